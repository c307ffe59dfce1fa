# r02i full pass: GPU parity tests, smoke, default bench, reference arm, every config, traffic, ncu
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r02i_pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/r02i_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02i_smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/r02i_bench_default.log 2>&1; echo default=$?; tail -1 gpurun_out/r02i_bench_default.log | cut -c1-300
timeout 600 python bench.py --impl reference > gpurun_out/r02i_bench_ref.log 2>&1; echo ref=$?
timeout 2400 python bench.py --all --steps 10 > gpurun_out/r02i_bench_all.log 2>&1; echo all=$?
timeout 2400 python tools/traffic.py gpurun_out/r02i_traffic.json > gpurun_out/r02i_traffic.log 2>&1; echo traffic=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02i_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02i_ncu_launch.log 2>&1; echo launch=$?
S="cfg2:4:2 cfg2:3:2 cfg3:2:2 cfg3:4:2 cfg4:2:2 cfg5:2:2 cfg5:4:2 cfg1:2:2"
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:^(sell|long|pad)_" -f -o gpurun_out/r02i_prof_all python tools/kbench.py --steps 1 --warmup 0 $S > gpurun_out/r02i_prof.log 2>&1; echo ncu=$?
