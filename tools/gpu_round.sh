# One GPU pass: parity tests, smoke, default bench, all-config bench, launch list, one ncu capture.
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
nproc > gpurun_out/host.txt; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket" >> gpurun_out/host.txt
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; tail -3 gpurun_out/bench_default.log
timeout 900 python bench.py --all --steps 10 --no-e2e > gpurun_out/bench_all.log 2>&1; tail -12 gpurun_out/bench_all.log
B="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --secondary none"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sell_real -s 2 -c 1 -o gpurun_out/prof_cfg2_qd $B > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/ncu_full.log
