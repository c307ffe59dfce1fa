# One GPU pass: parity tests, smoke, default bench, reference arm, all-config bench,
# then the ncu launch list of the default bench and a full capture of its top kernel.
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; tail -1 gpurun_out/bench_default.log | cut -c1-300
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-200
timeout 1800 python bench.py --all --steps 10 --no-e2e > gpurun_out/bench_all.log 2>&1; tail -2 gpurun_out/bench_all.log | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --secondary none > gpurun_out/ncu_launch.log 2>&1; echo launch=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sell_real" -c 1 -o gpurun_out/top_kernel \
  python tools/kbench.py --steps 1 --warmup 0 cfg2:4:2 > gpurun_out/ncu_top.log 2>&1; echo top=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cg_|kr_" -s 40 -c 12 -o gpurun_out/solver_kernels \
  python tools/kr_probe.py 4 bicgstab 4 > gpurun_out/ncu_solver.log 2>&1; echo solver=$?
