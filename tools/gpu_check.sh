set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_cg.py -x -q -m gpu 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; tail -3 gpurun_out/bench_default.log
timeout 900 python bench.py --all --steps 10 --no-e2e > gpurun_out/bench_all.log 2>&1; tail -12 gpurun_out/bench_all.log
