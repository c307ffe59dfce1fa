# r02b baseline pass of HEAD: GPU parity tests, smoke, default bench, reference arm, every config
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/g13_pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/g13_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g13_smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/g13_bench_default.log 2>&1; echo default=$?; tail -1 gpurun_out/g13_bench_default.log | cut -c1-400
timeout 600 python bench.py --impl reference > gpurun_out/g13_bench_ref.log 2>&1; echo ref=$?
timeout 2400 python bench.py --all --steps 10 > gpurun_out/g13_bench_all.log 2>&1; echo all=$?
