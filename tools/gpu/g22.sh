cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_cg.py tests/test_gpu_dist.py -q -m gpu -x > gpurun_out/g22_pytest.log 2>&1; echo pytest=$?
tail -30 gpurun_out/g22_pytest.log
