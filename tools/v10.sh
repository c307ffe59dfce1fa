cd $GRAFT_REPO_ROOT
timeout 900 ./oracle/_ref/dropin_test > gpurun_out/dropin.log 2>&1; echo dropin rc=$?; grep -c PASS gpurun_out/dropin.log; grep FAIL gpurun_out/dropin.log | head
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
