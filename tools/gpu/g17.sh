cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S="cfg2:3:2 cfg5:3:2 cfg2:3:2:mixed"
MPSG_TD_PAD=0 timeout 300 python tools/kbench.py --tag nopad --steps 20 $S 2>&1 | grep -v "^#" | cut -c1-200
timeout 300 python tools/kbench.py --tag pad --steps 20 $S 2>&1 | grep -v "^#" | cut -c1-200
timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_fast_accuracy.py tests/test_gpu_mixed_sptmv.py -q -m gpu -x > gpurun_out/g17_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/g17_pytest.log
