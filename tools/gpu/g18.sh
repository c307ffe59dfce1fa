cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S="cfg2:4:2 cfg2:3:2 cfg5:4:2 cfg5:3:2 cfg2:4:2:mixed cfg2:3:2:mixed"
MPSG_LIB=variants/nolvl.so timeout 300 python tools/kbench.py --tag nolvl --steps 20 $S 2>&1 | grep -v "^#" | cut -c1-200
timeout 300 python tools/kbench.py --tag lvl --steps 20 $S 2>&1 | grep -v "^#" | cut -c1-200
timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_fast_accuracy.py tests/test_gpu_mixed_sptmv.py -q -m gpu -x > gpurun_out/g18_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/g18_pytest.log
