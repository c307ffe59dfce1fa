cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MPSG_WS=1
S="cfg2:4:2 cfg2:3:2 cfg5:4:2 cfg5:3:2"
timeout 300 python tools/kbench.py --tag p4 --steps 10 $S 2>&1 | grep -v "^#" | cut -c1-200
for v in p4b5 p2b5 p2b6; do
MPSG_LIB=variants/$v.so timeout 300 python tools/kbench.py --tag $v --steps 10 $S 2>&1 | grep -v "^#" | cut -c1-200
done
timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_fast_accuracy.py -q -m gpu -x > gpurun_out/g15_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/g15_pytest.log
