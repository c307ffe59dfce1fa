cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MPSG_TMA=1
S="cfg2:4:2 cfg2:3:2 cfg5:4:2 cfg5:3:2 cfg2:4:2:mixed"
timeout 300 python tools/kbench.py --tag tg2s2 --steps 20 $S 2>&1 | grep -v "^#" | cut -c1-200
for v in tc50 tg1s4 tg2s3 tg2s2b7; do
MPSG_LIB=variants/$v.so timeout 300 python tools/kbench.py --tag $v --steps 20 $S 2>&1 | grep -v "^#" | cut -c1-200
done
timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_fast_accuracy.py tests/test_gpu_mixed_sptmv.py -q -m gpu -x > gpurun_out/g21_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/g21_pytest.log
