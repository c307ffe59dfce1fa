cd $GRAFT_REPO_ROOT
S="cfg4:2:2"
timeout 300 python tools/kbench.py --tag lu4 --steps 20 $S 2>&1 | grep -v "^#" | cut -c1-200
for v in lu1 lu2 lu8; do
MPSG_LIB=variants/$v.so timeout 300 python tools/kbench.py --tag $v --steps 20 $S 2>&1 | grep -v "^#" | cut -c1-200
done
timeout 600 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_fast_accuracy.py -q -m gpu -x 2>&1 | tail -2
