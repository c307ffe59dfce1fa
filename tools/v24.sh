cd $GRAFT_REPO_ROOT
S="cfg1:2:2 cfg5:2:2 cfg4:2:2 cfg5:2:0"
python tools/kbench.py --tag small8 $S 2>&1 | grep -v Warn
for v in nosmall small6; do MPSG_LIB=$PWD/variants/$v.so python tools/kbench.py --tag $v $S 2>&1 | grep -v Warn; done
timeout 900 python -m pytest tests/test_gpu_spmv.py -x -q -m gpu 2>&1 | tail -1
