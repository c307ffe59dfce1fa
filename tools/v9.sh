cd $GRAFT_REPO_ROOT
S="cfg2:4:2 cfg2:3:2 cfg3:4:2 cfg3:2:2 cfg4:2:2 cfg5:2:2 cfg5:4:2 cfg1:2:2 cfg5:2:1 cfg3:2:1 cfg3:4:1"
python tools/kbench.py --tag base $S 2>&1 | grep -v Warn
MPSG_LIB=$PWD/variants/cl4.so python tools/kbench.py --tag cl4 cfg3:4:2 cfg3:2:2 2>&1 | grep -v Warn
timeout 900 python -m pytest tests/test_gpu_spmv.py -x -q -m gpu 2>&1 | tail -3
