cd $GRAFT_REPO_ROOT
S="cfg2:4:1 cfg2:3:1 cfg3:4:1 cfg3:2:1 cfg4:2:2 cfg4:2:1 cfg5:2:1 cfg5:2:0 cfg5:4:1 cfg1:2:1 cfg1:2:0"
python tools/kbench.py --tag v4 $S 2>&1 | grep -v Warn
timeout 900 python -m pytest tests/test_gpu_spmv.py -x -q -m gpu 2>&1 | tail -3
