cd $GRAFT_REPO_ROOT
S="cfg2:4:2 cfg2:3:2 cfg5:4:2 cfg5:4:1 cfg3:4:2 cfg2:4:1"
python tools/kbench.py --tag early $S 2>&1 | grep -v Warn
timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_cg.py -x -q -m gpu 2>&1 | tail -2
