cd $GRAFT_REPO_ROOT
S="cfg2:4:2 cfg2:3:2 cfg5:4:2 cfg3:4:2 cfg3:2:2 cfg2:4:1 cfg2:3:1 cfg3:4:1"
python tools/kbench.py --tag pf2 $S 2>&1 | grep -v Warn
for v in g1 g3; do MPSG_LIB=$PWD/variants/$v.so python tools/kbench.py --tag $v cfg2:4:2 cfg2:3:2 cfg5:4:2 2>&1 | grep -v Warn; done
timeout 900 python -m pytest tests/test_gpu_spmv.py -x -q -m gpu 2>&1 | tail -2
