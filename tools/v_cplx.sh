cd $GRAFT_REPO_ROOT
S="cfg3:2:2 cfg3:2:0 cfg3:4:2"
python tools/kbench.py --check $S
MPSG_LIB=$PWD/variants/cplxg2.so python tools/kbench.py --check --tag g2 $S
