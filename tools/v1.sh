cd $GRAFT_REPO_ROOT
S="cfg2:4:1 cfg2:3:1 cfg5:4:1 cfg3:4:1 cfg3:2:1 cfg4:2:1 cfg5:2:1 cfg1:2:1"
python tools/kbench.py --tag base $S 2>&1 | grep -v Warn
MPSG_LIB=$PWD/variants/minb6.so python tools/kbench.py --tag minb6 cfg2:4:1 cfg2:3:1 cfg5:4:1 2>&1 | grep -v Warn
MPSG_LIB=$PWD/variants/minb8.so python tools/kbench.py --tag minb8 cfg2:4:1 cfg2:3:1 cfg5:4:1 2>&1 | grep -v Warn
