cd $GRAFT_REPO_ROOT
S="cfg2:4:2 cfg2:3:2 cfg5:4:2 cfg3:4:2"
python tools/kbench.py --tag base $S 2>&1 | grep -v Warn
for v in g2 pf4 pf2 m8 g2m8 pf2m8; do MPSG_LIB=$PWD/variants/$v.so python tools/kbench.py --tag $v $S 2>&1 | grep -v Warn; done
