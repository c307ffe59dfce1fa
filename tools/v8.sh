cd $GRAFT_REPO_ROOT
S="cfg4:2:2 cfg5:2:1 cfg5:2:0 cfg1:2:1 cfg1:2:0 cfg3:2:1"
python tools/kbench.py --tag base $S 2>&1 | grep -v Warn
for v in minb12 minb16 ch4 ch4m12; do MPSG_LIB=$PWD/variants/$v.so python tools/kbench.py --tag $v $S 2>&1 | grep -v Warn; done
