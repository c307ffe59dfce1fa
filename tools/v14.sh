cd $GRAFT_REPO_ROOT
S="cfg4:2:2 cfg2:4:2 cfg2:3:2 cfg3:2:2 cfg5:2:2 cfg1:2:2 cfg4:2:1"
python tools/kbench.py --tag base $S 2>&1 | grep -v Warn
for v in xh ah xah; do MPSG_LIB=$PWD/variants/$v.so python tools/kbench.py --tag $v $S 2>&1 | grep -v Warn; done
