cd $GRAFT_REPO_ROOT
python tools/kbench.py --tag base cfg4:2:2 2>&1 | grep -v Warn
for v in u4 m12 u4m12 u1 m16; do MPSG_LIB=$PWD/variants/$v.so python tools/kbench.py --tag $v cfg4:2:2 2>&1 | grep -v Warn; done
