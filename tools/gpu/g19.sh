cd $GRAFT_REPO_ROOT
S="cfg3:2:2 cfg3:2:1 cfg3:2:0"
timeout 300 python tools/kbench.py --tag base --steps 20 --check $S 2>&1 | grep -v "^#" | cut -c1-200
for v in cb10 cb12 cb16; do
MPSG_LIB=variants/$v.so timeout 300 python tools/kbench.py --tag $v --steps 20 --check $S 2>&1 | grep -v "^#" | cut -c1-200
done
