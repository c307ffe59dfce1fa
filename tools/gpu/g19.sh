cd $GRAFT_REPO_ROOT
S="cfg2:4:2 cfg5:4:2"
timeout 300 python tools/kbench.py --tag base --steps 20 --check $S 2>&1 | grep -v "^#" | cut -c1-200
for v in th64 th32; do
MPSG_LIB=variants/$v.so timeout 300 python tools/kbench.py --tag $v --steps 20 --check $S 2>&1 | grep -v "^#" | cut -c1-200
done
