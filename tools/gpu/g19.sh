cd $GRAFT_REPO_ROOT
S="cfg2:3:2 cfg5:3:2 cfg2:3:2:mixed"
for v in t37 t47 t36 t26 t46; do
MPSG_LIB=variants/$v.so timeout 300 python tools/kbench.py --tag $v --steps 20 $S 2>&1 | grep -v "^#" | cut -c1-200
done
