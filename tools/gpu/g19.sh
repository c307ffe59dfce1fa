cd $GRAFT_REPO_ROOT
S="cfg2:4:2 cfg5:4:2"
for v in b9g4 b9g3 b9g2; do
MPSG_LIB=variants/$v.so timeout 300 python tools/kbench.py --tag $v --steps 20 $S 2>&1 | grep -v "^#" | cut -c1-200
done
MPSG_TMA=1 MPSG_LIB=variants/tmag4.so timeout 300 python tools/kbench.py --tag tmag4 --steps 20 $S 2>&1 | grep -v "^#" | cut -c1-200
