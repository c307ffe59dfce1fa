cd $GRAFT_REPO_ROOT
S="cfg2:4:2 cfg5:4:2 cfg2:4:1 cfg2:4:0 cfg5:4:1"
MPSG_LIB=variants/aos.so timeout 300 python tools/kbench.py --tag aos --steps 20 --check $S 2>&1 | grep -v "^#" | cut -c1-200
timeout 300 python tools/kbench.py --tag base --steps 20 --check $S 2>&1 | grep -v "^#" | cut -c1-200
