cd $GRAFT_REPO_ROOT
S="cfg5:2:2 cfg5:2:0 cfg4:2:2 cfg4:2:0 cfg1:2:2"
MPSG_PERSIST=0 python tools/kbench.py --check --tag off $S
python tools/kbench.py --check --tag on $S
MPSG_PERSIST=0 python tools/cg_probe.py 2 128
python tools/cg_probe.py 2 128
