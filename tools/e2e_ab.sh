cd $GRAFT_REPO_ROOT
for K in 4 3; do python tools/e2e_probe.py $K; MPSG_PARTS=8 python tools/e2e_probe.py $K; MPSG_PARTS=3 python tools/e2e_probe.py $K; done
