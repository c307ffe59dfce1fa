cd $GRAFT_REPO_ROOT
for g in 0 1 2 4; do for f in 0 1; do echo "grid=$g fuse=$f: $(MPSG_CG_GRID=$g MPSG_CG_FUSE=$f python tools/cg_probe.py 4 128) | $(MPSG_CG_GRID=$g MPSG_CG_FUSE=$f python tools/cg_probe.py 2 128)"; done; done
