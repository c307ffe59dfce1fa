cd $GRAFT_REPO_ROOT
for g in 0 1; do echo "grid=$g: $(MPSG_CG_GRID=$g python tools/cg_probe.py 4 128) | $(MPSG_CG_GRID=$g python tools/cg_probe.py 2 128)"; done
timeout 900 python -m pytest tests/test_gpu_cg.py tests/test_gpu_dist.py -x -q -m gpu 2>&1 | tail -2
