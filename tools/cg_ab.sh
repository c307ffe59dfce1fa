cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_krylov.py tests/test_gpu_cg.py tests/test_gpu_dist.py -q -m gpu 2>&1 | tail -3
for K in 4 2; do
  echo "$(python tools/cg_probe.py $K 128)"
  echo "$(python tools/kr_probe.py $K cg 64) | $(python tools/kr_probe.py $K bicgstab 32) | $(python tools/kr_probe.py $K gpbicg 32)"
  echo "tiny: $(python tools/kr_probe.py $K cg 64 2 10) | $(python tools/kr_probe.py $K bicgstab 32 2 10)"
done
