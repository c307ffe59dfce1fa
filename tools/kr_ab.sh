cd $GRAFT_REPO_ROOT
for occ in 0 2 4 6 8 12; do
  echo "occ=$occ $(MPSG_KR_OCC=$occ python tools/kr_probe.py 4 bicgstab 32) | $(MPSG_KR_OCC=$occ python tools/kr_probe.py 4 cg 64) | $(MPSG_KR_OCC=$occ python tools/kr_probe.py 2 bicgstab 32)"
done
python tools/kbench.py cfg1:2:2 cfg5:2:2 cfg4:2:2 cfg1:2:1
for v in minb14 minb16; do MPSG_LIB=$PWD/variants/$v.so python tools/kbench.py --tag $v cfg1:2:2 cfg5:2:2 cfg4:2:2 cfg1:2:1; done
