cd $GRAFT_REPO_ROOT
echo "base: $(python tools/cg_probe.py 4 128) | $(python tools/cg_probe.py 2 128)"
for v in t128 t128m8 t256m4 t64; do echo "$v: $(MPSG_LIB=$PWD/variants/$v.so python tools/cg_probe.py 4 128) | $(MPSG_LIB=$PWD/variants/$v.so python tools/cg_probe.py 2 128)"; done
