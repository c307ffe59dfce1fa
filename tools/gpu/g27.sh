cd $GRAFT_REPO_ROOT
echo -n "base   "; python tools/cg_probe.py 4 256
for v in dm3 dm4 t128m6 t128m8 t128; do
echo -n "$v   "; MPSG_LIB=variants/$v.so python tools/cg_probe.py 4 256
done
echo -n "base   "; python tools/cg_probe.py 4 256
