cd $GRAFT_REPO_ROOT
for i in 1 2 3; do
for lib in "" variants/before.so; do
echo -n "lib=$lib  "; MPSG_LIB=$lib python tools/cg_probe.py 4 256
done; done
