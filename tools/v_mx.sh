cd $GRAFT_REPO_ROOT
python tools/x_locality_probe.py mixed 1
for v in mxu2 mxu4; do MPSG_LIB=$PWD/variants/$v.so python tools/x_locality_probe.py mixed 1; done
