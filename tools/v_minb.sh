cd $GRAFT_REPO_ROOT
python tools/kbench.py cfg1:2:2 cfg5:2:2 cfg4:2:2 cfg1:2:1
for v in minb14 minb16; do MPSG_LIB=$PWD/variants/$v.so python tools/kbench.py --tag $v cfg1:2:2 cfg5:2:2 cfg4:2:2 cfg1:2:1; done
