cd $GRAFT_REPO_ROOT
S="cfg2:4:2 cfg2:3:2 cfg5:4:2 cfg3:4:2"
python tools/kbench.py $S
for v in pf1 pf2; do MPSG_LIB=$PWD/variants/$v.so python tools/kbench.py --tag $v $S; done
