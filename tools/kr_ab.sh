cd $GRAFT_REPO_ROOT
for p1 in 10 40; do for K in 4 2; do
  echo "p1=$p1 $(python tools/kr_probe.py $K cg 64 2 $p1) | $(python tools/kr_probe.py $K bicgstab 32 2 $p1)"
done; done
