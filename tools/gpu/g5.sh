cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SPECS="cfg2:4:2 cfg2:3:2 cfg5:4:2 cfg5:3:2"
for v in default g1m10 g1m12 g2m10 g4m10 g2m12 g4m9 default; do
  if [ $v = default ]; then L=""; else L=variants/$v.so; fi
  MPSG_LIB=$L timeout 600 python tools/kbench.py --tag $v --steps 20 --check $SPECS >> gpurun_out/g5_kbench.log 2>&1
done
echo done
