cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SPECS="cfg2:4:2 cfg2:3:2 cfg5:4:2 cfg5:3:2"
for v in default p4_4 p2_6 p4_5 p3_5 p2_5 default; do
  if [ $v = default ]; then L=""; else L=variants/$v.so; fi
  MPSG_LIB=$L timeout 600 python tools/kbench.py --tag $v --steps 20 --check $SPECS >> gpurun_out/g2_kbench.log 2>&1
done
echo done
