cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SPECS="cfg2:4:2 cfg5:4:2 cfg3:4:2 cfg2:4:0 cfg2:4:1"
for v in default ld256 default ld256; do
  if [ $v = default ]; then L=""; else L=variants/$v.so; fi
  MPSG_LIB=$L timeout 600 python tools/kbench.py --tag $v --steps 20 --check $SPECS >> gpurun_out/g3_kbench.log 2>&1
done
MPSG_LIB=variants/ld256.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sell_real" -c 1 -o gpurun_out/g3_ld256 python tools/kbench.py --steps 1 --warmup 0 cfg2:4:2 > gpurun_out/g3_ncu.log 2>&1
echo done
