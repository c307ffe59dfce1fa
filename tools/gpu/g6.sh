cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SPECS="cfg2:4:2 cfg2:3:2 cfg5:4:2"
for v in default memonly a2s2w4 memonly_a; do
  if [ $v = default ]; then L=""; else L=variants/$v.so; fi
  MPSG_LIB=$L timeout 600 python tools/kbench.py --tag $v --steps 20 $SPECS >> gpurun_out/g6_kbench.log 2>&1
done
MPSG_LIB=variants/a2s2w4.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sell_fast_async" -c 1 -o gpurun_out/g6_async python tools/kbench.py --steps 1 --warmup 0 cfg2:4:2 > gpurun_out/g6_ncu.log 2>&1
MPSG_LIB=variants/memonly.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sell_real" -c 1 -o gpurun_out/g6_memonly python tools/kbench.py --steps 1 --warmup 0 cfg2:4:2 >> gpurun_out/g6_ncu.log 2>&1
echo done
