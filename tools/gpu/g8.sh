cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SPECS="cfg2:4:2 cfg5:4:2"
for v in default t2s3 t2s2 t4s2 t1s4 t2s4 default; do
  if [ $v = default ]; then L=""; else L=variants/$v.so; fi
  MPSG_LIB=$L timeout 300 python tools/kbench.py --tag $v --steps 20 --check $SPECS >> gpurun_out/g8_kbench.log 2>&1
done
MPSG_LIB=variants/t2s2.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sell_fast_tma" -c 1 -o gpurun_out/g8_tma python tools/kbench.py --steps 1 --warmup 0 cfg2:4:2 > gpurun_out/g8_ncu.log 2>&1
echo done
