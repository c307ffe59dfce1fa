cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SPECS="cfg2:4:2 cfg2:3:2 cfg5:4:2 cfg5:3:2 cfg3:4:2"
for v in default a4s2w4 a2s3w4 a2s2w4 a1s4w4 a2s3ca default; do
  if [ $v = default ]; then L=""; else L=variants/$v.so; fi
  MPSG_LIB=$L timeout 600 python tools/kbench.py --tag $v --steps 20 --check $SPECS >> gpurun_out/g4_kbench.log 2>&1
done
echo done
