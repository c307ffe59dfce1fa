cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SPECS="cfg2:4:2 cfg5:4:2"
for v in default a2s2n2 a2s2n1 a4s2n2 a2s3n2 a4s2n4 a1s3n1 default; do
  if [ $v = default ]; then L=""; else L=variants/$v.so; fi
  MPSG_LIB=$L timeout 600 python tools/kbench.py --tag $v --steps 20 --check $SPECS >> gpurun_out/g7_kbench.log 2>&1
done
echo done
