cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SPECS="cfg2:4:2 cfg5:4:2 cfg2:3:2"
for v in default two2m8 two1m8 two2m6 two1m10 t2s3 default; do
  if [ $v = default ]; then L=""; else L=variants/$v.so; fi
  MPSG_LIB=$L timeout 300 python tools/kbench.py --tag $v --steps 20 --check $SPECS >> gpurun_out/g9_kbench.log 2>&1
done
echo done
