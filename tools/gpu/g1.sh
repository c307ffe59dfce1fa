cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,compute_mode,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt 2>&1
timeout 1500 python -m pytest -q -x tests/test_gpu_arith.py tests/test_gpu_fast_full.py tests/test_gpu_fast_accuracy.py "tests/test_gpu_cg.py::test_cg_full_config5_500_iterations" "tests/test_gpu_dist.py::test_failing_rank_fails_every_rank_without_hanging" -s > gpurun_out/g1_pytest.log 2>&1; echo pytest=$? 
SPECS="cfg2:4:2 cfg2:3:2 cfg5:4:2 cfg5:2:2 cfg4:2:2 cfg1:2:2 cfg2:4:0 cfg5:2:0"
for v in default pf1 pf2 pf4 default pf2; do
  if [ $v = default ]; then L=""; else L=variants/$v.so; fi
  MPSG_LIB=$L timeout 600 python tools/kbench.py --tag $v --steps 20 $SPECS >> gpurun_out/g1_kbench.log 2>&1
done
echo done
