# warp-specialised FAST short-row kernel: correctness (bound tests) and A/B timing
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S="cfg2:4:2 cfg2:3:2 cfg5:4:2 cfg5:3:2"
MPSG_WS=0 timeout 300 python tools/kbench.py --tag plain --steps 20 $S > gpurun_out/g14_kbench_plain.log 2>&1; echo plain=$?
timeout 300 python tools/kbench.py --tag ws --steps 20 $S > gpurun_out/g14_kbench_ws.log 2>&1; echo ws=$?
cat gpurun_out/g14_kbench_plain.log gpurun_out/g14_kbench_ws.log | grep -v "^#" | cut -c1-200
timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_fast_accuracy.py -q -m gpu -x > gpurun_out/g14_pytest.log 2>&1; echo pytest=$?
tail -5 gpurun_out/g14_pytest.log
