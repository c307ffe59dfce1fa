cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SPECS="cfg2:4:2 cfg2:3:2 cfg5:4:2 cfg5:3:2 cfg2:3:0 cfg2:3:1 cfg2:4:0 cfg2:4:1"
timeout 300 python tools/kbench.py --tag new --steps 20 --check $SPECS > gpurun_out/g10_kbench.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/g10_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/g10_pytest.log
