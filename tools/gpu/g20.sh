cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S="cfg2:4:2 cfg2:3:2 cfg5:4:2 cfg5:3:2 cfg3:4:2 cfg3:2:2 cfg4:2:2 cfg1:2:2 cfg3:4:2:mixed cfg2:4:2:sptmv"
timeout 600 python tools/kbench.py --tag r02c --steps 20 $S 2>&1 | grep -v "^#" | cut -c1-200
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/g20_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/g20_pytest.log
