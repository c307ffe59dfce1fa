cd $GRAFT_REPO_ROOT
python tools/fused_adversarial.py
python tools/fused_probe.py
python tools/kbench.py cfg2:4:2 cfg2:3:2 cfg5:4:2 cfg3:4:2 cfg3:2:2 cfg4:2:2 cfg5:2:2
python tools/cg_probe.py 4 128; python tools/kr_probe.py 4 bicgstab 32
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
