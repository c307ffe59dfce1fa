cd $GRAFT_REPO_ROOT
python tools/kbench.py --tag cb16m4096 cfg4:2:2 2>&1 | grep -v Warn
MPSG_COLBLOCK_BYTES=0 python tools/kbench.py --tag cb_off cfg4:2:2 2>&1 | grep -v Warn
MPSG_COLBLOCK_BYTES=8388608 python tools/kbench.py --tag cb8 cfg4:2:2 2>&1 | grep -v Warn
MPSG_COLBLOCK_BYTES=33554432 python tools/kbench.py --tag cb32 cfg4:2:2 2>&1 | grep -v Warn
MPSG_COLBLOCK_MIN=1024 python tools/kbench.py --tag cb16m1024 cfg4:2:2 2>&1 | grep -v Warn
MPSG_COLBLOCK_MIN=16384 python tools/kbench.py --tag cb16m16k cfg4:2:2 2>&1 | grep -v Warn
MPSG_COLBLOCK_BYTES=4194304 MPSG_COLBLOCK_MIN=2048 python tools/kbench.py --tag cb4m2048 cfg4:2:2 2>&1 | grep -v Warn
timeout 900 python -m pytest tests/test_gpu_spmv.py -x -q -m gpu -k "fast" 2>&1 | tail -2
