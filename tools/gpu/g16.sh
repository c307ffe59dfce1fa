cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
MPSG_TMA=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sell_real" -c 1 -f -o gpurun_out/g16_tma python tools/kbench.py --steps 1 --warmup 0 cfg2:4:2 > gpurun_out/g16_ncu.log 2>&1; echo ncu=$?
