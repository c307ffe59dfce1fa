cd $GRAFT_REPO_ROOT
C="python tools/kbench.py --steps 1 --warmup 0 cfg4:2:2"
$C > gpurun_out/p16_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none -k regex:"sell_|long_" -o gpurun_out/prof_cfg4_cb $C > gpurun_out/p16_ncu.log 2>&1; echo ncu=$?
MPSG_COLBLOCK_BYTES=0 $C > gpurun_out/p16_plain.log 2>&1 && MPSG_COLBLOCK_BYTES=0 timeout 900 ncu --set full --clock-control none -k regex:"sell_|long_" -o gpurun_out/prof_cfg4_nocb $C > gpurun_out/p16_ncu2.log 2>&1; echo ncu=$?
