cd $GRAFT_REPO_ROOT
C="python tools/kbench.py --steps 1 --warmup 0 cfg4:2:1 cfg4:2:0"
$C > gpurun_out/p23_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none -k regex:"sell_|long_" -o gpurun_out/prof_cfg4_det $C > gpurun_out/p23_ncu.log 2>&1; echo ncu=$?
cat gpurun_out/p23_plain.log | grep -v Warn
