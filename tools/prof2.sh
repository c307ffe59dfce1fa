cd $GRAFT_REPO_ROOT
A="python tools/kbench.py --steps 2 cfg2:4:1"
B="python tools/kbench.py --steps 2 cfg4:2:2"
$A > gpurun_out/plainA.log 2>&1 && $B > gpurun_out/plainB.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sell_real -s 3 -c 1 -o gpurun_out/prof_qd_sell $A > gpurun_out/ncuA.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sell_real|long_fast" -s 6 -c 2 -o gpurun_out/prof_cfg4_dd $B > gpurun_out/ncuB.log 2>&1
echo rc=$?
cat gpurun_out/plainA.log gpurun_out/plainB.log | grep -v Warn
