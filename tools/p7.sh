cd $GRAFT_REPO_ROOT
export MPSG_LIB=$PWD/variants/ch0.so
A="python tools/kbench.py --steps 1 cfg5:2:1 cfg5:2:0"
$A > gpurun_out/plainA.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sell_real -s 3 -c 5 -o gpurun_out/prof_cfg5_orders $A > gpurun_out/ncuA.log 2>&1; echo ncu=$?
