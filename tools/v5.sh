cd $GRAFT_REPO_ROOT
S="cfg4:2:2 cfg5:2:1 cfg1:2:1 cfg3:2:1"
python tools/kbench.py --tag base $S 2>&1 | grep -v Warn
for v in small8 longu2 par1dd par4dd; do MPSG_LIB=$PWD/variants/$v.so python tools/kbench.py --tag $v $S 2>&1 | grep -v Warn; done
A="python tools/kbench.py --steps 2 cfg5:2:1"
$A > gpurun_out/plainA.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sell_real -s 3 -c 1 -o gpurun_out/prof_cfg5_dd $A > gpurun_out/ncuA.log 2>&1; echo ncu=$?
