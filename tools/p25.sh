cd $GRAFT_REPO_ROOT
C="python tools/cg_probe.py 4 2"
$C > gpurun_out/p25_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cg_|sell_" -o gpurun_out/prof_cg_qd $C > gpurun_out/p25_ncu.log 2>&1; echo ncu=$?
