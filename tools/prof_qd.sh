cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/kbench.py --steps 3 --warmup 1 cfg2:4:2 > gpurun_out/qd_plain.log 2>&1 && cat gpurun_out/qd_plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sell_real" -c 1 -o gpurun_out/qd_sell python tools/kbench.py --steps 1 --warmup 0 cfg2:4:2 > gpurun_out/qd_ncu.log 2>&1
echo ncu=$?
