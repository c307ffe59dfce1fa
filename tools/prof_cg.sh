# ncu of the config-5 CG iteration kernels (QD and DD), after plain runs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/cg_probe.py 4 64 > gpurun_out/cg_plain.log 2>&1 && python tools/cg_probe.py 2 64 >> gpurun_out/cg_plain.log 2>&1
cat gpurun_out/cg_plain.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cg_launches.csv python tools/cg_probe.py 4 8 > /dev/null 2>&1
echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cg_|sell_" -s 12 -c 6 -o gpurun_out/cg_qd python tools/cg_probe.py 4 8 > gpurun_out/cg_ncu.log 2>&1
echo full=$?
