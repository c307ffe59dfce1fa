# ncu --set full of every config's SpMV kernels (one launch each, cold L2), after a plain run
cd $GRAFT_REPO_ROOT
S="cfg2:4:2 cfg2:3:2 cfg3:2:2 cfg3:4:2 cfg4:2:2 cfg5:2:2 cfg5:4:2 cfg1:2:2"
C="python tools/kbench.py --steps 1 --warmup 0 $S"
$C > gpurun_out/prof_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"sell_|long_" -o gpurun_out/prof_all $C > gpurun_out/prof_ncu.log 2>&1
echo ncu=$?
B="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e"
$B > gpurun_out/plainB.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
echo launch=$?
