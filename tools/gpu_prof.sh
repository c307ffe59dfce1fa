# bench + launch list + one full ncu capture of the top kernel (cfg2 QD)
cd $GRAFT_REPO_ROOT
B="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --secondary none"
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; tail -1 gpurun_out/bench_default.log
timeout 900 python bench.py --all --steps 10 --no-e2e > gpurun_out/bench_all.log 2>&1; cut -c1-400 gpurun_out/bench_all.log | grep -o '"value": [0-9.]*\|"workload": "[^"]*"\|"frac": [0-9.]*'
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sell_real -s 2 -c 1 -o gpurun_out/prof_cfg2_qd $B > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/ncu_full.log
