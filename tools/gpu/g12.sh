cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python tools/traffic.py gpurun_out/g12_traffic.json > gpurun_out/g12_traffic.log 2>&1; echo traffic=$?
S="cfg2:4:2 cfg2:3:2 cfg3:2:2 cfg3:4:2 cfg4:2:2 cfg5:2:2 cfg5:4:2 cfg1:2:2"
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:^(sell|long)_" -o gpurun_out/g12_prof_all python tools/kbench.py --steps 1 --warmup 0 $S > gpurun_out/g12_prof.log 2>&1
echo ncu=$?
