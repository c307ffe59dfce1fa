cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/g11_bench_default.log 2>&1; echo default=$?
timeout 2400 python bench.py --all --steps 10 > gpurun_out/g11_bench_all.log 2>&1; echo all=$?
timeout 2400 python tools/traffic.py gpurun_out/g11_traffic.json > gpurun_out/g11_traffic.log 2>&1; echo traffic=$?
