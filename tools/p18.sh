cd $GRAFT_REPO_ROOT
python tools/cg_probe.py 4 64 && python tools/cg_probe.py 2 64 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cg_launches_qd.csv python tools/cg_probe.py 4 64 > /dev/null 2>&1; echo ncu=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cg_launches_dd.csv python tools/cg_probe.py 2 64 > /dev/null 2>&1; echo ncu=$?
