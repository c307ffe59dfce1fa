cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python bench.py --no-cpu --secondary none --steps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('overlap', d['value'], d['e2e'])"
MPSG_OVERLAP=0 python bench.py --no-cpu --secondary none --steps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('no-overlap', d['value'], d['e2e'])"
