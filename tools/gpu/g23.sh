cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for K in 2 4; do for v in 1 2; do
timeout 600 python bench.py --config cfg5 --K $K --cg --cg-variant $v --no-cpu --steps 10 --warmup 3 2>&1 | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('K',$K,'variant',$v, round(d['value'],1),'Gnnz/s', round(d['ms_per_iteration'],4),'ms/iter', d['config'].get('cg_form'), d['config']['iterations'], d['config']['rel_residual'], d['roofline']['frac'])"
done; done
