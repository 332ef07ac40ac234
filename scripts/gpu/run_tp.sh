cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in 1 2; do timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print(d['value'], d['ms_per_step'], d['load_balance'])
" >> gpurun_out/tp.log; done
