cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
ACCFEM_PROF_SO=paper_2503_06922_b200/libaccfem_prof.so timeout 300 python scripts/phase_profile.py cfg4 1776 > gpurun_out/polish_prof.log 2>&1
for i in 1 2; do timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print(d['value'], d['load_balance'], d['latency']['cfg3p']['p50_ms'])
" >> gpurun_out/polish_prof.log; done
