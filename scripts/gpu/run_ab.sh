cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in A B A B; do echo "variant $v" >> gpurun_out/ab.log; ACCFEM_LIB=paper_2503_06922_b200/libaccfem_$v.so timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print(d['value'], d['ms_per_step'], d['load_balance']['tail_frac'])
" >> gpurun_out/ab.log; done
