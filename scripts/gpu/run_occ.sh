cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for pad in 0 6000 16000; do echo "pad $pad" >> gpurun_out/occ.log; ACCFEM_SMEM_PAD=$pad timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print(d['value'], d['roofline']['kernel'], d['load_balance'])
" >> gpurun_out/occ.log; done
