cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
ACCFEM_MODE=cr timeout 300 python scripts/latency_probe.py cfg3p cfg4_s0 > gpurun_out/quick.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_quick.log 2>&1
python -c "
import sys; sys.path.insert(0,'.')
from paper_2503_06922_b200 import scenarios
from paper_2503_06922_b200.engine import Engine
e = Engine(**scenarios.cfg4(1).engine_kwargs(), device=0)
print('teams resident', e._lib.accfem_teams_resident(e._h), 'ws bytes', e._lib.accfem_workspace_bytes(e._h))
" >> gpurun_out/quick.log 2>&1
