cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python scripts/contact_scaling.py > gpurun_out/contact_scaling.json 2> gpurun_out/contact_scaling.err
ACCFEM_MODE=cr timeout 300 python scripts/latency_probe.py cfg3p cfg4_s0 > gpurun_out/quick.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_quick.log 2>&1
