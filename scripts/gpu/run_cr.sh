cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for m in cr team4; do ACCFEM_MODE=$m timeout 300 python scripts/latency_probe.py cfg3p cfg4_s0 cfg1 cfg4_148 >> gpurun_out/lat.log 2>&1; done
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "every_kernel_mode or static_solves or status" > gpurun_out/pytest_cr.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_cr.log
