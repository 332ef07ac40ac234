cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
ACCFEM_MODE=cr timeout 600 python scripts/latency_probe.py cfg3p cfg4_s0 cfg5 > gpurun_out/cr2.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/cr2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/cr2_pytest.log
