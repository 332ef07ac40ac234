cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/p4_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/p4_pytest.log
echo "== cr cfg5 1" >> gpurun_out/p4_prof.log; ACCFEM_MODE=cr ACCFEM_PROF_SO=paper_2503_06922_b200/libaccfem_prof.so timeout 300 python scripts/phase_profile.py cfg5 1 >> gpurun_out/p4_prof.log 2>&1
echo "== team2 cfg4 1776" >> gpurun_out/p4_prof.log; ACCFEM_PROF_SO=paper_2503_06922_b200/libaccfem_prof.so timeout 300 python scripts/phase_profile.py cfg4 1776 >> gpurun_out/p4_prof.log 2>&1
echo "== team2 cfg5 1184" >> gpurun_out/p4_prof.log; ACCFEM_PROF_SO=paper_2503_06922_b200/libaccfem_prof.so timeout 300 python scripts/phase_profile.py cfg5 1184 >> gpurun_out/p4_prof.log 2>&1
timeout 600 python scripts/latency_probe.py cfg3p cfg5 cfg5_296 cfg5_1184 > gpurun_out/p4_lat.log 2>&1
