cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for m in cr team4; do ACCFEM_MODE=$m timeout 600 python scripts/latency_probe.py cfg5 >> gpurun_out/cfg5.log 2>&1; done
ACCFEM_PROF_SO=paper_2503_06922_b200/libaccfem_prof.so ACCFEM_MODE=cr timeout 300 python scripts/phase_profile.py cfg5 1 >> gpurun_out/cfg5.log 2>&1
ACCFEM_PROF_SO=paper_2503_06922_b200/libaccfem_prof.so ACCFEM_MODE=team4 timeout 300 python scripts/phase_profile.py cfg5 1 >> gpurun_out/cfg5.log 2>&1
