cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in "cfg3p 1" "cfg4 1"; do echo "== cr $c" >> gpurun_out/prof3.log; ACCFEM_MODE=cr ACCFEM_PROF_SO=paper_2503_06922_b200/libaccfem_prof.so timeout 300 python scripts/phase_profile.py $c >> gpurun_out/prof3.log 2>&1; done
echo "== team2 cfg4 1776" >> gpurun_out/prof3.log; ACCFEM_PROF_SO=paper_2503_06922_b200/libaccfem_prof.so timeout 300 python scripts/phase_profile.py cfg4 1776 >> gpurun_out/prof3.log 2>&1
echo "== cr cfg5 1" >> gpurun_out/prof3.log; ACCFEM_MODE=cr ACCFEM_PROF_SO=paper_2503_06922_b200/libaccfem_prof.so timeout 300 python scripts/phase_profile.py cfg5 1 >> gpurun_out/prof3.log 2>&1
