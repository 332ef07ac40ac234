cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in c400_5 c400_50; do echo "== cr $c" >> gpurun_out/c400.log; ACCFEM_MODE=cr ACCFEM_PROF_SO=paper_2503_06922_b200/libaccfem_prof.so timeout 300 python scripts/phase_profile.py $c 1 >> gpurun_out/c400.log 2>&1; done
