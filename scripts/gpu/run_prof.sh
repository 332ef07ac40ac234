cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for m in cr team4; do for c in "cfg3p 1" "cfg4 1"; do echo "== mode $m $c" >> gpurun_out/prof.log; ACCFEM_MODE=$m ACCFEM_PROF_SO=paper_2503_06922_b200/libaccfem_prof.so timeout 300 python scripts/phase_profile.py $c >> gpurun_out/prof.log 2>&1; done; done
