cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for m in team4 team2; do ACCFEM_MODE=$m timeout 900 python scripts/latency_probe.py cfg5_1184 >> gpurun_out/cfg5tp2.log 2>&1; done
