cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
./scripts/micro/cr16_bench > gpurun_out/cr16.log 2>&1
