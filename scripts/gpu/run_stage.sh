cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
./scripts/micro/stage_bench > gpurun_out/stage.log 2>&1
