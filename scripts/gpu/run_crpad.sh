cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
./scripts/micro/crpad_bench > gpurun_out/crpad.log 2>&1
