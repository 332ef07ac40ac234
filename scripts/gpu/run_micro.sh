cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
#./scripts/micro/nd_bench > gpurun_out/nd.log 2>&1
./scripts/micro/chain1_bench > gpurun_out/chain1.log 2>&1
