cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
./scripts/micro/cr16_bench > gpurun_out/cr16_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bench -c 1 -o gpurun_out/cr16 ./scripts/micro/cr16_bench > gpurun_out/cr16_ncu.log 2>&1
