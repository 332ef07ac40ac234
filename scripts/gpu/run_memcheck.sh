cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python scripts/sanitize_probe.py > gpurun_out/sanitize_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 50 python scripts/sanitize_probe.py > gpurun_out/memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/memcheck.log
