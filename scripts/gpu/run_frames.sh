cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_frames.py tests/test_dropin_gpu.py -q -p no:cacheprovider > gpurun_out/pytest_frames.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_frames.log
