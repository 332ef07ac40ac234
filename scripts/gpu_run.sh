# development run: GPU tests, throughput, latency, linear-algebra microbenchmark
set -x
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python scripts/quick_tput.py 8192 2 > gpurun_out/tput.log 2>&1
timeout 300 python scripts/latency.py > gpurun_out/lat.log 2>&1
timeout 120 ./scripts/micro/cr_bench > gpurun_out/cr_bench.log 2>&1
