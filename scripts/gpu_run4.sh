# device grid build: parity tests, timing, ncu launch list of the grid kernels
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python scripts/grid_probe.py > gpurun_out/grid.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_grid -c 6 --csv \
  python scripts/grid_probe.py > gpurun_out/ncu_grid.csv 2> gpurun_out/ncu_grid.err
