# development run: tests, throughput, cfg5, phase profile, ncu dram of one wave
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python scripts/quick_tput.py 8192 3 > gpurun_out/tput.log 2>&1
timeout 300 python scripts/cfg5_probe.py > gpurun_out/cfg5.log 2>&1
ACCFEM_PROF_SO=paper_2503_06922_b200/libaccfem_prof.so timeout 300 python scripts/phase_profile.py cfg4 1776 > gpurun_out/prof.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_solve -c 1 python scripts/quick_tput.py 444 1 > gpurun_out/ncu_dram.log 2>&1
