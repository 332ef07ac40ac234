# round-end measurement: bench line, ncu launch list, one ncu --set full capture of k_solve
set -x
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --batch 2048 --no-cpu-baseline --no-e2e > gpurun_out/ncu_list.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_solve -c 1 -o gpurun_out/k_solve_full \
  python scripts/quick_tput.py 444 1 > gpurun_out/ncu_full.log 2>&1
