cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python scripts/ab_bitexact.py ab_prev_libaccfem.so paper_2503_06922_b200/libaccfem.so > gpurun_out/f8_ab.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/f8_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f8_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f8_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f8_smoke.log
timeout 600 python scripts/contact_scaling.py > gpurun_out/f8_contact_scaling.json 2>&1
ACCFEM_LIB=ab_prev_libaccfem.so timeout 600 python scripts/contact_scaling.py > gpurun_out/f8_contact_scaling_prev.json 2>&1
timeout 900 python scripts/latency_probe.py cfg3p cfg4_s0 cfg1 cfg5 cfg5_296 cfg5_1184 > gpurun_out/f8_latency.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/f8_bench.log 2>&1; echo "rc=$?" >> gpurun_out/f8_bench.log
python scripts/profile_ksolve.py 8192 > gpurun_out/f8_prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/ksolve_r02_f8 python scripts/profile_ksolve.py 8192 > gpurun_out/f8_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/f8_ncu.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f8_launches.csv python scripts/profile_ksolve.py 8192 > gpurun_out/f8_ncu_launches.log 2>&1
