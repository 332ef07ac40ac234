cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final_pytest.log
python scripts/profile_ksolve.py 8192 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/ksolve_r02_final python scripts/profile_ksolve.py 8192 > gpurun_out/ncu_ksolve.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_ksolve.log
python scripts/profile_ksolve.py 8192 > gpurun_out/prof_plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv python scripts/profile_ksolve.py 8192 > gpurun_out/ncu_launches.log 2>&1
