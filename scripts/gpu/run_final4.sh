cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/final_bench.log 2>&1; echo "rc=$?" >> gpurun_out/final_bench.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/final_bench_ref.log
timeout 600 python scripts/contact_scaling.py > gpurun_out/final_contact_scaling.json 2>&1
for m in cr team4; do ACCFEM_MODE=$m timeout 600 python scripts/latency_probe.py cfg3p cfg4_s0 cfg1 cfg5 >> gpurun_out/final_latency.log 2>&1; done
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final_smoke.log
