cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo "rc=$?" >> gpurun_out/bench_full.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 2 --warmup 3 --batch 2048 --dist-backend gloo --no-e2e > gpurun_out/bench_2rank_gloo.log 2>&1; echo "rc=$?" >> gpurun_out/bench_2rank_gloo.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --steps 2 --warmup 3 --batch 2048 --dist-backend gloo --chunk 512 --no-e2e > gpurun_out/bench_2rank_dyn.log 2>&1; echo "rc=$?" >> gpurun_out/bench_2rank_dyn.log
