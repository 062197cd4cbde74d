mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/probe_task_shape scripts/probe_task_shape.cu && timeout 300 /tmp/probe_task_shape > gpurun_out/r02_probe_task_shape.log 2>&1; echo "probe rc=$?"
cat gpurun_out/r02_probe_task_shape.log
timeout 900 python bench.py --workload cfg5 --csr-path shard --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_cfg5_shard.log 2>&1; echo "cfg5 shard rc=$?"
tail -3 gpurun_out/r2_bench_cfg5_shard.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --workload cfg5 --csr-path shard --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_cfg5_shard_nccl1.log 2>&1; echo "cfg5 shard torchrun rc=$?"
tail -2 gpurun_out/r2_bench_cfg5_shard_nccl1.log
