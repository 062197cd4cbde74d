# K3n (sharded CSR ranking): parity tests, then a world-1 timing of the product call on cfg5
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_rank_sharded.py -x -q -m gpu > gpurun_out/pytest_rank_sharded.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_rank_sharded.log
timeout 900 python scripts/probe_csr_shard.py > gpurun_out/r02_probe_csr_shard.log 2>&1; echo "probe rc=$?"
cat gpurun_out/r02_probe_csr_shard.log
