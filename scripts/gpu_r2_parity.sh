mkdir -p gpurun_out
timeout 2400 python -m pytest -q --timeout 1200 -m gpu "tests/test_gpu_dense.py::test_cfg3_end_to_end_vs_oracle" "tests/test_gpu_batched.py::test_cfg4_full_size" "tests/test_gpu_rank.py::test_cfg5_fixed_200_as_benched" tests/test_gpu_dense.py -k "cfg3_end_to_end or cfg4_full or fixed_200 or nonfinite" > gpurun_out/r2_parity.log 2>&1; tail -3 gpurun_out/r2_parity.log
timeout 900 python scripts/probe_cfg2_norms.py > gpurun_out/r2_cfg2_norms.log 2>&1; tail -12 gpurun_out/r2_cfg2_norms.log
