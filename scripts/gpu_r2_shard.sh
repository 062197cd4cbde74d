mkdir -p gpurun_out
timeout 1500 python -m pytest -q -x --timeout 900 tests/test_gpu_sharded.py 2>&1 | tail -5
timeout 900 python -m pytest -q -x --timeout 900 tests/test_gpu_dense.py -k "sym" 2>&1 | tail -2
