mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_random.py -q -x -k "sym or random or host" --timeout 600 > gpurun_out/pytest_quick.log 2>&1; tail -1 gpurun_out/pytest_quick.log
