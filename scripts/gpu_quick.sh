mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_random.py -q --timeout 600 > gpurun_out/pytest_random.log 2>&1; tail -15 gpurun_out/pytest_random.log
