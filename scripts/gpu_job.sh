mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_random.py -q -m gpu 2>&1 | tail -15
