HBS_HOST_TIMING=1 timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 4 2>/dev/null | grep "host pipeline" | tail -2
HBS_HOST_TIMING=1 HBS_HOST_CHUNKS=16 timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 4 2>/dev/null | grep "host pipeline" | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_distributed.py tests/test_gpu_large.py -m gpu -x -q 2>&1 | tail -2
