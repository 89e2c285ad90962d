timeout 600 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -25
timeout 300 python bench.py --steps 50 --no-cpu-baseline --no-e2e 2>&1 | tail -3
