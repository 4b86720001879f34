timeout 600 python -m pytest tests/test_concurrency_gpu.py -x -q 2>&1 | tail -15
