timeout 900 python -m pytest tests/test_gpu_sharding.py tests/test_gpu_parity.py -x -q --timeout 600 2>&1 | tail -4
timeout 300 python bench.py --workload 70b --steps 200 --warmup 10 2>&1 | tail -2
timeout 300 python bench.py --workload 70b --allgather peer --steps 200 --warmup 10 2>&1 | tail -2
