timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "tcgen05 or 70-256" 2>&1 | tail -15
