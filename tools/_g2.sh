timeout 900 python -m pytest tests/test_gpu_slab.py -q -x 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_slab.py -q -x 2>&1 | grep -E "^E " | head -10
