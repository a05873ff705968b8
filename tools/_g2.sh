timeout 900 python -m pytest tests/test_gpu_slab.py tests/test_gpu_det.py -q -x 2>&1 | tail -15
