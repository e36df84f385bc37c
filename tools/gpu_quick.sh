python paper_1711_03244_b200/build.py >/dev/null
timeout 900 python -m pytest tests/test_acceptance_gpu.py tests/test_gpu_parity.py -m gpu -q -k "c1 or c2 or c10 or c11 or simulate" 2>&1 | tail -25
