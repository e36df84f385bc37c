python paper_1711_03244_b200/build.py >/dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k corner 2>&1 | tail -25
