python paper_1711_03244_b200/build.py >/dev/null
python tools/bench_k4.py
timeout 600 python -m pytest tests -m gpu -q -k "normalize or pipeline" 2>&1 | tail -3
