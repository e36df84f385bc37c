python paper_1711_03244_b200/build.py >/dev/null || exit 1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 400 python bench.py --workload b3 --no-cpu-baseline 2>&1 | tail -1
