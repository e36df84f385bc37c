python paper_1711_03244_b200/build.py >/dev/null
VMC_DEBUG_TIMING=1 python tools/e2e_probe.py 2>&1 | grep -v "^\[vmc\] \(alloc\|enqueue\|finish\)" | tail -30
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
