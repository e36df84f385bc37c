python paper_1711_03244_b200/build.py >/dev/null
echo "== v1"; VMC_KERNEL=v1 python tools/quick_tp.py 2>&1 | grep -E "tp"
for pct in 35 50 70; do echo "pct=$pct"; VMC_KERNEL=v1 VMC_SCATTER_PCT=$pct python tools/quick_tp.py 2>&1 | grep -E "b1|b2"; done
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
