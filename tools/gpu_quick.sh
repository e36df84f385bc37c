python paper_1711_03244_b200/build.py >/dev/null
echo "== v1"; VMC_KERNEL=v1 python tools/quick_tp.py 2>&1 | grep -E "tp"
echo "== pool default"; python tools/quick_tp.py 2>&1 | grep -E "tp|Error|error"
for pct in 60 80 120; do echo "pool pct=$pct"; VMC_POOL_SCATTER_PCT=$pct python tools/quick_tp.py 2>&1 | grep -E "b1|b2"; done
for rf in 2 16; do echo "pool refill=$rf"; VMC_POOL_REFILL_MIN=$rf python tools/quick_tp.py 2>&1 | grep -E "b1|b2"; done
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
