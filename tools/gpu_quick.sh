python paper_1711_03244_b200/build.py >/dev/null
for pct in 0 35 50 65; do for rf in 1 2 4; do echo "pct=$pct refill=$rf"; VMC_SCATTER_PCT=$pct VMC_REFILL_MIN=$rf python tools/quick_tp.py 2>&1 | grep -E "b2|b1"; done; done
