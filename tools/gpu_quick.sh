python paper_1711_03244_b200/build.py >/dev/null
for pct in 40 45 50 55 60; do echo "pct=$pct"; VMC_SCATTER_PCT=$pct python tools/quick_tp.py | grep -E "b1|b2|head"; done
for rf in 1 3 4; do echo "refill=$rf"; VMC_REFILL_MIN=$rf python tools/quick_tp.py | grep -E "b2|head"; done
