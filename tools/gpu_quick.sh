python paper_1711_03244_b200/build.py >/dev/null || exit 1
python tools/map_digest.py ab/libvoxmc_b200.so
python tools/map_digest.py
python tools/quick_tp.py 2>&1 | grep tp
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
