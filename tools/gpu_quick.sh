for v in "-DVMC_MIN_BLOCKS=4" ""; do
  rm -f paper_1711_03244_b200/lib/obj/transport_f32.o
  VMC_NVCC_EXTRA="$v" python paper_1711_03244_b200/build.py >/dev/null
  echo "== $v"; python tools/quick_tp.py 2>&1 | grep -E "tp"
done
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
