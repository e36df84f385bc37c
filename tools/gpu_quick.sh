for v in "-DVMC_SUBSTEPS=1" "-DVMC_SUBSTEPS=2" "-DVMC_SUBSTEPS=3"; do
  rm -f paper_1711_03244_b200/lib/obj/transport_f32.o
  VMC_NVCC_EXTRA="$v" python paper_1711_03244_b200/build.py >/dev/null
  echo "== $v"; python tools/quick_tp.py 2>&1 | grep -E "tp"
done
rm -f paper_1711_03244_b200/lib/obj/transport_f32.o; python paper_1711_03244_b200/build.py >/dev/null
