cp paper_1711_03244_b200/csrc/transport.cuh /tmp/transport_cur.cuh
for var in prev cur; do
  if [ $var = cur ]; then cp /tmp/transport_cur.cuh paper_1711_03244_b200/csrc/transport.cuh; else cp tools/ab/transport_$var.cuh paper_1711_03244_b200/csrc/transport.cuh; fi
  rm -f paper_1711_03244_b200/lib/obj/transport_f32.o paper_1711_03244_b200/lib/obj/transport_f64.o
  python paper_1711_03244_b200/build.py > /dev/null 2>&1 || echo BUILD FAILED $var
  echo "== $var"; python tools/quick_tp.py 2>&1 | grep tp
done
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
