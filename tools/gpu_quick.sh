python paper_1711_03244_b200/build.py >/dev/null
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -8
for w in b1 b3 head; do timeout 600 python bench.py --workload $w --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_$w.json; done
