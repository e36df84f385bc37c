# usage: bash tools/gpu_evidence.sh <tag> — the full evidence run for profiles/ (one gpurun call)
TAG=${1:-dev}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python paper_1711_03244_b200/build.py >/dev/null || exit 1
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1 | tee gpurun_out/smoke_$TAG.log
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2 | tee gpurun_out/pytest_gpu_$TAG.log
for W in b2 b1 b3 head; do
  timeout 600 python bench.py --workload $W 2>&1 | tail -1 > gpurun_out/bench_${W}_$TAG.json
done
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1 > gpurun_out/bench_ref_$TAG.json
python tools/quick_tp.py 2>&1 | tee gpurun_out/tp_$TAG.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --photons 10000000 > /dev/null 2>&1
for W in b2 b1; do
  timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:k_(flight|transport)' -s 1 -c 1 -o gpurun_out/prof_${W}_$TAG python tools/ncu_target.py $W 1e7 > gpurun_out/ncu_full_${W}_$TAG.log 2>&1
done
cp paper_1711_03244_b200/lib/obj/transport_f32.o gpurun_out/transport_f32_$TAG.o
bash tools/gpu_traffic.sh
