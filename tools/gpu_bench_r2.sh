# round 2: bench lines for every workload + FP64 + the reference arm + small-N sweep
mkdir -p gpurun_out/r2
TAG=${1:-r2}
python bench.py --steps 5 --warmup 3 > gpurun_out/r2/bench_scale_$TAG.json 2> gpurun_out/r2/bench_scale_$TAG.err; echo "scale rc=$?"
for W in b1 b2 b3 head; do
  python bench.py --workload $W --steps 5 --warmup 3 > gpurun_out/r2/bench_${W}_$TAG.json 2> gpurun_out/r2/bench_${W}_$TAG.err; echo "$W rc=$?"
done
python bench.py --workload b2 --precision fp64 --steps 3 --warmup 3 --photons 20000000 --no-cpu-baseline > gpurun_out/r2/bench_b2_fp64_$TAG.json 2> gpurun_out/r2/bench_b2_fp64_$TAG.err; echo "fp64 rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2/bench_reference_scale_$TAG.json 2>&1; echo "ref rc=$?"
python tools/small_n.py > gpurun_out/r2/small_n_$TAG.txt 2>&1; echo "small_n rc=$?"
