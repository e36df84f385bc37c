# usage: bash tools/gpu_round.sh <tag> [tests|notests] [ncu|noncu] [bench|nobench]
TAG=${1:-dev}; T=${2:-tests}; N=${3:-ncu}; B=${4:-bench}
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python paper_1711_03244_b200/build.py >/dev/null
timeout 300 python tools/probe_gpu.py 2>&1 | tee gpurun_out/probe_$TAG.log | tail -8
if [ "$T" = tests ]; then timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -25; fi
if [ "$B" = bench ]; then timeout 400 python bench.py 2>&1 | tail -2 | tee gpurun_out/bench_$TAG.json; fi
if [ "$N" = ncu ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_transport -s 1 -c 1 -o gpurun_out/prof_b2_$TAG python tools/ncu_target.py b2 1e7 > gpurun_out/ncu_full_$TAG.log 2>&1
tail -2 gpurun_out/ncu_full_$TAG.log
cp paper_1711_03244_b200/lib/obj/transport_f32.o gpurun_out/transport_f32_$TAG.o
fi
