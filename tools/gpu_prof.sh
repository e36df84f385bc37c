# usage: bash tools/gpu_prof.sh <tag> [workload] [photons] [kernel-regex] — one ncu --set full capture of the transport kernel
TAG=${1:-dev}; W=${2:-b2}; N=${3:-1e7}; K=${4:-k_flight}
python paper_1711_03244_b200/build.py >/dev/null || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/prof_${W}_$TAG python tools/ncu_target.py $W $N > gpurun_out/ncu_full_${W}_$TAG.log 2>&1
tail -1 gpurun_out/ncu_full_${W}_$TAG.log
cp paper_1711_03244_b200/lib/obj/transport_f32.o gpurun_out/transport_f32_$TAG.o
