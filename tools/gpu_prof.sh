# usage: bash tools/gpu_prof.sh <tag> [env...]  -> ncu full capture of the transport kernel on b2 1e7
TAG=$1; shift
python paper_1711_03244_b200/build.py >/dev/null
env "$@" timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_transport -s 1 -c 1 -o gpurun_out/prof_$TAG python tools/ncu_target.py b2 1e7 > gpurun_out/ncu_$TAG.log 2>&1
tail -1 gpurun_out/ncu_$TAG.log
cp paper_1711_03244_b200/lib/obj/transport_f32.o gpurun_out/transport_f32_$TAG.o
