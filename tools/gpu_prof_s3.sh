# session-3 capture: warp-scheduling stats + ncu --set full of the production kernels (b1, b3)
mkdir -p gpurun_out/s3
bash tools/gpu_stats.sh b1 b2 b3 head > gpurun_out/s3/stats.txt 2>&1
for W in b1 b3; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_flight -s 1 -c 1 -o gpurun_out/s3/prof_${W} python tools/ncu_target.py $W 1e7 > gpurun_out/s3/ncu_${W}.log 2>&1
done
cp paper_1711_03244_b200/lib/obj/transport_f32.o gpurun_out/s3/transport_f32.o
cat gpurun_out/s3/stats.txt
