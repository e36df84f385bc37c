mkdir -p gpurun_out/r2
bash tools/gpu_stats.sh b1 b2 b3 head > gpurun_out/r2/stats_a.txt 2>&1
for W in b1 b2; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_flight -s 1 -c 1 -o gpurun_out/r2/prof_${W}_a python tools/ncu_target.py $W 1e7 > gpurun_out/r2/ncu_${W}_a.log 2>&1
done
cp paper_1711_03244_b200/lib/obj/transport_f32.o gpurun_out/r2/transport_f32_a.o
python tools/small_n.py > gpurun_out/r2/small_n_a.txt 2>&1
cat gpurun_out/r2/stats_a.txt gpurun_out/r2/small_n_a.txt
