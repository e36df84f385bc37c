# round 2 evidence: one ncu --set full capture of the production transport
# kernel per workload (1e7 photons; head 2e6) + per-launch traffic / issue /
# red-sector metrics at the bench size (1e8; scale = B3), + the launch list of
# the default bench command. usage: bash tools/gpu_prof_r2.sh <tag>
TAG=${1:-r2}
mkdir -p gpurun_out/r2
python paper_1711_03244_b200/build.py > /dev/null || exit 1
cp paper_1711_03244_b200/lib/obj/transport_f32.o gpurun_out/r2/transport_f32_$TAG.o
for W in b1 b2 b3 head; do
  N=1e7; [ $W = head ] && N=2e6
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_flight -s 1 -c 1 \
    -o gpurun_out/r2/prof_${W}_$TAG python tools/ncu_target.py $W $N > gpurun_out/r2/ncu_full_${W}_$TAG.log 2>&1
  echo "full $W rc=$?"
done
M=dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.avg.per_cycle_active,smsp__thread_inst_executed_per_inst_executed.ratio,smsp__inst_executed.sum,gpu__time_duration.sum,lts__t_requests_op_red.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum,smsp__sass_inst_executed_op_global_red.sum
for W in b1 b2 b3 head; do
  timeout 900 ncu --metrics $M --clock-control none -k regex:k_flight -s 1 -c 1 --csv \
    --log-file gpurun_out/r2/traffic_${W}_$TAG.csv python tools/ncu_target.py $W 1e8 > /dev/null 2>&1
  echo "traffic $W rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r2/launches_bench_$TAG.csv python bench.py --steps 2 --warmup 3 --photons 100000000 \
  --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2/launches_bench_$TAG.log 2>&1
echo "launches rc=$?"
