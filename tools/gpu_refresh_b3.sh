# refresh the B3 / scale evidence after a kernel change: bench lines, ncu full, traffic
TAG=${1:-r2g}
mkdir -p gpurun_out/r2
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2/pytest_$TAG.log 2>&1; tail -1 gpurun_out/r2/pytest_$TAG.log
for W in scale b3 b1 b2 head; do
  python bench.py --workload $W --steps 5 --warmup 3 > gpurun_out/r2/bench_${W}_$TAG.json 2> gpurun_out/r2/bench_${W}_$TAG.err; echo "$W rc=$?"
done
python paper_1711_03244_b200/build.py > /dev/null
cp paper_1711_03244_b200/lib/obj/transport_f32.o gpurun_out/r2/transport_f32_$TAG.o
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_flight -s 1 -c 1 \
  -o gpurun_out/r2/prof_b3_$TAG python tools/ncu_target.py b3 1e7 > gpurun_out/r2/ncu_full_b3_$TAG.log 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.avg.per_cycle_active,smsp__thread_inst_executed_per_inst_executed.ratio,smsp__inst_executed.sum,gpu__time_duration.sum,lts__t_requests_op_red.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum,smsp__sass_inst_executed_op_global_red.sum
for W in b1 b2 b3 head; do
  timeout 900 ncu --metrics $M --clock-control none -k regex:k_flight -s 1 -c 1 --csv \
    --log-file gpurun_out/r2/traffic_${W}_$TAG.csv python tools/ncu_target.py $W 1e8 > /dev/null 2>&1
  echo "traffic $W rc=$?"
done
