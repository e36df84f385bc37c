# round 2 closing evidence after the last kernel changes (event order of the single-label
# kernels, small-run instantiation): GPU suite + smoke, bench lines, launch list, traffic,
# ncu --set full of the B1 and B2 production kernels, small-N table
TAG=${1:-r2zz}
mkdir -p gpurun_out/r2
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2/pytest_$TAG.log 2>&1; tail -2 gpurun_out/r2/pytest_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke_$TAG.log 2>&1; tail -1 gpurun_out/r2/smoke_$TAG.log
bash tools/gpu_bench_r2.sh $TAG
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2/launches_bench_$TAG.csv python bench.py --steps 2 --warmup 3 --photons 100000000 \
  --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2/launches_bench_$TAG.log 2>&1
echo "launches rc=$?"
M=dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.avg.per_cycle_active,smsp__thread_inst_executed_per_inst_executed.ratio,smsp__inst_executed.sum,gpu__time_duration.sum,lts__t_requests_op_red.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum,smsp__sass_inst_executed_op_global_red.sum
for W in b1 b2 b3 head; do
  timeout 900 ncu --metrics $M --clock-control none -k regex:k_flight -s 1 -c 1 --csv \
    --log-file gpurun_out/r2/traffic_${W}_$TAG.csv python tools/ncu_target.py $W 1e8 > /dev/null 2>&1
  echo "traffic $W rc=$?"
done
for W in b1 b2; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_flight -s 1 -c 1 -o gpurun_out/r2/prof_${W}_$TAG python tools/ncu_target.py $W 1e7 > gpurun_out/r2/ncu_full_${W}_$TAG.log 2>&1
  echo "ncu full $W rc=$?"
done
cp paper_1711_03244_b200/lib/obj/transport_f32.o gpurun_out/r2/transport_f32_$TAG.o
