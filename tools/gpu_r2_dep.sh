# round 2: deposit-path A/B (direct / warp-aggregated / hot box) + red-counter semantics
mkdir -p gpurun_out/r2
python paper_1711_03244_b200/build.py > /dev/null || exit 1
python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "deposit_paths" > gpurun_out/r2/dep_tests.log 2>&1; tail -3 gpurun_out/r2/dep_tests.log
python tools/deposit_ab.py 1e7 > gpurun_out/r2/deposit_ab.txt 2>&1; cat gpurun_out/r2/deposit_ab.txt | grep -v "^{"
M=lts__t_requests_op_red.sum,lts__t_sectors_op_red.sum,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum,smsp__sass_inst_executed_op_global_red.sum,gpu__time_duration.sum
timeout 300 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2/red_probe.csv paper_1711_03244_b200/lib/red_counter_probe > gpurun_out/r2/red_probe.out 2>&1
cat gpurun_out/r2/red_probe.out | grep pattern
M2=$M,sm__inst_executed.sum,smsp__thread_inst_executed_per_inst_executed.ratio,sm__inst_executed.avg.per_cycle_active,smsp__sass_inst_executed_op_shared_atom.sum
for D in direct warp hotbox; do
  for W in b1 b3; do
    VMC_DEPOSIT=$D timeout 600 ncu --metrics $M2 --clock-control none -k 'regex:k_flight' -s 1 -c 1 --csv --log-file gpurun_out/r2/dep_${D}_${W}.csv python tools/ncu_target.py $W 1e7 > /dev/null 2>&1
    echo "$D $W rc=$?"
  done
done
