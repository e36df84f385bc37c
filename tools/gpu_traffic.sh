# per-launch DRAM traffic and issue metrics of K1 at the bench size (1e8 photons) for every workload
python paper_1711_03244_b200/build.py >/dev/null || exit 1
M=dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.avg.per_cycle_active,smsp__thread_inst_executed_per_inst_executed.ratio,smsp__inst_executed.sum,gpu__time_duration.sum,lts__t_requests_op_red.sum,lts__t_sectors_srcunit_tex_lookup_miss.sum
for W in b1 b2 b3 head; do
  timeout 900 ncu --metrics $M --clock-control none -k 'regex:k_(flight|transport)' -s 1 -c 1 --csv --log-file gpurun_out/traffic_$W.csv python tools/ncu_target.py $W 1e8 > /dev/null 2>&1
  echo "$W rc=$?"
done
