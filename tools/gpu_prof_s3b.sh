# session-3 capture after the launch changes: production tests + ncu --set full of B3 (1e7)
mkdir -p gpurun_out/s3
timeout 900 python -m pytest tests/test_gpu_production.py -m gpu -q -x 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_flight -s 1 -c 1 -o gpurun_out/s3/prof_b3b python tools/ncu_target.py b3 1e7 > gpurun_out/s3/ncu_b3b.log 2>&1
cp paper_1711_03244_b200/lib/obj/transport_f32.o gpurun_out/s3/transport_f32_b.o
