# usage: bash tools/refresh_profiles.sh <tag> — copy an evidence run (tools/gpu_evidence.sh <tag>) into profiles/
T=$1
for W in b1 b2 b3 head; do cp gpurun_out/bench_${W}_$T.json profiles/r1_bench_${W}.json; cp gpurun_out/traffic_$W.csv profiles/r1_ncu_traffic_$W.csv; done
cp gpurun_out/bench_ref_$T.json profiles/r1_bench_reference_b2.json
cp gpurun_out/tp_$T.log profiles/r1_throughput.txt
cp gpurun_out/launches_$T.csv profiles/r1_launches_bench_b2.csv
[ -f gpurun_out/atomics_roofline_$T.json ] && cp gpurun_out/atomics_roofline_$T.json profiles/r1_atomics_roofline.json
python tools/traffic_json.py > /dev/null
python tools/regions_flight.py > tools/regions_flight.txt
R=$(cat tools/regions_flight.txt)
for W in b2 b1; do
  K=$(grep -o "k_flight<[0-9, -]*>" gpurun_out/ncu_full_${W}_$T.log | head -1)
  M=$(cuobjdump -sass gpurun_out/transport_f32_$T.o | grep -o "_ZN3vmc8k_flightILb0ELb0ELb0ELb1ELi0EEEvNS_10KernelArgsE" | head -1)
  CATFILE=flight.cuh python tools/make_profile_summary.py gpurun_out/prof_${W}_$T.ncu-rep gpurun_out/transport_f32_$T.o $M 1e7 profiles/r1_ncu_k_flight_${W}.txt "round 1 (K1f) — k_flight<float, uniform, small-mua> on ${W^^} (cube60), 1e7 photons, B200" "$R" > /dev/null
done
