# Strong-scaling emulation on ONE B200 (no 8-GPU box in this build's rounds): the per-rank
# share of BASELINE configs[4] (1e9 B3 photons in total, S1 split) at N = 1, 2, 4, 8 is run as
# a single-GPU bench step of 1e9/N photons (same kernel, same record sort), so T(1)/T(N)
# is the compute part of the strong-scaling speed-up; the N > 1 exchange (NCCL reduce of the
# 1.7 MB map + record gather) is not in it.
mkdir -p gpurun_out/r2
for N in 1 2 4 8; do
  P=$((1000000000 / N))
  python bench.py --steps 5 --warmup 3 --photons $P --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2/scale_emul_$N.json 2> gpurun_out/r2/scale_emul_$N.err
  echo "N=$N rc=$?"
done
python tools/small_n.py b1,b2,b3,head > gpurun_out/r2/small_n_r2z2.txt 2>&1
