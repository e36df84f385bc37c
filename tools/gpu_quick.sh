python paper_1711_03244_b200/build.py >/dev/null || exit 1
for U in 3 2; do
  touch paper_1711_03244_b200/csrc/transport_kernels.cu
  VMC_NVCC_EXTRA="-DVMC_AZ_UNROLL=$U" python paper_1711_03244_b200/build.py >/dev/null || exit 1
  echo "az_unroll=$U"; python tools/quick_tp.py 2>&1 | grep tp
done
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
