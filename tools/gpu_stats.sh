# usage: bash tools/gpu_stats.sh [workloads...] — debug build with -DVMC_STATS, one run each, then restore the normal build
touch paper_1711_03244_b200/csrc/flight.cuh
VMC_NVCC_EXTRA="-DVMC_STATS" python paper_1711_03244_b200/build.py > /dev/null
python tools/stats_run.py "$@" 2>&1 | grep -v "^$"
touch paper_1711_03244_b200/csrc/flight.cuh
python paper_1711_03244_b200/build.py > /dev/null
