# usage: bash tools/ab_build.sh <name> "<extra nvcc flags for transport_f32>"  -> ab/<name>.so (then VMC_LIB_PATH=ab/<name>.so)
mkdir -p ab
touch paper_1711_03244_b200/csrc/flight.cuh
VMC_NVCC_EXTRA="$2" python paper_1711_03244_b200/build.py > /dev/null && cp paper_1711_03244_b200/lib/libvoxmc_b200.so ab/$1.so
touch paper_1711_03244_b200/csrc/flight.cuh
python paper_1711_03244_b200/build.py > /dev/null
