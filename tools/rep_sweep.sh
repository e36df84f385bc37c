# kernel time vs fluence-map replicas and map placement (B1, B2)
for W in b1 b2; do for R in 1 4 8 16; do echo "== $W replicas $R"; VMC_MAP_REPLICAS=$R python tools/map_placement.py $W 2e7 | awk '{print $NF-1" "$0}' | cut -d' ' -f2- | grep offset | awk '{printf "%s ", $(NF-1)} END{print ""}'; done; done
