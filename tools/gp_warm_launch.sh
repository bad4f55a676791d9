#!/bin/bash
# warm-cache (--cache-control none) per-kernel launch lists of the c4 / c2 8-way slab steps and the c4 step
T=gpurun_out/${1:-warm}
mkdir -p $T
for c in c4 c2; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file $T/slab8_${c}_launches.csv python tools/slab_time.py $c 3 8 > $T/ncu_$c.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file $T/c4_launches.csv python tools/slab_time.py c4 3 1 > $T/ncu_c4full.log 2>&1
