#!/bin/bash
# c4 post-kernel tail: per-kernel launch lists of the c4 step and of the c4 8-way slab step (dev tool)
T=gpurun_out/${1:-c4tail}
mkdir -p $T
timeout 300 python tools/slab_time.py c4 30 1,8 > $T/slab.log 2>&1
timeout 300 python tools/slab_time.py c2 30 1,8 >> $T/slab.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $T/slab8_launches.csv \
  python tools/slab_time.py c4 3 8 > $T/ncu1.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $T/c4_launches.csv \
  python bench.py --config c4 --steps 2 --warmup 3 --no-rhosvd --no-e2e --no-cpu-baseline --no-per-config > $T/ncu2.log 2>&1
