#!/bin/bash
# ncu evidence per config: one --set full capture of the fused sketch kernel + the launch list of a 3-step run
# (random N(0,1) data of each config's shape: the counters do not depend on values).  usage: bash tools/ncu_configs.sh <tag> "<cfgs>"
TAG=${1:-r02b}; CFGS=${2:-"c2 c3 c4 c5"}
OUT=gpurun_out/$TAG; mkdir -p $OUT
for c in $CFGS; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:krp_tc_sketch_kernel -s 2 -c 1 \
    -o $OUT/sketch_full_$c python tools/tc_time.py $c 1 > $OUT/ncu_full_$c.log 2>&1; echo "rc=$?" >> $OUT/ncu_full_$c.log
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches_$c.csv \
    python tools/tc_time.py $c 3 > $OUT/ncu_launch_$c.log 2>&1; echo "rc=$?" >> $OUT/ncu_launch_$c.log
done
python tools/sass_counts.py > $OUT/sass_counts.txt 2>&1
echo done
