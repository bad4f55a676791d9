#!/bin/bash
# dev GPU pass: one ncu --set full capture of the sketch kernel.  usage: bash tools/ncu_one.sh <tag> <cfg> [lib name]
TAG=${1:-nc}; CFG=${2:-c2}; LIBN=${3:-prod}
OUT=gpurun_out/$TAG; mkdir -p $OUT
if [ "$LIBN" = "prod" ]; then L=""; else L="KRP_LIB=abtest/libkrp_$LIBN.so"; fi
env $L timeout 600 ncu --set full --clock-control none --import-source on -k regex:krp_tc_sketch_kernel -s 2 -c 1 \
  -o $OUT/sketch_full python tools/tc_time.py $CFG 1 > $OUT/ncu_full.log 2>&1; echo "ncu rc=$?" >> $OUT/ncu_full.log
echo done
