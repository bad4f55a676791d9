#!/bin/bash
# dev GPU pass: time the sketch with several libraries (abtest/libkrp_<name>.so, "prod" = in-tree)
#   usage: bash tools/lib_ab.sh <tag> "<cfgs>" "name1 name2 ..." [trace cfgs]
TAG=${1:-lab}; CFGS=${2:-"c2 c5"}; LIBS=${3:-"prod"}; TRC=${4:-""}
OUT=gpurun_out/$TAG; mkdir -p $OUT
for rep in 1 2; do
for c in $CFGS; do
  for n in $LIBS; do
    if [ "$n" = "prod" ]; then L=""; else L="KRP_LIB=abtest/libkrp_$n.so"; fi
    echo -n "$n rep$rep " >> $OUT/ab.log
    env $L timeout 300 python tools/tc_time.py $c 20 >> $OUT/ab.log 2>&1
  done
done
done
for c in $TRC; do
  KRP_LIB=abtest/libkrp_trace.so KRP_TC_TRACE=$OUT/trace_$c.txt timeout 300 python tools/tc_time.py $c 1 x >> $OUT/trace_time.log 2>&1
done
echo done
