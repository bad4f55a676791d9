#!/bin/bash
# dev GPU pass: production timing + role timeline of CTAs 0/1 with the trace build (abtest/libkrp_trace.so)
TAG=${1:-tr}; CFGS=${2:-"c2 c5"}
OUT=gpurun_out/$TAG; mkdir -p $OUT
for c in $CFGS; do
  timeout 300 python tools/tc_time.py $c 20 >> $OUT/time.log 2>&1
  KRP_LIB=abtest/libkrp_trace.so KRP_TC_TRACE=$OUT/trace_$c.txt timeout 300 python tools/tc_time.py $c 1 x >> $OUT/trace_time.log 2>&1
done
echo done
