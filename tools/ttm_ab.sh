#!/bin/bash
# dev A/B: krp_ttm timings for the production library and abtest/ variants.  usage: bash tools/ttm_ab.sh out.log v1 v2 ...
OUT=$1; shift
python tools/ttm_time.py > $OUT 2>&1
for v in "$@"; do echo "== $v" >> $OUT; KRP_LIB=abtest/libkrp_$v.so python tools/ttm_time.py >> $OUT 2>&1; done
