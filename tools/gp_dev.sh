#!/bin/bash
# dev pass: quick check, sketch parity subset, per-config kernel timing.  usage: bash tools/gp_dev.sh <tag> [pytest -k] [configs]
TAG=${1:-dev}; OUT=gpurun_out/$TAG; mkdir -p $OUT
K=${2:-"integer or random or recipes or deterministic or misaligned"}
CFGS=${3:-"c5 c2 c3 c4"}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $OUT/smi.txt 2>&1
timeout 60 python tools/tc_quick.py > $OUT/quick.log 2>&1; rc=$?; echo "quick rc=$rc" >> $OUT/quick.log; [ $rc -ne 0 ] && exit 1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "$K" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
for c in $CFGS; do timeout 90 python tools/tc_time.py $c 20 >> $OUT/time.log 2>&1; done
echo done
