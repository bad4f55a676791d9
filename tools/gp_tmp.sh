#!/bin/bash
# re-run of the default bench (both arms) after the oracle-sample calibration change
OUT=gpurun_out/r02m; mkdir -p $OUT
( time timeout 900 python bench.py ) > $OUT/bench_c5.log 2>&1; echo "rc=$?" >> $OUT/bench_c5.log
( time timeout 900 python bench.py --impl reference ) > $OUT/bench_reference_default.log 2>&1; echo "rc=$?" >> $OUT/bench_reference_default.log
( time timeout 900 python bench.py --config c4 --no-per-config ) > $OUT/bench_c4.log 2>&1; echo "rc=$?" >> $OUT/bench_c4.log
