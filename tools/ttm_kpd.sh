#!/bin/bash
OUT=$1
for k in 1 2 4; do echo "== kpd $k" >> $OUT; KRP_T0_KPD=$k python tools/ttm_time.py >> $OUT 2>&1; KRP_T0_KPD=$k python -m pytest tests/test_gpu_parity.py -q -k "ttm_positive" 2>&1 | grep -E "assert|passed|failed" >> $OUT; done
