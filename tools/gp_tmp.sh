T=gpurun_out/tq1
mkdir -p $T
for c in c2 c4 c5; do for v in 1 2 1 2; do echo "variant $v"; KRP_TTM0_VARIANT=$v timeout 120 python tools/rh_time.py $c 5; done; done > $T/log 2>&1
for v in 1 2; do KRP_TTM0_VARIANT=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ttm_mode0 -c 2 --csv --log-file $T/ttm_c2_$v.csv python tools/rh_time.py c2 1 > /dev/null 2>&1; done
timeout 1200 python -m pytest tests -m gpu -x -q -k "rhosvd or sthosvd or tucker or dist" > $T/pytest.log 2>&1
