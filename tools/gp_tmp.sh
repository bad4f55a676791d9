T=gpurun_out/rh14
mkdir -p $T
{
for c in c2 c4 c5; do
  echo "== new";  timeout 120 python tools/rh_time.py $c 5
done
} > $T/log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -k "rhosvd or sthosvd or tucker or dist" > $T/pytest.log 2>&1
for c in c2 c5; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ttm_mode0 -c 3 --csv --log-file $T/launches_$c.csv python tools/rh_time.py $c 1 > $T/ncu_$c.log 2>&1
done
