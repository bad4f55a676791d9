T=gpurun_out/tg2
mkdir -p $T
{
for c in c2 c4 c5; do
  echo "== head"; KRP_LIB=abtest/libkrp_head.so timeout 120 python tools/rh_time.py $c 5
  echo "== new";  timeout 120 python tools/rh_time.py $c 5
done
} > $T/log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -k "rhosvd or sthosvd or tucker" > $T/pytest.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ttm_mode0q -c 2 --csv --log-file $T/c4.csv python tools/rh_time.py c4 1 > /dev/null 2>&1
