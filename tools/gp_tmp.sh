T=gpurun_out/rh8
mkdir -p $T
{
for c in c2 c3 c4 c5; do
  echo "== head"; KRP_LIB=abtest/libkrp_head.so timeout 120 python tools/rh_time.py $c 5
  echo "== new";  timeout 120 python tools/rh_time.py $c 5
done
} > $T/log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $T/pytest.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $T/launches_c2.csv python tools/rh_time.py c2 1 > $T/ncu.log 2>&1
