T=gpurun_out/ch2
mkdir -p $T
{
for c in c2 c3 c2 c3; do
  echo "== head"; KRP_LIB=abtest/libkrp_head.so timeout 120 python tools/rh_time.py $c 10
  echo "== new";  timeout 120 python tools/rh_time.py $c 10
done
} > $T/log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $T/pytest.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:chol -c 3 --csv --log-file $T/chol.csv python tools/rh_time.py c2 1 > /dev/null 2>&1
