T=gpurun_out/rh17
mkdir -p $T
{
for c in c2 c3 c5; do
  echo "== head"; KRP_LIB=abtest/libkrp_head.so timeout 120 python tools/rh_time.py $c 5
  echo "== new";  timeout 120 python tools/rh_time.py $c 5
done
} > $T/log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -k "rhosvd or sthosvd or tucker or dist" > $T/pytest.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:chol -c 3 --csv --log-file $T/chol.csv python tools/rh_time.py c2 1 > $T/ncu.log 2>&1
