T=gpurun_out/rh18
mkdir -p $T
{
for c in c2 c3 c4; do
  echo "== head"; KRP_LIB=abtest/libkrp_head.so timeout 120 python tools/rh_time.py $c 5
  echo "== new";  timeout 120 python tools/rh_time.py $c 5
done
} > $T/log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -k "rhosvd or sthosvd or tucker or dist" > $T/pytest.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:mode_gram -c 8 --csv --log-file $T/mg.csv python tools/rh_time.py c3 1 > $T/ncu.log 2>&1
