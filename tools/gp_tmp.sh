mkdir -p gpurun_out/rh6
{
for c in c2 c3 c4; do
  echo "== head"; KRP_LIB=abtest/libkrp_head.so timeout 120 python tools/rh_time.py $c 5
  echo "== new";  timeout 120 python tools/rh_time.py $c 5
done
timeout 900 python -m pytest tests -m gpu -x -q -k "rhosvd or sthosvd or chol or jacobi or tucker or dist" 2>&1 | tail -5
} > gpurun_out/rh6/log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/rh6/launches_c2.csv python tools/rh_time.py c2 1 > gpurun_out/rh6/ncu.log 2>&1
