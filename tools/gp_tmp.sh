T=gpurun_out/tg4
mkdir -p $T
{
for c in c4 c3 c2 c4 c3 c2; do
  echo "== head"; KRP_LIB=abtest/libkrp_head.so timeout 120 python tools/rh_time.py $c 5
  echo "== new";  timeout 120 python tools/rh_time.py $c 5
done
} > $T/log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $T/pytest.log 2>&1
