T=gpurun_out/sw3
mkdir -p $T
timeout 300 python tools/tc_sweep.py 512 40 > $T/sweep.log 2>&1
for c in c2 c3 c4 c5; do timeout 120 python tools/tc_time.py $c 20 check; done > $T/time.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $T/pytest.log 2>&1
timeout 300 python tools/slab_time.py c2 30 > $T/slab.log 2>&1
