T=gpurun_out/sw4
mkdir -p $T
for c in c2 c3 c4 c5; do for lib in abtest/libkrp_head.so paper_2507_23207_b200/libkrp.so; do echo "lib $lib"; KRP_LIB=$lib timeout 120 python tools/tc_time.py $c 20 check; done; done > $T/time.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $T/pytest.log 2>&1
timeout 300 python tools/tc_sweep.py 512 40 > $T/sweep.log 2>&1
