T=gpurun_out/sw8
mkdir -p $T
for c in c2 c3 c4 c5; do for lib in abtest/libkrp_head.so paper_2507_23207_b200/libkrp.so abtest/libkrp_head.so paper_2507_23207_b200/libkrp.so; do echo "lib $lib"; KRP_LIB=$lib timeout 120 python tools/tc_time.py $c 30; done; done > $T/time.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $T/pytest.log 2>&1
timeout 300 python tools/slab_time.py c2 30 > $T/slab.log 2>&1
