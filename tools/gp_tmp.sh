T=gpurun_out/ro2
mkdir -p $T
timeout 1500 python -m pytest tests -m gpu -x -q > $T/pytest.log 2>&1
for c in c2 c4 c5; do for lib in abtest/libkrp_head.so paper_2507_23207_b200/libkrp.so abtest/libkrp_head.so paper_2507_23207_b200/libkrp.so; do echo "lib $lib"; KRP_LIB=$lib timeout 120 python tools/tc_time.py $c 30; done; done > $T/time.log 2>&1
