T=gpurun_out/sl2
mkdir -p $T
for c in c2 c4 c3; do for lib in paper_2507_23207_b200/libkrp.so abtest/libkrp_A.so abtest/libkrp_B.so abtest/libkrp_C.so abtest/libkrp_D.so paper_2507_23207_b200/libkrp.so; do echo "lib $lib"; KRP_LIB=$lib timeout 120 python tools/tc_time.py $c 30; done; done > $T/time.log 2>&1
