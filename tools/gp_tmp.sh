T=gpurun_out/sl3
mkdir -p $T
for c in c2 c3 c4; do for lib in abtest/libkrp_head.so abtest/libkrp_E.so abtest/libkrp_A16.so abtest/libkrp_A32.so abtest/libkrp_A64.so abtest/libkrp_head.so abtest/libkrp_E.so abtest/libkrp_A16.so abtest/libkrp_A32.so abtest/libkrp_A64.so; do echo "lib $lib"; KRP_LIB=$lib timeout 120 python tools/tc_time.py $c 30; done; done > $T/time.log 2>&1
