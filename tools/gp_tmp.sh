mkdir -p gpurun_out/ab12
for rep in 1 2; do for c in c2 c3 c4 c5; do
 echo "head"; KRP_LIB=$PWD/abtest/libkrp_head.so timeout 60 python tools/tc_time.py $c 20
 echo "new"; timeout 60 python tools/tc_time.py $c 20
done; done > gpurun_out/ab12/time.log 2>&1
