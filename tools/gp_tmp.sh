mkdir -p gpurun_out/ab3
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/ab3/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab3/pytest_gpu.log
for c in c2 c3 c4 c5; do
 echo "old"; KRP_LIB=$PWD/abtest/libkrp_old.so KRP_TC_OPT=1 timeout 60 python tools/tc_time.py $c 20
 echo "new"; timeout 60 python tools/tc_time.py $c 20
done > gpurun_out/ab3/time.log 2>&1
