mkdir -p gpurun_out/ab19
for rep in 1 2; do for c in c2 c3 c4 c5; do for ns in 10000000 0; do echo "ns $ns"; KRP_TC_WAIT_NS=$ns timeout 60 python tools/tc_time.py $c 20; done; done; done > gpurun_out/ab19/time.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/ab19/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab19/pytest_gpu.log
