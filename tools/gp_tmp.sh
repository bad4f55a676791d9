mkdir -p gpurun_out/ab7
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/ab7/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab7/pytest_gpu.log
for c in c2 c3 c4 c5; do timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/ab7/launches_$c.csv python tools/tc_time.py $c 2 > /dev/null 2>&1; done
