mkdir -p gpurun_out/rh2
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "rhosvd or sthosvd" > gpurun_out/rh2/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rh2/pytest.log
for c in c2 c3 c4; do timeout 120 python tools/rh_time.py $c 3; done > gpurun_out/rh2/time.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/rh2/launches_c2.csv python tools/rh_time.py c2 1 > /dev/null 2>&1
