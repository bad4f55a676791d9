mkdir -p gpurun_out/d1
timeout 300 python -m pytest tests/test_gpu_dist1.py -x -q > gpurun_out/d1/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/d1/pytest.log
