mkdir -p gpurun_out/r01q
timeout 1500 python -m pytest tests -m gpu -x -q -rs --durations=15 > gpurun_out/r01q/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r01q/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01q/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r01q/smoke.log
free -g > gpurun_out/r01q/mem.txt; nproc >> gpurun_out/r01q/mem.txt
