#!/bin/bash
# Final evidence pass: tests, smoke, c2 bench + ncu (gpu_round.sh), then bench lines for the other configs.
TAG=${1:-r01j}
bash tools/gpu_round.sh $TAG c2
for c in c3 c4 c5 c1; do
  timeout 900 python bench.py --config $c > gpurun_out/$TAG/bench_$c.log 2>&1; echo "rc=$?" >> gpurun_out/$TAG/bench_$c.log
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/$TAG/bench_reference.log 2>&1
