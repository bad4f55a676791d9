#!/bin/bash
# Final round-2 evidence pass at HEAD: tests, smoke, c5 bench + launch list + full capture, other configs' bench lines, reference arm.
TAG=${1:-r02l}
OUT=gpurun_out/$TAG
mkdir -p $OUT
bash tools/gpu_round.sh $TAG c5
for c in c2 c3 c4; do
  timeout 600 python bench.py --config $c --no-per-config > $OUT/bench_$c.log 2>&1; echo "rc=$?" >> $OUT/bench_$c.log
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference.log 2>&1; echo "rc=$?" >> $OUT/bench_reference.log
echo done > $OUT/done.txt
