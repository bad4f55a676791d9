#!/bin/bash
# evidence pass after the per-plan L2 prefetch distance: quick timings, GPU suite, smoke, default bench, per-config lines
OUT=gpurun_out/r02p; mkdir -p $OUT
for c in c2 c3 c4 c5; do timeout 300 python tools/tc_time.py $c 20 >> $OUT/tc_time.log 2>&1; done
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench_c5.log 2>&1; echo "rc=$?" >> $OUT/bench_c5.log
for c in c2 c3 c4; do
  timeout 600 python bench.py --config $c --no-per-config > $OUT/bench_$c.log 2>&1; echo "rc=$?" >> $OUT/bench_$c.log
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-rhosvd --no-e2e \
  --no-cpu-baseline > $OUT/ncu_launch.log 2>&1; echo "ncu rc=$?" >> $OUT/ncu_launch.log
bash tools/ncu_configs.sh r02p "c2 c3 c4 c5" > /dev/null 2>&1
for c in c4 c5; do timeout 300 python tools/slab_time.py $c 50 1,8 > $OUT/slab_$c.log 2>&1; done
echo done > $OUT/done.txt
