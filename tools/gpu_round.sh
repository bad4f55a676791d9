#!/bin/bash
# One gpurun call: GPU parity tests, smoke, a bench line, the ncu launch list and a full capture of the
# fused sketch kernel.  usage (on the box): bash tools/gpu_round.sh <tag> [config]
TAG=${1:-r01}
CFG=${2:-c2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $OUT/smi.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
fi
timeout 600 python bench.py --config $CFG > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches.csv python bench.py --config $CFG --steps 2 --warmup 3 --no-rhosvd --no-e2e \
  --no-cpu-baseline > $OUT/ncu_launch.log 2>&1; echo "ncu rc=$?" >> $OUT/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:krp_tc_sketch_kernel -s 3 -c 1 \
  -o $OUT/sketch_full python bench.py --config $CFG --steps 1 --warmup 3 --no-rhosvd --no-e2e \
  --no-cpu-baseline > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?" >> $OUT/ncu_full.log
