#!/bin/bash
# dev GPU pass: parity tests of the sketch + per-config kernel timing.  usage: bash tools/dev_run.sh <tag> [pytest -k expr]
TAG=${1:-dev}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $OUT/smi.txt 2>&1
python -c "import sys; sys.path.insert(0,'.'); from paper_2507_23207_b200 import build; build.build()" > $OUT/build.log 2>&1
timeout 120 python tools/tc_quick.py > $OUT/quick.log 2>&1; echo "quick rc=$?" >> $OUT/quick.log
if [ -n "$2" ]; then
  timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "$2" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
else
  timeout 900 python -m pytest tests/test_gpu_parity.py -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
fi
for c in c2 c3 c4 c5; do timeout 300 python tools/tc_time.py $c 20 >> $OUT/time.log 2>&1; done
echo done
