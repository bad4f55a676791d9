#!/bin/bash
# dev GPU pass: kernel time for env-variable variants.  usage: bash tools/ab_run.sh <tag> "<cfgs>" "<VAR=val ...>|..."
TAG=${1:-ab}; CFGS=${2:-"c2 c5"}; VARIANTS=${3:-"BASE"}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import sys; sys.path.insert(0,'.'); from paper_2507_23207_b200 import build; build.build()" > $OUT/build.log 2>&1
IFS='|' read -ra VS <<< "$VARIANTS"
for c in $CFGS; do
  for v in "${VS[@]}"; do
    echo "== $c $v" >> $OUT/ab.log
    if [ "$v" = "BASE" ]; then envs=""; else envs="$v"; fi
    env $envs timeout 300 python tools/tc_time.py $c 20 >> $OUT/ab.log 2>&1
  done
done
if [ -n "$NCU_CFG" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:krp_tc_sketch_kernel -s 2 -c 1 \
    -o $OUT/sketch_full python tools/tc_time.py $NCU_CFG 1 > $OUT/ncu_full.log 2>&1; echo "ncu rc=$?" >> $OUT/ncu_full.log
fi
echo done
