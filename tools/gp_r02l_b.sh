#!/bin/bash
# Second half of the final round-2 evidence pass: ncu captures of c2-c4 at HEAD, per-rank slab timings, decomposition times.
TAG=${1:-r02l}
OUT=gpurun_out/$TAG
mkdir -p $OUT
bash tools/ncu_configs.sh $TAG "c2 c3 c4"
for c in c2 c3 c4 c5; do
  timeout 300 python tools/slab_time.py $c 50 > $OUT/slab_$c.log 2>&1; echo "rc=$?" >> $OUT/slab_$c.log
done
timeout 300 python tools/rh_back_to_back.py > $OUT/rh_back_to_back.log 2>&1
python tools/decomp_launches.py rhosvd c5 > $OUT/decomp.log 2>&1
python tools/decomp_launches.py sthosvd c3 >> $OUT/decomp.log 2>&1
python tools/decomp_launches.py rhosvd c2 >> $OUT/decomp.log 2>&1
python tools/decomp_launches.py rhosvd c4 >> $OUT/decomp.log 2>&1
echo done > $OUT/done_b.txt
