#!/bin/bash
# Round-2 evidence pass on one B200: tests, smoke, the default (c5) bench line + ncu, the other configs'
# bench lines, the reference arm, decomposition launch lists, ncu captures of the TTM and the eigensolver.
TAG=${1:-r02d}
OUT=gpurun_out/$TAG
mkdir -p $OUT
bash tools/gpu_round.sh $TAG c5
for c in c2 c3 c4; do
  timeout 900 python bench.py --config $c --no-per-config > $OUT/bench_$c.log 2>&1; echo "rc=$?" >> $OUT/bench_$c.log
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference.log 2>&1; echo "rc=$?" >> $OUT/bench_reference.log
python tools/decomp_launches.py rhosvd c5 > $OUT/decomp.log 2>&1
python tools/decomp_launches.py sthosvd c3 >> $OUT/decomp.log 2>&1
python tools/decomp_launches.py rhosvd c2 >> $OUT/decomp.log 2>&1
python tools/decomp_launches.py rhosvd c4 >> $OUT/decomp.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/rhosvd_c5_launches.csv python tools/decomp_launches.py rhosvd c5 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/sthosvd_c3_launches.csv python tools/decomp_launches.py sthosvd c3 > /dev/null 2>&1
python tools/ttm_time.py > $OUT/ttm_time.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ttm0_tc_kernel -s 3 -c 1 -o $OUT/ttm0_full python tools/ttm_time.py > $OUT/ncu_ttm0.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:jacobi_top -s 2 -c 1 -o $OUT/jacobi_full python tools/decomp_launches.py rhosvd c5 > $OUT/ncu_jacobi.log 2>&1
echo done > $OUT/done.txt
