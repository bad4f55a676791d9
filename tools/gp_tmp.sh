mkdir -p gpurun_out/r01f
for c in c3 c4 c5; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r01f/bench_$c.log 2>&1; done
