mkdir -p gpurun_out/dbg6
for m in 7 15; do echo "dbg $m"; KRP_TC_DEBUG=$m timeout 60 python tools/tc_time.py c2 20; done > gpurun_out/dbg6/time.log 2>&1
