T=gpurun_out/df1
mkdir -p $T
for c in c4 c2; do for o in 0 9 0 9; do echo "opt $o"; KRP_LIB=abtest/libkrp_df.so KRP_TC_OPT=$o timeout 60 python tools/tc_time.py $c 30 check | grep -v "mode [1-9]"; done; done > $T/time.log 2>&1
echo "current lib" >> $T/time.log
for c in c4 c2; do timeout 60 python tools/tc_time.py $c 30; done >> $T/time.log 2>&1
