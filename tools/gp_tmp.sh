T=gpurun_out/jt1
mkdir -p $T
for n in 1024 512 256 128; do echo "threads $n"; for c in c2 c3; do KRP_JACOBI_THREADS=$n timeout 120 python tools/rh_time.py $c 10; done; done > $T/log 2>&1
for n in 1024 256 128; do KRP_JACOBI_THREADS=$n timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:jacobi -c 2 --csv --log-file $T/jac_$n.csv python tools/rh_time.py c2 1 > /dev/null 2>&1; done
timeout 900 python -m pytest tests -m gpu -x -q -k "rhosvd or sthosvd" > $T/pytest.log 2>&1
