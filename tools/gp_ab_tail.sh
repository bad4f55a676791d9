#!/bin/bash
# same-box A/B of the sketch tail (head .so vs the working tree's): per-rank slab steps and step/kernel times
T=gpurun_out/${1:-abtail}
mkdir -p $T
{
for i in 1 2; do
  for c in c4 c2 c3; do
    echo "== head $c"; KRP_LIB=abtest/libkrp_head.so timeout 300 python tools/slab_time.py $c 40 1,8 2>&1 | grep -v NCCL
    echo "== new $c";  timeout 300 python tools/slab_time.py $c 40 1,8 2>&1 | grep -v NCCL
  done
done
} > $T/ab.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $T/pytest.log 2>&1; echo "pytest rc=$?" >> $T/pytest.log
