#!/bin/bash
for m in ${2:-4 1 2 3 0}; do
  echo "KRP_TC_DEBUG=$m"; KRP_TC_DEBUG=$m timeout 120 python tools/tc_time.py ${1:-c2} 10
done
