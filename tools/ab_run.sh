#!/bin/bash
# A/B: ab/libold.so vs ab/libnew.so, alternating, same box.
for r in 1 2; do
  for v in old new; do
    echo "== $v"
    python tools/ab_perf.py ab/lib$v.so --scale 22 --ef 16 --ns 1,4 "$@" 2>&1 | grep -E "N=.*par-ws"
    python tools/ab_perf.py ab/lib$v.so --scale 20 --ef 16 --ns 1 --skew uniform 2>&1 | grep -E "N=.*par-ws"
  done
done
