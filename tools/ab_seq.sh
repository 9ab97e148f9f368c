#!/bin/bash
# A/B of library builds on the seq-ws sweep (dev tool): tools/ab_seq.sh name1 name2 ...
# (ab/lib<name>.so), alternating, cfg2's matrix at N=32/64/128 and uniform N=32.
for r in 1 2; do
  for v in "$@"; do
    echo "== $v"
    python tools/ab_perf.py ab/lib$v.so --scale 20 --ef 16 --ns 32,64,128 --reps 20 2>&1 | grep -E "seq-ws"
    python tools/ab_perf.py ab/lib$v.so --scale 20 --ef 16 --ns 32 --skew uniform --reps 20 2>&1 | grep -E "seq-ws"
  done
done
