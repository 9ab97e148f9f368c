#!/bin/bash
# SASS statistics of one kernel of a translation unit (dev tool, runs here):
#   tools/sass_stats.sh <file.cu> <kernel-name-regex>
# prints registers and an opcode histogram of the matching function.
set -e
cu=$1; pat=$2
out=/tmp/sass_stats.cubin
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -cubin -o $out "$cu" -I"$(dirname "$0")/../include"
cuobjdump -res-usage $out 2>/dev/null | grep -A1 -E "$pat" | grep -oE "REG:[0-9]+|SHARED:[0-9]+" | head -2
cuobjdump -sass $out | awk -v pat="$pat" '/Function :/ {on = ($0 ~ pat)} on && /^ +\/\*[0-9a-f]{4}\*\// {print}' \
  | sed -E 's/ +\/\* 0x[0-9a-f]+ \*\///; s/^ +\/\*[0-9a-f]+\*\/ +//; s/^@!?U?P[0-9T] +//' \
  | awk '{split($1,a,"."); print a[1]}' | sort | uniq -c | sort -rn | head -${3:-25}
