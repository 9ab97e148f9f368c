for m in 4 5 6; do echo "MINB $m"; for sk in heavy uniform; do SPMK_PARWS_MINB=$m timeout 300 python tools/probe_perf.py --skew $sk --scale 20 --ef 16 --ns 1,4 2>&1 | grep "par-ws"; done; done
