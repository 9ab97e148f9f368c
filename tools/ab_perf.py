"""A/B timing of two builds of the library in one process pair (dev tool):
python tools/ab_perf.py <lib.so> <probe_perf args...>"""
import os
import runpy
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_16064_b200.spmk as m  # noqa: E402

m.load_library(sys.argv[1])
sys.argv = [os.path.join(os.path.dirname(os.path.abspath(__file__)), "probe_perf.py")] + sys.argv[2:]
runpy.run_path(sys.argv[0], run_name="__main__")
