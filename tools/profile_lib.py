"""profile_one.py against a variant library: python tools/profile_lib.py <lib.so> [profile_one args]"""
import os
import runpy
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_16064_b200.spmk as m  # noqa: E402

m.load_library(sys.argv[1])
sys.argv = [os.path.join(os.path.dirname(os.path.abspath(__file__)), "profile_one.py")] + sys.argv[2:]
runpy.run_path(sys.argv[0], run_name="__main__")
