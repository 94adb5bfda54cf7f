"""Run tools/run_case.py-style timing against an alternative build of
libcwcsim.so (experiments): python tools/variant_run.py LIB CONFIG [env...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1010_2438_b200 import cwc  # noqa: E402

cwc.LIB_PATH = os.path.abspath(sys.argv[1])
sys.argv = [sys.argv[0], "--config", sys.argv[2], "--repeat", "3"]
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "run_case.py")).read())
