"""Scratch: v6 ring-size sweep (BB_V6_R) on the headline."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.quick_v5 import time_cfg
os.environ["BB_V6_G"] = "4"
for dt, Rs in (("f32", (9, 11, 13, 17)), ("f64", (9,))):
    for R in Rs:
        os.environ["BB_V6_R"] = str(R)
        print(dt, "R", R, flush=True)
        time_cfg(32768, 128, dt, 32, reps=2)
