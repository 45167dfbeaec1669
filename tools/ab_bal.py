"""A/B of the balanced softmax plan (MPC_SOFTMAX_BAL=0 / 1) with tools/ab_half.py's timing code."""
import os
import subprocess
import sys

code = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "ab_half.py")).read().split("code = r'''")[1].split("'''")[0]
for rep in range(2):
    for v in ("0", "1"):
        print("MPC_SOFTMAX_BAL=" + v, flush=True)
        subprocess.run([sys.executable, "-c", code], env=dict(os.environ, MPC_SOFTMAX_BAL=v, MPC_TAIL_HALF="0"), check=True)
