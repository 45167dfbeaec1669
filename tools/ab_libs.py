"""A/B of library builds (MPC200_LIB) on tools/ab_half.py's workloads, one process per build, L2
flushed between steps.  Usage: python tools/ab_libs.py lib1.so lib2.so ... (env KEY=VAL pairs after
a '+' apply to the following library: python tools/ab_libs.py a.so + MPC_MAXTREE_DF=0 a.so)"""
import os
import subprocess
import sys

code = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "ab_half.py")).read().split("code = r'''")[1].split("'''")[0]
runs, env = [], {}
args = sys.argv[1:]
i = 0
while i < len(args):
    if args[i] == "+":
        k, v = args[i + 1].split("=", 1)
        env[k] = v
        i += 2
        continue
    runs.append((args[i], dict(env)))
    env = {}
    i += 1
for rep in range(2):
    for lib, e in runs:
        print(os.path.basename(lib), e, flush=True)
        subprocess.run([sys.executable, "-c", code], env=dict(os.environ, MPC200_LIB=os.path.abspath(lib), **e), check=True)
