"""PAIR-loopback cfg2 softmax and cfg3-sized GELU (1M) in both exchange wire formats (LL, LL63), for
each library build given on the command line (MPC200_LIB; one process each)."""
import os
import subprocess
import sys

code = r'''
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2511_19711_b200 as m, workloads
res = []
for fmt in (0, 1):
    c = m.Ctx.for_cfg(workloads.keys(2), mode=m.binding.MODE_PAIR_LOOPBACK)
    c.set_exchange(fmt)
    rows, cols = workloads.SHAPES["cfg2_softmax"]
    x = c.share(torch.from_numpy(workloads.softmax_inputs(rows, cols).ravel()).cuda())
    g = c.share(torch.from_numpy(workloads.normal_inputs(1 << 20, 3)).cuda())
    s = torch.cuda.current_stream()
    def t(fn, reps=5):
        fn(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(reps): fn()
        b.record(s); torch.cuda.synchronize()
        return a.elapsed_time(b) / reps
    res += [f"fmt{fmt} softmax {t(lambda: c.softmax(x, rows, cols)):.4f}",
            f"fmt{fmt} gelu1M {t(lambda: c.gelu(g, form='poly_abs', degree=4)):.4f}"]
    c.sync()
print(os.path.basename(os.environ.get("MPC200_LIB", "default")), " | ".join(res), flush=True)
'''
for rep in range(2):
    for lib in sys.argv[1:]:
        subprocess.run([sys.executable, "-c", code], env=dict(os.environ, MPC200_LIB=os.path.abspath(lib)), check=True)
