"""Tile latency / throughput of the softmax row kernel vs CTA size: cfg2 rows at several tile
counts, default library vs an A/B build (MPC200_LIB), one process per library."""
import os, subprocess, sys

code = r'''
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2511_19711_b200 as m, workloads
rows, cols = workloads.SHAPES["cfg2_softmax"]
c = m.Ctx.for_cfg(workloads.keys(2))
x = c.share(torch.from_numpy(workloads.softmax_inputs(rows, cols)).cuda())
out = c._empty(rows * cols)
s = torch.cuda.current_stream()
res = []
for tiles in (88, 148, 296, 384):
    r = tiles * 32
    xs = tuple(t[: r * cols] for t in x); os_ = tuple(t[: r * cols] for t in out)
    for _ in range(3): c.softmax(xs, r, cols, out=os_)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(20): c.softmax(xs, r, cols, out=os_)
    b.record(s); torch.cuda.synchronize()
    res.append(f"{tiles} tiles {a.elapsed_time(b) / 20:.4f}")
print(os.environ.get("MPC200_LIB", "default"), " | ".join(res))
'''
for lib in [None] + sys.argv[1:]:
    env = dict(os.environ)
    if lib:
        env["MPC200_LIB"] = lib
    subprocess.run([sys.executable, "-c", code], env=env, check=True)
