"""End-to-end (host buffers) cfg2 softmax: sequential H2D -> op -> D2H on one stream vs the
pipelined mpc_softmax_hostio at several chunk sizes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_19711_b200 as m
import workloads

rows, cols = workloads.SHAPES["cfg2_softmax"]
c = m.Ctx.for_cfg(workloads.keys(2))
x = c.share(torch.from_numpy(workloads.softmax_inputs(rows, cols)).cuda())
hx = tuple(t.cpu().pin_memory() for t in x)
hz = tuple(torch.empty_like(t).pin_memory() for t in hx)
din = [torch.empty_like(t) for t in x]
out = c._empty(rows * cols)
s = torch.cuda.current_stream()


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def seq():
    for d, h in zip(din, hx):
        d.copy_(h, non_blocking=True)
    c.softmax(tuple(din), rows, cols, out=out)
    for h, o in zip(hz, out):
        h.copy_(o, non_blocking=True)


ms = timeit(seq)
print(f"sequential       {ms:.4f} ms  {rows * cols / ms / 1e6:.3f} G el/s")
for slots in (4, 8, 12, 16):
    os.environ["MPC_HIO_SLOTS"] = str(slots)          # read when a context creates its pipeline
    cs = m.Ctx.for_cfg(workloads.keys(2))
    for ch in (0, 768, 1024, 1536, 2048, 3072):
        ms = timeit(lambda: cs.softmax_hostio(hx, hz, rows, cols, chunk_rows=ch))
        print(f"hostio slots {slots:2d} chunk {ch:5d} {ms:.4f} ms  {rows * cols / ms / 1e6:.3f} G el/s")
ms = timeit(lambda: c.softmax(x, rows, cols, out=out))
print(f"device only      {ms:.4f} ms")
for r in (512, 1024, 2048, 3072, 4096, 6144):
    xs = tuple(t[: r * cols] for t in x)
    os_ = tuple(t[: r * cols] for t in out)
    ms = timeit(lambda: c.softmax(xs, r, cols, out=os_))
    print(f"device only {r:5d} rows ({r // 32:3d} tiles) {ms:.4f} ms")
h2d = timeit(lambda: [d.copy_(h, non_blocking=True) for d, h in zip(din, hx)])
d2h = timeit(lambda: [h.copy_(o, non_blocking=True) for h, o in zip(hz, out)])
print(f"H2D 2x{hx[0].numel() * 8 / 1e6:.1f} MB {h2d:.4f} ms ({2 * hx[0].numel() * 8 / h2d / 1e6:.1f} GB/s); D2H {d2h:.4f} ms")
