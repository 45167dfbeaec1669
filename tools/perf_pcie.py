"""PCIe copy microbenchmark: H2D alone, D2H alone and both directions concurrently (separate
streams, pinned host memory) -- the ceiling of the host-buffer e2e path."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

MB = 1 << 20


def run(nbytes, reps=10):
    n = nbytes // 8
    hs = torch.empty(n, dtype=torch.int64).pin_memory()
    hd = torch.empty(n, dtype=torch.int64).pin_memory()
    ds = torch.empty(n, dtype=torch.int64, device="cuda")
    dd = torch.empty(n, dtype=torch.int64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    main = torch.cuda.current_stream()

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main)
        for _ in range(reps):
            fn()
        b.record(main)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    def h2d():
        ds.copy_(hs, non_blocking=True)

    def d2h():
        hd.copy_(dd, non_blocking=True)

    def both():
        ev = torch.cuda.Event()
        ev.record(main)
        s1.wait_event(ev); s2.wait_event(ev)
        with torch.cuda.stream(s1):
            ds.copy_(hs, non_blocking=True)
        with torch.cuda.stream(s2):
            hd.copy_(dd, non_blocking=True)
        main.wait_stream(s1); main.wait_stream(s2)

    t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
    gb = nbytes / 1e9
    print(f"{nbytes / MB:7.1f} MB  H2D {t1:.4f} ms {gb / t1 * 1e3:6.1f} GB/s   D2H {t2:.4f} ms {gb / t2 * 1e3:6.1f} GB/s"
          f"   both {t3:.4f} ms ({2 * gb / t3 * 1e3:6.1f} GB/s aggregate; serial would be {t1 + t2:.4f})")


for mb in (3, 6, 12, 25, 100):
    run(int(mb * MB))


def chunked(nbytes=25 * MB, nchunks=8, with_kernel=False, reps=10):
    """Both directions concurrently, each as nchunks copies (the hostio pattern), optionally with a
    softmax kernel running on a third stream."""
    n = nbytes // 8
    hs = torch.empty(n, dtype=torch.int64).pin_memory()
    hd = torch.empty(n, dtype=torch.int64).pin_memory()
    ds = torch.empty(n, dtype=torch.int64, device="cuda")
    dd = torch.empty(n, dtype=torch.int64, device="cuda")
    s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    main = torch.cuda.current_stream()
    k = None
    if with_kernel:
        import paper_2511_19711_b200 as m
        import workloads
        c = m.Ctx.for_cfg(workloads.keys(2))
        rows, cols = 12288, 128
        xs = c.share(torch.from_numpy(workloads.softmax_inputs(rows, cols)).cuda())
        out = c._empty(rows * cols)
        k = (c, xs, out, rows, cols)
    step = n // nchunks

    def both():
        ev = torch.cuda.Event()
        ev.record(main)
        for s in (s1, s2, s3):
            s.wait_event(ev)
        with torch.cuda.stream(s1):
            for i in range(nchunks):
                ds[i * step:(i + 1) * step].copy_(hs[i * step:(i + 1) * step], non_blocking=True)
        with torch.cuda.stream(s2):
            for i in range(nchunks):
                hd[i * step:(i + 1) * step].copy_(dd[i * step:(i + 1) * step], non_blocking=True)
        if k:
            with torch.cuda.stream(s3):
                c, xs, out, rows, cols = k
                for _ in range(2):
                    c.softmax(xs, rows, cols, out=out)
        for s in (s1, s2, s3):
            main.wait_stream(s)

    for _ in range(3):
        both()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(main)
    for _ in range(reps):
        both()
    b.record(main)
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / reps
    print(f"both directions {nbytes / MB:.0f} MB as {nchunks} copies{' + softmax x2' if k else ''}: {t:.4f} ms "
          f"({2 * nbytes / t / 1e6:.1f} GB/s aggregate)")


for nch in (1, 4, 8, 16):
    chunked(nchunks=nch)
chunked(nchunks=8, with_kernel=True)
