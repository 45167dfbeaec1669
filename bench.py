#!/usr/bin/env python
"""bench.py -- secret-shared elements/s of the 2-party nonlinear-operator path on B200.

Step = one mpc_softmax over BASELINE config 2 (BERT-base attention softmax,
8 x 12 x 128 x 128 scores, exp-limit t=8 + Newton-Raphson reciprocal 10 iters,
window 33) for both parties.  N = 1: one GPU holds both parties (MPC_MODE_BOTH).
N > 1 (torchrun): every rank runs its own batch shard (global row offset
rank * rows, weak scaling, no data-path collective).
Also reported (`per_op`): GELU over config 3 (8x128x3072, |x|-form deg 4) and
ReLU over one 8-image shard of ResNet-50's first ReLU layer (config 4).

--impl reference times the CPU oracle (oracle/, plain C, 1 thread) on a bounded
sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

METRIC = "secret-shared elements/s per op (Softmax, GELU, ReLU) at 1/2/4/8 B200; % HBM roofline"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
SM_COUNT, SMSP, LANES = 148, 4, 32
# Philox4x32-10 = 10 rounds x (2 IMAD.WIDE.U32 + 2 LOP3); IMAD on the fma pipe and LOP3 on the
# alu pipe each take 2 cycles per warp instruction (B300_MICROARCH "Pipe rates"): 40 pipe-cycles
# per 32 blocks per SMSP on either pipe.  Peak = 148 * 4 * 32 / 40 * f_max.
CYCLES_PER_WARP_BLOCK = 40.0


def load_peaks():
    try:
        return json.load(open(PEAKS_PATH))
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "_fallback": True}


def philox_peak_gblocks(sm_mhz):
    return SM_COUNT * SMSP * LANES / CYCLES_PER_WARP_BLOCK * sm_mhz * 1e6 / 1e9


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([v.strip() for v in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows if len(r) >= 9 for k in range(4)
                          if r[5 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------- mpc200 arm ----
def run_mpc200(args):
    import torch
    import torch.distributed as dist
    import paper_2511_19711_b200 as m

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    keys = workloads.keys(2)
    rows, cols = workloads.SHAPES["cfg2_softmax"]
    n = rows * cols
    row_off = rank * rows                      # this rank's global batch shard
    ctx = m.Ctx.for_cfg(keys, device=local)
    stream = torch.cuda.current_stream(dev)

    # inputs: shares of synthetic scores (sharing is setup, not timed: SURVEY 8(d))
    x = workloads.softmax_inputs(rows, cols)
    xs = ctx.share(torch.from_numpy(x).to(dev), off=row_off * cols)
    out = (torch.empty_like(xs[0]), torch.empty_like(xs[1]))
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)   # 512 MB > 126 MB L2
    sm_kw = dict(window=33, exp_t=8, exp_clamp=0, recip_iters=10, recip_t=8)

    def step():
        ctx.softmax(xs, rows, cols, row_off=row_off, out=out, **sm_kw)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, per-step events, L2 flushed between steps ----
    ctx.reset_stats()
    ctx.enable_kernel_timing(True)
    ctx.kernel_times()
    clocks = Clocks(local)
    clocks.start()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        flush.fill_(k)
        evs[k][0].record(stream)
        step()
        evs[k][1].record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = sum(a.elapsed_time(b) for a, b in evs)
    st = ctx.stats()
    ktimes = ctx.kernel_times()
    ctx.enable_kernel_timing(False)
    if ws > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = ws * n / (ms_step / 1e3)

    # ---- roofline of the dominant kernel (ALU bound: Philox blocks) ----
    agg = {}
    for name, kms, ph, _u in ktimes:
        a = agg.setdefault(name, [0.0, 0, 0])
        a[0] += kms; a[1] += ph; a[2] += 1
    tot = sum(v[0] for v in agg.values()) or 1.0
    dom = max(agg, key=lambda k: agg[k][0])
    peaks = load_peaks()
    fmax = float(peaks.get("sm_max_mhz", 1965.0))
    peak = philox_peak_gblocks(fmax)
    ach = agg[dom][1] / (agg[dom][0] / 1e3) / 1e9
    roof = {"bound": "alu", "kernel": dom, "achieved": round(ach, 2), "peak": round(peak, 2),
            "unit": "Gphilox/s", "frac": round(ach / peak, 4), "traffic": None,
            "share_of_step": round(agg[dom][0] / tot, 3), "launches_per_step": agg[dom][2] // args.steps,
            "peak_basis": f"148 SM x 4 SMSP x 32 lanes / 40 cycles per warp-block x {fmax:.0f} MHz "
                          f"({'measured' if not peaks.get('_fallback') else 'fallback'} sm_max)",
            "step_philox_frac": round(st["philox_calls"] / args.steps / (ms_step / 1e3) / 1e9 / peak, 4),
            "kernels": {k: {"ms_per_step": round(v[0] / args.steps, 4), "gphilox_s": round(v[1] / (v[0] / 1e3) / 1e9, 2) if v[0] else None}
                        for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])}}
    hbm_bytes = 32 * n     # BOTH: read x0,x1 + write z0,z1 (algorithmic)
    roof["hbm_frac"] = round(hbm_bytes / (ms_step / 1e3) / 1e9 / float(peaks.get("hbm_gbs", 6650.0)), 5)

    # ---- e2e: host buffers through the public API (H2D inputs, D2H outputs inside the region) ----
    h0 = xs[0].cpu().pin_memory(); h1 = xs[1].cpu().pin_memory()
    o0 = torch.empty_like(h0).pin_memory(); o1 = torch.empty_like(h1).pin_memory()
    d0, d1 = torch.empty_like(xs[0]), torch.empty_like(xs[1])
    e2e_steps = max(3, min(args.steps, 10))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ea.record(stream)
    for _ in range(e2e_steps):
        d0.copy_(h0, non_blocking=True); d1.copy_(h1, non_blocking=True)
        ctx.softmax((d0, d1), rows, cols, row_off=row_off, out=out, **sm_kw)
        o0.copy_(out[0], non_blocking=True); o1.copy_(out[1], non_blocking=True)
    eb.record(stream)
    torch.cuda.synchronize()
    e_ms = ea.elapsed_time(eb) / e2e_steps
    if ws > 1:
        t = torch.tensor([e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item())

    # ---- per-op lines (GELU cfg3, ReLU cfg4 shard), same timing rules ----
    per_op = {"softmax": {"elements": n, "elements_per_s": value / ws, "ms": round(ms_step, 4)}}
    if not args.no_per_op:
        per_op.update(time_per_op(m, ctx, dev, stream, flush, args, rank))

    res = None
    if rank == 0:
        res = {"metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": ws, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
               "config": {"workload": "cfg2: BERT-base attention softmax 8x12x128x128 (2-party, Z_2^64, f=16)",
                          "rows": rows, "cols": cols, "exp": "limit t=8", "recip": "NR 10 iters (exp t=8)",
                          "window": 33, "mode": "BOTH (1 GPU holds both parties)" if ws == 1 else
                          f"BOTH per rank, batch-sharded x{ws}", "l2": "flushed between steps (512 MB write)",
                          "parallelism": f"dp{ws}"},
               "roofline": roof,
               "e2e": {"value": ws * n / (e_ms / 1e3), "unit": "elements/s",
                       "h2d_bytes_per_step": 16 * n, "d2h_bytes_per_step": 16 * n,
                       "ms_per_step": round(e_ms, 4)},
               "gpu_launches": st["launches"],
               "launches_per_step": st["launches"] / args.steps,
               "protocol_per_step": {"philox_blocks": st["philox_calls"] // args.steps,
                                     "bytes_per_party": st["bytes_per_party"] // args.steps,
                                     "rounds": st["rounds"] // args.steps},
               "clocks": clk, "per_op": per_op}
        if not args.no_cpu_baseline:
            res["cpu_baseline"] = cpu_baseline(args)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return res


def time_per_op(m, ctx, dev, stream, flush, args, rank):
    import torch
    out = {}
    # GELU cfg3 (|x|-form deg 4, B=3: the paper's BOLT structure)
    n3 = workloads.SHAPES["cfg3_gelu"]
    g = ctx.share(torch.from_numpy(workloads.normal_inputs(n3, 3)).to(dev), off=rank * n3)
    z = (torch.empty_like(g[0]), torch.empty_like(g[1]))
    knobs = m.default_act("gelu", "poly_abs", degree=4)
    fn = lambda: ctx._act(m.binding._L.mpc_gelu, "mpc_gelu", g, rank * n3, knobs, z)  # noqa: E731
    out["gelu"] = _time(fn, n3, ctx, flush, stream, args)
    out["gelu"]["config"] = "cfg3: BERT-base FFN 8x128x3072, |x|-form deg 4, B=3"
    del g, z
    # ReLU: one 8-image shard of ResNet-50's first ReLU layer (32x64x112x112 / 4 pairs)
    N, C, H, W = workloads.SHAPES["cfg4_relu_first"]
    n4 = N * C * H * W // 4
    r = ctx.share(torch.from_numpy(workloads.relu_inputs(n4)).to(dev), off=rank * n4)
    z = (torch.empty_like(r[0]), torch.empty_like(r[1]))
    out["relu"] = _time(lambda: ctx.relu(r, off=rank * n4, out=z), n4, ctx, flush, stream, args)
    out["relu"]["config"] = "cfg4: ResNet-50 first ReLU, 8 images x 64 x 112 x 112, window 33"
    del r, z
    # LayerNorm: GPT-2 small, 8 x 1024 tokens x 768 (cfg5), rsqrt 3 iters (exp t=8)
    rows5, cols5 = workloads.SHAPES["cfg5_ln"]
    ln = ctx.share(torch.from_numpy(workloads.layernorm_inputs(rows5, cols5)).to(dev), off=rank * rows5 * cols5)
    z = (torch.empty_like(ln[0]), torch.empty_like(ln[1]))
    out["layernorm"] = _time(lambda: ctx.layernorm(ln, rows5, cols5, row_off=rank * rows5, out=z),
                             rows5 * cols5, ctx, flush, stream, args)
    out["layernorm"]["config"] = "cfg5: GPT-2 LayerNorm 8192 x 768, rsqrt 3 iters, mean x E(1/d)"
    del ln, z
    # GPT-2 softmax rows (1024 wide), 1/8 of one layer's 8x12x1024x1024 scores
    rs, cs = 8 * 12 * 128, 1024
    sm = ctx.share(torch.from_numpy(workloads.softmax_inputs(rs, cs, seed_cfg=5)).to(dev), off=rank * rs * cs)
    z = (torch.empty_like(sm[0]), torch.empty_like(sm[1]))
    out["softmax1024"] = _time(lambda: ctx.softmax(sm, rs, cs, row_off=rank * rs, out=z), rs * cs, ctx, flush,
                               stream, args)
    out["softmax1024"]["config"] = "cfg5: GPT-2 softmax rows of 1024 (12288 rows = 1/8 layer), t=8, NR 10"
    del sm, z
    # Beaver multiply alone (S4), 16M elements
    nm = 1 << 24
    a = ctx.share(torch.from_numpy(workloads.act_inputs(nm)).to(dev))
    b = ctx.share(torch.from_numpy(workloads.act_inputs(nm, seed_cfg=7)).to(dev))
    z = (torch.empty_like(a[0]), torch.empty_like(a[1]))
    out["mul"] = _time(lambda: ctx.mul(a, b, trunc_bits=16, out=z), nm, ctx, flush, stream, args)
    out["mul"]["config"] = "Beaver multiply + trunc, 16M elements"
    return out


def _time(fn, n, ctx, flush, stream, args):
    import torch
    for _ in range(max(1, args.warmup)):
        fn()
    torch.cuda.synchronize()
    ctx.enable_kernel_timing(True)
    ctx.kernel_times()
    ph0 = ctx.stats()["philox_calls"]
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for k in range(args.steps):
        flush.fill_(k)
        evs[k][0].record(stream)
        fn()
        evs[k][1].record(stream)
    torch.cuda.synchronize()
    kt = ctx.kernel_times()
    ctx.enable_kernel_timing(False)
    ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
    ph = (ctx.stats()["philox_calls"] - ph0) / args.steps
    peak = philox_peak_gblocks(float(load_peaks().get("sm_max_mhz", 1965.0)))
    kms = sum(t[1] for t in kt) / args.steps
    return {"elements": n, "elements_per_s": n / (ms / 1e3), "ms": round(ms, 4),
            "gphilox_s": round(ph / (kms / 1e3) / 1e9, 2), "alu_frac": round(ph / (kms / 1e3) / 1e9 / peak, 4)}


# ------------------------------------------------------------------------ CPU oracle ----
def _oracle_softmax_sample(rows_s):
    from oracle import Oracle
    rows, cols = workloads.SHAPES["cfg2_softmax"]
    keys = workloads.keys(2)
    x = workloads.softmax_inputs(rows, cols)[:rows_s]
    o = Oracle.for_cfg(keys)
    s = o.share(x)
    t0 = time.perf_counter()
    o.softmax(s, rows_s, cols)
    return time.perf_counter() - t0


def cpu_baseline(args):
    """The oracle as it stands (plain C, 1 thread) on a bounded sample of cfg2."""
    rows, cols = workloads.SHAPES["cfg2_softmax"]
    rows_s = int(os.environ.get("MPC_CPU_SAMPLE_ROWS", "2048"))
    dt = _oracle_softmax_sample(rows_s)
    return {"value": rows_s * cols / dt, "unit": "elements/s", "cores": 1, "kind": "oracle",
            "sample": f"{rows_s} of {rows} rows of cfg2 softmax ({rows_s * cols} elements), 1 pass, {dt:.2f} s",
            "host_cpus": os.cpu_count()}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return None
    rows, cols = workloads.SHAPES["cfg2_softmax"]
    # size each step so that warmup + steps finish in ~2 minutes
    dt32 = _oracle_softmax_sample(32)
    per_row = dt32 / 32
    budget = float(os.environ.get("MPC_REF_BUDGET_S", "120"))
    rows_s = int(max(32, min(rows, budget / (args.steps + args.warmup) / per_row)) // 32 * 32)
    for _ in range(args.warmup):
        _oracle_softmax_sample(rows_s)
    ts = [_oracle_softmax_sample(rows_s) for _ in range(args.steps)]
    ms = 1e3 * sum(ts) / len(ts)
    v = rows_s * cols / (ms / 1e3)
    sample = f"{rows_s} of {rows} rows of cfg2 softmax per step (oracle/, plain C, 1 thread)"
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": "elements/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": "cfg2: BERT-base attention softmax 8x12x128x128 (2-party, Z_2^64, f=16)",
                       "rows": rows, "cols": cols, "sample_rows": rows_s},
            "cpu_baseline": {"value": v, "unit": "elements/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="mpc200", choices=["mpc200", "reference"])
    ap.add_argument("--no-per-op", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    res = run_reference(args) if args.impl == "reference" else run_mpc200(args)
    if res is not None:
        print(json.dumps(res))


if __name__ == "__main__":
    main()
