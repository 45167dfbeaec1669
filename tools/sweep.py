#!/usr/bin/env python
"""Per-row / per-config measurement sweep (MPC_MODE_BOTH, cuda:0).

Every row of SURVEY.md §8(a) and every BASELINE.json config is timed here with the same
rules as bench.py (CUDA events on the ctx stream, L2 flushed between steps by a 512 MB
write, warm-up first) and reported with its protocol cost (Philox blocks, bytes per party
and rounds a PAIR execution would send) and its integer-ALU roofline fraction.
bench.py keeps the headline (cfg2 softmax) and a compact per_op; this tool writes the full
table:  python tools/sweep.py [--steps K] [--out gpurun_out/sweep.json] [--only cfg3,...]

Sections
  rows    S1..S15 at a common size (one line per ABI entry point, default knobs)
  cfg1    4096 elements: exp t in {8, 8+clamp, 4, 2, 0+clamp}, reciprocal 10 it, GELU forms (us/call)
  cfg2    BERT-base softmax 8x12x128x128: default, +clamp, spike rows, NEXT variants
  cfg3    BERT-base FFN GELU 8x128x3072: x-form deg 4/2 (B=5), |x|-form deg 4/2 (B=3), ReLU, erf K 4/6/8
  cfg4    ResNet-50 v1.5 batch-32 shard of one pair (8 images): all 49 ReLU layers as one pass,
          first ReLU layer, MaxPool 3x3/2 pad 1; windows 33 vs HummingBird-style 21
  cfg5    GPT-2 small layer set for one pair's shard (2 sequences x 1024): LN1, softmax, LN2, GELU per
          layer x 12 + final LN, under three synthetic knob schedules
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_19711_b200 as m  # noqa: E402
import workloads  # noqa: E402

# ResNet-50 v1.5 at 224x224: ReLU output shapes (C, H, W) per image, in network order.
# stem 1; layer1 3 blocks x 3 ReLU at 56^2 (64, 64, 256); layer2 4 blocks (first block's
# first ReLU at 56^2 -- v1.5 puts the stride on the 3x3); layer3 6; layer4 3.
def resnet50_relu_shapes():
    s = [(64, 112, 112)]
    def stage(blocks, width, out, hw_in, hw):
        for b in range(blocks):
            s.append((width, hw_in if b == 0 else hw, hw_in if b == 0 else hw))
            s.append((width, hw, hw))
            s.append((out, hw, hw))
    stage(3, 64, 256, 56, 56)
    stage(4, 128, 512, 56, 28)
    stage(6, 256, 1024, 28, 14)
    stage(3, 512, 2048, 14, 7)
    return s


class Sweep:
    def __init__(self, steps, warmup):
        self.job = bench.Job(m, torch, torch.distributed)
        self.args = argparse.Namespace(steps=steps, warmup=warmup)
        self.flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.int32, device=self.job.dev)
        self.ctxs = {}

    def ctx(self, cfg):
        if cfg not in self.ctxs:
            self.ctxs[cfg] = self.job.ctx(cfg)
        return self.ctxs[cfg]

    def share(self, c, x):
        return self.job.share(c, x, 0)

    def line(self, c, fn, n, config, circuit=0):
        c.set_ltz_circuit(circuit)
        try:
            r = bench._op_line(self.job, c, fn, n, self.flush, self.args, config)
        finally:
            c.set_ltz_circuit(0)
        r["us_per_call"] = round(r["ms"] * 1e3, 2)
        return r


def sec_rows(S):
    c = S.ctx(1)
    n = 1 << 22
    out = {}
    x = S.share(c, workloads.act_inputs(n))
    y = S.share(c, workloads.act_inputs(n, seed_cfg=7))
    z = c._empty(n)
    xf = torch.from_numpy(workloads.act_inputs(n)).to(S.job.dev)
    out["S1_share"] = S.line(c, lambda: c.share(xf, owner=0), n, "encode + share 4M f64 values")
    out["S2_open"] = S.line(c, lambda: c.open(x), n, "open + decode 4M (ring and f64 outputs)")
    out["S4_mul"] = S.line(c, lambda: c.mul(x, y, trunc_bits=0, out=z), n, "Beaver multiply 4M, no trunc")
    out["S4_mul_trunc"] = S.line(c, lambda: c.mul(x, y, trunc_bits=16, out=z), n, "Beaver multiply + trunc 4M")
    yr = S.share(c, workloads.recip_inputs(n // 128))
    out["S4_mul_bcast"] = S.line(c, lambda: c.mul_bcast(x, yr, n // 128, 128, trunc_bits=16, out=z), n,
                                 "broadcast-triple multiply 32768 x 128 by a per-row factor (NEXT #2)")
    out["S4_square"] = S.line(c, lambda: c.square(x, trunc_bits=16, out=z), n, "square-pair triple 4M (NEXT #2)")
    out["S5_trunc"] = S.line(c, lambda: c.trunc(x, 16, out=z), n, "local truncation 4M")
    for w in (33, 64):
        out[f"S7_cmp_w{w}"] = S.line(c, lambda w=w: c.cmp(x, window=w, out=z), n, f"LTZ window {w}, 4M")
        out[f"S7_cmp_w{w}_cone"] = S.line(c, lambda w=w: c.cmp(x, window=w, out=z), n,
                                          f"LTZ window {w}, carry cone, 4M", circuit=1)
    out["S8_relu"] = S.line(c, lambda: c.relu(x, out=z), n, "ReLU w33, 4M")
    rows, cols = 32768, 128
    mx = S.share(c, workloads.softmax_inputs(rows, cols, seed_cfg=1))
    zr = c._empty(rows)
    out["S9_max"] = S.line(c, lambda: c.max(mx, rows, cols, out=zr), rows * cols, "row max 32768 x 128")
    e = S.share(c, workloads.exp_inputs(n))
    out["S10_exp_t8"] = S.line(c, lambda: c.exp(e, out=z), n, "exp t=8, 4M")
    out["S10_exp_t8_clamp"] = S.line(c, lambda: c.exp(e, clamp=1, out=z), n, "exp t=8+clamp, 4M")
    rc = S.share(c, workloads.recip_inputs(n))
    out["S11_recip"] = S.line(c, lambda: c.recip(rc, out=z), n, "reciprocal NR 10 it (exp t=8), 4M")
    rq = S.share(c, workloads.rsqrt_inputs(n))
    out["S12_rsqrt"] = S.line(c, lambda: c.rsqrt(rq, out=z), n, "rsqrt NR 3 it (exp t=8), 4M")
    a = S.share(c, workloads.act_inputs(n, lo=-8.0, hi=8.0))
    out["S13_gelu_abs4"] = S.line(c, lambda: c.gelu(a, form="poly_abs", degree=4, out=z), n, "GELU |x|-form deg 4, 4M")
    out["S13_silu_abs4"] = S.line(c, lambda: c.silu(a, form="poly_abs", degree=4, out=z), n, "SiLU |x|-form deg 4, 4M")
    out["S13_sigmoid_x4"] = S.line(c, lambda: c.sigmoid(a, form="poly_x", degree=4, out=z), n,
                                   "Sigmoid x-form deg 4, 4M")
    sm = S.share(c, workloads.softmax_inputs(rows, cols, seed_cfg=1))
    zs = c._empty(rows * cols)
    out["S14_softmax"] = S.line(c, lambda: c.softmax(sm, rows, cols, out=zs), rows * cols, "softmax 32768 x 128")
    ln = S.share(c, workloads.layernorm_inputs(4096, 1024, seed_cfg=1))
    zl = c._empty(4096 * 1024)
    out["S15_layernorm"] = S.line(c, lambda: c.layernorm(ln, 4096, 1024, out=zl), 4096 * 1024,
                                  "layernorm 4096 x 1024, rsqrt 3 it")
    return out


def graph_us_per_call(fn, calls=20, replays=10):
    """Device-side latency of one call: `calls` calls captured into one CUDA graph (the library's
    launches are stream-capturable), replayed; us per call.  Replays reuse the captured step ids,
    so this is a timing device only (never reuse randomness in a real protocol run)."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()                                            # warm-up: scratch allocated, occupancy cached
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(calls):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(replays):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) * 1e3 / (replays * calls), 2)


def sec_cfg1(S):
    c = S.ctx(1)
    n = workloads.SHAPES["cfg1_elems"]
    out = {}
    e = S.share(c, workloads.exp_inputs(n, tail_frac=0.05))
    z = c._empty(n)
    for t, cl in ((8, 0), (8, 1), (4, 0), (2, 0), (2, 1), (0, 1)):
        out[f"exp_t{t}{'_clamp' if cl else ''}"] = S.line(c, lambda t=t, cl=cl: c.exp(e, t=t, clamp=cl, out=z), n,
                                                          f"cfg1 exp-limit t={t}{'+clamp' if cl else ''}, 4096")
    r = S.share(c, workloads.recip_inputs(n))
    out["recip_10"] = S.line(c, lambda: c.recip(r, out=z), n, "cfg1 reciprocal NR 10 it, 4096")
    a = S.share(c, workloads.act_inputs(n))
    for form, deg in (("poly_x", 4), ("poly_abs", 4), ("erf", 8), ("relu", 0)):
        out[f"gelu_{form}{deg}"] = S.line(c, lambda form=form, deg=deg: c.gelu(a, form=form, degree=deg,
                                                                             erf_terms=8, out=z),
                                          n, f"cfg1 GELU {form} deg {deg}, 4096")
    # the same calls replayed from a CUDA graph: device latency without the host launch path
    fns = {"exp_t8": lambda: c.exp(e, t=8, out=z), "exp_t8_clamp": lambda: c.exp(e, t=8, clamp=1, out=z),
           "exp_t2_clamp": lambda: c.exp(e, t=2, clamp=1, out=z), "recip_10": lambda: c.recip(r, out=z),
           "gelu_poly_abs4": lambda: c.gelu(a, form="poly_abs", degree=4, out=z),
           "gelu_erf8": lambda: c.gelu(a, form="erf", erf_terms=8, out=z)}
    for k, fn in fns.items():
        out[k]["us_per_call_graph"] = graph_us_per_call(fn)
    return out


def sec_cfg2(S):
    c = S.ctx(2)
    rows, cols = workloads.SHAPES["cfg2_softmax"]
    n = rows * cols
    out = {}
    x = S.share(c, workloads.softmax_inputs(rows, cols))
    xs = S.share(c, workloads.softmax_inputs(rows, cols, spike=True))
    z = c._empty(n)
    out["softmax_t8"] = S.line(c, lambda: c.softmax(x, rows, cols, out=z), n, "cfg2 t=8, NR 10 (headline)")
    out["softmax_t8_clamp"] = S.line(c, lambda: c.softmax(x, rows, cols, exp_clamp=1, out=z), n, "cfg2 t=8+clamp")
    out["softmax_t8_spike"] = S.line(c, lambda: c.softmax(xs, rows, cols, out=z), n, "cfg2 +6 spike rows")
    out["softmax_t2_clamp"] = S.line(c, lambda: c.softmax(x, rows, cols, exp_t=2, exp_clamp=1, out=z), n,
                                     "cfg2 t=2+clamp (moderate)")
    out["softmax_t0_clamp"] = S.line(c, lambda: c.softmax(x, rows, cols, exp_t=0, exp_clamp=1, out=z), n,
                                     "cfg2 t=0+clamp (aggressive)")
    out["softmax_cone"] = S.line(c, lambda: c.softmax(x, rows, cols, out=z), n, "cfg2 carry cone", circuit=1)
    out["softmax_cone_square"] = S.line(c, lambda: c.softmax(x, rows, cols, exp_square=1, recip_square=1, out=z),
                                        n, "cfg2 carry cone + square triples", circuit=1)
    out["softmax_bcast"] = S.line(c, lambda: c.softmax(x, rows, cols, bcast=1, out=z), n, "cfg2 broadcast triple")
    out["softmax_next_all"] = S.line(c, lambda: c.softmax(x, rows, cols, exp_square=1, recip_square=1, bcast=1,
                                                          out=z), n, "cfg2 cone + square + broadcast", circuit=1)
    return out


def sec_cfg3(S):
    c = S.ctx(3)
    n = workloads.SHAPES["cfg3_gelu"]
    out = {}
    g = S.share(c, workloads.normal_inputs(n, 3))
    z = c._empty(n)
    for form, deg in (("poly_x", 4), ("poly_x", 2), ("poly_abs", 4), ("poly_abs", 2), ("relu", 0)):
        out[f"gelu_{form}{deg}"] = S.line(c, lambda form=form, deg=deg: c.gelu(g, form=form, degree=deg, out=z), n,
                                          f"cfg3 GELU {form} deg {deg}")
    for K in (4, 6, 8):
        out[f"gelu_erf{K}"] = S.line(c, lambda K=K: c.gelu(g, form="erf", erf_terms=K, out=z), n,
                                     f"cfg3 GELU erf-series K={K}, B=2.5")
    out["gelu_poly_abs4_cone"] = S.line(c, lambda: c.gelu(g, form="poly_abs", degree=4, out=z), n,
                                        "cfg3 GELU |x|-form deg 4, carry cone", circuit=1)
    out["gelu_poly_abs4_power"] = S.line(c, lambda: c.gelu(g, form="poly_abs", degree=4, basis=1, out=z), n,
                                         "cfg3 GELU |x|-form deg 4, power basis (NEXT #2)")
    out["gelu_poly_x4_power"] = S.line(c, lambda: c.gelu(g, form="poly_x", degree=4, basis=1, out=z), n,
                                       "cfg3 GELU x-form deg 4, power basis (NEXT #2)")
    return out


def sec_cfg4(S):
    c = S.ctx(4)
    out = {}
    per_img = sum(a * b * d for a, b, d in resnet50_relu_shapes())
    imgs = 8                                            # one pair's shard of batch 32 (4 pairs)
    n = per_img * imgs
    n = (n + 31) // 32 * 32
    r = S.share(c, workloads.relu_inputs(n))
    z = c._empty(n)
    out["relu_all49_w33"] = S.line(c, lambda: c.relu(r, out=z), n,
                                   f"cfg4 all 49 ReLU layers, 8 images ({per_img} per image), w33")
    out["relu_all49_w33_cone"] = S.line(c, lambda: c.relu(r, out=z), n, "cfg4 all 49 ReLU layers, carry cone",
                                        circuit=1)
    out["relu_all49_w21_cone"] = S.line(c, lambda: c.relu(r, window=21, out=z), n,
                                        "cfg4 all 49 ReLU layers, window 21 (HummingBird-style), carry cone",
                                        circuit=1)
    del r, z
    N, C, H, W = workloads.SHAPES["cfg4_maxpool_in"]
    N = imgs
    mp = S.share(c, workloads.maxpool_inputs((N, C, H, W)))
    no = N * C * 56 * 56
    zo = c._empty(no)
    out["maxpool_3x3s2"] = S.line(c, lambda: c.maxpool2d(mp, N, C, H, W, 3, 2, 1, out=zo), no,
                                  "cfg4 MaxPool 3x3/2 pad 1, 8 x 64 x 112^2 -> 56^2 (elements = outputs)")
    out["maxpool_3x3s2_cone"] = S.line(c, lambda: c.maxpool2d(mp, N, C, H, W, 3, 2, 1, out=zo), no,
                                       "cfg4 MaxPool, carry cone", circuit=1)
    return out


SCHEDULES = {
    # three synthetic per-layer knob schedules (the tuner is out of scope)
    "max_accuracy": lambda l: dict(sm=dict(exp_t=8, exp_clamp=1), gelu=dict(form="poly_abs", degree=4),
                                   ln1=dict(rsqrt_t=8), ln2=dict(rsqrt_t=8)),
    "moderate_like": lambda l: dict(sm=dict(exp_t=8 if l >= 8 else 2, exp_clamp=0 if l >= 8 else 1),
                                    gelu=dict(form="poly_abs", degree=4 if l < 6 else 2),
                                    ln1=dict(rsqrt_t=8), ln2=dict(rsqrt_t=0)),
    "aggressive": lambda l: dict(sm=dict(exp_t=0, exp_clamp=1), gelu=dict(form="relu", degree=0),
                                 ln1=dict(rsqrt_t=0), ln2=dict(rsqrt_t=0)),
}


def sec_cfg5(S):
    c = S.ctx(5)
    seqs, ctxlen, heads, d, ff = 2, 1024, 12, 768, 3072   # one pair's shard of batch 8 over 4 pairs
    rs, cs = seqs * heads * ctxlen, ctxlen
    rl = seqs * ctxlen
    ng = rl * ff
    sm = S.share(c, workloads.softmax_inputs(rs, cs, seed_cfg=5))
    ln = S.share(c, workloads.layernorm_inputs(rl, d))
    g = S.share(c, workloads.normal_inputs(ng, 5))
    zs, zl, zg = c._empty(rs * cs), c._empty(rl * d), c._empty(ng)
    out = {}
    n_layer = rs * cs + 2 * rl * d + ng
    for name, sched in SCHEDULES.items():
        def step(sched=sched):
            for l in range(12):
                k = sched(l)
                c.layernorm(ln, rl, d, out=zl, **k["ln1"])
                c.softmax(sm, rs, cs, out=zs, **k["sm"])
                c.layernorm(ln, rl, d, out=zl, **k["ln2"])
                c.gelu(g, out=zg, **k["gelu"])
            c.layernorm(ln, rl, d, out=zl)
        out[f"gpt2_12layers_{name}"] = S.line(c, step, 12 * n_layer + rl * d,
                                              f"cfg5 GPT-2 small 12 layers x (LN, softmax 24576x1024, LN, GELU "
                                              f"2048x3072) + final LN, 2 sequences, schedule {name}")
    # BASELINE cfg5 "per-layer auto-tuned approximation choices": the NEXT #4 tuner over the 49
    # layers, calibration samples per layer (score spread and LN row statistics vary with depth),
    # quality = summed per-layer max error vs the most accurate candidate, cost = measured MPC
    # time on this shard's shapes plus the paper's LAN model
    from paper_2511_19711_b200 import tuner as T
    dev = S.job.dev
    layers = []
    for l in range(12):
        sig = 1.0 + 0.25 * l
        layers.append(T.Layer(f"ln1_{l}", "layernorm", rl, d, torch.from_numpy(
            workloads.layernorm_inputs(64, d, seed_cfg=100 + l)).to(dev), 64))
        layers.append(T.Layer(f"attn_{l}", "softmax", rs, cs, torch.from_numpy(
            workloads.softmax_inputs(64, cs, seed_cfg=200 + l, sigma=sig)).to(dev), 64))
        layers.append(T.Layer(f"ln2_{l}", "layernorm", rl, d, torch.from_numpy(
            workloads.layernorm_inputs(64, d, seed_cfg=300 + l) * (0.5 + 0.1 * l)).to(dev), 64))
        layers.append(T.Layer(f"ffn_{l}", "gelu", 1, 8192, torch.from_numpy(
            workloads.normal_inputs(8192, 400 + l, sigma=sig)).to(dev), 1))
    ev = T.Evaluator(c, mpc_inputs={"softmax": (sm, rs), "layernorm": (ln, rl), "gelu": (g, 1)}, objective="lan")
    tuned = T.HillClimbTuner(layers, ev, threshold=0.25).run()
    knobs = tuned["knobs"]

    def step_tuned():
        for l in range(12):
            c.layernorm(ln, rl, d, out=zl, **knobs[f"ln1_{l}"])
            c.softmax(sm, rs, cs, out=zs, **knobs[f"attn_{l}"])
            c.layernorm(ln, rl, d, out=zl, **knobs[f"ln2_{l}"])
            c.gelu(g, out=zg, **knobs[f"ffn_{l}"])
        c.layernorm(ln, rl, d, out=zl)
    r = S.line(c, step_tuned, 12 * n_layer + rl * d, "cfg5 GPT-2 small 12 layers, per-layer knobs from the "
               "NEXT #4 hill-climbing tuner (LAN objective, summed max-error budget 0.25)")
    r["tuned"] = {"knobs": knobs, "quality_loss": tuned["quality_loss"], "lan_cost_ms": tuned["cost"],
                  "lan_cost_most_accurate_ms": tuned["cost_most_accurate"], "steps": tuned["steps"]}
    out["gpt2_12layers_autotuned"] = r
    out["softmax1024_t8"] = S.line(c, lambda: c.softmax(sm, rs, cs, out=zs), rs * cs, "cfg5 softmax layer, t=8 NR 10")
    out["softmax1024_t8_causal"] = S.line(c, lambda: c.softmax(sm, rs, cs, causal=1, out=zs), rs * cs,
                                          "cfg5 causal softmax layer (DESIGN.md 2.12), t=8 NR 10")
    out["gelu_poly_abs4"] = S.line(c, lambda: c.gelu(g, form="poly_abs", degree=4, out=zg), ng,
                                   "cfg5 GELU layer |x|-form deg 4")
    out["layernorm_r3"] = S.line(c, lambda: c.layernorm(ln, rl, d, out=zl), rl * d, "cfg5 LN 2048 x 768, rsqrt 3 it")
    return out


def sec_matmul(S):
    """NEXT #3 Beaver matmul on BERT-base shapes, SIMT vs tensor-core engine (same shares)."""
    c = S.ctx(2)
    out = {}
    for name, (B, M, K, N) in {"qkT_96x128x64x128": (96, 128, 64, 128), "av_96x128x128x64": (96, 128, 128, 64),
                               "ffn_1024x768x3072": (1, 1024, 768, 3072)}.items():
        x = S.share(c, workloads.act_inputs(B * M * K, lo=-2, hi=2))
        y = S.share(c, workloads.act_inputs(B * K * N, seed_cfg=5, lo=-2, hi=2))
        z = c._empty(B * M * N)
        for eng, tag in ((1, "simt"), (2, "tc")):
            c.set_matmul_engine(eng)
            r = S.line(c, lambda: c.matmul(x, y, B, M, K, N, trunc_bits=16, out=z), B * M * N,
                       f"Beaver matmul {name}, engine {tag} (elements = outputs)")
            r["ring_macs_per_s"] = B * M * K * N / (r["ms"] / 1e3)
            out[f"{name}_{tag}"] = r
        c.set_matmul_engine(0)
    return out


SECTIONS = {"rows": sec_rows, "cfg1": sec_cfg1, "cfg2": sec_cfg2, "cfg3": sec_cfg3, "cfg4": sec_cfg4,
            "cfg5": sec_cfg5, "matmul": sec_matmul}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--only", default="")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.json"))
    args = ap.parse_args()
    S = Sweep(args.steps, args.warmup)
    res = {"device": torch.cuda.get_device_name(0), "mode": "BOTH", "steps": args.steps, "warmup": args.warmup,
           "peak_gphilox_derived": round(bench.philox_peak_gblocks(1965.0), 2),
           "philox_peak_basis": "profiles/r02_microbench.json (IMAD.WIDE.U32 rate)", "philox_only_measured": bench.philox_only_measured(), "sections": {}}
    clocks = bench.Clocks(0)
    clocks.start()
    t0 = time.time()
    for name, fn in SECTIONS.items():
        if args.only and name not in args.only.split(","):
            continue
        res["sections"][name] = fn(S)
        torch.cuda.synchronize()
        print(f"[sweep] {name} done at {time.time() - t0:.1f}s", file=sys.stderr, flush=True)
    res["clocks"] = clocks.stop()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)
    for sec, d in res["sections"].items():
        for k, v in d.items():
            print(f"{sec:5s} {k:28s} {v['ms']:9.4f} ms {v['elements_per_s'] / 1e9:8.3f} Gel/s "
                  f"{v['gphilox_s']:7.1f} Gph/s  B/party {v['bytes_per_party']:>12d} rounds {v['rounds']}"
                  + (f"  graph {v['us_per_call_graph']} us/call" if "us_per_call_graph" in v else ""))


if __name__ == "__main__":
    main()
