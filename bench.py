#!/usr/bin/env python
"""bench.py -- secret-shared elements/s of the 2-party nonlinear-operator path on B200.

Step = one mpc_softmax over BASELINE config 2 (BERT-base attention softmax, 8 x 12 x
128 x 128 scores, exp-limit t=8 + Newton-Raphson reciprocal 10 iters (exp t=8), window 33).
  N = 1 : one GPU holds both parties (MPC_MODE_BOTH).
  N > 1 : (torchrun) ranks (2k, 2k+1) form party pair k (MPC_MODE_PAIR): every opening is
          exchanged between the pair's GPUs through NVLink peer memory inside the fused
          kernels; pair k processes batch shard k (global row offset k*rows) -- weak
          scaling, no inter-pair collective.  value = pairs x elements / max-over-ranks time.
Also reported (`per_op`): GELU (cfg3), ReLU (cfg4 shard), LayerNorm and 1024-wide softmax
(cfg5), Beaver multiply; at N = 1 also the PAIR protocol in loopback (both parties' kernels
on one GPU).  --impl reference times the CPU oracle (plain C, 1 thread) on a bounded sample.
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
# ALU roofline.  A Philox4x32-10 block is 10 rounds x (2 IMAD.WIDE.U32 + 2 LOP3).
# tools/microbench.cu (profiles/r02_microbench.json) measures IMAD.WIDE.U32 in isolation at one warp
# instruction per 4.04 cycles per SMSP (fmaheavy, quarter rate) and LOP3 at one per 2.02 on the alu
# pipe, the two overlapping: a block costs 20 x 4.04 = 80.7 fmaheavy cycles per warp, so
# peak = 148 SM x 4 SMSP x 32 lanes / 80.7 x f_max = 461 G blocks/s at 1965 MHz.
MICROBENCH_PATH = os.path.join(ROOT, "profiles", "r02_microbench.json")
IMADW_CYCLES_FALLBACK = 4.037
NVLINK_PEER_GBS = 770.0      # B200_PROFILING.md: measured peer copy per direction
# PAIR exchange wire bytes per payload byte: LL (format 0) sends every 8-byte payload word
# as two {half | round} words; LL63 (format 1, the MPC_MODE_PAIR default) sends 33 tagged words per 32
WIRE_FACTOR = {0: 2.0, 1: 33.0 / 32.0}


def imadw_cycles():
    try:
        return float(json.load(open(MICROBENCH_PATH))["derived"]["imad_wide_u32_cycles_per_warp_instr"])
    except Exception:
        return IMADW_CYCLES_FALLBACK


def philox_only_measured():
    try:
        return float(json.load(open(MICROBENCH_PATH))["derived"]["philox_only_best_measured_gblocks_s"])
    except Exception:
        return None


def load_peaks():
    try:
        return json.load(open(PEAKS_PATH))
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "_fallback": True}


def philox_peak_gblocks(sm_mhz):
    return SM_COUNT * SMSP * LANES / (20.0 * imadw_cycles()) * sm_mhz * 1e6 / 1e9


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
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
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
        ok = [r for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        sm = [float(r[1]) for r in ok]
        mx = [float(r[2]) for r in ok if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in ok for k in range(4) if r[5 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Job:
    """The run's layout: mode, party, pair index, and helpers that work in both modes."""

    def __init__(self, m, torch, dist):
        self.m, self.torch, self.dist = m, torch, dist
        self.ws, self.rank, self.local = dist_env()
        # MPC_BENCH_ONE_GPU=1 (validation only): every rank on cuda:0 with gloo for the host-side
        # collectives -- exercises the whole N > 1 path (pairs, cudaIpc exchange, max-over-ranks
        # timing, JSON) on a one-GPU box; the parties' kernels time-slice, so its numbers are not
        # throughput (tests/test_gpu_bench_pair.py)
        self.one_gpu = os.environ.get("MPC_BENCH_ONE_GPU") == "1"
        if self.one_gpu:
            self.local = 0
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        if self.ws > 1:
            if self.one_gpu:
                dist.init_process_group("gloo")
            else:
                # NCCL's own init lines (rank / nRanks per communicator) on stderr, so the driver's
                # scaling run can check the rank count; the JSON line stays alone on stdout
                os.environ.setdefault("NCCL_DEBUG", "INFO")
                os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
                dist.init_process_group("nccl", device_id=self.dev)
                print(f"[bench] rank {self.rank}: NCCL process group of {self.ws} ranks on cuda:{self.local}",
                      file=sys.stderr, flush=True)
            from paper_2511_19711_b200 import pair
            self.party, self.peer, self.pair_idx, self.npairs = pair.pair_layout(self.rank, self.ws)
            self.mode = m.binding.MODE_PAIR
        else:
            self.party, self.peer, self.pair_idx, self.npairs = 0, None, 0, 1
            self.mode = m.binding.MODE_BOTH
        self.stream = torch.cuda.current_stream(self.dev)
        self.dealer = None                 # PAIR party 1: the trusted dealer's offline context
        self.stream_words = 0              # correction words party 1 read in the last prefed block

    def ctx(self, cfg, mode=None):
        mode = self.mode if mode is None else mode
        keys = workloads.keys(cfg)
        if mode == self.m.binding.MODE_PAIR and self.party == 1 and os.environ.get("MPC_BENCH_DEALER", "1") == "1":
            # party 1 never receives K_0; the trusted dealer makes its
            # correction words OFFLINE, before each timed block (prefeed), on party 1's GPU
            self.dealer = self.m.Ctx.dealer(keys, device=self.local)
            keys = dict(keys, key_p0=0)
        c = self.m.Ctx.for_cfg(keys, device=self.local, mode=mode, party=self.party)
        if mode == self.m.binding.MODE_PAIR:
            from paper_2511_19711_b200 import pair
            pair.connect(c)
        return c

    def prefeed(self, ctx, fn, count):
        """PAIR party 1 with a dealer: the dealer runs the next `count` calls fn(c) offline (same
        shapes and step ids; it ignores the share pointers) and party 1 will read that stream."""
        if self.dealer is None or ctx.mode != self.m.binding.MODE_PAIR:
            return
        self.torch.cuda.synchronize()
        d = self.dealer
        d.dealer_reset()
        d.set_step(ctx.step, force=True)
        d.set_ltz_circuit(ctx.circuit)
        for _ in range(count):
            fn(d)
        stream = d.dealer_stream()
        self.stream_words = stream[1]
        ctx.set_corrections(stream)
        self.torch.cuda.synchronize()

    def share(self, ctx, x, off):
        """Party 0 owns the activations: in PAIR mode party 1 derives its share r
        from the pairwise key alone (no communication)."""
        xt = self.torch.from_numpy(np.ascontiguousarray(x).ravel()).to(self.dev)
        if ctx.mode == self.m.binding.MODE_PAIR and self.party == 1:
            return ctx.share(None, owner=0, off=off, n=xt.numel())
        return ctx.share(xt, owner=0, off=off)

    def maxr(self, v):
        if self.ws == 1:
            return v
        t = self.torch.tensor([v], device="cpu" if self.one_gpu else self.dev, dtype=self.torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def barrier(self):
        if self.ws > 1:
            self.dist.barrier()


def timed(job, ctx, fn, steps, flush, clocks=None):
    """K steps, CUDA events per step on the launching stream, L2 flushed between steps;
    returns (ms per step, max over ranks), kernel records, stats delta."""
    torch = job.torch
    ctx.reset_stats()
    ctx.enable_kernel_timing(True)
    ctx.kernel_times()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    job.barrier()
    torch.cuda.synchronize()
    if clocks:
        clocks.start()
    for k in range(steps):
        flush.fill_(k)
        evs[k][0].record(job.stream)
        fn()
        evs[k][1].record(job.stream)
    torch.cuda.synchronize()
    clk = clocks.stop() if clocks else None
    job.barrier()
    ms = sum(a.elapsed_time(b) for a, b in evs) / steps
    kt = ctx.kernel_times()
    ctx.enable_kernel_timing(False)
    st = ctx.stats()
    if ctx.mode != job.m.binding.MODE_BOTH:
        ctx.sync()                       # raises MPC_ERR_TIMEOUT if an exchange failed
    return job.maxr(ms), kt, st, clk


def roofline(job, ctx_mode, kt, st, steps, ms_step, n, xfmt=1):
    """Dominant kernel's achieved rate vs its roofline."""
    agg = {}
    for name, kms, ph, _u in kt:
        a = agg.setdefault(name, [0.0, 0, 0])
        a[0] += kms; a[1] += ph; a[2] += 1
    tot = sum(v[0] for v in agg.values()) or 1.0
    dom = max(agg, key=lambda k: agg[k][0])
    peaks = load_peaks()
    fmax = float(peaks.get("sm_max_mhz", 1965.0))
    peak = philox_peak_gblocks(fmax)
    dms = agg[dom][0] / agg[dom][2]                # average launch duration
    ach = (agg[dom][1] / agg[dom][2]) / (dms / 1e3) / 1e9
    traffic, tsrc = None, None
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        if dom in tj and ctx_mode == job.m.binding.MODE_BOTH:
            traffic, tsrc = tj[dom]["dram_bytes"], f"profiles/{tj[dom]['report']} (ncu --set full, one launch)"
    except Exception:
        pass
    r = {"bound": "alu", "kernel": dom, "achieved": round(ach, 2), "peak": round(peak, 2), "unit": "Gphilox/s",
         "frac": round(ach / peak, 4), "traffic": traffic, "traffic_source": tsrc,
         "traffic_algorithmic_bytes": 32 * n, "avg_launch_ms": round(dms, 4),
         "share_of_step": round(agg[dom][0] / tot, 3),
         "peak_basis": f"148 SM x 4 SMSP x 32 lanes / (20 IMAD.WIDE.U32 per block x {imadw_cycles():.3f} cycles, "
                       f"measured in isolation: profiles/r02_microbench.json) x {fmax:.0f} MHz "
                       f"({'measured' if not peaks.get('_fallback') else 'fallback'} sm_max, MEASURED_PEAKS.json)",
         "philox_only_measured": philox_only_measured(),
         "hbm_frac": round(32 * n / (ms_step / 1e3) / 1e9 / float(peaks.get("hbm_gbs", 6650.0)), 5)}
    if ctx_mode != job.m.binding.MODE_BOTH:
        bps = st["bytes_per_party"] / steps
        fmt = xfmt
        wps = bps * WIRE_FACTOR[fmt]
        r["nvlink"] = {"payload_bytes_per_party_per_step": int(bps), "wire_bytes_per_party_per_step": int(wps),
                       "wire_gbs": round(wps / (ms_step / 1e3) / 1e9, 2), "peak_gbs": NVLINK_PEER_GBS,
                       "wire_frac": round(wps / (ms_step / 1e3) / 1e9 / NVLINK_PEER_GBS, 4),
                       "payload_roofline_frac": round(bps / NVLINK_PEER_GBS / 1e9 / (ms_step / 1e3), 4),
                       "rounds_per_step": st["rounds"] // steps, "exchange_format": ["LL", "LL63"][fmt],
                       "wire_over_payload": WIRE_FACTOR[fmt]}
        r["note"] = ("PAIR: philox counts both parties + dealer (the BOTH-mode work) per pair; "
                     "each party's GPU executes its part plus party 1's dealer corrections")
    return r


# ---------------------------------------------------------------------------- mpc200 arm ----
def run_mpc200(args):
    import torch
    import torch.distributed as dist
    import paper_2511_19711_b200 as m

    job = Job(m, torch, dist)
    rows, cols = workloads.SHAPES["cfg2_softmax"]
    n = rows * cols
    row_off = job.pair_idx * rows                     # this pair's global batch shard
    ctx = job.ctx(2)
    xs = job.share(ctx, workloads.softmax_inputs(rows, cols), row_off * cols)
    out = ctx._empty(n)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.int32, device=job.dev)   # 512 MB > 126 MB L2
    sm_kw = dict(window=33, exp_t=8, exp_clamp=0, recip_iters=10, recip_t=8)

    def step(c=ctx):
        c.softmax(xs, rows, cols, row_off=row_off, out=out, **sm_kw)

    job.prefeed(ctx, step, args.warmup + args.steps)              # PAIR party 1: the dealer's offline pass
    stream_words_per_step = job.stream_words / max(1, args.warmup + args.steps)

    s_before = ctx.step
    for _ in range(args.warmup):
        step()
    steps_per_call = (ctx.step - s_before) // max(1, args.warmup)
    torch.cuda.synchronize()
    ms_step, kt, st, clk = timed(job, ctx, step, args.steps, flush, Clocks(job.local))
    value = job.npairs * n / (ms_step / 1e3)
    roof = roofline(job, ctx.mode, kt, st, args.steps, ms_step, n, ctx.exchange)
    if job.ws > 1:
        sw = job.maxr(stream_words_per_step)          # party 1's rank holds the stream
        roof["dealer"] = ({"party1_stream_bytes_per_step": int(8 * sw),
                           "party1_stream_hbm_frac": round(8 * sw / (ms_step / 1e3) / 1e9 /
                                                           float(load_peaks().get("hbm_gbs", 6650.0)), 5),
                           "how": "party 1 reads the trusted dealer's correction words (made offline before the "
                                  "timed block, DESIGN.md 7.1); its context has no K_0"}
                          if dealer_on(job) else {"simulated_by_party1": True})
    parity = check_timed_output(job, ctx.step - steps_per_call, xs, out, rows, cols, row_off, sm_kw)

    # ---- e2e: host buffers through the public API (H2D inputs, D2H outputs inside the region) ----
    # mpc_softmax_hostio: chunks of 1536 rows, H2D / compute / D2H of neighbouring chunks overlapped
    # on separate streams (tools/perf_e2e.py: 1.21 ms sequential -> 0.80 ms per cfg2 step)
    # both parties' shares in ONE pinned [2][n] host tensor each way, so a chunk's two party copies
    # are one pitched 2D DMA submission (copy_pair in mpc200.cu)
    def pinned_pair(src):
        live = [s for s in src if s is not None]
        buf = torch.empty((2, live[0].numel()), dtype=live[0].dtype).pin_memory()
        out = []
        for q, s in enumerate(src):
            if s is None:
                out.append(None)
            else:
                buf[q].copy_(s.reshape(-1).cpu())
                out.append(buf[q])
        return tuple(out)
    hin = pinned_pair(xs)
    hout = pinned_pair(tuple(torch.empty_like(s) if s is not None else None for s in xs))
    e2e_steps = max(3, min(args.steps, 10))
    job.prefeed(ctx, lambda c=ctx: c.softmax_hostio(hin, hout, rows, cols, row_off=row_off, chunk_rows=1536, **sm_kw),
                1 + e2e_steps)
    ctx.softmax_hostio(hin, hout, rows, cols, row_off=row_off, chunk_rows=1536, **sm_kw)    # warm-up
    job.barrier()
    torch.cuda.synchronize()
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ea.record(job.stream)
    for _ in range(e2e_steps):
        ctx.softmax_hostio(hin, hout, rows, cols, row_off=row_off, chunk_rows=1536, **sm_kw)
    eb.record(job.stream)
    torch.cuda.synchronize()
    e_ms = job.maxr(ea.elapsed_time(eb) / e2e_steps)
    pcie = pcie_floor(job, hin, hout)

    per_op = {"softmax": {"elements": n, "elements_per_s": value / job.npairs, "ms": round(ms_step, 4)}}
    if not args.no_per_op:
        per_op.update(time_per_op(job, m, ctx, flush, args))
        if job.ws == 1:
            per_op.update(time_loopback(job, m, flush, args))

    res = None
    if job.rank == 0:
        mode = ("BOTH (1 GPU holds both parties)" if job.ws == 1 else
                f"PAIR: {job.npairs} party pair(s), openings over NVLink peer memory, batch-sharded")
        res = {"metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": job.ws, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
               "config": {"workload": "cfg2: BERT-base attention softmax 8x12x128x128 (2-party, Z_2^64, f=16)",
                          "rows": rows, "cols": cols, "elements_per_pair": n, "exp": "limit t=8",
                          "recip": "NR 10 iters (exp t=8)", "window": 33, "mode": mode,
                          "l2": "flushed between steps (512 MB write)", "parallelism": f"pairs{job.npairs}"},
               "roofline": roof,
               "parity_ok": parity.get("ok"), "parity": parity,
               "e2e": {"value": job.npairs * n / (e_ms / 1e3), "unit": "elements/s",
                       "h2d_bytes_per_step": 16 * n * job.npairs, "d2h_bytes_per_step": 16 * n * job.npairs,
                       "ms_per_step": round(e_ms, 4),
                       "api": "mpc_softmax_hostio (pinned host shares in/out, 1536-row chunks, copies overlapped)",
                       "pcie_floor_ms": pcie, "frac_of_pcie_floor": round(pcie / e_ms, 3) if pcie else None,
                       "pcie_floor_how": "the step's H2D and D2H bytes as one copy per direction on two streams "
                                         "at once (no compute): the transfer-only time of a step"},
               "gpu_launches": st["launches"],
               "launches_per_step": st["launches"] / args.steps,
               "protocol_per_step": {"philox_blocks": st["philox_calls"] // args.steps,
                                     "bytes_per_party": st["bytes_per_party"] // args.steps,
                                     "rounds": st["rounds"] // args.steps},
               "clocks": clk, "per_op": per_op}
        if not args.no_cpu_baseline and job.ws == 1:      # rank 0 at N = 1 only
            res["cpu_baseline"] = cpu_baseline(args)
            res["cpu_baseline_all_cores"] = cpu_baseline_all_cores(args)
    if job.ws > 1:
        job.barrier()
        dist.destroy_process_group()
    return res


def pcie_floor(job, hin, hout, reps=5):
    """Transfer-only floor of one e2e step: every party buffer H2D and D2H, one copy per direction
    per buffer, the two directions on two streams at once."""
    torch = job.torch
    try:
        dev_in = [torch.empty_like(h, device=job.dev) if h is not None else None for h in hin]
        s1, s2 = torch.cuda.Stream(job.dev), torch.cuda.Stream(job.dev)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(job.stream)
        for _ in range(reps):
            s1.wait_stream(job.stream); s2.wait_stream(job.stream)
            with torch.cuda.stream(s1):
                for h, d in zip(hin, dev_in):
                    if h is not None:
                        d.copy_(h, non_blocking=True)
            with torch.cuda.stream(s2):
                for h, d in zip(hout, dev_in):
                    if h is not None:
                        h.copy_(d, non_blocking=True)
            job.stream.wait_stream(s1); job.stream.wait_stream(s2)
        b.record(job.stream)
        torch.cuda.synchronize()
        return round(a.elapsed_time(b) / reps, 4)
    except Exception:
        return None


def check_timed_output(job, step_id, xs, out, rows, cols, row_off, sm_kw, tiles=8):
    """Bit-exact check of the TIMED output: `tiles` 32-row tiles spread over the last timed step's
    output (every share of both parties) against oracle/ run at that step's id on the same input
    shares (the PRG is keyed by global row, so a 32-row slice with its row_off is exactly that part
    of the op).  PAIR: pair 0's two ranks contribute their party's shares."""
    r0s = sorted({int(v) // 32 * 32 for v in np.linspace(0, rows - 32, tiles)})
    mine = {}
    for r0 in r0s:
        sl = slice(r0 * cols, (r0 + 32) * cols)
        mine[r0] = [(None if xs[p] is None else xs[p][sl].cpu().numpy(),
                     None if out[p] is None else out[p][sl].cpu().numpy()) for p in (0, 1)]
    if job.ws > 1:
        allp = [None] * job.ws
        job.dist.all_gather_object(allp, (job.pair_idx, job.party, mine))
        if job.rank != 0:
            return {"ok": None, "checked_on": "rank 0"}
        got = {}
        for pidx, party, d in allp:
            if pidx != 0:
                continue
            for r0, v in d.items():
                got.setdefault(r0, [None, None])[party] = v[party]
        mine = {r0: [v[0], v[1]] for r0, v in got.items()}
    try:
        from oracle import Oracle                 # test infrastructure: the checker, not the product path
        bad = []
        for r0 in r0s:
            (x0, z0), (x1, z1) = mine[r0]
            o = Oracle.for_cfg(workloads.keys(2), step_id)
            r = o.softmax((x0, x1), 32, cols, row_off=row_off + r0, **sm_kw)
            if not (np.array_equal(r[0], z0) and np.array_equal(r[1], z1)):
                bad.append(r0)
        return {"ok": not bad, "rows_checked": 32 * len(r0s), "tile_rows": r0s, "mismatching_tiles": bad,
                "step_id": int(step_id), "how": "every share of both parties vs oracle/ (plain C) at the last "
                                                "timed step's id, same input shares"}
    except Exception as e:                       # never fail the bench line on the checker itself
        return {"ok": None, "error": f"{type(e).__name__}: {e}"[:200]}


def dealer_on(job):
    """PAIR with the trusted dealer's correction stream for party 1 (uniform over ranks)."""
    return job.ws > 1 and os.environ.get("MPC_BENCH_DEALER", "1") == "1"


def _op_line(job, ctx, fn, n, flush, args, config):
    job.prefeed(ctx, fn, max(1, args.warmup) + args.steps)       # PAIR party 1: the dealer's offline pass
    for _ in range(max(1, args.warmup)):
        fn()
    job.torch.cuda.synchronize()
    ms, kt, st, _ = timed(job, ctx, fn, args.steps, flush)
    kms = sum(t[1] for t in kt) / args.steps
    ph = st["philox_calls"] / args.steps
    peak = philox_peak_gblocks(float(load_peaks().get("sm_max_mhz", 1965.0)))
    line = {"elements": n, "elements_per_s": n * job.npairs / (ms / 1e3), "ms": round(ms, 4),
            "gphilox_s": round(ph / (kms / 1e3) / 1e9, 2), "alu_frac": round(ph / (kms / 1e3) / 1e9 / peak, 4),
            "bytes_per_party": st["bytes_per_party"] // args.steps, "rounds": st["rounds"] // args.steps,
            "config": config}
    if ctx.mode == job.m.binding.MODE_PAIR_LOOPBACK:
        # both parties' kernels on ONE GPU exchanging through local HBM: no NVLink involved
        f = WIRE_FACTOR[ctx.exchange]
        wire = line["bytes_per_party"] * f
        line["exchange"] = {"where": "local HBM (loopback, no NVLink)", "format": ["LL", "LL63"][ctx.exchange],
                            "payload_bytes_per_party": line["bytes_per_party"],
                            "wire_bytes_per_party": int(wire), "wire_over_payload": f,
                            "wire_gbs_per_party": round(wire / (ms / 1e3) / 1e9, 2)}
    elif ctx.mode == job.m.binding.MODE_PAIR:
        wire = line["bytes_per_party"] * WIRE_FACTOR[ctx.exchange]
        line["nvlink"] = {"payload_bytes_per_party": line["bytes_per_party"], "wire_bytes_per_party": int(wire),
                          "wire_gbs": round(wire / (ms / 1e3) / 1e9, 2), "peak_gbs": NVLINK_PEER_GBS,
                          "wire_frac": round(wire / (ms / 1e3) / 1e9 / NVLINK_PEER_GBS, 4),
                          "payload_roofline_frac": round(line["bytes_per_party"] / NVLINK_PEER_GBS / 1e9 / (ms / 1e3), 4)}
    return line


def time_per_op(job, m, ctx, flush, args):
    torch = job.torch
    k = job.pair_idx
    out = {}
    n3 = workloads.SHAPES["cfg3_gelu"]
    g = job.share(ctx, workloads.normal_inputs(n3, 3), k * n3)
    z = ctx._empty(n3)
    out["gelu"] = _op_line(job, ctx, lambda c=ctx: c.gelu(g, off=k * n3, form="poly_abs", degree=4, out=z), n3, flush,
                           args, "cfg3: BERT-base FFN 8x128x3072, |x|-form deg 4, B=3")
    del g, z
    N, C, H, W = workloads.SHAPES["cfg4_relu_first"]
    n4 = N * C * H * W // 4
    r = job.share(ctx, workloads.relu_inputs(n4), k * n4)
    z = ctx._empty(n4)
    out["relu"] = _op_line(job, ctx, lambda c=ctx: c.relu(r, off=k * n4, out=z), n4, flush, args,
                           "cfg4: ResNet-50 first ReLU, 8 images x 64 x 112 x 112, window 33")
    del r, z
    Np, Cp, Hp, Wp = 8, 64, 112, 112                  # one pair's 8-image shard of the MaxPool input
    mp = job.share(ctx, workloads.maxpool_inputs((Np, Cp, Hp, Wp)), k * Np * Cp * Hp * Wp)
    no = Np * Cp * 56 * 56
    z = ctx._empty(no)
    out["maxpool"] = _op_line(job, ctx, lambda c=ctx: c.maxpool2d(mp, Np, Cp, Hp, Wp, 3, 2, 1, img_off=k * Np, out=z),
                              no, flush, args, "cfg4: ResNet-50 MaxPool 3x3/2 pad 1, 8 x 64 x 112^2 -> 56^2 "
                              "(elements = outputs, 8 comparisons each)")
    del mp, z
    rows5, cols5 = workloads.SHAPES["cfg5_ln"]
    ln = job.share(ctx, workloads.layernorm_inputs(rows5, cols5), k * rows5 * cols5)
    z = ctx._empty(rows5 * cols5)
    out["layernorm"] = _op_line(job, ctx, lambda c=ctx: c.layernorm(ln, rows5, cols5, row_off=k * rows5, out=z),
                                rows5 * cols5, flush, args, "cfg5: GPT-2 LayerNorm 8192 x 768, rsqrt 3 iters")
    del ln, z
    rs, cs = 8 * 12 * 128, 1024
    sm = job.share(ctx, workloads.softmax_inputs(rs, cs, seed_cfg=5), k * rs * cs)
    z = ctx._empty(rs * cs)
    out["softmax1024"] = _op_line(job, ctx, lambda c=ctx: c.softmax(sm, rs, cs, row_off=k * rs, out=z), rs * cs, flush,
                                  args, "cfg5: GPT-2 softmax rows of 1024 (12288 rows = 1/8 layer), t=8, NR 10")
    out["softmax1024_causal"] = _op_line(job, ctx, lambda c=ctx: c.softmax(sm, rs, cs, row_off=k * rs, causal=1, out=z),
                                         rs * cs, flush, args,
                                         "cfg5: GPT-2 causal softmax (12 x 1024 x 1024 blocks, DESIGN.md 2.12)")
    del sm, z
    # NEXT #1 / #2 variants of the same ops (same approximation; the cone's output shares are
    # bit-identical to the Kogge-Stone contract's, square triples change the shares)
    x2 = job.share(ctx, workloads.softmax_inputs(*workloads.SHAPES["cfg2_softmax"]), k * 12288 * 128)
    z = ctx._empty(12288 * 128)
    out["softmax_clamp"] = _op_line(job, ctx, lambda c=ctx: c.softmax(x2, 12288, 128, row_off=k * 12288, exp_clamp=1,
                                                                  out=z), 12288 * 128, flush, args,
                                    "cfg2 softmax with exp t=8+clamp (max-accuracy knob)")
    out["softmax_bcast"] = _op_line(job, ctx, lambda c=ctx: c.softmax(x2, 12288, 128, row_off=k * 12288, bcast=1, out=z),
                                    12288 * 128, flush, args, "cfg2 softmax, broadcast triple for e*r (NEXT #2)")
    out["softmax_square"] = _op_line(job, ctx, lambda c=ctx: c.softmax(x2, 12288, 128, row_off=k * 12288, exp_square=1,
                                                                   recip_square=1, out=z), 12288 * 128, flush, args,
                                     "cfg2 softmax with square-pair triples in every exp squaring (NEXT #2)")
    ctx.set_ltz_circuit(1)
    out["softmax_cone"] = _op_line(job, ctx, lambda c=ctx: c.softmax(x2, 12288, 128, row_off=k * 12288, out=z),
                                   12288 * 128, flush, args, "cfg2 softmax, carry-cone LTZ in the max tree (NEXT #1)")
    out["softmax_cone_square"] = _op_line(
        job, ctx, lambda c=ctx: c.softmax(x2, 12288, 128, row_off=k * 12288, exp_square=1, recip_square=1, out=z),
        12288 * 128, flush, args, "cfg2 softmax, carry-cone LTZ + square-pair triples (NEXT #1 + #2)")
    out["softmax_next_all"] = _op_line(
        job, ctx, lambda c=ctx: c.softmax(x2, 12288, 128, row_off=k * 12288, exp_square=1, recip_square=1, bcast=1,
                                      out=z),
        12288 * 128, flush, args, "cfg2 softmax, carry cone + square-pair triples + broadcast triple (NEXT #1 + #2)")
    del x2, z
    g = job.share(ctx, workloads.normal_inputs(n3, 3), k * n3)
    z = ctx._empty(n3)
    out["gelu_cone"] = _op_line(job, ctx, lambda c=ctx: c.gelu(g, off=k * n3, form="poly_abs", degree=4, out=z), n3,
                                flush, args, "cfg3 GELU |x|-form deg 4, carry-cone LTZ (NEXT #1)")
    out["gelu_cone_power"] = _op_line(
        job, ctx, lambda c=ctx: c.gelu(g, off=k * n3, form="poly_abs", degree=4, basis=1, out=z), n3, flush, args,
        "cfg3 GELU |x|-form deg 4, carry-cone LTZ + power basis (NEXT #1 + #2)")
    del g, z
    r = job.share(ctx, workloads.relu_inputs(n4), k * n4)
    z = ctx._empty(n4)
    out["relu_cone"] = _op_line(job, ctx, lambda c=ctx: c.relu(r, off=k * n4, out=z), n4, flush, args,
                                "cfg4 ReLU shard, carry-cone LTZ (NEXT #1)")
    del r, z
    ctx.set_ltz_circuit(0)
    Bm, Mm, Km, Nm = 1, 1024, 768, 3072           # BERT-base FFN Linear (8 x 128 tokens), NEXT #3
    if True:
        xm = job.share(ctx, workloads.act_inputs(Mm * Km, lo=-2, hi=2), k * Mm * Km)
        ym = job.share(ctx, workloads.act_inputs(Km * Nm, seed_cfg=5, lo=-2, hi=2), k * Km * Nm)
        z = ctx._empty(Mm * Nm)
        out["matmul_tc"] = _op_line(job, ctx, lambda c=ctx: c.matmul(xm, ym, Bm, Mm, Km, Nm, batch_off=k,
                                                                     trunc_bits=16, out=z), Mm * Nm, flush, args,
                                    "Beaver matmul 1024 x 768 x 3072 (BERT FFN Linear), tcgen05 kind::i8 on 8-bit "
                                    "limbs (elements = outputs; 2.4 G ring MACs)")
        del xm, ym, z
    nm = 1 << 24
    a = job.share(ctx, workloads.act_inputs(nm), k * nm)
    b = job.share(ctx, workloads.act_inputs(nm, seed_cfg=7), k * nm)
    z = ctx._empty(nm)
    out["mul"] = _op_line(job, ctx, lambda c=ctx: c.mul(a, b, off=k * nm, trunc_bits=16, out=z), nm, flush, args,
                          "Beaver multiply + trunc, 16M elements")
    del a, b, z
    torch.cuda.synchronize()
    return out


def time_loopback(job, m, flush, args):
    """The PAIR protocol on one GPU: both parties' kernels in one launch (MPC_MODE_PAIR_LOOPBACK),
    every opening exchanged through memory exactly as across NVLink."""
    rows, cols = workloads.SHAPES["cfg2_softmax"]
    c = job.ctx(2, mode=m.binding.MODE_PAIR_LOOPBACK)
    xs = c.share(job.torch.from_numpy(workloads.softmax_inputs(rows, cols).ravel()).to(job.dev))
    z = c._empty(rows * cols)
    line = _op_line(job, c, lambda: c.softmax(xs, rows, cols, out=z), rows * cols, flush, args,
                    "cfg2 softmax, PAIR protocol in loopback (both parties on this GPU)")
    n3 = workloads.SHAPES["cfg3_gelu"]
    g = c.share(job.torch.from_numpy(workloads.normal_inputs(n3, 3)).to(job.dev))
    z2 = c._empty(n3)
    line2 = _op_line(job, c, lambda: c.gelu(g, form="poly_abs", degree=4, out=z2), n3, flush, args,
                     "cfg3 GELU |x|-form deg 4, PAIR protocol in loopback")
    # the same two ops with the LL63 wire format (the MPC_MODE_PAIR default): 33/32 wire bytes per
    # payload byte instead of 2 -- the format whose bytes set a real pair's NVLink time
    c2 = job.ctx(2, mode=m.binding.MODE_PAIR_LOOPBACK)
    c2.set_exchange(1)
    xs2 = c2.share(job.torch.from_numpy(workloads.softmax_inputs(rows, cols).ravel()).to(job.dev))
    line3 = _op_line(job, c2, lambda: c2.softmax(xs2, rows, cols, out=z), rows * cols, flush, args,
                     "cfg2 softmax, PAIR protocol in loopback, LL63 wire format")
    g2 = c2.share(job.torch.from_numpy(workloads.normal_inputs(n3, 3)).to(job.dev))
    line4 = _op_line(job, c2, lambda: c2.gelu(g2, form="poly_abs", degree=4, out=z2), n3, flush, args,
                     "cfg3 GELU |x|-form deg 4, PAIR protocol in loopback, LL63 wire format")
    return {"softmax_pair_loopback": line, "gelu_pair_loopback": line2, "softmax_pair_loopback_ll63": line3,
            "gelu_pair_loopback_ll63": line4}


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


_BAR = None


def _oracle_pool_init(bar):
    global _BAR
    _BAR = bar


def _oracle_rows_worker(a, b):
    """Rows [a, b) of cfg2 through the oracle, as it stands (row_off = a: the PRG is keyed by
    global row, so the slices together are exactly the whole op).  Returns (t_start, t_end) on
    the system-wide monotonic clock, the compute only."""
    from oracle import Oracle
    rows, cols = workloads.SHAPES["cfg2_softmax"]
    o = Oracle.for_cfg(workloads.keys(2))
    s = o.share(workloads.softmax_inputs(rows, cols)[a:b], off=a * cols)
    _BAR.wait()
    t0 = time.perf_counter()
    o.softmax(s, b - a, cols, row_off=a)
    return t0, time.perf_counter()


def _oracle_softmax_all_cores(rows_s, ncores, reps=1):
    """The same oracle in one process per host core (at most 128) over 32-row-aligned row slices
    (SURVEY 8(d) oracle timing, 'all host cores'); per rep, wall time = last end - first start
    of the compute.  Returns ([seconds per rep], processes used)."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    ncores = max(1, min(ncores, 128, rows_s // 32))
    per = (rows_s // 32 + ncores - 1) // ncores * 32
    parts = [(a, min(rows_s, a + per)) for a in range(0, rows_s, per)]
    bar = ctx.Barrier(len(parts))
    out = []
    with ctx.Pool(len(parts), initializer=_oracle_pool_init, initargs=(bar,)) as pool:
        for _ in range(reps):
            spans = pool.starmap_async(_oracle_rows_worker, parts, chunksize=1).get(timeout=600)
            out.append(max(t1 for _, t1 in spans) - min(t0 for t0, _ in spans))
    return out, len(parts)


def _host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_baseline_all_cores(args):
    """The oracle on every host core (process per core over row slices), whole cfg2."""
    rows, cols = workloads.SHAPES["cfg2_softmax"]
    try:
        dts, used = _oracle_softmax_all_cores(rows, _host_cores())
    except Exception as e:                      # a reported baseline only: never fail the bench line
        return {"unavailable": f"{type(e).__name__}: {e}"[:200]}
    dt = dts[0]
    return {"value": rows * cols / dt, "unit": "elements/s", "cores": used, "kind": "oracle",
            "sample": f"all {rows} rows of cfg2 softmax, one process per core over 32-row-aligned slices, "
                      f"{dt:.2f} s wall", "host_cpus": os.cpu_count()}


def cpu_baseline(args):
    """The oracle as it stands (plain C, 1 thread) on a bounded sample of cfg2."""
    rows, cols = workloads.SHAPES["cfg2_softmax"]
    rows_s = int(os.environ.get("MPC_CPU_SAMPLE_ROWS", "4096"))
    dt = _oracle_softmax_sample(rows_s)
    return {"value": rows_s * cols / dt, "unit": "elements/s", "cores": 1, "kind": "oracle",
            "sample": f"{rows_s} of {rows} rows of cfg2 softmax ({rows_s * cols} elements), 1 pass, {dt:.2f} s",
            "host_cpus": os.cpu_count()}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return None
    rows, cols = workloads.SHAPES["cfg2_softmax"]
    dt32 = _oracle_softmax_sample(32)          # size each step so the whole run takes ~2 minutes
    per_row = dt32 / 32
    budget = float(os.environ.get("MPC_REF_BUDGET_S", "120"))
    cores = _host_cores()
    rows_s = int(max(32, min(rows, budget / (args.steps + args.warmup) / per_row * min(cores, 128))) // 32 * 32)
    try:                                       # the oracle on every host core (process per core, row slices)
        dts, used = _oracle_softmax_all_cores(rows_s, cores, reps=args.warmup + args.steps)
        ts = dts[args.warmup:]
        how = f"one process per core on {used} cores over 32-row-aligned slices"
    except Exception:                          # no process pool here: one thread, as before
        rows_s = int(max(32, min(rows, budget / (args.steps + args.warmup) / per_row)) // 32 * 32)
        for _ in range(args.warmup):
            _oracle_softmax_sample(rows_s)
        ts = [_oracle_softmax_sample(rows_s) for _ in range(args.steps)]
        used, how = 1, "1 thread"
    ms = 1e3 * sum(ts) / len(ts)
    v = rows_s * cols / (ms / 1e3)
    sample = f"{rows_s} of {rows} rows of cfg2 softmax per step (oracle/, plain C, {how})"
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": "elements/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": "cfg2: BERT-base attention softmax 8x12x128x128 (2-party, Z_2^64, f=16)",
                       "rows": rows, "cols": cols, "sample_rows": rows_s},
            "cpu_baseline": {"value": v, "unit": "elements/s", "cores": used, "kind": "oracle", "sample": sample},
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
