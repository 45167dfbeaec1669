"""Approximation auto-tuner ("Auto-tuning").

CrypTorch's tuner picks, per operator instance (layer), the cheapest approximation whose output
quality stays within a user threshold of the maximally accurate one ("The output quality
is compared with the maximally accurate approximation, and the difference is compared with the
user-given threshold"), scoring candidates on a non-MPC runtime.  This module is the
search machinery over the library's knobs:

* a Layer: an op kind ("softmax", "gelu", "silu", "sigmoid", "layernorm", "relu" (comparison
  window, HummingBird-style), "exp", "recip", "rsqrt"), its MPC shape, calibration inputs (a float64 device tensor) and candidate knob sets
  ordered from the most accurate to the cheapest (``CANDIDATES``);
* quality: the plaintext fixed-point emulation of each candidate (``Ctx.plain_eval`` ->
  mpc_plain_eval, CUDA) against the most accurate candidate's emulation on the same inputs --
  max abs error per layer, summed over the layers (reading: without a trained model the paper's
  end-to-end loss is replaced by this additive per-layer error budget);
* cost: measured per candidate by running the MPC op once on the layer's shape (MPC_MODE_BOTH,
  CUDA events) and reading the protocol counters (bytes per party, rounds), then combined by an
  objective: "gpu" (ms), or the paper's emulated networks "lan" (0.3 ms, 10 Gbps) and "wan"
  (40 ms, 352 Mbps);
* strategies (``Tuner.generate_next_candidate``): GreedyTuner -- layer by layer,
  take the next cheaper candidate while the quality holds, roll back on failure; HillClimbTuner
  -- every step applies the single-layer move with the largest cost reduction that keeps the
  quality.

Host-side search only: every evaluation runs in the library's kernels.
"""
from __future__ import annotations

import dataclasses
from typing import Callable, Dict, List, Optional, Sequence

NETWORKS = {"lan": (0.3e-3, 10e9 / 8), "wan": (40e-3, 352e6 / 8)}   # (latency s, bytes/s)

# candidate knob sets per op kind, most accurate first (the knob ranges of P:206-219)
CANDIDATES: Dict[str, List[dict]] = {
    # (the NEXT #2 protocol variants -- square-pair triples, the broadcast triple, power-basis
    # polynomials -- are candidates too: same approximation, fewer bytes / rounds, their own
    # fixed-point rounding)
    "softmax": [dict(exp_t=8, exp_clamp=1), dict(exp_t=8, exp_clamp=0),
                dict(exp_t=8, exp_clamp=0, exp_square=1, recip_square=1, bcast=1), dict(exp_t=4, exp_clamp=1),
                dict(exp_t=2, exp_clamp=1), dict(exp_t=2, exp_clamp=1, recip_iters=7),
                dict(exp_t=0, exp_clamp=1, recip_iters=7)],
    "gelu": [dict(form="poly_abs", degree=4), dict(form="poly_abs", degree=4, basis=1), dict(form="poly_abs", degree=2),
             dict(form="relu", degree=0)],
    "silu": [dict(form="poly_abs", degree=4), dict(form="poly_abs", degree=2), dict(form="relu", degree=0)],
    "sigmoid": [dict(form="poly_x", degree=4), dict(form="poly_x", degree=2), dict(form="relu", degree=0)],
    "layernorm": [dict(rsqrt_iters=3, rsqrt_t=8), dict(rsqrt_iters=2, rsqrt_t=8), dict(rsqrt_iters=3, rsqrt_t=4),
                  dict(rsqrt_iters=3, rsqrt_t=0), dict(rsqrt_iters=2, rsqrt_t=0)],
    # HummingBird-style per-site comparison windows: the sign is
    # exact while |x| < 2^(w-17); a smaller window means fewer carry-circuit gates and bytes
    "relu": [dict(window=33), dict(window=29), dict(window=25), dict(window=21), dict(window=19), dict(window=17)],
    "exp": [dict(t=8, clamp=1), dict(t=8), dict(t=4), dict(t=2), dict(t=0, clamp=1)],
    "recip": [dict(iters=10), dict(iters=8), dict(iters=6)],
    "rsqrt": [dict(iters=3), dict(iters=2), dict(iters=1)],
}


@dataclasses.dataclass
class Layer:
    name: str
    op: str
    rows: int
    cols: int
    calib: object                      # float64 CUDA tensor (rows_c x cols) of calibration inputs
    calib_rows: int
    candidates: Optional[List[dict]] = None
    mpc_rows: Optional[int] = None     # MPC shape for the cost (defaults to the calibration shape)

    def cands(self) -> List[dict]:
        return self.candidates if self.candidates is not None else CANDIDATES[self.op]


class Evaluator:
    """Quality (plaintext emulation) and cost (one MPC run) of candidate knob sets, cached."""

    def __init__(self, ctx, mpc_inputs: Optional[Dict[str, tuple]] = None, objective: str = "gpu"):
        """mpc_inputs: op kind -> (shares, rows) of the MPC shape to cost on (default: the layer's
        calibration inputs); costs are cached per (op, shape, knobs), so layers of the same shape
        are measured once."""
        self.ctx = ctx
        self.objective = objective
        self.mpc_inputs = mpc_inputs or {}
        self._ref: Dict[str, object] = {}
        self._err: Dict[tuple, float] = {}
        self._cost: Dict[tuple, dict] = {}

    def _plain(self, layer: Layer, knobs: dict):
        return self.ctx.plain_eval(layer.op, layer.calib, rows=layer.calib_rows, cols=layer.cols, **knobs)

    def error(self, layer: Layer, k: int) -> float:
        key = (layer.name, k)
        if key not in self._err:
            if layer.name not in self._ref:
                self._ref[layer.name] = self._plain(layer, layer.cands()[0])
            y = self._plain(layer, layer.cands()[k])
            self._err[key] = float((y - self._ref[layer.name]).abs().max().item())
        return self._err[key]

    def cost(self, layer: Layer, k: int) -> dict:
        knobs = layer.cands()[k]
        shares, rows = self.mpc_inputs.get(layer.op, (None, layer.mpc_rows or layer.calib_rows))
        key = (layer.op, rows, layer.cols, tuple(sorted(knobs.items())))
        if key not in self._cost:
            self._cost[key] = measure_cost(self.ctx, layer, knobs, shares, rows)
        return self._cost[key]

    def objective_value(self, layer: Layer, k: int) -> float:
        c = self.cost(layer, k)
        if self.objective == "gpu":
            return c["ms"]
        lat, bw = NETWORKS[self.objective]
        return 1e3 * (c["rounds"] * lat + c["bytes_per_party"] / bw) + c["ms"]


def measure_cost(ctx, layer: Layer, knobs: dict, shares=None, rows: Optional[int] = None, reps: int = 3) -> dict:
    """One MPC run of the layer's op with these knobs (BOTH mode): ms (CUDA events, mean of reps after
    a warm-up), bytes per party and rounds from the context's protocol counters."""
    import torch
    rows = rows or layer.mpc_rows or layer.calib_rows
    if shares is None:
        shares = ctx.share(layer.calib.reshape(-1)[: rows * layer.cols].contiguous())
    fn = _mpc_call(ctx, layer, knobs, shares, rows)
    fn()
    torch.cuda.synchronize()
    ctx.reset_stats()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    st = ctx.stats()
    return {"ms": a.elapsed_time(b) / reps, "bytes_per_party": st["bytes_per_party"] // reps,
            "rounds": st["rounds"] // reps}


def _mpc_call(ctx, layer: Layer, knobs: dict, x, rows) -> Callable[[], object]:
    op, cols = layer.op, layer.cols
    if op == "softmax":
        return lambda: ctx.softmax(x, rows, cols, **knobs)
    if op == "layernorm":
        return lambda: ctx.layernorm(x, rows, cols, **knobs)
    if op in ("gelu", "silu", "sigmoid"):
        return lambda: getattr(ctx, op)(x, **knobs)
    return lambda: getattr(ctx, op)(x, **knobs)


class Tuner:
    """Search over per-layer candidate indices (0 = most accurate).  Subclasses implement
    generate_next_candidate(state, history) -> Optional[list]."""

    def __init__(self, layers: Sequence[Layer], evaluator: Evaluator, threshold: float):
        self.layers = list(layers)
        self.ev = evaluator
        self.threshold = threshold
        self.history: List[tuple] = []

    def quality_loss(self, state: Sequence[int]) -> float:
        return sum(self.ev.error(l, k) for l, k in zip(self.layers, state))

    def total_cost(self, state: Sequence[int]) -> float:
        return sum(self.ev.objective_value(l, k) for l, k in zip(self.layers, state))

    def accept(self, state: Sequence[int]) -> bool:
        return self.quality_loss(state) <= self.threshold

    def generate_next_candidate(self, state: List[int]) -> Optional[List[int]]:
        raise NotImplementedError

    def run(self, max_steps: int = 10_000) -> dict:
        state = [0] * len(self.layers)
        for _ in range(max_steps):
            nxt = self.generate_next_candidate(state)
            if nxt is None:
                break
            state = nxt
        return {"state": state, "knobs": {l.name: l.cands()[k] for l, k in zip(self.layers, state)},
                "quality_loss": self.quality_loss(state), "cost": self.total_cost(state),
                "cost_most_accurate": self.total_cost([0] * len(self.layers)), "steps": len(self.history)}


class GreedyTuner(Tuner):
    """Linear greedy search: layer by layer, step to the next cheaper candidate while the quality
    threshold holds; on failure roll back and move on to the next layer."""

    def __init__(self, layers, evaluator, threshold):
        super().__init__(layers, evaluator, threshold)
        self._layer = 0

    def generate_next_candidate(self, state):
        while self._layer < len(self.layers):
            l = self._layer
            if state[l] + 1 < len(self.layers[l].cands()):
                trial = list(state)
                trial[l] += 1
                ok = self.accept(trial)
                self.history.append((l, trial[l], ok))
                if ok:
                    return trial
            self._layer += 1
        return None


class HillClimbTuner(Tuner):
    """Each step applies the single-layer move (one candidate cheaper) with the largest cost
    reduction among the moves that keep the quality; stops when no move helps."""

    def generate_next_candidate(self, state):
        best, best_gain = None, 0.0
        cur = [self.ev.objective_value(l, k) for l, k in zip(self.layers, state)]
        for l, layer in enumerate(self.layers):
            if state[l] + 1 >= len(layer.cands()):
                continue
            trial = list(state)
            trial[l] += 1
            gain = cur[l] - self.ev.objective_value(layer, trial[l])
            if gain > best_gain and self.accept(trial):
                best, best_gain = trial, gain
        if best is not None:
            self.history.append((best, best_gain))
        return best
