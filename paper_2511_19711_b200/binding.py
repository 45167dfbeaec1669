"""Thin ctypes binding of include/mpc200.h (argument marshalling only).

Every compute step runs in libmpc200.so's CUDA kernels; this module only passes
torch tensor device pointers, the current CUDA stream and knob structs.  There is
no CPU fallback: importing fails loudly if the shared library is missing.
Names follow the C ABI (mpc_share, mpc_open, mpc_mul, ...), exposed as methods of
`Ctx` without the prefix.
"""
from __future__ import annotations

import ctypes
import json
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MPC200_LIB") or os.path.join(_PKG, "libmpc200.so")   # override: A/B experiments

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libmpc200.so not found at {LIB_PATH}: run `python paper_2511_19711_b200/build.py` "
                      "(there is no CPU fallback)")
_L = ctypes.CDLL(LIB_PATH)

u64 = ctypes.c_uint64
i64 = ctypes.c_int64
INT = ctypes.c_int
VP = ctypes.c_void_p

MODE_BOTH, MODE_PAIR, MODE_PAIR_LOOPBACK, MODE_DEALER = 0, 1, 2, 3
PAIR_HANDLE_BYTES = 64
FORM = {"poly_x": 0, "poly_abs": 1, "relu": 2, "erf": 3}
STATUS = {0: "OK", 1: "INVALID", 2: "RANGE", 3: "CUDA", 4: "NCCL", 5: "PROTOCOL", 6: "REUSE",
          7: "TIMEOUT", 8: "NOMEM", 9: "UNSUPPORTED"}


class Config(ctypes.Structure):
    _fields_ = [("mode", INT), ("party", INT), ("frac_bits", INT), ("device", INT),
                ("key_share", u64), ("key_p0", u64), ("key_p1", u64),
                ("cuda_stream", VP), ("reserved", VP)]


class Shares(ctypes.Structure):
    _fields_ = [("sh", VP * 2)]


class Stats(ctypes.Structure):
    _fields_ = [("steps", u64), ("philox_calls", u64), ("bytes_per_party", u64), ("rounds", u64),
                ("launches", u64), ("calls", u64)]


class KernelTime(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("ms", ctypes.c_float), ("philox", u64), ("units", u64)]


class CorrSeg(ctypes.Structure):
    _fields_ = [("base", u64), ("threads", u64), ("depth", u64), ("tag", u64)]


class ExpP(ctypes.Structure):
    _fields_ = [("t", INT), ("clamp", INT), ("window", INT), ("square", INT)]


class NrP(ctypes.Structure):
    _fields_ = [("iters", INT), ("exp", ExpP)]


class ActP(ctypes.Structure):
    _fields_ = [("form", INT), ("degree", INT), ("B", ctypes.c_double),
                ("coeffs", ctypes.POINTER(ctypes.c_double)), ("erf_terms", INT), ("window", INT),
                ("basis", INT)]


class SoftmaxP(ctypes.Structure):
    _fields_ = [("window", INT), ("exp", ExpP), ("recip", NrP), ("bcast", INT), ("causal", INT)]


class LnP(ctypes.Structure):
    _fields_ = [("eps", ctypes.c_double), ("mean_mode", INT), ("rsqrt", NrP), ("bcast", INT)]


C = ctypes.POINTER
_SIGS = {
    "mpc_ctx_create": [C(Config), C(VP)],
    "mpc_ctx_destroy": [VP],
    "mpc_ctx_set_step": [VP, u64, INT],
    "mpc_ctx_get_step": [VP],
    "mpc_ctx_set_stream": [VP, VP],
    "mpc_ctx_stats": [VP, C(Stats)],
    "mpc_ctx_reset_stats": [VP],
    "mpc_last_error": [VP],
    "mpc_version": [],
    "mpc_last_call_philox": [VP],
    "mpc_ctx_enable_kernel_timing": [VP, INT],
    "mpc_ctx_set_ltz_circuit": [VP, INT],
    "mpc_ctx_set_matmul_engine": [VP, INT],
    "mpc_dealer_set_target": [VP, INT],
    "mpc_dealer_stream": [VP, C(VP), C(u64), C(VP), C(i64)],
    "mpc_dealer_reset": [VP],
    "mpc_ctx_set_corrections": [VP, VP, u64, VP, i64],
    "mpc_ctx_corrections_left": [VP],
    "mpc_pair_export": [VP, VP],
    "mpc_pair_connect": [VP, VP],
    "mpc_ctx_sync": [VP],
    "mpc_ctx_kernel_times": [VP, VP, INT],
    "mpc_prg_fill": [VP, u64, u64, ctypes.c_uint32, ctypes.c_uint32, VP, i64, INT],
    "mpc_share": [VP, VP, INT, INT, Shares, i64, i64],
    "mpc_open": [VP, Shares, i64, VP, VP, INT],
    "mpc_open_to": [VP, Shares, i64, INT, VP, VP, INT],
    "mpc_ctx_set_debug": [VP, INT],
    "mpc_ctx_set_exchange": [VP, INT],
    "mpc_ctx_get_exchange": [VP],
    "mpc_mul": [VP, Shares, Shares, Shares, i64, i64, INT],
    "mpc_square": [VP, Shares, Shares, i64, i64, INT],
    "mpc_mul_bcast": [VP, Shares, Shares, Shares, i64, i64, i64, i64, INT],
    "mpc_matmul": [VP, Shares, Shares, Shares, i64, i64, i64, i64, i64, INT],
    "mpc_plain_eval": [VP, INT, VP, VP, VP, i64, i64],
    "mpc_trunc": [VP, Shares, Shares, i64, INT],
    "mpc_cmp": [VP, Shares, Shares, i64, i64, INT],
    "mpc_relu": [VP, Shares, Shares, i64, i64, INT],
    "mpc_exp": [VP, Shares, Shares, i64, i64, C(ExpP)],
    "mpc_recip": [VP, Shares, Shares, i64, i64, C(NrP)],
    "mpc_rsqrt": [VP, Shares, Shares, i64, i64, C(NrP)],
    "mpc_gelu": [VP, Shares, Shares, i64, i64, C(ActP)],
    "mpc_silu": [VP, Shares, Shares, i64, i64, C(ActP)],
    "mpc_sigmoid": [VP, Shares, Shares, i64, i64, C(ActP)],
    "mpc_max": [VP, Shares, Shares, i64, i64, i64, INT],
    "mpc_maxpool2d": [VP, Shares, Shares, INT, INT, INT, INT, INT, INT, INT, i64, INT],
    "mpc_softmax": [VP, Shares, Shares, i64, i64, i64, C(SoftmaxP)],
    "mpc_softmax_hostio": [VP, Shares, Shares, i64, i64, i64, C(SoftmaxP), i64],
    "mpc_layernorm": [VP, Shares, Shares, i64, i64, i64, C(LnP)],
}
_RESTYPE = {"mpc_ctx_get_step": u64, "mpc_last_error": ctypes.c_char_p, "mpc_version": ctypes.c_char_p,
            "mpc_last_call_philox": u64, "mpc_ctx_corrections_left": i64}
_OPTIONAL = {"mpc_ctx_set_exchange", "mpc_ctx_get_exchange", "mpc_dealer_set_target", "mpc_dealer_stream",
             "mpc_dealer_reset", "mpc_ctx_set_corrections", "mpc_ctx_corrections_left"}   # absent in older A/B builds
for _n, _a in list(_SIGS.items()):
    try:
        _f = getattr(_L, _n)
    except AttributeError:
        if _n in _OPTIONAL and os.environ.get("MPC200_LIB"):
            del _SIGS[_n]
            continue
        raise
    _f.argtypes = _a
    _f.restype = _RESTYPE.get(_n, INT)

EXPORTS = sorted(_SIGS)


def version() -> str:
    return _L.mpc_version().decode()


def load_coeffs():
    path = os.path.join(os.path.dirname(_PKG), "fixtures", "coeffs.json")
    return json.load(open(path))["fits"]


def default_act(act="gelu", form="poly_x", degree=4, erf_terms=8, window=33, B=None, coeffs=None, basis=0):
    """Knob struct for S13 using fixtures/coeffs.json (SPEC S:239 least-squares fits).
    basis: 0 Horner, 1 power basis (NEXT #2; x- and |x|-forms)."""
    if form == "erf":
        return dict(form="erf", degree=0, B=2.5 if B is None else B, coeffs=None, erf_terms=erf_terms,
                    window=window, basis=basis)
    if form == "relu" or degree == 0:
        return dict(form=form, degree=0, B=5.0 if B is None else B, coeffs=None, erf_terms=0, window=window,
                    basis=basis)
    if coeffs is None:
        fit = [f for f in load_coeffs() if f["op"] == act and f["form"] == form and f.get("degree") == degree]
        if not fit:
            raise ValueError(f"no fitted coefficients for {act}/{form}/deg {degree}")
        coeffs, B = fit[0]["coefficients"], fit[0]["interval"][1]
    return dict(form=form, degree=degree, B=B, coeffs=list(coeffs), erf_terms=0, window=window, basis=basis)


class MPCError(RuntimeError):
    pass


def _ptr(t):
    if t is None or t.device.type == "meta":      # meta: a shape-only operand (the dealer's calls)
        return None
    if not t.is_cuda:
        raise ValueError("mpc200 compute calls take CUDA tensors")
    if not t.is_contiguous():
        raise ValueError("tensors must be contiguous")
    return t.data_ptr()


def _sh(pair):
    s = Shares()
    s.sh[0] = _ptr(pair[0]) if pair[0] is not None else None
    s.sh[1] = _ptr(pair[1]) if pair[1] is not None else None
    return s


def _sh_host(pair):
    s = Shares()
    for p in (0, 1):
        t = pair[p]
        if t is None:
            s.sh[p] = None
            continue
        if t.is_cuda or t.dtype != torch.uint64 or not t.is_contiguous():
            raise ValueError("host-buffer calls take contiguous CPU uint64 tensors (pinned for overlap)")
        s.sh[p] = t.data_ptr()
    return s


class Ctx:
    """An mpc_ctx: keys, step counter, stream.  MODE_BOTH holds both parties on one GPU."""

    def __init__(self, key_share: int, key_p0: int, key_p1: int, device: int = 0, mode: int = MODE_BOTH,
                 party: int = 0):
        self.device = torch.device("cuda", device)
        self.mode, self.party = mode, party
        cfg = Config(mode, party, 16, device, key_share, key_p0, key_p1, None, None)
        h = VP()
        st = _L.mpc_ctx_create(ctypes.byref(cfg), ctypes.byref(h))
        if st != 0:
            raise MPCError(f"mpc_ctx_create: {STATUS.get(st, st)}")
        self._h = h

    @classmethod
    def for_cfg(cls, keys: dict, device: int = 0, **kw):
        return cls(keys["key_share"], keys["key_p0"], keys["key_p1"], device, **kw)

    # ---- the trusted dealer's correction stream ----
    @classmethod
    def dealer(cls, keys: dict, device: int = 0, target: int = MODE_PAIR):
        """An MPC_MODE_DEALER context for party 1 of a PAIR (or, target=MODE_PAIR_LOOPBACK, loopback)
        execution: call the same ops with the same shapes as party 1 (operands may be shape-only
        `meta` tensors, see `like`); its stream then feeds party 1 (set_corrections)."""
        d = cls(keys["key_share"], keys["key_p0"], keys["key_p1"], device, mode=MODE_DEALER, party=1)
        d._chk(_L.mpc_dealer_set_target(d._h, target), "mpc_dealer_set_target")
        return d

    @staticmethod
    def like(n: int):
        """A shape-only share pair for the dealer's calls (no device memory)."""
        return (torch.empty(n, dtype=torch.uint64, device="meta"), None)

    def dealer_stream(self):
        """(device word pointer, n_words, [segments]) of the dealer's stream so far; the words stay
        owned by this (dealer) context."""
        w, nw, sg, ns = VP(), u64(), VP(), i64()
        self._chk(_L.mpc_dealer_stream(self._h, ctypes.byref(w), ctypes.byref(nw), ctypes.byref(sg), ctypes.byref(ns)),
                  "mpc_dealer_stream")
        segs = (CorrSeg * max(ns.value, 1))()
        if ns.value:
            ctypes.memmove(segs, sg.value, ctypes.sizeof(CorrSeg) * ns.value)
        return w.value, int(nw.value), list(segs)[:ns.value]

    def dealer_reset(self):
        self._chk(_L.mpc_dealer_reset(self._h), "mpc_dealer_reset")

    def set_corrections(self, stream):
        """Party 1: read the dealer's correction words (a `dealer_stream()` triple, words on this
        device) instead of deriving them from K_0; None clears."""
        if stream is None:
            self._chk(_L.mpc_ctx_set_corrections(self._h, None, 0, None, 0), "mpc_ctx_set_corrections")
            return
        w, nw, segs = stream
        arr = (CorrSeg * max(len(segs), 1))(*segs)
        self._chk(_L.mpc_ctx_set_corrections(self._h, w, nw, ctypes.cast(arr, VP), len(segs)), "mpc_ctx_set_corrections")

    def corrections_left(self) -> int:
        return int(_L.mpc_ctx_corrections_left(self._h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _L.mpc_ctx_destroy(h)
            self._h = None

    # ---- bookkeeping ----
    def _chk(self, st, name):
        if st != 0:
            raise MPCError(f"{name}: {STATUS.get(st, st)}: {_L.mpc_last_error(self._h).decode()}")

    # ---- PAIR plumbing ----
    def pair_export(self) -> bytes:
        buf = ctypes.create_string_buffer(PAIR_HANDLE_BYTES)
        self._chk(_L.mpc_pair_export(self._h, ctypes.cast(buf, VP)), "mpc_pair_export")
        return buf.raw

    def pair_connect(self, peer_handle: bytes):
        buf = ctypes.create_string_buffer(bytes(peer_handle), PAIR_HANDLE_BYTES)
        self._chk(_L.mpc_pair_connect(self._h, ctypes.cast(buf, VP)), "mpc_pair_connect")

    def set_debug(self, on: bool = True):
        """PAIR modes: exchange and compare an op header before every op (MPC_ERR_PROTOCOL at sync)."""
        self._chk(_L.mpc_ctx_set_debug(self._h, int(on)), "mpc_ctx_set_debug")

    def set_exchange(self, fmt: int):
        """PAIR wire format: 0 = LL (2 wire bytes per payload byte), 1 = LL63 (33/32); same shares.
        Only before the context's first exchange (both parties alike)."""
        self._chk(_L.mpc_ctx_set_exchange(self._h, int(fmt)), "mpc_ctx_set_exchange")

    @property
    def exchange(self) -> int:
        if "mpc_ctx_get_exchange" not in _SIGS:                 # an older A/B build: LL only
            return 0
        return int(_L.mpc_ctx_get_exchange(self._h))

    circuit = 0

    def set_ltz_circuit(self, circuit: int):
        """0 = Kogge-Stone (default, the S7 contract), 1 = carry cone (NEXT #1): same output shares."""
        self._chk(_L.mpc_ctx_set_ltz_circuit(self._h, circuit), "mpc_ctx_set_ltz_circuit")
        self.circuit = circuit

    def set_matmul_engine(self, engine: int):
        """0 auto, 1 SIMT, 2 tensor cores (tcgen05 on 8-bit limbs); same output shares."""
        self._chk(_L.mpc_ctx_set_matmul_engine(self._h, engine), "mpc_ctx_set_matmul_engine")

    def sync(self):
        self._stream()
        self._chk(_L.mpc_ctx_sync(self._h), "mpc_ctx_sync")

    def _stream(self):
        _L.mpc_ctx_set_stream(self._h, torch.cuda.current_stream(self.device).cuda_stream)

    @property
    def step(self) -> int:
        return int(_L.mpc_ctx_get_step(self._h))

    def set_step(self, step: int, force: bool = False):
        self._chk(_L.mpc_ctx_set_step(self._h, step, int(force)), "mpc_ctx_set_step")

    def stats(self) -> dict:
        s = Stats()
        self._chk(_L.mpc_ctx_stats(self._h, ctypes.byref(s)), "mpc_ctx_stats")
        return {k: int(getattr(s, k)) for k, _ in Stats._fields_}

    def reset_stats(self):
        _L.mpc_ctx_reset_stats(self._h)

    def enable_kernel_timing(self, on: bool = True):
        self._chk(_L.mpc_ctx_enable_kernel_timing(self._h, int(on)), "mpc_ctx_enable_kernel_timing")

    def kernel_times(self, cap: int = 65536):
        """Drain per-launch records: list of (name, ms, philox_blocks, units)."""
        buf = (KernelTime * cap)()
        n = _L.mpc_ctx_kernel_times(self._h, ctypes.cast(buf, VP), cap)
        return [(buf[i].name.decode(), float(buf[i].ms), int(buf[i].philox), int(buf[i].units))
                for i in range(max(n, 0))]

    def last_call_philox(self) -> int:
        return int(_L.mpc_last_call_philox(self._h))

    def _empty(self, n):
        if self.mode == MODE_DEALER:
            return self.like(n)
        mk = lambda: torch.empty(n, dtype=torch.uint64, device=self.device)  # noqa: E731
        if self.mode in (MODE_BOTH, MODE_PAIR_LOOPBACK):
            return (mk(), mk())
        return (mk(), None) if self.party == 0 else (None, mk())

    # ---- S3 ----
    def prg_fill(self, key: int, unit0: int, step: int, slot: int, n: int, reps: int = 1):
        out = torch.empty(4 * n, dtype=torch.int32, device=self.device)
        self._stream()
        self._chk(_L.mpc_prg_fill(self._h, key, unit0, step, slot, out.data_ptr(), n, reps), "mpc_prg_fill")
        return out

    # ---- S1 / S2 ----
    def share(self, x: torch.Tensor | None, owner: int = 0, off: int = 0, n: int | None = None):
        if x is not None:
            if x.dtype not in (torch.float32, torch.float64):
                raise ValueError("share takes float32 / float64")
            x = x.contiguous().view(-1)
            n = x.numel()
        z = self._empty(n)
        self._stream()
        self._chk(_L.mpc_share(self._h, _ptr(x) if x is not None else None,
                               int(x is not None and x.dtype == torch.float64), owner, _sh(z), n, off),
                  "mpc_share")
        return z

    def open(self, s, scale_bits: int = 16, want_ring=True, want_f64=True):
        n = (s[0] if s[0] is not None else s[1]).numel()
        if self.mode == MODE_DEALER:
            want_ring = want_f64 = False
        ring = torch.empty(n, dtype=torch.uint64, device=self.device) if want_ring else None
        f = torch.empty(n, dtype=torch.float64, device=self.device) if want_f64 else None
        self._stream()
        self._chk(_L.mpc_open(self._h, _sh(s), n, _ptr(ring), _ptr(f), scale_bits), "mpc_open")
        return ring, f

    def open_to(self, s, reveal_to: int, scale_bits: int = 16, want_ring=True, want_f64=True):
        """Open to one party (reveal_to 0 | 1; -1 = both): in the PAIR modes only that party learns
        and writes the result; the other party's outputs are left untouched."""
        n = (s[0] if s[0] is not None else s[1]).numel()
        ring = torch.zeros(n, dtype=torch.uint64, device=self.device) if want_ring else None
        f = torch.zeros(n, dtype=torch.float64, device=self.device) if want_f64 else None
        self._stream()
        self._chk(_L.mpc_open_to(self._h, _sh(s), n, int(reveal_to), _ptr(ring), _ptr(f), scale_bits), "mpc_open_to")
        return ring, f

    # ---- S4 / S5 ----
    def mul(self, x, y, off=0, trunc_bits=0, out=None):
        n = x[0].numel() if x[0] is not None else x[1].numel()
        z = out if out is not None else self._empty(n)
        self._stream()
        self._chk(_L.mpc_mul(self._h, _sh(x), _sh(y), _sh(z), n, off, trunc_bits), "mpc_mul")
        return z

    def mul_bcast(self, x, y, rows, cols, off=0, row_off=0, trunc_bits=0, out=None):
        """z[r, j] = x[r, j] * y[r] with the broadcast triple."""
        z = out if out is not None else self._empty(rows * cols)
        self._stream()
        self._chk(_L.mpc_mul_bcast(self._h, _sh(x), _sh(y), _sh(z), rows, cols, off, row_off, trunc_bits),
                  "mpc_mul_bcast")
        return z

    def matmul(self, x, y, batch, M, K, N, batch_off=0, trunc_bits=0, out=None):
        """Z[b] = X[b] (M x K) @ Y[b] (K x N) over Z_2^64 with a matrix Beaver triple."""
        z = out if out is not None else self._empty(batch * M * N)
        self._stream()
        self._chk(_L.mpc_matmul(self._h, _sh(x), _sh(y), _sh(z), batch, M, K, N, batch_off, trunc_bits), "mpc_matmul")
        return z

    # ---- NEXT #4: plaintext fixed-point emulation (the auto-tuner's evaluator) ----
    PLAIN = {"exp": 0, "recip": 1, "rsqrt": 2, "gelu": 3, "silu": 4, "sigmoid": 5, "softmax": 6, "layernorm": 7,
             "relu": 3}

    def plain_eval(self, op: str, x: torch.Tensor, rows: int = 1, cols: int | None = None, **kw):
        """Run one approximation schedule on plaintext fixed-point values (float64 in / out, device).
        Knobs as the MPC op's keyword arguments."""
        if x.dtype != torch.float64 or not x.is_cuda:
            raise ValueError("plain_eval takes a float64 CUDA tensor")
        x = x.contiguous().view(-1)
        cols = x.numel() // rows if cols is None else cols
        y = torch.empty_like(x)
        if op == "exp":
            knobs = ExpP(kw.get("t", 8), int(kw.get("clamp", 0)), kw.get("window", 33), 0)
        elif op in ("recip", "rsqrt"):
            knobs = NrP(kw.get("iters", 10 if op == "recip" else 3),
                        ExpP(kw.get("t", 8), int(kw.get("clamp", 0)), kw.get("window", 33), 0))
        elif op in ("gelu", "silu", "sigmoid", "relu"):
            if op == "relu":                         # ReLU = the degree-0 segment form, x * NOT ltz_w(x)
                kw = dict(form="relu", degree=0, window=kw.get("window", 33))
            k = default_act("gelu" if op == "relu" else op,
                            **{a: b for a, b in kw.items() if a in ("form", "degree", "erf_terms", "window", "B",
                                                                  "coeffs", "basis")})
            coeffs = k.get("coeffs")
            arr = (ctypes.c_double * len(coeffs))(*coeffs) if coeffs else None
            knobs = ActP(FORM[k["form"]], int(k.get("degree", 0)), float(k.get("B", 5.0)),
                         ctypes.cast(arr, ctypes.POINTER(ctypes.c_double)) if arr is not None else None,
                         int(k.get("erf_terms", 0)), int(k.get("window", 33)), int(k.get("basis", 0)))
        elif op == "softmax":
            # (square triples / broadcast triple change only the MPC rounding, not the emulated value)
            knobs = SoftmaxP(kw.get("window", 33), ExpP(kw.get("exp_t", 8), int(kw.get("exp_clamp", 0)), 33, 0),
                             NrP(kw.get("recip_iters", 10), ExpP(kw.get("recip_t", 8), int(kw.get("recip_clamp", 0)),
                                                                  33, 0)), 0, int(kw.get("causal", 0)))
        elif op == "layernorm":
            knobs = LnP(kw.get("eps", 1e-5), kw.get("mean_mode", 0),
                        NrP(kw.get("rsqrt_iters", 3), ExpP(kw.get("rsqrt_t", 8), int(kw.get("rsqrt_clamp", 0)), 33, 0)), 0)
        else:
            raise ValueError(op)
        self._stream()
        self._chk(_L.mpc_plain_eval(self._h, self.PLAIN[op], ctypes.byref(knobs), _ptr(x), _ptr(y), rows, cols),
                  "mpc_plain_eval")
        return y

    def square(self, x, off=0, trunc_bits=0, out=None):
        n = x[0].numel() if x[0] is not None else x[1].numel()
        z = out if out is not None else self._empty(n)
        self._stream()
        self._chk(_L.mpc_square(self._h, _sh(x), _sh(z), n, off, trunc_bits), "mpc_square")
        return z

    def trunc(self, x, bits=16, out=None):
        n = x[0].numel() if x[0] is not None else x[1].numel()
        z = out if out is not None else self._empty(n)
        self._stream()
        self._chk(_L.mpc_trunc(self._h, _sh(x), _sh(z), n, bits), "mpc_trunc")
        return z

    # ---- element-wise ops ----
    def _un(self, fn, name, x, out, *args):
        n = x[0].numel() if x[0] is not None else x[1].numel()
        z = out if out is not None else self._empty(n)
        self._stream()
        self._chk(fn(self._h, _sh(x), _sh(z), n, *args), name)
        return z

    def cmp(self, x, off=0, window=33, out=None):
        return self._un(_L.mpc_cmp, "mpc_cmp", x, out, off, window)

    def relu(self, x, off=0, window=33, out=None):
        return self._un(_L.mpc_relu, "mpc_relu", x, out, off, window)

    def exp(self, x, off=0, t=8, clamp=0, window=33, square=0, out=None):
        return self._un(_L.mpc_exp, "mpc_exp", x, out, off, ctypes.byref(ExpP(t, int(clamp), window, int(square))))

    def recip(self, x, off=0, iters=10, t=8, clamp=0, window=33, square=0, out=None):
        p = NrP(iters, ExpP(t, int(clamp), window, int(square)))
        return self._un(_L.mpc_recip, "mpc_recip", x, out, off, ctypes.byref(p))

    def rsqrt(self, x, off=0, iters=3, t=8, clamp=0, window=33, square=0, out=None):
        p = NrP(iters, ExpP(t, int(clamp), window, int(square)))
        return self._un(_L.mpc_rsqrt, "mpc_rsqrt", x, out, off, ctypes.byref(p))

    def _act(self, fn, name, x, off, knobs, out):
        k = dict(knobs)
        coeffs = k.get("coeffs")
        arr = (ctypes.c_double * len(coeffs))(*coeffs) if coeffs else None
        p = ActP(FORM[k["form"]], int(k.get("degree", 0)), float(k.get("B", 5.0)),
                 ctypes.cast(arr, ctypes.POINTER(ctypes.c_double)) if arr is not None else None,
                 int(k.get("erf_terms", 0)), int(k.get("window", 33)), int(k.get("basis", 0)))
        return self._un(fn, name, x, out, off, ctypes.byref(p))

    def gelu(self, x, off=0, out=None, **knobs):
        return self._act(_L.mpc_gelu, "mpc_gelu", x, off, default_act("gelu", **knobs), out)

    def silu(self, x, off=0, out=None, **knobs):
        return self._act(_L.mpc_silu, "mpc_silu", x, off, default_act("silu", **knobs), out)

    def sigmoid(self, x, off=0, out=None, **knobs):
        return self._act(_L.mpc_sigmoid, "mpc_sigmoid", x, off, default_act("sigmoid", **knobs), out)

    # ---- row ops ----
    def max(self, x, rows, cols, row_off=0, window=33, out=None):
        z = out if out is not None else self._empty(rows)
        self._stream()
        self._chk(_L.mpc_max(self._h, _sh(x), _sh(z), rows, cols, row_off, window), "mpc_max")
        return z

    def maxpool2d(self, x, N, C, H, W, k=3, stride=2, pad=1, img_off=0, window=33, out=None):
        Ho, Wo = (H + 2 * pad - k) // stride + 1, (W + 2 * pad - k) // stride + 1
        z = out if out is not None else self._empty(N * C * Ho * Wo)
        self._stream()
        self._chk(_L.mpc_maxpool2d(self._h, _sh(x), _sh(z), N, C, H, W, k, stride, pad, img_off, window),
                  "mpc_maxpool2d")
        return z

    def softmax(self, x, rows, cols, row_off=0, window=33, exp_t=8, exp_clamp=0, exp_window=33,
                recip_iters=10, recip_t=8, recip_clamp=0, recip_window=33, exp_square=0, recip_square=0,
                bcast=0, causal=0, out=None):
        p = SoftmaxP(window, ExpP(exp_t, int(exp_clamp), exp_window, int(exp_square)),
                     NrP(recip_iters, ExpP(recip_t, int(recip_clamp), recip_window, int(recip_square))), int(bcast),
                     int(causal))
        z = out if out is not None else self._empty(rows * cols)
        self._stream()
        self._chk(_L.mpc_softmax(self._h, _sh(x), _sh(z), rows, cols, row_off, ctypes.byref(p)), "mpc_softmax")
        return z

    def softmax_hostio(self, hx, hz, rows, cols, row_off=0, chunk_rows=1536, window=33, exp_t=8, exp_clamp=0,
                       exp_window=33, recip_iters=10, recip_t=8, recip_clamp=0, recip_window=33, exp_square=0,
                       recip_square=0, bcast=0, causal=0):
        """Softmax over HOST buffers (hx, hz: per-party CPU uint64 tensors, pinned): chunked, with the
        H2D copies, the compute and the D2H copies of neighbouring chunks overlapped."""
        p = SoftmaxP(window, ExpP(exp_t, int(exp_clamp), exp_window, int(exp_square)),
                     NrP(recip_iters, ExpP(recip_t, int(recip_clamp), recip_window, int(recip_square))), int(bcast),
                     int(causal))
        self._stream()
        self._chk(_L.mpc_softmax_hostio(self._h, _sh_host(hx), _sh_host(hz), rows, cols, row_off, ctypes.byref(p),
                                        chunk_rows), "mpc_softmax_hostio")
        return hz

    def layernorm(self, x, rows, cols, row_off=0, eps=1e-5, mean_mode=0, rsqrt_iters=3, rsqrt_t=8,
                  rsqrt_clamp=0, rsqrt_window=33, rsqrt_square=0, bcast=0, out=None):
        p = LnP(eps, mean_mode, NrP(rsqrt_iters, ExpP(rsqrt_t, int(rsqrt_clamp), rsqrt_window, int(rsqrt_square))),
                int(bcast))
        z = out if out is not None else self._empty(rows * cols)
        self._stream()
        self._chk(_L.mpc_layernorm(self._h, _sh(x), _sh(z), rows, cols, row_off, ctypes.byref(p)),
                  "mpc_layernorm")
        return z
