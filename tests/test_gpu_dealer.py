"""The trusted dealer's correction stream ("distributed in advance by a
trusted third-party").  An MPC_MODE_DEALER context runs party 1's kernels in the dealer role and
writes party 1's correction words (Beaver / square / broadcast c1, AND-triple c1, daBit r1A);
party 1 then reads them instead of deriving them from K_0.  The output shares must be
bit-identical to MPC_MODE_BOTH's (hence to the oracle's) for every op, the stream must be consumed
exactly, and a stream recorded for other calls must be refused (MPC_ERR_PROTOCOL).  Loopback here;
tools/pair_ipc_check.py --dealer runs party 1 in its own process with key_p0 = 0."""
import pytest

import workloads

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def m():
    import paper_2511_19711_b200 as mod
    return mod


def eq(a, b):
    torch.cuda.synchronize()
    return torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


def run_case(m, n, fn, step=5, circuit=0, cfg=1, scale=1.0):
    """fn(ctx, x_shares) -> output shares; x = seeded U[-8, 8] * scale of n elements."""
    keys = workloads.keys(cfg)
    b = m.Ctx.for_cfg(keys)
    p = m.Ctx.for_cfg(keys, mode=m.binding.MODE_PAIR_LOOPBACK)
    d = m.Ctx.dealer(keys, target=m.binding.MODE_PAIR_LOOPBACK)
    for c in (b, p, d):
        c.set_ltz_circuit(circuit)
        c.set_step(step)
    xs = b.share(torch.from_numpy(workloads.act_inputs(n) * scale).cuda())
    p.set_step(b.step)
    d.set_step(b.step)
    zb = fn(b, xs)
    fn(d, m.Ctx.like(n))                     # offline: the dealer's pass over the same calls
    stream = d.dealer_stream()
    p.set_corrections(stream)
    zp = fn(p, xs)
    p.sync()
    assert p.corrections_left() == 0, "party 1 did not consume the whole stream"
    assert p.step == b.step == d.step
    return zb, zp, stream


CASES = {
    "mul": (10_001, lambda c, x: c.mul(x, x, off=2, trunc_bits=16)),
    "square": (4097, lambda c, x: c.square(x, trunc_bits=16)),
    "mul_bcast": (64 * 96, lambda c, x: c.mul_bcast(x, c.max(x, 64, 96), 64, 96, trunc_bits=16)),
    "cmp_w1": (4096 + 32, lambda c, x: c.cmp(x, window=1)),
    "cmp_w13": (4096 + 32, lambda c, x: c.cmp(x, window=13)),
    "cmp_w33": (4096 + 32, lambda c, x: c.cmp(x, window=33)),
    "cmp_w34": (4096 + 32, lambda c, x: c.cmp(x, window=34)),
    "cmp_w64": (4096 + 32, lambda c, x: c.cmp(x, window=64)),
    "relu": (8192, lambda c, x: c.relu(x)),
    "exp": (5000, lambda c, x: c.exp(x, t=8)),
    "exp_clamp": (5000, lambda c, x: c.exp(x, t=4, clamp=1)),
    "exp_square": (5000, lambda c, x: c.exp(x, t=8, square=1)),
    "recip": (3000, lambda c, x: c.recip(x)),
    "rsqrt": (3000, lambda c, x: c.rsqrt(x)),
    "gelu_abs": (4096, lambda c, x: c.gelu(x, form="poly_abs", degree=4)),
    "gelu_x_power": (4096, lambda c, x: c.gelu(x, form="poly_x", degree=4, basis=1)),
    "gelu_erf": (4096, lambda c, x: c.gelu(x, form="erf", erf_terms=8)),
    "silu": (4096, lambda c, x: c.silu(x, form="poly_abs", degree=4)),
    "sigmoid": (4096, lambda c, x: c.sigmoid(x, form="poly_x", degree=4)),
    "max": (64 * 37, lambda c, x: c.max(x, 64, 37)),
    "maxpool": (2 * 4 * 14 * 14, lambda c, x: c.maxpool2d(x, 2, 4, 14, 14)),
    "maxpool_5x5": (1 * 4 * 20 * 20, lambda c, x: c.maxpool2d(x, 1, 4, 20, 20, k=5, stride=2, pad=2)),
    "softmax": (96 * 128, lambda c, x: c.softmax(x, 96, 128)),
    "softmax_causal": (64 * 64, lambda c, x: c.softmax(x, 64, 64, causal=1)),
    "softmax_bcast_square": (64 * 128, lambda c, x: c.softmax(x, 64, 128, bcast=1, exp_square=1, recip_square=1)),
    "softmax_clamp": (64 * 100, lambda c, x: c.softmax(x, 64, 100, exp_clamp=1)),
    "softmax_wide_rows": (32 * 1024, lambda c, x: c.softmax(x, 32, 1024)),
    "layernorm": (64 * 768, lambda c, x: c.layernorm(x, 64, 768)),
    "layernorm_bcast_mode1": (64 * 300, lambda c, x: c.layernorm(x, 64, 300, bcast=1, mean_mode=1)),
    "layernorm_clamp": (64 * 256, lambda c, x: c.layernorm(x, 64, 256, rsqrt_clamp=1, rsqrt_t=4)),
    "open": (5000, lambda c, x: (c.mul(x, x, trunc_bits=16), c.open(x)[0])[0]),
    # the matrix triple: the dealer's GEMM writes C1 = (A0+A1)(B0+B1) - C0 as one segment
    "matmul_tc": (64 * 96, lambda c, x: c.matmul(x, x, 1, 64, 96, 64, trunc_bits=16)),
    "matmul_batched": (3 * 40 * 32, lambda c, x: c.matmul(x, x, 3, 40, 32, 40, batch_off=2)),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_dealer_stream_loopback_bit_identical(m, name):
    n, fn = CASES[name]
    zb, zp, stream = run_case(m, n, fn)
    assert eq(zb, zp), name


@pytest.mark.parametrize("name,w", [("relu", 21), ("relu", 33), ("relu", 64), ("gelu_abs", 33), ("softmax", 33),
                                    ("max", 33)])
def test_dealer_stream_carry_cone(m, name, w):
    n, fn = CASES[name]
    f = (lambda c, x: c.relu(x, window=w)) if name == "relu" else fn
    zb, zp, _ = run_case(m, n, f, circuit=1, scale=0.25)
    assert eq(zb, zp), (name, w)


def test_dealer_stream_words_per_op(m):
    """The stream carries party 1's corrections only: a Beaver multiply is one word per element."""
    n = 1 << 20
    _, _, (_, nwords, segs) = run_case(m, n, lambda c, x: c.mul(x, x, trunc_bits=16))
    assert len(segs) == 1
    g = segs[0]
    assert g.depth * g.threads >= n and nwords == g.depth * g.threads
    # one c1 per unit, plus at most one pass (2 unit pairs per lane) of padding in the last pass
    assert nwords <= n + 4 * g.threads, (nwords, n, g.threads)


def test_dealer_stream_mismatch_is_refused(m):
    keys = workloads.keys(1)
    p = m.Ctx.for_cfg(keys, mode=m.binding.MODE_PAIR_LOOPBACK)
    d = m.Ctx.dealer(keys, target=m.binding.MODE_PAIR_LOOPBACK)
    xs = p.share(torch.from_numpy(workloads.act_inputs(4096)).cuda())
    d.set_step(p.step)
    d.relu(m.Ctx.like(4096))
    p.set_corrections(d.dealer_stream())
    with pytest.raises(m.MPCError, match="PROTOCOL"):
        p.exp(xs, t=8)                       # the stream holds a ReLU's corrections
    p.set_corrections(d.dealer_stream())
    p.relu(xs)
    with pytest.raises(m.MPCError, match="PROTOCOL"):
        p.relu(xs)                           # exhausted
    p.set_corrections(None)
    assert p.corrections_left() == -1
    p.relu(xs)                               # back to the simulated dealer
    p.sync()


def test_dealer_hostio_softmax(m):
    """The host-buffer softmax's chunks in PAIR_LOOPBACK read their corrections from the stream."""
    keys = workloads.keys(2)
    rows, cols = 256, 128
    b = m.Ctx.for_cfg(keys)
    p = m.Ctx.for_cfg(keys, mode=m.binding.MODE_PAIR_LOOPBACK)
    d = m.Ctx.dealer(keys, target=m.binding.MODE_PAIR_LOOPBACK)
    xs = b.share(torch.from_numpy(workloads.softmax_inputs(rows, cols).ravel()).cuda())
    p.set_step(b.step)
    d.set_step(b.step)
    zb = b.softmax(xs, rows, cols)
    hx = tuple(t.cpu().pin_memory() for t in xs)
    hz = tuple(torch.empty_like(t).pin_memory() for t in hx)
    d.softmax_hostio((torch.empty(rows * cols, dtype=torch.uint64), torch.empty(rows * cols, dtype=torch.uint64)),
                     (torch.empty(rows * cols, dtype=torch.uint64), torch.empty(rows * cols, dtype=torch.uint64)),
                     rows, cols, chunk_rows=64)
    p.set_corrections(d.dealer_stream())
    p.softmax_hostio(hx, hz, rows, cols, chunk_rows=64)
    p.sync()
    torch.cuda.synchronize()
    assert p.corrections_left() == 0
    assert torch.equal(hz[0], zb[0].cpu()) and torch.equal(hz[1], zb[1].cpu())


def test_dealer_matmul_simt_engine(m):
    def fn(c, x):
        c.set_matmul_engine(1)
        return c.matmul(x, x, 2, 24, 40, 24, trunc_bits=16)
    zb, zp, _ = run_case(m, 2 * 24 * 40, fn)
    assert eq(zb, zp)


def test_dealer_refuses_party0(m):
    keys = workloads.keys(1)
    d = m.Ctx.dealer(keys)
    b = m.Ctx.for_cfg(keys)
    with pytest.raises(m.MPCError, match="INVALID"):
        b.set_corrections(d.dealer_stream())
