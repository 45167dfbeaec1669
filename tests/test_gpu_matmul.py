"""GPU parity for the Beaver matrix multiplication:
bit-exact shares vs the oracle in MPC_MODE_BOTH and the PAIR protocol (loopback), ragged
shapes (not multiples of the 64 x 64 tile), batches with a global offset, truncation."""
import numpy as np
import pytest

import workloads
from oracle import Oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def m():
    import paper_2511_19711_b200 as mod
    return mod


def np_(t):
    return t.cpu().numpy()


def same(g, o):
    a0, a1 = np_(g[0]), np_(g[1])
    bad = np.nonzero((a0 != o[0]) | (a1 != o[1]))[0]
    assert bad.size == 0, f"{bad.size} mismatching shares, first at {bad[:5]}"


@pytest.mark.parametrize("batch,M,K,N,boff,tb", [(1, 1, 1, 1, 0, 0), (1, 5, 7, 3, 0, 16), (2, 64, 64, 64, 1, 16),
                                                 (3, 70, 33, 129, 5, 16), (1, 128, 200, 65, 0, 0),
                                                 (1, 257, 96, 130, 2, 16)])
@pytest.mark.parametrize("engine", [1, 2])
def test_matmul_vs_oracle(m, batch, M, K, N, boff, tb, engine):
    keys = workloads.keys(2)
    c = m.Ctx.for_cfg(keys)
    c.set_matmul_engine(engine)
    c.set_step(3)
    o = Oracle.for_cfg(keys, 3)
    x = workloads.act_inputs(batch * M * K, lo=-2, hi=2)
    y = workloads.act_inputs(batch * K * N, seed_cfg=7, lo=-2, hi=2)
    gx, gy = c.share(torch.from_numpy(x).cuda()), c.share(torch.from_numpy(y).cuda())
    ox, oy = o.share(x), o.share(y)
    same(c.matmul(gx, gy, batch, M, K, N, batch_off=boff, trunc_bits=tb),
         o.matmul(ox, oy, batch, M, K, N, batch_off=boff, trunc_bits=tb))
    assert c.step == o.step


def test_matmul_bert_attention_scores_sampled(m):
    """BERT-base QK^T shape (12 heads x 128 x 64 x 128, 2 sequences): reconstruction against the
    float product of the decoded inputs, shares bit-exact on one sampled head."""
    batch, M, K, N = 24, 128, 64, 128
    keys = workloads.keys(2)
    c = m.Ctx.for_cfg(keys)
    x = workloads.normal_inputs(batch * M * K, 2, sigma=1.0)
    y = workloads.normal_inputs(batch * K * N, 2, sigma=1.0, stream=9)
    gx, gy = c.share(torch.from_numpy(x).cuda()), c.share(torch.from_numpy(y).cuda())
    s0 = c.step
    z = c.matmul(gx, gy, batch, M, K, N, trunc_bits=16)
    xd = np_(c.open(gx)[1]).reshape(batch, M, K)
    yd = np_(c.open(gy)[1]).reshape(batch, K, N)
    got = np_(c.open(z)[1]).reshape(batch, M, N)
    assert np.max(np.abs(got - xd @ yd)) <= 2 * 2.0 ** -16 + 1e-9
    h = 17
    o = Oracle.for_cfg(keys, s0)
    sl = slice(h * M * K, (h + 1) * M * K)
    slb = slice(h * K * N, (h + 1) * K * N)
    r = o.matmul((np_(gx[0])[sl], np_(gx[1])[sl]), (np_(gy[0])[slb], np_(gy[1])[slb]), 1, M, K, N,
                 batch_off=h, trunc_bits=16)
    zs = slice(h * M * N, (h + 1) * M * N)
    assert np.array_equal(np_(z[0])[zs], r[0]) and np.array_equal(np_(z[1])[zs], r[1])


def test_matmul_loopback(m):
    keys = workloads.keys(3)
    b = m.Ctx.for_cfg(keys)
    p = m.Ctx.for_cfg(keys, mode=m.binding.MODE_PAIR_LOOPBACK)
    for (batch, M, K, N) in [(2, 70, 33, 129), (1, 128, 64, 128)]:
        x = b.share(torch.from_numpy(workloads.act_inputs(batch * M * K)).cuda())
        y = b.share(torch.from_numpy(workloads.act_inputs(batch * K * N, seed_cfg=5)).cuda())
        p.set_step(b.step)
        zb = b.matmul(x, y, batch, M, K, N, batch_off=1, trunc_bits=16)
        zp = p.matmul(x, y, batch, M, K, N, batch_off=1, trunc_bits=16)
        torch.cuda.synchronize()
        assert torch.equal(zb[0], zp[0]) and torch.equal(zb[1], zp[1])
    p.sync()


def test_matmul_engines_agree_on_random_ring_values(m):
    """Full-range u64 shares (not fixed-point encodings): every limb of both operands is
    exercised; the tensor-core and SIMT engines must give the same shares."""
    keys = workloads.keys(4)
    batch, M, K, N = 2, 200, 160, 96
    g = np.random.default_rng(5)
    mk = lambda n: (torch.from_numpy(g.integers(0, 2**64, n, dtype=np.uint64, endpoint=False)).cuda(),
                    torch.from_numpy(g.integers(0, 2**64, n, dtype=np.uint64, endpoint=False)).cuda())
    x, y = mk(batch * M * K), mk(batch * K * N)
    out = []
    for engine in (1, 2):
        c = m.Ctx.for_cfg(keys)
        c.set_matmul_engine(engine)
        out.append(c.matmul(x, y, batch, M, K, N, batch_off=7))
    torch.cuda.synchronize()
    assert torch.equal(out[0][0], out[1][0]) and torch.equal(out[0][1], out[1][1])
    o = Oracle.for_cfg(keys)
    r = o.matmul((np_(x[0]), np_(x[1])), (np_(y[0]), np_(y[1])), batch, M, K, N, batch_off=7)
    same(out[1], r)


def test_matmul_tc_engine_rejects_long_k(m):
    c = m.Ctx.for_cfg(workloads.keys(1))
    c.set_matmul_engine(2)
    x = c.share(torch.zeros(6000, dtype=torch.float64).cuda())
    with pytest.raises(m.MPCError):
        c.matmul(x, x, 1, 1, 6000, 1)
