"""GPU parity for the SURVEY §8(f) NEXT #2 variants: the broadcast triple (mpc_mul_bcast, the
softmax / layernorm `bcast` knob) and power-basis polynomials (the `basis`
knob of mpc_act_p).  Bit-exact on every share against the oracle, in
MPC_MODE_BOTH (Kogge-Stone and carry-cone LTZ) and in the PAIR protocol (loopback)."""
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


def ctx(m, cfg=1, step=0, mode=None):
    keys = workloads.keys(cfg)
    kw = {} if mode is None else {"mode": mode}
    c = m.Ctx.for_cfg(keys, **kw)
    c.set_step(step)
    return c, Oracle.for_cfg(keys, step)


@pytest.mark.parametrize("rows,cols,off,row_off,tb", [(1, 1, 0, 0, 0), (7, 13, 3, 5, 16), (64, 128, 0, 32, 16),
                                                      (1000, 3, 10, 7, 0), (5, 4097, 1, 0, 16)])
def test_mul_bcast(m, rows, cols, off, row_off, tb):
    c, o = ctx(m, step=4)
    x = workloads.act_inputs(rows * cols)
    y = workloads.recip_inputs(rows)
    gx, gy = c.share(torch.from_numpy(x).cuda()), c.share(torch.from_numpy(y).cuda())
    ox, oy = o.share(x), o.share(y)
    same(c.mul_bcast(gx, gy, rows, cols, off=off, row_off=row_off, trunc_bits=tb),
         o.mul_bcast(ox, oy, rows, cols, off=off, row_off=row_off, trunc_bits=tb))
    assert c.step == o.step


@pytest.mark.parametrize("rows,cols,clamp", [(64, 128, 0), (32, 1024, 0), (45, 77, 1), (40, 9, 0)])
@pytest.mark.parametrize("circuit", [0, 1])
def test_softmax_bcast(m, rows, cols, clamp, circuit):
    c, o = ctx(m, 2, step=1)
    c.set_ltz_circuit(circuit)
    x = workloads.softmax_inputs(rows, cols, spike=bool(clamp))
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    kw = dict(exp_clamp=clamp, bcast=1)
    same(c.softmax(gx, rows, cols, row_off=32, **kw), o.softmax(ox, rows, cols, row_off=32, **kw))
    assert c.step == o.step


@pytest.mark.parametrize("rows,cols,mean_mode", [(64, 768, 0), (45, 100, 1)])
def test_layernorm_bcast(m, rows, cols, mean_mode):
    c, o = ctx(m, 5, step=2)
    x = workloads.layernorm_inputs(rows, cols)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.layernorm(gx, rows, cols, row_off=64, mean_mode=mean_mode, bcast=1),
         o.layernorm(ox, rows, cols, row_off=64, mean_mode=mean_mode, bcast=1))


POWER = [("gelu", "poly_x", 4), ("gelu", "poly_x", 2), ("gelu", "poly_abs", 4), ("gelu", "poly_abs", 2),
         ("silu", "poly_abs", 4), ("silu", "poly_x", 4), ("sigmoid", "poly_x", 4), ("sigmoid", "poly_x", 2)]


@pytest.mark.parametrize("act,form,deg", POWER)
@pytest.mark.parametrize("circuit", [0, 1])
def test_power_basis(m, act, form, deg, circuit):
    c, o = ctx(m, step=4)
    c.set_ltz_circuit(circuit)
    n = 4096 + 99
    x = workloads.act_inputs(n)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    k = m.default_act(act, form, degree=deg, basis=1)
    g = getattr(c, act)(gx, off=0, form=form, degree=deg, basis=1)
    r = o.act(ox, act, form, deg, k["B"], k["coeffs"], basis=1)
    same(g, r)
    assert c.step == o.step


def test_power_basis_degree3_custom_coeffs(m):
    c, o = ctx(m, step=7)
    coeffs = [0.01, 0.5, 0.2, -0.03]
    x = workloads.act_inputs(2048)
    gx, ox = c.share(torch.from_numpy(x).cuda()), o.share(x)
    same(c.gelu(gx, form="poly_x", degree=3, B=4.0, coeffs=coeffs, basis=1),
         o.act(ox, "gelu", "poly_x", 3, 4.0, coeffs, basis=1))


def test_bad_knobs(m):
    c, _ = ctx(m)
    gx = c.share(torch.zeros(64, dtype=torch.float64).cuda())
    with pytest.raises(m.MPCError):
        c.gelu(gx, form="erf", erf_terms=8, basis=1)
    with pytest.raises(m.MPCError):
        c.mul_bcast(gx, c.share(torch.zeros(8, dtype=torch.float64).cuda()), 8, 8, trunc_bits=3)


# ------------------------------------------------------------- PAIR loopback ----
def eq(a, b):
    torch.cuda.synchronize()
    return torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


@pytest.mark.parametrize("circuit", [0, 1])
def test_next2_loopback(m, circuit):
    keys = workloads.keys(2)
    b = m.Ctx.for_cfg(keys)
    p = m.Ctx.for_cfg(keys, mode=m.binding.MODE_PAIR_LOOPBACK)
    b.set_ltz_circuit(circuit)
    p.set_ltz_circuit(circuit)
    x = b.share(torch.from_numpy(workloads.act_inputs(777 * 9)).cuda())
    y = b.share(torch.from_numpy(workloads.recip_inputs(777)).cuda())
    p.set_step(b.step)
    assert eq(b.mul_bcast(x, y, 777, 9, off=1, row_off=3, trunc_bits=16),
              p.mul_bcast(x, y, 777, 9, off=1, row_off=3, trunc_bits=16))
    s = b.share(torch.from_numpy(workloads.softmax_inputs(70, 128)).cuda())
    p.set_step(b.step)
    assert eq(b.softmax(s, 70, 128, bcast=1), p.softmax(s, 70, 128, bcast=1))
    ln = b.share(torch.from_numpy(workloads.layernorm_inputs(40, 768)).cuda())
    p.set_step(b.step)
    assert eq(b.layernorm(ln, 40, 768, bcast=1), p.layernorm(ln, 40, 768, bcast=1))
    g = b.share(torch.from_numpy(workloads.act_inputs(4096 + 64)).cuda())
    for form in ("poly_x", "poly_abs"):
        p.set_step(b.step)
        assert eq(b.gelu(g, form=form, degree=4, basis=1), p.gelu(g, form=form, degree=4, basis=1))
    p.set_step(b.step)
    assert eq(b.gelu(g, form="poly_x", degree=3, B=4.0, coeffs=[0.0, 0.5, 0.2, -0.03], basis=1),
              p.gelu(g, form="poly_x", degree=3, B=4.0, coeffs=[0.0, 0.5, 0.2, -0.03], basis=1))
    p.sync()
