"""The library's launches are CUDA-graph capturable (stream capture of whole MPC ops; the ctx
switches to the capturing stream without cross-capture dependencies): a captured and replayed
softmax / GELU / matmul gives the eager call's output shares at the same step ids."""
import pytest

import workloads

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def m():
    import paper_2511_19711_b200 as mod
    return mod


def test_graph_replay_equals_eager(m):
    c = m.Ctx.for_cfg(workloads.keys(2))
    x = c.share(torch.from_numpy(workloads.softmax_inputs(96, 128)).cuda())
    g = c.share(torch.from_numpy(workloads.act_inputs(4096)).cuda())
    a = c.share(torch.from_numpy(workloads.act_inputs(2 * 64 * 32)).cuda())
    s0 = c.step
    z1 = c.softmax(x, 96, 128)
    y1 = c.gelu(g, form="poly_abs", degree=4)
    w1 = c.matmul(a, a, 2, 64, 32, 64)
    torch.cuda.synchronize()
    z2, y2, w2 = c._empty(96 * 128), c._empty(4096), c._empty(2 * 64 * 64)
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):                       # warm-up on a side stream (scratch sized)
        c.set_step(s0, force=True)
        c.softmax(x, 96, 128, out=z2)
    torch.cuda.current_stream().wait_stream(st)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    c.set_step(s0, force=True)
    with torch.cuda.graph(graph):
        c.softmax(x, 96, 128, out=z2)
        c.gelu(g, form="poly_abs", degree=4, out=y2)
        c.matmul(a, a, 2, 64, 32, 64, out=w2)
    for t in (*z2, *y2, *w2):
        t.zero_()
    graph.replay()
    torch.cuda.synchronize()
    for e, r in ((z1, z2), (y1, y2), (w1, w2)):
        assert torch.equal(e[0], r[0]) and torch.equal(e[1], r[1])
