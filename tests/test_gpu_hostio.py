"""mpc_softmax_hostio: the chunked, copy-overlapped host-buffer softmax gives the same output
shares as mpc_softmax on device buffers (same steps and units), in BOTH and PAIR loopback."""
import numpy as np
import pytest

import workloads

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def m():
    import paper_2511_19711_b200 as mod
    return mod


@pytest.mark.parametrize("rows,cols,chunk", [(12288, 128, 2048), (1000, 77, 96), (64, 1024, 32)])
@pytest.mark.parametrize("mode", [0, 2])
def test_hostio_equals_device_softmax(m, rows, cols, chunk, mode):
    keys = workloads.keys(2)
    c = m.Ctx.for_cfg(keys, mode=mode)
    x = c.share(torch.from_numpy(workloads.softmax_inputs(rows, cols)).cuda())
    s0 = c.step
    z = c.softmax(x, rows, cols, row_off=64)
    s1 = c.step
    hx = tuple(t.cpu().pin_memory() for t in x)
    hz = tuple(torch.empty_like(t).pin_memory() for t in hx)
    c.set_step(s0, force=True)
    c.softmax_hostio(hx, hz, rows, cols, row_off=64, chunk_rows=chunk)
    torch.cuda.synchronize()
    assert c.step == s1                     # the same step ids as one mpc_softmax call
    assert torch.equal(hz[0], z[0].cpu()) and torch.equal(hz[1], z[1].cpu())
    if mode:
        c.sync()


@pytest.mark.parametrize("mode", [0, 2])
def test_hostio_adjacent_party_buffers(m, mode):
    """Both parties' host shares in ONE pinned [2][n] tensor each way: every chunk's two party
    copies go as one pitched 2D DMA (copy_pair); same output shares as the device softmax."""
    keys = workloads.keys(2)
    rows, cols = 3000, 128
    c = m.Ctx.for_cfg(keys, mode=mode)
    x = c.share(torch.from_numpy(workloads.softmax_inputs(rows, cols)).cuda())
    s0 = c.step
    z = c.softmax(x, rows, cols)
    hin = torch.empty((2, rows * cols), dtype=torch.uint64).pin_memory()
    hout = torch.empty((2, rows * cols), dtype=torch.uint64).pin_memory()
    hin[0].copy_(x[0].cpu()); hin[1].copy_(x[1].cpu())
    c.set_step(s0, force=True)
    c.softmax_hostio((hin[0], hin[1]), (hout[0], hout[1]), rows, cols, chunk_rows=768)
    torch.cuda.synchronize()
    assert torch.equal(hout[0], z[0].cpu()) and torch.equal(hout[1], z[1].cpu())
    if mode:
        c.sync()
