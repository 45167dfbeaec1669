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
