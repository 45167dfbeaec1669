"""Host-side logic of the PAIR bootstrap on CPU (gloo, world_size 2 and 4): pair layout and
the handle exchange that lets each party map its peer's receive buffers."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("pairmod", os.path.join(root, "paper_2511_19711_b200", "pair.py"))
    pairmod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(pairmod)

    class FakeCtx:
        def __init__(self):
            self.peer = None

        def pair_export(self):
            return bytes([rank]) * 64

        def pair_connect(self, h):
            self.peer = h

    c = pairmod.connect(FakeCtx())
    q.put((rank, pairmod.pair_layout(rank, world), c.peer))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_handle_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, (party, peer, pair, npairs), got in res:
        assert party == rank % 2 and peer == rank ^ 1 and pair == rank // 2 and npairs == world // 2
        assert got == bytes([rank ^ 1]) * 64


def test_pair_layout_rejects_odd_world():
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("pairmod", os.path.join(root, "paper_2511_19711_b200", "pair.py"))
    pairmod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(pairmod)
    with pytest.raises(ValueError):
        pairmod.pair_layout(0, 3)
