"""Two-process MPC_MODE_PAIR check: ranks 0 and 1 are party 0 and party 1 in
separate processes, each with its own mpc_ctx, exchanging every opening through the other
process's cudaIpc-mapped exchange memory -- the remote code path bench.py runs for N > 1.
With one GPU both processes share cuda:0 (the driver time-slices their contexts, so every
exchange round costs a context switch: correctness only, tiny shapes); with two or more GPUs
rank r uses cuda:r.  Each op's output shares are gathered on rank 0 and compared bit for bit
with MPC_MODE_BOTH on the same seeds and step ids (share, mul, ReLU, GELU, softmax dense /
cone + square triples / causal, LayerNorm, Beaver matmul, broadcast-triple mul / softmax /
LayerNorm), and an open to party 1 only.

  python tools/pair_ipc_check.py             (prints PAIR_IPC_OK on success, exit code 0)
  python tools/pair_ipc_check.py --mismatch  (debug header check: the parties issue different ops;
                                              prints PAIR_IPC_PROTOCOL_DETECTED)
  python tools/pair_ipc_check.py --exchange=0 (the LL wire format instead of the LL63 default)
  python tools/pair_ipc_check.py --dealer    (party 1's context is created WITHOUT K_0 (key_p0 = 0) and
                                              reads its corrections from a trusted-dealer stream made
                                              offline by an MPC_MODE_DEALER context)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import workloads  # noqa: E402


def ops(c, x, party, n_rows, n_cols, matmul=True):
    """The op sequence both modes run; returns the list of this party's output shares."""
    out = []
    xs = x if x is not None else None
    if c.mode in (1, 3) and party == 1:
        s = c.share(None, owner=0, n=n_rows * n_cols)
    else:
        s = c.share(xs, owner=0)
    out.append(s)
    out.append(c.mul(s, s, trunc_bits=16))
    out.append(c.relu(s))
    out.append(c.gelu(s, form="poly_abs", degree=4))
    out.append(c.softmax(s, n_rows, n_cols))
    out.append(c.layernorm(s, n_rows, n_cols))
    c.set_ltz_circuit(1)
    out.append(c.relu(s))
    out.append(c.softmax(s, n_rows, n_cols, exp_square=1, recip_square=1))
    c.set_ltz_circuit(0)
    out.append(c.softmax(s, n_rows, n_cols, causal=1))
    # X = s as n_rows x n_cols, Y = the same buffer as n_cols x n_rows (tensor-core engine)
    if matmul:
        out.append(c.matmul(s, s, 1, n_rows, n_cols, n_rows, trunc_bits=16))
    # broadcast triple (NEXT #2): per-row record scratch is per party in PAIR
    out.append(c.mul_bcast(s, s, n_rows, n_cols, trunc_bits=16))
    out.append(c.softmax(s, n_rows, n_cols, bcast=1))
    out.append(c.layernorm(s, n_rows, n_cols, bcast=1))
    return out


def worker(rank, world, port, q, mismatch=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2511_19711_b200 as m
    from paper_2511_19711_b200 import pair
    ngpu = torch.cuda.device_count()
    dev = rank % ngpu
    torch.cuda.set_device(dev)
    rows, cols = 32, 64
    x = torch.from_numpy(workloads.softmax_inputs(rows, cols).ravel()).cuda(dev)
    keys = workloads.keys(2)
    dealer = "--dealer" in sys.argv
    if dealer and rank == 1:
        # party 1 never receives K_0: its corrections come from the dealer's offline pass
        c = m.Ctx(keys["key_share"], 0, keys["key_p1"], dev, mode=m.binding.MODE_PAIR, party=1)
        d = m.Ctx.dealer(keys, device=dev)
        d.set_step(c.step)
        ops(d, None, 1, rows, cols)
        d.open_to(m.Ctx.like(rows * cols), 1)          # the final open's (empty) segment
        c.set_corrections(d.dealer_stream())
    else:
        c = m.Ctx.for_cfg(keys, device=dev, mode=m.binding.MODE_PAIR, party=rank)
    if "--exchange=0" in sys.argv:
        c.set_exchange(0)                             # LL instead of the LL63 default
    pair.connect(c)
    if mismatch:
        # debug header check: party 0 issues mul, party 1 square (same step count and rounds, so
        # the exchange itself completes) -- both must report MPC_ERR_PROTOCOL at sync
        c.set_debug(True)
        s = c.share(x if rank == 0 else None, owner=0, n=rows * cols)
        c.sync()
        if rank == 0:
            c.mul(s, s, trunc_bits=16)
        else:
            c.square(s, trunc_bits=16)
        try:
            c.sync()
            got = "OK"
        except m.MPCError as e:
            got = str(e)
        res = [None, None]
        dist.all_gather_object(res, got)
        if rank == 0:
            q.put([] if all("PROTOCOL" in r for r in res) else [("mismatch", res)])
        dist.barrier()
        dist.destroy_process_group()
        return
    res = ops(c, x if rank == 0 else None, rank, rows, cols)
    ring1, _ = c.open_to(res[0], 1)                   # only party 1 learns rec(x)
    c.sync()
    if dealer and rank == 1 and c.corrections_left() != 0:
        raise RuntimeError(f"party 1 left {c.corrections_left()} correction segments")
    mine = [r[rank].cpu().numpy() for r in res] + [ring1.cpu().numpy()]
    gathered = [None, None]
    dist.all_gather_object(gathered, mine)
    if rank == 0:
        b = m.Ctx.for_cfg(keys, device=dev)
        ref = ops(b, x, 0, rows, cols)
        ring_ref, _ = b.open(ref[0])
        torch.cuda.synchronize()
        bad = []
        for k, r in enumerate(ref):
            for p in (0, 1):
                if not np.array_equal(gathered[p][k], r[p].cpu().numpy()):
                    bad.append((k, p))
        if not np.array_equal(gathered[1][-1], ring_ref.cpu().numpy()):
            bad.append(("open_to", 1))
        if np.any(gathered[0][-1]):                   # party 0 received nothing, wrote nothing
            bad.append(("open_to", 0))
        q.put(bad)
    dist.barrier()
    dist.destroy_process_group()


def main():
    port = 29600 + (os.getpid() % 1000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mismatch = "--mismatch" in sys.argv
    mp.start_processes(worker, args=(2, port, q, mismatch), nprocs=2, join=True, start_method="spawn")
    bad = q.get(timeout=5)
    if bad:
        print("PAIR_IPC_MISMATCH", bad)
        sys.exit(1)
    print(("PAIR_IPC_PROTOCOL_DETECTED" if mismatch else "PAIR_IPC_OK") + f" ({torch.cuda.device_count()} GPU(s))")


if __name__ == "__main__":
    main()
