"""Quick BOTH-mode timings of the hot ops on cuda:0 (CUDA events, L2 flushed between reps)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_19711_b200 as m
import workloads

flush = torch.empty(128 << 20, dtype=torch.int32, device="cuda")

def t(c, fn, reps=10):
    fn(); torch.cuda.synchronize()
    c.reset_stats()
    tot = 0.0
    for i in range(reps):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    ms = tot / reps
    ph = c.stats()["philox_calls"] / reps
    return f"{ms:.4f} ms  {ph / ms / 1e6:.1f} Gphilox/s"

mode = int(sys.argv[1]) if len(sys.argv) > 1 else 0
c = m.Ctx.for_cfg(workloads.keys(2), mode=mode)
sh = lambda x: c.share(torch.from_numpy(x.ravel()).cuda())
rows, cols = workloads.SHAPES["cfg2_softmax"]
x = sh(workloads.softmax_inputs(rows, cols))
print("softmax cfg2 ", t(c, lambda: c.softmax(x, rows, cols)))
c.set_ltz_circuit(1)
print("softmax cone ", t(c, lambda: c.softmax(x, rows, cols)))
print("softmax c+sq ", t(c, lambda: c.softmax(x, rows, cols, exp_square=1, recip_square=1)))
c.set_ltz_circuit(0)
g = sh(workloads.normal_inputs(workloads.SHAPES["cfg3_gelu"], 3))
print("gelu cfg3    ", t(c, lambda: c.gelu(g, form="poly_abs", degree=4)))
c.set_ltz_circuit(1)
print("gelu cone    ", t(c, lambda: c.gelu(g, form="poly_abs", degree=4)))
c.set_ltz_circuit(0)
r = sh(workloads.relu_inputs(32 * 64 * 112 * 112 // 4))
print("relu 6.4M    ", t(c, lambda: c.relu(r)))
c.set_ltz_circuit(1)
print("relu cone    ", t(c, lambda: c.relu(r)))
c.set_ltz_circuit(0)
ln = sh(workloads.layernorm_inputs(8192, 768))
print("ln 8192x768  ", t(c, lambda: c.layernorm(ln, 8192, 768)))
s2 = sh(workloads.softmax_inputs(12288, 1024))
print("softmax1024  ", t(c, lambda: c.softmax(s2, 12288, 1024)))
mm = sh(workloads.act_inputs(1 << 24))
print("mul 16M      ", t(c, lambda: c.mul(mm, mm, trunc_bits=16)))
e = sh(workloads.exp_inputs(1 << 22))
print("exp t8 4M    ", t(c, lambda: c.exp(e)))
if mode:
    c.sync()
