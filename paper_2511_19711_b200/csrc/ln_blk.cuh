// ln_blk.cuh -- LayerNorm (BOTH) on row blocks staged in shared memory by bulk copies.
// LAYERNORM: mu = rowsum(x) E(1/d) (or per-share floor / d), c = x - mu,
// v = mean(rowsum MT(c, c)) + eps, r = RSQRT(v) (row units), out = MT(c, r) (element units).
// A CTA walks row blocks of RB rows (round-robin over the grid); each block's two share arrays are
// ONE contiguous range per share, so a block arrives as two cp.async.bulk copies completing on an
// mbarrier, double-buffered: block k+1 is in flight while block k computes.  x is read from HBM
// exactly once (k_ln_fused reads it three times and, with the output, overflows L2: 240 MB read for
// 100 MB of input at cfg5).  W = 8 / RB warps share a row (chunk ranges of its element pairs); the
// row sums combine through shared memory at two CTA barriers per block; every warp of a row runs the
// row's RSQRT chain from its own table of the chain's triples (lanes 0..ns-1 generate one step each,
// kernels.cuh row_tab_step), so the chain needs no barrier.  Same steps, units, PRG words and output
// bits as k_ln_fused.  BOTH only, no clamp in the rsqrt's exp, no broadcast triple, ns <= 32.
#pragma once
#include "kernels.cuh"
#include "matmul_tc.cuh"

namespace mpc {

struct LnBArgs {
    u32 s_sq, s_rs, s_mul; NrK rk; SP x; SO z; i64 rows, cols; u64 row_off;
    int mean_mode; u64 e_invd, e_eps;
    int RB;                 // rows per block: 1, 2, 4 or 8 (W = 8 / RB warps per row)
};
__host__ __device__ inline size_t lnb_smem_bytes(i64 cols, int RB) { return sizeof(u64) * 4 * (size_t)RB * (size_t)cols; }

template <class PA>
__global__ void __launch_bounds__(MPC_ROW_TPB, MPC_SM_MINB) k_ln_blk(const __grid_constant__ PA pa, LnBArgs a)
{
    extern __shared__ __align__(128) u64 lbuf[];              // [2 buffers][2 shares][RB x C]
    __shared__ __align__(8) u64 bar[2];
    __shared__ u64 part[MPC_ROW_TPB / 32][2][2];              // [warp][mu | var][share]
    __shared__ u64 tabs[MPC_ROW_TPB / 32][MPC_NR_TAB_MAX_STEPS * NR_TAB_F];
    int cta, ncta;
    auto pr = pa.make(cta, ncta);
    using P = decltype(pr);
    using S = typename P::S;
    static_assert(!P::kPair, "BOTH only");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
    const i64 C = a.cols, hc = C / 2, nk = (hc + 31) / 32;   // pairs per row, pair chunks per lane
    const int RB = a.RB, W = NW / RB;                        // warps per row
    const int rw = warp / W, hf = warp % W;                   // the warp's row in the block, its part
    const i64 kb = hf * nk / W, ke = (hf + 1) * nk / W;       // the warp's chunks of that row
    const int ns = nr_tab_steps(1, a.rk.exp.t, a.rk.iters);
    const i64 nblk = (a.rows + RB - 1) / RB, bw = (i64)RB * C;
    u64* T = tabs[warp];
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](i64 blk, int b) {                        // thread 0: block blk -> buffer b
        const i64 r0 = blk * RB, R = min((i64)RB, a.rows - r0);
        const u32 bytes = (u32)(R * C * 8);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic reads before async writes
        mbar_expect_tx(&bar[b], 2 * bytes);
        bulk_g2s(lbuf + (i64)b * 2 * bw, a.x.p[0] + r0 * C, bytes, &bar[b]);
        bulk_g2s(lbuf + (i64)b * 2 * bw + bw, a.x.p[1] + r0 * C, bytes, &bar[b]);
    };
    if (threadIdx.x == 0 && cta < nblk) issue(cta, 0);
    u32 ph0 = 0, ph1 = 0;
    int b = 0;
    for (i64 blk = cta; blk < nblk; blk += ncta, b ^= 1) {
        if (threadIdx.x == 0 && blk + ncta < nblk) issue(blk + ncta, b ^ 1);
        mbar_wait(&bar[b], b ? ph1 : ph0);
        if (b) ph1 ^= 1; else ph0 ^= 1;
        const i64 r0 = blk * RB;
        const int R = (int)min((i64)RB, a.rows - r0);
        const bool live = rw < R;                             // warp-uniform
        u64* xb = lbuf + (i64)b * 2 * bw + (i64)rw * C;
        const SP xs{{xb, xb + bw}};
        const u64 g = a.row_off + (u64)(r0 + rw);             // global row = the rsqrt's unit
        const u64 ub = g * (u64)C;                            // even (C is)
        const SO zr{{a.z.p[0] + (r0 + rw) * C, a.z.p[1] + (r0 + rw) * C}};
        // A: row sum -> mu
        S acc = pr.zero();
        if (live)
            for (i64 k = kb; k < ke; ++k) {
                const i64 p2 = lane + 32 * k;
                if (p2 < hc) {
                    S xa, xc;
                    pr.ld_pair(xs, 2 * p2, true, true, xa, xc);
                    acc = pr.add(acc, pr.add(xa, xc));
                }
            }
        acc = pr.sumw(acc);
        if (lane == 0) { part[warp][0][0] = acc.s0; part[warp][0][1] = acc.s1; }
        // the chain's triples: lane j < ns generates step j (data-independent)
        if (live && lane < ns) row_tab_step(*pr.Kp, g, a.s_rs + (u32)lane, lane < a.rk.exp.t && a.rk.exp.sq, T + lane * NR_TAB_F);
        __syncthreads();
        S mu = pr.zero();
        for (int q = 0; q < W; ++q) mu = pr.add(mu, S{part[rw * W + q][0][0], part[rw * W + q][0][1]});
        mu = a.mean_mode == 0 ? pr.mulf(mu, a.e_invd) : pr.divp(mu, C);
        // B: sum of MT(c, c), c = x - mu
        S qs = pr.zero();
        if (live)
            for (i64 k = kb; k < ke; ++k) {
                const i64 p2 = lane + 32 * k;
                S xa = pr.zero(), xc = pr.zero();
                if (p2 < hc) pr.ld_pair(xs, 2 * p2, true, true, xa, xc);
                u64 u[1] = {ub + 2 * (u64)p2};
                S ca[1] = {pr.sub(xa, mu)}, cb[1] = {pr.sub(xc, mu)}, za[1], zz[1];
                pr.template bm2v<1>(u, a.s_sq, ca, ca, cb, cb, za, zz);
                if (p2 < hc) qs = pr.add(qs, pr.add(pr.shr_(za[0], FRAC), pr.shr_(zz[0], FRAC)));
            }
        qs = pr.sumw(qs);
        if (lane == 0) { part[warp][1][0] = qs.s0; part[warp][1][1] = qs.s1; }
        __syncthreads();
        if (live) {
            S var = pr.zero();
            for (int q = 0; q < W; ++q) var = pr.add(var, S{part[rw * W + q][1][0], part[rw * W + q][1][1]});
            var = a.mean_mode == 0 ? pr.mulf(var, a.e_invd) : pr.divp(var, C);
            var = pr.addp(var, a.e_eps);
            // C: r = RSQRT(var), unit g, every lane the same chain from the warp's table
            BothRowTabP tp;
            tp.Kp = pr.Kp; tp.T = T; tp.sb = a.s_rs;
            const S rr = rsqrt_group<false>(tp, g, g >> 5, a.s_rs, a.rk, var, lane);
            // D: out = MT(c, r)
            for (i64 k = kb; k < ke; ++k) {
                const i64 p2 = lane + 32 * k;
                S xa = pr.zero(), xc = pr.zero();
                if (p2 < hc) pr.ld_pair(xs, 2 * p2, true, true, xa, xc);
                u64 u[1] = {ub + 2 * (u64)p2};
                S ca[1] = {pr.sub(xa, mu)}, cb[1] = {pr.sub(xc, mu)}, rv[1] = {rr}, za[1], zz[1];
                pr.template bm2v<1>(u, a.s_mul, ca, rv, cb, rv, za, zz);
                if (p2 < hc) pr.st_pair(zr, 2 * p2, true, true, pr.shr_(za[0], FRAC), pr.shr_(zz[0], FRAC));
            }
        }
        __syncthreads();                                      // buffer b and part[] are free
    }
    pa.done(pr);
}

}  // namespace mpc
