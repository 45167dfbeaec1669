// plain.cuh -- plaintext fixed-point emulation of the approximation schedules (the auto-tuner's
// evaluator).
//
// CrypTorch's tuner scores a candidate set of approximations by running the approximated graph
// WITHOUT MPC ("directly lowering the graph to a (non-MPC) PyTorch GPU runtime").  Here
// the candidate schedules of DESIGN.md 2.5 run on the plaintext ring values (int64 at scale 2^16)
// with the same public constants, the same step structure and deterministic floor truncation:
// the MPC output equals this emulation up to the per-share truncation's (-1, 0] ulp per product
// (P:1016), so the emulation captures every approximation- and fixed-point-induced error at a
// fraction of the cost (no PRG, no openings).  One thread per element (one per row for the row
// ops); input / output are float64 device arrays.
#pragma once
#include "sched.cuh"

namespace mpc {

__device__ __forceinline__ i64 pl_mt(i64 x, i64 y) { return (i64)((u64)x * (u64)y) >> FRAC; }   // MT, floor
__device__ __forceinline__ i64 pl_mulf(i64 x, u64 e) { return (i64)((u64)x * e) >> FRAC; }      // pmulF
__device__ __forceinline__ i64 pl_ltz(i64 x, int w) { return (i64)(((u64)x >> (w - 1)) & 1ull); }

__device__ i64 pl_exp(i64 x, const ExpK& p)
{
    i64 y = (x >> p.t) + (i64)p.e_one;
    if (p.clamp) y = y * (1 - pl_ltz(x + (i64)p.e_2t, p.w));          // value x mask, no truncation
    for (int k = 0; k < p.t; ++k) y = pl_mt(y, y);
    return y;
}
__device__ i64 pl_recip(i64 x, const NrK& p)
{
    const i64 g = pl_exp((i64)p.e_half - x, p.exp);
    i64 y = 3 * g + (i64)p.e_c003;
    for (int it = 0; it < p.iters; ++it) {
        const i64 q = pl_mt(x, y);
        y = pl_mt(y, (i64)p.e_two - q);
    }
    return y;
}
__device__ i64 pl_rsqrt(i64 x, const NrK& p)
{
    const i64 g = pl_exp(-((x >> 1) + (i64)p.e_02), p.exp);
    i64 y = pl_mulf(g, p.e_22) + (i64)p.e_02;
    for (int it = 0; it < p.iters; ++it) {
        const i64 q = pl_mt(y, y), r = pl_mt(x, q);
        y = pl_mulf(pl_mt(y, (i64)p.e_three - r), p.e_half);
    }
    return y;
}
__device__ i64 pl_poly(i64 v, const ActK& p, int d, const u64* c)
{
    if (p.basis) {                                                       // POWER
        i64 h = pl_mulf(v, c[1]);
        if (d >= 2) {
            const i64 v2 = pl_mt(v, v);
            h += pl_mulf(v2, c[2]);
            if (d >= 3) h += pl_mulf(pl_mt(v2, v), c[3]);
            if (d >= 4) h += pl_mulf(pl_mt(v2, v2), c[4]);
        }
        return h + (i64)c[0];
    }
    i64 h = pl_mulf(v, c[d]) + (i64)c[d - 1];                            // HORNER
    for (int k = d - 2; k >= 0; --k) h = pl_mt(h, v) + (i64)c[k];
    return h;
}
__device__ i64 pl_act(i64 x, const ActK& p)
{
    if (p.form == 2 || p.deg == 0) {
        const i64 nl = 1 - pl_ltz(x, p.w);
        return p.act == 2 ? nl << FRAC : x * nl;
    }
    const i64 l1 = pl_ltz(x + (i64)p.e_B, p.w), l2 = pl_ltz(x + (i64)p.e_mB, p.w);
    i64 h;
    if (p.form == 0) {
        h = pl_poly(x, p, p.deg, p.c);
    } else if (p.form == 1) {
        const i64 ax = x * (1 - 2 * pl_ltz(x, p.w));
        h = pl_mulf(x, p.e_half) + pl_poly(ax, p, p.deg, p.c);
    } else {
        const i64 z = pl_mulf(x, p.e_isqrt2), z2 = pl_mt(z, z);
        ActK q = p;
        q.basis = 0;
        const i64 S = pl_poly(z2, q, p.deg, p.c);
        const i64 erf = pl_mulf(pl_mt(z, S), p.e_2sqrtpi);
        h = pl_mulf(pl_mt(x, erf + (i64)p.e_one), p.e_half);
    }
    const i64 nl2 = 1 - l2;
    return h * (l2 - l1) + (p.act == 2 ? nl2 << FRAC : x * nl2);
}

__device__ __forceinline__ i64 pl_enc(double v) { return __double2ll_rn(v * 65536.0); }
__device__ __forceinline__ double pl_dec(i64 v) { return (double)v * (1.0 / 65536.0); }

// op: 0 exp, 1 recip, 2 rsqrt, 3 activation (ActK), 4 softmax rows, 5 layernorm rows
struct PlainArgs {
    int op; ExpK ek; NrK nk; ActK ak; int w; int causal;   // causal: softmax row r sees columns <= r mod cols
    int mean_mode; u64 e_invd, e_eps;
    const double* x; double* y; i64 rows, cols;
};

__global__ void __launch_bounds__(256) k_plain(const __grid_constant__ PlainArgs a)
{
    const i64 stride = (i64)gridDim.x * blockDim.x;
    if (a.op <= 3) {
        const i64 n = a.rows * a.cols;
        for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += stride) {
            const i64 x = pl_enc(a.x[i]);
            const i64 r = a.op == 0 ? pl_exp(x, a.ek) : a.op == 1 ? pl_recip(x, a.nk) : a.op == 2 ? pl_rsqrt(x, a.nk)
                                                                                                : pl_act(x, a.ak);
            a.y[i] = pl_dec(r);
        }
        return;
    }
    for (i64 row = blockIdx.x * (i64)blockDim.x + threadIdx.x; row < a.rows; row += stride) {
        const double* xr = a.x + row * a.cols;
        double* yr = a.y + row * a.cols;
        if (a.op == 4) {                                  // SOFTMAX (causal 2.12)
            const i64 nv = a.causal ? row % a.cols + 1 : a.cols;    // visible columns
            // MAX_row as the schedule's half-split tree (R22) with the mux x_h + d (1 - LTZ_w(d)),
            // in the output row (reinterpreted as int64) as workspace; masked entries -2^(w-2)
            i64* v = reinterpret_cast<i64*>(yr);
            const i64 L = a.w >= 2 ? -((i64)1 << (a.w - 2)) : -1;
            for (i64 j = 0; j < a.cols; ++j) v[j] = j < nv ? pl_enc(xr[j]) : L;
            for (i64 m = a.cols; m > 1;) {
                const i64 h = m / 2;
                for (i64 i = 0; i < h; ++i) {
                    const i64 d = (i64)((u64)v[i] - (u64)v[i + h]);
                    v[i] = (i64)((u64)v[i + h] + (u64)d * (u64)(1 - pl_ltz(d, a.w)));
                }
                if (m & 1) v[h] = v[m - 1];
                m = h + (m & 1);
            }
            const i64 m = v[0];
            i64 S = 0;
            for (i64 j = 0; j < nv; ++j) S = (i64)((u64)S + (u64)pl_exp(pl_enc(xr[j]) - m, a.ek));
            const i64 r = pl_recip(S, a.nk);
            for (i64 j = 0; j < a.cols; ++j) yr[j] = j < nv ? pl_dec(pl_mt(pl_exp(pl_enc(xr[j]) - m, a.ek), r)) : 0.0;
        } else {                                          // LAYERNORM
            i64 s = 0;
            for (i64 j = 0; j < a.cols; ++j) s += pl_enc(xr[j]);
            const i64 mu = a.mean_mode == 0 ? pl_mulf(s, a.e_invd) : (s >= 0 ? s / a.cols : -((-s + a.cols - 1) / a.cols));
            i64 q = 0;
            for (i64 j = 0; j < a.cols; ++j) { const i64 c = pl_enc(xr[j]) - mu; q += pl_mt(c, c); }
            const i64 v = (a.mean_mode == 0 ? pl_mulf(q, a.e_invd) : (q >= 0 ? q / a.cols : -((-q + a.cols - 1) / a.cols)))
                          + (i64)a.e_eps;
            const i64 r = pl_rsqrt(v, a.nk);
            for (i64 j = 0; j < a.cols; ++j) yr[j] = pl_dec(pl_mt(pl_enc(xr[j]) - mu, r));
        }
    }
}

}  // namespace mpc
