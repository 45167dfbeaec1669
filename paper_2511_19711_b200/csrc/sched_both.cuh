// sched_both.cuh -- L2 fused schedules (MPC_MODE_BOTH) for one element / row unit:
// EXP, RECIP, RSQRT, HORNER and the segment forms of DESIGN.md 2.5.  Each function
// consumes step ids s, s+1, ... in exactly the order of the decomposition.
#pragma once
#include "proto_both.cuh"

namespace mpc {

// knobs with their public constants already encoded (E(c), host side)
struct ExpK { int t, clamp, w; u64 e_one, e_2t; };
struct NrK  { int iters; ExpK exp; u64 e_half, e_c003, e_two, e_three, e_02, e_22; };
constexpr int MAX_COEF = 13;
struct ActK {
    int act;          // 0 gelu, 1 silu, 2 sigmoid
    int form;         // 0 poly_x, 1 poly_abs, 2 relu, 3 erf
    int deg;          // polynomial degree (HORNER degree for erf = K-1)
    int w;
    u64 e_B, e_mB, e_half, e_one, e_isqrt2, e_2sqrtpi;
    u64 c[MAX_COEF];  // E(c_k) (poly) or E(a_k) (erf series)
};

__device__ __forceinline__ int exp_steps(const ExpK& e) { return e.t + 2 * e.clamp; }

// ---- EXP(x; t, clamp, w) ------------------------------------
// GROUP variant: lane <-> unit u (LTZ group q); usable with or without clamp.
template <bool WIDE>
__device__ __forceinline__ Sh exp_group(const Keys& K, u64 u, u64 q, u32 s, const ExpK& p, Sh x, int lane)
{
    Sh y = sh_addp(sh_shr(x, p.t), p.e_one);
    if (p.clamp) {
        const Sh l = ltz<WIDE>(K, q, s, p.w, sh_addp(x, p.e_2t), lane);
        y = bm(K, u, s + 1, y, sh_not(l));
        s += 2;
    }
    for (int k = 0; k < p.t; ++k) y = mt(K, u, s + k, y, y);
    return y;
}

// PAIR variant (no clamp): two consecutive units u (even), u+1 in one thread.
__device__ __forceinline__ void exp_pair(const Keys& K, u64 u, u32 s, const ExpK& p, Sh& y0, Sh& y1)
{
    y0 = sh_addp(sh_shr(y0, p.t), p.e_one);
    y1 = sh_addp(sh_shr(y1, p.t), p.e_one);
    for (int k = 0; k < p.t; ++k) {
        Sh a, b;
        bm2(K, u, s + k, y0, y0, y1, y1, a, b);
        y0 = sh_shr(a, FRAC); y1 = sh_shr(b, FRAC);
    }
}

// ---- RECIP(x; iters, exp) --------------------------------
template <bool WIDE>
__device__ __forceinline__ Sh recip_group(const Keys& K, u64 u, u64 q, u32 s, const NrK& p, Sh x, int lane)
{
    Sh g = exp_group<WIDE>(K, u, q, s, p.exp, sh_addp(sh_neg(x), p.e_half), lane);
    s += exp_steps(p.exp);
    Sh y = sh_addp(sh_muli(g, 3ull), p.e_c003);
    for (int it = 0; it < p.iters; ++it) {
        const Sh pr = mt(K, u, s, x, y);
        y = mt(K, u, s + 1, y, sh_addp(sh_neg(pr), p.e_two));
        s += 2;
    }
    return y;
}

__device__ __forceinline__ void recip_pair(const Keys& K, u64 u, u32 s, const NrK& p, Sh x0, Sh x1, Sh& y0, Sh& y1)
{
    Sh g0 = sh_addp(sh_neg(x0), p.e_half), g1 = sh_addp(sh_neg(x1), p.e_half);
    exp_pair(K, u, s, p.exp, g0, g1);
    s += exp_steps(p.exp);
    y0 = sh_addp(sh_muli(g0, 3ull), p.e_c003);
    y1 = sh_addp(sh_muli(g1, 3ull), p.e_c003);
    for (int it = 0; it < p.iters; ++it) {
        Sh a, b;
        bm2(K, u, s, x0, y0, x1, y1, a, b);
        a = sh_addp(sh_neg(sh_shr(a, FRAC)), p.e_two);
        b = sh_addp(sh_neg(sh_shr(b, FRAC)), p.e_two);
        Sh c, d;
        bm2(K, u, s + 1, y0, a, y1, b, c, d);
        y0 = sh_shr(c, FRAC); y1 = sh_shr(d, FRAC);
        s += 2;
    }
}

// ---- RSQRT(x; iters, exp) ---------------------------------
template <bool WIDE>
__device__ __forceinline__ Sh rsqrt_group(const Keys& K, u64 u, u64 q, u32 s, const NrK& p, Sh x, int lane)
{
    Sh g = exp_group<WIDE>(K, u, q, s, p.exp, sh_neg(sh_addp(sh_shr(x, 1), p.e_02)), lane);
    s += exp_steps(p.exp);
    Sh y = sh_addp(sh_mulf(g, p.e_22), p.e_02);
    for (int it = 0; it < p.iters; ++it) {
        const Sh qq = mt(K, u, s, y, y);
        const Sh pp = mt(K, u, s + 1, x, qq);
        const Sh uu = mt(K, u, s + 2, y, sh_addp(sh_neg(pp), p.e_three));
        y = sh_mulf(uu, p.e_half);
        s += 3;
    }
    return y;
}

__device__ __forceinline__ void rsqrt_pair(const Keys& K, u64 u, u32 s, const NrK& p, Sh x0, Sh x1, Sh& y0, Sh& y1)
{
    Sh g0 = sh_neg(sh_addp(sh_shr(x0, 1), p.e_02)), g1 = sh_neg(sh_addp(sh_shr(x1, 1), p.e_02));
    exp_pair(K, u, s, p.exp, g0, g1);
    s += exp_steps(p.exp);
    y0 = sh_addp(sh_mulf(g0, p.e_22), p.e_02);
    y1 = sh_addp(sh_mulf(g1, p.e_22), p.e_02);
    for (int it = 0; it < p.iters; ++it) {
        Sh a, b, c, d;
        bm2(K, u, s, y0, y0, y1, y1, a, b);
        a = sh_shr(a, FRAC); b = sh_shr(b, FRAC);
        bm2(K, u, s + 1, x0, a, x1, b, c, d);
        c = sh_addp(sh_neg(sh_shr(c, FRAC)), p.e_three);
        d = sh_addp(sh_neg(sh_shr(d, FRAC)), p.e_three);
        bm2(K, u, s + 2, y0, c, y1, d, a, b);
        y0 = sh_mulf(sh_shr(a, FRAC), p.e_half);
        y1 = sh_mulf(sh_shr(b, FRAC), p.e_half);
        s += 3;
    }
}

// ---- HORNER(v; c_0..c_d), d >= 1 ------------------------------------------------------
__device__ __forceinline__ Sh horner(const Keys& K, u64 u, u32 s, const u64* c, int d, Sh v)
{
    Sh h = sh_addp(sh_mulf(v, c[d]), c[d - 1]);
    for (int k = d - 2; k >= 0; --k) {
        h = sh_addp(mt(K, u, s, h, v), c[k]);
        ++s;
    }
    return h;
}

// ---- segment forms of S13 (R21, R30) ---------------------------
template <bool WIDE>
__device__ __forceinline__ Sh act_group(const Keys& K, u64 u, u64 q, u32 s, const ActK& p, Sh x, int lane)
{
    if (p.form == 2 || p.deg == 0) {
        const Sh nl = sh_not(ltz<WIDE>(K, q, s, p.w, x, lane));
        if (p.act == 2) return {nl.s0 << FRAC, nl.s1 << FRAC};
        return bm(K, u, s + 1, x, nl);
    }
    Sh sgn = {0, 0};
    if (p.form == 1) { sgn = ltz<WIDE>(K, q, s, p.w, x, lane); ++s; }
    const Sh l1 = ltz<WIDE>(K, q, s, p.w, sh_addp(x, p.e_B), lane);
    const Sh l2 = ltz<WIDE>(K, q, s + 1, p.w, sh_addp(x, p.e_mB), lane);
    s += 2;
    Sh h;
    if (p.form == 0) {
        h = horner(K, u, s, p.c, p.deg, x);
        s += p.deg - 1;
    } else if (p.form == 1) {
        const Sh ax = bm(K, u, s, x, {1ull - 2ull * sgn.s0, 0ull - 2ull * sgn.s1});
        ++s;
        h = sh_add(sh_mulf(x, p.e_half), horner(K, u, s, p.c, p.deg, ax));
        s += p.deg - 1;
    } else {
        const Sh z = sh_mulf(x, p.e_isqrt2);
        const Sh z2 = mt(K, u, s, z, z);
        ++s;
        const Sh S = horner(K, u, s, p.c, p.deg, z2);
        s += p.deg - 1;
        const Sh erf = sh_mulf(mt(K, u, s, z, S), p.e_2sqrtpi);
        h = sh_mulf(mt(K, u, s + 1, x, sh_addp(erf, p.e_one)), p.e_half);
        s += 2;
    }
    Sh out = bm(K, u, s, h, sh_sub(l2, l1));
    const Sh nl2 = sh_not(l2);
    if (p.act == 2) out = sh_add(out, {nl2.s0 << FRAC, nl2.s1 << FRAC});
    else out = sh_add(out, bm(K, u, s + 1, x, nl2));
    return out;
}

}  // namespace mpc
