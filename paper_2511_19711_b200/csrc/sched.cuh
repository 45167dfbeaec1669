// sched.cuh -- L2 fused schedules of DESIGN.md 2.5, written once against a protocol policy
// P (BothP or PairP, proto.cuh).  Each function consumes step ids s, s+1, ... exactly in
// the order of the decomposition (so fused = composed).  In PairP every bm/ltz is a
// warp-level exchange: all 32 lanes of a warp must call these functions together.
#pragma once
#include "proto.cuh"

namespace mpc {

// knobs with their public constants already encoded (E(c), host side)
struct ExpK { int t, clamp, w, sq; u64 e_one, e_2t; };   // sq: square-pair triples (NEXT #2)
struct NrK  { int iters; ExpK exp; u64 e_half, e_c003, e_two, e_three, e_02, e_22; };
constexpr int MAX_COEF = 13;
struct ActK {
    int act;          // 0 gelu, 1 silu, 2 sigmoid
    int form;         // 0 poly_x, 1 poly_abs, 2 relu, 3 erf
    int deg;          // polynomial degree (HORNER degree for erf = K-1)
    int w;
    int basis;        // 0 Horner, 1 power basis (NEXT #2)
    u64 e_B, e_mB, e_half, e_one, e_isqrt2, e_2sqrtpi;
    u64 c[MAX_COEF];  // E(c_k) (poly) or E(a_k) (erf series)
};

__device__ __forceinline__ int exp_steps(const ExpK& e) { return e.t + 2 * e.clamp; }

// ---- EXP(x; t, clamp, w) -------------------------------------------------
// GROUP variant: lane <-> unit u of LTZ group q (with or without clamp).
template <bool WIDE, class P>
__device__ __forceinline__ typename P::S exp_group(P& pr, u64 u, u64 q, u32 s, const ExpK& p,
                                                   typename P::S x, int lane)
{
    typename P::S y = pr.addp(pr.shr_(x, p.t), p.e_one);
    if (p.clamp) {
        const typename P::S l = pr.template ltz_o<WIDE>(q, s, p.w, pr.addp(x, p.e_2t), lane);
        y = pr.bm(u, s + 1, y, pr.notb(l));
        s += 2;
    }
    for (int k = 0; k < p.t; ++k) y = pr.shr_(p.sq ? pr.sq(u, s + k, y) : pr.bm(u, s + k, y, y), FRAC);
    return y;
}

// PAIR variant (no clamp): units u (even) and u+1 in one thread; one c0 block per pair.
template <class P>
__device__ __forceinline__ void exp_pair(P& pr, u64 u, u32 s, const ExpK& p, typename P::S& y0, typename P::S& y1)
{
    y0 = pr.addp(pr.shr_(y0, p.t), p.e_one);
    y1 = pr.addp(pr.shr_(y1, p.t), p.e_one);
    for (int k = 0; k < p.t; ++k) {
        typename P::S a, b;
        if (p.sq) pr.sq2(u, s + k, y0, y1, a, b);
        else pr.bm2(u, s + k, y0, y0, y1, y1, a, b);
        y0 = pr.shr_(a, FRAC); y1 = pr.shr_(b, FRAC);
    }
}

// Clamp head of EXP (steps s, s+1; group layout): y = BM(addP(shr(x,t),1), NOT(LTZ_w(addP(x,2^t)))).
// Splitting it from the squarings lets the t squarings run in the pair layout (one c0 block per
// unit pair, 5 independent Philox blocks per thread and step) -- same units, same output bits.
template <bool WIDE, class P>
__device__ __forceinline__ typename P::S exp_clamp_head(P& pr, u64 u, u64 q, u32 s, const ExpK& p,
                                                        typename P::S x, int lane)
{
    const typename P::S y = pr.addp(pr.shr_(x, p.t), p.e_one);
    const typename P::S l = pr.template ltz_o<WIDE>(q, s, p.w, pr.addp(x, p.e_2t), lane);
    return pr.bm(u, s + 1, y, pr.notb(l));
}

// The t squarings of EXP (steps s .. s+t-1) on V unit pairs per lane.
template <int V, class P>
__device__ __forceinline__ void exp_squarings_pairv(P& pr, const u64 (&u)[V], u32 s, const ExpK& p,
                                                    typename P::S (&y0)[V], typename P::S (&y1)[V])
{
    for (int k = 0; k < p.t; ++k) {
        typename P::S a[V], b[V];
        if (p.sq) pr.template sq2v<V>(u, s + k, y0, y1, a, b);
        else pr.template bm2v<V>(u, s + k, y0, y0, y1, y1, a, b);
#pragma unroll
        for (int v = 0; v < V; ++v) { y0[v] = pr.shr_(a[v], FRAC); y1[v] = pr.shr_(b[v], FRAC); }
    }
}

// V pairs per lane (P::kV): the same schedule on V unit pairs, one exchange per step in PAIR.
template <int V, class P>
__device__ __forceinline__ void exp_pairv(P& pr, const u64 (&u)[V], u32 s, const ExpK& p,
                                          typename P::S (&y0)[V], typename P::S (&y1)[V])
{
#pragma unroll
    for (int v = 0; v < V; ++v) { y0[v] = pr.addp(pr.shr_(y0[v], p.t), p.e_one); y1[v] = pr.addp(pr.shr_(y1[v], p.t), p.e_one); }
    exp_squarings_pairv<V>(pr, u, s, p, y0, y1);
}

template <int V, class P>
__device__ __forceinline__ void recip_pairv(P& pr, const u64 (&u)[V], u32 s, const NrK& p, const typename P::S (&x0)[V],
                                            const typename P::S (&x1)[V], typename P::S (&y0)[V], typename P::S (&y1)[V])
{
    using S = typename P::S;
    S g0[V], g1[V];
#pragma unroll
    for (int v = 0; v < V; ++v) { g0[v] = pr.addp(pr.neg(x0[v]), p.e_half); g1[v] = pr.addp(pr.neg(x1[v]), p.e_half); }
    exp_pairv<V>(pr, u, s, p.exp, g0, g1);
    s += exp_steps(p.exp);
#pragma unroll
    for (int v = 0; v < V; ++v) { y0[v] = pr.addp(pr.muli(g0[v], 3ull), p.e_c003); y1[v] = pr.addp(pr.muli(g1[v], 3ull), p.e_c003); }
    for (int it = 0; it < p.iters; ++it) {
        S a[V], b[V], c[V], d[V];
        pr.template bm2v<V>(u, s, x0, y0, x1, y1, a, b);
#pragma unroll
        for (int v = 0; v < V; ++v) {
            a[v] = pr.addp(pr.neg(pr.shr_(a[v], FRAC)), p.e_two);
            b[v] = pr.addp(pr.neg(pr.shr_(b[v], FRAC)), p.e_two);
        }
        pr.template bm2v<V>(u, s + 1, y0, a, y1, b, c, d);
#pragma unroll
        for (int v = 0; v < V; ++v) { y0[v] = pr.shr_(c[v], FRAC); y1[v] = pr.shr_(d[v], FRAC); }
        s += 2;
    }
}

template <int V, class P>
__device__ __forceinline__ void rsqrt_pairv(P& pr, const u64 (&u)[V], u32 s, const NrK& p, const typename P::S (&x0)[V],
                                            const typename P::S (&x1)[V], typename P::S (&y0)[V], typename P::S (&y1)[V])
{
    using S = typename P::S;
    S g0[V], g1[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
        g0[v] = pr.neg(pr.addp(pr.shr_(x0[v], 1), p.e_02));
        g1[v] = pr.neg(pr.addp(pr.shr_(x1[v], 1), p.e_02));
    }
    exp_pairv<V>(pr, u, s, p.exp, g0, g1);
    s += exp_steps(p.exp);
#pragma unroll
    for (int v = 0; v < V; ++v) { y0[v] = pr.addp(pr.mulf(g0[v], p.e_22), p.e_02); y1[v] = pr.addp(pr.mulf(g1[v], p.e_22), p.e_02); }
    for (int it = 0; it < p.iters; ++it) {
        S a[V], b[V], c[V], d[V];
        pr.template bm2v<V>(u, s, y0, y0, y1, y1, a, b);
#pragma unroll
        for (int v = 0; v < V; ++v) { a[v] = pr.shr_(a[v], FRAC); b[v] = pr.shr_(b[v], FRAC); }
        pr.template bm2v<V>(u, s + 1, x0, a, x1, b, c, d);
#pragma unroll
        for (int v = 0; v < V; ++v) {
            c[v] = pr.addp(pr.neg(pr.shr_(c[v], FRAC)), p.e_three);
            d[v] = pr.addp(pr.neg(pr.shr_(d[v], FRAC)), p.e_three);
        }
        pr.template bm2v<V>(u, s + 2, y0, c, y1, d, a, b);
#pragma unroll
        for (int v = 0; v < V; ++v) {
            y0[v] = pr.mulf(pr.shr_(a[v], FRAC), p.e_half);
            y1[v] = pr.mulf(pr.shr_(b[v], FRAC), p.e_half);
        }
        s += 3;
    }
}

// ---- RECIP(x; iters, exp) -------------------------------------------
template <bool WIDE, class P>
__device__ __forceinline__ typename P::S recip_group(P& pr, u64 u, u64 q, u32 s, const NrK& p,
                                                     typename P::S x, int lane)
{
    typename P::S g = exp_group<WIDE>(pr, u, q, s, p.exp, pr.addp(pr.neg(x), p.e_half), lane);
    s += exp_steps(p.exp);
    typename P::S y = pr.addp(pr.muli(g, 3ull), p.e_c003);
    for (int it = 0; it < p.iters; ++it) {
        const typename P::S pp = pr.shr_(pr.bm(u, s, x, y), FRAC);
        y = pr.shr_(pr.bm(u, s + 1, y, pr.addp(pr.neg(pp), p.e_two)), FRAC);
        s += 2;
    }
    return y;
}

template <class P>
__device__ __forceinline__ void recip_pair(P& pr, u64 u, u32 s, const NrK& p, typename P::S x0, typename P::S x1,
                                           typename P::S& y0, typename P::S& y1)
{
    typename P::S g0 = pr.addp(pr.neg(x0), p.e_half), g1 = pr.addp(pr.neg(x1), p.e_half);
    exp_pair(pr, u, s, p.exp, g0, g1);
    s += exp_steps(p.exp);
    y0 = pr.addp(pr.muli(g0, 3ull), p.e_c003);
    y1 = pr.addp(pr.muli(g1, 3ull), p.e_c003);
    for (int it = 0; it < p.iters; ++it) {
        typename P::S a, b;
        pr.bm2(u, s, x0, y0, x1, y1, a, b);
        a = pr.addp(pr.neg(pr.shr_(a, FRAC)), p.e_two);
        b = pr.addp(pr.neg(pr.shr_(b, FRAC)), p.e_two);
        typename P::S c, d;
        pr.bm2(u, s + 1, y0, a, y1, b, c, d);
        y0 = pr.shr_(c, FRAC); y1 = pr.shr_(d, FRAC);
        s += 2;
    }
}

// ---- RSQRT(x; iters, exp) ---------------------------------------------
template <bool WIDE, class P>
__device__ __forceinline__ typename P::S rsqrt_group(P& pr, u64 u, u64 q, u32 s, const NrK& p,
                                                     typename P::S x, int lane)
{
    typename P::S g = exp_group<WIDE>(pr, u, q, s, p.exp, pr.neg(pr.addp(pr.shr_(x, 1), p.e_02)), lane);
    s += exp_steps(p.exp);
    typename P::S y = pr.addp(pr.mulf(g, p.e_22), p.e_02);
    for (int it = 0; it < p.iters; ++it) {
        const typename P::S qq = pr.shr_(pr.bm(u, s, y, y), FRAC);
        const typename P::S pp = pr.shr_(pr.bm(u, s + 1, x, qq), FRAC);
        const typename P::S uu = pr.shr_(pr.bm(u, s + 2, y, pr.addp(pr.neg(pp), p.e_three)), FRAC);
        y = pr.mulf(uu, p.e_half);
        s += 3;
    }
    return y;
}

template <class P>
__device__ __forceinline__ void rsqrt_pair(P& pr, u64 u, u32 s, const NrK& p, typename P::S x0, typename P::S x1,
                                           typename P::S& y0, typename P::S& y1)
{
    typename P::S g0 = pr.neg(pr.addp(pr.shr_(x0, 1), p.e_02)), g1 = pr.neg(pr.addp(pr.shr_(x1, 1), p.e_02));
    exp_pair(pr, u, s, p.exp, g0, g1);
    s += exp_steps(p.exp);
    y0 = pr.addp(pr.mulf(g0, p.e_22), p.e_02);
    y1 = pr.addp(pr.mulf(g1, p.e_22), p.e_02);
    for (int it = 0; it < p.iters; ++it) {
        typename P::S a, b, c, d;
        pr.bm2(u, s, y0, y0, y1, y1, a, b);
        a = pr.shr_(a, FRAC); b = pr.shr_(b, FRAC);
        pr.bm2(u, s + 1, x0, a, x1, b, c, d);
        c = pr.addp(pr.neg(pr.shr_(c, FRAC)), p.e_three);
        d = pr.addp(pr.neg(pr.shr_(d, FRAC)), p.e_three);
        pr.bm2(u, s + 2, y0, c, y1, d, a, b);
        y0 = pr.mulf(pr.shr_(a, FRAC), p.e_half);
        y1 = pr.mulf(pr.shr_(b, FRAC), p.e_half);
        s += 3;
    }
}

// ---- HORNER(v; c_0..c_d), d >= 1 ---------------------------------------------------------------
template <class P>
__device__ __forceinline__ typename P::S horner(P& pr, u64 u, u32 s, const u64* c, int d, typename P::S v)
{
    typename P::S h = pr.addp(pr.mulf(v, c[d]), c[d - 1]);
    for (int k = d - 2; k >= 0; --k) {
        h = pr.addp(pr.shr_(pr.bm(u, s, h, v), FRAC), c[k]);
        ++s;
    }
    return h;
}

// ---- POWER(v; c_0..c_d), 1 <= d <= 4 (NEXT #2): v2 = MT(v,v) at s; v3 = MT(v2,v)
// at s+1 and v4 = MT(v2,v2) at s+2 in ONE exchange; h = addP(sum_k pmulF(v^k, c_k), c_0).
template <class P>
__device__ __forceinline__ typename P::S poly_power(P& pr, u64 u, u32 s, const u64* c, int d, typename P::S v)
{
    using S = typename P::S;
    S h = pr.mulf(v, c[1]);
    if (d >= 2) {
        const S v2 = pr.shr_(pr.bm(u, s, v, v), FRAC);
        h = pr.add(h, pr.mulf(v2, c[2]));
        if (d == 3) {
            h = pr.add(h, pr.mulf(pr.shr_(pr.bm(u, s + 1, v2, v), FRAC), c[3]));
        } else if (d >= 4) {
            S v3, v4;
            pr.bm_dual(u, s + 1, v2, v, s + 2, v2, v2, v3, v4);
            h = pr.add(h, pr.add(pr.mulf(pr.shr_(v3, FRAC), c[3]), pr.mulf(pr.shr_(v4, FRAC), c[4])));
        }
    }
    return pr.addp(h, c[0]);
}
template <class P>
__device__ __forceinline__ void poly_power2(P& pr, u64 u, u32 s, const u64* c, int d, typename P::S v0,
                                            typename P::S v1, typename P::S& h0, typename P::S& h1)
{
    using S = typename P::S;
    h0 = pr.mulf(v0, c[1]);
    h1 = pr.mulf(v1, c[1]);
    if (d >= 2) {
        S a, b;
        pr.bm2(u, s, v0, v0, v1, v1, a, b);
        const S q0 = pr.shr_(a, FRAC), q1 = pr.shr_(b, FRAC);
        h0 = pr.add(h0, pr.mulf(q0, c[2]));
        h1 = pr.add(h1, pr.mulf(q1, c[2]));
        if (d == 3) {
            pr.bm2(u, s + 1, q0, v0, q1, v1, a, b);
            h0 = pr.add(h0, pr.mulf(pr.shr_(a, FRAC), c[3]));
            h1 = pr.add(h1, pr.mulf(pr.shr_(b, FRAC), c[3]));
        } else if (d >= 4) {
            S t0, t1, w0, w1;
            pr.bm2_dual(u, s + 1, q0, v0, q1, v1, s + 2, q0, q0, q1, q1, t0, t1, w0, w1);
            h0 = pr.add(h0, pr.add(pr.mulf(pr.shr_(t0, FRAC), c[3]), pr.mulf(pr.shr_(w0, FRAC), c[4])));
            h1 = pr.add(h1, pr.add(pr.mulf(pr.shr_(t1, FRAC), c[3]), pr.mulf(pr.shr_(w1, FRAC), c[4])));
        }
    }
    h0 = pr.addp(h0, c[0]);
    h1 = pr.addp(h1, c[0]);
}

template <class P>
__device__ __forceinline__ typename P::S act_tail(P& pr, u64 u, u32 s, const ActK& p, typename P::S x,
                                                  typename P::S sgn, typename P::S l1, typename P::S l2);

// ---- segment forms of S13 (R21, R30) ------------------------------------
template <bool WIDE, class P>
__device__ __forceinline__ typename P::S act_group(P& pr, u64 u, u64 q, u32 s, const ActK& p,
                                                   typename P::S x, int lane)
{
    using S = typename P::S;
    if (p.form == 2 || p.deg == 0) {
        const S nl = pr.notb(pr.template ltz_o<WIDE>(q, s, p.w, x, lane));
        if (p.act == 2) return pr.shl(nl, FRAC);
        return pr.bm(u, s + 1, x, nl);
    }
    S sgn = pr.zero();
    if (p.form == 1) { sgn = pr.template ltz_o<WIDE>(q, s, p.w, x, lane); ++s; }
    const S l1 = pr.template ltz_o<WIDE>(q, s, p.w, pr.addp(x, p.e_B), lane);
    const S l2 = pr.template ltz_o<WIDE>(q, s + 1, p.w, pr.addp(x, p.e_mB), lane);
    return act_tail(pr, u, s + 2, p, x, sgn, l1, l2);
}

// the non-comparison part of S13 (after the segment LTZs), steps from s on
template <class P>
__device__ __forceinline__ typename P::S act_tail(P& pr, u64 u, u32 s, const ActK& p, typename P::S x,
                                                  typename P::S sgn, typename P::S l1, typename P::S l2)
{
    using S = typename P::S;
    S h;
    if (p.form == 0) {
        h = p.basis ? poly_power(pr, u, s, p.c, p.deg, x) : horner(pr, u, s, p.c, p.deg, x);
        s += p.deg - 1;
    } else if (p.form == 1) {
        const S ax = pr.bm(u, s, x, pr.pm1(sgn));
        ++s;
        h = pr.add(pr.mulf(x, p.e_half), p.basis ? poly_power(pr, u, s, p.c, p.deg, ax) : horner(pr, u, s, p.c, p.deg, ax));
        s += p.deg - 1;
    } else {
        const S z = pr.mulf(x, p.e_isqrt2);
        const S z2 = pr.shr_(pr.bm(u, s, z, z), FRAC);
        ++s;
        const S Ssum = horner(pr, u, s, p.c, p.deg, z2);
        s += p.deg - 1;
        const S erf = pr.mulf(pr.shr_(pr.bm(u, s, z, Ssum), FRAC), p.e_2sqrtpi);
        h = pr.mulf(pr.shr_(pr.bm(u, s + 1, x, pr.addp(erf, p.e_one)), FRAC), p.e_half);
        s += 2;
    }
    S out = pr.bm(u, s, h, pr.sub(l2, l1));
    const S nl2 = pr.notb(l2);
    if (p.act == 2) out = pr.add(out, pr.shl(nl2, FRAC));
    else out = pr.add(out, pr.bm(u, s + 1, x, nl2));
    return out;
}

// ---- the same tails on a unit PAIR (u even, u+1) per thread: one c0 block per pair and step,
// two independent chains per thread.  Same steps, units and output bits as act_tail.
template <class P>
__device__ __forceinline__ void horner2(P& pr, u64 u, u32 s, const u64* c, int d, typename P::S v0,
                                        typename P::S v1, typename P::S& h0, typename P::S& h1)
{
    h0 = pr.addp(pr.mulf(v0, c[d]), c[d - 1]);
    h1 = pr.addp(pr.mulf(v1, c[d]), c[d - 1]);
    for (int k = d - 2; k >= 0; --k) {
        typename P::S a, b;
        pr.bm2(u, s, h0, v0, h1, v1, a, b);
        h0 = pr.addp(pr.shr_(a, FRAC), c[k]);
        h1 = pr.addp(pr.shr_(b, FRAC), c[k]);
        ++s;
    }
}

template <class P>
__device__ __forceinline__ void act_tail2(P& pr, u64 u, u32 s, const ActK& p, typename P::S x0, typename P::S x1,
                                          typename P::S sg0, typename P::S sg1, typename P::S la0, typename P::S la1,
                                          typename P::S lb0, typename P::S lb1, typename P::S& r0, typename P::S& r1)
{
    using S = typename P::S;
    S h0, h1;
    if (p.form == 0) {
        if (p.basis) poly_power2(pr, u, s, p.c, p.deg, x0, x1, h0, h1);
        else horner2(pr, u, s, p.c, p.deg, x0, x1, h0, h1);
        s += p.deg - 1;
    } else if (p.form == 1) {
        S ax0, ax1, t0, t1;
        pr.bm2(u, s, x0, pr.pm1(sg0), x1, pr.pm1(sg1), ax0, ax1);
        ++s;
        if (p.basis) poly_power2(pr, u, s, p.c, p.deg, ax0, ax1, t0, t1);
        else horner2(pr, u, s, p.c, p.deg, ax0, ax1, t0, t1);
        h0 = pr.add(pr.mulf(x0, p.e_half), t0);
        h1 = pr.add(pr.mulf(x1, p.e_half), t1);
        s += p.deg - 1;
    } else {
        const S z0 = pr.mulf(x0, p.e_isqrt2), z1 = pr.mulf(x1, p.e_isqrt2);
        S a, b, q0, q1;
        pr.bm2(u, s, z0, z0, z1, z1, a, b);
        ++s;
        horner2(pr, u, s, p.c, p.deg, pr.shr_(a, FRAC), pr.shr_(b, FRAC), q0, q1);
        s += p.deg - 1;
        pr.bm2(u, s, z0, q0, z1, q1, a, b);
        const S e0 = pr.mulf(pr.shr_(a, FRAC), p.e_2sqrtpi), e1 = pr.mulf(pr.shr_(b, FRAC), p.e_2sqrtpi);
        pr.bm2(u, s + 1, x0, pr.addp(e0, p.e_one), x1, pr.addp(e1, p.e_one), a, b);
        h0 = pr.mulf(pr.shr_(a, FRAC), p.e_half);
        h1 = pr.mulf(pr.shr_(b, FRAC), p.e_half);
        s += 2;
    }
    pr.bm2(u, s, h0, pr.sub(lb0, la0), h1, pr.sub(lb1, la1), r0, r1);
    const S n0 = pr.notb(lb0), n1 = pr.notb(lb1);
    if (p.act == 2) {
        r0 = pr.add(r0, pr.shl(n0, FRAC));
        r1 = pr.add(r1, pr.shl(n1, FRAC));
    } else {
        S a, b;
        pr.bm2(u, s + 1, x0, n0, x1, n1, a, b);
        r0 = pr.add(r0, a);
        r1 = pr.add(r1, b);
    }
}

}  // namespace mpc
