// proto_both.cuh -- L1 protocol steps, MPC_MODE_BOTH: one thread holds both parties'
// shares of an element; an "opening" is the sum of the two masked shares, formed in
// registers (the value each party would send and receive in a PAIR execution).
// Contract: DESIGN.md 2.3 (PRG layout) and 2.4 (protocol steps).
#pragma once
#include "dev_common.cuh"

namespace mpc {

struct Sh { u64 s0, s1; };   // [x]_0, [x]_1

__device__ __forceinline__ Sh sh_add(Sh a, Sh b) { return {a.s0 + b.s0, a.s1 + b.s1}; }
__device__ __forceinline__ Sh sh_sub(Sh a, Sh b) { return {a.s0 - b.s0, a.s1 - b.s1}; }
__device__ __forceinline__ Sh sh_neg(Sh a) { return {0ull - a.s0, 0ull - a.s1}; }
__device__ __forceinline__ Sh sh_addp(Sh a, u64 e) { return {a.s0 + e, a.s1}; }        // addP: party 0
__device__ __forceinline__ Sh sh_shr(Sh a, int k) { return {shr(a.s0, k), shr(a.s1, k)}; }
__device__ __forceinline__ Sh sh_muli(Sh a, u64 k) { return {a.s0 * k, a.s1 * k}; }    // pmulI
__device__ __forceinline__ Sh sh_mulf(Sh a, u64 e) { return {shr(a.s0 * e, FRAC), shr(a.s1 * e, FRAC)}; } // pmulF
__device__ __forceinline__ Sh sh_not(Sh b) { return {1ull - b.s0, 0ull - b.s1}; }      // 1 - bit

// Beaver step on element-unit u at step s.
// (a0,b0) = PRG(K0,u,s,0); (a1,b1) = PRG(K1,u,s,0); c0 = half (u&1) of PRG(K0,u>>1,s,1).
// Party 1's share is z1 = c1 + e b1 + f a1 with c1 = (a0+a1)(b0+b1) - c0; since Beaver is exact,
// z0 + z1 = (x0+x1)(y0+y1) = X Y, so one thread holding both parties forms the SAME z1 as
// X Y - z0: 3 ring multiplies instead of 5 (identical bits; the PAIR policy computes z1 the
// protocol's way, tests compare both against the oracle).
__device__ __forceinline__ Sh bm_with_c0(const Keys& K, u64 u, u32 s, Sh x, Sh y, u64 c0)
{
    const uint4 A0 = prg(K.k0, u, s, 0);
    const uint4 A1 = prg(K.k1, u, s, 0);
    const u64 a0 = w64(A0.x, A0.y), b0 = w64(A0.z, A0.w);
    const u64 a1 = w64(A1.x, A1.y), b1 = w64(A1.z, A1.w);
    const u64 X = x.s0 + x.s1, Y = y.s0 + y.s1;
    const u64 e = X - (a0 + a1);                       // open(x - a)
    const u64 f = Y - (b0 + b1);                       // open(y - b)
    const u64 z0 = c0 + e * (b0 + f) + f * a0;         // party 0: e b0 + e f = e (b0 + f)
    return {z0, X * Y - z0};
}

__device__ __forceinline__ u64 beaver_c0(const Keys& K, u64 u, u32 s)
{
    const uint4 C = prg(K.k0, u >> 1, s, 1);
    return (u & 1) ? w64(C.z, C.w) : w64(C.x, C.y);
}

__device__ __forceinline__ Sh bm(const Keys& K, u64 u, u32 s, Sh x, Sh y)
{
    return bm_with_c0(K, u, s, x, y, beaver_c0(K, u, s));
}
__device__ __forceinline__ Sh mt(const Keys& K, u64 u, u32 s, Sh x, Sh y)
{
    return sh_shr(bm(K, u, s, x, y), FRAC);
}

// Two consecutive units (u even, u+1) share one c0 block: 5 Philox blocks per pair.
__device__ __forceinline__ void bm2(const Keys& K, u64 u, u32 s, Sh x0, Sh y0, Sh x1, Sh y1,
                                   Sh& z0, Sh& z1)
{
    const uint4 C = prg(K.k0, u >> 1, s, 1);
    z0 = bm_with_c0(K, u, s, x0, y0, w64(C.x, C.y));
    z1 = bm_with_c0(K, u + 1, s, x1, y1, w64(C.z, C.w));
}

// Square with a square-pair triple:
// (a0, c0) = PRG(K0,u,s,2); a1 = half (u&1) of PRG(K1,u>>1,s,3); c1 = (a0+a1)^2 - c0;
// e = open(y - a); z0 = c0 + 2 e a0 + e^2; z1 = c1 + 2 e a1.  One opening, 8 B/party.
__device__ __forceinline__ Sh sq_with_a1(const Keys& K, u64 u, u32 s, Sh y, u64 a1)
{
    const uint4 A0 = prg(K.k0, u, s, 2);
    const u64 a0 = w64(A0.x, A0.y), c0 = w64(A0.z, A0.w);
    const u64 Y = y.s0 + y.s1;
    const u64 e = Y - (a0 + a1);                       // open(y - a)
    const u64 z0 = c0 + e * (2ull * a0 + e);
    return {z0, Y * Y - z0};                           // = c1 + 2 e a1 with c1 = a^2 - c0 (exact square)
}
__device__ __forceinline__ Sh sq1(const Keys& K, u64 u, u32 s, Sh y)
{
    const uint4 A1 = prg(K.k1, u >> 1, s, 3);
    return sq_with_a1(K, u, s, y, (u & 1) ? w64(A1.z, A1.w) : w64(A1.x, A1.y));
}
__device__ __forceinline__ void sq2(const Keys& K, u64 u, u32 s, Sh y0, Sh y1, Sh& z0, Sh& z1)
{
    const uint4 A1 = prg(K.k1, u >> 1, s, 3);
    z0 = sq_with_a1(K, u, s, y0, w64(A1.x, A1.y));
    z1 = sq_with_a1(K, u + 1, s, y1, w64(A1.z, A1.w));
}

// Broadcast triple: z = x * y_row with ONE mask per row.
// Row part: b0 = PRG(K0,r,s,6)[0..1], b1 = PRG(K1,r,s,6)[0..1], f = open(y - b).
// Element part: (a0,c0) = PRG(K0,u,s,4); a1 = half (u&1) of PRG(K1,u>>1,s,5);
// c1 = (a0+a1)(b0+b1) - c0 (dealer -> party 1); e = open(x - a);
// z0 = c0 + e b0 + f a0 + e f; z1 = c1 + e b1 + f a1.
struct BRow { u64 b0, b1, f; };   // PAIR: party 0 holds b0; party 1 b1 and (as dealer) b0
__device__ __forceinline__ BRow bmb_row(const Keys& K, u64 r, u32 s, Sh y)
{
    const uint4 B0 = prg(K.k0, r, s, 6), B1 = prg(K.k1, r, s, 6);
    const u64 b0 = w64(B0.x, B0.y), b1 = w64(B1.x, B1.y);
    return {b0, b1, (y.s0 - b0) + (y.s1 - b1)};
}
__device__ __forceinline__ Sh bmb_elem(const Keys& K, u64 u, u32 s, Sh x, const BRow& r, u64 a1)
{
    const uint4 A0 = prg(K.k0, u, s, 4);
    const u64 a0 = w64(A0.x, A0.y), c0 = w64(A0.z, A0.w);
    const u64 X = x.s0 + x.s1;
    const u64 e = X - (a0 + a1);                       // open(x - a)
    const u64 z0 = c0 + e * (r.b0 + r.f) + r.f * a0;
    return {z0, X * (r.b0 + r.b1 + r.f) - z0};         // = c1 + e b1 + f a1 (exact: rec = x y_row)
}
// unit pair (u even, u+1): one K1 block serves both a1 halves (1.5 blocks per element)
__device__ __forceinline__ void bmb2(const Keys& K, u64 u, u32 s, Sh x0, Sh x1, const BRow& r0, const BRow& r1,
                                     Sh& z0, Sh& z1)
{
    const uint4 A1 = prg(K.k1, u >> 1, s, 5);
    z0 = bmb_elem(K, u, s, x0, r0, w64(A1.x, A1.y));
    z1 = bmb_elem(K, u + 1, s, x1, r1, w64(A1.z, A1.w));
}

// AND on XOR-shared 32-bit plane words with triple (a0,b0,c0 | a1,b1).
// (party 1's z1 = c1 ^ d&b1 ^ e&a1 with c1 = (a0^a1)&(b0^b1) ^ c0 equals (X & Y) ^ z0, X = x0^x1,
// Y = y0^y1: the AND is exact on XOR shares -- fewer LOP3s for the thread holding both parties)
__device__ __forceinline__ void and_both(u32 x0, u32 x1, u32 y0, u32 y1,
                                         u32 a0, u32 b0, u32 c0, u32 a1, u32 b1,
                                         u32& z0, u32& z1)
{
    const u32 X = x0 ^ x1, Y = y0 ^ y1;
    const u32 d = X ^ a0 ^ a1;                          // open(x ^ a)
    const u32 e = Y ^ b0 ^ b1;                          // open(y ^ b)
    z0 = c0 ^ (d & b0) ^ (e & a0) ^ (d & e);
    z1 = (X & Y) ^ z0;
}

// LTZ_w for w <= 33 (one bit plane per lane), branch-free: every lane issues the three
// Philox blocks of each Kogge-Stone level and keeps the result only if its plane is
// active.  At the last level (d = 16, when w > 17) lanes 0..15 have no gate, so their
// blocks compute the daBit words instead: D0 of element l and l+16 and the K1 word --
// exactly the contract's blocks, issued in slots that would idle.
__device__ __forceinline__ Sh ltz_narrow(const Keys& K, u64 q, u32 s, int w, Sh x, int lane)
{
    const int m = w - 1;
    const PrgQ Q0 = prg_q(K.k0, q, s), Q1 = prg_q(K.k1, q, s);
    u32 P0 = transpose32((u32)x.s0, lane), P1 = transpose32((u32)x.s1, lane), G0 = 0, G1 = 0;
    {   // g-layer: g_j = AND((x0_j, 0), (0, x1_j))
        const uint4 t0 = prg(Q0, ltz_slot(0, lane, 0));
        const uint4 t1 = prg(Q1, ltz_slot(0, lane, 0));
        u32 g0, g1;
        and_both(P0, 0u, 0u, P1, t0.x, t0.y, t0.z, t1.x, t1.y, g0, g1);
        if (lane < m) { G0 = g0; G1 = g1; }
    }
    const int L = (m > 0) ? ceil_log2i(m) : 0;
    const bool trick = m > 16;                      // last level has d = 16
    uint4 Dlo = make_uint4(0, 0, 0, 0), Dhi = make_uint4(0, 0, 0, 0);
    u32 k1w = 0;
    for (int k = 0; k < L; ++k) {
        const int d = 1 << k;
        const int src = (lane - d) & 31;
        const u32 g0 = __shfl_sync(FULL, G0, src), g1 = __shfl_sync(FULL, G1, src);
        const u32 p0 = __shfl_sync(FULL, P0, src), p1 = __shfl_sync(FULL, P1, src);
        const bool act = lane >= d && lane < m;
        const bool dab = trick && k == L - 1 && lane < 16;
        const uint4 tg = prg(Q0, dab ? 2u + (u32)lane : ltz_slot(k + 1, lane, 0));
        const uint4 tp = prg(Q0, dab ? 18u + (u32)lane : ltz_slot(k + 1, lane, 1));
        const uint4 t1 = prg(Q1, dab ? 1u : ltz_slot(k + 1, lane, 0));
        u32 ng0, ng1, np0, np1;
        and_both(P0, P1, g0, g1, tg.x, tg.y, tg.z, t1.x, t1.y, ng0, ng1);
        and_both(P0, P1, p0, p1, tp.x, tp.y, tp.z, t1.z, t1.w, np0, np1);
        if (act) { G0 ^= ng0; G1 ^= ng1; P0 = np0; P1 = np1; }
        if (dab) { Dlo = tg; Dhi = tp; k1w = t1.x; }
    }
    u32 b0, b1;
    if (m == 0) {
        b0 = (u32)(x.s0 & 1ull); b1 = (u32)(x.s1 & 1ull);
    } else {
        const u32 gm0 = __shfl_sync(FULL, G0, m - 1), gm1 = __shfl_sync(FULL, G1, m - 1);
        b0 = (u32)((x.s0 >> (w - 1)) & 1ull) ^ ((gm0 >> lane) & 1u);
        b1 = (u32)((x.s1 >> (w - 1)) & 1ull) ^ ((gm1 >> lane) & 1u);
    }
    uint4 D0;
    u32 d1x;
    if (trick) {
        const u32 hx = __shfl_sync(FULL, Dhi.x, lane & 15), hy = __shfl_sync(FULL, Dhi.y, lane & 15);
        const u32 hz = __shfl_sync(FULL, Dhi.z, lane & 15);
        D0 = lane < 16 ? Dlo : make_uint4(hx, hy, hz, 0u);
        d1x = __shfl_sync(FULL, k1w, 0);
    } else {
        D0 = prg(Q0, 2u + (u32)lane);
        d1x = prg(Q1, 1u).x;
    }
    const u64 r0A = w64(D0.x, D0.y);
    const u32 r0B = D0.z & 1u;
    const u32 r1B = (d1x >> lane) & 1u;
    const u64 r1A = (u64)(r0B ^ r1B) - r0A;
    const u64 c = (u64)((b0 ^ r0B) ^ (b1 ^ r1B));
    const u64 sg = 1ull - 2ull * c;
    return {c + sg * r0A, sg * r1A};
}

// LTZ at w = 33 (m = 32 planes, L = 5 Kogge-Stone levels) with the levels' Philox rebalanced over
// idle lanes.  At level k the lanes j < 2^k have no gate; instead of issuing blocks nobody uses they
// generate the blocks of the LAST level's gate nodes (planes 16..31; item t = 2^k - 1 + lane, t < 15)
// into a per-warp shared-memory stash, and lanes 1..3 generate item 15 (plane 31) in the daBit pass in
// place of the redundant copies of the K1 daBit word.  The last level then issues no Philox at all:
// 16 warp-blocks per LTZ instead of 19 (the algorithmic count is 15.1).  Same blocks, same gate
// words, same output bits as ltz<false> (DESIGN.md 2.3 / 2.4); needs <= 8 warps per CTA.
__device__ __forceinline__ Sh ltz33_rebal(const Keys& K, u64 q, u32 s, Sh x, int lane)
{
    __shared__ __align__(16) u32 stash_all[8][16][12];          // [warp][item][tg.xyz tp.xyz t1.xyzw]
    u32 (*stash)[12] = stash_all[(threadIdx.x >> 5) & 7];
    const PrgQ Q0 = prg_q(K.k0, q, s), Q1 = prg_q(K.k1, q, s);
    // daBit pass: D0 on every lane; the K1 word D1 on lane 0 (broadcast); item 15 on lanes 1..3
    const uint4 D0 = prg(Q0, 2u + (u32)lane);
    const u32 sd = lane == 1 ? ltz_slot(5, 31, 0) : lane == 2 ? ltz_slot(5, 31, 1) : lane == 3 ? ltz_slot(5, 31, 0) : 1u;
    const uint4 DX = prg((lane == 1 || lane == 2) ? K.k0 : K.k1, q, s, sd);       // (a key select: 2 registers)
    const u32 d1x = __shfl_sync(FULL, DX.x, 0);
    if (lane == 1) { stash[15][0] = DX.x; stash[15][1] = DX.y; stash[15][2] = DX.z; }
    if (lane == 2) { stash[15][3] = DX.x; stash[15][4] = DX.y; stash[15][5] = DX.z; }
    if (lane == 3) { stash[15][6] = DX.x; stash[15][7] = DX.y; stash[15][8] = DX.z; stash[15][9] = DX.w; }
    // A2B and the g-layer (every plane is a leaf at m = 32)
    u32 P0 = transpose32((u32)x.s0, lane), P1 = transpose32((u32)x.s1, lane), G0, G1;
    {
        const uint4 t0 = prg(Q0, ltz_slot(0, lane, 0)), t1 = prg(Q1, ltz_slot(0, lane, 0));
        and_both(P0, 0u, 0u, P1, t0.x, t0.y, t0.z, t1.x, t1.y, G0, G1);
    }
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int d = 1 << k;
        const int src = (lane - d) & 31;
        const u32 g0 = __shfl_sync(FULL, G0, src), g1 = __shfl_sync(FULL, G1, src);
        const u32 p0 = __shfl_sync(FULL, P0, src), p1 = __shfl_sync(FULL, P1, src);
        const bool act = lane >= d;
        uint4 tg, tp, t1;
        if (k < 4) {
            const int t = d - 1 + lane;                            // the last level's item of an idle lane
            const int jj = act ? lane : 16 + t, kk = act ? k : 4;
            tg = prg(Q0, ltz_slot(kk + 1, jj, 0));
            tp = prg(Q0, ltz_slot(kk + 1, jj, 1));
            t1 = prg(Q1, ltz_slot(kk + 1, jj, 0));
            if (!act) {
                u32* w = stash[t];
                w[0] = tg.x; w[1] = tg.y; w[2] = tg.z; w[3] = tp.x; w[4] = tp.y; w[5] = tp.z;
                w[6] = t1.x; w[7] = t1.y; w[8] = t1.z; w[9] = t1.w;
            }
            if (k == 3) __syncwarp();
        } else {                                                     // every item is in the stash
            const u32* w = stash[lane & 15];
            tg = make_uint4(w[0], w[1], w[2], 0u); tp = make_uint4(w[3], w[4], w[5], 0u);
            t1 = make_uint4(w[6], w[7], w[8], w[9]);
        }
        u32 ng0, ng1, np0, np1;
        and_both(P0, P1, g0, g1, tg.x, tg.y, tg.z, t1.x, t1.y, ng0, ng1);
        and_both(P0, P1, p0, p1, tp.x, tp.y, tp.z, t1.z, t1.w, np0, np1);
        if (act) { G0 ^= ng0; G1 ^= ng1; P0 = np0; P1 = np1; }
    }
    __syncwarp();                                                    // the stash is free for the next call
    // sign b = p_32 ^ G_31, then the daBit B2A (as ltz<false>)
    const u32 gm0 = __shfl_sync(FULL, G0, 31), gm1 = __shfl_sync(FULL, G1, 31);
    const u32 b0 = (u32)((x.s0 >> 32) & 1ull) ^ ((gm0 >> lane) & 1u);
    const u32 b1 = (u32)((x.s1 >> 32) & 1ull) ^ ((gm1 >> lane) & 1u);
    const u64 r0A = w64(D0.x, D0.y);
    const u32 r0B = D0.z & 1u;
    const u32 r1B = (d1x >> lane) & 1u;
    const u64 r1A = (u64)(r0B ^ r1B) - r0A;
    const u64 c = (u64)((b0 ^ r0B) ^ (b1 ^ r1B));
    const u64 sg = 1ull - 2ull * c;
    return {c + sg * r0A, sg * r1A};
}

// LTZ_w on the warp's 32-element group q (lane l <-> element 32q+l); DESIGN.md 2.4.
// All 32 lanes must call it (tail lanes with any value).  Returns the scale-1
// arithmetic sharing of bit (w-1) of rec(x).  WIDE: w > 33 (two planes per lane).
template <bool WIDE, bool RB = false>
__device__ __forceinline__ Sh ltz(const Keys& K, u64 q, u32 s, int w, Sh x, int lane)
{
#ifndef MPC_LTZ_NARROW
#define MPC_LTZ_NARROW 0   // measured: the branchy form is 3-7% faster (register pressure)
#endif
    if constexpr (!WIDE && MPC_LTZ_NARROW) return ltz_narrow(K, q, s, w, x, lane);
#ifndef MPC_LTZ_REBAL
#define MPC_LTZ_REBAL 1
#endif
    if constexpr (!WIDE && RB && MPC_LTZ_REBAL)
        if (w == 33 && blockDim.x <= 256) return ltz33_rebal(K, q, s, x, lane);
    const int m = w - 1;
    const PrgQ Q0 = prg_q(K.k0, q, s), Q1 = prg_q(K.k1, q, s);
#ifndef MPC_LTZ_HOIST
#define MPC_LTZ_HOIST 1       // the daBit blocks first (interleave with the g-layer's); with UNIFORM: max tree -4 %
#endif
#ifndef MPC_LTZ_UNIFORM
#define MPC_LTZ_UNIFORM 1     // every lane issues each level's blocks (no divergence; SIMT issues them anyway)
#endif
    uint4 D0h = make_uint4(0, 0, 0, 0), D1h = D0h;
    if (MPC_LTZ_HOIST) { D0h = prg(Q0, 2u + (u32)lane); D1h = prg(Q1, 1u); }
    // A2B (local): lane j receives plane j of both parties' shares.
    u32 P0[2], P1[2], G0[2], G1[2];
    P0[0] = transpose32((u32)x.s0, lane);
    P1[0] = transpose32((u32)x.s1, lane);
    if (WIDE) {
        P0[1] = transpose32((u32)(x.s0 >> 32), lane);
        P1[1] = transpose32((u32)(x.s1 >> 32), lane);
    }
    constexpr int H = WIDE ? 2 : 1;
    // g-layer: g_j = AND((x0_j, 0), (0, x1_j))
#pragma unroll
    for (int h = 0; h < H; ++h) {
        const int j = lane + 32 * h;
        G0[h] = 0; G1[h] = 0;
        if (j < m) {
            const uint4 t0 = prg(Q0, ltz_slot(0, j, 0));
            const uint4 t1 = prg(Q1, ltz_slot(0, j, 0));
            and_both(P0[h], 0u, 0u, P1[h], t0.x, t0.y, t0.z, t1.x, t1.y, G0[h], G1[h]);
        }
    }
    // Kogge-Stone levels: G_j ^= P_j & G_{j-d};  P_j &= P_{j-d}   (old values)
    const int L = (m > 0) ? ceil_log2i(m) : 0;
    for (int k = 0; k < L; ++k) {
        const int d = 1 << k;
        u32 sG0[2], sG1[2], sP0[2], sP1[2];
        const int src = (lane - d) & 31;
#pragma unroll
        for (int h = 0; h < H; ++h) {
            sG0[h] = __shfl_sync(FULL, G0[h], src);
            sG1[h] = __shfl_sync(FULL, G1[h], src);
            sP0[h] = __shfl_sync(FULL, P0[h], src);
            sP1[h] = __shfl_sync(FULL, P1[h], src);
        }
#pragma unroll
        for (int h = 0; h < H; ++h) {
            const int j = lane + 32 * h;
            const bool act = j >= d && j < m;
            if (MPC_LTZ_UNIFORM || act) {
                // source plane j-d lives in lane src, half h (if lane >= d) or h-1
                int hs = h;
                if (d < 32) hs = (lane >= d) ? h : h - 1;
                else hs = h - 1;                       // d == 32 (WIDE only): same lane, lower half
                u32 g0 = sG0[0], g1 = sG1[0], p0 = sP0[0], p1 = sP1[0];
                if (WIDE && hs == 1) { g0 = sG0[1]; g1 = sG1[1]; p0 = sP0[1]; p1 = sP1[1]; }
                if (WIDE && d == 32) { g0 = G0[0]; g1 = G1[0]; p0 = P0[0]; p1 = P1[0]; }
                const uint4 tg = prg(Q0, ltz_slot(k + 1, j, 0));
                const uint4 tp = prg(Q0, ltz_slot(k + 1, j, 1));
                const uint4 t1 = prg(Q1, ltz_slot(k + 1, j, 0));
                u32 ng0, ng1, np0, np1;
                and_both(P0[h], P1[h], g0, g1, tg.x, tg.y, tg.z, t1.x, t1.y, ng0, ng1);
                and_both(P0[h], P1[h], p0, p1, tp.x, tp.y, tp.z, t1.z, t1.w, np0, np1);
                if (act) {
                    G0[h] ^= ng0; G1[h] ^= ng1;
                    P0[h] = np0; P1[h] = np1;
                }
            }
        }
    }
    // sign: b = p_{w-1} ^ G_{m-1}
    u32 b0, b1;
    if (m == 0) {
        b0 = (u32)(x.s0 & 1ull); b1 = (u32)(x.s1 & 1ull);
    } else {
        const int jm = m - 1;
        u32 gm0 = G0[0], gm1 = G1[0];
        if (WIDE && jm >= 32) { gm0 = G0[1]; gm1 = G1[1]; }
        gm0 = __shfl_sync(FULL, gm0, jm & 31);
        gm1 = __shfl_sync(FULL, gm1, jm & 31);
        b0 = (u32)((x.s0 >> (w - 1)) & 1ull) ^ ((gm0 >> lane) & 1u);
        b1 = (u32)((x.s1 >> (w - 1)) & 1ull) ^ ((gm1 >> lane) & 1u);
    }
    // daBit + B2A: c = open(b ^ r); z0 = c + (1-2c) r0A; z1 = (1-2c) r1A
    const uint4 D0 = MPC_LTZ_HOIST ? D0h : prg(Q0, 2u + (u32)lane);
    const uint4 D1 = MPC_LTZ_HOIST ? D1h : prg(Q1, 1u);
    const u64 r0A = w64(D0.x, D0.y);
    const u32 r0B = D0.z & 1u;
    const u32 r1B = (D1.x >> lane) & 1u;
    const u64 r1A = (u64)(r0B ^ r1B) - r0A;
    const u64 c = (u64)((b0 ^ r0B) ^ (b1 ^ r1B));
    const u64 sg = 1ull - 2ull * c;
    return {c + sg * r0A, sg * r1A};
}

// Philox blocks used per 32-element group by LTZ_w (algorithmic count).
__host__ __device__ inline u64 ltz_philox_per_group(int w)
{
    const int m = w - 1;
    if (m <= 0) return 32 + 1;
    const int L = ceil_log2i(m);
    u64 c = 2ull * (u64)m + 32 + 1;
    for (int k = 0; k < L; ++k) c += 3ull * (u64)(m - (1 << k));
    return c;
}

}  // namespace mpc
