// ltz_cone.cuh -- LTZ with the carry-cone circuit, G groups per warp.
//
// Only G_{m-1} (the carry into bit w-1) is needed for the sign, so instead of the full
// Kogge-Stone prefix the carry is computed by a binary tree over the 2^L leaves (L =
// ceil(log2 m)); leaves j >= m are the public pads (G, P) = (0, 1).  A node over leaves
// [i*2^(k+1), (i+1)*2^(k+1)) at level k combines lo = node 2i and hi = node 2i+1 of level k-1:
//   G = G_hi ^ AND(P_hi, G_lo),   P = AND(P_hi, P_lo).
// Gates: m (g-layer) + 2(2^L - 1) -- 94 at w = 33 against Kogge-Stone's 290; same rounds.
// PRG: g-layer as Kogge-Stone; node (k, i): G-gate K0 slot SLOT(k+1,i,0),
// P-gate K0 slot SLOT(k+1,i,1), K1 slot SLOT(k+1,i,0) (words 0-1 G, 2-3 P).
// The output shares depend only on the sign bit and the daBit, so they are
// bit-identical to the Kogge-Stone LTZ -- the parity tests compare against the same oracle.
//
// A warp evaluates G consecutive 32-element groups q0..q0+G-1 at once (lane l holds element l
// of each); the tree's nodes of all G groups are spread over the 32 lanes through a per-warp
// shared-memory array, so the 16, 8, 4, 2, 1 nodes per level do not leave lanes idle.
#pragma once
#include "proto.cuh"

namespace mpc {

// per-warp shared memory ConeSmem<G> (proto.cuh): [G][32 positions][4 words] -- BOTH: (G0, G1,
// P0, P1), PAIR: (G, P) of this party -- of the node stored at its leftmost leaf's position.

__host__ __device__ inline int cone_gate_count(int w)
{
    const int m = w - 1;
    if (m <= 0) return 0;
    const int L = ceil_log2i(m);
    return m + 2 * ((1 << L) - 1);
}
// Philox blocks per 32-element group (both parties + dealer): g-layer 2m, nodes 3 each, daBit 33
__host__ __device__ inline u64 cone_philox_per_group(int w)
{
    const int m = w - 1;
    if (m <= 0) return 33;
    const int L = ceil_log2i(m);
    return 2ull * (u64)m + 3ull * (u64)((1 << L) - 1) + 33ull;
}

// ---------------------------------------------------------------- BOTH ----
template <int G>
__device__ void ltz_cone_both(const Keys& K, u64 q0, u32 s, int w, const Sh (&x)[G], Sh (&z)[G],
                                              int lane, ConeSmem<G>& sm)
{
    const int m = w - 1;                      // 0..32
    const int L = (m > 0) ? ceil_log2i(m) : 0;
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const u32 P0 = transpose32((u32)x[g].s0, lane), P1 = transpose32((u32)x[g].s1, lane);
        const uint4 t0 = prg(K.k0, q0 + g, s, ltz_slot(0, lane, 0));
        const uint4 t1 = prg(K.k1, q0 + g, s, ltz_slot(0, lane, 0));
        u32 g0, g1;
        and_both(P0, 0u, 0u, P1, t0.x, t0.y, t0.z, t1.x, t1.y, g0, g1);
        const bool leaf = lane < m;
        sm.w[g][lane][0] = leaf ? g0 : 0u;
        sm.w[g][lane][1] = leaf ? g1 : 0u;
        sm.w[g][lane][2] = leaf ? P0 : 0xffffffffu;    // pad P = public 1: party 0 holds 1
        sm.w[g][lane][3] = leaf ? P1 : 0u;
    }
    __syncwarp();
    for (int k = 0; k < L; ++k) {
        const int nn = 1 << (L - 1 - k);              // nodes per group at this level
        for (int base = 0; base < G * nn; base += 32) {
            const int t = base + lane;
            const bool valid = t < G * nn;
            const int g = valid ? t >> (L - 1 - k) : 0, i = valid ? t & (nn - 1) : 0;
            const int lo = i << (k + 1), hi = lo + (1 << k);
            u32 gl0 = 0, gl1 = 0, pl0 = 0, pl1 = 0, gh0 = 0, gh1 = 0, ph0 = 0, ph1 = 0;
            if (valid) {
                gl0 = sm.w[g][lo][0]; gl1 = sm.w[g][lo][1]; pl0 = sm.w[g][lo][2]; pl1 = sm.w[g][lo][3];
                gh0 = sm.w[g][hi][0]; gh1 = sm.w[g][hi][1]; ph0 = sm.w[g][hi][2]; ph1 = sm.w[g][hi][3];
            }
            const u64 q = q0 + (u64)g;
            const uint4 tg = prg(K.k0, q, s, ltz_slot(k + 1, i, 0));
            const uint4 tp = prg(K.k0, q, s, ltz_slot(k + 1, i, 1));
            const uint4 t1 = prg(K.k1, q, s, ltz_slot(k + 1, i, 0));
            u32 ng0, ng1, np0, np1;
            and_both(ph0, ph1, gl0, gl1, tg.x, tg.y, tg.z, t1.x, t1.y, ng0, ng1);
            and_both(ph0, ph1, pl0, pl1, tp.x, tp.y, tp.z, t1.z, t1.w, np0, np1);
            if (valid) {
                sm.w[g][lo][0] = gh0 ^ ng0; sm.w[g][lo][1] = gh1 ^ ng1;
                sm.w[g][lo][2] = np0; sm.w[g][lo][3] = np1;
            }
        }
        __syncwarp();
    }
    // K1 daBit words: lane g computes group g's, broadcast
    u32 k1w = 0;
    if (lane < G) k1w = prg(K.k1, q0 + lane, s, 1u).x;
#pragma unroll
    for (int g = 0; g < G; ++g) {
        u32 b0, b1;
        if (m == 0) { b0 = (u32)(x[g].s0 & 1ull); b1 = (u32)(x[g].s1 & 1ull); }
        else {
            b0 = (u32)((x[g].s0 >> (w - 1)) & 1ull) ^ ((sm.w[g][0][0] >> lane) & 1u);
            b1 = (u32)((x[g].s1 >> (w - 1)) & 1ull) ^ ((sm.w[g][0][1] >> lane) & 1u);
        }
        const uint4 D0 = prg(K.k0, q0 + g, s, 2u + (u32)lane);
        const u32 d1x = __shfl_sync(FULL, k1w, g);
        const u64 r0A = w64(D0.x, D0.y);
        const u32 r0B = D0.z & 1u;
        const u32 r1B = (d1x >> lane) & 1u;
        const u64 r1A = (u64)(r0B ^ r1B) - r0A;
        const u64 c = (u64)((b0 ^ r0B) ^ (b1 ^ r1B));
        const u64 sg = 1ull - 2ull * c;
        z[g] = Sh{c + sg * r0A, sg * r1A};
    }
    __syncwarp();
}

// ---------------------------------------------------------------- PAIR ----
// Same circuit, one party's shares; every g-layer / tree pass / B2A is one warp exchange that
// carries all G groups' words (so 1 + (passes) + 1 exchanges per G groups).
template <int G>
__device__ void ltz_cone_pair(PairP& pr, u64 q0, u32 s, int w, const u64 (&x)[G], u64 (&z)[G], int lane,
                              ConeSmem<G>& sm)
{
    static_assert(G <= XW, "one exchange carries at most XW words per lane");
    const int m = w - 1;
    const int L = (m > 0) ? ceil_log2i(m) : 0;
    const int pty = pr.pty;
    const Keys& K = *pr.Kp;
    {   // g-layer for all G groups in one exchange
        u32 ta[G], tb[G], tc[G], dd[G], ee[G], Pp[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            Pp[g] = transpose32((u32)x[g], lane);
            const uint4 t0 = prg(K.k0, q0 + g, s, ltz_slot(0, lane, 0));
            uint4 t1 = make_uint4(0, 0, 0, 0);
            if (pty == 1) t1 = prg(K.k1, q0 + g, s, ltz_slot(0, lane, 0));
            pr.and_triple(t0, t1, 0, ta[g], tb[g], tc[g]);
            dd[g] = (pty == 0 ? Pp[g] : 0u) ^ ta[g];
            ee[g] = (pty == 0 ? 0u : Pp[g]) ^ tb[g];
            pr.put(lane, g, (u64)dd[g] | ((u64)ee[g] << 32));
        }
        pr.exch(lane);
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const u64 pw = pr.get(lane, g);
            const u32 gg = pr.and_finish(ta[g], tb[g], tc[g], dd[g] ^ (u32)pw, ee[g] ^ (u32)(pw >> 32));
            const bool leaf = lane < m;
            sm.w[g][lane][0] = leaf ? gg : 0u;
            sm.w[g][lane][2] = leaf ? Pp[g] : (pty == 0 ? 0xffffffffu : 0u);   // pad P = public 1
        }
    }
    __syncwarp();
    for (int k = 0; k < L; ++k) {
        const int nn = 1 << (L - 1 - k);
        for (int base = 0; base < G * nn; base += 32) {
            const int t = base + lane;
            const bool valid = t < G * nn;
            const int g = valid ? t >> (L - 1 - k) : 0, i = valid ? t & (nn - 1) : 0;
            const int lo = i << (k + 1), hi = lo + (1 << k);
            u32 gl = 0, pl = 0, gh = 0, ph = 0;         // idle lanes read nothing (no benign races)
            if (valid) { gl = sm.w[g][lo][0]; pl = sm.w[g][lo][2]; gh = sm.w[g][hi][0]; ph = sm.w[g][hi][2]; }
            const u64 q = q0 + (u64)g;
            const uint4 tg = prg(K.k0, q, s, ltz_slot(k + 1, i, 0));
            const uint4 tp = prg(K.k0, q, s, ltz_slot(k + 1, i, 1));
            uint4 t1 = make_uint4(0, 0, 0, 0);
            if (pty == 1) t1 = prg(K.k1, q, s, ltz_slot(k + 1, i, 0));
            u32 ga, gb, gc, pa, pb, pc;
            pr.and_triple(tg, t1, 0, ga, gb, gc);
            pr.and_triple(tp, t1, 1, pa, pb, pc);
            const u32 dG = ph ^ ga, eG = gl ^ gb, dP = ph ^ pa, eP = pl ^ pb;
            pr.put(lane, 0, (u64)dG | ((u64)eG << 32));
            pr.put(lane, 1, (u64)dP | ((u64)eP << 32));
            pr.exch(lane);
            const u64 w0 = pr.get(lane, 0), w1 = pr.get(lane, 1);
            const u32 ng = pr.and_finish(ga, gb, gc, dG ^ (u32)w0, eG ^ (u32)(w0 >> 32));
            const u32 np = pr.and_finish(pa, pb, pc, dP ^ (u32)w1, eP ^ (u32)(w1 >> 32));
            if (valid) { sm.w[g][lo][0] = gh ^ ng; sm.w[g][lo][2] = np; }
        }
        __syncwarp();
    }
    u32 k1w = 0;
    if (pty == 1 && lane < G) k1w = prg(K.k1, q0 + lane, s, 1u).x;
    u64 rA[G];
    u32 mine[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        u32 bp;
        if (m == 0) bp = (u32)(x[g] & 1ull);
        else bp = (u32)((x[g] >> (w - 1)) & 1ull) ^ ((sm.w[g][0][0] >> lane) & 1u);
        const uint4 D0 = prg(K.k0, q0 + g, s, 2u + (u32)lane);
        const u64 r0A = w64(D0.x, D0.y);
        const u32 r0B = D0.z & 1u;
        const u32 d1x = __shfl_sync(FULL, k1w, g);
        u32 rB;
        if (pty == 0) { rA[g] = r0A; rB = r0B; }
        else { rB = (d1x >> lane) & 1u; rA[g] = (u64)(r0B ^ rB) - r0A; }
        mine[g] = bp ^ rB;
        pr.put(lane, g, (u64)mine[g]);
    }
    pr.exch(lane);
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const u64 c = (u64)(mine[g] ^ ((u32)pr.get(lane, g) & 1u));
        const u64 sg = 1ull - 2ull * c;
        z[g] = pty == 0 ? c + sg * rA[g] : sg * rA[g];
    }
    __syncwarp();
}

}  // namespace mpc
