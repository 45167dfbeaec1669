// ltz_cone.cuh -- LTZ with the pruned carry-cone circuit, G groups per
// warp, every window w in [1, 64].
//
// The sign b = p_{w-1} ^ c_{w-1} needs only the carry into bit w-1, i.e. the generate signal of
// the whole prefix [0, m), m = w - 1.  Instead of Kogge-Stone's full prefix (290 AND gates at
// w = 33, 693 at w = 64) it is computed by a binary tree over the 2^L leaves (L = ceil(log2 m)):
// leaf j < m is (g_j, p_j) = (AND(x0_j, x1_j), x0_j ^ x1_j) and leaves j >= m are the PUBLIC pads
// (G, P) = (0, 1).  Node (k, i) covers leaves [i 2^(k+1), (i+1) 2^(k+1)) with children lo = node
// 2i and hi = node 2i+1 of level k-1:   G = G_hi ^ AND(P_hi, G_lo),   P = AND(P_hi, P_lo).
// Pruning:
//  * a node whose hi child lies entirely in the pads IS its lo child (G_hi = 0, P_hi = 1): no
//    gate, no round-trip -- and since a node is stored at its leftmost leaf's position, nothing
//    is even copied; a node entirely in the pads stays the public (0, 1);
//  * so the gate nodes of level k are i < ng_k = ceil((m - 2^k) / 2^(k+1));
//  * P is used only by the parent's G (a hi child) or the parent's own P, so it is never needed
//    on the left spine (i = 0, the root included) and always needed for i > 0.
// Gates: m + sum_k ng_k + sum_k (ng_k - 1) -- 89 at w = 33 (Kogge-Stone 290), 181 at w = 64
// (693), 53 at w = 21 (HummingBird window, 158).  Same rounds as Kogge-Stone (1 + L + 1).
// PRG: g-layer plane j as Kogge-Stone, SLOT(0, j, 0); gate node (k, i): G-gate
// K0 block SLOT(k+1, i, 0), P-gate K0 block SLOT(k+1, i, 1), K1 block SLOT(k+1, i, 0) (words 0-1
// G, 2-3 P).  The output shares depend only on the sign bit and the daBit, so they
// are bit-identical to the Kogge-Stone LTZ -- the parity tests compare against the same oracle.
//
// A warp evaluates G consecutive 32-element groups q0..q0+G-1 at once (lane l holds element l of
// each); a level's G * ng_k gate nodes are spread over the 32 lanes (up to 4 per lane) through a
// per-warp shared-memory array, so the 16, 8, 4, 2, 1 nodes per level do not leave lanes idle, and
// in PAIR mode every level is ONE exchange round for all G groups.
#pragma once
#include "proto.cuh"

namespace mpc {

// per-warp shared memory ConeSmem<G, NL> (proto.cuh): [G][NL positions][4 words] -- BOTH: (G0, G1,
// P0, P1), PAIR: (G, P) of this party in words 0 and 2 -- of the node stored at its leftmost leaf.
// NL = 32 (w <= 33) or 64 (w <= 65).

__host__ __device__ inline int cone_nodes(int m, int k)      // gate nodes at level k
{
    const int d = 1 << k;
    return m > d ? (m - d + 2 * d - 1) / (2 * d) : 0;
}
__host__ __device__ inline int cone_gate_count(int w)
{
    const int m = w - 1;
    if (m <= 0) return 0;
    const int L = ceil_log2i(m);
    int g = m;
    for (int k = 0; k < L; ++k) { const int n = cone_nodes(m, k); g += n + (n > 0 ? n - 1 : 0); }
    return g;
}
// Philox blocks per 32-element group (both parties + dealer): g-layer 2 per plane, G-only node 2,
// G+P node 3, daBit 32 (K0) + 1 (K1)
__host__ __device__ inline u64 cone_philox_per_group(int w)
{
    const int m = w - 1;
    if (m <= 0) return 33;
    const int L = ceil_log2i(m);
    u64 c = 2ull * (u64)m + 33ull;
    for (int k = 0; k < L; ++k) { const int n = cone_nodes(m, k); c += 2ull * (u64)n + (n > 0 ? (u64)(n - 1) : 0ull); }
    return c;
}

// item t of a level -> (group, node): t / ng for t < 128, ng <= 32, by a 16-bit reciprocal
__device__ __forceinline__ int cone_div(int t, int ng) { return (t * ((65536 + ng - 1) / ng)) >> 16; }

// ---------------------------------------------------------------- BOTH ----
template <int G, int NL>
__device__ void ltz_cone_both(const Keys& K, u64 q0, u32 s, int w, const Sh (&x)[G], Sh (&z)[G],
                              int lane, ConeSmem<G, NL>& sm)
{
    static_assert(NL == 32 || NL == 64, "32 or 64 leaf positions");
    constexpr int H = NL / 32;
    const int m = w - 1;                      // 0..63
    const int L = (m > 0) ? ceil_log2i(m) : 0;
#pragma unroll
    for (int g = 0; g < G; ++g) {
#pragma unroll
        for (int h = 0; h < H; ++h) {
            if (h == 1 && m <= 32) break;     // warp-uniform: the upper plane half is all pads
            const int j = lane + 32 * h;
            const u32 P0 = transpose32((u32)(x[g].s0 >> (32 * h)), lane), P1 = transpose32((u32)(x[g].s1 >> (32 * h)), lane);
            const bool leaf = j < m;
            u32 g0 = 0, g1 = 0;
            if (leaf) {
                const uint4 t0 = prg(K.k0, q0 + g, s, ltz_slot(0, j, 0));
                const uint4 t1 = prg(K.k1, q0 + g, s, ltz_slot(0, j, 0));
                and_both(P0, 0u, 0u, P1, t0.x, t0.y, t0.z, t1.x, t1.y, g0, g1);
            }
            sm.w[g][j][0] = g0;
            sm.w[g][j][1] = g1;
            sm.w[g][j][2] = leaf ? P0 : 0xffffffffu;    // pad P = public 1: party 0 holds 1
            sm.w[g][j][3] = leaf ? P1 : 0u;
        }
    }
    __syncwarp();
    // Flat gate triples (G x the tree's gate nodes <= 64): the tree's Philox blocks are data-
    // independent, so every lane generates the blocks of its items t = lane + 32 r (level-major over
    // all levels) up front -- one or two passes of 3 blocks with full ILP instead of a pass per level
    // with most lanes idle -- and evaluates those items in the level passes from registers.
    constexpr int RF = (G * (NL - 1) + 31) / 32;
#ifndef MPC_CONE_FLAT
#define MPC_CONE_FLAT 1
#endif
    if constexpr (MPC_CONE_FLAT && RF <= 2) {
        int tot = 0;
        for (int k = 0; k < L; ++k) tot += G * cone_nodes(m, k);
        uint4 TG[RF], TP[RF], T1[RF];
        int kk[RF], gg[RF], ii[RF];
#pragma unroll
        for (int r = 0; r < RF; ++r) {
            int t = lane + 32 * r, k = 0, ng = 0;
            kk[r] = -1; gg[r] = 0; ii[r] = 0;
            if (t < tot) {
                for (; k < L; ++k) { ng = cone_nodes(m, k); if (t < G * ng) break; t -= G * ng; }
                kk[r] = k; gg[r] = G == 1 ? 0 : cone_div(t, ng); ii[r] = t - gg[r] * ng;
            }
            const u64 q = q0 + (u64)gg[r];
            const int kq = kk[r] < 0 ? 0 : kk[r];
            TG[r] = prg(K.k0, q, s, ltz_slot(kq + 1, ii[r], 0));
            TP[r] = prg(K.k0, q, s, ltz_slot(kq + 1, ii[r], 1));
            T1[r] = prg(K.k1, q, s, ltz_slot(kq + 1, ii[r], 0));
        }
        for (int k = 0; k < L; ++k) {
#pragma unroll
            for (int r = 0; r < RF; ++r) {
                if (kk[r] != k) continue;
                const int g = gg[r], i = ii[r], lo = i << (k + 1), hi = lo + (1 << k);
                const u32 gl0 = sm.w[g][lo][0], gl1 = sm.w[g][lo][1], pl0 = sm.w[g][lo][2], pl1 = sm.w[g][lo][3];
                const u32 gh0 = sm.w[g][hi][0], gh1 = sm.w[g][hi][1], ph0 = sm.w[g][hi][2], ph1 = sm.w[g][hi][3];
                u32 ng0, ng1, np0, np1;
                and_both(ph0, ph1, gl0, gl1, TG[r].x, TG[r].y, TG[r].z, T1[r].x, T1[r].y, ng0, ng1);
                and_both(ph0, ph1, pl0, pl1, TP[r].x, TP[r].y, TP[r].z, T1[r].z, T1[r].w, np0, np1);
                sm.w[g][lo][0] = gh0 ^ ng0; sm.w[g][lo][1] = gh1 ^ ng1;
                if (i > 0) { sm.w[g][lo][2] = np0; sm.w[g][lo][3] = np1; }   // P off the left spine only
            }
            __syncwarp();
        }
    } else
    for (int k = 0; k < L; ++k) {
        const int ng = cone_nodes(m, k), items = G * ng;
        for (int base = 0; base < items; base += 32) {
            // uniform control flow: every lane issues the three blocks (SIMT issues them for the warp
            // anyway) so the compiler interleaves the independent Philox chains; stores are masked
            const int t = base + lane;
            const bool valid = t < items;
            const int g = valid ? cone_div(t, ng) : 0, i = valid ? t - g * ng : 0;
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
                if (i > 0) { sm.w[g][lo][2] = np0; sm.w[g][lo][3] = np1; }   // P off the left spine only
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
// Same circuit, one party's shares; the g-layer, every tree level and the B2A are ONE warp
// exchange each, carrying all G groups' words (so 1 + L + 1 rounds per G groups).
template <int G, int NL, int R>
__device__ void ltz_cone_pair(PairP<R>& pr, u64 q0, u32 s, int w, const u64 (&x)[G], u64 (&z)[G], int lane,
                              ConeSmem<G, NL>& sm)
{
    constexpr int H = NL / 32;
    static_assert(G * H <= XW, "one exchange carries at most XW words per lane");
    static_assert(2 * ((G * NL / 2 + 31) / 32) <= XW, "a level's gate nodes fit one exchange");
    const int m = w - 1;
    const int L = (m > 0) ? ceil_log2i(m) : 0;
    const int pty = pr.pty;
    const Keys& K = *pr.Kp;
    {   // g-layer for all G groups (and both plane halves) in one exchange
        u32 ta[G][H], tb[G][H], tc[G][H], dd[G][H], ee[G][H], Pp[G][H];
#pragma unroll
        for (int g = 0; g < G; ++g) {
#pragma unroll
            for (int h = 0; h < H; ++h) {
                if (h == 1 && m <= 32) break;
                const int j = lane + 32 * h;
                Pp[g][h] = transpose32((u32)(x[g] >> (32 * h)), lane);
                ta[g][h] = tb[g][h] = tc[g][h] = 0;
                dd[g][h] = ee[g][h] = 0;
                if (j < m) {
                    const uint4 t0 = pr.k0ok() ? prg(K.k0, q0 + g, s, ltz_slot(0, j, 0)) : make_uint4(0, 0, 0, 0);
                    uint4 t1 = make_uint4(0, 0, 0, 0);
                    if (pty == 1) t1 = prg(K.k1, q0 + g, s, ltz_slot(0, j, 0));
                    pr.and_triple(t0, t1, 0, ta[g][h], tb[g][h], tc[g][h]);
                    dd[g][h] = (pty == 0 ? Pp[g][h] : 0u) ^ ta[g][h];
                    ee[g][h] = (pty == 0 ? 0u : Pp[g][h]) ^ tb[g][h];
                }
                pr.put(lane, g * H + h, (u64)dd[g][h] | ((u64)ee[g][h] << 32), j < m);
            }
        }
        pr.exch(lane);
#pragma unroll
        for (int g = 0; g < G; ++g) {
#pragma unroll
            for (int h = 0; h < H; ++h) {
                if (h == 1 && m <= 32) break;
                const int j = lane + 32 * h;
                const bool leaf = j < m;
                u32 gg = 0;
                if (leaf) {
                    const u64 pw = pr.get(lane, g * H + h);
                    gg = pr.and_finish(ta[g][h], tb[g][h], tc[g][h], dd[g][h] ^ (u32)pw, ee[g][h] ^ (u32)(pw >> 32));
                }
                sm.w[g][j][0] = gg;
                sm.w[g][j][2] = leaf ? Pp[g][h] : (pty == 0 ? 0xffffffffu : 0u);   // pad P = public 1
            }
        }
    }
    __syncwarp();
    for (int k = 0; k < L; ++k) {
        const int ng = cone_nodes(m, k), items = G * ng;
        constexpr int IPL = (G * NL / 2 + 31) / 32;      // items per lane (level 0 is the largest)
        u32 ga[IPL], gb[IPL], gc[IPL], pa[IPL], pb[IPL], pc[IPL], dG[IPL], eG[IPL], dP[IPL], eP[IPL], gh[IPL];
        int lo_[IPL], gi[IPL], ii[IPL];
#pragma unroll
        for (int v = 0; v < IPL; ++v) {
            const int t = v * 32 + lane;
            ii[v] = -1;
            if (v * 32 < items) {                 // warp-uniform: blocks issued by every lane of the pass
                const bool valid = t < items;
                const int g = valid ? cone_div(t, ng) : 0, i = valid ? t - g * ng : 0;
                const int lo = i << (k + 1), hi = lo + (1 << k);
                gi[v] = g; lo_[v] = lo;
                if (valid) ii[v] = i;
                u32 gl = 0, pl = 0, ph = 0;
                gh[v] = 0;
                if (valid) { gl = sm.w[g][lo][0]; pl = sm.w[g][lo][2]; ph = sm.w[g][hi][2]; gh[v] = sm.w[g][hi][0]; }
                const u64 q = q0 + (u64)g;
                uint4 tg = make_uint4(0, 0, 0, 0), tp = tg;
                if (pr.k0ok()) { tg = prg(K.k0, q, s, ltz_slot(k + 1, i, 0)); tp = prg(K.k0, q, s, ltz_slot(k + 1, i, 1)); }
                uint4 t1 = make_uint4(0, 0, 0, 0);
                if (pty == 1) t1 = prg(K.k1, q, s, ltz_slot(k + 1, i, 0));
                pr.and_triple2(tg, tp, t1, ga[v], gb[v], gc[v], pa[v], pb[v], pc[v]);
                dG[v] = ph ^ ga[v]; eG[v] = gl ^ gb[v];
                dP[v] = ph ^ pa[v]; eP[v] = pl ^ pb[v];
                pr.put(lane, 2 * v, (u64)dG[v] | ((u64)eG[v] << 32), valid);
                pr.put(lane, 2 * v + 1, (u64)dP[v] | ((u64)eP[v] << 32), valid && i > 0);
            }
        }
        pr.exch(lane);
#pragma unroll
        for (int v = 0; v < IPL; ++v) {
            if (ii[v] < 0) continue;
            const u64 w0 = pr.get(lane, 2 * v);
            const u32 ngv = pr.and_finish(ga[v], gb[v], gc[v], dG[v] ^ (u32)w0, eG[v] ^ (u32)(w0 >> 32));
            sm.w[gi[v]][lo_[v]][0] = gh[v] ^ ngv;
            if (ii[v] > 0) {
                const u64 w1 = pr.get(lane, 2 * v + 1);
                sm.w[gi[v]][lo_[v]][2] = pr.and_finish(pa[v], pb[v], pc[v], dP[v] ^ (u32)w1, eP[v] ^ (u32)(w1 >> 32));
            }
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
        const uint4 D0 = pr.k0ok() ? prg(K.k0, q0 + g, s, 2u + (u32)lane) : make_uint4(0, 0, 0, 0);
        const u32 d1x = __shfl_sync(FULL, k1w, g);
        u32 rB;
        if (pty == 0) { rA[g] = w64(D0.x, D0.y); rB = D0.z & 1u; }
        else { rB = (d1x >> lane) & 1u; rA[g] = pr.dabit_r1A(D0, rB); }
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
