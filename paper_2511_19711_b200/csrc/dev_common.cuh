// dev_common.cuh -- L0 device primitives for sm_100a: Philox4x32-10, ring helpers,
// warp bit-plane transpose.  (DESIGN.md 2.1 / 2.3.)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mpc {

typedef uint64_t u64;
typedef int64_t i64;
typedef unsigned int u32;
typedef uint8_t u8;

constexpr u32 FULL = 0xffffffffu;
constexpr int FRAC = 16;

// A 64-bit Philox key split into (lo32, hi32).  Keys are warp-uniform, so the per-round
// key bumps run on the uniform datapath (UIADD3) and LOP3 reads the key from a uniform
// register.  (Precomputed round-key tables were tried: 40 round keys overflow the 63
// uniform registers inside the LTZ kernels and turn into IMAD.U32 moves on the FMA pipe.)
struct Key { u32 lo, hi; };

struct Keys {
    Key ks, k0, k1;   // K_s, K_0, K_1
};

__host__ __device__ inline Key make_key(u64 k) { return Key{(u32)k, (u32)(k >> 32)}; }

// Philox4x32-10 (Salmon et al. SC'11).  Counter (c0..c3), key (k0, k1); the key is
// bumped by the Weyl constants before every round but the first.  The multiplies
// are 32x32->64 (IMAD.WIDE.U32).
__device__ __forceinline__ uint4 philox(const Key& key, u32 c0, u32 c1, u32 c2, u32 c3)
{
    u32 k0 = key.lo, k1 = key.hi;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const u64 p0 = (u64)0xD2511F53u * (u64)c0;
        const u64 p1 = (u64)0xCD9E8D57u * (u64)c2;
        const u32 n0 = (u32)(p1 >> 32) ^ c1 ^ k0;
        const u32 n2 = (u32)(p0 >> 32) ^ c3 ^ k1;
        c1 = (u32)p1;
        c3 = (u32)p0;
        c0 = n0;
        c2 = n2;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return make_uint4(c0, c1, c2, c3);
}

// ---- Philox4x32-10 split at the shared prefix -------------------------------------------
// Many blocks of one protocol step share counter words, so the first rounds' products that
// depend only on the shared words are computed once per thread and reused (identical output
// bits; the tests compare with the oracle's plain Philox).
// The "slot" form: counters (c0, c1, c2, c3) with only c3 varying (the LTZ gate, daBit and
// K1-word blocks of one group and step): 4 of the 20 products are shared, 16 per block remain.
// (The analogous "unit" form for Beaver blocks -- 2 of 20 shared -- measured no gain: the
// element-wise kernels are not multiply-bound.)
constexpr u32 PH_M0 = 0xD2511F53u, PH_M1 = 0xCD9E8D57u, PH_W0 = 0x9E3779B9u, PH_W1 = 0xBB67AE85u;

__device__ __forceinline__ void ph_rounds(u32 k0, u32 k1, int r0, u32& c0, u32& c1, u32& c2, u32& c3)
{
    k0 += (u32)r0 * PH_W0; k1 += (u32)r0 * PH_W1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r < r0) continue;
        const u64 p0 = (u64)PH_M0 * (u64)c0;
        const u64 p1 = (u64)PH_M1 * (u64)c2;
        const u32 n0 = (u32)(p1 >> 32) ^ c1 ^ k0;
        const u32 n2 = (u32)(p0 >> 32) ^ c3 ^ k1;
        c1 = (u32)p1; c3 = (u32)p0; c0 = n0; c2 = n2;
        k0 += PH_W0; k1 += PH_W1;
    }
}

struct PhSlot { u32 x2, y, w, z0, c1; };           // shared prefix, slot form
__device__ __forceinline__ PhSlot ph_slot_pre(const Key& k, u32 c0, u32 c1, u32 c2)
{
    const u64 p0 = (u64)PH_M0 * c0, p1 = (u64)PH_M1 * c2;                 // round 0
    const u32 A0 = (u32)(p1 >> 32) ^ c1 ^ k.lo, A1 = (u32)p1, A3 = (u32)p0;
    const u32 X2 = (u32)(p0 >> 32) ^ k.hi;                                 // A2 = X2 ^ c3
    const u64 q0 = (u64)PH_M0 * A0;                                        // round 1, P0
    const u32 B2 = (u32)(q0 >> 32) ^ A3 ^ (k.hi + PH_W1), B3 = (u32)q0;
    const u64 r1 = (u64)PH_M1 * B2;                                        // round 2, P1
    PhSlot P;
    P.x2 = X2;
    P.y = A1 ^ (k.lo + PH_W0);                                             // B0 = hi(M1 A2) ^ y
    P.z0 = (u32)(r1 >> 32) ^ (k.lo + 2u * PH_W0);                          // C0 = z0 ^ B1
    P.c1 = (u32)r1;
    P.w = B3 ^ (k.hi + 2u * PH_W1);                                        // C2 = hi(M0 B0) ^ w
    return P;
}
__device__ __forceinline__ uint4 ph_slot_post(const Key& k, const PhSlot& P, u32 c3)
{
    const u64 p1 = (u64)PH_M1 * (P.x2 ^ c3);                               // round 1, P1
    const u32 B0 = (u32)(p1 >> 32) ^ P.y, B1 = (u32)p1;
    const u64 p0 = (u64)PH_M0 * B0;                                        // round 2, P0
    u32 c0 = P.z0 ^ B1, c1 = P.c1, c2 = (u32)(p0 >> 32) ^ P.w, c3o = (u32)p0;
    ph_rounds(k.lo, k.hi, 3, c0, c1, c2, c3o);
    return make_uint4(c0, c1, c2, c3o);
}

// PRG(K, unit, step, slot) of DESIGN.md 2.3.
__device__ __forceinline__ uint4 prg(const Key& key, u64 unit, u32 step, u32 slot)
{
    return philox(key, (u32)unit, (u32)(unit >> 32), step, slot);
}

// PRG(K, unit, step, *) with the slot varying: prefix once per (K, unit, step).
struct PrgQ { Key k; PhSlot p; };
__device__ __forceinline__ PrgQ prg_q(const Key& key, u64 unit, u32 step)
{
    return PrgQ{key, ph_slot_pre(key, (u32)unit, (u32)(unit >> 32), step)};
}
__device__ __forceinline__ uint4 prg(const PrgQ& P, u32 slot) { return ph_slot_post(P.k, P.p, slot); }

__device__ __forceinline__ u64 w64(u32 lo, u32 hi) { return (u64)lo | ((u64)hi << 32); }

// per-share arithmetic shift (local truncation)
__device__ __forceinline__ u64 shr(u64 v, int k) { return (u64)(((i64)v) >> k); }

// LTZ gate slot
__device__ __forceinline__ u32 ltz_slot(int lv, int j, int c)
{
    return 64u + 128u * (u32)lv + 2u * (u32)j + (u32)c;
}

// 32x32 bit-matrix transpose across a warp: lane l holds row l (bit j = column j);
// on return lane j holds column j (bit l = row l).  5 butterfly stages.
__device__ __forceinline__ u32 transpose32(u32 v, int lane)
{
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        const u32 m = (s == 16) ? 0x0000FFFFu : (s == 8) ? 0x00FF00FFu
                    : (s == 4) ? 0x0F0F0F0Fu : (s == 2) ? 0x33333333u : 0x55555555u;
        const u32 o = __shfl_xor_sync(FULL, v, s);
        v = (lane & s) ? ((v & ~m) | ((o >> s) & m)) : ((v & m) | ((o << s) & ~m));
    }
    return v;
}

// q = n / d for n < 2^31 with one IMAD.HI + shift (round-up multiplier, p = 31 + ceil(log2 d))
struct FastDiv { u32 d, m, s; };
__host__ __device__ inline FastDiv make_fastdiv(u32 d)
{
    FastDiv f{d, 0u, 0u};
    if (d > 1) {
        int l = 0;
        while ((1ull << l) < d) ++l;
        const int p = 31 + l;
        f.m = (u32)(((1ull << p) + d - 1) / d);
        f.s = (u32)(p - 32);
    }
    return f;
}
__device__ __forceinline__ u32 fdiv(u32 n, const FastDiv& f)
{
    return f.d == 1 ? n : (__umulhi(n, f.m) >> f.s);
}

__host__ __device__ inline int ceil_log2i(int m)
{
    int L = 0;
    while ((1 << L) < m) ++L;
    return L;
}

}  // namespace mpc
