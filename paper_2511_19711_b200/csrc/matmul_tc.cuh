// matmul_tc.cuh -- the ring GEMM of mpc_matmul on the 5th-generation tensor cores (sm_100a).
//
// Z_2^64 products through 8-bit limbs: with a = sum_i 2^(8i) a_i and
// b = sum_j 2^(8j) b_j (unsigned bytes),
//     a * b mod 2^64 = sum_{s=0..7} 2^(8s) S_s,   S_s = sum_{i+j=s} a_i b_j,
// so a ring GEMM is 36 u8 x u8 -> s32 GEMMs accumulated into 8 TMEM accumulators S_0..S_7.
// Each S_s is exact as long as (s+1) K' 255^2 < 2^32 for s <= 3 (K' < 16513); for s >= 4 only
// its low 64 - 8s <= 32 bits survive the shift, so the 32-bit wrap of the accumulator is
// harmless.  The epilogue forms sum_s (u64)S_s << 8s, adds +-C0 from the PRG and truncates.
//
// Operands are pre-tiled by k_mm_limbs_lhs / _rhs into the UMMA canonical K-major layout without
// swizzle (core matrix = 8 rows x 16 B; LBO = 128 B between the two 16-B K-chunks, SBO = 256 B
// between 8-row groups), one contiguous chunk per (row block, K block of 32) holding all 8
// limbs: A chunk = 8 x (128 x 32 B) = 32 KB, B chunk = 8 x (TC_BN x 32 B) = 8 KB at TC_BN = 32.
// A stage is therefore two flat cp.async.bulk copies (TMA without tensor maps) completing on an
// mbarrier.
// One CTA = one 128 x TC_BN output tile (8 accumulators x TC_BN TMEM columns); thread 0 issues
// the copies (2-3 stage ring) and one tcgen05.mma per A limb i against the stacked B limbs
// 0..7-i (N = TC_BN (8-i) <= 256; split in two at TC_BN = 64) per K block; all 4 warps run the
// epilogue (warp w owns TMEM lanes 32w..32w+31 = rows).
#pragma once
#include "matmul.cuh"

namespace mpc {

// Output tile 128 x TC_BN: 8 accumulators take 8 * TC_BN TMEM columns.  TC_BN = 32 (default) uses
// 256 columns and ~80 KB of shared memory, so TWO CTAs share an SM and one CTA's epilogue overlaps
// the other's MMAs; TC_BN = 64 fills TMEM (one CTA per SM, epilogue serialised with the MMAs).
#ifndef MPC_TC_BN
#define MPC_TC_BN 32
#endif
constexpr int TC_BM = 128, TC_BN = MPC_TC_BN, TC_BK = 32, TC_STAGES = TC_BN == 32 ? 2 : 3;
constexpr int TC_CTAS_PER_SM = TC_BN == 32 ? 2 : 1, TC_TMEM_COLS = 8 * TC_BN;
constexpr int TC_A_TILE = TC_BM * TC_BK, TC_B_TILE = TC_BN * TC_BK;          // bytes per limb tile
constexpr int TC_A_CHUNK = 8 * TC_A_TILE, TC_B_CHUNK = 8 * TC_B_TILE;          // bytes per stage
constexpr int TC_SMEM = TC_STAGES * (TC_A_CHUNK + TC_B_CHUNK) + 1024;

// byte offset of (row r, k byte kb) inside one limb tile (canonical K-major, no swizzle)
__host__ __device__ inline int tc_tile_off(int r, int kb) { return (r >> 3) * 256 + (kb >> 4) * 128 + (r & 7) * 16 + (kb & 15); }

// ---- limb tiling ------------------------------------------------------------------------------
// Operand of one party: up to three terms concatenated along K (K' = nt * K).  LHS terms are
// [batch][M][K] (rows = m), RHS terms [batch][K][N] (rows = n, transposed to K-major).  Output:
// [batch][row block][K block][limb][tile], zero padded to whole blocks.  A thread packs one
// 16-byte core-matrix row (16 consecutive k' of one row) for all 8 limbs.
struct LimbArgs {
    const u64* t[3]; int nt; int rows, K, Kp, rhs, rows_blk; int batch; i64 in_stride; u8* out;
};
// Each term occupies its own whole K blocks: term t holds k' in [t Kpad, t Kpad + K), Kpad =
// 32 ceil(K / 32), the rest zero (zeros add nothing to the products), so Kp = nt Kpad and the
// fused BOTH-mode kernels below can write a term's tile without touching its neighbours.
__host__ __device__ inline int tc_kpad(int K) { return (K + TC_BK - 1) / TC_BK * TC_BK; }
// RHS limb tiling through a shared-memory transpose: one CTA per (batch, 64-column block, K block
// of 32): coalesced loads of 32 rows x 64 columns, then 128 threads pack the 64 x 2 core-matrix
// rows of all 8 limbs and write the 16 KB chunk contiguously.
__global__ void __launch_bounds__(2 * TC_BN) k_mm_limbs_rhs(LimbArgs a)
{
    __shared__ u64 sm[TC_BK][TC_BN + 1];
    const int KB = a.Kp / TC_BK, NB = (a.rows + TC_BN - 1) / TC_BN;
    const int Kpad = tc_kpad(a.K);
    const i64 ntile = (i64)a.batch * NB * KB;
    for (i64 tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
        const int b = (int)(tile / ((i64)NB * KB));
        const int rem = (int)(tile - (i64)b * NB * KB), nb = rem / KB, kb = rem - (rem / KB) * KB;
        for (int l = threadIdx.x; l < TC_BK * TC_BN; l += blockDim.x) {
            const int kr = l / TC_BN, nc = l - kr * TC_BN;
            const int kk = kb * TC_BK + kr, n = nb * TC_BN + nc;
            u64 v = 0;
            const int t = kk / Kpad, k = kk - t * Kpad;
            if (t < a.nt && k < a.K && n < a.rows) v = a.t[t][(i64)b * a.in_stride + (i64)k * a.rows + n];
            sm[kr][nc] = v;
        }
        __syncthreads();
        if (threadIdx.x < 2 * TC_BN) {
            const int n = threadIdx.x >> 1, ch = threadIdx.x & 1;
            uint4 limb[8];
            u32* lw = reinterpret_cast<u32*>(limb);
#pragma unroll
            for (int q = 0; q < 32; ++q) lw[q] = 0;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const u64 v = sm[ch * 16 + e][n];
#pragma unroll
                for (int i = 0; i < 8; ++i) lw[i * 4 + (e >> 2)] |= ((u32)(v >> (8 * i)) & 0xffu) << (8 * (e & 3));
            }
            u8* dst = a.out + (((i64)b * NB + nb) * KB + kb) * (i64)TC_B_CHUNK;
            const int off = tc_tile_off(n, ch * 16);
#pragma unroll
            for (int i = 0; i < 8; ++i) *reinterpret_cast<uint4*>(dst + (i64)i * TC_B_TILE + off) = limb[i];
        }
        __syncthreads();
    }
}

// LHS limb tiling through shared memory: one CTA per (batch, 128-row block, K block of 32):
// coalesced loads of 128 rows x 32 k' (each row 256 contiguous bytes), then 256 threads pack the
// 128 x 2 core-matrix rows of all 8 limbs and write the 32 KB chunk contiguously.
__global__ void __launch_bounds__(256) k_mm_limbs_lhs(LimbArgs a)
{
    __shared__ u64 sm[TC_BM][TC_BK + 1];
    const int KB = a.Kp / TC_BK, MB = (a.rows + TC_BM - 1) / TC_BM;
    const int Kpad = tc_kpad(a.K);
    const i64 ntile = (i64)a.batch * MB * KB;
    for (i64 tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
        const int b = (int)(tile / ((i64)MB * KB));
        const int rem = (int)(tile - (i64)b * MB * KB), mb = rem / KB, kb = rem - (rem / KB) * KB;
        for (int l = threadIdx.x; l < TC_BM * TC_BK; l += blockDim.x) {
            const int r = l / TC_BK, kc = l - r * TC_BK;
            const int kk = kb * TC_BK + kc, m = mb * TC_BM + r;
            u64 v = 0;
            const int t = kk / Kpad, k = kk - t * Kpad;
            if (t < a.nt && k < a.K && m < a.rows) v = a.t[t][(i64)b * a.in_stride + (i64)m * a.K + k];
            sm[r][kc] = v;
        }
        __syncthreads();
        {
            const int r = threadIdx.x >> 1, ch = threadIdx.x & 1;
            uint4 limb[8];
            u32* lw = reinterpret_cast<u32*>(limb);
#pragma unroll
            for (int q = 0; q < 32; ++q) lw[q] = 0;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const u64 v = sm[r][ch * 16 + e];
#pragma unroll
                for (int i = 0; i < 8; ++i) lw[i * 4 + (e >> 2)] |= ((u32)(v >> (8 * i)) & 0xffu) << (8 * (e & 3));
            }
            u8* dst = a.out + (((i64)b * MB + mb) * KB + kb) * (i64)TC_A_CHUNK;
            const int off = tc_tile_off(r, ch * 16);
#pragma unroll
            for (int i = 0; i < 8; ++i) *reinterpret_cast<uint4*>(dst + (i64)i * TC_A_TILE + off) = limb[i];
        }
        __syncthreads();
    }
}

// ---- BOTH mode: Beaver masking fused with the limb tiling ------------------------------------
// One pass over the input shares of one operand writes every limb tile the GEMM reads (DESIGN.md
// 2.10): the thread derives the triple shares r0 = A_0 (key K_0), r1 = A_1 (key K_1) of its
// elements from the PRG (unit = global element index, slot 8 for X, 9 for Y; the same values as
// the mask pass of the PAIR path), opens E = (x_0 - r0) + (x_1 - r1) in registers, and packs the
// terms of both parties:
//   X: party 0 [E, A0],        party 1 [As = A0 + A1, E, A1]
//   Y: party 0 [B0 + F, F],    party 1 [Bs = B0 + B1, B1, F]
// in term-padded K blocks (tc_kpad).  The mask pass wrote 4 planes (32 B / element) that the limb
// pass read back (40 B) before writing the limbs (40 B); here 16 B are read and 40 B written.
struct FuseArgs {
    Keys keys; u32 s; const u64* x0; const u64* x1; int rows, K, batch; u64 goff; u8* out0; u8* out1;
};

// pack FW (4 or 8) u64 into the 8 limbs' FW-byte pieces (piece i = bytes i of v[0..FW-1]) and
// store them at (row r, k byte kb) of the 8 consecutive limb tiles of a chunk
constexpr int FW = 4;                                  // elements (k) per thread in the fused kernels
__device__ __forceinline__ void tc_store(u8* chunk, int tile_bytes, int r, int kb, const u64 (&v)[FW])
{
    const int off = tc_tile_off(r, kb);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        u32 w = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) w |= ((u32)(v[e] >> (8 * i)) & 0xffu) << (8 * e);
        *reinterpret_cast<u32*>(chunk + (i64)i * tile_bytes + off) = w;
    }
}

__device__ __forceinline__ u64 prg_pick(const uint4& R, u64 u) { return (u & 1) ? w64(R.z, R.w) : w64(R.x, R.y); }

// X (LHS, [batch][M][K]): CTA = 32 rows x 32 k of one (batch, 128-row block, K block); thread =
// (row, FW consecutive k): loads first, then the PRG blocks of the (at most 3) unit pairs.
__global__ void __launch_bounds__(256) k_mm_fuse_lhs(FuseArgs a)
{
    constexpr int TPR = TC_BK / FW, RPC = 256 / TPR, QB = TC_BM / RPC;   // threads per row, rows per CTA
    const int KB = tc_kpad(a.K) / TC_BK, MB = (a.rows + TC_BM - 1) / TC_BM;
    const i64 ntile = (i64)a.batch * QB * MB * KB;
    const int kq = threadIdx.x % TPR, rl = threadIdx.x / TPR;
    for (i64 tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
        const int b = (int)(tile / ((i64)QB * MB * KB));
        const int rem = (int)(tile - (i64)b * QB * MB * KB), hb = rem / KB, kb = rem - hb * KB;
        const int mb = hb / QB, r = (hb % QB) * RPC + rl, m = mb * TC_BM + r, k0 = kb * TC_BK + kq * FW;
        const i64 base = ((i64)b * a.rows + m) * a.K;
        const u64 u0 = (a.goff + (u64)b) * (u64)a.rows * (u64)a.K + (u64)m * (u64)a.K + (u64)k0;
        u64 x0[FW], x1[FW];
        bool ok[FW];
#pragma unroll
        for (int e = 0; e < FW; ++e) {
            ok[e] = m < a.rows && k0 + e < a.K;
            x0[e] = ok[e] ? __ldg(a.x0 + base + k0 + e) : 0;
            x1[e] = ok[e] ? __ldg(a.x1 + base + k0 + e) : 0;
        }
        uint4 R0[FW / 2 + 1], R1[FW / 2 + 1];
#pragma unroll
        for (int j = 0; j <= FW / 2; ++j) {
            if (j < FW / 2 || (u0 & 1)) {
                R0[j] = prg(a.keys.k0, (u0 >> 1) + j, a.s, 8u);
                R1[j] = prg(a.keys.k1, (u0 >> 1) + j, a.s, 8u);
            } else R0[j] = R1[j] = make_uint4(0, 0, 0, 0);
        }
        u64 E[FW], A0[FW], A1[FW];
#pragma unroll
        for (int e = 0; e < FW; ++e) {
            const u64 u = u0 + e;
            const int j = (e + (int)(u0 & 1)) >> 1;              // block of unit u (register select, no local array)
            uint4 P0 = R0[0], P1 = R1[0];
#pragma unroll
            for (int q = 1; q <= FW / 2; ++q) if (j == q) { P0 = R0[q]; P1 = R1[q]; }
            const u64 r0 = ok[e] ? prg_pick(P0, u) : 0, r1 = ok[e] ? prg_pick(P1, u) : 0;
            A0[e] = r0; A1[e] = r1;
            E[e] = ok[e] ? (x0[e] - r0) + (x1[e] - r1) : 0;
        }
        const int kbyte = kq * FW;
        u8* c0 = a.out0 + (((i64)b * MB + mb) * 2 * KB) * (i64)TC_A_CHUNK;
        u8* c1 = a.out1 + (((i64)b * MB + mb) * 3 * KB) * (i64)TC_A_CHUNK;
        tc_store(c0 + (i64)(0 * KB + kb) * TC_A_CHUNK, TC_A_TILE, r, kbyte, E);
        tc_store(c0 + (i64)(1 * KB + kb) * TC_A_CHUNK, TC_A_TILE, r, kbyte, A0);
        tc_store(c1 + (i64)(1 * KB + kb) * TC_A_CHUNK, TC_A_TILE, r, kbyte, E);
        tc_store(c1 + (i64)(2 * KB + kb) * TC_A_CHUNK, TC_A_TILE, r, kbyte, A1);
#pragma unroll
        for (int e = 0; e < FW; ++e) A0[e] += A1[e];
        tc_store(c1 + (i64)(0 * KB + kb) * TC_A_CHUNK, TC_A_TILE, r, kbyte, A0);
    }
}

// Y (RHS, [batch][K][N], packed K-major per column n): CTA = 64 columns x 32 k of one (batch,
// 64-column group, K block); thread = (2 adjacent columns, FW consecutive k), so both halves of a
// PRG block are used when the column pair is unit-aligned.
__global__ void __launch_bounds__(256) k_mm_fuse_rhs(FuseArgs a)
{
    constexpr int TPC = TC_BK / FW, CPC = 2 * (256 / TPC);              // threads per column pair, columns per CTA
    const int KB = tc_kpad(a.K) / TC_BK, NB = (a.rows + TC_BN - 1) / TC_BN, NG = (a.rows + CPC - 1) / CPC;
    const i64 ntile = (i64)a.batch * NG * KB;
    const int kq = threadIdx.x % TPC, np = threadIdx.x / TPC;
    for (i64 tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
        const int b = (int)(tile / ((i64)NG * KB));
        const int rem = (int)(tile - (i64)b * NG * KB), ng = rem / KB, kb = rem - ng * KB;
        const int n = ng * CPC + 2 * np, k0 = kb * TC_BK + kq * FW;
        const i64 base = (i64)b * a.K * a.rows;
        const u64 ub = (a.goff + (u64)b) * (u64)a.K * (u64)a.rows;
        u64 y0[2][FW], y1[2][FW];
#pragma unroll
        for (int e = 0; e < FW; ++e)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const bool v = k0 + e < a.K && n + j < a.rows;
                const i64 idx = base + (i64)(k0 + e) * a.rows + n + j;
                y0[j][e] = v ? __ldg(a.x0 + idx) : 0;
                y1[j][e] = v ? __ldg(a.x1 + idx) : 0;
            }
        u64 F[2][FW], B0[2][FW], B1[2][FW];
#pragma unroll
        for (int e = 0; e < FW; ++e) {
            const int k = k0 + e;
            const u64 u = ub + (u64)k * (u64)a.rows + (u64)n;
            const bool v0 = k < a.K && n < a.rows, v1 = k < a.K && n + 1 < a.rows;
            uint4 R0 = make_uint4(0, 0, 0, 0), R1 = R0, S0, S1;
            if (v0) { R0 = prg(a.keys.k0, u >> 1, a.s, 9u); R1 = prg(a.keys.k1, u >> 1, a.s, 9u); }
            S0 = R0; S1 = R1;
            if (v1 && (u & 1)) { S0 = prg(a.keys.k0, (u >> 1) + 1, a.s, 9u); S1 = prg(a.keys.k1, (u >> 1) + 1, a.s, 9u); }
            const u64 r00 = v0 ? prg_pick(R0, u) : 0, r10 = v0 ? prg_pick(R1, u) : 0;
            const u64 r01 = v1 ? prg_pick(S0, u + 1) : 0, r11 = v1 ? prg_pick(S1, u + 1) : 0;
            B0[0][e] = r00; B1[0][e] = r10; F[0][e] = v0 ? (y0[0][e] - r00) + (y1[0][e] - r10) : 0;
            B0[1][e] = r01; B1[1][e] = r11; F[1][e] = v1 ? (y0[1][e] - r01) + (y1[1][e] - r11) : 0;
        }
        const int kbyte = kq * FW;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int nn = n + j, nb = nn / TC_BN, rr = nn - nb * TC_BN;
            if (nb >= NB) continue;
            u8* c0 = a.out0 + (((i64)b * NB + nb) * 2 * KB) * (i64)TC_B_CHUNK;
            u8* c1 = a.out1 + (((i64)b * NB + nb) * 3 * KB) * (i64)TC_B_CHUNK;
            u64 G[FW], Bs[FW];
#pragma unroll
            for (int e = 0; e < FW; ++e) { G[e] = B0[j][e] + F[j][e]; Bs[e] = B0[j][e] + B1[j][e]; }
            tc_store(c0 + (i64)(0 * KB + kb) * TC_B_CHUNK, TC_B_TILE, rr, kbyte, G);
            tc_store(c0 + (i64)(1 * KB + kb) * TC_B_CHUNK, TC_B_TILE, rr, kbyte, F[j]);
            tc_store(c1 + (i64)(0 * KB + kb) * TC_B_CHUNK, TC_B_TILE, rr, kbyte, Bs);
            tc_store(c1 + (i64)(1 * KB + kb) * TC_B_CHUNK, TC_B_TILE, rr, kbyte, B1[j]);
            tc_store(c1 + (i64)(2 * KB + kb) * TC_B_CHUNK, TC_B_TILE, rr, kbyte, F[j]);
        }
    }
}

// ---- PTX helpers ------------------------------------------------------------------------------
__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u64* bar, u32 count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(u64* bar, u32 bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* bar, u32 phase)
{
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" :: "r"(smem_u32(bar)), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, u32 bytes, u64* bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// UMMA shared-memory descriptor: canonical K-major, SWIZZLE_NONE, LBO 128 B, SBO 256 B, version 1
__device__ __forceinline__ u64 umma_desc(const void* p)
{
    const u64 addr = (u64)(smem_u32(p) >> 4) & 0x3fffull;
    return addr | ((u64)(128 >> 4) << 16) | ((u64)(256 >> 4) << 32) | (1ull << 46);
}
// instruction descriptor: kind::i8, D = s32, A = B = u8, K-major, M = 128, N = n (multiple of 16, <= 256)
__host__ __device__ constexpr u32 tc_idesc(int n)
{
    return (2u << 4) | (0u << 7) | (0u << 10) | ((u32)(n >> 3) << 17) | ((u32)(TC_BM >> 4) << 24);
}

__device__ __forceinline__ void umma_i8(u32 tmem_d, u64 adesc, u64 bdesc, u32 idesc, u32 accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
        :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory");
}
__device__ __forceinline__ void umma_commit(u64* bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tmem_ld16(u32 taddr, u32 (&v)[16])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(taddr));
}

// ---- the tensor-core ring GEMM ------------------------------------------------------------------
struct TcArgs {
    MmArgs mm;                 // shapes, keys, step, outputs, truncation
    const u8* A[2]; const u8* B[2];   // tiled limb operands per party
    int Kp[2];                 // padded K' per party
};

__global__ void __launch_bounds__(128, TC_CTAS_PER_SM) k_mm_tc(const __grid_constant__ TcArgs t)
{
    extern __shared__ __align__(1024) u8 smem_raw[];
    u8* smem = (u8*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ __align__(8) u64 full_bar[TC_STAGES], empty_bar[TC_STAGES], done_bar;
    __shared__ u32 tmem_base_sh;
    const MmArgs& a = t.mm;
    const int p = a.p0 + (int)(blockIdx.z % a.np), b = (int)(blockIdx.z / a.np);
    const int nb = blockIdx.x, mb = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int KB = t.Kp[p] / TC_BK;
    const int MB = (a.M + TC_BM - 1) / TC_BM, NB = (a.N + TC_BN - 1) / TC_BN;
    const u8* Ag = t.A[p] + (((i64)b * MB + mb) * KB) * (i64)TC_A_CHUNK;
    const u8* Bg = t.B[p] + (((i64)b * NB + nb) * KB) * (i64)TC_B_CHUNK;
    u8* sA = smem;
    u8* sB = smem + TC_STAGES * TC_A_CHUNK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < TC_STAGES; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], 1); }
        mbar_init(&done_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tmem_base_sh)), "n"(TC_TMEM_COLS) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const u32 tmem = tmem_base_sh;

    if (threadIdx.x == 0) {
        auto load = [&](int kb) {
            const int s = kb % TC_STAGES;
            mbar_expect_tx(&full_bar[s], TC_A_CHUNK + TC_B_CHUNK);
            bulk_g2s(sA + s * TC_A_CHUNK, Ag + (i64)kb * TC_A_CHUNK, TC_A_CHUNK, &full_bar[s]);
            bulk_g2s(sB + s * TC_B_CHUNK, Bg + (i64)kb * TC_B_CHUNK, TC_B_CHUNK, &full_bar[s]);
        };
        for (int kb = 0; kb < KB && kb < TC_STAGES; ++kb) load(kb);
        for (int kb = 0; kb < KB; ++kb) {
            const int s = kb % TC_STAGES;
            mbar_wait(&full_bar[s], (u32)((kb / TC_STAGES) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const u8* As_ = sA + s * TC_A_CHUNK;
            const u8* Bs_ = sB + s * TC_B_CHUNK;
            // A limb i times ALL B limbs j = 0 .. 7-i at once: the 8 B limb tiles are stacked along
            // N in the canonical layout (tile j = rows 64j .. 64j+63), and accumulators S_i .. S_7
            // are the contiguous TMEM columns [64 i, 512) -- one MMA of N = 64 (8 - i), split at
            // N = 256: 12 MMAs per K block instead of 36 (each A tile is read from shared memory
            // 1-2 times instead of 8 - i times).
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const u64 ad = umma_desc(As_ + i * TC_A_TILE);
                const u32 acc = (kb > 0 || i > 0) ? 1u : 0u;     // S_0..S_7 all first written at i = 0
                const int nj = 8 - i;
                constexpr int JMAX = 256 / TC_BN;                 // limbs per MMA (N <= 256)
                const int n1 = nj > JMAX ? JMAX : nj;
                umma_i8(tmem + (u32)(i * TC_BN), ad, umma_desc(Bs_), tc_idesc(n1 * TC_BN), acc);
                if (nj > JMAX)
                    umma_i8(tmem + (u32)((i + JMAX) * TC_BN), ad, umma_desc(Bs_ + JMAX * TC_B_TILE),
                            tc_idesc((nj - JMAX) * TC_BN), acc);
            }
            umma_commit(&empty_bar[s]);                   // frees stage s once these MMAs complete
            if (kb + TC_STAGES < KB) {
                mbar_wait(&empty_bar[s], (u32)((kb / TC_STAGES) & 1));
                load(kb + TC_STAGES);
            }
        }
        umma_commit(&done_bar);
    }
    __syncwarp();
    mbar_wait(&done_bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    // epilogue: thread <-> row m0 + 32 warp + lane, 16 columns at a time
    const int m = mb * TC_BM + warp * 32 + lane;
    const u32 trow = tmem + ((u32)(warp * 32) << 16);
    for (int c0 = 0; c0 < TC_BN; c0 += 16) {
        u64 r[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) r[q] = 0;
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            u32 v[16];
            tmem_ld16(trow + (u32)(s * TC_BN + c0), v);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int q = 0; q < 16; ++q) r[q] += (u64)v[q] << (8 * s);
        }
        if (m < a.M) {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const int n = nb * TC_BN + c0 + q;
                if (n < a.N) a.z[p][(i64)b * a.M * a.N + (i64)m * a.N + n] = mm_epilogue(a, p, b, m, n, r[q]);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "n"(TC_TMEM_COLS) : "memory");
}

}  // namespace mpc
