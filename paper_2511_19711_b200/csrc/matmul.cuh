// matmul.cuh -- Beaver matrix multiplication over Z_2^64.
//
// Z = X Y for `batch` products, with a matrix Beaver triple generated on device:
//   A_p = half (uA&1) of PRG(K_p, uA>>1, s, 8), B_p likewise at slot 9, C0 at slot 10 (K_0),
//   C1 = (A0+A1)(B0+B1) - C0, E = open(X - A), F = open(Y - B),
//   Z0 = C0 + E B0 + A0 F + E F = C0 + E (B0 + F) + A0 F
//   Z1 = C1 + E B1 + A1 F       = (A0+A1)(B0+B1) - C0 + E B1 + A1 F
// Stage 1 (k_pairs + MmMaskBody): masks, openings (one exchange per warp in PAIR mode) and the
// operand planes the parties' GEMMs read.  Stage 2: the ring GEMMs (sum of up to three
// products per party) with C0 from the PRG and the truncation in the epilogue.
#pragma once
#include "kernels.cuh"

namespace mpc {

// Operand planes of one part (A part: n = batch*M*K units; B part: batch*K*N):
//   A part: [0] E = open(X - A), [1] A0, [2] A1, [3] A0 + A1
//   B part: [0] F = open(Y - B), [1] B0 + F, [2] B1, [3] B0 + B1
// In PAIR mode each party writes the planes its GEMM reads (party 0: E, A0 / F, B0+F; party 1
// simulating the dealer: E, A1, A0+A1 / F, B1, B0+B1 -- with the dealer's stream only E, A1 / F, B1
// are used: party 1's GEMM reads the dealer's C1).
struct MmMaskBody {
    u32 s, slot; SP x; i64 n; u64* out; int bpart;
    template <int V, class P>
    __device__ void run(P& pr, const u64 (&u)[V], const i64 (&i0)[V], const bool (&ok)[V]) const {
        using S = typename P::S;
        const int p = pr.party();
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const bool va = ok[v] && i0[v] >= 0, vb = ok[v] && i0[v] + 1 < n;
            const uint4 R0 = pr.k0ok() ? prg(pr.Kp->k0, u[v] >> 1, s, slot) : make_uint4(0, 0, 0, 0);
            uint4 R1 = make_uint4(0, 0, 0, 0);
            if (p != 0) R1 = prg(pr.Kp->k1, u[v] >> 1, s, slot);
            const u64 r0a = w64(R0.x, R0.y), r0b = w64(R0.z, R0.w), r1a = w64(R1.x, R1.y), r1b = w64(R1.z, R1.w);
            const S xa = va ? pr.ld(x, i0[v]) : pr.zero(), xb = vb ? pr.ld(x, i0[v] + 1) : pr.zero();
            u64 ea, eb;
            pr.open2(pr.mask2(xa, r0a, r1a), pr.mask2(xb, r0b, r1b), ea, eb);
            const u64 oa[4] = {ea, bpart ? r0a + ea : r0a, r1a, r0a + r1a};
            const u64 ob[4] = {eb, bpart ? r0b + eb : r0b, r1b, r0b + r1b};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const bool mine = p < 0 || k == 0 || (p == 0 ? k == 1 : k >= 2);
                if (!mine) continue;
                if (va) out[(i64)k * n + i0[v]] = oa[k];
                if (vb) out[(i64)k * n + i0[v] + 1] = ob[k];
            }
        }
    }
};

struct MmTerm { const u64* a; const u64* b; };      // a: [batch][M][K], b: [batch][K][N]
struct MmArgs {
    Keys K; u32 s; int M, Kd, N, batch; u64 goff; int tb;
    int p0, np;                                      // parties computed by this launch
    MmTerm t[2][3]; int nt[2];
    u64* z[2];
    const u64* cin[2];      // party p's C term read from memory (party 1: the dealer's C1)
};

// C0 epilogue + truncation for output element (b, m, n) of party p
__device__ __forceinline__ u64 mm_epilogue(const MmArgs& a, int p, int b, int m, int n, u64 acc)
{
    u64 v;
    if (a.cin[p]) {
        v = acc + a.cin[p][(i64)b * a.M * a.N + (i64)m * a.N + n];
    } else {
        const u64 uC = (a.goff + (u64)b) * (u64)a.M * (u64)a.N + (u64)m * (u64)a.N + (u64)n;
        const uint4 C = prg(a.K.k0, uC >> 1, a.s, 10);
        const u64 c0 = (uC & 1) ? w64(C.z, C.w) : w64(C.x, C.y);
        v = p == 0 ? acc + c0 : acc - c0;
    }
    return a.tb ? shr(v, a.tb) : v;
}

// SIMT ring GEMM (IMAD): 64 x 64 output tile per CTA, 4 x 4 per thread, K step 16.
// blockIdx.z = b * np + (p - p0).
__global__ void __launch_bounds__(256) k_mm_simt(const __grid_constant__ MmArgs a)
{
    __shared__ u64 sA[16][64 + 1], sB[16][64];
    const int p = a.p0 + (int)(blockIdx.z % a.np), b = (int)(blockIdx.z / a.np);
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
    const i64 MK = (i64)a.M * a.Kd, KN = (i64)a.Kd * a.N;
    u64 acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0;
    for (int t = 0; t < a.nt[p]; ++t) {
        const u64* A_ = a.t[p][t].a + (i64)b * MK;
        const u64* B_ = a.t[p][t].b + (i64)b * KN;
        for (int k0 = 0; k0 < a.Kd; k0 += 16) {
            for (int l = threadIdx.x; l < 1024; l += 256) {
                const int r = l >> 4, c = l & 15, m = m0 + r, k = k0 + c;
                sA[c][r] = (m < a.M && k < a.Kd) ? A_[(i64)m * a.Kd + k] : 0ull;
            }
            for (int l = threadIdx.x; l < 1024; l += 256) {
                const int r = l >> 6, c = l & 63, k = k0 + r, n = n0 + c;
                sB[r][c] = (k < a.Kd && n < a.N) ? B_[(i64)k * a.N + n] : 0ull;
            }
            __syncthreads();
#pragma unroll
            for (int kk = 0; kk < 16; ++kk) {
                u64 ra[4], rb[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) { ra[i] = sA[kk][ty + 16 * i]; rb[i] = sB[kk][tx + 16 * i]; }
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] += ra[i] * rb[j];
            }
            __syncthreads();
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int m = m0 + ty + 16 * i, n = n0 + tx + 16 * j;
            if (m < a.M && n < a.N) a.z[p][(i64)b * a.M * a.N + (i64)m * a.N + n] = mm_epilogue(a, p, b, m, n, acc[i][j]);
        }
}

}  // namespace mpc
