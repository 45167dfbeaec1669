// rows_both.cuh -- fused row operators (MPC_MODE_BOTH): one CTA owns a tile of 32
// consecutive rows (32-aligned in global row index) and runs the whole schedule
// of DESIGN.md 2.5 on it -- every max-tree level (whose LTZ groups of row*h+i
// stay inside the 32-row tile), exp, row sums, the per-row Newton-Raphson and the
// final broadcast product -- with the intermediates in shared memory (or, for
// long rows, in a per-CTA global scratch tile that stays L2-resident).
// Persistent grid: CTAs loop over tiles.
#pragma once
#include "sched_both.cuh"

namespace mpc {

struct RowPtr2 { const u64* p0; const u64* p1; };
struct RowOut2 { u64* p0; u64* p1; };

constexpr int ROW_TILE = 32;

// ---- MAX_row tree over a 32-row tile (R22) --------------------------------
// in: row-major, row stride ldi (tile-local row 0 = global row g0).  Levels write into
// the ping-pong buffers A/B (stride H = ceil(cols/2)); the last level writes mx[rr].
// R = valid rows in the tile.  Steps s + 2*lv, s + 2*lv + 1.
template <bool WIDE>
__device__ __forceinline__ void tile_max(const Keys& K, u32 s, int w, RowPtr2 in, i64 ldi, i64 cols,
                                         int R, u64 g0, u64* A0, u64* A1, u64* B0, u64* B1, i64 H,
                                         u64* mx0, u64* mx1)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
    i64 m = cols;
    int lv = 0;
    const u64* i0 = in.p0; const u64* i1 = in.p1;
    i64 li = ldi;
    while (m > 1) {
        const i64 h = m / 2, mn = h + (m & 1);
        u64* o0; u64* o1; i64 lo;
        if (mn == 1) { o0 = mx0; o1 = mx1; lo = 1; }
        else if (lv & 1) { o0 = B0; o1 = B1; lo = H; }
        else { o0 = A0; o1 = A1; lo = H; }
        const u32 sl = s + 2u * (u32)lv;
        const u64 ubase = g0 * (u64)h;                 // multiple of 32 (g0 is)
        const FastDiv dh = make_fastdiv((u32)h);
        for (i64 g = warp; g < h; g += NW) {            // 32*h units = h groups
            const i64 v = g * 32 + lane;
            const bool valid = v < (i64)R * h;
            i64 rr = 0, i = 0;
            Sh d = {0, 0}, y = {0, 0};
            if (valid) {
                rr = fdiv((u32)v, dh); i = v - rr * h;
                const Sh a = {i0[rr * li + i], i1[rr * li + i]};
                y = Sh{i0[rr * li + i + h], i1[rr * li + i + h]};
                d = sh_sub(a, y);
            }
            const u64 q = (ubase >> 5) + (u64)g;
            const Sh c = sh_not(ltz<WIDE>(K, q, sl, w, d, lane));
            const Sh sel = sh_add(y, bm(K, ubase + (u64)v, sl + 1, d, c));
            if (valid) {
                o0[rr * lo + i] = sel.s0; o1[rr * lo + i] = sel.s1;
                if ((m & 1) && i == h - 1) { o0[rr * lo + h] = i0[rr * li + m - 1]; o1[rr * lo + h] = i1[rr * li + m - 1]; }
            }
        }
        __syncthreads();
        i0 = o0; i1 = o1; li = lo;
        m = mn;
        ++lv;
    }
    if (cols == 1) {
        for (int rr = threadIdx.x; rr < R; rr += blockDim.x) { mx0[rr] = in.p0[rr * ldi]; mx1[rr] = in.p1[rr * ldi]; }
        __syncthreads();
    }
}

// per-row Newton-Raphson over the tile's rows: warp 0, lane <-> row (LTZ group = tile)
template <int KIND, bool WIDE>
__device__ __forceinline__ void tile_nr(const Keys& K, u32 s, const NrK& p, int R, u64 g0,
                                        const u64* x0, const u64* x1, u64* y0, u64* y1)
{
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        const bool valid = lane < R;
        Sh x = {0, 0};
        if (valid) x = Sh{x0[lane], x1[lane]};
        Sh y;
        if (KIND == 0) y = recip_group<WIDE>(K, g0 + lane, g0 >> 5, s, p, x, lane);
        else y = rsqrt_group<WIDE>(K, g0 + lane, g0 >> 5, s, p, x, lane);
        if (valid) { y0[lane] = y.s0; y1[lane] = y.s1; }
    }
    __syncthreads();
}

// warp per row: S[rr] = sum_j E[rr][j]
__device__ __forceinline__ void tile_rowsum(const u64* e0, const u64* e1, i64 ld, i64 cols, int R, u64* S0, u64* S1)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
    for (int rr = warp; rr < R; rr += NW) {
        u64 a = 0, b = 0;
        for (i64 j = lane; j < cols; j += 32) { a += e0[rr * ld + j]; b += e1[rr * ld + j]; }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) { a += __shfl_xor_sync(FULL, a, o); b += __shfl_xor_sync(FULL, b, o); }
        if (lane == 0) { S0[rr] = a; S1[rr] = b; }
    }
    __syncthreads();
}

struct SoftmaxArgs {
    Keys K;
    u32 s_max, s_exp, s_rec, s_mul;
    int w;
    ExpK ek;
    NrK rk;
    RowPtr2 x;
    RowOut2 z;
    i64 rows, cols;
    u64 row_off;
    u64* gscratch;          // per-CTA work tiles when they do not fit in shared memory
    i64 work_u64;           // u64 words of one work tile
    int use_smem;
};

// work tile layout (u64 words), H = ceil(cols/2):
//   A0 A1 B0 B1 : 4 x 32H  (max ping-pong; reused as E0 E1 : 2 x 32 cols <= 4 x 32H)
//   MX0 MX1 S0 S1 R0 R1 : 6 x 32
__host__ __device__ inline i64 softmax_work_u64(i64 cols) { return 4 * 32 * ((cols + 1) / 2) + 6 * 32; }

template <bool WIDE>
__global__ void __launch_bounds__(256, 3) k_softmax_fused(SoftmaxArgs a)
{
    extern __shared__ __align__(16) u64 smem[];
    u64* W = a.use_smem ? smem : a.gscratch + (i64)blockIdx.x * a.work_u64;
    const i64 C = a.cols, H = (C + 1) / 2;
    u64 *A0 = W, *A1 = W + 32 * H, *B0 = W + 64 * H, *B1 = W + 96 * H;
    u64 *E0 = W, *E1 = W + 32 * C;
    u64 *MX0 = W + 128 * H, *MX1 = MX0 + 32, *S0 = MX0 + 64, *S1 = MX0 + 96, *R0 = MX0 + 128, *R1 = MX0 + 160;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
    const i64 ntiles = (a.rows + 31) / 32;
    const FastDiv dC = make_fastdiv((u32)C);
    for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const i64 r0 = tile * 32;
        const int R = (int)min((i64)32, a.rows - r0);
        const u64 g0 = a.row_off + (u64)r0;                       // global row of the tile
        const RowPtr2 xt = {a.x.p0 + r0 * C, a.x.p1 + r0 * C};
        // 1. m = MAX_row(x)
        tile_max<WIDE>(a.K, a.s_max, a.w, xt, C, C, R, g0, A0, A1, B0, B1, H, MX0, MX1);
        // 2-3. e = EXP(x - m), element units g0*C + e
        const i64 ne = (i64)R * C;
        const u64 ub = g0 * (u64)C;
        if (a.ek.clamp) {
            for (i64 g = warp; g < (ne + 31) / 32; g += NW) {
                const i64 e = g * 32 + lane;
                const bool valid = e < ne;
                Sh d = {0, 0};
                if (valid) { const i64 rr = fdiv((u32)e, dC); d = Sh{xt.p0[e] - MX0[rr], xt.p1[e] - MX1[rr]}; }
                const Sh y = exp_group<WIDE>(a.K, ub + e, (ub >> 5) + g, a.s_exp, a.ek, d, lane);
                if (valid) { E0[e] = y.s0; E1[e] = y.s1; }
            }
        } else {
            for (i64 p = threadIdx.x; p < (ne + 1) / 2; p += blockDim.x) {
                const i64 e = 2 * p;
                const i64 ra = fdiv((u32)e, dC), rb = fdiv((u32)(e + 1), dC);
                Sh da = {xt.p0[e] - MX0[ra], xt.p1[e] - MX1[ra]}, db = {0, 0};
                const bool vb = e + 1 < ne;
                if (vb) db = Sh{xt.p0[e + 1] - MX0[rb], xt.p1[e + 1] - MX1[rb]};
                exp_pair(a.K, ub + e, a.s_exp, a.ek, da, db);
                E0[e] = da.s0; E1[e] = da.s1;
                if (vb) { E0[e + 1] = db.s0; E1[e + 1] = db.s1; }
            }
        }
        __syncthreads();
        // 4. S = rowsum(e)
        tile_rowsum(E0, E1, C, C, R, S0, S1);
        // 5. r = RECIP(S), row units
        tile_nr<0, WIDE>(a.K, a.s_rec, a.rk, R, g0, S0, S1, R0, R1);
        // 6. out = MT(e, r), element units
        for (i64 p = threadIdx.x; p < (ne + 1) / 2; p += blockDim.x) {
            const i64 e = 2 * p;
            const bool vb = e + 1 < ne;
            const i64 ra = fdiv((u32)e, dC), rb = fdiv((u32)(e + 1), dC);
            const Sh ea = {E0[e], E1[e]}, eb = vb ? Sh{E0[e + 1], E1[e + 1]} : Sh{0, 0};
            const Sh xa = {R0[ra], R1[ra]}, xb = vb ? Sh{R0[rb], R1[rb]} : Sh{0, 0};
            Sh za, zb;
            bm2(a.K, ub + e, a.s_mul, ea, xa, eb, xb, za, zb);
            a.z.p0[r0 * C + e] = shr(za.s0, FRAC); a.z.p1[r0 * C + e] = shr(za.s1, FRAC);
            if (vb) { a.z.p0[r0 * C + e + 1] = shr(zb.s0, FRAC); a.z.p1[r0 * C + e + 1] = shr(zb.s1, FRAC); }
        }
        __syncthreads();
    }
}

struct MaxArgs {
    Keys K; u32 s; int w; RowPtr2 x; RowOut2 z; i64 rows, cols; u64 row_off;
    u64* gscratch; i64 work_u64; int use_smem;
};
__host__ __device__ inline i64 max_work_u64(i64 cols) { return 4 * 32 * ((cols + 1) / 2) + 2 * 32; }

template <bool WIDE>
__global__ void __launch_bounds__(256, 3) k_max_fused(MaxArgs a)
{
    extern __shared__ __align__(16) u64 smem[];
    u64* W = a.use_smem ? smem : a.gscratch + (i64)blockIdx.x * a.work_u64;
    const i64 C = a.cols, H = (C + 1) / 2;
    u64 *A0 = W, *A1 = W + 32 * H, *B0 = W + 64 * H, *B1 = W + 96 * H, *MX0 = W + 128 * H, *MX1 = MX0 + 32;
    const i64 ntiles = (a.rows + 31) / 32;
    for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const i64 r0 = tile * 32;
        const int R = (int)min((i64)32, a.rows - r0);
        tile_max<WIDE>(a.K, a.s, a.w, RowPtr2{a.x.p0 + r0 * C, a.x.p1 + r0 * C}, C, C, R, a.row_off + (u64)r0,
                 A0, A1, B0, B1, H, MX0, MX1);
        for (int rr = threadIdx.x; rr < R; rr += blockDim.x) { a.z.p0[r0 + rr] = MX0[rr]; a.z.p1[r0 + rr] = MX1[rr]; }
        __syncthreads();
    }
}

struct LnArgs {
    Keys K; u32 s_sq, s_rs, s_mul; NrK rk; RowPtr2 x; RowOut2 z; i64 rows, cols; u64 row_off;
    int mean_mode; u64 e_invd, e_eps;
};

__device__ __forceinline__ u64 floordiv_s(u64 a, i64 d)
{
    const i64 x = (i64)a;
    i64 q = x / d;
    if ((x % d) != 0 && x < 0) --q;
    return (u64)q;
}

// LAYERNORM: mu, c = x - mu, v = mean(MT(c,c)) + eps, r = RSQRT(v), out = MT(c, r)
template <bool WIDE>
__global__ void __launch_bounds__(256, 3) k_ln_fused(LnArgs a)
{
    __shared__ u64 MU0[32], MU1[32], V0[32], V1[32], RS0[32], RS1[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
    const i64 C = a.cols;
    const i64 ntiles = (a.rows + 31) / 32;
    const FastDiv dC = make_fastdiv((u32)C);
    for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const i64 r0 = tile * 32;
        const int R = (int)min((i64)32, a.rows - r0);
        const u64 g0 = a.row_off + (u64)r0;
        const u64* x0 = a.x.p0 + r0 * C;
        const u64* x1 = a.x.p1 + r0 * C;
        for (int rr = warp; rr < R; rr += NW) {
            u64 s0 = 0, s1 = 0;
            for (i64 j = lane; j < C; j += 32) { s0 += x0[rr * C + j]; s1 += x1[rr * C + j]; }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) { s0 += __shfl_xor_sync(FULL, s0, o); s1 += __shfl_xor_sync(FULL, s1, o); }
            Sh mu = {s0, s1};
            mu = a.mean_mode == 0 ? sh_mulf(mu, a.e_invd) : Sh{floordiv_s(mu.s0, C), floordiv_s(mu.s1, C)};
            // q = MT(c, c) over the row, element units; lanes take element pairs (2j, 2j+1)
            u64 q0 = 0, q1 = 0;
            const u64 ub = (g0 + (u64)rr) * (u64)C;
            for (i64 j = 2 * lane - (i64)(ub & 1); j < C; j += 64) {
                const bool va = j >= 0, vb = j + 1 < C;
                Sh ca = {0, 0}, cb = {0, 0};
                if (va) ca = sh_sub(Sh{x0[rr * C + j], x1[rr * C + j]}, mu);
                if (vb) cb = sh_sub(Sh{x0[rr * C + j + 1], x1[rr * C + j + 1]}, mu);
                Sh za, zb;
                bm2(a.K, ub + (u64)j, a.s_sq, ca, ca, cb, cb, za, zb);
                if (va) { q0 += shr(za.s0, FRAC); q1 += shr(za.s1, FRAC); }
                if (vb) { q0 += shr(zb.s0, FRAC); q1 += shr(zb.s1, FRAC); }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) { q0 += __shfl_xor_sync(FULL, q0, o); q1 += __shfl_xor_sync(FULL, q1, o); }
            Sh v = {q0, q1};
            v = a.mean_mode == 0 ? sh_mulf(v, a.e_invd) : Sh{floordiv_s(v.s0, C), floordiv_s(v.s1, C)};
            v = sh_addp(v, a.e_eps);
            if (lane == 0) { MU0[rr] = mu.s0; MU1[rr] = mu.s1; V0[rr] = v.s0; V1[rr] = v.s1; }
        }
        __syncthreads();
        tile_nr<1, WIDE>(a.K, a.s_rs, a.rk, R, g0, V0, V1, RS0, RS1);
        const i64 ne = (i64)R * C;
        const u64 ub = g0 * (u64)C;            // even: g0 is a multiple of 32
        for (i64 p = threadIdx.x; p < (ne + 1) / 2; p += blockDim.x) {
            const i64 e = 2 * p;
            const bool vb = e + 1 < ne;
            const i64 ra = fdiv((u32)e, dC), rb = fdiv((u32)(e + 1), dC);
            const Sh ca = sh_sub(Sh{x0[e], x1[e]}, Sh{MU0[ra], MU1[ra]});
            const Sh cb = vb ? sh_sub(Sh{x0[e + 1], x1[e + 1]}, Sh{MU0[rb], MU1[rb]}) : Sh{0, 0};
            const Sh ra_ = {RS0[ra], RS1[ra]}, rb_ = vb ? Sh{RS0[rb], RS1[rb]} : Sh{0, 0};
            Sh za, zb;
            bm2(a.K, ub + e, a.s_mul, ca, ra_, cb, rb_, za, zb);
            a.z.p0[r0 * C + e] = shr(za.s0, FRAC); a.z.p1[r0 * C + e] = shr(za.s1, FRAC);
            if (vb) { a.z.p0[r0 * C + e + 1] = shr(zb.s0, FRAC); a.z.p1[r0 * C + e + 1] = shr(zb.s1, FRAC); }
        }
        __syncthreads();
    }
}

}  // namespace mpc
