// microbench.cu -- integer-pipe microbenchmarks on sm_100a that pin the ALU roofline
// of DESIGN.md 6: IMAD.WIDE.U32 vs IMAD vs IMAD.HI vs LOP3 throughput, and the
// Philox4x32-10 block rate at several ILP / occupancy points.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
#define CHAINS 8

__global__ void k_imad_wide(uint32_t* out, uint32_t seed)
{
    uint32_t a[CHAINS], b[CHAINS];
    for (int c = 0; c < CHAINS; ++c) { a[c] = seed + threadIdx.x * 7 + c; b[c] = a[c] ^ 0x1234567u; }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) {
            uint64_t p = (uint64_t)a[c] * 0xD2511F53u;
            a[c] = (uint32_t)(p >> 32) + b[c];   // keeps the chain dependent (IMAD.WIDE consumes b)
            b[c] = (uint32_t)p;
        }
    }
    uint32_t s = 0;
    for (int c = 0; c < CHAINS; ++c) s ^= a[c] ^ b[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_imad_lo(uint32_t* out, uint32_t seed)
{
    uint32_t a[CHAINS];
    for (int c = 0; c < CHAINS; ++c) a[c] = seed + threadIdx.x * 7 + c;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) a[c] = a[c] * 0xD2511F53u + c;
    }
    uint32_t s = 0;
    for (int c = 0; c < CHAINS; ++c) s ^= a[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_imad_hi(uint32_t* out, uint32_t seed)
{
    uint32_t a[CHAINS];
    for (int c = 0; c < CHAINS; ++c) a[c] = seed + threadIdx.x * 7 + c;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) a[c] = __umulhi(a[c], 0xD2511F53u) + a[c];
    }
    uint32_t s = 0;
    for (int c = 0; c < CHAINS; ++c) s ^= a[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_lop3(uint32_t* out, uint32_t seed)
{
    uint32_t a[CHAINS], b = seed * 3 + 1, d = seed * 5 + 7;
    for (int c = 0; c < CHAINS; ++c) a[c] = seed + threadIdx.x * 7 + c;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) a[c] = (a[c] ^ b ^ (d + it));
    }
    uint32_t s = 0;
    for (int c = 0; c < CHAINS; ++c) s ^= a[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}


// ---- pure-pipe kernels (one SASS instruction per chained step; checked with cuobjdump -sass) ----
// IMAD.WIDE.U32 alone: p = (u64)hi32(p) * M (one IMAD.WIDE.U32 per step, 8 independent chains)
__global__ void k_imadw_pure(uint32_t* out, uint32_t seed)
{
    uint64_t p[CHAINS];
    for (int c = 0; c < CHAINS; ++c) p[c] = ((uint64_t)((seed + threadIdx.x) * (c + 3)) << 32) | (uint64_t)(c * 977u + threadIdx.x);
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c)
            asm volatile("{.reg .u32 lo, hi; mov.b64 {lo, hi}, %0; mul.wide.u32 %0, hi, 0xD2511F53;}" : "+l"(p[c]));
    }
    uint32_t s = 0;
    for (int c = 0; c < CHAINS; ++c) s ^= (uint32_t)p[c] ^ (uint32_t)(p[c] >> 32);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// LOP3 alone: a = a ^ b ^ d with loop-invariant b, d
__global__ void k_lop3_pure(uint32_t* out, uint32_t seed)
{
    uint32_t a[CHAINS], b = seed * 3 + 1 + threadIdx.x, d = seed * 5 + 7;
    for (int c = 0; c < CHAINS; ++c) a[c] = seed + threadIdx.x * 7 + c;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c)
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[c]) : "r"(b), "r"(d));
    }
    uint32_t s = 0;
    for (int c = 0; c < CHAINS; ++c) s ^= a[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// the Philox round's instruction pair without the key bumps: IMAD.WIDE + LOP3 per step
__global__ void k_imadw_lop3(uint32_t* out, uint32_t seed)
{
    uint64_t p[CHAINS];
    uint32_t x[CHAINS];
    const uint32_t k = seed * 0x9E3779B9u + threadIdx.x;
    for (int c = 0; c < CHAINS; ++c) { p[c] = (uint64_t)(seed + threadIdx.x + c) << 7; x[c] = c; }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) {
            asm volatile("{.reg .u32 lo, hi, plo, phi; mov.b64 {plo, phi}, %1; mul.wide.u32 %1, %0, 0xD2511F53;"
                         " mov.b64 {lo, hi}, %1; lop3.b32 %0, hi, plo, %2, 0x96;}" : "+r"(x[c]), "+l"(p[c]) : "r"(k));
        }
    }
    uint32_t s = 0;
    for (int c = 0; c < CHAINS; ++c) s ^= x[c] ^ (uint32_t)p[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

struct Key { uint32_t lo, hi; };
__device__ __forceinline__ uint4 philox(Key key, uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3)
{
    uint32_t k0 = key.lo, k1 = key.hi;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        c1 = (uint32_t)p1; c3 = (uint32_t)p0; c0 = n0; c2 = n2;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    return make_uint4(c0, c1, c2, c3);
}

// same rounds with the 64-bit product split into IMAD.HI + IMAD (lo) -- tests whether the
// low half can leave the fmaheavy pipe
__device__ __forceinline__ uint4 philox_split(Key key, uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3)
{
    uint32_t k0 = key.lo, k1 = key.hi;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t h0, l0, h1, l1;
        asm volatile("mul.hi.u32 %0, %1, 0xD2511F53;" : "=r"(h0) : "r"(c0));
        asm volatile("mad.lo.u32 %0, %1, 0xD2511F52, %1;" : "=r"(l0) : "r"(c0));
        asm volatile("mul.hi.u32 %0, %1, 0xCD9E8D57;" : "=r"(h1) : "r"(c2));
        asm volatile("mad.lo.u32 %0, %1, 0xCD9E8D56, %1;" : "=r"(l1) : "r"(c2));
        const uint32_t n0 = h1 ^ c1 ^ k0;
        const uint32_t n2 = h0 ^ c3 ^ k1;
        c1 = l1; c3 = l0; c0 = n0; c2 = n2;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    return make_uint4(c0, c1, c2, c3);
}

template <int ILP>
__global__ void k_philox_split(uint32_t* out, Key key, int reps)
{
    uint32_t acc = 0;
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int j = 0; j < ILP; ++j) {
            const uint4 v = philox_split(key, t, (uint32_t)r, (uint32_t)j, 7u);
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    }
    out[t] = acc;
}

template <int ILP>
__global__ void k_philox(uint32_t* out, Key key, int reps)
{
    uint32_t acc = 0;
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int j = 0; j < ILP; ++j) {
            const uint4 v = philox(key, t, (uint32_t)r, (uint32_t)j, 7u);
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    }
    out[t] = acc;
}

template <class F>
static float timeit(F launch)
{
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
}

int main()
{
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    uint32_t* out;
    cudaMalloc(&out, 64 << 20);
    const int blocks = sms * 8, threads = 256;
    const double nthr = (double)blocks * threads;
    printf("{\"sms\": %d, \"clock_khz\": %d", sms, clk);
    float ms = timeit([&] { k_imad_wide<<<blocks, threads>>>(out, 1); });
    printf(", \"imad_wide_per_clk_per_sm\": %.2f", nthr * ITERS * CHAINS / (ms * 1e-3) / sms / (clk * 1e3));
    ms = timeit([&] { k_imad_lo<<<blocks, threads>>>(out, 1); });
    printf(", \"imad_per_clk_per_sm\": %.2f", nthr * ITERS * CHAINS / (ms * 1e-3) / sms / (clk * 1e3));
    ms = timeit([&] { k_imad_hi<<<blocks, threads>>>(out, 1); });
    printf(", \"imad_hi_plus_iadd_per_clk_per_sm\": %.2f", nthr * ITERS * CHAINS / (ms * 1e-3) / sms / (clk * 1e3));
    ms = timeit([&] { k_lop3<<<blocks, threads>>>(out, 1); });
    printf(", \"lop3_plus_iadd_per_clk_per_sm\": %.2f", nthr * ITERS * CHAINS / (ms * 1e-3) / sms / (clk * 1e3));
    ms = timeit([&] { k_imadw_pure<<<blocks, threads>>>(out, 1); });
    printf(", \"imadw_pure_warp_instr_per_clk_per_smsp\": %.4f", nthr / 32 * ITERS * CHAINS / (ms * 1e-3) / (sms * 4.0) / (clk * 1e3));
    ms = timeit([&] { k_lop3_pure<<<blocks, threads>>>(out, 1); });
    printf(", \"lop3_pure_warp_instr_per_clk_per_smsp\": %.4f", nthr / 32 * ITERS * CHAINS / (ms * 1e-3) / (sms * 4.0) / (clk * 1e3));
    ms = timeit([&] { k_imadw_lop3<<<blocks, threads>>>(out, 1); });
    printf(", \"imadw_plus_lop3_pairs_per_clk_per_smsp\": %.4f", nthr / 32 * ITERS * CHAINS / (ms * 1e-3) / (sms * 4.0) / (clk * 1e3));
    const int reps = 256;
    for (int tpb : {128, 256, 512, 1024}) {
        const int nb = sms * (2048 / tpb);
        const double n = (double)nb * tpb;
        ms = timeit([&] { k_philox<1><<<nb, tpb>>>(out, Key{1, 2}, reps); });
        printf(", \"philox_ilp1_%dthr_gblk_s\": %.1f", tpb * (2048 / tpb), n * reps / (ms * 1e-3) / 1e9);
        ms = timeit([&] { k_philox<2><<<nb, tpb>>>(out, Key{1, 2}, reps / 2); });
        printf(", \"philox_ilp2_%dthr_gblk_s\": %.1f", tpb * (2048 / tpb), n * reps / (ms * 1e-3) / 1e9);
    }
    {
        const int nb = sms * 2, tpb = 256;   // 16 warps / SM
        const double n = (double)nb * tpb;
        ms = timeit([&] { k_philox<1><<<nb, tpb>>>(out, Key{1, 2}, reps); });
        printf(", \"philox_ilp1_512thr_per_sm_gblk_s\": %.1f", n * reps / (ms * 1e-3) / 1e9);
        ms = timeit([&] { k_philox<4><<<nb, tpb>>>(out, Key{1, 2}, reps / 4); });
        printf(", \"philox_ilp4_512thr_per_sm_gblk_s\": %.1f", n * reps / (ms * 1e-3) / 1e9);
    }
    for (int tpb : {256, 512}) {
        const int nb = sms * (2048 / tpb);
        const double n = (double)nb * tpb;
        ms = timeit([&] { k_philox_split<2><<<nb, tpb>>>(out, Key{1, 2}, reps / 2); });
        printf(", \"philox_split_ilp2_%dthr_gblk_s\": %.1f", tpb * (2048 / tpb), n * reps / (ms * 1e-3) / 1e9);
        ms = timeit([&] { k_philox_split<4><<<nb, tpb>>>(out, Key{1, 2}, reps / 4); });
        printf(", \"philox_split_ilp4_%dthr_gblk_s\": %.1f", tpb * (2048 / tpb), n * reps / (ms * 1e-3) / 1e9);
        ms = timeit([&] { k_philox<4><<<nb, tpb>>>(out, Key{1, 2}, reps / 4); });
        printf(", \"philox_ilp4_%dthr_gblk_s\": %.1f", tpb * (2048 / tpb), n * reps / (ms * 1e-3) / 1e9);
    }
    printf("}\n");
    return 0;
}
