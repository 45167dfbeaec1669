// microbench_dfma.cu -- Philox4x32-10 with the high halves of its 32x32 products taken on the
// FP64 pipe instead of IMAD.WIDE.U32 (the fmaheavy pipe's quarter-rate instruction, the ALU roofline
// of DESIGN.md 6).
//
// The exact identity (round toward -inf, one rounding in a fused multiply-add):
//   D(n) = the double with bit pattern {hi = 0x43380000, lo = n}  (= 1.5*2^52 + n, n < 2^32)
//   fma.rm(D(n), M*2^-32, 1.5*2^52 - 1.5*2^20*M) = 1.5*2^52 + floor(n*M / 2^32)
// so the low word of the result IS mulhi(n, M), and its high word is again 0x43380000: the next
// round's XOR writes the low word in place and the pair is the next round's operand.  The low half
// of the product is a 32-bit IMAD.  Checked bit for bit against the integer Philox below.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_dfma tools/microbench_dfma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

typedef uint32_t u32;
struct Key { u32 lo, hi; };

__device__ __forceinline__ uint4 philox(Key key, u32 c0, u32 c1, u32 c2, u32 c3)
{
    u32 k0 = key.lo, k1 = key.hi;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const u32 n0 = (u32)(p1 >> 32) ^ c1 ^ k0;
        const u32 n2 = (u32)(p0 >> 32) ^ c3 ^ k1;
        c1 = (u32)p1; c3 = (u32)p0; c0 = n0; c2 = n2;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    return make_uint4(c0, c1, c2, c3);
}

#define PH_M0 0xD2511F53u
#define PH_M1 0xCD9E8D57u
// M * 2^-32 and the addend 1.5*2^52 - 1.5*2^20*M, both exact doubles
__device__ __forceinline__ double dm(u32 M) { return (double)M * 0x1p-32; }
__device__ __forceinline__ double da(u32 M) { return 6755399441055744.0 - 1572864.0 * (double)M; }
__device__ __forceinline__ u32 mulhi_df(u32 n, u32 M)
{
    const double d = __hiloint2double(0x43380000, (int)n);
    return (u32)__double2loint(__fma_rd(d, dm(M), da(M)));
}

// the product's high word as the low word of the FMA result; the result's high word is 0x43380000
__device__ __forceinline__ unsigned long long fmahi(unsigned long long D, u32 M)
{
    return (unsigned long long)__double_as_longlong(__fma_rd(__longlong_as_double((long long)D), dm(M), da(M)));
}
#define DHI 0x4338000000000000ull
// MODE 0: both highs on FP64; 1: M0 product on IMAD.WIDE, M1 on FP64; 2: alternate per round.
// c0 / c2 live as D(n) bit patterns: the XOR of the next round writes their low word in place
template <int MODE>
__device__ __forceinline__ uint4 philox_df(Key key, u32 c0, u32 c1, u32 c2, u32 c3)
{
    u32 k0 = key.lo, k1 = key.hi;
    unsigned long long D0 = DHI | c0, D2 = DHI | c2;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const bool df0 = MODE == 0 || (MODE == 2 && (r & 1));
        const bool df1 = MODE == 0 || MODE == 1 || (MODE == 2 && !(r & 1));
        unsigned long long H0, H1;
        u32 l0, l1;
        if (df0) { H0 = fmahi(D0, PH_M0); l0 = (u32)D0 * PH_M0; }
        else { const uint64_t p = (uint64_t)PH_M0 * (u32)D0; H0 = DHI | (p >> 32); l0 = (u32)p; }
        if (df1) { H1 = fmahi(D2, PH_M1); l1 = (u32)D2 * PH_M1; }
        else { const uint64_t p = (uint64_t)PH_M1 * (u32)D2; H1 = DHI | (p >> 32); l1 = (u32)p; }
        D0 = H1 ^ (unsigned long long)(c1 ^ k0);
        D2 = H0 ^ (unsigned long long)(c3 ^ k1);
        c1 = l1; c3 = l0;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    return make_uint4((u32)D0, c1, (u32)D2, c3);
}

// all four counter words vary at run time (no folded products)
template <int MODE, int ILP>
__global__ void k_ph(u32* out, Key key, int reps, u32 salt)
{
    u32 acc = 0;
    const u32 t = blockIdx.x * blockDim.x + threadIdx.x;
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int j = 0; j < ILP; ++j) {
            const u32 a = t ^ salt, b = (u32)r * 977u + salt, c = (u32)j + (acc & 1u) + salt, d = salt * 3u + (u32)r;
            const uint4 v = MODE < 0 ? philox(key, a, b, c, d) : philox_df<MODE < 0 ? 0 : MODE>(key, a, b, c, d);
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    }
    out[t] = acc;
}

// correctness: every mode against the integer Philox on n counters (including edge words)
__global__ void k_check(int* bad, Key key, int n)
{
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const u32 a = (u32)i * 2654435761u, b = (i & 7) == 0 ? 0xffffffffu : (u32)i, c = (i & 15) == 1 ? 0u : ~(u32)i * 40503u,
                  d = (i & 3) == 2 ? 0xffffffffu : (u32)i >> 3;
        const uint4 r = philox(key, a, b, c, d);
        const uint4 x = philox_df<0>(key, a, b, c, d), y = philox_df<1>(key, a, b, c, d), z = philox_df<2>(key, a, b, c, d);
        if (r.x != x.x || r.y != x.y || r.z != x.z || r.w != x.w) atomicAdd(bad, 1);
        if (r.x != y.x || r.y != y.y || r.z != y.z || r.w != y.w) atomicAdd(bad + 1, 1);
        if (r.x != z.x || r.y != z.y || r.z != z.z || r.w != z.w) atomicAdd(bad + 2, 1);
        // mulhi identity on raw words, including 0 and 2^32-1
        const u32 m = (i & 1) ? PH_M0 : PH_M1;
        const u32 w = (i & 31) == 5 ? 0xffffffffu : (i & 31) == 6 ? 0u : a ^ d;
        if (mulhi_df(w, m) != __umulhi(w, m)) atomicAdd(bad + 3, 1);
    }
}

// Random123 known-answer vector (philox4x32-10, ctr = key = 0 / all-ones / pi digits)
__global__ void k_kat(uint4* o)
{
    o[0] = philox_df<0>(Key{0, 0}, 0, 0, 0, 0);
    o[1] = philox_df<0>(Key{0xffffffffu, 0xffffffffu}, 0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
    o[2] = philox_df<0>(Key{0xa4093822u, 0x299f31d0u}, 0x243f6a88u, 0x85a308d3u, 0x13198a2eu, 0x03707344u);
}

__global__ void k_dfma_pure(double* out, double seed)
{
    double a[8];
    for (int c = 0; c < 8; ++c) a[c] = seed + threadIdx.x + c;
    for (int it = 0; it < 4096; ++it) {
#pragma unroll
        for (int c = 0; c < 8; ++c) a[c] = __fma_rd(a[c], 0.999999, 1e-3);
    }
    double s = 0;
    for (int c = 0; c < 8; ++c) s += a[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
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
    u32* out;
    cudaMalloc(&out, 64 << 20);
    int* bad;
    cudaMalloc(&bad, 16);
    cudaMemset(bad, 0, 16);
    k_check<<<sms * 8, 256>>>(bad, Key{0x12345678u, 0x9abcdef0u}, 1 << 24);
    int hb[4];
    cudaMemcpy(hb, bad, 16, cudaMemcpyDeviceToHost);
    uint4* kat;
    cudaMalloc(&kat, 3 * sizeof(uint4));
    k_kat<<<1, 1>>>(kat);
    uint4 hk[3];
    cudaMemcpy(hk, kat, sizeof hk, cudaMemcpyDeviceToHost);
    const bool kat_ok = hk[0].x == 0x6627e8d5u && hk[0].y == 0xe169c58du && hk[0].z == 0xbc57ac4cu && hk[0].w == 0x9b00dbd8u &&
                        hk[1].x == 0x408f276du && hk[1].y == 0x41c83b0eu && hk[1].z == 0xa20bc7c6u && hk[1].w == 0x6d5451fdu &&
                        hk[2].x == 0xd16cfe09u && hk[2].y == 0x94fdccebu && hk[2].z == 0x5001e420u && hk[2].w == 0x24126ea1u;
    printf("{\"sms\": %d, \"clock_khz\": %d, \"check_counters\": %d, \"mismatch_df_both\": %d, \"mismatch_df_mix\": %d, "
           "\"mismatch_df_alt\": %d, \"mismatch_mulhi\": %d, \"kat_random123_ok\": %s",
           sms, clk, 1 << 24, hb[0], hb[1], hb[2], hb[3], kat_ok ? "true" : "false");
    {
        const int blocks = sms * 8, threads = 256;
        float ms = timeit([&] { k_dfma_pure<<<blocks, threads>>>((double*)out, 1.0); });
        printf(", \"dfma_warp_instr_per_clk_per_smsp\": %.4f",
               (double)blocks * threads / 32 * 4096 * 8 / (ms * 1e-3) / (sms * 4.0) / (clk * 1e3));
    }
    const int reps = 256;
    for (int tpb : {256, 512}) {
        const int nb = sms * (2048 / tpb);
        const double n = (double)nb * tpb;
        float ms;
#define RUN(MODE, ILP, NAME) \
        ms = timeit([&] { k_ph<MODE, ILP><<<nb, tpb>>>(out, Key{1, 2}, reps / ILP, 5u); }); \
        printf(", \"%s_ilp%d_%dthr_gblk_s\": %.1f", NAME, ILP, tpb * (2048 / tpb), n * reps / (ms * 1e-3) / 1e9);
        RUN(-1, 1, "int") RUN(-1, 2, "int") RUN(-1, 4, "int")
        RUN(0, 1, "df") RUN(0, 2, "df") RUN(0, 4, "df")
        RUN(1, 1, "mix") RUN(1, 2, "mix") RUN(1, 4, "mix")
        RUN(2, 2, "alt") RUN(2, 4, "alt")
    }
    {
        const int nb = sms * 2, tpb = 256;   // 16 warps / SM: the row kernels' occupancy
        const double n = (double)nb * tpb;
        float ms;
        RUN(-1, 2, "int_16w") RUN(0, 2, "df_16w") RUN(1, 2, "mix_16w") RUN(-1, 4, "int_16w") RUN(0, 4, "df_16w") RUN(1, 4, "mix_16w")
    }
    printf("}\n");
    return 0;
}
