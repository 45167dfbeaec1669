// PCIe copy microbenchmark for the host-buffer path: DMA copies (cudaMemcpyAsync, one per party and
// chunk, as mpc_softmax_hostio issued them) vs SM-driven copy kernels that read / write the pinned
// host buffers directly (one launch per chunk and direction, both parties), both directions at once.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pcie_copy tools/pcie_copy.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

struct Pair { const uint4* src[2]; uint4* dst[2]; long long n16; };

__global__ void k_copy2(Pair p)
{
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (int q = 0; q < 2; ++q) {
        const uint4* __restrict__ s = p.src[q];
        uint4* __restrict__ d = p.dst[q];
        long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
        // 4 independent 16-B loads in flight per thread (PCIe read latency is ~1-2 us)
        for (; i + 3 * stride < p.n16; i += 4 * stride) {
            uint4 a = s[i], b = s[i + stride], c = s[i + 2 * stride], e = s[i + 3 * stride];
            d[i] = a; d[i + stride] = b; d[i + 2 * stride] = c; d[i + 3 * stride] = e;
        }
        for (; i < p.n16; i += stride) d[i] = s[i];
    }
}

int main()
{
    const size_t half = 12582912;                 // one party's cfg2 shares: 12288 x 128 x 8 B
    uint64_t *hx[2], *hz[2], *dx[2], *dz[2];
    for (int q = 0; q < 2; ++q) {
        CK(cudaHostAlloc(&hx[q], half, cudaHostAllocDefault));
        CK(cudaHostAlloc(&hz[q], half, cudaHostAllocDefault));
        CK(cudaMalloc(&dx[q], half));
        CK(cudaMalloc(&dz[q], half));
        memset(hx[q], 1, half);
        CK(cudaMemset(dz[q], 2, half));
    }
    cudaStream_t s1, s2;
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    cudaEvent_t a, b, f;
    cudaEventCreate(&a); cudaEventCreate(&b); cudaEventCreate(&f);
    auto timeit = [&](auto fn, const char* what, double dirs = 2.0) {
        for (int r = 0; r < 3; ++r) fn();
        cudaDeviceSynchronize();
        const int reps = 10;
        cudaEventRecord(a, 0);
        for (int r = 0; r < reps; ++r) {
            cudaEventRecord(f, 0);
            cudaStreamWaitEvent(s1, f, 0); cudaStreamWaitEvent(s2, f, 0);
            fn();
            cudaEventRecord(f, s1); cudaStreamWaitEvent(0, f, 0);
            cudaEventRecord(f, s2); cudaStreamWaitEvent(0, f, 0);
        }
        cudaEventRecord(b, 0);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= reps;
        printf("%-58s %.4f ms  %6.1f GB/s aggregate\n", what, ms, dirs * 2.0 * half / ms / 1e6);
    };
    for (int nch : {1, 2, 3, 4, 6, 8}) {
        const size_t cb = half / nch;
        char name[128];
        snprintf(name, sizeof name, "DMA, both directions, %d chunks x 2 parties", nch);
        timeit([&] {
            for (int i = 0; i < nch; ++i)
                for (int q = 0; q < 2; ++q) {
                    cudaMemcpyAsync((char*)dx[q] + i * cb, (char*)hx[q] + i * cb, cb, cudaMemcpyHostToDevice, s1);
                    cudaMemcpyAsync((char*)hz[q] + i * cb, (char*)dz[q] + i * cb, cb, cudaMemcpyDeviceToHost, s2);
                }
        }, name);
        if (hx[1] > hx[0] && hz[1] > hz[0] && dx[1] > dx[0] && dz[1] > dz[0]) {
            snprintf(name, sizeof name, "DMA 2D (both parties one copy), %d chunks", nch);
            timeit([&] {
                for (int i = 0; i < nch; ++i) {
                    cudaMemcpy2DAsync((char*)dx[0] + i * cb, (char*)dx[1] - (char*)dx[0], (char*)hx[0] + i * cb,
                                      (char*)hx[1] - (char*)hx[0], cb, 2, cudaMemcpyHostToDevice, s1);
                    cudaMemcpy2DAsync((char*)hz[0] + i * cb, (char*)hz[1] - (char*)hz[0], (char*)dz[0] + i * cb,
                                      (char*)dz[1] - (char*)dz[0], cb, 2, cudaMemcpyDeviceToHost, s2);
                }
            }, name);
            CK(cudaGetLastError());
        } else {
            printf("(2D variant skipped: allocation order)\n");
        }
        for (int G : {32}) {
            snprintf(name, sizeof name, "SM copy, both directions, %d chunks, %d CTAs x 512", nch, G);
            timeit([&] {
                for (int i = 0; i < nch; ++i) {
                    Pair in{{(const uint4*)((char*)hx[0] + i * cb), (const uint4*)((char*)hx[1] + i * cb)},
                            {(uint4*)((char*)dx[0] + i * cb), (uint4*)((char*)dx[1] + i * cb)}, (long long)(cb / 16)};
                    Pair out{{(const uint4*)((char*)dz[0] + i * cb), (const uint4*)((char*)dz[1] + i * cb)},
                             {(uint4*)((char*)hz[0] + i * cb), (uint4*)((char*)hz[1] + i * cb)}, (long long)(cb / 16)};
                    k_copy2<<<G, 512, 0, s1>>>(in);
                    k_copy2<<<G, 512, 0, s2>>>(out);
                }
            }, name);
        }
    }
    for (int G : {32}) {
        char name[128];
        snprintf(name, sizeof name, "SM copy, H2D only, 1 chunk, %d CTAs", G);
        Pair in{{(const uint4*)hx[0], (const uint4*)hx[1]}, {(uint4*)dx[0], (uint4*)dx[1]}, (long long)(half / 16)};
        timeit([&] { k_copy2<<<G, 512, 0, s1>>>(in); }, name, 1.0);
        snprintf(name, sizeof name, "SM copy, D2H only, 1 chunk, %d CTAs", G);
        Pair out{{(const uint4*)dz[0], (const uint4*)dz[1]}, {(uint4*)hz[0], (uint4*)hz[1]}, (long long)(half / 16)};
        timeit([&] { k_copy2<<<G, 512, 0, s2>>>(out); }, name, 1.0);
    }
    CK(cudaGetLastError());
    uint64_t chk = 0;
    CK(cudaMemcpy(&chk, dx[1] + 12345, 8, cudaMemcpyDeviceToHost));
    printf("check %s\n", chk == 0x0101010101010101ull && hz[0][777] == 0x0202020202020202ull ? "ok" : "BAD");
    return 0;
}
