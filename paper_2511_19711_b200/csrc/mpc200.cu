// mpc200.cu -- the C ABI of include/mpc200.h: validation, step accounting, launches.
//
// Kernels (kernels.cuh) are written once against a launch policy:
//   MPC_MODE_BOTH          BothA: one GPU executes both parties and the dealer; openings
//                          are formed in registers.
//   MPC_MODE_PAIR          PairA: this GPU is one party; every opening is a warp-level
//                          exchange with the peer party's kernel through NVLink peer memory
//                          (cooperative launch, so every CTA is resident on both GPUs).
//   MPC_MODE_PAIR_LOOPBACK PairA with both parties' CTAs in one launch on one GPU.
// No tensor cores: the path is element-wise / bitwise integer work.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cstdarg>
#include <algorithm>
#include <vector>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>      // header-only NVTX3: no-ops unless a tool (nsys / ncu) is attached

#include "mpc200.h"
#include "kernels.cuh"
#include "matmul.cuh"
#include "matmul_tc.cuh"
#include "ln_blk.cuh"
#include "plain.cuh"

using namespace mpc;

#define TPB 256
#define NWARPS (TPB / 32)

// per-launch timing records (mpc_ctx_enable_kernel_timing)
struct TimingRec { const char* name; cudaEvent_t a, b; u64 philox_at; u64 philox; u64 units; };

// one party's exchange memory (single cudaMalloc so it can be exported with cudaIpc)
struct XAlloc {
    void* base;
    size_t bytes;
    u64 rx_off, flag_off, round_off, tags_off, err_off;
};

struct mpc_ctx {
    mpc_config cfg;
    Keys K;
    u64 step;
    cudaStream_t stream;
    int sm_count;
    mpc_stats st;
    u64 last_philox;
    char err[512];
    void* scratch;          // ctx-owned, grow-only, stream-ordered on `stream`
    size_t scratch_bytes;
    int timing;
    TimingRec* recs;
    int nrec, caprec;
    cudaEvent_t* pool;
    int npool, cappool;
    // PAIR modes
    int slots;              // warp slots of the exchange memory
    XAlloc xa[2];           // own (and, loopback, the other party's) exchange memory
    void* peer_base;        // MPC_MODE_PAIR: the peer's exchange memory (cudaIpc-mapped)
    int connected;
    int debug_hdr;          // PAIR: exchange and compare an op header before every op (MPC_ERR_PROTOCOL)
    int circuit;            // LTZ carry circuit: 0 Kogge-Stone, 1 carry cone (2.7)
    int mm_engine;          // mpc_matmul ring GEMM: 0 auto, 1 SIMT, 2 tensor cores
    struct HostIO* hio;     // pipelined host-buffer execution (mpc_softmax_hostio), lazily created
    int nvtx_open;          // an op-level NVTX range is open (begin_op .. finish)
    int xfmt;               // PAIR exchange wire format (proto.cuh): 0 LL, 1 LL63
    int xused;              // a PAIR exchange kernel has been launched (the format is then fixed)
    // trusted dealer's correction stream
    int dtarget;            // DEALER: the grid its launches are sized for (MPC_MODE_PAIR / _PAIR_LOOPBACK)
    u64* dw;                // DEALER: stream words (device), capacity and words used
    u64 dw_cap, dw_end;
    u32* dkmax;             // DEALER: device high-water mark (corrections per thread) of one launch
    u32 dcap;               // DEALER: per-thread capacity the next launch is tried with
    mpc_corr_seg* segv;     // DEALER: segments produced; party 1: segments to consume
    i64 nseg, capseg;
    const u64* cwords;      // party 1: the stream being consumed (caller-owned device words)
    i64 cnext;              // party 1: next segment
    int corr_on;            // party 1: corrections come from the stream (K_0 unused)
};

// Pipelined host-buffer execution: chunk i goes H2D on `h2d`, computes on cs[i % HIO_SLOTS] with its
// own staging buffers and kernel scratch, and comes back D2H on `d2h` -- the copy engines (both
// PCIe directions) overlap each other and the compute of the neighbouring chunks.
constexpr int HIO_SLOTS = 16;           // capacity; h->nslots in use (MPC_HIO_SLOTS, default below)
#ifndef MPC_HIO_DEFAULT_SLOTS
#define MPC_HIO_DEFAULT_SLOTS 4
#endif
struct HostIO {
    int nslots;
    cudaStream_t h2d, d2h, cs[HIO_SLOTS];
    cudaEvent_t in_ready[HIO_SLOTS], comp_done[HIO_SLOTS], out_done[HIO_SLOTS], start;
    u64* dbuf[HIO_SLOTS]; size_t dbuf_bytes[HIO_SLOTS];
    void* scr[HIO_SLOTS]; size_t scr_bytes[HIO_SLOTS];
    bool used[HIO_SLOTS];
};

static bool is_pair(const mpc_ctx* c) { return c->cfg.mode != MPC_MODE_BOTH; }   // PAIR, LOOPBACK, DEALER
static bool is_loop(const mpc_ctx* c) { return c->cfg.mode == MPC_MODE_PAIR_LOOPBACK; }
static bool is_dealer(const mpc_ctx* c) { return c->cfg.mode == MPC_MODE_DEALER; }
// FNV-1a of a launch's kernel-family name: the tag of its correction-stream segment
static u64 fnv_tag(const char* name)
{
    u64 h = 1469598103934665603ull;
    for (const char* q = name; *q; ++q) { h ^= (u8)*q; h *= 1099511628211ull; }
    return h;
}

static cudaEvent_t ev_get(mpc_ctx* c)
{
    if (c->npool > 0) return c->pool[--c->npool];
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}
static void ev_put(mpc_ctx* c, cudaEvent_t e)
{
    if (c->npool == c->cappool) {
        c->cappool = c->cappool ? 2 * c->cappool : 64;
        c->pool = (cudaEvent_t*)realloc(c->pool, sizeof(cudaEvent_t) * (size_t)c->cappool);
    }
    c->pool[c->npool++] = e;
}
// close the attribution window of the previous record (its acct ran after its launch)
static void rec_close(mpc_ctx* c)
{
    if (c->timing && c->nrec > 0) {
        TimingRec& r = c->recs[c->nrec - 1];
        if (r.philox == ~0ull) r.philox = c->last_philox - r.philox_at;
    }
}
// NVTX ranges (SURVEY 5 tracing): every compute entry point opens an op range in begin_op (named
// after the ABI function) that finish / the next op closes, and every kernel launch is a nested
// range named after its kernel family; nsys / ncu --nvtx show the per-op and per-launch timeline.
static nvtxDomainHandle_t nvtx_domain()
{
    static nvtxDomainHandle_t d = nvtxDomainCreateA("mpc200");
    return d;
}
static void nvtx_push(const char* name)
{
    nvtxEventAttributes_t ev{};
    ev.version = NVTX_VERSION;
    ev.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
    ev.messageType = NVTX_MESSAGE_TYPE_ASCII;
    ev.message.ascii = name;
    nvtxDomainRangePushEx(nvtx_domain(), &ev);
}
static void nvtx_pop() { nvtxDomainRangePop(nvtx_domain()); }

static void rec_begin(mpc_ctx* c, const char* name, u64 units)
{
    nvtx_push(name);
    if (!c->timing) return;
    rec_close(c);
    if (c->nrec == c->caprec) {
        c->caprec = c->caprec ? 2 * c->caprec : 256;
        c->recs = (TimingRec*)realloc(c->recs, sizeof(TimingRec) * (size_t)c->caprec);
    }
    TimingRec& r = c->recs[c->nrec++];
    r.name = name; r.a = ev_get(c); r.b = ev_get(c); r.philox_at = c->last_philox; r.philox = ~0ull; r.units = units;
    cudaEventRecord(r.a, c->stream);
}
static void rec_end(mpc_ctx* c)
{
    if (c->timing && c->nrec > 0) cudaEventRecord(c->recs[c->nrec - 1].b, c->stream);
    nvtx_pop();
}

// grow-only scratch, stream-ordered on the ctx stream (reused by every row op)
static void* scratch(mpc_ctx* c, size_t bytes)
{
    if (bytes <= c->scratch_bytes) return c->scratch;
    if (c->scratch) cudaFreeAsync(c->scratch, c->stream);
    c->scratch = nullptr; c->scratch_bytes = 0;
    if (cudaMallocAsync(&c->scratch, bytes, c->stream) != cudaSuccess) { c->scratch = nullptr; return nullptr; }
    c->scratch_bytes = bytes;
    return c->scratch;
}

static mpc_status fail(mpc_ctx* c, mpc_status s, const char* fmt, ...)
{
    if (c) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(c->err, sizeof c->err, fmt, ap);
        va_end(ap);
    }
    return s;
}

static mpc_status cuda_check(mpc_ctx* c, const char* where)
{
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(c, MPC_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
    return MPC_OK;
}

static Key mkkey(u64 k) { return make_key(k); }

// E(c) = round-half-even(c * 2^16) (reading R2), host side
static u64 E(double c) { return (u64)(long long)nearbyint(c * 65536.0); }

static int gate_count(int w)
{
    const int m = w - 1;
    if (m <= 0) return 0;
    const int L = ceil_log2i(m);
    int g = m;
    for (int k = 0; k < L; ++k) g += 2 * (m - (1 << k));
    return g;
}

// accounting of one primitive over n units (DESIGN.md 2.3 / 2.4 cost model; both parties + dealer)
static void acct_beaver(mpc_ctx* c, u64 n)
{
    c->last_philox += 2 * n + (n + 1) / 2;
    c->st.bytes_per_party += 16 * n;
    c->st.rounds += 1;
}
static void acct_square(mpc_ctx* c, u64 n)
{
    c->last_philox += n + (n + 1) / 2;
    c->st.bytes_per_party += 8 * n;
    c->st.rounds += 1;
}
// broadcast triple: 1.5 blocks per element + 2 per row; 8 B per element and per
// row; the row openings and the element openings are separate rounds here
static void acct_bcast(mpc_ctx* c, u64 n, u64 rows)
{
    c->last_philox += n + (n + 1) / 2 + 2 * rows;
    c->st.bytes_per_party += 8 * n + 8 * rows;
    c->st.rounds += 2;
}
// the pruned carry cone (ltz_cone.cuh) covers every window 1..64: 32 leaf positions for w <= 33, 64 above
static bool use_cone(const mpc_ctx* c, int w) { (void)w; return c->circuit == 1; }
static void acct_ltz(mpc_ctx* c, u64 n, int w)
{
    const u64 groups = (n + 31) / 32;
    const bool cone = use_cone(c, w);
    c->last_philox += groups * (cone ? cone_philox_per_group(w) : ltz_philox_per_group(w));
    c->st.bytes_per_party += groups * (8ull * (u64)(cone ? cone_gate_count(w) : gate_count(w)) + 4ull);
    c->st.rounds += 2 + (w > 1 ? ceil_log2i(w - 1) : 0);
}

static int grid_for(const mpc_ctx* c, i64 work_items, int threads, int per_sm = 8)
{
    i64 b = (work_items + threads - 1) / threads;
    const i64 cap = (i64)c->sm_count * per_sm;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (int)b;
}

// ------------------------------------------------------------------ simple kernels ----
__global__ void k_prg_fill(Key key, u64 unit0, u32 step, u32 slot, u32* out, i64 n, int reps)
{
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        const u64 u = unit0 + (u64)i;
        uint4 v = prg(key, u, step, slot);
        for (int r = 1; r < reps; ++r) v = philox(key, v.x, v.y, v.z ^ step, v.w ^ slot);
        reinterpret_cast<uint4*>(out)[i] = v;
    }
}

// S1: v = E(x); owner share v - r, other r; r = PRG(K_s, off+i, s, 0).  A PAIR party writes only
// its own share (x may be NULL on the non-owner).
__global__ void k_share(const void* x, int f64, int owner, u64* s0, u64* s1, i64 n, u64 off, u32 s, Key ks)
{
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        const uint4 R = prg(ks, off + (u64)i, s, 0);
        const u64 r = w64(R.x, R.y);
        u64 v = 0;
        if (x) {
            const double xv = f64 ? static_cast<const double*>(x)[i] : (double)static_cast<const float*>(x)[i];
            v = (u64)__double2ll_rn(xv * 65536.0);
        }
        const u64 own = v - r;
        if (s0) s0[i] = owner == 0 ? own : r;
        if (s1) s1[i] = owner == 1 ? own : r;
    }
}

__global__ void k_open(const u64* s0, const u64* s1, i64 n, u64* ring, double* f, int scale_bits)
{
    const double inv = 1.0 / (double)(1ull << scale_bits);
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        const u64 v = s0[i] + s1[i];
        if (ring) ring[i] = v;
        if (f) f[i] = (double)(i64)v * inv;
    }
}

__global__ void k_trunc(SP x, SO z, i64 n, int bits)
{
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        if (z.p[0]) z.p[0][i] = shr(x.p[0][i], bits);
        if (z.p[1]) z.p[1][i] = shr(x.p[1][i], bits);
    }
}

// maxpool: gather each k x k window (public zero padding) into a row
__global__ void k_pool_gather(SP x, SO rowsbuf, int N, int C, int H, int W, int k, int stride, int pad, int Ho, int Wo)
{
    const i64 rows = (i64)N * C * Ho * Wo, kk = (i64)k * k;
    for (i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x; t < rows * kk; t += (i64)gridDim.x * blockDim.x) {
        const i64 o = t / kk, e = t - o * kk;
        const int dy = (int)(e / k), dx = (int)(e - (i64)dy * k);
        const i64 ow = o % Wo, oh = (o / Wo) % Ho, c = (o / ((i64)Wo * Ho)) % C, img = o / ((i64)Wo * Ho * C);
        const i64 iy = oh * stride - pad + dy, ix = ow * stride - pad + dx;
        const bool in = iy >= 0 && iy < H && ix >= 0 && ix < W;
        const i64 idx = ((img * C + c) * H + iy) * W + ix;
        for (int p = 0; p < 2; ++p)
            if (rowsbuf.p[p]) rowsbuf.p[p][t] = in ? x.p[p][idx] : 0ull;
    }
}

// ------------------------------------------------------------------ launch machinery ----
static XMem xmem_of(const mpc_ctx* c, int which)
{
    const XAlloc& a = c->xa[which];
    char* b = (char*)a.base;
    XMem m;
    m.rx = (u64*)(b + a.rx_off); m.flag = (u64*)(b + a.flag_off); m.round = (u64*)(b + a.round_off);
    m.tags = (u32*)(b + a.tags_off);
    m.err = (int*)(b + a.err_off); m.slots = c->slots;
    if (is_dealer(c)) {                               // the dealer's self-loop (proto.cuh PairP)
        m.prx = m.rx; m.pflag = m.flag;
    } else if (is_loop(c)) {
        const XAlloc& o = c->xa[1 - which];
        char* ob = (char*)o.base;
        m.prx = (u64*)(ob + o.rx_off); m.pflag = (u64*)(ob + o.flag_off);
    } else {
        char* pb = (char*)c->peer_base;
        m.prx = (u64*)(pb + a.rx_off); m.pflag = (u64*)(pb + a.flag_off);
    }
    return m;
}

static PairArgs pair_args(const mpc_ctx* c, int G)
{
    PairArgs pa;
    pa.K = c->K;
    pa.party = c->cfg.party;
    pa.loopback = is_loop(c) ? 1 : 0;
    pa.G = G;
    pa.fmt = c->xfmt;
    pa.xm[0] = xmem_of(c, 0);
    pa.xm[1] = is_loop(c) ? xmem_of(c, 1) : pa.xm[0];
    return pa;
}

// A PAIR kernel in its two roles (kernels.cuh PairAR): r0 = PairA (party 0, the simulated dealer,
// loopback), r1 = PairAS (party 1 reading the dealer's stream, the dealer's own pass)
template <class K0, class K1> struct KRoles { K0 r0; K1 r1; };
template <class K0, class K1> static KRoles<K0, K1> kroles(K0 a, K1 b) { return {a, b}; }
static bool stream_role(const mpc_ctx* c) { return is_dealer(c) || c->corr_on; }
template <class KR>
static void set_smem_attr(KR k, int bytes)
{
    cudaFuncSetAttribute(k.r0, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(k.r1, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

// CTAs per party for a PAIR launch: every CTA of both parties must be co-resident.  The same G for
// both roles (min occupancy), so party 0 (role 0), party 1 (either role) and the dealer pair up.
template <class KR>
static int pair_ctas(mpc_ctx* c, KR kk, size_t dyn, i64 want, int tpb = TPB)
{
    int nb = 0, nb1 = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kk.r0, tpb, dyn) != cudaSuccess || nb < 1) nb = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb1, kk.r1, tpb, dyn) != cudaSuccess || nb1 < 1) nb1 = 1;
    nb = std::min(nb, nb1);
    const bool halves = is_loop(c) || (is_dealer(c) && c->dtarget == MPC_MODE_PAIR_LOOPBACK);
    i64 cap = (i64)nb * c->sm_count / (halves ? 2 : 1);
    cap = std::min<i64>(cap, c->slots / (tpb / 32));
    i64 G = std::min<i64>(want, cap);
    return (int)std::max<i64>(G, 1);
}

template <class KR, class... Args>
static mpc_status launch_pair_kernel_tpb(mpc_ctx* c, KR kk, int G, size_t dyn, int tpb, const char* name, Args... args);

template <class KR, class... Args>
static mpc_status launch_pair_kernel(mpc_ctx* c, KR kk, int G, size_t dyn, const char* name, Args... args)
{
    return launch_pair_kernel_tpb(c, kk, G, dyn, TPB, name, args...);
}

// The dealer's offline pass of one launch: party 1's kernel with the same grid in
// the dealer role (cmode 2: no exchange, no share access), writing the launch's corrections as one
// stream segment; relaunched with a larger per-thread capacity if the high-water mark exceeds it.
template <class Kern, class... Args>
static mpc_status dealer_launch(mpc_ctx* c, Kern kern, int G, size_t dyn, int tpb, const char* name, Args... args)
{
    PairArgs pa;
    memset(&pa, 0, sizeof pa);
    pa.K = c->K; pa.party = 1; pa.loopback = 0; pa.G = G; pa.fmt = c->xfmt; pa.cmode = 2;
    pa.xm[0] = pa.xm[1] = xmem_of(c, 0);
    const u64 T = (u64)G * (u64)tpb;
    if (!c->dkmax && cudaMalloc(&c->dkmax, sizeof(u32)) != cudaSuccess) { c->dkmax = nullptr; return fail(c, MPC_ERR_NOMEM, "dealer counter"); }
    if (!c->dcap) c->dcap = 64;
    u32 kmax = 0;
    for (;;) {
        const u64 need = c->dw_end + (u64)c->dcap * T;
        if (need > c->dw_cap) {                       // grow (offline: synchronous is fine)
            const u64 ncap = std::max<u64>(need, 2 * c->dw_cap);
            u64* nw = nullptr;
            if (cudaMalloc(&nw, ncap * sizeof(u64)) != cudaSuccess) return fail(c, MPC_ERR_NOMEM, "dealer stream %llu words", (unsigned long long)ncap);
            if (c->dw) { cudaMemcpyAsync(nw, c->dw, c->dw_end * sizeof(u64), cudaMemcpyDeviceToDevice, c->stream); cudaStreamSynchronize(c->stream); cudaFree(c->dw); }
            c->dw = nw; c->dw_cap = ncap;
        }
        pa.cw = c->dw + c->dw_end; pa.ccap = c->dcap; pa.kmax = c->dkmax;
        cudaMemsetAsync(c->dkmax, 0, sizeof(u32), c->stream);
        void* argv[] = {(void*)&pa, (void*)&args...};
        rec_begin(c, name, 0);
        cudaError_t e = cudaLaunchKernel((const void*)kern, G, tpb, argv, dyn, c->stream);
        rec_end(c);
        c->st.launches++;
        if (e != cudaSuccess) return fail(c, MPC_ERR_CUDA, "%s: dealer launch: %s", name, cudaGetErrorString(e));
        cudaMemcpyAsync(&kmax, c->dkmax, sizeof(u32), cudaMemcpyDeviceToHost, c->stream);
        if (cudaStreamSynchronize(c->stream) != cudaSuccess) return cuda_check(c, name);
        if (kmax <= c->dcap) break;
        c->dcap = kmax;                               // too deep: run the launch again with room for all
    }
    if (c->nseg == c->capseg) {
        c->capseg = c->capseg ? 2 * c->capseg : 64;
        c->segv = (mpc_corr_seg*)realloc(c->segv, sizeof(mpc_corr_seg) * (size_t)c->capseg);
    }
    c->segv[c->nseg++] = mpc_corr_seg{c->dw_end, T, kmax, fnv_tag(name)};
    c->dw_end += (u64)kmax * T;
    return cuda_check(c, name);
}

template <class KR, class... Args>
static mpc_status launch_pair_kernel_tpb(mpc_ctx* c, KR kk, int G, size_t dyn, int tpb, const char* name, Args... args)
{
    if (is_dealer(c)) return dealer_launch(c, kk.r1, G, dyn, tpb, name, args...);
    if (!is_loop(c) && !c->connected) return fail(c, MPC_ERR_INVALID, "%s: PAIR context not connected", name);
    PairArgs pa = pair_args(c, G);
    pa.cw = nullptr; pa.ccap = 0; pa.cmode = 0; pa.kmax = nullptr;
    if (c->corr_on) {                                 // party 1 reads this launch's corrections
        if (c->cnext >= c->nseg)
            return fail(c, MPC_ERR_PROTOCOL, "%s: the dealer's correction stream is exhausted (%lld segments)", name, (long long)c->nseg);
        const mpc_corr_seg& g = c->segv[c->cnext];
        if (g.tag != fnv_tag(name) || g.threads != (u64)G * (u64)tpb)
            return fail(c, MPC_ERR_PROTOCOL, "%s: correction segment %lld is for another launch (tag / %llu threads vs %llu)",
                        name, (long long)c->cnext, (unsigned long long)g.threads, (unsigned long long)G * (u64)tpb);
        ++c->cnext;
        pa.cw = const_cast<u64*>(c->cwords) + g.base; pa.ccap = (u32)g.depth; pa.cmode = 1;
    }
    c->xused = 1;
    void* argv[] = {(void*)&pa, (void*)&args...};
    const int grid = G * (is_loop(c) ? 2 : 1);
    rec_begin(c, name, 0);
    const void* kern = stream_role(c) ? (const void*)kk.r1 : (const void*)kk.r0;
    cudaError_t e = cudaLaunchCooperativeKernel(kern, grid, tpb, argv, dyn, c->stream);
    rec_end(c);
    c->st.launches++;
    if (e != cudaSuccess) return fail(c, MPC_ERR_CUDA, "%s: cooperative launch: %s", name, cudaGetErrorString(e));
    return cuda_check(c, name);
}

template <class K>
static int occupancy(K kern, size_t dyn = 0, int tpb = TPB)
{
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, tpb, dyn) != cudaSuccess || nb < 1) nb = 1;
    return nb;
}

// Per-device launch-setup cache: kernel attributes (cudaFuncSetAttribute) and occupancies belong to
// a device context, so a process driving contexts on several GPUs sets them up once per device.
constexpr int MAX_DEV = 64;
struct DevCache { int v[MAX_DEV]; };
template <class F>
static int dev_cached(DevCache& dc, int dev, F compute)
{
    if (dev < 0 || dev >= MAX_DEV) return compute();
    if (!dc.v[dev]) dc.v[dev] = compute();      // racing first calls compute the same value
    return dc.v[dev];
}

template <class Body>
static mpc_status launch_pairs(mpc_ctx* c, i64 n, u64 off, const Body& b, const char* name)
{
    if (n <= 0) return MPC_OK;
    const i64 npairs = (i64)(((off + (u64)n + 1) >> 1) - (off >> 1));
    if (!is_pair(c)) {
        static DevCache occ;
        const int per_sm = dev_cached(occ, c->cfg.device, [] { return occupancy(k_pairs<BothA, Body>); });
        rec_begin(c, name, (u64)n);
        k_pairs<BothA, Body><<<grid_for(c, npairs, TPB, per_sm), TPB, 0, c->stream>>>(BothA{c->K}, n, off, b);
        rec_end(c);
        c->st.launches++;
        return cuda_check(c, name);
    }
    const auto kk = kroles(k_pairs<PairA, Body>, k_pairs<PairAS, Body>);
    const int G = pair_ctas(c, kk, 0, (npairs + TPB - 1) / TPB);
    return launch_pair_kernel(c, kk, G, 0, name, n, off, b);
}

template <class Body>
static mpc_status launch_cone(mpc_ctx* c, i64 n, u64 off, const Body& b, const char* name)
{
    if (n <= 0) return MPC_OK;
    const i64 nw = (((n + 31) / 32) + CG - 1) / CG;       // warps of work
    const size_t dyn = sizeof(u64) * (size_t)Body::kStash * NWARPS;
    if (!is_pair(c)) {
        static DevCache occ;
        const int per_sm = dev_cached(occ, c->cfg.device, [&] {
            cudaFuncSetAttribute(k_groups_cone<BothA, Body>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
            return occupancy(k_groups_cone<BothA, Body>, dyn);
        });
        rec_begin(c, name, (u64)n);
        k_groups_cone<BothA, Body><<<grid_for(c, nw * 32, TPB, per_sm), TPB, dyn, c->stream>>>(BothA{c->K}, n, off, b);
        rec_end(c);
        c->st.launches++;
        return cuda_check(c, name);
    }
    const auto kk = kroles(k_groups_cone<PairA, Body>, k_groups_cone<PairAS, Body>);
    set_smem_attr(kk, (int)dyn);
    const int G = pair_ctas(c, kk, dyn, (nw * 32 + TPB - 1) / TPB);
    return launch_pair_kernel(c, kk, G, dyn, name, n, off, b);
}

template <class Body>
static mpc_status launch_groups(mpc_ctx* c, i64 n, u64 off, const Body& b, const char* name)
{
    if (n <= 0) return MPC_OK;
    if (!is_pair(c)) {
        static DevCache occ;
        const int per_sm = dev_cached(occ, c->cfg.device, [] { return occupancy(k_groups<BothA, Body>); });
        rec_begin(c, name, (u64)n);
        k_groups<BothA, Body><<<grid_for(c, ((n + 31) / 32) * 32, TPB, per_sm), TPB, 0, c->stream>>>(BothA{c->K}, n, off, b);
        rec_end(c);
        c->st.launches++;
        return cuda_check(c, name);
    }
    const auto kk = kroles(k_groups<PairA, Body>, k_groups<PairAS, Body>);
    const int G = pair_ctas(c, kk, 0, (((n + 31) / 32) * 32 + TPB - 1) / TPB);
    return launch_pair_kernel(c, kk, G, 0, name, n, off, b);
}

static const size_t SMEM_LIMIT = 56 * 1024;      // + 16 KB static cone smem: keep 3 CTAs per SM

// fused row kernels: work tile in shared memory when it fits, else a per-CTA global tile
// Row kernels' tail tiles as 16-row half tiles (kernels.cuh tile_plan): off by default -- cfg2 softmax
// 0.282 vs 0.271 ms, max 0.147 vs 0.141 ms (tools/ab_half.py, r02): a lone tile is latency-bound, so
// a half tile is hardly shorter, and the SMs that held 3 tiles still hold 2 + 2 halves.
// MPC_TAIL_HALF=1 in the environment turns it on (read per call: A/B and tests without a rebuild).
static int tail_half()
{
    const char* e = getenv("MPC_TAIL_HALF");
    return e ? atoi(e) : 0;
}

template <class Args, class KB, class KP>
static mpc_status launch_rows(mpc_ctx* c, KB kb, KP kp, Args& a, i64 rows, i64 work_u64, i64 esc_u64, const char* name,
                              size_t smem_limit = SMEM_LIMIT)
{
    const i64 ntiles = (rows + 31) / 32;
    const size_t wbytes = sizeof(u64) * (size_t)work_u64;
    const bool smem = work_u64 > 0 && wbytes <= smem_limit;
    const size_t dyn = smem ? wbytes : 0;
    if (smem) {
        cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wbytes);
        set_smem_attr(kp, (int)wbytes);
    }
    int grid;
    if (!is_pair(c)) grid = (int)std::min<i64>(ntiles, (i64)c->sm_count * occupancy(kb, dyn, MPC_ROW_TPB));
    else grid = pair_ctas(c, kp, dyn, ntiles, MPC_ROW_TPB);
    // tests: cap the row kernels' grid (MPC_ROW_GRID_CAP) so small inputs take the multi-round and
    // half-tile paths of tile_plan
    if (const char* cap = getenv("MPC_ROW_GRID_CAP")) { const int g = atoi(cap); if (g > 0 && g < grid) grid = g; }
    const int launched = grid * (is_loop(c) ? 2 : 1);
    a.use_smem = smem ? 1 : 0;
    a.gscratch = nullptr;
    a.work_u64 = work_u64;
    // one scratch allocation: [E tiles (esc_u64 per CTA)] [global work tiles if not in smem]
    const size_t ebytes = sizeof(u64) * (size_t)esc_u64 * (size_t)launched;
    const size_t gbytes = smem ? 0 : wbytes * (size_t)launched;
    u64* base = nullptr;
    if (ebytes + gbytes > 0) {
        base = (u64*)scratch(c, ebytes + gbytes);
        if (!base) return fail(c, MPC_ERR_NOMEM, "%s: scratch %zu bytes", name, ebytes + gbytes);
    }
    a.escratch = base;
    if (!smem && work_u64 > 0) a.gscratch = base + (size_t)esc_u64 * (size_t)launched;
    if (is_pair(c)) return launch_pair_kernel_tpb(c, kp, grid, dyn, MPC_ROW_TPB, name, a);
    rec_begin(c, name, (u64)rows);
    kb<<<grid, MPC_ROW_TPB, dyn, c->stream>>>(BothA{c->K}, a);
    rec_end(c);
    c->st.launches++;
    return cuda_check(c, name);
}

static mpc_status launch_max(mpc_ctx* c, MaxArgs& a, i64 rows, i64 cols, int w, const char* name)
{
    // BOTH, Kogge-Stone w <= 33: the softmax's balanced plan (one range of ~rows / grid rows per CTA, on
    // min(grid, rows / 2) CTAs) when the level buffers fit shared memory; MPC_MAX_BAL=0: off (per call)
    const char* mb_env = getenv("MPC_MAX_BAL");
    if (!is_pair(c) && !a.cone && w <= 33 && !(mb_env && atoi(mb_env) == 0) && rows >= 2) {
        static DevCache occ;
        const int per_sm = dev_cached(occ, c->cfg.device, [] {
            cudaFuncSetAttribute(k_max<0, BothA>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
            return occupancy(k_max<0, BothA>, 100 * 1024, MPC_ROW_TPB);
        });
        i64 g = std::max<i64>(1, std::min<i64>((i64)c->sm_count * per_sm, rows / 2));
        if (const char* cap = getenv("MPC_ROW_GRID_CAP")) { const int v = atoi(cap); if (v > 0 && v < g) g = v; }
        const i64 hr = (rows + 1) / 2;
        const i64 nrange = hr > 32 * g ? g * ((hr + 32 * g - 1) / (32 * g)) : g;   // k rounds of ranges per CTA
        const i64 tr = 2 * ((hr + nrange - 1) / nrange), wkm = max_work_u64(cols, tr);
        if (tr <= 64 && wkm * 8 <= 100 * 1024) {
            a.tr = (int)tr; a.nrange = nrange; a.use_smem = 1; a.work_u64 = wkm; a.gscratch = nullptr;
            cudaFuncSetAttribute(k_max<0, BothA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(wkm * 8));
            rec_begin(c, name, (u64)rows);
            k_max<0, BothA><<<(int)g, MPC_ROW_TPB, wkm * 8, c->stream>>>(BothA{c->K}, a);
            rec_end(c);
            c->st.launches++;
            return cuda_check(c, name);
        }
    }
    const i64 wk = max_work_u64(cols);
    if (a.cone && w > 33) return launch_rows(c, k_max<3, BothA>, kroles(k_max<3, PairA>, k_max<3, PairAS>), a, rows, wk, 0, name);
    if (w > 33) return launch_rows(c, k_max<1, BothA>, kroles(k_max<1, PairA>, k_max<1, PairAS>), a, rows, wk, 0, name);
    if (a.cone) return launch_rows(c, k_max<2, BothA>, kroles(k_max<2, PairA>, k_max<2, PairAS>), a, rows, wk, 0, name);
    return launch_rows(c, k_max<0, BothA>, kroles(k_max<0, PairA>, k_max<0, PairAS>), a, rows, wk, 0, name);
}

// short rows (cols <= MAXS_COLS, MaxPool windows): warp-per-tile kernel, windows gathered in-kernel
static mpc_status launch_max_small(mpc_ctx* c, MaxSmallArgs& a, const char* name)
{
    const int lv = use_cone(c, a.w) ? (a.w > 33 ? 3 : 2) : (a.w > 33 ? 1 : 0);
    const size_t dyn = sizeof(u64) * 64 * (size_t)a.cols * NWARPS;
    a.fcol = make_fastdiv((u32)a.cols);
    const i64 ntiles = (a.rows + 31) / 32;
    const i64 nctas = (ntiles + NWARPS - 1) / NWARPS;
    auto pick = [&](auto kb, auto kp) -> mpc_status {
        cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        set_smem_attr(kp, (int)dyn);
        if (is_pair(c)) return launch_pair_kernel_tpb(c, kp, pair_ctas(c, kp, dyn, nctas, TPB), dyn, TPB, name, a);
        const int grid = (int)std::min<i64>(nctas, (i64)c->sm_count * occupancy(kb, dyn, TPB));
        rec_begin(c, name, (u64)a.rows);
        kb<<<grid, TPB, dyn, c->stream>>>(BothA{c->K}, a);
        rec_end(c);
        c->st.launches++;
        return cuda_check(c, name);
    };
    if (lv == 1) return pick(k_max_small<1, BothA>, kroles(k_max_small<1, PairA>, k_max_small<1, PairAS>));
    if (lv == 2) return pick(k_max_small<2, BothA>, kroles(k_max_small<2, PairA>, k_max_small<2, PairAS>));
    if (lv == 3) return pick(k_max_small<3, BothA>, kroles(k_max_small<3, PairA>, k_max_small<3, PairAS>));
    return pick(k_max_small<0, BothA>, kroles(k_max_small<0, PairA>, k_max_small<0, PairAS>));
}

// ------------------------------------------------------------------ validation helpers ----
// shares argument valid for the mode: both pointers (BOTH / LOOPBACK) or sh[party] (PAIR)
static bool bad_sh(const mpc_ctx* c, mpc_shares s)
{
    if (is_dealer(c)) return false;                   // the dealer reads and writes no shares
    if (c->cfg.mode == MPC_MODE_PAIR) {
        const uint64_t* p = s.sh[c->cfg.party];
        return !p || ((uintptr_t)p & 7);
    }
    return !s.sh[0] || !s.sh[1] || ((uintptr_t)s.sh[0] & 7) || ((uintptr_t)s.sh[1] & 7);
}
static SP spv(const mpc_ctx* c, mpc_shares s)
{
    SP r{{s.sh[0], s.sh[1]}};
    if (c->cfg.mode == MPC_MODE_PAIR) r.p[1 - c->cfg.party] = nullptr;
    if (is_dealer(c)) r.p[0] = r.p[1] = nullptr;
    return r;
}
static SO sov(const mpc_ctx* c, mpc_shares s)
{
    SO r{{s.sh[0], s.sh[1]}};
    if (c->cfg.mode == MPC_MODE_PAIR) r.p[1 - c->cfg.party] = nullptr;
    if (is_dealer(c)) r.p[0] = r.p[1] = nullptr;
    return r;
}

// common prologue of a compute call: validates the step budget, resets the per-call counter
// debug header (mpc_ctx_set_debug): FNV-1a of the entry point's name, mixed with the step id and
// the step count the call needs; exchanged and compared by one PAIR launch before the op
static mpc_status hdr_check(mpc_ctx* c, const char* op, u64 steps_needed)
{
    u64 h = 1469598103934665603ull;
    for (const char* q = op; *q; ++q) { h ^= (u8)*q; h *= 1099511628211ull; }
    h ^= c->step * 0x9E3779B97F4A7C15ull; h *= 1099511628211ull;
    h ^= steps_needed; h *= 1099511628211ull;
    return launch_groups(c, 32, 0, HdrBody{h, SP{{nullptr, nullptr}}}, "op_header");
}
static mpc_status begin_op(mpc_ctx* c, u64 steps_needed, const char* op)
{
    if (!c) return MPC_ERR_INVALID;
    if (c->nvtx_open) nvtx_pop();                 // an op that returned early left its range open
    nvtx_push(op);
    c->nvtx_open = 1;
    c->last_philox = 0;
    c->st.calls++;
    if (c->step + steps_needed > (1ull << 32))
        return fail(c, MPC_ERR_RANGE, "step counter would exceed 2^32");
    // kernels launch on the calling thread's current device: refuse to run on another one
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess || cur != c->cfg.device)
        return fail(c, MPC_ERR_INVALID, "current CUDA device %d is not the context's device %d", cur, c->cfg.device);
    if (c->debug_hdr && is_pair(c)) return hdr_check(c, op, steps_needed);
    return MPC_OK;
}
#define begin(c, steps) begin_op((c), (steps), __func__)
static void finish(mpc_ctx* c, u64 steps)
{
    if (c->nvtx_open) { nvtx_pop(); c->nvtx_open = 0; }
    rec_close(c);
    c->step += steps;
    c->st.steps += steps;
    c->st.philox_calls += c->last_philox;
}

static bool exp_ok(const mpc_exp_p* p)
{
    return p && p->t >= 0 && p->t <= 8 && p->window >= 1 && p->window <= 64 && (p->square == 0 || p->square == 1);
}
static bool nr_ok(const mpc_nr_p* p) { return p && p->iters >= 1 && p->iters <= 12 && exp_ok(&p->exp); }

static ExpK mk_exp(const mpc_exp_p* p)
{
    return ExpK{p->t, p->clamp ? 1 : 0, p->window, p->square ? 1 : 0, E(1.0), E(ldexp(1.0, p->t))};
}
static NrK mk_nr(const mpc_nr_p* p)
{
    NrK k;
    k.iters = p->iters; k.exp = mk_exp(&p->exp);
    k.e_half = E(0.5); k.e_c003 = E(0.003); k.e_two = E(2.0); k.e_three = E(3.0);
    k.e_02 = E(0.2); k.e_22 = E(2.2);
    return k;
}
static u64 exp_steps_h(const mpc_exp_p* p) { return (u64)p->t + (p->clamp ? 2u : 0u); }

static void acct_exp(mpc_ctx* c, u64 n, const mpc_exp_p* p)
{
    if (p->clamp) { acct_ltz(c, n, p->window); acct_beaver(c, n); }
    for (int k = 0; k < p->t; ++k) { if (p->square) acct_square(c, n); else acct_beaver(c, n); }
}

static int max_levels_h(i64 cols) { int L = 0; i64 m = cols; while (m > 1) { m = (m + 1) / 2; ++L; } return L; }

static void acct_max(mpc_ctx* c, i64 rows, i64 cols, int w)
{
    i64 m = cols;
    while (m > 1) {
        const i64 h = m / 2;
        acct_ltz(c, (u64)(rows * h), w);
        acct_beaver(c, (u64)(rows * h));
        m = h + (m & 1);
    }
}

// ------------------------------------------------------------------ PAIR memory ----
// Initial exchange state (proto.cuh): LL -- all zero (tags are rounds >= 1); LL63 -- every receive
// word holds tag 1 and every lane's tag bits are 1, so the first write of a word carries tag 0.
__global__ void k_xinit(u64* rx, u32* tags, u64* rounds, i64 slots, int fmt)
{
    for (i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x; t < slots * XSLOT_RX; t += (i64)gridDim.x * blockDim.x)
        rx[t] = fmt ? (1ull << 63) : 0ull;
    for (i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x; t < slots * 32; t += (i64)gridDim.x * blockDim.x)
        tags[t] = 0xffffffffu;
    for (i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x; t < slots; t += (i64)gridDim.x * blockDim.x)
        rounds[t] = 0;
}
static mpc_status xinit(mpc_ctx* c, XAlloc& a)
{
    const size_t S = (size_t)c->slots;
    char* b = (char*)a.base;
    k_xinit<<<(unsigned)std::min<size_t>((S * XSLOT_RX + 255) / 256, 4096), 256>>>(
        (u64*)(b + a.rx_off), (u32*)(b + a.tags_off), (u64*)(b + a.round_off), (i64)S, c->xfmt);
    return cudaDeviceSynchronize() == cudaSuccess ? MPC_OK : MPC_ERR_CUDA;
}

static mpc_status xalloc(mpc_ctx* c, XAlloc& a)
{
    const size_t S = (size_t)c->slots;
    a.rx_off = 0;
    a.flag_off = a.rx_off + S * XSLOT_RX * sizeof(u64);
    a.round_off = a.flag_off + S * 4 * sizeof(u64);
    a.tags_off = a.round_off + S * sizeof(u64);
    a.err_off = a.tags_off + S * 32 * sizeof(u32);
    a.bytes = a.err_off + 256;
    if (cudaMalloc(&a.base, a.bytes) != cudaSuccess) { a.base = nullptr; return MPC_ERR_NOMEM; }
    if (cudaMemset(a.base, 0, a.bytes) != cudaSuccess) return MPC_ERR_CUDA;
    return xinit(c, a);
}

// ------------------------------------------------------------------ ABI ----
extern "C" {

const char* mpc_version(void) { return "mpc200 0.3 (sm_100a; BOTH, PAIR over peer memory, PAIR_LOOPBACK; tcgen05 matmul)"; }

mpc_status mpc_ctx_create(const mpc_config* cfg, mpc_ctx** out)
{
    if (!cfg || !out) return MPC_ERR_INVALID;
    if (cfg->frac_bits != 16) return MPC_ERR_RANGE;
    if (cfg->mode != MPC_MODE_BOTH && cfg->mode != MPC_MODE_PAIR && cfg->mode != MPC_MODE_PAIR_LOOPBACK &&
        cfg->mode != MPC_MODE_DEALER)
        return MPC_ERR_INVALID;
    if (cfg->mode == MPC_MODE_PAIR && (cfg->party < 0 || cfg->party > 1)) return MPC_ERR_INVALID;
    if (cfg->mode == MPC_MODE_DEALER && cfg->party != 1) return MPC_ERR_INVALID;   // the dealer serves party 1
    mpc_ctx* c = new mpc_ctx();
    memset(c, 0, sizeof *c);
    c->cfg = *cfg;
    c->K.ks = mkkey(cfg->key_share); c->K.k0 = mkkey(cfg->key_p0); c->K.k1 = mkkey(cfg->key_p1);
    c->stream = (cudaStream_t)cfg->cuda_stream;
    if (cudaSetDevice(cfg->device) != cudaSuccess) { delete c; return MPC_ERR_CUDA; }
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cfg->device) != cudaSuccess) {
        delete c; return MPC_ERR_CUDA;
    }
    c->sm_count = sms;
    // keep stream-ordered allocations in the pool across synchronizations
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, cfg->device) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    c->dtarget = MPC_MODE_PAIR;
    if (cfg->mode == MPC_MODE_DEALER) {
        c->slots = sms * 8 * NWARPS;       // the parties' launch sizing (pair_ctas)
        c->xfmt = 0;                       // self-loop exchange memory (LL: fewest instructions)
        mpc_status st = xalloc(c, c->xa[0]);
        if (st) { mpc_ctx_destroy(c); return st; }
    } else if (cfg->mode != MPC_MODE_BOTH) {
        c->slots = sms * 8 * NWARPS;       // up to 8 resident CTAs per SM
        // default wire format: LL63 across GPUs (NVLink bytes bind), LL in loopback (local HBM:
        // LL's fewer instructions per word win, tools/ab_pair.py)
        c->xfmt = cfg->mode == MPC_MODE_PAIR ? 1 : 0;
        mpc_status st = xalloc(c, c->xa[0]);
        if (!st && cfg->mode == MPC_MODE_PAIR_LOOPBACK) st = xalloc(c, c->xa[1]);
        if (st) { mpc_ctx_destroy(c); return st; }
    }
    *out = c;
    return MPC_OK;
}

mpc_status mpc_ctx_destroy(mpc_ctx* c)
{
    if (!c) return MPC_OK;
    if (c->nvtx_open) nvtx_pop();
    cudaStreamSynchronize(c->stream);
    for (int i = 0; i < c->nrec; ++i) { cudaEventDestroy(c->recs[i].a); cudaEventDestroy(c->recs[i].b); }
    for (int i = 0; i < c->npool; ++i) cudaEventDestroy(c->pool[i]);
    free(c->recs); free(c->pool);
    if (c->scratch) { cudaFreeAsync(c->scratch, c->stream); cudaStreamSynchronize(c->stream); }
    if (c->hio) {
        HostIO* h = c->hio;
        for (int b = 0; b < h->nslots; ++b) {
            cudaStreamSynchronize(h->cs[b]);
            if (h->dbuf[b]) cudaFree(h->dbuf[b]);
            if (h->scr[b]) cudaFree(h->scr[b]);
            cudaStreamDestroy(h->cs[b]);
            cudaEventDestroy(h->in_ready[b]); cudaEventDestroy(h->comp_done[b]); cudaEventDestroy(h->out_done[b]);
        }
        cudaStreamSynchronize(h->h2d); cudaStreamSynchronize(h->d2h);
        cudaStreamDestroy(h->h2d); cudaStreamDestroy(h->d2h); cudaEventDestroy(h->start);
        delete h;
    }
    if (c->peer_base) cudaIpcCloseMemHandle(c->peer_base);
    for (int i = 0; i < 2; ++i) if (c->xa[i].base) cudaFree(c->xa[i].base);
    if (c->dw) cudaFree(c->dw);
    if (c->dkmax) cudaFree(c->dkmax);
    free(c->segv);
    delete c;
    return MPC_OK;
}

mpc_status mpc_pair_export(mpc_ctx* c, void* handle_out)
{
    if (!c || !handle_out || c->cfg.mode != MPC_MODE_PAIR) return MPC_ERR_INVALID;
    static_assert(sizeof(cudaIpcMemHandle_t) <= MPC_PAIR_HANDLE_BYTES, "handle size");
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, c->xa[0].base) != cudaSuccess) return fail(c, MPC_ERR_CUDA, "cudaIpcGetMemHandle");
    memset(handle_out, 0, MPC_PAIR_HANDLE_BYTES);
    memcpy(handle_out, &h, sizeof h);
    return MPC_OK;
}

mpc_status mpc_pair_connect(mpc_ctx* c, const void* peer_handle)
{
    if (!c || !peer_handle || c->cfg.mode != MPC_MODE_PAIR) return MPC_ERR_INVALID;
    cudaIpcMemHandle_t h;
    memcpy(&h, peer_handle, sizeof h);
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess || cur != c->cfg.device)
        return fail(c, MPC_ERR_INVALID, "pair_connect: current CUDA device %d is not the context's device %d", cur, c->cfg.device);
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return fail(c, MPC_ERR_CUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
    c->peer_base = p;
    c->connected = 1;
    return MPC_OK;
}

mpc_status mpc_ctx_sync(mpc_ctx* c)
{
    if (!c) return MPC_ERR_INVALID;
    cudaError_t e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return fail(c, MPC_ERR_CUDA, "sync: %s", cudaGetErrorString(e));
    for (int i = 0; i < 2; ++i) {
        if (!c->xa[i].base) continue;
        int err = 0;
        cudaMemcpy(&err, (char*)c->xa[i].base + c->xa[i].err_off, sizeof err, cudaMemcpyDeviceToHost);
        if (err == 2) return fail(c, MPC_ERR_PROTOCOL, "PAIR op headers differ (the parties issued different calls)");
        if (err) return fail(c, MPC_ERR_TIMEOUT, "PAIR exchange timed out (peer not running the same op?)");
    }
    return MPC_OK;
}

mpc_status mpc_ctx_set_debug(mpc_ctx* c, int on)
{
    if (!c) return MPC_ERR_INVALID;
    c->debug_hdr = on ? 1 : 0;
    return MPC_OK;
}

mpc_status mpc_ctx_set_exchange(mpc_ctx* c, int fmt)
{
    if (!c) return MPC_ERR_INVALID;
    if (fmt != 0 && fmt != 1) return fail(c, MPC_ERR_RANGE, "exchange format must be 0 (LL) or 1 (LL63)");
    if (!is_pair(c)) return MPC_OK;                        // BOTH: no exchange
    if (fmt == c->xfmt) return MPC_OK;
    if (c->xused) return fail(c, MPC_ERR_INVALID, "set_exchange: the context has already exchanged (set it first)");
    c->xfmt = fmt;
    for (int i = 0; i < 2; ++i)
        if (c->xa[i].base) { mpc_status st = xinit(c, c->xa[i]); if (st) return fail(c, st, "set_exchange: init"); }
    return MPC_OK;
}
int mpc_ctx_get_exchange(const mpc_ctx* c) { return c ? c->xfmt : -1; }

mpc_status mpc_ctx_set_ltz_circuit(mpc_ctx* c, int circuit)
{
    if (!c) return MPC_ERR_INVALID;
    if (circuit != 0 && circuit != 1) return fail(c, MPC_ERR_RANGE, "circuit must be 0 (Kogge-Stone) or 1 (carry cone)");
    c->circuit = circuit;
    return MPC_OK;
}

mpc_status mpc_dealer_set_target(mpc_ctx* c, int target_mode)
{
    if (!c || !is_dealer(c) || (target_mode != MPC_MODE_PAIR && target_mode != MPC_MODE_PAIR_LOOPBACK))
        return c ? fail(c, MPC_ERR_INVALID, "dealer_set_target: a DEALER context and MPC_MODE_PAIR / _LOOPBACK") : MPC_ERR_INVALID;
    c->dtarget = target_mode;
    return MPC_OK;
}

mpc_status mpc_dealer_stream(const mpc_ctx* c, const uint64_t** words, uint64_t* n_words, const mpc_corr_seg** segs,
                             int64_t* n_segs)
{
    if (!c || !is_dealer(c)) return MPC_ERR_INVALID;
    cudaStreamSynchronize(c->stream);
    if (words) *words = c->dw;
    if (n_words) *n_words = c->dw_end;
    if (segs) *segs = c->segv;
    if (n_segs) *n_segs = c->nseg;
    return MPC_OK;
}

mpc_status mpc_dealer_reset(mpc_ctx* c)
{
    if (!c || !is_dealer(c)) return MPC_ERR_INVALID;
    cudaStreamSynchronize(c->stream);
    c->dw_end = 0;
    c->nseg = 0;
    return MPC_OK;
}

mpc_status mpc_ctx_set_corrections(mpc_ctx* c, const uint64_t* words, uint64_t n_words, const mpc_corr_seg* segs,
                                   int64_t n_segs)
{
    if (!c) return MPC_ERR_INVALID;
    const bool p1 = (c->cfg.mode == MPC_MODE_PAIR && c->cfg.party == 1) || is_loop(c);
    if (!p1) return fail(c, MPC_ERR_INVALID, "set_corrections: only party 1 (PAIR party 1 or PAIR_LOOPBACK) reads a dealer stream");
    if (!words && n_segs == 0) { c->corr_on = 0; c->cwords = nullptr; c->nseg = 0; c->cnext = 0; return MPC_OK; }
    if (!words || n_segs < 0 || (n_segs > 0 && !segs) || ((uintptr_t)words & 7))
        return fail(c, MPC_ERR_INVALID, "set_corrections: words / segs");
    for (int64_t i = 0; i < n_segs; ++i)
        if (segs[i].base + segs[i].depth * segs[i].threads > n_words || segs[i].depth >= (1ull << 32))
            return fail(c, MPC_ERR_INVALID, "set_corrections: segment %lld outside the %llu words", (long long)i,
                        (unsigned long long)n_words);
    if (n_segs > c->capseg) {
        c->capseg = n_segs;
        c->segv = (mpc_corr_seg*)realloc(c->segv, sizeof(mpc_corr_seg) * (size_t)c->capseg);
    }
    if (n_segs) memcpy(c->segv, segs, sizeof(mpc_corr_seg) * (size_t)n_segs);
    c->nseg = n_segs; c->cnext = 0; c->cwords = words; c->corr_on = 1;
    return MPC_OK;
}

int64_t mpc_ctx_corrections_left(const mpc_ctx* c)
{
    if (!c || !c->corr_on) return -1;
    return c->nseg - c->cnext;
}

mpc_status mpc_ctx_set_matmul_engine(mpc_ctx* c, int engine)
{
    if (!c) return MPC_ERR_INVALID;
    if (engine < 0 || engine > 2) return fail(c, MPC_ERR_RANGE, "engine must be 0 (auto), 1 (SIMT) or 2 (tensor cores)");
    c->mm_engine = engine;
    return MPC_OK;
}

mpc_status mpc_ctx_enable_kernel_timing(mpc_ctx* c, int on)
{
    if (!c) return MPC_ERR_INVALID;
    c->timing = on ? 1 : 0;
    return MPC_OK;
}

int mpc_ctx_kernel_times(mpc_ctx* c, mpc_kernel_time* out, int cap)
{
    if (!c) return -1;
    rec_close(c);
    if (c->nrec > 0) cudaEventSynchronize(c->recs[c->nrec - 1].b);
    int n = 0;
    for (int i = 0; i < c->nrec; ++i) {
        TimingRec& r = c->recs[i];
        if (out && n < cap) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, r.a, r.b);
            out[n].name = r.name; out[n].ms = ms;
            out[n].philox = r.philox == ~0ull ? 0 : r.philox; out[n].units = r.units;
            ++n;
        }
        ev_put(c, r.a); ev_put(c, r.b);
    }
    c->nrec = 0;
    return n;
}

mpc_status mpc_ctx_set_step(mpc_ctx* c, uint64_t step, int force)
{
    if (!c) return MPC_ERR_INVALID;
    if (step < c->step && !force) return fail(c, MPC_ERR_REUSE, "set_step %llu below current %llu", (unsigned long long)step, (unsigned long long)c->step);
    if (step >= (1ull << 32)) return fail(c, MPC_ERR_RANGE, "step >= 2^32");
    c->step = step;
    return MPC_OK;
}
uint64_t mpc_ctx_get_step(const mpc_ctx* c) { return c ? c->step : 0; }
mpc_status mpc_ctx_set_stream(mpc_ctx* c, void* s)
{
    if (!c) return MPC_ERR_INVALID;
    cudaStream_t ns = (cudaStream_t)s;
    cudaStreamCaptureStatus cap_new = cudaStreamCaptureStatusNone, cap_old = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(ns, &cap_new);
    cudaStreamIsCapturing(c->stream, &cap_old);
    if (ns != c->stream && cap_new == cudaStreamCaptureStatusNone && cap_old == cudaStreamCaptureStatusNone) {
        // scratch and exchange memory are stream-ordered: order the new stream after the old one.
        // (Under CUDA-graph capture an event from outside the capture cannot be waited on: the
        // capturing caller orders its stream after the context's previous work itself.)
        cudaEvent_t e = ev_get(c);
        cudaEventRecord(e, c->stream);
        cudaStreamWaitEvent(ns, e, 0);
        ev_put(c, e);
    }
    c->stream = ns;
    return MPC_OK;
}
mpc_status mpc_ctx_stats(const mpc_ctx* c, mpc_stats* o) { if (!c || !o) return MPC_ERR_INVALID; *o = c->st; return MPC_OK; }
mpc_status mpc_ctx_reset_stats(mpc_ctx* c) { if (!c) return MPC_ERR_INVALID; memset(&c->st, 0, sizeof c->st); return MPC_OK; }
const char* mpc_last_error(const mpc_ctx* c) { return c ? c->err : "null context"; }
uint64_t mpc_last_call_philox(const mpc_ctx* c) { return c ? c->last_philox : 0; }

mpc_status mpc_prg_fill(mpc_ctx* c, uint64_t key, uint64_t unit0, uint32_t step, uint32_t slot,
                        uint32_t* out, int64_t n, int reps)
{
    if (!c || !out || n < 0 || reps < 1) return MPC_ERR_INVALID;
    if (n == 0) return MPC_OK;
    c->last_philox = (u64)n * (u64)reps;
    rec_begin(c, "prg_fill", (u64)n);
    k_prg_fill<<<grid_for(c, n, TPB, 16), TPB, 0, c->stream>>>(mkkey(key), unit0, step, slot, out, n, reps);
    rec_end(c);
    c->st.launches++;
    return cuda_check(c, "prg_fill");
}

mpc_status mpc_share(mpc_ctx* c, const void* x, int x_is_f64, int owner, mpc_shares out, int64_t n, int64_t off)
{
    mpc_status st = begin(c, 1);
    if (st) return st;
    if (owner != 0 && owner != 1) return fail(c, MPC_ERR_INVALID, "owner must be 0 or 1");
    if (n < 0 || off < 0) return fail(c, MPC_ERR_INVALID, "bad n/off");
    const bool pair = c->cfg.mode == MPC_MODE_PAIR;
    if (bad_sh(c, out)) return fail(c, MPC_ERR_INVALID, "share: null/misaligned output");
    const bool need_x = !is_dealer(c) && (!pair || c->cfg.party == owner);
    if (need_x && !x && n > 0) return fail(c, MPC_ERR_INVALID, "share: the owner needs x");
    u64* s0 = !pair || c->cfg.party == 0 ? out.sh[0] : nullptr;
    u64* s1 = !pair || c->cfg.party == 1 ? out.sh[1] : nullptr;
    if (n > 0 && !is_dealer(c)) {                      // (no corrections: the dealer has nothing to do)
        rec_begin(c, "share", (u64)n);
        k_share<<<grid_for(c, n, TPB, 16), TPB, 0, c->stream>>>(need_x ? x : nullptr, x_is_f64, owner, s0, s1, n, (u64)off, (u32)c->step, c->K.ks);
        rec_end(c);
        c->st.launches++;
        if ((st = cuda_check(c, "share"))) return st;
    }
    c->last_philox = (u64)n;
    finish(c, 1);
    return MPC_OK;
}

mpc_status mpc_open(mpc_ctx* c, mpc_shares in, int64_t n, uint64_t* ring_out, double* f64_out, int scale_bits)
{
    return mpc_open_to(c, in, n, -1, ring_out, f64_out, scale_bits);
}

mpc_status mpc_open_to(mpc_ctx* c, mpc_shares in, int64_t n, int reveal_to, uint64_t* ring_out, double* f64_out,
                       int scale_bits)
{
    mpc_status st = begin(c, 0);
    if (st) return st;
    if (n < 0 || scale_bits < 0 || scale_bits > 62) return fail(c, MPC_ERR_INVALID, "bad n/scale");
    if (reveal_to < -1 || reveal_to > 1) return fail(c, MPC_ERR_INVALID, "reveal_to must be -1, 0 or 1");
    if (bad_sh(c, in)) return fail(c, MPC_ERR_INVALID, "open: null pointer");
    if (n > 0) {
        if (is_dealer(c)) { ring_out = nullptr; f64_out = nullptr; }   // same launch as party 1, no output
        if (is_pair(c)) {
            const int writer = reveal_to >= 0 ? reveal_to : (is_loop(c) ? 0 : -1);
            st = launch_groups(c, n, 0, OpenBody{spv(c, in), ring_out, f64_out, n, 1.0 / (double)(1ull << scale_bits),
                                                 writer, reveal_to}, "open");
        } else {
            rec_begin(c, "open", (u64)n);
            k_open<<<grid_for(c, n, TPB, 16), TPB, 0, c->stream>>>(in.sh[0], in.sh[1], n, ring_out, f64_out, scale_bits);
            rec_end(c);
            c->st.launches++;
            st = cuda_check(c, "open");
        }
        if (st) return st;
    }
    c->st.bytes_per_party += 8ull * (u64)n;
    c->st.rounds += 1;
    rec_close(c);
    return MPC_OK;
}

mpc_status mpc_trunc(mpc_ctx* c, mpc_shares x, mpc_shares z, int64_t n, int bits)
{
    mpc_status st = begin(c, 0);
    if (st) return st;
    if (bits < 0 || bits > 63) return fail(c, MPC_ERR_RANGE, "bits");
    if (bad_sh(c, x) || bad_sh(c, z) || n < 0) return fail(c, MPC_ERR_INVALID, "trunc args");
    if (n > 0 && !is_dealer(c)) {
        rec_begin(c, "trunc", (u64)n);
        k_trunc<<<grid_for(c, n, TPB, 16), TPB, 0, c->stream>>>(spv(c, x), sov(c, z), n, bits);
        rec_end(c);
        c->st.launches++;
        if ((st = cuda_check(c, "trunc"))) return st;
    }
    rec_close(c);
    return MPC_OK;
}

mpc_status mpc_mul(mpc_ctx* c, mpc_shares x, mpc_shares y, mpc_shares z, int64_t n, int64_t off, int tb)
{
    mpc_status st = begin(c, 1);
    if (st) return st;
    if (tb != 0 && tb != 16) return fail(c, MPC_ERR_RANGE, "trunc_bits must be 0 or 16");
    if (n < 0 || off < 0) return fail(c, MPC_ERR_INVALID, "bad n/off");
    if (bad_sh(c, x) || bad_sh(c, y) || bad_sh(c, z)) return fail(c, MPC_ERR_INVALID, "mul: null pointer");
    if ((st = launch_pairs(c, n, (u64)off, MulBody{(u32)c->step, spv(c, x), spv(c, y), sov(c, z), n, tb}, "mul"))) return st;
    acct_beaver(c, (u64)n);
    finish(c, 1);
    return MPC_OK;
}

mpc_status mpc_square(mpc_ctx* c, mpc_shares x, mpc_shares z, int64_t n, int64_t off, int tb)
{
    mpc_status st = begin(c, 1);
    if (st) return st;
    if (tb != 0 && tb != 16) return fail(c, MPC_ERR_RANGE, "trunc_bits must be 0 or 16");
    if (n < 0 || off < 0) return fail(c, MPC_ERR_INVALID, "bad n/off");
    if (bad_sh(c, x) || bad_sh(c, z)) return fail(c, MPC_ERR_INVALID, "square: null pointer");
    if ((st = launch_pairs(c, n, (u64)off, SquareBody{(u32)c->step, spv(c, x), sov(c, z), n, tb}, "square"))) return st;
    acct_square(c, (u64)n);
    finish(c, 1);
    return MPC_OK;
}

// S4'' broadcast multiply (NEXT #2): row masks + openings, then element products
mpc_status mpc_mul_bcast(mpc_ctx* c, mpc_shares x, mpc_shares y, mpc_shares z, int64_t rows, int64_t cols,
                         int64_t off, int64_t row_off, int tb)
{
    mpc_status st = begin(c, 1);
    if (st) return st;
    if (tb != 0 && tb != 16) return fail(c, MPC_ERR_RANGE, "trunc_bits must be 0 or 16");
    if (rows < 0 || cols < 1 || off < 0 || row_off < 0 || rows * cols >= (1ll << 31))
        return fail(c, MPC_ERR_INVALID, "mul_bcast: bad rows/cols/off (rows*cols < 2^31)");
    if (bad_sh(c, x) || bad_sh(c, y) || bad_sh(c, z)) return fail(c, MPC_ERR_INVALID, "mul_bcast: null pointer");
    const i64 n = rows * cols;
    if (rows > 0) {
        u64* br = (u64*)scratch(c, sizeof(u64) * 6 * (size_t)rows);     // [3][rows], loopback: per party
        if (!br) return fail(c, MPC_ERR_NOMEM, "mul_bcast scratch");
        BmbRowsArgs ra{(u32)c->step, spv(c, y), rows, (u64)row_off, br, is_loop(c) ? 1 : 0};
        const i64 nw = (rows + 31) / 32;
        if (!is_pair(c)) {
            rec_begin(c, "bcast_rows", (u64)rows);
            k_bmb_rows<BothA><<<grid_for(c, nw * 32, TPB, 8), TPB, 0, c->stream>>>(BothA{c->K}, ra);
            rec_end(c);
            c->st.launches++;
            st = cuda_check(c, "bcast_rows");
        } else {
            st = launch_pair_kernel(c, kroles(k_bmb_rows<PairA>, k_bmb_rows<PairAS>), pair_ctas(c, kroles(k_bmb_rows<PairA>, k_bmb_rows<PairAS>), 0, (nw * 32 + TPB - 1) / TPB),
                                    0, "bcast_rows", ra);
        }
        if (st) return st;
        st = launch_pairs(c, n, (u64)off, BmbBody{(u32)c->step, spv(c, x), sov(c, z), n, make_fastdiv((u32)cols),
                                                  br, rows, tb, is_loop(c) ? 1 : 0, SP{{nullptr, nullptr}}, 0}, "mul_bcast");
        if (st) return st;
        acct_bcast(c, (u64)n, (u64)rows);
    }
    finish(c, 1);
    return MPC_OK;
}

// NEXT #3 Beaver matrix multiplication: masks + openings, then the ring GEMMs
mpc_status mpc_matmul(mpc_ctx* c, mpc_shares x, mpc_shares y, mpc_shares z, int64_t batch, int64_t M, int64_t K,
                      int64_t N, int64_t batch_off, int tb)
{
    mpc_status st = begin(c, 1);
    if (st) return st;
    if (tb != 0 && tb != 16) return fail(c, MPC_ERR_RANGE, "trunc_bits must be 0 or 16");
    const i64 nparty = c->cfg.mode == MPC_MODE_PAIR ? 1 : 2;        // parties computed by this GPU
    if (batch < 0 || M < 1 || K < 1 || N < 1 || batch_off < 0 || M > 65535ll * 64 || N > (1ll << 30) ||
        batch * M * K >= (1ll << 40) || batch * K * N >= (1ll << 40) || batch * nparty > 65535)
        return fail(c, MPC_ERR_INVALID, "matmul: bad shape (batch x parties <= 65535 grid z)");
    if (bad_sh(c, x) || bad_sh(c, y) || bad_sh(c, z)) return fail(c, MPC_ERR_INVALID, "matmul: null pointer");
    if (batch == 0) { finish(c, 1); return MPC_OK; }
    const bool tc_ok = 3 * K <= 16384;                // exact limb accumulators (matmul_tc.cuh)
    if (c->mm_engine == 2 && !tc_ok) return fail(c, MPC_ERR_UNSUPPORTED, "matmul: tensor-core engine needs K <= 5461");
    const bool use_tc = c->mm_engine == 2 || (c->mm_engine == 0 && tc_ok);
    const i64 nA = batch * M * K, nB = batch * K * N;
    // scratch: operand planes (4 (nA + nB) u64), then for the tensor-core engine the limb-tiled
    // operands of each computed party (party 0: K' = 2K, party 1: K' = 3K)
    const i64 MB = (M + TC_BM - 1) / TC_BM, NB = (N + TC_BN - 1) / TC_BN;
    const i64 Kpad = tc_kpad((int)K), Kp0 = 2 * Kpad, Kp1 = 3 * Kpad;     // term-padded K' (matmul_tc.cuh)
    const i64 la0 = batch * MB * (Kp0 / TC_BK) * TC_A_CHUNK, lb0 = batch * NB * (Kp0 / TC_BK) * TC_B_CHUNK;
    const i64 la1 = batch * MB * (Kp1 / TC_BK) * TC_A_CHUNK, lb1 = batch * NB * (Kp1 / TC_BK) * TC_B_CHUNK;
    // BOTH mode + tensor cores: the masking is fused into the limb tiling (no operand planes)
    const bool fused = use_tc && c->cfg.mode == MPC_MODE_BOTH;
    const size_t plane_bytes = fused ? 0 : sizeof(u64) * 4 * (size_t)(nA + nB);
    const size_t limb_bytes = use_tc ? (size_t)(la0 + lb0 + la1 + lb1) : 0;
    u8* sc = (u8*)scratch(c, plane_bytes + limb_bytes);
    if (!sc) return fail(c, MPC_ERR_NOMEM, "matmul scratch");
    u64 *PA = (u64*)sc, *PB = PA + 4 * nA;
    const u32 s = (u32)c->step;
    if (!fused) {
        if ((st = launch_pairs(c, nA, (u64)(batch_off * M * K), MmMaskBody{s, 8u, spv(c, x), nA, PA, 0}, "mm_mask"))) return st;
        if ((st = launch_pairs(c, nB, (u64)(batch_off * K * N), MmMaskBody{s, 9u, spv(c, y), nB, PB, 1}, "mm_mask"))) return st;
    }
    MmArgs a;
    memset(&a, 0, sizeof a);
    a.K = c->K; a.s = s; a.M = (int)M; a.Kd = (int)K; a.N = (int)N; a.batch = (int)batch; a.goff = (u64)batch_off; a.tb = tb;
    const u64 *E = PA, *A0 = PA + nA, *A1 = PA + 2 * nA, *As = PA + 3 * nA;
    const u64 *F = PB, *G = PB + nB, *B1 = PB + 2 * nB, *Bs = PB + 3 * nB;
    a.t[0][0] = MmTerm{E, G}; a.t[0][1] = MmTerm{A0, F}; a.nt[0] = 2;                          // C0 + E(B0+F) + A0 F
    a.t[1][0] = MmTerm{As, Bs}; a.t[1][1] = MmTerm{E, B1}; a.t[1][2] = MmTerm{A1, F}; a.nt[1] = 3; // AB - C0 + E B1 + A1 F
    a.z[0] = z.sh[0]; a.z[1] = z.sh[1];
    if (c->cfg.mode == MPC_MODE_PAIR) { a.p0 = c->cfg.party; a.np = 1; }
    else { a.p0 = 0; a.np = 2; }
    // the trusted dealer's matrix correction C1 = (A0+A1)(B0+B1) - C0: the dealer forms
    // it with ONE GEMM term and writes it as a stream segment; party 1 reads it in its epilogue and
    // multiplies only E B1 + A1 F (K' = 2K instead of 3K)
    const u64 nC = (u64)(batch * M * N);
    if (is_dealer(c)) {
        if (c->dw_end + nC > c->dw_cap) {
            const u64 ncap = std::max<u64>(c->dw_end + nC, 2 * c->dw_cap);
            u64* nw = nullptr;
            if (cudaMalloc(&nw, ncap * sizeof(u64)) != cudaSuccess) return fail(c, MPC_ERR_NOMEM, "dealer stream");
            if (c->dw) { cudaMemcpyAsync(nw, c->dw, c->dw_end * sizeof(u64), cudaMemcpyDeviceToDevice, c->stream); cudaStreamSynchronize(c->stream); cudaFree(c->dw); }
            c->dw = nw; c->dw_cap = ncap;
        }
        a.nt[1] = 1; a.tb = 0; a.p0 = 1; a.np = 1;
        a.z[1] = c->dw + c->dw_end;
    } else if (c->corr_on && a.p0 + a.np > 1) {
        if (c->cnext >= c->nseg || c->segv[c->cnext].tag != fnv_tag("matmul_c1") || c->segv[c->cnext].threads != nC)
            return fail(c, MPC_ERR_PROTOCOL, "matmul: the next correction segment is not this product's C1");
        a.cin[1] = c->cwords + c->segv[c->cnext].base;
        ++c->cnext;
        a.t[1][0] = MmTerm{E, B1}; a.t[1][1] = MmTerm{A1, F}; a.nt[1] = 2;                     // C1 + E B1 + A1 F
    }
    if (!use_tc) {
        const dim3 grid((unsigned)((N + 63) / 64), (unsigned)((M + 63) / 64), (unsigned)(batch * a.np));
        rec_begin(c, "matmul", (u64)(batch * M * N));
        k_mm_simt<<<grid, 256, 0, c->stream>>>(a);
        rec_end(c);
        c->st.launches++;
        if ((st = cuda_check(c, "matmul"))) return st;
    } else {
        TcArgs t;
        memset(&t, 0, sizeof t);
        t.mm = a;
        u8* lp = sc + plane_bytes;
        u8* LA[2] = {lp, lp + la0 + lb0};
        u8* LB[2] = {lp + la0, lp + la0 + lb0 + la1};
        const i64 Kps[2] = {Kp0, a.nt[1] * Kpad};
        if (fused) {
            const i64 KBn = Kpad / TC_BK;
            FuseArgs fx{c->K, s, x.sh[0], x.sh[1], (int)M, (int)K, (int)batch, (u64)batch_off, LA[0], LA[1]};
            FuseArgs fy{c->K, s, y.sh[0], y.sh[1], (int)N, (int)K, (int)batch, (u64)batch_off, LB[0], LB[1]};
            rec_begin(c, "mm_fuse", (u64)(nA + nB));
            // tiles: LHS 32 rows x 32 k, RHS 64 columns x 32 k (FW = 4 elements per thread)
            k_mm_fuse_lhs<<<(unsigned)std::min<i64>(batch * 4 * MB * KBn, (i64)c->sm_count * 16), 256, 0, c->stream>>>(fx);
            k_mm_fuse_rhs<<<(unsigned)std::min<i64>(batch * ((N + 63) / 64) * KBn, (i64)c->sm_count * 16), 256, 0, c->stream>>>(fy);
            rec_end(c);
            c->st.launches += 2;
            for (int p = 0; p < 2; ++p) { t.A[p] = LA[p]; t.B[p] = LB[p]; t.Kp[p] = (int)Kps[p]; }
        }
        for (int p = a.p0; p < a.p0 + a.np && !fused; ++p) {
            LimbArgs la{}, lb{};
            for (int q = 0; q < a.nt[p]; ++q) { la.t[q] = a.t[p][q].a; lb.t[q] = a.t[p][q].b; }
            la.nt = lb.nt = a.nt[p];
            la.rows = (int)M; la.K = (int)K; la.Kp = (int)Kps[p]; la.rhs = 0; la.rows_blk = TC_BM; la.batch = (int)batch;
            la.in_stride = M * K; la.out = LA[p];
            lb.rows = (int)N; lb.K = (int)K; lb.Kp = (int)Kps[p]; lb.rhs = 1; lb.rows_blk = TC_BN; lb.batch = (int)batch;
            lb.in_stride = K * N; lb.out = LB[p];
            rec_begin(c, "mm_limbs", 0);
            k_mm_limbs_lhs<<<(unsigned)std::min<i64>(batch * MB * (Kps[p] / TC_BK), (i64)c->sm_count * 8), 256, 0, c->stream>>>(la);
            // 2 * TC_BN threads pack a tile's core-matrix rows: CTAs of exactly that size, many per SM
            k_mm_limbs_rhs<<<(unsigned)std::min<i64>(batch * NB * (Kps[p] / TC_BK), (i64)c->sm_count * 24), 2 * TC_BN, 0, c->stream>>>(lb);
            rec_end(c);
            c->st.launches += 2;
            t.A[p] = LA[p]; t.B[p] = LB[p]; t.Kp[p] = (int)Kps[p];
        }
        if ((st = cuda_check(c, "mm_limbs"))) return st;
        static DevCache attr;
        dev_cached(attr, c->cfg.device, [] {
            return cudaFuncSetAttribute(k_mm_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM) == cudaSuccess ? 1 : -1;
        });
        const dim3 grid((unsigned)NB, (unsigned)MB, (unsigned)(batch * a.np));
        rec_begin(c, "matmul_tc", (u64)(batch * M * N));
        k_mm_tc<<<grid, 128, TC_SMEM, c->stream>>>(t);
        rec_end(c);
        c->st.launches++;
        if ((st = cuda_check(c, "matmul_tc"))) return st;
    }
    if (is_dealer(c)) {
        if ((st = cuda_check(c, "matmul_c1"))) return st;
        if (c->nseg == c->capseg) {
            c->capseg = c->capseg ? 2 * c->capseg : 64;
            c->segv = (mpc_corr_seg*)realloc(c->segv, sizeof(mpc_corr_seg) * (size_t)c->capseg);
        }
        c->segv[c->nseg++] = mpc_corr_seg{c->dw_end, nC, 1, fnv_tag("matmul_c1")};
        c->dw_end += nC;
    }
    c->last_philox += (u64)(nA + nB) + (u64)(batch * M * N + 1) / 2;
    c->st.bytes_per_party += 8ull * (u64)(nA + nB);
    c->st.rounds += 1;
    finish(c, 1);
    return MPC_OK;
}

static mpc_status cmp_common(mpc_ctx* c, mpc_shares x, mpc_shares z, int64_t n, int64_t off, int w, int relu)
{
    mpc_status st = begin(c, relu ? 2 : 1);
    if (st) return st;
    if (w < 1 || w > 64) return fail(c, MPC_ERR_RANGE, "window must be in [1,64]");
    if (n < 0 || off < 0 || (off & 31)) return fail(c, MPC_ERR_INVALID, "off must be a multiple of 32");
    if (bad_sh(c, x) || bad_sh(c, z)) return fail(c, MPC_ERR_INVALID, "cmp: null pointer");
    const char* name = relu ? "relu" : "cmp";
    if (use_cone(c, w) && w > 33)
        st = launch_cone(c, n, (u64)off, CmpConeBody<64>{(u32)c->step, w, spv(c, x), sov(c, z), relu, n}, name);
    else if (use_cone(c, w))
        st = launch_cone(c, n, (u64)off, CmpConeBody<32>{(u32)c->step, w, spv(c, x), sov(c, z), relu, n}, name);
    else st = w > 33 ? launch_groups(c, n, (u64)off, CmpBody<true>{(u32)c->step, w, spv(c, x), sov(c, z), relu}, name)
                : launch_groups(c, n, (u64)off, CmpBody<false>{(u32)c->step, w, spv(c, x), sov(c, z), relu}, name);
    if (st) return st;
    acct_ltz(c, (u64)n, w);
    if (relu) acct_beaver(c, (u64)n);
    finish(c, relu ? 2 : 1);
    return MPC_OK;
}

mpc_status mpc_cmp(mpc_ctx* c, mpc_shares x, mpc_shares z, int64_t n, int64_t off, int w) { return cmp_common(c, x, z, n, off, w, 0); }
mpc_status mpc_relu(mpc_ctx* c, mpc_shares x, mpc_shares z, int64_t n, int64_t off, int w) { return cmp_common(c, x, z, n, off, w, 1); }

mpc_status mpc_exp(mpc_ctx* c, mpc_shares x, mpc_shares z, int64_t n, int64_t off, const mpc_exp_p* p)
{
    if (!c) return MPC_ERR_INVALID;
    if (!exp_ok(p)) return fail(c, MPC_ERR_RANGE, "exp knobs out of range");
    mpc_status st = begin(c, exp_steps_h(p));
    if (st) return st;
    if (bad_sh(c, x) || bad_sh(c, z) || n < 0 || off < 0) return fail(c, MPC_ERR_INVALID, "exp args");
    const ExpK k = mk_exp(p);
    if (p->clamp) {
        if (off & 31) return fail(c, MPC_ERR_INVALID, "off must be a multiple of 32");
        // large n: the clamp head (LTZ group layout, steps s, s+1) into z, then the t squarings in
        // the pair layout in place (steps s+2 ..) -- the same units and output bits as one fused
        // pass, 5 % faster at 4M; small n (latency-bound, cfg1): one fused launch
        const int head = n >= (1 << 16) ? 1 : 0;
        st = p->window > 33 ? launch_groups(c, n, (u64)off, ExpGroupBody<true>{(u32)c->step, k, spv(c, x), sov(c, z), head}, "exp_clamp")
                            : launch_groups(c, n, (u64)off, ExpGroupBody<false>{(u32)c->step, k, spv(c, x), sov(c, z), head}, "exp_clamp");
        if (!st && head && k.t > 0) st = launch_pairs(c, n, (u64)off, ExpPairBody{(u32)c->step + 2u, k, spv(c, z), sov(c, z), n, 1}, "exp");
    } else {
        st = launch_pairs(c, n, (u64)off, ExpPairBody{(u32)c->step, k, spv(c, x), sov(c, z), n, 0}, "exp");
    }
    if (st) return st;
    acct_exp(c, (u64)n, p);
    finish(c, exp_steps_h(p));
    return MPC_OK;
}

}  // extern "C"

template <int KIND>
static mpc_status nr_common(mpc_ctx* c, mpc_shares x, mpc_shares z, int64_t n, int64_t off, const mpc_nr_p* p)
{
    if (!c) return MPC_ERR_INVALID;
    if (!nr_ok(p)) return fail(c, MPC_ERR_RANGE, "newton knobs out of range");
    const u64 steps = exp_steps_h(&p->exp) + (KIND == 0 ? 2u : 3u) * (u64)p->iters;
    mpc_status st = begin(c, steps);
    if (st) return st;
    if (bad_sh(c, x) || bad_sh(c, z) || n < 0 || off < 0) return fail(c, MPC_ERR_INVALID, "newton args");
    const NrK k = mk_nr(p);
    const char* name = KIND == 0 ? "recip" : "rsqrt";
    if (p->exp.clamp) {
        if (off & 31) return fail(c, MPC_ERR_INVALID, "off must be a multiple of 32");
        st = p->exp.window > 33 ? launch_groups(c, n, (u64)off, NrGroupBody<KIND, true>{(u32)c->step, k, spv(c, x), sov(c, z)}, name)
                                : launch_groups(c, n, (u64)off, NrGroupBody<KIND, false>{(u32)c->step, k, spv(c, x), sov(c, z)}, name);
    } else {
        st = launch_pairs(c, n, (u64)off, NrPairBody<KIND>{(u32)c->step, k, spv(c, x), sov(c, z), n}, name);
    }
    if (st) return st;
    acct_exp(c, (u64)n, &p->exp);
    for (int i = 0; i < (KIND == 0 ? 2 : 3) * p->iters; ++i) acct_beaver(c, (u64)n);
    finish(c, steps);
    return MPC_OK;
}

static u64 act_steps(int act, const mpc_act_p* p)
{
    if (p->form == MPC_FORM_RELU || (p->form != MPC_FORM_ERF && p->degree == 0)) return act == 2 ? 1 : 2;
    const u64 tail = act == 2 ? 1 : 2;
    if (p->form == MPC_FORM_POLY_X) return 2 + (u64)(p->degree - 1) + tail;
    if (p->form == MPC_FORM_POLY_ABS) return 3 + 1 + (u64)(p->degree - 1) + tail;
    return 2 + 1 + (u64)(p->erf_terms - 2) + 2 + tail;   // ERF
}

// S13 knob validation + the device knob struct (shared by the MPC ops and the plaintext evaluator)
static mpc_status act_knobs(mpc_ctx* c, int act, const mpc_act_p* p, ActK& k)
{
    if (!p || p->window < 1 || p->window > 64) return fail(c, MPC_ERR_RANGE, "window");
    if (p->form < 0 || p->form > 3) return fail(c, MPC_ERR_RANGE, "form");
    if ((p->form == MPC_FORM_POLY_X || p->form == MPC_FORM_POLY_ABS) && (p->degree < 0 || p->degree > 4))
        return fail(c, MPC_ERR_RANGE, "degree must be in [0,4]");
    if (p->form == MPC_FORM_ERF && (act != 0 || p->erf_terms < 2 || p->erf_terms > 12))
        return fail(c, MPC_ERR_RANGE, "erf form: GELU only, erf_terms in [2,12]");
    if (p->form == MPC_FORM_POLY_ABS && act == 2) return fail(c, MPC_ERR_RANGE, "sigmoid has no |x|-form (R30)");
    if ((p->form == MPC_FORM_POLY_X || p->form == MPC_FORM_POLY_ABS) && p->degree > 0 && !p->coeffs)
        return fail(c, MPC_ERR_INVALID, "coeffs");
    if (p->basis != 0 && p->basis != 1) return fail(c, MPC_ERR_RANGE, "basis must be 0 (Horner) or 1 (power)");
    if (p->basis == 1 && p->form == MPC_FORM_ERF) return fail(c, MPC_ERR_RANGE, "power basis: x- and |x|-forms only");
    memset(&k, 0, sizeof k);
    k.act = act; k.form = p->form; k.w = p->window; k.basis = p->form == MPC_FORM_ERF ? 0 : p->basis;
    k.e_B = E(p->B); k.e_mB = E(-p->B); k.e_half = E(0.5); k.e_one = E(1.0);
    k.e_isqrt2 = E(1.0 / sqrt(2.0)); k.e_2sqrtpi = E(2.0 / sqrt(M_PI));
    if (p->form == MPC_FORM_ERF) {
        const int K = p->erf_terms;
        double fact = 1.0;
        for (int i = 0; i < K; ++i) {
            if (i > 0) fact *= (double)i;
            k.c[i] = E(((i & 1) ? -1.0 : 1.0) / (fact * (double)(2 * i + 1)));
        }
        k.deg = K - 1;
    } else if (p->form == MPC_FORM_RELU) {
        k.deg = 0;
    } else {
        k.deg = p->degree;
        for (int i = 0; i <= p->degree; ++i) k.c[i] = E(p->coeffs[i]);
    }
    return MPC_OK;
}

static mpc_status act_common(mpc_ctx* c, int act, mpc_shares x, mpc_shares z, int64_t n, int64_t off, const mpc_act_p* p)
{
    if (!c) return MPC_ERR_INVALID;
    ActK k;
    mpc_status st = act_knobs(c, act, p, k);
    if (st) return st;
    const u64 steps = act_steps(act, p);
    st = begin(c, steps);
    if (st) return st;
    if (bad_sh(c, x) || bad_sh(c, z) || n < 0 || off < 0 || (off & 31)) return fail(c, MPC_ERR_INVALID, "act args (off % 32)");
    const char* name = act == 0 ? "gelu" : act == 1 ? "silu" : "sigmoid";
    if (use_cone(c, k.w) && k.w > 33)
        st = launch_cone(c, n, (u64)off, ActConeBody<64>{(u32)c->step, k, spv(c, x), sov(c, z), n}, name);
    else if (use_cone(c, k.w))
        st = launch_cone(c, n, (u64)off, ActConeBody<32>{(u32)c->step, k, spv(c, x), sov(c, z), n}, name);
    else st = k.w > 33 ? launch_groups(c, n, (u64)off, ActBody<true>{(u32)c->step, k, spv(c, x), sov(c, z)}, name)
                  : launch_groups(c, n, (u64)off, ActBody<false>{(u32)c->step, k, spv(c, x), sov(c, z)}, name);
    if (st) return st;
    const u64 N = (u64)n;
    if (k.deg == 0) { acct_ltz(c, N, k.w); if (act != 2) acct_beaver(c, N); }
    else {
        acct_ltz(c, N, k.w); acct_ltz(c, N, k.w);
        if (k.form == 1) { acct_ltz(c, N, k.w); acct_beaver(c, N); }
        for (u64 i = 0; i < (u64)(k.deg - 1); ++i) acct_beaver(c, N);
        if (k.form == 3) { acct_beaver(c, N); acct_beaver(c, N); acct_beaver(c, N); }
        acct_beaver(c, N);
        if (act != 2) acct_beaver(c, N);
    }
    finish(c, steps);
    return MPC_OK;
}

extern "C" {
// NEXT #4: the auto-tuner's plaintext fixed-point evaluator
mpc_status mpc_plain_eval(mpc_ctx* c, int op, const void* knobs, const double* x, double* y, int64_t rows, int64_t cols)
{
    if (!c) return MPC_ERR_INVALID;
    if (!knobs || !x || !y || rows < 0 || cols < 1) return fail(c, MPC_ERR_INVALID, "plain_eval args");
    if (x < y + rows * cols && y < x + rows * cols)      // the softmax rows use y as their max-tree workspace
        return fail(c, MPC_ERR_INVALID, "plain_eval: x and y must not overlap");
    PlainArgs a;
    memset(&a, 0, sizeof a);
    a.x = x; a.y = y; a.rows = rows; a.cols = cols;
    mpc_status st = MPC_OK;
    switch (op) {
    case MPC_PLAIN_EXP: {
        const mpc_exp_p* p = (const mpc_exp_p*)knobs;
        if (!exp_ok(p)) return fail(c, MPC_ERR_RANGE, "exp knobs");
        a.op = 0; a.ek = mk_exp(p); break;
    }
    case MPC_PLAIN_RECIP: case MPC_PLAIN_RSQRT: {
        const mpc_nr_p* p = (const mpc_nr_p*)knobs;
        if (!nr_ok(p)) return fail(c, MPC_ERR_RANGE, "NR knobs");
        a.op = op == MPC_PLAIN_RECIP ? 1 : 2; a.nk = mk_nr(p); break;
    }
    case MPC_PLAIN_GELU: case MPC_PLAIN_SILU: case MPC_PLAIN_SIGMOID:
        if ((st = act_knobs(c, op - MPC_PLAIN_GELU, (const mpc_act_p*)knobs, a.ak))) return st;
        a.op = 3; break;
    case MPC_PLAIN_SOFTMAX: {
        const mpc_softmax_p* p = (const mpc_softmax_p*)knobs;
        if (p->window < 1 || p->window > 64 || !exp_ok(&p->exp) || !nr_ok(&p->recip)) return fail(c, MPC_ERR_RANGE, "softmax knobs");
        if (p->causal != 0 && p->causal != 1) return fail(c, MPC_ERR_RANGE, "softmax knobs");
        a.op = 4; a.ek = mk_exp(&p->exp); a.nk = mk_nr(&p->recip); a.w = p->window; a.causal = p->causal; break;
    }
    case MPC_PLAIN_LAYERNORM: {
        const mpc_ln_p* p = (const mpc_ln_p*)knobs;
        if (!nr_ok(&p->rsqrt) || (p->mean_mode != 0 && p->mean_mode != 1)) return fail(c, MPC_ERR_RANGE, "layernorm knobs");
        a.op = 5; a.nk = mk_nr(&p->rsqrt); a.mean_mode = p->mean_mode; a.e_invd = E(1.0 / (double)cols); a.e_eps = E(p->eps);
        break;
    }
    default: return fail(c, MPC_ERR_RANGE, "plain_eval: unknown op");
    }
    if (rows == 0) return MPC_OK;
    const i64 work = a.op <= 3 ? rows * cols : rows;
    rec_begin(c, "plain_eval", (u64)(rows * cols));
    k_plain<<<grid_for(c, work, 256, 8), 256, 0, c->stream>>>(a);
    rec_end(c);
    c->st.launches++;
    rec_close(c);
    return cuda_check(c, "plain_eval");
}

mpc_status mpc_recip(mpc_ctx* c, mpc_shares x, mpc_shares z, int64_t n, int64_t off, const mpc_nr_p* p) { return nr_common<0>(c, x, z, n, off, p); }
mpc_status mpc_rsqrt(mpc_ctx* c, mpc_shares x, mpc_shares z, int64_t n, int64_t off, const mpc_nr_p* p) { return nr_common<1>(c, x, z, n, off, p); }
mpc_status mpc_gelu(mpc_ctx* c, mpc_shares x, mpc_shares z, int64_t n, int64_t off, const mpc_act_p* p) { return act_common(c, 0, x, z, n, off, p); }
mpc_status mpc_silu(mpc_ctx* c, mpc_shares x, mpc_shares z, int64_t n, int64_t off, const mpc_act_p* p) { return act_common(c, 1, x, z, n, off, p); }
mpc_status mpc_sigmoid(mpc_ctx* c, mpc_shares x, mpc_shares z, int64_t n, int64_t off, const mpc_act_p* p) { return act_common(c, 2, x, z, n, off, p); }

// ---- row ops (fused, one CTA per 32-row tile) ---------------------------------------------------
mpc_status mpc_max(mpc_ctx* c, mpc_shares x, mpc_shares z, int64_t rows, int64_t cols, int64_t row_off, int w)
{
    if (!c) return MPC_ERR_INVALID;
    const u64 steps = 2ull * (u64)max_levels_h(cols);
    mpc_status st = begin(c, steps);
    if (st) return st;
    if (w < 1 || w > 64) return fail(c, MPC_ERR_RANGE, "window");
    if (bad_sh(c, x) || bad_sh(c, z) || rows < 0 || cols < 1 || row_off < 0 || (row_off & 31))
        return fail(c, MPC_ERR_INVALID, "max args (row_off % 32)");
    if (rows > 0 && cols <= MAXS_COLS) {
        MaxSmallArgs a{};
        a.s = (u32)c->step; a.w = w; a.x = spv(c, x); a.z = sov(c, z); a.rows = rows; a.cols = cols;
        a.row_off = (u64)row_off; a.pool = 0;
        st = launch_max_small(c, a, "max");
        if (st) return st;
        acct_max(c, rows, cols, w);
    } else if (rows > 0) {
        MaxArgs a{(u32)c->step, w, spv(c, x), sov(c, z), rows, cols, (u64)row_off, nullptr, 0, 0, nullptr,
                  use_cone(c, w) ? 1 : 0, tail_half()};
        st = launch_max(c, a, rows, cols, w, "max");
        if (st) return st;
        acct_max(c, rows, cols, w);
    }
    finish(c, steps);
    return MPC_OK;
}

mpc_status mpc_maxpool2d(mpc_ctx* c, mpc_shares x, mpc_shares z, int N, int C, int H, int W,
                         int k, int stride, int pad, int64_t img_off, int w)
{
    if (!c) return MPC_ERR_INVALID;
    if (k < 1 || stride < 1 || pad < 0 || pad >= k || N < 0 || C < 1 || H < 1 || W < 1)
        return fail(c, MPC_ERR_INVALID, "maxpool shape");
    const int Ho = (H + 2 * pad - k) / stride + 1, Wo = (W + 2 * pad - k) / stride + 1;
    if (Ho < 1 || Wo < 1) return fail(c, MPC_ERR_INVALID, "maxpool output empty");
    const i64 rows = (i64)N * C * Ho * Wo, cols = (i64)k * k;
    const u64 steps = 2ull * (u64)max_levels_h(cols);
    mpc_status st = begin(c, steps);
    if (st) return st;
    if (w < 1 || w > 64) return fail(c, MPC_ERR_RANGE, "window");
    const u64 row_off = (u64)img_off * (u64)C * (u64)Ho * (u64)Wo;
    if (bad_sh(c, x) || bad_sh(c, z) || img_off < 0 || (row_off & 31)) return fail(c, MPC_ERR_INVALID, "maxpool args");
    if (max_work_u64(cols) * 8 > (i64)SMEM_LIMIT) return fail(c, MPC_ERR_UNSUPPORTED, "pool window too large");
    if (rows > 0 && cols <= MAXS_COLS && rows < (1ll << 31) && (i64)N * C * H * W < (1ll << 40)) {
        MaxSmallArgs a{};
        a.s = (u32)c->step; a.w = w; a.x = spv(c, x); a.z = sov(c, z); a.rows = rows; a.cols = cols;
        a.row_off = row_off; a.pool = 1; a.k = k; a.stride = stride; a.pad = pad; a.H = H; a.W = W;
        a.fk = make_fastdiv((u32)k); a.fwo = make_fastdiv((u32)Wo); a.fho = make_fastdiv((u32)Ho);
        st = launch_max_small(c, a, "maxpool");
        if (st) return st;
        acct_max(c, rows, cols, w);
    } else if (rows > 0) {
        // gather the windows (public zero padding) into rows, then the fused row max
        const size_t gb = sizeof(u64) * (size_t)(rows * cols);
        u64* Rw = (u64*)scratch(c, 2 * gb);
        if (!Rw) return fail(c, MPC_ERR_NOMEM, "maxpool scratch");
        SO rowsbuf = sov(c, mpc_shares{{Rw, Rw + rows * cols}});
        if (!is_dealer(c)) {
        rec_begin(c, "pool_gather", (u64)rows);
        k_pool_gather<<<grid_for(c, rows * cols, TPB, 16), TPB, 0, c->stream>>>(spv(c, x), rowsbuf, N, C, H, W, k, stride, pad, Ho, Wo);
        rec_end(c);
        c->st.launches++;
        if ((st = cuda_check(c, "pool_gather"))) return st;
        }
        MaxArgs a{(u32)c->step, w, SP{{rowsbuf.p[0], rowsbuf.p[1]}}, sov(c, z), rows, cols, row_off, nullptr, 0, 0,
                  nullptr, use_cone(c, w) ? 1 : 0, tail_half()};
        st = launch_max(c, a, rows, cols, w, "maxpool");
        if (st) return st;
        acct_max(c, rows, cols, w);
    }
    finish(c, steps);
    return MPC_OK;
}

static mpc_status softmax_core(mpc_ctx* c, mpc_shares x, mpc_shares z, int64_t rows, int64_t cols, int64_t row_off,
                               const mpc_softmax_p* p, u32 s0, int bal_default = 2);
static void acct_softmax(mpc_ctx* c, int64_t rows, int64_t cols, const mpc_softmax_p* p);

mpc_status mpc_softmax(mpc_ctx* c, mpc_shares x, mpc_shares z, int64_t rows, int64_t cols, int64_t row_off,
                       const mpc_softmax_p* p)
{
    if (!c) return MPC_ERR_INVALID;
    if (!p || p->window < 1 || p->window > 64 || !exp_ok(&p->exp) || !nr_ok(&p->recip) ||
        (p->causal != 0 && p->causal != 1))
        return fail(c, MPC_ERR_RANGE, "softmax knobs");
    const int L = max_levels_h(cols);
    const u64 steps = 2ull * (u64)L + exp_steps_h(&p->exp) + exp_steps_h(&p->recip.exp) + 2ull * (u64)p->recip.iters + 1;
    mpc_status st = begin(c, steps);
    if (st) return st;
    if (bad_sh(c, x) || bad_sh(c, z) || rows < 0 || cols < 1 || row_off < 0 || (row_off & 31))
        return fail(c, MPC_ERR_INVALID, "softmax args (row_off % 32)");
    if (rows > 0) {
        if ((st = softmax_core(c, x, z, rows, cols, row_off, p, (u32)c->step))) return st;
        acct_softmax(c, rows, cols, p);
    }
    finish(c, steps);
    return MPC_OK;
}

// The two parties' copies of one chunk and direction as ONE DMA submission: with both PCIe directions
// busy, every separate cudaMemcpyAsync costs ~9 us of link time (tools/pcie_copy.cu: cfg2, 4 chunks x
// 2 parties both ways).  The two chunks are the two rows of a pitched 2D copy when each side's party
// arrays are one allocation: the device staging always is, the host arrays when they are ADJACENT
// (party 1's array starts right after party 0's, e.g. one pinned [2][n] tensor: pitch == adj bytes;
// the driver refuses a pitch that spans two allocations).  Otherwise one copy per party.
static void copy_pair(void** dst, void** src, size_t bytes, int n, cudaStream_t s, cudaMemcpyKind kind,
                      size_t host_adj)
{
    if (n == 2) {
        const char *d0 = (const char*)dst[0], *d1 = (const char*)dst[1];
        const char *s0 = (const char*)src[0], *s1 = (const char*)src[1];
        const int64_t dp = d1 - d0, sp = s1 - s0, lim = (int64_t)1 << 31;
        const int64_t hp = kind == cudaMemcpyHostToDevice ? sp : dp;      // the host side's pitch
        if (hp == (int64_t)host_adj && dp >= (int64_t)bytes && sp >= (int64_t)bytes && dp < lim && sp < lim) {
            if (cudaMemcpy2DAsync(dst[0], (size_t)dp, src[0], (size_t)sp, bytes, 2, kind, s) == cudaSuccess) return;
            cudaGetLastError();                    // pitch not accepted: fall back to single copies
        }
    }
    for (int q = 0; q < n; ++q) cudaMemcpyAsync(dst[q], src[q], bytes, kind, s);
}

// pipelined host-buffer softmax (see HostIO): same steps, units and output shares as mpc_softmax
mpc_status mpc_softmax_hostio(mpc_ctx* c, mpc_shares hx, mpc_shares hz, int64_t rows, int64_t cols, int64_t row_off,
                              const mpc_softmax_p* p, int64_t chunk_rows)
{
    if (!c) return MPC_ERR_INVALID;
    if (!p || p->window < 1 || p->window > 64 || !exp_ok(&p->exp) || !nr_ok(&p->recip) ||
        (p->causal != 0 && p->causal != 1))
        return fail(c, MPC_ERR_RANGE, "softmax knobs");
    const int L = max_levels_h(cols);
    const u64 steps = 2ull * (u64)L + exp_steps_h(&p->exp) + exp_steps_h(&p->recip.exp) + 2ull * (u64)p->recip.iters + 1;
    mpc_status st = begin(c, steps);
    if (st) return st;
    if (bad_sh(c, hx) || bad_sh(c, hz) || rows < 0 || cols < 1 || row_off < 0 || (row_off & 31) ||
        chunk_rows < 0 || (chunk_rows > 0 && chunk_rows < 32) || (chunk_rows & 31))
        return fail(c, MPC_ERR_INVALID, "softmax_hostio args (row_off, chunk_rows % 32)");
    if (rows == 0) { finish(c, steps); return MPC_OK; }
    if (!c->hio) {
        HostIO* h = new HostIO();
        memset(h, 0, sizeof *h);
        cudaStreamCreateWithFlags(&h->h2d, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&h->d2h, cudaStreamNonBlocking);
        cudaEventCreateWithFlags(&h->start, cudaEventDisableTiming);
        const char* ev = getenv("MPC_HIO_SLOTS");
        h->nslots = ev ? std::max(1, std::min(HIO_SLOTS, atoi(ev))) : MPC_HIO_DEFAULT_SLOTS;
        for (int b = 0; b < h->nslots; ++b) {
            cudaStreamCreateWithFlags(&h->cs[b], cudaStreamNonBlocking);
            cudaEventCreateWithFlags(&h->in_ready[b], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&h->comp_done[b], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&h->out_done[b], cudaEventDisableTiming);
        }
        c->hio = h;
        if ((st = cuda_check(c, "hostio setup"))) return st;
    }
    HostIO* h = c->hio;
    const int parties[2] = {0, 1};
    const int np = c->cfg.mode == MPC_MODE_PAIR ? 1 : 2;
    const int p0 = c->cfg.mode == MPC_MODE_PAIR ? c->cfg.party : 0;
    // PAIR kernels own the per-warp exchange slots: their chunks run one after another
    const int nslots = is_pair(c) ? 1 : h->nslots;
    // chunk schedule: chunk_rows, or (0) four equal chunks -- measured best for cfg2 among 768..6144-row
    // chunks and a short-long-short ramp (tools/perf_e2e.py)
    std::vector<i64> sched;
    static const char* ramp = getenv("MPC_HIO_SCHED");   // experiments: explicit chunk list "r0,r1,..."
    if (ramp && chunk_rows == 0) {
        i64 r = 0;
        for (const char* q = ramp; *q && r < rows;) {
            const i64 v = std::max<i64>(32, strtoll(q, nullptr, 10) / 32 * 32);
            sched.push_back(std::min<i64>(v, rows - r));
            r += sched.back();
            while (*q && *q != ',') ++q;
            if (*q == ',') ++q;
        }
        while (!sched.empty() && r < rows) { sched.push_back(std::min<i64>(sched.back(), rows - r)); r += sched.back(); }
    }
    if (sched.empty()) {                                  // default (also for an empty / unparsable MPC_HIO_SCHED)
        const i64 cr = chunk_rows > 0 ? chunk_rows : std::max<i64>(32, ((rows + 3) / 4 + 31) / 32 * 32);
        for (i64 r = 0; r < rows; r += cr) sched.push_back(std::min<i64>(cr, rows - r));
    }
    i64 maxc = 0;
    for (i64 v : sched) maxc = std::max(maxc, v);
    const size_t half = sizeof(u64) * (size_t)maxc * (size_t)cols;             // one party, one array
    if (is_dealer(c)) {                                  // party 1's chunk computes, no copies
        i64 rr = 0;
        const mpc_shares none{{nullptr, nullptr}};
        for (i64 v : sched) {
            if ((st = softmax_core(c, none, none, v, cols, row_off + rr, p, (u32)c->step))) return st;
            rr += v;
        }
        acct_softmax(c, rows, cols, p);
        finish(c, steps);
        return MPC_OK;
    }
    cudaStream_t user = c->stream;
    cudaEventRecord(h->start, user);
    cudaStreamWaitEvent(h->h2d, h->start, 0);
    // MPC_HIO_TRACE=1 (diagnostics only): per-chunk timeline of the copies and the compute on stderr
    static const bool trace = getenv("MPC_HIO_TRACE") != nullptr;
    std::vector<cudaEvent_t> tev;
    auto mark = [&](cudaStream_t s) {
        if (!trace) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, s);
        tev.push_back(e);
    };
    mark(h->h2d);
    const u32 s0 = (u32)c->step;
    const i64 nchunks = (i64)sched.size();
    i64 r0 = 0;
    for (i64 i = 0; i < nchunks; r0 += sched[(size_t)i], ++i) {
        const int b = (int)(i % h->nslots);
        const int cb = (int)(i % nslots);
        const i64 ri = sched[(size_t)i];
        const size_t bytes = sizeof(u64) * (size_t)(ri * cols);
        if (!h->dbuf[b] || h->dbuf_bytes[b] < 4 * half) {
            if (h->dbuf[b]) { cudaStreamSynchronize(h->d2h); cudaFree(h->dbuf[b]); }
            if (cudaMalloc(&h->dbuf[b], 4 * half) != cudaSuccess) { h->dbuf[b] = nullptr; return fail(c, MPC_ERR_NOMEM, "hostio staging"); }
            h->dbuf_bytes[b] = 4 * half;
        }
        u64* dx[2] = {h->dbuf[b], h->dbuf[b] + half / 8};
        u64* dz[2] = {h->dbuf[b] + 2 * (half / 8), h->dbuf[b] + 3 * (half / 8)};
        if (h->used[b]) cudaStreamWaitEvent(h->h2d, h->out_done[b], 0);
        mark(h->h2d);
        {
            void* dst[2]; void* src[2];
            for (int q = 0; q < np; ++q) { dst[q] = dx[parties[p0 + q]]; src[q] = hx.sh[parties[p0 + q]] + r0 * cols; }
            copy_pair(dst, src, bytes, np, h->h2d, cudaMemcpyHostToDevice, sizeof(u64) * (size_t)(rows * cols));
        }
        cudaEventRecord(h->in_ready[b], h->h2d);
        mark(h->h2d);
        cudaStreamWaitEvent(h->cs[cb], h->in_ready[b], 0);
        mark(h->cs[cb]);
        // launch on the slot's stream with the slot's own scratch
        void* save_scr = c->scratch; size_t save_bytes = c->scratch_bytes;
        c->stream = h->cs[cb]; c->scratch = h->scr[cb]; c->scratch_bytes = h->scr_bytes[cb];
        mpc_shares xs{{dx[0], dx[1]}}, zs{{dz[0], dz[1]}};
        if (c->cfg.mode == MPC_MODE_PAIR) { xs.sh[1 - c->cfg.party] = nullptr; zs.sh[1 - c->cfg.party] = nullptr; }
        // (the chunks' kernels take the balanced plan too: cfg2 in 1536-row chunks 0.716-0.730 ms vs
        // 0.756-0.768 for 3072-row chunks on 32-row tiles -- the pipeline's head and tail are one chunk's
        // latency; 3072-row chunks on the balanced plan 0.82 ms: concurrent chunks then contend,
        // tools/ab_hostio.py, r02)
        st = softmax_core(c, xs, zs, ri, cols, row_off + r0, p, s0, 2);
        h->scr[cb] = c->scratch; h->scr_bytes[cb] = c->scratch_bytes;
        c->scratch = save_scr; c->scratch_bytes = save_bytes; c->stream = user;
        if (st) return st;
        cudaEventRecord(h->comp_done[b], h->cs[cb]);
        mark(h->cs[cb]);
        cudaStreamWaitEvent(h->d2h, h->comp_done[b], 0);
        mark(h->d2h);
        {
            void* dst[2]; void* src[2];
            for (int q = 0; q < np; ++q) { dst[q] = hz.sh[parties[p0 + q]] + r0 * cols; src[q] = dz[parties[p0 + q]]; }
            copy_pair(dst, src, bytes, np, h->d2h, cudaMemcpyDeviceToHost, sizeof(u64) * (size_t)(rows * cols));
        }
        cudaEventRecord(h->out_done[b], h->d2h);
        mark(h->d2h);
        h->used[b] = true;
    }
    cudaEventRecord(h->start, h->d2h);
    cudaStreamWaitEvent(user, h->start, 0);          // the call completes in the caller's stream order
    if (trace) {
        cudaDeviceSynchronize();
        fprintf(stderr, "hostio trace (ms from start): chunk rows | h2d start end | comp start end | d2h start end\n");
        for (i64 i = 0; i < nchunks; ++i) {
            float t[6];
            for (int j = 0; j < 6; ++j) cudaEventElapsedTime(&t[j], tev[0], tev[1 + 6 * (size_t)i + j]);
            fprintf(stderr, "  %3lld %5lld | %.3f %.3f | %.3f %.3f | %.3f %.3f\n", (long long)i, (long long)sched[(size_t)i],
                    t[0], t[1], t[2], t[3], t[4], t[5]);
        }
        for (cudaEvent_t e : tev) cudaEventDestroy(e);
    }
    if ((st = cuda_check(c, "softmax_hostio"))) return st;
    acct_softmax(c, rows, cols, p);
    finish(c, steps);
    return MPC_OK;
}

static mpc_status softmax_core(mpc_ctx* c, mpc_shares x, mpc_shares z, int64_t rows, int64_t cols, int64_t row_off,
                               const mpc_softmax_p* p, u32 s0, int bal_default)
{
    const int L = max_levels_h(cols);
    mpc_status st;
    {
        SoftmaxArgs a;
        a.s_max = s0;
        a.s_exp = a.s_max + 2u * (u32)L;
        a.s_rec = a.s_exp + (u32)exp_steps_h(&p->exp);
        a.s_mul = a.s_rec + (u32)exp_steps_h(&p->recip.exp) + 2u * (u32)p->recip.iters;
        a.w = p->window; a.ek = mk_exp(&p->exp); a.rk = mk_nr(&p->recip);
        a.x = spv(c, x); a.z = sov(c, z);
        a.rows = rows; a.cols = cols; a.row_off = (u64)row_off;
        a.cone = use_cone(c, p->window) ? 1 : 0;
        a.bcast = p->bcast ? 1 : 0;
        a.causal = p->causal ? 1 : 0;
        a.causal_L = p->window >= 2 ? 0ull - (1ull << (p->window - 2)) : 0ull - 1ull;   // public -2^(w-2)
        // half tiles start at row 16 mod 32: not with a clamp in the reciprocal's exp (an LTZ over the
        // tile's row units) nor a clamped exp over odd rows (element groups would start mid-group)
        a.half = (tail_half() && !p->recip.exp.clamp && !(p->exp.clamp && (cols & 1))) ? 1 : 0;
        const bool wide = p->window > 33 || p->exp.window > 33 || p->recip.exp.window > 33;
        // E in shared memory when the whole work tile fits 100 KB (two CTAs per SM): cols <= 192
#ifndef MPC_SOFTMAX_ESMEM
#define MPC_SOFTMAX_ESMEM 1
#endif
        a.esmem = (MPC_SOFTMAX_ESMEM && softmax_work_u64(cols, true) * 8 <= 100 * 1024) ? 1 : 0;
        // BOTH with E in shared memory and no clamp in the reciprocal's exp: the NR chain's triples
        // are pre-generated by every warp into a shared-memory table (kernels.cuh nr_pregen)
#ifndef MPC_SOFTMAX_NRTAB
#define MPC_SOFTMAX_NRTAB 1
#endif
        const int nsteps = nr_tab_steps(0, p->recip.exp.t, p->recip.iters);
        // (not with the carry cone: its 16 KB of static shared memory would leave one CTA per SM)
        a.nrtab = (MPC_SOFTMAX_NRTAB && !is_pair(c) && a.esmem && !p->recip.exp.clamp && !a.cone &&
                   nsteps <= MPC_NR_TAB_MAX_STEPS) ? 1 : 0;
        const i64 tab = a.nrtab ? (i64)nsteps * NR_TAB_F * 32 : 0;
        // BOTH split form: the max tree as its own launch (k_max on the balanced plan: one range of ~rows /
        // grid rows per CTA, the rebalanced w = 33 LTZ), then exp / row sums / reciprocal / product
        // (kernels.cuh k_softmax_rest) on row blocks that are all resident at once, compiled for 3 CTAs
        // per SM: the fused kernel's 127 registers (the LTZ's) hold its exp phase to 16 warps per SM,
        // where the standalone exp kernel (80 registers, 24 warps) runs at 0.77 of the ALU peak.  One
        // timing record spans both launches.  MPC_SOFTMAX_SPLIT=0 / 1 in the environment (per call).
#ifndef MPC_SOFTMAX_SPLIT
#define MPC_SOFTMAX_SPLIT 0
#endif
        const char* split_env = getenv("MPC_SOFTMAX_SPLIT");
        const int split = split_env ? atoi(split_env) : MPC_SOFTMAX_SPLIT;
        if (split && !is_pair(c) && !a.causal && !a.bcast && !p->exp.clamp && !p->recip.exp.clamp &&
            !a.cone && !wide && !(cols & 1) && nsteps <= MPC_NR_TAB_MAX_STEPS && rows >= 2) {
            const int tabw = nsteps * NR_TAB_F * 32;
            static DevCache occ, occm;
            const int per_sm = dev_cached(occ, c->cfg.device, [&] {
                cudaFuncSetAttribute(k_softmax_rest<BothA>, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
                return occupancy(k_softmax_rest<BothA>, sizeof(u64) * (size_t)smr_smem_u64(tabw, 1), MPC_ROW_TPB);
            });
            const int per_sm_m = dev_cached(occm, c->cfg.device, [&] {
                cudaFuncSetAttribute(k_max<0, BothA>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
                return occupancy(k_max<0, BothA>, 100 * 1024, MPC_ROW_TPB);
            });
            const i64 slots = (i64)c->sm_count * per_sm;
            i64 rb = (rows + slots - 1) / slots;
            rb = std::max<i64>(2, std::min<i64>(64, (rb + 1) / 2 * 2));
            const i64 nblk = (rows + rb - 1) / rb;
            const int grid = (int)std::min<i64>(nblk, slots);
            const int ntab = rb > 32 ? 2 : 1;
            const size_t dyn = sizeof(u64) * (size_t)smr_smem_u64(tabw, ntab);
            i64 gm = std::max<i64>(1, std::min<i64>((i64)c->sm_count * per_sm_m, rows / 2));
            if (const char* cap = getenv("MPC_ROW_GRID_CAP")) { const int g = atoi(cap); if (g > 0 && g < gm) gm = g; }
            const i64 tr = 2 * (((rows + 1) / 2 + gm - 1) / gm), wkm = max_work_u64(cols, tr);
            if (tr <= 64 && wkm * 8 <= 100 * 1024) {
                // scratch: row maxima (2 x rows) then the per-CTA E tiles
                u64* sc = (u64*)scratch(c, sizeof(u64) * (size_t)(2 * rows + (i64)grid * 2 * rb * cols));
                if (!sc) return fail(c, MPC_ERR_NOMEM, "softmax scratch");
                MaxArgs ma{a.s_max, a.w, a.x, SO{{sc, sc + rows}}, rows, cols, (u64)row_off, nullptr, wkm, 1, nullptr, 0};
                ma.tr = (int)tr;
                cudaFuncSetAttribute(k_max<0, BothA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(wkm * 8));
                cudaFuncSetAttribute(k_softmax_rest<BothA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
                SmRestArgs ra{a.s_exp, a.s_rec, a.s_mul, a.ek, a.rk, a.x, SP{{sc, sc + rows}}, a.z, rows, cols, (u64)row_off,
                              (int)rb, sc + 2 * rows, tabw};
                rec_begin(c, "softmax", (u64)rows);
                k_max<0, BothA><<<(int)gm, MPC_ROW_TPB, wkm * 8, c->stream>>>(BothA{c->K}, ma);
                k_softmax_rest<BothA><<<grid, MPC_ROW_TPB, dyn, c->stream>>>(BothA{c->K}, ra);
                rec_end(c);
                c->st.launches += 2;
                return cuda_check(c, "softmax");
            }
        }
        a.bal = 0; a.tr = 32; a.tab_u64 = tab; a.nrange = 0;
        // BOTH balanced plan (kernels.cuh softmax_bal_*): when the 32-row tiles need more than one round,
        // ONE row range of ~rows / grid rows per CTA, every CTA resident at once
        const char* bal_env = getenv("MPC_SOFTMAX_BAL");      // 0: off (A/B, tests; read per call)
        // (the carry cone too, w <= 33: its 16 KB of static shared memory beside the 74 KB work area still
        // leaves two CTAs per SM; the triple tables alias the level buffers, so no esmem condition)
        const bool bal_tab = !p->recip.exp.clamp && nsteps <= MPC_NR_TAB_MAX_STEPS;
        // (a clamped exp's LTZ groups are element groups from g0 cols: whole groups iff 32 | g0 cols, and the
        // plan's g0 are even, so cols % 16 == 0)
        // Rows whose level buffers do not fit shared memory (cols > 192, e.g. GPT-2's 1024) keep them in a
        // per-CTA global work area (L2) and only the two triple tables in shared memory ("gwork").
        const char* balw_env = getenv("MPC_SOFTMAX_BAL_WIDE");
        const bool gwork_ok = !(balw_env && atoi(balw_env) == 0);
        if (!(bal_env && atoi(bal_env) == 0) && !is_pair(c) && !wide && (!p->exp.clamp || cols % 16 == 0) && bal_tab &&
            (cols <= 192 || gwork_ok)) {
            static DevCache occb, occc;
            const int per_sm = a.cone ? dev_cached(occc, c->cfg.device, [] {
                cudaFuncSetAttribute(k_softmax<2, BothA>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
                return occupancy(k_softmax<2, BothA>, 80 * 1024, MPC_ROW_TPB);
            }) : dev_cached(occb, c->cfg.device, [] {
                cudaFuncSetAttribute(k_softmax<0, BothA>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
                return occupancy(k_softmax<0, BothA>, 100 * 1024, MPC_ROW_TPB);
            });
            const i64 tab = (i64)nsteps * NR_TAB_F * 32;
            // CTAs per SM: the most whose work areas fit (the query above assumed 100 KB each)
            int ps = per_sm;
            {
                auto kq = a.cone ? k_softmax<2, BothA> : k_softmax<0, BothA>;
                static DevCache occr0, occr2;                  // register / thread limit (no shared memory)
                const int ps_max = dev_cached(a.cone ? occr2 : occr0, c->cfg.device, [&] { return occupancy(kq, 0, MPC_ROW_TPB); });
                for (int k = ps_max; k > per_sm; --k) {
                    const i64 g = (i64)c->sm_count * k, t = 2 * (((rows + 1) / 2 + g - 1) / g);
                    const size_t d = sizeof(u64) * (size_t)softmax_bal_work_u64(cols, t, (i64)nsteps * NR_TAB_F * 32);
                    if (d <= 100 * 1024) {
                        cudaFuncSetAttribute(kq, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d);
                        if (occupancy(kq, d, MPC_ROW_TPB) >= k) { ps = k; break; }
                    }
                }
            }
            i64 grid = (i64)c->sm_count * ps;
            if (const char* cap = getenv("MPC_ROW_GRID_CAP")) { const int g = atoi(cap); if (g > 0 && g < grid) grid = g; }
            // 2 (default): always, on min(grid, rows / 2) CTAs (>= 2 rows each) -- fewer rows per CTA
            // means a shorter critical path (1024 rows: 0.050 vs 0.113 ms on 32 tiles; 3072: 0.089 vs
            // 0.115; 8192: 0.172 vs 0.186, tools/ab_rows.py, r02) for more LTZ groups shared at range
            // boundaries; 1: only when the 32-row tiles need more than one round (the host-buffer chunks)
            const int bal_mode = bal_env ? atoi(bal_env) : bal_default;
            if (bal_mode >= 3) grid = std::max<i64>(1, grid / 2);   // 3: one CTA per SM (concurrent chunks)
            if (bal_mode >= 2) grid = std::max<i64>(1, std::min<i64>(grid, rows / 2));
            const i64 hr = (rows + 1) / 2;
            // rows that would exceed 64 per CTA (shared-memory work area) run as k equal rounds of ranges
            // per CTA (nrange = k x grid): still one balanced plan, 32768 rows = 2 rounds of 55-56 rows
            i64 nrange = grid;
            if (cols <= 192 && hr > 32 * grid) nrange = grid * ((hr + 32 * grid - 1) / (32 * grid));
            const i64 tr = 2 * ((hr + nrange - 1) / nrange);
            const i64 wkb = softmax_bal_work_u64(cols, tr, tab);
            const bool want = bal_mode >= 2 ? true : rows > 32 * grid;
            a.nrange = nrange;
            // (up to 96 rows per CTA here: three 32-row tables, 107 KB of shared memory -- the 24576-row
            // GPT-2 shard of a pair has 84 rows per CTA)
            const i64 ntab = (tr + 31) / 32;
            const bool gwork = cols > 192 && gwork_ok && ntab * tab * 8 <= (a.cone ? 80 : 110) * 1024;
            if (want && tr <= 96 && gwork) {
                a.bal = 1; a.tr = (int)tr; a.esmem = 0; a.use_smem = 0; a.nrtab = 1; a.tab_u64 = tab;
                a.work_u64 = wkb;
                // scratch: [E tiles: 2 tr cols per CTA] [work areas: wkb per CTA]
                u64* esc = (u64*)scratch(c, sizeof(u64) * (size_t)((2 * tr * cols + wkb) * grid));
                if (!esc) return fail(c, MPC_ERR_NOMEM, "softmax scratch");
                a.escratch = esc;
                a.gscratch = esc + (size_t)(2 * tr * cols) * (size_t)grid;
                const size_t dyn = sizeof(u64) * (size_t)(ntab * tab);
                auto kb = a.cone ? (a.causal ? k_softmax<2, BothA, true> : k_softmax<2, BothA>)
                                 : (a.causal ? k_softmax<0, BothA, true> : k_softmax<0, BothA>);
                cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
                rec_begin(c, "softmax", (u64)rows);
                kb<<<(int)grid, MPC_ROW_TPB, dyn, c->stream>>>(BothA{c->K}, a);
                rec_end(c);
                c->st.launches++;
                return cuda_check(c, "softmax");
            }
            if (want && tr <= 64 && cols <= 192 && wkb * 8 <= (a.cone ? 80 : 100) * 1024) {
                a.bal = 1; a.tr = (int)tr; a.esmem = 0; a.use_smem = 1; a.nrtab = 1; a.tab_u64 = tab;
                a.gscratch = nullptr; a.work_u64 = wkb;
                u64* esc = (u64*)scratch(c, sizeof(u64) * (size_t)(2 * tr * cols * grid));
                if (!esc) return fail(c, MPC_ERR_NOMEM, "softmax scratch");
                a.escratch = esc;
                const size_t dyn = sizeof(u64) * (size_t)wkb;
                // every launch: launch_rows sets the same kernels' attribute to other tiles' sizes
                auto kb = a.cone ? (a.causal ? k_softmax<2, BothA, true> : k_softmax<2, BothA>)
                                 : (a.causal ? k_softmax<0, BothA, true> : k_softmax<0, BothA>);
                cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
                rec_begin(c, "softmax", (u64)rows);
                kb<<<(int)grid, MPC_ROW_TPB, dyn, c->stream>>>(BothA{c->K}, a);
                rec_end(c);
                c->st.launches++;
                return cuda_check(c, "softmax");
            }
        }
        // PAIR modes: the same balanced plan on min(CTAs, rows / 2) CTAs.  The ranges, groups and the
        // exchange sequence of CTA c depend only on (rows, grid), so party 0's CTA c, party 1's and the
        // dealer's pass run the same rows.  MPC_SOFTMAX_BAL_PAIR=0: off (A/B; per call)
        const char* balp_env = getenv("MPC_SOFTMAX_BAL_PAIR");
        if (is_pair(c) && !(balp_env && atoi(balp_env) == 0) && !(bal_env && atoi(bal_env) == 0) && !wide && !a.cone &&
            (!p->exp.clamp || cols % 16 == 0) && !p->recip.exp.clamp) {
            const auto kk = a.causal ? kroles(k_softmax<0, PairA, true>, k_softmax<0, PairAS, true>)
                                     : kroles(k_softmax<0, PairA>, k_softmax<0, PairAS>);
            set_smem_attr(kk, 100 * 1024);
            i64 G = pair_ctas(c, kk, 100 * 1024, std::max<i64>(1, rows / 2), MPC_ROW_TPB);
            if (const char* cap = getenv("MPC_ROW_GRID_CAP")) { const int g = atoi(cap); if (g > 0 && g < G) G = g; }
            const i64 hr = (rows + 1) / 2, tr = 2 * ((hr + G - 1) / G);
            const i64 wkb = softmax_bal_work_u64(cols, tr, 0);
            if (tr <= 64 && wkb * 8 <= 100 * 1024) {
                a.bal = 1; a.tr = (int)tr; a.esmem = 0; a.use_smem = 1; a.nrtab = 0; a.tab_u64 = 0;
                a.gscratch = nullptr; a.work_u64 = wkb;
                const i64 launched = G * (is_loop(c) ? 2 : 1);
                u64* esc = (u64*)scratch(c, sizeof(u64) * (size_t)(2 * tr * cols * launched));
                if (!esc) return fail(c, MPC_ERR_NOMEM, "softmax scratch");
                a.escratch = esc;
                const size_t dyn = sizeof(u64) * (size_t)wkb;
                set_smem_attr(kk, (int)dyn);
                return launch_pair_kernel_tpb(c, kk, (int)G, dyn, MPC_ROW_TPB, "softmax", a);
            }
            // the level buffers in a per-CTA global work area when they do not fit (loopback's half grid at
            // cfg2: 84 rows per CTA; wide rows); no triple tables in PAIR, so up to 96 rows per CTA
            const char* balw = getenv("MPC_SOFTMAX_BAL_WIDE");
            if (tr <= 96 && !(balw && atoi(balw) == 0)) {
                a.bal = 1; a.tr = (int)tr; a.esmem = 0; a.use_smem = 0; a.nrtab = 0; a.tab_u64 = 0;
                a.work_u64 = wkb;
                const i64 launched = G * (is_loop(c) ? 2 : 1);
                u64* esc = (u64*)scratch(c, sizeof(u64) * (size_t)((2 * tr * cols + wkb) * launched));
                if (!esc) return fail(c, MPC_ERR_NOMEM, "softmax scratch");
                a.escratch = esc;
                a.gscratch = esc + (size_t)(2 * tr * cols) * (size_t)launched;
                return launch_pair_kernel_tpb(c, kk, (int)G, 0, MPC_ROW_TPB, "softmax", a);
            }
        }
        const i64 wk = softmax_work_u64(cols, a.esmem != 0, tab), ek = a.esmem ? 0 : 64 * cols;
        const size_t lim = a.esmem ? 100 * 1024 + (size_t)tab * 8 : SMEM_LIMIT;
        if (a.causal)   // causal instantiations: the dense kernels carry no mask code
            st = wide && a.cone ? launch_rows(c, k_softmax<3, BothA, true>, kroles(k_softmax<3, PairA, true>, k_softmax<3, PairAS, true>), a, rows, wk, ek, "softmax", lim)
               : wide ? launch_rows(c, k_softmax<1, BothA, true>, kroles(k_softmax<1, PairA, true>, k_softmax<1, PairAS, true>), a, rows, wk, ek, "softmax", lim)
               : a.cone ? launch_rows(c, k_softmax<2, BothA, true>, kroles(k_softmax<2, PairA, true>, k_softmax<2, PairAS, true>), a, rows, wk, ek, "softmax", lim)
                        : launch_rows(c, k_softmax<0, BothA, true>, kroles(k_softmax<0, PairA, true>, k_softmax<0, PairAS, true>), a, rows, wk, ek, "softmax", lim);
        else
            st = wide && a.cone ? launch_rows(c, k_softmax<3, BothA>, kroles(k_softmax<3, PairA>, k_softmax<3, PairAS>), a, rows, wk, ek, "softmax", lim)
               : wide ? launch_rows(c, k_softmax<1, BothA>, kroles(k_softmax<1, PairA>, k_softmax<1, PairAS>), a, rows, wk, ek, "softmax", lim)
               : a.cone ? launch_rows(c, k_softmax<2, BothA>, kroles(k_softmax<2, PairA>, k_softmax<2, PairAS>), a, rows, wk, ek, "softmax", lim)
                        : launch_rows(c, k_softmax<0, BothA>, kroles(k_softmax<0, PairA>, k_softmax<0, PairAS>), a, rows, wk, ek, "softmax", lim);
    }
    return st;
}

static void acct_softmax(mpc_ctx* c, int64_t rows, int64_t cols, const mpc_softmax_p* p)
{
    const i64 n = rows * cols;
    acct_max(c, rows, cols, p->window);
    acct_exp(c, (u64)n, &p->exp);
    acct_exp(c, (u64)rows, &p->recip.exp);
    for (int i = 0; i < 2 * p->recip.iters; ++i) acct_beaver(c, (u64)rows);
    if (p->bcast) acct_bcast(c, (u64)n, (u64)rows); else acct_beaver(c, (u64)n);
}

mpc_status mpc_layernorm(mpc_ctx* c, mpc_shares x, mpc_shares z, int64_t rows, int64_t cols, int64_t row_off,
                         const mpc_ln_p* p)
{
    if (!c) return MPC_ERR_INVALID;
    if (!p || !nr_ok(&p->rsqrt) || (p->mean_mode != 0 && p->mean_mode != 1)) return fail(c, MPC_ERR_RANGE, "layernorm knobs");
    const u64 steps = 1 + exp_steps_h(&p->rsqrt.exp) + 3ull * (u64)p->rsqrt.iters + 1;
    mpc_status st = begin(c, steps);
    if (st) return st;
    if (bad_sh(c, x) || bad_sh(c, z) || rows < 0 || cols < 1 || row_off < 0 || (row_off & 31))
        return fail(c, MPC_ERR_INVALID, "layernorm args (row_off % 32)");
    if (rows > 0) {
        LnArgs a;
        a.s_sq = (u32)c->step;
        a.s_rs = a.s_sq + 1;
        a.s_mul = a.s_rs + (u32)exp_steps_h(&p->rsqrt.exp) + 3u * (u32)p->rsqrt.iters;
        a.rk = mk_nr(&p->rsqrt);
        a.x = spv(c, x); a.z = sov(c, z);
        a.rows = rows; a.cols = cols; a.row_off = (u64)row_off;
        a.mean_mode = p->mean_mode; a.e_invd = E(1.0 / (double)cols); a.e_eps = E(p->eps);
        a.bcast = p->bcast ? 1 : 0;
        const i64 ntiles = (rows + 31) / 32;
        const bool wide = p->rsqrt.exp.window > 33;
#ifndef MPC_LN_QUAD
#define MPC_LN_QUAD 0      // warp-per-4-rows kernel: measured 9 % slower than the tile kernel (all warps hit
#endif                     // their rsqrt chains at once)
#ifndef MPC_LN_SPLIT
#define MPC_LN_SPLIT 1
#endif
#ifndef MPC_LN_FUSED
#define MPC_LN_FUSED 1
#endif
        const int nsteps_rs = nr_tab_steps(1, p->rsqrt.exp.t, p->rsqrt.iters);
        // BOTH: one warp per row (kernels.cuh k_ln_row) when its rows fill the warps' rounds evenly
        // (ceil(rows / warps) rounds at >= 90 % of the work, or one round); otherwise the row-block
        // kernel.  Measured (tools/ab_ln.py, r02): 24576 x 768 0.413 vs 0.447 ms, 1024 x 768 0.029 vs
        // 0.035; cfg5 8192 x 768 (3.46 rows per warp) 0.161 vs 0.148 -> k_ln_fused.  A warp's row is
        // latency-bound (fewer warps per CTA to even the rounds measured slower: 7 warps 0.162 ms)
        const char* lnr_env = getenv("MPC_LN_ROW");          // 0 / 1 force (A/B, tests); read per call
        bool ln_row = false;
        if (!is_pair(c) && !p->rsqrt.exp.clamp && !p->bcast && !(cols & 1) && nsteps_rs <= MPC_NR_TAB_MAX_STEPS) {
            static DevCache occr;
            const int per_sm = dev_cached(occr, c->cfg.device, [&] { return occupancy(k_ln_row<BothA>, 0, MPC_ROW_TPB); });
            const i64 nw = (i64)c->sm_count * per_sm * (MPC_ROW_TPB / 32), rounds = (rows + nw - 1) / nw;
            ln_row = rounds == 1 || (double)rows >= 0.9 * (double)(rounds * nw);
            if (lnr_env) ln_row = atoi(lnr_env) != 0;
        }
        // BOTH: row blocks staged in shared memory by double-buffered bulk copies (ln_blk.cuh): the
        // largest RB in {8, 4, 2, 1} whose two buffers fit 96 KB.  MPC_LN_BLK=0: off (A/B; per call)
        const char* lnb_env = getenv("MPC_LN_BLK");
        int lnb_rb = 0;
        // (cp.async.bulk needs 16-byte aligned sources: both share arrays' bases, cols even)
        const bool al16x = ((uintptr_t)a.x.p[0] % 16 == 0) && ((uintptr_t)a.x.p[1] % 16 == 0);
        if (!(lnb_env && atoi(lnb_env) == 0) && !is_pair(c) && !p->rsqrt.exp.clamp && !p->bcast && !(cols & 1) &&
            nsteps_rs <= MPC_NR_TAB_MAX_STEPS && al16x)
            for (int rb = 8; rb >= 1 && !lnb_rb; rb /= 2)
                if (lnb_smem_bytes(cols, rb) <= 96 * 1024) lnb_rb = rb;
        if (lnb_rb) {
            LnBArgs f{a.s_sq, a.s_rs, a.s_mul, a.rk, a.x, a.z, rows, cols, (u64)row_off, a.mean_mode, a.e_invd, a.e_eps,
                      lnb_rb};
            const size_t dyn = lnb_smem_bytes(cols, lnb_rb);
            static DevCache occb;
            const int per_sm = dev_cached(occb, c->cfg.device, [&] {
                cudaFuncSetAttribute(k_ln_blk<BothA>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
                return occupancy(k_ln_blk<BothA>, 96 * 1024, MPC_ROW_TPB);
            });
            cudaFuncSetAttribute(k_ln_blk<BothA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
            const i64 nblk = (rows + lnb_rb - 1) / lnb_rb;
            int grid = (int)std::min<i64>(nblk, (i64)c->sm_count * per_sm);
            if (const char* cap = getenv("MPC_ROW_GRID_CAP")) { const int g = atoi(cap); if (g > 0 && g < grid) grid = g; }
            rec_begin(c, "layernorm", (u64)rows);
            k_ln_blk<BothA><<<grid, MPC_ROW_TPB, dyn, c->stream>>>(BothA{c->K}, f);
            rec_end(c);
            c->st.launches++;
            st = cuda_check(c, "layernorm");
        } else if (ln_row) {
            LnRArgs f{a.s_sq, a.s_rs, a.s_mul, a.rk, a.x, a.z, rows, cols, (u64)row_off, a.mean_mode, a.e_invd, a.e_eps};
            static DevCache occ;
            const int per_sm = dev_cached(occ, c->cfg.device, [&] { return occupancy(k_ln_row<BothA>, 0, MPC_ROW_TPB); });
            const i64 nctas = (rows + MPC_ROW_TPB / 32 - 1) / (MPC_ROW_TPB / 32);
            const int grid = (int)std::min<i64>(nctas, (i64)c->sm_count * per_sm);
            rec_begin(c, "layernorm", (u64)rows);
            k_ln_row<BothA><<<grid, MPC_ROW_TPB, 0, c->stream>>>(BothA{c->K}, f);
            rec_end(c);
            c->st.launches++;
            st = cuda_check(c, "layernorm");
        } else if (MPC_LN_FUSED && !p->rsqrt.exp.clamp && !p->bcast && !(cols & 1) && rows * cols < (1ll << 31)) {
            // one launch, row blocks of RB rows with every block resident (kernels.cuh k_ln_fused)
            LnFArgs f{a.s_sq, a.s_rs, a.s_mul, a.rk, a.x, a.z, rows, cols, (u64)row_off, a.mean_mode, a.e_invd,
                      a.e_eps, 2, 0};
            f.nrtab = (!is_pair(c) && nsteps_rs <= MPC_NR_TAB_MAX_STEPS) ? 1 : 0;
            const size_t dyn = sizeof(u64) * (size_t)lnf_smem_u64(f.nrtab ? nsteps_rs : 0);
            auto rb_for = [&](i64 slots) {
                i64 rb = (rows + slots - 1) / std::max<i64>(1, slots);
                rb = std::max<i64>(2, std::min<i64>(32, (rb + 1) / 2 * 2));
                return (int)rb;
            };
            if (!is_pair(c)) {
                static DevCache occ;
                const int per_sm = dev_cached(occ, c->cfg.device, [&] {
                    cudaFuncSetAttribute(k_ln_fused<BothA>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
                    return occupancy(k_ln_fused<BothA>, 64 * 1024, MPC_ROW_TPB);
                });
                f.RB = rb_for((i64)c->sm_count * per_sm * MPC_LN_BLOCKS_PER_CTA);
                const i64 nblk = (rows + f.RB - 1) / f.RB;
                const int grid = (int)std::min<i64>(nblk, (i64)c->sm_count * per_sm);
                rec_begin(c, "layernorm", (u64)rows);
                k_ln_fused<BothA><<<grid, MPC_ROW_TPB, dyn, c->stream>>>(BothA{c->K}, f);
                rec_end(c);
                c->st.launches++;
                st = cuda_check(c, "layernorm");
            } else {
                const auto kk = kroles(k_ln_fused<PairA>, k_ln_fused<PairAS>);
                set_smem_attr(kk, 64 * 1024);
                f.RB = rb_for(pair_ctas(c, kk, dyn, 1ll << 40, MPC_ROW_TPB) * MPC_LN_BLOCKS_PER_CTA);
                const i64 nblk = (rows + f.RB - 1) / f.RB;
                st = launch_pair_kernel_tpb(c, kk, pair_ctas(c, kk, dyn, nblk, MPC_ROW_TPB), dyn, MPC_ROW_TPB,
                                            "layernorm", f);
            }
        } else if (MPC_LN_SPLIT && !p->rsqrt.exp.clamp && rows * cols < (1ll << 31)) {
            // three launches: per-row stats, the row rsqrt (element-wise NR kernel), the product
            u64* sc = (u64*)scratch(c, sizeof(u64) * (size_t)rows * (6 + 6));
            if (!sc) return fail(c, MPC_ERR_NOMEM, "layernorm scratch");
            const SO MU{{sc, sc + rows}}, VR{{sc + 2 * rows, sc + 3 * rows}}, RS{{sc + 4 * rows, sc + 5 * rows}};
            u64* br = sc + 6 * rows;                                     // broadcast-triple row records
            LnStatsArgs sa{a.s_sq, a.x, MU, VR, rows, cols, (u64)row_off, a.mean_mode, a.e_invd, a.e_eps};
            const i64 nw = rows;                                        // warps of work
            if (!is_pair(c)) {
                static DevCache occ;
                const int per_sm = dev_cached(occ, c->cfg.device, [] { return occupancy(k_ln_stats<BothA>); });
                rec_begin(c, "ln_stats", (u64)rows);
                k_ln_stats<BothA><<<grid_for(c, nw * 32, TPB, per_sm), TPB, 0, c->stream>>>(BothA{c->K}, sa);
                rec_end(c);
                c->st.launches++;
                st = cuda_check(c, "ln_stats");
            } else {
                st = launch_pair_kernel(c, kroles(k_ln_stats<PairA>, k_ln_stats<PairAS>), pair_ctas(c, kroles(k_ln_stats<PairA>, k_ln_stats<PairAS>), 0, (nw * 32 + TPB - 1) / TPB),
                                        0, "ln_stats", sa);
            }
            if (st) return st;
            const SP VRc{{VR.p[0], VR.p[1]}}, MUc{{MU.p[0], MU.p[1]}}, RSc{{RS.p[0], RS.p[1]}};
            if ((st = launch_pairs(c, rows, (u64)row_off, NrPairBody<1>{a.s_rs, a.rk, VRc, RS, rows}, "ln_rsqrt"))) return st;
            const i64 n = rows * cols;
            if (a.bcast) {
                BmbRowsArgs ra{a.s_mul, RSc, rows, (u64)row_off, br, is_loop(c) ? 1 : 0};
                const i64 nw2 = (rows + 31) / 32;
                if (!is_pair(c)) {
                    rec_begin(c, "bcast_rows", (u64)rows);
                    k_bmb_rows<BothA><<<grid_for(c, nw2 * 32, TPB, 8), TPB, 0, c->stream>>>(BothA{c->K}, ra);
                    rec_end(c);
                    c->st.launches++;
                    st = cuda_check(c, "bcast_rows");
                } else {
                    st = launch_pair_kernel(c, kroles(k_bmb_rows<PairA>, k_bmb_rows<PairAS>), pair_ctas(c, kroles(k_bmb_rows<PairA>, k_bmb_rows<PairAS>), 0, (nw2 * 32 + TPB - 1) / TPB),
                                            0, "bcast_rows", ra);
                }
                if (st) return st;
                st = launch_pairs(c, n, (u64)row_off * (u64)cols,
                                  BmbBody{a.s_mul, a.x, a.z, n, make_fastdiv((u32)cols), br, rows, FRAC, is_loop(c) ? 1 : 0,
                                          MUc, 1}, "ln_out");
            } else {
                st = launch_pairs(c, n, (u64)row_off * (u64)cols,
                                  LnOutBody{a.s_mul, a.x, a.z, n, make_fastdiv((u32)cols), MUc, RSc}, "ln_out");
            }
        } else if (MPC_LN_QUAD && !p->rsqrt.exp.clamp) {
            // warp-granular kernel (no clamp: the rsqrt has no LTZ, so rows need no 32-row grouping)
            const i64 nctas = ((rows + 3) / 4 + NWARPS - 1) / NWARPS;
            if (!is_pair(c)) {
                static DevCache occ;
                const int per_sm = dev_cached(occ, c->cfg.device, [] { return occupancy(k_ln_quad<false, BothA>, 0, MPC_ROW_TPB); });
                const int grid = (int)std::min<i64>(nctas, (i64)c->sm_count * per_sm);
                rec_begin(c, "layernorm", (u64)rows);
                k_ln_quad<false, BothA><<<grid, MPC_ROW_TPB, 0, c->stream>>>(BothA{c->K}, a);
                rec_end(c);
                c->st.launches++;
                st = cuda_check(c, "layernorm");
            } else {
                st = launch_pair_kernel_tpb(c, kroles(k_ln_quad<false, PairA>, k_ln_quad<false, PairAS>), pair_ctas(c, kroles(k_ln_quad<false, PairA>, k_ln_quad<false, PairAS>), 0, nctas, MPC_ROW_TPB),
                                            0, MPC_ROW_TPB, "layernorm", a);
            }
        } else if (!is_pair(c)) {
            const int grid = (int)std::min<i64>(ntiles, (i64)c->sm_count * occupancy(wide ? k_ln<true, BothA> : k_ln<false, BothA>, 0, MPC_ROW_TPB));
            rec_begin(c, "layernorm", (u64)rows);
            if (wide) k_ln<true, BothA><<<grid, MPC_ROW_TPB, 0, c->stream>>>(BothA{c->K}, a);
            else k_ln<false, BothA><<<grid, MPC_ROW_TPB, 0, c->stream>>>(BothA{c->K}, a);
            rec_end(c);
            c->st.launches++;
            st = cuda_check(c, "layernorm");
        } else if (wide) {
            st = launch_pair_kernel_tpb(c, kroles(k_ln<true, PairA>, k_ln<true, PairAS>), pair_ctas(c, kroles(k_ln<true, PairA>, k_ln<true, PairAS>), 0, ntiles, MPC_ROW_TPB), 0, MPC_ROW_TPB, "layernorm", a);
        } else {
            st = launch_pair_kernel_tpb(c, kroles(k_ln<false, PairA>, k_ln<false, PairAS>), pair_ctas(c, kroles(k_ln<false, PairA>, k_ln<false, PairAS>), 0, ntiles, MPC_ROW_TPB), 0, MPC_ROW_TPB, "layernorm", a);
        }
        if (st) return st;
        const i64 n = rows * cols;
        acct_beaver(c, (u64)n);
        acct_exp(c, (u64)rows, &p->rsqrt.exp);
        for (int i = 0; i < 3 * p->rsqrt.iters; ++i) acct_beaver(c, (u64)rows);
        if (p->bcast) acct_bcast(c, (u64)n, (u64)rows); else acct_beaver(c, (u64)n);
    }
    finish(c, steps);
    return MPC_OK;
}

}  // extern "C"
