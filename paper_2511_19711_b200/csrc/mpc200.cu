// mpc200.cu -- kernels (MPC_MODE_BOTH) and the C ABI of include/mpc200.h.
//
// Every kernel here executes the protocol of DESIGN.md section 2 for BOTH parties
// and the dealer on one GPU: Philox triples in registers, masked values formed
// and "opened" in registers, both parties' share updates.  No tensor cores: the
// path is element-wise / bitwise integer work.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdarg>
#include <algorithm>
#include <cuda_runtime.h>

#include "mpc200.h"
#include "sched_both.cuh"
#include "rows_both.cuh"

using namespace mpc;

// ------------------------------------------------------------------ context ----
// per-launch timing records (mpc_ctx_enable_kernel_timing): CUDA events on the ctx
// stream around every launch, plus the launch's algorithmic Philox count.
struct TimingRec { const char* name; cudaEvent_t a, b; u64 philox_at; u64 philox; u64 units; };

struct mpc_ctx {
    mpc_config cfg;
    Keys K;
    u64 step;
    cudaStream_t stream;
    int sm_count;
    mpc_stats st;
    u64 last_philox;
    char err[512];
    void* scratch;         // ctx-owned, grow-only, stream-ordered on `stream`
    size_t scratch_bytes;
    int timing;
    TimingRec* recs;
    int nrec, caprec;
    cudaEvent_t* pool;
    int npool, cappool;
};

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
static void rec_begin(mpc_ctx* c, const char* name, u64 units)
{
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

static Key mkkey(u64 k) { return Key{(u32)k, (u32)(k >> 32)}; }

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

// accounting of one primitive over n units (DESIGN.md 2.3 / 2.4 cost model)
static void acct_beaver(mpc_ctx* c, u64 n)
{
    c->last_philox += 2 * n + (n + 1) / 2;
    c->st.bytes_per_party += 16 * n;
    c->st.rounds += 1;
}
static void acct_ltz(mpc_ctx* c, u64 n, int w)
{
    const u64 groups = (n + 31) / 32;
    c->last_philox += groups * ltz_philox_per_group(w);
    c->st.bytes_per_party += groups * (8ull * (u64)gate_count(w) + 4ull);
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

// ------------------------------------------------------------------ kernels ----
__global__ void k_prg_fill(Key key, u64 unit0, u32 step, u32 slot, u32* out, i64 n, int reps)
{
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        const u64 u = unit0 + (u64)i;
        uint4 v = prg(key, u, step, slot);
        for (int r = 1; r < reps; ++r) v = philox(key, v.x, v.y, v.z ^ step, v.w ^ slot);
        reinterpret_cast<uint4*>(out)[i] = v;
    }
}

// S1: v = E(x); owner share v - r, other r; r = PRG(K_s, off+i, s, 0)
__global__ void k_share(const void* x, int f64, int owner, u64* s0, u64* s1, i64 n, u64 off,
                        u32 s, Key ks)
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

__global__ void k_trunc(const u64* x0, const u64* x1, u64* z0, u64* z1, i64 n, int bits)
{
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        z0[i] = shr(x0[i], bits);
        z1[i] = shr(x1[i], bits);
    }
}

// ---- generic drivers ---------------------------------------------------------------
// PAIR driver: thread <-> global unit pair (2P, 2P+1) covering [off, off+n).
template <class Body>
__global__ void __launch_bounds__(256, 3) k_pairs(i64 n, u64 off, Body body)
{
    const u64 p0 = off >> 1, p1 = (off + (u64)n + 1) >> 1;
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 P = p0 + blockIdx.x * (u64)blockDim.x + threadIdx.x; P < p1; P += stride) {
        const u64 u = 2 * P;
        const i64 i0 = (i64)(u - off);    // may be -1 when off is odd
        body(u, i0);
    }
}

// GROUP driver: warp <-> 32-unit LTZ group, lane <-> unit.  off % 32 == 0.
template <class Body>
__global__ void __launch_bounds__(256, 3) k_groups(i64 n, u64 off, Body body)
{
    const int lane = threadIdx.x & 31;
    const i64 ng = (n + 31) >> 5;
    const i64 nw = ((i64)gridDim.x * blockDim.x) >> 5;
    for (i64 g = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < ng; g += nw) {
        const i64 i = g * 32 + lane;
        body(off + (u64)i, (off >> 5) + (u64)g, i, lane, i < n);
    }
}

struct Ptr2 { const u64* p0; const u64* p1; };
struct Out2 { u64* p0; u64* p1; };

__device__ __forceinline__ Sh ld(Ptr2 a, i64 i) { return {a.p0[i], a.p1[i]}; }
__device__ __forceinline__ void st(Out2 a, i64 i, Sh v) { a.p0[i] = v.s0; a.p1[i] = v.s1; }

// ---- element-wise bodies ----------------------------------------------------------------
struct MulBody {
    Keys K; u32 s; Ptr2 x, y; Out2 z; i64 n; int tb;
    __device__ void operator()(u64 u, i64 i0) const {
        const bool v0 = i0 >= 0, v1 = i0 + 1 < n;
        Sh xa = {0, 0}, ya = {0, 0}, xb = {0, 0}, yb = {0, 0};
        if (v0) { xa = ld(x, i0); ya = ld(y, i0); }
        if (v1) { xb = ld(x, i0 + 1); yb = ld(y, i0 + 1); }
        Sh za, zb;
        bm2(K, u, s, xa, ya, xb, yb, za, zb);
        if (tb) { za = sh_shr(za, tb); zb = sh_shr(zb, tb); }
        if (v0) st(z, i0, za);
        if (v1) st(z, i0 + 1, zb);
    }
};

template <bool WIDE>
struct CmpBody {
    Keys K; u32 s; int w; Ptr2 x; Out2 z; int relu;
    __device__ void operator()(u64 u, u64 q, i64 i, int lane, bool valid) const {
        Sh xv = {0, 0};
        if (valid) xv = ld(x, i);
        Sh l = ltz<WIDE>(K, q, s, w, xv, lane);
        if (relu) l = bm(K, u, s + 1, xv, sh_not(l));
        if (valid) st(z, i, l);
    }
};

template <bool WIDE>
struct ExpGroupBody {
    Keys K; u32 s; ExpK p; Ptr2 x; Out2 z;
    __device__ void operator()(u64 u, u64 q, i64 i, int lane, bool valid) const {
        Sh xv = {0, 0};
        if (valid) xv = ld(x, i);
        const Sh y = exp_group<WIDE>(K, u, q, s, p, xv, lane);
        if (valid) st(z, i, y);
    }
};

struct ExpPairBody {
    Keys K; u32 s; ExpK p; Ptr2 x; Out2 z; i64 n;
    __device__ void operator()(u64 u, i64 i0) const {
        const bool v0 = i0 >= 0, v1 = i0 + 1 < n;
        Sh a = {0, 0}, b = {0, 0};
        if (v0) a = ld(x, i0);
        if (v1) b = ld(x, i0 + 1);
        exp_pair(K, u, s, p, a, b);
        if (v0) st(z, i0, a);
        if (v1) st(z, i0 + 1, b);
    }
};

template <int KIND, bool WIDE>   // 0 recip, 1 rsqrt
struct NrGroupBody {
    Keys K; u32 s; NrK p; Ptr2 x; Out2 z;
    __device__ void operator()(u64 u, u64 q, i64 i, int lane, bool valid) const {
        Sh xv = {0, 0};
        if (valid) xv = ld(x, i);
        Sh y;
        if (KIND == 0) y = recip_group<WIDE>(K, u, q, s, p, xv, lane);
        else y = rsqrt_group<WIDE>(K, u, q, s, p, xv, lane);
        if (valid) st(z, i, y);
    }
};

template <int KIND>
struct NrPairBody {
    Keys K; u32 s; NrK p; Ptr2 x; Out2 z; i64 n;
    __device__ void operator()(u64 u, i64 i0) const {
        const bool v0 = i0 >= 0, v1 = i0 + 1 < n;
        Sh a = {0, 0}, b = {0, 0};
        if (v0) a = ld(x, i0);
        if (v1) b = ld(x, i0 + 1);
        Sh ya, yb;
        if (KIND == 0) recip_pair(K, u, s, p, a, b, ya, yb);
        else rsqrt_pair(K, u, s, p, a, b, ya, yb);
        if (v0) st(z, i0, ya);
        if (v1) st(z, i0 + 1, yb);
    }
};

template <bool WIDE>
struct ActBody {
    Keys K; u32 s; ActK p; Ptr2 x; Out2 z;
    __device__ void operator()(u64 u, u64 q, i64 i, int lane, bool valid) const {
        Sh xv = {0, 0};
        if (valid) xv = ld(x, i);
        const Sh y = act_group<WIDE>(K, u, q, s, p, xv, lane);
        if (valid) st(z, i, y);
    }
};

// maxpool: gather each k x k window (public zero padding) into a row
__global__ void k_pool_gather(Ptr2 x, Out2 rowsbuf, int N, int C, int H, int W, int k, int stride,
                              int pad, int Ho, int Wo)
{
    const i64 rows = (i64)N * C * Ho * Wo, kk = (i64)k * k;
    for (i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x; t < rows * kk; t += (i64)gridDim.x * blockDim.x) {
        const i64 o = t / kk, e = t - o * kk;
        const int dy = (int)(e / k), dx = (int)(e - (i64)dy * k);
        const i64 ow = o % Wo, oh = (o / Wo) % Ho, c = (o / ((i64)Wo * Ho)) % C, img = o / ((i64)Wo * Ho * C);
        const i64 iy = oh * stride - pad + dy, ix = ow * stride - pad + dx;
        u64 a = 0, b = 0;
        if (iy >= 0 && iy < H && ix >= 0 && ix < W) {
            const i64 idx = ((img * C + c) * H + iy) * W + ix;
            a = x.p0[idx]; b = x.p1[idx];
        }
        rowsbuf.p0[t] = a; rowsbuf.p1[t] = b;
    }
}

// ------------------------------------------------------------------ host helpers ----
#define TPB 256

// resident CTAs per SM of a kernel at TPB threads (queried once per instantiation)
template <class K>
static int occupancy(K kern)
{
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, TPB, 0) != cudaSuccess || nb < 1) nb = 1;
    return nb;
}

template <class Body>
static mpc_status launch_pairs(mpc_ctx* c, i64 n, u64 off, const Body& b, const char* name)
{
    if (n <= 0) return MPC_OK;
    static int per_sm = occupancy(k_pairs<Body>);
    const i64 npairs = (i64)(((off + (u64)n + 1) >> 1) - (off >> 1));
    rec_begin(c, name, (u64)n);
    k_pairs<Body><<<grid_for(c, npairs, TPB, per_sm), TPB, 0, c->stream>>>(n, off, b);
    rec_end(c);
    c->st.launches++;
    return cuda_check(c, name);
}

template <class Body>
static mpc_status launch_groups(mpc_ctx* c, i64 n, u64 off, const Body& b, const char* name)
{
    if (n <= 0) return MPC_OK;
    static int per_sm = occupancy(k_groups<Body>);
    rec_begin(c, name, (u64)n);
    k_groups<Body><<<grid_for(c, ((n + 31) / 32) * 32, TPB, per_sm), TPB, 0, c->stream>>>(n, off, b);
    rec_end(c);
    c->st.launches++;
    return cuda_check(c, name);
}

static bool bad2(const mpc_ctx* c, mpc_shares s)
{
    (void)c;
    return !s.sh[0] || !s.sh[1] || ((uintptr_t)s.sh[0] & 7) || ((uintptr_t)s.sh[1] & 7);
}

static Ptr2 P(mpc_shares s) { return Ptr2{s.sh[0], s.sh[1]}; }
static Out2 O(mpc_shares s) { return Out2{s.sh[0], s.sh[1]}; }

// common prologue of a compute call: validates mode and step budget, resets counters
static mpc_status begin(mpc_ctx* c, u64 steps_needed)
{
    if (!c) return MPC_ERR_INVALID;
    c->last_philox = 0;
    c->st.calls++;
    if (c->step + steps_needed > (1ull << 32))
        return fail(c, MPC_ERR_RANGE, "step counter would exceed 2^32");
    return MPC_OK;
}
static void finish(mpc_ctx* c, u64 steps)
{
    rec_close(c);
    c->step += steps;
    c->st.steps += steps;
    c->st.philox_calls += c->last_philox;
}

static bool exp_ok(const mpc_exp_p* p) { return p && p->t >= 0 && p->t <= 8 && p->window >= 1 && p->window <= 64; }
static bool nr_ok(const mpc_nr_p* p) { return p && p->iters >= 1 && p->iters <= 12 && exp_ok(&p->exp); }

static ExpK mk_exp(const mpc_exp_p* p)
{
    return ExpK{p->t, p->clamp ? 1 : 0, p->window, E(1.0), E(ldexp(1.0, p->t))};
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
    for (int k = 0; k < p->t; ++k) acct_beaver(c, n);
}

// ------------------------------------------------------------------ ABI ----
extern "C" {

const char* mpc_version(void) { return "mpc200 0.1 (sm_100a; BOTH + PAIR_HOST)"; }

mpc_status mpc_ctx_create(const mpc_config* cfg, mpc_ctx** out)
{
    if (!cfg || !out) return MPC_ERR_INVALID;
    if (cfg->frac_bits != 16) return MPC_ERR_RANGE;
    if (cfg->mode != MPC_MODE_BOTH && cfg->mode != MPC_MODE_PAIR_HOST) return MPC_ERR_INVALID;
    if (cfg->mode != MPC_MODE_BOTH) return MPC_ERR_UNSUPPORTED;   /* PAIR modes: mpc200_pair */
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
    *out = c;
    return MPC_OK;
}

mpc_status mpc_ctx_destroy(mpc_ctx* c)
{
    if (!c) return MPC_OK;
    for (int i = 0; i < c->nrec; ++i) { cudaEventDestroy(c->recs[i].a); cudaEventDestroy(c->recs[i].b); }
    for (int i = 0; i < c->npool; ++i) cudaEventDestroy(c->pool[i]);
    free(c->recs); free(c->pool);
    if (c->scratch) { cudaFreeAsync(c->scratch, c->stream); cudaStreamSynchronize(c->stream); }
    delete c;
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
    if (ns != c->stream && c->scratch) {
        // the scratch tile is stream-ordered: order the new stream after the old one
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
    rec_begin(c, "prg_fill", 0);
    k_prg_fill<<<grid_for(c, n, TPB, 16), TPB, 0, c->stream>>>(mkkey(key), unit0, step, slot, out, n, reps);
    rec_end(c);
    c->st.launches++;
    return cuda_check(c, "prg_fill");
}

mpc_status mpc_share(mpc_ctx* c, const void* x, int x_is_f64, int owner, mpc_shares out,
                     int64_t n, int64_t off)
{
    mpc_status st = begin(c, 1);
    if (st) return st;
    if (owner != 0 && owner != 1) return fail(c, MPC_ERR_INVALID, "owner must be 0 or 1");
    if (n < 0 || off < 0) return fail(c, MPC_ERR_INVALID, "bad n/off");
    if (c->cfg.mode == MPC_MODE_BOTH) {
        if (bad2(c, out) || (!x && n > 0)) return fail(c, MPC_ERR_INVALID, "share: null pointer");
    } else {
        if (!out.sh[c->cfg.party] || (c->cfg.party == owner && !x && n > 0))
            return fail(c, MPC_ERR_INVALID, "share: null pointer");
    }
    u64* s0 = c->cfg.mode == MPC_MODE_BOTH || c->cfg.party == 0 ? out.sh[0] : nullptr;
    u64* s1 = c->cfg.mode == MPC_MODE_BOTH || c->cfg.party == 1 ? out.sh[1] : nullptr;
    const void* xin = (c->cfg.mode == MPC_MODE_BOTH || c->cfg.party == owner) ? x : nullptr;
    if (n > 0) {
        rec_begin(c, "share", 0);
        k_share<<<grid_for(c, n, TPB, 16), TPB, 0, c->stream>>>(xin, x_is_f64, owner, s0, s1, n, (u64)off, (u32)c->step, c->K.ks);
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
    mpc_status st = begin(c, 0);
    if (st) return st;
    if (n < 0 || scale_bits < 0 || scale_bits > 62) return fail(c, MPC_ERR_INVALID, "bad n/scale");
    if (bad2(c, in)) return fail(c, MPC_ERR_INVALID, "open: null pointer");
    if (n > 0) {
        rec_begin(c, "open", 0);
        k_open<<<grid_for(c, n, TPB, 16), TPB, 0, c->stream>>>(in.sh[0], in.sh[1], n, ring_out, f64_out, scale_bits);
        rec_end(c);
        c->st.launches++;
        if ((st = cuda_check(c, "open"))) return st;
    }
    c->st.bytes_per_party += 8ull * (u64)n;
    c->st.rounds += 1;
    return MPC_OK;
}

mpc_status mpc_trunc(mpc_ctx* c, mpc_shares x, mpc_shares z, int64_t n, int bits)
{
    mpc_status st = begin(c, 0);
    if (st) return st;
    if (bits < 0 || bits > 63) return fail(c, MPC_ERR_RANGE, "bits");
    if (bad2(c, x) || bad2(c, z) || n < 0) return fail(c, MPC_ERR_INVALID, "trunc args");
    if (n > 0) {
        rec_begin(c, "trunc", 0);
        k_trunc<<<grid_for(c, n, TPB, 16), TPB, 0, c->stream>>>(x.sh[0], x.sh[1], z.sh[0], z.sh[1], n, bits);
        rec_end(c);
        c->st.launches++;
        if ((st = cuda_check(c, "trunc"))) return st;
    }
    return MPC_OK;
}

#define CHECK_BOTH_ONLY(c) \
    if ((c)->cfg.mode != MPC_MODE_BOTH) return fail((c), MPC_ERR_UNSUPPORTED, "op not available in this mode")

mpc_status mpc_mul(mpc_ctx* c, mpc_shares x, mpc_shares y, mpc_shares z, int64_t n, int64_t off, int tb)
{
    mpc_status st = begin(c, 1);
    if (st) return st;
    if (tb != 0 && tb != 16) return fail(c, MPC_ERR_RANGE, "trunc_bits must be 0 or 16");
    if (n < 0 || off < 0) return fail(c, MPC_ERR_INVALID, "bad n/off");
    if (bad2(c, x) || bad2(c, y) || bad2(c, z)) return fail(c, MPC_ERR_INVALID, "mul: null pointer");
    if ((st = launch_pairs(c, n, (u64)off, MulBody{c->K, (u32)c->step, P(x), P(y), O(z), n, tb}, "mul"))) return st;
    acct_beaver(c, (u64)n);
    finish(c, 1);
    return MPC_OK;
}

static mpc_status cmp_common(mpc_ctx* c, mpc_shares x, mpc_shares z, int64_t n, int64_t off, int w, int relu)
{
    mpc_status st = begin(c, relu ? 2 : 1);
    if (st) return st;
    if (w < 1 || w > 64) return fail(c, MPC_ERR_RANGE, "window must be in [1,64]");
    if (n < 0 || off < 0 || (off & 31)) return fail(c, MPC_ERR_INVALID, "off must be a multiple of 32");
    if (bad2(c, x) || bad2(c, z)) return fail(c, MPC_ERR_INVALID, "cmp: null pointer");
    st = w > 33 ? launch_groups(c, n, (u64)off, CmpBody<true>{c->K, (u32)c->step, w, P(x), O(z), relu}, relu ? "relu" : "cmp")
                : launch_groups(c, n, (u64)off, CmpBody<false>{c->K, (u32)c->step, w, P(x), O(z), relu}, relu ? "relu" : "cmp");
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
    CHECK_BOTH_ONLY(c);
    if (bad2(c, x) || bad2(c, z) || n < 0 || off < 0) return fail(c, MPC_ERR_INVALID, "exp args");
    const ExpK k = mk_exp(p);
    if (p->clamp) {
        if (off & 31) return fail(c, MPC_ERR_INVALID, "off must be a multiple of 32");
        st = p->window > 33 ? launch_groups(c, n, (u64)off, ExpGroupBody<true>{c->K, (u32)c->step, k, P(x), O(z)}, "exp")
                            : launch_groups(c, n, (u64)off, ExpGroupBody<false>{c->K, (u32)c->step, k, P(x), O(z)}, "exp");
    } else {
        st = launch_pairs(c, n, (u64)off, ExpPairBody{c->K, (u32)c->step, k, P(x), O(z), n}, "exp");
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
    CHECK_BOTH_ONLY(c);
    if (bad2(c, x) || bad2(c, z) || n < 0 || off < 0) return fail(c, MPC_ERR_INVALID, "newton args");
    const NrK k = mk_nr(p);
    if (p->exp.clamp) {
        if (off & 31) return fail(c, MPC_ERR_INVALID, "off must be a multiple of 32");
        st = p->exp.window > 33 ? launch_groups(c, n, (u64)off, NrGroupBody<KIND, true>{c->K, (u32)c->step, k, P(x), O(z)}, "newton")
                                : launch_groups(c, n, (u64)off, NrGroupBody<KIND, false>{c->K, (u32)c->step, k, P(x), O(z)}, "newton");
    } else {
        st = launch_pairs(c, n, (u64)off, NrPairBody<KIND>{c->K, (u32)c->step, k, P(x), O(z), n}, "newton");
    }
    if (st) return st;
    acct_exp(c, (u64)n, &p->exp);
    for (int i = 0; i < (KIND == 0 ? 2 : 3) * p->iters; ++i) acct_beaver(c, (u64)n);
    finish(c, steps);
    return MPC_OK;
}
extern "C" {
mpc_status mpc_recip(mpc_ctx* c, mpc_shares x, mpc_shares z, int64_t n, int64_t off, const mpc_nr_p* p) { return nr_common<0>(c, x, z, n, off, p); }
mpc_status mpc_rsqrt(mpc_ctx* c, mpc_shares x, mpc_shares z, int64_t n, int64_t off, const mpc_nr_p* p) { return nr_common<1>(c, x, z, n, off, p); }

static u64 act_steps(int act, const mpc_act_p* p)
{
    if (p->form == MPC_FORM_RELU || (p->form != MPC_FORM_ERF && p->degree == 0)) return act == 2 ? 1 : 2;
    const u64 tail = act == 2 ? 1 : 2;
    if (p->form == MPC_FORM_POLY_X) return 2 + (u64)(p->degree - 1) + tail;
    if (p->form == MPC_FORM_POLY_ABS) return 3 + 1 + (u64)(p->degree - 1) + tail;
    return 2 + 1 + (u64)(p->erf_terms - 2) + 2 + tail;   // ERF
}

static mpc_status act_common(mpc_ctx* c, int act, mpc_shares x, mpc_shares z, int64_t n, int64_t off, const mpc_act_p* p)
{
    if (!c) return MPC_ERR_INVALID;
    if (!p || p->window < 1 || p->window > 64) return fail(c, MPC_ERR_RANGE, "window");
    if (p->form < 0 || p->form > 3) return fail(c, MPC_ERR_RANGE, "form");
    if ((p->form == MPC_FORM_POLY_X || p->form == MPC_FORM_POLY_ABS) && (p->degree < 0 || p->degree > 4))
        return fail(c, MPC_ERR_RANGE, "degree must be in [0,4]");
    if (p->form == MPC_FORM_ERF && (act != 0 || p->erf_terms < 2 || p->erf_terms > 12))
        return fail(c, MPC_ERR_RANGE, "erf form: GELU only, erf_terms in [2,12]");
    if (p->form == MPC_FORM_POLY_ABS && act == 2) return fail(c, MPC_ERR_RANGE, "sigmoid has no |x|-form (R30)");
    if ((p->form == MPC_FORM_POLY_X || p->form == MPC_FORM_POLY_ABS) && p->degree > 0 && !p->coeffs)
        return fail(c, MPC_ERR_INVALID, "coeffs");
    const u64 steps = act_steps(act, p);
    mpc_status st = begin(c, steps);
    if (st) return st;
    CHECK_BOTH_ONLY(c);
    if (bad2(c, x) || bad2(c, z) || n < 0 || off < 0 || (off & 31)) return fail(c, MPC_ERR_INVALID, "act args (off % 32)");
    ActK k;
    memset(&k, 0, sizeof k);
    k.act = act; k.form = p->form; k.w = p->window;
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
    st = k.w > 33 ? launch_groups(c, n, (u64)off, ActBody<true>{c->K, (u32)c->step, k, P(x), O(z)}, "act")
                  : launch_groups(c, n, (u64)off, ActBody<false>{c->K, (u32)c->step, k, P(x), O(z)}, "act");
    if (st) return st;
    // accounting
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
mpc_status mpc_gelu(mpc_ctx* c, mpc_shares x, mpc_shares z, int64_t n, int64_t off, const mpc_act_p* p) { return act_common(c, 0, x, z, n, off, p); }
mpc_status mpc_silu(mpc_ctx* c, mpc_shares x, mpc_shares z, int64_t n, int64_t off, const mpc_act_p* p) { return act_common(c, 1, x, z, n, off, p); }
mpc_status mpc_sigmoid(mpc_ctx* c, mpc_shares x, mpc_shares z, int64_t n, int64_t off, const mpc_act_p* p) { return act_common(c, 2, x, z, n, off, p); }

}  // extern "C"

// ---- row ops (fused, one CTA per 32-row tile; rows_both.cuh) -------------------------------------
static int max_levels_h(i64 cols) { int L = 0; i64 m = cols; while (m > 1) { m = (m + 1) / 2; ++L; } return L; }

static const size_t SMEM_LIMIT = 72 * 1024;      // keep 3 CTAs per SM

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

template <class Args>
static mpc_status launch_rows(mpc_ctx* c, void (*kern)(Args), Args& a, i64 rows, i64 work_u64, const char* name)
{
    const i64 ntiles = (rows + 31) / 32;
    const size_t smem = sizeof(u64) * (size_t)work_u64;
    int grid = (int)std::min<i64>(ntiles, (i64)c->sm_count * 3);
    if (grid < 1) grid = 1;
    size_t dyn = 0;
    if (work_u64 > 0 && smem <= SMEM_LIMIT) {
        a.use_smem = 1; a.gscratch = nullptr; dyn = smem;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    } else if (work_u64 > 0) {
        a.use_smem = 0;
        a.gscratch = (u64*)scratch(c, smem * (size_t)grid);
        if (!a.gscratch) return fail(c, MPC_ERR_NOMEM, "%s: scratch %zu bytes", name, smem * (size_t)grid);
    }
    a.work_u64 = work_u64;
    rec_begin(c, name, (u64)rows);
    kern<<<grid, 256, dyn, c->stream>>>(a);
    rec_end(c);
    c->st.launches++;
    return cuda_check(c, name);
}

extern "C" {

mpc_status mpc_max(mpc_ctx* c, mpc_shares x, mpc_shares z, int64_t rows, int64_t cols, int64_t row_off, int w)
{
    if (!c) return MPC_ERR_INVALID;
    const u64 steps = 2ull * (u64)max_levels_h(cols);
    mpc_status st = begin(c, steps);
    if (st) return st;
    CHECK_BOTH_ONLY(c);
    if (w < 1 || w > 64) return fail(c, MPC_ERR_RANGE, "window");
    if (bad2(c, x) || bad2(c, z) || rows < 0 || cols < 1 || row_off < 0 || (row_off & 31))
        return fail(c, MPC_ERR_INVALID, "max args (row_off % 32)");
    if (rows > 0) {
        MaxArgs a{c->K, (u32)c->step, w, RowPtr2{x.sh[0], x.sh[1]}, RowOut2{z.sh[0], z.sh[1]}, rows, cols,
                  (u64)row_off, nullptr, 0, 0};
        if ((st = launch_rows(c, w > 33 ? k_max_fused<true> : k_max_fused<false>, a, rows, max_work_u64(cols), "max_fused"))) return st;
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
    CHECK_BOTH_ONLY(c);
    if (w < 1 || w > 64) return fail(c, MPC_ERR_RANGE, "window");
    const u64 row_off = (u64)img_off * (u64)C * (u64)Ho * (u64)Wo;
    if (bad2(c, x) || bad2(c, z) || img_off < 0 || (row_off & 31)) return fail(c, MPC_ERR_INVALID, "maxpool args");
    if (rows > 0) {
        // gather the windows (public zero padding) into rows, then the fused row max
        u64* Rw = (u64*)scratch(c, sizeof(u64) * 2 * (size_t)(rows * cols));
        if (!Rw) return fail(c, MPC_ERR_NOMEM, "maxpool scratch");
        rec_begin(c, "pool_gather", 0);
        k_pool_gather<<<grid_for(c, rows * cols, TPB, 16), TPB, 0, c->stream>>>(P(x), Out2{Rw, Rw + rows * cols}, N, C, H, W, k, stride, pad, Ho, Wo);
        rec_end(c);
        c->st.launches++;
        if ((st = cuda_check(c, "pool_gather"))) return st;
        MaxArgs a{c->K, (u32)c->step, w, RowPtr2{Rw, Rw + rows * cols}, RowOut2{z.sh[0], z.sh[1]}, rows, cols,
                  row_off, nullptr, 0, 0};
        if (max_work_u64(cols) * 8 > (i64)SMEM_LIMIT) return fail(c, MPC_ERR_UNSUPPORTED, "pool window too large");
        if ((st = launch_rows(c, w > 33 ? k_max_fused<true> : k_max_fused<false>, a, rows, max_work_u64(cols), "maxpool_fused"))) return st;
        acct_max(c, rows, cols, w);
    }
    finish(c, steps);
    return MPC_OK;
}

mpc_status mpc_softmax(mpc_ctx* c, mpc_shares x, mpc_shares z, int64_t rows, int64_t cols, int64_t row_off,
                       const mpc_softmax_p* p)
{
    if (!c) return MPC_ERR_INVALID;
    if (!p || p->window < 1 || p->window > 64 || !exp_ok(&p->exp) || !nr_ok(&p->recip))
        return fail(c, MPC_ERR_RANGE, "softmax knobs");
    const int L = max_levels_h(cols);
    const u64 steps = 2ull * (u64)L + exp_steps_h(&p->exp) + exp_steps_h(&p->recip.exp) + 2ull * (u64)p->recip.iters + 1;
    mpc_status st = begin(c, steps);
    if (st) return st;
    CHECK_BOTH_ONLY(c);
    if (bad2(c, x) || bad2(c, z) || rows < 0 || cols < 1 || row_off < 0 || (row_off & 31))
        return fail(c, MPC_ERR_INVALID, "softmax args (row_off % 32)");
    if (rows > 0) {
        SoftmaxArgs a;
        a.K = c->K;
        a.s_max = (u32)c->step;
        a.s_exp = a.s_max + 2u * (u32)L;
        a.s_rec = a.s_exp + (u32)exp_steps_h(&p->exp);
        a.s_mul = a.s_rec + (u32)exp_steps_h(&p->recip.exp) + 2u * (u32)p->recip.iters;
        a.w = p->window; a.ek = mk_exp(&p->exp); a.rk = mk_nr(&p->recip);
        a.x = RowPtr2{x.sh[0], x.sh[1]}; a.z = RowOut2{z.sh[0], z.sh[1]};
        a.rows = rows; a.cols = cols; a.row_off = (u64)row_off;
        const bool wide = p->window > 33 || p->exp.window > 33 || p->recip.exp.window > 33;
        if ((st = launch_rows(c, wide ? k_softmax_fused<true> : k_softmax_fused<false>, a, rows,
                              softmax_work_u64(cols), "softmax_fused"))) return st;
        const i64 n = rows * cols;
        acct_max(c, rows, cols, p->window);
        acct_exp(c, (u64)n, &p->exp);
        acct_exp(c, (u64)rows, &p->recip.exp);
        for (int i = 0; i < 2 * p->recip.iters; ++i) acct_beaver(c, (u64)rows);
        acct_beaver(c, (u64)n);
    }
    finish(c, steps);
    return MPC_OK;
}

mpc_status mpc_layernorm(mpc_ctx* c, mpc_shares x, mpc_shares z, int64_t rows, int64_t cols, int64_t row_off,
                         const mpc_ln_p* p)
{
    if (!c) return MPC_ERR_INVALID;
    if (!p || !nr_ok(&p->rsqrt) || (p->mean_mode != 0 && p->mean_mode != 1)) return fail(c, MPC_ERR_RANGE, "layernorm knobs");
    const u64 steps = 1 + exp_steps_h(&p->rsqrt.exp) + 3ull * (u64)p->rsqrt.iters + 1;
    mpc_status st = begin(c, steps);
    if (st) return st;
    CHECK_BOTH_ONLY(c);
    if (bad2(c, x) || bad2(c, z) || rows < 0 || cols < 1 || row_off < 0 || (row_off & 31))
        return fail(c, MPC_ERR_INVALID, "layernorm args (row_off % 32)");
    if (rows > 0) {
        LnArgs a;
        a.K = c->K;
        a.s_sq = (u32)c->step;
        a.s_rs = a.s_sq + 1;
        a.s_mul = a.s_rs + (u32)exp_steps_h(&p->rsqrt.exp) + 3u * (u32)p->rsqrt.iters;
        a.rk = mk_nr(&p->rsqrt);
        a.x = RowPtr2{x.sh[0], x.sh[1]}; a.z = RowOut2{z.sh[0], z.sh[1]};
        a.rows = rows; a.cols = cols; a.row_off = (u64)row_off;
        a.mean_mode = p->mean_mode; a.e_invd = E(1.0 / (double)cols); a.e_eps = E(p->eps);
        const i64 ntiles = (rows + 31) / 32;
        const int grid = (int)std::min<i64>(ntiles, (i64)c->sm_count * 3);
        rec_begin(c, "layernorm_fused", (u64)rows);
        if (p->rsqrt.exp.window > 33) k_ln_fused<true><<<grid, 256, 0, c->stream>>>(a);
        else k_ln_fused<false><<<grid, 256, 0, c->stream>>>(a);
        rec_end(c);
        c->st.launches++;
        if ((st = cuda_check(c, "layernorm_fused"))) return st;
        const i64 n = rows * cols;
        acct_beaver(c, (u64)n);
        acct_exp(c, (u64)rows, &p->rsqrt.exp);
        for (int i = 0; i < 3 * p->rsqrt.iters; ++i) acct_beaver(c, (u64)rows);
        acct_beaver(c, (u64)n);
    }
    finish(c, steps);
    return MPC_OK;
}

}  // extern "C"
