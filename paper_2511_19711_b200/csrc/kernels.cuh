// kernels.cuh -- every kernel of the library, written once against a launch policy PA:
//   BothA : MPC_MODE_BOTH (policy BothP)
//   PairA : MPC_MODE_PAIR (one party per GPU, grid = that party's CTAs) and
//           MPC_MODE_PAIR_LOOPBACK (one launch, CTAs [0,G) are party 0 and [G,2G) party 1,
//           exchanging through local memory -- the same code path as two GPUs).
// All loops that contain an opening are warp-uniform (PairP exchanges per warp).
#pragma once
#include "sched.cuh"
#include "ltz_cone.cuh"

#ifndef MPC_SM_MINB
#define MPC_SM_MINB 2      // resident CTAs/SM the row kernels are compiled for (<= 128 regs; 3 measured slower: spills)
#endif
#ifndef MPC_SM_MINB_KS
#define MPC_SM_MINB_KS 2   // same for the Kogge-Stone (LV 0) row kernels
#endif
#ifndef MPC_ROW_TPB
#define MPC_ROW_TPB 256    // threads per CTA of the row kernels (softmax / max / layernorm)
#endif
#ifndef MPC_GROUP_PREFETCH
#define MPC_GROUP_PREFETCH 1   // element-wise drivers prefetch the next pass's input shares to L2
#endif
#ifndef MPC_MAXS_PAIRS
#define MPC_MAXS_PAIRS 0      // A/B: short-row max with the cone in BOTH: 4-group batches as 2 x 2 flat
#endif
#ifndef MPC_EW_MINB
#define MPC_EW_MINB 2      // same for the element-wise drivers
#endif

namespace mpc {

// ------------------------------------------------------------------ launch policies ----
struct BothA {
    Keys K;
    __device__ __forceinline__ BothP make(int& cta, int& ncta) const { cta = blockIdx.x; ncta = gridDim.x; return BothP{&K}; }
    __device__ __forceinline__ void done(BothP&) const {}
};

// launch arguments of both PAIR roles (identical layout: the host fills one PairArgs for either)
struct PairArgs {
    Keys K;
    int party;        // remote mode: this GPU's party
    int loopback;     // 1: both parties in one launch
    int G;            // CTAs per party
    int fmt;          // exchange wire format (proto.cuh): 0 LL, 1 LL63
    XMem xm[2];       // exchange memory of party 0 / 1 (remote: xm[0] only)
    // dealer correction stream (proto.cuh PairP::corr): cmode 1 = party 1 reads it,
    // 2 = this launch is the dealer and writes it (party 1's role over a self-loop exchange); the
    // segment is [ccap or depth][G * blockDim] words at cw; kmax: the dealer's words-per-thread
    // high-water mark.  Used by the stream role (R = 1) only.
    u64* cw;
    u32 ccap;
    int cmode;
    u32* kmax;
};
template <int R>
struct PairAR : PairArgs {
    __device__ __forceinline__ PairP<R> make(int& cta, int& ncta) const {
        PairP<R> p;
        p.Kp = &K;
        int slot_cta;
        if (loopback) { p.pty = blockIdx.x >= (unsigned)G ? 1 : 0; slot_cta = blockIdx.x - p.pty * G; }
        else { p.pty = party; slot_cta = blockIdx.x; }
        cta = slot_cta; ncta = G;
        p.local = loopback;
        p.fmt = fmt;
        if constexpr (R == 1) {
            p.cmode = p.pty == 1 ? cmode : 0;
            p.cst = (u32)G * blockDim.x;
            p.cw = p.cmode ? cw + (u64)slot_cta * blockDim.x + threadIdx.x : nullptr;
            p.ck = 0;
            p.ccap = ccap;
        }
        p.bind(xm[loopback ? p.pty : 0], slot_cta * (blockDim.x >> 5) + (threadIdx.x >> 5));
        return p;
    }
    __device__ __forceinline__ void done(PairP<R>& p) const {
        p.unbind(threadIdx.x & 31);
        if constexpr (R == 1)
            if (p.cmode == 2 && p.ck) atomicMax(kmax, p.ck);
    }
};
using PairA = PairAR<0>;     // party 0; party 1 simulating the dealer; loopback
using PairAS = PairAR<1>;    // the stream roles: party 1 reading the dealer's stream, the dealer itself
static_assert(sizeof(PairA) == sizeof(PairArgs) && sizeof(PairAS) == sizeof(PairArgs), "one argument layout");

// ------------------------------------------------------------------ drivers ----
// GROUP driver: warp <-> 32-unit LTZ group, lane <-> unit.  off % 32 == 0.
template <class PA, class Body>
__global__ void __launch_bounds__(256, MPC_EW_MINB) k_groups(const __grid_constant__ PA pa, i64 n, u64 off, Body body)
{
    int cta, ncta;
    auto pr = pa.make(cta, ncta);
    const int lane = threadIdx.x & 31, NW = blockDim.x >> 5;
    const i64 ng = (n + 31) >> 5;
    const i64 gstep = (i64)ncta * NW;
    for (i64 g = (i64)cta * NW + (threadIdx.x >> 5); g < ng; g += gstep) {
        const i64 i = g * 32 + lane;
        if (MPC_GROUP_PREFETCH) {       // the next group's input shares to L2 while this one computes
            const i64 inext = i + gstep * 32;
            if (inext < n) {
#pragma unroll
                for (int p = 0; p < 2; ++p)
                    if (body.x.p[p]) asm volatile("prefetch.global.L2 [%0];" :: "l"(body.x.p[p] + inext));
            }
        }
        body(pr, off + (u64)i, (off >> 5) + (u64)g, i, lane, i < n);
    }
    pa.done(pr);
}

// PAIR driver: lane <-> V = P::kV global unit pairs (2P, 2P+1) per pass (pairs base + lane + 32v),
// covering [off, off+n); warp-uniform loop.
template <class PA, class Body>
__global__ void __launch_bounds__(256, MPC_EW_MINB) k_pairs(const __grid_constant__ PA pa, i64 n, u64 off, Body body)
{
    int cta, ncta;
    auto pr = pa.make(cta, ncta);
    constexpr int V = decltype(pr)::kV;
    const int lane = threadIdx.x & 31, NW = blockDim.x >> 5;
    const u64 p0 = off >> 1, p1 = (off + (u64)n + 1) >> 1;
    const u64 pstep = (u64)ncta * NW * 32 * V;
    for (u64 base = ((u64)cta * NW + (threadIdx.x >> 5)) * 32 * V; p0 + base < p1; base += pstep) {
        if (MPC_GROUP_PREFETCH && p0 + base + pstep + lane < p1) {   // next pass's input shares to L2
            const i64 inext = (i64)(2 * (p0 + base + pstep + lane) - off);
            if (inext >= 0)
#pragma unroll
                for (int q = 0; q < 2; ++q)
                    if (body.x.p[q]) asm volatile("prefetch.global.L2 [%0];" :: "l"(body.x.p[q] + inext));
        }
        u64 u[V];
        i64 i0[V];
        bool ok[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const u64 P = p0 + base + lane + 32 * v;
            u[v] = 2 * P;
            i0[v] = (i64)(u[v] - off);
            ok[v] = P < p1;
        }
        body.template run<V>(pr, u, i0, ok);
    }
    pa.done(pr);
}

// CONE driver: warp <-> CG consecutive 32-unit groups; shared memory for the carry trees.
constexpr int CG = 4;
template <class PA, class Body>
__global__ void __launch_bounds__(256, MPC_EW_MINB) k_groups_cone(const __grid_constant__ PA pa, i64 n, u64 off, Body body)
{
    __shared__ ConeSmem<CG, Body::kNL> sm[8];
    extern __shared__ __align__(16) u64 stash[];       // per-warp staging (Body::kStash u64)
    int cta, ncta;
    auto pr = pa.make(cta, ncta);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
    const i64 ng = (n + 31) >> 5;
    for (i64 gb = ((i64)cta * NW + warp) * CG; gb < ng; gb += (i64)ncta * NW * CG)
        body(pr, off, gb, lane, sm[warp], stash + (i64)warp * Body::kStash);
    pa.done(pr);
}

// cmp / relu with the carry-cone LTZ over CG groups per warp (NL = 32: w <= 33, 64: w <= 64)
template <int NL>
struct CmpConeBody {
    static constexpr int kStash = 0, kNL = NL;
    u32 s; int w; SP x; SO z; int relu; i64 n;
    template <class P>
    __device__ void operator()(P& pr, u64 off, i64 gb, int lane, ConeSmem<CG, NL>& sm, u64*) const {
        using S = typename P::S;
        S xv[CG], l[CG];
#pragma unroll
        for (int g = 0; g < CG; ++g) {
            const i64 i = (gb + g) * 32 + lane;
            xv[g] = i < n ? pr.ld(x, i) : pr.zero();
        }
        pr.template ltz_cone<CG, NL>((off >> 5) + (u64)gb, s, w, xv, l, lane, sm);
#pragma unroll
        for (int g = 0; g < CG; ++g) {
            const i64 i = (gb + g) * 32 + lane;
            S r = l[g];
            if (relu) r = pr.bm(off + (u64)i, s + 1, xv[g], pr.notb(l[g]));
            if (i < n) pr.st(z, i, r);
        }
    }
};

// S13 with carry-cone LTZs: the 2-3 segment comparisons of CG groups run first (stashed in
// shared memory), then the polynomial / final products run in the PAIR layout -- thread <-> unit
// pairs (2p, 2p+1), one c0 block per pair, two independent Beaver chains per thread (act_tail2).
// Same step ids, units and output bits as act_group.  (The same body with Kogge-Stone LTZs per
// group measured 10 % slower than ActBody, so the Kogge-Stone path keeps the group layout.)
template <int NL>
struct ActConeBody {
    static constexpr int kStash = 3 * CG * 32 * 2, kNL = NL;      // [3 ltz][CG][32 lanes][2 words]
    u32 s; ActK p; SP x; SO z; i64 n;
    template <class P>
    __device__ __forceinline__ void ltzs(P& pr, u64 q0, u32 sl, typename P::S (&in)[CG], typename P::S (&out)[CG],
                                         int lane, ConeSmem<CG, NL>& sm) const {
        pr.template ltz_cone<CG, NL>(q0, sl, p.w, in, out, lane, sm);
    }
    template <class P>
    __device__ void operator()(P& pr, u64 off, i64 gb, int lane, ConeSmem<CG, NL>& sm, u64* st) const {
        using S = typename P::S;
        static_assert(sizeof(S) <= 16, "stash holds up to two words per share");
        S xv[CG], t[CG];
        S* stS = reinterpret_cast<S*>(st);              // [3][CG][32]
#pragma unroll
        for (int g = 0; g < CG; ++g) {
            const i64 i = (gb + g) * 32 + lane;
            xv[g] = i < n ? pr.ld(x, i) : pr.zero();
        }
        const u64 q0 = (off >> 5) + (u64)gb;
        const bool relu_form = p.form == 2 || p.deg == 0;
        u32 sl = s;
        if (relu_form || p.form == 1) {                 // ltz(x): the ReLU mask or the sign of x
            ltzs(pr, q0, sl, xv, t, lane, sm);
#pragma unroll
            for (int g = 0; g < CG; ++g) stS[(0 * CG + g) * 32 + lane] = t[g];
            ++sl;
        }
        if (!relu_form) {
#pragma unroll
            for (int g = 0; g < CG; ++g) t[g] = pr.addp(xv[g], p.e_B);
            ltzs(pr, q0, sl, t, t, lane, sm);
#pragma unroll
            for (int g = 0; g < CG; ++g) stS[(1 * CG + g) * 32 + lane] = t[g];
#pragma unroll
            for (int g = 0; g < CG; ++g) t[g] = pr.addp(xv[g], p.e_mB);
            ltzs(pr, q0, sl + 1, t, t, lane, sm);
#pragma unroll
            for (int g = 0; g < CG; ++g) stS[(2 * CG + g) * 32 + lane] = t[g];
            sl += 2;
        }
        __syncwarp();
#pragma unroll 1
        for (int j = 0; j < CG / 2; ++j) {              // pair lane + 32 j: elements e, e + 1 of the block
            const int e = 2 * (lane + 32 * j);
            const int o = e;                            // stash [k][g][lane]: element e of the block at k*CG*32 + e
            const i64 i = gb * 32 + e;
            const u64 u = off + (u64)i;
            const S x0 = i < n ? pr.ld(x, i) : pr.zero(), x1 = i + 1 < n ? pr.ld(x, i + 1) : pr.zero();
            S r0, r1;
            if (relu_form) {
                const S n0 = pr.notb(stS[o]), n1 = pr.notb(stS[o + 1]);
                if (p.act == 2) { r0 = pr.shl(n0, FRAC); r1 = pr.shl(n1, FRAC); }
                else pr.bm2(u, sl, x0, n0, x1, n1, r0, r1);
            } else {
                act_tail2(pr, u, sl, p, x0, x1, stS[o], stS[o + 1], stS[CG * 32 + o], stS[CG * 32 + o + 1],
                          stS[2 * CG * 32 + o], stS[2 * CG * 32 + o + 1], r0, r1);
            }
            if (i < n) pr.st(z, i, r0);
            if (i + 1 < n) pr.st(z, i + 1, r1);
        }
        __syncwarp();
    }
};

// ------------------------------------------------------------------ element-wise bodies ----
struct SquareBody {
    u32 s; SP x; SO z; i64 n; int tb;
    template <int V, class P>
    __device__ void run(P& pr, const u64 (&u)[V], const i64 (&i0)[V], const bool (&ok)[V]) const {
        using S = typename P::S;
        S xa[V], xb[V], za[V], zb[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            pr.ld_pair(x, i0[v], ok[v] && i0[v] >= 0, ok[v] && i0[v] + 1 < n, xa[v], xb[v]);
        }
        pr.template sq2v<V>(u, s, xa, xb, za, zb);
#pragma unroll
        for (int v = 0; v < V; ++v) {
            if (tb) { za[v] = pr.shr_(za[v], tb); zb[v] = pr.shr_(zb[v], tb); }
            pr.st_pair(z, i0[v], ok[v] && i0[v] >= 0, ok[v] && i0[v] + 1 < n, za[v], zb[v]);
        }
    }
};

struct MulBody {
    u32 s; SP x, y; SO z; i64 n; int tb;
    template <int V, class P>
    __device__ void run(P& pr, const u64 (&u)[V], const i64 (&i0)[V], const bool (&ok)[V]) const {
        using S = typename P::S;
        S xa[V], ya[V], xb[V], yb[V], za[V], zb[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const bool va = ok[v] && i0[v] >= 0, vb = ok[v] && i0[v] + 1 < n;
            pr.ld_pair(x, i0[v], va, vb, xa[v], xb[v]);
            pr.ld_pair(y, i0[v], va, vb, ya[v], yb[v]);
        }
        pr.template bm2v<V>(u, s, xa, ya, xb, yb, za, zb);
#pragma unroll
        for (int v = 0; v < V; ++v) {
            if (tb) { za[v] = pr.shr_(za[v], tb); zb[v] = pr.shr_(zb[v], tb); }
            pr.st_pair(z, i0[v], ok[v] && i0[v] >= 0, ok[v] && i0[v] + 1 < n, za[v], zb[v]);
        }
    }
};

template <bool WIDE>
struct CmpBody {
    u32 s; int w; SP x; SO z; int relu;
    template <class P>
    __device__ void operator()(P& pr, u64 u, u64 q, i64 i, int lane, bool valid) const {
        typename P::S xv = pr.zero();
        if (valid) xv = pr.ld(x, i);
        typename P::S l = pr.template ltz_rb<WIDE>(q, s, w, xv, lane);
        if (relu) l = pr.bm(u, s + 1, xv, pr.notb(l));
        if (valid) pr.st(z, i, l);
    }
};

template <bool WIDE>
struct ExpGroupBody {
    u32 s; ExpK p; SP x; SO z; int head_only;   // head_only: the clamp head (steps s, s+1) alone
    template <class P>
    __device__ void operator()(P& pr, u64 u, u64 q, i64 i, int lane, bool valid) const {
        typename P::S xv = pr.zero();
        if (valid) xv = pr.ld(x, i);
        const typename P::S y = head_only ? exp_clamp_head<WIDE>(pr, u, q, s, p, xv, lane)
                                          : exp_group<WIDE>(pr, u, q, s, p, xv, lane);
        if (valid) pr.st(z, i, y);
    }
};

struct ExpPairBody {
    u32 s; ExpK p; SP x; SO z; i64 n; int sq_only;   // sq_only: x holds the clamp head's y
    template <int V, class P>
    __device__ void run(P& pr, const u64 (&u)[V], const i64 (&i0)[V], const bool (&ok)[V]) const {
        typename P::S a[V], b[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            pr.ld_pair(x, i0[v], ok[v] && i0[v] >= 0, ok[v] && i0[v] + 1 < n, a[v], b[v]);
        }
        if (sq_only) exp_squarings_pairv<V>(pr, u, s, p, a, b);
        else exp_pairv<V>(pr, u, s, p, a, b);
#pragma unroll
        for (int v = 0; v < V; ++v) pr.st_pair(z, i0[v], ok[v] && i0[v] >= 0, ok[v] && i0[v] + 1 < n, a[v], b[v]);
    }
};

template <int KIND, bool WIDE>   // 0 recip, 1 rsqrt
struct NrGroupBody {
    u32 s; NrK p; SP x; SO z;
    template <class P>
    __device__ void operator()(P& pr, u64 u, u64 q, i64 i, int lane, bool valid) const {
        typename P::S xv = pr.zero();
        if (valid) xv = pr.ld(x, i);
        typename P::S y;
        if (KIND == 0) y = recip_group<WIDE>(pr, u, q, s, p, xv, lane);
        else y = rsqrt_group<WIDE>(pr, u, q, s, p, xv, lane);
        if (valid) pr.st(z, i, y);
    }
};

template <int KIND>
struct NrPairBody {
    u32 s; NrK p; SP x; SO z; i64 n;
    template <int V, class P>
    __device__ void run(P& pr, const u64 (&u)[V], const i64 (&i0)[V], const bool (&ok)[V]) const {
        typename P::S a[V], b[V], ya[V], yb[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            pr.ld_pair(x, i0[v], ok[v] && i0[v] >= 0, ok[v] && i0[v] + 1 < n, a[v], b[v]);
        }
        if (KIND == 0) recip_pairv<V>(pr, u, s, p, a, b, ya, yb);
        else rsqrt_pairv<V>(pr, u, s, p, a, b, ya, yb);
#pragma unroll
        for (int v = 0; v < V; ++v) pr.st_pair(z, i0[v], ok[v] && i0[v] >= 0, ok[v] && i0[v] + 1 < n, ya[v], yb[v]);
    }
};

template <bool WIDE>
struct ActBody {
    u32 s; ActK p; SP x; SO z;
    template <class P>
    __device__ void operator()(P& pr, u64 u, u64 q, i64 i, int lane, bool valid) const {
        typename P::S xv = pr.zero();
        if (valid) xv = pr.ld(x, i);
        const typename P::S y = act_group<WIDE>(pr, u, q, s, p, xv, lane);
        if (valid) pr.st(z, i, y);
    }
};

// S2 in PAIR modes: exchange the shares, both parties learn rec (reveal_to both)
// reveal >= 0 (mpc_open_to): only that party learns rec -- it sends zeros in place of its share
// (the exchange keeps its lockstep; the peer receives nothing about x) and adds its own share.
struct OpenBody {
    SP x; u64* ring; double* f; i64 n; double inv; int writer;   // writer: party that stores (-1: own)
    int reveal;                                                  // -1: both parties learn rec
    template <class P>
    __device__ void operator()(P& pr, u64 u, u64 q, i64 i, int lane, bool valid) const {
        (void)u; (void)q;
        typename P::S mine = pr.zero();
        if (valid) mine = pr.ld(x, i);
        u64 v;
        if constexpr (std::is_same<typename P::S, u64>::value) {     // PAIR: one party's share per thread
            const bool recv_only = reveal >= 0 && pr.party() == reveal;
            v = pr.open(recv_only ? pr.zero() : mine);
            if (recv_only) v += mine;
        } else {
            v = pr.open(mine);
        }
        if (valid && (writer < 0 || pr.party() == writer)) {
            if (ring) ring[i] = v;
            if (f) f[i] = (double)(i64)v * inv;
        }
    }
};

// Debug header exchange (mpc_ctx_set_debug, PAIR modes): each party opens its op header; a
// mismatch (rec != 2 hdr) marks the context's error word with 2 (MPC_ERR_PROTOCOL at sync).
struct HdrBody {
    u64 hdr;
    SP x;                 // unused (no inputs); keeps the group driver's prefetch interface
    template <class P>
    __device__ void operator()(P& pr, u64 u, u64 q, i64 i, int lane, bool valid) const {
        (void)u; (void)q; (void)i; (void)lane; (void)valid;
        if constexpr (std::is_same<typename P::S, u64>::value) {
            const u64 v = pr.open(hdr);
            if (v != 2ull * hdr) atomicCAS(pr.err, 0, 2);
        }
    }
};

// ------------------------------------------------------------------ row tiles ----
// One CTA owns a tile of 32 consecutive rows (32-aligned global row index); persistent loop.
// Tile plan: tiles of 32 rows, round-robin over the ncta CTAs.  When the last round would hold
// P = ntiles mod ncta tiles with 2P <= ncta (cfg2: 384 tiles on 296 CTAs leave 88 lone tiles on 88
// SMs while 60 idle), those P tiles run as 2P half tiles of 16 rows on twice the CTAs: the tail wave
// is one half-tile latency instead of one tile latency.  A half tile starts at a row = 16 mod 32, so
// the levels whose LTZ groups span more than 16 rows see a group offset (tile_max handles any
// alignment: the group's lanes outside the tile are evaluated and dropped).
struct TilePlan { i64 nfull, ntot; };
__device__ __forceinline__ TilePlan tile_plan(i64 rows, int ncta, int half)
{
    const i64 nt = (rows + 31) / 32, P = nt % ncta;
    if (!half || nt <= ncta || P == 0 || 2 * P > ncta) return TilePlan{nt, nt};
    return TilePlan{nt - P, nt + P};
}
// rows [r0, r0 + R) of plan tile t (R <= 0: past the end)
__device__ __forceinline__ void tile_rows(const TilePlan& tp, i64 t, i64 rows, i64& r0, int& R)
{
    if (t < tp.nfull) { r0 = t * 32; R = (int)min((i64)32, rows - r0); }
    else { r0 = tp.nfull * 32 + (t - tp.nfull) * 16; R = (int)min((i64)16, rows - r0); }
}

// MAX_row tree (R22): levels ping-pong in A/B (stride H = ceil(cols/2));
// the last level writes mx[rr].  Steps s + 2*lv (LTZ), s + 2*lv + 1 (mux BM).
// A holds levels 0, 2, 4.. (stride HA = ceil(cols/2)), B levels 1, 3, .. (stride HB = ceil(HA/2)).
// cone: the level's LTZs use the carry-cone circuit, CG groups per warp (ltz_cone.cuh).
template <bool WIDE, bool CONE, class P, bool CAUSAL = false, bool RBL = false>
__device__ __forceinline__ void tile_max(P& pr, u32 s, int w, SP in, i64 ldi, i64 cols, int R, u64 g0,
                                         SO A, SO B, i64 HA, i64 HB, SO mx, ConeSmem<CG, WIDE ? 64 : 32>* cone,
                                         u64 cL = 0)
{
    using S = typename P::S;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
    i64 m = cols;
    int lv = 0;
    SP cur = in;
    i64 li = ldi;
    // level-0 entry (row rr, column col); causal softmax: columns past the row's
    // position g mod cols enter as the public constant cL (party 0 holds it)
    u32 g0m = 0;                                   // g0 mod cols, once per tile (positions g0m + rr, rr < 32)
    FastDiv dcol{};
    if constexpr (CAUSAL) { g0m = (u32)(g0 % (u64)cols); dcol = make_fastdiv((u32)cols); }
    auto ldc = [&](i64 rr, i64 col) -> S {
        if constexpr (CAUSAL) {
            const u32 v = g0m + (u32)rr, pos = v - fdiv(v, dcol) * (u32)cols;
            if (lv == 0 && col > (i64)pos) return pr.addp(pr.zero(), cL);
        }
        return pr.ld(cur, rr * li + col);
    };
    // Warp-local levels: warp w owns rows [w rw, (w+1) rw) (rw = 32 / NW = 4).  When rw h is a
    // multiple of 32 (h % 8 == 0: every level of 128-wide rows down to h = 8, i.e. 120 of a tile's 127
    // comparison groups) the warp's units are whole LTZ groups of its own rows, so the level needs
    // no CTA barrier -- only the levels whose groups span warps (h = 4, 2, 1) synchronize the CTA.
    const int rw = 32 / NW;
#ifndef MPC_MAX_WARP_LOCAL
#define MPC_MAX_WARP_LOCAL 0   // measured 2 % slower on cfg2 (tools/ab_ops_quick.py, r02)
#endif
    auto warp_local = [&](i64 hh) { return MPC_MAX_WARP_LOCAL && 32 % NW == 0 && ((i64)rw * hh) % 32 == 0; };
    while (m > 1) {
        const i64 h = m / 2, mn = h + (m & 1);
        SO o; i64 lo;
        if (mn == 1) { o = mx; lo = 1; }
        else if (lv & 1) { o = B; lo = HB; }
        else { o = A; lo = HA; }
        const u32 sl = s + 2u * (u32)lv;
        const u64 ubase = g0 * (u64)h;                 // multiple of 32 for a full tile (g0 is); a half
        const int ua = (int)(ubase & 31);              // tile may start inside a group: ua lanes before it
        const u64 qb = ubase >> 5;
        const i64 nu = (i64)R * h;                     // the tile's units at this level
        const FastDiv dh = make_fastdiv((u32)h);
        const bool wl = warp_local(h) && R == 32 && ua == 0;
        const i64 gpw = (i64)rw * h / 32;              // groups per warp when warp-local
        const i64 gend = wl ? (warp + 1) * gpw : (ua + nu + 31) / 32;
        if constexpr (CONE) {
            constexpr int GB = CG;     // (one group per call in BOTH measured 4 % slower on softmax_cone)
            for (i64 gb = wl ? warp * gpw : (i64)warp * GB; gb < gend; gb += wl ? GB : (i64)NW * GB) {
                S d[GB], l[GB];
#pragma unroll
                for (int g = 0; g < GB; ++g) {
                    const i64 v = (gb + g) * 32 + lane - ua;
                    d[g] = pr.zero();
                    if (gb + g < gend && v >= 0 && v < nu) {
                        const i64 rr = fdiv((u32)v, dh), i = v - rr * h;
                        d[g] = pr.sub(ldc(rr, i), ldc(rr, i + h));
                    }
                }
                pr.template ltz_cone<GB, WIDE ? 64 : 32>(qb + (u64)gb, sl, w, d, l, lane,
                                                         *reinterpret_cast<ConeSmem<GB, WIDE ? 64 : 32>*>(&cone[warp]));
#pragma unroll
                for (int g = 0; g < GB; ++g) {
                    const i64 v = (gb + g) * 32 + lane - ua;
                    const bool valid = gb + g < gend && v >= 0 && v < nu;
                    i64 rr = 0, i = 0;
                    S y = pr.zero();
                    if (valid) { rr = fdiv((u32)v, dh); i = v - rr * h; y = ldc(rr, i + h); }
                    const S sel = pr.add(y, pr.bm(ubase + (u64)v, sl + 1, d[g], pr.notb(l[g])));
                    if (valid) {
                        pr.st(o, rr * lo + i, sel);
                        if ((m & 1) && i == h - 1) pr.st(o, rr * lo + h, ldc(rr, m - 1));
                    }
                }
            }
        } else {
            for (i64 g = wl ? warp * gpw : warp; g < gend; g += wl ? 1 : NW) {
                const i64 v = g * 32 + lane - ua;
                const bool valid = v >= 0 && v < nu;
                i64 rr = 0, i = 0;
                S d = pr.zero(), y = pr.zero();
                if (valid) {
                    rr = fdiv((u32)v, dh); i = v - rr * h;
                    y = ldc(rr, i + h);
                    d = pr.sub(ldc(rr, i), y);
                }
                const u64 q = qb + (u64)g;
#ifndef MPC_MAXTREE_REBAL
#define MPC_MAXTREE_REBAL 0      // A/B: the softmax / max tree with the rebalanced w = 33 LTZ
#endif
                const S c = pr.notb((MPC_MAXTREE_REBAL || RBL) ? pr.template ltz_rb<WIDE>(q, sl, w, d, lane)
                                                               : pr.template ltz_o<WIDE>(q, sl, w, d, lane));
                const S sel = pr.add(y, pr.bm(ubase + (u64)v, sl + 1, d, c));
                if (valid) {
                    pr.st(o, rr * lo + i, sel);
                    if ((m & 1) && i == h - 1) pr.st(o, rr * lo + h, ldc(rr, m - 1));
                }
            }
        }
        if (wl && mn > 1 && warp_local(mn / 2)) __syncwarp();   // next level reads only this warp's rows
        else __syncthreads();
        cur = SP{{o.p[0], o.p[1]}};
        li = lo;
        m = mn;
        ++lv;
    }
    if (cols == 1) {
        for (int rr = threadIdx.x; rr < R; rr += blockDim.x) pr.st(mx, rr, pr.ld(in, rr * ldi));
        __syncthreads();
    }
}

// ---- BOTH mode: the per-row Newton-Raphson chain with its triples generated ahead ----------------
// The NR chain (exp squarings + iters x 2 (recip) / 3 (rsqrt) Beaver steps on the tile's 32 row
// units) is one warp's serial dependency chain, and each step used to wait on its own 2.5 Philox
// blocks.  The triples are data-independent, so ALL warps of the CTA generate them first (nr_pregen,
// unit pairs: 5 blocks per pair and Beaver step, the contract's c0 sharing) into a
// shared-memory table; the chain (warp 0, BothTabP) then only opens and forms the shares.  Same
// steps, units, PRG words and output bits as recip_group / rsqrt_group on BothP.  Clamped exp
// (an LTZ inside the chain) keeps the direct path.
constexpr int NR_TAB_F = 5;                           // words per (step, row): a0 b0 c0 a b (square: a0 - c0 a)
__host__ __device__ inline int nr_tab_steps(int kind, int t, int iters) { return t + (kind ? 3 : 2) * iters; }
#ifndef MPC_NR_TAB_MAX_STEPS
#define MPC_NR_TAB_MAX_STEPS 32                       // 32 steps x 32 rows x 5 words = 40 KB of shared memory
#endif
template <int KIND>
__device__ __forceinline__ void nr_pregen(const Keys& K, u32 s, const NrK& p, u64 g0, u64* T, int nrows = 32)
{
    // the table's first nrows rows (unit pairs; the chain reads rows < R only)
    const int t = p.exp.t, ns = nr_tab_steps(KIND, t, p.iters), np = (min(nrows, 32) + 1) / 2;
    for (int it = threadIdx.x; it < ns * np; it += blockDim.x) {
        const int j = it / np, l = 2 * (it - j * np);
        const u64 u = g0 + (u64)l;                    // even (g0 is a multiple of 32)
        const u32 sj = s + (u32)j;
        u64* R = T + (i64)j * NR_TAB_F * 32 + l;
        if (j < t && p.exp.sq) {                      // square-pair triple
            const uint4 A0u = prg(K.k0, u, sj, 2), A0v = prg(K.k0, u + 1, sj, 2), A1 = prg(K.k1, u >> 1, sj, 3);
            R[0] = w64(A0u.x, A0u.y); R[1] = w64(A0v.x, A0v.y);
            R[64] = w64(A0u.z, A0u.w); R[65] = w64(A0v.z, A0v.w);
            R[96] = R[0] + w64(A1.x, A1.y); R[97] = R[1] + w64(A1.z, A1.w);
        } else {                                      // Beaver triple
            const uint4 A0u = prg(K.k0, u, sj, 0), A1u = prg(K.k1, u, sj, 0);
            const uint4 A0v = prg(K.k0, u + 1, sj, 0), A1v = prg(K.k1, u + 1, sj, 0);
            const uint4 C = prg(K.k0, u >> 1, sj, 1);
            R[0] = w64(A0u.x, A0u.y); R[1] = w64(A0v.x, A0v.y);
            R[32] = w64(A0u.z, A0u.w); R[33] = w64(A0v.z, A0v.w);
            R[64] = w64(C.x, C.y); R[65] = w64(C.z, C.w);
            R[96] = R[0] + w64(A1u.x, A1u.y); R[97] = R[1] + w64(A1v.x, A1v.y);
            R[128] = R[32] + w64(A1u.z, A1u.w); R[129] = R[33] + w64(A1v.z, A1v.w);
        }
    }
}
// BothP with bm / sq of the chain's steps read from the table (lane <-> row unit g0 + lane)
struct BothTabP : BothP {
    const u64* T; u32 sb;
    __device__ __forceinline__ S bm(u64, u32 s, S x, S y) const {
        const u64* R = T + (i64)(s - sb) * NR_TAB_F * 32 + (threadIdx.x & 31);
        const u64 a0 = R[0], b0 = R[32], c0 = R[64], a = R[96], b = R[128];
        const u64 X = x.s0 + x.s1, Y = y.s0 + y.s1;
        const u64 e = X - a, f = Y - b;               // open(x - a), open(y - b)
        const u64 z0 = c0 + e * (b0 + f) + f * a0;    // = mpc::bm_with_c0
        return {z0, X * Y - z0};
    }
    __device__ __forceinline__ S sq(u64, u32 s, S y) const {
        const u64* R = T + (i64)(s - sb) * NR_TAB_F * 32 + (threadIdx.x & 31);
        const u64 a0 = R[0], c0 = R[64], a = R[96];
        const u64 Y = y.s0 + y.s1, e = Y - a;
        const u64 z0 = c0 + e * (2ull * a0 + e);      // = mpc::sq_with_a1
        return {z0, Y * Y - z0};
    }
};

// per-row Newton-Raphson over the tile's rows: warp 0, lane <-> row (LTZ group = the tile)
// tab (BOTH mode only): the chain's triples, already generated by nr_pregen<KIND> for (s, g0)
// R > 32 (the balanced softmax plan, BOTH): warp w < ceil(R / 32) runs rows 32 w + lane (units g0 + 32 w
// + lane) from the w-th table (tab + w * tab2)
template <int KIND, bool WIDE, class P>
__device__ __forceinline__ void tile_nr(P& pr, u32 s, const NrK& p, int R, u64 g0, SP x, SO y, const u64* tab = nullptr,
                                        i64 tab2 = 0)
{
    const int warp = threadIdx.x >> 5;
    if (warp == 0 || 32 * warp < R) {
        const int lane = threadIdx.x & 31, row = (int)threadIdx.x;
        const u64 gw = g0 + 32u * (u64)warp;
        const bool valid = row < R;
        typename P::S xv = pr.zero();
        if (valid) xv = pr.ld(x, row);
        typename P::S r;
        bool done = false;
        if constexpr (!P::kPair) {
            if (tab) {
                BothTabP tp;
                tp.Kp = pr.Kp; tp.T = tab + warp * tab2; tp.sb = s;
                if (KIND == 0) r = recip_group<WIDE>(tp, gw + lane, gw >> 5, s, p, xv, lane);
                else r = rsqrt_group<WIDE>(tp, gw + lane, gw >> 5, s, p, xv, lane);
                done = true;
            }
        }
        if (!done) {
            if (KIND == 0) r = recip_group<WIDE>(pr, gw + lane, gw >> 5, s, p, xv, lane);
            else r = rsqrt_group<WIDE>(pr, gw + lane, gw >> 5, s, p, xv, lane);
        }
        if (valid) pr.st(y, row, r);
    }
    __syncthreads();
}

// L2 prefetch of the next tile's input rows (rows [r0n, r0n + 32) of a rows x C share array)
__device__ __forceinline__ void prefetch_rows(SP x, i64 r0n, i64 rows, i64 C)
{
    if (!MPC_GROUP_PREFETCH || r0n >= rows) return;
    const i64 nel = (rows - r0n < 32 ? rows - r0n : 32) * C;
    for (i64 l = (i64)threadIdx.x * 16; l < nel; l += (i64)blockDim.x * 16)       // one 128-B line each
#pragma unroll
        for (int q = 0; q < 2; ++q)
            if (x.p[q]) asm volatile("prefetch.global.L2 [%0];" :: "l"(x.p[q] + r0n * C + l));
}

// out = MT(x, bcast r) over a tile of R rows x C with the BROADCAST triple (NEXT #2, DESIGN.md
// 2.8): warp 0 opens f = r - b for the tile's 32 rows (lane <-> row, one round), the CTA then
// forms the element products (e = x - a opened per element) on unit pairs.  val(e, row) yields
// the element's share.  brs: 3 x 32 u64 of shared / per-CTA scratch (b0, b1, f per row).
template <class P, class Val>
__device__ __forceinline__ void tile_bcast_mul(P& pr, u32 s, int R, i64 C, u64 g0, const FastDiv& dC,
                                               SP Rr, SO zt, u64* brs, Val val, int BS = 32)
{
    using S = typename P::S;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
    if (warp == 0 || 32 * warp < R) {                   // BS > 32 (balanced plan): warp w < ceil(R / 32)
        const int row = (int)threadIdx.x;
        const S y = row < R ? pr.ld(Rr, row) : pr.zero();
        const BRow b = pr.bmb_row(g0 + (u64)row, s, y);
        if (row < BS) { brs[row] = b.b0; brs[BS + row] = b.b1; brs[2 * BS + row] = b.f; }
    }
    __syncthreads();
    const i64 ne = (i64)R * C;
    const u64 ub = g0 * (u64)C;                         // even: g0 is a multiple of 32
    for (i64 base = (i64)warp * 32; base < (ne + 1) / 2; base += (i64)NW * 32) {
        const i64 e = 2 * (base + lane);
        S xa = pr.zero(), xb = pr.zero();
        int ra = 0, rb = 0;
        if (e < ne) { ra = (int)fdiv((u32)e, dC); xa = val(e, ra); }
        if (e + 1 < ne) { rb = (int)fdiv((u32)(e + 1), dC); xb = val(e + 1, rb); }
        const BRow b0{brs[ra], brs[BS + ra], brs[2 * BS + ra]}, b1{brs[rb], brs[BS + rb], brs[2 * BS + rb]};
        S za, zb;
        pr.bmb2(ub + (u64)e, s, xa, xb, b0, b1, za, zb);
        if (e < ne) pr.st(zt, e, pr.shr_(za, FRAC));
        if (e + 1 < ne) pr.st(zt, e + 1, pr.shr_(zb, FRAC));
    }
}

struct SoftmaxArgs {
    u32 s_max, s_exp, s_rec, s_mul;
    int w;
    ExpK ek;
    NrK rk;
    SP x;
    SO z;
    i64 rows, cols;
    u64 row_off;
    u64* gscratch;          // per-CTA work tiles when they do not fit in shared memory
    i64 work_u64;           // u64 words of one work tile
    int use_smem;
    u64* escratch;          // per-CTA exp tile E (2 x 32 x cols), global (L2-resident)
    int cone;               // carry-cone LTZ in the max tree (NEXT #1)
    int bcast;              // broadcast triple for the final e * r (NEXT #2)
    int esmem;              // E tile in the work area (aliasing the dead max-tree levels), not escratch
    int causal;             // causal attention rows
    u64 causal_L;           // public constant of the masked max-tree inputs, -2^(w-2)
    int nrtab;              // BOTH: the reciprocal chain's triples pre-generated into smem (nr_pregen)
    int half;               // tail tiles as 16-row half tiles (tile_plan)
    int bal;                // BOTH balanced plan: ONE row range of <= tr rows per CTA (softmax_bal_*)
    int tr;                 // rows per CTA capacity of the balanced plan
    i64 tab_u64;            // balanced plan: u64 words of one 32-row NR table
    i64 nrange;             // balanced plan: ranges (0: one per CTA; k x grid: k rounds per CTA)
};

// Balanced plan (BOTH, no clamp / broadcast triple / cone): CTA c of ncta owns rows
// [2 floor(c hr / ncta), 2 floor((c+1) hr / ncta)), hr = ceil(rows / 2) -- every CTA resident at once,
// each SM ~rows / #SMs rows (cfg2: 41-42 rows per CTA instead of 384 32-row tiles on 296 CTAs, whose
// last round left 88 SMs with a third tile).  Work area: the max-tree levels A0 A1 B0 B1 (2 tr HA +
// 2 tr HB), aliased after the tree by the reciprocal chains' triple tables (two 32-row tables); then
// X: MX0 MX1 S0 S1 R0 R1 (6 tr).  E (2 x tr x cols) lives in the per-CTA global escratch (L2).
__host__ __device__ inline i64 softmax_bal_x_off(i64 cols, i64 tr, i64 tab_u64)
{
    const i64 HA = (cols + 1) / 2, HB = (HA + 1) / 2, lv = 2 * tr * (HA + HB);
    return lv > 2 * tab_u64 ? lv : 2 * tab_u64;
}
__host__ __device__ inline i64 softmax_bal_work_u64(i64 cols, i64 tr, i64 tab_u64)
{
    return softmax_bal_x_off(cols, tr, tab_u64) + 9 * tr;        // X: MX S R (6 tr), broadcast rows (3 tr)
}

// work tile (u64 words), HA = ceil(cols/2), HB = ceil(HA/2): A0 A1 (2 x 32HA), B0 B1 (2 x 32HB),
// then at softmax_x_off: MX0 MX1 S0 S1 R0 R1 (6 x 32), broadcast-triple rows b0 b1 f (3 x 32).
// With esmem the exp tile E (2 x 32 x cols) reuses the max-tree levels' space (they are dead
// once the row maxima are in MX), so X starts after max(64 HA + 64 HB, 64 cols); otherwise E
// lives in the per-CTA global escratch (L2).
__host__ __device__ inline i64 softmax_x_off(i64 cols, bool esmem)
{
    const i64 HA = (cols + 1) / 2, HB = (HA + 1) / 2;
    return esmem ? (64 * cols > 64 * HA + 64 * HB ? 64 * cols : 64 * HA + 64 * HB) : 64 * HA + 64 * HB;
}
__host__ __device__ inline i64 softmax_work_u64(i64 cols, bool esmem = false, i64 tab_u64 = 0)
{
    return softmax_x_off(cols, esmem) + 9 * 32 + tab_u64;   // [.. X (9 x 32)] [NR triple table]
}

#ifndef MPC_SOFTMAX_EXP_V
#define MPC_SOFTMAX_EXP_V 1    // BOTH: unit pairs per thread and pass in the softmax exp phase
#endif
// LV: 0 Kogge-Stone LTZ (w <= 33), 1 Kogge-Stone wide (w > 33), 2 carry cone (w <= 33), 3 carry cone
// wide (w <= 64) -- separate instantiations so the cone's registers / shared memory do not cost the
// others occupancy
template <int LV, class PA, bool CAUSAL = false>
__global__ void __launch_bounds__(MPC_ROW_TPB, LV == 0 ? MPC_SM_MINB_KS : MPC_SM_MINB) k_softmax(const __grid_constant__ PA pa, SoftmaxArgs a)
{
    constexpr bool WIDE = LV == 1 || LV == 3, CONE = LV >= 2;
    extern __shared__ __align__(16) u64 smem[];
    __shared__ ConeSmem<CG, WIDE ? 64 : 32> cone_sm[CONE ? MPC_ROW_TPB / 32 : 1];
    int cta, ncta;
    auto pr = pa.make(cta, ncta);
    using S = typename decltype(pr)::S;
    // loopback: the two parties' CTAs need separate tiles of scratch
    const int wslot = blockIdx.x;
    u64* W = a.use_smem ? smem : a.gscratch + (i64)wslot * a.work_u64;
    const i64 C = a.cols, HA = (C + 1) / 2, HB = (HA + 1) / 2;
    const i64 TR = a.bal ? a.tr : 32;                             // rows per tile capacity
    SO A{{W, W + TR * HA}}, B{{W + 2 * TR * HA, W + 2 * TR * HA + TR * HB}};
    u64* Ew = a.esmem ? W : a.escratch + (i64)wslot * 2 * TR * C;
    SO E{{Ew, Ew + TR * C}};
    u64* X = W + (a.bal ? softmax_bal_x_off(C, TR, a.tab_u64) : softmax_x_off(C, a.esmem != 0));
    SO MX{{X, X + TR}}, SS{{X + 2 * TR, X + 3 * TR}}, RR{{X + 4 * TR, X + 5 * TR}};
    // balanced plan: the triple tables alias the dead level buffers in shared memory, or (global work
    // area, wide rows) are the dynamic shared memory itself
    u64* const nrt = a.nrtab ? (a.bal ? (a.use_smem ? W : smem) : X + 9 * 32) : nullptr;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
    const TilePlan tp = tile_plan(a.rows, ncta, a.half);
    const FastDiv dC = make_fastdiv((u32)C);
    // balanced plan: nrange ranges (a multiple of the grid: k equal rounds per CTA), default one per CTA
    const i64 ntl = a.bal ? (a.nrange > 0 ? a.nrange : (i64)ncta) : tp.ntot;
    for (i64 tile = cta; tile < ntl; tile += ncta) {
        i64 r0; int R;
        if (a.bal) {
            const i64 hr = (a.rows + 1) / 2;
            r0 = min(a.rows, 2 * (tile * hr / ntl));
            R = (int)(min(a.rows, 2 * ((tile + 1) * hr / ntl)) - r0);
            if (R <= 0) continue;
        } else {
            tile_rows(tp, tile, a.rows, r0, R);
            if (R <= 0) break;
        }
        const u64 g0 = a.row_off + (u64)r0;                       // global row of the tile
        const SP xt{{a.x.p[0] ? a.x.p[0] + r0 * C : nullptr, a.x.p[1] ? a.x.p[1] + r0 * C : nullptr}};
        // (no next-tile prefetch here: measured neutral to 0.6 % slower for softmax, 2 % faster for k_max)
        // 1. m = MAX_row(x)
#ifndef MPC_SOFTMAX_SKIP
#define MPC_SOFTMAX_SKIP 0   // profiling only: bitmask of phases to skip (1 max, 2 exp, 4 recip, 8 mul)
#endif
        if (!(MPC_SOFTMAX_SKIP & 1))
        tile_max<WIDE, CONE, decltype(pr), CAUSAL>(pr, a.s_max, a.w, xt, C, C, R, g0, A, B, HA, HB, MX, cone_sm, a.causal_L);
        // BOTH: every warp generates the reciprocal chain's triples now (tile_nr's warp-0 chain then
        // only opens and multiplies); the exp phase's closing barrier orders it before the chain
        if constexpr (!decltype(pr)::kPair)
            if (nrt)                                              // one 32-row table per 32 rows (<= 3)
                for (int t = 0; 32 * t < R; ++t)
                    nr_pregen<0>(*pr.Kp, a.s_rec, a.rk, g0 + 32u * (u64)t, nrt + t * a.tab_u64, R - 32 * t);
        // 2-3. e = EXP(x - m), element units g0*C + e
        const i64 ne = (i64)R * C;
        const u64 ub = g0 * (u64)C;
        const SP MXc{{MX.p[0], MX.p[1]}};
        if (MPC_SOFTMAX_SKIP & 2) {
        } else if (a.ek.clamp) {
            // clamp head in the LTZ group layout, then the squarings in the pair layout (E in place)
            for (i64 g = warp; g < (ne + 31) / 32; g += NW) {
                const i64 e = g * 32 + lane;
                const bool valid = e < ne;
                S d = pr.zero();
                if (valid) d = pr.sub(pr.ld(xt, e), pr.ld(MXc, fdiv((u32)e, dC)));
                const S y = exp_clamp_head<WIDE>(pr, ub + e, (ub >> 5) + g, a.s_exp, a.ek, d, lane);
                if (valid) pr.st(E, e, y);
            }
            __syncthreads();
            const SP Ec{{E.p[0], E.p[1]}};
            constexpr int V = decltype(pr)::kV;
            for (i64 base = (i64)warp * 32 * V; base < (ne + 1) / 2; base += (i64)NW * 32 * V) {
                u64 uv[V];
                S da[V], db[V];
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const i64 e = 2 * (base + lane + 32 * v);
                    uv[v] = ub + (u64)e;
                    da[v] = db[v] = pr.zero();
                    if (e < ne) da[v] = pr.ld(Ec, e);
                    if (e + 1 < ne) db[v] = pr.ld(Ec, e + 1);
                }
                exp_squarings_pairv<V>(pr, uv, a.s_exp + 2, a.ek, da, db);
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const i64 e = 2 * (base + lane + 32 * v);
                    if (e < ne) pr.st(E, e, da[v]);
                    if (e + 1 < ne) pr.st(E, e + 1, db[v]);
                }
            }
        } else {
            constexpr int V = decltype(pr)::kPair ? decltype(pr)::kV : MPC_SOFTMAX_EXP_V;   // BOTH: A/B knob
            for (i64 base = (i64)warp * 32 * V; base < (ne + 1) / 2; base += (i64)NW * 32 * V) {
                u64 uv[V];
                S da[V], db[V];
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const i64 e = 2 * (base + lane + 32 * v);
                    uv[v] = ub + (u64)e;
                    pr.ld_pair(xt, e, e < ne, e + 1 < ne, da[v], db[v]);      // 16-byte loads (row pairs)
                    if (e < ne) da[v] = pr.sub(da[v], pr.ld(MXc, fdiv((u32)e, dC)));
                    if (e + 1 < ne) db[v] = pr.sub(db[v], pr.ld(MXc, fdiv((u32)(e + 1), dC)));
                }
                exp_pairv<V>(pr, uv, a.s_exp, a.ek, da, db);
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const i64 e = 2 * (base + lane + 32 * v);
                    pr.st_pair(E, e, e < ne, e + 1 < ne, da[v], db[v]);
                }
            }
        }
        __syncthreads();
        // causal: the masked exponentials are the public 0
        const u32 g0m = CAUSAL ? (u32)(g0 % (u64)C) : 0u;
        auto masked = [&](i64 e) {
            const u32 rr = fdiv((u32)e, dC), v = g0m + rr;
            return (u32)e - rr * (u32)C > v - fdiv(v, dC) * (u32)C;
        };
        if constexpr (CAUSAL) {
            for (i64 e = threadIdx.x; e < ne; e += blockDim.x)
                if (masked(e)) pr.st(E, e, pr.zero());
            __syncthreads();
        }
        // 4. S = rowsum(e) (local): warp per row
        const SP Ec{{E.p[0], E.p[1]}};
        for (int rr = warp; rr < R; rr += NW) {
            S acc = pr.zero();
            for (i64 j = lane; j < C; j += 32) acc = pr.add(acc, pr.ld(Ec, rr * C + j));
            acc = pr.sumw(acc);
            if (lane == 0) pr.st(SS, rr, acc);
        }
        __syncthreads();
        // 5. r = RECIP(S), row units
        if (!(MPC_SOFTMAX_SKIP & 4)) tile_nr<0, WIDE>(pr, a.s_rec, a.rk, R, g0, SP{{SS.p[0], SS.p[1]}}, RR, nrt, a.tab_u64);
        // 6. out = MT(e, r), element units
        const SP Rc{{RR.p[0], RR.p[1]}};
        const SO zt{{a.z.p[0] ? a.z.p[0] + r0 * C : nullptr, a.z.p[1] ? a.z.p[1] + r0 * C : nullptr}};
        if (a.bcast) {
            tile_bcast_mul(pr, a.s_mul, R, C, g0, dC, Rc, zt, X + 6 * TR, [&](i64 e, int) { return pr.ld(Ec, e); }, (int)TR);
        } else if (!(MPC_SOFTMAX_SKIP & 8)) {
            constexpr int V = decltype(pr)::kV;
            for (i64 base = (i64)warp * 32 * V; base < (ne + 1) / 2; base += (i64)NW * 32 * V) {
                u64 uv[V];
                S ea[V], eb[V], ra[V], rb[V], za[V], zb[V];
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const i64 e = 2 * (base + lane + 32 * v);
                    uv[v] = ub + (u64)e;
                    ra[v] = rb[v] = pr.zero();
                    pr.ld_pair(Ec, e, e < ne, e + 1 < ne, ea[v], eb[v]);
                    if (e < ne) ra[v] = pr.ld(Rc, fdiv((u32)e, dC));
                    if (e + 1 < ne) rb[v] = pr.ld(Rc, fdiv((u32)(e + 1), dC));
                }
                pr.template bm2v<V>(uv, a.s_mul, ea, ra, eb, rb, za, zb);
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const i64 e = 2 * (base + lane + 32 * v);
                    pr.st_pair(zt, e, e < ne, e + 1 < ne, pr.shr_(za[v], FRAC), pr.shr_(zb[v], FRAC));
                }
            }
        }
        if constexpr (CAUSAL) {                           // masked outputs: the public 0
            __syncthreads();
            for (i64 e = threadIdx.x; e < ne; e += blockDim.x)
                if (masked(e)) pr.st(zt, e, pr.zero());
        }
        __syncthreads();
    }
    pa.done(pr);
}

struct MaxArgs {
    u32 s; int w; SP x; SO z; i64 rows, cols; u64 row_off;
    u64* gscratch; i64 work_u64; int use_smem;
    u64* escratch; int cone;
    int half;               // tail tiles as 16-row half tiles (tile_plan)
    int tr;                 // > 0: the balanced plan (k_softmax's): one range of <= tr rows per CTA
    i64 nrange;             // balanced plan: ranges (0: one per CTA; k x grid: k rounds per CTA)
};
__host__ __device__ inline i64 max_work_u64(i64 cols, i64 tr = 32)
{
    const i64 HA = (cols + 1) / 2, HB = (HA + 1) / 2;
    return 2 * tr * HA + 2 * tr * HB + 2 * tr;
}

template <int LV, class PA>   // LV as k_softmax
__global__ void __launch_bounds__(MPC_ROW_TPB, LV == 0 ? MPC_SM_MINB_KS : MPC_SM_MINB) k_max(const __grid_constant__ PA pa, MaxArgs a)
{
    constexpr bool WIDE = LV == 1 || LV == 3, CONE = LV >= 2;
    extern __shared__ __align__(16) u64 smem[];
    __shared__ ConeSmem<CG, WIDE ? 64 : 32> cone_sm[CONE ? MPC_ROW_TPB / 32 : 1];
    int cta, ncta;
    auto pr = pa.make(cta, ncta);
    u64* W = a.use_smem ? smem : a.gscratch + (i64)blockIdx.x * a.work_u64;
    const i64 C = a.cols, HA = (C + 1) / 2, HB = (HA + 1) / 2;
    const i64 TR = a.tr > 0 ? a.tr : 32;
    SO A{{W, W + TR * HA}}, B{{W + 2 * TR * HA, W + 2 * TR * HA + TR * HB}};
    SO MX{{W + 2 * TR * HA + 2 * TR * HB, W + 2 * TR * HA + 2 * TR * HB + TR}};
    const TilePlan tp = tile_plan(a.rows, ncta, a.half);
    const i64 ntl = a.tr > 0 ? (a.nrange > 0 ? a.nrange : (i64)ncta) : tp.ntot;
    for (i64 tile = cta; tile < ntl; tile += ncta) {
        i64 r0; int R;
        if (a.tr > 0) {                                   // balanced plan (k_softmax's softmax_bal_*)
            const i64 hr = (a.rows + 1) / 2;
            r0 = min(a.rows, 2 * (tile * hr / ntl));
            R = (int)(min(a.rows, 2 * ((tile + 1) * hr / ntl)) - r0);
            if (R <= 0) continue;
        } else {
            tile_rows(tp, tile, a.rows, r0, R);
            if (R <= 0) break;
        }
        const SP xt{{a.x.p[0] ? a.x.p[0] + r0 * C : nullptr, a.x.p[1] ? a.x.p[1] + r0 * C : nullptr}};
        if (a.tr <= 0) prefetch_rows(a.x, r0 + (i64)ncta * 32, a.rows, C);
        // standalone max (and softmax's split max pass): the rebalanced w = 33 LTZ (k_max has the registers)
        tile_max<WIDE, CONE, decltype(pr), false, true>(pr, a.s, a.w, xt, C, C, R, a.row_off + (u64)r0, A, B, HA, HB, MX, cone_sm);
        const SP MXc{{MX.p[0], MX.p[1]}};
        const SO zt{{a.z.p[0] ? a.z.p[0] + r0 : nullptr, a.z.p[1] ? a.z.p[1] + r0 : nullptr}};
        for (int rr = threadIdx.x; rr < R; rr += blockDim.x) pr.st(zt, rr, pr.ld(MXc, rr));
        __syncthreads();
    }
    pa.done(pr);
}

// mpc_mul_bcast (NEXT #2): rows' masks and openings (warp <-> 32 rows), then the
// element products on unit pairs (pairs driver) reading the row records.
struct BmbRowsArgs { u32 s; SP y; i64 rows; u64 row_off; u64* br; int loop; };   // br: [3][rows] ([2][3][rows] in loopback)
template <class PA>
__global__ void __launch_bounds__(256, MPC_EW_MINB) k_bmb_rows(const __grid_constant__ PA pa, BmbRowsArgs a)
{
    int cta, ncta;
    auto pr = pa.make(cta, ncta);
    const int lane = threadIdx.x & 31, NW = blockDim.x >> 5;
    const i64 ng = (a.rows + 31) >> 5;
    for (i64 g = (i64)cta * NW + (threadIdx.x >> 5); g < ng; g += (i64)ncta * NW) {
        const i64 r = g * 32 + lane;
        const typename decltype(pr)::S y = r < a.rows ? pr.ld(a.y, r) : pr.zero();
        const BRow b = pr.bmb_row(a.row_off + (u64)r, a.s, y);
        u64* br = a.br + (a.loop && pr.party() > 0 ? 3 * a.rows : 0);   // loopback: one record set per party
        if (r < a.rows) { br[r] = b.b0; br[a.rows + r] = b.b1; br[2 * a.rows + r] = b.f; }
    }
    pa.done(pr);
}
struct BmbBody {
    u32 s; SP x; SO z; i64 n; FastDiv dC; const u64* br; i64 rows; int tb; int loop;
    SP mu; int has_mu;      // LayerNorm: the left operand is x - mu[row] (k_ln_stats' means)
    template <int V, class P>
    __device__ void run(P& pr, const u64 (&u)[V], const i64 (&i0)[V], const bool (&ok)[V]) const {
        using S = typename P::S;
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const bool va = ok[v] && i0[v] >= 0, vb = ok[v] && i0[v] + 1 < n;
            S xa = pr.zero(), xb = pr.zero();
            i64 ra = 0, rb = 0;
            if (va) { ra = fdiv((u32)i0[v], dC); xa = pr.ld(x, i0[v]); if (has_mu) xa = pr.sub(xa, pr.ld(mu, ra)); }
            if (vb) { rb = fdiv((u32)(i0[v] + 1), dC); xb = pr.ld(x, i0[v] + 1); if (has_mu) xb = pr.sub(xb, pr.ld(mu, rb)); }
            const u64* bp = br + (loop && pr.party() > 0 ? 3 * rows : 0);   // loopback: party 1's records
            const BRow b0{bp[ra], bp[rows + ra], bp[2 * rows + ra]}, b1{bp[rb], bp[rows + rb], bp[2 * rows + rb]};
            S za, zb;
            pr.bmb2(u[v], s, xa, xb, b0, b1, za, zb);
            if (va) pr.st(z, i0[v], pr.shr_(za, tb));
            if (vb) pr.st(z, i0[v] + 1, pr.shr_(zb, tb));
        }
    }
};

// Short-row MAX_row (cols <= MAXS_COLS; MaxPool windows).  The same contract as k_max (R22:
// half-split tree with the odd entry carried, LTZ at step s + 2 lv and the mux at s + 2 lv + 1,
// units row * h + i), but ONE WARP owns a 32-row tile: a 3x3 window's levels have h = 4, 2, 1,
// 1 groups per tile, which would leave most of a CTA's warps idle at its level barriers.  The
// warp's tile lives in its own shared-memory slice (levels in place: a level writes only
// positions i < h, which no other unit of the level reads; the odd carry moves after the level)
// and MaxPool gathers its k x k windows (public zero padding, R26) straight from the NCHW input.
constexpr int MAXS_COLS = 16;
struct MaxSmallArgs {
    u32 s; int w; SP x; SO z; i64 rows, cols; u64 row_off;
    int pool, k, stride, pad, H, W;
    FastDiv fcol, fk, fwo, fho;        // cols, k, Wo, Ho
};
template <int LV, class PA>
__global__ void __launch_bounds__(256, MPC_EW_MINB) k_max_small(const __grid_constant__ PA pa, MaxSmallArgs a)
{
    constexpr bool WIDE = LV == 1 || LV == 3, CONE = LV >= 2;
    constexpr int NL = WIDE ? 64 : 32;
    extern __shared__ __align__(16) u64 smem[];                 // per warp: 2 parties x 32 rows x cols
    __shared__ ConeSmem<CG, NL> cone_sm[CONE ? 8 : 1];
    int cta, ncta;
    auto pr = pa.make(cta, ncta);
    using S = typename decltype(pr)::S;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
    const int C = (int)a.cols;
    u64* wb = smem + (i64)warp * 64 * C;
    const SO X{{wb, wb + 32 * C}};
    const SP Xc{{wb, wb + 32 * C}};
    const i64 ntiles = (a.rows + 31) / 32;
    for (i64 tile = (i64)cta * NW + warp; tile < ntiles; tile += (i64)ncta * NW) {
        const i64 r0 = tile * 32;
        const int R = (int)min((i64)32, a.rows - r0);
        for (int t = lane; t < R * C; t += 32) {
            const u32 rr = fdiv((u32)t, a.fcol);
            const u32 e = (u32)t - rr * (u32)C;
            S v;
            if (a.pool) {                                      // window element e of output r0 + rr
                const u32 o = (u32)(r0 + rr);
                const u32 q1 = fdiv(o, a.fwo), ow = o - q1 * a.fwo.d;
                const u32 q2 = fdiv(q1, a.fho), oh = q1 - q2 * a.fho.d;     // q2 = img * C + c
                const u32 dy = fdiv(e, a.fk), dx = e - dy * a.fk.d;
                const int iy = (int)(oh * a.stride + dy) - a.pad, ix = (int)(ow * a.stride + dx) - a.pad;
                const bool in = iy >= 0 && iy < a.H && ix >= 0 && ix < a.W;
                v = in ? pr.ld(a.x, ((i64)q2 * a.H + iy) * a.W + ix) : pr.zero();
            } else {
                v = pr.ld(a.x, (r0 + rr) * (i64)C + e);
            }
            pr.st(X, t, v);
        }
        __syncwarp();
        const u64 g0 = a.row_off + (u64)r0;
        int m = C, lv = 0;
        while (m > 1) {
            const int h = m / 2;
            const u32 sl = a.s + 2u * (u32)lv;
            const u64 ubase = g0 * (u64)h;                     // multiple of 32 (g0 is)
            const FastDiv dh = make_fastdiv((u32)h);
            if constexpr (CONE) {
                for (int b = 0; b < h; b += CG) {
                    S d[CG], l[CG], y[CG];
                    int at[CG];
#pragma unroll
                    for (int g = 0; g < CG; ++g) {
                        const int v = (b + g) * 32 + lane;
                        d[g] = pr.zero(); y[g] = pr.zero(); at[g] = -1;
                        if (b + g < h && v < R * h) {
                            const int rr = (int)fdiv((u32)v, dh), i = v - rr * h;
                            at[g] = rr * C + i;
                            y[g] = pr.ld(Xc, at[g] + h);
                            d[g] = pr.sub(pr.ld(Xc, at[g]), y[g]);
                        }
                    }
                    const int ng = min(CG, h - b);
                    const u64 q = (ubase >> 5) + (u64)b;
                    if (ng == 3 || (ng == 4 && !(!decltype(pr)::kPair && MPC_MAXS_PAIRS))) {
                        pr.template ltz_cone<CG, NL>(q, sl, a.w, d, l, lane, cone_sm[warp]);
                    } else if (ng == 1) {
                        S d1[1] = {d[0]}, l1[1];
                        pr.template ltz_cone<1, NL>(q, sl, a.w, d1, l1, lane, *reinterpret_cast<ConeSmem<1, NL>*>(&cone_sm[warp]));
                        l[0] = l1[0];
                    } else if (ng == 2) {
                        S d2[2] = {d[0], d[1]}, l2[2];
                        pr.template ltz_cone<2, NL>(q, sl, a.w, d2, l2, lane, *reinterpret_cast<ConeSmem<2, NL>*>(&cone_sm[warp]));
                        l[0] = l2[0]; l[1] = l2[1];
                    } else if (!decltype(pr)::kPair && MPC_MAXS_PAIRS) {
                        // BOTH: two flat-triple calls of 2 groups (ltz_cone.cuh) instead of one of 4
                        S da[2] = {d[0], d[1]}, la[2], db[2] = {d[2], d[3]}, lb[2];
                        pr.template ltz_cone<2, NL>(q, sl, a.w, da, la, lane, *reinterpret_cast<ConeSmem<2, NL>*>(&cone_sm[warp]));
                        pr.template ltz_cone<2, NL>(q + 2, sl, a.w, db, lb, lane, *reinterpret_cast<ConeSmem<2, NL>*>(&cone_sm[warp]));
                        l[0] = la[0]; l[1] = la[1]; l[2] = lb[0]; l[3] = lb[1];
                    } else {
                        pr.template ltz_cone<CG, NL>(q, sl, a.w, d, l, lane, cone_sm[warp]);
                    }
#pragma unroll
                    for (int g = 0; g < CG; ++g) {
                        if (g >= ng) break;                    // warp-uniform
                        const S sel = pr.add(y[g], pr.bm(ubase + (u64)((b + g) * 32 + lane), sl + 1, d[g], pr.notb(l[g])));
                        if (at[g] >= 0) pr.st(X, at[g], sel);
                    }
                }
            } else {
                for (int g = 0; g < h; ++g) {                  // 32*h units = h groups
                    const int v = g * 32 + lane;
                    int at = -1;
                    S d = pr.zero(), y = pr.zero();
                    if (v < R * h) {
                        const int rr = (int)fdiv((u32)v, dh), i = v - rr * h;
                        at = rr * C + i;
                        y = pr.ld(Xc, at + h);
                        d = pr.sub(pr.ld(Xc, at), y);
                    }
                    const S c = pr.notb(pr.template ltz_rb<WIDE>((ubase >> 5) + (u64)g, sl, a.w, d, lane));
                    const S sel = pr.add(y, pr.bm(ubase + (u64)v, sl + 1, d, c));
                    if (at >= 0) pr.st(X, at, sel);
                }
            }
            __syncwarp();
            if (m & 1) {
                for (int rr = lane; rr < R; rr += 32) pr.st(X, rr * C + h, pr.ld(Xc, rr * C + m - 1));
                __syncwarp();
            }
            m = h + (m & 1);
            ++lv;
        }
        for (int rr = lane; rr < R; rr += 32) pr.st(a.z, r0 + rr, pr.ld(Xc, rr * C));
        __syncwarp();
    }
    pa.done(pr);
}

struct LnArgs {
    u32 s_sq, s_rs, s_mul; NrK rk; SP x; SO z; i64 rows, cols; u64 row_off;
    int mean_mode; u64 e_invd, e_eps;
    int bcast;              // broadcast triple for the final c * r (NEXT #2)
};

// LAYERNORM: mu, c = x - mu, v = mean(MT(c,c)) + eps, r = RSQRT(v), out = MT(c, r)
template <bool WIDE, class PA>
__global__ void __launch_bounds__(MPC_ROW_TPB, MPC_SM_MINB) k_ln(const __grid_constant__ PA pa, LnArgs a)
{
    __shared__ u64 MU[2][32], V[2][32], RS[2][32], BR[3 * 32];
    int cta, ncta;
    auto pr = pa.make(cta, ncta);
    using S = typename decltype(pr)::S;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
    const i64 C = a.cols;
    const i64 ntiles = (a.rows + 31) / 32;
    const FastDiv dC = make_fastdiv((u32)C);
    const SO MUo{{MU[0], MU[1]}}, Vo{{V[0], V[1]}}, RSo{{RS[0], RS[1]}};
    const SP MUc{{MU[0], MU[1]}}, Vc{{V[0], V[1]}}, RSc{{RS[0], RS[1]}};
    for (i64 tile = cta; tile < ntiles; tile += ncta) {
        const i64 r0 = tile * 32;
        const int R = (int)min((i64)32, a.rows - r0);
        const u64 g0 = a.row_off + (u64)r0;
        const SP xt{{a.x.p[0] ? a.x.p[0] + r0 * C : nullptr, a.x.p[1] ? a.x.p[1] + r0 * C : nullptr}};
        prefetch_rows(a.x, r0 + (i64)ncta * 32, a.rows, C);
        for (int rr = warp; rr < R; rr += NW) {
            S acc = pr.zero();
            for (i64 j = lane; j < C; j += 32) acc = pr.add(acc, pr.ld(xt, rr * C + j));
            S mu = pr.sumw(acc);
            mu = a.mean_mode == 0 ? pr.mulf(mu, a.e_invd) : pr.divp(mu, C);
            // q = MT(c, c) over the row, element units; lanes take unit pairs (2j, 2j+1)
            S qs = pr.zero();
            const u64 ub = (g0 + (u64)rr) * (u64)C;
            const i64 j0 = -(i64)(ub & 1);
            for (i64 j = j0 + 2 * lane, jb = j0; jb < C; j += 64, jb += 64) {
                const bool va = j >= 0 && j < C, vb = j + 1 >= 0 && j + 1 < C;
                S ca = pr.zero(), cb = pr.zero();
                if (va) ca = pr.sub(pr.ld(xt, rr * C + j), mu);
                if (vb) cb = pr.sub(pr.ld(xt, rr * C + j + 1), mu);
                S za, zb;
                pr.bm2(ub + (u64)j, a.s_sq, ca, ca, cb, cb, za, zb);
                if (va) qs = pr.add(qs, pr.shr_(za, FRAC));
                if (vb) qs = pr.add(qs, pr.shr_(zb, FRAC));
            }
            S v = pr.sumw(qs);
            v = a.mean_mode == 0 ? pr.mulf(v, a.e_invd) : pr.divp(v, C);
            v = pr.addp(v, a.e_eps);
            if (lane == 0) { pr.st(MUo, rr, mu); pr.st(Vo, rr, v); }
        }
        __syncthreads();
        tile_nr<1, WIDE>(pr, a.s_rs, a.rk, R, g0, Vc, RSo);
        const i64 ne = (i64)R * C;
        const u64 ub = g0 * (u64)C;            // even: g0 is a multiple of 32
        const SO zt{{a.z.p[0] ? a.z.p[0] + r0 * C : nullptr, a.z.p[1] ? a.z.p[1] + r0 * C : nullptr}};
        constexpr int V = decltype(pr)::kV;
        if (a.bcast) {
            tile_bcast_mul(pr, a.s_mul, R, C, g0, dC, RSc, zt, BR,
                           [&](i64 e, int r) { return pr.sub(pr.ld(xt, e), pr.ld(MUc, r)); });
        } else
        for (i64 base = (i64)warp * 32 * V; base < (ne + 1) / 2; base += (i64)NW * 32 * V) {
            u64 uv[V];
            S ca[V], cb[V], ra[V], rb[V], za[V], zb[V];
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const i64 e = 2 * (base + lane + 32 * v);
                uv[v] = ub + (u64)e;
                ca[v] = cb[v] = ra[v] = rb[v] = pr.zero();
                if (e < ne) { const i64 r = fdiv((u32)e, dC); ca[v] = pr.sub(pr.ld(xt, e), pr.ld(MUc, r)); ra[v] = pr.ld(RSc, r); }
                if (e + 1 < ne) { const i64 r = fdiv((u32)(e + 1), dC); cb[v] = pr.sub(pr.ld(xt, e + 1), pr.ld(MUc, r)); rb[v] = pr.ld(RSc, r); }
            }
            pr.template bm2v<V>(uv, a.s_mul, ca, ra, cb, rb, za, zb);
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const i64 e = 2 * (base + lane + 32 * v);
                if (e < ne) pr.st(zt, e, pr.shr_(za[v], FRAC));
                if (e + 1 < ne) pr.st(zt, e + 1, pr.shr_(zb[v], FRAC));
            }
        }
        __syncthreads();
    }
    pa.done(pr);
}

// LAYERNORM as three launches (rsqrt without clamp; DESIGN.md 2.5 / 6):
//  k_ln_stats : warp per row -- mu = mean(x) (x E(1/d) or floor / d), v = mean(MT(c, c)) + eps,
//               element units (unit pairs over the row), step s_sq; writes mu, v per row
//  RSQRT      : the element-wise Newton-Raphson kernel over the rows (k_pairs<NrPairBody<1>>,
//               row units g = row_off + r, steps s_rs..) -- a short latency-bound launch instead of
//               one warp per 32-row tile holding seven warps at a barrier
//  LnOutBody  : out = MT(x - mu, r) on element unit pairs (step s_mul), perfectly balanced
// Same steps, units and output bits as k_ln (tests compare both against the oracle).
struct LnStatsArgs { u32 s_sq; SP x; SO mu; SO var; i64 rows, cols; u64 row_off; int mean_mode; u64 e_invd, e_eps; };
template <class PA>
__global__ void __launch_bounds__(256, MPC_EW_MINB) k_ln_stats(const __grid_constant__ PA pa, LnStatsArgs a)
{
    int cta, ncta;
    auto pr = pa.make(cta, ncta);
    using S = typename decltype(pr)::S;
    const int lane = threadIdx.x & 31, NW = blockDim.x >> 5;
    const i64 C = a.cols;
    for (i64 r = (i64)cta * NW + (threadIdx.x >> 5); r < a.rows; r += (i64)ncta * NW) {
        const SP xr{{a.x.p[0] ? a.x.p[0] + r * C : nullptr, a.x.p[1] ? a.x.p[1] + r * C : nullptr}};
        S acc = pr.zero();
        for (i64 j = lane; j < C; j += 32) acc = pr.add(acc, pr.ld(xr, j));
        S mu = pr.sumw(acc);
        mu = a.mean_mode == 0 ? pr.mulf(mu, a.e_invd) : pr.divp(mu, C);
        S qs = pr.zero();
        const u64 ub = (a.row_off + (u64)r) * (u64)C;
        const i64 j0 = -(i64)(ub & 1);
        for (i64 j = j0 + 2 * lane, jb = j0; jb < C; j += 64, jb += 64) {
            const bool va = j >= 0 && j < C, vb = j + 1 >= 0 && j + 1 < C;
            S ca = pr.zero(), cb = pr.zero();
            if (va) ca = pr.sub(pr.ld(xr, j), mu);
            if (vb) cb = pr.sub(pr.ld(xr, j + 1), mu);
            S za, zb;
            pr.bm2(ub + (u64)j, a.s_sq, ca, ca, cb, cb, za, zb);
            if (va) qs = pr.add(qs, pr.shr_(za, FRAC));
            if (vb) qs = pr.add(qs, pr.shr_(zb, FRAC));
        }
        S v = pr.sumw(qs);
        v = a.mean_mode == 0 ? pr.mulf(v, a.e_invd) : pr.divp(v, C);
        v = pr.addp(v, a.e_eps);
        if (lane == 0) { pr.st(a.mu, r, mu); pr.st(a.var, r, v); }
    }
    pa.done(pr);
}
struct LnOutBody {
    u32 s; SP x; SO z; i64 n; FastDiv dC; SP mu; SP rs;
    template <int V, class P>
    __device__ void run(P& pr, const u64 (&u)[V], const i64 (&i0)[V], const bool (&ok)[V]) const {
        using S = typename P::S;
        S ca[V], cb[V], ra[V], rb[V], za[V], zb[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            ca[v] = cb[v] = ra[v] = rb[v] = pr.zero();
            if (ok[v] && i0[v] >= 0) {
                const i64 r = fdiv((u32)i0[v], dC);
                ca[v] = pr.sub(pr.ld(x, i0[v]), pr.ld(mu, r)); ra[v] = pr.ld(rs, r);
            }
            if (ok[v] && i0[v] + 1 < n) {
                const i64 r = fdiv((u32)(i0[v] + 1), dC);
                cb[v] = pr.sub(pr.ld(x, i0[v] + 1), pr.ld(mu, r)); rb[v] = pr.ld(rs, r);
            }
        }
        pr.template bm2v<V>(u, s, ca, ra, cb, rb, za, zb);
#pragma unroll
        for (int v = 0; v < V; ++v) {
            if (ok[v] && i0[v] >= 0) pr.st(z, i0[v], pr.shr_(za[v], FRAC));
            if (ok[v] && i0[v] + 1 < n) pr.st(z, i0[v] + 1, pr.shr_(zb[v], FRAC));
        }
    }
};

// LAYERNORM, warp-granular (rsqrt without clamp: no LTZ, so row units need no 32-row grouping).
// A warp owns a QUAD of 4 consecutive rows (4-aligned global rows, so the rsqrt unit pairs (2p, 2p+1)
// are aligned) and runs the whole schedule on them with no CTA barrier: mean and sum MT(c, c) per
// row (element units, unit pairs over the row), RSQRT over the quad's rows (lanes 0-1 hold the two
// unit pairs; every lane runs the chain, so it costs one warp's issue, not 8 warps' barrier wait),
// then the final MT(c, r) (element units).  Same steps, units and output bits as k_ln.  Persistent
// over quads (8192 rows = 2048 quads, one wave of 2048 warps for cfg5).
template <bool WIDE, class PA>
__global__ void __launch_bounds__(MPC_ROW_TPB, MPC_SM_MINB) k_ln_quad(const __grid_constant__ PA pa, LnArgs a)
{
    __shared__ u64 RSH[MPC_ROW_TPB / 32][2][4];          // per warp: r of the quad's rows (per party)
    int cta, ncta;
    auto pr = pa.make(cta, ncta);
    using S = typename decltype(pr)::S;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
    const i64 C = a.cols;
    const i64 nq = (a.rows + 3) / 4;
    const FastDiv dC = make_fastdiv((u32)C);
    const SO RSo{{RSH[warp][0], RSH[warp][1]}};
    const SP RSc{{RSH[warp][0], RSH[warp][1]}};
    for (i64 Q = (i64)cta * NW + warp; Q < nq; Q += (i64)ncta * NW) {
        const i64 r0 = 4 * Q;
        const int R = (int)min((i64)4, a.rows - r0);
        const u64 g0 = a.row_off + (u64)r0;                           // global row of the quad (4-aligned)
        const SP xt{{a.x.p[0] ? a.x.p[0] + r0 * C : nullptr, a.x.p[1] ? a.x.p[1] + r0 * C : nullptr}};
        S mu[4], var[4];
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
            mu[rr] = var[rr] = pr.zero();
            if (rr >= R) continue;                                   // warp-uniform
            S acc = pr.zero();
            for (i64 j = lane; j < C; j += 32) acc = pr.add(acc, pr.ld(xt, rr * C + j));
            S m = pr.sumw(acc);
            m = a.mean_mode == 0 ? pr.mulf(m, a.e_invd) : pr.divp(m, C);
            // q = MT(c, c) over the row, element units; lanes take unit pairs (2j, 2j+1)
            S qs = pr.zero();
            const u64 ub = (g0 + (u64)rr) * (u64)C;
            const i64 j0 = -(i64)(ub & 1);
            for (i64 j = j0 + 2 * lane, jb = j0; jb < C; j += 64, jb += 64) {
                const bool va = j >= 0 && j < C, vb = j + 1 >= 0 && j + 1 < C;
                S ca = pr.zero(), cb = pr.zero();
                if (va) ca = pr.sub(pr.ld(xt, rr * C + j), m);
                if (vb) cb = pr.sub(pr.ld(xt, rr * C + j + 1), m);
                S za, zb;
                pr.bm2(ub + (u64)j, a.s_sq, ca, ca, cb, cb, za, zb);
                if (va) qs = pr.add(qs, pr.shr_(za, FRAC));
                if (vb) qs = pr.add(qs, pr.shr_(zb, FRAC));
            }
            S v = pr.sumw(qs);
            v = a.mean_mode == 0 ? pr.mulf(v, a.e_invd) : pr.divp(v, C);
            mu[rr] = m;
            var[rr] = pr.addp(v, a.e_eps);
        }
        {   // RSQRT of the quad's rows: lane p (0, 1) <-> unit pair (g0 + 2p, g0 + 2p + 1)
            const int p = lane & 1;
            S y0, y1;
            rsqrt_pair(pr, g0 + 2u * (u64)p, a.s_rs, a.rk, p ? var[2] : var[0], p ? var[3] : var[1], y0, y1);
            if (lane < 2) { pr.st(RSo, 2 * lane, y0); pr.st(RSo, 2 * lane + 1, y1); }
        }
        __syncwarp();
        const i64 ne = (i64)R * C;
        const u64 ub = g0 * (u64)C;                                  // even: g0 is a multiple of 4
        const SO zt{{a.z.p[0] ? a.z.p[0] + r0 * C : nullptr, a.z.p[1] ? a.z.p[1] + r0 * C : nullptr}};
        auto cval = [&](i64 e, int r) {
            const S m = r == 0 ? mu[0] : r == 1 ? mu[1] : r == 2 ? mu[2] : mu[3];
            return pr.sub(pr.ld(xt, e), m);
        };
        if (a.bcast) {                                              // broadcast triple (NEXT #2)
            const S yr = lane < R ? pr.ld(RSc, lane) : pr.zero();
            const BRow br = pr.bmb_row(g0 + (u64)lane, a.s_mul, yr);   // lanes >= 4: unused rows
            for (i64 base = 0; base < (ne + 1) / 2; base += 32) {
                const i64 e = 2 * (base + lane);
                S xa = pr.zero(), xb = pr.zero();
                int ra = 0, rb = 0;
                if (e < ne) { ra = (int)fdiv((u32)e, dC); xa = cval(e, ra); }
                if (e + 1 < ne) { rb = (int)fdiv((u32)(e + 1), dC); xb = cval(e + 1, rb); }
                const BRow b0{__shfl_sync(FULL, br.b0, ra), __shfl_sync(FULL, br.b1, ra), __shfl_sync(FULL, br.f, ra)};
                const BRow b1{__shfl_sync(FULL, br.b0, rb), __shfl_sync(FULL, br.b1, rb), __shfl_sync(FULL, br.f, rb)};
                S za, zb;
                pr.bmb2(ub + (u64)e, a.s_mul, xa, xb, b0, b1, za, zb);
                if (e < ne) pr.st(zt, e, pr.shr_(za, FRAC));
                if (e + 1 < ne) pr.st(zt, e + 1, pr.shr_(zb, FRAC));
            }
        } else {
            constexpr int V = decltype(pr)::kV;
            for (i64 base = 0; base < (ne + 1) / 2; base += 32 * V) {
                u64 uv[V];
                S ca[V], cb[V], ra[V], rb[V], za[V], zb[V];
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const i64 e = 2 * (base + lane + 32 * v);
                    uv[v] = ub + (u64)e;
                    ca[v] = cb[v] = ra[v] = rb[v] = pr.zero();
                    if (e < ne) { const int r = (int)fdiv((u32)e, dC); ca[v] = cval(e, r); ra[v] = pr.ld(RSc, r); }
                    if (e + 1 < ne) { const int r = (int)fdiv((u32)(e + 1), dC); cb[v] = cval(e + 1, r); rb[v] = pr.ld(RSc, r); }
                }
                pr.template bm2v<V>(uv, a.s_mul, ca, ra, cb, rb, za, zb);
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const i64 e = 2 * (base + lane + 32 * v);
                    if (e < ne) pr.st(zt, e, pr.shr_(za[v], FRAC));
                    if (e + 1 < ne) pr.st(zt, e + 1, pr.shr_(zb[v], FRAC));
                }
            }
        }
        __syncwarp();
    }
    pa.done(pr);
}

// ---------------------------------------------------------------- fused row-block LayerNorm ----
// LAYERNORM in ONE launch, element-balanced: a CTA owns RB consecutive rows (RB even, <= 32,
// chosen so that every CTA is resident at once) and its 8 warps split the block's ELEMENT PAIRS
// evenly; a warp walks its range ROW SEGMENT by row segment (the row is warp-uniform inside a segment:
// mu / r are one register, and the per-row sums are a warp reduction into wpart[warp][segment] --
// no shared-memory atomics, which are CAS loops for u64):
//   A  row sums -> mu = x E(1/d) | floor / d
//   B  MT(c, c), c = x - mu (element units, unit pairs), summed per row -> v = mean + eps
//   C  RSQRT(v) over the block's rows (row units; BOTH: the chain's triples generated by all warps
//      first, nr_pregen<1>), warp 0 lane <-> row
//   D  out = MT(c, r) (element units, unit pairs)
// Same steps, units, PRG words and output bits as k_ln / the stats-rsqrt-product launches (units:
// rows for the rsqrt, global elements for the two Beaver passes); no clamp (an LTZ in the rsqrt would
// need 32-row groups) and no broadcast triple -- those keep the other paths.  x is read three times
// (the block's rows stay L2-resident between the passes).
struct LnFArgs {
    u32 s_sq, s_rs, s_mul; NrK rk; SP x; SO z; i64 rows, cols; u64 row_off;
    int mean_mode; u64 e_invd, e_eps;
    int RB;                 // rows per block (even)
    int nrtab;              // BOTH: rsqrt triples pre-generated into shared memory
};
constexpr int LNF_SEG = 34;                    // row segments per warp (<= RB + 1)
#ifndef MPC_LN_NEXT_PREFETCH
#define MPC_LN_NEXT_PREFETCH 0     // A/B: 2 blocks per CTA + the next block's rows to L2 during the rsqrt
#endif                             // phase -- measured 2 % slower than one resident block per CTA (r02)
#ifndef MPC_LN_BLOCKS_PER_CTA
#define MPC_LN_BLOCKS_PER_CTA 1
#endif
__host__ __device__ inline int lnf_smem_u64(int nsteps_tab) { return 256 + 8 * LNF_SEG * 2 + nsteps_tab * NR_TAB_F * 32; }
template <class PA>
__global__ void __launch_bounds__(MPC_ROW_TPB, MPC_SM_MINB) k_ln_fused(const __grid_constant__ PA pa, LnFArgs a)
{
    extern __shared__ __align__(16) u64 lsm[];
    int cta, ncta;
    auto pr = pa.make(cta, ncta);
    using P = decltype(pr);
    using S = typename P::S;
    constexpr int V = P::kV;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
    const i64 C = a.cols, hc = C / 2;                        // pairs per row (C even)
    // shared: means MU, variances VR, rsqrt RS (each 2 x 32), per-warp segment sums, NR table
    u64* MUw = lsm; u64* VRw = lsm + 64; u64* RSw = lsm + 128;
    u64* wpart = lsm + 256;                                   // [NW][LNF_SEG][2]
    u64* tab = a.nrtab ? lsm + 256 + 8 * LNF_SEG * 2 : nullptr;
    const SO MU{{MUw, MUw + 32}}, VR{{VRw, VRw + 32}}, RS{{RSw, RSw + 32}};
    const SP MUc{{MUw, MUw + 32}}, VRc{{VRw, VRw + 32}}, RSc{{RSw, RSw + 32}};
    auto put_part = [&](int seg, S v) {                       // lane 0: the warp's sum of one segment
        if constexpr (P::kPair) wpart[(warp * LNF_SEG + seg) * 2 + pr.party()] = v;
        else { wpart[(warp * LNF_SEG + seg) * 2] = v.s0; wpart[(warp * LNF_SEG + seg) * 2 + 1] = v.s1; }
    };
    auto get_part = [&](int w, int seg) -> S {
        if constexpr (P::kPair) return wpart[(w * LNF_SEG + seg) * 2 + pr.party()];
        else return S{wpart[(w * LNF_SEG + seg) * 2], wpart[(w * LNF_SEG + seg) * 2 + 1]};
    };
    const i64 nblk = (a.rows + a.RB - 1) / a.RB;
    for (i64 blk = cta; blk < nblk; blk += ncta) {
        const i64 r0 = blk * a.RB;
        const int R = (int)min((i64)a.RB, a.rows - r0);
        const u64 g0 = a.row_off + (u64)r0;                   // even
        const i64 np = (i64)R * hc;                          // element pairs of the block
        const i64 wbeg = np * warp / NW, wend = np * (warp + 1) / NW;
        const int rw0 = (int)(wbeg / hc);                     // the warp's first row (segment 0)
        const int nseg = wend > wbeg ? (int)((wend - 1) / hc) - rw0 + 1 : 0;
        const u64 ub = g0 * (u64)C;                           // global unit of the block's element 0
        const SP xb{{a.x.p[0] ? a.x.p[0] + r0 * C : nullptr, a.x.p[1] ? a.x.p[1] + r0 * C : nullptr}};
        const SO zb{{a.z.p[0] ? a.z.p[0] + r0 * C : nullptr, a.z.p[1] ? a.z.p[1] + r0 * C : nullptr}};
        // row sum of the warps' segments that cover row r (a row spans at most a few warps)
        auto row_total = [&](int r) -> S {
            S t = pr.zero();
            for (int w = 0; w < NW; ++w) {
                const i64 b0 = np * w / NW, e0 = np * (w + 1) / NW;
                if (e0 <= b0) continue;
                const int f = (int)(b0 / hc), l = (int)((e0 - 1) / hc);
                if (r >= f && r <= l) t = pr.add(t, get_part(w, r - f));
            }
            return t;
        };
        // A: row sums (loads LA pairs ahead: this pass has no arithmetic to hide them)
        for (int sg = 0; sg < nseg; ++sg) {
            const int r = rw0 + sg;
            const i64 sb = max(wbeg, (i64)r * hc), se = min(wend, (i64)(r + 1) * hc);
            constexpr int LA = 8;
            S acc = pr.zero();
            for (i64 base = sb + lane; base < se; base += 32 * LA) {
                S xa[LA], xc[LA];
#pragma unroll
                for (int q = 0; q < LA; ++q) {
                    xa[q] = xc[q] = pr.zero();
                    if (base + 32 * q < se) pr.ld_pair(xb, 2 * (base + 32 * q), true, true, xa[q], xc[q]);
                }
#pragma unroll
                for (int q = 0; q < LA; ++q) acc = pr.add(acc, pr.add(xa[q], xc[q]));
            }
            acc = pr.sumw(acc);
            if (lane == 0) put_part(sg, acc);
        }
        __syncthreads();
        if (threadIdx.x < R) {
            S mu = row_total(threadIdx.x);
            mu = a.mean_mode == 0 ? pr.mulf(mu, a.e_invd) : pr.divp(mu, C);
            pr.st(MU, threadIdx.x, mu);
        }
        __syncthreads();
        // B: sum of MT(c, c); the next iteration's pairs load while this one computes
        for (int sg = 0; sg < nseg; ++sg) {
            const int r = rw0 + sg;
            const i64 sb = max(wbeg, (i64)r * hc), se = min(wend, (i64)(r + 1) * hc);
            const S m = pr.ld(MUc, r);
            const i64 iters = (se - sb + 32 * V - 1) / (32 * V);
            S acc = pr.zero();
            S nxa[V], nxc[V];
#pragma unroll
            for (int v = 0; v < V; ++v) {
                nxa[v] = nxc[v] = pr.zero();
                if (sb + v * 32 + lane < se) pr.ld_pair(xb, 2 * (sb + v * 32 + lane), true, true, nxa[v], nxc[v]);
            }
            for (i64 it = 0; it < iters; ++it) {
                u64 u[V];
                S ca[V], cb[V], za[V], zz[V];
                bool ok[V];
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const i64 P2 = sb + (it * V + v) * 32 + lane;
                    ok[v] = P2 < se;
                    u[v] = ub + 2 * (u64)P2;
                    ca[v] = pr.sub(nxa[v], m); cb[v] = pr.sub(nxc[v], m);
                    const i64 Q2 = P2 + 32 * V;
                    nxa[v] = nxc[v] = pr.zero();
                    if (Q2 < se) pr.ld_pair(xb, 2 * Q2, true, true, nxa[v], nxc[v]);
                }
                pr.template bm2v<V>(u, a.s_sq, ca, ca, cb, cb, za, zz);
#pragma unroll
                for (int v = 0; v < V; ++v)
                    if (ok[v]) acc = pr.add(acc, pr.add(pr.shr_(za[v], FRAC), pr.shr_(zz[v], FRAC)));
            }
            acc = pr.sumw(acc);
            if (lane == 0) put_part(sg, acc);
        }
        __syncthreads();
        if (threadIdx.x < R) {
            S v = row_total(threadIdx.x);
            v = a.mean_mode == 0 ? pr.mulf(v, a.e_invd) : pr.divp(v, C);
            pr.st(VR, threadIdx.x, pr.addp(v, a.e_eps));
        }
        if constexpr (!P::kPair)
            if (tab) nr_pregen<1>(*pr.Kp, a.s_rs, a.rk, g0, tab);
        // the CTA's NEXT block: its rows to L2 now (the rsqrt chain below leaves 7 warps idle and the
        // product pass is ALU-bound), so its row-sum pass reads L2 instead of waiting on HBM
        if (MPC_LN_NEXT_PREFETCH && blk + ncta < nblk) {
            const i64 rn = (blk + ncta) * a.RB, nel = min((i64)a.RB, a.rows - rn) * C;
            for (i64 l = (i64)threadIdx.x * 16; l < nel; l += (i64)blockDim.x * 16)      // one 128-B line each
#pragma unroll
                for (int q = 0; q < 2; ++q)
                    if (a.x.p[q]) asm volatile("prefetch.global.L2 [%0];" :: "l"(a.x.p[q] + rn * C + l));
        }
        __syncthreads();
        // C: r = RSQRT(v), row units g0 + lane
        tile_nr<1, false>(pr, a.s_rs, a.rk, R, g0, VRc, RS, tab);
        // D: out = MT(c, r)
        for (int sg = 0; sg < nseg; ++sg) {
            const int r = rw0 + sg;
            const i64 sb = max(wbeg, (i64)r * hc), se = min(wend, (i64)(r + 1) * hc);
            const S m = pr.ld(MUc, r), rr = pr.ld(RSc, r);
            const i64 iters = (se - sb + 32 * V - 1) / (32 * V);
            S nxa[V], nxc[V];
#pragma unroll
            for (int v = 0; v < V; ++v) {
                nxa[v] = nxc[v] = pr.zero();
                if (sb + v * 32 + lane < se) pr.ld_pair(xb, 2 * (sb + v * 32 + lane), true, true, nxa[v], nxc[v]);
            }
            for (i64 it = 0; it < iters; ++it) {
                u64 u[V];
                S ca[V], cb[V], rv[V], za[V], zz[V];
                i64 e0[V];
                bool ok[V];
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const i64 P2 = sb + (it * V + v) * 32 + lane;
                    ok[v] = P2 < se;
                    e0[v] = 2 * P2;
                    u[v] = ub + 2 * (u64)P2;
                    ca[v] = pr.sub(nxa[v], m); cb[v] = pr.sub(nxc[v], m); rv[v] = rr;
                    const i64 Q2 = P2 + 32 * V;
                    nxa[v] = nxc[v] = pr.zero();
                    if (Q2 < se) pr.ld_pair(xb, 2 * Q2, true, true, nxa[v], nxc[v]);
                }
                pr.template bm2v<V>(u, a.s_mul, ca, rv, cb, rv, za, zz);
#pragma unroll
                for (int v = 0; v < V; ++v)
                    if (ok[v]) pr.st_pair(zb, e0[v], true, true, pr.shr_(za[v], FRAC), pr.shr_(zz[v], FRAC));
            }
        }
        __syncthreads();
    }
    pa.done(pr);
}


// ------------------------------------------------------------- warp-per-row LayerNorm (BOTH) ----
// LAYERNORM with one WARP per row and no CTA barrier: the row's element pairs are the
// lanes' (pair p = lane + 32 k, 16-byte loads of both shares), the row sums are warp reductions, and
// the row's RSQRT chain (row unit g) runs on every lane from a per-warp table of its triples that
// lanes 0..ns-1 generate one step each while the row's first pass is in flight (3 Philox blocks per
// lane instead of ns x 2.5 serial blocks on the chain).  x is read from HBM once per pass A (the next
// row is prefetched to L2) and from L2 in passes B and D.  Same steps, units, PRG words and output
// bits as k_ln_fused (units: global rows for the rsqrt, global elements for the two Beaver passes);
// BOTH only, no clamp in the rsqrt's exp, no broadcast triple, ns <= 32.
struct LnRArgs {
    u32 s_sq, s_rs, s_mul; NrK rk; SP x; SO z; i64 rows, cols; u64 row_off;
    int mean_mode; u64 e_invd, e_eps;
};
// BothP with the chain's bm / sq read from a per-warp table [step][5] (a0 b0 c0 a b; square-pair
// steps: a0 . c0 a), all lanes reading the same words (shared-memory broadcast)
struct BothRowTabP : BothP {
    const u64* T; u32 sb;
    __device__ __forceinline__ S bm(u64, u32 s, S x, S y) const {
        const u64* R = T + (i64)(s - sb) * NR_TAB_F;
        const u64 a0 = R[0], b0 = R[1], c0 = R[2], a = R[3], b = R[4];
        const u64 X = x.s0 + x.s1, Y = y.s0 + y.s1;
        const u64 e = X - a, f = Y - b;               // open(x - a), open(y - b)
        const u64 z0 = c0 + e * (b0 + f) + f * a0;    // = mpc::bm_with_c0
        return {z0, X * Y - z0};
    }
    __device__ __forceinline__ S sq(u64, u32 s, S y) const {
        const u64* R = T + (i64)(s - sb) * NR_TAB_F;
        const u64 a0 = R[0], c0 = R[2], a = R[3];
        const u64 Y = y.s0 + y.s1, e = Y - a;
        const u64 z0 = c0 + e * (2ull * a0 + e);      // = mpc::sq_with_a1
        return {z0, Y * Y - z0};
    }
};
// one step's triple of row unit u (the words nr_pregen writes for a unit, DESIGN.md 2.3 / 2.6)
__device__ __forceinline__ void row_tab_step(const Keys& K, u64 u, u32 sj, bool square, u64* R)
{
    if (square) {
        const uint4 A0 = prg(K.k0, u, sj, 2), A1 = prg(K.k1, u >> 1, sj, 3);
        const u64 a0 = w64(A0.x, A0.y);
        R[0] = a0; R[1] = 0; R[2] = w64(A0.z, A0.w);
        R[3] = a0 + ((u & 1) ? w64(A1.z, A1.w) : w64(A1.x, A1.y)); R[4] = 0;
    } else {
        const uint4 A0 = prg(K.k0, u, sj, 0), A1 = prg(K.k1, u, sj, 0), Cb = prg(K.k0, u >> 1, sj, 1);
        const u64 a0 = w64(A0.x, A0.y), b0 = w64(A0.z, A0.w);
        R[0] = a0; R[1] = b0; R[2] = (u & 1) ? w64(Cb.z, Cb.w) : w64(Cb.x, Cb.y);
        R[3] = a0 + w64(A1.x, A1.y); R[4] = b0 + w64(A1.z, A1.w);
    }
}
#ifndef MPC_LNR_V
#define MPC_LNR_V 1            // unit pairs per lane per Beaver call in passes B and D
#endif
template <class PA>
__global__ void __launch_bounds__(MPC_ROW_TPB, MPC_SM_MINB) k_ln_row(const __grid_constant__ PA pa, LnRArgs a)
{
    __shared__ u64 tabs[MPC_ROW_TPB / 32][MPC_NR_TAB_MAX_STEPS * NR_TAB_F];
    int cta, ncta;
    auto pr = pa.make(cta, ncta);
    using P = decltype(pr);
    using S = typename P::S;
    static_assert(!P::kPair, "BOTH only (PAIR keeps k_ln_fused)");
    constexpr int V = MPC_LNR_V;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
    const i64 C = a.cols, hc = C / 2;                        // pairs per row (C even)
    const i64 nk = (hc + 31) / 32;                           // pair chunks per lane
    const i64 nwarp = (i64)ncta * NW;
    const int ns = nr_tab_steps(1, a.rk.exp.t, a.rk.iters);
    u64* T = tabs[warp];
    for (i64 r = (i64)cta * NW + warp; r < a.rows; r += nwarp) {
        const u64 g = a.row_off + (u64)r;                    // global row = the rsqrt's unit
        const u64 ub = g * (u64)C;                           // even (C is)
        const SP xr{{a.x.p[0] + r * C, a.x.p[1] + r * C}};
        const SO zr{{a.z.p[0] + r * C, a.z.p[1] + r * C}};
        if (MPC_GROUP_PREFETCH && r + nwarp < a.rows)        // the warp's next row to L2 (128-B lines)
            for (i64 l = (i64)lane * 16; l < C; l += 32 * 16)
#pragma unroll
                for (int q = 0; q < 2; ++q) asm volatile("prefetch.global.L2 [%0];" :: "l"(a.x.p[q] + (r + nwarp) * C + l));
        // A: row sum -> mu (all chunks' loads in flight at once)
        S acc = pr.zero();
        for (i64 k0 = 0; k0 < nk; k0 += 4) {
            S xa[4], xc[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                xa[q] = xc[q] = pr.zero();
                const i64 p2 = lane + 32 * (k0 + q);
                if (k0 + q < nk && p2 < hc) pr.ld_pair(xr, 2 * p2, true, true, xa[q], xc[q]);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) acc = pr.add(acc, pr.add(xa[q], xc[q]));
        }
        S mu = pr.sumw(acc);
        mu = a.mean_mode == 0 ? pr.mulf(mu, a.e_invd) : pr.divp(mu, C);
        // the chain's triples: lane j < ns generates step j (data-independent; overlaps pass B)
        if (lane < ns) row_tab_step(*pr.Kp, g, a.s_rs + (u32)lane, lane < a.rk.exp.t && a.rk.exp.sq, T + lane * NR_TAB_F);
        // B: sum of MT(c, c), c = x - mu; the next chunk's pairs load while this one computes
        S qs = pr.zero();
        {
            S nxa[V], nxc[V];
#pragma unroll
            for (int v = 0; v < V; ++v) {
                nxa[v] = nxc[v] = pr.zero();
                const i64 p2 = lane + 32 * v;
                if (v < nk && p2 < hc) pr.ld_pair(xr, 2 * p2, true, true, nxa[v], nxc[v]);
            }
            for (i64 k0 = 0; k0 < nk; k0 += V) {
                u64 u[V];
                S ca[V], cb[V], za[V], zz[V];
                bool ok[V];
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const i64 p2 = lane + 32 * (k0 + v);
                    ok[v] = k0 + v < nk && p2 < hc;
                    u[v] = ub + 2 * (u64)p2;
                    ca[v] = pr.sub(nxa[v], mu); cb[v] = pr.sub(nxc[v], mu);
                    const i64 q2 = p2 + 32 * V;
                    nxa[v] = nxc[v] = pr.zero();
                    if (k0 + v + V < nk && q2 < hc) pr.ld_pair(xr, 2 * q2, true, true, nxa[v], nxc[v]);
                }
                pr.template bm2v<V>(u, a.s_sq, ca, ca, cb, cb, za, zz);
#pragma unroll
                for (int v = 0; v < V; ++v)
                    if (ok[v]) qs = pr.add(qs, pr.add(pr.shr_(za[v], FRAC), pr.shr_(zz[v], FRAC)));
            }
        }
        S var = pr.sumw(qs);
        var = a.mean_mode == 0 ? pr.mulf(var, a.e_invd) : pr.divp(var, C);
        var = pr.addp(var, a.e_eps);
        __syncwarp();
        // C: r = RSQRT(var), unit g, every lane the same chain from the table
        BothRowTabP tp;
        tp.Kp = pr.Kp; tp.T = T; tp.sb = a.s_rs;
        const S rr = rsqrt_group<false>(tp, g, g >> 5, a.s_rs, a.rk, var, lane);
        // D: out = MT(c, r)
        {
            S nxa[V], nxc[V];
#pragma unroll
            for (int v = 0; v < V; ++v) {
                nxa[v] = nxc[v] = pr.zero();
                const i64 p2 = lane + 32 * v;
                if (v < nk && p2 < hc) pr.ld_pair(xr, 2 * p2, true, true, nxa[v], nxc[v]);
            }
            for (i64 k0 = 0; k0 < nk; k0 += V) {
                u64 u[V];
                S ca[V], cb[V], rv[V], za[V], zz[V];
                bool ok[V];
                i64 e0[V];
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const i64 p2 = lane + 32 * (k0 + v);
                    ok[v] = k0 + v < nk && p2 < hc;
                    e0[v] = 2 * p2;
                    u[v] = ub + 2 * (u64)p2;
                    ca[v] = pr.sub(nxa[v], mu); cb[v] = pr.sub(nxc[v], mu); rv[v] = rr;
                    const i64 q2 = p2 + 32 * V;
                    nxa[v] = nxc[v] = pr.zero();
                    if (k0 + v + V < nk && q2 < hc) pr.ld_pair(xr, 2 * q2, true, true, nxa[v], nxc[v]);
                }
                pr.template bm2v<V>(u, a.s_mul, ca, rv, cb, rv, za, zz);
#pragma unroll
                for (int v = 0; v < V; ++v)
                    if (ok[v]) pr.st_pair(zr, e0[v], true, true, pr.shr_(za[v], FRAC), pr.shr_(zz[v], FRAC));
            }
        }
        __syncwarp();                                         // T is rewritten for the next row
    }
    pa.done(pr);
}

// ------------------------------------------------- softmax after the max tree (BOTH, split form) ----
// cfg2-shaped softmax as two launches: the row max tree (k_max, 32-row tiles, the rebalanced w = 33
// LTZ) and this kernel -- e = EXP(x - m), S = rowsum(e), r = RECIP(S), out = MT(e, r) -- on row
// blocks of RB <= 64 rows sized so that every block is resident at once (no tail wave), the warps
// splitting the block's element pairs evenly along warp-uniform row segments (as k_ln_fused), E in
// an L2-resident per-block scratch, the reciprocal chains' triples pre-generated (two 32-row
// tables, warps 0 and 1).  Same steps, units and output bits as k_softmax (dense, no clamp, the
// expanded product).
struct SmRestArgs {
    u32 s_exp, s_rec, s_mul; ExpK ek; NrK rk; SP x; SP mx; SO z; i64 rows, cols; u64 row_off;
    int RB;                 // rows per block (even, <= 64)
    u64* escr;              // per-CTA E scratch: 2 x RB x cols u64
    int tab_u64;            // u64 words of one 32-row NR table
};
constexpr int SMR_SEG = 66;                    // row segments per warp (<= RB + 2)
__host__ __device__ inline int smr_smem_u64(int tab_u64, int ntab = 2) { return 6 * 64 + 8 * SMR_SEG * 2 + ntab * tab_u64; }
#ifndef MPC_SMR_MINB
#define MPC_SMR_MINB 3         // resident CTAs per SM of k_softmax_rest (<= 85 registers: 24 warps per SM)
#endif
template <class PA>
__global__ void __launch_bounds__(MPC_ROW_TPB, MPC_SMR_MINB) k_softmax_rest(const __grid_constant__ PA pa, SmRestArgs a)
{
    extern __shared__ __align__(16) u64 rsm[];
    int cta, ncta;
    auto pr = pa.make(cta, ncta);
    using P = decltype(pr);
    using S = typename P::S;
    static_assert(!P::kPair, "BOTH only (PAIR keeps the fused k_softmax)");
    constexpr int V = P::kV;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
    const i64 C = a.cols, hc = C / 2;
    u64* MXw = rsm; u64* SSw = rsm + 128; u64* RRw = rsm + 256;
    u64* wpart = rsm + 384;                                        // [NW][SMR_SEG][2]
    u64* tab = rsm + 384 + 8 * SMR_SEG * 2;                        // two 32-row NR tables
    const SO MX{{MXw, MXw + 64}}, SS{{SSw, SSw + 64}}, RR{{RRw, RRw + 64}};
    const SP MXc{{MXw, MXw + 64}}, SSc{{SSw, SSw + 64}}, RRc{{RRw, RRw + 64}};
    u64* Ew = a.escr + (i64)blockIdx.x * 2 * a.RB * C;
    const SO E{{Ew, Ew + (i64)a.RB * C}};
    const SP Ec{{Ew, Ew + (i64)a.RB * C}};
    const i64 nblk = (a.rows + a.RB - 1) / a.RB;
    for (i64 blk = cta; blk < nblk; blk += ncta) {
        const i64 r0 = blk * a.RB;
        const int R = (int)min((i64)a.RB, a.rows - r0);
        const u64 g0 = a.row_off + (u64)r0;                         // even
        const i64 np = (i64)R * hc;
        const i64 wbeg = np * warp / NW, wend = np * (warp + 1) / NW;
        const int rw0 = (int)(wbeg / hc);
        const int nseg = wend > wbeg ? (int)((wend - 1) / hc) - rw0 + 1 : 0;
        const u64 ub = g0 * (u64)C;
        const SP xb{{a.x.p[0] + r0 * C, a.x.p[1] + r0 * C}};
        const SO zb{{a.z.p[0] + r0 * C, a.z.p[1] + r0 * C}};
        for (int r = threadIdx.x; r < R; r += blockDim.x) pr.st(MX, r, pr.ld(a.mx, r0 + r));
        __syncthreads();
        // 1. e = EXP(x - m) into E, and the per-row sums of e
        for (int sg = 0; sg < nseg; ++sg) {
            const int r = rw0 + sg;
            const i64 sb = max(wbeg, (i64)r * hc), se = min(wend, (i64)(r + 1) * hc);
            const S m = pr.ld(MXc, r);
            S acc = pr.zero();
            for (i64 base = sb + lane; base - lane < se; base += 32 * V) {     // warp-uniform trip count
                u64 uv[V];
                S da[V], db[V];
                bool ok[V];
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const i64 P2 = base + 32 * v;
                    ok[v] = P2 < se;
                    uv[v] = ub + 2 * (u64)P2;
                    da[v] = db[v] = pr.zero();
                    if (ok[v]) { pr.ld_pair(xb, 2 * P2, true, true, da[v], db[v]); da[v] = pr.sub(da[v], m); db[v] = pr.sub(db[v], m); }
                }
                exp_pairv<V>(pr, uv, a.s_exp, a.ek, da, db);
#pragma unroll
                for (int v = 0; v < V; ++v)
                    if (ok[v]) {
                        const i64 P2 = base + 32 * v;
                        pr.st_pair(E, 2 * P2, true, true, da[v], db[v]);
                        acc = pr.add(acc, pr.add(da[v], db[v]));
                    }
            }
            acc = pr.sumw(acc);
            if (lane == 0) { wpart[(warp * SMR_SEG + sg) * 2] = acc.s0; wpart[(warp * SMR_SEG + sg) * 2 + 1] = acc.s1; }
        }
        __syncthreads();
        if (threadIdx.x < R) {                                       // S[r] = the warps' segments of row r
            S t = pr.zero();
            for (int w = 0; w < NW; ++w) {
                const i64 b0 = np * w / NW, e0 = np * (w + 1) / NW;
                if (e0 <= b0) continue;
                const int f = (int)(b0 / hc), l = (int)((e0 - 1) / hc);
                if ((int)threadIdx.x >= f && (int)threadIdx.x <= l)
                    t = pr.add(t, S{wpart[(w * SMR_SEG + (threadIdx.x - f)) * 2], wpart[(w * SMR_SEG + (threadIdx.x - f)) * 2 + 1]});
            }
            pr.st(SS, threadIdx.x, t);
        }
        nr_pregen<0>(*pr.Kp, a.s_rec, a.rk, g0, tab);
        if (R > 32) nr_pregen<0>(*pr.Kp, a.s_rec, a.rk, g0 + 32, tab + a.tab_u64);
        __syncthreads();
        // 2. r = RECIP(S): warp w < 2 runs rows 32 w + lane, units g0 + 32 w + lane
        if (warp < 2 && 32 * warp < R) {
            const int row = 32 * warp + lane;
            BothTabP tp;
            tp.Kp = pr.Kp; tp.T = tab + warp * a.tab_u64; tp.sb = a.s_rec;
            const S xv = row < R ? pr.ld(SSc, row) : pr.zero();
            const S rv = recip_group<false>(tp, g0 + (u64)row, (g0 + 32 * warp) >> 5, a.s_rec, a.rk, xv, lane);
            if (row < R) pr.st(RR, row, rv);
        }
        __syncthreads();
        // 3. out = MT(e, r)
        for (int sg = 0; sg < nseg; ++sg) {
            const int r = rw0 + sg;
            const i64 sb = max(wbeg, (i64)r * hc), se = min(wend, (i64)(r + 1) * hc);
            const S rv = pr.ld(RRc, r);
            for (i64 base = sb + lane; base - lane < se; base += 32 * V) {
                u64 uv[V];
                S ea[V], eb[V], rr[V], za[V], zz[V];
                bool ok[V];
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const i64 P2 = base + 32 * v;
                    ok[v] = P2 < se;
                    uv[v] = ub + 2 * (u64)P2;
                    ea[v] = eb[v] = pr.zero(); rr[v] = rv;
                    if (ok[v]) pr.ld_pair(Ec, 2 * P2, true, true, ea[v], eb[v]);
                }
                pr.template bm2v<V>(uv, a.s_mul, ea, rr, eb, rr, za, zz);
#pragma unroll
                for (int v = 0; v < V; ++v)
                    if (ok[v]) pr.st_pair(zb, 2 * (base + 32 * v), true, true, pr.shr_(za[v], FRAC), pr.shr_(zz[v], FRAC));
            }
        }
        __syncthreads();
    }
    pa.done(pr);
}

}  // namespace mpc
