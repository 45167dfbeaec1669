// proto.cuh -- the two protocol "policies" every schedule is written against.
//
//  BothP : MPC_MODE_BOTH -- one thread holds both parties' shares of a unit; an opening
//          is the sum of the two masked shares, formed in registers (proto_both.cuh).
//  PairP : MPC_MODE_PAIR / MPC_MODE_PAIR_LOOPBACK -- a thread holds ITS party's share;
//          each opening is a warp-level exchange with the matching warp of the peer
//          party through NVLink peer memory (or, loopback, through local memory):
//          every lane stores its masked words into the peer's receive buffer, fences at
//          system scope, lane 0 publishes a monotonically increasing round number in the
//          peer's flag word and waits (acquire, with a timeout) for the peer's flag.
//          Receive buffers are double-buffered by round parity; the round counter of each
//          warp slot persists across launches, so consecutive ops never alias.
// Both policies implement exactly the contract of DESIGN.md 2.3 / 2.4, so their output
// shares are bit-identical (test T4).
#pragma once
#include "proto_both.cuh"

namespace mpc {

// ---- shares in memory: one pointer per party ------------------------------------------------
struct SP { const u64* p[2]; };
struct SO { u64* p[2]; };

// carry-cone LTZ over G groups per warp (ltz_cone.cuh); NL leaf positions (32: w <= 33, 64: w <= 65)
template <int G, int NL = 32>
struct ConeSmem { u32 w[G][NL][4]; };
template <int G, int NL>
__device__ void ltz_cone_both(const Keys& K, u64 q0, u32 s, int w, const Sh (&x)[G], Sh (&z)[G], int lane,
                              ConeSmem<G, NL>& sm);
template <int R> struct PairP;
template <int G, int NL, int R>
__device__ void ltz_cone_pair(PairP<R>& pr, u64 q0, u32 s, int w, const u64 (&x)[G], u64 (&z)[G], int lane,
                              ConeSmem<G, NL>& sm);

// 16-byte (LDG.E.128 / STG.E.128) access to an element pair (i, i+1) of one party's array
__device__ __forceinline__ bool al16(const u64* p) { return ((uintptr_t)p & 15u) == 0; }
__device__ __forceinline__ ulonglong2 ld128(const u64* p) { return *reinterpret_cast<const ulonglong2*>(p); }
__device__ __forceinline__ void st128(u64* p, u64 a, u64 b) { *reinterpret_cast<ulonglong2*>(p) = make_ulonglong2(a, b); }

// ================================================================================ BOTH ====
struct BothP {
    const Keys* Kp;          // points into the kernel's parameter space (__grid_constant__)
    using S = Sh;
    static constexpr bool kPair = false;
#ifndef MPC_BOTH_KV
#define MPC_BOTH_KV 1
#endif
    static constexpr int kV = MPC_BOTH_KV;   // unit pairs per lane per pass (registers hold both parties)
    __device__ __forceinline__ int party() const { return -1; }
    __device__ __forceinline__ bool k0ok() const { return true; }
    __device__ __forceinline__ S zero() const { return {0, 0}; }
    __device__ __forceinline__ S ld(SP a, i64 i) const { return {a.p[0][i], a.p[1][i]}; }
    __device__ __forceinline__ void st(SO a, i64 i, S v) const { a.p[0][i] = v.s0; a.p[1][i] = v.s1; }
    // element pair (i, i+1): plain 8-byte accesses here (two per party, together fully coalesced) --
    // the 16-byte form of PairP measured 3 % (softmax) to 15 % (Beaver mul) slower in this mode
    __device__ __forceinline__ void ld_pair(SP a, i64 i, bool va, bool vb, S& x0, S& x1) const {
        x0 = x1 = zero();
        if (va) x0 = ld(a, i);
        if (vb) x1 = ld(a, i + 1);
    }
    __device__ __forceinline__ void st_pair(SO a, i64 i, bool va, bool vb, S x0, S x1) const {
        if (va) st(a, i, x0);
        if (vb) st(a, i + 1, x1);
    }
    __device__ __forceinline__ S add(S a, S b) const { return sh_add(a, b); }
    __device__ __forceinline__ S sub(S a, S b) const { return sh_sub(a, b); }
    __device__ __forceinline__ S neg(S a) const { return sh_neg(a); }
    __device__ __forceinline__ S addp(S a, u64 e) const { return sh_addp(a, e); }
    __device__ __forceinline__ S shr_(S a, int k) const { return sh_shr(a, k); }
    __device__ __forceinline__ S muli(S a, u64 k) const { return sh_muli(a, k); }
    __device__ __forceinline__ S mulf(S a, u64 e) const { return sh_mulf(a, e); }
    __device__ __forceinline__ S notb(S b) const { return sh_not(b); }
    __device__ __forceinline__ S pm1(S s) const { return {1ull - 2ull * s.s0, 0ull - 2ull * s.s1}; }   // 1 - 2s
    __device__ __forceinline__ S shl(S a, int k) const { return {a.s0 << k, a.s1 << k}; }
    __device__ __forceinline__ S sumw(S a) const {                     // warp sum (local)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) { a.s0 += __shfl_xor_sync(FULL, a.s0, o); a.s1 += __shfl_xor_sync(FULL, a.s1, o); }
        return a;
    }
    __device__ __forceinline__ S divp(S a, i64 d) const;               // per-share floor division
    __device__ __forceinline__ S bm(u64 u, u32 s, S x, S y) { return mpc::bm(*Kp, u, s, x, y); }
    __device__ __forceinline__ void bm2(u64 u, u32 s, S x0, S y0, S x1, S y1, S& z0, S& z1) {
        mpc::bm2(*Kp, u, s, x0, y0, x1, y1, z0, z1);
    }
    template <bool WIDE>
    __device__ __forceinline__ S ltz(u64 q, u32 s, int w, S x, int lane) { return mpc::ltz<WIDE>(*Kp, q, s, w, x, lane); }
    // w = 33 with the levels' Philox rebalanced over idle lanes (proto_both.cuh ltz33_rebal): faster where
    // the kernel has registers to spare (cmp / ReLU -9 %, short-row max), slower inside GELU's schedule
    template <bool WIDE>
    __device__ __forceinline__ S ltz_rb(u64 q, u32 s, int w, S x, int lane) { return mpc::ltz<WIDE, true>(*Kp, q, s, w, x, lane); }
#ifndef MPC_BOTH_LTZ_O_INLINE
#define MPC_BOTH_LTZ_O_INLINE 1
#endif
    template <bool WIDE>
#if MPC_BOTH_LTZ_O_INLINE
    __device__ __forceinline__ S ltz_o(u64 q, u32 s, int w, S x, int lane) { return ltz<WIDE>(q, s, w, x, lane); }
#else
    __device__ __noinline__ S ltz_o(u64 q, u32 s, int w, S x, int lane) { return ltz<WIDE>(q, s, w, x, lane); }
#endif
    __device__ __forceinline__ S sq(u64 u, u32 s, S y) { return mpc::sq1(*Kp, u, s, y); }
    // two Beaver steps of one unit (power basis: v^3 at sA, v^4 at sB -- one round in PAIR)
    __device__ __forceinline__ void bm_dual(u64 u, u32 sA, S xA, S yA, u32 sB, S xB, S yB, S& zA, S& zB) {
        zA = mpc::bm(*Kp, u, sA, xA, yA); zB = mpc::bm(*Kp, u, sB, xB, yB);
    }
    __device__ __forceinline__ void bm2_dual(u64 u, u32 sA, S xA0, S yA0, S xA1, S yA1, u32 sB, S xB0, S yB0, S xB1,
                                             S yB1, S& zA0, S& zA1, S& zB0, S& zB1) {
        mpc::bm2(*Kp, u, sA, xA0, yA0, xA1, yA1, zA0, zA1);
        mpc::bm2(*Kp, u, sB, xB0, yB0, xB1, yB1, zB0, zB1);
    }
    // broadcast triple: row mask + opening, then the element products
    __device__ __forceinline__ BRow bmb_row(u64 r, u32 s, S y) { return mpc::bmb_row(*Kp, r, s, y); }
    __device__ __forceinline__ void bmb2(u64 u, u32 s, S x0, S x1, const BRow& r0, const BRow& r1, S& z0, S& z1) {
        mpc::bmb2(*Kp, u, s, x0, x1, r0, r1, z0, z1);
    }
    template <int G, int NL>
    __device__ __forceinline__ void ltz_cone(u64 q0, u32 s, int w, const S (&x)[G], S (&z)[G], int lane, ConeSmem<G, NL>& sm) {
        ltz_cone_both<G, NL>(*Kp, q0, s, w, x, z, lane, sm);
    }
    __device__ __forceinline__ void sq2(u64 u, u32 s, S y0, S y1, S& z0, S& z1) { mpc::sq2(*Kp, u, s, y0, y1, z0, z1); }
    __device__ __forceinline__ u64 open(S x) const { return x.s0 + x.s1; }
    // matrix-triple masking: this party's share minus its mask half; two openings
    __device__ __forceinline__ S mask2(S x, u64 r0, u64 r1) const { return {x.s0 - r0, x.s1 - r1}; }
    __device__ __forceinline__ void open2(S a, S b, u64& ea, u64& eb) const { ea = a.s0 + a.s1; eb = b.s0 + b.s1; }
    template <int V>
    __device__ __forceinline__ void bm2v(const u64 (&u)[V], u32 s, const S (&x0)[V], const S (&y0)[V],
                                         const S (&x1)[V], const S (&y1)[V], S (&z0)[V], S (&z1)[V]) {
#pragma unroll
        for (int v = 0; v < V; ++v) mpc::bm2(*Kp, u[v], s, x0[v], y0[v], x1[v], y1[v], z0[v], z1[v]);
    }
    template <int V>
    __device__ __forceinline__ void sq2v(const u64 (&u)[V], u32 s, const S (&y0)[V], const S (&y1)[V],
                                         S (&z0)[V], S (&z1)[V]) {
#pragma unroll
        for (int v = 0; v < V; ++v) mpc::sq2(*Kp, u[v], s, y0[v], y1[v], z0[v], z1[v]);
    }
};

__device__ __forceinline__ u64 floordiv_share(u64 a, i64 d)
{
    const i64 x = (i64)a;
    i64 q = x / d;
    if ((x % d) != 0 && x < 0) --q;
    return (u64)q;
}
__device__ __forceinline__ Sh BothP::divp(Sh a, i64 d) const { return {floordiv_share(a.s0, d), floordiv_share(a.s1, d)}; }

// ================================================================================ PAIR ====
constexpr int XW = 8;                // u64 words per lane per round (max)
constexpr int XSLOT_RX = 2 * XW * 32 * 2;   // u64 per warp slot: LL [buf][word][lane][2]; LL63 uses the
                                            // first [buf][word][lane] main words, then [buf][word] top-bit
                                            // words
constexpr u64 M63 = 0x7fffffffffffffffull;

// Device view of one party's exchange memory.
struct XMem {
    u64* rx;          // [slots][2][XW][32] receive buffers (peer writes)
    u64* flag;        // [slots][4]          my flags (peer writes word 0)
    u64* round;       // [slots]             persistent round counters (local only)
    u32* tags;        // [slots][32]         persistent per-lane LL63 tag bits (local only)
    int* err;         // error word (1 = exchange timeout)
    u64* prx;         // peer's rx   (remote or, loopback, the other party's local buffer)
    u64* pflag;       // peer's flag
    int slots;
};

__device__ __forceinline__ u64 ld_acquire_sys(const u64* p)
{
    u64 v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(u64* p, u64 v)
{
    asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u64 ld_acquire_gpu(const u64* p)
{
    u64 v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(u64* p, u64 v)
{
    asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u64 ld_volatile(const u64* p)
{
    u64 v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ u64 globaltimer()
{
    u64 t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Dealer correction-stream state: only the stream role (R = 1) carries it, so the
// R = 0 kernels (party 0, the simulated dealer, loopback without a stream) compile exactly as
// without the feature.
template <int R> struct StreamState {
    static constexpr int cmode = 0;
};
template <> struct StreamState<1> {
    u64* cw;                 // this thread's column of the launch's stream segment
    u32 cst, ck, ccap;       // stride (threads of the party's launch), next k, dealer capacity (words per thread)
    int cmode;               // 0 (party 0 CTAs of a loopback launch), 1 read the stream, 2 the dealer
};

// R: 0 = party 0, or party 1 simulating the dealer from K_0 (reading R7); 1 = the stream roles:
// party 1 reading the dealer's correction stream (cmode 1) or the dealer's own pass (cmode 2).
template <int R>
struct PairP : StreamState<R> {
    using StreamState<R>::cmode;
#ifndef MPC_PAIR_KV
#define MPC_PAIR_KV 2
#endif
    static constexpr int kV = MPC_PAIR_KV;   // unit pairs per lane per exchange round (2: loopback softmax 5 %, mul 18 % faster than 1)
    const Keys* Kp;          // kernel parameter space (__grid_constant__)
    int pty;                 // 0 | 1
    // per-warp exchange state (set by bind())
    u64* rx; u64* prx; u64* flag; u64* pflag; u64* rstate; u32* tstate; int* err;
    u64 rnd;
    u32 tg;                  // LL63 tag bits: main word (b, k) at bit 8b + k, top-bit word at 16 + 8b + k
    int dead;
    int local;               // loopback: the peer is on this GPU -> gpu-scope release/acquire
    int fmt;                 // exchange wire format: 0 LL, 1 LL63 (warp-uniform)
    // Dealer correction stream: party 1's correction words -- Beaver / square /
    // broadcast c1, AND-triple c1 (G and P gate of a level packed in one word), daBit r1A -- are the
    // only values party 1 would need K_0 for.  cmode 0: derived from K_0 (the dealer simulated by
    // party 1, reading R7); 1: read from the dealer's stream (party 1 never touches K_0); 2: this
    // launch IS the dealer (derives them and writes the stream; its exchange memory is a self-loop --
    // every put comes back to the same warp -- so it runs party 1's exact code path).  The k-th
    // correction of thread t is word cw[k * cst] (cw = stream base + t): coalesced across a warp,
    // and the same (thread, k) in the dealer's launch and party 1's because both run the same kernel
    // with the same grid and data-independent control flow.
    using S = u64;
    static constexpr bool kPair = true;
    static constexpr u64 kTimeoutNs = 10ull * 1000 * 1000 * 1000;   // 10 s, then poison

    __device__ __forceinline__ void bind(const XMem& m, int slot) {
        dead = 0;
        rx = m.rx + (i64)slot * XSLOT_RX;
        prx = m.prx + (i64)slot * XSLOT_RX;
        flag = m.flag + (i64)slot * 4;
        pflag = m.pflag + (i64)slot * 4;
        rstate = m.round + slot;
        tstate = m.tags + (i64)slot * 32;
        err = m.err;
        rnd = *rstate;
        tg = tstate[threadIdx.x & 31];
        dead = 0;
    }
    __device__ __forceinline__ void unbind(int lane) {
        if (lane == 0) *rstate = rnd;
        tstate[lane] = tg;
    }
    __device__ __forceinline__ int party() const { return pty; }
    // K_0 is this thread's to use: party 0 always; party 1 only while it simulates the dealer
    __device__ __forceinline__ bool k0ok() const {
        if constexpr (R == 0) return true;
        else return pty == 0 || cmode != 1;
    }
    __device__ __forceinline__ bool sread() const {          // party 1 reads the stream
        if constexpr (R == 0) return false;
        else return cmode == 1;
    }
    // party 1's next correction word: derive() (K_0) unless it comes from the dealer's stream
    template <class F>
    __device__ __forceinline__ u64 corr(F derive) {
        if constexpr (R == 0) {
            return derive();
        } else {
            if (cmode == 1) { const u64 v = this->cw[(u64)this->ck * this->cst]; ++this->ck; return v; }
            const u64 v = derive();
            if (cmode == 2) { if (this->ck < this->ccap) this->cw[(u64)this->ck * this->cst] = v; ++this->ck; }
            return v;
        }
    }
    // ---- exchange: put words, exch(), get peer's words ----
    // Two wire formats, both "LL"-style (the idea of NCCL's low-latency protocol: the data carries
    // its own readiness tag, so there are no fences, flags or warp barriers on the data path), chosen
    // per context (mpc_ctx_set_exchange):
    //  LL   (fmt 0): payload word = two 8-byte words {lo32 | tag32, hi32 | tag32}, tag = the 32-bit
    //                round, one 16-byte store / load.  2 wire bytes per payload byte, fewest
    //                instructions -- the default in PAIR_LOOPBACK (local HBM, instruction-bound).
    //  LL63 (fmt 1): payload word = ONE 8-byte store {bits 0..62 | tag << 63}; the 32 lanes' bit 63
    //                is gathered with a ballot and lane 0 sends it as one extra tagged word per
    //                (round, word): 33 words per 32 (wire / payload 1.031) -- the default in
    //                MPC_MODE_PAIR (NVLink, bytes-bound).  The one-bit tag FLIPS on every write of
    //                a receive word: both parties issue the same put / get sequence, so each lane
    //                tracks its words' current tags (register tg, persisted per warp slot).
    // Both: round r uses receive buffer r mod 2 (a sender is at most one round ahead of its peer, so
    // it never overwrites a word the peer has not read), and aligned 8-byte stores are single-copy
    // atomic.  put / get must be issued by all 32 lanes together (LL63's ballot); a lane with
    // live = false sends, reads and (LL63) flips nothing for that word -- both parties pass the same
    // live pattern.
    // (both inline: an out-of-line LL63 put / get kept its code out of the loopback kernels' stream
    // but cost 20 % in LL63 loopback -- call overhead per word; inline costs LL 2 %)
#ifndef MPC_XFMT_LL_ONLY
#define MPC_XFMT_LL_ONLY 0     // A/B builds: compile the LL63 path out
#endif
    __device__ __forceinline__ void put(int lane, int k, u64 v, bool live = true) {
        const u64 r = rnd + 1;                                   // the round being sent
        const int b = (int)(r & 1);
        if (MPC_XFMT_LL_ONLY || !fmt) {
            const u64 tag = r << 32;
            u64* d = prx + ((b * XW + k) * 32 + lane) * 2;
            const u64 lo = (v & 0xffffffffull) | tag, hi = (v >> 32) | tag;
            if (live) asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" :: "l"(d), "l"(lo), "l"(hi) : "memory");
            return;
        }
        put63(lane, k, v, live, b);
    }
#ifndef MPC_LL63_INLINE
#define MPC_LL63_INLINE 1      // LL63 put / get inline: loopback LL63 softmax 2.03 -> 1.63 ms, GELU 1M 1.59 -> 1.34 ms; LL +2 % (r02)
#endif
#if MPC_LL63_INLINE
    __device__ __forceinline__ void put63(int lane, int k, u64 v, bool live, int b) {
#else
    __device__ __noinline__ void put63(int lane, int k, u64 v, bool live, int b) {
#endif
        const u32 mb = 1u << (8 * b + k), eb = 1u << (16 + 8 * b + k);
        tg ^= eb;
        if (live) tg ^= mb;
        const u32 top = __ballot_sync(FULL, live && (v >> 63));
        u64* d = prx + (b * XW + k) * 32 + lane;
        if (live) asm volatile("st.volatile.global.u64 [%0], %1;" :: "l"(d), "l"((v & M63) | ((u64)((tg & mb) != 0) << 63)) : "memory");
        if (lane == 0) {
            u64* e = prx + 2 * XW * 32 + b * XW + k;
            asm volatile("st.volatile.global.u64 [%0], %1;" :: "l"(e), "l"((u64)top | ((u64)((tg & eb) != 0) << 63)) : "memory");
        }
    }
    __device__ __forceinline__ void exch(int lane) {
        (void)lane;
        ++rnd;                                   // the round now being received
    }
    __device__ __forceinline__ u64 get(int lane, int k) {
        const int b = (int)(rnd & 1);                            // this round's buffer (tags set by put)
        if (MPC_XFMT_LL_ONLY || !fmt) {
            const u64* sp = rx + ((b * XW + k) * 32 + lane) * 2;
            const u64 want = rnd & 0xffffffffull;
            u64 lo, hi;
            asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(sp) : "memory");
            if (((lo >> 32) != want || (hi >> 32) != want) && !dead) {
                const u64 t0 = globaltimer();
                unsigned spins = 0;
                do {                             // (a __nanosleep backoff here measured 2x slower)
                    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(sp) : "memory");
                    if ((++spins & 1023) == 0 && globaltimer() - t0 > kTimeoutNs) { atomicCAS(err, 0, 1); dead = 1; break; }
                } while ((lo >> 32) != want || (hi >> 32) != want);
            }
            return (lo & 0xffffffffull) | (hi << 32);
        }
        return get63(lane, k, b);
    }
#if MPC_LL63_INLINE
    __device__ __forceinline__ u64 get63(int lane, int k, int b) {
#else
    __device__ __noinline__ u64 get63(int lane, int k, int b) {
#endif
        const u64* sp = rx + (b * XW + k) * 32 + lane;
        const u64* ep = rx + 2 * XW * 32 + b * XW + k;
        const u64 want = (tg >> (8 * b + k)) & 1u, wante = (tg >> (16 + 8 * b + k)) & 1u;
        u64 v, e;
        asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(sp) : "memory");
        asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(e) : "l"(ep) : "memory");
        if (((v >> 63) != want || (e >> 63) != wante) && !dead) {
            const u64 t0 = globaltimer();
            unsigned spins = 0;
            do {
                asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(sp) : "memory");
                asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(e) : "l"(ep) : "memory");
                if ((++spins & 1023) == 0 && globaltimer() - t0 > kTimeoutNs) { atomicCAS(err, 0, 1); dead = 1; break; }
            } while ((v >> 63) != want || (e >> 63) != wante);
        }
        return (v & M63) | ((u64)((u32)e >> lane & 1u) << 63);
    }

    // ---- local share ops (party 0 carries public addends) ----
    __device__ __forceinline__ S zero() const { return 0; }
#ifndef MPC_DEALER_LDST
#define MPC_DEALER_LDST 1     // A/B only: 0 drops the dealer's share-access guards (unsafe for the dealer)
#endif
    __device__ __forceinline__ bool nosh() const {          // the dealer: no shares
        if constexpr (R == 0) return false;
        else return MPC_DEALER_LDST && cmode == 2;
    }
    __device__ __forceinline__ S ld(SP a, i64 i) const { return nosh() ? 0ull : a.p[pty][i]; }
    __device__ __forceinline__ void st(SO a, i64 i, S v) const { if (!nosh()) a.p[pty][i] = v; }
    // element pair (i, i+1) of this party's array: one 16-byte access (LDG.E.128 / STG.E.128) when both
    // are valid and aligned (loopback Beaver mul 5 % faster)
    __device__ __forceinline__ void ld_pair(SP a, i64 i, bool va, bool vb, S& x0, S& x1) const {
        x0 = x1 = 0;
        if (nosh()) return;
        if (va && vb && al16(a.p[pty] + i)) { const ulonglong2 t = ld128(a.p[pty] + i); x0 = t.x; x1 = t.y; }
        else { if (va) x0 = ld(a, i); if (vb) x1 = ld(a, i + 1); }
    }
    __device__ __forceinline__ void st_pair(SO a, i64 i, bool va, bool vb, S x0, S x1) const {
        if (nosh()) return;
        if (va && vb && al16(a.p[pty] + i)) st128(a.p[pty] + i, x0, x1);
        else { if (va) st(a, i, x0); if (vb) st(a, i + 1, x1); }
    }
    __device__ __forceinline__ S add(S a, S b) const { return a + b; }
    __device__ __forceinline__ S sub(S a, S b) const { return a - b; }
    __device__ __forceinline__ S neg(S a) const { return 0ull - a; }
    __device__ __forceinline__ S addp(S a, u64 e) const { return pty == 0 ? a + e : a; }
    __device__ __forceinline__ S shr_(S a, int k) const { return shr(a, k); }
    __device__ __forceinline__ S muli(S a, u64 k) const { return a * k; }
    __device__ __forceinline__ S mulf(S a, u64 e) const { return shr(a * e, FRAC); }
    __device__ __forceinline__ S notb(S b) const { return pty == 0 ? 1ull - b : 0ull - b; }
    __device__ __forceinline__ S pm1(S s) const { return pty == 0 ? 1ull - 2ull * s : 0ull - 2ull * s; }
    __device__ __forceinline__ S shl(S a, int k) const { return a << k; }
    __device__ __forceinline__ S sumw(S a) const {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(FULL, a, o);
        return a;
    }
    __device__ __forceinline__ S divp(S a, i64 d) const { return floordiv_share(a, d); }

    // ---- Beaver (DESIGN.md 2.3/2.4); party 1 also plays the dealer's correction (R7) ----
    // c0: party 0's c share (K_0; ignored -- and not computed by the caller -- when party 1 reads the stream)
    __device__ __forceinline__ void triple(u64 u, u32 s, u64 c0, u64& a, u64& b, u64& c) {
        if (pty == 0) {
            const uint4 A0 = prg(Kp->k0, u, s, 0);
            a = w64(A0.x, A0.y); b = w64(A0.z, A0.w); c = c0;
        } else if (sread()) {                         // the dealer's c1 from the stream
            const uint4 A1 = prg(Kp->k1, u, s, 0);
            a = w64(A1.x, A1.y); b = w64(A1.z, A1.w);
            c = corr([] { return 0ull; });
        } else {                                      // both blocks in one basic block (ILP)
            const uint4 A0 = prg(Kp->k0, u, s, 0), A1 = prg(Kp->k1, u, s, 0);
            a = w64(A1.x, A1.y); b = w64(A1.z, A1.w);
            const u64 cc = (w64(A0.x, A0.y) + a) * (w64(A0.z, A0.w) + b) - c0;
            c = corr([&] { return cc; });
        }
    }
    // the triples of unit pair (u, u+1) (u even): one c0 block serves both; each path keeps all its
    // Philox blocks in one basic block so they interleave (ILP)
    __device__ __forceinline__ void triple_pair(u64 u, u32 s, u64& a0, u64& b0, u64& c0, u64& a1, u64& b1, u64& c1) {
        if (pty == 0) {
            const uint4 C = prg(Kp->k0, u >> 1, s, 1), Au = prg(Kp->k0, u, s, 0), Av = prg(Kp->k0, u + 1, s, 0);
            a0 = w64(Au.x, Au.y); b0 = w64(Au.z, Au.w); a1 = w64(Av.x, Av.y); b1 = w64(Av.z, Av.w);
            c0 = w64(C.x, C.y); c1 = w64(C.z, C.w);
        } else if (sread()) {
            const uint4 Au = prg(Kp->k1, u, s, 0), Av = prg(Kp->k1, u + 1, s, 0);
            a0 = w64(Au.x, Au.y); b0 = w64(Au.z, Au.w); a1 = w64(Av.x, Av.y); b1 = w64(Av.z, Av.w);
            c0 = corr([] { return 0ull; }); c1 = corr([] { return 0ull; });
        } else {
            const uint4 C = prg(Kp->k0, u >> 1, s, 1), Au = prg(Kp->k0, u, s, 0), Av = prg(Kp->k0, u + 1, s, 0);
            const uint4 Bu = prg(Kp->k1, u, s, 0), Bv = prg(Kp->k1, u + 1, s, 0);
            a0 = w64(Bu.x, Bu.y); b0 = w64(Bu.z, Bu.w); a1 = w64(Bv.x, Bv.y); b1 = w64(Bv.z, Bv.w);
            const u64 cu = (w64(Au.x, Au.y) + a0) * (w64(Au.z, Au.w) + b0) - w64(C.x, C.y);
            const u64 cv = (w64(Av.x, Av.y) + a1) * (w64(Av.z, Av.w) + b1) - w64(C.z, C.w);
            c0 = corr([&] { return cu; }); c1 = corr([&] { return cv; });
        }
    }
    __device__ __forceinline__ uint4 cblk(u64 u, u32 s) const {          // the c0 block of unit pair (u, u+1)
        return k0ok() ? prg(Kp->k0, u >> 1, s, 1) : make_uint4(0, 0, 0, 0);
    }
    __device__ __forceinline__ S bm_finish(u64 a, u64 b, u64 c, u64 e, u64 f) const {
        return pty == 0 ? c + e * (b + f) + f * a : c + e * b + f * a;   // party 0: e b + e f = e (b + f)
    }
#if MPC_PAIR_BM_INLINE
    __device__ __forceinline__ S bm(u64 u, u32 s, S x, S y) {
#else
    __device__ __noinline__ S bm(u64 u, u32 s, S x, S y) {
#endif
        const int lane = threadIdx.x & 31;
        u64 a, b, c;
        const uint4 C = cblk(u, s);
        triple(u, s, (u & 1) ? w64(C.z, C.w) : w64(C.x, C.y), a, b, c);
        put(lane, 0, x - a); put(lane, 1, y - b);
        exch(lane);
        const u64 e = (x - a) + get(lane, 0), f = (y - b) + get(lane, 1);
        return bm_finish(a, b, c, e, f);
    }
#if MPC_PAIR_BM_INLINE
    __device__ __forceinline__ void bm2(u64 u, u32 s, S x0, S y0, S x1, S y1, S& z0, S& z1) {
#else
    __device__ __noinline__ void bm2(u64 u, u32 s, S x0, S y0, S x1, S y1, S& z0, S& z1) {
#endif
        const int lane = threadIdx.x & 31;
        u64 a0, b0, c0, a1, b1, c1;
        triple_pair(u, s, a0, b0, c0, a1, b1, c1);
        put(lane, 0, x0 - a0); put(lane, 1, y0 - b0); put(lane, 2, x1 - a1); put(lane, 3, y1 - b1);
        exch(lane);
        z0 = bm_finish(a0, b0, c0, (x0 - a0) + get(lane, 0), (y0 - b0) + get(lane, 1));
        z1 = bm_finish(a1, b1, c1, (x1 - a1) + get(lane, 2), (y1 - b1) + get(lane, 3));
    }

    // two Beaver steps of one unit / unit pair in ONE round (power basis)
    __device__ __forceinline__ void bm_dual(u64 u, u32 sA, S xA, S yA, u32 sB, S xB, S yB, S& zA, S& zB) {
        const int lane = threadIdx.x & 31;
        u64 aA, bA, cA, aB, bB, cB;
        const uint4 CA = cblk(u, sA), CB = cblk(u, sB);
        triple(u, sA, (u & 1) ? w64(CA.z, CA.w) : w64(CA.x, CA.y), aA, bA, cA);
        triple(u, sB, (u & 1) ? w64(CB.z, CB.w) : w64(CB.x, CB.y), aB, bB, cB);
        put(lane, 0, xA - aA); put(lane, 1, yA - bA); put(lane, 2, xB - aB); put(lane, 3, yB - bB);
        exch(lane);
        zA = bm_finish(aA, bA, cA, (xA - aA) + get(lane, 0), (yA - bA) + get(lane, 1));
        zB = bm_finish(aB, bB, cB, (xB - aB) + get(lane, 2), (yB - bB) + get(lane, 3));
    }
    __device__ __forceinline__ void bm2_dual(u64 u, u32 sA, S xA0, S yA0, S xA1, S yA1, u32 sB, S xB0, S yB0, S xB1,
                                             S yB1, S& zA0, S& zA1, S& zB0, S& zB1) {
        static_assert(8 <= XW, "exchange width");
        const int lane = threadIdx.x & 31;
        u64 a[4], b[4], c[4];
        triple_pair(u, sA, a[0], b[0], c[0], a[1], b[1], c[1]);
        triple_pair(u, sB, a[2], b[2], c[2], a[3], b[3], c[3]);
        const S xs[4] = {xA0, xA1, xB0, xB1}, ys[4] = {yA0, yA1, yB0, yB1};
#pragma unroll
        for (int k = 0; k < 4; ++k) { put(lane, 2 * k, xs[k] - a[k]); put(lane, 2 * k + 1, ys[k] - b[k]); }
        exch(lane);
        S zs[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            zs[k] = bm_finish(a[k], b[k], c[k], (xs[k] - a[k]) + get(lane, 2 * k), (ys[k] - b[k]) + get(lane, 2 * k + 1));
        zA0 = zs[0]; zA1 = zs[1]; zB0 = zs[2]; zB1 = zs[3];
    }

    // ---- broadcast triple (NEXT #2): f opened once per row, e per element ----
    __device__ __forceinline__ BRow bmb_row(u64 r, u32 s, S y) {
        const int lane = threadIdx.x & 31;
        const uint4 B0 = k0ok() ? prg(Kp->k0, r, s, 6) : make_uint4(0, 0, 0, 0);
        BRow Rw;
        Rw.b0 = w64(B0.x, B0.y); Rw.b1 = 0;
        if (pty == 1) { const uint4 B1 = prg(Kp->k1, r, s, 6); Rw.b1 = w64(B1.x, B1.y); }
        const u64 m = y - (pty == 0 ? Rw.b0 : Rw.b1);
        put(lane, 0, m);
        exch(lane);
        Rw.f = m + get(lane, 0);
        return Rw;
    }
    __device__ __forceinline__ void bmb2(u64 u, u32 s, S x0, S x1, const BRow& r0, const BRow& r1, S& z0, S& z1) {
        const int lane = threadIdx.x & 31;
        uint4 Au = make_uint4(0, 0, 0, 0), Av = Au;
        if (k0ok()) { Au = prg(Kp->k0, u, s, 4); Av = prg(Kp->k0, u + 1, s, 4); }
        u64 au = w64(Au.x, Au.y), cu = w64(Au.z, Au.w), av = w64(Av.x, Av.y), cv = w64(Av.z, Av.w);
        if (pty == 1) {                                  // party 1: own a1, dealer's c1
            const uint4 A1 = prg(Kp->k1, u >> 1, s, 5);
            const u64 a1u = w64(A1.x, A1.y), a1v = w64(A1.z, A1.w);
            const u64 a0u = au, c0u = cu, a0v = av, c0v = cv;
            cu = corr([&] { return (a0u + a1u) * (r0.b0 + r0.b1) - c0u; });
            cv = corr([&] { return (a0v + a1v) * (r1.b0 + r1.b1) - c0v; });
            au = a1u; av = a1v;
        }
        put(lane, 0, x0 - au); put(lane, 1, x1 - av);
        exch(lane);
        const u64 eu = (x0 - au) + get(lane, 0), ev = (x1 - av) + get(lane, 1);
        const u64 bu = pty == 0 ? r0.b0 : r0.b1, bv = pty == 0 ? r1.b0 : r1.b1;
        z0 = cu + eu * bu + r0.f * au + (pty == 0 ? eu * r0.f : 0ull);
        z1 = cv + ev * bv + r1.f * av + (pty == 0 ? ev * r1.f : 0ull);
    }

    // ---- squares with square-pair triples (NEXT #2): one word per element per round ----
    __device__ __forceinline__ void sq_triple(u64 u, u32 s, u64 a1_other_half, u64& a, u64& c) {
        if (pty == 0) { const uint4 A0 = prg(Kp->k0, u, s, 2); a = w64(A0.x, A0.y); c = w64(A0.z, A0.w); }
        else {
            a = a1_other_half;
            const u64 a1 = a;
            c = corr([&] { const uint4 A0 = prg(Kp->k0, u, s, 2); const u64 t = w64(A0.x, A0.y) + a1; return t * t - w64(A0.z, A0.w); });
        }
    }
    __device__ __forceinline__ S sq_finish(u64 a, u64 c, u64 e) const {
        return pty == 0 ? c + e * (2ull * a + e) : c + 2ull * e * a;
    }
    __device__ __forceinline__ S sq(u64 u, u32 s, S y) {
        const int lane = threadIdx.x & 31;
        u64 a1 = 0;
        if (pty == 1) { const uint4 A1 = prg(Kp->k1, u >> 1, s, 3); a1 = (u & 1) ? w64(A1.z, A1.w) : w64(A1.x, A1.y); }
        u64 a, c;
        sq_triple(u, s, a1, a, c);
        put(lane, 0, y - a);
        exch(lane);
        return sq_finish(a, c, (y - a) + get(lane, 0));
    }
    __device__ __forceinline__ void sq2(u64 u, u32 s, S y0, S y1, S& z0, S& z1) {
        const int lane = threadIdx.x & 31;
        u64 a1e = 0, a1o = 0;
        if (pty == 1) { const uint4 A1 = prg(Kp->k1, u >> 1, s, 3); a1e = w64(A1.x, A1.y); a1o = w64(A1.z, A1.w); }
        u64 a0, c0, a1, c1;
        sq_triple(u, s, a1e, a0, c0);
        sq_triple(u + 1, s, a1o, a1, c1);
        put(lane, 0, y0 - a0); put(lane, 1, y1 - a1);
        exch(lane);
        z0 = sq_finish(a0, c0, (y0 - a0) + get(lane, 0));
        z1 = sq_finish(a1, c1, (y1 - a1) + get(lane, 1));
    }

    // V unit pairs in one exchange round (4V / 2V words per lane)
    template <int V>
    __device__ __forceinline__ void bm2v(const u64 (&u)[V], u32 s, const S (&x0)[V], const S (&y0)[V],
                                         const S (&x1)[V], const S (&y1)[V], S (&z0)[V], S (&z1)[V]) {
        static_assert(4 * V <= XW, "exchange width");
        const int lane = threadIdx.x & 31;
        u64 a0[V], b0[V], c0[V], a1[V], b1[V], c1[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            triple_pair(u[v], s, a0[v], b0[v], c0[v], a1[v], b1[v], c1[v]);
            put(lane, 4 * v + 0, x0[v] - a0[v]); put(lane, 4 * v + 1, y0[v] - b0[v]);
            put(lane, 4 * v + 2, x1[v] - a1[v]); put(lane, 4 * v + 3, y1[v] - b1[v]);
        }
        exch(lane);
#pragma unroll
        for (int v = 0; v < V; ++v) {
            z0[v] = bm_finish(a0[v], b0[v], c0[v], (x0[v] - a0[v]) + get(lane, 4 * v + 0), (y0[v] - b0[v]) + get(lane, 4 * v + 1));
            z1[v] = bm_finish(a1[v], b1[v], c1[v], (x1[v] - a1[v]) + get(lane, 4 * v + 2), (y1[v] - b1[v]) + get(lane, 4 * v + 3));
        }
    }
    template <int V>
    __device__ __forceinline__ void sq2v(const u64 (&u)[V], u32 s, const S (&y0)[V], const S (&y1)[V],
                                         S (&z0)[V], S (&z1)[V]) {
        static_assert(2 * V <= XW, "exchange width");
        const int lane = threadIdx.x & 31;
        u64 a0[V], c0[V], a1[V], c1[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            u64 a1e = 0, a1o = 0;
            if (pty == 1) { const uint4 A1 = prg(Kp->k1, u[v] >> 1, s, 3); a1e = w64(A1.x, A1.y); a1o = w64(A1.z, A1.w); }
            sq_triple(u[v], s, a1e, a0[v], c0[v]);
            sq_triple(u[v] + 1, s, a1o, a1[v], c1[v]);
            put(lane, 2 * v, y0[v] - a0[v]); put(lane, 2 * v + 1, y1[v] - a1[v]);
        }
        exch(lane);
#pragma unroll
        for (int v = 0; v < V; ++v) {
            z0[v] = sq_finish(a0[v], c0[v], (y0[v] - a0[v]) + get(lane, 2 * v));
            z1[v] = sq_finish(a1[v], c1[v], (y1[v] - a1[v]) + get(lane, 2 * v + 1));
        }
    }

    // ---- AND gates on XOR-shared plane words; up to 2 gates (4 words) per round ----
    __device__ __forceinline__ void and_triple(uint4 t0, uint4 t1, int which, u32& a, u32& b, u32& c) {
        // which = 0: (a1,b1) = t1.x,t1.y ; 1: t1.z,t1.w
        const u32 a1 = which ? t1.z : t1.x, b1 = which ? t1.w : t1.y;
        if (pty == 0) { a = t0.x; b = t0.y; c = t0.z; }
        else { a = a1; b = b1; c = (u32)corr([&] { return (u64)(((t0.x ^ a1) & (t0.y ^ b1)) ^ t0.z); }); }
    }
    // the G and P gates of one Kogge-Stone / cone node: party 1's two c1 words in ONE stream word
    __device__ __forceinline__ void and_triple2(uint4 tg, uint4 tp, uint4 t1, u32& ga, u32& gb, u32& gc,
                                                u32& pa, u32& pb, u32& pc) {
        if (pty == 0) { ga = tg.x; gb = tg.y; gc = tg.z; pa = tp.x; pb = tp.y; pc = tp.z; return; }
        ga = t1.x; gb = t1.y; pa = t1.z; pb = t1.w;
        const u64 cc = corr([&] {
            return (u64)(((tg.x ^ t1.x) & (tg.y ^ t1.y)) ^ tg.z) | ((u64)(((tp.x ^ t1.z) & (tp.y ^ t1.w)) ^ tp.z) << 32);
        });
        gc = (u32)cc; pc = (u32)(cc >> 32);
    }
    // this lane's daBit r1A (party 1): (r0B ^ r1B) - r0A with D0 = PRG(K_0, q, s, 2 + lane)
    __device__ __forceinline__ u64 dabit_r1A(uint4 D0, u32 r1B) {
        return corr([&] { return (u64)((D0.z & 1u) ^ r1B) - w64(D0.x, D0.y); });
    }
    __device__ __forceinline__ u32 and_finish(u32 a, u32 b, u32 c, u32 d, u32 e) const {
        return pty == 0 ? (c ^ (d & b) ^ (e & a) ^ (d & e)) : (c ^ (d & b) ^ (e & a));
    }

    // w <= 33, branch-free, daBit words in the idle slots of the last level (as ltz_narrow)
    __device__ __forceinline__ S ltz_narrow(u64 q, u32 s, int w, S x, int lane) {
        const int m = w - 1;
        const bool k0 = k0ok();
        const PrgQ Q0 = prg_q(Kp->k0, q, s), Q1 = prg_q(Kp->k1, q, s);
        u32 Pp = transpose32((u32)x, lane), Gp = 0;
        {
            const uint4 t0 = k0 ? prg(Q0, ltz_slot(0, lane, 0)) : make_uint4(0, 0, 0, 0);
            uint4 t1 = make_uint4(0, 0, 0, 0);
            if (pty == 1) t1 = prg(Q1, ltz_slot(0, lane, 0));
            u32 ta, tb, tc;
            and_triple(t0, t1, 0, ta, tb, tc);
            const u32 dd = (pty == 0 ? Pp : 0u) ^ ta, ee = (pty == 0 ? 0u : Pp) ^ tb;
            put(lane, 0, (u64)dd | ((u64)ee << 32));
            exch(lane);
            const u64 pw = get(lane, 0);
            const u32 g = and_finish(ta, tb, tc, dd ^ (u32)pw, ee ^ (u32)(pw >> 32));
            if (lane < m) Gp = g;
        }
        const int L = (m > 0) ? ceil_log2i(m) : 0;
        const bool trick = m > 16;
        uint4 Dlo = make_uint4(0, 0, 0, 0), Dhi = make_uint4(0, 0, 0, 0);
        u32 k1w = 0;
        for (int k = 0; k < L; ++k) {
            const int dl = 1 << k;
            const int src = (lane - dl) & 31;
            const u32 g = __shfl_sync(FULL, Gp, src), p = __shfl_sync(FULL, Pp, src);
            const bool act = lane >= dl && lane < m;
            const bool dab = trick && k == L - 1 && lane < 16;
            uint4 tg = make_uint4(0, 0, 0, 0), tp = tg;
            if (k0) { tg = prg(Q0, dab ? 2u + (u32)lane : ltz_slot(k + 1, lane, 0)); tp = prg(Q0, dab ? 18u + (u32)lane : ltz_slot(k + 1, lane, 1)); }
            uint4 t1 = make_uint4(0, 0, 0, 0);
            if (pty == 1) t1 = prg(Q1, dab ? 1u : ltz_slot(k + 1, lane, 0));
            u32 ga, gb, gc, pa, pb, pc;
            and_triple2(tg, tp, t1, ga, gb, gc, pa, pb, pc);
            const u32 dG = Pp ^ ga, eG = g ^ gb, dP = Pp ^ pa, eP = p ^ pb;
            put(lane, 0, (u64)dG | ((u64)eG << 32));
            put(lane, 1, (u64)dP | ((u64)eP << 32));
            exch(lane);
            const u64 w0 = get(lane, 0), w1 = get(lane, 1);
            const u32 ng = and_finish(ga, gb, gc, dG ^ (u32)w0, eG ^ (u32)(w0 >> 32));
            const u32 np = and_finish(pa, pb, pc, dP ^ (u32)w1, eP ^ (u32)(w1 >> 32));
            if (act) { Gp ^= ng; Pp = np; }
            if (dab) { Dlo = tg; Dhi = tp; k1w = t1.x; }
        }
        u32 bp;
        if (m == 0) bp = (u32)(x & 1ull);
        else bp = (u32)((x >> (w - 1)) & 1ull) ^ ((__shfl_sync(FULL, Gp, m - 1) >> lane) & 1u);
        uint4 D0;
        u32 d1x = 0;
        if (trick) {
            const u32 hx = __shfl_sync(FULL, Dhi.x, lane & 15), hy = __shfl_sync(FULL, Dhi.y, lane & 15);
            const u32 hz = __shfl_sync(FULL, Dhi.z, lane & 15);
            D0 = lane < 16 ? Dlo : make_uint4(hx, hy, hz, 0u);
            d1x = __shfl_sync(FULL, k1w, 0);
        } else {
            D0 = k0 ? prg(Q0, 2u + (u32)lane) : make_uint4(0, 0, 0, 0);
            if (pty == 1) d1x = prg(Q1, 1u).x;
        }
        u64 rA;
        u32 rB;
        if (pty == 0) { rA = w64(D0.x, D0.y); rB = D0.z & 1u; }
        else { rB = (d1x >> lane) & 1u; rA = dabit_r1A(D0, rB); }
        const u32 mine = bp ^ rB;
        put(lane, 0, (u64)mine);
        exch(lane);
        const u64 c = (u64)(mine ^ ((u32)get(lane, 0) & 1u));
        const u64 sg = 1ull - 2ull * c;
        return pty == 0 ? c + sg * rA : sg * rA;
    }

    // Out-of-line LTZ for schedules with several comparison sites (S13's 2-3 segment masks, the
    // clamp inside exp / NR): one copy of the circuit and its polling loops per kernel instead of
    // one per site.  Measured in loopback: GELU 2.6x faster (the inlined copies made the kernel's
    // instruction fetch the top stall); single-site kernels (ReLU) stay inlined (8 % faster).
    template <bool WIDE>
    __device__ __noinline__ S ltz_o(u64 q, u32 s, int w, S x, int lane) { return ltz<WIDE>(q, s, w, x, lane); }
    template <bool WIDE>
    __device__ __forceinline__ S ltz_rb(u64 q, u32 s, int w, S x, int lane) { return ltz<WIDE>(q, s, w, x, lane); }
#ifndef MPC_PAIR_BM_INLINE
#define MPC_PAIR_BM_INLINE 1
#endif
    template <bool WIDE>
    __device__ __forceinline__ S ltz(u64 q, u32 s, int w, S x, int lane) {
        if constexpr (!WIDE && MPC_LTZ_NARROW) return ltz_narrow(q, s, w, x, lane);
        const int m = w - 1;
        const bool k0 = k0ok();
        const PrgQ Q0 = prg_q(Kp->k0, q, s), Q1 = prg_q(Kp->k1, q, s);
        constexpr int H = WIDE ? 2 : 1;
        u32 Pp[2], Gp[2];                                  // this party's shares of P_j, G_j
        Pp[0] = transpose32((u32)x, lane);
        if (WIDE) Pp[1] = transpose32((u32)(x >> 32), lane);
        // g-layer: AND((x0_j, 0), (0, x1_j)) -- party 0 holds the x-input, party 1 the y-input
        {
            u32 ta[2], tb[2], tc[2], dd[2], ee[2];
#pragma unroll
            for (int h = 0; h < H; ++h) {
                const int j = lane + 32 * h;
                ta[h] = tb[h] = tc[h] = 0;
                if (j < m) {
                    const uint4 t0 = k0 ? prg(Q0, ltz_slot(0, j, 0)) : make_uint4(0, 0, 0, 0);
                    uint4 t1 = make_uint4(0, 0, 0, 0);
                    if (pty == 1) t1 = prg(Q1, ltz_slot(0, j, 0));
                    and_triple(t0, t1, 0, ta[h], tb[h], tc[h]);
                }
                const u32 xin = pty == 0 ? Pp[h] : 0u, yin = pty == 0 ? 0u : Pp[h];
                dd[h] = xin ^ ta[h]; ee[h] = yin ^ tb[h];
                put(lane, h, (u64)dd[h] | ((u64)ee[h] << 32));
            }
            exch(lane);
#pragma unroll
            for (int h = 0; h < H; ++h) {
                const u64 pw = get(lane, h);
                const u32 d = dd[h] ^ (u32)pw, e = ee[h] ^ (u32)(pw >> 32);
                Gp[h] = (lane + 32 * h < m) ? and_finish(ta[h], tb[h], tc[h], d, e) : 0u;
            }
        }
        const int L = (m > 0) ? ceil_log2i(m) : 0;
        for (int k = 0; k < L; ++k) {
            const int dl = 1 << k;
            const int src = (lane - dl) & 31;
            u32 sG[2], sP[2];
#pragma unroll
            for (int h = 0; h < H; ++h) { sG[h] = __shfl_sync(FULL, Gp[h], src); sP[h] = __shfl_sync(FULL, Pp[h], src); }
            u32 ga[2], gb[2], gc[2], pa[2], pb[2], pc[2], dG[2], eG[2], dP[2], eP[2];
            bool act[2];
#pragma unroll
            for (int h = 0; h < H; ++h) {
                const int j = lane + 32 * h;
                act[h] = (j >= dl && j < m);
                int hs = h;
                if (dl < 32) hs = (lane >= dl) ? h : h - 1; else hs = h - 1;
                u32 g = sG[0], p = sP[0];
                if (WIDE && hs == 1) { g = sG[1]; p = sP[1]; }
                if (WIDE && dl == 32) { g = Gp[0]; p = Pp[0]; }
                ga[h] = gb[h] = gc[h] = pa[h] = pb[h] = pc[h] = 0;
                if (act[h]) {
                    uint4 tg = make_uint4(0, 0, 0, 0), tp = tg;
                    if (k0) { tg = prg(Q0, ltz_slot(k + 1, j, 0)); tp = prg(Q0, ltz_slot(k + 1, j, 1)); }
                    uint4 t1 = make_uint4(0, 0, 0, 0);
                    if (pty == 1) t1 = prg(Q1, ltz_slot(k + 1, j, 0));
                    and_triple2(tg, tp, t1, ga[h], gb[h], gc[h], pa[h], pb[h], pc[h]);
                }
                dG[h] = Pp[h] ^ ga[h]; eG[h] = g ^ gb[h];
                dP[h] = Pp[h] ^ pa[h]; eP[h] = p ^ pb[h];
                put(lane, 2 * h, (u64)dG[h] | ((u64)eG[h] << 32));
                put(lane, 2 * h + 1, (u64)dP[h] | ((u64)eP[h] << 32));
            }
            exch(lane);
#pragma unroll
            for (int h = 0; h < H; ++h) {
                if (act[h]) {
                    const u64 w0 = get(lane, 2 * h), w1 = get(lane, 2 * h + 1);
                    const u32 d1 = dG[h] ^ (u32)w0, e1 = eG[h] ^ (u32)(w0 >> 32);
                    const u32 d2 = dP[h] ^ (u32)w1, e2 = eP[h] ^ (u32)(w1 >> 32);
                    Gp[h] ^= and_finish(ga[h], gb[h], gc[h], d1, e1);
                    Pp[h] = and_finish(pa[h], pb[h], pc[h], d2, e2);
                }
            }
        }
        u32 bp;
        if (m == 0) bp = (u32)(x & 1ull);
        else {
            const int jm = m - 1;
            u32 gm = Gp[0];
            if (WIDE && jm >= 32) gm = Gp[1];
            gm = __shfl_sync(FULL, gm, jm & 31);
            bp = (u32)((x >> (w - 1)) & 1ull) ^ ((gm >> lane) & 1u);
        }
        // daBit + B2A: party 0 holds (r0A, r0B); party 1 (r1A, r1B), r1A = (r0B ^ r1B) - r0A
        const uint4 D0 = k0 ? prg(Q0, 2u + (u32)lane) : make_uint4(0, 0, 0, 0);
        u64 rA;
        u32 rB;
        if (pty == 0) { rA = w64(D0.x, D0.y); rB = D0.z & 1u; }
        else {
            const uint4 D1 = prg(Q1, 1u);
            rB = (D1.x >> lane) & 1u;
            rA = dabit_r1A(D0, rB);
        }
        const u32 mine = bp ^ rB;
        put(lane, 0, (u64)mine);
        exch(lane);
        const u64 c = (u64)(mine ^ ((u32)get(lane, 0) & 1u));
        const u64 sg = 1ull - 2ull * c;
        return pty == 0 ? c + sg * rA : sg * rA;
    }

    template <int G, int NL>
    __device__ __forceinline__ void ltz_cone(u64 q0, u32 s, int w, const S (&x)[G], S (&z)[G], int lane, ConeSmem<G, NL>& sm) {
        ltz_cone_pair<G, NL, R>(*this, q0, s, w, x, z, lane, sm);
    }

    // ---- S2 open: exchange the shares themselves ----
    __device__ __forceinline__ u64 open(u64 x) {
        const int lane = threadIdx.x & 31;
        put(lane, 0, x);
        exch(lane);
        return x + get(lane, 0);
    }
    __device__ __forceinline__ S mask2(S x, u64 r0, u64 r1) const { return pty == 0 ? x - r0 : x - r1; }
    __device__ __forceinline__ void open2(S a, S b, u64& ea, u64& eb) {
        const int lane = threadIdx.x & 31;
        put(lane, 0, a); put(lane, 1, b);
        exch(lane);
        ea = a + get(lane, 0); eb = b + get(lane, 1);
    }
};

}  // namespace mpc
