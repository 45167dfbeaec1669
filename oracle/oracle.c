/*
 * oracle.c -- plain, slow, scalar CPU oracle for the 2-party nonlinear-operator
 * path of arxiv 2511.19711 (CrypTorch / CrypTen++).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  It shares no code,
 * header, table or constant generator with the CUDA path under
 * paper_2511_19711_b200/ and includes nothing from it.
 *
 * Citations: "P:n" = line n of /root/reference/PAPER.md, "S:n" = line n of
 * /root/reference/SPEC.md, "R<k>" = reading k in DESIGN.md section 3 (the
 * places where the paper is silent and we fixed a reading).
 *
 * Every operation simulates BOTH parties in lockstep on plain arrays
 * (x0[i], x1[i]) of uint64 ring elements of Z_2^64 (P:997-1000, P:1026:
 * "CrypTen uses s=2^16 and a 64-bit integer ring").  Steps of each schedule are
 * executed in the order DESIGN.md section 2 lists them, over the whole array,
 * one step at a time (no fusion, no blocking).
 *
 * Pinning: every function here is pinned by tests/test_oracle_*.py against
 * closed forms, brute force, the paper's printed values and invariants
 * (DESIGN.md section 4).  None is "parity unpinned".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

typedef uint64_t u64;
typedef int64_t i64;
typedef uint32_t u32;

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon et al., SC'11; the Random123 reference algorithm).   */
/* Reading R8: the paper's TTP dealer and SPEC's "own seed"  */
/* fix no generator; we fix Philox4x32-10 with counter (unit_lo, unit_hi,     */
/* step, slot) and a 64-bit key (lo32, hi32).                                 */
/* ------------------------------------------------------------------------ */
void orc_philox4x32_10(const u32 ctr_in[4], const u32 key_in[2], u32 out[4])
{
    u32 c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
    u32 k[2] = {key_in[0], key_in[1]};
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k[0] += 0x9E3779B9u; k[1] += 0xBB67AE85u; }
        u64 p0 = (u64)0xD2511F53u * (u64)c[0];
        u64 p1 = (u64)0xCD9E8D57u * (u64)c[2];
        u32 hi0 = (u32)(p0 >> 32), lo0 = (u32)p0;
        u32 hi1 = (u32)(p1 >> 32), lo1 = (u32)p1;
        u32 n0 = hi1 ^ c[1] ^ k[0];
        u32 n1 = lo1;
        u32 n2 = hi0 ^ c[3] ^ k[1];
        u32 n3 = lo0;
        c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
    }
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

/* PRG(key, unit, step, slot) -> 4 words. */
static void prg(u64 key, u64 unit, u64 step, u32 slot, u32 w[4])
{
    u32 ctr[4] = {(u32)unit, (u32)(unit >> 32), (u32)step, slot};
    u32 k[2] = {(u32)key, (u32)(key >> 32)};
    orc_philox4x32_10(ctr, k, w);
}
static u64 w64(u32 lo, u32 hi) { return (u64)lo | ((u64)hi << 32); }

typedef struct {
    u64 key_share, key_p0, key_p1;   /* K_s, K_0, K_1 */
    u64 step;                        /* next unused step id */
} orc_ctx;

/* ------------------------------------------------------------------------ */
/* Fixed-point encoding E(c) = round-half-even(c * 2^16)  ("round it  */
/* to the nearest integer"; reading R2: ties to even).                       */
/* ------------------------------------------------------------------------ */
#define FRAC 16
i64 orc_encode(double c) { return (i64)nearbyint(c * 65536.0); }

/* per-share arithmetic shift (local truncation; R3: floor) */
static u64 shr(u64 v, int k) { return (u64)(((i64)v) >> k); }

/* ------------------------------------------------------------------------ */
/* S1 share: owner's share = v - r, other = r, r from the pairwise key K_s   */
/* ("[x]_0 = x - r and [x]_1 = r").  One step per call.           */
/* ------------------------------------------------------------------------ */
void orc_share(orc_ctx* ctx, const double* x, int owner, u64* s0, u64* s1, i64 n, i64 off)
{
    u64 s = ctx->step++;
    for (i64 i = 0; i < n; ++i) {
        u32 w[4];
        prg(ctx->key_share, (u64)(off + i), s, 0, w);
        u64 r = w64(w[0], w[1]);
        u64 v = (u64)orc_encode(x[i]);
        if (owner == 0) { s0[i] = v - r; s1[i] = r; }
        else            { s0[i] = r;     s1[i] = v - r; }
    }
}

/* S2 open: rec = x0 + x1 mod 2^64; decode (int64)rec / 2^scale_bits */
void orc_open(const u64* s0, const u64* s1, i64 n, u64* ring, double* f, int scale_bits)
{
    for (i64 i = 0; i < n; ++i) {
        u64 v = s0[i] + s1[i];
        if (ring) ring[i] = v;
        if (f) f[i] = (double)(i64)v / (double)((u64)1 << scale_bits);
    }
}

/* ------------------------------------------------------------------------ */
/* S3 + S4: Beaver multiplication with a trusted-dealer triple (P:1009-1011,  */
/* S:432-440).  Triple layout:                               */
/*   (a0,b0) = PRG(K0, u, s, 0) ;  (a1,b1) = PRG(K1, u, s, 0)                 */
/*   c0      = half (u&1) of PRG(K0, u>>1, s, 1) ; c1 = (a0+a1)(b0+b1) - c0  */
/* e = open(x - a), f = open(y - b);                                          */
/* z0 = c0 + e*b0 + f*a0 + e*f  (party 0 adds e*f, R6) ; z1 = c1 + e*b1 + f*a1 */
/* ------------------------------------------------------------------------ */
static void beaver_triple(const orc_ctx* ctx, u64 s, u64 u,
                          u64* a0, u64* b0, u64* c0, u64* a1, u64* b1, u64* c1)
{
    u32 w[4];
    prg(ctx->key_p0, u, s, 0, w); *a0 = w64(w[0], w[1]); *b0 = w64(w[2], w[3]);
    prg(ctx->key_p1, u, s, 0, w); *a1 = w64(w[0], w[1]); *b1 = w64(w[2], w[3]);
    prg(ctx->key_p0, u >> 1, s, 1, w);
    *c0 = (u & 1) ? w64(w[2], w[3]) : w64(w[0], w[1]);
    *c1 = (*a0 + *a1) * (*b0 + *b1) - *c0;   /* dealer correction to party 1 (R7) */
}

/* BM over an array; element i uses unit units0 + i.  One step. */
static void BM(orc_ctx* ctx, i64 n, u64 units0,
               const u64* x0, const u64* x1, const u64* y0, const u64* y1, u64* z0, u64* z1)
{
    u64 s = ctx->step++;
    for (i64 i = 0; i < n; ++i) {
        u64 a0, b0, c0, a1, b1, c1;
        beaver_triple(ctx, s, units0 + (u64)i, &a0, &b0, &c0, &a1, &b1, &c1);
        /* each party masks its own shares; the opening is the sum (one round) */
        u64 e = (x0[i] - a0) + (x1[i] - a1);
        u64 f = (y0[i] - b0) + (y1[i] - b1);
        u64 r0 = c0 + e * b0 + f * a0 + e * f;
        u64 r1 = c1 + e * b1 + f * a1;
        z0[i] = r0; z1[i] = r1;
    }
}

/* MT(x,y) = trunc(BM(x,y), 16): Sec-Sec Mul rule ("mul_MPC then trunc by s_min") */
static void MT(orc_ctx* ctx, i64 n, u64 units0,
               const u64* x0, const u64* x1, const u64* y0, const u64* y1, u64* z0, u64* z1)
{
    BM(ctx, n, units0, x0, x1, y0, y1, z0, z1);
    for (i64 i = 0; i < n; ++i) { z0[i] = shr(z0[i], FRAC); z1[i] = shr(z1[i], FRAC); }
}

/* ------------------------------------------------------------------------ */
/* Square with a square-pair triple (a, c = a^2) -- SURVEY 8(f) NEXT #2; the     */
/* way CrypTen squares (its exp loop calls square(), P:653 default t=8).       */
/* Layout: (a0, c0) = PRG(K0, u, s, 2) ; a1 = half (u&1) of     */
/* PRG(K1, u>>1, s, 3) ; c1 = (a0+a1)^2 - c0.  e = open(y - a) (one word);      */
/* z0 = c0 + 2 e a0 + e^2 ; z1 = c1 + 2 e a1.                                   */
/* ------------------------------------------------------------------------ */
static void SQ(orc_ctx* ctx, i64 n, u64 units0, const u64* y0, const u64* y1, u64* z0, u64* z1)
{
    u64 s = ctx->step++;
    for (i64 i = 0; i < n; ++i) {
        u64 u = units0 + (u64)i;
        u32 w[4];
        prg(ctx->key_p0, u, s, 2, w);
        u64 a0 = w64(w[0], w[1]), c0 = w64(w[2], w[3]);
        prg(ctx->key_p1, u >> 1, s, 3, w);
        u64 a1 = (u & 1) ? w64(w[2], w[3]) : w64(w[0], w[1]);
        u64 a = a0 + a1;
        u64 c1 = a * a - c0;                        /* dealer correction -> party 1 */
        u64 e = (y0[i] - a0) + (y1[i] - a1);        /* opened */
        u64 r0 = c0 + 2 * e * a0 + e * e;
        u64 r1 = c1 + 2 * e * a1;
        z0[i] = r0; z1[i] = r1;
    }
}

static void MS(orc_ctx* ctx, i64 n, u64 units0, const u64* y0, const u64* y1, u64* z0, u64* z1)
{
    SQ(ctx, n, units0, y0, y1, z0, z1);
    for (i64 i = 0; i < n; ++i) { z0[i] = shr(z0[i], FRAC); z1[i] = shr(z1[i], FRAC); }
}

void orc_square(orc_ctx* ctx, const u64* x0, const u64* x1, u64* z0, u64* z1, i64 n, i64 off, int trunc_bits)
{
    SQ(ctx, n, (u64)off, x0, x1, z0, z1);
    if (trunc_bits)
        for (i64 i = 0; i < n; ++i) { z0[i] = shr(z0[i], trunc_bits); z1[i] = shr(z1[i], trunc_bits); }
}

void orc_mul(orc_ctx* ctx, const u64* x0, const u64* x1, const u64* y0, const u64* y1,
             u64* z0, u64* z1, i64 n, i64 off, int trunc_bits)
{
    BM(ctx, n, (u64)off, x0, x1, y0, y1, z0, z1);
    if (trunc_bits)
        for (i64 i = 0; i < n; ++i) { z0[i] = shr(z0[i], trunc_bits); z1[i] = shr(z1[i], trunc_bits); }
}

/* ------------------------------------------------------------------------ */
/* Broadcast-triple product z_i = x_i * y_{row(i)} (SURVEY 8(f) NEXT #2 "a     */
/* broadcast triple for softmax's e*r"; the expanded product of S:435 opens    */
/* y once per ELEMENT, this one once per ROW).  Layout:        */
/*   (a0, c0) = PRG(K0, u, s, 4) ; a1 = half (u&1) of PRG(K1, u>>1, s, 5)      */
/*   b0 = PRG(K0, r, s, 6)[0..1] ; b1 = PRG(K1, r, s, 6)[0..1]                 */
/*   c1 = (a0+a1)(b0+b1) - c0            (dealer correction -> party 1, R7)    */
/* e_i = open(x_i - a_i) per element, f_r = open(y_r - b_r) per row;           */
/* z0 = c0 + e b0 + f a0 + e f (party 0 adds e f, R6) ; z1 = c1 + e b1 + f a1. */
/* u = element unit (units0 + i), r = row unit (row0 + row).  One step.        */
/* ------------------------------------------------------------------------ */
static void BMB(orc_ctx* ctx, i64 rows, i64 cols, u64 units0, u64 row0,
                const u64* x0, const u64* x1, const u64* y0, const u64* y1, u64* z0, u64* z1)
{
    u64 s = ctx->step++;
    for (i64 r = 0; r < rows; ++r) {
        u32 w[4];
        prg(ctx->key_p0, row0 + (u64)r, s, 6, w);
        u64 b0 = w64(w[0], w[1]);
        prg(ctx->key_p1, row0 + (u64)r, s, 6, w);
        u64 b1 = w64(w[0], w[1]);
        u64 f = (y0[r] - b0) + (y1[r] - b1);             /* opened once per row */
        for (i64 j = 0; j < cols; ++j) {
            i64 i = r * cols + j;
            u64 u = units0 + (u64)i;
            prg(ctx->key_p0, u, s, 4, w);
            u64 a0 = w64(w[0], w[1]), c0 = w64(w[2], w[3]);
            prg(ctx->key_p1, u >> 1, s, 5, w);
            u64 a1 = (u & 1) ? w64(w[2], w[3]) : w64(w[0], w[1]);
            u64 c1 = (a0 + a1) * (b0 + b1) - c0;
            u64 e = (x0[i] - a0) + (x1[i] - a1);         /* opened per element */
            z0[i] = c0 + e * b0 + f * a0 + e * f;
            z1[i] = c1 + e * b1 + f * a1;
        }
    }
}

void orc_mul_bcast(orc_ctx* ctx, const u64* x0, const u64* x1, const u64* y0, const u64* y1,
                   u64* z0, u64* z1, i64 rows, i64 cols, i64 off, i64 row_off, int trunc_bits)
{
    BMB(ctx, rows, cols, (u64)off, (u64)row_off, x0, x1, y0, y1, z0, z1);
    if (trunc_bits)
        for (i64 i = 0; i < rows * cols; ++i) { z0[i] = shr(z0[i], trunc_bits); z1[i] = shr(z1[i], trunc_bits); }
}

/* S5 local truncation: z_i = (int64)x_i >> k at each party */
void orc_trunc(const u64* x0, const u64* x1, u64* z0, u64* z1, i64 n, int bits)
{
    for (i64 i = 0; i < n; ++i) { z0[i] = shr(x0[i], bits); z1[i] = shr(x1[i], bits); }
}

/* ------------------------------------------------------------------------ */
/* S7 LTZ: GMW sign bit realised as A2B + Kogge-Stone carry    */
/* circuit + daBit B2A (readings R9, R10, R11, R12).        */
/*                                                                           */
/* Per element, with m = w-1 carry positions and L = ceil(log2 m) levels:     */
/*   p_j = x0_j ^ x1_j   (XOR-shared as (x0_j, x1_j), local)                  */
/*   g_j = x0_j & x1_j   (AND gate on ((x0_j,0),(0,x1_j)))                    */
/*   level k, d = 2^k, j in [d, m):  G_j ^= P_j & G_{j-d};  P_j &= P_{j-d}     */
/*   b = p_{w-1} ^ G_{m-1}            (b = p_0 when w == 1)                    */
/* The triple WORDS of each gate are defined per 32-element group q (bit l of */
/* a word belongs to element 32q+l); the oracle reads the element's bit.      */
/* Gate triple layout:                                        */
/*   SLOT(lv, j, c) = 64 + 128*lv + 2*j + c                                   */
/*   g-layer plane j:   (a0,b0,c0)=PRG(K0,q,s,SLOT(0,j,0))[0..2],             */
/*                      (a1,b1)   =PRG(K1,q,s,SLOT(0,j,0))[0..1]              */
/*   level k plane j:   G-gate (a0,b0,c0)=PRG(K0,q,s,SLOT(k+1,j,0))[0..2]     */
/*                      P-gate (a0,b0,c0)=PRG(K0,q,s,SLOT(k+1,j,1))[0..2]     */
/*                      T1 = PRG(K1,q,s,SLOT(k+1,j,0)):                       */
/*                        G-gate (a1,b1)=T1[0..1], P-gate (a1,b1)=T1[2..3]     */
/*   c1 = ((a0^a1)&(b0^b1))^c0  (dealer correction to party 1)                */
/* daBit of element l:  D0=PRG(K0,q,s,2+l): r0A=w64(D0[0],D0[1]), r0B=D0[2]&1 */
/*                      r1B = bit l of PRG(K1,q,s,1)[0] ; r=r0B^r1B ; r1A=r-r0A */
/* B2A: c = open(b ^ r); z0 = c + (1-2c) r0A ; z1 = (1-2c) r1A                 */
/* ------------------------------------------------------------------------ */
#define SLOT(lv, j, c) (64u + 128u * (u32)(lv) + 2u * (u32)(j) + (u32)(c))

typedef struct { u32 a0, b0, c0, a1, b1, c1; } btriple;

static btriple and_triple_words(const u32 t0[4], u32 a1, u32 b1)
{
    btriple t;
    t.a0 = t0[0]; t.b0 = t0[1]; t.c0 = t0[2];
    t.a1 = a1; t.b1 = b1;
    t.c1 = ((t.a0 ^ t.a1) & (t.b0 ^ t.b1)) ^ t.c0;
    return t;
}

/* AND of XOR-shared bits (x0^x1)&(y0^y1) with a bit-triple (one round).      */
static void and_gate(int x0, int x1, int y0, int y1, const btriple* t, int l, int* z0, int* z1)
{
    int a0 = (t->a0 >> l) & 1, b0 = (t->b0 >> l) & 1, c0 = (t->c0 >> l) & 1;
    int a1 = (t->a1 >> l) & 1, b1 = (t->b1 >> l) & 1, c1 = (t->c1 >> l) & 1;
    int d = (x0 ^ a0) ^ (x1 ^ a1);     /* opened */
    int e = (y0 ^ b0) ^ (y1 ^ b1);     /* opened */
    *z0 = c0 ^ (d & b0) ^ (e & a0) ^ (d & e);
    *z1 = c1 ^ (d & b1) ^ (e & a1);
}

static int ceil_log2(int m) { int L = 0; while ((1 << L) < m) ++L; return L; }

/* Number of AND gates of the full Kogge-Stone LTZ at window w (R9). */
int orc_ltz_gate_count(int w)
{
    int m = w - 1;
    if (m <= 0) return 0;
    int L = ceil_log2(m), g = m;
    for (int k = 0; k < L; ++k) g += 2 * (m - (1 << k));
    return g;
}

/* the group's triples, generated once per (q, s) and then read bit by bit  */
typedef struct {
    btriple g[64];          /* g-layer, plane j */
    btriple G[7][64];       /* level k, plane j: G-gate */
    btriple P[7][64];       /* level k, plane j: P-gate */
} ltz_group_triples;

static void gen_group_triples(const orc_ctx* ctx, u64 s, u64 q, int w, ltz_group_triples* T)
{
    int m = w - 1, L = (m > 0) ? ceil_log2(m) : 0;
    u32 t0[4], t0p[4], t1[4];
    for (int j = 0; j < m; ++j) {
        prg(ctx->key_p0, q, s, SLOT(0, j, 0), t0);
        prg(ctx->key_p1, q, s, SLOT(0, j, 0), t1);
        T->g[j] = and_triple_words(t0, t1[0], t1[1]);
    }
    for (int k = 0; k < L; ++k)
        for (int j = (1 << k); j < m; ++j) {
            prg(ctx->key_p0, q, s, SLOT(k + 1, j, 0), t0);
            prg(ctx->key_p0, q, s, SLOT(k + 1, j, 1), t0p);
            prg(ctx->key_p1, q, s, SLOT(k + 1, j, 0), t1);
            T->G[k][j] = and_triple_words(t0, t1[0], t1[1]);
            T->P[k][j] = and_triple_words(t0p, t1[2], t1[3]);
        }
}

/* LTZ over an array whose element i has unit units0 + i.  One step.         */
/* Output: arithmetic shares of b = bit (w-1) of rec(x), at scale 1.          */
static void LTZ(orc_ctx* ctx, i64 n, u64 units0, int w,
                const u64* x0, const u64* x1, u64* z0, u64* z1)
{
    u64 s = ctx->step++;
    int m = w - 1, L = (m > 0) ? ceil_log2(m) : 0;
    ltz_group_triples* T = (ltz_group_triples*)malloc(sizeof(ltz_group_triples));
    u64 cur_q = ~(u64)0;
    u32 r1b_word = 0;
    for (i64 i = 0; i < n; ++i) {
        u64 u = units0 + (u64)i, q = u >> 5;
        int l = (int)(u & 31);
        if (q != cur_q) {
            gen_group_triples(ctx, s, q, w, T);
            u32 d1[4];
            prg(ctx->key_p1, q, s, 1, d1);
            r1b_word = d1[0];
            cur_q = q;
        }
        /* A2B: each party bit-decomposes its own share (local) */
        int X0[64], X1[64];
        for (int j = 0; j < w; ++j) { X0[j] = (int)((x0[i] >> j) & 1); X1[j] = (int)((x1[i] >> j) & 1); }
        int G0[64], G1[64], P0[64], P1[64];
        for (int j = 0; j < m; ++j) {
            P0[j] = X0[j]; P1[j] = X1[j];                            /* p_j shares */
            and_gate(X0[j], 0, 0, X1[j], &T->g[j], l, &G0[j], &G1[j]); /* g_j = x0_j & x1_j */
        }
        for (int k = 0; k < L; ++k) {
            int d = 1 << k;
            int nG0[64], nG1[64], nP0[64], nP1[64];
            for (int j = 0; j < m; ++j) { nG0[j] = G0[j]; nG1[j] = G1[j]; nP0[j] = P0[j]; nP1[j] = P1[j]; }
            for (int j = d; j < m; ++j) {     /* G-updates */
                int t0, t1;
                and_gate(P0[j], P1[j], G0[j - d], G1[j - d], &T->G[k][j], l, &t0, &t1);
                nG0[j] = G0[j] ^ t0; nG1[j] = G1[j] ^ t1;
            }
            for (int j = d; j < m; ++j)       /* P-updates */
                and_gate(P0[j], P1[j], P0[j - d], P1[j - d], &T->P[k][j], l, &nP0[j], &nP1[j]);
            memcpy(G0, nG0, sizeof G0); memcpy(G1, nG1, sizeof G1);
            memcpy(P0, nP0, sizeof P0); memcpy(P1, nP1, sizeof P1);
        }
        int b0, b1;
        if (m == 0) { b0 = X0[0]; b1 = X1[0]; }
        else        { b0 = X0[w - 1] ^ G0[m - 1]; b1 = X1[w - 1] ^ G1[m - 1]; }
        /* daBit + B2A */
        u32 d0[4];
        prg(ctx->key_p0, q, s, 2u + (u32)l, d0);
        u64 r0A = w64(d0[0], d0[1]);
        int r0B = (int)(d0[2] & 1u);
        int r1B = (int)((r1b_word >> l) & 1u);
        u64 r = (u64)(r0B ^ r1B);
        u64 r1A = r - r0A;
        u64 c = (u64)((b0 ^ r0B) ^ (b1 ^ r1B));     /* opened bit */
        u64 sgn = (u64)1 - 2 * c;                    /* 1 - 2c mod 2^64 */
        z0[i] = c + sgn * r0A;
        z1[i] = sgn * r1A;
    }
    free(T);
}

void orc_ltz(orc_ctx* ctx, const u64* x0, const u64* x1, u64* z0, u64* z1, i64 n, i64 off, int w)
{
    LTZ(ctx, n, (u64)off, w, x0, x1, z0, z1);
}

/* ------------------------------------------------------------------------ */
/* Local public operations (rules P:398-483)          */
/* ------------------------------------------------------------------------ */
static void addP(u64* x0, i64 n, double c) { u64 e = (u64)orc_encode(c); for (i64 i = 0; i < n; ++i) x0[i] += e; }
static void notmask(u64* b0, u64* b1, i64 n) { for (i64 i = 0; i < n; ++i) { b0[i] = 1 - b0[i]; b1[i] = (u64)0 - b1[i]; } }
static void pmulF(u64* x0, u64* x1, i64 n, double c)
{
    u64 e = (u64)orc_encode(c);
    for (i64 i = 0; i < n; ++i) { x0[i] = shr(x0[i] * e, FRAC); x1[i] = shr(x1[i] * e, FRAC); }
}

/* per-share floor division by a public positive integer (reading R25) */
static i64 floordiv(i64 a, i64 d) { i64 q = a / d; if ((a % d) != 0 && (a < 0)) --q; return q; }
static void divP(u64* x0, u64* x1, i64 n, i64 d)
{
    for (i64 i = 0; i < n; ++i) { x0[i] = (u64)floordiv((i64)x0[i], d); x1[i] = (u64)floordiv((i64)x1[i], d); }
}

static u64* A(i64 n) { return (u64*)malloc(sizeof(u64) * (size_t)(n > 0 ? n : 1)); }

/* S8 ReLU = BM(x, NOT(LTZ(x)))  ("x x (x >= 0)"; no truncation: */
/* the mask has scale 1, s_min = 1, R5).  2 steps.                            */
void orc_relu(orc_ctx* ctx, const u64* x0, const u64* x1, u64* z0, u64* z1, i64 n, i64 off, int w)
{
    u64 *l0 = A(n), *l1 = A(n);
    LTZ(ctx, n, (u64)off, w, x0, x1, l0, l1);
    notmask(l0, l1, n);
    BM(ctx, n, (u64)off, x0, x1, l0, l1, z0, z1);
    free(l0); free(l1);
}

/* ------------------------------------------------------------------------ */
/* S10 EXP(x; t, clamp, w): (1 + x/2^t)^(2^t) (Fig. pass_lang)*/
/*   y = addP(shr(x,t), 1.0)            x/2^t as a shift (R4)                 */
/*   clamp: y = BM(y, NOT(LTZ_w(addP(x, 2^t))))     mask [x >= -2^t] (R13)     */
/*   t times: y = MT(y, y)                                                    */
/* Steps: t + 2*clamp.                                                        */
/* ------------------------------------------------------------------------ */
static void EXP(orc_ctx* ctx, i64 n, u64 units0, int t, int clamp, int w, int sq,
                const u64* x0, const u64* x1, u64* y0, u64* y1)
{
    u64 e1 = (u64)orc_encode(1.0);
    u64 *c0 = A(n), *c1 = A(n);                       /* x + 2^t, taken before y may alias x */
    memcpy(c0, x0, sizeof(u64) * (size_t)n); memcpy(c1, x1, sizeof(u64) * (size_t)n);
    addP(c0, n, ldexp(1.0, t));
    for (i64 i = 0; i < n; ++i) { y0[i] = shr(x0[i], t) + e1; y1[i] = shr(x1[i], t); }
    if (clamp) {
        u64 *l0 = A(n), *l1 = A(n);
        LTZ(ctx, n, units0, w, c0, c1, l0, l1);
        notmask(l0, l1, n);
        BM(ctx, n, units0, y0, y1, l0, l1, y0, y1);
        free(l0); free(l1);
    }
    free(c0); free(c1);
    for (int k = 0; k < t; ++k) {
        if (sq) MS(ctx, n, units0, y0, y1, y0, y1);          /* square-pair triple (NEXT #2) */
        else MT(ctx, n, units0, y0, y1, y0, y1, y0, y1);
    }
}

void orc_exp(orc_ctx* ctx, const u64* x0, const u64* x1, u64* z0, u64* z1, i64 n, i64 off,
             int t, int clamp, int w, int sq)
{
    EXP(ctx, n, (u64)off, t, clamp, w, sq, x0, x1, z0, z1);
}

/* S11 RECIP: Newton-Raphson y <- y(2 - x y) from y0 = 3 exp(0.5 - x) + 0.003  */
/* ("Newton-Raphson method"; S:208-216, S:240 initialisation).          */
static void RECIP(orc_ctx* ctx, i64 n, u64 units0, int iters, int t, int clamp, int w, int sq,
                  const u64* x0, const u64* x1, u64* y0, u64* y1)
{
    u64 *g0 = A(n), *g1 = A(n), *p0 = A(n), *p1 = A(n);
    for (i64 i = 0; i < n; ++i) { g0[i] = (u64)0 - x0[i]; g1[i] = (u64)0 - x1[i]; }
    addP(g0, n, 0.5);
    EXP(ctx, n, units0, t, clamp, w, sq, g0, g1, g0, g1);
    for (i64 i = 0; i < n; ++i) { y0[i] = g0[i] * 3; y1[i] = g1[i] * 3; }   /* pmulI(g,3) */
    addP(y0, n, 0.003);
    for (int it = 0; it < iters; ++it) {
        MT(ctx, n, units0, x0, x1, y0, y1, p0, p1);                             /* p = x*y */
        for (i64 i = 0; i < n; ++i) { p0[i] = (u64)0 - p0[i]; p1[i] = (u64)0 - p1[i]; }
        addP(p0, n, 2.0);                                                       /* 2 - p */
        MT(ctx, n, units0, y0, y1, p0, p1, y0, y1);                             /* y*(2-p) */
    }
    free(g0); free(g1); free(p0); free(p1);
}

void orc_recip(orc_ctx* ctx, const u64* x0, const u64* x1, u64* z0, u64* z1, i64 n, i64 off,
               int iters, int t, int clamp, int w, int sq)
{
    RECIP(ctx, n, (u64)off, iters, t, clamp, w, sq, x0, x1, z0, z1);
}

/* S12 RSQRT: y <- y (3 - x y^2) / 2 from y0 = 2.2 exp(-(x/2 + 0.2)) + 0.2     */
/* ("uses e^x in its approximation of inverse sqrt").  */
static void RSQRT(orc_ctx* ctx, i64 n, u64 units0, int iters, int t, int clamp, int w, int sq,
                  const u64* x0, const u64* x1, u64* y0, u64* y1)
{
    u64 *g0 = A(n), *g1 = A(n), *q0 = A(n), *q1 = A(n), *p0 = A(n), *p1 = A(n);
    for (i64 i = 0; i < n; ++i) { g0[i] = shr(x0[i], 1); g1[i] = shr(x1[i], 1); }
    addP(g0, n, 0.2);
    for (i64 i = 0; i < n; ++i) { g0[i] = (u64)0 - g0[i]; g1[i] = (u64)0 - g1[i]; }
    EXP(ctx, n, units0, t, clamp, w, sq, g0, g1, g0, g1);
    memcpy(y0, g0, sizeof(u64) * (size_t)n); memcpy(y1, g1, sizeof(u64) * (size_t)n);
    pmulF(y0, y1, n, 2.2);
    addP(y0, n, 0.2);
    for (int it = 0; it < iters; ++it) {
        MT(ctx, n, units0, y0, y1, y0, y1, q0, q1);                 /* q = y*y  */
        MT(ctx, n, units0, x0, x1, q0, q1, p0, p1);                 /* p = x*q  */
        for (i64 i = 0; i < n; ++i) { p0[i] = (u64)0 - p0[i]; p1[i] = (u64)0 - p1[i]; }
        addP(p0, n, 3.0);                                            /* 3 - p    */
        MT(ctx, n, units0, y0, y1, p0, p1, y0, y1);                 /* u = y*(3-p) */
        pmulF(y0, y1, n, 0.5);                                       /* y = u*0.5 */
    }
    free(g0); free(g1); free(q0); free(q1); free(p0); free(p1);
}

void orc_rsqrt(orc_ctx* ctx, const u64* x0, const u64* x1, u64* z0, u64* z1, i64 n, i64 off,
               int iters, int t, int clamp, int w, int sq)
{
    RSQRT(ctx, n, (u64)off, iters, t, clamp, w, sq, x0, x1, z0, z1);
}

/* ------------------------------------------------------------------------ */
/* S13 segment polynomials ("order-4 polynomial from BOLT ...   */
/* order-2 polynomial and ReLU").                                   */
/* HORNER(v; c_0..c_d), d >= 1:  h = addP(pmulF(v, c_d), c_{d-1});            */
/*   for k = d-2..0: h = addP(MT(h, v), c_k).   d-1 steps.                      */
/* ------------------------------------------------------------------------ */
static void HORNER(orc_ctx* ctx, i64 n, u64 units0, const u64* v0, const u64* v1,
                   const double* c, int d, u64* h0, u64* h1)
{
    memcpy(h0, v0, sizeof(u64) * (size_t)n); memcpy(h1, v1, sizeof(u64) * (size_t)n);
    pmulF(h0, h1, n, c[d]);
    addP(h0, n, c[d - 1]);
    for (int k = d - 2; k >= 0; --k) {
        MT(ctx, n, units0, h0, h1, v0, v1, h0, h1);
        addP(h0, n, c[k]);
    }
}

/* POWER(v; c_0..c_d), 1 <= d <= 4 (SURVEY 8(f) NEXT #2 "power-basis polynomials   */
/* (2 rounds instead of 3)"):  v2 = MT(v,v); v3 = MT(v2,v); v4 = MT(v2,v2) (steps   */
/* in this order; v3 and v4 need only v2, so they share one round);                */
/* h = addP(sum_{k=1..d} pmulF(v^k, c_k), c_0).  d-1 steps, like HORNER.            */
static void POWER(orc_ctx* ctx, i64 n, u64 units0, const u64* v0, const u64* v1,
                  const double* c, int d, u64* h0, u64* h1)
{
    u64 *p0[5] = {0}, *p1[5] = {0};
    u64 *t0 = A(n), *t1 = A(n);
    p0[1] = (u64*)v0; p1[1] = (u64*)v1;
    for (int k = 2; k <= d; ++k) { p0[k] = A(n); p1[k] = A(n); }
    if (d >= 2) MT(ctx, n, units0, v0, v1, v0, v1, p0[2], p1[2]);
    if (d >= 3) MT(ctx, n, units0, p0[2], p1[2], v0, v1, p0[3], p1[3]);
    if (d >= 4) MT(ctx, n, units0, p0[2], p1[2], p0[2], p1[2], p0[4], p1[4]);
    memset(h0, 0, sizeof(u64) * (size_t)n); memset(h1, 0, sizeof(u64) * (size_t)n);
    for (int k = 1; k <= d; ++k) {
        memcpy(t0, p0[k], sizeof(u64) * (size_t)n); memcpy(t1, p1[k], sizeof(u64) * (size_t)n);
        pmulF(t0, t1, n, c[k]);
        for (i64 i = 0; i < n; ++i) { h0[i] += t0[i]; h1[i] += t1[i]; }
    }
    addP(h0, n, c[0]);
    for (int k = 2; k <= d; ++k) { free(p0[k]); free(p1[k]); }
    free(t0); free(t1);
}

enum { ACT_GELU = 0, ACT_SILU = 1, ACT_SIGMOID = 2 };
enum { FORM_POLY_X = 0, FORM_POLY_ABS = 1, FORM_RELU = 2, FORM_ERF = 3 };

/* segment masks + final masked sum shared by the x-, |x|- and erf- forms:   */
/*   l1 = LTZ(x + B), l2 = LTZ(x - B)   (two steps, listed order)              */
/*   out = BM(inner, l2 - l1) + tail,  tail = BM(x, NOT(l2)) (GELU/SiLU) or    */
/*                                     pmulI(NOT(l2), 2^16) (Sigmoid, local)   */
/* basis: 0 HORNER, 1 POWER (x- and |x|-forms, degree <= 4) */
void orc_act(orc_ctx* ctx, const u64* x0, const u64* x1, u64* z0, u64* z1, i64 n, i64 off,
             int act, int form, int degree, double B, const double* coeffs, int erf_terms, int w, int basis)
{
    u64 U = (u64)off;
    u64 *l0 = A(n), *l1 = A(n), *m0 = A(n), *m1 = A(n), *h0 = A(n), *h1 = A(n), *t0 = A(n), *t1 = A(n);
    if (form == FORM_RELU || degree == 0) {
        /* degree 0: ReLU for GELU/SiLU, unit step 1 - ltz(x) for Sigmoid */
        LTZ(ctx, n, U, w, x0, x1, l0, l1);
        notmask(l0, l1, n);
        if (act == ACT_SIGMOID) {
            for (i64 i = 0; i < n; ++i) { z0[i] = l0[i] << FRAC; z1[i] = l1[i] << FRAC; }
        } else {
            BM(ctx, n, U, x0, x1, l0, l1, z0, z1);
        }
        goto done;
    }
    {
        u64 *s0 = NULL, *s1 = NULL;
        if (form == FORM_POLY_ABS) {                     /* s = ltz(x) first */
            s0 = A(n); s1 = A(n);
            LTZ(ctx, n, U, w, x0, x1, s0, s1);
        }
        memcpy(t0, x0, sizeof(u64) * (size_t)n); memcpy(t1, x1, sizeof(u64) * (size_t)n);
        addP(t0, n, B);
        LTZ(ctx, n, U, w, t0, t1, l0, l1);               /* l1 = [x < -B] */
        memcpy(t0, x0, sizeof(u64) * (size_t)n); memcpy(t1, x1, sizeof(u64) * (size_t)n);
        addP(t0, n, -B);
        LTZ(ctx, n, U, w, t0, t1, m0, m1);               /* l2 = [x < B]  */
        if (form == FORM_POLY_X) {
            if (basis) POWER(ctx, n, U, x0, x1, coeffs, degree, h0, h1);
            else HORNER(ctx, n, U, x0, x1, coeffs, degree, h0, h1);
        } else if (form == FORM_POLY_ABS) {
            /* |x| = BM(x, 1 - 2s) ; h = 0.5 x + P(|x|) (BOLT structure) */
            u64 *sg0 = A(n), *sg1 = A(n), *ax0 = A(n), *ax1 = A(n);
            for (i64 i = 0; i < n; ++i) { sg0[i] = 1 - 2 * s0[i]; sg1[i] = (u64)0 - 2 * s1[i]; }
            BM(ctx, n, U, x0, x1, sg0, sg1, ax0, ax1);
            if (basis) POWER(ctx, n, U, ax0, ax1, coeffs, degree, h0, h1);
            else HORNER(ctx, n, U, ax0, ax1, coeffs, degree, h0, h1);
            memcpy(t0, x0, sizeof(u64) * (size_t)n); memcpy(t1, x1, sizeof(u64) * (size_t)n);
            pmulF(t0, t1, n, 0.5);
            for (i64 i = 0; i < n; ++i) { h0[i] += t0[i]; h1[i] += t1[i]; }
            free(sg0); free(sg1); free(ax0); free(ax1);
        } else { /* FORM_ERF: GELU(x) = 0.5 x (1 + erf(x/sqrt2)), Maclaurin erf (R21) */
            int K = erf_terms;
            double* a = (double*)malloc(sizeof(double) * (size_t)K);
            double fact = 1.0;
            for (int k = 0; k < K; ++k) {
                if (k > 0) fact *= (double)k;
                a[k] = ((k & 1) ? -1.0 : 1.0) / (fact * (double)(2 * k + 1));
            }
            u64 *zz0 = A(n), *zz1 = A(n), *z20 = A(n), *z21 = A(n), *S0 = A(n), *S1 = A(n);
            memcpy(zz0, x0, sizeof(u64) * (size_t)n); memcpy(zz1, x1, sizeof(u64) * (size_t)n);
            pmulF(zz0, zz1, n, 1.0 / sqrt(2.0));                     /* z = x / sqrt 2 */
            MT(ctx, n, U, zz0, zz1, zz0, zz1, z20, z21);             /* z^2 */
            HORNER(ctx, n, U, z20, z21, a, K - 1, S0, S1);           /* sum a_k z^(2k) */
            MT(ctx, n, U, zz0, zz1, S0, S1, t0, t1);                 /* z * S */
            pmulF(t0, t1, n, 2.0 / sqrt(M_PI));                      /* erf */
            addP(t0, n, 1.0);                                        /* 1 + erf */
            MT(ctx, n, U, x0, x1, t0, t1, h0, h1);                   /* x (1 + erf) */
            pmulF(h0, h1, n, 0.5);
            free(a); free(zz0); free(zz1); free(z20); free(z21); free(S0); free(S1);
        }
        /* segment mask (l2 - l1) and masked sum */
        for (i64 i = 0; i < n; ++i) { t0[i] = m0[i] - l0[i]; t1[i] = m1[i] - l1[i]; }
        BM(ctx, n, U, h0, h1, t0, t1, z0, z1);
        notmask(m0, m1, n);
        if (act == ACT_SIGMOID) {
            for (i64 i = 0; i < n; ++i) { z0[i] += m0[i] << FRAC; z1[i] += m1[i] << FRAC; }
        } else {
            BM(ctx, n, U, x0, x1, m0, m1, t0, t1);
            for (i64 i = 0; i < n; ++i) { z0[i] += t0[i]; z1[i] += t1[i]; }
        }
        if (s0) { free(s0); free(s1); }
    }
done:
    free(l0); free(l1); free(m0); free(m1); free(h0); free(h1); free(t0); free(t1);
}

/* ------------------------------------------------------------------------ */
/* S9 MAX_row: half-split tree (R22) with mux y + c (x - y) ("one       */
/* (y + c x (x - y))").  Level with m live entries: h = m/2;       */
/*   d_i = x_i - x_{i+h};  c_i = NOT(LTZ(d_i));  x_i' = x_{i+h} + BM(d_i, c_i) */
/*   units row*h + i (global row); odd m: last entry carried to position h.   */
/* Each level: 2 steps, batched over all rows.                                 */
/* ------------------------------------------------------------------------ */
static int max_levels(i64 cols) { int L = 0; i64 m = cols; while (m > 1) { m = (m + 1) / 2; ++L; } return L; }

static void MAXROW(orc_ctx* ctx, i64 rows, i64 cols, i64 row_off, int w,
                   const u64* x0, const u64* x1, u64* mx0, u64* mx1)
{
    u64 *v0 = A(rows * cols), *v1 = A(rows * cols);
    memcpy(v0, x0, sizeof(u64) * (size_t)(rows * cols));
    memcpy(v1, x1, sizeof(u64) * (size_t)(rows * cols));
    i64 m = cols;
    while (m > 1) {
        i64 h = m / 2;
        i64 nn = rows * h;
        u64 *d0 = A(nn), *d1 = A(nn), *c0 = A(nn), *c1 = A(nn), *p0 = A(nn), *p1 = A(nn);
        for (i64 r = 0; r < rows; ++r)
            for (i64 i = 0; i < h; ++i) {
                d0[r * h + i] = v0[r * cols + i] - v0[r * cols + i + h];
                d1[r * h + i] = v1[r * cols + i] - v1[r * cols + i + h];
            }
        u64 U = (u64)(row_off * h);
        LTZ(ctx, nn, U, w, d0, d1, c0, c1);
        notmask(c0, c1, nn);
        BM(ctx, nn, U, d0, d1, c0, c1, p0, p1);
        for (i64 r = 0; r < rows; ++r) {
            for (i64 i = 0; i < h; ++i) {
                u64 y0 = v0[r * cols + i + h], y1 = v1[r * cols + i + h];
                v0[r * cols + i] = y0 + p0[r * h + i];
                v1[r * cols + i] = y1 + p1[r * h + i];
            }
            if (m & 1) { v0[r * cols + h] = v0[r * cols + m - 1]; v1[r * cols + h] = v1[r * cols + m - 1]; }
        }
        m = h + (m & 1);
        free(d0); free(d1); free(c0); free(c1); free(p0); free(p1);
    }
    for (i64 r = 0; r < rows; ++r) { mx0[r] = v0[r * cols]; mx1[r] = v1[r * cols]; }
    free(v0); free(v1);
}

void orc_max(orc_ctx* ctx, const u64* x0, const u64* x1, u64* z0, u64* z1, i64 rows, i64 cols,
             i64 row_off, int w)
{
    if (rows <= 0 || cols <= 0) { ctx->step += 2 * (u64)max_levels(cols); return; }
    MAXROW(ctx, rows, cols, row_off, w, x0, x1, z0, z1);
}

int orc_max_levels(i64 cols) { return max_levels(cols); }

/* MaxPool2d: each output window (public zero padding, R26) becomes one row of */
/* k*k entries, row index = global output index; then MAX_row.   */
void orc_maxpool2d(orc_ctx* ctx, const u64* x0, const u64* x1, u64* z0, u64* z1,
                   int N, int C, int H, int W, int k, int stride, int pad, i64 img_off, int w)
{
    int Ho = (H + 2 * pad - k) / stride + 1, Wo = (W + 2 * pad - k) / stride + 1;
    i64 rows = (i64)N * C * Ho * Wo, cols = (i64)k * k;
    u64 *r0 = A(rows * cols), *r1 = A(rows * cols);
    for (i64 o = 0; o < rows; ++o) {
        i64 ow = o % Wo, oh = (o / Wo) % Ho, c = (o / ((i64)Wo * Ho)) % C, nimg = o / ((i64)Wo * Ho * C);
        for (int dy = 0; dy < k; ++dy)
            for (int dx = 0; dx < k; ++dx) {
                i64 iy = oh * stride - pad + dy, ix = ow * stride - pad + dx;
                u64 a = 0, b = 0;
                if (iy >= 0 && iy < H && ix >= 0 && ix < W) {
                    i64 idx = ((nimg * C + c) * H + iy) * W + ix;
                    a = x0[idx]; b = x1[idx];
                }
                r0[o * cols + dy * k + dx] = a; r1[o * cols + dy * k + dx] = b;
            }
    }
    i64 row_off = img_off * (i64)C * Ho * Wo;
    orc_max(ctx, r0, r1, z0, z1, rows, cols, row_off, w);
    free(r0); free(r1);
}

/* ------------------------------------------------------------------------ */
/* S14 SOFTMAX: e^{x - max} / sum e^{x - max} (P:604 footnote)     */
/*   m = MAX_row(x); d = x - m; e = EXP(d) [units: element index];             */
/*   S = rowsum(e); r = RECIP(S) [units: row]; out = MT(e, bcast r) [element]  */
/* ------------------------------------------------------------------------ */
/* causal (reading R24c): the rows are the T x T score blocks of causal attention,
 * T = cols; global row g attends to columns j <= g mod T.  The masked entries enter the max as
 * the public constant -2^(w-2) (below every in-window value, so never the maximum), their
 * exponentials are replaced by the public 0 before the row sum, and their outputs are the
 * public 0.  Same units and steps as the dense softmax.                                        */
static int causal_masked(i64 row_off, i64 r, i64 j, i64 cols) { return j > (row_off + r) % cols; }

void orc_softmax(orc_ctx* ctx, const u64* x0, const u64* x1, u64* z0, u64* z1,
                 i64 rows, i64 cols, i64 row_off, int w,
                 int exp_t, int exp_clamp, int exp_w, int exp_sq,
                 int rc_iters, int rc_t, int rc_clamp, int rc_w, int rc_sq, int bcast, int causal)
{
    i64 n = rows * cols;
    u64 *mx0 = A(rows), *mx1 = A(rows), *e0 = A(n), *e1 = A(n), *S0 = A(rows), *S1 = A(rows);
    u64 *r0 = A(rows), *r1 = A(rows), *b0 = A(n), *b1 = A(n);
    if (rows > 0 && cols > 0) {
        if (causal) {                                  /* masked inputs of the max: public -2^(w-2) */
            u64 *m0 = A(n), *m1 = A(n);
            const u64 L = w >= 2 ? (u64)0 - ((u64)1 << (w - 2)) : (u64)0 - 1;
            for (i64 r = 0; r < rows; ++r)
                for (i64 j = 0; j < cols; ++j) {
                    int msk = causal_masked(row_off, r, j, cols);
                    m0[r * cols + j] = msk ? L : x0[r * cols + j];
                    m1[r * cols + j] = msk ? 0 : x1[r * cols + j];
                }
            MAXROW(ctx, rows, cols, row_off, w, m0, m1, mx0, mx1);
            free(m0); free(m1);
        } else {
            MAXROW(ctx, rows, cols, row_off, w, x0, x1, mx0, mx1);
        }
    } else ctx->step += 2 * (u64)max_levels(cols);
    for (i64 r = 0; r < rows; ++r)
        for (i64 j = 0; j < cols; ++j) {
            e0[r * cols + j] = x0[r * cols + j] - mx0[r];
            e1[r * cols + j] = x1[r * cols + j] - mx1[r];
        }
    u64 Ue = (u64)(row_off * cols);
    EXP(ctx, n, Ue, exp_t, exp_clamp, exp_w, exp_sq, e0, e1, e0, e1);
    if (causal)
        for (i64 r = 0; r < rows; ++r)
            for (i64 j = 0; j < cols; ++j)
                if (causal_masked(row_off, r, j, cols)) e0[r * cols + j] = e1[r * cols + j] = 0;
    for (i64 r = 0; r < rows; ++r) {
        u64 a = 0, b = 0;
        for (i64 j = 0; j < cols; ++j) { a += e0[r * cols + j]; b += e1[r * cols + j]; }
        S0[r] = a; S1[r] = b;
    }
    RECIP(ctx, rows, (u64)row_off, rc_iters, rc_t, rc_clamp, rc_w, rc_sq, S0, S1, r0, r1);
    if (bcast) {                                      /* NEXT #2: one opening of r per row */
        BMB(ctx, rows, cols, Ue, (u64)row_off, e0, e1, r0, r1, z0, z1);
        for (i64 i = 0; i < n; ++i) { z0[i] = shr(z0[i], FRAC); z1[i] = shr(z1[i], FRAC); }
    } else {
        for (i64 r = 0; r < rows; ++r)
            for (i64 j = 0; j < cols; ++j) { b0[r * cols + j] = r0[r]; b1[r * cols + j] = r1[r]; }
        MT(ctx, n, Ue, e0, e1, b0, b1, z0, z1);
    }
    if (causal)
        for (i64 r = 0; r < rows; ++r)
            for (i64 j = 0; j < cols; ++j)
                if (causal_masked(row_off, r, j, cols)) z0[r * cols + j] = z1[r * cols + j] = 0;
    free(mx0); free(mx1); free(e0); free(e1); free(S0); free(S1); free(r0); free(r1); free(b0); free(b1);
}

/* ------------------------------------------------------------------------ */
/* S15 LAYERNORM (mean as Sec-PubFloat Mul by 1/d):          */
/*   mean_mode 0: x 1/d as pmulF(., 1/d)  (E(1/768) = 85, R25)      */
/*   mean_mode 1: per-share floor division by the public integer d (R25),       */
/*                same wrap probability as local truncation           */
/*   mu = pmulF(rowsum(x), 1/d); c = x - mu;                                   */
/*   v = addP(pmulF(rowsum(MT(c,c)), 1/d), eps); r = RSQRT(v) [units: row];    */
/*   out = MT(c, bcast r) [units: element]                                     */
/* ------------------------------------------------------------------------ */
void orc_layernorm(orc_ctx* ctx, const u64* x0, const u64* x1, u64* z0, u64* z1,
                   i64 rows, i64 cols, i64 row_off, double eps, int mean_mode,
                   int rs_iters, int rs_t, int rs_clamp, int rs_w, int rs_sq, int bcast)
{
    i64 n = rows * cols;
    u64 *mu0 = A(rows), *mu1 = A(rows), *c0 = A(n), *c1 = A(n), *q0 = A(n), *q1 = A(n);
    u64 *v0 = A(rows), *v1 = A(rows), *r0 = A(rows), *r1 = A(rows), *b0 = A(n), *b1 = A(n);
    double inv_d = 1.0 / (double)cols;
    for (i64 r = 0; r < rows; ++r) {
        u64 a = 0, b = 0;
        for (i64 j = 0; j < cols; ++j) { a += x0[r * cols + j]; b += x1[r * cols + j]; }
        mu0[r] = a; mu1[r] = b;
    }
    if (mean_mode == 0) pmulF(mu0, mu1, rows, inv_d);
    else divP(mu0, mu1, rows, cols);
    for (i64 r = 0; r < rows; ++r)
        for (i64 j = 0; j < cols; ++j) {
            c0[r * cols + j] = x0[r * cols + j] - mu0[r];
            c1[r * cols + j] = x1[r * cols + j] - mu1[r];
        }
    u64 Ue = (u64)(row_off * cols);
    MT(ctx, n, Ue, c0, c1, c0, c1, q0, q1);
    for (i64 r = 0; r < rows; ++r) {
        u64 a = 0, b = 0;
        for (i64 j = 0; j < cols; ++j) { a += q0[r * cols + j]; b += q1[r * cols + j]; }
        v0[r] = a; v1[r] = b;
    }
    if (mean_mode == 0) pmulF(v0, v1, rows, inv_d);
    else divP(v0, v1, rows, cols);
    addP(v0, rows, eps);
    RSQRT(ctx, rows, (u64)row_off, rs_iters, rs_t, rs_clamp, rs_w, rs_sq, v0, v1, r0, r1);
    if (bcast) {                                      /* NEXT #2: one opening of r per row */
        BMB(ctx, rows, cols, Ue, (u64)row_off, c0, c1, r0, r1, z0, z1);
        for (i64 i = 0; i < n; ++i) { z0[i] = shr(z0[i], FRAC); z1[i] = shr(z1[i], FRAC); }
    } else {
        for (i64 r = 0; r < rows; ++r)
            for (i64 j = 0; j < cols; ++j) { b0[r * cols + j] = r0[r]; b1[r * cols + j] = r1[r]; }
        MT(ctx, n, Ue, c0, c1, b0, b1, z0, z1);
    }
    free(mu0); free(mu1); free(c0); free(c1); free(q0); free(q1);
    free(v0); free(v1); free(r0); free(r1); free(b0); free(b1);
}

/* ------------------------------------------------------------------------ */
/* Beaver MATMUL over Z_2^64 (the CrypTen++ Beaver       */
/* matmul, P:563 / P:846; the same algebra as S4 with matrix triples).        */
/* Z = X Y for `batch` independent products X[b] (M x K), Y[b] (K x N),       */
/* row-major, contiguous.  One step s.  Units (global batch index g = boff+b):  */
/*   uA = g*M*K + m*K + k ; uB = g*K*N + k*N + n ; uC = g*M*N + m*N + n        */
/* Triple:                                                    */
/*   A_p = half (uA&1) of PRG(K_p, uA>>1, s, 8)   (p = 0, 1)                     */
/*   B_p = half (uB&1) of PRG(K_p, uB>>1, s, 9)                                  */
/*   C0  = half (uC&1) of PRG(K_0, uC>>1, s, 10) ; C1 = (A0+A1)(B0+B1) - C0     */
/*   (matrix product mod 2^64; dealer correction to party 1, R7)               */
/* E = open(X - A), F = open(Y - B) (one round, 8 (MK + KN) B per party);      */
/* Z0 = C0 + E B0 + A0 F + E F ;  Z1 = C1 + E B1 + A1 F  (party 0 adds E F).    */
/* ------------------------------------------------------------------------ */
static u64 prg_half(u64 key, u64 u, u64 s, u32 slot)
{
    u32 w[4];
    prg(key, u >> 1, s, slot, w);
    return (u & 1) ? w64(w[2], w[3]) : w64(w[0], w[1]);
}

/* R = P Q (rows x inner) (inner x cols), mod 2^64, plain triple loop */
static void ring_matmul(const u64* P, const u64* Q, u64* R, i64 rows, i64 inner, i64 cols)
{
    for (i64 i = 0; i < rows; ++i)
        for (i64 j = 0; j < cols; ++j) {
            u64 acc = 0;
            for (i64 k = 0; k < inner; ++k) acc += P[i * inner + k] * Q[k * cols + j];
            R[i * cols + j] = acc;
        }
}

void orc_matmul(orc_ctx* ctx, const u64* x0, const u64* x1, const u64* y0, const u64* y1,
                u64* z0, u64* z1, i64 batch, i64 M, i64 K, i64 N, i64 batch_off, int trunc_bits)
{
    u64 s = ctx->step++;
    i64 MK = M * K, KN = K * N, MN = M * N;
    u64 *A0 = A(MK), *A1 = A(MK), *As = A(MK), *E = A(MK);
    u64 *B0 = A(KN), *B1 = A(KN), *Bs = A(KN), *F = A(KN);
    u64 *C0 = A(MN), *C1 = A(MN), *T = A(MN);
    for (i64 b = 0; b < batch; ++b) {
        u64 g = (u64)(batch_off + b);
        const u64 *xb0 = x0 + b * MK, *xb1 = x1 + b * MK, *yb0 = y0 + b * KN, *yb1 = y1 + b * KN;
        for (i64 i = 0; i < MK; ++i) {
            u64 u = g * (u64)MK + (u64)i;
            A0[i] = prg_half(ctx->key_p0, u, s, 8);
            A1[i] = prg_half(ctx->key_p1, u, s, 8);
            As[i] = A0[i] + A1[i];
            E[i] = (xb0[i] - A0[i]) + (xb1[i] - A1[i]);          /* opened */
        }
        for (i64 i = 0; i < KN; ++i) {
            u64 u = g * (u64)KN + (u64)i;
            B0[i] = prg_half(ctx->key_p0, u, s, 9);
            B1[i] = prg_half(ctx->key_p1, u, s, 9);
            Bs[i] = B0[i] + B1[i];
            F[i] = (yb0[i] - B0[i]) + (yb1[i] - B1[i]);          /* opened */
        }
        for (i64 i = 0; i < MN; ++i) C0[i] = prg_half(ctx->key_p0, g * (u64)MN + (u64)i, s, 10);
        ring_matmul(As, Bs, C1, M, K, N);                          /* dealer: A B */
        for (i64 i = 0; i < MN; ++i) C1[i] -= C0[i];
        u64 *zb0 = z0 + b * MN, *zb1 = z1 + b * MN;
        /* party 0: C0 + E B0 + A0 F + E F */
        memcpy(zb0, C0, sizeof(u64) * (size_t)MN);
        ring_matmul(E, B0, T, M, K, N);  for (i64 i = 0; i < MN; ++i) zb0[i] += T[i];
        ring_matmul(A0, F, T, M, K, N);  for (i64 i = 0; i < MN; ++i) zb0[i] += T[i];
        ring_matmul(E, F, T, M, K, N);   for (i64 i = 0; i < MN; ++i) zb0[i] += T[i];
        /* party 1: C1 + E B1 + A1 F */
        memcpy(zb1, C1, sizeof(u64) * (size_t)MN);
        ring_matmul(E, B1, T, M, K, N);  for (i64 i = 0; i < MN; ++i) zb1[i] += T[i];
        ring_matmul(A1, F, T, M, K, N);  for (i64 i = 0; i < MN; ++i) zb1[i] += T[i];
        if (trunc_bits)
            for (i64 i = 0; i < MN; ++i) { zb0[i] = shr(zb0[i], trunc_bits); zb1[i] = shr(zb1[i], trunc_bits); }
    }
    free(A0); free(A1); free(As); free(E); free(B0); free(B1); free(Bs); free(F);
    free(C0); free(C1); free(T);
}

/* ------------------------------------------------------------------------ */
/* Small-ring truncation statistics (acceptance 4): ring Z_2^N with    */
/* N < 64, shares uniform in the ring, per-share arithmetic shift by k bits.  */
/* Returns the number of trials whose reconstruction is not within            */
/* {floor(x/2^k), floor(x/2^k) - 1} mod 2^N.  Uses its own PRG key stream.    */
/* ------------------------------------------------------------------------ */
i64 orc_trunc_wrap_trials(int N, int k, i64 x, i64 trials, u64 key)
{
    u64 mask = (N == 64) ? ~(u64)0 : (((u64)1 << N) - 1);
    i64 bad = 0;
    for (i64 t = 0; t < trials; ++t) {
        u32 wd[4];
        prg(key, (u64)t, 0, 0, wd);
        u64 r = w64(wd[0], wd[1]) & mask;
        u64 xv = (u64)x & mask;
        u64 s0 = (xv - r) & mask, s1 = r;
        /* signed interpretation of an N-bit share, then arithmetic shift */
        i64 v0 = (i64)(s0 << (64 - N)) >> (64 - N);
        i64 v1 = (i64)(s1 << (64 - N)) >> (64 - N);
        u64 z = ((u64)(v0 >> k) + (u64)(v1 >> k)) & mask;
        i64 zs = (i64)(z << (64 - N)) >> (64 - N);
        i64 expect = x >> k;
        if (!(zs == expect || zs == expect - 1)) ++bad;
    }
    return bad;
}

/* ======================================================================== */
/* PLAINTEXT-RING SCHEDULES: the auto-tuner's non-MPC evaluator (SURVEY      */
/* 8(f) NEXT #4; "directly lowering the graph to a (non-MPC)       */
/* PyTorch GPU runtime").  Each schedule of DESIGN.md 2.5 is  */
/* run on ONE plaintext ring value per element (int64 at scale 2^16) instead */
/* of two shares -- no PRG, no openings:                                     */
/*   BM(x, y)     -> the wrapping ring product x*y mod 2^64                  */
/*   MT(x, y)     -> floor((x*y mod 2^64) / 2^16)  (arithmetic shift)         */
/*   pmulF(x, c)  -> floor((x*E(c) mod 2^64) / 2^16)                          */
/*   addP(x, c)   -> x + E(c)                                                */
/*   shr(x, k)    -> floor(x / 2^k)                                          */
/*   LTZ_w(x)     -> bit (w-1) of x  (the value LTZ reconstructs, R12)        */
/*   NOT(b)       -> 1 - b                                                   */
/* Inputs are doubles, encoded with E (round half even, R2); outputs are the */
/* ring results decoded as (double)(int64)v / 2^16.  The MPC schedules differ */
/* from these only by the per-share truncation of each product.     */
/* ======================================================================== */
static i64 pl_mt(i64 x, i64 y) { return (i64)((u64)x * (u64)y) >> FRAC; }
static i64 pl_mulf(i64 x, double c) { return (i64)((u64)x * (u64)orc_encode(c)) >> FRAC; }
static i64 pl_ltz(i64 x, int w) { return (i64)(((u64)x >> (w - 1)) & 1); }
static double pl_dec(i64 v) { return (double)v / 65536.0; }

/* EXP(x; t, clamp, w) on plaintext (R4, R13) */
static i64 pl_exp(i64 x, int t, int clamp, int w)
{
    i64 y = (x >> t) + orc_encode(1.0);
    if (clamp) y = (i64)((u64)y * (u64)(1 - pl_ltz(x + orc_encode(ldexp(1.0, t)), w)));  /* no truncation */
    for (int k = 0; k < t; ++k) y = pl_mt(y, y);
    return y;
}
/* RECIP: y0 = 3 EXP(0.5 - x) + 0.003; iters x y <- y (2 - x y) */
static i64 pl_recip(i64 x, int iters, int t, int clamp, int w)
{
    i64 g = pl_exp(orc_encode(0.5) - x, t, clamp, w);
    i64 y = (i64)((u64)g * 3u) + orc_encode(0.003);
    for (int it = 0; it < iters; ++it) {
        i64 p = pl_mt(x, y);
        y = pl_mt(y, orc_encode(2.0) - p);
    }
    return y;
}
/* RSQRT: y0 = 2.2 EXP(-(x/2 + 0.2)) + 0.2; iters x y <- (y (3 - x y^2)) * 0.5 */
static i64 pl_rsqrt(i64 x, int iters, int t, int clamp, int w)
{
    i64 g = pl_exp(-((x >> 1) + orc_encode(0.2)), t, clamp, w);
    i64 y = pl_mulf(g, 2.2) + orc_encode(0.2);
    for (int it = 0; it < iters; ++it) {
        i64 q = pl_mt(y, y);
        i64 p = pl_mt(x, q);
        i64 u = pl_mt(y, orc_encode(3.0) - p);
        y = pl_mulf(u, 0.5);
    }
    return y;
}
/* HORNER(v; c_0..c_d) and POWER(v; c_0..c_d) on plaintext */
static i64 pl_horner(i64 v, const double* c, int d)
{
    i64 h = pl_mulf(v, c[d]) + orc_encode(c[d - 1]);
    for (int k = d - 2; k >= 0; --k) h = pl_mt(h, v) + orc_encode(c[k]);
    return h;
}
static i64 pl_power(i64 v, const double* c, int d)
{
    i64 p[5] = {0, v, 0, 0, 0};
    if (d >= 2) p[2] = pl_mt(v, v);
    if (d >= 3) p[3] = pl_mt(p[2], v);
    if (d >= 4) p[4] = pl_mt(p[2], p[2]);
    i64 h = 0;
    for (int k = 1; k <= d; ++k) h += pl_mulf(p[k], c[k]);
    return h + orc_encode(c[0]);
}
/* S13 segment forms on plaintext (R21, R30) */
static i64 pl_act(i64 x, int act, int form, int degree, double B, const double* coeffs,
                  const double* erf_a, int erf_terms, int w, int basis)
{
    if (form == FORM_RELU || (form != FORM_ERF && degree == 0)) {
        i64 nl = 1 - pl_ltz(x, w);
        return act == ACT_SIGMOID ? (i64)((u64)nl << FRAC) : (i64)((u64)x * (u64)nl);
    }
    i64 l1 = pl_ltz(x + orc_encode(B), w), l2 = pl_ltz(x + orc_encode(-B), w);
    i64 h;
    if (form == FORM_POLY_X) {
        h = basis ? pl_power(x, coeffs, degree) : pl_horner(x, coeffs, degree);
    } else if (form == FORM_POLY_ABS) {
        i64 ax = (i64)((u64)x * (u64)(1 - 2 * pl_ltz(x, w)));      /* |x| = x (1 - 2 s) */
        h = pl_mulf(x, 0.5) + (basis ? pl_power(ax, coeffs, degree) : pl_horner(ax, coeffs, degree));
    } else {                                                         /* erf series (R21) */
        i64 z = pl_mulf(x, 1.0 / sqrt(2.0));
        i64 z2 = pl_mt(z, z);
        i64 S = pl_horner(z2, erf_a, erf_terms - 1);
        i64 erf = pl_mulf(pl_mt(z, S), 2.0 / sqrt(M_PI));
        h = pl_mulf(pl_mt(x, erf + orc_encode(1.0)), 0.5);
    }
    i64 out = (i64)((u64)h * (u64)(l2 - l1));
    i64 nl2 = 1 - l2;
    out += act == ACT_SIGMOID ? (i64)((u64)nl2 << FRAC) : (i64)((u64)x * (u64)nl2);
    return out;
}

void orc_plain_exp(const double* x, double* y, i64 n, int t, int clamp, int w)
{
    for (i64 i = 0; i < n; ++i) y[i] = pl_dec(pl_exp(orc_encode(x[i]), t, clamp, w));
}
void orc_plain_recip(const double* x, double* y, i64 n, int iters, int t, int clamp, int w)
{
    for (i64 i = 0; i < n; ++i) y[i] = pl_dec(pl_recip(orc_encode(x[i]), iters, t, clamp, w));
}
void orc_plain_rsqrt(const double* x, double* y, i64 n, int iters, int t, int clamp, int w)
{
    for (i64 i = 0; i < n; ++i) y[i] = pl_dec(pl_rsqrt(orc_encode(x[i]), iters, t, clamp, w));
}
void orc_plain_act(const double* x, double* y, i64 n, int act, int form, int degree, double B,
                   const double* coeffs, int erf_terms, int w, int basis)
{
    double a[16];
    double fact = 1.0;
    for (int k = 0; k < erf_terms && k < 16; ++k) {                 /* (-1)^k / (k! (2k+1)) */
        if (k > 0) fact *= (double)k;
        a[k] = ((k & 1) ? -1.0 : 1.0) / (fact * (double)(2 * k + 1));
    }
    for (i64 i = 0; i < n; ++i)
        y[i] = pl_dec(pl_act(orc_encode(x[i]), act, form, degree, B, coeffs, a, erf_terms, w, basis));
}

/* MAX_row on plaintext: the half-split tree of DESIGN.md 2.5 (R22) with the mux               */
/* x_i' = x_{i+h} + d (1 - LTZ_w(d)), d = x_i - x_{i+h}; odd m carries x_{m-1} to position h.   */
/* In place over v[0..cols); returns the row maximum (exact when every d is inside the window). */
static i64 pl_maxrow(i64* v, i64 cols, int w)
{
    i64 m = cols;
    while (m > 1) {
        i64 h = m / 2;
        for (i64 i = 0; i < h; ++i) {
            i64 d = v[i] - v[i + h];
            v[i] = v[i + h] + (i64)((u64)d * (u64)(1 - pl_ltz(d, w)));
        }
        if (m & 1) v[h] = v[m - 1];
        m = h + (m & 1);
    }
    return v[0];
}
void orc_plain_max(const double* x, double* y, i64 rows, i64 cols, int w)
{
    i64* v = (i64*)malloc(sizeof(i64) * (size_t)(cols > 0 ? cols : 1));
    for (i64 r = 0; r < rows; ++r) {
        for (i64 j = 0; j < cols; ++j) v[j] = orc_encode(x[r * cols + j]);
        y[r] = pl_dec(pl_maxrow(v, cols, w));
    }
    free(v);
}

/* SOFTMAX rows on plaintext (causal 2.12 with row r of the call at position  */
/* r mod cols): MAX_row as the half-split tree with the mux x_i' = x_{i+h} + d (1 - LTZ_w(d)),  */
/* d = x_i - x_{i+h} (masked entries enter as -2^(w-2)); e = EXP(x - m) (masked -> 0);        */
/* S = rowsum(e); r = RECIP(S); out = MT(e, r) (masked -> 0).                                  */
void orc_plain_softmax(const double* x, double* y, i64 rows, i64 cols, int w,
                       int exp_t, int exp_clamp, int exp_w, int rc_iters, int rc_t, int rc_clamp, int rc_w,
                       int causal)
{
    i64* v = (i64*)malloc(sizeof(i64) * (size_t)(cols > 0 ? cols : 1));
    i64* e = (i64*)malloc(sizeof(i64) * (size_t)(cols > 0 ? cols : 1));
    const i64 L = w >= 2 ? -((i64)1 << (w - 2)) : -1;
    for (i64 r = 0; r < rows; ++r) {
        const double* xr = x + r * cols;
        double* yr = y + r * cols;
        i64 pos = r % cols;
        for (i64 j = 0; j < cols; ++j) v[j] = (causal && j > pos) ? L : orc_encode(xr[j]);
        const i64 mx = pl_maxrow(v, cols, w);
        i64 S = 0;
        for (i64 j = 0; j < cols; ++j) {
            e[j] = (causal && j > pos) ? 0 : pl_exp(orc_encode(xr[j]) - mx, exp_t, exp_clamp, exp_w);
            S += e[j];
        }
        const i64 rc = pl_recip(S, rc_iters, rc_t, rc_clamp, rc_w);
        for (i64 j = 0; j < cols; ++j) yr[j] = (causal && j > pos) ? 0.0 : pl_dec(pl_mt(e[j], rc));
    }
    free(v); free(e);
}

/* LAYERNORM rows on plaintext (R25): mu = pmulF(rowsum x, 1/d) (mode 0) or     */
/* floor(rowsum x / d) (mode 1); c = x - mu; v = (same mean of rowsum MT(c,c)) + E(eps);    */
/* r = RSQRT(v); out = MT(c, r).                                                            */
void orc_plain_layernorm(const double* x, double* y, i64 rows, i64 cols, double eps, int mean_mode,
                         int rs_iters, int rs_t, int rs_clamp, int rs_w)
{
    const double inv_d = 1.0 / (double)cols;
    for (i64 r = 0; r < rows; ++r) {
        const double* xr = x + r * cols;
        double* yr = y + r * cols;
        i64 s = 0;
        for (i64 j = 0; j < cols; ++j) s += orc_encode(xr[j]);
        const i64 mu = mean_mode == 0 ? pl_mulf(s, inv_d) : floordiv(s, cols);
        i64 q = 0;
        for (i64 j = 0; j < cols; ++j) { i64 c = orc_encode(xr[j]) - mu; q += pl_mt(c, c); }
        const i64 v = (mean_mode == 0 ? pl_mulf(q, inv_d) : floordiv(q, cols)) + orc_encode(eps);
        const i64 rs = pl_rsqrt(v, rs_iters, rs_t, rs_clamp, rs_w);
        for (i64 j = 0; j < cols; ++j) yr[j] = pl_dec(pl_mt(orc_encode(xr[j]) - mu, rs));
    }
}
