/*
 * mpc200.h -- C ABI of the B200-native two-party nonlinear-operator library.
 *
 * Method: arxiv 2511.19711 (CrypTorch / CrypTen++), the approximated nonlinear
 * operators its characterization finds dominant, over
 * 2-party additive secret shares in Z_2^64 with 16 fractional bits,
 * trusted-dealer Beaver triples, local truncation and a
 * GMW comparison.  The bit-exact contract every entry point
 * implements is DESIGN.md section 2 (PRG layout 2.3, schedules 2.5).
 *
 * Conventions for every compute entry point:
 *  - All data pointers are DEVICE pointers on the context's device, owned and
 *    allocated by the caller; the library never frees caller memory.  Shares are
 *    uint64_t arrays (ring elements of Z_2^64), 8-byte aligned, dense, row-major.
 *  - mpc_shares carries one pointer per party.  MPC_MODE_BOTH and
 *    MPC_MODE_PAIR_LOOPBACK need sh[0] and sh[1]; MPC_MODE_PAIR needs sh[party] only.
 *  - Every call is ASYNCHRONOUS on the context's CUDA stream (cudaStream_t passed
 *    as void*); results are valid after the stream is synchronized.  The calling thread's
 *    current CUDA device must be the context's device (MPC_ERR_INVALID otherwise).
 *  - `off` / `row_off` is the global index of this shard's first element / row:
 *    the PRG is keyed by global unit, so shards reproduce the unsharded shares.
 *    Ops that contain a comparison need off (and row_off * per-row units)
 *    divisible by 32 (MPC_ERR_INVALID otherwise).
 *  - In-place operation (z == x) is allowed for element-wise ops and softmax.
 *  - Each randomness-consuming primitive advances the context's step counter by
 *    one; the step counts of every op are listed below.
 *  - Errors: the call returns a status and leaves the step counter unchanged;
 *    mpc_last_error() gives a message.  CUDA launch errors surface as
 *    MPC_ERR_CUDA at the call (or, for asynchronous faults, at the next call).
 */
#ifndef MPC200_H
#define MPC200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MPC_OK = 0,
    MPC_ERR_INVALID = 1,   /* null / misaligned pointer, bad shape, bad mode      */
    MPC_ERR_RANGE = 2,     /* knob out of range, step counter exhausted (2^32)    */
    MPC_ERR_CUDA = 3,      /* CUDA runtime or launch failure                       */
    MPC_ERR_NCCL = 4,      /* exchange failure in a PAIR mode                      */
    MPC_ERR_PROTOCOL = 5,  /* parties disagree on the op header (debug mode)      */
    MPC_ERR_REUSE = 6,     /* set_step below the current step (triple reuse)      */
    MPC_ERR_TIMEOUT = 7,
    MPC_ERR_NOMEM = 8,
    MPC_ERR_UNSUPPORTED = 9
} mpc_status;

typedef enum {
    MPC_MODE_BOTH = 0,          /* one GPU simulates both parties; openings add in registers   */
    MPC_MODE_PAIR = 1,          /* one GPU (process) per party; every opening is exchanged by  *
                                 * the fused kernels through NVLink peer memory. *
                                 * TRUST MODEL: party 1's correction terms (Beaver / square /  *
                                 * broadcast c1, AND-triple c1, daBit r1A) come from the       *
                                 * trusted dealer as a correction stream              *
                                 * (mpc_ctx_set_corrections, produced offline by an            *
                                 * MPC_MODE_DEALER context): party 1's context then never      *
                                 * uses K_0 (its key_p0 may be 0).  Without a stream, party 1  *
                                 * SIMULATES the dealer from key_p0 (reading R7) and can       *
                                 * regenerate party 0's masks: no privacy against party 1.    */
    MPC_MODE_PAIR_LOOPBACK = 2, /* both parties' PAIR kernels in one launch on one GPU,        *
                                 * exchanging through local memory (same code path; tests)    */
    MPC_MODE_DEALER = 3         /* the trusted dealer's offline pass for party 1 (DESIGN.md    *
                                 * 7.1): holds K_0 and K_1, issues the SAME calls with the     *
                                 * same shapes, offsets and knobs as party 1 (share pointers   *
                                 * may be NULL: no share is read or written, nothing is        *
                                 * exchanged) and appends party 1's correction words to its    *
                                 * stream (mpc_dealer_stream).  cfg.party must be 1.          */
} mpc_mode;

typedef struct {
    int mode;               /* mpc_mode                                              */
    int party;              /* 0 | 1 (ignored in MPC_MODE_BOTH)                       */
    int frac_bits;          /* must be 16                                    */
    int device;             /* CUDA device ordinal                                    */
    uint64_t key_share;     /* K_s: pairwise share-mask key          */
    uint64_t key_p0;        /* K_0: dealer -> party 0 key                             */
    uint64_t key_p1;        /* K_1: dealer -> party 1 key                             */
    void* cuda_stream;      /* cudaStream_t the calls are enqueued on (NULL = legacy) */
    void* reserved;         /* must be NULL                                            */
} mpc_config;

typedef struct mpc_ctx mpc_ctx;

typedef struct { uint64_t* sh[2]; } mpc_shares;

typedef struct {
    uint64_t steps;          /* step ids consumed                                        */
    uint64_t philox_calls;   /* Philox4x32-10 blocks generated (algorithmic count)        */
    uint64_t bytes_per_party;/* bytes each party sends in a PAIR execution (model; 2.4)   */
    uint64_t rounds;         /* communication rounds                                     */
    uint64_t launches;       /* kernels launched                                         */
    uint64_t calls;          /* ABI calls                                                */
} mpc_stats;

/* ---- context -------------------------------------------------------------- */
mpc_status mpc_ctx_create(const mpc_config* cfg, mpc_ctx** out);
mpc_status mpc_ctx_destroy(mpc_ctx* ctx);
/* Replay support: set the next step id.  Below the current step -> MPC_ERR_REUSE
 * unless force != 0 (the triple-reuse analogue of S:440). */
mpc_status mpc_ctx_set_step(mpc_ctx* ctx, uint64_t step, int force);
uint64_t   mpc_ctx_get_step(const mpc_ctx* ctx);
mpc_status mpc_ctx_set_stream(mpc_ctx* ctx, void* cuda_stream);
mpc_status mpc_ctx_stats(const mpc_ctx* ctx, mpc_stats* out);
mpc_status mpc_ctx_reset_stats(mpc_ctx* ctx);
const char* mpc_last_error(const mpc_ctx* ctx);
const char* mpc_version(void);
/* Philox4x32-10 blocks generated per element by each op (algorithmic),
 * used for the ALU roofline.  Returns the count for the last call on ctx. */
uint64_t mpc_last_call_philox(const mpc_ctx* ctx);

/* ---- PAIR mode plumbing ---------------------------------------------------------
 * MPC_MODE_PAIR: each party's context allocates its exchange memory (receive buffers and
 * flags) at creation; the parties swap the opaque handles out of band
 * (bench/binding use torch.distributed) and connect.  Both parties must then issue the
 * same sequence of calls with the same shapes; each fused kernel exchanges its openings
 * with the peer kernel through peer memory.  An exchange that does not complete within
 * 10 s poisons the context (results undefined) and mpc_ctx_sync returns MPC_ERR_TIMEOUT. */
#define MPC_PAIR_HANDLE_BYTES 64
mpc_status mpc_pair_export(mpc_ctx* ctx, void* handle_out /* MPC_PAIR_HANDLE_BYTES */);
mpc_status mpc_pair_connect(mpc_ctx* ctx, const void* peer_handle);
/* Synchronize the context stream; MPC_ERR_PROTOCOL if the debug header check found the parties
 * issuing different calls, MPC_ERR_TIMEOUT if a PAIR exchange timed out, MPC_ERR_CUDA on an
 * asynchronous CUDA error. */
mpc_status mpc_ctx_sync(mpc_ctx* ctx);
/* Debug mode (PAIR modes; default off): before every op the parties exchange an op header (a hash
 * of the entry point, the step id and the op's step count) in one extra round; a mismatch marks
 * the context and mpc_ctx_sync returns MPC_ERR_PROTOCOL.  No effect in MPC_MODE_BOTH. */
mpc_status mpc_ctx_set_debug(mpc_ctx* ctx, int on);
/* PAIR exchange wire format (transport only -- openings, rounds and output shares are
 * unchanged, reading R33): 0 = LL (each 8-byte payload word travels as two {half | round} words:
 * 2 wire bytes per payload byte, fewest instructions; default in MPC_MODE_PAIR_LOOPBACK), 1 = LL63
 * (one {63 payload bits | 1 tag bit} word per payload word plus one tagged top-bit word per warp and
 * word: 33 / 32 wire bytes per payload byte; default in MPC_MODE_PAIR).  Both parties must use the
 * same format.  Only before the context's first PAIR exchange (MPC_ERR_INVALID afterwards);
 * MPC_ERR_RANGE for other values; no effect in MPC_MODE_BOTH. */
mpc_status mpc_ctx_set_exchange(mpc_ctx* ctx, int fmt);
int        mpc_ctx_get_exchange(const mpc_ctx* ctx);   /* current format, -1 for a NULL context */

/* LTZ carry circuit: 0 = full Kogge-Stone (the S7 contract, default),
 * 1 = carry cone (only the carry into bit w-1, pruned: 89 AND gates at w = 33 instead of 290,
 * 181 at w = 64 instead of 693, same rounds), every window 1..64.  The output shares of every op are
 * bit-identical under both circuits (they depend only on the sign and the daBit); only the
 * transcript, the PRG work and the bytes sent change. */
mpc_status mpc_ctx_set_ltz_circuit(mpc_ctx* ctx, int circuit);

/* ---- the trusted dealer's correction stream ("distributed in advance by a trusted
 * third-party") ---------------------------------------------------------------
 * Every PAIR kernel launch of party 1 consumes one SEGMENT of the stream: words
 * [base, base + depth * threads) of the device word array, where word base + k * threads + t is
 * the k-th correction of the launch's thread t (threads = the party's CTAs x block size, depth =
 * corrections per thread, tag = a hash of the kernel family).  A DEALER context appends one
 * segment per launch, in the order party 1 will launch; it runs the same kernels with the same
 * grid as party 1 and synchronizes after each launch (an offline pass). */
typedef struct { uint64_t base, threads, depth, tag; } mpc_corr_seg;
/* Grid the dealer sizes its launches for: MPC_MODE_PAIR (default, party 1 on its own GPU) or
 * MPC_MODE_PAIR_LOOPBACK (party 1's CTAs inside a loopback launch).  MPC_ERR_INVALID on a
 * non-dealer context or another mode. */
mpc_status mpc_dealer_set_target(mpc_ctx* dealer, int target_mode);
/* View of the stream so far: *words is a device pointer owned by the dealer context (valid until
 * its next call or destruction), *segs a host array owned by it. */
mpc_status mpc_dealer_stream(const mpc_ctx* dealer, const uint64_t** words, uint64_t* n_words,
                             const mpc_corr_seg** segs, int64_t* n_segs);
/* Start a new, empty stream (keeps the allocation). */
mpc_status mpc_dealer_reset(mpc_ctx* dealer);
/* Party 1 (MPC_MODE_PAIR with party 1, or MPC_MODE_PAIR_LOOPBACK): consume these corrections,
 * segment by segment in launch order, instead of deriving them from K_0.  words: device pointer
 * on the context's device, owned by the caller, valid until consumed; segs is copied.  A launch
 * whose next segment is missing or does not match (tag, threads) fails with MPC_ERR_PROTOCOL.
 * words == NULL and n_segs == 0 clears the stream (party 1 derives from K_0 again).
 * MPC_ERR_INVALID on party 0, BOTH or DEALER contexts.  mpc_matmul's matrix correction
 * C1 = (A0+A1)(B0+B1) - C0 is one segment of batch*M*N words (tag "matmul_c1", depth 1) that the
 * dealer forms with a ring GEMM and party 1 adds in its GEMM epilogue. */
mpc_status mpc_ctx_set_corrections(mpc_ctx* ctx, const uint64_t* words, uint64_t n_words,
                                   const mpc_corr_seg* segs, int64_t n_segs);
/* Segments not consumed yet; -1 when no stream is set. */
int64_t    mpc_ctx_corrections_left(const mpc_ctx* ctx);

/* Ring-GEMM engine of mpc_matmul: 0 = auto (tensor cores whenever the limb
 * accumulators are exact, i.e. K <= 5461), 1 = SIMT (IMAD u64 multiply-adds), 2 = tensor cores
 * (tcgen05 kind::i8 on 8-bit limbs; MPC_ERR_UNSUPPORTED if K > 5461).  All engines give the
 * same ring product, hence bit-identical output shares. */
mpc_status mpc_ctx_set_matmul_engine(mpc_ctx* ctx, int engine);

/* Per-launch timing (for the roofline in bench.py): when enabled, every kernel the
 * context launches is bracketed by CUDA events on the context stream and tagged with
 * its algorithmic Philox4x32-10 block count.  mpc_ctx_kernel_times synchronizes on
 * the last event, copies up to cap records (oldest first), clears the list and
 * returns the number copied (-1 on a null ctx). */
typedef struct { const char* name; float ms; uint64_t philox; uint64_t units; } mpc_kernel_time;
mpc_status mpc_ctx_enable_kernel_timing(mpc_ctx* ctx, int on);
int        mpc_ctx_kernel_times(mpc_ctx* ctx, mpc_kernel_time* out, int cap);

/* ---- S3: the device PRG itself (known-answer tests, rate microbenchmark) ----
 * out[4*i .. 4*i+3] = Philox4x32-10(key, ctr = (lo32(unit0+i), hi32(unit0+i), step, slot))
 * for i < n.  `reps` > 1 chains the counter through the generator reps times
 * (out = the last block) to measure the generator rate without memory traffic. */
mpc_status mpc_prg_fill(mpc_ctx* ctx, uint64_t key, uint64_t unit0, uint32_t step, uint32_t slot,
                        uint32_t* out, int64_t n, int reps);

/* ---- S1 / S2 ---------------------------------------------------------------- */
/* S1 share: v = E(x) = round-half-even(x * 2^16) (|x| < 2^31);
 * owner's share = v - r, the other party's = r, r = PRG(K_s, off+i, step, 0).
 * x: device float (x_is_f64 = 0) or double (1) array of n; 1 step. */
mpc_status mpc_share(mpc_ctx* ctx, const void* x, int x_is_f64, int owner, mpc_shares out,
                     int64_t n, int64_t off);
/* S2 open: ring_out[i] = x0+x1 mod 2^64 (may be NULL);
 * f64_out[i] = (int64)ring / 2^scale_bits (may be NULL).  No step.  In MPC_MODE_PAIR both
 * parties exchange their shares (1 round, 8 B/element) and both receive the result. */
mpc_status mpc_open(mpc_ctx* ctx, mpc_shares in, int64_t n, uint64_t* ring_out,
                    double* f64_out, int scale_bits);
/* S2 open to one party (SURVEY 8(b) reveal_to): as mpc_open with reveal_to = -1 (both);
 * reveal_to = p in {0, 1}: only party p learns rec -- in the PAIR modes p sends zeros in place
 * of its share (the exchange keeps its lockstep and the peer receives no data from p's
 * share -- but see the MPC_MODE_PAIR trust model: party 1 holds key_p0) and only p writes
 * ring_out / f64_out (the other party may pass NULL).  In MPC_MODE_BOTH the caller holds both
 * parties and the outputs are written as by mpc_open.  MPC_ERR_INVALID for other reveal_to. */
mpc_status mpc_open_to(mpc_ctx* ctx, mpc_shares in, int64_t n, int reveal_to, uint64_t* ring_out,
                       double* f64_out, int scale_bits);

/* ---- S4 / S5 ---------------------------------------------------------------- */
/* S4 Beaver multiply: z = x*y mod 2^64, then per-share
 * arithmetic shift by trunc_bits (0 or 16).  1 step, 1 round, 16 B/elem/party. */
mpc_status mpc_mul(mpc_ctx* ctx, mpc_shares x, mpc_shares y, mpc_shares z, int64_t n,
                   int64_t off, int trunc_bits);
/* S4' square with a square-pair triple (NEXT #2): z = x*x mod 2^64, then
 * per-share shift by trunc_bits (0 or 16).  1 step, 1 round, 8 B/elem/party. */
mpc_status mpc_square(mpc_ctx* ctx, mpc_shares x, mpc_shares z, int64_t n, int64_t off, int trunc_bits);
/* S4'' broadcast multiply (NEXT #2 "broadcast triple"): x is rows x cols
 * (row-major), y is rows; z[r*cols+j] = x[r*cols+j] * y[r] mod 2^64, then per-share shift by
 * trunc_bits (0 or 16).  One mask per row for y: 1 step, 1 round, 8 B/elem + 8 B/row per
 * party.  off = global element index of x[0] (multiple of 2), row_off = global row of y[0]. */
mpc_status mpc_mul_bcast(mpc_ctx* ctx, mpc_shares x, mpc_shares y, mpc_shares z, int64_t rows,
                         int64_t cols, int64_t off, int64_t row_off, int trunc_bits);
/* NEXT #3 Beaver matrix multiplication over Z_2^64 (CrypTen++'s Beaver matmul, P:563,
 * P:846): for b < batch, Z[b] = X[b] Y[b] mod 2^64 with X[b] M x K, Y[b]
 * K x N, Z[b] M x N, all row-major and contiguous; then per-share shift by trunc_bits (0 or
 * 16).  A matrix Beaver triple (A, B, C = AB) from the PRG keyed by global units (batch_off =
 * global index of the first product); 1 step, 1 round, 8 (MK + KN) B per product per party.
 * Caller-owned device buffers.  Library scratch per product: the operand planes, 32 (MK + KN) B
 * (SIMT engine and PAIR modes), plus for the tensor-core engine the limb tiles of both parties,
 * 40 (M' Kpad + Kpad N') B (5 terms x 8 limb bytes; Kpad = 32 ceil(K/32), M' and N' rounded
 * up to the tile).  In MPC_MODE_BOTH the masking is fused into the limb tiling and only the
 * limb tiles are kept. */
mpc_status mpc_matmul(mpc_ctx* ctx, mpc_shares x, mpc_shares y, mpc_shares z, int64_t batch,
                      int64_t M, int64_t K, int64_t N, int64_t batch_off, int trunc_bits);
/* S5 local truncation: z_i = (int64)x_i >> bits, bits in [0,63].
 * No step, no communication. */
mpc_status mpc_trunc(mpc_ctx* ctx, mpc_shares x, mpc_shares z, int64_t n, int bits);

/* ---- S7 / S8 ---------------------------------------------------------------- */
/* S7 comparison: z = [x < 0] as a scale-1 arithmetic
 * sharing; exactly bit (window-1) of rec(x), so correct for rec(x) in
 * [-2^(window-1), 2^(window-1)) (HummingBird window).  window in [1,64].
 * 1 step; 2 + ceil(log2(window-1)) rounds. */
mpc_status mpc_cmp(mpc_ctx* ctx, mpc_shares x, mpc_shares z, int64_t n, int64_t off, int window);
/* S8 ReLU: z = BM(x, 1 - ltz(x)), exact (no truncation).  2 steps. */
mpc_status mpc_relu(mpc_ctx* ctx, mpc_shares x, mpc_shares z, int64_t n, int64_t off, int window);

/* ---- S10 - S13 ------------------------------------------------------------------ */
/* exp-limit knobs: t in [0,8]; clamp 0|1; window of the clamp comparison;
 * square 0|1: squarings with square-pair triples (NEXT #2) instead of Beaver
 * triples -- a different (cheaper) protocol with its own output shares. */
typedef struct { int t; int clamp; int window; int square; } mpc_exp_p;
typedef struct { int iters; mpc_exp_p exp; } mpc_nr_p;       /* iters in [1,12]          */

/* S10 exp-limit: (1 + x/2^t)^(2^t), zeroed below -2^t when clamp.
 * Steps t + 2*clamp. */
mpc_status mpc_exp(mpc_ctx* ctx, mpc_shares x, mpc_shares z, int64_t n, int64_t off,
                   const mpc_exp_p* p);
/* S11 Newton-Raphson reciprocal. Steps exp + 2*iters. */
mpc_status mpc_recip(mpc_ctx* ctx, mpc_shares x, mpc_shares z, int64_t n, int64_t off,
                     const mpc_nr_p* p);
/* S12 Newton-Raphson inverse square root. Steps exp + 3*iters. */
mpc_status mpc_rsqrt(mpc_ctx* ctx, mpc_shares x, mpc_shares z, int64_t n, int64_t off,
                     const mpc_nr_p* p);

typedef enum { MPC_FORM_POLY_X = 0, MPC_FORM_POLY_ABS = 1, MPC_FORM_RELU = 2, MPC_FORM_ERF = 3 } mpc_act_form;
/* The segment table of S13: inside [-B, B) the value is
 * the form's polynomial, outside its asymptote.  coeffs: HOST array of degree+1
 * doubles, low -> high (POLY_X / POLY_ABS); erf_terms K in [2,12] for ERF.
 * basis: 0 Horner; 1 power basis (NEXT #2: v^2, then v^3 and v^4 in
 * one round; POLY_X / POLY_ABS only) -- its own output shares, the same step count. */
typedef struct {
    int form; int degree; double B; const double* coeffs; int erf_terms; int window; int basis;
} mpc_act_p;
/* S13 GELU: POLY_X steps 2+(d-1)+2, POLY_ABS 3+1+(d-1)+2, ERF 2+1+(K-2)+1+1+2,
 * RELU or degree 0: 2. */
mpc_status mpc_gelu(mpc_ctx* ctx, mpc_shares x, mpc_shares z, int64_t n, int64_t off,
                    const mpc_act_p* p);
/* S13 SiLU: forms POLY_X, POLY_ABS, RELU. */
mpc_status mpc_silu(mpc_ctx* ctx, mpc_shares x, mpc_shares z, int64_t n, int64_t off,
                    const mpc_act_p* p);
/* S13 Sigmoid: forms POLY_X, RELU (unit step); tail is the public 1 (R30). */
mpc_status mpc_sigmoid(mpc_ctx* ctx, mpc_shares x, mpc_shares z, int64_t n, int64_t off,
                       const mpc_act_p* p);

/* ---- S9 ---------------------------------------------------------------------------- */
/* S9 row max: x is rows x cols, z is rows; exact.
 * 2 * ceil(log2(cols)) steps. */
mpc_status mpc_max(mpc_ctx* ctx, mpc_shares x, mpc_shares z, int64_t rows, int64_t cols,
                   int64_t row_off, int window);
/* S9 MaxPool2d over NCHW (public zero padding, R26); z is N x C x Ho x Wo.
 * img_off = global index of the first image.  2 * ceil(log2(k*k)) steps. */
mpc_status mpc_maxpool2d(mpc_ctx* ctx, mpc_shares x, mpc_shares z, int N, int C, int H, int W,
                         int k, int stride, int pad, int64_t img_off, int window);

/* ---- S14 / S15 ---------------------------------------------------------------------- */
/* bcast: 0 the final e * r with per-element Beaver triples; 1 with the broadcast
 * triple of mpc_mul_bcast (NEXT #2) -- its own output shares, same steps. */
/* causal: 0 dense; 1 causal attention (reading R24c): the rows are T x T score
 * blocks with T = cols and global row g attends to columns j <= g mod T; masked entries enter the
 * max as the public -2^(window-2), their exponentials and outputs are the public 0 (both shares
 * 0).  Same units and steps as dense.  mpc_plain_eval: row r of the call sees columns <= r mod cols. */
typedef struct { int window; mpc_exp_p exp; mpc_nr_p recip; int bcast; int causal; } mpc_softmax_p;
/* S14 softmax over rows (P:604 footnote).  Steps: 2*levels(cols) + exp +
 * recip + 1.  The library allocates row scratch on the context's device. */
mpc_status mpc_softmax(mpc_ctx* ctx, mpc_shares x, mpc_shares z, int64_t rows, int64_t cols,
                       int64_t row_off, const mpc_softmax_p* p);
/* S14 over HOST buffers (pinned for overlap): hx / hz carry host pointers (rows x cols per
 * party).  The rows are processed in chunks of chunk_rows (multiple of 32; 0 = four equal
 * chunks): chunk i is copied in
 * on one stream, computed on its own stream with its own staging and scratch, and copied out on
 * a third, so both PCIe directions overlap each other and the compute.  The same steps, units
 * and output shares as mpc_softmax on the same rows; completes in the ctx stream's order. */
mpc_status mpc_softmax_hostio(mpc_ctx* ctx, mpc_shares hx, mpc_shares hz, int64_t rows, int64_t cols,
                              int64_t row_off, const mpc_softmax_p* p, int64_t chunk_rows);
typedef struct { double eps; int mean_mode; mpc_nr_p rsqrt; int bcast; } mpc_ln_p;   /* bcast as softmax */
/* S15 layernorm over rows, without the public affine.
 * mean_mode 0: x E(1/d) (SPEC); 1: per-share floor division by d (R25).
 * Steps 1 + rsqrt + 1. */
mpc_status mpc_layernorm(mpc_ctx* ctx, mpc_shares x, mpc_shares z, int64_t rows, int64_t cols,
                         int64_t row_off, const mpc_ln_p* p);

/* ---- NEXT #4: the auto-tuner's evaluator ---------------------------------------------- */
/* Plaintext fixed-point emulation of one approximation schedule, the scoring
 * step of CrypTorch's auto-tuner, which evaluates candidate approximations on a non-MPC runtime
 * (P:237-241).  x, y: DEVICE float64 arrays of rows x cols (rows = 1 for element-wise ops);
 * x is encoded at 2^16 (round half even), the op's schedule runs on the plaintext ring values
 * with floor truncation, y is decoded.  The MPC output differs from it only by the per-share
 * truncation's (-1, 0] ulp per product.  knobs points to the op's knob struct (mpc_exp_p,
 * mpc_nr_p, mpc_act_p, mpc_softmax_p, mpc_ln_p).  No step, no randomness, no communication.
 * x and y must not overlap (MPC_ERR_INVALID).  Bit-exact contract: oracle orc_plain_* (DESIGN.md
 * 2.11; the row max is the schedule's half-split tree with LTZ_w, as in MAX_row). */
typedef enum { MPC_PLAIN_EXP = 0, MPC_PLAIN_RECIP = 1, MPC_PLAIN_RSQRT = 2, MPC_PLAIN_GELU = 3,
               MPC_PLAIN_SILU = 4, MPC_PLAIN_SIGMOID = 5, MPC_PLAIN_SOFTMAX = 6,
               MPC_PLAIN_LAYERNORM = 7 } mpc_plain_op;
mpc_status mpc_plain_eval(mpc_ctx* ctx, int op, const void* knobs, const double* x, double* y,
                          int64_t rows, int64_t cols);

#ifdef __cplusplus
}
#endif
#endif /* MPC200_H */
