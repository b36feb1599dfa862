/*
 * sonic.h -- C ABI of libsonic, a B200 (sm_100a) implementation of the hot path
 * of SonicMoE (arXiv 2512.14080): the forward and backward pass of a
 * fine-grained sparse MoE expert layer.
 *
 * Citations: P:n = line n of the paper text; S:n = SPEC.md line n;
 * Qk = reading k in DESIGN.md section 3.
 *
 * Conventions (all entry points):
 *  - Every tensor pointer is a DEVICE pointer, row-major, caller-allocated and
 *    caller-owned.  bf16 tensors are passed as `const void *` (2-byte elements).
 *  - `stream` is a cudaStream_t passed as `void *` (NULL = legacy default stream).
 *  - sonic_route / sonic_moe_fwd / sonic_moe_bwd are asynchronous on `stream`:
 *    they allocate nothing, never synchronise the host with the device and never
 *    copy device data to the host.  The routed row count R lives on the device
 *    (routing.pad_offsets[E]); buffers are sized with the host-side upper bound
 *    sonic_rows_max().
 *  - Validation is synchronous and happens before any launch: a bad argument
 *    returns SONIC_ERR_INVALID_ARG (or SONIC_ERR_UNSUPPORTED for a legal shape
 *    the kernels do not cover; SONIC_ERR_WORKSPACE for a short workspace) and
 *    launches nothing.  A failed launch returns SONIC_ERR_CUDA.  Device-side
 *    index checks do not exist in release builds.  No C++ exception crosses
 *    the ABI.
 *  - Supported shapes: 1 <= K <= min(E, 16), E <= 4096 (the paper's top-K range,
 *    P:1076), d % 64 == 0, n == 32 or n % 64 == 0, m_tile 128 or 256 (the GEMM M
 *    tile of one CTA or of a 2-CTA pair, P:1238 footnote "M_tile is GPU-dependent", Q16),
 *    rows_max (sonic_rows_max) < 2^31.  All pointers 16-byte aligned.
 *
 * Grouped-row layout.  Expert e owns the grouped rows
 * [pad_offsets[e], pad_offsets[e+1]); the first f_rounded[e] of them hold e's
 * kept tokens in ascending token order (Q17), the rest (< 128, TC mode only)
 * are pad rows with row_token = -1 and row_gate = 0.  pad_offsets[e] is a
 * multiple of 128, so every 128-row GEMM tile belongs to exactly one expert.
 * Under token rounding every f_rounded[e] is a multiple of 128 and there are no
 * pad rows.  All values computed on pad rows are exactly zero.
 */
#ifndef SONIC_H
#define SONIC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SONIC_OK = 0,
  SONIC_ERR_INVALID_ARG = -1,
  SONIC_ERR_UNSUPPORTED = -2,
  SONIC_ERR_WORKSPACE = -3,
  SONIC_ERR_CUDA = -4,
  SONIC_ERR_NCCL = -5
} sonic_status;

typedef enum {
  SONIC_ROUTE_TC = 0,      /* token-choice top-K */
  SONIC_ROUTE_TR_NRF = 1,  /* token rounding, Alg. 4 with NR-f */
  SONIC_ROUTE_GIVEN = 2,   /* arbitrary routing input: S is the gate matrix, t -> e iff
                              the bits of S[t,e] are not +0.0 (a routed pair with a zero gate is
                              passed as -0.0, which sonic_ep_build_plan does), gate = S[t,e] (no
                              renormalisation); topk_ids/topk_s are
                              not written; K may be up to E.  Used by the expert-parallel receive side. */
  /* Token rounding with the other subroutines of the ablation; selection, rescue and
   * gates as for SONIC_ROUTE_TR_NRF. */
  SONIC_ROUTE_TR_UP = 3,       /* always pad: f_r = min(ceil_M(f), T) */
  SONIC_ROUTE_TR_DOWN = 4,     /* always drop: f_r = floor_M(f) */
  SONIC_ROUTE_TR_BALANCE = 5,  /* Balance-f, Alg. 6: sequential residual accumulator */
  SONIC_ROUTE_TR_SR = 6,       /* SR-f: pad with probability (f - floor_M f)/M; the draw of
                                  expert e is SplitMix64 from state (seed << 32 | e), top 24 bits (Q21) */
  SONIC_ROUTE_EC = 7,          /* expert choice (NEXT-3, Q22): each expert keeps its C best tokens,
                                  C = min(ceil_M(ceil(T K / E)), T); no orphan rescue (tokens no expert
                                  chose have no rows and get O = dX = 0) */
  SONIC_ROUTE_TR_NRS = 8       /* NR-s (Q25): pad with probability (sum s - sum floor s) /
                                  (sum ceil s - sum floor s) over Alg. 4's ranking; SR-f's draws (seed) */
} sonic_route_mode;

/* flags */
#define SONIC_F_GATE_RAW         1  /* gate = S_te (no renormalisation over the kept set, Q13) */
#define SONIC_F_NO_ORPHAN_RESCUE 2  /* TR: skip the orphan rescue (Q14) */
#define SONIC_F_BWD_NO_DW        8  /* sonic_moe_bwd part 1: dH, dS, dX only (dW1/dW2 may be NULL);
                                       dH and A' are left in ws */
#define SONIC_F_BWD_DW_ONLY     16  /* sonic_moe_bwd part 2: dW2, dW1 from the dH / A' a preceding
                                       SONIC_F_BWD_NO_DW call left in the same ws (dX/dS may be NULL).
                                       Lets a caller overlap the dX exchange with the weight gradients. */
#define SONIC_F_DW_BF16         32  /* sonic_moe_bwd: dW1 / dW2 are written as bf16 (the float* arguments point
                                       at bf16 [E,d,2n] / [E,n,d] buffers): half the weight-gradient store
                                       traffic; fp32 accumulation as always.  Not with SONIC_F_DW_ACCUMULATE. */
#define SONIC_F_NO_FUSED_UPDOWN 64  /* sonic_moe_fwd: force the up- and down-projection to run as two kernels
                                       with A in the workspace (the default). */
#define SONIC_F_FUSED_UPDOWN   128  /* sonic_moe_fwd: the fused up/down kernel (NEXT-1: A = SwiGLU(H) stays in
                                       shared memory, never written to HBM) where n is 128 or 256 and
                                       d % 128 == 0; sonic_fwd_workspace_size then holds Y only.  Opt-in:
                                       measured slower than the two kernels at 7B. */
#define SONIC_F_FP8_UP         256  /* sonic_moe_fwd: the up-projection on e4m3 operands (NEXT-4, the paper's
                                       FP8 future work P:1553-1556): X quantised per token row and W1 per
                                       output column (sonic_quantize_e4m3_rows / _cols: scale = amax/448 in
                                       fp32, round to nearest even, satfinite), e4m3 x e4m3 -> fp32 tensor-core
                                       sums (tcgen05 kind::f8f6f4), H = sum * sx[t] * sw[e][c], then the
                                       usual SwiGLU epilogue (H, A in bf16).  Everything else stays bf16;
                                       the backward differentiates the quantised forward through the
                                       cached H.  Needs n % 128 == 0 and d % 128 == 0 (else
                                       SONIC_ERR_UNSUPPORTED); the fwd workspace then also holds the e4m3
                                       copies and scales.  Not with the fused up/down kernel. */
#define SONIC_F_FP8_W1_CACHED  512  /* with SONIC_F_FP8_UP: the e4m3 copy of W1 and its scales in the fwd
                                       workspace are still valid (a previous sonic_moe_fwd with the same W1
                                       and this workspace wrote them, e.g. the earlier micro-batches of a
                                       gradient-accumulation step): only X is quantised.  The caller
                                       guarantees it; stale weights are not detected. */
#define SONIC_F_FP8_DXT       1024  /* sonic_moe_bwd: dX~ = dH W1_e^T on e4m3 operands (NEXT-4, reading Q25):
                                       W1 quantised per output column exactly as SONIC_F_FP8_UP does (with
                                       SONIC_F_FP8_W1_CACHED: the copy in THIS bwd workspace is reused), the
                                       stored bf16 dH multiplied by those column scales in fp32 and quantised
                                       per row, dX~ = (e4m3 x e4m3 -> fp32 sum) * row scale; dH, dS, dW1, dW2
                                       stay bf16-path results.  Needs n % 64 == 0 and d % 256 == 0 (else
                                       SONIC_ERR_UNSUPPORTED); the bwd workspace then also holds the e4m3
                                       copies and scales.  Not with SONIC_F_BWD_DW_ONLY. */
#define SONIC_F_DW_ACCUMULATE    4  /* sonic_moe_bwd: dW1 += ..., dW2 += ... (fp32 element-wise adds done by
                                       the TMA store unit; one add per element per call, so deterministic)
                                       instead of overwriting -- gradient accumulation over microbatches */

typedef struct {
  int64_t T;           /* tokens in the microbatch */
  int32_t d, n;        /* embedding dim, expert intermediate dim (H has 2n columns: [gate | up], Q1) */
  int32_t E, K;        /* experts, experts per token */
  int32_t m_tile;      /* TR / EC rounding tile: 128 (one CTA's M tile) or 256 (a 2-CTA pair's M tile,
                          Q16): with 256 every expert gets an even number of 128-row tiles, so no
                          pair is half empty (the grouped-row layout stays in 128-row tiles) */
  int32_t route_mode;  /* sonic_route_mode */
  int32_t flags;       /* SONIC_F_* */
  uint32_t seed;       /* SONIC_ROUTE_TR_SR: seed of the rounding draws (ignored otherwise) */
  int64_t rows_cap;    /* SONIC_ROUTE_GIVEN: upper bound on the routed (token, expert) pairs, i.e. the
                          nonzero gates of S (0 = T*K).  Sizes rows_max = rows_cap + E*(m_tile-1) rounded
                          up to m_tile, so the expert-parallel receive side (K = L local experts) does not
                          reserve T*L rows.  The caller guarantees it (more nonzero gates than rows_cap
                          is undefined behaviour); must be 0 for the other modes. */
} sonic_moe_desc;

/* Routing metadata: written by sonic_route, read by sonic_moe_fwd/bwd.
 * Sizes in elements; byte sizes via sonic_routing_sizes().  All device memory. */
typedef struct {
  int32_t *topk_ids;     /* [T,K]  TC choice, value-descending, ties -> lower expert id (Q9) */
  float   *topk_s;       /* [T,K]  the chosen scores */
  int32_t *f;            /* [E]    TC token count per expert (Alg. 4 step (2)) */
  int32_t *f_rounded;    /* [E]    kept count per expert (== f under TC) */
  int32_t *offsets;      /* [E+1]  exclusive prefix of f_rounded */
  int32_t *pad_offsets;  /* [E+1]  exclusive prefix of ceil(f_rounded/128)*128; pad_offsets[E] = R_pad */
  int32_t *row_token;    /* [rows_max] token of each grouped row (the gather map); -1 on pad rows */
  float   *row_gate;     /* [rows_max] gate g_te of each grouped row; 0 on pad rows */
  int32_t *token_rowptr; /* [T+1]  CSR over tokens */
  int32_t *token_rows;   /* [rows_max] grouped rows of each token, expert-ascending (the scatter map) */
  int32_t *tile_expert;  /* [rows_max/128] expert owning each 128-row tile */
  int32_t *num_tiles;    /* [1]    R_pad / 128 */
  int32_t *tile_pairs;   /* [rows_max/128 + 1] 2-CTA schedule: first 128-row tile of each pair of
                            same-expert tiles, bit 31 set when the second tile exists */
  int32_t *num_pairs;    /* [1]    number of tile pairs */
} sonic_routing;

#define SONIC_ROUTING_NFIELDS 14

/* Upper bound on grouped rows (incl. pad rows): min(T*K + E*(max(m_tile,128)-1), E*ceil(T/128)*128),
 * rounded up to a multiple of 128; for SONIC_ROUTE_EC exactly E*ceil_128(C) with the capacity
 * C = min(ceil_m_tile(ceil(T*K/E)), T) (Q22).  Returns -1 on an invalid descriptor. */
int64_t sonic_rows_max(const sonic_moe_desc *desc);

/* Byte size of each sonic_routing field, in declaration order. */
sonic_status sonic_routing_sizes(const sonic_moe_desc *desc, size_t bytes_out[SONIC_ROUTING_NFIELDS]);

size_t sonic_route_workspace_size(const sonic_moe_desc *desc);
size_t sonic_fwd_workspace_size(const sonic_moe_desc *desc);  /* Y [rows_max,d] (bf16), + A [rows_max,n] when the
                                                                up/down projections are not fused */
size_t sonic_bwd_workspace_size(const sonic_moe_desc *desc);  /* dH, A', dX~ (bf16) + dS partials (fp32) */

/* Byte offsets of the named transients inside the fwd / bwd workspace, for
 * inspection by tests: fwd {A, Y}; bwd {dH, A_prime, dXt, dS_part}; bwd e4m3 buffers of
 * SONIC_F_FP8_DXT {dH' codes, dH' row scales, W1 codes, W1 column scales}.  which = 0 (fwd), 1 (bwd)
 * or 2 (bwd fp8).  The fwd A offset is SIZE_MAX when the up/down projections are fused (A is never
 * materialised); the which = 2 offsets are SIZE_MAX without SONIC_F_FP8_DXT. */
sonic_status sonic_workspace_offsets(const sonic_moe_desc *desc, int which, size_t offs_out[4]);

/*
 * sonic_route -- router top-K, counts, token rounding and the index build
 * (Alg. 4; TC routing P:358; "routing metadata computation" P:944).
 *   S      [T,E] fp32 router scores (softmax probabilities; router GEMM and softmax
 *          are the caller's, P:284 footnote).  Finite values only (Q24).  TR needs
 *          the full S, not only the top-K entries (Q10).
 *   out    routing metadata, every field written (rows past pad_offsets[E] untouched).
 * Integer outputs are deterministic and equal the fp64 oracle's bit for bit.
 * Gate: g_te = S_te / sum_{e' kept for t} S_te' (fp32, ascending-e sum), or S_te
 * with SONIC_F_GATE_RAW.
 */
sonic_status sonic_route(const sonic_moe_desc *desc, const float *S, sonic_routing *out,
                         void *ws, size_t ws_bytes, void *stream);

/*
 * sonic_route_given_capped -- SONIC_ROUTE_GIVEN routing whose routed pairs may exceed the descriptor's
 * rows_cap (the host-sync-free expert-parallel receive side, NEXT-2, sizes its buffers from a
 * capacity instead of the exact received count).  Counts the pairs first; within rows_cap it is
 * exactly sonic_route and *overflow = 0; beyond it the routing is made EMPTY (no rows: nothing is
 * written out of bounds and the GEMMs / aggregation of that step do nothing) and *overflow = 1 --
 * the caller must treat the step as invalid (re-run it with exact sizing).  overflow: device int.
 */
sonic_status sonic_route_given_capped(const sonic_moe_desc *desc, const float *S, sonic_routing *out, void *ws,
                                      size_t ws_bytes, int *overflow, void *stream);

/*
 * sonic_route_logits -- sonic_route with the router softmax fused in ("an optional softmax
 * fusion ... within the top-K kernel"; SURVEY 8(b) SONIC_F_FUSED_SOFTMAX).
 *   logits [T,E] fp32 router logits (finite, Q24), read once.
 *   S_out  [T,E] fp32 output: S_t = softmax(logits_t) per token, computed in fp32 -- max-subtracted
 *          expf, the sum over each lane's experts in order then a fixed butterfly across the warp,
 *          IEEE division (deterministic; within (E + 64) * 2^-24 relative of the exact softmax).
 *          It is the S of sonic_route / sonic_router_bwd: keep it for the backward.
 *   out    as sonic_route; the routing is exactly sonic_route(desc, S_out) (bit for bit).
 * Under TC with E % 32 == 0 and E <= 128 the softmax runs inside the warp-per-token top-K kernel
 * (logits in, S out, no extra pass); otherwise a row-softmax kernel writes S_out first (same
 * arithmetic).  Not for SONIC_ROUTE_GIVEN (SONIC_ERR_INVALID_ARG).  logits and S_out must not alias.
 */
sonic_status sonic_route_logits(const sonic_moe_desc *desc, const float *logits, float *S_out,
                                sonic_routing *out, void *ws, size_t ws_bytes, void *stream);

/*
 * sonic_moe_fwd -- Alg. 2: up-proj A kernel (gather fused, SwiGLU
 * epilogue), down-proj Y kernel (gate applied in the epilogue, Q2), expert
 * aggregation O kernel (gather-and-sum, no atomics).
 *   X  [T,d] bf16;  W1 [E,d,2n] bf16;  W2 [E,n,d] bf16;  rt from sonic_route.
 *   O        [T,d] bf16 output.
 *   H_cache  [rows_max,2n] bf16 output: H = X_e W1_e per grouped row, the only
 *            activation kept for the backward (section 3.2).
 */
sonic_status sonic_moe_fwd(const sonic_moe_desc *desc, const void *X, const void *W1, const void *W2,
                           const sonic_routing *rt, void *O, void *H_cache,
                           void *ws, size_t ws_bytes, void *stream);

/*
 * sonic_moe_bwd -- Alg. 3 + Alg. 5: dH kernel (gather
 * of dO fused; epilogue recomputes A from H, applies dSwiGLU, writes dH, A' and
 * dS = <dA', A>), dW2 = A'^T dO_e, dX~ = dH W1_e^T, dW1 = X_e^T dH,
 * dX aggregation.
 *   dO [T,d] bf16; X, H_cache, W1, W2, rt as in the forward.
 *   dX  [T,d] bf16 output.
 *   dW1 [E,d,2n] fp32, dW2 [E,n,d] fp32 outputs, overwritten (experts with no rows get 0), or
 *       accumulated into with SONIC_F_DW_ACCUMULATE (experts with no rows unchanged), or bf16
 *       buffers of the same shapes with SONIC_F_DW_BF16 (the fp32 result rounded to nearest even).
 *   Split form: SONIC_F_BWD_NO_DW computes dH, dS, dX only (dW1/dW2 may be NULL) and leaves dH, A'
 *       in ws; a following SONIC_F_BWD_DW_ONLY call with the same ws computes dW2, dW1 (dX/dS may
 *       be NULL) -- the expert-parallel path overlaps its dX~ exchange with the second call.
 *   Streams: the dX aggregation may run on an internal side stream forked from and joined back
 *       into `stream` before return (SONIC_BWD_OVERLAP); callers see ordinary stream semantics.
 *   dS  [rows_max] fp32 output: dL/dg for each grouped row (0 on pad rows).  The router
 *       backward (renormalisation/softmax Jacobian) is outside the boundary.
 */
sonic_status sonic_moe_bwd(const sonic_moe_desc *desc, const void *dO, const void *X, const void *H_cache,
                           const void *W1, const void *W2, const sonic_routing *rt,
                           void *dX, float *dW1, float *dW2, float *dS,
                           void *ws, size_t ws_bytes, void *stream);

/*
 * sonic_router_bwd -- NEXT-4: the router's backward from dS to d logits for the routing in rt
 * (the top-K / rounding choice is piecewise constant: no gradient through it).
 *   g_te = S_te / Z_t, Z_t = sum of S over t's kept experts (Q13; g = S with
 *   SONIC_F_GATE_RAW).  dS_full_te = (dS_te - sum_e' dS_te' g_te') / Z_t on kept (t,e), 0 elsewhere;
 *   d logit_tj = S_tj (dS_full_tj - sum_i S_ti dS_full_ti)  (S = softmax(logits) row-wise).
 *   S [T,E] fp32 (the scores sonic_route used); dS [rows_max] fp32 from sonic_moe_bwd;
 *   dlogits [T,E] fp32 output (every entry written; tokens with no expert get 0).
 * Not valid for SONIC_ROUTE_GIVEN (no softmax there): returns SONIC_ERR_INVALID_ARG.
 */
sonic_status sonic_router_bwd(const sonic_moe_desc *desc, const float *S, const sonic_routing *rt,
                              const float *dS, float *dlogits, void *stream);

const char *sonic_status_string(sonic_status s);

/*
 * e4m3 quantisation (NEXT-4, SONIC_F_FP8_UP): one fp32 scale per slice along the reduction dim,
 * scale = amax / 448 (1 where amax = 0), q = cvt.rn.satfinite.e4m3(fl32(x / scale)).
 *   _rows: X [rows, cols] bf16 (cols % 8 == 0, 16-byte aligned) -> q [rows, cols] e4m3, scale [rows]
 *   _cols: W [batch, K, N] bf16 (N % 8 == 0, 16-byte aligned) -> q [batch, K, N] e4m3 (same layout),
 *          scale [batch, N] (per column)
 * Caller-owned device buffers; asynchronous on `stream`.
 */
sonic_status sonic_quantize_e4m3_rows(const void *X, int64_t rows, int32_t cols, void *q, float *scale,
                                      void *stream);
sonic_status sonic_quantize_e4m3_cols(const void *W, int32_t batch, int32_t K, int32_t N, void *q, float *scale,
                                      void *stream);

/*
 * sonic_router_fwd -- the router GEMM before the routing (NEXT-4; the router "computes" the scores,
 * P:284 footnote): logits = X W_r.
 *   X      [T,d] bf16 row-major (the layer input, as sonic_moe_fwd's X)
 *   Wr     [d,E] bf16 row-major router weight
 *   logits [T,E] fp32 output (fp32 accumulation), the input of sonic_route_logits.
 * A plain dense GEMM, run by cuBLAS (cublasGemmEx), loaded with dlopen at first use:
 * SONIC_ERR_UNSUPPORTED if libcublas.so.12 cannot be loaded.  Asynchronous on `stream`.
 */
sonic_status sonic_router_fwd(const sonic_moe_desc *desc, const void *X, const void *Wr, float *logits,
                              void *stream);

/*
 * sonic_router_grad -- the router's share of the input and weight gradients (NEXT-4), from the
 * d logits of sonic_router_bwd (which carries dS through the gate renormalisation and softmax):
 *   dlogits [T,E] fp32; rounded to bf16 in ws for the tensor-core GEMMs (the operand precision
 *           of every GEMM of the layer)
 *   dX      [T,d] bf16 in/out, may be NULL: dX += dlogits W_r^T (pass sonic_moe_bwd's dX to get
 *           the layer's full input gradient; fp32 accumulation, one bf16 rounding)
 *   dWr     [d,E] fp32 out, may be NULL: dWr = X^T dlogits (overwritten)
 *   ws      >= sonic_router_grad_workspace_size(desc) bytes, 16-byte aligned.
 * Both NULL is SONIC_ERR_INVALID_ARG.  cuBLAS as sonic_router_fwd.
 */
size_t sonic_router_grad_workspace_size(const sonic_moe_desc *desc);
sonic_status sonic_router_grad(const sonic_moe_desc *desc, const void *X, const void *Wr, const float *dlogits,
                               void *dX, float *dWr, void *ws, size_t ws_bytes, void *stream);

/* Number of kernels the last sonic_route / sonic_moe_fwd / sonic_moe_bwd / sonic_ep_* compute call on
 * this thread launched. */
int sonic_last_launch_count(void);

/* Optional timing instrumentation (per calling thread).  When enabled, every kernel (the
 * route sequence counts as one record, "route") is bracketed by CUDA events on its stream.
 * sonic_profile_collect synchronises on the recorded events, writes up to max_records
 * (name, milliseconds) pairs -- names as NUL-terminated strings of name_len bytes each --
 * clears the record list and returns the number written. */
void sonic_profile_enable(int on);
int sonic_profile_collect(char *names, int name_len, float *ms, int max_records);

/*
 * ---------------------------------------------------------------- expert parallelism
 * G ranks; rank g owns experts [g*L, (g+1)*L), L = E/G (E % G == 0, G <= 32).  Each rank routes its
 * own T tokens over all E experts with sonic_route; the calls below build and use the dispatch plan
 * of one rank.  The all-to-all itself (NCCL over NVLink) is the caller's (torch.distributed):
 * send row i of the send buffer goes to rank g for send_offsets[g] <= i < send_offsets[g+1].
 * All pointers are device pointers; calls are asynchronous on `stream`; invalid arguments return
 * SONIC_ERR_INVALID_ARG before any launch.
 */
typedef struct {
  int32_t  *dmask;        /* [T]      bit g set when token t has a kept expert on rank g */
  uint32_t *bm;           /* [G, W]   per-rank token bitmaps, W = ceil(T/32) */
  int32_t  *wprefix;      /* [G, W]   exclusive popcount prefix per rank */
  int32_t  *send_counts;  /* [G]      rows sent to each rank (one per token per rank: de-duplicated) */
  int32_t  *send_offsets; /* [G+1]    exclusive prefix of send_counts; send_offsets[G] = rows to send */
  int32_t  *tokcnt;       /* [T]      ranks per token */
  int32_t  *ep_rowptr;    /* [T+1]    CSR over tokens of their send rows (ascending rank) */
  int32_t  *ep_rows;      /* [T*G]    */
  int32_t  *send_token;   /* [T*G]    token of each send row (ascending token within a rank) */
  float    *send_gate;    /* [T*G, L] the token's gates for the destination's L experts, 0 = not routed */
} sonic_ep_plan;
#define SONIC_EP_PLAN_NFIELDS 10

sonic_status sonic_ep_plan_sizes(const sonic_moe_desc *desc, int G, size_t bytes_out[SONIC_EP_PLAN_NFIELDS]);
/* Build the plan from this rank's routing (the sonic_route output for desc). */
sonic_status sonic_ep_build_plan(const sonic_moe_desc *desc, int G, const sonic_routing *rt, sonic_ep_plan *plan,
                                 void *stream);
/* send[i] = src[send_token[i]] for i < send_offsets[G] (src: [T,d] bf16 -- X forward, dO backward). */
sonic_status sonic_ep_pack(const sonic_moe_desc *desc, int G, const sonic_ep_plan *plan, const void *src,
                           void *send, void *stream);
/* out[t] = sum of back[ep_rows[ep_rowptr[t] .. ep_rowptr[t+1])] in ascending rank order, fp32
 * accumulation (back: the returned rows, laid out like the send buffer; out: [T,d] bf16). */
sonic_status sonic_ep_combine(const sonic_moe_desc *desc, int G, const sonic_ep_plan *plan, const void *back,
                              void *out, void *stream);
/* Receive side: dS of the local grouped rows (local desc = GIVEN routing of the received rows over
 * the L local experts) -> dense [rows_in, L] fp32 (zeros where not routed). */
sonic_status sonic_ep_ds_dense(const sonic_moe_desc *local_desc, const sonic_routing *local_rt, const float *dS,
                               float *dense, void *stream);
/* Source side: returned dense dS rows (laid out like the send buffer, [*, L]) -> dS [rows_max] of
 * this rank's routing. */
sonic_status sonic_ep_ds_scatter(const sonic_moe_desc *desc, int G, const sonic_routing *rt,
                                 const sonic_ep_plan *plan, const float *back, float *dS, void *stream);

/*
 * ---------------------------------------------------------------- peer-memory exchange (NEXT-2)
 * The EP all-to-all-v without NCCL (the paper's future work on
 * communication).  Each rank of the group allocates one symmetric region of `bytes` and maps
 * every other rank's region over CUDA IPC (NVLink peer memory on an NVSwitch box).  Kernels store
 * rows straight into the destination rank's region; sonic_peer_barrier orders the phases on the
 * stream (system-scope release/acquire flags), with no host synchronisation.
 * Ownership: sonic_peer_create allocates the region and the flags (cudaMalloc on the current
 * device) and sonic_peer_destroy frees them (it synchronises the device first).  Every rank must
 * issue the same sequence of sonic_peer_barrier calls.  All calls return SONIC_ERR_INVALID_ARG on
 * bad arguments (before any launch) and SONIC_ERR_CUDA on a CUDA failure.
 */
#define SONIC_PEER_MAX 32
#define SONIC_PEER_HANDLE_BYTES 256
typedef struct sonic_peer sonic_peer;
/* Allocate this rank's region and flags; write the exportable handle blob (SONIC_PEER_HANDLE_BYTES
 * bytes) to `handle` -- the caller exchanges the blobs (e.g. all_gather) and passes all of them,
 * rank-ordered, to sonic_peer_open.  Ranks created in the same process (virtual ranks on one GPU,
 * each driving its own stream) are mapped by their raw pointers instead of CUDA IPC. */
sonic_status sonic_peer_create(int rank, int world, size_t bytes, sonic_peer **out, void *handle);
sonic_status sonic_peer_open(sonic_peer *peer, const void *handles /* [world][SONIC_PEER_HANDLE_BYTES] */);
/* Device address of rank r's region as mapped in this process (r == own rank: the own region). */
void        *sonic_peer_base(const sonic_peer *peer, int r);
sonic_status sonic_peer_destroy(sonic_peer *peer);
/* Stream-ordered barrier over the group: the work queued before it on `stream` on every rank
 * (its peer stores) is visible to the work queued after it on every rank. */
sonic_status sonic_peer_barrier(sonic_peer *peer, void *stream);
/* Fused dispatch: send row i of the plan (destination g: send_offsets[g] <= i < send_offsets[g+1])
 * = src[send_token[i]] ([T,d] bf16) is stored as row dst_row0[g] + (i - send_offsets[g]) of the
 * [*, d] bf16 array at byte offset region_off of rank g's region.  dst_row0: HOST array [G] (the
 * rows the lower source ranks put there, from the count matrix).  The caller sizes the regions
 * (capacity T*G rows per source block is always enough). */
sonic_status sonic_ep_pack_peer(const sonic_moe_desc *desc, int G, const sonic_ep_plan *plan, const void *src,
                                const sonic_peer *peer, size_t region_off, const int32_t *dst_row0, void *stream);
/* Block put: rows [src_row0[g], src_row0[g] + cnt[g]) of the device array src (row_bytes each, a
 * multiple of 4; 16-byte vectors when row_bytes, src and region_off allow) to rows [dst_row0[g], ...) of the array at byte offset region_off of rank g's
 * region, for every g < G (= world).  src_row0 / cnt / dst_row0: HOST arrays [G].  Returns
 * SONIC_ERR_INVALID_ARG if a block would end past the region. */
sonic_status sonic_peer_put_rows(const sonic_peer *peer, int G, const void *src, size_t row_bytes,
                                 const int32_t *src_row0, const int32_t *cnt, const int32_t *dst_row0,
                                 size_t region_off, void *stream);

/*
 * Host-sync-free variants (NEXT-2): the block offsets are read on the device from the count matrix
 * at byte offset counts_off of the rank's OWN region (row s = the vector rank s stored in the count
 * exchange; M[s][g] = rows s sends g = the first G of its count_cols int32), so no host read of the
 * counts is needed and the calls can be captured in a CUDA graph.  Same stores as the host-offset
 * versions.
 *   sonic_ep_pack_peer_dev:  dispatch, dst_row0[g] = sum_{s < rank} M[s][g].
 *   sonic_peer_put_rows_dev: direction 0 (dispatch, rank -> g): rows [sum_{g'<g} M[rank][g'],
 *       +M[rank][g]) of src to rows [sum_{s<rank} M[s][g], ...) of rank g; direction 1 (return,
 *       rank = destination, g = source): rows [sum_{s<g} M[s][rank], +M[g][rank]) to rows
 *       [sum_{g'<rank} M[g][g'], ...) of rank g.  The caller sizes the regions for the worst case
 *       (T*G rows per array, as PeerComm does); blocks are not bounds-checked on the host.
 *   sonic_peer_zero_tail: zero rows [R_in, cap_rows) of the own-region array at region_off, R_in =
 *       sum_s M[s][rank] (stale rows of an earlier step past this step's received rows).
 */
sonic_status sonic_ep_pack_peer_dev(const sonic_moe_desc *desc, int G, const sonic_ep_plan *plan, const void *src,
                                    const sonic_peer *peer, size_t region_off, size_t counts_off, int count_cols,
                                    void *stream);
sonic_status sonic_peer_put_rows_dev(const sonic_peer *peer, int G, const void *src, size_t row_bytes, int direction,
                                     size_t counts_off, int count_cols, size_t region_off, void *stream);
sonic_status sonic_peer_zero_tail(const sonic_peer *peer, int G, size_t row_bytes, size_t counts_off, int count_cols,
                                  size_t region_off, long long cap_rows, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SONIC_H */
