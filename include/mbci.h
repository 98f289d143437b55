/*
 * mbci.h — C ABI of the B200-native fused MBCI chain  E = op(A·B)·D.
 *
 * The operation (MCFuser, arXiv 2506.22169; citations are PAPER.md line numbers):
 *   PAPER.md:196 (§III-A, Fig. 3)  "the GEMM chain (C = A×B, E = C×D)" with cross-tile
 *                                  loops m, n, k, h;
 *   PAPER.md:489 (§VI-B1)          batched layouts "(batch, M, K) × (batch, K, N)" then
 *                                  "(batch, M, N) × (batch, N, H)";  this ABI writes L for H;
 *   PAPER.md:498 (§VI-B2)          self-attention: a softmax between the two contractions;
 *   PAPER.md:253 (§III-B)          with K <= 128 the k loop is dead, A is loaded once per
 *                                  CTA and C never leaves the chip (one fused kernel);
 *   PAPER.md:426-441 (Table II)    G3-G6: H (= L) up to 256 and K up to 1024 — larger K runs a
 *                                  live k loop (A and B streamed in 64-column chunks), larger
 *                                  L is cut into <= 128-column h chunks bound to the grid.
 * For every batch index b (b = batch x heads):
 *   C[m,n] = sum_k A[b,m,k] * B[b,k,n]                  (fp32 accumulate)
 *   NONE:    C' = C
 *   SCALE:   C' = scale * C
 *   RELU / GELU: C' = act(scale * C)  (elementwise, R19)
 *   SOFTMAX: C'[m,:] = softmax_n(scale * C[m,:] + mask), mask = -inf for keys
 *            n >= valid_len[b] (KEY_PADDING); a row with no valid key gives E = 0
 *   E[b,m,l] = sum_n C'[m,n] * D[b,n,l]                 (fp32 accumulate, stored as dtype)
 * The readings behind scale / mask / softmax axis are DESIGN.md §2 R1-R4.
 *
 * Conventions: all sizes and strides are int64 ELEMENT counts; pointers are
 * plain host or device pointers as stated per call; no C++ exception crosses
 * the ABI; every call returns an mbci_status_t; a thread-local detail string is
 * available from mbci_last_error().
 */
#ifndef MBCI_H_
#define MBCI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MBCI_ABI_VERSION 1

typedef struct mbci_chain* mbci_chain_t;   /* opaque; created/owned by the library */

typedef enum { MBCI_F32 = 0, MBCI_F16 = 1, MBCI_BF16 = 2 } mbci_dtype_t;
/* Inter-GEMM op on C = A·B: NONE C, SCALE s·C, SOFTMAX softmax_n(s·C + mask), and the elementwise
 * activations RELU max(s·C, 0), GELU g(s·C) with g(x) = x/2 (1 + erf(x / sqrt 2)) (the MLP-style
 * chain; R19). */
typedef enum {
  MBCI_OP_NONE = 0,
  MBCI_OP_SCALE = 1,
  MBCI_OP_SOFTMAX = 2,
  MBCI_OP_RELU = 3,
  MBCI_OP_GELU = 4
} mbci_op_t;
/* Masks (bit flags, SOFTMAX only).  KEY_PADDING: keys n >= valid_len[b] get -inf.  CAUSAL: key n
 * is visible to query row m only if n <= m (top-left aligned, as torch SDPA is_causal; DESIGN.md
 * R18).  CAUSAL_KEY_PADDING: both (row limit min(valid_len[b], m + 1)). */
typedef enum {
  MBCI_MASK_NONE = 0,
  MBCI_MASK_KEY_PADDING = 1,
  MBCI_MASK_CAUSAL = 2,
  MBCI_MASK_CAUSAL_KEY_PADDING = 3
} mbci_mask_t;
typedef enum {
  MBCI_OK = 0,
  MBCI_ERR_INVALID = 1,      /* user error: NULL pointer, negative dim, bad enum, missing valid_len */
  MBCI_ERR_UNSUPPORTED = 2,  /* legal but outside this build: K or L > 65536, misaligned TMA strides
                                with no fallback, no sm_100 device */
  MBCI_ERR_CUDA = 3,         /* CUDA runtime / driver failure (detail in mbci_last_error) */
  MBCI_ERR_NOMEM = 4         /* host or device allocation failed */
} mbci_status_t;

/* Problem descriptor.  A, B, D, E share `dtype`; accumulation is fp32.
 * Layouts (row-major inside each batch slice, strides in elements):
 *   A  [batch, M, K]  element (b,m,k) at  b*bs_a + m*ld_a + k
 *   B  b_layout 0: [batch, K, N]  (b,k,n) at b*bs_b + k*ld_b + n
 *      b_layout 1: [batch, N, K]  (b,n,k) at b*bs_b + n*ld_b + k   (attention's K matrix)
 *   D  [batch, N, L]  (b,n,l) at  b*bs_d + n*ld_d + l
 *   E  [batch, M, L]  (b,m,l) at  b*bs_e + m*ld_e + l
 * A stride of 0 means "packed" (ld = inner extent, bs = rows*ld). */
typedef struct {
  int64_t batch, M, N, K, L;
  int32_t dtype;        /* mbci_dtype_t */
  int32_t op;           /* mbci_op_t */
  float scale;          /* SCALE / SOFTMAX multiplier; NaN selects 1/sqrt(K) (DESIGN R1) */
  int32_t mask;         /* mbci_mask_t; any mask only with SOFTMAX */
  int32_t b_layout;     /* 0 or 1, see above */
  int64_t ld_a, ld_b, ld_d, ld_e;
  int64_t bs_a, bs_b, bs_d, bs_e;
  int32_t tune;         /* 0: analytical model picks the plan; 1: also time the top-8 at create;
                           2: PAPER.md Algorithm 1 (mbci_plan_search with GPU timing) at create */
} mbci_chain_desc_t;

/* Hardware description used by the tile selector (Eqs. 2-5). */
typedef struct {
  double W;             /* HBM bandwidth, bytes/s */
  double P;             /* dense 16-bit tensor throughput, FLOP/s */
  int32_t n_sm;         /* streaming multiprocessors */
  int32_t smem_max;     /* max dynamic shared memory per CTA, bytes */
  int32_t tmem_cols;    /* tensor-memory columns per SM (512 on sm_100) */
  double sfu_per_clk_sm;/* ex2 results per clock per SM (16 on sm_100) */
  double clock_hz;      /* SM clock used for the SFU term */
} mbci_hw_t;

/* One candidate plan: the paper's tile sizes (T_M, T_N, T_K, T_H) for the
 * flat expression mh(n(k(L_A,L_B,C_C),L_D,C_E),S_E), plus B200 pipeline parameters and the
 * model terms of Eqs. (2)-(5).  kernel: 4 = persistent ping-pong tcgen05 chain (default for
 * 16-bit inputs: pairs of 128-row Q tiles per CTA, BM = 256, BN = 128, TL = L padded to 16,
 * stages >= 3 when L <= 64; stages >= 4 enables half items for the last partial round),
 * 0 = one tcgen05 CTA per (β, 128-row tile, h-chunk), 2 / 3 = persistent stream-K variants,
 * 1 = SIMT (CUDA cores; fp32 and TMA-illegal strides).  n_block: CTAs (kernel 0/1) or work
 * items (kernels 2-4) of the created plan. */
typedef struct {
  int32_t kernel;
  int32_t BM, BN, TK, TL;   /* T_M, T_N, T_K (= padded K: dead k loop), T_H */
  int32_t stages;           /* B/D shared-memory ring depth */
  int32_t smem_bytes, tmem_cols;
  int64_t n_block;          /* CTAs = batch * l_m * l_h */
  double t_mem, t_comp, alpha, t_estm;   /* PAPER.md Eqs. (3), (4), (5), (2), seconds */
  double t_b200;            /* B200 extension: max(HBM, tensor, SFU) x wave quantisation */
} mbci_plan_t;

/* ---- lifecycle -------------------------------------------------------------------------- */

/* Validate `desc`, pick a plan (tile selector) for `device`, and return a handle.
 * Host-only unless desc->tune == 1 (then it allocates scratch and times candidates on
 * `device`).  Errors: INVALID (NULL, negative dims, bad enums), UNSUPPORTED (K or L > 65536,
 * no legal plan, device is not sm_100), CUDA, NOMEM. */
mbci_status_t mbci_chain_create(const mbci_chain_desc_t* desc, int device, mbci_chain_t* out);

/* As mbci_chain_create with an explicit plan (tests: plan invariance).  Fields used: kernel,
 * BN, TL, stages; the rest is recomputed.  UNSUPPORTED if the plan is illegal for desc. */
mbci_status_t mbci_chain_create_with_plan(const mbci_chain_desc_t* desc, int device,
                                          const mbci_plan_t* plan, mbci_chain_t* out);

/* Enqueue one evaluation of the chain on `stream` (cudaStream_t; NULL = legacy default).
 * A, B, D, E are DEVICE pointers on the handle's device with the descriptor's layout, each
 * 16-byte aligned for the tcgen05 path; E must not alias A, B or D.  valid_len is a DEVICE
 * int32[batch] (required iff mask == KEY_PADDING; values clamp to [0, N]).
 * Asynchronous: no allocation, no host synchronisation.  Degenerate shapes: batch, M or
 * L == 0 launch nothing; N == 0 (or every key masked) writes E = 0; K == 0 treats C as 0.
 * Errors: INVALID (NULL handle/pointers), UNSUPPORTED (misaligned pointer on the tensor-core
 * path), CUDA (launch failure). */
mbci_status_t mbci_chain_run(mbci_chain_t h, const void* A, const void* B, const void* D,
                             void* E, const int32_t* valid_len, void* stream);

/* End-to-end convenience: A, B, D, E and valid_len are HOST pointers (pinned memory gives
 * asynchronous copies).  Copies the inputs to handle-owned device buffers (allocated on
 * first use and kept), runs the chain, copies E back, and returns when E is on the host.
 * The batch is cut into up to 4 chunks pipelined over two handle-owned streams (after the work
 * already queued on `stream`): the H2D copy of one chunk, the kernel of another and the D2H copy
 * of a third overlap.  Same layouts, strides and errors as mbci_chain_run, plus NOMEM. */
mbci_status_t mbci_chain_run_host(mbci_chain_t h, const void* A, const void* B, const void* D,
                                  void* E, const int32_t* valid_len, void* stream);

/* ---- split-N: the key axis n cut into disjoint ranges ---------------------
 * One part of the chain over the keys [key_offset, key_offset + N) of a longer sequence: the
 * handle's desc has N = this part's key count, and B / D point at its first key row.  E receives
 * the part's own result (softmax normalised over ITS keys); for SOFTMAX, lse
 * (DEVICE, fp32 [batch][M] packed, owned by the caller) receives the natural-log row
 * log-sum-exp ln Σ_{n in part} exp(scale · C[m,n]) over the part's unmasked keys (−inf when none).
 * valid_len (KEY_PADDING) counts keys of the FULL sequence; the part sees
 * clamp(valid_len[β] − key_offset, 0, N).  Other ops ignore lse (it may be NULL).  Errors as
 * mbci_chain_run, plus INVALID (SOFTMAX without lse, key_offset < 0 or > 2^31 − 1) and
 * UNSUPPORTED (the causal mask, three-contraction handles, kernel-6 plans). */
mbci_status_t mbci_chain_run_partial(mbci_chain_t h, const void* A, const void* B, const void* D, void* E,
                                     float* lse, const int32_t* valid_len, int64_t key_offset, void* stream);

/* The reduce step of split-N: E[β,m,:] from `parts` partial results over disjoint key ranges,
 * E_parts [parts][batch][M][L] and lse_parts [parts][batch][M] packed (DEVICE; e.g. gathered
 * from the ranks over NCCL), E [batch][M][L] packed (DEVICE, must not alias the parts).
 * SOFTMAX: E = Σ_r w_r E_r / Σ_r w_r with w_r = exp(lse_r − max lse), exact in real arithmetic
 * (each E_r·exp(lse_r) is the part's unnormalised product; a row with no valid key anywhere gives
 * 0).  NONE / SCALE / RELU / GELU: E = Σ_r E_r.  fp32 arithmetic, one rounding to dtype
 * (mbci_dtype_t).  Asynchronous on stream.  INVALID on bad sizes / enums / NULL buffers. */
mbci_status_t mbci_merge_partials(int32_t parts, const void* E_parts, const float* lse_parts, void* E,
                                  int64_t batch, int64_t M, int64_t L, int32_t dtype, int32_t op, void* stream);

/* Free the handle and its device scratch.  The caller must have synchronised every stream
 * the handle ran on.  NULL is a no-op. */
mbci_status_t mbci_chain_destroy(mbci_chain_t h);

/* ---- three-contraction chains (R20) -------------------
 * E3[b,m,h] = sum_l op2(E[b,m,l]) * F[b,l,h] with E = op(A·B)·D as above: a third contraction whose
 * inputs never leave the chip (kernel 0: O -> P2 in tensor memory -> tcgen05.mma with F staged by
 * TMA; H cut into chunks of <= 128 columns on the grid).  op2 in {NONE, SCALE (scale2), RELU, GELU}
 * (activations on scale2 · x; NaN scale2 -> 1).  fp16 / bf16, packed row-major layouts only:
 * A [b,M,K], B [b,K,N] or [b,N,K], D [b,N,L], F [b,L,H], E3 [b,M,H]; 1 <= L <= 128, K, N, L, H
 * multiples of 8 (16-byte TMA rows).  Masks and ops of the first two contractions as mbci_chain_*.
 * The handle is an mbci_chain_t: mbci_chain_plan / describe / destroy apply. */
typedef struct {
  int64_t batch, M, N, K, L, H;
  int32_t dtype, op;
  float scale;
  int32_t mask, b_layout;
  int32_t op2;
  float scale2;
} mbci_chain3_desc_t;
mbci_status_t mbci_chain3_create(const mbci_chain3_desc_t* desc, int device, mbci_chain_t* out);
/* A, B, D, F, E3: DEVICE pointers, 16-byte aligned; valid_len as mbci_chain_run.  Asynchronous. */
mbci_status_t mbci_chain3_run(mbci_chain_t h, const void* A, const void* B, const void* D, const void* F,
                              void* E3, const int32_t* valid_len, void* stream);

/* ---- introspection ---------------------------------------------------------------------- */

/* The chosen plan (copy). */
mbci_status_t mbci_chain_plan(mbci_chain_t h, mbci_plan_t* out);

/* Human-readable plan description into buf (NUL-terminated, truncated to len). */
mbci_status_t mbci_chain_describe(mbci_chain_t h, char* buf, size_t len);

/* Debug tracing (tensor-core path): when buf (DEVICE, >= n_block * 1024 bytes) is non-NULL,
 * every later run writes 128 uint64 per CTA: %globaltimer ns at start / setup / per n-tile
 * pipeline events / epilogue / end, and the SM id.  NULL turns tracing off.  INVALID if
 * the buffer is too small. */
mbci_status_t mbci_chain_set_trace(mbci_chain_t h, void* buf, int64_t cap_bytes);

/* Number of kernel launches one mbci_chain_run performs for this handle (0 or 1). */
int32_t mbci_chain_launches_per_run(mbci_chain_t h);

const char* mbci_status_string(mbci_status_t s);
const char* mbci_last_error(void);   /* thread-local; valid until the next call on this thread */
int32_t mbci_abi_version(void);

/* ---- tile selector (host only; never touches a GPU) ------------------------------------- */

/* PAPER.md Algorithm 1 (§IV-B) over the legal plans of desc on hw: a population of N
 * random candidates, each round ranked by the analytical model (model 0: the paper's t_estm,
 * Eqs. 2-5; 1: the B200 score t_b200), the n best-estimated measured by `measure` (seconds; a
 * plan is measured once), stop when |top1 - best| / best < eps (returning top1, as the paper's
 * pseudocode), else mutate: N draws weighted by 1 / estimate, each moving one tile parameter
 * (BN, TL or the pipeline depth) to an adjacent legal value; the kernel family (the tiling
 * expression) never mutates.  Host only: `measure` decides what a measurement is (GPU timing in
 * mbci_chain_create with tune = 2).  Defaults (params NULL): N 512, n 8, eps 0.01, seed 1,
 * max_rounds 64, model 0.  round_log (optional) receives 3 doubles per round: best estimate,
 * measured top 1, best measured so far.  Errors: INVALID, UNSUPPORTED (no legal plan). */
typedef struct {
  int32_t N, n;
  double eps;
  uint64_t seed;
  int32_t max_rounds, model;
} mbci_search_params_t;
typedef double (*mbci_measure_fn)(const mbci_plan_t* plan, void* user);
typedef struct {
  int32_t rounds, measurements, space_size;
  double best_measured, history_min;
} mbci_search_result_t;
mbci_status_t mbci_plan_search(const mbci_chain_desc_t* desc, const mbci_hw_t* hw,
                               const mbci_search_params_t* params, mbci_measure_fn measure, void* user,
                               mbci_plan_t* best, mbci_search_result_t* result, double* round_log);

/* Rounds and measurements of the Algorithm-1 search a tune = 2 handle ran at create (0, 0 otherwise). */
mbci_status_t mbci_chain_search_stats(mbci_chain_t h, int32_t* rounds, int32_t* measurements);

/* Default B200 hardware description: W and P from MEASURED_PEAKS-style figures, 148 SMs,
 * 232448 B shared memory, 512 TMEM columns, 16 ex2/clk/SM at 1.965 GHz. */
void mbci_hw_default(mbci_hw_t* hw);

/* Enumerate the legal candidate plans for desc on hw (after Rule 3, and the
 * exact SMEM / TMEM budgets that replace Rule 4's estimate), each with its
 * model terms.  Writes at most cap plans; *n_out receives the total count.  INVALID on
 * bad desc; UNSUPPORTED if no plan is legal. */
mbci_status_t mbci_plan_enumerate(const mbci_chain_desc_t* desc, const mbci_hw_t* hw,
                                  mbci_plan_t* plans, int32_t cap, int32_t* n_out);

/* The plan the selector picks without measurement (smallest t_b200; ties -> t_estm). */
mbci_status_t mbci_plan_select(const mbci_chain_desc_t* desc, const mbci_hw_t* hw,
                               mbci_plan_t* out);

/* Paper model terms (Eqs. 2-5) for an arbitrary tile vector of the flat chain schedule
 * mh(n(k(L_A,L_B,C_C),L_D,C_E),S_E) with dead-loop elimination.
 * elem_bytes = s.  Writes {t_mem, t_comp, alpha, t_estm} into out[0..3] and N_block to
 * out[4]. */
mbci_status_t mbci_model_terms(int64_t batch, int64_t M, int64_t N, int64_t K, int64_t L,
                               int64_t TM, int64_t TN, int64_t TK, int64_t TH, int32_t elem_bytes,
                               const mbci_hw_t* hw, double out[5]);

/* The paper's search space for the two-GEMM chain and its pruning funnel (Fig. 7):
 * 26 tiling expressions x tile vectors of multiples of 16, then Rule 1
 * (deduplicate by the sub-tiling expression left after deleting the blockIdx-bound loops m and h,
 * P:285), Rule 2 (drop `kn`-type classes), Rule 3 (padding) and Rule 4 (Eq. 1 over
 * the A, B, C, D, E tiles x elem_bytes > 1.2 shm_max); R21.  Counts
 * are candidates (expression class x tile vector) retained after each rule.  Host only.
 * INVALID on non-positive sizes or a NULL out; UNSUPPORTED if more than 2^30 tile vectors survive
 * Rule 3 (the Rule-4 pass enumerates them). */
typedef struct {
  int32_t expr_raw, expr_rule1, expr_rule2;                 /* tiling expressions / classes */
  int64_t tile_vectors, tile_vectors_rule3, tile_vectors_rule4;
  int64_t raw, after_rule1, after_rule2, after_rule3, after_rule4;
} mbci_funnel_t;
mbci_status_t mbci_prune_funnel(int64_t M, int64_t N, int64_t K, int64_t H, int32_t elem_bytes,
                                int64_t shm_max, mbci_funnel_t* out);

#ifdef __cplusplus
}
#endif
#endif /* MBCI_H_ */
