/*
 * mbci_oracle.c — CPU oracle for the fused MBCI chain E = op(A·B)·D.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_2506_22169_b200/csrc); neither includes the other.
 *
 * What it computes (the plain, UNFUSED definition, in fp64):
 *   PAPER.md:196 (§III-A, Fig. 3): "the GEMM chain (C = A×B, E = C×D)";
 *   PAPER.md:489 (§VI-B1): "(batch, M, K) × (batch, K, N) specifies the size for
 *     the first batch GEMM operator, while (batch, M, N) × (batch, N, H) delineates
 *     the size of the subsequent batch GEMM operator";
 *   PAPER.md:498 (§VI-B2): the self-attention module "includes ... softmax".
 * Fusion (§III-B) only reorders and hoists Load/Compute/Store
 * statements, so in exact arithmetic the fused kernel computes exactly this
 * unfused chain.  The in-between op follows the readings of DESIGN.md §2
 * (scale s, softmax over the key axis n, key-padding mask -> -inf, a fully
 * masked row -> 0, two-pass max-shifted softmax).
 *
 * Steps per batch β and row m (no blocking, no fusion, no reordering):
 *   1. decode every input element exactly to double (own IEEE decoders below);
 *   2. C[n] = sum_{k<K} A[β,m,k] * B[β,k,n]            (B per b_layout)
 *   3. op:  NONE  C'[n] = C[n]
 *           SCALE C'[n] = s*C[n]
 *           RELU  C'[n] = max(s*C[n], 0)              (R19: elementwise inter-ops,
 *           GELU  C'[n] = g(s*C[n]), g(x) = x/2 (1 + erf(x/sqrt 2))   PAPER.md:194)
 *           SOFTMAX z[n] = s*C[n] (or -inf if n >= valid_len[β], or, with the causal
 *                   mask, if n > m — top-left aligned as torch SDPA is_causal; R18,
 *                   SURVEY §8(f) f4 / PAPER.md:194 "more ... operators");
 *                   mu = max_n z[n]; if mu == -inf: C'[n] = 0 for all n;
 *                   else e[n] = exp(z[n]-mu), Z = sum_n e[n], C'[n] = e[n]/Z
 *   4. E[β,m,l] = sum_{n<N} C'[n] * D[β,n,l]
 * oracle_chain3 (R20): a third contraction
 *   5. O2[l] = op2(E[β,m,l])  (NONE, SCALE s2·x, RELU, GELU as in step 3)
 *   6. E3[β,m,h] = sum_{l<L} O2[l] * F[β,l,h]
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { ORC_F32 = 0, ORC_F16 = 1, ORC_BF16 = 2 };
enum { ORC_OP_NONE = 0, ORC_OP_SCALE = 1, ORC_OP_SOFTMAX = 2, ORC_OP_RELU = 3, ORC_OP_GELU = 4 };

/* IEEE 754 binary16: 1 sign, 5 exponent (bias 15), 10 fraction bits. */
double oracle_decode_f16(uint16_t h) {
  int sign = (h >> 15) & 1, e = (h >> 10) & 0x1F, f = h & 0x3FF;
  double v;
  if (e == 0) v = ldexp((double)f, -24);                 /* subnormal: f * 2^-24 */
  else if (e == 31) v = f ? NAN : INFINITY;
  else v = ldexp((double)(1024 + f), e - 25);            /* (1 + f/2^10) * 2^(e-15) */
  return sign ? -v : v;
}

/* bfloat16: 1 sign, 8 exponent (bias 127), 7 fraction bits. */
double oracle_decode_bf16(uint16_t b) {
  int sign = (b >> 15) & 1, e = (b >> 7) & 0xFF, f = b & 0x7F;
  double v;
  if (e == 0) v = ldexp((double)f, -133);                /* f * 2^-7 * 2^-126 */
  else if (e == 255) v = f ? NAN : INFINITY;
  else v = ldexp((double)(128 + f), e - 134);            /* (1 + f/2^7) * 2^(e-127) */
  return sign ? -v : v;
}

/* IEEE 754 binary32: 1 sign, 8 exponent (bias 127), 23 fraction bits. */
double oracle_decode_f32(uint32_t u) {
  int sign = (u >> 31) & 1, e = (u >> 23) & 0xFF;
  uint32_t f = u & 0x7FFFFF;
  double v;
  if (e == 0) v = ldexp((double)f, -149);
  else if (e == 255) v = f ? NAN : INFINITY;
  else v = ldexp((double)(8388608u + f), e - 150);
  return sign ? -v : v;
}

static double elem(const void* p, int dtype, int64_t i) {
  if (dtype == ORC_F32) return oracle_decode_f32(((const uint32_t*)p)[i]);
  if (dtype == ORC_F16) return oracle_decode_f16(((const uint16_t*)p)[i]);
  return oracle_decode_bf16(((const uint16_t*)p)[i]);
}

/* step 1: decode n elements starting at element offset off into double. */
static void decode_span(const void* p, int dtype, int64_t off, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = elem(p, dtype, off + i);
}

/* One output row E[β, m, 0:L] (and optionally the op(C) row C'[0:N]).
 * a: decoded A[β,m,0:K]; b: decoded B[β] (layout as stored); d: decoded D[β]. */
static void chain_row(const double* a, const double* b, const double* d,
                      int64_t N, int64_t K, int64_t L, int op, double s, int b_layout,
                      int64_t vlen, double* C /* scratch [N] */, double* Erow,
                      double* Cprime_out) {
  /* step 2: C[n] = sum_k A[m,k] B[k,n] */
  for (int64_t n = 0; n < N; ++n) {
    double acc = 0.0;
    for (int64_t k = 0; k < K; ++k)
      acc += a[k] * (b_layout == 0 ? b[k * N + n]     /* B[β,k,n] */
                                   : b[n * K + k]);   /* Bᵀ stored as [β,n,k] */
    C[n] = acc;
  }
  /* step 3: op */
  if (op == ORC_OP_SCALE) {
    for (int64_t n = 0; n < N; ++n) C[n] = s * C[n];
  } else if (op == ORC_OP_RELU) {
    for (int64_t n = 0; n < N; ++n) C[n] = (s * C[n] > 0.0) ? s * C[n] : 0.0;
  } else if (op == ORC_OP_GELU) {
    for (int64_t n = 0; n < N; ++n) C[n] = 0.5 * (s * C[n]) * (1.0 + erf((s * C[n]) / sqrt(2.0)));
  } else if (op == ORC_OP_SOFTMAX) {
    double mu = -INFINITY;
    for (int64_t n = 0; n < N; ++n) {
      C[n] = (n < vlen) ? s * C[n] : -INFINITY;
      if (C[n] > mu) mu = C[n];
    }
    if (mu == -INFINITY) {
      for (int64_t n = 0; n < N; ++n) C[n] = 0.0;
    } else {
      double Z = 0.0;
      for (int64_t n = 0; n < N; ++n) { C[n] = (n < vlen) ? exp(C[n] - mu) : 0.0; Z += C[n]; }
      for (int64_t n = 0; n < N; ++n) C[n] = C[n] / Z;
    }
  }
  if (Cprime_out) memcpy(Cprime_out, C, (size_t)N * sizeof(double));
  /* step 4: E[l] = sum_n C'[n] D[n,l] */
  for (int64_t l = 0; l < L; ++l) {
    double acc = 0.0;
    for (int64_t n = 0; n < N; ++n) acc += C[n] * d[n * L + l];
    Erow[l] = acc;
  }
}

static int64_t clamp_vlen(int op, const int32_t* valid_len, int64_t beta, int64_t N) {
  int64_t v = N;
  if (op == ORC_OP_SOFTMAX && valid_len) {
    v = valid_len[beta];
    if (v < 0) v = 0;
    if (v > N) v = N;
  }
  return v;
}

#define ORC_MAX1(x) ((x) > 0 ? (x) : 1)

/*
 * Full chain (rows == NULL: E is [batch, M, L]) or selected rows
 * (rows = nrows pairs (β, m): E is [nrows, L]).  Inputs are packed row-major
 * raw storage bits: A [batch,M,K], B [batch,K,N] (b_layout 0) or [batch,N,K]
 * (b_layout 1), D [batch,N,L].  valid_len: NULL or int32[batch] (only used by
 * SOFTMAX; values clamp to [0, N]).  Cprime: NULL or double[rows, N].
 * Returns 0, or -1 on invalid arguments / allocation failure.
 */
/* the key limit of row m: valid_len (clamped) and, with the causal mask, keys n <= m only */
static int64_t row_limit(int64_t vlen, int causal, int64_t m) {
  return (causal && m + 1 < vlen) ? m + 1 : vlen;
}

int oracle_chain_ex(const void* A, const void* B, const void* D, double* E, int dtype,
                    int64_t batch, int64_t M, int64_t N, int64_t K, int64_t L, int op,
                    double scale, int b_layout, const int32_t* valid_len, int causal,
                    const int64_t* rows, int64_t nrows, int nthreads, double* Cprime);

int oracle_chain(const void* A, const void* B, const void* D, double* E, int dtype,
                 int64_t batch, int64_t M, int64_t N, int64_t K, int64_t L, int op,
                 double scale, int b_layout, const int32_t* valid_len,
                 const int64_t* rows, int64_t nrows, int nthreads, double* Cprime) {
  return oracle_chain_ex(A, B, D, E, dtype, batch, M, N, K, L, op, scale, b_layout, valid_len, 0, rows,
                         nrows, nthreads, Cprime);
}

/* As oracle_chain; causal != 0 adds the causal mask to SOFTMAX (key n visible to row m iff n <= m). */
int oracle_chain_ex(const void* A, const void* B, const void* D, double* E, int dtype,
                    int64_t batch, int64_t M, int64_t N, int64_t K, int64_t L, int op,
                    double scale, int b_layout, const int32_t* valid_len, int causal,
                    const int64_t* rows, int64_t nrows, int nthreads, double* Cprime) {
  if (op != ORC_OP_SOFTMAX) causal = 0;
  if (batch < 0 || M < 0 || N < 0 || K < 0 || L < 0 || nrows < 0) return -1;
  if (dtype < 0 || dtype > 2 || op < 0 || op > 4 || b_layout < 0 || b_layout > 1) return -1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  int err = 0;
  if (!rows) {
    /* all rows: decode each batch slice once, then every row m of it */
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t beta = 0; beta < batch; ++beta) {
      double* a = (double*)malloc((size_t)ORC_MAX1(M * K) * sizeof(double));
      double* b = (double*)malloc((size_t)ORC_MAX1(K * N) * sizeof(double));
      double* d = (double*)malloc((size_t)ORC_MAX1(N * L) * sizeof(double));
      double* C = (double*)malloc((size_t)ORC_MAX1(N) * sizeof(double));
      if (!a || !b || !d || !C) {
#pragma omp atomic write
        err = 1;
      } else {
        decode_span(A, dtype, beta * M * K, M * K, a);
        decode_span(B, dtype, beta * K * N, K * N, b);
        decode_span(D, dtype, beta * N * L, N * L, d);
        int64_t vlen = clamp_vlen(op, valid_len, beta, N);
        for (int64_t m = 0; m < M; ++m)
          chain_row(a + m * K, b, d, N, K, L, op, scale, b_layout, row_limit(vlen, causal, m), C,
                    E + (beta * M + m) * L, Cprime ? Cprime + (beta * M + m) * N : NULL);
      }
      free(a); free(b); free(d); free(C);
    }
  } else {
    /* selected rows: decode the slices each row needs */
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t r = 0; r < nrows; ++r) {
      int64_t beta = rows[2 * r], m = rows[2 * r + 1];
      double* a = (double*)malloc((size_t)ORC_MAX1(K) * sizeof(double));
      double* b = (double*)malloc((size_t)ORC_MAX1(K * N) * sizeof(double));
      double* d = (double*)malloc((size_t)ORC_MAX1(N * L) * sizeof(double));
      double* C = (double*)malloc((size_t)ORC_MAX1(N) * sizeof(double));
      if (!a || !b || !d || !C || beta < 0 || beta >= batch || m < 0 || m >= M) {
#pragma omp atomic write
        err = 1;
      } else {
        decode_span(A, dtype, (beta * M + m) * K, K, a);
        decode_span(B, dtype, beta * K * N, K * N, b);
        decode_span(D, dtype, beta * N * L, N * L, d);
        chain_row(a, b, d, N, K, L, op, scale, b_layout,
                  row_limit(clamp_vlen(op, valid_len, beta, N), causal, m), C, E + r * L,
                  Cprime ? Cprime + r * N : NULL);
      }
      free(a); free(b); free(d); free(C);
    }
  }
  return err ? -1 : 0;
}

/* Row log-sum-exp of the SOFTMAX op (the statistic a split-N partial result carries, SURVEY §8(f)
 * f1): lse[β, m] = ln Σ_{n < v} exp(scale · C[m, n]) with C = A·B (step 2) and v the clamped
 * valid_len (all N keys when NULL); −inf when v = 0.  Two-pass stable evaluation
 * μ + ln Σ exp(z − μ), as chain_row's softmax.  lse is [batch, M].  Returns 0 or -1. */
int oracle_row_lse(const void* A, const void* B, double* lse, int dtype, int64_t batch, int64_t M,
                   int64_t N, int64_t K, double scale, int b_layout, const int32_t* valid_len,
                   int nthreads) {
  if (batch < 0 || M < 0 || N < 0 || K < 0 || dtype < 0 || dtype > 2 || b_layout < 0 || b_layout > 1) return -1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  int err = 0;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t beta = 0; beta < batch; ++beta) {
    double* a = (double*)malloc((size_t)ORC_MAX1(M * K) * sizeof(double));
    double* b = (double*)malloc((size_t)ORC_MAX1(K * N) * sizeof(double));
    double* z = (double*)malloc((size_t)ORC_MAX1(N) * sizeof(double));
    if (!a || !b || !z) {
#pragma omp atomic write
      err = 1;
    } else {
      decode_span(A, dtype, beta * M * K, M * K, a);
      decode_span(B, dtype, beta * K * N, K * N, b);
      const int64_t v = clamp_vlen(ORC_OP_SOFTMAX, valid_len, beta, N);
      for (int64_t m = 0; m < M; ++m) {
        double mu = -INFINITY;
        for (int64_t n = 0; n < v; ++n) {
          double acc = 0.0;
          for (int64_t k = 0; k < K; ++k) acc += a[m * K + k] * (b_layout == 0 ? b[k * N + n] : b[n * K + k]);
          z[n] = scale * acc;
          if (z[n] > mu) mu = z[n];
        }
        if (mu == -INFINITY) {
          lse[beta * M + m] = -INFINITY;
        } else {
          double Z = 0.0;
          for (int64_t n = 0; n < v; ++n) Z += exp(z[n] - mu);
          lse[beta * M + m] = mu + log(Z);
        }
      }
    }
    free(a); free(b); free(z);
  }
  return err ? -1 : 0;
}

/* Three-contraction chain: E3 [batch, M, H] = op2(op(A·B)·D) · F, F [batch, L, H] packed row-major
 * storage bits; op2 in {NONE, SCALE, RELU, GELU} with scale2; the rest as oracle_chain_ex.
 * Plain and unfused: the two-contraction row of steps 1-4, then steps 5-6 per row. */
int oracle_chain3(const void* A, const void* B, const void* D, const void* F, double* E3, int dtype,
                  int64_t batch, int64_t M, int64_t N, int64_t K, int64_t L, int64_t H, int op,
                  double scale, int b_layout, const int32_t* valid_len, int causal, int op2, double scale2,
                  int nthreads) {
  if (batch < 0 || M < 0 || N < 0 || K < 0 || L < 0 || H < 0) return -1;
  if (dtype < 0 || dtype > 2 || op < 0 || op > 4 || b_layout < 0 || b_layout > 1) return -1;
  if (op2 != ORC_OP_NONE && op2 != ORC_OP_SCALE && op2 != ORC_OP_RELU && op2 != ORC_OP_GELU) return -1;
  if (op != ORC_OP_SOFTMAX) causal = 0;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  int err = 0;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t beta = 0; beta < batch; ++beta) {
    double* a = (double*)malloc((size_t)ORC_MAX1(M * K) * sizeof(double));
    double* b = (double*)malloc((size_t)ORC_MAX1(K * N) * sizeof(double));
    double* d = (double*)malloc((size_t)ORC_MAX1(N * L) * sizeof(double));
    double* f = (double*)malloc((size_t)ORC_MAX1(L * H) * sizeof(double));
    double* C = (double*)malloc((size_t)ORC_MAX1(N) * sizeof(double));
    double* e = (double*)malloc((size_t)ORC_MAX1(L) * sizeof(double));
    if (!a || !b || !d || !f || !C || !e) {
#pragma omp atomic write
      err = 1;
    } else {
      decode_span(A, dtype, beta * M * K, M * K, a);
      decode_span(B, dtype, beta * K * N, K * N, b);
      decode_span(D, dtype, beta * N * L, N * L, d);
      decode_span(F, dtype, beta * L * H, L * H, f);
      int64_t vlen = clamp_vlen(op, valid_len, beta, N);
      for (int64_t m = 0; m < M; ++m) {
        chain_row(a + m * K, b, d, N, K, L, op, scale, b_layout, row_limit(vlen, causal, m), C, e, NULL);
        for (int64_t l = 0; l < L; ++l) {       /* step 5 */
          double x = e[l];
          if (op2 == ORC_OP_SCALE) x = scale2 * x;
          else if (op2 == ORC_OP_RELU) x = (scale2 * x > 0.0) ? scale2 * x : 0.0;
          else if (op2 == ORC_OP_GELU) x = 0.5 * (scale2 * x) * (1.0 + erf((scale2 * x) / sqrt(2.0)));
          e[l] = x;
        }
        for (int64_t hh = 0; hh < H; ++hh) {    /* step 6 */
          double acc = 0.0;
          for (int64_t l = 0; l < L; ++l) acc += e[l] * f[l * H + hh];
          E3[(beta * M + m) * H + hh] = acc;
        }
      }
    }
    free(a); free(b); free(d); free(f); free(C); free(e);
  }
  return err ? -1 : 0;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Decode n storage elements to double with the decoders above (step 1). */
int oracle_decode_array(const void* p, int dtype, int64_t n, double* out) {
  if (dtype < 0 || dtype > 2 || n < 0) return -1;
  decode_span(p, dtype, 0, n, out);
  return 0;
}
