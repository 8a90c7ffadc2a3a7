/*
 * atom_oracle.c -- plain, slow, obviously-correct CPU oracle for the Atom W4A4 hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header, table or constant with
 * the CUDA path (paper_2310_19102_b200/csrc); neither side includes or links the other.
 *
 * Paper: Atom, arXiv 2310.19102, /root/reference/PAPER.md ("P:n" = line n).  Readings of places
 * where the paper is silent/ambiguous follow SURVEY.md §8(c) G1-G18 and are listed in DESIGN.md.
 *
 * Steps, in the paper's order:
 *   O2 reorder        x'[j] = X[r][perm[j]]                       P:242 (§4.1), Fig 4 caption P:237
 *   O3 group amax     amax = max_{j in group} |x'_j|                P:118 (§2, symmetric quantization)
 *   O4 scale          s = 2*max|X|*c/(2^n-1), evaluated as
 *                     alpha = RN32(RN32(2c)/RN32(2^n-1)); s = RN32(amax*alpha); s = FLT_MIN if amax==0
 *   O5 code           q = clamp(round_half_even(RN32(x' * RN32(1/s))), -2^(n-1), 2^(n-1)-1)
 *   O6 pack           INT4 two's-complement nibbles, low nibble = even channel; INT8 outliers
 *                     (the last k_o reordered channels, §4.1 mixed precision)
 *   O7 partials       P_t[m][n] = sum_{j in group t} qa*qw  in int64 (Fig 6 Step 1)
 *   O8 output         C[m][n] = sum_t (double)s_a[t][m] * (double)s_w[t][n] * P_t[m][n]
 *                     (Fig 6 Steps 2-3), groups ascending, in double.
 *
 * Group size g = 128 (§4.2 "a group size of 128"); K counts the outlier channels (P:256 fn:
 * 4096 = 3968 normal + 128 outliers).  Groups 0..G4-1 are INT4 (n = 4), group G-1 is the INT8
 * outlier group (n = 8) when k_o == 128 (one scale per token / per output channel).
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC (no -ffast-math: every float op below is
 * a single IEEE-754 binary32 operation in round-to-nearest-even, never contracted into an FMA).
 *
 * Parity pins: see tests/test_oracle_pins.py (P1-P10 of SURVEY §8(c)).  Every function below is
 * pinned; none is "parity unpinned".
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_GROUP 128

/* status codes (independent of the CUDA library's) */
#define ORC_OK 0
#define ORC_ERR_NULL 1
#define ORC_ERR_SHAPE 2
#define ORC_ERR_ARG 4
#define ORC_ERR_OVERFLOW 8

int oracle_version(void) { return 1; }

void oracle_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* O1: validate (SPEC S:152 shape errors, S:186 group divides channels, S:314 split multiple of g) */
static int check_shape(int64_t K, int32_t k_o) {
  if (K <= 0 || K % ORACLE_GROUP != 0) return ORC_ERR_SHAPE;
  if (!(k_o == 0 || k_o == ORACLE_GROUP)) return ORC_ERR_ARG;
  if (K - k_o < 0) return ORC_ERR_SHAPE;
  return ORC_OK;
}

/* O4, first half: alpha = 2c/(2^n - 1) as two rounded binary32 operations. */
static float oracle_alpha(float clip, int nbits) {
  float two_c = 2.0f * clip;                     /* exact: multiplication by 2 */
  float levels = (float)((1 << nbits) - 1);      /* 15 or 255, exact */
  return two_c / levels;                         /* IEEE division, round to nearest even */
}

/* O5: round-half-to-even and clamp to the signed n-bit range. */
static int oracle_code(float x, float inv, int nbits) {
  float v = x * inv;                             /* one IEEE multiply */
  float r = nearbyintf(v);                       /* default rounding mode = ties-to-even */
  float lo = -(float)(1 << (nbits - 1));
  float hi = (float)((1 << (nbits - 1)) - 1);
  if (r < lo) r = lo;
  if (r > hi) r = hi;
  return (int)r;
}

/*
 * O2-O6 for `rows` rows of the row-major fp32 matrix x (row stride ldx).  The values of x are the
 * fp16 inputs converted to fp32 (exact).  Outputs:
 *   q4     uint8 [rows][(K-k_o)/2]   byte b = (q[2b] & 0xF) | (q[2b+1] & 0xF) << 4
 *   q8     int8  [rows][k_o]         (may be NULL iff k_o == 0)
 *   scales fp32  [K/128][rows]       group-major
 * clip4 applies to the INT4 groups, clip8 to the INT8 outlier group (P:299 clip factors).
 */
int oracle_quantize_rows(const float* x, int64_t rows, int64_t ldx, const int32_t* perm, int64_t K,
                         int32_t k_o, float clip4, float clip8, uint8_t* q4, int8_t* q8,
                         float* scales) {
  int st = check_shape(K, k_o);
  if (st) return st;
  if (!x || !perm || !scales || (K - k_o > 0 && !q4) || (k_o > 0 && !q8)) return ORC_ERR_NULL;
  if (!(clip4 > 0.0f && clip4 <= 1.0f) || !(clip8 > 0.0f && clip8 <= 1.0f)) return ORC_ERR_ARG;
  for (int64_t j = 0; j < K; ++j)
    if (perm[j] < 0 || perm[j] >= ldx) return ORC_ERR_ARG;

  const int64_t G = K / ORACLE_GROUP;
  const int64_t G4 = (K - k_o) / ORACLE_GROUP;   /* number of INT4 groups */
  const int64_t row4 = (K - k_o) / 2;            /* bytes per packed INT4 row */

#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r) {
    float xr[ORACLE_GROUP];
    int q[ORACLE_GROUP];
    for (int64_t t = 0; t < G; ++t) {
      const int is_int4 = (t < G4);
      const int nbits = is_int4 ? 4 : 8;
      const float clip = is_int4 ? clip4 : clip8;
      /* O2: reorder (gather by perm) */
      for (int jj = 0; jj < ORACLE_GROUP; ++jj)
        xr[jj] = x[r * ldx + perm[t * ORACLE_GROUP + jj]];
      /* O3: group absolute maximum */
      float amax = 0.0f;
      for (int jj = 0; jj < ORACLE_GROUP; ++jj) {
        float a = fabsf(xr[jj]);
        if (a > amax) amax = a;
      }
      /* O4: scale (degenerate all-zero group -> smallest normal, SURVEY G6 / SPEC S:115) */
      float s = (amax == 0.0f) ? FLT_MIN : amax * oracle_alpha(clip, nbits);
      float inv = 1.0f / s;
      scales[t * rows + r] = s;
      /* O5: codes */
      for (int jj = 0; jj < ORACLE_GROUP; ++jj) q[jj] = oracle_code(xr[jj], inv, nbits);
      /* O6: pack */
      if (is_int4) {
        uint8_t* dst = q4 + r * row4 + t * (ORACLE_GROUP / 2);
        for (int b = 0; b < ORACLE_GROUP / 2; ++b)
          dst[b] = (uint8_t)((q[2 * b] & 0xF) | ((q[2 * b + 1] & 0xF) << 4));
      } else {
        int8_t* dst = q8 + r * k_o;
        for (int jj = 0; jj < ORACLE_GROUP; ++jj) dst[jj] = (int8_t)q[jj];
      }
    }
  }
  return ORC_OK;
}

/*
 * Sum of x_c^2 over fp16-valued x, EXACTLY, rounded once to double (reading G19): an
 * fp16 value is an integer multiple of 2^-24, so x^2 * 2^48 is an integer (< 2^80) and the sum of
 * up to 2^13 of them fits a 128-bit integer; the exact sum is then rounded to the nearest double
 * (the compiler's __int128 -> double conversion, round-to-nearest-even) and scaled by 2^-48
 * (exact).  Order-independent by construction.
 */
static double oracle_sum_squares(const float* x, int64_t C) {
  unsigned __int128 acc = 0;
  for (int64_t c = 0; c < C; ++c) {
    const double v = fabs((double)x[c]) * 16777216.0;   /* |x| * 2^24: an exact integer */
    const unsigned __int128 m = (unsigned __int128)(uint64_t)v;
    acc += m * m;                                      /* x^2 * 2^48, exact */
  }
  return ldexp((double)acc, -48);
}

/*
 * N1 (NEXT-1, the "prior operator" the paper fuses reordering and quantization into: "fuses
 * the activation matrix reordering operators into the prior operator", "we fuse the
 * quantization operator into the prior operator (e.g., LayerNorm)").  The paper does not define
 * the norm; the Llama models it evaluates use RMSNorm (reading G19):
 *     y_c = x_c / sqrt(mean_c(x_c^2) + eps) * gamma_c,   c in [0, C)
 * with the arithmetic pinned as follows (x and gamma are fp16 values widened exactly to fp32):
 *     ss = RN64( sum_c x_c^2 )                   (the exact sum, one rounding: oracle_sum_squares)
 *     r  = RN32( 1.0 / sqrt(ss / C + (double)eps) )   (double ops, one final rounding to fp32)
 *     y_c = RN32( RN32(x_c * r) * gamma_c )      (two binary32 multiplies, in this order)
 * The caller rounds y to fp16 (round-to-nearest-even) before the quantizer, as an fp16 RMSNorm
 * layer followed by a quantized linear layer would.  Output: y32 fp32 [rows][C].
 */
int oracle_rmsnorm_rows(const float* x, int64_t rows, int64_t ldx, int64_t C, const float* gamma,
                        float eps, float* y32) {
  if (!x || !gamma || !y32) return ORC_ERR_NULL;
  if (C <= 0 || C > ldx || !(eps >= 0.0f)) return ORC_ERR_ARG;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r) {
    const float* xr = x + r * ldx;
    const double ss = oracle_sum_squares(xr, C);
    const float rinv = (float)(1.0 / sqrt(ss / (double)C + (double)eps));
    for (int64_t c = 0; c < C; ++c) {
      const float t = xr[c] * rinv;              /* one IEEE multiply */
      y32[r * C + c] = t * gamma[c];             /* one IEEE multiply */
    }
  }
  return ORC_OK;
}

/*
 * The binary32 exponential of the SwiGLU (reading G20), written out operation by
 * operation so that any implementation reproduces it bit for bit (each line one IEEE operation,
 * fmaf = fused multiply-add with one rounding):
 *     x > 88           -> +inf              x < -87 -> 0      (beyond: silu(g) = g or -0 in fp16)
 *     n = rint(x * L2E)                     L2E = 0x3FB8AA3B (log2 e), round half to even
 *     r = fmaf(-n, LN2_HI, x)               LN2_HI = 0x3F317200 (0.693145751953125)
 *     r = fmaf(-n, LN2_LO, r)               LN2_LO = 0x35BFBE8E (1.42860677e-06)
 *     p = 1/720;  p = fmaf(p, r, 1/120);  p = fmaf(p, r, 1/24);  p = fmaf(p, r, 1/6);
 *     p = fmaf(p, r, 1/2);  p = fmaf(p, r, 1);  p = fmaf(p, r, 1)     (Taylor, |r| <= 0.35)
 *     e = p * 2^n                           (ldexpf: exact, normal range)
 * Accurate to a few binary32 ulps of exp(x) on [-87, 88] (pinned against libm's double exp in
 * tests/test_oracle_pins.py).
 */
float oracle_expf_pinned(float x) {
  if (x > 88.0f) return INFINITY;
  if (x < -87.0f) return 0.0f;
  const float L2E = 1.44269502162933349609375f, LN2_HI = 0.693145751953125f;
  const float LN2_LO = 1.428606765330187045037746429443359375e-06f;
  const float n = rintf(x * L2E);
  float r = fmaf(-n, LN2_HI, x);
  r = fmaf(-n, LN2_LO, r);
  float p = 1.0f / 720.0f;
  p = fmaf(p, r, 1.0f / 120.0f);
  p = fmaf(p, r, 1.0f / 24.0f);
  p = fmaf(p, r, 1.0f / 6.0f);
  p = fmaf(p, r, 0.5f);
  p = fmaf(p, r, 1.0f);
  p = fmaf(p, r, 1.0f);
  return ldexpf(p, (int)n);
}

/*
 * N4 (NEXT-4 piece: the down projection's prior operator in a Llama MLP, "we fuse the
 * quantization operator into the prior operator").  The paper does not define the MLP; Llama's is
 * down(silu(gate(x)) * up(x)) (reading G20), with the elementwise step pinned in
 * binary32 as
 *     e_c = oracle_expf_pinned(-g_c)
 *     s_c = RN32( g_c / RN32(1 + e_c) )                        (IEEE add, IEEE division)
 *     h_c = RN32( s_c * u_c )                                  (one binary32 multiply)
 * g and u are the fp16 gate / up outputs widened exactly to fp32; the caller rounds h to fp16
 * (round-to-nearest-even) before the quantizer.  Output: h32 fp32 [rows][C], C = ldx.
 */
int oracle_silu_mul_rows(const float* g, const float* u, int64_t rows, int64_t ldx, float* h32) {
  if (!g || !u || !h32) return ORC_ERR_NULL;
  if (ldx <= 0 || rows < 0) return ORC_ERR_ARG;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t c = 0; c < ldx; ++c) {
      const float gc = g[r * ldx + c];
      const float e = oracle_expf_pinned(-gc);
      const float d = 1.0f + e;                 /* one IEEE add */
      const float s = gc / d;                   /* one IEEE division */
      h32[r * ldx + c] = s * u[r * ldx + c];     /* one IEEE multiply */
    }
  return ORC_OK;
}

/* Decode one signed nibble (two's complement). */
static int oracle_nibble(uint8_t byte, int high) {
  int v = high ? (byte >> 4) & 0xF : byte & 0xF;
  return v >= 8 ? v - 16 : v;
}

/* Reordered code j (0 <= j < K) of one quantized row. */
static int oracle_row_code(const uint8_t* q4row, const int8_t* q8row, int64_t K, int32_t k_o,
                           int64_t j) {
  if (j < K - k_o) return oracle_nibble(q4row[j / 2], (int)(j & 1));
  return (int)q8row[j - (K - k_o)];
}

/* O7 for one (m, n, t): exact integer dot product over group t (Fig 6 Step 1). */
static int64_t oracle_partial(const uint8_t* a_q4, const int8_t* a_q8, const uint8_t* w_q4,
                              const int8_t* w_q8, int64_t K, int32_t k_o, int64_t m, int64_t n,
                              int64_t t) {
  const int64_t row4 = (K - k_o) / 2;
  const uint8_t* a4 = a_q4 ? a_q4 + m * row4 : NULL;
  const uint8_t* w4 = w_q4 ? w_q4 + n * row4 : NULL;
  const int8_t* a8 = a_q8 ? a_q8 + m * k_o : NULL;
  const int8_t* w8 = w_q8 ? w_q8 + n * k_o : NULL;
  int64_t acc = 0;
  for (int64_t j = t * ORACLE_GROUP; j < (t + 1) * ORACLE_GROUP; ++j)
    acc += (int64_t)oracle_row_code(a4, a8, K, k_o, j) * (int64_t)oracle_row_code(w4, w8, K, k_o, j);
  return acc;
}

/*
 * O7: all group partials, int32 [G][M][N].  Returns ORC_ERR_OVERFLOW if any partial does not fit
 * int32 (SPEC S:309 no-overflow invariant; never happens for |q| <= 128 and g = 128).
 */
int oracle_group_partials(const uint8_t* a_q4, const int8_t* a_q8, const uint8_t* w_q4,
                          const int8_t* w_q8, int64_t M, int64_t N, int64_t K, int32_t k_o,
                          int32_t* partials) {
  int st = check_shape(K, k_o);
  if (st) return st;
  if (!partials) return ORC_ERR_NULL;
  const int64_t G = K / ORACLE_GROUP;
  int overflow = 0;
#pragma omp parallel for schedule(static) reduction(| : overflow)
  for (int64_t m = 0; m < M; ++m)
    for (int64_t t = 0; t < G; ++t)
      for (int64_t n = 0; n < N; ++n) {
        int64_t p = oracle_partial(a_q4, a_q8, w_q4, w_q8, K, k_o, m, n, t);
        if (p > INT32_MAX || p < INT32_MIN) overflow = 1;
        partials[(t * M + m) * N + n] = (int32_t)p;
      }
  return overflow ? ORC_ERR_OVERFLOW : ORC_OK;
}

/* O8: C[m][n] = sum_t s_a[t][m] * s_w[t][n] * P_t[m][n] in double, t ascending. */
int oracle_gemm_output(const int32_t* partials, const float* a_scales, const float* w_scales,
                       int64_t M, int64_t N, int64_t G, double* c) {
  if (!partials || !a_scales || !w_scales || !c) return ORC_ERR_NULL;
#pragma omp parallel for schedule(static)
  for (int64_t m = 0; m < M; ++m)
    for (int64_t n = 0; n < N; ++n) {
      double acc = 0.0;
      for (int64_t t = 0; t < G; ++t)
        acc += (double)a_scales[t * M + m] * (double)w_scales[t * N + n] *
               (double)partials[(t * M + m) * N + n];
      c[m * N + n] = acc;
    }
  return ORC_OK;
}

/*
 * O7+O8 for a list of token rows without materialising [G][M][N] partials (used for sampled
 * parity at full BASELINE sizes and for the timed CPU baseline).  Same arithmetic, same order as
 * oracle_group_partials followed by oracle_gemm_output.  a_scales is [G][M] (full M), output
 * c is [n_rows][N].
 */
int oracle_output_rows(const uint8_t* a_q4, const int8_t* a_q8, const float* a_scales,
                       const uint8_t* w_q4, const int8_t* w_q8, const float* w_scales, int64_t M,
                       int64_t N, int64_t K, int32_t k_o, const int64_t* rows, int64_t n_rows,
                       double* c) {
  int st = check_shape(K, k_o);
  if (st) return st;
  if (!rows || !a_scales || !w_scales || !c) return ORC_ERR_NULL;
  const int64_t G = K / ORACLE_GROUP;
  int overflow = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : overflow)
  for (int64_t i = 0; i < n_rows; ++i) {
    const int64_t m = rows[i];
    for (int64_t n = 0; n < N; ++n) {
      double acc = 0.0;
      for (int64_t t = 0; t < G; ++t) {
        int64_t p = oracle_partial(a_q4, a_q8, w_q4, w_q8, K, k_o, m, n, t);
        if (p > INT32_MAX || p < INT32_MIN) overflow = 1;
        acc += (double)a_scales[t * M + m] * (double)w_scales[t * N + n] * (double)(int32_t)p;
      }
      c[i * N + n] = acc;
    }
  }
  return overflow ? ORC_ERR_OVERFLOW : ORC_OK;
}
