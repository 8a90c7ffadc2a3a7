/* mx_oracle.c -- CPU oracle for Atom (FP), the paper's FP4 variant on the MX format (NEXT-2).
 * TEST INFRASTRUCTURE ONLY: called by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs; the product library never links or calls it.
 *
 * Paper: "we also evaluate the effectiveness of Atom in FP4 ... quantizing both weights and
 * activations into FP4" and "group quantization with the MX format is supported by NVIDIA
 * Blackwell GPUs.  We expect this hardware feature can mitigate the group quantization overhead"
 * (Section 6; Table 5 P:527 "Atom (FP)").  The method is Atom's
 * (channel reorder P:242, mixed precision for the outlier channels P:230, fine-grained group
 * quantization P:252) with MX elements and MX block scales.  Readings (G21-G24):
 *   G21  normal channels: MXFP4 = E2M1 elements, blocks of 32 consecutive reordered channels,
 *        one UE8M0 (power-of-two) scale per block and row (the MX block size is 32);
 *   G22  the k_o = 128 outlier channels: MXFP8 = E4M3 elements, blocks of 32, UE8M0 scales;
 *   G23  conversion as written in the OCP Microscaling spec v1.0 (Section 6.3):
 *        shared_exp = floor(log2(amax)) - emax_elem (emax_elem = 2 for E2M1, 8 for E4M3),
 *        clamped to [-127, 127]; amax == 0 -> shared_exp = -127 (UE8M0 byte 0);
 *        element = round-to-nearest-even of x / 2^shared_exp to the element format, saturating
 *        to +-max normal (6 for E2M1, 448 for E4M3); the sign of a zero result is the sign of x;
 *        the clip ratios of the INT path do not apply (power-of-two scales);
 *   G24  output C[m][n] = sum over reordered channels j (ascending) of deq(a[m][j]) * deq(w[n][j])
 *        in double (every product is exact; the GPU sums in its tensor cores' fp32).
 * Each step below is written out in the spec's order; nothing here is shared with the GPU path.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MX_OK 0
#define MX_ERR_SHAPE 2
#define MX_BLOCK 32

/* E2M1 (OCP MX v1.0 Table 1: 1 sign, 2 exponent bits with bias 1, 1 mantissa bit, no inf/nan):
 * code c in [0, 8) -> magnitude; exponent field e = c >> 1, mantissa m = c & 1;
 * e == 0: subnormal m * 2^(1-1) * 0.5 = 0.5 m; e > 0: 2^(e-1) * (1 + m / 2). */
double oracle_e2m1_value(int code) {
  const int c = code & 7, e = c >> 1, m = c & 1;
  const double mag = (e == 0) ? 0.5 * m : ldexp(1.0 + 0.5 * m, e - 1);
  return (code & 8) ? -mag : mag;
}

/* E4M3 (OCP OFP8 E4M3: bias 7, 3 mantissa bits, max normal 448, S.1111.111 = NaN):
 * e == 0: subnormal m * 2^-9; else 2^(e-7) * (1 + m / 8). */
double oracle_e4m3_value(int code) {
  const int c = code & 0x7F, e = c >> 3, m = c & 7;
  const double mag = (e == 0) ? ldexp((double)m, -9) : ldexp(1.0 + m / 8.0, e - 7);
  return (code & 0x80) ? -mag : mag;
}

/* Round-to-nearest-even onto a format given by its ordered non-negative code values
 * 0..ncodes-1 (code value strictly increasing), saturating to the largest. */
static int rne_code(double a, double (*value)(int), int ncodes) {
  if (a >= value(ncodes - 1)) return ncodes - 1;                 /* saturate */
  int lo = 0;
  while (lo + 1 < ncodes && value(lo + 1) <= a) ++lo;             /* value(lo) <= a < value(lo+1) */
  if (value(lo) == a) return lo;
  const double dlo = a - value(lo), dhi = value(lo + 1) - a;
  if (dlo < dhi) return lo;
  if (dhi < dlo) return lo + 1;
  return (lo & 1) ? lo + 1 : lo;                                  /* tie: even mantissa bit */
}

/* x (a finite float) -> E2M1 nibble, RNE with saturation; sign of x kept on zero. */
int oracle_e2m1_code(float x) {
  const int c = rne_code(fabs((double)x), oracle_e2m1_value, 8);
  return c | (signbit(x) ? 8 : 0);
}

/* x -> E4M3 byte, RNE with saturation to 448 (codes 0..0x7E). */
int oracle_e4m3_code(float x) {
  const int c = rne_code(fabs((double)x), oracle_e4m3_value, 0x7F);
  return c | (signbit(x) ? 0x80 : 0);
}

/* OCP MX v1.0 Section 6.3: shared_exp = floor(log2(amax)) - emax_elem, in [-127, 127];
 * returned as the UE8M0 byte (shared_exp + 127).  floor(log2(amax)) from frexp: amax = f 2^E,
 * f in [0.5, 1) -> E - 1 (exact). */
int oracle_mx_scale_byte(float amax, int emax_elem) {
  if (amax == 0.0f) return 0;
  int E;
  (void)frexp((double)amax, &E);
  int se = (E - 1) - emax_elem;
  if (se < -127) se = -127;
  if (se > 127) se = 127;
  return se + 127;
}

/* Reorder (x'[j] = x[perm[j]]) and MX-quantize rows.  fp4: [rows][(K-k_o)/2] packed E2M1
 * (low nibble = even channel), fp8: [rows][k_o] E4M3, sexp: [rows][K/32] UE8M0 bytes (block b
 * covers reordered channels 32b .. 32b+31; the last k_o/32 blocks are the outlier blocks). */
int oracle_mx_quantize_rows(const float* x, int64_t rows, int64_t ldx, const int32_t* perm,
                            int64_t K, int32_t k_o, uint8_t* fp4, uint8_t* fp8, uint8_t* sexp) {
  if (K % 128 != 0 || (k_o != 0 && k_o != 128) || K < k_o) return MX_ERR_SHAPE;
  const int64_t K4 = K - k_o, nb = K / MX_BLOCK;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r) {
    const float* xr = x + r * ldx;
    for (int64_t b = 0; b < nb; ++b) {
      const int64_t j0 = b * MX_BLOCK;
      const int is_fp4 = j0 < K4;
      float amax = 0.0f;                                           /* step 1: block amax */
      for (int64_t j = j0; j < j0 + MX_BLOCK; ++j) {
        const float a = fabsf(xr[perm[j]]);
        if (a > amax) amax = a;
      }
      const int sb = oracle_mx_scale_byte(amax, is_fp4 ? 2 : 8);   /* step 2: shared exponent */
      sexp[r * nb + b] = (uint8_t)sb;
      const double X = ldexp(1.0, sb - 127);
      for (int64_t j = j0; j < j0 + MX_BLOCK; ++j) {               /* step 3: elements */
        const float v = (float)((double)xr[perm[j]] / X);           /* exact: X is 2^k */
        if (is_fp4) {
          const int c = oracle_e2m1_code(v);
          uint8_t* byte = fp4 + r * (K4 / 2) + j / 2;
          if ((j & 1) == 0) *byte = (uint8_t)c;
          else *byte = (uint8_t)(*byte | (c << 4));
        } else {
          fp8[r * k_o + (j - K4)] = (uint8_t)oracle_e4m3_code(v);
        }
      }
    }
  }
  return MX_OK;
}

/* Dequantized reordered row: out[j] = element j * 2^(scale byte of block j/32 - 127). */
static void mx_dequant_row(const uint8_t* q4row, const uint8_t* q8row, const uint8_t* srow,
                           int64_t K, int64_t K4, double* out) {
  for (int64_t j = 0; j < K; ++j) {
    const double X = ldexp(1.0, (int)srow[j / MX_BLOCK] - 127);
    if (j < K4) {
      const uint8_t byte = q4row[j / 2];
      out[j] = X * oracle_e2m1_value((j & 1) ? (byte >> 4) : (byte & 15));
    } else {
      out[j] = X * oracle_e4m3_value(q8row[j - K4]);
    }
  }
}

/* G24: out[i][n] = sum_j deq(a[rows[i]][j]) deq(w[n][j]), j ascending, double. */
int oracle_mx_output_rows(const uint8_t* a4, const uint8_t* a8, const uint8_t* asf,
                          const uint8_t* w4, const uint8_t* w8, const uint8_t* wsf, int64_t M,
                          int64_t N, int64_t K, int32_t k_o, const int64_t* rows, int64_t nrows,
                          double* out) {
  if (K % 128 != 0 || (k_o != 0 && k_o != 128) || K < k_o) return MX_ERR_SHAPE;
  const int64_t K4 = K - k_o, nb = K / MX_BLOCK;
  for (int64_t i = 0; i < nrows; ++i)
    if (rows[i] < 0 || rows[i] >= M) return MX_ERR_SHAPE;
  double* ad = (double*)malloc(sizeof(double) * (size_t)(nrows * K));
  if (!ad) return MX_ERR_SHAPE;
  for (int64_t i = 0; i < nrows; ++i) {
    const int64_t m = rows[i];
    mx_dequant_row(a4 + m * (K4 / 2), a8 + m * k_o, asf + m * nb, K, K4, ad + i * K);
  }
#pragma omp parallel
  {
    double* wd = (double*)malloc(sizeof(double) * (size_t)K);
#pragma omp for schedule(static)
    for (int64_t n = 0; n < N; ++n) {
      mx_dequant_row(w4 + n * (K4 / 2), w8 + n * k_o, wsf + n * nb, K, K4, wd);
      for (int64_t i = 0; i < nrows; ++i) {
        double acc = 0.0;
        for (int64_t j = 0; j < K; ++j) acc += ad[i * K + j] * wd[j];
        out[i * N + n] = acc;
      }
    }
    free(wd);
  }
  free(ad);
  return MX_OK;
}
