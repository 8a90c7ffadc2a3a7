/* kv_oracle.c -- CPU oracle for Atom's quantized KV cache and the dequantize-on-load decode
 * attention (NEXT-3).  TEST INFRASTRUCTURE ONLY: called by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs; the product library never links or calls it.
 *
 * Paper (Section 4.4): "Atom loads the KV-cache in low-bit
 * precision and directly dequantizes it before performing the FP16 calculation"; "Atom uses
 * asymmetric quantization on KV-cache"; "directly applies asymmetric low-bit quantization with
 * the granularity of attention head"; attention: "the Query vector of the incoming token is
 * multiplied by the K cache.  The result is normalized using Softmax and further multiplied with
 * the V cache"; PageAttention for memory management.  Readings (G25-G28):
 *   G25  one (scale, min) pair per (token, head) vector of head_dim values (the only causally
 *        appendable head granularity), INT4 codes in [0, 15], no clipping:
 *          mn = min x, mx = max x;  s = RN32(RN32(mx - mn) / 15);  inv = s > 0 ? RN32(1 / s) : 0
 *          q = clamp(rint_half_even(RN32(RN32(x - mn) * inv)), 0, 15)      (each op one IEEE step)
 *        dequantized value = q * s + mn (a real number; kernels may re-associate it);
 *        codes packed two per byte, low nibble = even dimension;
 *   G26  pages of 16 tokens: page p holds, per head h, tokens [0, 16) of the page contiguously
 *        (codes [page][head][16][head_dim/2], params [page][head][16][2] fp32 (s, mn));
 *        block_table[b][j] = page of tokens [16 j, 16 j + 16) of sequence b; numerics do not
 *        depend on the paging;
 *   G27  decode attention per (sequence b, head h): score_t = sum_i q_i k_ti / sqrt(head_dim)
 *        over the dequantized keys of tokens t < seq_len[b], p = softmax(score), out_i =
 *        sum_t p_t v_ti, all in double here (the GPU computes in fp32);
 *   G28  the query is fp16 (the model's activation precision), the output fp32.
 * Nothing here is shared with the GPU path.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#define KV_OK 0
#define KV_ERR 2
#define KV_PAGE 16

/* G25: quantize `T` token vectors of n_heads x head_dim values (x row-major [T][H][d]) into the
 * paged cache at slots slot[t] (= page * 16 + offset). */
int oracle_kv_quantize(const float* x, int64_t T, int32_t H, int32_t d, const int64_t* slot,
                       uint8_t* codes, float* params) {
  if (d <= 0 || d % 2 != 0 || H <= 0) return KV_ERR;
  for (int64_t t = 0; t < T; ++t) {
    const int64_t page = slot[t] / KV_PAGE, off = slot[t] % KV_PAGE;
    for (int32_t h = 0; h < H; ++h) {
      const float* v = x + (t * H + h) * d;
      float mn = v[0], mx = v[0];
      for (int32_t i = 1; i < d; ++i) {           /* step 1: range of the head vector */
        if (v[i] < mn) mn = v[i];
        if (v[i] > mx) mx = v[i];
      }
      const float range = mx - mn;                /* step 2: scale (binary32, one rounding each) */
      const float s = range / 15.0f;
      const float inv = s > 0.0f ? 1.0f / s : 0.0f;
      const int64_t base = (page * H + h) * KV_PAGE + off;
      params[2 * base] = s;
      params[2 * base + 1] = mn;
      uint8_t* out = codes + base * (d / 2);
      for (int32_t i = 0; i < d; ++i) {           /* step 3: codes */
        const float u = (v[i] - mn) * inv;
        float r = rintf(u);                       /* round half to even (default FE_TONEAREST) */
        if (r < 0.0f) r = 0.0f;
        if (r > 15.0f) r = 15.0f;
        const int q = (int)r;
        if ((i & 1) == 0) out[i / 2] = (uint8_t)q;
        else out[i / 2] = (uint8_t)(out[i / 2] | (q << 4));
      }
    }
  }
  return KV_OK;
}

/* dequantized head vector of token t (of sequence b) into out[d] (double, exact) */
static void kv_dequant(const uint8_t* codes, const float* params, const int32_t* block_table,
                       int64_t max_pages, int64_t b, int64_t t, int32_t H, int32_t h, int32_t d,
                       double* out) {
  const int64_t page = block_table[b * max_pages + t / KV_PAGE], off = t % KV_PAGE;
  const int64_t base = (page * H + h) * KV_PAGE + off;
  const double s = params[2 * base], mn = params[2 * base + 1];
  const uint8_t* c = codes + base * (d / 2);
  for (int32_t i = 0; i < d; ++i) {
    const int q = (i & 1) ? (c[i / 2] >> 4) : (c[i / 2] & 15);
    out[i] = q * s + mn;
  }
}

/* G27: out[b][h][:] (double) for every sequence b < B and head h < H. */
int oracle_decode_attention(const float* q, int64_t B, int32_t H, int32_t d,
                            const uint8_t* k_codes, const float* k_params,
                            const uint8_t* v_codes, const float* v_params,
                            const int32_t* block_table, int64_t max_pages,
                            const int32_t* seq_lens, double* out) {
  if (d <= 0 || d % 2 != 0 || H <= 0) return KV_ERR;
  for (int64_t b = 0; b < B; ++b)
    if (seq_lens[b] <= 0 || seq_lens[b] > max_pages * KV_PAGE) return KV_ERR;
  const double scale = 1.0 / sqrt((double)d);
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int64_t b = 0; b < B; ++b) {
    for (int32_t h = 0; h < H; ++h) {
      const int64_t L = seq_lens[b];
      const float* qv = q + (b * H + h) * d;
      double* kd = (double*)malloc(sizeof(double) * d);
      double* sc = (double*)malloc(sizeof(double) * L);
      double mx = -INFINITY;
      for (int64_t t = 0; t < L; ++t) {           /* scores over the dequantized keys */
        kv_dequant(k_codes, k_params, block_table, max_pages, b, t, H, h, d, kd);
        double acc = 0.0;
        for (int32_t i = 0; i < d; ++i) acc += (double)qv[i] * kd[i];
        sc[t] = acc * scale;
        if (sc[t] > mx) mx = sc[t];
      }
      double den = 0.0;                           /* softmax */
      for (int64_t t = 0; t < L; ++t) {
        sc[t] = exp(sc[t] - mx);
        den += sc[t];
      }
      double* o = out + (b * H + h) * d;
      for (int32_t i = 0; i < d; ++i) o[i] = 0.0;
      for (int64_t t = 0; t < L; ++t) {           /* weighted sum of the dequantized values */
        kv_dequant(v_codes, v_params, block_table, max_pages, b, t, H, h, d, kd);
        const double p = sc[t] / den;
        for (int32_t i = 0; i < d; ++i) o[i] += p * kd[i];
      }
      free(kd);
      free(sc);
    }
  }
  return KV_OK;
}
