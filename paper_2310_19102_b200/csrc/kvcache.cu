// kvcache.cu -- NEXT-3: Atom's quantized KV cache and the dequantize-on-load decode attention.
//
// Paper (Section 4.4): "Atom loads the KV-cache in low-bit precision and directly
// dequantizes it before performing the FP16 calculation"; "asymmetric quantization ... with the
// granularity of attention head"; the query is multiplied by the K cache, normalised by softmax
// and multiplied with the V cache; PageAttention manages the memory.  Readings G25-G28
// (DESIGN.md): one (scale, min) per (token, head) vector, INT4 codes in [0, 15], 16-token pages.
//
// B200 design: decode attention is HBM-bound (each cached byte is used once per step); every
// token-head vector is 64 bytes of codes + 8 bytes of (s, mn).  Split-K ("flash decoding"): a CTA
// of 4 warps handles one (sequence, head, chunk of tokens); a warp takes 8 tokens at a time,
// 4 lanes per token, each lane 32 dimensions = one 16-byte load of codes, so a warp reads 8
// tokens' 64-byte vectors of one page as 512 contiguous bytes.  The dequantization is folded
// algebraically (sum_i q_i (c_i s + mn) = s sum_i q_i c_i + mn sum_i q_i; sum_t p_t (c_t s + mn)
// = sum_t (p_t s) c_t + sum_t p_t mn_t), so the inner loops are one code extraction and one FMA
// per element.  Scores of the chunk are kept in shared memory (exact two-pass softmax inside the
// chunk); chunks are merged by a small combine kernel (log-sum-exp).
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "internal.h"
#include "ptx.cuh"

namespace atom {

constexpr int kKvPage = 16;
constexpr int kKvD = 128;                 // head dimension of the kernels (Llama)
constexpr int kAttThreads = 128;
constexpr int kMaxChunk = 1024;           // tokens per CTA (scores in shared memory)

// ---------------------------------------------------------------------------------------------
// quantize: one warp per (token, head) vector, a lane owns 4 dimensions
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
kv_quantize_kernel(const __half* __restrict__ x, int64_t T, int64_t ldx, int32_t H,
                   const int32_t* __restrict__ slots, uint8_t* __restrict__ codes,
                   float* __restrict__ params) {
  griddep_wait();
  griddep_launch();
  const int lane = threadIdx.x % 32;
  const int64_t nvec = T * H;
  for (int64_t v = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32; v < nvec;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x / 32) {
    const int64_t t = v / H;
    const int h = static_cast<int>(v % H);
    const uint2 raw = *reinterpret_cast<const uint2*>(x + t * ldx + h * kKvD + 4 * lane);
    const __half2* hp = reinterpret_cast<const __half2*>(&raw);
    const float2 a = __half22float2(hp[0]), b = __half22float2(hp[1]);
    const float xv[4] = {a.x, a.y, b.x, b.y};
    float mn = fminf(fminf(xv[0], xv[1]), fminf(xv[2], xv[3]));
    float mx = fmaxf(fmaxf(xv[0], xv[1]), fmaxf(xv[2], xv[3]));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, off));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    }
    // G25, each step one IEEE operation: s = RN(RN(mx - mn) / 15), inv = RN(1 / s)
    const float s = __fdiv_rn(__fsub_rn(mx, mn), 15.0f);
    const float inv = s > 0.0f ? __frcp_rn(s) : 0.0f;
    uint32_t packed = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float r = fminf(fmaxf(rintf(__fmul_rn(__fsub_rn(xv[k], mn), inv)), 0.0f), 15.0f);
      packed |= static_cast<uint32_t>(r) << (4 * k);
    }
    const int64_t slot = slots[t];
    const int64_t base = ((slot / kKvPage) * H + h) * kKvPage + slot % kKvPage;
    reinterpret_cast<uint16_t*>(codes + base * (kKvD / 2))[lane] = static_cast<uint16_t>(packed);
    if (lane == 0) reinterpret_cast<float2*>(params)[base] = make_float2(s, mn);
  }
}

cudaError_t launch_kv_quantize(const void* x, int64_t T, int64_t ldx, int32_t H,
                               const int32_t* slots, uint8_t* codes, float* params,
                               cudaStream_t stream, int num_sms) {
  int64_t blocks = (T * H * 32 + 255) / 256;
  if (blocks > 16LL * num_sms) blocks = 16LL * num_sms;
  return launch_pdl(kv_quantize_kernel, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, stream,
                    static_cast<const __half*>(x), T, ldx, H, slots, codes, params);
}

// ---------------------------------------------------------------------------------------------
// decode attention
// ---------------------------------------------------------------------------------------------
// The 8 codes of a 32-bit word (dimensions 8j .. 8j+7) as 4 float pairs (dims 2k, 2k+1):
// the even / odd nibbles are split into bytes once, a PRMT places each byte under the exponent
// of 2^23 (0x4B0000nn = 2^23 + n), one FFMA2 subtracts 2^23 (exact).
__device__ __forceinline__ void code_pairs(uint32_t w, float2 (&c)[4]) {
  const uint32_t ev = w & 0x0F0F0F0Fu, od = (w >> 4) & 0x0F0F0F0Fu;
  const float2 one = make_float2(1.0f, 1.0f), off = make_float2(-8388608.0f, -8388608.0f);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t sel = 0x7540u | static_cast<uint32_t>(k);   // byte k of the word, then 0x4B0000
    const float2 f = make_float2(__uint_as_float(__byte_perm(ev, 0x4B000000u, sel)),
                                 __uint_as_float(__byte_perm(od, 0x4B000000u, sel)));
    c[k] = __ffma2_rn(f, one, off);
  }
}

// The nibbles at bits 4i and 4i + 16 of w as an exact half2 (n_lo, n_hi): the nibbles land in
// the low mantissa bits under the exponent of 1024 (0x6400 = 1024 + n), one HSUB2 removes 1024.
__device__ __forceinline__ uint32_t nibble_h2(uint32_t w, int i) {
  uint32_t x = ((w >> (4 * i)) & 0x000F000Fu) | 0x64006400u;
  const __half2 h = __hsub2(*reinterpret_cast<const __half2*>(&x),
                            __half2half2(__ushort_as_half(static_cast<unsigned short>(0x6400))));
  return *reinterpret_cast<const uint32_t*>(&h);
}

// D (16 x 8, fp32) += A (16 x 16, f16, row) * B (16 x 8, f16, col) on the tensor cores
__device__ __forceinline__ void mma_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                          uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// CTA (b, h, chunk): tokens [c0, c1) of sequence b.  splits > 1: writes the chunk's (max, sum,
// unnormalised output) to the workspace; splits == 1: the normalised output.
__global__ void __launch_bounds__(kAttThreads)
decode_attention_kernel(const __half* __restrict__ q, int32_t H,
                        const uint8_t* __restrict__ kc, const float* __restrict__ kp,
                        const uint8_t* __restrict__ vc, const float* __restrict__ vp,
                        const int32_t* __restrict__ block_table, int64_t max_pages,
                        const int32_t* __restrict__ seq_lens, int32_t chunk, int32_t splits,
                        float* __restrict__ out, float* __restrict__ part) {
  __shared__ float sc[kMaxChunk];
  __shared__ float red[kAttThreads / 32][kKvD + 2];
  const int bh = blockIdx.x, split = blockIdx.y;
  const int b = bh / H, h = bh % H;
  griddep_wait();
  griddep_launch();
  const int L = seq_lens[b];
  const int c0 = split * chunk, c1 = min(L, c0 + chunk);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tj = lane >> 2, part4 = lane & 3;         // token slot within 8, dimension quarter
  // sum of q over this lane's 32 dimensions (the (s, mn) form of a dequantized dot product:
  // q . (s n + mn) = s (q . n) + mn sum(q))
  float qsum = 0.0f;
  {
    const __half2* qp = reinterpret_cast<const __half2*>(q + static_cast<int64_t>(bh) * kKvD +
                                                         32 * part4);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float2 f = __half22float2(qp[i]);
      qsum += f.x;
      qsum += f.y;
    }
  }
  constexpr float kRsqrtD = 0.08838834764831845f;     // 1 / sqrt(128)
  const int32_t* bt = block_table + static_cast<int64_t>(b) * max_pages;
  // the 16 tokens t0 .. t0+15 of a warp step lie in one page (t0 % 16 == 0): one table lookup
  auto vec0 = [&](int t0) {                           // (page, head, offset) index of token t0
    return (static_cast<int64_t>(__ldg(bt + t0 / kKvPage)) * H + h) * kKvPage + t0 % kKvPage;
  };
  // q as the B operand of m16n8k16 (column 0 = lanes tj == 0; the other columns zero): k-tile
  // kt = 2 wi + e, slots (2 part4, +1) <-> dims 32 part4 + 8 wi + 2e + (0, 4), slots
  // (2 part4 + 8, +9) <-> dims 32 part4 + 8 wi + 2e + (1, 5) -- the pairs nibble_h2 makes
  uint32_t qb[8][2];
  {
    const __half* qh = q + static_cast<int64_t>(bh) * kKvD + 32 * part4;
#pragma unroll
    for (int wi = 0; wi < 4; ++wi)
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int dm = 8 * wi + 2 * e + r;
          const __half2 v = __halves2half2(qh[dm], qh[dm + 4]);
          qb[2 * wi + e][r] = tj == 0 ? *reinterpret_cast<const uint32_t*>(&v) : 0u;
        }
  }
  float qsum_all = qsum + __shfl_xor_sync(0xffffffffu, qsum, 1);
  qsum_all += __shfl_xor_sync(0xffffffffu, qsum_all, 2);

  // A warp step covers 8 kTpl tokens (kTpl / 2 whole pages): lane (tj, part4) loads dims
  // 32 part4 .. +31 of tokens t0 + 8 u + tj, u < kTpl -- in pass 1 exactly its A fragment of
  // the page's m16n8k16 (rows tj, tj + 8); every step's codes and (s, mn) are loaded one step
  // ahead.
  constexpr int kTpl = 2;     // tokens per lane per step (4: 191.6 vs 183.2 us at B=128 L=1024)
  static_assert(kTpl % 2 == 0, "a warp step covers whole pages");
  constexpr int kStep = 8 * kTpl * (kAttThreads / 32);
  auto load = [&](const uint8_t* codes, const float* prm, int t0, uint4 (&w)[kTpl],
                  float2 (&sm)[kTpl]) {
#pragma unroll
    for (int pg = 0; pg < kTpl / 2; ++pg) {
      const int tp = t0 + 16 * pg;
      if (tp < c1) {
        const int64_t v0 = vec0(tp) + tj;
#pragma unroll
        for (int u = 2 * pg; u < 2 * pg + 2; ++u)
          if (t0 + 8 * u + tj < c1) {
            const int64_t v = v0 + 8 * (u - 2 * pg);
            w[u] = __ldg(reinterpret_cast<const uint4*>(codes + v * (kKvD / 2) + 16 * part4));
            sm[u] = __ldg(reinterpret_cast<const float2*>(prm) + v);
          }
      }
    }
  };

  // ---- pass 1: scores of the chunk into shared memory ----
  float wmax = -INFINITY;
  uint4 wn[kTpl];
  float2 smn[kTpl];
#pragma unroll
  for (int u = 0; u < kTpl; ++u) {
    wn[u] = make_uint4(0, 0, 0, 0);
    smn[u] = make_float2(0.0f, 0.0f);
  }
  load(kc, kp, c0 + 8 * kTpl * warp, wn, smn);
  for (int t0 = c0 + 8 * kTpl * warp; t0 < c1; t0 += kStep) {
    uint4 w[kTpl];
    float2 sm[kTpl];
#pragma unroll
    for (int u = 0; u < kTpl; ++u) {
      w[u] = wn[u];
      sm[u] = smn[u];
    }
    load(kc, kp, t0 + kStep, wn, smn);
    // one m16n8k16 chain per page: A = the page's codes (row = token t0 + 16 pt + tj (+8),
    // k-slots = this lane's dimensions, see qb), B = q in column 0; column 0 of D holds the
    // exact-product fp32 dot products sum_i q_i n_ti of tokens tj and tj + 8 (lanes part4 == 0)
#pragma unroll
    for (int pt = 0; pt < kTpl / 2; ++pt) {
      float d[4] = {0.0f, 0.0f, 0.0f, 0.0f};
      const uint32_t r0[4] = {w[2 * pt].x, w[2 * pt].y, w[2 * pt].z, w[2 * pt].w};
      const uint32_t r1[4] = {w[2 * pt + 1].x, w[2 * pt + 1].y, w[2 * pt + 1].z, w[2 * pt + 1].w};
#pragma unroll
      for (int wi = 0; wi < 4; ++wi) {
#pragma unroll
        for (int e = 0; e < 2; ++e)
          mma_16816(d, nibble_h2(r0[wi], 2 * e), nibble_h2(r1[wi], 2 * e),
                    nibble_h2(r0[wi], 2 * e + 1), nibble_h2(r1[wi], 2 * e + 1), qb[2 * wi + e][0],
                    qb[2 * wi + e][1]);
      }
      if (part4 == 0) {
#pragma unroll
        for (int u2 = 0; u2 < 2; ++u2) {
          const int t = t0 + 16 * pt + 8 * u2 + tj;
          if (t < c1) {
            const float2 m = sm[2 * pt + u2];
            const float score = fmaf(m.x, d[2 * u2], m.y * qsum_all) * kRsqrtD;
            sc[t - c0] = score;
            wmax = fmaxf(wmax, score);
          }
        }
      }
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) wmax = fmaxf(wmax, __shfl_xor_sync(0xffffffffu, wmax, off));
  if (lane == 0) red[warp][0] = wmax;
  __syncthreads();
  float cmax = red[0][0];
#pragma unroll
  for (int w = 1; w < kAttThreads / 32; ++w) cmax = fmaxf(cmax, red[w][0]);
  __syncthreads();

  // ---- pass 2: p_t = exp(score - max), out = sum_t p_t v_t ----
  float acc[32];
  float2* acc2 = reinterpret_cast<float2*>(acc);
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = 0.0f;
  float psum = 0.0f, pmn = 0.0f;                      // sum p_t, sum p_t mn_t (this lane's tokens)
  load(vc, vp, c0 + 8 * kTpl * warp, wn, smn);
  for (int t0 = c0 + 8 * kTpl * warp; t0 < c1; t0 += kStep) {
    uint4 w[kTpl];
    float2 sm[kTpl];
#pragma unroll
    for (int u = 0; u < kTpl; ++u) {
      w[u] = wn[u];
      sm[u] = smn[u];
    }
    load(vc, vp, t0 + kStep, wn, smn);
#pragma unroll
    for (int u = 0; u < kTpl; ++u) {
      const int t = t0 + 8 * u + tj;
      if (t < c1) {
        const float p = __expf(sc[t - c0] - cmax);
        const float ps = p * sm[u].x;
        psum += p;
        pmn = fmaf(p, sm[u].y, pmn);
        const uint32_t ww[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
        const float2 ps2 = make_float2(ps, ps);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float2 c[4];
          code_pairs(ww[i], c);
#pragma unroll
          for (int k = 0; k < 4; ++k) acc2[4 * i + k] = __ffma2_rn(ps2, c[k], acc2[4 * i + k]);
        }
      }
    }
  }
  // reduce over the 8 token slots of the warp (lanes with the same dimension quarter)
#pragma unroll
  for (int off = 4; off < 32; off <<= 1) {
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], off);
    psum += __shfl_xor_sync(0xffffffffu, psum, off);
    pmn += __shfl_xor_sync(0xffffffffu, pmn, off);
  }
  // psum / pmn were counted once per token by each of its 4 lanes: use lane part4's own copy
  if (tj == 0) {
#pragma unroll
    for (int i = 0; i < 32; ++i) red[warp][32 * part4 + i] = acc[i];
    if (part4 == 0) {
      red[warp][kKvD] = psum;
      red[warp][kKvD + 1] = pmn;
    }
  }
  __syncthreads();
  // combine the 4 warps: thread i < 128 owns output dimension i
  const int i = threadIdx.x;
  float o = 0.0f, l = 0.0f, lm = 0.0f;
#pragma unroll
  for (int w = 0; w < kAttThreads / 32; ++w) {
    o += red[w][i];
    l += red[w][kKvD];
    lm += red[w][kKvD + 1];
  }
  o += lm;                                            // + sum_t p_t mn_t (same for every dim)
  if (splits == 1) {
    out[static_cast<int64_t>(bh) * kKvD + i] = c1 > c0 ? o / l : 0.0f;
  } else {
    float* pp = part + (static_cast<int64_t>(bh) * splits + split) * (kKvD + 2);
    pp[i] = o;
    if (i == 0) {
      pp[kKvD] = c1 > c0 ? cmax : -INFINITY;
      pp[kKvD + 1] = l;
    }
  }
}

// log-sum-exp merge of the chunks: one warp per (sequence, head), a lane owns 4 dimensions
__global__ void __launch_bounds__(128)
decode_combine_kernel(int64_t BH, int32_t splits, const float* __restrict__ part,
                      float* __restrict__ out) {
  griddep_wait();
  griddep_launch();
  const int lane = threadIdx.x % 32;
  const int64_t bh = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32;
  if (bh >= BH) return;
  const float* pp = part + bh * splits * (kKvD + 2);
  float m = -INFINITY;
  for (int s = 0; s < splits; ++s) m = fmaxf(m, pp[s * (kKvD + 2) + kKvD]);
  float l = 0.0f, o[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  for (int s = 0; s < splits; ++s) {
    const float ms = pp[s * (kKvD + 2) + kKvD];
    if (ms == -INFINITY) continue;
    const float f = __expf(ms - m);
    l = fmaf(f, pp[s * (kKvD + 2) + kKvD + 1], l);
#pragma unroll
    for (int k = 0; k < 4; ++k) o[k] = fmaf(f, pp[s * (kKvD + 2) + 4 * lane + k], o[k]);
  }
  *reinterpret_cast<float4*>(out + bh * kKvD + 4 * lane) =
      make_float4(o[0] / l, o[1] / l, o[2] / l, o[3] / l);
}

// chunk (multiple of the page) and split count for a batch: enough CTAs for ~2 waves
void plan_decode_attention(int64_t BH, int32_t max_seq_len, int num_sms, int32_t* chunk,
                           int32_t* splits) {
  int64_t s = (2LL * num_sms + BH - 1) / BH;
  const int64_t max_split = (max_seq_len + 63) / 64;   // at least 64 tokens per chunk
  if (s > max_split) s = max_split;
  if (s < 1) s = 1;
  int64_t c = (max_seq_len + s - 1) / s;
  c = ((c + kKvPage - 1) / kKvPage) * kKvPage;
  if (c > kMaxChunk) c = kMaxChunk;
  *chunk = static_cast<int32_t>(c);
  *splits = static_cast<int32_t>((max_seq_len + c - 1) / c);
}

cudaError_t launch_decode_attention(const void* q, int64_t B, int32_t H, const uint8_t* kc,
                                    const float* kp, const uint8_t* vc, const float* vp,
                                    const int32_t* block_table, int64_t max_pages,
                                    const int32_t* seq_lens, int32_t max_seq_len, float* out,
                                    float* workspace, cudaStream_t stream, int num_sms,
                                    int* launches) {
  int32_t chunk, splits;
  plan_decode_attention(B * H, max_seq_len, num_sms, &chunk, &splits);
  cudaError_t e = launch_pdl(decode_attention_kernel,
                             dim3(static_cast<unsigned>(B * H), static_cast<unsigned>(splits)),
                             dim3(kAttThreads), 0, stream, static_cast<const __half*>(q), H, kc,
                             kp, vc, vp, block_table, max_pages, seq_lens, chunk, splits, out,
                             workspace);
  if (e != cudaSuccess) return e;
  *launches = 1;
  if (splits > 1) {
    const int64_t blocks = (B * H * 32 + 127) / 128;
    e = launch_pdl(decode_combine_kernel, dim3(static_cast<unsigned>(blocks)), dim3(128), 0,
                   stream, B * H, splits, static_cast<const float*>(workspace), out);
    if (e != cudaSuccess) return e;
    *launches = 2;
  }
  return cudaSuccess;
}

size_t decode_attention_workspace_bytes(int64_t B, int32_t H, int32_t max_seq_len, int num_sms) {
  int32_t chunk, splits;
  plan_decode_attention(B * H, max_seq_len, num_sms, &chunk, &splits);
  return splits > 1 ? static_cast<size_t>(B * H) * splits * (kKvD + 2) * sizeof(float) : 0;
}

}  // namespace atom
