// quantize.cu -- a0/a1: fused channel reorder + dynamic symmetric quantization (sm_100a).
//
// Paper: reorder activations by the offline calibration index so the outlier channels sit at the
// tail (Fig 4), keep the last 128 reordered channels in INT8, quantize the
// rest to INT4 in groups of 128, with dynamically computed symmetric scales
// s = 2*max|X|*c/(2^n-1) and codes clamp(round(X/s)).  The same kernel
// quantizes weights offline (rows = output channels, clip 0.85).
//
// B200 design: HBM-bound gather.  One CTA per (row, group-chunk); the fp16 row is staged once in
// shared memory with 128-bit streaming loads (coalesced), the gather x'[j] = x[perm[j]] then
// reads shared memory.  One half-warp per 128-channel group: each lane owns 8 reordered
// channels (two 128-bit perm loads), the group |max| is a 4-step shuffle reduction, codes are
// packed in registers and written as 64 contiguous bytes (INT4) or 128 bytes (INT8), plus the
// GEMM operand form a_f8 (one E4M3 byte per code) and the per-row dequant constants a_ab
// (include/atom.h).
// Numerics are pinned to the oracle's binary32 steps: __fdiv_rn / __fmul_rn / __frcp_rn are
// IEEE round-to-nearest and never contracted; cvt.rni gives round-half-to-even.
#include <cfloat>
#include <cstdint>
#include <cuda_fp16.h>

#include "internal.h"
#include "ptx.cuh"

namespace atom {

constexpr int kQuantThreads = 256;
constexpr int kQuantWarps = kQuantThreads / 32;

__device__ __forceinline__ uint4 ld_stream_u4(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// kNorm (NEXT-1): the RMSNorm the paper fuses the quantizer into is applied to the
// staged row first: r = RN32(1/sqrt(ss/ldx + eps)) where ss is the EXACT sum of squares rounded
// once to double (128-bit integer accumulation of x^2 * 2^48: order-independent by
// construction), and the gathered value becomes y = fp16_rn(RN32(RN32(x*r) * gamma)) (oracle N1,
// reading G19).
// kPre: 0 = plain a1; 1 = RMSNorm first (NEXT-1); 2 = SwiGLU first (NEXT-4 piece): x is the
// gate projection and `up` the up projection of a Llama MLP, and the staged value is
// h = fp16_rn(RN32(s * u)), s = RN32(g / RN32(1 + e)), e = the pinned binary32 exp(-g) of reading
// G20 (expf_pinned below), i.e. the down projection's input, quantized without an fp16 round
// trip through HBM.

// The binary32 exponential of reading G20 (oracle_expf_pinned), one IEEE operation per step.
__device__ __forceinline__ float expf_pinned(float x) {
  if (x > 88.0f) return __int_as_float(0x7F800000);
  if (x < -87.0f) return 0.0f;
  const float L2E = 1.44269502162933349609375f, LN2_HI = 0.693145751953125f;
  const float LN2_LO = 1.428606765330187045037746429443359375e-06f;
  const float n = rintf(__fmul_rn(x, L2E));
  float r = __fmaf_rn(-n, LN2_HI, x);
  r = __fmaf_rn(-n, LN2_LO, r);
  float p = 1.0f / 720.0f;
  p = __fmaf_rn(p, r, 1.0f / 120.0f);
  p = __fmaf_rn(p, r, 1.0f / 24.0f);
  p = __fmaf_rn(p, r, 1.0f / 6.0f);
  p = __fmaf_rn(p, r, 0.5f);
  p = __fmaf_rn(p, r, 1.0f);
  p = __fmaf_rn(p, r, 1.0f);
  // p * 2^n with one rounding (= ldexpf): 2^n is a normal binary32 for n in [-126, 127]
  return __fmul_rn(p, __int_as_float((static_cast<int>(n) + 127) << 23));
}

// 128-bit unsigned accumulator (hi, lo) of x^2 * 2^48 for fp16-valued x (exact).
struct U128 {
  unsigned long long lo = 0, hi = 0;
  __device__ __forceinline__ void add(unsigned long long plo, unsigned long long phi) {
    lo += plo;
    hi += phi + (lo < plo ? 1ull : 0ull);
  }
  __device__ __forceinline__ void add_square(float x) {
    const unsigned long long m = __float2ull_rz(fabsf(x) * 16777216.0f);   // |x| * 2^24, exact
    add(m * m, __umul64hi(m, m));
  }
  // round-to-nearest-even conversion of the 128-bit integer to double
  __device__ __forceinline__ double to_double() const {
    if (hi == 0) return __ull2double_rn(lo);
    const int sh = 64 - __clzll(static_cast<long long>(hi));   // bits of hi: shift right by sh
    unsigned long long m = (hi << (64 - sh)) | (lo >> sh);
    if ((lo & ((1ull << sh) - 1ull)) != 0) m |= 1ull;          // sticky, far below bit 11
    return ldexp(__ull2double_rn(m), sh);
  }
};
template <int kPre>
__global__ void __launch_bounds__(kQuantThreads)
reorder_quantize_kernel(const __half* __restrict__ x, int64_t rows, int64_t ldx,
                        const int32_t* __restrict__ perm, int32_t G, int32_t G4,
                        int32_t groups_per_cta, float clip4, float clip8,
                        uint8_t* __restrict__ q4, int8_t* __restrict__ q8,
                        uint8_t* __restrict__ af8, float* __restrict__ ab, int64_t Mp,
                        int64_t K, float* __restrict__ scales, float* __restrict__ wsp,
                        const __half* __restrict__ gamma, float eps,
                        const __half* __restrict__ up) {
  constexpr bool kNorm = kPre == 1;
  extern __shared__ uint4 srow4[];
  const __half* srow = reinterpret_cast<const __half*>(srow4);
  const int64_t row = blockIdx.x;
  const int g_begin = blockIdx.y * groups_per_cta;
  const int g_end = min(G, g_begin + groups_per_cta);

  // PDL: x (and the outputs) may belong to the previous kernel of the stream
  griddep_wait();
  griddep_launch();
  // Stage the whole source row (the gather may touch any channel).  Plain a1 and the RMSNorm:
  // one bulk copy (a single HBM round trip per row, no per-thread load -> store chains); the
  // SwiGLU combines two rows element-wise on the way in, with 4 loads of each in flight.
  const uint4* src = reinterpret_cast<const uint4*>(x + row * ldx);
  const int n16 = static_cast<int>(ldx / 8);
  U128 ss;
  if constexpr (kPre != 2) {
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      fence_mbar_init();
      mbar_arrive_expect_tx(&bar, static_cast<uint32_t>(ldx) * 2);
      bulk_g2s(srow4, src, static_cast<uint32_t>(ldx) * 2, &bar);
    }
    __syncthreads();
    mbar_wait(&bar, 0);
    if constexpr (kNorm) {
      for (int i = threadIdx.x; i < n16; i += kQuantThreads) {
        const uint4 v = srow4[i];
        const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = __half22float2(h[k]);
          ss.add_square(f.x);
          ss.add_square(f.y);
        }
      }
    }
  } else {
    const uint4* upr = reinterpret_cast<const uint4*>(up + row * ldx);
    constexpr int U = 4;
    for (int i0 = threadIdx.x; i0 < n16; i0 += U * kQuantThreads) {
      uint4 gv[U], uv[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int i = i0 + j * kQuantThreads;
        if (i < n16) {
          gv[j] = ld_stream_u4(src + i);
          uv[j] = ld_stream_u4(upr + i);
        }
      }
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int i = i0 + j * kQuantThreads;
        if (i >= n16) continue;
        __half2* hg = reinterpret_cast<__half2*>(&gv[j]);
        const __half2* hu = reinterpret_cast<const __half2*>(&uv[j]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 g = __half22float2(hg[k]), u = __half22float2(hu[k]);
          const float sx = __fdiv_rn(g.x, __fadd_rn(1.0f, expf_pinned(-g.x)));
          const float sy = __fdiv_rn(g.y, __fadd_rn(1.0f, expf_pinned(-g.y)));
          hg[k] = __floats2half2_rn(__fmul_rn(sx, u.x), __fmul_rn(sy, u.y));
        }
        srow4[i] = gv[j];
      }
    }
  }
  float rinv = 1.0f;
  if constexpr (kNorm) {
    // exact 128-bit sum over the CTA (integer additions: any order gives the same sum)
    __shared__ unsigned long long red[kQuantThreads / 32][2];
    __shared__ float rs;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
      ss.add(__shfl_xor_sync(0xffffffffu, ss.lo, off), __shfl_xor_sync(0xffffffffu, ss.hi, off));
    if ((threadIdx.x & 31) == 0) {
      red[threadIdx.x / 32][0] = ss.lo;
      red[threadIdx.x / 32][1] = ss.hi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      U128 t;
      for (int w = 0; w < kQuantThreads / 32; ++w) t.add(red[w][0], red[w][1]);
      const double sum = ldexp(t.to_double(), -48);          // RN64 of the exact sum
      rs = __double2float_rn(
          __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(__ddiv_rn(sum, static_cast<double>(ldx)),
                                              static_cast<double>(eps)))));
    }
    __syncthreads();
    rinv = rs;
  } else {
    __syncthreads();
  }

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // alpha = fl(fl(2c) / (2^n - 1))
  const float alpha4 = __fdiv_rn(__fmul_rn(2.0f, clip4), 15.0f);
  const float alpha8 = __fdiv_rn(__fmul_rn(2.0f, clip8), 255.0f);
  const int64_t row4 = static_cast<int64_t>(G4) * 64;

  // Two groups per warp, one per half-warp; a lane owns 8 consecutive reordered channels (two
  // 128-bit perm loads), the group |max| is a 4-step shuffle.  Codes: v = fl(x * fl(1/s)) (one
  // RN multiply), clamped to the code range (clamping to integer bounds commutes with
  // rounding), then rounded half-to-even by adding 1.5*2^23 in binary32 -- the sum's low bits
  // ARE the two's-complement code (0x4B400000 is a multiple of 256), so no float->int
  // conversion is needed; bytes are gathered with PRMT.
  const int hw = lane >> 4, hl = lane & 15;
  constexpr float kRint = 12582912.0f;   // 1.5 * 2^23
  // the perm slices are software-prefetched one iteration ahead (an L2 round trip per group
  // would otherwise sit on the critical path)
  auto perm_at = [&](int t0, int4& a, int4& b) {
    const int t = t0 + hw;
    const int tt = t < g_end ? t : t0;
    a = __ldg(reinterpret_cast<const int4*>(perm + tt * 128 + 8 * hl));
    b = __ldg(reinterpret_cast<const int4*>(perm + tt * 128 + 8 * hl + 4));
  };
  int4 pa_n, pb_n;
  if (g_begin + 2 * warp < g_end) perm_at(g_begin + 2 * warp, pa_n, pb_n);
  for (int t0 = g_begin + 2 * warp; t0 < g_end; t0 += 2 * kQuantWarps) {
    const int t = t0 + hw;
    const bool valid = t < g_end;
    const int tt = valid ? t : t0;
    const int4 pa = pa_n, pb = pb_n;
    if (t0 + 2 * kQuantWarps < g_end) perm_at(t0 + 2 * kQuantWarps, pa_n, pb_n);
    float v[8];
    v[0] = __half2float(srow[pa.x]); v[1] = __half2float(srow[pa.y]);
    v[2] = __half2float(srow[pa.z]); v[3] = __half2float(srow[pa.w]);
    v[4] = __half2float(srow[pb.x]); v[5] = __half2float(srow[pb.y]);
    v[6] = __half2float(srow[pb.z]); v[7] = __half2float(srow[pb.w]);
    if constexpr (kNorm) {
      const int src_c[8] = {pa.x, pa.y, pa.z, pa.w, pb.x, pb.y, pb.z, pb.w};
#pragma unroll
      for (int k = 0; k < 8; ++k)
        v[k] = __half2float(__float2half_rn(
            __fmul_rn(__fmul_rn(v[k], rinv), __half2float(__ldg(gamma + src_c[k])))));
    }
    float amax = fabsf(v[0]);
#pragma unroll
    for (int k = 1; k < 8; ++k) amax = fmaxf(amax, fabsf(v[k]));
#pragma unroll
    for (int off = 8; off > 0; off >>= 1)
      amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
    const bool is_int4 = tt < G4;
    const float s = (amax == 0.0f) ? FLT_MIN : __fmul_rn(amax, is_int4 ? alpha4 : alpha8);
    const float inv = __frcp_rn(s);
    const float lo = is_int4 ? -8.0f : -128.0f, hi = is_int4 ? 7.0f : 127.0f;
    uint32_t f[8];   // bit patterns of 1.5*2^23 + q: low byte = q (two's complement)
#pragma unroll
    for (int k = 0; k < 8; ++k)
      f[k] = __float_as_uint(__fadd_rn(fminf(fmaxf(__fmul_rn(v[k], inv), lo), hi), kRint));
    // even / odd channels, one byte each: E = [q0 q2 q4 q6], O = [q1 q3 q5 q7]
    const uint32_t ev = __byte_perm(__byte_perm(f[0], f[2], 0x0040), __byte_perm(f[4], f[6], 0x0040),
                                    0x5410);
    const uint32_t od = __byte_perm(__byte_perm(f[1], f[3], 0x0040), __byte_perm(f[5], f[7], 0x0040),
                                    0x5410);
    // group code sum (the GEMM's offset-binary correction, include/atom.h "a_ab")
    int qs = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) qs += static_cast<int>(f[k] - 0x4B400000u);
#pragma unroll
    for (int off = 8; off > 0; off >>= 1) qs += __shfl_xor_sync(0xffffffffu, qs, off);
    if (valid) {
      uint8_t* ag = af8 ? af8 + row * K + t * 128 : nullptr;
      if (is_int4) {
        // packed byte j = (q_2j & 0xF) | (q_2j+1 << 4)   (low nibble = even channel)
        if (q4)
          reinterpret_cast<uint32_t*>(q4 + row * row4 + t * 64)[hl] =
              (ev & 0x0F0F0F0Fu) | ((od << 4) & 0xF0F0F0F0u);
        if (ag) {
          // GEMM operand: E4M3 sign-magnitude byte of q (value q * 2^-9); channel 32c + 8i +
          // 2b + h of the group sits at byte 32c + 16h + 4i + b (include/atom.h "a_f8")
          auto sm4 = [](uint32_t w) {   // 4 two's-complement nibbles (low bits of each byte)
            const uint32_t n = w & 0x0F0F0F0Fu;
            const uint32_t neg = (n >> 3) & 0x01010101u;
            return (((n ^ (neg * 0x0Fu)) + neg) & 0x0F0F0F0Fu) | (neg << 7);
          };
          const int p = 32 * (hl >> 2) + 4 * (hl & 3);
          *reinterpret_cast<uint32_t*>(ag + p) = sm4(ev);
          *reinterpret_cast<uint32_t*>(ag + p + 16) = sm4(od);
        }
      } else {
        const uint32_t w0 = __byte_perm(ev, od, 0x5140), w1 = __byte_perm(ev, od, 0x7362);
        if (q8) reinterpret_cast<uint2*>(q8 + row * 128)[hl] = make_uint2(w0, w1);
        if (ag) reinterpret_cast<uint2*>(ag)[hl] = make_uint2(w0, w1);
      }
      if (hl == 0) {
        scales[static_cast<int64_t>(t) * rows + row] = s;
        if (wsp) {   // weights: the GEMM's channel order of the scales (include/atom.h "w_sp")
          const int64_t nl = row & 127, k = nl >> 3;
          const int64_t pos = (row - nl) + 32 * (k >> 2) + 8 * ((nl & 7) >> 1) + 2 * (k & 3) +
                              (nl & 1);
          wsp[static_cast<int64_t>(t) * rows + pos] = s;
        }
        if (ab) {   // (alpha, beta) of include/atom.h "a_ab", in its row order
          const int64_t r = row & 31;
          const int64_t pos = (row - r) + 4 * (r & 7) + (r >> 3);
          const float2 v = is_int4 ? make_float2(s * 262144.0f,
                                                 __fmul_rn(static_cast<float>(-8 * qs), s))
                                   : make_float2(s, 0.0f);
          reinterpret_cast<float2*>(ab)[static_cast<int64_t>(t) * Mp + pos] = v;
        }
      }
    }
  }
}

cudaError_t launch_reorder_quantize(const void* x, int64_t rows, int64_t ldx,
                                    const int32_t* perm, int64_t K, int32_t k_outlier,
                                    float clip4, float clip8, uint8_t* q4, int8_t* q8,
                                    uint8_t* af8, float* ab, float* scales, float* wsp,
                                    cudaStream_t stream, int num_sms, const void* gamma,
                                    float eps, const void* up) {
  const int G = static_cast<int>(K / 128);
  const int G4 = static_cast<int>((K - k_outlier) / 128);
  // Enough CTAs to cover the SMs ~4 times; each extra split re-stages the row (from L2).
  int splits = static_cast<int>((4LL * num_sms + rows - 1) / rows);
  const int max_splits = (G + 2 * kQuantWarps - 1) / (2 * kQuantWarps);
  splits = max(1, min(splits, max_splits));
  const int gpc = (G + splits - 1) / splits;
  splits = (G + gpc - 1) / gpc;
  const size_t smem = static_cast<size_t>(ldx) * sizeof(__half);
  auto kern = up ? reorder_quantize_kernel<2>
                 : gamma ? reorder_quantize_kernel<1> : reorder_quantize_kernel<0>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  dim3 grid(static_cast<unsigned>(rows), static_cast<unsigned>(splits));
  return launch_pdl(kern, grid, dim3(kQuantThreads), smem, stream, static_cast<const __half*>(x),
                    rows, ldx, perm, G, G4, gpc, clip4, clip8, q4, q8, af8, ab, ab_rows(rows), K, scales, wsp,
                    static_cast<const __half*>(gamma), eps, static_cast<const __half*>(up));
}

// ---------------------------------------------------------------------------------------------
// perm validation (test helper)
// ---------------------------------------------------------------------------------------------
__global__ void perm_count_kernel(const int32_t* perm, int64_t K, int64_t ldx, int32_t* counts,
                                  int32_t* bad) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < K;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = perm[j];
    if (p < 0 || p >= ldx) atomicOr(bad, 1);
    else atomicAdd(counts + p, 1);
  }
}

__global__ void perm_check_kernel(const int32_t* counts, int64_t K, int64_t ldx, int32_t* bad,
                                  int32_t* ok) {
  __shared__ int any;
  if (threadIdx.x == 0) any = *bad;
  __syncthreads();
  for (int64_t c = threadIdx.x; c < ldx; c += blockDim.x) {
    const int32_t n = counts[c];
    if (n > 1 || (ldx == K && n != 1)) atomicOr(&any, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) *ok = any ? 0 : 1;
}

cudaError_t launch_validate_perm(const int32_t* perm, int64_t K, int64_t ldx, int32_t* scratch,
                                 int32_t* ok, cudaStream_t stream) {
  cudaError_t e = cudaMemsetAsync(scratch, 0, sizeof(int32_t) * ldx, stream);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(ok, 0, sizeof(int32_t), stream);
  if (e != cudaSuccess) return e;
  perm_count_kernel<<<64, 256, 0, stream>>>(perm, K, ldx, scratch, ok);
  // `ok` doubles as the `bad` accumulator until the check kernel overwrites it.
  perm_check_kernel<<<1, 1024, 0, stream>>>(scratch, K, ldx, ok, ok);
  return cudaGetLastError();
}

}  // namespace atom
