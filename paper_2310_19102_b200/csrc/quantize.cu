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
// packed in registers and written as 64 contiguous bytes (INT4) or 128 bytes (INT8).
// Numerics are pinned to the oracle's binary32 steps: __fdiv_rn / __fmul_rn / __frcp_rn are
// IEEE round-to-nearest and never contracted; cvt.rni gives round-half-to-even.
#include <cfloat>
#include <cstdint>
#include <cuda_fp16.h>

#include "internal.h"

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

__device__ __forceinline__ int quant_code(float x, float inv, int lo, int hi) {
  int q = __float2int_rn(__fmul_rn(x, inv));  // single RN multiply, then round-half-even
  return min(max(q, lo), hi);
}

__global__ void __launch_bounds__(kQuantThreads)
reorder_quantize_kernel(const __half* __restrict__ x, int64_t rows, int64_t ldx,
                        const int32_t* __restrict__ perm, int32_t G, int32_t G4,
                        int32_t groups_per_cta, float clip4, float clip8,
                        uint8_t* __restrict__ q4, int8_t* __restrict__ q8,
                        int8_t* __restrict__ x8, int64_t K, float* __restrict__ scales) {
  extern __shared__ uint4 srow4[];
  const __half* srow = reinterpret_cast<const __half*>(srow4);
  const int64_t row = blockIdx.x;
  const int g_begin = blockIdx.y * groups_per_cta;
  const int g_end = min(G, g_begin + groups_per_cta);

  // Stage the whole source row (the gather may touch any channel).
  const uint4* src = reinterpret_cast<const uint4*>(x + row * ldx);
  const int n16 = static_cast<int>(ldx / 8);
  for (int i = threadIdx.x; i < n16; i += kQuantThreads) srow4[i] = ld_stream_u4(src + i);
  __syncthreads();

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // alpha = fl(fl(2c) / (2^n - 1))
  const float alpha4 = __fdiv_rn(__fmul_rn(2.0f, clip4), 15.0f);
  const float alpha8 = __fdiv_rn(__fmul_rn(2.0f, clip8), 255.0f);
  const int64_t row4 = static_cast<int64_t>(G4) * 64;

  // Each warp quantizes two groups at a time, one per half-warp; a lane owns 8 consecutive
  // reordered channels (two 128-bit perm loads), the group |max| is a 4-step shuffle.
  const int hw = lane >> 4, hl = lane & 15;
  for (int t0 = g_begin + 2 * warp; t0 < g_end; t0 += 2 * kQuantWarps) {
    const int t = t0 + hw;
    const bool valid = t < g_end;
    const int tt = valid ? t : t0;
    const int4 pa = __ldg(reinterpret_cast<const int4*>(perm + tt * 128 + 8 * hl));
    const int4 pb = __ldg(reinterpret_cast<const int4*>(perm + tt * 128 + 8 * hl + 4));
    float v[8];
    v[0] = __half2float(srow[pa.x]); v[1] = __half2float(srow[pa.y]);
    v[2] = __half2float(srow[pa.z]); v[3] = __half2float(srow[pa.w]);
    v[4] = __half2float(srow[pb.x]); v[5] = __half2float(srow[pb.y]);
    v[6] = __half2float(srow[pb.z]); v[7] = __half2float(srow[pb.w]);
    float amax = fabsf(v[0]);
#pragma unroll
    for (int k = 1; k < 8; ++k) amax = fmaxf(amax, fabsf(v[k]));
#pragma unroll
    for (int off = 8; off > 0; off >>= 1)
      amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
    const bool is_int4 = tt < G4;
    const float s = (amax == 0.0f) ? FLT_MIN : __fmul_rn(amax, is_int4 ? alpha4 : alpha8);
    const float inv = __frcp_rn(s);
    if (valid) {
      int8_t* xg = x8 ? x8 + row * K + t * 128 : nullptr;
      if (is_int4) {
        int q[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) q[k] = quant_code(v[k], inv, -8, 7);
        if (q4) {
          uint32_t packed = 0;
#pragma unroll
          for (int k = 0; k < 8; ++k) packed |= static_cast<uint32_t>(q[k] & 0xF) << (4 * k);
          reinterpret_cast<uint32_t*>(q4 + row * row4 + t * 64)[hl] = packed;
        }
        if (xg) {
          // GEMM operand order (atom.h "x8"): channel 32c + 8i + 2b + h of the group sits at
          // byte 32c + 16h + 4i + b -- the order in which the GEMM unpacks weight nibbles.
          uint32_t ev = 0, od = 0;
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            ev |= static_cast<uint32_t>(q[2 * b] & 0xFF) << (8 * b);
            od |= static_cast<uint32_t>(q[2 * b + 1] & 0xFF) << (8 * b);
          }
          const int p = 32 * (hl >> 2) + 4 * (hl & 3);
          *reinterpret_cast<uint32_t*>(xg + p) = ev;
          *reinterpret_cast<uint32_t*>(xg + p + 16) = od;
        }
      } else {
        uint32_t lo = 0, hi = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          lo |= static_cast<uint32_t>(quant_code(v[k], inv, -128, 127) & 0xFF) << (8 * k);
          hi |= static_cast<uint32_t>(quant_code(v[k + 4], inv, -128, 127) & 0xFF) << (8 * k);
        }
        if (q8) reinterpret_cast<uint2*>(q8 + row * 128)[hl] = make_uint2(lo, hi);
        if (xg) reinterpret_cast<uint2*>(xg)[hl] = make_uint2(lo, hi);
      }
      if (hl == 0) scales[static_cast<int64_t>(t) * rows + row] = s;
    }
  }
}

cudaError_t launch_reorder_quantize(const void* x, int64_t rows, int64_t ldx,
                                    const int32_t* perm, int64_t K, int32_t k_outlier,
                                    float clip4, float clip8, uint8_t* q4, int8_t* q8,
                                    int8_t* x8, float* scales, cudaStream_t stream, int num_sms) {
  const int G = static_cast<int>(K / 128);
  const int G4 = static_cast<int>((K - k_outlier) / 128);
  // Enough CTAs to cover the SMs ~4 times; each extra split re-stages the row (from L2).
  int splits = static_cast<int>((4LL * num_sms + rows - 1) / rows);
  const int max_splits = (G + 2 * kQuantWarps - 1) / (2 * kQuantWarps);
  splits = max(1, min(splits, max_splits));
  const int gpc = (G + splits - 1) / splits;
  splits = (G + gpc - 1) / gpc;
  const size_t smem = static_cast<size_t>(ldx) * sizeof(__half);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(reorder_quantize_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  dim3 grid(static_cast<unsigned>(rows), static_cast<unsigned>(splits));
  reorder_quantize_kernel<<<grid, kQuantThreads, smem, stream>>>(
      static_cast<const __half*>(x), rows, ldx, perm, G, G4, gpc, clip4, clip8, q4, q8, x8, K, scales);
  return cudaGetLastError();
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
