// drain_bench2.cu -- the GEMM epilogue's inner loop in isolation (LDTM 32x32b, LOP3 magic
// conversion, 2 FFMA2 per column pair, s_a via 16-byte broadcast loads), NW epilogue warps
// sharing 256 columns of one 128-lane group, with the tensor pipe busy on the other TMEM half.
// Variants: warps per lane quarter (3 or 4), load batch width (16 or 32 columns).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2310_19102_b200/csrc -o tools/drain_bench2 tools/drain_bench2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace atom;

template <int WPQ, int JB, int LOP>
__global__ void __launch_bounds__(WPQ * 128 + 128, 1) drain(int iters, int mma, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* A = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* B = A + 128 * 128;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ __align__(16) float sa[256];
  __shared__ volatile int stop;
  for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(A)[i] = i * 2654435761u;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) sa[i] = 1.0f + i;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); stop = 0; }
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) tmem_alloc(&tbase, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  constexpr int NCOLMAX = (256 / 8 + WPQ - 1) / WPQ * 8;
  if (warp == 1) {
    if (lane == 0 && mma) {
      const uint32_t idesc = umma_idesc_i8(128, 256);
      const uint64_t da = umma_desc_sw128(smem_u32(A)), db = umma_desc_sw128(smem_u32(B));
      int n = 0;
      while (!stop && n < 4000000) { umma_i8(tbase + 256, da, db, idesc, 1u); ++n; }
      umma_commit(&bar);
      mbar_wait(&bar, 0);
    }
  } else if (warp >= 4) {
    const int e = warp - 4, q = warp & 3, third = e >> 2;
    constexpr int NC = 32, kBase = NC / WPQ, kRem = NC % WPQ;
    const int ncol = 8 * (kBase + (third < kRem ? 1 : 0));
    const int c0 = 8 * (third * kBase + (third < kRem ? third : kRem));
    const uint32_t tq = tbase + ((uint32_t)(q * 32) << 16) + c0;
    float acc[NCOLMAX];
#pragma unroll
    for (int i = 0; i < NCOLMAX; ++i) acc[i] = 0.f;
    const float sw = 0.5f + lane;
    const float2 sw2 = make_float2(sw, sw), nc2 = make_float2(-12582912.0f * sw, -12582912.0f * sw);
    const uint32_t magic = 0x4B400000u;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j0 = 0; j0 < NCOLMAX; j0 += JB) {
        uint32_t r[JB];
#pragma unroll
        for (int j = j0; j < j0 + JB && j < NCOLMAX; j += 16) {
          if (JB >= 32 && j == j0 && j + JB <= ncol) {
#pragma unroll
            for (int jj = 0; jj < JB; jj += 32) tmem_ld32(tq + j + jj, *reinterpret_cast<uint32_t(*)[32]>(r + jj));
            j += JB - 16; continue;
          }
          if (j + 16 <= ncol) tmem_ld16p(tq + j, r + (j - j0));
          else if (j + 8 <= ncol) tmem_ld8(tq + j, r + (j - j0));
        }
        tmem_ld_wait();
#pragma unroll
        for (int j = j0; j < j0 + JB && j < NCOLMAX; j += 4) {
          if (j < ncol) {
            uint32_t* rv = r + (j - j0);
            if (LOP) {
#pragma unroll
              for (int v = 0; v < 4; ++v) rv[v] = __float_as_uint(__uint_as_float(and_xor(rv[v], 0x7FFFFF, magic)));
            }
            const float4 s4 = *reinterpret_cast<const float4*>(&sa[c0 + j]);
            const float2 g0 = __ffma2_rn(make_float2(__uint_as_float(rv[0]), __uint_as_float(rv[1])), sw2, nc2);
            const float2 g1 = __ffma2_rn(make_float2(__uint_as_float(rv[2]), __uint_as_float(rv[3])), sw2, nc2);
            const float2 a0 = __ffma2_rn(make_float2(s4.x, s4.y), g0, make_float2(acc[j], acc[j + 1]));
            const float2 a1 = __ffma2_rn(make_float2(s4.z, s4.w), g1, make_float2(acc[j + 2], acc[j + 3]));
            acc[j] = a0.x; acc[j + 1] = a0.y; acc[j + 2] = a1.x; acc[j + 3] = a1.y;
          }
        }
      }
    }
    long long t1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NCOLMAX; ++i) s += acc[i];
    if (s == 1.2345f) out[100] = 1;
    if (threadIdx.x == 128) out[blockIdx.x * 2] = t1 - t0;
    named_bar_sync(1, WPQ * 128);
    if (threadIdx.x == 128) stop = 1;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tbase, 512); }
}

template <int WPQ, int JB, int LOP>
void run(int sms, int mma, long long* d) {
  const int iters = 2000;
  const int smem = (128 + 256) * 128 + 1024;
  cudaFuncSetAttribute(drain<WPQ, JB, LOP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  drain<WPQ, JB, LOP><<<sms, WPQ * 128 + 128, smem>>>(iters, mma, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[2]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("warps/quarter=%d batch=%d lop=%d mma=%d: %.1f clk per 128x256 group (%s)\n", WPQ, JB,
         LOP, mma, (double)h[0] / iters, cudaGetErrorString(e));
  fflush(stdout);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d; cudaMalloc(&d, 512 * sizeof(long long));
  run<3, 16, 1>(sms, 1, d);
  run<2, 16, 1>(sms, 1, d); run<2, 32, 1>(sms, 1, d); run<2, 64, 1>(sms, 1, d);
  run<2, 32, 0>(sms, 1, d); run<2, 64, 0>(sms, 1, d);
  return 0;
}
