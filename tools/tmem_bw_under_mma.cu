// tmem_bw_under_mma.cu -- TMEM load throughput of 8 warps while thread 0 keeps the tensor pipe
// busy with i8 128x256x32 MMAs into columns [0,256); loads read columns [256,384).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2310_19102_b200/csrc -o tools/tmem_bw_under_mma tools/tmem_bw_under_mma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace atom;

__global__ void probe(int nmma, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* A = smem + ((1024 - (smem_u32(smem) & 1023)) & 1023);
  uint8_t* B = A + 128 * 128;
  for (int i = threadIdx.x; i < 128 * 128 + 256 * 128; i += blockDim.x) A[i] = 1;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&tbase, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t idesc = umma_idesc_i8(128, 256);
    const uint64_t da = umma_desc_sw128(smem_u32(A)), db = umma_desc_sw128(smem_u32(B));
    long long t0 = clock64();
    for (int i = 0; i < nmma; ++i) umma_i8(tbase, da, db, idesc, 1u);
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    out[blockIdx.x * 4 + 0] = clock64() - t0;
  }
  if (warp >= 8) {
    const uint32_t t = tbase + ((uint32_t)((warp & 3) * 32) << 16) + 256 + ((warp >> 2) & 1) * 64;
    uint32_t x = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      uint32_t r[16];
      tmem_ld16(t, r); tmem_ld_wait();
#pragma unroll
      for (int k = 0; k < 16; ++k) x ^= r[k];
      tmem_ld16(t + 16, r); tmem_ld_wait();
#pragma unroll
      for (int k = 0; k < 16; ++k) x ^= r[k];
    }
    long long t1 = clock64();
    if ((threadIdx.x & 255) == 0) out[blockIdx.x * 4 + 1] = t1 - t0;
    if (x == 0x12345) out[blockIdx.x * 4 + 3] = x;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tbase, 512); }
}

int main() {
  long long* d; cudaMalloc(&d, 64 * sizeof(long long));
  const int smem = 128 * 128 + 256 * 128 + 2048;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  for (int n : {0, 2000}) {
    probe<<<1, 512, smem>>>(n, iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[4]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const double bytes = 8.0 * 32 * 32 * 4 * iters;   // 8 warps x 32 lanes x 32 cols x 4 B
    printf("MMAs %4d (%lld clk): 8-warp TMEM ld %.1f B/clk over %lld clk (%s)\n", n, h[0],
           bytes / h[1], h[1], cudaGetErrorString(e));
  }
}
