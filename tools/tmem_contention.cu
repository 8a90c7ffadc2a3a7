// tmem_contention.cu -- does tcgen05.ld wait behind queued tcgen05.mma of another thread?
// Thread 0 (warp 0) issues NMMA back-to-back i8 MMAs (128x128x32, 64 clk each) into TMEM cols
// [0,128); warps 4..7 then time tcgen05.ld (x32) from cols [256,288) while the MMAs run.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2310_19102_b200/csrc -o tools/tmem_contention tools/tmem_contention.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace atom;

__global__ void probe(int nmma, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, go;
  __shared__ uint32_t tbase;
  uint8_t* A = smem + ((1024 - (smem_u32(smem) & 1023)) & 1023);
  uint8_t* B = A + 128 * 128;
  for (int i = threadIdx.x; i < 2 * 128 * 128; i += blockDim.x) A[i] = 1;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&go, 1); fence_mbar_init(); }
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&tbase, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  long long t_issue0 = 0, t_issue1 = 0;
  if (threadIdx.x == 0) {
    const uint32_t idesc = umma_idesc_i8(128, 128);
    const uint64_t da = umma_desc_sw128(smem_u32(A)), db = umma_desc_sw128(smem_u32(B));
    t_issue0 = clock64();
    for (int i = 0; i < nmma; ++i) umma_i8(tbase, da, db, idesc, 1u);
    umma_commit(&bar);
    t_issue1 = clock64();
    mbar_arrive(&go);                 // tell the loaders the MMAs are queued
    mbar_wait(&bar, 0);
    long long t_done = clock64();
    out[blockIdx.x * 8 + 0] = t_issue1 - t_issue0;
    out[blockIdx.x * 8 + 1] = t_done - t_issue0;
  }
  if (warp >= 4) {
    mbar_wait(&go, 0);
    long long t0 = clock64();
    uint32_t r[32];
    tmem_ld32(tbase + ((uint32_t)((warp & 3) * 32) << 16) + 256, r);
    tmem_ld_wait();
    long long t1 = clock64();
    uint32_t x = 0;
    for (int k = 0; k < 32; ++k) x ^= r[k];
    if (threadIdx.x == 128) { out[blockIdx.x * 8 + 2] = t1 - t0; out[blockIdx.x * 8 + 3] = x; }
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tbase, 512); }
}

int main() {
  long long* d; cudaMalloc(&d, 8 * 8 * sizeof(long long));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  for (int n : {0, 4, 16, 64}) {
    probe<<<1, 256, 40000>>>(n, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[8]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("queued MMAs %3d: issue %lld clk, MMAs done after %lld clk, LDTM x32 latency %lld clk (%s)\n",
           n, h[0], h[1], h[2], cudaGetErrorString(e));
  }
}
