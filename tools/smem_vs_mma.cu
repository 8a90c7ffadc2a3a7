// smem_vs_mma.cu -- does generic shared-memory traffic (LDS/STS) compete with the tensor core's
// SMEM operand reads?  Thread 0 issues NMMA i8 128x256x32 SS MMAs (12 KB of operands each) while
// 8 other warps stream LDS.128+STS.128 over a separate 32 KB region.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2310_19102_b200/csrc -o tools/smem_vs_mma tools/smem_vs_mma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace atom;

__global__ void probe(int nmma, int iters, int mode, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* A = smem + ((1024 - (smem_u32(smem) & 1023)) & 1023);
  uint8_t* B = A + 128 * 128;
  uint8_t* X = B + 256 * 128;   // 32 KB scratch for LDS/STS traffic
  for (int i = threadIdx.x; i < 128 * 128 + 256 * 128 + 32768; i += blockDim.x) A[i] = 1;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&tbase, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x == 0 && nmma > 0) {
    const uint32_t idesc = umma_idesc_i8(128, 256);
    const uint64_t da = umma_desc_sw128(smem_u32(A)), db = umma_desc_sw128(smem_u32(B));
    long long t0 = clock64();
    for (int i = 0; i < nmma; ++i) umma_i8(tbase, da, db, idesc, 1u);
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    out[0] = clock64() - t0;
  }
  if (warp >= 8 && iters > 0) {
    const int t = threadIdx.x - 256;   // 0..255
    uint4* x = reinterpret_cast<uint4*>(X);
    uint4 v = make_uint4(t, 1, 2, 3);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      // 2 KB read + 2 KB write per warp-iteration... 256 threads x 16 B = 4 KB per phase
      if (mode != 2) {   // loads
        uint4 a = x[(t + 256 * (i & 3)) & 2047];
        v.x ^= a.x; v.y += a.y; v.z ^= a.z; v.w += a.w;
        if (mode == 1) {
          uint4 b = x[(t + 256 * ((i + 2) & 3)) & 2047];
          v.x ^= b.x; v.y += b.y; v.z ^= b.z; v.w += b.w;
        }
      }
      if (mode != 1)     // stores
        x[(t + 256 * ((i + 1) & 3) + 1024) & 2047] = make_uint4(v.x, v.y + i, v.z, v.w);
      if (mode == 2) x[(t + 256 * ((i + 3) & 3) + 1024) & 2047] = make_uint4(v.x, v.y, v.z + i, v.w);
    }
    long long t1 = clock64();
    if (t == 0) out[1] = t1 - t0;
    if (v.x == 0x1234567) out[2] = v.y;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tbase, 512); }
}

int main() {
  long long* d; cudaMalloc(&d, 8 * sizeof(long long));
  const int smem = 128 * 128 + 256 * 128 + 32768 + 2048;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4000, nmma = 1000;
  long long h[4];
  for (int mode = 0; mode < 3; ++mode)
  for (int cfg = 0; cfg < 3; ++cfg) {
    if (mode > 0 && cfg == 0) continue;
    const int nm = cfg == 1 ? 0 : nmma, it = cfg == 0 ? 0 : iters;
    cudaMemset(d, 0, 8 * sizeof(long long));
    probe<<<1, 512, smem>>>(nm, it, mode, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const double bytes = 256.0 * 16 * 2 * iters;   // LDS + STS bytes
    printf("[%s] %s: MMA %lld clk (%.1f clk/MMA)  smem %lld clk (%.1f B/clk)  [%s]\n",
           mode == 0 ? "LDS+STS" : mode == 1 ? "LDSx2  " : "STSx2  ",
           cfg == 0 ? "MMA only    " : cfg == 1 ? "smem only   " : "MMA + smem  ",
           h[0], nm ? (double)h[0] / nm : 0.0, h[1], h[1] ? bytes / h[1] : 0.0, cudaGetErrorString(e));
  }
}
