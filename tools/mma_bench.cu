// mma_bench.cu -- raw tcgen05.mma throughput on one SM per CTA (grid = #SMs): back-to-back
// dispatches from shared-memory operands into one TMEM accumulator.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2310_19102_b200/csrc -o tools/mma_bench tools/mma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace atom;

// KIND 0 = i8 (K=32), 1 = f16 (K=16), 2 = 1 f16 + 4 i8 per "group", 3 = i8 rotating over 4
// accumulators every 4 dispatches, 4 = as 3 plus 2 commits per group, 5 = i8, accumulate=0 on
// the first dispatch of every 4 (same accumulator)
template <int KIND, int N>
__global__ void mma_loop(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint64_t bar2[2];
  __shared__ uint32_t tbase;
  uint8_t* A = smem + ((1024 - (smem_u32(smem) & 1023)) & 1023);
  uint8_t* B = A + 128 * 128;
  for (int i = threadIdx.x; i < 128 * 128 + N * 128; i += blockDim.x) A[i] = 0;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar2[0], 1); mbar_init(&bar2[1], 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tbase, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t idesc = KIND != 1 ? umma_idesc_i8(128, N) : umma_idesc_f16_f32(128, N);
    const uint64_t da = umma_desc_sw128(smem_u32(A)), db = umma_desc_sw128(smem_u32(B));
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (KIND == 0) umma_i8(tbase, da, db, idesc, 1u);
      else if (KIND == 1) umma_f16(tbase, da, db, idesc, 1u);
      else if (KIND == 2) {
        if ((i % 5) == 0) umma_f16(tbase, da, db, umma_idesc_f16_f32(128, N), 0u);
        else umma_i8(tbase, da, db, umma_idesc_i8(128, N), 1u);
      } else if (KIND == 3 || KIND == 4) {
        const uint32_t acc = tbase + ((i / 4) % 4) * N;
        umma_i8(acc, da, db, idesc, 1u);
        if (KIND == 4 && (i % 4) == 3) { umma_commit(&bar2[0]); umma_commit(&bar2[1]); }
      } else {
        umma_i8(tbase, da, db, idesc, (i % 4) != 0);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tbase, 512); }
}

template <int KIND, int N>
void run(const char* name, int sms, unsigned long long* d) {
  const int iters = 4096;
  size_t smem = 128 * 128 + N * 128 + 2048;
  cudaFuncSetAttribute(mma_loop<KIND, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mma_loop<KIND, N><<<sms, 128, smem>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double k = KIND == 1 ? 16 : 32;
  printf("%-16s M=128 N=%3d : %.1f clk/dispatch, %.0f MAC/clk/SM  (%s)\n", name, N, (double)h / iters,
         128.0 * N * k * iters / h, cudaGetErrorString(e));
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d; cudaMalloc(&d, sms * 8);
  run<0, 64>("i8", sms, d); run<0, 128>("i8", sms, d); run<0, 256>("i8", sms, d);
  run<1, 128>("f16", sms, d); run<1, 256>("f16", sms, d);
  run<2, 128>("f16+4i8", sms, d);
  run<3, 128>("i8 rot4", sms, d);
  run<4, 128>("i8 rot4+commit", sms, d);
  run<5, 128>("i8 acc0/4", sms, d);
  return 0;
}
