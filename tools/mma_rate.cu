// mma_rate.cu -- tcgen05.mma kind::i8 rate with the GEMM's operand pattern: SW128 K-major
// operands in RS rotating shared-memory slots, 4 dispatches (K = 32 each) per 128-channel group,
// accumulator rotation over RT TMEM buffers, one commit per group.  Operand DATA varies: zeros,
// random int8, random 16*q4.  Development tool (not part of the product).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2310_19102_b200/csrc -o tools/mma_rate tools/mma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace atom;

// VAR: bit0 = tcgen05.fence::after_thread_sync per group; bit1 = two mbarrier.test_wait per
// group (on completed barriers); bit2 = 12 other warps spin on try_wait of the commit barrier;
// bit3 = other warps loop on tcgen05.wait::ld + fence::before_thread_sync; bit4 = commit to a
// rotating barrier per group (3 barriers)
template <int N, int RS, int VAR = 0>
__global__ void mma_loop(int groups, int fill, unsigned long long* cyc, int spin = 0) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t bar;
  __shared__ uint64_t bars[3];
  __shared__ uint64_t done_bar;
  __shared__ volatile int stop;
  __shared__ uint32_t tbase;
  const int bytes = RS * (128 + N) * 128;
  uint32_t x = 12345u + threadIdx.x * 7919u + blockIdx.x * 104729u;
  for (int i = threadIdx.x * 4; i < bytes; i += blockDim.x * 4) {
    x = x * 1664525u + 1013904223u;
    uint32_t v = fill == 0 ? 0u : fill == 1 ? x : (x & 0xF0F0F0F0u);
    *reinterpret_cast<uint32_t*>(base + i) = v;
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1); mbar_init(&done_bar, 1);
    for (int i = 0; i < 3; ++i) mbar_init(&bars[i], 1);
    stop = 0;
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&tbase, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = umma_idesc_i8(128, N);
    constexpr int RT = 512 / N;
    long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
      const int u = g % RS;
      const uint32_t a = smem_u32(base + u * 128 * 128);
      const uint32_t b = smem_u32(base + RS * 128 * 128 + u * N * 128);
      const uint32_t d = tbase + (g % RT) * N;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        umma_i8(d, umma_desc_sw128(a + 32 * k), umma_desc_sw128(b + 32 * k), idesc, k > 0);
        if constexpr ((VAR & 64) != 0) {
          if (k == 2) {
            uint32_t z = g;
            for (int i = 0; i < spin; ++i) z = z * 1664525u + 1013904223u;
            if (z == 0x12345678u) cyc[1001] = z;
          }
        }
      }
      if constexpr ((VAR & 16) != 0) umma_commit(&bars[g % 3]);
      else umma_commit(&bar);
      if constexpr ((VAR & 1) != 0) tc_fence_after();
      if constexpr ((VAR & 32) != 0) {   // dependent integer work after the commit
        uint32_t z = g;
        for (int i = 0; i < spin; ++i) z = z * 1664525u + 1013904223u;
        if (z == 0x12345678u) cyc[1001] = z;
      }
      if constexpr ((VAR & 64) != 0) {   // same work between dispatch 2 and 3 (next iteration)
      }
      if constexpr ((VAR & 2) != 0) {
        if (!mbar_test(&done_bar, 1)) cyc[1000] = 1;
      }
    }
    if constexpr ((VAR & 16) != 0) mbar_wait(&bars[(groups - 1) % 3], ((groups - 1) / 3) & 1);
    else mbar_wait(&bar, (groups - 1) & 1);
    long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
    stop = 1;
  } else if (threadIdx.x >= 32 && (threadIdx.x & 31) == 0 && (VAR & 12) != 0) {
    int it = 0;
    while (!stop && it < 50000000) {
      if constexpr ((VAR & 4) != 0) mbar_test(&bar, it & 1);
      if constexpr ((VAR & 8) != 0) { tmem_ld_wait(); tc_fence_before(); }
      ++it;
    }
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tbase, 512); }
}

template <int N, int RS, int VAR = 0>
void run(int sms, int fill, unsigned long long* d, int spin = 0) {
  const int groups = 2000;
  size_t smem = RS * (128 + N) * 128 + 1024;
  cudaFuncSetAttribute(mma_loop<N, RS, VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mma_loop<N, RS, VAR><<<sms, 512, smem>>>(groups, fill, d, spin);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, d, 8 * sms, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0, mn = ~0ull;
  for (int i = 0; i < sms; ++i) { mx = h[i] > mx ? h[i] : mx; mn = h[i] < mn ? h[i] : mn; }
  const char* fs[] = {"zeros", "rand-i8", "rand-16q4"};
  printf("spin=%4d VAR=%2d N=%3d RS=%d %-10s grid=%3d: %.1f clk/group (min %.1f), %.0f MAC/clk/SM  (%s)\n", spin, VAR, N, RS,
         fs[fill], sms, (double)mx / groups, (double)mn / groups,
         128.0 * N * 128 * groups / mx, cudaGetErrorString(e));
  fflush(stdout);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d; cudaMalloc(&d, 2048 * 8);
  run<256, 3, 0>(sms, 1, d);
  run<256, 3, 16>(sms, 1, d);
  run<256, 3, 17>(sms, 1, d);
  run<256, 3, 18>(sms, 1, d);
  run<256, 3, 19>(sms, 1, d);
  run<128, 4, 0>(sms, 1, d);
  run<128, 4, 19>(sms, 1, d);
  return 0;
}
