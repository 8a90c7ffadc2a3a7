// l2_bw.cu -- L2 -> shared memory throughput on B200 (development probe, not product).
// Every CTA (one per SM) streams CHUNK-byte cp.async.bulk copies from an L2-resident buffer into
// a ring of shared-memory slots (one issuing thread, mbarrier completion).  `share` CTAs with
// consecutive ids read the same addresses at about the same time (the activation-tile reuse
// pattern of the GEMM); the working set is ws bytes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2310_19102_b200/csrc -o tools/l2_bw tools/l2_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace atom;

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

constexpr int NB = 6;
__global__ void __launch_bounds__(32, 1) l2bw(const uint8_t* buf, size_t ws, int chunk, int iters,
                                              int share, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((128 - (smem_u32(smem_raw) & 127)) & 127);
  __shared__ uint64_t bar[NB];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < NB; ++i) mbar_init(&bar[i], 1);
  fence_mbar_init();
  const int grp = blockIdx.x / share;
  const int ngrp = (gridDim.x + share - 1) / share;
  const size_t slice = ws / ngrp / chunk * chunk;
  const uint8_t* src0 = buf + grp * slice;
  size_t off = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int s = it % NB;
    if (it >= NB) mbar_wait_spin(&bar[s], ((it / NB) - 1) & 1);
    mbar_arrive_expect_tx(&bar[s], chunk);
    bulk_g2s(base + s * chunk, src0 + off, chunk, &bar[s]);
    off += chunk;
    if (off >= slice) off = 0;
  }
  for (int it = iters - NB; it < iters; ++it) mbar_wait_spin(&bar[it % NB], (it / NB) & 1);
  out[blockIdx.x] = clock64() - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t max_ws = 256ull << 20;
  uint8_t* buf;
  cudaMalloc(&buf, max_ws);
  cudaMemset(buf, 1, max_ws);
  long long* out;
  cudaMalloc(&out, sizeof(long long) * 1024);
  cudaFuncSetAttribute(l2bw, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t wss[] = {8ull << 20, 32ull << 20, 64ull << 20, 96ull << 20, 256ull << 20};
  const int chunks[] = {8192, 16384, 32768};
  const int shares[] = {1, 2, 4, 8};
  for (size_t ws : wss)
    for (int chunk : chunks)
      for (int share : shares) {
        if (share > 1 && chunk != 16384) continue;
        const int iters = 2000;
        const size_t smem = NB * chunk + 128;
        l2bw<<<sms, 32, smem>>>(buf, ws, chunk, iters, share, out);   // warm
        cudaEventRecord(e0);
        for (int r = 0; r < 3; ++r) l2bw<<<sms, 32, smem>>>(buf, ws, chunk, iters, share, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = 3.0 * sms * iters * (double)chunk;
        long long h[1024];
        cudaMemcpy(h, out, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("ws=%4zu MiB chunk=%5d share=%d : %7.2f TB/s  (%.1f B/clk/SM by clock64, max CTA)\n",
               ws >> 20, chunk, share, bytes / (ms * 1e-3) / 1e12,
               (double)iters * chunk / (double)mx);
      }
  cudaError_t err = cudaDeviceSynchronize();
  printf("rc=%d %s\n", (int)err, cudaGetErrorString(err));
  return 0;
}
