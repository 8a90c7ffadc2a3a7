// microbench.cu -- sm_100a pipe/TMEM throughput probes that decide the GEMM epilogue design.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
// Prints per-SM throughputs measured with clock64 on one CTA per SM (grid = #SMs).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int NCOL>
__device__ __forceinline__ void ld_x(uint32_t taddr, uint32_t* r);

template <>
__device__ __forceinline__ void ld_x<16>(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

__device__ __forceinline__ void st16(uint32_t taddr, uint32_t v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr), "r"(v));
}

// mode 0: LDTM x16 chunks, wait after every 4 loads; mode 1: STTM x16
__global__ void tmem_bw(int iters, int mode, unsigned long long* cycles, uint32_t* sink) {
  __shared__ uint32_t base;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = base + ((uint32_t)((warp & 3) * 32) << 16) + ((warp / 4) % 8) * 64;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (mode == 0) {
      uint32_t r[64];
      ld_x<16>(t, r);
      ld_x<16>(t + 16, r + 16);
      ld_x<16>(t + 32, r + 32);
      ld_x<16>(t + 48, r + 48);
      asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
      for (int k = 0; k < 64; ++k) acc ^= r[k];
    } else if (mode == 2) {
      uint32_t r[64];
      ld_x<16>(t, r);
      ld_x<16>(t + 16, r + 16);
      ld_x<16>(t + 32, r + 32);
      ld_x<16>(t + 48, r + 48);
      asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
      for (int k = 0; k < 64; ++k) acc ^= r[k];
      st16(t, i);
      st16(t + 16, i);
      st16(t + 32, i);
      st16(t + 48, i);
      asm volatile("tcgen05.wait::st.sync.aligned;");
    } else {
      st16(t, i);
      st16(t + 16, i);
      st16(t + 32, i);
      st16(t + 48, i);
      asm volatile("tcgen05.wait::st.sync.aligned;");
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}

// FP pipe probes: mode 0 FFMA, 1 FFMA2, 2 FADD2, 3 FMUL2, 4 I2FP, 5 FFMA with imm
__global__ void fp_tput(int iters, int mode, unsigned long long* cycles, float* sink) {
  float a[8], b = 1.0001f * threadIdx.x;
  float2 a2[8], b2 = make_float2(b, b + 1.f), c2 = make_float2(0.999f, 0.998f);
  int ia[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    a[k] = k;
    a2[k] = make_float2(k, k + 0.5f);
    ia[k] = k * 7 + threadIdx.x;
  }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (mode == 0) a[k] = fmaf(a[k], b, 0.5f * b);
      else if (mode == 1) a2[k] = __ffma2_rn(a2[k], b2, c2);
      else if (mode == 2) a2[k] = __fadd2_rn(a2[k], b2);
      else if (mode == 3) a2[k] = __fmul2_rn(a2[k], c2);
      else if (mode == 4) { a[k] += __int2float_rn(ia[k]); ia[k] += 3; }
      else a[k] = fmaf(a[k], 0.999f, 1.0f);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k] + a2[k].x + a2[k].y;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, sms * sizeof(unsigned long long));
  cudaMalloc(&sink, sms * 1024 * sizeof(uint32_t));
  unsigned long long h[256];
  for (int mode = 0; mode < 3; ++mode)
    for (int warps : {4, 8, 16}) {
      int iters = 2000;
      tmem_bw<<<sms, warps * 32>>>(iters, mode, cyc, sink);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("tmem err %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
      double bytes = (double)iters * warps * 32 * 64 * 4 * (mode == 2 ? 2 : 1);
      printf("TMEM %s warps=%d : %.1f B/clk/SM (cycles %llu)\n",
             mode == 0 ? "ld" : mode == 1 ? "st" : "ld+st", warps, bytes / h[0], h[0]);
    }
  const char* names[] = {"FFMA", "FFMA2", "FADD2", "FMUL2", "I2FP+FADD", "FFMA-imm"};
  for (int mode = 0; mode < 6; ++mode)
    for (int warps : {8, 16}) {
      int iters = 4000;
      fp_tput<<<sms, warps * 32>>>(iters, mode, cyc, reinterpret_cast<float*>(sink));
      cudaDeviceSynchronize();
      cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
      double inst = (double)iters * 8 * warps;  // warp-instructions (per mode unit)
      printf("%-10s warps=%2d : %.2f warp-inst/clk/SM  (%.0f lane-results/clk/SM)\n", names[mode],
             warps, inst / h[0], inst * 32 * ((mode >= 1 && mode <= 3) ? 2 : 1) / h[0]);
    }
  return 0;
}
