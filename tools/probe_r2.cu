// probe_r2.cu -- round-2 design probes for the W4A4 GEMM on B200 (development tool, not product).
//   E1  tcgen05.mma kind::f8f6f4 (E4M3) rate, cta_group::1, N = 256 / 128
//   E2  the same MMA stream while 8 warps stream LDS.128 + STS.128 (shared-memory contention)
//   E3  the same MMA stream while one thread streams cp.async.bulk global->shared (TMA writes)
//   E4  cta_group::2 kind::f8f6f4, M = 256, N = 256 / 128 (CTA pair), leader-timed
//   E5  TMEM -> register load bandwidth: 8 warps, 32x32b.x16/x32/x64 and 16x256b.x8/x16
//   E6  synthetic epilogue: 8 warps x {TMEM load 128 cols, FMUL2 + FFMA2 per column pair with
//       the column scales from shared memory} per "group", alone and under a running MMA stream
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2310_19102_b200/csrc -o tools/probe_r2 tools/probe_r2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace atom;

__host__ __device__ constexpr uint32_t idesc_f8(uint32_t m, uint32_t n) {
  return (1u << 4) | ((n >> 3) << 17) | ((m >> 4) << 24);   // D f32, A = B = E4M3, K-major
}
__device__ __forceinline__ void umma_f8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void umma_f8_cg2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit_cg2(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---- TMEM loads of several shapes ---------------------------------------------------------
#define R8(b) "=r"(r[b + 0]), "=r"(r[b + 1]), "=r"(r[b + 2]), "=r"(r[b + 3]), "=r"(r[b + 4]), \
              "=r"(r[b + 5]), "=r"(r[b + 6]), "=r"(r[b + 7])
__device__ __forceinline__ void ld32x32b_x32(uint32_t t, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,"
               "%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31},"
               " [%32];"
               : R8(0), R8(8), R8(16), R8(24) : "r"(t) : "memory");
}
__device__ __forceinline__ void ld32x32b_x64(uint32_t t, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,"
               "%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
               "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,"
               "%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
               : R8(0), R8(8), R8(16), R8(24), R8(32), R8(40), R8(48), R8(56) : "r"(t) : "memory");
}
__device__ __forceinline__ void ld16x256b_x8(uint32_t t, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,"
               "%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31},"
               " [%32];"
               : R8(0), R8(8), R8(16), R8(24) : "r"(t) : "memory");
}
__device__ __forceinline__ void ld16x256b_x16(uint32_t t, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,"
               "%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
               "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,"
               "%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
               : R8(0), R8(8), R8(16), R8(24), R8(32), R8(40), R8(48), R8(56) : "r"(t) : "memory");
}

// ---- E1/E2/E3: cta_group::1 MMA stream with optional LSU / bulk-copy contention -------------
// smem: A [RS][128][128] | B [RS][N][128] | X 64 KB scratch (LSU or bulk-copy target)
template <int N>
__global__ void __launch_bounds__(512, 1) e123(int groups, int lsu_iters, int bulk_iters,
                                               const uint8_t* gsrc, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  constexpr int RS = 2;
  uint8_t* A = base;
  uint8_t* B = A + RS * 128 * 128;
  uint8_t* X = B + RS * N * 128;
  __shared__ uint64_t bar, bbar[2];
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x * 16; i < RS * (128 + N) * 128 + 65536; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(base + i) = make_uint4(0x38383838u, 0x40404040u, 0xB8B8B8B8u, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bbar[0], 1); mbar_init(&bbar[1], 1); fence_mbar_init(); }
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&tbase, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x == 0 && groups > 0) {
    constexpr uint32_t id = idesc_f8(128, N);
    constexpr int RT = 512 / N;
    long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
      const uint32_t a = smem_u32(A + (g % RS) * 128 * 128), b = smem_u32(B + (g % RS) * N * 128);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        umma_f8(tbase + (g % RT) * N, umma_desc_sw128(a + 32 * k), umma_desc_sw128(b + 32 * k), id,
                k > 0);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    out[0] = clock64() - t0;
  }
  if (threadIdx.x == 32 && bulk_iters > 0) {   // one thread streams 16 KB bulk copies into X
    long long t0 = clock64();                    // two 32 KB batches in flight (bars bbar[0/1])
    uint32_t ph[2] = {0, 0};
    for (int i = 0; i < bulk_iters + 2; ++i) {
      const int s = i & 1;
      if (i >= 2) { mbar_wait(&bbar[s], ph[s]); ph[s] ^= 1; }
      if (i < bulk_iters) {
        mbar_arrive_expect_tx(&bbar[s], 2 * 16384);
        for (int j = 0; j < 2; ++j)
          bulk_g2s(X + (s * 2 + j) * 16384, gsrc + ((i * 2 + j) & 63) * 16384, 16384, &bbar[s]);
      }
    }
    out[2] = clock64() - t0;
  }
  if (warp >= 8 && lsu_iters > 0) {
    const int t = threadIdx.x - 256;
    uint4* x = reinterpret_cast<uint4*>(X);
    uint4 v = make_uint4(t, 1, 2, 3);
    long long t0 = clock64();
    for (int i = 0; i < lsu_iters; ++i) {
      uint4 a = x[(t + 256 * (i & 3)) & 4095];
      v.x ^= a.x; v.y += a.y; v.z ^= a.z; v.w += a.w;
      x[(t + 256 * ((i + 1) & 3) + 2048) & 4095] = make_uint4(v.x, v.y + i, v.z, v.w);
    }
    long long t1 = clock64();
    if (t == 0) out[1] = t1 - t0;
    if (v.x == 0x1234567) out[3] = v.y;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tbase, 512); }
}

// ---- E4: cta_group::2 -----------------------------------------------------------------------
template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) e4(int groups, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* A = base;                  // this CTA's 128 rows of A (M = 256 over the pair)
  uint8_t* B = A + 2 * 128 * 128;     // this CTA's N/2 rows of B
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x * 16; i < 2 * (128 + N / 2) * 128; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(base + i) = make_uint4(0x38383838u, 0x40404040u, 0xB8B8B8B8u, 0);
  fence_proxy_async_smem();
  const uint32_t rank = cluster_rank();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tbase)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (rank == 0 && threadIdx.x == 0) {
    constexpr uint32_t id = idesc_f8(256, N);
    constexpr int RT = 512 / N;
    long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
      const uint32_t a = smem_u32(A + (g & 1) * 128 * 128), b = smem_u32(B + (g & 1) * (N / 2) * 128);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        umma_f8_cg2(tbase + (g % RT) * N, umma_desc_sw128(a + 32 * k), umma_desc_sw128(b + 32 * k),
                    id, k > 0);
    }
    commit_cg2(&bar, 3);
    mbar_wait(&bar, 0);
    out[0] = clock64() - t0;
  }
  if (rank == 1 && threadIdx.x == 0) {
    mbar_wait(&bar, 0);
    out[1] = 1;
  }
  tc_fence_before();
  cluster_sync_all();
  if (threadIdx.x < 32) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512)
                 : "memory");
  }
}

// ---- E5/E6: TMEM loads and the synthetic epilogue --------------------------------------------
// MODE: 0 = 32x32b.x16 (8 loads per 128 cols), 1 = x32, 2 = x64, 3 = 16x256b.x8, 4 = 16x256b.x16
// MATH: 0 = loads only; 1 = + FMUL2/FFMA2 dequant-accumulate (32x32b: column scales by LDS.128;
//       16x256b: LDS.64)
// mma: a concurrent kind::f8f6f4 128x256 stream into TMEM columns 256..511 (reads 0..255 here)
template <int MODE, int MATH>
__global__ void __launch_bounds__(384, 1) e56(int groups, int mma_groups, long long* out,
                                              float* sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ __align__(16) float sa[256];
  for (int i = threadIdx.x * 16; i < (128 + 256) * 128; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(base + i) = make_uint4(0x38383838u, 0x40404040u, 0xB8B8B8B8u, 0);
  for (int i = threadIdx.x; i < 256; i += blockDim.x) sa[i] = 1.0f + i * 1e-3f;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) tmem_alloc(&tbase, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 8 && lane == 0 && mma_groups > 0) {
    constexpr uint32_t id = idesc_f8(128, 256);
    const uint32_t a = smem_u32(base), b = smem_u32(base + 128 * 128);
    long long t0 = clock64();
    for (int g = 0; g < mma_groups; ++g)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        umma_f8(tbase + 256, umma_desc_sw128(a + 32 * k), umma_desc_sw128(b + 32 * k), id, k > 0);
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    out[1] = clock64() - t0;
  }
  if (warp < 8) {
    const int q = warp & 3, half = warp >> 2;          // lane quarter, column half (128 cols)
    const uint32_t t0a = tbase + (static_cast<uint32_t>(q * 32) << 16) + half * 128;
    float acc[128];
#pragma unroll
    for (int i = 0; i < 128; ++i) acc[i] = 0.0f;
    const float sw = 0.5f + lane * 1e-3f;
    uint32_t r[64];
    long long c0 = clock64();
    for (int g = 0; g < groups; ++g) {
      if constexpr (MODE <= 2) {
        constexpr int W = MODE == 0 ? 16 : MODE == 1 ? 32 : 64;
#pragma unroll
        for (int c = 0; c < 128; c += W) {
          if constexpr (W == 16) tmem_ld16p(t0a + c, r);
          else if constexpr (W == 32) ld32x32b_x32(t0a + c, r);
          else ld32x32b_x64(t0a + c, r);
          tmem_ld_wait();
          if constexpr (MATH) {
#pragma unroll
            for (int j = 0; j < W; j += 4) {
              const float4 s4 = *reinterpret_cast<const float4*>(&sa[half * 128 + c + j]);
              float2 g0 = __fmul2_rn(make_float2(__uint_as_float(r[j]), __uint_as_float(r[j + 1])),
                                     make_float2(sw, sw));
              float2 g1 = __fmul2_rn(make_float2(__uint_as_float(r[j + 2]), __uint_as_float(r[j + 3])),
                                     make_float2(sw, sw));
              float2 a0 = __ffma2_rn(make_float2(s4.x, s4.y), g0, make_float2(acc[c + j], acc[c + j + 1]));
              float2 a1 = __ffma2_rn(make_float2(s4.z, s4.w), g1, make_float2(acc[c + j + 2], acc[c + j + 3]));
              acc[c + j] = a0.x; acc[c + j + 1] = a0.y; acc[c + j + 2] = a1.x; acc[c + j + 3] = a1.y;
            }
          } else {
#pragma unroll
            for (int j = 0; j < W; ++j) acc[(c + j) & 127] += __uint_as_float(r[j]);
          }
        }
      } else {
        // 16x256b: two loads (lanes +0 and +16 of the quarter) per 8*X columns; thread holds,
        // per 8-col chunk, cols 2(l%4)+{0,1} of rows l/4 and l/4+8
        constexpr int X = MODE == 3 ? 8 : 16;   // chunks per load
#pragma unroll
        for (int c = 0; c < 128; c += 8 * X) {  // this warp: 128 columns x 32 lanes = 2 x 16 lanes
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if constexpr (X == 8) ld16x256b_x8(t0a + (static_cast<uint32_t>(16 * h) << 16) + c, r);
            else ld16x256b_x16(t0a + (static_cast<uint32_t>(16 * h) << 16) + c, r);
            tmem_ld_wait();
#pragma unroll
            for (int ch = 0; ch < X; ++ch) {
              const int ai = (h * 64 + (c / 8 + ch) * 4) & 127;
              if constexpr (MATH) {
                const float2 s2 = *reinterpret_cast<const float2*>(&sa[half * 128 + c + 8 * ch + 2 * (lane & 3)]);
                float2 g0 = __fmul2_rn(make_float2(__uint_as_float(r[4 * ch]), __uint_as_float(r[4 * ch + 1])),
                                       make_float2(sw, sw));
                float2 g1 = __fmul2_rn(make_float2(__uint_as_float(r[4 * ch + 2]), __uint_as_float(r[4 * ch + 3])),
                                       make_float2(sw, sw));
                float2 a0 = __ffma2_rn(s2, g0, make_float2(acc[ai], acc[ai + 1]));
                float2 a1 = __ffma2_rn(s2, g1, make_float2(acc[ai + 2], acc[ai + 3]));
                acc[ai] = a0.x; acc[ai + 1] = a0.y; acc[ai + 2] = a1.x; acc[ai + 3] = a1.y;
              } else {
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[ai + v] += __uint_as_float(r[4 * ch + v]);
              }
            }
          }
        }
      }
    }
    long long c1 = clock64();
    if (lane == 0) out[2 + warp] = c1 - c0;
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < 128; ++i) s += acc[i];
    if (s == 1.2345f) sink[threadIdx.x] = s;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tbase, 512); }
}


// ---- E7: epilogue math under an MMA stream: where does the slowdown come from? ----------------
// NW epilogue warps (8: 128 cols each; 16: 64 cols each), software-pipelined x16 TMEM loads,
// FMUL2 + FFMA2 per column pair; MMA thread in warp MW with PACE: 0 = back-to-back issue,
// 1 = 4 MMAs + commit + wait (suspend) per group, 2 = as 1 with spin test_wait.
template <int NW, int PACE>
__global__ void __launch_bounds__((NW + 2) * 32, 1) e7(int groups, int mma_groups, int mw, long long* out,
                                             float* sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tbase;
  __shared__ __align__(16) float sa[256];
  for (int i = threadIdx.x * 16; i < (128 + 256) * 128; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(base + i) = make_uint4(0x38383838u, 0x40404040u, 0xB8B8B8B8u, 0);
  for (int i = threadIdx.x; i < 256; i += blockDim.x) sa[i] = 1.0f + i * 1e-3f;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); fence_mbar_init(); }
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) tmem_alloc(&tbase, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == mw && lane == 0 && mma_groups > 0) {
    constexpr uint32_t id = idesc_f8(128, 256);
    const uint32_t a = smem_u32(base), b = smem_u32(base + 128 * 128);
    long long t0 = clock64();
    uint32_t ph = 0;
    for (int g = 0; g < mma_groups; ++g) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        umma_f8(tbase + 256, umma_desc_sw128(a + 32 * k), umma_desc_sw128(b + 32 * k), id, k > 0);
      if (PACE != 0) {
        umma_commit(&bar[g & 1]);
        if (g >= 1) {   // keep one group queued behind the running one
          if (PACE == 1) mbar_wait(&bar[(g - 1) & 1], ((g - 1) >> 1) & 1);
          else mbar_wait_test(&bar[(g - 1) & 1], ((g - 1) >> 1) & 1);
        }
      }
    }
    if (PACE == 0) { umma_commit(&bar[0]); mbar_wait(&bar[0], 0); }
    else {
      const int g = mma_groups - 1;
      mbar_wait(&bar[g & 1], (g >> 1) & 1);
    }
    out[1] = clock64() - t0;
  }
  if (warp < NW) {
    constexpr int COLS = 128 * 8 / NW;                  // columns per warp
    const int q = warp & 3, part = warp >> 2;
    const uint32_t t0a = tbase + (static_cast<uint32_t>(q * 32) << 16) + part * COLS;
    float acc[COLS];
#pragma unroll
    for (int i = 0; i < COLS; ++i) acc[i] = 0.0f;
    const float sw = 0.5f + lane * 1e-3f;
    uint32_t r[2][16];
    long long c0 = clock64();
    for (int g = 0; g < groups; ++g) {
      tmem_ld16p(t0a, r[0]);
#pragma unroll
      for (int bi = 0; bi < COLS / 16; ++bi) {
        if (bi + 1 < COLS / 16) tmem_ld16p(t0a + 16 * (bi + 1), r[(bi + 1) & 1]);
        else tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; j += 4) {
          const int c = bi * 16 + j;
          uint32_t* rv = r[bi & 1] + j;
          const float4 s4 = *reinterpret_cast<const float4*>(&sa[part * COLS + c]);
          float2 g0 = __fmul2_rn(make_float2(__uint_as_float(rv[0]), __uint_as_float(rv[1])), make_float2(sw, sw));
          float2 g1 = __fmul2_rn(make_float2(__uint_as_float(rv[2]), __uint_as_float(rv[3])), make_float2(sw, sw));
          float2 a0 = __ffma2_rn(make_float2(s4.x, s4.y), g0, make_float2(acc[c], acc[c + 1]));
          float2 a1 = __ffma2_rn(make_float2(s4.z, s4.w), g1, make_float2(acc[c + 2], acc[c + 3]));
          acc[c] = a0.x; acc[c + 1] = a0.y; acc[c + 2] = a1.x; acc[c + 3] = a1.y;
        }
      }
    }
    long long c1 = clock64();
    if (lane == 0) out[2 + warp] = c1 - c0;
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < COLS; ++i) s += acc[i];
    if (s == 1.2345f) sink[threadIdx.x] = s;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tbase, 512); }
}

// ---- E8: which part of the epilogue does a running MMA stream slow down? ---------------------
// V: 0 = TMEM loads + math with scales in registers (no LDS); 1 = no TMEM loads (partials in
// registers) + math with LDS.128 column scales; 2 = dependent LDS chain latency (lane 0 of each
// warp); 3 = TMEM loads + math with LDS, scales for the NEXT 16 columns prefetched one batch ahead
template <int V>
__global__ void __launch_bounds__(320, 1) e8(int groups, int mma_groups, long long* out, float* sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ __align__(16) float sa[256];
  __shared__ int chain[1024];
  for (int i = threadIdx.x * 16; i < (128 + 256) * 128; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(base + i) = make_uint4(0x38383838u, 0x40404040u, 0xB8B8B8B8u, 0);
  for (int i = threadIdx.x; i < 256; i += blockDim.x) sa[i] = 1.0f + i * 1e-3f;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) chain[i] = (i * 37 + 11) & 1023;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) tmem_alloc(&tbase, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 8 && lane == 0 && mma_groups > 0) {
    constexpr uint32_t id = idesc_f8(128, 256);
    const uint32_t a = smem_u32(base), b = smem_u32(base + 128 * 128);
    long long t0 = clock64();
    for (int g = 0; g < mma_groups; ++g)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        umma_f8(tbase + 256, umma_desc_sw128(a + 32 * k), umma_desc_sw128(b + 32 * k), id, k > 0);
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    out[1] = clock64() - t0;
  }
  if (warp < 8) {
    const int q = warp & 3, part = warp >> 2;
    const uint32_t t0a = tbase + (static_cast<uint32_t>(q * 32) << 16) + part * 128;
    float acc[128];
#pragma unroll
    for (int i = 0; i < 128; ++i) acc[i] = 0.0f;
    const float sw = 0.5f + lane * 1e-3f;
    uint32_t r[2][16];
    float4 s4n[4];
    long long c0 = clock64();
    if constexpr (V == 2) {
      int idx = lane;
      for (int g = 0; g < groups * 16; ++g) idx = chain[idx];
      acc[0] = idx;
    } else
    for (int g = 0; g < groups; ++g) {
      if constexpr (V != 1) tmem_ld16p(t0a, r[0]);
      else {
#pragma unroll
        for (int v = 0; v < 16; ++v) { r[0][v] = __float_as_uint(g + v * 0.5f); r[1][v] = r[0][v] ^ 1; }
      }
      if constexpr (V == 3) {
#pragma unroll
        for (int j = 0; j < 4; ++j) s4n[j] = *reinterpret_cast<const float4*>(&sa[part * 128 + 4 * j]);
      }
#pragma unroll
      for (int bi = 0; bi < 8; ++bi) {
        if constexpr (V != 1) {
          if (bi + 1 < 8) tmem_ld16p(t0a + 16 * (bi + 1), r[(bi + 1) & 1]);
          else tmem_ld_wait();
        }
        float4 s4c[4];
        if constexpr (V == 3) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            s4c[j] = s4n[j];
            if (bi + 1 < 8) s4n[j] = *reinterpret_cast<const float4*>(&sa[part * 128 + 16 * (bi + 1) + 4 * j]);
          }
        }
#pragma unroll
        for (int j = 0; j < 16; j += 4) {
          const int c = bi * 16 + j;
          uint32_t* rv = r[(V == 1) ? (j >> 3) & 1 : bi & 1] + j;
          float4 s4;
          if constexpr (V == 0) s4 = make_float4(sw, sw + 1, sw + 2, sw + 3);
          else if constexpr (V == 3) s4 = s4c[j / 4];
          else s4 = *reinterpret_cast<const float4*>(&sa[part * 128 + c]);
          float2 g0 = __fmul2_rn(make_float2(__uint_as_float(rv[0]), __uint_as_float(rv[1])), make_float2(sw, sw));
          float2 g1 = __fmul2_rn(make_float2(__uint_as_float(rv[2]), __uint_as_float(rv[3])), make_float2(sw, sw));
          float2 a0 = __ffma2_rn(make_float2(s4.x, s4.y), g0, make_float2(acc[c], acc[c + 1]));
          float2 a1 = __ffma2_rn(make_float2(s4.z, s4.w), g1, make_float2(acc[c + 2], acc[c + 3]));
          acc[c] = a0.x; acc[c + 1] = a0.y; acc[c + 2] = a1.x; acc[c + 3] = a1.y;
        }
      }
    }
    long long c1 = clock64();
    if (lane == 0) out[2 + warp] = c1 - c0;
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < 128; ++i) s += acc[i];
    if (s == 1.2345f) sink[threadIdx.x] = s;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tbase, 512); }
}

int main(int argc, char** argv) {
  const int only7 = argc > 1;
  long long* d;
  float* sink;
  uint8_t* gsrc;
  cudaMalloc(&d, 64 * sizeof(long long));
  cudaMalloc(&sink, 4096 * sizeof(float));
  cudaMalloc(&gsrc, 64 * 16384);
  cudaMemset(gsrc, 0, 64 * 16384);
  long long h[64];
  auto run = [&](const char* what) {
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) printf("%s: ERROR %s\n", what, cudaGetErrorString(e));
    return e == cudaSuccess;
  };
  // ---- E1/E2/E3
  if (!only7) {
    const int G = 2000, LI = 20000, BI = 1600;
    const int smem256 = 2 * (128 + 256) * 128 + 65536 + 1024, smem128 = 2 * (128 + 128) * 128 + 65536 + 1024;
    cudaFuncSetAttribute(e123<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem256);
    cudaFuncSetAttribute(e123<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem128);
    struct { int g, l, b; const char* name; } cs[] = {
        {G, 0, 0, "MMA only"}, {0, LI, 0, "LSU only"}, {G, LI, 0, "MMA + LSU"},
        {0, 0, BI, "bulk only"}, {G, 0, BI, "MMA + bulk"}, {G, LI, BI, "MMA + LSU + bulk"}};
    for (int n = 0; n < 2; ++n)
      for (auto& c : cs) {
        cudaMemset(d, 0, sizeof(h));
        if (n == 0) e123<256><<<1, 512, smem256>>>(c.g, c.l, c.b, gsrc, d);
        else e123<128><<<1, 512, smem128>>>(c.g, c.l, c.b, gsrc, d);
        if (!run(c.name)) continue;
        printf("E1-3 N=%d %-18s MMA %7.1f clk/group | LSU %6.1f B/clk | bulk %6.1f B/clk\n",
               n == 0 ? 256 : 128, c.name, c.g ? (double)h[0] / c.g : 0.0,
               h[1] ? 256.0 * 32 * c.l / h[1] : 0.0, h[2] ? 32768.0 * c.b / h[2] : 0.0);
      }
  }
  // ---- E4
  if (!only7) {
    const int G = 2000;
    const int s256 = 2 * (128 + 128) * 128 + 1024, s128 = 2 * (128 + 64) * 128 + 1024;
    cudaFuncSetAttribute(e4<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, s256);
    cudaFuncSetAttribute(e4<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, s128);
    cudaMemset(d, 0, sizeof(h));
    e4<256><<<2, 128, s256>>>(G, d);
    if (run("E4 N=256")) printf("E4 cta_group::2 M=256 N=256: %.1f clk/group (per SM 128x256x128)\n", (double)h[0] / G);
    cudaMemset(d, 0, sizeof(h));
    e4<128><<<2, 128, s128>>>(G, d);
    if (run("E4 N=128")) printf("E4 cta_group::2 M=256 N=128: %.1f clk/group (per SM 128x128x128)\n", (double)h[0] / G);
  }
  // ---- E5/E6
  if (!only7) {
    const int G = 400, smem = (128 + 256) * 128 + 1024;
#define E56(MO, MA)                                                                                \
  do {                                                                                             \
    cudaFuncSetAttribute(e56<MO, MA>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);          \
    for (int withmma = 0; withmma < 2; ++withmma) {                                                \
      cudaMemset(d, 0, sizeof(h));                                                                 \
      e56<MO, MA><<<1, 384, smem>>>(G, withmma ? 4 * G : 0, d, sink);                              \
      if (!run("E56")) break;                                                                      \
      long long mx = 0;                                                                            \
      for (int w = 0; w < 8; ++w) mx = h[2 + w] > mx ? h[2 + w] : mx;                              \
      printf("E5/6 mode %d math %d mma %d: %.1f clk per 128x256 group (%.0f B/clk TMEM read)%s\n", \
             MO, MA, withmma, (double)mx / G, 131072.0 * G / mx,                                   \
             withmma ? "" : "");                                                                   \
      if (withmma) printf("      (MMA stream %.1f clk/group)\n", (double)h[1] / (4 * G));        \
    }                                                                                              \
  } while (0)
    E56(0, 0); E56(1, 0); E56(2, 0); E56(3, 0); E56(4, 0);
    E56(0, 1); E56(1, 1); E56(2, 1); E56(3, 1); E56(4, 1);
  }
  // ---- E7
  if (argc > 1 && argv[1][0] == '7') {
    const int G = 400, smem = (128 + 256) * 128 + 1024;
#define E7(NW, PACE, MW)                                                                           \
  do {                                                                                             \
    cudaFuncSetAttribute(e7<NW, PACE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);         \
    for (int withmma = 0; withmma < 2; ++withmma) {                                                \
      if (!withmma && (PACE != 0 || MW != NW)) continue;                                           \
      cudaMemset(d, 0, sizeof(h));                                                                 \
      e7<NW, PACE><<<1, (NW + 2) * 32, smem>>>(G, withmma ? 4 * G : 0, MW, d, sink);                         \
      if (!run("E7")) break;                                                                       \
      long long mx = 0;                                                                            \
      printf("E7 NW=%d pace=%d mma_warp=%d mma=%d: per-warp clk/group:", NW, PACE, MW, withmma);   \
      for (int w = 0; w < NW; ++w) { mx = h[2 + w] > mx ? h[2 + w] : mx; printf(" %.0f", (double)h[2 + w] / G); } \
      printf(" | max %.1f", (double)mx / G);                                                       \
      if (withmma) printf(" | MMA %.1f clk/group", (double)h[1] / (4 * G));                       \
      printf("\n");                                                                                \
    }                                                                                              \
  } while (0)
    E7(8, 0, 8); E7(8, 0, 9); E7(8, 1, 8); E7(8, 2, 8); E7(8, 1, 9);
    E7(16, 0, 16); E7(16, 1, 16); E7(16, 2, 16); E7(16, 1, 17);
  }
  // ---- E8
  {
    const int G = 400, smem = (128 + 256) * 128 + 1024;
#define E8(V)                                                                                      \
  do {                                                                                             \
    cudaFuncSetAttribute(e8<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);                \
    for (int withmma = 0; withmma < 2; ++withmma) {                                                \
      cudaMemset(d, 0, sizeof(h));                                                                 \
      e8<V><<<1, 320, smem>>>(G, withmma ? 4 * G : 0, d, sink);                                    \
      if (!run("E8")) break;                                                                       \
      long long mx = 0;                                                                            \
      for (int w = 0; w < 8; ++w) mx = h[2 + w] > mx ? h[2 + w] : mx;                              \
      if (V == 2) printf("E8 V=2 mma=%d: dependent LDS latency %.1f clk\n", withmma, (double)mx / (16 * G)); \
      else printf("E8 V=%d mma=%d: %.1f clk per group%s\n", V, withmma, (double)mx / G, withmma ? "" : ""); \
    }                                                                                              \
  } while (0)
    E8(0); E8(1); E8(2); E8(3);
  }
  return 0;
}
