// mxfp.cu -- NEXT-2, Atom (FP): the paper's FP4 variant on Blackwell's MX block-scaled tensor
// cores (sm_100a).
//
// Paper: "we also evaluate the effectiveness of Atom in FP4 ... quantizing both weights and
// activations into FP4" and "group quantization with the MX format is supported by NVIDIA
// Blackwell GPUs.  We expect this hardware feature can mitigate the group quantization overhead"
// (Section 6; Table 5).  Same method as the INT path -- channel reorder,
// outlier channels kept in higher precision, fine-grained group quantization --
// with MX elements and scales (readings G21-G24):
//   normal channels  MXFP4: E2M1, blocks of 32 reordered channels, one UE8M0 scale per block/row
//   128 outliers     MXFP8: E4M3, blocks of 32, UE8M0 scales
//   conversion       OCP MX v1.0 6.3: shared_exp = floor(log2 amax) - emax_elem, RNE, saturate
//
// B200 design: the group dequantization the INT path pays in its epilogue (2 fp32 ops per output
// per group) is done by the tensor core itself: tcgen05.mma.kind::mxf4.block_scale.block32 reads
// packed E2M1 operands straight from the TMA-written (128B-swizzled) shared memory -- no weight
// expansion warps -- and applies the per-block scales from TMEM; the outlier group runs
// kind::mxf8f6f4.block_scale into the same fp32 accumulator.  One accumulator per tile over all
// of K; the epilogue only converts fp32 -> fp16 once per tile.
//   * Tile 128 tokens (MMA M, TMEM lanes) x 224 channels (MMA N): two accumulator buffers
//     (2 x 224 TMEM columns) plus 24 scale-factor columns fit the 512-column TMEM, so the
//     epilogue of tile i overlaps the MMAs of tile i+1 (at N = 28672: 1024 tiles = 6.9 waves).
//   * Stage = 256 K-elements (128 bytes of packed E2M1 per row = one SW128 atom): TMA of the
//     activation and weight tiles and of the canonical scale bytes [rows][16 B] (two stages'
//     worth; the stage uses 8), a transposer warp turns the scale bytes into the
//     tcgen05.cp 32x128b.warpx4 images (TMEM lane l, column c = the 4 scale bytes of row 32c+l of
//     a 128-row block), the MMA thread copies them to TMEM (tcgen05.cp and tcgen05.mma execute
//     in issue order) and issues 4 MMAs of K = 64 (scale ids 0 / 2 of the chunk's word).
//   * Warp roles (12 warps): 0 TMA producer, 1 MMA issuer, 2 scale transposer, 3 idle,
//     4-11 epilogue (warp % 4 = TMEM lane quarter, (warp - 4) / 4 = column half).
#include <cstdint>
#include <mutex>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "internal.h"
#include "ptx.cuh"

namespace atom {

// =============================================================================================
// MX reorder + quantize (activations online, weights offline)
// =============================================================================================
constexpr int kMxqThreads = 256;

__device__ __forceinline__ uint32_t cvt_e2m1x2(float hi, float lo) {
  uint32_t r;   // RNE, saturating to +-6; lo -> bits 0-3, hi -> bits 4-7
  asm("{\n\t.reg .b8 t;\n\tcvt.rn.satfinite.e2m1x2.f32 t, %1, %2;\n\tcvt.u32.u8 %0, t;\n\t}"
      : "=r"(r)
      : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ uint32_t cvt_e4m3x2(float hi, float lo) {
  uint32_t r;   // RNE, saturating to +-448; lo -> bits 0-7, hi -> bits 8-15
  asm("{\n\t.reg .b16 t;\n\tcvt.rn.satfinite.e4m3x2.f32 t, %1, %2;\n\tcvt.u32.u16 %0, t;\n\t}"
      : "=r"(r)
      : "f"(hi), "f"(lo));
  return r;
}

// One CTA per (row, group chunk); the fp16 row is staged in shared memory (one bulk copy), each
// warp quantizes 128-channel groups: lane l owns reordered channels 4l .. 4l+3 (MX block l / 8).
__global__ void __launch_bounds__(kMxqThreads)
mx_reorder_quantize_kernel(const __half* __restrict__ x, int64_t rows, int64_t ldx,
                           const int32_t* __restrict__ perm, int32_t G, int32_t G4,
                           int32_t groups_per_cta, uint8_t* __restrict__ fp4,
                           uint8_t* __restrict__ fp8, uint8_t* __restrict__ sf, int64_t ldsf) {
  extern __shared__ uint4 srow4[];
  const __half* srow = reinterpret_cast<const __half*>(srow4);
  __shared__ uint64_t bar;
  const int64_t row = blockIdx.x;
  const int g_begin = blockIdx.y * groups_per_cta;
  const int g_end = min(G, g_begin + groups_per_cta);
  griddep_wait();
  griddep_launch();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(&bar, static_cast<uint32_t>(ldx) * 2);
    bulk_g2s(srow4, x + row * ldx, static_cast<uint32_t>(ldx) * 2, &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t row4 = static_cast<int64_t>(G4) * 64;
  for (int t = g_begin + warp; t < g_end; t += kMxqThreads / 32) {
    const int4 pj = __ldg(reinterpret_cast<const int4*>(perm + t * 128 + 4 * lane));
    float v[4] = {__half2float(srow[pj.x]), __half2float(srow[pj.y]), __half2float(srow[pj.z]),
                  __half2float(srow[pj.w])};
    float amax = fmaxf(fmaxf(fabsf(v[0]), fabsf(v[1])), fmaxf(fabsf(v[2]), fabsf(v[3])));
#pragma unroll
    for (int off = 1; off < 8; off <<= 1)       // the 8 lanes of one MX block
      amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
    const bool is_fp4 = t < G4;
    // shared_exp = floor(log2 amax) - emax_elem: amax is a normal binary32 (fp16 values are),
    // so floor(log2 amax) is its unbiased exponent field
    const int se = static_cast<int>((__float_as_uint(amax) >> 23) & 0xFFu) - 127 - (is_fp4 ? 2 : 8);
    const uint32_t sbyte = amax == 0.0f ? 0u : static_cast<uint32_t>(se + 127);
    const float mul = amax == 0.0f ? 1.0f : __uint_as_float(static_cast<uint32_t>(127 - se) << 23);
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = __fmul_rn(v[k], mul);   // x / 2^se, exact
    if (is_fp4) {
      const uint32_t b = cvt_e2m1x2(v[1], v[0]) | (cvt_e2m1x2(v[3], v[2]) << 8);
      reinterpret_cast<uint16_t*>(fp4 + row * row4 + t * 64)[lane] = static_cast<uint16_t>(b);
    } else {
      const uint32_t b = cvt_e4m3x2(v[1], v[0]) | (cvt_e4m3x2(v[3], v[2]) << 16);
      reinterpret_cast<uint32_t*>(fp8 + row * 128)[lane] = b;
    }
    // the group's 4 block scale bytes: lanes 0, 8, 16, 24 -> one 32-bit store
    const uint32_t s1 = __shfl_sync(0xffffffffu, sbyte, 8), s2 = __shfl_sync(0xffffffffu, sbyte, 16),
                   s3 = __shfl_sync(0xffffffffu, sbyte, 24);
    if (lane == 0)
      *reinterpret_cast<uint32_t*>(sf + row * ldsf + 4 * t) = sbyte | (s1 << 8) | (s2 << 16) | (s3 << 24);
  }
}

cudaError_t launch_mx_reorder_quantize(const void* x, int64_t rows, int64_t ldx,
                                       const int32_t* perm, int64_t K, int32_t k_outlier,
                                       uint8_t* fp4, uint8_t* fp8, uint8_t* sf, int64_t ldsf,
                                       cudaStream_t stream, int num_sms) {
  const int G = static_cast<int>(K / 128), G4 = static_cast<int>((K - k_outlier) / 128);
  int splits = static_cast<int>((4LL * num_sms + rows - 1) / rows);
  const int max_splits = (G + 7) / 8;
  splits = max(1, min(splits, max_splits));
  const int gpc = (G + splits - 1) / splits;
  splits = (G + gpc - 1) / gpc;
  const size_t smem = static_cast<size_t>(ldx) * sizeof(__half);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(mx_reorder_quantize_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  dim3 grid(static_cast<unsigned>(rows), static_cast<unsigned>(splits));
  return launch_pdl(mx_reorder_quantize_kernel, grid, dim3(kMxqThreads), smem, stream,
                    static_cast<const __half*>(x), rows, ldx, perm, G, G4, gpc, fp4, fp8, sf,
                    ldsf);
}

// =============================================================================================
// MX GEMM: C[m][n] = sum over blocks of 2^(sa + sw) * sum_j a_j w_j, fp32 accumulate, fp16 out
// =============================================================================================
template <int N>
struct MxRing {   // ring slot + phase parity
  uint32_t i = 0, ph = 0;
  __device__ __forceinline__ void next() {
    if (++i == N) {
      i = 0;
      ph ^= 1;
    }
  }
};

constexpr int kMxThreads = 384;
#ifndef ATOM_MX_TN
#define ATOM_MX_TN 224
#endif
constexpr int kMxTN = ATOM_MX_TN;
constexpr int kMxEpi0 = 4, kMxNumEpi = 8;
constexpr uint32_t kMxTmemCols = 512;

// Token-tile configurations: kTM = 128 (two accumulator buffers: the epilogue of tile i overlaps
// the MMAs of tile i + 1) or kTM = 256 (two 128-row MMA halves sharing the weight tile: 32% fewer
// operand bytes into the SM per MMA, which bounds this kernel (an MMA-free variant of it runs at
// 125 us at cfg5), one accumulator buffer).  The launcher picks per shape (waves x bytes).
template <int kTM>
struct MxCfg {
  static constexpr int TM = kTM, TN = ATOM_MX_TN;
  static constexpr int H = TM / 128;                  // 128-row MMA halves per tile
  static constexpr int AB = H == 1 ? 2 : 1;           // accumulator buffers (TMEM: 512 columns)
  static constexpr int KS = H == 1 ? 4 : 3;           // pipeline stages (shared memory)
  static constexpr uint32_t AccCols = AB * H * TN;    // 448
  static constexpr uint32_t SfaCol = AccCols;         // A scales: (half h, chunk c) at + 8h + 4c
  static constexpr uint32_t SfbCol = SfaCol + 8 * H;  // B scales: (chunk c, block k) at + 8c + 4k
  static constexpr uint32_t SfSet = 8 * H + 16;       // columns of one scale set
  static constexpr int Imgs = 2 * H + 4;              // tcgen05.cp images per stage
  static_assert(TM == 128 || TM == 256, "token tile");
  static_assert(SfaCol + 2 * SfSet <= 512, "two scale-column sets");
};

template <class C>
struct __align__(1024) MxSmem {
  uint8_t a[C::KS][C::TM * 128];         // packed E2M1 (or E4M3) activation stage, SW128
  uint8_t b[C::KS][C::TN * 128];         // weight stage, SW128
  uint8_t sfa[C::KS][C::TM * 16];        // canonical scale bytes of the stage, [row][16 B]
  uint8_t sfb[C::KS][C::TN * 16];
  uint32_t img[C::KS][C::Imgs][128];     // tcgen05.cp images: A (h, c) at 2h + c, then
                                         // B (c, k) at 2H + 2c + k
  uint64_t full[C::KS], sfready[C::KS], empty[C::KS];
  uint64_t tfull[C::AB], tempty[C::AB];
  uint32_t tmem_base;
};
static_assert(sizeof(MxSmem<MxCfg<128>>) + 1024 <= 232448, "shared memory");
static_assert(sizeof(MxSmem<MxCfg<256>>) + 1024 <= 232448, "shared memory");

// Instruction descriptor, block-scaled kinds: F32 accumulate, K-major A/B, UE8M0 scales.
__host__ __device__ constexpr uint32_t mx_idesc(uint32_t fmt, uint32_t m, uint32_t n,
                                                uint32_t sf_id) {
  return (sf_id << 4)          // B scale-factor id          [4, 6)
         | (fmt << 7)          // A format                   [7, 10)
         | (fmt << 10)         // B format                   [10, 13)
         | ((n >> 3) << 17)    // N >> 3                     [17, 23)
         | (1u << 23)          // scale format UE8M0         [23]
         | ((m >> 4) << 24)    // M >> 4                     [24, 29)
         | (sf_id << 29);      // A scale-factor id          [29, 31)
}
constexpr uint32_t kFmtE2M1 = 1;   // kind::mxf4 element format
constexpr uint32_t kFmtE4M3 = 0;   // kind::mxf8f6f4 element format

__device__ __forceinline__ void umma_mxf4(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t sfa, uint32_t sfb, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;"
      "\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb)
      : "memory");
}
__device__ __forceinline__ void umma_mxf8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t sfa, uint32_t sfb, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6],"
      " p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb)
      : "memory");
}
// 32 rows x 16 bytes of shared memory -> TMEM lanes 0-31 (replicated to the 4 lane quarters),
// 4 columns; the descriptor: no swizzle, 8-row core matrices 128 bytes apart.
__device__ __forceinline__ void tmem_cp_32x128b_x4(uint32_t taddr, uint32_t smem_addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(128u >> 4) << 32;   // SBO
  d |= static_cast<uint64_t>(1u) << 46;          // version
  asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(taddr), "l"(d)
               : "memory");
}

struct MxParams {
  void* c;
  int64_t ldc;
  int M, N;
  int s4;          // FP4 stages (256 K-elements each; the last may hold one 128-chunk)
  int ch_last;     // chunks of the last FP4 stage (1 or 2)
  int has8;        // 1 if the 128 outlier channels (one FP8 stage) are present
  int sf_off8;     // scale-byte column of the first outlier block (= (K - 128) / 32)
  int m_tiles, num_tiles;
  int ksplit, num_items;   // split-K: item = tile * ksplit + j covers stages [j nst / ksplit, ..)
  float* part;             // ksplit > 1: fp32 partials [ksplit][M][N]
};

template <int kTM>
__global__ void __launch_bounds__(kMxThreads, 1)
mx_gemm_kernel(const __grid_constant__ CUtensorMap tm_a4, const __grid_constant__ CUtensorMap tm_b4,
               const __grid_constant__ CUtensorMap tm_a8, const __grid_constant__ CUtensorMap tm_b8,
               const __grid_constant__ CUtensorMap tm_asf,
               const __grid_constant__ CUtensorMap tm_bsf, const MxParams p) {
  extern __shared__ uint8_t smem_raw[];
  using C = MxCfg<kTM>;
  constexpr int kMxTM = C::TM, kMxKS = C::KS, kMxH = C::H, kMxAB = C::AB;
  constexpr uint32_t kMxSfaCol = C::SfaCol, kMxSfbCol = C::SfbCol, kMxSfSet = C::SfSet;
  MxSmem<C>& sm = *reinterpret_cast<MxSmem<C>*>(smem_raw +
                                                ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kMxKS; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.sfready[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    for (int b = 0; b < kMxAB; ++b) {
      mbar_init(&sm.tfull[b], 1);
      mbar_init(&sm.tempty[b], kMxNumEpi);
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_a4);
    tma_prefetch_desc(&tm_b4);
    tma_prefetch_desc(&tm_a8);
    tma_prefetch_desc(&tm_b8);
    tma_prefetch_desc(&tm_asf);
    tma_prefetch_desc(&tm_bsf);
  }
  if (warp == 1) tmem_alloc(&sm.tmem_base, kMxTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  const int nst = p.s4 + p.has8;                      // stages per tile
  auto s_lo = [&](int it) { return (it % p.ksplit) * nst / p.ksplit; };
  auto s_hi = [&](int it) { return (it % p.ksplit + 1) * nst / p.ksplit; };
  if (threadIdx.x == 0) griddep_launch();

  if (warp == 0) {
    // ============ producer: activation / weight / scale-byte tiles of each stage (TMA) ============
    if (lane == 0) {
      const uint64_t pol_a = l2_policy_evict_last(), pol_w = l2_policy_evict_first();
      griddep_wait();
      MxRing<kMxKS> st;
      for (int it = blockIdx.x; it < p.num_items; it += gridDim.x) {
        const int tile = it / p.ksplit;
        const int m0 = (tile % p.m_tiles) * kMxTM, n0 = (tile / p.m_tiles) * kMxTN;
        for (int s = s_lo(it); s < s_hi(it); ++s, st.next()) {
          mbar_wait(&sm.empty[st.i], st.ph ^ 1);
          mbar_arrive_expect_tx(&sm.full[st.i], (kMxTM + kMxTN) * (128 + 16));
          const bool fp8 = s >= p.s4;
          const int sfc = fp8 ? p.sf_off8 : 8 * s;
          tma_load_2d_hint(sm.a[st.i], fp8 ? &tm_a8 : &tm_a4, &sm.full[st.i], fp8 ? 0 : 128 * s,
                           m0, pol_a);
          tma_load_2d_hint(sm.b[st.i], fp8 ? &tm_b8 : &tm_b4, &sm.full[st.i], fp8 ? 0 : 128 * s,
                           n0, pol_w);
          // the box starts on a 16-byte boundary (TMA requires it); the stage's 8 (or 4) scale
          // bytes of a row never straddle one
          tma_load_2d_hint(sm.sfa[st.i], &tm_asf, &sm.full[st.i], sfc & ~15, m0, pol_a);
          tma_load_2d_hint(sm.sfb[st.i], &tm_bsf, &sm.full[st.i], sfc & ~15, n0, pol_w);
        }
      }
    }
  } else if (warp == 1) {
    // ============ MMA issuer: scale copies to TMEM, 4 block-scaled MMAs per stage ============
    if (lane == 0) {
      const uint64_t da0 = umma_desc_sw128(smem_u32(sm.a[0]));
      const uint64_t db0 = umma_desc_sw128(smem_u32(sm.b[0]));
      MxRing<kMxKS> st;
      MxRing<kMxAB> tb;
      uint32_t sfpar = 0;
      for (int it = blockIdx.x; it < p.num_items; it += gridDim.x, tb.next()) {
        mbar_wait(&sm.tempty[tb.i], tb.ph ^ 1);        // the epilogue drained this buffer
        const int s0 = s_lo(it);
        tc_fence_after();
        const uint32_t d = tmem + tb.i * (kMxH * kMxTN);   // half h at + h kMxTN
        for (int s = s0; s < s_hi(it); ++s, st.next()) {
          mbar_wait(&sm.full[st.i], st.ph);
          mbar_wait(&sm.sfready[st.i], st.ph);
          tc_fence_after();
          const bool fp8 = s >= p.s4;
          const int nch = fp8 ? 1 : (s + 1 == p.s4 ? p.ch_last : 2);
          // scale columns alternate between two sets by stage parity, so a copy never overwrites
          // scales the previous stage's MMAs may still read
          const uint32_t sfa = tmem + kMxSfaCol + (sfpar ? kMxSfSet : 0u);
          const uint32_t sfb = tmem + kMxSfbCol + (sfpar ? kMxSfSet : 0u);
          sfpar ^= 1u;
          for (int c = 0; c < nch; ++c) {
#pragma unroll
            for (int h = 0; h < kMxH; ++h)
              tmem_cp_32x128b_x4(sfa + 8 * h + 4 * c, smem_u32(sm.img[st.i][2 * h + c]));
            tmem_cp_32x128b_x4(sfb + 8 * c, smem_u32(sm.img[st.i][2 * kMxH + 2 * c]));
            tmem_cp_32x128b_x4(sfb + 8 * c + 4, smem_u32(sm.img[st.i][2 * kMxH + 2 * c + 1]));
          }
          const uint64_t da = da0 + st.i * (kMxTM * 128 / 16), db = db0 + st.i * (kMxTN * 128 / 16);
          if (!fp8) {
            // K = 64 per MMA (32 bytes of packed E2M1): chunk c = k / 2, scale bytes 2 (k % 2), +1
            for (int k = 0; k < 2 * nch; ++k) {
              const uint32_t c = k >> 1, id = (k & 1) * 2;
#pragma unroll
              for (int h = 0; h < kMxH; ++h)
                umma_mxf4(d + h * kMxTN, da + h * (128 * 128 / 16) + 2 * k, db + 2 * k,
                          mx_idesc(kFmtE2M1, 128, kMxTN, id), sfa + 8 * h + 4 * c, sfb + 8 * c,
                          (s > s0 || k > 0));
            }
          } else {
            // K = 32 per MMA (32 bytes of E4M3): scale byte k
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
              for (int h = 0; h < kMxH; ++h)
                umma_mxf8(d + h * kMxTN, da + h * (128 * 128 / 16) + 2 * k, db + 2 * k,
                          mx_idesc(kFmtE4M3, 128, kMxTN, k), sfa + 8 * h, sfb, (s > s0 || k > 0));
          }
          umma_commit(&sm.empty[st.i]);
        }
        umma_commit(&sm.tfull[tb.i]);
      }
    }
  } else if (warp == 2) {
    // ============ scale transposer: canonical [row][bytes] -> tcgen05.cp 32x128b images ============
    // image word 4l + c = the chunk's 4 scale bytes of row 32c + l of the 128-row block
    MxRing<kMxKS> st;
    for (int it = blockIdx.x; it < p.num_items; it += gridDim.x) {
      for (int s = s_lo(it); s < s_hi(it); ++s, st.next()) {
        mbar_wait(&sm.full[st.i], st.ph);
        const bool fp8 = s >= p.s4;
        const int nch = fp8 ? 1 : (s + 1 == p.s4 ? p.ch_last : 2);
        const int off = (fp8 ? p.sf_off8 : 8 * s) & 15;   // the stage's bytes in the 16-byte box
        for (int c = 0; c < nch; ++c) {
          const int o = off + 4 * c;
#pragma unroll
          for (int h = 0; h < kMxH; ++h) {
            uint32_t wa[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
              wa[q] = *reinterpret_cast<const uint32_t*>(sm.sfa[st.i] +
                                                         (128 * h + 32 * q + lane) * 16 + o);
            reinterpret_cast<uint4*>(sm.img[st.i][2 * h + c])[lane] =
                make_uint4(wa[0], wa[1], wa[2], wa[3]);
          }
          uint32_t wb0[4], wb1[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int r = 32 * q + lane;
            wb0[q] = *reinterpret_cast<const uint32_t*>(sm.sfb[st.i] + r * 16 + o);
            wb1[q] = r + 128 < kMxTN
                         ? *reinterpret_cast<const uint32_t*>(sm.sfb[st.i] + (r + 128) * 16 + o)
                         : 0u;
          }
          reinterpret_cast<uint4*>(sm.img[st.i][2 * kMxH + 2 * c])[lane] =
              make_uint4(wb0[0], wb0[1], wb0[2], wb0[3]);
          reinterpret_cast<uint4*>(sm.img[st.i][2 * kMxH + 2 * c + 1])[lane] =
              make_uint4(wb1[0], wb1[1], wb1[2], wb1[3]);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.sfready[st.i]);
      }
    }
  } else if (warp >= kMxEpi0) {
    // ============ epilogue: TMEM fp32 -> fp16 C, once per tile ============
    // kMxH = 2: warp e drains row half e / 4 (TMEM lane quarter e % 4), all kMxTN columns in
    // two passes of 112; kMxH = 1: column half e / 4.
    const int e = warp - kMxEpi0, q = warp & 3, hf = e >> 2;
    constexpr int kPasses = kMxH == 2 ? 2 : 1;
    griddep_wait();
    MxRing<kMxAB> tb;
    for (int it = blockIdx.x; it < p.num_items; it += gridDim.x, tb.next()) {
      const int tile = it / p.ksplit;
      const int m0 = (tile % p.m_tiles) * kMxTM, n0 = (tile / p.m_tiles) * kMxTN;
      mbar_wait(&sm.tfull[tb.i], tb.ph);
      tc_fence_after();
      const int row = (kMxH == 2 ? 128 * hf : 0) + q * 32 + lane;
      const uint32_t ta = tmem + (static_cast<uint32_t>(q * 32) << 16) +
                          tb.i * (kMxH * kMxTN) + (kMxH == 2 ? hf * kMxTN : hf * 112);
      const int m = m0 + row;
      __half* crow = static_cast<__half*>(p.c) + static_cast<int64_t>(m < p.M ? m : 0) * p.ldc;
      for (int pass = 0; pass < kPasses; ++pass) {
        uint32_t r[7][16];
#pragma unroll
        for (int cb = 0; cb < 7; ++cb) tmem_ld_32x32b<16>(ta + 112 * pass + 16 * cb, r[cb]);
        tmem_ld_wait();
        if (pass + 1 == kPasses) {       // every column of this thread's rows is in registers
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.tempty[tb.i]);
        }
        if (m < p.M && p.ksplit > 1) {   // split-K: the fp32 partial of stages [s_lo, s_hi)
          float* prow = p.part + (static_cast<int64_t>(it % p.ksplit) * p.M + m) * p.N;
#pragma unroll
          for (int cb = 0; cb < 7; ++cb) {
            const int n = n0 + (kMxH == 2 ? 0 : hf * 112) + 112 * pass + 16 * cb;
            if (n >= p.N) break;
            float4* dst = reinterpret_cast<float4*>(prow + n);
#pragma unroll
            for (int i = 0; i < 4; ++i)
              dst[i] = make_float4(__uint_as_float(r[cb][4 * i]), __uint_as_float(r[cb][4 * i + 1]),
                                   __uint_as_float(r[cb][4 * i + 2]),
                                   __uint_as_float(r[cb][4 * i + 3]));
          }
        } else if (m < p.M) {
#pragma unroll
          for (int cb = 0; cb < 7; ++cb) {
            const int n = n0 + (kMxH == 2 ? 0 : hf * 112) + 112 * pass + 16 * cb;
            if (n >= p.N) break;
            uint32_t h[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const __half2 v = __floats2half2_rn(__uint_as_float(r[cb][2 * i]),
                                                  __uint_as_float(r[cb][2 * i + 1]));
              h[i] = *reinterpret_cast<const uint32_t*>(&v);
            }
            uint4* dst = reinterpret_cast<uint4*>(crow + n);
            dst[0] = make_uint4(h[0], h[1], h[2], h[3]);
            dst[1] = make_uint4(h[4], h[5], h[6], h[7]);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, kMxTmemCols);
  }
}

// split-K reduction: C[m][n] = fp16(sum_j part[j][m][n]), j ascending (deterministic)
__global__ void __launch_bounds__(256)
mx_splitk_reduce_kernel(const float* __restrict__ part, int32_t ksplit, int64_t M, int64_t N,
                        __half* __restrict__ c, int64_t ldc) {
  griddep_wait();
  griddep_launch();
  const int64_t n4 = N / 4, total = M * n4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t m = i / n4, n = 4 * (i % n4);
    float4 acc = reinterpret_cast<const float4*>(part + m * N + n)[0];
    for (int j = 1; j < ksplit; ++j) {
      const float4 v = reinterpret_cast<const float4*>(part + (j * M + m) * N + n)[0];
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    const __half2 lo = __floats2half2_rn(acc.x, acc.y), hi = __floats2half2_rn(acc.z, acc.w);
    uint2 o;
    o.x = *reinterpret_cast<const uint32_t*>(&lo);
    o.y = *reinterpret_cast<const uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(c + m * ldc + n) = o;
  }
}

// Split-K factor: when the output tiles cannot fill the SMs, the K stages of a tile are divided
// among ksplit CTAs (at least 4 stages each) and an fp32 reduction follows.
static int mx_ksplit(int64_t tiles, int nst, int num_sms) {
  if (tiles * 2 > num_sms) return 1;
  int k = static_cast<int>(num_sms / tiles);
  if (k > nst / 4) k = nst / 4;
  return k < 1 ? 1 : k;
}

// Launch plan.  Token tile: the one with fewer (waves x operand bytes into the SM per stage); the
// 256-row tile pays ~10% for its single accumulator buffer.  Small shapes: split-K over 128-row
// tiles.  Wave tail: when the 256-row tiles leave a partial last wave, they cover only the first
// n_full column tiles (whole waves) and a second launch covers the rest with 128-row tiles
// (twice the tiles, each ~2/3 of the time).  Split-K of the tail's 256-row tiles instead was
// measured slower (cfg5 149.8 vs 137.1 us).
struct MxPlan {
  int tm, ksplit;
  int64_t n_full;          // column tiles of the first launch (== all of them: one launch)
};
static MxPlan mx_plan(int64_t M, int64_t N, int64_t K, int32_t k_o, int num_sms) {
  const int64_t K4 = K - k_o;
  const int nst = static_cast<int>((K4 / 128 + 1) / 2) + (k_o ? 1 : 0);
  const int64_t n_tiles = (N + kMxTN - 1) / kMxTN;
  auto waves = [&](int64_t t) { return (t + num_sms - 1) / num_sms; };
  auto cost = [&](int tm, double f) {
    return static_cast<double>(waves(((M + tm - 1) / tm) * n_tiles)) * (tm + kMxTN) * f;
  };
  MxPlan pl;
  pl.tm = cost(256, 1.1) < cost(128, 1.0) ? 256 : 128;
  pl.ksplit = pl.tm == 128 ? mx_ksplit(((M + 127) / 128) * n_tiles, nst, num_sms) : 1;
  pl.n_full = n_tiles;
  if (pl.tm == 256) {
    const int64_t m256 = (M + 255) / 256, m128 = (M + 127) / 128;
    const int64_t nf = (waves(m256 * n_tiles) - 1) * num_sms / m256;
    if (nf > 0 && nf < n_tiles) {
      const double split = static_cast<double>(waves(m256 * nf)) * (256 + kMxTN) * 1.1 +
                           static_cast<double>(waves(m128 * (n_tiles - nf))) * (128 + kMxTN);
      if (split < 0.97 * cost(256, 1.1)) pl.n_full = nf;
    }
  }
  return pl;
}

int mx_gemm_launches(int64_t M, int64_t N, int64_t K, int32_t k_outlier, int num_sms) {
  const MxPlan pl = mx_plan(M, N, K, k_outlier, num_sms);
  return 1 + (pl.ksplit > 1) + (pl.n_full * kMxTN < N ? 1 : 0);
}

size_t mx_gemm_workspace_bytes(int64_t M, int64_t N, int64_t K, int32_t k_outlier, int num_sms) {
  const MxPlan pl = mx_plan(M, N, K, k_outlier, num_sms);
  return pl.ksplit > 1 ? static_cast<size_t>(pl.ksplit) * M * N * sizeof(float) : 0;
}

// ---------------------------------------------------------------------------------------------
typedef CUresult (*PFN_encodeTiledMx)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                      const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                      const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                      CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_encodeTiledMx mx_encode_fn() {
  static const PFN_encodeTiledMx fn = []() -> PFN_encodeTiledMx {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_encodeTiledMx>(ptr);
    return nullptr;
  }();
  return fn;
}
// 2D uint8 tensor [rows][cols] with row stride ld bytes, box [box_rows][box_cols bytes]
static bool mx_map(CUtensorMap* map, const void* base, uint64_t cols, uint64_t ld, uint64_t rows,
                   uint32_t box_cols, uint32_t box_rows, CUtensorMapSwizzle swz) {
  PFN_encodeTiledMx enc = mx_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// One launch over the output columns [n_off, n_end) with token tile tm (split-K only when
// ksplit > 1, which implies the whole range [0, N)).
static cudaError_t launch_mx_cols(const MxGemmArgs& a, cudaStream_t stream, int num_sms, int tm,
                                  int64_t n_off, int64_t n_end, int ksplit) {
  const int64_t K4 = a.K - a.k_outlier;
  const void* any = K4 ? static_cast<const void*>(a.a_fp4) : static_cast<const void*>(a.a_fp8);
  const void* anyw = K4 ? static_cast<const void*>(a.w_fp4) : static_cast<const void*>(a.w_fp8);
  const int64_t N = n_end - n_off;
  const int64_t n_tiles = (N + kMxTN - 1) / kMxTN;
  if (ksplit > 1 && (a.workspace == nullptr ||
                     a.workspace_bytes < static_cast<size_t>(ksplit) * a.M * N * sizeof(float)))
    return cudaErrorInvalidValue;
  CUtensorMap m_a4, m_b4, m_a8, m_b8, m_asf, m_bsf;
  // an absent operand (no FP4 channels / no outliers) aliases the other one and is never read
  const void* a4 = K4 ? a.a_fp4 : any;
  const void* a8 = a.k_outlier ? a.a_fp8 : any;
  const uint64_t c4 = K4 ? K4 / 2 : 128, c8 = a.k_outlier ? 128 : K4 / 2;
  const uint64_t nsf = a.K / 32;
  // weight rows (and their scale rows) from n_off on: every row pitch is a multiple of 16 bytes
  const uint8_t* b4 = static_cast<const uint8_t*>(K4 ? a.w_fp4 : anyw) + n_off * c4;
  const uint8_t* b8 = static_cast<const uint8_t*>(a.k_outlier ? a.w_fp8 : anyw) + n_off * c8;
  const uint8_t* bsf = a.w_sf + n_off * a.ldw_sf;
  if (!mx_map(&m_a4, a4, c4, c4, a.M, 128, tm, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !mx_map(&m_b4, b4, c4, c4, N, 128, kMxTN, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !mx_map(&m_a8, a8, c8, c8, a.M, 128, tm, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !mx_map(&m_b8, b8, c8, c8, N, 128, kMxTN, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !mx_map(&m_asf, a.a_sf, nsf, a.lda_sf, a.M, 16, tm, CU_TENSOR_MAP_SWIZZLE_NONE) ||
      !mx_map(&m_bsf, bsf, nsf, a.ldw_sf, N, 16, kMxTN, CU_TENSOR_MAP_SWIZZLE_NONE))
    return cudaErrorInvalidValue;
  MxParams p;
  p.c = static_cast<__half*>(a.c) + n_off;
  p.ldc = a.ldc;
  p.M = static_cast<int>(a.M);
  p.N = static_cast<int>(N);
  const int64_t chunks = K4 / 128;
  p.s4 = static_cast<int>((chunks + 1) / 2);
  p.ch_last = (chunks % 2) ? 1 : 2;
  p.has8 = a.k_outlier ? 1 : 0;
  p.sf_off8 = static_cast<int>(K4 / 32);
  p.m_tiles = static_cast<int>((a.M + tm - 1) / tm);
  p.num_tiles = p.m_tiles * static_cast<int>(n_tiles);
  p.ksplit = ksplit;
  p.num_items = p.num_tiles * ksplit;
  p.part = static_cast<float*>(a.workspace);
  const int grid = p.num_items < num_sms ? p.num_items : num_sms;
  auto go = [&](auto tm_tag) -> cudaError_t {
    constexpr int kTM = decltype(tm_tag)::value;
    const size_t smem = sizeof(MxSmem<MxCfg<kTM>>) + 1024;
    static std::once_flag once[64];
    static cudaError_t attr_err[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    std::call_once(once[dev], [&]() {
      attr_err[dev] = cudaFuncSetAttribute(mx_gemm_kernel<kTM>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem));
    });
    if (attr_err[dev] != cudaSuccess) return attr_err[dev];
    return launch_pdl(mx_gemm_kernel<kTM>, dim3(grid), dim3(kMxThreads), smem, stream, m_a4, m_b4,
                      m_a8, m_b8, m_asf, m_bsf, p);
  };
  cudaError_t e = tm == 256 ? go(std::integral_constant<int, 256>{})
                            : go(std::integral_constant<int, 128>{});
  if (e != cudaSuccess) return e;
  if (ksplit > 1) {
    int64_t blocks = (a.M * N / 4 + 255) / 256;
    if (blocks > 4LL * num_sms) blocks = 4LL * num_sms;
    e = launch_pdl(mx_splitk_reduce_kernel, dim3(static_cast<unsigned>(blocks)), dim3(256), 0,
                   stream, static_cast<const float*>(a.workspace), ksplit, a.M, N,
                   static_cast<__half*>(a.c) + n_off, a.ldc);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

cudaError_t launch_mx_gemm(const MxGemmArgs& a, cudaStream_t stream, int num_sms) {
  if (a.M == 0) return cudaSuccess;
  const MxPlan pl = mx_plan(a.M, a.N, a.K, a.k_outlier, num_sms);
  const int64_t n_mid = pl.n_full * kMxTN < a.N ? pl.n_full * kMxTN : a.N;
  cudaError_t e = launch_mx_cols(a, stream, num_sms, pl.tm, 0, n_mid, pl.ksplit);
  if (e != cudaSuccess || n_mid == a.N) return e;
  return launch_mx_cols(a, stream, num_sms, 128, n_mid, a.N, 1);
}

}  // namespace atom
