// gemm.cu -- a2-a5: fused W4A4 mixed-precision group GEMM on sm_100a tensor cores.
//
// Paper (Fig 6): per (activation group, weight group) compute the low-bit product on
// the tensor cores (Step 1), dequantize each temporary result with its two group scales (Step 2)
// and sum (Step 3), all fused in the MMA pipeline; the 128 INT8 outlier channels are one more
// group of the same K loop (mixed precision via reordering P:242).
//
// B200 design:
//   * swap-AB: the MMA M side (128 TMEM lanes) is 128 output channels n of W, the MMA N side is a
//     tile of BT tokens.  D[n][m] = sum_k W'[n][k] A'[m][k].
//   * TMA streams the PACKED INT4 tiles (64 B per row per group) into a 4-stage ring; the INT8
//     outlier group arrives as two 64-byte halves through the same ring.
//   * 4 unpack warps expand nibbles to int8 16*q (high nibbles: one LOP per 4 codes; low nibbles:
//     SHL + LOP; exact two's complement) directly into the 128B-swizzled K-major layout the UMMA
//     descriptor reads, with the same intra-group channel permutation for both operands (the dot
//     product is order-invariant).  tcgen05 has no s4 kind, so this is the INT4 -> INT8 step.
//   * 1 MMA thread per group: 4 x kind::i8 (K = 32) into a fresh TMEM int32 accumulator (4 TMEM
//     buffers rotate ACROSS groups so later groups multiply while the epilogue drains earlier
//     ones) and ONE tcgen05.commit that both frees the unpacked operands and publishes the
//     partial.  INT4 partials come out as R = 256*P_t (exact, |R| <= 2^21).
//   * 8 epilogue warps (thread = output channel = TMEM lane) tcgen05.ld the partials, turn R into
//     the float 1.5*2^23 + R with one LOP3 ((R & 0x7FFFFF) ^ 0x4B400000, exact for |R| < 2^22)
//     and dequantize with two FFMA2 per column pair; fp32
//     accumulators live in registers; after the last group they write fp16 (or fp32 for K-shards).
//   * persistent CTAs (one per SM) walk output tiles; consecutive CTAs share the weight tile.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "internal.h"
#include "ptx.cuh"

namespace atom {

constexpr int kStages = 4;      // packed-tile TMA ring depth
constexpr int kUbuf = 4;        // unpacked int8 operand buffers
constexpr int kThreads = 448;   // 14 warps
constexpr int kUnpackWarp0 = 2; // warps 2..5
constexpr int kNumUnpackWarps = 4;
constexpr int kEpiWarp0 = 6;    // warps 6..13
constexpr int kNumEpiWarps = 8;
constexpr int kTileN = 128;     // output channels per tile (MMA M)
constexpr int kSRing = 16;      // group-scale ring depth
constexpr int kTBuf = 4;        // TMEM accumulator buffers (4 x BT <= 512 columns)
static_assert(kTBuf == kUbuf, "one mdone barrier ring serves both the operand and TMEM rings");

constexpr uint32_t kMagicBits = 0x4B400000u;   // bit pattern of 1.5*2^23
constexpr float kMagic = 12582912.0f;          // 1.5*2^23

struct GemmParams {
  const float* a_scales;
  const float* w_scales;
  void* c;
  int64_t ldc;
  int32_t* debug;
  int M, N, G, G4, k_o, c_f32;
  int m_tiles, num_tiles;
  long long* trace;   // development timeline probe (CTA 0): [3][256] clock64 stamps, or null
};

template <int BT>
struct __align__(1024) GemmSmem {
  uint8_t ubuf_w[kUbuf][kTileN * 128];  // unpacked weight group, SW128 K-major
  uint8_t ubuf_a[kUbuf][BT * 128];      // unpacked activation group, SW128 K-major
  uint8_t stage_w[kStages][kTileN * 64];// packed weight group (or half of the INT8 group)
  uint8_t stage_a[kStages][BT * 64];    // packed activation group
  float ssw[kSRing][kTileN];            // weight scales of a group (ring, filled by cp.async)
  float ssa[kSRing][BT];                // activation scales of a group
  uint64_t full[kStages], empty[kStages];
  uint64_t ufull[kUbuf];
  uint64_t mdone[kUbuf];                // MMAs of a group done: operands free + partial ready
  uint64_t tempty[kTBuf];
  uint64_t sready[kSRing], sfree[kSRing];
  uint32_t tmem_base;
};

template <int BT>
__host__ __device__ constexpr uint32_t tmem_cols() {
  return (kTBuf * BT) <= 32 ? 32 : (kTBuf * BT) <= 64 ? 64 : (kTBuf * BT) <= 128 ? 128
       : (kTBuf * BT) <= 256 ? 256 : 512;
}

// rotl(v, 4) & 0xF0F0F0F0 == (v << 4) & 0xF0F0F0F0, but as SHF.L.W + LOP3 on the integer pipe
// (a plain shift is compiled to IMAD.SHL on the FMA pipe, which the epilogue saturates).
__device__ __forceinline__ uint32_t lo_nib(uint32_t v) {
  return __funnelshift_l(v, v, 4) & 0xF0F0F0F0u;
}
__device__ __forceinline__ uint4 unpack_lo(uint4 v) {  // even channels -> 16*q bytes
  return make_uint4(lo_nib(v.x), lo_nib(v.y), lo_nib(v.z), lo_nib(v.w));
}
// float(1.5*2^23 + R) from the int32 partial R, |R| < 2^22: the low 23 bits of R with bit 22
// flipped are R + 2^22 in [0, 2^23); OR-ing the exponent of 2^23 gives 2^23 + 2^22 + R exactly.
__device__ __forceinline__ float biased(uint32_t r) {
  return __uint_as_float((r & 0x007FFFFFu) ^ kMagicBits);
}

__device__ __forceinline__ uint4 unpack_hi(uint4 v) {  // odd channels -> 16*q bytes
  return make_uint4(v.x & 0xF0F0F0F0u, v.y & 0xF0F0F0F0u, v.z & 0xF0F0F0F0u, v.w & 0xF0F0F0F0u);
}

// One operand tile of ROWS rows: packed stage [ROWS][64 B] -> unpacked SW128 [ROWS][128 B].
// Thread ut owns the 16-byte packed chunk (ut & 3) of rows (ut >> 2) + 32k; rows 32 apart share
// their swizzle phase, so every address below is a per-thread base plus an immediate.
template <int ROWS>
__device__ __forceinline__ void unpack_tile(const uint8_t* stage, uint8_t* ubuf, int ut,
                                            bool int4, int h) {
  constexpr int KR = ROWS / 32;
  const uint32_t r0 = static_cast<uint32_t>(ut) >> 2, c = static_cast<uint32_t>(ut) & 3u;
  const uint32_t r7 = r0 & 7u;
  const uint8_t* src = stage + ut * 16;
  uint4 v[KR];
#pragma unroll
  for (int k = 0; k < KR; ++k) v[k] = *reinterpret_cast<const uint4*>(src + k * 32 * 64);
  uint8_t* dst = ubuf + r0 * 128;
  if (int4) {
    const uint32_t olo = ((2 * c) ^ r7) << 4, ohi = ((2 * c + 1) ^ r7) << 4;
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      *reinterpret_cast<uint4*>(dst + k * 32 * 128 + olo) = unpack_lo(v[k]);
      *reinterpret_cast<uint4*>(dst + k * 32 * 128 + ohi) = unpack_hi(v[k]);
    }
  } else {
    const uint32_t o = ((4 * h + c) ^ r7) << 4;
#pragma unroll
    for (int k = 0; k < KR; ++k) *reinterpret_cast<uint4*>(dst + k * 32 * 128 + o) = v[k];
  }
}

// kMode (development timing probes, never used for results): bit 0 = epilogue skips its
// arithmetic; bit 1 = unpack skips its data movement; bit 2 = producer skips the TMA loads;
// bit 3 = epilogue skips the TMEM loads; bit 4 = waits spin without the suspend-time hint.
template <int BT, bool kDebug, int kMode = 0>
__global__ void __launch_bounds__(kThreads, 1)
w4a4_gemm_kernel(const __grid_constant__ CUtensorMap tm_wq4,
                 const __grid_constant__ CUtensorMap tm_aq4,
                 const __grid_constant__ CUtensorMap tm_wq8,
                 const __grid_constant__ CUtensorMap tm_aq8, const GemmParams p) {
  static_assert(BT % 32 == 0 && BT >= 32 && BT * kTBuf <= 512, "token tile");
  auto wait = [](uint64_t* bar, uint32_t parity) {
    if constexpr ((kMode & 16) != 0) mbar_wait_spin(bar, parity);
    else mbar_wait(bar, parity);
  };
  extern __shared__ uint8_t smem_raw[];
  GemmSmem<BT>& sm = *reinterpret_cast<GemmSmem<BT>*>(
      smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  constexpr uint32_t kTmemCols = tmem_cols<BT>();

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kNumUnpackWarps);
    }
    for (int u = 0; u < kUbuf; ++u) {
      mbar_init(&sm.ufull[u], kNumUnpackWarps);
      mbar_init(&sm.mdone[u], 1);
    }
    for (int b = 0; b < kTBuf; ++b) {
      mbar_init(&sm.tempty[b], kNumEpiWarps);
    }
    for (int r = 0; r < kSRing; ++r) {
      mbar_init(&sm.sready[r], 32);  // one cp.async-arrive per producer-warp thread
      mbar_init(&sm.sfree[r], kNumEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_wq4);
    tma_prefetch_desc(&tm_aq4);
    tma_prefetch_desc(&tm_wq8);
    tma_prefetch_desc(&tm_aq8);
  }
  if (warp == 1) tmem_alloc(&sm.tmem_base, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  const int G = p.G, G4 = p.G4;
  const int loads_per_tile = G4 + (p.k_o ? 2 : 0);

  if (warp == 0) {
    // ===================== producer warp: group scales (cp.async) + TMA =====================
    // The scales of a group are staged into the scale ring when its first stage is loaded, i.e.
    // kStages + kUbuf + kTBuf groups ahead of the epilogue, which hides the L2 latency of the
    // 4-byte copies (cp.async works for any M; TMA would need 16-byte aligned rows).
    uint32_t it = 0, g_it = 0;
    for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
      const int n0 = (tile / p.m_tiles) * kTileN;
      const int m0 = (tile % p.m_tiles) * BT;
      for (int l = 0; l < loads_per_tile; ++l, ++it) {
        if (l <= G4) {   // first load of group t = l (the outlier group's 2nd half is l = G4+1)
          const int t = l;
          const uint32_t sr = g_it % kSRing, sph = (g_it / kSRing) & 1;
          wait(&sm.sfree[sr], sph ^ 1);
          const float* ws = p.w_scales + static_cast<int64_t>(t) * p.N + n0;
          const float* as = p.a_scales + static_cast<int64_t>(t) * p.M;
#pragma unroll
          for (int j = lane; j < kTileN; j += 32) cp_async_4(&sm.ssw[sr][j], ws + j);
#pragma unroll
          for (int j = lane; j < BT; j += 32)
            // rows past M: any finite scale works, their partials are exactly zero (TMA
            // zero-fills out-of-range activation rows) and they are never stored
            cp_async_4(&sm.ssa[sr][j], as + min(m0 + j, p.M - 1));
          cp_async_mbar_arrive(&sm.sready[sr]);
          ++g_it;
        }
        const uint32_t s = it % kStages, ph = (it / kStages) & 1;
        wait(&sm.empty[s], ph ^ 1);
        if (lane == 0) {
          if constexpr ((kMode & 4) != 0) {   // probe: no TMA traffic
            mbar_arrive(&sm.full[s]);
          } else {
            mbar_arrive_expect_tx(&sm.full[s], kTileN * 64 + BT * 64);
            if (l < G4) {
              tma_load_2d(sm.stage_w[s], &tm_wq4, &sm.full[s], l * 64, n0);
              tma_load_2d(sm.stage_a[s], &tm_aq4, &sm.full[s], l * 64, m0);
            } else {
              const int h = l - G4;
              tma_load_2d(sm.stage_w[s], &tm_wq8, &sm.full[s], h * 64, n0);
              tma_load_2d(sm.stage_a[s], &tm_aq8, &sm.full[s], h * 64, m0);
            }
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (single thread) =====================
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_i8(kTileN, BT);
      uint32_t g_it = 0;
      for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
        for (int t = 0; t < G; ++t, ++g_it) {
          const uint32_t u = g_it % kUbuf, uph = (g_it / kUbuf) & 1;
          const uint32_t b = g_it % kTBuf, bph = (g_it / kTBuf) & 1;
          wait(&sm.tempty[b], bph ^ 1);
          tc_fence_after();
          const uint32_t d = tmem + b * BT;
          wait(&sm.ufull[u], uph);
          tc_fence_after();
          if (p.trace != nullptr && blockIdx.x == 0 && g_it < 256) p.trace[g_it] = clock64();
          const uint32_t a_base = smem_u32(sm.ubuf_w[u]);
          const uint32_t b_base = smem_u32(sm.ubuf_a[u]);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_i8(d, umma_desc_sw128(a_base + 32 * k), umma_desc_sw128(b_base + 32 * k), idesc,
                    k > 0 ? 1u : 0u);
          umma_commit(&sm.mdone[u]);
        }
      }
    }
  } else if (warp < kEpiWarp0) {
    // ===================== unpack warps: packed INT4 -> int8 (16*q), SW128 =====================
    const int ut = threadIdx.x - kUnpackWarp0 * 32;  // 0..127
    uint32_t it = 0, g_it = 0;
    for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
      for (int t = 0; t < G; ++t, ++g_it) {
        const uint32_t u = g_it % kUbuf, uph = (g_it / kUbuf) & 1;
        wait(&sm.mdone[u], uph ^ 1);   // MMAs of group g - kUbuf finished with this buffer
        const bool int4 = t < G4;
        const int nh = int4 ? 1 : 2;
        for (int h = 0; h < nh; ++h, ++it) {
          const uint32_t s = it % kStages, ph = (it / kStages) & 1;
          wait(&sm.full[s], ph);
          if constexpr ((kMode & 2) == 0) {
            unpack_tile<kTileN>(sm.stage_w[s], sm.ubuf_w[u], ut, int4, h);
            unpack_tile<BT>(sm.stage_a[s], sm.ubuf_a[u], ut, int4, h);
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.empty[s]);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (p.trace != nullptr && blockIdx.x == 0 && g_it < 256 && ut == 0)
          p.trace[256 + g_it] = clock64();
        if (lane == 0) mbar_arrive(&sm.ufull[u]);
      }
    }
  } else {
    // ===================== epilogue warps =====================
    constexpr int COLS = BT / 2;  // tokens per thread
    constexpr int CH = COLS >= 32 ? 32 : 16;
    const int e = warp - kEpiWarp0;
    const int q = warp & 3;       // TMEM lane quarter this warp may access
    const int half = e >> 2;
    const int n_local = q * 32 + lane;
    const uint32_t tlane = tmem + (static_cast<uint32_t>(q * 32) << 16) + half * COLS;
    uint32_t g_it = 0;
    for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
      const int n0 = (tile / p.m_tiles) * kTileN;
      const int m0 = (tile % p.m_tiles) * BT;
      const int n = n0 + n_local;
      const int mc0 = m0 + half * COLS;
      float2 acc[COLS / 2];
#pragma unroll
      for (int j = 0; j < COLS / 2; ++j) acc[j] = make_float2(0.0f, 0.0f);
      for (int t = 0; t < G; ++t, ++g_it) {
        const uint32_t b = g_it % kTBuf, bph = (g_it / kTBuf) & 1;
        const uint32_t sr = g_it % kSRing, sph = (g_it / kSRing) & 1;
        const bool int4 = t < G4;
        wait(&sm.sready[sr], sph);
        float sw = sm.ssw[sr][n_local];
        if (int4) sw *= (1.0f / 256.0f);  // undo the 16*16 operand pre-scaling (exact)
        // Dequantize T = float(1.5*2^23 + R) with ONE fma: g = T*sw' - 1.5*2^23*sw' = sw'*R,
        // rounded once.  sw' = sw with its 2 lowest mantissa bits cleared (relative change
        // < 2^-22) so that 1.5*2^23*sw' is exact; see DESIGN.md "Epilogue arithmetic".
        const float swh = __uint_as_float(__float_as_uint(sw) & 0xFFFFFFFCu);
        const float2 sw2 = make_float2(swh, swh);
        const float2 nc2 = make_float2(-kMagic * swh, -kMagic * swh);
        const float4* sa4 = reinterpret_cast<const float4*>(&sm.ssa[sr][half * COLS]);
        wait(&sm.mdone[b], bph);
        tc_fence_after();
        if (p.trace != nullptr && blockIdx.x == 0 && g_it < 256 && e == 0 && lane == 0)
          p.trace[512 + g_it] = clock64();
        const uint32_t taddr = tlane + b * BT;
#pragma unroll
        for (int ch = 0; ch < COLS / CH; ++ch) {
          uint32_t r[CH];
          if constexpr ((kMode & 8) == 0) {
            tmem_ld<CH>(taddr + ch * CH, r);
            tmem_ld_wait();
          } else {
#pragma unroll
            for (int k = 0; k < CH; ++k) r[k] = 0;
          }
          if (ch == COLS / CH - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.tempty[b]);
          }
          if constexpr (kDebug) {
#pragma unroll
            for (int k = 0; k < CH; ++k) {
              const int m = mc0 + ch * CH + k;
              const int v = static_cast<int>(r[k]);
              if (m < p.M)
                p.debug[(static_cast<int64_t>(t) * p.M + m) * p.N + n] = int4 ? (v >> 8) : v;
            }
          }
#pragma unroll
          for (int k4 = 0; k4 < ((kMode & 1) ? 0 : CH / 4); ++k4) {
            const float4 s = sa4[ch * (CH / 4) + k4];
            const int j = ch * (CH / 2) + 2 * k4;
            const float2 g0 = __ffma2_rn(make_float2(biased(r[4 * k4 + 0]), biased(r[4 * k4 + 1])),
                                         sw2, nc2);
            const float2 g1 = __ffma2_rn(make_float2(biased(r[4 * k4 + 2]), biased(r[4 * k4 + 3])),
                                         sw2, nc2);
            acc[j] = __ffma2_rn(make_float2(s.x, s.y), g0, acc[j]);
            acc[j + 1] = __ffma2_rn(make_float2(s.z, s.w), g1, acc[j + 1]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.sfree[sr]);
      }
      // ---- tile output ----
#pragma unroll
      for (int j = 0; j < COLS; ++j) {
        const int m = mc0 + j;
        const float v = (j & 1) ? acc[j >> 1].y : acc[j >> 1].x;
        if (m < p.M) {
          if (p.c_f32)
            static_cast<float*>(p.c)[static_cast<int64_t>(m) * p.ldc + n] = v;
          else
            static_cast<__half*>(p.c)[static_cast<int64_t>(m) * p.ldc + n] = __float2half_rn(v);
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}

// ---------------------------------------------------------------------------------------------
// host side: tensor maps + launch
// ---------------------------------------------------------------------------------------------
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode_fn() {
  static PFN_encodeTiled fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(ptr);
  }
  return fn;
}

// 2D uint8 tensor [rows][cols] (row stride = cols bytes), box [box_rows][64 bytes].
static bool make_map_u8(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows,
                        uint32_t box_rows) {
  PFN_encodeTiled enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BT>
static cudaError_t launch_bt(const GemmArgs& a, cudaStream_t stream, int num_sms) {
  const int M = static_cast<int>(a.M), N = static_cast<int>(a.N), K = static_cast<int>(a.K);
  const int k_o = a.k_outlier;
  const uint64_t kp = static_cast<uint64_t>(K - k_o) / 2;
  CUtensorMap m_wq4, m_aq4, m_wq8, m_aq8;
  // A map is always encoded (a valid descriptor is required as a kernel parameter); the unused
  // INT4 or INT8 maps alias the other operand and are never read.
  const void* w4 = kp ? static_cast<const void*>(a.w_q4) : static_cast<const void*>(a.w_q8);
  const void* a4 = kp ? static_cast<const void*>(a.a_q4) : static_cast<const void*>(a.a_q8);
  const void* w8 = k_o ? static_cast<const void*>(a.w_q8) : static_cast<const void*>(a.w_q4);
  const void* a8 = k_o ? static_cast<const void*>(a.a_q8) : static_cast<const void*>(a.a_q4);
  const uint64_t c4 = kp ? kp : 128, c8 = k_o ? 128 : kp;
  if (!make_map_u8(&m_wq4, w4, c4, N, kTileN) || !make_map_u8(&m_aq4, a4, c4, M, BT) ||
      !make_map_u8(&m_wq8, w8, c8, N, kTileN) || !make_map_u8(&m_aq8, a8, c8, M, BT))
    return cudaErrorInvalidValue;

  GemmParams p;
  p.a_scales = a.a_scales;
  p.w_scales = a.w_scales;
  p.c = a.c;
  p.ldc = a.ldc;
  p.debug = a.debug_partials;
  p.M = M;
  p.N = N;
  p.G = K / 128;
  p.G4 = (K - k_o) / 128;
  p.k_o = k_o;
  p.c_f32 = a.c_f32;
  p.m_tiles = (M + BT - 1) / BT;
  p.num_tiles = p.m_tiles * (N / kTileN);

  const size_t smem = sizeof(GemmSmem<BT>) + 1024;
  auto kern = p.debug ? w4a4_gemm_kernel<BT, true> : w4a4_gemm_kernel<BT, false>;
  if constexpr (BT == 128) {
    static const char* mode_env = getenv("ATOM_GEMM_PROBE_MODE");   // development probe only
    const int mode = mode_env ? atoi(mode_env) : 0;
    if (mode == 1) kern = w4a4_gemm_kernel<BT, false, 1>;
    if (mode == 2) kern = w4a4_gemm_kernel<BT, false, 2>;
    if (mode == 3) kern = w4a4_gemm_kernel<BT, false, 3>;
    if (mode == 4) kern = w4a4_gemm_kernel<BT, false, 4>;
    if (mode == 7) kern = w4a4_gemm_kernel<BT, false, 7>;
    if (mode == 15) kern = w4a4_gemm_kernel<BT, false, 15>;
    if (mode == 16) kern = w4a4_gemm_kernel<BT, false, 16>;
    if (mode == 23) kern = w4a4_gemm_kernel<BT, false, 23>;

  }
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int grid = p.num_tiles < num_sms ? p.num_tiles : num_sms;
  static long long* trace = nullptr;
  static const bool want_trace = getenv("ATOM_GEMM_TRACE") != nullptr;   // development probe only
  if (want_trace && trace == nullptr) cudaMalloc(&trace, 3 * 256 * sizeof(long long));
  p.trace = want_trace ? trace : nullptr;
  kern<<<grid, kThreads, smem, stream>>>(m_wq4, m_aq4, m_wq8, m_aq8, p);
  if (want_trace) {
    long long h[768];
    cudaMemcpy(h, trace, sizeof(h), cudaMemcpyDeviceToHost);
    fprintf(stderr, "trace g: ufull_arrive mma_issue epi_seen (clk rel. to mma_issue[0])\n");
    for (int g = 0; g < 256 && g < p.G * 2; ++g)
      fprintf(stderr, "%3d %9lld %9lld %9lld\n", g, h[256 + g] - h[0], h[g] - h[0], h[512 + g] - h[0]);
  }
  return cudaGetLastError();
}

cudaError_t launch_w4a4_gemm(const GemmArgs& a, cudaStream_t stream, int num_sms,
                             int* launches) {
  *launches = 0;
  if (a.M == 0) return cudaSuccess;
  const int64_t n_tiles = a.N / kTileN;
  auto tiles = [&](int bt) { return n_tiles * ((a.M + bt - 1) / bt); };
  cudaError_t e;
  if (tiles(128) >= num_sms) e = launch_bt<128>(a, stream, num_sms);
  else if (tiles(64) >= num_sms) e = launch_bt<64>(a, stream, num_sms);
  else e = launch_bt<32>(a, stream, num_sms);
  if (e == cudaSuccess) *launches = 1;
  return e;
}

}  // namespace atom
