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
#include <type_traits>
#include <cstdlib>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "internal.h"
#include "ptx.cuh"

namespace atom {

// Warp roles (16 warps, 4 warpgroups):
//   WG0: warp 0 producer (scales via cp.async + TMA), warp 1 MMA issuer, warps 2-3 unpack
//   WG1: warps 4-7 unpack
//   WG2, WG3: warps 8-15 epilogue (warp % 4 = TMEM lane quarter; WG2 = token columns [0, BT/2),
//             WG3 = [BT/2, BT))
// setmaxnreg moves registers from WG0/WG1 (72 each) to the epilogue warpgroups (184 each), which
// hold the fp32 accumulators of a 128 x BT tile (BT/2 per thread).
constexpr int kThreads = 512;
constexpr int kUnpackWarp0 = 2;
constexpr int kNumUnpackWarps = 6;
constexpr int kEpiWarp0 = 8;
constexpr int kNumEpiWarps = 8;
constexpr int kRegsLow = 64, kRegsHigh = 192;           // 8*32*64 + 8*32*192 = 65536
constexpr int kTileN = 128;     // output channels per tile (MMA M)
constexpr int kStages = 4;      // packed-tile TMA ring depth
constexpr int kSRing = 8;       // group-scale ring depth

template <int BT> struct Cfg {
  static constexpr int kRing = BT >= 256 ? 2 : 4;       // unpacked operands == TMEM accumulators
  static constexpr uint32_t kTmemCols = kRing * BT <= 32 ? 32 : kRing * BT <= 64 ? 64
                                      : kRing * BT <= 128 ? 128 : kRing * BT <= 256 ? 256 : 512;
  static_assert(kRing * BT <= 512, "TMEM holds at most 512 columns");
};

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
  int ksplit, num_items;     // split-K: item = tile * ksplit + split
  float* partials;           // [num_tiles][ksplit][128][BT] fp32 (ksplit > 1)
  int* counters;             // [num_tiles] arrival counters, zeroed by the launcher (ksplit > 1)
  long long* trace;   // development timeline probe (CTA 0): [3][256] clock64 stamps, or null
};

template <int BT>
struct __align__(1024) GemmSmem {
  static constexpr int R = Cfg<BT>::kRing;
  uint8_t ubuf_w[R][kTileN * 128];      // unpacked weight group, SW128 K-major
  uint8_t ubuf_a[R][BT * 128];          // unpacked activation group, SW128 K-major
  uint8_t stage_w[kStages][kTileN * 64];// packed weight group (or half of the INT8 group)
  uint8_t stage_a[kStages][BT * 64];    // packed activation group
  float ssw[kSRing][kTileN];            // weight scales of a group (ring, filled by cp.async)
  float ssa[kSRing][BT];                // activation scales of a group
  uint8_t ostg[kNumEpiWarps][1280];     // per-warp output staging (2 x 8 rows x 80 B)
  uint32_t magic4[4];                   // 4 copies of the magic bit pattern
  uint64_t full[kStages], empty[kStages];
  uint64_t ufull[R];
  uint64_t mdone[R];                    // MMAs of a group done: operands free + partial ready
  uint64_t tempty[R];
  uint64_t sready[kSRing], sfree[kSRing];
  uint32_t tmem_base;
};

// rotl(v, 4) & 0xF0F0F0F0 == (v << 4) & 0xF0F0F0F0, but as SHF.L.W + LOP3 on the integer pipe
// (a plain shift is compiled to IMAD.SHL on the FMA pipe, which the epilogue saturates).
__device__ __forceinline__ uint32_t lo_nib(uint32_t v) {
  return __funnelshift_l(v, v, 4) & 0xF0F0F0F0u;
}
__device__ __forceinline__ uint4 unpack_lo(uint4 v) {  // even channels -> 16*q bytes
  return make_uint4(lo_nib(v.x), lo_nib(v.y), lo_nib(v.z), lo_nib(v.w));
}
__device__ __forceinline__ uint4 unpack_hi(uint4 v) {  // odd channels -> 16*q bytes
  return make_uint4(v.x & 0xF0F0F0F0u, v.y & 0xF0F0F0F0u, v.z & 0xF0F0F0F0u, v.w & 0xF0F0F0F0u);
}
// float(1.5*2^23 + R) from the int32 partial R, |R| < 2^22: the low 23 bits of R with bit 22
// flipped are R + 2^22 in [0, 2^23); OR-ing the exponent of 2^23 gives 2^23 + 2^22 + R exactly.
// One LOP3; `magic` holds kMagicBits in a register.
__device__ __forceinline__ float biased(uint32_t r, uint32_t magic) {
  return __uint_as_float(and_xor(r, 0x007FFFFFu, magic));
}

// KR rows of an operand tile, ROW_STEP apart (a multiple of 8, so all share one swizzle phase):
// packed stage [rows][64 B] -> unpacked SW128 [rows][128 B].  This thread owns the 16-byte
// packed chunk c of rows r0 + k*ROW_STEP; every address is a per-thread base plus an immediate.
template <int KR, int ROW_STEP>
__device__ __forceinline__ void unpack_rows(const uint8_t* stage, uint8_t* ubuf, uint32_t r0,
                                            uint32_t c, bool int4, int h) {
  static_assert(ROW_STEP % 8 == 0, "rows must share the swizzle phase");
  const uint32_t r7 = r0 & 7u;
  const uint8_t* src = stage + r0 * 64 + c * 16;
  uint4 v[KR];
#pragma unroll
  for (int k = 0; k < KR; ++k) v[k] = *reinterpret_cast<const uint4*>(src + k * ROW_STEP * 64);
  uint8_t* dst = ubuf + r0 * 128;
  if (int4) {
    const uint32_t olo = ((2 * c) ^ r7) << 4, ohi = ((2 * c + 1) ^ r7) << 4;
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      *reinterpret_cast<uint4*>(dst + k * ROW_STEP * 128 + olo) = unpack_lo(v[k]);
      *reinterpret_cast<uint4*>(dst + k * ROW_STEP * 128 + ohi) = unpack_hi(v[k]);
    }
  } else {
    const uint32_t o = ((4 * h + c) ^ r7) << 4;
#pragma unroll
    for (int k = 0; k < KR; ++k) *reinterpret_cast<uint4*>(dst + k * ROW_STEP * 128 + o) = v[k];
  }
}

__device__ __forceinline__ long long globaltimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// One work item = (output tile, K split).  Splits cover contiguous group ranges; the INT8 outlier
// group (the last one) therefore always lands in the last split.
struct Item {
  int n0, m0, t0, t1, tile, split;
};
template <int BT>
__device__ __forceinline__ Item make_item(const GemmParams& p, int item) {
  Item it;
  it.tile = item / p.ksplit;
  it.split = item - it.tile * p.ksplit;
  it.n0 = (it.tile / p.m_tiles) * kTileN;
  it.m0 = (it.tile % p.m_tiles) * BT;
  it.t0 = it.split * p.G / p.ksplit;
  it.t1 = (it.split + 1) * p.G / p.ksplit;
  return it;
}

// kMode (development timing probes, never used for results): bit 0 = epilogue skips its
// arithmetic; bit 1 = unpack skips its data movement; bit 2 = producer skips the TMA loads;
// bit 3 = epilogue skips the TMEM loads; bit 4 = waits spin without the suspend-time hint;
// bit 5 = no output stores; bit 6 = no magic prefill (every buffer converted with LOP3).
template <int BT, bool kDebug, int kMode = 0>
__global__ void __launch_bounds__(kThreads, 1)
w4a4_gemm_kernel(const __grid_constant__ CUtensorMap tm_wq4,
                 const __grid_constant__ CUtensorMap tm_aq4,
                 const __grid_constant__ CUtensorMap tm_wq8,
                 const __grid_constant__ CUtensorMap tm_aq8, const GemmParams p) {
  static_assert(BT % 32 == 0 && BT >= 32 && BT <= 256, "token tile");
  constexpr int R = Cfg<BT>::kRing;
  constexpr uint32_t kTmemCols = Cfg<BT>::kTmemCols;
  constexpr bool kPrefillEven = (kMode & 64) == 0;   // even buffers carry the magic bias
  auto wait = [](uint64_t* bar, uint32_t parity) {
    if constexpr ((kMode & 16) != 0) mbar_wait_spin(bar, parity);
    else mbar_wait(bar, parity);
  };
  extern __shared__ uint8_t smem_raw[];
  GemmSmem<BT>& sm = *reinterpret_cast<GemmSmem<BT>*>(
      smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (p.trace != nullptr && threadIdx.x == 0 && blockIdx.x < 256)
    p.trace[768 + blockIdx.x] = globaltimer();

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kNumUnpackWarps);
    }
    for (int u = 0; u < R; ++u) {
      mbar_init(&sm.ufull[u], kNumUnpackWarps);
      mbar_init(&sm.mdone[u], 1);
      mbar_init(&sm.tempty[u], kNumEpiWarps);
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
  if (threadIdx.x < 4) sm.magic4[threadIdx.x] = kMagicBits;
  if (warp == 1) tmem_alloc(&sm.tmem_base, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  const int G4 = p.G4;

  if (warp < kEpiWarp0) setmaxnreg_dec<kRegsLow>();
  if (warp == 0) {
    // ===================== producer warp: group scales (cp.async) + TMA =====================
    // The scales of a group are staged into the scale ring when its first stage is loaded,
    // several groups ahead of the epilogue, which hides the L2 latency of the 4-byte copies
    // (cp.async works for any M; TMA would need 16-byte aligned rows).
    uint32_t it = 0, g_it = 0;
    for (int item = blockIdx.x; item < p.num_items; item += gridDim.x) {
      const Item w = make_item<BT>(p, item);
      for (int t = w.t0; t < w.t1; ++t, ++g_it) {
        {
          const uint32_t sr = g_it % kSRing, sph = (g_it / kSRing) & 1;
          wait(&sm.sfree[sr], sph ^ 1);
          const float* ws = p.w_scales + static_cast<int64_t>(t) * p.N + w.n0;
          const float* as = p.a_scales + static_cast<int64_t>(t) * p.M;
#pragma unroll
          for (int j = lane; j < kTileN; j += 32) cp_async_4(&sm.ssw[sr][j], ws + j);
#pragma unroll
          for (int j = lane; j < BT; j += 32)
            // rows past M: any finite scale works, their partials are exactly zero (TMA
            // zero-fills out-of-range activation rows) and they are never stored
            cp_async_4(&sm.ssa[sr][j], as + min(w.m0 + j, p.M - 1));
          cp_async_mbar_arrive(&sm.sready[sr]);
        }
        const int nh = t < G4 ? 1 : 2;      // the INT8 outlier group arrives in two halves
        for (int h = 0; h < nh; ++h, ++it) {
          const uint32_t s = it % kStages, ph = (it / kStages) & 1;
          wait(&sm.empty[s], ph ^ 1);
          if (lane == 0) {
            if constexpr ((kMode & 4) != 0) {   // probe: no TMA traffic
              mbar_arrive(&sm.full[s]);
            } else {
              mbar_arrive_expect_tx(&sm.full[s], kTileN * 64 + BT * 64);
              if (t < G4) {
                tma_load_2d(sm.stage_w[s], &tm_wq4, &sm.full[s], t * 64, w.n0);
                tma_load_2d(sm.stage_a[s], &tm_aq4, &sm.full[s], t * 64, w.m0);
              } else {
                tma_load_2d(sm.stage_w[s], &tm_wq8, &sm.full[s], h * 64, w.n0);
                tma_load_2d(sm.stage_a[s], &tm_aq8, &sm.full[s], h * 64, w.m0);
              }
            }
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (single thread) =====================
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_i8(kTileN, BT);
      uint32_t g_it = 0;
      for (int item = blockIdx.x; item < p.num_items; item += gridDim.x) {
        const Item w = make_item<BT>(p, item);
        for (int t = w.t0; t < w.t1; ++t, ++g_it) {
          const uint32_t u = g_it % R, uph = (g_it / R) & 1;
          wait(&sm.tempty[u], uph);            // epilogue drained (and re-armed) this accumulator
          wait(&sm.ufull[u], uph);             // operands unpacked
          tc_fence_after();
          if (p.trace != nullptr && blockIdx.x == 0 && g_it < 256) p.trace[g_it] = clock64();
          const uint32_t d = tmem + u * BT;
          const uint32_t a_base = smem_u32(sm.ubuf_w[u]);
          const uint32_t b_base = smem_u32(sm.ubuf_a[u]);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            // even buffers hold the magic 1.5*2^23 (re-armed by the epilogue): always accumulate;
            // odd buffers start from zero and the epilogue converts with one LOP3
            umma_i8(d, umma_desc_sw128(a_base + 32 * k), umma_desc_sw128(b_base + 32 * k), idesc,
                    (k > 0 || (kPrefillEven && (u & 1u) == 0)) ? 1u : 0u);
          umma_commit(&sm.mdone[u]);
          if (p.trace != nullptr && blockIdx.x == 0 && g_it < 256) p.trace[1536 + g_it] = clock64();
        }
      }
    }
  } else if (warp < kEpiWarp0) {
    // ===================== unpack warps: packed INT4 -> int8 (16*q), SW128 =====================
    // threads 0-127: the 128 weight rows + activation rows [0, min(BT,128));
    // threads 128-191: activation rows [128, BT) (BT = 256 only).
    const int ut = threadIdx.x - kUnpackWarp0 * 32;  // 0..191
    const uint32_t r0 = static_cast<uint32_t>(ut & 127) >> 2, c = static_cast<uint32_t>(ut) & 3u;
    uint32_t it = 0, g_it = 0;
    for (int item = blockIdx.x; item < p.num_items; item += gridDim.x) {
      const Item w = make_item<BT>(p, item);
      for (int t = w.t0; t < w.t1; ++t, ++g_it) {
        const uint32_t u = g_it % R, uph = (g_it / R) & 1;
        wait(&sm.mdone[u], uph ^ 1);   // MMAs of group g - R finished with this buffer
        const bool int4 = t < G4;
        const int nh = int4 ? 1 : 2;
        for (int h = 0; h < nh; ++h, ++it) {
          const uint32_t s = it % kStages, ph = (it / kStages) & 1;
          wait(&sm.full[s], ph);
          if constexpr ((kMode & 2) == 0) {
            if (ut < 128) {
              unpack_rows<4, 32>(sm.stage_w[s], sm.ubuf_w[u], r0, c, int4, h);
              unpack_rows<(BT < 128 ? BT : 128) / 32, 32>(sm.stage_a[s], sm.ubuf_a[u], r0, c,
                                                          int4, h);
            } else if constexpr (BT > 128) {
              unpack_rows<(BT - 128) / 16, 16>(sm.stage_a[s] + 128 * 64, sm.ubuf_a[u] + 128 * 128,
                                               r0 & 15u, c, int4, h);
            }
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
    // TMEM is read with the 16x256b shape: thread (tr = lane/4, tc = lane%4) holds, for each
    // 16-lane block blk of its warp's lane quarter and each 8-column chunk j, the MMA-fragment
    // values (row tr, cols 2tc, 2tc+1) and (row tr+8, same cols).  Column pairs share one s_a
    // pair (one 8-byte shared load per chunk for the whole warp), and at the tile end the fp16
    // fragments go through stmatrix.trans into [token][channel] rows for 16-byte global stores.
    setmaxnreg_inc<kRegsHigh>();
    constexpr int COLS = BT / 2;         // token columns per warp (column half of the tile)
    constexpr int NJ = COLS / 8;         // 8-column chunks
    constexpr int JL = NJ >= 4 ? 4 : NJ; // chunks per TMEM load (16x256b.xJL)
    const int e = warp - kEpiWarp0;
    const int q = warp & 3;              // TMEM lane quarter this warp may access
    const int half = e >> 2;
    const int tr = lane >> 2, tc = lane & 3;
    const uint32_t tq = tmem + (static_cast<uint32_t>(q * 32) << 16) + half * COLS;
    const uint32_t magic = kMagicBits;
    // Resident copies of the magic as tcgen05.st sources (see the STTM re-arm below).
    uint32_t mg[4];
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(mg[0]), "=r"(mg[1]), "=r"(mg[2]), "=r"(mg[3])
                 : "r"(smem_u32(sm.magic4)));
    // Even accumulator buffers carry the magic bias (tcgen05.st, TMEM write port); odd ones are
    // converted with a LOP3 (ALU) -- see DESIGN.md "Epilogue arithmetic".
    if constexpr (kPrefillEven) {
#pragma unroll
      for (int b = 0; b < R; b += 2)
#pragma unroll
        for (int c = 0; c < COLS; c += 4) tmem_st4(tq + b * BT + c, mg);
      tmem_st_wait();
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0)
      for (int b = 0; b < R; ++b) mbar_arrive(&sm.tempty[b]);
    uint8_t* stg = sm.ostg[e];           // per-warp staging for the transposed output
    uint32_t g_it = 0;
    for (int item = blockIdx.x; item < p.num_items; item += gridDim.x) {
      const Item w = make_item<BT>(p, item);
      const int n0 = w.n0, m0 = w.m0;
      const int mc0 = m0 + half * COLS;
      // acc[blk][j][h]: rows 32q + 16 blk + tr + 8 h, columns (token) 8j + 2tc + {0, 1}
      float2 acc[2][NJ][2];
#pragma unroll
      for (int bk = 0; bk < 2; ++bk)
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          acc[bk][j][0] = make_float2(0.0f, 0.0f);
          acc[bk][j][1] = make_float2(0.0f, 0.0f);
        }
      for (int t = w.t0; t < w.t1; ++t, ++g_it) {
        const uint32_t b = g_it % R, bph = (g_it / R) & 1;
        const uint32_t sr = g_it % kSRing, sph = (g_it / kSRing) & 1;
        const bool int4 = t < G4;
        wait(&sm.sready[sr], sph);
        // Dequantize T = float(1.5*2^23 + R) with ONE fma: g = T*sw' - 1.5*2^23*sw' = sw'*R,
        // rounded once.  sw' = sw (x1/256 for INT4 groups, exact) with its 2 lowest mantissa
        // bits cleared so that 1.5*2^23*sw' is exact; see DESIGN.md "Epilogue arithmetic".
        float2 sw2[2][2], nc2[2][2];
#pragma unroll
        for (int bk = 0; bk < 2; ++bk)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float sw = sm.ssw[sr][q * 32 + 16 * bk + 8 * h + tr];
            if (int4) sw *= (1.0f / 256.0f);
            const float swh = __uint_as_float(__float_as_uint(sw) & 0xFFFFFFFCu);
            sw2[bk][h] = make_float2(swh, swh);
            nc2[bk][h] = make_float2(-kMagic * swh, -kMagic * swh);
          }
        const float2* sa2 = reinterpret_cast<const float2*>(&sm.ssa[sr][half * COLS + 2 * tc]);
        wait(&sm.mdone[b], bph);
        tc_fence_after();
        if (p.trace != nullptr && blockIdx.x == 0 && g_it < 256 && e == 0 && lane == 0)
          p.trace[512 + g_it] = clock64();
        const uint32_t taddr = tq + b * BT;
        auto drain = [&](auto pre_tag) {
          constexpr bool kPre = decltype(pre_tag)::value;
#pragma unroll
          for (int jl = 0; jl < NJ / JL; ++jl) {
            uint32_t r[2][4 * JL];
            if constexpr ((kMode & 8) == 0) {
              tmem_ld_16x256b<JL>(taddr + jl * 8 * JL, r[0]);
              tmem_ld_16x256b<JL>(taddr + (16u << 16) + jl * 8 * JL, r[1]);
              tmem_ld_wait();
            } else {
#pragma unroll
              for (int k = 0; k < 4 * JL; ++k) r[0][k] = r[1][k] = 0;
            }
            if (jl == NJ / JL - 1) {
              if constexpr (kPre && (kMode & 8) == 0) {   // re-arm the whole region
#pragma unroll
                for (int c = 0; c < COLS; c += 4) tmem_st4(taddr + c, mg);
                tmem_st_wait();
              }
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&sm.tempty[b]);
            }
            if constexpr (!kPre) {
#pragma unroll
              for (int k = 0; k < 4 * JL; ++k) {
                r[0][k] = __float_as_uint(biased(r[0][k], magic));
                r[1][k] = __float_as_uint(biased(r[1][k], magic));
              }
            }
#pragma unroll
            for (int jj = 0; jj < JL; ++jj) {
              const int j = jl * JL + jj;
              if constexpr (kDebug) {
#pragma unroll
                for (int bk = 0; bk < 2; ++bk)
#pragma unroll
                  for (int v = 0; v < 4; ++v) {
                    const int m = mc0 + 8 * j + 2 * tc + (v & 1);
                    const int n = n0 + q * 32 + 16 * bk + tr + 8 * (v >> 1);
                    const int raw = static_cast<int>(r[bk][4 * jj + v] - kMagicBits);
                    if (m < p.M)
                      p.debug[(static_cast<int64_t>(t) * p.M + m) * p.N + n] = int4 ? (raw >> 8) : raw;
                  }
              }
              if constexpr ((kMode & 1) == 0) {
                const float2 sa = sa2[4 * j];   // s_a of columns 8j + 2tc, +1
#pragma unroll
                for (int bk = 0; bk < 2; ++bk)
#pragma unroll
                  for (int h = 0; h < 2; ++h) {
                    const float2 g = __ffma2_rn(
                        make_float2(__uint_as_float(r[bk][4 * jj + 2 * h]),
                                    __uint_as_float(r[bk][4 * jj + 2 * h + 1])),
                        sw2[bk][h], nc2[bk][h]);
                    acc[bk][j][h] = __ffma2_rn(sa, g, acc[bk][j][h]);
                  }
              }
            }
          }
        };
        if (kPrefillEven && (b & 1u) == 0) drain(std::true_type{});
        else drain(std::false_type{});
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.sfree[sr]);
      }
      if (p.trace != nullptr && threadIdx.x == kEpiWarp0 * 32 && blockIdx.x < 256)
        p.trace[1024 + blockIdx.x] = globaltimer();
      if constexpr ((kMode & 32) != 0) continue;

      // ---- split-K: publish this split's fp32 partial in the fragment layout; the last
      //      split to arrive sums all partials in split order (deterministic) into acc ----
      if (p.ksplit > 1) {
        float* slot = p.partials + (static_cast<int64_t>(w.tile) * p.ksplit + w.split) * kTileN * BT;
        auto frag_ptr = [&](float* base, int bk, int j, int h) {
          return reinterpret_cast<float2*>(
              base + static_cast<int64_t>(q * 32 + 16 * bk + 8 * h + tr) * BT + half * COLS +
              8 * j + 2 * tc);
        };
#pragma unroll
        for (int bk = 0; bk < 2; ++bk)
#pragma unroll
          for (int j = 0; j < NJ; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) *frag_ptr(slot, bk, j, h) = acc[bk][j][h];
        __threadfence();
        named_bar_sync(1, kNumEpiWarps * 32);   // all epilogue threads of this CTA have written
        __shared__ int arrived;
        if (threadIdx.x == kEpiWarp0 * 32) arrived = atomicAdd(p.counters + w.tile, 1);
        named_bar_sync(1, kNumEpiWarps * 32);
        const bool last = arrived == p.ksplit - 1;
        named_bar_sync(1, kNumEpiWarps * 32);   // everyone has read `arrived`
        if (!last) continue;
        __threadfence();
        if (threadIdx.x == kEpiWarp0 * 32) p.counters[w.tile] = 0;   // self-cleaning
        float* slot0 = p.partials + static_cast<int64_t>(w.tile) * p.ksplit * kTileN * BT;
#pragma unroll
        for (int bk = 0; bk < 2; ++bk)
#pragma unroll
          for (int j = 0; j < NJ; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) acc[bk][j][h] = make_float2(0.0f, 0.0f);
        for (int sp = 0; sp < p.ksplit; ++sp) {
          float* sl = slot0 + static_cast<int64_t>(sp) * kTileN * BT;
#pragma unroll
          for (int bk = 0; bk < 2; ++bk)
#pragma unroll
            for (int j = 0; j < NJ; ++j)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const float2 o = __ldcg(frag_ptr(sl, bk, j, h));
                acc[bk][j][h].x += o.x;
                acc[bk][j][h].y += o.y;
              }
        }
      }

      // ---- tile output: stmatrix.trans turns the 8x8 (channel, token) fragments into
      //      [token][channel] rows of the per-warp staging; each lane then moves 16 bytes
      //      (8 channels of one token) to C.  fp32 output transposes the high and low 16-bit
      //      halves separately and re-interleaves them. ----
      // staging rows: 8 tokens x (32 channels) with an 80-byte pitch (bank-conflict free)
      const uint32_t st_addr = smem_u32(stg) + (lane & 7) * 80 + (lane >> 3) * 16;
      const int om = lane >> 2, op = lane & 3;                 // readback: token row, 8-ch piece
      const int ncol = n0 + q * 32 + 8 * op;
      for (int j = 0; j < NJ; ++j) {
        const int m = mc0 + 8 * j + om;
        if (!p.c_f32) {
          uint32_t h4[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const __half2 hh = __floats2half2_rn(acc[i >> 1][j][i & 1].x, acc[i >> 1][j][i & 1].y);
            h4[i] = *reinterpret_cast<const uint32_t*>(&hh);
          }
          stmatrix_x4_trans(st_addr, h4);
          __syncwarp();
          const uint4 v = *reinterpret_cast<const uint4*>(stg + om * 80 + op * 16);
          __syncwarp();
          if (m < p.M)
            *reinterpret_cast<uint4*>(static_cast<__half*>(p.c) + static_cast<int64_t>(m) * p.ldc +
                                      ncol) = v;
        } else {
          uint32_t hi4[4], lo4[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint32_t a = __float_as_uint(acc[i >> 1][j][i & 1].x);
            const uint32_t c = __float_as_uint(acc[i >> 1][j][i & 1].y);
            hi4[i] = __byte_perm(a, c, 0x7632);   // (hi(a), hi(c))
            lo4[i] = __byte_perm(a, c, 0x5410);   // (lo(a), lo(c))
          }
          stmatrix_x4_trans(st_addr, hi4);
          stmatrix_x4_trans(st_addr + 640, lo4);
          __syncwarp();
          const uint4 hv = *reinterpret_cast<const uint4*>(stg + om * 80 + op * 16);
          const uint4 lv = *reinterpret_cast<const uint4*>(stg + 640 + om * 80 + op * 16);
          __syncwarp();
          if (m < p.M) {
            float4* dst = reinterpret_cast<float4*>(static_cast<float*>(p.c) +
                                                    static_cast<int64_t>(m) * p.ldc + ncol);
            dst[0] = make_float4(__uint_as_float(__byte_perm(lv.x, hv.x, 0x5410)),
                                 __uint_as_float(__byte_perm(lv.x, hv.x, 0x7632)),
                                 __uint_as_float(__byte_perm(lv.y, hv.y, 0x5410)),
                                 __uint_as_float(__byte_perm(lv.y, hv.y, 0x7632)));
            dst[1] = make_float4(__uint_as_float(__byte_perm(lv.z, hv.z, 0x5410)),
                                 __uint_as_float(__byte_perm(lv.z, hv.z, 0x7632)),
                                 __uint_as_float(__byte_perm(lv.w, hv.w, 0x5410)),
                                 __uint_as_float(__byte_perm(lv.w, hv.w, 0x7632)));
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (p.trace != nullptr && threadIdx.x == 0 && blockIdx.x < 256)
    p.trace[1280 + blockIdx.x] = globaltimer();
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
static cudaError_t launch_bt(const GemmArgs& a, const GemmPlan& plan, void* workspace,
                             cudaStream_t stream, int num_sms, int* launches) {
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
  p.ksplit = plan.ksplit;
  p.num_items = p.num_tiles * p.ksplit;
  p.counters = nullptr;
  p.partials = nullptr;
  if (plan.ksplit > 1) {
    p.counters = static_cast<int*>(workspace);
    p.partials = reinterpret_cast<float*>(static_cast<char*>(workspace) + plan.counter_bytes);
    cudaError_t e = cudaMemsetAsync(p.counters, 0, plan.counter_bytes, stream);
    if (e != cudaSuccess) return e;
    ++*launches;
  }

  const size_t smem = sizeof(GemmSmem<BT>) + 1024;
  auto kern = p.debug ? w4a4_gemm_kernel<BT, true> : w4a4_gemm_kernel<BT, false>;
  if constexpr (BT == 256) {
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
    if (mode == 32) kern = w4a4_gemm_kernel<BT, false, 32>;
    if (mode == 64) kern = w4a4_gemm_kernel<BT, false, 64>;
    if (mode == 33) kern = w4a4_gemm_kernel<BT, false, 33>;
    if (mode == 34) kern = w4a4_gemm_kernel<BT, false, 34>;
    if (mode == 39) kern = w4a4_gemm_kernel<BT, false, 39>;


  }
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int grid = p.num_items < num_sms ? p.num_items : num_sms;
  static long long* trace = nullptr;
  static const bool want_trace = getenv("ATOM_GEMM_TRACE") != nullptr;   // development probe only
  if (want_trace && trace == nullptr) cudaMalloc(&trace, 7 * 256 * sizeof(long long));
  p.trace = want_trace ? trace : nullptr;
  kern<<<grid, kThreads, smem, stream>>>(m_wq4, m_aq4, m_wq8, m_aq8, p);
  ++*launches;
  if (want_trace) {
    long long h[1792];
    cudaMemcpy(h, trace, sizeof(h), cudaMemcpyDeviceToHost);
    fprintf(stderr, "plan: BT=%d ksplit=%d tiles=%d items=%d grid=%d\n", BT, p.ksplit,
            p.num_tiles, p.num_items, grid);
    fprintf(stderr, "trace g: ufull_arrive mma_issue mma_committed epi_seen (clk rel. to mma_issue[0])\n");
    for (int g = 0; g < 256 && g < p.G * 2; ++g)
      fprintf(stderr, "%3d %9lld %9lld %9lld %9lld\n", g, h[256 + g] - h[0], h[g] - h[0],
              h[1536 + g] - h[0], h[512 + g] - h[0]);
    long long t0 = h[768];
    for (int b = 0; b < grid && b < 256; ++b) t0 = h[768 + b] < t0 ? h[768 + b] : t0;
    fprintf(stderr, "cta: start_ns groups_done_ns end_ns (rel. to first start)\n");
    for (int b = 0; b < grid && b < 256; ++b)
      fprintf(stderr, "%3d %8lld %8lld %8lld\n", b, h[768 + b] - t0, h[1024 + b] - t0,
              h[1280 + b] - t0);
  }
  return cudaGetLastError();
}

// Tile / split-K plan.  BT = 256 tokens when the 128 x 256 tiles fill the SMs; otherwise the
// smallest power of two >= M (no wasted token columns) and the K groups are split S ways so that
// the (tile, split) items fill one wave as evenly as possible (each split >= 4 groups).  Splits
// publish fp32 partials in the workspace; the last split to arrive reduces (no spinning).
GemmPlan plan_w4a4_gemm(int64_t M, int64_t N, int64_t K, int num_sms) {
  GemmPlan pl;
  const int64_t n_tiles = N / kTileN;
  const int G = static_cast<int>(K / 128);
  auto tiles = [&](int bt) { return n_tiles * ((M + bt - 1) / bt); };
  if (tiles(256) >= num_sms) {
    pl.bt = 256;
  } else {
    pl.bt = 32;
    while (pl.bt < 256 && pl.bt < M) pl.bt *= 2;
  }
  const int64_t t = tiles(pl.bt);
  pl.ksplit = 1;
  if (t < 2 * num_sms) {
    double best = 1e30;
    for (int sp = 1; sp <= G / 4 && sp <= 16; ++sp) {
      const double cost = static_cast<double>((t * sp + num_sms - 1) / num_sms) / sp;
      if (cost < best - 1e-9) {
        best = cost;
        pl.ksplit = sp;
      }
    }
  }
  pl.num_tiles = t;
  if (pl.ksplit > 1) {
    pl.counter_bytes = ((t * sizeof(int) + 255) / 256) * 256;
    pl.workspace_bytes = pl.counter_bytes + t * pl.ksplit * kTileN * pl.bt * sizeof(float);
  }
  return pl;
}

cudaError_t launch_w4a4_gemm(const GemmArgs& a, void* workspace, size_t workspace_bytes,
                             cudaStream_t stream, int num_sms, int* launches) {
  *launches = 0;
  if (a.M == 0) return cudaSuccess;
  const GemmPlan pl = plan_w4a4_gemm(a.M, a.N, a.K, num_sms);
  if (workspace_bytes < pl.workspace_bytes) return cudaErrorInvalidValue;
  switch (pl.bt) {
    case 256: return launch_bt<256>(a, pl, workspace, stream, num_sms, launches);
    case 128: return launch_bt<128>(a, pl, workspace, stream, num_sms, launches);
    case 64: return launch_bt<64>(a, pl, workspace, stream, num_sms, launches);
    default: return launch_bt<32>(a, pl, workspace, stream, num_sms, launches);
  }
}

}  // namespace atom
