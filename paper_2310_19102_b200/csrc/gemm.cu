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
  float oscr[kNumEpiWarps][4][72];      // per-warp 8x8 transpose scratch for the tile output
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
    setmaxnreg_inc<kRegsHigh>();
    constexpr int COLS = BT / 2;  // tokens per thread
    constexpr int CH = (COLS >= 32 && COLS < 128) ? 32 : 16;   // x16 at COLS = 128: register budget
    const int e = warp - kEpiWarp0;
    const int q = warp & 3;       // TMEM lane quarter this warp may access
    const int half = e >> 2;
    const int n_local = q * 32 + lane;
    const uint32_t tlane = tmem + (static_cast<uint32_t>(q * 32) << 16) + half * COLS;
    const uint32_t magic = kMagicBits;
    // Resident copies of the magic as tcgen05.st sources: loaded once from shared memory so the
    // compiler cannot re-materialise them with 4 IMAD.MOV (FMA pipe) before every store.
    uint32_t mg[4];
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(mg[0]), "=r"(mg[1]), "=r"(mg[2]), "=r"(mg[3])
                 : "r"(smem_u32(sm.magic4)));
    // Even accumulator buffers carry the magic bias (tcgen05.st, TMEM write port); odd ones are
    // converted with a LOP3 (ALU).  Splitting the conversion between the two keeps both the TMEM
    // bandwidth and the ALU pipe below the MMA time.
    if constexpr (kPrefillEven) {
#pragma unroll
      for (int b = 0; b < R; b += 2)
#pragma unroll
        for (int ch = 0; ch < COLS / CH; ++ch) tmem_st_const<CH>(tlane + b * BT + ch * CH, magic);
      tmem_st_wait();
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0)
      for (int b = 0; b < R; ++b) mbar_arrive(&sm.tempty[b]);
    uint32_t g_it = 0;
    for (int item = blockIdx.x; item < p.num_items; item += gridDim.x) {
      const Item w = make_item<BT>(p, item);
      const int n0 = w.n0, m0 = w.m0;
      const int n = n0 + n_local;
      const int mc0 = m0 + half * COLS;
      float2 acc[COLS / 2];
#pragma unroll
      for (int j = 0; j < COLS / 2; ++j) acc[j] = make_float2(0.0f, 0.0f);
      for (int t = w.t0; t < w.t1; ++t, ++g_it) {
        const uint32_t b = g_it % R, bph = (g_it / R) & 1;
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
        // Two specialised copies of the drain: even buffers are magic-prefilled (re-armed with
        // tcgen05.st), odd ones are converted with a LOP3; no per-element select.
        auto drain = [&](auto pre_tag) {
          constexpr bool kPre = decltype(pre_tag)::value;
          constexpr int NCH = COLS / CH;
          // software-pipelined: chunk ch+1 is loaded from TMEM while chunk ch is computed
          uint32_t rb[2][CH];
          if constexpr ((kMode & 8) == 0) {
            tmem_ld<CH>(taddr, rb[0]);
            tmem_ld_wait();
          } else {
#pragma unroll
            for (int k = 0; k < CH; ++k) rb[0][k] = 0;
          }
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) {
            uint32_t (&r)[CH] = rb[ch & 1];
            if constexpr (kPre && (kMode & 8) == 0) {   // re-arm this chunk with the magic
#pragma unroll
              for (int k = 0; k < CH; k += 4) tmem_st4(taddr + ch * CH + k, mg);
            }
            if (ch + 1 < NCH) {
              if constexpr ((kMode & 8) == 0) tmem_ld<CH>(taddr + (ch + 1) * CH, rb[(ch + 1) & 1]);
              else {
#pragma unroll
                for (int k = 0; k < CH; ++k) rb[(ch + 1) & 1][k] = 0;
              }
            } else {
              if constexpr (kPre) tmem_st_wait();
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&sm.tempty[b]);
            }
            if constexpr (!kPre) {
#pragma unroll
              for (int k = 0; k < CH; ++k) r[k] = __float_as_uint(biased(r[k], magic));
            }
            if constexpr (kDebug) {
#pragma unroll
              for (int k = 0; k < CH; ++k) {
                const int m = mc0 + ch * CH + k;
                const int v = static_cast<int>(r[k] - kMagicBits);
                if (m < p.M)
                  p.debug[(static_cast<int64_t>(t) * p.M + m) * p.N + n] = int4 ? (v >> 8) : v;
              }
            }
#pragma unroll
            for (int k4 = 0; k4 < ((kMode & 1) ? 0 : CH / 4); ++k4) {
              const float4 s = sa4[ch * (CH / 4) + k4];
              const int j = ch * (CH / 2) + 2 * k4;
              const float2 g0 = __ffma2_rn(make_float2(__uint_as_float(r[4 * k4 + 0]),
                                                       __uint_as_float(r[4 * k4 + 1])), sw2, nc2);
              const float2 g1 = __ffma2_rn(make_float2(__uint_as_float(r[4 * k4 + 2]),
                                                       __uint_as_float(r[4 * k4 + 3])), sw2, nc2);
              acc[j] = __ffma2_rn(make_float2(s.x, s.y), g0, acc[j]);
              acc[j + 1] = __ffma2_rn(make_float2(s.z, s.w), g1, acc[j + 1]);
            }
            if (ch + 1 < NCH) {
              if constexpr ((kMode & 8) == 0) tmem_ld_wait();
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
      // ---- tile output ----
      // Thread = output channel n, registers = tokens m; C is [M][N] with n contiguous.  Each
      // 8x8 (m, n) block is transposed through a per-warp shared scratch so that every lane
      // stores 8 consecutive n of one token as one 16-byte vector (4 lanes per 64-byte row
      // segment), instead of 2-byte scattered stores.  With split-K the same fp32 path writes the
      // split's partial tile [BT][128] to the workspace; the last split to arrive then sums the
      // partials in split order (deterministic) with coalesced 16-byte loads and stores C.
      if constexpr ((kMode & 32) != 0) continue;
      const int ga = lane >> 3, gb = lane & 7;
      float* scr = &sm.oscr[e][ga][0];
      const bool split = p.ksplit > 1;
      float* f32_base;
      int64_t f32_ld;
      int row0, col0, row_limit;
      if (split) {
        f32_base = p.partials + (static_cast<int64_t>(w.tile) * p.ksplit + w.split) * BT * kTileN;
        f32_ld = kTileN;
        row0 = half * COLS;
        col0 = q * 32 + 8 * ga;
        row_limit = BT;
      } else {
        f32_base = static_cast<float*>(p.c);
        f32_ld = p.ldc;
        row0 = mc0;
        col0 = n0 + q * 32 + 8 * ga;
        row_limit = p.M;
      }
      if (split || p.c_f32) {
#pragma unroll
        for (int c8 = 0; c8 < COLS / 8; ++c8) {
          float4* wv = reinterpret_cast<float4*>(scr + gb * 8);
          wv[0] = make_float4(acc[4 * c8].x, acc[4 * c8].y, acc[4 * c8 + 1].x, acc[4 * c8 + 1].y);
          wv[1] = make_float4(acc[4 * c8 + 2].x, acc[4 * c8 + 2].y, acc[4 * c8 + 3].x,
                              acc[4 * c8 + 3].y);
          __syncwarp();
          float v[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] = scr[k * 8 + gb];
          __syncwarp();
          const int m = row0 + 8 * c8 + gb;
          if (m < row_limit) {
            float4* dst = reinterpret_cast<float4*>(f32_base + static_cast<int64_t>(m) * f32_ld + col0);
            dst[0] = make_float4(v[0], v[1], v[2], v[3]);
            dst[1] = make_float4(v[4], v[5], v[6], v[7]);
          }
        }
      } else {
        // fp16 first: halves the live registers before the transpose
        uint32_t hp[COLS / 2];
#pragma unroll
        for (int j = 0; j < COLS / 2; ++j) {
          const __half2 h = __floats2half2_rn(acc[j].x, acc[j].y);
          hp[j] = *reinterpret_cast<const uint32_t*>(&h);
        }
        uint16_t* hs = reinterpret_cast<uint16_t*>(scr);
        __half* crow = static_cast<__half*>(p.c) + static_cast<int64_t>(mc0 + gb) * p.ldc + col0;
        const int64_t step = 8 * p.ldc;
#pragma unroll
        for (int c8 = 0; c8 < COLS / 8; ++c8) {
          *reinterpret_cast<uint4*>(hs + gb * 8) =
              make_uint4(hp[4 * c8], hp[4 * c8 + 1], hp[4 * c8 + 2], hp[4 * c8 + 3]);
          __syncwarp();
          uint32_t wv[4];
#pragma unroll
          for (int k = 0; k < 4; ++k)
            wv[k] = static_cast<uint32_t>(hs[(2 * k) * 8 + gb]) |
                    (static_cast<uint32_t>(hs[(2 * k + 1) * 8 + gb]) << 16);
          __syncwarp();
          if (mc0 + 8 * c8 + gb < p.M)
            *reinterpret_cast<uint4*>(crow + c8 * step) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        }
      }
      if (split) {
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
        const float* slot0 = p.partials + static_cast<int64_t>(w.tile) * p.ksplit * BT * kTileN;
        const int et = threadIdx.x - kEpiWarp0 * 32;   // 0..255
        constexpr int kChunks = BT * (kTileN / 4);       // float4 chunks of the tile
        constexpr int kPerThread = kChunks / (kNumEpiWarps * 32);
        constexpr int kBatch = kPerThread < 4 ? kPerThread : 4;
        // batches of kBatch chunks: all loads of a batch are issued before any use (L2 latency)
        for (int b0 = 0; b0 < kPerThread; b0 += kBatch) {
          float4 sum[kBatch];
#pragma unroll
          for (int k = 0; k < kBatch; ++k) sum[k] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
          for (int sp = 0; sp < p.ksplit; ++sp) {
            float4 o[kBatch];
#pragma unroll
            for (int k = 0; k < kBatch; ++k)
              o[k] = __ldcg(reinterpret_cast<const float4*>(
                         slot0 + static_cast<int64_t>(sp) * BT * kTileN) +
                     et + (b0 + k) * (kNumEpiWarps * 32));
#pragma unroll
            for (int k = 0; k < kBatch; ++k) {
              sum[k].x += o[k].x; sum[k].y += o[k].y; sum[k].z += o[k].z; sum[k].w += o[k].w;
            }
          }
#pragma unroll
          for (int k = 0; k < kBatch; ++k) {
            const int idx = et + (b0 + k) * (kNumEpiWarps * 32);
            const int ml = idx / (kTileN / 4), nl = (idx % (kTileN / 4)) * 4;
            const int m = m0 + ml;
            if (m >= p.M) continue;
            if (p.c_f32) {
              *reinterpret_cast<float4*>(static_cast<float*>(p.c) + static_cast<int64_t>(m) * p.ldc +
                                         n0 + nl) = sum[k];
            } else {
              const __half2 h0 = __floats2half2_rn(sum[k].x, sum[k].y);
              const __half2 h1 = __floats2half2_rn(sum[k].z, sum[k].w);
              *reinterpret_cast<uint2*>(static_cast<__half*>(p.c) + static_cast<int64_t>(m) * p.ldc +
                                        n0 + nl) =
                  make_uint2(*reinterpret_cast<const uint32_t*>(&h0),
                             *reinterpret_cast<const uint32_t*>(&h1));
            }
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
