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
//   * weights stay PACKED in HBM: TMA streams 64-byte-per-row INT4 tiles into a 4-stage ring and
//     2 unpack warps expand the nibbles to int8 16*q (high nibbles: one LOP per 4 codes; low
//     nibbles: SHF.L.W + LOP; exact two's complement) directly into the 128B-swizzled K-major
//     layout the UMMA descriptor reads.  tcgen05 has no s4 kind, so this is the INT4 -> INT8 step.
//     The INT8 outlier group arrives as two 64-byte halves through the same ring.
//   * activations arrive MMA-ready: atom_reorder_quantize writes the codes one per byte in the
//     same intra-group order the weight unpack produces (atom.h "x8"), so TMA (SWIZZLE_128B)
//     drops them straight into the operand buffer; no SM work, a third of the old SMEM traffic.
//   * 1 MMA thread per group: 4 x kind::i8 (K = 32) into a TMEM int32 accumulator (RT buffers
//     rotate across groups so later groups multiply while the epilogue drains earlier ones) and
//     ONE tcgen05.commit that frees the operand slot and publishes the partial.  INT4 partials
//     come out as R = 16*P_t (exact, |R| <= 2^17).
//   * 12 epilogue warps (thread = output channel = TMEM lane, 3 warps per lane quarter, each a
//     third of the token columns) tcgen05.ld the partials, read them as the float
//     1.5*2^23 + R (magic-prefilled accumulators, or one LOP3), dequantize with one FFMA2 and
//     accumulate with one more; fp32 accumulators live in
//     registers; after the tile's last group they write fp16 (or fp32 for K-shards).
//   * stream-K schedule: the (tile, group) units are divided evenly over one persistent CTA per
//     SM.  A tile cut between CTAs is computed in K segments; every segment but the last
//     publishes its fp32 partial in the workspace, the CTA with the last segment adds them in a
//     fixed order (deterministic) and stores.  Each CTA walks its tiles in descending order, so
//     the segments it publishes are its first work and the one it reduces is its last.
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
//   WG0: warp 0 packed-weight producer (TMA), warp 1 MMA issuer, warp 2 activation-tile
//        loader (TMA), warp 3 group-scale loader (cp.async)
//   WG1: warps 4-7 unpack (one per SM sub-partition, so it never queues behind 2 others)
//   WG2-WG3: warps 8-15 epilogue (warp % 4 = TMEM lane quarter, (warp - 8) / 4 = column half)
// setmaxnreg moves registers from WG0/WG1 (56 each) to the epilogue warpgroups (200 each),
// which hold the fp32 accumulators of a 128 x BT tile (BT/2 per thread).
constexpr int kThreads = 512;
constexpr int kALoaderWarp = 2;
constexpr int kScaleWarp = 3;
constexpr int kUnpackWarp0 = 4;
constexpr int kNumUnpackWarps = 4;
constexpr int kEpiWarp0 = 8;
constexpr int kNumEpiWarps = 8;
constexpr int kEpiPerQuarter = kNumEpiWarps / 4;   // warps sharing one TMEM lane quarter
constexpr int kEpiThreads = kNumEpiWarps * 32;
constexpr int kRegsLow = 56, kRegsHigh = 200;           // 8*32*56 + 8*32*200 = 65536
constexpr int kTileN = 128;     // output channels per tile (MMA M)

template <int BT> struct Cfg {
  static constexpr int RT = BT >= 256 ? 2 : 4;          // TMEM accumulator buffers
  static constexpr int RS = 4;                          // activation slots (= go / mdone ring)
  static constexpr int RW = BT >= 256 ? 2 : 4;          // unpacked weight slots
  static constexpr int kStages = BT >= 256 ? 3 : 4;     // weight TMA ring depth (16 KB stages)
  static constexpr uint32_t kTmemCols = RT * BT <= 32 ? 32 : RT * BT <= 64 ? 64
                                      : RT * BT <= 128 ? 128 : RT * BT <= 256 ? 256 : 512;
  static constexpr int NC = BT / 8;                     // 8-column chunks of the tile
  static constexpr int NJ = (NC + kEpiPerQuarter - 1) / kEpiPerQuarter;   // chunks per warp
  // split-tile partial of one CTA: thread-linear, [epi warps][NJ*8/4 column quads][32 lanes] float4
  static constexpr size_t kSlotFloats = static_cast<size_t>(kNumEpiWarps) * NJ * 8 * 32;
  static_assert(RT * BT <= 512, "TMEM holds at most 512 columns");
  static_assert(RS >= RT && RS >= RW, "ring sizes");
};

constexpr uint32_t kMagicBits = 0x4B400000u;   // bit pattern of 1.5*2^23
constexpr float kMagic = 12582912.0f;          // 1.5*2^23

struct GemmParams {
  const float* a_scales;
  const float* w_scales;
  void* c;
  int64_t ldc;
  int32_t* debug;
  int M, N, G, G4, c_f32;
  int m_tiles, num_tiles;
  int dp_waves;              // whole tiles per CTA dealt round-robin
  int64_t sk_base;           // first stream-K unit (= dp_waves * grid * G)
  int64_t sk_units;          // stream-K (tile, group) units
  float* partials;           // [gridDim.x][kSlotFloats] split-tile partials
  int* counters;             // [gridDim.x] arrivals per reducing CTA (zero between launches)
  long long* trace;          // development timeline probe (ATOM_GEMM_TRACE): [8][kTraceN] clocks
};
constexpr int kTraceN = 512;
__device__ __forceinline__ long long globaltimer_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// development probe: clock64 of event ev for group g of CTA 0 (no-op unless p.trace is set)
#define TRACE(ev, g)                                                                          \
  do {                                                                                        \
    if (p.trace != nullptr && blockIdx.x == 0 && (g) < kTraceN)                               \
      p.trace[(ev) * kTraceN + (g)] = clock64();                                              \
  } while (0)

template <int BT>
struct __align__(1024) GemmSmem {
  static constexpr int RS = Cfg<BT>::RS;
  static constexpr int RW = Cfg<BT>::RW;
  static constexpr int RT = Cfg<BT>::RT;
  uint8_t ubuf_w[RW][kTileN * 128];     // unpacked weight group, SW128 K-major
  uint8_t ubuf_a[RS][BT * 128];         // activation group (x8), SW128 K-major, written by TMA
  uint8_t stage_w[Cfg<BT>::kStages][kTileN * 128];  // packed weights: 2 INT4 groups or INT8
  float ssw[RS][kTileN];                // weight scales of group g in slot g % RS (cp.async)
  float ssa[RS][BT];                    // activation scales of the same group
  uint8_t ostg[kNumEpiWarps][1024];     // per-warp output staging ([8 tokens][32 ch] fp32)
  uint64_t full[Cfg<BT>::kStages], empty[Cfg<BT>::kStages];
  // go[u]: group g (slot u = g % RS) may be issued -- its weights are unpacked (2 arrivals),
  // its activations landed (1 arrival + tx bytes) and its TMEM buffer was drained (12 epilogue
  // arrivals, made when group g - RT was released).  One barrier, one probe per group.
  uint64_t go[RS];
  uint64_t mdone[RS];                   // MMAs of a group done: slot free + partial ready
  uint64_t sfree[RS];                   // epilogue done with the scales in slot g % RS
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
// The same value as an integer add, R * 1 + 0x4B400000 (= the LOP3 result for |R| < 2^22).
// ptxas emits it as VIADD, which does not issue to the ALU pipe the LOP3s (and the unpack warps)
// load; used for half of the columns (measured best of 0, 1/4, 1/2, 3/4).
__device__ __forceinline__ float biased_fma(uint32_t r, uint32_t one, uint32_t magic) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(r), "r"(one), "r"(magic));
  return __uint_as_float(d);
}

// KR rows of the weight tile, ROW_STEP apart (a multiple of 8, so all share one swizzle phase):
// packed stage [rows][128 B] (two INT4 groups, or the INT8 group) -> unpacked SW128 [rows][128 B].
// This thread owns the 16-byte packed chunk c (< 4) of group `sub` of rows r0 + k*ROW_STEP;
// every address is a per-thread base plus an immediate.  Packed chunk c holds channels
// 32c..32c+31; its low nibbles (even channels) become 16-byte chunk 2c and its high nibbles (odd
// channels) chunk 2c+1 -- the x8 order of atom.h.  The INT8 group is copied as is (chunks c and
// c + 4 of the 128-byte row).
template <int KR, int ROW_STEP>
__device__ __forceinline__ void unpack_rows(const uint8_t* stage, uint8_t* ubuf, uint32_t r0,
                                            uint32_t c, bool int4, int sub) {
  static_assert(ROW_STEP % 8 == 0, "rows must share the swizzle phase");
  const uint32_t r7 = r0 & 7u;
  uint8_t* dst = ubuf + r0 * 128;
  if (int4) {
    const uint8_t* src = stage + r0 * 128 + sub * 64 + c * 16;
    uint4 v[KR];
#pragma unroll
    for (int k = 0; k < KR; ++k) v[k] = *reinterpret_cast<const uint4*>(src + k * ROW_STEP * 128);
    const uint32_t olo = ((2 * c) ^ r7) << 4, ohi = ((2 * c + 1) ^ r7) << 4;
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      *reinterpret_cast<uint4*>(dst + k * ROW_STEP * 128 + olo) = unpack_lo(v[k]);
      *reinterpret_cast<uint4*>(dst + k * ROW_STEP * 128 + ohi) = unpack_hi(v[k]);
    }
  } else {
    const uint8_t* src = stage + r0 * 128 + c * 16;
    const uint32_t o0 = (c ^ r7) << 4, o1 = ((c + 4) ^ r7) << 4;
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      const uint4 a = *reinterpret_cast<const uint4*>(src + k * ROW_STEP * 128);
      const uint4 b = *reinterpret_cast<const uint4*>(src + k * ROW_STEP * 128 + 64);
      *reinterpret_cast<uint4*>(dst + k * ROW_STEP * 128 + o0) = a;
      *reinterpret_cast<uint4*>(dst + k * ROW_STEP * 128 + o1) = b;
    }
  }
}

// Weight stages: 128-byte packed rows = two consecutive INT4 groups of the same work item (or a
// single one at an item / INT4-region boundary), or the INT8 outlier group.  Producer and unpack
// warps walk an item's groups in these stage units.
__device__ __forceinline__ int stage_groups(int t, int t1, int G4) {
  return (t < G4 && t + 1 < t1 && t + 1 < G4) ? 2 : 1;
}

// ---- schedule ("data-parallel waves + stream-K tail"): the first dp_waves * gridDim.x tiles are
//      whole tiles dealt round-robin (CTA i takes tiles i, i + grid, ...: neighbouring CTAs
//      share a weight tile at the same time, so it is read from HBM once); the remaining tiles'
//      (tile, group) units are divided evenly, CTA i owning [sk_start(i), sk_start(i+1)).  A tile
//      cut by those boundaries is computed in K segments by consecutive CTAs.  Each CTA first
//      works on its highest stream-K tile (a tile head it publishes, or a whole tile), then its
//      data-parallel tiles, then its remaining stream-K tiles in descending order (the last one
//      may be a tile tail it reduces), so reducers find the published segments ready. ----
__device__ __forceinline__ int64_t sk_start(const GemmParams& p, int64_t i) {
  return p.sk_base + i * p.sk_units / gridDim.x;
}
// CTA whose stream-K range contains unit u (u >= sk_base).
__device__ __forceinline__ int cta_of(const GemmParams& p, int64_t u) {
  int64_t i = ((u - p.sk_base) * gridDim.x) / p.sk_units;
  while (i + 1 < gridDim.x && sk_start(p, i + 1) <= u) ++i;
  while (i > 0 && sk_start(p, i) > u) --i;
  return static_cast<int>(i);
}

struct Sched {
  int64_t u0, u1;   // this CTA's stream-K units
  int t_hi;         // highest stream-K tile touched
  int ns, nd;       // number of stream-K items / data-parallel tiles
  __device__ __forceinline__ int count() const { return ns + nd; }
};
__device__ __forceinline__ Sched make_sched(const GemmParams& p) {
  Sched s;
  s.u0 = sk_start(p, blockIdx.x);
  s.u1 = sk_start(p, blockIdx.x + 1);
  s.nd = p.dp_waves;
  if (s.u1 > s.u0) {
    s.t_hi = static_cast<int>((s.u1 - 1) / p.G);
    s.ns = s.t_hi - static_cast<int>(s.u0 / p.G) + 1;
  } else {
    s.t_hi = 0;
    s.ns = 0;
  }
  return s;
}

struct Item {
  int n0, m0, t0, t1, tile;
};
template <int BT>
__device__ __forceinline__ Item get_item(const GemmParams& p, const Sched& s, int k) {
  Item it;
  int tile;
  bool sk = true;
  if (s.ns > 0 && k == 0) {
    tile = s.t_hi;
  } else {
    const int kk = k - (s.ns > 0 ? 1 : 0);
    if (kk < s.nd) {
      tile = static_cast<int>(blockIdx.x) + kk * static_cast<int>(gridDim.x);
      sk = false;
    } else {
      tile = s.t_hi - (kk - s.nd + 1);
    }
  }
  it.tile = tile;
  if (sk) {
    const int64_t base = static_cast<int64_t>(tile) * p.G;
    it.t0 = static_cast<int>((s.u0 > base ? s.u0 : base) - base);
    it.t1 = static_cast<int>((s.u1 < base + p.G ? s.u1 : base + p.G) - base);
  } else {
    it.t0 = 0;
    it.t1 = p.G;
  }
  it.n0 = (tile / p.m_tiles) * kTileN;
  it.m0 = (tile % p.m_tiles) * BT;
  return it;
}

// Walks this CTA's (item, group) sequence one group at a time.
template <int BT>
struct GroupCursor {
  int k, t, t1, m0, tile;
  __device__ __forceinline__ bool valid(const Sched& s) const { return k < s.count(); }
  __device__ __forceinline__ void load(const GemmParams& p, const Sched& s) {
    if (k < s.count()) {
      const Item w = get_item<BT>(p, s, k);
      t = w.t0;
      t1 = w.t1;
      m0 = w.m0;
      tile = w.tile;
    }
  }
  __device__ __forceinline__ void next(const GemmParams& p, const Sched& s) {
    if (++t >= t1) {
      ++k;
      load(p, s);
    }
  }
};

// ring position: slot index + phase parity, advanced one step at a time (no division)
template <int N>
struct Ring {
  uint32_t i = 0, ph = 0;
  __device__ __forceinline__ void next() {
    if (++i == N) {
      i = 0;
      ph ^= 1;
    }
  }
};

// kMode (development timing probes, never used for results): bit 0 = the epilogue skips its
// arithmetic; bit 1 = it skips the TMEM loads; bit 2 = magic re-arm of even buffers by tcgen05.st
// instead of the LOP3 conversion; bit 3 = no output stores; bit 4 = no activation TMA (arrive only); bit 5 = no
// weight TMA; bit 6 = unpack skips its data movement.
template <int BT, bool kDebug, int kMode = 0>
__global__ void __launch_bounds__(kThreads, 1)
w4a4_gemm_kernel(const __grid_constant__ CUtensorMap tm_wq4,
                 const __grid_constant__ CUtensorMap tm_wq8,
                 const __grid_constant__ CUtensorMap tm_ax8, const GemmParams p) {
  static_assert(BT % 32 == 0 && BT >= 32 && BT <= 256, "token tile");
  using C = Cfg<BT>;
  constexpr int RS = C::RS, RW = C::RW, RT = C::RT, NJ = C::NJ, NC = C::NC, KS = C::kStages;
  constexpr uint32_t kTmemCols = C::kTmemCols;
  extern __shared__ uint8_t smem_raw[];
  GemmSmem<BT>& sm = *reinterpret_cast<GemmSmem<BT>*>(
      smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (p.trace != nullptr && threadIdx.x == 0)
    p.trace[8 * kTraceN + blockIdx.x * 4 + 0] = globaltimer_ns();
  // waits on the MMA <-> epilogue critical loop: spin (bit 7 of kMode: suspend-hinted instead)
  auto wait_hot = [](uint64_t* bar, uint32_t parity) {
    if constexpr ((kMode & 128) != 0) mbar_wait(bar, parity);
    else if constexpr ((kMode & 4096) != 0) mbar_wait_spin(bar, parity);
    else mbar_wait_test(bar, parity);
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < KS; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kNumUnpackWarps);
    }
    for (int u = 0; u < RS; ++u) {
      // unpack warps, activation tile, epilogue release, group scales (32 cp.async lanes)
      mbar_init(&sm.go[u], kNumUnpackWarps + 1 + kNumEpiWarps + 32);   // unpack, A tile, epilogue
      mbar_init(&sm.mdone[u], 1);
    }
    for (int r = 0; r < RS; ++r) mbar_init(&sm.sfree[r], kNumEpiWarps);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_wq4);
    tma_prefetch_desc(&tm_wq8);
    tma_prefetch_desc(&tm_ax8);
  }
  if (warp == 1) tmem_alloc(&sm.tmem_base, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  const int G4 = p.G4;
  const Sched sch = make_sched(p);
  const int n_items = sch.count();

  if (threadIdx.x == 0) griddep_launch();   // the next kernel still waits for this grid's end
  if (warp < kEpiWarp0) setmaxnreg_dec<kRegsLow>();
  if (warp == 0) {
    // ===================== producer warp: packed weights (TMA) =====================
    // Not tied to the operand or scale slots, so the weight stream runs up to KS stages ahead
    // of the unpack warps.
    if (lane == 0) {
      Ring<KS> st;
      int gp = 0;
      const uint64_t pol_w = l2_policy_evict_first();
      if (n_items > 0) {   // PDL: warm L2 with the first weight stages while the previous kernel ends
        const Item w = get_item<BT>(p, sch, 0);
        for (int t = w.t0, s = 0; t < w.t1 && s < KS; t += stage_groups(t, w.t1, G4), ++s) {
          if (t < G4) tma_prefetch_2d(&tm_wq4, t * 64, w.n0);
          else tma_prefetch_2d(&tm_wq8, 0, w.n0);
        }
      }
      griddep_wait();
      for (int k = 0; k < n_items; ++k) {
        const Item w = get_item<BT>(p, sch, k);
        for (int t = w.t0; t < w.t1; st.next()) {
          const int n = stage_groups(t, w.t1, G4);
          mbar_wait(&sm.empty[st.i], st.ph ^ 1);
          TRACE(0, gp);
          if constexpr ((kMode & 32) != 0) {
            mbar_arrive(&sm.full[st.i]);
          } else {
            mbar_arrive_expect_tx(&sm.full[st.i], kTileN * 128);
            // weights: read by the 4 CTAs sharing the n-tile at about the same time, then dead.
            // A single INT4 group at the end of the INT4 region reads 64 bytes past the row
            // (zero-filled by TMA, unused).
            if (t < G4)
              tma_load_2d_hint(sm.stage_w[st.i], &tm_wq4, &sm.full[st.i], t * 64, w.n0, pol_w);
            else
              tma_load_2d_hint(sm.stage_w[st.i], &tm_wq8, &sm.full[st.i], 0, w.n0, pol_w);
          }
          t += n;
          gp += n;
        }
      }
    }
  } else if (warp == kScaleWarp) {
    // ===================== scale loader warp: group scales (cp.async) =====================
    // The scales complete group g's go barrier: the MMA (and hence the epilogue, which waits
    // for the MMA) never sees a group before its scales landed.  Slot g % RS is reused once
    // the epilogue is done with group g - RS.
    Ring<RS> sr;
    int gp = 0;
    griddep_wait();                      // scales may come from the previous kernel (quantize)
    for (int k = 0; k < n_items; ++k) {
      const Item w = get_item<BT>(p, sch, k);
      for (int t = w.t0; t < w.t1; ++t, sr.next(), ++gp) {
        mbar_wait(&sm.sfree[sr.i], sr.ph ^ 1);
        const float* ws = p.w_scales + static_cast<int64_t>(t) * p.N + w.n0;
        const float* as = p.a_scales + static_cast<int64_t>(t) * p.M;
#pragma unroll
        for (int j = lane; j < kTileN; j += 32) cp_async_4(&sm.ssw[sr.i][j], ws + j);
#pragma unroll
        for (int j = lane; j < BT; j += 32)
          // rows past M: any finite scale works, their partials are exactly zero (TMA
          // zero-fills out-of-range activation rows) and they are never stored
          cp_async_4(&sm.ssa[sr.i][j], as + min(w.m0 + j, p.M - 1));
        cp_async_mbar_arrive(&sm.go[sr.i]);
      }
    }
  } else if (warp == kALoaderWarp) {
    // ===================== activation-tile loader (single thread) =====================
    // Slot u is free exactly when the MMAs of the group that used it complete; the tile of
    // group g (x8, TMA, SWIZZLE_128B straight into the operand slot) is issued right then.
    if (lane == 0) {
      Ring<RS> u;
      const uint64_t pol_a = l2_policy_evict_last();
      griddep_wait();                    // the activation tiles come from the previous kernel
      int ga = 0;
      for (int k = 0; k < n_items; ++k) {
        const Item w = get_item<BT>(p, sch, k);
        for (int t = w.t0; t < w.t1; ++t, u.next(), ++ga) {
          wait_hot(&sm.mdone[u.i], u.ph ^ 1);
          if constexpr ((kMode & 16) != 0) {
            mbar_arrive(&sm.go[u.i]);
          } else {
            mbar_arrive_expect_tx(&sm.go[u.i], BT * 128);
            // activations: re-read by every n-tile, keep them in L2
            TRACE(1, ga);
            tma_load_2d_hint(sm.ubuf_a[u.i], &tm_ax8, &sm.go[u.i], t * 128, w.m0, pol_a);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (single thread) =====================
    // Every instruction this thread executes between dispatches idles the tensor pipe for as
    // long (measured, tools/mma_rate.cu: tcgen05.mma issue returns only as the previous dispatch
    // drains), so the loop is one barrier probe, 4 dispatches and one commit per group.
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_i8(kTileN, BT);
      int total = 0;
      for (int k = 0; k < n_items; ++k) {
        const Item w = get_item<BT>(p, sch, k);
        total += w.t1 - w.t0;
      }
      const uint64_t da0 = umma_desc_sw128(smem_u32(sm.ubuf_w[0]));
      const uint64_t db0 = umma_desc_sw128(smem_u32(sm.ubuf_a[0]));
      Ring<RS> u;
      Ring<RW> uw;
      Ring<RT> b;
      for (int gm = 0; gm < total; ++gm) {
        wait_hot(&sm.go[u.i], u.ph);
        tc_fence_after();
        TRACE(3, gm);
        const uint32_t d = tmem + b.i * BT;
        // descriptor start address field counts 16-byte units: slot u, K step kk (32 bytes)
        const uint64_t da = da0 + uw.i * (kTileN * 128 / 16);
        const uint64_t db = db0 + u.i * (BT * 128 / 16);
        const uint32_t acc0 = ((kMode & 4) != 0 && (b.i & 1u) == 0) ? 1u : 0u;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          // even buffers hold the magic 1.5*2^23 (re-armed by the epilogue): always accumulate;
          // odd buffers start from zero and the epilogue converts with one LOP3
          umma_i8(d, da + 2 * kk, db + 2 * kk, idesc, kk > 0 ? 1u : acc0);
        umma_commit(&sm.mdone[u.i]);
        if constexpr ((kMode & 256) != 0)   // probe: MMA latency (issue -> completion)
          mbar_wait_spin(&sm.mdone[u.i], u.ph);
        u.next();
        uw.next();
        b.next();
      }
    }
  } else if (warp >= kUnpackWarp0 && warp < kEpiWarp0) {
    // ===================== unpack warps: packed INT4 weights -> int8 (16*q), SW128 ============
    // 128 threads: thread ut owns packed chunk (ut & 3) of rows (ut >> 2) + 32k, k < 4.
    const int ut = threadIdx.x - kUnpackWarp0 * 32;
    const uint32_t r0 = static_cast<uint32_t>(ut) >> 2, c = static_cast<uint32_t>(ut) & 3u;
    Ring<KS> st;
    Ring<RS> u;                          // go slot of group g
    Ring<RS> lag;                        // mdone slot of group g - RW
    Ring<RW> uw;                         // unpacked-weight slot of group g
    int gu = 0;
#ifndef ATOM_UNPACK_PAIRS
#define ATOM_UNPACK_PAIRS 1
#endif
    // With 4 unpacked-weight slots (BT <= 128) a whole stage (two INT4 groups) is expanded in
    // one pass: twice the loads in flight and one fence / warp sync for both groups.
    if constexpr (RW >= 4 && ATOM_UNPACK_PAIRS != 0) {
      for (int k = 0; k < n_items; ++k) {
        const Item w = get_item<BT>(p, sch, k);
        for (int t = w.t0; t < w.t1;) {
          const int n = stage_groups(t, w.t1, G4);
          for (int i = 0; i < n; ++i)
            if (gu + i >= RW) {          // MMAs of group g + i - RW finished with its slot
              wait_hot(&sm.mdone[lag.i], lag.ph);
              lag.next();
            }
          wait_hot(&sm.full[st.i], st.ph);
          if (ut == 0) TRACE(2, gu);
          const bool int4 = t < G4;
          Ring<RW> uw1 = uw;
          uw1.next();
          if constexpr ((kMode & 64) == 0) {
            unpack_rows<4, 32>(sm.stage_w[st.i], sm.ubuf_w[uw.i], r0, c, int4, 0);
            if (n == 2) unpack_rows<4, 32>(sm.stage_w[st.i], sm.ubuf_w[uw1.i], r0, c, int4, 1);
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.empty[st.i]);
          st.next();
          if constexpr ((kMode & 512) == 0) fence_proxy_async_smem();
          __syncwarp();
          if (ut == 0) TRACE(4, gu);
          if (lane == 0) {
            mbar_arrive(&sm.go[u.i]);
            if (n == 2) {
              Ring<RS> u1 = u;
              u1.next();
              mbar_arrive(&sm.go[u1.i]);
            }
          }
          for (int i = 0; i < n; ++i) {
            u.next();
            uw.next();
          }
          gu += n;
          t += n;
        }
      }
    } else
    for (int k = 0; k < n_items; ++k) {
      const Item w = get_item<BT>(p, sch, k);
      int sub = 0, n = 0;                // position inside the current weight stage
      for (int t = w.t0; t < w.t1; ++t, u.next(), uw.next(), ++gu) {
        if (gu >= RW) {                  // MMAs of group g - RW finished with this weight slot
          wait_hot(&sm.mdone[lag.i], lag.ph);
          lag.next();
        }
        const bool int4 = t < G4;
        if (sub == 0) {                  // first group of a stage: wait for its TMA
          n = stage_groups(t, w.t1, G4);
          wait_hot(&sm.full[st.i], st.ph);
          if (ut == 0) TRACE(2, gu);
        }
        if constexpr ((kMode & 64) == 0)
          unpack_rows<4, 32>(sm.stage_w[st.i], sm.ubuf_w[uw.i], r0, c, int4, sub);
        if (++sub == n) {                // stage consumed
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.empty[st.i]);
          st.next();
          sub = 0;
        }
        if constexpr ((kMode & 512) == 0) fence_proxy_async_smem();
        __syncwarp();
        if (ut == 0) TRACE(4, gu);
        if (lane == 0) mbar_arrive(&sm.go[u.i]);
      }
    }
  } else if (warp >= kEpiWarp0) {
    // ===================== epilogue warps =====================
    // TMEM is read with the 32x32b shape: thread = TMEM lane = output channel n (its weight
    // scale is one scalar per group), consecutive registers = consecutive tokens of this warp's
    // column third.  Per column: dequantize T = float(1.5*2^23 + R) with one FFMA,
    // g = T*sw' - 1.5*2^23*sw' = sw'*R, and accumulate acc += s_a*g with one more (FFMA2 on
    // column pairs; s_a of 4 columns per broadcast 16-byte shared load).  The FP32 pipe is the
    // binding resource of the whole kernel (2 FMAs per output per group).
    setmaxnreg_inc<kRegsHigh>();
    const int e = warp - kEpiWarp0;
    const int q = warp & 3;              // TMEM lane quarter this warp may access
    const int third = e >> 2;            // column part (kEpiPerQuarter parts)
    constexpr int kBase = NC / kEpiPerQuarter, kRem = NC % kEpiPerQuarter;
    constexpr int NCOL = NJ * 8;         // columns of the widest third
    const int ncol = 8 * (kBase + (third < kRem ? 1 : 0));             // this warp (uniform)
    const int col0 = 8 * (third * kBase + (third < kRem ? third : kRem));
    const uint32_t tq = tmem + (static_cast<uint32_t>(q * 32) << 16) + col0;
    const uint32_t magic = kMagicBits;
    uint32_t one = 1u;
    asm volatile("" : "+r"(one));        // opaque to ptxas (see biased_fma)
    const bool a_issuer = e == 0 && lane == 0;
    const int n_local = q * 32 + lane;   // output channel within the tile
    uint32_t mg[8];                      // resident tcgen05.st sources for the magic re-arm
#pragma unroll
    for (int i = 0; i < 8; ++i) mg[i] = magic;
    asm volatile("" : "+r"(mg[0]), "+r"(mg[1]), "+r"(mg[2]), "+r"(mg[3]), "+r"(mg[4]),
                 "+r"(mg[5]), "+r"(mg[6]), "+r"(mg[7]));
    auto rearm = [&](uint32_t taddr) {   // this warp's columns of one buffer := 1.5*2^23
#pragma unroll
      for (int j = 0; j < NCOL; j += 8)
        if (j + 8 <= ncol) tmem_st8(taddr + j, mg);
      tmem_st_wait();
    };
    if constexpr ((kMode & 4) != 0) {
#pragma unroll
      for (int b = 0; b < RT; b += 2) rearm(tq + b * BT);
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0)   // the first RT groups find their TMEM buffers free
      for (int b = 0; b < RT; ++b) mbar_arrive(&sm.go[b % RS]);
    uint8_t* stg = sm.ostg[e];           // per-warp staging for the transposed output
    Ring<RS> u;
    Ring<RT> b;
    Ring<RS> sr;
    int ge = 0;
    for (int k = 0; k < n_items; ++k) {
      const Item w = get_item<BT>(p, sch, k);
      const int n0 = w.n0;
      const int mc0 = w.m0 + col0;       // first token of this warp's columns
      float acc[NCOL];
#pragma unroll
      for (int j = 0; j < NCOL; ++j) acc[j] = 0.0f;
      for (int t = w.t0; t < w.t1; ++t, u.next(), b.next(), sr.next(), ++ge) {
        const bool int4 = t < G4;
        if (a_issuer) TRACE(5, ge);
        wait_hot(&sm.mdone[u.i], u.ph);      // also implies the group's scales have landed
        if (a_issuer) TRACE(6, ge);
        if (p.trace != nullptr && a_issuer && ge == 0)
          p.trace[8 * kTraceN + blockIdx.x * 4 + 1] = globaltimer_ns();
        // sw' = sw (x1/16 for INT4 groups, exact) with its 2 lowest mantissa bits cleared so
        // that 1.5*2^23*sw' is exact; see DESIGN.md "Epilogue arithmetic".
        float sw = sm.ssw[sr.i][n_local];
        if (int4) sw *= (1.0f / 16.0f);
        const float swh = __uint_as_float(__float_as_uint(sw) & 0xFFFFFFFCu);
        const float2 sw2 = make_float2(swh, swh);
        const float2 nc2 = make_float2(-kMagic * swh, -kMagic * swh);
        const float* sa = &sm.ssa[sr.i][col0];
        tc_fence_after();
        const uint32_t taddr = tq + b.i * BT;
        const uint32_t go_next = u.i + RT >= RS ? u.i + RT - RS : u.i + RT;   // slot of g + RT
        const bool pre = (kMode & 4) != 0 && (b.i & 1u) == 0;
        auto drain = [&](auto pre_tag) {
          constexpr bool kPre = decltype(pre_tag)::value;
          // 16-column batches, software-pipelined one batch ahead: the load of batch i+1 is in
          // flight while batch i is computed (the LDTM destination registers are scoreboarded;
          // tcgen05.wait::ld, which waits for ALL loads, is only issued before the buffer is
          // released, once the last batch has been requested)
          constexpr int NB = (NCOL + 15) / 16;
          uint32_t r[2][16];
          auto load = [&](int bi, uint32_t* dst) {
            const int j = bi * 16;
            if constexpr ((kMode & 2) == 0) {
              if (j + 16 <= ncol) tmem_ld16p(taddr + j, dst);
              else if (j + 8 <= ncol) tmem_ld8(taddr + j, dst);
            } else {
#pragma unroll
              for (int v = 0; v < 16; ++v) dst[v] = taddr + v;
            }
          };
          load(0, r[0]);
#pragma unroll
          for (int bi = 0; bi < NB; ++bi) {
            if (bi + 1 < NB) {
              load(bi + 1, r[(bi + 1) & 1]);
            } else {                                  // all loads issued: release the buffer
              tmem_ld_wait();
              if constexpr (kPre) rearm(taddr);
              tc_fence_before();
              __syncwarp();
              if (a_issuer) TRACE(7, ge);
              if (lane == 0) mbar_arrive(&sm.go[go_next]);   // buffer b free for g + RT
            }
#pragma unroll
            for (int jj = 0; jj < 16; jj += 4) {
              const int j = bi * 16 + jj;
              if (j < NCOL && j < ncol) {
                uint32_t* rv = r[bi & 1] + jj;
#ifndef ATOM_I2F_MASK
#define ATOM_I2F_MASK 0xFF   // all column quads (A/B of the mixes: profiles/r01/NOTES.md)
#endif
                // int32 -> float by I2FP (measured faster than the LOP3 / VIADD magic-number
                // conversions, alone or mixed, once the epilogue is dequant-bound); the I2FP
                // columns dequantize as g = RN(sw' * float(R)) -- the same single rounding as
                // the magic path's fused multiply-add, so either form gives identical bits.
                // The debug-partials kernel keeps the magic path (it reads R back from it).
                const bool i2f = !kDebug && kMode == 0 && !kPre &&
                                 ((ATOM_I2F_MASK >> ((bi & 1) * 4 + jj / 4)) & 1) != 0;
                if constexpr (!kPre) {
#pragma unroll
                  for (int v = 0; v < 4; ++v)
                    rv[v] = i2f ? __float_as_uint(__int2float_rn(static_cast<int>(rv[v])))
                                : __float_as_uint(((kMode & 8192) == 0 && (jj & 4) != 0)
                                                      ? biased_fma(rv[v], one, magic)
                                                      : biased(rv[v], magic));
                }
                if constexpr (kDebug) {
#pragma unroll
                  for (int v = 0; v < 4; ++v) {
                    const int m = mc0 + j + v;
                    const int raw = static_cast<int>(rv[v] - kMagicBits);
                    if (m < p.M)
                      p.debug[(static_cast<int64_t>(t) * p.M + m) * p.N + n0 + n_local] =
                          int4 ? (raw >> 4) : raw;
                  }
                }
                const float4 s4 = *reinterpret_cast<const float4*>(sa + j);
                if constexpr ((kMode & 1) != 0) {
                  acc[j] += __uint_as_float(rv[0] ^ rv[3]);
                  continue;
                }
                const float2 ncq = i2f ? make_float2(0.0f, 0.0f) : nc2;
                const float2 g0 = __ffma2_rn(
                    make_float2(__uint_as_float(rv[0]), __uint_as_float(rv[1])), sw2, ncq);
                const float2 g1 = __ffma2_rn(
                    make_float2(__uint_as_float(rv[2]), __uint_as_float(rv[3])), sw2, ncq);
                const float2 a0 = __ffma2_rn(make_float2(s4.x, s4.y), g0,
                                             make_float2(acc[j], acc[j + 1]));
                const float2 a1 = __ffma2_rn(make_float2(s4.z, s4.w), g1,
                                             make_float2(acc[j + 2], acc[j + 3]));
                acc[j] = a0.x;
                acc[j + 1] = a0.y;
                acc[j + 2] = a1.x;
                acc[j + 3] = a1.y;
              }
            }
          }
        };
        if (pre) drain(std::true_type{});
        else drain(std::false_type{});
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.sfree[sr.i]);
      }

      // ---- split tile: every segment but the tile's last publishes its fp32 partial; the CTA
      //      holding the last segment adds the others (in CTA order, deterministic) ----
      if (w.t1 < p.G || w.t0 > 0) {
        // thread-linear float4 fragments: warp e, column quad i, lane -> one 512-byte row
        auto frag = [&](float* slot, int i) {
          return reinterpret_cast<float4*>(slot) + (e * (NCOL / 4) + i) * 32 + lane;
        };
        if (w.t1 < p.G) {                    // publisher (this CTA's first item)
          float* slot = p.partials + static_cast<int64_t>(blockIdx.x) * C::kSlotFloats;
#pragma unroll
          for (int i = 0; i < NCOL / 4; ++i)
            if (4 * i < ncol)
              __stcg(frag(slot, i), make_float4(acc[4 * i], acc[4 * i + 1], acc[4 * i + 2],
                                                acc[4 * i + 3]));
          __threadfence();
          named_bar_sync(1, kEpiThreads);
          if (e == 0 && lane == 0)
            red_release_add(p.counters + cta_of(p, static_cast<int64_t>(w.tile + 1) * p.G - 1), 1);
          continue;
        }
        // reducer (this CTA's last item): the other segments belong to CTAs first..blockIdx-1
        const int first = cta_of(p, static_cast<int64_t>(w.tile) * p.G);
        const int nseg = static_cast<int>(blockIdx.x) - first;
        if (e == 0 && lane == 0) {
          while (ld_acquire(p.counters + blockIdx.x) < nseg) __nanosleep(64);
          p.counters[blockIdx.x] = 0;        // self-cleaning for the next launch
        }
        named_bar_sync(1, kEpiThreads);
        for (int i0 = first; i0 < static_cast<int>(blockIdx.x); ++i0) {
          float* slot = p.partials + static_cast<int64_t>(i0) * C::kSlotFloats;
#pragma unroll
          for (int i = 0; i < NCOL / 4; ++i)
            if (4 * i < ncol) {
              const float4 o = __ldcg(frag(slot, i));
              acc[4 * i] += o.x;
              acc[4 * i + 1] += o.y;
              acc[4 * i + 2] += o.z;
              acc[4 * i + 3] += o.w;
            }
        }
      }
      if constexpr ((kMode & 8) != 0) {
        if (acc[0] == 1.2345f) p.debug[0] = 1;   // keep acc alive
        continue;
      }

      // ---- tile output: 8 tokens at a time, this lane's channel is written into a per-warp
      //      [8 tokens][32 channels] staging (conflict-free rows), then each lane stores 16
      //      contiguous bytes of one token row of C ----
      const int om = lane >> 2, op = lane & 3;           // readback: token row, channel piece
#pragma unroll
      for (int j = 0; j < NCOL; j += 8) {
        if (j >= ncol) continue;
        const int m = mc0 + j + om;
        if (!p.c_f32) {
          __half* s16 = reinterpret_cast<__half*>(stg);
#pragma unroll
          for (int v = 0; v < 8; ++v) s16[v * 32 + lane] = __float2half_rn(acc[j + v]);
          __syncwarp();
          const uint4 val = *reinterpret_cast<const uint4*>(s16 + om * 32 + op * 8);
          __syncwarp();
          if (m < p.M)
            *reinterpret_cast<uint4*>(static_cast<__half*>(p.c) + static_cast<int64_t>(m) * p.ldc +
                                      n0 + q * 32 + op * 8) = val;
        } else {
          float* s32 = reinterpret_cast<float*>(stg);
#pragma unroll
          for (int v = 0; v < 8; ++v) s32[v * 32 + lane] = acc[j + v];
          __syncwarp();
          const float4 v0 = *reinterpret_cast<const float4*>(s32 + om * 32 + op * 8);
          const float4 v1 = *reinterpret_cast<const float4*>(s32 + om * 32 + op * 8 + 4);
          __syncwarp();
          if (m < p.M) {
            float4* dst = reinterpret_cast<float4*>(static_cast<float*>(p.c) +
                                                    static_cast<int64_t>(m) * p.ldc + n0 +
                                                    q * 32 + op * 8);
            dst[0] = v0;
            dst[1] = v1;
          }
        }
      }
    }
  }

  if (p.trace != nullptr && threadIdx.x == kEpiWarp0 * 32)
    p.trace[8 * kTraceN + blockIdx.x * 4 + 2] = globaltimer_ns();
  tc_fence_before();
  __syncthreads();
  if (p.trace != nullptr && threadIdx.x == 0)
    p.trace[8 * kTraceN + blockIdx.x * 4 + 3] = globaltimer_ns();
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

// 2D uint8 tensor [rows][cols] (row stride = cols bytes), box [box_rows][box_cols bytes].
static bool make_map_u8(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows,
                        uint32_t box_cols, uint32_t box_rows, CUtensorMapSwizzle swz) {
  PFN_encodeTiled enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BT>
static size_t slot_bytes() {
  return Cfg<BT>::kSlotFloats * sizeof(float);
}
static size_t slot_bytes_for(int bt) {
  switch (bt) {
    case 256: return slot_bytes<256>();
    case 128: return slot_bytes<128>();
    case 64: return slot_bytes<64>();
    default: return slot_bytes<32>();
  }
}

template <int BT>
static cudaError_t launch_bt(const GemmArgs& a, const GemmPlan& plan, void* workspace,
                             cudaStream_t stream, int* launches) {
  const int M = static_cast<int>(a.M), N = static_cast<int>(a.N), K = static_cast<int>(a.K);
  const int k_o = a.k_outlier;
  const uint64_t kp = static_cast<uint64_t>(K - k_o) / 2;
  CUtensorMap m_wq4, m_wq8, m_ax8;
  // A map is always encoded (a valid descriptor is required as a kernel parameter); an unused
  // INT4 or INT8 weight map aliases the other one and is never read.
  const void* w4 = kp ? static_cast<const void*>(a.w_q4) : static_cast<const void*>(a.w_q8);
  const void* w8 = k_o ? static_cast<const void*>(a.w_q8) : static_cast<const void*>(a.w_q4);
  const uint64_t c4 = kp ? kp : 128, c8 = k_o ? 128 : kp;
  if (!make_map_u8(&m_wq4, w4, c4, N, 128, kTileN, CU_TENSOR_MAP_SWIZZLE_NONE) ||
      !make_map_u8(&m_wq8, w8, c8, N, 128, kTileN, CU_TENSOR_MAP_SWIZZLE_NONE) ||
      !make_map_u8(&m_ax8, a.a_x8, K, M, 128, BT, CU_TENSOR_MAP_SWIZZLE_128B))
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
  p.c_f32 = a.c_f32;
  p.m_tiles = (M + BT - 1) / BT;
  p.num_tiles = p.m_tiles * (N / kTileN);
  p.dp_waves = plan.dp_waves;
  p.sk_base = static_cast<int64_t>(plan.dp_waves) * plan.grid * p.G;
  p.sk_units = plan.sk_units;
  p.counters = nullptr;
  p.partials = nullptr;
  p.trace = nullptr;
  if (plan.workspace_bytes > 0) {
    p.counters = static_cast<int*>(workspace);
    p.partials = reinterpret_cast<float*>(static_cast<char*>(workspace) + plan.counter_bytes);
  }

  const size_t smem = sizeof(GemmSmem<BT>) + 1024;
  auto kern = p.debug ? w4a4_gemm_kernel<BT, true> : w4a4_gemm_kernel<BT, false>;
#ifdef ATOM_DEV_PROBES
  // development timing probes (results WRONG by design): only in builds made with
  // ATOM_NVCC_EXTRA=-DATOM_DEV_PROBES, never in the shipped library
  if constexpr (BT == 256 || BT == 128) {
    static const char* mode_env = getenv("ATOM_GEMM_PROBE_MODE");
    switch (mode_env ? atoi(mode_env) : 0) {
      case 1: kern = w4a4_gemm_kernel<BT, false, 1>; break;
      case 2: kern = w4a4_gemm_kernel<BT, false, 2>; break;
      case 3: kern = w4a4_gemm_kernel<BT, false, 3>; break;
      case 4: kern = w4a4_gemm_kernel<BT, false, 4>; break;
      case 8: kern = w4a4_gemm_kernel<BT, false, 8>; break;
      case 16: kern = w4a4_gemm_kernel<BT, false, 16>; break;
      case 32: kern = w4a4_gemm_kernel<BT, false, 32>; break;
      case 64: kern = w4a4_gemm_kernel<BT, false, 64>; break;
      case 115: kern = w4a4_gemm_kernel<BT, false, 115>; break;
      case 512: kern = w4a4_gemm_kernel<BT, false, 512>; break;
      case 1024: kern = w4a4_gemm_kernel<BT, false, 1024>; break;
      case 8192: kern = w4a4_gemm_kernel<BT, false, 8192>; break;
      default: break;
    }
  }
#endif
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  static long long* trace = nullptr;
  static const bool want_trace = getenv("ATOM_GEMM_TRACE") != nullptr;   // development only
  constexpr size_t kTraceBytes = (8 * kTraceN + 4 * 1024) * sizeof(long long);
  if (want_trace && trace == nullptr) cudaMalloc(&trace, kTraceBytes);
  p.trace = want_trace ? trace : nullptr;
  if (want_trace) cudaMemsetAsync(trace, 0, kTraceBytes, stream);
  e = launch_pdl(kern, dim3(plan.grid), dim3(kThreads), smem, stream, m_wq4, m_wq8, m_ax8, p);
  if (e != cudaSuccess) return e;
  ++*launches;
  if (want_trace) {
    static long long h[8 * kTraceN + 4 * 1024];
    cudaMemcpy(h, trace, sizeof(h), cudaMemcpyDeviceToHost);
    fprintf(stderr, "plan: BT=%d grid=%d dp_waves=%d sk_units=%lld tiles=%d\n", BT, plan.grid,
            plan.dp_waves, static_cast<long long>(plan.sk_units), p.num_tiles);
    fprintf(stderr, "g   W_tma  A_issue W_landed mma_issue unp_done epi_top epi_mdone epi_release\n");
    const long long t0 = h[0];
    for (int g = 0; g < kTraceN && (g < 40 || g % 25 == 0); ++g) {
      if (h[3 * kTraceN + g] == 0) break;
      fprintf(stderr, "%3d %8lld %8lld %8lld %8lld %8lld %8lld %8lld %8lld\n", g, h[g] - t0,
              h[kTraceN + g] - t0, h[2 * kTraceN + g] - t0, h[3 * kTraceN + g] - t0,
              h[4 * kTraceN + g] - t0, h[5 * kTraceN + g] - t0, h[6 * kTraceN + g] - t0,
              h[7 * kTraceN + g] - t0);
    }
    long long c0 = h[8 * kTraceN];
    for (int b = 0; b < plan.grid; ++b) c0 = h[8 * kTraceN + 4 * b] < c0 ? h[8 * kTraceN + 4 * b] : c0;
    fprintf(stderr, "cta: start first_mdone epi_done end (ns rel. to first start)\n");
    for (int b = 0; b < plan.grid; ++b) {
      const long long* q = h + 8 * kTraceN + 4 * b;
      fprintf(stderr, "%3d %7lld %7lld %7lld %7lld\n", b, q[0] - c0, q[1] - c0, q[2] - c0,
              q[3] - c0);
    }
  }
  return cudaGetLastError();
}

// Tile plan.  Every plan runs one persistent CTA per SM (or per unit, if fewer): whole tiles in
// round-robin waves while at least two waves remain, then the rest as evenly divided
// (tile, group) units (stream-K).  The only choice is the token tile BT: the largest power of
// two <= 256 that does not exceed the padded M, traded (by a simple clock-count model) against
// the cost of reducing split tiles when there are few units per CTA.
GemmPlan plan_w4a4_gemm(int64_t M, int64_t N, int64_t K, int num_sms) {
  GemmPlan best;
  const int64_t n_tiles = N / kTileN;
  const int64_t G = K / 128;
  int bt_max = 32;
  static const char* btm = getenv("ATOM_GEMM_BT_MAX");   // development override
  const int bt_cap = btm ? atoi(btm) : 256;
  while (bt_max < bt_cap && bt_max < M) bt_max *= 2;
  double best_cost = 1e300;
  for (int bt = bt_max; bt >= 32; bt /= 2) {
    GemmPlan pl;
    pl.bt = bt;
    pl.num_tiles = n_tiles * ((M + bt - 1) / bt);
    const int64_t units = pl.num_tiles * G;
    pl.grid = static_cast<int>(units < num_sms ? units : num_sms);
    const int64_t T = pl.num_tiles, P = pl.grid;
    if (T % P == 0) pl.dp_waves = static_cast<int>(T / P);
    else if (T >= 2 * P) pl.dp_waves = static_cast<int>(T / P - 1);
    else pl.dp_waves = 0;
    pl.sk_units = (T - static_cast<int64_t>(pl.dp_waves) * P) * G;
    // per group: MMA 2*BT clk (full rate at N >= 128, measured 67% at N = 64), weight unpack
    // ~200 clk; a split tile costs its reducer one partial slot read per extra segment
    const double per_unit = bt >= 128 ? 2.0 * bt : bt == 64 ? 192.0 : 160.0;
    const double unit_cost = per_unit > 200.0 ? per_unit : 200.0;
    const double per_cta = static_cast<double>((units + P - 1) / P);
    const double sk_per_cta = static_cast<double>(pl.sk_units) / P;
    const double segs = sk_per_cta > 0 ? static_cast<double>(G) / sk_per_cta : 0.0;
    const double cost = per_cta * unit_cost +
                        (segs > 1.0 ? segs - 1.0 : 0.0) * slot_bytes_for(bt) / 64.0;
    bool split = false;
    for (int64_t i = 1; i < P && !split && pl.sk_units > 0; ++i)
      split = (i * pl.sk_units / P) % G != 0;
    if (split) {
      // counters are indexed by the reducing CTA, so their region has the same size and place
      // for every shape on this device (only it must stay zero between calls)
      pl.counter_bytes = ((num_sms * sizeof(int) + 255) / 256) * 256;
      pl.workspace_bytes = pl.counter_bytes + pl.grid * slot_bytes_for(bt);
    }
    if (cost < best_cost * 0.97) {
      best_cost = cost;
      best = pl;
    }
  }
  return best;
}

cudaError_t launch_w4a4_gemm(const GemmArgs& a, void* workspace, size_t workspace_bytes,
                             cudaStream_t stream, int num_sms, int* launches) {
  *launches = 0;
  if (a.M == 0) return cudaSuccess;
  const GemmPlan pl = plan_w4a4_gemm(a.M, a.N, a.K, num_sms);
  if (workspace_bytes < pl.workspace_bytes) return cudaErrorInvalidValue;
  switch (pl.bt) {
    case 256: return launch_bt<256>(a, pl, workspace, stream, launches);
    case 128: return launch_bt<128>(a, pl, workspace, stream, launches);
    case 64: return launch_bt<64>(a, pl, workspace, stream, launches);
    default: return launch_bt<32>(a, pl, workspace, stream, launches);
  }
}

}  // namespace atom
