// gemm.cu -- a2-a5: fused W4A4 mixed-precision group GEMM on sm_100a tensor cores.
//
// Paper (Fig 6): per (activation group, weight group) compute the low-bit product on
// the tensor cores (Step 1), dequantize each temporary result with its two group scales (Step 2)
// and sum (Step 3), all fused in the MMA pipeline; the 128 INT8 outlier channels are one more
// group of the same K loop (mixed precision via reordering P:242).
//
// B200 design:
//   * Tile = 128 tokens (MMA M = TMEM lanes) x 256 output channels (MMA N = TMEM columns), one
//     persistent CTA per SM, 2 TMEM accumulator buffers of 256 columns.
//   * INT4 groups run on tcgen05 kind::f8f6f4.  tcgen05 has no 4-bit integer kind and I2FP runs
//     at quarter rate, so both operands are E4M3 bytes whose values are integers times 2^-9
//     (bytes 0x00..0x0F are exactly k * 2^-9, the subnormal-linear range of E4M3):
//       activations  sign-magnitude byte of q_a       (value q_a * 2^-9), written by the
//                    quantize kernel in the GEMM operand form (include/atom.h "a_f8")
//       weights      offset-binary byte nibble ^ 8     (value (q_w + 8) * 2^-9), expanded on the
//                    SM from the canonical packed two's-complement nibbles by one LOP3 per 4
//                    codes (low nibbles) / SHF + LOP3 (high nibbles)
//     The fp32 accumulator then holds P' = 2^-18 (P_t + 8 ca), exactly (|P_t + 8 ca| < 2^15), where
//     P_t is the exact integer group partial and ca = sum of the group's activation codes of the
//     token.  The quantize kernel also writes, per token and group, alpha = s_a * 2^18 and
//     beta = RN(-8 ca * s_a) (include/atom.h "a_ab"), in a row order that gives each epilogue
//     thread its 4 rows in two 16-byte loads.
//   * INT8 outlier group: kind::i8 on the canonical int8 codes, int32 accumulator (one kind
//     switch per tile).
//   * Epilogue (8 warps, 16x256b TMEM loads: a thread holds 4 token rows x 32 channel columns of
//     its warp's 32 x 128 quarter-tile): per output and group exactly two fp32 operations,
//       h = fma(P', alpha_m, beta_m)       alpha = s_a * 2^18, beta = RN(-8 ca * s_a)  (per row)
//       acc = fma(s_w[n], h, acc)                                                     (per col)
//     as FFMA2 on column pairs.  The per-row values and the thread's 32 column scales are read
//     from global memory (L1/L2, LDG) one group ahead: shared-memory loads issued while the
//     tensor core streams its operands stall the drain loop ~3x (profiles/r02/probe_epi.txt).
//   * Stream-K schedule: data-parallel waves of whole tiles, then the remaining (tile, group)
//     units divided evenly; a split tile's segments publish fp32 partials, the CTA holding the
//     last segment adds them in a fixed order (deterministic).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "internal.h"
#include "ptx.cuh"

namespace atom {

// Warp roles (16 warps, 4 warpgroups):
//   WG0: warp 0 packed-weight producer (TMA), warp 1 MMA issuer, warp 2 activation-tile loader
//        (TMA), warp 3 idle
//   WG1: warps 4-7 weight expansion (one per SM sub-partition)
//   WG2-WG3: warps 8-15 epilogue (warp % 4 = TMEM lane quarter, (warp - 8) / 4 = column half)
constexpr int kThreads = 512;
constexpr int kALoaderWarp = 2;
constexpr int kUnpackWarp0 = 4;
constexpr int kNumUnpackWarps = 4;
constexpr int kEpiWarp0 = 8;
constexpr int kNumEpiWarps = 8;
constexpr int kEpiThreads = kNumEpiWarps * 32;
constexpr int kRegsProd = 24, kRegsUnpack = 48, kRegsHigh = 216;   // 128*(24+48) + 256*216 <= 65536
#ifndef ATOM_SWAP_MAX_M
#define ATOM_SWAP_MAX_M 64
#endif
#ifndef ATOM_RW
#define ATOM_RW 2
#endif
#ifndef ATOM_KS
#define ATOM_KS 4
#endif
#ifndef ATOM_LDX
#define ATOM_LDX 2
#endif
constexpr int kRS0 = 4;         // activation slots (= go / mdone ring), kBT = 0 tiles
constexpr int kRW0 = ATOM_RW;   // expanded weight slots, kBT = 0 tiles
constexpr int kLdX = ATOM_LDX;  // 8-column chunks per 16x256b TMEM load
// development timing probes (results wrong by design; only with -DATOM_PROBE_MODE=n):
// bit 0 = the weight expansion moves no data; bit 1 = the epilogue skips its arithmetic;
// bit 2 = the epilogue also skips its TMEM loads; bit 3 = the epilogue keeps the first group's
// scales (no per-group scale loads)
#ifndef ATOM_PROBE_MODE
#define ATOM_PROBE_MODE 0
#endif
#if ATOM_PROBE_MODE != 0 && !defined(ATOM_DEV_PROBES)
#error "ATOM_PROBE_MODE is a development probe: build with -DATOM_DEV_PROBES"
#endif
#ifndef ATOM_LD_AHEAD
#define ATOM_LD_AHEAD 1
#endif
constexpr int kLdAhead = ATOM_LD_AHEAD;   // TMEM loads in flight ahead of the one being used
// split-tile partial of one CTA: [epi warps][32 float4][32 lanes]
constexpr size_t kSlotFloats = static_cast<size_t>(kNumEpiWarps) * 128 * 32;

// Tile configuration.  kBT = 0: the throughput tile, 128 tokens (MMA M, TMEM lanes) x 256 output
// channels (MMA N, TMEM columns).  kBT in {16, 32, 64} (small M, weight streaming): swap-AB,
// the weights are the MMA A operand (128 channels = TMEM lanes) and the kBT tokens the B operand
// (TMEM columns), so the epilogue drains 128 x kBT values per group instead of 128 x 256 of
// which all but M rows would be padding.
template <int kBT>
struct TileCfg {
  static constexpr bool kSwap = kBT > 0;
  static constexpr int TT = kSwap ? kBT : 128;      // tokens per tile
  static constexpr int TN = kSwap ? 128 : 256;      // output channels per tile
  // swap-AB tiles are cheap to drain, so the rings are deeper there: the loop MMA(g - RW) done
  // -> expand group g -> MMA(g) would otherwise bound the group rate (~900 clk per group with
  // 2 expanded-weight slots)
  static constexpr int RS = kSwap ? 8 : kRS0;       // activation slots (= go / mdone ring)
  static constexpr int RW = kSwap ? 4 : kRW0;       // expanded weight slots
  static constexpr int KS = kSwap ? 8 : ATOM_KS;    // packed weight stages (TN x 64 B each)
  static constexpr int RT = kSwap ? 8 : 2;          // TMEM accumulator buffers
  // swap-AB: per-group scales staged in shared memory by the activation loader (bulk copies
  // counted on go[]): the 128 weight scales of the tile (w_sp order) and the a_ab rows of the
  // 32-row block(s) holding the tile's tokens.  The loader writes group g's slot once MMA(g - RS)
  // is done, i.e. after the epilogue released group g - RS - RT, so RA > RS + RT slots never
  // overwrite a slot the epilogue still reads.
  static constexpr int AB_ROWS = kBT < 32 ? 32 : kBT;
  static constexpr int RA = kSwap ? 32 : 1;
  static constexpr int SC_FLOATS = kSwap ? 128 + 2 * AB_ROWS : 4;
  static_assert(!kSwap || RA > RS + RT, "scale ring");
  static constexpr int TC = kSwap ? kBT : 256;      // TMEM columns per buffer
  static constexpr uint32_t kTmemCols = RT * TC < 32 ? 32u : static_cast<uint32_t>(RT * TC);
  static_assert(RT * TC <= 512, "TMEM holds at most 512 columns");
  static_assert((kTmemCols & (kTmemCols - 1)) == 0, "TMEM allocations are powers of two");
  static_assert(RS >= RT && RS >= RW, "ring sizes");
  static_assert(!kSwap || (kBT == 16 || kBT == 32 || kBT == 64), "swap-AB token tiles");
};

struct GemmParams {
  const float* a_ab;         // [G][Mp][2] per-row dequant constants (include/atom.h "a_ab")
  const float* w_sp;         // [G][N] weight scales, GEMM channel order (include/atom.h "w_sp")
  void* c;
  int64_t ldc;
  int32_t* debug;
  int M, N, G, G4, c_f32;
  int Mp;                    // rows of a_ab per group (M rounded up to 128)
  int m_tiles, num_tiles;
  int dp_waves;              // whole tiles per CTA dealt round-robin (at most)
  int64_t sk_base;           // first stream-K unit (= dp_waves * grid * G)
  int64_t sk_units;          // stream-K (tile, group) units
  float* partials;           // [gridDim.x][kSlotFloats] split-tile partials
  int* counters;             // [gridDim.x] arrivals per reducing CTA (zero between launches)
#ifdef ATOM_DEV_PROBES
  long long* trace;          // development timeline probe: [kTraceEv][kTraceN] clock64 of CTA 0
#endif
};

#ifdef ATOM_DEV_PROBES
// Development-only timeline probe (never in the shipped library): clock64 of event ev for group
// g of CTA 0.  Built with ATOM_NVCC_EXTRA=-DATOM_DEV_PROBES, enabled by ATOM_GEMM_TRACE=1.
constexpr int kTraceN = 512, kTraceEv = 31;
#define TRACE(ev, g)                                                                      \
  do {                                                                                    \
    if (p.trace != nullptr && blockIdx.x == 0 && (g) < kTraceN)                           \
      p.trace[(ev) * kTraceN + (g)] = clock64();                                          \
  } while (0)
#else
#define TRACE(ev, g) \
  do {               \
  } while (0)
#endif

template <class C>
struct __align__(1024) GemmSmem {
  uint8_t a[C::RS][C::TT * 128];           // activation group, E4M3 / int8, SW128 K-major (TMA)
  uint8_t w[C::RW][C::TN * 128];           // expanded weight group, SW128 K-major
  uint8_t stage[C::KS][C::TN * 64];      // packed weight group (TMA, no swizzle)
  float sc[C::RA][C::SC_FLOATS];          // swap-AB: staged group scales (16-byte aligned rows)
  uint64_t full[C::KS], empty[C::KS];
  // go[u]: group g (slot u = g % kRS) may be issued -- its weights are expanded (4 arrivals),
  // its activations landed (1 arrival + tx bytes) and its TMEM buffer was drained (8 epilogue
  // arrivals, made when group g - kRT was released).
  uint64_t go[C::RS];
  uint64_t mdone[C::RS];                   // MMAs of a group done: slots free + partial ready
  uint32_t tmem_base;
};
static_assert(sizeof(GemmSmem<TileCfg<0>>) + 1024 <= 232448, "shared memory");
static_assert(sizeof(GemmSmem<TileCfg<64>>) + 1024 <= 232448, "shared memory");

// Packed INT4 weights -> E4M3 offset-binary bytes (nibble ^ 8 = q + 8 in [0, 15]: the E4M3 byte
// of (q + 8) * 2^-9).  Low nibbles (even channels) and high nibbles (odd channels) of a 16-byte
// packed chunk become two 16-byte operand chunks (the channel order of include/atom.h "a_f8").
__device__ __forceinline__ uint32_t lop_and_xor(uint32_t a, uint32_t mask, uint32_t x) {
  uint32_t d;   // (a & mask) ^ x in one LOP3
  asm("lop3.b32 %0, %1, %2, %3, 0x6A;" : "=r"(d) : "r"(a), "r"(mask), "r"(x));
  return d;
}

// ---- schedule ("data-parallel waves + stream-K tail"): the first dp_waves * gridDim.x tiles are
//      whole tiles dealt round-robin (CTA i takes tiles i, i + grid, ...: the m-tiles of an n-tile
//      are neighbours, so they read a weight tile from HBM once); the remaining tiles' (tile,
//      group) units are divided evenly, CTA i owning [sk_start(i), sk_start(i+1)).  A tile cut
//      by those boundaries is computed in K segments by consecutive CTAs.  Each CTA first works
//      on its highest stream-K tile (a tile head it publishes, or a whole tile), then its
//      data-parallel tiles, then its remaining stream-K tiles in descending order (the last
//      one may be a tile tail it reduces), so reducers find the published segments ready. ----
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
  // whole tiles blockIdx.x + i * grid, i < dp_waves, that exist (a split-free plan's last wave
  // may be partial)
  const int avail = (p.num_tiles - static_cast<int>(blockIdx.x) + static_cast<int>(gridDim.x) - 1) /
                    static_cast<int>(gridDim.x);
  s.nd = p.dp_waves < avail ? p.dp_waves : avail;
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
template <class C>
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
  it.n0 = (tile / p.m_tiles) * C::TN;
  it.m0 = (tile % p.m_tiles) * C::TT;
  return it;
}

// Waits of the roles off the MMA <-> epilogue critical loop (producer, activation loader,
// weight expansion): hardware-suspended try_wait, so they do not take issue slots from the
// epilogue warps of their SM sub-partition.
__device__ __forceinline__ void wait_off(uint64_t* bar, uint32_t parity) {
  mbar_wait(bar, parity);
}

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

// 32-byte global load (LDG.E.ENL2.256 on sm_100a)
__device__ __forceinline__ void ldg_v8(const float* p, float (&v)[8]) {
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]),
                 "=f"(v[6]), "=f"(v[7])
               : "l"(p));
}
__device__ __forceinline__ float2 u2f2(uint32_t a, uint32_t b) {
  return make_float2(__uint_as_float(a), __uint_as_float(b));
}

template <int kBT, bool kDebug>
__global__ void __launch_bounds__(kThreads, 1)
w4a4_gemm_kernel(const __grid_constant__ CUtensorMap tm_wq4,
                 const __grid_constant__ CUtensorMap tm_wq8,
                 const __grid_constant__ CUtensorMap tm_af8, const GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
#ifdef ATOM_DEV_PROBES
  auto gtimer = []() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return static_cast<long long>(t);
  };
  if (p.trace != nullptr && threadIdx.x == 0 && blockIdx.x < kTraceN)
    p.trace[25 * kTraceN + blockIdx.x] = gtimer();
#endif
  using C = TileCfg<kBT>;
  constexpr int kKS = C::KS, kRT = C::RT, kRS = C::RS, kRW = C::RW;
  GemmSmem<C>& sm = *reinterpret_cast<GemmSmem<C>*>(
      smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kKS; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], C::kSwap ? 1 : kNumUnpackWarps);
    }
    for (int u = 0; u < kRS; ++u) {
      mbar_init(&sm.go[u], (C::kSwap ? 1 : kNumUnpackWarps) + 1 + kNumEpiWarps);
      mbar_init(&sm.mdone[u], 1);
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_wq4);
    tma_prefetch_desc(&tm_wq8);
    tma_prefetch_desc(&tm_af8);
  }
  if (warp == 1) tmem_alloc(&sm.tmem_base, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  const int G4 = p.G4;
  const Sched sch = make_sched(p);
  const int n_items = sch.count();

  if (threadIdx.x == 0) griddep_launch();   // the next kernel still waits for this grid's end
  // setmaxnreg sits at the top of each warpgroup's branch, so ptxas allocates every role's code
  // with its own register budget
  if (warp < kUnpackWarp0) {
    setmaxnreg_dec<kRegsProd>();
    if (warp == 0) {
      // ===================== producer: packed weight groups (TMA) =====================
      // INT4 group: one stage [256 rows][64 B]; INT8 group: two stages (bytes 0-63, 64-127).
      if (lane == 0) {
        Ring<kKS> st;
        const uint64_t pol_w = l2_policy_evict_first();
        if (n_items > 0) {   // PDL: warm L2 with the first weight groups while the previous ends
          const Item w = get_item<C>(p, sch, 0);
          for (int t = w.t0, s = 0; t < w.t1 && t < G4 && s < kKS; ++t, ++s)
            tma_prefetch_2d(&tm_wq4, t * 64, w.n0);
        }
        griddep_wait();
        int gp = 0;
        for (int k = 0; k < n_items; ++k) {
          const Item w = get_item<C>(p, sch, k);
          for (int t = w.t0; t < w.t1; ++t, ++gp) {
            const int nst = t < G4 ? 1 : 2;
            for (int h = 0; h < nst; ++h, st.next()) {
              mbar_wait(&sm.empty[st.i], st.ph ^ 1);
              TRACE(0, gp);
              mbar_arrive_expect_tx(&sm.full[st.i], C::TN * 64);
              // read by the m-tiles of this n-tile at about the same time, then dead
              if (t < G4)
                tma_load_2d_hint(sm.stage[st.i], &tm_wq4, &sm.full[st.i], t * 64, w.n0, pol_w);
              else
                tma_load_2d_hint(sm.stage[st.i], &tm_wq8, &sm.full[st.i], h * 64, w.n0, pol_w);
            }
          }
        }
      }
    } else if (warp == kALoaderWarp) {
      // ===================== activation-tile loader (single thread) =====================
      // Slot u is free exactly when the MMAs of the group that used it complete.  The group's
      // scales (weight scales of the tile's channels, activation scales and code sums of its
      // tokens) are prefetched into L2 at the same time, kRS groups ahead of the epilogue that
      // reads them with plain loads.
      if (lane == 0) {
        Ring<kRS> u;
        const uint64_t pol_a = l2_policy_evict_last();
        griddep_wait();                  // activations and scales come from the previous kernel
        int ga = 0;
        for (int k = 0; k < n_items; ++k) {
          const Item w = get_item<C>(p, sch, k);
          const uint32_t sw_bytes = static_cast<uint32_t>(min(C::TN, p.N - w.n0)) * 4;
          for (int t = w.t0; t < w.t1; ++t, u.next(), ++ga) {
            wait_off(&sm.mdone[u.i], u.ph ^ 1);
            TRACE(1, ga);
            if constexpr (C::kSwap) {
              float* sc = sm.sc[ga % C::RA];
              mbar_arrive_expect_tx(&sm.go[u.i], C::TT * 128 + 512 + C::AB_ROWS * 8);
              tma_load_2d_hint(sm.a[u.i], &tm_af8, &sm.go[u.i], t * 128, w.m0, pol_a);
              bulk_g2s(sc, p.w_sp + static_cast<int64_t>(t) * p.N + w.n0, 512, &sm.go[u.i]);
              bulk_g2s(sc + 128, p.a_ab + 2 * (static_cast<int64_t>(t) * p.Mp + (w.m0 & ~31)),
                       C::AB_ROWS * 8, &sm.go[u.i]);
              continue;
            }
            mbar_arrive_expect_tx(&sm.go[u.i], C::TT * 128);
            // re-read by every n-tile: keep in L2
            tma_load_2d_hint(sm.a[u.i], &tm_af8, &sm.go[u.i], t * 128, w.m0, pol_a);
            prefetch_l2_bulk(p.w_sp + static_cast<int64_t>(t) * p.N + w.n0, sw_bytes);
            prefetch_l2_bulk(p.a_ab + 2 * (static_cast<int64_t>(t) * p.Mp + w.m0), C::TT * 8);
          }
        }
      }
#ifdef ATOM_DEV_PROBES
    } else if (warp == 3) {
      // development probe: observe every group's MMA completion (event 8)
      if (lane == 0 && p.trace != nullptr && blockIdx.x == 0) {
        Ring<kRS> u;
        int go_ = 0;
        for (int k = 0; k < n_items; ++k) {
          const Item w = get_item<C>(p, sch, k);
          for (int t = w.t0; t < w.t1; ++t, u.next(), ++go_) {
            mbar_wait_spin(&sm.mdone[u.i], u.ph);
            TRACE(8, go_);
          }
        }
      }
#endif
    } else if (warp == 1) {
      // ===================== MMA issuer (single thread) =====================
      // Every instruction this thread executes between dispatches idles the tensor pipe for as
      // long (tcgen05.mma issue returns only as the previous dispatch drains), so the loop is
      // one barrier probe, 4 dispatches and one commit per group.  (Swap-AB: a 128 x kBT x 32
      // dispatch takes ~130 clk from issue to drain whatever kBT is; a second issuing thread
      // for alternate groups measured no faster.)
      if (lane == 0) {
        // swap-AB: A = the weights (128 channels), B = the kBT tokens
        constexpr uint32_t id4 = umma_idesc_e4m3(128, C::kSwap ? kBT : C::TN);
        constexpr uint32_t id8 = umma_idesc_i8(128, C::kSwap ? kBT : C::TN);
        const uint64_t da0 = umma_desc_sw128(smem_u32(sm.a[0]));
        const uint64_t db0 = umma_desc_sw128(smem_u32(sm.w[0]));
        Ring<kRS> u;
        Ring<kRW> uw;
        Ring<kRT> b;
        int gm = 0;
        for (int k = 0; k < n_items; ++k) {
          const Item w = get_item<C>(p, sch, k);
          for (int t = w.t0; t < w.t1; ++t, u.next(), uw.next(), b.next(), ++gm) {
            mbar_wait_test(&sm.go[u.i], u.ph);
            TRACE(3, gm);
            tc_fence_after();
            const uint32_t d = tmem + b.i * C::TC;
            // descriptor start address field counts 16-byte units: slot, K step kk (32 bytes)
            const uint64_t da = da0 + u.i * (C::TT * 128 / 16);
            const uint64_t db = db0 + uw.i * (C::TN * 128 / 16);
            const uint64_t dA = C::kSwap ? db : da, dB = C::kSwap ? da : db;
            if (t < G4) {
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) umma_e4m3(d, dA + 2 * kk, dB + 2 * kk, id4, kk > 0);
            } else {
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) umma_i8(d, dA + 2 * kk, dB + 2 * kk, id8, kk > 0);
            }
            umma_commit(&sm.mdone[u.i]);
          }
        }
      }
    }
  } else if (warp < kEpiWarp0) {
    setmaxnreg_dec<kRegsUnpack>();
    if constexpr (C::kSwap) {
      // ===== swap-AB weight expansion: unpack warp uw expands every 4th group on its own
      //       (groups g = uw mod 4), so 4 groups are in flight (one warp per group keeps the
      //       expansion off the MMA's critical loop; the cooperative 4-warp form of kBT = 0
      //       took ~850 clk per group there).  Lane l owns 16-byte chunk c = l & 3 of stage
      //       rows (l >> 2) + 8 j, j < 16; row r is operand row r (TMEM lane r), swizzle phase
      //       r & 7 = l >> 2. ----
      const int uwi = warp - kUnpackWarp0;
      const uint32_t rr = static_cast<uint32_t>(lane) >> 2, cc = static_cast<uint32_t>(lane) & 3u;
      uint32_t m0f = 0x0F0F0F0Fu, x08 = 0x08080808u;
      asm volatile("" : "+r"(m0f), "+r"(x08));
      Ring<kKS> st;
      Ring<kRS> u;
      Ring<kRS> lag;                     // mdone slot of group g - kRW
      Ring<kRW> uw;
      int gu = 0;
      griddep_wait();
      for (int k = 0; k < n_items; ++k) {
        const Item w = get_item<C>(p, sch, k);
        for (int t = w.t0; t < w.t1; ++t, u.next(), uw.next(), ++gu) {
          const int nst = t < G4 ? 1 : 2;
          if ((gu & 3) != uwi) {         // another warp's group: advance the rings only
            for (int h = 0; h < nst; ++h) st.next();
            if (gu >= kRW) lag.next();
            continue;
          }
          if (gu >= kRW) {               // MMAs of group g - kRW finished with this slot
            wait_off(&sm.mdone[lag.i], lag.ph);
            lag.next();
          }
          if (lane == 0) TRACE(2, gu);
          uint8_t* dst = sm.w[uw.i];
          if (t < G4) {
            wait_off(&sm.full[st.i], st.ph);
            const uint8_t* src = sm.stage[st.i] + rr * 64 + cc * 16;
#pragma unroll
            for (int j0 = 0; j0 < 16; j0 += 4) {
              uint4 v[4];
#pragma unroll
              for (int j = 0; j < 4; ++j)
                v[j] = *reinterpret_cast<const uint4*>(src + (j0 + j) * 8 * 64);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                uint8_t* d = dst + (rr + 8 * (j0 + j)) * 128;
                *reinterpret_cast<uint4*>(d + (((2 * cc) ^ rr) << 4)) =
                    make_uint4(lop_and_xor(v[j].x, m0f, x08), lop_and_xor(v[j].y, m0f, x08),
                               lop_and_xor(v[j].z, m0f, x08), lop_and_xor(v[j].w, m0f, x08));
                *reinterpret_cast<uint4*>(d + (((2 * cc + 1) ^ rr) << 4)) = make_uint4(
                    lop_and_xor(v[j].x >> 4, m0f, x08), lop_and_xor(v[j].y >> 4, m0f, x08),
                    lop_and_xor(v[j].z >> 4, m0f, x08), lop_and_xor(v[j].w >> 4, m0f, x08));
              }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.empty[st.i]);
            st.next();
          } else {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              wait_off(&sm.full[st.i], st.ph);
              const uint8_t* src = sm.stage[st.i] + rr * 64 + cc * 16;
#pragma unroll
              for (int j0 = 0; j0 < 16; j0 += 4) {
                uint4 v[4];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                  v[j] = *reinterpret_cast<const uint4*>(src + (j0 + j) * 8 * 64);
#pragma unroll
                for (int j = 0; j < 4; ++j)
                  *reinterpret_cast<uint4*>(dst + (rr + 8 * (j0 + j)) * 128 +
                                            (((4 * h + cc) ^ rr) << 4)) = v[j];
              }
              __syncwarp();
              if (lane == 0) mbar_arrive(&sm.empty[st.i]);
              st.next();
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) TRACE(4, gu);
          if (lane == 0) mbar_arrive(&sm.go[u.i]);
        }
      }
    } else {
    // ===================== weight expansion -> E4M3 offset-binary / int8, SW128 =============
    // 128 threads: thread ut owns 16-byte chunk c = ut & 3 of the 64-byte stage rows
    // r0 + 32k, k < TN / 32 (r0 = ut >> 2).  Weight row r of the tile is operand row r: TMEM
    // column r (kBT = 0, B operand) or TMEM lane r (swap-AB, A operand) holds output channel
    // n0 + r.  The SW128 swizzle phase of row r is r0 & 7.
    constexpr int kRowsPT = C::TN / 32;
    const int ut = threadIdx.x - kUnpackWarp0 * 32;
    const uint32_t r0 = static_cast<uint32_t>(ut) >> 2, c = static_cast<uint32_t>(ut) & 3u;
    const uint32_t jb = r0;              // operand row of k = 0
    uint32_t m0f = 0x0F0F0F0Fu, x08 = 0x08080808u;
    asm volatile("" : "+r"(m0f), "+r"(x08));   // keep the LOP3 constants in registers
    Ring<kKS> st;
    Ring<kRS> u;                         // go slot of group g
    Ring<kRS> lag;                       // mdone slot of group g - kRW
    Ring<kRW> uw;                        // expanded-weight slot of group g
    int gu = 0;
    griddep_wait();
    for (int k = 0; k < n_items; ++k) {
      const Item w = get_item<C>(p, sch, k);
      for (int t = w.t0; t < w.t1; ++t, u.next(), uw.next(), ++gu) {
        if (gu >= kRW) {                 // MMAs of group g - kRW finished with this slot
          wait_off(&sm.mdone[lag.i], lag.ph);
          lag.next();
        }
        if (ut == 0) TRACE(2, gu);
        uint8_t* dst = sm.w[uw.i];
        if (t < G4) {
          wait_off(&sm.full[st.i], st.ph);
          const uint8_t* src = sm.stage[st.i] + r0 * 64 + c * 16;
          // all 8 shared-memory loads first: their latency grows several-fold while the tensor
          // core streams operands, so it is paid once per group
          uint4 v[kRowsPT];
#pragma unroll
          for (int j = 0; j < kRowsPT; ++j)
            if constexpr ((ATOM_PROBE_MODE & 1) == 0)
              v[j] = *reinterpret_cast<const uint4*>(src + j * 32 * 64);
#pragma unroll
          for (int j = 0; j < kRowsPT; ++j) {
            if constexpr ((ATOM_PROBE_MODE & 1) != 0) break;
            const uint32_t row = jb + 32 * j, ph = r0 & 7;
            uint8_t* d = dst + row * 128;
            *reinterpret_cast<uint4*>(d + (((2 * c) ^ ph) << 4)) =
                make_uint4(lop_and_xor(v[j].x, m0f, x08), lop_and_xor(v[j].y, m0f, x08),
                           lop_and_xor(v[j].z, m0f, x08), lop_and_xor(v[j].w, m0f, x08));
            *reinterpret_cast<uint4*>(d + (((2 * c + 1) ^ ph) << 4)) =
                make_uint4(lop_and_xor(v[j].x >> 4, m0f, x08), lop_and_xor(v[j].y >> 4, m0f, x08),
                           lop_and_xor(v[j].z >> 4, m0f, x08), lop_and_xor(v[j].w >> 4, m0f, x08));
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.empty[st.i]);
          st.next();
        } else {
          // INT8 outlier group: bytes 0-63 of each row in one stage, 64-127 in the next; copied
          // with the same row permutation
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            wait_off(&sm.full[st.i], st.ph);
            const uint8_t* src = sm.stage[st.i] + r0 * 64 + c * 16;
            uint4 v[kRowsPT];
#pragma unroll
            for (int j = 0; j < kRowsPT; ++j)
              v[j] = *reinterpret_cast<const uint4*>(src + j * 32 * 64);
#pragma unroll
            for (int j = 0; j < kRowsPT; ++j) {
              const uint32_t row = jb + 32 * j, ph = r0 & 7;
              *reinterpret_cast<uint4*>(dst + row * 128 + (((4 * h + c) ^ ph) << 4)) = v[j];
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.empty[st.i]);
            st.next();
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (ut == 0) TRACE(4, gu);
        if (lane == 0) mbar_arrive(&sm.go[u.i]);
      }
    }
    }   // kBT = 0 weight expansion
  } else {
    // ===================== epilogue warps =====================
    setmaxnreg_inc<kRegsHigh>();
    if constexpr (C::kSwap) {
      // ---- swap-AB (small M): thread = TMEM lane = output channel n0 + 32 q + lane; the two
      //      warps of a lane quarter drain token columns [h * kBT/2, (h + 1) * kBT/2).  Per
      //      output and group the same two fp32 operations as the kBT = 0 epilogue:
      //      h = fma(P', alpha_m, beta_m), acc = fma(s_w[n], h, acc). ----
      constexpr int NH = kBT / 2;
      const int e = warp - kEpiWarp0;
      const int q = warp & 3, hf = e >> 2;
      const int nl = q * 32 + lane;
      const int et = e * 32 + lane;
      const uint32_t tq = tmem + (static_cast<uint32_t>(q * 32) << 16) + hf * NH;
      const int kq = nl >> 3;   // position of channel nl in the w_sp order (include/atom.h)
      const int spos = 32 * (kq >> 2) + 8 * ((nl & 7) >> 1) + 2 * (kq & 3) + (nl & 1);
      griddep_wait();
      if (lane == 0)
        for (int bb = 0; bb < kRT; ++bb) mbar_arrive(&sm.go[bb % kRS]);
      // token m0 + hf NH + i of group t sits at a_ab row t Mp + (m0 & ~31) + tb + 4 (i % 8) + i / 8
      // (include/atom.h "a_ab"): tb = mb - rb + rb / 8, mb = m0 % 32 + hf NH, rb = mb % 32
      auto tok_base = [&](int m0) {
        const int mb = (m0 & 31) + hf * NH, rb = mb & 31;
        return mb - rb + (rb >> 3);
      };
      constexpr auto ab_off = [](int i) { return 4 * (i & 7) + (i >> 3); };
      Ring<kRS> u;
      Ring<kRT> b;
      int ge = 0;
      for (int k = 0; k < n_items; ++k) {
        const Item w = get_item<C>(p, sch, k);
        const int tb = tok_base(w.m0);
        float acc[NH];
#pragma unroll
        for (int i = 0; i < NH; ++i) acc[i] = 0.0f;
        for (int t = w.t0; t < w.t1; ++t, u.next(), b.next(), ++ge) {
          mbar_wait_test(&sm.mdone[u.i], u.ph);
          // the group's staged scales: go[u] (completed by the bulk copies) cannot advance
          // before this warp's release below, so the probe returns at once and makes the
          // async-proxy writes visible here
          mbar_wait_test(&sm.go[u.i], u.ph);
          if (e == 0 && lane == 0) TRACE(5, ge);
          const float* sc = sm.sc[ge % C::RA];
          const float sw_c = sc[spos];
          const float2* abr = reinterpret_cast<const float2*>(sc + 128) + tb;
          float2 ab_c[NH];
#pragma unroll
          for (int i = 0; i < NH; ++i) ab_c[i] = abr[ab_off(i)];
          tc_fence_after();
          uint32_t r[NH];
          tmem_ld_32x32b<NH>(tq + b.i * C::TC, r);
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          const uint32_t go_next = u.i + kRT >= kRS ? u.i + kRT - kRS : u.i + kRT;
          if (lane == 0) mbar_arrive(&sm.go[go_next]);
          if (e == 0 && lane == 0) TRACE(6, ge);
          const bool int4 = t < G4;
#pragma unroll
          for (int i = 0; i < NH; ++i) {
            const float pv = int4 ? __uint_as_float(r[i]) : __int2float_rn(static_cast<int>(r[i]));
            if constexpr (kDebug) {
              const int m = w.m0 + hf * NH + i, n = w.n0 + nl;
              if (m < p.M) {
                int pi;
                if (int4) {   // P = P' * 2^18 - 8 ca, exact (see the kBT = 0 epilogue)
                  const int ca = __double2int_rn(-static_cast<double>(ab_c[i].y) * 32768.0 /
                                                 static_cast<double>(ab_c[i].x));
                  pi = __float2int_rn(pv * 262144.0f) - 8 * ca;
                } else {
                  pi = static_cast<int>(r[i]);
                }
                p.debug[(static_cast<int64_t>(t) * p.M + m) * p.N + n] = pi;
              }
            }
            acc[i] = __fmaf_rn(sw_c, __fmaf_rn(pv, ab_c[i].x, ab_c[i].y), acc[i]);
          }
          if (e == 0 && lane == 0) TRACE(7, ge);
        }
        // split tile: publish / reduce as in the kBT = 0 epilogue (thread-linear slot layout)
        if (w.t1 < p.G || w.t0 > 0) {
          if (w.t1 < p.G) {
            float* slot = p.partials + static_cast<int64_t>(blockIdx.x) * kSlotFloats;
#pragma unroll
            for (int i = 0; i < NH; ++i) __stcg(slot + i * kEpiThreads + et, acc[i]);
            __threadfence();
            named_bar_sync(1, kEpiThreads);
            if (e == 0 && lane == 0)
              red_release_add(p.counters + cta_of(p, static_cast<int64_t>(w.tile + 1) * p.G - 1), 1);
            continue;
          }
          const int first = cta_of(p, static_cast<int64_t>(w.tile) * p.G);
          const int nseg = static_cast<int>(blockIdx.x) - first;
          if (e == 0 && lane == 0) {
            flag_wait_ge(p.counters + blockIdx.x, nseg);
            p.counters[blockIdx.x] = 0;
          }
          named_bar_sync(1, kEpiThreads);
          for (int i0 = first; i0 < static_cast<int>(blockIdx.x); ++i0) {
            const float* slot = p.partials + static_cast<int64_t>(i0) * kSlotFloats;
#pragma unroll
            for (int i = 0; i < NH; ++i) acc[i] += __ldcg(slot + i * kEpiThreads + et);
          }
        }
        const int n = w.n0 + nl;
#pragma unroll
        for (int i = 0; i < NH; ++i) {
          const int m = w.m0 + hf * NH + i;
          if (m >= p.M) continue;
          if (!p.c_f32)
            static_cast<__half*>(p.c)[static_cast<int64_t>(m) * p.ldc + n] = __float2half_rn(acc[i]);
          else
            static_cast<float*>(p.c)[static_cast<int64_t>(m) * p.ldc + n] = acc[i];
        }
      }
    } else {
    const int e = warp - kEpiWarp0;
    const int q = warp & 3;              // TMEM lane quarter this warp may access
    const int half = e >> 2;             // column half
    const uint32_t tq = tmem + (static_cast<uint32_t>(q * 32) << 16) + half * 128;
    const int rl = q * 32 + (lane >> 2);           // + 8 ri: the thread's 4 tile rows
    const int cl = half * 128 + 2 * (lane & 3);    // + 8 k (+1): its 16 channel pairs
    griddep_wait();
    if (lane == 0)                       // the first kRT groups find their TMEM buffers free
      for (int b = 0; b < kRT; ++b) mbar_arrive(&sm.go[b % kRS]);

    // scales of the group being drained: 16 channel-pair weight scales and per-row alpha /
    // beta, loaded (LDG: unaffected by the tensor core's shared-memory traffic, unlike LDS)
    // one group ahead, the weight scales 4 pairs at a time as their registers fall free.
    // w_sp holds each thread's 4 pairs of a load in 32 contiguous bytes, the 4 threads of a
    // pair column in one 128-byte line (include/atom.h "w_sp"): 4 32-byte loads per group.  The right half of a partial n-tile (N % 256 == 128) reads the left half's
    // scales (its outputs are never stored).
    const int cs_off = half * 128 + 8 * (lane & 3);
    const int cs_ld = cs_off - ((half == 1 && (p.N & 255) != 0) ? 128 : 0);
    float2 sw[16];
    float al[4], be[4];
    auto sw_base = [&](int t, int n0) {
      return p.w_sp + static_cast<int64_t>(t) * p.N + n0 + ((n0 + C::TN <= p.N) ? cs_off : cs_ld);
    };
    auto load_sw = [&](const float* ws, int k0, int nk) {   // channel pairs k0 .. k0+nk (k0 % 4 == 0)
#pragma unroll
      for (int k = 0; k < 16; k += 4)
        if (k >= k0 && k < k0 + nk) {
          float v[8];
          ldg_v8(ws + 8 * k, v);     // pairs k..k+3: 32 (k / 4) floats in
          sw[k] = make_float2(v[0], v[1]);
          sw[k + 1] = make_float2(v[2], v[3]);
          sw[k + 2] = make_float2(v[4], v[5]);
          sw[k + 3] = make_float2(v[6], v[7]);
        }
    };
    // per-row alpha / beta of rows rl + 8 ri: two 16-byte loads (a_ab row order)
    auto load_ab = [&](int t, int m0, float* a, float* bb) {
      const float* pa = p.a_ab + 2 * (static_cast<int64_t>(t) * p.Mp + m0 + q * 32 + 4 * (lane >> 2));
      float v[8];
      ldg_v8(pa, v);
      a[0] = v[0]; bb[0] = v[1]; a[1] = v[2]; bb[1] = v[3];
      a[2] = v[4]; bb[2] = v[5]; a[3] = v[6]; bb[3] = v[7];
    };
    if (n_items > 0) {
      const Item w0 = get_item<C>(p, sch, 0);
      load_ab(w0.t0, w0.m0, al, be);
      load_sw(sw_base(w0.t0, w0.n0), 0, 16);
    }
    Ring<kRS> u;
    Ring<kRT> b;
    int ge = 0;
    for (int k = 0; k < n_items; ++k) {
      const Item w = get_item<C>(p, sch, k);
      // first group of the next item (after the last group, "next" is the last group itself:
      // harmless reloads, no branches)
      int nt0 = w.t1 - 1, nn0 = w.n0, nm0 = w.m0;
      if (k + 1 < n_items) {
        const Item wn = get_item<C>(p, sch, k + 1);
        nt0 = wn.t0;
        nn0 = wn.n0;
        nm0 = wn.m0;
      }
      float2 acc[4][16];
#pragma unroll
      for (int ri = 0; ri < 4; ++ri)
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[ri][j] = make_float2(0.0f, 0.0f);
      for (int t = w.t0; t < w.t1; ++t, u.next(), b.next(), ++ge) {
        const bool last = t + 1 >= w.t1;
        const int xt = last ? nt0 : t + 1;     // next group
        const int xn0 = last ? nn0 : w.n0, xm0 = last ? nm0 : w.m0;
        const float* xws = sw_base(xt, xn0);
        float al_n[4], be_n[4];
        if constexpr ((ATOM_PROBE_MODE & 32) == 0) load_ab(xt, xm0, al_n, be_n);
        // the next group's last 4 channel pairs are loaded now too (into temporaries): a load
        // issued at the very end of the group would hold the scoreboard that the next group's
        // first instructions wait on
        float sw_last[8];
        ldg_v8(xws + 8 * 12, sw_last);
        mbar_wait_test(&sm.mdone[u.i], u.ph);
        if (e == 0 && lane == 0) TRACE(5, ge);
        if (lane == 0) TRACE(17 + e, ge);
        tc_fence_after();
        const uint32_t taddr = tq + b.i * C::TC;
        const uint32_t go_next = u.i + kRT >= kRS ? u.i + kRT - kRS : u.i + kRT;
        // loads j = 2 cb + hh: 16 lanes (half hh of the quarter) x kLdX chunks (block cb),
        // software-pipelined kLdAhead loads ahead
        auto drain = [&](auto int4_tag) {
          constexpr bool kInt4 = decltype(int4_tag)::value;
          constexpr int NL = 2 * (16 / kLdX);
          constexpr int NB = kLdAhead + 1;               // load buffers in flight
          uint32_t r[NB][4 * kLdX];
          auto ld = [&](int j, uint32_t* dst) {
            const int hh = j & 1, cb = j >> 1;
            if constexpr ((ATOM_PROBE_MODE & 4) != 0) {
#pragma unroll
              for (int v = 0; v < 4 * kLdX; ++v) dst[v] = taddr + v + j;
            } else {
              tmem_ld_16x256b<kLdX>(
                  taddr + (static_cast<uint32_t>(16 * hh) << 16) + 8 * kLdX * cb, dst);
            }
          };
#pragma unroll
          for (int j = 0; j < kLdAhead; ++j) ld(j, r[j]);
#pragma unroll
          for (int j = 0; j < NL; ++j) {
            uint32_t* rv = r[j % NB];
            if (j + kLdAhead < NL) {
              ld(j + kLdAhead, r[(j + kLdAhead) % NB]);
              // keep the registers of the loads in flight live across this issue (the LDTM
              // destination registers are scoreboarded)
#pragma unroll
              for (int a = 0; a < kLdAhead; ++a)
#pragma unroll
                for (int v = 0; v < 4 * kLdX; ++v) asm volatile("" : "+r"(r[(j + a) % NB][v]));
            }
            if (j + kLdAhead == NL) {                  // all loads issued: release the buffer
              tmem_ld_wait();
              tc_fence_before();
              __syncwarp();
              if (e == 0 && lane == 0) TRACE(6, ge);
              if (lane == 0) TRACE(9 + e, ge);
              if (lane == 0) mbar_arrive(&sm.go[go_next]);
            }
            const int hh = j & 1, cb = j >> 1;
#pragma unroll
            for (int ch = 0; ch < kLdX; ++ch) {
              const int kc = cb * kLdX + ch;           // channel-pair index of this chunk
#pragma unroll
              for (int s = 0; s < 2; ++s) {            // tile row 2 hh + s
                const int ri = 2 * hh + s;
                const uint32_t x0 = rv[4 * ch + 2 * s], x1 = rv[4 * ch + 2 * s + 1];
                float2 pv;
                if constexpr (kInt4) pv = u2f2(x0, x1);
                else   // INT8 group: exact int32 partial
                  pv = make_float2(__int2float_rn(static_cast<int>(x0)),
                                   __int2float_rn(static_cast<int>(x1)));
                if constexpr (kDebug) {
                  const int m = w.m0 + rl + 8 * ri;
                  const int n = w.n0 + cl + 8 * kc;
                  if (m < p.M && n < p.N) {
                    int p0, p1;
                    if constexpr (kInt4) {   // P = P' * 2^18 - 8 ca, exact
                      // ca = -beta / (8 s_a) rounded: beta = RN(-8 ca s_a) is within 2^-11 s_a
                      const int ca = __double2int_rn(-static_cast<double>(be[ri]) * 32768.0 /
                                                     static_cast<double>(al[ri]));
                      p0 = __float2int_rn(pv.x * 262144.0f) - 8 * ca;
                      p1 = __float2int_rn(pv.y * 262144.0f) - 8 * ca;
                    } else {
                      p0 = static_cast<int>(x0);
                      p1 = static_cast<int>(x1);
                    }
                    int32_t* dp = p.debug + (static_cast<int64_t>(t) * p.M + m) * p.N + n;
                    dp[0] = p0;
                    dp[1] = p1;
                  }
                }
                if constexpr ((ATOM_PROBE_MODE & 2) != 0) {
                  acc[ri][kc].x += pv.x;
                  continue;
                }
                const float2 h = __ffma2_rn(pv, make_float2(al[ri], al[ri]),
                                            make_float2(be[ri], be[ri]));
                acc[ri][kc] = __ffma2_rn(sw[kc], h, acc[ri][kc]);
              }
            }
            // block cb done for both lane halves: its channel scales are free for the next group
            if constexpr ((ATOM_PROBE_MODE & 16) == 0)
              // blocks cb - 1, cb done for both lane halves: 4 pairs of scales free
              if (hh == 1 && ((cb + 1) * kLdX) % 4 == 0) {
                if ((cb + 1) * kLdX < 16) {
                  load_sw(xws, (cb + 1) * kLdX - 4, 4);
                } else {
#pragma unroll
                  for (int v = 0; v < 4; ++v) sw[12 + v] = make_float2(sw_last[2 * v], sw_last[2 * v + 1]);
                }
              }
          }
        };
        if (t < G4) drain(std::true_type{});
        else drain(std::false_type{});
#pragma unroll
        for (int ri = 0; ri < 4; ++ri) {
          if constexpr ((ATOM_PROBE_MODE & 32) == 0) {
            al[ri] = al_n[ri];
            be[ri] = be_n[ri];
          }
        }
        if (e == 0 && lane == 0) TRACE(7, ge);
      }

      // ---- split tile: every segment but the tile's last publishes its fp32 partial; the CTA
      //      holding the last segment adds the others (in CTA order, deterministic) ----
      // fragment i (float4) of this thread: row i / 8, channel pairs 2 (i % 8), 2 (i % 8) + 1
      if (w.t1 < p.G || w.t0 > 0) {
        auto frag = [&](float* slot, int i) {
          return reinterpret_cast<float4*>(slot) + (e * 32 + i) * 32 + lane;
        };
        if (w.t1 < p.G) {                    // publisher (this CTA's first item)
          float* slot = p.partials + static_cast<int64_t>(blockIdx.x) * kSlotFloats;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float2 x = acc[i / 8][2 * (i % 8)], y = acc[i / 8][2 * (i % 8) + 1];
            __stcg(frag(slot, i), make_float4(x.x, x.y, y.x, y.y));
          }
          __threadfence();
          named_bar_sync(1, kEpiThreads);
          if (e == 0 && lane == 0) {
            red_release_add(p.counters + cta_of(p, static_cast<int64_t>(w.tile + 1) * p.G - 1), 1);
#ifdef ATOM_DEV_PROBES
            if (p.trace != nullptr && blockIdx.x < kTraceN) p.trace[30 * kTraceN + blockIdx.x] = gtimer();
#endif
          }
          continue;
        }
        // reducer (this CTA's last item): the other segments belong to CTAs first..blockIdx-1
        const int first = cta_of(p, static_cast<int64_t>(w.tile) * p.G);
        const int nseg = static_cast<int>(blockIdx.x) - first;
        if (e == 0 && lane == 0) {
#ifdef ATOM_DEV_PROBES
          if (p.trace != nullptr && blockIdx.x < kTraceN) {
            p.trace[27 * kTraceN + blockIdx.x] = gtimer();
            p.trace[29 * kTraceN + blockIdx.x] = nseg;
          }
#endif
          flag_wait_ge(p.counters + blockIdx.x, nseg);
#ifdef ATOM_DEV_PROBES
          if (p.trace != nullptr && blockIdx.x < kTraceN) p.trace[28 * kTraceN + blockIdx.x] = gtimer();
#endif
          p.counters[blockIdx.x] = 0;        // self-cleaning for the next launch
        }
        named_bar_sync(1, kEpiThreads);
        for (int i0 = first; i0 < static_cast<int>(blockIdx.x); ++i0) {
          float* slot = p.partials + static_cast<int64_t>(i0) * kSlotFloats;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float4 o = __ldcg(frag(slot, i));
            float2& x = acc[i / 8][2 * (i % 8)];
            float2& y = acc[i / 8][2 * (i % 8) + 1];
            x.x += o.x;
            x.y += o.y;
            y.x += o.z;
            y.y += o.w;
          }
        }
      }

      // ---- tile output: rows m0 + rl + 8 ri, 32 consecutive channels n0 + cl .. +32 ----
      if (w.n0 + half * 128 >= p.N) continue;          // right half of a partial n-tile
#pragma unroll
      for (int ri = 0; ri < 4; ++ri) {
        const int m = w.m0 + rl + 8 * ri;
        if (m >= p.M) continue;
        if (!p.c_f32) {
          __half2* crow = reinterpret_cast<__half2*>(static_cast<__half*>(p.c) +
                                                     static_cast<int64_t>(m) * p.ldc + w.n0 + cl);
#pragma unroll
          for (int kc = 0; kc < 16; ++kc) crow[4 * kc] = __float22half2_rn(acc[ri][kc]);
        } else {
          float2* crow = reinterpret_cast<float2*>(static_cast<float*>(p.c) +
                                                   static_cast<int64_t>(m) * p.ldc + w.n0 + cl);
#pragma unroll
          for (int kc = 0; kc < 16; ++kc) crow[4 * kc] = acc[ri][kc];
        }
      }
    }
    }   // kBT = 0 epilogue
  }

  tc_fence_before();
  __syncthreads();
#ifdef ATOM_DEV_PROBES
  if (p.trace != nullptr && threadIdx.x == 0 && blockIdx.x < kTraceN)
    p.trace[26 * kTraceN + blockIdx.x] = gtimer();
#endif
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, C::kTmemCols);
  }
}

// ---------------------------------------------------------------------------------------------
// activation operand expansion (canonical packed codes + scales -> a_f8 + a_ab), for
// atom_w4a4_gemm
// ---------------------------------------------------------------------------------------------
// One thread per 16-byte packed chunk (32 codes) of an INT4 group, 4 threads per group: the
// two's-complement nibbles become E4M3 sign-magnitude bytes (value q * 2^-9) in the a_f8 order
// (within each 32-channel chunk the even channels first, then the odd ones); the group's code
// sum is reduced over the 4 threads and turned into (alpha, beta).  INT8 outlier group: the
// codes are copied, (alpha, beta) = (s_a, 0).
__device__ __forceinline__ uint32_t nib_to_sm(uint32_t n) {
  // n: 4 bytes, each a two's-complement nibble in its low 4 bits
  const uint32_t neg = (n >> 3) & 0x01010101u;            // 1 per negative byte
  const uint32_t mag = (n ^ (neg * 0x0Fu)) + neg;         // |q| (16 - n for negatives)
  return (mag & 0x0F0F0F0Fu) | (neg << 7);
}
__device__ __forceinline__ int nib_sum(uint32_t n) {     // sum of 4 two's-complement nibbles
  int s = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int v = static_cast<int>((n >> (8 * b)) & 0xFu);
    s += v >= 8 ? v - 16 : v;
  }
  return s;
}

__global__ void __launch_bounds__(256)
expand_activations_kernel(const uint8_t* __restrict__ q4, const int8_t* __restrict__ q8,
                          const float* __restrict__ scales, int64_t M, int64_t Mp, int G, int G4,
                          uint8_t* __restrict__ af8, float* __restrict__ ab) {
  griddep_wait();
  griddep_launch();
  const int64_t K = static_cast<int64_t>(G) * 128;
  const int64_t nchunks = M * G * 4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nchunks;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i & 3);
    const int64_t mg = i >> 2;
    const int t = static_cast<int>(mg % G);
    const int64_t m = mg / G;
    int s = 0;
    if (t < G4) {
      const uint4 v = *reinterpret_cast<const uint4*>(q4 + m * (static_cast<int64_t>(G4) * 64) +
                                                      t * 64 + c * 16);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
      uint32_t lo[4], hi[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        lo[j] = w[j] & 0x0F0F0F0Fu;
        hi[j] = (w[j] >> 4) & 0x0F0F0F0Fu;
        s += nib_sum(lo[j]) + nib_sum(hi[j]);
      }
      uint8_t* dst = af8 + m * K + t * 128 + c * 32;
      *reinterpret_cast<uint4*>(dst) =
          make_uint4(nib_to_sm(lo[0]), nib_to_sm(lo[1]), nib_to_sm(lo[2]), nib_to_sm(lo[3]));
      *reinterpret_cast<uint4*>(dst + 16) =
          make_uint4(nib_to_sm(hi[0]), nib_to_sm(hi[1]), nib_to_sm(hi[2]), nib_to_sm(hi[3]));
    } else {
      const uint4 v = *reinterpret_cast<const uint4*>(q8 + m * 128 + c * 32);
      const uint4 v2 = *reinterpret_cast<const uint4*>(q8 + m * 128 + c * 32 + 16);
      uint8_t* dst = af8 + m * K + t * 128 + c * 32;
      *reinterpret_cast<uint4*>(dst) = v;
      *reinterpret_cast<uint4*>(dst + 16) = v2;
    }
    // all 4 threads of a group are consecutive lanes of one warp (4 | 32)
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    if (c == 0) {
      const float sa = scales[static_cast<int64_t>(t) * M + m];
      const int64_t r = m & 31;
      const int64_t pos = (m - r) + 4 * (r & 7) + (r >> 3);     // a_ab row order
      float2 v;
      if (t < G4) v = make_float2(sa * 262144.0f, __fmul_rn(static_cast<float>(-8 * s), sa));
      else v = make_float2(sa, 0.0f);
      reinterpret_cast<float2*>(ab)[static_cast<int64_t>(t) * Mp + pos] = v;
    }
  }
}

// w_scales [G][N] -> w_sp: within every 128 channels, channel 8k + 2c + b (k < 16, c < 4,
// b < 2) moves to 32 (k / 4) + 8c + 2 (k % 4) + b: the 4 pairs k = 4i..4i+3 of the epilogue
// thread with lane % 4 = c are 32 contiguous bytes, and the 4 threads c = 0..3 read one line.
__global__ void __launch_bounds__(256)
prepare_w_scales_kernel(const float* __restrict__ ws, int64_t total, float* __restrict__ wsp) {
  griddep_wait();
  griddep_launch();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t nl = i & 127, k = nl >> 3;
    wsp[(i - nl) + 32 * (k >> 2) + 8 * ((nl & 7) >> 1) + 2 * (k & 3) + (nl & 1)] = ws[i];
  }
}

cudaError_t launch_prepare_w_scales(const float* w_scales, int64_t G, int64_t N, float* w_sp,
                                    cudaStream_t stream, int num_sms) {
  const int64_t total = G * N;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 8LL * num_sms) blocks = 8LL * num_sms;
  return launch_pdl(prepare_w_scales_kernel, dim3(static_cast<unsigned>(blocks)), dim3(256), 0,
                    stream, w_scales, total, w_sp);
}

// ---------------------------------------------------------------------------------------------
// host side: tensor maps + launch
// ---------------------------------------------------------------------------------------------
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// Resolved once, thread-safely (function-local static initialisation).
static PFN_encodeTiled get_encode_fn() {
  static const PFN_encodeTiled fn = []() -> PFN_encodeTiled {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_encodeTiled>(ptr);
    return nullptr;
  }();
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

// cudaFuncSetAttribute once per (device, kernel instantiation).
template <int kBT, bool kDebug>
static cudaError_t set_smem_attr(size_t smem) {
  constexpr int kMaxDev = 64;
  static std::once_flag once[kMaxDev];
  static cudaError_t err[kMaxDev];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDev) return cudaErrorInvalidDevice;
  std::call_once(once[dev], [&]() {
    err[dev] = cudaFuncSetAttribute(w4a4_gemm_kernel<kBT, kDebug>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem));
  });
  return err[dev];
}

// Tile plan: one persistent CTA per SM (or per unit, if fewer); whole tiles in round-robin waves
// while at least two waves remain, then the rest as evenly divided (tile, group) units.
// Small M (<= ATOM_SWAP_MAX_M = 64 tokens) takes the swap-AB tile of kBT = 16 / 32 / 64 tokens x
// 128 channels (at M = 128, two 64-token tiles measured mixed in the L2-cold sweep: down
// projection 45 -> 41 us, up/gate 39 -> 43 us; not used).
GemmPlan plan_w4a4_gemm(int64_t M, int64_t N, int64_t K, int num_sms, bool split_free) {
  GemmPlan pl;
  const int64_t G = K / 128;
  pl.bt = M <= 16 ? 16 : M <= 32 ? 32 : M <= ATOM_SWAP_MAX_M ? 64 : 0;
  pl.tile_m = pl.bt ? pl.bt : 128;
  pl.tile_n = pl.bt ? 128 : 256;
  pl.num_tiles = ((N + pl.tile_n - 1) / pl.tile_n) * ((M + pl.tile_m - 1) / pl.tile_m);
  if (split_free) {   // every tile by one CTA over all of K: the same fp32 chain for any shape
    pl.grid = static_cast<int>(pl.num_tiles < num_sms ? pl.num_tiles : num_sms);
    pl.dp_waves = static_cast<int>((pl.num_tiles + pl.grid - 1) / pl.grid);
    pl.sk_units = 0;
    return pl;
  }
  const int64_t units = pl.num_tiles * G;
  pl.grid = static_cast<int>(units < num_sms ? units : num_sms);
  // fewer tiles than SMs: a grid of a whole multiple of the tile count (when it keeps >= 85% of
  // the SMs), so every tile is cut into the same number of equal K segments -- each segment then
  // has one publisher role or one reducer role instead of straddling two tiles (cfg2 23.4 ->
  // 20.6 us, M = 128 up/gate 24.9 -> 22.3 us, graph-replayed)
  if (!split_free && pl.num_tiles < num_sms && pl.num_tiles * G >= num_sms) {
    const int64_t even = pl.num_tiles * (num_sms / pl.num_tiles);
    if (even * 100 >= 85LL * num_sms) pl.grid = static_cast<int>(even);
  }
  const int64_t T = pl.num_tiles, P = pl.grid;
  if (T % P == 0) pl.dp_waves = static_cast<int>(T / P);
  else if (T >= 2 * P) pl.dp_waves = static_cast<int>(T / P - 1);
  // (one data-parallel wave for P <= T < 2P measured slower: cfg4 63.1 -> 65.5 us)
  else pl.dp_waves = 0;
  pl.sk_units = (T - static_cast<int64_t>(pl.dp_waves) * P) * G;
  bool split = false;
  for (int64_t i = 1; i < P && !split && pl.sk_units > 0; ++i)
    split = (i * pl.sk_units / P) % G != 0;
  if (split) {
    // counters are indexed by the reducing CTA, so their region has the same size and place
    // for every shape on this device (only it must stay zero between calls)
    pl.counter_bytes = ((num_sms * sizeof(int) + 255) / 256) * 256;
    pl.workspace_bytes = pl.counter_bytes + pl.grid * kSlotFloats * sizeof(float);
  }
  return pl;
}

int64_t ab_rows(int64_t M) { return ((M + 127) / 128) * 128; }

size_t expand_bytes(int64_t M, int64_t K) {
  const size_t f8 = ((static_cast<size_t>(M) * K + 255) / 256) * 256;
  return f8 + static_cast<size_t>(ab_rows(M)) * (K / 128) * 8;
}

cudaError_t launch_expand_activations(const uint8_t* q4, const int8_t* q8, const float* scales,
                                      int64_t M, int64_t K, int32_t k_outlier, uint8_t* af8,
                                      float* ab, cudaStream_t stream, int num_sms) {
  const int G = static_cast<int>(K / 128), G4 = static_cast<int>((K - k_outlier) / 128);
  const int64_t threads = M * G * 4;
  int64_t blocks = (threads + 255) / 256;
  if (blocks > 8LL * num_sms) blocks = 8LL * num_sms;
  return launch_pdl(expand_activations_kernel, dim3(static_cast<unsigned>(blocks)), dim3(256), 0,
                    stream, q4, q8, scales, M, ab_rows(M), G, G4, af8, ab);
}

cudaError_t launch_w4a4_gemm(const GemmArgs& a, void* workspace, size_t workspace_bytes,
                             cudaStream_t stream, int num_sms, int* launches) {
  *launches = 0;
  if (a.M == 0) return cudaSuccess;
  const GemmPlan plan = plan_w4a4_gemm(a.M, a.N, a.K, num_sms, a.split_free != 0);
  if (workspace_bytes < plan.workspace_bytes) return cudaErrorInvalidValue;
  const int M = static_cast<int>(a.M), N = static_cast<int>(a.N), K = static_cast<int>(a.K);
  const int k_o = a.k_outlier;
  const uint64_t kp = static_cast<uint64_t>(K - k_o) / 2;
  CUtensorMap m_wq4, m_wq8, m_af8;
  // A map is always encoded (a valid descriptor is required as a kernel parameter); an unused
  // INT4 or INT8 weight map aliases the other one and is never read.
  const void* w4 = kp ? static_cast<const void*>(a.w_q4) : static_cast<const void*>(a.w_q8);
  const void* w8 = k_o ? static_cast<const void*>(a.w_q8) : static_cast<const void*>(a.w_q4);
  const uint64_t c4 = kp ? kp : 128, c8 = k_o ? 128 : kp;
  const uint32_t tn = static_cast<uint32_t>(plan.tile_n), tt = static_cast<uint32_t>(plan.tile_m);
  if (!make_map_u8(&m_wq4, w4, c4, N, 64, tn, CU_TENSOR_MAP_SWIZZLE_NONE) ||
      !make_map_u8(&m_wq8, w8, c8, N, 64, tn, CU_TENSOR_MAP_SWIZZLE_NONE) ||
      !make_map_u8(&m_af8, a.a_f8, K, M, 128, tt, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;

  GemmParams p;
  p.a_ab = a.a_ab;
  p.Mp = static_cast<int>(ab_rows(a.M));
  p.w_sp = a.w_sp;
  p.c = a.c;
  p.ldc = a.ldc;
  p.debug = a.debug_partials;
  p.M = M;
  p.N = N;
  p.G = K / 128;
  p.G4 = (K - k_o) / 128;
  p.c_f32 = a.c_f32;
  p.m_tiles = (M + plan.tile_m - 1) / plan.tile_m;
  p.num_tiles = static_cast<int>(plan.num_tiles);
  p.dp_waves = plan.dp_waves;
  p.sk_base = static_cast<int64_t>(plan.dp_waves) * plan.grid * p.G;
  p.sk_units = plan.sk_units;
  p.counters = nullptr;
  p.partials = nullptr;
  if (plan.workspace_bytes > 0) {
    p.counters = static_cast<int*>(workspace);
    p.partials = reinterpret_cast<float*>(static_cast<char*>(workspace) + plan.counter_bytes);
  }

#ifdef ATOM_DEV_PROBES
  static long long* trace = nullptr;
  static const bool want_trace = std::getenv("ATOM_GEMM_TRACE") != nullptr;
  constexpr size_t kTraceBytes = static_cast<size_t>(kTraceEv) * kTraceN * sizeof(long long);
  if (want_trace && trace == nullptr) cudaMalloc(&trace, kTraceBytes);
  p.trace = want_trace ? trace : nullptr;
  if (want_trace) cudaMemsetAsync(trace, 0, kTraceBytes, stream);
#endif
  auto go = [&](auto bt_tag, auto dbg_tag) {
    constexpr int kBT = decltype(bt_tag)::value;
    constexpr bool kDbg = decltype(dbg_tag)::value;
    const size_t smem = sizeof(GemmSmem<TileCfg<kBT>>) + 1024;
    cudaError_t err = set_smem_attr<kBT, kDbg>(smem);
    if (err != cudaSuccess) return err;
    return launch_pdl(w4a4_gemm_kernel<kBT, kDbg>, dim3(plan.grid), dim3(kThreads), smem, stream,
                      m_wq4, m_wq8, m_af8, p);
  };
  auto go_bt = [&](auto dbg_tag) {
    switch (plan.bt) {
      case 16: return go(std::integral_constant<int, 16>{}, dbg_tag);
      case 32: return go(std::integral_constant<int, 32>{}, dbg_tag);
      case 64: return go(std::integral_constant<int, 64>{}, dbg_tag);
      default: return go(std::integral_constant<int, 0>{}, dbg_tag);
    }
  };
  const cudaError_t e = p.debug ? go_bt(std::true_type{}) : go_bt(std::false_type{});
  if (e != cudaSuccess) return e;
  ++*launches;
#ifdef ATOM_DEV_PROBES
  if (want_trace) {
    static long long h[kTraceEv * kTraceN];
    cudaMemcpy(h, trace, sizeof(h), cudaMemcpyDeviceToHost);
    std::fprintf(stderr, "plan grid=%d dp_waves=%d sk_units=%lld\n", plan.grid, plan.dp_waves,
                 static_cast<long long>(plan.sk_units));
    std::fprintf(stderr, "g  W_tma A_tma unp_start unp_done mma_issue mma_done epi_start epi_release epi_end\n");
    {
      long long s0 = -1, s1 = 0, e0 = -1, e1 = 0;
      for (int b = 0; b < plan.grid && b < kTraceN; ++b) {
        const long long a = h[25 * kTraceN + b], z = h[26 * kTraceN + b];
        if (s0 < 0 || a < s0) s0 = a;
        if (a > s1) s1 = a;
        if (e0 < 0 || z < e0) e0 = z;
        if (z > e1) e1 = z;
      }
      std::fprintf(stderr, "CTA globaltimer ns: start spread %lld, end first %lld last %lld\n",
                   s1 - s0, e0 - s0, e1 - s0);
      for (int b = 0; b < plan.grid && b < kTraceN; b += 4)
        std::fprintf(stderr, "  cta %3d start %6lld end %6lld published %6lld red_wait %6lld..%6lld nseg %lld\n",
                     b, h[25 * kTraceN + b] - s0, h[26 * kTraceN + b] - s0,
                     h[30 * kTraceN + b] ? h[30 * kTraceN + b] - s0 : -1,
                     h[27 * kTraceN + b] ? h[27 * kTraceN + b] - s0 : -1,
                     h[28 * kTraceN + b] ? h[28 * kTraceN + b] - s0 : -1, h[29 * kTraceN + b]);
    }
    const long long t0 = h[3 * kTraceN];
    for (int g = 0; g < kTraceN; ++g) {
      if (h[3 * kTraceN + g] == 0) break;
      if (g > 40 && g % 4 != 0) continue;
      std::fprintf(stderr, "%3d %8lld %8lld %8lld %8lld %8lld %8lld %8lld %8lld %8lld |", g,
                   h[g] - t0, h[kTraceN + g] - t0, h[2 * kTraceN + g] - t0,
                   h[4 * kTraceN + g] - t0, h[3 * kTraceN + g] - t0, h[8 * kTraceN + g] - t0,
                   h[5 * kTraceN + g] - t0, h[6 * kTraceN + g] - t0, h[7 * kTraceN + g] - t0);
      for (int e = 0; e < 8; ++e)
        std::fprintf(stderr, " %lld/%lld", h[(17 + e) * kTraceN + g] - t0,
                     h[(9 + e) * kTraceN + g] - t0);
      std::fprintf(stderr, "\n");
    }
  }
#endif
  return cudaGetLastError();
}

}  // namespace atom
