// internal.h -- launchers shared between the kernel translation units and the C-ABI layer.
#pragma once
#include <cstddef>
#include <cstdint>
#include <utility>
#include <cuda.h>
#include <cuda_runtime.h>

namespace atom {

// Launch with programmatic stream serialization (PDL): the kernel may be scheduled while the
// previous kernel of the stream is finishing; every kernel of this library calls griddep_wait()
// before touching global memory another kernel may write, so the semantics are those of a plain
// launch.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t stream, Args&&... args) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

cudaError_t launch_reorder_quantize(const void* x, int64_t rows, int64_t ldx,
                                    const int32_t* perm, int64_t K, int32_t k_outlier,
                                    float clip4, float clip8, uint8_t* q4, int8_t* q8,
                                    uint8_t* af8, float* ab, float* scales, float* wsp,
                                    cudaStream_t stream, int num_sms,
                                    const void* gamma = nullptr, float eps = 0.0f,
                                    const void* up = nullptr);

cudaError_t launch_validate_perm(const int32_t* perm, int64_t K, int64_t ldx, int32_t* scratch,
                                 int32_t* ok, cudaStream_t stream);

struct GemmArgs {
  const uint8_t* a_f8;      // activation operand form (include/atom.h "a_f8", "a_ab")
  const float* a_ab;
  const uint8_t* w_q4;
  const int8_t* w_q8;
  const float* w_sp;        // weight scales in the GEMM channel order (include/atom.h "w_sp")
  int64_t M, N, K;
  int32_t k_outlier;
  void* c;
  int64_t ldc;
  int c_f32;
  int32_t* debug_partials;
  int split_free;           // ATOM_GEMM_SPLIT_FREE: no K-split of any output tile
};

struct GemmPlan {
  int grid = 0;                 // persistent CTAs (<= SMs)
  int dp_waves = 0;             // whole-tile round-robin waves
  int64_t sk_units = 0;         // (tile, group) units divided evenly after the waves
  int64_t num_tiles = 0;
  int bt = 0;                   // 0: 128-token x 256-channel tiles; 16/32/64: swap-AB small-M tiles
  int tile_m = 128, tile_n = 256;   // tokens / channels per tile
  size_t counter_bytes = 0;
  size_t workspace_bytes = 0;   // 0 when no tile is split between CTAs
};

GemmPlan plan_w4a4_gemm(int64_t M, int64_t N, int64_t K, int num_sms, bool split_free = false);

// Rows of a_ab per group: M rounded up to a multiple of 128.
int64_t ab_rows(int64_t M);

// Bytes of workspace the canonical entry needs for a_f8 + a_ab (after the GEMM's own part).
size_t expand_bytes(int64_t M, int64_t K);

cudaError_t launch_expand_activations(const uint8_t* q4, const int8_t* q8, const float* scales,
                                      int64_t M, int64_t K, int32_t k_outlier, uint8_t* af8,
                                      float* ab, cudaStream_t stream, int num_sms);

// w_scales [G][N] -> w_sp (the GEMM's channel order), for atom_w4a4_gemm.
cudaError_t launch_prepare_w_scales(const float* w_scales, int64_t G, int64_t N, float* w_sp,
                                    cudaStream_t stream, int num_sms);

// Returns the number of kernel launches issued through *launches.
cudaError_t launch_w4a4_gemm(const GemmArgs& a, void* workspace, size_t workspace_bytes,
                             cudaStream_t stream, int num_sms, int* launches);

// NEXT-2, Atom (FP) on the MX format (mxfp.cu, include/atom.h "Atom (FP)")
cudaError_t launch_mx_reorder_quantize(const void* x, int64_t rows, int64_t ldx,
                                       const int32_t* perm, int64_t K, int32_t k_outlier,
                                       uint8_t* fp4, uint8_t* fp8, uint8_t* sf, int64_t ldsf,
                                       cudaStream_t stream, int num_sms);

struct MxGemmArgs {
  const uint8_t* a_fp4;
  const uint8_t* a_fp8;
  const uint8_t* a_sf;
  int64_t lda_sf;
  const uint8_t* w_fp4;
  const uint8_t* w_fp8;
  const uint8_t* w_sf;
  int64_t ldw_sf;
  int64_t M, N, K;
  int32_t k_outlier;
  void* c;
  int64_t ldc;
  void* workspace;          // split-K partials (mx_gemm_workspace_bytes)
  size_t workspace_bytes;
};
cudaError_t launch_mx_gemm(const MxGemmArgs& a, cudaStream_t stream, int num_sms);
size_t mx_gemm_workspace_bytes(int64_t M, int64_t N, int64_t K, int32_t k_outlier, int num_sms);
int mx_gemm_launches(int64_t M, int64_t N, int64_t K, int32_t k_outlier, int num_sms);

// NEXT-3: quantized paged KV cache + decode attention (kvcache.cu, include/atom.h "KV cache")
cudaError_t launch_kv_quantize(const void* x, int64_t T, int64_t ldx, int32_t H,
                               const int32_t* slots, uint8_t* codes, float* params,
                               cudaStream_t stream, int num_sms);
cudaError_t launch_decode_attention(const void* q, int64_t B, int32_t H, const uint8_t* kc,
                                    const float* kp, const uint8_t* vc, const float* vp,
                                    const int32_t* block_table, int64_t max_pages,
                                    const int32_t* seq_lens, int32_t max_seq_len, float* out,
                                    float* workspace, cudaStream_t stream, int num_sms,
                                    int* launches);
size_t decode_attention_workspace_bytes(int64_t B, int32_t H, int32_t max_seq_len, int num_sms);

}  // namespace atom
