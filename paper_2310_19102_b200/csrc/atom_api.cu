// atom_api.cu -- the C ABI (include/atom.h): host-side validation, device checks, launches.
//
// Nothing here computes the method; it validates arguments exactly as documented in atom.h
// (SPEC S:152 / S:283 "shape error" conventions), then calls the launchers in quantize.cu and
// gemm.cu on the caller's stream.  No allocation, no synchronization, no exceptions.
#include <cstdint>
#include <cuda_runtime.h>
#include <mutex>

#include "atom.h"
#include "internal.h"

namespace {

thread_local int g_last_launches = 0;

struct DeviceInfo {
  bool ok = false;
  bool is_sm100 = false;
  int num_sms = 0;
};

constexpr int kMaxDevices = 64;
DeviceInfo g_dev[kMaxDevices];
std::once_flag g_dev_once[kMaxDevices];

// Per-device attribute cache (the only global state; initialised once per device).
atom_status_t current_device(DeviceInfo* out) {
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return ATOM_ERR_CUDA;
  std::call_once(g_dev_once[dev], [dev]() {
    int major = 0, minor = 0, sms = 0;
    DeviceInfo d;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess) {
      d.ok = true;
      d.is_sm100 = (major == 10 && minor == 0);
      d.num_sms = sms;
    }
    g_dev[dev] = d;
  });
  *out = g_dev[dev];
  if (!out->ok) return ATOM_ERR_CUDA;
  if (!out->is_sm100) return ATOM_ERR_UNSUPPORTED;
  return ATOM_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

bool clip_ok(float c) { return c > 0.0f && c <= 1.0f; }

atom_status_t check_quant_args(const void* x, int64_t rows, int64_t ld, const int32_t* perm,
                               int64_t K, int32_t k_o, float clip4, float clip8,
                               const uint8_t* q4, const int8_t* q8, const uint8_t* af8,
                               const float* ab, const float* scales, bool packed_required) {
  if (rows < 0) return ATOM_ERR_SHAPE;
  if (!(k_o == 0 || k_o == ATOM_GROUP)) return ATOM_ERR_ARG;
  if (K <= 0 || K % ATOM_GROUP != 0 || K < k_o) return ATOM_ERR_SHAPE;
  if (!clip_ok(clip4) || !clip_ok(clip8)) return ATOM_ERR_ARG;
  if (rows > 0x7fffffffLL || K > (1LL << 30)) return ATOM_ERR_SHAPE;
  if (ld <= 0 || ld % 8 != 0 || ld > (1LL << 30)) return ATOM_ERR_SHAPE;
  if (ld * 2 > 227 * 1024) return ATOM_ERR_SHAPE;  // the source row is staged in shared memory
  if (rows == 0) return ATOM_OK;
  if (!x || !perm || !scales) return ATOM_ERR_NULL;
  // forbidden outputs: q4 without INT4 groups, q8 without the outlier block
  if ((K == k_o && q4 != nullptr) || (k_o == 0 && q8 != nullptr)) return ATOM_ERR_NULL;
  if (packed_required) {
    if ((K > k_o) != (q4 != nullptr) || (k_o > 0) != (q8 != nullptr)) return ATOM_ERR_NULL;
  } else if (!q4 && !q8 && !af8) {
    return ATOM_ERR_NULL;
  }
  if ((af8 == nullptr) != (ab == nullptr)) return ATOM_ERR_NULL;   // the operand form is a pair
  if (!aligned16(x) || !aligned16(perm) || !aligned16(scales) || (q4 && !aligned16(q4)) ||
      (q8 && !aligned16(q8)) || (af8 && !aligned16(af8)) || (ab && !aligned16(ab)))
    return ATOM_ERR_ALIGN;
  return ATOM_OK;
}

atom_status_t quantize_common(const void* x, int64_t rows, int64_t ld, const int32_t* perm,
                              int64_t K, int32_t k_o, float clip4, float clip8, uint8_t* q4,
                              int8_t* q8, uint8_t* af8, float* ab, float* scales,
                              bool packed_required,
                              void* stream, const void* gamma = nullptr, float eps = 0.0f,
                              const void* up = nullptr, float* wsp = nullptr) {
  g_last_launches = 0;
  atom_status_t st = check_quant_args(x, rows, ld, perm, K, k_o, clip4, clip8, q4, q8, af8, ab,
                                      scales, packed_required);
  if (st != ATOM_OK || rows == 0) return st;
  DeviceInfo dev;
  if ((st = current_device(&dev)) != ATOM_OK) return st;
  cudaError_t e = atom::launch_reorder_quantize(x, rows, ld, perm, K, k_o, clip4, clip8, q4, q8,
                                                af8, ab, scales, wsp,
                                                static_cast<cudaStream_t>(stream), dev.num_sms,
                                                gamma, eps, up);
  if (e != cudaSuccess) return ATOM_ERR_CUDA;
  g_last_launches = 1;
  return ATOM_OK;
}

size_t counter_region(int num_sms) {
  return ((static_cast<size_t>(num_sms) * sizeof(int) + 255) / 256) * 256;
}

// The GEMM's own workspace part (counters + split-tile slots), rounded so the canonical entry's
// operand area that follows it starts 256-byte aligned; at least the counter region, so one
// buffer serves both entries.
size_t gemm_part_bytes(const atom::GemmPlan& pl, int num_sms) {
  const size_t b = pl.workspace_bytes > 0 ? pl.workspace_bytes : counter_region(num_sms);
  return ((b + 255) / 256) * 256;
}

atom_status_t check_gemm_args(const uint8_t* w_q4, const int8_t* w_q8, const float* w_scales,
                              int64_t M, int64_t N, int64_t K, int32_t k_outlier, const void* c,
                              int64_t ldc, atom_dtype_t c_dtype, const int32_t* debug_partials) {
  if (M < 0 || N <= 0 || N % 128 != 0) return ATOM_ERR_SHAPE;
  if (!(k_outlier == 0 || k_outlier == ATOM_GROUP)) return ATOM_ERR_ARG;
  if (K <= 0 || K % ATOM_GROUP != 0 || K < k_outlier) return ATOM_ERR_SHAPE;
  if (M > 0x7fffffffLL || N > 0x7fffffffLL || K > (1LL << 30)) return ATOM_ERR_SHAPE;
  if (ldc < N || ldc % 8 != 0) return ATOM_ERR_SHAPE;
  if (!(c_dtype == ATOM_F16 || c_dtype == ATOM_F32)) return ATOM_ERR_ARG;
  if (M == 0) return ATOM_OK;
  if (!w_scales || !c) return ATOM_ERR_NULL;
  const bool has4 = K > k_outlier, has8 = k_outlier > 0;
  if (has4 != (w_q4 != nullptr)) return ATOM_ERR_NULL;
  if (has8 != (w_q8 != nullptr)) return ATOM_ERR_NULL;
  if (!aligned16(w_scales) || !aligned16(c) ||
      (w_q4 && !aligned16(w_q4)) || (w_q8 && !aligned16(w_q8)) ||
      (debug_partials && !aligned16(debug_partials)))
    return ATOM_ERR_ALIGN;
  return ATOM_OK;
}

cudaError_t run_gemm(const uint8_t* af8, const float* ab, const uint8_t* w_q4,
                     const int8_t* w_q8, const float* w_sp, int64_t M,
                     int64_t N, int64_t K, int32_t k_outlier, void* c, int64_t ldc,
                     atom_dtype_t c_dtype, int32_t* debug_partials, void* workspace,
                     size_t workspace_bytes, void* stream, const DeviceInfo& dev, int* launches,
                     int split_free = 0) {
  atom::GemmArgs a;
  a.a_f8 = af8;
  a.a_ab = ab;
  a.w_q4 = w_q4;
  a.w_q8 = w_q8;
  a.w_sp = w_sp;
  a.M = M;
  a.N = N;
  a.K = K;
  a.k_outlier = k_outlier;
  a.c = c;
  a.ldc = ldc;
  a.c_f32 = c_dtype == ATOM_F32;
  a.debug_partials = debug_partials;
  a.split_free = split_free;
  return atom::launch_w4a4_gemm(a, workspace, workspace_bytes, static_cast<cudaStream_t>(stream),
                                dev.num_sms, launches);
}

}  // namespace

extern "C" {

atom_status_t atom_reorder_quantize(const void* x_f16, int64_t M, int64_t ldx,
                                    const int32_t* perm, int64_t K, int32_t k_outlier,
                                    float clip_int4, float clip_int8, uint8_t* q4, int8_t* q8,
                                    uint8_t* a_f8, float* a_ab, float* scales, void* stream) {
  return quantize_common(x_f16, M, ldx, perm, K, k_outlier, clip_int4, clip_int8, q4, q8, a_f8,
                         a_ab, scales, false, stream);
}

atom_status_t atom_rmsnorm_reorder_quantize(const void* x_f16, int64_t M, int64_t ldx,
                                            const void* gamma_f16, float eps,
                                            const int32_t* perm, int64_t K, int32_t k_outlier,
                                            float clip_int4, float clip_int8, uint8_t* q4,
                                            int8_t* q8, uint8_t* a_f8, float* a_ab,
                                            float* scales, void* stream) {
  g_last_launches = 0;
  if (!(eps >= 0.0f)) return ATOM_ERR_ARG;
  if (M > 0 && !gamma_f16) return ATOM_ERR_NULL;
  if (gamma_f16 && !aligned16(gamma_f16)) return ATOM_ERR_ALIGN;
  return quantize_common(x_f16, M, ldx, perm, K, k_outlier, clip_int4, clip_int8, q4, q8, a_f8,
                         a_ab, scales, false, stream, gamma_f16, eps);
}

atom_status_t atom_silu_mul_reorder_quantize(const void* gate_f16, const void* up_f16, int64_t M,
                                             int64_t ldx, const int32_t* perm, int64_t K,
                                             int32_t k_outlier, float clip_int4, float clip_int8,
                                             uint8_t* q4, int8_t* q8, uint8_t* a_f8,
                                             float* a_ab, float* scales, void* stream) {
  g_last_launches = 0;
  if (M > 0 && !up_f16) return ATOM_ERR_NULL;
  if (up_f16 && !aligned16(up_f16)) return ATOM_ERR_ALIGN;
  return quantize_common(gate_f16, M, ldx, perm, K, k_outlier, clip_int4, clip_int8, q4, q8, a_f8,
                         a_ab, scales, false, stream, nullptr, 0.0f, up_f16);
}

atom_status_t atom_quantize_weights(const void* w_f16, int64_t N, int64_t ldw,
                                    const int32_t* perm, int64_t K, int32_t k_outlier,
                                    float clip_int4, float clip_int8, uint8_t* q4, int8_t* q8,
                                    float* scales, float* w_sp, void* stream) {
  g_last_launches = 0;
  if (w_sp && N % 128 != 0) return ATOM_ERR_SHAPE;
  if (w_sp && !aligned16(w_sp)) return ATOM_ERR_ALIGN;
  return quantize_common(w_f16, N, ldw, perm, K, k_outlier, clip_int4, clip_int8, q4, q8, nullptr,
                         nullptr, scales, true, stream, nullptr, 0.0f, nullptr, w_sp);
}

size_t atom_w4a4_gemm_workspace_size(int64_t M, int64_t N, int64_t K, int32_t k_outlier) {
  (void)k_outlier;
  if (M <= 0 || N <= 0 || N % 128 != 0 || K <= 0 || K % ATOM_GROUP != 0) return 0;
  DeviceInfo dev;
  if (current_device(&dev) != ATOM_OK) return 0;   // no sm_100 device: the GEMM cannot run
  const atom::GemmPlan pl = atom::plan_w4a4_gemm(M, N, K, dev.num_sms);
  return gemm_part_bytes(pl, dev.num_sms) + atom::expand_bytes(M, K) +
         static_cast<size_t>(N) * (K / ATOM_GROUP) * sizeof(float);
}

size_t atom_w4a4_gemm_f8_workspace_size(int64_t M, int64_t N, int64_t K, int32_t k_outlier) {
  (void)k_outlier;
  if (M <= 0 || N <= 0 || N % 128 != 0 || K <= 0 || K % ATOM_GROUP != 0) return 0;
  DeviceInfo dev;
  if (current_device(&dev) != ATOM_OK) return 0;
  return atom::plan_w4a4_gemm(M, N, K, dev.num_sms).workspace_bytes;
}

size_t atom_w4a4_gemm_counter_bytes(void) {
  DeviceInfo dev;
  if (current_device(&dev) != ATOM_OK) return 0;
  return counter_region(dev.num_sms);
}

atom_status_t atom_w4a4_gemm_f8(const uint8_t* a_f8, const float* a_ab, const uint8_t* w_q4,
                                const int8_t* w_q8, const float* w_sp, int64_t M, int64_t N,
                                int64_t K, int32_t k_outlier, void* c, int64_t ldc,
                                atom_dtype_t c_dtype, int32_t* debug_partials, int32_t flags,
                                void* workspace, size_t workspace_bytes, void* stream) {
  g_last_launches = 0;
  atom_status_t st = check_gemm_args(w_q4, w_q8, w_sp, M, N, K, k_outlier, c, ldc, c_dtype,
                                     debug_partials);
  if (st != ATOM_OK || M == 0) return st;
  if ((flags & ~ATOM_GEMM_SPLIT_FREE) != 0) return ATOM_ERR_ARG;
  if (!a_f8 || !a_ab) return ATOM_ERR_NULL;
  if (!aligned16(a_f8) || !aligned16(a_ab)) return ATOM_ERR_ALIGN;
  DeviceInfo dev;
  if ((st = current_device(&dev)) != ATOM_OK) return st;
  const bool split_free = (flags & ATOM_GEMM_SPLIT_FREE) != 0;
  const size_t ws = atom::plan_w4a4_gemm(M, N, K, dev.num_sms, split_free).workspace_bytes;
  if (ws > 0 && (workspace == nullptr || workspace_bytes < ws || !aligned16(workspace)))
    return ATOM_ERR_WORKSPACE;
  int launches = 0;
  if (run_gemm(a_f8, a_ab, w_q4, w_q8, w_sp, M, N, K, k_outlier, c, ldc, c_dtype,
               debug_partials, workspace, workspace_bytes, stream, dev, &launches,
               split_free ? 1 : 0) != cudaSuccess)
    return ATOM_ERR_CUDA;
  g_last_launches = launches;
  return ATOM_OK;
}

atom_status_t atom_w4a4_gemm(const uint8_t* a_q4, const int8_t* a_q8, const float* a_scales,
                             const uint8_t* w_q4, const int8_t* w_q8, const float* w_scales,
                             int64_t M, int64_t N, int64_t K, int32_t k_outlier, void* c,
                             int64_t ldc, atom_dtype_t c_dtype, int32_t* debug_partials,
                             void* workspace, size_t workspace_bytes, void* stream) {
  g_last_launches = 0;
  atom_status_t st = check_gemm_args(w_q4, w_q8, w_scales, M, N, K, k_outlier, c, ldc, c_dtype,
                                     debug_partials);
  if (st != ATOM_OK || M == 0) return st;
  if (!a_scales) return ATOM_ERR_NULL;
  if ((K > k_outlier) != (a_q4 != nullptr) || (k_outlier > 0) != (a_q8 != nullptr))
    return ATOM_ERR_NULL;
  if ((a_q4 && !aligned16(a_q4)) || (a_q8 && !aligned16(a_q8)) || !aligned16(a_scales))
    return ATOM_ERR_ALIGN;
  DeviceInfo dev;
  if ((st = current_device(&dev)) != ATOM_OK) return st;
  const atom::GemmPlan pl = atom::plan_w4a4_gemm(M, N, K, dev.num_sms);
  const size_t part = gemm_part_bytes(pl, dev.num_sms);
  const size_t exp = atom::expand_bytes(M, K);
  const size_t need = part + exp + static_cast<size_t>(N) * (K / ATOM_GROUP) * sizeof(float);
  if (workspace == nullptr || workspace_bytes < need || !aligned16(workspace))
    return ATOM_ERR_WORKSPACE;
  // the operand forms live after the GEMM's own part of the workspace
  uint8_t* af8 = static_cast<uint8_t*>(workspace) + part;
  float* ab = reinterpret_cast<float*>(af8 + ((static_cast<size_t>(M) * K + 255) / 256) * 256);
  float* wsp = reinterpret_cast<float*>(af8 + exp);
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (atom::launch_expand_activations(a_q4, a_q8, a_scales, M, K, k_outlier, af8, ab, s,
                                      dev.num_sms) != cudaSuccess ||
      atom::launch_prepare_w_scales(w_scales, K / ATOM_GROUP, N, wsp, s, dev.num_sms) !=
          cudaSuccess)
    return ATOM_ERR_CUDA;
  int launches = 0;
  if (run_gemm(af8, ab, w_q4, w_q8, wsp, M, N, K, k_outlier, c, ldc, c_dtype,
               debug_partials, workspace, part, stream, dev, &launches) != cudaSuccess)
    return ATOM_ERR_CUDA;
  g_last_launches = launches + 2;
  return ATOM_OK;
}

atom_status_t atom_mx_reorder_quantize(const void* x_f16, int64_t rows, int64_t ldx,
                                       const int32_t* perm, int64_t K, int32_t k_outlier,
                                       uint8_t* fp4, uint8_t* fp8, uint8_t* sf, int64_t ldsf,
                                       void* stream) {
  g_last_launches = 0;
  if (rows < 0) return ATOM_ERR_SHAPE;
  if (!(k_outlier == 0 || k_outlier == ATOM_GROUP)) return ATOM_ERR_ARG;
  if (K <= 0 || K % ATOM_GROUP != 0 || K < k_outlier || K > (1LL << 30)) return ATOM_ERR_SHAPE;
  if (rows > 0x7fffffffLL || ldx <= 0 || ldx % 8 != 0 || ldx * 2 > 227 * 1024)
    return ATOM_ERR_SHAPE;
  if (ldsf < K / 32 || ldsf % 16 != 0) return ATOM_ERR_SHAPE;
  if (rows == 0) return ATOM_OK;
  if (!x_f16 || !perm || !sf) return ATOM_ERR_NULL;
  if ((K > k_outlier) != (fp4 != nullptr) || (k_outlier > 0) != (fp8 != nullptr))
    return ATOM_ERR_NULL;
  if (!aligned16(x_f16) || !aligned16(perm) || !aligned16(sf) || (fp4 && !aligned16(fp4)) ||
      (fp8 && !aligned16(fp8)))
    return ATOM_ERR_ALIGN;
  DeviceInfo dev;
  atom_status_t st = current_device(&dev);
  if (st != ATOM_OK) return st;
  if (atom::launch_mx_reorder_quantize(x_f16, rows, ldx, perm, K, k_outlier, fp4, fp8, sf, ldsf,
                                       static_cast<cudaStream_t>(stream), dev.num_sms) !=
      cudaSuccess)
    return ATOM_ERR_CUDA;
  g_last_launches = 1;
  return ATOM_OK;
}

atom_status_t atom_mx_gemm(const uint8_t* a_fp4, const uint8_t* a_fp8, const uint8_t* a_sf,
                           int64_t lda_sf, const uint8_t* w_fp4, const uint8_t* w_fp8,
                           const uint8_t* w_sf, int64_t ldw_sf, int64_t M, int64_t N, int64_t K,
                           int32_t k_outlier, void* c_f16, int64_t ldc, void* workspace,
                           size_t workspace_bytes, void* stream) {
  g_last_launches = 0;
  if (M < 0 || N <= 0 || N % 128 != 0) return ATOM_ERR_SHAPE;
  if (!(k_outlier == 0 || k_outlier == ATOM_GROUP)) return ATOM_ERR_ARG;
  if (K <= 0 || K % ATOM_GROUP != 0 || K < k_outlier || K > (1LL << 30)) return ATOM_ERR_SHAPE;
  if (M > 0x7fffffffLL || N > 0x7fffffffLL || ldc < N || ldc % 8 != 0) return ATOM_ERR_SHAPE;
  if (lda_sf < K / 32 || lda_sf % 16 != 0 || ldw_sf < K / 32 || ldw_sf % 16 != 0)
    return ATOM_ERR_SHAPE;
  if (M == 0) return ATOM_OK;
  const bool has4 = K > k_outlier, has8 = k_outlier > 0;
  if (!a_sf || !w_sf || !c_f16 || has4 != (a_fp4 != nullptr) || has4 != (w_fp4 != nullptr) ||
      has8 != (a_fp8 != nullptr) || has8 != (w_fp8 != nullptr))
    return ATOM_ERR_NULL;
  if (!aligned16(a_sf) || !aligned16(w_sf) || !aligned16(c_f16) || (a_fp4 && !aligned16(a_fp4)) ||
      (w_fp4 && !aligned16(w_fp4)) || (a_fp8 && !aligned16(a_fp8)) || (w_fp8 && !aligned16(w_fp8)))
    return ATOM_ERR_ALIGN;
  DeviceInfo dev;
  atom_status_t st = current_device(&dev);
  if (st != ATOM_OK) return st;
  atom::MxGemmArgs a;
  a.a_fp4 = a_fp4;
  a.a_fp8 = a_fp8;
  a.a_sf = a_sf;
  a.lda_sf = lda_sf;
  a.w_fp4 = w_fp4;
  a.w_fp8 = w_fp8;
  a.w_sf = w_sf;
  a.ldw_sf = ldw_sf;
  a.M = M;
  a.N = N;
  a.K = K;
  a.k_outlier = k_outlier;
  a.c = c_f16;
  a.ldc = ldc;
  a.workspace = workspace;
  a.workspace_bytes = workspace_bytes;
  const size_t need = atom::mx_gemm_workspace_bytes(M, N, K, k_outlier, dev.num_sms);
  if (need > 0 && (!workspace || workspace_bytes < need || !aligned16(workspace)))
    return ATOM_ERR_WORKSPACE;
  if (atom::launch_mx_gemm(a, static_cast<cudaStream_t>(stream), dev.num_sms) != cudaSuccess)
    return ATOM_ERR_CUDA;
  g_last_launches = atom::mx_gemm_launches(M, N, K, k_outlier, dev.num_sms);
  return ATOM_OK;
}

size_t atom_mx_gemm_workspace_size(int64_t M, int64_t N, int64_t K, int32_t k_outlier) {
  if (M <= 0 || N <= 0 || N % 128 != 0 || K <= 0 || K % ATOM_GROUP != 0 || K < k_outlier)
    return 0;
  DeviceInfo dev;
  if (current_device(&dev) != ATOM_OK) return 0;
  return atom::mx_gemm_workspace_bytes(M, N, K, k_outlier, dev.num_sms);
}

atom_status_t atom_kv_quantize(const void* x_f16, int64_t T, int64_t ldx, int32_t H,
                               int32_t head_dim, const int32_t* slots, uint8_t* codes,
                               float* params, void* stream) {
  g_last_launches = 0;
  if (T < 0 || H <= 0 || head_dim != 128 || ldx < 128LL * H || ldx % 4 != 0) return ATOM_ERR_SHAPE;
  if (T == 0) return ATOM_OK;
  if (!x_f16 || !slots || !codes || !params) return ATOM_ERR_NULL;
  if (!aligned16(codes) || !aligned16(params) || (reinterpret_cast<uintptr_t>(x_f16) & 7u) ||
      (reinterpret_cast<uintptr_t>(slots) & 3u))
    return ATOM_ERR_ALIGN;
  DeviceInfo dev;
  atom_status_t st = current_device(&dev);
  if (st != ATOM_OK) return st;
  if (atom::launch_kv_quantize(x_f16, T, ldx, H, slots, codes, params,
                               static_cast<cudaStream_t>(stream), dev.num_sms) != cudaSuccess)
    return ATOM_ERR_CUDA;
  g_last_launches = 1;
  return ATOM_OK;
}

size_t atom_decode_attention_workspace_size(int64_t B, int32_t H, int32_t max_seq_len) {
  if (B <= 0 || H <= 0 || max_seq_len <= 0) return 0;
  DeviceInfo dev;
  if (current_device(&dev) != ATOM_OK) return 0;
  return atom::decode_attention_workspace_bytes(B, H, max_seq_len, dev.num_sms);
}

atom_status_t atom_decode_attention(const void* q_f16, int64_t B, int32_t H, int32_t head_dim,
                                    const uint8_t* k_codes, const float* k_params,
                                    const uint8_t* v_codes, const float* v_params,
                                    const int32_t* block_table, int64_t max_pages,
                                    const int32_t* seq_lens, int32_t max_seq_len, float* out,
                                    void* workspace, size_t workspace_bytes, void* stream) {
  g_last_launches = 0;
  if (B < 0 || H <= 0 || head_dim != 128 || max_pages <= 0 || max_seq_len <= 0 ||
      max_seq_len > 16 * max_pages || B * H > 0x7fffffffLL)
    return ATOM_ERR_SHAPE;
  if (B == 0) return ATOM_OK;
  if (!q_f16 || !k_codes || !k_params || !v_codes || !v_params || !block_table || !seq_lens ||
      !out)
    return ATOM_ERR_NULL;
  if (!aligned16(q_f16) || !aligned16(k_codes) || !aligned16(v_codes) || !aligned16(k_params) ||
      !aligned16(v_params) || !aligned16(out))
    return ATOM_ERR_ALIGN;
  DeviceInfo dev;
  atom_status_t st = current_device(&dev);
  if (st != ATOM_OK) return st;
  const size_t need = atom::decode_attention_workspace_bytes(B, H, max_seq_len, dev.num_sms);
  if (need > 0 && (!workspace || workspace_bytes < need || !aligned16(workspace)))
    return ATOM_ERR_WORKSPACE;
  int launches = 0;
  if (atom::launch_decode_attention(q_f16, B, H, k_codes, k_params, v_codes, v_params,
                                    block_table, max_pages, seq_lens, max_seq_len, out,
                                    static_cast<float*>(workspace),
                                    static_cast<cudaStream_t>(stream), dev.num_sms,
                                    &launches) != cudaSuccess)
    return ATOM_ERR_CUDA;
  g_last_launches = launches;
  return ATOM_OK;
}

atom_status_t atom_validate_perm(const int32_t* perm, int64_t K, int64_t ldx, int32_t* scratch,
                                 int32_t* ok_flag, void* stream) {
  g_last_launches = 0;
  if (!perm || !scratch || !ok_flag) return ATOM_ERR_NULL;
  if (K <= 0 || ldx < K) return ATOM_ERR_SHAPE;
  DeviceInfo dev;
  atom_status_t st = current_device(&dev);
  if (st != ATOM_OK) return st;
  if (atom::launch_validate_perm(perm, K, ldx, scratch, ok_flag,
                                 static_cast<cudaStream_t>(stream)) != cudaSuccess)
    return ATOM_ERR_CUDA;
  g_last_launches = 2;
  return ATOM_OK;
}

const char* atom_status_string(atom_status_t s) {
  switch (s) {
    case ATOM_OK: return "ATOM_OK";
    case ATOM_ERR_NULL: return "ATOM_ERR_NULL: required pointer missing or forbidden pointer given";
    case ATOM_ERR_SHAPE: return "ATOM_ERR_SHAPE: invalid shape or leading dimension";
    case ATOM_ERR_ALIGN: return "ATOM_ERR_ALIGN: pointer not 16-byte aligned";
    case ATOM_ERR_ARG: return "ATOM_ERR_ARG: invalid k_outlier, clip factor or dtype";
    case ATOM_ERR_WORKSPACE: return "ATOM_ERR_WORKSPACE: workspace missing or too small";
    case ATOM_ERR_UNSUPPORTED: return "ATOM_ERR_UNSUPPORTED: device is not sm_100 (B200)";
    case ATOM_ERR_CUDA: return "ATOM_ERR_CUDA: CUDA call or kernel launch failed";
  }
  return "ATOM_ERR_UNKNOWN";
}

int atom_abi_version(void) { return ATOM_ABI_VERSION; }

int atom_last_launch_count(void) { return g_last_launches; }

}  // extern "C"
