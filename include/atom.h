/*
 * atom.h -- C ABI of the B200-native Atom W4A4 hot path (arXiv 2310.19102).
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (the paper), "S:n" = SPEC.md line n.
 *
 * The path:
 *   a0  atom_quantize_weights   offline: reorder weight columns by the calibration index and
 *                               quantize them (RTN; GPTQ is out of scope)
 *   a1  atom_reorder_quantize   online: reorder activation channels and dynamically quantize
 *                               them (INT4 groups of 128 + INT8 outlier block)
 *   a2-a5 atom_w4a4_gemm        fused mixed-precision group GEMM: exact int32 partial per
 *                               K-group on the tensor cores, dequantized with s_a*s_w and
 *                               accumulated in fp32, outlier INT8 group fused, fp16 out
 *                                                                                P:254, Fig 6
 *
 * Conventions shared by every entry point
 *   - Pointers are DEVICE pointers owned by the caller (e.g. torch tensors' data_ptr()).  The
 *     library never allocates, frees, retains or synchronizes; every call is asynchronous on
 *     `stream` (a cudaStream_t passed as void*, NULL = legacy default stream).
 *   - Arguments are validated on the host BEFORE anything is launched; on error nothing is
 *     launched and a non-zero atom_status_t is returned.  Nothing aborts or throws across the ABI.
 *   - Device faults (e.g. an out-of-range perm entry, which is a precondition and not checked on
 *     the hot path) surface at the caller's next synchronization.  atom_validate_perm() checks a
 *     perm on the device for tests.
 *   - All base pointers must be 16-byte aligned.  Calls are reentrant; the only global state is
 *     per-device attribute caches and the driver's tensor-map encoder entry point, each
 *     initialised once, thread-safely (std::call_once / function-local statics).
 *   - Group size is fixed at g = 128 ("group size of 128"); k_outlier is 0 or 128
 *     ("128 channels ... keep them in INT8"); K counts the outlier channels (P:256 fn).
 *
 * Quantized formats (bit-exact with the CPU oracle in oracle/)
 *   q4      uint8 [rows][(K - k_outlier)/2]  symmetric INT4 codes in [-8, 7], two's-complement
 *           nibbles, low nibble = even (lower) reordered channel
 *   q8      int8  [rows][k_outlier]          symmetric INT8 codes of the outlier block
 *   scales  fp32  [K/128][rows]              group-major; row t < G4 = (K-k_o)/128 is INT4 group
 *           t, the last row is the outlier scale when k_outlier == 128 (one per token / channel)
 *   a_f8    uint8 [rows][K]  GEMM operand form of the activations (written by the quantize
 *           calls when requested, read by atom_w4a4_gemm_f8): one byte per code.  INT4 group t
 *           (t < G4) occupies bytes [128t, 128t+128) of a row, each code as the E4M3 byte of
 *           q * 2^-9 (sign-magnitude: q for q >= 0, 0x80 | -q for q < 0; bytes 0x00..0x0F of
 *           E4M3 are exactly k * 2^-9), reordered channel 128t + 32c + 8i + 2b + h (c, i, b < 4,
 *           h < 2) at byte 128t + 32c + 16h + 4i + b -- within every 32-channel chunk the even
 *           channels first, then the odd ones, the order in which the GEMM expands a packed
 *           weight nibble pair (low nibble = even channel).  The permutation is the same for both
 *           operands, so every group dot product is unchanged (P:254 Step 1 sums over the
 *           group).  INT8 outlier group: the int8 codes in natural order (= q8).
 *   a_ab    fp32 [K/128][Mp][2], Mp = rows rounded up to 128: per token and group the dequant
 *           constants (alpha, beta) = (s * 2^18, RN(-8 ca * s)) for an INT4 group (ca = sum of
 *           its 128 codes, s its scale) and (s, 0) for the outlier group.  Row order within
 *           every 32 rows: token 32b + r at position 32b + 4 (r % 8) + r / 8 (so a GEMM thread
 *           finds its 4 tokens r, r + 8, r + 16, r + 24 in 32 contiguous bytes); rows past
 *           `rows` are padding (never read for stored outputs).
 *           Why this form: tcgen05 has no 4-bit integer MMA kind and converting int32 partials to
 *           float runs at a quarter of the FP32 rate, so INT4 groups run on kind::f8f6f4 with
 *           integer-valued E4M3 operands (fp32 accumulator = exact integer partial).  The
 *           weights are expanded on the SM from the canonical packed nibbles as offset-binary
 *           bytes (nibble ^ 8, one LOP3 per 4 codes), which adds 8 * ca to each partial; the
 *           GEMM removes it with h = alpha * P' + beta (P' = 2^-18 (P + 8 ca), the fp32
 *           accumulator), i.e. h = s * P up to one rounding.  The activations are expanded once
 *           in the quantize kernel instead of once per output tile.
 *   w_sp    fp32 [K/128][N]  the weight scales in the GEMM's channel order (written by
 *           atom_quantize_weights when requested, read by atom_w4a4_gemm_f8; N % 128 == 0):
 *           within every 128 channels, channel 8k + 2c + b (k < 16, c < 4, b < 2) is stored at
 *           32 (k / 4) + 8c + 2 (k % 4) + b, so the GEMM thread that owns channel pairs 2c + 8k
 *           loads 4 of its pairs as 32 contiguous bytes and the 4 threads c = 0..3 one 128-byte
 *           line (four 32-byte loads per group instead of sixteen 8-byte ones).
 *   Quantizer: s = 2*max|x|*c/(2^n - 1), evaluated as alpha = fl(fl(2c)/(2^n-1)),
 *   s = fl(amax*alpha) (s = FLT_MIN for an all-zero group), q = clamp(rint_even(fl(x*fl(1/s))),
 *   -2^(n-1), 2^(n-1)-1).
 */
#ifndef ATOM_H_
#define ATOM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ATOM_ABI_VERSION 6
#define ATOM_GROUP 128

typedef enum {
  ATOM_OK = 0,
  ATOM_ERR_NULL = 1,        /* a required pointer is NULL (or a forbidden one is non-NULL) */
  ATOM_ERR_SHAPE = 2,       /* K % 128, N % 128, M < 0, ld too small, ... */
  ATOM_ERR_ALIGN = 3,       /* a pointer or leading dimension breaks the alignment rules */
  ATOM_ERR_ARG = 4,         /* k_outlier not in {0,128}, clip not in (0,1], bad dtype */
  ATOM_ERR_WORKSPACE = 5,   /* workspace missing or smaller than atom_w4a4_gemm_workspace_size */
  ATOM_ERR_UNSUPPORTED = 6, /* current device is not sm_100 (B200) */
  ATOM_ERR_CUDA = 7         /* a CUDA runtime/driver call or the launch itself failed */
} atom_status_t;

typedef enum { ATOM_F16 = 0, ATOM_F32 = 1 } atom_dtype_t;

/* atom_w4a4_gemm_f8 flags.  ATOM_GEMM_SPLIT_FREE: no output tile is split over K between CTAs
 * (plain round-robin tiles, no stream-K tail, no workspace), so every output is the same fp32
 * chain -- groups ascending -- for ANY N, and a column shard of the GEMM (tensor-parallel
 * N-sharding) reproduces the unsharded output bit for bit.  Default (0): stream-K load balance,
 * deterministic for a given shape but with split points that depend on the shape. */
#define ATOM_GEMM_SPLIT_FREE 1

/*
 * a1: reorder + dynamic quantize activations ("fuses the activation matrix reordering
 * operators", "tailoring quantization parameters for each activation matrix").
 *   x_f16      fp16 [M][ldx] row-major; token m, source channel c at x_f16[m*ldx + c]
 *   perm       int32 [K]: reordered channel j reads source channel perm[j] (gather).  The last
 *              k_outlier entries are the outlier channels (Fig 4).  A K-shard passes
 *              perm + k0 with its own K (multiple of 128) and k_outlier = 128 only on the shard
 *              that owns the tail.  Precondition (unchecked): 0 <= perm[j] < ldx.
 *   K          number of reordered channels, K % 128 == 0, K >= k_outlier
 *   k_outlier  0 or 128
 *   clip_int4  clipping factor of the INT4 groups, in (0,1]; the paper's 0.9 for activations
 *   clip_int8  clipping factor of the INT8 outlier block, in (0,1]; 1.0
 *   q4, q8, a_f8, a_ab, scales  outputs as described above.  scales is required.  q4 (when
 *              K > k_outlier), q8 (when k_outlier == 128) and the pair (a_f8, a_ab) are each
 *              optional (NULL = not written; a_f8 and a_ab are given together or not at all),
 *              but q4 must be NULL when K == k_outlier, q8 must be NULL when k_outlier == 0, and
 *              at least one code output must be given.  q4/q8 are the canonical packed storage
 *              format (read by atom_w4a4_gemm); a_f8/a_ab the operand form (read by
 *              atom_w4a4_gemm_f8).  All bit-exact with the oracle.
 *              ldx % 8 == 0 (16-byte rows).
 *   M == 0 is a no-op.
 */
atom_status_t atom_reorder_quantize(const void* x_f16, int64_t M, int64_t ldx,
                                    const int32_t* perm, int64_t K, int32_t k_outlier,
                                    float clip_int4, float clip_int8,
                                    uint8_t* q4, int8_t* q8, uint8_t* a_f8, float* a_ab,
                                    float* scales, void* stream);

/*
 * NEXT-1: RMSNorm fused with a1 -- the "prior operator" the paper fuses reordering and
 * quantization into ("fuses the activation matrix reordering operators into the prior
 * operator"; "we fuse the quantization operator into the prior operator (e.g., LayerNorm)").
 * Every row of x_f16 [M][ldx] is first normalized over its ldx channels (the hidden size; rows
 * must be dense):  y_c = fp16_rn( RN32( RN32(x_c * r) * gamma[c] ) ),
 *   r = RN32( 1 / sqrt(sum_c x_c^2 / ldx + eps) )   (sum of squares in double, reading G19),
 * and y is then reordered and quantized exactly as atom_reorder_quantize does (same arguments,
 * formats and errors).  gamma_f16: fp16 [ldx], device; eps >= 0.  y itself is not written.
 */
atom_status_t atom_rmsnorm_reorder_quantize(const void* x_f16, int64_t M, int64_t ldx,
                                            const void* gamma_f16, float eps,
                                            const int32_t* perm, int64_t K, int32_t k_outlier,
                                            float clip_int4, float clip_int8,
                                            uint8_t* q4, int8_t* q8, uint8_t* a_f8,
                                            float* a_ab, float* scales, void* stream);

/*
 * NEXT-4 piece: the SwiGLU of a Llama MLP fused with a1 for the down projection (the "prior
 * operator" of the down projection's quantizer).  gate_f16 and up_f16 are the fp16
 * outputs [M][ldx] of the gate and up projections (same row stride ldx, rows dense in the
 * sense of atom_reorder_quantize).  The value reordered and quantized is
 *   h_c = fp16_rn( RN32( RN32(silu(g_c)) * u_c ) ),  silu(g) = g / (1 + exp(-g)) in double
 * (reading G20), with the same arguments, formats and errors as atom_reorder_quantize;
 * up_f16 must be non-NULL (ATOM_ERR_NULL) and 16-byte aligned (ATOM_ERR_ALIGN).  h is not written.
 */
atom_status_t atom_silu_mul_reorder_quantize(const void* gate_f16, const void* up_f16, int64_t M,
                                             int64_t ldx, const int32_t* perm, int64_t K,
                                             int32_t k_outlier, float clip_int4, float clip_int8,
                                             uint8_t* q4, int8_t* q8, uint8_t* a_f8,
                                             float* a_ab, float* scales, void* stream);

/*
 * a0: offline weight reorder + quantize (Fig 4 P:237 "The weight matrix (W) is statically
 * reordered"; P:299 RTN stands in for GPTQ, which only changes the codes offline).  Same math
 * and formats as atom_reorder_quantize with rows = output channels n of W [N][ldw] (nn.Linear
 * layout); the paper's clip is 0.85 for weights.  scales are fp32 [K/128][N].  q4 and
 * q8 are required (when K > k_outlier / k_outlier == 128): the weights stay packed in HBM.
 * w_sp: NULL, or fp32 [K/128][N] receiving the same scales in the GEMM channel order (above);
 * requires N % 128 == 0 (else ATOM_ERR_SHAPE).
 */
atom_status_t atom_quantize_weights(const void* w_f16, int64_t N, int64_t ldw,
                                    const int32_t* perm, int64_t K, int32_t k_outlier,
                                    float clip_int4, float clip_int8,
                                    uint8_t* q4, int8_t* q8, float* scales, float* w_sp,
                                    void* stream);

/*
 * a2-a5: fused mixed-precision group GEMM (P:254 Steps 1-3, Fig 6, outliers P:230):
 *     P_t[m][n] = sum_{j in group t} qa[m][j] * qw[n][j]            exact integer (tensor cores)
 *     C[m][n]   = sum_t a_scales[t][m] * w_scales[t][n] * P_t[m][n]  fp32 accumulation
 *   written to c[m*ldc + n] as fp16 (c_dtype = ATOM_F16) or as the fp32 partial sum (ATOM_F32,
 *   for K-sharded tensor parallelism where partials are all-reduced in fp32).
 *   a_q4/a_q8/a_scales  activations in the canonical packed format (M rows), as written by
 *                       atom_reorder_quantize; expanded on the device into the
 *                       operand form (a_f8, a_ab) in the workspace, then multiplied
 *   w_q4/w_q8/w_scales  weights from atom_quantize_weights (N rows), same perm and K
 *   M >= 0 (M == 0 is a no-op), N % 128 == 0, K % 128 == 0, k_outlier in {0,128}; a_q4 / w_q4
 *   are required iff K > k_outlier, a_q8 / w_q8 iff k_outlier == 128.
 *   ldc >= N, ldc % 8 == 0 (an N-shard can write its column block into a wider buffer).
 *   debug_partials  NULL, or int32 [K/128][M][N]: every exact group partial P_t (test-only).
 *   workspace       device buffer of at least atom_w4a4_gemm_workspace_size(M, N, K, k_outlier)
 *                   bytes, 16-byte aligned.  The (tile, K-group) work is divided evenly over one
 *                   persistent CTA per SM ("stream-K"), so an output tile may be computed in K
 *                   segments by consecutive CTAs; the segments publish fp32 partials and
 *                   per-tile arrival counters there and the CTA holding the tile's last segment
 *                   sums them in a fixed order (deterministic).  The first
 *                   atom_w4a4_gemm_counter_bytes() bytes hold arrival counters: they MUST be zero
 *                   before the first use, and every completed call leaves them zero again
 *                   (self-cleaning), so no per-call memset is launched and one buffer can serve
 *                   every shape on the device; the rest is scratch.  Must not be shared by calls
 *                   that may run concurrently, and the counters must be re-zeroed if a call was
 *                   aborted.
 */
atom_status_t atom_w4a4_gemm(const uint8_t* a_q4, const int8_t* a_q8, const float* a_scales,
                             const uint8_t* w_q4, const int8_t* w_q8, const float* w_scales,
                             int64_t M, int64_t N, int64_t K, int32_t k_outlier,
                             void* c, int64_t ldc, atom_dtype_t c_dtype,
                             int32_t* debug_partials, void* workspace, size_t workspace_bytes,
                             void* stream);

/*
 * The same GEMM on the activation operand form (a_f8, a_ab) that atom_reorder_quantize writes
 * in the same pass as the scales: the hot path (quantize -> GEMM) then writes and reads only
 * what the GEMM consumes; the weight scales come in the GEMM channel order w_sp that
 * atom_quantize_weights writes offline.  Same results (bit for bit) and errors as
 * atom_w4a4_gemm; a_f8 and a_ab are required (the activation scales are inside a_ab).  flags: 0 or
 * ATOM_GEMM_SPLIT_FREE (above; other bits: ATOM_ERR_ARG).  Workspace:
 * atom_w4a4_gemm_f8_workspace_size bytes (may be 0; any atom_w4a4_gemm workspace also serves).
 */
atom_status_t atom_w4a4_gemm_f8(const uint8_t* a_f8, const float* a_ab,
                                const uint8_t* w_q4, const int8_t* w_q8, const float* w_sp,
                                int64_t M, int64_t N, int64_t K, int32_t k_outlier,
                                void* c, int64_t ldc, atom_dtype_t c_dtype,
                                int32_t* debug_partials, int32_t flags, void* workspace,
                                size_t workspace_bytes, void* stream);

/* Bytes of device workspace atom_w4a4_gemm needs for this shape on the CURRENT device (0 when
 * the current device is not an sm_100 GPU). */
size_t atom_w4a4_gemm_workspace_size(int64_t M, int64_t N, int64_t K, int32_t k_outlier);

/* Bytes of device workspace atom_w4a4_gemm_f8 needs (0 when no output tile is split between
 * CTAs, or when the current device is not an sm_100 GPU). */
size_t atom_w4a4_gemm_f8_workspace_size(int64_t M, int64_t N, int64_t K, int32_t k_outlier);

/* Size of the leading counter region of every GEMM workspace on the CURRENT device (the part
 * that must be zero before first use; 0 when the device is not an sm_100 GPU). */
size_t atom_w4a4_gemm_counter_bytes(void);

/* ------------------------------------------------------------------------------------------
 * Atom (FP) on the MX format (NEXT-2).  The paper's FP4 variant: "quantizing both weights and
 * activations into FP4" with "group quantization with the MX format ... supported by NVIDIA
 * Blackwell GPUs" (Section 6; Table 5).  Same reorder and outlier split
 * as above; readings G21-G24 of DESIGN.md fix the format:
 *   fp4   uint8 [rows][(K - k_outlier)/2]  MXFP4 elements, E2M1 nibbles (sign, 2-bit exponent
 *         with bias 1, 1 mantissa bit), low nibble = even reordered channel
 *   fp8   uint8 [rows][k_outlier]          MXFP8 elements of the outlier channels, E4M3
 *   sf    uint8 [rows][ldsf]               UE8M0 block scales: byte b of a row = 127 + the
 *         shared exponent of reordered channels [32b, 32b + 32) (b < K/32; the last k_o/32 are
 *         the outlier blocks); ldsf >= K/32 and a multiple of 16; bytes past K/32 are not written
 *   Conversion (OCP MX v1.0 6.3): shared_exp = floor(log2(amax of the block)) - emax_elem
 *   (2 for E2M1, 8 for E4M3), byte 0 for an all-zero block; element = x / 2^shared_exp rounded
 *   to nearest-even in the element format, saturating to +-6 / +-448, the sign of x kept on
 *   zero.  Bit-exact with oracle/mx_oracle.c.
 * ------------------------------------------------------------------------------------------ */

/* Reorder + MX-quantize `rows` fp16 rows (x[r * ldx + perm[j]] is reordered channel j).  Used
 * online for activations and offline for weights (rows = N).  K % 128 == 0, k_outlier in {0, 128},
 * ldx % 8 == 0, ldx >= max(perm) + 1, 2 * ldx <= 227 KiB.  fp4 NULL iff K == k_outlier, fp8 NULL
 * iff k_outlier == 0. */
atom_status_t atom_mx_reorder_quantize(const void* x_f16, int64_t rows, int64_t ldx,
                                       const int32_t* perm, int64_t K, int32_t k_outlier,
                                       uint8_t* fp4, uint8_t* fp8, uint8_t* sf, int64_t ldsf,
                                       void* stream);

/* C[m*ldc + n] = fp16( sum_j deq(a[m][j]) * deq(w[n][j]) ), deq = element * 2^shared_exp, on
 * tcgen05 block-scaled MMAs (kind::mxf4 for the FP4 channels, kind::mxf8f6f4 for the outliers)
 * with fp32 accumulation.  Activations [M][..] and weights [N][..] in the formats above (weights
 * quantized with the same perm).  N % 128 == 0, ldc >= N, ldc % 8 == 0, lda_sf / ldw_sf as ldsf.
 * workspace: atom_mx_gemm_workspace_size bytes (0 unless the output tiles cannot fill the GPU,
 * when the K loop is split and an fp32 reduction in a fixed order follows). */
atom_status_t atom_mx_gemm(const uint8_t* a_fp4, const uint8_t* a_fp8, const uint8_t* a_sf,
                           int64_t lda_sf, const uint8_t* w_fp4, const uint8_t* w_fp8,
                           const uint8_t* w_sf, int64_t ldw_sf, int64_t M, int64_t N, int64_t K,
                           int32_t k_outlier, void* c_f16, int64_t ldc, void* workspace,
                           size_t workspace_bytes, void* stream);
size_t atom_mx_gemm_workspace_size(int64_t M, int64_t N, int64_t K, int32_t k_outlier);

/* ------------------------------------------------------------------------------------------
 * Quantized KV cache + decode attention (NEXT-3).  "Atom loads the KV-cache in low-bit
 * precision and directly dequantizes it before performing the FP16 calculation", "asymmetric
 * quantization ... with the granularity of attention head" (Section 4.4), paged as in
 * PageAttention.  Readings G25-G28 of DESIGN.md; bit-exact with oracle/kv_oracle.c.
 *   pages of 16 tokens; head_dim = 128
 *   codes   uint8 [num_pages][H][16][64]   INT4 codes in [0, 15], low nibble = even dimension
 *   params  fp32  [num_pages][H][16][2]    (s, mn) per (token, head): value = code * s + mn
 *   slot of a token = page * 16 + offset; block_table int32 [B][max_pages]: page of tokens
 *   [16 j, 16 j + 16) of sequence b
 *   Quantization per (token, head) vector, each step one binary32 IEEE operation:
 *   s = RN(RN(max - min) / 15); inv = s > 0 ? RN(1 / s) : 0; code = clamp(rint(RN(RN(x - min) *
 *   inv)), 0, 15) (round half to even).
 * ------------------------------------------------------------------------------------------ */

/* Quantize T new tokens' K (or V) vectors x_f16 [T][ldx] (head h of token t at x[t*ldx + 128h])
 * into the cache at slots[t] (int32).  H >= 1, head_dim == 128, ldx >= 128 H, ldx % 4 == 0.  The
 * slots must be distinct and inside the caller's cache (not checked). */
atom_status_t atom_kv_quantize(const void* x_f16, int64_t T, int64_t ldx, int32_t H,
                               int32_t head_dim, const int32_t* slots, uint8_t* codes,
                               float* params, void* stream);

/* One decode step: out[b][h][:] (fp32 [B][H][128]) = softmax(q k^T / sqrt(128)) v over the
 * dequantized tokens t < seq_lens[b] of sequence b (1 <= seq_lens[b] <= max_seq_len <=
 * 16 max_pages; seq_lens on the device, max_seq_len a host-side bound used to split the work).
 * q_f16 [B][H][128].  workspace: atom_decode_attention_workspace_size bytes (may be 0). */
atom_status_t atom_decode_attention(const void* q_f16, int64_t B, int32_t H, int32_t head_dim,
                                    const uint8_t* k_codes, const float* k_params,
                                    const uint8_t* v_codes, const float* v_params,
                                    const int32_t* block_table, int64_t max_pages,
                                    const int32_t* seq_lens, int32_t max_seq_len, float* out,
                                    void* workspace, size_t workspace_bytes, void* stream);
size_t atom_decode_attention_workspace_size(int64_t B, int32_t H, int32_t max_seq_len);

/* Test helper: on `stream`, sets *ok_flag (device int32) to 1 iff perm[0..K) is a bijection of
 * [0,K) (ldx == K) or an injection into [0,ldx).  scratch: device int32 [ldx], clobbered. */
atom_status_t atom_validate_perm(const int32_t* perm, int64_t K, int64_t ldx, int32_t* scratch,
                                 int32_t* ok_flag, void* stream);

const char* atom_status_string(atom_status_t s);
int atom_abi_version(void);
/* Number of kernel launches the last successful call on this thread issued (for bench
 * accounting of "gpu_launches"). */
int atom_last_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* ATOM_H_ */
