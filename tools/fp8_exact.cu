// fp8_exact.cu -- feasibility probe for a conversion-free epilogue: does tcgen05.mma
// kind::f8f6f4 with E4M3 operands holding the INT4 codes (-8..7, exact in E4M3) give the exact
// integer group partial in its fp32 accumulator, and at what rate compared with kind::i8?
// One CTA: W tile 128 x 128 and activation tile 256 x 128 (one group), SW128 K-major, 4 MMAs of
// K = 32; the same codes as int8 through kind::i8.  Development tool (not part of the product).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2310_19102_b200/csrc -o tools/fp8_exact tools/fp8_exact.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace atom;

constexpr int N = 256;
constexpr uint32_t idesc_e4m3 = (1u << 4)    // D = F32
                                | (0u << 7)  // A = E4M3
                                | (0u << 10) // B = E4M3
                                | ((N >> 3) << 17) | ((128 >> 4) << 24);

__device__ __forceinline__ void umma_f8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

// smem: A8 (int8 W) | B8 (int8 X) | AF (e4m3 W) | BF (e4m3 X); out: [2][128][N] (f32 bits, s32)
__global__ void probe(const uint8_t* gin, uint32_t* out, int reps, long long* cyc) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  const int bytes = 2 * (128 + N) * 128;
  for (int i = threadIdx.x; i < bytes; i += blockDim.x) base[i] = gin[i];
  fence_proxy_async_smem();
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tbase, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t a8 = smem_u32(base), b8 = a8 + 128 * 128;
  const uint32_t af = b8 + N * 128, bf = af + 128 * 128;
  uint32_t ph = 0;
  if (threadIdx.x == 0) {
    for (int pass = 0; pass < 2; ++pass) {      // pass 0: exactness (1 group); pass 1: rate
      const int n = pass == 0 ? 1 : reps;
      for (int kind = 0; kind < 2; ++kind) {
        long long t0 = clock64();
        for (int g = 0; g < n; ++g) {
          const uint32_t d = tbase + kind * N;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (kind == 0)
              umma_i8(d, umma_desc_sw128(a8 + 32 * k), umma_desc_sw128(b8 + 32 * k),
                      umma_idesc_i8(128, N), k > 0);
            else
              umma_f8(d, umma_desc_sw128(af + 32 * k), umma_desc_sw128(bf + 32 * k), idesc_e4m3,
                      k > 0);
          }
        }
        umma_commit(&bar);
        mbar_wait(&bar, ph);
        ph ^= 1;
        if (pass == 1) cyc[kind] = clock64() - t0;
      }
    }
  }
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 128) {
    const int w = threadIdx.x / 32;
    for (int kind = 0; kind < 2; ++kind)
      for (int c = 0; c < N; c += 8) {
        uint32_t r[8];
        tmem_ld8(tbase + (static_cast<uint32_t>(w * 32) << 16) + kind * N + c, r);
        tmem_ld_wait();
        for (int v = 0; v < 8; ++v) out[(kind * 128 + threadIdx.x) * N + c + v] = r[v];
      }
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tbase, 512); }
}

static uint8_t e4m3(int v) {
  if (v == 0) return 0;
  const uint8_t s = v < 0 ? 0x80 : 0;
  int a = v < 0 ? -v : v, e = 0;
  while ((a >> (e + 1)) != 0) ++e;
  const int m = (a << 3 >> e) & 7;          // 3 mantissa bits of a / 2^e
  return s | static_cast<uint8_t>(((e + 7) << 3) | m);
}

int main() {
  const int bytes = 2 * (128 + N) * 128;
  uint8_t* h = static_cast<uint8_t*>(malloc(bytes));
  int* qa = static_cast<int*>(malloc(sizeof(int) * 128 * 128));
  int* qb = static_cast<int*>(malloc(sizeof(int) * N * 128));
  uint8_t *d_in;
  uint32_t* d_out;
  long long* d_cyc;
  cudaMalloc(&d_in, bytes);
  cudaMalloc(&d_out, 2 * 128 * N * 4);
  cudaMalloc(&d_cyc, 16);
  uint32_t* out = static_cast<uint32_t*>(malloc(2 * 128 * N * 4));
  const int smem = bytes + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int bad_total = 0;
  for (int trial = 0; trial < 4; ++trial) {
    srand(trial + 1);
    for (int r = 0; r < 128; ++r)
      for (int k = 0; k < 128; ++k)   // trial 0: all -8 (max |P| = 8192); else random
        qa[r * 128 + k] = trial == 0 ? -8 : trial == 1 ? 7 : rand() % 16 - 8;
    for (int r = 0; r < N; ++r)
      for (int k = 0; k < 128; ++k)
        qb[r * 128 + k] = trial == 0 ? -8 : trial == 1 ? (r & 1 ? 7 : -8) : rand() % 16 - 8;
    // SW128 K-major: byte (r, k) at r*128 + ((k/16) ^ (r%8))*16 + k%16
    auto put = [&](uint8_t* dst, int rows, const int* q, bool fp8) {
      for (int r = 0; r < rows; ++r)
        for (int k = 0; k < 128; ++k)
          dst[r * 128 + (((k >> 4) ^ (r & 7)) << 4) + (k & 15)] =
              fp8 ? e4m3(q[r * 128 + k]) : static_cast<uint8_t>(static_cast<int8_t>(q[r * 128 + k]));
    };
    put(h, 128, qa, false);
    put(h + 128 * 128, N, qb, false);
    put(h + (128 + N) * 128, 128, qa, true);
    put(h + (128 + N) * 128 + 128 * 128, N, qb, true);
    cudaMemcpy(d_in, h, bytes, cudaMemcpyHostToDevice);
    probe<<<1, 128, smem>>>(d_in, d_out, 2000, d_cyc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(out, d_out, 2 * 128 * N * 4, cudaMemcpyDeviceToHost);
    long long cyc[2];
    cudaMemcpy(cyc, d_cyc, 16, cudaMemcpyDeviceToHost);
    int bad_i8 = 0, bad_f8 = 0;
    for (int n = 0; n < 128; ++n)
      for (int m = 0; m < N; ++m) {
        long long p = 0;
        for (int k = 0; k < 128; ++k) p += qa[n * 128 + k] * qb[m * 128 + k];
        const int32_t di = static_cast<int32_t>(out[n * N + m]);
        float df;
        memcpy(&df, &out[(128 + n) * N + m], 4);
        bad_i8 += di != p;
        bad_f8 += df != static_cast<float>(p);
      }
    bad_total += bad_i8 + bad_f8;
    printf("trial %d: i8 mismatches %d, e4m3 mismatches %d | rate i8 %.1f clk/group, "
           "e4m3 %.1f clk/group (128x%dx128)\n", trial, bad_i8, bad_f8, cyc[0] / 2000.0,
           cyc[1] / 2000.0, N);
  }
  printf(bad_total ? "NOT EXACT\n" : "EXACT\n");
  return 0;
}
