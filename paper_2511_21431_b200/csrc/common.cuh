// common.cuh — shared device/host helpers of libmemfine.so (product code; no oracle code).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp8.h>
#include <stdint.h>
#include <stdlib.h>
#include <utility>
#include "../../include/memfine.h"

namespace memfine {

constexpr int kRowAlign = 128;   // every local expert's row segment is padded to 128 rows
constexpr int kTokPerBlk = 32;   // tokens per dispatch block (ranking pass: 32*k copies per CTA)
constexpr int kMaxSub = 64;      // max sub-chunks / chunks per call (memfine_stats.rows)

// info[] words written by the dispatch scan kernel, read by the GEMM schedulers.
enum InfoWord {
  kInfoRows = 0,       // s''_{r,j}: real rows received this chunk
  kInfoRowsPad = 1,    // padded rows (multiple of 128)
  kInfoSend = 2,       // copies of this rank's chunk tokens (valid ids)
  kInfoSkip = 3,       // 1 => capacity exceeded, every kernel of the chunk is a no-op
  kInfoPairs = 4,      // 256-row tile pairs (two 128-row m-tiles of one expert) for 2-CTA GEMMs
  kInfoWords = 8
};

// Latched device status word (pinned, mapped host memory, owned by the handle).
__device__ __forceinline__ void latch_error(int* status, int code) {
  if (status) atomicCAS(status, 0, code);
}

__host__ __device__ __forceinline__ int64_t ceil_div64(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ __forceinline__ int64_t round_up64(int64_t a, int64_t b) { return ceil_div64(a, b) * b; }
__host__ __device__ __forceinline__ int64_t chunk_begin(int64_t T, int C, int j) {
  // chunk j = [floor(jT/C), floor((j+1)T/C)) (reading R1).  T < 2^40 keeps j*T in range.
  return (int64_t)((j * (long long)T) / C);
}

// Element type helpers: the data path stores activations in bf16 (MEMFINE_BF16)
// or fp32 (MEMFINE_FP32); arithmetic is always fp32.
template <typename T> struct Elt;
template <> struct Elt<__nv_bfloat16> {
  static __device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
  static __device__ __forceinline__ __nv_bfloat16 from_f(float v) { return __float2bfloat16_rn(v); }
};
template <> struct Elt<float> {
  static __device__ __forceinline__ float to_f(float v) { return v; }
  static __device__ __forceinline__ float from_f(float v) { return v; }
};

// MUFU-based (ex2 + rcp, ~2 ulp): ample for bf16 outputs; the fp32-mode FFMA path uses the
// IEEE-exact forms (1e-5 parity).
// Programmatic dependent launch: a kernel launched with the PDL attribute may start while its
// predecessor on the stream drains; pdl_wait() blocks until that predecessor has completed and its
// memory is visible (a no-op without the attribute).  pdl_trigger() lets the successor launch early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// PDL on the hot path's launches (MEMFINE_PDL=0 turns it off).  Off for the calling thread while a
// call runs kernels on two streams (MEMFINE_FLAG_OVERLAP): early-launched CTAs waiting on their
// predecessor would hold SMs the comm stream's kernels need (measured: overlap mode 1.5-3 ms slower).
inline thread_local int tl_pdl_off = 0;
struct PdlOff {
  int prev;
  explicit PdlOff(bool off) : prev(tl_pdl_off) { if (off) tl_pdl_off = 1; }
  ~PdlOff() { tl_pdl_off = prev; }
};
inline bool use_pdl() {
  static const int v = [] {
    const char* s = getenv("MEMFINE_PDL");
    return (s && s[0] == '0') ? 0 : 1;
  }();
  return v == 1 && !tl_pdl_off;
}
// <<<grid, block, smem, st>>> with the PDL attribute: the kernel must call pdl_wait() before it
// touches global memory a predecessor writes or reads.
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = a;
  cfg.numAttrs = use_pdl() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);   // errors surface via latch_cuda
}

__device__ __forceinline__ float silu_f(float z) { return __fdividef(z, 1.0f + __expf(-z)); }
__device__ __forceinline__ float sigmoid_f(float z) { return __fdividef(1.0f, 1.0f + __expf(-z)); }
__device__ __forceinline__ float silu_exact(float z) { return z / (1.0f + expf(-z)); }
__device__ __forceinline__ float sigmoid_exact(float z) { return 1.0f / (1.0f + expf(-z)); }

// Binary search: the local expert owning padded row `row` (seg has El+1 entries).
__device__ __forceinline__ int expert_of_row(const int* __restrict__ seg, int El, int row) {
  int lo = 0, hi = El;  // seg[lo] <= row < seg[hi]
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (__ldg(seg + mid) <= row) lo = mid; else hi = mid;
  }
  return lo;
}

// The local expert owning 256-row pair `pair` (pseg: prefix of ceil(m_tiles_e / 2)).
__device__ __forceinline__ int expert_of_pair(const int* __restrict__ pseg, int El, int pair) {
  return expert_of_row(pseg, El, pair);
}

// ------------------------------------------------------------------ MXFP8 (DESIGN reading R28)
// Block of 32 consecutive elements along K, one E8M0 scale 2^E: E is the smallest integer with
// amax <= 448 * 2^E (448 = E4M3 max, so no element clips), E = 0 for an all-zero block, clamped
// to [-127, 126]; elements v * 2^-E rounded to E4M3 (round-to-nearest-even, satfinite).
__device__ __forceinline__ int mx_exp(float amax) {
  if (!(amax > 0.f)) return 0;
  int e;
  const float m = frexpf(amax, &e);              // amax = m 2^e, m in [0.5, 1): exact
  int E = e - 9 + (m > 0.875f ? 1 : 0);          // floor(log2 amax) - 8 (+1 if mantissa > 1.75)
  return E < -127 ? -127 : (E > 126 ? 126 : E);
}
// 2^-E as a float (exact: 127 - E in [1, 254])
__device__ __forceinline__ float mx_inv_scale(int E) { return __uint_as_float((uint32_t)(127 - E) << 23); }
// two floats -> packed E4M3 pair (lo byte = a)
__device__ __forceinline__ uint32_t mx_e4m3x2(float a, float b) {
  return (uint32_t)__nv_cvt_float2_to_fp8x2(make_float2(a, b), __NV_SATFINITE, __NV_E4M3);
}
// Scale-factor chunk layout read by tcgen05.cp 32x128b.warpx4 + the block-scaled MMA: a 512-byte
// chunk per 128 rows x 128 K (4 blocks); chunk (r/128, k/128) at ((r/128) * (K/128) + k/128) * 512,
// row r, block kb (= k/32) at byte (r % 32) * 16 + ((r % 128) / 32) * 4 + kb % 4.
__host__ __device__ __forceinline__ int64_t mx_sf_off(int64_t r, int64_t kb, int64_t K) {
  return ((r >> 7) * (K >> 7) + (kb >> 2)) * 512 + (r & 31) * 16 + ((r & 127) >> 5) * 4 + (kb & 3);
}

}  // namespace memfine

#define MF_CUDA_OK(expr)                                              \
  do {                                                                \
    cudaError_t _e = (expr);                                          \
    if (_e != cudaSuccess) { return MEMFINE_ERR_CUDA; }               \
  } while (0)
