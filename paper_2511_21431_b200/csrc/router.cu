// router.cu — the router step before the chunked MoE layer (Table 2 rows 9-10,
// PAPER.md:83-84): logits = x W_r^T (fp32 accumulate), the k largest logits (ties: lower expert id),
// scores = softmax over the k selected logits; and its backward consuming the layer's d_score.
#include <algorithm>
#include "kernels.h"

namespace memfine {

// ------------------------------------------------------------------ logits = x W_r^T (CUDA cores)
// 64 tokens x 64 experts per block, 256 threads x (4 x 4) outputs, K step 32.
template <typename T>
__global__ void __launch_bounds__(256) router_logits_kernel(const T* __restrict__ x, const T* __restrict__ wr,
                                                            int64_t ntok, int E, int h, float* __restrict__ logits) {
  __shared__ float xs[32][64 + 4];
  __shared__ float ws[32][64 + 4];
  const int64_t t0 = (int64_t)blockIdx.y * 64;
  const int e0 = blockIdx.x * 64;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < h; k0 += 32) {
    for (int i = threadIdx.x; i < 32 * 64; i += 256) {
      const int r = i / 32, kk = i % 32;   // kk fastest: coalesced along h
      const int64_t t = t0 + r;
      const int e = e0 + r;
      xs[kk][r] = (t < ntok && k0 + kk < h) ? Elt<T>::to_f(x[t * h + k0 + kk]) : 0.f;
      ws[kk][r] = (e < E && k0 + kk < h) ? Elt<T>::to_f(wr[(int64_t)e * h + k0 + kk]) : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < 32; kk++) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; i++) { a[i] = xs[kk][ty * 4 + i]; b[i] = ws[kk][tx * 4 + i]; }
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  for (int i = 0; i < 4; i++) {
    const int64_t t = t0 + ty * 4 + i;
    if (t >= ntok) continue;
    for (int j = 0; j < 4; j++) {
      const int e = e0 + tx * 4 + j;
      if (e < E) logits[t * E + e] = acc[i][j];
    }
  }
}

// ------------------------------------------------------------------ top-k + softmax, one warp per token
// logits row stride ld (>= E); out (nullable): the logits copied to a dense [T][E] array
__global__ void __launch_bounds__(256) router_topk_kernel(const float* __restrict__ logits, int64_t ntok, int E, int k,
                                                          int32_t* __restrict__ ids, float* __restrict__ scores,
                                                          int64_t ld, float* __restrict__ out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (t >= ntok) return;
  const float* lg = logits + t * ld;
  if (out)
    for (int e = lane; e < E; e += 32) out[t * E + e] = lg[e];
  uint32_t taken = 0;   // bit s: this lane's s-th expert (lane + 32 s) is chosen (E <= 1024)
  float sel_v[16];
  int sel_i[16];
  for (int j = 0; j < k; j++) {
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int e = lane, s = 0; e < E; e += 32, s++) {
      if ((taken >> s) & 1u) continue;
      const float v = lg[e];
      if (v > bv || (v == bv && e < bi)) { bv = v; bi = e; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    sel_v[j] = bv;
    sel_i[j] = bi;
    if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
  }
  if (lane == 0) {
    const float mx = sel_v[0];
    float z = 0.f;
    for (int j = 0; j < k; j++) z += __expf(sel_v[j] - mx);
    const float iz = 1.f / z;
    for (int j = 0; j < k; j++) {
      ids[t * k + j] = sel_i[j];
      scores[t * k + j] = __expf(sel_v[j] - mx) * iz;
    }
  }
}

// ------------------------------------------------------------------ backward, one warp per token
// d_logit_j = s_j (ds_j - sum_q s_q ds_q) on the selected slots; dx = sum_j d_logit_j W_r[id_j].
// dense (bf16 path): the [T][E] d_logits as an exact-to-2^-17 bf16 pair hi + lo (zero off the selected
// slots), the operands of the dW_r GEMM.  dx moves 16 B per lane when h allows.
template <typename T>
__global__ void __launch_bounds__(256) router_bwd_rows_kernel(const T* __restrict__ wr, const int32_t* __restrict__ ids,
                                                              const float* __restrict__ scores,
                                                              const float* __restrict__ dscore, int64_t ntok, int k,
                                                              int h, int E, float* __restrict__ dlog,
                                                              __nv_bfloat16* __restrict__ dhi,
                                                              __nv_bfloat16* __restrict__ dlo, T* __restrict__ dx,
                                                              int accumulate, int ldd) {
  constexpr int V = 16 / sizeof(T);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (t >= ntok) return;
  float dot = 0.f;
  for (int j = 0; j < k; j++) dot += scores[t * k + j] * dscore[t * k + j];
  float dl[16];
  int id[16];
  for (int j = 0; j < k; j++) {
    dl[j] = scores[t * k + j] * (dscore[t * k + j] - dot);
    id[j] = ids[t * k + j];
    if (lane == 0) dlog[t * k + j] = dl[j];
  }
  if (dhi) {
    for (int e = lane; e < E; e += 32) {
      float v = 0.f;
      for (int j = 0; j < k; j++) v = (id[j] == e) ? dl[j] : v;
      const __nv_bfloat16 hi = __float2bfloat16(v);
      dhi[t * ldd + e] = hi;
      dlo[t * ldd + e] = __float2bfloat16(v - __bfloat162float(hi));
    }
  }
  if (h % V == 0) {
    for (int c = lane * V; c < h; c += 32 * V) {
      float acc[V];
      if (accumulate) {
        const uint4 u = *reinterpret_cast<const uint4*>(dx + t * h + c);
        const T* pv = reinterpret_cast<const T*>(&u);
#pragma unroll
        for (int i = 0; i < V; i++) acc[i] = Elt<T>::to_f(pv[i]);
      } else {
#pragma unroll
        for (int i = 0; i < V; i++) acc[i] = 0.f;
      }
      for (int j = 0; j < k; j++) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(wr + (int64_t)id[j] * h + c));
        const T* pv = reinterpret_cast<const T*>(&u);
#pragma unroll
        for (int i = 0; i < V; i++) acc[i] = fmaf(dl[j], Elt<T>::to_f(pv[i]), acc[i]);
      }
      uint4 o;
      T* po = reinterpret_cast<T*>(&o);
#pragma unroll
      for (int i = 0; i < V; i++) po[i] = Elt<T>::from_f(acc[i]);
      *reinterpret_cast<uint4*>(dx + t * h + c) = o;
    }
    return;
  }
  for (int c = lane; c < h; c += 32) {
    float acc = accumulate ? Elt<T>::to_f(dx[t * h + c]) : 0.f;
    for (int j = 0; j < k; j++) acc = fmaf(dl[j], Elt<T>::to_f(wr[(int64_t)id[j] * h + c]), acc);
    dx[t * h + c] = Elt<T>::from_f(acc);
  }
}

// dW_r[e] = sum over the copies routed to e (contiguous after the counting sort) of d_logit x_token.
template <typename T>
__global__ void __launch_bounds__(256) router_dw_kernel(const T* __restrict__ x, const float* __restrict__ dlog,
                                                        const int* __restrict__ seg, const int* __restrict__ cnt,
                                                        const int* __restrict__ row_src, int k, int h,
                                                        float* __restrict__ dwr, int accumulate) {
  const int e = blockIdx.x;
  const int c = blockIdx.y * blockDim.x + threadIdx.x;
  if (c >= h) return;
  const int r0 = seg[e], r1 = r0 + cnt[e];
  float acc = 0.f;
  for (int r = r0; r < r1; r++) {
    const int q = __ldg(row_src + r);
    acc = fmaf(__ldg(dlog + q), Elt<T>::to_f(x[(int64_t)(q / k) * h + c]), acc);
  }
  float* o = dwr + (int64_t)e * h + c;
  *o = accumulate ? *o + acc : acc;
}

template <typename T>
void launch_router_fwd(const T* x, const T* wr, int64_t ntok, int E, int h, int k, float* logits, int32_t* ids,
                       float* scores, cudaStream_t st) {
  if (ntok == 0) return;
  dim3 grid((unsigned)ceil_div64(E, 64), (unsigned)ceil_div64(ntok, 64));
  router_logits_kernel<T><<<grid, 256, 0, st>>>(x, wr, ntok, E, h, logits);
  router_topk_kernel<<<(unsigned)ceil_div64(ntok, 8), 256, 0, st>>>(logits, ntok, E, k, ids, scores, E, nullptr);
}

// bf16 forward epilogue: top-k + softmax over the fp32 logits [T][ld] the tcgen05 GEMM wrote (memfine.cu
// runs the logits GEMM on the expert-GEMM kernels); out (nullable) receives the dense [T][E] logits.
void launch_router_topk(const float* logits, int64_t ld, int64_t ntok, int E, int k, int32_t* ids, float* scores,
                        float* out, cudaStream_t st) {
  if (ntok == 0) return;
  router_topk_kernel<<<(unsigned)ceil_div64(ntok, 8), 256, 0, st>>>(logits, ntok, E, k, ids, scores, ld, out);
}

// bf16 backward rows: d_logits, dx (+)= d_logits W_r, and the dense d_logits [T][ldd] as the bf16 pair hi + lo
// (exact to ~2^-17 relative; zero off the selected slots) - the operands of the tcgen05 dW_r GEMMs.
void launch_router_bwd_rows_bf16(const __nv_bfloat16* wr, const int32_t* ids, const float* scores, const float* dscore,
                                 int64_t ntok, int E, int h, int k, float* dlog, __nv_bfloat16* dhi,
                                 __nv_bfloat16* dlo, int ldd, __nv_bfloat16* dx, int acc_dx, cudaStream_t st) {
  if (ntok == 0) return;
  router_bwd_rows_kernel<__nv_bfloat16><<<(unsigned)ceil_div64(ntok, 8), 256, 0, st>>>(
      wr, ids, scores, dscore, ntok, k, h, E, dlog, dhi, dlo, dx, acc_dx, ldd);
}

template <typename T>
void launch_router_bwd(const T* x, const T* wr, const int32_t* ids, const float* scores, const float* dscore,
                       int64_t ntok, int E, int h, int k, float* dlog, T* dx, int acc_dx, float* dwr, int acc_dw,
                       const ChunkMeta& m, cudaStream_t st) {
  if (ntok > 0)
    router_bwd_rows_kernel<T><<<(unsigned)ceil_div64(ntok, 8), 256, 0, st>>>(wr, ids, scores, dscore, ntok, k, h, E,
                                                                             dlog, nullptr, nullptr, dx, acc_dx, E);
  dim3 grid((unsigned)E, (unsigned)ceil_div64(h, 256));
  router_dw_kernel<T><<<grid, 256, 0, st>>>(x, dlog, m.seg, m.recv_cnt, m.src_of, k, h, dwr, acc_dw);
}

template void launch_router_fwd<__nv_bfloat16>(const __nv_bfloat16*, const __nv_bfloat16*, int64_t, int, int, int,
                                               float*, int32_t*, float*, cudaStream_t);
template void launch_router_fwd<float>(const float*, const float*, int64_t, int, int, int, float*, int32_t*, float*,
                                       cudaStream_t);
template void launch_router_bwd<__nv_bfloat16>(const __nv_bfloat16*, const __nv_bfloat16*, const int32_t*,
                                               const float*, const float*, int64_t, int, int, int, float*,
                                               __nv_bfloat16*, int, float*, int, const ChunkMeta&, cudaStream_t);
template void launch_router_bwd<float>(const float*, const float*, const int32_t*, const float*, const float*, int64_t,
                                       int, int, int, float*, float*, int, float*, int, const ChunkMeta&,
                                       cudaStream_t);

const void* kernel_anchor_router() { return (const void*)router_topk_kernel; }

}  // namespace memfine
