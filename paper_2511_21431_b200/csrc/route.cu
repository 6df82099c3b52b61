// route.cu — routing histogram, stable dispatch permute, combine, unpermute-reduce and the
// MACT tuner kernel.  HBM-bound data movement:
// 16-byte vector loads/stores along contiguous rows, one warp per routed copy / token.
#include <algorithm>
#include <cstdio>
#include <type_traits>
#include "kernels.h"

namespace memfine {

// ------------------------------------------------------------------------------------------
// A1: per-sub-chunk expert histogram ("first notification").
// Token i belongs to sub-chunk j = floor((nsub*(i+1) - 1) / T)  (inverse of floor(jT/nsub)).
// ------------------------------------------------------------------------------------------
constexpr int kHistTok = 256;
constexpr int kHistSpan = 4;  // sub-chunks one block may privatise in smem

__global__ void route_hist_kernel(const int32_t* __restrict__ ids, int64_t T, int k, int E, int nsub,
                                  int* __restrict__ counts, int* status) {
  extern __shared__ int sh[];
  int64_t b0 = (int64_t)blockIdx.x * kHistTok;
  int64_t b1 = min(b0 + kHistTok, T);
  if (b0 >= b1) return;
  int j0 = (int)((nsub * (b0 + 1) - 1) / T);
  int j1 = (int)((nsub * b1 - 1) / T);
  bool priv = (j1 - j0 + 1) <= kHistSpan;
  if (priv) {
    for (int i = threadIdx.x; i < (j1 - j0 + 1) * E; i += blockDim.x) sh[i] = 0;
    __syncthreads();
  }
  for (int64_t q = b0 * k + threadIdx.x; q < b1 * k; q += blockDim.x) {
    int e = __ldg(ids + q);
    int64_t i = q / k;
    int j = (int)((nsub * (i + 1) - 1) / T);
    if (e < 0 || e >= E) { latch_error(status, MEMFINE_ERR_ROUTING); continue; }
    if (priv) atomicAdd(&sh[(j - j0) * E + e], 1);
    else atomicAdd(&counts[(int64_t)j * E + e], 1);
  }
  if (priv) {
    __syncthreads();
    for (int i = threadIdx.x; i < (j1 - j0 + 1) * E; i += blockDim.x)
      if (sh[i]) atomicAdd(&counts[(int64_t)j0 * E + i], sh[i]);
  }
}

void launch_route_hist(const int32_t* ids, int64_t T, int k, int E, int nsub, int* counts, int* status,
                       cudaStream_t st) {
  cudaMemsetAsync(counts, 0, sizeof(int) * (size_t)nsub * E, st);
  if (T == 0) return;
  int64_t nb = ceil_div64(T, kHistTok);
  size_t smem = sizeof(int) * (size_t)kHistSpan * E;
  route_hist_kernel<<<(unsigned)nb, 256, smem, st>>>(ids, T, k, E, nsub, counts, status);
}

// ------------------------------------------------------------------------------------------
// A5 dispatch, pass 1: per token-block expert histogram of the chunk.
// ------------------------------------------------------------------------------------------
__global__ void dispatch_hist_kernel(const int32_t* __restrict__ ids, int64_t t0, int64_t t1, int k, int E,
                                     int* __restrict__ blk_cnt, int* status) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ int sc[];
  for (int e = threadIdx.x; e < E; e += blockDim.x) sc[e] = 0;
  __syncthreads();
  int64_t b0 = t0 + (int64_t)blockIdx.x * kTokPerBlk;
  int64_t b1 = min(b0 + kTokPerBlk, t1);
  for (int64_t q = b0 * k + threadIdx.x; q < b1 * k; q += blockDim.x) {
    int e = __ldg(ids + q);
    if (e >= 0 && e < E) atomicAdd(&sc[e], 1);
    else latch_error(status, MEMFINE_ERR_ROUTING);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) blk_cnt[(int64_t)blockIdx.x * E + e] = sc[e];
}

void launch_dispatch_hist(const int32_t* ids, int64_t t0, int64_t t1, int k, int E, const ChunkMeta& m,
                          int* status, cudaStream_t st) {
  int NB = (int)ceil_div64(t1 - t0, kTokPerBlk);
  if (NB == 0) return;
  launch_pdl(dispatch_hist_kernel, dim3(NB), dim3(256), sizeof(int) * E, st, ids, t0, t1, k, E, m.blk_cnt, status);
}

// ------------------------------------------------------------------------------------------
// A5 dispatch, pass 2 (one CTA): exclusive scan over blocks per expert, expert bases, info.
//  send_layout == 0 (EP = 1): base[e] = padded prefix (every local expert's segment padded to
//                128 rows);
//  send_layout == 1 (the EP path): base[e] = unpadded prefix over global experts (the NCCL send
//                layout: dest rank major because ranks hold contiguous expert blocks).
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

__global__ void __launch_bounds__(1024) dispatch_scan_kernel(int NB, int E, int El, int send_layout, int64_t rows_cap,
                                     int* __restrict__ blk, int* __restrict__ exp_cnt, int* __restrict__ recv_cnt,
                                     int* __restrict__ seg, int* __restrict__ pseg, int* __restrict__ info,
                                     int64_t* stats_rows, int64_t* stats_rows_pad, int chunk) {
  pdl_wait();
  pdl_trigger();
  __shared__ int base[1024];
  __shared__ int cnt_s[1024];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  // per expert (one warp each): exclusive scan over the token blocks, 32 blocks per step
  for (int e = warp; e < E; e += nw) {
    int carry = 0;
    for (int b0 = 0; b0 < NB; b0 += 256) {  // 8 independent loads per lane per round trip
      int c[8];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int b = b0 + u * 32 + lane;
        c[u] = b < NB ? blk[(int64_t)b * E + e] : 0;
      }
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int b = b0 + u * 32 + lane;
        const int incl = warp_incl_scan(c[u], lane);
        if (b < NB) blk[(int64_t)b * E + e] = carry + incl - c[u];
        carry += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    if (lane == 0) { exp_cnt[e] = carry; cnt_s[e] = carry; }
  }
  __syncthreads();
  // expert bases (warp 0, 32 experts per step)
  if (warp == 0) {
    int acc = 0, send = 0, pairs = 0;
    for (int e0 = 0; e0 < E; e0 += 32) {
      const int e = e0 + lane;
      const int c = e < E ? cnt_s[e] : 0;
      const int ic = warp_incl_scan(c, lane);
      if (!send_layout) {
        const int pad = (int)round_up64(c, kRowAlign);
        const int pr = e < E ? (pad / kRowAlign + 1) / 2 : 0;
        const int ipad = warp_incl_scan(pad, lane), ipr = warp_incl_scan(pr, lane);
        if (e < E) {
          base[e] = acc + ipad - pad;
          seg[e] = acc + ipad - pad;
          pseg[e] = pairs + ipr - pr;
          recv_cnt[e] = c;
        }
        acc += __shfl_sync(0xffffffffu, ipad, 31);
        pairs += __shfl_sync(0xffffffffu, ipr, 31);
      } else {
        if (e < E) base[e] = acc + ic - c;
        acc += __shfl_sync(0xffffffffu, ic, 31);
      }
      send += __shfl_sync(0xffffffffu, ic, 31);
    }
    if (lane == 0) {
      if (!send_layout) {
        seg[El] = acc;
        pseg[El] = pairs;
        info[kInfoPairs] = pairs;
        info[kInfoRows] = send;
        info[kInfoRowsPad] = acc;
        info[kInfoSkip] = (acc > rows_cap) ? 1 : 0;
        if (stats_rows) { stats_rows[chunk] = send; stats_rows_pad[chunk] = acc; }
      } else {
        info[kInfoSkip] = 0;  // EP>1: the host checked the capacity exactly (it knows the counts)
      }
      info[kInfoSend] = send;
    }
  }
  __syncthreads();
  const int64_t n = (int64_t)NB * E;
  if ((E & 3) == 0) {
    int4* b4 = reinterpret_cast<int4*>(blk);
#pragma unroll 4
    for (int64_t i = threadIdx.x; i < n / 4; i += blockDim.x) {
      int4 v = b4[i];
      const int e = (int)((i * 4) % E);
      v.x += base[e]; v.y += base[e + 1]; v.z += base[e + 2]; v.w += base[e + 3];
      b4[i] = v;
    }
  } else {
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) blk[i] += base[i % E];
  }
}

void launch_dispatch_scan(int NB, int E, int El, int send_layout, int64_t rows_cap, const ChunkMeta& m,
                          int64_t* stats_rows, int64_t* stats_rows_pad, int chunk, cudaStream_t st) {
  launch_pdl(dispatch_scan_kernel, dim3(1), dim3(1024), 0, st, NB, E, El, send_layout, rows_cap, m.blk_cnt, m.exp_cnt, m.recv_cnt,
                                           m.seg, m.pseg, m.info, stats_rows, stats_rows_pad, chunk);
}

// ------------------------------------------------------------------------------------------
// A5/B1 dispatch, pass 3: stable in-block rank (canonical order (expert, token, slot),
// reading R3) then one warp per copy moves the token row(s) with 16-byte vectors.
// ------------------------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void copy_row(T* __restrict__ dst, const T* __restrict__ src, int h, int lane) {
  constexpr int V = 16 / sizeof(T);
  const uint4* s = reinterpret_cast<const uint4*>(src);
  uint4* d = reinterpret_cast<uint4*>(dst);
  int nv = h / V;
  int i = lane;
  for (; i + 96 < nv; i += 128) {
    uint4 a = __ldg(s + i), b = __ldg(s + i + 32), c = __ldg(s + i + 64), e = __ldg(s + i + 96);
    d[i] = a; d[i + 32] = b; d[i + 64] = c; d[i + 96] = e;
  }
  for (; i < nv; i += 32) d[i] = __ldg(s + i);
}

// Pass 3a: stable in-block rank -> dest_of[copy], row_src[row] = copy index, row scores.
__global__ void __launch_bounds__(256) dispatch_index_kernel(
    const int32_t* __restrict__ ids, const float* __restrict__ w, int64_t t0, int64_t t1, int k, int E,
    const int* __restrict__ blk_off, int* __restrict__ dest_of, int* __restrict__ row_src,
    float* __restrict__ w_row, float* __restrict__ dw_row, const int* __restrict__ info) {
  pdl_wait();
  pdl_trigger();
  if (info[kInfoSkip]) return;
  extern __shared__ int smem[];
  int* run = smem;        // [E]
  int* spos = smem + E;   // [kTokPerBlk * k]
  int64_t b0 = t0 + (int64_t)blockIdx.x * kTokPerBlk;
  int64_t b1 = min(b0 + kTokPerBlk, t1);
  int ncp = (int)(b1 - b0) * k;
  for (int e = threadIdx.x; e < E; e += blockDim.x) run[e] = blk_off[(int64_t)blockIdx.x * E + e];
  for (int q = threadIdx.x; q < ncp; q += blockDim.x) spos[q] = __ldg(ids + b0 * k + q);  // ids, coalesced
  __syncthreads();
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    unsigned lt = (1u << lane) - 1u;
    for (int base = 0; base < ncp; base += 32) {
      int q = base + lane;
      int e = -1;
      if (q < ncp) {
        e = spos[q];
        if (e < 0 || e >= E) e = -1;
      }
      unsigned peers = __match_any_sync(0xffffffffu, e);
      int p = -1;
      if (e >= 0) p = run[e] + __popc(peers & lt);
      __syncwarp();
      bool last = (peers >> lane) == 1u;  // highest lane of its group
      if (e >= 0 && last) run[e] += __popc(peers);
      __syncwarp();
      if (q < ncp) spos[q] = p;
    }
  }
  __syncthreads();
  for (int q = threadIdx.x; q < ncp; q += blockDim.x) {
    int p = spos[q];
    int64_t qg = b0 * k + q;  // global copy index i*k + slot
    dest_of[qg - t0 * k] = p;
    if (p < 0) continue;
    row_src[p] = (int)qg;
    if (w_row) w_row[p] = __ldg(w + qg);
    if (dw_row) dw_row[p] = 0.0f;
  }
}

// Pass 3b': one warp per SOURCE token reads its row(s) once and writes them to the token's k
// destination rows (dest_of from pass 3a).  Every token row crosses HBM once instead of once per
// copy (the destination-order gather re-reads it k times: 6.2x x's bytes at DeepSeek-V3's k = 8),
// so the kernel moves the algorithmic bytes, T_j*h read + T_j*k*h written per tensor.  With `seg`
// (the expert-major layout) the same launch then zeroes the padding rows.
template <typename T>
__global__ void __launch_bounds__(256) dispatch_scatter_kernel(
    const T* __restrict__ x, const T* __restrict__ dy, int64_t t0, int64_t t1, int k, int h,
    const int* __restrict__ dest_of, const int* __restrict__ info, T* __restrict__ xd, T* __restrict__ dyd,
    const int* __restrict__ seg, const int* __restrict__ cnt, int El, int* __restrict__ src_of,
    float* __restrict__ w_row, float* __restrict__ dw_row) {
  pdl_wait();
  pdl_trigger();
  if (info[kInfoSkip]) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  constexpr int V = 16 / sizeof(T);
  const int nv = h / V;
  for (int64_t i = t0 + (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; i < t1; i += nwarps) {
    __shared__ int pos_s[8][16];
    int* pos = pos_s[warp];
    const int kk = k < 16 ? k : 16;
    __syncwarp();
    if (lane < 16) pos[lane] = lane < kk ? __ldg(dest_of + (i - t0) * k + lane) : -1;
    __syncwarp();
    const uint4* s1 = reinterpret_cast<const uint4*>(x + i * h);
    const uint4* s2 = dy ? reinterpret_cast<const uint4*>(dy + i * h) : nullptr;
    int c = lane;
    for (; c + 96 < nv; c += 128) {
      uint4 a0 = __ldg(s1 + c), a1 = __ldg(s1 + c + 32), a2 = __ldg(s1 + c + 64), a3 = __ldg(s1 + c + 96);
      uint4 b0, b1, b2, b3;
      if (s2) { b0 = __ldg(s2 + c); b1 = __ldg(s2 + c + 32); b2 = __ldg(s2 + c + 64); b3 = __ldg(s2 + c + 96); }
#pragma unroll
      for (int s = 0; s < 16; s++) {
        if (s >= kk) break;
        if (pos[s] < 0) continue;
        uint4* d = reinterpret_cast<uint4*>(xd + (int64_t)pos[s] * h) + c;
        d[0] = a0; d[32] = a1; d[64] = a2; d[96] = a3;
        if (s2) {
          uint4* d2 = reinterpret_cast<uint4*>(dyd + (int64_t)pos[s] * h) + c;
          d2[0] = b0; d2[32] = b1; d2[64] = b2; d2[96] = b3;
        }
      }
    }
    for (; c < nv; c += 32) {
      uint4 a = __ldg(s1 + c), b;
      if (s2) b = __ldg(s2 + c);
#pragma unroll
      for (int s = 0; s < 16; s++) {
        if (s >= kk) break;
        if (pos[s] < 0) continue;
        reinterpret_cast<uint4*>(xd + (int64_t)pos[s] * h)[c] = a;
        if (s2) reinterpret_cast<uint4*>(dyd + (int64_t)pos[s] * h)[c] = b;
      }
    }
  }
  if (!seg) return;
  // expert-major layout: zero the padding rows [seg[e] + cnt[e], seg[e+1]) (<= 127 per expert),
  // one warp per (expert, padding slot), so padded rows add exact zeros to the dW reductions
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  for (int64_t q = gw; q < (int64_t)El * kRowAlign; q += nwarps) {
    const int e = (int)(q / kRowAlign);
    const int r = __ldg(seg + e) + __ldg(cnt + e) + (int)(q % kRowAlign);
    if (r >= __ldg(seg + e + 1)) continue;
    const uint4 z = make_uint4(0, 0, 0, 0);
    uint4* a = reinterpret_cast<uint4*>(xd + (int64_t)r * h);
    for (int i = lane; i < nv; i += 32) a[i] = z;
    if (dyd) {
      uint4* b = reinterpret_cast<uint4*>(dyd + (int64_t)r * h);
      for (int i = lane; i < nv; i += 32) b[i] = z;
    }
    if (lane == 0) {
      src_of[r] = -1;
      w_row[r] = 0.0f;
      if (dw_row) dw_row[r] = 0.0f;
    }
  }
}

// The MX gather as a token-order scatter: one warp per source token quantises its x row ONCE
// (codes are per row along h, so every copy of a token has the same codes and scales) and writes
// the codes, scale bytes (tcgen05 chunk layout at each destination row) and, when asked, the bf16
// x / dY rows to the token's k destinations.  Padding rows: zero codes, scale code 127 (E = 0),
// zero bf16 rows.
__device__ __forceinline__ void mx_quant8(const uint4& a, uint2& o, int& E) {
  const uint32_t wv[4] = {a.x, a.y, a.z, a.w};
  float v[8];
  float amax = 0.f;
#pragma unroll
  for (int j = 0; j < 4; j++) {
    v[2 * j] = __uint_as_float(wv[j] << 16);
    v[2 * j + 1] = __uint_as_float(wv[j] & 0xFFFF0000u);
    amax = fmaxf(amax, fmaxf(fabsf(v[2 * j]), fabsf(v[2 * j + 1])));
  }
  amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 1));
  amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 2));
  E = mx_exp(amax);
  const float inv = mx_inv_scale(E);
  o.x = mx_e4m3x2(v[0] * inv, v[1] * inv) | (mx_e4m3x2(v[2] * inv, v[3] * inv) << 16);
  o.y = mx_e4m3x2(v[4] * inv, v[5] * inv) | (mx_e4m3x2(v[6] * inv, v[7] * inv) << 16);
}

__global__ void __launch_bounds__(256) dispatch_scatter_mx_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ dy, int64_t t0, int64_t t1, int k, int h,
    const int* __restrict__ dest_of, const int* __restrict__ seg, const int* __restrict__ cnt, int El,
    int* __restrict__ src_of, float* __restrict__ w_row, float* __restrict__ dw_row, const int* __restrict__ info,
    int write_x, __nv_bfloat16* __restrict__ xd, __nv_bfloat16* __restrict__ dyd, uint8_t* __restrict__ xq,
    uint8_t* __restrict__ xsf) {
  pdl_wait();
  pdl_trigger();
  if (info[kInfoSkip]) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int nv = h / 8;   // uint4 per row (h % 32 == 0: blocks never straddle a quad of lanes)
  __shared__ int pos_s[8][16];
  int* pos = pos_s[warp];
  const int kk = k < 16 ? k : 16;
  for (int64_t t = t0 + (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; t < t1; t += nwarps) {
    __syncwarp();
    if (lane < 16) pos[lane] = lane < kk ? __ldg(dest_of + (t - t0) * k + lane) : -1;
    __syncwarp();
    const uint4* s = reinterpret_cast<const uint4*>(x + t * h);
    const uint4* s2 = dy ? reinterpret_cast<const uint4*>(dy + t * h) : nullptr;
    for (int base = 0; base < nv; base += 64) {
      const int i0 = base + lane, i1 = base + 32 + lane;
      const bool ok0 = i0 < nv, ok1 = i1 < nv;   // whole quads (nv % 4 == 0)
      uint4 a0 = make_uint4(0, 0, 0, 0), a1 = a0, b0 = a0, b1 = a0;
      if (ok0) a0 = __ldg(s + i0);
      if (ok1) a1 = __ldg(s + i1);
      if (s2 && ok0) b0 = __ldg(s2 + i0);
      if (s2 && ok1) b1 = __ldg(s2 + i1);
      uint2 o0, o1;
      int E0, E1;
      mx_quant8(a0, o0, E0);
      mx_quant8(a1, o1, E1);
#pragma unroll
      for (int q = 0; q < 16; q++) {
        if (q >= kk) break;
        const int64_t r = pos[q];
        if (r < 0) continue;
        if (ok0) {
          *reinterpret_cast<uint2*>(xq + r * h + (int64_t)i0 * 8) = o0;
          if ((i0 & 3) == 0) xsf[mx_sf_off(r, i0 >> 2, h)] = (uint8_t)(E0 + 127);
          if (write_x) reinterpret_cast<uint4*>(xd + r * h)[i0] = a0;
          if (s2) reinterpret_cast<uint4*>(dyd + r * h)[i0] = b0;
        }
        if (ok1) {
          *reinterpret_cast<uint2*>(xq + r * h + (int64_t)i1 * 8) = o1;
          if ((i1 & 3) == 0) xsf[mx_sf_off(r, i1 >> 2, h)] = (uint8_t)(E1 + 127);
          if (write_x) reinterpret_cast<uint4*>(xd + r * h)[i1] = a1;
          if (s2) reinterpret_cast<uint4*>(dyd + r * h)[i1] = b1;
        }
      }
    }
  }
  // padding rows of each local expert segment
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  for (int64_t q = gw; q < (int64_t)El * kRowAlign; q += nwarps) {
    const int e = (int)(q / kRowAlign);
    const int64_t r = __ldg(seg + e) + __ldg(cnt + e) + (int)(q % kRowAlign);
    if (r >= __ldg(seg + e + 1)) continue;
    const uint4 z = make_uint4(0, 0, 0, 0);
    for (int i = lane; i < nv; i += 32) {
      *reinterpret_cast<uint2*>(xq + r * h + (int64_t)i * 8) = make_uint2(0, 0);
      if ((i & 3) == 0) xsf[mx_sf_off(r, i >> 2, h)] = (uint8_t)127;
      if (write_x) reinterpret_cast<uint4*>(xd + r * h)[i] = z;
      if (dy) reinterpret_cast<uint4*>(dyd + r * h)[i] = z;
    }
    if (lane == 0) {
      src_of[r] = -1;
      w_row[r] = 0.0f;
      if (dw_row) dw_row[r] = 0.0f;
    }
  }
}

void launch_dispatch_index(const int32_t* ids, const float* w, int64_t t0, int64_t t1, int k, int E,
                           const ChunkMeta& m, int* row_src, float* w_row, cudaStream_t st) {
  int NB = (int)ceil_div64(t1 - t0, kTokPerBlk);
  if (NB == 0) return;
  size_t smem = sizeof(int) * ((size_t)E + (size_t)kTokPerBlk * k);
  launch_pdl(dispatch_index_kernel, dim3(NB), dim3(256), smem, st, ids, w, t0, t1, k, E, m.blk_cnt, m.dest_of, row_src, w_row, nullptr,
                                               m.info);
}

template <typename T>
void launch_dispatch_scatter(const T* x, const T* dy, const int32_t* ids, const float* w, int64_t t0, int64_t t1,
                             int k, int E, int h, const ChunkMeta& m, T* xd, T* dyd, int El, bool expert_major,
                             int64_t rows_cap, cudaStream_t st, uint8_t* xq, uint8_t* xsf, bool write_x) {
  (void)rows_cap;
  int NB = (int)ceil_div64(t1 - t0, kTokPerBlk);
  if (NB == 0) return;
  size_t smem = sizeof(int) * ((size_t)E + (size_t)kTokPerBlk * k);
  int* row_src = expert_major ? m.src_of : m.send_src;
  launch_pdl(dispatch_index_kernel, dim3(NB), dim3(256), smem, st, ids, w, t0, t1, k, E, m.blk_cnt, m.dest_of, row_src, m.w_row,
                                               dy ? m.dw_row : nullptr, m.info);
  // token-order scatter (each source row read once; k <= 16, memfine_create checks) + the padding
  // rows of the expert-major layout zeroed in the same launch
  const int blocks = (int)std::min<int64_t>(std::max<int64_t>(ceil_div64(t1 - t0, 8), expert_major ? El * 16 : 1),
                                            148 * 16);
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    if (xq && expert_major) {
      launch_pdl(dispatch_scatter_mx_kernel, dim3(blocks), dim3(256), 0, st, x, dy, t0, t1, k, h, m.dest_of, m.seg, m.recv_cnt, El,
                                                          m.src_of, m.w_row, dy ? m.dw_row : nullptr, m.info,
                                                          write_x ? 1 : 0, xd, dyd, xq, xsf);
      return;
    }
  }
  launch_pdl(dispatch_scatter_kernel<T>, dim3(blocks), dim3(256), 0, st, x, dy, t0, t1, k, h, m.dest_of, m.info, xd, dyd,
                                                     expert_major ? m.seg : nullptr, m.recv_cnt, El, m.src_of,
                                                     m.w_row, dy ? m.dw_row : nullptr);
}

// Zero the padding rows of each local expert segment (so padded rows contribute exact
// zeros to the weight-gradient reductions over tokens).
template <typename T>
__global__ void zero_padding_kernel(const int* __restrict__ seg, const int* __restrict__ recv_cnt, int h,
                                    const int* __restrict__ info, T* __restrict__ xd, T* __restrict__ dyd,
                                    int* __restrict__ src_of, float* __restrict__ w_row, float* __restrict__ dw_row) {
  pdl_wait();
  pdl_trigger();
  if (info[kInfoSkip]) return;
  int e = blockIdx.x;
  int r0 = seg[e] + recv_cnt[e], r1 = seg[e + 1];
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  constexpr int V = 16 / sizeof(T);
  for (int r = r0 + blockIdx.y * nw + warp; r < r1; r += nw * gridDim.y) {
    uint4 z = make_uint4(0, 0, 0, 0);
    uint4* a = reinterpret_cast<uint4*>(xd + (int64_t)r * h);
    for (int i = lane; i < h / V; i += 32) a[i] = z;
    if (dyd) {
      uint4* b = reinterpret_cast<uint4*>(dyd + (int64_t)r * h);
      for (int i = lane; i < h / V; i += 32) b[i] = z;
    }
    if (lane == 0) {
      if (src_of) src_of[r] = -1;
      if (w_row) w_row[r] = 0.0f;
      if (dw_row) dw_row[r] = 0.0f;
    }
  }
}

template <typename T>
void launch_zero_padding(int El, int h, const ChunkMeta& m, T* xd, T* dyd, cudaStream_t st) {
  launch_pdl(zero_padding_kernel<T>, dim3(dim3(El, kRowAlign / 8)), dim3(256), 0, st, m.seg, m.recv_cnt, h, m.info, xd, dyd, m.src_of,
                                                                 m.w_row, dyd ? m.dw_row : nullptr);
}

// ------------------------------------------------------------------------------------------
// A10: combine fused into the unpermute: Y_i = sum_{slot asc} w_{i,slot} * o[pos(i,slot)],
// fp32 accumulation, one rounding (Table 2 row 13 "score mul").
// ------------------------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void load8(const T* p, float v[8]);
template <>
__device__ __forceinline__ void load8<__nv_bfloat16>(const __nv_bfloat16* p, float v[8]) {
  uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
  const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; i++) { float2 f = __bfloat1622float2(b[i]); v[2 * i] = f.x; v[2 * i + 1] = f.y; }
}
template <>
__device__ __forceinline__ void load8<float>(const float* p, float v[8]) {
  float4 a = __ldg(reinterpret_cast<const float4*>(p)), b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
template <typename T>
__device__ __forceinline__ void store8(T* p, const float v[8]);
template <>
__device__ __forceinline__ void store8<__nv_bfloat16>(__nv_bfloat16* p, const float v[8]) {
  uint4 u;
  __nv_bfloat162* b = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; i++) b[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = u;
}
template <>
__device__ __forceinline__ void store8<float>(float* p, const float v[8]) {
  reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
}

// Raw 8-element vectors: all k rows of a column chunk are loaded before any FMA, so a lane keeps
// k (x NC column chunks) independent 16-byte loads in flight - the loop over slots would otherwise
// issue one load, wait for it at the FMA, then issue the next.
template <typename T> struct Raw8;
template <> struct Raw8<__nv_bfloat16> {
  uint4 u;
  __device__ __forceinline__ void load(const __nv_bfloat16* p) { u = __ldg(reinterpret_cast<const uint4*>(p)); }
  __device__ __forceinline__ void zero() { u = make_uint4(0, 0, 0, 0); }
  __device__ __forceinline__ void to_float(float v[8]) const {
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; i++) { float2 f = __bfloat1622float2(b[i]); v[2 * i] = f.x; v[2 * i + 1] = f.y; }
  }
};
template <> struct Raw8<float> {
  float4 a, b;
  __device__ __forceinline__ void load(const float* p) {
    a = __ldg(reinterpret_cast<const float4*>(p)); b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  }
  __device__ __forceinline__ void zero() { a = b = make_float4(0, 0, 0, 0); }
  __device__ __forceinline__ void to_float(float v[8]) const {
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
};

// One warp per token; per iteration NC column chunks of 8 elements per lane.  Slots are
// accumulated in ascending order from 0 (fma(w_s, v, acc)), exactly as before the loads were
// hoisted, so results are bit-identical; slots with pos < 0 (invalid ids) contribute nothing.
template <typename T, bool WEIGHTED>
__global__ void __launch_bounds__(256, 2) gather_reduce_kernel(
    const T* __restrict__ rows, const float* __restrict__ w, int64_t t0, int64_t t1, int k, int h,
    const int* __restrict__ dest_of, const int* __restrict__ info, T* __restrict__ out,
    const float* __restrict__ dw_row, float* __restrict__ dscore) {
  pdl_wait();
  pdl_trigger();
  if (info[kInfoSkip]) return;
  constexpr int SG = 8;                       // slots loaded per group
  constexpr int NC = sizeof(T) == 2 ? 2 : 1;  // column chunks per iteration
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t i = t0 + (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (i >= t1) return;
  __shared__ int pos_s[8][16];   // per warp: destination row and score of each slot
  __shared__ float ws_s[8][16];
  int* pos = pos_s[warp];
  float* ws = ws_s[warp];
  const int kk = k < 16 ? k : 16;
  if (lane < 16) {
    pos[lane] = lane < kk ? dest_of[(i - t0) * k + lane] : -1;
    ws[lane] = (WEIGHTED && lane < kk) ? __ldg(w + i * k + lane) : 1.0f;
  }
  __syncwarp();
  if (dscore && lane < k) {
    int p = dest_of[(i - t0) * k + lane];
    dscore[i * k + lane] = p >= 0 ? dw_row[p] : 0.0f;
  }
  for (int c0 = lane * 8; c0 < h; c0 += 256 * NC) {
    float acc[NC][8];
#pragma unroll
    for (int q = 0; q < NC; q++)
#pragma unroll
      for (int u = 0; u < 8; u++) acc[q][u] = 0.f;
#pragma unroll
    for (int g0 = 0; g0 < 16; g0 += SG) {
      if (g0 >= kk) break;
      Raw8<T> raw[SG][NC];
#pragma unroll
      for (int s = 0; s < SG; s++)
#pragma unroll
        for (int q = 0; q < NC; q++) {
          const int c = c0 + q * 256;
          if (g0 + s < kk && pos[g0 + s] >= 0 && c < h) raw[s][q].load(rows + (int64_t)pos[g0 + s] * h + c);
          else raw[s][q].zero();
        }
#pragma unroll
      for (int s = 0; s < SG; s++) {
        if (g0 + s >= kk || pos[g0 + s] < 0) continue;
#pragma unroll
        for (int q = 0; q < NC; q++) {
          float v[8];
          raw[s][q].to_float(v);
#pragma unroll
          for (int u = 0; u < 8; u++) acc[q][u] = fmaf(ws[g0 + s], v[u], acc[q][u]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < NC; q++)
      if (c0 + q * 256 < h) store8<T>(out + i * h + c0 + q * 256, acc[q]);
  }
}

// bf16 combine / unpermute-reduce (A10, B7): one warp per token, 32 B per lane per load (LDG.256),
// NC = 2 column chunks of 512 per iteration and SG slots loaded before the FMAs, so a warp keeps
// SG x 2 x 1 KB in flight (the per-slot loop had 512 B).  Slots are accumulated in ascending order
// from 0 with fma(w_s, v, acc) - bit-identical to the generic kernel above.
__device__ __forceinline__ void ldg256_nc(const void* p, uint32_t (&v)[8]) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "l"(p));
}
__device__ __forceinline__ void stg256(void* p, const uint32_t (&v)[8]) {
  asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
               "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}

template <bool WEIGHTED, int SG>
__global__ void __launch_bounds__(256, SG <= 2 ? 3 : 2) gather_reduce_bf16_kernel(
    const __nv_bfloat16* __restrict__ rows, const float* __restrict__ w, int64_t t0, int64_t t1, int k, int h,
    const int* __restrict__ dest_of, const int* __restrict__ info, __nv_bfloat16* __restrict__ out,
    const float* __restrict__ dw_row, float* __restrict__ dscore) {
  pdl_wait();
  pdl_trigger();
  if (info[kInfoSkip]) return;
  constexpr int NC = 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i = t0 + (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (i >= t1) return;
  __shared__ int pos_s[8][16];
  __shared__ float ws_s[8][16];
  int* pos = pos_s[warp];
  float* ws = ws_s[warp];
  const int kk = k < 16 ? k : 16;
  if (lane < 16) {
    pos[lane] = lane < kk ? dest_of[(i - t0) * k + lane] : -1;
    ws[lane] = (WEIGHTED && lane < kk) ? __ldg(w + i * k + lane) : 1.0f;
  }
  __syncwarp();
  if (dscore && lane < k) {
    const int p = dest_of[(i - t0) * k + lane];
    dscore[i * k + lane] = p >= 0 ? dw_row[p] : 0.0f;
  }
  for (int c0 = lane * 16; c0 < h; c0 += 512 * NC) {
    float acc[NC][16];
#pragma unroll
    for (int q = 0; q < NC; q++)
#pragma unroll
      for (int u = 0; u < 16; u++) acc[q][u] = 0.f;
    for (int g0 = 0; g0 < kk; g0 += SG) {
      uint32_t raw[SG][NC][8];
#pragma unroll
      for (int s = 0; s < SG; s++)
#pragma unroll
        for (int q = 0; q < NC; q++) {
          const int c = c0 + q * 512;
          if (g0 + s < kk && pos[g0 + s] >= 0 && c < h) {
            ldg256_nc(rows + (int64_t)pos[g0 + s] * h + c, raw[s][q]);
          } else {
#pragma unroll
            for (int u = 0; u < 8; u++) raw[s][q][u] = 0u;
          }
        }
#pragma unroll
      for (int s = 0; s < SG; s++) {
        if (g0 + s >= kk || pos[g0 + s] < 0) continue;
        const float ww = ws[g0 + s];
#pragma unroll
        for (int q = 0; q < NC; q++)
#pragma unroll
          for (int u = 0; u < 8; u++) {
            acc[q][2 * u] = fmaf(ww, __uint_as_float(raw[s][q][u] << 16), acc[q][2 * u]);
            acc[q][2 * u + 1] = fmaf(ww, __uint_as_float(raw[s][q][u] & 0xFFFF0000u), acc[q][2 * u + 1]);
          }
      }
    }
#pragma unroll
    for (int q = 0; q < NC; q++) {
      const int c = c0 + q * 512;
      if (c >= h) continue;
      uint32_t o[8];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        __nv_bfloat162 b = __floats2bfloat162_rn(acc[q][2 * u], acc[q][2 * u + 1]);
        o[u] = *reinterpret_cast<uint32_t*>(&b);
      }
      stg256(out + i * h + c, o);
    }
  }
}

template <bool WEIGHTED>
void launch_gather_reduce_bf16(const __nv_bfloat16* rows, const float* w, int64_t t0, int64_t t1, int k, int h,
                               const ChunkMeta& m, __nv_bfloat16* out, const float* dw_row, float* dscore,
                               cudaStream_t st) {
  const dim3 grid((unsigned)ceil_div64(t1 - t0, 8));
  if (k <= 2)
    launch_pdl(gather_reduce_bf16_kernel<WEIGHTED, 2>, grid, dim3(256), 0, st, rows, w, t0, t1, k, h, m.dest_of,
               m.info, out, dw_row, dscore);
  else
    launch_pdl(gather_reduce_bf16_kernel<WEIGHTED, 4>, grid, dim3(256), 0, st, rows, w, t0, t1, k, h, m.dest_of,
               m.info, out, dw_row, dscore);
}

template <typename T>
void launch_combine(const T* O, const float* w, int64_t t0, int64_t t1, int k, int h, const ChunkMeta& m, T* y,
                    cudaStream_t st) {
  int64_t n = t1 - t0;
  if (n == 0) return;
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    if (h % 16 == 0) return launch_gather_reduce_bf16<true>(O, w, t0, t1, k, h, m, y, nullptr, nullptr, st);
  }
  launch_pdl(gather_reduce_kernel<T, true>, dim3((unsigned)ceil_div64(n, 8)), dim3(256), 0, st, O, w, t0, t1, k, h, m.dest_of, m.info,
                                                                           y, nullptr, nullptr);
}

template <typename T>
void launch_unpermute_reduce(const T* dXd, int64_t t0, int64_t t1, int k, int h, const ChunkMeta& m, T* dx,
                             float* dscore, cudaStream_t st) {
  int64_t n = t1 - t0;
  if (n == 0) return;
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    if (h % 16 == 0) return launch_gather_reduce_bf16<false>(dXd, nullptr, t0, t1, k, h, m, dx, m.dw_row, dscore, st);
  }
  launch_pdl(gather_reduce_kernel<T, false>, dim3((unsigned)ceil_div64(n, 8)), dim3(256), 0, st, dXd, nullptr, t0, t1, k, h, m.dest_of,
                                                                            m.info, dx, m.dw_row, dscore);
}

// EP > 1: received rows per local expert for chunk j from the all-gathered counts
// [EP][C][E]; padded segment starts (expert-major: local expert, then src rank, reading R3).
__global__ void ep_recv_seg_kernel(const int* __restrict__ counts, int C, int j, int E, int El, int me, int EP,
                                   int64_t rows_cap, int* __restrict__ seg, int* __restrict__ pseg,
                                   int* __restrict__ recv_cnt, int* __restrict__ info, int64_t* stats_rows,
                                   int64_t* stats_rows_pad, const int* __restrict__ gskip) {
  if (threadIdx.x != 0) return;
  int acc = 0, rows = 0, pairs = 0;
  for (int el = 0; el < El; el++) {
    int c = 0;
    for (int src = 0; src < EP; src++) c += counts[((int64_t)src * C + j) * E + me * El + el];
    recv_cnt[el] = c;
    seg[el] = acc;
    pseg[el] = pairs;
    int pad = (int)round_up64(c, kRowAlign);
    acc += pad;
    pairs += (pad / kRowAlign + 1) / 2;
    rows += c;
  }
  seg[El] = acc;
  pseg[El] = pairs;
  info[kInfoPairs] = pairs;
  info[kInfoRows] = rows;
  info[kInfoRowsPad] = acc;
  info[kInfoSkip] = (acc > rows_cap || (gskip && gskip[j])) ? 1 : 0;
  if (stats_rows) { stats_rows[j] = rows; stats_rows_pad[j] = acc; }
}

void launch_ep_recv_seg(const int* counts, int C, int j, int E, int El, int me, int EP, int64_t rows_cap,
                        const ChunkMeta& m, int64_t* stats_rows, int64_t* stats_rows_pad, cudaStream_t st,
                        const int* gskip) {
  ep_recv_seg_kernel<<<1, 32, 0, st>>>(counts, C, j, E, El, me, EP, rows_cap, m.seg, m.pseg, m.recv_cnt, m.info,
                                       stats_rows, stats_rows_pad, gskip);
}

// ------------------------------------------------------------------------------------------
// Fused EP exchange over peer memory.
// ------------------------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) p2p_push_kernel(const T* __restrict__ x, const T* __restrict__ dy,
                                                       const float* __restrict__ w, int k, int h, int E, int El,
                                                       const int* __restrict__ tab, const int* __restrict__ send_src,
                                                       const int* __restrict__ info, PeerTable pt) {
  if (info[kInfoSkip]) return;
  const int rows = info[kInfoSend];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  const int* send_off = tab;
  const int* land = tab + E + 1;
  constexpr int V = 16 / sizeof(T);
  const int nv = h / V;
  for (int r = blockIdx.x * (blockDim.x >> 5) + warp; r < rows; r += nwarps) {
    // expert of send row r: last e with send_off[e] <= r
    int lo = 0, hi = E;
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (__ldg(send_off + mid) <= r) lo = mid; else hi = mid;
    }
    const int e = lo, dst = e / El, el = e % El;
    const int64_t drow = (int64_t)__ldg(land + dst * El + el) + (r - __ldg(send_off + e));
    const int q = __ldg(send_src + r);
    const int64_t tok = q / k;
    const uint4* s = reinterpret_cast<const uint4*>(x + tok * h);
    uint4* d = reinterpret_cast<uint4*>(pt.X[dst] + drow * h * (int64_t)sizeof(T));
    const uint4* s2 = dy ? reinterpret_cast<const uint4*>(dy + tok * h) : nullptr;
    uint4* d2 = dy ? reinterpret_cast<uint4*>(pt.DY[dst] + drow * h * (int64_t)sizeof(T)) : nullptr;
    int i = lane;
    for (; i + 96 < nv; i += 128) {
      uint4 a0 = __ldg(s + i), a1 = __ldg(s + i + 32), a2 = __ldg(s + i + 64), a3 = __ldg(s + i + 96);
      if (s2) {
        uint4 b0 = __ldg(s2 + i), b1 = __ldg(s2 + i + 32), b2 = __ldg(s2 + i + 64), b3 = __ldg(s2 + i + 96);
        d2[i] = b0; d2[i + 32] = b1; d2[i + 64] = b2; d2[i + 96] = b3;
      }
      d[i] = a0; d[i + 32] = a1; d[i + 64] = a2; d[i + 96] = a3;
    }
    for (; i < nv; i += 32) {
      d[i] = __ldg(s + i);
      if (s2) d2[i] = __ldg(s2 + i);
    }
    if (lane == 0) reinterpret_cast<float*>(pt.w_row[dst])[drow] = __ldg(w + q);
  }
}

template <typename T>
void launch_p2p_push(const T* x, const T* dy, const float* w, int k, int h, int E, int El, int EP, const int* tab,
                     const int* send_src, const int* info, const PeerTable& pt, int64_t rows_ub, cudaStream_t st) {
  (void)EP;
  if (rows_ub <= 0) return;
  int blocks = (int)std::min<int64_t>(ceil_div64(rows_ub, 8), 148 * 16);
  p2p_push_kernel<T><<<blocks, 256, 0, st>>>(x, dy, w, k, h, E, El, tab, send_src, info, pt);
}

__global__ void p2p_row_addr_kernel(const int* __restrict__ seg, const int* __restrict__ recv_cnt, int El, int EP,
                                    const int* __restrict__ tab, int E, const int* __restrict__ info, PeerTable pt,
                                    int row_bytes, uint64_t* __restrict__ row_addr, uint64_t* __restrict__ row_addr_w) {
  const int rows = info[kInfoSkip] ? 0 : info[kInfoRowsPad];
  const int* recv_off = tab + E + 1 + EP * El;
  const int* ret = recv_off + EP * El;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
    const int el = expert_of_row(seg, El, r);
    uint64_t a = 0, aw = 0;
    if (r < __ldg(seg + el) + __ldg(recv_cnt + el)) {
      // source rank: last s with recv_off[s][el] <= r (segments of one expert are src-ordered)
      int s = 0;
      for (int s2 = 1; s2 < EP; s2++)
        if (__ldg(recv_off + s2 * El + el) <= r) s = s2;
      const int64_t pos = (int64_t)__ldg(ret + s * El + el) + (r - __ldg(recv_off + s * El + el));
      a = (uint64_t)(pt.send[s] + pos * row_bytes);
      aw = pt.send_w[s] ? (uint64_t)(pt.send_w[s] + pos * 4) : 0;
    }
    row_addr[r] = a;
    if (row_addr_w) row_addr_w[r] = aw;
  }
}

void launch_p2p_row_addr(const int* seg, const int* recv_cnt, int El, int EP, const int* tab, int E, const int* info,
                         const PeerTable& pt, int row_bytes, uint64_t* row_addr, uint64_t* row_addr_w,
                         int64_t rows_cap, cudaStream_t st) {
  if (rows_cap <= 0) return;
  int blocks = (int)std::min<int64_t>(ceil_div64(rows_cap, 256), 148 * 8);
  p2p_row_addr_kernel<<<blocks, 256, 0, st>>>(seg, recv_cnt, El, EP, tab, E, info, pt, row_bytes, row_addr,
                                               row_addr_w);
}

__global__ void p2p_push_dw_kernel(const float* __restrict__ dw_row, const uint64_t* __restrict__ row_addr_w,
                                   const int* __restrict__ info) {
  if (info[kInfoSkip]) return;
  const int rows = info[kInfoRowsPad];
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
    uint64_t a = row_addr_w[r];
    if (a) *reinterpret_cast<float*>(a) = dw_row[r];
  }
}

void launch_p2p_push_dw(const float* dw_row, const uint64_t* row_addr_w, const int* info, int64_t rows_cap,
                        cudaStream_t st) {
  if (rows_cap <= 0) return;
  int blocks = (int)std::min<int64_t>(ceil_div64(rows_cap, 256), 148 * 8);
  p2p_push_dw_kernel<<<blocks, 256, 0, st>>>(dw_row, row_addr_w, info);
}

// ------------------------------------------------------------------------------------------
// N1: device-planned exchange ("first notification"): the count
// all-gather, the chunk tables and the fences run on the device; the host never waits.
// ------------------------------------------------------------------------------------------
uint64_t sync_area_bytes(int E) {
  return sizeof(uint64_t) * (1 + (uint64_t)kSyncPhases * kMaxPeers) +
         sizeof(int) * 2ull * kMaxPeers * kMaxSub * (uint64_t)E;
}
__device__ __forceinline__ uint64_t* sync_flags(uint64_t* area) { return area + 1; }
__device__ __forceinline__ int* sync_counts(uint64_t* area, int E, int parity, int src) {
  return reinterpret_cast<int*>(area + 1 + kSyncPhases * kMaxPeers) + ((int64_t)parity * kMaxPeers + src) * kMaxSub * E;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void sync_epoch_kernel(uint64_t* area) {
  if (threadIdx.x == 0 && blockIdx.x == 0) area[0] += 1;
}
void launch_sync_epoch(uint64_t* area, cudaStream_t st) { sync_epoch_kernel<<<1, 32, 0, st>>>(area); }

// block p: this rank's counts into peer p's landing zone, then (after the block's stores) its flag
__global__ void sync_push_counts_kernel(const int* __restrict__ mine, int n, int E, SyncPeers sp, int me) {
  const int p = blockIdx.x;
  const uint64_t ep = sp.area[me][0];
  int* dst = sync_counts(sp.area[p], E, (int)(ep & 1), me);
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = mine[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    st_release_sys(sync_flags(sp.area[p]) + 0 * kMaxPeers + me, ep * 256);
  }
}
void launch_sync_push_counts(const int* mine, int C, int E, const SyncPeers& sp, int me, cudaStream_t st) {
  sync_push_counts_kernel<<<sp.n, 256, 0, st>>>(mine, C * E, E, sp, me);
}

__global__ void sync_signal_kernel(SyncPeers sp, int me, int phase, int code) {
  if (threadIdx.x != 0) return;
  const uint64_t v = sp.area[me][0] * 256 + (uint64_t)code;
  __threadfence_system();   // this stream's earlier kernels (their peer stores) before the flag
  for (int p = 0; p < sp.n; p++) st_release_sys(sync_flags(sp.area[p]) + phase * kMaxPeers + me, v);
}
void launch_sync_signal(const SyncPeers& sp, int me, int phase, int code, cudaStream_t st) {
  sync_signal_kernel<<<1, 32, 0, st>>>(sp, me, phase, code);
}

__global__ void sync_wait_kernel(uint64_t* area, int EP, int me, int phase, int code, int* status) {
  const int p = threadIdx.x;
  if (p >= EP || p == me) return;
  const uint64_t target = (uint64_t)((int64_t)area[0] * 256 + code);
  const uint64_t* f = sync_flags(area) + phase * kMaxPeers + p;
  const uint64_t t0 = globaltimer();
  while (ld_acquire_sys(f) < target) {
    if (globaltimer() - t0 > 20000000000ull) {   // 20 s: a peer never arrived - latch, do not hang
      printf("memfine: rank %d timed out waiting for rank %d, phase %d: flag %llu < target %llu (epoch %llu)\n", me,
             p, phase, (unsigned long long)ld_acquire_sys(f), (unsigned long long)target,
             (unsigned long long)area[0]);
      latch_error(status, MEMFINE_ERR_CUDA);
      return;
    }
    __nanosleep(256);
  }
}
void launch_sync_wait(uint64_t* area, int EP, int me, int phase, int code, int* status, cudaStream_t st) {
  sync_wait_kernel<<<1, 32, 0, st>>>(area, EP, me, phase, code, status);
}

// One block per chunk j: the landed counts -> counts_all [EP][C][E] (block 0 copies), and chunk j's
// table: send_off (this rank's chunk copies over global experts), land[p][el] (where this rank's rows of
// expert (p, el) start in p's expert-major buffer), recv_off[s][el] (where s's rows of my local expert el
// start in mine), ret[s][el] (s's send-layout position of its copies of (me, el)); plus the global skip.
__global__ void p2p_tables_kernel(const uint64_t* __restrict__ area_c, int C, int E, int El, int EP, int me,
                                  int64_t rows_cap, int64_t send_cap, int* __restrict__ counts_all,
                                  int* __restrict__ p2p_tab, int* __restrict__ gskip, int* status) {
  uint64_t* area = const_cast<uint64_t*>(area_c);
  const int parity = (int)(area[0] & 1);
  const int j = blockIdx.x;
  auto cnt = [&](int src, int e) -> int { return sync_counts(area, E, parity, src)[(int64_t)j * E + e]; };
  if (j == 0)
    for (int i = threadIdx.x; i < EP * C * E; i += blockDim.x) {
      const int src = i / (C * E), r = i % (C * E);
      counts_all[i] = sync_counts(area, E, parity, src)[r];
    }
  int* tab = p2p_tab + (int64_t)j * (4 * E + 1);
  int* send_off = tab;
  int* land = tab + E + 1;
  int* roff = land + EP * El;
  int* ret = roff + EP * El;
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int e = 0; e < E; e++) { send_off[e] = acc; acc += cnt(me, e); }
    send_off[E] = acc;
  }
  // per rank p (one thread each): p's padded expert-major layout for chunk j and its send prefix
  for (int p = threadIdx.x; p < EP; p += blockDim.x) {
    int64_t acc = 0, sendp = 0;
    for (int e = 0; e < E; e++) sendp += cnt(p, e);
    for (int el = 0; el < El; el++) {
      int64_t run = acc;
      for (int s = 0; s < EP; s++) {
        const int c = cnt(s, p * El + el);
        if (s == me) land[p * El + el] = (int)run;   // my rows of expert (p, el) in p's buffer
        if (p == me) roff[s * El + el] = (int)run;   // s's rows of my expert el in my buffer
        run += c;
      }
      acc += (run - acc + kRowAlign - 1) / kRowAlign * kRowAlign;
    }
    // ret[p][el]: p's send-layout position of its copies of my expert el = prefix over global experts
    int64_t pre = 0;
    for (int e = 0; e < me * El; e++) pre += cnt(p, e);
    for (int el = 0; el < El; el++) {
      ret[p * El + el] = (int)pre;
      pre += cnt(p, me * El + el);
    }
    if (acc > rows_cap || sendp > send_cap) atomicOr(&bad, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    gskip[j] = bad;
    if (bad) latch_error(status, MEMFINE_ERR_WORKSPACE);
  }
}
void launch_p2p_tables(const uint64_t* area, int C, int E, int El, int EP, int me, int64_t rows_cap,
                       int64_t send_cap, int* counts_all, int* p2p_tab, int* gskip, int* status, cudaStream_t st) {
  p2p_tables_kernel<<<C, 256, 0, st>>>(area, C, E, El, EP, me, rows_cap, send_cap, counts_all, p2p_tab, gskip,
                                       status);
}

// ------------------------------------------------------------------------------------------
// A3: MACT tuner.  plan_from_subsums is the one evaluation used by both the host path and
// the device kernel (same integer arithmetic, so both are bit-identical by construction).
// ------------------------------------------------------------------------------------------
__host__ __device__ int plan_from_subsums(const int64_t* sub, const PlanParams& p, memfine_plan_info* out) {
  memfine_plan_info o;
  o.C = o.c_theory = o.clamped = o.feasible = o.hot_rank = o.exact_peak = 0;
  o.s_dd_max = o.s_prime_max = o.s_chunk_max = 0;
  o.predicted_peak_bytes = 0;
  // Eq. 8 numerator (bytes): B - M^sta - s-term.
  unsigned long long B = p.budget;
  unsigned long long used = p.static_bytes + p.other_bytes;
  if (used < p.static_bytes || B <= used) { *out = o; return MEMFINE_ERR_INFEASIBLE; }
  unsigned long long num = B - used;
  // s'_max = floor(num * tp * cp / (m_g * D_t * b * (2h + 2g)))
  unsigned long long den = (unsigned long long)p.m_g * p.D_t * p.micro_batch * (2ull * p.h + 2ull * p.g);
  unsigned long long tc = (unsigned long long)p.tp * p.cp;
  // num * tc may overflow 64 bits only beyond 2^64 bytes * tc; split the division.
  unsigned long long q1 = num / den, r1 = num % den;
  unsigned long long spm = q1 * tc + (r1 * tc) / den;
  o.s_prime_max = (int64_t)spm;
  if (spm == 0) { *out = o; return MEMFINE_ERR_INFEASIBLE; }
  int64_t sdd = -1;
  int hot = 0;
  for (int r = 0; r < p.EP; r++) {
    int64_t s = 0;
    for (int j = 0; j < p.nsub; j++) s += sub[r * p.nsub + j];
    if (s > sdd) { sdd = s; hot = r; }
  }
  o.s_dd_max = sdd;
  o.hot_rank = hot;
  int64_t c = (sdd + (int64_t)spm - 1) / (int64_t)spm;
  if (c < 1) c = 1;
  o.c_theory = (int32_t)(c > 0x7fffffff ? 0x7fffffff : c);
  int C = -1;
  if (p.rule == MEMFINE_RULE_EQ9) {
    for (int i = 0; i < p.nbins; i++)
      if (p.bins[i] >= c) { C = p.bins[i]; break; }
  } else {
    for (int i = 0; i < p.nbins; i++)
      if (p.nsub % p.bins[i] != 0) { *out = o; return MEMFINE_ERR_INVALID_ARG; }
    for (int i = 0; i < p.nbins && C < 0; i++) {
      int Cb = p.bins[i], per = p.nsub / Cb;
      int64_t mx = 0;
      for (int r = 0; r < p.EP; r++)
        for (int jc = 0; jc < Cb; jc++) {
          int64_t s = 0;
          for (int j = jc * per; j < (jc + 1) * per; j++) s += sub[r * p.nsub + j];
          if (s > mx) mx = s;
        }
      if (mx <= (int64_t)spm) C = Cb;
    }
  }
  if (C < 0) { C = p.bins[p.nbins - 1]; o.clamped = 1; }
  o.C = C;
  int64_t mx = 0;
  if (p.nsub % C == 0) {
    int per = p.nsub / C;
    o.exact_peak = 1;
    for (int r = 0; r < p.EP; r++)
      for (int jc = 0; jc < C; jc++) {
        int64_t s = 0;
        for (int j = jc * per; j < (jc + 1) * per; j++) s += sub[r * p.nsub + j];
        if (s > mx) mx = s;
      }
  } else {
    o.exact_peak = 0;
    mx = (sdd + C - 1) / C;
  }
  o.s_chunk_max = mx;
  o.feasible = mx <= (int64_t)spm ? 1 : 0;
  o.predicted_peak_bytes =
      ((unsigned long long)p.m_g * p.D_t * p.micro_batch * (unsigned long long)mx * (2ull * p.h + 2ull * p.g)) / tc;
  *out = o;
  return MEMFINE_OK;
}

// One CTA: per-(rank, sub-chunk) received-copy sums via smem reduction, then thread 0
// evaluates Eqs. 8-9 and the bins; the result lands in pinned mapped host memory.
__global__ void plan_kernel(const int32_t* __restrict__ counts, PlanParams p, memfine_plan_info* out, int* rc,
                            unsigned long long* sub_g) {
  extern __shared__ unsigned long long sub_s[];  // [EP * nsub] (in global memory when it exceeds 48 KB)
  unsigned long long* sub_u = sub_g ? sub_g : sub_s;
  int n = p.EP * p.nsub;
  for (int i = threadIdx.x; i < n; i += blockDim.x) sub_u[i] = 0ull;
  __syncthreads();
  int El = p.E / p.EP;
  int64_t total = (int64_t)p.EP * p.nsub * p.E;
  for (int64_t q = threadIdx.x; q < total; q += blockDim.x) {
    int e = (int)(q % p.E);
    int j = (int)((q / p.E) % p.nsub);
    int r = e / El;
    int v = counts[q];
    if (v) atomicAdd(&sub_u[r * p.nsub + j], (unsigned long long)v);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *rc = plan_from_subsums(reinterpret_cast<const int64_t*>(sub_u), p, out);
    __threadfence_system();
  }
}

int launch_plan_kernel(const int32_t* counts_dev, const PlanParams& p, memfine_plan_info* out_mapped, int* rc_mapped,
                       cudaStream_t st) {
  // per-(rank, sub-chunk) sums: shared memory up to 48 KB (EP * nsub <= 6144), else a device scratch
  const size_t bytes = sizeof(unsigned long long) * (size_t)p.EP * p.nsub;
  unsigned long long* scratch = nullptr;
  if (bytes > 48 * 1024 && cudaMallocAsync((void**)&scratch, bytes, st) != cudaSuccess) return -1;
  plan_kernel<<<1, 1024, scratch ? 0 : bytes, st>>>(counts_dev, p, out_mapped, rc_mapped, scratch);
  const cudaError_t e = cudaGetLastError();
  if (scratch) cudaFreeAsync(scratch, st);
  return e == cudaSuccess ? 0 : -1;
}

// ------------------------------------------------------------------------------------------
template void launch_dispatch_scatter<__nv_bfloat16>(const __nv_bfloat16*, const __nv_bfloat16*, const int32_t*,
                                                     const float*, int64_t, int64_t, int, int, int, const ChunkMeta&,
                                                     __nv_bfloat16*, __nv_bfloat16*, int, bool, int64_t, cudaStream_t,
                                                     uint8_t*, uint8_t*, bool);
template void launch_dispatch_scatter<float>(const float*, const float*, const int32_t*, const float*, int64_t,
                                             int64_t, int, int, int, const ChunkMeta&, float*, float*, int, bool,
                                             int64_t, cudaStream_t, uint8_t*, uint8_t*, bool);
template void launch_p2p_push<__nv_bfloat16>(const __nv_bfloat16*, const __nv_bfloat16*, const float*, int, int, int,
                                             int, int, const int*, const int*, const int*, const PeerTable&,
                                             int64_t, cudaStream_t);
template void launch_p2p_push<float>(const float*, const float*, const float*, int, int, int, int, int, const int*,
                                     const int*, const int*, const PeerTable&, int64_t, cudaStream_t);
template void launch_zero_padding<__nv_bfloat16>(int, int, const ChunkMeta&, __nv_bfloat16*, __nv_bfloat16*,
                                                 cudaStream_t);
template void launch_zero_padding<float>(int, int, const ChunkMeta&, float*, float*, cudaStream_t);
template void launch_combine<__nv_bfloat16>(const __nv_bfloat16*, const float*, int64_t, int64_t, int, int,
                                            const ChunkMeta&, __nv_bfloat16*, cudaStream_t);
template void launch_combine<float>(const float*, const float*, int64_t, int64_t, int, int, const ChunkMeta&, float*,
                                    cudaStream_t);
template void launch_unpermute_reduce<__nv_bfloat16>(const __nv_bfloat16*, int64_t, int64_t, int, int,
                                                     const ChunkMeta&, __nv_bfloat16*, float*, cudaStream_t);
template void launch_unpermute_reduce<float>(const float*, int64_t, int64_t, int, int, const ChunkMeta&, float*,
                                             float*, cudaStream_t);

const void* kernel_anchor_route() { return (const void*)sync_wait_kernel; }

}  // namespace memfine
