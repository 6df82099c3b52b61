// mx.cu — MXFP8 operand quantisation for the block-scaled expert GEMMs (
// DESIGN.md reading R28): E4M3 codes, K-major, with E8M0 block scales written straight into the
// tcgen05 scale-factor chunk layout (common.cuh mx_sf_off), so the GEMM producer moves them with
// one 512-byte bulk copy per 128 rows x 128 K.
#include <algorithm>
#include "kernels.h"

namespace memfine {

// Row-wise: src [rows][K] bf16 (row stride ld) -> q [rows][K] E4M3, sf chunks.  One thread per 8
// consecutive elements (one 16-B load), 4 threads per 32-element block (amax by two shuffles).
// With a chunk's info words: rows = its padded rows (0 when the chunk is skipped), at most rows_max.
__global__ void __launch_bounds__(256) mx_quant_rows_kernel(const __nv_bfloat16* __restrict__ src, int64_t ld,
                                                            int64_t rows_max, const int* __restrict__ info,
                                                            int K, uint8_t* __restrict__ q,
                                                            uint8_t* __restrict__ sf) {
  pdl_wait();
  pdl_trigger();
  int64_t rows = rows_max;
  if (info) rows = __ldg(info + kInfoSkip) ? 0 : min(rows_max, (int64_t)__ldg(info + kInfoRowsPad));
  const int per_row = K >> 3;
  const int64_t n = rows * per_row;
  // whole warps iterate together (full-mask shuffles); the 4 threads of a block share ok
  // (n and per_row are multiples of 4)
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i - (threadIdx.x & 31) < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool ok = i < n;
    const int64_t r = ok ? i / per_row : 0;
    const int s = ok ? (int)(i % per_row) : 0;
    uint4 u = ok ? *reinterpret_cast<const uint4*>(src + r * ld + (int64_t)s * 8) : make_uint4(0, 0, 0, 0);
    float v[8];
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int j = 0; j < 4; j++) {
      v[2 * j] = __uint_as_float(w[j] << 16);
      v[2 * j + 1] = __uint_as_float(w[j] & 0xFFFF0000u);
    }
    float amax = 0.f;
#pragma unroll
    for (int j = 0; j < 8; j++) amax = fmaxf(amax, fabsf(v[j]));
    amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 1));
    amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 2));
    const int E = mx_exp(amax);
    const float inv = mx_inv_scale(E);
    uint2 o;
    o.x = mx_e4m3x2(v[0] * inv, v[1] * inv) | (mx_e4m3x2(v[2] * inv, v[3] * inv) << 16);
    o.y = mx_e4m3x2(v[4] * inv, v[5] * inv) | (mx_e4m3x2(v[6] * inv, v[7] * inv) << 16);
    if (ok) {
      *reinterpret_cast<uint2*>(q + r * K + (int64_t)s * 8) = o;
      if ((s & 3) == 0) sf[mx_sf_off(r, s >> 2, K)] = (uint8_t)(E + 127);
    }
  }
}

// Both layouts of one weight in one pass (W_gate, W_up): src [B][R][Cc] bf16 ->
//   q_rows [B][R][Cc] blocked along Cc (the forward's K = h) and q_t [B][Cc][R] blocked along R
//   (dX's K = g), each with its scale chunks.  Tile 128 x 128 through smem, read once.
__global__ void __launch_bounds__(256) mx_quant_dual_kernel(const __nv_bfloat16* __restrict__ src, int R, int Cc,
                                                            uint8_t* __restrict__ q_rows, uint8_t* __restrict__ sf_rows,
                                                            uint8_t* __restrict__ q_t, uint8_t* __restrict__ sf_t) {
  // rows of 65 words: a warp reading one word per lane is conflict-free both along a row (lanes =
  // adjacent column pairs) and down a column (lanes = adjacent rows, 65 = 1 mod 32)
  __shared__ uint32_t t[128][65];
  const int b = blockIdx.z, r0 = blockIdx.y * 128, c0 = blockIdx.x * 128;
  const __nv_bfloat16* s = src + (int64_t)b * R * Cc;
#pragma unroll
  for (int pass = 0; pass < 8; pass++) {
    const int idx = pass * 256 + threadIdx.x;    // 16 x uint4 per row
    const int rr = idx >> 4, cw = (idx & 15) * 4;
    const uint4 u = *reinterpret_cast<const uint4*>(s + (int64_t)(r0 + rr) * Cc + c0 + cw * 2);
    t[rr][cw] = u.x; t[rr][cw + 1] = u.y; t[rr][cw + 2] = u.z; t[rr][cw + 3] = u.w;
  }
  __syncthreads();
  auto quant32 = [](const float (&v)[32], float amax, uint8_t* q, uint8_t* sf) {
    const int E = mx_exp(amax);
    const float inv = mx_inv_scale(E);
    uint32_t o[8];
#pragma unroll
    for (int j = 0; j < 8; j++)
      o[j] = mx_e4m3x2(v[4 * j] * inv, v[4 * j + 1] * inv) | (mx_e4m3x2(v[4 * j + 2] * inv, v[4 * j + 3] * inv) << 16);
    reinterpret_cast<uint4*>(q)[0] = make_uint4(o[0], o[1], o[2], o[3]);
    reinterpret_cast<uint4*>(q)[1] = make_uint4(o[4], o[5], o[6], o[7]);
    *sf = (uint8_t)(E + 127);
  };
  {
    // row-wise: thread = (row, half of the 128 columns): two 32-column blocks along Cc
    const int row = threadIdx.x & 127, hf = threadIdx.x >> 7;
    const int64_t gr = (int64_t)b * R + r0 + row;
#pragma unroll
    for (int k2 = 0; k2 < 2; k2++) {
      const int kb = hf * 2 + k2;
      float v[32];
      float amax = 0.f;
#pragma unroll
      for (int i = 0; i < 16; i++) {
        const uint32_t u = t[row][16 * kb + i];
        v[2 * i] = __uint_as_float(u << 16);
        v[2 * i + 1] = __uint_as_float(u & 0xFFFF0000u);
        amax = fmaxf(amax, fmaxf(fabsf(v[2 * i]), fabsf(v[2 * i + 1])));
      }
      quant32(v, amax, q_rows + gr * Cc + c0 + 32 * kb, sf_rows + mx_sf_off(gr, (c0 >> 5) + kb, Cc));
    }
  }
  {
    // column-wise: thread = (column pair, 32-row block), two columns at once along R
    const int cp = threadIdx.x & 63, kb = threadIdx.x >> 6;
    float v0[32], v1[32];
    float a0 = 0.f, a1 = 0.f;
#pragma unroll
    for (int i = 0; i < 32; i++) {
      const uint32_t u = t[32 * kb + i][cp];
      v0[i] = __uint_as_float(u << 16);
      v1[i] = __uint_as_float(u & 0xFFFF0000u);
      a0 = fmaxf(a0, fabsf(v0[i]));
      a1 = fmaxf(a1, fabsf(v1[i]));
    }
#pragma unroll
    for (int hh = 0; hh < 2; hh++) {
      const int64_t gc = c0 + 2 * cp + hh;
      quant32(hh ? v1 : v0, hh ? a1 : a0, q_t + ((int64_t)b * Cc + gc) * R + r0 + 32 * kb,
              sf_t + (int64_t)b * Cc * (R / 32) + mx_sf_off(gc, (r0 >> 5) + kb, R));
    }
  }
}

// Columnwise ("transposed") quantisation of a chunk's activation rows for the MXFP8 weight
// gradients (reading R28c): per tensor z, src [rows][Cc] bf16 (row stride ld; rows = the chunk's
// padded rows from info) -> q_t [Cc][Rcap] E4M3 blocked along the rows (K = the copies), scales at
// mx_sf_off(col, row / 32, Rcap).  Expert segments start at multiples of 128 rows, so every 32-row
// block lies inside one segment (its padding rows are zero).  One launch for all tensors
// (blockIdx.z); tile 128 x 128 through smem; a warp quantises 32 adjacent columns of one 32-row
// block (conflict-free shared-memory reads along a row).
__global__ void __launch_bounds__(256) mx_quant_t_kernel(MxColTensors tz, const int* __restrict__ info, int64_t Rcap) {
  pdl_wait();
  pdl_trigger();
  // flat grid over the tensors' 128-column tiles (no empty blocks for the narrower tensors)
  int z = 0;
  while (z + 1 < tz.n && (int)blockIdx.x >= tz.tile0[z + 1]) z++;
  const MxColTensor& tt = tz.t[z];
  const int64_t rows = __ldg(info + kInfoSkip) ? 0 : min(Rcap, (int64_t)__ldg(info + kInfoRowsPad));
  const int64_t r0 = (int64_t)blockIdx.y * 128;
  const int c0 = ((int)blockIdx.x - tz.tile0[z]) * 128;
  if (r0 >= rows) return;
  __shared__ __nv_bfloat16 t[128][128 + 8];
  const __nv_bfloat16* src = tt.src;
#pragma unroll
  for (int pass = 0; pass < 8; pass++) {
    const int idx = pass * 256 + threadIdx.x;    // 16 x uint4 per row
    const int rr = idx >> 4, cc = (idx & 15) * 8;
    *reinterpret_cast<uint4*>(&t[rr][cc]) = *reinterpret_cast<const uint4*>(src + (r0 + rr) * tt.ld + c0 + cc);
  }
  __syncthreads();
  // thread = (column pair, 32-row block): 64 pairs x 4 blocks; a warp reads 32 adjacent bf16x2 words
  // of one row per step (conflict-free) and quantises two column blocks at once
  const int cp = threadIdx.x & 63, kb = threadIdx.x >> 6;
  float v0[32], v1[32];
  float a0 = 0.f, a1 = 0.f;
#pragma unroll
  for (int i = 0; i < 32; i++) {
    const uint32_t u = *reinterpret_cast<const uint32_t*>(&t[32 * kb + i][2 * cp]);
    v0[i] = __uint_as_float(u << 16);
    v1[i] = __uint_as_float(u & 0xFFFF0000u);
    a0 = fmaxf(a0, fabsf(v0[i]));
    a1 = fmaxf(a1, fabsf(v1[i]));
  }
  auto emit = [&](const float (&v)[32], float amax, int64_t gc) {
    const int E = mx_exp(amax);
    const float inv = mx_inv_scale(E);
    uint32_t o[8];
#pragma unroll
    for (int j = 0; j < 8; j++)
      o[j] = mx_e4m3x2(v[4 * j] * inv, v[4 * j + 1] * inv) | (mx_e4m3x2(v[4 * j + 2] * inv, v[4 * j + 3] * inv) << 16);
    uint4* q = reinterpret_cast<uint4*>(tt.q_t + gc * Rcap + r0 + 32 * kb);
    q[0] = make_uint4(o[0], o[1], o[2], o[3]);
    q[1] = make_uint4(o[4], o[5], o[6], o[7]);
    tt.sf_t[mx_sf_off(gc, (r0 >> 5) + kb, Rcap)] = (uint8_t)(E + 127);
  };
  emit(v0, a0, c0 + 2 * cp);
  emit(v1, a1, c0 + 2 * cp + 1);
}

void launch_mx_quant_t(const MxColTensors& tz, const int* info, int64_t Rcap, cudaStream_t st) {
  if (Rcap <= 0 || tz.n <= 0) return;
  MxColTensors f = tz;
  int tiles = 0;
  for (int i = 0; i < f.n; i++) { f.tile0[i] = tiles; tiles += f.t[i].Cc / 128; }
  for (int i = f.n; i < 5; i++) f.tile0[i] = tiles;
  if (tiles <= 0) return;
  dim3 grid((unsigned)tiles, (unsigned)(Rcap / 128));
  launch_pdl(mx_quant_t_kernel, dim3(grid), dim3(256), 0, st, f, info, Rcap);
}

void launch_mx_quant_dual(const __nv_bfloat16* src, int B, int R, int Cc, uint8_t* q_rows, uint8_t* sf_rows,
                          uint8_t* q_t, uint8_t* sf_t, cudaStream_t st) {
  if (B <= 0 || R <= 0 || Cc <= 0) return;
  dim3 grid((unsigned)(Cc / 128), (unsigned)(R / 128), (unsigned)B);
  mx_quant_dual_kernel<<<grid, 256, 0, st>>>(src, R, Cc, q_rows, sf_rows, q_t, sf_t);
}

void launch_mx_quant_rows(const __nv_bfloat16* src, int64_t ld, int64_t rows_max, const int* info, int K,
                          uint8_t* q, uint8_t* sf, cudaStream_t st) {
  const int64_t n = rows_max * (K / 8);
  if (n <= 0) return;
  const int64_t blocks = std::min<int64_t>(ceil_div64(n, 256), (int64_t)sm100_num_sms() * 16);
  launch_pdl(mx_quant_rows_kernel, dim3((unsigned)blocks), dim3(256), 0, st, src, ld, rows_max, info, K, q, sf);
}


const void* kernel_anchor_mx() { return (const void*)mx_quant_t_kernel; }

}  // namespace memfine
