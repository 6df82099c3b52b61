// gemm_simt.cu — CUDA-core (FFMA) grouped expert GEMMs with the fused MoE epilogues.
// This is the MEMFINE_FP32 path (tcgen05 kind::tf32 cannot meet 1e-5),
// fp32 accumulation in a fixed k order.  The bf16 hot path is gemm_sm100.cu (tcgen05).
//
// Operand conventions (row-major storage, per local expert e, padded segment rows):
//   GATEUP   A = X[R,h]        B = W_gate[e], W_up[e]  [g,h]     (K-major both)
//   DOWN     A = a[R,g]        B = W_down[e] [h,g]              (K-major both)
//   DACT     A = dY[R,h]       B(n,k) = W_down[e][k][n]         (B MN-major)
//   DX       A = dGU[R,2g]     B(n,k) = W_gate/up[e][k][n]      (B MN-major, K split at g)
//   WGRAD_*  A(m,k) = rows[s0+k][m], B(n,k) = rows[s0+k][n]     (both MN-major, K = tokens)
#include "kernels.h"

namespace memfine {

constexpr int SB = 64;   // tile M and N
constexpr int SK = 16;   // tile K

template <typename T>
struct SimtOps {
  const GemmProblem<T>& p;
  int e, row0;  // expert, first padded row (M-tiled kinds) or segment start (WGRAD)
  __device__ SimtOps(const GemmProblem<T>& pp, int ee, int r0) : p(pp), e(ee), row0(r0) {}
  __device__ float a(int m, int k) const {
    switch (p.kind) {
      case GK_GATEUP: return Elt<T>::to_f(p.X[(int64_t)(row0 + m) * p.h + k]);
      case GK_DOWN: return Elt<T>::to_f(p.A[(int64_t)(row0 + m) * p.g + k]);
      case GK_DACT: return Elt<T>::to_f(p.DY[(int64_t)(row0 + m) * p.h + k]);
      case GK_DX: return Elt<T>::to_f(p.GU[(int64_t)(row0 + m) * 2 * p.g + k]);
      case GK_WGRAD_DOWN: return Elt<T>::to_f(p.DY[(int64_t)(row0 + k) * p.h + m]);
      default: return Elt<T>::to_f(p.GU[(int64_t)(row0 + k) * 2 * p.g + m]);
    }
  }
  // second B (W_up) only for GATEUP
  __device__ float b(int n, int k, int which) const {
    switch (p.kind) {
      case GK_GATEUP:
        return Elt<T>::to_f((which ? p.Wu : p.Wg)[((int64_t)e * p.g + n) * p.h + k]);
      case GK_DOWN: return Elt<T>::to_f(p.Wd[((int64_t)e * p.h + n) * p.g + k]);
      case GK_DACT: return Elt<T>::to_f(p.Wd[((int64_t)e * p.h + k) * p.g + n]);
      case GK_DX:
        return k < p.g ? Elt<T>::to_f(p.Wg[((int64_t)e * p.g + k) * p.h + n])
                       : Elt<T>::to_f(p.Wu[((int64_t)e * p.g + (k - p.g)) * p.h + n]);
      case GK_WGRAD_DOWN: return Elt<T>::to_f(p.A[(int64_t)(row0 + k) * p.g + n]);
      default: return Elt<T>::to_f(p.X[(int64_t)(row0 + k) * p.h + n]);
    }
  }
};

template <typename T, bool DUAL>
__global__ void __launch_bounds__(256) gemm_simt_kernel(GemmProblem<T> p, int M, int N, int K) {
  const bool wgrad = p.kind >= GK_WGRAD_DOWN;
  int e, row0, m0;
  int Kc = K;
  if (wgrad) {
    e = blockIdx.z;
    row0 = p.seg[e];
    Kc = p.seg[e + 1] - row0;
    m0 = blockIdx.y * SB;
    if (p.info[kInfoSkip]) return;
    if (Kc == 0 && p.wgrad_beta) return;
  } else {
    int rows = p.info[kInfoRowsPad];
    m0 = blockIdx.y * SB;
    if (p.info[kInfoSkip] || m0 >= rows) return;
    e = expert_of_row(p.seg, p.El, m0);
    row0 = m0;
    m0 = 0;
  }
  SimtOps<T> op(p, e, row0);
  int n0 = blockIdx.x * SB;
  __shared__ float As[SK][SB + 4];
  __shared__ float Bs[SK][SB + 4];
  __shared__ float Bs2[DUAL ? SK : 1][SB + 4];
  int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {}, acc2[DUAL ? 4 : 1][DUAL ? 4 : 1] = {};
  for (int k0 = 0; k0 < Kc; k0 += SK) {
    for (int i = threadIdx.x; i < SK * SB; i += 256) {
      int kk = i / SB, mm = i % SB;   // mm fastest: coalesced for MN-major operands
      int kg = k0 + kk;
      int mg = m0 + mm, ng = n0 + mm;
      As[kk][mm] = (kg < Kc && mg < M) ? op.a(mg, kg) : 0.f;
      Bs[kk][mm] = (kg < Kc && ng < N) ? op.b(ng, kg, 0) : 0.f;
      if (DUAL) Bs2[kk][mm] = (kg < Kc && ng < N) ? op.b(ng, kg, 1) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SK; kk++) {
      float av[4], bv[4], bv2[4];
#pragma unroll
      for (int i = 0; i < 4; i++) { av[i] = As[kk][ty * 4 + i]; bv[i] = Bs[kk][tx * 4 + i]; }
      if (DUAL) {
#pragma unroll
        for (int i = 0; i < 4; i++) bv2[i] = Bs2[kk][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) {
          acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
          if (DUAL) acc2[i][j] = fmaf(av[i], bv2[j], acc2[i][j]);
        }
    }
    __syncthreads();
  }
  // ---------------------------------------------------------------- epilogues
  for (int i = 0; i < 4; i++) {
    int m = m0 + ty * 4 + i;
    if (m >= M) continue;
    int64_t row = row0 + m;  // for M-tiled kinds
    float dwp = 0.f;
    for (int j = 0; j < 4; j++) {
      int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      float v = acc[i][j];
      switch (p.kind) {
        case GK_GATEUP: {
          float G = v, U = DUAL ? acc2[i][j] : 0.f;
          if (p.store_a) p.A[row * p.g + n] = Elt<T>::from_f(silu_exact(G) * U);
          if (p.store_gu) {
            p.GU[row * 2 * p.g + n] = Elt<T>::from_f(G);
            p.GU[row * 2 * p.g + p.g + n] = Elt<T>::from_f(U);
          }
          break;
        }
        case GK_DOWN:
        case GK_DX:
          if (p.row_addr) {
            const uint64_t a = p.row_addr[row];
            if (a) reinterpret_cast<T*>(a)[n] = Elt<T>::from_f(v);
          } else {
            p.O[row * p.h + n] = Elt<T>::from_f(v);
          }
          break;
        case GK_DACT: {
          float G = Elt<T>::to_f(p.GU[row * 2 * p.g + n]);
          float U = Elt<T>::to_f(p.GU[row * 2 * p.g + p.g + n]);
          float ws = p.w_row[row];
          float sg = sigmoid_exact(G);
          float a = G * sg * U;
          dwp = fmaf(v, a, dwp);
          float dA = ws * v;
          p.GU[row * 2 * p.g + n] = Elt<T>::from_f(dA * U * sg * (1.f + G * (1.f - sg)));
          p.GU[row * 2 * p.g + p.g + n] = Elt<T>::from_f(dA * G * sg);
          p.A[row * p.g + n] = Elt<T>::from_f(ws * a);
          break;
        }
        case GK_WGRAD_DOWN: {
          float* d = p.dWd + ((int64_t)e * p.h + m) * p.g + n;
          *d = p.wgrad_beta ? *d + v : v;
          break;
        }
        default: {
          float* d = (m < p.g) ? p.dWg + ((int64_t)e * p.g + m) * p.h + n
                               : p.dWu + ((int64_t)e * p.g + (m - p.g)) * p.h + n;
          *d = p.wgrad_beta ? *d + v : v;
          break;
        }
      }
    }
    if (p.kind == GK_DACT) atomicAdd(p.dw_row + row, dwp);
  }
}

template <typename T>
int launch_gemm_simt(const GemmProblem<T>& p, cudaStream_t st) {
  int M, N, K, gz = 1;
  int64_t mt = ceil_div64(p.rows_cap, SB);
  switch (p.kind) {
    case GK_GATEUP: N = p.g; K = p.h; break;
    case GK_DOWN: N = p.h; K = p.g; break;
    case GK_DACT: N = p.g; K = p.h; break;
    case GK_DX: N = p.h; K = 2 * p.g; break;
    case GK_WGRAD_DOWN: M = p.h; N = p.g; K = 0; gz = p.El; mt = ceil_div64(M, SB); break;
    default: M = 2 * p.g; N = p.h; K = 0; gz = p.El; mt = ceil_div64(M, SB); break;
  }
  if (p.kind < GK_WGRAD_DOWN) M = SB;  // per-tile rows (all rows valid: segments padded)
  if (mt == 0) return 0;
  dim3 grid((unsigned)ceil_div64(N, SB), (unsigned)mt, (unsigned)gz);
  if (p.kind == GK_GATEUP) gemm_simt_kernel<T, true><<<grid, 256, 0, st>>>(p, M, N, K);
  else gemm_simt_kernel<T, false><<<grid, 256, 0, st>>>(p, M, N, K);
  return 1;
}

template int launch_gemm_simt<float>(const GemmProblem<float>&, cudaStream_t);
template int launch_gemm_simt<__nv_bfloat16>(const GemmProblem<__nv_bfloat16>&, cudaStream_t);

const void* kernel_anchor_simt() { return (const void*)gemm_simt_kernel<float, true>; }

}  // namespace memfine
