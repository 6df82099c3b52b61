// tma_rmw_bench.cu — how fast can an epilogue read-modify-write fp32 in HBM on B200?
//
// The chunked backward accumulates the fp32 weight gradients across chunks (reading R18): every
// chunk after the first read-modify-writes dW.  The GEMM epilogue does it with
// cp.reduce.async.bulk.tensor .add.f32 from 32x32 swizzled staging boxes.  This microbenchmark
// measures the HBM rate of that primitive against the alternatives, on a 2 GB fp32 array
// (> L2), one CTA per SM, 8 warps each streaming 4 KB boxes:
//   reduce   TMA tensor reduce-add smem -> global           (8 B of DRAM traffic per element)
//   store    TMA tensor store smem -> global                  (4 B)
//   ldst     TMA tensor load global -> smem, then TMA store   (8 B; the "preload + overwrite" path)
//   ldg      LDG.128 / STG.128 read-add-write by threads      (8 B)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_rmw_bench tools/tma_rmw_bench.cu
//   ./tools/tma_rmw_bench            (prints one JSON line)
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("cuda %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int ROWS = 16384, COLS = 32768;   // 2 GiB fp32
constexpr int BOX = 32;                     // 32 x 32 fp32 = 4 KB boxes
constexpr int WARPS = 8, DEPTH = 4;         // boxes in flight per warp

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void __launch_bounds__(WARPS * 32) rmw_kernel(const __grid_constant__ CUtensorMap map, float* base) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (su32(smem_raw) & 1023)) & 1023);   // 128B swizzle: 1 KB aligned
  uint64_t (*bars)[DEPTH] = reinterpret_cast<uint64_t (*)[DEPTH]>(smem + WARPS * DEPTH * 4096);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* buf = smem + warp * DEPTH * 4096;
  const int nbx = COLS / BOX, nby = ROWS / BOX;
  const int64_t nbox = (int64_t)nbx * nby;
  const int64_t gw = (int64_t)blockIdx.x * WARPS + warp, nw = (int64_t)gridDim.x * WARPS;
  if (MODE == 4) {
    // red.global.add.v4.f32 from registers (fire-and-forget vector reductions at L2, no smem staging)
    for (int64_t b = gw; b < nbox; b += nw) {
      const int bx = (int)(b % nbx), by = (int)(b / nbx);
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const int r = by * BOX + i * 4 + (lane >> 3), c = bx * BOX + (lane & 7) * 4;
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(base + (int64_t)r * COLS + c), "f"(1.f),
                     "f"(1.f), "f"(1.f), "f"(1.f)
                     : "memory");
      }
    }
    return;
  }
  if (MODE == 5) {
    // the GEMM epilogue's layout: each lane owns one row and 32 consecutive columns (128 B)
    for (int64_t b = gw; b < nbox; b += nw) {
      const int bx = (int)(b % nbx), by = (int)(b / nbx);
      float* row = base + (int64_t)(by * BOX + lane) * COLS + bx * BOX;
#pragma unroll
      for (int i = 0; i < 8; i++)
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(row + 4 * i), "f"(1.f), "f"(1.f), "f"(1.f),
                     "f"(1.f)
                     : "memory");
    }
    return;
  }
  if (MODE == 3) {
    // thread read-add-write: each warp takes a box row by row (32 rows x 128 B)
    for (int64_t b = gw; b < nbox; b += nw) {
      const int bx = (int)(b % nbx), by = (int)(b / nbx);
      float4 v[8];
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const int r = by * BOX + i * 4 + (lane >> 3), c = bx * BOX + (lane & 7) * 4;
        v[i] = *reinterpret_cast<const float4*>(base + (int64_t)r * COLS + c);
      }
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const int r = by * BOX + i * 4 + (lane >> 3), c = bx * BOX + (lane & 7) * 4;
        v[i].x += 1.f; v[i].y += 1.f; v[i].z += 1.f; v[i].w += 1.f;
        *reinterpret_cast<float4*>(base + (int64_t)r * COLS + c) = v[i];
      }
    }
    return;
  }
  if (lane == 0) for (int d = 0; d < DEPTH; d++) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&bars[warp][d])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  if (lane != 0) return;
  int it = 0;
  uint32_t phase[DEPTH] = {0, 0, 0, 0};
  for (int64_t b = gw; b < nbox; b += nw, it++) {
    const int bx = (int)(b % nbx), by = (int)(b / nbx);
    const int slot = it % DEPTH;
    uint8_t* s = buf + slot * 4096;
    if (MODE == 6) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // one box in flight per warp
    else if (it >= DEPTH) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(DEPTH - 1) : "memory");
    if (MODE == 2) {
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&bars[warp][slot])), "r"(4096));
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              su32(s)), "l"(&map), "r"(bx * BOX), "r"(by * BOX), "r"(su32(&bars[warp][slot]))
          : "memory");
      asm volatile(
          "{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t@!p bra W;\n}" ::"r"(
              su32(&bars[warp][slot])), "r"(phase[slot])
          : "memory");
      phase[slot] ^= 1;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (MODE == 0 || MODE == 6)
      asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                       &map), "r"(su32(s)), "r"(bx * BOX), "r"(by * BOX)
                   : "memory");
    else
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&map),
                   "r"(su32(s)), "r"(bx * BOX), "r"(by * BOX)
                   : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  float* d = nullptr;
  const size_t bytes = (size_t)ROWS * COLS * 4;
  CK(cudaMalloc(&d, bytes));
  CK(cudaMemset(d, 0, bytes));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  auto enc = (CUresult(*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill))fn;
  CUtensorMap map;
  cuuint64_t gd[2] = {COLS, ROWS}, gs[1] = {(cuuint64_t)COLS * 4};
  cuuint32_t bx[2] = {BOX, BOX}, es[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, gd, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  const int smem = WARPS * DEPTH * 4096 + 2048;
  CK(cudaFuncSetAttribute(rmw_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(rmw_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(rmw_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(rmw_kernel<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const char* names[7] = {"reduce", "store", "ldst", "ldg", "redv4", "redv4_rowlane", "reduce_depth1"};
  const double traffic[7] = {8.0, 4.0, 8.0, 8.0, 8.0, 8.0, 8.0};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("{");
  // grid: every SM (x1, x2), then a subset of the SMs (how many SMs the HBM-bound dW accumulation
  // needs if it shares the GPU with a tensor-bound GEMM)
  const int grids[6] = {nsm, 2 * nsm, 16, 32, 64, 96};
  for (int gi = 0; gi < 6; gi++)
    for (int m = 0; m < 7; m++) {
      auto launch = [&]() {
        const int g = grids[gi];
        if (m == 0) rmw_kernel<0><<<g, WARPS * 32, smem>>>(map, d);
        if (m == 1) rmw_kernel<1><<<g, WARPS * 32, smem>>>(map, d);
        if (m == 2) rmw_kernel<2><<<g, WARPS * 32, smem>>>(map, d);
        if (m == 3) rmw_kernel<3><<<g, WARPS * 32, 0>>>(map, d);
        if (m == 4) rmw_kernel<4><<<g, WARPS * 32, 0>>>(map, d);
        if (m == 5) rmw_kernel<5><<<g, WARPS * 32, 0>>>(map, d);
        if (m == 6) rmw_kernel<6><<<g, WARPS * 32, smem>>>(map, d);
      };
      launch();
      CK(cudaDeviceSynchronize());
      const int reps = 5;
      cudaEventRecord(e0);
      for (int r = 0; r < reps; r++) launch();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double gbs = traffic[m] * ROWS * (double)COLS * reps / (ms * 1e-3) / 1e9;
      printf("%s\"%s_g%d\": %.0f", (gi == 0 && m == 0) ? "" : ", ", names[m], grids[gi], gbs);
    }
  printf(", \"unit\": \"GB/s of DRAM traffic (algorithmic)\", \"array_gb\": %.2f}\n", bytes / 1e9);
  return 0;
}
