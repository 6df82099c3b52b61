// gemm_sm100.cu — grouped expert GEMMs on the 5th-generation tensor cores (sm_100a).
//
// One persistent, warp-specialised kernel template serves the six expert GEMMs of the
// chunked MoE layer.  Per CTA (one per SM, 320 threads = 10 warps):
//   warp 0      TMA producer: cp.async.bulk.tensor 2D/3D loads, 128B swizzle, mbarrier tx
//   warp 1      TMEM allocator + MMA issuer: tcgen05.mma (BF16 kind::f16 or MXFP8
//               kind::mxf8f6f4.block_scale), FP32 accumulators in TMEM, tcgen05.commit -> mbarriers
//   warps 2..9  epilogue: tcgen05.ld 32x32b -> registers -> fused MoE epilogue -> global;
//               two warps per TMEM lane quarter (warp % 4), each taking half of the columns
// Default tiles are 256 x 256 per 2-CTA cluster (tcgen05.mma.cta_group::2, M = 256, issued by the
// even CTA; each CTA stages its 128 A rows and half of B): 32 KB per stage per CTA, as many stages as
// fit next to the epilogue staging (up to 6; nstage()).  Two TMEM accumulator stages (2 x 256 columns)
// let the epilogue of tile i overlap the mainloop of tile i+1 (MXFP8 N = 256: one stage + scale
// columns, drained early into registers).  MEMFINE_GEMM_CTA=1: 1-CTA 128 x 256 tiles (cta_group::1).
//
// Rows are the expert-major padded layout (every local expert's segment padded to 128
// rows), so an M tile never straddles experts and the weight-gradient K loop (over tokens)
// never straddles either; padded rows are zero.  Tile order is grouped (group_m M tiles x all N
// tiles, group_m sized per kind so the group's A strips fit an L2 budget).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <mutex>
#include <atomic>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <cmath>
#include "kernels.h"

namespace memfine {
namespace sm100 {

constexpr int BM = 128, BK = 64, EPI_WARPS = 8, THREADS = 64 + 32 * EPI_WARPS;
constexpr int A_BYTES = BM * BK * 2;  // 16 KB

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          su32(dst)),
      "l"(m), "r"(su32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(su32(dst)),
      "l"(m), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(m) : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// SMEM matrix descriptor (sm_100 UMMA): start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46),
// version 1 at [46,48), base offset 0, layout SWIZZLE_128B (2) at [61,64).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// Instruction descriptor, kind::f16: D f32, A/B bf16, majorness, N>>3, M>>4.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// the same without the wait (issue several, then one tmem_wait_ld)
__device__ __forceinline__ void tmem_ld32_nw(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_ftz(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}
// 32-byte global accesses (LDG/STG.E.ENL2.256 on sm_100): one thread moves half a 64-B row
// chunk per instruction, halving the L1 wavefronts of the row-per-thread epilogue.
__device__ __forceinline__ void st256(void* p, const uint32_t (&v)[8]) {
  asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
               "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void ld256(const void* p, uint32_t (&v)[8]) {
  asm volatile("ld.global.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "l"(p));
}
__device__ __forceinline__ void store32_bf16(__nv_bfloat16* dst, const float* v) {
#pragma unroll
  for (int i = 0; i < 2; i++) {
    uint32_t u[8];
#pragma unroll
    for (int j = 0; j < 8; j++) u[j] = pack_bf16(v[16 * i + 2 * j], v[16 * i + 2 * j + 1]);
    st256(dst + 16 * i, u);
  }
}
// raw bf16 pairs of a 32-element row chunk (two 32-byte loads)
__device__ __forceinline__ void load32_raw(const __nv_bfloat16* src, uint32_t (&u)[16]) {
  uint32_t a[8], b[8];
  ld256(src, a);
  ld256(src + 16, b);
#pragma unroll
  for (int j = 0; j < 8; j++) { u[j] = a[j]; u[8 + j] = b[j]; }
}
__device__ __forceinline__ void unpack32(const uint32_t (&u)[16], float* v) {
#pragma unroll
  for (int j = 0; j < 16; j++) {
    v[2 * j] = __uint_as_float(u[j] << 16);
    v[2 * j + 1] = __uint_as_float(u[j] & 0xFFFF0000u);
  }
}
__device__ __forceinline__ void store32_f32(float* dst, const float* v) {
#pragma unroll
  for (int i = 0; i < 4; i++) {
    uint32_t u[8];
#pragma unroll
    for (int j = 0; j < 8; j++) u[j] = __float_as_uint(v[8 * i + j]);
    st256(dst + 8 * i, u);
  }
}
__device__ __forceinline__ void add32_f32(float* dst, const float* v) {
#pragma unroll
  for (int i = 0; i < 4; i++) {
    uint32_t u[8];
    ld256(dst + 8 * i, u);
#pragma unroll
    for (int j = 0; j < 8; j++) u[j] = __float_as_uint(__uint_as_float(u[j]) + v[8 * i + j]);
    st256(dst + 8 * i, u);
  }
}

// One MXFP8 block from 32 bf16 values (two packed halves of 8 words): E4M3 codes (32 B, one
// 256-bit store) and the E8M0 scale byte (reading R28; the values are the stored bf16 ones, R28b).
__device__ __forceinline__ void mx_store_block_bf16(const uint32_t (&lo)[8], const uint32_t (&hi)[8], uint8_t* q,
                                                    uint8_t* sf) {
  float f[32];
  float amax = 0.f;
#pragma unroll
  for (int j = 0; j < 8; j++) {
    f[2 * j] = __uint_as_float(lo[j] << 16);
    f[2 * j + 1] = __uint_as_float(lo[j] & 0xFFFF0000u);
    f[16 + 2 * j] = __uint_as_float(hi[j] << 16);
    f[16 + 2 * j + 1] = __uint_as_float(hi[j] & 0xFFFF0000u);
  }
#pragma unroll
  for (int j = 0; j < 32; j++) amax = fmaxf(amax, fabsf(f[j]));
  const int E = mx_exp(amax);
  const float inv = mx_inv_scale(E);
  uint32_t o[8];
#pragma unroll
  for (int j = 0; j < 8; j++)
    o[j] = mx_e4m3x2(f[4 * j] * inv, f[4 * j + 1] * inv) | (mx_e4m3x2(f[4 * j + 2] * inv, f[4 * j + 3] * inv) << 16);
  st256(q, o);
  *sf = (uint8_t)(E + 127);
}

// TMA stores from shared memory (bulk async groups).  reduce = 1: element-wise add into global.
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* m, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(m),
               "r"(su32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* m, const void* src, int c0, int c1, int c2,
                                             bool reduce) {
  if (reduce)
    asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::
                     "l"(m),
                 "r"(su32(src)), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
  else
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(m),
                 "r"(su32(src)), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Staging writes in the TMA swizzle layouts.  bf16: 32 rows x 64 B, SWIZZLE_64B (16-B chunk c of
// row r at chunk c ^ ((r >> 1) & 3)); fp32: 32 rows x 128 B, SWIZZLE_128B (chunk c ^ (r & 7)).
// Both are bank-conflict-free for the row-per-thread writes of the 32x32b TMEM layout.
__device__ __forceinline__ void stage_bf16_row(uint8_t* buf, int r, const float* v) {
  uint8_t* row = buf + r * 64;
#pragma unroll
  for (int c = 0; c < 4; c++) {
    uint4 u = make_uint4(pack_bf16(v[8 * c], v[8 * c + 1]), pack_bf16(v[8 * c + 2], v[8 * c + 3]),
                         pack_bf16(v[8 * c + 4], v[8 * c + 5]), pack_bf16(v[8 * c + 6], v[8 * c + 7]));
    *reinterpret_cast<uint4*>(row + ((c ^ ((r >> 1) & 3)) << 4)) = u;
  }
}
__device__ __forceinline__ void stage_bf16_row_packed(uint8_t* buf, int r, const uint32_t (&u)[16]) {
  uint8_t* row = buf + r * 64;
#pragma unroll
  for (int c = 0; c < 4; c++)
    *reinterpret_cast<uint4*>(row + ((c ^ ((r >> 1) & 3)) << 4)) =
        make_uint4(u[4 * c], u[4 * c + 1], u[4 * c + 2], u[4 * c + 3]);
}
// fp32, 16 columns: 32 rows x 64 B in the SWIZZLE_64B layout (the bf16 staging's row shape)
__device__ __forceinline__ void stage_f32_row16(uint8_t* buf, int r, const float* v) {
  uint8_t* row = buf + r * 64;
#pragma unroll
  for (int c = 0; c < 4; c++)
    *reinterpret_cast<float4*>(row + ((c ^ ((r >> 1) & 3)) << 4)) =
        make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
}
__device__ __forceinline__ void stage_f32_row(uint8_t* buf, int r, const float* v) {
  uint8_t* row = buf + r * 128;
#pragma unroll
  for (int c = 0; c < 8; c++)
    *reinterpret_cast<float4*>(row + ((c ^ (r & 7)) << 4)) =
        make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
}

// ------------------------------------------------------------------ MXFP8 (block-scaled) helpers
// Instruction descriptor, kind::mxf8f6f4.block_scale: A/B E4M3 (format 0), K-major, N>>3 at 17,
// scale format E8M0 (bit 23), M>>4 at 24; the scale-factor byte ids (which of the 4 blocks of a
// 128-K chunk) of B at [4,6) and of A at [29,31).
__host__ __device__ constexpr uint32_t idesc_mx(int M, int N) {
  return ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_mx(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc,
                                       uint32_t tsfa, uint32_t tsfb) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], %1, %2, %3, [%5], [%6], p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(tsfa), "r"(tsfb)
      : "memory");
}
// SMEM descriptor of one 512-byte scale chunk (32 rows x 16 B, no swizzle; 8-row groups 128 B apart)
__device__ __forceinline__ uint64_t sdesc_sf(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)(128 >> 4) << 16;
  d |= (uint64_t)(128 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// smem chunk -> TMEM: 32 lanes x 128 bits, replicated to the 4 lane quarters (4 columns)
__device__ __forceinline__ void utccp_sf(uint32_t taddr, uint64_t sd) {
  asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(taddr), "l"(sd) : "memory");
}
// plain bulk copy global -> shared, completing on an mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}
// cta_group::2 variants (MX pairs): the leader issues for both CTAs; each CTA's scale chunk goes
// from its own smem to its own TMEM.
__device__ __forceinline__ void mma_mx_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc,
                                            uint32_t tsfa, uint32_t tsfb) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::mxf8f6f4.block_scale [%0], %1, %2, %3, [%5], [%6], p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(tsfa), "r"(tsfb)
      : "memory");
}
__device__ __forceinline__ void utccp_sf_pair(uint32_t taddr, uint64_t sd) {
  asm volatile("tcgen05.cp.cta_group::2.32x128b.warpx4 [%0], %1;" ::"r"(taddr), "l"(sd) : "memory");
}
// 0: one N=256 block-scaled MMA (B scales of rows 128..255 four TMEM columns after rows 0..127);
// 1: two N=128 MMAs (each with its own B scale chunk).  MEMFINE_MX_SPLITN selects 1 at launch.
constexpr int kMxSf = 12;   // TMEM columns of scale factors: A 4, B 2 x 4

// ------------------------------------------------------------------ per-kind configuration
template <int KIND>
struct Cfg;
// A7/B2: X[R,h] x W_gate/W_up[g,h]^T: the W_gate and W_up tiles land back to back in smem and
// form one 256-row B operand, so a single N=256 MMA produces G (cols 0..127) and U (128..255).
template <> struct Cfg<GK_GATEUP> { static constexpr int BN = 128, NACC = 2, A_MN = 0, B_MN = 0; };
// A8: a[R,g] x W_down[h,g]^T.
template <> struct Cfg<GK_DOWN> { static constexpr int BN = 256, NACC = 1, A_MN = 0, B_MN = 0; };
// B3: dY[R,h] x W_down[h,g]  (B(n,k) = W_down[k][n], MN-major).
template <> struct Cfg<GK_DACT> { static constexpr int BN = 256, NACC = 1, A_MN = 0, B_MN = 1; };
// B4: dGU[R,2g] x [W_gate; W_up][2g,h]  (MN-major B, K split at g).
template <> struct Cfg<GK_DX> { static constexpr int BN = 256, NACC = 1, A_MN = 0, B_MN = 1; };
// B5: dW[e] += rows^T rows  (A(m,k) = rows[s0+k][m], B(n,k) = rows[s0+k][n]; both MN-major).
template <> struct Cfg<GK_WGRAD_DOWN> { static constexpr int BN = 256, NACC = 1, A_MN = 1, B_MN = 1; };
template <> struct Cfg<GK_WGRAD_GU> { static constexpr int BN = 256, NACC = 1, A_MN = 1, B_MN = 1; };

// MX kernels (gate/up, down, dX): the same tiles, both operands K-major.
template <int KIND, bool MX>
struct CfgX {
  static constexpr int BN = Cfg<KIND>::BN;
  static constexpr int NACC = Cfg<KIND>::NACC;
  static constexpr int A_MN = MX ? 0 : Cfg<KIND>::A_MN;
  static constexpr int B_MN = MX ? 0 : Cfg<KIND>::B_MN;
};

// Epilogue staging per epilogue warp and chunk of 32 columns: output slots x slot bytes,
// double-buffered across chunks.
template <int KIND, bool MX = false>
struct Epi {
  static constexpr int SLOTS = KIND == GK_DACT ? 3 : (KIND == GK_GATEUP ? 2 : 1);
  // dA works in 16-column sub-chunks (32 rows x 32 B, SWIZZLE_32B) so its staging is 24 KB
  static constexpr int SLOT_BYTES = KIND >= GK_WGRAD_DOWN ? 4096 : (KIND == GK_DACT ? 1024 : 2048);
  static constexpr int CHUNK_BYTES = SLOTS * SLOT_BYTES;
  // dA and dW: single-buffered staging so the mainloop keeps one more stage of operands in flight
  // (measured: dA 72% -> 82% tensor-active going from 4 to 5 stages); the others double-buffer.
  static constexpr int BUFS = (KIND == GK_DACT || KIND >= GK_WGRAD_DOWN) ? 1 : 2;
  static constexpr int WARP_BYTES = BUFS * CHUNK_BYTES;
  // MX N=256 kinds store straight from registers (early accumulator release): no staging, so the
  // mainloop gets the smem for more stages.
  // (MX weight gradients keep the fp32 staging: dW goes out by TMA store / reduce-add)
  static constexpr int TOTAL = (MX && KIND < GK_WGRAD_DOWN) ? 0 : EPI_WARPS * WARP_BYTES;
};

struct Params {
  int El, h, g;
  int M, N, K;       // M: rows of dW for WGRAD kinds; N: output columns; K: reduction (M-tiled kinds)
  int num_mt_w;      // WGRAD: M tiles (of 128 or 256 rows) per expert
  int64_t rows_cap;
  const int* seg;
  const int* pseg;
  const int* info;
  __nv_bfloat16* GU;
  __nv_bfloat16* A;
  __nv_bfloat16* O;
  const float* w_row;
  float* dw_row;
  float* dW0;        // WGRAD_DOWN: dW_down; WGRAD_GU: dW_gate
  float* dW1;        // WGRAD_GU: dW_up
  int store_a, store_gu;
  int beta;          // WGRAD: 1 = dW += acc (accumulate), 0 = dW = acc (first chunk, overwrite)
  const uint64_t* row_addr;  // DOWN / DX fused EP combine: per-row peer destination (0 = padding)
  int group_m;       // M tiles per raster group (host-sized so a wave's operands stay in L2)
  int* wave_ctr;     // wave pacing: steps started by all units, zeroed per launch (null = off)
  int pace_kb;       // k-blocks per pacing step of M-tiled kinds (<= 0: one step per tile)
  int pace_slack;    // steps a unit may run ahead of the slowest unit (>= 1)
  // MXFP8 (MX kernels): scale chunks of A and B, GATEUP forward's quantised a
  const uint8_t* mx_a_sf;
  const uint8_t* mx_b0_sf;
  const uint8_t* mx_b1_sf;
  uint8_t* mx_aq;
  uint8_t* mx_aq_sf;
  uint8_t* mx_gq;      // dA (BF16 GEMM) in the MX variant: dG||dU also quantised for the dX GEMM
  uint8_t* mx_gq_sf;
  int mx_split_n;
  int out_f32;         // DOWN: fp32 output (the router's logits), 16-column TMA stores
};

struct Tile {
  int e;      // local expert
  int m0;     // first row of the (pair) tile: padded row (M-tiled kinds) or dW row (WGRAD)
  int m_end;  // rows >= m_end are not stored (expert segment end / M)
  int n0, k0, nkb;
  int halves = 1;   // QD (quad) tiles: 2 = two 256-row pair halves sharing the B tile, 1 = the last odd pair
};

// 2-CTA helpers (cta_group::2): the pair's leader is the even CTA of the cluster.
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // clears the CTA-in-pair bit of a shared::cluster address
__device__ __forceinline__ uint32_t cta_rank_in_cluster() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_2d_pair(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(su32(dst)),
      "l"(m), "r"(su32(bar) & kPeerMask), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_3d_pair(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4, %5}], [%2];" ::"r"(su32(dst)),
      "l"(m), "r"(su32(bar) & kPeerMask), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void mma_bf16_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// commit -> arrive on the barrier at the same smem offset in both CTAs of the pair
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          su32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
// arrive on the leader CTA's copy of a barrier (own copy when this is the leader)
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(su32(b) & kPeerMask) : "memory");
}

template <int KIND, bool PAIR, bool MX = false, bool QD = false>
__device__ __forceinline__ int num_tiles(const Params& p, const int* qseg = nullptr) {
  constexpr int BN = CfgX<KIND, MX>::BN;
  int nt = (p.N + BN - 1) / BN;
  if (KIND >= GK_WGRAD_DOWN) return p.El * p.num_mt_w * nt;
  if (p.info[kInfoSkip]) return 0;
  if (QD) return qseg[p.El] * nt;
  return (PAIR ? p.info[kInfoPairs] : p.info[kInfoRowsPad] / BM) * nt;
}

template <int KIND, bool PAIR, bool MX = false, bool QD = false>
__device__ __forceinline__ Tile tile_of(const Params& p, int t, const int* qseg = nullptr) {
  constexpr int BN = CfgX<KIND, MX>::BN;
  constexpr int TM = PAIR ? 2 * BM : BM;  // rows per (pair) tile
  int nt = (p.N + BN - 1) / BN;
  Tile T;
  if (QD) {
    // quad tiles: two consecutive 256-row pairs of one expert (qseg: shared-memory prefix of
    // ceil(pairs_e / 2)); an expert's odd last pair makes a one-half tile
    const int nq = qseg[p.El];
    const int gsz = p.group_m * nt;
    const int gi = t / gsz, first = gi * p.group_m;
    const int gm = min(nq - first, p.group_m);
    const int r = t % gsz;
    const int mq = first + r % gm;
    T.n0 = (r / gm) * BN;
    int lo = 0, hi = p.El;   // qseg[lo] <= mq < qseg[hi]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (qseg[mid] <= mq) lo = mid; else hi = mid;
    }
    T.e = lo;
    const int ps0 = __ldg(p.pseg + lo), pair = ps0 + (mq - qseg[lo]) * 2;
    T.halves = min(2, __ldg(p.pseg + lo + 1) - pair);
    T.m0 = __ldg(p.seg + lo) + (pair - ps0) * TM;
    T.m_end = __ldg(p.seg + lo + 1);
    T.k0 = 0;
    T.nkb = p.K / BK;
    return T;
  }
  if (KIND >= GK_WGRAD_DOWN) {
    int per = p.num_mt_w * nt;
    T.e = t / per;
    int r0 = t % per;
    int gsz = p.group_m * nt;
    int gi = r0 / gsz, first = gi * p.group_m;
    int gm = min(p.num_mt_w - first, p.group_m);
    int r = r0 % gsz;
    T.m0 = (first + r % gm) * TM;
    T.m_end = p.M;
    T.n0 = (r / gm) * BN;
    int s0 = __ldg(p.seg + T.e), s1 = __ldg(p.seg + T.e + 1);
    T.k0 = s0;
    T.nkb = (s1 - s0) / (MX ? 128 : BK);   // segments are 128-row padded
    return T;
  }
  int num_mt = PAIR ? p.info[kInfoPairs] : p.info[kInfoRowsPad] / BM;
  int gsz = p.group_m * nt;
  int gi = t / gsz, first = gi * p.group_m;
  int gm = min(num_mt - first, p.group_m);
  int r = t % gsz;
  int mt = first + r % gm;
  T.n0 = (r / gm) * BN;
  if (PAIR) {
    T.e = expert_of_pair(p.pseg, p.El, mt);
    T.m0 = __ldg(p.seg + T.e) + (mt - __ldg(p.pseg + T.e)) * TM;
    T.m_end = __ldg(p.seg + T.e + 1);
  } else {
    T.m0 = mt * BM;
    T.e = expert_of_row(p.seg, p.El, T.m0);
    T.m_end = T.m0 + BM;
  }
  T.k0 = 0;
  T.nkb = p.K / (MX ? 128 : BK);
  return T;
}

// MX stage: A 128 x 128 B + B (N rows) x 128 B (E4M3, 128 K per stage) + 1.5 KB scale chunks, 1 KB aligned
template <int KIND, bool PAIR, bool MX = false, bool QD = false>
__host__ __device__ constexpr int stage_bytes() {
  return MX ? (A_BYTES + CfgX<KIND, MX>::NACC * CfgX<KIND, MX>::BN * 128 / (PAIR ? 2 : 1) + 1536 + 1023) / 1024 * 1024
            : A_BYTES * (QD ? 2 : 1) +
                  (PAIR ? Cfg<KIND>::NACC * Cfg<KIND>::BN / 2 : Cfg<KIND>::NACC * Cfg<KIND>::BN) * BK * 2;
}
// QD: 1 KB more for the quad prefix (E_l <= 255)
constexpr int kQsegBytes = 1024;
// as many 1024-aligned stages as fit next to the epilogue staging (227 KB per CTA)
template <int KIND, bool PAIR, bool MX = false, bool QD = false>
__host__ __device__ constexpr int nstage() {
  return (232448 - 1024 - 512 - (QD ? kQsegBytes : 0) - Epi<KIND, MX>::TOTAL) / stage_bytes<KIND, PAIR, MX, QD>() > 6
             ? 6
             : (232448 - 1024 - 512 - (QD ? kQsegBytes : 0) - Epi<KIND, MX>::TOTAL) / stage_bytes<KIND, PAIR, MX, QD>();
}
template <int KIND, bool PAIR, bool MX = false, bool QD = false>
__host__ __device__ constexpr int smem_bytes() {
  return nstage<KIND, PAIR, MX, QD>() * stage_bytes<KIND, PAIR, MX, QD>() + Epi<KIND, MX>::TOTAL + 1024 + 512 +
         (QD ? kQsegBytes : 0);
}

// ------------------------------------------------------------------ the kernel
// PAIR = false: one CTA per 128-row tile, tcgen05.mma.cta_group::1 (M=128).
// PAIR = true : a 2-CTA cluster per 256-row tile, tcgen05.mma.cta_group::2 (M=256) issued by the
//               even CTA; each CTA stages 128 rows of A and half of B's columns, each CTA's TMEM
//               holds its 128 rows x N accumulator.  Per-CTA operand traffic drops by a third.
// MX = true: MXFP8 operands (kind::mxf8f6f4.block_scale, cta_group::1, K-major A and B, 128 K
//            per stage, N=256 tiles with one accumulator stage + 12 scale-factor columns in TMEM,
//            drained early into registers by the epilogue).  MX && PAIR: cta_group::2 (M = 256) like the BF16 pairs - each CTA
//            stages its 128 A rows and half of B, so the tensor core's smem reads per CTA halve;
//            scale chunks come by TMA (uint32 rows of 512 B): each CTA holds its own A scales and
//            the full B tile's scales.
// QD = true (BF16 DOWN / DX, pairs): 512 x 256 tiles per CTA pair - two M = 256 halves sharing each staged B
//            tile, so every B byte feeds twice the rows (a quarter fewer operand fills per FLOP); each CTA
//            stages 2 x 128 A rows, the two halves' accumulators fill all 512 TMEM columns (one stage:
//            the epilogue of a tile is not overlapped, which the long K of these two GEMMs hides).
template <int KIND, bool PAIR, bool MX = false, bool QD = false>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_kernel(const __grid_constant__ Params p, const __grid_constant__ CUtensorMap tmA,
                const __grid_constant__ CUtensorMap tmB0, const __grid_constant__ CUtensorMap tmB1,
                const __grid_constant__ CUtensorMap tmO0, const __grid_constant__ CUtensorMap tmO1,
                const __grid_constant__ CUtensorMap tmSA, const __grid_constant__ CUtensorMap tmSB0,
                const __grid_constant__ CUtensorMap tmSB1) {
  using CF = CfgX<KIND, MX>;
  constexpr int BN = CF::BN, NACC = CF::NACC;
  constexpr int MMA_N = NACC * BN;                      // GATEUP: G||U in one MMA (N = 256)
  static_assert(MMA_N <= 256, "MMA N");
  constexpr bool G2 = PAIR;                             // cta_group::2 pair
  constexpr int B_ROWS = G2 ? MMA_N / 2 : MMA_N;        // B rows (N) staged per CTA
  constexpr int B_BYTES = B_ROWS * BK * 2;               // (MX: B_ROWS x 128 E4M3 = the same bytes)
  constexpr int STAGE_BYTES = stage_bytes<KIND, PAIR, MX, QD>();
  constexpr int NSTAGE = nstage<KIND, PAIR, MX, QD>();
  constexpr int A_ST = QD ? 2 * A_BYTES : A_BYTES;       // A bytes per stage (QD: both halves' rows)
  static_assert(!QD || (PAIR && !MX && MMA_N == 256 && (KIND == GK_DOWN || KIND == GK_DX)), "QD tiles");
  constexpr int ACC_COLS = MMA_N;                       // per accumulator stage (QD: per half)
  constexpr int ACC_ST = ((MX && MMA_N == 256) || QD) ? 1 : 2;  // accumulator stages (MX N=256: scales take TMEM)
  constexpr uint32_t TMEM_COLS = MX ? 512 : 2 * ACC_COLS;
  constexpr uint32_t SF_COL = ACC_ST * ACC_COLS;        // MX: A scales at +0..3, B at +4..11
  static_assert(TMEM_COLS <= 512 && (!MX || ACC_ST * ACC_COLS + kMxSf <= 512), "TMEM");
  static_assert(!MX || KIND != GK_DACT, "MX: gate/up, down, dX, weight gradients (R28c)");
  constexpr uint32_t IDESC = idesc_bf16(PAIR ? 2 * BM : BM, MMA_N, CF::A_MN, CF::B_MN);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* epi_smem = smem + NSTAGE * STAGE_BYTES;      // 1024-aligned (STAGE_BYTES is)
  uint64_t* full = (uint64_t*)(epi_smem + Epi<KIND, MX>::TOTAL);
  uint64_t* empty = full + NSTAGE;
  uint64_t* tfull = empty + NSTAGE;
  uint64_t* tempty = tfull + 2;
  uint64_t* ebar = tempty + 2;                          // [EPI_WARPS][2] epilogue TMA-load barriers (dA)
  uint32_t* tmem_slot = (uint32_t*)(ebar + 2 * EPI_WARPS);
  int* qseg = (int*)(epi_smem + Epi<KIND, MX>::TOTAL + 512);   // QD: [E_l + 1] quad prefix (after the barriers)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = PAIR ? cta_rank_in_cluster() : 0;
  const bool leader = rank == 0;
  const int cid = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;     // tile-loop index
  const int ncid = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB0);
    if (KIND == GK_GATEUP || KIND == GK_DX) prefetch_tmap(&tmB1);
    prefetch_tmap(&tmO0);
    if (KIND == GK_GATEUP || KIND == GK_DACT || KIND == GK_WGRAD_GU) prefetch_tmap(&tmO1);
    if (MX) {
      prefetch_tmap(&tmSA);
      prefetch_tmap(&tmSB0);
      if (KIND == GK_GATEUP || KIND == GK_DX) prefetch_tmap(&tmSB1);
    }
    for (int s = 0; s < NSTAGE; s++) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
    for (int a = 0; a < 2; a++) { mbar_init(tfull + a, 1); mbar_init(tempty + a, (G2 ? 2 : 1) * EPI_WARPS); }
    for (int i = 0; i < 2 * EPI_WARPS; i++) mbar_init(ebar + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    if (G2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                   "r"(TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                   "r"(TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  fence_before();
  if (PAIR) cluster_sync(); else __syncthreads();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // everything above (barrier init, TMEM alloc, descriptor prefetch) overlaps the predecessor's tail
  pdl_wait();
  pdl_trigger();
  if constexpr (QD) {
    // the quad prefix qseg[e] = sum over e' < e of ceil(pairs_e' / 2), from the pair prefix the dispatch scan
    // wrote (read after griddepcontrol.wait); warp 2, 32 experts per step
    if (warp == 2) {
      int carry = 0;
      if (lane == 0) qseg[0] = 0;
      for (int base = 0; base < p.El; base += 32) {
        const int e = base + lane;
        int v = e < p.El ? (__ldg(p.pseg + e + 1) - __ldg(p.pseg + e) + 1) >> 1 : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int u = __shfl_up_sync(0xffffffffu, v, o);
          if (lane >= o) v += u;
        }
        if (e < p.El) qseg[e + 1] = carry + v;
        carry += __shfl_sync(0xffffffffu, v, 31);
      }
    }
    __syncthreads();
  }
  const int ntiles = num_tiles<KIND, PAIR, MX, QD>(p, qseg);
  (void)SF_COL;

  if (warp == 0) {
    // ================================================================ TMA producer (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int step = 0;  // pacing steps this unit has started
      int seen = 0;  // pacing counter as loaded half a step ago
      // Wave pacing: a unit starts its pacing step s only once every unit has started step s - 1, so
      // the units of one wave (which share A strips along n and B strips along m) stay within a step
      // of each other and their operand loads meet in L2 instead of each missing to DRAM.  A step is
      // a tile, or PACE_KB k-blocks of a long-K tile (every tile of an M-tiled launch has the same K,
      // so the steps line up across units; weight-gradient tiles pace per tile).  The counter is
      // loaded half a step ahead, so a unit that is not ahead never waits on the load.  Spin bounded
      // (~1 ms): pacing is a hint, a non-resident unit cannot deadlock the others.
      const int PACE_KB = (KIND >= GK_WGRAD_DOWN || p.pace_kb <= 0) ? (1 << 30) : p.pace_kb;
      auto pace = [&]() {
        const int target = ncid * (step + 1 - p.pace_slack);   // every unit started step - slack
        if (step >= p.pace_slack && seen < target) {
          for (int spin = 0; spin < 1000; spin++) {
            int v;
            asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p.wave_ctr) : "memory");
            if (v >= target) break;
            __nanosleep(64);
          }
        }
        atomicAdd(p.wave_ctr, 1);
        step++;
      };
      for (int t = cid; t < ntiles; t += ncid) {
        Tile T = tile_of<KIND, PAIR, MX, QD>(p, t, qseg);
        const int am0 = T.m0 + (int)rank * BM;              // this CTA's A rows
        if (KIND >= GK_WGRAD_DOWN && p.wave_ctr && leader) {
          // weight gradients: one step per tile, taken even by tiles without rows (nkb = 0)
          pace();
          if (T.nkb == 0)
            asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(seen) : "l"(p.wave_ctr) : "memory");
        }
        for (int kb = 0; kb < T.nkb; kb++) {
          if (p.wave_ctr && leader) {
            const int ks = kb % PACE_KB, slen = min(PACE_KB, T.nkb - (kb - ks));
            if (ks == 0 && KIND < GK_WGRAD_DOWN) pace();
            if (ks == (slen >> 1))
              asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(seen) : "l"(p.wave_ctr) : "memory");
          }
          mbar_wait(empty + stage, phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_ST;
          if constexpr (MX) {
            // E4M3 A [128 rows x 128 K], this CTA's B rows (all, or its half in a pair) and the scale
            // chunks: own A rows' chunk, the whole B tile's chunks (TMA zero-fills chunks and rows
            // past the end - ragged N tiles, a pair's second m-tile past the buffer)
            const int kc = (KIND >= GK_WGRAD_DOWN ? T.k0 : 0) + kb * 128;
            uint8_t* ssf = sb + B_BYTES;
            // K chunks per 128 operand rows: the weight-gradient operands are the chunk's columnwise
            // codes [M or N rows][rows_cap] (K = the copies, reading R28c)
            const int KB = KIND >= GK_WGRAD_DOWN ? (int)(p.rows_cap >> 7) : p.K >> 7;
            constexpr int SFB_CH = MMA_N / 128;
            if (leader) mbar_expect_tx(full + stage, (PAIR ? 2 : 1) * (A_BYTES + B_BYTES + 512 + 512 * SFB_CH));
            auto L2 = [&](void* dst, const CUtensorMap* m, int c0, int c1) {
              if (PAIR) tma_2d_pair(dst, m, full + stage, c0, c1); else tma_2d(dst, m, full + stage, c0, c1);
            };
            auto L3 = [&](void* dst, const CUtensorMap* m, int c0, int c1, int c2) {
              if (PAIR) tma_3d_pair(dst, m, full + stage, c0, c1, c2); else tma_3d(dst, m, full + stage, c0, c1, c2);
            };
            L2(sa, &tmA, kc, am0);
            L2(ssf, &tmSA, 0, (am0 >> 7) * KB + (kc >> 7));
            if (KIND >= GK_WGRAD_DOWN) {
              // B(n, k) = codes_t[n][k]: this CTA's rows of the N tile, the whole tile's scale chunks
              L2(sb, &tmB0, kc, T.n0 + (PAIR ? (int)rank * B_ROWS : 0));
              const int nch = p.N >> 7;
#pragma unroll
              for (int i = 0; i < SFB_CH; i++) {
                const int nc = (T.n0 >> 7) + i;
                L2(ssf + 512 + 512 * i, &tmSB0, 0, (nc < nch ? nc : (T.n0 >> 7)) * KB + (kc >> 7));
              }
            } else if (KIND == GK_GATEUP) {
              if (PAIR) {
                L3(sb, rank ? &tmB1 : &tmB0, kc, T.n0, T.e);       // CTA0: W_gate rows, CTA1: W_up rows
              } else {
                L3(sb, &tmB0, kc, T.n0, T.e);
                L3(sb + B_BYTES / 2, &tmB1, kc, T.n0, T.e);
              }
              const int ci = (T.e * (p.N >> 7) + (T.n0 >> 7)) * KB + kb;
              L2(ssf + 512, &tmSB0, 0, ci);
              L2(ssf + 1024, &tmSB1, 0, ci);
            } else {
              // DOWN: W_down rows; DACT: W_down^T rows; DX: W_gate^T (k < g) / W_up^T rows
              const bool lo = KIND != GK_DX || kc < p.g;
              const int kk = lo ? kc : kc - p.g;
              const int KW = KIND == GK_DX ? (p.g >> 7) : KB;       // K chunks of the weight
              L3(sb, lo ? &tmB0 : &tmB1, kk, T.n0 + (PAIR ? (int)rank * B_ROWS : 0), T.e);
              const int ci = (T.e * (p.N >> 7) + (T.n0 >> 7)) * KW + (kk >> 7);
              const int nvalid = (p.N - T.n0 + 127) >> 7;           // B chunks inside this expert
#pragma unroll
              for (int i = 0; i < SFB_CH; i++)
                L2(ssf + 512 + 512 * i, lo ? &tmSB0 : &tmSB1, 0, i < nvalid ? ci + i * KW : ci);
            }
            if (++stage == NSTAGE) { stage = 0; phase ^= 1; }
            continue;
          }
          if (leader)
            mbar_expect_tx(full + stage, (PAIR ? 2 : 1) * (QD ? A_BYTES * T.halves + (STAGE_BYTES - A_ST) : STAGE_BYTES));
          int kc = T.k0 + kb * BK;
          auto LA = [&](void* dst, const CUtensorMap* m, int c0, int c1) {
            if (PAIR) tma_2d_pair(dst, m, full + stage, c0, c1); else tma_2d(dst, m, full + stage, c0, c1);
          };
          auto L2 = LA;
          auto L3 = [&](void* dst, const CUtensorMap* m, int c0, int c1, int c2) {
            if (PAIR) tma_3d_pair(dst, m, full + stage, c0, c1, c2); else tma_3d(dst, m, full + stage, c0, c1, c2);
          };
          if (CF::A_MN) {
            // A(m,k) = rows[kc + k][am0 + m]: two 64-wide MN atoms of 64 K rows
            LA(sa, &tmA, am0, kc);
            LA(sa + 8192, &tmA, am0 + 64, kc);
          } else {
            LA(sa, &tmA, kc, am0);
            if (QD && T.halves == 2) LA(sa + A_BYTES, &tmA, kc, am0 + 2 * BM);   // the second half's rows
          }
          // B: this CTA's share of the N columns
          const int bn0 = T.n0 + (PAIR ? (int)rank * B_ROWS : 0);
          if (KIND == GK_GATEUP) {
            if (PAIR) {
              L3(sb, rank ? &tmB1 : &tmB0, kc, T.n0, T.e);      // CTA0: W_gate rows, CTA1: W_up rows
            } else {
              L3(sb, &tmB0, kc, T.n0, T.e);
              L3(sb + B_BYTES / 2, &tmB1, kc, T.n0, T.e);
            }
          } else if (KIND == GK_DOWN) {
            L3(sb, &tmB0, kc, bn0, T.e);
          } else if (KIND == GK_DACT) {
#pragma unroll
            for (int i = 0; i < B_ROWS / 64; i++) L3(sb + i * 8192, &tmB0, bn0 + 64 * i, kc, T.e);
          } else if (KIND == GK_DX) {
            const CUtensorMap* mb = kc < p.g ? &tmB0 : &tmB1;
            int kk = kc < p.g ? kc : kc - p.g;
#pragma unroll
            for (int i = 0; i < B_ROWS / 64; i++) L3(sb + i * 8192, mb, bn0 + 64 * i, kk, T.e);
          } else {
#pragma unroll
            for (int i = 0; i < B_ROWS / 64; i++) L2(sb + i * 8192, &tmB0, bn0 + 64 * i, kc);
          }
          if (++stage == NSTAGE) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ================================================================ MMA issuer (leader CTA only)
    if (lane == 0 && leader) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = cid; t < ntiles; t += ncid) {
        Tile T = tile_of<KIND, PAIR, MX, QD>(p, t, qseg);
        if (T.nkb == 0) continue;
        int as = it % ACC_ST;
        uint32_t aph = (it / ACC_ST) & 1;
        mbar_wait(tempty + as, aph ^ 1);
        fence_after();
        uint32_t dbase = tmem_base + as * ACC_COLS;
        for (int kb = 0; kb < T.nkb; kb++) {
          mbar_wait(full + stage, phase);
          fence_after();
          uint32_t sa = su32(smem + stage * STAGE_BYTES);
          uint32_t sb = sa + A_ST;
          if constexpr (MX) {
            // scales smem -> TMEM (executes in order with the MMAs: the previous stage's MMAs
            // have read the columns before these copies land)
            const uint32_t ssf = sb + B_BYTES;
            const uint32_t tsf = tmem_base + SF_COL;
            constexpr int SFB_CH = MMA_N / 128;
#pragma unroll
            for (int i = 0; i <= SFB_CH; i++) {
              if (PAIR) utccp_sf_pair(tsf + 4 * i, sdesc_sf(ssf + 512 * i));
              else utccp_sf(tsf + 4 * i, sdesc_sf(ssf + 512 * i));
            }
#pragma unroll
            for (int k = 0; k < 4; k++) {
              const uint64_t ad = sdesc(sa + k * 32, 16, 1024);
              const uint32_t ids = ((uint32_t)k << 29) | ((uint32_t)k << 4);
              if (PAIR) {
                const uint64_t bd = sdesc(sb + k * 32, 16, 1024);
                mma_mx_pair(dbase, ad, bd, idesc_mx(2 * BM, MMA_N) | ids, (kb | k) != 0, tsf, tsf + 4);
              } else if (MMA_N == 128 || !(p.mx_split_n & 1)) {
                const uint64_t bd = sdesc(sb + k * 32, 16, 1024);
                mma_mx(dbase, ad, bd, idesc_mx(BM, MMA_N) | ids, (kb | k) != 0, tsf, tsf + 4);
              } else {
#pragma unroll
                for (int hn = 0; hn < 2; hn++) {
                  const uint64_t bd = sdesc(sb + hn * (B_BYTES / 2) + k * 32, 16, 1024);
                  mma_mx(dbase + hn * (MMA_N / 2), ad, bd, idesc_mx(BM, MMA_N >= 256 ? 128 : MMA_N) | ids,
                         (kb | k) != 0, tsf, tsf + 4 + 4 * hn);
                }
              }
            }
            if (PAIR) mma_commit_pair(empty + stage); else mma_commit(empty + stage);
            if (++stage == NSTAGE) { stage = 0; phase ^= 1; }
            continue;
          }
#pragma unroll
          for (int k = 0; k < BK / 16; k++) {
            uint64_t ad = CF::A_MN ? sdesc(sa + k * 2048, 8192, 1024) : sdesc(sa + k * 32, 16, 1024);
            uint64_t bd = CF::B_MN ? sdesc(sb + k * 2048, 8192, 1024) : sdesc(sb + k * 32, 16, 1024);
            if (PAIR) mma_bf16_pair(dbase, ad, bd, IDESC, (kb | k) != 0);
            else mma_bf16(dbase, ad, bd, IDESC, (kb | k) != 0);
          }
          if (QD && T.halves == 2) {
            // the second half: its own A rows, the same staged B tile, the other 256 TMEM columns
#pragma unroll
            for (int k = 0; k < BK / 16; k++)
              mma_bf16_pair(dbase + ACC_COLS, sdesc(sa + A_BYTES + k * 32, 16, 1024),
                            CF::B_MN ? sdesc(sb + k * 2048, 8192, 1024) : sdesc(sb + k * 32, 16, 1024), IDESC,
                            (kb | k) != 0);
          }
          if (PAIR) mma_commit_pair(empty + stage); else mma_commit(empty + stage);
          if (++stage == NSTAGE) { stage = 0; phase ^= 1; }
        }
        if (G2) mma_commit_pair(tfull + as); else mma_commit(tfull + as);
        it++;
      }
    }
  } else {
    // ================================================================ epilogue (warps 2..9, both CTAs)
    // TMEM -> registers (tcgen05.ld 32x32b: lane = row) -> fused MoE math -> swizzled smem
    // staging -> TMA store (or TMA reduce-add for accumulated dW), one bulk group per chunk,
    // double-buffered per warp.
    const int q = warp & 3;               // TMEM lane quarter this warp may access
    const int half = (warp - 2) >> 2;     // which half of the tile's columns
    const int ew = warp - 2;              // epilogue warp index 0..7
    const int rloc = q * 32 + lane;       // row within this CTA's 128 rows
    constexpr int CPW = BN / 2;           // columns per epilogue warp
    using EP = Epi<KIND, MX>;
    uint8_t* wbuf = epi_smem + ew * EP::WARP_BYTES;
    int sbuf = 0;
    int it = 0;
    uint32_t ephase[2] = {0, 0};   // dA: phase of this warp's two G||U load barriers
    // dA: TMA-load the G||U sub-tile (32 rows x 32 cols each) of chunk column n into buffer b
    auto dact_load = [&](int b, int n, int row0) {
      if (lane == 0) {
        bulk_wait_read<0>();   // the buffer's previous stores have read it
        uint8_t* buf = wbuf + b * EP::CHUNK_BYTES;
        mbar_expect_tx(ebar + 2 * ew + b, 2 * EP::SLOT_BYTES);
        tma_2d(buf, &tmO0, ebar + 2 * ew + b, n, row0);
        tma_2d(buf + EP::SLOT_BYTES, &tmO0, ebar + 2 * ew + b, p.g + n, row0);
      }
      __syncwarp();
    };
    auto next_buf = [&]() -> uint8_t* {
      // the group that last used this buffer must have finished reading it
      if (lane == 0) {
        if (EP::BUFS == 2) bulk_wait_read<1>(); else bulk_wait_read<0>();
      }
      __syncwarp();
      uint8_t* b = wbuf + sbuf * EP::CHUNK_BYTES;
      if (EP::BUFS == 2) sbuf ^= 1;
      return b;
    };
    for (int t = cid; t < ntiles; t += ncid) {
      Tile T = tile_of<KIND, PAIR, MX, QD>(p, t, qseg);
      int row0 = T.m0 + (int)rank * BM + q * 32;           // first row of this warp's 32 rows
      int rowi = row0 + lane;
      bool rows_ok = row0 < T.m_end;                       // warp-uniform (halves are 128-row aligned)
      if (T.nkb == 0) {
        if (KIND >= GK_WGRAD_DOWN && !p.beta && rows_ok) {
          // an expert without rows in the first chunk: its dW tile is zero
          float z[32];
#pragma unroll
          for (int i = 0; i < 32; i++) z[i] = 0.f;
          for (int c = half * CPW; c < (half + 1) * CPW; c += 32) {
            uint8_t* buf = next_buf();
            stage_f32_row(buf, lane, z);
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
              const int n = T.n0 + c;
              if (KIND == GK_WGRAD_DOWN) tma_store_3d(&tmO0, buf, n, row0, T.e, false);
              else if (row0 < p.g) tma_store_3d(&tmO0, buf, n, row0, T.e, false);
              else tma_store_3d(&tmO1, buf, n, row0 - p.g, T.e, false);
              bulk_commit();
            }
          }
        }
        continue;
      }
      int as = it % ACC_ST;
      uint32_t aph = (it / ACC_ST) & 1;
      int64_t row = rowi;
      if constexpr (MX && ACC_ST == 1) {
        // One accumulator stage (the scales take the rest of TMEM): drain this warp's slice of
        // the tile into registers, free TMEM for the next tile's MMAs, then run the epilogue from
        // registers - the mainloop of tile i+1 overlaps the math and stores of tile i.
        constexpr int NCH = CPW / 32;
        uint32_t acc[NCH][32];
        uint32_t acc2[KIND == GK_GATEUP ? NCH : 1][32];
        mbar_wait(tfull + as, aph);
        fence_after();
        const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16);
#pragma unroll
        for (int i = 0; i < NCH; i++) {
          tmem_ld32_nw(tb + half * CPW + 32 * i, acc[i]);
          if constexpr (KIND == GK_GATEUP) tmem_ld32_nw(tb + BN + half * CPW + 32 * i, acc2[i]);
        }
        tmem_wait_ld();
        fence_before();
        __syncwarp();
        if (lane == 0) {
          if (PAIR) mbar_arrive_leader(tempty + as); else mbar_arrive(tempty + as);
        }
#pragma unroll
        for (int i = 0; i < NCH; i++) {
          const int n = T.n0 + half * CPW + 32 * i;
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; j++) v[j] = __uint_as_float(acc[i][j]);
          if constexpr (KIND >= GK_WGRAD_DOWN) {
            // MX weight gradients (R28c): fp32 dW tile by TMA store (first chunk) / reduce-add
            if (!rows_ok || n >= p.N) continue;
            uint8_t* buf = next_buf();
            stage_f32_row(buf, lane, v);
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
              if (KIND == GK_WGRAD_DOWN) tma_store_3d(&tmO0, buf, n, row0, T.e, p.beta != 0);
              else if (row0 < p.g) tma_store_3d(&tmO0, buf, n, row0, T.e, p.beta != 0);
              else tma_store_3d(&tmO1, buf, n, row0 - p.g, T.e, p.beta != 0);
              bulk_commit();
            }
          } else if constexpr (KIND == GK_GATEUP) {
            if (!rows_ok || n >= p.g) continue;
            if (!p.store_gu) {
              // a = silu(G) U straight to MXFP8: this thread's 32 columns are one block
              float a[32];
              float amax = 0.f;
#pragma unroll
              for (int j = 0; j < 32; j++) {
                a[j] = silu_f(v[j]) * __uint_as_float(acc2[i][j]);
                amax = fmaxf(amax, fabsf(a[j]));
              }
              const int E = mx_exp(amax);
              const float inv = mx_inv_scale(E);
              uint32_t o[8];
#pragma unroll
              for (int j = 0; j < 8; j++)
                o[j] = mx_e4m3x2(a[4 * j] * inv, a[4 * j + 1] * inv) |
                       (mx_e4m3x2(a[4 * j + 2] * inv, a[4 * j + 3] * inv) << 16);
              st256(p.mx_aq + row * p.g + n, o);
              p.mx_aq_sf[mx_sf_off(row, n >> 5, p.g)] = (uint8_t)(E + 127);
            } else {
              // G -> GU[row, n..n+31], U -> GU[row, g + n..]: 64 B each, straight from registers
              float u[32];
#pragma unroll
              for (int j = 0; j < 32; j++) u[j] = __uint_as_float(acc2[i][j]);
              __nv_bfloat16* gu = p.GU + row * (2 * (int64_t)p.g);
              store32_bf16(gu + n, v);
              store32_bf16(gu + p.g + n, u);
            }
          } else {
            if (!rows_ok || n >= p.h) continue;                 // DOWN / DX: N = h
            if (p.row_addr) {
              // fused EP combine (P2P transport): the row goes straight into its source rank's send
              // buffer (peer memory) as the tile is produced
              const uint64_t a = __ldg(p.row_addr + row);
              if (a) store32_bf16(reinterpret_cast<__nv_bfloat16*>(a) + n, v);
            } else {
              store32_bf16(p.O + row * (int64_t)p.h + n, v);
            }
          }
        }
        it++;
        continue;
      }
      float dwp = 0.f;
      float2 dwp2 = make_float2(0.f, 0.f);   // dA: d_w partials of the even / odd columns
      float wrow = 0.f;
      if (KIND == GK_DACT && rows_ok) {
        wrow = p.w_row[row];
        const int n0c = T.n0 + half * CPW;
        if (n0c < p.g) dact_load(0, n0c, row0);   // first chunk's G||U, overlapping the MMA
      }
      mbar_wait(tfull + as, aph);
      fence_after();
      uint32_t tb = tmem_base + as * ACC_COLS + ((uint32_t)(q * 32) << 16);
      for (int hh = 0; hh < (QD ? T.halves : 1); hh++) {
      if (QD && hh) {   // the quad tile's second half: 256 rows further, the other 256 TMEM columns
        row0 += 2 * BM;
        rowi += 2 * BM;
        row += 2 * BM;
        rows_ok = row0 < T.m_end;
        tb += ACC_COLS;
      }
#pragma unroll 1
      for (int c = half * CPW; c < (half + 1) * CPW; c += 32) {
        const int n = T.n0 + c;
        uint32_t r[32];
        tmem_ld32(tb + c, r);
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; i++) v[i] = __uint_as_float(r[i]);
        if (KIND == GK_GATEUP) {
          uint32_t r2[32];
          tmem_ld32(tb + BN + c, r2);
          if (rows_ok && n < p.g) {
            uint8_t* buf = next_buf();
            float u[32];
#pragma unroll
            for (int i = 0; i < 32; i++) u[i] = __uint_as_float(r2[i]);
            if (p.store_gu) {
              stage_bf16_row(buf, lane, v);
              stage_bf16_row(buf + 2048, lane, u);
            } else {
              // a = silu(G) U on packed fp32x2 (FMUL2 / FADD2, ftz ex2 / rcp; see the dA epilogue)
              float a[32];
              const float2 one2 = make_float2(1.f, 1.f);
              const float2 nl2e = make_float2(-1.4426950408889634f, -1.4426950408889634f);
#pragma unroll
              for (int i = 0; i < 32; i += 2) {
                const float2 G2 = make_float2(v[i], v[i + 1]);
                const float2 t2 = __fmul2_rn(G2, nl2e);
                const float2 den = __fadd2_rn(make_float2(ex2_ftz(t2.x), ex2_ftz(t2.y)), one2);
                const float2 a2 = __fmul2_rn(__fmul2_rn(G2, make_float2(rcp_ftz(den.x), rcp_ftz(den.y))),
                                             make_float2(u[i], u[i + 1]));
                a[i] = a2.x;
                a[i + 1] = a2.y;
              }
              stage_bf16_row(buf, lane, a);
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
              if (p.store_gu) {
                tma_store_2d(&tmO0, buf, n, row0);               // G -> GU[:, n]
                tma_store_2d(&tmO0, buf + 2048, p.g + n, row0);  // U -> GU[:, g + n]
              } else {
                tma_store_2d(&tmO1, buf, n, row0);               // a -> A[:, n]
              }
              bulk_commit();
            }
          }
        } else if ((KIND == GK_DOWN || KIND == GK_DX) && p.row_addr) {
          // fused combine exchange: the row goes straight into its source rank's send buffer
          // (peer memory) as the tile is produced
          if (rows_ok && n < p.h) {
            const uint64_t a = __ldg(p.row_addr + row);
            if (a) store32_bf16(reinterpret_cast<__nv_bfloat16*>(a) + n, v);
          }
        } else if (KIND == GK_DOWN || KIND == GK_DX) {
          if (rows_ok && n < p.h) {
            if (KIND == GK_DOWN && p.out_f32) {
              // fp32 output (the router's logits): two 16-column stores per 32-column chunk
#pragma unroll
              for (int h2 = 0; h2 < 2; h2++) {
                uint8_t* buf = next_buf();
                stage_f32_row16(buf, lane, v + 16 * h2);
                fence_async_smem();
                __syncwarp();
                if (lane == 0) {
                  tma_store_2d(&tmO0, buf, n + 16 * h2, row0);
                  bulk_commit();
                }
              }
            } else {
              uint8_t* buf = next_buf();
              stage_bf16_row(buf, lane, v);
              fence_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_store_2d(&tmO0, buf, n, row0);
                bulk_commit();
              }
            }
          }
        } else if (KIND == GK_DACT) {
          if (rows_ok && n < p.g) {
            uint8_t* buf = wbuf;
            uint32_t qg[8], qu[8];   // MX: the first 16 columns' dG / dU (bf16 pairs) of this block
#pragma unroll
            for (int h2 = 0; h2 < 2; h2++) {
              const int n2 = n + 16 * h2;
              if (c != half * CPW || h2) dact_load(0, n2, row0);   // (the first load was issued early)
              mbar_wait(ebar + 2 * ew, ephase[0]);
              ephase[0] ^= 1;
              // this row's 16 G and 16 U (bf16) from the SWIZZLE_32B staging rows (32 B each)
              uint32_t gcur[8], ucur[8];
#pragma unroll
              for (int cc = 0; cc < 2; cc++) {
                const int off = lane * 32 + ((cc ^ ((lane >> 2) & 1)) << 4);
                const uint4 gv = *reinterpret_cast<const uint4*>(buf + off);
                const uint4 uv = *reinterpret_cast<const uint4*>(buf + 1024 + off);
                gcur[4 * cc] = gv.x; gcur[4 * cc + 1] = gv.y; gcur[4 * cc + 2] = gv.z; gcur[4 * cc + 3] = gv.w;
                ucur[4 * cc] = uv.x; ucur[4 * cc + 1] = uv.y; ucur[4 * cc + 2] = uv.z; ucur[4 * cc + 3] = uv.w;
              }
              __syncwarp();
              uint32_t og[8], ou[8], oa[8];
              // the two columns of each bf16 pair in one register pair: packed fp32x2 FMUL2 / FADD2 / FFMA2 (half
              // the FP32 issue of scalar math - the epilogue's instruction stream is what slows the MMA stream
              // beside it, profiles/r02_dact_and_tail_experiments.md §7); per element the same fp32 formulas:
              //   s = 1 / (1 + 2^(-G log2 e)), silu = G s, a = silu U, dA = w u, dU = dA silu,
              //   dG = dA U (s + silu (1 - s)), a_w = w a, d_w += u a
              const float2 w2 = make_float2(wrow, wrow);
              const float2 one2 = make_float2(1.f, 1.f), mone2 = make_float2(-1.f, -1.f);
              const float2 nl2e = make_float2(-1.4426950408889634f, -1.4426950408889634f);
#pragma unroll
              for (int j = 0; j < 8; j++) {
                const uint32_t gw = gcur[j], uw = ucur[j];
                const float2 G2 = make_float2(__uint_as_float(gw << 16), __uint_as_float(gw & 0xFFFF0000u));
                const float2 U2 = make_float2(__uint_as_float(uw << 16), __uint_as_float(uw & 0xFFFF0000u));
                const float2 v2 = make_float2(v[16 * h2 + 2 * j], v[16 * h2 + 2 * j + 1]);
                const float2 t2 = __fmul2_rn(G2, nl2e);
                const float2 den = __fadd2_rn(make_float2(ex2_ftz(t2.x), ex2_ftz(t2.y)), one2);
                const float2 sg = make_float2(rcp_ftz(den.x), rcp_ftz(den.y));
                const float2 silu = __fmul2_rn(G2, sg);
                const float2 a2 = __fmul2_rn(silu, U2);
                dwp2 = __ffma2_rn(v2, a2, dwp2);
                const float2 dA2 = __fmul2_rn(w2, v2);
                const float2 ds = __ffma2_rn(silu, __ffma2_rn(sg, mone2, one2), sg);   // s + silu (1 - s)
                const float2 dG2 = __fmul2_rn(__fmul2_rn(dA2, U2), ds);
                const float2 dU2 = __fmul2_rn(dA2, silu);
                const float2 aw2 = __fmul2_rn(w2, a2);
                og[j] = pack_bf16(dG2.x, dG2.y);
                ou[j] = pack_bf16(dU2.x, dU2.y);
                oa[j] = pack_bf16(aw2.x, aw2.y);
              }
              if (p.mx_gq) {
                // MX variant: dG and dU of this 32-column block -> E4M3 + scale for the dX GEMM
                if (h2 == 0) {
#pragma unroll
                  for (int j = 0; j < 8; j++) { qg[j] = og[j]; qu[j] = ou[j]; }
                } else {
                  const int64_t K2 = 2 * (int64_t)p.g;
                  mx_store_block_bf16(qg, og, p.mx_gq + row * K2 + n, p.mx_gq_sf + mx_sf_off(row, n >> 5, K2));
                  mx_store_block_bf16(qu, ou, p.mx_gq + row * K2 + p.g + n,
                                      p.mx_gq_sf + mx_sf_off(row, (p.g + n) >> 5, K2));
                }
              }
#pragma unroll
              for (int cc = 0; cc < 2; cc++) {
                const int off = lane * 32 + ((cc ^ ((lane >> 2) & 1)) << 4);
                *reinterpret_cast<uint4*>(buf + off) = make_uint4(og[4 * cc], og[4 * cc + 1], og[4 * cc + 2], og[4 * cc + 3]);
                *reinterpret_cast<uint4*>(buf + 1024 + off) =
                    make_uint4(ou[4 * cc], ou[4 * cc + 1], ou[4 * cc + 2], ou[4 * cc + 3]);
                *reinterpret_cast<uint4*>(buf + 2048 + off) =
                    make_uint4(oa[4 * cc], oa[4 * cc + 1], oa[4 * cc + 2], oa[4 * cc + 3]);
              }
              fence_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_store_2d(&tmO0, buf, n2, row0);               // dG over G
                tma_store_2d(&tmO0, buf + 1024, p.g + n2, row0);  // dU over U
                tma_store_2d(&tmO1, buf + 2048, n2, row0);        // a_w
                bulk_commit();
              }
            }
          }
        } else {
          // WGRAD: fp32 dW tile: TMA store (first chunk) or TMA reduce-add (later chunks)
          if (rows_ok && n < p.N) {
            uint8_t* buf = next_buf();
            stage_f32_row(buf, lane, v);
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
              if (KIND == GK_WGRAD_DOWN) tma_store_3d(&tmO0, buf, n, row0, T.e, p.beta != 0);
              else if (row0 < p.g) tma_store_3d(&tmO0, buf, n, row0, T.e, p.beta != 0);
              else tma_store_3d(&tmO1, buf, n, row0 - p.g, T.e, p.beta != 0);
              bulk_commit();
            }
          }
        }
      }
      }   // halves
      if (KIND == GK_DACT && rows_ok) atomicAdd(p.dw_row + row, dwp + dwp2.x + dwp2.y);
      fence_before();
      __syncwarp();
      if (lane == 0) {
        if (G2) mbar_arrive_leader(tempty + as); else mbar_arrive(tempty + as);
      }
      it++;
    }
    if (lane == 0) bulk_wait_all();
    __syncwarp();
  }
  fence_before();
  if (PAIR) cluster_sync(); else __syncthreads();
  fence_after();
  if (warp == 1) {
    if (G2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                   : "memory");
  }
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  });
  return fn;
}

// bf16 tensor map, 128B swizzle; dims/box innermost first; strides in bytes for dims 1..
bool make_map(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
              const uint32_t* box) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t gd[3], gs[2];
  cuuint32_t bx[3], es[3] = {1, 1, 1};
  for (int i = 0; i < rank; i++) { gd[i] = dims[i]; bx[i] = box[i]; }
  for (int i = 0; i < rank - 1; i++) gs[i] = strides_bytes[i];
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), gd, gs, bx, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_map_t(CUtensorMap* m, CUtensorMapDataType dt, int esize, CUtensorMapSwizzle sw, const void* base, int rank,
                const uint64_t* dims, const uint32_t* box) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t gd[3], gs[2];
  cuuint32_t bx[3], es[3] = {1, 1, 1};
  uint64_t stride = esize;
  for (int i = 0; i < rank; i++) {
    gd[i] = dims[i];
    bx[i] = box[i];
    if (i < rank - 1) { stride *= dims[i]; gs[i] = stride; }
  }
  return fn(m, dt, rank, const_cast<void*>(base), gd, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// epilogue store maps: bf16 [outer][inner] boxes of 32 x 32 (SWIZZLE_64B); fp32 dW [El][rows][cols]
// boxes of 32 x 32 x 1 (SWIZZLE_128B); out-of-range rows / columns are clipped by the TMA unit.
bool map2d_st(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer) {
  if (!base) { memset(m, 0, sizeof *m); return true; }
  uint64_t d[2] = {inner, outer};
  uint32_t b[2] = {32, 32};
  return make_map_t(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, CU_TENSOR_MAP_SWIZZLE_64B, base, 2, d, b);
}
bool map2d_st16(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer) {
  uint64_t d[2] = {inner, outer};
  uint32_t b[2] = {16, 32};
  return make_map_t(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, CU_TENSOR_MAP_SWIZZLE_32B, base, 2, d, b);
}
bool map3d_f32(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2) {
  uint64_t d[3] = {d0, d1, d2};
  uint32_t b[3] = {32, 32, 1};
  return make_map_t(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, CU_TENSOR_MAP_SWIZZLE_128B, base, 3, d, b);
}

bool map2d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint32_t box_in, uint32_t box_out,
           uint64_t ld = 0) {
  uint64_t d[2] = {inner, outer}, s[1] = {(ld ? ld : inner) * 2};
  uint32_t b[2] = {box_in, box_out};
  return make_map(m, base, 2, d, s, b);
}
// fp32 [outer][ld] store map over the first `inner` columns, boxes of 16 x 32 (SWIZZLE_64B)
bool map2d_st_f32(CUtensorMap* m, const void* base, uint64_t inner, uint64_t ld, uint64_t outer) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t gd[2] = {inner, outer}, gs[1] = {ld * 4};
  cuuint32_t bx[2] = {16, 32}, es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), gd, gs, bx, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
bool map3d(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0, uint32_t b1) {
  uint64_t d[3] = {d0, d1, d2}, s[2] = {d0 * 2, d0 * d1 * 2};
  uint32_t b[3] = {b0, b1, 1};
  return make_map(m, base, 3, d, s, b);
}

// Wave pacing (profiles/r01_gemm_dram_pacing.md): opt-in, MEMFINE_WAVE_SYNC=1.  It cuts DRAM traffic
// 2-15 %, but the step time moved -5 % on two boxes and +3..6 % on another (lock-stepped units hit
// the same L2 lines at once), so it is not the default.  Even when asked for, it is used only where
// the caller guarantees no concurrent kernel holds SMs (gp.pace: EP = 1, one stream) - elsewhere a
// non-resident unit would make the others sit out the spin bound.  One counter per launch from a
// ring, zeroed on the launch's stream.
int setup_pacing(Params& p, const GemmProblem<__nv_bfloat16>& gp, cudaStream_t st) {
  static const int env_wave = [] {
    const char* s = getenv("MEMFINE_WAVE_SYNC");
    return s ? atoi(s) : -1;
  }();
  static const int env_kb = [] {
    const char* s = getenv("MEMFINE_PACE_KB");
    return s ? atoi(s) : 0;   // sub-tile steps measured worse (dX 7.3 -> 9.3 ms at 64)
  }();
  static int* ctr_ring = nullptr;
  static std::atomic<unsigned> ctr_next{0};
  p.wave_ctr = nullptr;
  if (!(env_wave == 1 && gp.pace && gp.sm_limit <= 0)) return 0;
  static std::once_flag once;
  std::call_once(once, [] { if (cudaMalloc(&ctr_ring, 4096 * sizeof(int)) != cudaSuccess) ctr_ring = nullptr; });
  if (!ctr_ring) return -1;
  p.wave_ctr = ctr_ring + (ctr_next++ & 4095u);
  p.pace_kb = env_kb;
  static const int env_slack = [] {
    const char* s = getenv("MEMFINE_PACE_SLACK");
    return s ? std::max(1, atoi(s)) : 1;
  }();
  p.pace_slack = env_slack;
  return cudaMemsetAsync(p.wave_ctr, 0, sizeof(int), st) == cudaSuccess ? 0 : -1;
}

int g_num_sms = 0;


bool use_pairs() {
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("MEMFINE_GEMM_CTA");
    v = (s && s[0] == '1') ? 0 : 1;  // default: 2-CTA pairs (cta_group::2); MEMFINE_GEMM_CTA=1 for 1-CTA
  }
  return v == 1;
}

template <int KIND, bool PAIR, bool QD = false>
int launch(const GemmProblem<__nv_bfloat16>& gp, cudaStream_t st) {
  using CF = Cfg<KIND>;
  constexpr int BN = CF::BN;
  constexpr int MMA_N = CF::NACC * BN;
  constexpr int B_ROWS = PAIR ? MMA_N / 2 : MMA_N;
  constexpr int SMEM = smem_bytes<KIND, PAIR, false, QD>();
  static_assert(SMEM <= 232448, "smem");
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(gemm_kernel<KIND, PAIR, false, QD>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM) !=
        cudaSuccess)
      return -1;
    attr_set = true;
  }
  if (!g_num_sms) {
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  Params p{};
  p.El = gp.El;
  p.h = gp.h;
  p.g = gp.g;
  p.rows_cap = gp.rows_cap;
  p.seg = gp.seg;
  p.pseg = gp.pseg;
  p.info = gp.info;
  p.GU = gp.GU;
  p.A = gp.A;
  p.O = gp.O;
  p.w_row = gp.w_row;
  p.dw_row = gp.dw_row;
  p.store_a = gp.store_a;
  p.store_gu = gp.store_gu;
  p.beta = gp.wgrad_beta;
  p.row_addr = gp.row_addr;
  p.mx_gq = gp.mx_gq;
  p.mx_gq_sf = gp.mx_gq_sf;
  p.out_f32 = gp.out_f32;
  const uint64_t R = (uint64_t)gp.rows_cap, h = gp.h, g = gp.g, El = gp.El;
  if (R == 0) return 0;
  const uint64_t Rin = gp.rows_in > 0 ? (uint64_t)gp.rows_in : R;   // rows the operand maps hold
  CUtensorMap mA, mB0, mB1, mO0, mO1;
  bool ok = true;
  const uint32_t gu_rows = PAIR ? BN : BN;  // per-CTA B box rows for GATEUP (one of W_gate / W_up)
  switch (KIND) {
    case GK_GATEUP:
      p.N = gp.g; p.K = gp.h;
      ok &= map2d(&mA, gp.X, h, R, BK, BM);
      ok &= map3d(&mB0, gp.Wg, h, g, El, BK, gu_rows);
      ok &= map3d(&mB1, gp.Wu, h, g, El, BK, gu_rows);
      ok &= map2d_st(&mO0, gp.GU ? (const void*)gp.GU : (const void*)gp.A, gp.GU ? 2 * g : g, R);
      ok &= map2d_st(&mO1, gp.A ? (const void*)gp.A : (const void*)gp.GU, gp.A ? g : 2 * g, R);
      break;
    case GK_DOWN:
      p.N = gp.h; p.K = gp.g;
      ok &= map2d(&mA, gp.A, g, Rin, BK, BM);
      ok &= map3d(&mB0, gp.Wd, g, h, El, BK, B_ROWS);
      mB1 = mB0;
      if (gp.out_f32) ok &= map2d_st_f32(&mO0, gp.O, h, gp.ld_out > 0 ? (uint64_t)gp.ld_out : h, Rin);
      else ok &= map2d_st(&mO0, gp.O, h, R);
      mO1 = mO0;
      break;
    case GK_DACT:
      p.N = gp.g; p.K = gp.h;
      ok &= map2d(&mA, gp.DY, h, R, BK, BM);
      ok &= map3d(&mB0, gp.Wd, g, h, El, 64, BK);   // B(n,k) = W_down[e][k][n]
      mB1 = mB0;
      ok &= map2d_st16(&mO0, gp.GU, 2 * g, R);
      ok &= map2d_st16(&mO1, gp.A, g, R);
      break;
    case GK_DX:
      p.N = gp.h; p.K = 2 * gp.g;
      ok &= map2d(&mA, gp.GU, 2 * g, R, BK, BM);
      ok &= map3d(&mB0, gp.Wg, h, g, El, 64, BK);   // B(n,k) = W_gate[e][k][n]
      ok &= map3d(&mB1, gp.Wu, h, g, El, 64, BK);
      ok &= map2d_st(&mO0, gp.O, h, R);
      mO1 = mO0;
      break;
    case GK_WGRAD_DOWN:
      p.M = gp.h; p.N = gp.g;
      ok &= map2d(&mA, gp.DY, h, Rin, 64, BK, gp.ld_a > 0 ? (uint64_t)gp.ld_a : 0);   // A(m,k) = dY[s0+k][m]
      ok &= map2d(&mB0, gp.A, g, Rin, 64, BK);      // B(n,k) = a_w[s0+k][n]
      mB1 = mB0;
      p.dW0 = gp.dWd;
      ok &= map3d_f32(&mO0, gp.dWd, g, h, El);
      mO1 = mO0;
      break;
    default:
      p.M = 2 * gp.g; p.N = gp.h;
      ok &= map2d(&mA, gp.GU, 2 * g, R, 64, BK);    // A(m,k) = dGU[s0+k][m]
      ok &= map2d(&mB0, gp.X, h, R, 64, BK);        // B(n,k) = X[s0+k][n]
      mB1 = mB0;
      p.dW0 = gp.dWg;
      p.dW1 = gp.dWu;
      ok &= map3d_f32(&mO0, gp.dWg, h, g, El);
      ok &= map3d_f32(&mO1, gp.dWu, h, g, El);
      break;
  }
  if (!ok) return -1;
  constexpr int TM = PAIR ? 2 * BM : BM;
  int nt = (p.N + BN - 1) / BN;
  const int per_unit = PAIR ? 2 : 1;
  const int units_hw = (gp.sm_limit > 0 ? std::min(gp.sm_limit, g_num_sms) : g_num_sms) / per_unit;
  {
    // Raster group: gm M tiles x all N tiles, gm sized so the group's A strips take a per-kind L2
    // budget.  Cycles do not depend on it, DRAM traffic does - and under the power cap DRAM energy
    // costs SM clock (profiles/r01_l2_group_sweep.md: 8..96 MB, same cycles, 72..123 GB per step,
    // 1.10..1.30 GHz).  Per-kind minima of the Mixtral step: gate/up and dA 24 MB, down, dX and
    // dW_gate/up 8 MB, dW_down 48 MB.  MEMFINE_L2_GROUP_MB overrides every kind (0 = square-ish
    // wave block, gm ~ sqrt(units * B_strip / A_strip)).
    static const int64_t env_budget = [] {
      const char* s = getenv("MEMFINE_L2_GROUP_MB");
      return s ? (int64_t)atoi(s) << 20 : (int64_t)-1;
    }();
    constexpr int64_t kind_mb = (KIND == GK_DOWN || KIND == GK_DX || KIND == GK_WGRAD_GU) ? 8
                                : KIND == GK_WGRAD_DOWN ? 48 : 24;
    const int64_t budget = env_budget >= 0 ? env_budget : kind_mb << 20;
    int64_t kdim = (KIND >= GK_WGRAD_DOWN) ? (int64_t)std::max<int64_t>(1, R / std::max<uint64_t>(1, El)) : p.K;
    int64_t a_strip = (int64_t)TM * (QD ? 2 : 1) * kdim * 2, b_strip = (int64_t)BN * kdim * 2;
    if (budget) {
      p.group_m = (int)std::max<int64_t>(1, std::min<int64_t>(64, budget / std::max<int64_t>(1, a_strip)));
    } else {
      double gm = std::sqrt((double)units_hw * (double)b_strip / (double)a_strip);
      p.group_m = (int)std::max<double>(1.0, std::min<double>(64.0, std::floor(gm + 0.5)));
    }
  }
  if (setup_pacing(p, gp, st)) return -1;
  int64_t max_tiles;
  if (KIND >= GK_WGRAD_DOWN) {
    p.num_mt_w = (p.M + TM - 1) / TM;
    max_tiles = (int64_t)p.El * p.num_mt_w * nt;
  } else {
    max_tiles = QD ? (int64_t)((R / BM + 3 * El) / 4 + 1) * nt
                   : (int64_t)((R / BM + (PAIR ? El : 0)) / (PAIR ? 2 : 1) + 1) * nt;
  }
  int units = (int)std::min<int64_t>(max_tiles, units_hw);
  if (units <= 0) return 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(units * per_unit);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = per_unit;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (use_pdl() && !p.wave_ctr) ? 2 : 1;   // (a pacing memset precedes a paced launch)
  CUtensorMap none;
  memset(&none, 0, sizeof none);
  if (cudaLaunchKernelEx(&cfg, gemm_kernel<KIND, PAIR, false, QD>, p, mA, mB0, mB1, mO0, mO1, none, none, none) !=
      cudaSuccess)
    return -1;
  return 1;
}

constexpr int64_t kQuadMinK = 8192;

template <int KIND>
int launch_kind(const GemmProblem<__nv_bfloat16>& gp, cudaStream_t st) {
  if constexpr (KIND == GK_DOWN || KIND == GK_DX) {
    // 512 x 256 quad tiles for the two long-K GEMMs (MEMFINE_QUAD=0: 256 x 256 pairs; =2: quads whatever the
    // size - tests); the quad prefix lives in 1 KB of shared memory (E_l <= 255); the router's fp32-output DOWN
    // launch keeps pairs.  Read per launch (a test flips it).
    const char* qs = getenv("MEMFINE_QUAD");
    const int env_quad = qs ? atoi(qs) : 1;
    // quads halve the tile count, so they need enough work per launch to keep the last wave's tail small:
    // at least 8 waves of quad tiles at the chunk's row capacity (the full-size C = 1 Mixtral layer has 14)
    const int64_t quads = gp.rows_cap / (4 * BM) + 1, nt_q = (gp.h + 255) / 256;
    const int units = (g_num_sms ? g_num_sms : 148) / 2;
    // and a long K: a quad's accumulator is single-buffered, so its drain is exposed once per tile; at
    // K >= 8192 (Mixtral's down, K = g = 14336, and dX, K = 2g) that is a few % of the mainloop, at the
    // short K of DeepSeek-V3 / Qwen3 (down K = 2048 / 1536, dX 4096 / 3072) the pairs' double-buffered
    // accumulators win (profiles/r02d_lib_ab_quad_k)
    const int64_t K = KIND == GK_DOWN ? (int64_t)gp.g : 2 * (int64_t)gp.g;
    if (use_pairs() && env_quad && !gp.out_f32 && gp.El <= 255 &&
        (env_quad == 2 || (quads * nt_q >= 8 * units && K >= kQuadMinK)))
      return launch<KIND, true, true>(gp, st);
  }
  return use_pairs() ? launch<KIND, true>(gp, st) : launch<KIND, false>(gp, st);
}

// E4M3 maps: K-major rows, 128 K (bytes) x box rows, 128B swizzle
bool map_fp8_2d(CUtensorMap* m, const void* base, uint64_t K, uint64_t rows) {
  uint64_t d[2] = {K, rows};
  uint32_t b[2] = {128, 128};
  return make_map_t(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, CU_TENSOR_MAP_SWIZZLE_128B, base, 2, d, b);
}
bool map_fp8_2d_box(CUtensorMap* m, const void* base, uint64_t K, uint64_t rows, uint32_t box_rows) {
  uint64_t d[2] = {K, rows};
  uint32_t b[2] = {128, box_rows};
  return make_map_t(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, CU_TENSOR_MAP_SWIZZLE_128B, base, 2, d, b);
}
bool map_fp8_3d(CUtensorMap* m, const void* base, uint64_t K, uint64_t rows, uint64_t El, uint32_t box_rows) {
  uint64_t d[3] = {K, rows, El};
  uint32_t b[3] = {128, box_rows, 1};
  return make_map_t(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, CU_TENSOR_MAP_SWIZZLE_128B, base, 3, d, b);
}

// MEMFINE_MX_SPLITN=1 (1-CTA only): two N=128 block-scaled MMAs instead of one N=256
int mx_flags() {
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("MEMFINE_MX_SPLITN");
    v = (s && s[0] == '1') ? 1 : 0;
  }
  return v;
}

bool mx_pairs() {
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("MEMFINE_MX_CTA");
    v = (s && s[0] == '1') ? 0 : 1;   // default: cta_group::2 pairs; MEMFINE_MX_CTA=1 for 1-CTA
  }
  return v == 1;
}
// scale chunks as uint32 rows of 128 words (512 B), one TMA box per chunk
bool map_sf(CUtensorMap* m, const void* base, uint64_t nchunks) {
  uint64_t d[2] = {128, nchunks};
  uint32_t b[2] = {128, 1};
  return make_map_t(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, CU_TENSOR_MAP_SWIZZLE_NONE, base, 2, d, b);
}

// MXFP8 launch (K-major E4M3 operands, block scales): the four M-tiled kinds; PAIR = cta_group::2.
template <int KIND, bool PAIR>
int launch_mx(const GemmProblem<__nv_bfloat16>& gp, cudaStream_t st) {
  constexpr int SMEM = smem_bytes<KIND, PAIR, true>();
  static_assert(SMEM <= 232448, "smem");
  constexpr int BROWS = CfgX<KIND, true>::NACC * CfgX<KIND, true>::BN;     // B tile rows
  constexpr uint32_t BOX = KIND == GK_GATEUP ? 128 : (PAIR ? BROWS / 2 : BROWS);  // B rows per TMA load
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(gemm_kernel<KIND, PAIR, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM) !=
        cudaSuccess)
      return -1;
    attr_set = true;
  }
  if (!g_num_sms) {
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  Params p{};
  p.El = gp.El;
  p.h = gp.h;
  p.g = gp.g;
  p.rows_cap = gp.rows_cap;
  p.seg = gp.seg;
  p.pseg = gp.pseg;
  p.info = gp.info;
  p.GU = gp.GU;
  p.A = gp.A;
  p.O = gp.O;
  p.w_row = gp.w_row;
  p.dw_row = gp.dw_row;
  p.store_a = gp.store_a;
  p.store_gu = gp.store_gu;
  p.row_addr = gp.row_addr;
  p.mx_a_sf = gp.mx_a.sf;
  p.mx_b0_sf = gp.mx_b0.sf;
  p.mx_b1_sf = gp.mx_b1.sf;
  p.mx_aq = gp.mx_aq;
  p.mx_aq_sf = gp.mx_aq_sf;
  p.mx_split_n = mx_flags();
  const uint64_t R = (uint64_t)gp.rows_cap, h = gp.h, g = gp.g, El = gp.El;
  if (R == 0) return 0;
  if (h % 128 || g % 128 || R % 128) return -1;
  CUtensorMap mA, mB0, mB1, mO0, mO1, mSA, mSB0, mSB1;
  bool ok = true;
  const uint64_t wch = El * (h / 128) * (g / 128);   // scale chunks of one weight operand
  switch (KIND) {
    case GK_GATEUP:
      p.N = gp.g; p.K = gp.h;
      ok &= map_sf(&mSB0, gp.mx_b0.sf, wch);
      ok &= map_sf(&mSB1, gp.mx_b1.sf, wch);
      ok &= map_fp8_2d(&mA, gp.mx_a.q, h, R);
      ok &= map_fp8_3d(&mB0, gp.mx_b0.q, h, g, El, 128);
      ok &= map_fp8_3d(&mB1, gp.mx_b1.q, h, g, El, 128);
      if (gp.store_gu) {
        ok &= map2d_st(&mO0, gp.GU, 2 * g, R);
        mO1 = mO0;
      } else {
        memset(&mO0, 0, sizeof mO0);
        memset(&mO1, 0, sizeof mO1);
      }
      break;
    case GK_DOWN:
      p.N = gp.h; p.K = gp.g;
      ok &= map_fp8_2d(&mA, gp.mx_a.q, g, R);
      ok &= map_fp8_3d(&mB0, gp.mx_b0.q, g, h, El, BOX);
      mB1 = mB0;
      ok &= map_sf(&mSB0, gp.mx_b0.sf, wch);
      mSB1 = mSB0;
      ok &= map2d_st(&mO0, gp.O, h, R);
      mO1 = mO0;
      break;
    case GK_WGRAD_DOWN:
      // dW_down[e] (+)= dY^T a_w over the expert's copies: A = dY columnwise codes [h][R],
      // B = a_w columnwise codes [g][R] (reading R28c)
      p.M = gp.h; p.N = gp.g; p.K = (int)R;
      ok &= map_fp8_2d(&mA, gp.mx_a.q, R, h);
      ok &= map_fp8_2d_box(&mB0, gp.mx_b0.q, R, g, BOX);
      mB1 = mB0;
      ok &= map_sf(&mSB0, gp.mx_b0.sf, (g / 128) * (R / 128));
      mSB1 = mSB0;
      p.dW0 = gp.dWd;
      p.beta = gp.wgrad_beta;
      ok &= map3d_f32(&mO0, gp.dWd, g, h, El);
      mO1 = mO0;
      break;
    case GK_WGRAD_GU:
      // dW_gate || dW_up[e] (+)= dGU^T x: A = dG || dU columnwise codes [2g][R], B = x's [h][R]
      p.M = 2 * gp.g; p.N = gp.h; p.K = (int)R;
      ok &= map_fp8_2d(&mA, gp.mx_a.q, R, 2 * g);
      ok &= map_fp8_2d_box(&mB0, gp.mx_b0.q, R, h, BOX);
      mB1 = mB0;
      ok &= map_sf(&mSB0, gp.mx_b0.sf, (h / 128) * (R / 128));
      mSB1 = mSB0;
      p.dW0 = gp.dWg;
      p.dW1 = gp.dWu;
      p.beta = gp.wgrad_beta;
      ok &= map3d_f32(&mO0, gp.dWg, h, g, El);
      ok &= map3d_f32(&mO1, gp.dWu, h, g, El);
      break;
    default:  // GK_DX
      p.N = gp.h; p.K = 2 * gp.g;
      ok &= map_fp8_2d(&mA, gp.mx_a.q, 2 * g, R);
      ok &= map_fp8_3d(&mB0, gp.mx_b0.q, g, h, El, BOX);    // W_gate^T [El][h][g]
      ok &= map_fp8_3d(&mB1, gp.mx_b1.q, g, h, El, BOX);    // W_up^T
      ok &= map_sf(&mSB0, gp.mx_b0.sf, wch);
      ok &= map_sf(&mSB1, gp.mx_b1.sf, wch);
      ok &= map2d_st(&mO0, gp.O, h, R);
      mO1 = mO0;
      break;
  }
  ok &= map_sf(&mSA, gp.mx_a.sf,
                KIND >= GK_WGRAD_DOWN ? (uint64_t)(p.M / 128) * (R / 128) : (R / 128) * (uint64_t)(p.K / 128));
  if (!ok) return -1;
  constexpr int BN = CfgX<KIND, true>::BN;
  int nt = (p.N + BN - 1) / BN;
  {
    // the same per-kind raster budgets as the BF16 kernels (launch<>); MEMFINE_L2_GROUP_MB overrides
    static const int64_t env_budget = [] {
      const char* s = getenv("MEMFINE_L2_GROUP_MB");
      return s ? (int64_t)atoi(s) << 20 : (int64_t)-1;
    }();
    constexpr int64_t kind_mb = (KIND == GK_DOWN || KIND == GK_DX || KIND == GK_WGRAD_GU) ? 8
                                : KIND == GK_WGRAD_DOWN ? 48 : 24;
    const int64_t budget = env_budget > 0 ? env_budget : kind_mb << 20;
    const int64_t kdim = KIND >= GK_WGRAD_DOWN ? std::max<int64_t>(1, (int64_t)(R / El)) : p.K;
    int64_t a_strip = (int64_t)(PAIR ? 2 : 1) * BM * kdim;   // E4M3: one byte per element
    p.group_m = (int)std::max<int64_t>(1, std::min<int64_t>(64, budget / a_strip));
  }
  if (setup_pacing(p, gp, st)) return -1;
  const int per_unit = PAIR ? 2 : 1;
  int64_t max_tiles;
  if (KIND >= GK_WGRAD_DOWN) {
    p.num_mt_w = (p.M + (PAIR ? 2 : 1) * BM - 1) / ((PAIR ? 2 : 1) * BM);
    max_tiles = (int64_t)p.El * p.num_mt_w * nt;
  } else {
    max_tiles = (int64_t)((R / BM + (PAIR ? El : 0)) / per_unit + 1) * nt;
  }
  const int sms = gp.sm_limit > 0 ? std::min(gp.sm_limit, g_num_sms) : g_num_sms;
  int units = (int)std::min<int64_t>(max_tiles, sms / per_unit);
  if (units <= 0) return 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(units * per_unit);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = per_unit;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = use_pdl() ? 2 : 1;
  if (cudaLaunchKernelEx(&cfg, gemm_kernel<KIND, PAIR, true>, p, mA, mB0, mB1, mO0, mO1, mSA, mSB0, mSB1) !=
      cudaSuccess)
    return -1;
  return 1;
}

template <int KIND>
int launch_mx_kind(const GemmProblem<__nv_bfloat16>& gp, cudaStream_t st) {
  return mx_pairs() ? launch_mx<KIND, true>(gp, st) : launch_mx<KIND, false>(gp, st);
}

}  // namespace sm100

int launch_gemm_sm100(const GemmProblem<__nv_bfloat16>& p, cudaStream_t st) {
  if (p.mx) {
    switch (p.kind) {
      case GK_GATEUP: return sm100::launch_mx_kind<GK_GATEUP>(p, st);
      case GK_DOWN: return sm100::launch_mx_kind<GK_DOWN>(p, st);
      case GK_DX: return sm100::launch_mx_kind<GK_DX>(p, st);
      case GK_WGRAD_DOWN: return sm100::launch_mx_kind<GK_WGRAD_DOWN>(p, st);   // reading R28c
      case GK_WGRAD_GU: return sm100::launch_mx_kind<GK_WGRAD_GU>(p, st);
      default: break;   // dA stays BF16 (reading R28)
    }
  }
  switch (p.kind) {
    case GK_GATEUP: return sm100::launch_kind<GK_GATEUP>(p, st);
    case GK_DOWN: return sm100::launch_kind<GK_DOWN>(p, st);
    case GK_DACT: return sm100::launch_kind<GK_DACT>(p, st);
    case GK_DX: return sm100::launch_kind<GK_DX>(p, st);
    case GK_WGRAD_DOWN: return sm100::launch_kind<GK_WGRAD_DOWN>(p, st);
    case GK_WGRAD_GU: return sm100::launch_kind<GK_WGRAD_GU>(p, st);
  }
  return -1;
}

int sm100_num_sms() { return sm100::g_num_sms ? sm100::g_num_sms : 148; }

const void* kernel_anchor_sm100() { return (const void*)sm100::gemm_kernel<GK_DOWN, true>; }

}  // namespace memfine
