// gemm_sm100.cu — grouped expert GEMMs on the 5th-generation tensor cores (sm_100a).
//
// One persistent, warp-specialised kernel template serves the six expert GEMMs of the
// chunked MoE layer.  Per CTA (one per SM, 192 threads):
//   warp 0      TMA producer: cp.async.bulk.tensor 2D/3D loads, 128B swizzle, mbarrier tx
//   warp 1      TMEM allocator + MMA issuer: tcgen05.mma.cta_group::1.kind::f16, BF16 in,
//               FP32 accumulators in TMEM, tcgen05.commit -> mbarriers
//   warps 2..9  epilogue: tcgen05.ld 32x32b -> registers -> fused MoE epilogue -> global;
//               two warps per TMEM lane quarter (warp % 4), each taking half of the columns
// A 4-stage smem ring (48 KB/stage) feeds the MMA; two TMEM accumulator stages (512 cols)
// let the epilogue of tile i overlap the mainloop of tile i+1.
//
// Rows are the expert-major padded layout (every local expert's segment padded to 128
// rows), so an M tile never straddles experts and the weight-gradient K loop (over tokens)
// never straddles either; padded rows are zero.  Tile order is grouped (8 M tiles x all N
// tiles) so the weights and activations a wave touches stay in the 126 MB L2.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <mutex>
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

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
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
__device__ __forceinline__ void stage_f32_row(uint8_t* buf, int r, const float* v) {
  uint8_t* row = buf + r * 128;
#pragma unroll
  for (int c = 0; c < 8; c++)
    *reinterpret_cast<float4*>(row + ((c ^ (r & 7)) << 4)) =
        make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
}

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

// Epilogue staging per epilogue warp and chunk of 32 columns: output slots x slot bytes,
// double-buffered across chunks.
template <int KIND>
struct Epi {
  static constexpr int SLOTS = KIND == GK_DACT ? 3 : (KIND == GK_GATEUP ? 2 : 1);
  // dA works in 16-column sub-chunks (32 rows x 32 B, SWIZZLE_32B) so its staging is 24 KB
  static constexpr int SLOT_BYTES = KIND >= GK_WGRAD_DOWN ? 4096 : (KIND == GK_DACT ? 1024 : 2048);
  static constexpr int CHUNK_BYTES = SLOTS * SLOT_BYTES;
  // dA and dW: single-buffered staging so the mainloop keeps one more stage of operands in flight
  // (measured: dA 72% -> 82% tensor-active going from 4 to 5 stages); the others double-buffer.
  static constexpr int BUFS = (KIND == GK_DACT || KIND >= GK_WGRAD_DOWN) ? 1 : 2;
  static constexpr int WARP_BYTES = BUFS * CHUNK_BYTES;
  static constexpr int TOTAL = EPI_WARPS * WARP_BYTES;
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
};

struct Tile {
  int e;      // local expert
  int m0;     // first row of the (pair) tile: padded row (M-tiled kinds) or dW row (WGRAD)
  int m_end;  // rows >= m_end are not stored (expert segment end / M)
  int n0, k0, nkb;
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

template <int KIND, bool PAIR>
__device__ __forceinline__ int num_tiles(const Params& p) {
  constexpr int BN = Cfg<KIND>::BN;
  int nt = (p.N + BN - 1) / BN;
  if (KIND >= GK_WGRAD_DOWN) return p.El * p.num_mt_w * nt;
  if (p.info[kInfoSkip]) return 0;
  return (PAIR ? p.info[kInfoPairs] : p.info[kInfoRowsPad] / BM) * nt;
}

template <int KIND, bool PAIR>
__device__ __forceinline__ Tile tile_of(const Params& p, int t) {
  constexpr int BN = Cfg<KIND>::BN;
  constexpr int TM = PAIR ? 2 * BM : BM;  // rows per (pair) tile
  int nt = (p.N + BN - 1) / BN;
  Tile T;
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
    T.nkb = (s1 - s0) / BK;
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
  T.nkb = p.K / BK;
  return T;
}

template <int KIND, bool PAIR>
__host__ __device__ constexpr int stage_bytes() {
  return A_BYTES + (PAIR ? Cfg<KIND>::NACC * Cfg<KIND>::BN / 2 : Cfg<KIND>::NACC * Cfg<KIND>::BN) * BK * 2;
}
// as many 1024-aligned stages as fit next to the epilogue staging (227 KB per CTA)
template <int KIND, bool PAIR>
__host__ __device__ constexpr int nstage() {
  return (232448 - 1024 - 512 - Epi<KIND>::TOTAL) / stage_bytes<KIND, PAIR>() > 6
             ? 6
             : (232448 - 1024 - 512 - Epi<KIND>::TOTAL) / stage_bytes<KIND, PAIR>();
}
template <int KIND, bool PAIR>
__host__ __device__ constexpr int smem_bytes() {
  return nstage<KIND, PAIR>() * stage_bytes<KIND, PAIR>() + Epi<KIND>::TOTAL + 1024 + 512;
}

// ------------------------------------------------------------------ the kernel
// PAIR = false: one CTA per 128-row tile, tcgen05.mma.cta_group::1 (M=128).
// PAIR = true : a 2-CTA cluster per 256-row tile, tcgen05.mma.cta_group::2 (M=256) issued by the
//               even CTA; each CTA stages 128 rows of A and half of B's columns, each CTA's TMEM
//               holds its 128 rows x N accumulator.  Per-CTA operand traffic drops by a third.
template <int KIND, bool PAIR>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_kernel(const __grid_constant__ Params p, const __grid_constant__ CUtensorMap tmA,
                const __grid_constant__ CUtensorMap tmB0, const __grid_constant__ CUtensorMap tmB1,
                const __grid_constant__ CUtensorMap tmO0, const __grid_constant__ CUtensorMap tmO1) {
  using CF = Cfg<KIND>;
  constexpr int BN = CF::BN, NACC = CF::NACC;
  constexpr int MMA_N = NACC * BN;                      // GATEUP: G||U in one MMA (N = 256)
  static_assert(MMA_N <= 256, "MMA N");
  constexpr int B_ROWS = PAIR ? MMA_N / 2 : MMA_N;      // B rows (N) staged per CTA
  constexpr int B_BYTES = B_ROWS * BK * 2;
  constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr int NSTAGE = nstage<KIND, PAIR>();
  constexpr int ACC_COLS = MMA_N;                       // per accumulator stage
  constexpr uint32_t TMEM_COLS = 2 * ACC_COLS;          // double-buffered
  static_assert(TMEM_COLS <= 512, "TMEM");
  constexpr uint32_t IDESC = idesc_bf16(PAIR ? 2 * BM : BM, MMA_N, CF::A_MN, CF::B_MN);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* epi_smem = smem + NSTAGE * STAGE_BYTES;      // 1024-aligned (STAGE_BYTES is)
  uint64_t* full = (uint64_t*)(epi_smem + Epi<KIND>::TOTAL);
  uint64_t* empty = full + NSTAGE;
  uint64_t* tfull = empty + NSTAGE;
  uint64_t* tempty = tfull + 2;
  uint64_t* ebar = tempty + 2;                          // [EPI_WARPS][2] epilogue TMA-load barriers (dA)
  uint32_t* tmem_slot = (uint32_t*)(ebar + 2 * EPI_WARPS);

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
    for (int s = 0; s < NSTAGE; s++) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
    for (int a = 0; a < 2; a++) { mbar_init(tfull + a, 1); mbar_init(tempty + a, (PAIR ? 2 : 1) * EPI_WARPS); }
    for (int i = 0; i < 2 * EPI_WARPS; i++) mbar_init(ebar + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    if (PAIR) {
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
  const int ntiles = num_tiles<KIND, PAIR>(p);

  if (warp == 0) {
    // ================================================================ TMA producer (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cid; t < ntiles; t += ncid) {
        Tile T = tile_of<KIND, PAIR>(p, t);
        const int am0 = T.m0 + (int)rank * BM;              // this CTA's A rows
        for (int kb = 0; kb < T.nkb; kb++) {
          mbar_wait(empty + stage, phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          if (leader) mbar_expect_tx(full + stage, (PAIR ? 2 : 1) * STAGE_BYTES);
          int kc = T.k0 + kb * BK;
          auto L2 = [&](void* dst, const CUtensorMap* m, int c0, int c1) {
            if (PAIR) tma_2d_pair(dst, m, full + stage, c0, c1); else tma_2d(dst, m, full + stage, c0, c1);
          };
          auto L3 = [&](void* dst, const CUtensorMap* m, int c0, int c1, int c2) {
            if (PAIR) tma_3d_pair(dst, m, full + stage, c0, c1, c2); else tma_3d(dst, m, full + stage, c0, c1, c2);
          };
          if (CF::A_MN) {
            // A(m,k) = rows[kc + k][am0 + m]: two 64-wide MN atoms of 64 K rows
            L2(sa, &tmA, am0, kc);
            L2(sa + 8192, &tmA, am0 + 64, kc);
          } else {
            L2(sa, &tmA, kc, am0);
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
        Tile T = tile_of<KIND, PAIR>(p, t);
        if (T.nkb == 0) continue;
        int as = it & 1;
        uint32_t aph = (it >> 1) & 1;
        mbar_wait(tempty + as, aph ^ 1);
        fence_after();
        uint32_t dbase = tmem_base + as * ACC_COLS;
        for (int kb = 0; kb < T.nkb; kb++) {
          mbar_wait(full + stage, phase);
          fence_after();
          uint32_t sa = su32(smem + stage * STAGE_BYTES);
          uint32_t sb = sa + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; k++) {
            uint64_t ad = CF::A_MN ? sdesc(sa + k * 2048, 8192, 1024) : sdesc(sa + k * 32, 16, 1024);
            uint64_t bd = CF::B_MN ? sdesc(sb + k * 2048, 8192, 1024) : sdesc(sb + k * 32, 16, 1024);
            if (PAIR) mma_bf16_pair(dbase, ad, bd, IDESC, (kb | k) != 0);
            else mma_bf16(dbase, ad, bd, IDESC, (kb | k) != 0);
          }
          if (PAIR) mma_commit_pair(empty + stage); else mma_commit(empty + stage);
          if (++stage == NSTAGE) { stage = 0; phase ^= 1; }
        }
        if (PAIR) mma_commit_pair(tfull + as); else mma_commit(tfull + as);
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
    using EP = Epi<KIND>;
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
      Tile T = tile_of<KIND, PAIR>(p, t);
      const int row0 = T.m0 + (int)rank * BM + q * 32;     // first row of this warp's 32 rows
      const int rowi = row0 + lane;
      const bool rows_ok = row0 < T.m_end;                 // warp-uniform (halves are 128-row aligned)
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
      int as = it & 1;
      uint32_t aph = (it >> 1) & 1;
      const int64_t row = rowi;
      float dwp = 0.f;
      float wrow = 0.f;
      if (KIND == GK_DACT && rows_ok) {
        wrow = p.w_row[row];
        const int n0c = T.n0 + half * CPW;
        if (n0c < p.g) dact_load(0, n0c, row0);   // first chunk's G||U, overlapping the MMA
      }
      mbar_wait(tfull + as, aph);
      fence_after();
      uint32_t tb = tmem_base + as * ACC_COLS + ((uint32_t)(q * 32) << 16);
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
              float a[32];
#pragma unroll
              for (int i = 0; i < 32; i++) a[i] = silu_f(v[i]) * u[i];
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
            uint8_t* buf = next_buf();
            stage_bf16_row(buf, lane, v);
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&tmO0, buf, n, row0);
              bulk_commit();
            }
          }
        } else if (KIND == GK_DACT) {
          if (rows_ok && n < p.g) {
            uint8_t* buf = wbuf;
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
#pragma unroll
              for (int j = 0; j < 8; j++) {
                float r2v[2][3];
#pragma unroll
                for (int q2 = 0; q2 < 2; q2++) {
                  const int i = 16 * h2 + 2 * j + q2;
                  const uint32_t gw = gcur[j], uw = ucur[j];
                  const float G = __uint_as_float(q2 ? (gw & 0xFFFF0000u) : (gw << 16));
                  const float U = __uint_as_float(q2 ? (uw & 0xFFFF0000u) : (uw << 16));
                  const float sg = sigmoid_f(G);
                  const float a = G * sg * U;
                  dwp = fmaf(v[i], a, dwp);
                  const float dA = wrow * v[i];
                  r2v[q2][0] = dA * U * sg * (1.f + G * (1.f - sg));
                  r2v[q2][1] = dA * G * sg;
                  r2v[q2][2] = wrow * a;
                }
                og[j] = pack_bf16(r2v[0][0], r2v[1][0]);
                ou[j] = pack_bf16(r2v[0][1], r2v[1][1]);
                oa[j] = pack_bf16(r2v[0][2], r2v[1][2]);
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
      if (KIND == GK_DACT && rows_ok) atomicAdd(p.dw_row + row, dwp);
      fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR) mbar_arrive_leader(tempty + as); else mbar_arrive(tempty + as);
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
    if (PAIR)
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

bool map2d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint32_t box_in, uint32_t box_out) {
  uint64_t d[2] = {inner, outer}, s[1] = {inner * 2};
  uint32_t b[2] = {box_in, box_out};
  return make_map(m, base, 2, d, s, b);
}
bool map3d(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0, uint32_t b1) {
  uint64_t d[3] = {d0, d1, d2}, s[2] = {d0 * 2, d0 * d1 * 2};
  uint32_t b[3] = {b0, b1, 1};
  return make_map(m, base, 3, d, s, b);
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

template <int KIND, bool PAIR>
int launch(const GemmProblem<__nv_bfloat16>& gp, cudaStream_t st) {
  using CF = Cfg<KIND>;
  constexpr int BN = CF::BN;
  constexpr int MMA_N = CF::NACC * BN;
  constexpr int B_ROWS = PAIR ? MMA_N / 2 : MMA_N;
  constexpr int SMEM = smem_bytes<KIND, PAIR>();
  static_assert(SMEM <= 232448, "smem");
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(gemm_kernel<KIND, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM) !=
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
  const uint64_t R = (uint64_t)gp.rows_cap, h = gp.h, g = gp.g, El = gp.El;
  if (R == 0) return 0;
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
      ok &= map2d(&mA, gp.A, g, R, BK, BM);
      ok &= map3d(&mB0, gp.Wd, g, h, El, BK, B_ROWS);
      mB1 = mB0;
      ok &= map2d_st(&mO0, gp.O, h, R);
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
      ok &= map2d(&mA, gp.DY, h, R, 64, BK);        // A(m,k) = dY[s0+k][m]
      ok &= map2d(&mB0, gp.A, g, R, 64, BK);        // B(n,k) = a_w[s0+k][n]
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
  const int units_hw = g_num_sms / per_unit;
  {
    // Raster group: gm M tiles x all N tiles, gm sized so the group's A strips take ~24 MB of L2
    // (measured best on the Mixtral-size step: less DRAM traffic -> less power -> higher clocks
    // under the 1 kW cap; 48 and 96 MB were slower).  MEMFINE_L2_GROUP_MB=0 selects a square-ish
    // wave block (gm ~ sqrt(units * B_strip / A_strip)) instead; other values set the budget.
    static int64_t budget = [] {
      const char* s = getenv("MEMFINE_L2_GROUP_MB");
      return (int64_t)(s ? atoi(s) : 24) << 20;
    }();
    int64_t kdim = (KIND >= GK_WGRAD_DOWN) ? (int64_t)std::max<int64_t>(1, R / std::max<uint64_t>(1, El)) : p.K;
    int64_t a_strip = (int64_t)TM * kdim * 2, b_strip = (int64_t)BN * kdim * 2;
    if (budget) {
      p.group_m = (int)std::max<int64_t>(1, std::min<int64_t>(64, budget / std::max<int64_t>(1, a_strip)));
    } else {
      double gm = std::sqrt((double)units_hw * (double)b_strip / (double)a_strip);
      p.group_m = (int)std::max<double>(1.0, std::min<double>(64.0, std::floor(gm + 0.5)));
    }
  }
  int64_t max_tiles;
  if (KIND >= GK_WGRAD_DOWN) {
    p.num_mt_w = (p.M + TM - 1) / TM;
    max_tiles = (int64_t)p.El * p.num_mt_w * nt;
  } else {
    max_tiles = (int64_t)((R / BM + (PAIR ? El : 0)) / (PAIR ? 2 : 1) + 1) * nt;
  }
  int units = (int)std::min<int64_t>(max_tiles, units_hw);
  if (units <= 0) return 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(units * per_unit);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = per_unit;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, gemm_kernel<KIND, PAIR>, p, mA, mB0, mB1, mO0, mO1) != cudaSuccess) return -1;
  return 1;
}

template <int KIND>
int launch_kind(const GemmProblem<__nv_bfloat16>& gp, cudaStream_t st) {
  return use_pairs() ? launch<KIND, true>(gp, st) : launch<KIND, false>(gp, st);
}

}  // namespace sm100

int launch_gemm_sm100(const GemmProblem<__nv_bfloat16>& p, cudaStream_t st) {
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

}  // namespace memfine
