// kernels.h — host-side launchers of the libmemfine.so kernels (internal header).
#pragma once
#include "common.cuh"

namespace memfine {

// Per-chunk device metadata carved from the workspace.
struct ChunkMeta {
  int* blk_cnt;    // [NBmax][E]   per token-block expert counts, then (in place) block offsets
  int* exp_cnt;    // [E]          this rank's chunk copies per global expert
  int* recv_cnt;   // [E_l]        rows received per local expert (EP>1; == exp_cnt slice at EP=1)
  int* seg;        // [E_l+1]      padded row segment starts of the local experts
  int* pseg;       // [E_l+1]      prefix of 256-row tile pairs per local expert (2-CTA GEMMs)
  int* info;       // [kInfoWords]
  int* dest_of;    // [Tmax*k]     position of copy (i,slot): expert-major row (EP=1) or send row
  int* src_of;     // [rows_cap]   copy index feeding each row (EP=1, debug/gather), -1 padding
  int* send_src;   // [Tmax*k]     copy index feeding each send row (EP>1)
  int* p2p_tab;    // [C][4E+1]    fused-exchange tables (EP>1, see PeerTable)
  uint64_t* row_addr;    // [rows_cap] fused combine: destination of each row in its source's send buffer
  uint64_t* row_addr_w;  // [rows_cap] ... and of its d_score slot
  float* w_row;    // [rows_cap]   top-k score of each row (0 on padding)
  float* dw_row;   // [rows_cap]   d_score of each row (bwd)
};

// ---------------------------------------------------------------- routing (A1, A5, A10, B7)
void launch_route_hist(const int32_t* ids, int64_t T, int k, int E, int nsub, int* counts,
                       int* status, cudaStream_t st);
void launch_dispatch_hist(const int32_t* ids, int64_t t0, int64_t t1, int k, int E, const ChunkMeta& m,
                          int* status, cudaStream_t st);
// send_layout 0: EP=1 expert-major padded layout; 1: EP send layout (global expert order).
void launch_dispatch_scan(int NB, int E, int El, int send_layout, int64_t rows_cap, const ChunkMeta& m,
                          int64_t* stats_rows, int64_t* stats_rows_pad, int chunk, cudaStream_t st);
// gskip (nullable): per-chunk global skip flags (N1 device plan) OR-ed into the chunk's info word
void launch_ep_recv_seg(const int* counts, int C, int j, int E, int El, int me, int EP, int64_t rows_cap,
                        const ChunkMeta& m, int64_t* stats_rows, int64_t* stats_rows_pad, cudaStream_t st,
                        const int* gskip = nullptr);
// Index pass (stable ranks) + row gather.  expert_major: EP=1 padded layout (padding rows zeroed,
// rows_cap bounds the grid); otherwise the EP send layout.
template <typename T>
void launch_dispatch_scatter(const T* x, const T* dy, const int32_t* ids, const float* w, int64_t t0,
                             int64_t t1, int k, int E, int h, const ChunkMeta& m, T* xd, T* dyd, int El,
                             bool expert_major, int64_t rows_cap, cudaStream_t st,
                             uint8_t* xq = nullptr, uint8_t* xsf = nullptr, bool write_x = true);
// Index pass only (stable ranks -> dest_of, row_src, scores), for the fused P2P dispatch.
void launch_dispatch_index(const int32_t* ids, const float* w, int64_t t0, int64_t t1, int k, int E,
                           const ChunkMeta& m, int* row_src, float* w_row, cudaStream_t st);
template <typename T>
void launch_zero_padding(int El, int h, const ChunkMeta& m, T* xd, T* dyd, cudaStream_t st);
template <typename T>
void launch_combine(const T* O, const float* w, int64_t t0, int64_t t1, int k, int h, const ChunkMeta& m,
                    T* y, cudaStream_t st);
template <typename T>
void launch_unpermute_reduce(const T* dXd, int64_t t0, int64_t t1, int k, int h, const ChunkMeta& m,
                             T* dx, float* dscore, cudaStream_t st);

// ---------------------------------------------------------------- fused EP exchange over peer memory
// Peer buffers of every EP rank, mapped into this process (in-process group: other ranks'
// workspaces on the same device; multi-process: CUDA IPC mappings).
constexpr int kMaxPeers = 16;
struct PeerTable {
  char* X[kMaxPeers];       // expert-major token rows [R][h]
  char* DY[kMaxPeers];      // expert-major dY rows (bwd)
  char* w_row[kMaxPeers];   // per-row scores
  char* send[kMaxPeers];    // send-layout rows: where o / dX rows come back
  char* send_w[kMaxPeers];  // send-layout d_score slots (bwd)
  int n;
};
// Per-chunk table (ints): send_off[E+1] | land[EP*El] | recv_off[EP*El] | ret[EP*El]
//   send_off: prefix of this rank's chunk copies over global experts (its send layout)
//   land[p*El+el]: first row of this rank's copies in rank p's expert-major buffer, expert (p, el)
//   recv_off[s*El+el]: first row of rank s's copies in THIS rank's buffer, local expert el
//   ret[s*El+el]: rank s's send-layout position of its copies of expert (this rank, el)
// A5+A6 fused: one warp per send row writes the token row straight into the receiver's buffer.
template <typename T>
void launch_p2p_push(const T* x, const T* dy, const float* w, int k, int h, int E, int El, int EP,
                     const int* tab, const int* send_src, const int* info, const PeerTable& pt, int64_t rows_ub,
                     cudaStream_t st);
// Row -> destination addresses for the combine direction (0 for padding rows).
void launch_p2p_row_addr(const int* seg, const int* recv_cnt, int El, int EP, const int* tab, int E,
                         const int* info, const PeerTable& pt, int row_bytes, uint64_t* row_addr,
                         uint64_t* row_addr_w, int64_t rows_cap, cudaStream_t st);
// B6 for d_score: each received row's d_w straight into its source rank's send_w slot.
void launch_p2p_push_dw(const float* dw_row, const uint64_t* row_addr_w, const int* info, int64_t rows_cap,
                        cudaStream_t st);

// ---------------------------------------------------------------- N1: device-planned exchange, no host sync
// Every rank owns a small sync area (memfine_register_workspace), mapped by every peer:
//   epoch (uint64, this rank's call counter) | flags[kSyncPhases][kMaxPeers] (uint64, written by peers) |
//   counts[2][kMaxPeers][kMaxSub * E] (int32, the count all-gather landing zone, by call parity)
// A flag value is epoch * 256 + code; waits spin (acquire, system scope) until every peer's flag reaches
// the target, with a bounded spin (latched error, never a hang).
constexpr int kSyncPhases = 4;   // 0 counts, 1 pushed(j), 2 combined(j), 3 done(j)
constexpr int kSyncDoneCall = 255;
struct SyncPeers {
  uint64_t* area[kMaxPeers];     // every rank's sync area (own entry = local)
  int n;
};
uint64_t sync_area_bytes(int E);
// epoch += 1 (one thread; the first kernel of every device-planned call)
void launch_sync_epoch(uint64_t* area, cudaStream_t st);
// this rank's counts [C][E] -> every peer's counts slot (call parity), then flag phase 0 = epoch*256
void launch_sync_push_counts(const int* mine, int C, int E, const SyncPeers& sp, int me, cudaStream_t st);
// flag `phase` of this rank in every peer's area := epoch * 256 + code (after a system-scope fence)
void launch_sync_signal(const SyncPeers& sp, int me, int phase, int code, cudaStream_t st);
// wait until every peer's flag `phase` in the local area >= epoch * 256 + code (code may be negative)
void launch_sync_wait(uint64_t* area, int EP, int me, int phase, int code, int* status, cudaStream_t st);
// the landed counts of this call [EP][C][E] -> counts_all; then, per chunk j, the fused-exchange table
// (see PeerTable's comment) into p2p_tab + j (4E+1), and gskip[j] = 1 if ANY rank's padded rows exceed
// rows_cap or its send rows exceed send_cap (identical on every rank: the same counts)
void launch_p2p_tables(const uint64_t* area, int C, int E, int El, int EP, int me, int64_t rows_cap,
                       int64_t send_cap, int* counts_all, int* p2p_tab, int* gskip, int* status, cudaStream_t st);

// ---------------------------------------------------------------- router (N3)
template <typename T>
void launch_router_fwd(const T* x, const T* wr, int64_t ntok, int E, int h, int k, float* logits, int32_t* ids,
                       float* scores, cudaStream_t st);
// m: a counting sort of ids by expert (dispatch_hist/scan/index with ep_size 1): seg, recv_cnt, src_of
template <typename T>
void launch_router_bwd(const T* x, const T* wr, const int32_t* ids, const float* scores, const float* dscore,
                       int64_t ntok, int E, int h, int k, float* dlog, T* dx, int acc_dx, float* dwr, int acc_dw,
                       const ChunkMeta& m, cudaStream_t st);
// bf16: the logits GEMM (x W_r^T, fp32 out) and the dW_r GEMMs (d_logits^T x over the hi and lo halves) run
// on the expert-GEMM kernels (GK_DOWN with out_f32, GK_WGRAD_DOWN); these are the row kernels around them.
void launch_router_topk(const float* logits, int64_t ld, int64_t ntok, int E, int k, int32_t* ids, float* scores,
                        float* out, cudaStream_t st);
void launch_router_bwd_rows_bf16(const __nv_bfloat16* wr, const int32_t* ids, const float* scores, const float* dscore,
                                 int64_t ntok, int E, int h, int k, float* dlog, __nv_bfloat16* dhi,
                                 __nv_bfloat16* dlo, int ldd, __nv_bfloat16* dx, int acc_dx, cudaStream_t st);

// ---------------------------------------------------------------- MACT tuner (A3)
struct PlanParams {
  int32_t EP, nsub, E, h, g, D_t, nbins, rule;
  int32_t bins[16];
  uint64_t budget, static_bytes, other_bytes;
  int64_t m_g, tp, cp, micro_batch;
};
// Shared host/device evaluation from per-(rank, sub-chunk) sums sub[r*nsub + j].
__host__ __device__ int plan_from_subsums(const int64_t* sub, const PlanParams& p, memfine_plan_info* out);
// 0 = launched; -1 = launch failure (the result words are then not written)
int launch_plan_kernel(const int32_t* counts_dev, const PlanParams& p, memfine_plan_info* out_mapped,
                       int* rc_mapped, cudaStream_t st);

// ---------------------------------------------------------------- expert GEMMs (A7, A8, B2-B5)
enum GemmKind {
  GK_GATEUP = 0,      // A7/B2: [R,h] x W_gate/W_up^T -> a = silu(G)*U (fwd) and/or G||U (bwd)
  GK_DOWN = 1,        // A8:    [R,g] x W_down^T -> o
  GK_DACT = 2,        // B3:    dY [R,h] x W_down -> u; epilogue d_w, dG, dU, a_w
  GK_DX = 3,          // B4:    dGU [R,2g] x [W_gate; W_up] -> dX_disp
  GK_WGRAD_DOWN = 4,  // B5:    dW_down[e] += dY^T a_w
  GK_WGRAD_GU = 5     // B5:    dW_gate[e] || dW_up[e] += dGU^T X
};

// One MXFP8 operand: E4M3 codes (K-major rows) and its scale-factor chunks.
struct MxOp {
  const uint8_t* q;
  const uint8_t* sf;
};

template <typename T>
struct GemmProblem {
  int kind;
  int El, h, g;
  int64_t rows_cap;
  const int* seg;    // [El+1]
  const int* pseg;   // [El+1]  pair prefix
  const int* info;   // chunk info words
  const T* X;        // X_disp [R][h]
  const T* DY;       // dY_disp [R][h]
  T* GU;             // [R][2g]   G||U (recompute), overwritten by dG||dU
  T* A;              // [R][g]    a (fwd) / a_w (bwd)
  T* O;              // [R][h]    o (fwd) / dX_disp (bwd)
  const T* Wg;       // [El][g][h]
  const T* Wu;       // [El][g][h]
  const T* Wd;       // [El][h][g]
  const float* w_row;
  float* dw_row;
  float* dWg;        // [El][g][h] fp32
  float* dWu;
  float* dWd;        // [El][h][g]
  int store_a;       // GATEUP: store a
  int store_gu;      // GATEUP: store G||U
  int wgrad_beta;    // WGRAD: 1 accumulate into dW, 0 overwrite (zero tiles for experts without rows)
  const uint64_t* row_addr;  // DOWN / DX (fused EP combine): per-row destination address in the
                             // source rank's send buffer (peer memory), 0 = padding; null = local O
  // MXFP8 variant (mx = 1, sm100 path only): E4M3 operands + E8M0 block scales (mx_sf_off layout)
  int mx;
  MxOp mx_a;                 // A operand: Xq (GATEUP), Aq (DOWN), DYq (DACT), dGUq (DX)
  MxOp mx_b0, mx_b1;         // B: W_gate / W_up rows (GATEUP), W_down rows (DOWN), W_down^T (DACT),
                             //    W_gate^T / W_up^T (DX; K split at g)
  uint8_t* mx_aq;            // GATEUP forward output: a quantised (codes [R][g]) ...
  uint8_t* mx_aq_sf;         // ... and its block scales
  uint8_t* mx_gq;            // DACT (BF16) in the MX variant: dG||dU also quantised ([R][2g]) ...
  uint8_t* mx_gq_sf;         // ... with scales (non-null = on)
  int sm_limit;              // > 0: launch on at most this many SMs (MEMFINE_FLAG_OVERLAP comm reserve)
  int pace;                  // 1: no other kernel shares the SMs (EP = 1, one stream): wave pacing is safe
  // the router's GEMMs on the same kernels (N3): logits = x W_r^T as a DOWN launch storing fp32, and
  // dW_r = d_logits^T x as a WGRAD_DOWN launch (0 = off / defaults)
  int out_f32;               // DOWN: O is fp32 [rows][ld_out] (columns >= h clipped)
  int64_t ld_out;            // DOWN out_f32: O's row stride in elements (default h)
  int64_t ld_a;              // WGRAD_DOWN: DY's row stride in elements (default h)
  int64_t rows_in;           // rows present in the row-major operands (TMA zero-fills rows up to the
                             // 128-padded K / M loops; default rows_cap)
};

// CUDA-core FFMA path (MEMFINE_FP32 mode; K12 of SURVEY §2.4).
template <typename T>
int launch_gemm_simt(const GemmProblem<T>& p, cudaStream_t st);
// tcgen05 / TMEM / TMA path (MEMFINE_BF16).  Returns number of launches or <0 on error.
int launch_gemm_sm100(const GemmProblem<__nv_bfloat16>& p, cudaStream_t st);
int sm100_num_sms();
// One kernel of each translation unit (each .cu registers its own module): memfine.cu's preload finds the
// module of each and loads every function in it (lazy loading vs spinning inter-rank waits).
const void* kernel_anchor_route();
const void* kernel_anchor_mx();
const void* kernel_anchor_router();
const void* kernel_anchor_simt();
const void* kernel_anchor_sm100();

// ---------------------------------------------------------------- MXFP8 quantisation (mx.cu)
// info != null: rows = the chunk's padded rows (0 if skipped), capped at rows_max; else rows_max.
// Rows and K multiples of 128 (scale chunks).
void launch_mx_quant_rows(const __nv_bfloat16* src, int64_t ld, int64_t rows_max, const int* info, int K,
                          uint8_t* q, uint8_t* sf, cudaStream_t st);
// columnwise (R28c): per tensor, src [rows][Cc] (ld; rows = info's padded rows) -> q_t [Cc][Rcap]
// blocked along the rows, with scales; up to 4 tensors in one launch
struct MxColTensor {
  const __nv_bfloat16* src;
  int64_t ld;
  int Cc;
  uint8_t* q_t;
  uint8_t* sf_t;
};
struct MxColTensors {
  MxColTensor t[4];
  int n;
  int tile0[5];   // set by launch_mx_quant_t: first 128-column tile of each tensor in the flat grid
};
void launch_mx_quant_t(const MxColTensors& tz, const int* info, int64_t Rcap, cudaStream_t st);
// src [B][R][Cc] -> q_rows [B][R][Cc] blocked along Cc and q_t [B][Cc][R] blocked along R, one read
void launch_mx_quant_dual(const __nv_bfloat16* src, int B, int R, int Cc, uint8_t* q_rows, uint8_t* sf_rows,
                          uint8_t* q_t, uint8_t* sf_t, cudaStream_t st);


}  // namespace memfine
