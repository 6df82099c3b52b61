// memfine.cu — the C ABI of libmemfine.so: handle, MACT plan, workspace carving and the
// FCDA chunk loops (Eq. 6 forward, Eq. 7 recompute backward).
#include <nvtx3/nvToolsExt.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>
#include <string>
#include <algorithm>
#include <type_traits>
#include <mutex>
#include <condition_variable>
#include <array>

#include "kernels.h"
#include <cuda.h>
#include <cudaTypedefs.h>
#include "nccl_shim.h"

using namespace memfine;

// In-process EP group (memfine_local_group_create): a host barrier plus per-rank events and
// published buffer pointers; exchanges are pull-based device copies.
struct memfine_group_s {
  int n = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0, gen = 0;
  std::vector<cudaEvent_t> ready, done;
  std::vector<std::array<char*, 20>> ptrs;  // per rank: buffers of the current call ([slot*8 + kind];
                                            // kPtrWs: workspace, kPtrSync: P2P sync area)
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    int g = gen;
    if (++arrived == n) {
      arrived = 0;
      gen++;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

struct memfine_handle_s;
memfine_status register_local(memfine_handle_s* h, void* ws, uint64_t ws_bytes);

struct memfine_handle_s {
  memfine_dims d;
  memfine_group_s* lg = nullptr;   // in-process EP group (instead of NCCL)
  int p2p = 0;                     // fused exchange over peer memory (MEMFINE_EP_P2P)
  int ipc_only = 0;                // memfine_create_ipc: no NCCL; mappings via memfine_ipc_export / _import
  void* exp_ws = nullptr;          // memfine_ipc_export: the exported workspace
  uint64_t exp_bytes = 0;
  // P2P (N1, device-planned): the registered workspace and sync area of every rank (own entries local;
  // in-process peers directly, other processes through CUDA IPC), the all-gathered counts and the
  // per-chunk global skip flags
  void* reg_ws = nullptr;
  uint64_t reg_bytes = 0;
  std::vector<char*> peer_ws;      // [EP] (own entry = reg_ws)
  std::vector<uint64_t*> peer_sync;// [EP] (own entry = sync_d)
  uint64_t* sync_d = nullptr;      // this rank's sync area (sync_area_bytes)
  int* gskip_d = nullptr;          // [kMaxSub]
  std::vector<void*> ipc_bases;    // opened peer allocation bases (to close)
  // MXFP8: the bound quantised weights (memfine_mx_quantize_weights)
  const uint8_t* mx_w = nullptr;
  // router scratch (lazily allocated): logits, d_logits, counting sort of ids by expert
  char* router_scratch = nullptr;
  size_t router_bytes = 0;
  int device = 0;
  int num_sms = 148;
  int* status_h = nullptr;     // pinned, mapped: device-latched error word
  int* status_d = nullptr;
  int64_t* rows_h = nullptr;   // pinned, mapped: [2][kMaxSub] rows / padded rows per chunk
  int64_t* rows_d = nullptr;
  memfine_stats last{};
  uint64_t last_meta = 0, last_row_bytes = 0;
  int debug = 0;
  std::vector<std::vector<int64_t>> debug_perm;
  // debug (EP = 1): per chunk of the last call, the expert-major rows' copy indices and the MXFP8
  // decisions (codes + scale chunks) of the operands the kernels quantise (memfine_debug_mx)
  struct DbgMx { std::vector<uint8_t> q, sf; int64_t rows = 0, cols = 0; };
  std::vector<std::array<DbgMx, 6>> dbg_mx;
  std::vector<std::vector<int32_t>> dbg_src;
  // expert parallel
  NcclComm comm{};
  int* counts_d = nullptr;     // [EP][C][E] all-gathered chunk counts (device)
  int* counts_h = nullptr;     // pinned mirror
  size_t counts_cap = 0;
  cudaEvent_t ev = nullptr;
  // MEMFINE_FLAG_OVERLAP: the comm stream (highest priority) and its fork/join events
  cudaStream_t cs = nullptr;
  cudaEvent_t ev_disp[2] = {nullptr, nullptr}, ev_gemm[2] = {nullptr, nullptr};
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int comm_sms = 0;
  // measurement (memfine_profile_enable)
  int prof = 0;
  struct Rec { int slot; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  size_t pool_used = 0;
  int open_slot = -1;
  cudaEvent_t open_ev = nullptr;
};

namespace {
// NVTX ranges (no-ops unless a tool injects NVTX): one per layer call and one per FCDA chunk, so ncu
// `--nvtx --nvtx-include` / a timeline tool can select e.g. the backward of chunk 3.
struct Nvtx {
  explicit Nvtx(const char* s) { nvtxRangePushA(s); }
  ~Nvtx() { nvtxRangePop(); }
};
const char* chunk_range_name(int pass, int j) {
  static char names[2][64][24];
  static bool init = false;
  if (!init) {
    for (int p = 0; p < 2; p++)
      for (int c = 0; c < 64; c++) snprintf(names[p][c], sizeof names[p][c], "%s chunk %d", p ? "bwd" : "fwd", c);
    init = true;
  }
  return names[pass ? 1 : 0][j & 63];
}

cudaEvent_t pool_event(memfine_handle_s* h) {
  if (h->pool_used == h->pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    h->pool.push_back(e);
  }
  return h->pool[h->pool_used++];
}
// Bracket a launch (or a group of launches) of class `slot` with events on stream st.
void prof_begin(memfine_handle_s* h, int slot, cudaStream_t st) {
  if (!h->prof) return;
  h->open_slot = slot;
  h->open_ev = pool_event(h);
  cudaEventRecord(h->open_ev, st);
}
void prof_end(memfine_handle_s* h, cudaStream_t st) {
  if (!h->prof || h->open_slot < 0) return;
  cudaEvent_t b = pool_event(h);
  cudaEventRecord(b, st);
  h->recs.push_back({h->open_slot, h->open_ev, b});
  h->open_slot = -1;
}
}  // namespace

namespace {

bool dims_ok(const memfine_dims* d) {
  if (!d) return false;
  if (d->tokens < 0 || d->tokens > (int64_t(1) << 31) / 64) return false;
  if (d->hidden <= 0 || d->hidden % 64 || d->ffn <= 0 || d->ffn % 64) return false;
  if (d->num_experts < 1 || d->topk < 1 || d->topk > d->num_experts || d->topk > 16) return false;
  if (d->ep_size < 1 || d->num_experts % d->ep_size || d->ep_rank < 0 || d->ep_rank >= d->ep_size) return false;
  if (d->num_experts > 1024) return false;
  if (d->dtype != MEMFINE_BF16 && d->dtype != MEMFINE_FP32 && d->dtype != MEMFINE_MXFP8) return false;
  if (d->dtype == MEMFINE_MXFP8 && (d->hidden % 128 || d->ffn % 128)) return false;
  if (d->flags & ~(MEMFINE_FLAG_OVERLAP | MEMFINE_FLAG_EP_PATH | MEMFINE_FLAG_MX_WGRAD)) return false;
  if ((d->flags & MEMFINE_FLAG_EP_PATH) && d->ep_size != 1) return false;
  if ((d->flags & MEMFINE_FLAG_MX_WGRAD) && d->dtype != MEMFINE_MXFP8) return false;
  return true;
}

// The expert-parallel data path runs for ep_size > 1, or at ep_size == 1 over a 1-rank NCCL
// communicator with MEMFINE_FLAG_EP_PATH (the NCCL transport exercised on one GPU).
bool ep_path(const memfine_dims& d) { return d.ep_size > 1 || (d.flags & MEMFINE_FLAG_EP_PATH); }

int elt_bytes(const memfine_dims& d) { return d.dtype == MEMFINE_FP32 ? 4 : 2; }  // MXFP8: bf16 storage

// ------------------------------------------------------------------ workspace carving
// One bump allocator (256-byte aligned) defines the layout; the byte count it reaches is
// the predicted high-water (memfine_workspace_bytes) and the carve used by fwd/bwd.
struct Bump {
  char* base;
  uint64_t off = 0;
  explicit Bump(void* b) : base((char*)b) {}
  template <typename T>
  T* take(uint64_t n) {
    off = (off + 255) & ~uint64_t(255);
    T* p = base ? (T*)(base + off) : nullptr;
    off += n * sizeof(T);
    return p;
  }
};

struct Layout {
  ChunkMeta m{};
  void* X = nullptr;   // [R][h]
  void* DY = nullptr;  // [R][h]   (bwd)
  void* GU = nullptr;  // [R][2g]  (bwd)
  void* A = nullptr;   // [R][g]
  void* O = nullptr;   // [R][h]   (fwd: o; bwd: dX_disp aliases X)
  void* send = nullptr;      // [S][h]   EP>1 staging (x out / o back)
  void* send_dy = nullptr;   // [S][h]   EP>1 bwd
  float* send_w = nullptr;   // [S]      EP>1 scores out / d_score back
  // MXFP8 operands (E4M3 codes + scale chunks): X, a (fwd) / X, dG||dU (bwd)
  uint8_t *Xq = nullptr, *Xsf = nullptr, *Aq = nullptr, *Asf = nullptr;
  uint8_t *GUq = nullptr, *GUsf = nullptr;
  uint8_t *DYt = nullptr, *DYtsf = nullptr, *GUt = nullptr, *GUtsf = nullptr, *At = nullptr, *Atsf = nullptr;
  int64_t rows_cap = 0;
  uint64_t meta_bytes = 0, row_bytes = 0, total = 0;
  bool o_alias = false;   // O is carved over X (by layout, not by address: zero-row arrays share one)
};

// MEMFINE_FLAG_OVERLAP: two slots of the exchanged rows (chunk j+1 lands while chunk j computes).
int ep_slots(const memfine_dims& d, int C) {
  return (d.flags & MEMFINE_FLAG_OVERLAP) && ep_path(d) && C > 1 && d.dtype != MEMFINE_MXFP8 ? 2 : 1;
}

uint64_t row_bytes_of(const memfine_dims& d, int pass, int slots = 1) {
  uint64_t D = elt_bytes(d), h = d.hidden, g = d.ffn;
  uint64_t ep = ep_path(d) ? 16 : 0;                               // row_addr, row_addr_w (EP>1)
  if (d.dtype == MEMFINE_MXFP8) {
    // fwd: x gathered straight to Xq + scales, a straight to Aq + scales, O (bf16)
    if (pass == MEMFINE_FWD) return ep + 8 + (h + h / 32) + (g + g / 32) + D * h;
    // bwd: bf16 X, dY, G||U, a_w (dA stays BF16) + Xq, dGUq with scales; O aliases X.  MX_WGRAD:
    // + the columnwise codes of dY, dG || dU and a_w (x's reuse Xq, dead after the recompute)
    const uint64_t wg = (d.flags & MEMFINE_FLAG_MX_WGRAD) ? (h + h / 32) + (3 * g + 3 * g / 32) : 0;
    return ep + 12 + D * (h + h + 2 * g + g) + (h + h / 32) + (2 * g + 2 * g / 32) + wg;
  }
  if (slots == 2) {
    // per slot: src_of, w_row, row addresses, (bwd: dw_row, dY_disp), X_disp (o / dX_disp written
    // over it); shared: a (fwd) / G||U + a_w (bwd)
    if (pass == MEMFINE_FWD) return 2 * (ep + 8 + D * h) + D * g;
    return 2 * (ep + 12 + D * 2 * h) + D * 3 * g;
  }
  if (pass == MEMFINE_FWD) return ep + 4 + 4 + D * (h + g + h);   // src_of, w_row, X, A, O
  return ep + 4 + 4 + 4 + D * (h + h + 2 * g + g);                 // + dw_row, DY, GU; O aliases X
}

int64_t tmax_chunk(const memfine_dims& d, int C) { return ceil_div64(d.tokens, C); }

// Carve: metadata, optional EP send staging (send_rows), then rows_cap rows.  With two slots
// (ep_slots) the metadata + staging and the exchanged row arrays are carved twice; slot s is
// returned in L2[s] (L2 may be null when slots == 1).  The returned Layout is slot 0 and carries
// the totals.
Layout carve(const memfine_dims& d, int C, int pass, void* ws, int64_t rows_cap, int64_t send_rows,
             Layout* L2 = nullptr) {
  const int S = ep_slots(d, C);
  Layout Ls[2];
  Bump b(ws);
  int E = d.num_experts, El = E / d.ep_size;
  int64_t Tm = tmax_chunk(d, C);
  int64_t NB = ceil_div64(Tm, kTokPerBlk);
  uint64_t D = elt_bytes(d);
  for (int s = 0; s < S; s++) {
    Layout& L = Ls[s];
    L.m.blk_cnt = b.take<int>((uint64_t)NB * E);
    L.m.exp_cnt = b.take<int>(E);
    L.m.recv_cnt = b.take<int>(El);
    L.m.seg = b.take<int>(El + 1);
    L.m.pseg = b.take<int>(El + 1);
    L.m.info = b.take<int>(kInfoWords);
    L.m.dest_of = b.take<int>((uint64_t)Tm * d.topk);
    if (ep_path(d)) {
      L.m.send_src = b.take<int>((uint64_t)Tm * d.topk);
      L.m.p2p_tab = b.take<int>((uint64_t)C * (4 * (uint64_t)E + 1));
      L.send = b.take<char>((uint64_t)send_rows * d.hidden * D);
      if (pass == MEMFINE_BWD) L.send_dy = b.take<char>((uint64_t)send_rows * d.hidden * D);
      L.send_w = b.take<float>((uint64_t)send_rows);
    }
  }
  b.off = (b.off + 255) & ~uint64_t(255);
  const uint64_t meta_bytes = b.off;
  int64_t R = rows_cap;
  if (S == 2) {
    for (int s = 0; s < 2; s++) {
      Layout& L = Ls[s];
      L.m.src_of = b.take<int>(R);
      L.m.w_row = b.take<float>(R);
      L.m.row_addr = b.take<uint64_t>(R);
      L.m.row_addr_w = b.take<uint64_t>(R);
      if (pass == MEMFINE_BWD) {
        L.m.dw_row = b.take<float>(R);
        L.DY = b.take<char>((uint64_t)R * d.hidden * D);
      }
      L.X = b.take<char>((uint64_t)R * d.hidden * D);
      L.O = L.X;
      L.o_alias = true;
    }
    void* GU = pass == MEMFINE_BWD ? b.take<char>((uint64_t)R * 2 * d.ffn * D) : nullptr;
    void* A = b.take<char>((uint64_t)R * d.ffn * D);
    for (int s = 0; s < 2; s++) {
      Ls[s].GU = GU;
      Ls[s].A = A;
    }
  } else {
    Layout& L = Ls[0];
    L.m.src_of = b.take<int>(R);
    L.m.w_row = b.take<float>(R);
    if (ep_path(d)) {
      L.m.row_addr = b.take<uint64_t>(R);
      L.m.row_addr_w = b.take<uint64_t>(R);
    }
    if (pass == MEMFINE_BWD) L.m.dw_row = b.take<float>(R);
    // (the MX forward at EP = 1 keeps no bf16 copy of the dispatched rows: the gather writes E4M3
    // only; on the EP path X_disp receives the bf16 rows and o is later written over it)
    if (!(d.dtype == MEMFINE_MXFP8 && pass == MEMFINE_FWD) || ep_path(d))
      L.X = b.take<char>((uint64_t)R * d.hidden * D);
    if (d.dtype == MEMFINE_MXFP8) {
      const uint64_t hh = d.hidden, gg = d.ffn;
      L.Xq = b.take<uint8_t>((uint64_t)R * hh);
      L.Xsf = b.take<uint8_t>((uint64_t)R * hh / 32);
      if (pass == MEMFINE_BWD) {
        L.DY = b.take<char>((uint64_t)R * hh * D);
        L.GU = b.take<char>((uint64_t)R * 2 * gg * D);
        L.A = b.take<char>((uint64_t)R * gg * D);
        L.GUq = b.take<uint8_t>((uint64_t)R * 2 * gg);
        L.GUsf = b.take<uint8_t>((uint64_t)R * 2 * gg / 32);
        if (d.flags & MEMFINE_FLAG_MX_WGRAD) {   // columnwise codes [cols][R] (reading R28c)
          L.DYt = b.take<uint8_t>((uint64_t)R * hh);
          L.DYtsf = b.take<uint8_t>((uint64_t)R * hh / 32);
          L.GUt = b.take<uint8_t>((uint64_t)R * 2 * gg);
          L.GUtsf = b.take<uint8_t>((uint64_t)R * 2 * gg / 32);
          L.At = b.take<uint8_t>((uint64_t)R * gg);
          L.Atsf = b.take<uint8_t>((uint64_t)R * gg / 32);
        }
        L.O = L.X;
        L.o_alias = true;
      } else {
        L.Aq = b.take<uint8_t>((uint64_t)R * gg);
        L.Asf = b.take<uint8_t>((uint64_t)R * gg / 32);
        L.o_alias = ep_path(d);
        L.O = ep_path(d) ? L.X : b.take<char>((uint64_t)R * hh * D);
      }
    } else if (pass == MEMFINE_BWD) {
      L.DY = b.take<char>((uint64_t)R * d.hidden * D);
      L.GU = b.take<char>((uint64_t)R * 2 * d.ffn * D);
      L.A = b.take<char>((uint64_t)R * d.ffn * D);
      L.O = L.X;
      L.o_alias = true;
    } else {
      L.A = b.take<char>((uint64_t)R * d.ffn * D);
      L.O = b.take<char>((uint64_t)R * d.hidden * D);
    }
  }
  b.off = (b.off + 255) & ~uint64_t(255);
  for (int s = 0; s < S; s++) {
    Ls[s].meta_bytes = meta_bytes;
    Ls[s].row_bytes = row_bytes_of(d, pass, S);
    Ls[s].rows_cap = rows_cap;
    Ls[s].total = b.off;
  }
  if (L2) {
    L2[0] = Ls[0];
    L2[1] = Ls[S - 1];
  }
  return Ls[0];
}

// rows_cap that fits ws_bytes (multiple of 128; each row array then stays 256-aligned).
int64_t rows_fitting(const memfine_dims& d, int C, int pass, uint64_t ws_bytes, int64_t send_rows) {
  Layout L0 = carve(d, C, pass, nullptr, 0, send_rows);
  if (ws_bytes < L0.meta_bytes) return -1;
  int64_t R = (int64_t)((ws_bytes - L0.meta_bytes) / L0.row_bytes);
  R = (R / kRowAlign) * kRowAlign;
  while (R > 0 && carve(d, C, pass, nullptr, R, send_rows).total > ws_bytes) R -= kRowAlign;
  return R;
}

// Padded rows per chunk on rank r from host counts [EP][nsub][E] (C | nsub).
void chunk_rows(const int32_t* counts, int nsub, const memfine_dims& d, int C, int r, std::vector<int64_t>& rows,
                std::vector<int64_t>& rows_pad, std::vector<int64_t>* send) {
  int E = d.num_experts, El = E / d.ep_size, per = nsub / C;
  rows.assign(C, 0);
  rows_pad.assign(C, 0);
  if (send) send->assign(C, 0);
  for (int jc = 0; jc < C; jc++) {
    for (int e = r * El; e < (r + 1) * El; e++) {
      int64_t c = 0;
      for (int src = 0; src < d.ep_size; src++)
        for (int j = jc * per; j < (jc + 1) * per; j++) c += counts[((int64_t)src * nsub + j) * E + e];
      rows[jc] += c;
      rows_pad[jc] += round_up64(c, kRowAlign);
    }
    if (send)
      for (int e = 0; e < E; e++)
        for (int j = jc * per; j < (jc + 1) * per; j++) (*send)[jc] += counts[((int64_t)r * nsub + j) * E + e];
  }
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int budget_to_params(const memfine_dims* d, const memfine_budget* b, int nsub, PlanParams* p) {
  static const int32_t kDefaultBins[4] = {1, 2, 4, 8};
  if (!dims_ok(d) || !b || nsub < 1 || nsub > kMaxSub) return MEMFINE_ERR_INVALID_ARG;
  const int32_t* bins = b->bins ? b->bins : kDefaultBins;
  int nb = b->bins ? b->nbins : 4;
  if (nb < 1 || nb > 16) return MEMFINE_ERR_INVALID_ARG;
  for (int i = 0; i < nb; i++) {
    if (bins[i] < 1) return MEMFINE_ERR_INVALID_ARG;
    if (i && bins[i] <= bins[i - 1]) return MEMFINE_ERR_INVALID_ARG;
    p->bins[i] = bins[i];
  }
  if (!(b->alpha > 0.0) || !std::isfinite(b->alpha)) return MEMFINE_ERR_INVALID_ARG;
  if (b->m_g < 1 || b->tp < 1 || b->cp < 1 || b->micro_batch < 1) return MEMFINE_ERR_INVALID_ARG;
  if (b->rule != MEMFINE_RULE_EQ9 && b->rule != MEMFINE_RULE_EXACT) return MEMFINE_ERR_INVALID_ARG;
  if (b->model != MEMFINE_MODEL_PAPER && b->model != MEMFINE_MODEL_IMPL) return MEMFINE_ERR_INVALID_ARG;
  if (b->pass != MEMFINE_FWD && b->pass != MEMFINE_BWD) return MEMFINE_ERR_INVALID_ARG;
  long double B = (long double)b->alpha * (long double)b->gpu_capacity_bytes;
  if (B >= 18446744073709551615.0L) B = 18446744073709551615.0L;
  p->budget = (uint64_t)floorl(B);
  p->EP = d->ep_size;
  p->nsub = nsub;
  p->E = d->num_experts;
  p->h = d->hidden;
  p->g = d->ffn;
  p->D_t = elt_bytes(*d);
  p->nbins = nb;
  p->rule = b->rule;
  p->static_bytes = b->static_bytes;
  p->other_bytes = b->other_act_bytes;
  p->m_g = b->m_g;
  p->tp = b->tp;
  p->cp = b->cp;
  p->micro_batch = b->micro_batch;
  return MEMFINE_OK;
}

template <typename T>
GemmProblem<T> base_problem(const memfine_handle_s* h, const Layout& L, const void* wg, const void* wu,
                            const void* wd) {
  GemmProblem<T> p{};
  p.El = h->d.num_experts / h->d.ep_size;
  p.h = h->d.hidden;
  p.g = h->d.ffn;
  p.rows_cap = L.rows_cap;
  p.seg = L.m.seg;
  p.pseg = L.m.pseg;
  p.info = L.m.info;
  p.X = (const T*)L.X;
  p.DY = (const T*)L.DY;
  p.GU = (T*)L.GU;
  p.A = (T*)L.A;
  p.O = (T*)L.O;
  p.Wg = (const T*)wg;
  p.Wu = (const T*)wu;
  p.Wd = (const T*)wd;
  p.w_row = L.m.w_row;
  p.dw_row = L.m.dw_row;
  // wave pacing of the persistent GEMM units needs every unit resident: not when GEMMs of other
  // ranks (in-process group) or comm kernels (EP path) may hold SMs concurrently
  p.pace = (h->d.ep_size == 1 && !(h->d.flags & MEMFINE_FLAG_EP_PATH) && !h->lg) ? 1 : 0;
  return p;
}

bool bf16_use_simt() {
  const char* s = getenv("MEMFINE_BF16_GEMM");
  return s && !strcmp(s, "simt");
}

template <typename T>
int run_gemm(memfine_handle_s* h, const GemmProblem<T>& p, cudaStream_t st) {
  int n;
  prof_begin(h, p.kind, st);
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    if (bf16_use_simt()) n = launch_gemm_simt<T>(p, st);
    else n = launch_gemm_sm100(p, st);
  } else {
    n = launch_gemm_simt<T>(p, st);
  }
  prof_end(h, st);
  if (n < 0) return MEMFINE_ERR_UNSUPPORTED;
  h->last.gemm_launches += n;
  h->last.kernel_launches += n;
  return MEMFINE_OK;
}

memfine_status latch_cuda(memfine_handle_s* h) {
  (void)h;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MEMFINE_OK : MEMFINE_ERR_CUDA;
}

// ------------------------------------------------------------------ MXFP8 weights (N4, reading R28)
// Five E4M3 operands of E_l*g*h codes each, then their scale chunks (E_l*g*h/32 each), 256-aligned:
//   0 W_gate rows (K = h)  1 W_up rows (K = h)  2 W_down rows (K = g)
//   3 W_gate^T [E_l][h][g] (K = g, dX)   4 W_up^T (K = g, dX)
constexpr int kMxW = 5;
struct MxWeightsLayout {
  MxOp op[kMxW];
  uint64_t total = 0;
};
MxWeightsLayout mx_weights_layout(const memfine_dims& d, const void* base) {
  MxWeightsLayout W;
  Bump b(const_cast<void*>(base));
  const uint64_t n = (uint64_t)(d.num_experts / d.ep_size) * d.hidden * d.ffn;
  uint8_t* q[kMxW];
  for (int i = 0; i < kMxW; i++) q[i] = b.take<uint8_t>(n);
  for (int i = 0; i < kMxW; i++) W.op[i] = {q[i], b.take<uint8_t>(n / 32)};
  b.off = (b.off + 255) & ~uint64_t(255);
  W.total = b.off;
  return W;
}

void set_mx(GemmProblem<__nv_bfloat16>& p, const MxOp& a, const MxOp& b0, const MxOp& b1) {
  p.mx = 1;
  p.mx_a = a;
  p.mx_b0 = b0;
  p.mx_b1 = b1;
}

// B5: the chunk's weight-gradient GEMMs (W_grad = sum over chunks, reading R18; p.wgrad_beta set by
// the caller).  MEMFINE_FLAG_MX_WGRAD (reading R28c): one launch writes the columnwise E4M3 codes of
// x (into Xq: dead after the recompute), dY, dG || dU and a_w, then block-scaled GEMMs over them.
template <typename T>
int run_wgrad(memfine_handle_s* h, GemmProblem<T>& p, const Layout& L, cudaStream_t st) {
  if (p.rows_cap == 0) {
    // No chunk of this call reaches this rank's experts (EP: every copy routed elsewhere).  The
    // GEMM launchers return early on an empty row buffer, so the first chunk's overwrite of dW
    // (beta = 0) is done here; later chunks add nothing.
    if (!p.wgrad_beta) {
      const memfine_dims& d = h->d;
      const size_t wb = sizeof(float) * (size_t)(d.num_experts / d.ep_size) * d.ffn * d.hidden;
      prof_begin(h, 8, st);
      float* dws[3] = {p.dWg, p.dWu, p.dWd};
      for (float* dw : dws)
        if (cudaMemsetAsync(dw, 0, wb, st) != cudaSuccess) return MEMFINE_ERR_CUDA;
      prof_end(h, st);
      h->last.kernel_launches += 3;
    }
    return MEMFINE_OK;
  }
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    const memfine_dims& d = h->d;
    if (d.dtype == MEMFINE_MXFP8 && (d.flags & MEMFINE_FLAG_MX_WGRAD)) {
      const int hd = d.hidden, g = d.ffn;
      prof_begin(h, 10, st);
      MxColTensors tz{};
      tz.t[0] = {(const __nv_bfloat16*)L.X, hd, hd, L.Xq, L.Xsf};
      tz.t[1] = {(const __nv_bfloat16*)L.DY, hd, hd, L.DYt, L.DYtsf};
      tz.t[2] = {(const __nv_bfloat16*)L.GU, 2 * g, 2 * g, L.GUt, L.GUtsf};
      tz.t[3] = {(const __nv_bfloat16*)L.A, g, g, L.At, L.Atsf};
      tz.n = 4;
      launch_mx_quant_t(tz, L.m.info, L.rows_cap, st);
      prof_end(h, st);
      h->last.kernel_launches += 1;
      p.kind = GK_WGRAD_DOWN;
      set_mx(p, {L.DYt, L.DYtsf}, {L.At, L.Atsf}, {L.At, L.Atsf});
      if (int rc = run_gemm<T>(h, p, st)) return rc;
      p.kind = GK_WGRAD_GU;
      set_mx(p, {L.GUt, L.GUtsf}, {L.Xq, L.Xsf}, {L.Xq, L.Xsf});
      if (int rc = run_gemm<T>(h, p, st)) return rc;
      p.mx = 0;
      return 0;
    }
  }
  p.kind = GK_WGRAD_DOWN;
  if (int rc = run_gemm<T>(h, p, st)) return rc;
  p.kind = GK_WGRAD_GU;
  return run_gemm<T>(h, p, st);
}

// ------------------------------------------------------------------ debug capture (EP = 1)
// Synchronises and copies device state to the host; only with memfine_set_debug(1).
void dbg_rows(memfine_handle_s* h, int j, const int* src_of, cudaStream_t st) {
  cudaStreamSynchronize(st);
  if ((int)h->dbg_src.size() <= j) h->dbg_src.resize(j + 1);
  const int64_t rp = h->rows_h[kMaxSub + j];
  h->dbg_src[j].assign(rp > 0 ? rp : 0, -1);
  if (rp > 0) cudaMemcpy(h->dbg_src[j].data(), src_of, sizeof(int) * rp, cudaMemcpyDeviceToHost);
}
// which: 0 a [rows_pad][g], 1 dG||dU [rows_pad][2g] (rowwise); 2 x, 3 dY [h][Rcap], 4 dG||dU [2g][Rcap],
// 5 a_w [g][Rcap] (columnwise, reading R28c).  Scales in the tcgen05 chunk layout with K = cols.
void dbg_mx(memfine_handle_s* h, int j, int which, const uint8_t* q, const uint8_t* sf, int64_t rows, int64_t cols,
            cudaStream_t st) {
  cudaStreamSynchronize(st);
  if ((int)h->dbg_mx.size() <= j) h->dbg_mx.resize(j + 1);
  auto& D = h->dbg_mx[j][which];
  D.rows = rows;
  D.cols = cols;
  D.q.assign((size_t)(rows * cols), 0);
  D.sf.assign((size_t)(rows * cols / 32), 0);
  if (rows * cols > 0) {
    cudaMemcpy(D.q.data(), q, D.q.size(), cudaMemcpyDeviceToHost);
    cudaMemcpy(D.sf.data(), sf, D.sf.size(), cudaMemcpyDeviceToHost);
  }
}

// ------------------------------------------------------------------ the FCDA chunk loops (EP = 1)
template <typename T>
memfine_status fwd_ep1(memfine_handle_s* h, const T* x, const int32_t* ids, const float* w, const void* wg,
                       const void* wu, const void* wd, int C, T* y, void* ws, uint64_t ws_bytes, cudaStream_t st) {
  const memfine_dims& d = h->d;
  int64_t R = rows_fitting(d, C, MEMFINE_FWD, ws_bytes, 0);
  if (R < 0) return MEMFINE_ERR_WORKSPACE;
  Layout L = carve(d, C, MEMFINE_FWD, ws, R, 0);
  int E = d.num_experts, El = E, k = d.topk, hd = d.hidden;
  const bool mx = d.dtype == MEMFINE_MXFP8;
  if (mx && !h->mx_w) return MEMFINE_ERR_INVALID_ARG;   // memfine_mx_quantize_weights first
  MxWeightsLayout W = mx_weights_layout(d, h->mx_w);
  h->last_meta = L.meta_bytes;
  h->last_row_bytes = L.row_bytes;
  if (h->debug) h->debug_perm.assign(C, {});
  for (int j = 0; j < C; j++) {
    int64_t t0 = chunk_begin(d.tokens, C, j), t1 = chunk_begin(d.tokens, C, j + 1);
    if (t1 == t0) continue;
    Nvtx chunk_range(chunk_range_name(0, j));
    int NB = (int)ceil_div64(t1 - t0, kTokPerBlk);
    prof_begin(h, 6, st);
    launch_dispatch_hist(ids, t0, t1, k, E, L.m, h->status_d, st);
    launch_dispatch_scan(NB, E, El, 0, R, L.m, h->rows_d, h->rows_d + kMaxSub, j, st);
    // (MX: the gather writes x's E4M3 codes + scales only - the forward needs no bf16 copy)
    launch_dispatch_scatter<T>(x, nullptr, ids, w, t0, t1, k, E, hd, L.m, (T*)L.X, nullptr, El, true, R, st,
                               mx ? L.Xq : nullptr, mx ? L.Xsf : nullptr, !mx);
    prof_end(h, st);
    h->last.kernel_launches += 4;
    if (h->debug) {
      cudaStreamSynchronize(st);
      int rp = (int)h->rows_h[kMaxSub + j];
      std::vector<int> tmp(rp > 0 ? rp : 0);
      if (rp > 0) cudaMemcpy(tmp.data(), L.m.src_of, sizeof(int) * rp, cudaMemcpyDeviceToHost);
      for (int v : tmp)
        if (v >= 0) h->debug_perm[j].push_back(v);
    }
    GemmProblem<T> p = base_problem<T>(h, L, wg, wu, wd);
    p.kind = GK_GATEUP;
    p.store_a = 1;
    if constexpr (std::is_same<T, __nv_bfloat16>::value)
      if (mx) {
        set_mx(p, {L.Xq, L.Xsf}, W.op[0], W.op[1]);
        p.mx_aq = L.Aq;
        p.mx_aq_sf = L.Asf;
      }
    if (int rc = run_gemm<T>(h, p, st)) return (memfine_status)rc;
    if (h->debug) {
      dbg_rows(h, j, L.m.src_of, st);
      if (mx) dbg_mx(h, j, 0, L.Aq, L.Asf, h->rows_h[kMaxSub + j], d.ffn, st);
    }
    p.kind = GK_DOWN;
    if constexpr (std::is_same<T, __nv_bfloat16>::value)
      if (mx) set_mx(p, {L.Aq, L.Asf}, W.op[2], W.op[2]);
    if (int rc = run_gemm<T>(h, p, st)) return (memfine_status)rc;
    prof_begin(h, 7, st);
    launch_combine<T>((const T*)L.O, w, t0, t1, k, hd, L.m, y, st);
    prof_end(h, st);
    h->last.kernel_launches += 1;
  }
  return latch_cuda(h);
}

template <typename T>
memfine_status bwd_ep1(memfine_handle_s* h, const T* dy, const T* x, const int32_t* ids, const float* w,
                       const void* wg, const void* wu, const void* wd, int C, T* dx, float* dwg, float* dwu,
                       float* dwd, float* dscore, int accumulate, void* ws, uint64_t ws_bytes, cudaStream_t st) {
  const memfine_dims& d = h->d;
  int64_t R = rows_fitting(d, C, MEMFINE_BWD, ws_bytes, 0);
  if (R < 0) return MEMFINE_ERR_WORKSPACE;
  Layout L = carve(d, C, MEMFINE_BWD, ws, R, 0);
  int E = d.num_experts, El = E, k = d.topk, hd = d.hidden, g = d.ffn;
  const bool mx = d.dtype == MEMFINE_MXFP8;
  if (mx && !h->mx_w) return MEMFINE_ERR_INVALID_ARG;   // memfine_mx_quantize_weights first
  MxWeightsLayout W = mx_weights_layout(d, h->mx_w);
  h->last_meta = L.meta_bytes;
  h->last_row_bytes = L.row_bytes;
  // dW is overwritten by the first non-empty chunk's weight-gradient GEMMs (beta = 0) and
  // accumulated by the later ones; only a call with no tokens at all needs a memset.
  int beta = accumulate ? 1 : 0;
  prof_begin(h, 8, st);
  if (!accumulate && d.tokens == 0) {
    size_t wb = sizeof(float) * (size_t)El * g * hd;
    MF_CUDA_OK(cudaMemsetAsync(dwg, 0, wb, st));
    MF_CUDA_OK(cudaMemsetAsync(dwu, 0, wb, st));
    MF_CUDA_OK(cudaMemsetAsync(dwd, 0, wb, st));
  }
  if (dscore && d.tokens > 0) MF_CUDA_OK(cudaMemsetAsync(dscore, 0, sizeof(float) * d.tokens * k, st));
  prof_end(h, st);
  for (int j = 0; j < C; j++) {
    int64_t t0 = chunk_begin(d.tokens, C, j), t1 = chunk_begin(d.tokens, C, j + 1);
    if (t1 == t0) continue;
    Nvtx chunk_range(chunk_range_name(1, j));
    int NB = (int)ceil_div64(t1 - t0, kTokPerBlk);
    // B1: re-dispatch x and dy of the chunk (the recompute of Eq. 7 starts from X_j)
    prof_begin(h, 6, st);
    launch_dispatch_hist(ids, t0, t1, k, E, L.m, h->status_d, st);
    launch_dispatch_scan(NB, E, El, 0, R, L.m, h->rows_d, h->rows_d + kMaxSub, j, st);
    launch_dispatch_scatter<T>(x, dy, ids, w, t0, t1, k, E, hd, L.m, (T*)L.X, (T*)L.DY, El, true, R, st,
                               mx ? L.Xq : nullptr, mx ? L.Xsf : nullptr, true);
    prof_end(h, st);
    h->last.kernel_launches += 4;
    GemmProblem<T> p = base_problem<T>(h, L, wg, wu, wd);
    p.dWg = dwg;
    p.dWu = dwu;
    p.dWd = dwd;
    // B2: recompute G || U for this chunk only
    p.kind = GK_GATEUP;
    p.store_a = 0;
    p.store_gu = 1;
    if constexpr (std::is_same<T, __nv_bfloat16>::value)
      if (mx) set_mx(p, {L.Xq, L.Xsf}, W.op[0], W.op[1]);
    if (int rc = run_gemm<T>(h, p, st)) return (memfine_status)rc;
    // B3: u = dY W_down, fused d_w / dG / dU / a_w epilogue (BF16 operands in the MX variant too:
    // the GEMM is bound by its epilogue - reading R28)
    p.kind = GK_DACT;
    p.mx = 0;
    if (mx) {   // ... whose epilogue also writes dG || dU as E4M3 + scales for the dX GEMM
      p.mx_gq = L.GUq;
      p.mx_gq_sf = L.GUsf;
    }
    if (int rc = run_gemm<T>(h, p, st)) return (memfine_status)rc;
    p.mx_gq = nullptr;
    p.mx_gq_sf = nullptr;
    if (h->debug) {
      dbg_rows(h, j, L.m.src_of, st);
      if (mx) dbg_mx(h, j, 1, L.GUq, L.GUsf, h->rows_h[kMaxSub + j], 2 * (int64_t)g, st);
    }
    // B5: weight gradients accumulate across chunks (reading R18)
    p.wgrad_beta = beta;
    if (int rc = run_wgrad<T>(h, p, L, st)) return (memfine_status)rc;
    beta = 1;
    if (h->debug && mx && (d.flags & MEMFINE_FLAG_MX_WGRAD)) {
      dbg_mx(h, j, 2, L.Xq, L.Xsf, hd, L.rows_cap, st);
      dbg_mx(h, j, 3, L.DYt, L.DYtsf, hd, L.rows_cap, st);
      dbg_mx(h, j, 4, L.GUt, L.GUtsf, 2 * (int64_t)g, L.rows_cap, st);
      dbg_mx(h, j, 5, L.At, L.Atsf, g, L.rows_cap, st);
    }
    // B4: dX_disp = dG W_gate + dU W_up (overwrites X_disp, dead after B5)
    p.kind = GK_DX;
    if constexpr (std::is_same<T, __nv_bfloat16>::value)
      if (mx) set_mx(p, {L.GUq, L.GUsf}, W.op[3], W.op[4]);
    if (int rc = run_gemm<T>(h, p, st)) return (memfine_status)rc;
    // B7: dX_i = sum_slot dX_disp[pos], d_score
    prof_begin(h, 7, st);
    launch_unpermute_reduce<T>((const T*)L.O, t0, t1, k, hd, L.m, dx, dscore, st);
    prof_end(h, st);
    h->last.kernel_launches += 1;
  }
  return latch_cuda(h);
}

// ------------------------------------------------------------------ expert parallel (EP > 1)
// Per chunk: dispatch permute into the send layout (dest rank, local expert, token, slot),
// NCCL all-to-allv with one message per (peer, local expert) segment so rows land directly in
// the receiver's padded expert-major layout (local expert, src rank, token, slot; reading R3),
// expert GEMMs, and the reverse exchange back into the send layout for the combine.
struct EpChunk {
  std::vector<int64_t> send_off;  // [E+1] prefix of my chunk copies over global experts
  std::vector<int64_t> recv_off;  // [EP][El] row where src's rows of local expert el start
  std::vector<int64_t> recv_cnt;  // [EP][El]
  int64_t rows = 0, rows_pad = 0, send = 0;
};

EpChunk ep_chunk_table(const memfine_dims& d, const int* counts, int C, int j) {
  int E = d.num_experts, EP = d.ep_size, El = E / EP, me = d.ep_rank;
  EpChunk t;
  t.send_off.assign(E + 1, 0);
  for (int e = 0; e < E; e++) t.send_off[e + 1] = t.send_off[e] + counts[((int64_t)me * C + j) * E + e];
  t.send = t.send_off[E];
  t.recv_off.assign((size_t)EP * El, 0);
  t.recv_cnt.assign((size_t)EP * El, 0);
  int64_t acc = 0;
  for (int el = 0; el < El; el++) {
    int64_t run = acc;
    for (int src = 0; src < EP; src++) {
      int64_t c = counts[((int64_t)src * C + j) * E + me * El + el];
      t.recv_off[(size_t)src * El + el] = run;
      t.recv_cnt[(size_t)src * El + el] = c;
      run += c;
      t.rows += c;
    }
    acc += round_up64(run - acc, kRowAlign);
  }
  t.rows_pad = acc;
  return t;
}

// ---- in-process group transport
enum { kPtrSend = 0, kPtrSendDy = 1, kPtrSendW = 2, kPtrX = 3, kPtrDY = 4, kPtrO = 5, kPtrWRow = 6, kPtrDWRow = 7,
       kPtrWs = 16, kPtrSync = 17, kPtrWsBytes = 18 };

// all ranks' device work before this point is visible to every rank's stream after it
void local_fence(memfine_handle_s* h, cudaStream_t st, std::vector<cudaEvent_t>& evs) {
  memfine_group_s* g = h->lg;
  cudaEventRecord(evs[h->d.ep_rank], st);
  g->barrier();
  for (int r = 0; r < g->n; r++)
    if (r != h->d.ep_rank) cudaStreamWaitEvent(st, evs[r], 0);
}

EpChunk ep_chunk_table(const memfine_dims& d, const int* counts, int C, int j);

// Pull-based exchange.  forward: copy the rows peers send me (their send layout) into my
// expert-major buffer; reverse: copy the rows peers computed for my tokens (their expert-major
// buffer) into my send layout.  Both tables are derived from the shared counts.
int local_exchange(memfine_handle_s* h, const int* counts, int C, int j, bool forward, int kind_send,
                   int kind_expert, size_t row_bytes, cudaStream_t st) {
  memfine_group_s* g = h->lg;
  const memfine_dims& d = h->d;
  int E = d.num_experts, EP = d.ep_size, El = E / EP, me = d.ep_rank;
  local_fence(h, st, g->ready);
  EpChunk mine = ep_chunk_table(d, counts, C, j);
  for (int p = 0; p < EP; p++) {
    memfine_dims dp = d;
    dp.ep_rank = p;
    EpChunk theirs = ep_chunk_table(dp, counts, C, j);
    for (int el = 0; el < El; el++) {
      if (forward) {
        // p's copies for my expert (me, el) -> my rows recv_off[p][el]
        int eg = me * El + el;
        int64_t s0 = theirs.send_off[eg], n = theirs.send_off[eg + 1] - s0;
        if (!n) continue;
        char* src = g->ptrs[p][kind_send] + s0 * row_bytes;
        char* dst = g->ptrs[me][kind_expert] + mine.recv_off[(size_t)p * El + el] * row_bytes;
        if (cudaMemcpyAsync(dst, src, n * row_bytes, cudaMemcpyDeviceToDevice, st)) return 1;
        h->last.comm_ops++;
      } else {
        // rows p computed for my copies of its expert (p, el) -> my send layout
        int eg = p * El + el;
        int64_t s0 = mine.send_off[eg], n = mine.send_off[eg + 1] - s0;
        if (!n) continue;
        char* src = g->ptrs[p][kind_expert] + theirs.recv_off[(size_t)me * El + el] * row_bytes;
        char* dst = g->ptrs[me][kind_send] + s0 * row_bytes;
        if (cudaMemcpyAsync(dst, src, n * row_bytes, cudaMemcpyDeviceToDevice, st)) return 1;
        h->last.comm_ops++;
      }
    }
  }
  local_fence(h, st, g->done);  // nobody reuses a buffer until every rank's copies are done
  return 0;
}

// One grouped exchange.  forward=true: send-layout rows -> receiver's expert-major rows;
// forward=false: expert-major rows -> the source's send layout.  width = elements per row,
// esize = bytes per element (row payload moved as bytes; NCCL dtype uint8) or 4 for fp32 scalars.
// ks / ke: the buffers' kinds in the in-process group's pointer table (slot * 8 + kPtr*), passed
// explicitly - a zero-row rank's arrays share one address, so they cannot be looked up by pointer.
int ep_exchange(memfine_handle_s* h, const EpChunk& t, const int* counts, int C, int j, bool forward, char* send_buf,
                char* expert_buf, size_t row_bytes, cudaStream_t st, int ks, int ke) {
  const memfine_dims& d = h->d;
  int E = d.num_experts, EP = d.ep_size, El = E / EP, me = d.ep_rank;
  if (h->lg) return local_exchange(h, counts, C, j, forward, ks, ke, row_bytes, st);
  if (nccl_group_start()) return 1;
  int rc = 0;
  for (int peer = 0; peer < EP && !rc; peer++) {
    for (int el = 0; el < El && !rc; el++) {
      // my copies for expert (peer, el): contiguous in my send layout
      int eg = peer * El + el;
      int64_t s0 = t.send_off[eg], sn = t.send_off[eg + 1] - s0;
      // rows of src=peer for my local expert el in my expert-major buffer
      int64_t r0 = t.recv_off[(size_t)peer * El + el], rn = t.recv_cnt[(size_t)peer * El + el];
      if (peer == me && !(d.flags & MEMFINE_FLAG_EP_PATH)) {
        if (sn) {
          char* a = send_buf + s0 * row_bytes;
          char* b = expert_buf + r0 * row_bytes;
          if (cudaMemcpyAsync(forward ? b : a, forward ? a : b, sn * row_bytes, cudaMemcpyDeviceToDevice, st))
            rc = 1;
          h->last.comm_ops++;
        }
        continue;
      }
      if (forward) {
        if (sn) rc |= nccl_send(&h->comm, send_buf + s0 * row_bytes, sn * row_bytes, 0, peer, st);
        if (rn) rc |= nccl_recv(&h->comm, expert_buf + r0 * row_bytes, rn * row_bytes, 0, peer, st);
      } else {
        if (rn) rc |= nccl_send(&h->comm, expert_buf + r0 * row_bytes, rn * row_bytes, 0, peer, st);
        if (sn) rc |= nccl_recv(&h->comm, send_buf + s0 * row_bytes, sn * row_bytes, 0, peer, st);
      }
      h->last.comm_ops += (sn ? 1 : 0) + (rn ? 1 : 0);
    }
  }
  (void)counts; (void)C; (void)j;
  rc |= nccl_group_end();
  return rc;
}

// All-gathered per-chunk counts [EP][C][E] on device and host (the layer's one D2H sync).
int ep_gather_counts(memfine_handle_s* h, const int32_t* ids, int C, cudaStream_t st) {
  const memfine_dims& d = h->d;
  size_t need = (size_t)d.ep_size * C * d.num_experts;
  if (need > h->counts_cap) {
    if (h->counts_d) cudaFree(h->counts_d);
    if (h->counts_h) cudaFreeHost(h->counts_h);
    h->counts_d = nullptr;
    h->counts_h = nullptr;
    h->counts_cap = 0;
    if (cudaMalloc((void**)&h->counts_d, need * sizeof(int)) ||
        cudaHostAlloc((void**)&h->counts_h, need * sizeof(int), cudaHostAllocDefault))
      return MEMFINE_ERR_CUDA;
    h->counts_cap = need;
  }
  int* mine = h->counts_d + (int64_t)d.ep_rank * C * d.num_experts;
  launch_route_hist(ids, d.tokens, d.topk, d.num_experts, C, mine, h->status_d, st);
  if (h->lg) {
    h->lg->ptrs[d.ep_rank][0] = (char*)mine;
    local_fence(h, st, h->lg->ready);
    size_t nb = sizeof(int) * (size_t)C * d.num_experts;
    for (int r = 0; r < d.ep_size; r++)
      if (r != d.ep_rank)
        MF_CUDA_OK(cudaMemcpyAsync(h->counts_d + (int64_t)r * C * d.num_experts, h->lg->ptrs[r][0], nb,
                                   cudaMemcpyDeviceToDevice, st));
    local_fence(h, st, h->lg->done);
  } else if (nccl_all_gather_int(&h->comm, mine, h->counts_d, (size_t)C * d.num_experts, st)) {
    return MEMFINE_ERR_NCCL;
  }
  MF_CUDA_OK(cudaMemcpyAsync(h->counts_h, h->counts_d, need * sizeof(int), cudaMemcpyDeviceToHost, st));
  MF_CUDA_OK(cudaStreamSynchronize(st));
  if (*h->status_h) return __atomic_exchange_n(h->status_h, 0, __ATOMIC_SEQ_CST);
  return MEMFINE_OK;
}

// EP with the exchange fused into the kernels over peer memory, planned on the device:
// the count all-gather ("the first notification") is a push into every peer's sync area, the
// per-chunk tables and the capacity check come from a device kernel, and ranks fence with per-peer flags
// (epoch-stamped, spin-waited on the device) - the host never waits, so a call is graph-capturable.  The
// workspace layout does not depend on the counts: rows_cap follows from ws_bytes (as at EP = 1) and the send
// staging holds the chunk's T_j k copies, so every rank derives every peer's buffer addresses from the
// registered workspaces (all ranks register the same ws_bytes).  Per chunk j:
//   wait done(j-1) of every peer -> push rows into the receivers' expert-major buffers -> signal pushed(j),
//   wait pushed(j) -> GEMMs, whose down / dX epilogues store each output row into its source's send buffer
//   -> signal combined(j), wait combined(j) -> combine / unpermute -> signal done(j).
// A rank pushes chunk j+1 as soon as its receivers are done with chunk j, while it may still compute.
int ensure_comm_stream(memfine_handle_s* h);

template <typename T>
memfine_status ep_run_p2p(memfine_handle_s* h, int pass, const T* dy, const T* x, const int32_t* ids, const float* w,
                          const void* wg, const void* wu, const void* wd, int C, T* out, float* dwg, float* dwu,
                          float* dwd, float* dscore, int accumulate, void* ws, uint64_t ws_bytes, cudaStream_t st) {
  const memfine_dims& d = h->d;
  const int E = d.num_experts, EP = d.ep_size, El = E / EP, k = d.topk, hd = d.hidden, me = d.ep_rank;
  if (EP > kMaxPeers) return MEMFINE_ERR_UNSUPPORTED;
  const bool mx = d.dtype == MEMFINE_MXFP8;
  if (mx && !h->mx_w) return MEMFINE_ERR_INVALID_ARG;   // memfine_mx_quantize_weights first
  MxWeightsLayout W = mx_weights_layout(d, h->mx_w);
  if (ws != h->reg_ws || ws_bytes != h->reg_bytes || (int)h->peer_ws.size() != EP) {
    // in-process groups register on first use (every rank's call reaches the same point); across
    // processes memfine_register_workspace(ws, ws_bytes) (or memfine_ipc_import) must come first, on every rank
    if (!h->lg) return MEMFINE_ERR_INVALID_ARG;
    if (memfine_status rc = register_local(h, ws, ws_bytes)) return rc;
  }
  // MEMFINE_FLAG_OVERLAP (C > 1, not MXFP8): two workspace slots; chunk j's pushes (and j-1's combine) run on
  // the comm stream while chunk j-1's GEMMs run on the caller's stream
  const int S = ep_slots(d, C);
  const int64_t Srows = tmax_chunk(d, C) * k;
  const int64_t R = rows_fitting(d, C, pass, ws_bytes, Srows);
  if (R <= 0) return MEMFINE_ERR_WORKSPACE;
  Layout Ls[2];
  carve(d, C, pass, ws, R, Srows, Ls);
  h->last_meta = Ls[0].meta_bytes;
  h->last_row_bytes = Ls[0].row_bytes;
  PeerTable pt[2] = {};
  SyncPeers sp{};
  sp.n = EP;
  for (int r = 0; r < EP; r++) {
    memfine_dims dr = d;
    dr.ep_rank = r;
    Layout Lr[2];
    carve(dr, C, pass, h->peer_ws[r], R, Srows, Lr);   // the same offsets in every rank's workspace
    for (int sl = 0; sl < S; sl++) {
      pt[sl].n = EP;
      pt[sl].X[r] = (char*)Lr[sl].X;
      pt[sl].DY[r] = (char*)Lr[sl].DY;
      pt[sl].w_row[r] = (char*)Lr[sl].m.w_row;
      pt[sl].send[r] = (char*)Lr[sl].send;
      pt[sl].send_w[r] = pass == MEMFINE_BWD ? (char*)Lr[sl].send_w : nullptr;
    }
    sp.area[r] = h->peer_sync[r];
  }
  uint64_t* area = h->sync_d;
  // A1 + A2 on the device: this rank's per-chunk counts, pushed into every peer's landing zone
  launch_sync_epoch(area, st);
  int* mine = h->counts_d + (int64_t)me * C * E;
  launch_route_hist(ids, d.tokens, k, E, C, mine, h->status_d, st);
  launch_sync_push_counts(mine, C, E, sp, me, st);
  launch_sync_wait(area, EP, me, 0, 0, h->status_d, st);
  // A3's per-chunk split and offset tables (every chunk's, in slot 0's array), and the capacity check
  int* tabs = Ls[0].m.p2p_tab;
  launch_p2p_tables(area, C, E, El, EP, me, R, Srows, h->counts_d, tabs, h->gskip_d, h->status_d, st);
  h->last.kernel_launches += 6;
  int beta = accumulate ? 1 : 0;
  if (pass == MEMFINE_BWD && dscore && d.tokens > 0)
    MF_CUDA_OK(cudaMemsetAsync(dscore, 0, sizeof(float) * d.tokens * k, st));
  cudaStream_t cs = st;
  if (S == 2) {
    if (ensure_comm_stream(h)) return MEMFINE_ERR_CUDA;
    cs = h->cs;
    MF_CUDA_OK(cudaEventRecord(h->ev_fork, st));   // counts, tables, dscore zeroing
    MF_CUDA_OK(cudaStreamWaitEvent(cs, h->ev_fork, 0));
  }
  const int rb = hd * (int)sizeof(T);
  const size_t per = 4 * (size_t)E + 1;
  // Per chunk j (slot j % S), flags epoch-stamped with code j + 1:
  //   dispatch(j) [cs]: wait done(j - S) of every peer (their slot is free) -> push rows -> signal pushed(j),
  //                     wait pushed(j) -> padding, row addresses
  //   compute(j)  [st]: GEMMs, whose down / dX epilogues store each output row into its source's send buffer
  //                     -> signal combined(j)
  //   combine(j)  [cs]: wait combined(j) -> combine / unpermute -> signal done(j)
  // With one slot everything runs in that order on st; with two, cs issues dispatch(j+1) before combine(j).
  auto dispatch = [&](int j) -> memfine_status {
    const Layout& L = Ls[j % S];
    const int* tab_j = tabs + per * j;
    int64_t t0 = chunk_begin(d.tokens, C, j), t1 = chunk_begin(d.tokens, C, j + 1);
    int NB = (int)ceil_div64(t1 - t0, kTokPerBlk);
    if (NB) {
      launch_dispatch_hist(ids, t0, t1, k, E, L.m, h->status_d, cs);
      launch_dispatch_scan(NB, E, El, 1, L.rows_cap, L.m, nullptr, nullptr, j, cs);
      launch_dispatch_index(ids, w, t0, t1, k, E, L.m, L.m.send_src, nullptr, cs);
      h->last.kernel_launches += 3;
    }
    launch_ep_recv_seg(h->counts_d, C, j, E, El, me, EP, L.rows_cap, L.m, h->rows_d, h->rows_d + kMaxSub, cs,
                       h->gskip_d);
    prof_begin(h, 9, cs);
    // every peer is done with its buffers of slot j % S (chunk j - S, or the previous call)
    launch_sync_wait(area, EP, me, 3, j < S ? -1 : j - S + 1, h->status_d, cs);
    if (NB)
      launch_p2p_push<T>(x, pass == MEMFINE_BWD ? dy : nullptr, w, k, hd, E, El, EP, tab_j, L.m.send_src, L.m.info,
                         pt[j % S], (t1 - t0) * k, cs);
    launch_sync_signal(sp, me, 1, j + 1, cs);
    launch_sync_wait(area, EP, me, 1, j + 1, h->status_d, cs);   // every row pushed into this rank landed
    prof_end(h, cs);
    launch_zero_padding<T>(El, hd, L.m, (T*)L.X, pass == MEMFINE_BWD ? (T*)L.DY : nullptr, cs);
    if (pass == MEMFINE_BWD) MF_CUDA_OK(cudaMemsetAsync(L.m.dw_row, 0, sizeof(float) * L.rows_cap, cs));
    launch_p2p_row_addr(L.m.seg, L.m.recv_cnt, El, EP, tab_j, E, L.m.info, pt[j % S], rb, L.m.row_addr,
                        pass == MEMFINE_BWD ? L.m.row_addr_w : nullptr, L.rows_cap, cs);
    h->last.kernel_launches += 6;
    if constexpr (std::is_same<T, __nv_bfloat16>::value)
      if (mx) {   // MXFP8 (reading R28): the landed bf16 rows -> E4M3 + scale chunks
        launch_mx_quant_rows((const __nv_bfloat16*)L.X, hd, L.rows_cap, L.m.info, hd, L.Xq, L.Xsf, cs);
        h->last.kernel_launches += 1;
      }
    if (S == 2) MF_CUDA_OK(cudaEventRecord(h->ev_disp[j % 2], cs));
    return MEMFINE_OK;
  };
  auto compute = [&](int j) -> memfine_status {
    const Layout& L = Ls[j % S];
    if (S == 2) MF_CUDA_OK(cudaStreamWaitEvent(st, h->ev_disp[j % 2], 0));
    GemmProblem<T> p = base_problem<T>(h, L, wg, wu, wd);
    p.dWg = dwg;
    p.dWu = dwu;
    p.dWd = dwd;
    if (S == 2) p.sm_limit = h->num_sms - h->comm_sms;
    if (pass == MEMFINE_FWD) {
      p.kind = GK_GATEUP;
      p.store_a = 1;
      if constexpr (std::is_same<T, __nv_bfloat16>::value)
        if (mx) {
          set_mx(p, {L.Xq, L.Xsf}, W.op[0], W.op[1]);
          p.mx_aq = L.Aq;
          p.mx_aq_sf = L.Asf;
        }
      if (int rc = run_gemm<T>(h, p, st)) return (memfine_status)rc;
      p.kind = GK_DOWN;
      p.row_addr = L.m.row_addr;   // A8 + A9 fused: o rows stored into their source's send buffer
      if constexpr (std::is_same<T, __nv_bfloat16>::value)
        if (mx) set_mx(p, {L.Aq, L.Asf}, W.op[2], W.op[2]);
      if (int rc = run_gemm<T>(h, p, st)) return (memfine_status)rc;
    } else {
      p.kind = GK_GATEUP;
      p.store_a = 0;
      p.store_gu = 1;
      if constexpr (std::is_same<T, __nv_bfloat16>::value)
        if (mx) set_mx(p, {L.Xq, L.Xsf}, W.op[0], W.op[1]);
      if (int rc = run_gemm<T>(h, p, st)) return (memfine_status)rc;
      p.kind = GK_DACT;
      p.mx = 0;
      if (mx) {   // BF16 dA GEMM whose epilogue also writes dG || dU as E4M3 + scales
        p.mx_gq = L.GUq;
        p.mx_gq_sf = L.GUsf;
      }
      if (int rc = run_gemm<T>(h, p, st)) return (memfine_status)rc;
      p.mx_gq = nullptr;
      p.mx_gq_sf = nullptr;
      p.wgrad_beta = beta;
      if (int rc = run_wgrad<T>(h, p, L, st)) return (memfine_status)rc;
      beta = 1;
      p.kind = GK_DX;
      p.row_addr = L.m.row_addr;   // B4 + B6 fused: dX rows stored into their source's send buffer
      if constexpr (std::is_same<T, __nv_bfloat16>::value)
        if (mx) set_mx(p, {L.GUq, L.GUsf}, W.op[3], W.op[4]);
      if (int rc = run_gemm<T>(h, p, st)) return (memfine_status)rc;
      launch_p2p_push_dw(L.m.dw_row, L.m.row_addr_w, L.m.info, L.rows_cap, st);
      h->last.kernel_launches += 1;
    }
    launch_sync_signal(sp, me, 2, j + 1, st);
    h->last.kernel_launches += 1;
    if (S == 2) MF_CUDA_OK(cudaEventRecord(h->ev_gemm[j % 2], st));
    return MEMFINE_OK;
  };
  auto combine = [&](int j) -> memfine_status {
    const Layout& L = Ls[j % S];
    int64_t t0 = chunk_begin(d.tokens, C, j), t1 = chunk_begin(d.tokens, C, j + 1);
    if (S == 2) MF_CUDA_OK(cudaStreamWaitEvent(cs, h->ev_gemm[j % 2], 0));
    launch_sync_wait(area, EP, me, 2, j + 1, h->status_d, cs);   // every o / dX row of this rank's tokens landed
    if (pass == MEMFINE_FWD) {
      if (t1 > t0) launch_combine<T>((const T*)L.send, w, t0, t1, k, hd, L.m, out, cs);
    } else {
      ChunkMeta mb = L.m;
      mb.dw_row = L.send_w;
      if (t1 > t0) launch_unpermute_reduce<T>((const T*)L.send, t0, t1, k, hd, mb, out, dscore, cs);
    }
    // this rank's buffers of slot j % S are free for the peers' pushes / stores of chunk j + S (or the next call)
    launch_sync_signal(sp, me, 3, j + 1 == C ? kSyncDoneCall : j + 1, cs);
    h->last.kernel_launches += 3;
    return MEMFINE_OK;
  };
  if (S == 1) {
    for (int j = 0; j < C; j++) {
      if (memfine_status rc = dispatch(j)) return rc;
      if (memfine_status rc = compute(j)) return rc;
      if (memfine_status rc = combine(j)) return rc;
    }
  } else {
    if (memfine_status rc = dispatch(0)) return rc;
    for (int j = 0; j < C; j++) {
      if (j + 1 < C)
        if (memfine_status rc = dispatch(j + 1)) return rc;
      if (memfine_status rc = compute(j)) return rc;
      if (memfine_status rc = combine(j)) return rc;
    }
    MF_CUDA_OK(cudaEventRecord(h->ev_join, cs));
    MF_CUDA_OK(cudaStreamWaitEvent(st, h->ev_join, 0));
  }
  return latch_cuda(h);
}



// The comm stream of MEMFINE_FLAG_OVERLAP (created on first use, highest priority).
int ensure_comm_stream(memfine_handle_s* h) {
  if (h->cs) return 0;
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  if (cudaStreamCreateWithPriority(&h->cs, cudaStreamNonBlocking, hi)) return 1;
  for (cudaEvent_t* e : {&h->ev_disp[0], &h->ev_disp[1], &h->ev_gemm[0], &h->ev_gemm[1], &h->ev_fork, &h->ev_join})
    if (cudaEventCreateWithFlags(e, cudaEventDisableTiming)) return 1;
  return 0;
}

// The FCDA chunk loop with EP > 1 over send buffers + all-to-allv (MEMFINE_EP_COPY).
// One slot: every step of chunk j on the caller's stream, in the order of Eq. 6 / Eq. 7.
// Two slots (MEMFINE_FLAG_OVERLAP): the exchange side of each chunk - permute, dispatch
// all-to-allv, (after the chunk's GEMMs) combine all-to-allv and unpermute - runs on the comm
// stream cs, the GEMMs on st; chunk j uses slot j % 2.  Issue order on cs is
//   dispatch(0) dispatch(1) combine(0) dispatch(2) combine(1) dispatch(3) ...
// so chunk j+1's rows move while chunk j multiplies, and chunk j's results return while chunk
// j+1 multiplies.  Hazards: GEMMs(j) wait ev_disp[j%2] (their rows and metadata arrived);
// combine(j) waits ev_gemm[j%2] (o / dX_disp, d_w written); dispatch(j+2) reuses slot j%2 after
// combine(j) in cs order; G||U and a are touched by st only.  Results are bit-identical to the
// one-slot order: every kernel sees the same inputs.
template <typename T>
memfine_status ep_run(memfine_handle_s* h, int pass, const T* dy, const T* x, const int32_t* ids, const float* w,
                      const void* wg, const void* wu, const void* wd, int C, T* out, float* dwg, float* dwu,
                      float* dwd, float* dscore, int accumulate, void* ws, uint64_t ws_bytes, cudaStream_t st) {
  if (h->p2p)
    return ep_run_p2p<T>(h, pass, dy, x, ids, w, wg, wu, wd, C, out, dwg, dwu, dwd, dscore, accumulate, ws, ws_bytes,
                         st);
  const memfine_dims& d = h->d;
  int E = d.num_experts, El = E / d.ep_size, k = d.topk, hd = d.hidden;
  const bool mx = d.dtype == MEMFINE_MXFP8;
  if (mx && !h->mx_w) return MEMFINE_ERR_INVALID_ARG;   // memfine_mx_quantize_weights first
  MxWeightsLayout W = mx_weights_layout(d, h->mx_w);
  if (int rc = ep_gather_counts(h, ids, C, st)) return (memfine_status)rc;
  std::vector<EpChunk> tab;
  int64_t rows_max = 0, send_max = 0;
  for (int j = 0; j < C; j++) {
    tab.push_back(ep_chunk_table(d, h->counts_h, C, j));
    rows_max = std::max(rows_max, tab[j].rows_pad);
    send_max = std::max(send_max, tab[j].send);
  }
  Layout Ls[2];
  carve(d, C, pass, ws, rows_max, send_max, Ls);
  if (Ls[0].total > ws_bytes) return MEMFINE_ERR_WORKSPACE;
  const int S = ep_slots(d, C);
  if (h->lg) {
    auto& P = h->lg->ptrs[d.ep_rank];
    for (int s = 0; s < S; s++) {
      const Layout& L = Ls[s];
      char** Q = P.data() + 8 * s;
      Q[kPtrSend] = (char*)L.send;
      Q[kPtrSendDy] = (char*)L.send_dy;
      Q[kPtrSendW] = (char*)L.send_w;
      Q[kPtrX] = (char*)L.X;
      Q[kPtrDY] = (char*)L.DY;
      Q[kPtrO] = L.o_alias ? nullptr : (char*)L.O;  // O aliases X in the backward and with two slots
      Q[kPtrWRow] = (char*)L.m.w_row;
      Q[kPtrDWRow] = (char*)L.m.dw_row;
    }
  }
  h->last_meta = Ls[0].meta_bytes;
  h->last_row_bytes = Ls[0].row_bytes;
  size_t rb = (size_t)hd * sizeof(T);
  if (pass == MEMFINE_BWD && dscore && d.tokens > 0)
    MF_CUDA_OK(cudaMemsetAsync(dscore, 0, sizeof(float) * d.tokens * k, st));
  cudaStream_t cs = st;
  if (S == 2) {
    if (ensure_comm_stream(h)) return MEMFINE_ERR_CUDA;
    cs = h->cs;
    MF_CUDA_OK(cudaEventRecord(h->ev_fork, st));   // inputs, dscore zeroing, counts
    MF_CUDA_OK(cudaStreamWaitEvent(cs, h->ev_fork, 0));
  }

  // A5/B1 permute + A6 dispatch all-to-allv of chunk j into slot j % S (on cs)
  auto dispatch = [&](int j) -> memfine_status {
    const Layout& L = Ls[j % S];
    const EpChunk& t = tab[j];
    int64_t t0 = chunk_begin(d.tokens, C, j), t1 = chunk_begin(d.tokens, C, j + 1);
    int NB = (int)ceil_div64(t1 - t0, kTokPerBlk);
    ChunkMeta ms = L.m;
    ms.src_of = nullptr;
    ms.w_row = L.send_w;
    ms.dw_row = nullptr;
    if (NB) {
      launch_dispatch_hist(ids, t0, t1, k, E, L.m, h->status_d, cs);
      launch_dispatch_scan(NB, E, El, 1, L.rows_cap, L.m, nullptr, nullptr, j, cs);
      launch_dispatch_scatter<T>(x, pass == MEMFINE_BWD ? dy : nullptr, ids, w, t0, t1, k, E, hd, ms, (T*)L.send,
                                 pass == MEMFINE_BWD ? (T*)L.send_dy : nullptr, El, false, 0, cs);
      h->last.kernel_launches += 4;
    }
    launch_ep_recv_seg(h->counts_d, C, j, E, El, d.ep_rank, d.ep_size, L.rows_cap, L.m, h->rows_d,
                       h->rows_d + kMaxSub, cs);
    prof_begin(h, 9, cs);
    const int ko = 8 * (j % S);   // this slot's kinds in the in-process pointer table
    // B1: x, dY and the scores of the chunk move in ONE NCCL group (one fused launch per chunk)
    const bool grp = pass == MEMFINE_BWD && !h->lg;
    if (grp && nccl_group_start()) return MEMFINE_ERR_NCCL;
    int erc = ep_exchange(h, t, h->counts_h, C, j, true, (char*)L.send, (char*)L.X, rb, cs, ko + kPtrSend, ko + kPtrX);
    if (pass == MEMFINE_BWD) {
      erc |= ep_exchange(h, t, h->counts_h, C, j, true, (char*)L.send_dy, (char*)L.DY, rb, cs, ko + kPtrSendDy,
                         ko + kPtrDY);
      erc |= ep_exchange(h, t, h->counts_h, C, j, true, (char*)L.send_w, (char*)L.m.w_row, 4, cs, ko + kPtrSendW,
                         ko + kPtrWRow);
    }
    if (grp && nccl_group_end()) return MEMFINE_ERR_NCCL;
    if (erc) return MEMFINE_ERR_NCCL;
    if (pass == MEMFINE_BWD) {
      if (t.rows_pad) MF_CUDA_OK(cudaMemsetAsync(L.m.dw_row, 0, sizeof(float) * t.rows_pad, cs));
    }
    prof_end(h, cs);
    launch_zero_padding<T>(El, hd, L.m, (T*)L.X, pass == MEMFINE_BWD ? (T*)L.DY : nullptr, cs);
    h->last.kernel_launches += 2;
    if (S == 2) MF_CUDA_OK(cudaEventRecord(h->ev_disp[j % 2], cs));
    return MEMFINE_OK;
  };
  // A9/B6 combine all-to-allv + A10/B7 unpermute of chunk j (on cs)
  auto combine = [&](int j) -> memfine_status {
    const Layout& L = Ls[j % S];
    const EpChunk& t = tab[j];
    int64_t t0 = chunk_begin(d.tokens, C, j), t1 = chunk_begin(d.tokens, C, j + 1);
    if (S == 2) MF_CUDA_OK(cudaStreamWaitEvent(cs, h->ev_gemm[j % 2], 0));
    const int ko = 8 * (j % S);
    // B6: dX rows and d_score of the chunk in ONE NCCL group
    const bool grp = pass == MEMFINE_BWD && !h->lg;
    if (grp && nccl_group_start()) return MEMFINE_ERR_NCCL;
    int erc = ep_exchange(h, t, h->counts_h, C, j, false, (char*)L.send, (char*)L.O, rb, cs, ko + kPtrSend,
                          ko + (L.o_alias ? kPtrX : kPtrO));
    if (pass == MEMFINE_BWD)
      erc |= ep_exchange(h, t, h->counts_h, C, j, false, (char*)L.send_w, (char*)L.m.dw_row, 4, cs, ko + kPtrSendW,
                         ko + kPtrDWRow);
    if (grp && nccl_group_end()) return MEMFINE_ERR_NCCL;
    if (erc) return MEMFINE_ERR_NCCL;
    if (pass == MEMFINE_FWD) {
      if (t1 > t0) launch_combine<T>((const T*)L.send, w, t0, t1, k, hd, L.m, out, cs);
    } else {
      ChunkMeta mb = L.m;
      mb.dw_row = L.send_w;
      if (t1 > t0) launch_unpermute_reduce<T>((const T*)L.send, t0, t1, k, hd, mb, out, dscore, cs);
    }
    h->last.kernel_launches += 1;
    return MEMFINE_OK;
  };
  int beta = accumulate ? 1 : 0;  // first chunk overwrites dW, later chunks accumulate
  // A7-A8 / B2-B5 expert GEMMs of chunk j (on st)
  auto compute = [&](int j) -> memfine_status {
    Nvtx chunk_range(chunk_range_name(pass == MEMFINE_BWD, j));
    const Layout& L = Ls[j % S];
    if (S == 2) MF_CUDA_OK(cudaStreamWaitEvent(st, h->ev_disp[j % 2], 0));
    GemmProblem<T> p = base_problem<T>(h, L, wg, wu, wd);
    p.dWg = dwg;
    p.dWu = dwu;
    p.dWd = dwd;
    if (S == 2) p.sm_limit = h->num_sms - h->comm_sms;
    if constexpr (std::is_same<T, __nv_bfloat16>::value)
      if (mx) {   // MXFP8 (reading R28): the received bf16 rows -> E4M3 + scale chunks
        prof_begin(h, 6, st);
        launch_mx_quant_rows((const __nv_bfloat16*)L.X, hd, L.rows_cap, L.m.info, hd, L.Xq, L.Xsf, st);
        prof_end(h, st);
        h->last.kernel_launches += 1;
      }
    if (pass == MEMFINE_FWD) {
      p.kind = GK_GATEUP;
      p.store_a = 1;
      if constexpr (std::is_same<T, __nv_bfloat16>::value)
        if (mx) {
          set_mx(p, {L.Xq, L.Xsf}, W.op[0], W.op[1]);
          p.mx_aq = L.Aq;
          p.mx_aq_sf = L.Asf;
        }
      if (int rc = run_gemm<T>(h, p, st)) return (memfine_status)rc;
      p.kind = GK_DOWN;   // (two slots / MX: o written over X_disp, dead after gate/up)
      if constexpr (std::is_same<T, __nv_bfloat16>::value)
        if (mx) set_mx(p, {L.Aq, L.Asf}, W.op[2], W.op[2]);
      if (int rc = run_gemm<T>(h, p, st)) return (memfine_status)rc;
    } else {
      p.kind = GK_GATEUP;
      p.store_a = 0;
      p.store_gu = 1;
      if constexpr (std::is_same<T, __nv_bfloat16>::value)
        if (mx) set_mx(p, {L.Xq, L.Xsf}, W.op[0], W.op[1]);
      if (int rc = run_gemm<T>(h, p, st)) return (memfine_status)rc;
      p.kind = GK_DACT;
      p.mx = 0;
      if (mx) {   // BF16 dA GEMM whose epilogue also writes dG || dU as E4M3 + scales
        p.mx_gq = L.GUq;
        p.mx_gq_sf = L.GUsf;
      }
      if (int rc = run_gemm<T>(h, p, st)) return (memfine_status)rc;
      p.mx_gq = nullptr;
      p.mx_gq_sf = nullptr;
      p.wgrad_beta = beta;
      if (int rc = run_wgrad<T>(h, p, L, st)) return (memfine_status)rc;
      beta = 1;
      p.kind = GK_DX;
      if constexpr (std::is_same<T, __nv_bfloat16>::value)
        if (mx) set_mx(p, {L.GUq, L.GUsf}, W.op[3], W.op[4]);
      if (int rc = run_gemm<T>(h, p, st)) return (memfine_status)rc;
    }
    if (S == 2) MF_CUDA_OK(cudaEventRecord(h->ev_gemm[j % 2], st));
    return MEMFINE_OK;
  };

  if (S == 1) {
    for (int j = 0; j < C; j++) {
      if (memfine_status rc = dispatch(j)) return rc;
      if (memfine_status rc = compute(j)) return rc;
      if (memfine_status rc = combine(j)) return rc;
    }
  } else {
    if (memfine_status rc = dispatch(0)) return rc;
    for (int j = 0; j < C; j++) {
      if (j + 1 < C)
        if (memfine_status rc = dispatch(j + 1)) return rc;
      if (memfine_status rc = compute(j)) return rc;
      if (memfine_status rc = combine(j)) return rc;
    }
    MF_CUDA_OK(cudaEventRecord(h->ev_join, cs));
    MF_CUDA_OK(cudaStreamWaitEvent(st, h->ev_join, 0));
  }
  return latch_cuda(h);
}

memfine_status memfine_ep_fwd(memfine_handle_s* h, const void* x, const int32_t* ids, const float* w, const void* wg,
                              const void* wu, const void* wd, int C, void* y, void* ws, uint64_t ws_bytes,
                              cudaStream_t st) {
  if (h->d.dtype != MEMFINE_FP32)   // BF16 and MXFP8 (bf16 storage)
    return ep_run<__nv_bfloat16>(h, MEMFINE_FWD, nullptr, (const __nv_bfloat16*)x, ids, w, wg, wu, wd, C,
                                 (__nv_bfloat16*)y, nullptr, nullptr, nullptr, nullptr, 0, ws, ws_bytes, st);
  return ep_run<float>(h, MEMFINE_FWD, nullptr, (const float*)x, ids, w, wg, wu, wd, C, (float*)y, nullptr, nullptr,
                       nullptr, nullptr, 0, ws, ws_bytes, st);
}

memfine_status memfine_ep_bwd(memfine_handle_s* h, const void* dy, const void* x, const int32_t* ids, const float* w,
                              const void* wg, const void* wu, const void* wd, int C, void* dx, float* dwg, float* dwu,
                              float* dwd, float* dscore, int accumulate, void* ws, uint64_t ws_bytes,
                              cudaStream_t st) {
  if (h->d.dtype != MEMFINE_FP32)   // BF16 and MXFP8 (bf16 storage)
    return ep_run<__nv_bfloat16>(h, MEMFINE_BWD, (const __nv_bfloat16*)dy, (const __nv_bfloat16*)x, ids, w, wg, wu,
                                 wd, C, (__nv_bfloat16*)dx, dwg, dwu, dwd, dscore, accumulate, ws, ws_bytes, st);
  return ep_run<float>(h, MEMFINE_BWD, (const float*)dy, (const float*)x, ids, w, wg, wu, wd, C, (float*)dx, dwg,
                       dwu, dwd, dscore, accumulate, ws, ws_bytes, st);
}

void begin_call(memfine_handle_s* h, int C, int pass, uint64_t ws_bytes, cudaStream_t st) {
  h->last = memfine_stats{};
  if (h->debug) {
    h->dbg_mx.assign(C, {});
    h->dbg_src.assign(C, {});
  }
  h->last.C = C;
  h->last.pass = pass;
  h->last.workspace_given_bytes = ws_bytes;
  // rows_h is written by the scan kernels in stream order; clear it in stream order too.
  cudaMemsetAsync(h->rows_d, 0, sizeof(int64_t) * 2 * kMaxSub, st);
}

}  // namespace

// =================================================================================== C ABI
// Per-handle device state of the device-planned P2P exchange (N1): sync area (zeroed; the "done" flags
// start at the previous-call marker so the first call's chunk 0 may push), skip flags, counts.
// Lazy module loading (CUDA_MODULE_LOADING=LAZY, the CUDA 12 default) loads a kernel at its first launch, and a
// load waits for the kernels already running on the device.  The device-planned P2P exchange has kernels of one
// rank spin-wait on flags raised by another rank's kernels; in an in-process group a first launch in one rank's
// thread would wait behind the other rank's spinning kernel, which waits for this rank (measured: 20-60 s stalls
// until the bounded spin latches an error, in ~half the runs).  So every function of every module of the library
// is loaded before the first P2P call.  Driver entry points through the runtime (no -lcuda).
memfine_status preload_all_kernels() {
  static std::once_flag once;
  static memfine_status rc = MEMFINE_OK;
  std::call_once(once, [] {
    void *p_mod = nullptr, *p_cnt = nullptr, *p_enum = nullptr, *p_load = nullptr;
    cudaDriverEntryPointQueryResult q;
    bool ok = cudaGetDriverEntryPoint("cuFuncGetModule", &p_mod, cudaEnableDefault, &q) == cudaSuccess && p_mod &&
              cudaGetDriverEntryPoint("cuModuleGetFunctionCount", &p_cnt, cudaEnableDefault, &q) == cudaSuccess &&
              p_cnt && cudaGetDriverEntryPoint("cuModuleEnumerateFunctions", &p_enum, cudaEnableDefault, &q) ==
              cudaSuccess && p_enum && cudaGetDriverEntryPoint("cuFuncLoad", &p_load, cudaEnableDefault, &q) ==
              cudaSuccess && p_load;
    if (!ok) { cudaGetLastError(); rc = MEMFINE_ERR_CUDA; return; }
    auto get_mod = (PFN_cuFuncGetModule_v11000)p_mod;
    auto count = (PFN_cuModuleGetFunctionCount_v12040)p_cnt;
    auto enumerate = (PFN_cuModuleEnumerateFunctions_v12040)p_enum;
    auto load = (PFN_cuFuncLoad_v12040)p_load;
    const void* anchors[] = {kernel_anchor_route(), kernel_anchor_mx(), kernel_anchor_router(), kernel_anchor_simt(),
                             kernel_anchor_sm100()};
    for (const void* a : anchors) {
      cudaFunction_t f;
      CUmodule mod;
      unsigned n = 0;
      if (cudaGetFuncBySymbol(&f, a) != cudaSuccess || get_mod(&mod, (CUfunction)f) != CUDA_SUCCESS ||
          count(&n, mod) != CUDA_SUCCESS) {
        cudaGetLastError();
        rc = MEMFINE_ERR_CUDA;
        return;
      }
      std::vector<CUfunction> fs(n);
      if (n && enumerate(fs.data(), n, mod) != CUDA_SUCCESS) { rc = MEMFINE_ERR_CUDA; return; }
      for (CUfunction fn : fs)
        if (load(fn) != CUDA_SUCCESS) { rc = MEMFINE_ERR_CUDA; return; }
    }
  });
  return rc;
}

memfine_status p2p_alloc_sync(memfine_handle_s* h) {
  const memfine_dims& d = h->d;
  if (memfine_status rc = preload_all_kernels()) return rc;
  const size_t sb = sync_area_bytes(d.num_experts);
  if (!h->sync_d) {
    MF_CUDA_OK(cudaMalloc((void**)&h->sync_d, sb));
    MF_CUDA_OK(cudaMalloc((void**)&h->gskip_d, sizeof(int) * kMaxSub));
  }
  const size_t need = (size_t)d.ep_size * kMaxSub * d.num_experts;
  if (need > h->counts_cap) {
    if (h->counts_d) cudaFree(h->counts_d);
    if (h->counts_h) cudaFreeHost(h->counts_h);
    h->counts_d = nullptr;
    h->counts_h = nullptr;
    h->counts_cap = 0;
    MF_CUDA_OK(cudaMalloc((void**)&h->counts_d, need * sizeof(int)));
    MF_CUDA_OK(cudaHostAlloc((void**)&h->counts_h, need * sizeof(int), cudaHostAllocDefault));
    h->counts_cap = need;
  }
  std::vector<uint64_t> init(1 + (size_t)kSyncPhases * kMaxPeers, 0);
  for (int p = 0; p < kMaxPeers; p++) init[1 + 3 * kMaxPeers + p] = kSyncDoneCall;   // epoch 0, call done
  MF_CUDA_OK(cudaMemset(h->sync_d, 0, sb));
  MF_CUDA_OK(cudaMemcpy(h->sync_d, init.data(), init.size() * sizeof(uint64_t), cudaMemcpyHostToDevice));
  MF_CUDA_OK(cudaDeviceSynchronize());
  return MEMFINE_OK;
}

memfine_status register_local(memfine_handle_s* h, void* ws, uint64_t ws_bytes) {
  memfine_group_s* g = h->lg;
  const int EP = h->d.ep_size, me = h->d.ep_rank;
  memfine_status rc = p2p_alloc_sync(h);
  g->ptrs[me][kPtrWs] = (char*)ws;
  g->ptrs[me][kPtrSync] = (char*)h->sync_d;
  g->ptrs[me][kPtrWsBytes] = (char*)(uintptr_t)(rc == MEMFINE_OK ? ws_bytes : 0);
  g->barrier();   // every rank published its workspace and sync area
  h->peer_ws.assign(EP, nullptr);
  h->peer_sync.assign(EP, nullptr);
  bool same = true;
  for (int r = 0; r < EP; r++) {
    h->peer_ws[r] = g->ptrs[r][kPtrWs];
    h->peer_sync[r] = (uint64_t*)g->ptrs[r][kPtrSync];
    same = same && (uint64_t)(uintptr_t)g->ptrs[r][kPtrWsBytes] == ws_bytes;
  }
  g->barrier();   // nobody republishes before every rank has read
  if (rc != MEMFINE_OK) return rc;
  if (!same) return MEMFINE_ERR_INVALID_ARG;   // the fused exchange needs one workspace size on every rank
  h->reg_ws = ws;
  h->reg_bytes = ws_bytes;
  return MEMFINE_OK;
}

extern "C" {

int32_t memfine_abi_version(void) { return MEMFINE_ABI_VERSION; }

memfine_status memfine_m_g(int32_t v, int32_t p, int32_t r_pp, int32_t full_recompute, int32_t* m_g) {
  if (!m_g || v < 1 || p < 1 || r_pp < 0 || r_pp >= p) return MEMFINE_ERR_INVALID_ARG;
  // m_g = v p + p - 2 r_pp - 1 (>= 1 for 0 <= r_pp < p); 1 under full recomputation
  *m_g = full_recompute ? 1 : v * p + p - 2 * r_pp - 1;
  return MEMFINE_OK;
}

const char* memfine_status_str(memfine_status s) {
  switch (s) {
    case MEMFINE_OK: return "ok";
    case MEMFINE_ERR_INVALID_ARG: return "invalid argument";
    case MEMFINE_ERR_INFEASIBLE: return "infeasible: the static memory or the budget leaves no room (Eq. 3/8)";
    case MEMFINE_ERR_ROUTING: return "routing: expert id outside [0, E)";
    case MEMFINE_ERR_CUDA: return "CUDA error (or no sm_100 device)";
    case MEMFINE_ERR_NCCL: return "NCCL error (or libnccl.so.2 not loadable)";
    case MEMFINE_ERR_WORKSPACE: return "workspace smaller than memfine_workspace_bytes()";
    case MEMFINE_ERR_UNSUPPORTED: return "unsupported shape";
  }
  return "unknown status";
}

memfine_status memfine_nccl_unique_id(uint8_t out_id[128]) {
  if (!out_id) return MEMFINE_ERR_INVALID_ARG;
  return nccl_get_unique_id(out_id) ? MEMFINE_ERR_NCCL : MEMFINE_OK;
}

memfine_status memfine_create(const memfine_dims* dims, const uint8_t* nccl_unique_id, memfine_handle_t* out) {
  if (!out || !dims_ok(dims)) return MEMFINE_ERR_INVALID_ARG;
  if (ep_path(*dims) != (nccl_unique_id != nullptr)) return MEMFINE_ERR_INVALID_ARG;
  *out = nullptr;
  int dev;
  if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return MEMFINE_ERR_CUDA; }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) { cudaGetLastError(); return MEMFINE_ERR_CUDA; }
  if (prop.major != 10 || prop.minor != 0) return MEMFINE_ERR_CUDA;  // built for sm_100a only
  memfine_handle_s* h = new memfine_handle_s();
  h->d = *dims;
  h->device = dev;
  h->num_sms = prop.multiProcessorCount;
  if (cudaHostAlloc((void**)&h->status_h, sizeof(int) * 4, cudaHostAllocMapped) != cudaSuccess ||
      cudaHostAlloc((void**)&h->rows_h, sizeof(int64_t) * 2 * kMaxSub, cudaHostAllocMapped) != cudaSuccess) {
    memfine_destroy(h);
    return MEMFINE_ERR_CUDA;
  }
  memset(h->status_h, 0, sizeof(int) * 4);
  memset(h->rows_h, 0, sizeof(int64_t) * 2 * kMaxSub);
  cudaHostGetDevicePointer((void**)&h->status_d, h->status_h, 0);
  cudaHostGetDevicePointer((void**)&h->rows_d, h->rows_h, 0);
  cudaEventCreateWithFlags(&h->ev, cudaEventDisableTiming);
  if (ep_path(*dims)) {
    if (nccl_comm_init(&h->comm, nccl_unique_id, dims->ep_size, dims->ep_rank)) {
      memfine_destroy(h);
      return MEMFINE_ERR_NCCL;
    }
  }
  *out = h;
  return MEMFINE_OK;
}

memfine_status memfine_local_group_create(int32_t nranks, memfine_group_t* out) {
  if (!out || nranks < 1 || nranks > 64) return MEMFINE_ERR_INVALID_ARG;
  memfine_group_s* g = new memfine_group_s();
  g->n = nranks;
  g->ready.resize(nranks);
  g->done.resize(nranks);
  g->ptrs.assign(nranks, {});
  for (int r = 0; r < nranks; r++) {
    if (cudaEventCreateWithFlags(&g->ready[r], cudaEventDisableTiming) ||
        cudaEventCreateWithFlags(&g->done[r], cudaEventDisableTiming)) {
      cudaGetLastError();
      memfine_local_group_destroy(g);
      return MEMFINE_ERR_CUDA;
    }
  }
  *out = g;
  return MEMFINE_OK;
}

memfine_status memfine_local_group_destroy(memfine_group_t g) {
  if (!g) return MEMFINE_ERR_INVALID_ARG;
  for (auto e : g->ready) if (e) cudaEventDestroy(e);
  for (auto e : g->done) if (e) cudaEventDestroy(e);
  delete g;
  return MEMFINE_OK;
}

memfine_status memfine_create_local(const memfine_dims* dims, memfine_group_t group, memfine_handle_t* out) {
  if (!group || !dims || !out || dims->ep_size != group->n) return MEMFINE_ERR_INVALID_ARG;
  memfine_dims d1 = *dims;
  int ep = d1.ep_size, rk = d1.ep_rank;
  d1.ep_size = 1;   // create with the single-rank path, then switch to the group
  d1.ep_rank = 0;
  if (!dims_ok(dims)) return MEMFINE_ERR_INVALID_ARG;
  memfine_status st = memfine_create(&d1, nullptr, out);
  if (st != MEMFINE_OK) return st;
  (*out)->d.ep_size = ep;
  (*out)->d.ep_rank = rk;
  (*out)->lg = group;
  return MEMFINE_OK;
}

memfine_status memfine_set_comm_sms(memfine_handle_t h, int32_t n) {
  if (!h || n < 0 || n >= h->num_sms) return MEMFINE_ERR_INVALID_ARG;
  h->comm_sms = n;
  return MEMFINE_OK;
}

memfine_status memfine_set_ep_transport(memfine_handle_t h, int32_t transport) {
  if (!h || (transport != MEMFINE_EP_COPY && transport != MEMFINE_EP_P2P)) return MEMFINE_ERR_INVALID_ARG;
  if (transport == MEMFINE_EP_P2P && h->d.ep_size > kMaxPeers) return MEMFINE_ERR_UNSUPPORTED;
  if (h->ipc_only) return transport == MEMFINE_EP_P2P ? MEMFINE_OK : MEMFINE_ERR_UNSUPPORTED;   // no NCCL
  if (transport == MEMFINE_EP_P2P && !h->lg && h->d.ep_size > 1 && !h->comm.comm) return MEMFINE_ERR_UNSUPPORTED;
  h->p2p = transport == MEMFINE_EP_P2P;
  return MEMFINE_OK;
}

// Multi-process P2P: export the allocation holding ws (base + offset) through CUDA IPC, all-gather
// the records over the handle's NCCL communicator, open every peer's mapping.
// CUDA IPC mapping record of one rank (memfine_ipc_export / memfine_register_workspace)
struct IpcRec {
  cudaIpcMemHandle_t hdl, sync;
  uint64_t offset, bytes;
};
static_assert(sizeof(IpcRec) <= MEMFINE_IPC_RECORD_BYTES, "record");

memfine_status ipc_export_rec(memfine_handle_s* h, void* ws, uint64_t ws_bytes, IpcRec* out) {
  if (memfine_status rc = p2p_alloc_sync(h)) return rc;
  // allocation base of ws
  typedef CUresult (*RangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
  static RangeFn range_fn = nullptr;
  if (!range_fn) {
    cudaDriverEntryPointQueryResult q;
    void* fp = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fp, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return MEMFINE_ERR_CUDA;
    range_fn = (RangeFn)fp;
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range_fn(&base, &size, (CUdeviceptr)ws) != CUDA_SUCCESS) return MEMFINE_ERR_CUDA;
  memset(out, 0, sizeof *out);
  if (cudaIpcGetMemHandle(&out->hdl, (void*)base) != cudaSuccess ||
      cudaIpcGetMemHandle(&out->sync, (void*)h->sync_d) != cudaSuccess) {
    cudaGetLastError();
    return MEMFINE_ERR_CUDA;
  }
  out->offset = (uint64_t)((char*)ws - (char*)base);
  out->bytes = ws_bytes;
  return MEMFINE_OK;
}

// map every peer's workspace and sync area (all[r], rank order); this rank's entries stay local
memfine_status ipc_import_recs(memfine_handle_s* h, const IpcRec* all, void* ws, uint64_t ws_bytes) {
  const int EP = h->d.ep_size, me = h->d.ep_rank;
  for (void* b : h->ipc_bases) cudaIpcCloseMemHandle(b);
  h->ipc_bases.clear();
  h->peer_ws.assign(EP, nullptr);
  h->peer_sync.assign(EP, nullptr);
  h->reg_ws = nullptr;
  h->reg_bytes = 0;
  for (int r = 0; r < EP; r++)
    if (all[r].bytes != ws_bytes) return MEMFINE_ERR_INVALID_ARG;   // one workspace size on every rank
  for (int r = 0; r < EP; r++) {
    if (r == me) {
      h->peer_ws[r] = (char*)ws;
      h->peer_sync[r] = h->sync_d;
      continue;
    }
    void* pb = nullptr;
    void* ps = nullptr;
    if (cudaIpcOpenMemHandle(&pb, all[r].hdl, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
        cudaIpcOpenMemHandle(&ps, all[r].sync, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      return MEMFINE_ERR_CUDA;
    }
    h->ipc_bases.push_back(pb);
    h->ipc_bases.push_back(ps);
    h->peer_ws[r] = (char*)pb + all[r].offset;
    h->peer_sync[r] = (uint64_t*)ps;
  }
  h->reg_ws = ws;
  h->reg_bytes = ws_bytes;
  return MEMFINE_OK;
}

memfine_status memfine_register_workspace(memfine_handle_t h, void* ws, uint64_t ws_bytes, void* stream) {
  if (!h || !ws) return MEMFINE_ERR_INVALID_ARG;
  if (h->lg) return register_local(h, ws, ws_bytes);
  if (h->ipc_only) return MEMFINE_ERR_INVALID_ARG;   // memfine_ipc_export / memfine_ipc_import
  if (!ep_path(h->d)) {   // a single rank without the EP path: nothing to map
    h->reg_ws = ws;
    h->reg_bytes = ws_bytes;
    return MEMFINE_OK;
  }
  if (!h->comm.comm) return MEMFINE_ERR_NCCL;
  cudaStream_t st = (cudaStream_t)stream;
  IpcRec mine;
  if (memfine_status rc = ipc_export_rec(h, ws, ws_bytes, &mine)) return rc;
  const int EP = h->d.ep_size;
  char* dbuf = nullptr;
  MF_CUDA_OK(cudaMalloc((void**)&dbuf, sizeof(IpcRec) * (EP + 1)));
  MF_CUDA_OK(cudaMemcpyAsync(dbuf + sizeof(IpcRec) * EP, &mine, sizeof(IpcRec), cudaMemcpyHostToDevice, st));
  if (nccl_all_gather_bytes(&h->comm, dbuf + sizeof(IpcRec) * EP, dbuf, sizeof(IpcRec), st)) {
    cudaFree(dbuf);
    return MEMFINE_ERR_NCCL;
  }
  std::vector<IpcRec> all(EP);
  cudaMemcpyAsync(all.data(), dbuf, sizeof(IpcRec) * EP, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  cudaFree(dbuf);
  if (memfine_status rc = ipc_import_recs(h, all.data(), ws, ws_bytes)) return rc;
  // every rank has opened every mapping and initialised its flags before anyone signals
  if (nccl_stream_barrier(&h->comm, h->gskip_d, st)) return MEMFINE_ERR_NCCL;
  MF_CUDA_OK(cudaStreamSynchronize(st));
  return MEMFINE_OK;
}

memfine_status memfine_create_ipc(const memfine_dims* dims, memfine_handle_t* out) {
  if (!out || !dims || !dims_ok(dims)) return MEMFINE_ERR_INVALID_ARG;
  if (dims->ep_size < 2 || dims->ep_size > kMaxPeers) return MEMFINE_ERR_INVALID_ARG;
  if (dims->flags & MEMFINE_FLAG_EP_PATH) return MEMFINE_ERR_INVALID_ARG;
  memfine_dims d1 = *dims;
  d1.ep_size = 1;   // create with the single-rank path (no communicator), then switch to the EP layout
  d1.ep_rank = 0;
  d1.flags &= ~MEMFINE_FLAG_OVERLAP;
  memfine_status st = memfine_create(&d1, nullptr, out);
  if (st != MEMFINE_OK) return st;
  (*out)->d.ep_size = dims->ep_size;
  (*out)->d.ep_rank = dims->ep_rank;
  (*out)->d.flags = dims->flags;   // (MEMFINE_FLAG_OVERLAP: the two-slot pipeline of the peer-memory exchange)
  (*out)->ipc_only = 1;
  (*out)->p2p = 1;
  return MEMFINE_OK;
}

memfine_status memfine_ipc_export(memfine_handle_t h, void* ws, uint64_t ws_bytes, uint8_t* record) {
  if (!h || !ws || !record || !h->ipc_only) return MEMFINE_ERR_INVALID_ARG;
  IpcRec mine;
  if (memfine_status rc = ipc_export_rec(h, ws, ws_bytes, &mine)) return rc;
  memset(record, 0, MEMFINE_IPC_RECORD_BYTES);
  memcpy(record, &mine, sizeof mine);
  h->exp_ws = ws;
  h->exp_bytes = ws_bytes;
  return MEMFINE_OK;
}

memfine_status memfine_ipc_import(memfine_handle_t h, const uint8_t* records) {
  if (!h || !records || !h->ipc_only || !h->exp_ws) return MEMFINE_ERR_INVALID_ARG;
  std::vector<IpcRec> all(h->d.ep_size);
  for (int r = 0; r < h->d.ep_size; r++) memcpy(&all[r], records + (size_t)r * MEMFINE_IPC_RECORD_BYTES, sizeof(IpcRec));
  return ipc_import_recs(h, all.data(), h->exp_ws, h->exp_bytes);
}

memfine_status memfine_destroy(memfine_handle_t h) {
  if (!h) return MEMFINE_ERR_INVALID_ARG;
  if (h->router_scratch) cudaFree(h->router_scratch);
  for (void* b : h->ipc_bases) cudaIpcCloseMemHandle(b);
  if (h->sync_d) cudaFree(h->sync_d);
  if (h->gskip_d) cudaFree(h->gskip_d);
  if (h->comm.comm) nccl_comm_destroy(&h->comm);
  if (h->status_h) cudaFreeHost(h->status_h);
  if (h->rows_h) cudaFreeHost(h->rows_h);
  if (h->counts_d) cudaFree(h->counts_d);
  if (h->counts_h) cudaFreeHost(h->counts_h);
  if (h->ev) cudaEventDestroy(h->ev);
  for (cudaEvent_t e : {h->ev_disp[0], h->ev_disp[1], h->ev_gemm[0], h->ev_gemm[1], h->ev_fork, h->ev_join})
    if (e) cudaEventDestroy(e);
  if (h->cs) cudaStreamDestroy(h->cs);
  for (auto e : h->pool) cudaEventDestroy(e);
  delete h;
  return MEMFINE_OK;
}

memfine_status memfine_route_counts(memfine_handle_t h, const int32_t* ids_dev, int32_t nsub, int32_t* counts_dev,
                                    void* stream) {
  if (!h || (!ids_dev && h->d.tokens > 0) || !counts_dev || nsub < 1 || nsub > kMaxSub)
    return MEMFINE_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const memfine_dims& d = h->d;
  int* mine = counts_dev + (int64_t)d.ep_rank * nsub * d.num_experts;
  launch_route_hist(ids_dev, d.tokens, d.topk, d.num_experts, nsub, mine, h->status_d, st);
  if (cudaGetLastError() != cudaSuccess) return MEMFINE_ERR_CUDA;
  if (d.ep_size > 1 && h->lg) {
    h->lg->ptrs[d.ep_rank][0] = (char*)mine;
    local_fence(h, st, h->lg->ready);
    size_t nb = sizeof(int) * (size_t)nsub * d.num_experts;
    for (int r = 0; r < d.ep_size; r++)
      if (r != d.ep_rank)
        MF_CUDA_OK(cudaMemcpyAsync(counts_dev + (int64_t)r * nsub * d.num_experts, h->lg->ptrs[r][0], nb,
                                   cudaMemcpyDeviceToDevice, st));
    local_fence(h, st, h->lg->done);
  } else if (ep_path(d) && !h->ipc_only) {   // (IPC handles: the caller all-gathers)
    if (nccl_all_gather_int(&h->comm, mine, counts_dev, (size_t)nsub * d.num_experts, st)) return MEMFINE_ERR_NCCL;
  }
  return MEMFINE_OK;
}

memfine_status plan_host(const int32_t* counts, int32_t nsub, const memfine_dims* dims, const memfine_budget* budget,
                         memfine_plan_info* info);
memfine_status plan_impl(const int32_t* counts_host, int32_t nsub, const memfine_dims* dims,
                         const memfine_budget* budget, memfine_plan_info* info);

// ordered = true: device counts are read in `stream` order and only `stream` is synchronised (the other
// streams of the caller keep running); false: the whole device is synchronised first (counts may come
// from any stream).
memfine_status plan_any(const int32_t* counts, int32_t nsub, const memfine_dims* dims, const memfine_budget* budget,
                        memfine_plan_info* info, cudaStream_t stream, bool ordered) {
  if (!counts || !info) return MEMFINE_ERR_INVALID_ARG;
  PlanParams p;
  if (int rc = budget_to_params(dims, budget, nsub, &p)) return (memfine_status)rc;
  memset(info, 0, sizeof *info);
  // per host thread and device: pinned result words and a stream (a layer plans every step)
  struct PlanCtx { int dev = -1; memfine_plan_info* out_h = nullptr; cudaStream_t st = nullptr;
                   std::vector<int32_t> hc; int32_t* pin = nullptr; size_t pin_n = 0; };
  static thread_local PlanCtx ctx;
  const bool dev_counts = is_device_ptr(counts);
  if (dev_counts) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return MEMFINE_ERR_CUDA; }
    if (ctx.dev != dev) {
      if (ctx.out_h) cudaFreeHost(ctx.out_h);
      if (ctx.pin) cudaFreeHost(ctx.pin);
      if (ctx.st) cudaStreamDestroy(ctx.st);
      ctx = PlanCtx{};
      if (cudaHostAlloc((void**)&ctx.out_h, sizeof(memfine_plan_info) + 16, cudaHostAllocMapped) != cudaSuccess ||
          cudaStreamCreateWithFlags(&ctx.st, cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        return MEMFINE_ERR_CUDA;
      }
      ctx.dev = dev;
    }
  }
  cudaStream_t st = ordered ? stream : ctx.st;
  if (dev_counts && !ordered) cudaDeviceSynchronize();   // counts may come from any stream of the caller
  if (budget->model == MEMFINE_MODEL_IMPL) {
    if (dev_counts) {
      const size_t n = (size_t)p.EP * nsub * p.E;
      if (ctx.pin_n < n) {
        if (ctx.pin) cudaFreeHost(ctx.pin);
        ctx.pin = nullptr;
        ctx.pin_n = 0;
        MF_CUDA_OK(cudaHostAlloc((void**)&ctx.pin, n * sizeof(int32_t), cudaHostAllocDefault));
        ctx.pin_n = n;
      }
      MF_CUDA_OK(cudaMemcpyAsync(ctx.pin, counts, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      MF_CUDA_OK(cudaStreamSynchronize(st));
      return plan_impl(ctx.pin, nsub, dims, budget, info);
    }
    return plan_impl(counts, nsub, dims, budget, info);
  }
  if (dev_counts) {
    // A3 on the device: the single-CTA tuner kernel reads the (all-gathered) counts in HBM; its result
    // lands in pinned mapped memory
    memfine_plan_info* out_h = ctx.out_h;
    int* rc_h = (int*)(out_h + 1);
    *rc_h = -1;
    memfine_plan_info* out_d;
    cudaHostGetDevicePointer((void**)&out_d, out_h, 0);
    int* rc_d = (int*)(out_d + 1);
    const int lrc = launch_plan_kernel(counts, p, out_d, rc_d, st);
    cudaError_t e = cudaStreamSynchronize(st);
    int rc = *rc_h;
    if (lrc || e != cudaSuccess || rc < 0) {   // launch failure: the result words were never written
      cudaGetLastError();
      return MEMFINE_ERR_CUDA;
    }
    *info = *out_h;
    return (memfine_status)rc;
  }
  return plan_host(counts, nsub, dims, budget, info);
}

memfine_status memfine_plan(const int32_t* counts, int32_t nsub, const memfine_dims* dims, const memfine_budget* budget,
                            memfine_plan_info* info) {
  return plan_any(counts, nsub, dims, budget, info, nullptr, false);
}

memfine_status memfine_plan_stream(const int32_t* counts, int32_t nsub, const memfine_dims* dims,
                                   const memfine_budget* budget, memfine_plan_info* info, void* stream) {
  return plan_any(counts, nsub, dims, budget, info, (cudaStream_t)stream, true);
}

memfine_status plan_host(const int32_t* counts, int32_t nsub, const memfine_dims* dims, const memfine_budget* budget,
                         memfine_plan_info* info) {
  PlanParams p;
  if (int rc = budget_to_params(dims, budget, nsub, &p)) return (memfine_status)rc;
  // Host counts: same evaluation on the CPU.
  std::vector<int64_t> sub((size_t)p.EP * nsub, 0);
  int El = p.E / p.EP;
  for (int src = 0; src < p.EP; src++)
    for (int j = 0; j < nsub; j++)
      for (int e = 0; e < p.E; e++) sub[(size_t)(e / El) * nsub + j] += counts[((int64_t)src * nsub + j) * p.E + e];
  return (memfine_status)plan_from_subsums(sub.data(), p, info);
}

// MEMFINE_MODEL_IMPL: smallest bin whose exact workspace high-water fits the budget (host).
memfine_status plan_impl(const int32_t* counts_host, int32_t nsub, const memfine_dims* dims,
                         const memfine_budget* budget, memfine_plan_info* info) {
  memfine_budget paper = *budget;
  paper.model = MEMFINE_MODEL_PAPER;
  paper.rule = MEMFINE_RULE_EQ9;
  memfine_status st = plan_host(counts_host, nsub, dims, &paper, info);
  if (st != MEMFINE_OK && st != MEMFINE_ERR_INFEASIBLE) return st;
  static const int32_t kDefaultBins[4] = {1, 2, 4, 8};
  const int32_t* bins = budget->bins ? budget->bins : kDefaultBins;
  int nb = budget->bins ? budget->nbins : 4;
  for (int i = 0; i < nb; i++)
    if (nsub % bins[i]) return MEMFINE_ERR_INVALID_ARG;
  long double Bl = (long double)budget->alpha * (long double)budget->gpu_capacity_bytes;
  uint64_t B = Bl >= 18446744073709551615.0L ? ~0ull : (uint64_t)floorl(Bl);
  uint64_t used = budget->static_bytes + budget->other_act_bytes;
  if (B <= used) return MEMFINE_ERR_INFEASIBLE;
  uint64_t room = B - used;
  auto ws_of = [&](int Cb) {
    uint64_t mx = 0;
    memfine_dims d = *dims;
    for (int r = 0; r < dims->ep_size; r++) {
      d.ep_rank = r;
      uint64_t w = 0;
      memfine_workspace_bytes(counts_host, nsub, &d, Cb, budget->pass == MEMFINE_FWD ? MEMFINE_FWD : MEMFINE_BWD, &w);
      mx = std::max(mx, w);
    }
    return mx;
  };
  int C = -1;
  uint64_t wsC = 0;
  for (int i = 0; i < nb && C < 0; i++) {
    uint64_t w = ws_of(bins[i]);
    if (w <= room) { C = bins[i]; wsC = w; }
  }
  info->clamped = 0;
  info->feasible = 1;
  if (C < 0) {
    C = bins[nb - 1];
    wsC = ws_of(C);
    info->clamped = 1;
    info->feasible = 0;
  }
  info->C = C;
  info->exact_peak = 1;
  info->predicted_peak_bytes = wsC;
  // s_chunk_max for the chosen C (paper quantity, exact because C | nsub)
  int El = dims->num_experts / dims->ep_size, per = nsub / C, E = dims->num_experts;
  int64_t mx = 0;
  for (int r = 0; r < dims->ep_size; r++)
    for (int jc = 0; jc < C; jc++) {
      int64_t sum = 0;
      for (int src = 0; src < dims->ep_size; src++)
        for (int j = jc * per; j < (jc + 1) * per; j++)
          for (int e = r * El; e < (r + 1) * El; e++) sum += counts_host[((int64_t)src * nsub + j) * E + e];
      mx = std::max(mx, sum);
    }
  info->s_chunk_max = mx;
  return MEMFINE_OK;
}

memfine_status memfine_workspace_bytes(const int32_t* counts_host, int32_t nsub, const memfine_dims* dims, int32_t C,
                                       int32_t pass, uint64_t* bytes) {
  if (!dims_ok(dims) || !bytes || C < 1 || C > kMaxSub || (pass != MEMFINE_FWD && pass != MEMFINE_BWD))
    return MEMFINE_ERR_INVALID_ARG;
  const memfine_dims& d = *dims;
  int El = d.num_experts / d.ep_size;
  int64_t rows_pad_max = 0, send_max = 0;
  if (counts_host) {
    if (nsub < 1 || nsub > kMaxSub || nsub % C) return MEMFINE_ERR_INVALID_ARG;
    std::vector<int64_t> rows, rows_pad, send;
    chunk_rows(counts_host, nsub, d, C, d.ep_rank, rows, rows_pad, &send);
    for (int j = 0; j < C; j++) {
      rows_pad_max = std::max(rows_pad_max, rows_pad[j]);
      send_max = std::max(send_max, send[j]);
    }
  } else {
    int64_t Tm = tmax_chunk(d, C);
    int64_t total = (int64_t)d.ep_size * Tm * d.topk;  // duplicates in a token's top-k are legal
    rows_pad_max = round_up64(total + (int64_t)El * (kRowAlign - 1), kRowAlign);
    send_max = Tm * d.topk;
  }
  Layout L = carve(d, C, pass, nullptr, rows_pad_max, ep_path(d) ? send_max : 0);
  *bytes = L.total;
  return MEMFINE_OK;
}

memfine_status memfine_a2a_plan(const int32_t* counts_host, int32_t nsub, const memfine_dims* dims, int32_t C,
                                int32_t chunk, int64_t* send_rows, int64_t* recv_rows, int64_t* recv_offsets,
                                int64_t* rows_padded) {
  if (!counts_host || !dims_ok(dims) || C < 1 || C > kMaxSub || nsub < 1 || nsub > kMaxSub || nsub % C ||
      chunk < 0 || chunk >= C || !send_rows || !recv_rows || !recv_offsets)
    return MEMFINE_ERR_INVALID_ARG;
  const memfine_dims& d = *dims;
  int E = d.num_experts, EP = d.ep_size, El = E / EP, per = nsub / C;
  std::vector<int> agg((size_t)EP * C * E, 0);  // [EP][C][E]
  for (int src = 0; src < EP; src++)
    for (int j = 0; j < nsub; j++)
      for (int e = 0; e < E; e++) agg[((size_t)src * C + j / per) * E + e] += counts_host[((int64_t)src * nsub + j) * E + e];
  EpChunk t = ep_chunk_table(d, agg.data(), C, chunk);
  for (int peer = 0; peer < EP; peer++) {
    send_rows[peer] = t.send_off[(peer + 1) * El] - t.send_off[peer * El];
    int64_t r = 0;
    for (int el = 0; el < El; el++) {
      r += t.recv_cnt[(size_t)peer * El + el];
      recv_offsets[(size_t)peer * El + el] = t.recv_off[(size_t)peer * El + el];
    }
    recv_rows[peer] = r;
  }
  if (rows_padded) *rows_padded = t.rows_pad;
  return MEMFINE_OK;
}

memfine_status memfine_moe_fwd(memfine_handle_t h, const void* x, const int32_t* ids, const float* w,
                               const void* w_gate, const void* w_up, const void* w_down, int32_t C, void* y, void* ws,
                               uint64_t ws_bytes, void* stream) {
  if (!h || C < 1 || C > kMaxSub) return MEMFINE_ERR_INVALID_ARG;
  if (h->d.tokens > 0 && (!x || !ids || !w || !y)) return MEMFINE_ERR_INVALID_ARG;
  if (!w_gate || !w_up || !w_down || !ws) return MEMFINE_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  Nvtx call_range("memfine_moe_fwd");
  PdlOff pdl_off(ep_slots(h->d, C) == 2);
  begin_call(h, C, MEMFINE_FWD, ws_bytes, st);
  if (ep_path(h->d)) return memfine_ep_fwd(h, x, ids, w, w_gate, w_up, w_down, C, y, ws, ws_bytes, st);
  if (h->d.dtype != MEMFINE_FP32)
    return fwd_ep1<__nv_bfloat16>(h, (const __nv_bfloat16*)x, ids, w, w_gate, w_up, w_down, C, (__nv_bfloat16*)y, ws,
                                  ws_bytes, st);
  return fwd_ep1<float>(h, (const float*)x, ids, w, w_gate, w_up, w_down, C, (float*)y, ws, ws_bytes, st);
}

memfine_status memfine_moe_bwd(memfine_handle_t h, const void* dy, const void* x, const int32_t* ids, const float* w,
                               const void* w_gate, const void* w_up, const void* w_down, int32_t C, void* dx,
                               float* dw_gate, float* dw_up, float* dw_down, float* dscore, int32_t accumulate_dw,
                               void* ws, uint64_t ws_bytes, void* stream) {
  if (!h || C < 1 || C > kMaxSub) return MEMFINE_ERR_INVALID_ARG;
  if (h->d.tokens > 0 && (!dy || !x || !ids || !w || !dx)) return MEMFINE_ERR_INVALID_ARG;
  if (!w_gate || !w_up || !w_down || !dw_gate || !dw_up || !dw_down || !ws) return MEMFINE_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  Nvtx call_range("memfine_moe_bwd");
  PdlOff pdl_off(ep_slots(h->d, C) == 2);
  begin_call(h, C, MEMFINE_BWD, ws_bytes, st);
  if (ep_path(h->d))
    return memfine_ep_bwd(h, dy, x, ids, w, w_gate, w_up, w_down, C, dx, dw_gate, dw_up, dw_down, dscore,
                          accumulate_dw, ws, ws_bytes, st);
  if (h->d.dtype != MEMFINE_FP32)
    return bwd_ep1<__nv_bfloat16>(h, (const __nv_bfloat16*)dy, (const __nv_bfloat16*)x, ids, w, w_gate, w_up, w_down,
                                  C, (__nv_bfloat16*)dx, dw_gate, dw_up, dw_down, dscore, accumulate_dw, ws, ws_bytes,
                                  st);
  return bwd_ep1<float>(h, (const float*)dy, (const float*)x, ids, w, w_gate, w_up, w_down, C, (float*)dx, dw_gate,
                        dw_up, dw_down, dscore, accumulate_dw, ws, ws_bytes, st);
}

// ---------------------------------------------------------------- MXFP8 (N4, reading R28)
memfine_status memfine_mx_weights_bytes(const memfine_dims* dims, uint64_t* bytes) {
  if (!dims_ok(dims) || !bytes || dims->dtype != MEMFINE_MXFP8) return MEMFINE_ERR_INVALID_ARG;
  *bytes = mx_weights_layout(*dims, nullptr).total;
  return MEMFINE_OK;
}

memfine_status memfine_mx_quantize_weights(memfine_handle_t h, const void* w_gate, const void* w_up,
                                           const void* w_down, void* wq, uint64_t wq_bytes, void* stream) {
  if (!h || h->d.dtype != MEMFINE_MXFP8 || !w_gate || !w_up || !w_down || !wq) return MEMFINE_ERR_INVALID_ARG;
  const memfine_dims& d = h->d;
  MxWeightsLayout W = mx_weights_layout(d, wq);
  if (wq_bytes < W.total) return MEMFINE_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  const int El = d.num_experts / d.ep_size, hd = d.hidden, g = d.ffn;
  auto q = [&](int i) { return const_cast<uint8_t*>(W.op[i].q); };
  auto sf = [&](int i) { return const_cast<uint8_t*>(W.op[i].sf); };
  const __nv_bfloat16 *wg = (const __nv_bfloat16*)w_gate, *wu = (const __nv_bfloat16*)w_up,
                      *wd = (const __nv_bfloat16*)w_down;
  // W_gate / W_up: rows (blocks along h) and transposed (blocks along g) from one read each
  launch_mx_quant_dual(wg, El, g, hd, q(0), sf(0), q(3), sf(3), st);
  launch_mx_quant_dual(wu, El, g, hd, q(1), sf(1), q(4), sf(4), st);
  launch_mx_quant_rows(wd, g, (int64_t)El * hd, nullptr, g, q(2), sf(2), st);
  h->mx_w = (const uint8_t*)wq;
  return latch_cuda(h);
}

memfine_status memfine_mx_quantize(const void* src, int64_t rows, int32_t K, void* codes, void* scales, void* stream) {
  if (!src || !codes || !scales || rows < 0 || rows % 128 || K <= 0 || K % 128) return MEMFINE_ERR_INVALID_ARG;
  launch_mx_quant_rows((const __nv_bfloat16*)src, K, rows, nullptr, K, (uint8_t*)codes, (uint8_t*)scales,
                       (cudaStream_t)stream);
  return cudaGetLastError() == cudaSuccess ? MEMFINE_OK : MEMFINE_ERR_CUDA;
}

// ---------------------------------------------------------------- router (N3)
namespace {
// Router scratch (per handle, allocated on first use): the GEMM-written logits [T][E4] (fp32, row stride a
// multiple of 16 B for TMA), d_logits, the dense bf16 hi / lo d_logits [T_pad][E8] (rows and columns past
// T, E stay zero: the dW_r GEMM's K loop runs over whole 128-row blocks), the one-segment metadata the
// expert-GEMM scheduler reads (seg, pseg, info), and the fp32 path's counting sort.
struct RouterScratch {
  float* logits;
  float* dlog;
  __nv_bfloat16* dhi;
  __nv_bfloat16* dlo;
  int* gseg;     // {0, T_pad}
  int* gpseg;    // {0, pairs}
  int* ginfo;    // kInfoWords
  ChunkMeta m;
  int64_t rows_cap, T_pad;
  int E4, E8;
};
memfine_status router_scratch(memfine_handle_s* h, RouterScratch* rs) {
  const memfine_dims& d = h->d;
  const int E = d.num_experts, k = d.topk;
  const int64_t T = d.tokens, NB = std::max<int64_t>(1, ceil_div64(T, kTokPerBlk));
  const int64_t rows_cap = round_up64(T * k + (int64_t)E * (kRowAlign - 1), kRowAlign);
  const int64_t T_pad = round_up64(std::max<int64_t>(T, 1), kRowAlign);
  const int E4 = (int)round_up64(E, 4), E8 = (int)round_up64(E, 8);
  auto layout = [&](Bump& b, RouterScratch* o) {
    float* lg = b.take<float>((uint64_t)T * E4);
    float* dl = b.take<float>((uint64_t)T * k);
    __nv_bfloat16* hi = b.take<__nv_bfloat16>((uint64_t)T_pad * E8);
    __nv_bfloat16* lo = b.take<__nv_bfloat16>((uint64_t)T_pad * E8);
    int* gs = b.take<int>(2);
    int* gp = b.take<int>(2);
    int* gi = b.take<int>(kInfoWords);
    ChunkMeta m{};
    m.blk_cnt = b.take<int>((uint64_t)NB * E);
    m.exp_cnt = b.take<int>(E + 1);
    m.recv_cnt = b.take<int>(E + 1);
    m.seg = b.take<int>(E + 1);
    m.pseg = b.take<int>(E + 1);
    m.info = b.take<int>(kInfoWords);
    m.dest_of = b.take<int>((uint64_t)T * k);
    m.src_of = b.take<int>((uint64_t)rows_cap);
    if (o) *o = RouterScratch{lg, dl, hi, lo, gs, gp, gi, m, rows_cap, T_pad, E4, E8};
  };
  Bump b(nullptr);
  layout(b, nullptr);
  if (b.off > h->router_bytes) {
    if (h->router_scratch) cudaFree(h->router_scratch);
    h->router_scratch = nullptr;
    h->router_bytes = 0;
    MF_CUDA_OK(cudaMalloc((void**)&h->router_scratch, b.off));
    h->router_bytes = b.off;
    Bump c(h->router_scratch);
    layout(c, rs);
    // zero padding of hi / lo, and the scheduler's metadata of the one T-row segment (fixed per handle)
    MF_CUDA_OK(cudaMemset(rs->dhi, 0, sizeof(__nv_bfloat16) * (size_t)T_pad * E8));
    MF_CUDA_OK(cudaMemset(rs->dlo, 0, sizeof(__nv_bfloat16) * (size_t)T_pad * E8));
    const int mt = (int)(T_pad / kRowAlign), pairs = (mt + 1) / 2;
    int meta[4 + kInfoWords] = {0, (int)T_pad, 0, pairs};
    meta[4 + kInfoRows] = (int)T;
    meta[4 + kInfoRowsPad] = (int)T_pad;
    meta[4 + kInfoSend] = (int)T;
    meta[4 + kInfoSkip] = 0;
    meta[4 + kInfoPairs] = pairs;
    MF_CUDA_OK(cudaMemcpy(rs->gseg, meta, sizeof(int) * 2, cudaMemcpyHostToDevice));
    MF_CUDA_OK(cudaMemcpy(rs->gpseg, meta + 2, sizeof(int) * 2, cudaMemcpyHostToDevice));
    MF_CUDA_OK(cudaMemcpy(rs->ginfo, meta + 4, sizeof(int) * kInfoWords, cudaMemcpyHostToDevice));
    return MEMFINE_OK;
  }
  Bump c(h->router_scratch);
  layout(c, rs);
  return MEMFINE_OK;
}

// The router's dense contractions on the expert-GEMM kernels: one "expert" whose rows are the T tokens.
GemmProblem<__nv_bfloat16> router_problem(const memfine_handle_s* h, const RouterScratch& rs) {
  GemmProblem<__nv_bfloat16> p{};
  p.El = 1;
  p.h = h->d.num_experts;    // N of the logits GEMM, M of the dW_r GEMM
  p.g = h->d.hidden;         // K of the logits GEMM, N of the dW_r GEMM
  p.rows_cap = rs.T_pad;
  p.rows_in = h->d.tokens;
  p.seg = rs.gseg;
  p.pseg = rs.gpseg;
  p.info = rs.ginfo;
  return p;
}
}  // namespace

memfine_status memfine_router_fwd(memfine_handle_t h, const void* x, const void* w_router, int32_t* ids,
                                  float* scores, float* logits, void* stream) {
  if (!h || !w_router || (h->d.tokens > 0 && (!x || !ids || !scores))) return MEMFINE_ERR_INVALID_ARG;
  const memfine_dims& d = h->d;
  cudaStream_t st = (cudaStream_t)stream;
  RouterScratch rs;
  if (int rc = router_scratch(h, &rs)) return (memfine_status)rc;
  if (d.dtype != MEMFINE_FP32) {
    if (d.tokens == 0) return MEMFINE_OK;
    // logits = x W_r^T: a DOWN launch (A = x [T][h] K-major, B = W_r [1][E][h]) storing fp32 [T][E4]
    GemmProblem<__nv_bfloat16> p = router_problem(h, rs);
    p.kind = GK_DOWN;
    p.A = (__nv_bfloat16*)x;
    p.Wd = (const __nv_bfloat16*)w_router;
    p.O = (__nv_bfloat16*)rs.logits;
    p.out_f32 = 1;
    p.ld_out = rs.E4;
    if (int rc = run_gemm<__nv_bfloat16>(h, p, st)) return (memfine_status)rc;
    launch_router_topk(rs.logits, rs.E4, d.tokens, d.num_experts, d.topk, ids, scores, logits, st);
    h->last.kernel_launches += 1;
    return latch_cuda(h);
  }
  float* lg = logits ? logits : rs.logits;
  launch_router_fwd<float>((const float*)x, (const float*)w_router, d.tokens, d.num_experts, d.hidden, d.topk, lg,
                           ids, scores, st);
  return latch_cuda(h);
}

memfine_status memfine_router_bwd(memfine_handle_t h, const void* x, const void* w_router, const int32_t* ids,
                                  const float* scores, const float* dscore, void* dx, int32_t accumulate_dx,
                                  float* dw_router, int32_t accumulate_dw, void* stream) {
  if (!h || !w_router || !dw_router || (h->d.tokens > 0 && (!x || !ids || !scores || !dscore || !dx)))
    return MEMFINE_ERR_INVALID_ARG;
  const memfine_dims& d = h->d;
  cudaStream_t st = (cudaStream_t)stream;
  RouterScratch rs;
  if (int rc = router_scratch(h, &rs)) return (memfine_status)rc;
  const int E = d.num_experts, k = d.topk;
  if (d.dtype != MEMFINE_FP32) {
    if (d.tokens == 0) {
      if (!accumulate_dw) MF_CUDA_OK(cudaMemsetAsync(dw_router, 0, sizeof(float) * (size_t)E * d.hidden, st));
      return MEMFINE_OK;
    }
    launch_router_bwd_rows_bf16((const __nv_bfloat16*)w_router, ids, scores, dscore, d.tokens, E, d.hidden, k,
                                rs.dlog, rs.dhi, rs.dlo, rs.E8, (__nv_bfloat16*)dx, accumulate_dx, st);
    h->last.kernel_launches += 1;
    // dW_r (+)= d_logits^T x = hi^T x + lo^T x: two WGRAD_DOWN launches (K = the T_pad token rows)
    GemmProblem<__nv_bfloat16> p = router_problem(h, rs);
    p.kind = GK_WGRAD_DOWN;
    p.A = (__nv_bfloat16*)x;
    p.ld_a = rs.E8;
    p.dWd = dw_router;
    p.DY = rs.dhi;
    p.wgrad_beta = accumulate_dw ? 1 : 0;
    if (int rc = run_gemm<__nv_bfloat16>(h, p, st)) return (memfine_status)rc;
    p.DY = rs.dlo;
    p.wgrad_beta = 1;
    if (int rc = run_gemm<__nv_bfloat16>(h, p, st)) return (memfine_status)rc;
    return latch_cuda(h);
  }
  // fp32: counting sort of the copies by expert (stable): segment e = rows [seg[e], seg[e] + cnt[e])
  int NB = (int)ceil_div64(d.tokens, kTokPerBlk);
  if (NB) {
    launch_dispatch_hist(ids, 0, d.tokens, k, E, rs.m, h->status_d, st);
    launch_dispatch_scan(NB, E, E, 0, rs.rows_cap, rs.m, nullptr, nullptr, 0, st);
    launch_dispatch_index(ids, nullptr, 0, d.tokens, k, E, rs.m, rs.m.src_of, nullptr, st);
  } else {
    MF_CUDA_OK(cudaMemsetAsync(rs.m.seg, 0, sizeof(int) * (E + 1), st));
    MF_CUDA_OK(cudaMemsetAsync(rs.m.recv_cnt, 0, sizeof(int) * (E + 1), st));
  }
  launch_router_bwd<float>((const float*)x, (const float*)w_router, ids, scores, dscore, d.tokens, E, d.hidden, k,
                             rs.dlog, (float*)dx, accumulate_dx, dw_router, accumulate_dw, rs.m, st);
  return latch_cuda(h);
}

memfine_status memfine_sync(memfine_handle_t h, void* stream) {
  if (!h) return MEMFINE_ERR_INVALID_ARG;
  if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) { cudaGetLastError(); return MEMFINE_ERR_CUDA; }
  int e = __atomic_exchange_n(h->status_h, 0, __ATOMIC_SEQ_CST);
  if (e) {
    h->last.device_error = e;
    fflush(stdout);   // device-side diagnostics (printf of the timed-out waits) before the caller reports
  }
  // stats: rows per chunk and the workspace high-water they imply
  uint64_t maxpad = 0;
  for (int j = 0; j < h->last.C && j < kMaxSub; j++) {
    h->last.rows[j] = h->rows_h[j];
    h->last.rows_padded[j] = h->rows_h[kMaxSub + j];
    maxpad = std::max<uint64_t>(maxpad, (uint64_t)h->rows_h[kMaxSub + j]);
  }
  if (h->last.C) h->last.workspace_used_bytes = h->last_meta + maxpad * h->last_row_bytes;
  if (!e && h->last.workspace_used_bytes > h->last.workspace_given_bytes && h->last.C) e = MEMFINE_ERR_WORKSPACE;
  return (memfine_status)e;
}

memfine_status memfine_last_stats(memfine_handle_t h, memfine_stats* out) {
  if (!h || !out) return MEMFINE_ERR_INVALID_ARG;
  *out = h->last;
  return MEMFINE_OK;
}

memfine_status memfine_profile_enable(memfine_handle_t h, int32_t enable) {
  if (!h) return MEMFINE_ERR_INVALID_ARG;
  h->prof = enable ? 1 : 0;
  return MEMFINE_OK;
}

memfine_status memfine_profile_read(memfine_handle_t h, memfine_profile* out) {
  if (!h || !out) return MEMFINE_ERR_INVALID_ARG;
  memset(out, 0, sizeof *out);
  for (auto& r : h->recs) {
    if (cudaEventSynchronize(r.b) != cudaSuccess) { cudaGetLastError(); return MEMFINE_ERR_CUDA; }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    out->launches[r.slot] += 1;
    out->ms[r.slot] += ms;
  }
  h->recs.clear();
  h->pool_used = 0;
  return MEMFINE_OK;
}

memfine_status memfine_set_debug(memfine_handle_t h, int32_t enable) {
  if (!h) return MEMFINE_ERR_INVALID_ARG;
  h->debug = enable ? 1 : 0;
  return MEMFINE_OK;
}

memfine_status memfine_debug_rows(memfine_handle_t h, int32_t chunk, int32_t* src_of_host, int64_t cap, int64_t* n) {
  if (!h || !n || chunk < 0 || chunk >= (int)h->dbg_src.size()) return MEMFINE_ERR_INVALID_ARG;
  const auto& v = h->dbg_src[chunk];
  *n = (int64_t)v.size();
  if (src_of_host) {
    if (cap < (int64_t)v.size()) return MEMFINE_ERR_INVALID_ARG;
    std::copy(v.begin(), v.end(), src_of_host);
  }
  return MEMFINE_OK;
}

memfine_status memfine_debug_mx(memfine_handle_t h, int32_t chunk, int32_t which, uint8_t* codes_host,
                                uint8_t* scales_host, int64_t cap_codes, int64_t* rows, int64_t* cols) {
  if (!h || !rows || !cols || chunk < 0 || chunk >= (int)h->dbg_mx.size() || which < 0 || which >= 6)
    return MEMFINE_ERR_INVALID_ARG;
  const auto& D = h->dbg_mx[chunk][which];
  *rows = D.rows;
  *cols = D.cols;
  if (codes_host) {
    if (cap_codes < (int64_t)D.q.size() || !scales_host) return MEMFINE_ERR_INVALID_ARG;
    std::copy(D.q.begin(), D.q.end(), codes_host);
    std::copy(D.sf.begin(), D.sf.end(), scales_host);
  }
  return MEMFINE_OK;
}

memfine_status memfine_debug_perm(memfine_handle_t h, int32_t chunk, int64_t* perm_host, int64_t cap, int64_t* n) {
  if (!h || !n || chunk < 0 || chunk >= (int)h->debug_perm.size()) return MEMFINE_ERR_INVALID_ARG;
  const auto& v = h->debug_perm[chunk];
  *n = (int64_t)v.size();
  if (perm_host) {
    if (cap < (int64_t)v.size()) return MEMFINE_ERR_INVALID_ARG;
    for (size_t i = 0; i < v.size(); i++) perm_host[i] = v[i];
  }
  return MEMFINE_OK;
}

}  // extern "C"
