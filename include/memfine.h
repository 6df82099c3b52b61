/*
 * memfine.h — C ABI of libmemfine.so, the B200 (sm_100a) MemFine chunked MoE layer.
 *
 * MemFine (arXiv 2511.21431, PAPER.md) trains MoE layers without capping expert
 * capacity by running dispatch -> expert -> combine in C token chunks (FCDA,
 * Eq. 6), recomputing each chunk's expert activations just
 * before its gradients (Eq. 7), with C chosen by the paper's
 * activation-memory model under a memory threshold (MACT, Eqs. 8-9 and bins,
 * PAPER.md:191-206).
 *
 * Conventions (all entry points):
 *  - Plain C types and raw pointers only.  "dev" pointers are CUDA device
 *    pointers on the handle's device; "host" pointers are CPU memory.
 *  - The caller owns every buffer, including the workspace.  The library owns
 *    only small per-handle metadata (counts mirror, status word, NCCL comm).
 *  - Stream-ordered: kernels are enqueued on the given cudaStream_t (passed as
 *    void*; NULL = legacy default stream).  One host thread per handle.
 *  - No exception or longjmp crosses the ABI; every call returns a status code.
 *    Synchronous argument checks return immediately.  Errors detected on the
 *    device (bad expert id, workspace too small) are latched in the handle and
 *    returned by the next memfine_sync() (or by the call itself when it already
 *    synchronises, e.g. every call with ep_size > 1).
 *  - There is no CPU fallback: every compute step runs in the library's CUDA
 *    kernels; on a machine without a usable sm_100 device, memfine_create
 *    returns MEMFINE_ERR_CUDA.
 *
 * Symbols (Table 1; SURVEY.md symbol table):
 *   T tokens per rank (b*s), h hidden, g expert FFN size (g_e), E experts,
 *   k top-k (t_k), EP expert-parallel size (e), E_l = E/EP local experts,
 *   C chunk count (the paper's c of Eq. 9 — NOT its context-parallel c).
 */
#ifndef MEMFINE_H
#define MEMFINE_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MEMFINE_ABI_VERSION 2

/* Status codes.  1 and 2 mirror the SPEC CLI exit codes. */
typedef enum {
    MEMFINE_OK = 0,
    MEMFINE_ERR_INVALID_ARG = 1,   /* null pointer, bad dims, bad bins, C < 1, ...        */
    MEMFINE_ERR_INFEASIBLE = 2,    /* static + other >= alpha*M^GPU, or s'_max <= 0        */
    MEMFINE_ERR_ROUTING = 3,       /* an expert id outside [0, E) (device-detected)        */
    MEMFINE_ERR_CUDA = 4,          /* CUDA runtime error / no sm_100 device                */
    MEMFINE_ERR_NCCL = 5,          /* NCCL missing or failed                               */
    MEMFINE_ERR_WORKSPACE = 6,     /* workspace smaller than memfine_workspace_bytes()     */
    MEMFINE_ERR_UNSUPPORTED = 7    /* shape outside what the kernels support (see below)  */
} memfine_status;

enum { MEMFINE_BF16 = 0, MEMFINE_FP32 = 1, MEMFINE_MXFP8 = 2 }; /* memfine_dims.dtype */
enum { MEMFINE_RULE_EXACT = 0, MEMFINE_RULE_EQ9 = 1 }; /* memfine_budget.rule (0 = EXACT, the default) */
enum { MEMFINE_FWD = 0, MEMFINE_BWD = 1 };           /* workspace pass      */
enum { MEMFINE_MODEL_PAPER = 0, MEMFINE_MODEL_IMPL = 1 }; /* memfine_budget.model */

typedef struct memfine_handle_s* memfine_handle_t;

/* Layer dimensions.  Supported: tokens >= 0; hidden % 64 == 0; ffn % 64 == 0;
 * 1 <= topk <= num_experts; num_experts % ep_size == 0; 0 <= ep_rank < ep_size. */
typedef struct {
    int64_t tokens;       /* T: tokens on this rank (every rank the same T)          */
    int32_t hidden;       /* h                                                       */
    int32_t ffn;          /* g (= g_e)                                               */
    int32_t num_experts;  /* E (global)                                              */
    int32_t topk;         /* k (= t_k)                                               */
    int32_t ep_size;      /* EP; ranks hold contiguous expert blocks (reading R4)    */
    int32_t ep_rank;      /* this rank                                               */
    int32_t dtype;        /* MEMFINE_BF16 (bf16 storage, fp32 accumulate, tcgen05)    *
                           * MEMFINE_FP32 (fp32 everywhere, CUDA-core FFMA; <=1e-5)   *
                           * MEMFINE_MXFP8 (bf16 storage; the gate/up, down and dX   *
                           *   GEMMs on MXFP8 operands, see memfine_mx_*; hidden,     *
                           *   ffn % 128 == 0; with EP the rows travel in bf16 and are *
                           *   quantised on arrival; both EP transports)               */
    int32_t flags;        /* MEMFINE_FLAG_* (0 = none).  Part of the workspace layout:  *
                           * memfine_workspace_bytes and the fwd/bwd calls must see the *
                           * same flags.                                                */
} memfine_dims;

/* memfine_dims.flags
 *  MEMFINE_FLAG_OVERLAP (ep_size > 1, C > 1; either transport): pipeline the FCDA chunk loop
 *    over two streams, "the per-chunk dispatch and combine overlapped chunk by chunk with the
 *    grouped GEMM" (north star; Eq. 6 / 7 order is unchanged): chunk j+1's
 *    permute + dispatch all-to-allv and chunk j-1's combine all-to-allv + unpermute run on the
 *    handle's high-priority comm stream while chunk j's GEMMs run on the caller's stream.  The
 *    workspace holds two slots of the exchanged rows (send staging, X_disp, dY_disp, per-row
 *    scores and metadata); G||U and a stay single (compute-only).  In the forward o is written
 *    over X_disp, so the forward's per-row bytes do not grow; the backward's grow by 2h*D_t.
 *    With MEMFINE_EP_P2P the comm stream runs chunk j+1's permute + pushes into the peers' buffers
 *    and chunk j-1's flag wait + combine / unpermute; chunk j's GEMMs (whose epilogues store into
 *    the sources' buffers) run on the caller's stream; slot reuse is fenced by the peers' done(j-2)
 *    flags.  Ignored (layout and bytes identical to flags = 0) when ep_size == 1 (without EP_PATH),
 *    C == 1 or MXFP8.
 *  MEMFINE_FLAG_EP_PATH (ep_size == 1 only): run the expert-parallel data path - count
 *    all-gather, send staging, per-(peer, local expert) all-to-allv, combine exchange - over a
 *    1-rank NCCL communicator, every segment (including the self segment) through ncclSend /
 *    ncclRecv.  memfine_create then takes a unique id.  Results equal the EP = 1 path; this is
 *    how the NCCL transport is exercised on a single GPU (NCCL refuses two ranks on one device).
 *  MEMFINE_FLAG_MX_WGRAD (dtype MEMFINE_MXFP8; EP copy transport): the weight-gradient
 *    GEMMs also take MXFP8 operands - x, dY, dG || dU and a_w quantised columnwise (blocks of 32
 *    copies of an expert within a chunk, reading R28c) - instead of BF16 ones.  Adds the
 *    columnwise codes to the backward workspace ((h + 3g) * 33/32 bytes per row). */
enum { MEMFINE_FLAG_OVERLAP = 1, MEMFINE_FLAG_EP_PATH = 2, MEMFINE_FLAG_MX_WGRAD = 4 };

/* Memory budget for MACT (Eq. 3; Eq. 8). */
typedef struct {
    uint64_t gpu_capacity_bytes; /* M^GPU                                                  */
    double   alpha;              /* available ratio; budget B = floor(alpha * M^GPU) bytes  */
    uint64_t static_bytes;       /* M^sta (Eq. 1), supplied by the caller                   */
    uint64_t other_act_bytes;    /* the s-term of Eq. 2 (attention, norms, router), caller  */
    uint32_t m_g;                /* Eq. 2 multiplier; 1 under full recompute */
    uint32_t tp, cp;             /* the (t c) divisor of Eqs. 2 and 8; 1 on this path       */
    uint32_t micro_batch;        /* b                                                       */
    const int32_t* bins;         /* host; strictly increasing, bins[0] >= 1; NULL = {1,2,4,8}
                                                                         */
    int32_t  nbins;
    int32_t  rule;               /* MEMFINE_RULE_EXACT (0, the default): smallest bin whose true
                                    per-chunk maximum max_j s''_{r,j}(C) fits s'_max (every bin
                                    must divide nsub) - Eq. 3 holds for the chunks actually run;
                                    MEMFINE_RULE_EQ9: C = smallest bin >= ceil(s''/s'_max)
                                    (Eq. 9 + "the large bin closest to c", reading R8), the
                                    paper's estimate, which assumes the chunk maximum is s''/C
                                    (reading R11)                                            */
    int32_t  model;              /* MEMFINE_MODEL_PAPER: the paper's per-copy activation
                                    beta = D_t(2h+2g) (Table 2 rows 11-13; Eqs. 8-9 as above).
                                    MEMFINE_MODEL_IMPL: C = smallest bin whose EXACT workspace
                                    high-water (memfine_workspace_bytes, backward pass, max over
                                    EP ranks) fits B - static - other; every bin must divide
                                    nsub; s'_max / c_theory are still reported per Eqs. 8-9 and
                                    predicted_peak_bytes is that exact workspace.  Evaluated on
                                    the host (device counts are copied, 4*EP*nsub*E bytes).    */
    int32_t  pass;               /* MEMFINE_MODEL_IMPL only: size for MEMFINE_BWD (default, the
                                    larger live set) or MEMFINE_FWD (a forward-only C)          */
} memfine_budget;

/* Result of memfine_plan. */
typedef struct {
    int32_t  C;                  /* chosen chunk count                                      */
    int32_t  c_theory;           /* Eq. 9: max(1, ceil(s''_max / s'_max))                   */
    int32_t  clamped;            /* c exceeded the largest bin                */
    int32_t  feasible;           /* max_{r,j} s''_{r,j}(C) <= s'_max                        */
    int32_t  hot_rank;           /* argmax_r s''_r (lowest index on ties)                   */
    int32_t  exact_peak;         /* 1: s_chunk_max exact (C | nsub); 0: ceil(s''_max / C)   */
    int64_t  s_dd_max;           /* max_r s''_r: routed copies received by the hottest rank */
    int64_t  s_prime_max;        /* Eq. 8 in integer bytes (reading R9)                     */
    int64_t  s_chunk_max;        /* max_{r,j} s''_{r,j}(C)                                  */
    uint64_t predicted_peak_bytes; /* paper model: m_g D_t b s_chunk_max (2h+2g) / (tp cp)
                                      (Table 2 rows 11-13)                  */
} memfine_plan_info;

/* Statistics of the last fwd / bwd call on a handle (valid after memfine_sync). */
typedef struct {
    int32_t  C;
    int32_t  pass;                  /* MEMFINE_FWD / MEMFINE_BWD                            */
    int64_t  rows[64];              /* s''_{r,j}: rows this rank received per chunk (C<=64)  */
    int64_t  rows_padded[64];       /* the same, each local expert padded to 128 rows       */
    uint64_t workspace_used_bytes;  /* high-water of the workspace bump allocator           */
    uint64_t workspace_given_bytes;
    int32_t  device_error;          /* latched memfine_status from the device, or 0         */
    int32_t  gemm_launches;         /* kernels launched by the last call                    */
    int32_t  kernel_launches;
    int32_t  comm_ops;              /* point-to-point operations of the call's exchanges (EP path,
                                       copy transport: ncclSend + ncclRecv calls, or device copies
                                       in an in-process group); all chunks                      */
} memfine_stats;

/* ---------------------------------------------------------------------------------- */

int32_t     memfine_abi_version(void);
const char* memfine_status_str(memfine_status s);

/* NCCL bootstrap for ep_size > 1: rank 0 calls this, broadcasts the 128 bytes over
 * the caller's process group (e.g. torch.distributed), every rank passes them to
 * memfine_create.  Returns MEMFINE_ERR_NCCL if libnccl.so.2 cannot be loaded. */
memfine_status memfine_nccl_unique_id(uint8_t out_id[128]);

/* Create a handle on the CURRENT CUDA device.  nccl_unique_id: host, 128 bytes from
 * memfine_nccl_unique_id(), NULL iff dims->ep_size == 1 and MEMFINE_FLAG_EP_PATH is not
 * set.  Collective over the EP
 * group when ep_size > 1 (ncclCommInitRank).  Fails with MEMFINE_ERR_CUDA if the
 * current device is not sm_100. */
memfine_status memfine_create(const memfine_dims* dims, const uint8_t* nccl_unique_id,
                              memfine_handle_t* out);
memfine_status memfine_destroy(memfine_handle_t h);

/* In-process EP group: ep_size ranks of one layer in ONE process on ONE device, one host
 * thread per rank, exchanging rows with stream-ordered device copies instead of NCCL (the
 * same send layout, per-(peer, local expert) segments and receive offsets as the NCCL path).
 * For validating the expert-parallel data path on a single GPU; every rank's calls must be
 * made concurrently from its own thread (they rendezvous like collectives).  The group must
 * outlive its handles. */
typedef struct memfine_group_s* memfine_group_t;
memfine_status memfine_local_group_create(int32_t nranks, memfine_group_t* out);
memfine_status memfine_local_group_destroy(memfine_group_t g);
memfine_status memfine_create_local(const memfine_dims* dims, memfine_group_t group, memfine_handle_t* out);

/* EP transport of a handle (ep_size > 1).
 *  MEMFINE_EP_COPY (default): the permute writes a send buffer; the dispatch / combine
 *    all-to-allv move rows between ranks (ncclSend/Recv per (peer, local expert) segment, or
 *    stream-ordered device copies inside an in-process group).
 *  MEMFINE_EP_P2P: the exchange is fused into the kernels over peer memory:
 *    the permute kernel stores each token row straight into the receiving rank's expert-major
 *    buffer, and the down / dX GEMM epilogues store each output row straight into its source
 *    rank's combine buffer as the tile is produced; ranks fence with events (in-process group).
 *    ep_size <= 16.  In-process groups map peers directly; across processes (NCCL handles) the
 *    workspace must first be registered with memfine_register_workspace (or, without NCCL, exported
 *    and imported: memfine_create_ipc), and ranks fence with epoch-stamped per-peer flags in each
 *    other's sync areas, waited on by device kernels (no host synchronisation inside a call).
 * The workspace layout and size are the same for both (with MEMFINE_FLAG_OVERLAP: two slots for either,
 * sized by memfine_workspace_bytes from the dims). */
enum { MEMFINE_EP_COPY = 0, MEMFINE_EP_P2P = 1 };
memfine_status memfine_set_ep_transport(memfine_handle_t h, int32_t transport);

/* MEMFINE_FLAG_OVERLAP only: number of SMs the expert GEMMs leave free for the comm stream's
 * kernels (NCCL send/recv, permute, unpermute) while chunks overlap; 0 (default) = the GEMMs
 * take every SM and the comm kernels interleave at kernel boundaries (the comm stream has the
 * highest priority).  0 <= n < SM count, else MEMFINE_ERR_INVALID_ARG. */
memfine_status memfine_set_comm_sms(memfine_handle_t h, int32_t n);

/* Collective over the EP group (NCCL handles): export the device allocation holding `ws`
 * through CUDA IPC, all-gather (handle, offset) over the handle's communicator and map every
 * peer's workspace (cudaIpcMemLazyEnablePeerAccess).  MEMFINE_EP_P2P calls must then pass this
 * same ws (MEMFINE_ERR_INVALID_ARG otherwise).  For in-process groups and ep_size == 1 it only
 * records ws.  Synchronises `stream`. */
memfine_status memfine_register_workspace(memfine_handle_t h, void* ws, uint64_t ws_bytes, void* stream);

/* N1 across processes WITHOUT NCCL (EP data flow PAPER.md:30, the count exchange
 * PAPER.md:200): an expert-parallel handle whose only transport is the device-planned peer-memory
 * exchange (MEMFINE_EP_P2P), for ranks in separate processes that exchange their workspace mappings
 * through the caller's own channel (e.g. torch.distributed over gloo) - two processes sharing one
 * device included.  dims->ep_size in [2, 16]; flags without MEMFINE_FLAG_EP_PATH (MEMFINE_FLAG_OVERLAP selects
 * the two-slot, two-stream chunk pipeline of the exchange).
 * memfine_route_counts on such a handle fills only this rank's rows of counts_dev (the caller
 * all-gathers them to size the workspace); the layer calls themselves need no host collective (the
 * counts travel through the peers' sync areas).  memfine_set_ep_transport accepts MEMFINE_EP_P2P only. */
memfine_status memfine_create_ipc(const memfine_dims* dims, memfine_handle_t* out);
#define MEMFINE_IPC_RECORD_BYTES 256
/* This rank's mapping record (MEMFINE_IPC_RECORD_BYTES bytes, opaque: CUDA IPC handles of the allocation
 * holding ws and of the handle's sync area, ws's offset and ws_bytes) written to `record`; allocates and
 * initialises the sync area and loads every kernel of the library (a first launch must not wait behind a
 * peer's spinning kernel).  Synchronises the device.  Every rank must pass the same ws_bytes. */
memfine_status memfine_ipc_export(memfine_handle_t h, void* ws, uint64_t ws_bytes, uint8_t* record);
/* Map every peer's workspace and sync area from the ep_size records (rank order, record r at
 * records + r * MEMFINE_IPC_RECORD_BYTES; this rank's own must come from memfine_ipc_export on this
 * handle).  The caller runs a host barrier after every rank's import and before the first layer call;
 * fwd / bwd must then pass the exported ws and ws_bytes.  MEMFINE_ERR_INVALID_ARG if the ranks' ws_bytes
 * differ or this rank did not export; MEMFINE_ERR_CUDA if a mapping fails. */
memfine_status memfine_ipc_import(memfine_handle_t h, const uint8_t* records);

/* A1 + A2: per-sub-chunk expert histogram of this rank's routing,
 * then the all-gather of every rank's histogram ("the first notification",
 * PAPER.md:200).  ids_dev: int32 [T][k] row-major.  counts_dev: int32
 * [EP][nsub][E]; counts_dev[r][j][e] = copies of rank r's sub-chunk j routed to
 * expert e, sub-chunk j = tokens [floor(jT/nsub), floor((j+1)T/nsub)).  Ids outside
 * [0,E) are not counted and latch MEMFINE_ERR_ROUTING.  1 <= nsub <= 64.
 * Collective when ep_size > 1. */
memfine_status memfine_route_counts(memfine_handle_t h, const int32_t* ids_dev, int32_t nsub,
                                    int32_t* counts_dev, void* stream);

/* m_g of Eq. 2 (§3): the number of micro-batches whose activations a pipeline stage
 * holds, m_g = v*p + p - 2*r_pp - 1 for virtual-pipeline size v, pipeline size p and stage r_pp
 * (0-based; reading R29), and m_g = 1 under full recomputation (full_recompute != 0).  MACT's s'_max
 * is per PP stage: pass the result as memfine_budget.m_g of that stage's plan.
 * v >= 1, p >= 1, 0 <= r_pp < p, else MEMFINE_ERR_INVALID_ARG. */
memfine_status memfine_m_g(int32_t v, int32_t p, int32_t r_pp, int32_t full_recompute, int32_t* m_g);

/* A3 (MACT): choose C from the counts.  counts: int32
 * [EP][nsub][E], HOST or DEVICE memory (detected).  Device counts are evaluated
 * by the library's single-CTA tuner kernel on the current device (one D2H of the
 * 64-byte result); host counts by the identical host routine.  Pure: no handle,
 * no communication.  Integer math throughout (reading R9):
 *   B = floor(alpha*M^GPU); num = B - static - other (<= 0 -> INFEASIBLE);
 *   s'_max = floor(num*tp*cp / (m_g*D_t*b*(2h+2g))) (<= 0 -> INFEASIBLE);
 *   s''_r = sum of counts routed to rank r's experts; c = max(1, ceil(max_r s''_r / s'_max));
 *   C = smallest bin >= c, else the largest bin with clamped = 1.
 * D_t = 2 for MEMFINE_BF16, 4 for MEMFINE_FP32. */
memfine_status memfine_plan(const int32_t* counts, int32_t nsub, const memfine_dims* dims,
                            const memfine_budget* budget, memfine_plan_info* info);
/* memfine_plan with device counts read in `stream` order: the tuner kernel (or, for MEMFINE_MODEL_IMPL,
 * the D2H copy of the counts) runs on `stream` and only `stream` is synchronised - the caller's other
 * streams (e.g. the next step's input copies) keep running.  memfine_plan instead synchronises the whole
 * device first, because its counts may come from any stream.  Host counts: identical to memfine_plan. */
memfine_status memfine_plan_stream(const int32_t* counts, int32_t nsub, const memfine_dims* dims,
                                   const memfine_budget* budget, memfine_plan_info* info, void* stream);

/* Exact workspace bytes the fwd (pass = MEMFINE_FWD) or bwd (MEMFINE_BWD) call
 * needs for this routing and C.  counts_host: int32 [EP][nsub][E] from
 * memfine_route_counts (copied to the host), C must divide nsub; or NULL for the
 * routing-independent worst case.  The result is the byte high-water of the
 * library's bump allocator: (per-row bytes) * max_j padded rows of chunk j +
 * send/receive staging (ep_size > 1) + metadata.  See DESIGN.md "Workspace". */
memfine_status memfine_workspace_bytes(const int32_t* counts_host, int32_t nsub,
                                       const memfine_dims* dims, int32_t C, int32_t pass,
                                       uint64_t* bytes);

/* A6 (EP > 1), host only: the all-to-allv the layer performs for chunk `chunk` of C on
 * rank dims->ep_rank.  counts_host: int32 [EP][nsub][E] (the all-gathered routing counts),
 * C | nsub.  Outputs (host):
 *   send_rows[EP]        rows this rank sends to each peer (its chunk copies, by dest rank)
 *   recv_rows[EP]        rows it receives from each source rank
 *   recv_offsets[EP*E_l] first row of (src, local expert) in the padded expert-major receive
 *                        buffer: local expert major, src rank minor (reading R3), each local
 *                        expert's segment padded to 128 rows
 *   rows_padded          total padded receive rows of the chunk (nullable)
 * Pure; no GPU, no communication. */
memfine_status memfine_a2a_plan(const int32_t* counts_host, int32_t nsub, const memfine_dims* dims, int32_t C,
                                int32_t chunk, int64_t* send_rows, int64_t* recv_rows, int64_t* recv_offsets,
                                int64_t* rows_padded);

/* FCDA forward (Eq. 6): Y = concat_j combine(expert(dispatch(X_j))).
 *   x       dev [T][h]        bf16 or fp32 (dims.dtype)
 *   ids     dev [T][k]        int32 global expert ids
 *   w       dev [T][k]        fp32 top-k scores
 *   w_gate  dev [E_l][g][h]   local experts only (nn.Linear [out,in])
 *   w_up    dev [E_l][g][h]
 *   w_down  dev [E_l][h][g]
 *   y       dev [T][h]        output (overwritten)
 *   ws      dev, ws_bytes >= memfine_workspace_bytes(counts, C, MEMFINE_FWD)
 * Nothing is saved for the backward (A11: the recompute discipline, m_g = 1).
 * Collective when ep_size > 1 (then it synchronises once on the counts). */
memfine_status memfine_moe_fwd(memfine_handle_t h, const void* x, const int32_t* ids, const float* w,
                               const void* w_gate, const void* w_up, const void* w_down, int32_t C,
                               void* y, void* ws, uint64_t ws_bytes, void* stream);

/* FCDA backward (Eq. 7): for each chunk j, recompute the chunk's gate/up
 * activations, then back-propagate dY_j.  Inputs as in memfine_moe_fwd plus
 *   dy      dev [T][h]        upstream gradient
 * Outputs:
 *   dx      dev [T][h]        (overwritten)
 *   dw_gate dev fp32 [E_l][g][h], dw_up fp32 [E_l][g][h], dw_down fp32 [E_l][h][g]
 *           overwritten, or accumulated into when accumulate_dw != 0
 *   dscore  dev fp32 [T][k]   dL/dw (nullable); 0 for ids outside [0,E)
 * Collective when ep_size > 1. */
memfine_status memfine_moe_bwd(memfine_handle_t h, const void* dy, const void* x, const int32_t* ids,
                               const float* w, const void* w_gate, const void* w_up, const void* w_down,
                               int32_t C, void* dx, float* dw_gate, float* dw_up, float* dw_down,
                               float* dscore, int32_t accumulate_dw, void* ws, uint64_t ws_bytes,
                               void* stream);

/* N3: the router step before the layer (Table 2 rows 9-10).
 *   logits = x W_r^T (fp32 accumulation), ids = the k largest logits (ties: lower expert id),
 *   scores = softmax over the k selected logits (the renormalised top-k convention).
 *   x dev [T][h], w_router dev [E][h] (dims.dtype, replicated on every EP rank), ids dev int32
 *   [T][k], scores dev fp32 [T][k], logits dev fp32 [T][E] (nullable: library scratch).
 *   BF16/MXFP8 handles: the logits GEMM and the backward's dW_r GEMMs run on the library's tcgen05
 *   expert-GEMM kernels (bf16 operands, fp32 accumulation in TMEM; the T tokens form one 128-row-padded
 *   segment, TMA zero-fills past T and E); top-k, softmax and the backward's row kernel are the
 *   library's.  FP32 handles use the library's CUDA-core GEMM (fp32 FMA, no TF32).  Stream-ordered; not
 *   graph-capture safe on the first call of a handle (it allocates and initialises scratch). */
memfine_status memfine_router_fwd(memfine_handle_t h, const void* x, const void* w_router, int32_t* ids,
                                  float* scores, float* logits, void* stream);
/* Router backward from the layer's d_score (memfine_moe_bwd's dscore):
 *   d_logit = s (ds - <s, ds>) on the selected slots (0 elsewhere);
 *   dx (dev [T][h]) = d_logits W_r, added to dx when accumulate_dx (the router shares the layer input);
 *   dw_router (dev fp32 [E][h]) = d_logits^T x, accumulated when accumulate_dw. */
memfine_status memfine_router_bwd(memfine_handle_t h, const void* x, const void* w_router, const int32_t* ids,
                                  const float* scores, const float* dscore, void* dx, int32_t accumulate_dx,
                                  float* dw_router, int32_t accumulate_dw, void* stream);

/* ---- MXFP8 variant of the expert GEMMs (reading R28) ----
 * The paper trains in BF16; this variant is the build's extension.  Block format:
 * 32 consecutive elements along a GEMM's K share one E8M0 scale 2^E, E the smallest integer with
 * amax <= 448 * 2^E (no element clips; E = 0 for an all-zero block); elements are E4M3,
 * round-to-nearest-even.  Quantised operands: x and W_gate/W_up rows along h, a and W_down rows
 * along g (forward and recompute); dG||dU and W_gate/W_up columns along g (dX).  The dA GEMM
 * (bound by its fused epilogue) stays BF16 x BF16 -> fp32; so do the weight gradients unless
 * MEMFINE_FLAG_MX_WGRAD (reading R28c: x, dY, dG||dU and a_w quantised along each expert's copies
 * in a chunk, blocks of 32, "columnwise").  With EP > 1
 * (EP_COPY transport) the dispatched rows travel in bf16 and each rank quantises the rows it
 * received (the same codes: x is blocked along h, per row); over EP_P2P the pushed bf16 rows are quantised
 * on arrival and the MX down / dX epilogues store o / dX rows into the sources' buffers.
 *
 * memfine_mx_weights_bytes: bytes of the quantised-weights buffer for dims (dtype MXFP8).
 * memfine_mx_quantize_weights: quantise the handle's local experts' bf16 weights (dev, the
 *   layouts of memfine_moe_fwd) into wq (dev, caller-owned, >= memfine_mx_weights_bytes;
 *   MEMFINE_ERR_WORKSPACE if smaller) and bind wq to the handle: every later fwd/bwd of an
 *   MXFP8 handle reads it (call again after each weight update; fwd/bwd before the first call
 *   return MEMFINE_ERR_INVALID_ARG).  Stream-ordered.
 * memfine_mx_quantize: the block format on its own: src dev bf16 [rows][K] -> codes dev uint8
 *   [rows][K] (E4M3) and scales dev uint8 [rows*K/32] (E + 127) in the tcgen05 scale-chunk
 *   layout (byte of row r, block b: ((r/128)*(K/128) + b/4)*512 + (r%32)*16 + ((r%128)/32)*4
 *   + b%4).  rows % 128 == 0, K % 128 == 0. */
memfine_status memfine_mx_weights_bytes(const memfine_dims* dims, uint64_t* bytes);
memfine_status memfine_mx_quantize_weights(memfine_handle_t h, const void* w_gate, const void* w_up,
                                           const void* w_down, void* wq, uint64_t wq_bytes, void* stream);
memfine_status memfine_mx_quantize(const void* src, int64_t rows, int32_t K, void* codes, void* scales,
                                   void* stream);

/* Synchronise `stream` and return (and clear) any device-latched error. */
memfine_status memfine_sync(memfine_handle_t h, void* stream);

/* Statistics of the last fwd/bwd (call memfine_sync first). */
memfine_status memfine_last_stats(memfine_handle_t h, memfine_stats* out);

/* Measurement: when enabled, the library brackets each of its launches with CUDA events
 * recorded on the launch stream and accumulates per-kernel-class device time.  Slots:
 * 0..5 the expert GEMMs (0 gate/up+SwiGLU, 1 down, 2 dA+fused epilogue, 3 dX,
 * 4 dW_down, 5 dW_gate||dW_up), 6 dispatch (histogram, scan, permute, padding), 7 combine /
 * unpermute-reduce, 8 memsets, 9 NCCL exchanges, 10 the MX weight gradients' columnwise quantisation
 * (MEMFINE_FLAG_MX_WGRAD).  memfine_profile_read synchronises on the
 * recorded events, returns the totals since the last read, and resets them. */
#define MEMFINE_PROF_SLOTS 11
typedef struct {
    int32_t launches[MEMFINE_PROF_SLOTS];
    double  ms[MEMFINE_PROF_SLOTS];
} memfine_profile;
memfine_status memfine_profile_enable(memfine_handle_t h, int32_t enable);
memfine_status memfine_profile_read(memfine_handle_t h, memfine_profile* out);

/* Debug: when enabled, fwd records each chunk's canonical dispatch order
 * (reading R3: ascending local expert, src rank, token, slot; padding rows
 * dropped) as src*T*k + i*k + slot.  memfine_debug_perm copies chunk `chunk`
 * of the last fwd into perm_host (capacity cap) and sets *n. */
memfine_status memfine_set_debug(memfine_handle_t h, int32_t enable);
memfine_status memfine_debug_perm(memfine_handle_t h, int32_t chunk, int64_t* perm_host, int64_t cap,
                                  int64_t* n);
/* Debug, ep_size == 1 (test infrastructure: the debug capture synchronises after each chunk's GEMMs).
 * memfine_debug_rows: chunk `chunk` of the last fwd or bwd call, its expert-major padded rows' copy
 *   index (i*k + slot) or -1 for a padding row; *n = the chunk's padded rows.  src_of_host NULL:
 *   only *n.
 * memfine_debug_mx (MXFP8 handles): the decisions the kernels took on one quantised operand of chunk
 *   `chunk` of the last call - codes_host [rows][cols] E4M3 bytes, scales_host [rows*cols/32] E8M0
 *   bytes in the scale-chunk layout of memfine_mx_quantize with K = cols.  which:
 *     0 a (fwd), rows = the chunk's padded rows, cols = g (blocks along g)
 *     1 dG || dU (bwd, the dX operand), rows = padded rows, cols = 2g
 *     2 x, 3 dY, 4 dG || dU, 5 a_w: MEMFINE_FLAG_MX_WGRAD's columnwise operands (reading R28c),
 *       rows = h / h / 2g / g operand columns, cols = the workspace's row capacity (blocks of 32
 *       rows along it; only the chunk's padded rows are meaningful).
 *   codes_host NULL: only *rows and *cols; cap_codes < rows*cols: MEMFINE_ERR_INVALID_ARG. */
memfine_status memfine_debug_rows(memfine_handle_t h, int32_t chunk, int32_t* src_of_host, int64_t cap, int64_t* n);
memfine_status memfine_debug_mx(memfine_handle_t h, int32_t chunk, int32_t which, uint8_t* codes_host,
                                uint8_t* scales_host, int64_t cap_codes, int64_t* rows, int64_t* cols);

#ifdef __cplusplus
}
#endif
#endif /* MEMFINE_H */
