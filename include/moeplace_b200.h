/*
 * moeplace_b200.h -- C ABI of the B200-native distributed MoE-layer forward.
 *
 * The reference (`moeplace`, arXiv 2508.12851) is a pure-Python placement
 * library + simulator; it has no FFI.  Its hot path -- the per-layer dispatch
 * `_EventLoop._dispatch_layer` (reference pkg/src/moeplace/sim.py:441-463) with
 * the target rule `_choose_target` (sim.py:433-439), the activation counting
 * `ActivationStats.ingest` (stats.py:82-96), the analytic `comp_time` /
 * `comm_time` estimators (cost.py:132-149) and the migration slot diff of
 * `migration_cost` (cost.py:171-191) -- is replaced by the entry points below.
 * Each entry point names the reference interface it replaces.
 *
 * Conventions
 *   - Plain pointers and sizes only.  Device pointers are `void*` / typed
 *     pointers into GPU memory; `stream` is a cudaStream_t passed as void*.
 *   - Every call returns 0 (MP_OK) or a negative MP_E_* code; the message of
 *     the last failure on the calling thread is available from mp_last_error.
 *   - bf16 buffers are row-major, 2 bytes per element.
 *   - The library owns only what mp_layer_create allocates (the NVLink-shared
 *     window, the expert-weight slot pool and per-layer scratch); caller
 *     buffers are never freed by the library.
 *   - One host thread per mp_layer; calls on one layer are not re-entrant
 *     (the reference event loop is single-threaded).
 */
#ifndef MOEPLACE_B200_H
#define MOEPLACE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MP_ABI_VERSION 3
#define MP_MAX_GROUPS 128 /* expert groups per mp_grouped_gemm call */

#define MP_OK 0
#define MP_E_ARG -1        /* bad argument (null pointer, unknown mode)                  */
#define MP_E_SHAPE -2      /* shape mismatch      -> moeplace.DimensionMismatch           */
#define MP_E_CAPACITY -3   /* slot / buffer cap   -> moeplace.InfeasibleError             */
#define MP_E_UNPLACED -4   /* route w/o holder    -> moeplace.UnplacedExpertError         */
#define MP_E_CUDA -5       /* CUDA runtime / driver failure -> RuntimeError               */
#define MP_E_PEER -6       /* IPC / NVLink peer failure or barrier timeout -> RuntimeError */

/* Router score modes (public model definitions; the reference has no router,
 * SPEC.md:416). */
#define MP_SCORE_TOPK_SOFTMAX 0 /* Mixtral: top-k logits, softmax over the k            */
#define MP_SCORE_SOFTMAX_TOPK 1 /* Qwen1.5-MoE / DeepSeek-V2-Lite: softmax over E, top-k */

int mp_abi_version(void);
/* Copies the last error message of the calling thread (NUL-terminated). */
int mp_last_error(char* buf, int buf_len);

/* ------------------------------------------------------------------------
 * Stateless kernels (used by the layer, exported for parity tests).
 * --------------------------------------------------------------------- */

/* Bytes of the packed router operand for E_tot weight rows of width d. */
size_t mp_router_packed_bytes(int E_tot, int d);

/* Pack router weights Wg [E_tot, d] bf16 into K1's exact-integer operand:
 * each row on its own integer grid (q = rint(w * 2^(21 - E(row))), see
 * csrc/router.cu), as three 8-bit limb planes [3][N][d] (N = E_tot rounded up
 * to a multiple of 16, zero rows), then int64 row sums [N] and int32 row
 * exponents [N].  `packed` must hold mp_router_packed_bytes(E_tot, d) bytes
 * (16-byte aligned); d % 256 == 0.  E_tot = E, or E+1 with the shared-expert
 * gate row. */
int mp_router_pack(const void* wg_bf16, int E_tot, int d, void* packed, void* stream);

/* K1 -- replaces ActivationStats.ingest (stats.py:82-96) fed by sampled expert
 * sets (sim.py:181-185): top-k routing of T tokens plus a fused histogram.
 *   x        [T, d] bf16           packed  from mp_router_pack (E + has_gate rows)
 *   bias     [E] fp32 or NULL      per-origin routing skew (log p, sim.py:161-164)
 *   idx      [T, k] int32 out      experts, descending logit, ties -> lower id
 *   w        [T, k] fp32 out       gate weights
 *   gate_out [T] fp32 out or NULL  sigmoid shared-expert gate (has_gate = 1)
 *   hist     [E] uint32 in/out     += tokens routed to each expert (token_count 1)
 */
int mp_router_topk_hist(const void* x, const void* packed, const float* bias, int T, int d, int E, int has_gate,
                        int k, int score_mode, int renorm, int32_t* idx, float* w, float* gate_out, uint32_t* hist,
                        void* stream);
/* Logits-in parity variant of K1's selection stage: top-k (descending, ties ->
 * lower id), gate weights and histogram from fp32 logits [T][ld] (+ bias [E]
 * or NULL) -- pins the selection rule independently of the dot products. */
int mp_router_topk_logits(const float* logits, int ld, const float* bias, int T, int E, int k, int score_mode,
                          int renorm, int32_t* idx, float* w, uint32_t* hist, void* stream);

/* K3 -- replaces comp_time (cost.py:132-136).  Grouped GEMM on tcgen05:
 *   for g < *n_groups: rows [a_row, a_row+m) of A [a_rows, K] times slot `slot`
 *   of B (rows slot*N .. slot*N+N of B [b_rows, K]) -> out rows [o_row, o_row+m).
 *   swiglu = 1: B holds interleaved gate/up blocks of 128 rows, out [*, N/2].
 *   groups (device) = n x {a_row, m, slot, o_row}; n_groups (device) int32,
 *   at most MP_MAX_GROUPS (else MP_E_SHAPE; this parity entry reads it with a
 *   stream sync).                                                             */
int mp_grouped_gemm(const void* a, int64_t a_rows, const void* b, int64_t b_rows, const int32_t* groups,
                    const int32_t* n_groups, int N, int K, void* out, int out_ld, int swiglu, void* stream);

/* ------------------------------------------------------------------------
 * The MoE layer: one per (process, GPU); rank r of G ranks = reference server r
 * with one GPU (ClusterSpec servers, domain.py:73-155).
 * --------------------------------------------------------------------- */
typedef struct mp_layer mp_layer;

typedef struct mp_layer_desc {
  int32_t rank;         /* this GPU = reference server id                      */
  int32_t world;        /* G: number of GPUs (servers), 1..8                    */
  int32_t device;       /* CUDA device ordinal                                   */
  int32_t max_tokens;   /* T capacity per forward on this origin                */
  int32_t d;            /* hidden width  (ModelSpec.hidden_width)               */
  int32_t f;            /* expert FFN width                                     */
  int32_t E;            /* routed experts (ModelSpec.experts_per_layer[l])      */
  int32_t top_k;        /* ModelSpec.top_k                                      */
  int32_t score_mode;   /* MP_SCORE_*                                           */
  int32_t renorm;       /* renormalise top-k weights (softmax_topk mode)        */
  int32_t n_slots;      /* expert slots on this GPU: floor(GpuSpec.memory / m_e) */
  int32_t shared_f;     /* shared-expert FFN width, 0 = none                    */
  int32_t shared_gate;  /* 1: shared output scaled by sigmoid(x . w_sg)          */
} mp_layer_desc;

/* Device pointers of the layer's buffers (for filling weights and for
 * parity inspection).  Sizes in elements. */
typedef struct mp_layer_ptrs {
  void* pool;        /* expert slot s at pool + s * slot_bytes (n_slots slots), holding
                        [W13: 2f x d bf16, gate/up rows interleaved per 128 rows | W2: d x f bf16]
                        -- one contiguous m_e-byte block per slot (migration copies it whole) */
  void* wg;          /* [E + shared_gate][d] bf16 router weights (packed on set)  */
  float* bias;       /* [E] fp32                                                 */
  void* w13_shared;  /* [2*shared_f][d] bf16 or NULL                             */
  void* w2_shared;   /* [d][shared_f] bf16 or NULL                               */
  int32_t* idx;      /* [max_tokens][k]                                          */
  float* w;          /* [max_tokens][k]                                          */
  int32_t* pos_dst;  /* [max_tokens][k] target GPU of each (token, slot)         */
  int32_t* pos_row;  /* [max_tokens][k] row in the target's receive buffer       */
  void* recv;        /* [recv_cap][d] bf16 rows received for local experts       */
  void* h;           /* [recv_cap][f] bf16 SwiGLU activations                    */
  void* ret;         /* [max_tokens][k][d] bf16 this origin's expert outputs, in (token, slot)
                        order, written back by the (local or peer) GEMM2 epilogues      */
  int32_t* recv_src; /* [recv_cap] (origin rank << 24 | pair index) of each received row */
  uint32_t* hist;    /* [E] cumulative activation histogram (this origin)        */
  int32_t* counts;   /* [2][G][E] exchanged batch counts C[src][e] (parity halves) */
  float* shared_gate;/* [max_tokens] or NULL                                     */
  int32_t* batch_counts; /* [E] this origin's counts of the last routed batch      */
  int64_t recv_cap;  /* rows                                                     */
  int64_t slot_bytes;/* bytes of one expert slot (w13 + w2) = ModelSpec.expert_size */
} mp_layer_ptrs;

int mp_layer_create(const mp_layer_desc* desc, mp_layer** out);
int mp_layer_destroy(mp_layer* layer);
int mp_layer_get_ptrs(mp_layer* layer, mp_layer_ptrs* out);

/* NVLink window setup (G > 1): export this rank's IPC handles (2 x 64 bytes:
 * exchange window, weight pool), then open all ranks' handles (G x 128 bytes,
 * ordered by rank; this rank's own entry is ignored). */
int mp_layer_export_handles(mp_layer* layer, void* handles_out /* 128 bytes */);
int mp_layer_open_peers(mp_layer* layer, const void* all_handles /* G * 128 bytes */);

/* Route table -- replaces `_choose_target` (sim.py:433-439) evaluated per
 * invocation: route[s*E + e] = target GPU for origin s and expert e (origin if
 * it holds e, else the cheapest holder, ties to the lowest id); slot_of[e] =
 * local slot holding e on this GPU or -1.  Host arrays; validated
 * (MP_E_UNPLACED when a route points at a GPU without the expert here). */
int mp_layer_set_routes(mp_layer* layer, const int32_t* route, const int32_t* slot_of, void* stream);

/* Packs layer->wg (+ bias) after the caller filled them. */
int mp_layer_prepare_router(mp_layer* layer, void* stream);

/* One MoE-layer forward of T tokens originating on this GPU -- replaces
 * `_dispatch_layer` (sim.py:441-463).  x, out: [T, d] bf16 device.  SPMD: all
 * G ranks must call it with their own T (T = 0 allowed).  Kernels: router +
 * histogram (its tail publishes the counts to every peer), permute + dispatch
 * (NVLink stores), grouped SwiGLU GEMMs on tcgen05 (shared expert fused in;
 * GEMM2's epilogue stores each row back to its origin GPU over NVLink),
 * combine (local).  The cross-GPU ordering is a flag protocol inside those
 * kernels; there is no separate barrier launch. */
int mp_layer_forward(mp_layer* layer, const void* x, void* out, int T, void* stream);

/* Same forward, recording MP_NUM_STAGE_EVENTS cudaEvent_t (created by the
 * caller with timing enabled; NULL entries are skipped) on `stream` at the
 * stage boundaries:
 *   0 start | 1 router (+ count exchange) | 2, 3 (folded) | 4 permute+dispatch |
 *   5 shared expert (empty when fused into K3) | 6 (folded) | 7 GEMM1 SwiGLU |
 *   8 GEMM2 | 9 (folded) | 10 combine+return
 * and, on the side stream when the small-group chain runs (MP_CFG_SPLIT_M):
 *   11 side chain start | 12 side chain end                                   */
#define MP_NUM_STAGE_EVENTS 13
int mp_layer_forward_timed(mp_layer* layer, const void* x, void* out, int T, void* stream, void* const* events);

/* ---- The same forward as separate stages, for a host-driven transport (the
 * NCCL all-to-all-v arm: paper_2508_12851_b200/nccl_path.py) and for standalone
 * K1 / K2 / K3 / K5 parity tests.  Between the stages the caller moves rows:
 *   mp_layer_route     K1 only: idx, w, gate, histogram and this origin's batch
 *                      counts (ptrs.batch_counts); no peer exchange.
 *   mp_layer_permute   K2 against a caller-assembled count table counts_all
 *                      [G][E] (device): rows for this GPU go into recv, rows
 *                      for GPU D != rank into `staging` + (D * recv_cap + r) * d,
 *                      r = the row in D's receive layout (pos_row) -- so every
 *                      (source, expert) chunk has the same offsets in the
 *                      sender's image and in D's receive buffer.
 *   mp_layer_experts   K3 over recv (groups from counts_all and the routes);
 *                      the expert outputs overwrite their received rows.
 *   mp_layer_combine_gather
 *                      K5 reading pair (t, j)'s output from recv (own GPU) or
 *                      `ret_stage` + (D * recv_cap + pos_row) * d (GPU D's
 *                      rows, returned into the same image layout).
 * staging / ret_stage: G * recv_cap * d bf16 (device), unused when G == 1. */
int mp_layer_route(mp_layer* layer, const void* x, int T, void* stream);
int mp_layer_permute(mp_layer* layer, const void* x, int T, const int32_t* counts_all, void* staging, void* stream);
int mp_layer_experts(mp_layer* layer, const void* x, int T, const int32_t* counts_all, void* stream);
int mp_layer_combine_gather(mp_layer* layer, const void* ret_stage, int T, void* out, void* stream);

/* Number of kernels the last mp_layer_forward launched. */
int mp_layer_last_launches(mp_layer* layer);

/* K3 execution plan of the last forward (before any forward: the plan chosen at
 * creation from the shape; MP_* environment knobs override), for reporting.
 * Small batches (G*T*k/E below MP_STREAM_ROWS, default 256) stream every
 * expert group over all SMs on the 1-CTA kernel instead of splitting off a
 * side chain; the shared expert rides in the routed launches either way. */
#define MP_CFG_PAIR_ROUTED 0   /* routed experts on CTA-pair (256-row) tiles   */
#define MP_CFG_SPLIT_M 1       /* groups below this many rows: side-stream chain */
#define MP_CFG_SMALL_GRID 2    /* SMs given to that side chain                   */
#define MP_CFG_FUSE_SHARED 3   /* shared expert fused into the routed launches   */
int mp_layer_config(mp_layer* layer, int key);

/* Host copy of the last forward's exchanged count table C[src][e] (G*E int32;
 * synchronises the stream).  C feeds the reference accounting: remote pairs
 * (sim.py:452-456), remote_volume (cost.py:120-129). */
int mp_layer_read_counts(mp_layer* layer, int32_t* host_counts, void* stream);

/* Barrier/peer error word (0 = ok); synchronises the stream. */
int mp_layer_check(mp_layer* layer, void* stream);

/* Diagnostic: the NVLink flag protocol's device state at a quiescent point (synchronises
 * `stream` and the layer's side stream).  out[16]: [0] epoch, [1] forwards seen, [2] count
 * parity, [3] router / [4] permute / [5] GEMM2 arrival tickets, [6] timeout bits, [7] nonzero
 * router count accumulators, [8 + p] flags[p] of this rank's window (p < G).  Between
 * forwards every rank holds the same epoch, every flag equals it and [3..7] are 0. */
int mp_layer_sync_state(mp_layer* layer, uint32_t* out, void* stream);

/* K6 -- executes the slot diff of migration_cost (cost.py:186-187) adopted by
 * should_migrate (cost.py:217-248): copy expert slots into local slots, from a
 * peer GPU's pool over NVLink (src_rank != rank) or locally, on `stream`
 * (a side stream), then record `done_event` (cudaEvent_t, may be NULL).  The
 * caller swaps routes (mp_layer_set_routes) only after the event completes,
 * matching migration_complete (sim.py:520-525). */
typedef struct mp_copy_op {
  int32_t src_rank;
  int32_t src_slot;
  int32_t dst_slot;
} mp_copy_op;
int mp_layer_migrate(mp_layer* layer, const mp_copy_op* ops, int n_ops, void* stream, void* done_event);

/* Link probe for the measured-cost inputs of the reference's TimeModel (comm_time,
 * cost.py:139-149) and migration_cost's load bandwidth (cost.py:171-191): `reps`
 * back-to-back copies of `bytes` from peer's receive region into ours over the
 * NVLink mapping, timed with CUDA events on `stream` (synchronises).  Small sizes
 * give the per-transfer latency, large sizes the bandwidth.  Overwrites the
 * receive region (call between forwards). */
int mp_layer_peer_probe(mp_layer* layer, int peer, int64_t bytes, int reps, void* stream, float* ms_per_copy);

#ifdef __cplusplus
}
#endif

#endif /* MOEPLACE_B200_H */
