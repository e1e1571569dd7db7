// extern "C" boundary (include/moeplace_b200.h) and the MoE layer object.
//
// The layer composes the kernels of one distributed MoE-layer forward; it is
// the B200 counterpart of `_EventLoop._dispatch_layer` (reference
// pkg/src/moeplace/sim.py:441-463).  Memory per GPU:
//   pool    (IPC-exported)  expert weight slots, n_slots = floor(GpuSpec.memory / m_e)
//                           (domain.py:395-401): the per-GPU memory cap is real
//   window  (IPC-exported)  receive rows, expert outputs, count tables, flags
//   scratch (private)       router/permutation state, SwiGLU activations, maps
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "mp_internal.h"

namespace mp {

static thread_local char g_err[1024] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

bool pdl_enabled() {
  static const bool on = [] {
    // measured: within noise on Mixtral, slower with the concurrent small-group chain
    // (Qwen / DeepSeek) -- opt in with MP_PDL=1
    const char* env = getenv("MP_PDL");
    return env != nullptr && atoi(env) != 0;
  }();
  return on;
}

int set_cuda_error(cudaError_t e, const char* what) {
  return set_error(MP_E_CUDA, "%s: %s (%d)", what, cudaGetErrorString(e), int(e));
}

int ensure_max_dyn_smem(const void* kernel, size_t bytes, const char* what) {
  if (bytes == 0) return MP_OK;  // the 48 KB default covers static + dynamic: set it for any dynamic size
  struct Entry {
    const void* fn;
    int dev;
    size_t bytes;
  };
  static std::mutex mu;
  static std::vector<Entry> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaGetDevice");
  std::lock_guard<std::mutex> lock(mu);
  for (Entry& x : done)
    if (x.fn == kernel && x.dev == dev) {
      if (x.bytes >= bytes) return MP_OK;
      e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
      if (e != cudaSuccess) return set_cuda_error(e, what);
      x.bytes = bytes;
      return MP_OK;
    }
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
  if (e != cudaSuccess) return set_cuda_error(e, what);
  done.push_back({kernel, dev, bytes});
  return MP_OK;
}

}  // namespace mp

using namespace mp;

#define MP_CUDA(call)                                                  \
  do {                                                                 \
    cudaError_t _e = (call);                                           \
    if (_e != cudaSuccess) return set_cuda_error(_e, #call);           \
  } while (0)
#define MP_TRY(call)                 \
  do {                               \
    int _r = (call);                 \
    if (_r != MP_OK) return _r;      \
  } while (0)

struct mp_layer {
  mp_layer_desc desc;
  int G = 1, rank = 0, nb_max = 0;
  int64_t recv_cap = 0;
  size_t w13_slot_elems = 0, w2_slot_elems = 0, slot_bytes = 0;

  // allocations
  uint8_t* pool = nullptr;
  size_t pool_bytes = 0;
  uint8_t* window = nullptr;
  size_t window_bytes = 0;
  uint8_t* scratch = nullptr;
  size_t scratch_bytes = 0;
  size_t off_recv = 0, off_ret = 0, off_src = 0, off_counts = 0, off_flags = 0;

  // pool / window views
  __nv_bfloat16 *w13 = nullptr, *w2 = nullptr, *recv = nullptr, *ret = nullptr;
  int32_t* recv_src = nullptr;
  int32_t* counts = nullptr;
  uint32_t* flags = nullptr;
  // scratch views
  __nv_bfloat16 *h = nullptr, *wg = nullptr, *w13s = nullptr, *w2s = nullptr, *hs = nullptr, *ys = nullptr;
  uint8_t* wg_packed = nullptr;  // router operand: Wg limbs, row sums, row exponents
  float *bias = nullptr, *w = nullptr, *sgate = nullptr;
  int32_t *idx = nullptr, *pos_dst = nullptr, *pos_row = nullptr, *blk_counts = nullptr, *count_acc = nullptr,
          *batch_counts = nullptr, *route_d = nullptr,
          *slot_of_d = nullptr;
  uint32_t *hist = nullptr, *err = nullptr, *ticket = nullptr, *sync_state = nullptr;
  // peer-timeout bits mirrored into mapped pinned host memory: read by the next forward
  volatile uint32_t* err_host = nullptr;
  uint32_t* err_host_d = nullptr;
  uint32_t *perm_ticket = nullptr, *ret_ticket = nullptr;  // arrival counters of the raising kernels
  void** ptr_arrays = nullptr;  // device: recv[8], ret[8], flags[8], counts0[8], counts1[8], recv_src[8]
  // stage entries (host-driven transport): device [recv images 8 | recv_src images 8 | combine bases 8]
  void** stage_ptrs = nullptr;
  void* stage_host[24] = {};
  bool stage_uploaded = false;
  int32_t* src_image = nullptr;  // [G][recv_cap] recv_src images of the peers' layouts (never read)

  uint8_t* peer_window[8] = {};
  uint8_t* peer_pool[8] = {};
  bool peers_open = false, routes_set = false, router_ready = false;

  CUtensorMap tm_recv, tm_w13, tm_h, tm_w2, tm_w13s, tm_hs, tm_w2s, tm_x;
  // B maps with 128-row boxes for the CTA-pair GEMM (each CTA loads half of N)
  CUtensorMap tm_w13_p, tm_w2_p, tm_w13s_p, tm_w2s_p;
  int pair_routed = 0, pair_shared = 1;
  // shared expert fused into the routed CTA-pair launches (one GEMM1 and one GEMM2
  // launch cover both problems; no per-launch tails / wave quantisation of its own)
  int fuse_shared = 0;
  // below this many rows per expert on average (G*T*k/E) a forward streams every group
  // over all SMs on the 1-CTA kernel (no side chain, shared expert in its own launches)
  int stream_rows = 256;
  int last_pair = -1, last_split = -1, last_fused = -1;  // plan of the last forward (-1: none yet)
  int last_small_grid = 0;
  // small-group split: groups below split_m rows run on a side stream over small_grid SMs
  int split_m = 0, small_grid = 20;
  int tail_max = 0;  // split plans: pair-tile tails of up to tail_max rows go to the side chain
  int side_shared_rows = 0;  // split plans: the fused shared expert's last rows run on the side chain
  bool small_grid_fixed = false;  // MP_GEMM_SMALL_GRID pins it; else chosen per forward
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  const void* tm_x_ptr = nullptr;
  int tm_x_rows = -1;

  int last_launches = 0;
};

namespace {

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct Carver {
  uint8_t* base;
  size_t off = 0;
  template <typename T>
  T* take(size_t count) {
    off = align_up(off, 256);
    T* p = reinterpret_cast<T*>(base + off);
    off += count * sizeof(T);
    return p;
  }
};

int validate_desc(const mp_layer_desc& d) {
  if (d.world < 1 || d.world > 8) return set_error(MP_E_SHAPE, "world=%d outside [1, 8]", d.world);
  if (d.rank < 0 || d.rank >= d.world) return set_error(MP_E_SHAPE, "rank=%d outside [0, %d)", d.rank, d.world);
  if (d.max_tokens < 1) return set_error(MP_E_SHAPE, "max_tokens=%d", d.max_tokens);
  if (d.E < 1 || d.E > 64) return set_error(MP_E_SHAPE, "E=%d outside [1, 64]", d.E);
  if (d.top_k < 1 || d.top_k > 8 || d.top_k > d.E) return set_error(MP_E_SHAPE, "top_k=%d invalid", d.top_k);
  if (d.d % 256 != 0) return set_error(MP_E_SHAPE, "hidden width d=%d must be a multiple of 256", d.d);
  if (d.f % 128 != 0) return set_error(MP_E_SHAPE, "FFN width f=%d must be a multiple of 128", d.f);
  if (d.shared_f % 128 != 0 || d.shared_f < 0)
    return set_error(MP_E_SHAPE, "shared FFN width %d must be a multiple of 128", d.shared_f);
  if (d.score_mode != MP_SCORE_TOPK_SOFTMAX && d.score_mode != MP_SCORE_SOFTMAX_TOPK)
    return set_error(MP_E_ARG, "score_mode=%d", d.score_mode);
  if (d.n_slots < 0) return set_error(MP_E_CAPACITY, "n_slots=%d", d.n_slots);
  if (d.shared_gate && d.shared_f == 0) return set_error(MP_E_ARG, "shared_gate without a shared expert");
  return MP_OK;
}

}  // namespace

extern "C" {

int mp_abi_version(void) { return MP_ABI_VERSION; }

int mp_last_error(char* buf, int buf_len) {
  if (!buf || buf_len <= 0) return MP_E_ARG;
  strncpy(buf, g_err, size_t(buf_len) - 1);
  buf[buf_len - 1] = 0;
  return MP_OK;
}

size_t mp_router_packed_bytes(int E_tot, int d) { return router_packed_bytes(E_tot, d); }

int mp_router_pack(const void* wg_bf16, int E_tot, int d, void* packed, void* stream) {
  if (!wg_bf16 || !packed) return set_error(MP_E_ARG, "mp_router_pack: null pointer");
  return launch_router_pack(static_cast<const __nv_bfloat16*>(wg_bf16), E_tot, d, static_cast<uint8_t*>(packed),
                            static_cast<cudaStream_t>(stream));
}

int mp_router_topk_hist(const void* x, const void* packed, const float* bias, int T, int d, int E, int has_gate,
                        int k, int score_mode, int renorm, int32_t* idx, float* w, float* gate_out, uint32_t* hist,
                        void* stream) {
  if (!x || !packed || !idx || !w) return set_error(MP_E_ARG, "mp_router_topk_hist: null pointer");
  return launch_router(static_cast<const __nv_bfloat16*>(x), static_cast<const uint8_t*>(packed), bias, T, d, E,
                       has_gate, k, score_mode, renorm, idx, w, gate_out, hist, nullptr, nullptr, nullptr, nullptr,
                       static_cast<cudaStream_t>(stream));
}

int mp_router_topk_logits(const float* logits, int ld, const float* bias, int T, int E, int k, int score_mode,
                          int renorm, int32_t* idx, float* w, uint32_t* hist, void* stream) {
  if ((!logits || !idx || !w) && T > 0) return set_error(MP_E_ARG, "mp_router_topk_logits: null pointer");
  return launch_router_logits(logits, ld, bias, T, E, k, score_mode, renorm, idx, w, hist,
                              static_cast<cudaStream_t>(stream));
}

int mp_grouped_gemm(const void* a, int64_t a_rows, const void* b, int64_t b_rows, const int32_t* groups,
                    const int32_t* n_groups, int N, int K, void* out, int out_ld, int swiglu, void* stream) {
  if (!a || !b || !groups || !n_groups || !out) return set_error(MP_E_ARG, "mp_grouped_gemm: null pointer");
  // the group count lives on the device (the kernel reads it in its prologue); this
  // stateless entry reads it once so an oversized table fails instead of being clipped
  int32_t ng = 0;
  MP_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  MP_CUDA(cudaMemcpy(&ng, n_groups, 4, cudaMemcpyDeviceToHost));
  if (ng < 0 || ng > MP_MAX_GROUPS)
    return set_error(MP_E_SHAPE, "mp_grouped_gemm: n_groups=%d outside [0, %d]", ng, MP_MAX_GROUPS);
  CUtensorMap ta, tb;
  int pair = 0;
  if (const char* env = getenv("MP_GEMM_PAIR")) pair = atoi(env);
  MP_TRY(encode_tmap_bf16_2d(&ta, a, uint64_t(a_rows), uint64_t(K), 128));
  MP_TRY(encode_tmap_bf16_2d(&tb, b, uint64_t(b_rows), uint64_t(K), pair ? 128 : 256));
  GroupSpec gs;
  gs.mode = 0;
  gs.groups = groups;
  gs.n_groups = n_groups;
  return launch_grouped_gemm(ta, tb, gs, N, K, N, 0, static_cast<__nv_bfloat16*>(out), out_ld, swiglu, 0,
                             static_cast<cudaStream_t>(stream), pair);
}

int mp_layer_create(const mp_layer_desc* desc, mp_layer** out) {
  if (!desc || !out) return set_error(MP_E_ARG, "mp_layer_create: null pointer");
  MP_TRY(validate_desc(*desc));
  DeviceGuard dg(desc->device);
  MP_CUDA(dg.status);
  cudaDeviceProp prop;
  MP_CUDA(cudaGetDeviceProperties(&prop, desc->device));
  if (prop.major != 10)
    return set_error(MP_E_CUDA, "device %d is sm_%d%d; this library is built for sm_100a (B200)", desc->device,
                     prop.major, prop.minor);

  mp_layer* L = new mp_layer();
  L->desc = *desc;
  const mp_layer_desc& D = L->desc;
  L->G = D.world;
  L->rank = D.rank;
  L->nb_max = (D.max_tokens + router_block_tokens() - 1) / router_block_tokens();
  L->recv_cap = int64_t(D.world) * D.max_tokens * D.top_k;
  L->w13_slot_elems = size_t(2) * D.f * D.d;
  L->w2_slot_elems = size_t(D.d) * D.f;

  auto fail = [&](int code) {
    mp_layer_destroy(L);
    return code;
  };
  cudaError_t e;

  // ---- pool: slot s = [w13 (2f x d) | w2 (d x f)], exactly m_e = 3*d*f*2 bytes
  L->slot_bytes = (L->w13_slot_elems + L->w2_slot_elems) * 2;
  L->pool_bytes = std::max<size_t>(256, size_t(D.n_slots) * L->slot_bytes);
  if ((e = cudaMalloc(&L->pool, L->pool_bytes)) != cudaSuccess)
    return fail(set_error(MP_E_CAPACITY, "cannot allocate %d expert slots (%zu bytes): %s", D.n_slots,
                          L->pool_bytes, cudaGetErrorString(e)));
  L->w13 = reinterpret_cast<__nv_bfloat16*>(L->pool);
  L->w2 = L->w13 + L->w13_slot_elems;

  // ---- window (identical layout on every rank)
  {
    size_t off = 0;
    L->off_recv = off;
    off = align_up(off + size_t(L->recv_cap) * D.d * 2, 1024);
    L->off_ret = off;
    off = align_up(off + size_t(D.max_tokens) * D.top_k * D.d * 2, 1024);
    L->off_src = off;
    off = align_up(off + size_t(L->recv_cap) * 4, 1024);
    L->off_counts = off;
    off = align_up(off + size_t(2) * 8 * 64 * 4, 256);
    L->off_flags = off;
    off = align_up(off + 64 * 4, 256);
    L->window_bytes = off;
  }
  if ((e = cudaMalloc(&L->window, L->window_bytes)) != cudaSuccess)
    return fail(set_error(MP_E_CAPACITY, "cannot allocate the exchange window (%zu bytes): %s", L->window_bytes,
                          cudaGetErrorString(e)));
  L->recv = reinterpret_cast<__nv_bfloat16*>(L->window + L->off_recv);
  L->ret = reinterpret_cast<__nv_bfloat16*>(L->window + L->off_ret);
  L->recv_src = reinterpret_cast<int32_t*>(L->window + L->off_src);
  L->counts = reinterpret_cast<int32_t*>(L->window + L->off_counts);
  L->flags = reinterpret_cast<uint32_t*>(L->window + L->off_flags);
  if ((e = cudaMemset(L->window + L->off_counts, 0, L->window_bytes - L->off_counts)) != cudaSuccess)
    return fail(set_cuda_error(e, "cudaMemset(window)"));

  // ---- scratch
  {
    const int T = D.max_tokens, k = D.top_k, E = D.E;
    const int E_tot = E + (D.shared_gate ? 1 : 0);
    Carver c{nullptr};
    auto plan = [&](Carver& cv) {
      L->h = cv.take<__nv_bfloat16>(size_t(L->recv_cap) * D.f);
      L->wg = cv.take<__nv_bfloat16>(size_t(E_tot) * D.d);
      L->wg_packed = cv.take<uint8_t>(router_packed_bytes(E_tot, D.d));
      L->bias = cv.take<float>(E);
      L->w = cv.take<float>(size_t(T) * k);
      L->sgate = D.shared_gate ? cv.take<float>(T) : nullptr;
      L->idx = cv.take<int32_t>(size_t(T) * k);
      L->pos_dst = cv.take<int32_t>(size_t(T) * k);
      L->pos_row = cv.take<int32_t>(size_t(T) * k);
      L->blk_counts = cv.take<int32_t>(size_t(L->nb_max) * E);
      L->count_acc = cv.take<int32_t>(64);  // router batch-count accumulator (reset by its last CTA)
      L->batch_counts = cv.take<int32_t>(64);
      L->route_d = cv.take<int32_t>(8 * 64);
      L->slot_of_d = cv.take<int32_t>(64);
      L->hist = cv.take<uint32_t>(64);
      L->err = cv.take<uint32_t>(4);
      L->ticket = cv.take<uint32_t>(4);
      L->perm_ticket = cv.take<uint32_t>(4);
      L->ret_ticket = cv.take<uint32_t>(4);
      L->sync_state = cv.take<uint32_t>(4);
      L->ptr_arrays = cv.take<void*>(6 * 8);
      L->stage_ptrs = cv.take<void*>(3 * 8);
      if (D.shared_f > 0) {
        L->w13s = cv.take<__nv_bfloat16>(size_t(2) * D.shared_f * D.d);
        L->w2s = cv.take<__nv_bfloat16>(size_t(D.d) * D.shared_f);
        L->hs = cv.take<__nv_bfloat16>(size_t(T) * D.shared_f);
        L->ys = cv.take<__nv_bfloat16>(size_t(T) * D.d);
      }
    };
    plan(c);
    L->scratch_bytes = align_up(c.off, 256);
    if ((e = cudaMalloc(&L->scratch, L->scratch_bytes)) != cudaSuccess)
      return fail(set_error(MP_E_CAPACITY, "cannot allocate layer scratch (%zu bytes): %s", L->scratch_bytes,
                            cudaGetErrorString(e)));
    Carver real{L->scratch};
    plan(real);
    // zero the small control region (everything but the big activation buffers)
    if ((e = cudaMemset(L->scratch, 0, L->scratch_bytes)) != cudaSuccess)
      return fail(set_cuda_error(e, "cudaMemset(scratch)"));
  }

  // ---- peer-error word in mapped pinned host memory (no sync needed to read it)
  {
    void* hp = nullptr;
    if ((e = cudaHostAlloc(&hp, 64, cudaHostAllocMapped | cudaHostAllocPortable)) != cudaSuccess)
      return fail(set_cuda_error(e, "cudaHostAlloc(error word)"));
    memset(hp, 0, 64);
    L->err_host = static_cast<volatile uint32_t*>(hp);
    void* dp = nullptr;
    if ((e = cudaHostGetDevicePointer(&dp, hp, 0)) != cudaSuccess)
      return fail(set_cuda_error(e, "cudaHostGetDevicePointer(error word)"));
    L->err_host_d = static_cast<uint32_t*>(dp);
  }

  // ---- own pointer arrays (peers filled by mp_layer_open_peers)
  {
    void* host[6 * 8] = {};
    host[0 * 8 + L->rank] = L->recv;
    host[1 * 8 + L->rank] = L->ret;
    host[5 * 8 + L->rank] = L->recv_src;
    host[2 * 8 + L->rank] = L->flags;
    host[3 * 8 + L->rank] = L->counts;
    host[4 * 8 + L->rank] = L->counts + L->G * D.E;
    if ((e = cudaMemcpy(L->ptr_arrays, host, sizeof(host), cudaMemcpyHostToDevice)) != cudaSuccess)
      return fail(set_cuda_error(e, "cudaMemcpy(ptr arrays)"));
  }

  // ---- tensor maps over fixed buffers
  int r;
  if ((r = encode_tmap_bf16_2d(&L->tm_recv, L->recv, uint64_t(L->recv_cap), uint64_t(D.d), 128)) != MP_OK)
    return fail(r);
  if ((r = encode_tmap_bf16_2d(&L->tm_h, L->h, uint64_t(L->recv_cap), uint64_t(D.f), 128)) != MP_OK) return fail(r);
  if (D.n_slots > 0) {
    // W13 viewed as [n_slots * 3f, d] (slot s rows start at 3f*s); W2 as
    // [n_slots * 3d, f] (slot s rows start at 3d*s + 2d)
    if ((r = encode_tmap_bf16_2d(&L->tm_w13, L->pool, uint64_t(D.n_slots) * 3 * D.f, uint64_t(D.d), 256)) != MP_OK)
      return fail(r);
    if ((r = encode_tmap_bf16_2d(&L->tm_w2, L->pool, uint64_t(D.n_slots) * 3 * D.d, uint64_t(D.f), 256)) != MP_OK)
      return fail(r);
    if ((r = encode_tmap_bf16_2d(&L->tm_w13_p, L->pool, uint64_t(D.n_slots) * 3 * D.f, uint64_t(D.d), 128)) != MP_OK)
      return fail(r);
    if ((r = encode_tmap_bf16_2d(&L->tm_w2_p, L->pool, uint64_t(D.n_slots) * 3 * D.d, uint64_t(D.f), 128)) != MP_OK)
      return fail(r);
  }
  // CTA pairs (256-row tiles) when the average expert group is large
  L->pair_routed = int64_t(D.world) * D.max_tokens * D.top_k >= int64_t(512) * D.E ? 1 : 0;
  // many small expert groups (Qwen / DeepSeek): weight-bound small groups run concurrently
  // with the compute-bound large ones on a disjoint set of SMs
  L->split_m = D.E >= 16 ? 256 : 0;
  if (const char* env = getenv("MP_GEMM_SPLIT_M")) L->split_m = atoi(env);
  if (const char* env = getenv("MP_GEMM_SMALL_GRID")) {
    L->small_grid = std::max(2, atoi(env)) & ~1;
    L->small_grid_fixed = true;
  }
  // with the small groups split off, the remaining (>= split_m rows) groups run on CTA pairs
  if (L->split_m >= 256) L->pair_routed = 1;
  if (const char* env = getenv("MP_GEMM_PAIR")) L->pair_routed = L->pair_shared = atoi(env) ? 1 : 0;
  if (L->split_m > 0) {
    if ((e = cudaStreamCreateWithFlags(&L->side, cudaStreamNonBlocking)) != cudaSuccess)
      return fail(set_cuda_error(e, "cudaStreamCreate(side)"));
    if ((e = cudaEventCreateWithFlags(&L->ev_fork, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&L->ev_join, cudaEventDisableTiming)) != cudaSuccess)
      return fail(set_cuda_error(e, "cudaEventCreate(split)"));
  }
  // the shared expert rides in the routed launches (either kernel) as the aux problem
  L->fuse_shared = (D.shared_f > 0 && D.n_slots > 0) ? 1 : 0;
  if (const char* env = getenv("MP_STREAM_ROWS")) L->stream_rows = atoi(env);
  if (const char* env = getenv("MP_GEMM_TAILS")) L->tail_max = atoi(env);
  if (const char* env = getenv("MP_SIDE_SHARED_ROWS")) L->side_shared_rows = atoi(env);
  if (const char* env = getenv("MP_FUSE_SHARED")) L->fuse_shared = L->fuse_shared && atoi(env) != 0;
  if (D.shared_f > 0) {
    if ((r = encode_tmap_bf16_2d(&L->tm_w13s, L->w13s, uint64_t(2) * D.shared_f, uint64_t(D.d), 256)) != MP_OK)
      return fail(r);
    if ((r = encode_tmap_bf16_2d(&L->tm_w2s, L->w2s, uint64_t(D.d), uint64_t(D.shared_f), 256)) != MP_OK)
      return fail(r);
    if ((r = encode_tmap_bf16_2d(&L->tm_hs, L->hs, uint64_t(D.max_tokens), uint64_t(D.shared_f), 128)) != MP_OK)
      return fail(r);
    if ((r = encode_tmap_bf16_2d(&L->tm_w13s_p, L->w13s, uint64_t(2) * D.shared_f, uint64_t(D.d), 128)) != MP_OK)
      return fail(r);
    if ((r = encode_tmap_bf16_2d(&L->tm_w2s_p, L->w2s, uint64_t(D.d), uint64_t(D.shared_f), 128)) != MP_OK)
      return fail(r);
  }
  if (L->G == 1) L->peers_open = true;
  *out = L;
  return MP_OK;
}

int mp_layer_destroy(mp_layer* L) {
  if (!L) return MP_OK;
  DeviceGuard dg(L->desc.device);
  for (int p = 0; p < 8; ++p) {
    if (L->peer_window[p]) cudaIpcCloseMemHandle(L->peer_window[p]);
    if (L->peer_pool[p]) cudaIpcCloseMemHandle(L->peer_pool[p]);
  }
  if (L->ev_fork) cudaEventDestroy(L->ev_fork);
  if (L->ev_join) cudaEventDestroy(L->ev_join);
  if (L->side) cudaStreamDestroy(L->side);
  if (L->scratch) cudaFree(L->scratch);
  if (L->err_host) cudaFreeHost(const_cast<uint32_t*>(L->err_host));
  if (L->src_image) cudaFree(L->src_image);
  if (L->window) cudaFree(L->window);
  if (L->pool) cudaFree(L->pool);
  delete L;
  return MP_OK;
}

int mp_layer_get_ptrs(mp_layer* L, mp_layer_ptrs* o) {
  if (!L || !o) return set_error(MP_E_ARG, "mp_layer_get_ptrs: null pointer");
  memset(o, 0, sizeof(*o));
  o->pool = L->pool;
  o->wg = L->wg;
  o->bias = L->bias;
  o->w13_shared = L->w13s;
  o->w2_shared = L->w2s;
  o->idx = L->idx;
  o->w = L->w;
  o->pos_dst = L->pos_dst;
  o->pos_row = L->pos_row;
  o->recv = L->recv;
  o->h = L->h;
  o->ret = L->ret;
  o->recv_src = L->recv_src;
  o->hist = L->hist;
  o->counts = L->counts;
  o->shared_gate = L->sgate;
  o->batch_counts = L->batch_counts;
  o->recv_cap = L->recv_cap;
  o->slot_bytes = int64_t(L->slot_bytes);
  return MP_OK;
}

int mp_layer_export_handles(mp_layer* L, void* handles_out) {
  if (!L || !handles_out) return set_error(MP_E_ARG, "mp_layer_export_handles: null pointer");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  DeviceGuard dg(L->desc.device);
  MP_CUDA(dg.status);
  cudaIpcMemHandle_t hw, hp;
  MP_CUDA(cudaIpcGetMemHandle(&hw, L->window));
  MP_CUDA(cudaIpcGetMemHandle(&hp, L->pool));
  memcpy(handles_out, &hw, 64);
  memcpy(static_cast<uint8_t*>(handles_out) + 64, &hp, 64);
  return MP_OK;
}

int mp_layer_open_peers(mp_layer* L, const void* all_handles) {
  if (!L || !all_handles) return set_error(MP_E_ARG, "mp_layer_open_peers: null pointer");
  DeviceGuard dg(L->desc.device);
  MP_CUDA(dg.status);
  const uint8_t* h = static_cast<const uint8_t*>(all_handles);
  void* host[6 * 8] = {};
  for (int p = 0; p < L->G; ++p) {
    uint8_t* win;
    if (p == L->rank) {
      win = L->window;
    } else {
      if (!L->peer_window[p]) {
        cudaIpcMemHandle_t hw, hp;
        memcpy(&hw, h + 128 * p, 64);
        memcpy(&hp, h + 128 * p + 64, 64);
        void* pw = nullptr;
        void* pp = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&pw, hw, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess)
          return set_error(MP_E_PEER, "cudaIpcOpenMemHandle(window of rank %d): %s", p, cudaGetErrorString(e));
        e = cudaIpcOpenMemHandle(&pp, hp, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess)
          return set_error(MP_E_PEER, "cudaIpcOpenMemHandle(pool of rank %d): %s", p, cudaGetErrorString(e));
        L->peer_window[p] = static_cast<uint8_t*>(pw);
        L->peer_pool[p] = static_cast<uint8_t*>(pp);
      }
      win = L->peer_window[p];
    }
    host[0 * 8 + p] = win + L->off_recv;
    host[1 * 8 + p] = win + L->off_ret;
    host[5 * 8 + p] = win + L->off_src;
    host[2 * 8 + p] = win + L->off_flags;
    host[3 * 8 + p] = win + L->off_counts;
    host[4 * 8 + p] = win + L->off_counts + size_t(L->G) * L->desc.E * 4;
  }
  MP_CUDA(cudaMemcpy(L->ptr_arrays, host, sizeof(host), cudaMemcpyHostToDevice));
  L->peers_open = true;
  return MP_OK;
}

int mp_layer_set_routes(mp_layer* L, const int32_t* route, const int32_t* slot_of, void* stream) {
  if (!L || !route || !slot_of) return set_error(MP_E_ARG, "mp_layer_set_routes: null pointer");
  const int G = L->G, E = L->desc.E;
  for (int s = 0; s < G; ++s)
    for (int e = 0; e < E; ++e) {
      const int t = route[s * E + e];
      if (t < 0 || t >= G)
        return set_error(MP_E_UNPLACED, "expert %d routed from GPU %d to GPU %d: placed nowhere", e, s, t);
      if (t == L->rank && (slot_of[e] < 0 || slot_of[e] >= L->desc.n_slots))
        return set_error(MP_E_UNPLACED, "expert %d of GPU %d's traffic is routed here but holds no slot (slot %d)", e,
                         s, slot_of[e]);
    }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DeviceGuard dg(L->desc.device);
  MP_CUDA(dg.status);
  // small synchronous staging: route tables change once per placement
  std::vector<int32_t> r(route, route + G * E), so(slot_of, slot_of + E);
  MP_CUDA(cudaMemcpyAsync(L->route_d, r.data(), r.size() * 4, cudaMemcpyHostToDevice, st));
  MP_CUDA(cudaMemcpyAsync(L->slot_of_d, so.data(), so.size() * 4, cudaMemcpyHostToDevice, st));
  MP_CUDA(cudaStreamSynchronize(st));
  L->routes_set = true;
  return MP_OK;
}

int mp_layer_prepare_router(mp_layer* L, void* stream) {
  if (!L) return set_error(MP_E_ARG, "mp_layer_prepare_router: null layer");
  DeviceGuard dg(L->desc.device);
  MP_CUDA(dg.status);
  MP_TRY(launch_router_pack(L->wg, L->desc.E + (L->desc.shared_gate ? 1 : 0), L->desc.d, L->wg_packed,
                            static_cast<cudaStream_t>(stream)));
  L->router_ready = true;
  return MP_OK;
}

namespace {

// Stage-boundary events of mp_layer_forward_timed (NULL entries skipped).
struct Marker {
  void* const* events;
  cudaStream_t st;
  int i = 0;
  int mark() {
    if (events && events[i]) {
      cudaError_t e = cudaEventRecord(static_cast<cudaEvent_t>(events[i]), st);
      if (e != cudaSuccess) return set_cuda_error(e, "cudaEventRecord(stage)");
    }
    ++i;
    return MP_OK;
  }
  int mark_on(int idx, cudaStream_t s) {
    if (events && events[idx]) {
      cudaError_t e = cudaEventRecord(static_cast<cudaEvent_t>(events[idx]), s);
      if (e != cudaSuccess) return set_cuda_error(e, "cudaEventRecord(stage)");
    }
    return MP_OK;
  }
};

int check_forward_args(mp_layer* L, const void* x, const void* out, int T, const char* who) {
  if (!L) return set_error(MP_E_ARG, "%s: null layer", who);
  if ((!x || !out) && T > 0) return set_error(MP_E_ARG, "%s: null x/out with T=%d", who, T);
  const mp_layer_desc& D = L->desc;
  if (T < 0 || T > D.max_tokens) return set_error(MP_E_SHAPE, "T=%d exceeds max_tokens=%d", T, D.max_tokens);
  if (!L->routes_set) return set_error(MP_E_UNPLACED, "%s: route table not set", who);
  if (!L->router_ready) return set_error(MP_E_ARG, "%s: router weights not prepared", who);
  // a peer wait of an earlier forward timed out: its outputs were garbage and the
  // protocol is out of step -- refuse to run (read from mapped host memory, no sync)
  if (const uint32_t bad = *L->err_host)
    return set_error(MP_E_PEER, "an earlier forward timed out waiting for NVLink peers (ranks mask 0x%x)", bad);
  return MP_OK;
}

// The shared expert's dense tensor map over this forward's x.
int bind_x(mp_layer* L, const void* x, int T) {
  if (L->desc.shared_f > 0 && T > 0 && (L->tm_x_ptr != x || L->tm_x_rows != T)) {
    MP_TRY(encode_tmap_bf16_2d(&L->tm_x, x, uint64_t(std::max(T, 1)), uint64_t(L->desc.d), 128));
    L->tm_x_ptr = x;
    L->tm_x_rows = T;
  }
  return MP_OK;
}

// K3: the local experts' grouped SwiGLU GEMMs over the receive buffer, groups derived from
// the count table (counts_all [+ parity half]) and the route table; the shared expert rides in
// the routed launches when the plan fuses it.  GEMM2 writes each row to ret_ptrs[origin][pair]
// (scatter, the fused NVLink return) or, ret_ptrs == nullptr, in place of its received row.
int stage_experts(mp_layer* L, int T, const int32_t* counts_all, const uint32_t* parity, cudaStream_t st,
                  Marker& mk, const PeerSync* sw, PeerSync* ps_ret, __nv_bfloat16* const* ret_ptrs, int& launches) {
  const mp_layer_desc& D = L->desc;
  const int G = L->G, E = D.E, k = D.top_k;
  // Per-forward K3 plan.  With few rows per expert (small batches) every group is
  // weight-bound: stream all of them over every SM on the 1-CTA kernel instead of
  // confining them to the small-group side chain (the shared expert rides along as
  // the aux problem of those launches).
  const int64_t avg_rows = int64_t(G) * T * k / std::max(1, E);
  const bool stream_plan = L->split_m > 0 && avg_rows < L->stream_rows;
  const bool split = L->split_m > 0 && !stream_plan;
  const bool fused = L->fuse_shared && D.shared_f > 0 && T > 0;
  L->last_split = split ? L->split_m : 0;
  L->last_fused = fused ? 1 : 0;
  L->last_pair = stream_plan ? 0 : L->pair_routed;
  if (D.shared_f > 0 && T > 0 && !fused) {
    GroupSpec gsh;
    gsh.mode = 2;
    gsh.single_m = T;
    const int ps = L->pair_shared;
    MP_TRY(launch_grouped_gemm(L->tm_x, ps ? L->tm_w13s_p : L->tm_w13s, gsh, 2 * D.shared_f, D.d, 0, 0, L->hs,
                               D.shared_f, 1, 0, st, ps));
    MP_TRY(launch_grouped_gemm(L->tm_hs, ps ? L->tm_w2s_p : L->tm_w2s, gsh, D.d, D.shared_f, 0, 0, L->ys, D.d, 0, 0,
                               st, ps));
    launches += 2;
  }
  MP_TRY(mk.mark());  // 5 shared expert
  MP_TRY(mk.mark());  // 6 (dispatch barrier: folded into the permute tail / GEMM1 producers)
  if (D.n_slots > 0) {
    GroupSpec gs;
    gs.mode = 1;
    // F2 per-source dispatch waits: measured 2-4% slower than one wait for every rank's epoch
    // B before the first routed tile (G = 2 / 4, Mixtral and DeepSeek), so off unless MP_F2=1
    static const bool per_source = [] {
      const char* env = getenv("MP_F2");
      return env != nullptr && atoi(env) != 0;
    }();
    gs.per_source = per_source ? 1 : 0;
    gs.counts = counts_all;
    gs.parity = parity;
    gs.route = L->route_d;
    gs.slot_of = L->slot_of_d;
    gs.G = G;
    gs.E = E;
    gs.rank = L->rank;
    const int pr = stream_plan ? 0 : L->pair_routed;
    // side-chain SMs: with many rows per expert (G*T*k/E >= 1024, e.g. 4+ GPUs) few groups
    // stay below split_m, so the chain gets 8 SMs instead of 20 (measured: +3-5% at G = 4)
    const int small_grid = L->small_grid_fixed ? L->small_grid : (avg_rows >= 1024 ? 8 : 20);
    L->last_small_grid = small_grid;
    const int big_grid = split ? kNumSMs - small_grid : 0;
    // C is raised by the last GEMM2 CTA of both chains
    if (ps_ret) ps_ret->total = grouped_gemm_ctas(big_grid, pr) + (split ? grouped_gemm_ctas(small_grid, 0) : 0);
    const int32_t* scatter_src = ret_ptrs ? L->recv_src : nullptr;
    __nv_bfloat16* out2 = ret_ptrs ? L->ret : L->recv;
    // the fused shared expert's last ms rows (a multiple of 256, so neither chain pads a tile)
    // can ride on the side chain, whose weight-bound small groups leave it slack
    const int ms = (split && fused) ? std::min(L->side_shared_rows / 256 * 256, T / 256 * 256) : 0;
    AuxProblem saux1, saux2;
    if (ms > 0) {
      const size_t r0 = size_t(T - ms);
      MP_TRY(encode_tmap_bf16_2d(&saux1.tmA, static_cast<const __nv_bfloat16*>(L->tm_x_ptr) + r0 * D.d,
                                 uint64_t(ms), uint64_t(D.d), 128));
      saux1.tmB = L->tm_w13s;
      saux1.out = L->hs + r0 * D.shared_f;
      saux1.out_ld = D.shared_f;
      saux1.m = ms;
      saux1.N = 2 * D.shared_f;
      saux1.K = D.d;
      MP_TRY(encode_tmap_bf16_2d(&saux2.tmA, L->hs + r0 * D.shared_f, uint64_t(ms), uint64_t(D.shared_f), 128));
      saux2.tmB = L->tm_w2s;
      saux2.out = L->ys + r0 * D.d;
      saux2.out_ld = D.d;
      saux2.m = ms;
      saux2.N = D.d;
      saux2.K = D.shared_f;
    }
    if (split) {
      // fork: small groups (weight-bound) on the side stream over small_grid SMs, large
      // groups (compute-bound) on the main stream over the rest, then join
      GroupSpec gsmall = gs;
      gsmall.m_hi = L->split_m;
      gs.m_lo = L->split_m;
      if (pr && L->tail_max > 0) {  // big groups' short pair-tile tails -> the 1-CTA side chain
        gs.tail_role = 1;
        gsmall.tail_role = 2;
        gs.tail_max = gsmall.tail_max = L->tail_max;
        gs.tail_block = gsmall.tail_block = 256;
      }
      MP_CUDA(cudaEventRecord(L->ev_fork, st));
      MP_CUDA(cudaStreamWaitEvent(L->side, L->ev_fork, 0));
      MP_TRY(mk.mark_on(11, L->side));
      // (no PDL on the split chains: early-scheduled CTAs would contend for the other chain's SMs)
      MP_TRY(launch_grouped_gemm(L->tm_recv, L->tm_w13, gsmall, 2 * D.f, D.d, 3 * D.f, 0, L->h, D.f, 1,
                                 small_grid, L->side, 0, nullptr, nullptr, false, ms > 0 ? &saux1 : nullptr, sw));
      MP_TRY(launch_grouped_gemm(L->tm_h, L->tm_w2, gsmall, D.d, D.f, 3 * D.d, 2 * D.d, out2, D.d, 0,
                                 small_grid, L->side, 0, scatter_src, ret_ptrs, false, ms > 0 ? &saux2 : nullptr,
                                 ps_ret));
      MP_TRY(mk.mark_on(12, L->side));
      MP_CUDA(cudaEventRecord(L->ev_join, L->side));
      launches += 2;
    }
    const bool pdl = !split;
    // fused shared expert: its GEMM1 / GEMM2 tiles ride in the routed launches
    AuxProblem aux1, aux2;
    if (fused) {
      aux1.tmA = L->tm_x;
      aux1.tmB = pr ? L->tm_w13s_p : L->tm_w13s;
      aux1.out = L->hs;
      aux1.out_ld = D.shared_f;
      aux1.m = T - ms;
      aux1.N = 2 * D.shared_f;
      aux1.K = D.d;
      aux2.tmA = L->tm_hs;
      aux2.tmB = pr ? L->tm_w2s_p : L->tm_w2s;
      aux2.out = L->ys;
      aux2.out_ld = D.d;
      aux2.m = T - ms;
      aux2.N = D.d;
      aux2.K = D.shared_f;
    }
    MP_TRY(launch_grouped_gemm(L->tm_recv, pr ? L->tm_w13_p : L->tm_w13, gs, 2 * D.f, D.d, 3 * D.f, 0, L->h, D.f, 1,
                               big_grid, st, pr, nullptr, nullptr, pdl, fused ? &aux1 : nullptr, sw));
    MP_TRY(mk.mark());  // 7 GEMM1 (SwiGLU)
    // GEMM2 epilogue returns every output row to its origin GPU (NVLink stores)
    MP_TRY(launch_grouped_gemm(L->tm_h, pr ? L->tm_w2_p : L->tm_w2, gs, D.d, D.f, 3 * D.d, 2 * D.d, out2, D.d, 0,
                               big_grid, st, pr, scatter_src, ret_ptrs, pdl, fused ? &aux2 : nullptr, ps_ret));
    if (split) MP_CUDA(cudaStreamWaitEvent(st, L->ev_join, 0));
    launches += 2;
  } else {
    MP_TRY(mk.mark());
    if (ps_ret && G > 1) {  // no GEMM2 here to raise C
      MP_TRY(launch_peer_sync(*ps_ret, nullptr, E, 1, st));
      ++launches;
    }
  }
  MP_TRY(mk.mark());  // 8 GEMM2
  return MP_OK;
}

}  // namespace

static int layer_forward(mp_layer* L, const void* x, void* out, int T, void* stream, void* const* events) {
  MP_TRY(check_forward_args(L, x, out, T, "mp_layer_forward"));
  if (!L->peers_open) return set_error(MP_E_PEER, "mp_layer_forward: peers not opened (G=%d)", L->G);
  const mp_layer_desc& D = L->desc;
  DeviceGuard dg(D.device);
  MP_CUDA(dg.status);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int G = L->G, E = D.E, k = D.top_k, rank = L->rank;
  auto** recv_ptrs = reinterpret_cast<__nv_bfloat16**>(L->ptr_arrays + 0 * 8);
  auto** ret_ptrs = reinterpret_cast<__nv_bfloat16**>(L->ptr_arrays + 1 * 8);
  auto** src_ptrs = reinterpret_cast<int32_t**>(L->ptr_arrays + 5 * 8);
  auto** flag_ptrs = reinterpret_cast<uint32_t**>(L->ptr_arrays + 2 * 8);
  auto** count_ptrs = reinterpret_cast<int32_t**>(L->ptr_arrays + 3 * 8);  // [parity][peer]
  int launches = 0;
  Marker mk{events, st};
  MP_TRY(bind_x(L, x, T));

  // NVLink flag protocol (G > 1), folded into the kernels: router tail raises A
  // (counts published), permute waits A and its tail raises B (rows sent), GEMM1
  // producers wait B, the GEMM2 tails raise C (rows returned), combine waits C
  PeerSync ps0;
  if (G > 1) {
    ps0.flag_ptrs = flag_ptrs;
    ps0.count_ptrs = count_ptrs;
    ps0.state = L->sync_state;
    ps0.err = L->err;
    ps0.err_host = L->err_host_d;
    ps0.G = G;
    // one bounded peer wait: 30 s, or MP_PEER_TIMEOUT_MS (tests), capped below the 40 s
    // mbarrier bound of the warps that wait behind a waiting producer
    static const uint64_t timeout_ns = [] {
      const char* env = getenv("MP_PEER_TIMEOUT_MS");
      const long long ms = env ? atoll(env) : 30000;
      return uint64_t(std::min(std::max(ms, 1ll), 30000ll)) * 1000000ull;
    }();
    ps0.timeout_ns = timeout_ns;
    ps0.rank = rank;
  }
  PeerSync ps_wait = ps0, ps_perm = ps0, ps_ret = ps0;
  ps_wait.wait = 1;
  ps_perm.wait = 1;
  ps_perm.ticket = L->perm_ticket;
  ps_perm.total = 1;  // launch_permute sets its grid
  ps_ret.ticket = L->ret_ticket;

  MP_TRY(mk.mark());  // 0
  if (T > 0) {
    MP_TRY(launch_router(static_cast<const __nv_bfloat16*>(x), L->wg_packed, L->bias, T, D.d, E, D.shared_gate, k,
                         D.score_mode, D.renorm, L->idx, L->w, L->sgate, L->hist, L->blk_counts, L->batch_counts,
                         L->ticket, L->count_acc, st, G > 1 ? &ps0 : nullptr));
    ++launches;
  } else if (G > 1) {
    // no router / permute on this origin: publish zero counts, raise A and B
    MP_TRY(launch_peer_sync(ps0, L->batch_counts, E, 2, st));
    ++launches;
  } else {
    MP_CUDA(cudaMemsetAsync(L->batch_counts, 0, size_t(E) * 4, st));
  }
  MP_TRY(mk.mark());  // 1 router (+ per-batch counts, count exchange)
  const int32_t* counts_all = G > 1 ? L->counts : L->batch_counts;
  const uint32_t* parity = G > 1 ? L->sync_state + 2 : nullptr;
  MP_TRY(mk.mark());  // 2 (count exchange: folded into the router tail / permute prologue)
  MP_TRY(mk.mark());  // 3 (layout: folded into permute / GEMM prologues)
  if (T > 0) {
    MP_TRY(launch_permute(static_cast<const __nv_bfloat16*>(x), L->idx, L->route_d, counts_all, parity,
                          L->blk_counts, src_ptrs, rank, G, T, D.d, E, k, recv_ptrs, L->pos_dst, L->pos_row, st,
                          G > 1 ? &ps_perm : nullptr));
    ++launches;
  }
  MP_TRY(mk.mark());  // 4 permute + dispatch
  MP_TRY(stage_experts(L, T, counts_all, parity, st, mk, G > 1 ? &ps_wait : nullptr, G > 1 ? &ps_ret : nullptr,
                       ret_ptrs, launches));
  MP_TRY(mk.mark());  // 9 (return barrier: folded into the GEMM2 tails / combine prologue)
  if (T > 0) {
    MP_TRY(launch_combine(L->ret, L->w, T, D.d, k, D.shared_f > 0 ? L->ys : nullptr,
                          D.shared_gate ? L->sgate : nullptr, static_cast<__nv_bfloat16*>(out), st,
                          G > 1 ? &ps_wait : nullptr));
    ++launches;
  }
  MP_TRY(mk.mark());  // 10 combine + return
  L->last_launches = launches;
  return MP_OK;
}

int mp_layer_forward(mp_layer* L, const void* x, void* out, int T, void* stream) {
  return layer_forward(L, x, out, T, stream, nullptr);
}

int mp_layer_forward_timed(mp_layer* L, const void* x, void* out, int T, void* stream, void* const* events) {
  if (!events) return set_error(MP_E_ARG, "mp_layer_forward_timed: null events");
  return layer_forward(L, x, out, T, stream, events);
}

// ---- stage entries (host-driven transport, e.g. NCCL all-to-all-v; standalone K1 / K2 / K3 / K5)
namespace {
// Points the permute's destinations / the combine's sources at receive-layout images:
// slot 8*a + D (a = 0 permute rows, 1 permute recv_src, 2 combine rows) = own buffer for
// D == rank, else image D of the caller's staging buffer.
int upload_stage_ptrs(mp_layer* L, int which, void* base, size_t elem_bytes, void* own, cudaStream_t st) {
  bool changed = !L->stage_uploaded;
  for (int D = 0; D < 8; ++D) {
    void* p = nullptr;
    if (D < L->G)
      p = D == L->rank ? own
                       : (base ? static_cast<uint8_t*>(base) + size_t(D) * size_t(L->recv_cap) * elem_bytes : nullptr);
    changed |= L->stage_host[8 * which + D] != p;
    L->stage_host[8 * which + D] = p;
  }
  if (!changed) return MP_OK;
  MP_CUDA(cudaMemcpyAsync(L->stage_ptrs, L->stage_host, sizeof(L->stage_host), cudaMemcpyHostToDevice, st));
  MP_CUDA(cudaStreamSynchronize(st));
  L->stage_uploaded = true;
  return MP_OK;
}
}  // namespace

int mp_layer_route(mp_layer* L, const void* x, int T, void* stream) {
  MP_TRY(check_forward_args(L, x, x, T, "mp_layer_route"));
  DeviceGuard dg(L->desc.device);
  MP_CUDA(dg.status);
  const mp_layer_desc& D = L->desc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (T == 0) {
    MP_CUDA(cudaMemsetAsync(L->batch_counts, 0, size_t(D.E) * 4, st));
    return MP_OK;
  }
  return launch_router(static_cast<const __nv_bfloat16*>(x), L->wg_packed, L->bias, T, D.d, D.E, D.shared_gate,
                       D.top_k, D.score_mode, D.renorm, L->idx, L->w, L->sgate, L->hist, L->blk_counts,
                       L->batch_counts, L->ticket, L->count_acc, st, nullptr);
}

int mp_layer_permute(mp_layer* L, const void* x, int T, const int32_t* counts_all, void* staging, void* stream) {
  MP_TRY(check_forward_args(L, x, x, T, "mp_layer_permute"));
  if (!counts_all) return set_error(MP_E_ARG, "mp_layer_permute: null count table");
  if (L->G > 1 && !staging) return set_error(MP_E_ARG, "mp_layer_permute: G=%d needs a staging buffer", L->G);
  DeviceGuard dg(L->desc.device);
  MP_CUDA(dg.status);
  const mp_layer_desc& D = L->desc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (L->G > 1 && !L->src_image) {
    cudaError_t e = cudaMalloc(&L->src_image, size_t(L->G) * size_t(L->recv_cap) * 4);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaMalloc(recv_src images)");
  }
  MP_TRY(upload_stage_ptrs(L, 0, staging, size_t(D.d) * 2, L->recv, st));
  MP_TRY(upload_stage_ptrs(L, 1, L->src_image, 4, L->recv_src, st));
  if (T == 0) return MP_OK;
  return launch_permute(static_cast<const __nv_bfloat16*>(x), L->idx, L->route_d, counts_all, nullptr, L->blk_counts,
                        reinterpret_cast<int32_t* const*>(L->stage_ptrs + 8), L->rank, L->G, T, D.d, D.E, D.top_k,
                        reinterpret_cast<__nv_bfloat16* const*>(L->stage_ptrs), L->pos_dst, L->pos_row, st, nullptr);
}

int mp_layer_experts(mp_layer* L, const void* x, int T, const int32_t* counts_all, void* stream) {
  MP_TRY(check_forward_args(L, x, x, T, "mp_layer_experts"));
  if (!counts_all) return set_error(MP_E_ARG, "mp_layer_experts: null count table");
  DeviceGuard dg(L->desc.device);
  MP_CUDA(dg.status);
  MP_TRY(bind_x(L, x, T));
  Marker mk{nullptr, static_cast<cudaStream_t>(stream)};
  int launches = 0;
  return stage_experts(L, T, counts_all, nullptr, static_cast<cudaStream_t>(stream), mk, nullptr, nullptr, nullptr,
                       launches);
}

int mp_layer_combine_gather(mp_layer* L, const void* ret_stage, int T, void* out, void* stream) {
  MP_TRY(check_forward_args(L, out, out, T, "mp_layer_combine_gather"));
  if (L->G > 1 && !ret_stage) return set_error(MP_E_ARG, "mp_layer_combine_gather: G=%d needs the return images", L->G);
  DeviceGuard dg(L->desc.device);
  MP_CUDA(dg.status);
  const mp_layer_desc& D = L->desc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  MP_TRY(upload_stage_ptrs(L, 2, const_cast<void*>(ret_stage), size_t(D.d) * 2, L->recv, st));
  if (T == 0) return MP_OK;
  return launch_combine(nullptr, L->w, T, D.d, D.top_k, D.shared_f > 0 ? L->ys : nullptr,
                        D.shared_gate ? L->sgate : nullptr, static_cast<__nv_bfloat16*>(out), st, nullptr,
                        reinterpret_cast<const __nv_bfloat16* const*>(L->stage_ptrs + 16), L->pos_dst, L->pos_row);
}

int mp_layer_last_launches(mp_layer* L) { return L ? L->last_launches : 0; }

int mp_layer_config(mp_layer* L, int key) {
  if (!L) return set_error(MP_E_ARG, "mp_layer_config: null layer");
  switch (key) {
    case MP_CFG_PAIR_ROUTED: return L->last_pair >= 0 ? L->last_pair : L->pair_routed;
    case MP_CFG_SPLIT_M: return L->last_split >= 0 ? L->last_split : L->split_m;
    case MP_CFG_SMALL_GRID:
      return (L->last_split >= 0 ? L->last_split : L->split_m) > 0
                 ? (L->last_small_grid > 0 ? L->last_small_grid : L->small_grid)
                 : 0;
    case MP_CFG_FUSE_SHARED: return L->last_fused >= 0 ? L->last_fused : L->fuse_shared;
    default: return set_error(MP_E_ARG, "mp_layer_config: key %d", key);
  }
}

int mp_layer_read_counts(mp_layer* L, int32_t* host_counts, void* stream) {
  if (!L || !host_counts) return set_error(MP_E_ARG, "mp_layer_read_counts: null pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DeviceGuard dg(L->desc.device);
  MP_CUDA(dg.status);
  MP_CUDA(cudaStreamSynchronize(st));
  const int G = L->G, E = L->desc.E;
  if (G == 1) {
    MP_CUDA(cudaMemcpy(host_counts, L->batch_counts, size_t(E) * 4, cudaMemcpyDeviceToHost));
  } else {
    uint32_t par = 0;  // parity of the last completed forward (device state)
    MP_CUDA(cudaMemcpy(&par, L->sync_state + 2, 4, cudaMemcpyDeviceToHost));
    MP_CUDA(cudaMemcpy(host_counts, L->counts + size_t(par & 1) * G * E, size_t(G) * E * 4, cudaMemcpyDeviceToHost));
  }
  return MP_OK;
}

int mp_layer_check(mp_layer* L, void* stream) {
  if (!L) return set_error(MP_E_ARG, "mp_layer_check: null layer");
  DeviceGuard dg(L->desc.device);
  MP_CUDA(dg.status);
  MP_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  uint32_t err = 0;
  MP_CUDA(cudaMemcpy(&err, L->err, 4, cudaMemcpyDeviceToHost));
  err |= *L->err_host;
  if (err) return set_error(MP_E_PEER, "NVLink flag wait timed out on ranks mask 0x%x", err);
  return MP_OK;
}

int mp_layer_sync_state(mp_layer* L, uint32_t* out, void* stream) {
  if (!L || !out) return set_error(MP_E_ARG, "mp_layer_sync_state: null pointer");
  DeviceGuard dg(L->desc.device);
  MP_CUDA(dg.status);
  MP_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  if (L->side) MP_CUDA(cudaStreamSynchronize(L->side));
  for (int i = 0; i < 16; ++i) out[i] = 0;
  MP_CUDA(cudaMemcpy(out, L->sync_state, 3 * 4, cudaMemcpyDeviceToHost));
  MP_CUDA(cudaMemcpy(out + 3, L->ticket, 4, cudaMemcpyDeviceToHost));
  MP_CUDA(cudaMemcpy(out + 4, L->perm_ticket, 4, cudaMemcpyDeviceToHost));
  MP_CUDA(cudaMemcpy(out + 5, L->ret_ticket, 4, cudaMemcpyDeviceToHost));
  MP_CUDA(cudaMemcpy(out + 6, L->err, 4, cudaMemcpyDeviceToHost));
  int32_t acc[64];
  MP_CUDA(cudaMemcpy(acc, L->count_acc, sizeof(acc), cudaMemcpyDeviceToHost));
  for (int e = 0; e < 64; ++e) out[7] += acc[e] != 0;
  if (L->G > 1) MP_CUDA(cudaMemcpy(out + 8, L->flags, size_t(L->G) * 4, cudaMemcpyDeviceToHost));
  return MP_OK;
}

int mp_layer_peer_probe(mp_layer* L, int peer, int64_t bytes, int reps, void* stream, float* ms_per_copy) {
  if (!L || !ms_per_copy) return set_error(MP_E_ARG, "mp_layer_peer_probe: null pointer");
  if (peer < 0 || peer >= L->G || peer == L->rank) return set_error(MP_E_ARG, "mp_layer_peer_probe: peer %d", peer);
  if (!L->peer_window[peer]) return set_error(MP_E_PEER, "mp_layer_peer_probe: peer %d not opened", peer);
  const int64_t cap = int64_t(L->off_ret - L->off_recv);  // the receive region of both windows
  if (bytes <= 0 || bytes > cap || reps < 1) return set_error(MP_E_ARG, "mp_layer_peer_probe: %lld bytes x %d",
                                                              (long long)bytes, reps);
  DeviceGuard dg(L->desc.device);
  MP_CUDA(dg.status);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaEvent_t a, b;
  MP_CUDA(cudaEventCreate(&a));
  MP_CUDA(cudaEventCreate(&b));
  // the peer's receive region -> ours, over the NVLink mapping opened by mp_layer_open_peers
  const uint8_t* src = L->peer_window[peer] + L->off_recv;
  uint8_t* dst = L->window + L->off_recv;
  cudaError_t e = cudaSuccess;
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) e = cudaMemcpyAsync(dst, src, size_t(bytes), cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = cudaEventRecord(a, st);
  for (int i = 0; i < reps && e == cudaSuccess; ++i)
    e = cudaMemcpyAsync(dst, src, size_t(bytes), cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = cudaEventRecord(b, st);
  if (e == cudaSuccess) e = cudaEventSynchronize(b);
  float ms = 0.f;
  if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (e != cudaSuccess) return set_cuda_error(e, "mp_layer_peer_probe");
  *ms_per_copy = ms / float(reps);
  return MP_OK;
}

int mp_layer_migrate(mp_layer* L, const mp_copy_op* ops, int n_ops, void* stream, void* done_event) {
  if (!L || (n_ops > 0 && !ops)) return set_error(MP_E_ARG, "mp_layer_migrate: null pointer");
  DeviceGuard dg(L->desc.device);
  MP_CUDA(dg.status);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int S = L->desc.n_slots;
  for (int i = 0; i < n_ops; ++i) {
    const mp_copy_op& op = ops[i];
    if (op.dst_slot < 0 || op.dst_slot >= S)
      return set_error(MP_E_CAPACITY, "migration target slot %d outside [0, %d)", op.dst_slot, S);
    if (op.src_rank < 0 || op.src_rank >= L->G) return set_error(MP_E_ARG, "migration source rank %d", op.src_rank);
    if (op.src_slot < 0) return set_error(MP_E_ARG, "migration source slot %d", op.src_slot);
    const uint8_t* src_pool = op.src_rank == L->rank ? L->pool : L->peer_pool[op.src_rank];
    if (!src_pool) return set_error(MP_E_PEER, "pool of rank %d not opened", op.src_rank);
    if (op.src_rank == L->rank && op.src_slot == op.dst_slot) continue;
    // one contiguous m_e-byte copy per slot; peer sources go over NVLink
    MP_CUDA(cudaMemcpyAsync(L->pool + size_t(op.dst_slot) * L->slot_bytes, src_pool + size_t(op.src_slot) * L->slot_bytes,
                            L->slot_bytes, cudaMemcpyDeviceToDevice, st));
  }
  if (done_event) MP_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(done_event), st));
  return MP_OK;
}

}  // extern "C"
