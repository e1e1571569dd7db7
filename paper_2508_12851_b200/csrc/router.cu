// K1: top-k softmax router with a fused, block-aggregated expert histogram.
//
// The reference has no router: expert sets are sampled per request
// (reference pkg/src/moeplace/sim.py:153-191) and folded into token-weighted
// activation counts by ActivationStats.ingest (reference
// pkg/src/moeplace/stats.py:82-96).  This kernel produces both from real
// activations in one pass over x:
//   logits[t,e] = <x[t], Wg[e]>  (+ bias[e])       -- exact contract below
//   idx[t,:]    = top-k experts by logit, descending, ties -> lower expert id
//   w[t,:]      = softmax weights (mode 0: softmax over the k selected logits,
//                 Mixtral; mode 1: softmax over all E, no renorm unless asked,
//                 Qwen1.5-MoE / DeepSeek-V2-Lite)
//   hist[e]    += #tokens whose top-k contains e   (token_count = 1 per token)
//
// Numerics contract (restated by oracle/moe_oracle.py:router_logits).  Every row
// a of x and of Wg (bf16) is put on an integer grid fixed by the row's largest
// magnitude:  E(a) = max(ef(max_k |a_k|) - 126, -100)  (ef = the bf16 exponent
// field, so max |a| < 2^E(a)),  q_k = rint(a_k * 2^(win - E(a)))  (round half to
// even), win = 21 for token rows and 14 for router-weight rows: |q| <= 2^win, and
// every bf16 element within 2^-13 (x) / 2^-6 (Wg) of its row maximum is exact.  Then
//   S[t,e]      = sum_k qx[t,k] * qw[e,k]          EXACT (an integer, |S| < 2^52)
//   logits[t,e] = f32( f64(rn_f32(S)) * 2^(E(x_t) + E(w_e) - 35) ) (+ bias[e], fp32)
// S is computed on the tensor cores from 8-bit limbs (x: three unsigned limbs of
// q + 2^22, Wg: two balanced signed limbs) with tcgen05.mma.kind::i8 into s32
// accumulators in TMEM -- integer arithmetic is associative, so the result does
// not depend on tile shapes, K splits or accumulation order, and the logits are
// bit-reproducible by any exact method.  The quantisation error (<= 2^-22 of the
// token row maximum, 2^-15 of the weight row maximum, per element) sits between
// fp32 and bf16 rounding.
//
// Kernel (router_i8_kernel): a cluster of `split` CTAs per 128-token tile, each
// CTA one contiguous K range of d:
//   1. every CTA reads its x range once for the per-token maxima; the maxima go to
//      every CTA of the cluster through DSMEM, so all CTAs share E(x_t);
//   2. the x range comes again (L2) by TMA, one 128-k block at a time into a 3-stage
//      shared-memory ring; each producer lane converts its row (limb j = byte j of the fp32
//      pattern of q + 1.5 * 2^23: an FFMA and byte permutes) and writes the three limb tiles
//      into TMEM (tcgen05.st); both Wg limbs arrive by one TMA as a [2N][128] tile; one thread
//      issues one MMA per (32-k step, x limb) with A from TMEM and N' = 2N, into four s32
//      accumulators, one per limb shift 8 (i + j);
//   3. the epilogue folds the four accumulators into int64 per (token, expert), the
//      cluster sums its K ranges through DSMEM (integer, exact), and each 32-token
//      router block is selected by one CTA: one warp per token, top-k by two
//      redux.sync rounds, gate weights, block histogram; the last CTA of the grid
//      produces the batch counts, the per-block prefix the permute needs and, at
//      G > 1, the count exchange with epoch A.
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "mp_internal.h"
#include "peer_sync.cuh"

namespace mp {

namespace rt {
constexpr int kTokens = 32;    // tokens per router block (the permute / histogram block)
constexpr int kMaxE = 64;      // routed experts
constexpr int kMaxK = 8;
constexpr int kWinX = 21;      // token rows: |q| <= 2^21 (three unsigned limbs, the top one biased)
constexpr int kWinW = 14;      // Wg rows:    |q| <= 2^14 (two balanced signed limbs)
constexpr int kMinExp = -100;  // E(a) floor: 2^(win - E) stays a normal fp32
constexpr float kMagic = 12582912.0f;           // 1.5 * 2^23
constexpr uint32_t kMagicBits = 0x4B400000u;    // its bit pattern
}  // namespace rt

int router_block_tokens() { return rt::kTokens; }
// MMA N: routed experts + gate row, rounded up to a multiple of 16
__host__ __device__ int router_n_pad(int E_tot) { return E_tot <= 16 ? 16 : (E_tot + 15) / 16 * 16; }

size_t router_packed_bytes(int E_tot, int d) {
  const size_t N = size_t(router_n_pad(E_tot));
  return 2 * N * size_t(d) + 8 * N + 4 * N;
}

#define MP_TRY_R(call)             \
  do {                             \
    const int _r = (call);         \
    if (_r != MP_OK) return _r;    \
  } while (0)

// E(a) from the largest |bf16| bit pattern of a row.
MP_DEV int row_exponent(uint32_t max_bits) { return max(int(max_bits >> 7) - 126, rt::kMinExp); }
// 2^(win - E) as fp32 bits
MP_DEV float row_scale(int e, int win) { return __uint_as_float(uint32_t(127 + win - e) << 23); }
// bit pattern of rn(a * scale + 1.5 * 2^23) = 0x4B400000 + rint(a * scale)
MP_DEV uint32_t quant_bits(float a, float scale) { return __float_as_uint(fmaf(a, scale, rt::kMagic)); }

// ---------------------------------------------------------------- Wg packing
// packed = [2][N][d] limbs | int64 R[N] | int32 E[N]: q = b0 + 2^8 b1 with balanced signed
// digits b0, b1 in [-128, 127] (|q| <= 2^14), R[e] = sum_k q[e][k].  Pad rows (e >= E_tot)
// are zero.  One CTA per row.
__global__ void __launch_bounds__(256) router_pack_kernel(const __nv_bfloat16* __restrict__ wg, int E_tot, int N,
                                                          int d, uint8_t* __restrict__ packed) {
  const int e = blockIdx.x, tid = threadIdx.x;
  const uint16_t* row = reinterpret_cast<const uint16_t*>(wg) + size_t(e) * d;
  const bool real = e < E_tot;
  __shared__ uint32_t mx_s[8];
  __shared__ long long sum_s[8];
  uint32_t m = 0;
  if (real)
    for (int k = tid; k < d; k += blockDim.x) m = max(m, uint32_t(row[k] & 0x7fffu));
  m = __reduce_max_sync(0xffffffffu, m);
  if ((tid & 31) == 0) mx_s[tid >> 5] = m;
  __syncthreads();
  m = 0;
  for (int i = 0; i < 8; ++i) m = max(m, mx_s[i]);
  const int ex = row_exponent(m);
  const float sc = row_scale(ex, rt::kWinW);
  long long s = 0;
  for (int k = tid; k < d; k += blockDim.x) {
    int q = 0;
    if (real) q = int(quant_bits(__uint_as_float(uint32_t(row[k]) << 16), sc) - rt::kMagicBits);
    s += q;
    const int b0 = ((q + 128) & 255) - 128, b1 = (q - b0) / 256;
    packed[(size_t(0) * N + e) * d + k] = uint8_t(int8_t(b0));
    packed[(size_t(1) * N + e) * d + k] = uint8_t(int8_t(b1));
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((tid & 31) == 0) sum_s[tid >> 5] = s;
  __syncthreads();
  if (tid == 0) {
    long long tot = 0;
    for (int i = 0; i < 8; ++i) tot += sum_s[i];
    reinterpret_cast<long long*>(packed + 2 * size_t(N) * d)[e] = tot;
    reinterpret_cast<int*>(packed + 2 * size_t(N) * d + 8 * size_t(N))[e] = real ? ex : 0;
  }
}

int launch_router_pack(const __nv_bfloat16* wg, int E_tot, int d, uint8_t* packed, cudaStream_t stream) {
  if (d % 256 != 0) return set_error(MP_E_SHAPE, "router d=%d not a multiple of 256", d);
  if (E_tot < 1 || E_tot > rt::kMaxE + 1) return set_error(MP_E_SHAPE, "router: %d weight rows", E_tot);
  const int N = router_n_pad(E_tot);
  router_pack_kernel<<<unsigned(N), 256, 0, stream>>>(wg, E_tot, N, d, packed);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MP_OK : set_cuda_error(e, "router_pack_kernel launch");
}

// ---------------------------------------------------------------- selection
// Order-preserving 32-bit key of an fp32 logit (-0 canonicalised to +0, so equal logits get
// equal keys): larger logit <=> larger unsigned key.
MP_DEV uint32_t logit_key(float v) {
  const uint32_t u = __float_as_uint(v + 0.0f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Warp-collective top-k + gate weights of NT tokens in lockstep (their warp reductions are
// independent, so they pipeline) from their logits (lane l holds experts l and l + 32 of token
// i in v0[i], v1[i]): k rounds of a warp arg-max -- larger logit, ties -> lower id, as two
// redux.sync reductions over order-preserving keys -- then softmax over the k (mode 0) or
// over all E (mode 1, optional renormalisation).  Lane j < k writes idx_row[i][j] /
// w_row[i][j] and bumps cnt_s.  Tokens with valid[i] == false only ride along.
template <int NT>
MP_DEV void select_topk_store(const float (&v0)[NT], const float (&v1)[NT], const bool (&valid)[NT], int E, int k,
                              int score_mode, int renorm, int32_t* const (&idx_row)[NT],
                              float* const (&w_row)[NT], int* cnt_s) {
  const int lane = lane_id();
  // candidates of this lane: expert lane (v0) and lane + 32 (v1); taken/absent -> key 0
  uint32_t k0[NT], k1[NT];
  float my_v[NT], mx[NT];  // lane j < k keeps the j-th selected logit and expert
  int my_i[NT];
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    k0[i] = lane < E ? logit_key(v0[i]) : 0u;
    k1[i] = lane + 32 < E ? logit_key(v1[i]) : 0u;
    my_v[i] = -INFINITY;
    mx[i] = 0.f;
    my_i[i] = 0;
  }
#pragma unroll 1
  for (int j = 0; j < k; ++j) {
    uint32_t bk[NT], bi[NT];
    bool use1[NT];
#pragma unroll
    for (int i = 0; i < NT; ++i) {
      use1[i] = k1[i] > k0[i];  // ties inside the lane: the lower id (lane) wins
      bk[i] = use1[i] ? k1[i] : k0[i];
    }
    uint32_t mk[NT];
#pragma unroll
    for (int i = 0; i < NT; ++i) mk[i] = __reduce_max_sync(0xffffffffu, bk[i]);
#pragma unroll
    for (int i = 0; i < NT; ++i) {
      const uint32_t cand = (bk[i] == mk[i] && mk[i] != 0u) ? uint32_t(use1[i] ? lane + 32 : lane) : 0xffffffffu;
      bi[i] = __reduce_min_sync(0xffffffffu, cand);
    }
#pragma unroll
    for (int i = 0; i < NT; ++i) {
      const float bv = __shfl_sync(0xffffffffu, bi[i] >= 32 ? v1[i] : v0[i], bi[i] & 31);
      if (j == 0) mx[i] = bv;
      if (lane == j) { my_v[i] = bv; my_i[i] = int(bi[i]); }
      if (bi[i] == uint32_t(lane)) k0[i] = 0u;
      if (bi[i] == uint32_t(lane + 32)) k1[i] = 0u;
    }
  }
  // weights: lane j < k owns w_j
  float ej[NT], denom[NT];
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    ej[i] = lane < k ? __expf(my_v[i] - mx[i]) : 0.f;
    denom[i] = score_mode == 0 ? ej[i]
                               : (lane < E ? __expf(v0[i] - mx[i]) : 0.f) + (lane + 32 < E ? __expf(v1[i] - mx[i]) : 0.f);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
#pragma unroll
    for (int i = 0; i < NT; ++i) denom[i] += __shfl_xor_sync(0xffffffffu, denom[i], off);
  float wj[NT];
#pragma unroll
  for (int i = 0; i < NT; ++i) wj[i] = __fdividef(ej[i], denom[i]);
  if (score_mode == 1 && renorm) {
    float wsum[NT];
#pragma unroll
    for (int i = 0; i < NT; ++i) wsum[i] = wj[i];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
      for (int i = 0; i < NT; ++i) wsum[i] += __shfl_xor_sync(0xffffffffu, wsum[i], off);
#pragma unroll
    for (int i = 0; i < NT; ++i) wj[i] = __fdividef(wj[i], wsum[i]);
  }
#pragma unroll
  for (int i = 0; i < NT; ++i)
    if (lane < k && valid[i]) {
      idx_row[i][lane] = my_i[i];
      w_row[i][lane] = wj[i];
      atomicAdd(&cnt_s[my_i[i]], 1);
    }
}

// The last CTA of a routing launch (all its threads): the batch counts every CTA added into
// count_acc (integer sums: order-independent) move to batch_counts and count_acc is reset for
// the next launch; at G > 1 they are published into every rank's count table and epoch A is
// raised.  (The per-block prefix the permute needs is its own prologue's job.)
MP_DEV void router_batch_tail(int E, int32_t* count_acc, int32_t* batch_counts, const PeerSync& sync) {
  const int tid = threadIdx.x;
  __shared__ int tot_s[64];
  for (int e = tid; e < E; e += blockDim.x) {
    const int c = __ldcg(count_acc + e);
    tot_s[e] = c;
    batch_counts[e] = c;
    count_acc[e] = 0;
  }
  // count exchange (G > 1): this origin's batch counts go into every rank's
  // count table (half = forward parity), then epoch A is raised
  if (peer_on(sync)) {
    __syncthreads();
    const uint32_t fwd = sync.state[1], par = fwd & 1u;
    int32_t* const* half = sync.count_ptrs + 8 * par;
    for (int i = tid; i < sync.G * E; i += blockDim.x) {
      const int pp = i / E, e2 = i - (i / E) * E;
      half[pp][sync.rank * E + e2] = tot_s[e2];
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence_system();  // cumulative over the CTA's count stores (ordered by the barrier)
      const uint32_t ep = sync.state[0] + 1;
      peer_raise(sync, ep);
      sync.state[0] = ep;
      sync.state[1] = fwd + 1;
      sync.state[2] = par;
    }
  }
}

// ---------------------------------------------------------------- the tensor-core router
namespace ri {
constexpr int kM = 128;                  // tokens per tile (MMA M, TMEM lanes)
constexpr int kKB = 128;                 // k per block: one 128-byte swizzled row of 8-bit limbs
constexpr int kThreads = 256;            // producer / epilogue warps 0-7
constexpr int kMmaWarp = 8;              // + one warp that issues the TMA and MMA work
constexpr int kBlock = kThreads + 32;
constexpr int kStages = 2;
constexpr int kABytes = kM * kKB;        // one limb tile, 16 KB
constexpr int kAStage = 3 * kABytes;
constexpr int kMaxSplit = 4;             // CTAs per cluster (K ranges per tile); a 32-token block each

template <int N>
struct Cfg {
  static constexpr int kBStage = 2 * N * kKB;                   // both Wg limbs: one [2N][128] tile
  // s32 accumulators, one per limb shift s = i + j (x limb i, Wg limb j), at columns [s N, s N + N):
  // x limb i's MMA (N' = 2N over both Wg limbs) lands at column i N, so shifts 1 and 2 collect
  // two MMAs each -- the accumulators are zeroed first and every MMA accumulates
  static constexpr int kCols = 4 * N;
  // the x limb tiles live in TMEM (columns 320.., 2 stages x 3 limbs x 32 columns): the MMAs read
  // no A operand from shared memory and the producers need no proxy fence
  static constexpr int kTmemACol = 320;
  static constexpr int kTmemCols = 512;
  static_assert(kCols <= kTmemACol, "accumulators overlap the A stages");
  static constexpr size_t kOffB = size_t(kStages) * kAStage;
  // partial sums pushed by the other K ranges of the cluster: [split - 1][owned rows][N] int64
  static constexpr size_t kOffRecv = kOffB + size_t(kStages) * kBStage;
  static constexpr int kRow = N + 2;  // int64 per staged row (16-byte pad: conflict-free row-per-lane stores)
  static constexpr size_t kRecvBytes = size_t(kM) * kRow * 8 * (kMaxSplit - 1) / kMaxSplit;
  static constexpr size_t kOffMax = kOffRecv + kRecvBytes;             // [kMaxSplit][kM] row maxima
  static constexpr size_t kOffBar = kOffMax + size_t(kMaxSplit) * kM * 4;
  static constexpr size_t kSmem = kOffBar + 256 + 1024;          // + alignment slack
  static_assert(size_t(kM) * kRow * 8 <= kOffB, "the fold staging must fit in the A ring");
};
}  // namespace ri

// Limb bytes j of four quantised values (bit patterns of q + 1.5 * 2^23), element i in byte i.
MP_DEV void limb_words(uint32_t y0, uint32_t y1, uint32_t y2, uint32_t y3, uint32_t& l0, uint32_t& l1,
                       uint32_t& l2) {
  const uint32_t t01 = __byte_perm(y0, y1, 0x5140), t23 = __byte_perm(y2, y3, 0x5140);
  l0 = __byte_perm(t01, t23, 0x5410);
  l1 = __byte_perm(t01, t23, 0x7632);
  const uint32_t u01 = __byte_perm(y0, y1, 0x0062), u23 = __byte_perm(y2, y3, 0x0062);
  l2 = __byte_perm(u01, u23, 0x5410);
}

// logit = f32( f64(rn_f32(S)) * 2^sh ): rn_f32(S) = m * 2^drop (m <= 2^24) with integer ops, then
// one fp32 multiply by an exact power of two -- the same single rounding as the fp64 product.
// Exponents outside fp32's normal range (rows of tiny / huge magnitude) take the fp64 path.
MP_DEV float exact_logit(long long s, int sh) {
  const unsigned long long a = s < 0 ? 0ull - (unsigned long long)s : (unsigned long long)s;
  if (a == 0) return 0.f;
  const int nb = 64 - __clzll((long long)a);
  const int drop = nb > 24 ? nb - 24 : 0;
  uint32_t m = uint32_t(a >> drop);
  if (drop > 0) {
    const unsigned long long rem = a & ((1ull << drop) - 1), half = 1ull << (drop - 1);
    m += (rem > half || (rem == half && (m & 1u))) ? 1u : 0u;
  }
  const float f = s < 0 ? -float(m) : float(m);  // exact: m <= 2^24
  const int k = drop + sh;
  if (k >= -126 && k <= 127) return f * __uint_as_float(uint32_t(127 + k) << 23);
  return __double2float_rn(double(f) * __hiloint2double((1023 + k) << 20, 0));
}

template <int N>
__global__ void __launch_bounds__(ri::kBlock, 1)
    router_i8_kernel(const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmX,
                     const __nv_bfloat16* __restrict__ x,
                     const uint8_t* __restrict__ packed, const float* __restrict__ bias, int T, int d, int E,
                     int has_gate, int k, int score_mode, int renorm, int split, int32_t* __restrict__ idx,
                     float* __restrict__ wout, float* __restrict__ shared_gate, uint32_t* __restrict__ hist,
                     int32_t* __restrict__ blk_counts, int32_t* __restrict__ batch_counts,
                     uint32_t* __restrict__ ticket, int32_t* __restrict__ count_acc, const PeerSync sync) {
  using C = ri::Cfg<N>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smA = sm;
  uint8_t* smB = sm + C::kOffB;
  uint32_t* xmax = reinterpret_cast<uint32_t*>(sm + C::kOffMax);  // [split][kM]
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + C::kOffBar);  // [2] Wg limbs landed
  uint64_t* empty = full + 2;                                     // [2] MMAs of the stage done
  uint64_t* done = full + 4;                                      // every MMA done
  uint64_t* recv_bar = full + 5;                                  // the cluster's partials landed
  uint64_t* full_a = full + 6;                                    // [2] x limbs written (8 warps)
  uint64_t* xfull = full + 8;                                     // [3] x tiles landed (TMEM-A path)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(full + 12);
  long long* recv = reinterpret_cast<long long*>(sm + C::kOffRecv);
  __shared__ int ex_s[ri::kM];  // E(x_t) of the tile's rows
  __shared__ long long rw_s[N];  // Wg row sums and exponents
  __shared__ int ew_s[N];
  __shared__ float bias_s[N];
  __shared__ int cnt_s[rt::kMaxE];
  __shared__ int last_s;

  const int tid = threadIdx.x, warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const int row0 = blockIdx.y * ri::kM;
  const int n_kb = d / ri::kKB;
  const int kb0 = int(rank) * n_kb / split, kb1 = (int(rank) + 1) * n_kb / split, nk = kb1 - kb0;

  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    mbar_init(recv_bar, 1);
    for (int s = 0; s < 2; ++s) mbar_init(&full_a[s], ri::kThreads / 32);
    for (int s = 0; s < 3; ++s) mbar_init(&xfull[s], 1);
    fence_barrier_init();
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmX);
  }
  if (warp == 0) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  cluster_arrive_relaxed();  // this CTA has started (waited on before the first DSMEM store)
  const uint32_t tmem = *tmem_slot;
  // rows of the tile this CTA selects: router blocks b (32 tokens) with b % split == rank
  const int own_blocks = (4 - int(rank) + split - 1) / split;
  if (tid == 0 && split > 1)  // bytes the other K ranges push here (set before the cluster barrier)
    mbar_arrive_expect_tx(recv_bar, uint32_t((split - 1) * own_blocks * rt::kTokens * C::kRow * 8));

  griddep_launch_dependents();
  griddep_wait();  // x may come from the previous kernel in the stream
  if (tid < ri::kM && row0 + tid < T)  // this CTA's x range, row by row, toward L2 (both passes read it)
    bulk_prefetch_l2(x + size_t(row0 + tid) * d + size_t(kb0) * ri::kKB, uint32_t(nk * ri::kKB * 2));
  for (int e = tid; e < N; e += blockDim.x) {
    rw_s[e] = reinterpret_cast<const long long*>(packed + 2 * size_t(N) * d)[e];
    ew_s[e] = reinterpret_cast<const int*>(packed + 2 * size_t(N) * d + 8 * size_t(N))[e];
    bias_s[e] = (bias != nullptr && e < E) ? bias[e] : 0.f;
  }

  auto issue_b = [&](int i) {  // both Wg limbs of local k-block i into stage i & 1
    const int s = i & 1;
    mbar_arrive_expect_tx(&full[s], uint32_t(C::kBStage));
    tma_load_2d(smB + size_t(s) * C::kBStage, &tmB, &full[s], (kb0 + i) * ri::kKB, 0);
  };
  // the k-block's x tile (128 rows x 128 k bf16, two 64-k SWIZZLE_128B boxes) by TMA into a
  // 3-stage ring at the head of shared memory; rows past T arrive as zeros
  auto issue_x = [&](int i) {
    const int xs = i % 3;
    mbar_arrive_expect_tx(&xfull[xs], uint32_t(ri::kM * ri::kKB * 2));
#pragma unroll
    for (int h = 0; h < 2; ++h)
      tma_load_2d(smA + size_t(xs) * (ri::kM * ri::kKB * 2) + size_t(h) * (ri::kM * 128), &tmX, &xfull[xs],
                  (kb0 + i) * ri::kKB + 64 * h, row0);
  };
  if (warp == ri::kMmaWarp && lane == 0) {
    for (int i = 0; i < min(2, nk); ++i) issue_b(i);
    for (int i = 0; i < min(3, nk); ++i) issue_x(i);
  }

  // ---- 1. per-row maxima of |x| over this CTA's K range, shared with the cluster.  A warp
  // takes 8 rows at a time with every lane's loads of all 8 in flight before any is used.
  cluster_wait();  // every CTA of the cluster has started: its shared memory takes remote stores
  {
    const int kc = nk * ri::kKB / 8;  // 16-byte chunks of one row's range (a multiple of 16)
    const int per = kc / 16;          // chunks per half-warp and row: lanes 0-15 / 16-31 split a row
    for (int r0 = warp * 16; r0 < warp * 16 + 16 && warp < ri::kMmaWarp; r0 += 8) {
      uint32_t m2[4] = {0, 0, 0, 0};   // rows r0 + 2i + (lane >> 4)
      for (int c0 = 0; c0 < per; c0 += 4) {
        uint4 v[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int t = min(row0 + r0 + 2 * i + (lane >> 4), T - 1);
          const uint4* src = reinterpret_cast<const uint4*>(x + size_t(t) * d + size_t(kb0) * ri::kKB) + (lane & 15);
#pragma unroll
          for (int c = 0; c < 4; ++c)
            v[i][c] = c0 + c < per ? ld_nc_v4(src + 16 * (c0 + c)) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int c = 0; c < 4; ++c)
            m2[i] = __vmaxu2(m2[i], __vmaxu2(__vmaxu2(v[i][c].x & 0x7fff7fffu, v[i][c].y & 0x7fff7fffu),
                                             __vmaxu2(v[i][c].z & 0x7fff7fffu, v[i][c].w & 0x7fff7fffu)));
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint32_t m = max(m2[i] & 0xffffu, m2[i] >> 16);
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));  // within the half-warp
        const int r = r0 + 2 * i + (lane >> 4);
        if ((lane & 15) < split) st_cluster_u32(&xmax[rank * ri::kM + r], uint32_t(lane & 15), m);
      }
    }
  }
  cluster_sync();
  if (tid < ri::kM) {
    uint32_t m = 0;
    for (int q = 0; q < split; ++q) m = max(m, xmax[q * ri::kM + tid]);
    ex_s[tid] = row_exponent(m);
  }
  __syncthreads();

  // ---- 2. limbs -> swizzled A tiles, Wg limbs by TMA, 9 MMAs per 32-k step
  if (warp < ri::kMmaWarp) {
    // TMEM-A producers: warp w owns TMEM lanes 32 (w & 3) .. +31 (= tile rows) and k-half w >> 2
    // of every 128-k block: a lane reads its row's 128 bytes from the swizzled x tile (8 x 16 B,
    // conflict-free), converts 64 elements -> 16 words per limb -> three tcgen05.st.  No proxy
    // fence: the tiles come by TMA several blocks ahead.
    const int q = warp & 3, hk = warp >> 2, r = q * 32 + lane;
    const float sc = row_scale(ex_s[r], rt::kWinX);
    {  // zero this warp's half of the accumulator columns (ordered before the first MMA by the
       // tcgen05.wait::st + full_a arrival of block 0)
      uint32_t z[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) z[j] = 0u;
#pragma unroll
      for (int c = 0; c < 2 * N; c += 16)
        tmem_st_32x32b_x16(tmem + (uint32_t(q * 32) << 16) + uint32_t(hk * 2 * N + c), z);
    }
#pragma unroll 1
    for (int i = 0; i < nk; ++i) {
      const int s = i & 1, xs = i % 3;
      if (i >= 2) {
        if (lane == 0) mbar_wait(&empty[s], ((i >> 1) - 1) & 1);
        __syncwarp();
        tc_fence_after();
      }
      if (lane == 0) mbar_wait(&xfull[xs], (i / 3) & 1);
      __syncwarp();
      const uint8_t* xt = smA + size_t(xs) * (ri::kM * ri::kKB * 2) + size_t(hk) * (ri::kM * 128) + r * 128;
      uint4 v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = *reinterpret_cast<const uint4*>(xt + ((j ^ (r & 7)) << 4));
      uint32_t l0[16], l1[16], l2[16];
#pragma unroll
      for (int j = 0; j < 8; ++j) {  // 8 elements per uint4 -> two 4-element words per limb
        const uint32_t w[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
        uint32_t y[8];
#pragma unroll
        for (int e2 = 0; e2 < 4; ++e2) {
          y[2 * e2] = quant_bits(bf16_lo(w[e2]), sc);
          y[2 * e2 + 1] = quant_bits(bf16_hi(w[e2]), sc);
        }
        limb_words(y[0], y[1], y[2], y[3], l0[2 * j], l1[2 * j], l2[2 * j]);
        limb_words(y[4], y[5], y[6], y[7], l0[2 * j + 1], l1[2 * j + 1], l2[2 * j + 1]);
      }
      const uint32_t ta = tmem + (uint32_t(q * 32) << 16) + uint32_t(C::kTmemACol + s * 96 + hk * 16);
      tmem_st_32x32b_x16(ta, l0);
      tmem_st_32x32b_x16(ta + 32, l1);
      tmem_st_32x32b_x16(ta + 64, l2);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_a[s]);  // also: this warp is done with x stage xs
    }
  } else if (lane == 0) {
    // MMA warp: one MMA per (32-k step, x limb), N' = 2N columns = (x limb ia) x (Wg limbs 0, 1)
    for (int i = 0; i < nk; ++i) {
      const int s = i & 1;
      if (i >= 2) {  // Wg stage s is free once the MMAs of block i - 2 completed
        mbar_wait(&empty[s], ((i >> 1) - 1) & 1);
        issue_b(i);
      }
      mbar_wait(&full_a[s], (i >> 1) & 1);
      if (i + 3 < nk) issue_x(i + 3);  // every producer is past x stage i % 3
      mbar_wait(&full[s], (i >> 1) & 1);
      tc_fence_after();
      const uint64_t bd = make_sdesc_sw128(smem_u32(smB + size_t(s) * C::kBStage));
#pragma unroll
      for (int ks = 0; ks < ri::kKB / 32; ++ks)
#pragma unroll
        for (int ia = 0; ia < 3; ++ia) {  // A tile: 8 TMEM columns (32 k) per step of limb ia's 32
          const uint32_t at = tmem + uint32_t(C::kTmemACol + s * 96 + ia * 32 + ks * 8);
          umma_i8_ts(tmem + uint32_t(ia * N), at, bd + uint64_t(2 * ks), make_idesc_i8(ri::kM, 2 * N, true), 1u);
        }
      umma_commit(&empty[s]);
      if (i == nk - 1) umma_commit(done);
    }
  }

  if (tid == 0) mbar_wait(done, 0);
  __syncthreads();
  tc_fence_after();
  // ---- 3. fold the four accumulators into int64 per (row, expert).  Rows of a router block
  // another CTA selects are staged (over the A ring: every MMA is done) and sent there as one
  // bulk copy per block (completing on its recv_bar); rows selected here wait for those copies.
  long long* stage = reinterpret_cast<long long*>(smA);  // [kM][kRow] int64
  const int E_tot = E + (has_gate ? 1 : 0);
  const int own_rows = own_blocks * rt::kTokens;
  if (warp < ri::kMmaWarp) {
    constexpr int H = N / 2;                             // columns per warp quartet
    const int r = (warp & 3) * 32 + lane, h0 = (warp >> 2) * H;
    const uint32_t lane_base = uint32_t((warp & 3) * 32) << 16;
    long long acc[H];
#pragma unroll
    for (int j = 0; j < H; ++j) acc[j] = 0;
#pragma unroll 1
    for (int sh = 0; sh < 4; ++sh) {  // accumulator of limb shift sh, weight 2^(8 sh)
      const long long wgt = 1ll << (8 * sh);
#pragma unroll
      for (int j0 = 0; j0 < H; j0 += 8) {
        uint32_t rv[8];
        tmem_ld_32x32b_x8(tmem + lane_base + uint32_t(sh * N + h0 + j0), rv);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j0 + j] += (long long)int32_t(rv[j]) * wgt;
      }
    }
#pragma unroll
    for (int j = 0; j < H; j += 2)
      *reinterpret_cast<longlong2*>(stage + size_t(r) * C::kRow + h0 + j) = make_longlong2(acc[j], acc[j + 1]);
  }
  fence_proxy_async_shared();
  __syncthreads();
  if (tid == 0) {
    for (int bb = 0; bb < 4; ++bb) {
      const int ow = bb % split;
      if (ow == int(rank)) continue;
      const int slot = int(rank) < ow ? int(rank) : int(rank) - 1;
      const int ow_rows = (4 - ow + split - 1) / split * rt::kTokens;
      const int r_loc = (bb / split) * rt::kTokens;
      bulk_s2s_cluster(recv + (size_t(slot) * ow_rows + r_loc) * C::kRow, stage + size_t(bb) * rt::kTokens * C::kRow,
                       uint32_t(rt::kTokens * C::kRow * 8), recv_bar, uint32_t(ow));
    }
    bulk_commit();
    if (split > 1) mbar_wait(recv_bar, 0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem);
  }
  // logits of this CTA's rows, (row, expert) items over every thread: own partial + the other
  // K ranges' partials - the x-limb bias term, rounded once; into lg [own rows][N] (B ring)
  float* lg = reinterpret_cast<float*>(smB);
  {
    // warp w takes rows w, w + 9, ...; lane l experts l, l + 32 (, l + 64).  Compact code on
    // purpose: each CTA runs this once, so instruction fetch, not issue, sets its time.
    constexpr int EP = (N + 31) / 32;
    constexpr int kWarps = ri::kBlock / 32;
#pragma unroll 1
    for (int rl = warp; rl < own_rows; rl += kWarps) {
      const int r = (int(rank) + (rl / rt::kTokens) * split) * rt::kTokens + rl % rt::kTokens;  // tile row
      const int shr = ex_s[r] - rt::kWinX - rt::kWinW;
#pragma unroll 1
      for (int u = 0; u < EP; ++u) {
        const int e = lane + 32 * u;
        if (e >= E_tot) break;
        long long sum = stage[size_t(r) * C::kRow + e] - rw_s[e] * (1ll << 22);  // q = A' - 2^22
#pragma unroll 1
        for (int p = 0; p < split - 1; ++p) sum += recv[(size_t(p) * own_rows + rl) * C::kRow + e];
        float v = exact_logit(sum, shr + ew_s[e]);
        if (e < E && bias != nullptr) v = __fadd_rn(v, bias_s[e]);
        lg[rl * N + e] = v;
      }
    }
  }
  __syncthreads();

  // ---- 4. selection of this CTA's router blocks: 4 tokens per warp in lockstep, block histogram
  int handled = 0;
  for (int bl = 0; bl < own_blocks; ++bl) {
    const int b = int(rank) + bl * split;
    const int t0 = row0 + b * rt::kTokens;
    if (t0 >= T) break;
    const int nt = min(rt::kTokens, T - t0);
    for (int e = tid; e < E; e += blockDim.x) cnt_s[e] = 0;
    __syncthreads();
    {
      constexpr int NT = 2;  // tokens per warp in lockstep; pairs q, q + 1 over the block's warps
      const float* lgb = lg + size_t(bl) * rt::kTokens * N;
#pragma unroll 1
      for (int q0 = NT * warp; q0 < nt; q0 += NT * (ri::kBlock / 32)) {
        float a[NT], c[NT];
        bool ok[NT];
        int32_t* ir[NT];
        float* wr[NT];
#pragma unroll
        for (int i = 0; i < NT; ++i) {
          const int q = q0 + i, qq = min(q, nt - 1);
          ok[i] = q < nt;
          a[i] = lane < E ? lgb[qq * N + lane] : -INFINITY;
          c[i] = lane + 32 < E ? lgb[qq * N + lane + 32] : -INFINITY;
          ir[i] = idx + size_t(t0 + qq) * k;
          wr[i] = wout + size_t(t0 + qq) * k;
        }
        int32_t* const (&irc)[NT] = ir;
        float* const (&wrc)[NT] = wr;
        select_topk_store<NT>(a, c, ok, E, k, score_mode, renorm, irc, wrc, cnt_s);
        if (lane < NT && has_gate && shared_gate != nullptr) {
          const int q = q0 + lane;
          if (q < nt) shared_gate[t0 + q] = 1.0f / (1.0f + __expf(-lgb[q * N + E]));
        }
      }
    }
    __syncthreads();
    const int blk = t0 / rt::kTokens;
    for (int e = tid; e < E; e += blockDim.x) {
      const int cc = cnt_s[e];
      if (blk_counts) blk_counts[size_t(blk) * E + e] = cc;
      if (cc && hist) atomicAdd(&hist[e], uint32_t(cc));
      if (cc && count_acc) atomicAdd(&count_acc[e], cc);
    }
    ++handled;
    __syncthreads();
  }
  if (tid == 0) bulk_wait_read0();  // the staging rows were read out before the CTA may exit
  if (batch_counts == nullptr || count_acc == nullptr || handled == 0) return;
  // the CTA completing the grid's router blocks reduces the per-block counts
  const int n_blk = (T + rt::kTokens - 1) / rt::kTokens;
  __syncthreads();
  if (tid == 0) {
    __threadfence();  // cumulative over the CTA's count stores (ordered by the barrier)
    last_s = atomicAdd(ticket, uint32_t(handled)) + uint32_t(handled) == uint32_t(n_blk);
    if (last_s) __threadfence();
  }
  __syncthreads();
  if (!last_s) return;
  router_batch_tail(E, count_acc, batch_counts, sync);
  if (tid == 0) *ticket = 0u;  // ready for the next launch (stream-ordered)
}

// Logits-in parity variant of K1's selection stage: the same warp top-k, gate
// weights and block-aggregated histogram, from caller-given fp32 logits [T][ld]
// (+ bias).  One warp per token, 8 tokens per CTA.
__global__ void __launch_bounds__(256) router_logits_kernel(const float* __restrict__ logits, int ld,
                                                            const float* __restrict__ bias, int T, int E, int k,
                                                            int score_mode, int renorm, int32_t* __restrict__ idx,
                                                            float* __restrict__ wout, uint32_t* __restrict__ hist) {
  __shared__ int cnt_s[rt::kMaxE];
  const int tid = threadIdx.x, lane = lane_id(), warp = warp_id();
  for (int e = tid; e < E; e += blockDim.x) cnt_s[e] = 0;
  __syncthreads();
  const int t = blockIdx.x * (blockDim.x / 32) + warp;
  if (t < T) {
    const float* row = logits + size_t(t) * ld;
    float v0 = lane < E ? row[lane] : -INFINITY;
    float v1 = lane + 32 < E ? row[lane + 32] : -INFINITY;
    if (bias != nullptr) {
      if (lane < E) v0 = __fadd_rn(v0, bias[lane]);
      if (lane + 32 < E) v1 = __fadd_rn(v1, bias[lane + 32]);
    }
    const float a[1] = {v0}, c[1] = {v1};
    const bool ok[1] = {true};
    int32_t* const ir[1] = {idx + size_t(t) * k};
    float* const wr[1] = {wout + size_t(t) * k};
    select_topk_store<1>(a, c, ok, E, k, score_mode, renorm, ir, wr, cnt_s);
  }
  __syncthreads();
  if (hist != nullptr)
    for (int e = tid; e < E; e += blockDim.x)
      if (cnt_s[e]) atomicAdd(&hist[e], uint32_t(cnt_s[e]));
}

int launch_router_logits(const float* logits, int ld, const float* bias, int T, int E, int k, int score_mode,
                         int renorm, int32_t* idx, float* w, uint32_t* hist, cudaStream_t stream) {
  if (E < 1 || E > rt::kMaxE) return set_error(MP_E_SHAPE, "router: E=%d outside [1, %d]", E, rt::kMaxE);
  if (k < 1 || k > E || k > rt::kMaxK) return set_error(MP_E_SHAPE, "router: top_k=%d invalid for E=%d", k, E);
  if (ld < E) return set_error(MP_E_SHAPE, "router: logits row stride %d < E=%d", ld, E);
  if (score_mode != 0 && score_mode != 1) return set_error(MP_E_ARG, "router: score_mode %d", score_mode);
  if (T <= 0) return MP_OK;
  router_logits_kernel<<<unsigned((T + 7) / 8), 256, 0, stream>>>(logits, ld, bias, T, E, k, score_mode, renorm,
                                                                   idx, w, hist);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MP_OK : set_cuda_error(e, "router_logits_kernel launch");
}

// K ranges per 128-token tile: enough CTAs to cover the SMs, at most 8 (one cluster)
// and at most one per 128-k block.  MP_ROUTER_SPLIT overrides (tests: the logits do
// not depend on it).
int router_split(int T, int d) {
  const int tiles = (T + ri::kM - 1) / ri::kM, n_kb = d / ri::kKB;
  int split = 1;
  if (const char* env = getenv("MP_ROUTER_SPLIT")) {
    split = atoi(env);
  } else {
    while (split < ri::kMaxSplit && tiles * split * 2 <= kNumSMs) split *= 2;
  }
  split = std::max(1, std::min({split, ri::kMaxSplit, n_kb}));
  return split == 3 ? 2 : split;  // a power of two: the tile's 4 router blocks divide evenly
}

template <int N>
static cudaError_t launch_i8(const CUtensorMap& tmB, const CUtensorMap& tmX, int split, int tiles, cudaStream_t stream, bool pdl,
                             const __nv_bfloat16* x, const uint8_t* packed, const float* bias, int T, int d, int E,
                             int has_gate, int k, int score_mode, int renorm, int32_t* idx, float* w,
                             float* shared_gate, uint32_t* hist, int32_t* blk_counts, int32_t* batch_counts,
                             uint32_t* ticket, int32_t* count_acc, const PeerSync& ps) {
  using C = ri::Cfg<N>;
  const int r = ensure_max_dyn_smem(reinterpret_cast<const void*>(router_i8_kernel<N>), C::kSmem,
                                    "cudaFuncSetAttribute(router_i8)");
  if (r != MP_OK) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(split), unsigned(tiles));
  cfg.blockDim = dim3(ri::kBlock);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = unsigned(split);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, router_i8_kernel<N>, tmB, tmX, x, packed, bias, T, d, E, has_gate, k, score_mode, renorm,
                            split, idx, w, shared_gate, hist, blk_counts, batch_counts, ticket, count_acc, ps);
}

int launch_router(const __nv_bfloat16* x, const uint8_t* packed, const float* bias, int T, int d, int E,
                  int has_gate, int k, int score_mode, int renorm, int32_t* idx, float* w, float* shared_gate,
                  uint32_t* hist, int32_t* blk_counts, int32_t* batch_counts, uint32_t* ticket,
                  int32_t* count_acc, cudaStream_t stream, const PeerSync* sync) {
  if (batch_counts && (!ticket || !count_acc || !blk_counts))
    return set_error(MP_E_ARG, "router: batch counts need the block counts, a ticket word and an accumulator");
  if (E < 1 || E > rt::kMaxE) return set_error(MP_E_SHAPE, "router: E=%d outside [1, %d]", E, rt::kMaxE);
  if (k < 1 || k > E || k > rt::kMaxK) return set_error(MP_E_SHAPE, "router: top_k=%d invalid for E=%d", k, E);
  if (d % 256 != 0 || d > 16384) return set_error(MP_E_SHAPE, "router: d=%d not a multiple of 256 in [256, 16384]", d);
  if (score_mode != 0 && score_mode != 1) return set_error(MP_E_ARG, "router: score_mode %d", score_mode);
  if (T <= 0) return MP_OK;
  if (sync && sync->G > 1 && (!batch_counts || !blk_counts))
    return set_error(MP_E_ARG, "router: the count exchange needs the batch counts");
  if (reinterpret_cast<uintptr_t>(x) % 16 != 0) return set_error(MP_E_ARG, "router: x not 16-byte aligned");
  const int E_tot = E + (has_gate ? 1 : 0), N = router_n_pad(E_tot);
  CUtensorMap tmB, tmX;
  MP_TRY_R(encode_tmap_u8_2d(&tmB, packed, uint64_t(2) * N, uint64_t(d), uint32_t(2 * N)));
  MP_TRY_R(encode_tmap_bf16_2d(&tmX, x, uint64_t(T), uint64_t(d), uint32_t(ri::kM)));  // TMEM-A path
  const int split = router_split(T, d), tiles = (T + ri::kM - 1) / ri::kM;
  const PeerSync ps = sync ? *sync : PeerSync();
  // programmatic dependent launch: scheduled while the previous kernel drains (the
  // kernel's griddepcontrol.wait orders x before use); MP_ROUTER_PDL=0 disables
  static const bool pdl = [] {
    const char* env = getenv("MP_ROUTER_PDL");
    return env == nullptr || atoi(env) != 0;
  }();
  cudaError_t e;
#define MP_ROUTER_LAUNCH(NN)                                                                                       \
  e = launch_i8<NN>(tmB, tmX, split, tiles, stream, pdl, x, packed, bias, T, d, E, has_gate, k, score_mode, renorm, idx, \
                    w, shared_gate, hist, blk_counts, batch_counts, ticket, count_acc, ps)
  switch (N) {
    case 16: MP_ROUTER_LAUNCH(16); break;
    case 32: MP_ROUTER_LAUNCH(32); break;
    case 48: MP_ROUTER_LAUNCH(48); break;
    case 64: MP_ROUTER_LAUNCH(64); break;
    case 80: MP_ROUTER_LAUNCH(80); break;
    default: return set_error(MP_E_SHAPE, "router: %d weight rows", E_tot);
  }
#undef MP_ROUTER_LAUNCH
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? MP_OK : set_cuda_error(e, "router_i8_kernel launch");
}

}  // namespace mp
