// K1: top-k softmax router with a fused, block-aggregated expert histogram.
//
// The reference has no router: expert sets are sampled per request
// (reference pkg/src/moeplace/sim.py:153-191) and folded into token-weighted
// activation counts by ActivationStats.ingest (reference
// pkg/src/moeplace/stats.py:82-96).  This kernel produces both from real
// activations in one pass over x:
//   logits[t,e] = sum_k x[t,k] * Wg[e,k]  (+ bias[e])
//   idx[t,:]    = top-k experts by logit, descending, ties -> lower expert id
//   w[t,:]      = softmax weights (mode 0: softmax over the k selected logits,
//                 Mixtral; mode 1: softmax over all E, no renorm unless asked,
//                 Qwen1.5-MoE / DeepSeek-V2-Lite)
//   hist[e]    += #tokens whose top-k contains e   (token_count = 1 per token)
//
// Bit-exactness contract (restated by oracle/moe_oracle.py:router_logits):
//   * L = 32 n_lg logical lanes, n_lg = router_lane_groups(d) in {1, 2, 4}; lane
//     (g, l) owns the k-slices [8 L s + 8 (32 g + l), +8), s = 0..d/(8L)-1 -- i.e.
//     the 256-k steps g, g + n_lg, g + 2 n_lg, ... at offset 8 l; its partial is ONE
//     sequential fp32 FMA chain over those k ascending, from 0; x and Wg are bf16, so
//     each product is exact and fma == rn(acc + x*w);
//   * inside a group the 32 partials are combined by the butterfly tree
//     p[l] <- p[l] + p[l + o] for o = 16, 8, 4, 2, 1 (fp add is commutative, so a
//     warp reduce-scatter yields exactly this tree); the group sums by
//     q[g] <- q[g] + q[g + o], o = n_lg/2 .. 1; then + bias[e];
//   * selection compares logits only (independent of the exp implementation).
//
// Two kernels.  router_chain_kernel: persistent over every SM, one warp per unit =
// (8-expert pass, lane group, 4-token quad) -- 4 x 8 = 32 accumulators per lane as
// 16 FFMA2 chains while the lanes walk the group's k-steps (x straight from HBM,
// 512 B coalesced per token per step; Wg fp32 in consumption order through L1/L2);
// a reduce-scatter leaves lane l holding (token l/8, expert l%8), stored as a group
// partial.  Lane groups split d so that even one expert pass (Mixtral) yields enough
// units to fill the SMs.  router_select_kernel: one CTA per 32-token block combines
// the partials by the contract's tree and runs top-k, weights and the histogram.
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "mp_internal.h"
#include "peer_sync.cuh"

namespace mp {

namespace rt {
constexpr int kTokens = 32;    // tokens per CTA (also the permute / histogram block)
constexpr int kMaxE = 64;      // routed experts
constexpr int kMaxK = 8;
}  // namespace rt

int router_block_tokens() { return rt::kTokens; }
__host__ __device__ int router_e_pad(int E_tot) { return (E_tot + 7) / 8 * 8; }

#define MP_TRY_R(call)             \
  do {                             \
    const int _r = (call);         \
    if (_r != MP_OK) return _r;    \
  } while (0)

// packed[E_pad][d] bf16 = Wg (zero rows pad E_tot up to a multiple of 8)
__global__ void router_pack_kernel(const __nv_bfloat16* __restrict__ wg, int E_tot, int E_pad, int d,
                                   __nv_bfloat16* __restrict__ packed) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;  // over E_pad * d
  if (i >= size_t(E_pad) * d) return;
  packed[i] = i < size_t(E_tot) * d ? wg[i] : __float2bfloat16(0.0f);
}

int launch_router_pack(const __nv_bfloat16* wg, int E_tot, int d, __nv_bfloat16* packed, cudaStream_t stream) {
  if (d % 256 != 0) return set_error(MP_E_SHAPE, "router d=%d not a multiple of 256", d);
  const int E_pad = router_e_pad(E_tot);
  const size_t n = size_t(E_pad) * d;
  router_pack_kernel<<<unsigned((n + 255) / 256), 256, 0, stream>>>(wg, E_tot, E_pad, d, packed);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MP_OK : set_cuda_error(e, "router_pack_kernel launch");
}

// Wg pre-converted to fp32 in the order the router's lanes consume it: float4
// number t of lane l in (pass, step) sits at ((pass * S + step) * 16 + t) * 32 + l
// (a warp's load of float4 t is 512 contiguous bytes) and holds experts
// 8 pass + 4 (t & 1) .. +3 at k = 256 step + 8 l + (t >> 1) -- two
// (expert 2i, 2i+1) pairs ready for FFMA2, no bf16 conversions in the FMA loop.
// Same products and chains as the bf16 path (bit-identical logits).
__global__ void router_pack32_kernel(const __nv_bfloat16* __restrict__ wg, int E_tot, int E_pad, int d,
                                     float* __restrict__ w32) {
  const size_t o = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (o >= size_t(E_pad) * d) return;
  const int S = d / 256;
  const int i = int(o & 3), l = int((o >> 2) & 31), t = int((o >> 7) & 15);
  const size_t rest = o >> 11;  // pass * S + step
  const int st = int(rest % S), p = int(rest / S);
  const int e = 8 * p + 4 * (t & 1) + i, kk = 256 * st + 8 * l + (t >> 1);
  w32[o] = e < E_tot ? __bfloat162float(wg[size_t(e) * d + kk]) : 0.0f;
}

int launch_router_pack32(const __nv_bfloat16* wg, int E_tot, int d, float* w32, cudaStream_t stream) {
  if (d % 256 != 0) return set_error(MP_E_SHAPE, "router d=%d not a multiple of 256", d);
  const size_t n = size_t(router_e_pad(E_tot)) * d;
  router_pack32_kernel<<<unsigned((n + 255) / 256), 256, 0, stream>>>(wg, E_tot, router_e_pad(E_tot), d, w32);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MP_OK : set_cuda_error(e, "router_pack32_kernel launch");
}

// acc = (acc.lo + x*w.lo, acc.hi + x*w.hi): two independent fp32 FMAs (FFMA2),
// each rounded exactly like fmaf -- the per-lane chain contract is unchanged.
MP_DEV void ffma2(unsigned long long& acc, float x, unsigned long long w) {
  const unsigned long long xx = (unsigned long long)__float_as_uint(x) | ((unsigned long long)__float_as_uint(x) << 32);
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(xx), "l"(w));
}
MP_DEV unsigned long long pack2(float lo, float hi) {
  return (unsigned long long)__float_as_uint(lo) | ((unsigned long long)__float_as_uint(hi) << 32);
}

// Warp-collective top-k + gate weights of one token from its logits (lane l holds
// experts l and l + 32): k rounds of a warp arg-max -- larger logit, ties -> lower id,
// as two redux.sync reductions over order-preserving keys -- then softmax over the k
// (mode 0) or over all E (mode 1, optional renormalisation).  Lane j < k writes
// idx_row[j] / w_row[j] and bumps cnt_s.
// Order-preserving 32-bit key of an fp32 logit (-0 canonicalised to +0, so equal logits get
// equal keys): larger logit <=> larger unsigned key.
MP_DEV uint32_t logit_key(float v) {
  const uint32_t u = __float_as_uint(v + 0.0f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

MP_DEV void select_topk_store(float v0, float v1, int E, int k, int score_mode, int renorm, int32_t* idx_row,
                              float* w_row, int* cnt_s) {
  const int lane = lane_id();
  // candidates of this lane: expert lane (v0) and lane + 32 (v1); taken/absent -> key 0
  uint32_t k0 = lane < E ? logit_key(v0) : 0u, k1 = lane + 32 < E ? logit_key(v1) : 0u;
  float my_v = -INFINITY, mx = 0.f;  // lane j < k keeps the j-th selected logit and expert
  int my_i = 0;
#pragma unroll 1
  for (int j = 0; j < k; ++j) {
    // round j: the largest key over the warp (redux), then the lowest expert id holding it
    const bool use1 = k1 > k0;  // ties inside the lane: the lower id (lane) wins
    const uint32_t bk = use1 ? k1 : k0;
    const uint32_t mk = __reduce_max_sync(0xffffffffu, bk);
    const uint32_t cand = (bk == mk && mk != 0u) ? uint32_t(use1 ? lane + 32 : lane) : 0xffffffffu;
    const uint32_t bi = __reduce_min_sync(0xffffffffu, cand);
    const float bv = __shfl_sync(0xffffffffu, bi >= 32 ? v1 : v0, bi & 31);
    if (j == 0) mx = bv;
    if (lane == j) { my_v = bv; my_i = int(bi); }
    if (bi == uint32_t(lane)) k0 = 0u;
    if (bi == uint32_t(lane + 32)) k1 = 0u;
  }
  // weights: lane j < k owns w_j
  const float ej = lane < k ? expf(my_v - mx) : 0.f;
  float denom;
  if (score_mode == 0) {
    denom = ej;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) denom += __shfl_xor_sync(0xffffffffu, denom, off);
  } else {
    float sum = (lane < E ? expf(v0 - mx) : 0.f) + (lane + 32 < E ? expf(v1 - mx) : 0.f);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
    denom = sum;
  }
  float wj = ej / denom;
  if (score_mode == 1 && renorm) {
    float wsum = wj;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, off);
    wj = wj / wsum;
  }
  if (lane < k) {
    idx_row[lane] = my_i;
    w_row[lane] = wj;
    atomicAdd(&cnt_s[my_i], 1);
  }
}

constexpr int kTokPerWarp = 4;  // a chain unit: 4 tokens (one quad) x 8 experts (one pass)
constexpr int kExpPerPass = 8;
constexpr int kChainWarps = 16;  // warps per CTA of the chain kernel

// Lane groups of the numerics contract (oracle.router_lane_groups): with n_lg groups
// of 32 logical lanes, the chain of lane (g, l) walks the 256-k steps g, g + n_lg, ...
// so every unit of work is one 32-lane warp over d / n_lg of the k range.
__host__ __device__ int router_lane_groups(int d) {
  if (d >= 4096 && d % 1024 == 0) return 4;
  if (d >= 2048 && d % 512 == 0) return 2;
  return 1;
}

// Stage 1 (chains).  Unit = (expert pass p, lane group g, token quad q): one warp keeps
// 4 tokens x 8 experts = 16 FFMA2 accumulator pairs per lane while its lanes walk the
// group's k-steps (x: 512 B coalesced per token per step, straight from HBM; Wg: the
// fp32 consumption-order operand or the bf16 rows, through L1/L2).  A reduce-scatter
// butterfly leaves lane l holding the group partial of (token l/8, expert l%8), stored
// to partial[g][t][E_pad].  Persistent: warps stride over the units, quads fastest.
template <bool kW32>
__global__ void __launch_bounds__(kChainWarps * 32, 1)
    router_chain_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wp,
                        const float4* __restrict__ w32, int T, int d, int E_pad, int n_lg,
                        float* __restrict__ partial) {
  griddep_launch_dependents();
  griddep_wait();
  const int lane = lane_id();
  const int n_quads = (T + kTokPerWarp - 1) / kTokPerWarp;
  const int n_pass = E_pad / kExpPerPass;
  const int S_all = d / 256;          // 256-k steps in d
  const int S = S_all / n_lg;         // steps of one lane group's chain
  const int n_units = n_quads * n_pass * n_lg;
  const int gw = blockIdx.x * (blockDim.x >> 5) + warp_id();
  const int n_warps = gridDim.x * (blockDim.x >> 5);
  for (int u = gw; u < n_units; u += n_warps) {
    const int q = u % n_quads, pg = u / n_quads;
    const int g = pg % n_lg, pass = pg / n_lg;
    const int t0 = q * kTokPerWarp;
    const __nv_bfloat16* xr[kTokPerWarp];
#pragma unroll
    for (int i = 0; i < kTokPerWarp; ++i)
      xr[i] = x + size_t(t0 + i < T ? t0 + i : 0) * d + 256 * g + 8 * lane;  // rows past T: discarded
    unsigned long long acc[kTokPerWarp][kExpPerPass / 2];
#pragma unroll
    for (int i = 0; i < kTokPerWarp; ++i)
#pragma unroll
      for (int j = 0; j < kExpPerPass / 2; ++j) acc[i][j] = 0ull;
    if (kW32) {
      // fp32 pairs straight from the pre-converted Wg (two halves of 4 k each); the
      // step of this group's chain number s is the 256-k step g + n_lg * s
      const float4* w4 = w32 + (size_t(pass) * S_all + g) * 16 * 32 + lane;
      uint4 xv[kTokPerWarp], xn[kTokPerWarp];
#pragma unroll
      for (int i = 0; i < kTokPerWarp; ++i) xv[i] = ld_nc_v4(xr[i]);
#pragma unroll 1
      for (int s = 0; s < S; ++s, w4 += size_t(n_lg) * 16 * 32) {
        // the next step's x rows are in flight while this step's FFMA2 chains run
        if (s + 1 < S) {
#pragma unroll
          for (int i = 0; i < kTokPerWarp; ++i) xn[i] = ld_nc_v4(xr[i] + size_t(256) * n_lg * (s + 1));
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float4 wv[8];
#pragma unroll
          for (int t2 = 0; t2 < 8; ++t2) wv[t2] = __ldg(w4 + (8 * h + t2) * 32);
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {  // strictly ascending k inside the lane's slice
            const int qk = 4 * h + qq;
            float xs[kTokPerWarp];
#pragma unroll
            for (int i = 0; i < kTokPerWarp; ++i) {
              const uint32_t uu = (&xv[i].x)[qk >> 1];
              xs[i] = (qk & 1) ? bf16_hi(uu) : bf16_lo(uu);
            }
            const float4 a = wv[2 * qq], b = wv[2 * qq + 1];
            const unsigned long long w2[4] = {pack2(a.x, a.y), pack2(a.z, a.w), pack2(b.x, b.y), pack2(b.z, b.w)};
#pragma unroll
            for (int j = 0; j < kExpPerPass / 2; ++j)
#pragma unroll
              for (int i = 0; i < kTokPerWarp; ++i) ffma2(acc[i][j], xs[i], w2[j]);
          }
        }
#pragma unroll
        for (int i = 0; i < kTokPerWarp; ++i) xv[i] = xn[i];
      }
    } else {
      const __nv_bfloat16* wr = wp + size_t(kExpPerPass) * pass * d + 256 * g + 8 * lane;
#pragma unroll 1
      for (int s = 0; s < S; ++s) {
        const size_t ko = size_t(256) * n_lg * s;
        uint4 xv[kTokPerWarp], wv[kExpPerPass];
#pragma unroll
        for (int i = 0; i < kTokPerWarp; ++i) xv[i] = ld_nc_v4(xr[i] + ko);
#pragma unroll
        for (int j = 0; j < kExpPerPass; ++j) wv[j] = __ldg(reinterpret_cast<const uint4*>(wr + size_t(j) * d + ko));
#pragma unroll
        for (int qk = 0; qk < 8; ++qk) {  // strictly ascending k inside the lane's slice
          float xs[kTokPerWarp];
#pragma unroll
          for (int i = 0; i < kTokPerWarp; ++i) {
            const uint32_t uu = (&xv[i].x)[qk >> 1];
            xs[i] = (qk & 1) ? bf16_hi(uu) : bf16_lo(uu);
          }
#pragma unroll
          for (int j = 0; j < kExpPerPass / 2; ++j) {
            const uint32_t u0 = (&wv[2 * j].x)[qk >> 1], u1 = (&wv[2 * j + 1].x)[qk >> 1];
            const unsigned long long w2 =
                (qk & 1) ? pack2(bf16_hi(u0), bf16_hi(u1)) : pack2(bf16_lo(u0), bf16_lo(u1));
#pragma unroll
            for (int i = 0; i < kTokPerWarp; ++i) ffma2(acc[i][j], xs[i], w2);
          }
        }
      }
    }
    // butterfly reduce-scatter over the 32 lane partials of 32 values
    // (value v = token v/8, expert v%8); afterwards lane l holds value l
    float v[32];
#pragma unroll
    for (int i = 0; i < kTokPerWarp; ++i)
#pragma unroll
      for (int j = 0; j < kExpPerPass / 2; ++j) {
        v[i * 8 + 2 * j] = __uint_as_float(uint32_t(acc[i][j]));
        v[i * 8 + 2 * j + 1] = __uint_as_float(uint32_t(acc[i][j] >> 32));
      }
#pragma unroll
    for (int o = 16, n = 32; o >= 1; o >>= 1, n >>= 1) {
      const bool upper = (lane & o) != 0;
#pragma unroll
      for (int i = 0; i < n / 2; ++i) {
        const float send = upper ? v[i] : v[i + n / 2];
        const float keep = upper ? v[i + n / 2] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
    const int tt = t0 + (lane >> 3);
    if (tt < T) partial[(size_t(g) * T + tt) * E_pad + kExpPerPass * pass + (lane & 7)] = v[0];
  }
}

// Stage 1, octet form (the layer's default).  Unit = (expert pass p, lane group g, token
// octet o): one warp keeps 8 tokens x 8 experts = 32 FFMA2 accumulator pairs per lane, so
// every Wg value a lane loads feeds 8 tokens (half the L1 traffic per FMA of the quad form).
// Wg comes as bf16 rows [E_pad][d] (one uint4 = 8 k of one expert per lane and step); the
// pair (e, e + 1) at one k is two ALU ops.  With one warp's 32 x 8 accumulators the register
// file holds only 8 warps per SM, too few to hide load latency, so every lane streams its own
// operands (8 x rows + 8 Wg rows, 16 B each per step) through a kStages-deep shared-memory
// ring with cp.async, running ahead across unit boundaries -- a lane only ever reads back the
// bytes it copied itself, so no warp or CTA synchronisation is involved.  Same chains, same
// butterfly, same partial layout as the quad form.
constexpr int kOctTok = 8;
constexpr int kOctWarps = 8;
constexpr int kOctStages = 3;
constexpr int kOctChunks = kOctTok + kExpPerPass;  // 16-B chunks per lane and step
constexpr size_t kOctSmem = size_t(kOctWarps) * kOctStages * kOctChunks * 32 * 16;  // 192 KB

__global__ void __launch_bounds__(kOctWarps * 32, 1)
    router_chain8_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wp, int T, int d,
                         int E_pad, int n_lg, float* __restrict__ partial) {
  extern __shared__ __align__(16) uint8_t ring_raw[];
  griddep_launch_dependents();
  griddep_wait();
  const int lane = lane_id(), warp = warp_id();
  // this lane's ring: [stage][chunk] 16-B slots, lane-interleaved (conflict-free LDS.128)
  uint4* ring = reinterpret_cast<uint4*>(ring_raw) + size_t(warp) * kOctStages * kOctChunks * 32 + lane;
  const int n_oct = (T + kOctTok - 1) / kOctTok;
  const int n_pass = E_pad / kExpPerPass;
  const int S = d / 256 / n_lg;
  const int n_units = n_oct * n_pass * n_lg;
  const int gw = blockIdx.x * kOctWarps + warp;
  const int n_warps = gridDim.x * kOctWarps;
  // (unit, step) pairs of this warp in order: unit u_i = gw + i * n_warps, steps 0..S-1
  const int my_units = gw < n_units ? (n_units - 1 - gw) / n_warps + 1 : 0;
  const int total = my_units * S;
  // producer cursor: the (unit, step) whose copies are issued next, with its row / Wg bases
  // recomputed only when it crosses into the next unit
  int f_s = 0, f_u = gw;
  const __nv_bfloat16* fx = nullptr;   // x row of the octet's first token at this step and lane
  const __nv_bfloat16* fw = nullptr;   // Wg row of the pass's first expert at this step and lane
  uint32_t frow[kOctTok];              // element offsets of the octet's rows from the first one
  auto unit_bases = [&]() {
    const int o = f_u % n_oct, pg = f_u / n_oct;
    const int g = pg % n_lg, pass = pg / n_lg;
    const int t0 = o * kOctTok;
    fx = x + size_t(t0) * d + 256 * g + 8 * lane;
    fw = wp + size_t(kExpPerPass) * pass * d + 256 * g + 8 * lane;
#pragma unroll
    for (int i = 0; i < kOctTok; ++i) frow[i] = uint32_t(t0 + i < T ? i : -t0) * uint32_t(d);  // past T: row 0
  };
  if (total > 0) unit_bases();
  const size_t step_elems = size_t(256) * n_lg;
  int f_slot = 0;
  auto fetch = [&]() {  // issue the copies of the producer's (unit, step) into its ring stage
    uint4* slot = ring + size_t(f_slot) * kOctChunks * 32;
    const __nv_bfloat16* xs = fx + step_elems * f_s;
    const __nv_bfloat16* ws = fw + step_elems * f_s;
#pragma unroll
    for (int i = 0; i < kOctTok; ++i) cp_async_16(slot + i * 32, xs + int32_t(frow[i]));
#pragma unroll
    for (int j = 0; j < kExpPerPass; ++j) cp_async_16(slot + (kOctTok + j) * 32, ws + size_t(j) * d);
    if (++f_slot == kOctStages) f_slot = 0;
    if (++f_s == S) {
      f_s = 0;
      f_u += n_warps;
      if (f_u < n_units) unit_bases();
    }
  };
#pragma unroll
  for (int f = 0; f < kOctStages - 1; ++f) {
    if (f < total) fetch();
    cp_async_commit();
  }
  unsigned long long acc[kOctTok][kExpPerPass / 2];
  int c_s = 0, c_u = gw, c_slot = 0;  // consumer cursor
#pragma unroll 1
  for (int c = 0; c < total; ++c) {
    if (c + kOctStages - 1 < total) fetch();
    cp_async_commit();
    cp_async_wait<kOctStages - 1>();  // this lane's copies of step c have landed
    const int s = c_s;
    if (s == 0) {
#pragma unroll
      for (int i = 0; i < kOctTok; ++i)
#pragma unroll
        for (int j = 0; j < kExpPerPass / 2; ++j) acc[i][j] = 0ull;
    }
    const uint4* slot = ring + size_t(c_slot) * kOctChunks * 32;
    if (++c_slot == kOctStages) c_slot = 0;
    uint4 wv[kExpPerPass];
#pragma unroll
    for (int j = 0; j < kExpPerPass; ++j) wv[j] = slot[(kOctTok + j) * 32];
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // two halves of the octet's x rows
      uint4 xv[kOctTok / 2];
#pragma unroll
      for (int i = 0; i < kOctTok / 2; ++i) xv[i] = slot[(4 * h + i) * 32];
#pragma unroll
      for (int qk = 0; qk < 8; ++qk) {  // strictly ascending k inside the lane's slice
        unsigned long long w2[kExpPerPass / 2];
#pragma unroll
        for (int j = 0; j < kExpPerPass / 2; ++j) {
          const uint32_t u0 = (&wv[2 * j].x)[qk >> 1], u1 = (&wv[2 * j + 1].x)[qk >> 1];
          w2[j] = (qk & 1) ? pack2(bf16_hi(u0), bf16_hi(u1)) : pack2(bf16_lo(u0), bf16_lo(u1));
        }
#pragma unroll
        for (int i = 0; i < kOctTok / 2; ++i) {
          const uint32_t uu = (&xv[i].x)[qk >> 1];
          const float xs = (qk & 1) ? bf16_hi(uu) : bf16_lo(uu);
#pragma unroll
          for (int j = 0; j < kExpPerPass / 2; ++j) ffma2(acc[4 * h + i][j], xs, w2[j]);
        }
      }
    }
    if (++c_s == S) {
      c_s = 0;
      const int u = c_u;
      c_u += n_warps;
      const int o = u % n_oct, pg = u / n_oct;
      const int g = pg % n_lg, pass = pg / n_lg;
      // two butterfly reduce-scatters (tokens 0-3 and 4-7), as in the quad form
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float v[32];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < kExpPerPass / 2; ++j) {
            v[i * 8 + 2 * j] = __uint_as_float(uint32_t(acc[4 * h + i][j]));
            v[i * 8 + 2 * j + 1] = __uint_as_float(uint32_t(acc[4 * h + i][j] >> 32));
          }
#pragma unroll
        for (int off = 16, n = 32; off >= 1; off >>= 1, n >>= 1) {
          const bool upper = (lane & off) != 0;
#pragma unroll
          for (int i = 0; i < n / 2; ++i) {
            const float send = upper ? v[i] : v[i + n / 2];
            const float keep = upper ? v[i + n / 2] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
          }
        }
        const int tt = o * kOctTok + 4 * h + (lane >> 3);
        if (tt < T) partial[(size_t(g) * T + tt) * E_pad + kExpPerPass * pass + (lane & 7)] = v[0];
      }
    }
  }
  cp_async_wait<0>();
}

// Stage 2 (selection).  CTA = one router block of 32 tokens (the histogram / permute
// block), 32 warps, one warp per token: lane l reads the partials of experts l
// and l + 32 straight from L2 (all of a warp's loads issued before any is used),
// combines them by the contract's tree (q[g] += q[g + o], o = n_lg/2..1) + bias, then
// top-k, gate weights and the block-aggregated histogram; the last CTA produces the
// batch counts, the block prefix and (G > 1) the count exchange with epoch A.
MP_DEV float combine_groups(const float* pp, size_t gs, int n_lg) {
  // pp: the partial of (token, expert) in group 0; gs: stride between groups
  float v = __ldcg(pp);
  if (n_lg == 2) {
    v = v + __ldcg(pp + gs);
  } else if (n_lg == 4) {  // q[g] += q[g + 2], then q[0] += q[1]
    const float a1 = __ldcg(pp + gs), a2 = __ldcg(pp + 2 * gs), a3 = __ldcg(pp + 3 * gs);
    v = (v + a2) + (a1 + a3);
  }
  return v;
}

constexpr int kSelectThreads = rt::kTokens * 32;
__global__ void __launch_bounds__(kSelectThreads)
    router_select_kernel(const float* __restrict__ partial, int n_lg, int E_pad, const float* __restrict__ bias,
                         int T, int E, int has_gate, int k, int score_mode, int renorm, int32_t* __restrict__ idx,
                         float* __restrict__ wout, float* __restrict__ shared_gate, uint32_t* __restrict__ hist,
                         int32_t* __restrict__ blk_counts, int32_t* __restrict__ batch_counts,
                         uint32_t* __restrict__ ticket, int32_t* __restrict__ blk_prefix, const PeerSync sync,
                         int stage_counts) {
  __shared__ int cnt_s[rt::kMaxE];
  extern __shared__ __align__(128) uint8_t dsm[];  // last CTA: the [nb][E] block counts
  int* bc = reinterpret_cast<int*>(dsm);
  const int blk = blockIdx.x, n_blk = gridDim.x;
  const int t0 = blk * rt::kTokens;
  const int tid = threadIdx.x, lane = lane_id(), warp = warp_id();
  for (int e = tid; e < E; e += blockDim.x) cnt_s[e] = 0;
  const float bz0 = (bias != nullptr && lane < E) ? bias[lane] : 0.f;
  const float bz1 = (bias != nullptr && lane + 32 < E) ? bias[lane + 32] : 0.f;
  griddep_launch_dependents();
  griddep_wait();  // the chain kernel's partials
  __syncthreads();

  // ---- logits, top-k + weights: one warp per token
  const size_t gs = size_t(T) * E_pad;
  auto load = [&](int t, float& a0, float& a1, float& ag) {
    const float* pp = partial + size_t(min(t, T - 1)) * E_pad;
    a0 = lane < E ? combine_groups(pp + lane, gs, n_lg) : -INFINITY;
    a1 = lane + 32 < E ? combine_groups(pp + lane + 32, gs, n_lg) : -INFINITY;
    ag = has_gate ? combine_groups(pp + E, gs, n_lg) : 0.f;
  };
  // one warp per token of the block (32 warps): the selection is a chain of dependent shuffles,
  // so its latency is hidden by warps, not by work per warp
  const int t = t0 + warp;
  if (warp < rt::kTokens && t < T) {
    float c0, c1, cg;
    load(t, c0, c1, cg);
    const float a = (lane < E && bias != nullptr) ? __fadd_rn(c0, bz0) : c0;
    const float c = (lane + 32 < E && bias != nullptr) ? __fadd_rn(c1, bz1) : c1;
    select_topk_store(a, c, E, k, score_mode, renorm, idx + size_t(t) * k, wout + size_t(t) * k, cnt_s);
    if (lane == 0 && has_gate && shared_gate != nullptr) shared_gate[t] = 1.0f / (1.0f + expf(-cg));
  }
  __syncthreads();
  for (int e = tid; e < E; e += blockDim.x) {
    const int c = cnt_s[e];
    if (blk_counts) blk_counts[size_t(blk) * E + e] = c;
    if (c && hist) atomicAdd(&hist[e], uint32_t(c));
  }
  if (batch_counts == nullptr || blk_counts == nullptr) return;
  // The last CTA to finish reduces the per-block counts into this batch's
  // per-expert counts (integer sums: order-independent), so they are ready when
  // the kernel completes -- no memset, no second pass.
  __shared__ int is_last;
  // one gpu-scope fence per CTA, from thread 0 after the barrier (cumulative over the CTA's
  // count stores), as in a cooperative grid barrier -- not one per thread
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    is_last = atomicAdd(ticket, 1u) == uint32_t(n_blk - 1);
    if (is_last) __threadfence();
  }
  __syncthreads();
  if (!is_last) return;
  const int nb = n_blk;
  // stage the [nb][E] block-count matrix in shared memory with coalesced loads
  // (when it fits: up to 200 KB), then per-expert scans run from there
  const bool staged = stage_counts != 0;
  if (staged)
    for (int i = tid; i < nb * E; i += blockDim.x) bc[i] = __ldcg(&blk_counts[i]);
  __syncthreads();
  __shared__ int seg_sum[64][17];
  int P = 1;
  while (P * 2 * E <= int(blockDim.x) && P * 2 <= 16) P *= 2;
  const int e = tid / P, p = tid - (tid / P) * P;
  const int seg = (nb + P - 1) / P;
  const int b0 = min(nb, p * seg), b1 = min(nb, b0 + seg);
  auto cnt = [&](int blk) { return staged ? bc[blk * E + e] : __ldcg(&blk_counts[size_t(blk) * E + e]); };
  if (e < E) {
    int sum = 0;
    for (int blk = b0; blk < b1; ++blk) sum += cnt(blk);
    seg_sum[e][p] = sum;
  }
  __syncthreads();
  if (e < E) {
    int run = 0;
    for (int q = 0; q < p; ++q) run += seg_sum[e][q];
    if (p == P - 1) {
      int tot = run;
      for (int blk = b0; blk < b1; ++blk) tot += cnt(blk);
      batch_counts[e] = tot;
    }
    // exclusive prefix over blocks: blk_prefix[b][e] = sum_{b' < b} blk_counts[b'][e]
    if (blk_prefix != nullptr)
      for (int blk = b0; blk < b1; ++blk) {
        blk_prefix[size_t(blk) * E + e] = run;
        run += cnt(blk);
      }
  }
  // count exchange (G > 1): this origin's batch counts go into every rank's
  // count table (half = forward parity), then epoch A is raised
  if (peer_on(sync)) {
    __syncthreads();
    const uint32_t fwd = sync.state[1], par = fwd & 1u;
    int32_t* const* half = sync.count_ptrs + 8 * par;
    for (int i = tid; i < sync.G * E; i += blockDim.x) {
      const int p = i / E, e2 = i - (i / E) * E;
      half[p][sync.rank * E + e2] = batch_counts[e2];
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
    select_topk_store(v0, v1, E, k, score_mode, renorm, idx + size_t(t) * k, wout + size_t(t) * k, cnt_s);
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

// Partial-logit scratch of the stateless entries (the layer passes its own): per device,
// grown on demand, never freed.
static float* stateless_partial(size_t floats) {
  static std::mutex mu;
  static float* buf[16] = {};
  static size_t cap[16] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (cap[dev] < floats) {
    if (buf[dev]) cudaFree(buf[dev]);
    buf[dev] = nullptr;
    cap[dev] = 0;
    if (cudaMalloc(&buf[dev], floats * sizeof(float)) != cudaSuccess) return nullptr;
    cap[dev] = floats;
  }
  return buf[dev];
}

size_t router_partial_floats(int T, int d, int E_tot) {
  return size_t(router_lane_groups(d)) * size_t(T) * size_t(router_e_pad(E_tot));
}

int launch_router(const __nv_bfloat16* x, const __nv_bfloat16* wg_packed, const float* bias, int T, int d, int E,
                  int has_gate, int k, int score_mode, int renorm, int32_t* idx, float* w, float* shared_gate,
                  uint32_t* hist, int32_t* blk_counts, int32_t* batch_counts, uint32_t* ticket,
                  int32_t* blk_prefix, cudaStream_t stream, const PeerSync* sync, const float* w32, float* partial) {
  if (batch_counts && !ticket) return set_error(MP_E_ARG, "router: batch counts need a ticket word");
  if (E < 1 || E > rt::kMaxE) return set_error(MP_E_SHAPE, "router: E=%d outside [1, %d]", E, rt::kMaxE);
  if (k < 1 || k > E || k > rt::kMaxK) return set_error(MP_E_SHAPE, "router: top_k=%d invalid for E=%d", k, E);
  if (d % 256 != 0) return set_error(MP_E_SHAPE, "router: d=%d not a multiple of 256", d);
  if (score_mode != 0 && score_mode != 1) return set_error(MP_E_ARG, "router: score_mode %d", score_mode);
  if (T <= 0) return MP_OK;
  if (sync && sync->G > 1 && (!batch_counts || !blk_counts))
    return set_error(MP_E_ARG, "router: the count exchange needs the batch counts");
  if (reinterpret_cast<uintptr_t>(x) % 16 != 0) return set_error(MP_E_ARG, "router: x not 16-byte aligned");
  const int E_tot = E + (has_gate ? 1 : 0), E_pad = router_e_pad(E_tot), n_lg = router_lane_groups(d);
  if (!partial) partial = stateless_partial(router_partial_floats(T, d, E_tot));
  if (!partial) return set_error(MP_E_CUDA, "router: cannot allocate the partial-logit scratch");
  const char* w32env = getenv("MP_ROUTER_W32");
  const bool use32 = w32 != nullptr && (w32env == nullptr || atoi(w32env) != 0);

  // stage 1: the chains, persistent over every SM (MP_ROUTER_GRID overrides, for tests)
  const int n_units = ((T + kTokPerWarp - 1) / kTokPerWarp) * (E_pad / kExpPerPass) * n_lg;
  int grid1 = std::min(kNumSMs, (n_units + kChainWarps - 1) / kChainWarps);
  if (const char* ge = getenv("MP_ROUTER_GRID")) grid1 = std::max(1, atoi(ge));
  // the octet form over the bf16 rows is the default; an fp32 operand runs the quad form
  // (MP_ROUTER_CHAIN=4 also runs the quad form over the bf16 rows)
  const char* chain_env = getenv("MP_ROUTER_CHAIN");
  const int chain = use32 ? 4 : (chain_env ? atoi(chain_env) : 8);
  cudaError_t e;
  if (chain == 8) {
    const int n_units8 = ((T + kOctTok - 1) / kOctTok) * (E_pad / kExpPerPass) * n_lg;
    int grid8 = std::min(kNumSMs, (n_units8 + kOctWarps - 1) / kOctWarps);
    if (const char* ge = getenv("MP_ROUTER_GRID")) grid8 = std::max(1, atoi(ge));
    MP_TRY_R(ensure_max_dyn_smem(reinterpret_cast<const void*>(router_chain8_kernel), kOctSmem,
                                 "cudaFuncSetAttribute(router_chain8)"));
    e = launch_pdl(router_chain8_kernel, dim3(grid8), dim3(kOctWarps * 32), kOctSmem, stream, x, wg_packed, T, d,
                   E_pad, n_lg, partial);
  } else if (use32) {
    e = launch_pdl(router_chain_kernel<true>, dim3(grid1), dim3(kChainWarps * 32), 0, stream, x, wg_packed,
                   reinterpret_cast<const float4*>(w32), T, d, E_pad, n_lg, partial);
  } else {
    e = launch_pdl(router_chain_kernel<false>, dim3(grid1), dim3(kChainWarps * 32), 0, stream, x, wg_packed,
                   static_cast<const float4*>(nullptr), T, d, E_pad, n_lg, partial);
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "router_chain_kernel launch");

  // stage 2: selection per 32-token block (+ last-CTA scan and count exchange)
  const int grid2 = (T + rt::kTokens - 1) / rt::kTokens;
  size_t bc_bytes = blk_counts && batch_counts ? size_t(grid2) * E * 4 : 0;
  const bool stage_counts = bc_bytes <= 200 * 1024;  // larger T: the last CTA scans from global memory
  if (!stage_counts) bc_bytes = 0;
  MP_TRY_R(ensure_max_dyn_smem(reinterpret_cast<const void*>(router_select_kernel), bc_bytes,
                               "cudaFuncSetAttribute(router_select)"));
  // programmatic dependent launch: the selection grid is scheduled while the chains drain
  // (its griddepcontrol.wait still orders every partial before use); MP_ROUTER_PDL=0 disables
  static const bool sel_pdl = [] {
    const char* env = getenv("MP_ROUTER_PDL");
    return env == nullptr || atoi(env) != 0;
  }();
  e = launch_pdl_if(sel_pdl || pdl_enabled(), router_select_kernel, dim3(grid2), dim3(kSelectThreads), bc_bytes,
                    stream,
                    static_cast<const float*>(partial), n_lg, E_pad, bias, T, E, has_gate ? 1 : 0, k, score_mode,
                    renorm, idx, w, shared_gate, hist, blk_counts, batch_counts, ticket, blk_prefix,
                    sync ? *sync : PeerSync(), stage_counts ? 1 : 0);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? MP_OK : set_cuda_error(e, "router_select_kernel launch");
}

}  // namespace mp
