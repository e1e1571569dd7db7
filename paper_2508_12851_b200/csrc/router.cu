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
// Bit-exactness contract (checked against oracle/moe_oracle.py): every logit
// is ONE sequential fp32 FMA chain over k = 0..d-1 ascending, starting at 0.
// x and Wg are bf16, so every product is exact in fp32 and fma(x,w,acc) ==
// rn(acc + x*w); the oracle restates this with numpy float32 adds.  Selection
// compares logits only, so the indices do not depend on the exp implementation.
//
// Layout: Wg is repacked once into [d][E_pad] fp32 (Wg^T, E_pad = E_tot
// rounded up to 8, zero columns), so the TE weights of one k are contiguous.  A CTA owns 32 tokens (one per lane) and all experts (TE per
// warp); x rows and Wg columns are staged through shared memory in k-chunks by
// a double-buffered cp.async pipeline.
#include <cstdlib>

#include "common.cuh"
#include "mp_internal.h"

namespace mp {

namespace rt {
constexpr int kTokens = 32;    // tokens per CTA (also the permute / histogram block)
constexpr int kMaxE = 64;      // routed experts
constexpr int kMaxK = 8;
}  // namespace rt

int router_block_tokens() { return rt::kTokens; }
__host__ __device__ int router_e_pad(int E_tot) { return (E_tot + 7) / 8 * 8; }

// packed[k][E_pad] fp32 = Wg[e][k] (Wg transposed; zero columns pad E_tot up to E_pad)
__global__ void router_pack_kernel(const __nv_bfloat16* __restrict__ wg, int E_tot, int E_pad, int d,
                                   float* __restrict__ packed) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;  // over d * E_pad
  if (i >= E_pad * d) return;
  const int k = i / E_pad, e = i - k * E_pad;
  packed[i] = e < E_tot ? __bfloat162float(wg[size_t(e) * d + k]) : 0.0f;
}

int launch_router_pack(const __nv_bfloat16* wg, int E_tot, int d, float* packed, cudaStream_t stream) {
  if (d % 8 != 0) return set_error(MP_E_SHAPE, "router d=%d not a multiple of 8", d);
  const int E_pad = router_e_pad(E_tot);
  const int n = E_pad * d;
  router_pack_kernel<<<(n + 255) / 256, 256, 0, stream>>>(wg, E_tot, E_pad, d, packed);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MP_OK : set_cuda_error(e, "router_pack_kernel launch");
}

// acc = (acc.lo + x*w.lo, acc.hi + x*w.hi): two independent fp32 FMAs (FFMA2),
// each rounded exactly like fmaf -- the per-logit chain contract is unchanged.
MP_DEV void ffma2(unsigned long long& acc, float x, unsigned long long w) {
  const unsigned long long xx = (unsigned long long)__float_as_uint(x) | ((unsigned long long)__float_as_uint(x) << 32);
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(xx), "l"(w));
}
MP_DEV unsigned long long pack2(float lo, float hi) {
  return (unsigned long long)__float_as_uint(lo) | ((unsigned long long)__float_as_uint(hi) << 32);
}

// Larger logit wins; equal logits -> lower expert id.
MP_DEV bool better(float a, int ia, float b, int ib) { return a > b || (a == b && ia < ib); }

MP_DEV void cp_async_16(void* smem, const void* gmem, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem), "r"(src_bytes)
               : "memory");
}
MP_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
MP_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// CTA = 32 tokens x (E_pad / TE) warps.  Lane = token, warp = a group of TE
// consecutive experts: every x element is loaded once per thread and feeds TE
// independent fp32 chains, two per FFMA2 instruction; the Wg values of one k
// are warp-uniform (shared-memory broadcast).  Per stage, shared memory holds
// the x chunk [32][kc+8] bf16 (padded rows: conflict-free 16 B lane loads) and
// the Wg chunk [kc][E_pad] fp32; kStages-deep cp.async ring.
constexpr int kStages = 4;
template <int TE>
__global__ void __launch_bounds__(512)
    router_kernel(const __nv_bfloat16* __restrict__ x, const uint4* __restrict__ wp, const float* __restrict__ bias,
                  int T, int d, int E, int has_gate, int k, int score_mode, int renorm, int kc,
                  int32_t* __restrict__ idx, float* __restrict__ wout, float* __restrict__ shared_gate,
                  uint32_t* __restrict__ hist, int32_t* __restrict__ blk_counts, int32_t* __restrict__ batch_counts,
                  uint32_t* __restrict__ ticket, int32_t* __restrict__ blk_prefix) {
  extern __shared__ __align__(16) uint8_t rsm[];
  __shared__ float logits[rt::kTokens][rt::kMaxE + 2];
  __shared__ int cnt_s[rt::kMaxE];

  const int E_tot = E + has_gate;
  const int E_pad = router_e_pad(E_tot);
  const int t0 = blockIdx.x * rt::kTokens;
  const int tid = threadIdx.x, lane = lane_id(), warp = warp_id();
  const int pitch = kc + 8;                       // bf16 elements per staged x row
  const int x_bytes = rt::kTokens * pitch * 2;
  const int w_bytes = kc * E_pad * 4;
  const int stage_bytes = x_bytes + w_bytes;
  for (int e = tid; e < E; e += blockDim.x) cnt_s[e] = 0;

  unsigned long long acc[TE / 2];
#pragma unroll
  for (int j = 0; j < TE / 2; ++j) acc[j] = 0ull;
  const int e0 = warp * TE;
  const int n_chunks = d / kc;

  auto issue = [&](int c) {
    uint8_t* base = rsm + (c % kStages) * stage_bytes;
    const int k0 = c * kc;
    const int xv = kc / 8;
    for (int v = tid; v < rt::kTokens * xv; v += blockDim.x) {
      const int tt = v / xv, c8 = (v - tt * xv) * 8;
      const bool ok = t0 + tt < T;
      const __nv_bfloat16* src = ok ? x + size_t(t0 + tt) * d + k0 + c8 : x;
      cp_async_16(base + (tt * pitch + c8) * 2, src, ok ? 16u : 0u);
    }
    const uint4* wsrc = wp + size_t(k0) * E_pad / 4;
    uint4* wdst = reinterpret_cast<uint4*>(base + x_bytes);
    for (int v = tid; v < kc * E_pad / 4; v += blockDim.x) cp_async_16(wdst + v, wsrc + v, 16u);
  };

  // prologue: kStages-1 chunks in flight (one commit group per chunk, empty groups past the end)
#pragma unroll
  for (int c = 0; c < kStages - 1; ++c) {
    if (c < n_chunks) issue(c);
    cp_async_commit();
  }
  for (int c = 0; c < n_chunks; ++c) {
    if (c + kStages - 1 < n_chunks) issue(c + kStages - 1);
    cp_async_commit();
    cp_async_wait<kStages - 1>();
    __syncthreads();
    const uint8_t* base = rsm + (c % kStages) * stage_bytes;
    const uint4* xrow = reinterpret_cast<const uint4*>(base + size_t(lane) * pitch * 2);
    const float* ws = reinterpret_cast<const float*>(base + x_bytes) + e0;
#pragma unroll 2
    for (int kk = 0; kk < kc; kk += 8) {
      const uint4 xv = xrow[kk >> 3];
      const float xs[8] = {bf16_lo(xv.x), bf16_hi(xv.x), bf16_lo(xv.y), bf16_hi(xv.y),
                           bf16_lo(xv.z), bf16_hi(xv.z), bf16_lo(xv.w), bf16_hi(xv.w)};
#pragma unroll
      for (int q = 0; q < 8; ++q) {   // strictly ascending k
        const float* wr = ws + size_t(kk + q) * E_pad;
        if constexpr (TE == 2) {
          const float2 w = *reinterpret_cast<const float2*>(wr);
          ffma2(acc[0], xs[q], pack2(w.x, w.y));
        } else {
#pragma unroll
          for (int j = 0; j < TE / 4; ++j) {
            const float4 w = reinterpret_cast<const float4*>(wr)[j];
            ffma2(acc[2 * j], xs[q], pack2(w.x, w.y));
            ffma2(acc[2 * j + 1], xs[q], pack2(w.z, w.w));
          }
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < TE; ++j) {
    const int e = e0 + j;
    if (e < E_tot) {
      float v = __uint_as_float(uint32_t(acc[j >> 1] >> ((j & 1) * 32)));
      if (bias != nullptr && e < E) v = __fadd_rn(v, bias[e]);
      logits[lane][e] = v;
    }
  }
  __syncthreads();

  // ---- top-k + weights: one warp per token
  for (int tt = warp; tt < rt::kTokens; tt += blockDim.x / 32) {
    const int t = t0 + tt;
    if (t >= T) break;
    float v0 = lane < E ? logits[tt][lane] : -INFINITY;
    float v1 = lane + 32 < E ? logits[tt][lane + 32] : -INFINITY;
    bool taken0 = lane >= E, taken1 = lane + 32 >= E;
    float sel_v[rt::kMaxK];
    int sel_i[rt::kMaxK];
    for (int j = 0; j < k; ++j) {
      float bv = -INFINITY;
      int bi = 0x7fffffff;
      if (!taken0) { bv = v0; bi = lane; }
      if (!taken1 && (bi == 0x7fffffff || better(v1, lane + 32, bv, bi))) { bv = v1; bi = lane + 32; }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (oi != 0x7fffffff && (bi == 0x7fffffff || better(ov, oi, bv, bi))) { bv = ov; bi = oi; }
      }
      sel_v[j] = bv;
      sel_i[j] = bi;
      if (bi == lane) taken0 = true;
      if (bi == lane + 32) taken1 = true;
    }
    // weights
    const float mx = sel_v[0];
    float denom;
    if (score_mode == 0) {
      denom = 0.f;
      for (int j = 0; j < k; ++j) denom += expf(sel_v[j] - mx);
    } else {
      float s = (lane < E ? expf(v0 - mx) : 0.f) + (lane + 32 < E ? expf(v1 - mx) : 0.f);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      denom = s;
    }
    if (lane == 0) {
      float wsum = 0.f;
      float wj[rt::kMaxK];
      for (int j = 0; j < k; ++j) {
        wj[j] = expf(sel_v[j] - mx) / denom;
        wsum += wj[j];
      }
      for (int j = 0; j < k; ++j) {
        idx[size_t(t) * k + j] = sel_i[j];
        wout[size_t(t) * k + j] = (score_mode == 1 && renorm) ? wj[j] / wsum : wj[j];
        atomicAdd(&cnt_s[sel_i[j]], 1);
      }
      if (has_gate && shared_gate != nullptr) {
        const float g = logits[tt][E];
        shared_gate[t] = 1.0f / (1.0f + expf(-g));
      }
    }
  }
  __syncthreads();
  for (int e = tid; e < E; e += blockDim.x) {
    const int c = cnt_s[e];
    if (blk_counts) blk_counts[size_t(blockIdx.x) * E + e] = c;
    if (c && hist) atomicAdd(&hist[e], uint32_t(c));
  }
  if (batch_counts == nullptr || blk_counts == nullptr) return;
  // The last CTA to finish reduces the per-block counts into this batch's
  // per-expert counts (integer sums: order-independent), so they are ready when
  // the kernel completes -- no memset, no second pass.
  __shared__ int is_last;
  __threadfence();
  __syncthreads();
  if (tid == 0) is_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  const int nb = gridDim.x;
  // stage the [nb][E] block-count matrix in the (now idle) dynamic smem ring with
  // coalesced loads, then per-expert scans run from shared memory
  int* bc = reinterpret_cast<int*>(rsm);
  const bool staged = size_t(nb) * E * 4 <= size_t(kStages) * stage_bytes;
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
  if (tid == 0) *ticket = 0u;  // ready for the next launch (stream-ordered)
}

int launch_router(const __nv_bfloat16* x, const float* wg_packed, const float* bias, int T, int d, int E,
                  int has_gate, int k, int score_mode, int renorm, int32_t* idx, float* w, float* shared_gate,
                  uint32_t* hist, int32_t* blk_counts, int32_t* batch_counts, uint32_t* ticket,
                  int32_t* blk_prefix, cudaStream_t stream) {
  if (batch_counts && !ticket) return set_error(MP_E_ARG, "router: batch counts need a ticket word");
  if (E < 1 || E > rt::kMaxE) return set_error(MP_E_SHAPE, "router: E=%d outside [1, %d]", E, rt::kMaxE);
  if (k < 1 || k > E || k > rt::kMaxK) return set_error(MP_E_SHAPE, "router: top_k=%d invalid for E=%d", k, E);
  if (d % 8 != 0) return set_error(MP_E_SHAPE, "router: d=%d not a multiple of 8", d);
  if (score_mode != 0 && score_mode != 1) return set_error(MP_E_ARG, "router: score_mode %d", score_mode);
  if (T <= 0) return MP_OK;
  const int E_tot = E + (has_gate ? 1 : 0);
  const int E_pad = router_e_pad(E_tot);
  int TE = E_pad <= 16 ? 2 : 4;
  if (const char* env = getenv("MP_ROUTER_TE")) {  // tuning override (2, 4 or 8)
    const int v = atoi(env);
    if ((v == 2 || v == 4 || v == 8) && E_pad % v == 0 && E_pad / v <= 16) TE = v;
  }
  const int warps = E_pad / TE;
  const int grid = (T + rt::kTokens - 1) / rt::kTokens;
  const uint4* wp = reinterpret_cast<const uint4*>(wg_packed);
  int kc = E_pad <= 16 ? 256 : 128;
  while (d % kc) kc >>= 1;
  const size_t smem = size_t(kStages) * (rt::kTokens * (kc + 8) * 2 + size_t(kc) * E_pad * 4);
  cudaError_t e;
#define MP_ROUTER_LAUNCH(N)                                                                                    \
  e = cudaFuncSetAttribute(router_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));        \
  if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(router)");                            \
  router_kernel<N><<<grid, 32 * warps, smem, stream>>>(x, wp, bias, T, d, E, has_gate ? 1 : 0, k, score_mode, \
                                                       renorm, kc, idx, w, shared_gate, hist, blk_counts,     \
                                                       batch_counts, ticket, blk_prefix)
  if (TE == 2) {
    MP_ROUTER_LAUNCH(2);
  } else if (TE == 4) {
    MP_ROUTER_LAUNCH(4);
  } else {
    MP_ROUTER_LAUNCH(8);
  }
#undef MP_ROUTER_LAUNCH
  e = cudaGetLastError();
  return e == cudaSuccess ? MP_OK : set_cuda_error(e, "router_kernel launch");
}

}  // namespace mp
