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
// Layout: Wg is repacked once into [d/4][E_tot][4] fp32 so that threads owning
// consecutive experts read consecutive 16 B words.  A CTA owns 16 tokens; the x
// rows and the matching Wg columns are staged through shared memory in k-chunks
// by a double-buffered cp.async pipeline, so the FMA chains only see LDS latency.
#include "common.cuh"
#include "mp_internal.h"

namespace mp {

namespace rt {
constexpr int kThreads = 128;
constexpr int kTokens = 16;    // tokens per CTA
constexpr int kMaxE = 64;      // routed experts
constexpr int kMaxItems = (kTokens * (kMaxE + 1) + kThreads - 1) / kThreads;
constexpr int kMaxK = 8;
}  // namespace rt

int router_block_tokens() { return rt::kTokens; }

__global__ void router_pack_kernel(const __nv_bfloat16* __restrict__ wg, int E_tot, int d, float* __restrict__ packed) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;  // over E_tot * d
  if (i >= E_tot * d) return;
  const int e = i / d, k = i - e * d;
  packed[(size_t(k >> 2) * E_tot + e) * 4 + (k & 3)] = __bfloat162float(wg[i]);
}

int launch_router_pack(const __nv_bfloat16* wg, int E_tot, int d, float* packed, cudaStream_t stream) {
  if (d % 4 != 0) return set_error(MP_E_SHAPE, "router d=%d not a multiple of 4", d);
  const int n = E_tot * d;
  router_pack_kernel<<<(n + 255) / 256, 256, 0, stream>>>(wg, E_tot, d, packed);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MP_OK : set_cuda_error(e, "router_pack_kernel launch");
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

// Shared memory per stage: x chunk [16][kc] bf16 + Wg chunk [kc/4][E_tot][4] fp32,
// double-buffered and filled with cp.async while the previous chunk is consumed.
template <int kItems>
__global__ void __launch_bounds__(rt::kThreads)
    router_kernel(const __nv_bfloat16* __restrict__ x, const float4* __restrict__ wp, const float* __restrict__ bias,
                  int T, int d, int E, int has_gate, int k, int score_mode, int renorm, int kc,
                  int32_t* __restrict__ idx, float* __restrict__ wout, float* __restrict__ shared_gate,
                  uint32_t* __restrict__ hist, int32_t* __restrict__ blk_counts, int32_t* __restrict__ batch_counts) {
  extern __shared__ __align__(16) uint8_t rsm[];
  __shared__ float logits[rt::kTokens][rt::kMaxE + 1];
  __shared__ int cnt_s[rt::kMaxE];

  const int E_tot = E + has_gate;
  const int t0 = blockIdx.x * rt::kTokens;
  const int tid = threadIdx.x;
  const int x_bytes = rt::kTokens * kc * 2;
  const int w_bytes = E_tot * kc * 4;
  const int stage_bytes = x_bytes + w_bytes;
  for (int e = tid; e < E; e += blockDim.x) cnt_s[e] = 0;

  int it_t[kItems], it_e[kItems];
  float acc[kItems];
#pragma unroll
  for (int m = 0; m < kItems; ++m) {
    const int i = tid + m * rt::kThreads;
    it_t[m] = i / E_tot;
    it_e[m] = i - it_t[m] * E_tot;
    acc[m] = 0.0f;
  }
  const int n_items = rt::kTokens * E_tot;
  const int n_chunks = d / kc;

  auto issue = [&](int c) {
    uint8_t* base = rsm + (c & 1) * stage_bytes;
    const int k0 = c * kc;
    const int xv = kc / 8;  // 16 B vectors per token row
    for (int v = tid; v < rt::kTokens * xv; v += blockDim.x) {
      const int tt = v / xv, c8 = (v - tt * xv) * 8;
      const bool ok = t0 + tt < T;
      const __nv_bfloat16* src = ok ? x + size_t(t0 + tt) * d + k0 + c8 : x;
      cp_async_16(base + (tt * kc + c8) * 2, src, ok ? 16u : 0u);
    }
    const float4* wsrc = wp + size_t(k0 >> 2) * E_tot;
    float4* wdst = reinterpret_cast<float4*>(base + x_bytes);
    for (int v = tid; v < (kc >> 2) * E_tot; v += blockDim.x) cp_async_16(wdst + v, wsrc + v, 16u);
    cp_async_commit();
  };

  issue(0);
  for (int c = 0; c < n_chunks; ++c) {
    if (c + 1 < n_chunks) {
      issue(c + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const uint8_t* base = rsm + (c & 1) * stage_bytes;
    const __nv_bfloat16* xs = reinterpret_cast<const __nv_bfloat16*>(base);
    const float4* ws = reinterpret_cast<const float4*>(base + x_bytes);
#pragma unroll
    for (int m = 0; m < kItems; ++m) {
      if (tid + m * rt::kThreads < n_items) {
        const uint4* xrow = reinterpret_cast<const uint4*>(xs + it_t[m] * kc);
        const float4* wcol = ws + it_e[m];
        float a = acc[m];
#pragma unroll 4
        for (int kk = 0; kk < kc; kk += 8) {
          const uint4 xv = xrow[kk >> 3];
          const float4 w0 = wcol[(kk >> 2) * E_tot];
          const float4 w1 = wcol[((kk >> 2) + 1) * E_tot];
          // strictly ascending k: one fp32 FMA chain per logit
          a = fmaf(bf16_lo(xv.x), w0.x, a);
          a = fmaf(bf16_hi(xv.x), w0.y, a);
          a = fmaf(bf16_lo(xv.y), w0.z, a);
          a = fmaf(bf16_hi(xv.y), w0.w, a);
          a = fmaf(bf16_lo(xv.z), w1.x, a);
          a = fmaf(bf16_hi(xv.z), w1.y, a);
          a = fmaf(bf16_lo(xv.w), w1.z, a);
          a = fmaf(bf16_hi(xv.w), w1.w, a);
        }
        acc[m] = a;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int m = 0; m < kItems; ++m) {
    if (tid + m * rt::kThreads < n_items) {
      float v = acc[m];
      if (bias != nullptr && it_e[m] < E) v = __fadd_rn(v, bias[it_e[m]]);
      logits[it_t[m]][it_e[m]] = v;
    }
  }
  __syncthreads();

  // ---- top-k + weights: one warp per token (4 warps x 4 rounds)
  const int warp = warp_id(), lane = lane_id();
  for (int tt = warp; tt < rt::kTokens; tt += rt::kThreads / 32) {
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
    if (c) {
      if (hist) atomicAdd(&hist[e], uint32_t(c));
      if (batch_counts) atomicAdd(&batch_counts[e], c);
    }
  }
}

int launch_router(const __nv_bfloat16* x, const float* wg_packed, const float* bias, int T, int d, int E,
                  int has_gate, int k, int score_mode, int renorm, int32_t* idx, float* w, float* shared_gate,
                  uint32_t* hist, int32_t* blk_counts, int32_t* batch_counts, cudaStream_t stream) {
  if (E < 1 || E > rt::kMaxE) return set_error(MP_E_SHAPE, "router: E=%d outside [1, %d]", E, rt::kMaxE);
  if (k < 1 || k > E || k > rt::kMaxK) return set_error(MP_E_SHAPE, "router: top_k=%d invalid for E=%d", k, E);
  if (d % 8 != 0) return set_error(MP_E_SHAPE, "router: d=%d not a multiple of 8", d);
  if (score_mode != 0 && score_mode != 1) return set_error(MP_E_ARG, "router: score_mode %d", score_mode);
  if (T <= 0) return MP_OK;
  const int E_tot = E + (has_gate ? 1 : 0);
  const int items = (rt::kTokens * E_tot + rt::kThreads - 1) / rt::kThreads;
  const int grid = (T + rt::kTokens - 1) / rt::kTokens;
  const float4* wp = reinterpret_cast<const float4*>(wg_packed);
  int kc = E_tot <= 16 ? 256 : 128;
  while (d % kc) kc >>= 1;
  if (kc < 8) return set_error(MP_E_SHAPE, "router: d=%d not a multiple of 8", d);
  const size_t smem = size_t(2) * (rt::kTokens * kc * 2 + E_tot * kc * 4);
#define MP_ROUTER_CASE(N)                                                                                       \
  case N:                                                                                                      \
    if (smem > 48 * 1024)                                                                                      \
      cudaFuncSetAttribute(router_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));          \
    router_kernel<N><<<grid, rt::kThreads, smem, stream>>>(x, wp, bias, T, d, E, has_gate ? 1 : 0, k, score_mode, \
                                                           renorm, kc, idx, w, shared_gate, hist, blk_counts,    \
                                                           batch_counts);                                        \
    break;
  switch (items) {
    MP_ROUTER_CASE(1)
    MP_ROUTER_CASE(2)
    MP_ROUTER_CASE(3)
    MP_ROUTER_CASE(4)
    MP_ROUTER_CASE(5)
    MP_ROUTER_CASE(6)
    MP_ROUTER_CASE(7)
    MP_ROUTER_CASE(8)
    MP_ROUTER_CASE(9)
    default:
      return set_error(MP_E_SHAPE, "router: %d items per thread unsupported", items);
  }
#undef MP_ROUTER_CASE
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MP_OK : set_cuda_error(e, "router_kernel launch");
}

}  // namespace mp
