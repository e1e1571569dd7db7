// K2 permute+dispatch and K5 combine.
//
// Reference anchors:
//   * target rule  `_choose_target` (reference pkg/src/moeplace/sim.py:433-439):
//     folded into route[origin][expert] on the host once per placement;
//   * per-target grouping in `_dispatch_layer` (sim.py:446-457): here every
//     (token, slot) pair is stably counting-sorted by (target GPU, expert);
//   * remote payload accounting 2*tokens*d*bpe (sim.py:454, domain.py:193-194):
//     the rows written to a peer's receive buffer here, and returned by the
//     peer's GEMM2 epilogue, are exactly the reference's "remote invocations"
//     at token granularity (payload out + result back).
//
// Receive-buffer layout on GPU D (identical formula on every rank, so no
// per-row metadata crosses NVLink): rows grouped by expert id ascending; inside
// an expert group, rows ordered by source GPU ascending, then by (token, slot)
// of that source.  M[D][e] = sum_s [route[s][e]==D] * C[s][e].  The offsets are
// recomputed where they are needed (permute CTAs, GEMM prologues) from the
// exchanged count table -- there is no separate layout kernel.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "mp_internal.h"
#include "peer_sync.cuh"

namespace mp {

// ------------------------------------------------------------------ K2 permute + dispatch
// CTA = one router block of 32 tokens (the histogram blocks), 256 threads.
// Prologue (the "layout", recomputed per CTA from tiny inputs, no extra launch):
//   * my_base[e]: first row of this origin's expert-e rows in the target GPU's
//     receive buffer = rows of lower experts on that GPU + rows of lower-ranked
//     sources for e (from the exchanged counts C[G][E] and the route table);
//   * prefix[e]: rows of expert e in this origin's earlier router blocks, summed
//     here from the router's per-block counts (coalesced over experts, loads in flight).
// Phase 1: one thread per (token, slot) pair computes its stable in-block rank
//          (__match_any_sync within a warp, a per-expert prefix across warps).
// Phase 2: one warp per token loads the x row once (16 B per lane per step) and
//          stores it to its k destinations, local or peer (NVLink) rows.
template <int kVecPerLane>
__global__ void __launch_bounds__(256)
    permute_kernel(const __nv_bfloat16* __restrict__ x, const int32_t* __restrict__ idx,
                   const int32_t* __restrict__ route, const int32_t* __restrict__ counts_all,
                   const uint32_t* __restrict__ parity, const int32_t* __restrict__ blk_counts,
                   int32_t* const* __restrict__ src_ptrs, int rank, int G, int T, int d, int E, int k,
                   __nv_bfloat16* const* __restrict__ recv_ptrs, int32_t* __restrict__ pos_dst,
                   int32_t* __restrict__ pos_row, const PeerSync sync) {
  constexpr int kTok = 32;
  __shared__ int s_e[kTok * 8];
  __shared__ int s_dst[kTok * 8];
  __shared__ int s_row[kTok * 8];
  __shared__ int C[8][64], R[8][64];
  __shared__ int base_s[64];
  __shared__ int wcnt[8][64];  // per-warp, per-expert pair counts -> exclusive prefix over warps
  __shared__ int Mpre[8][64];  // rows of lower experts on GPU D (exclusive prefix over experts)
  __shared__ int pre_s[64];  // this origin's rows of each expert in earlier router blocks
  __shared__ int pre_seg[4][64];
  const int b = blockIdx.x;
  const int t0 = b * kTok;
  const int nt = min(kTok, T - t0);
  const int np = nt * k;
  const int tid = threadIdx.x;
  griddep_launch_dependents();
  griddep_wait();
  // count exchange: every rank's counts of this forward are in our table once
  // all flags reached epoch A (raised by each rank's router)
  if (peer_on(sync) && sync.wait) peer_wait_cta(sync);
  if (parity != nullptr) counts_all += size_t(*parity) * G * E;
  for (int i = tid; i < G * E; i += blockDim.x) {
    C[i / E][i % E] = __ldcg(counts_all + i);
    R[i / E][i % E] = route[i];
  }
  if (tid < np) s_e[tid] = idx[size_t(t0) * k + tid];
  for (int i = tid; i < 8 * 64; i += blockDim.x) (&wcnt[0][0])[i] = 0;
  {  // block prefix: thread (segment, expert) sums blocks seg, seg + S, ... below b -- lanes over
    // consecutive experts (coalesced), 32 loads in flight per thread -- then a sum over segments
    const int S = blockDim.x / 64, e = tid & 63, seg = tid >> 6;
    int sum = 0;
    if (e < E)
      for (int b0 = seg; b0 < b; b0 += 32 * S) {
        int v[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          const int bb = b0 + u * S;
          v[u] = bb < b ? __ldcg(blk_counts + size_t(bb) * E + e) : 0;
        }
#pragma unroll
        for (int u = 0; u < 32; ++u) sum += v[u];
      }
    pre_seg[seg][e] = sum;
  }
  __syncthreads();
  if (tid < 64) {
    int t = 0;
    for (int q = 0; q < int(blockDim.x / 64); ++q) t += pre_seg[q][tid];
    pre_s[tid] = t;
  }
  __syncthreads();
  // receive layout of every GPU D: rows of expert e2 on D = sum over sources routing e2 to D;
  // warp D scans them over the experts (exclusive), so each expert's base is O(G) work
  {
    const int w = tid >> 5, l = tid & 31;
    if (w < G) {
      int m[2] = {0, 0};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int e2 = l + 32 * h;
        if (e2 < E)
          for (int s = 0; s < G; ++s)
            if (R[s][e2] == w) m[h] += C[s][e2];
      }
      int p0 = m[0], p1 = m[1];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t0 = __shfl_up_sync(0xffffffffu, p0, o), t1 = __shfl_up_sync(0xffffffffu, p1, o);
        if (l >= o) {
          p0 += t0;
          p1 += t1;
        }
      }
      const int tot0 = __shfl_sync(0xffffffffu, p0, 31);
      Mpre[w][l] = p0 - m[0];
      Mpre[w][l + 32] = tot0 + p1 - m[1];
    }
  }
  __syncthreads();
  if (tid < E) {
    const int e = tid, D = R[rank][e];
    int base = pre_s[e] + Mpre[D][e];
    for (int s = 0; s < rank; ++s)
      if (R[s][e] == D) base += C[s][e];
    base_s[e] = base;
  }
  // stable in-block rank of each pair among the block's pairs of the same expert:
  // within a warp from __match_any_sync, across warps from a per-expert prefix
  const int w = tid >> 5, l = tid & 31;
  const int e_my = tid < np ? s_e[tid] : -1;
  const unsigned act = __ballot_sync(0xffffffffu, tid < np);
  int lrank = 0;
  if (tid < np) {
    const unsigned m = __match_any_sync(act, e_my);
    lrank = __popc(m & ((1u << l) - 1u));
    if (lrank == 0) wcnt[w][e_my] = __popc(m);
  }
  __syncthreads();
  if (tid < E) {
    int run = 0;
    for (int w2 = 0; w2 < 8; ++w2) {
      const int c = wcnt[w2][tid];
      wcnt[w2][tid] = run;
      run += c;
    }
  }
  __syncthreads();
  if (tid < np) {
    const int e = e_my;
    const int r = wcnt[w][e] + lrank;
    const int dst = R[rank][e];
    const int row = base_s[e] + r;
    s_dst[tid] = dst;
    s_row[tid] = row;
    if (blockIdx.y == 0) {
      pos_dst[size_t(t0) * k + tid] = dst;
      pos_row[size_t(t0) * k + tid] = row;
      // where this row's expert output must return: (origin rank, pair index)
      src_ptrs[dst][row] = int32_t((uint32_t(rank) << 24) | uint32_t(t0 * k + tid));
    }
  }
  __syncthreads();
  const int warp = warp_id(), lane = lane_id();
  // blockIdx.y: this CTA's column slice of the rows (small batches spread the row
  // copies over more SMs; the pair bookkeeping above is repeated, slice 0 writes it)
  const int nvec_all = d / 8;  // 16 B vectors per row
  const int per = nvec_all / gridDim.y;
  const int c_lo = blockIdx.y * per;
  const int nvec = per;
  // the next token's row is loaded before this token's k stores are issued (the asm
  // loads / stores keep program order): one load round trip per warp, not per token
  auto load_row = [&](int tt, uint4 (&v)[kVecPerLane]) {
    const __nv_bfloat16* src = x + size_t(t0 + tt) * d + 8 * c_lo;
#pragma unroll
    for (int i = 0; i < kVecPerLane; ++i) {
      const int c = lane + 32 * i;
      if (c < nvec) v[i] = ld_nc_v4(src + 8 * c);
    }
  };
  auto store_row = [&](int tt, const uint4 (&v)[kVecPerLane]) {
    for (int j = 0; j < k; ++j) {
      __nv_bfloat16* dst = recv_ptrs[s_dst[tt * k + j]] + size_t(s_row[tt * k + j]) * d + 8 * c_lo;
#pragma unroll
      for (int i = 0; i < kVecPerLane; ++i) {
        const int c = lane + 32 * i;
        if (c < nvec) st_v4(dst + 8 * c, v[i]);
      }
    }
  };
  if (kVecPerLane <= 8) {
    uint4 va[kVecPerLane], vb[kVecPerLane];
    int tt = warp;
    if (tt < nt) load_row(tt, va);
    for (; tt < nt; tt += 16) {
      if (tt + 8 < nt) load_row(tt + 8, vb);
      store_row(tt, va);
      if (tt + 8 >= nt) break;
      if (tt + 16 < nt) load_row(tt + 16, va);
      store_row(tt + 8, vb);
    }
  } else {
    for (int tt = warp; tt < nt; tt += 8) {
      uint4 v[kVecPerLane];
      load_row(tt, v);
      store_row(tt, v);
    }
  }
  // dispatch done: the last CTA raises epoch B once every CTA's rows are visible
  if (peer_on(sync) && sync.total > 0) peer_arrive_and_raise(sync);
}

int launch_permute(const __nv_bfloat16* x, const int32_t* idx, const int32_t* route, const int32_t* counts_all,
                   const uint32_t* parity, const int32_t* blk_counts, int32_t* const* src_ptrs, int rank, int G,
                   int T, int d, int E, int k,
                   __nv_bfloat16* const* recv_ptrs, int32_t* pos_dst, int32_t* pos_row, cudaStream_t stream,
                   const PeerSync* sync) {
  if (d % 8 != 0) return set_error(MP_E_SHAPE, "permute: d=%d not a multiple of 8", d);
  if (k > 8) return set_error(MP_E_SHAPE, "permute: top_k=%d > 8", k);
  if (G < 1 || G > 8 || E < 1 || E > 64) return set_error(MP_E_SHAPE, "permute: G=%d E=%d", G, E);
  if (T <= 0) return MP_OK;
  const int grid = (T + 31) / 32;
  // split each block's row copies into column slices until the grid holds about two CTAs
  // per SM (they are small: 8 warps, no dynamic smem, so several are co-resident) -- the
  // copies are bound by the memory-level parallelism of the warps in flight per SM
  int ny = 1;
  while (ny < 16 && grid * ny < 2 * kNumSMs && (d / 8) % (ny * 2) == 0 && (d / 8) / (ny * 2) >= 32) ny *= 2;
  if (const char* env = getenv("MP_PERMUTE_SLICES")) ny = std::max(1, atoi(env));
  if ((d / 8) % ny != 0) return set_error(MP_E_SHAPE, "permute: %d column slices do not divide d=%d", ny, d);
  const int vpl = ((d / 8) / ny + 31) / 32;
  PeerSync ps = sync ? *sync : PeerSync();
  if (ps.total > 0) ps.total = grid * ny;
  cudaError_t e;
#define MP_PERM_LAUNCH(N)                                                                                    \
  e = launch_pdl(permute_kernel<N>, dim3(grid, ny), dim3(256), 0, stream, x, idx, route, counts_all, parity, blk_counts, \
                 src_ptrs, rank, G, T, d, E, k, recv_ptrs, pos_dst, pos_row, ps)
  if (vpl <= 1) MP_PERM_LAUNCH(1);
  else if (vpl <= 2) MP_PERM_LAUNCH(2);
  else if (vpl <= 4) MP_PERM_LAUNCH(4);
  else if (vpl <= 8) MP_PERM_LAUNCH(8);
  else if (vpl <= 16) MP_PERM_LAUNCH(16);
  else if (vpl <= 32) MP_PERM_LAUNCH(32);
  else return set_error(MP_E_SHAPE, "permute: d=%d too large", d);
#undef MP_PERM_LAUNCH
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? MP_OK : set_cuda_error(e, "permute_kernel launch");
}

// ------------------------------------------------------------------ K5 combine
// One warp per token.  The k expert outputs of token t were written back into
// this GPU's return buffer by the (local or remote) GEMM2 epilogues, at rows
// t*k .. t*k+k-1, so the combine is a local, fully coalesced read:
// out[t] = bf16( sum_{j<k} w[t,j] * ret[t*k+j] (+ g[t] * ysh[t]) ), fp32, ascending j.
// Gather form (bases != nullptr; the host-driven NCCL transport): pair (t, j)'s row
// is bases[pos_dst[t,j]] + pos_row[t,j] * d -- the expert output left in the
// receive-layout image of the GPU that computed it.
template <int K>
__global__ void __launch_bounds__(256)
    combine_kernel(const __nv_bfloat16* __restrict__ ret, const float* __restrict__ w, int T, int d,
                   const __nv_bfloat16* __restrict__ shared_y, const float* __restrict__ shared_gate,
                   __nv_bfloat16* __restrict__ out, const PeerSync sync,
                   const __nv_bfloat16* const* __restrict__ bases, const int32_t* __restrict__ pos_dst,
                   const int32_t* __restrict__ pos_row) {
  griddep_launch_dependents();
  griddep_wait();
  // every rank's GEMM2 stored its rows of our tokens into ret (epoch C)
  if (peer_on(sync) && sync.wait) peer_wait_cta(sync);
  const int t = blockIdx.x * 8 + warp_id();
  if (t >= T) return;
  const int lane = lane_id();
  const __nv_bfloat16* src = ret + size_t(t) * K * d;
  const __nv_bfloat16* rows[K];
#pragma unroll
  for (int j = 0; j < K; ++j)
    rows[j] = bases ? bases[pos_dst[size_t(t) * K + j]] + size_t(pos_row[size_t(t) * K + j]) * d
                    : src + size_t(j) * d;
  float wj[K];
#pragma unroll
  for (int j = 0; j < K; ++j) wj[j] = w[size_t(t) * K + j];
  const float g = shared_gate ? shared_gate[t] : 1.0f;
  // blockIdx.y: this CTA's column slice of the token rows (more, smaller CTAs even out the
  // per-SM work of a one-wave grid)
  const int nvec = d / 8 / int(gridDim.y), c_base = int(blockIdx.y) * nvec;
#pragma unroll
  for (int j = 0; j < K; ++j) rows[j] += size_t(8) * c_base;
  if (shared_y) shared_y += size_t(8) * c_base;
  out += size_t(8) * c_base;
  // U column vectors per lane per batch: all their loads are issued before any
  // of their stores (the asm loads / stores keep program order, so an unbatched
  // loop would serialise one load round trip per vector)
  constexpr int U = K <= 4 ? 4 : 2;
  for (int c0 = lane; c0 < nvec; c0 += 32 * U) {
    uint4 v[U][K], sv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + 32 * u;
      if (c < nvec) {
#pragma unroll
        for (int j = 0; j < K; ++j) v[u][j] = ld_cg_v4(rows[j] + 8 * c);  // peer-written: L2
        if (shared_y) sv[u] = ld_nc_v4(shared_y + size_t(t) * d + 8 * c);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + 32 * u;
      if (c >= nvec) break;
      float acc[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = 0.f;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const uint32_t q4[4] = {v[u][j].x, v[u][j].y, v[u][j].z, v[u][j].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          acc[2 * q] = fmaf(wj[j], bf16_lo(q4[q]), acc[2 * q]);
          acc[2 * q + 1] = fmaf(wj[j], bf16_hi(q4[q]), acc[2 * q + 1]);
        }
      }
      if (shared_y) {
        const uint32_t q4[4] = {sv[u].x, sv[u].y, sv[u].z, sv[u].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          acc[2 * q] = fmaf(g, bf16_lo(q4[q]), acc[2 * q]);
          acc[2 * q + 1] = fmaf(g, bf16_hi(q4[q]), acc[2 * q + 1]);
        }
      }
      uint4 o;
      o.x = pack_bf16x2(acc[0], acc[1]);
      o.y = pack_bf16x2(acc[2], acc[3]);
      o.z = pack_bf16x2(acc[4], acc[5]);
      o.w = pack_bf16x2(acc[6], acc[7]);
      st_v4(out + size_t(t) * d + 8 * c, o);
    }
  }
}

int launch_combine(const __nv_bfloat16* ret, const float* w, int T, int d, int k, const __nv_bfloat16* shared_y,
                   const float* shared_gate, __nv_bfloat16* out, cudaStream_t stream, const PeerSync* sync,
                   const __nv_bfloat16* const* bases, const int32_t* pos_dst, const int32_t* pos_row) {
  if (d % 8 != 0) return set_error(MP_E_SHAPE, "combine: d=%d not a multiple of 8", d);
  if (k < 1 || k > 8) return set_error(MP_E_SHAPE, "combine: top_k=%d outside [1, 8]", k);
  if (T <= 0) return MP_OK;
  const int grid = (T + 7) / 8;
  // column slices: 1 unless MP_COMBINE_SLICES asks (each slice keeps >= 32 vectors per row)
  int ny = 1;
  if (const char* env = getenv("MP_COMBINE_SLICES")) ny = std::max(1, atoi(env));
  while (ny > 1 && ((d / 8) % ny != 0 || (d / 8) / ny < 32)) ny /= 2;
  const PeerSync ps = sync ? *sync : PeerSync();
  cudaError_t e = cudaSuccess;
  switch (k) {
#define MP_COMBINE_CASE(N) \
  case N:                                                                                                  \
    e = launch_pdl(combine_kernel<N>, dim3(grid, ny), dim3(256), 0, stream, ret, w, T, d, shared_y, shared_gate, out, ps, \
                   bases, pos_dst, pos_row);                                                                \
    break;
    MP_COMBINE_CASE(1) MP_COMBINE_CASE(2) MP_COMBINE_CASE(3) MP_COMBINE_CASE(4)
    MP_COMBINE_CASE(5) MP_COMBINE_CASE(6) MP_COMBINE_CASE(7) MP_COMBINE_CASE(8)
#undef MP_COMBINE_CASE
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? MP_OK : set_cuda_error(e, "combine_kernel launch");
}

}  // namespace mp
