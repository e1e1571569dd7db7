// K3: grouped expert FFN on the 5th-generation tensor cores (sm_100a).
//
// Stands in for the reference's analytic compute estimate
// `comp_time = (comp_base + comp_per_token * tokens) * load` (reference
// pkg/src/moeplace/cost.py:132-136): here the expert work is real.
//
// For every local expert slot s with M_s routed rows (contiguous in the
// receive buffer), the layer runs two launches of one persistent kernel:
//   GEMM1  H[M_s, f] = silu(X W1^T) * (X W3^T)      (SwiGLU fused in the epilogue)
//   GEMM2  Y[M_s, d] = H W2^T
// W13 is stored per slot as [2f, d] with gate/up rows interleaved in blocks of
// 128 (rows 256b..256b+127 = gate rows 128b.., rows 256b+128.. = up rows
// 128b..), so one 128x256 accumulator tile holds matching gate and up columns.
//
// Kernel anatomy (one CTA per SM, persistent, static round-robin tiles):
//   warp 0      TMA producer: A (128x64) + B (256x64) bf16 tiles, 128B swizzle,
//               4-stage smem ring guarded by full/empty mbarriers
//   warp 1      MMA issuer: one thread issues tcgen05.mma M=128 N=256 K=16 into
//               a double-buffered TMEM accumulator (2 x 256 fp32 columns)
//   warp 2      TMEM allocator (512 columns)
//   warps 4..7  epilogue: tcgen05.ld -> (SwiGLU) -> bf16 -> global
#include <cstdlib>

#include "common.cuh"
#include "mp_internal.h"
#include "peer_sync.cuh"

namespace mp {

namespace gg {
constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 64;
constexpr int kStages = 4;
constexpr int kABytes = BM * BK * 2;  // 16 KB
constexpr int kBBytes = BN * BK * 2;  // 32 KB
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kMaxGroups = MP_MAX_GROUPS;
constexpr int kThreads = 256;
constexpr int kTmemCols = 512;
constexpr size_t kSmemBytes = 1024 /*align slack*/ + size_t(kStages) * kStageBytes + 4096;
}  // namespace gg

struct GemmSmemTail {
  uint64_t full[gg::kStages];
  uint64_t empty[gg::kStages];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
  int n_groups;
  int total_tiles;
  int tile_prefix[gg::kMaxGroups + 1];
  int g_arow[gg::kMaxGroups];
  int g_m[gg::kMaxGroups];
  int g_slot[gg::kMaxGroups];
  int g_orow[gg::kMaxGroups];
  int g_expert[gg::kMaxGroups];  // mode 1: the group's expert id (per-source dispatch waits)
  int g_tmp[64];
};

struct TileCoord {
  int g, m_blk, n_blk;
};

// Source ranks whose dispatched rows fall in rows [r0, r1) of group g (mode 1: the receive
// layout orders an expert's rows by source rank), as a bit mask; other modes: every rank.
template <class Tail>
MP_DEV uint32_t group_row_sources(const Tail& st, const GroupSpec& gs, int g, int r0, int r1) {
  if (gs.mode != 1 || !gs.per_source) return 0xffu;
  const int e = st.g_expert[g] & 0xff, roff = st.g_expert[g] >> 8;  // a tail group starts at roff
  r0 += roff;
  r1 += roff;
  const int32_t* counts = gs.counts + (gs.parity ? size_t(*gs.parity) * gs.G * gs.E : 0);
  uint32_t mask = 0;
  int acc = 0;
  for (int s = 0; s < gs.G && acc < r1; ++s) {
    if (gs.route[s * gs.E + e] != gs.rank) continue;
    const int c = __ldcg(counts + s * gs.E + e);
    if (c > 0 && acc + c > r0) mask |= 1u << s;
    acc += c;
  }
  return mask;
}

// Inclusive warp scan (Kogge-Stone over the 32 lanes).
MP_DEV int warp_incl_scan(int v) {
  const int lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// Prologue shared by both kernels: build the group table in shared memory
// (explicit, derived from the exchanged counts, or a single dense group) and
// the per-group tile prefix.  Called by every thread; warp 0 does the
// compaction and the scans with warp collectives (no serial thread-0 loops
// over the experts on the critical path of every launch).
template <class Tail>
MP_DEV void load_groups(Tail& st, const GroupSpec& gs, int bm, int n_blocks) {
  const int tid = threadIdx.x, lane = lane_id();
  if (gs.mode == 1) {
    if (tid < 32) {
      // experts lane and lane + 32 (E <= 64): rows this GPU computes for them
      const int32_t* counts = gs.counts + (gs.parity ? size_t(*gs.parity) * gs.G * gs.E : 0);
      int m[2] = {0, 0}, slot[2] = {-1, -1};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int e = lane + 32 * h;
        if (e < gs.E) {
          for (int s = 0; s < gs.G; ++s)
            if (gs.route[s * gs.E + e] == gs.rank) m[h] += counts[s * gs.E + e];
          slot[h] = gs.slot_of[e];
        }
      }
      // rows of lower experts (receive layout: expert-major) and the compacted group index
      const int p0 = warp_incl_scan(m[0]);
      const int tot0 = __shfl_sync(0xffffffffu, p0, 31);
      const int p1 = warp_incl_scan(m[1]);
      const int row[2] = {p0 - m[0], tot0 + p1 - m[1]};
      bool sel[2];
      int gm[2], roff[2] = {0, 0};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int mh = m[h];
        sel[h] = mh > 0 && mh >= gs.m_lo && mh < gs.m_hi;
        gm[h] = mh;
        if (gs.tail_role != 0) {  // big group: m >= the split threshold
          const bool big = mh >= (gs.tail_role == 1 ? gs.m_lo : gs.m_hi);
          const int tail = big ? mh % gs.tail_block : 0;
          if (tail > 0 && tail <= gs.tail_max) {
            if (gs.tail_role == 1) {
              gm[h] = mh - tail;  // body
            } else {
              sel[h] = true;      // tail
              gm[h] = tail;
              roff[h] = mh - tail;
            }
          }
        }
      }
      const unsigned b0 = __ballot_sync(0xffffffffu, sel[0]), b1 = __ballot_sync(0xffffffffu, sel[1]);
      const unsigned lt = (1u << lane) - 1u;
      const int idx[2] = {__popc(b0 & lt), __popc(b0) + __popc(b1 & lt)};
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (sel[h]) {
          st.g_arow[idx[h]] = row[h] + roff[h];
          st.g_m[idx[h]] = gm[h];
          st.g_slot[idx[h]] = slot[h];
          st.g_orow[idx[h]] = row[h] + roff[h];
          st.g_expert[idx[h]] = (lane + 32 * h) | (roff[h] << 8);
        }
      if (lane == 0) st.n_groups = __popc(b0) + __popc(b1);
    }
  } else if (gs.mode == 2) {
    if (tid == 0) {
      st.g_arow[0] = 0;
      st.g_m[0] = gs.single_m;
      st.g_slot[0] = 0;
      st.g_orow[0] = 0;
      st.n_groups = gs.single_m > 0 ? 1 : 0;
    }
  } else {
    if (tid == 0) st.n_groups = min(*gs.n_groups, gg::kMaxGroups);
    __syncthreads();
    for (int g = tid; g < st.n_groups; g += blockDim.x) {
      st.g_arow[g] = gs.groups[4 * g + 0];
      st.g_m[g] = gs.groups[4 * g + 1];
      st.g_slot[g] = gs.groups[4 * g + 2];
      st.g_orow[g] = gs.groups[4 * g + 3];
    }
  }
  __syncthreads();
  if (tid < 32) {  // tile prefix over the groups, 32 at a time
    const int ng = st.n_groups;
    int carry = 0;
    if (lane == 0) st.tile_prefix[0] = 0;
    for (int g0 = 0; g0 < ng; g0 += 32) {
      const int g = g0 + lane;
      const int tiles = g < ng ? ((st.g_m[g] + bm - 1) / bm) * n_blocks : 0;
      const int incl = warp_incl_scan(tiles);
      if (g < ng) st.tile_prefix[g + 1] = carry + incl;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) st.total_tiles = carry;
  }
}

template <class Tail>
MP_DEV TileCoord decode_any(const Tail& s, int tile, int n_blocks, int bm) {
  TileCoord c;
  // the group holding `tile`: the last g with tile_prefix[g] <= tile (binary search: every warp
  // role decodes every tile, so a linear scan over up to 128 groups sat on the producer's path)
  int lo = 0, hi = s.n_groups - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (s.tile_prefix[mid] <= tile) lo = mid;
    else hi = mid - 1;
  }
  const int g = lo;  // (an empty group shares its prefix with the next: the last such g is the owner)
  const int local = tile - s.tile_prefix[g];
  const int m_blocks = (s.g_m[g] + bm - 1) / bm;
  c.g = g;
  c.n_blk = local / m_blocks;
  c.m_blk = local - c.n_blk * m_blocks;
  return c;
}


// Output row of the epilogue.  Plain mode: out + orow * out_ld.  Scatter mode
// (GEMM2 of the layer): the row goes straight back to its origin GPU's return
// buffer, at the origin's (token, slot) pair index -- recorded per receive row
// by the permute kernel as (source rank << 24 | pair) -- so the return transfer
// rides NVLink inside the GEMM, tile by tile.
MP_DEV __nv_bfloat16* out_row_ptr(__nv_bfloat16* out, size_t orow, int out_ld, const int32_t* scatter_src,
                                   __nv_bfloat16* const* scatter_ptrs, bool valid) {
  if (scatter_src == nullptr || !valid) return out + orow * size_t(out_ld);
  const uint32_t info = uint32_t(__ldg(scatter_src + orow));
  return scatter_ptrs[info >> 24] + size_t(info & 0xFFFFFFu) * size_t(out_ld);
}

// Epilogue of one 128-row x 256-column accumulator: this thread owns one row
// (TMEM lane), reads 32 columns per tcgen05.ld, applies SwiGLU (GEMM1: columns
// [0,128) gate, [128,256) up) and writes bf16.
MP_DEV void epilogue_store(uint32_t taddr, bool valid, __nv_bfloat16* __restrict__ rowp, int n_blk, int swiglu) {
  if (swiglu) {
    __nv_bfloat16* dst = rowp + size_t(n_blk) * (gg::BN / 2);
#pragma unroll 1
    for (int cc = 0; cc < gg::BN / 2; cc += 32) {
      uint32_t gv[32], uv[32];
      tmem_ld_32x32b_x32(taddr + cc, gv);
      tmem_ld_32x32b_x32(taddr + gg::BN / 2 + cc, uv);
      tmem_ld_wait();
      uint32_t packed[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        float g0 = __uint_as_float(gv[2 * i]), g1 = __uint_as_float(gv[2 * i + 1]);
        float u0 = __uint_as_float(uv[2 * i]), u1 = __uint_as_float(uv[2 * i + 1]);
        float h0 = __fdividef(g0, 1.0f + __expf(-g0)) * u0;
        float h1 = __fdividef(g1, 1.0f + __expf(-g1)) * u1;
        packed[i] = pack_bf16x2(h0, h1);
      }
      if (valid) {
        uint4* p = reinterpret_cast<uint4*>(dst + cc);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          p[i] = make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2], packed[4 * i + 3]);
      }
    }
  } else {
    __nv_bfloat16* dst = rowp + size_t(n_blk) * gg::BN;
#pragma unroll 1
    for (int cc = 0; cc < gg::BN; cc += 32) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(taddr + cc, v);
      tmem_ld_wait();
      uint32_t packed[16];
#pragma unroll
      for (int i = 0; i < 16; ++i)
        packed[i] = pack_bf16x2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
      if (valid) {
        uint4* p = reinterpret_cast<uint4*>(dst + cc);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          p[i] = make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2], packed[4 * i + 3]);
      }
    }
  }
}

// One tile of work (a CTA pair's 256-row tile, or a CTA's 128-row tile): where its
// A / B rows come from, how many k-blocks it runs and where its output goes.
struct TileJob {
  const CUtensorMap* ma;
  const CUtensorMap* mb;
  int a_row, b_row;   // first row of the tile (A) and of its 256 N rows (B)
  int k_blocks;
  int n_blk;
  int m_row0, m_rows;  // tile's first row inside its group, and the group's row count
  bool aux;
  int g;               // routed group (aux: -1)
};

// Static schedule of one cluster.  Without an aux problem: routed tiles
// round-robin.  With one: aux tiles round-robin (tile t -> cluster t mod C),
// then the routed tiles round-robin in reversed cluster order, except the last
// few, which go only to the clusters that drew one aux tile fewer (about
// aux K / routed K tiles each) -- so every cluster ends with about the same
// number of k-blocks while concurrently running clusters still share weight
// tiles in L2.  (Contiguous k-balanced ranges per cluster lose that sharing:
// measured 30% slower.)
struct TileSched {
  int A, aux_mb, aux_kb;
  int s1_begin, s1_end, s1_step;
  int s2_begin, s2_end, s2_step;
};

template <int BM_>
MP_DEV TileSched make_sched(const AuxProblem& aux, int R, int k_blocks, int cluster_id, int C) {
  TileSched ps;
  ps.aux_mb = aux.m > 0 ? (aux.m + BM_ - 1) / BM_ : 0;
  ps.A = ps.aux_mb * (aux.N / gg::BN);
  ps.aux_kb = aux.K / gg::BK;
  ps.s2_begin = ps.s2_end = 0;
  ps.s2_step = 1;
  if (ps.A == 0) {
    ps.s1_begin = cluster_id;
    ps.s1_end = R;
    ps.s1_step = C;
    return ps;
  }
  const int rem = ps.A % C;
  const int extra = rem > 0 ? (ps.aux_kb + k_blocks / 2) / k_blocks : 0;
  const int X = min(R, (C - rem) * extra);
  const int R1 = R - X;
  ps.s1_begin = C - 1 - cluster_id;
  ps.s1_end = R1;
  ps.s1_step = C;
  if (cluster_id >= rem && X > 0) {
    ps.s2_begin = R1 + (cluster_id - rem);
    ps.s2_end = R;
    ps.s2_step = C - rem;
  }
  return ps;
}

template <int BM_, class Tail, class Fn>
MP_DEV void for_each_job(const TileSched& ps, const Tail& st, const AuxProblem& aux,
                              const CUtensorMap* tmA, const CUtensorMap* tmB, int n_blocks, int k_blocks,
                              int b_slot_stride, int b_offset, int cluster_id, int C, Fn&& fn) {
  for (int t = cluster_id; t < ps.A; t += C) {
    TileJob j;
    j.aux = true;
    j.g = -1;
    j.n_blk = t / ps.aux_mb;
    const int m_blk = t - j.n_blk * ps.aux_mb;
    j.ma = &aux.tmA;
    j.mb = &aux.tmB;
    j.m_row0 = m_blk * BM_;
    j.m_rows = aux.m;
    j.a_row = j.m_row0;
    j.b_row = j.n_blk * gg::BN;
    j.k_blocks = ps.aux_kb;
    fn(j);
  }
  for (int seg = 0; seg < 2; ++seg) {
    const int t0 = seg ? ps.s2_begin : ps.s1_begin, t1 = seg ? ps.s2_end : ps.s1_end;
    const int dt = seg ? ps.s2_step : ps.s1_step;
    for (int t = t0; t < t1; t += dt) {
    const TileCoord c = decode_any(st, t, n_blocks, BM_);
    TileJob j;
    j.aux = false;
    j.g = c.g;
    j.n_blk = c.n_blk;
    j.ma = tmA;
    j.mb = tmB;
    j.m_row0 = c.m_blk * BM_;
    j.m_rows = st.g_m[c.g];
    j.a_row = st.g_arow[c.g] + j.m_row0;
    j.b_row = st.g_slot[c.g] * b_slot_stride + b_offset + c.n_blk * gg::BN;
    j.k_blocks = k_blocks;
    fn(j);
    }
  }
}

__global__ void __launch_bounds__(gg::kThreads, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ GroupSpec gs, int N, int K, int b_slot_stride, int b_offset, __nv_bfloat16* __restrict__ out,
                        int out_ld, int swiglu, const int32_t* __restrict__ scatter_src,
                        __nv_bfloat16* const* __restrict__ scatter_ptrs, const PeerSync sync,
                        const __grid_constant__ AuxProblem aux) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smA = smem;
  uint8_t* smB = smem + gg::kStages * gg::kABytes;
  static_assert(sizeof(GemmSmemTail) <= 4096, "GEMM smem tail exceeds its reservation");
  GemmSmemTail& st = *reinterpret_cast<GemmSmemTail*>(smem + gg::kStages * gg::kStageBytes);

  const int warp = warp_id();
  const int lane = lane_id();
  const int n_blocks = N / gg::BN;
  const int k_blocks = K / gg::BK;

  // ---- prologue: barriers, TMEM and descriptor prefetch overlap the previous
  // kernel's tail (PDL); the group table needs its results, so it comes after
  griddep_launch_dependents();
  if (threadIdx.x == 0) {
    for (int i = 0; i < gg::kStages; ++i) {
      mbar_init(&st.full[i], 1);
      mbar_init(&st.empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&st.tfull[i], 1);
      mbar_init(&st.tempty[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (aux.m > 0) {
      tma_prefetch_desc(&aux.tmA);
      tma_prefetch_desc(&aux.tmB);
    }
  }
  if (warp == 2) tmem_alloc<gg::kTmemCols>(&st.tmem_base);
  griddep_wait();
  load_groups(st, gs, gg::BM, n_blocks);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = st.tmem_base;
  const TileSched ts = make_sched<gg::BM>(aux, st.total_tiles, k_blocks, blockIdx.x, gridDim.x);
  auto each_job = [&](auto&& fn) {
    for_each_job<gg::BM>(ts, st, aux, &tmA, &tmB, n_blocks, k_blocks, b_slot_stride, b_offset, blockIdx.x,
                         gridDim.x, fn);
  };

  if (warp == 0) {
    if (lane == 0) {
      // ================= TMA producer
      int stage = 0;
      uint32_t phase = 0;
      // F2: a routed tile waits only for the ranks whose dispatched rows it reads (epoch B
      // of each); this GPU's own rows are complete by stream order
      const bool waits = peer_on(sync) && sync.wait;
      const uint32_t epoch = waits ? sync.state[0] : 0u;
      uint32_t ready = waits ? (1u << sync.rank) : 0xffu;
      if (waits) fence_proxy_async_global();
      each_job([&](const TileJob& j) {
        if (waits && !j.aux) {
          uint32_t need = group_row_sources(st, gs, j.g, j.m_row0, min(j.m_row0 + gg::BM, j.m_rows)) & ~ready;
          if (need) {
            const uint64_t t0 = globaltimer_ns();
            for (int p = 0; p < sync.G; ++p)
              if (need >> p & 1u) peer_wait_one(sync, p, epoch, t0);
            fence_proxy_async_global();
            ready |= need;
          }
        }
        for (int kb = 0; kb < j.k_blocks; ++kb) {
          mbar_wait(&st.empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&st.full[stage], gg::kStageBytes);
          tma_load_2d(smA + stage * gg::kABytes, j.ma, &st.full[stage], kb * gg::BK, j.a_row);
          tma_load_2d(smB + stage * gg::kBBytes, j.mb, &st.full[stage], kb * gg::BK, j.b_row);
          if (++stage == gg::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      });
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ================= MMA issuer
      constexpr uint32_t idesc = make_idesc_bf16(gg::BM, gg::BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      each_job([&](const TileJob& j) {
        mbar_wait(&st.tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + uint32_t(acc * gg::BN);
        for (int kb = 0; kb < j.k_blocks; ++kb) {
          mbar_wait(&st.full[stage], phase);
          tc_fence_after();
          const uint64_t adesc = make_sdesc_sw128(smem_u32(smA + stage * gg::kABytes));
          const uint64_t bdesc = make_sdesc_sw128(smem_u32(smB + stage * gg::kBBytes));
#pragma unroll
          for (int k = 0; k < gg::BK / 16; ++k) {
            // advance 16 bf16 (32 B) along K inside the 128 B swizzle atom
            umma_bf16(d_tmem, adesc + uint64_t(2 * k), bdesc + uint64_t(2 * k), idesc,
                      (kb | k) != 0 ? 1u : 0u);
          }
          umma_commit(&st.empty[stage]);
          if (++stage == gg::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&st.tfull[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      });
    }
  } else if (warp >= 4) {
    // ================= epilogue (warp w owns TMEM lanes 32*(w%4) .. +31)
    const int q = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    each_job([&](const TileJob& j) {
      const int row = j.m_row0 + q * 32 + lane;
      const bool valid = row < j.m_rows;
      __nv_bfloat16* rowp =
          j.aux ? aux.out + size_t(row) * aux.out_ld
                : out_row_ptr(out, size_t(st.g_orow[j.g] + row), out_ld, scatter_src, scatter_ptrs, valid);
      mbar_wait(&st.tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * gg::BN);
      epilogue_store(taddr, valid, rowp, j.n_blk, swiglu);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&st.tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    });
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<gg::kTmemCols>(tmem_base);
  }
  // GEMM2: the rows this CTA returned over NVLink are counted towards epoch C
  if (peer_on(sync) && sync.total > 0) peer_arrive_and_raise(sync);
}

// ------------------------------------------------------------------ CTA-pair variant
// Same tile math with tcgen05.mma.cta_group::2: a cluster of two CTAs on one
// TPC computes a 256 x 256 tile.  CTA r loads A rows [128r, 128r+128) and B
// rows (N) [128r, 128r+128) of the tile; the leader (r = 0) issues M=256 N=256
// MMAs that read both CTAs' smem and write each CTA's 128 rows into its own
// TMEM.  Per CTA and k-block only 32 KB cross L2 -> smem instead of 48 KB.
//   * full[s]   (leader)  : leader's expect_tx(64 KB) + both CTAs' 2-SM TMA bytes
//   * empty[s]  (both)    : multicast tcgen05.commit from the leader's MMA thread
//   * tfull[a]  (both)    : multicast commit after the tile's last k-block
//   * tempty[a] (leader)  : 8 arrivals = 4 epilogue warps x 2 CTAs (remote arrive)
namespace g2 {
constexpr int BM = 256;  // rows per pair tile (128 per CTA)
constexpr int BN = 256;
constexpr int BK = 64;
constexpr int kStages = 6;
constexpr int kABytes = 128 * BK * 2;  // 16 KB per CTA
constexpr int kBBytes = 128 * BK * 2;  // 16 KB per CTA (its half of N)
constexpr int kStageBytes = kABytes + kBBytes;
constexpr size_t kSmemBytes = 1024 + size_t(kStages) * kStageBytes + 4096;
}  // namespace g2

struct Gemm2SmemTail {
  uint64_t full[g2::kStages];
  uint64_t empty[g2::kStages];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
  int n_groups;
  int total_tiles;
  int tile_prefix[gg::kMaxGroups + 1];
  int g_arow[gg::kMaxGroups];
  int g_m[gg::kMaxGroups];
  int g_slot[gg::kMaxGroups];
  int g_orow[gg::kMaxGroups];
  int g_expert[gg::kMaxGroups];  // mode 1: the group's expert id (per-source dispatch waits)
  int g_tmp[64];
};


__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(gg::kThreads, 1)
    grouped_gemm_2sm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                            const __grid_constant__ GroupSpec gs, int N, int K, int b_slot_stride, int b_offset,
                            __nv_bfloat16* __restrict__ out, int out_ld, int swiglu,
                            const int32_t* __restrict__ scatter_src, __nv_bfloat16* const* __restrict__ scatter_ptrs,
                            const __grid_constant__ AuxProblem aux, const PeerSync sync) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smA = smem;
  uint8_t* smB = smem + g2::kStages * g2::kABytes;
  static_assert(sizeof(Gemm2SmemTail) <= 4096, "GEMM smem tail exceeds its reservation");
  Gemm2SmemTail& st = *reinterpret_cast<Gemm2SmemTail*>(smem + g2::kStages * g2::kStageBytes);

  const int warp = warp_id();
  const int lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster_id = blockIdx.x >> 1;
  const int n_clusters = gridDim.x >> 1;
  const int n_blocks = N / g2::BN;
  const int k_blocks = K / g2::BK;

  griddep_launch_dependents();
  if (threadIdx.x == 0) {
    for (int i = 0; i < g2::kStages; ++i) {
      mbar_init(&st.full[i], 1);
      mbar_init(&st.empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&st.tfull[i], 1);
      mbar_init(&st.tempty[i], 8);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (aux.m > 0) {
      tma_prefetch_desc(&aux.tmA);
      tma_prefetch_desc(&aux.tmB);
    }
  }
  if (warp == 2) tmem_alloc_2sm<gg::kTmemCols>(&st.tmem_base);
  griddep_wait();
  load_groups(st, gs, g2::BM, n_blocks);
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the peer's barriers are initialised before any remote arrive / TMA
  tc_fence_after();
  const uint32_t tmem_base = st.tmem_base;
  const TileSched ps = make_sched<g2::BM>(aux, st.total_tiles, k_blocks, cluster_id, n_clusters);
  auto each_job = [&](auto&& fn) {
    for_each_job<g2::BM>(ps, st, aux, &tmA, &tmB, n_blocks, k_blocks, b_slot_stride, b_offset, cluster_id,
                         n_clusters, fn);
  };

  if (warp == 0) {
    if (lane == 0) {
      // ================= TMA producer (both CTAs load their halves)
      int stage = 0;
      uint32_t phase = 0;
      // F2: a routed tile waits only for the ranks whose dispatched rows this CTA's half of
      // it reads (epoch B of each); own rows are complete by stream order, and the
      // shared-expert tiles scheduled first overlap the waits
      const bool waits = peer_on(sync) && sync.wait;
      const uint32_t epoch = waits ? sync.state[0] : 0u;
      uint32_t ready = waits ? (1u << sync.rank) : 0xffu;
      if (waits) fence_proxy_async_global();
      each_job([&](const TileJob& j) {
        if (waits && !j.aux) {
          const int r0 = j.m_row0 + int(rank) * 128;
          uint32_t need = r0 < j.m_rows ? group_row_sources(st, gs, j.g, r0, min(r0 + 128, j.m_rows)) & ~ready : 0u;
          if (need) {
            const uint64_t t0 = globaltimer_ns();
            for (int p = 0; p < sync.G; ++p)
              if (need >> p & 1u) peer_wait_one(sync, p, epoch, t0);
            fence_proxy_async_global();
            ready |= need;
          }
        }
        const int a_row = j.a_row + int(rank) * 128;
        const int b_row = j.b_row + int(rank) * 128;
        for (int kb = 0; kb < j.k_blocks; ++kb) {
          mbar_wait(&st.empty[stage], phase ^ 1);
          if (leader) mbar_arrive_expect_tx(&st.full[stage], 2 * g2::kStageBytes);
          tma_load_2d_2sm(smA + stage * g2::kABytes, j.ma, &st.full[stage], kb * g2::BK, a_row);
          tma_load_2d_2sm(smB + stage * g2::kBBytes, j.mb, &st.full[stage], kb * g2::BK, b_row);
          if (++stage == g2::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      });
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      // ================= MMA issuer (leader CTA only)
      constexpr uint32_t idesc = make_idesc_bf16(g2::BM, g2::BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      each_job([&](const TileJob& j) {
        mbar_wait(&st.tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + uint32_t(acc * g2::BN);
        for (int kb = 0; kb < j.k_blocks; ++kb) {
          mbar_wait(&st.full[stage], phase);
          tc_fence_after();
          const uint64_t adesc = make_sdesc_sw128(smem_u32(smA + stage * g2::kABytes));
          const uint64_t bdesc = make_sdesc_sw128(smem_u32(smB + stage * g2::kBBytes));
#pragma unroll
          for (int k = 0; k < g2::BK / 16; ++k)
            umma_bf16_2sm(d_tmem, adesc + uint64_t(2 * k), bdesc + uint64_t(2 * k), idesc, (kb | k) != 0 ? 1u : 0u);
          umma_commit_2sm_mc(&st.empty[stage], 0x3);
          if (++stage == g2::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_2sm_mc(&st.tfull[acc], 0x3);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      });
    }
  } else if (warp >= 4) {
    // ================= epilogue (both CTAs: own 128 rows of the pair tile)
    const int q = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    each_job([&](const TileJob& j) {
      const int row = j.m_row0 + int(rank) * 128 + q * 32 + lane;
      const bool valid = row < j.m_rows;
      __nv_bfloat16* rowp =
          j.aux ? aux.out + size_t(row) * aux.out_ld
                : out_row_ptr(out, size_t(st.g_orow[j.g] + row), out_ld, scatter_src, scatter_ptrs, valid);
      mbar_wait(&st.tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * g2::BN);
      epilogue_store(taddr, valid, rowp, j.n_blk, swiglu);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&st.tempty[acc], 0);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    });
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();  // both CTAs are done with TMEM and each other's barriers
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_2sm<gg::kTmemCols>(tmem_base);
  }
  if (peer_on(sync) && sync.total > 0) peer_arrive_and_raise(sync);
}

// ------------------------------------------------------------------ host side
namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn tmap_encoder() {
  static const EncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return EncodeFn(nullptr);
    return reinterpret_cast<EncodeFn>(p);
  }();
  return fn;
}

// 2-D map with a 128-byte inner box and SWIZZLE_128B (the UMMA K-major layout)
int encode_tmap_2d(CUtensorMap* map, CUtensorMapDataType dt, int esize, const void* ptr, uint64_t rows, uint64_t cols,
                   uint32_t box_rows) {
  const EncodeFn fn = tmap_encoder();
  if (!fn) return set_error(MP_E_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  const uint64_t inner = 128 / esize;
  if (cols % inner != 0)
    return set_error(MP_E_SHAPE, "tensor map inner dimension %llu not a multiple of %llu", (unsigned long long)cols,
                     (unsigned long long)inner);
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * esize};
  cuuint32_t box[2] = {uint32_t(inner), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(MP_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", int(r));
  return MP_OK;
}
}  // namespace

int encode_tmap_bf16_2d(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  return encode_tmap_2d(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ptr, rows, cols, box_rows);
}
int encode_tmap_u8_2d(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  return encode_tmap_2d(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, ptr, rows, cols, box_rows);
}

int launch_grouped_gemm(const CUtensorMap& tmA, const CUtensorMap& tmB, const GroupSpec& gs, int N, int K,
                        int b_slot_stride, int b_offset,
                        __nv_bfloat16* out, int out_ld, int swiglu, int grid, cudaStream_t stream, int pair,
                        const int32_t* scatter_src, __nv_bfloat16* const* scatter_ptrs, bool pdl,
                        const AuxProblem* aux, const PeerSync* sync) {
  const PeerSync ps = sync ? *sync : PeerSync();
  if (N % gg::BN != 0) return set_error(MP_E_SHAPE, "grouped GEMM N=%d not a multiple of %d", N, gg::BN);
  if (K % gg::BK != 0) return set_error(MP_E_SHAPE, "grouped GEMM K=%d not a multiple of %d", K, gg::BK);
  AuxProblem no_aux;
  if (aux && aux->m > 0) {
    if (aux->N % g2::BN != 0 || aux->K % g2::BK != 0 || aux->K <= 0)
      return set_error(MP_E_SHAPE, "grouped GEMM aux problem N=%d K=%d", aux->N, aux->K);
    if (swiglu && aux->out_ld < aux->N / 2) return set_error(MP_E_SHAPE, "aux out_ld %d", aux->out_ld);
  }
  const AuxProblem& ax = (aux && aux->m > 0) ? *aux : no_aux;
  if (pair) {  // the B map must have 128-row boxes (each CTA loads half of N)
    const int ra = ensure_max_dyn_smem(reinterpret_cast<const void*>(grouped_gemm_2sm_kernel), g2::kSmemBytes,
                                       "cudaFuncSetAttribute(grouped_gemm_2sm)");
    if (ra != MP_OK) return ra;
    if (grid <= 0) grid = kNumSMs;
    grid &= ~1;
    cudaError_t e = launch_pdl_if(pdl && pdl_enabled(), grouped_gemm_2sm_kernel, dim3(grid), dim3(gg::kThreads), g2::kSmemBytes, stream, tmA,
                               tmB, gs, N, K, b_slot_stride, b_offset, out, out_ld, swiglu, scatter_src,
                               scatter_ptrs, ax, ps);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error(e, "grouped_gemm_2sm_kernel launch");
    return MP_OK;
  }
  const int ra = ensure_max_dyn_smem(reinterpret_cast<const void*>(grouped_gemm_kernel), gg::kSmemBytes,
                                     "cudaFuncSetAttribute(grouped_gemm)");
  if (ra != MP_OK) return ra;
  if (grid <= 0) grid = kNumSMs;
  cudaError_t e = launch_pdl_if(pdl && pdl_enabled(), grouped_gemm_kernel, dim3(grid), dim3(gg::kThreads), gg::kSmemBytes, stream, tmA, tmB,
                             gs, N, K, b_slot_stride, b_offset, out, out_ld, swiglu, scatter_src, scatter_ptrs, ps,
                             ax);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "grouped_gemm_kernel launch");
  return MP_OK;
}

int grouped_gemm_ctas(int grid, int pair) {
  if (grid <= 0) grid = kNumSMs;
  return pair ? (grid & ~1) : grid;
}

}  // namespace mp
