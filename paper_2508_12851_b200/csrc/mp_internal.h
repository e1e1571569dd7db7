// Internal (C++) declarations shared by the kernel translation units and the
// C-ABI layer in abi.cu.  Nothing here crosses the extern "C" boundary.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/moeplace_b200.h"

namespace mp {

// Kernel launch with programmatic stream serialization (PDL): the kernel may be
// scheduled while its predecessor drains; every kernel calls griddep_wait()
// before touching memory its predecessor produces.  Off by default; MP_PDL=1 enables.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_if(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                          cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args&&... args) {
  return launch_pdl_if(pdl_enabled(), kernel, grid, block, smem, stream, static_cast<Args&&>(args)...);
}

// NVLink synchronisation folded into the layer's own kernels (G > 1).  Each
// rank owns flags[G] in its window; "raise e" = st.release.sys e into
// flags[rank] of every peer, "wait e" = ld.acquire.sys until every flags[p]
// of this rank reached e.  The epoch lives in device memory (state[0]), so a
// captured graph replays correctly: a raising kernel sets state[0] = e after
// raising, and later kernels in stream order wait for state[0].
//   router (last CTA)   publishes its batch counts, raises A   (count exchange)
//   permute             waits A in its prologue; last CTA raises B (rows sent)
//   GEMM1 producers     wait B before the first routed tile (the fused shared-
//                       expert tiles go first and hide the wait)
//   GEMM2 (both chains) last CTA of all raises C (rows returned)
//   combine             waits C in its prologue
struct PeerSync {
  uint32_t* const* flag_ptrs = nullptr;  // [G] device array -> each rank's flags[G]
  int32_t* const* count_ptrs = nullptr;  // [2][8] count-table halves (router only)
  uint32_t* state = nullptr;             // [0] epoch, [1] forwards seen, [2] count parity
  uint32_t* err = nullptr;               // timeout bits (mp_layer_check)
  uint32_t* err_host = nullptr;          // the same bits in mapped pinned host memory: the next
                                         // mp_layer_forward reads them without a sync
  uint32_t* ticket = nullptr;            // arrival counter of a raising kernel
  int G = 1, rank = 0;
  int wait = 0;    // this launch waits for state[0] before touching peer-written rows
  int total = 0;   // this launch raises once `total` CTAs (across launches sharing ticket) arrived
  uint64_t timeout_ns = 30ull * 1000ull * 1000ull * 1000ull;  // bound of one wait (MP_PEER_TIMEOUT_MS)
};

// Error state (thread-local, read through mp_last_error).
int set_error(int code, const char* fmt, ...);
int set_cuda_error(cudaError_t e, const char* what);

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device attribute: raise it
// once per (kernel, current device) to at least `bytes` (thread-safe).
int ensure_max_dyn_smem(const void* kernel, size_t bytes, const char* what);

// Makes `device` current for the scope and restores the caller's device after.
struct DeviceGuard {
  int prev = -1;
  cudaError_t status = cudaSuccess;
  explicit DeviceGuard(int device) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != device) status = cudaSetDevice(device);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// ---- K1 router (tensor-core exact-integer logits; contract in router.cu)
int launch_router(const __nv_bfloat16* x, const uint8_t* packed, const float* bias, int T, int d, int E,
                  int has_gate, int k, int score_mode, int renorm, int32_t* idx, float* w, float* shared_gate,
                  uint32_t* hist, int32_t* blk_counts, int32_t* batch_counts, uint32_t* ticket,
                  int32_t* count_acc, cudaStream_t stream, const PeerSync* sync = nullptr);
int launch_router_logits(const float* logits, int ld, const float* bias, int T, int E, int k, int score_mode,
                         int renorm, int32_t* idx, float* w, uint32_t* hist, cudaStream_t stream);
int router_block_tokens();
__host__ __device__ int router_n_pad(int E_tot);
// Bytes of the packed router operand of E_tot weight rows ([3][N][d] limbs | R[N] | E[N]).
size_t router_packed_bytes(int E_tot, int d);
int launch_router_pack(const __nv_bfloat16* wg, int E_tot, int d, uint8_t* packed, cudaStream_t stream);
// K ranges (CTAs per 128-token tile) the router uses for T tokens.
int router_split(int T, int d);

// ---- K2 permute (+ dispatch through peer pointers)
int launch_permute(const __nv_bfloat16* x, const int32_t* idx, const int32_t* route, const int32_t* counts_all,
                   const uint32_t* parity, const int32_t* blk_counts, int32_t* const* src_ptrs, int rank, int G, int T, int d, int E, int k,
                   __nv_bfloat16* const* recv_ptrs, int32_t* pos_dst, int32_t* pos_row, cudaStream_t stream,
                   const PeerSync* sync = nullptr);

// ---- K3 grouped GEMM
// Where the GEMM takes its expert groups from (read in the kernel prologue).
struct GroupSpec {
  const int32_t* groups = nullptr;    // mode 0: explicit table [n][4] = {a_row, m, slot, out_row}
  const int32_t* n_groups = nullptr;  //         and its length (device)
  const int32_t* counts = nullptr;    // mode 1: derived -- exchanged counts C[G][E] (+ parity half
  const uint32_t* parity = nullptr;   //         *parity * G * E when non-null),
  const int32_t* route = nullptr;     //         route[G][E] and slot_of[E]: groups are the
  const int32_t* slot_of = nullptr;   //         experts routed to `rank`, ascending, rows packed
  int G = 1, E = 0, rank = 0;
  int single_m = 0;                   // mode 2: one group {0, single_m, slot 0, 0}
  int mode = 0;
  int m_lo = 0, m_hi = 1 << 30;       // mode 1: only groups with m_lo <= m < m_hi
  // mode 1, split plans: a big group's last partial CTA-pair tile (tail = m % tail_block rows,
  // 0 < tail <= tail_max) runs on the 1-CTA side chain as its own group, so the pair tile does
  // not pad it to tail_block rows.  tail_role 1: this launch takes the big groups less their
  // tails (m_lo = the threshold); 2: the small groups plus the tails (m_hi = the threshold)
  int tail_role = 0, tail_block = 256, tail_max = 0;
  int per_source = 1;                 // mode 1: a routed tile waits only for its rows' source ranks
};
// A second, dense problem fused into the same CTA-pair launch (the shared
// expert): its tiles are scheduled first, round-robin over the clusters, and
// the routed tiles fill each cluster up to an equal share of k-blocks.
struct alignas(64) AuxProblem {
  CUtensorMap tmA;                // A rows [m, K] (box 128 rows)
  CUtensorMap tmB;                // B rows [N, K] (box 128 rows)
  __nv_bfloat16* out = nullptr;   // [m, out_ld]
  int out_ld = 0;
  int m = 0, N = 0, K = 0;        // m == 0: no aux problem
};
int encode_tmap_bf16_2d(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows);
// 8-bit elements, 128-byte inner box, SWIZZLE_128B
int encode_tmap_u8_2d(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows);
int launch_grouped_gemm(const CUtensorMap& tmA, const CUtensorMap& tmB, const GroupSpec& gs, int N, int K,
                        int b_slot_stride, int b_offset,
                        __nv_bfloat16* out, int out_ld, int swiglu, int grid, cudaStream_t stream,
                        int pair = 0, const int32_t* scatter_src = nullptr,
                        __nv_bfloat16* const* scatter_ptrs = nullptr, bool pdl = true,
                        const AuxProblem* aux = nullptr, const PeerSync* sync = nullptr);
// CTAs a grouped-GEMM launch with this grid request runs (for PeerSync::total).
int grouped_gemm_ctas(int grid, int pair);

// ---- K5 combine (the expert outputs are already back in this GPU's return buffer)
int launch_combine(const __nv_bfloat16* ret /*[T][k][d]*/, const float* w, int T, int d, int k,
                   const __nv_bfloat16* shared_y, const float* shared_gate, __nv_bfloat16* out,
                   cudaStream_t stream, const PeerSync* sync = nullptr,
                   const __nv_bfloat16* const* bases = nullptr, const int32_t* pos_dst = nullptr,
                   const int32_t* pos_row = nullptr);

// ---- stand-in flag raises over NVLink peer memory (exchange.cu)
// Stand-ins when a raising kernel does not run (T == 0: no router / permute;
// no local slots: no GEMM2): publish zero counts + raise A, then raise B
// (`raise_count` = 2), or raise one epoch (`raise_count` = 1, counts unused).
int launch_peer_sync(const PeerSync& sync, int32_t* batch_counts, int E, int raise_count, cudaStream_t stream);


}  // namespace mp
