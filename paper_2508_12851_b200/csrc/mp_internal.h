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
  cfg.numAttrs = (pdl && pdl_enabled()) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args&&... args) {
  return launch_pdl_if(true, kernel, grid, block, smem, stream, static_cast<Args&&>(args)...);
}

// Error state (thread-local, read through mp_last_error).
int set_error(int code, const char* fmt, ...);
int set_cuda_error(cudaError_t e, const char* what);

// ---- K1 router
int launch_router(const __nv_bfloat16* x, const __nv_bfloat16* wg_packed, const float* bias, int T, int d, int E,
                  int has_gate, int k, int score_mode, int renorm, int32_t* idx, float* w, float* shared_gate,
                  uint32_t* hist, int32_t* blk_counts, int32_t* batch_counts, uint32_t* ticket,
                  int32_t* blk_prefix, cudaStream_t stream);
int router_block_tokens();
__host__ __device__ int router_e_pad(int E_tot);
int launch_router_pack(const __nv_bfloat16* wg, int E_tot, int d, __nv_bfloat16* packed, cudaStream_t stream);

// ---- K2 permute (+ dispatch through peer pointers)
int launch_permute(const __nv_bfloat16* x, const int32_t* idx, const int32_t* route, const int32_t* counts_all,
                   const uint32_t* parity, const int32_t* blk_prefix, int32_t* const* src_ptrs, int rank, int G, int T, int d, int E, int k,
                   __nv_bfloat16* const* recv_ptrs, int32_t* pos_dst, int32_t* pos_row, cudaStream_t stream);

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
  int order = 0;                      // tile order: 0 group-major, 1 n-block-major
  int m_lo = 0, m_hi = 1 << 30;       // mode 1: only groups with m_lo <= m < m_hi
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
  int sched = 0;                  // tile schedule (grouped_swiglu.cu: make_sched)
};
int encode_tmap_bf16_2d(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows);
int launch_grouped_gemm(const CUtensorMap& tmA, const CUtensorMap& tmB, const GroupSpec& gs, int N, int K,
                        int b_slot_stride, int b_offset,
                        __nv_bfloat16* out, int out_ld, int swiglu, int grid, cudaStream_t stream,
                        int pair = 0, const int32_t* scatter_src = nullptr,
                        __nv_bfloat16* const* scatter_ptrs = nullptr, bool pdl = true,
                        const AuxProblem* aux = nullptr);

// ---- K5 combine (the expert outputs are already back in this GPU's return buffer)
int launch_combine(const __nv_bfloat16* ret /*[T][k][d]*/, const float* w, int T, int d, int k,
                   const __nv_bfloat16* shared_y, const float* shared_gate, __nv_bfloat16* out,
                   cudaStream_t stream);

// ---- exchange / barrier over NVLink peer memory
int launch_publish_barrier(uint32_t* const* flag_ptrs /*[G] device array, each -> flags[G]*/,
                           int32_t* const* count_ptrs /*[2][8] device array -> table halves, or null*/,
                           const int32_t* my_counts, int E, int G, int rank, uint32_t* state /*[3] device*/,
                           uint32_t* error_word, cudaStream_t stream);

}  // namespace mp
