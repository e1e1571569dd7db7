// Count exchange + cross-GPU barrier over NVLink peer memory.
//
// Replaces the reference's analytic round trip `comm_time = lat + 2*payload/bw`
// (reference pkg/src/moeplace/cost.py:139-149) for the control part of the
// exchange: each rank writes its per-expert batch counts C[rank][:] into every
// peer's count table and then raises its epoch flag there; a rank leaves the
// barrier once all G flags in its own window carry the current epoch.  The data
// part (token rows out, expert outputs back) moves inside the permute and
// combine kernels as direct peer stores / loads, so no NCCL call sits on the
// layer's critical path.
//
// Safety: the spin is bounded (kBarrierTimeoutNs); on timeout the kernel sets
// an error word the host checks, instead of hanging the GPU.
#include "common.cuh"
#include "mp_internal.h"

namespace mp {

constexpr uint64_t kBarrierTimeoutNs = 30ull * 1000ull * 1000ull * 1000ull;

// Barrier state lives on the device (graph-replayable): state[0] = barrier
// epoch, state[1] = forwards seen by the count exchange, state[2] = count-table
// parity of the current forward (read by the permute kernel and the GEMM
// prologue).  Stream order serialises the single-CTA barrier kernels.
__global__ void __launch_bounds__(256)
    publish_barrier_kernel(uint32_t* const* __restrict__ flag_ptrs, int32_t* const* __restrict__ count_ptrs,
                           const int32_t* __restrict__ my_counts, int E, int G, int rank,
                           uint32_t* __restrict__ state, uint32_t* __restrict__ error_word) {
  __shared__ uint32_t s_epoch, s_par, s_fwd;
  const int tid = threadIdx.x;
  griddep_launch_dependents();
  griddep_wait();
  if (tid == 0) {
    s_epoch = state[0] + 1;
    s_fwd = state[1];
    s_par = s_fwd & 1u;
  }
  // everything this stream wrote before (permute rows, expert outputs) must be
  // visible system-wide before the flag goes up
  __threadfence_system();
  __syncthreads();
  const uint32_t epoch = s_epoch;
  if (count_ptrs != nullptr) {
    int32_t* const* half = count_ptrs + 8 * s_par;  // [parity][peer]
    for (int i = tid; i < G * E; i += blockDim.x) {
      const int p = i / E, e = i - p * E;
      half[p][rank * E + e] = my_counts[e];
    }
  }
  __threadfence_system();
  __syncthreads();
  if (tid < G) st_release_sys_u32(flag_ptrs[tid] + rank, epoch);
  if (tid < G) {
    const uint32_t* mine = flag_ptrs[rank] + tid;
    const uint64_t t0 = globaltimer_ns();
    while (int32_t(ld_acquire_sys_u32(mine) - epoch) < 0) {
      if (globaltimer_ns() - t0 > kBarrierTimeoutNs) {
        atomicOr(error_word, 1u << tid);
        break;
      }
      __nanosleep(32);
    }
  }
  __syncthreads();
  if (tid == 0) {
    state[0] = epoch;
    if (count_ptrs != nullptr) {
      state[1] = s_fwd + 1;
      state[2] = s_par;
    }
  }
}

int launch_publish_barrier(uint32_t* const* flag_ptrs, int32_t* const* count_ptrs, const int32_t* my_counts, int E,
                           int G, int rank, uint32_t* state, uint32_t* error_word, cudaStream_t stream) {
  cudaError_t e = launch_pdl(publish_barrier_kernel, dim3(1), dim3(256), 0, stream, flag_ptrs, count_ptrs, my_counts, E,
                             G, rank, state, error_word);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? MP_OK : set_cuda_error(e, "publish_barrier_kernel launch");
}

}  // namespace mp
