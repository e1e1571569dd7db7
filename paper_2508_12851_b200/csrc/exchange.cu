// Stand-in raise kernels for the NVLink flag protocol (PeerSync, mp_internal.h).
//
// Replaces the reference's analytic round trip `comm_time = lat + 2*payload/bw`
// (reference pkg/src/moeplace/cost.py:139-149) for the control part of the
// exchange.  In a normal forward the flags are raised and awaited inside the
// layer kernels themselves (router tail: counts + epoch A; permute tail: B;
// GEMM2 tail: C) -- there is no barrier kernel on the critical path.  The
// kernel here runs only when the raising kernel does not: an origin with T = 0
// tokens launches no router / permute (zero counts are published, A is raised
// and awaited -- the GEMM prologues read the count table -- then B is raised),
// and a GPU without expert slots launches no GEMM2 (C is raised).
#include "common.cuh"
#include "mp_internal.h"
#include "peer_sync.cuh"

namespace mp {

__global__ void __launch_bounds__(256)
    peer_sync_kernel(const PeerSync ps, int32_t* __restrict__ batch_counts, int E, int raise_count) {
  const int tid = threadIdx.x;
  griddep_launch_dependents();
  griddep_wait();
  __shared__ uint32_t s_fwd;
  if (raise_count == 2) {
    if (tid == 0) s_fwd = ps.state[1];
    for (int e = tid; e < E; e += blockDim.x) batch_counts[e] = 0;
    __syncthreads();
    int32_t* const* half = ps.count_ptrs + 8 * (s_fwd & 1u);
    for (int i = tid; i < ps.G * E; i += blockDim.x) {
      const int p = i / E, e = i - (i / E) * E;
      half[p][ps.rank * E + e] = 0;
    }
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence_system();
    uint32_t ep = ps.state[0];
    peer_raise(ps, ++ep);
    if (raise_count == 2) {
      // the GEMM prologues that follow read the count table: every rank's counts
      // must have landed (A) before B is raised and this kernel completes
      peer_wait(ps, ep);
      peer_raise(ps, ++ep);
    }
    ps.state[0] = ep;
    if (raise_count == 2) {
      ps.state[1] = s_fwd + 1;
      ps.state[2] = s_fwd & 1u;
    }
  }
}

int launch_peer_sync(const PeerSync& sync, int32_t* batch_counts, int E, int raise_count, cudaStream_t stream) {
  if (raise_count < 1 || raise_count > 2) return set_error(MP_E_ARG, "peer sync: raise_count %d", raise_count);
  cudaError_t e = launch_pdl(peer_sync_kernel, dim3(1), dim3(256), 0, stream, sync, batch_counts, E, raise_count);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? MP_OK : set_cuda_error(e, "peer_sync_kernel launch");
}

}  // namespace mp
