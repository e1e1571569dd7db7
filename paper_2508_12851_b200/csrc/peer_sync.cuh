// Device side of PeerSync (mp_internal.h): the NVLink flag protocol folded into
// the layer kernels.  All waits are bounded (PeerSync::timeout_ns, 30 s): on timeout the
// missing ranks' bits are set in the error word -- in device memory for
// mp_layer_check and in mapped host memory, which the next mp_layer_forward
// reads before launching anything and turns into MP_E_PEER -- and the kernel
// proceeds (its outputs are garbage) instead of hanging the GPU.
#pragma once

#include "common.cuh"
#include "mp_internal.h"

namespace mp {

MP_DEV bool peer_on(const PeerSync& ps) { return ps.G > 1 && ps.flag_ptrs != nullptr; }

// One thread: spin until rank p's flag in this rank's window reached `epoch`, at most until
// t0 + ps.timeout_ns -- t0 is the start of the caller's whole wait, so a wait on several
// ranks is bounded once (below the 40 s mbarrier bound of the warps waiting behind it).  A
// rank this layer already marked lost is not waited for again.
MP_DEV void peer_wait_one(const PeerSync& ps, int p, uint32_t epoch, uint64_t t0) {
  const uint32_t* mine = ps.flag_ptrs[ps.rank];
  while (int32_t(ld_acquire_sys_u32(mine + p) - epoch) < 0) {
    if ((*reinterpret_cast<volatile uint32_t*>(ps.err) >> p) & 1u) break;
    if (globaltimer_ns() - t0 > ps.timeout_ns) {
      const uint32_t bits = atomicOr(ps.err, 1u << p) | (1u << p);
      if (ps.err_host != nullptr) st_release_sys_u32(ps.err_host, bits);
      break;
    }
    __nanosleep(64);
  }
}

// One thread: spin until every rank's flag in this rank's window reached `epoch`.
MP_DEV void peer_wait(const PeerSync& ps, uint32_t epoch) {
  const uint64_t t0 = globaltimer_ns();
  for (int p = 0; p < ps.G; ++p) peer_wait_one(ps, p, epoch, t0);
}

// One thread: raise `epoch` in every rank's window (flags[rank]).
MP_DEV void peer_raise(const PeerSync& ps, uint32_t epoch) {
  for (int p = 0; p < ps.G; ++p) st_release_sys_u32(ps.flag_ptrs[p] + ps.rank, epoch);
}

// Whole CTA, at kernel end: this CTA's peer stores are made visible system-wide
// and counted; the CTA that completes `ps.total` arrivals raises the next epoch
// and publishes it in state[0] for the kernels that follow in stream order.
MP_DEV void peer_arrive_and_raise(const PeerSync& ps) {
  // the CTA barrier orders every thread's stores before thread 0's system-scope
  // fence (cumulative), as in a cooperative grid barrier: one fence per CTA
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    if (atomicAdd(ps.ticket, 1u) == uint32_t(ps.total - 1)) {
      __threadfence_system();
      const uint32_t e = ps.state[0] + 1;
      peer_raise(ps, e);
      ps.state[0] = e;
      *ps.ticket = 0u;  // ready for the next forward (stream-ordered)
    }
  }
}

// Whole CTA, in a prologue: thread 0 waits for the epoch the preceding raising
// kernel published; the rest of the CTA is released by the barrier.
MP_DEV void peer_wait_cta(const PeerSync& ps) {
  if (threadIdx.x == 0) peer_wait(ps, ps.state[0]);
  __syncthreads();
}

}  // namespace mp
