// Peer-window device helpers shared by the peer-memory collectives
// (comm_p2p.cu: all-reduce, fused all-reduce+RMSNorm; moe_ep.cu: expert-
// parallel dispatch / combine).
//
// Window of every rank (one cudaMalloc, CUDA-IPC mapped into all peers):
//   [staging bytes | flags [kMaxCtas][kMaxWorld] u32 | epochs [kMaxCtas] u32 | err u32]
// A barrier on slot b: bump my epoch[b] (device memory, so replays stay in
// lock-step), st.release.sys it into flag[b][me] of every peer, spin (bounded)
// until my flag[b][p] >= epoch for all p.  Collectives are serialised by the
// engine's comm chain, so one slot sequence is shared by all of them; slot
// kBarrierSlot is reserved for whole-rank (1-CTA) barriers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "opflow/comm.hpp"

namespace opflow {

constexpr int kMaxWorld = 8;
constexpr int kMaxCtas = 1024;
constexpr int kBarrierSlot = kMaxCtas - 1;  // rank-wide barriers (EP dispatch / combine)
// spin bound: a barrier that waits longer than this raises the window's error
// flag instead of hanging the GPU (generous: ranks sharing one GPU time-slice)
constexpr uint64_t kSpinTimeoutNs = 10ull * 1000 * 1000 * 1000;

struct PeerPtrs {
  const void* buf[kMaxWorld];  // staging region of each rank
  uint32_t* flags[kMaxWorld];  // flag array of each rank [kMaxCtas][kMaxWorld]
};

// GEMM -> all-reduce push protocol (gemm_ar_push: the row-parallel GEMM's
// epilogue stores each 32-row slab of its partial straight into the owner
// rank's window): per-slab arrival counters, per-slab publish epochs and one
// call epoch, after the error flag.
constexpr int kMaxSlabs = 4096;  // 32-row slabs per owner block (blk <= 131072 rows)

inline size_t window_layout(size_t stage_bytes, size_t* flags_off, size_t* epoch_off) {
  const size_t s = (stage_bytes + 255) / 256 * 256;
  *flags_off = s;
  *epoch_off = s + sizeof(uint32_t) * kMaxCtas * kMaxWorld;
  return *epoch_off + sizeof(uint32_t) * kMaxCtas + sizeof(uint32_t) /*error flag*/ +
         sizeof(uint32_t) * (2 * kMaxSlabs + 1) /*push counters, publish epochs, call epoch*/;
}
// offset of the push area: [cnt kMaxSlabs | pub kMaxSlabs | call epoch]
inline size_t window_push_off(size_t stage_bytes) {
  size_t fo, eo;
  window_layout(stage_bytes, &fo, &eo);
  return eo + sizeof(uint32_t) * kMaxCtas + sizeof(uint32_t);
}

// Host: peer pointers + my epochs / error flag of a windowed communicator.
struct WindowView {
  PeerPtrs pp{};
  char* base = nullptr;
  uint32_t* epochs = nullptr;
  uint32_t* err = nullptr;
  size_t stage_bytes = 0;
};
inline bool window_view(const opf_comm* c, WindowView* w) {
  if (!c || c->peer_buf.empty()) return false;
  size_t fo, eo;
  window_layout(c->peer_bytes, &fo, &eo);
  for (int p = 0; p < c->world; ++p) {
    w->pp.buf[p] = c->peer_buf[p];
    w->pp.flags[p] = c->peer_flag[p];
  }
  w->base = static_cast<char*>(c->window_base);
  w->epochs = reinterpret_cast<uint32_t*>(w->base + eo);
  w->err = reinterpret_cast<uint32_t*>(w->base + eo + sizeof(uint32_t) * kMaxCtas);
  w->stage_bytes = c->peer_bytes;
  return true;
}

#ifdef __CUDACC__
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Spin until *p reaches `target` in wrap-safe serial-number order (epochs and
// counters are u32 that grow forever in device memory).  Returns false, after
// setting *err, when kSpinTimeoutNs passes first.
__device__ __forceinline__ bool spin_until_reached(const uint32_t* p, uint32_t target, uint32_t* err) {
  if (static_cast<int32_t>(ld_acquire_sys(p) - target) >= 0) return true;
  const uint64_t t0 = global_ns();
  uint32_t n = 0;
  while (static_cast<int32_t>(ld_acquire_sys(p) - target) < 0) {
    if ((++n & 255u) == 0 && global_ns() - t0 > kSpinTimeoutNs) {
      atomicExch(err, 1u);
      return false;
    }
  }
  return true;
}

// Barrier of CTA slot `slot` across all ranks; called by every thread of the CTA.
__device__ __forceinline__ bool slot_barrier(const PeerPtrs& pp, uint32_t* my_epoch, int slot, int world, int rank,
                                             uint32_t* err) {
  __syncthreads();
  __shared__ uint32_t ok;
  if (threadIdx.x == 0) {
    ok = 1;
    if (*reinterpret_cast<volatile uint32_t*>(err)) {  // poisoned by an earlier timeout: fail fast
      ok = 0;
    }
  }
  __syncthreads();
  if (!ok) return false;
  if (threadIdx.x == 0) {
    const uint32_t e = ++my_epoch[slot];
    __threadfence_system();
    for (int p = 0; p < world; ++p) st_release_sys(pp.flags[p] + slot * kMaxWorld + rank, e);
    for (int p = 0; p < world; ++p)
      if (!spin_until_reached(pp.flags[rank] + slot * kMaxWorld + p, e, err)) {
        ok = 0;
        break;
      }
  }
  __syncthreads();
  return ok != 0;
}
#endif

}  // namespace opflow
