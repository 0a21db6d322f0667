// Tensor-/expert-parallel communicator: one process (rank) per GPU, NCCL over
// NVLink 5 / NVSwitch for the plumbing, plus a symmetric peer-buffer window
// (CUDA IPC handles exchanged out of band) for the fused all-reduce+RMSNorm
// kernel that reads peers' partial sums directly over NVLink.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <vector>

#include "opflow_b200.h"

struct opf_comm {
  ncclComm_t nccl = nullptr;
  int world = 1;
  int rank = 0;
  int device = 0;
  // Peer window (optional): every rank's staging buffer mapped into this
  // process, plus a per-rank flag array used as a cross-GPU barrier.
  std::vector<void*> peer_buf;      // [world] device pointers (local one included)
  std::vector<uint32_t*> peer_flag; // [world]
  size_t peer_bytes = 0;
  void** d_peer_buf = nullptr;      // device copy of peer_buf
  uint32_t** d_peer_flag = nullptr;
  uint32_t epoch = 0;               // (unused: epochs live in device memory)
  void* window_base = nullptr;      // my symmetric window (staging | flags | epochs)
  size_t window_bytes = 0;
  std::vector<void*> opened;        // IPC-opened peer windows (closed on free)
  bool virtual_rank = false;        // one-device test rank (no NCCL)
  // Symmetric session arenas (expert-parallel ops write peers' tensors directly)
  void* arena_base = nullptr;       // my arena
  size_t arena_bytes = 0;
  std::vector<void*> peer_arena;    // [world] (mine included)
  std::vector<void*> opened_arenas; // IPC-opened peer arenas (closed on free)
};

namespace opflow {
void comm_window_alloc(opf_comm* c, size_t stage_bytes, void* ipc_handle_out);
void comm_window_open(opf_comm* c, const void* handles);
void comm_window_link_local(opf_comm* const* comms, int world);
uint32_t comm_window_error(const opf_comm* c);
uint32_t comm_push_calls(const opf_comm* c);
void comm_window_set_epochs(opf_comm* c, uint32_t v);
struct opf_view_fwd;
}  // namespace opflow
