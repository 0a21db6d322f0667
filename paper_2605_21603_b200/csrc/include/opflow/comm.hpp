// Tensor-/expert-parallel communicator: one process (rank) per GPU, NCCL over
// NVLink 5 / NVSwitch for the plumbing, plus a symmetric peer-buffer window
// (CUDA IPC handles exchanged out of band) for the fused all-reduce+RMSNorm
// kernel that reads peers' partial sums directly over NVLink.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <vector>

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
  uint32_t epoch = 0;               // barrier generation, bumped per fused call (host side)
};
