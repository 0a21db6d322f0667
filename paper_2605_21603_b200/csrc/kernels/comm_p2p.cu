// Fused all-reduce + residual add + RMSNorm over peer memory (TokenWeave's
// partial-overlap kernel, Fig. 7; north star: "a fused
// all-reduce+RMSNorm kernel that writes to peer buffers over NVSwitch").
//
// Every rank owns a symmetric window (one cudaMalloc, CUDA-IPC mapped into all
// peers): [staging rows | per-CTA signal flags | per-CTA local epochs].
// One launch per rank, same grid on every rank; CTA b owns rows b, b+G, ...:
//   1. copy my partial rows into my staging window;
//   2. barrier: bump my epoch for CTA b, store it into flag[b][me] of every
//      peer (st.release.sys over NVLink), spin until flag[b][p] >= epoch for
//      all p (ld.acquire.sys) — pairwise per CTA, no grid-wide sync;
//   3. reduce: sum the W partial rows by P2P loads, add the residual, write
//      x1, normalise and write h (one pass, rows in registers/smem);
//   4. barrier again ("done reading") so peers may overwrite their staging.
// Epochs live in device memory and advance inside the kernel, so the launch
// is CUDA-graph capturable and replays stay in lock-step across ranks.  The
// spin loops are bounded: on timeout the kernel raises an error flag instead
// of hanging the GPU.
#include <cuda_bf16.h>

#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "opflow/comm.hpp"
#include "opflow/device.hpp"
#include "opflow/p2p.cuh"

namespace opflow {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ bool cta_barrier(const PeerPtrs& pp, uint32_t* my_epoch, int world, int rank,
                                            uint32_t* err) {
  return slot_barrier(pp, my_epoch, blockIdx.x, world, rank, err);
}

__global__ void __launch_bounds__(kThreads) ar_add_rmsnorm_p2p_kernel(
    PeerPtrs pp, int world, int rank, const __nv_bfloat16* __restrict__ partial,
    __nv_bfloat16* __restrict__ my_stage, uint32_t* my_epoch, const __nv_bfloat16* __restrict__ resid,
    const __nv_bfloat16* __restrict__ gamma, __nv_bfloat16* __restrict__ x_out,
    __nv_bfloat16* __restrict__ y, int64_t rows, int64_t H, float eps, uint32_t* err) {
  extern __shared__ float rowbuf[];
  __shared__ float red[kThreads / 32];
  const int64_t n8 = H / 8;
  // 1. publish my partial rows
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x)
    for (int64_t c = threadIdx.x; c < n8; c += kThreads)
      reinterpret_cast<uint4*>(my_stage + r * H)[c] = reinterpret_cast<const uint4*>(partial + r * H)[c];
  // 2. all peers' rows for this CTA are in place
  if (!cta_barrier(pp, my_epoch, world, rank, err)) return;
  // 3. reduce + residual + norm
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    float ss = 0.0f;
    for (int64_t c = threadIdx.x; c < n8; c += kThreads) {
      float acc[8];
      {
        const uint4 u = reinterpret_cast<const uint4*>(resid + r * H)[c];
        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = __bfloat1622float2(h2[i]);
          acc[2 * i] = f.x;
          acc[2 * i + 1] = f.y;
        }
      }
      for (int p = 0; p < world; ++p) {
        const uint4 u = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(pp.buf[p]) + r * H)[c];
        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = __bfloat1622float2(h2[i]);
          acc[2 * i] += f.x;
          acc[2 * i + 1] += f.y;
        }
      }
      uint4 o;
      __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        o2[i] = __floats2bfloat162_rn(acc[2 * i], acc[2 * i + 1]);
        rowbuf[c * 8 + 2 * i] = acc[2 * i];
        rowbuf[c * 8 + 2 * i + 1] = acc[2 * i + 1];
        ss += acc[2 * i] * acc[2 * i] + acc[2 * i + 1] * acc[2 * i + 1];
      }
      reinterpret_cast<uint4*>(x_out + r * H)[c] = o;
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, s);
    if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = ss;
    __syncthreads();
    float tot = 0.0f;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) tot += red[w];
    const float inv = rsqrtf(tot / static_cast<float>(H) + eps);
    for (int64_t c = threadIdx.x; c < H; c += kThreads)
      y[r * H + c] = __float2bfloat16(rowbuf[c] * inv * __bfloat162float(gamma[c]));
    __syncthreads();
  }
  // 4. peers are done reading my staging rows
  cta_barrier(pp, my_epoch, world, rank, err);
}

// One-shot, push form ("writes to peer buffers"): every rank STORES its
// partial rows into slot `rank` of every peer's window ([world][rows][H]), so
// the NVLink traffic is posted writes; after the barrier each rank sums the
// world slots from its own HBM.  Same bytes as the pull form, no remote-read
// round trips.  Needs world x rows x H x 2 bytes of window.
template <bool NORM>
__global__ void __launch_bounds__(kThreads) ar_push_kernel(
    PeerPtrs pp, int world, int rank, const __nv_bfloat16* __restrict__ partial, uint32_t* my_epoch,
    const __nv_bfloat16* __restrict__ resid, const __nv_bfloat16* __restrict__ gamma,
    __nv_bfloat16* __restrict__ x_out, __nv_bfloat16* __restrict__ y, int64_t rows, int64_t H, float eps,
    uint32_t* err) {
  extern __shared__ float rowbuf[];
  __shared__ float red[kThreads / 32];
  const int64_t n8 = H / 8;
  // 1. push my partial rows into every rank's slot `rank`
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x)
    for (int64_t c = threadIdx.x; c < n8; c += kThreads) {
      const uint4 v = reinterpret_cast<const uint4*>(partial + r * H)[c];
      for (int p = 0; p < world; ++p)
        reinterpret_cast<uint4*>(const_cast<__nv_bfloat16*>(static_cast<const __nv_bfloat16*>(pp.buf[p])) +
                                 (static_cast<int64_t>(rank) * rows + r) * H)[c] = v;
    }
  __threadfence_system();
  if (!cta_barrier(pp, my_epoch, world, rank, err)) return;
  // 2. reduce my world slots (local HBM) [+ residual + norm]
  const __nv_bfloat16* mine = static_cast<const __nv_bfloat16*>(pp.buf[rank]);
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    float ss = 0.0f;
    for (int64_t c = threadIdx.x; c < n8; c += kThreads) {
      float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if constexpr (NORM) {
        const uint4 u = reinterpret_cast<const uint4*>(resid + r * H)[c];
        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(h2[e]);
          acc[2 * e] = f.x;
          acc[2 * e + 1] = f.y;
        }
      }
      for (int p = 0; p < world; ++p) {
        const uint4 u = reinterpret_cast<const uint4*>(mine + (static_cast<int64_t>(p) * rows + r) * H)[c];
        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(h2[e]);
          acc[2 * e] += f.x;
          acc[2 * e + 1] += f.y;
        }
      }
      uint4 o;
      __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        o2[e] = __floats2bfloat162_rn(acc[2 * e], acc[2 * e + 1]);
        if constexpr (NORM) {
          rowbuf[c * 8 + 2 * e] = acc[2 * e];
          rowbuf[c * 8 + 2 * e + 1] = acc[2 * e + 1];
          ss += acc[2 * e] * acc[2 * e] + acc[2 * e + 1] * acc[2 * e + 1];
        }
      }
      reinterpret_cast<uint4*>(x_out + r * H)[c] = o;
    }
    if constexpr (NORM) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = ss;
      __syncthreads();
      float tot = 0.0f;
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) tot += red[w];
      const float inv = rsqrtf(tot / static_cast<float>(H) + eps);
      for (int64_t c = threadIdx.x; c < H; c += kThreads)
        y[r * H + c] = __float2bfloat16(rowbuf[c] * inv * __bfloat162float(gamma[c]));
      __syncthreads();
    }
  }
  // 3. every rank has read its slots before anyone pushes the next call's rows
  cta_barrier(pp, my_epoch, world, rank, err);
}

// Two-shot variant (reduce-scatter -> residual add + RMSNorm -> all-gather)
// for large messages at W >= 4: rank q reduces and normalises only row block
// q (rows [q*B, (q+1)*B)), publishes x1 / h of its block in its window, and
// every rank then gathers all blocks.  NVLink bytes pulled per rank:
// 3 (W-1)/W x rows x H x 2 instead of the one-shot's (W-1) x rows x H x 2.
// Row r's in-block index i decides its CTA (i mod grid) in every phase and on
// every rank, so each CTA's pairwise per-slot barrier orders exactly the rows
// it reads next (no grid-wide barrier).  Window: [partials | x1 | h].
__global__ void __launch_bounds__(kThreads) ar2_add_rmsnorm_p2p_kernel(
    PeerPtrs pp, int world, int rank, const __nv_bfloat16* __restrict__ partial,
    __nv_bfloat16* __restrict__ my_stage, uint32_t* my_epoch, const __nv_bfloat16* __restrict__ resid,
    const __nv_bfloat16* __restrict__ gamma, __nv_bfloat16* __restrict__ x_out,
    __nv_bfloat16* __restrict__ y, int64_t rows, int64_t H, float eps, uint32_t* err) {
  extern __shared__ float rowbuf[];
  __shared__ float red[kThreads / 32];
  const int64_t n8 = H / 8;
  const int64_t blk = (rows + world - 1) / world;
  const int64_t plane = rows * H;  // elements per window plane
  // 1. publish my partial rows (every block)
  for (int64_t i = blockIdx.x; i < blk; i += gridDim.x)
    for (int q = 0; q < world; ++q) {
      const int64_t r = q * blk + i;
      if (r >= rows) continue;
      for (int64_t c = threadIdx.x; c < n8; c += kThreads)
        reinterpret_cast<uint4*>(my_stage + r * H)[c] = reinterpret_cast<const uint4*>(partial + r * H)[c];
    }
  if (!cta_barrier(pp, my_epoch, world, rank, err)) return;
  // 2. reduce-scatter + residual + norm for my block, results into my window
  for (int64_t i = blockIdx.x; i < blk; i += gridDim.x) {
    const int64_t r = rank * blk + i;
    if (r >= rows) continue;
    float ss = 0.0f;
    for (int64_t c = threadIdx.x; c < n8; c += kThreads) {
      float acc[8];
      {
        const uint4 u = reinterpret_cast<const uint4*>(resid + r * H)[c];
        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(h2[e]);
          acc[2 * e] = f.x;
          acc[2 * e + 1] = f.y;
        }
      }
      for (int p = 0; p < world; ++p) {
        const uint4 u = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(pp.buf[p]) + r * H)[c];
        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(h2[e]);
          acc[2 * e] += f.x;
          acc[2 * e + 1] += f.y;
        }
      }
      uint4 o;
      __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        o2[e] = __floats2bfloat162_rn(acc[2 * e], acc[2 * e + 1]);
        rowbuf[c * 8 + 2 * e] = acc[2 * e];
        rowbuf[c * 8 + 2 * e + 1] = acc[2 * e + 1];
        ss += acc[2 * e] * acc[2 * e] + acc[2 * e + 1] * acc[2 * e + 1];
      }
      reinterpret_cast<uint4*>(my_stage + plane + r * H)[c] = o;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = ss;
    __syncthreads();
    float tot = 0.0f;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) tot += red[w];
    const float inv = rsqrtf(tot / static_cast<float>(H) + eps);
    for (int64_t c = threadIdx.x; c < H; c += kThreads)
      my_stage[2 * plane + r * H + c] = __float2bfloat16(rowbuf[c] * inv * __bfloat162float(gamma[c]));
    __syncthreads();
  }
  if (!cta_barrier(pp, my_epoch, world, rank, err)) return;
  // 3. all-gather x1 / h of every block from its owner
  for (int64_t i = blockIdx.x; i < blk; i += gridDim.x)
    for (int q = 0; q < world; ++q) {
      const int64_t r = q * blk + i;
      if (r >= rows) continue;
      const __nv_bfloat16* src = static_cast<const __nv_bfloat16*>(pp.buf[q]);
      for (int64_t c = threadIdx.x; c < n8; c += kThreads) {
        reinterpret_cast<uint4*>(x_out + r * H)[c] = reinterpret_cast<const uint4*>(src + plane + r * H)[c];
        reinterpret_cast<uint4*>(y + r * H)[c] = reinterpret_cast<const uint4*>(src + 2 * plane + r * H)[c];
      }
    }
  // 4. peers are done reading my window
  cta_barrier(pp, my_epoch, world, rank, err);
}

// One-shot all-reduce (sum) over peer memory: same protocol, no norm.
__global__ void __launch_bounds__(kThreads) allreduce_p2p_kernel(
    PeerPtrs pp, int world, int rank, const __nv_bfloat16* __restrict__ partial,
    __nv_bfloat16* __restrict__ my_stage, uint32_t* my_epoch, __nv_bfloat16* __restrict__ out,
    int64_t rows, int64_t H, uint32_t* err) {
  const int64_t n8 = H / 8;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x)
    for (int64_t c = threadIdx.x; c < n8; c += kThreads)
      reinterpret_cast<uint4*>(my_stage + r * H)[c] = reinterpret_cast<const uint4*>(partial + r * H)[c];
  if (!cta_barrier(pp, my_epoch, world, rank, err)) return;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x)
    for (int64_t c = threadIdx.x; c < n8; c += kThreads) {
      float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int p = 0; p < world; ++p) {
        const uint4 u = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(pp.buf[p]) + r * H)[c];
        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = __bfloat1622float2(h2[i]);
          acc[2 * i] += f.x;
          acc[2 * i + 1] += f.y;
        }
      }
      uint4 o;
      __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int i = 0; i < 4; ++i) o2[i] = __floats2bfloat162_rn(acc[2 * i], acc[2 * i + 1]);
      reinterpret_cast<uint4*>(out + r * H)[c] = o;
    }
  cta_barrier(pp, my_epoch, world, rank, err);
}


// GEMM -> all-reduce -> residual add -> RMSNorm with the transfer inside the
// GEMM (gemm_ar_add_rmsnorm_push).  The row-parallel GEMM of every rank pushed
// its partial rows into the owner's window (rank q owns rows [q*blk,(q+1)*blk),
// slot p = rank p's partial) and counted each 32-row slab in the owner's
// cnt[slab]; this kernel, on every rank:
//   1. per slab of MY block: wait cnt == world x n_tiles, sum the world slots
//      (local HBM), add the residual, write x1 (local output + my window's x1
//      plane) and h = rmsnorm(x1) * g; reset cnt, publish pub[slab] = epoch;
//   2. per 8-row quarter of every OTHER owner's slab: wait that owner's
//      pub[slab] >= epoch, pull x1 over NVLink, normalise locally.
// NVLink bytes per rank: (W-1)/W of the partial pushed during the GEMM plus
// (W-1)/W of x1 pulled here — one all-reduce's worth, the first half hidden
// under the GEMM's math.  Between two push calls no extra barrier is needed
// (a rank pushes call k+1 only after its call-k kernel gathered from every
// owner, i.e. after every owner reset its counters and published); the final
// barrier keeps the window invariant shared by all collectives here: each
// ends after its last window access on every rank, so whichever collective
// comes next may write into any peer's window (e.g. a one-shot push into the
// region this call's x1 plane occupied).
__global__ void __launch_bounds__(kThreads) push_reduce_norm_kernel(
    PeerPtrs pp, int world, int rank, unsigned long long push_off, const __nv_bfloat16* __restrict__ resid,
    const __nv_bfloat16* __restrict__ gamma, __nv_bfloat16* __restrict__ x_out, __nv_bfloat16* __restrict__ y,
    int64_t rows, int64_t H, float eps, int n_tiles, uint32_t* my_epoch, uint32_t* err) {
  extern __shared__ float rowbuf[];
  __shared__ float red[kThreads / 32];
  __shared__ uint32_t ok;
  const int64_t n8 = H / 8;
  const int64_t blk = rows / world, slabs = blk / 32, plane = rows * H;
  char* mine = const_cast<char*>(static_cast<const char*>(pp.buf[rank]));
  uint32_t* cnt = reinterpret_cast<uint32_t*>(mine + push_off);
  uint32_t* pub = cnt + kMaxSlabs;
  const uint32_t epoch = *reinterpret_cast<volatile uint32_t*>(cnt + 2 * kMaxSlabs);
  const __nv_bfloat16* part = reinterpret_cast<const __nv_bfloat16*>(mine);
  __nv_bfloat16* x1w = reinterpret_cast<__nv_bfloat16*>(mine) + plane;
  // one row: v[c] = x1 (bf16-rounded) from `src8` (+ partial slots when reducing); y = rmsnorm(v) * g
  auto norm_row = [&](int64_t r) {
    float ss = 0.0f;
    for (int64_t c = threadIdx.x; c < n8; c += kThreads) {
      const float* v = rowbuf + c * 8;
#pragma unroll
      for (int e = 0; e < 8; ++e) ss += v[e] * v[e];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = ss;
    __syncthreads();
    float tot = 0.0f;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) tot += red[w];
    const float inv = rsqrtf(tot / static_cast<float>(H) + eps);
    for (int64_t c = threadIdx.x; c < n8; c += kThreads) {
      const uint4 gu = reinterpret_cast<const uint4*>(gamma)[c];
      const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gu);
      uint4 o;
      __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 gf = __bfloat1622float2(g2[e]);
        o2[e] = __floats2bfloat162_rn(rowbuf[c * 8 + 2 * e] * inv * gf.x, rowbuf[c * 8 + 2 * e + 1] * inv * gf.y);
      }
      reinterpret_cast<uint4*>(y + r * H)[c] = o;
    }
    __syncthreads();  // rowbuf / red reused by the next row
  };
  // 1. reduce my block
  for (int64_t s = blockIdx.x; s < slabs; s += gridDim.x) {
    if (threadIdx.x == 0) {
      ok = 1;
      const uint32_t need = static_cast<uint32_t>(world * n_tiles);
      if (!spin_until_reached(cnt + s, need, err)) ok = 0;
    }
    __syncthreads();
    if (!ok) return;
    for (int rr = 0; rr < 32; ++rr) {
      const int64_t lr = s * 32 + rr, r = rank * blk + lr;
      for (int64_t c = threadIdx.x; c < n8; c += kThreads) {
        float acc[8];
        const uint4 u = reinterpret_cast<const uint4*>(resid + r * H)[c];
        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(h2[e]);
          acc[2 * e] = f.x;
          acc[2 * e + 1] = f.y;
        }
        for (int p = 0; p < world; ++p) {
          const uint4 pu = reinterpret_cast<const uint4*>(part + (p * blk + lr) * H)[c];
          const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&pu);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(p2[e]);
            acc[2 * e] += f.x;
            acc[2 * e + 1] += f.y;
          }
        }
        uint4 o;
        __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          o2[e] = __floats2bfloat162_rn(acc[2 * e], acc[2 * e + 1]);
          const float2 f = __bfloat1622float2(o2[e]);
          rowbuf[c * 8 + 2 * e] = f.x;
          rowbuf[c * 8 + 2 * e + 1] = f.y;
        }
        reinterpret_cast<uint4*>(x_out + r * H)[c] = o;
        reinterpret_cast<uint4*>(x1w + r * H)[c] = o;
      }
      norm_row(r);
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
      cnt[s] = 0;  // every partial of this slab is consumed
      __threadfence_system();
      st_release_sys(pub + s, epoch);
    }
  }
  // 2. gather the other owners' x1 rows (8-row quarters of their slabs)
  const int64_t units = static_cast<int64_t>(world - 1) * slabs * 4;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int qi = static_cast<int>(u / (slabs * 4));
    const int q = qi < rank ? qi : qi + 1;
    const int64_t s = (u % (slabs * 4)) / 4, qu = u % 4;
    const char* theirs = static_cast<const char*>(pp.buf[q]);
    if (threadIdx.x == 0) {
      ok = 1;
      const uint32_t* qpub = reinterpret_cast<const uint32_t*>(theirs + push_off) + kMaxSlabs;
      if (!spin_until_reached(qpub + s, epoch, err)) ok = 0;
    }
    __syncthreads();
    if (!ok) return;
    const __nv_bfloat16* qx1 = reinterpret_cast<const __nv_bfloat16*>(theirs) + plane;
    for (int rr = 0; rr < 8; ++rr) {
      const int64_t r = q * blk + s * 32 + qu * 8 + rr;
      for (int64_t c = threadIdx.x; c < n8; c += kThreads) {
        const uint4 u4 = reinterpret_cast<const uint4*>(qx1 + r * H)[c];
        reinterpret_cast<uint4*>(x_out + r * H)[c] = u4;
        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u4);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(h2[e]);
          rowbuf[c * 8 + 2 * e] = f.x;
          rowbuf[c * 8 + 2 * e + 1] = f.y;
        }
      }
      norm_row(r);
    }
  }
  // 3. every window collective ends with a barrier after its last window
  //    access, so the next one (of any kind) may write into any peer's window
  cta_barrier(pp, my_epoch, world, rank, err);
}

}  // namespace

// ----------------------------------------------------------------- window API
void comm_window_alloc(opf_comm* c, size_t stage_bytes, void* ipc_handle_out) {
  size_t fo, eo;
  const size_t total = window_layout(stage_bytes, &fo, &eo);
  void* base = nullptr;
  OPF_CUDA(cudaMalloc(&base, total));
  OPF_CUDA(cudaMemset(base, 0, total));
  c->window_base = base;
  c->window_bytes = total;
  c->peer_bytes = stage_bytes;
  if (ipc_handle_out) {
    cudaIpcMemHandle_t h;
    OPF_CUDA(cudaIpcGetMemHandle(&h, base));
    std::memcpy(ipc_handle_out, &h, sizeof(h));
  }
}

void comm_window_open(opf_comm* c, const void* handles) {
  require(c->world <= kMaxWorld, Errc::ConfigError, "peer window supports world <= 8");
  size_t fo, eo;
  window_layout(c->peer_bytes, &fo, &eo);
  c->peer_buf.assign(c->world, nullptr);
  c->peer_flag.assign(c->world, nullptr);
  for (int p = 0; p < c->world; ++p) {
    void* base = c->window_base;
    if (p != c->rank) {
      cudaIpcMemHandle_t h;
      std::memcpy(&h, static_cast<const char*>(handles) + p * sizeof(cudaIpcMemHandle_t), sizeof(h));
      OPF_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
      c->opened.push_back(base);
    }
    c->peer_buf[p] = base;
    c->peer_flag[p] = reinterpret_cast<uint32_t*>(static_cast<char*>(base) + fo);
  }
}

// virtual ranks on ONE device (tests): windows are plain allocations wired
// together without IPC.
void comm_window_link_local(opf_comm* const* comms, int world) {
  size_t fo, eo;
  for (int r = 0; r < world; ++r) {
    opf_comm* c = comms[r];
    window_layout(c->peer_bytes, &fo, &eo);
    c->peer_buf.assign(world, nullptr);
    c->peer_flag.assign(world, nullptr);
    for (int p = 0; p < world; ++p) {
      c->peer_buf[p] = comms[p]->window_base;
      c->peer_flag[p] = reinterpret_cast<uint32_t*>(static_cast<char*>(comms[p]->window_base) + fo);
    }
  }
}

uint32_t comm_window_error(const opf_comm* c) {
  size_t fo, eo;
  window_layout(c->peer_bytes, &fo, &eo);
  uint32_t e = 0;
  OPF_CUDA(cudaMemcpy(&e, static_cast<char*>(c->window_base) + eo + sizeof(uint32_t) * kMaxCtas,
                      sizeof(e), cudaMemcpyDeviceToHost));
  return e;
}

void comm_window_set_epochs(opf_comm* c, uint32_t v) {
  size_t fo, eo;
  window_layout(c->peer_bytes, &fo, &eo);
  char* base = static_cast<char*>(c->window_base);
  const std::vector<uint32_t> flags(static_cast<size_t>(kMaxCtas) * kMaxWorld, v);
  OPF_CUDA(cudaMemcpy(base + fo, flags.data(), flags.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
  OPF_CUDA(cudaMemcpy(base + eo, flags.data(), kMaxCtas * sizeof(uint32_t), cudaMemcpyHostToDevice));
  // push protocol: publish epochs [kMaxSlabs] + the call epoch (arrival counters stay 0)
  char* push = base + window_push_off(c->peer_bytes);
  OPF_CUDA(cudaMemcpy(push + sizeof(uint32_t) * kMaxSlabs, flags.data(), (kMaxSlabs + 1) * sizeof(uint32_t),
                      cudaMemcpyHostToDevice));
}

uint32_t comm_push_calls(const opf_comm* c) {
  if (!c || !c->window_base) return 0;
  uint32_t e = 0;
  OPF_CUDA(cudaMemcpy(&e, static_cast<char*>(c->window_base) + window_push_off(c->peer_bytes) +
                              sizeof(uint32_t) * 2 * kMaxSlabs,
                      sizeof(e), cudaMemcpyDeviceToHost));
  return e;
}

bool ar_add_rmsnorm_p2p(const opf_comm* c, const opf_view& o, const opf_view& x, const opf_view& g,
                        opf_view& x_out, opf_view& y, int64_t rows, float eps, int max_ctas, int mode,
                        cudaStream_t s) {
  if (!c || c->peer_buf.empty() || o.dtype != OPF_BF16) return false;
  const int64_t H = view_row_elems(o);
  if (H % 8 || static_cast<size_t>(rows * H * 2) > c->peer_bytes || H * 4 > 48 * 1024) return false;
  size_t fo, eo;
  window_layout(c->peer_bytes, &fo, &eo);
  PeerPtrs pp{};
  for (int p = 0; p < c->world; ++p) {
    pp.buf[p] = c->peer_buf[p];
    pp.flags[p] = c->peer_flag[p];
  }
  char* base = static_cast<char*>(c->window_base);
  int grid = max_ctas > 0 ? max_ctas : num_sms();
  // two-shot for large messages at W >= 4 (3(W-1)/W vs (W-1) row-planes over
  // NVLink) when the window holds partials + x1 + h; OPF_AR=oneshot|twoshot forces
  static const int ar_mode = [] {
    const char* e = std::getenv("OPF_AR");
    if (e && std::string(e) == "oneshot") return 1;  // pull form
    if (e && std::string(e) == "twoshot") return 2;
    if (e && std::string(e) == "push") return 3;
    return 0;
  }();
  const bool fits2 = static_cast<size_t>(3 * rows * H * 2) <= c->peer_bytes;
  const bool fits_push = static_cast<size_t>(c->world) * rows * H * 2 <= c->peer_bytes;
  const int m = mode ? mode : ar_mode;
  const bool two = fits2 && (m == 2 || (m == 0 && c->world >= 4 && rows * H * 2 >= (1 << 20)));
  if (!two && fits_push && (m == 0 || m == 3)) {  // one-shot, push form (default when the window holds W planes)
    grid = static_cast<int>(std::min<int64_t>(std::min(grid, kBarrierSlot), rows));
    ar_push_kernel<true><<<std::max(grid, 1), kThreads, H * sizeof(float), s>>>(
        pp, c->world, c->rank, vptr<__nv_bfloat16>(o), reinterpret_cast<uint32_t*>(base + eo),
        vptr<__nv_bfloat16>(x), vptr<__nv_bfloat16>(g), vptr<__nv_bfloat16>(x_out), vptr<__nv_bfloat16>(y), rows,
        H, eps, reinterpret_cast<uint32_t*>(base + eo + sizeof(uint32_t) * kMaxCtas));
    return true;
  }
  if (two) {
    const int64_t blk = (rows + c->world - 1) / c->world;
    grid = static_cast<int>(std::min<int64_t>(std::min(grid, kBarrierSlot), blk));
    ar2_add_rmsnorm_p2p_kernel<<<std::max(grid, 1), kThreads, H * sizeof(float), s>>>(
        pp, c->world, c->rank, vptr<__nv_bfloat16>(o), reinterpret_cast<__nv_bfloat16*>(base),
        reinterpret_cast<uint32_t*>(base + eo), vptr<__nv_bfloat16>(x), vptr<__nv_bfloat16>(g),
        vptr<__nv_bfloat16>(x_out), vptr<__nv_bfloat16>(y), rows, H, eps,
        reinterpret_cast<uint32_t*>(base + eo + sizeof(uint32_t) * kMaxCtas));
    return true;
  }
  grid = static_cast<int>(std::min<int64_t>(std::min(grid, kBarrierSlot), rows));
  ar_add_rmsnorm_p2p_kernel<<<std::max(grid, 1), kThreads, H * sizeof(float), s>>>(
      pp, c->world, c->rank, vptr<__nv_bfloat16>(o), reinterpret_cast<__nv_bfloat16*>(base),
      reinterpret_cast<uint32_t*>(base + eo), vptr<__nv_bfloat16>(x), vptr<__nv_bfloat16>(g),
      vptr<__nv_bfloat16>(x_out), vptr<__nv_bfloat16>(y), rows, H, eps,
      reinterpret_cast<uint32_t*>(base + eo + sizeof(uint32_t) * kMaxCtas));
  return true;
}

bool allreduce_p2p(const opf_comm* c, const opf_view& in, opf_view& out, int64_t rows, int max_ctas,
                   cudaStream_t s) {
  if (!c || c->peer_buf.empty() || in.dtype != OPF_BF16) return false;
  const int64_t H = view_row_elems(in);
  if (H % 8 || static_cast<size_t>(rows * H * 2) > c->peer_bytes) return false;
  size_t fo, eo;
  window_layout(c->peer_bytes, &fo, &eo);
  PeerPtrs pp{};
  for (int p = 0; p < c->world; ++p) {
    pp.buf[p] = c->peer_buf[p];
    pp.flags[p] = c->peer_flag[p];
  }
  char* base = static_cast<char*>(c->window_base);
  int grid = max_ctas > 0 ? max_ctas : num_sms();
  grid = static_cast<int>(std::min<int64_t>(std::min(grid, kBarrierSlot), rows));
  static const bool pull = [] {
    const char* e = std::getenv("OPF_AR");
    return e && std::string(e) == "oneshot";
  }();
  if (!pull && static_cast<size_t>(c->world) * rows * H * 2 <= c->peer_bytes) {  // push form
    ar_push_kernel<false><<<std::max(grid, 1), kThreads, 0, s>>>(
        pp, c->world, c->rank, vptr<__nv_bfloat16>(in), reinterpret_cast<uint32_t*>(base + eo), nullptr, nullptr,
        vptr<__nv_bfloat16>(out), nullptr, rows, H, 0.0f,
        reinterpret_cast<uint32_t*>(base + eo + sizeof(uint32_t) * kMaxCtas));
    return true;
  }
  allreduce_p2p_kernel<<<std::max(grid, 1), kThreads, 0, s>>>(
      pp, c->world, c->rank, vptr<__nv_bfloat16>(in), reinterpret_cast<__nv_bfloat16*>(base),
      reinterpret_cast<uint32_t*>(base + eo), vptr<__nv_bfloat16>(out), rows, H,
      reinterpret_cast<uint32_t*>(base + eo + sizeof(uint32_t) * kMaxCtas));
  return true;
}

bool gemm_ar_add_rmsnorm_push(const opf_comm* c, const GemmArgs& g, const opf_view& x, const opf_view& gam,
                              opf_view& x_out, opf_view& y, float eps, cudaStream_t s) {
  if (!c || c->peer_buf.empty() || c->world < 2) return false;
  const int W = c->world;
  const int64_t rows = g.m, H = g.n;
  if (rows % (32 * W) || H % 256 || rows <= 128 || H * 4 > 48 * 1024 || x.dtype != OPF_BF16) return false;
  if (static_cast<size_t>(2 * rows * H * 2) > c->peer_bytes) return false;  // partials + x1 planes
  const int64_t blk = rows / W;
  if (blk / 32 > kMaxSlabs) return false;
  const size_t push_off = window_push_off(c->peer_bytes);
  PushArgs p{};
  PeerPtrs pp{};
  for (int q = 0; q < W; ++q) {
    char* base = static_cast<char*>(c->peer_buf[q]);
    p.dst[q] = base + static_cast<size_t>(c->rank) * blk * H * 2;
    p.cnt[q] = reinterpret_cast<uint32_t*>(base + push_off);
    pp.buf[q] = base;
    pp.flags[q] = c->peer_flag[q];
  }
  p.epoch = reinterpret_cast<uint32_t*>(static_cast<char*>(c->window_base) + push_off) + 2 * kMaxSlabs;
  p.blk = blk;
  p.world = W;
  gemm_bf16_push(g, p, s);
  size_t fo, eo;
  window_layout(c->peer_bytes, &fo, &eo);
  const int64_t slabs = blk / 32;
  int grid = g.max_ctas > 0 ? g.max_ctas : num_sms();
  grid = static_cast<int>(std::min<int64_t>(std::min(grid, kBarrierSlot),
                                             std::max<int64_t>(slabs, (W - 1) * slabs * 4)));
  push_reduce_norm_kernel<<<std::max(grid, 1), kThreads, H * sizeof(float), s>>>(
      pp, W, c->rank, static_cast<unsigned long long>(push_off), vptr<__nv_bfloat16>(x), vptr<__nv_bfloat16>(gam),
      vptr<__nv_bfloat16>(x_out), vptr<__nv_bfloat16>(y), rows, H, eps, static_cast<int>(H / 256),
      reinterpret_cast<uint32_t*>(static_cast<char*>(c->window_base) + eo),
      reinterpret_cast<uint32_t*>(static_cast<char*>(c->window_base) + eo + sizeof(uint32_t) * kMaxCtas));
  return true;
}

}  // namespace opflow
