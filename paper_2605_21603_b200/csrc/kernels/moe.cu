// Mixture-of-experts operators (Qwen3-30B-A3B-shaped MoE layer).
//
// Graph-level decomposition (one Custom op each, so strategies can place the
// dispatch/combine — the expert-parallel all-to-all sites — on the network lane
// and overlap them with the other micro-batch's expert GEMMs, DBO-style):
//
//   logits [T,E] = MatMul(x_norm, W_router)                  (tcgen05 GEMM)
//   moe_topk     logits -> ids [T,k] (i64), w [T,k] (f32)     top-k by (value desc,
//                index asc); w = softmax over the k selected logits (renorm=1, Qwen3
//                norm_topk_prob) or the full-softmax probabilities (renorm=0)
//   moe_dispatch x [T,H], ids -> xd [T, k*H] (= [T*k, H] rows sorted by expert,
//                stable in (token, j) order), slot [T,k] (i64 row of (t,j) in xd)
//   moe_gate_up  xd, ids, W_gu [E,H,2I] -> hd [T, k*I]       grouped tcgen05 GEMM,
//                SiLU-mul fused in the epilogue
//   moe_down     hd, ids, W_d [E,I,H] -> yd [T, k*H]         grouped tcgen05 GEMM
//   moe_combine  yd, slot, w -> y [T,H] = sum_j w[t,j] * yd[slot[t,j]]  (j ascending)
//
// Routing is a stable counting sort over the T*k (token, j) slots: per-chunk
// expert histograms, then one CTA per chunk derives its bases from the whole
// count matrix and ranks equal experts (per-warp counts + __match_any_sync) so
// positions follow slot order — bit-identical to a stable argsort (the
// oracle's restatement).  Ids outside [0,E) are dropped
// (slot = -1, no contribution).  All index work is exact; the grouped GEMM's
// tile table (row0, row_end, expert per 128-row tile) is rebuilt on the device
// by each GEMM op from `ids`, so every launch is graph-capturable (no host sync).
#include <cuda_bf16.h>

#include <algorithm>
#include <cfloat>
#include <mutex>

#include "opflow/device.hpp"
#include "opflow/p2p.cuh"

namespace opflow {

namespace {

constexpr int kMaxE = 1024;

__device__ __forceinline__ bool valid_id(int64_t e, int E) { return e >= 0 && e < E; }

// ---------------------------------------------------------------- top-k
template <typename T>
__device__ __forceinline__ float ldf(const T* p);
template <>
__device__ __forceinline__ float ldf<float>(const float* p) { return *p; }
template <>
__device__ __forceinline__ float ldf<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }

// One warp per token; lane l holds logits l, l+32, ...  k rounds of a warp
// argmax with (value desc, index asc) ordering.
template <typename T, int PER>
__global__ void __launch_bounds__(256) topk_kernel(const T* __restrict__ logits, int64_t* __restrict__ ids,
                                                   float* __restrict__ w, int64_t rows, int E, int k,
                                                   int renorm) {
  pdl_wait();
  pdl_trigger();
  const int64_t t = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (t >= rows) return;
  float v[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int e = lane + 32 * i;
    v[i] = e < E ? ldf<T>(logits + t * E + e) : -FLT_MAX;
  }
  float vmax = -FLT_MAX;
  float sel[32];
  int64_t* out_ids = ids + t * k;
  for (int j = 0; j < k; ++j) {
    float bv = -FLT_MAX;
    int bi = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int e = lane + 32 * i;
      if (e < E && (v[i] > bv || (v[i] == bv && e < bi))) {
        bv = v[i];
        bi = e;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
#pragma unroll
    for (int i = 0; i < PER; ++i)  // remove the winner (owner lane)
      if (lane + 32 * i == bi) v[i] = -INFINITY;
    if (j == 0) vmax = bv;
    sel[j & 31] = bv;
    if (lane == 0) out_ids[j] = bi;
  }
  float denom = 0.0f;
  if (renorm) {
    for (int j = 0; j < k; ++j) denom += __expf(sel[j & 31] - vmax);
  } else {  // full softmax over all E logits (restore the removed values first)
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int e = lane + 32 * i;
      if (e < E) denom += __expf(ldf<T>(logits + t * E + e) - vmax);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) denom += __shfl_xor_sync(0xffffffffu, denom, o);
  }
  if (lane == 0)
    for (int j = 0; j < k; ++j) w[t * k + j] = __expf(sel[j & 31] - vmax) / denom;
}

// ---------------------------------------------------------------- routing
// Stable counting sort of the n = T*k slots by expert in THREE launches:
//   route_hist_kernel   C CTAs, one chunk of `chunk` slots each -> cnt[c][e]
//   route_assign_kernel C CTAs: every CTA reduces the whole C x E count
//                       matrix (all 1024 threads, strided over chunks) to
//                       its own bases (expert offsets + the counts of earlier
//                       chunks) — no separate scan launch — then ranks its slots round
//                       by round (1024 per round: per-warp expert counts,
//                       a scan over the 32 warps, __match_any_sync inside a warp)
//   gather_tokens_kernel one warp per token: the row is read once and
//                       written to its k expert-sorted rows
// The grouped GEMMs only need the tile table: route_hist + route_tiles_kernel.
// C <= 64 chunks (C * E <= 16384 counts).
constexpr int kRouteThreads = 1024;

int64_t route_chunk(int64_t n, int E) {
  const int64_t cmax = std::max<int64_t>(1, std::min<int64_t>(64, 16384 / E));
  const int64_t per = (n + cmax - 1) / cmax;
  return std::max<int64_t>(kRouteThreads, (per + kRouteThreads - 1) / kRouteThreads * kRouteThreads);
}
int64_t route_chunks(int64_t n, int E) { return n > 0 ? (n + route_chunk(n, E) - 1) / route_chunk(n, E) : 0; }

__global__ void __launch_bounds__(kRouteThreads) route_hist_kernel(const int64_t* __restrict__ ids, int64_t n, int E,
                                                                   int64_t chunk, int32_t* __restrict__ cnt) {
  pdl_wait();
  extern __shared__ int32_t h[];
  for (int e = threadIdx.x; e < E; e += blockDim.x) h[e] = 0;
  __syncthreads();
  const int64_t s0 = static_cast<int64_t>(blockIdx.x) * chunk;
  const int64_t s1 = s0 + chunk < n ? s0 + chunk : n;
  for (int64_t s = s0 + threadIdx.x; s < s1; s += blockDim.x) {
    const int64_t e = ids[s];
    if (valid_id(e, E)) atomicAdd(&h[e], 1);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) cnt[static_cast<int64_t>(blockIdx.x) * E + e] = h[e];
  pdl_trigger();
}

// exclusive block scan of one value per thread (1024 threads); returns the
// exclusive prefix, *total = the sum over the block
__device__ __forceinline__ int32_t block_excl_scan(int32_t v, int32_t* warp_tot, int32_t* total) {
  const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
  int32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    int32_t t = warp_tot[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    warp_tot[lane] = t;  // inclusive over warps
  }
  __syncthreads();
  const int32_t r = x - v + (w ? warp_tot[w - 1] : 0);
  if (total) *total = warp_tot[31];
  __syncthreads();
  return r;
}

// shared memory of route_assign_kernel: partial sums [2][kRouteThreads] i32,
// run [E] i32, per-warp counts [32][E] u16, 32 warp totals
size_t route_assign_smem(int C, int E) {
  (void)C;
  return 2 * static_cast<size_t>(kRouteThreads) * 4 + static_cast<size_t>(E) * 4 + 32 * static_cast<size_t>(E) * 2 +
         32 * 4;
}

__global__ void __launch_bounds__(kRouteThreads) route_assign_kernel(const int64_t* __restrict__ ids, int64_t n, int E,
                                                                     int64_t chunk, int C,
                                                                     const int32_t* __restrict__ cnt,
                                                                     int64_t* __restrict__ slot,
                                                                     int32_t* __restrict__ tot_out,
                                                                     int32_t* __restrict__ off_out) {
  pdl_wait();
  extern __shared__ __align__(16) uint8_t rs[];
  int32_t* ps = reinterpret_cast<int32_t*>(rs);  // [2][kRouteThreads] partial (total, before-me) sums
  int32_t* run = ps + 2 * kRouteThreads;
  uint16_t* wh = reinterpret_cast<uint16_t*>(run + E);
  int32_t* wt = reinterpret_cast<int32_t*>(wh + 32 * E);
  const int tid = threadIdx.x, lane = tid % 32, warp = tid / 32;
  for (int i = tid; i < 32 * E; i += blockDim.x) wh[i] = 0;
  // bases of this chunk (thread e owns expert e): off[e] = exclusive scan of
  // the expert totals, plus the counts of the chunks before this one.  Every
  // thread sums a strided share of one expert's chunk counts straight from
  // global memory (C / parts loads each), reduced through shared memory.
  const int parts = kRouteThreads / E;  // E <= kRouteThreads
  if (tid < parts * E) {
    int32_t a = 0, b = 0;
    for (int c = tid / E; c < C; c += parts) {
      const int32_t v = cnt[static_cast<int64_t>(c) * E + tid % E];
      a += v;
      if (c < static_cast<int>(blockIdx.x)) b += v;
    }
    ps[tid] = a;
    ps[kRouteThreads + tid] = b;
  }
  __syncthreads();
  int32_t tot = 0, pre = 0;
  if (tid < E)
    for (int p2 = 0; p2 < parts; ++p2) {
      tot += ps[p2 * E + tid];
      pre += ps[kRouteThreads + p2 * E + tid];
    }
  const int32_t off = block_excl_scan(tid < E ? tot : 0, wt, nullptr);
  if (tid < E) {
    run[tid] = off + pre;
    if (blockIdx.x == 0) {
      if (tot_out) tot_out[tid] = tot;
      if (off_out) off_out[tid] = off;
    }
  }
  const int64_t s0 = static_cast<int64_t>(blockIdx.x) * chunk;
  const int64_t s1 = s0 + chunk < n ? s0 + chunk : n;
  for (int64_t r0 = s0; r0 < s1; r0 += blockDim.x) {  // rounds of 1024 slots, in slot order
    const int64_t s = r0 + tid;
    int key = -1 - lane;  // unique per lane when the slot is absent or its id invalid
    if (s < s1) {
      const int64_t e = ids[s];
      if (valid_id(e, E)) key = static_cast<int>(e);
    }
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    const int below = __popc(peers & ((1u << lane) - 1u));  // same-expert slots earlier in my warp
    if (key >= 0 && below == 0) wh[warp * E + key] = static_cast<uint16_t>(__popc(peers));
    __syncthreads();
    int32_t round_tot = 0;
    if (tid < E) {  // per-warp counts -> exclusive offsets over the 32 warps
#pragma unroll 8
      for (int w = 0; w < 32; ++w) {
        const int32_t v = wh[w * E + tid];
        wh[w * E + tid] = static_cast<uint16_t>(round_tot);
        round_tot += v;
      }
    }
    __syncthreads();
    if (key >= 0)
      slot[s] = static_cast<int64_t>(run[key] + wh[warp * E + key] + below);
    else if (s < s1)
      slot[s] = -1;
    __syncthreads();
    if (tid < E) {
      run[tid] += round_tot;
      for (int w = 0; w < 32; ++w) wh[w * E + tid] = 0;
    }
    __syncthreads();
  }
  pdl_trigger();
}

// shared memory of route_tiles_kernel: counts [C][E] i32 + 32 warp totals
// Grouped-GEMM tile table from the chunk counts (one CTA): gtab[0] = tiles,
// then (row0, row_end, expert) per tile_m-row tile, experts in order.
__global__ void __launch_bounds__(kRouteThreads) route_tiles_kernel(const int32_t* __restrict__ cnt, int C, int E,
                                                                    int tile_m, int32_t* __restrict__ gtab) {
  pdl_wait();
  __shared__ int32_t wt[32];
  __shared__ int32_t part_sum[kRouteThreads];
  const int tid = threadIdx.x;
  // every thread sums a strided share of the chunk counts of one expert
  // (C / parts independent loads each instead of C dependent ones on E threads)
  const int parts = kRouteThreads / E;  // E <= kRouteThreads
  if (tid < parts * E) {
    int32_t acc = 0;
    for (int c = tid / E; c < C; c += parts) acc += cnt[static_cast<int64_t>(c) * E + tid % E];
    part_sum[tid] = acc;
  }
  __syncthreads();
  int32_t tot = 0;
  if (tid < E)
    for (int p2 = 0; p2 < parts; ++p2) tot += part_sum[p2 * E + tid];
  const int32_t tiles = tid < E ? (tot + tile_m - 1) / tile_m : 0;
  const int32_t off = block_excl_scan(tid < E ? tot : 0, wt, nullptr);
  int32_t n_tiles = 0;
  const int32_t tbase = block_excl_scan(tiles, wt, &n_tiles);
  if (tid == 0) gtab[0] = n_tiles;
  if (tid < E) {
    int32_t* g = gtab + 1 + 3 * tbase;
    for (int32_t i = 0; i < tiles; ++i) {
      g[3 * i] = off + i * tile_m;
      g[3 * i + 1] = off + tot;
      g[3 * i + 2] = tid;
    }
  }
  pdl_trigger();
}

// xd[slot[t, j]] = x[t] for j < k: one warp per token, the row read once into
// registers (8 x 16 B per lane per 4 KB) and written to its k expert-sorted rows
__global__ void __launch_bounds__(256) gather_tokens_kernel(const __nv_bfloat16* __restrict__ x,
                                                            const int64_t* __restrict__ slot, int64_t T, int k,
                                                            int64_t H, __nv_bfloat16* __restrict__ xd) {
  pdl_wait();
  pdl_trigger();
  const int64_t t = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (t >= T) return;
  const int64_t my_slot = lane < k ? slot[t * k + lane] : -1;
  const uint4* src = reinterpret_cast<const uint4*>(x + t * H);
  const int64_t nv = H / 8;
  for (int64_t v0 = 0; v0 < nv; v0 += 8 * 32) {
    uint4 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t idx = v0 + i * 32 + lane;
      if (idx < nv) v[i] = __ldcs(src + idx);
    }
    for (int j = 0; j < k; ++j) {
      const int64_t d = __shfl_sync(0xffffffffu, my_slot, j);
      if (d < 0) continue;
      uint4* dst = reinterpret_cast<uint4*>(xd + d * H);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int64_t idx = v0 + i * 32 + lane;
        if (idx < nv) dst[idx] = v[i];
      }
    }
  }
}

// y[t] = sum_j w[t,j] * yd[slot[t,j]]  (fp32, j ascending), one CTA per token
__global__ void __launch_bounds__(256) combine_kernel(const __nv_bfloat16* __restrict__ yd,
                                                      const int64_t* __restrict__ slot, const float* __restrict__ w,
                                                      int k, int64_t H, __nv_bfloat16* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  const int64_t t = blockIdx.x;
  for (int64_t c = threadIdx.x; c < H / 8; c += blockDim.x) {
    float acc[8] = {};
    for (int j = 0; j < k; ++j) {
      const int64_t d = slot[t * k + j];
      if (d < 0) continue;
      const float wj = w[t * k + j];
      const uint4 u = *reinterpret_cast<const uint4*>(yd + d * H + c * 8);
      const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(h2[i]);
        acc[2 * i] += wj * f.x;
        acc[2 * i + 1] += wj * f.y;
      }
    }
    uint4 o;
    __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int i = 0; i < 4; ++i) o2[i] = __floats2bfloat162_rn(acc[2 * i], acc[2 * i + 1]);
    *reinterpret_cast<uint4*>(y + t * H + c * 8) = o;
  }
}

// ---------------------------------------------------------------- expert parallel
// W ranks, rank r owns experts [r*El, (r+1)*El).  Every rank runs the same
// plan, so a tensor sits at the same arena offset everywhere: peers write the
// dispatched rows straight into the owner's xr tensor (and results straight
// back into the source's yc tensor) over NVLink.  Receive layout on the owner:
// rows sorted by (local expert, source rank, source slot order); rinfo =
// [El per-local-expert row counts | per-row source code (rank * T*k + slot)].
struct PeerArena {
  char* base[kMaxWorld];
};

// counts all-gather through the window + the offsets every rank derives from it
__global__ void __launch_bounds__(1024) ep_exchange_kernel(PeerPtrs pp, uint32_t* epochs, uint32_t* err, int W,
                                                           int rank, int E, int El,
                                                           const int32_t* __restrict__ tot,
                                                           int32_t* __restrict__ send_off,
                                                           int64_t* __restrict__ rinfo_head) {
  pdl_wait();
  if (!slot_barrier(pp, epochs, kBarrierSlot, W, rank, err)) return;  // all ranks reached the dispatch
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    for (int p = 0; p < W; ++p) static_cast<int32_t*>(const_cast<void*>(pp.buf[p]))[rank * E + e] = tot[e];
  __threadfence_system();
  if (!slot_barrier(pp, epochs, kBarrierSlot, W, rank, err)) return;  // count matrix complete
  const int32_t* M = static_cast<const int32_t*>(pp.buf[rank]);         // [W][E]
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int o = e / El, el = e % El;
    int32_t acc = 0;
    for (int e2 = o * El; e2 < o * El + el; ++e2)
      for (int src = 0; src < W; ++src) acc += M[src * E + e2];
    for (int src = 0; src < rank; ++src) acc += M[src * E + e];
    send_off[e] = acc;
  }
  for (int el = threadIdx.x; el < El; el += blockDim.x) {
    int32_t r = 0;
    for (int src = 0; src < W; ++src) r += M[src * E + rank * El + el];
    rinfo_head[el] = r;
  }
  pdl_trigger();
}

// one warp per local slot: row x[s / k] -> owner's xr, source code -> owner's rinfo
__global__ void __launch_bounds__(256) ep_send_kernel(PeerArena pa, int64_t xr_off, int64_t rinfo_off,
                                                      const __nv_bfloat16* __restrict__ x,
                                                      const int64_t* __restrict__ ids,
                                                      const int64_t* __restrict__ slot_local,
                                                      const int32_t* __restrict__ off_local,
                                                      const int32_t* __restrict__ send_off, int64_t n, int k,
                                                      int64_t H, int E, int El, int rank, int64_t cap,
                                                      const uint32_t* __restrict__ err) {
  pdl_wait();
  if (*reinterpret_cast<const volatile uint32_t*>(err)) return;  // poisoned window: the counts are not valid
  const int lane = threadIdx.x % 32;
  for (int64_t s = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32; s < n;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x / 32) {
    const int64_t e = ids[s];
    if (!valid_id(e, E)) continue;
    const int o = static_cast<int>(e / El);
    const int64_t dest = send_off[e] + (slot_local[s] - off_local[e]);
    if (dest < 0 || dest >= cap) continue;  // never write outside the owner's receive tensor
    const uint4* src = reinterpret_cast<const uint4*>(x + (s / k) * H);
    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(pa.base[o] + xr_off) + dest * H);
    for (int64_t i = lane; i < H / 8; i += 32) dst[i] = src[i];
    if (lane == 0) reinterpret_cast<int64_t*>(pa.base[o] + rinfo_off)[El + dest] = static_cast<int64_t>(rank) * n + s;
  }
  __threadfence_system();
}

__global__ void ep_barrier_kernel(PeerPtrs pp, uint32_t* epochs, uint32_t* err, int W, int rank) {
  pdl_wait();
  slot_barrier(pp, epochs, kBarrierSlot, W, rank, err);
  pdl_trigger();
}

// one warp per received row: expert output row -> the source rank's yc[slot]
__global__ void __launch_bounds__(256) ep_return_kernel(PeerArena pa, int64_t yc_off,
                                                        const __nv_bfloat16* __restrict__ yr,
                                                        const int64_t* __restrict__ rinfo, int El, int64_t n,
                                                        int64_t H, int W, int64_t cap,
                                                        const uint32_t* __restrict__ err) {
  pdl_wait();
  if (*reinterpret_cast<const volatile uint32_t*>(err)) return;  // poisoned window: rinfo is not valid
  __shared__ int64_t n_recv;
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int el = 0; el < El; ++el) t += rinfo[el];
    n_recv = t < cap ? t : cap;
  }
  __syncthreads();
  const int lane = threadIdx.x % 32;
  for (int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32; i < n_recv;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x / 32) {
    const int64_t code = rinfo[El + i];
    const int p = static_cast<int>(code / n);
    const int64_t s = code % n;
    if (code < 0 || p >= W) continue;  // never follow a corrupt source code
    const uint4* src = reinterpret_cast<const uint4*>(yr + i * H);
    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(pa.base[p] + yc_off) + s * H);
    for (int64_t c = lane; c < H / 8; c += 32) dst[c] = src[c];
  }
  __threadfence_system();
}

// y[t] = sum_j w[t,j] * yc[t*k + j]  (valid ids only, j ascending)
__global__ void __launch_bounds__(256) combine_slots_kernel(const __nv_bfloat16* __restrict__ yc,
                                                            const int64_t* __restrict__ ids,
                                                            const float* __restrict__ w, int k, int E, int64_t H,
                                                            __nv_bfloat16* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  const int64_t t = blockIdx.x;
  for (int64_t c = threadIdx.x; c < H / 8; c += blockDim.x) {
    float acc[8] = {};
    for (int j = 0; j < k; ++j) {
      if (!valid_id(ids[t * k + j], E)) continue;
      const float wj = w[t * k + j];
      const uint4 u = *reinterpret_cast<const uint4*>(yc + (t * k + j) * H + c * 8);
      const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(h2[i]);
        acc[2 * i] += wj * f.x;
        acc[2 * i + 1] += wj * f.y;
      }
    }
    uint4 o;
    __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int i = 0; i < 4; ++i) o2[i] = __floats2bfloat162_rn(acc[2 * i], acc[2 * i + 1]);
    *reinterpret_cast<uint4*>(y + t * H + c * 8) = o;
  }
}

// grouped-GEMM tile table from per-local-expert row counts (EP receive side)
__global__ void tiles_from_counts_kernel(const int64_t* __restrict__ counts, int El, int32_t* __restrict__ gtab,
                                         int tile_m, int64_t cap) {
  pdl_wait();
  if (threadIdx.x == 0) {
    int32_t row = 0, t = 0;
    for (int el = 0; el < El; ++el) {
      // clamp to the receive tensor's rows: tiles never address past it
      const int64_t c64 = counts[el] < 0 ? 0 : counts[el];
      const int32_t c = static_cast<int32_t>(c64 < cap - row ? c64 : cap - row);
      for (int32_t r = 0; r < c; r += tile_m, ++t) {
        gtab[1 + 3 * t] = row + r;
        gtab[2 + 3 * t] = row + c;
        gtab[3 + 3 * t] = el;
      }
      row += c;
    }
    gtab[0] = t;
  }
  pdl_trigger();
}

// ---------------------------------------------------------------- host ops
int64_t max_tiles(int64_t n, int E) { return n / moe_tile_m() + E + 1; }
size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

int topk_param(const opf_op_ctx& c) { return static_cast<int>(ctx_param(c, "topk", 8)); }
int experts_param(const opf_op_ctx& c) { return static_cast<int>(ctx_param(c, "experts", 128)); }

size_t cnt_bytes(int64_t n, int E) { return align256(static_cast<size_t>(route_chunks(n, E)) * E * 4); }

// per-chunk expert histograms into ws (C x E i32)
void route_hist(const int64_t* ids, int64_t n, int E, int32_t* cnt, cudaStream_t s) {
  const int64_t C = route_chunks(n, E);
  if (C > 0)
    launch_pdl(route_hist_kernel, dim3(static_cast<unsigned>(C)), dim3(kRouteThreads), static_cast<size_t>(E) * 4, s,
               ids, n, E, route_chunk(n, E), cnt);
}
// slot[s] = row of slot s in the expert-sorted layout (-1: invalid id); tot / off per expert (optional)
void route_assign(const int64_t* ids, int64_t n, int E, const int32_t* cnt, int64_t* slot, cudaStream_t s,
                  int32_t* tot = nullptr, int32_t* off = nullptr) {
  const int C = static_cast<int>(route_chunks(n, E));
  const size_t smem = route_assign_smem(C, E);
  static std::once_flag once;
  std::call_once(once, [] {
    OPF_CUDA(cudaFuncSetAttribute(route_assign_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(route_assign_smem(16, 1024))));
  });
  launch_pdl(route_assign_kernel, dim3(static_cast<unsigned>(std::max(C, 1))), dim3(kRouteThreads), smem, s, ids, n,
             E, route_chunk(n, E), C, cnt, slot, tot, off);
}

opf_status op_moe_topk(const opf_op_ctx* c, const opf_view* in, int32_t n_in, opf_view* out, int32_t n_out,
                       int64_t rows, void* stream) {
  if (n_in != 1 || n_out != 2) return op_error(Errc::ShapeMismatch, "moe_topk takes (logits) -> (ids, w)");
  const int E = static_cast<int>(view_row_elems(in[0]));
  const int k = topk_param(*c);
  if (E > 256 || k > 32 || k > E || k < 1) return op_error(Errc::ShapeMismatch, "moe_topk: E <= 256, 1 <= k <= min(32, E)");
  if (view_row_elems(out[0]) != k || view_row_elems(out[1]) != k || out[0].dtype != OPF_I64 || out[1].dtype != OPF_F32)
    return op_error(Errc::ShapeMismatch, "moe_topk: outputs are ids [T,k] i64 and w [T,k] f32");
  if (rows == 0) return 0;
  const int renorm = static_cast<int>(ctx_param(*c, "renorm", 1));
  auto s = static_cast<cudaStream_t>(stream);
  const unsigned grid = static_cast<unsigned>((rows * 32 + 255) / 256);
  int64_t* ids = vptr<int64_t>(out[0]);
  float* w = vptr<float>(out[1]);
  const int per = (E + 31) / 32;
#define OPF_TOPK(T, P)                                                                                 \
  launch_pdl(topk_kernel<T, P>, dim3(grid), dim3(256), 0, s, static_cast<const T*>(vptr<T>(in[0])), ids, w, \
             rows, E, k, renorm)
  if (in[0].dtype == OPF_BF16) {
    if (per <= 4) OPF_TOPK(__nv_bfloat16, 4); else OPF_TOPK(__nv_bfloat16, 8);
  } else if (in[0].dtype == OPF_F32) {
    if (per <= 4) OPF_TOPK(float, 4); else OPF_TOPK(float, 8);
  } else {
    return op_error(Errc::ShapeMismatch, "moe_topk: logits dtype");
  }
#undef OPF_TOPK
  return launch_status("moe_topk");
}

size_t ws_dispatch(const opf_op_ctx& c, const opf_view*, int, const opf_view*, int, int64_t rows) {
  return cnt_bytes(rows * topk_param(c), experts_param(c)) + 256;
}
size_t ws_grouped(const opf_op_ctx& c, const opf_view*, int, const opf_view*, int, int64_t rows) {
  const int64_t n = rows * topk_param(c);
  return cnt_bytes(n, experts_param(c)) + align256(static_cast<size_t>(1 + 3 * max_tiles(n, experts_param(c))) * 4) +
         256;
}

opf_status need_ws(const opf_op_ctx* c, size_t bytes, const char* who) {
  if (!c->workspace || c->workspace_bytes < bytes)
    return op_error(Errc::ConfigError, std::string(who) + ": workspace missing or too small");
  return 0;
}

opf_status op_moe_dispatch(const opf_op_ctx* c, const opf_view* in, int32_t n_in, opf_view* out,
                           int32_t n_out, int64_t rows, void* stream) {
  if (n_in != 2 || n_out != 2) return op_error(Errc::ShapeMismatch, "moe_dispatch takes (x, ids) -> (xd, slot)");
  const int k = topk_param(*c), E = experts_param(*c);
  const int64_t H = view_row_elems(in[0]);
  if (in[0].dtype != OPF_BF16 || out[0].dtype != OPF_BF16 || H % 8 || E > kMaxE ||
      view_row_elems(in[1]) != k || view_row_elems(out[0]) != k * H || view_row_elems(out[1]) != k ||
      out[1].dtype != OPF_I64)
    return op_error(Errc::ShapeMismatch, "moe_dispatch: x [T,H] bf16, ids [T,k] -> xd [T,k*H], slot [T,k] i64");
  if (rows == 0) return 0;
  if (opf_status e = need_ws(c, ws_dispatch(*c, in, n_in, out, n_out, rows), "moe_dispatch")) return e;
  auto s = static_cast<cudaStream_t>(stream);
  const int64_t n = rows * k;
  const int64_t* ids = vptr<int64_t>(in[1]);
  int64_t* slot = vptr<int64_t>(out[1]);
  auto* cnt = static_cast<int32_t*>(c->workspace);
  route_hist(ids, n, E, cnt, s);
  route_assign(ids, n, E, cnt, slot, s);
  launch_pdl(gather_tokens_kernel, dim3(static_cast<unsigned>((rows * 32 + 255) / 256)), dim3(256), 0, s,
             static_cast<const __nv_bfloat16*>(vptr<__nv_bfloat16>(in[0])), static_cast<const int64_t*>(slot), rows,
             k, H, vptr<__nv_bfloat16>(out[0]));
  return launch_status("moe_dispatch");
}

int ep_param(const opf_op_ctx& c) { return static_cast<int>(ctx_param(c, "ep", 1)); }

size_t ws_grouped_any(const opf_op_ctx& c, const opf_view* in, int n_in, const opf_view* out, int n_out,
                      int64_t rows) {
  const int ep = ep_param(c);
  if (ep <= 1) return ws_grouped(c, in, n_in, out, n_out, rows);
  const int64_t n = rows * topk_param(c) * ep;
  return align256(static_cast<size_t>(1 + 3 * max_tiles(n, experts_param(c) / ep)) * 4) + 256;
}

// shared body of the two grouped expert GEMMs.  ep == 1: (act, ids, w[E,K,N]),
// tile table from a routing pass over ids.  ep > 1: (act = received rows,
// rinfo, w = this rank's [E/ep, K, N] shard), tile table from rinfo's counts.
opf_status grouped(const opf_op_ctx* c, const opf_view* in, int32_t n_in, opf_view* out, int32_t n_out,
                   int64_t rows, void* stream, bool gate_up) {
  const char* who = gate_up ? "moe_gate_up" : "moe_down";
  if (n_in != 3 || n_out != 1) return op_error(Errc::ShapeMismatch, std::string(who) + " takes (act, ids|rinfo, w) -> out");
  const int k = topk_param(*c), ep = ep_param(*c), E = experts_param(*c);
  if (ep < 1 || E % ep) return op_error(Errc::ConfigError, std::string(who) + ": experts % ep");
  const int El = E / ep;  // experts whose weights this rank holds
  // w: [El, K, N] reference layout (per-expert [K,N] MatMul weight)
  const int64_t route_w = ep == 1 ? k : static_cast<int64_t>(ep) * k + El;
  if (in[2].rank != 3 || in[2].shape[0] != El || in[0].dtype != OPF_BF16 || in[2].dtype != OPF_BF16 ||
      out[0].dtype != OPF_BF16 || view_row_elems(in[1]) != route_w || in[1].dtype != OPF_I64)
    return op_error(Errc::ShapeMismatch, std::string(who) + ": w must be [experts/ep, K, N] bf16, ids [T, k] "
                                                            "(ep 1) or rinfo [T, ep*k + experts/ep] (ep > 1)");
  const int64_t K = in[2].shape[1], N = in[2].shape[2];
  const int64_t n_out_cols = gate_up ? N / 2 : N;
  const int64_t slots = static_cast<int64_t>(k) * ep;  // row capacity per token
  if (view_row_elems(in[0]) != slots * K || view_row_elems(out[0]) != slots * n_out_cols)
    return op_error(Errc::ShapeMismatch, std::string(who) + ": activation widths");
  if (rows == 0) return 0;
  const void* packed = c->aux ? c->aux : (ctx_param(*c, "packed", 0.0) != 0.0 ? view_ptr(in[2]) : nullptr);
  if (!packed)
    return op_error(Errc::ConfigError, std::string(who) + ": expert weights not packed (run through a Session, "
                                                          "or pass packed [E,N,K] weights with params.packed=1)");
  if (opf_status e = need_ws(c, ws_grouped_any(*c, in, n_in, out, n_out, rows), who)) return e;
  auto s = static_cast<cudaStream_t>(stream);
  const int64_t n = rows * slots;
  char* ws = static_cast<char*>(c->workspace);
  int32_t* gtab;
  if (ep == 1) {
    auto* cnt = reinterpret_cast<int32_t*>(ws);
    gtab = reinterpret_cast<int32_t*>(ws + cnt_bytes(n, E));
    route_hist(vptr<int64_t>(in[1]), n, E, cnt, s);
    launch_pdl(route_tiles_kernel, dim3(1), dim3(kRouteThreads), 0, s, static_cast<const int32_t*>(cnt),
               static_cast<int>(route_chunks(n, E)), E, moe_tile_m(), gtab);
  } else {
    gtab = reinterpret_cast<int32_t*>(ws);
    launch_pdl(tiles_from_counts_kernel, dim3(1), dim3(32), 0, s, static_cast<const int64_t*>(vptr<int64_t>(in[1])),
               El, gtab, moe_tile_m(), n);
  }
  GemmArgs g{};
  g.a = view_ptr(in[0]);
  g.bt = packed;
  g.c = view_ptr(out[0]);
  g.m = n;
  g.n = N;
  g.k = K;
  g.lda = K;
  g.ldc = n_out_cols;
  g.max_ctas = c->max_ctas;
  g.epi = gate_up ? 1 : 0;
  gemm_bf16_grouped(g, gtab, max_tiles(n, El), N, El, s);
  return launch_status(who);
}

// ---- expert-parallel dispatch / combine (peer-arena all-to-all)
struct EpCtx {
  WindowView w;
  PeerArena pa{};
  int W = 1, rank = 0;
};
opf_status ep_ctx(const opf_op_ctx* c, const char* who, EpCtx* x, std::initializer_list<const opf_view*> arena_views) {
  const opf_comm* cm = static_cast<const opf_comm*>(c->comm);
  const int ep = ep_param(*c);
  if (!cm || cm->world != ep || ep > kMaxWorld)
    return op_error(Errc::ConfigError, std::string(who) + ": needs a communicator with world == params.ep (<= 8)");
  if (!window_view(cm, &x->w))
    return op_error(Errc::ConfigError, std::string(who) + ": communicator has no peer window");
  if (cm->peer_arena.size() != static_cast<size_t>(ep) || !cm->arena_base)
    return op_error(Errc::ConfigError, std::string(who) + ": peer arenas not mapped (opf_session_arena_open / _link_local)");
  const char* base = static_cast<const char*>(cm->arena_base);
  for (const opf_view* v : arena_views) {
    const char* p = view_ptr(*v);
    if (p < base || p >= base + cm->arena_bytes)
      return op_error(Errc::ConfigError, std::string(who) + ": peer-written tensors must live in the session arena");
  }
  for (int r = 0; r < ep; ++r) x->pa.base[r] = static_cast<char*>(cm->peer_arena[r]);
  x->W = ep;
  x->rank = cm->rank;
  return 0;
}

size_t ws_ep_dispatch(const opf_op_ctx& c, const opf_view*, int, const opf_view*, int, int64_t rows) {
  const int64_t n = rows * topk_param(c);
  const int E = experts_param(c);
  return cnt_bytes(n, E) + align256(static_cast<size_t>(n) * 8) + 3 * align256(static_cast<size_t>(E) * 4) + 256;
}

opf_status op_moe_ep_dispatch(const opf_op_ctx* c, const opf_view* in, int32_t n_in, opf_view* out,
                              int32_t n_out, int64_t rows, void* stream) {
  if (n_in != 2 || n_out != 2)
    return op_error(Errc::ShapeMismatch, "moe_ep_dispatch takes (x, ids) -> (xr, rinfo)");
  const int k = topk_param(*c), E = experts_param(*c), ep = ep_param(*c);
  if (ep < 2 || E % ep || E > kMaxE) return op_error(Errc::ConfigError, "moe_ep_dispatch: ep >= 2 dividing experts");
  const int El = E / ep;
  const int64_t H = view_row_elems(in[0]);
  if (in[0].dtype != OPF_BF16 || out[0].dtype != OPF_BF16 || H % 8 || view_row_elems(in[1]) != k ||
      view_row_elems(out[0]) != static_cast<int64_t>(ep) * k * H || out[1].dtype != OPF_I64 ||
      view_row_elems(out[1]) != static_cast<int64_t>(ep) * k + El)
    return op_error(Errc::ShapeMismatch,
                    "moe_ep_dispatch: x [T,H] bf16, ids [T,k] -> xr [T, ep*k*H] bf16, rinfo [T, ep*k + experts/ep] i64");
  EpCtx x;
  if (opf_status e = ep_ctx(c, "moe_ep_dispatch", &x, {&out[0], &out[1]})) return e;
  if (x.w.stage_bytes < static_cast<size_t>(ep) * E * 4)
    return op_error(Errc::ConfigError, "moe_ep_dispatch: peer window smaller than the count matrix");
  if (opf_status e = need_ws(c, ws_ep_dispatch(*c, in, n_in, out, n_out, rows), "moe_ep_dispatch")) return e;
  auto s = static_cast<cudaStream_t>(stream);
  const int64_t n = rows * k;
  char* ws = static_cast<char*>(c->workspace);
  auto* cnt = reinterpret_cast<int32_t*>(ws);
  auto* slot_local = reinterpret_cast<int64_t*>(ws + cnt_bytes(n, E));
  auto* tot = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(slot_local) + align256(static_cast<size_t>(n) * 8));
  auto* off = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(tot) + align256(static_cast<size_t>(E) * 4));
  auto* send_off = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(off) + align256(static_cast<size_t>(E) * 4));
  const int64_t* ids = vptr<int64_t>(in[1]);
  if (n > 0) {
    route_hist(ids, n, E, cnt, s);
    route_assign(ids, n, E, cnt, slot_local, s, tot, off);
  } else {
    OPF_CUDA(cudaMemsetAsync(tot, 0, E * 4, s));
  }
  launch_pdl(ep_exchange_kernel, dim3(1), dim3(1024), 0, s, x.w.pp, x.w.epochs, x.w.err, ep, x.rank, E, El,
             static_cast<const int32_t*>(tot), send_off, vptr<int64_t>(out[1]));
  const char* base = static_cast<const char*>(static_cast<const opf_comm*>(c->comm)->arena_base);
  const int64_t xr_off = view_ptr(out[0]) - base, rinfo_off = view_ptr(out[1]) - base;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n * 32 + 255) / 256, num_sms() * 8LL)));
  launch_pdl(ep_send_kernel, dim3(grid), dim3(256), 0, s, x.pa, xr_off, rinfo_off,
             static_cast<const __nv_bfloat16*>(vptr<__nv_bfloat16>(in[0])), ids,
             static_cast<const int64_t*>(slot_local), static_cast<const int32_t*>(off),
             static_cast<const int32_t*>(send_off), n, k, H, E, El, x.rank, n * ep,
             static_cast<const uint32_t*>(x.w.err));
  launch_pdl(ep_barrier_kernel, dim3(1), dim3(32), 0, s, x.w.pp, x.w.epochs, x.w.err, ep, x.rank);
  return launch_status("moe_ep_dispatch");
}

// The returned rows land in the combine's workspace (planned inside the arena,
// so it sits at the same offset on every rank and lives exactly as long as the
// combine: peers write it only between the two barriers).
size_t ws_ep_combine(const opf_op_ctx& c, const opf_view*, int, const opf_view* out, int, int64_t rows) {
  return align256(static_cast<size_t>(rows) * topk_param(c) * view_row_elems(out[0]) * 2) + 256;
}

opf_status op_moe_ep_combine(const opf_op_ctx* c, const opf_view* in, int32_t n_in, opf_view* out,
                             int32_t n_out, int64_t rows, void* stream) {
  if (n_in != 4 || n_out != 1)
    return op_error(Errc::ShapeMismatch, "moe_ep_combine takes (yr, rinfo, w, ids) -> y");
  const int k = topk_param(*c), E = experts_param(*c), ep = ep_param(*c);
  if (ep < 2 || E % ep) return op_error(Errc::ConfigError, "moe_ep_combine: ep >= 2 dividing experts");
  const int El = E / ep;
  const int64_t H = view_row_elems(out[0]);
  if (in[0].dtype != OPF_BF16 || out[0].dtype != OPF_BF16 || H % 8 ||
      view_row_elems(in[0]) != static_cast<int64_t>(ep) * k * H ||
      view_row_elems(in[1]) != static_cast<int64_t>(ep) * k + El || in[2].dtype != OPF_F32 ||
      view_row_elems(in[2]) != k || view_row_elems(in[3]) != k)
    return op_error(Errc::ShapeMismatch, "moe_ep_combine: yr [T, ep*k*H], rinfo, w [T,k] f32, ids [T,k] -> y [T,H]");
  if (opf_status e = need_ws(c, ws_ep_combine(*c, in, n_in, out, n_out, rows), "moe_ep_combine")) return e;
  opf_view yc = out[0];
  yc.base = c->workspace;
  yc.elem_offset = 0;
  EpCtx x;
  if (opf_status e = ep_ctx(c, "moe_ep_combine", &x, {&yc})) return e;
  auto s = static_cast<cudaStream_t>(stream);
  const int64_t n = rows * k;
  const int64_t yc_off = static_cast<const char*>(c->workspace) -
                         static_cast<const char*>(static_cast<const opf_comm*>(c->comm)->arena_base);
  launch_pdl(ep_barrier_kernel, dim3(1), dim3(32), 0, s, x.w.pp, x.w.epochs, x.w.err, ep, x.rank);
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n * ep * 32 + 255) / 256, num_sms() * 8LL)));
  launch_pdl(ep_return_kernel, dim3(grid), dim3(256), 0, s, x.pa, yc_off,
             static_cast<const __nv_bfloat16*>(vptr<__nv_bfloat16>(in[0])),
             static_cast<const int64_t*>(vptr<int64_t>(in[1])), El, n, H, ep, n * ep,
             static_cast<const uint32_t*>(x.w.err));
  launch_pdl(ep_barrier_kernel, dim3(1), dim3(32), 0, s, x.w.pp, x.w.epochs, x.w.err, ep, x.rank);
  if (rows > 0)
    launch_pdl(combine_slots_kernel, dim3(static_cast<unsigned>(rows)), dim3(256), 0, s,
               static_cast<const __nv_bfloat16*>(c->workspace),
               static_cast<const int64_t*>(vptr<int64_t>(in[3])), static_cast<const float*>(vptr<float>(in[2])), k, E,
               H, vptr<__nv_bfloat16>(out[0]));
  return launch_status("moe_ep_combine");
}

opf_status op_moe_gate_up(const opf_op_ctx* c, const opf_view* in, int32_t n_in, opf_view* out, int32_t n_out,
                          int64_t rows, void* stream) {
  return grouped(c, in, n_in, out, n_out, rows, stream, true);
}
opf_status op_moe_down(const opf_op_ctx* c, const opf_view* in, int32_t n_in, opf_view* out, int32_t n_out,
                       int64_t rows, void* stream) {
  return grouped(c, in, n_in, out, n_out, rows, stream, false);
}

opf_status op_moe_combine(const opf_op_ctx* c, const opf_view* in, int32_t n_in, opf_view* out, int32_t n_out,
                          int64_t rows, void* stream) {
  if (n_in != 3 || n_out != 1) return op_error(Errc::ShapeMismatch, "moe_combine takes (yd, slot, w) -> y");
  const int k = topk_param(*c);
  const int64_t H = view_row_elems(out[0]);
  if (in[0].dtype != OPF_BF16 || out[0].dtype != OPF_BF16 || in[1].dtype != OPF_I64 || in[2].dtype != OPF_F32 ||
      H % 8 || view_row_elems(in[0]) != k * H || view_row_elems(in[1]) != k || view_row_elems(in[2]) != k)
    return op_error(Errc::ShapeMismatch, "moe_combine: yd [T,k*H] bf16, slot [T,k] i64, w [T,k] f32 -> y [T,H]");
  if (rows == 0) return 0;
  auto s = static_cast<cudaStream_t>(stream);
  launch_pdl(combine_kernel, dim3(static_cast<unsigned>(rows)), dim3(256), 0, s,
             static_cast<const __nv_bfloat16*>(vptr<__nv_bfloat16>(in[0])),
             static_cast<const int64_t*>(vptr<int64_t>(in[1])), static_cast<const float*>(vptr<float>(in[2])), k,
             H, vptr<__nv_bfloat16>(out[0]));
  return launch_status("moe_combine");
}

}  // namespace

void register_moe_ops(OpRegistry& r) {
  r.add({"moe_topk", op_moe_topk, ResourceClass::kMemory, 1, 2, {}});
  r.add({"moe_dispatch", op_moe_dispatch, ResourceClass::kNetwork, 2, 2, ws_dispatch});
  r.add({"moe_gate_up", op_moe_gate_up, ResourceClass::kCompute, 3, 1, ws_grouped_any, 2, 2});
  r.add({"moe_down", op_moe_down, ResourceClass::kCompute, 3, 1, ws_grouped_any, 2, 3});
  r.add({"moe_combine", op_moe_combine, ResourceClass::kNetwork, 3, 1, {}});
  r.add({"moe_ep_dispatch", op_moe_ep_dispatch, ResourceClass::kNetwork, 2, 2, ws_ep_dispatch});
  r.add({"moe_ep_combine", op_moe_ep_combine, ResourceClass::kNetwork, 4, 1, ws_ep_combine});
}

}  // namespace opflow
