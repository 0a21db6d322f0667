// Paged decode attention on tensor cores (memory-bound hot kernel of the
// decode config).  qkv_rot [B, (nq+2nkv)*128] holds the current token; K/V
// cache [pages, 16, nkv, 128] bf16 with a per-sequence block table; the
// sequence attends to its `ctx` cached tokens plus itself.
//
// Persistent: one CTA per SM (8 warps) walks (sequence, kv head) items; warp w streams pages w, w+8, ...
// (16 tokens x 256 B of K and of V each) with cp.async into a 3-deep per-warp
// ring (XOR-swizzled): 192 KB per SM in flight.  The grid size is the SM budget.  The GQA group is the
// MMA M dimension: S[16 x 16 tokens] = Q[16 x 128] K^T and O[16 x 128] += P V
// are 32 mma.sync m16n8k16 per page per warp (rows >= group are zero padding),
// i.e. ~2 tensor instructions per token instead of ~60 SIMT ones — the
// kernel becomes HBM-bound.  Online softmax in fp32 on the accumulator
// fragments; the 4 warps' (m, l, O) and the current token merge in smem.
// Algorithmic bytes per (sequence, kv head) = 2 * ctx * 128 * 2.
#include <cuda_bf16.h>

#include <cfloat>

#include "opflow/device.hpp"

namespace opflow {

namespace {

constexpr int HD = 128;
constexpr int PAGE = 16;
constexpr int kWarps = 8;
constexpr int kDepth = 3;                  // pages in flight per warp
constexpr int kPageBytes = PAGE * HD * 2;  // 4 KB (one tensor, one page, one kv head)
constexpr int kWarpRing = kDepth * 2 * kPageBytes;
constexpr int kSmemRing = kWarps * kWarpRing;  // 192 KB -> 1 CTA per SM

__device__ __forceinline__ uint32_t saddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t swz(int r, int c) {
  return static_cast<uint32_t>(r * (HD * 2) + ((c ^ (r & 7)) << 4));
}
__device__ __forceinline__ void cp16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void ldsm4(uint32_t a, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(a));
}
__device__ __forceinline__ void ldsm4t(uint32_t a, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(a));
}
__device__ __forceinline__ void mma(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pk(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

__global__ void __launch_bounds__(kWarps * 32)
    decode_mma_kernel(const __nv_bfloat16* __restrict__ qkv, const __nv_bfloat16* __restrict__ kc,
                      const __nv_bfloat16* __restrict__ vc, const int64_t* __restrict__ table,
                      const int64_t* __restrict__ ctx_len, __nv_bfloat16* __restrict__ out, int nq,
                      int nkv, int64_t max_pages, float scale_log2, int64_t n_items) {
  extern __shared__ __align__(128) uint8_t smem[];
  pdl_wait();
  pdl_trigger();
  // persistent: a CTA (one per SM) walks (sequence, kv head) items, so the
  // launch occupies exactly gridDim.x SMs (SM partitioning under overlap)
  for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
  const int64_t b = item / nkv;
  const int kh = static_cast<int>(item % nkv);
  const int G = nq / nkv;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int g = lane >> 2, t = lane & 3;
  const int64_t W = static_cast<int64_t>(nq + 2 * nkv) * HD;
  const __nv_bfloat16* row = qkv + b * W;
  const int64_t ctx = ctx_len[b];
  const int n_pages = static_cast<int>((ctx + PAGE - 1) / PAGE);
  const int64_t tok_stride = static_cast<int64_t>(nkv) * HD;  // elements between tokens of a page

  uint8_t* ring = smem + warp * kWarpRing;
  auto k_slot = [&](int s) { return ring + s * 2 * kPageBytes; };
  auto v_slot = [&](int s) { return ring + s * 2 * kPageBytes + kPageBytes; };
  auto issue = [&](int page_idx, int s) {
    const int64_t pg = table[b * max_pages + page_idx];
    const __nv_bfloat16* kp = kc + (pg * PAGE * nkv + kh) * HD;
    const __nv_bfloat16* vp = vc + (pg * PAGE * nkv + kh) * HD;
    const uint32_t kd = saddr(k_slot(s)), vd = saddr(v_slot(s));
#pragma unroll
    for (int i = 0; i < 8; ++i) {  // 16 rows x 16 chunks = 256 chunks per tensor
      const int idx = i * 32 + lane;
      const int r = idx >> 4, c = idx & 15;
      cp16(kd + swz(r, c), kp + r * tok_stride + c * 8);
      cp16(vd + swz(r, c), vp + r * tok_stride + c * 8);
    }
  };

  // Q fragments (rows = heads of the group; rows >= G are zero)
  uint32_t qf[8][4];
  {
    const bool valid = g < G;
    const __nv_bfloat16* qrow = row + static_cast<int64_t>(kh * G + (valid ? g : 0)) * HD;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      qf[kk][0] = valid ? *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 2 * t) : 0u;
      qf[kk][1] = 0u;
      qf[kk][2] = valid ? *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 8 + 2 * t) : 0u;
      qf[kk][3] = 0u;
    }
  }
  float o[16][4];
#pragma unroll
  for (int d = 0; d < 16; ++d) o[d][0] = o[d][1] = o[d][2] = o[d][3] = 0.0f;
  float m_r = -FLT_MAX, l_r = 0.0f;

  // prologue: fill the ring
  int my_pages = 0;
  for (int p = warp; p < n_pages; p += kWarps) ++my_pages;
#pragma unroll
  for (int s = 0; s < kDepth; ++s) {
    if (s < my_pages) issue(warp + s * kWarps, s);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int i = 0; i < my_pages; ++i) {
    const int s = i % kDepth;
    const int page_idx = warp + i * kWarps;
    asm volatile("cp.async.wait_group %0;" ::"n"(kDepth - 1) : "memory");
    __syncwarp();
    // S = Q K^T for 16 tokens
    float sc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
    const uint32_t kb = saddr(k_slot(s)), vb = saddr(v_slot(s));
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      uint32_t b0, b1, b2, b3;
      ldsm4(kb + swz((lane & 7) + (lane >> 4) * 8, kk * 2 + ((lane >> 3) & 1)), b0, b1, b2, b3);
      mma(sc[0], qf[kk], b0, b1);
      mma(sc[1], qf[kk], b2, b3);
    }
    // online softmax over this page (rows g < G meaningful)
    const int64_t tok0 = static_cast<int64_t>(page_idx) * PAGE;
    float mx = m_r;
#pragma unroll
    for (int n = 0; n < 2; ++n)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t tok = tok0 + n * 8 + 2 * t + e;
        float v = sc[n][e] * scale_log2;
        if (tok >= ctx) v = -FLT_MAX;
        sc[n][e] = v;
        mx = fmaxf(mx, v);
      }
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float corr = exp2f(m_r - mx);
    float p[2][2], rs = 0.0f;
#pragma unroll
    for (int n = 0; n < 2; ++n)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        p[n][e] = exp2f(sc[n][e] - mx);
        rs += p[n][e];
      }
    l_r = l_r * corr + rs;
    m_r = mx;
    const uint32_t pa[4] = {pk(p[0][0], p[0][1]), 0u, pk(p[1][0], p[1][1]), 0u};
#pragma unroll
    for (int d = 0; d < 16; ++d) {
      o[d][0] *= corr;
      o[d][1] *= corr;
    }
    // O += P V  (k = 16 tokens, n = 128 dims)
#pragma unroll
    for (int dp = 0; dp < 8; ++dp) {
      uint32_t b0, b1, b2, b3;
      ldsm4t(vb + swz((lane & 7) + ((lane >> 3) & 1) * 8, dp * 2 + (lane >> 4)), b0, b1, b2, b3);
      mma(o[2 * dp], pa, b0, b1);
      mma(o[2 * dp + 1], pa, b2, b3);
    }
    __syncwarp();
    // refill this slot with the page kDepth ahead
    if (i + kDepth < my_pages) issue(warp + (i + kDepth) * kWarps, s);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");

  // ---- merge: per-warp partial states -> smem (reuses the ring)
  __syncthreads();
  float* sm_m = reinterpret_cast<float*>(smem);                  // [kWarps][16]
  float* sm_l = sm_m + kWarps * 16;                              // [kWarps][16]
  float* sm_o = sm_l + kWarps * 16;                              // [kWarps][16][HD]
  l_r += __shfl_xor_sync(0xffffffffu, l_r, 1);
  l_r += __shfl_xor_sync(0xffffffffu, l_r, 2);
  if (t == 0) {
    sm_m[warp * 16 + g] = m_r;
    sm_l[warp * 16 + g] = l_r;
  }
#pragma unroll
  for (int d = 0; d < 16; ++d) {
    sm_o[(warp * 16 + g) * HD + d * 8 + 2 * t] = o[d][0];
    sm_o[(warp * 16 + g) * HD + d * 8 + 2 * t + 1] = o[d][1];
  }
  __syncthreads();
  // current token (in qkv): one warp per head computes its score
  float* sm_cur = sm_o + kWarps * 16 * HD;  // [16]: scaled score of the current token per head
  const __nv_bfloat16* kcur = row + static_cast<int64_t>(nq + kh) * HD;
  const __nv_bfloat16* vcur = row + static_cast<int64_t>(nq + nkv + kh) * HD;
  for (int h = warp; h < G; h += kWarps) {
    const __nv_bfloat16* q = row + static_cast<int64_t>(kh * G + h) * HD;
    float dot = 0.0f;
    for (int d = lane; d < HD; d += 32) dot += __bfloat162float(q[d]) * __bfloat162float(kcur[d]);
#pragma unroll
    for (int s2 = 16; s2 > 0; s2 >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, s2);
    if (lane == 0) sm_cur[h] = dot * scale_log2;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < G * HD; idx += blockDim.x) {
    const int h = idx / HD, d = idx % HD;
    float M = sm_cur[h];
    for (int w = 0; w < kWarps; ++w) M = fmaxf(M, sm_m[w * 16 + h]);
    const float cc = exp2f(sm_cur[h] - M);
    float L = cc, A = cc * __bfloat162float(vcur[d]);
    for (int w = 0; w < kWarps; ++w) {
      if (sm_l[w * 16 + h] == 0.0f) continue;
      const float c = exp2f(sm_m[w * 16 + h] - M);
      L += sm_l[w * 16 + h] * c;
      A += sm_o[(w * 16 + h) * HD + d] * c;
    }
    out[b * static_cast<int64_t>(nq) * HD + static_cast<int64_t>(kh * G + h) * HD + d] =
        __float2bfloat16(A / L);
  }
  __syncthreads();  // smem is reused by the next item's ring
  }
}

}  // namespace

bool decode_bf16_mma(const __nv_bfloat16* qkv, const __nv_bfloat16* kc, const __nv_bfloat16* vc,
                     const int64_t* table, const int64_t* ctx, __nv_bfloat16* out, int64_t B, int nq,
                     int nkv, int hd, int page, int64_t max_pages, float scale, int max_ctas,
                     cudaStream_t s) {
  if (hd != HD || page != PAGE || nq % nkv != 0 || nq / nkv > 8) return false;
  static bool attr = [] {
    return cudaFuncSetAttribute(decode_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kSmemRing) == cudaSuccess;
  }();
  if (!attr) return false;
  const int64_t items = B * nkv;
  int64_t grid = max_ctas > 0 ? std::min<int64_t>(max_ctas, num_sms()) : num_sms();
  grid = std::max<int64_t>(1, std::min(grid, items));
  launch_pdl(decode_mma_kernel, dim3(static_cast<unsigned>(grid)), dim3(kWarps * 32), kSmemRing, s,
             qkv, kc, vc, table, ctx, out, nq, nkv, max_pages, scale * 1.4426950408889634f, items);
  return true;
}

}  // namespace opflow
