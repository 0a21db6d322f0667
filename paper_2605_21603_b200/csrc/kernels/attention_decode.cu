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
#include <cuda.h>
#include <cuda_bf16.h>

#include <cfloat>
#include <cstdlib>

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


// ------------------------------------------------------------------ transposed variant
// Tokens on the MMA M dimension, the GQA group on N (8): S^T[16 tok x 8 heads]
// = K[16 x 128] Q^T and O^T[128 dims x 8 heads] += V^T P^T — 8 + 8 m16n8k16
// per page instead of 16 + 16 with the group padded to M = 16, and a 32-float
// accumulator instead of 64.  P^T reaches the B-fragment layout through 8
// shuffles; the softmax reduces over tokens (lane bits 2..4).  W warps with
// D-deep private cp.async page rings (W x D x 8 KB of smem).
template <int W, int D>
__global__ void __launch_bounds__(W * 32)
    decode_t_kernel(const __nv_bfloat16* __restrict__ qkv, const __nv_bfloat16* __restrict__ kc,
                    const __nv_bfloat16* __restrict__ vc, const int64_t* __restrict__ table,
                    const int64_t* __restrict__ ctx_len, __nv_bfloat16* __restrict__ out, int nq, int nkv,
                    int64_t max_pages, float scale_log2, int64_t n_items, int hnd) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int kRing = D * 2 * kPageBytes;
  pdl_wait();
  pdl_trigger();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int g = lane >> 2, t = lane & 3;
  for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int64_t b = item / nkv;
    const int kh = static_cast<int>(item % nkv);
    const int G = nq / nkv;
    const int64_t Wd = static_cast<int64_t>(nq + 2 * nkv) * HD;
    const __nv_bfloat16* row = qkv + b * Wd;
    const int64_t ctx = ctx_len[b];
    const int n_pages = static_cast<int>((ctx + PAGE - 1) / PAGE);
    // NHD pages [16 tokens][nkv][128] (reference / vLLM layout) or HND pages
    // [nkv][16 tokens][128]: one (page, kv head) block is 4 KB contiguous, which
    // DRAM streams ~2-5% faster than 16 rows of 256 B at 2 KB stride
    const int64_t tok_stride = hnd ? HD : static_cast<int64_t>(nkv) * HD;
    const int64_t head_off = hnd ? static_cast<int64_t>(kh) * PAGE * HD : static_cast<int64_t>(kh) * HD;
    uint8_t* ring = smem + warp * kRing;
    auto k_slot = [&](int s) { return ring + s * 2 * kPageBytes; };
    auto v_slot = [&](int s) { return ring + s * 2 * kPageBytes + kPageBytes; };
    auto issue = [&](int page_idx, int s) {
      const int64_t pg = table[b * max_pages + page_idx];
      const __nv_bfloat16* kp = kc + pg * PAGE * nkv * HD + head_off;
      const __nv_bfloat16* vp = vc + pg * PAGE * nkv * HD + head_off;
      const uint32_t kd = saddr(k_slot(s)), vd = saddr(v_slot(s));
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int idx = i * 32 + lane;
        const int r = idx >> 4, c = idx & 15;
        cp16(kd + swz(r, c), kp + r * tok_stride + c * 8);
        cp16(vd + swz(r, c), vp + r * tok_stride + c * 8);
      }
    };
    // Q^T as the B operand: n = head g of the group (zero for g >= G), k = dims
    uint32_t qb[8][2];
    {
      const bool valid = g < G;
      const __nv_bfloat16* qrow = row + static_cast<int64_t>(kh * G + (valid ? g : 0)) * HD;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        qb[kk][0] = valid ? *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 2 * t) : 0u;
        qb[kk][1] = valid ? *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 8 + 2 * t) : 0u;
      }
    }
    float o[8][4];  // O^T: [dim tile][(dim g | g+8) x (head 2t | 2t+1)]
#pragma unroll
    for (int d = 0; d < 8; ++d) o[d][0] = o[d][1] = o[d][2] = o[d][3] = 0.0f;
    float m_r[2] = {-FLT_MAX, -FLT_MAX}, l_r[2] = {0.0f, 0.0f};  // heads 2t, 2t+1 (l: this lane's tokens)
    int my_pages = 0;
    for (int p = warp; p < n_pages; p += W) ++my_pages;
#pragma unroll
    for (int s2 = 0; s2 < D; ++s2) {
      if (s2 < my_pages) issue(warp + s2 * W, s2);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    const int srcA = 8 * t + (g >> 1), srcB = srcA + 4;  // lanes holding tokens 2t / 2t+1 (and +8)
    const bool odd = g & 1;
    for (int i = 0; i < my_pages; ++i) {
      const int sl = i % D;
      const int page_idx = warp + i * W;
      asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
      __syncwarp();
      const uint32_t kb = saddr(k_slot(sl)), vb = saddr(v_slot(sl));
      float sc[4] = {0, 0, 0, 0};  // (tok g, heads 2t|2t+1), (tok g+8, ...)
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        uint32_t a[4];
        ldsm4(kb + swz((lane & 7) + ((lane >> 3) & 1) * 8, kk * 2 + (lane >> 4)), a[0], a[1], a[2], a[3]);
        mma(sc, a, qb[kk][0], qb[kk][1]);
      }
      const int64_t tok0 = static_cast<int64_t>(page_idx) * PAGE;
      const bool v0 = tok0 + g < ctx, v1 = tok0 + g + 8 < ctx;
      float p[4];
      float corr[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float x0 = v0 ? sc[e] * scale_log2 : -FLT_MAX;
        const float x1 = v1 ? sc[2 + e] * scale_log2 : -FLT_MAX;
        float mx = fmaxf(x0, x1);
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
        mx = fmaxf(mx, m_r[e]);
        corr[e] = exp2f(m_r[e] - mx);
        p[e] = exp2f(x0 - mx);
        p[2 + e] = exp2f(x1 - mx);
        l_r[e] = l_r[e] * corr[e] + p[e] + p[2 + e];
        m_r[e] = mx;
      }
      // P^T as the B operand: (tok 2t | 2t+1, head g) and (tok 2t+8 | 2t+9, head g)
      const float a0 = __shfl_sync(0xffffffffu, p[0], srcA), a1 = __shfl_sync(0xffffffffu, p[1], srcA);
      const float a2 = __shfl_sync(0xffffffffu, p[2], srcA), a3 = __shfl_sync(0xffffffffu, p[3], srcA);
      const float b0 = __shfl_sync(0xffffffffu, p[0], srcB), b1 = __shfl_sync(0xffffffffu, p[1], srcB);
      const float b2 = __shfl_sync(0xffffffffu, p[2], srcB), b3 = __shfl_sync(0xffffffffu, p[3], srcB);
      const uint32_t pb0 = pk(odd ? a1 : a0, odd ? b1 : b0);
      const uint32_t pb1 = pk(odd ? a3 : a2, odd ? b3 : b2);
#pragma unroll
      for (int d = 0; d < 8; ++d) {
        o[d][0] *= corr[0];
        o[d][1] *= corr[1];
        o[d][2] *= corr[0];
        o[d][3] *= corr[1];
      }
#pragma unroll
      for (int dm = 0; dm < 8; ++dm) {
        uint32_t a[4];
        ldsm4t(vb + swz((lane & 7) + (lane >> 4) * 8, dm * 2 + ((lane >> 3) & 1)), a[0], a[1], a[2], a[3]);
        mma(o[dm], a, pb0, pb1);
      }
      __syncwarp();
      if (i + D < my_pages) issue(warp + (i + D) * W, sl);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    // ---- merge
    __syncthreads();
    float* sm_m = reinterpret_cast<float*>(smem);  // [W][8]
    float* sm_l = sm_m + W * 8;                     // [W][8]
    float* sm_o = sm_l + W * 8;                     // [W][8][HD]
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      l_r[e] += __shfl_xor_sync(0xffffffffu, l_r[e], 4);
      l_r[e] += __shfl_xor_sync(0xffffffffu, l_r[e], 8);
      l_r[e] += __shfl_xor_sync(0xffffffffu, l_r[e], 16);
    }
    if (g == 0) {
      sm_m[warp * 8 + 2 * t] = m_r[0];
      sm_m[warp * 8 + 2 * t + 1] = m_r[1];
      sm_l[warp * 8 + 2 * t] = l_r[0];
      sm_l[warp * 8 + 2 * t + 1] = l_r[1];
    }
#pragma unroll
    for (int dm = 0; dm < 8; ++dm) {
      sm_o[(warp * 8 + 2 * t) * HD + dm * 16 + g] = o[dm][0];
      sm_o[(warp * 8 + 2 * t + 1) * HD + dm * 16 + g] = o[dm][1];
      sm_o[(warp * 8 + 2 * t) * HD + dm * 16 + g + 8] = o[dm][2];
      sm_o[(warp * 8 + 2 * t + 1) * HD + dm * 16 + g + 8] = o[dm][3];
    }
    __syncthreads();
    float* sm_cur = sm_o + W * 8 * HD;  // [8]
    const __nv_bfloat16* kcur = row + static_cast<int64_t>(nq + kh) * HD;
    const __nv_bfloat16* vcur = row + static_cast<int64_t>(nq + nkv + kh) * HD;
    for (int h = warp; h < G; h += W) {
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
      for (int w = 0; w < W; ++w) M = fmaxf(M, sm_m[w * 8 + h]);
      const float cc = exp2f(sm_cur[h] - M);
      float L = cc, A = cc * __bfloat162float(vcur[d]);
      for (int w = 0; w < W; ++w) {
        if (sm_l[w * 8 + h] == 0.0f) continue;
        const float c = exp2f(sm_m[w * 8 + h] - M);
        L += sm_l[w * 8 + h] * c;
        A += sm_o[(w * 8 + h) * HD + d] * c;
      }
      out[b * static_cast<int64_t>(nq) * HD + static_cast<int64_t>(kh * G + h) * HD + d] = __float2bfloat16(A / L);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ TMA variant
// Same math, decoupled loads: warp 0 (one lane) is a TMA producer streaming the
// (K, V) pages of this CTA's items, in order, into ONE shared ring of kSlots
// 8 KB slots (4 TMA boxes per page: K/V x two 64-dim halves, 128B-swizzled
// [16 tokens][128 B]); consumer warps 1..8 take pages j = w, w+8, ... of the
// current item (slot = running page count mod kSlots), free the slot after
// their MMAs, and merge the 8 partial softmax states at the item's end while
// the producer already streams the next item.  Bytes in flight per SM are the
// whole ring (~190 KB) instead of each warp's 3-page private ring, so fewer
// SMs reach the HBM roofline (the pure-read probe gets 7.4 TB/s from 74 SMs,
// tools/hbm_read_bench.cu) — the SM budget NanoFlow partitioning needs.
constexpr int kTmaCons = 8;                      // consumer warps
constexpr int kTmaThreads = (kTmaCons + 1) * 32;
constexpr int kMaxG = 8;                         // GQA group rows merged
constexpr int kMergeBytes = (kTmaCons * kMaxG * (HD + 2) + kMaxG) * 4;  // m, l, o per warp; current-token scores
constexpr int kSlotBytes = 2 * kPageBytes;       // K + V page
constexpr int kSlots = (227 * 1024 - kMergeBytes - 1024 - 2048) / kSlotBytes;
constexpr int kTmaSmem = 1024 + kSlots * kSlotBytes + kMergeBytes + 1024;

// TMA SW128 image of one page of one kv head: [16 tokens][2 halves][128 B];
// 128 B line L = 2 * token + half, 16 B chunk c stored at c ^ (L & 7)
__device__ __forceinline__ uint32_t swz2(int r, int c16) {
  const int line = 2 * r + (c16 >> 3);
  return static_cast<uint32_t>(line * 128 + (((c16 & 7) ^ (line & 7)) << 4));
}
__device__ __forceinline__ void mbar_init_d(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_wait_d(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma4(uint32_t dst, const CUtensorMap* map, uint32_t bar, int kh, int tok0) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(0), "r"(0), "r"(kh), "r"(tok0)
      : "memory");
}

__global__ void __launch_bounds__(kTmaThreads, 1)
    decode_tma_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
                      const __nv_bfloat16* __restrict__ qkv, const int64_t* __restrict__ table,
                      const int64_t* __restrict__ ctx_len, __nv_bfloat16* __restrict__ out, int nq, int nkv,
                      int64_t max_pages, float scale_log2, int64_t n_items) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* sm_m = reinterpret_cast<float*>(ring + kSlots * kSlotBytes);  // [cons][kMaxG]
  float* sm_l = sm_m + kTmaCons * kMaxG;
  float* sm_o = sm_l + kTmaCons * kMaxG;                                  // [cons][kMaxG][HD]
  float* sm_cur = sm_o + kTmaCons * kMaxG * HD;                           // [kMaxG]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm_cur + kMaxG);
  const uint32_t full0 = saddr(bars), empty0 = saddr(bars + kSlots);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int G = nq / nkv;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlots; ++s) {
      mbar_init_d(full0 + 8 * s, 1);
      mbar_init_d(empty0 + 8 * s, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();

  if (warp == 0) {  // ---------------- producer (whole warp: block-table entries 32 at a time)
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&kmap)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&vmap)) : "memory");
    }
    int64_t g = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int64_t b = item / nkv;
      const int kh = static_cast<int>(item % nkv);
      const int n_pages = static_cast<int>((ctx_len[b] + PAGE - 1) / PAGE);
      const int64_t* trow = table + b * max_pages;
      int64_t nxt = lane < n_pages ? trow[lane] : 0;
      for (int j0 = 0; j0 < n_pages; j0 += 32) {
        const int64_t cur = nxt;
        if (j0 + 32 + lane < n_pages) nxt = trow[j0 + 32 + lane];  // next chunk in flight
        const int cnt = min(32, n_pages - j0);
        for (int i = 0; i < cnt; ++i, ++g) {
          const int tok0 = static_cast<int>(__shfl_sync(0xffffffffu, cur, i) * PAGE);
          if (lane == 0) {
            const int s = static_cast<int>(g % kSlots);
            const uint32_t ph = static_cast<uint32_t>((g / kSlots) & 1);
            mbar_wait_d(empty0 + 8 * s, ph ^ 1);
            const uint32_t dst = saddr(ring + s * kSlotBytes), bar = full0 + 8 * s;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kSlotBytes)
                         : "memory");
            tma4(dst, &kmap, bar, kh, tok0);
            tma4(dst + kPageBytes, &vmap, bar, kh, tok0);
          }
          __syncwarp();
        }
      }
    }
    return;
  }
  // ---------------- consumers (warps 1..8)
  const int cw = warp - 1;
  const int g8 = lane >> 2, t = lane & 3;
  int64_t gbase = 0;  // pages of this CTA's previous items
  for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int64_t b = item / nkv;
    const int kh = static_cast<int>(item % nkv);
    const int64_t W = static_cast<int64_t>(nq + 2 * nkv) * HD;
    const __nv_bfloat16* row = qkv + b * W;
    const int64_t ctx = ctx_len[b];
    const int n_pages = static_cast<int>((ctx + PAGE - 1) / PAGE);
    uint32_t qf[8][4];
    {
      const bool valid = g8 < G;
      const __nv_bfloat16* qrow = row + static_cast<int64_t>(kh * G + (valid ? g8 : 0)) * HD;
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
    for (int j = cw; j < n_pages; j += kTmaCons) {
      const int64_t gp = gbase + j;
      const int s = static_cast<int>(gp % kSlots);
      mbar_wait_d(full0 + 8 * s, static_cast<uint32_t>((gp / kSlots) & 1));
      const uint32_t kb = saddr(ring + s * kSlotBytes), vb = kb + kPageBytes;
      float sc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        uint32_t b0, b1, b2, b3;
        ldsm4(kb + swz2((lane & 7) + (lane >> 4) * 8, kk * 2 + ((lane >> 3) & 1)), b0, b1, b2, b3);
        mma(sc[0], qf[kk], b0, b1);
        mma(sc[1], qf[kk], b2, b3);
      }
      const int64_t tok0 = static_cast<int64_t>(j) * PAGE;
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
#pragma unroll
      for (int dp = 0; dp < 8; ++dp) {
        uint32_t b0, b1, b2, b3;
        ldsm4t(vb + swz2((lane & 7) + ((lane >> 3) & 1) * 8, dp * 2 + (lane >> 4)), b0, b1, b2, b3);
        mma(o[2 * dp], pa, b0, b1);
        mma(o[2 * dp + 1], pa, b2, b3);
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty0 + 8 * s) : "memory");
    }
    gbase += n_pages;
    // ---- merge the 8 partial states (+ the current token) -> out
    l_r += __shfl_xor_sync(0xffffffffu, l_r, 1);
    l_r += __shfl_xor_sync(0xffffffffu, l_r, 2);
    if (g8 < G) {
      if (t == 0) {
        sm_m[cw * kMaxG + g8] = m_r;
        sm_l[cw * kMaxG + g8] = l_r;
      }
#pragma unroll
      for (int d = 0; d < 16; ++d) {
        sm_o[(cw * kMaxG + g8) * HD + d * 8 + 2 * t] = o[d][0];
        sm_o[(cw * kMaxG + g8) * HD + d * 8 + 2 * t + 1] = o[d][1];
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kTmaCons * 32) : "memory");
    const __nv_bfloat16* kcur = row + static_cast<int64_t>(nq + kh) * HD;
    const __nv_bfloat16* vcur = row + static_cast<int64_t>(nq + nkv + kh) * HD;
    for (int h = cw; h < G; h += kTmaCons) {  // current token's score per head
      const __nv_bfloat16* q = row + static_cast<int64_t>(kh * G + h) * HD;
      float dot = 0.0f;
      for (int d = lane; d < HD; d += 32) dot += __bfloat162float(q[d]) * __bfloat162float(kcur[d]);
#pragma unroll
      for (int s2 = 16; s2 > 0; s2 >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, s2);
      if (lane == 0) sm_cur[h] = dot * scale_log2;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kTmaCons * 32) : "memory");
    for (int idx = threadIdx.x - 32; idx < G * HD; idx += kTmaCons * 32) {
      const int h = idx / HD, d = idx % HD;
      const float cur = sm_cur[h];
      float M = cur;
      for (int w = 0; w < kTmaCons; ++w) M = fmaxf(M, sm_m[w * kMaxG + h]);
      const float cc = exp2f(cur - M);
      float L = cc, A = cc * __bfloat162float(vcur[d]);
      for (int w = 0; w < kTmaCons; ++w) {
        if (sm_l[w * kMaxG + h] == 0.0f) continue;
        const float c = exp2f(sm_m[w * kMaxG + h] - M);
        L += sm_l[w * kMaxG + h] * c;
        A += sm_o[(w * kMaxG + h) * HD + d] * c;
      }
      out[b * static_cast<int64_t>(nq) * HD + static_cast<int64_t>(kh * G + h) * HD + d] = __float2bfloat16(A / L);
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kTmaCons * 32) : "memory");  // merge buffers reused next item
  }
}

__device__ __forceinline__ void tma4b(uint32_t dst, const CUtensorMap* map, uint32_t bar, int blk) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %3, %3, %4}], "
      "[%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(0), "r"(blk)
      : "memory");
}

// TMA-fed variant of decode_t_kernel for HND pages (OPF_DECODE=tt): one 4 KB
// TMA per page and tensor (lane 0) instead of 16 cp.async per lane, per-slot
// mbarriers, the same tokens-on-M math.
template <int W, int D>
__global__ void __launch_bounds__(W * 32)
    decode_tt_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
                     const __nv_bfloat16* __restrict__ qkv, const __nv_bfloat16* __restrict__ kc,
                    const __nv_bfloat16* __restrict__ vc, const int64_t* __restrict__ table,
                    const int64_t* __restrict__ ctx_len, __nv_bfloat16* __restrict__ out, int nq, int nkv,
                    int64_t max_pages, float scale_log2, int64_t n_items, int hnd) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int kRing = D * 2 * kPageBytes;
  const uint32_t full0 = saddr(smem + W * kRing);  // [W][D] mbarriers
  if (threadIdx.x < W * D) mbar_init_d(full0 + 8 * threadIdx.x, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  uint32_t issued = 0, consumed = 0;  // this warp's pages, across items (slot = n % D, phase = n / D)
  pdl_wait();
  pdl_trigger();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int g = lane >> 2, t = lane & 3;
  for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int64_t b = item / nkv;
    const int kh = static_cast<int>(item % nkv);
    const int G = nq / nkv;
    const int64_t Wd = static_cast<int64_t>(nq + 2 * nkv) * HD;
    const __nv_bfloat16* row = qkv + b * Wd;
    const int64_t ctx = ctx_len[b];
    const int n_pages = static_cast<int>((ctx + PAGE - 1) / PAGE);
    // NHD pages [16 tokens][nkv][128] (reference / vLLM layout) or HND pages
    // [nkv][16 tokens][128]: one (page, kv head) block is 4 KB contiguous, which
    // DRAM streams ~2-5% faster than 16 rows of 256 B at 2 KB stride
    const int64_t tok_stride = hnd ? HD : static_cast<int64_t>(nkv) * HD;
    const int64_t head_off = hnd ? static_cast<int64_t>(kh) * PAGE * HD : static_cast<int64_t>(kh) * HD;
    uint8_t* ring = smem + warp * kRing;
    auto k_slot = [&](int s) { return ring + s * 2 * kPageBytes; };
    auto v_slot = [&](int s) { return ring + s * 2 * kPageBytes + kPageBytes; };
    auto issue = [&](int page_idx, int) {
      // HND pages: one 4 KB (page, kv head) block per tensor, one TMA each
      const int blk = static_cast<int>(table[b * max_pages + page_idx] * nkv + kh);
      const int s = static_cast<int>(issued % D);
      if (lane == 0) {
        const uint32_t bar = full0 + 8 * (warp * D + s);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(2 * kPageBytes)
                     : "memory");
        tma4b(saddr(k_slot(s)), &kmap, bar, blk);
        tma4b(saddr(v_slot(s)), &vmap, bar, blk);
      }
      ++issued;
    };
    // Q^T as the B operand: n = head g of the group (zero for g >= G), k = dims
    uint32_t qb[8][2];
    {
      const bool valid = g < G;
      const __nv_bfloat16* qrow = row + static_cast<int64_t>(kh * G + (valid ? g : 0)) * HD;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        qb[kk][0] = valid ? *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 2 * t) : 0u;
        qb[kk][1] = valid ? *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 8 + 2 * t) : 0u;
      }
    }
    float o[8][4];  // O^T: [dim tile][(dim g | g+8) x (head 2t | 2t+1)]
#pragma unroll
    for (int d = 0; d < 8; ++d) o[d][0] = o[d][1] = o[d][2] = o[d][3] = 0.0f;
    float m_r[2] = {-FLT_MAX, -FLT_MAX}, l_r[2] = {0.0f, 0.0f};  // heads 2t, 2t+1 (l: this lane's tokens)
    int my_pages = 0;
    for (int p = warp; p < n_pages; p += W) ++my_pages;
#pragma unroll
    for (int s2 = 0; s2 < D; ++s2)
      if (s2 < my_pages) issue(warp + s2 * W, s2);
    const int srcA = 8 * t + (g >> 1), srcB = srcA + 4;  // lanes holding tokens 2t / 2t+1 (and +8)
    const bool odd = g & 1;
    for (int i = 0; i < my_pages; ++i) {
      const int sl = static_cast<int>(consumed % D);
      const int page_idx = warp + i * W;
      mbar_wait_d(full0 + 8 * (warp * D + sl), (consumed / D) & 1u);
      ++consumed;
      const uint32_t kb = saddr(k_slot(sl)), vb = saddr(v_slot(sl));
      float sc[4] = {0, 0, 0, 0};  // (tok g, heads 2t|2t+1), (tok g+8, ...)
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        uint32_t a[4];
        ldsm4(kb + swz2((lane & 7) + ((lane >> 3) & 1) * 8, kk * 2 + (lane >> 4)), a[0], a[1], a[2], a[3]);
        mma(sc, a, qb[kk][0], qb[kk][1]);
      }
      const int64_t tok0 = static_cast<int64_t>(page_idx) * PAGE;
      const bool v0 = tok0 + g < ctx, v1 = tok0 + g + 8 < ctx;
      float p[4];
      float corr[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float x0 = v0 ? sc[e] * scale_log2 : -FLT_MAX;
        const float x1 = v1 ? sc[2 + e] * scale_log2 : -FLT_MAX;
        float mx = fmaxf(x0, x1);
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
        mx = fmaxf(mx, m_r[e]);
        corr[e] = exp2f(m_r[e] - mx);
        p[e] = exp2f(x0 - mx);
        p[2 + e] = exp2f(x1 - mx);
        l_r[e] = l_r[e] * corr[e] + p[e] + p[2 + e];
        m_r[e] = mx;
      }
      // P^T as the B operand: (tok 2t | 2t+1, head g) and (tok 2t+8 | 2t+9, head g)
      const float a0 = __shfl_sync(0xffffffffu, p[0], srcA), a1 = __shfl_sync(0xffffffffu, p[1], srcA);
      const float a2 = __shfl_sync(0xffffffffu, p[2], srcA), a3 = __shfl_sync(0xffffffffu, p[3], srcA);
      const float b0 = __shfl_sync(0xffffffffu, p[0], srcB), b1 = __shfl_sync(0xffffffffu, p[1], srcB);
      const float b2 = __shfl_sync(0xffffffffu, p[2], srcB), b3 = __shfl_sync(0xffffffffu, p[3], srcB);
      const uint32_t pb0 = pk(odd ? a1 : a0, odd ? b1 : b0);
      const uint32_t pb1 = pk(odd ? a3 : a2, odd ? b3 : b2);
#pragma unroll
      for (int d = 0; d < 8; ++d) {
        o[d][0] *= corr[0];
        o[d][1] *= corr[1];
        o[d][2] *= corr[0];
        o[d][3] *= corr[1];
      }
#pragma unroll
      for (int dm = 0; dm < 8; ++dm) {
        uint32_t a[4];
        ldsm4t(vb + swz2((lane & 7) + (lane >> 4) * 8, dm * 2 + ((lane >> 3) & 1)), a[0], a[1], a[2], a[3]);
        mma(o[dm], a, pb0, pb1);
      }
      __syncwarp();
      if (i + D < my_pages) issue(warp + (i + D) * W, sl);
    }
    // ---- merge
    __syncthreads();
    float* sm_m = reinterpret_cast<float*>(smem);  // [W][8]
    float* sm_l = sm_m + W * 8;                     // [W][8]
    float* sm_o = sm_l + W * 8;                     // [W][8][HD]
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      l_r[e] += __shfl_xor_sync(0xffffffffu, l_r[e], 4);
      l_r[e] += __shfl_xor_sync(0xffffffffu, l_r[e], 8);
      l_r[e] += __shfl_xor_sync(0xffffffffu, l_r[e], 16);
    }
    if (g == 0) {
      sm_m[warp * 8 + 2 * t] = m_r[0];
      sm_m[warp * 8 + 2 * t + 1] = m_r[1];
      sm_l[warp * 8 + 2 * t] = l_r[0];
      sm_l[warp * 8 + 2 * t + 1] = l_r[1];
    }
#pragma unroll
    for (int dm = 0; dm < 8; ++dm) {
      sm_o[(warp * 8 + 2 * t) * HD + dm * 16 + g] = o[dm][0];
      sm_o[(warp * 8 + 2 * t + 1) * HD + dm * 16 + g] = o[dm][1];
      sm_o[(warp * 8 + 2 * t) * HD + dm * 16 + g + 8] = o[dm][2];
      sm_o[(warp * 8 + 2 * t + 1) * HD + dm * 16 + g + 8] = o[dm][3];
    }
    __syncthreads();
    float* sm_cur = sm_o + W * 8 * HD;  // [8]
    const __nv_bfloat16* kcur = row + static_cast<int64_t>(nq + kh) * HD;
    const __nv_bfloat16* vcur = row + static_cast<int64_t>(nq + nkv + kh) * HD;
    for (int h = warp; h < G; h += W) {
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
      for (int w = 0; w < W; ++w) M = fmaxf(M, sm_m[w * 8 + h]);
      const float cc = exp2f(sm_cur[h] - M);
      float L = cc, A = cc * __bfloat162float(vcur[d]);
      for (int w = 0; w < W; ++w) {
        if (sm_l[w * 8 + h] == 0.0f) continue;
        const float c = exp2f(sm_m[w * 8 + h] - M);
        L += sm_l[w * 8 + h] * c;
        A += sm_o[(w * 8 + h) * HD + d] * c;
      }
      out[b * static_cast<int64_t>(nq) * HD + static_cast<int64_t>(kh * G + h) * HD + d] = __float2bfloat16(A / L);
    }
    __syncthreads();
  }
}

using EncodeFnD = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

bool cache_map(CUtensorMap* m, const void* base, int nkv, int64_t pages) {
  static EncodeFnD fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeFnD>(nullptr);
    return reinterpret_cast<EncodeFnD>(p);
  }();
  if (!fn) return false;
  // [pages * 16 tokens][nkv heads][2 halves][64 dims] bf16 -> box [16][1][2][64]
  // (one TMA per page per tensor; 128 B lines, SW128)
  const cuuint64_t dims[4] = {64, 2, static_cast<cuuint64_t>(nkv), static_cast<cuuint64_t>(pages * PAGE)};
  const cuuint64_t strides[3] = {128, static_cast<cuuint64_t>(HD) * 2, static_cast<cuuint64_t>(nkv) * HD * 2};
  const cuuint32_t box[4] = {64, 2, 1, PAGE};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool cache_map_hnd(CUtensorMap* m, const void* base, int nkv, int64_t pages) {
  static EncodeFnD fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeFnD>(nullptr);
    return reinterpret_cast<EncodeFnD>(p);
  }();
  if (!fn) return false;
  // HND: [pages * nkv blocks][16 tokens][2 halves][64 dims] -> box [1][16][2][64] (one block)
  const cuuint64_t dims[4] = {64, 2, PAGE, static_cast<cuuint64_t>(pages * nkv)};
  const cuuint64_t strides[3] = {128, 256, static_cast<cuuint64_t>(PAGE) * HD * 2};
  const cuuint32_t box[4] = {64, 2, PAGE, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

template <int W, int D>
bool launch_decode_tt(const __nv_bfloat16* qkv, const __nv_bfloat16* kc, const __nv_bfloat16* vc,
                      const int64_t* table, const int64_t* ctx, __nv_bfloat16* out, int nq, int nkv,
                      int64_t max_pages, int64_t cache_pages, float scale_log2, int64_t items, int64_t grid,
                      cudaStream_t s) {
  constexpr int kSmem = 1024 + W * D * 2 * kPageBytes + 1024;
  static bool attr = cudaFuncSetAttribute(decode_tt_kernel<W, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          kSmem) == cudaSuccess;
  if (!attr) return false;
  CUtensorMap km, vm;
  if (!cache_map_hnd(&km, kc, nkv, cache_pages) || !cache_map_hnd(&vm, vc, nkv, cache_pages)) return false;
  launch_pdl(decode_tt_kernel<W, D>, dim3(static_cast<unsigned>(grid)), dim3(W * 32), kSmem, s, km, vm, qkv, kc, vc,
             table, ctx, out, nq, nkv, max_pages, scale_log2, items, 1);
  return true;
}

template <int W, int D>
bool launch_decode_t(const __nv_bfloat16* qkv, const __nv_bfloat16* kc, const __nv_bfloat16* vc,
                     const int64_t* table, const int64_t* ctx, __nv_bfloat16* out, int nq, int nkv,
                     int64_t max_pages, float scale_log2, int64_t items, int64_t grid, int hnd,
                     cudaStream_t s) {
  constexpr int kSmem = W * D * 2 * kPageBytes;
  static_assert(kSmem >= (W * 8 * (HD + 2) + 8) * 4, "merge buffers fit in the rings");
  static bool attr = cudaFuncSetAttribute(decode_t_kernel<W, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          kSmem) == cudaSuccess;
  if (!attr) return false;
  launch_pdl(decode_t_kernel<W, D>, dim3(static_cast<unsigned>(grid)), dim3(W * 32), kSmem, s, qkv, kc, vc, table,
             ctx, out, nq, nkv, max_pages, scale_log2, items, hnd);
  return true;
}

bool decode_bf16_mma(const __nv_bfloat16* qkv, const __nv_bfloat16* kc, const __nv_bfloat16* vc,
                     const int64_t* table, const int64_t* ctx, __nv_bfloat16* out, int64_t B, int nq,
                     int nkv, int hd, int page, int64_t max_pages, float scale, int max_ctas, int hnd,
                     int64_t cache_pages, cudaStream_t s) {
  if (hd != HD || page != PAGE || nq % nkv != 0 || nq / nkv > 8) return false;
  // OPF_DECODE: t12x2 (default) | t8x3 | mma16 (group padded to M = 16)
  static const int variant = [] {
    const char* e = std::getenv("OPF_DECODE");
    if (e && std::string(e) == "mma16") return 0;
    if (e && std::string(e) == "t8x3") return 1;
    if (e && std::string(e) == "t14x2") return 3;
    if (e && std::string(e) == "t16x1") return 4;
    if (e && std::string(e) == "t6x4") return 5;
    if (e && std::string(e) == "tt") return 6;
    return 2;
  }();
  const int64_t items = B * nkv;
  int64_t grid = max_ctas > 0 ? std::min<int64_t>(max_ctas, num_sms()) : num_sms();
  grid = std::max<int64_t>(1, std::min(grid, items));
  const float sl2 = scale * 1.4426950408889634f;
  if (variant == 6 && hnd && (reinterpret_cast<uintptr_t>(kc) | reinterpret_cast<uintptr_t>(vc)) % 16 == 0)
    return launch_decode_tt<12, 2>(qkv, kc, vc, table, ctx, out, nq, nkv, max_pages, cache_pages, sl2, items, grid,
                                   s);
  if (variant == 1) return launch_decode_t<8, 3>(qkv, kc, vc, table, ctx, out, nq, nkv, max_pages, sl2, items, grid, hnd, s);
  if (variant == 2) return launch_decode_t<12, 2>(qkv, kc, vc, table, ctx, out, nq, nkv, max_pages, sl2, items, grid, hnd, s);
  if (variant == 3) return launch_decode_t<14, 2>(qkv, kc, vc, table, ctx, out, nq, nkv, max_pages, sl2, items, grid, hnd, s);
  if (variant == 4) return launch_decode_t<16, 1>(qkv, kc, vc, table, ctx, out, nq, nkv, max_pages, sl2, items, grid, hnd, s);
  if (variant == 5) return launch_decode_t<6, 4>(qkv, kc, vc, table, ctx, out, nq, nkv, max_pages, sl2, items, grid, hnd, s);
  static bool attr = [] {
    return cudaFuncSetAttribute(decode_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kSmemRing) == cudaSuccess;
  }();
  if (!attr || hnd) return false;  // the M = 16 kernel reads NHD pages only
  launch_pdl(decode_mma_kernel, dim3(static_cast<unsigned>(grid)), dim3(kWarps * 32), kSmemRing, s,
             qkv, kc, vc, table, ctx, out, nq, nkv, max_pages, sl2, items);
  return true;
}

// TMA-ring variant (opt-in with OPF_DECODE=tma; the per-warp cp.async rings are the default)
bool decode_bf16_tma(const __nv_bfloat16* qkv, const __nv_bfloat16* kc, const __nv_bfloat16* vc,
                     const int64_t* table, const int64_t* ctx, __nv_bfloat16* out, int64_t B, int nq, int nkv,
                     int hd, int page, int64_t max_pages, int64_t cache_pages, float scale, int max_ctas,
                     cudaStream_t s) {
  static const bool off = [] {
    const char* e = std::getenv("OPF_DECODE");
    return !(e && std::string(e) == "tma");  // opt-in: measured slower than the per-warp rings (see DESIGN)
  }();
  if (off || hd != HD || page != PAGE || nq % nkv != 0 || nq / nkv > kMaxG) return false;
  if ((reinterpret_cast<uintptr_t>(kc) | reinterpret_cast<uintptr_t>(vc)) % 16) return false;
  static bool attr = [] {
    return cudaFuncSetAttribute(decode_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem) ==
           cudaSuccess;
  }();
  if (!attr) return false;
  CUtensorMap km, vm;
  if (!cache_map(&km, kc, nkv, cache_pages) || !cache_map(&vm, vc, nkv, cache_pages)) return false;
  const int64_t items = B * nkv;
  int64_t grid = max_ctas > 0 ? std::min<int64_t>(max_ctas, num_sms()) : num_sms();
  grid = std::max<int64_t>(1, std::min(grid, items));
  launch_pdl(decode_tma_kernel, dim3(static_cast<unsigned>(grid)), dim3(kTmaThreads), kTmaSmem, s, km, vm, qkv,
             table, ctx, out, nq, nkv, max_pages, scale * 1.4426950408889634f, items);
  return true;
}

}  // namespace opflow
