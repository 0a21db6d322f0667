// Paged decode attention on tensor cores (the memory-bound hot kernel of the
// decode config, BASELINE configs[3]).  qkv_rot [B, (nq+2nkv)*128] holds the
// current token; the K/V caches are paged ([pages, 16, nkv, 128] NHD or
// [pages, nkv, 16, 128] HND, bf16) with a per-sequence block table; each
// sequence attends to its `ctx` cached tokens plus itself.
//
// One (sequence, kv head) item per CTA — or, under an explicit SM budget, a
// persistent grid of the budget walking the items — so every K/V byte is read
// once.  Warp w of W streams pages w, w+W, ... (16
// tokens x 256 B of K and of V each) with cp.async into its private D-deep ring
// (XOR-swizzled).  Tokens sit on the MMA M dimension and the GQA group on N:
// S^T = K Q^T and O^T += V^T P^T are 8 + 8 mma.sync m16n8k16 per page, so the
// kernel is HBM-bound (tcgen05 has no use at N = 8 GQA rows).  Online softmax in
// fp32 on the fragments; the W warps' (m, l, O) and the current token merge in
// shared memory.  Algorithmic bytes per (sequence, kv head) = 2 * ctx * 128 * 2.
//
// Shipped shapes: W = 6 warps, D = 2 pages per warp (96 KB of rings, 165
// registers), two CTAs per SM, one item each; under an explicit SM budget
// (NanoFlow lane partitions) W = 12, one persistent CTA per SM.  0.97 of the
// measured HBM read peak at 512 x 4K.  Measured losers (an M = 16 padded-group kernel, a shared TMA
// ring, TMA-fed per-warp rings, other W x D shapes, and the co-resident 4/8-warp
// shapes of commit 7418aec) live in the git history and DESIGN §5.1 / §8.
#include <cuda.h>
#include <cuda_bf16.h>

#include <cfloat>
#include <cstdlib>
#include <string>

#include "opflow/device.hpp"

namespace opflow {

namespace {

constexpr int HD = 128;
constexpr int PAGE = 16;
constexpr int kPageBytes = PAGE * HD * 2;  // 4 KB (one tensor, one page, one kv head)

__device__ __forceinline__ uint32_t saddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t swz(int r, int c) {
  return static_cast<uint32_t>(r * (HD * 2) + ((c ^ (r & 7)) << 4));
}
__device__ __forceinline__ void cp16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
// KV bytes are read exactly once per step: mark their L2 lines evict-first so
// the 8.6 GB/layer stream does not evict the operands a concurrent GEMM (the
// other nano-batch's projections) re-reads across its N tiles.
__device__ __forceinline__ void cp16_ef(uint32_t dst, const void* src, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "l"(pol)
               : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
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

// Tokens on the MMA M dimension, the GQA group on N (8): S^T[16 tok x 8 heads]
// = K[16 x 128] Q^T and O^T[128 dims x 8 heads] += V^T P^T — 8 + 8 m16n8k16
// per page, a 32-float accumulator.  P^T reaches the B-fragment layout through 8
// shuffles; the softmax reduces over tokens (lane bits 2..4).  W warps with
// D-deep private cp.async page rings (W x D x 8 KB of smem).
template <int W, int D, int MinBlocks, bool EF>
__global__ void __launch_bounds__(W * 32, MinBlocks)
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
  const uint64_t pol = EF ? evict_first_policy() : 0;
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
        if constexpr (EF) {
          cp16_ef(kd + swz(r, c), kp + r * tok_stride + c * 8, pol);
          cp16_ef(vd + swz(r, c), vp + r * tok_stride + c * 8, pol);
        } else {
          cp16(kd + swz(r, c), kp + r * tok_stride + c * 8);
          cp16(vd + swz(r, c), vp + r * tok_stride + c * 8);
        }
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

}  // namespace

template <int W, int D, int MinBlocks, bool EF>
bool launch_decode_t(const __nv_bfloat16* qkv, const __nv_bfloat16* kc, const __nv_bfloat16* vc,
                     const int64_t* table, const int64_t* ctx, __nv_bfloat16* out, int nq, int nkv,
                     int64_t max_pages, float scale_log2, int64_t items, int64_t grid, int hnd,
                     cudaStream_t s) {
  constexpr int kSmem = W * D * 2 * kPageBytes;
  static_assert(kSmem >= (W * 8 * (HD + 2) + 8) * 4, "merge buffers fit in the rings");
  static bool attr = cudaFuncSetAttribute(decode_t_kernel<W, D, MinBlocks, EF>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem) == cudaSuccess &&
                     cudaFuncSetAttribute(decode_t_kernel<W, D, MinBlocks, EF>,
                                          cudaFuncAttributePreferredSharedMemoryCarveout, 100) == cudaSuccess;
  if (!attr) return false;
  launch_pdl(decode_t_kernel<W, D, MinBlocks, EF>, dim3(static_cast<unsigned>(grid)), dim3(W * 32), kSmem, s, qkv,
             kc, vc, table, ctx, out, nq, nkv, max_pages, scale_log2, items, hnd);
  return true;
}

bool decode_bf16_mma(const __nv_bfloat16* qkv, const __nv_bfloat16* kc, const __nv_bfloat16* vc,
                     const int64_t* table, const int64_t* ctx, __nv_bfloat16* out, int64_t B, int nq,
                     int nkv, int hd, int page, int64_t max_pages, float scale, int max_ctas, int hnd,
                     cudaStream_t s) {
  if (hd != HD || page != PAGE || nq % nkv != 0 || nq / nkv > 8) return false;
  const int64_t items = B * nkv;
  const int64_t grid = max_ctas > 0 ? std::min<int64_t>(max_ctas, num_sms()) : num_sms();  // SM budget
  const float sl2 = scale * 1.4426950408889634f;
  static const bool ef = [] {
    const char* e = std::getenv("OPF_DECODE_L2");  // "normal": plain cp.async (A/B switch)
    return !(e && std::string(e) == "normal");
  }();
  // An explicit SM budget (a NanoFlow lane partition) keeps the persistent
  // form, one 12-warp CTA per SM, so the CTA count bounds the SMs the lane
  // occupies.  Otherwise one (sequence, kv head) item per CTA of 6 warps
  // (96 KB of rings, two per SM) and the hardware scheduler refills an SM as
  // soon as one of its CTAs finishes: no round quantisation, and a new item's
  // ring fill overlaps the other CTA's streaming.  Same box, 512 x 4K: the
  // persistent 12-warp form 1229 us, persistent 6-warp x 2 per SM 1223 us,
  // one item per CTA 1189 us (7.22 TB/s, 0.97 of the read peak); TP=8 per-rank
  // shape 170 / 159 / 159 us (profiles/r02_decode_half_cta_ab.txt).
  if (max_ctas > 0) {
    const int64_t g1 = std::max<int64_t>(1, std::min<int64_t>(grid, items));
    if (ef)
      return launch_decode_t<12, 2, 1, true>(qkv, kc, vc, table, ctx, out, nq, nkv, max_pages, sl2, items, g1, hnd, s);
    return launch_decode_t<12, 2, 1, false>(qkv, kc, vc, table, ctx, out, nq, nkv, max_pages, sl2, items, g1, hnd, s);
  }
  const int64_t g2 = std::max<int64_t>(1, items);
  if (ef)
    return launch_decode_t<6, 2, 2, true>(qkv, kc, vc, table, ctx, out, nq, nkv, max_pages, sl2, items, g2, hnd, s);
  return launch_decode_t<6, 2, 2, false>(qkv, kc, vc, table, ctx, out, nq, nkv, max_pages, sl2, items, g2, hnd, s);
}

}  // namespace opflow
