// Attention ops for the Llama-shaped graphs.
//
//  attn_decode  (memory-bound, the north star's paged decode attention)
//    qkv_rot [B, (nq+2nkv)*hd], k_cache / v_cache [pages, page, nkv, hd],
//    block_table [B, max_pages] (i64), ctx_len [B] (i64) -> out [B, nq*hd].
//    One CTA per (sequence, kv head) serves the whole GQA group, so every
//    cached K/V byte is read from HBM exactly once: algorithmic bytes per
//    (sequence, kv head) = 2 * ctx * hd * 2 B.  Each token's K (or V) row is
//    256 contiguous bytes read by 16 lanes with 16-byte loads; a warp covers
//    two tokens per step and four steps are kept in flight (8 x 16 B per lane).
//    Online softmax in fp32; the 4 warps' partial states merge in smem.
//
//  attn_prefill (causal GQA within fixed-length sequences; SIMT reference
//    path here, tensor-core path in attention_tc.cu).
#include <cuda_bf16.h>

#include <cfloat>
#include <cstdlib>
#include <string>

#include "opflow/device.hpp"

namespace opflow {

namespace {

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16(v); }

// ---------------------------------------------------------------- prefill (SIMT)
// One warp per (row, q head); lanes split head_dim.  Correctness path for fp32
// graphs and the numerics reference of the tensor-core kernel.
template <typename T>
__global__ void prefill_simt_kernel(const T* __restrict__ qkv, T* __restrict__ out, int64_t rows,
                                    int nq, int nkv, int hd, int S, float scale) {
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (gw >= rows * nq) return;
  const int64_t r = gw / nq;
  const int h = static_cast<int>(gw % nq), kh = h / (nq / nkv);
  const int64_t W = static_cast<int64_t>(nq + 2 * nkv) * hd;
  const int64_t s0 = r - r % S;
  constexpr int MAXD = 8;  // hd <= 256
  float q[MAXD], acc[MAXD];
#pragma unroll
  for (int i = 0; i < MAXD; ++i) {
    const int d = lane + 32 * i;
    q[i] = d < hd ? to_f(qkv[r * W + h * hd + d]) * scale : 0.0f;
    acc[i] = 0.0f;
  }
  float m = -FLT_MAX, l = 0.0f;
  for (int64_t j = s0; j <= r; ++j) {
    const T* k = qkv + j * W + static_cast<int64_t>(nq + kh) * hd;
    float dot = 0.0f;
#pragma unroll
    for (int i = 0; i < MAXD; ++i) {
      const int d = lane + 32 * i;
      if (d < hd) dot += q[i] * to_f(k[d]);
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, s);
    const float mn = fmaxf(m, dot);
    const float corr = expf(m - mn), p = expf(dot - mn);
    l = l * corr + p;
    const T* v = qkv + j * W + static_cast<int64_t>(nq + nkv + kh) * hd;
#pragma unroll
    for (int i = 0; i < MAXD; ++i) {
      const int d = lane + 32 * i;
      acc[i] = acc[i] * corr + (d < hd ? p * to_f(v[d]) : 0.0f);
    }
    m = mn;
  }
#pragma unroll
  for (int i = 0; i < MAXD; ++i) {
    const int d = lane + 32 * i;
    if (d < hd) out[r * nq * hd + h * hd + d] = from_f<T>(acc[i] / l);
  }
}

// ------------------------------------------------- prefill (fp32, short sequences)
// One CTA per (sequence, q head, row slice): the sequence's K and V rows of
// the head's kv head staged once in shared memory (K rows padded to hd + 1
// floats so lanes reading different keys hit different banks).  Each warp
// takes query rows; per row the lanes split the keys (scores for keys
// lane, lane + 32, ... <= row), one warp max / sum gives the softmax, the
// probabilities go through a per-warp shared buffer and the lanes split
// head_dim for P V.  Exact two-pass softmax per row (the SIMT kernel above
// is online); both are within the fp32 tolerance of the fp64 oracle.  Used
// when S <= 256, hd <= 128 and K / V fit in shared memory (the C1 toy:
// S = 128, hd = 64).
constexpr int kSmallWarps = 8;
template <int MAXT>
__global__ void __launch_bounds__(kSmallWarps * 32) prefill_small_f32_kernel(
    const float* __restrict__ qkv, float* __restrict__ out, int nq, int nkv, int hd, int S, float scale,
    int slices) {
  extern __shared__ __align__(16) float sm[];
  const int hdp = hd + 4;  // K row stride: 16-byte aligned, and 8 lanes' float4 reads of 8 rows hit 8 bank quads
  const int S4 = (S + 3) & ~3;
  float* ks = sm;                                  // [S][hd + 4]
  float* vs = ks + static_cast<int64_t>(S) * hdp;  // [S rounded up to 4][hd], rows past `last` zero
  float* qs = vs + static_cast<int64_t>(S4) * hd;  // [warps][hd]
  float* ps = qs + kSmallWarps * hd;               // [warps][S rounded up to 4]
  const int seq = blockIdx.x / nq, h = blockIdx.x % nq, slice = blockIdx.y;
  const int kh = h / (nq / nkv);
  const int64_t W = static_cast<int64_t>(nq + 2 * nkv) * hd;
  const float* base = qkv + static_cast<int64_t>(seq) * S * W;
  // rows this CTA handles: slice, slice + slices, ...; keys needed: 0..last row
  const int last = slice + ((S - 1 - slice) / slices) * slices;
  const int hd4 = hd / 4;
  for (int i = threadIdx.x; i < S4 * hd4; i += blockDim.x) {
    const int j = i / hd4, d = (i % hd4) * 4;
    if (j <= last) {
      const float* row = base + j * W;
      *reinterpret_cast<float4*>(ks + j * hdp + d) =
          *reinterpret_cast<const float4*>(row + static_cast<int64_t>(nq + kh) * hd + d);
      *reinterpret_cast<float4*>(vs + j * hd + d) =
          *reinterpret_cast<const float4*>(row + static_cast<int64_t>(nq + nkv + kh) * hd + d);
    } else {  // P V reads whole float4s of p: the rows it touches past the last key must be finite (zero)
      *reinterpret_cast<float4*>(vs + j * hd + d) = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    }
  }
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  float* q = qs + warp * hd;
  float* p = ps + warp * S4;
  for (int r = slice + warp * slices; r < S; r += kSmallWarps * slices) {
    for (int d = lane * 4; d < hd; d += 128) {
      float4 v = *reinterpret_cast<const float4*>(base + r * W + static_cast<int64_t>(h) * hd + d);
      v.x *= scale, v.y *= scale, v.z *= scale, v.w *= scale;
      *reinterpret_cast<float4*>(q + d) = v;
    }
    __syncwarp();
    float sc[MAXT];
    float m = -FLT_MAX;
#pragma unroll
    for (int t = 0; t < MAXT; ++t) {
      const int j = lane + 32 * t;
      float dot = -FLT_MAX;
      if (j <= r) {
        dot = 0.0f;
        const float* kr = ks + j * hdp;
        for (int d = 0; d < hd; d += 4) {
          const float4 q4 = *reinterpret_cast<const float4*>(q + d);  // broadcast
          const float4 k4 = *reinterpret_cast<const float4*>(kr + d);
          dot += q4.x * k4.x + q4.y * k4.y + q4.z * k4.z + q4.w * k4.w;
        }
      }
      sc[t] = dot;
      m = fmaxf(m, dot);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float l = 0.0f;
#pragma unroll
    for (int t = 0; t < MAXT; ++t) {
      const int j = lane + 32 * t;
      if (j < S4) {  // keys past the row (and the pad to 4) get probability 0
        const float e = j <= r ? expf(sc[t] - m) : 0.0f;
        l += e;
        p[j] = e;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    __syncwarp();
    const float inv = 1.0f / l;
    const int jn = (r + 4) & ~3;  // keys 0..r, rounded up to whole float4s of p (zeros past r)
    for (int d = lane; d < hd; d += 32) {
      float acc = 0.0f;
      for (int j = 0; j < jn; j += 4) {
        const float4 p4 = *reinterpret_cast<const float4*>(p + j);  // broadcast
        acc += p4.x * vs[j * hd + d];
        acc += p4.y * vs[(j + 1) * hd + d];
        acc += p4.z * vs[(j + 2) * hd + d];
        acc += p4.w * vs[(j + 3) * hd + d];
      }
      out[(static_cast<int64_t>(seq) * S + r) * nq * hd + static_cast<int64_t>(h) * hd + d] = acc * inv;
    }
    __syncwarp();  // q / p of this row are read before the next row overwrites them
  }
}

// ---------------------------------------------------------------- decode (paged)
constexpr int kDecWarps = 4;
constexpr int kMaxGroup = 8;   // q heads per kv head
constexpr int kUnroll = 4;     // token pairs in flight per warp

template <int GRP>
__global__ void __launch_bounds__(kDecWarps * 32) decode_bf16_kernel(
    const __nv_bfloat16* __restrict__ qkv, const __nv_bfloat16* __restrict__ kc,
    const __nv_bfloat16* __restrict__ vc, const int64_t* __restrict__ table,
    const int64_t* __restrict__ ctx_len, __nv_bfloat16* __restrict__ out, int nq, int nkv,
    int64_t max_pages, int page, float scale) {
  constexpr int HD = 128;  // 16 lanes x 8 bf16
  const int64_t b = blockIdx.x / nkv;
  const int kh = blockIdx.x % nkv;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int half = lane / 16, sub = lane % 16;  // token parity, 16-byte chunk index
  const int64_t W = static_cast<int64_t>(nq + 2 * nkv) * HD;
  const int64_t ctx = ctx_len[b];
  const int64_t total = ctx + 1;  // cached tokens + the current one
  const __nv_bfloat16* row = qkv + b * W;

  float q[GRP][8];
#pragma unroll
  for (int g = 0; g < GRP; ++g) {
    const uint4 u = *reinterpret_cast<const uint4*>(row + (kh * GRP + g) * HD + sub * 8);
    const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h2[i]);
      q[g][2 * i] = f.x * scale;
      q[g][2 * i + 1] = f.y * scale;
    }
  }
  float m[GRP], l[GRP], acc[GRP][8];
#pragma unroll
  for (int g = 0; g < GRP; ++g) {
    m[g] = -FLT_MAX;
    l[g] = 0.0f;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[g][i] = 0.0f;
  }
  const int64_t kv_stride = static_cast<int64_t>(nkv) * HD;
  auto kv_ptr = [&](const __nv_bfloat16* cache, const __nv_bfloat16* cur, int64_t j) {
    if (j == ctx) return cur;
    const int64_t pg = table[b * max_pages + j / page];
    return cache + (pg * page + j % page) * kv_stride + static_cast<int64_t>(kh) * HD;
  };
  const __nv_bfloat16* kcur = row + static_cast<int64_t>(nq + kh) * HD;
  const __nv_bfloat16* vcur = row + static_cast<int64_t>(nq + nkv + kh) * HD;

  // token j handled by (warp, half) = ((j/2) % kDecWarps, j % 2)
  for (int64_t base = 2 * warp; base < total; base += 2 * kDecWarps * kUnroll) {
    uint4 kr[kUnroll], vr[kUnroll];
    bool ok[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t j = base + static_cast<int64_t>(u) * 2 * kDecWarps + half;
      ok[u] = j < total;
      if (ok[u]) {
        kr[u] = __ldg(reinterpret_cast<const uint4*>(kv_ptr(kc, kcur, j) + sub * 8));
        vr[u] = __ldg(reinterpret_cast<const uint4*>(kv_ptr(vc, vcur, j) + sub * 8));
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      float kf[8], vf[8];
      const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&kr[u]);
      const __nv_bfloat162* v2 = reinterpret_cast<const __nv_bfloat162*>(&vr[u]);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 a = __bfloat1622float2(k2[i]), c = __bfloat1622float2(v2[i]);
        kf[2 * i] = a.x;
        kf[2 * i + 1] = a.y;
        vf[2 * i] = c.x;
        vf[2 * i + 1] = c.y;
      }
#pragma unroll
      for (int g = 0; g < GRP; ++g) {
        float s = 0.0f;
#pragma unroll
        for (int i = 0; i < 8; ++i) s += q[g][i] * kf[i];
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);  // within 16 lanes
        if (ok[u]) {
          const float mn = fmaxf(m[g], s);
          const float corr = __expf(m[g] - mn), p = __expf(s - mn);
          l[g] = l[g] * corr + p;
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[g][i] = acc[g][i] * corr + p * vf[i];
          m[g] = mn;
        }
      }
    }
  }
  // merge the two half-warps, then the warps, through shared memory
  __shared__ float sm_m[kDecWarps * 2][GRP], sm_l[kDecWarps * 2][GRP];
  __shared__ float sm_acc[kDecWarps * 2][GRP][HD];
  const int slot = warp * 2 + half;
#pragma unroll
  for (int g = 0; g < GRP; ++g) {
    if (sub == 0) {
      sm_m[slot][g] = m[g];
      sm_l[slot][g] = l[g];
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) sm_acc[slot][g][sub * 8 + i] = acc[g][i];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < GRP * HD; idx += blockDim.x) {
    const int g = idx / HD, d = idx % HD;
    float M = -FLT_MAX;
    for (int sl = 0; sl < kDecWarps * 2; ++sl) M = fmaxf(M, sm_m[sl][g]);
    float L = 0.0f, A = 0.0f;
    for (int sl = 0; sl < kDecWarps * 2; ++sl) {
      if (sm_l[sl][g] == 0.0f) continue;
      const float c = __expf(sm_m[sl][g] - M);
      L += sm_l[sl][g] * c;
      A += sm_acc[sl][g][d] * c;
    }
    out[b * static_cast<int64_t>(nq) * HD + (kh * GRP + g) * HD + d] = __float2bfloat16(A / L);
  }
}

// Generic (any dtype / head_dim) decode: one warp per (sequence, q head).
template <typename T>
__global__ void decode_simt_kernel(const T* __restrict__ qkv, const T* __restrict__ kc,
                                   const T* __restrict__ vc, const int64_t* __restrict__ table,
                                   const int64_t* __restrict__ ctx_len, T* __restrict__ out,
                                   int64_t B, int nq, int nkv, int hd, int64_t max_pages, int page,
                                   float scale) {
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (gw >= B * nq) return;
  const int64_t b = gw / nq;
  const int h = static_cast<int>(gw % nq), kh = h / (nq / nkv);
  const int64_t W = static_cast<int64_t>(nq + 2 * nkv) * hd, ctx = ctx_len[b];
  constexpr int MAXD = 8;
  float q[MAXD], acc[MAXD];
#pragma unroll
  for (int i = 0; i < MAXD; ++i) {
    const int d = lane + 32 * i;
    q[i] = d < hd ? to_f(qkv[b * W + h * hd + d]) * scale : 0.0f;
    acc[i] = 0.0f;
  }
  float m = -FLT_MAX, l = 0.0f;
  for (int64_t j = 0; j <= ctx; ++j) {
    const T *k, *v;
    if (j == ctx) {
      k = qkv + b * W + static_cast<int64_t>(nq + kh) * hd;
      v = qkv + b * W + static_cast<int64_t>(nq + nkv + kh) * hd;
    } else {
      const int64_t pg = table[b * max_pages + j / page];
      const int64_t off = ((pg * page + j % page) * nkv + kh) * static_cast<int64_t>(hd);
      k = kc + off;
      v = vc + off;
    }
    float dot = 0.0f;
#pragma unroll
    for (int i = 0; i < MAXD; ++i) {
      const int d = lane + 32 * i;
      if (d < hd) dot += q[i] * to_f(k[d]);
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, s);
    const float mn = fmaxf(m, dot), corr = expf(m - mn), p = expf(dot - mn);
    l = l * corr + p;
#pragma unroll
    for (int i = 0; i < MAXD; ++i) {
      const int d = lane + 32 * i;
      acc[i] = acc[i] * corr + (d < hd ? p * to_f(v[d]) : 0.0f);
    }
    m = mn;
  }
#pragma unroll
  for (int i = 0; i < MAXD; ++i) {
    const int d = lane + 32 * i;
    if (d < hd) out[b * nq * hd + h * hd + d] = from_f<T>(acc[i] / l);
  }
}

}  // namespace

// attention_decode.cu (tensor-core paged decode); false when unsupported.
bool decode_bf16_mma(const __nv_bfloat16* qkv, const __nv_bfloat16* kc, const __nv_bfloat16* vc,
                     const int64_t* table, const int64_t* ctx, __nv_bfloat16* out, int64_t B, int nq,
                     int nkv, int hd, int page, int64_t max_pages, float scale, int max_ctas, int hnd,
                     cudaStream_t s);

// implemented in attention_tc.cu (tensor-core prefill); returns false when the
// shape is not supported there.
bool prefill_bf16_tc(const __nv_bfloat16* qkv, __nv_bfloat16* out, int64_t rows, int nq, int nkv,
                     int hd, int S, float scale, cudaStream_t s);
// attention_fa_tc.cu: tcgen05/TMEM flash attention (hd 128, S % 128 == 0)
bool prefill_bf16_tcgen05(const __nv_bfloat16* qkv, __nv_bfloat16* out, int64_t rows, int nq, int nkv,
                          int hd, int S, float scale, int max_ctas, cudaStream_t s);

opf_status attn_prefill_simt(const opf_view& in, opf_view& out, int64_t rows, int nq, int nkv,
                             int hd, int S, cudaStream_t s) {
  const float scale = 1.0f / sqrtf(static_cast<float>(hd));
  const size_t small_smem =
      (static_cast<size_t>(S) * (hd + 4) + static_cast<size_t>((S + 3) & ~3) * hd +
       static_cast<size_t>(kSmallWarps) * (hd + ((S + 3) & ~3))) * sizeof(float);
  if (in.dtype == OPF_F32 && S <= 256 && hd <= 128 && hd % 4 == 0 && small_smem <= 200 * 1024 &&
      (reinterpret_cast<uintptr_t>(vptr<float>(in)) | reinterpret_cast<uintptr_t>(vptr<float>(out))) % 16 == 0) {
    // enough CTAs for the SMs: split each (sequence, head)'s rows into slices
    const int64_t units = (rows / S) * nq;
    int slices = 1;
    while (slices < 16 && units * slices < 2 * num_sms() && S / (slices * 2) >= kSmallWarps) slices *= 2;
    const dim3 grid(static_cast<unsigned>(units), static_cast<unsigned>(slices));
    static const bool attr_ok = [] {  // every instantiation (they share one function-pointer type)
      bool ok = true;
      for (auto k : {prefill_small_f32_kernel<2>, prefill_small_f32_kernel<4>, prefill_small_f32_kernel<8>})
        ok = ok && cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) == cudaSuccess;
      return ok;
    }();
    if (!attr_ok) return op_error(Errc::SchedulerError, "attn_prefill_small_f32: shared-memory attribute");
    auto launch = [&](auto kern) {
      kern<<<grid, kSmallWarps * 32, small_smem, s>>>(vptr<float>(in), vptr<float>(out), nq, nkv, hd, S, scale,
                                                      slices);
    };
    if (S <= 64)
      launch(prefill_small_f32_kernel<2>);
    else if (S <= 128)
      launch(prefill_small_f32_kernel<4>);
    else
      launch(prefill_small_f32_kernel<8>);
    return launch_status("attn_prefill_small_f32");
  }
  const int64_t warps = rows * nq;
  const int threads = 128;
  const unsigned grid = static_cast<unsigned>((warps * 32 + threads - 1) / threads);
  if (in.dtype == OPF_BF16)
    prefill_simt_kernel<__nv_bfloat16><<<grid, threads, 0, s>>>(
        vptr<__nv_bfloat16>(in), vptr<__nv_bfloat16>(out), rows, nq, nkv, hd, S, scale);
  else
    prefill_simt_kernel<float><<<grid, threads, 0, s>>>(vptr<float>(in), vptr<float>(out), rows, nq,
                                                        nkv, hd, S, scale);
  return launch_status("attn_prefill_simt");
}

namespace {

opf_status op_attn_prefill(const opf_op_ctx* c, const opf_view* in, int32_t n_in, opf_view* out,
                           int32_t n_out, int64_t rows, void* stream) {
  if (n_in != 1 || n_out != 1) return op_error(Errc::ShapeMismatch, "attn_prefill takes (qkv) -> o");
  const int nq = static_cast<int>(ctx_param(*c, "heads", 1));
  const int nkv = static_cast<int>(ctx_param(*c, "kv_heads", 1));
  const int hd = static_cast<int>(ctx_param(*c, "head_dim", 128));
  const int S = static_cast<int>(ctx_param(*c, "seq_len", 1));
  if (nq % nkv || hd > 256) return op_error(Errc::ShapeMismatch, "attn_prefill: heads");
  if (view_row_elems(in[0]) != static_cast<int64_t>(nq + 2 * nkv) * hd ||
      view_row_elems(out[0]) != static_cast<int64_t>(nq) * hd)
    return op_error(Errc::ShapeMismatch, "attn_prefill: widths");
  if (rows % S)
    return op_error(Errc::ShapeMismatch, "attn_prefill: rows " + std::to_string(rows) +
                                             " not a multiple of seq_len " + std::to_string(S));
  if (rows == 0) return 0;
  auto s = static_cast<cudaStream_t>(stream);
  // impl: 0 auto (tcgen05 -> mma.sync -> SIMT), 1 mma.sync FA2, 2 SIMT; OPF_PREFILL=fa2|simt overrides auto
  static const int env_impl = [] {
    const char* e = std::getenv("OPF_PREFILL");
    if (!e) return 0;
    return std::string(e) == "fa2" ? 1 : std::string(e) == "simt" ? 2 : 0;
  }();
  int impl = static_cast<int>(ctx_param(*c, "impl", 0.0));
  if (ctx_param(*c, "simt", 0.0) != 0.0) impl = 2;
  if (impl == 0) impl = env_impl;
  const float scale = 1.0f / sqrtf(static_cast<float>(hd));
  if (in[0].dtype == OPF_BF16 && impl == 0 &&
      prefill_bf16_tcgen05(vptr<__nv_bfloat16>(in[0]), vptr<__nv_bfloat16>(out[0]), rows, nq, nkv, hd, S,
                           scale, c->max_ctas, s))
    return launch_status("attn_prefill_tcgen05");
  if (in[0].dtype == OPF_BF16 && impl <= 1 &&
      prefill_bf16_tc(vptr<__nv_bfloat16>(in[0]), vptr<__nv_bfloat16>(out[0]), rows, nq, nkv, hd, S,
                      scale, s))
    return launch_status("attn_prefill_tc");
  return attn_prefill_simt(in[0], out[0], rows, nq, nkv, hd, S, s);
}

opf_status op_attn_decode(const opf_op_ctx* c, const opf_view* in, int32_t n_in, opf_view* out,
                          int32_t n_out, int64_t rows, void* stream) {
  if (n_in != 5 || n_out != 1)
    return op_error(Errc::ShapeMismatch, "attn_decode takes (qkv, k_cache, v_cache, table, ctx)");
  const int nq = static_cast<int>(ctx_param(*c, "heads", 1));
  const int nkv = static_cast<int>(ctx_param(*c, "kv_heads", 1));
  const int hd = static_cast<int>(ctx_param(*c, "head_dim", 128));
  const int page = static_cast<int>(ctx_param(*c, "page_size", 16));
  if (nq % nkv || hd > 256) return op_error(Errc::ShapeMismatch, "attn_decode: heads");
  const int hnd = static_cast<int>(ctx_param(*c, "kv_layout", 0.0));  // 0 NHD, 1 HND
  if (hnd == 0 && (in[1].rank != 4 || in[1].shape[1] != page || in[1].shape[2] != nkv || in[1].shape[3] != hd))
    return op_error(Errc::ShapeMismatch, "attn_decode: cache must be [pages, page, kv_heads, hd]");
  if (hnd == 1 && (in[1].rank != 4 || in[1].shape[1] != nkv || in[1].shape[2] != page || in[1].shape[3] != hd))
    return op_error(Errc::ShapeMismatch, "attn_decode: kv_layout 1 (HND) cache must be [pages, kv_heads, page, hd]");
  if (hnd != 0 && hnd != 1) return op_error(Errc::ConfigError, "attn_decode: kv_layout is 0 (NHD) or 1 (HND)");
  bool same_kv = in[2].rank == in[1].rank;
  for (int i = 0; same_kv && i < in[1].rank; ++i) same_kv = in[2].shape[i] == in[1].shape[i];
  if (!same_kv) return op_error(Errc::ShapeMismatch, "attn_decode: K and V caches must have identical shapes");
  if (in[0].dtype != in[1].dtype || in[2].dtype != in[1].dtype || out[0].dtype != in[0].dtype ||
      (in[0].dtype != OPF_BF16 && in[0].dtype != OPF_F32))
    return op_error(Errc::ShapeMismatch, "attn_decode: qkv, caches and output share one float dtype");
  if (in[3].dtype != OPF_I64 || in[4].dtype != OPF_I64 || in[3].rank != 2 || in[4].rank != 1)
    return op_error(Errc::ShapeMismatch, "attn_decode: block table [B, max_pages] and context lengths [B] are i64");
  if (view_row_elems(in[0]) != static_cast<int64_t>(nq + 2 * nkv) * hd || view_row_elems(out[0]) != int64_t{nq} * hd)
    return op_error(Errc::ShapeMismatch, "attn_decode: qkv rows are (heads + 2 kv_heads) * head_dim wide, "
                                         "outputs heads * head_dim");
  if (rows == 0) return 0;
  const int64_t max_pages = view_row_elems(in[3]);
  const float scale = 1.0f / sqrtf(static_cast<float>(hd));
  auto s = static_cast<cudaStream_t>(stream);
  const int grp = nq / nkv;
  const int impl = static_cast<int>(ctx_param(*c, "impl", 0.0));  // 0 auto, 1 warp-SIMT, 2 generic
  if (in[0].dtype == OPF_BF16 && impl == 0 && ctx_param(*c, "simt", 0.0) == 0.0 &&
      decode_bf16_mma(vptr<__nv_bfloat16>(in[0]), vptr<__nv_bfloat16>(in[1]), vptr<__nv_bfloat16>(in[2]),
                      vptr<int64_t>(in[3]), vptr<int64_t>(in[4]), vptr<__nv_bfloat16>(out[0]), rows, nq,
                      nkv, hd, page, max_pages, scale, c->max_ctas, hnd, s))
    return launch_status("attn_decode_mma");
  if (hnd) return op_error(Errc::ShapeMismatch, "attn_decode: HND pages need the tensor-core path (bf16, hd 128, group <= 8)");
  if (in[0].dtype == OPF_BF16 && hd == 128 && grp <= kMaxGroup && impl != 2 &&
      ctx_param(*c, "simt", 0.0) == 0.0) {
    const unsigned grid = static_cast<unsigned>(rows * nkv);
    auto args = [&](auto kern) {
      kern<<<grid, kDecWarps * 32, 0, s>>>(vptr<__nv_bfloat16>(in[0]), vptr<__nv_bfloat16>(in[1]),
                                           vptr<__nv_bfloat16>(in[2]), vptr<int64_t>(in[3]),
                                           vptr<int64_t>(in[4]), vptr<__nv_bfloat16>(out[0]), nq,
                                           nkv, max_pages, page, scale);
    };
    switch (grp) {
      case 1: args(decode_bf16_kernel<1>); break;
      case 2: args(decode_bf16_kernel<2>); break;
      case 4: args(decode_bf16_kernel<4>); break;
      case 8: args(decode_bf16_kernel<8>); break;
      default: goto generic;
    }
    return launch_status("attn_decode");
  }
generic:
  {
    const int threads = 128;
    const unsigned grid = static_cast<unsigned>((rows * nq * 32 + threads - 1) / threads);
    if (in[0].dtype == OPF_BF16)
      decode_simt_kernel<__nv_bfloat16><<<grid, threads, 0, s>>>(
          vptr<__nv_bfloat16>(in[0]), vptr<__nv_bfloat16>(in[1]), vptr<__nv_bfloat16>(in[2]),
          vptr<int64_t>(in[3]), vptr<int64_t>(in[4]), vptr<__nv_bfloat16>(out[0]), rows, nq, nkv, hd,
          max_pages, page, scale);
    else
      decode_simt_kernel<float><<<grid, threads, 0, s>>>(
          vptr<float>(in[0]), vptr<float>(in[1]), vptr<float>(in[2]), vptr<int64_t>(in[3]),
          vptr<int64_t>(in[4]), vptr<float>(out[0]), rows, nq, nkv, hd, max_pages, page, scale);
  }
  return launch_status("attn_decode_simt");
}

}  // namespace

void register_attention_ops(OpRegistry& r) {
  r.add({"attn_prefill", op_attn_prefill, ResourceClass::kCompute, 1, 1, {}});
  r.add({"attn_decode", op_attn_decode, ResourceClass::kMemory, 5, 1, {}});
}

}  // namespace opflow
