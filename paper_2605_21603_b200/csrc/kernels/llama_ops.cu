// Memory-bound Llama-layer ops on sm_100a: rmsnorm, add_rmsnorm (fused
// residual + norm), rope (rotate-half), silu_mul.  One CTA per row, 16-byte
// vector loads/stores, the row held in registers between the reduction and the
// write (one HBM read + one write per element), warp-shuffle + smem reduction.
// Algorithmic bytes/row: rmsnorm 2*H*b (+H*b gamma, L2-resident), add_rmsnorm
// 4*H*b, rope 2*W*b, silu_mul 3*I*b (b = dtype bytes).  CPU references:
// oracle/ref_shim.cpp (Custom ops registered in the reference's CustomRegistry)
// and oracle/oracle.py.
#include <cuda_bf16.h>

#include "opflow/device.hpp"

namespace opflow {

namespace {

constexpr int kThreads = 128;
constexpr int kMaxVec = 8;  // 16-byte vectors per thread held in registers

template <typename T>
struct Vec;
template <>
struct Vec<__nv_bfloat16> {
  static constexpr int N = 8;
  __device__ static void load(const __nv_bfloat16* p, float* f) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 v = __bfloat1622float2(h[i]);
      f[2 * i] = v.x;
      f[2 * i + 1] = v.y;
    }
  }
  __device__ static void store(__nv_bfloat16* p, const float* f) {
    uint4 u;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    *reinterpret_cast<uint4*>(p) = u;
  }
};
template <>
struct Vec<float> {
  static constexpr int N = 4;
  __device__ static void load(const float* p, float* f) {
    const float4 u = *reinterpret_cast<const float4*>(p);
    f[0] = u.x;
    f[1] = u.y;
    f[2] = u.z;
    f[3] = u.w;
  }
  __device__ static void store(float* p, const float* f) {
    *reinterpret_cast<float4*>(p) = make_float4(f[0], f[1], f[2], f[3]);
  }
};

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float t = 0.0f;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) t += red[w];
  __syncthreads();
  return t;
}

// y = x * rsqrt(mean(x^2) + eps) * g; with RES, s = x + r is also stored and normalised.
template <typename T, bool RES>
__global__ void __launch_bounds__(kThreads) rmsnorm_kernel(const T* __restrict__ x,
                                                           const T* __restrict__ r,
                                                           const T* __restrict__ g,
                                                           T* __restrict__ s_out,
                                                           T* __restrict__ y, int64_t H, float eps) {
  pdl_wait();
  pdl_trigger();
  constexpr int V = Vec<T>::N;
  __shared__ float red[kThreads / 32];
  const int64_t row = blockIdx.x;
  const T* xr = x + row * H;
  const int64_t nvec = H / V;
  float v[kMaxVec][V];
  float ss = 0.0f;
#pragma unroll
  for (int i = 0; i < kMaxVec; ++i) {
    const int64_t c = (static_cast<int64_t>(i) * kThreads + threadIdx.x);
    if (c < nvec) {
      Vec<T>::load(xr + c * V, v[i]);
      if constexpr (RES) {
        float rv[V];
        Vec<T>::load(r + row * H + c * V, rv);
#pragma unroll
        for (int k = 0; k < V; ++k) v[i][k] += rv[k];
        Vec<T>::store(s_out + row * H + c * V, v[i]);
      }
#pragma unroll
      for (int k = 0; k < V; ++k) ss += v[i][k] * v[i][k];
    }
  }
  const float inv = rsqrtf(block_sum(ss, red) / static_cast<float>(H) + eps);
#pragma unroll
  for (int i = 0; i < kMaxVec; ++i) {
    const int64_t c = (static_cast<int64_t>(i) * kThreads + threadIdx.x);
    if (c < nvec) {
      float gv[V], o[V];
      Vec<T>::load(g + c * V, gv);
#pragma unroll
      for (int k = 0; k < V; ++k) o[k] = v[i][k] * inv * gv[k];
      Vec<T>::store(y + row * H + c * V, o);
    }
  }
}

// Norm half of a MatMul fused with add_rmsnorm: the epi-4 GEMM stored
// x1 = x + A W and per-(row, 256-column tile) sums of squares; one warp per
// row sums those (fixed order: deterministic) and writes y = x1 * rsqrt(ms + eps) * g.
__global__ void __launch_bounds__(256) rmsnorm_stats_kernel(const __nv_bfloat16* __restrict__ x1,
                                                            const float* __restrict__ ssq, int64_t n_tiles,
                                                            const __nv_bfloat16* __restrict__ g,
                                                            __nv_bfloat16* __restrict__ y, int64_t rows, int64_t H,
                                                            float eps) {
  pdl_wait();
  pdl_trigger();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + warp;
  if (row >= rows) return;
  float t = 0.0f;
  for (int64_t i = lane; i < n_tiles; i += 32) t += ssq[row * n_tiles + i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  const float inv = rsqrtf(t / static_cast<float>(H) + eps);
  const uint4* xr = reinterpret_cast<const uint4*>(x1 + row * H);
  const uint4* gr = reinterpret_cast<const uint4*>(g);
  uint4* yr = reinterpret_cast<uint4*>(y + row * H);
  for (int64_t c = lane; c < H / 8; c += 32) {
    const uint4 u = xr[c], gu = gr[c];
    const __nv_bfloat162* a = reinterpret_cast<const __nv_bfloat162*>(&u);
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&gu);
    uint4 o;
    __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 fa = __bfloat1622float2(a[e]), fb = __bfloat1622float2(b[e]);
      o2[e] = __floats2bfloat162_rn(fa.x * inv * fb.x, fa.y * inv * fb.y);
    }
    yr[c] = o;
  }
}

// HF rotate-half rope on the q and k heads of a fused qkv row; v is copied.
template <typename T>
__global__ void __launch_bounds__(256) rope_kernel(const T* __restrict__ qkv,
                                                   const int64_t* __restrict__ pos,
                                                   T* __restrict__ out, int n_rot_heads,
                                                   int n_v_heads, int hd, float log2_theta) {
  pdl_wait();
  pdl_trigger();
  constexpr int V = Vec<T>::N;
  const int64_t row = blockIdx.x;
  const int64_t W = static_cast<int64_t>(n_rot_heads + n_v_heads) * hd;
  const T* in = qkv + row * W;
  T* o = out + row * W;
  const float p = static_cast<float>(pos[row]);
  const int half = hd / 2, chunks_per_head = half / V;
  const int n_rot = n_rot_heads * chunks_per_head;
  const int n_cpy = n_v_heads * hd / V;
  for (int item = threadIdx.x; item < n_rot + n_cpy; item += blockDim.x) {
    if (item < n_rot) {
      const int h = item / chunks_per_head, i0 = (item % chunks_per_head) * V;
      float a[V], b[V], ra[V], rb[V];
      Vec<T>::load(in + h * hd + i0, a);
      Vec<T>::load(in + h * hd + half + i0, b);
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const float inv_freq = exp2f(-2.0f * static_cast<float>(i0 + k) / hd * log2_theta);
        float sn, cs;
        sincosf(p * inv_freq, &sn, &cs);
        ra[k] = a[k] * cs - b[k] * sn;
        rb[k] = b[k] * cs + a[k] * sn;
      }
      Vec<T>::store(o + h * hd + i0, ra);
      Vec<T>::store(o + h * hd + half + i0, rb);
    } else {
      const int64_t c = static_cast<int64_t>(n_rot_heads) * hd + static_cast<int64_t>(item - n_rot) * V;
      float a[V];
      Vec<T>::load(in + c, a);
      Vec<T>::store(o + c, a);
    }
  }
}

// Qwen3 attention prologue: per-head RMSNorm of every q and k head (weights
// q_norm / k_norm, [hd]) followed by rotate-half RoPE; v heads copied.  One
// warp per head (hd = 128: 4 elements per lane, rotate-half partner = lane ^ 16).
__global__ void __launch_bounds__(256) qk_norm_rope_kernel(const __nv_bfloat16* __restrict__ qkv,
                                                           const int64_t* __restrict__ pos,
                                                           const __nv_bfloat16* __restrict__ qn,
                                                           const __nv_bfloat16* __restrict__ kn,
                                                           __nv_bfloat16* __restrict__ out, int nq, int nkv,
                                                           float log2_theta, float eps) {
  pdl_wait();
  pdl_trigger();
  constexpr int HD = 128;
  const int64_t row = blockIdx.x;
  const int64_t W = static_cast<int64_t>(nq + 2 * nkv) * HD;
  const __nv_bfloat16* in = qkv + row * W;
  __nv_bfloat16* o = out + row * W;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const float p = static_cast<float>(pos[row]);
  const int i0 = lane * 4;
  // the rotation depends only on (position, dim): one sincos per lane element
  // per row, shared by all q/k heads (reduced argument, MUFU sin/cos)
  float cs[4], sn[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int j = (i0 + k) % (HD / 2);
    const float ang = p * exp2f(-2.0f * static_cast<float>(j) / HD * log2_theta);
    const float q = rintf(ang * 0.15915494309189535f);
    const float red = fmaf(-q, 6.28318548202514648f, fmaf(-q, -1.7484556e-07f, ang));
    __sincosf(red, &sn[k], &cs[k]);
  }
  for (int h = warp; h < nq + nkv; h += blockDim.x / 32) {
    const uint2 u = *reinterpret_cast<const uint2*>(in + h * HD + i0);
    const __nv_bfloat162* x2 = reinterpret_cast<const __nv_bfloat162*>(&u);
    const uint2 gu = *reinterpret_cast<const uint2*>((h < nq ? qn : kn) + i0);
    const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gu);
    float x[4], g[4];
    for (int k = 0; k < 2; ++k) {
      const float2 a = __bfloat1622float2(x2[k]), b = __bfloat1622float2(g2[k]);
      x[2 * k] = a.x;
      x[2 * k + 1] = a.y;
      g[2 * k] = b.x;
      g[2 * k + 1] = b.y;
    }
    float ss = x[0] * x[0] + x[1] * x[1] + x[2] * x[2] + x[3] * x[3];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    const float inv = rsqrtf(ss / HD + eps);
    float y[4], r[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) y[k] = x[k] * inv * g[k];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float partner = __shfl_xor_sync(0xffffffffu, y[k], 16);
      r[k] = lane < 16 ? y[k] * cs[k] - partner * sn[k] : y[k] * cs[k] + partner * sn[k];
    }
    uint2 w;
    __nv_bfloat162* w2 = reinterpret_cast<__nv_bfloat162*>(&w);
    w2[0] = __floats2bfloat162_rn(r[0], r[1]);
    w2[1] = __floats2bfloat162_rn(r[2], r[3]);
    *reinterpret_cast<uint2*>(o + h * HD + i0) = w;
  }
  // v heads: straight copy
  const int64_t v0 = static_cast<int64_t>(nq + nkv) * HD;
  for (int64_t c = threadIdx.x * 8; c < static_cast<int64_t>(nkv) * HD; c += blockDim.x * 8)
    *reinterpret_cast<uint4*>(o + v0 + c) = *reinterpret_cast<const uint4*>(in + v0 + c);
}

template <typename T>
__global__ void silu_mul_kernel(const T* __restrict__ gu, T* __restrict__ out, int64_t rows,
                                int64_t I) {
  pdl_wait();
  pdl_trigger();
  constexpr int V = Vec<T>::N;
  const int64_t per_row = I / V, n = rows * per_row;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / per_row, c = (i % per_row) * V;
    float g[V], u[V], o[V];
    Vec<T>::load(gu + r * 2 * I + c, g);
    Vec<T>::load(gu + r * 2 * I + I + c, u);
#pragma unroll
    for (int k = 0; k < V; ++k) o[k] = g[k] / (1.0f + expf(-g[k])) * u[k];
    Vec<T>::store(out + r * I + c, o);
  }
}

template <typename T>
opf_status run_rmsnorm(const opf_view* in, opf_view* out, int64_t rows, float eps, bool res,
                       cudaStream_t s) {
  const int64_t H = view_row_elems(in[0]);
  if (H % Vec<T>::N != 0 || H / Vec<T>::N > static_cast<int64_t>(kThreads) * kMaxVec)
    return op_error(Errc::ShapeMismatch, "rmsnorm: hidden " + std::to_string(H) + " unsupported");
  if (rows == 0) return 0;
  if (res)
    launch_pdl(rmsnorm_kernel<T, true>, dim3(static_cast<unsigned>(rows)), dim3(kThreads), 0, s,
               static_cast<const T*>(vptr<T>(in[0])), static_cast<const T*>(vptr<T>(in[1])),
               static_cast<const T*>(vptr<T>(in[2])), vptr<T>(out[0]), vptr<T>(out[1]), H, eps);
  else
    launch_pdl(rmsnorm_kernel<T, false>, dim3(static_cast<unsigned>(rows)), dim3(kThreads), 0, s,
               static_cast<const T*>(vptr<T>(in[0])), static_cast<const T*>(nullptr),
               static_cast<const T*>(vptr<T>(in[1])), static_cast<T*>(nullptr), vptr<T>(out[0]), H, eps);
  return launch_status("rmsnorm");
}

opf_status op_rmsnorm(const opf_op_ctx* c, const opf_view* in, int32_t n_in, opf_view* out,
                      int32_t n_out, int64_t rows, void* stream) {
  if (n_in != 2 || n_out != 1) return op_error(Errc::ShapeMismatch, "rmsnorm takes (x, g) -> y");
  const float eps = static_cast<float>(ctx_param(*c, "eps", 1e-5));
  auto s = static_cast<cudaStream_t>(stream);
  if (in[0].dtype == OPF_BF16) return run_rmsnorm<__nv_bfloat16>(in, out, rows, eps, false, s);
  if (in[0].dtype == OPF_F32) return run_rmsnorm<float>(in, out, rows, eps, false, s);
  return op_error(Errc::ShapeMismatch, "rmsnorm: dtype");
}

opf_status op_add_rmsnorm(const opf_op_ctx* c, const opf_view* in, int32_t n_in, opf_view* out,
                          int32_t n_out, int64_t rows, void* stream) {
  if (n_in != 3 || n_out != 2)
    return op_error(Errc::ShapeMismatch, "add_rmsnorm takes (x, r, g) -> (x+r, y)");
  const float eps = static_cast<float>(ctx_param(*c, "eps", 1e-5));
  auto s = static_cast<cudaStream_t>(stream);
  if (in[0].dtype == OPF_BF16) return run_rmsnorm<__nv_bfloat16>(in, out, rows, eps, true, s);
  if (in[0].dtype == OPF_F32) return run_rmsnorm<float>(in, out, rows, eps, true, s);
  return op_error(Errc::ShapeMismatch, "add_rmsnorm: dtype");
}

opf_status op_rope(const opf_op_ctx* c, const opf_view* in, int32_t n_in, opf_view* out,
                   int32_t n_out, int64_t rows, void* stream) {
  if (n_in != 2 || n_out != 1) return op_error(Errc::ShapeMismatch, "rope takes (qkv, pos) -> qkv");
  const int nq = static_cast<int>(ctx_param(*c, "heads", 1));
  const int nkv = static_cast<int>(ctx_param(*c, "kv_heads", 1));
  const int hd = static_cast<int>(ctx_param(*c, "head_dim", 128));
  const float l2t = static_cast<float>(std::log2(ctx_param(*c, "theta", 10000.0)));
  if (view_row_elems(in[0]) != static_cast<int64_t>(nq + 2 * nkv) * hd)
    return op_error(Errc::ShapeMismatch, "rope: qkv width does not match heads");
  if (rows == 0) return 0;
  auto s = static_cast<cudaStream_t>(stream);
  const int64_t* pos = vptr<int64_t>(in[1]);
  if (in[0].dtype == OPF_BF16) {
    if ((hd / 2) % 8) return op_error(Errc::ShapeMismatch, "rope: head_dim/2 must be a multiple of 8");
    launch_pdl(rope_kernel<__nv_bfloat16>, dim3(static_cast<unsigned>(rows)), dim3(256), 0, s,
               static_cast<const __nv_bfloat16*>(vptr<__nv_bfloat16>(in[0])), pos,
               vptr<__nv_bfloat16>(out[0]), nq + nkv, nkv, hd, l2t);
  } else if (in[0].dtype == OPF_F32) {
    if ((hd / 2) % 4) return op_error(Errc::ShapeMismatch, "rope: head_dim/2 must be a multiple of 4");
    rope_kernel<float><<<static_cast<unsigned>(rows), 256, 0, s>>>(vptr<float>(in[0]), pos,
                                                                    vptr<float>(out[0]), nq + nkv,
                                                                    nkv, hd, l2t);
  } else {
    return op_error(Errc::ShapeMismatch, "rope: dtype");
  }
  return launch_status("rope");
}

opf_status op_silu_mul(const opf_op_ctx*, const opf_view* in, int32_t n_in, opf_view* out,
                       int32_t n_out, int64_t rows, void* stream) {
  if (n_in != 1 || n_out != 1) return op_error(Errc::ShapeMismatch, "silu_mul takes (gu) -> a");
  const int64_t I = view_row_elems(out[0]);
  if (view_row_elems(in[0]) != 2 * I) return op_error(Errc::ShapeMismatch, "silu_mul: width");
  if (rows == 0) return 0;
  auto s = static_cast<cudaStream_t>(stream);
  const int threads = 256;
  if (in[0].dtype == OPF_BF16) {
    if (I % 8) return op_error(Errc::ShapeMismatch, "silu_mul: inter % 8");
    const int64_t n = rows * I / 8;
    const int g = static_cast<int>(std::min<int64_t>((n + threads - 1) / threads, num_sms() * 16LL));
    launch_pdl(silu_mul_kernel<__nv_bfloat16>, dim3(g), dim3(threads), 0, s,
               static_cast<const __nv_bfloat16*>(vptr<__nv_bfloat16>(in[0])), vptr<__nv_bfloat16>(out[0]),
               rows, I);
  } else if (in[0].dtype == OPF_F32) {
    if (I % 4) return op_error(Errc::ShapeMismatch, "silu_mul: inter % 4");
    const int64_t n = rows * I / 4;
    const int g = static_cast<int>(std::min<int64_t>((n + threads - 1) / threads, num_sms() * 16LL));
    silu_mul_kernel<float><<<g, threads, 0, s>>>(vptr<float>(in[0]), vptr<float>(out[0]), rows, I);
  } else {
    return op_error(Errc::ShapeMismatch, "silu_mul: dtype");
  }
  return launch_status("silu_mul");
}

opf_status op_qk_norm_rope(const opf_op_ctx* c, const opf_view* in, int32_t n_in, opf_view* out,
                           int32_t n_out, int64_t rows, void* stream) {
  if (n_in != 4 || n_out != 1)
    return op_error(Errc::ShapeMismatch, "qk_norm_rope takes (qkv, pos, q_norm, k_norm) -> qkv");
  const int nq = static_cast<int>(ctx_param(*c, "heads", 1));
  const int nkv = static_cast<int>(ctx_param(*c, "kv_heads", 1));
  const int hd = static_cast<int>(ctx_param(*c, "head_dim", 128));
  const float l2t = static_cast<float>(std::log2(ctx_param(*c, "theta", 1000000.0)));
  const float eps = static_cast<float>(ctx_param(*c, "eps", 1e-6));
  if (hd != 128 || in[0].dtype != OPF_BF16 || view_row_elems(in[0]) != static_cast<int64_t>(nq + 2 * nkv) * hd ||
      view_numel(in[2]) != hd || view_numel(in[3]) != hd)
    return op_error(Errc::ShapeMismatch, "qk_norm_rope: bf16, head_dim 128, norm weights [head_dim]");
  if (rows == 0) return 0;
  launch_pdl(qk_norm_rope_kernel, dim3(static_cast<unsigned>(rows)), dim3(256), 0, static_cast<cudaStream_t>(stream),
             static_cast<const __nv_bfloat16*>(vptr<__nv_bfloat16>(in[0])),
             static_cast<const int64_t*>(vptr<int64_t>(in[1])),
             static_cast<const __nv_bfloat16*>(vptr<__nv_bfloat16>(in[2])),
             static_cast<const __nv_bfloat16*>(vptr<__nv_bfloat16>(in[3])), vptr<__nv_bfloat16>(out[0]), nq, nkv,
             l2t, eps);
  return launch_status("qk_norm_rope");
}

}  // namespace

void rmsnorm_from_stats(const void* x1, const float* ssq, int64_t n_tiles, const void* gamma, void* y, int64_t rows,
                        int64_t H, float eps, cudaStream_t s) {
  launch_pdl(rmsnorm_stats_kernel, dim3(static_cast<unsigned>((rows + 7) / 8)), dim3(256), 0, s,
             static_cast<const __nv_bfloat16*>(x1), ssq, n_tiles, static_cast<const __nv_bfloat16*>(gamma),
             static_cast<__nv_bfloat16*>(y), rows, H, eps);
}

void register_llama_ops(OpRegistry& r) {
  r.add({"rmsnorm", op_rmsnorm, ResourceClass::kMemory, 2, 1, {}});
  r.add({"add_rmsnorm", op_add_rmsnorm, ResourceClass::kMemory, 3, 2, {}});
  r.add({"rope", op_rope, ResourceClass::kMemory, 2, 1, {}});
  r.add({"silu_mul", op_silu_mul, ResourceClass::kMemory, 1, 1, {}});
  r.add({"qk_norm_rope", op_qk_norm_rope, ResourceClass::kMemory, 4, 1, {}});
}

}  // namespace opflow
