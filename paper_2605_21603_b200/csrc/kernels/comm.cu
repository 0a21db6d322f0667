// Fused communication + normalisation replacement ops (TokenWeave-style
// partial overlap; Fig. 7):
//
//   allreduce_rowscale     (x)        -> rowscale(allreduce(x))          stand-in graphs
//   allreduce_add_rmsnorm  (o, x, g)  -> (x + allreduce(o), rmsnorm(..)*g) Llama layers
//
// Single device (no communicator, or world 1): allreduce is the reference's
// stand-in "sum of world_size identical replicas" (x * world_size), fused
// into the norm pass so the tensor is read once.  The fp32 / i64 stand-in
// path reproduces AllReduce-then-RowScale to the bit (same rounding sequence
// as /root/reference/proj/src/kernels_scalar.cpp:21-38).
//
// Multi-GPU (world > 1): when the communicator carries a peer window the fused
// kernel pulls every rank's partial row over NVLink (P2P loads), reduces,
// adds the residual and normalises in one pass — no separate all-reduce
// kernel, no extra HBM round trip.  Without a window it falls back to
// ncclAllReduce + the fused add+norm pass.
#include <cuda_bf16.h>

#include "opflow/comm.hpp"
#include "opflow/nccl_api.hpp"
#include "opflow/device.hpp"

namespace opflow {

bool ar_add_rmsnorm_p2p(const opf_comm* c, const opf_view& o, const opf_view& x, const opf_view& g,
                        opf_view& x_out, opf_view& y, int64_t rows, float eps, int max_ctas, int mode,
                        cudaStream_t s);
bool gemm_ar_add_rmsnorm_push(const opf_comm* c, const GemmArgs& g, const opf_view& x, const opf_view& gam,
                              opf_view& x_out, opf_view& y, float eps, cudaStream_t s);

namespace {

constexpr int kThreads = 128;

__device__ __forceinline__ float bsum(float v, float* red) {
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = v;
  __syncthreads();
  float t = 0.0f;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) t += red[w];
  __syncthreads();
  return t;
}

// exact stand-in: y = RowScale(x * ws), fp32 (one warp per row, serial sum)
__global__ void ar_rowscale_f32_kernel(const float* __restrict__ x, float* __restrict__ y,
                                       int64_t rows, int64_t cols, float ws) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * 4 + warp;
  if (r >= rows) return;
  const float* xr = x + r * cols;
  float sumsq = 0.0f;
  if (lane == 0)
    for (int64_t c = 0; c < cols; ++c) {
      const float t = __fmul_rn(xr[c], ws);
      sumsq = __fadd_rn(sumsq, __fmul_rn(t, t));
    }
  float inv = 0.0f;
  if (lane == 0)
    inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(sumsq, static_cast<float>(cols)), 1e-6f)));
  inv = __shfl_sync(0xffffffffu, inv, 0);
  for (int64_t c = lane; c < cols; c += 32) y[r * cols + c] = __fmul_rn(__fmul_rn(xr[c], ws), inv);
}

__global__ void ar_rowscale_i64_kernel(const int64_t* __restrict__ x, int64_t* __restrict__ y,
                                       int64_t rows, int64_t cols, int64_t ws) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * 4 + warp;
  if (r >= rows) return;
  auto t_of = [&](int64_t c) {
    return static_cast<int64_t>(static_cast<uint64_t>(x[r * cols + c]) * static_cast<uint64_t>(ws));
  };
  int64_t stat = 1;
  for (int64_t c = lane; c < cols; c += 32) {
    const int64_t v = t_of(c);
    const int64_t mag = v < 0 ? static_cast<int64_t>(0ull - static_cast<uint64_t>(v)) : v;
    stat = mag > stat ? mag : stat;
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    const int64_t o = __shfl_xor_sync(0xffffffffu, stat, s);
    stat = o > stat ? o : stat;
  }
  for (int64_t c = lane; c < cols; c += 32) y[r * cols + c] = t_of(c) / stat;
}

// bf16 / generic: one CTA per row.  `partials` = world pointers to the rows'
// partial sums (peer window) or just {o} on one device (scaled by ws).
struct PartList {
  const void* p[8];
};

template <typename T, bool RESID>
__global__ void __launch_bounds__(kThreads) ar_norm_kernel(
    const PartList partials, int n_part, float scale, const T* __restrict__ resid,
    const T* __restrict__ g, T* __restrict__ x_out, T* __restrict__ y, int64_t H, float eps,
    bool rowscale_semantics) {
  __shared__ float red[kThreads / 32];
  extern __shared__ float rowbuf[];
  const int64_t row = blockIdx.x;
  float ss = 0.0f;
  for (int64_t c = threadIdx.x; c < H; c += kThreads) {
    float v = 0.0f;
    for (int p = 0; p < n_part; ++p) {
      if constexpr (std::is_same_v<T, float>)
        v += static_cast<const T*>(partials.p[p])[row * H + c];
      else
        v += __bfloat162float(static_cast<const T*>(partials.p[p])[row * H + c]);
    }
    v *= scale;
    if constexpr (RESID) {
      if constexpr (std::is_same_v<T, float>)
        v += resid[row * H + c];
      else
        v += __bfloat162float(resid[row * H + c]);
      if constexpr (std::is_same_v<T, float>)
        x_out[row * H + c] = v;
      else
        x_out[row * H + c] = __float2bfloat16(v);
    }
    rowbuf[c] = v;
    ss += v * v;
  }
  const float tot = bsum(ss, red);
  const float inv = rowscale_semantics ? rsqrtf(tot / static_cast<float>(H) + 1e-6f)
                                       : rsqrtf(tot / static_cast<float>(H) + eps);
  for (int64_t c = threadIdx.x; c < H; c += kThreads) {
    float o = rowbuf[c] * inv;
    if (g) {
      if constexpr (std::is_same_v<T, float>)
        o *= g[c];
      else
        o *= __bfloat162float(g[c]);
    }
    if constexpr (std::is_same_v<T, float>)
      y[row * H + c] = o;
    else
      y[row * H + c] = __float2bfloat16(o);
  }
}

template <typename T>
opf_status launch_ar_norm(const opf_comm* comm, const opf_view& o, const opf_view* resid,
                          const opf_view* g, opf_view* x_out, opf_view& y, int64_t rows, float eps,
                          int64_t ws, bool rowscale, void* workspace, cudaStream_t s) {
  const int64_t H = view_row_elems(o);
  const size_t smem = static_cast<size_t>(H) * sizeof(float);
  if (smem > 48 * 1024) return op_error(Errc::ShapeMismatch, "fused norm: row too wide");
  const T* src = vptr<T>(o);
  float scale = static_cast<float>(ws);
  if (comm && comm->world > 1 && !comm->nccl)
    return op_error(Errc::ConfigError, "allreduce_norm: peer-only communicator and the message does not "
                                       "fit its window");
  if (comm && comm->world > 1) {
    // NCCL all-reduce into the workspace, then one fused add+norm pass.
    T* red = static_cast<T*>(workspace);
    const ncclResult_t r = nccl().AllReduce(src, red, static_cast<size_t>(rows * H),
                                         std::is_same_v<T, float> ? ncclFloat32 : ncclBfloat16,
                                         ncclSum, comm->nccl, s);
    if (r != ncclSuccess)
      return op_error(Errc::SchedulerError, std::string("ncclAllReduce: ") + nccl().GetErrorString(r));
    src = red;
    scale = 1.0f;
  }
  PartList d_parts{};
  d_parts.p[0] = src;
  if (resid)
    ar_norm_kernel<T, true><<<static_cast<unsigned>(rows), kThreads, smem, s>>>(
        d_parts, 1, scale, vptr<T>(*resid), g ? vptr<T>(*g) : nullptr, vptr<T>(*x_out), vptr<T>(y),
        H, eps, rowscale);
  else
    ar_norm_kernel<T, false><<<static_cast<unsigned>(rows), kThreads, smem, s>>>(
        d_parts, 1, scale, nullptr, g ? vptr<T>(*g) : nullptr, nullptr, vptr<T>(y), H, eps,
        rowscale);
  return launch_status("allreduce_norm");
}

size_t ws_ar(const opf_op_ctx& c, const opf_view* in, int, const opf_view*, int, int64_t rows) {
  const opf_comm* comm = static_cast<const opf_comm*>(c.comm);
  size_t bytes = 0;
  if (comm && comm->world > 1)
    bytes += static_cast<size_t>(rows * view_row_elems(in[0]) * dtype_bytes(Dtype(in[0].dtype)));
  return bytes;
}

opf_status op_ar_rowscale(const opf_op_ctx* c, const opf_view* in, int32_t n_in, opf_view* out,
                          int32_t n_out, int64_t rows, void* stream) {
  if (n_in != 1 || n_out != 1)
    return op_error(Errc::SignatureMismatch, "allreduce_rowscale takes (x) -> y");
  if (rows == 0) return 0;
  auto s = static_cast<cudaStream_t>(stream);
  const opf_comm* comm = static_cast<const opf_comm*>(c->comm);
  const int64_t cols = view_row_elems(in[0]);
  if (!(comm && comm->world > 1)) {
    if (in[0].dtype == OPF_F32) {
      ar_rowscale_f32_kernel<<<static_cast<unsigned>((rows + 3) / 4), 128, 0, s>>>(
          vptr<float>(in[0]), vptr<float>(out[0]), rows, cols, static_cast<float>(c->world_size));
      return launch_status("allreduce_rowscale");
    }
    if (in[0].dtype == OPF_I64) {
      ar_rowscale_i64_kernel<<<static_cast<unsigned>((rows + 3) / 4), 128, 0, s>>>(
          vptr<int64_t>(in[0]), vptr<int64_t>(out[0]), rows, cols, c->world_size);
      return launch_status("allreduce_rowscale");
    }
  }
  if (in[0].dtype == OPF_BF16)
    return launch_ar_norm<__nv_bfloat16>(comm, in[0], nullptr, nullptr, nullptr, out[0], rows, 1e-6f,
                                         c->world_size, true, c->workspace, s);
  if (in[0].dtype == OPF_F32)
    return launch_ar_norm<float>(comm, in[0], nullptr, nullptr, nullptr, out[0], rows, 1e-6f,
                                 c->world_size, true, c->workspace, s);
  return op_error(Errc::ShapeMismatch, "allreduce_rowscale: dtype with communicator");
}

opf_status op_ar_add_rmsnorm(const opf_op_ctx* c, const opf_view* in, int32_t n_in, opf_view* out,
                             int32_t n_out, int64_t rows, void* stream) {
  if (n_in != 3 || n_out != 2)
    return op_error(Errc::SignatureMismatch, "allreduce_add_rmsnorm takes (o, x, g) -> (x1, y)");
  if (rows == 0) return 0;
  auto s = static_cast<cudaStream_t>(stream);
  const opf_comm* comm = static_cast<const opf_comm*>(c->comm);
  const float eps = static_cast<float>(ctx_param(*c, "eps", 1e-5));
  // peer-memory kernel (one-shot, or two-shot for large messages at W >= 4;
  // params.ar_mode 1 / 2 forces one / two-shot) when the communicator has a window
  const int mode = static_cast<int>(ctx_param(*c, "ar_mode", 0.0));
  if (comm && comm->world > 1 && !comm->peer_buf.empty() &&
      ar_add_rmsnorm_p2p(comm, in[0], in[1], in[2], out[0], out[1], rows, eps, c->max_ctas, mode, s))
    return launch_status("allreduce_add_rmsnorm_p2p");
  if (in[0].dtype == OPF_BF16)
    return launch_ar_norm<__nv_bfloat16>(comm, in[0], &in[1], &in[2], &out[0], out[1], rows, eps,
                                         c->world_size, false, c->workspace, s);
  if (in[0].dtype == OPF_F32)
    return launch_ar_norm<float>(comm, in[0], &in[1], &in[2], &out[0], out[1], rows, eps,
                                 c->world_size, false, c->workspace, s);
  return op_error(Errc::ShapeMismatch, "allreduce_add_rmsnorm: dtype");
}

// matmul_allreduce_add_rmsnorm (a, w, x, g) -> (x1, y): the row-parallel
// projection (o_proj / down) + its AllReduce + the residual add + RMSNorm as
// ONE op (the fuse_norm_comm strategy with "fuse_gemm": 1).  With a peer
// window the GEMM epilogue pushes partial slabs to their owner ranks over
// NVLink while later tiles compute, and one kernel reduces, normalises and
// gathers (gemm_ar_add_rmsnorm_p2p in comm_p2p.cu).  Otherwise: GEMM into the
// workspace, then the allreduce_add_rmsnorm path on it.
size_t ws_mm_ar(const opf_op_ctx& c, const opf_view* in, int n_in, const opf_view* out, int n_out, int64_t rows) {
  if (n_in != 4 || n_out != 2) return 0;
  const size_t o_bytes = (static_cast<size_t>(rows * view_row_elems(out[0]) * 2) + 255) / 256 * 256;
  opf_view o = out[0];
  return o_bytes + ws_ar(c, &o, 1, nullptr, 0, rows);
}

opf_status op_mm_ar_add_rmsnorm(const opf_op_ctx* c, const opf_view* in, int32_t n_in, opf_view* out,
                                int32_t n_out, int64_t rows, void* stream) {
  if (n_in != 4 || n_out != 2)
    return op_error(Errc::SignatureMismatch, "matmul_allreduce_add_rmsnorm takes (a, w, x, g) -> (x1, y)");
  if (rows == 0) return 0;
  auto s = static_cast<cudaStream_t>(stream);
  const int64_t K = view_row_elems(in[0]), N = view_row_elems(out[0]);
  if (in[0].dtype != OPF_BF16 || in[1].dtype != OPF_BF16 || in[1].shape[0] != K || in[1].shape[1] != N)
    return op_error(Errc::ShapeMismatch, "matmul_allreduce_add_rmsnorm: bf16 a [rows,K] and w [K,N]");
  if (!c->aux) return op_error(Errc::ShapeMismatch, "matmul_allreduce_add_rmsnorm needs the packed weight");
  const opf_comm* comm = static_cast<const opf_comm*>(c->comm);
  const float eps = static_cast<float>(ctx_param(*c, "eps", 1e-5));
  GemmArgs g{};
  g.a = view_ptr(in[0]);
  g.bt = c->aux;
  g.m = rows;
  g.n = N;
  g.k = K;
  g.lda = K;
  g.ldc = N;
  g.max_ctas = c->max_ctas;
  if (comm && comm->world > 1 && !comm->peer_buf.empty() && ctx_param(*c, "push", 1.0) != 0.0 &&
      gemm_ar_add_rmsnorm_push(comm, g, in[2], in[3], out[0], out[1], eps, s))
    return launch_status("matmul_allreduce_add_rmsnorm_push");
  // unfused fallback: partial product in the workspace, then the fused AR + add + norm
  const size_t o_bytes = (static_cast<size_t>(rows * N * 2) + 255) / 256 * 256;
  if (!c->workspace || c->workspace_bytes < o_bytes)
    return op_error(Errc::ShapeMismatch, "matmul_allreduce_add_rmsnorm: workspace too small");
  g.c = c->workspace;
  gemm_bf16_tc(g, s);
  opf_view o = make_view(c->workspace, 0, Dtype::kBF16, {rows, N}, true);
  opf_op_ctx c2 = *c;
  c2.workspace = static_cast<char*>(c->workspace) + o_bytes;
  c2.workspace_bytes = c->workspace_bytes - o_bytes;
  opf_view ins[3] = {o, in[2], in[3]};
  return op_ar_add_rmsnorm(&c2, ins, 3, out, 2, rows, stream);
}

}  // namespace

void register_comm_ops(OpRegistry& r) {
  r.add({"allreduce_rowscale", op_ar_rowscale, ResourceClass::kNetwork, 1, 1, ws_ar});
  r.add({"allreduce_add_rmsnorm", op_ar_add_rmsnorm, ResourceClass::kNetwork, 3, 2, ws_ar});
  OpEntry mm{"matmul_allreduce_add_rmsnorm", op_mm_ar_add_rmsnorm, ResourceClass::kNetwork, 4, 2, ws_mm_ar};
  mm.prepack_input = 1;  // [K,N] weight -> K-major [N,K] (tcgen05 B operand)
  r.add(mm);
}

}  // namespace opflow
