// Device-op registry and the built-in kind dispatch (device eval_op_into,
// /root/reference/proj/src/eval.cpp:31-107).
#include <cstring>
#include <map>

#include "opflow/comm.hpp"
#include "opflow/nccl_api.hpp"
#include "opflow/device.hpp"

#include <cmath>

namespace opflow {

bool allreduce_p2p(const opf_comm* c, const opf_view& in, opf_view& out, int64_t rows, int max_ctas,
                   cudaStream_t s);

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }
const std::string& last_error_ref() { return g_last_error; }

opf_status op_error(Errc code, const std::string& msg) {
  set_last_error(msg);
  return static_cast<opf_status>(code) + 1;
}

opf_status launch_status(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) return 0;
  return op_error(Errc::SchedulerError, std::string(what) + ": " + cudaGetErrorString(e));
}

opf_view make_view(void* base, int64_t elem_offset, Dtype dt, const std::vector<int64_t>& shape,
                   bool batched) {
  opf_view v{};
  v.base = base;
  v.elem_offset = elem_offset;
  v.dtype = static_cast<int32_t>(dt);
  v.rank = static_cast<int32_t>(shape.size());
  for (std::size_t i = 0; i < shape.size() && i < 4; ++i) v.shape[i] = shape[i];
  v.batched = batched ? 1 : 0;
  return v;
}

double ctx_param(const opf_op_ctx& c, const char* name, double dflt) {
  for (int i = 0; i < c.n_params; ++i)
    if (std::strcmp(c.param_names[i], name) == 0) return c.param_values[i];
  return dflt;
}

OpRegistry::OpRegistry() {
  register_llama_ops(*this);
  register_attention_ops(*this);
  register_comm_ops(*this);
  register_moe_ops(*this);
  register_kv_ops(*this);
}

OpRegistry& OpRegistry::global() {
  static OpRegistry r;
  return r;
}

void OpRegistry::add(OpEntry e) {
  std::lock_guard<std::mutex> g(mu_);
  ops_[e.name] = std::move(e);
}

const OpEntry* OpRegistry::find(const std::string& name) const {
  std::lock_guard<std::mutex> g(mu_);
  auto it = ops_.find(name);
  return it == ops_.end() ? nullptr : &it->second;
}

const void* alltoall_perm_device(uint64_t seed, int64_t cols) {
  static std::mutex mu;
  static std::map<std::pair<uint64_t, int64_t>, void*> cache;
  std::lock_guard<std::mutex> g(mu);
  auto key = std::make_pair(seed, cols);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  std::vector<uint32_t> host(static_cast<std::size_t>(cols));
  opf_alltoall_permutation(seed, static_cast<uint32_t>(cols), host.data());
  void* d = nullptr;
  OPF_CUDA(cudaMalloc(&d, cols * sizeof(uint32_t)));
  OPF_CUDA(cudaMemcpy(d, host.data(), cols * sizeof(uint32_t), cudaMemcpyHostToDevice));
  cache[key] = d;
  return d;
}

namespace {

ncclDataType_t nccl_type(int32_t dt) {
  return dt == OPF_F32 ? ncclFloat32 : (dt == OPF_BF16 ? ncclBfloat16 : ncclInt64);
}

}  // namespace

size_t kind_workspace(const opf_op_ctx& c, const opf_view* in, int n_in, const opf_view* out, int n_out,
                      int64_t rows) {
  // bf16 MatMul on the tcgen05 path: split-K partials for under-filled grids
  if (static_cast<OperatorKind>(c.kind) == OperatorKind::kMatMul && n_in >= 2 && n_out >= 1 &&
      in[0].dtype == OPF_BF16) {
    const int epi = static_cast<int>(ctx_param(c, "epi", 0.0));
    if (epi == 2) return 0;  // RoPE epilogue runs unsplit
    if (epi == 4)            // residual-norm epilogue: per-row, per-column-tile sums of squares
      return (static_cast<size_t>(rows * (out[0].shape[1] / 256)) * sizeof(float) + 255) / 256 * 256;
    const int64_t N = out[0].shape[1] * (epi == 1 ? 2 : 1);
    return gemm_splitk_workspace(rows, N, in[0].shape[1], c.max_ctas);
  }
  return 0;
}

opf_status launch_kind(const opf_op_ctx& c, const opf_view* in, int n_in, opf_view* out, int n_out,
                       int64_t rows, cudaStream_t s) {
  const auto kind = static_cast<OperatorKind>(c.kind);
  if (n_out < 1) return op_error(Errc::ShapeMismatch, "operator without outputs");
  const Dtype dt = static_cast<Dtype>(in[0].dtype);
  for (int i = 0; i < n_out; ++i)
    if (out[i].dtype != in[0].dtype)
      return op_error(Errc::ShapeMismatch, "output dtype differs from input dtype");
  if (rows == 0) return 0;
  try {
    switch (kind) {
      case OperatorKind::kMatMul: {
        // 1: fused SiLU-mul, 2: fused RoPE, 4: fused residual add + RMSNorm (add_rmsnorm)
        const int epi = static_cast<int>(ctx_param(c, "epi", 0.0));
        if (n_in != (epi == 2 ? 3 : epi == 4 ? 4 : 2) || n_out != (epi == 4 ? 2 : 1))
          return op_error(Errc::ShapeMismatch, epi == 2   ? "MatMul+RoPE takes (x, w, positions)"
                                               : epi == 4 ? "MatMul+add_rmsnorm takes (a, w, x, g) -> (x1, y)"
                                                          : "MatMul takes 2 inputs");
        const int64_t K = in[0].shape[1];
        const int64_t N = out[0].shape[1] * (epi == 1 ? 2 : 1);
        if (in[1].shape[0] != K || in[1].shape[1] != N)
          return op_error(Errc::ShapeMismatch, "MatMul weight must be [K,N]");
        if (epi >= 1 && (dt != Dtype::kBF16 || !c.aux))
          return op_error(Errc::ShapeMismatch, "fused epilogues need the packed bf16 weight");
        if (dt == Dtype::kBF16) {
          GemmArgs g{};
          g.a = view_ptr(in[0]);
          g.c = view_ptr(out[0]);
          g.m = rows;
          g.n = N;
          g.k = K;
          g.lda = K;
          g.ldc = out[0].shape[1];
          g.max_ctas = c.max_ctas;
          g.epi = epi;
          g.ws = c.workspace;
          g.ws_bytes = c.workspace_bytes;
          if (epi == 2) {  // RoPE epilogue: rotate-half on q/k heads (params of the fused rope op)
            const int nq = static_cast<int>(ctx_param(c, "heads", 1));
            const int nkv = static_cast<int>(ctx_param(c, "kv_heads", 1));
            if (static_cast<int>(ctx_param(c, "head_dim", 128)) != 128 || N != static_cast<int64_t>(nq + 2 * nkv) * 128)
              return op_error(Errc::ShapeMismatch, "RoPE epilogue needs head_dim 128 and N = (heads + 2 kv_heads) * 128");
            if (in[2].dtype != OPF_I64) return op_error(Errc::ShapeMismatch, "RoPE positions must be i64");
            g.pos = vptr<const int64_t>(in[2]);
            g.rot_heads = nq + nkv;
            g.log2_theta = static_cast<float>(std::log2(ctx_param(c, "theta", 10000.0)));
          }
          if (epi == 4) {  // C = x + A W, row statistics into the workspace, then the norm pass
            if (view_row_elems(in[2]) != N || view_numel(in[3]) != N || N % 256 != 0)
              return op_error(Errc::ShapeMismatch, "MatMul+add_rmsnorm: residual [rows,N], gamma [N], N % 256 == 0");
            const size_t need = static_cast<size_t>(rows * (N / 256)) * sizeof(float);
            if (!c.workspace || c.workspace_bytes < need)
              return op_error(Errc::ShapeMismatch, "MatMul+add_rmsnorm: workspace too small");
            g.resid = view_ptr(in[2]);
            g.ssq = static_cast<float*>(c.workspace);
            g.ws = nullptr;
            g.ws_bytes = 0;
            g.bt = c.aux;
            gemm_bf16_tc(g, s);
            rmsnorm_from_stats(view_ptr(out[0]), g.ssq, N / 256, view_ptr(in[3]), view_ptr(out[1]), rows, N,
                               static_cast<float>(ctx_param(c, "eps", 1e-5)), s);
            return launch_status("MatMul+add_rmsnorm");
          }
          if (c.aux) {  // pre-packed [N,K] weight -> tcgen05 path
            g.bt = c.aux;
            gemm_bf16_tc(g, s);
          } else {      // direct opf_launch on a [K,N] weight: CUDA-core path
            g.bt = view_ptr(in[1]);
            g.b_kn = true;
            gemm_bf16_simt(g, s);
          }
        } else {
          k_matmul_exact(dt, view_ptr(in[0]), view_ptr(in[1]), view_ptr(out[0]), rows, K, N, s);
        }
        return launch_status("MatMul");
      }
      case OperatorKind::kElemAdd:
        if (n_in != 2) return op_error(Errc::ShapeMismatch, "ElemAdd takes 2 inputs");
        k_add(dt, view_ptr(in[0]), view_ptr(in[1]), view_ptr(out[0]), view_numel(out[0]), s);
        return launch_status("ElemAdd");
      case OperatorKind::kRowScale:
        k_row_scale(dt, view_ptr(in[0]), view_ptr(out[0]), rows, view_row_elems(in[0]), s);
        return launch_status("RowScale");
      case OperatorKind::kAllReduce: {
        const opf_comm* comm = static_cast<const opf_comm*>(c.comm);
        // one-shot peer-memory all-reduce for small (decode-size) messages; large
        // (prefill) ones go to NCCL's bandwidth-optimal algorithms, whose
        // per-rank NVLink traffic is 2(W-1)/W instead of (W-1) row-planes
        const int64_t msg = view_numel(in[0]) * (in[0].dtype == OPF_F32 ? 4 : in[0].dtype == OPF_I64 ? 8 : 2);
        // a peer-only communicator (no NCCL) takes the peer path at every size
        if (comm && comm->world > 1 && !comm->peer_buf.empty() && comm->world == c.world_size &&
            (msg <= (int64_t{4} << 20) || !comm->nccl) &&
            allreduce_p2p(comm, in[0], out[0], rows, c.max_ctas, s))
          return launch_status("AllReduce(p2p)");
        if (comm && comm->world > 1 && !comm->nccl)
          return op_error(Errc::ConfigError, "AllReduce: peer-only communicator and the message does not "
                                             "fit its window (or is not bf16)");
        if (comm && comm->world > 1) {
          if (comm->world != c.world_size)
            return op_error(Errc::ConfigError, "AllReduce world_size " +
                                                   std::to_string(c.world_size) +
                                                   " != communicator size " +
                                                   std::to_string(comm->world));
          const ncclResult_t r =
              nccl().AllReduce(view_ptr(in[0]), view_ptr(out[0]), static_cast<size_t>(view_numel(in[0])),
                            nccl_type(in[0].dtype), ncclSum, comm->nccl, s);
          if (r != ncclSuccess)
            return op_error(Errc::SchedulerError, std::string("ncclAllReduce: ") + nccl().GetErrorString(r));
          return 0;
        }
        // single device: the reference stand-in (sum of world_size identical replicas)
        k_scale(dt, view_ptr(in[0]), c.world_size, view_ptr(out[0]), view_numel(in[0]), s);
        return launch_status("AllReduce");
      }
      case OperatorKind::kAllToAll: {
        const int64_t cols = view_row_elems(in[0]);
        const void* perm = c.aux ? c.aux : alltoall_perm_device(c.seed, cols);
        k_permute_cols(dt, view_ptr(in[0]), view_ptr(out[0]), rows, cols,
                       static_cast<const uint32_t*>(perm), s);
        return launch_status("AllToAll");
      }
      case OperatorKind::kAttention:
        if (dt == Dtype::kBF16) return op_error(Errc::ShapeMismatch, "Attention stand-in: bf16");
        k_prefix_sum(dt, view_ptr(in[0]), view_ptr(out[0]), rows, view_row_elems(in[0]), s);
        return launch_status("Attention");
      case OperatorKind::kCustom:
        return op_error(Errc::ConfigError, "Custom ops go through the registry");
    }
  } catch (const Error& e) {
    return op_error(e.code(), e.what());
  }
  return op_error(Errc::ConfigError, "unknown operator kind");
}

}  // namespace opflow
