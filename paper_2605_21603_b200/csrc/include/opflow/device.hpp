// Device-op registry and launch helpers.
//
// The device twin of the reference's CustomRegistry
// (/root/reference/proj/include/opflow/eval.hpp:19-28): name -> kernel entry.
// Built-in OperatorKinds dispatch through launch_kind(), the device
// counterpart of eval_op_into (/root/reference/proj/src/eval.cpp:31-107):
// outputs are caller-provided (possibly merge-buffer slices), written in place.
#pragma once

#include <cuda_runtime.h>

#include <functional>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "opflow/graph.hpp"
#include "opflow_b200.h"

namespace opflow {

#define OPF_CUDA(expr)                                                                 \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess)                                                             \
      ::opflow::fail(::opflow::Errc::SchedulerError,                                  \
                     std::string(#expr) + ": " + cudaGetErrorString(_e));              \
  } while (0)

// Workspace bytes an op needs for one launch (0 when none).
using WorkspaceFn = std::function<size_t(const opf_op_ctx&, const opf_view* in, int n_in,
                                         const opf_view* out, int n_out, int64_t rows)>;

struct OpEntry {
  std::string name;
  opf_kernel_fn fn = nullptr;
  ResourceClass rc = ResourceClass::kCompute;
  int n_in = -1;   // -1: any arity
  int n_out = -1;
  WorkspaceFn workspace;
  // weight input packed once per binding by the session (ctx.aux = packed copy):
  // mode 2 = per-expert gate|up pack ([E,K,2I] -> [E,2I,K] interleaved),
  // mode 3 = per-expert transpose ([E,K,N] -> [E,N,K])
  int prepack_input = -1;
  int prepack_mode = 0;
};

class OpRegistry {
 public:
  static OpRegistry& global();
  void add(OpEntry e);
  const OpEntry* find(const std::string& name) const;

 private:
  OpRegistry();
  mutable std::mutex mu_;
  std::unordered_map<std::string, OpEntry> ops_;
};

// View helpers.
inline int64_t view_row_elems(const opf_view& v) {
  int64_t n = 1;
  for (int i = 1; i < v.rank; ++i) n *= v.shape[i];
  return n;
}
inline int64_t view_numel(const opf_view& v) {
  int64_t n = 1;
  for (int i = 0; i < v.rank; ++i) n *= v.shape[i];
  return n;
}
inline char* view_ptr(const opf_view& v) {
  return static_cast<char*>(v.base) + v.elem_offset * dtype_bytes(static_cast<Dtype>(v.dtype));
}
template <class T>
inline T* vptr(const opf_view& v) {
  return reinterpret_cast<T*>(view_ptr(v));
}
opf_view make_view(void* base, int64_t elem_offset, Dtype dt, const std::vector<int64_t>& shape,
                   bool batched);

double ctx_param(const opf_op_ctx& c, const char* name, double dflt);
// Device copy of the AllToAll column permutation (cached; first call uploads,
// so it must happen outside stream capture).
const void* alltoall_perm_device(uint64_t seed, int64_t cols);

// Thread-local C-ABI error message (read back through opf_last_error()).
void set_last_error(const std::string& msg);
// Return a C-ABI status for `code`, recording `msg`.
opf_status op_error(Errc code, const std::string& msg);
// Check the last launch of a kernel wrapper; returns 0 or an error status.
opf_status launch_status(const char* what);

// Built-in kinds (MatMul, ElemAdd, RowScale, AllReduce, AllToAll, Attention).
opf_status launch_kind(const opf_op_ctx& ctx, const opf_view* in, int n_in, opf_view* out,
                       int n_out, int64_t rows, cudaStream_t s);
size_t kind_workspace(const opf_op_ctx& ctx, const opf_view* in, int n_in, const opf_view* out,
                      int n_out, int64_t rows);

// Registration hooks implemented by the kernel translation units.
void register_norm_ops(OpRegistry& r);
void register_llama_ops(OpRegistry& r);
void register_attention_ops(OpRegistry& r);
void register_comm_ops(OpRegistry& r);
void register_moe_ops(OpRegistry& r);
void register_kv_ops(OpRegistry& r);

// ---- kernel launchers used across translation units -------------------------------
// Stand-in kinds (bit-exact with the reference kernels for i64 / f32).
void k_matmul_exact(Dtype dt, const void* a, const void* w, void* out, int64_t rows, int64_t k,
                    int64_t n, cudaStream_t s);
void k_add(Dtype dt, const void* a, const void* b, void* out, int64_t n, cudaStream_t s);
void k_scale(Dtype dt, const void* x, int64_t factor, void* out, int64_t n, cudaStream_t s);
void k_row_scale(Dtype dt, const void* x, void* out, int64_t rows, int64_t cols, cudaStream_t s);
void k_prefix_sum(Dtype dt, const void* x, void* out, int64_t rows, int64_t cols, cudaStream_t s);
void k_permute_cols(Dtype dt, const void* x, void* out, int64_t rows, int64_t cols,
                    const uint32_t* perm, cudaStream_t s);
void k_copy_rows(const void* src, void* dst, int64_t bytes, cudaStream_t s);
void k_transpose_bf16(const void* src, void* dst, int64_t rows, int64_t cols, cudaStream_t s);

// bf16 tensor-core GEMM: C[M,N] = A[M,K] * Bt[N,K]^T (fp32 accumulate in TMEM).
struct GemmArgs {
  const void* a;   // [M,K] row-major bf16, row stride lda elements
  const void* bt;  // [N,K] row-major bf16 (pre-packed weight)
  void* c;         // [M,N] row-major bf16, row stride ldc elements
  int64_t m, n, k, lda, ldc;
  int max_ctas;    // 0 = all SMs
  bool b_kn;       // simt path only: B given as [K,N] row-major instead of [N,K]
  int epi;         // 0 plain; 1 SiLU-mul (Bt packed by k_pack_gate_up, C is [M, N/2]);
                   // 2 rotate-half RoPE on 128-wide q/k heads (C = rope(A B^T))
  const int64_t* pos;  // epi 2: per-row positions
  int rot_heads;       // epi 2: heads [0, rot_heads) rotated, the rest copied
  float log2_theta;    // epi 2
  void* ws;        // split-K workspace (gemm_splitk_workspace bytes), nullptr = no split
  size_t ws_bytes;
  // epi 4: C = x + A B^T (x = resid [M,N]) and per-row, per-256-column-tile sums
  // of squares of the rounded C in ssq [M, N/256] (input of rmsnorm_from_stats)
  const void* resid;
  float* ssq;
};
void gemm_bf16_tc(const GemmArgs& g, cudaStream_t s);
// y = x1 * rsqrt(sum(ssq[row, :]) / H + eps) * g  (the norm half of a MatMul
// fused with add_rmsnorm: x1 and ssq come from the epi-4 GEMM)
void rmsnorm_from_stats(const void* x1, const float* ssq, int64_t n_tiles, const void* gamma, void* y, int64_t rows,
                        int64_t H, float eps, cudaStream_t s);
// Push epilogue (row-parallel GEMM -> all-reduce over peer memory): output row
// r of this rank's partial belongs to owner q = r / blk; the 32-row slab is
// stored at dst[q] + (r - q*blk) * N (this rank's slot in q's window) and
// counted in q's cnt[(r - q*blk) / 32] (red.release.sys) once written.
struct PushArgs {
  void* dst[8];
  uint32_t* cnt[8];
  uint32_t* epoch;  // my call epoch (CTA 0 bumps it; the reduce kernel reads it)
  int64_t blk;
  int world;
};
void gemm_bf16_push(const GemmArgs& g, const PushArgs& p, cudaStream_t s);
// K splits the 2-CTA kernel uses for an (m, n, k) launch on `max_ctas` SMs
// (1 = none) and the workspace they need (fp32 partials + tile semaphores).
int gemm_splitk_splits(int64_t m, int64_t n, int64_t k, int max_ctas);
size_t gemm_splitk_workspace(int64_t m, int64_t n, int64_t k, int max_ctas);
// Grouped per-expert GEMM (MoE): gtab = device tile table [n, (row0, row_end, expert) x n],
// bt = [n_groups * group_n, K]; g.m bounds the rows of a / c, g.n is unused.
// rows per grouped-GEMM tile (128: 1-SM, default; 256: 2-CTA pairs, OPF_MOE_TILE=256);
// the routing kernels build the tile table with the same height
int moe_tile_m();
void gemm_bf16_grouped(const GemmArgs& g, const int32_t* gtab, int64_t max_mtiles, int64_t group_n,
                       int64_t n_groups, cudaStream_t s);
void k_pack_gate_up(const void* src, void* dst, int64_t K, int64_t I, cudaStream_t s);
// Reference CUDA-core GEMM (bf16 in, fp32 accumulate) used by tests as a
// numerics cross-check of the tcgen05 path.
void gemm_bf16_simt(const GemmArgs& g, cudaStream_t s);
int num_sms();

// ---- Programmatic Dependent Launch (PDL) -----------------------------------------
// Hot-path kernels are launched with programmatic stream serialization: the
// next kernel on a stream may be scheduled before this one finishes; it runs
// its prologue (barrier init, TMEM alloc, descriptor prefetch) and blocks in
// pdl_wait() until the previous grid has completed and flushed.  Inside CUDA
// graphs this becomes a programmatic edge.  OPF_PDL=0 disables it.
bool pdl_enabled();
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
#endif

}  // namespace opflow
