// kv_write: store the K / V of new tokens (from the roped fused qkv rows) into
// their paged-cache slots (slot = page * page_size + offset, from the KV-cache
// manager; negative = padding, skipped).  Inputs (qkv_rot [T, (nq+2nkv)*hd],
// slots [T] i64, k_cache, v_cache) -> written [T] i64 (the slots, so the DAG
// can order readers after the write).  Half a warp moves one 256-byte head
// row of K or V with 16-byte vectors; HBM-bound: 2 * nkv * hd * 2 B per token.
#include <cuda_bf16.h>

#include "opflow/device.hpp"

namespace opflow {

namespace {

__global__ void __launch_bounds__(256) kv_write_kernel(const __nv_bfloat16* __restrict__ qkv,
                                                       const int64_t* __restrict__ slots,
                                                       __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc,
                                                       int64_t* __restrict__ written, int64_t T, int nq, int nkv,
                                                       int hd, int page, int hnd, int64_t n_slots) {
  pdl_wait();
  pdl_trigger();
  const int64_t gid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 16;  // (token, head, K|V)
  const int l16 = threadIdx.x % 16;
  const int64_t per_tok = 2LL * nkv;
  const int64_t t = gid / per_tok;
  if (t >= T) return;
  const int rem = static_cast<int>(gid % per_tok);
  const int kh = rem >> 1, is_v = rem & 1;
  const int64_t slot = slots[t];
  if (rem == 0 && l16 == 0) written[t] = slot;
  if (slot < 0 || slot >= n_slots) return;  // padding, or outside the pool (never write past it)
  const int64_t pg = slot / page, off = slot % page;
  const int64_t W = static_cast<int64_t>(nq + 2 * nkv) * hd;
  const __nv_bfloat16* src = qkv + t * W + static_cast<int64_t>(nq + is_v * nkv + kh) * hd;
  const int64_t dst_row = hnd ? ((pg * nkv + kh) * page + off) : ((pg * page + off) * nkv + kh);
  __nv_bfloat16* dst = (is_v ? vc : kc) + dst_row * hd;
  for (int c = l16; c < hd / 8; c += 16)
    reinterpret_cast<uint4*>(dst)[c] = reinterpret_cast<const uint4*>(src)[c];
}

opf_status op_kv_write(const opf_op_ctx* c, const opf_view* in, int32_t n_in, opf_view* out, int32_t n_out,
                       int64_t rows, void* stream) {
  if (n_in != 4 || n_out != 1) return op_error(Errc::ShapeMismatch, "kv_write takes (qkv, slots, k_cache, v_cache) -> slots");
  const int nq = static_cast<int>(ctx_param(*c, "heads", 1));
  const int nkv = static_cast<int>(ctx_param(*c, "kv_heads", 1));
  const int hd = static_cast<int>(ctx_param(*c, "head_dim", 128));
  const int page = static_cast<int>(ctx_param(*c, "page_size", 16));
  const int hnd = static_cast<int>(ctx_param(*c, "kv_layout", 0.0));
  if (in[0].dtype != OPF_BF16 || in[2].dtype != OPF_BF16 || in[3].dtype != OPF_BF16 || in[1].dtype != OPF_I64 ||
      out[0].dtype != OPF_I64 || hd % 8 || view_row_elems(in[0]) != static_cast<int64_t>(nq + 2 * nkv) * hd)
    return op_error(Errc::ShapeMismatch, "kv_write: bf16 qkv / caches, i64 slots, qkv width (heads + 2 kv_heads) * hd");
  const bool shape_ok = in[2].rank == 4 && in[2].shape[3] == hd &&
                        (hnd ? (in[2].shape[1] == nkv && in[2].shape[2] == page)
                             : (in[2].shape[1] == page && in[2].shape[2] == nkv));
  if (!shape_ok) return op_error(Errc::ShapeMismatch, "kv_write: cache shape does not match kv_layout / heads / page");
  bool same = in[3].rank == in[2].rank;
  for (int i = 0; same && i < in[2].rank; ++i) same = in[3].shape[i] == in[2].shape[i];
  if (!same) return op_error(Errc::ShapeMismatch, "kv_write: K and V caches must have identical shapes");
  const int64_t n_slots = in[2].shape[0] * page;
  if (rows == 0) return 0;
  const int64_t threads = rows * 2 * nkv * 16;
  launch_pdl(kv_write_kernel, dim3(static_cast<unsigned>((threads + 255) / 256)), dim3(256), 0,
             static_cast<cudaStream_t>(stream), static_cast<const __nv_bfloat16*>(vptr<__nv_bfloat16>(in[0])),
             static_cast<const int64_t*>(vptr<int64_t>(in[1])), vptr<__nv_bfloat16>(in[2]), vptr<__nv_bfloat16>(in[3]),
             vptr<int64_t>(out[0]), rows, nq, nkv, hd, page, hnd, n_slots);
  return launch_status("kv_write");
}

}  // namespace

void register_kv_ops(OpRegistry& r) { r.add({"kv_write", op_kv_write, ResourceClass::kMemory, 4, 1, {}}); }

}  // namespace opflow
