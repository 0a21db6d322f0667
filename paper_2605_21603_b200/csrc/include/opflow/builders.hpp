// Workload graph builders.
//
// dense_tp / moe_ep / fuse_chain reproduce the reference's canonical stand-in
// graphs op-for-op (/root/reference/proj/src/builders.cpp:43-132, world_size 2
// hard-coded there and here).  llama / llama_decode describe Llama-3-shaped
// decoder layers with Custom device ops (rmsnorm, rope, attn_prefill,
// attn_decode, silu_mul) around reference MatMul / ElemAdd / AllReduce kinds,
// so the same description runs on the CPU oracle and on the B200 engine.
#pragma once

#include <string>

#include "opflow/graph.hpp"

namespace opflow::builders {

struct KindCosts {
  CostParams attention;
  CostParams matmul;
  CostParams allreduce;
  CostParams alltoall;
  CostParams rowscale;
};

GraphDescription dense_tp_graph(int layers, int64_t batch, int64_t hidden, const KindCosts& costs,
                                Dtype dtype = Dtype::kI64);
GraphDescription moe_ep_graph(int layers, int64_t batch, int64_t hidden, const KindCosts& costs,
                              Dtype dtype = Dtype::kI64);
GraphDescription fuse_chain_graph(int layers, int64_t batch, int64_t hidden,
                                  const KindCosts& costs, Dtype dtype = Dtype::kI64);

struct LlamaShape {
  int layers = 1;
  int64_t tokens = 8192;     // rows of the residual stream
  int64_t seq_len = 1024;    // prefill: tokens are tokens/seq_len sequences
  int64_t hidden = 4096;
  int64_t heads = 32;
  int64_t kv_heads = 8;
  int64_t head_dim = 128;
  int64_t inter = 14336;
  int64_t tp = 1;            // tensor-parallel degree (weights are per-rank shards)
  double eps = 1e-5;
  double theta = 500000.0;
  Dtype dtype = Dtype::kBF16;
  // decode only
  bool decode = false;
  int64_t ctx_len = 4096;    // cached context per sequence
  int64_t page_size = 16;
  int64_t num_pages = 0;     // 0 = tokens * ctx_len / page_size
  int64_t kv_layout = 0;     // decode KV pages: 0 NHD [pages, page, kv, hd]; 1 HND [pages, kv, page, hd]
  // paged KV-cache writes: every layer stores the rows' roped K / V into their
  // cache slots (graph input "slots" [T] i64, -1 = skip); prefill needs num_pages
  bool kv_write = false;
  // Qwen3 options: per-head q/k RMSNorm before RoPE; MoE FFN when experts > 0
  bool qk_norm = false;
  int64_t experts = 0;
  int64_t topk = 8;
  int64_t moe_inter = 768;
  int64_t ep = 1;  // expert parallelism: this rank holds experts / ep experts' weights
};

GraphDescription llama_graph(const LlamaShape& s);

// JSON entry used by the C-ABI (opf_builder_json).
std::string build_json(const std::string& name, const std::string& params_json);

}  // namespace opflow::builders
