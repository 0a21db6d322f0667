#include "opflow/builders.hpp"

#include <map>

#include "opflow/json.hpp"

namespace opflow::builders {

namespace {

class DescWriter {
 public:
  explicit DescWriter(Dtype dt) : dtype_(dt) {}

  std::string tensor(const std::string& name, std::vector<int64_t> shape, BatchSemantics b,
                     TensorRole role, std::optional<Dtype> dt = std::nullopt) {
    d_.tensors.push_back(TensorDecl{name, std::move(shape), b, dt ? *dt : dtype_, role});
    return name;
  }
  std::string act(const std::string& name, std::vector<int64_t> shape, bool is_out = false) {
    return tensor(name, std::move(shape), BatchSemantics::kBatched,
                  is_out ? TensorRole::kGraphOutput : TensorRole::kIntermediate);
  }
  std::string weight(const std::string& name, std::vector<int64_t> shape,
                     std::optional<Dtype> dt = std::nullopt) {
    return tensor(name, std::move(shape), BatchSemantics::kReplicated, TensorRole::kWeight, dt);
  }
  OpDecl& op(const std::string& name, OperatorKind kind, std::vector<std::string> ins,
             std::vector<std::string> outs, const std::string& module, CostParams cost) {
    OpDecl o;
    o.name = name;
    o.kind = kind;
    o.inputs = std::move(ins);
    o.outputs = std::move(outs);
    o.module_path = module;
    o.cost = cost;
    d_.operators.push_back(std::move(o));
    return d_.operators.back();
  }
  OpDecl& custom(const std::string& name, const std::string& fn, std::vector<std::string> ins,
                 std::vector<std::string> outs, const std::string& module, ResourceClass rc,
                 CostParams cost) {
    OpDecl& o = op(name, OperatorKind::kCustom, std::move(ins), std::move(outs), module, cost);
    o.attrs.custom_name = fn;
    o.resource_class = rc;
    return o;
  }
  GraphDescription take() { return std::move(d_); }

 private:
  Dtype dtype_;
  GraphDescription d_;
};

std::string L(int l) { return "layer" + std::to_string(l); }

}  // namespace

GraphDescription dense_tp_graph(int layers, int64_t B, int64_t H, const KindCosts& c, Dtype dt) {
  DescWriter w(dt);
  std::string x = w.tensor("x", {B, H}, BatchSemantics::kBatched, TensorRole::kGraphInput);
  for (int l = 0; l < layers; ++l) {
    const std::string p = L(l);
    const std::string wt = w.weight(p + ".w", {H, H});
    const std::string a = w.act(p + ".attn_out", {B, H});
    const std::string m = w.act(p + ".mm_out", {B, H});
    const std::string r = w.act(p + ".ar_out", {B, H});
    const std::string o = w.act(p + ".out", {B, H}, l == layers - 1);
    w.op(p + ".attn", OperatorKind::kAttention, {x}, {a}, p + ".attn", c.attention);
    w.op(p + ".mlp", OperatorKind::kMatMul, {a, wt}, {m}, p + ".mlp", c.matmul);
    w.op(p + ".comm", OperatorKind::kAllReduce, {m}, {r}, p + ".comm", c.allreduce)
        .attrs.world_size = 2;
    w.op(p + ".norm", OperatorKind::kRowScale, {r}, {o}, p + ".norm", c.rowscale);
    x = o;
  }
  return w.take();
}

GraphDescription moe_ep_graph(int layers, int64_t B, int64_t H, const KindCosts& c, Dtype dt) {
  DescWriter w(dt);
  std::string x = w.tensor("x", {B, H}, BatchSemantics::kBatched, TensorRole::kGraphInput);
  for (int l = 0; l < layers; ++l) {
    const std::string p = L(l);
    const std::string wt = w.weight(p + ".w_exp", {H, H});
    const std::string a = w.act(p + ".attn_out", {B, H});
    const std::string d = w.act(p + ".disp_out", {B, H});
    const std::string e = w.act(p + ".exp_out", {B, H});
    const std::string cb = w.act(p + ".comb_out", {B, H});
    const std::string o = w.act(p + ".out", {B, H}, l == layers - 1);
    w.op(p + ".attn", OperatorKind::kAttention, {x}, {a}, p + ".attn", c.attention);
    w.op(p + ".dispatch", OperatorKind::kAllToAll, {a}, {d}, p + ".moe.dispatch", c.alltoall)
        .attrs.seed = static_cast<uint64_t>(l) + 1;
    w.op(p + ".experts", OperatorKind::kMatMul, {d, wt}, {e}, p + ".moe.experts", c.matmul);
    w.op(p + ".combine", OperatorKind::kAllReduce, {e}, {cb}, p + ".moe.combine", c.allreduce)
        .attrs.world_size = 2;
    w.op(p + ".post", OperatorKind::kRowScale, {cb}, {o}, p + ".post", c.rowscale);
    x = o;
  }
  return w.take();
}

GraphDescription fuse_chain_graph(int layers, int64_t B, int64_t H, const KindCosts& c, Dtype dt) {
  DescWriter w(dt);
  std::string x = w.tensor("x", {B, H}, BatchSemantics::kBatched, TensorRole::kGraphInput);
  for (int l = 0; l < layers; ++l) {
    const std::string p = L(l);
    const std::string wt = w.weight(p + ".w", {H, H});
    const std::string m = w.act(p + ".mm_out", {B, H});
    const std::string r = w.act(p + ".ar_out", {B, H});
    const std::string o = w.act(p + ".out", {B, H}, l == layers - 1);
    w.op(p + ".mlp", OperatorKind::kMatMul, {x, wt}, {m}, p + ".mlp", c.matmul);
    w.op(p + ".comm", OperatorKind::kAllReduce, {m}, {r}, p + ".comm", c.allreduce)
        .attrs.world_size = 2;
    w.op(p + ".norm", OperatorKind::kRowScale, {r}, {o}, p + ".norm", c.rowscale);
    x = o;
  }
  return w.take();
}

GraphDescription llama_graph(const LlamaShape& s) {
  require(s.tp >= 1 && s.heads % s.tp == 0 && s.kv_heads % s.tp == 0 && s.inter % s.tp == 0,
          Errc::ConfigError, "llama: tp must divide heads, kv_heads and inter");
  require(s.decode || s.tokens % s.seq_len == 0, Errc::ConfigError,
          "llama: tokens must be a multiple of seq_len");
  require(s.experts == 0 || (s.tp == 1 && s.topk >= 1 && s.topk <= s.experts), Errc::ConfigError,
          "moe: experts need tp == 1 and 1 <= topk <= experts");
  require(s.ep >= 1 && s.ep <= 8 && (s.experts == 0 ? s.ep == 1 : s.experts % s.ep == 0), Errc::ConfigError,
          "moe: ep must be 1..8 and divide experts");
  DescWriter w(s.dtype);
  const int64_t T = s.tokens, H = s.hidden, hd = s.head_dim;
  const int64_t nq = s.heads / s.tp, nkv = s.kv_heads / s.tp, I = s.inter / s.tp;
  const int64_t nqkv = (nq + 2 * nkv) * hd;
  // Cost model (alpha = fixed launch + weight read, beta = per-token), in
  // microseconds at B200 roofline; only used for dominant-class labels and the
  // strategies' threshold guard.
  auto gemm_cost = [&](int64_t k, int64_t n) {
    return CostParams{2.0 + (2.0 * k * n) / 6.5e3 * 1e-3, 2.0 * k * n / 1.4e6 * 1e-3};
  };
  const CostParams mem_cost{2.0, H * 4.0 / 6.5e6};
  std::string x = w.tensor("x", {T, H}, BatchSemantics::kBatched, TensorRole::kGraphInput);
  const std::string pos =
      w.tensor("positions", {T}, BatchSemantics::kBatched, TensorRole::kGraphInput, Dtype::kI64);
  std::string table, kc, vc;
  const int64_t max_pages = (s.ctx_len + s.page_size - 1) / s.page_size;
  if (s.decode)
    table = w.tensor("block_table", {T, max_pages}, BatchSemantics::kBatched,
                     TensorRole::kGraphInput, Dtype::kI64);
  require(!s.kv_write || s.decode || s.num_pages > 0, Errc::ConfigError,
          "llama: kv_write in prefill needs num_pages (the cache pool size)");
  std::string slots;
  if (s.kv_write)
    slots = w.tensor("slots", {T}, BatchSemantics::kBatched, TensorRole::kGraphInput, Dtype::kI64);
  // Layer l: [rmsnorm (l==0)] qkv -> rope -> attn -> o_proj [-> AllReduce]
  //   -> add_rmsnorm (residual + mlp norm) -> gate_up -> silu_mul -> down
  //   [-> AllReduce] -> add_rmsnorm with layer l+1's attn norm (ElemAdd on the
  //   last layer).  Fused residual+norm is the vLLM/TokenWeave layer shape.
  std::string h1 = w.act("layer0.h1", {T, H});
  w.custom("layer0.attn_norm", "rmsnorm", {x, w.weight("layer0.attn_norm.w", {H})}, {h1},
           "layer0.attn.norm", ResourceClass::kMemory, mem_cost)
      .attrs.params = {{"eps", s.eps}};
  for (int l = 0; l < s.layers; ++l) {
    const std::string p = L(l);
    const bool last = l == s.layers - 1;
    const std::string wqkv = w.weight(p + ".qkv.w", {H, nqkv});
    const std::string wo = w.weight(p + ".o.w", {nq * hd, H});
    const std::string g2 = w.weight(p + ".mlp_norm.w", {H});
    const bool moe = s.experts > 0;
    const int64_t E = s.experts, K = s.topk, MI = s.moe_inter, EP = s.ep, El = moe ? E / EP : 0;
    const std::string wgu = moe ? w.weight(p + ".experts.gate_up.w", {El, H, 2 * MI})
                                : w.weight(p + ".gate_up.w", {H, 2 * I});
    const std::string wd = moe ? w.weight(p + ".experts.down.w", {El, MI, H}) : w.weight(p + ".down.w", {I, H});
    if (s.decode || s.kv_write) {
      const int64_t pages = s.num_pages ? s.num_pages : T * max_pages;
      const std::vector<int64_t> cshape = s.kv_layout == 1 ? std::vector<int64_t>{pages, nkv, s.page_size, hd}
                                                           : std::vector<int64_t>{pages, s.page_size, nkv, hd};
      kc = w.weight(p + ".k_cache", cshape);
      vc = w.weight(p + ".v_cache", cshape);
    }
    const std::string qkv = w.act(p + ".qkv", {T, nqkv});
    const std::string qkvr = w.act(p + ".qkv_rot", {T, nqkv});
    const std::string ctx = w.act(p + ".ctx", {T, nq * hd});
    const std::string o = w.act(p + ".o", {T, H});
    const std::string x1 = w.act(p + ".x1", {T, H});
    const std::string h2 = w.act(p + ".h2", {T, H});
    const std::string dn = w.act(p + ".down_out", {T, H});

    w.op(p + ".qkv_proj", OperatorKind::kMatMul, {h1, wqkv}, {qkv}, p + ".attn.qkv",
         gemm_cost(H, nqkv));
    if (s.qk_norm) {
      w.custom(p + ".rope", "qk_norm_rope",
               {qkv, pos, w.weight(p + ".q_norm.w", {hd}), w.weight(p + ".k_norm.w", {hd})}, {qkvr},
               p + ".attn.rope", ResourceClass::kMemory, mem_cost)
          .attrs.params = {{"heads", double(nq)}, {"kv_heads", double(nkv)}, {"head_dim", double(hd)},
                           {"theta", s.theta}, {"eps", s.eps}};
    } else {
      w.custom(p + ".rope", "rope", {qkv, pos}, {qkvr}, p + ".attn.rope", ResourceClass::kMemory,
               mem_cost)
          .attrs.params = {{"heads", double(nq)}, {"kv_heads", double(nkv)},
                           {"head_dim", double(hd)}, {"theta", s.theta}};
    }
    if (s.kv_write) {  // this step's rows join the paged cache (decode reads ctx < their position)
      // a graph output (the graph model allows no dead intermediates); unbound,
      // it lives in the session arena
      const std::string wr = w.tensor(p + ".kv_written", {T}, BatchSemantics::kBatched,
                                      TensorRole::kGraphOutput, Dtype::kI64);
      w.custom(p + ".kv_write", "kv_write", {qkvr, slots, kc, vc}, {wr}, p + ".attn.kv", ResourceClass::kMemory,
               CostParams{2.0, nkv * hd * 4.0 / 6.5e6})
          .attrs.params = {{"heads", double(nq)}, {"kv_heads", double(nkv)}, {"head_dim", double(hd)},
                           {"page_size", double(s.page_size)}, {"kv_layout", double(s.kv_layout)}};
    }
    if (s.decode) {
      w.custom(p + ".attn", "attn_decode", {qkvr, kc, vc, table, pos}, {ctx}, p + ".attn.core",
               ResourceClass::kMemory, mem_cost)
          .attrs.params = {{"heads", double(nq)}, {"kv_heads", double(nkv)},
                           {"head_dim", double(hd)}, {"page_size", double(s.page_size)},
                           {"kv_layout", double(s.kv_layout)}};
    } else {
      w.custom(p + ".attn", "attn_prefill", {qkvr}, {ctx}, p + ".attn.core",
               ResourceClass::kCompute, mem_cost)
          .attrs.params = {{"heads", double(nq)}, {"kv_heads", double(nkv)},
                           {"head_dim", double(hd)}, {"seq_len", double(s.seq_len)}};
    }
    w.op(p + ".o_proj", OperatorKind::kMatMul, {ctx, wo}, {o}, p + ".attn.o",
         gemm_cost(nq * hd, H));
    std::string o_in = o;
    if (s.tp > 1) {
      o_in = w.act(p + ".o_ar", {T, H});
      w.op(p + ".o_allreduce", OperatorKind::kAllReduce, {o}, {o_in}, p + ".attn.comm",
           CostParams{5.0, H * 2.0 / 0.8e6})
          .attrs.world_size = s.tp;
    }
    w.custom(p + ".attn_resid_norm", "add_rmsnorm", {x, o_in, g2}, {x1, h2}, p + ".attn.resid",
             ResourceClass::kMemory, mem_cost)
        .attrs.params = {{"eps", s.eps}};
    if (moe) {
      // Qwen3 MoE FFN: router GEMM -> top-k -> dispatch (EP all-to-all site)
      // -> grouped expert GEMMs -> combine (EP all-to-all site)
      const std::string logits = w.act(p + ".router_logits", {T, E});
      const std::string ids = w.tensor(p + ".topk_ids", {T, K}, BatchSemantics::kBatched,
                                       TensorRole::kIntermediate, Dtype::kI64);
      const std::string wts = w.tensor(p + ".topk_w", {T, K}, BatchSemantics::kBatched,
                                       TensorRole::kIntermediate, Dtype::kF32);
      const std::vector<std::pair<std::string, double>> mp = {
          {"experts", double(E)}, {"topk", double(K)}, {"ep", double(EP)}};
      auto params = [&](std::initializer_list<std::pair<const std::string, double>> extra) {
        std::map<std::string, double> m(mp.begin(), mp.end());
        for (const auto& kv : extra) m[kv.first] = kv.second;
        return m;
      };
      w.op(p + ".router", OperatorKind::kMatMul, {h2, w.weight(p + ".router.w", {H, E})}, {logits},
           p + ".moe.router", gemm_cost(H, E));
      w.custom(p + ".topk", "moe_topk", {logits}, {ids, wts}, p + ".moe.topk", ResourceClass::kMemory,
               CostParams{2.0, E * 2.0 / 6.5e6})
          .attrs.params = params({{"renorm", 1.0}});
      const CostParams a2a{5.0, K * H * 4.0 / (EP > 1 ? 0.8e6 : 6.5e6)};
      if (EP == 1) {
        const std::string xd = w.act(p + ".dispatched", {T, K * H});
        const std::string slot = w.tensor(p + ".slot", {T, K}, BatchSemantics::kBatched,
                                          TensorRole::kIntermediate, Dtype::kI64);
        const std::string hd_ = w.act(p + ".expert_act", {T, K * MI});
        const std::string yd = w.act(p + ".expert_out", {T, K * H});
        w.custom(p + ".dispatch", "moe_dispatch", {h2, ids}, {xd, slot}, p + ".moe.dispatch",
                 ResourceClass::kNetwork, a2a)
            .attrs.params = params({});
        w.custom(p + ".experts_gate_up", "moe_gate_up", {xd, ids, wgu}, {hd_}, p + ".moe.experts",
                 ResourceClass::kCompute, CostParams{2.0, K * 2.0 * H * 2 * MI / 1.4e9})
            .attrs.params = params({});
        w.custom(p + ".experts_down", "moe_down", {hd_, ids, wd}, {yd}, p + ".moe.experts",
                 ResourceClass::kCompute, CostParams{2.0, K * 2.0 * MI * H / 1.4e9})
            .attrs.params = params({});
        w.custom(p + ".combine", "moe_combine", {yd, slot, wts}, {dn}, p + ".moe.combine",
                 ResourceClass::kNetwork, CostParams{5.0, K * H * 2.0 / 6.5e6})
            .attrs.params = params({});
      } else {
        // expert parallel: rows travel to the owner rank's arena and back
        const std::string xr = w.act(p + ".dispatched", {T, EP * K * H});
        const std::string rinfo = w.tensor(p + ".recv_info", {T, EP * K + El}, BatchSemantics::kBatched,
                                           TensorRole::kIntermediate, Dtype::kI64);
        const std::string hr = w.act(p + ".expert_act", {T, EP * K * MI});
        const std::string yr = w.act(p + ".expert_out", {T, EP * K * H});
        w.custom(p + ".dispatch", "moe_ep_dispatch", {h2, ids}, {xr, rinfo}, p + ".moe.dispatch",
                 ResourceClass::kNetwork, a2a)
            .attrs.params = params({});
        w.custom(p + ".experts_gate_up", "moe_gate_up", {xr, rinfo, wgu}, {hr}, p + ".moe.experts",
                 ResourceClass::kCompute, CostParams{2.0, K * 2.0 * H * 2 * MI / 1.4e9})
            .attrs.params = params({});
        w.custom(p + ".experts_down", "moe_down", {hr, rinfo, wd}, {yr}, p + ".moe.experts",
                 ResourceClass::kCompute, CostParams{2.0, K * 2.0 * MI * H / 1.4e9})
            .attrs.params = params({});
        w.custom(p + ".combine", "moe_ep_combine", {yr, rinfo, wts, ids}, {dn}, p + ".moe.combine",
                 ResourceClass::kNetwork, a2a)
            .attrs.params = params({});
      }
    } else {
      const std::string gu = w.act(p + ".gu", {T, 2 * I});
      const std::string a = w.act(p + ".act", {T, I});
      w.op(p + ".gate_up", OperatorKind::kMatMul, {h2, wgu}, {gu}, p + ".mlp.gate_up",
           gemm_cost(H, 2 * I));
      w.custom(p + ".act", "silu_mul", {gu}, {a}, p + ".mlp.act", ResourceClass::kMemory, mem_cost);
      w.op(p + ".down", OperatorKind::kMatMul, {a, wd}, {dn}, p + ".mlp.down", gemm_cost(I, H));
    }
    std::string d_in = dn;
    if (s.tp > 1) {
      d_in = w.act(p + ".down_ar", {T, H});
      w.op(p + ".down_allreduce", OperatorKind::kAllReduce, {dn}, {d_in}, p + ".mlp.comm",
           CostParams{5.0, H * 2.0 / 0.8e6})
          .attrs.world_size = s.tp;
    }
    if (last) {
      const std::string out = w.act(p + ".out", {T, H}, true);
      w.op(p + ".mlp_resid", OperatorKind::kElemAdd, {x1, d_in}, {out}, p + ".mlp.resid",
           mem_cost);
    } else {
      const std::string nx = L(l + 1);
      const std::string xn = w.act(p + ".out", {T, H});
      const std::string h1n = w.act(nx + ".h1", {T, H});
      w.custom(p + ".mlp_resid_norm", "add_rmsnorm",
               {x1, d_in, w.weight(nx + ".attn_norm.w", {H})}, {xn, h1n}, p + ".mlp.resid",
               ResourceClass::kMemory, mem_cost)
          .attrs.params = {{"eps", s.eps}};
      x = xn;
      h1 = h1n;
    }
  }
  return w.take();
}

namespace {

CostParams cost_of(const json::Value* costs, const char* key, CostParams dflt) {
  if (!costs) return dflt;
  const json::Value* v = costs->get(key);
  if (!v) return dflt;
  return CostParams{v->arr().at(0).num(), v->arr().at(1).num()};
}

int64_t geti(const json::Value& p, const char* k, int64_t d) {
  const json::Value* v = p.get(k);
  return v ? v->as_i64() : d;
}
double getd(const json::Value& p, const char* k, double d) {
  const json::Value* v = p.get(k);
  return v ? v->num() : d;
}

}  // namespace

std::string build_json(const std::string& name, const std::string& params_json) {
  json::Value p;
  try {
    p = json::parse(params_json.empty() ? "{}" : params_json);
  } catch (const std::exception& e) {
    fail(Errc::ConfigError, e.what());
  }
  const json::Value* dtv = p.get("dtype");
  const Dtype dt = dtv ? dtype_from_name(dtv->str()) : Dtype::kI64;
  if (name == "dense_tp" || name == "moe_ep" || name == "fuse_chain") {
    const json::Value* c = p.get("costs");
    KindCosts k;
    k.attention = cost_of(c, "attention", {1.0, 0.1});
    k.matmul = cost_of(c, "matmul", {1.0, 0.3});
    k.allreduce = cost_of(c, "allreduce", {1.0, 0.1});
    k.alltoall = cost_of(c, "alltoall", {1.0, 0.1});
    k.rowscale = cost_of(c, "rowscale", {1.0, 0.05});
    const int layers = static_cast<int>(geti(p, "layers", 2));
    const int64_t B = geti(p, "batch", 8), H = geti(p, "hidden", 4);
    GraphDescription d = name == "dense_tp"  ? dense_tp_graph(layers, B, H, k, dt)
                         : name == "moe_ep"  ? moe_ep_graph(layers, B, H, k, dt)
                                             : fuse_chain_graph(layers, B, H, k, dt);
    return description_to_json(d);
  }
  if (name == "llama" || name == "llama_decode" || name == "toy_decoder" || name == "qwen3_moe") {
    LlamaShape s;
    if (name == "qwen3_moe") {  // BASELINE.json configs[4]: Qwen3-30B-A3B-shaped layer
      s.layers = 1;
      s.hidden = 2048;
      s.heads = 32;
      s.kv_heads = 4;
      s.head_dim = 128;
      s.inter = 6144;
      s.eps = 1e-6;
      s.theta = 1000000.0;
      s.qk_norm = true;
      s.experts = 128;
      s.topk = 8;
      s.moe_inter = 768;
    }
    if (name == "toy_decoder") {  // BASELINE.json configs[0]
      s.layers = 2;
      s.tokens = 8 * 128;
      s.seq_len = 128;
      s.hidden = 512;
      s.heads = 8;
      s.kv_heads = 8;
      s.head_dim = 64;
      s.inter = 1536;
      s.dtype = Dtype::kF32;
    }
    s.decode = name == "llama_decode";
    if (s.decode) {
      s.tokens = 512;
      s.seq_len = 1;
    }
    s.layers = static_cast<int>(geti(p, "layers", s.layers));
    s.tokens = geti(p, "tokens", s.tokens);
    s.seq_len = geti(p, "seq_len", s.seq_len);
    s.hidden = geti(p, "hidden", s.hidden);
    s.heads = geti(p, "heads", s.heads);
    s.kv_heads = geti(p, "kv_heads", s.kv_heads);
    s.head_dim = geti(p, "head_dim", s.head_dim);
    s.inter = geti(p, "inter", s.inter);
    s.tp = geti(p, "tp", s.tp);
    s.eps = getd(p, "eps", s.eps);
    s.theta = getd(p, "theta", s.theta);
    s.ctx_len = geti(p, "ctx_len", s.ctx_len);
    s.page_size = geti(p, "page_size", s.page_size);
    s.num_pages = geti(p, "num_pages", s.num_pages);
    s.kv_layout = geti(p, "kv_layout", s.kv_layout);
    s.kv_write = geti(p, "kv_write", s.kv_write ? 1 : 0) != 0;
    s.experts = geti(p, "experts", s.experts);
    s.topk = geti(p, "topk", s.topk);
    s.moe_inter = geti(p, "moe_inter", s.moe_inter);
    s.ep = geti(p, "ep", s.ep);
    s.qk_norm = geti(p, "qk_norm", s.qk_norm ? 1 : 0) != 0;
    if (dtv) s.dtype = dt;
    return description_to_json(llama_graph(s));
  }
  fail(Errc::ConfigError, "unknown builder '" + name + "'");
}

}  // namespace opflow::builders
