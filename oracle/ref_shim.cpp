// TEST INFRASTRUCTURE ONLY — the parity checker, never the product path.
//
// C-ABI shim over the UNMODIFIED reference sources (/root/reference/proj/src/*.cpp,
// compiled in place by oracle/Makefile into oracle/_ref/libopflow_ref.so).  It lets
// the Python tests and bench.py's CPU-baseline leg drive the reference's own
//   build_graph   (/root/reference/proj/src/graph.cpp:108-252)
//   partition     (/root/reference/proj/src/partition.cpp:121-230)
//   validate_plan (/root/reference/proj/src/partition.cpp:240-315)
//   eval_reference(/root/reference/proj/src/eval.cpp:109-165)
//   alltoall_permutation (/root/reference/proj/src/eval.cpp:14-20)
// on the same JSON graph descriptions the B200 engine consumes.
//
// Oracle EXTENSIONS (parity unpinned in the reference, which has no Llama op
// semantics — SURVEY.md §8c item 6): CPU reference functions for the Custom ops
// rmsnorm / rope / attn_prefill / attn_decode / silu_mul / add_rmsnorm, registered
// in the reference's own CustomRegistry (proj/include/opflow/eval.hpp:19-28).
// They are cross-checked against oracle/oracle.py (numpy) and torch fp32 in tests.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "opflow/builders.hpp"
#include "opflow/eval.hpp"
#include "opflow/graph.hpp"
#include "opflow/kernels.hpp"
#include "opflow/partition.hpp"
// header-only JSON reader shared with the product (parsing only)
#include "../paper_2605_21603_b200/csrc/include/opflow/json.hpp"

using namespace opflow;

namespace {

thread_local std::string g_err;

int fail_code(const Error& e) {
  g_err = e.what();
  return static_cast<int>(e.code()) + 1;
}

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

Dtype dtype_of(const std::string& s) { return s == "i64" ? Dtype::kI64 : Dtype::kF32; }

OperatorKind kind_of(const std::string& s) {
  static const std::map<std::string, OperatorKind> m = {
      {"MatMul", OperatorKind::kMatMul},       {"ElemAdd", OperatorKind::kElemAdd},
      {"RowScale", OperatorKind::kRowScale},   {"AllReduce", OperatorKind::kAllReduce},
      {"AllToAll", OperatorKind::kAllToAll},   {"Attention", OperatorKind::kAttention},
      {"Custom", OperatorKind::kCustom}};
  auto it = m.find(s);
  if (it == m.end()) fail(Errc::ConfigError, "unknown kind " + s);
  return it->second;
}

struct Parsed {
  GraphDescription desc;
  std::map<std::string, std::map<std::string, double>> custom_params;  // custom_name -> params
};

Parsed parse_desc(const char* text) {
  Parsed out;
  const json::Value root = json::parse(text);
  for (const json::Value& tv : root.get("tensors")->arr()) {
    TensorDecl t;
    t.name = tv.get("name")->str();
    for (const json::Value& e : tv.get("shape")->arr()) t.shape.push_back(e.as_i64());
    if (const json::Value* b = tv.get("batch"))
      t.batch = b->str() == "replicated" ? BatchSemantics::kReplicated : BatchSemantics::kBatched;
    if (const json::Value* d = tv.get("dtype")) t.dtype = dtype_of(d->str());
    if (const json::Value* r = tv.get("role")) {
      const std::string& rs = r->str();
      t.role = rs == "input"    ? TensorRole::kGraphInput
               : rs == "weight" ? TensorRole::kWeight
               : rs == "output" ? TensorRole::kGraphOutput
                                : TensorRole::kIntermediate;
    }
    out.desc.tensors.push_back(std::move(t));
  }
  for (const json::Value& ov : root.get("operators")->arr()) {
    OpDecl o;
    o.name = ov.get("name")->str();
    o.kind = kind_of(ov.get("kind")->str());
    for (const json::Value& e : ov.get("inputs")->arr()) o.inputs.push_back(e.str());
    for (const json::Value& e : ov.get("outputs")->arr()) o.outputs.push_back(e.str());
    if (const json::Value* v = ov.get("resource_class"); v && !v->is_null()) {
      const std::string& s = v->str();
      o.resource_class = s == "memory"    ? ResourceClass::kMemory
                         : s == "network" ? ResourceClass::kNetwork
                                          : ResourceClass::kCompute;
    }
    if (const json::Value* v = ov.get("module_path")) o.module_path = v->str();
    if (const json::Value* v = ov.get("region_tags"))
      for (const json::Value& e : v->arr()) o.region_tags.push_back(e.str());
    if (const json::Value* v = ov.get("cost"); v && !v->is_null())
      o.cost = CostParams{v->arr()[0].num(), v->arr()[1].num()};
    if (const json::Value* a = ov.get("attrs")) {
      if (const json::Value* v = a->get("world_size")) o.attrs.world_size = v->as_i64();
      if (const json::Value* v = a->get("seed")) o.attrs.seed = v->as_u64();
      if (const json::Value* v = a->get("custom_name")) o.attrs.custom_name = v->str();
      if (const json::Value* v = a->get("params")) {
        std::map<std::string, double> ps;
        for (const auto& kv : v->obj()) ps[kv.first] = kv.second.num();
        if (o.kind == OperatorKind::kCustom) {
          auto it = out.custom_params.find(o.attrs.custom_name);
          if (it == out.custom_params.end())
            out.custom_params[o.attrs.custom_name] = ps;
          else if (it->second != ps)
            fail(Errc::ConfigError, "custom '" + o.attrs.custom_name +
                                        "' used with differing params (oracle registry is per name)");
        }
      }
    }
    out.desc.operators.push_back(std::move(o));
  }
  return out;
}

std::vector<PartitionRule> parse_rules(const char* text) {
  std::vector<PartitionRule> rules;
  if (!text || !*text) return rules;
  const json::Value root = json::parse(text);
  for (const json::Value& r : root.arr()) {
    const std::string& k = r.get("kind")->str();
    const std::string& p = r.get("pattern")->str();
    if (k == "module" || k == "by_module")
      rules.push_back(PartitionRule::by_module(p));
    else if (k == "func" || k == "by_func")
      rules.push_back(PartitionRule::by_func(p));
    else
      rules.push_back(PartitionRule::by_region(p));
  }
  return rules;
}

template <class T>
std::string ilist(const std::vector<T>& v) {
  std::string s = "[";
  for (std::size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
  return s + "]";
}

std::string graph_dump(const Graph& g) {
  std::string s = "{\"ops\":[";
  for (std::size_t i = 0; i < g.ops.size(); ++i) {
    const OperatorNode& op = g.ops[i];
    s += (i ? "," : "");
    s += "{\"name\":" + json::quote(op.name) + ",\"kind\":\"" + kind_name(op.kind) +
         "\",\"inputs\":" + ilist(op.inputs) + ",\"outputs\":" + ilist(op.outputs) +
         ",\"resource_class\":\"" + resource_class_name(op.resource_class) + "\"}";
  }
  s += "],\"tensors\":[";
  for (std::size_t t = 0; t < g.tensors.size(); ++t) {
    const TensorMeta& m = g.tensors[t];
    s += (t ? "," : "");
    s += "{\"name\":" + json::quote(m.name) + ",\"shape\":" + ilist(m.shape) +
         ",\"producer\":" + std::to_string(m.producer) + ",\"consumers\":" + ilist(m.consumers) +
         "}";
  }
  s += "],\"graph_inputs\":" + ilist(g.graph_inputs) + ",\"weights\":" + ilist(g.weights) +
       ",\"graph_outputs\":" + ilist(g.graph_outputs) + "}";
  return s;
}

std::string plan_dump(const PartitionPlan& p) {
  std::string s = "{\"subgraphs\":[";
  for (std::size_t i = 0; i < p.subgraphs.size(); ++i) {
    const Subgraph& sg = p.subgraphs[i];
    s += (i ? "," : "");
    s += "{\"id\":" + std::to_string(sg.id) + ",\"ops\":" + ilist(sg.ops) +
         ",\"boundary_inputs\":" + ilist(sg.boundary_inputs) +
         ",\"boundary_outputs\":" + ilist(sg.boundary_outputs) + ",\"label\":" +
         json::quote(sg.label) + ",\"dominant_class\":\"" +
         resource_class_name(sg.dominant_class) + "\"}";
  }
  s += "],\"sg_edges\":[";
  for (std::size_t i = 0; i < p.sg_edges.size(); ++i)
    s += (i ? "," : "") + std::string("[") + std::to_string(p.sg_edges[i].first) + "," +
         std::to_string(p.sg_edges[i].second) + "]";
  std::vector<std::string> tr = p.rule_trace;
  s += "],\"rule_trace\":[";
  for (std::size_t i = 0; i < tr.size(); ++i) s += (i ? "," : "") + json::quote(tr[i]);
  s += "],\"op_to_subgraph\":" + ilist(p.op_to_subgraph) + "}";
  return s;
}

// ---------------------------------------------------------------- Llama Custom ops (fp32)
double P(const std::map<std::string, double>& ps, const char* k, double d) {
  auto it = ps.find(k);
  return it == ps.end() ? d : it->second;
}

TensorValue like(const std::vector<int64_t>& shape) {
  return TensorValue::alloc(shape, Dtype::kF32, BatchSemantics::kBatched, nullptr);
}

void rms_row(const float* x, const float* g, float* y, int64_t n, float eps) {
  double ss = 0.0;
  for (int64_t i = 0; i < n; ++i) ss += double(x[i]) * x[i];
  const float inv = 1.0f / std::sqrt(float(ss / n) + eps);
  for (int64_t i = 0; i < n; ++i) y[i] = x[i] * inv * g[i];
}

CustomRegistry make_registry(const std::map<std::string, std::map<std::string, double>>& cp) {
  CustomRegistry reg;
  auto params = [&](const char* name) {
    auto it = cp.find(name);
    return it == cp.end() ? std::map<std::string, double>{} : it->second;
  };
  {
    const float eps = float(P(params("rmsnorm"), "eps", 1e-5));
    reg.fns["rmsnorm"] = [eps](const std::vector<TensorValue>& in, int64_t rows) {
      const int64_t H = in[0].row_elems();
      TensorValue y = like({rows, H});
      for (int64_t r = 0; r < rows; ++r) rms_row(in[0].f32() + r * H, in[1].f32(), y.f32() + r * H, H, eps);
      return std::vector<TensorValue>{y};
    };
  }
  {
    const float eps = float(P(params("add_rmsnorm"), "eps", 1e-5));
    reg.fns["add_rmsnorm"] = [eps](const std::vector<TensorValue>& in, int64_t rows) {
      const int64_t H = in[0].row_elems();
      TensorValue s = like({rows, H}), y = like({rows, H});
      for (int64_t i = 0; i < rows * H; ++i) s.f32()[i] = in[0].f32()[i] + in[1].f32()[i];
      for (int64_t r = 0; r < rows; ++r) rms_row(s.f32() + r * H, in[2].f32(), y.f32() + r * H, H, eps);
      return std::vector<TensorValue>{s, y};
    };
  }
  {
    const auto ps = params("silu_mul");
    (void)ps;
    reg.fns["silu_mul"] = [](const std::vector<TensorValue>& in, int64_t rows) {
      const int64_t I2 = in[0].row_elems(), I = I2 / 2;
      TensorValue y = like({rows, I});
      for (int64_t r = 0; r < rows; ++r)
        for (int64_t j = 0; j < I; ++j) {
          const float g = in[0].f32()[r * I2 + j], u = in[0].f32()[r * I2 + I + j];
          y.f32()[r * I + j] = g / (1.0f + std::exp(-g)) * u;
        }
      return std::vector<TensorValue>{y};
    };
  }
  {
    // external-operator test op (tests/bridge/ext_op.cu registers the device
    // kernel of the same name through opf_register_op): y = cap * tanh(x / cap)
    const float cap = float(P(params("softcap"), "cap", 30.0));
    reg.fns["softcap"] = [cap](const std::vector<TensorValue>& in, int64_t rows) {
      const int64_t W = in[0].row_elems();
      TensorValue y = like({rows, W});
      for (int64_t i = 0; i < rows * W; ++i) y.f32()[i] = cap * std::tanh(in[0].f32()[i] / cap);
      return std::vector<TensorValue>{y};
    };
  }
  {
    const auto ps = params("rope");
    const int64_t nq = int64_t(P(ps, "heads", 1)), nkv = int64_t(P(ps, "kv_heads", 1)),
                  hd = int64_t(P(ps, "head_dim", 2));
    const double theta = P(ps, "theta", 10000.0);
    reg.fns["rope"] = [=](const std::vector<TensorValue>& in, int64_t rows) {
      const int64_t W = in[0].row_elems();
      TensorValue y = like({rows, W});
      std::memcpy(y.f32(), in[0].f32(), sizeof(float) * rows * W);
      const int64_t half = hd / 2;
      for (int64_t r = 0; r < rows; ++r) {
        const double pos = double(in[1].i64()[r]);
        for (int64_t h = 0; h < nq + nkv; ++h) {  // rotate q heads then k heads, v untouched
          float* v = y.f32() + r * W + h * hd;
          const float* x = in[0].f32() + r * W + h * hd;
          for (int64_t i = 0; i < half; ++i) {
            const double inv = std::pow(theta, -2.0 * double(i) / double(hd));
            const float c = float(std::cos(pos * inv)), s = float(std::sin(pos * inv));
            v[i] = x[i] * c - x[i + half] * s;
            v[i + half] = x[i + half] * c + x[i] * s;
          }
        }
      }
      return std::vector<TensorValue>{y};
    };
  }
  {
    const auto ps = params("attn_prefill");
    const int64_t nq = int64_t(P(ps, "heads", 1)), nkv = int64_t(P(ps, "kv_heads", 1)),
                  hd = int64_t(P(ps, "head_dim", 1)), S = int64_t(P(ps, "seq_len", 1));
    reg.fns["attn_prefill"] = [=](const std::vector<TensorValue>& in, int64_t rows) {
      if (rows % S) fail(Errc::ShapeMismatch, "attn_prefill: rows not a multiple of seq_len");
      const int64_t W = in[0].row_elems(), grp = nq / nkv;
      TensorValue y = like({rows, nq * hd});
      const float scale = 1.0f / std::sqrt(float(hd));
      std::vector<double> p(S);
      for (int64_t r = 0; r < rows; ++r) {
        const int64_t s0 = r - r % S;
        for (int64_t h = 0; h < nq; ++h) {
          const int64_t kh = h / grp;
          const float* q = in[0].f32() + r * W + h * hd;
          double mx = -1e300;
          for (int64_t j = s0; j <= r; ++j) {
            const float* k = in[0].f32() + j * W + (nq + kh) * hd;
            double dot = 0;
            for (int64_t d = 0; d < hd; ++d) dot += double(q[d]) * k[d];
            p[j - s0] = dot * scale;
            mx = std::max(mx, p[j - s0]);
          }
          double den = 0;
          for (int64_t j = s0; j <= r; ++j) den += (p[j - s0] = std::exp(p[j - s0] - mx));
          float* o = y.f32() + r * nq * hd + h * hd;
          for (int64_t d = 0; d < hd; ++d) {
            double acc = 0;
            for (int64_t j = s0; j <= r; ++j)
              acc += p[j - s0] * in[0].f32()[j * W + (nq + nkv + kh) * hd + d];
            o[d] = float(acc / den);
          }
        }
      }
      return std::vector<TensorValue>{y};
    };
  }
  {
    const auto ps = params("attn_decode");
    const int64_t nq = int64_t(P(ps, "heads", 1)), nkv = int64_t(P(ps, "kv_heads", 1)),
                  hd = int64_t(P(ps, "head_dim", 1)), page = int64_t(P(ps, "page_size", 16));
    // in: qkv_rot [B, (nq+2nkv)hd], k_cache/v_cache [pages, page, nkv, hd],
    //     block_table [B, max_pages] (i64), positions = cached context length [B] (i64)
    reg.fns["attn_decode"] = [=](const std::vector<TensorValue>& in, int64_t rows) {
      const int64_t W = in[0].row_elems(), grp = nq / nkv, maxp = in[3].row_elems();
      TensorValue y = like({rows, nq * hd});
      const float scale = 1.0f / std::sqrt(float(hd));
      for (int64_t b = 0; b < rows; ++b) {
        const int64_t ctx = in[4].i64()[b];
        std::vector<double> p(ctx + 1);
        for (int64_t h = 0; h < nq; ++h) {
          const int64_t kh = h / grp;
          const float* q = in[0].f32() + b * W + h * hd;
          auto kptr = [&](int64_t j) -> const float* {
            if (j == ctx) return in[0].f32() + b * W + (nq + kh) * hd;
            const int64_t pg = in[3].i64()[b * maxp + j / page];
            return in[1].f32() + ((pg * page + j % page) * nkv + kh) * hd;
          };
          auto vptr = [&](int64_t j) -> const float* {
            if (j == ctx) return in[0].f32() + b * W + (nq + nkv + kh) * hd;
            const int64_t pg = in[3].i64()[b * maxp + j / page];
            return in[2].f32() + ((pg * page + j % page) * nkv + kh) * hd;
          };
          double mx = -1e300;
          for (int64_t j = 0; j <= ctx; ++j) {
            const float* k = kptr(j);
            double dot = 0;
            for (int64_t d = 0; d < hd; ++d) dot += double(q[d]) * k[d];
            p[j] = dot * scale;
            mx = std::max(mx, p[j]);
          }
          double den = 0;
          for (int64_t j = 0; j <= ctx; ++j) den += (p[j] = std::exp(p[j] - mx));
          float* o = y.f32() + b * nq * hd + h * hd;
          for (int64_t d = 0; d < hd; ++d) {
            double acc = 0;
            for (int64_t j = 0; j <= ctx; ++j) acc += p[j] * vptr(j)[d];
            o[d] = float(acc / den);
          }
        }
      }
      return std::vector<TensorValue>{y};
    };
  }
  return reg;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(char* p) { std::free(p); }

// Build + partition with the reference; dumps in the product's JSON format.
int ref_graph_plan(const char* desc_json, const char* rules_json, char** graph_out,
                   char** plan_out) {
  try {
    Parsed pd = parse_desc(desc_json);
    Graph g = build_graph(pd.desc);
    if (graph_out) *graph_out = dup(graph_dump(g));
    if (plan_out) {
      PartitionPlan p = partition(g, parse_rules(rules_json));
      validate_plan(p, g);
      *plan_out = dup(plan_dump(p));
    }
    return 0;
  } catch (const Error& e) {
    return fail_code(e);
  } catch (const std::exception& e) {
    g_err = e.what();
    return static_cast<int>(Errc::ConfigError) + 1;
  }
}

// Hand-assembled plan (list of op lists) -> finalize_plan + validate_plan.
int ref_validate_hand_plan(const char* desc_json, const int32_t* ops, const int32_t* counts,
                           int32_t n_sg, char** plan_out) {
  try {
    Graph g = build_graph(parse_desc(desc_json).desc);
    PartitionPlan p;
    int32_t k = 0;
    for (int32_t s = 0; s < n_sg; ++s) {
      Subgraph sg;
      for (int32_t j = 0; j < counts[s]; ++j) sg.ops.push_back(ops[k++]);
      sg.label = "hand" + std::to_string(s);
      p.subgraphs.push_back(sg);
      p.rule_trace.push_back("hand");
    }
    finalize_plan(p, g);
    if (plan_out) *plan_out = dup(plan_dump(p));
    validate_plan(p, g);
    return 0;
  } catch (const Error& e) {
    return fail_code(e);
  }
}

int ref_builder(const char* name, int layers, int64_t batch, int64_t hidden, int f32,
                char** graph_out, const char* rules_json, char** plan_out) {
  try {
    builders::KindCosts c;
    c.attention = {1.0, 0.1};
    c.matmul = {1.0, 0.3};
    c.allreduce = {1.0, 0.1};
    c.alltoall = {1.0, 0.1};
    c.rowscale = {1.0, 0.05};
    const Dtype dt = f32 ? Dtype::kF32 : Dtype::kI64;
    const std::string n = name;
    GraphDescription d = n == "dense_tp" ? builders::dense_tp_graph(layers, batch, hidden, c, dt)
                         : n == "moe_ep" ? builders::moe_ep_graph(layers, batch, hidden, c, dt)
                                         : builders::fuse_chain_graph(layers, batch, hidden, c, dt);
    Graph g = build_graph(d);
    if (graph_out) *graph_out = dup(graph_dump(g));
    if (plan_out) *plan_out = dup(plan_dump(partition(g, parse_rules(rules_json))));
    return 0;
  } catch (const Error& e) {
    return fail_code(e);
  }
}

int ref_alltoall_permutation(uint64_t seed, uint32_t cols, uint32_t* out) {
  std::vector<uint32_t> p = alltoall_permutation(seed, cols);
  std::memcpy(out, p.data(), sizeof(uint32_t) * cols);
  return 0;
}

// eval_reference on host buffers.  Inputs/weights are given by name with
// contiguous host data in the oracle dtype (i64 or f32; bf16 graphs evaluate in
// f32).  Batched inputs have `rows` rows.  Outputs are written to caller
// buffers in graph_outputs order.  Returns seconds spent in eval_reference.
int ref_eval(const char* desc_json, int64_t rows, int32_t n_bind, const char* const* names,
             const void* const* data, int32_t n_out, void* const* out_data, double* seconds) {
  try {
    Parsed pd = parse_desc(desc_json);
    Graph g = build_graph(pd.desc);
    CustomRegistry reg = make_registry(pd.custom_params);
    Bindings b;
    for (int32_t i = 0; i < n_bind; ++i) {
      const int32_t t = g.tensor_id(names[i]);
      const TensorMeta& m = g.tensors[t];
      std::vector<int64_t> shape = m.shape;
      if (m.batch == BatchSemantics::kBatched) shape[0] = rows;
      TensorValue v = TensorValue::alloc(shape, m.dtype, m.batch, nullptr);
      std::memcpy(m.dtype == Dtype::kI64 ? static_cast<void*>(v.i64()) : static_cast<void*>(v.f32()),
                  data[i], v.numel() * dtype_bytes(m.dtype));
      b.emplace(t, v);
    }
    const auto t0 = std::chrono::steady_clock::now();
    Bindings out = eval_reference(g, b, reg);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    if (n_out != static_cast<int32_t>(g.graph_outputs.size()))
      fail(Errc::ShapeMismatch, "ref_eval: output count mismatch");
    for (int32_t i = 0; i < n_out; ++i) {
      const TensorValue& v = out.at(g.graph_outputs[i]);
      std::memcpy(out_data[i],
                  v.dtype == Dtype::kI64 ? static_cast<const void*>(v.i64())
                                         : static_cast<const void*>(v.f32()),
                  v.numel() * dtype_bytes(v.dtype));
    }
    return 0;
  } catch (const Error& e) {
    return fail_code(e);
  } catch (const std::exception& e) {
    g_err = e.what();
    return static_cast<int>(Errc::ConfigError) + 1;
  }
}

// Reference kernels, exposed for known-answer tests of the restatement.
void ref_matmul_f32(const float* a, const float* w, float* o, uint64_t r, uint64_t k, uint64_t n) {
  kernels::matmul_f32(a, w, o, r, k, n);
}
void ref_row_scale_f32(const float* x, float* o, uint64_t r, uint64_t c) {
  kernels::row_scale_f32(x, o, r, c);
}
const char* ref_backend() { return kernels::backend_name(kernels::active_backend()); }

}  // extern "C"
