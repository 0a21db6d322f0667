// build_graph / infer_op_outputs for the B200 backend frontend.
// Observable behaviour (op order, wiring, error codes) is kept bit-identical
// to /root/reference/proj/src/graph.cpp so partition plans match exactly.
#include "opflow/graph.hpp"

#include <algorithm>
#include <queue>
#include <set>

#include "opflow/json.hpp"

namespace opflow {

const char* dtype_name(Dtype d) {
  switch (d) {
    case Dtype::kI64: return "i64";
    case Dtype::kF32: return "f32";
    case Dtype::kBF16: return "bf16";
  }
  return "?";
}

const char* kind_name(OperatorKind k) {
  static const char* names[] = {"MatMul",   "ElemAdd",  "RowScale", "AllReduce",
                                "AllToAll", "Attention", "Custom"};
  int i = static_cast<int>(k);
  return (i >= 0 && i < 7) ? names[i] : "?";
}

const char* resource_class_name(ResourceClass c) {
  static const char* names[] = {"compute", "memory", "network"};
  int i = static_cast<int>(c);
  return (i >= 0 && i < 3) ? names[i] : "?";
}

ResourceClass default_resource_class(OperatorKind k) {
  switch (k) {
    case OperatorKind::kElemAdd:
    case OperatorKind::kRowScale:
    case OperatorKind::kAttention: return ResourceClass::kMemory;
    case OperatorKind::kAllReduce:
    case OperatorKind::kAllToAll: return ResourceClass::kNetwork;
    default: return ResourceClass::kCompute;
  }
}

int32_t Graph::tensor_id(const std::string& name) const {
  auto it = tensor_index.find(name);
  if (it == tensor_index.end()) fail(Errc::UnknownTensor, "no tensor named '" + name + "'");
  return it->second;
}

int64_t Graph::nominal_rows() const {
  int64_t r = 1;
  for (int32_t t : graph_inputs)
    if (tensors[t].batch == BatchSemantics::kBatched) r = std::max(r, tensors[t].shape[0]);
  return r;
}

namespace {

std::vector<int64_t> rows_substituted(const TensorMeta& m, int64_t rows) {
  std::vector<int64_t> s = m.shape;
  if (m.batch == BatchSemantics::kBatched && !s.empty()) s[0] = rows;
  return s;
}

bool is_batched(const TensorMeta* m) { return m->batch == BatchSemantics::kBatched; }

}  // namespace

std::vector<InferredOutput> infer_op_outputs(OperatorKind kind,
                                             const std::vector<const TensorMeta*>& in,
                                             int64_t rows,
                                             const std::vector<const TensorMeta*>& declared) {
  std::vector<InferredOutput> out;
  const std::string kn = kind_name(kind);
  switch (kind) {
    case OperatorKind::kMatMul:
      require(in.size() == 2, Errc::ShapeMismatch, "MatMul takes 2 inputs");
      require(is_batched(in[0]) && in[0]->shape.size() == 2, Errc::ShapeMismatch,
              "MatMul lhs must be Batched rank-2");
      require(!is_batched(in[1]) && in[1]->shape.size() == 2, Errc::ShapeMismatch,
              "MatMul rhs must be Replicated rank-2");
      require(in[0]->shape[1] == in[1]->shape[0], Errc::ShapeMismatch,
              "MatMul inner extents disagree");
      out.push_back({{rows, in[1]->shape[1]}, BatchSemantics::kBatched});
      break;
    case OperatorKind::kElemAdd:
      require(in.size() == 2, Errc::ShapeMismatch, "ElemAdd takes 2 inputs");
      require(in[0]->batch == in[1]->batch, Errc::ShapeMismatch,
              "ElemAdd inputs must share batch semantics");
      require(in[0]->shape == in[1]->shape, Errc::ShapeMismatch, "ElemAdd shapes disagree");
      out.push_back({rows_substituted(*in[0], rows), in[0]->batch});
      break;
    case OperatorKind::kRowScale:
    case OperatorKind::kAllReduce:
    case OperatorKind::kAllToAll:
    case OperatorKind::kAttention:
      require(in.size() == 1, Errc::ShapeMismatch, kn + " takes 1 input");
      require(is_batched(in[0]) && !in[0]->shape.empty(), Errc::ShapeMismatch,
              kn + " input must be Batched rank>=1");
      out.push_back({rows_substituted(*in[0], rows), BatchSemantics::kBatched});
      break;
    case OperatorKind::kCustom:
      for (const TensorMeta* m : declared) out.push_back({rows_substituted(*m, rows), m->batch});
      break;
  }
  require(out.size() == declared.size(), Errc::ShapeMismatch, "operator output count mismatch");
  return out;
}

Graph build_graph(const GraphDescription& desc) {
  Graph g;
  // 1. tensor declarations
  for (const TensorDecl& td : desc.tensors) {
    require(!td.name.empty(), Errc::ConfigError, "tensor with empty name");
    require(g.tensor_index.find(td.name) == g.tensor_index.end(), Errc::DuplicateId,
            "duplicate tensor '" + td.name + "'");
    require(!td.shape.empty(), Errc::ShapeMismatch, "tensor '" + td.name + "' has empty shape");
    for (int64_t d : td.shape)
      require(d >= 0, Errc::ShapeMismatch, "tensor '" + td.name + "' has negative extent");
    if (td.batch == BatchSemantics::kBatched)
      require(td.shape[0] >= 1, Errc::ShapeMismatch,
              "batched tensor '" + td.name + "' needs a positive batch extent");
    if (td.role == TensorRole::kWeight)
      require(td.batch == BatchSemantics::kReplicated, Errc::ShapeMismatch,
              "weight '" + td.name + "' must be replicated");
    TensorMeta m;
    m.name = td.name;
    m.shape = td.shape;
    m.batch = td.batch;
    m.dtype = td.dtype;
    m.role = td.role;
    g.tensor_index.emplace(m.name, static_cast<int32_t>(g.tensors.size()));
    g.tensors.push_back(std::move(m));
  }

  // 2. operator resolution in declaration order
  const std::size_t n_ops = desc.operators.size();
  std::vector<OperatorNode> decl_ops;
  decl_ops.reserve(n_ops);
  std::unordered_map<std::string, int32_t> seen_ops;
  std::vector<int32_t> producer(g.tensors.size(), -1);
  for (const OpDecl& od : desc.operators) {
    require(!od.name.empty(), Errc::ConfigError, "operator with empty name");
    require(seen_ops.find(od.name) == seen_ops.end(), Errc::DuplicateId,
            "duplicate operator '" + od.name + "'");
    const int32_t self = static_cast<int32_t>(decl_ops.size());
    seen_ops.emplace(od.name, self);
    OperatorNode n;
    n.name = od.name;
    n.kind = od.kind;
    n.resource_class = od.resource_class ? *od.resource_class : default_resource_class(od.kind);
    n.module_path = od.module_path;
    n.region_tags = od.region_tags;
    n.cost = od.cost ? *od.cost : CostParams{};
    n.attrs = od.attrs;
    for (const std::string& in : od.inputs) n.inputs.push_back(g.tensor_id(in));
    for (const std::string& o : od.outputs) {
      const int32_t t = g.tensor_id(o);
      require(producer[t] < 0, Errc::DuplicateId, "tensor '" + o + "' produced twice");
      const TensorRole r = g.tensors[t].role;
      require(r == TensorRole::kIntermediate || r == TensorRole::kGraphOutput, Errc::DuplicateId,
              "tensor '" + o + "' is externally bound but has a producer");
      producer[t] = self;
      n.outputs.push_back(t);
    }
    require(!n.outputs.empty(), Errc::ConfigError, "operator '" + od.name + "' has no outputs");
    decl_ops.push_back(std::move(n));
  }
  for (std::size_t t = 0; t < g.tensors.size(); ++t) {
    const TensorRole r = g.tensors[t].role;
    if ((r == TensorRole::kIntermediate || r == TensorRole::kGraphOutput) && producer[t] < 0)
      fail(Errc::UnknownTensor, "tensor '" + g.tensors[t].name + "' has no producer");
  }

  // 3. Kahn's algorithm; the frontier is a min-heap on declaration index.
  std::vector<std::vector<int32_t>> succ(n_ops);
  std::vector<int32_t> indeg(n_ops, 0);
  for (std::size_t i = 0; i < n_ops; ++i) {
    std::vector<int32_t> preds;
    for (int32_t t : decl_ops[i].inputs) {
      const int32_t p = producer[t];
      if (p >= 0 && p != static_cast<int32_t>(i)) preds.push_back(p);
    }
    std::sort(preds.begin(), preds.end());
    preds.erase(std::unique(preds.begin(), preds.end()), preds.end());
    for (int32_t p : preds) {
      succ[p].push_back(static_cast<int32_t>(i));
      ++indeg[i];
    }
  }
  std::priority_queue<int32_t, std::vector<int32_t>, std::greater<int32_t>> ready;
  for (std::size_t i = 0; i < n_ops; ++i)
    if (indeg[i] == 0) ready.push(static_cast<int32_t>(i));
  std::vector<int32_t> order;
  order.reserve(n_ops);
  while (!ready.empty()) {
    const int32_t i = ready.top();
    ready.pop();
    order.push_back(i);
    for (int32_t s : succ[i])
      if (--indeg[s] == 0) ready.push(s);
  }
  require(order.size() == n_ops, Errc::CycleDetected, "operator dependency cycle");

  // 4. re-index into topological order and wire producers/consumers
  std::vector<int32_t> pos(n_ops);
  for (std::size_t k = 0; k < order.size(); ++k) pos[order[k]] = static_cast<int32_t>(k);
  g.ops.reserve(n_ops);
  for (int32_t old : order) g.ops.push_back(std::move(decl_ops[old]));
  for (std::size_t i = 0; i < n_ops; ++i) g.op_index.emplace(g.ops[i].name, static_cast<int32_t>(i));
  for (std::size_t t = 0; t < g.tensors.size(); ++t)
    g.tensors[t].producer = producer[t] >= 0 ? pos[producer[t]] : -1;
  for (std::size_t i = 0; i < n_ops; ++i)
    for (int32_t t : g.ops[i].inputs) g.tensors[t].consumers.push_back(static_cast<int32_t>(i));

  // 5. shape validation in topological order
  for (const OperatorNode& op : g.ops) {
    std::vector<const TensorMeta*> ins, outs;
    for (int32_t t : op.inputs) ins.push_back(&g.tensors[t]);
    for (int32_t t : op.outputs) outs.push_back(&g.tensors[t]);
    int64_t rows = 0;
    for (const TensorMeta* m : ins) {
      if (m->batch != BatchSemantics::kBatched || m->shape.empty()) continue;
      require(rows == 0 || rows == m->shape[0], Errc::ShapeMismatch,
              "operator '" + op.name + "' mixes batch extents");
      rows = m->shape[0];
    }
    if (rows == 0) rows = 1;
    const auto inferred = infer_op_outputs(op.kind, ins, rows, outs);
    for (std::size_t j = 0; j < inferred.size(); ++j)
      require(inferred[j].first == outs[j]->shape && inferred[j].second == outs[j]->batch,
              Errc::ShapeMismatch,
              "operator '" + op.name + "' output '" + outs[j]->name + "' shape mismatch");
    if (op.kind == OperatorKind::kAllReduce)
      require(op.attrs.world_size >= 1, Errc::ConfigError,
              "AllReduce '" + op.name + "' needs world_size >= 1");
  }

  // 6. role lists
  for (std::size_t t = 0; t < g.tensors.size(); ++t) {
    const TensorMeta& m = g.tensors[t];
    const int32_t id = static_cast<int32_t>(t);
    if (m.role == TensorRole::kGraphInput)
      g.graph_inputs.push_back(id);
    else if (m.role == TensorRole::kWeight)
      g.weights.push_back(id);
    else if (m.role == TensorRole::kGraphOutput)
      g.graph_outputs.push_back(id);
    else
      require(!m.consumers.empty(), Errc::ConfigError,
              "intermediate tensor '" + m.name + "' has no consumers");
  }
  return g;
}

// ---------------------------------------------------------------- JSON forms

Dtype dtype_from_name(const std::string& s) {
  if (s == "i64" || s == "I64" || s == "int64") return Dtype::kI64;
  if (s == "f32" || s == "F32" || s == "float32") return Dtype::kF32;
  if (s == "bf16" || s == "BF16" || s == "bfloat16") return Dtype::kBF16;
  fail(Errc::ConfigError, "unknown dtype '" + s + "'");
}

OperatorKind kind_from_name(const std::string& s) {
  for (int k = 0; k < 7; ++k)
    if (s == kind_name(static_cast<OperatorKind>(k))) return static_cast<OperatorKind>(k);
  fail(Errc::ConfigError, "unknown operator kind '" + s + "'");
}

ResourceClass resource_class_from_name(const std::string& s) {
  for (int c = 0; c < 3; ++c)
    if (s == resource_class_name(static_cast<ResourceClass>(c)))
      return static_cast<ResourceClass>(c);
  fail(Errc::ConfigError, "unknown resource class '" + s + "'");
}

namespace {

TensorRole role_from_name(const std::string& s) {
  if (s == "input") return TensorRole::kGraphInput;
  if (s == "weight") return TensorRole::kWeight;
  if (s == "intermediate") return TensorRole::kIntermediate;
  if (s == "output") return TensorRole::kGraphOutput;
  fail(Errc::ConfigError, "unknown tensor role '" + s + "'");
}

const char* role_name(TensorRole r) {
  static const char* n[] = {"input", "weight", "intermediate", "output"};
  return n[static_cast<int>(r)];
}

std::string num(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

}  // namespace

GraphDescription description_from_json(const std::string& text) {
  json::Value root;
  try {
    root = json::parse(text);
  } catch (const std::exception& e) {
    fail(Errc::ConfigError, e.what());
  }
  GraphDescription d;
  try {
    if (const json::Value* ts = root.get("tensors")) {
      for (const json::Value& tv : ts->arr()) {
        TensorDecl t;
        t.name = tv.get("name")->str();
        for (const json::Value& e : tv.get("shape")->arr()) t.shape.push_back(e.as_i64());
        if (const json::Value* b = tv.get("batch"))
          t.batch = b->str() == "replicated" ? BatchSemantics::kReplicated
                                              : BatchSemantics::kBatched;
        if (const json::Value* dt = tv.get("dtype")) t.dtype = dtype_from_name(dt->str());
        if (const json::Value* r = tv.get("role")) t.role = role_from_name(r->str());
        d.tensors.push_back(std::move(t));
      }
    }
    if (const json::Value* os = root.get("operators")) {
      for (const json::Value& ov : os->arr()) {
        OpDecl o;
        o.name = ov.get("name")->str();
        o.kind = kind_from_name(ov.get("kind")->str());
        if (const json::Value* v = ov.get("inputs"))
          for (const json::Value& e : v->arr()) o.inputs.push_back(e.str());
        if (const json::Value* v = ov.get("outputs"))
          for (const json::Value& e : v->arr()) o.outputs.push_back(e.str());
        if (const json::Value* v = ov.get("resource_class"); v && !v->is_null())
          o.resource_class = resource_class_from_name(v->str());
        if (const json::Value* v = ov.get("module_path")) o.module_path = v->str();
        if (const json::Value* v = ov.get("region_tags"))
          for (const json::Value& e : v->arr()) o.region_tags.push_back(e.str());
        if (const json::Value* v = ov.get("cost"); v && !v->is_null())
          o.cost = CostParams{v->arr().at(0).num(), v->arr().at(1).num()};
        if (const json::Value* a = ov.get("attrs")) {
          if (const json::Value* v = a->get("world_size")) o.attrs.world_size = v->as_i64();
          if (const json::Value* v = a->get("seed")) o.attrs.seed = v->as_u64();
          if (const json::Value* v = a->get("custom_name")) o.attrs.custom_name = v->str();
          if (const json::Value* v = a->get("params"))
            for (const auto& kv : v->obj()) o.attrs.params[kv.first] = kv.second.num();
        }
        d.operators.push_back(std::move(o));
      }
    }
  } catch (const Error&) {
    throw;
  } catch (const std::exception& e) {
    fail(Errc::ConfigError, std::string("malformed graph description: ") + e.what());
  }
  return d;
}

std::string description_to_json(const GraphDescription& d) {
  std::string s = "{\"tensors\":[";
  for (std::size_t i = 0; i < d.tensors.size(); ++i) {
    const TensorDecl& t = d.tensors[i];
    if (i) s += ',';
    s += "{\"name\":" + json::quote(t.name) + ",\"shape\":" + json::int_list(t.shape) +
         ",\"batch\":\"" + (t.batch == BatchSemantics::kBatched ? "batched" : "replicated") +
         "\",\"dtype\":\"" + dtype_name(t.dtype) + "\",\"role\":\"" + role_name(t.role) + "\"}";
  }
  s += "],\"operators\":[";
  for (std::size_t i = 0; i < d.operators.size(); ++i) {
    const OpDecl& o = d.operators[i];
    if (i) s += ',';
    s += "{\"name\":" + json::quote(o.name) + ",\"kind\":\"" + kind_name(o.kind) +
         "\",\"inputs\":" + json::str_list(o.inputs) + ",\"outputs\":" + json::str_list(o.outputs);
    if (o.resource_class)
      s += std::string(",\"resource_class\":\"") + resource_class_name(*o.resource_class) + "\"";
    s += ",\"module_path\":" + json::quote(o.module_path) +
         ",\"region_tags\":" + json::str_list(o.region_tags);
    if (o.cost) s += ",\"cost\":[" + num(o.cost->alpha) + "," + num(o.cost->beta) + "]";
    s += ",\"attrs\":{\"world_size\":" + std::to_string(o.attrs.world_size) +
         ",\"seed\":" + std::to_string(o.attrs.seed) +
         ",\"custom_name\":" + json::quote(o.attrs.custom_name) + ",\"params\":{";
    bool first = true;
    for (const auto& kv : o.attrs.params) {
      if (!first) s += ',';
      first = false;
      s += json::quote(kv.first) + ":" + num(kv.second);
    }
    s += "}}}";
  }
  s += "]}";
  return s;
}

std::string graph_to_json(const Graph& g) {
  std::string s = "{\"ops\":[";
  for (std::size_t i = 0; i < g.ops.size(); ++i) {
    const OperatorNode& op = g.ops[i];
    if (i) s += ',';
    s += "{\"name\":" + json::quote(op.name) + ",\"kind\":\"" + kind_name(op.kind) +
         "\",\"inputs\":" + json::int_list(op.inputs) + ",\"outputs\":" +
         json::int_list(op.outputs) + ",\"resource_class\":\"" +
         resource_class_name(op.resource_class) + "\"}";
  }
  s += "],\"tensors\":[";
  for (std::size_t t = 0; t < g.tensors.size(); ++t) {
    const TensorMeta& m = g.tensors[t];
    if (t) s += ',';
    s += "{\"name\":" + json::quote(m.name) + ",\"shape\":" + json::int_list(m.shape) +
         ",\"producer\":" + std::to_string(m.producer) +
         ",\"consumers\":" + json::int_list(m.consumers) + "}";
  }
  s += "],\"graph_inputs\":" + json::int_list(g.graph_inputs) +
       ",\"weights\":" + json::int_list(g.weights) +
       ",\"graph_outputs\":" + json::int_list(g.graph_outputs) + "}";
  return s;
}

}  // namespace opflow
