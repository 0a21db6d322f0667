// opflow_b200_bridge.hpp — the reference-side binding of the B200 backend.
//
// A header-only C++ adapter a reference maintainer includes next to the
// reference's own headers (/root/reference/proj/include).  It takes the
// reference's types — GraphDescription (graph.hpp:79-106), PartitionRule
// (partition.hpp:15-27), CustomFn-style operator registration (eval.hpp:19-28)
// — serialises them to the backend's JSON form, calls the C-ABI
// (include/opflow_b200.h) and rethrows every non-zero opf_status as the
// reference's own exception, opflow::Error{Errc} (common.hpp:50-58), so the
// reference's error contract holds unchanged.  Compiled and exercised against
// the reference headers by tests/test_bridge.py (tests/bridge/*).
#pragma once

#include <cstdio>
#include <string>
#include <utility>
#include <vector>

#include "opflow/common.hpp"
#include "opflow/graph.hpp"
#include "opflow/partition.hpp"
#include "opflow_b200.h"

namespace opflow::b200 {

// Errc ordinal + 1  ->  the reference exception (same Errc, same message).
inline void check(opf_status s) {
  if (s) throw opflow::Error(static_cast<opflow::Errc>(s - 1), opf_last_error());
}

inline std::string quote(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') {
      o += '\\';
      o += c;
    } else if (static_cast<unsigned char>(c) < 0x20) {
      char b[8];
      std::snprintf(b, sizeof b, "\\u%04x", c);
      o += b;
    } else {
      o += c;
    }
  }
  return o + "\"";
}

inline const char* dtype_json(opflow::Dtype d) {
  switch (d) {
    case opflow::Dtype::kI64: return "i64";
    case opflow::Dtype::kF32: return "f32";
  }
  return "i64";
}
inline const char* role_json(opflow::TensorRole r) {
  switch (r) {
    case opflow::TensorRole::kGraphInput: return "input";
    case opflow::TensorRole::kWeight: return "weight";
    case opflow::TensorRole::kIntermediate: return "intermediate";
    case opflow::TensorRole::kGraphOutput: return "output";
  }
  return "intermediate";
}

// GraphDescription -> the backend's description document.  `params` carries
// per-op numeric attributes the reference keeps outside OpAttrs (the
// reference's CustomFns capture them; the device ops read them from the op).
inline std::string to_json(const opflow::GraphDescription& d,
                           const std::vector<std::pair<std::string, std::vector<std::pair<std::string, double>>>>&
                               params = {}) {
  std::string s = "{\"tensors\":[";
  for (std::size_t i = 0; i < d.tensors.size(); ++i) {
    const auto& t = d.tensors[i];
    s += i ? "," : "";
    s += "{\"name\":" + quote(t.name) + ",\"shape\":[";
    for (std::size_t j = 0; j < t.shape.size(); ++j) s += (j ? "," : "") + std::to_string(t.shape[j]);
    s += std::string("],\"batch\":\"") + (t.batch == opflow::BatchSemantics::kBatched ? "batched" : "replicated") +
         "\",\"dtype\":\"" + dtype_json(t.dtype) + "\",\"role\":\"" + role_json(t.role) + "\"}";
  }
  s += "],\"operators\":[";
  for (std::size_t i = 0; i < d.operators.size(); ++i) {
    const auto& o = d.operators[i];
    s += i ? "," : "";
    s += "{\"name\":" + quote(o.name) + ",\"kind\":" + quote(opflow::kind_name(o.kind)) + ",\"inputs\":[";
    for (std::size_t j = 0; j < o.inputs.size(); ++j) s += (j ? "," : "") + quote(o.inputs[j]);
    s += "],\"outputs\":[";
    for (std::size_t j = 0; j < o.outputs.size(); ++j) s += (j ? "," : "") + quote(o.outputs[j]);
    s += "]";
    if (o.resource_class) s += ",\"resource_class\":" + quote(opflow::resource_class_name(*o.resource_class));
    s += ",\"module_path\":" + quote(o.module_path) + ",\"region_tags\":[";
    for (std::size_t j = 0; j < o.region_tags.size(); ++j) s += (j ? "," : "") + quote(o.region_tags[j]);
    s += "]";
    if (o.cost) {
      char b[96];
      std::snprintf(b, sizeof b, ",\"cost\":[%.17g,%.17g]", o.cost->alpha, o.cost->beta);
      s += b;
    }
    s += ",\"attrs\":{\"world_size\":" + std::to_string(o.attrs.world_size) +
         ",\"seed\":" + std::to_string(o.attrs.seed) + ",\"custom_name\":" + quote(o.attrs.custom_name) +
         ",\"params\":{";
    bool first = true;
    for (const auto& [op, kv] : params)
      if (op == o.name)
        for (const auto& [k, v] : kv) {
          char b[64];
          std::snprintf(b, sizeof b, "%.17g", v);
          s += (first ? "" : ",") + quote(k) + ":" + b;
          first = false;
        }
    s += "}}}";
  }
  return s + "]}";
}

inline std::string to_json(const std::vector<opflow::PartitionRule>& rules) {
  std::string s = "[";
  for (std::size_t i = 0; i < rules.size(); ++i) {
    const auto& r = rules[i];
    const char* k = r.kind == opflow::PartitionRule::Kind::kByModule ? "module"
                    : r.kind == opflow::PartitionRule::Kind::kByFunc ? "func"
                                                                      : "region";
    s += std::string(i ? "," : "") + "{\"kind\":\"" + k + "\",\"pattern\":" + quote(r.pattern) + "}";
  }
  return s + "]";
}

inline std::string take(char* p) {
  std::string s = p ? p : "";
  opf_free_string(p);
  return s;
}

struct Graph {
  opf_graph* h = nullptr;
  Graph() = default;
  Graph(Graph&& o) noexcept : h(std::exchange(o.h, nullptr)) {}
  ~Graph() { opf_graph_free(h); }
  std::string dump() const {
    char* p = nullptr;
    check(opf_graph_dump(h, &p));
    return take(p);
  }
};
struct Plan {
  opf_plan* h = nullptr;
  Plan() = default;
  Plan(Plan&& o) noexcept : h(std::exchange(o.h, nullptr)) {}
  ~Plan() { opf_plan_free(h); }
  std::string dump() const {
    char* p = nullptr;
    check(opf_plan_dump(h, &p));
    return take(p);
  }
};
struct Session {
  opf_session* h = nullptr;
  Session() = default;
  Session(Session&& o) noexcept : h(std::exchange(o.h, nullptr)) {}
  ~Session() { opf_session_free(h); }
};

// replaces opflow::build_graph(desc)                 (graph.hpp:106)
inline Graph build_graph(const opflow::GraphDescription& d) {
  Graph g;
  check(opf_graph_build(to_json(d).c_str(), &g.h));
  return g;
}
inline Graph build_graph(const std::string& desc_json) {
  Graph g;
  check(opf_graph_build(desc_json.c_str(), &g.h));
  return g;
}
// replaces opflow::partition(g, rules)               (partition.hpp:58)
inline Plan partition(const Graph& g, const std::vector<opflow::PartitionRule>& rules) {
  Plan p;
  check(opf_partition(g.h, to_json(rules).c_str(), &p.h));
  return p;
}
// replaces opflow::validate_plan(plan, g)            (partition.hpp:63)
inline void validate_plan(const Plan& p, const Graph& g) { check(opf_validate_plan(p.h, g.h)); }

// replaces CustomRegistry::fns[name] = fn            (eval.hpp:22-28): a
// device kernel registered under the name a Custom op's attrs.custom_name
// (and ByFunc) refer to.
inline void register_op(const std::string& name, opf_kernel_fn fn, opflow::ResourceClass rc, int n_in = -1,
                        int n_out = -1) {
  check(opf_register_op(name.c_str(), fn, static_cast<int32_t>(rc), n_in, n_out));
}

// eval_reference's device counterpart (eval.hpp:40-41): a session over a
// graph + plan, run under a strategy document, async on a CUDA stream.
inline Session make_session(const Graph& g, const Plan& p, const std::string& config_json = "{}") {
  Session s;
  check(opf_session_create(g.h, p.h, config_json.c_str(), nullptr, &s.h));
  return s;
}
inline void bind(Session& s, const std::string& tensor, const opf_view& v) {
  check(opf_session_bind(s.h, tensor.c_str(), &v));
}
inline void run(Session& s, const std::string& strategy_json, void* cuda_stream) {
  check(opf_session_run(s.h, strategy_json.c_str(), cuda_stream));
}
inline void synchronize(Session& s) { check(opf_session_check(s.h)); }

}  // namespace opflow::b200
