// Reference-side program: the reference's own C++ types and builders drive the
// B200 backend through include/opflow_b200_bridge.hpp, next to the reference's
// own build_graph / partition on the same descriptions.  Prints one JSON line
// per case; tests/test_bridge.py compares the two sides.  Compiled against
// /root/reference/proj/include + the reference's frontend sources (in place).
#include <cstdio>
#include <string>
#include <vector>

#include "opflow/builders.hpp"
#include "opflow/partition.hpp"
#include "opflow_b200_bridge.hpp"

using namespace opflow;
using b200::quote;

static std::string ints(const std::vector<int32_t>& v) {
  std::string s = "[";
  for (std::size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
  return s + "]";
}

// reference Graph -> the same document shape opf_graph_dump emits
static std::string ref_graph_json(const Graph& g) {
  std::string s = "{\"ops\":[";
  for (std::size_t i = 0; i < g.ops.size(); ++i) {
    const auto& o = g.ops[i];
    s += std::string(i ? "," : "") + "{\"name\":" + quote(o.name) + ",\"kind\":" + quote(kind_name(o.kind)) +
         ",\"inputs\":" + ints(o.inputs) + ",\"outputs\":" + ints(o.outputs) +
         ",\"resource_class\":" + quote(resource_class_name(o.resource_class)) + "}";
  }
  s += "],\"tensors\":[";
  for (std::size_t i = 0; i < g.tensors.size(); ++i) {
    const auto& t = g.tensors[i];
    std::string sh = "[";
    for (std::size_t j = 0; j < t.shape.size(); ++j) sh += (j ? "," : "") + std::to_string(t.shape[j]);
    s += std::string(i ? "," : "") + "{\"name\":" + quote(t.name) + ",\"shape\":" + sh +
         "],\"producer\":" + std::to_string(t.producer) + ",\"consumers\":" + ints(t.consumers) + "}";
  }
  return s + "],\"graph_inputs\":" + ints(g.graph_inputs) + ",\"weights\":" + ints(g.weights) +
         ",\"graph_outputs\":" + ints(g.graph_outputs) + "}";
}

static std::string ref_plan_json(const PartitionPlan& p) {
  std::string s = "{\"subgraphs\":[";
  for (std::size_t i = 0; i < p.subgraphs.size(); ++i) {
    const auto& sg = p.subgraphs[i];
    s += std::string(i ? "," : "") + "{\"id\":" + std::to_string(sg.id) + ",\"ops\":" + ints(sg.ops) +
         ",\"boundary_inputs\":" + ints(sg.boundary_inputs) + ",\"boundary_outputs\":" + ints(sg.boundary_outputs) +
         ",\"label\":" + quote(sg.label) + ",\"dominant_class\":" + quote(resource_class_name(sg.dominant_class)) +
         "}";
  }
  s += "],\"sg_edges\":[";
  for (std::size_t i = 0; i < p.sg_edges.size(); ++i)
    s += std::string(i ? "," : "") + "[" + std::to_string(p.sg_edges[i].first) + "," +
         std::to_string(p.sg_edges[i].second) + "]";
  s += "],\"rule_trace\":[";
  for (std::size_t i = 0; i < p.rule_trace.size(); ++i) s += (i ? "," : "") + quote(p.rule_trace[i]);
  return s + "],\"op_to_subgraph\":" + ints(p.op_to_subgraph) + "}";
}

static builders::KindCosts unit_costs() {  // proj/tests/test_partition.cpp:18-26
  builders::KindCosts c;
  c.attention = {1, 0.1};
  c.matmul = {1, 0.3};
  c.allreduce = {1, 0.1};
  c.alltoall = {1, 0.1};
  c.rowscale = {1, 0.05};
  return c;
}

static void run_case(const std::string& name, const GraphDescription& d, const std::vector<PartitionRule>& rules) {
  // the reference on its own structs
  std::string ref_g, ref_p, ref_err = "null", ours_g, ours_p, ours_err = "null";
  try {
    Graph g = build_graph(d);
    ref_g = ref_graph_json(g);
    ref_p = ref_plan_json(partition(g, rules));
  } catch (const Error& e) {
    ref_err = quote(errc_name(e.code()));
  }
  // the backend through the bridge (exceptions are the reference's opflow::Error)
  try {
    b200::Graph g = b200::build_graph(d);
    ours_g = g.dump();
    b200::Plan p = b200::partition(g, rules);
    b200::validate_plan(p, g);
    ours_p = p.dump();
  } catch (const Error& e) {
    ours_err = quote(errc_name(e.code()));
  }
  std::printf("{\"case\":%s,\"ref_error\":%s,\"ours_error\":%s,\"ref_graph\":%s,\"ours_graph\":%s,"
              "\"ref_plan\":%s,\"ours_plan\":%s}\n",
              quote(name).c_str(), ref_err.c_str(), ours_err.c_str(), ref_g.empty() ? "null" : ref_g.c_str(),
              ours_g.empty() ? "null" : ours_g.c_str(), ref_p.empty() ? "null" : ref_p.c_str(),
              ours_p.empty() ? "null" : ours_p.c_str());
}

int main() {
  const auto c = unit_costs();
  using R = PartitionRule;
  const std::vector<std::pair<std::string, std::vector<R>>> rulesets = {
      {"none", {}},
      {"func_allreduce", {R::by_func("AllReduce")}},
      {"module_layer", {R::by_module("layer*")}},
      {"dbo", {R::by_module("layer*.attn"), R::by_module("layer*.moe.dispatch"), R::by_module("layer*.moe.experts"),
               R::by_module("layer*.moe.combine")}},
      {"fuse", {R::by_func("AllReduce"), R::by_func("RowScale")}},
  };
  for (int layers : {1, 2, 3})
    for (int64_t batch : {4, 1024})
      for (Dtype dt : {Dtype::kI64, Dtype::kF32})
        for (const auto& [rn, rules] : rulesets) {
          const std::string sfx = "_L" + std::to_string(layers) + "_B" + std::to_string(batch) +
                                  (dt == Dtype::kI64 ? "_i64_" : "_f32_") + rn;
          run_case("dense_tp" + sfx, builders::dense_tp_graph(layers, batch, 8, c, dt), rules);
          run_case("moe_ep" + sfx, builders::moe_ep_graph(layers, batch, 8, c, dt), rules);
          run_case("fuse_chain" + sfx, builders::fuse_chain_graph(layers, batch, 8, c, dt), rules);
        }
  // error taxonomy: both sides must raise the same Errc as opflow::Error
  {
    GraphDescription d = builders::dense_tp_graph(1, 4, 8, c);
    d.operators[1].inputs[0] = "nope";
    run_case("err_unknown_tensor", d, {});
  }
  {
    GraphDescription d = builders::dense_tp_graph(1, 4, 8, c);
    d.operators.push_back(d.operators[0]);
    run_case("err_duplicate_op", d, {});
  }
  {
    GraphDescription d = builders::dense_tp_graph(2, 4, 8, c);
    d.operators[0].inputs[0] = d.operators.back().outputs[0];  // close a cycle through the last op
    run_case("err_cycle", d, {});
  }
  {
    GraphDescription d = builders::dense_tp_graph(1, 4, 8, c);
    d.tensors[0].shape = {4, 9};
    run_case("err_shape", d, {});
  }
  {
    GraphDescription d = builders::dense_tp_graph(2, 4, 8, c);
    d.operators[0].region_tags = {"r"};
    d.operators[5].region_tags = {"r"};
    run_case("err_noncontiguous_region", d, {R::by_region("r")});
  }
  run_case("err_empty_pattern", builders::dense_tp_graph(1, 4, 8, c), {R::by_func("")});
  return 0;
}
