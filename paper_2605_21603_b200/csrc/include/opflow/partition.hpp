// Graph-partition annotations (SplitModule / SplitFunc / mark analogues).
//
// Same rule kinds, precedence (ByRegion > ByFunc > ByModule), labels, filler
// naming and boundary/edge ordering as the reference partitioner
// (/root/reference/proj/include/opflow/partition.hpp:15-70,
//  /root/reference/proj/src/partition.cpp:12-230).  One documented
// divergence: two *different* ByFunc rules claiming one op raise
// OverlappingRules, as the reference's own test
// (/root/reference/proj/tests/test_partition.cpp:157-164) and SPEC.md:128
// require; the reference code does not raise there (partition.cpp:163 builds
// the claim key without the rule pattern).
#pragma once

#include <string>
#include <vector>

#include "opflow/graph.hpp"

namespace opflow {

struct PartitionRule {
  enum class Kind { kByModule, kByFunc, kByRegion };
  Kind kind = Kind::kByModule;
  std::string pattern;

  static PartitionRule by_module(std::string p) { return {Kind::kByModule, std::move(p)}; }
  static PartitionRule by_func(std::string p) { return {Kind::kByFunc, std::move(p)}; }
  static PartitionRule by_region(std::string p) { return {Kind::kByRegion, std::move(p)}; }
};

struct Subgraph {
  int32_t id = -1;
  std::vector<int32_t> ops;  // ascending, contiguous in topological order
  std::vector<int32_t> boundary_inputs;
  std::vector<int32_t> boundary_outputs;
  std::string label;
  ResourceClass dominant_class = ResourceClass::kCompute;
};

struct PartitionPlan {
  std::vector<Subgraph> subgraphs;
  std::vector<std::pair<int32_t, int32_t>> sg_edges;  // sorted
  std::vector<std::string> rule_trace;
  std::vector<int32_t> op_to_subgraph;
  std::vector<std::vector<int32_t>> sg_succ;
  std::vector<std::vector<int32_t>> sg_pred;

  std::size_t size() const { return subgraphs.size(); }
  const Subgraph* find_label(const std::string& label) const;
};

bool glob_match(const std::string& pattern, const std::string& text);
PartitionPlan partition(const Graph& g, const std::vector<PartitionRule>& rules);
void validate_plan(const PartitionPlan& plan, const Graph& g);
void finalize_plan(PartitionPlan& plan, const Graph& g);

std::vector<PartitionRule> rules_from_json(const std::string& text);
std::string plan_to_json(const PartitionPlan& plan);
PartitionPlan plan_from_json(const std::string& text);  // hand-assembled plans (tests)

}  // namespace opflow
