// Scheduling contract, Algorithm-1 static analysis
// and the built-in strategies.
#include <algorithm>
#include <numeric>

#include "opflow/engine.hpp"
#include "opflow/json.hpp"

namespace opflow {

// ------------------------------------------------------------------ static analysis
std::vector<MicroBatchContext> static_analysis(const Graph& g, const PartitionPlan& plan,
                                               const SplitSignature& sig) {
  for (int32_t s : sig.merge_set)
    require(s >= 0 && s < static_cast<int32_t>(plan.size()), Errc::UnknownSubgraph,
            "merge set names subgraph " + std::to_string(s));
  // out-degree of each tensor in the partitioned graph: distinct consumer subgraphs
  std::vector<int32_t> outdeg(g.tensors.size(), 0);
  std::vector<bool> pre(g.tensors.size(), false);
  for (const Subgraph& sg : plan.subgraphs)
    for (int32_t t : sg.boundary_inputs) {
      ++outdeg[t];
      if (sig.merge_set.count(sg.id) && g.tensors[t].producer >= 0) pre[t] = true;
    }
  std::vector<MicroBatchContext> ctxs;
  for (std::size_t u = 0; u < sig.sizes.size(); ++u) {
    MicroBatchContext c;
    c.ubatch_idx = static_cast<int32_t>(u);
    c.batch_rows = sig.sizes[u];
    c.states.resize(g.tensors.size());
    for (std::size_t t = 0; t < g.tensors.size(); ++t) {
      c.states[t].ref_count = outdeg[t] + (g.is_output(static_cast<int32_t>(t)) ? 1 : 0);
      c.states[t].prealloc = pre[t];
    }
    ctxs.push_back(std::move(c));
  }
  return ctxs;
}

// ------------------------------------------------------------------ SchedContext
SchedContext::SchedContext(const Graph& g, const PartitionPlan& p, int64_t rows, int num_lanes)
    : g_(g), p_(p), rows_(rows), lanes_(num_lanes) {}

void SchedContext::ensure_split() {
  if (split_done_) return;
  split_done_ = true;
  sizes_ = {rows_};
  done_.assign(p_.size(), std::vector<int32_t>(1, -1));
}

std::vector<int32_t> SchedContext::split(const std::vector<int64_t>& sizes) {
  require(!split_done_, Errc::AlreadySplit, "split() called twice or after execute()");
  require(!sizes.empty(), Errc::SizeMismatch, "split sizes empty");
  int64_t total = 0;
  for (int64_t s : sizes) {
    require(s >= 1, Errc::SizeMismatch, "split sizes must be >= 1");
    total += s;
  }
  require(total == rows_, Errc::SizeMismatch,
          "split sizes sum to " + std::to_string(total) + ", batch has " + std::to_string(rows_));
  split_done_ = true;
  sizes_ = sizes;
  done_.assign(p_.size(), std::vector<int32_t>(sizes.size(), -1));
  std::vector<int32_t> ids(sizes.size());
  std::iota(ids.begin(), ids.end(), 0);
  return ids;
}

int32_t SchedContext::num_ubatches() {
  ensure_split();
  return static_cast<int32_t>(sizes_.size());
}

int32_t SchedContext::find_label(const std::string& label) const {
  for (const Subgraph& sg : p_.subgraphs)
    if (sg.label == label) return sg.id;
  return -1;
}

bool SchedContext::deps_met(int32_t s, int32_t u, const std::set<int32_t>& also) const {
  for (int32_t p : p_.sg_pred[s])
    if (done_[p][u] < 0 && !also.count(p)) return false;
  return true;
}

std::vector<OpHandle> SchedContext::get_ready_ops(int32_t u) {
  ensure_split();
  require(u >= 0 && u < static_cast<int32_t>(sizes_.size()), Errc::InvalidUbatch,
          "ubatch " + std::to_string(u));
  std::vector<OpHandle> out;
  for (int32_t s = 0; s < static_cast<int32_t>(p_.size()); ++s)
    if (done_[s][u] < 0 && deps_met(s, u, {})) out.push_back({s, u, s});
  return out;
}

OpHandle SchedContext::handle(int32_t s, int32_t u) {
  ensure_split();
  require(s >= 0 && s < static_cast<int32_t>(p_.size()), Errc::UnknownSubgraph,
          "subgraph " + std::to_string(s));
  require(u >= 0 && u < static_cast<int32_t>(sizes_.size()), Errc::InvalidUbatch,
          "ubatch " + std::to_string(u));
  return {s, u, s};
}

void SchedContext::check_handle(const OpHandle& h) const {
  require(h.subgraph >= 0 && h.subgraph < static_cast<int32_t>(p_.size()), Errc::UnknownSubgraph,
          "handle names subgraph " + std::to_string(h.subgraph));
  require(h.ubatch >= 0 && h.ubatch < static_cast<int32_t>(sizes_.size()), Errc::InvalidUbatch,
          "handle names ubatch " + std::to_string(h.ubatch));
  require(done_[h.subgraph][h.ubatch] < 0, Errc::NotReady,
          "subgraph '" + p_.subgraphs[h.subgraph].label + "' ubatch " + std::to_string(h.ubatch) +
              " already executed");
}

void SchedContext::record(Dispatch d) {
  d.id = static_cast<int32_t>(dispatches_.size());
  for (int32_t s : d.subgraphs)
    for (int32_t u = d.u0; u < d.u1; ++u) done_[s][u] = d.id;
  dispatches_.push_back(std::move(d));
}

void SchedContext::execute(const std::vector<OpHandle>& ops, int32_t lane,
                           const std::string& replace_fn) {
  ensure_split();
  require(!ops.empty(), Errc::SchedulerError, "execute() with no handles");
  require(lane >= 0 && lane < lanes_, Errc::SchedulerError,
          "lane " + std::to_string(lane) + " out of range");
  std::set<std::pair<int32_t, int32_t>> seen;
  for (const OpHandle& h : ops) {
    check_handle(h);
    require(seen.insert({h.subgraph, h.ubatch}).second, Errc::DuplicateHandle,
            "handle listed twice");
  }
  const bool same_sg = std::all_of(ops.begin(), ops.end(),
                                   [&](const OpHandle& h) { return h.subgraph == ops[0].subgraph; });
  if (ops.size() == 1 || same_sg) {
    // single or merged execution of one subgraph over a contiguous ubatch range
    std::vector<int32_t> us;
    for (const OpHandle& h : ops) us.push_back(h.ubatch);
    std::sort(us.begin(), us.end());
    for (std::size_t i = 1; i < us.size(); ++i)
      require(us[i] == us[i - 1] + 1, Errc::MergeAcrossSplits,
              "merged ubatches must be a contiguous range");
    const int32_t s = ops[0].subgraph;
    for (int32_t u : us)
      require(deps_met(s, u, {}), Errc::NotReady,
              "subgraph '" + p_.subgraphs[s].label + "' ubatch " + std::to_string(u) +
                  " has unexecuted predecessors");
    Dispatch d;
    d.lane = lane;
    d.kind = ops.size() == 1 ? Dispatch::Kind::kSingle : Dispatch::Kind::kMerged;
    d.subgraphs = {s};
    d.u0 = us.front();
    d.u1 = us.back() + 1;
    if (!replace_fn.empty()) {  // replace a single subgraph's body
      d.kind = Dispatch::Kind::kFused;
      d.replace_fn = replace_fn;
      require(ops.size() == 1, Errc::MergeAcrossSplits, "fused+merged execution unsupported");
    }
    record(std::move(d));
    return;
  }
  if (!replace_fn.empty()) {
    // fused execution: one replacement op for several subgraphs of one ubatch
    const int32_t u = ops[0].ubatch;
    std::set<int32_t> members;
    for (const OpHandle& h : ops) {
      require(h.ubatch == u, Errc::MergeAcrossSplits, "fused handles span ubatches");
      members.insert(h.subgraph);
    }
    for (const OpHandle& h : ops)
      require(deps_met(h.subgraph, u, members), Errc::NotReady,
              "fused member '" + p_.subgraphs[h.subgraph].label + "' not ready");
    require(OpRegistry::global().find(replace_fn) != nullptr, Errc::SignatureMismatch,
            "no replacement op '" + replace_fn + "' registered");
    Dispatch d;
    d.lane = lane;
    d.kind = Dispatch::Kind::kFused;
    std::vector<OpHandle> sorted = ops;
    std::sort(sorted.begin(), sorted.end(),
              [](const OpHandle& a, const OpHandle& b) { return a.subgraph < b.subgraph; });
    for (const OpHandle& h : sorted) d.subgraphs.push_back(h.subgraph);
    d.u0 = u;
    d.u1 = u + 1;
    d.replace_fn = replace_fn;
    record(std::move(d));
    return;
  }
  // different subgraphs, no replacement: sequential fallback in handle order.
  // Readiness of the whole list is checked first (earlier handles of the same
  // ubatch count as done), so a NotReady leaves the context untouched.
  for (std::size_t i = 0; i < ops.size(); ++i) {
    std::set<int32_t> earlier;
    for (std::size_t j = 0; j < i; ++j)
      if (ops[j].ubatch == ops[i].ubatch) earlier.insert(ops[j].subgraph);
    require(deps_met(ops[i].subgraph, ops[i].ubatch, earlier), Errc::NotReady,
            "subgraph '" + p_.subgraphs[ops[i].subgraph].label + "' not ready");
  }
  for (const OpHandle& h : ops) {
    Dispatch d;
    d.lane = lane;
    d.subgraphs = {h.subgraph};
    d.u0 = h.ubatch;
    d.u1 = h.ubatch + 1;
    record(std::move(d));
  }
}

int32_t SchedContext::unfinished() const {
  if (!split_done_) return static_cast<int32_t>(p_.size());
  int32_t n = 0;
  for (const auto& row : done_)
    for (int32_t d : row) n += d < 0;
  return n;
}

void SchedContext::finish() {
  ensure_split();
  const int32_t n = unfinished();
  require(n == 0, Errc::IncompleteSchedule,
          std::to_string(n) + " subgraph instances were never executed");
}

// ------------------------------------------------------------------ strategies
namespace {

struct StrategyParams {
  std::string name = "sequential";
  int64_t threshold = 0;          // tokens; below -> sequential
  int32_t n_ub = 2;
  std::vector<int64_t> sizes;     // explicit split sizes (optional)
  int64_t align = 1;              // split sizes rounded to multiples (sequence boundary)
  std::string lane_mode = "class";  // class | ubatch
  int32_t lane_of[kNumResourceClasses] = {0, 1, 2};
  std::string replace_fn;         // fuse_norm_comm replacement name ("" = auto)
  std::vector<std::string> merged_labels = {"*.attn"};  // dbo: executed merged
  std::vector<int> lane_budget;   // per-lane SM budgets
  bool fuse_gemm = false;         // fuse_norm_comm: fold the producing row-parallel MatMul in too
  std::string raw;
};

StrategyParams parse_spec(const std::string& text) {
  StrategyParams p;
  p.raw = text;
  json::Value v;
  try {
    v = json::parse(text.empty() ? "{}" : text);
  } catch (const std::exception& e) {
    fail(Errc::ConfigError, std::string("strategy spec: ") + e.what());
  }
  if (v.t == json::Value::T::String) {
    p.name = v.str();
    return p;
  }
  if (const json::Value* x = v.get("name")) p.name = x->str();
  if (const json::Value* x = v.get("threshold")) p.threshold = x->as_i64();
  if (const json::Value* x = v.get("n_microbatches")) p.n_ub = static_cast<int32_t>(x->as_i64());
  if (const json::Value* x = v.get("sizes"))
    for (const json::Value& e : x->arr()) p.sizes.push_back(e.as_i64());
  if (const json::Value* x = v.get("align")) p.align = std::max<int64_t>(1, x->as_i64());
  if (const json::Value* x = v.get("lane_mode")) p.lane_mode = x->str();
  if (const json::Value* x = v.get("lanes")) {
    if (const json::Value* c = x->get("compute")) p.lane_of[0] = static_cast<int32_t>(c->as_i64());
    if (const json::Value* c = x->get("memory")) p.lane_of[1] = static_cast<int32_t>(c->as_i64());
    if (const json::Value* c = x->get("network")) p.lane_of[2] = static_cast<int32_t>(c->as_i64());
  }
  if (const json::Value* x = v.get("replace_fn")) p.replace_fn = x->str();
  if (const json::Value* x = v.get("fuse_gemm")) p.fuse_gemm = x->t == json::Value::T::Bool ? x->b : x->as_i64() != 0;
  if (const json::Value* x = v.get("lane_sm_budget"))
    for (const json::Value& e : x->arr()) p.lane_budget.push_back(static_cast<int>(e.as_i64()));
  if (const json::Value* x = v.get("merged")) {
    p.merged_labels.clear();
    for (const json::Value& e : x->arr()) p.merged_labels.push_back(e.str());
  }
  if (p.n_ub < 1) fail(Errc::ConfigError, "n_microbatches must be >= 1");
  return p;
}

std::vector<int64_t> split_sizes(const StrategyParams& p, int64_t rows) {
  if (!p.sizes.empty()) return p.sizes;
  // near-equal parts, rounded to the alignment; the last part takes the rest
  std::vector<int64_t> s;
  const int64_t units = rows / p.align;
  int64_t left = rows;
  for (int32_t i = 0; i < p.n_ub; ++i) {
    int64_t part = (i == p.n_ub - 1) ? left : ((units + p.n_ub - 1 - i) / (p.n_ub - i)) * p.align;
    part = std::min(part, left);
    if (part <= 0) break;
    s.push_back(part);
    left -= part;
  }
  if (left > 0) s.back() += left;
  return s;
}

void run_sequential(SchedContext& ctx) {
  // topological order, lane 0, no split ("falls back to a sequential execution")
  const int32_t n = static_cast<int32_t>(ctx.plan().size());
  for (int32_t s = 0; s < n; ++s) ctx.execute({ctx.handle(s, 0)}, 0);
}

int32_t lane_for(const StrategyParams& p, SchedContext& ctx, int32_t s, int32_t u) {
  const int32_t L = ctx.num_lanes();
  if (p.lane_mode == "ubatch") return u % L;
  return std::min(p.lane_of[static_cast<int>(ctx.plan().subgraphs[s].dominant_class)], L - 1);
}

class Sequential final : public Scheduler {
 public:
  explicit Sequential(StrategyParams p) : p_(std::move(p)) {}
  std::vector<int> lane_budgets() const override { return p_.lane_budget; }
  void schedule(SchedContext& ctx) override { run_sequential(ctx); }
  std::string key() const override { return "sequential"; }

 private:
  StrategyParams p_;
};

// NanoFlow-style split + overlap: greedy, ubatch-interleaved, each instance on
// the lane of its resource class (or of its ubatch).
class SplitOverlap final : public Scheduler {
 public:
  explicit SplitOverlap(StrategyParams p) : p_(std::move(p)) {}
  std::vector<int> lane_budgets() const override { return p_.lane_budget; }
  std::string key() const override { return p_.raw; }
  void schedule(SchedContext& ctx) override {
    if (ctx.rows() < p_.threshold || p_.n_ub == 1 || ctx.rows() < 2 * p_.align) {
      run_sequential(ctx);
      return;
    }
    ctx.split(split_sizes(p_, ctx.rows()));
    const int32_t U = ctx.num_ubatches();
    while (ctx.unfinished() > 0) {
      bool progressed = false;
      for (int32_t u = 0; u < U; ++u) {
        auto ready = ctx.get_ready_ops(u);
        if (ready.empty()) continue;
        const OpHandle h = ready.front();
        ctx.execute({h}, lane_for(p_, ctx, h.subgraph, u));
        progressed = true;
      }
      require(progressed, Errc::SchedulerError, "split_overlap made no progress");
    }
  }

 private:
  StrategyParams p_;
};

// Dual-batch overlap (Fig. 7): subgraphs whose label matches `merged` run once
// at full batch (merged ubatches); everything else is per-ubatch, interleaved,
// communication on the network lane and compute on the compute lane.
class Dbo final : public Scheduler {
 public:
  explicit Dbo(StrategyParams p) : p_(std::move(p)) {}
  std::vector<int> lane_budgets() const override { return p_.lane_budget; }
  std::string key() const override { return p_.raw; }
  void schedule(SchedContext& ctx) override {
    const PartitionPlan& plan = ctx.plan();
    std::vector<bool> merged(plan.size(), false);
    bool any = false, comm = false;
    for (const Subgraph& sg : plan.subgraphs) {
      for (const std::string& pat : p_.merged_labels)
        if (glob_match(pat, sg.label)) merged[sg.id] = any = true;
      comm = comm || sg.dominant_class == ResourceClass::kNetwork;
    }
    require(any && comm, Errc::MissingLabels,
            "dbo needs merged (attention) subgraphs and network subgraphs in the plan");
    if (ctx.rows() < p_.threshold || ctx.rows() < 2) {
      run_sequential(ctx);
      return;
    }
    StrategyParams two = p_;
    two.n_ub = 2;
    ctx.split(split_sizes(two, ctx.rows()));
    while (ctx.unfinished() > 0) {
      auto r0 = ctx.get_ready_ops(0), r1 = ctx.get_ready_ops(1);
      bool progressed = false;
      // merged instances first when both halves are ready
      for (const OpHandle& h : r0)
        if (merged[h.subgraph] &&
            std::any_of(r1.begin(), r1.end(), [&](const OpHandle& x) { return x.subgraph == h.subgraph; })) {
          ctx.execute({h, ctx.handle(h.subgraph, 1)}, lane_for(p_, ctx, h.subgraph, 0));
          progressed = true;
        }
      if (progressed) continue;
      // per-ubatch instances, interleaved u0,u1 so one half's comm overlaps the
      // other's compute
      for (int32_t u = 0; u < 2; ++u) {
        for (const OpHandle& h : ctx.get_ready_ops(u)) {
          if (merged[h.subgraph]) continue;
          ctx.execute({h}, lane_for(p_, ctx, h.subgraph, u));
          progressed = true;
          break;
        }
      }
      require(progressed, Errc::SchedulerError, "dbo made no progress");
    }
  }

 private:
  StrategyParams p_;
};

// TokenWeave-style fuse_norm_comm: every AllReduce subgraph followed by a
// norm subgraph is executed as ONE fused replacement op on the network lane,
// overlapped with the other ubatch's compute.
class FuseNormComm final : public Scheduler {
 public:
  explicit FuseNormComm(StrategyParams p) : p_(std::move(p)) {}
  std::vector<int> lane_budgets() const override { return p_.lane_budget; }
  std::string key() const override { return p_.raw; }
  void schedule(SchedContext& ctx) override {
    const Graph& g = ctx.graph();
    const PartitionPlan& plan = ctx.plan();
    // pair[s] = successor norm subgraph of AllReduce-only subgraph s
    std::vector<int32_t> pair(plan.size(), -1);
    std::vector<std::string> fn(plan.size());
    bool found = false;
    for (const Subgraph& sg : plan.subgraphs) {
      if (sg.ops.size() != 1 || g.ops[sg.ops[0]].kind != OperatorKind::kAllReduce) continue;
      if (plan.sg_succ[sg.id].size() != 1) continue;
      const Subgraph& nx = plan.subgraphs[plan.sg_succ[sg.id][0]];
      if (nx.ops.size() != 1) continue;
      const OperatorNode& nop = g.ops[nx.ops[0]];
      std::string f;
      if (nop.kind == OperatorKind::kRowScale) f = "allreduce_rowscale";
      if (nop.kind == OperatorKind::kCustom && nop.attrs.custom_name == "add_rmsnorm")
        f = "allreduce_add_rmsnorm";
      if (f.empty()) continue;
      pair[sg.id] = nx.id;
      fn[sg.id] = p_.replace_fn.empty() ? f : p_.replace_fn;
      found = true;
    }
    require(found, Errc::MissingPattern, "no AllReduce -> norm subgraph pairs in the plan");
    std::vector<bool> is_second(plan.size(), false);
    for (int32_t s = 0; s < static_cast<int32_t>(plan.size()); ++s)
      if (pair[s] >= 0) is_second[pair[s]] = true;
    // fuse_gemm: a single-MatMul subgraph whose only successor is the AllReduce
    // of an (AllReduce, add_rmsnorm) pair joins it — the row-parallel GEMM's
    // epilogue then pushes its partial to the owner ranks while later tiles
    // compute (matmul_allreduce_add_rmsnorm).  Isolate those MatMuls with
    // rules, e.g. by_module("layer*.attn.o"), by_module("layer*.mlp.down").
    std::vector<int32_t> gemm_of(plan.size(), -1);  // AR subgraph -> its MatMul subgraph
    std::vector<int32_t> ar_of(plan.size(), -1);    // MatMul subgraph -> its AR subgraph
    if (p_.fuse_gemm)
      for (int32_t s = 0; s < static_cast<int32_t>(plan.size()); ++s) {
        if (pair[s] < 0 || fn[s] != "allreduce_add_rmsnorm" || plan.sg_pred[s].size() != 1) continue;
        const int32_t m = plan.sg_pred[s][0];
        const Subgraph& ms = plan.subgraphs[m];
        if (ms.ops.size() != 1 || plan.sg_succ[m].size() != 1) continue;
        const OperatorNode& mop = g.ops[ms.ops[0]];
        if (mop.kind != OperatorKind::kMatMul || g.ops[plan.subgraphs[s].ops[0]].inputs[0] != mop.outputs[0]) continue;
        gemm_of[s] = m;
        ar_of[m] = s;
        fn[s] = p_.replace_fn.empty() ? "matmul_allreduce_add_rmsnorm" : p_.replace_fn;
      }
    const bool split = !(ctx.rows() < p_.threshold || ctx.rows() < 2 * p_.align);
    if (split) {
      StrategyParams two = p_;
      ctx.split(split_sizes(two, ctx.rows()));
    }
    const int32_t U = ctx.num_ubatches();
    const int32_t net = std::min(p_.lane_of[2], ctx.num_lanes() - 1);
    while (ctx.unfinished() > 0) {
      bool progressed = false;
      for (int32_t u = 0; u < U; ++u) {
        for (const OpHandle& h : ctx.get_ready_ops(u)) {
          if (is_second[h.subgraph]) continue;  // dispatched with its AllReduce
          if (ar_of[h.subgraph] >= 0) {         // MatMul -> AllReduce -> add_rmsnorm as one op
            const int32_t a = ar_of[h.subgraph];
            ctx.execute({h, ctx.handle(a, u), ctx.handle(pair[a], u)}, net, fn[a]);
          } else if (gemm_of[h.subgraph] >= 0) {
            continue;  // dispatched with its MatMul
          } else if (pair[h.subgraph] >= 0) {
            ctx.execute({h, ctx.handle(pair[h.subgraph], u)}, net, fn[h.subgraph]);
          } else {
            ctx.execute({h}, lane_for(p_, ctx, h.subgraph, u));
          }
          progressed = true;
          break;
        }
      }
      require(progressed, Errc::SchedulerError, "fuse_norm_comm made no progress");
    }
  }

 private:
  StrategyParams p_;
};

}  // namespace

std::unique_ptr<Scheduler> make_strategy(const std::string& spec) {
  StrategyParams p = parse_spec(spec);
  if (p.name == "sequential") return std::make_unique<Sequential>(p);
  if (p.name == "split_overlap" || p.name == "nanoflow") return std::make_unique<SplitOverlap>(p);
  if (p.name == "dbo") return std::make_unique<Dbo>(p);
  if (p.name == "fuse_norm_comm" || p.name == "tokenweave") return std::make_unique<FuseNormComm>(p);
  fail(Errc::ConfigError, "unknown strategy '" + p.name + "'");
}

}  // namespace opflow
