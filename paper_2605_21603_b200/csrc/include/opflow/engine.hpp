// The B200 execution backend: scheduling contract (split / get_ready_ops /
// execute), Algorithm-1 data-flow + memory management over one HBM arena, and
// a multi-stream executor whose resolved schedule is captured into one CUDA
// Graph and replayed from a plan cache.
//
// SPEC sources (the reference has no code for these layers):
//   dataflow_mem  SPEC.md:162-240, PAPER.md:377-420 (Algorithm 1)
//   sched_api     SPEC.md:242-320, PAPER.md:298-350 (Fig. 6)
//   engine
//   strategies
//
// Execution model.  A strategy runs against a SchedContext that *records*
// dispatches; "dispatched" satisfies a dependency for readiness because the
// device enforces ordering (same-lane FIFO on a CUDA stream, cross-lane via
// events) — the asynchronous-engine reading of SPEC.md:308.  The recorded
// dispatch list is then compiled once per key (strategy, split signature,
// rows): Algorithm 1 binds every boundary tensor instance to an arena block or a
// merge-buffer slice (zero copy), a lane-aware allocator reuses blocks only
// across happens-before edges, and the launch list is stream-captured into a
// CUDA Graph.  Steady state = one cudaGraphLaunch per forward.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "opflow/device.hpp"
#include "opflow/graph.hpp"
#include "opflow/partition.hpp"

struct opf_comm;

namespace opflow {

// ------------------------------------------------------------ dataflow (Algorithm 1)
struct SplitSignature {
  std::vector<int64_t> sizes;
  std::set<int32_t> merge_set;  // subgraphs executed merged (merge points)
};

enum class BindingKind { kUnmaterialized, kOwned, kSlice };

struct TensorState {
  int32_t ref_count = 0;
  bool prealloc = false;
  BindingKind binding = BindingKind::kUnmaterialized;
  int32_t buffer = -1;      // arena block id
  int64_t row_offset = 0;   // rows into the block
  int64_t row_extent = 0;
};

struct MicroBatchContext {
  int32_t ubatch_idx = 0;
  int64_t batch_rows = 0;
  std::vector<TensorState> states;  // indexed by tensor id
};

// ref_count = number of distinct subgraphs consuming t across a boundary
// (+1 sentinel for GraphOutputs); prealloc = boundary input of a merge point
// produced inside the graph.
std::vector<MicroBatchContext> static_analysis(const Graph& g, const PartitionPlan& plan,
                                               const SplitSignature& sig);

// ------------------------------------------------------------ schedule recording
struct OpHandle {
  int32_t subgraph = -1;
  int32_t ubatch = -1;
  int32_t topo_index = -1;
};

struct Dispatch {
  enum class Kind { kSingle, kMerged, kFused };
  int32_t id = -1;
  int32_t lane = 0;
  Kind kind = Kind::kSingle;
  std::vector<int32_t> subgraphs;  // >1 only for fused
  int32_t u0 = 0, u1 = 1;          // covered ubatches [u0, u1)
  std::string replace_fn;
};

class SchedContext {
 public:
  SchedContext(const Graph& g, const PartitionPlan& p, int64_t rows, int num_lanes);

  std::vector<int32_t> split(const std::vector<int64_t>& sizes);
  std::vector<OpHandle> get_ready_ops(int32_t ubatch);
  OpHandle handle(int32_t subgraph, int32_t ubatch);
  void execute(const std::vector<OpHandle>& ops, int32_t lane = 0,
               const std::string& replace_fn = "");

  int64_t rows() const { return rows_; }
  int32_t num_ubatches();
  int32_t num_lanes() const { return lanes_; }
  int32_t unfinished() const;
  const Graph& graph() const { return g_; }
  const PartitionPlan& plan() const { return p_; }
  bool is_split() const { return split_done_; }
  const std::vector<int64_t>& sizes() { ensure_split(); return sizes_; }
  int32_t find_label(const std::string& label) const;

  // recorded result
  const std::vector<Dispatch>& dispatches() const { return dispatches_; }
  void finish();  // IncompleteSchedule check

 private:
  void ensure_split();
  bool deps_met(int32_t s, int32_t u, const std::set<int32_t>& also) const;
  void check_handle(const OpHandle& h) const;
  void record(Dispatch d);

  const Graph& g_;
  const PartitionPlan& p_;
  int64_t rows_;
  int lanes_;
  bool split_done_ = false;
  std::vector<int64_t> sizes_;
  std::vector<std::vector<int32_t>> done_;  // [subgraph][ubatch] -> dispatch id or -1
  std::vector<Dispatch> dispatches_;
};

// Strategy (the paper's OpSchedulerBase.schedule).
class Scheduler {
 public:
  virtual ~Scheduler() = default;
  virtual void schedule(SchedContext& ctx) = 0;
  virtual std::string key() const = 0;  // plan-cache key component
  // Per-lane SM budgets (max SMs a lane's GEMM / attention launches occupy;
  // 0 = all).  NanoFlow-style SM partitioning between concurrent streams.
  virtual std::vector<int> lane_budgets() const { return {}; }
};

std::unique_ptr<Scheduler> make_strategy(const std::string& spec_json);

// ------------------------------------------------------------ session / engine
struct SessionConfig {
  int lanes = 3;
  bool prealloc = true;       // Algorithm-1 zero-copy merge buffers; false = copying fallback
  bool cuda_graph = true;     // capture + replay; false = eager launches every run
  bool fuse = true;           // GEMM epilogue fusion (MatMul -> silu_mul) inside a dispatch
  bool fuse_addnorm = true;   // ... and MatMul -> add_rmsnorm (residual add in the epilogue)
  int device = 0;
  int gemm_sm_budget = 0;     // max CTAs for tensor-core GEMMs on lane 0 when overlapping
  std::vector<int> lane_sm_budget;  // per-lane SM budget defaults (strategy may override)
  int world = 0;                    // dry sessions: communicator size to plan for (0 = the comm's)
};

struct PlannedView {
  enum class Src { kArena, kExternal, kPrepacked, kNone } src = Src::kNone;
  int64_t block_off = 0;   // arena byte offset of the block (kArena)
  int32_t tensor = -1;     // external / prepacked tensor id
  int64_t elem_offset = 0; // within the block / external view
  Dtype dtype = Dtype::kF32;
  std::vector<int64_t> shape;
  bool batched = true;
};

struct PlannedLaunch {
  int32_t op = -1;               // graph op index, -1 for fused replacement / copies
  std::string fn;                // registry name (Custom / fused), "" = built-in kind
  OperatorKind kind = OperatorKind::kCustom;
  OpAttrs attrs;
  std::string name;
  std::vector<PlannedView> in, out;
  int64_t rows = 0;
  int64_t ws_off = -1, ws_bytes = 0;  // arena workspace
  const void* aux = nullptr;
  int32_t prepacked = -1;        // MatMul bf16: weight tensor whose [N,K] copy is aux
  int prepack_mode = 0;          // 0 transposed, 1 gate/up interleaved (SiLU-mul epilogue)
  bool is_copy = false;          // concat fallback copy
  int max_ctas = 0;
};

struct PlannedDispatch {
  Dispatch d;
  std::vector<int32_t> wait_on;  // dispatch ids (other lanes) to wait for
  bool record_event = false;
  std::vector<PlannedLaunch> launches;
  int64_t rows = 0;
};

struct CompiledPlan {
  std::string key;
  std::vector<PlannedDispatch> dispatches;
  int64_t arena_bytes = 0;
  int64_t copied_elements = 0;
  int64_t analysis_ops = 0;    // graph-analysis work done at build (0 on replay)
  int64_t peak_live_bytes = 0;
  int64_t n_launches = 0;
  int lanes_used = 0;
  int64_t end_live_tensors = 0;  // non-output tensors still referenced after the run
  std::vector<std::pair<int32_t, int64_t>> outputs;  // graph output -> arena offset
  cudaGraphExec_t exec = nullptr;
  void* arena_base_at_capture = nullptr;
  std::vector<std::string> trace_names;
};

class Session {
 public:
  Session(const Graph& g, const PartitionPlan& p, SessionConfig cfg, opf_comm* comm);
  // Device-free session: records and compiles schedules (Algorithm 1, lanes,
  // events, arena plan) without touching a GPU — used by CPU tests and tools.
  static std::unique_ptr<Session> dry(const Graph& g, const PartitionPlan& p, SessionConfig cfg,
                                      int64_t rows);
  void plan_only(Scheduler& strat, const std::string& key);
  ~Session();

  void bind(const std::string& tensor, const opf_view& v);
  // Context-aware strategy selection: for
  // {"name":"auto","candidates":[spec, ...]} time every candidate's captured
  // schedule on the device for the current row count, cache the winner per
  // rows, and return its spec; any other spec is returned unchanged.
  std::string choose(const std::string& spec, cudaStream_t stream);
  void run(Scheduler& strat, const std::string& key, cudaStream_t stream);
  // Everything run() does except the launch: plan (cached), prepack weights,
  // size the arena, capture the CUDA graph.  Peer-memory ranks sharing one
  // device prepare all ranks before launching any (no allocation may then
  // synchronise the device while a peer's barrier kernel spins).
  CompiledPlan* prepare(Scheduler& strat, const std::string& key, cudaStream_t stream);
  opf_view output(const std::string& tensor);
  std::string stats_json() const;
  std::string schedule_json() const;
  std::string trace_json();

  const Graph& graph() const { return g_; }
  const PartitionPlan& plan() const { return p_; }
  int64_t rows() const;

  // Symmetric arena for peer-memory ops (expert-parallel dispatch / combine):
  // every rank compiles the same plans, so a tensor lives at the same arena
  // offset on every rank.  export_arena() allocates at least `bytes` and pins
  // the arena (later plans must fit); set_peer_arenas() hands all ranks' bases
  // (mine included) to the communicator.
  void* export_arena(int64_t bytes);
  void set_peer_arenas(const std::vector<void*>& bases);
  opf_comm* comm() const { return comm_; }
  // Peer-window health: every replay that may touch the communicator's window
  // copies its sticky barrier-timeout word to pinned host memory behind the
  // replay.  run() raises SchedulerError for an earlier replay whose copy has
  // landed; check_window() waits for the last one.  A timed-out barrier means
  // a peer never arrived, so that replay's activations are invalid.
  void check_window(bool wait);

 private:
  std::unique_ptr<CompiledPlan> compile(const SchedContext& ctx, const std::string& key,
                                        const std::vector<int>& budgets);
  void ensure_arena(int64_t bytes);
  void ensure_prepacked(cudaStream_t s);
  opf_view resolve(const PlannedView& v) const;
  void launch_plan(CompiledPlan& cp, cudaStream_t origin, bool capturing);
  void launch_one(const PlannedLaunch& l, cudaStream_t s);
  void warm_aux(const CompiledPlan& cp);

  const Graph& g_;
  const PartitionPlan& p_;
  SessionConfig cfg_;
  opf_comm* comm_;
  std::vector<cudaStream_t> lanes_;
  std::vector<opf_view> ext_;        // per tensor: bound external view (base == nullptr if unbound)
  std::vector<void*> prepacked_;     // per weight tensor: transposed bf16 copy for MatMul
  std::vector<void*> prepacked_act_; // per weight tensor: gate/up interleaved copy (SiLU epilogue)
  void ensure_packed_for(const CompiledPlan& cp, cudaStream_t s);
  bool prepack_dirty_ = true;
  void* arena_ = nullptr;
  int64_t arena_bytes_ = 0;
  bool arena_pinned_ = false;  // peer-mapped: never reallocated
  std::map<std::string, std::unique_ptr<CompiledPlan>> cache_;
  std::map<std::pair<uint64_t, int64_t>, void*> perms_;
  CompiledPlan* last_ = nullptr;
  std::vector<cudaEvent_t> events_;
  int64_t hits_ = 0, misses_ = 0, runs_ = 0;
  std::map<std::string, std::string> auto_choice_;        // (auto spec | rows) -> winner spec
  std::map<std::string, std::vector<double>> auto_times_;  // (auto spec | rows) -> ms per candidate
  bool dry_ = false;
  int64_t dry_rows_ = 0;
  uint32_t* win_err_host_ = nullptr;   // pinned copy of the window's error word
  cudaEvent_t win_err_ev_ = nullptr;   // recorded behind that copy
  bool win_err_pending_ = false;
  void note_window(cudaStream_t stream);
  CompiledPlan* lookup_or_build(Scheduler& strat, const std::string& key);
  std::vector<std::string> names_;  // storage for opf_op_ctx param names
};

}  // namespace opflow
