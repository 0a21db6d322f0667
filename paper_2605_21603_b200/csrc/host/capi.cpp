// extern "C" boundary of libopflow_b200.so (declared in include/opflow_b200.h).
// Every entry point converts opflow::Error into (Errc ordinal + 1) and keeps the
// message for opf_last_error(), mirroring the reference's exception contract.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <random>

#include "opflow/builders.hpp"
#include "opflow/comm.hpp"
#include "opflow/nccl_api.hpp"
#include "opflow/engine.hpp"
#include "opflow/graph.hpp"
#include "opflow/json.hpp"
#include "opflow/partition.hpp"
#include "opflow_b200.h"

using namespace opflow;

namespace opflow {
const std::string& last_error_ref();
}

struct opf_graph {
  Graph g;
};
struct opf_plan {
  PartitionPlan p;
};
struct opf_session {
  Graph g;
  PartitionPlan p;
  std::unique_ptr<Session> s;
};
struct opf_sched_ctx {
  SchedContext* ctx;
};

namespace {

template <class F>
opf_status guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    set_last_error(e.what());
    return static_cast<opf_status>(e.code()) + 1;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return static_cast<opf_status>(Errc::SchedulerError) + 1;
  }
}

char* dup_string(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

void need(const void* p, const char* what) {
  if (!p) fail(Errc::ConfigError, std::string("null ") + what);
}

// Direct (session-less) launch of a registered op: allocate its workspace
// stream-ordered for this one call (a Session plans it inside the arena instead).
opf_status call_with_workspace(const OpEntry& e, opf_op_ctx& c, const opf_view* in, int32_t n_in,
                               opf_view* out, int32_t n_out, int64_t rows, cudaStream_t s) {
  const size_t bytes = e.workspace ? e.workspace(c, in, n_in, out, n_out, rows) : 0;
  if (bytes == 0) return e.fn(&c, in, n_in, out, n_out, rows, s);
  void* ws = nullptr;
  OPF_CUDA(cudaMallocAsync(&ws, bytes, s));
  c.workspace = ws;
  c.workspace_bytes = bytes;
  const opf_status st = e.fn(&c, in, n_in, out, n_out, rows, s);
  OPF_CUDA(cudaFreeAsync(ws, s));
  return st;
}

SessionConfig parse_config(const char* text) {
  SessionConfig c;
  if (!text || !*text) return c;
  json::Value v;
  try {
    v = json::parse(text);
  } catch (const std::exception& e) {
    fail(Errc::ConfigError, std::string("session config: ") + e.what());
  }
  if (const json::Value* x = v.get("lanes")) c.lanes = static_cast<int>(x->as_i64());
  if (const json::Value* x = v.get("prealloc")) c.prealloc = x->b;
  if (const json::Value* x = v.get("cuda_graph")) c.cuda_graph = x->b;
  if (const json::Value* x = v.get("device")) c.device = static_cast<int>(x->as_i64());
  if (const json::Value* x = v.get("gemm_sm_budget")) c.gemm_sm_budget = static_cast<int>(x->as_i64());
  if (const json::Value* x = v.get("fuse")) c.fuse = x->b;
  if (const json::Value* x = v.get("fuse_addnorm")) c.fuse_addnorm = x->b;
  if (const json::Value* x = v.get("world")) c.world = static_cast<int>(x->as_i64());
  if (const json::Value* x = v.get("lane_sm_budget"))
    for (const json::Value& e : x->arr()) c.lane_sm_budget.push_back(static_cast<int>(e.as_i64()));
  require(c.lanes >= 1 && c.lanes <= 16, Errc::ConfigError, "lanes must be in [1,16]");
  return c;
}

class CallbackStrategy final : public Scheduler {
 public:
  CallbackStrategy(opf_schedule_fn fn, void* user, std::string key)
      : fn_(fn), user_(user), key_(std::move(key)) {}
  void schedule(SchedContext& ctx) override {
    opf_sched_ctx c{&ctx};
    const opf_status st = fn_(&c, user_);
    if (st != 0) {
      const int code = st - 1;
      fail(code >= 0 && code < static_cast<int>(Errc::kCount) ? static_cast<Errc>(code)
                                                              : Errc::SchedulerError,
           "user strategy: " + last_error_ref());
    }
  }
  std::string key() const override { return key_; }

 private:
  opf_schedule_fn fn_;
  void* user_;
  std::string key_;
};

}  // namespace

extern "C" {

const char* opf_last_error(void) { return last_error_ref().c_str(); }
const char* opf_errc_name(opf_status s) {
  if (s == 0) return "OK";
  return errc_name(static_cast<Errc>(s - 1));
}
const char* opf_version(void) { return "opflow-b200 0.1 (sm_100a)"; }
void opf_free_string(char* s) { std::free(s); }

// ------------------------------------------------------------------ frontend
opf_status opf_graph_build(const char* desc, opf_graph** out) {
  return guard([&] {
    need(desc, "description");
    need(out, "out");
    auto g = std::make_unique<opf_graph>();
    g->g = build_graph(description_from_json(desc));
    *out = g.release();
  });
}
void opf_graph_free(opf_graph* g) { delete g; }

opf_status opf_graph_dump(const opf_graph* g, char** json_out) {
  return guard([&] {
    need(g, "graph");
    *json_out = dup_string(graph_to_json(g->g));
  });
}

opf_status opf_graph_tensor_id(const opf_graph* g, const char* name, int32_t* id) {
  return guard([&] {
    need(g, "graph");
    *id = g->g.tensor_id(name);
  });
}

opf_status opf_partition(const opf_graph* g, const char* rules, opf_plan** out) {
  return guard([&] {
    need(g, "graph");
    auto p = std::make_unique<opf_plan>();
    p->p = partition(g->g, rules_from_json(rules ? rules : "[]"));
    *out = p.release();
  });
}

opf_status opf_plan_from_json(const opf_graph* g, const char* plan_json, opf_plan** out) {
  return guard([&] {
    need(g, "graph");
    auto p = std::make_unique<opf_plan>();
    p->p = plan_from_json(plan_json);
    finalize_plan(p->p, g->g);
    *out = p.release();
  });
}

opf_status opf_validate_plan(const opf_plan* p, const opf_graph* g) {
  return guard([&] {
    need(p, "plan");
    need(g, "graph");
    validate_plan(p->p, g->g);
  });
}

opf_status opf_plan_dump(const opf_plan* p, char** json_out) {
  return guard([&] {
    need(p, "plan");
    *json_out = dup_string(plan_to_json(p->p));
  });
}
void opf_plan_free(opf_plan* p) { delete p; }

opf_status opf_builder_json(const char* name, const char* params, char** json_out) {
  return guard([&] { *json_out = dup_string(builders::build_json(name, params ? params : "{}")); });
}

// Same algorithm as /root/reference/proj/src/eval.cpp:14-20 (libstdc++
// std::shuffle driven by mt19937_64 seeded with seed*golden+cols).
opf_status opf_alltoall_permutation(uint64_t seed, uint32_t cols, uint32_t* perm_out) {
  return guard([&] {
    std::vector<uint32_t> p(cols);
    std::iota(p.begin(), p.end(), 0u);
    std::mt19937_64 rng(seed * 0x9E3779B97F4A7C15ull + cols);
    std::shuffle(p.begin(), p.end(), rng);
    std::copy(p.begin(), p.end(), perm_out);
  });
}

// ------------------------------------------------------------------ device ops
opf_status opf_register_op(const char* name, opf_kernel_fn fn, int32_t rc, int32_t n_in,
                           int32_t n_out) {
  return guard([&] {
    need(name, "name");
    need(reinterpret_cast<const void*>(fn), "kernel fn");
    require(rc >= 0 && rc < kNumResourceClasses, Errc::ConfigError, "bad resource class");
    OpRegistry::global().add({name, fn, static_cast<ResourceClass>(rc), n_in, n_out, {}});
  });
}

opf_status opf_has_op(const char* name, int32_t* present) {
  return guard([&] { *present = OpRegistry::global().find(name) != nullptr; });
}

int32_t opf_gemm_splits(int64_t m, int64_t n, int64_t k, int32_t max_ctas) {
  try {
    return opflow::gemm_splitk_splits(m, n, k, max_ctas);
  } catch (...) {
    return 1;
  }
}

opf_status opf_launch(const char* op_json, const opf_view* in, int32_t n_in, opf_view* out,
                      int32_t n_out, int64_t rows, void* stream) {
  opf_status st = 0;
  const opf_status g = guard([&] {
    need(op_json, "op");
    GraphDescription d = description_from_json(std::string("{\"operators\":[") + op_json + "]}");
    const OpDecl& od = d.operators.at(0);
    std::vector<const char*> pn;
    std::vector<double> pv;
    for (const auto& kv : od.attrs.params) {
      pn.push_back(kv.first.c_str());
      pv.push_back(kv.second);
    }
    opf_op_ctx c{};
    c.op_name = od.name.c_str();
    c.kind = static_cast<int32_t>(od.kind);
    c.custom_name = od.attrs.custom_name.c_str();
    c.world_size = od.attrs.world_size;
    c.seed = od.attrs.seed;
    c.n_params = static_cast<int32_t>(pn.size());
    c.param_names = pn.data();
    c.param_values = pv.data();
    auto s = static_cast<cudaStream_t>(stream);
    if (od.kind == OperatorKind::kCustom) {
      const OpEntry* e = OpRegistry::global().find(od.attrs.custom_name);
      require(e != nullptr, Errc::ConfigError,
              "no custom function registered for '" + od.attrs.custom_name + "'");
      st = call_with_workspace(*e, c, in, n_in, out, n_out, rows, s);
    } else {
      st = launch_kind(c, in, n_in, out, n_out, rows, s);
    }
  });
  return g ? g : st;
}

opf_status opf_launch_comm(const char* op_json, const opf_view* in, int32_t n_in, opf_view* out,
                           int32_t n_out, int64_t rows, opf_comm* comm, int32_t max_ctas,
                           void* stream) {
  opf_status st = 0;
  const opf_status g = guard([&] {
    need(op_json, "op");
    GraphDescription d = description_from_json(std::string("{\"operators\":[") + op_json + "]}");
    const OpDecl& od = d.operators.at(0);
    std::vector<const char*> pn;
    std::vector<double> pv;
    for (const auto& kv : od.attrs.params) {
      pn.push_back(kv.first.c_str());
      pv.push_back(kv.second);
    }
    opf_op_ctx c{};
    c.op_name = od.name.c_str();
    c.kind = static_cast<int32_t>(od.kind);
    c.custom_name = od.attrs.custom_name.c_str();
    c.world_size = od.attrs.world_size;
    c.seed = od.attrs.seed;
    c.n_params = static_cast<int32_t>(pn.size());
    c.param_names = pn.data();
    c.param_values = pv.data();
    c.comm = comm;
    c.max_ctas = max_ctas;
    auto s = static_cast<cudaStream_t>(stream);
    if (od.kind == OperatorKind::kCustom) {
      const OpEntry* e = OpRegistry::global().find(od.attrs.custom_name);
      require(e != nullptr, Errc::ConfigError,
              "no custom function registered for '" + od.attrs.custom_name + "'");
      st = call_with_workspace(*e, c, in, n_in, out, n_out, rows, s);
    } else {
      st = launch_kind(c, in, n_in, out, n_out, rows, s);
    }
  });
  return g ? g : st;
}

opf_status opf_view_rows(const opf_view* v, int64_t row_off, int64_t nrows, opf_view* out) {
  return guard([&] {
    need(v, "view");
    require(v->rank >= 1 && row_off >= 0 && nrows >= 0 && row_off + nrows <= v->shape[0],
            Errc::SizeMismatch, "row view out of range");
    *out = *v;
    out->shape[0] = nrows;
    out->elem_offset = v->elem_offset + row_off * view_row_elems(*v);
  });
}

// ------------------------------------------------------------------ comm
opf_status opf_comm_unique_id(uint8_t id_out[128]) {
  return guard([&] {
    ncclUniqueId id;
    const ncclResult_t r = nccl().GetUniqueId(&id);
    require(r == ncclSuccess, Errc::SchedulerError, std::string("ncclGetUniqueId: ") + nccl().GetErrorString(r));
    static_assert(sizeof(id) == 128);
    std::memcpy(id_out, &id, 128);
  });
}

opf_status opf_comm_init(const uint8_t id[128], int32_t world, int32_t rank, int32_t device,
                         opf_comm** out) {
  return guard([&] {
    auto c = std::make_unique<opf_comm>();
    c->world = world;
    c->rank = rank;
    c->device = device;
    OPF_CUDA(cudaSetDevice(device));
    if (world > 1) {
      ncclUniqueId uid;
      std::memcpy(&uid, id, 128);
      const ncclResult_t r = nccl().CommInitRank(&c->nccl, world, uid, rank);
      require(r == ncclSuccess, Errc::SchedulerError,
              std::string("ncclCommInitRank: ") + nccl().GetErrorString(r));
    }
    *out = c.release();
  });
}

opf_status opf_comm_init_peer(int32_t world, int32_t rank, int32_t device, opf_comm** out) {
  return guard([&] {
    require(world >= 1 && world <= 8 && rank >= 0 && rank < world, Errc::ConfigError,
            "peer communicator: need 1 <= world <= 8 and 0 <= rank < world");
    auto c = std::make_unique<opf_comm>();
    c->world = world;
    c->rank = rank;
    c->device = device;
    OPF_CUDA(cudaSetDevice(device));
    *out = c.release();
  });
}

void opf_comm_free(opf_comm* c) {
  if (!c) return;
  if (c->nccl) nccl().CommDestroy(c->nccl);
  for (void* p : c->opened) cudaIpcCloseMemHandle(p);
  for (void* p : c->opened_arenas) cudaIpcCloseMemHandle(p);
  if (c->window_base) cudaFree(c->window_base);
  delete c;
}

opf_status opf_comm_window_alloc(opf_comm* c, size_t stage_bytes, uint8_t ipc_handle_out[64]) {
  return guard([&] {
    need(c, "comm");
    comm_window_alloc(c, stage_bytes, ipc_handle_out);
  });
}

opf_status opf_comm_window_open(opf_comm* c, const uint8_t* handles) {
  return guard([&] {
    need(c, "comm");
    need(handles, "handles");
    comm_window_open(c, handles);
  });
}

opf_status opf_comm_create_virtual(int32_t world, int32_t device, size_t stage_bytes, opf_comm** outs) {
  return guard([&] {
    require(world >= 1 && world <= 8, Errc::ConfigError, "virtual world must be 1..8");
    OPF_CUDA(cudaSetDevice(device));
    std::vector<opf_comm*> cs;
    for (int r = 0; r < world; ++r) {
      auto c = std::make_unique<opf_comm>();
      c->world = world;
      c->rank = r;
      c->device = device;
      c->virtual_rank = true;
      comm_window_alloc(c.get(), stage_bytes, nullptr);
      cs.push_back(c.release());
    }
    comm_window_link_local(cs.data(), world);
    for (int r = 0; r < world; ++r) outs[r] = cs[r];
  });
}

opf_status opf_comm_window_error(opf_comm* c, uint32_t* err) {
  return guard([&] {
    need(c, "comm");
    *err = comm_window_error(c);
  });
}

opf_status opf_comm_window_set_epochs(opf_comm* c, uint32_t value) {
  return guard([&] {
    need(c, "comm");
    require(c->window_base != nullptr, Errc::ConfigError, "communicator has no window");
    comm_window_set_epochs(c, value);
  });
}

opf_status opf_comm_push_calls(opf_comm* c, uint32_t* calls) {
  return guard([&] {
    need(c, "comm");
    *calls = comm_push_calls(c);
  });
}

// ------------------------------------------------------------------ sessions
opf_status opf_session_create(const opf_graph* g, const opf_plan* p, const char* config,
                              opf_comm* comm, opf_session** out) {
  return guard([&] {
    need(g, "graph");
    need(p, "plan");
    auto s = std::make_unique<opf_session>();
    s->g = g->g;
    s->p = p->p;
    validate_plan(s->p, s->g);
    s->s = std::make_unique<Session>(s->g, s->p, parse_config(config), comm);
    *out = s.release();
  });
}

void opf_session_free(opf_session* s) { delete s; }

opf_status opf_session_arena_export(opf_session* s, int64_t min_bytes, uint8_t ipc_handle_out[64]) {
  return guard([&] {
    need(s, "session");
    void* base = s->s->export_arena(min_bytes);
    if (ipc_handle_out) {
      cudaIpcMemHandle_t h;
      OPF_CUDA(cudaIpcGetMemHandle(&h, base));
      std::memcpy(ipc_handle_out, &h, sizeof(h));
    }
  });
}

opf_status opf_session_arena_open(opf_session* s, const uint8_t* handles) {
  return guard([&] {
    need(s, "session");
    need(handles, "handles");
    opf_comm* c = s->s->comm();
    require(c != nullptr, Errc::ConfigError, "session has no communicator");
    std::vector<void*> bases(c->world, nullptr);
    for (int p = 0; p < c->world; ++p) {
      if (p == c->rank) {
        bases[p] = s->s->export_arena(0);
        continue;
      }
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handles + p * sizeof(cudaIpcMemHandle_t), sizeof(h));
      OPF_CUDA(cudaIpcOpenMemHandle(&bases[p], h, cudaIpcMemLazyEnablePeerAccess));
      c->opened_arenas.push_back(bases[p]);
    }
    s->s->set_peer_arenas(bases);
  });
}

opf_status opf_session_arena_link_local(opf_session* const* sessions, int32_t world, int64_t min_bytes) {
  return guard([&] {
    need(sessions, "sessions");
    std::vector<void*> bases;
    for (int r = 0; r < world; ++r) {
      need(sessions[r], "session");
      bases.push_back(sessions[r]->s->export_arena(min_bytes));
    }
    for (int r = 0; r < world; ++r) sessions[r]->s->set_peer_arenas(bases);
  });
}

opf_status opf_session_bind(opf_session* s, const char* tensor, const opf_view* v) {
  return guard([&] {
    need(s, "session");
    need(v, "view");
    s->s->bind(tensor, *v);
  });
}

opf_status opf_session_run(opf_session* s, const char* strategy, void* stream) {
  return guard([&] {
    need(s, "session");
    const std::string spec = strategy ? strategy : "{}";
    auto cs = s->s->choose(spec, static_cast<cudaStream_t>(stream));
    auto strat = make_strategy(cs);
    s->s->run(*strat, "builtin:" + cs, static_cast<cudaStream_t>(stream));
  });
}

opf_status opf_session_check(opf_session* s) {
  return guard([&] {
    need(s, "session");
    s->s->check_window(true);
  });
}

opf_status opf_session_prepare(opf_session* s, const char* strategy, void* stream) {
  return guard([&] {
    need(s, "session");
    const std::string spec = strategy ? strategy : "{}";
    auto strat = make_strategy(spec);
    s->s->prepare(*strat, "builtin:" + spec, static_cast<cudaStream_t>(stream));
  });
}

opf_status opf_session_run_custom(opf_session* s, const char* key, opf_schedule_fn fn, void* user,
                                  void* stream) {
  return guard([&] {
    need(s, "session");
    CallbackStrategy strat(fn, user, key ? key : "custom");
    s->s->run(strat, std::string("custom:") + (key ? key : ""), static_cast<cudaStream_t>(stream));
  });
}

opf_status opf_session_output(opf_session* s, const char* tensor, opf_view* out) {
  return guard([&] {
    need(s, "session");
    *out = s->s->output(tensor);
  });
}

opf_status opf_session_stats(opf_session* s, char** json_out) {
  return guard([&] { *json_out = dup_string(s->s->stats_json()); });
}
opf_status opf_session_trace(opf_session* s, char** json_out) {
  return guard([&] { *json_out = dup_string(s->s->trace_json()); });
}
opf_status opf_session_schedule_dump(opf_session* s, char** json_out) {
  return guard([&] { *json_out = dup_string(s->s->schedule_json()); });
}

opf_status opf_dry_run(const opf_graph* g, const opf_plan* p, const char* config,
                       const char* strategy, int64_t rows, int32_t repeats, char** schedule_json,
                       char** stats_json) {
  return guard([&] {
    need(g, "graph");
    need(p, "plan");
    validate_plan(p->p, g->g);
    auto s = Session::dry(g->g, p->p, parse_config(config), rows);
    // a calibrated auto table resolves without a device; timed auto raises
    const std::string spec = s->choose(strategy ? strategy : "{}", nullptr);
    auto strat = make_strategy(spec);
    for (int32_t i = 0; i < std::max(1, repeats); ++i) s->plan_only(*strat, "builtin:" + spec);
    if (schedule_json) *schedule_json = dup_string(s->schedule_json());
    if (stats_json) *stats_json = dup_string(s->stats_json());
  });
}

opf_status opf_dry_run_custom(const opf_graph* g, const opf_plan* p, const char* config,
                              const char* key, opf_schedule_fn fn, void* user, int64_t rows,
                              char** schedule_json, char** stats_json) {
  return guard([&] {
    need(g, "graph");
    need(p, "plan");
    validate_plan(p->p, g->g);
    auto s = Session::dry(g->g, p->p, parse_config(config), rows);
    CallbackStrategy strat(fn, user, key ? key : "custom");
    s->plan_only(strat, std::string("custom:") + (key ? key : ""));
    if (schedule_json) *schedule_json = dup_string(s->schedule_json());
    if (stats_json) *stats_json = dup_string(s->stats_json());
  });
}

// ------------------------------------------------------------------ sched_api
opf_status opf_sched_split(opf_sched_ctx* c, const int64_t* sizes, int32_t n) {
  return guard([&] { c->ctx->split(std::vector<int64_t>(sizes, sizes + n)); });
}

opf_status opf_sched_ready(opf_sched_ctx* c, int32_t ubatch, opf_handle* out, int32_t cap,
                           int32_t* n_out) {
  return guard([&] {
    const auto hs = c->ctx->get_ready_ops(ubatch);
    *n_out = static_cast<int32_t>(hs.size());
    for (int32_t i = 0; i < *n_out && i < cap; ++i)
      out[i] = {hs[i].subgraph, hs[i].ubatch, hs[i].topo_index};
  });
}

opf_status opf_sched_handle(opf_sched_ctx* c, int32_t subgraph, int32_t ubatch, opf_handle* out) {
  return guard([&] {
    const OpHandle h = c->ctx->handle(subgraph, ubatch);
    *out = {h.subgraph, h.ubatch, h.topo_index};
  });
}

opf_status opf_sched_execute(opf_sched_ctx* c, const opf_handle* hs, int32_t n, int32_t lane,
                             const char* replace_fn) {
  return guard([&] {
    std::vector<OpHandle> v;
    for (int32_t i = 0; i < n; ++i) v.push_back({hs[i].subgraph, hs[i].ubatch, hs[i].topo_index});
    c->ctx->execute(v, lane, replace_fn ? replace_fn : "");
  });
}

opf_status opf_sched_rows(opf_sched_ctx* c, int64_t* rows) {
  return guard([&] { *rows = c->ctx->rows(); });
}
opf_status opf_sched_num_subgraphs(opf_sched_ctx* c, int32_t* n) {
  return guard([&] { *n = static_cast<int32_t>(c->ctx->plan().size()); });
}
opf_status opf_sched_label(opf_sched_ctx* c, int32_t subgraph, char* buf, int32_t cap) {
  return guard([&] {
    const auto& sgs = c->ctx->plan().subgraphs;
    require(subgraph >= 0 && subgraph < static_cast<int32_t>(sgs.size()), Errc::UnknownSubgraph,
            "subgraph index");
    std::snprintf(buf, static_cast<size_t>(cap), "%s", sgs[subgraph].label.c_str());
  });
}
opf_status opf_sched_unfinished(opf_sched_ctx* c, int32_t* n) {
  return guard([&] { *n = c->ctx->unfinished(); });
}

}  // extern "C"
