// Session: Algorithm-1 memory planning over one HBM arena, event-based
// multi-stream dispatch, CUDA-graph capture/replay with a plan cache.
#include "opflow/engine.hpp"

#include <algorithm>
#include <chrono>
#include <cstring>
#include <functional>
#include <numeric>

#include "opflow/comm.hpp"
#include "opflow/p2p.cuh"
#include "opflow/json.hpp"

namespace opflow {

namespace {

constexpr int64_t kAlign = 256;
int64_t align_up(int64_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

int64_t tensor_bytes_rows(const TensorMeta& m, int64_t rows) {
  return rows * m.row_elems() * dtype_bytes(m.dtype);
}

// Lane-aware block allocator: a freed block is handed out again only to a
// dispatch that happens-after every previous user (vector clocks over lanes).
struct Block {
  int64_t off = 0, bytes = 0;
  bool live = false;
  bool pinned = false;  // graph outputs: never recycled
  std::vector<int32_t> users;
};

struct Planner {
  std::vector<Block> blocks;
  int64_t top = 0, live = 0, peak = 0;
  const std::vector<std::vector<int32_t>>* vc = nullptr;  // per dispatch
  const std::vector<int32_t>* lane_of = nullptr;
  const std::vector<int32_t>* seq_of = nullptr;

  bool hb(int32_t x, int32_t d) const {
    if (x == d) return true;
    return (*vc)[d][(*lane_of)[x]] >= (*seq_of)[x];
  }
  // fresh: never recycle a freed block (merge buffers: later producers of other
  // ubatches write into them on lanes not ordered after the old tenant).
  int32_t alloc(int64_t bytes, int32_t d, bool pinned = false, bool fresh = false) {
    bytes = align_up(std::max<int64_t>(bytes, 1));
    int32_t best = -1;
    if (!pinned && !fresh) {
      for (int32_t i = 0; i < static_cast<int32_t>(blocks.size()); ++i) {
        const Block& b = blocks[i];
        if (b.live || b.pinned || b.bytes < bytes) continue;
        if (best >= 0 && blocks[best].bytes <= b.bytes) continue;
        bool ok = true;
        for (int32_t u : b.users) ok = ok && hb(u, d);
        if (ok) best = i;
      }
    }
    if (best < 0) {
      Block b;
      b.off = top;
      b.bytes = bytes;
      top += bytes;
      blocks.push_back(b);
      best = static_cast<int32_t>(blocks.size()) - 1;
    }
    Block& b = blocks[best];
    b.live = true;
    b.pinned = pinned;
    b.users.assign(1, d);
    live += b.bytes;
    peak = std::max(peak, live);
    return best;
  }
  void use(int32_t blk, int32_t d) {
    auto& u = blocks[blk].users;
    if (std::find(u.begin(), u.end(), d) == u.end()) u.push_back(d);
  }
  void release(int32_t blk) {
    Block& b = blocks[blk];
    if (!b.live || b.pinned) return;
    b.live = false;
    live -= b.bytes;
  }
};

struct InstBinding {
  int32_t block = -1;
  int64_t row_off = 0;   // rows into the block
  int32_t producer = -1; // dispatch id
};

}  // namespace

// ------------------------------------------------------------------ Session
Session::Session(const Graph& g, const PartitionPlan& p, SessionConfig cfg, opf_comm* comm)
    : g_(g), p_(p), cfg_(cfg), comm_(comm) {
  lanes_.assign(std::max(1, cfg_.lanes), nullptr);
  ext_.assign(g_.tensors.size(), opf_view{});
  prepacked_.assign(g_.tensors.size(), nullptr);
  prepacked_act_.assign(g_.tensors.size(), nullptr);
  if (cfg_.device < 0) return;  // dry session
  OPF_CUDA(cudaSetDevice(cfg_.device));
  for (auto& s : lanes_) OPF_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
}

std::unique_ptr<Session> Session::dry(const Graph& g, const PartitionPlan& p, SessionConfig cfg,
                                      int64_t rows) {
  cfg.device = -1;
  auto s = std::make_unique<Session>(g, p, cfg, nullptr);
  s->dry_ = true;
  s->dry_rows_ = rows;
  return s;
}

Session::~Session() {
  if (dry_) return;
  for (auto& kv : cache_)
    if (kv.second->exec) cudaGraphExecDestroy(kv.second->exec);
  for (auto& s : lanes_) cudaStreamDestroy(s);
  for (auto& e : events_) cudaEventDestroy(e);
  for (void* p : prepacked_)
    if (p) cudaFree(p);
  for (void* p : prepacked_act_)
    if (p) cudaFree(p);
  for (auto& kv : perms_) cudaFree(kv.second);
  if (arena_) cudaFree(arena_);
  if (win_err_ev_) cudaEventDestroy(win_err_ev_);
  if (win_err_host_) cudaFreeHost(win_err_host_);
}

void Session::check_window(bool wait) {
  if (!win_err_pending_) return;
  if (wait) {
    OPF_CUDA(cudaEventSynchronize(win_err_ev_));
  } else {
    const cudaError_t q = cudaEventQuery(win_err_ev_);
    if (q == cudaErrorNotReady) return;
    OPF_CUDA(q);
  }
  win_err_pending_ = false;
  if (*win_err_host_ != 0)
    fail(Errc::SchedulerError,
         "peer-window barrier timed out on rank " + std::to_string(comm_->rank) + " of " +
             std::to_string(comm_->world) +
             " (a peer never arrived): the outputs of that run are invalid and the window is poisoned");
}

void Session::note_window(cudaStream_t stream) {
  WindowView w;
  if (!window_view(comm_, &w)) return;
  if (!win_err_host_) {
    OPF_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&win_err_host_), sizeof(uint32_t), cudaHostAllocDefault));
    *win_err_host_ = 0;
    OPF_CUDA(cudaEventCreateWithFlags(&win_err_ev_, cudaEventDisableTiming));
  }
  OPF_CUDA(cudaMemcpyAsync(win_err_host_, w.err, sizeof(uint32_t), cudaMemcpyDeviceToHost, stream));
  OPF_CUDA(cudaEventRecord(win_err_ev_, stream));
  win_err_pending_ = true;
}

void Session::bind(const std::string& name, const opf_view& v) {
  const int32_t t = g_.tensor_id(name);
  const TensorMeta& m = g_.tensors[t];
  require(m.role != TensorRole::kIntermediate, Errc::ConfigError,
          "tensor '" + name + "' is an intermediate; only inputs, weights and outputs bind");
  require(v.dtype == static_cast<int32_t>(m.dtype), Errc::ShapeMismatch,
          "binding dtype mismatch for '" + name + "'");
  require(v.rank == static_cast<int32_t>(m.shape.size()), Errc::ShapeMismatch,
          "binding rank mismatch for '" + name + "'");
  for (int d = (m.batch == BatchSemantics::kBatched ? 1 : 0); d < v.rank; ++d)
    require(v.shape[d] == m.shape[d], Errc::ShapeMismatch,
            "binding extent mismatch for '" + name + "'");
  require(v.base != nullptr, Errc::MissingBinding, "null binding for '" + name + "'");
  const bool changed = ext_[t].base != v.base || ext_[t].elem_offset != v.elem_offset ||
                       ext_[t].shape[0] != v.shape[0];
  ext_[t] = v;
  if (changed) {
    if (m.role == TensorRole::kWeight) {
      prepack_dirty_ = true;
      for (std::vector<void*>* v : {&prepacked_, &prepacked_act_})
        if ((*v)[t]) {
          cudaFree((*v)[t]);
          (*v)[t] = nullptr;
        }
    }
    // captured graphs embed pointers: drop them (plans are rebuilt lazily)
    for (auto& kv : cache_)
      if (kv.second->exec) {
        cudaGraphExecDestroy(kv.second->exec);
        kv.second->exec = nullptr;
      }
  }
}

int64_t Session::rows() const {
  if (dry_) return dry_rows_;
  int64_t rows = 0;
  for (int32_t t : g_.graph_inputs) {
    const TensorMeta& m = g_.tensors[t];
    require(ext_[t].base != nullptr, Errc::MissingBinding,
            "no binding for tensor '" + m.name + "'");
    if (m.batch != BatchSemantics::kBatched) continue;
    if (rows == 0) rows = ext_[t].shape[0];
    require(ext_[t].shape[0] == rows, Errc::ShapeMismatch, "batched inputs disagree on rows");
  }
  for (int32_t t : g_.weights)
    require(ext_[t].base != nullptr, Errc::MissingBinding,
            "no binding for tensor '" + g_.tensors[t].name + "'");
  return rows == 0 ? 1 : rows;
}

void Session::ensure_prepacked(cudaStream_t) {}

void Session::ensure_packed_for(const CompiledPlan& cp, cudaStream_t s) {
  // MatMul bf16 weights are [K,N] (reference layout); the tcgen05 GEMM wants
  // K-major B ([N,K]), gate/up-interleaved for the SiLU-mul epilogue.  Packed
  // once per binding, outside any capture.
  for (const PlannedDispatch& pd : cp.dispatches)
    for (const PlannedLaunch& l : pd.launches) {
      if (l.prepacked < 0) continue;
      const int32_t w = l.prepacked;
      const TensorMeta& m = g_.tensors[w];
      std::vector<void*>& slot = l.prepack_mode == 1 ? prepacked_act_ : prepacked_;
      if (slot[w]) continue;
      OPF_CUDA(cudaMalloc(&slot[w], m.numel() * 2));
      if (l.prepack_mode == 1) {
        k_pack_gate_up(view_ptr(ext_[w]), slot[w], m.shape[0], m.shape[1] / 2, s);
      } else if (l.prepack_mode == 2 || l.prepack_mode == 3) {  // per-expert [E,K,N]
        require(m.shape.size() == 3, Errc::ShapeMismatch, "expert weight '" + m.name + "' must be [E,K,N]");
        const int64_t E = m.shape[0], K = m.shape[1], N = m.shape[2];
        const char* src = static_cast<const char*>(view_ptr(ext_[w]));
        char* dst = static_cast<char*>(slot[w]);
        for (int64_t e = 0; e < E; ++e) {
          if (l.prepack_mode == 2)
            k_pack_gate_up(src + e * K * N * 2, dst + e * K * N * 2, K, N / 2, s);
          else
            k_transpose_bf16(src + e * K * N * 2, dst + e * K * N * 2, K, N, s);
        }
      } else
        k_transpose_bf16(view_ptr(ext_[w]), slot[w], m.shape[0], m.shape[1], s);
    }
  OPF_CUDA(cudaGetLastError());
}

void Session::warm_aux(const CompiledPlan& cp) {
  for (const PlannedDispatch& pd : cp.dispatches)
    for (const PlannedLaunch& l : pd.launches)
      if (!l.is_copy && l.fn.empty() && l.kind == OperatorKind::kAllToAll)
        alltoall_perm_device(l.attrs.seed, l.in[0].shape.size() > 1 ? l.in[0].shape[1] : 1);
}

void Session::ensure_arena(int64_t bytes) {
  if (bytes <= arena_bytes_) return;
  require(!arena_pinned_, Errc::ConfigError,
          "plan needs a " + std::to_string(bytes) + "-byte arena but the arena is peer-mapped at " +
              std::to_string(arena_bytes_) + " bytes (export a larger arena before mapping peers)");
  if (arena_) {
    OPF_CUDA(cudaDeviceSynchronize());
    OPF_CUDA(cudaFree(arena_));
  }
  OPF_CUDA(cudaMalloc(&arena_, bytes));
  arena_bytes_ = bytes;
}

void* Session::export_arena(int64_t bytes) {
  require(!dry_, Errc::ConfigError, "dry sessions have no arena");
  require(comm_ != nullptr, Errc::ConfigError, "peer arena needs a communicator");
  ensure_arena(std::max<int64_t>(bytes, 1));
  arena_pinned_ = true;
  return arena_;
}

void Session::set_peer_arenas(const std::vector<void*>& bases) {
  require(comm_ != nullptr && static_cast<int>(bases.size()) == comm_->world, Errc::ConfigError,
          "peer arenas: one base per rank");
  require(arena_pinned_ && bases[comm_->rank] == arena_, Errc::ConfigError, "export the arena first");
  comm_->arena_base = arena_;
  comm_->arena_bytes = static_cast<size_t>(arena_bytes_);
  comm_->peer_arena = bases;
}

std::unique_ptr<CompiledPlan> Session::compile(const SchedContext& ctx, const std::string& key,
                                               const std::vector<int>& budgets_in) {
  const std::vector<int>& budgets = budgets_in.empty() ? cfg_.lane_sm_budget : budgets_in;
  auto cp = std::make_unique<CompiledPlan>();
  cp->key = key;
  const auto& ds = ctx.dispatches();
  const int32_t nd = static_cast<int32_t>(ds.size());
  SchedContext& mctx = const_cast<SchedContext&>(ctx);
  const std::vector<int64_t> sizes = mctx.sizes();
  const int32_t U = static_cast<int32_t>(sizes.size());
  std::vector<int64_t> offs(U + 1, 0);
  for (int32_t u = 0; u < U; ++u) offs[u + 1] = offs[u] + sizes[u];
  const int64_t total_rows = offs[U];

  SplitSignature sig;
  sig.sizes = sizes;
  for (const Dispatch& d : ds)
    if (d.kind == Dispatch::Kind::kMerged) sig.merge_set.insert(d.subgraphs[0]);
  std::vector<MicroBatchContext> mb = static_analysis(g_, p_, sig);
  cp->analysis_ops += static_cast<int64_t>(g_.tensors.size()) * U + p_.size();
  if (!cfg_.prealloc)
    for (auto& c : mb)
      for (auto& st : c.states) st.prealloc = false;

  const int L = static_cast<int>(lanes_.size());
  std::vector<std::vector<int32_t>> vc(nd, std::vector<int32_t>(L, 0));
  std::vector<int32_t> lane_of(nd), seq_of(nd), lane_last(L, -1), lane_seq(L, 0);
  Planner pl;
  pl.vc = &vc;
  pl.lane_of = &lane_of;
  pl.seq_of = &seq_of;

  const int32_t NT = static_cast<int32_t>(g_.tensors.size());
  std::vector<std::vector<InstBinding>> inst(NT, std::vector<InstBinding>(U));
  std::vector<int32_t> merge_buf(NT, -1);  // full-batch block of prealloc / output tensors
  std::vector<int32_t> block_pending;      // live (t,u) slices per block
  auto pending = [&](int32_t b) -> int32_t& {
    if (static_cast<int32_t>(block_pending.size()) <= b) block_pending.resize(b + 1, 0);
    return block_pending[b];
  };

  // Graph outputs not bound by the caller live in pinned arena blocks.
  for (int32_t t : g_.graph_outputs)
    if (!ext_[t].base) {
      merge_buf[t] = pl.alloc(tensor_bytes_rows(g_.tensors[t], total_rows), -1, true);
      pl.blocks[merge_buf[t]].users.clear();
    }

  auto ext_view = [&](int32_t t, int64_t r0, int64_t nrows) {
    const TensorMeta& m = g_.tensors[t];
    PlannedView v;
    v.src = PlannedView::Src::kExternal;
    v.tensor = t;
    v.dtype = m.dtype;
    v.batched = m.batch == BatchSemantics::kBatched;
    v.shape = m.shape;
    if (v.batched) {
      v.shape[0] = nrows;
      v.elem_offset = r0 * m.row_elems();
    }
    return v;
  };
  auto arena_view = [&](int32_t blk, int32_t t, int64_t row_off, int64_t nrows) {
    const TensorMeta& m = g_.tensors[t];
    PlannedView v;
    v.src = PlannedView::Src::kArena;
    v.block_off = pl.blocks[blk].off;
    v.tensor = blk;
    v.dtype = m.dtype;
    v.shape = m.shape;
    v.shape[0] = nrows;
    v.elem_offset = row_off * m.row_elems();
    v.batched = true;
    return v;
  };

  int32_t last_comm = -1;
  for (int32_t di = 0; di < nd; ++di) {
    const Dispatch& d = ds[di];
    PlannedDispatch pd;
    pd.d = d;
    const int64_t r0 = offs[d.u0], nrows = offs[d.u1] - offs[d.u0];
    pd.rows = nrows;
    lane_of[di] = d.lane;

    // ---- member ops, produced set, boundary inputs/outputs of the dispatch
    std::vector<int32_t> ops;
    std::set<int32_t> produced, member_set(d.subgraphs.begin(), d.subgraphs.end());
    for (int32_t s : d.subgraphs)
      for (int32_t op : p_.subgraphs[s].ops) ops.push_back(op);
    for (int32_t op : ops)
      for (int32_t t : g_.ops[op].outputs) produced.insert(t);
    std::vector<int32_t> b_in, b_out;  // ordered (first use / production order)
    for (int32_t op : ops)
      for (int32_t t : g_.ops[op].inputs)
        if (!produced.count(t) && std::find(b_in.begin(), b_in.end(), t) == b_in.end())
          b_in.push_back(t);
    for (int32_t op : ops)
      for (int32_t t : g_.ops[op].outputs) {
        bool leaves = g_.is_output(t);
        for (int32_t c : g_.tensors[t].consumers)
          leaves = leaves || !member_set.count(p_.op_to_subgraph[c]);
        if (leaves) b_out.push_back(t);
      }
    // boundary inputs as Algorithm 1 sees them: per member subgraph
    std::vector<std::pair<int32_t, int32_t>> consumed;  // (tensor, member subgraph)
    for (int32_t s : d.subgraphs)
      for (int32_t t : p_.subgraphs[s].boundary_inputs) consumed.push_back({t, s});

    // ---- dependencies from input producers
    std::set<int32_t> deps;
    for (int32_t t : b_in) {
      const TensorMeta& m = g_.tensors[t];
      if (m.producer < 0) {
        require(dry_ || ext_[t].base != nullptr, Errc::MissingBinding,
                "no binding for '" + m.name + "'");
        continue;
      }
      for (int32_t u = d.u0; u < d.u1; ++u) {
        const TensorState& st = mb[u].states[t];
        require(st.binding != BindingKind::kUnmaterialized, Errc::Unmaterialized,
                "tensor '" + m.name + "' ubatch " + std::to_string(u) + " not materialized");
        require(st.ref_count > 0, Errc::UseAfterFree,
                "tensor '" + m.name + "' ubatch " + std::to_string(u) + " already reclaimed");
        deps.insert(inst[t][u].producer);
      }
    }
    // Communicating dispatches form one global chain, identical on every rank:
    // two collectives (NCCL, or peer-window kernels sharing the staging window and
    // flags) must never run concurrently on different lanes.
    bool comm_dispatch = false;
    const int world = cfg_.world > 0 ? cfg_.world : (comm_ ? comm_->world : 1);
    if (world > 1)
      for (int32_t op : ops) comm_dispatch = comm_dispatch || g_.ops[op].resource_class == ResourceClass::kNetwork;
    if (comm_dispatch) {
      if (last_comm >= 0) deps.insert(last_comm);
      last_comm = di;
    }
    // vector clock of this dispatch
    std::vector<int32_t>& my = vc[di];
    if (lane_last[d.lane] >= 0) my = vc[lane_last[d.lane]];
    for (int32_t x : deps)
      for (int l = 0; l < L; ++l) my[l] = std::max(my[l], vc[x][l]);
    const std::vector<int32_t> before = lane_last[d.lane] >= 0 ? vc[lane_last[d.lane]]
                                                              : std::vector<int32_t>(L, 0);
    seq_of[di] = ++lane_seq[d.lane];
    my[d.lane] = seq_of[di];
    for (int32_t x : deps)
      if (lane_of[x] != d.lane && before[lane_of[x]] < seq_of[x]) {
        // not yet ordered by an earlier wait on this lane
        bool covered = false;
        for (int32_t y : pd.wait_on) covered = covered || (vc[y][lane_of[x]] >= seq_of[x]);
        if (!covered) pd.wait_on.push_back(x);
      }
    std::sort(pd.wait_on.begin(), pd.wait_on.end());

    // ---- input views (zero-copy slices, or counted concat copies in fallback mode)
    std::map<int32_t, PlannedView> view_of;
    std::vector<int32_t> scratch;  // blocks freed after this dispatch
    for (int32_t t : b_in) {
      const TensorMeta& m = g_.tensors[t];
      if (m.producer < 0) {
        view_of[t] = ext_view(t, r0, nrows);
        continue;
      }
      const InstBinding& first = inst[t][d.u0];
      bool contiguous = true;
      for (int32_t u = d.u0 + 1; u < d.u1; ++u)
        contiguous = contiguous && inst[t][u].block == first.block &&
                     inst[t][u].row_off == first.row_off + (offs[u] - offs[d.u0]);
      if (contiguous) {
        view_of[t] = first.block == -2 ? ext_view(t, r0, nrows)
                                       : arena_view(first.block, t, first.row_off, nrows);
        if (first.block >= 0)
          for (int32_t u = d.u0; u < d.u1; ++u) pl.use(inst[t][u].block, di);
        continue;
      }
      // copying fallback: concat_rows into a fresh block (copies counted)
      const int32_t blk = pl.alloc(tensor_bytes_rows(m, nrows), di);
      scratch.push_back(blk);
      for (int32_t u = d.u0; u < d.u1; ++u) {
        const InstBinding& ib = inst[t][u];
        PlannedLaunch cpy;
        cpy.is_copy = true;
        cpy.name = "concat_rows:" + m.name;
        cpy.rows = sizes[u];
        cpy.in.push_back(ib.block == -2 ? ext_view(t, offs[u], sizes[u])
                                        : arena_view(ib.block, t, ib.row_off, sizes[u]));
        cpy.out.push_back(arena_view(blk, t, offs[u] - offs[d.u0], sizes[u]));
        if (ib.block >= 0) pl.use(ib.block, di);
        pd.launches.push_back(std::move(cpy));
        cp->copied_elements += sizes[u] * m.row_elems();
      }
      view_of[t] = arena_view(blk, t, 0, nrows);
    }

    // ---- output bindings (on_outputs)
    for (int32_t t : b_out) {
      const TensorMeta& m = g_.tensors[t];
      for (int32_t u = d.u0; u < d.u1; ++u)
        require(mb[u].states[t].binding == BindingKind::kUnmaterialized, Errc::DoubleProduce,
                "tensor '" + m.name + "' produced twice in ubatch " + std::to_string(u));
      if (g_.is_output(t) && ext_[t].base) {
        for (int32_t u = d.u0; u < d.u1; ++u) {
          inst[t][u] = {-2, offs[u], di};
          mb[u].states[t].binding = BindingKind::kSlice;
        }
        view_of[t] = ext_view(t, r0, nrows);
        continue;
      }
      const bool full = g_.is_output(t) || mb[d.u0].states[t].prealloc;
      int32_t blk;
      int64_t base_row;
      if (full) {
        // MergeBuffer: one full-batch block; it stays live until every
        // ubatch's slice has been produced AND consumed (pending = U).
        if (merge_buf[t] < 0) {
          merge_buf[t] = pl.alloc(tensor_bytes_rows(m, total_rows), di, false, /*fresh=*/true);
          pending(merge_buf[t]) = U;
        }
        blk = merge_buf[t];
        pl.use(blk, di);
        base_row = r0;
      } else {
        blk = pl.alloc(tensor_bytes_rows(m, nrows), di);
        pending(blk) = d.u1 - d.u0;
        base_row = 0;
      }
      for (int32_t u = d.u0; u < d.u1; ++u) {
        inst[t][u] = {blk, base_row + (offs[u] - offs[d.u0]), di};
        mb[u].states[t].binding = full ? BindingKind::kSlice : BindingKind::kOwned;
        mb[u].states[t].buffer = blk;
        mb[u].states[t].row_offset = inst[t][u].row_off;
        mb[u].states[t].row_extent = sizes[u];
      }
      view_of[t] = arena_view(blk, t, base_row, nrows);
    }

    // workspace + SM budget of one planned launch; the workspace block is live
    // only for this launch (later launches of this dispatch may reuse it)
    auto plan_ws = [&](PlannedLaunch& l) {
      if (l.is_copy) return;
      if (cfg_.gemm_sm_budget > 0 && d.lane == 0) l.max_ctas = cfg_.gemm_sm_budget;
      if (d.lane < static_cast<int>(budgets.size()) && budgets[d.lane] > 0) l.max_ctas = budgets[d.lane];
      opf_op_ctx c{};
      c.kind = static_cast<int32_t>(l.kind);
      c.world_size = l.attrs.world_size;
      c.comm = comm_;
      c.max_ctas = l.max_ctas;
      std::vector<opf_view> iv, ov;
      for (const auto& v : l.in) iv.push_back(make_view(nullptr, v.elem_offset, v.dtype, v.shape, v.batched));
      for (const auto& v : l.out) ov.push_back(make_view(nullptr, v.elem_offset, v.dtype, v.shape, v.batched));
      std::vector<const char*> pn;
      std::vector<double> pv;
      for (const auto& kv : l.attrs.params) {
        pn.push_back(kv.first.c_str());
        pv.push_back(kv.second);
      }
      c.n_params = static_cast<int32_t>(pn.size());
      c.param_names = pn.data();
      c.param_values = pv.data();
      size_t ws = 0;
      if (l.fn.empty()) {
        ws = kind_workspace(c, iv.data(), static_cast<int>(iv.size()), ov.data(),
                            static_cast<int>(ov.size()), l.rows);
      } else if (const OpEntry* e = OpRegistry::global().find(l.fn); e && e->workspace) {
        ws = e->workspace(c, iv.data(), static_cast<int>(iv.size()), ov.data(),
                          static_cast<int>(ov.size()), l.rows);
      }
      if (ws > 0) {
        const int32_t blk = pl.alloc(static_cast<int64_t>(ws), di);
        l.ws_off = pl.blocks[blk].off;
        l.ws_bytes = static_cast<int64_t>(ws);
        pl.release(blk);
      }
    };

    // ---- launches
    auto weight_view = [&](int32_t t, const OperatorNode&) { return ext_view(t, 0, 0); };
    const bool fused = d.kind == Dispatch::Kind::kFused;
    if (fused) {
      PlannedLaunch l;
      l.fn = d.replace_fn;
      l.name = d.replace_fn;
      l.rows = nrows;
      for (int32_t op : ops) {  // merged attrs: max world_size, union of params
        const OpAttrs& a = g_.ops[op].attrs;
        l.attrs.world_size = std::max(l.attrs.world_size, a.world_size);
        if (!l.attrs.seed) l.attrs.seed = a.seed;
        for (const auto& kv : a.params) l.attrs.params.insert(kv);
        l.name += ":" + g_.ops[op].name;
      }
      l.attrs.custom_name = d.replace_fn;
      for (int32_t t : b_in)
        l.in.push_back(g_.tensors[t].role == TensorRole::kWeight ? ext_view(t, 0, 0) : view_of.at(t));
      for (int32_t t : b_out) l.out.push_back(view_of.at(t));
      const OpEntry* e = OpRegistry::global().find(d.replace_fn);
      require(e != nullptr, Errc::SignatureMismatch, "no replacement op '" + d.replace_fn + "'");
      require((e->n_in < 0 || e->n_in == static_cast<int>(l.in.size())) &&
                  (e->n_out < 0 || e->n_out == static_cast<int>(l.out.size())),
              Errc::SignatureMismatch,
              "replacement '" + d.replace_fn + "' takes " + std::to_string(e->n_in) + "->" +
                  std::to_string(e->n_out) + " tensors, fused subgraphs expose " +
                  std::to_string(l.in.size()) + "->" + std::to_string(l.out.size()));
      if (e->prepack_input >= 0 && e->prepack_input < static_cast<int>(b_in.size()) &&
          g_.tensors[b_in[e->prepack_input]].role == TensorRole::kWeight &&
          g_.tensors[b_in[e->prepack_input]].dtype == Dtype::kBF16) {
        l.prepacked = b_in[e->prepack_input];  // e.g. the GEMM weight of matmul_allreduce_add_rmsnorm
        l.prepack_mode = e->prepack_mode;
      }
      pd.launches.push_back(std::move(l));
      plan_ws(pd.launches.back());
    } else {
      // Epilogue fusion (per-subgraph compilation): a bf16
      // MatMul whose output feeds only a silu_mul (or a rope) of the same
      // dispatch runs as ONE tcgen05 GEMM with the SiLU-mul (RoPE) epilogue;
      // the un-activated [T, 2I] (un-rotated qkv) never touches HBM.
      std::map<int32_t, int32_t> fused_act;  // matmul op -> silu_mul op
      std::set<int32_t> skip;
      if (cfg_.fuse) {
        const std::set<int32_t> in_dispatch(ops.begin(), ops.end());
        std::map<int32_t, int32_t> pos_of;  // op -> position in this dispatch
        for (int32_t k = 0; k < static_cast<int32_t>(ops.size()); ++k) pos_of[ops[k]] = k;
        for (int32_t op : ops) {
          const OperatorNode& node = g_.ops[op];
          if (node.kind != OperatorKind::kMatMul) continue;
          const TensorMeta& w = g_.tensors[node.inputs[1]];
          const int32_t t = node.outputs[0];
          const auto& cons = g_.tensors[t].consumers;
          if (w.dtype != Dtype::kBF16 || w.role != TensorRole::kWeight || w.shape[1] % 256 != 0 ||
              cons.size() != 1 || !in_dispatch.count(cons[0]) || g_.is_output(t) ||
              std::find(b_out.begin(), b_out.end(), t) != b_out.end())
            continue;
          const OperatorNode& act = g_.ops[cons[0]];
          if (act.kind != OperatorKind::kCustom) continue;
          const bool silu = act.attrs.custom_name == "silu_mul";
          // RoPE epilogue: 128-wide heads tiling N (two per 256-column tile)
          const auto hd = act.attrs.params.find("head_dim");
          const bool rope = act.attrs.custom_name == "rope" && act.inputs.size() == 2 && act.inputs[0] == t &&
                            hd != act.attrs.params.end() && hd->second == 128.0;
          // residual add + RMSNorm: the MatMul output is add_rmsnorm's second
          // input; the residual and gamma must exist by the MatMul's position
          bool addnorm = cfg_.fuse_addnorm && act.attrs.custom_name == "add_rmsnorm" && act.inputs.size() == 3 &&
                         act.outputs.size() == 2 && act.inputs[1] == t && act.inputs[0] != t &&
                         g_.tensors[act.inputs[0]].dtype == Dtype::kBF16;
          if (addnorm) {  // only where the plain GEMM would not split K (decode-size rows keep split-K)
            int mc = 0;
            if (cfg_.gemm_sm_budget > 0 && d.lane == 0) mc = cfg_.gemm_sm_budget;
            if (d.lane < static_cast<int>(budgets.size()) && budgets[d.lane] > 0) mc = budgets[d.lane];
            addnorm = gemm_splitk_splits(nrows, w.shape[1], w.shape[0], mc) <= 1;
          }
          for (int32_t u : {act.inputs.size() == 3 ? act.inputs[0] : -1, act.inputs.size() == 3 ? act.inputs[2] : -1})
            if (addnorm && u >= 0) {
              const int32_t p = g_.tensors[u].producer;
              if (p >= 0 && in_dispatch.count(p) && pos_of[p] > pos_of[op]) addnorm = false;
            }
          if (!silu && !rope && !addnorm) continue;
          fused_act[op] = cons[0];
          skip.insert(cons[0]);
        }
      }
      // internal tensors of the subgraph get arena blocks from their producer to
      // their last consumer within this dispatch (launches of a dispatch run in
      // order on its lane, so a block freed after op k is reusable from op k+1)
      std::map<int32_t, int32_t> last_pos, int_blk;
      for (int32_t k = 0; k < static_cast<int32_t>(ops.size()); ++k)
        for (int32_t t : g_.ops[ops[k]].inputs) last_pos[t] = k;
      auto retire_inputs = [&](int32_t k, const std::vector<int32_t>& ins) {
        for (int32_t t : ins) {
          auto ib = int_blk.find(t);
          if (ib != int_blk.end() && last_pos[t] <= k) {
            pl.release(ib->second);
            int_blk.erase(ib);
          }
        }
      };
      for (int32_t k = 0; k < static_cast<int32_t>(ops.size()); ++k) {
        const int32_t op = ops[k];
        if (skip.count(op)) {  // ran inside its producer's GEMM epilogue: its inputs retire here
          retire_inputs(k, g_.ops[op].inputs);
          continue;
        }
        const OperatorNode& node = g_.ops[op];
        auto fa = fused_act.find(op);
        if (fa != fused_act.end()) {
          const OperatorNode& act = g_.ops[fa->second];
          for (int32_t a_out : act.outputs)
            if (!view_of.count(a_out)) {
              const int32_t blk = pl.alloc(tensor_bytes_rows(g_.tensors[a_out], nrows), di);
              scratch.push_back(blk);
              int_blk[a_out] = blk;
              view_of[a_out] = arena_view(blk, a_out, 0, nrows);
            }
          const bool rope = act.attrs.custom_name == "rope";
          const bool addnorm = act.attrs.custom_name == "add_rmsnorm";
          PlannedLaunch l;
          l.op = op;
          l.kind = OperatorKind::kMatMul;
          l.attrs = node.attrs;
          if (rope || addnorm)
            for (const auto& kv : act.attrs.params) l.attrs.params[kv.first] = kv.second;
          l.attrs.params["epi"] = rope ? 2.0 : (addnorm ? 4.0 : 1.0);
          l.name = node.name + "+" + act.name;
          l.rows = nrows;
          l.in.push_back(view_of.at(node.inputs[0]));
          l.in.push_back(weight_view(node.inputs[1], node));
          if (rope) l.in.push_back(view_of.at(act.inputs[1]));  // positions
          if (addnorm) {                                         // residual x, gamma
            l.in.push_back(view_of.at(act.inputs[0]));
            l.in.push_back(g_.tensors[act.inputs[2]].role == TensorRole::kWeight ? weight_view(act.inputs[2], act)
                                                                                 : view_of.at(act.inputs[2]));
          }
          for (int32_t o : act.outputs) l.out.push_back(view_of.at(o));
          l.prepacked = node.inputs[1];
          l.prepack_mode = (rope || addnorm) ? 0 : 1;
          pd.launches.push_back(std::move(l));
          plan_ws(pd.launches.back());
          // only inputs whose last consumer is this MatMul retire here (an input
          // also read by the skipped act or a later op stays to the dispatch end)
          retire_inputs(k, node.inputs);
          continue;
        }
        for (int32_t t : node.outputs)
          if (!view_of.count(t)) {
            const int32_t blk = pl.alloc(tensor_bytes_rows(g_.tensors[t], nrows), di);
            scratch.push_back(blk);
            int_blk[t] = blk;
            view_of[t] = arena_view(blk, t, 0, nrows);
          }
        PlannedLaunch l;
        l.op = op;
        l.kind = node.kind;
        l.fn = node.kind == OperatorKind::kCustom ? node.attrs.custom_name : "";
        l.attrs = node.attrs;
        l.name = node.name;
        l.rows = nrows;
        for (int32_t t : node.inputs)
          l.in.push_back(g_.tensors[t].role == TensorRole::kWeight ? weight_view(t, node)
                                                                     : view_of.at(t));
        for (int32_t t : node.outputs) l.out.push_back(view_of.at(t));
        if (node.kind == OperatorKind::kMatMul && g_.tensors[node.inputs[1]].dtype == Dtype::kBF16 &&
            g_.tensors[node.inputs[1]].role == TensorRole::kWeight)
          l.prepacked = node.inputs[1];  // aux = [N,K] copy, resolved at launch
        if (node.kind == OperatorKind::kCustom) {
          const OpEntry* e = OpRegistry::global().find(node.attrs.custom_name);
          require(e != nullptr, Errc::ConfigError,
                  "no device op registered for '" + node.attrs.custom_name + "'");
          if (e->prepack_input >= 0 && e->prepack_input < static_cast<int>(node.inputs.size()) &&
              g_.tensors[node.inputs[e->prepack_input]].role == TensorRole::kWeight) {
            l.prepacked = node.inputs[e->prepack_input];
            l.prepack_mode = e->prepack_mode;
          }
        }
        pd.launches.push_back(std::move(l));
        plan_ws(pd.launches.back());
        retire_inputs(k, node.inputs);
      }
    }
    // ---- on_inputs: decrement ref counts, reclaim dead slices after the dispatch
    for (const auto& [t, s] : consumed) {
      (void)s;
      if (g_.tensors[t].producer < 0) continue;
      const bool internal = produced.count(t) > 0;
      if (internal && std::find(b_out.begin(), b_out.end(), t) == b_out.end()) continue;
      for (int32_t u = d.u0; u < d.u1; ++u) {
        TensorState& st = mb[u].states[t];
        require(st.ref_count > 0, Errc::UseAfterFree,
                "tensor '" + g_.tensors[t].name + "' over-consumed");
        if (--st.ref_count == 0 && !g_.is_output(t)) {
          const int32_t blk = inst[t][u].block;
          if (blk >= 0 && --pending(blk) == 0) pl.release(blk);
        }
      }
    }
    // fused-internal tensors never materialize: retire their Algorithm-1 state
    if (fused)
      for (int32_t t : produced)
        if (std::find(b_out.begin(), b_out.end(), t) == b_out.end())
          for (int32_t u = d.u0; u < d.u1; ++u) mb[u].states[t].ref_count = 0;
    for (int32_t blk : scratch) pl.release(blk);
    lane_last[d.lane] = di;
    cp->n_launches += static_cast<int64_t>(pd.launches.size());
    cp->dispatches.push_back(std::move(pd));
  }
  // events are recorded only where another lane waits
  for (const PlannedDispatch& pd : cp->dispatches)
    for (int32_t x : pd.wait_on) cp->dispatches[x].record_event = true;
  std::set<int32_t> used;
  for (const Dispatch& d : ds) used.insert(d.lane);
  cp->lanes_used = static_cast<int>(used.size());
  for (int32_t t : g_.graph_outputs)
    if (merge_buf[t] >= 0) cp->outputs.push_back({t, pl.blocks[merge_buf[t]].off});
  cp->end_live_tensors = 0;
  for (int32_t t = 0; t < NT; ++t)
    for (int32_t u = 0; u < U; ++u)
      if (g_.tensors[t].producer >= 0 && !g_.is_output(t) && mb[u].states[t].ref_count > 0) {
        ++cp->end_live_tensors;
        break;
      }
  cp->arena_bytes = pl.top;
  cp->peak_live_bytes = pl.peak;
  return cp;
}

opf_view Session::resolve(const PlannedView& v) const {
  switch (v.src) {
    case PlannedView::Src::kArena:
      return make_view(static_cast<char*>(arena_) + v.block_off, v.elem_offset, v.dtype, v.shape,
                       v.batched);
    case PlannedView::Src::kExternal: {
      const opf_view& e = ext_[v.tensor];
      return make_view(e.base, e.elem_offset + v.elem_offset, v.dtype, v.shape, v.batched);
    }
    case PlannedView::Src::kPrepacked:
      return make_view(prepacked_[v.tensor], 0, v.dtype, v.shape, false);
    default:
      fail(Errc::Unmaterialized, "unresolved planned view");
  }
}

void Session::launch_one(const PlannedLaunch& l, cudaStream_t s) {
  if (l.is_copy) {
    const opf_view src = resolve(l.in[0]), dst = resolve(l.out[0]);
    k_copy_rows(view_ptr(src), view_ptr(dst), view_numel(src) * dtype_bytes(Dtype(src.dtype)), s);
    return;
  }
  std::vector<opf_view> iv, ov;
  for (const auto& v : l.in) iv.push_back(resolve(v));
  for (const auto& v : l.out) ov.push_back(resolve(v));
  std::vector<const char*> pn;
  std::vector<double> pv;
  for (const auto& kv : l.attrs.params) {
    pn.push_back(kv.first.c_str());
    pv.push_back(kv.second);
  }
  opf_op_ctx c{};
  c.op_name = l.name.c_str();
  c.kind = static_cast<int32_t>(l.kind);
  c.custom_name = l.attrs.custom_name.c_str();
  c.world_size = l.attrs.world_size;
  c.seed = l.attrs.seed;
  c.n_params = static_cast<int32_t>(pn.size());
  c.param_names = pn.data();
  c.param_values = pv.data();
  c.max_ctas = l.max_ctas;
  c.comm = comm_;
  c.aux = l.prepacked >= 0 ? (l.prepack_mode == 1 ? prepacked_act_ : prepacked_)[l.prepacked] : l.aux;
  if (l.kind == OperatorKind::kAllToAll && l.fn.empty())
    c.aux = alltoall_perm_device(l.attrs.seed, view_row_elems(iv[0]));
  c.workspace = l.ws_off >= 0 ? static_cast<char*>(arena_) + l.ws_off : nullptr;
  c.workspace_bytes = static_cast<size_t>(l.ws_bytes);
  opf_status st;
  if (l.fn.empty()) {
    st = launch_kind(c, iv.data(), static_cast<int>(iv.size()), ov.data(),
                     static_cast<int>(ov.size()), l.rows, s);
  } else {
    const OpEntry* e = OpRegistry::global().find(l.fn);
    require(e != nullptr, Errc::ConfigError, "no device op '" + l.fn + "'");
    st = e->fn(&c, iv.data(), static_cast<int>(iv.size()), ov.data(), static_cast<int>(ov.size()),
               l.rows, s);
  }
  if (st != 0)
    fail(static_cast<Errc>(st - 1), "op '" + l.name + "': " + std::string(opf_last_error()));
}

void Session::launch_plan(CompiledPlan& cp, cudaStream_t origin, bool capturing) {
  const int L = static_cast<int>(lanes_.size());
  const std::size_t need = cp.dispatches.size() + L + 1;
  while (events_.size() < need) {
    cudaEvent_t e;
    OPF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    events_.push_back(e);
  }
  cudaEvent_t fork = events_[cp.dispatches.size()];
  OPF_CUDA(cudaEventRecord(fork, origin));
  std::vector<bool> used(L, false);
  for (const PlannedDispatch& pd : cp.dispatches) used[pd.d.lane] = true;
  for (int l = 0; l < L; ++l)
    if (used[l]) OPF_CUDA(cudaStreamWaitEvent(lanes_[l], fork, 0));
  for (const PlannedDispatch& pd : cp.dispatches) {
    cudaStream_t s = lanes_[pd.d.lane];
    for (int32_t w : pd.wait_on) OPF_CUDA(cudaStreamWaitEvent(s, events_[w], 0));
    for (const PlannedLaunch& l : pd.launches) launch_one(l, s);
    if (pd.record_event) OPF_CUDA(cudaEventRecord(events_[pd.d.id], s));
  }
  for (int l = 0; l < L; ++l)
    if (used[l]) {
      cudaEvent_t j = events_[cp.dispatches.size() + 1 + l];
      OPF_CUDA(cudaEventRecord(j, lanes_[l]));
      OPF_CUDA(cudaStreamWaitEvent(origin, j, 0));
    }
  (void)capturing;
}

CompiledPlan* Session::lookup_or_build(Scheduler& strat, const std::string& key_in) {
  const int64_t r = rows();
  const std::string key = key_in + "|rows=" + std::to_string(r);
  ++runs_;
  auto it = cache_.find(key);
  if (it != cache_.end()) {
    ++hits_;
    return it->second.get();
  }
  ++misses_;
  SchedContext ctx(g_, p_, r, static_cast<int>(lanes_.size()));
  strat.schedule(ctx);
  ctx.finish();
  auto built = compile(ctx, key, strat.lane_budgets());
  CompiledPlan* cp = built.get();
  cache_[key] = std::move(built);
  return cp;
}

void Session::plan_only(Scheduler& strat, const std::string& key) {
  last_ = lookup_or_build(strat, key);
}

namespace {
// serialise a parsed spec back to text (plain objects of scalars / arrays)
std::string dump_json(const json::Value& x) {
  switch (x.t) {
    case json::Value::T::Null: return "null";
    case json::Value::T::Bool: return x.b ? "true" : "false";
    case json::Value::T::Int: return x.is_neg ? std::to_string(x.i) : std::to_string(x.u);
    case json::Value::T::Double: {
      char b[64];
      std::snprintf(b, sizeof b, "%.17g", x.d);
      return b;
    }
    case json::Value::T::String: return json::quote(x.s);
    case json::Value::T::Array: {
      std::string o = "[";
      for (std::size_t i = 0; i < x.a->size(); ++i) o += (i ? "," : "") + dump_json((*x.a)[i]);
      return o + "]";
    }
    case json::Value::T::Object: {
      std::string o = "{";
      for (std::size_t i = 0; i < x.o->size(); ++i)
        o += (i ? "," : "") + json::quote((*x.o)[i].first) + ":" + dump_json((*x.o)[i].second);
      return o + "}";
    }
  }
  return "null";
}
}  // namespace

std::string Session::choose(const std::string& spec, cudaStream_t stream) {
  json::Value v;
  try {
    v = json::parse(spec.empty() ? "{}" : spec);
  } catch (const std::exception& e) {
    fail(Errc::ConfigError, std::string("strategy spec: ") + e.what());
  }
  const json::Value* name = v.get("name");
  if (!name || name->t != json::Value::T::String || name->str() != "auto") return spec;
  const std::string key = spec + "|rows=" + std::to_string(rows());
  auto hit = auto_choice_.find(key);
  if (hit != auto_choice_.end()) return hit->second;
  // Calibrated form: {"name":"auto","table":[{"min_rows":R,"strategy":{...}},...]}
  // — a rows -> strategy decision table fitted offline from device timings
  // (selector.py): the entry with the largest min_rows <= rows
  // wins, no timing at run time, one cached CUDA graph per decision.
  if (const json::Value* table = v.get("table")) {
    require(table->t == json::Value::T::Array && !table->arr().empty(), Errc::ConfigError,
            "auto table must be a non-empty list");
    const json::Value* pick = nullptr;
    int64_t pick_min = -1;
    for (const json::Value& e : table->arr()) {
      const json::Value* mr = e.get("min_rows");
      const json::Value* st = e.get("strategy");
      require(mr && st && st->t == json::Value::T::Object, Errc::ConfigError,
              "auto table entries need 'min_rows' and a 'strategy' object");
      const int64_t m = mr->as_i64();
      require(m >= 0, Errc::ConfigError, "auto table: min_rows must be >= 0");
      if (m <= rows() && m > pick_min) {
        pick = st;
        pick_min = m;
      }
    }
    require(pick != nullptr, Errc::ConfigError,
            "auto table has no entry for rows=" + std::to_string(rows()) + " (add min_rows 0)");
    const std::string chosen = dump_json(*pick);
    auto_choice_[key] = chosen;
    auto_times_[key] = {};
    return chosen;
  }
  const json::Value* cands = v.get("candidates");
  require(cands && cands->t == json::Value::T::Array && !cands->arr().empty(), Errc::ConfigError,
          "auto strategy needs a non-empty 'candidates' list (or a 'table')");
  require(!dry_, Errc::EngineStopped, "auto strategy selection needs a device session");
  const int reps = v.get("reps") ? static_cast<int>(v.get("reps")->as_i64()) : 5;
  // candidates timed in interleaved rounds, median per candidate: a B200 under
  // its power cap drifts by several % within a second, so timing each
  // candidate once, back to back, let the drift pick the winner
  const int rounds = v.get("rounds") ? std::max(1, static_cast<int>(v.get("rounds")->as_i64())) : 3;
  const auto dump = dump_json;
  cudaEvent_t e0, e1;
  OPF_CUDA(cudaEventCreate(&e0));
  OPF_CUDA(cudaEventCreate(&e1));
  std::vector<std::string> specs;
  std::vector<std::unique_ptr<Scheduler>> strats;
  for (const json::Value& c : cands->arr()) {
    specs.push_back(dump(c));
    strats.push_back(make_strategy(specs.back()));
    run(*strats.back(), "builtin:" + specs.back(), stream);  // build + capture + warm-up
  }
  std::vector<std::vector<double>> per(specs.size());
  for (int r = 0; r < rounds; ++r)
    for (size_t i = 0; i < specs.size(); ++i) {
      OPF_CUDA(cudaEventRecord(e0, stream));
      for (int k = 0; k < reps; ++k) run(*strats[i], "builtin:" + specs[i], stream);
      OPF_CUDA(cudaEventRecord(e1, stream));
      OPF_CUDA(cudaEventSynchronize(e1));
      float ms = 0.0f;
      OPF_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      per[i].push_back(ms / reps);
    }
  std::vector<double> times;
  std::string best;
  double best_ms = 1e300;
  for (size_t i = 0; i < specs.size(); ++i) {
    std::vector<double> t = per[i];
    std::sort(t.begin(), t.end());
    const double med = t[t.size() / 2];
    times.push_back(med);
    if (med < best_ms) {
      best_ms = med;
      best = specs[i];
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  auto_choice_[key] = best;
  auto_times_[key] = times;
  log_info("auto strategy for rows=" + std::to_string(rows()) + ": " + best);
  return best;
}

void Session::run(Scheduler& strat, const std::string& key_in, cudaStream_t stream) {
  check_window(false);
  CompiledPlan* cp = prepare(strat, key_in, stream);
  last_ = cp;
  if (!cfg_.cuda_graph) {
    launch_plan(*cp, stream, false);
    OPF_CUDA(cudaGetLastError());
  } else {
    OPF_CUDA(cudaGraphLaunch(cp->exec, stream));
  }
  note_window(stream);
}

CompiledPlan* Session::prepare(Scheduler& strat, const std::string& key_in, cudaStream_t stream) {
  require(!dry_, Errc::EngineStopped, "dry session cannot execute");
  CompiledPlan* cp = lookup_or_build(strat, key_in);
  ensure_packed_for(*cp, stream);
  ensure_arena(cp->arena_bytes);
  warm_aux(*cp);
  if (!cfg_.cuda_graph) return cp;
  if (!cp->exec || cp->arena_base_at_capture != arena_) {
    if (cp->exec) {
      OPF_CUDA(cudaGraphExecDestroy(cp->exec));
      cp->exec = nullptr;
    }
    cudaStream_t cap;
    OPF_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    // prior work on `stream` (prepack, input uploads) must precede capture-free replay
    OPF_CUDA(cudaStreamSynchronize(stream));
    OPF_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    try {
      launch_plan(*cp, cap, true);
    } catch (...) {
      cudaGraph_t g;
      cudaStreamEndCapture(cap, &g);
      if (g) cudaGraphDestroy(g);
      cudaStreamDestroy(cap);
      throw;
    }
    cudaGraph_t graph;
    OPF_CUDA(cudaStreamEndCapture(cap, &graph));
    OPF_CUDA(cudaGraphInstantiate(&cp->exec, graph, 0));
    OPF_CUDA(cudaGraphDestroy(graph));
    OPF_CUDA(cudaStreamDestroy(cap));
    cp->arena_base_at_capture = arena_;
  }
  return cp;
}

opf_view Session::output(const std::string& name) {
  const int32_t t = g_.tensor_id(name);
  require(g_.is_output(t), Errc::ConfigError, "'" + name + "' is not a graph output");
  if (ext_[t].base) return ext_[t];
  require(last_ != nullptr, Errc::Unmaterialized, "no run yet");
  for (const auto& [tt, off] : last_->outputs)
    if (tt == t) {
      const TensorMeta& m = g_.tensors[t];
      std::vector<int64_t> shape = m.shape;
      shape[0] = rows();
      return make_view(static_cast<char*>(arena_) + off, 0, m.dtype, shape, true);
    }
  fail(Errc::Unmaterialized, "output '" + name + "' not found in last plan");
}

std::string Session::stats_json() const {
  std::string s = "{\"runs\":" + std::to_string(runs_) +
                  ",\"plan_cache_hits\":" + std::to_string(hits_) +
                  ",\"plan_cache_misses\":" + std::to_string(misses_) +
                  ",\"arena_bytes\":" + std::to_string(arena_bytes_) +
                  ",\"cached_plans\":" + std::to_string(cache_.size());
  s += ",\"auto\":[";
  bool first = true;
  for (const auto& [k, v] : auto_choice_) {
    s += std::string(first ? "" : ",") + "{\"key\":" + json::quote(k) + ",\"chosen\":" + json::quote(v);
    std::string ts = "[";
    for (std::size_t i = 0; i < auto_times_.at(k).size(); ++i) {
      char b[32];
      std::snprintf(b, sizeof b, "%s%.4f", i ? "," : "", auto_times_.at(k)[i]);
      ts += b;
    }
    s += ",\"ms\":" + ts + "]}";
    first = false;
  }
  s += "]";
  if (last_) {
    s += ",\"last\":{\"key\":" + json::quote(last_->key) +
         ",\"dispatches\":" + std::to_string(last_->dispatches.size()) +
         ",\"launches\":" + std::to_string(last_->n_launches) +
         ",\"copied_elements\":" + std::to_string(last_->copied_elements) +
         ",\"plan_arena_bytes\":" + std::to_string(last_->arena_bytes) +
         ",\"peak_live_bytes\":" + std::to_string(last_->peak_live_bytes) +
         ",\"analysis_ops\":" + std::to_string(last_->analysis_ops) +
         ",\"lanes_used\":" + std::to_string(last_->lanes_used) +
         ",\"end_live_tensors\":" + std::to_string(last_->end_live_tensors) +
         ",\"captured\":" + (last_->exec ? "true" : "false") + "}";
  }
  return s + "}";
}

std::string Session::schedule_json() const {
  require(last_ != nullptr, Errc::Unmaterialized, "no run yet");
  static const char* kinds[] = {"single", "merged", "fused"};
  std::string s = "{\"key\":" + json::quote(last_->key) + ",\"dispatches\":[";
  for (std::size_t i = 0; i < last_->dispatches.size(); ++i) {
    const PlannedDispatch& pd = last_->dispatches[i];
    if (i) s += ',';
    std::vector<std::string> labels;
    for (int32_t sg : pd.d.subgraphs) labels.push_back(p_.subgraphs[sg].label);
    s += "{\"id\":" + std::to_string(pd.d.id) + ",\"lane\":" + std::to_string(pd.d.lane) +
         ",\"kind\":\"" + kinds[static_cast<int>(pd.d.kind)] +
         "\",\"subgraphs\":" + json::int_list(pd.d.subgraphs) +
         ",\"labels\":" + json::str_list(labels) + ",\"u0\":" + std::to_string(pd.d.u0) +
         ",\"u1\":" + std::to_string(pd.d.u1) + ",\"rows\":" + std::to_string(pd.rows) +
         ",\"wait_on\":" + json::int_list(pd.wait_on) + ",\"replace_fn\":" +
         json::quote(pd.d.replace_fn) + ",\"launches\":[";
    for (std::size_t j = 0; j < pd.launches.size(); ++j) {
      const PlannedLaunch& l = pd.launches[j];
      if (j) s += ',';
      auto views = [&](const std::vector<PlannedView>& vs) {
        std::string o = "[";
        for (std::size_t k = 0; k < vs.size(); ++k) {
          static const char* src[] = {"arena", "external", "prepacked", "none"};
          if (k) o += ',';
          o += "{\"src\":\"" + std::string(src[static_cast<int>(vs[k].src)]) +
               "\",\"block_off\":" + std::to_string(vs[k].block_off) +
               ",\"tensor\":" + std::to_string(vs[k].tensor) +
               ",\"elem_offset\":" + std::to_string(vs[k].elem_offset) +
               ",\"elem_bytes\":" + std::to_string(dtype_bytes(vs[k].dtype)) +
               ",\"shape\":" + json::int_list(vs[k].shape) + "}";
        }
        return o + "]";
      };
      s += "{\"name\":" + json::quote(l.name) + ",\"op\":" + std::to_string(l.op) +
           ",\"copy\":" + (l.is_copy ? "true" : "false") + ",\"rows\":" + std::to_string(l.rows) +
           ",\"ws_off\":" + std::to_string(l.ws_off) + ",\"ws_bytes\":" + std::to_string(l.ws_bytes) +
           ",\"prepacked\":" + std::to_string(l.prepacked) +
           ",\"in\":" + views(l.in) + ",\"out\":" + views(l.out) + "}";
    }
    s += "]}";
  }
  return s + "]}";
}

std::string Session::trace_json() {
  require(last_ != nullptr, Errc::Unmaterialized, "no run yet");
  // Profiled eager replay: timing events around every dispatch on its lane
  // (OPF_TRACE_LAUNCHES=1: around every kernel launch instead — the in-situ
  // per-kernel breakdown of a step, unlike ncu's serialised cold-cache list).
  const char* per_env = std::getenv("OPF_TRACE_LAUNCHES");
  const bool per_launch = per_env && std::string(per_env) == "1";
  CompiledPlan& cp = *last_;
  struct Ev {
    cudaEvent_t b, e;
    std::string name;
    int lane;
  };
  std::vector<Ev> evs;
  std::vector<cudaEvent_t> disp_end(cp.dispatches.size());
  cudaEvent_t t0;
  OPF_CUDA(cudaEventCreate(&t0));
  OPF_CUDA(cudaDeviceSynchronize());
  OPF_CUDA(cudaEventRecord(t0, lanes_[0]));
  for (auto& l : lanes_) OPF_CUDA(cudaStreamWaitEvent(l, t0, 0));
  auto mk = [&](const std::string& name, int lane) {
    Ev e{};
    OPF_CUDA(cudaEventCreate(&e.b));
    OPF_CUDA(cudaEventCreate(&e.e));
    e.name = name;
    e.lane = lane;
    evs.push_back(e);
    return evs.size() - 1;
  };
  for (std::size_t i = 0; i < cp.dispatches.size(); ++i) {
    const PlannedDispatch& pd = cp.dispatches[i];
    cudaStream_t s = lanes_[pd.d.lane];
    for (int32_t w : pd.wait_on) OPF_CUDA(cudaStreamWaitEvent(s, disp_end[w], 0));
    std::string dname;
    for (int32_t sg : pd.d.subgraphs) dname += (dname.empty() ? "" : "+") + p_.subgraphs[sg].label;
    dname += " u" + std::to_string(pd.d.u0) + (pd.d.u1 - pd.d.u0 > 1 ? "-" + std::to_string(pd.d.u1 - 1) : "");
    std::size_t di = 0;
    if (!per_launch) {
      di = mk(dname, pd.d.lane);
      OPF_CUDA(cudaEventRecord(evs[di].b, s));
    }
    for (const PlannedLaunch& l : pd.launches) {
      std::size_t li = 0;
      if (per_launch) {
        li = mk(l.name + " u" + std::to_string(pd.d.u0), pd.d.lane);
        OPF_CUDA(cudaEventRecord(evs[li].b, s));
      }
      launch_one(l, s);
      if (per_launch) OPF_CUDA(cudaEventRecord(evs[li].e, s));
    }
    OPF_CUDA(cudaEventCreate(&disp_end[i]));
    OPF_CUDA(cudaEventRecord(disp_end[i], s));
    if (!per_launch) OPF_CUDA(cudaEventRecord(evs[di].e, s));
  }
  OPF_CUDA(cudaDeviceSynchronize());
  std::string out = "[";
  for (std::size_t i = 0; i < evs.size(); ++i) {
    float ts = 0, te = 0;
    OPF_CUDA(cudaEventElapsedTime(&ts, t0, evs[i].b));
    OPF_CUDA(cudaEventElapsedTime(&te, t0, evs[i].e));
    char buf[128];
    std::snprintf(buf, sizeof buf, ",\"ts\":%.3f,\"dur\":%.3f,\"pid\":0,\"tid\":%d}", ts * 1e3,
                  (te - ts) * 1e3, evs[i].lane);
    out += std::string(i ? "," : "") + "{\"name\":" + json::quote(evs[i].name) +
           ",\"cat\":\"" + (per_launch ? "launch" : "dispatch") + "\",\"ph\":\"X\"" + buf;
    cudaEventDestroy(evs[i].b);
    cudaEventDestroy(evs[i].e);
  }
  for (auto& e : disp_end) cudaEventDestroy(e);
  cudaEventDestroy(t0);
  return out + "]";
}

}  // namespace opflow
