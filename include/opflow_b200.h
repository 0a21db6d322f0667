/*
 * opflow_b200.h — C-ABI of the B200-native DynaFlow execution backend.
 *
 * Plain pointers and sizes only (no torch / C++ types).  Every function
 * returns an opf_status: 0 = OK, otherwise (opflow::Errc ordinal + 1), the
 * reference's error taxonomy (/root/reference/proj/include/opflow/common.hpp:12-46);
 * opf_last_error() returns the thread-local message of the last failure.
 * Description documents (graphs, rules, strategies) are UTF-8 JSON (SPEC.md:131,
 * "Graph description format is a declarative JSON document").
 *
 * Reference interfaces each group replaces (file:line under /root/reference):
 *   opf_graph_*      build_graph / GraphDescription     proj/include/opflow/graph.hpp:79-112
 *   opf_partition*   partition / validate_plan / finalize_plan
 *                                                       proj/include/opflow/partition.hpp:58-70
 *   opf_builder_json dense_tp_graph / moe_ep_graph / fuse_chain_graph
 *                                                       proj/include/opflow/builders.hpp:26-38
 *   opf_launch       eval_op_into (per-op boundary, outputs are caller-owned,
 *                    possibly views)                    proj/include/opflow/eval.hpp:32-36
 *   opf_register_op  CustomRegistry / CustomFn          proj/include/opflow/eval.hpp:19-28
 *   opf_view_rows    TensorValue::view_rows / split_rows proj/src/tensor.cpp:23-30,67-85
 *   opf_alltoall_permutation  alltoall_permutation      proj/include/opflow/eval.hpp:44
 *   opf_session_* / opf_sched_*  the SPEC-only sched_api + engine + dataflow_mem
 *                    (split / get_ready_ops / execute, run_scheduler, CompiledPlan cache,
 *                    Algorithm 1)
 */
#ifndef OPFLOW_B200_H_
#define OPFLOW_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t opf_status;

enum opf_dtype { OPF_I64 = 0, OPF_F32 = 1, OPF_BF16 = 2 };
enum opf_resource_class { OPF_COMPUTE = 0, OPF_MEMORY = 1, OPF_NETWORK = 2 };
enum opf_kind {
  OPF_MATMUL = 0, OPF_ELEMADD, OPF_ROWSCALE, OPF_ALLREDUCE, OPF_ALLTOALL, OPF_ATTENTION, OPF_CUSTOM
};

/* A (possibly row-sliced) device tensor: element (r, c...) lives at
 * base + (elem_offset + r*row_elems + ...) * dtype_bytes.  Mirrors
 * TensorValue{storage, offset, shape} (proj/include/opflow/tensor.hpp:84-113). */
typedef struct opf_view {
  void* base;
  int64_t elem_offset;
  int32_t dtype;   /* opf_dtype */
  int32_t rank;    /* 1..4 */
  int64_t shape[4];
  int32_t batched; /* 1 = Batched (dim 0 splittable), 0 = Replicated */
  int32_t _pad;
} opf_view;

/* Per-launch context handed to a device op (built-in or registered). */
typedef struct opf_op_ctx {
  const char* op_name;
  int32_t kind;            /* opf_kind */
  const char* custom_name; /* registry key for Custom / fused ops */
  int64_t world_size;
  uint64_t seed;
  int32_t n_params;
  const char* const* param_names;
  const double* param_values;
  int32_t max_ctas;        /* SM budget for this launch (0 = whole GPU) */
  int32_t _pad;
  void* comm;              /* opf_comm* when the session is tensor-parallel, else NULL */
  const void* aux;         /* op-private device data prepared at plan build (may be NULL) */
  void* workspace;         /* arena scratch, workspace_bytes long */
  size_t workspace_bytes;
} opf_op_ctx;

/* Device kernel entry point: async on `stream` (a cudaStream_t), never
 * allocates, outputs are caller-owned views (the zero-copy redirection hook). */
typedef opf_status (*opf_kernel_fn)(const opf_op_ctx* ctx, const opf_view* in, int32_t n_in,
                                    opf_view* out, int32_t n_out, int64_t rows, void* stream);

/* ---------------------------------------------------------------- errors */
const char* opf_last_error(void);
const char* opf_errc_name(opf_status s);
const char* opf_version(void);

/* ---------------------------------------------------------------- frontend */
typedef struct opf_graph opf_graph;
typedef struct opf_plan opf_plan;

opf_status opf_graph_build(const char* description_json, opf_graph** out);
void opf_graph_free(opf_graph* g);
/* Canonical dump (op order, tensor wiring, role lists) — caller frees with opf_free_string. */
opf_status opf_graph_dump(const opf_graph* g, char** json_out);
opf_status opf_graph_tensor_id(const opf_graph* g, const char* name, int32_t* id_out);

opf_status opf_partition(const opf_graph* g, const char* rules_json, opf_plan** out);
/* Hand-assembled plan ({"subgraphs":[{"ops":[..],"label":..}]}) + finalize_plan. */
opf_status opf_plan_from_json(const opf_graph* g, const char* plan_json, opf_plan** out);
opf_status opf_validate_plan(const opf_plan* p, const opf_graph* g);
opf_status opf_plan_dump(const opf_plan* p, char** json_out);
void opf_plan_free(opf_plan* p);

/* Builders: name in {dense_tp, moe_ep, fuse_chain, llama, toy_decoder, llama_decode};
 * params_json e.g. {"layers":2,"batch":1024,"hidden":512,"dtype":"f32","costs":{...}}. */
opf_status opf_builder_json(const char* name, const char* params_json, char** json_out);
void opf_free_string(char* s);

/* AllToAll column permutation (mt19937_64 + std::shuffle, libstdc++). */
opf_status opf_alltoall_permutation(uint64_t seed, uint32_t cols, uint32_t* perm_out);

/* ---------------------------------------------------------------- device ops */
opf_status opf_register_op(const char* name, opf_kernel_fn fn, int32_t resource_class,
                           int32_t n_in, int32_t n_out);
opf_status opf_has_op(const char* name, int32_t* present);
/* eval_op_into on the device: op_json = one OpDecl object ({"kind":..,"attrs":{..}}). */
opf_status opf_launch(const char* op_json, const opf_view* in, int32_t n_in, opf_view* out,
                      int32_t n_out, int64_t rows, void* stream);
opf_status opf_view_rows(const opf_view* v, int64_t row_off, int64_t nrows, opf_view* out);
/* K splits the tcgen05 GEMM takes for an (m, n, k) MatMul on max_ctas SMs
 * (0 = whole GPU) when the engine provides its workspace; 1 = no split. */
int32_t opf_gemm_splits(int64_t m, int64_t n, int64_t k, int32_t max_ctas);
/* opf_launch with a communicator (TP collectives / fused comm ops) and an SM budget. */
typedef struct opf_comm opf_comm;
opf_status opf_launch_comm(const char* op_json, const opf_view* in, int32_t n_in, opf_view* out,
                           int32_t n_out, int64_t rows, opf_comm* comm, int32_t max_ctas,
                           void* stream);

/* ---------------------------------------------------------------- paged KV cache */
/* Per-layer K / V page pools (bf16; layout 0 NHD [pages, page, kv, hd], 1 HND
 * [pages, kv, page, hd]) with a free-list page allocator.  dry = 1: host logic
 * only (no device pools).  Slots (page * page_size + offset) feed the kv_write
 * op; block tables feed attn_decode. */
typedef struct opf_kvcache opf_kvcache;
opf_status opf_kv_create(int32_t layers, int64_t pages, int32_t page_size, int32_t kv_heads, int32_t head_dim,
                         int32_t layout, int32_t device, int32_t dry, opf_kvcache** out);
void opf_kv_free(opf_kvcache* c);
opf_status opf_kv_cache_ptr(opf_kvcache* c, int32_t layer, int32_t which, void** out);
opf_status opf_kv_append(opf_kvcache* c, const int64_t* seq_ids, const int32_t* n_new, int32_t n,
                         int64_t* slots_out, int64_t* positions_out);
opf_status opf_kv_release(opf_kvcache* c, int64_t seq_id);
opf_status opf_kv_block_table(opf_kvcache* c, const int64_t* seq_ids, int32_t n, int64_t max_pages,
                              int64_t* table_out, int64_t* lens_out);
opf_status opf_kv_stats(opf_kvcache* c, int64_t* free_pages, int64_t* sequences);

/* ---------------------------------------------------------------- comm (TP/EP) */
typedef struct opf_comm opf_comm;
/* NCCL unique id is 128 bytes; exchange it with any out-of-band channel. */
opf_status opf_comm_unique_id(uint8_t id_out[128]);
opf_status opf_comm_init(const uint8_t id[128], int32_t world, int32_t rank, int32_t device,
                         opf_comm** out);
/* Peer-window-only communicator (no NCCL): every collective runs over the
 * CUDA-IPC window (opf_comm_window_alloc / _open), at any message size.  For
 * ranks that cannot form an NCCL communicator (two processes sharing one GPU)
 * or that want NCCL-free collectives. */
opf_status opf_comm_init_peer(int32_t world, int32_t rank, int32_t device, opf_comm** out);
void opf_comm_free(opf_comm* c);
/* Symmetric peer window for the fused all-reduce+RMSNorm kernel: allocate my
 * window (returns its 64-byte CUDA-IPC handle), exchange handles out of band,
 * then open all peers' windows (handles: world x 64 bytes, rank order). */
opf_status opf_comm_window_alloc(opf_comm* c, size_t stage_bytes, uint8_t ipc_handle_out[64]);
opf_status opf_comm_window_open(opf_comm* c, const uint8_t* handles);
/* `world` virtual ranks sharing one device (tests of the peer-memory protocol). */
opf_status opf_comm_create_virtual(int32_t world, int32_t device, size_t stage_bytes, opf_comm** outs);
opf_status opf_comm_window_error(opf_comm* c, uint32_t* err);
/* Test hook: set every barrier epoch / flag / publish epoch of my window to
 * `value` (all ranks the same, before any collective) — e.g. near 2^32 to
 * exercise the wrap-safe barrier comparisons. */
opf_status opf_comm_window_set_epochs(opf_comm* c, uint32_t value);
/* Fused GEMM -> all-reduce calls that ran the peer-memory push protocol on
 * this rank (matmul_allreduce_add_rmsnorm; 0 = every call took the fallback). */
opf_status opf_comm_push_calls(opf_comm* c, uint32_t* calls);

/* ---------------------------------------------------------------- sessions */
typedef struct opf_session opf_session;
typedef struct opf_sched_ctx opf_sched_ctx;

/* config_json: {"lanes":3,"prealloc":true,"cuda_graph":true,"device":0,
 *               "gemm_sm_budget":0, "overlap_sm_reserve":0} */
opf_status opf_session_create(const opf_graph* g, const opf_plan* p, const char* config_json,
                              opf_comm* comm, opf_session** out);
void opf_session_free(opf_session* s);

/* Symmetric arena for peer-memory (expert-parallel) ops: every rank runs the
 * same plans, so a tensor sits at the same arena offset on every rank.
 * opf_session_arena_export allocates (at least min_bytes) and pins the arena
 * (later plans must fit) and returns its CUDA IPC handle (NULL: skip);
 * opf_session_arena_open maps all peers' handles ([world][64] bytes) into the
 * session's communicator; opf_session_arena_link_local wires `world` sessions
 * of ONE process (virtual ranks on one device) without IPC.  No reference
 * counterpart: the reference's AllToAll is a single-process column
 * permutation (/root/reference/proj/src/eval.cpp:71-80). */
opf_status opf_session_arena_export(opf_session* s, int64_t min_bytes, uint8_t ipc_handle_out[64]);
opf_status opf_session_arena_open(opf_session* s, const uint8_t* handles);
opf_status opf_session_arena_link_local(opf_session* const* sessions, int32_t world, int64_t min_bytes);
/* Bind an external tensor (GraphInput / Weight, or a GraphOutput destination)
 * to caller-owned device memory. */
opf_status opf_session_bind(opf_session* s, const char* tensor, const opf_view* v);
/* Run one forward under a built-in strategy spec
 * ({"name":"sequential"|"split_overlap"|"dbo"|"fuse_norm_comm"|"nanoflow", ...}).
 * Record → Algorithm-1 plan → CUDA-graph capture on a cache miss, replay on a hit. */
opf_status opf_session_run(opf_session* s, const char* strategy_json, void* stream);
/* Plan, prepack and capture `strategy` for the bound row count without
 * launching (virtual peer ranks on one device prepare every rank first). */
opf_status opf_session_prepare(opf_session* s, const char* strategy, void* stream);
/* User-programmable strategy: `schedule` is called with a scheduling context
 * on which it calls opf_sched_split / opf_sched_ready / opf_sched_execute. */
typedef opf_status (*opf_schedule_fn)(opf_sched_ctx* ctx, void* user);
opf_status opf_session_run_custom(opf_session* s, const char* cache_key, opf_schedule_fn fn,
                                  void* user, void* stream);
/* Wait for the last run and fail with SchedulerError if any peer-window
 * barrier of the runs so far timed out (a peer never arrived; the outputs are
 * invalid).  opf_session_run also raises it for earlier runs it finds done. */
opf_status opf_session_check(opf_session* s);
opf_status opf_session_output(opf_session* s, const char* tensor, opf_view* out);
/* Metrics JSON: plan-cache hits/misses, analysis ops, dispatches, launches,
 * copied elements, arena bytes, last-run trace summary. */
opf_status opf_session_stats(opf_session* s, char** json_out);
/* Trace Event JSON of the last recorded schedule (SPEC.md:455 format). */
opf_status opf_session_trace(opf_session* s, char** json_out);
/* Resolved schedule of the last run (dispatch list + buffer plan) as JSON. */
opf_status opf_session_schedule_dump(opf_session* s, char** json_out);

/* Device-free planning: run a strategy against the scheduling state machine,
 * compile the Algorithm-1 memory plan / lane events, and dump the resolved
 * schedule and stats without a GPU (`repeats` > 1 exercises the plan cache). */
opf_status opf_dry_run(const opf_graph* g, const opf_plan* p, const char* config_json,
                       const char* strategy_json, int64_t rows, int32_t repeats,
                       char** schedule_json, char** stats_json);
opf_status opf_dry_run_custom(const opf_graph* g, const opf_plan* p, const char* config_json,
                              const char* cache_key, opf_schedule_fn fn, void* user, int64_t rows,
                              char** schedule_json, char** stats_json);

typedef struct opf_handle {
  int32_t subgraph;
  int32_t ubatch;
  int32_t topo_index;
} opf_handle;

opf_status opf_sched_split(opf_sched_ctx* c, const int64_t* sizes, int32_t n);
opf_status opf_sched_ready(opf_sched_ctx* c, int32_t ubatch, opf_handle* out, int32_t cap,
                           int32_t* n_out);
opf_status opf_sched_handle(opf_sched_ctx* c, int32_t subgraph, int32_t ubatch, opf_handle* out);
opf_status opf_sched_execute(opf_sched_ctx* c, const opf_handle* hs, int32_t n, int32_t lane,
                             const char* replace_fn);
opf_status opf_sched_rows(opf_sched_ctx* c, int64_t* rows);
opf_status opf_sched_num_subgraphs(opf_sched_ctx* c, int32_t* n);
opf_status opf_sched_label(opf_sched_ctx* c, int32_t subgraph, char* buf, int32_t cap);
opf_status opf_sched_unfinished(opf_sched_ctx* c, int32_t* n);

#ifdef __cplusplus
}
#endif
#endif /* OPFLOW_B200_H_ */
