// Reference-side program: an EXTERNAL device operator registered through the
// operator registry (opf_register_op via the bridge; the reference's
// CustomRegistry::fns[name] = fn, eval.hpp:19-28), declared as a Custom op in
// a reference GraphDescription, isolated by ByFunc(custom_name)
// (partition.cpp:161-162) and run by the backend under a 2-nano-batch split.
//
//   ext_op <in.bin> <out.bin> <desc.json>
// in.bin: x [R,H] f32 then w [H,H] f32 (R=256, H=256); writes the output
// [R,H] f32 and the description it ran, which tests/test_bridge.py evaluates
// with the reference's eval_reference + an oracle CustomFn of the same op.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "opflow/graph.hpp"
#include "opflow_b200_bridge.hpp"

using namespace opflow;

namespace {
constexpr int64_t R = 256, H = 256;
int g_calls = 0;  // host-side invocations (each nano-batch's launch, at capture)

__global__ void softcap_kernel(const float* x, float* y, int64_t n, float cap) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    y[i] = cap * tanhf(x[i] / cap);
}

float param(const opf_op_ctx* c, const char* name, float dflt) {
  for (int i = 0; i < c->n_params; ++i)
    if (std::string(c->param_names[i]) == name) return float(c->param_values[i]);
  return dflt;
}

// The registered kernel entry: outputs are caller-owned views (nano-batch row
// slices of the engine's arena), async on the given stream, no allocation.
opf_status softcap(const opf_op_ctx* c, const opf_view* in, int32_t n_in, opf_view* out, int32_t n_out,
                   int64_t rows, void* stream) {
  if (n_in != 1 || n_out != 1 || in[0].dtype != OPF_F32) return int32_t(Errc::SignatureMismatch) + 1;
  ++g_calls;
  const int64_t n = rows * in[0].shape[1];
  const float* x = static_cast<const float*>(in[0].base) + in[0].elem_offset;
  float* y = static_cast<float*>(out[0].base) + out[0].elem_offset;
  softcap_kernel<<<int((n + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(x, y, n, param(c, "cap", 30.f));
  return cudaGetLastError() == cudaSuccess ? 0 : int32_t(Errc::SchedulerError) + 1;
}

opf_view view(void* p, int64_t r, int64_t c, bool batched) {
  opf_view v{};
  v.base = p;
  v.dtype = OPF_F32;
  v.rank = 2;
  v.shape[0] = r;
  v.shape[1] = c;
  v.batched = batched;
  return v;
}
}  // namespace

int main(int argc, char** argv) {
  if (argc != 4) return 2;
  b200::register_op("softcap", softcap, ResourceClass::kMemory, 1, 1);

  GraphDescription d;
  d.tensors = {{"x", {R, H}, BatchSemantics::kBatched, Dtype::kF32, TensorRole::kGraphInput},
               {"w", {H, H}, BatchSemantics::kReplicated, Dtype::kF32, TensorRole::kWeight},
               {"mm", {R, H}, BatchSemantics::kBatched, Dtype::kF32, TensorRole::kIntermediate},
               {"capped", {R, H}, BatchSemantics::kBatched, Dtype::kF32, TensorRole::kIntermediate},
               {"y", {R, H}, BatchSemantics::kBatched, Dtype::kF32, TensorRole::kGraphOutput}};
  OpDecl mm{"blk.proj", OperatorKind::kMatMul, {"x", "w"}, {"mm"}};
  mm.module_path = "blk.proj";
  OpDecl cap{"blk.cap", OperatorKind::kCustom, {"mm"}, {"capped"}};
  cap.module_path = "blk.cap";
  cap.attrs.custom_name = "softcap";
  OpDecl norm{"blk.norm", OperatorKind::kRowScale, {"capped"}, {"y"}};
  norm.module_path = "blk.norm";
  d.operators = {mm, cap, norm};
  const std::string desc = b200::to_json(d, {{"blk.cap", {{"cap", 2.0}}}});

  b200::Graph g = b200::build_graph(desc);
  b200::Plan p = b200::partition(g, {PartitionRule::by_func("softcap")});
  std::vector<float> host(R * H + H * H);
  {
    std::ifstream f(argv[1], std::ios::binary);
    f.read(reinterpret_cast<char*>(host.data()), std::streamsize(host.size() * sizeof(float)));
    if (!f) return 3;
  }
  float *x, *w, *y;
  cudaMalloc(&x, R * H * sizeof(float));
  cudaMalloc(&w, H * H * sizeof(float));
  cudaMalloc(&y, R * H * sizeof(float));
  cudaMemcpy(x, host.data(), R * H * sizeof(float), cudaMemcpyHostToDevice);
  cudaMemcpy(w, host.data() + R * H, H * H * sizeof(float), cudaMemcpyHostToDevice);
  b200::Session s = b200::make_session(g, p, "{\"lanes\":2}");
  b200::bind(s, "x", view(x, R, H, true));
  b200::bind(s, "w", view(w, H, H, false));
  b200::bind(s, "y", view(y, R, H, true));
  const std::string strat = "{\"name\":\"split_overlap\",\"n_microbatches\":2,\"lane_mode\":\"ubatch\"}";
  for (int i = 0; i < 3; ++i) b200::run(s, strat, nullptr);  // capture once, replay
  b200::synchronize(s);
  cudaDeviceSynchronize();
  std::vector<float> out(R * H);
  cudaMemcpy(out.data(), y, out.size() * sizeof(float), cudaMemcpyDeviceToHost);
  std::ofstream(argv[2], std::ios::binary).write(reinterpret_cast<const char*>(out.data()),
                                                 std::streamsize(out.size() * sizeof(float)));
  std::ofstream(argv[3]) << desc;
  char* stats = nullptr;
  b200::check(opf_session_stats(s.h, &stats));
  std::printf("{\"calls\":%d,\"plan\":%s,\"stats\":%s}\n", g_calls, p.dump().c_str(), b200::take(stats).c_str());
  return 0;
}
