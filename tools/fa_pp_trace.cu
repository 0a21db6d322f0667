// Timeline harness for the two-head prefill attention (fa_pp_kernel):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DFA_TRACE \
//        -I paper_2605_21603_b200/csrc/include -I include tools/fa_pp_trace.cu -lcuda -o /tmp/fa_pp_trace
// Prints CTA 0's first tiles: K issue, S / PV issue per head, and when each
// head's softmax got S and released P (clock64 cycles from the first event).
#include <cuda_bf16.h>

#include <cstdio>
#include <vector>

#include "../paper_2605_21603_b200/csrc/kernels/attention_fa_tc.cu"

namespace opflow {
int num_sms() { return 148; }
bool pdl_enabled() { return false; }
}  // namespace opflow

int main(int argc, char** argv) {
  const int S = 1024, seqs = argc > 1 ? atoi(argv[1]) : 8, nq = 32, nkv = 8, hd = 128;
  const int64_t rows = int64_t(S) * seqs, W = int64_t(nq + 2 * nkv) * hd;
  std::vector<__nv_bfloat16> h(rows * W);
  uint32_t x = 1;
  for (auto& v : h) {
    x = x * 1664525u + 1013904223u;
    v = __float2bfloat16(((x >> 9) & 0xffff) / 32768.0f - 1.0f);
  }
  __nv_bfloat16 *qkv, *out;
  cudaMalloc(&qkv, h.size() * 2);
  cudaMalloc(&out, rows * nq * hd * 2);
  cudaMemcpy(qkv, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  for (int it = 0; it < 3; ++it)
    if (!opflow::prefill_bf16_tcgen05(qkv, out, rows, nq, nkv, hd, S, 0.0883883f, 0, 0)) return 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  cudaEventRecord(e0);
  opflow::prefill_bf16_tcgen05(qkv, out, rows, nq, nkv, hd, S, 0.0883883f, 0, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long t[12][64];
  cudaMemcpyFromSymbol(t, opflow::g_fa_trace, sizeof(t));
  printf("kernel %.1f us (%s)\n", ms * 1e3, cudaGetErrorString(cudaGetLastError()));
  long long t0 = t[0][0];
  const int ev[] = {0, 2, 3, 4, 5, 6, 7, 8, 9};
  const char* names[] = {"K issued", "S0 issue", "S1 issue", "PV0 issue", "PV1 issue", "h0 got S", "h0 P rdy",
                         "h1 got S", "h1 P rdy"};
  printf("%4s", "n");
  for (const char* nme : names) printf(" %10s", nme);
  printf("\n");
  for (int j = 0; j < 40; ++j) {
    printf("%4d", j);
    for (int e : ev) printf(" %10lld", t[e][j] - t0);
    printf("\n");
  }
  // item boundaries: Q load issued (producer), Q landed at the MMA warp, head-0 epilogue done
  printf("%4s %10s %10s %10s\n", "item", "Q issued", "Q at MMA", "epi0 done");
  for (int j = 0; j < 8; ++j) printf("%4d %10lld %10lld %10lld\n", j, t[1][j] - t0, t[10][j] - t0, t[11][j] - t0);
  return 0;
}
