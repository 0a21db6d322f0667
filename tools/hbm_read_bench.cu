// Pure-read HBM bandwidth probe (the decode-attention ceiling): every CTA
// streams a disjoint slice with 16-byte non-caching loads, N loads in flight
// per thread; the result is folded into one int so nothing is dead code.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hbm_read_bench tools/hbm_read_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int U>
__global__ void read_kernel(const uint4* __restrict__ p, size_t n, unsigned* out) {
  unsigned acc = 0;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x * U;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x * U + threadIdx.x; i < n; i += stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t j = i + static_cast<size_t>(u) * blockDim.x;
      v[u] = j < n ? __ldcs(p + j) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) atomicAdd(out, acc);
}

int main() {
  const size_t bytes = size_t(8) << 30;
  uint4* p;
  unsigned* out;
  cudaMalloc(&p, bytes);
  cudaMalloc(&out, 4);
  cudaMemset(p, 1, bytes);
  const size_t n = bytes / 16;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int ctas_per_sm : {1, 2, 4, 8}) {
    for (int threads : {256, 512, 1024}) {
      if (ctas_per_sm * threads > 2048) continue;
      const int grid = sms * ctas_per_sm;
      read_kernel<8><<<grid, threads>>>(p, n, out);
      cudaEventRecord(a);
      for (int r = 0; r < 5; ++r) read_kernel<8><<<grid, threads>>>(p, n, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("ctas/SM %d threads %4d: %.1f GB/s\n", ctas_per_sm, threads, 5.0 * bytes / (ms / 1e3) / 1e9);
    }
  }
  // SM-count scaling at the best shape (decode overlap: HBM share per SM)
  for (int used : {148, 124, 108, 92, 74, 48}) {
    if (used > sms) continue;
    read_kernel<8><<<used * 2, 1024>>>(p, n, out);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) read_kernel<8><<<used * 2, 1024>>>(p, n, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("SMs %3d (2 x 1024 thr): %.1f GB/s\n", used, 5.0 * bytes / (ms / 1e3) / 1e9);
  }
  return 0;
}
