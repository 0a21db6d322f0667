// Per-SM throughput of the softmax building blocks on this GPU (cycles per
// warp-instruction): ex2.approx (MUFU), cvt.rn.bf16x2.f32 (F2FP), FFMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mufu_bench.cu -o tools/mufu_bench.bin
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>

template <int OP>
__global__ void k(float* out, long long* cyc, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f - 0.5f;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      } else if (OP == 1) {
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 1) & 7]));
        acc += r;
        a[i] += 1e-7f;
      } else {
        asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a[i]));
      }
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
}

template <int OP>
void run(const char* name, int warps) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  k<OP><<<148, warps * 32>>>(out, cyc, iters);
  k<OP><<<148, warps * 32>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double warp_instr_per_smsp = double(iters) * 8 * warps / 4;
  printf("%-8s warps/SM %2d: %.2f cycles per warp-instruction per SMSP (%.1f lanes/clk/SM)\n", name, warps,
         c / warp_instr_per_smsp, 128.0 / (c / warp_instr_per_smsp));
}

int main() {
  for (int w : {4, 8, 16, 32}) run<0>("ex2", w);
  for (int w : {4, 8, 16, 32}) run<1>("f2fp", w);
  for (int w : {4, 16}) run<2>("ffma", w);
  return 0;
}
