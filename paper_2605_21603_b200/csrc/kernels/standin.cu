// Stand-in operator kinds on sm_100a, bit-exact with the reference CPU kernels
// (/root/reference/proj/src/kernels_scalar.cpp:13-113):
//   * fp32 products and sums use __fmul_rn / __fadd_rn in the reference's
//     accumulation order (no FMA contraction, which the reference also avoids:
//     proj/src/CMakeLists.txt:14-15), so results match to the bit;
//   * int64 arithmetic wraps (two's complement), like the reference.
// These serve the reference's own graphs (dense_tp / moe_ep / fuse_chain) and
// the C1 toy; the Llama-shaped hot path uses the bf16 kernels in gemm_tc.cu /
// norm.cu / llama_ops.cu / attention.cu.
#include <cuda_bf16.h>

#include "opflow/device.hpp"

namespace opflow {

namespace {

__device__ __forceinline__ int64_t wrap_mul(int64_t a, int64_t b) {
  return static_cast<int64_t>(static_cast<uint64_t>(a) * static_cast<uint64_t>(b));
}
__device__ __forceinline__ int64_t wrap_add(int64_t a, int64_t b) {
  return static_cast<int64_t>(static_cast<uint64_t>(a) + static_cast<uint64_t>(b));
}

// out[r][j] = sum_k a[r][k] * w[k][j], k ascending, one rounding per mul and add.
// 64x64 output tile per CTA, 16-deep k slabs staged in shared memory, 4x4 per
// thread.  Launched for int64 (wrapping); fp32 takes matmul_exact_f32_kernel.
template <typename T>
__global__ void __launch_bounds__(256) matmul_exact_kernel(const T* __restrict__ a,
                                                           const T* __restrict__ w, T* __restrict__ out,
                                                           int64_t rows, int64_t K, int64_t N) {
  constexpr int BM = 64, BN = 64, BK = 16;
  __shared__ T As[BK][BM + 1];
  __shared__ T Ws[BK][BN];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * BM, n0 = static_cast<int64_t>(blockIdx.x) * BN;
  T acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = T(0);
  for (int64_t k0 = 0; k0 < K; k0 += BK) {
    for (int idx = threadIdx.x; idx < BM * BK; idx += 256) {
      const int r = idx / BK, c = idx % BK;
      const int64_t gr = m0 + r, gc = k0 + c;
      As[c][r] = (gr < rows && gc < K) ? a[gr * K + gc] : T(0);
    }
    for (int idx = threadIdx.x; idx < BK * BN; idx += 256) {
      const int r = idx / BN, c = idx % BN;
      const int64_t gr = k0 + r, gc = n0 + c;
      Ws[r][c] = (gr < K && gc < N) ? w[gr * N + gc] : T(0);
    }
    __syncthreads();
    const int kend = static_cast<int>(K - k0 < BK ? K - k0 : BK);
    for (int kk = 0; kk < kend; ++kk) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const T av = As[kk][ty * 4 + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const T wv = Ws[kk][tx * 4 + j];
          if constexpr (std::is_same_v<T, float>)
            acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(av, wv));
          else
            acc[i][j] = wrap_add(acc[i][j], wrap_mul(av, wv));
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t r = m0 + ty * 4 + i, c = n0 + tx * 4 + j;
      if (r < rows && c < N) out[r * N + c] = acc[i][j];
    }
}

// fp32 form of the same contraction, register-tiled: BM x BN output tile per
// CTA of 256 threads (128x128: 8x8 outputs per thread; 64x64: 4x4, for grids
// that would not fill the SMs), 8-deep k slabs double-buffered in shared
// memory (A transposed so a thread reads its rows as float4), each thread's
// rows / columns in 4-wide groups 64 apart (conflict-free 128-bit shared
// loads).  Each output still accumulates k = 0..K-1 in order with one
// __fmul_rn and one __fadd_rn per term, so it is bit-identical to
// matmul_exact_kernel (and to kernels_scalar.cpp:40-66); the next slab's global
// loads are in flight while the current one is consumed.
constexpr int kXK = 8;
template <int BM, int BN>
__global__ void __launch_bounds__(256) matmul_exact_f32_kernel(const float* __restrict__ a,
                                                               const float* __restrict__ w,
                                                               float* __restrict__ out, int64_t rows,
                                                               int64_t K, int64_t N, bool vec) {
  constexpr int TM = BM / 16, TN = BN / 16;   // outputs per thread: TM rows x TN columns
  constexpr int VA = BM * kXK / 256, VW = BN * kXK / 256;  // slab elements each thread loads
  __shared__ __align__(16) float As[2][kXK][BM];
  __shared__ __align__(16) float Ws[2][kXK][BN];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * BM, n0 = static_cast<int64_t>(blockIdx.x) * BN;
  // loader roles: A — row lr, k columns lc..lc+VA-1; W — k row wr, columns wc..wc+VW-1
  const int lr = tid / (kXK / VA), lc = (tid % (kXK / VA)) * VA;
  const int wr = tid / (BN / VW), wc = (tid % (BN / VW)) * VW;
  float ra[VA], rw[VW];
  auto fetch = [&](int64_t k0) {
    const int64_t gr = m0 + lr, gk = k0 + lc;
    if (vec && gr < rows && gk + VA <= K) {
      if constexpr (VA == 4) {
        const float4 v = *reinterpret_cast<const float4*>(a + gr * K + gk);
        ra[0] = v.x, ra[1] = v.y, ra[2] = v.z, ra[3] = v.w;
      } else {
        const float2 v = *reinterpret_cast<const float2*>(a + gr * K + gk);
        ra[0] = v.x, ra[1] = v.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < VA; ++i) ra[i] = (gr < rows && gk + i < K) ? a[gr * K + gk + i] : 0.0f;
    }
    const int64_t gwr = k0 + wr, gwc = n0 + wc;
    if (vec && gwr < K && gwc + VW <= N) {
      if constexpr (VW == 4) {
        const float4 v = *reinterpret_cast<const float4*>(w + gwr * N + gwc);
        rw[0] = v.x, rw[1] = v.y, rw[2] = v.z, rw[3] = v.w;
      } else {
        const float2 v = *reinterpret_cast<const float2*>(w + gwr * N + gwc);
        rw[0] = v.x, rw[1] = v.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < VW; ++i) rw[i] = (gwr < K && gwc + i < N) ? w[gwr * N + gwc + i] : 0.0f;
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int i = 0; i < VA; ++i) As[buf][lc + i][lr] = ra[i];
#pragma unroll
    for (int i = 0; i < VW; ++i) Ws[buf][wr][wc + i] = rw[i];
  };
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;
  const int64_t n_slabs = (K + kXK - 1) / kXK;
  fetch(0);
  stash(0);
  __syncthreads();
  for (int64_t s = 0; s < n_slabs; ++s) {
    const int buf = static_cast<int>(s & 1);
    if (s + 1 < n_slabs) fetch((s + 1) * kXK);
    const int kend = static_cast<int>(K - s * kXK < kXK ? K - s * kXK : kXK);
    for (int kk = 0; kk < kend; ++kk) {
      float av[TM], wv[TN];
#pragma unroll
      for (int g = 0; g < TM / 4; ++g) {
        const float4 v = *reinterpret_cast<const float4*>(&As[buf][kk][g * 64 + ty * 4]);
        av[4 * g] = v.x, av[4 * g + 1] = v.y, av[4 * g + 2] = v.z, av[4 * g + 3] = v.w;
      }
#pragma unroll
      for (int g = 0; g < TN / 4; ++g) {
        const float4 v = *reinterpret_cast<const float4*>(&Ws[buf][kk][g * 64 + tx * 4]);
        wv[4 * g] = v.x, wv[4 * g + 1] = v.y, wv[4 * g + 2] = v.z, wv[4 * g + 3] = v.w;
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(av[i], wv[j]));
    }
    if (s + 1 < n_slabs) stash(buf ^ 1);  // the other buffer was last read before the previous barrier
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t r = m0 + (i / 4) * 64 + ty * 4 + i % 4;
    if (r >= rows) continue;
#pragma unroll
    for (int h = 0; h < TN / 4; ++h) {
      const int64_t c = n0 + h * 64 + tx * 4;
      if (vec && c + 4 <= N) {
        *reinterpret_cast<float4*>(out + r * N + c) =
            make_float4(acc[i][h * 4], acc[i][h * 4 + 1], acc[i][h * 4 + 2], acc[i][h * 4 + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (c + j < N) out[r * N + c + j] = acc[i][h * 4 + j];
      }
    }
  }
}

template <typename T>
__global__ void add_kernel(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ o,
                           int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if constexpr (std::is_same_v<T, int64_t>)
      o[i] = wrap_add(a[i], b[i]);
    else if constexpr (std::is_same_v<T, float>)
      o[i] = __fadd_rn(a[i], b[i]);
    else
      o[i] = __float2bfloat16(__bfloat162float(a[i]) + __bfloat162float(b[i]));
  }
}

__global__ void add_bf16x8_kernel(const uint4* __restrict__ a, const uint4* __restrict__ b,
                                  uint4* __restrict__ o, int64_t n8) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint4 x = a[i], y = b[i], z;
    const __nv_bfloat162* xp = reinterpret_cast<const __nv_bfloat162*>(&x);
    const __nv_bfloat162* yp = reinterpret_cast<const __nv_bfloat162*>(&y);
    __nv_bfloat162* zp = reinterpret_cast<__nv_bfloat162*>(&z);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 fx = __bfloat1622float2(xp[k]), fy = __bfloat1622float2(yp[k]);
      zp[k] = __floats2bfloat162_rn(fx.x + fy.x, fx.y + fy.y);
    }
    o[i] = z;
  }
}

template <typename T>
__global__ void scale_kernel(const T* __restrict__ x, int64_t f, T* __restrict__ o, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if constexpr (std::is_same_v<T, int64_t>)
      o[i] = wrap_mul(x[i], f);
    else if constexpr (std::is_same_v<T, float>)
      o[i] = __fmul_rn(x[i], static_cast<float>(f));
    else
      o[i] = __float2bfloat16(__bfloat162float(x[i]) * static_cast<float>(f));
  }
}

// One warp per row.  The row is staged in shared memory with coalesced loads,
// then lane 0 runs the reference's sequential reduction; the result is
// broadcast and all lanes write the row back coalesced.
constexpr int kRowWarps = 4;
constexpr int kRowChunk = 1024;  // elements staged per pass

__global__ void row_scale_f32_kernel(const float* __restrict__ x, float* __restrict__ o,
                                     int64_t rows, int64_t cols) {
  __shared__ float buf[kRowWarps][kRowChunk];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * kRowWarps + warp;
  if (r >= rows) return;
  const float* xr = x + r * cols;
  float sumsq = 0.0f;
  for (int64_t c0 = 0; c0 < cols; c0 += kRowChunk) {
    const int n = static_cast<int>(cols - c0 < kRowChunk ? cols - c0 : kRowChunk);
    for (int i = lane; i < n; i += 32) buf[warp][i] = xr[c0 + i];
    __syncwarp();
    if (lane == 0)
      for (int i = 0; i < n; ++i) sumsq = __fadd_rn(sumsq, __fmul_rn(buf[warp][i], buf[warp][i]));
    __syncwarp();
  }
  float inv = 0.0f;
  if (lane == 0)
    inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(sumsq, static_cast<float>(cols)), 1e-6f)));
  inv = __shfl_sync(0xffffffffu, inv, 0);
  for (int64_t c = lane; c < cols; c += 32) o[r * cols + c] = __fmul_rn(xr[c], inv);
}

__global__ void row_scale_i64_kernel(const int64_t* __restrict__ x, int64_t* __restrict__ o,
                                     int64_t rows, int64_t cols) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * kRowWarps + warp;
  if (r >= rows) return;
  const int64_t* xr = x + r * cols;
  int64_t stat = 1;
  for (int64_t c = lane; c < cols; c += 32) {
    const int64_t v = xr[c];
    const int64_t mag = v < 0 ? static_cast<int64_t>(0ull - static_cast<uint64_t>(v)) : v;
    stat = mag > stat ? mag : stat;
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    const int64_t other = __shfl_xor_sync(0xffffffffu, stat, s);
    stat = other > stat ? other : stat;
  }
  for (int64_t c = lane; c < cols; c += 32) o[r * cols + c] = xr[c] / stat;
}

__global__ void row_scale_bf16_kernel(const __nv_bfloat16* __restrict__ x,
                                      __nv_bfloat16* __restrict__ o, int64_t rows, int64_t cols) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * kRowWarps + warp;
  if (r >= rows) return;
  float ss = 0.0f;
  for (int64_t c = lane; c < cols; c += 32) {
    const float v = __bfloat162float(x[r * cols + c]);
    ss += v * v;
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, s);
  const float inv = rsqrtf(ss / static_cast<float>(cols) + 1e-6f);
  for (int64_t c = lane; c < cols; c += 32)
    o[r * cols + c] = __float2bfloat16(__bfloat162float(x[r * cols + c]) * inv);
}

template <typename T>
__global__ void prefix_sum_kernel(const T* __restrict__ x, T* __restrict__ o, int64_t rows,
                                  int64_t cols) {
  __shared__ T buf[kRowWarps][kRowChunk];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * kRowWarps + warp;
  if (r >= rows) return;
  T acc = T(0);
  for (int64_t c0 = 0; c0 < cols; c0 += kRowChunk) {
    const int n = static_cast<int>(cols - c0 < kRowChunk ? cols - c0 : kRowChunk);
    for (int i = lane; i < n; i += 32) buf[warp][i] = x[r * cols + c0 + i];
    __syncwarp();
    if (lane == 0)
      for (int i = 0; i < n; ++i) {
        if constexpr (std::is_same_v<T, float>)
          acc = __fadd_rn(acc, buf[warp][i]);
        else
          acc = wrap_add(acc, buf[warp][i]);
        buf[warp][i] = acc;
      }
    __syncwarp();
    for (int i = lane; i < n; i += 32) o[r * cols + c0 + i] = buf[warp][i];
    __syncwarp();
  }
}

template <typename T>
__global__ void permute_cols_kernel(const T* __restrict__ x, T* __restrict__ o, int64_t rows,
                                    int64_t cols, const uint32_t* __restrict__ perm) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols, c = i % cols;
    o[i] = x[r * cols + perm[c]];
  }
}

// [rows, cols] -> [cols, rows] bf16 via 32x32 shared tiles (weight pre-pack).
__global__ void transpose_bf16_kernel(const __nv_bfloat16* __restrict__ src,
                                      __nv_bfloat16* __restrict__ dst, int64_t rows, int64_t cols) {
  __shared__ __nv_bfloat16 tile[32][33];
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 32, r0 = static_cast<int64_t>(blockIdx.y) * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = src[r * cols + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) dst[c * rows + r] = tile[threadIdx.x][i];
  }
}

int grid_for(int64_t n, int threads) {
  const int64_t want = (n + threads - 1) / threads;
  const int64_t cap = static_cast<int64_t>(num_sms()) * 16;
  return static_cast<int>(want < 1 ? 1 : (want > cap ? cap : want));
}

}  // namespace

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("OPF_PDL");
    return e && e[0] == '1';  // opt-in: no measurable gain under the power cap (profiles/)
  }();
  return on;
}

int num_sms() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

void k_matmul_exact(Dtype dt, const void* a, const void* w, void* out, int64_t rows, int64_t k,
                    int64_t n, cudaStream_t s) {
  if (dt == Dtype::kF32) {
    const bool vec = k % 4 == 0 && n % 4 == 0 &&
                     (reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(out)) % 16 == 0;
    const int64_t big = ((n + 127) / 128) * ((rows + 127) / 128);
    if (big >= num_sms()) {  // 128x128 tiles fill the SMs: 8x8 outputs per thread
      dim3 g(static_cast<unsigned>((n + 127) / 128), static_cast<unsigned>((rows + 127) / 128));
      matmul_exact_f32_kernel<128, 128><<<g, 256, 0, s>>>(static_cast<const float*>(a), static_cast<const float*>(w),
                                                          static_cast<float*>(out), rows, k, n, vec);
    } else {
      dim3 g(static_cast<unsigned>((n + 63) / 64), static_cast<unsigned>((rows + 63) / 64));
      matmul_exact_f32_kernel<64, 64><<<g, 256, 0, s>>>(static_cast<const float*>(a), static_cast<const float*>(w),
                                                        static_cast<float*>(out), rows, k, n, vec);
    }
    return;
  }
  dim3 grid(static_cast<unsigned>((n + 63) / 64), static_cast<unsigned>((rows + 63) / 64));
  matmul_exact_kernel<int64_t><<<grid, 256, 0, s>>>(static_cast<const int64_t*>(a),
                                                      static_cast<const int64_t*>(w),
                                                      static_cast<int64_t*>(out), rows, k, n);
}

void k_add(Dtype dt, const void* a, const void* b, void* out, int64_t n, cudaStream_t s) {
  if (dt == Dtype::kBF16 && n % 8 == 0 && (reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) |
                                            reinterpret_cast<uintptr_t>(out)) % 16 == 0) {
    add_bf16x8_kernel<<<grid_for(n / 8, 256), 256, 0, s>>>(
        static_cast<const uint4*>(a), static_cast<const uint4*>(b), static_cast<uint4*>(out), n / 8);
    return;
  }
  const int g = grid_for(n, 256);
  if (dt == Dtype::kF32)
    add_kernel<float><<<g, 256, 0, s>>>(static_cast<const float*>(a), static_cast<const float*>(b),
                                        static_cast<float*>(out), n);
  else if (dt == Dtype::kI64)
    add_kernel<int64_t><<<g, 256, 0, s>>>(static_cast<const int64_t*>(a),
                                          static_cast<const int64_t*>(b),
                                          static_cast<int64_t*>(out), n);
  else
    add_kernel<__nv_bfloat16><<<g, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(a),
                                                static_cast<const __nv_bfloat16*>(b),
                                                static_cast<__nv_bfloat16*>(out), n);
}

void k_scale(Dtype dt, const void* x, int64_t f, void* out, int64_t n, cudaStream_t s) {
  const int g = grid_for(n, 256);
  if (dt == Dtype::kF32)
    scale_kernel<float><<<g, 256, 0, s>>>(static_cast<const float*>(x), f, static_cast<float*>(out), n);
  else if (dt == Dtype::kI64)
    scale_kernel<int64_t><<<g, 256, 0, s>>>(static_cast<const int64_t*>(x), f,
                                            static_cast<int64_t*>(out), n);
  else
    scale_kernel<__nv_bfloat16><<<g, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(x), f,
                                                  static_cast<__nv_bfloat16*>(out), n);
}

void k_row_scale(Dtype dt, const void* x, void* out, int64_t rows, int64_t cols, cudaStream_t s) {
  const unsigned g = static_cast<unsigned>((rows + kRowWarps - 1) / kRowWarps);
  if (dt == Dtype::kF32)
    row_scale_f32_kernel<<<g, 32 * kRowWarps, 0, s>>>(static_cast<const float*>(x),
                                                      static_cast<float*>(out), rows, cols);
  else if (dt == Dtype::kI64)
    row_scale_i64_kernel<<<g, 32 * kRowWarps, 0, s>>>(static_cast<const int64_t*>(x),
                                                      static_cast<int64_t*>(out), rows, cols);
  else
    row_scale_bf16_kernel<<<g, 32 * kRowWarps, 0, s>>>(static_cast<const __nv_bfloat16*>(x),
                                                       static_cast<__nv_bfloat16*>(out), rows, cols);
}

void k_prefix_sum(Dtype dt, const void* x, void* out, int64_t rows, int64_t cols, cudaStream_t s) {
  const unsigned g = static_cast<unsigned>((rows + kRowWarps - 1) / kRowWarps);
  if (dt == Dtype::kF32)
    prefix_sum_kernel<float><<<g, 32 * kRowWarps, 0, s>>>(static_cast<const float*>(x),
                                                          static_cast<float*>(out), rows, cols);
  else
    prefix_sum_kernel<int64_t><<<g, 32 * kRowWarps, 0, s>>>(static_cast<const int64_t*>(x),
                                                            static_cast<int64_t*>(out), rows, cols);
}

void k_permute_cols(Dtype dt, const void* x, void* out, int64_t rows, int64_t cols,
                    const uint32_t* perm, cudaStream_t s) {
  const int g = grid_for(rows * cols, 256);
  if (dt == Dtype::kF32)
    permute_cols_kernel<float><<<g, 256, 0, s>>>(static_cast<const float*>(x),
                                                 static_cast<float*>(out), rows, cols, perm);
  else if (dt == Dtype::kI64)
    permute_cols_kernel<int64_t><<<g, 256, 0, s>>>(static_cast<const int64_t*>(x),
                                                   static_cast<int64_t*>(out), rows, cols, perm);
  else
    permute_cols_kernel<__nv_bfloat16><<<g, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(x),
                                                         static_cast<__nv_bfloat16*>(out), rows,
                                                         cols, perm);
}

void k_copy_rows(const void* src, void* dst, int64_t bytes, cudaStream_t s) {
  OPF_CUDA(cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), cudaMemcpyDeviceToDevice, s));
}

void k_transpose_bf16(const void* src, void* dst, int64_t rows, int64_t cols, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((rows + 31) / 32));
  transpose_bf16_kernel<<<grid, dim3(32, 8), 0, s>>>(static_cast<const __nv_bfloat16*>(src),
                                                     static_cast<__nv_bfloat16*>(dst), rows, cols);
}

}  // namespace opflow
