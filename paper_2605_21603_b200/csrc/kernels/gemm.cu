// bf16 GEMM for the QKV / O / gate_up / down projections (the only dense
// contractions of the Llama layer):  C[M,N] = A[M,K] * Bt[N,K]^T, fp32
// accumulation, bf16 out.  A = activations (row-major), Bt = the weight
// pre-packed K-major at bind time (the reference MatMul weight is [K,N],
// /root/reference/proj/src/kernels_scalar.cpp:40-66).
//
// tcgen05 path (sm_100a), one CTA per SM, persistent over output tiles:
//   warp 0      TMA producer: A 128x64 and B 256x64 bf16 tiles (128B swizzle)
//               into a 4-stage shared-memory ring (48 KB / stage)
//   warp 1      MMA issuer: one elected thread issues tcgen05.mma
//               (M=128, N=256, K=16, kind::f16) into a double-buffered TMEM
//               accumulator (2 x 256 fp32 columns = all 512 TMEM columns)
//   warps 2..5  epilogue: tcgen05.ld 32x32b -> bf16 -> swizzled smem -> TMA
//               store; each warp owns 32 accumulator lanes (rows)
// Tiles are rasterised in groups of 16 M-blocks so concurrently resident CTAs
// share A and B tiles through L2.  `max_ctas` caps the grid (SM partitioning
// when the GEMM overlaps another stream).
//
// gemm_bf16_simt is a plain CUDA-core kernel kept as the numerics cross-check
// and for direct opf_launch calls on un-packed [K,N] weights.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <mutex>

#include "opflow/device.hpp"

namespace opflow {

namespace {

// ------------------------------------------------------------------ SIMT reference
__global__ void __launch_bounds__(256) gemm_simt_kernel(const __nv_bfloat16* __restrict__ A,
                                                        const __nv_bfloat16* __restrict__ B,
                                                        __nv_bfloat16* __restrict__ C, int64_t M,
                                                        int64_t N, int64_t K, int64_t lda,
                                                        int64_t ldc, bool b_kn) {
  constexpr int BM = 64, BN = 64, BK = 16;
  __shared__ float As[BK][BM + 1];
  __shared__ float Bs[BK][BN + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * BM, n0 = static_cast<int64_t>(blockIdx.x) * BN;
  float acc[4][4] = {};
  for (int64_t k0 = 0; k0 < K; k0 += BK) {
    for (int i = threadIdx.x; i < BM * BK; i += 256) {
      const int r = i / BK, c = i % BK;
      As[c][r] = (m0 + r < M && k0 + c < K) ? __bfloat162float(A[(m0 + r) * lda + k0 + c]) : 0.0f;
    }
    for (int i = threadIdx.x; i < BN * BK; i += 256) {
      const int n = i / BK, c = i % BK;
      float v = 0.0f;
      if (n0 + n < N && k0 + c < K)
        v = __bfloat162float(b_kn ? B[(k0 + c) * N + n0 + n] : B[(n0 + n) * K + k0 + c]);
      Bs[c][n] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += As[kk][ty * 4 + i] * Bs[kk][tx * 4 + j];
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t r = m0 + ty * 4 + i, c = n0 + tx * 4 + j;
      if (r < M && c < N) C[r * ldc + c] = __float2bfloat16(acc[i][j]);
    }
}

// ------------------------------------------------------------------ tcgen05 path
constexpr int BM = 128, BN = 256, BK = 64;
// EPI 2 (RoPE epilogue): a 256-column tile holds two 128-wide heads.
// EPI 4 (residual add + RMSNorm statistics): out = x + A B^T (the add_rmsnorm
// residual output) and this tile's per-row sum of squares of the rounded
// result in ssq[row * ssq_ld + n_tile] (one writer per entry: deterministic).
struct RopeArgs {
  const int64_t* pos;
  int rot_heads;
  float log2_theta;
  const __nv_bfloat16* resid = nullptr;  // EPI 4: x [M, N]
  float* ssq = nullptr;                  // EPI 4: [M, ssq_ld] partial sums of squares
  int64_t ssq_ld = 0;                    // EPI 4: N / 256 (column tiles)
  int64_t resid_ld = 0;                  // EPI 4: row stride of x (= N)
};
constexpr int kStages = 4;
constexpr int kAccStages = 2;
constexpr int kEpiWarps = 4;
constexpr int kThreads = 64 + kEpiWarps * 32;  // TMA warp, MMA warp, 4 epilogue warps
constexpr uint32_t kABytes = BM * BK * 2;      // 16 KB
constexpr uint32_t kBBytes = BN * BK * 2;      // 32 KB
constexpr uint32_t kStageBytes = kABytes + kBBytes;
constexpr uint32_t kEpiBytes = 32 * 128;       // one warp's 32 rows x 64 cols bf16 (swizzled)
constexpr uint32_t kSmemBytes = 1024 /*align slack*/ + kStages * kStageBytes +
                                kEpiWarps * 2 * kEpiBytes + 256 /*barriers*/;
constexpr int kGroupM = 16;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int32_t c0,
                                             int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}

// K-major, 128-byte swizzle UMMA shared-memory descriptor (sm_100 format:
// start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46), version=1 [46,48),
// layout SWIZZLE_128B=2 [61,64)).  Rows are 128 B, 8-row atoms are 1024 B apart.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;             // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;     // SBO
  d |= static_cast<uint64_t>(1) << 46;             // descriptor version
  d |= static_cast<uint64_t>(2) << 61;             // SWIZZLE_128B
  return d;
}

// kind::f16 instruction descriptor: D=f32, A=B=bf16, K-major both, M=128, N=256.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
                            (static_cast<uint32_t>(BM >> 4) << 24);

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(kIdesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

// SiLU(g) * u with the fast reciprocal (MUFU.RCP + FMUL; <= 2 ulp): the IEEE
// division is a ~15-instruction FCHK / Newton sequence per element, issued by
// the epilogue warps beside the producer and MMA warps of the same SM.
// g -> -inf: exp(-g) = inf and __fdividef returns 0, the SiLU limit.
__device__ __forceinline__ float silu_mul(float g, float u) { return __fdividef(g, 1.0f + __expf(-g)) * u; }

__device__ __forceinline__ uint32_t pack_bf16(uint32_t lo, uint32_t hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(__uint_as_float(lo), __uint_as_float(hi));
  return *reinterpret_cast<const uint32_t*>(&v);
}

__device__ __forceinline__ void tile_coords(int64_t t, int64_t m_blocks, int64_t n_blocks,
                                            int64_t& mb, int64_t& nb) {
  // 32-bit arithmetic: tile counts fit easily, and a 64-bit divide is a ~70
  // instruction software routine on the single producer / MMA thread, paid per
  // tile (measured ~600 cycles between two tiles' MMAs on K = 512 shapes)
  const uint32_t tt = static_cast<uint32_t>(t), mbk = static_cast<uint32_t>(m_blocks);
  const uint32_t per_group = static_cast<uint32_t>(kGroupM) * static_cast<uint32_t>(n_blocks);
  const uint32_t g = tt / per_group;
  const uint32_t first_m = g * kGroupM;
  const uint32_t gm = min(static_cast<uint32_t>(kGroupM), mbk - first_m);
  const uint32_t r = tt - g * per_group;
  const uint32_t q = r / gm;
  mb = first_m + (r - q * gm);
  nb = q;
}

// Epilogue of one accumulator tile for one warp (32 rows): TMEM -> registers
// -> (epilogue math) -> bf16 -> 128B-swizzled smem staging -> TMA store.
//   EPI 0: plain, 256 output columns at nb*256.
//   EPI 1: SiLU-mul, the weight was packed so tile columns [0,128) are gate and
//          [128,256) the matching up columns; 128 outputs at nb*128.
__device__ void store_tile_rope(const CUtensorMap* map_c, uint32_t tmem_col0, uint8_t* const (&stg)[2], int lane,
                                int64_t nb, int64_t row0, int64_t M, const RopeArgs& rope);

template <int EPI, int TN = BN>
__device__ __forceinline__ void store_tile(const CUtensorMap* map_c, uint32_t tmem_col0,
                                           uint8_t* const (&stg)[2], int& buf, int lane, int64_t nb,
                                           int64_t row0, int64_t M, int first = 0, int step = 1,
                                           const RopeArgs* rope = nullptr) {
  if constexpr (EPI == 2) {
    store_tile_rope(map_c, tmem_col0, stg, lane, nb, row0, M, *rope);
    return;
  }
  // EPI 1 needs TN = 256 (gate | up halves of 128); chunks are 64 output columns
  constexpr int kChunks = EPI == 1 ? 2 : TN / 64;
  float ss = 0.0f;  // EPI 4: this lane's row, this warp's columns of the tile
#pragma unroll 1
  for (int chunk = first; chunk < kChunks; chunk += step) {
    uint32_t v0[32], v1[32];
    uint4 xres[EPI == 4 ? 8 : 1];
    if constexpr (EPI == 4) {  // residual row segment, loads in flight under the TMEM loads
      const int64_t row = row0 + lane;
      if (row < M) {
        const uint4* xr = reinterpret_cast<const uint4*>(rope->resid + row * rope->resid_ld + nb * TN + chunk * 64);
#pragma unroll
        for (int j = 0; j < 8; ++j) xres[j] = __ldcs(xr + j);
      }
    }
    const uint32_t taddr = tmem_col0 + static_cast<uint32_t>(chunk * 64);
    tmem_ld32(taddr, v0);
    tmem_ld32(taddr + 32, v1);
    if constexpr (EPI == 1) {
      uint32_t u0[32], u1[32];
      tmem_ld32(taddr + 128, u0);
      tmem_ld32(taddr + 160, u1);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float g0 = __uint_as_float(v0[i]), g1 = __uint_as_float(v1[i]);
        v0[i] = __float_as_uint(silu_mul(g0, __uint_as_float(u0[i])));
        v1[i] = __float_as_uint(silu_mul(g1, __uint_as_float(u1[i])));
      }
    } else {
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    }
    if constexpr (EPI == 4) {  // + residual row (128 B of this lane's row), sum of squares of the rounded sum
      if (row0 + lane < M) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint4 u = xres[j];
          const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
          uint32_t* dst = j < 4 ? &v0[8 * j] : &v1[8 * (j - 4)];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(h2[e]);
            const float a = __bfloat162float(__float2bfloat16(__uint_as_float(dst[2 * e]) + f.x));
            const float b = __bfloat162float(__float2bfloat16(__uint_as_float(dst[2 * e + 1]) + f.y));
            ss += a * a + b * b;
            dst[2 * e] = __float_as_uint(a);
            dst[2 * e + 1] = __float_as_uint(b);
          }
        }
      }
    }
    // staging buffer reuse: the TMA store issued two chunks ago must have read it
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncwarp();
    uint8_t* sbuf = stg[buf];
    const int r = lane;  // accumulator row within this warp's 32
#pragma unroll
    for (int j = 0; j < 8; ++j) {  // 16-byte chunk j = columns 8j..8j+7
      const uint32_t* src = j < 4 ? &v0[8 * j] : &v1[8 * (j - 4)];
      uint4 q;
      q.x = pack_bf16(src[0], src[1]);
      q.y = pack_bf16(src[2], src[3]);
      q.z = pack_bf16(src[4], src[5]);
      q.w = pack_bf16(src[6], src[7]);
      *reinterpret_cast<uint4*>(sbuf + r * 128 + ((j ^ (r & 7)) * 16)) = q;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0 && row0 < M) {
      const int64_t col = EPI == 1 ? nb * (TN / 2) + chunk * 64 : nb * TN + chunk * 64;
      tma_store_2d(map_c, sbuf, static_cast<int32_t>(col), static_cast<int32_t>(row0));
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    buf ^= 1;
  }
  if constexpr (EPI == 4) {
    static_assert(EPI != 4 || TN == 256, "EPI 4 partials assume whole 256-column tiles per warp");
    if (row0 + lane < M) rope->ssq[(row0 + lane) * rope->ssq_ld + nb] = ss;
  }
}

// Grouped (MoE) epilogue: expert segments are not tile-aligned, so rows past
// the segment end belong to the next expert's tile and must not be written;
// each lane stores its own row (512 B contiguous per chunk pair) when valid.
template <int EPI>
__device__ __forceinline__ void store_tile_direct(uint32_t tmem_col0, __nv_bfloat16* __restrict__ c,
                                                  int64_t ldc, int64_t row, int64_t row_end, int64_t nb) {
  constexpr int kChunks = EPI == 1 ? 2 : BN / 64;
#pragma unroll 1
  for (int chunk = 0; chunk < kChunks; ++chunk) {
    uint32_t v0[32], v1[32];
    const uint32_t taddr = tmem_col0 + static_cast<uint32_t>(chunk * 64);
    tmem_ld32(taddr, v0);
    tmem_ld32(taddr + 32, v1);
    if constexpr (EPI == 1) {
      uint32_t u0[32], u1[32];
      tmem_ld32(taddr + 128, u0);
      tmem_ld32(taddr + 160, u1);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float g0 = __uint_as_float(v0[i]), g1 = __uint_as_float(v1[i]);
        v0[i] = __float_as_uint(silu_mul(g0, __uint_as_float(u0[i])));
        v1[i] = __float_as_uint(silu_mul(g1, __uint_as_float(u1[i])));
      }
    } else {
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    }
    if (row < row_end) {
      const int64_t col = EPI == 1 ? nb * (BN / 2) + chunk * 64 : nb * BN + chunk * 64;
      uint4* dst = reinterpret_cast<uint4*>(c + row * ldc + col);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t* src = j < 4 ? &v0[8 * j] : &v1[8 * (j - 4)];
        uint4 q;
        q.x = pack_bf16(src[0], src[1]);
        q.y = pack_bf16(src[2], src[3]);
        q.z = pack_bf16(src[4], src[5]);
        q.w = pack_bf16(src[6], src[7]);
        dst[j] = q;
      }
    }
  }
}

template <int EPI, bool GROUPED = false>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   const __grid_constant__ CUtensorMap map_c, int64_t M, int64_t N, int64_t K,
                   const int32_t* __restrict__ gtab, __nv_bfloat16* __restrict__ c_out, int64_t ldc,
                   RopeArgs rope) {
  // GROUPED: gtab = [n_tiles, (row0, row_end, expert) x n_tiles]; N is the per-expert
  // width, expert e's B rows start at e * N; M bounds the A rows.
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stage_base = smem;
  uint8_t* epi_base = smem + kStages * kStageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(epi_base + kEpiWarps * 2 * kEpiBytes);
  uint64_t* full = bars;                      // [kStages]
  uint64_t* empty = bars + kStages;           // [kStages]
  uint64_t* tfull = bars + 2 * kStages;       // [kAccStages]
  uint64_t* tempty = bars + 2 * kStages + kAccStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 2 * kAccStages);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  int64_t m_blocks = (M + BM - 1) / BM;
  const int64_t n_blocks = (N + BN - 1) / BN;
  const int k_blocks = static_cast<int>((K + BK - 1) / BK);

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_c)) : "memory");
    }
    // whole warp: allocate all 512 TMEM columns (2 accumulators x 256 fp32)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  } else if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < kAccStages; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();
  pdl_trigger();
  if constexpr (GROUPED) m_blocks = *reinterpret_cast<const volatile int32_t*>(gtab);  // written by the routing kernel
  const int64_t tiles = m_blocks * n_blocks;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        int64_t mb, nb;
        tile_coords(t, m_blocks, n_blocks, mb, nb);
        int32_t a_row = static_cast<int32_t>(mb * BM), b_row = static_cast<int32_t>(nb * BN);
        if constexpr (GROUPED) {
          a_row = gtab[1 + 3 * mb];
          b_row += static_cast<int32_t>(gtab[3 + 3 * mb] * N);
        }
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = stage_base + stage * kStageBytes;
          mbar_expect_tx(&full[stage], kStageBytes);
          tma_load_2d(sa, &map_a, &full[stage], kb * BK, a_row);
          tma_load_2d(sa + kABytes, &map_b, &full[stage], kb * BK, b_row);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&full[stage], phase);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sa = smem_u32(stage_base + stage * kStageBytes);
          const uint32_t sb = sa + kABytes;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_f16(d_tmem, umma_desc_sw128(sa + k * 32), umma_desc_sw128(sb + k * 32),
                     (kb | k) != 0);
          umma_commit(&empty[stage]);  // frees the smem slot once these MMAs retire
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);  // accumulator ready for the epilogue
        if (++acc == kAccStages) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {  // ---------------- epilogue warps
    const int ew = warp - 2;         // 0..3
    const int quarter = warp % 4;    // TMEM lane quarter this warp may access
    uint8_t* stg[2] = {epi_base + (ew * 2) * kEpiBytes, epi_base + (ew * 2 + 1) * kEpiBytes};
    int acc = 0;
    uint32_t acc_phase = 0;
    int buf = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
      int64_t mb, nb;
      tile_coords(t, m_blocks, n_blocks, mb, nb);
      mbar_wait(&tfull[acc], acc_phase);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t tcol = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(acc * BN);
      if constexpr (GROUPED) {
        // whole 32-row slabs inside the expert segment go out by TMA; only the
        // slab straddling the segment end (rows past it belong to the next
        // expert's tile) is stored row by row
        const int64_t r0 = gtab[1 + 3 * mb] + quarter * 32, r_end = gtab[2 + 3 * mb];
        if (r0 + 32 <= r_end)
          store_tile<EPI>(&map_c, tcol, stg, buf, lane, nb, r0, M);
        else
          store_tile_direct<EPI>(tcol, c_out, ldc, r0 + lane, r_end, nb);
      } else {
        store_tile<EPI>(&map_c, tcol, stg, buf, lane, nb, mb * BM + quarter * 32, M, 0, 1, &rope);
      }
      // accumulator fully read: hand it back to the MMA warp
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == kAccStages) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
}

// ------------------------------------------------------------------ split-K (2-CTA, TN = 256)
// Under-filled grids (decode / TP-sharded shapes: M = 256..512 rows, or few N
// tiles) split the K loop over S work units per output tile so every SM
// streams weights.  Each epilogue warp owns a fixed region of the 256x256 tile
// (CTA rank r, lane quarter, 4 pieces of 32 accumulator columns): it writes its
// fp32 partial to the workspace, bumps the region's semaphore, and the warp
// that arrives last sums the S partials in split order (its own from TMEM) —
// deterministic whatever the arrival order — applies the epilogue and stores.
constexpr int kRegionFloats = 32 * 128;  // 32 rows x 4 pieces x 32 columns

// accumulator column of piece p (0..3) of this warp's region
template <int EPI>
__device__ __forceinline__ uint32_t splitk_piece_col(int half, int p) {
  if constexpr (EPI == 1) return static_cast<uint32_t>((p >> 1) * 128 + half * 64 + (p & 1) * 32);
  return static_cast<uint32_t>(((p >> 1) * 2 + half) * 64 + (p & 1) * 32);
}

// acc = sum over splits j = 0..S-1 (in order) of piece p of a region, read
// from the workspace two splits at a time (16 x 16-byte loads in flight)
__device__ __forceinline__ void ld_piece(float (&t)[32], const float4* src) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float4 x = __ldcg(src + q * 32);
    t[4 * q] = x.x;
    t[4 * q + 1] = x.y;
    t[4 * q + 2] = x.z;
    t[4 * q + 3] = x.w;
  }
}
__device__ __forceinline__ void splitk_sum_piece(float (&acc)[32], const float4* __restrict__ regions,
                                                 int64_t split_stride, int S, int p, int lane) {
  const float4* src = regions + p * 8 * 32 + lane;
  ld_piece(acc, src);  // split 0 (0 + p0 == p0 exactly)
  int j = 1;
  for (; j + 1 < S; j += 2) {
    float t0[32], t1[32];
    ld_piece(t0, src + j * split_stride);
    ld_piece(t1, src + (j + 1) * split_stride);
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = (acc[i] + t0[i]) + t1[i];
  }
  if (j < S) {
    float t0[32];
    ld_piece(t0, src + j * split_stride);
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] += t0[i];
  }
}

// bf16-pack 32 columns of this lane's row into half h (16-byte chunks 4h..4h+3)
// of the 64-column swizzled staging buffer
__device__ __forceinline__ void stage_half(uint8_t* sbuf, const float (&v)[32], int h, int lane) {
#pragma unroll
  for (int jj = 0; jj < 4; ++jj) {
    const int j = 4 * h + jj;
    uint4 q;
    q.x = pack_bf16(__float_as_uint(v[8 * jj]), __float_as_uint(v[8 * jj + 1]));
    q.y = pack_bf16(__float_as_uint(v[8 * jj + 2]), __float_as_uint(v[8 * jj + 3]));
    q.z = pack_bf16(__float_as_uint(v[8 * jj + 4]), __float_as_uint(v[8 * jj + 5]));
    q.w = pack_bf16(__float_as_uint(v[8 * jj + 6]), __float_as_uint(v[8 * jj + 7]));
    *reinterpret_cast<uint4*>(sbuf + lane * 128 + ((j ^ (lane & 7)) * 16)) = q;
  }
}
__device__ __forceinline__ uint8_t* stage_begin(uint8_t* const (&stg)[2], int buf, int lane) {
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
  __syncwarp();
  return stg[buf];
}
__device__ __forceinline__ void stage_commit(const CUtensorMap* map_c, uint8_t* sbuf, int& buf, int lane,
                                             int64_t col, int64_t row0, int64_t M) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0 && row0 < M) {
    tma_store_2d(map_c, sbuf, static_cast<int32_t>(col), static_cast<int32_t>(row0));
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  buf ^= 1;
}

// RoPE epilogue (EPI 2, TN = 256): this warp's 32 rows of the two 128-wide
// heads of the tile.  Rotate-half on q/k heads (global head < rot_heads):
//   out[d] = a cos - b sin, out[d + 64] = b cos + a sin,  a = x[d], b = x[d + 64],
//   angle = pos * theta^(-d / 64)  (HF / the rope op in llama_ops.cu),
// applied to the fp32 accumulator before the bf16 rounding; v heads copied.
// Both staging buffers hold one head (dims 0-63 | 64-127).
__device__ void store_tile_rope(const CUtensorMap* map_c, uint32_t tmem_col0, uint8_t* const (&stg)[2], int lane,
                                int64_t nb, int64_t row0, int64_t M, const RopeArgs& rope) {
  const int64_t row = row0 + lane;
  const float p = row < M ? static_cast<float>(rope.pos[row]) : 0.0f;
#pragma unroll 1
  for (int hh = 0; hh < 2; ++hh) {
    const bool rot = nb * 2 + hh < rope.rot_heads;
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncwarp();
#pragma unroll 1
    for (int j = 0; j < 2; ++j) {
      uint32_t a[32], b[32];
      tmem_ld32(tmem_col0 + static_cast<uint32_t>(hh * 128 + j * 32), a);
      tmem_ld32(tmem_col0 + static_cast<uint32_t>(hh * 128 + 64 + j * 32), b);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      float ra[32], rb[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float x = __uint_as_float(a[i]), y = __uint_as_float(b[i]);
        if (rot) {
          // angle reduced to [-pi, pi] (two-constant Cody-Waite), then the MUFU
          // sin/cos (abs err ~2^-21 there; the bf16 output rounds at 2^-8)
          const float inv_freq = exp2f(-2.0f * static_cast<float>(j * 32 + i) / 128.0f * rope.log2_theta);
          const float ang = p * inv_freq;
          const float q = rintf(ang * 0.15915494309189535f);
          const float r = fmaf(-q, 6.28318548202514648f, fmaf(-q, -1.7484556e-07f, ang));
          float sn, cs;
          __sincosf(r, &sn, &cs);
          ra[i] = x * cs - y * sn;
          rb[i] = y * cs + x * sn;
        } else {
          ra[i] = x;
          rb[i] = y;
        }
      }
      stage_half(stg[0], ra, j, lane);
      stage_half(stg[1], rb, j, lane);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0 && row0 < M) {
      const int32_t col = static_cast<int32_t>(nb * 256 + hh * 128);
      tma_store_2d(map_c, stg[0], col, static_cast<int32_t>(row0));
      tma_store_2d(map_c, stg[1], col + 64, static_cast<int32_t>(row0));
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
}

// One epilogue warp's share of split `mine` of tile `tile`.  The accumulator
// is released (release_acc) as soon as the partial is in the workspace, so
// the last arriver's fixup overlaps the next unit's MMAs.
template <int EPI, typename Release>
__device__ __forceinline__ void store_tile_splitk(const CUtensorMap* map_c, uint32_t tcol, uint8_t* const (&stg)[2],
                                                  int& buf, int lane, int64_t nb, int64_t row0, int64_t M,
                                                  int half, int region, int64_t tile, int mine, int S,
                                                  float4* __restrict__ ws, int* __restrict__ sem,
                                                  Release release_acc) {
  const int64_t split_stride = 16LL * kRegionFloats / 4;  // float4s between splits of one region
  float4* regions = ws + (tile * S * 16 + region) * (kRegionFloats / 4);
  float4* my = regions + mine * split_stride;
  // 1. partial -> workspace (coalesced: a warp store covers 512 contiguous bytes)
#pragma unroll 1
  for (int p = 0; p < 4; ++p) {
    uint32_t v[32];
    tmem_ld32(tcol + splitk_piece_col<EPI>(half, p), v);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int q = 0; q < 8; ++q)
      __stcg(my + p * 8 * 32 + q * 32 + lane,
             make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                         __uint_as_float(v[4 * q + 3])));
  }
  release_acc();
  __threadfence();
  __syncwarp();
  int old = 0;
  int* sm = sem + tile * 16 + region;
  if (lane == 0) old = atomicAdd(sm, 1);
  old = __shfl_sync(0xffffffffu, old, 0);
  if (old != S - 1) return;
  // 2. last arriver: sum the S partials in split order, epilogue, store
  __threadfence();
  if (lane == 0) *sm = 0;  // self-cleaning for the next launch on this workspace
  if constexpr (EPI == 1) {
    uint8_t* sbuf = stage_begin(stg, buf, lane);
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      float g[32], u[32];
      splitk_sum_piece(g, regions, split_stride, S, h, lane);
      splitk_sum_piece(u, regions, split_stride, S, 2 + h, lane);
#pragma unroll
      for (int i = 0; i < 32; ++i) g[i] = silu_mul(g[i], u[i]);
      stage_half(sbuf, g, h, lane);
    }
    stage_commit(map_c, sbuf, buf, lane, nb * 128 + half * 64, row0, M);
  } else {
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      uint8_t* sbuf = stage_begin(stg, buf, lane);
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        float v[32];
        splitk_sum_piece(v, regions, split_stride, S, 2 * c + h, lane);
        stage_half(sbuf, v, h, lane);
      }
      stage_commit(map_c, sbuf, buf, lane, nb * 256 + (2 * c + half) * 64, row0, M);
    }
  }
}

// ------------------------------------------------------------------ 2-CTA (cta_group::2) path
// A CTA pair (cluster of 2 on one TPC) owns a 256x256 output tile.  Each CTA
// TMA-loads its own 128 A rows and 128 of the 256 B rows per 64-deep k-block
// (32 KB / stage instead of 48 KB: half the L2->SM operand traffic per MAC),
// the leader's single thread issues M=256 N=256 tcgen05.mma over both CTAs'
// shared memory, and each CTA's TMEM receives its 128 accumulator rows.
// Full barriers live in the leader (TMA complete_tx from both CTAs lands
// there); smem-slot and accumulator-ready commits multicast to both CTAs;
// both CTAs' epilogue warps release the accumulator on the leader's barrier.
//
// Tile width TN in {256, 384} (384: one-wave shapes, below).  Epilogue
// warps: 4 (one per TMEM lane quarter, 6-stage ring) for whole-K tiles; the
// split-K variant uses 8 (warp w reads lane quarter w % 4 and the 64-column
// chunks (w - 2) / 4, +2: 16 independent regions per tile for the partial
// fixup) with a 5-stage ring.  8 warps did not speed up the whole-K epilogue
// on short-K shapes (A/B in profiles/r01_gemm_ab_r0_vs_new.jsonl), so the
// lighter 4-warp / 6-stage configuration stays there.
//
// TN = 384 (one-wave shapes, e.g. the TP=8 QKV 8192x768: 64 tiles of 256x384
// on 74 clusters instead of 96 tiles of 256x256, a 1.3-wave tail): per k16 two
// MMAs, N = 256 (TMEM columns 0..255, B rows 0..127 of each CTA's half) and
// N = 128 (columns 256..383, B rows 128..191); one accumulator stage (384 of
// the 512 TMEM columns), plain-store epilogue only.
template <int TN, bool SPLIT>
struct Tc2Cfg {
  static constexpr int kEpiW = SPLIT ? 8 : 4;
  static constexpr int kThreads = 64 + kEpiW * 32;
  static constexpr int kAcc = TN == 384 ? 1 : 2;       // TMEM accumulator stages
  static constexpr int kStg = TN == 384 ? 1 : 2;       // 4 KB staging buffers per epilogue warp
  static constexpr uint32_t kStageBytes = kABytes + (TN / 2) * BK * 2;
  static constexpr uint32_t kFixed = 1024 + kEpiW * kStg * kEpiBytes + 512;
  static constexpr int kStages = ((232448 - kFixed) / kStageBytes) > 6 ? 6 : (232448 - kFixed) / kStageBytes;
  static constexpr uint32_t kSmemBytes = kFixed + kStages * kStageBytes;
  static constexpr uint32_t idesc(int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
           (static_cast<uint32_t>(256 >> 4) << 24);
  }
  static constexpr uint32_t kIdesc = idesc(TN == 384 ? 256 : TN);
};
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // clear the CTA-rank bit: address the pair leader

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint64_t* bar,
                                                 int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], "
      "[%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & kPeerMask), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void umma_f16_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                              uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], "
      "%1;" ::"r"(smem_u32(bar)),
      "h"(static_cast<uint16_t>(0x3))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(smem_u32(bar) & kPeerMask)
               : "memory");
}
// Accumulator hand-back: only the (already waited-for) TMEM loads must precede
// it, so no release semantics — a .release arrive would first drain every
// global store this thread issued (measured ~1.9k cycles per tile).
__device__ __forceinline__ void mbar_arrive_leader_relaxed(uint64_t* bar) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(smem_u32(bar) & kPeerMask)
               : "memory");
}

// Epilogue of one accumulator tile for one warp (32 rows) with plain global
// stores: TMEM -> registers (-> SiLU-mul / residual add) -> bf16 -> a 4 KB
// 128B-swizzled staging buffer (lane = row) -> read back so that 8 lanes
// cover one 128-byte row segment (each store instruction writes 4 whole
// rows x 128 B) -> st.global.  The accumulator is released as soon as its
// last TMEM load lands, so the next tile's MMAs never wait for the stores, and
// no TMA store shares the TMA unit with the operand loads (measured: the
// TMA-store epilogue took 4-6k cycles per 128x256 tile and bounded every
// short-K shape, tools/gemm_trace.py).
template <int EPI, int TN, typename Release, typename Mark>
__device__ __forceinline__ void store_tile_st(uint32_t tmem_col0, uint8_t* sbuf, int lane, int64_t nb, int64_t row0,
                                              int64_t M, int64_t n_out, __nv_bfloat16* __restrict__ c, int64_t ldc,
                                              const RopeArgs* rope, Release&& release, Mark&& mark,
                                              bool direct = false) {
  constexpr int kChunks = EPI == 1 ? 2 : TN / 64;
  float ss = 0.0f;  // EPI 4: this lane's row, this tile's columns
  const bool row_ok = row0 + lane < M;
#pragma unroll 1
  for (int chunk = 0; chunk < kChunks; ++chunk) {
    uint32_t v0[32], v1[32];
    uint4 xres[EPI == 4 ? 8 : 1];
    if constexpr (EPI == 4) {  // residual row segment, in flight under the TMEM loads
      if (row_ok) {
        const uint4* xr =
            reinterpret_cast<const uint4*>(rope->resid + (row0 + lane) * rope->resid_ld + nb * TN + chunk * 64);
#pragma unroll
        for (int j = 0; j < 8; ++j) xres[j] = __ldcs(xr + j);
      }
    }
    const uint32_t taddr = tmem_col0 + static_cast<uint32_t>(chunk * 64);
    tmem_ld32(taddr, v0);
    tmem_ld32(taddr + 32, v1);
    if constexpr (EPI == 1) {
      uint32_t u0[32], u1[32];
      tmem_ld32(taddr + 128, u0);
      tmem_ld32(taddr + 160, u1);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (chunk == kChunks - 1) release();
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float g0 = __uint_as_float(v0[i]), g1 = __uint_as_float(v1[i]);
        v0[i] = __float_as_uint(silu_mul(g0, __uint_as_float(u0[i])));
        v1[i] = __float_as_uint(silu_mul(g1, __uint_as_float(u1[i])));
      }
    } else {
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      mark(4);
      if (chunk == kChunks - 1) release();
    }
    if constexpr (EPI == 4) {  // + residual, sum of squares of the rounded sum
      if (row_ok) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint4 u = xres[j];
          const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
          uint32_t* dst = j < 4 ? &v0[8 * j] : &v1[8 * (j - 4)];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(h2[e]);
            const float a = __bfloat162float(__float2bfloat16(__uint_as_float(dst[2 * e]) + f.x));
            const float b = __bfloat162float(__float2bfloat16(__uint_as_float(dst[2 * e + 1]) + f.y));
            ss += a * a + b * b;
            dst[2 * e] = __float_as_uint(a);
            dst[2 * e + 1] = __float_as_uint(b);
          }
        }
      }
    }
    // direct (32-byte aligned rows only): each lane stores its own row's 64
    // columns (32 B per store, not allocated in L1) instead of staging them through shared memory for
    // 4-row coalesced stores.  The staging's shared-memory traffic (128 KB per
    // 256x256 tile) matters on short-K tiles (8-28 k-blocks: the TP=8 O and
    // down projections, -4% / -1.7%); on K >= 4096 the coalesced form is as
    // fast or faster (profiles/r02_gemm_epi_direct_na_ab.txt).
    if (direct) {
      const int64_t col0d = (EPI == 1 ? nb * (TN / 2) : nb * TN) + chunk * 64;
      if (col0d + 64 <= n_out) {
        if (row_ok) {
          __nv_bfloat16* dst = c + (row0 + lane) * ldc + col0d;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t* src = j < 2 ? &v0[16 * j] : &v1[16 * (j - 2)];
            uint32_t w[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) w[e] = pack_bf16(src[2 * e], src[2 * e + 1]);
            asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst + 16 * j),
                         "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                         : "memory");
          }
        }
        mark(5);
        continue;
      }
    }
    __syncwarp();  // the previous chunk's read-back of sbuf is done
#pragma unroll
    for (int j = 0; j < 8; ++j) {  // 16-byte piece j = columns 8j..8j+7 of this lane's row
      const uint32_t* src = j < 4 ? &v0[8 * j] : &v1[8 * (j - 4)];
      uint4 q;
      q.x = pack_bf16(src[0], src[1]);
      q.y = pack_bf16(src[2], src[3]);
      q.z = pack_bf16(src[4], src[5]);
      q.w = pack_bf16(src[6], src[7]);
      *reinterpret_cast<uint4*>(sbuf + lane * 128 + ((j ^ (lane & 7)) * 16)) = q;
    }
    __syncwarp();
    const int64_t col0 = (EPI == 1 ? nb * (TN / 2) : nb * TN) + chunk * 64;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int row = i * 4 + lane / 8, j = lane % 8;
      const int64_t col = col0 + j * 8;
      if (row0 + row < M && col < n_out) {
        const uint4 u = *reinterpret_cast<const uint4*>(sbuf + row * 128 + ((j ^ (row & 7)) * 16));
        *reinterpret_cast<uint4*>(c + (row0 + row) * ldc + col) = u;
      }
    }
    mark(5);
  }
  if constexpr (EPI == 4) {
    static_assert(EPI != 4 || TN == 256, "EPI 4 partials assume whole 256-column tiles per warp");
    if (row_ok) rope->ssq[(row0 + lane) * rope->ssq_ld + nb] = ss;
  }
}

// RoPE epilogue with plain stores (EPI 2, TN = 256 or 384: TN / 128 heads of
// 128 per tile).  For head h of the tile, dims d < 64 and d + 64 rotate as
// in store_tile_rope; the two 64-column halves go out one after the other
// through the warp's one 4 KB staging buffer (the half not being staged is
// recomputed from TMEM, which is cheaper than a second buffer's worth of
// pipeline stages).  Released after the last head's last TMEM load.
template <int TN, typename Release>
__device__ __forceinline__ void store_tile_rope_st(uint32_t tmem_col0, uint8_t* sbuf, int lane, int64_t nb,
                                                   int64_t row0, int64_t M, int64_t n_out,
                                                   __nv_bfloat16* __restrict__ c, int64_t ldc, const RopeArgs& rope,
                                                   Release&& release) {
  (void)sbuf;
  constexpr int kHeads = TN / 128;
  const bool row_ok = row0 + lane < M;
  const float p = row_ok ? static_cast<float>(rope.pos[row0 + lane]) : 0.0f;
  __nv_bfloat16* crow = c + (row0 + lane) * ldc + nb * TN;
  // Pair-chunk j (32 of the 64 rotation pairs) outermost: the cos / sin of
  // this lane's row for those pairs are computed ONCE per tile and reused by
  // every head and both halves (the per-element form, 2 x heads sincos + an
  // exp2 per pair, took ~40k cycles per decode tile).  Each lane owns one row
  // and stores its 8-column pieces directly (16 B per store; L2 merges the
  // sectors), so no staging order ties the heads together.
#pragma unroll 1
  for (int j = 0; j < 2; ++j) {
    float cs[32], sn[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float inv_freq = exp2f(-2.0f * static_cast<float>(j * 32 + i) / 128.0f * rope.log2_theta);
      const float ang = p * inv_freq;
      const float q = rintf(ang * 0.15915494309189535f);
      const float r = fmaf(-q, 6.28318548202514648f, fmaf(-q, -1.7484556e-07f, ang));
      __sincosf(r, &sn[i], &cs[i]);
    }
#pragma unroll 1
    for (int hh = 0; hh < kHeads; ++hh) {
      const bool rot = (nb * TN) / 128 + hh < rope.rot_heads;
      uint32_t a[32], b[32];
      tmem_ld32(tmem_col0 + static_cast<uint32_t>(hh * 128 + j * 32), a);
      tmem_ld32(tmem_col0 + static_cast<uint32_t>(hh * 128 + 64 + j * 32), b);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (hh == kHeads - 1 && j == 1) release();
      const int64_t col_lo = hh * 128 + j * 32;
#pragma unroll
      for (int q8 = 0; q8 < 4; ++q8) {
        float o0[8], o1[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int i = q8 * 8 + e;
          const float x = __uint_as_float(a[i]), y = __uint_as_float(b[i]);
          o0[e] = rot ? x * cs[i] - y * sn[i] : x;
          o1[e] = rot ? y * cs[i] + x * sn[i] : y;
        }
        if (row_ok && nb * TN + hh * 128 + 128 <= n_out) {
          uint4 u0, u1;
          u0.x = pack_bf16(__float_as_uint(o0[0]), __float_as_uint(o0[1]));
          u0.y = pack_bf16(__float_as_uint(o0[2]), __float_as_uint(o0[3]));
          u0.z = pack_bf16(__float_as_uint(o0[4]), __float_as_uint(o0[5]));
          u0.w = pack_bf16(__float_as_uint(o0[6]), __float_as_uint(o0[7]));
          u1.x = pack_bf16(__float_as_uint(o1[0]), __float_as_uint(o1[1]));
          u1.y = pack_bf16(__float_as_uint(o1[2]), __float_as_uint(o1[3]));
          u1.z = pack_bf16(__float_as_uint(o1[4]), __float_as_uint(o1[5]));
          u1.w = pack_bf16(__float_as_uint(o1[6]), __float_as_uint(o1[7]));
          *reinterpret_cast<uint4*>(crow + col_lo + q8 * 8) = u0;
          *reinterpret_cast<uint4*>(crow + col_lo + 64 + q8 * 8) = u1;
        }
      }
    }
  }
}

// Push epilogue (EPI 3): the 32-row slab of this warp goes straight into the
// owner rank's window (row r -> owner r / blk, this rank's slot there), 64
// columns at a time through the swizzled staging buffer so every store
// instruction writes 4 rows x 128 contiguous bytes (NVLink-friendly), then one
// system-scope release increment of the owner's slab counter per tile.  Never
// waits on a peer: the reduce side does all the waiting.
template <int TN, typename Release>
__device__ __forceinline__ void store_tile_push(uint32_t tmem_col0, uint8_t* sbuf, int lane, int64_t nb, int64_t row0,
                                                int64_t M, int64_t N, const PushArgs& pa, Release&& release) {
  const int q = static_cast<int>(row0 / pa.blk);
  const int64_t lr = row0 - q * pa.blk;
  __nv_bfloat16* dst = row0 < M ? static_cast<__nv_bfloat16*>(pa.dst[q]) + lr * N + nb * TN : nullptr;
#pragma unroll 1
  for (int chunk = 0; chunk < TN / 64; ++chunk) {
    uint32_t v0[32], v1[32];
    const uint32_t taddr = tmem_col0 + static_cast<uint32_t>(chunk * 64);
    tmem_ld32(taddr, v0);
    tmem_ld32(taddr + 32, v1);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (chunk == TN / 64 - 1) release();  // accumulator fully read
    __syncwarp();  // the previous chunk's read-back of sbuf is done
    const int r = lane;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t* src = j < 4 ? &v0[8 * j] : &v1[8 * (j - 4)];
      uint4 u;
      u.x = pack_bf16(src[0], src[1]);
      u.y = pack_bf16(src[2], src[3]);
      u.z = pack_bf16(src[4], src[5]);
      u.w = pack_bf16(src[6], src[7]);
      *reinterpret_cast<uint4*>(sbuf + r * 128 + ((j ^ (r & 7)) * 16)) = u;
    }
    __syncwarp();
    if (dst) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int row = i * 4 + lane / 8, j = lane % 8;
        const uint4 u = *reinterpret_cast<const uint4*>(sbuf + row * 128 + ((j ^ (row & 7)) * 16));
        *reinterpret_cast<uint4*>(dst + row * N + chunk * 64 + j * 8) = u;
      }
    }
  }
  if (!dst) return;
  __threadfence_system();
  __syncwarp();
  if (lane == 0)
    asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(pa.cnt[q] + lr / 32), "r"(1u) : "memory");
}

// Per-tile timeline of cluster 0's leader CTA (tools/gemm_trace.py), compiled
// in only with -DOPF_GEMM_TRACE: role r (0 producer, 1 MMA, 2 epilogue warp
// 2) appends (event, unit, clock64) records.
#ifdef OPF_GEMM_TRACE
__device__ unsigned long long g_gemm_trace[3][2048];
__device__ int g_gemm_trace_n[3];
// counters live in registers (a global read-modify-write per event would add
// an L2 round trip to the timeline it measures)
#define GTRACE(role, ev, unit)                                                                  \
  do {                                                                                          \
    if (blockIdx.x == 0 && gt_n < 2048)                                                         \
      g_gemm_trace[role][gt_n++] = (static_cast<unsigned long long>(ev) << 56) |                \
                                   (static_cast<unsigned long long>((unit) & 0xFFFF) << 40) |   \
                                   (clock64() & 0xFFFFFFFFFFull);                               \
  } while (0)
#define GTRACE_END(role) \
  do {                   \
    if (blockIdx.x == 0) g_gemm_trace_n[role] = gt_n; \
  } while (0)
#else
#define GTRACE(role, ev, unit) \
  do {                         \
  } while (0)
#define GTRACE_END(role) \
  do {                   \
  } while (0)
#endif

template <int EPI, int TN, bool SPLIT = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Tc2Cfg<TN, SPLIT>::kThreads, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                    const __grid_constant__ CUtensorMap map_c, int64_t M, int64_t N, int64_t K, int splits,
                    float4* __restrict__ ws, int* __restrict__ sem, RopeArgs rope, __nv_bfloat16* __restrict__ c_out,
                    int64_t ldc, PushArgs push) {
  using C = Tc2Cfg<TN, SPLIT>;
  constexpr int kStages2 = C::kStages;
  constexpr uint32_t kStageBytes2 = C::kStageBytes;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stage_base = smem;
  constexpr int kAcc = C::kAcc;
  uint8_t* epi_base = smem + kStages2 * kStageBytes2;
  uint64_t* bars = reinterpret_cast<uint64_t*>(epi_base + C::kEpiW * C::kStg * kEpiBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages2;
  uint64_t* tfull = bars + 2 * kStages2;
  uint64_t* tempty = bars + 2 * kStages2 + kAcc;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages2 + 2 * kAcc);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_rank();
#ifdef OPF_GEMM_TRACE
  int gt_n = 0;
#endif
  const bool leader = rank == 0;
  const int64_t m_blocks = (M + 2 * BM - 1) / (2 * BM);
  const int64_t n_blocks = (N + TN - 1) / TN;
  const int k_blocks = static_cast<int>((K + BK - 1) / BK);
  const int64_t cluster = blockIdx.x / 2, n_clusters = gridDim.x / 2;

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_c)) : "memory");
    }
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  } else if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < kAcc; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * C::kEpiW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();     // inputs of the previous kernel on this stream are visible from here
  pdl_trigger();  // persistent grid: let the next kernel stage its prologue on freed SMs
  if constexpr (EPI == 3)  // one new push call: the reduce kernel that follows waits for this epoch's publishes
    if (blockIdx.x == 0 && threadIdx.x == 0) *push.epoch += 1;
  const int64_t tiles = m_blocks * n_blocks;
  const int64_t units = tiles * splits;  // unit u = split (u % splits) of tile (u / splits)

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs)
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t u = cluster; u < units; u += n_clusters) {
        const int64_t t = splits == 1 ? u : static_cast<int64_t>(static_cast<uint32_t>(u) / static_cast<uint32_t>(splits));
        const int sp = static_cast<int>(u - t * splits);
        int64_t mb, nb;
        tile_coords(t, m_blocks, n_blocks, mb, nb);
        const int32_t m0 = static_cast<int32_t>(mb * 2 * BM + rank * BM);
        const int32_t n0 = static_cast<int32_t>(nb * TN + rank * (TN / 2));
        const int kb0 = splits == 1 ? 0 : sp * k_blocks / splits;
        const int kb1 = splits == 1 ? k_blocks : (sp + 1) * k_blocks / splits;
        GTRACE(0, 0, u);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (kb == kb0) GTRACE(0, 1, u);
          uint8_t* sa = stage_base + stage * kStageBytes2;
          if (leader) mbar_expect_tx(&full[stage], 2 * kStageBytes2);
          tma_load_2d_pair(sa, &map_a, &full[stage], kb * BK, m0);
          if constexpr (TN == 384) {  // B box = 64 rows: MMA-1 rows (2 boxes), then MMA-2 rows
            const int32_t nt = static_cast<int32_t>(nb * 384);
            tma_load_2d_pair(sa + kABytes, &map_b, &full[stage], kb * BK, nt + static_cast<int32_t>(rank) * 128);
            tma_load_2d_pair(sa + kABytes + 8192, &map_b, &full[stage], kb * BK,
                             nt + static_cast<int32_t>(rank) * 128 + 64);
            tma_load_2d_pair(sa + kABytes + 16384, &map_b, &full[stage], kb * BK,
                             nt + 256 + static_cast<int32_t>(rank) * 64);
          } else {
            tma_load_2d_pair(sa + kABytes, &map_b, &full[stage], kb * BK, n0);
          }
          if (++stage == kStages2) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      GTRACE_END(0);
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // ---------------- MMA issuer (leader CTA)
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int64_t u = cluster; u < units; u += n_clusters) {
        const int sp = splits == 1 ? 0 : static_cast<int>(static_cast<uint32_t>(u) % static_cast<uint32_t>(splits));
        const int kb0 = splits == 1 ? 0 : sp * k_blocks / splits;
        const int kb1 = splits == 1 ? k_blocks : (sp + 1) * k_blocks / splits;
        GTRACE(1, 0, u);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        GTRACE(1, 1, u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * TN);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          GTRACE(1, 2, u);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sa = smem_u32(stage_base + stage * kStageBytes2);
          const uint32_t sb = sa + kABytes;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            umma_f16_pair(d_tmem, umma_desc_sw128(sa + k * 32), umma_desc_sw128(sb + k * 32), C::kIdesc,
                          (kb != kb0 || k != 0) ? 1u : 0u);
            if constexpr (TN == 384)
              umma_f16_pair(d_tmem + 256, umma_desc_sw128(sa + k * 32), umma_desc_sw128(sb + 16384 + k * 32),
                            C::idesc(128), (kb != kb0 || k != 0) ? 1u : 0u);
          }
          umma_commit_pair(&empty[stage]);
          if (++stage == kStages2) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_pair(&tfull[acc]);
        GTRACE(1, 3, u);
        if (++acc == kAcc) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      GTRACE_END(1);
    }
  } else {  // ---------------- epilogue warps (both CTAs)
    const int ew = warp - 2;
    const int quarter = warp % 4;
    const int half = C::kEpiW == 8 ? ew / 4 : 0;  // column chunks half, half + step, ...
    constexpr int kStep = C::kEpiW == 8 ? 2 : 1;
    uint8_t* stg[2] = {epi_base + (ew * C::kStg) * kEpiBytes, epi_base + (ew * C::kStg + C::kStg - 1) * kEpiBytes};
    int acc = 0;
    uint32_t acc_phase = 0;
    int buf = 0;
    for (int64_t u = cluster; u < units; u += n_clusters) {
      const int64_t t = splits == 1 ? u : static_cast<int64_t>(static_cast<uint32_t>(u) / static_cast<uint32_t>(splits));
      int64_t mb, nb;
      tile_coords(t, m_blocks, n_blocks, mb, nb);
      if (warp == 2 && lane == 0) GTRACE(2, 0, u);
      mbar_wait(&tfull[acc], acc_phase);
      if (warp == 2 && lane == 0) GTRACE(2, 1, u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int64_t row0 = mb * 2 * BM + rank * BM + quarter * 32;
      const uint32_t tcol = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(acc * TN);
      auto release = [&]() {  // accumulator fully read: hand it back to the MMA warp
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive_leader_relaxed(&tempty[acc]);
        if (warp == 2 && lane == 0) GTRACE(2, 2, u);
      };
      if constexpr (EPI == 3) {
        store_tile_push<TN>(tcol, stg[0], lane, nb, row0, M, N, push, release);
      } else if constexpr (SPLIT && TN == 256) {
        store_tile_splitk<EPI>(&map_c, tcol, stg, buf, lane, nb, row0, M, half, static_cast<int>(rank) * 8 + ew, t,
                               static_cast<int>(u - t * splits), splits, ws, sem, release);
      } else if constexpr (EPI == 2) {
        store_tile_rope_st<TN>(tcol, stg[0], lane, nb, row0, M, N, c_out, ldc, rope, release);
      } else {
        auto mark = [&](int ev) {
          if (warp == 2 && lane == 0) GTRACE(2, ev, u);
        };
        store_tile_st<EPI, TN>(tcol, stg[0], lane, nb, row0, M, EPI == 1 ? N / 2 : N, c_out, ldc, &rope, release,
                               mark,
                               K <= 2048 && ldc % 16 == 0 && (reinterpret_cast<uintptr_t>(c_out) & 31) == 0);
      }
      if (warp == 2 && lane == 0) GTRACE(2, 3, u);
      if (++acc == kAcc) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (warp == 2 && lane == 0) GTRACE_END(2);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
}

// ------------------------------------------------------------------ host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fail(Errc::SchedulerError, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<EncodeFn>(p);
  }();
  return fn;
}

CUtensorMap make_map(const void* base, int64_t inner, int64_t outer, int64_t ld_elems,
                     uint32_t box_inner, uint32_t box_outer) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld_elems) * 2};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base),
                                 dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  require(r == CUDA_SUCCESS, Errc::SchedulerError,
          "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
  return m;
}

}  // namespace

void gemm_bf16_tc_init() {
  static std::once_flag once;
  std::call_once(once, [] {
    OPF_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kSmemBytes)));
    OPF_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kSmemBytes)));
    OPF_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kSmemBytes)));
    OPF_CUDA(cudaFuncSetAttribute(gemm_tc2_kernel<2, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(Tc2Cfg<256, false>::kSmemBytes)));
    OPF_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kSmemBytes)));
    OPF_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kSmemBytes)));
    OPF_CUDA(cudaFuncSetAttribute(gemm_tc2_kernel<0, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(Tc2Cfg<256, false>::kSmemBytes)));
    OPF_CUDA(cudaFuncSetAttribute(gemm_tc2_kernel<0, 384>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(Tc2Cfg<384, false>::kSmemBytes)));
    OPF_CUDA(cudaFuncSetAttribute(gemm_tc2_kernel<2, 384>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(Tc2Cfg<384, false>::kSmemBytes)));
    OPF_CUDA(cudaFuncSetAttribute(gemm_tc2_kernel<1, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(Tc2Cfg<256, false>::kSmemBytes)));
    OPF_CUDA(cudaFuncSetAttribute(gemm_tc2_kernel<4, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(Tc2Cfg<256, false>::kSmemBytes)));
    OPF_CUDA(cudaFuncSetAttribute(gemm_tc2_kernel<0, 256, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(Tc2Cfg<256, true>::kSmemBytes)));
    OPF_CUDA(cudaFuncSetAttribute(gemm_tc2_kernel<1, 256, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(Tc2Cfg<256, true>::kSmemBytes)));
  });
}

void gemm_bf16_simt(const GemmArgs& g, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>((g.n + 63) / 64), static_cast<unsigned>((g.m + 63) / 64));
  gemm_simt_kernel<<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(g.a),
                                        static_cast<const __nv_bfloat16*>(g.bt),
                                        static_cast<__nv_bfloat16*>(g.c), g.m, g.n, g.k, g.lda,
                                        g.ldc, g.b_kn);
}

// K splits for a 2-CTA launch.  Split only when every split of every tile
// fits in ONE round of clusters (measured on B200: in multi-round grids the
// partial write + fixup is paid by every unit and loses, e.g. 8192x768x4096
// 49 -> 67 us at S = 3), each split keeps >= 16 k-blocks, and the split saves
// >= 32 k-block steps (~9 us) against a ~10 us fixed prologue / drain / fixup
// cost (profiles/r01_gemm_splitk_ab.json).  Largest such S <= 8.
int gemm_splitk_splits(int64_t m, int64_t n, int64_t k, int max_ctas) {
  if (m <= BM) return 1;
  static const int forced = [] {
    const char* e = std::getenv("OPF_GEMM_SPLITK");
    return e ? std::atoi(e) : -1;
  }();
  int grid = num_sms();
  if (max_ctas > 0 && max_ctas < grid) grid = max_ctas;
  const int64_t clusters = std::max(grid / 2, 1);
  const int64_t tiles = ((m + 2 * BM - 1) / (2 * BM)) * ((n + 255) / 256);
  const int64_t kb = (k + BK - 1) / BK;
  if (forced >= 1) return static_cast<int>(std::min<int64_t>(forced, std::max<int64_t>(kb, 1)));
  int best = 1;
  for (int S = 2; S <= 8; ++S)
    if (tiles * S <= clusters && kb / S >= 16 && kb - kb / S >= 32) best = S;
  return best;
}

size_t gemm_splitk_workspace(int64_t m, int64_t n, int64_t k, int max_ctas) {
  const int S = gemm_splitk_splits(m, n, k, max_ctas);
  if (S <= 1) return 0;
  const int64_t tiles = ((m + 2 * BM - 1) / (2 * BM)) * ((n + 255) / 256);
  return static_cast<size_t>(tiles * S * 16 * kRegionFloats) * sizeof(float) +
         static_cast<size_t>(tiles * 16) * sizeof(int);
}

constexpr __nv_bfloat16* kNoOut = nullptr;
constexpr PushArgs kNoPush{};

void gemm_bf16_tc(const GemmArgs& g, cudaStream_t s) {
  require(g.k % 8 == 0 && g.lda % 8 == 0 && g.ldc % 8 == 0, Errc::ShapeMismatch,
          "tcgen05 GEMM needs 16-byte aligned rows (K, lda, ldc multiples of 8)");
  require((reinterpret_cast<uintptr_t>(g.a) | reinterpret_cast<uintptr_t>(g.bt) |
           reinterpret_cast<uintptr_t>(g.c)) % 16 == 0,
          Errc::ShapeMismatch, "tcgen05 GEMM needs 16-byte aligned base pointers");
  require(g.epi == 0 || g.n % BN == 0, Errc::ShapeMismatch,
          "SiLU-mul / RoPE epilogues need N to be a multiple of 256");
  require(g.epi != 2 || g.pos != nullptr, Errc::ShapeMismatch, "RoPE epilogue needs positions");
  require(g.epi != 4 || (g.n % 256 == 0 && g.resid && g.ssq), Errc::ShapeMismatch,
          "residual-norm epilogue needs N % 256 == 0, the residual and the statistics buffer");
  const RopeArgs rope{g.pos, g.rot_heads, g.log2_theta, static_cast<const __nv_bfloat16*>(g.resid), g.ssq,
                      g.n / 256, g.n};
  gemm_bf16_tc_init();
  static const int mode = [] {  // OPF_GEMM=1sm|2sm|auto
    const char* e = std::getenv("OPF_GEMM");
    if (e && std::string(e) == "1sm") return 1;
    if (e && std::string(e) == "2sm") return 2;
    return 0;
  }();
  const bool pair = mode == 2 || (mode == 0 && g.m > BM) || g.epi == 4;  // EPI 4 lives in the 2-CTA kernel
  const int64_t n_out = g.epi == 1 ? g.n / 2 : g.n;
  const CUtensorMap ma = make_map(g.a, g.k, g.m, g.lda, BK, BM);
  const CUtensorMap mc = make_map(g.c, n_out, g.m, g.ldc, 64, 32);
  int grid = num_sms();
  if (g.max_ctas > 0 && g.max_ctas < grid) grid = g.max_ctas;
  if (pair) {
    const int64_t mt = (g.m + 2 * BM - 1) / (2 * BM);
    const int cmax = std::max(grid / 2, 1);
    // Tile width 256, or 384 for one-wave shapes.  (Narrower 192 / 128 tiles
    // quantise better onto 74 clusters, e.g. N = 768: 96 -> 128 tiles, but
    // measured slower per FLOP on B200 — more L2 -> SMEM bytes per MAC —
    // profiles/r01_gemm_sweep*.json; they were removed in round 2.)
    int tn = 256;
    if (g.epi == 0 || g.epi == 2) {
      // 256x384 tiles when they fit one round of clusters and 256-wide ones
      // would need two (a ~1.3-wave tail): e.g. 8192 x 768 -> 64 tiles, not 96
      const int64_t t256 = mt * ((g.n + 255) / 256), t384 = mt * ((g.n + 383) / 384);
      const bool one_wave_384 = g.n % 384 == 0 && t384 <= cmax && t256 > cmax && g.k >= 1024;
      tn = one_wave_384 ? 384 : 256;
    }
    const CUtensorMap mb = make_map(g.bt, g.k, g.n, g.k, BK, static_cast<uint32_t>(tn == 384 ? 64 : tn / 2));
    const int64_t tiles = mt * ((g.n + tn - 1) / tn);
    int splits = tn == 256 && g.epi != 2 && g.epi != 4 ? gemm_splitk_splits(g.m, g.n, g.k, g.max_ctas) : 1;
    float4* ws = nullptr;
    int* sem = nullptr;
    if (splits > 1) {
      const size_t need = gemm_splitk_workspace(g.m, g.n, g.k, g.max_ctas);
      if (g.ws == nullptr || g.ws_bytes < need || (reinterpret_cast<uintptr_t>(g.ws) % 16) != 0) {
        splits = 1;  // direct launches without an engine workspace
      } else {
        ws = static_cast<float4*>(g.ws);
        sem = reinterpret_cast<int*>(static_cast<char*>(g.ws) + need - static_cast<size_t>(tiles * 16) * sizeof(int));
        // semaphores start at zero (the last arriver re-zeroes its own)
        OPF_CUDA(cudaMemsetAsync(sem, 0, static_cast<size_t>(tiles * 16) * sizeof(int), s));
      }
    }
    const int clusters = static_cast<int>(std::min<int64_t>(tiles * splits, cmax));
    const dim3 blocks(2u * static_cast<unsigned>(std::max(clusters, 1)));
    if (splits > 1 && g.epi == 1)
      launch_pdl(gemm_tc2_kernel<1, 256, true>, blocks, dim3(Tc2Cfg<256, true>::kThreads), Tc2Cfg<256, true>::kSmemBytes, s, ma, mb, mc,
                 g.m, g.n, g.k, splits, ws, sem, rope, static_cast<__nv_bfloat16*>(g.c), g.ldc, kNoPush);
    else if (splits > 1)
      launch_pdl(gemm_tc2_kernel<0, 256, true>, blocks, dim3(Tc2Cfg<256, true>::kThreads), Tc2Cfg<256, true>::kSmemBytes, s, ma, mb, mc,
                 g.m, g.n, g.k, splits, ws, sem, rope, static_cast<__nv_bfloat16*>(g.c), g.ldc, kNoPush);
    else if (g.epi == 4)
      launch_pdl(gemm_tc2_kernel<4, 256>, blocks, dim3(Tc2Cfg<256, false>::kThreads), Tc2Cfg<256, false>::kSmemBytes, s, ma, mb,
                 mc, g.m, g.n, g.k, 1, ws, sem, rope, static_cast<__nv_bfloat16*>(g.c), g.ldc, kNoPush);
    else if (g.epi == 2 && tn == 384)
      launch_pdl(gemm_tc2_kernel<2, 384>, blocks, dim3(Tc2Cfg<384, false>::kThreads), Tc2Cfg<384, false>::kSmemBytes, s, ma, mb,
                 mc, g.m, g.n, g.k, 1, ws, sem, rope, static_cast<__nv_bfloat16*>(g.c), g.ldc, kNoPush);
    else if (g.epi == 2)
      launch_pdl(gemm_tc2_kernel<2, 256>, blocks, dim3(Tc2Cfg<256, false>::kThreads), Tc2Cfg<256, false>::kSmemBytes, s, ma, mb,
                 mc, g.m, g.n, g.k, 1, ws, sem, rope, static_cast<__nv_bfloat16*>(g.c), g.ldc, kNoPush);
    else if (g.epi == 1)
      launch_pdl(gemm_tc2_kernel<1, 256>, blocks, dim3(Tc2Cfg<256, false>::kThreads), Tc2Cfg<256, false>::kSmemBytes, s, ma, mb, mc, g.m,
                 g.n, g.k, splits, ws, sem, rope, static_cast<__nv_bfloat16*>(g.c), g.ldc, kNoPush);
    else if (tn == 256)
      launch_pdl(gemm_tc2_kernel<0, 256>, blocks, dim3(Tc2Cfg<256, false>::kThreads), Tc2Cfg<256, false>::kSmemBytes, s, ma, mb, mc, g.m,
                 g.n, g.k, splits, ws, sem, rope, static_cast<__nv_bfloat16*>(g.c), g.ldc, kNoPush);
    else
      launch_pdl(gemm_tc2_kernel<0, 384>, blocks, dim3(Tc2Cfg<384, false>::kThreads), Tc2Cfg<384, false>::kSmemBytes, s, ma, mb, mc, g.m,
                 g.n, g.k, 1, ws, sem, rope, static_cast<__nv_bfloat16*>(g.c), g.ldc, kNoPush);
    return;
  }
  const CUtensorMap mb = make_map(g.bt, g.k, g.n, g.k, BK, BN);
  const int64_t tiles = ((g.m + BM - 1) / BM) * ((g.n + BN - 1) / BN);
  if (tiles < grid) grid = static_cast<int>(tiles);
  if (g.epi == 2)
    launch_pdl(gemm_tc_kernel<2>, dim3(grid), dim3(kThreads), kSmemBytes, s, ma, mb, mc, g.m, g.n, g.k,
               static_cast<const int32_t*>(nullptr), static_cast<__nv_bfloat16*>(nullptr), int64_t{0}, rope);
  else if (g.epi == 1)
    launch_pdl(gemm_tc_kernel<1>, dim3(grid), dim3(kThreads), kSmemBytes, s, ma, mb, mc, g.m, g.n, g.k,
               static_cast<const int32_t*>(nullptr), static_cast<__nv_bfloat16*>(nullptr), int64_t{0}, rope);
  else
    launch_pdl(gemm_tc_kernel<0>, dim3(grid), dim3(kThreads), kSmemBytes, s, ma, mb, mc, g.m, g.n, g.k,
               static_cast<const int32_t*>(nullptr), static_cast<__nv_bfloat16*>(nullptr), int64_t{0}, rope);
}

// Row-parallel GEMM whose epilogue pushes each 32-row slab of the partial
// product into its owner rank's peer window (EPI 3, store_tile_push).  2-CTA
// 256x256 tiles only; the caller checks m % (32 * world) == 0 and n % 256 == 0.
void gemm_bf16_push(const GemmArgs& g, const PushArgs& p, cudaStream_t s) {
  require(g.k % 8 == 0 && g.lda % 8 == 0 && g.n % 256 == 0 && p.blk % 32 == 0 && g.m > BM, Errc::ShapeMismatch,
          "push GEMM needs K % 8, N % 256, 32-row owner blocks and M > 128");
  gemm_bf16_tc_init();
  static std::once_flag once;
  std::call_once(once, [] {
    OPF_CUDA(cudaFuncSetAttribute(gemm_tc2_kernel<3, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(Tc2Cfg<256, false>::kSmemBytes)));
  });
  const CUtensorMap ma = make_map(g.a, g.k, g.m, g.lda, BK, BM);
  const CUtensorMap mb = make_map(g.bt, g.k, g.n, g.k, BK, 128);
  int grid = num_sms();
  if (g.max_ctas > 0 && g.max_ctas < grid) grid = g.max_ctas;
  const int64_t tiles = ((g.m + 2 * BM - 1) / (2 * BM)) * (g.n / 256);
  const int clusters = static_cast<int>(std::min<int64_t>(tiles, std::max(grid / 2, 1)));
  launch_pdl(gemm_tc2_kernel<3, 256>, dim3(2u * static_cast<unsigned>(std::max(clusters, 1))),
             dim3(Tc2Cfg<256, false>::kThreads), Tc2Cfg<256, false>::kSmemBytes, s, ma, mb, ma, g.m, g.n, g.k, 1,
             static_cast<float4*>(nullptr), static_cast<int*>(nullptr), RopeArgs{}, kNoOut, int64_t{0}, p);
}

// Grouped (per-expert) GEMM: rows of `a` are expert-sorted segments, gtab the
// device tile table built by the routing kernel, bt = [E * group_n, K] packed
// expert weights.  max_mtiles bounds the tile count (grid sizing happens on the
// host; the actual count is read on the device, so the launch is capturable).
int moe_tile_m() { return BM; }  // 128-row expert tiles: the 1-SM grouped kernel

void gemm_bf16_grouped(const GemmArgs& g, const int32_t* gtab, int64_t max_mtiles, int64_t group_n,
                       int64_t n_groups, cudaStream_t s) {
  require(g.k % 8 == 0 && g.lda % 8 == 0 && g.ldc % 8 == 0 && group_n % BN == 0, Errc::ShapeMismatch,
          "grouped GEMM needs K, lda, ldc multiples of 8 and a per-expert N multiple of 256");
  gemm_bf16_tc_init();
  auto* c = static_cast<__nv_bfloat16*>(g.c);
  const CUtensorMap ma = make_map(g.a, g.k, g.m, g.lda, BK, BM);
  const CUtensorMap mc = make_map(g.c, g.epi == 1 ? group_n / 2 : group_n, g.m, g.ldc, 64, 32);
  int grid = num_sms();
  if (g.max_ctas > 0 && g.max_ctas < grid) grid = g.max_ctas;
  const int64_t tiles = max_mtiles * (group_n / BN);
  const CUtensorMap mb = make_map(g.bt, g.k, group_n * n_groups, g.k, BK, BN);
  if (tiles < grid) grid = static_cast<int>(std::max<int64_t>(tiles, 1));
  if (g.epi == 1)
    launch_pdl(gemm_tc_kernel<1, true>, dim3(grid), dim3(kThreads), kSmemBytes, s, ma, mb, mc, g.m, group_n, g.k,
               gtab, c, g.ldc, RopeArgs{});
  else
    launch_pdl(gemm_tc_kernel<0, true>, dim3(grid), dim3(kThreads), kSmemBytes, s, ma, mb, mc, g.m, group_n, g.k,
               gtab, c, g.ldc, RopeArgs{});
}

// [K, 2I] gate|up weight -> K-major [2I, K] with gate/up interleaved in 128-row
// blocks (rows 256b..256b+127 = gate block b, +128..+255 = up block b), the
// layout the SiLU-mul epilogue consumes.
__global__ void pack_gate_up_kernel(const __nv_bfloat16* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                    int64_t K, int64_t I) {
  __shared__ __nv_bfloat16 tile[32][33];
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 32, r0 = static_cast<int64_t>(blockIdx.y) * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    if (r < K && c < 2 * I) tile[i][threadIdx.x] = src[r * 2 * I + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;  // source column c -> packed row
    if (r < K && c < 2 * I) {
      const bool up = c >= I;
      const int64_t j = up ? c - I : c;
      const int64_t prow = (j / 128) * 256 + (up ? 128 : 0) + j % 128;
      dst[prow * K + r] = tile[threadIdx.x][i];
    }
  }
}

void k_pack_gate_up(const void* src, void* dst, int64_t K, int64_t I, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>((2 * I + 31) / 32), static_cast<unsigned>((K + 31) / 32));
  pack_gate_up_kernel<<<grid, dim3(32, 8), 0, s>>>(static_cast<const __nv_bfloat16*>(src),
                                                   static_cast<__nv_bfloat16*>(dst), K, I);
}

}  // namespace opflow

#ifdef OPF_GEMM_TRACE
// tools/gemm_trace.py: read (and reset) the trace buffers of the last launch
extern "C" int opf_debug_gemm_trace(unsigned long long* out, int* counts) {
  if (cudaMemcpyFromSymbol(out, opflow::g_gemm_trace, sizeof(opflow::g_gemm_trace)) != cudaSuccess) return 1;
  if (cudaMemcpyFromSymbol(counts, opflow::g_gemm_trace_n, sizeof(opflow::g_gemm_trace_n)) != cudaSuccess) return 1;
  const int zero[3] = {0, 0, 0};
  return cudaMemcpyToSymbol(opflow::g_gemm_trace_n, zero, sizeof(zero)) == cudaSuccess ? 0 : 1;
}
#endif
