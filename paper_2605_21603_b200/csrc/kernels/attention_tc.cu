// Causal GQA prefill attention on tensor cores (flash-attention style):
// bf16 in, fp32 online softmax, bf16 out, for qkv rows laid out
// [rows, (nq + 2 nkv) * 128] with fixed-length sequences (seq_len | rows).
//
// One CTA = 128 query rows of one (sequence, q head); 8 warps x 16 rows.
// K/V tiles of 64 keys stream through a double-buffered, XOR-swizzled shared
// memory ring (cp.async 16 B), fragments come from ldmatrix (.trans for V),
// S = Q K^T and O += P V use mma.sync m16n8k16 (bf16, fp32 accumulate); P
// never leaves registers (the S accumulator layout is reused as the A
// fragment of the PV product).  Causal: a query tile reads keys up to its
// last row; only the two diagonal key tiles are masked.  Q tiles are issued
// longest-first so the causal triangle load-balances across the 148 SMs.
// FLOPs per (sequence, q head) = 4 * S^2/2 * 128 (2*S^2*hd for QK^T and PV).
#include <cuda_bf16.h>

#include <cfloat>

#include "opflow/device.hpp"

namespace opflow {

namespace {

constexpr int HD = 128;
constexpr int BQ = 128;
constexpr int BKV = 64;
constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kRowBytes = HD * 2;  // 256 B per row in smem (16 chunks of 16 B)
constexpr int kQBytes = BQ * kRowBytes;
constexpr int kKVBytes = BKV * kRowBytes;
constexpr int kSmem = kQBytes + 4 * kKVBytes;  // Q + 2 x (K, V)

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// byte offset of 16-byte chunk `c` of row `r` (XOR swizzle within 8-chunk groups)
__device__ __forceinline__ uint32_t swz(int r, int c) {
  return static_cast<uint32_t>(r * kRowBytes + ((c ^ (r & 7)) << 4));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// load `nrows` rows (128 bf16 each) starting at global row pointer base (row stride ld elems)
__device__ __forceinline__ void load_tile(uint8_t* sm, const __nv_bfloat16* g, int64_t ld, int nrows,
                                          int valid_rows) {
  const uint32_t s0 = smem_addr(sm);
  for (int i = threadIdx.x; i < nrows * 16; i += kThreads) {
    const int r = i >> 4, c = i & 15;
    if (r < valid_rows) {
      cp_async16(s0 + swz(r, c), g + static_cast<int64_t>(r) * ld + c * 8);
    } else {
      *reinterpret_cast<uint4*>(sm + swz(r, c)) = make_uint4(0, 0, 0, 0);
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    fa_prefill_kernel(const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* __restrict__ out,
                      int nq, int nkv, int S, int q_tiles, float scale_log2) {
  extern __shared__ __align__(128) uint8_t smem[];
  pdl_wait();
  pdl_trigger();
  uint8_t* sQ = smem;
  uint8_t* sK[2] = {smem + kQBytes, smem + kQBytes + 2 * kKVBytes};
  uint8_t* sV[2] = {smem + kQBytes + kKVBytes, smem + kQBytes + 3 * kKVBytes};

  // longest causal tiles first: blockIdx.x -> (q tile descending, head, sequence)
  const int per_tile = nq * (gridDim.x / (q_tiles * nq));
  const int qt = q_tiles - 1 - static_cast<int>(blockIdx.x) / per_tile;
  const int rem = static_cast<int>(blockIdx.x) % per_tile;
  const int h = rem % nq;
  const int seq = rem / nq;
  const int kh = h / (nq / nkv);
  const int64_t W = static_cast<int64_t>(nq + 2 * nkv) * HD;
  const int64_t row0 = static_cast<int64_t>(seq) * S;
  const int q0 = qt * BQ;
  const int q_valid = min(BQ, S - q0);
  const __nv_bfloat16* gQ = qkv + (row0 + q0) * W + static_cast<int64_t>(h) * HD;
  const __nv_bfloat16* gK = qkv + row0 * W + static_cast<int64_t>(nq + kh) * HD;
  const __nv_bfloat16* gV = qkv + row0 * W + static_cast<int64_t>(nq + nkv + kh) * HD;

  const int kv_end = q0 + q_valid;  // causal: keys [0, kv_end)
  const int n_tiles = (kv_end + BKV - 1) / BKV;

  load_tile(sQ, gQ, W, BQ, q_valid);
  load_tile(sK[0], gK, W, BKV, min(BKV, kv_end));
  load_tile(sV[0], gV, W, BKV, min(BKV, kv_end));
  cp_commit();

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int g = lane >> 2, t = lane & 3;
  const int wrow = warp * 16;  // this warp's first query row in the tile

  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.0f;
  float m_r[2] = {-FLT_MAX, -FLT_MAX}, l_r[2] = {0.0f, 0.0f};
  uint32_t qf[8][4];

  for (int j = 0; j < n_tiles; ++j) {
    const int buf = j & 1;
    if (j + 1 < n_tiles) {
      const int k1 = (j + 1) * BKV;
      load_tile(sK[buf ^ 1], gK + static_cast<int64_t>(k1) * W, W, BKV, min(BKV, kv_end - k1));
      load_tile(sV[buf ^ 1], gV + static_cast<int64_t>(k1) * W, W, BKV, min(BKV, kv_end - k1));
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    if (j == 0) {  // Q fragments into registers once
      const uint32_t qb = smem_addr(sQ);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int r = wrow + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = kk * 2 + (lane >> 4);
        ldsm_x4(qb + swz(r, c), qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
      }
    }
    // ---- S = Q K^T (16 x 64 per warp)
    float s[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.0f;
    const uint32_t kb = smem_addr(sK[buf]);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {  // pairs of 8-key n-tiles
        uint32_t b0, b1, b2, b3;
        const int r = np * 16 + (lane & 7) + (lane >> 4) * 8;
        const int c = kk * 2 + ((lane >> 3) & 1);
        ldsm_x4(kb + swz(r, c), b0, b1, b2, b3);
        mma16816(s[2 * np], qf[kk], b0, b1);
        mma16816(s[2 * np + 1], qf[kk], b2, b3);
      }
    }
    // ---- causal mask on diagonal tiles, online softmax
    const int kbase = j * BKV;
    const bool diag = kbase + BKV > q0;
    float mx[2] = {m_r[0], m_r[1]};
#pragma unroll
    for (int n = 0; n < 8; ++n) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int qi = q0 + wrow + g + (e >> 1) * 8;
        const int kj = kbase + n * 8 + 2 * t + (e & 1);
        float v = s[n][e] * scale_log2;
        if ((diag && kj > qi) || kj >= kv_end) v = -FLT_MAX;
        s[n][e] = v;
        mx[e >> 1] = fmaxf(mx[e >> 1], v);
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
    }
    float corr[2], rs[2] = {0.0f, 0.0f};
#pragma unroll
    for (int r = 0; r < 2; ++r) corr[r] = exp2f(m_r[r] - mx[r]);
    uint32_t pf[4][4];  // P as A fragments for the 4 k-steps of P V
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      float p[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        p[e] = exp2f(s[n][e] - mx[e >> 1]);
        rs[e >> 1] += p[e];
      }
      const int kk = n >> 1;
      if ((n & 1) == 0) {
        pf[kk][0] = pack2(p[0], p[1]);
        pf[kk][1] = pack2(p[2], p[3]);
      } else {
        pf[kk][2] = pack2(p[0], p[1]);
        pf[kk][3] = pack2(p[2], p[3]);
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      l_r[r] = l_r[r] * corr[r] + rs[r];
      m_r[r] = mx[r];
    }
#pragma unroll
    for (int d = 0; d < 16; ++d) {
      o[d][0] *= corr[0];
      o[d][1] *= corr[0];
      o[d][2] *= corr[1];
      o[d][3] *= corr[1];
    }
    // ---- O += P V  (V tile 64 keys x 128 dims; B fragments via ldmatrix.trans)
    const uint32_t vb = smem_addr(sV[buf]);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
      for (int dp = 0; dp < 8; ++dp) {  // pairs of 8-dim n-tiles
        uint32_t b0, b1, b2, b3;
        const int r = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = dp * 2 + (lane >> 4);
        ldsm_x4_t(vb + swz(r, c), b0, b1, b2, b3);
        mma16816(o[2 * dp], pf[kk], b0, b1);
        mma16816(o[2 * dp + 1], pf[kk], b2, b3);
      }
    }
    __syncthreads();  // this buffer is refilled two iterations later
  }
  // ---- finalize: reduce row sums across the quad, normalise, store bf16
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 1);
    l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 2);
    l_r[r] = l_r[r] > 0.0f ? 1.0f / l_r[r] : 0.0f;
  }
  const int64_t ldo = static_cast<int64_t>(nq) * HD;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int qi = wrow + g + r * 8;
    if (qi >= q_valid) continue;
    __nv_bfloat16* orow = out + (row0 + q0 + qi) * ldo + static_cast<int64_t>(h) * HD;
#pragma unroll
    for (int d = 0; d < 16; ++d) {
      const uint32_t v = pack2(o[d][2 * r] * l_r[r], o[d][2 * r + 1] * l_r[r]);
      *reinterpret_cast<uint32_t*>(orow + d * 8 + 2 * t) = v;
    }
  }
}

}  // namespace

bool prefill_bf16_tc(const __nv_bfloat16* qkv, __nv_bfloat16* out, int64_t rows, int nq, int nkv,
                     int hd, int S, float scale, cudaStream_t s) {
  if (hd != HD || nq % nkv != 0 || S < 1 || rows % S != 0) return false;
  if (reinterpret_cast<uintptr_t>(qkv) % 16 || reinterpret_cast<uintptr_t>(out) % 16) return false;
  static bool attr = [] {
    return cudaFuncSetAttribute(fa_prefill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kSmem) == cudaSuccess;
  }();
  if (!attr) return false;
  const int n_seqs = static_cast<int>(rows / S);
  const int q_tiles = (S + BQ - 1) / BQ;
  const unsigned grid = static_cast<unsigned>(q_tiles * nq * n_seqs);
  const float scale_log2 = scale * 1.4426950408889634f;
  launch_pdl(fa_prefill_kernel, dim3(grid), dim3(kThreads), kSmem, s, qkv, out, nq, nkv, S, q_tiles,
             scale_log2);
  return true;
}

}  // namespace opflow
