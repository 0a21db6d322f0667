// Causal GQA prefill attention on tcgen05 / TMEM (head_dim 128, seq_len % 128 == 0).
//
// Persistent CTAs (one per SM, 224 KB smem) walk (q-tile, head, sequence)
// items longest-first.  Per item (128 query rows of one head):
//   warp 0  TMA: Q tile once; K_j, V_j tiles (128 keys x 128 dims, two 64-dim
//           128B-swizzled halves each) into a 2-stage ring.  One tensor map over
//           the whole qkv buffer serves Q, K and V (column = head * 128).
//   warp 1  MMA (one thread): S_j = Q K_j^T -> TMEM S[j % 2] (M=N=K=128, both
//           operands K-major); O += P_j V_j -> TMEM O (A = P from smem,
//           B = V MN-major: LBO = 16 KB between the 64-dim halves, SBO = 1 KB).
//           Issue order S_0, S_1, PV_0, S_2, PV_1, ... keeps the tensor pipe
//           busy with PV_{j-1} + S_{j+1} while the softmax of S_j runs.
//   warp 2  completion tracker: waits every PV commit in order and publishes a
//           running count in smem (softmax warps read it before touching O or
//           overwriting a P buffer).
//   warps 4..7  softmax: thread = one query row (TMEM lane), whole 128-key row
//           in registers (tcgen05.ld 32x32b), row max / exp2 / sum without
//           shuffles, causal mask on the diagonal tile, P (bf16) written to a
//           double-buffered K-major SW128 smem tile.  Lazy rescaling: the
//           exponent base m only moves when the row max grows by > 8 (log2), then
//           O (TMEM) and l are rescaled; final O / l in the epilogue.
// FLOPs per item = 4 * 128 * 128 * 128 * (#key tiles) (diagonal tile half-masked).
#include <cuda.h>
#include <cuda_bf16.h>

#include <cfloat>
#include <mutex>

#include "opflow/device.hpp"

namespace opflow {

namespace {

constexpr int HD = 128, BQ = 128, BKV = 128;
constexpr int kThreads = 256;
constexpr uint32_t kHalf = 128 * 64 * 2;   // 16 KB: 128 rows x 64 bf16 (one swizzled half)
constexpr uint32_t kTile = 2 * kHalf;      // 32 KB: 128 rows x 128 bf16
constexpr int kStages = 2;
constexpr uint32_t kSmemQ = 0;
constexpr uint32_t kSmemK = kTile;                      // [kStages]
constexpr uint32_t kSmemV = kSmemK + kStages * kTile;   // [kStages]
constexpr uint32_t kSmemP = kSmemV + kStages * kTile;   // [2]
constexpr uint32_t kSmemBar = kSmemP + 2 * kTile;
constexpr uint32_t kSmemTotal = kSmemBar + 256 + 1024;  // + barriers + alignment slack
constexpr float kRescaleThresh = 8.0f;  // log2 units

// kind::f16, D f32, A/B bf16, M=128, N=128; b_mn: B operand MN-major
constexpr uint32_t idesc(bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn ? 1u : 0u) << 16) | ((128u >> 3) << 17) |
         ((128u >> 4) << 24);
}

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra W_%=;\n\t}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(su32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// smem matrix descriptor, 128B swizzle, version 1
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFF) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b))
               : "memory");
}
__device__ __forceinline__ void tld32(uint32_t a, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(a));
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tst32(uint32_t a, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31, %32};" ::"r"(a),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])),
      "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])),
      "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
      "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])),
      "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])),
      "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
      : "memory");
}
__device__ __forceinline__ uint32_t bf2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void __launch_bounds__(kThreads, 1)
    fa_tc_kernel(const __grid_constant__ CUtensorMap mqkv, __nv_bfloat16* __restrict__ out, int nq,
                 int nkv, int S, int n_seqs, float scale_log2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + kSmemBar);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;   // [2]
  uint64_t* v_full = bars + 4;   // [2]
  uint64_t* kv_empty = bars + 6; // [2]
  uint64_t* s_full = bars + 8;   // [2]
  uint64_t* s_free = bars + 10;  // [2]
  uint64_t* p_full = bars + 12;  // [2]
  uint64_t* o_done = bars + 14;  // one phase per PV
  uint64_t* o_free = bars + 15;  // epilogue finished reading O
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);
  volatile uint32_t* pv_count = reinterpret_cast<volatile uint32_t*>(bars + 17);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int q_tiles = S / BQ;
  const int64_t per_q = static_cast<int64_t>(nq) * n_seqs;
  const int64_t n_items = per_q * q_tiles;
  const int grp = nq / nkv;
  const int W = (nq + 2 * nkv) * HD;  // qkv row width (elements)

  if (warp == 0) {
    if (lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mqkv)) : "memory");
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  } else if (warp == 1 && lane == 0) {
    bar_init(q_full, 1);
    bar_init(q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      bar_init(&k_full[i], 1);
      bar_init(&v_full[i], 1);
      bar_init(&kv_empty[i], 1);
      bar_init(&s_full[i], 1);
      bar_init(&s_free[i], 4);
      bar_init(&p_full[i], 4);
    }
    bar_init(o_done, 1);
    bar_init(o_free, 4);
    *pv_count = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;  // S[0] cols 0..127, S[1] 128..255, O 256..383
  pdl_wait();
  pdl_trigger();

  auto decode_item = [&](int64_t i, int& qt, int& h, int& seq) {
    qt = q_tiles - 1 - static_cast<int>(i / per_q);  // longest (most key tiles) first
    const int64_t r = i % per_q;
    h = static_cast<int>(r % nq);
    seq = static_cast<int>(r / nq);
  };

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ TMA producer
      int stage = 0;
      uint32_t ph = 0, qph = 0;
      for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
        int qt, h, seq;
        decode_item(it, qt, h, seq);
        const int kh = h / grp;
        const int row0 = seq * S;
        bar_wait(q_empty, qph ^ 1);
        qph ^= 1;
        bar_expect(q_full, kTile);
        tma2d(su32(sm + kSmemQ), &mqkv, q_full, h * HD, row0 + qt * BQ);
        tma2d(su32(sm + kSmemQ + kHalf), &mqkv, q_full, h * HD + 64, row0 + qt * BQ);
        for (int j = 0; j <= qt; ++j) {
          bar_wait(&kv_empty[stage], ph ^ 1);
          const uint32_t kd = su32(sm + kSmemK + stage * kTile), vd = su32(sm + kSmemV + stage * kTile);
          bar_expect(&k_full[stage], kTile);
          tma2d(kd, &mqkv, &k_full[stage], (nq + kh) * HD, row0 + j * BKV);
          tma2d(kd + kHalf, &mqkv, &k_full[stage], (nq + kh) * HD + 64, row0 + j * BKV);
          bar_expect(&v_full[stage], kTile);
          tma2d(vd, &mqkv, &v_full[stage], (nq + nkv + kh) * HD, row0 + j * BKV);
          tma2d(vd + kHalf, &mqkv, &v_full[stage], (nq + nkv + kh) * HD + 64, row0 + j * BKV);
          if (++stage == kStages) {
            stage = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------------ MMA issuer
      int stage = 0;
      uint32_t ph = 0, qph = 0, ofree_ph = 0;
      uint32_t sfree_ph[2] = {0, 0}, pfull_ph[2] = {0, 0};
      int sbuf_uses[2] = {0, 0};
      bool first_item = true;
      const uint32_t S_id = idesc(false), PV_id = idesc(true);
      const uint32_t qa = su32(sm + kSmemQ);
      for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
        int qt, h, seq;
        decode_item(it, qt, h, seq);
        const int n = qt + 1;
        bar_wait(q_full, qph);
        qph ^= 1;
        int pv_stage = stage;
        uint32_t pv_ph = ph;
        auto issue_pv = [&](int j) {
          const int b = j & 1;
          bar_wait(&p_full[b], pfull_ph[b]);
          pfull_ph[b] ^= 1;
          bar_wait(&v_full[pv_stage], pv_ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t pa = su32(sm + kSmemP + b * kTile);
          const uint32_t vb = su32(sm + kSmemV + pv_stage * kTile);
#pragma unroll
          for (int k = 0; k < 8; ++k) {  // 16 keys per step
            const uint64_t ad = sdesc(pa + (k >> 2) * kHalf + (k & 3) * 32, 16, 1024);
            const uint64_t bd = sdesc(vb + k * 2048, kHalf, 1024);
            mma_ss(tmem + 256, ad, bd, PV_id, (j | k) != 0);
          }
          commit(&kv_empty[pv_stage]);
          commit(o_done);
          if (++pv_stage == kStages) {
            pv_stage = 0;
            pv_ph ^= 1;
          }
        };
        for (int j = 0; j < n; ++j) {
          const int b = j & 1;
          if (sbuf_uses[b]++ > 0) {  // S buffer b last held S_{j-2}: softmax must be done reading
            bar_wait(&s_free[b], sfree_ph[b]);
            sfree_ph[b] ^= 1;
          }
          bar_wait(&k_full[stage], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t kb = su32(sm + kSmemK + stage * kTile);
#pragma unroll
          for (int k = 0; k < 8; ++k) {  // 16 dims per step
            const uint64_t ad = sdesc(qa + (k >> 2) * kHalf + (k & 3) * 32, 16, 1024);
            const uint64_t bd = sdesc(kb + (k >> 2) * kHalf + (k & 3) * 32, 16, 1024);
            mma_ss(tmem + b * 128, ad, bd, S_id, k != 0);
          }
          commit(&s_full[b]);
          if (++stage == kStages) {
            stage = 0;
            ph ^= 1;
          }
          if (j == n - 1) commit(q_empty);
          if (j >= 1) {
            if (j == 1 && !first_item) {  // O of the previous item must be drained first
              bar_wait(o_free, ofree_ph);
              ofree_ph ^= 1;
            }
            issue_pv(j - 1);
          }
        }
        if (n == 1 && !first_item) {
          bar_wait(o_free, ofree_ph);
          ofree_ph ^= 1;
        }
        issue_pv(n - 1);
        first_item = false;
      }
    }
  } else if (warp == 2) {
    if (lane == 0) {  // ------------------------------------------------ PV completion tracker
      uint32_t oph = 0, count = 0;
      for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
        int qt, h, seq;
        decode_item(it, qt, h, seq);
        for (int j = 0; j <= qt; ++j) {
          bar_wait(o_done, oph);
          oph ^= 1;
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          *pv_count = ++count;
          __threadfence_block();
        }
      }
    }
  } else if (warp >= 4) {  // ---------------------------------------- softmax / epilogue
    const int q = warp & 3;          // TMEM lane quarter
    const int r = q * 32 + lane;     // query row within the tile
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(q * 32) << 16);
    uint32_t sfull_ph[2] = {0, 0};
    uint32_t pv_seen = 0;  // PV count at the start of this item
    for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
      int qt, h, seq;
      decode_item(it, qt, h, seq);
      const int n = qt + 1;
      float m_used = -FLT_MAX, l = 0.0f;
      for (int j = 0; j < n; ++j) {
        const int b = j & 1;
        bar_wait(&s_full[b], sfull_ph[b]);
        sfull_ph[b] ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        float s[128];
#pragma unroll
        for (int c = 0; c < 4; ++c) tld32(lane_base + b * 128 + c * 32, *reinterpret_cast<float(*)[32]>(&s[c * 32]));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) bar_arrive(&s_free[b]);
        // scale, causal mask (diagonal tile only), row max
        const bool diag = j == qt;
        float mx = -FLT_MAX;
#pragma unroll
        for (int c = 0; c < 128; ++c) {
          float v = s[c] * scale_log2;
          if (diag && c > r) v = -FLT_MAX;
          s[c] = v;
          mx = fmaxf(mx, v);
        }
        // lazy rescale of the exponent base
        float factor = 1.0f;
        const bool rescale = mx > m_used + kRescaleThresh;
        if (rescale) {
          factor = ex2(m_used - mx);  // 0 on the first tile
          m_used = mx;
        }
        l *= factor;
        float sum = 0.0f;
        // P buffer b was last read by PV_{j-2}
        if (j >= 2)
          while (*pv_count < pv_seen + static_cast<uint32_t>(j - 1)) {
          }
        uint8_t* pbuf = sm + kSmemP + b * kTile;
#pragma unroll
        for (int c8 = 0; c8 < 16; ++c8) {
          float p[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            p[e] = ex2(s[c8 * 8 + e] - m_used);
            sum += p[e];
          }
          const int half = c8 >> 3, chunk = c8 & 7;
          uint4 u;
          u.x = bf2(p[0], p[1]);
          u.y = bf2(p[2], p[3]);
          u.z = bf2(p[4], p[5]);
          u.w = bf2(p[6], p[7]);
          *reinterpret_cast<uint4*>(pbuf + half * kHalf + r * 128 + ((chunk ^ (r & 7)) << 4)) = u;
        }
        l += sum;
        // rescale O (TMEM) when any row of this warp moved its base (not on tile 0)
        if (j > 0 && __any_sync(0xffffffffu, rescale)) {
          while (*pv_count < pv_seen + static_cast<uint32_t>(j)) {  // PV_{j-1} complete
          }
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            float o[32];
            tld32(lane_base + 256 + c * 32, o);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] *= factor;
            tst32(lane_base + 256 + c * 32, o);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) bar_arrive(&p_full[b]);
      }
      // ---- epilogue: wait for the item's last PV, O / l -> bf16 -> global
      while (*pv_count < pv_seen + static_cast<uint32_t>(n)) {
      }
      pv_seen += n;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const float inv = l > 0.0f ? 1.0f / l : 0.0f;
      __nv_bfloat16* orow = out + (static_cast<int64_t>(seq) * S + qt * BQ + r) * (static_cast<int64_t>(nq) * HD) +
                            static_cast<int64_t>(h) * HD;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float o[32];
        tld32(lane_base + 256 + c * 32, o);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          uint4 u;
          u.x = bf2(o[v * 8 + 0] * inv, o[v * 8 + 1] * inv);
          u.y = bf2(o[v * 8 + 2] * inv, o[v * 8 + 3] * inv);
          u.z = bf2(o[v * 8 + 4] * inv, o[v * 8 + 5] * inv);
          u.w = bf2(o[v * 8 + 6] * inv, o[v * 8 + 7] * inv);
          *reinterpret_cast<uint4*>(orow + c * 32 + v * 8) = u;
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) bar_arrive(o_free);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

}  // namespace

bool prefill_bf16_tcgen05(const __nv_bfloat16* qkv, __nv_bfloat16* out, int64_t rows, int nq, int nkv,
                          int hd, int S, float scale, int max_ctas, cudaStream_t s) {
  if (hd != HD || S % BQ != 0 || nq % nkv != 0 || rows % S != 0) return false;
  if (reinterpret_cast<uintptr_t>(qkv) % 16 || reinterpret_cast<uintptr_t>(out) % 16) return false;
  static EncodeFn enc = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeFn>(nullptr);
    return reinterpret_cast<EncodeFn>(p);
  }();
  static bool attr = cudaFuncSetAttribute(fa_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(kSmemTotal)) == cudaSuccess;
  if (!enc || !attr) return false;
  const int64_t W = static_cast<int64_t>(nq + 2 * nkv) * HD;
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(W) * 2};
  const cuuint32_t box[2] = {64, 128};
  const cuuint32_t es[2] = {1, 1};
  if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<__nv_bfloat16*>(qkv), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  const int n_seqs = static_cast<int>(rows / S);
  const int64_t items = static_cast<int64_t>(S / BQ) * nq * n_seqs;
  int grid = max_ctas > 0 ? std::min(max_ctas, num_sms()) : num_sms();
  grid = static_cast<int>(std::min<int64_t>(grid, items));
  launch_pdl(fa_tc_kernel, dim3(grid), dim3(kThreads), kSmemTotal, s, m, out, nq, nkv, S, n_seqs,
             scale * 1.4426950408889634f);
  return true;
}

}  // namespace opflow
