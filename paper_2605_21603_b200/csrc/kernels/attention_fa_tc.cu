// Causal GQA prefill attention on tcgen05 / TMEM (head_dim 128, seq_len % 128 == 0).
//
// Persistent CTAs (one per SM, 224 KB smem) walk (q-tile, head, sequence)
// items longest-first.  Per item (128 query rows of one head):
//   warp 0  TMA: Q tile once, K_j tiles; warp 3 TMA: V_j tiles (128 keys x 128 dims,
//           two 64-dim 128B-swizzled halves each), separate 2-stage K and V rings
//           (K_j's slot frees when S_j retires, V_j's when PV_j retires).  One tensor map over
//           the whole qkv buffer serves Q, K and V (column = head * 128).
//   warp 1  MMA (one thread): S_j = Q K_j^T -> TMEM S[j % 2] (M=N=K=128, both
//           operands K-major); O += P_j V_j -> TMEM O (A = P from smem,
//           B = V MN-major: LBO = 16 KB between the 64-dim halves, SBO = 1 KB).
//           Issue order S_0, S_1, PV_0, S_2, PV_1, ... keeps the tensor pipe
//           busy with PV_{j-1} + S_{j+1} while the softmax of S_j runs.
//   warp 2  completion tracker: waits every PV commit in order and publishes a
//           running count in smem (softmax warps read it before touching O or
//           overwriting a P buffer).
//   warps 4..11 softmax: two warps per TMEM lane quarter, thread = one query
//           row x 64 key columns (tcgen05.ld 32x32b); causal mask on the diagonal
//           tile, row max halves exchanged through smem (64-thread named barrier),
//           exp2 with the scale folded into one FFMA, P (bf16) packed in registers
//           and stored to the single K-major SW128 P tile once PV_{j-1} retired.
//           Lazy rescaling: the exponent base m only moves when the row max grows
//           by > 8 (log2), then each half rescales its 64 O columns in TMEM;
//           final O / l (halves' sums exchanged) in the epilogue.
// FLOPs per item = 4 * 128 * 128 * 128 * (#key tiles) (diagonal tile half-masked).
#include <cuda.h>
#include <cuda_bf16.h>

#include <cfloat>
#include <cstdlib>
#include <mutex>
#include <string>

#include "opflow/device.hpp"

namespace opflow {

namespace {

constexpr int HD = 128, BQ = 128, BKV = 128;
constexpr int kThreads = 384;  // 4 role warps + 8 softmax warps
constexpr uint32_t kHalf = 128 * 64 * 2;   // 16 KB: 128 rows x 64 bf16 (one swizzled half)
constexpr uint32_t kTile = 2 * kHalf;      // 32 KB: 128 rows x 128 bf16
constexpr int kStages = 2;
constexpr uint32_t kSmemQ = 0;
constexpr uint32_t kSmemK = kTile;                      // [kStages]
constexpr uint32_t kSmemV = kSmemK + kStages * kTile;   // [kStages]
constexpr uint32_t kSmemBar = kSmemV + kStages * kTile;
// TMEM columns: S[0] 0..127, S[1] 128..255, O 256..383, P[0] 384..447, P[1] 448..511
constexpr uint32_t kColO = 256, kColP = 384;
constexpr uint32_t kSmemXch = kSmemBar + 256;           // row max / sum exchange [2][NP <= 4][128] f32
constexpr uint32_t kSmemTotal = kSmemXch + 4096 + 1024;  // + alignment slack
constexpr float kRescaleThresh = 8.0f;  // log2 units

// kind::f16, D f32, A/B bf16, M=128, N=128; b_mn: B operand MN-major
__host__ __device__ constexpr uint32_t idesc(bool b_mn) {
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
// 16-byte global store that does not allocate in L1 (the output epilogues)
__device__ __forceinline__ void st_na_v4(void* p, const uint32_t* w) {
  asm volatile("st.global.L1::no_allocate.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(w[0]), "r"(w[1]), "r"(w[2]),
               "r"(w[3])
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
// A operand from TMEM (P: lane = query row, 32-bit column = 2 consecutive bf16 keys)
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void tst32u(uint32_t a, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31, %32};" ::"r"(a),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
      "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
      "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tst16u(uint32_t a, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16};" ::"r"(a),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
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
__device__ __forceinline__ void st_release(uint32_t a, uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(uint32_t a) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
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
// 2^x on the FMA pipe: x = k + f (k = round(x) via the 1.5*2^23 magic add,
// f in [-0.5, 0.5]), 2^f by a cubic (max rel err ~1e-4, below bf16's 4e-3),
// 2^k added into the exponent bits.  x is clamped at -126 (result ~1e-38).
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -126.0f);
  const float t = x + 12582912.0f;
  const float f = x - (t - 12582912.0f);
  float p = fmaf(fmaf(fmaf(0.0555041086648216f, f, 0.2402264923172690f), f, 0.6931471805599453f), f, 1.0f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}
// packed fp32x2 FMA / add (sm_100 FFMA2 / FADD2): two softmax elements per instruction
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(r)
      : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)),
        "l"(*reinterpret_cast<uint64_t*>(&c)));
  return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  uint64_t r;
  asm("add.f32x2 %0, %1, %2;"
      : "=l"(r)
      : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)));
  return *reinterpret_cast<float2*>(&r);
}
#ifndef FA_POLY
#define FA_POLY 0  // measured: 8 of 32 pairs on the FMA pipe 128.0 us vs all-MUFU 125.3 us (one-head kernel)
#endif
constexpr int kPolyPairs = FA_POLY;  // of the 32 element pairs each softmax thread exponentiates

#ifdef FA_TRACE  // per-phase clock64 timeline of CTA 0 (tools/fa_trace.cu); compiled out otherwise
__device__ long long g_fa_trace[12][64];
#define FA_T(ev, j)                                       \
  do {                                                    \
    const int fa_j_ = (j);                                \
    if (blockIdx.x == 0 && fa_j_ < 64) g_fa_trace[ev][fa_j_] = clock64(); \
  } while (0)
#else
#define FA_T(ev, j) \
  do {              \
    (void)(j);      \
  } while (0)
#endif

// NP = column parts per query row: NP x 4 softmax warps, each thread owning
// one row x 128/NP key columns (NP = 2: 8 warps, the round-1 default; NP = 4:
// 16 warps with 32 columns each — more warps to hide the softmax latency chain).
template <int NP>
__global__ void __launch_bounds__(128 + NP * 128, 1)
    fa_tc_kernel(const __grid_constant__ CUtensorMap mqkv, __nv_bfloat16* __restrict__ out, int nq,
                 int nkv, int S, int n_seqs, float scale_log2) {
  constexpr int CP = 128 / NP;         // key (and O) columns per softmax thread
  constexpr int kSoftW = 4 * NP;       // softmax warps
  constexpr int kPoly = kPolyPairs * CP / 64;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + kSmemBar);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;   // [2]
  uint64_t* v_full = bars + 4;   // [2]
  uint64_t* k_empty = bars + 6;  // [2]  S_j retired (K slot free)
  uint64_t* v_empty = bars + 18; // [2]  PV_j retired (V slot free)
  uint64_t* s_full = bars + 8;   // [2]
  uint64_t* s_free = bars + 10;  // [2]
  // one barrier per P buffer: a fast softmax warp may store P_{j+1} before a
  // slow one stores P_j (S_{j+1} is already computed and P_{j+1} needs no PV
  // to retire when j + 1 < 2); with one barrier for both buffers its early
  // arrival completed P_j's phase and PV_j read a stale P quarter
  uint64_t* p_full = bars + 12;  // [2]
  uint64_t* o_done = bars + 14;  // one phase per PV
  uint64_t* o_free = bars + 15;  // epilogue finished reading O
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);
  volatile uint32_t* pv_count = reinterpret_cast<volatile uint32_t*>(bars + 17);
  const uint32_t pv_count_addr = su32(bars + 17);
  static_assert(20 * 8 <= 256, "barrier area");

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int q_tiles = S / BQ;
  const int64_t per_q = static_cast<int64_t>(nq) * n_seqs;
  const int64_t n_items = per_q * q_tiles;
  const int grp = nq / nkv;

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
      bar_init(&k_empty[i], 1);
      bar_init(&v_empty[i], 1);
      bar_init(&s_full[i], 1);
      bar_init(&s_free[i], kSoftW);
    }
    bar_init(&p_full[0], kSoftW);
    bar_init(&p_full[1], kSoftW);
    bar_init(o_done, 1);
    bar_init(o_free, kSoftW);
    *pv_count = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;  // S[0] cols 0..127, S[1] 128..255, O 256..383
  int tile_k = 0, tile_v = 0, tile_s = 0, tile_pv = 0, tile_sm = 0;  // trace indices
  (void)tile_k, (void)tile_v, (void)tile_s, (void)tile_pv, (void)tile_sm;
  pdl_wait();
  pdl_trigger();

  // Item order of this CTA: passes of gridDim.x items, longest first, walked
  // boustrophedon (even passes CTA c takes item c, odd passes item G-1-c), so
  // the CTA that got the longest item of one pass gets the shortest of the
  // next.  Plain round-robin left the busiest CTA 12 % above the mean at
  // 8 x 1024 tokens (35 vs 31.1 key tiles per head pair); this is within 3 %.
  auto snake_item = [&](int64_t k) -> int64_t {
    const int64_t G = gridDim.x, c = blockIdx.x;
    return k * G + ((k & 1) ? G - 1 - c : c);
  };
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
      for (int64_t kk = 0, it = snake_item(0); it < n_items; it = snake_item(++kk)) {
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
          bar_wait(&k_empty[stage], ph ^ 1);
          const uint32_t kd = su32(sm + kSmemK + stage * kTile);
          bar_expect(&k_full[stage], kTile);
          tma2d(kd, &mqkv, &k_full[stage], (nq + kh) * HD, row0 + j * BKV);
          tma2d(kd + kHalf, &mqkv, &k_full[stage], (nq + kh) * HD + 64, row0 + j * BKV);
          FA_T(0, tile_k++);
          if (++stage == kStages) {
            stage = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 3) {
    if (lane == 0) {  // ------------------------------------------------ TMA producer (V)
      int stage = 0;
      uint32_t ph = 0;
      for (int64_t kk = 0, it = snake_item(0); it < n_items; it = snake_item(++kk)) {
        int qt, h, seq;
        decode_item(it, qt, h, seq);
        const int kh = h / grp;
        const int row0 = seq * S;
        for (int j = 0; j <= qt; ++j) {
          bar_wait(&v_empty[stage], ph ^ 1);
          const uint32_t vd = su32(sm + kSmemV + stage * kTile);
          bar_expect(&v_full[stage], kTile);
          tma2d(vd, &mqkv, &v_full[stage], (nq + nkv + kh) * HD, row0 + j * BKV);
          tma2d(vd + kHalf, &mqkv, &v_full[stage], (nq + nkv + kh) * HD + 64, row0 + j * BKV);
          FA_T(1, tile_v++);
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
      uint32_t ph = 0, qph = 0, ofree_ph = 0, pfull_ph = 0;  // pfull_ph: per-P-buffer bits
      uint32_t sfree_ph = 0, sbuf_used = 0;  // per-S-buffer bits
      bool first_item = true;
      const uint32_t S_id = idesc(false), PV_id = idesc(true);
      const uint32_t qa = su32(sm + kSmemQ);
      for (int64_t kk = 0, it = snake_item(0); it < n_items; it = snake_item(++kk)) {
        int qt, h, seq;
        decode_item(it, qt, h, seq);
        const int n = qt + 1;
        bar_wait(q_full, qph);
        qph ^= 1;
        int pv_stage = stage;
        uint32_t pv_ph = ph;
        auto issue_pv = [&](int j) {
          bar_wait(&p_full[j & 1], (pfull_ph >> (j & 1)) & 1u);
          pfull_ph ^= 1u << (j & 1);
          bar_wait(&v_full[pv_stage], pv_ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t vb = su32(sm + kSmemV + pv_stage * kTile);
          const uint32_t pt = tmem + kColP + (j & 1) * 64;
#pragma unroll
          for (int k = 0; k < 8; ++k) {  // 16 keys (8 TMEM columns of P) per step
            const uint64_t bd = sdesc(vb + k * 2048, kHalf, 1024);
            mma_ts(tmem + kColO, pt + k * 8, bd, PV_id, (j | k) != 0);
          }
          commit(&v_empty[pv_stage]);
          commit(o_done);
          FA_T(3, tile_pv++);
          if (++pv_stage == kStages) {
            pv_stage = 0;
            pv_ph ^= 1;
          }
        };
        for (int j = 0; j < n; ++j) {
          const int b = j & 1;
          if (sbuf_used & (1u << b)) {  // S buffer b last held S_{j-2}: softmax must be done reading
            bar_wait(&s_free[b], (sfree_ph >> b) & 1u);
            sfree_ph ^= 1u << b;
          }
          sbuf_used |= 1u << b;
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
          FA_T(2, tile_s++);
          commit(&k_empty[stage]);
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
      for (int64_t kk = 0, it = snake_item(0); it < n_items; it = snake_item(++kk)) {
        int qt, h, seq;
        decode_item(it, qt, h, seq);
        for (int j = 0; j <= qt; ++j) {
          bar_wait(o_done, oph);
          oph ^= 1;
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          st_release(pv_count_addr, ++count);
          FA_T(4, static_cast<int>(count) - 1);
        }
      }
    }
  } else if (warp >= 4) {  // ---------------------------------------- softmax / epilogue
    // NP warps per TMEM lane quarter: part pt takes key columns pt*CP.. (and the
    // same O columns).  Row max / row sum parts meet in a double-buffered smem
    // exchange behind a per-quarter named barrier.
    const int q = warp & 3;             // TMEM lane quarter
    const int pt = (warp - 4) >> 2;     // column part
    const int r = q * 32 + lane;        // query row within the tile
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(q * 32) << 16) + pt * CP;   // S columns
    const uint32_t o_base = tmem + (static_cast<uint32_t>(q * 32) << 16) + kColO + pt * CP;
    const uint32_t p_base = tmem + (static_cast<uint32_t>(q * 32) << 16) + kColP + pt * (CP / 2);
    float* xch = reinterpret_cast<float*>(sm + kSmemXch);  // [2 parity][NP parts][128 rows]
    uint32_t xpar = 0;
    auto exchange = [&](float v, bool is_max) {  // reduction of v over the row's NP parts
      xch[(xpar * NP + pt) * 128 + r] = v;
      asm volatile("bar.sync %0, %1;" ::"r"(1 + q), "n"(NP * 32) : "memory");
      float acc = xch[(xpar * NP) * 128 + r];
#pragma unroll
      for (int o = 1; o < NP; ++o) {
        const float w = xch[(xpar * NP + o) * 128 + r];
        acc = is_max ? fmaxf(acc, w) : acc + w;
      }
      xpar ^= 1;
      return acc;
    };
    uint32_t sfull_ph = 0;  // per-S-buffer bits
    uint32_t pv_seen = 0;   // PV count at the start of this item
    for (int64_t kk = 0, it = snake_item(0); it < n_items; it = snake_item(++kk)) {
      int qt, h, seq;
      decode_item(it, qt, h, seq);
      const int n = qt + 1;
      float m_used = -FLT_MAX, l = 0.0f;  // m_used in scaled log2 units; l over this part
      for (int j = 0; j < n; ++j) {
        const int b = j & 1;
        bar_wait(&s_full[b], (sfull_ph >> b) & 1u);
        if (lane == 0 && warp == 4) FA_T(5, tile_sm);
        sfull_ph ^= 1u << b;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        float s[CP];
#pragma unroll
        for (int c = 0; c < CP / 32; ++c)
          tld32(lane_base + b * 128 + c * 32, *reinterpret_cast<float(*)[32]>(&s[c * 32]));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) bar_arrive(&s_free[b]);
        if (lane == 0 && warp == 4) FA_T(7, tile_sm);
        // causal mask (diagonal tile only) and row max on the raw scores; the
        // softmax scale folds into one FFMA per element below
        float mx8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) mx8[i] = -INFINITY;
        if (j == qt) {
#pragma unroll
          for (int c = 0; c < CP; ++c) {
            if (pt * CP + c > r) s[c] = -INFINITY;
            mx8[c & 7] = fmaxf(mx8[c & 7], s[c]);
          }
        } else {
#pragma unroll
          for (int c = 0; c < CP; ++c) mx8[c & 7] = fmaxf(mx8[c & 7], s[c]);
        }
        const float pm = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                               fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
        const float mx = scale_log2 * exchange(pm, true);  // identical in every part
        if (lane == 0 && warp == 4) FA_T(8, tile_sm);
        // lazy rescale of the exponent base (log2 units)
        float factor = 1.0f;
        const bool rescale = mx > m_used + kRescaleThresh;
        if (rescale) {
          factor = ex2(m_used - mx);  // 0 on the first tile
          m_used = mx;
        }
        l *= factor;
        float sum8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        uint32_t pk[CP / 2];  // P row part, packed bf16x2
#pragma unroll
        for (int c2 = 0; c2 < CP / 2; ++c2) {
          // FA4-style split: the first kPoly pairs use the FMA-pipe polynomial,
          // the rest MUFU ex2 (the pipes run concurrently)
          const float x0 = fmaf(s[2 * c2], scale_log2, -m_used), x1 = fmaf(s[2 * c2 + 1], scale_log2, -m_used);
          const float p0 = c2 < kPoly ? ex2_poly(x0) : ex2(x0);
          const float p1 = c2 < kPoly ? ex2_poly(x1) : ex2(x1);
          sum8[(2 * c2) & 7] += p0;
          sum8[(2 * c2 + 1) & 7] += p1;
          pk[c2] = bf2(p0, p1);
        }
        l += ((sum8[0] + sum8[1]) + (sum8[2] + sum8[3])) + ((sum8[4] + sum8[5]) + (sum8[6] + sum8[7]));
        if (lane == 0 && warp == 4) FA_T(9, tile_sm);
        // P buffer (j & 1) was last read by PV_{j-2}; O rescaling needs PV_{j-1} retired
        const bool any_rescale = j > 0 && __any_sync(0xffffffffu, rescale);
        const uint32_t need = any_rescale ? static_cast<uint32_t>(j) : (j >= 2 ? static_cast<uint32_t>(j - 1) : 0u);
        while (ld_acquire(pv_count_addr) < pv_seen + need) {
        }
        if (lane == 0 && warp == 4) FA_T(10, tile_sm);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (any_rescale) {  // this part's CP O columns
#pragma unroll
          for (int c = 0; c < CP / 32; ++c) {
            float o[32];
            tld32(o_base + c * 32, o);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] *= factor;
            tst32(o_base + c * 32, o);
          }
        }
        if constexpr (CP == 64)
          tst32u(p_base + (j & 1) * 64, pk);
        else
          tst16u(p_base + (j & 1) * 64, pk);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) bar_arrive(&p_full[j & 1]);
        if (lane == 0 && warp == 4) FA_T(6, tile_sm);
        ++tile_sm;
      }
      // ---- epilogue: wait for the item's last PV, O / l -> bf16 -> global
      const float l_all = exchange(l, false);
      while (ld_acquire(pv_count_addr) < pv_seen + static_cast<uint32_t>(n)) {
      }
      pv_seen += n;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const float inv = l_all > 0.0f ? 1.0f / l_all : 0.0f;
      __nv_bfloat16* orow = out + (static_cast<int64_t>(seq) * S + qt * BQ + r) * (static_cast<int64_t>(nq) * HD) +
                            static_cast<int64_t>(h) * HD + pt * CP;
      // 256-bit stores that do not allocate in L1 when the output base allows
      // (as in the two-head kernel)
      const bool out32 = (reinterpret_cast<uintptr_t>(out) & 31) == 0;
#pragma unroll
      for (int c = 0; c < CP / 32; ++c) {
        float o[32];
        tld32(o_base + c * 32, o);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          uint32_t w[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) w[e] = bf2(o[v * 16 + 2 * e] * inv, o[v * 16 + 2 * e + 1] * inv);
          if (out32) {
            asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(orow + c * 32 + v * 16),
                         "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                         : "memory");
          } else {
            st_na_v4(orow + c * 32 + v * 16, w);
            st_na_v4(orow + c * 32 + v * 16 + 8, w + 4);
          }
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

// ------------------------------------------------------------------ ping-pong variant
// Two heads of one GQA group per item (same q tile, same K_j / V_j tiles: one
// K/V load feeds two S and two PV MMAs).  TMEM: S0/P0 0..127, S1/P1 128..255,
// O0 256..383, O1 384..511.  Softmax warpgroup t (warps 4+4t..7+4t) owns head
// t: one thread = one query row x all 128 keys (two 64-column passes over
// TMEM, so no cross-warp exchange), P (bf16) written over the consumed S
// columns.  The MMA warp interleaves the two heads — S0_{j+1} / S1_{j+1} are
// issued right behind PV0_j / PV1_j — so one head's softmax overlaps the
// other head's tensor work (FA4's ping-pong).  A commit after S_t,j also
// covers PV_t,{j-1} (in-order tcgen05 completion), so the softmax may rescale
// O_t without a separate PV tracker.
constexpr int kPPThreads = 384;                  // 4 role warps + 2 softmax warpgroups
#ifndef FA_PP_TURNS
#define FA_PP_TURNS 1
#endif
constexpr bool kPPTurns = FA_PP_TURNS != 0;      // heads alternate the exp phase
#ifndef FA_PP_POLY_EVERY
#define FA_PP_POLY_EVERY 0
#endif
// exp2 pairs computed on the FMA pipe: 1 in N (0 = all on MUFU).  Measured at
// 8 x 1024 tokens: 1 in 2 / 3 / 4 / 8 / 16 -> 119 / 114 / 110 / 104 / 103 us,
// none (0) -> 101 us: in this kernel the softmax is issue-bound, not MUFU-bound.
constexpr int kPPPolyEvery = FA_PP_POLY_EVERY;
constexpr uint32_t kPPQ = 0;                     // Q0, Q1
constexpr uint32_t kPPK = 2 * kTile;             // [2 stages]
constexpr uint32_t kPPV = kPPK + 2 * kTile;      // [2 stages]
constexpr uint32_t kPPBar = kPPV + 2 * kTile;
constexpr uint32_t kPPSmem = kPPBar + 256 + 1024;

__global__ void __launch_bounds__(kPPThreads, 1)
    fa_pp_kernel(const __grid_constant__ CUtensorMap mqkv, __nv_bfloat16* __restrict__ out, int nq, int nkv,
                 int S, int n_seqs, float scale_log2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + kPPBar);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;    // [2]
  uint64_t* k_empty = bars + 4;   // [2]
  uint64_t* v_full = bars + 6;    // [2]
  uint64_t* v_empty = bars + 8;   // [2]
  uint64_t* s_full = bars + 10;   // [2 heads]
  uint64_t* p_full = bars + 12;   // [2 heads]
  uint64_t* o_full = bars + 14;   // [2 heads]
  uint64_t* o_free = bars + 16;   // [2 heads]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 18);
  static_assert(19 * 8 <= 256, "barrier area");

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int q_tiles = S / BQ;
  const int grp = nq / nkv;
  const int pairs = nq / 2;
  const int64_t per_q = static_cast<int64_t>(pairs) * n_seqs;
  const int64_t n_items = per_q * q_tiles;

  if (warp == 0) {
    if (lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mqkv)) : "memory");
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  } else if (warp == 1 && lane == 0) {
    bar_init(q_full, 1);
    bar_init(q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      bar_init(&k_full[i], 1);
      bar_init(&k_empty[i], 1);
      bar_init(&v_full[i], 1);
      bar_init(&v_empty[i], 1);
      bar_init(&s_full[i], 1);
      bar_init(&p_full[i], 4);
      bar_init(&o_full[i], 1);
      bar_init(&o_free[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_trigger();
  int pp_k = 0, pp_s[2] = {0, 0}, pp_pv[2] = {0, 0}, pp_sm = 0, pp_ep = 0;  // trace indices (FA_TRACE builds)
  (void)pp_k, (void)pp_s, (void)pp_pv, (void)pp_sm, (void)pp_ep;

  // Item order of this CTA: passes of gridDim.x items, longest first, walked
  // boustrophedon (even passes CTA c takes item c, odd passes item G-1-c), so
  // the CTA that got the longest item of one pass gets the shortest of the
  // next.  Plain round-robin left the busiest CTA 12 % above the mean at
  // 8 x 1024 tokens (35 vs 31.1 key tiles per head pair); this is within 3 %.
  auto snake_item = [&](int64_t k) -> int64_t {
    const int64_t G = gridDim.x, c = blockIdx.x;
    return k * G + ((k & 1) ? G - 1 - c : c);
  };
  auto decode_item = [&](int64_t i, int& qt, int& hp, int& seq) {
    qt = q_tiles - 1 - static_cast<int>(i / per_q);  // longest first
    const int64_t r = i % per_q;
    hp = static_cast<int>(r % pairs);
    seq = static_cast<int>(r / pairs);
  };
  // Register split (warpgroup granularity): the role warpgroup (TMA, MMA)
  // shrinks to 56, the two softmax warpgroups grow to 224 so a thread holds
  // its whole 128-column S row (one TMEM pass, no spills).
  // 128 x 56 + 256 x 224 = 384 x 168.
  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 88;\n" ::: "memory");
  if (warp == 0) {
    if (lane == 0) {  // ---------------------------------------------- TMA: Q pair, K tiles
      int stage = 0;
      uint32_t ph = 0, qph = 0;
      for (int64_t kk = 0, it = snake_item(0); it < n_items; it = snake_item(++kk)) {
        int qt, hp, seq;
        decode_item(it, qt, hp, seq);
        const int h0 = 2 * hp, kh = h0 / grp;
        const int row0 = seq * S;
        bar_wait(q_empty, qph ^ 1);
        qph ^= 1;
        FA_T(1, static_cast<int>(kk));
        bar_expect(q_full, 2 * kTile);
        for (int t = 0; t < 2; ++t) {
          tma2d(su32(sm + kPPQ + t * kTile), &mqkv, q_full, (h0 + t) * HD, row0 + qt * BQ);
          tma2d(su32(sm + kPPQ + t * kTile + kHalf), &mqkv, q_full, (h0 + t) * HD + 64, row0 + qt * BQ);
        }
        for (int j = 0; j <= qt; ++j) {
          bar_wait(&k_empty[stage], ph ^ 1);
          const uint32_t kd = su32(sm + kPPK + stage * kTile);
          bar_expect(&k_full[stage], kTile);
          tma2d(kd, &mqkv, &k_full[stage], (nq + kh) * HD, row0 + j * BKV);
          tma2d(kd + kHalf, &mqkv, &k_full[stage], (nq + kh) * HD + 64, row0 + j * BKV);
          FA_T(0, pp_k++);
          if (++stage == 2) {
            stage = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 3) {
    if (lane == 0) {  // ---------------------------------------------- TMA: V tiles
      int stage = 0;
      uint32_t ph = 0;
      for (int64_t kk = 0, it = snake_item(0); it < n_items; it = snake_item(++kk)) {
        int qt, hp, seq;
        decode_item(it, qt, hp, seq);
        const int kh = 2 * hp / grp;
        const int row0 = seq * S;
        for (int j = 0; j <= qt; ++j) {
          bar_wait(&v_empty[stage], ph ^ 1);
          const uint32_t vd = su32(sm + kPPV + stage * kTile);
          bar_expect(&v_full[stage], kTile);
          tma2d(vd, &mqkv, &v_full[stage], (nq + nkv + kh) * HD, row0 + j * BKV);
          tma2d(vd + kHalf, &mqkv, &v_full[stage], (nq + nkv + kh) * HD + 64, row0 + j * BKV);
          if (++stage == 2) {
            stage = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------------------------------------- MMA issuer
      int kst = 0, vst = 0;
      uint32_t kph = 0, vph = 0, qph = 0;
      uint32_t pph[2] = {0, 0}, ofph[2] = {0, 0};
      bool first_item = true;
      const uint32_t S_id = idesc(false), PV_id = idesc(true);
      auto issue_s = [&](int t) {  // S_t = Q_t K^T into TMEM cols t*128 (K tile in stage kst)
        const uint32_t qa = su32(sm + kPPQ + t * kTile);
        const uint32_t kb = su32(sm + kPPK + kst * kTile);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint64_t ad = sdesc(qa + (k >> 2) * kHalf + (k & 3) * 32, 16, 1024);
          const uint64_t bd = sdesc(kb + (k >> 2) * kHalf + (k & 3) * 32, 16, 1024);
          mma_ss(tmem + t * 128, ad, bd, S_id, k != 0);
        }
        commit(&s_full[t]);
        FA_T(2 + t, pp_s[t]++);
      };
      auto issue_pv = [&](int t, int j) {  // O_t += P_t V (P in TMEM over S_t's first 64 cols)
        bar_wait(&p_full[t], pph[t]);
        pph[t] ^= 1;
        if (j == 0 && !first_item) {  // the epilogue must have read O_t of the previous item
          bar_wait(&o_free[t], ofph[t]);
          ofph[t] ^= 1;
        }
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t vb = su32(sm + kPPV + vst * kTile);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint64_t bd = sdesc(vb + k * 2048, kHalf, 1024);
          mma_ts(tmem + kColO + t * 128, tmem + t * 128 + k * 8, bd, PV_id, (j | k) != 0);
        }
        FA_T(4 + t, pp_pv[t]++);
      };
      for (int64_t kk = 0, it = snake_item(0); it < n_items; it = snake_item(++kk)) {
        int qt, hp, seq;
        decode_item(it, qt, hp, seq);
        const int n = qt + 1;
        bar_wait(q_full, qph);
        qph ^= 1;
        FA_T(10, static_cast<int>(kk));
        bar_wait(&k_full[kst], kph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        issue_s(0);
        issue_s(1);
        commit(&k_empty[kst]);
        if (++kst == 2) {
          kst = 0;
          kph ^= 1;
        }
        if (n == 1) commit(q_empty);
        for (int j = 0; j < n; ++j) {
          bar_wait(&v_full[vst], vph);
          const bool more = j + 1 < n;
          if (more) {
            bar_wait(&k_full[kst], kph);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          }
          issue_pv(0, j);
          if (!more) commit(&o_full[0]);
          if (more) issue_s(0);
          issue_pv(1, j);
          commit(&v_empty[vst]);
          if (++vst == 2) {
            vst = 0;
            vph ^= 1;
          }
          if (!more) commit(&o_full[1]);
          if (more) {
            issue_s(1);
            commit(&k_empty[kst]);
            if (++kst == 2) {
              kst = 0;
              kph ^= 1;
            }
            if (j + 2 == n) commit(q_empty);
          }
        }
        first_item = false;
      }
    }
  }
  } else {  // ------------------------------------------------------------ softmax warpgroups
    asm volatile("setmaxnreg.inc.sync.aligned.u32 192;\n" ::: "memory");
    const int t = (warp - 4) >> 2;  // head of the pair
    if (kPPTurns && t == 1 && blockIdx.x < n_items) asm volatile("bar.arrive 1, 256;" ::: "memory");  // head 0 first
    const int q = warp & 3;         // TMEM lane quarter
    const int r = q * 32 + lane;    // query row within the tile
    const uint32_t srow = tmem + (static_cast<uint32_t>(q * 32) << 16) + t * 128;
    const uint32_t orow = tmem + (static_cast<uint32_t>(q * 32) << 16) + kColO + t * 128;
    uint32_t sph = 0, oph = 0;
    // Epilogue of an item (O_t / l -> bf16 -> global), deferred until the next
    // item's first P is stored: that softmax overlaps the last PV of this item
    // instead of waiting behind it (the next PV needs O free anyway).
    struct Done {
      int64_t row0;  // first output row of the item's q tile
      int head;
      float l;
    } prev{0, 0, 0.0f};
    bool pending = false;
    const bool out32 = (reinterpret_cast<uintptr_t>(out) & 31) == 0;  // rows are 256 B multiples
    auto epilogue = [&](const Done& d) {
      bar_wait(&o_full[t], oph);
      oph ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const float inv = d.l > 0.0f ? 1.0f / d.l : 0.0f;
      __nv_bfloat16* op = out + (d.row0 + r) * (static_cast<int64_t>(nq) * HD) + static_cast<int64_t>(d.head) * HD;
      // Output rows go out with 32-byte stores that do not allocate in L1.
      // This warp's 32 rows are 8 KB apart, so every store instruction
      // scatters over 32 lines, and that traffic shares the L1 / shared
      // memory array the MMAs read Q, K and V from: allocating the lines in
      // L1 cost 6%, and 16-byte pieces (twice the sectors) another 3%
      // (profiles/r02_attention_st256_ab.txt).
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float o[32];
        tld32(orow + c * 32, o);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          uint32_t w[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) w[e] = bf2(o[v * 16 + 2 * e] * inv, o[v * 16 + 2 * e + 1] * inv);
          if (out32) {
            asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(op + c * 32 + v * 16),
                         "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                         : "memory");
          } else {  // output base only 16-byte aligned (a caller-owned view)
            st_na_v4(op + c * 32 + v * 16, w);
            st_na_v4(op + c * 32 + v * 16 + 8, w + 4);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) bar_arrive(&o_free[t]);
      if (lane == 0 && warp == 4) FA_T(11, pp_ep++);
    };
    for (int64_t kk = 0, it = snake_item(0); it < n_items; it = snake_item(++kk)) {
      int qt, hp, seq;
      decode_item(it, qt, hp, seq);
      const int n = qt + 1;
      float m_used = -FLT_MAX, l = 0.0f;
      for (int j = 0; j < n; ++j) {
        bar_wait(&s_full[t], sph);
        sph ^= 1;
        if (lane == 0 && (warp & 3) == 0) FA_T(6 + 2 * t, pp_sm);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const bool diag = j == qt;
        // the whole 128-key S row in registers (one TMEM pass), row max in-thread
        float sv[128];
#pragma unroll
        for (int c = 0; c < 4; ++c) tld32(srow + c * 32, *reinterpret_cast<float(*)[32]>(&sv[c * 32]));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        float mx8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) mx8[i] = -INFINITY;
        if (diag) {
#pragma unroll
          for (int c = 0; c < 128; ++c) {
            if (c > r) sv[c] = -INFINITY;
            mx8[c & 7] = fmaxf(mx8[c & 7], sv[c]);
          }
        } else {
#pragma unroll
          for (int c = 0; c < 128; ++c) mx8[c & 7] = fmaxf(mx8[c & 7], sv[c]);
        }
        const float pm = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                               fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
        const float mx = scale_log2 * pm;
        float factor = 1.0f;
        const bool rescale = mx > m_used + kRescaleThresh;
        if (rescale) {
          factor = ex2(m_used - mx);  // 0 on the first tile
          m_used = mx;
        }
        l *= factor;
        // O_t is stable here (this S's commit covered PV_t,{j-1})
        if (j > 0 && __any_sync(0xffffffffu, rescale)) {
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            float o[32];
            tld32(orow + c * 32, o);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] *= factor;
            tst32(orow + c * 32, o);
          }
        }
        // P = 2^(s * scale - m) (bf16) over the consumed S columns, 32 keys per store.
        // The two heads take turns in this MUFU-bound phase (named barriers
        // 1 / 2): one head exponentiates while the other loads / reduces /
        // stores and its MMAs run, so the phases interleave instead of both
        // heads contending for the SFU in lock-step.
        if (kPPTurns) asm volatile("bar.sync %0, 256;" ::"r"(1 + t) : "memory");
        float2 sum4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        const float2 sc2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-m_used, -m_used);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          uint32_t pk[16];
#pragma unroll
          for (int c2 = 0; c2 < 16; ++c2) {
            const int c0 = h * 32 + 2 * c2;
            const float2 xv = ffma2(make_float2(sv[c0], sv[c0 + 1]), sc2, nm2);
            const bool poly = kPPPolyEvery > 0 && (h * 16 + c2) % (kPPPolyEvery > 0 ? kPPPolyEvery : 1) == 0;
            const float p0 = poly ? ex2_poly(xv.x) : ex2(xv.x);
            const float p1 = poly ? ex2_poly(xv.y) : ex2(xv.y);
            sum4[c2 & 3] = fadd2(sum4[c2 & 3], make_float2(p0, p1));
            pk[c2] = bf2(p0, p1);
          }
          tst16u(srow + h * 16, pk);
        }
        float sum8[8] = {sum4[0].x, sum4[0].y, sum4[1].x, sum4[1].y, sum4[2].x, sum4[2].y, sum4[3].x, sum4[3].y};
        // hand the turn to the other head (head 1's very last hand-off has no taker)
        if (kPPTurns && !(t == 1 && j == n - 1 && snake_item(kk + 1) >= n_items))
          asm volatile("bar.arrive %0, 256;" ::"r"(2 - t) : "memory");
        l += ((sum8[0] + sum8[1]) + (sum8[2] + sum8[3])) + ((sum8[4] + sum8[5]) + (sum8[6] + sum8[7]));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) bar_arrive(&p_full[t]);
        if (lane == 0 && (warp & 3) == 0) FA_T(7 + 2 * t, pp_sm);
        ++pp_sm;
        if (j == 0 && pending) {
          epilogue(prev);
          pending = false;
        }
      }
      prev = Done{static_cast<int64_t>(seq) * S + static_cast<int64_t>(qt) * BQ, 2 * hp + t, l};
      pending = true;
    }
    if (pending) epilogue(prev);
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
  static bool attr = cudaFuncSetAttribute(fa_tc_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(kSmemTotal)) == cudaSuccess &&
                     cudaFuncSetAttribute(fa_pp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(kPPSmem)) == cudaSuccess;
  if (!enc || !attr) return false;
  // Two heads of one GQA group per item (fa_pp_kernel: registers rebalanced
  // with setmaxnreg, whole S row per thread) for even groups — measured 111 vs
  // 126 us at 8 x 1024 tokens, 32 / 8 heads (620 vs 547 TFLOP/s); odd groups
  // take the one-head kernel with two softmax column parts per row.
  static const int fa_mode = [] {  // OPF_FA=one|pair forces a kernel (A/B runs)
    const char* e = std::getenv("OPF_FA");
    if (e && std::string(e) == "one") return 1;
    if (e && std::string(e) == "pair") return 2;
    return 0;
  }();
  bool pp = (nq / nkv) % 2 == 0;
  if (fa_mode == 1) pp = false;
  // Fewer head-pair items than SMs (e.g. the TP=8 per-rank shape, 4 q heads:
  // 128 items of up to 8 key tiles on 148 SMs) leaves SMs idle behind the
  // longest item; one head per item doubles the items.  Measured per rank at
  // 8 x 1024 tokens (tools/attn_tp8.py): TP=8 25.5 -> 21.9 us; TP=4 (256 pair
  // items) stays on the pair kernel (29.3 vs 37.1 us).
  const int64_t pair_items = static_cast<int64_t>(S / BQ) * (nq / 2) * (rows / S);
  const int sm_grid = max_ctas > 0 ? std::min(max_ctas, num_sms()) : num_sms();
  if (fa_mode == 0 && pp && pair_items < sm_grid) pp = false;
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
  const int64_t items = static_cast<int64_t>(S / BQ) * (pp ? nq / 2 : nq) * n_seqs;
  int grid = max_ctas > 0 ? std::min(max_ctas, num_sms()) : num_sms();
  grid = static_cast<int>(std::min<int64_t>(grid, items));
  if (pp)
    launch_pdl(fa_pp_kernel, dim3(grid), dim3(kPPThreads), kPPSmem, s, m, out, nq, nkv, S, n_seqs,
               scale * 1.4426950408889634f);
  else
    launch_pdl(fa_tc_kernel<2>, dim3(grid), dim3(128 + 2 * 128), kSmemTotal, s, m, out, nq, nkv, S, n_seqs,
               scale * 1.4426950408889634f);
  return true;
}

}  // namespace opflow
