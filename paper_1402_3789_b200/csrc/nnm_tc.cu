// nnm_tc.cu -- tensor-core screening scan for Euclidean Boruvka rounds (sm_100a).
//
// Replaces, for the Euclidean metric, the reference's distance + nearest-pair
// selection stack (metrics.internal_pairwise -> scipy cdist, metrics.py:67-73;
// pairgen._mask_ineligible / _chunk_candidates, pairgen.py:190-244) inside a
// Boruvka round with a tcgen05 GEMM whose accumulator IS the screened distance:
//
//   every tile T is centred on its own fp32 centre c_T; x_t = tf32(fl(x32 - c_T))
//   for a row point x (tile I) and a column point y (tile J), D = c_J - c_I:
//     |x - y|^2 ~= v = r_i - 2 G'_ij,   r_i = |x_t - D|^2              (CUDA cores, per row)
//     G'_ij = x_t . y_t + s_hi + s_lo,   s_hi + s_lo = -(|y_t|^2 + 2 D.y_t)/2
//   G' is one M=128 x N=128 x K=32 kind::tf32 MMA: K holds the d coordinates,
//   the (1, 1) x (s_hi, s_lo) column term, and component slots (-2^50 x 1) that
//   push same-component pairs out of range.  The tf32 products are exact
//   (x_t, y_t are tf32 values); the only rounding inside the tensor core is the
//   fp32 accumulation.
//
// Rigorous filter: with E (squared-domain evaluation error) and eta (distance-domain
// rounding of inputs / centring / tf32 / D), L = (sqrt(v - E) - eta)^2 <= S, the
// exact scipy value.  A pair is skipped only when L exceeds the row's current
// second-best key; a pair that passes gets its exact FP64 value (rounded down) as
// key.  Keys stay lower bounds of S (the FP32 dot form's contract, nnm_common.cuh
// DotModel), so refine / certification / ambiguity handling is unchanged -- and
// since inserted keys are exact, rows are ambiguous only at true FP64 near-ties.
//
// Selection: the full square of the pruned tile-pair list is scanned (each
// unordered tile pair as (I, J) and (J, I)), so a thread owns one row of the
// accumulator (TMEM lane) and keeps that row's top-2 in registers for the whole
// row tile: a 128-column block costs 4 tcgen05.ld + 43 FMNMX3 + 1 compare per
// row; only blocks whose maximum G' passes the row threshold take the exact
// (FP64-bounded) insert path.
//
// Warp roles (320 threads, 1 CTA / SM, persistent over a contiguous item range):
//   warps 0-3  epilogue (TMEM lane quadrant = warp): thresholds, filter, top-2
//   warps 4-7  prep: row-tile slots, per-item D, s_j and column slots into smem
//   warp 8     producer: 16 KB bulk copies (cp.async.bulk) of operand tiles
//   warp 9     MMA issuer + TMEM owner (2 accumulators x 128 columns)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "nnm_common.cuh"
#include "nnm_tc.cuh"

namespace nnm {
namespace {

constexpr int TC_STAGES = 8;
constexpr int TC_EPI_WARPS = 12;                       // warps 0-11: 3 groups x 4 lane quadrants
constexpr int TC_EPI_GROUPS = 3;                       // epilogue groups, items q % 3
constexpr int TC_PREP_GROUPS = 2;                      // 2 single-warp prep groups, items q % 2
constexpr int TC_PREP_THREADS = 32;                    // per group; each lane owns 4 rows / columns
constexpr int TC_PRODUCER_WARP = TC_EPI_WARPS + TC_PREP_GROUPS * TC_PREP_THREADS / 32;
constexpr int TC_MMA_WARP = TC_PRODUCER_WARP + 1;
constexpr int TC_THREADS = (TC_MMA_WARP + 1) * 32;     // 512: 16 warps x 128 registers
constexpr int TC_RING = 64;                            // item ring (>> stages: see prep)
constexpr int TC_ACC = 4;                              // TMEM accumulators (4 x 128 columns)
constexpr uint32_t TC_TILE_BYTES = TC_TILE_FLOATS * 4;
constexpr float TC_MASK = -1125899906842624.0f;   // -2^50: component-slot weight (A side)
constexpr float TC_PAD = -1152921504606846976.0f; // -2^60: s_hi of a pad column
constexpr float TC_U = 5.9604644775390625e-08f;   // 2^-24
// tensor-core fp32 accumulation error per unit of sum |terms|: 2^-16, about 64x the
// classical (K + 8) 2^-22 bound -- validated on the GPU by tests/test_tc.py
constexpr float TC_CACC = 1.52587890625e-05f;

struct TcSmem {
  float A[2][TC_TILE_FLOATS];          // row-tile operand (+ per-row-tile tail)
  float B[TC_STAGES][TC_TILE_FLOATS];  // column-tile operands (+ per-item tail)
  float metaA[2][TC_META];             // tile records (centre, radius, eta bound)
  float metaB[TC_STAGES][TC_META];
  int acomp[2][TILE];                  // component labels of the row / column tiles
  int bcomp[TC_STAGES][TILE];
  float asq[2][TILE];                  // |x_t|^2 of the row tile's positions
  float atn[2][TILE];                  // |x_t| and eta of the row tile's positions
  float aeta[2][TILE];
  float bsq[TC_STAGES][TILE];          // |y_t|^2 of the column tile's positions
  // per-row data of the item's ROW tile, staged with every item (so the epilogue never
  // waits on global memory at a row-tile change): component labels, the rows' global
  // second-best keys at copy time (a valid threshold: keys only decrease) and, on capped
  // exact passes, the per-position component caps
  int rcomp[TC_STAGES][TILE];
  unsigned long long rb2[TC_STAGES][TILE];
  unsigned rcap[TC_STAGES][TILE];
  float rrow[TC_STAGES][TILE];         // per row of the item: r_i, E and eta (prep -> epilogue)
  float erow[TC_STAGES][TILE];
  float etarow[TC_STAGES][TILE];
  int2 ring[TC_RING];                  // (I, J) of item q at q % TC_RING (written by the producer)
  int4 ringtr[TC_RING];                // component-label ranges of I and J (x, y: I; z, w: J)
  int ringrt[TC_RING];                 // row-tile index of item q, negated-minus-one when item q
                                       // is the first of its row tile (producer)
  int arec[2][16];                     // row tile's slot record: [0..7] component slots,
                                       // [8] distinct components (tc_tails_kernel, per round)
  int chk[TC_STAGES];                  // item may hold unmasked same-component pairs (prep)
  unsigned lbw[TC_EPI_GROUPS][2][4];   // tile-pair bound: per-quadrant minima of an item
  int lbcnt[TC_EPI_GROUPS][2];         // (epilogue group, item parity) arrivals
  unsigned long long full[TC_STAGES], prepped[TC_STAGES], empty[TC_STAGES];
  unsigned long long tfull[TC_ACC], tempty[TC_ACC], afull[2], aprepped[2], aempty[2];
  uint32_t tmem_base;
};

// ---------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(su32(b)),
      "r"(parity), "r"(0x989680u)  // suspend-time hint: a waiting warp sleeps, it does not poll
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// K-major, 128-byte swizzled operand: rows of 128 B, 8-row atoms 1024 B apart (SBO),
// descriptor version 1 (sm_100), layout type 2 (SWIZZLE_128B).
__device__ __forceinline__ uint64_t sw128_desc(const void* p) {
  const uint64_t a = su32(p);
  return ((a >> 4) & 0x3FFFull) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
// kind::tf32 instruction descriptor: D f32, A/B tf32, both K-major, N = 128, M = 128
constexpr uint32_t TC_IDESC =
    (1u << 4) | (2u << 7) | (2u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(TC_IDESC), "r"(accum)
      : "memory");
}
__device__ __forceinline__ void mma_commit(unsigned long long* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
      : "memory");
}

#define TC_R8(i) "=r"(r[i]), "=r"(r[i + 1]), "=r"(r[i + 2]), "=r"(r[i + 3]), \
                 "=r"(r[i + 4]), "=r"(r[i + 5]), "=r"(r[i + 6]), "=r"(r[i + 7])
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, float (&v)[64]) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : TC_R8(0), TC_R8(8), TC_R8(16), TC_R8(24)
      : "r"(taddr));
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : TC_R8(32), TC_R8(40), TC_R8(48), TC_R8(56)
      : "r"(taddr + 32));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
#undef TC_R8
// timing trace (NNM_TC_TRACE): CTA 0 stamps clock64 per role / item / event
__device__ __forceinline__ void trace(const TcArgs& p, int role, int q, int ev) {
  if (p.trace && blockIdx.x == 0 && q < 256) p.trace[(role * 256 + q) * 2 + ev] = clock64();
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// float offset of chunk c (4 floats) of row r inside a swizzled tile image
__device__ __forceinline__ int swz(int r, int c) { return r * TC_K + ((c ^ (r & 7)) << 2); }

__device__ __forceinline__ void insert_top2_g(unsigned long long* G1, unsigned long long* G2,
                                              unsigned long long k1, unsigned long long k2) {
  if (!key_valid(k1)) return;
  const unsigned long long old = atomicMin(G1, k1);
  const unsigned long long disp = (k1 < old) ? old : k1;
  const unsigned long long m = disp < k2 ? disp : k2;
  if (key_valid(m)) atomicMin(G2, m);
}

// Rigorous lower bound of S from the computed v (see file header): the |v| term
// of the evaluation error is added here, E holds the rest.
__device__ __forceinline__ float lower_key(float v, float E, float eta) {
  const double w = (double)v - (double)E * (1.0 + 1e-9) - 1.02 * 5.9604644775390625e-08 * fabs((double)v);
  if (!(w > 0.0)) return 0.f;
  const double sq = sqrt(w) * (1.0 - 1e-15) - (double)eta;
  if (!(sq > 0.0)) return 0.f;
  return float_down(sq * sq * (1.0 - 1e-15));
}

// Tail of one operand row: positions d .. d+1+kc of the K = 32 floats (the image has
// zeros beyond), written as whole 16-byte chunks (coordinates sharing the first chunk
// are re-written unchanged).  A side (row tile): (1, 1, -2^50 per matching slot);
// B side (column tile): (s_hi, s_lo, 1 per matching slot).  hits: bit k = slot k matches.
// With a compile-time d every index below folds to a constant (straight-line code).
__device__ __forceinline__ void write_tail(float* tile, int r, int d, int kc, float t0, float t1,
                                          uint32_t hits, float hit) {
  const int c0 = d >> 2, c1 = (d + 1 + kc) >> 2;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    if (c < c0 || c > c1) continue;
    float4* q = reinterpret_cast<float4*>(tile + swz(r, c));
    float e[4] = {0.f, 0.f, 0.f, 0.f};
    if (c == c0 && (d & 3)) {
      const float4 v = *q;
      e[0] = v.x; e[1] = v.y; e[2] = v.z; e[3] = v.w;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int t = 4 * c + u - d;
      const float val = t == 0 ? t0 : t == 1 ? t1 : ((hits >> ((t - 2) & 31)) & 1u) ? hit : 0.f;
      e[u] = t < 0 ? e[u] : val;
    }
    *q = make_float4(e[0], e[1], e[2], e[3]);
  }
}

__device__ __forceinline__ uint32_t slot_hits(int comp, const int (&slot)[8]) {
  uint32_t h = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) h |= (comp >= 0 && comp == slot[k]) ? (1u << k) : 0u;
  return h;
}

// Per-item quantities (shared by the prep warps and the probe so both round
// identically; any summation order is inside the error bound):
//   D = c_J - c_I (fp32), |D|^2, r_i = |x_t|^2 - 2 x_t.D + |D|^2, s_j = |y_t|^2 + 2 D.y_t
// with |x_t|^2 / |y_t|^2 precomputed per position (tc_prepare_kernel).
__device__ __forceinline__ float tc_delta(const float* __restrict__ mj, const float* __restrict__ mi,
                                          int d, float (&dl)[32]) {
  float n2[2] = {0.f, 0.f};
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    if (4 * c >= d) {
      dl[4 * c] = dl[4 * c + 1] = dl[4 * c + 2] = dl[4 * c + 3] = 0.f;
      continue;
    }
    const float4 a = *reinterpret_cast<const float4*>(mj + 4 * c);
    const float4 b = *reinterpret_cast<const float4*>(mi + 4 * c);
    dl[4 * c] = a.x - b.x; dl[4 * c + 1] = a.y - b.y; dl[4 * c + 2] = a.z - b.z; dl[4 * c + 3] = a.w - b.w;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (4 * c + u < d) n2[u & 1] = fmaf(dl[4 * c + u], dl[4 * c + u], n2[u & 1]);
  }
  return n2[0] + n2[1];
}
__device__ __forceinline__ float tc_dot(const float (&x)[32], const float (&dl)[32], int d) {
  float q4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int k = 0; k < 32; ++k)
    if (k < d) q4[k & 3] = fmaf(x[k], dl[k], q4[k & 3]);
  return (q4[0] + q4[1]) + (q4[2] + q4[3]);
}
__device__ __forceinline__ float tc_r(float xsq, float q, float dn2) {
  return __fmaf_rn(-2.f, q, xsq) + dn2;
}
__device__ __forceinline__ float tc_dnorm(float dn2, int d) {
  return sqrtf(dn2) * (1.0f + (d + 4) * TC_U * 2.f);
}

// Squared-domain evaluation bound E of a row's pairs with tile J (all terms but the |v|
// one, which lower_key adds) and the distance-domain rounding bound eta (file header).
// r error <= (d+3) u (|x_t| + |D|)^2, s error <= (d+3) u (|y_t|^2 + 2 |y_t||D|) with
// sb = RJ (RJ + 2|D|) >= |s_j|, split 2^-22 |s|, tensor-core accumulation.
__device__ __forceinline__ void tc_bounds(float dnorm, int d, float tn_i, float eta_i, float RJ,
                                          float etaJ, float& Erow, float& eta_row) {
  const float sb = RJ * (RJ + 2.f * dnorm);
  const float xr = tn_i + dnorm;
  Erow = ((d + 3) * TC_U * 1.02f * xr * xr + (d + 3) * TC_U * 1.01f * sb + 2.4e-7f * sb +
          2.f * TC_CACC * (tn_i * RJ + 0.51f * sb)) * 1.01f + 1e-30f;
  eta_row = (eta_i + etaJ + TC_U * 1.001f * dnorm) * 1.0001f;
}

__device__ __forceinline__ void load_row(const float* tile, int r, int d, float (&x)[32]) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    if (4 * c < d) {
      const float4 v = *reinterpret_cast<const float4*>(tile + swz(r, c));
      x[4 * c] = v.x; x[4 * c + 1] = v.y; x[4 * c + 2] = v.z; x[4 * c + 3] = v.w;
    } else {
      x[4 * c] = x[4 * c + 1] = x[4 * c + 2] = x[4 * c + 3] = 0.f;
    }
  }
}

// Mask slots of a row tile: the first kc distinct components in position order
// (parallel first-occurrence test + warp ballots).  Called by one prep warp: lane l owns
// rows l, l + 32, l + 64, l + 96 (one 32-row block per ballot, in position order).
__device__ __forceinline__ void select_slots(const int* comp, int* slot, int* nslot, int lane, int kc) {
  int c[4];
  bool f[4];
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    c[b] = comp[lane + 32 * b];
    f[b] = c[b] >= 0;
  }
#pragma unroll 8
  for (int r = 0; r < TILE; ++r) {
    const int cr = comp[r];
#pragma unroll
    for (int b = 0; b < 4; ++b) f[b] &= !(r < lane + 32 * b && cr == c[b]);
  }
  int base = 0;
  const unsigned below = (1u << lane) - 1u;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const unsigned m = __ballot_sync(0xFFFFFFFFu, f[b]);
    const int rank = base + __popc(m & below);
    if (f[b] && rank < kc) slot[rank] = c[b];
    base += __popc(m);
  }
  if (lane < 8 && lane >= min(base, kc)) slot[lane] = -2;
  if (lane == 0) *nslot = base;
  __syncwarp();
}

template <int DC>
__global__ void __maxnreg__(128) tc_scan_kernel(TcArgs p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // pointer arithmetic on the shared array keeps the shared state space (no generic LD/ST)
  TcSmem& S = *reinterpret_cast<TcSmem*>(smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t total = p.w_end - p.w_begin;
  const int64_t per = (total + gridDim.x - 1) / gridDim.x;
  const int64_t w0 = p.w_begin + (int64_t)blockIdx.x * per;
  const int64_t w1 = min(w0 + per, p.w_end);
  if (w0 >= w1) return;
  const int nq = (int)(w1 - w0);
  const int d = DC ? DC : p.d;  // compile-time for the specialised instantiations
  const int kc = min(8, TC_K - d - 2);

  if (tid == 0) {
    for (int s = 0; s < TC_STAGES; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.prepped[s], 1);
      mbar_init(&S.empty[s], 1 + TC_EPI_WARPS / TC_EPI_GROUPS);
    }
    for (int a = 0; a < TC_ACC; ++a) {
      mbar_init(&S.tfull[a], 1);
      mbar_init(&S.tempty[a], TC_EPI_WARPS / TC_EPI_GROUPS);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&S.afull[a], 1);
      mbar_init(&S.aprepped[a], 1);
      mbar_init(&S.aempty[a], 1);
    }
    for (int g = 0; g < TC_EPI_GROUPS; ++g)
      for (int b = 0; b < 2; ++b) S.lbcnt[g][b] = 0;
    fence_barrier_init();
  }
  if (warp == TC_MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     su32(&S.tmem_base))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = S.tmem_base;

  if (warp == TC_PRODUCER_WARP) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int rt = -1, prevI = -1;
      int2 nxt = __ldg(p.items + w0);
      // component-label ranges of the item's tiles (the prep's slot-check decision), one
      // item ahead like the item itself; no trange: always check
      auto ranges = [&](int2 t) {
        if (!p.trange) return make_int4(0, 0x7FFFFFFF, 0, 0x7FFFFFFF);
        const int2 a = __ldg(p.trange + t.x), b = __ldg(p.trange + t.y);
        return make_int4(a.x, a.y, b.x, b.y);
      };
      int4 nxtr = ranges(nxt);
      for (int q = 0; q < nq; ++q) {
        const int2 it = nxt;
        const int4 itr = nxtr;
        if (q + 1 < nq) {  // one item of lookahead
          nxt = __ldg(p.items + w0 + q + 1);
          nxtr = ranges(nxt);
        }
        if (it.x != prevI) {
          ++rt;
          prevI = it.x;
          const int xb = rt & 1;
          if (rt >= 2) mbar_wait(&S.aempty[xb], ((rt - 2) >> 1) & 1);
          mbar_expect_tx(&S.afull[xb], TC_TILE_BYTES + TC_META * 4 + 4 * TILE * 4 + 64);
          bulk_g2s(S.arec[xb], p.slots + (int64_t)it.x * 16, 64, &S.afull[xb]);
          bulk_g2s(S.A[xb], p.img + (int64_t)it.x * TC_TILE_FLOATS, TC_TILE_BYTES, &S.afull[xb]);
          bulk_g2s(S.metaA[xb], p.meta + (int64_t)it.x * TC_META, TC_META * 4, &S.afull[xb]);
          bulk_g2s(S.acomp[xb], p.comp + (int64_t)it.x * TILE, TILE * 4, &S.afull[xb]);
          bulk_g2s(S.asq[xb], p.sq + (int64_t)it.x * TILE, TILE * 4, &S.afull[xb]);
          bulk_g2s(S.atn[xb], p.tnorm + (int64_t)it.x * TILE, TILE * 4, &S.afull[xb]);
          bulk_g2s(S.aeta[xb], p.eta + (int64_t)it.x * TILE, TILE * 4, &S.afull[xb]);
        }
        const int s = q % TC_STAGES;
        if (q >= TC_STAGES) mbar_wait(&S.empty[s], ((q / TC_STAGES) - 1) & 1);
        trace(p, 0, q, 0);
        S.ring[q % TC_RING] = it;  // published to the other roles by the full barrier
        S.ringtr[q % TC_RING] = itr;
        S.ringrt[q % TC_RING] = (q == 0 || it.x != S.ring[(q - 1) % TC_RING].x) ? -rt - 1 : rt;
        const bool rows_b2 = !p.bound_only && !p.dump;
        const bool rows_cap = rows_b2 && p.capp;
        mbar_expect_tx(&S.full[s], TC_TILE_BYTES + TC_META * 4 + 3 * TILE * 4 +
                                       (rows_b2 ? TILE * 8 : 0) + (rows_cap ? TILE * 4 : 0));
        bulk_g2s(S.B[s], p.img + (int64_t)it.y * TC_TILE_FLOATS, TC_TILE_BYTES, &S.full[s]);
        bulk_g2s(S.metaB[s], p.meta + (int64_t)it.y * TC_META, TC_META * 4, &S.full[s]);
        bulk_g2s(S.bcomp[s], p.comp + (int64_t)it.y * TILE, TILE * 4, &S.full[s]);
        bulk_g2s(S.bsq[s], p.sq + (int64_t)it.y * TILE, TILE * 4, &S.full[s]);
        bulk_g2s(S.rcomp[s], p.comp + (int64_t)it.x * TILE, TILE * 4, &S.full[s]);
        if (rows_b2) bulk_g2s(S.rb2[s], p.B2 + (int64_t)it.x * TILE, TILE * 8, &S.full[s]);
        if (rows_cap) bulk_g2s(S.rcap[s], p.capp + (int64_t)it.x * TILE, TILE * 4, &S.full[s]);
      }
    }
  } else if (warp == TC_MMA_WARP) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      int rt = -1, prevI = -1;
      for (int q = 0; q < nq; ++q) {
        const int s = q % TC_STAGES;
        mbar_wait(&S.prepped[s], (q / TC_STAGES) & 1);
        const int2 it = S.ring[q % TC_RING];
        if (it.x != prevI) {
          if (rt >= 0) mma_commit(&S.aempty[rt & 1]);  // previous A buffer free once its MMAs land
          ++rt;
          prevI = it.x;
          mbar_wait(&S.afull[rt & 1], (rt >> 1) & 1);  // A tails written per round
        }
        const int a = q % TC_ACC;
        if (q >= TC_ACC) mbar_wait(&S.tempty[a], ((q / TC_ACC) - 1) & 1);
        trace(p, 1, q, 0);
        tc_after();
        const uint64_t ad = sw128_desc(S.A[rt & 1]), bd = sw128_desc(S.B[s]);
        const int reps = (p.dbg & 512) ? 0 : (p.dbg & 32) ? 8 : 1;  // timing experiments
        for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
          for (int kk = 0; kk < TC_K / 8; ++kk)  // K = 8 tf32 (32 B) per instruction
            mma_tf32(tmem + a * TILE, ad + 2 * kk, bd + 2 * kk, kk > 0 ? 1u : 0u);
        }
        mma_commit(&S.empty[s]);
        mma_commit(&S.tfull[a]);
      }
    }
  } else if (warp >= TC_EPI_WARPS) {
    // ------------------------------------------------------------ prep groups
    // group g (one warp) preps items q = g, g + 4, ...; lane l owns rows / columns
    // l + 32k (k < 4).  Row-tile changes are read from the item ring (entries q-4 .. q
    // are still live: the producer runs at most TC_STAGES items ahead of the slowest
    // consumer and TC_RING >> TC_STAGES + 4)
    const int g = warp - TC_EPI_WARPS;
    const int pt = lane;
    int rt = -1, myI = -1;
    float tn4[4] = {0.f, 0.f, 0.f, 0.f}, eta4[4] = {0.f, 0.f, 0.f, 0.f};
    int slot[8];
    for (int q = g; q < nq; q += TC_PREP_GROUPS) {
      const int s = q % TC_STAGES;
      mbar_wait(&S.full[s], (q / TC_STAGES) & 1);
      if (pt == 0) trace(p, 2, q, 0);
      // row-tile index of item q and whether it opens its row tile (from the producer)
      const int I = S.ring[q % TC_RING].x;
      const int rtq = S.ringrt[q % TC_RING];
      const bool opens = rtq < 0;
      rt = opens ? -rtq - 1 : rtq;
      const int xb = rt & 1;
      if (I != myI) {
        myI = I;
        // the A operand (coordinates + per-round tails) and its slot record arrive as copied
        mbar_wait(&S.afull[xb], (rt >> 1) & 1);
#pragma unroll
        for (int k = 0; k < 8; ++k) slot[k] = S.arec[xb][k];
#pragma unroll
        for (int k = 0; k < 4; ++k) {  // staged with the row tile (no global latency)
          tn4[k] = S.atn[xb][pt + 32 * k];
          eta4[k] = S.aeta[xb][pt + 32 * k];
        }
      }
      if (p.dbg & 2) {  // timing experiment: no prep work
        __syncwarp();
        if (pt == 0) mbar_arrive(&S.prepped[s]);
        continue;
      }
      if (pt == 0) trace(p, 5, q, 0);
      float dl[32];
      const float dn2 = tc_delta(S.metaB[s], S.metaA[xb], d, dl);
      const float dnorm = tc_dnorm(dn2, d);
      const float RJ = S.metaB[s][32], etaJ = S.metaB[s][33];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        // row pt + 32k: r_i and its bounds for the epilogue (coordinates read from the
        // A tile: the tail chunk holds the A-side constants, not coordinates < d)
        const int row = pt + 32 * k;
        float x[32];
        load_row(S.A[xb], row, d, x);
        const float r = tc_r(S.asq[xb][row], tc_dot(x, dl, d), dn2);
        float Erow, eta_row;
        tc_bounds(dnorm, d, tn4[k], eta4[k], RJ, etaJ, Erow, eta_row);
        S.rrow[s][row] = r;
        S.erow[s][row] = Erow;
        S.etarow[s][row] = eta_row;
        // column pt + 32k: s_j = |y|^2 + 2 D.y into the K tail (hi / lo), slot hits
        const int col = row;
        float y[32];
        load_row(S.B[s], col, d, y);
        const int cj = S.bcomp[s][col];
        float hi, lo;
        if (cj >= 0) {
          const float sj = __fmaf_rn(2.f, tc_dot(y, dl, d), S.bsq[s][col]);
          const float hh = -0.5f * sj;
          hi = tf32_rna(hh);
          lo = tf32_rna(hh - hi);
        } else {
          hi = TC_PAD;
          lo = 0.f;
        }
        write_tail(S.B[s], col, d, kc, hi, lo, slot_hits(cj, slot), 1.f);
      }
      if (pt == 0) {
        trace(p, 5, q, 1);
        // unmasked same-component pairs are possible only if the row tile has more
        // components than slots and the two tiles' component ranges overlap
        const int4 tr = S.ringtr[q % TC_RING];
        const bool chk = S.arec[xb][8] > kc && !(tr.w < tr.x || tr.y < tr.z);
        S.chk[s] = chk ? 1 : 0;
      }
      if (!(p.dbg & 4)) fence_proxy_async();  // (dbg 4: timing experiment only)
      if (pt == 0) trace(p, 7, q, 0);
      __syncwarp();
      if (pt == 0) {
        trace(p, 2, q, 1);
        mbar_arrive(&S.prepped[s]);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue warps
    // group e = warp / 4 takes items q = e, e + 2, ... (two items in flight); warp w owns
    // TMEM lane quadrant w % 4 (rows 32(w%4) ..) and all 128 columns of its items.  Each
    // group keeps its own per-row top-2 for the row tile and merges it atomically.
    const int e = warp >> 2;
    const int i = (warp & 3) * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    int prevI = -1;
    unsigned long long k1 = NONE_KEY, k2 = NONE_KEY;
    float gT = INFINITY, tup = INFINITY;  // tup: seeded upper bound of the second best
    float capT = INFINITY;                // the component's cap (exact mode)
    float rowU = INFINITY;                // best screened upper bound of the row (bound mode)
    int ci = -1;
    int64_t g = 0;
    // Row-tile flush of the top-2 into the global keys, split in two so that the latency of
    // the returning atomicMin on B1 overlaps the next item's work: step 1 at the row-tile
    // change issues it; step 2 (the displaced key into B2, a non-returning atomicMin) runs
    // after the next item.  Both epilogue groups merge into the same rows this way.
    bool pend = false;
    unsigned long long pold = 0, pk1 = NONE_KEY, pk2 = NONE_KEY;
    int64_t pg = 0;
    auto finish_flush = [&]() {
      if (!pend) return;
      pend = false;
      const unsigned long long disp = (pk1 < pold) ? pold : pk1;
      const unsigned long long m = disp < pk2 ? disp : pk2;
      if (key_valid(m)) atomicMin(p.B2 + pg, m);
    };
    auto flush_row = [&]() {
      if (ci < 0 || p.dump) return;
      if (p.bound_only) {
        if (p.ucap && rowU < INFINITY) atomicMin(p.ucap + ci, __float_as_uint(rowU));
      } else if (key_valid(k1)) {
        finish_flush();
        pend = true;
        pg = g;
        pk1 = k1;
        pk2 = k2;
        pold = atomicMin(p.B1 + g, k1);
      }
    };
    for (int q = e; q < nq; q += TC_EPI_GROUPS) {
      const int s = q % TC_STAGES;
      if (tid == 0) trace(p, 6, q, 0);
      mbar_wait(&S.prepped[s], (q / TC_STAGES) & 1);
      if (tid == 0) trace(p, 4, q, 0);
      const int2 it = S.ring[q % TC_RING];
      const int I = it.x, J = it.y;
      if (I != prevI) {
        if (prevI >= 0) flush_row();
        prevI = I;
        g = (int64_t)I * TILE + i;
        ci = S.rcomp[s][i];
        if (p.bound_only || p.dump) {
          gT = INFINITY;
        } else {
          const unsigned long long gb = S.rb2[s][i];
          gT = key_valid(gb) ? key_value(gb) : INFINITY;
        }
        capT = (!p.bound_only && !p.dump && p.capp && ci >= 0) ? __uint_as_float(S.rcap[s][i]) : INFINITY;
        k1 = k2 = NONE_KEY;
        tup = INFINITY;
        rowU = INFINITY;
      }
      const float r = S.rrow[s][i], Erow = S.erow[s][i], eta_row = S.etarow[s][i];
      // G' threshold equivalent to "L <= T may hold" (vthr: largest v with L <= T)
      auto gamma_of = [&](float T) -> float {
        if (!(T < INFINITY)) return -INFINITY;
        const float st = sqrtf(T) * 1.000001f + eta_row;
        const float vthr = (st * st + Erow) * 1.00001f;
        return (r - vthr) * 0.5f - (fabsf(r) + vthr) * 1e-6f - 1e-30f;
      };
      float T = fminf(fminf(k2 == NONE_KEY ? INFINITY : key_value(k2), fminf(gT, tup)),
                      fminf(p.thr_hi, capT));
      float gam = gamma_of(T);
      const int a = q % TC_ACC;
      mbar_wait(&S.tfull[a], (q / TC_ACC) & 1);
      if (tid == 0) trace(p, 3, q, 0);
      tc_after();
      if (!(p.dbg & 1)) {
        // fast filter, 64 columns at a time: maxima of the 8-column groups (the first
        // levels of the reduction tree) -> bit mask of groups that may hold a candidate
        uint32_t gm = 0;
        float rmax = -INFINITY;  // largest G' of the row (tile-pair bound)
        float gmax[16];          // 8-column group maxima (bound mode skips groups below b1)
#pragma unroll 1
        for (int hb = 0; hb < 2; ++hb) {
          float v[64];
          tmem_ld64(lane_base + a * TILE + hb * 64, v);
          if (p.dump) {
            float* o = p.dump + ((w0 + q - p.w_begin) * TILE + i) * TILE + hb * 64;
#pragma unroll
            for (int jj = 0; jj < 64; ++jj) o[jj] = v[jj];
          } else {
            float g8[8];
#pragma unroll
            for (int k = 0; k < 8; ++k)
              g8[k] = fmaxf(fmaxf(fmaxf(v[8 * k], v[8 * k + 1]), fmaxf(v[8 * k + 2], v[8 * k + 3])),
                            fmaxf(fmaxf(v[8 * k + 4], v[8 * k + 5]), fmaxf(v[8 * k + 6], v[8 * k + 7])));
            rmax = fmaxf(rmax, fmaxf(fmaxf(fmaxf(g8[0], g8[1]), fmaxf(g8[2], g8[3])),
                                     fmaxf(fmaxf(g8[4], g8[5]), fmaxf(g8[6], g8[7]))));
            uint32_t m = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              m |= (g8[k] >= gam) ? (1u << k) : 0u;
              gmax[8 * hb + k] = g8[k];
            }
            gm |= (ci >= 0 ? m : 0u) << (8 * hb);
          }
        }
        if (p.bound_only) {
          // bound mode: the largest G' over the row's valid cross-component columns gives a
          // real eligible-or-farther partner with S <= (sqrt(v + E) + eta)^2: the row's
          // rigorous upper bound, min over the row tile's items, atomicMin into its
          // component's cap at the end of the row tile (flush_row)
          // every same-component pair is masked by the slots (or none exists): the row
          // maximum over all columns is over valid cross-component columns (pads sit at
          // -2^60 and cannot win while the tile holds a real point)
          const bool chk = S.chk[s] != 0;
          float b1 = chk ? -INFINITY : rmax;
#pragma unroll 1
          for (int gidx = 0; gidx < TILE / 8; ++gidx) {
            if (!chk) break;
            if (!__any_sync(0xFFFFFFFFu, ci >= 0 && gmax[gidx] > b1)) continue;
            float w[8];
            tmem_ld8(lane_base + a * TILE + gidx * 8, w);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int cj = S.bcomp[s][gidx * 8 + u];
              if (cj >= 0 && cj != ci) b1 = fmaxf(b1, w[u]);
            }
          }
          if (ci >= 0 && b1 > -INFINITY) {
            // the same bound as the seed's below, in fp32 with every step rounded up (a
            // rigorous upper bound; the FP64 form cost a DSQRT per row and item)
            const float v1 = __fmaf_rn(-2.f, b1, r);
            const float e = __fmaf_ru(1.03f * 5.9604644775390625e-08f, fabsf(v1),
                                      __fmul_ru(Erow, 1.000001f));
            const float up = __fadd_ru(__fsqrt_ru(fmaxf(0.f, __fadd_ru(v1, e))), eta_row);
            rowU = fminf(rowU, __fmul_ru(up, up));
          }
          gm = 0;  // no exact work in bound mode
        } else
        // threshold seed: a row with no finite threshold yet (first items of a row tile in
        // phase 1) would send every column to the FP64 path.  The two largest valid G' of the
        // item give two distinct eligible partners with S <= (sqrt(v + E) + eta)^2, so the
        // larger of those upper bounds caps the row's second-best exact value.
        if (__any_sync(0xFFFFFFFFu, ci >= 0 && !(T < INFINITY))) {
          float b1 = -INFINITY, b2 = -INFINITY;
#pragma unroll 1
          for (int gidx = 0; gidx < TILE / 8; ++gidx) {
            float w[8];
            tmem_ld8(lane_base + a * TILE + gidx * 8, w);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int cj = S.bcomp[s][gidx * 8 + u];
              if (cj >= 0 && cj != ci) {
                b2 = fmaxf(b2, fminf(b1, w[u]));
                b1 = fmaxf(b1, w[u]);
              }
            }
          }
          if (p.trace && lane == 0) atomicAdd((unsigned long long*)(p.trace + 8 * 256 * 2 + 1), 1ull);
          if (ci >= 0 && !(T < INFINITY) && b2 > -INFINITY) {
            const double v2 = (double)__fmaf_rn(-2.f, b2, r);
            const double e = (double)Erow * (1.0 + 1e-9) + 1.02 * 5.9604644775390625e-08 * fabs(v2);
            const double up = sqrt(fmax(0.0, v2 + e)) * (1.0 + 1e-15) + (double)eta_row;
            tup = float_up(up * up * (1.0 + 1e-15));
            T = fminf(T, tup);
            gam = gamma_of(T);
          }
        }
        // exact insert path (rare): the warp re-reads only the 8-column groups where some
        // lane may hold a candidate (tcgen05.ld is warp-collective) and each lane marks its
        // candidates (value, component and rigorous lower bound checks) in a 128-bit mask;
        // then the lanes evaluate their candidates in lockstep -- each iteration every lane
        // takes its next one -- so FP64 gather latencies are paid per candidate of the
        // busiest lane, not per column position.  A candidate gets its exact scipy-order
        // FP64 value (rounded down) as key.
        uint32_t wm = __reduce_or_sync(0xFFFFFFFFu, gm);
#pragma unroll 1
        while (wm) {
          const int gidx = __ffs(wm) - 1;
          wm &= wm - 1;
          if (p.trace && lane == 0) atomicAdd((unsigned long long*)(p.trace + 8 * 256 * 2 + 2), 1ull);
          float w[8];
          tmem_ld8(lane_base + a * TILE + gidx * 8, w);
          uint32_t m8 = 0;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (ci < 0 || !(w[u] >= gam)) continue;
            const int cj = S.bcomp[s][gidx * 8 + u];
            if (cj < 0 || cj == ci) continue;
            if (!(lower_key(__fmaf_rn(-2.f, w[u], r), Erow, eta_row) <= T)) continue;
            m8 |= 1u << u;
          }
          if (p.cand && m8) {  // deferred: append, evaluated after the scan (tc_exact)
            const unsigned nc8 = __popc(m8);
            const unsigned long long at = atomicAdd(p.ccount, (unsigned long long)nc8);
            if (at + nc8 <= p.ccap) {
              unsigned long long* o = p.cand + at;
              while (m8) {
                const int u = __ffs(m8) - 1;
                m8 &= m8 - 1;
                *o++ = ((unsigned long long)g << 32) | (unsigned)((int64_t)J * TILE + gidx * 8 + u);
              }
            }  // else: the buffer is full -- these lanes evaluate in place below
          }
          // lockstep: each iteration every lane evaluates its next candidate of the group
#pragma unroll 1
          while (__any_sync(0xFFFFFFFFu, m8 != 0u)) {
            if (m8 == 0u) continue;
            const int u = __ffs(m8) - 1;
            m8 &= m8 - 1;
            const int64_t gj = (int64_t)J * TILE + gidx * 8 + u;
            if (p.trace) atomicAdd((unsigned long long*)(p.trace + 8 * 256 * 2), 1ull);
            const float L = float_down(exact_dist<EUCLIDEAN>(p.X64 + g * d, p.X64 + gj * d, d));
            if (!(L <= T)) continue;  // cannot enter the top-2 (T: second best, global, dmax)
            const unsigned long long key = ((unsigned long long)__float_as_uint(L) << 32) | (unsigned)gj;
            if (key < k2) {
              if (key < k1) {
                k2 = k1;
                k1 = key;
              } else {
                k2 = key;
              }
              T = fminf(fminf(key_value(k2), fminf(gT, tup)), fminf(p.thr_hi, capT));
              gam = gamma_of(T);
            }
          }
        }
        // tile-pair lower bound (DESIGN 3.1): min over the item's rows of L(r_i - 2 max_j G'),
        // a rigorous lower bound of S over every pair not masked as same-component now,
        // hence of every cross-component pair in later rounds.  The 4 quadrant warps
        // combine through shared memory (the last to arrive publishes with atomicMax:
        // both orientations and all rounds give valid bounds, the largest is kept).
        if (p.tpmin && !p.dump) {
          const float lbr = ci >= 0 ? lower_key(__fmaf_rn(-2.f, rmax, r), Erow, eta_row) : INFINITY;
          const unsigned mw = __reduce_min_sync(0xFFFFFFFFu, __float_as_uint(lbr));
          if (lane == 0) {
            const int par = (q / TC_EPI_GROUPS) & 1;
            volatile unsigned* lw = S.lbw[e][par];
            lw[warp & 3] = mw;
            __threadfence_block();
            if (atomicAdd(&S.lbcnt[e][par], 1) == 3) {
              __threadfence_block();
              const unsigned mm = min(min(lw[0], lw[1]), min(lw[2], lw[3]));
              S.lbcnt[e][par] = 0;
              const int lo = min(I, J), hi = max(I, J);
              const int64_t w = (int64_t)lo * p.T - (int64_t)lo * (lo - 1) / 2 + (hi - lo);
              if (mm != 0u) atomicMax(p.tpmin + w, mm);
            }
          }
        }
      }
      tc_before();
      __syncwarp();
      if (lane == 0) {
        if (tid == 0) trace(p, 3, q, 1);
        mbar_arrive(&S.tempty[a]);
        mbar_arrive(&S.empty[s]);
      }
      finish_flush();  // step 2 of the previous row tile's flush (its atomic has landed)
    }
    if (prevI >= 0) flush_row();
    finish_flush();
  }

  tc_before();
  __syncthreads();
  tc_after();
  if (warp == TC_MMA_WARP)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

// ---------------------------------------------------------------- per-round A tails
// Once per round (components changed): for every tile, its component slots (the first kc
// distinct components in position order, -2 unused) and distinct count into the slot
// record [T][16], and the A-side K tail of every row written into the operand image:
// (1, 1, -2^50 at each slot holding the row's component).  The scan then takes the row
// tile as copied (no per-row-tile prep); B tails are rewritten per item in shared memory.
__global__ void tc_tails_kernel(float* __restrict__ img, const int* __restrict__ comp, int T,
                                int d, int* __restrict__ slots) {
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  const int kc = min(8, TC_K - d - 2);
  int* rec = slots + (int64_t)t * 16;
  const int* c = comp + (int64_t)t * TILE;
  select_slots(c, rec, rec + 8, lane, kc);
  int slot[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) slot[k] = rec[k];
  float* tile = img + (int64_t)t * TC_TILE_FLOATS;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int row = lane + 32 * k;
    write_tail(tile, row, d, kc, 1.f, 1.f, slot_hits(c[row], slot), TC_MASK);
  }
}

// ---------------------------------------------------------------- operand image
__global__ void tc_prepare_kernel(const double* __restrict__ X64p, const int* __restrict__ porig,
                                  const double* __restrict__ tcenter64,
                                  const double* __restrict__ normp, int64_t np, int d,
                                  float* __restrict__ img, float* __restrict__ tnorm,
                                  float* __restrict__ eta, float* __restrict__ meta,
                                  float* __restrict__ sq) {
  const int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= np) return;
  const int64_t T0 = pos / TILE;
  const int r = (int)(pos % TILE);
  if (r < TC_META && r != 32 && r != 33)  // centre (zero padded); tR / tEta: tc_tile_max_kernel
    meta[T0 * TC_META + r] = r < d ? __double2float_rn(tcenter64[T0 * d + r]) : 0.f;
  float xt[TC_K];
#pragma unroll
  for (int k = 0; k < TC_K; ++k) xt[k] = 0.f;
  if (porig[pos] >= 0) {
    double xc2 = 0.0, tn2 = 0.0;
#pragma unroll
    for (int k = 0; k < TC_K; ++k) {
      if (k < d) {
        const float x32 = __double2float_rn(X64p[pos * d + k]);
        const float c = __double2float_rn(tcenter64[T0 * d + k]);
        const float xc = __fsub_rn(x32, c);
        const float t = tf32_rna(xc);
        xt[k] = t;
        xc2 += (double)xc * (double)xc;
        tn2 += (double)t * (double)t;
      }
    }
    const double u = 5.9604644775390625e-08;
    tnorm[pos] = float_up(sqrt(tn2) * (1.0 + 1e-12));
    float q = 0.f;  // |x_t|^2 as an fp32 FMA chain (inside the (d+3) u (|x_t| + |D|)^2 term)
#pragma unroll
    for (int k = 0; k < TC_K; ++k)
      if (k < d) q = fmaf(xt[k], xt[k], q);
    sq[pos] = q;
    eta[pos] = float_up((u * normp[pos] + (1.001 * u + 4.8828125e-04) * sqrt(xc2)) * 1.0001 + 1e-30);
  } else {
    tnorm[pos] = 0.f;
    eta[pos] = 0.f;
    sq[pos] = 0.f;
  }
  float* o = img + T0 * TC_TILE_FLOATS;
#pragma unroll
  for (int c = 0; c < 8; ++c)
    *reinterpret_cast<float4*>(o + swz(r, c)) =
        make_float4(xt[4 * c], xt[4 * c + 1], xt[4 * c + 2], xt[4 * c + 3]);
}

__global__ void tc_tile_max_kernel(const float* __restrict__ tnorm, const float* __restrict__ eta,
                                   float* __restrict__ meta) {
  const int T0 = blockIdx.x;
  float a = tnorm[(int64_t)T0 * TILE + threadIdx.x], b = eta[(int64_t)T0 * TILE + threadIdx.x];
  for (int o = 16; o > 0; o >>= 1) {
    a = fmaxf(a, __shfl_xor_sync(0xFFFFFFFFu, a, o));
    b = fmaxf(b, __shfl_xor_sync(0xFFFFFFFFu, b, o));
  }
  __shared__ float sa[4], sb[4];
  if ((threadIdx.x & 31) == 0) {
    sa[threadIdx.x >> 5] = a;
    sb[threadIdx.x >> 5] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    meta[(int64_t)T0 * TC_META + 32] = fmaxf(fmaxf(sa[0], sa[1]), fmaxf(sa[2], sa[3]));
    meta[(int64_t)T0 * TC_META + 33] = fmaxf(fmaxf(sb[0], sb[1]), fmaxf(sb[2], sb[3]));
  }
}

// Error-model probe: for dumped accumulators of `items`, compare the rigorous key L
// and the bound with the exact scipy-order FP64 value S of every real, distinct pair.
// out[0] = max |v - S| / bound (atomicMax on the bits of a nonnegative float),
// out[1] = pairs with L > S (must be 0), out[2] = pairs checked.
__global__ void tc_probe_kernel(TcArgs p, const double* __restrict__ X64p, const int2* __restrict__ items,
                                int64_t nitems, unsigned long long* out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nitems * TILE) return;
  const int64_t q = t / TILE;
  const int i = (int)(t % TILE);
  const int2 it = items[q];
  const int I = it.x, J = it.y, d = p.d;
  const int64_t gi = (int64_t)I * TILE + i;
  if (p.comp[gi] < 0) return;
  float x[32], dl[32];
  load_row(p.img + (int64_t)I * TC_TILE_FLOATS, i, d, x);
  const float dn2 = tc_delta(p.meta + (int64_t)J * TC_META, p.meta + (int64_t)I * TC_META, d, dl);
  const float r = tc_r(p.sq[gi], tc_dot(x, dl, d), dn2);
  float Erow, eta_row;
  tc_bounds(tc_dnorm(dn2, d), d, p.tnorm[gi], p.eta[gi], p.meta[(int64_t)J * TC_META + 32],
            p.meta[(int64_t)J * TC_META + 33], Erow, eta_row);
  float worst = 0.f;
  unsigned long long bad = 0, cnt = 0;
  for (int j = 0; j < TILE; ++j) {
    const int64_t gj = (int64_t)J * TILE + j;
    if (gj == gi || p.comp[gj] < 0 || p.comp[gj] == p.comp[gi]) continue;
    const float G = p.dump[(q * TILE + i) * TILE + j];
    const float v = __fmaf_rn(-2.f, G, r);
    const float L = lower_key(v, Erow, eta_row);
    double S = 0.0;
    for (int k = 0; k < d; ++k) {
      const double dd = __dsub_rn(X64p[gi * d + k], X64p[gj * d + k]);
      S = __dadd_rn(S, __dmul_rn(dd, dd));
    }
    const double e = (double)eta_row;
    const double bound = (double)Erow + 1.02 * 5.9604644775390625e-08 * fabs((double)v) +
                         2.0 * e * sqrt(S) + e * e;
    const float ratio = (float)(fabs((double)v - S) / bound);
    worst = fmaxf(worst, ratio);
    bad += ((double)L > S);
    ++cnt;
  }
  atomicMax(out, (unsigned long long)__float_as_uint(worst));
  if (bad) atomicAdd(out + 1, bad);
  atomicAdd(out + 2, cnt);
}

}  // namespace

cudaError_t launch_tc_probe(const TcArgs& a, const double* X64p, const int2* items, int64_t n,
                            unsigned long long* out, cudaStream_t st) {
  tc_probe_kernel<<<(unsigned)((n * TILE + 127) / 128), 128, 0, st>>>(a, X64p, items, n, out);
  return cudaGetLastError();
}

size_t tc_smem_bytes() { return sizeof(TcSmem) + 1024; }

bool tc_supported(int d) { return d >= 1 && d <= TC_MAX_D; }

template <int DC>
static cudaError_t launch_tc_d(const TcArgs& a, int grid, cudaStream_t st) {
  const size_t sm = tc_smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(tc_scan_kernel<DC>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) {
    fprintf(stderr, "[nnm] tc_scan smem attribute (%zu B) failed: %s\n", sm, cudaGetErrorString(e));
    return e;
  }
  tc_scan_kernel<DC><<<grid, TC_THREADS, sm, st>>>(a);
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, tc_scan_kernel<DC>) == cudaSuccess)
      fprintf(stderr, "[nnm] tc_scan launch failed: regs %d maxThreads %d smem %zu+%zu localBytes %zu\n",
              fa.numRegs, fa.maxThreadsPerBlock, fa.sharedSizeBytes, sm, fa.localSizeBytes);
  }
  return e;
}

__global__ void tc_exact_kernel(const unsigned long long* __restrict__ cand,
                                const unsigned long long* __restrict__ count, int64_t cap,
                                const double* __restrict__ X64, int d, float thr_hi,
                                unsigned long long* B1, unsigned long long* B2) {
  const int64_t n = min((int64_t)*count, cap);
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long c = cand[t];
    const int64_t g = (int64_t)(c >> 32), gj = (int64_t)(c & 0xFFFFFFFFull);
    const float L = float_down(exact_dist<EUCLIDEAN>(X64 + g * d, X64 + gj * d, d));
    if (!(L <= thr_hi)) continue;
    const unsigned long long key = ((unsigned long long)__float_as_uint(L) << 32) | (unsigned)gj;
    const unsigned long long old = atomicMin(B1 + g, key);  // atomic top-2 insert
    const unsigned long long disp = key < old ? old : key;
    if (key_valid(disp)) atomicMin(B2 + g, disp);
  }
}

cudaError_t launch_tc_exact(const unsigned long long* cand, const unsigned long long* count,
                            int64_t cap, const double* X64, int d, float thr_hi,
                            unsigned long long* B1, unsigned long long* B2, cudaStream_t st) {
  tc_exact_kernel<<<148 * 8, 256, 0, st>>>(cand, count, cap, X64, d, thr_hi, B1, B2);
  return cudaGetLastError();
}

cudaError_t launch_tc_tails(float* img, const int* comp, int T, int d, int* slots, cudaStream_t st) {
  tc_tails_kernel<<<(T + 7) / 8, 256, 0, st>>>(img, comp, T, d, slots);
  return cudaGetLastError();
}

cudaError_t launch_tc_scan(const TcArgs& a, int grid, cudaStream_t st) {
  // the BASELINE shapes get compile-time d (straight-line tails); others run generic
  if (a.d == 25) return launch_tc_d<25>(a, grid, st);
  if (a.d == 8) return launch_tc_d<8>(a, grid, st);
  return launch_tc_d<0>(a, grid, st);
}

cudaError_t launch_tc_prepare(const double* X64p, const int* porig, const double* tcenter64,
                              const double* normp, int64_t np, int d, int T, float* img,
                              float* tnorm, float* eta, float* meta, float* sq, cudaStream_t st) {
  tc_prepare_kernel<<<(unsigned)((np + 255) / 256), 256, 0, st>>>(X64p, porig, tcenter64, normp, np,
                                                                  d, img, tnorm, eta, meta, sq);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  tc_tile_max_kernel<<<T, TILE, 0, st>>>(tnorm, eta, meta);
  return cudaGetLastError();
}


}  // namespace nnm
