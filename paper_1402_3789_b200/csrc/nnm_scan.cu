// nnm_scan.cu -- fused FP32 distance + eligibility + nearest-pair kernels (sm_100a).
//
// Replaces the reference's distance/selection stack
//   metrics.internal_pairwise -> scipy cdist      (metrics.py:67-73)
//   pairgen._mask_ineligible                       (pairgen.py:190-210)
//   pairgen._chunk_candidates / scan_block_pair    (pairgen.py:213-298)
// with one kernel that never materialises the n x n matrix.  The FP32 values
// computed here only SCREEN; every order-deciding key is re-evaluated in FP64
// (nnm_exact.cu) with a rigorous error margin (nnm_common.cuh ErrModel).
//
// Tiling: a CTA owns a contiguous run of upper-triangular 128x128 tile pairs
// (I <= J) in row-major order, so the row tile I stays in shared memory and
// its per-row best keys accumulate in shared memory across consecutive J.
// 8 warps as 4 (rows) x 2 (cols); a warp covers 32 rows x 64 cols; a thread
// covers 8 x 8 pairs with FADD2/FFMA2 (packed fp32x2) arithmetic.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "nnm_common.cuh"
#include "nnm_kernels.cuh"

namespace nnm {

// ----------------------------------------------------------------------------
// helpers
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint32_t umin3(uint32_t a, uint32_t b, uint32_t c) {
  return min(min(a, b), c);
}

// Insert a top-2 pair (k1 <= k2) into an atomic top-2 (G1, G2).  Order
// independent: after all inserts G1 = min key, G2 = second-smallest key.
__device__ __forceinline__ void insert_top2(unsigned long long* G1, unsigned long long* G2,
                                            unsigned long long k1, unsigned long long k2) {
  if (!key_valid(k1)) return;
  unsigned long long old = atomicMin(G1, k1);
  if (G2 == nullptr) return;
  unsigned long long disp = (k1 < old) ? old : k1;
  unsigned long long m = disp < k2 ? disp : k2;
  if (key_valid(m)) atomicMin(G2, m);
}

// The same insert split in two so that the returning atomicMin's latency overlaps the next
// item's arithmetic: start() issues the G1 atomic and keeps (k1, k2, old); finish() -- at the
// thread's next start() or at the end of the kernel -- derives the displaced key and issues
// the (non-returning) G2 atomic.  The protocol stays order independent (each displacement
// is decided by the atomic's return value); other readers of G2 in between only see a
// looser (larger) second-best key, which is safe for thresholds.
struct Top2Flush {
  bool pend = false;
  unsigned long long* g2 = nullptr;
  unsigned long long k1 = 0, k2 = 0, old = 0;
  __device__ __forceinline__ void finish() {
    if (!pend) return;
    pend = false;
    const unsigned long long disp = (k1 < old) ? old : k1;
    const unsigned long long m = disp < k2 ? disp : k2;
    if (key_valid(m)) atomicMin(g2, m);
  }
  __device__ __forceinline__ void start(unsigned long long* G1, unsigned long long* G2,
                                        unsigned long long a1, unsigned long long a2) {
    finish();
    if (!key_valid(a1)) return;
    if (G2 == nullptr) {
      atomicMin(G1, a1);
      return;
    }
    old = atomicMin(G1, a1);
    k1 = a1;
    k2 = a2;
    g2 = G2;
    pend = true;
  }
};

__device__ __forceinline__ void decode_work(int64_t w, int T, int& I, int& J) {
  // start(I) = I*T - I*(I-1)/2 ; find the largest I with start(I) <= w
  double tt = 2.0 * T + 1.0;
  double disc = tt * tt - 8.0 * (double)w;
  int i = (int)floor((tt - sqrt(disc > 0 ? disc : 0)) * 0.5);
  if (i < 0) i = 0;
  if (i > T - 1) i = T - 1;
  auto start = [T](int64_t x) { return x * T - x * (x - 1) / 2; };
  while (i + 1 < T && start(i + 1) <= w) ++i;
  while (i > 0 && start(i) > w) --i;
  I = i;
  J = i + (int)(w - start(i));
}

// Work item w -> tile pair (I, J): either the row-major upper triangle or an
// explicit list (pruned scans), in both cases sorted by I so row tiles are reused.
__device__ __forceinline__ void first_item(const ScanArgs& p, int64_t w, int& I, int& J) {
  if (p.items) {
    const int2 it = __ldg(p.items + w);
    I = it.x;
    J = it.y;
  } else {
    decode_work(w, p.T, I, J);
  }
}

__device__ __forceinline__ void next_item(const ScanArgs& p, int64_t w, int I, int J, int& In,
                                          int& Jn) {
  if (p.items) {
    const int2 it = (w + 1 < p.w_end) ? __ldg(p.items + w + 1) : make_int2(I, J);
    In = it.x;
    Jn = it.y;
  } else {
    In = I;
    Jn = J + 1;
    if (Jn == p.T) {
      ++In;
      Jn = In;
    }
  }
}

template <int M>
__device__ __forceinline__ void accumulate(float2& acc, float2 y, float x) {
  float2 dd = __fadd2_rn(y, make_float2(-x, -x));
  if (M == EUCLIDEAN || M == SQEUCLIDEAN) {
    acc = __ffma2_rn(dd, dd, acc);
  } else if (M == MANHATTAN) {
    acc = __fadd2_rn(acc, make_float2(fabsf(dd.x), fabsf(dd.y)));
  } else {
    acc.x = fmaxf(acc.x, fabsf(dd.x));
    acc.y = fmaxf(acc.y, fabsf(dd.y));
  }
}

// Warp-local column of a thread's column slot c (0..7): two float4 groups 32
// columns apart, so the 8 lanes of an LDS.128 phase read 128 contiguous bytes
// (bank-conflict free).  Within the CTA tile: wc*64 + wcol(tc, c).
__device__ __forceinline__ int wcol(int tc, int c) { return (c >> 2) * 32 + tc * 4 + (c & 3); }

template <int M>
__device__ __forceinline__ void fma_step(float2 (&acc)[8][4], float4 xa, float4 xb, float4 ya,
                                         float4 yb) {
  const float xr[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
  const float2 yc[4] = {make_float2(ya.x, ya.y), make_float2(ya.z, ya.w), make_float2(yb.x, yb.y),
                        make_float2(yb.z, yb.w)};
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int q = 0; q < 4; ++q) accumulate<M>(acc[r][q], yc[q], xr[r]);
}

// 8x8 register tile: rows row0..row0+7 of sX, columns colw + wcol(tc, 0..7) of sY.
template <int M>
__device__ __forceinline__ void tile_8x8(const float* __restrict__ sX, const float* __restrict__ sY,
                                         int d, int row0, int colw, int tc, float2 (&acc)[8][4]) {
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[r][q] = make_float2(0.f, 0.f);
  const float* __restrict__ xp = sX + row0;
  const float* __restrict__ yp = sY + colw + tc * 4;
  // software-pipelined with two register sets (no copies: IMAD.MOV would run on
  // the FMA pipe): operands of k+1 load while k computes, hiding LDS latency
  // behind 64 FMA-pipe instructions even at 2 compute warps per SMSP.
  // Pointers advance by TILE floats per k (integer adds on the ALU pipe; IMAD
  // address math would take FMA-pipe cycles from FFMA2/FADD2).
  float4 a0 = *reinterpret_cast<const float4*>(xp), a1 = *reinterpret_cast<const float4*>(xp + 4);
  float4 a2 = *reinterpret_cast<const float4*>(yp), a3 = *reinterpret_cast<const float4*>(yp + 32);
  int k = 0;
#pragma unroll 1
  for (; k + 2 < d; k += 2) {
    const float4 b0 = *reinterpret_cast<const float4*>(xp + TILE);
    const float4 b1 = *reinterpret_cast<const float4*>(xp + TILE + 4);
    const float4 b2 = *reinterpret_cast<const float4*>(yp + TILE);
    const float4 b3 = *reinterpret_cast<const float4*>(yp + TILE + 32);
    fma_step<M>(acc, a0, a1, a2, a3);
    xp += 2 * TILE;
    yp += 2 * TILE;
    a0 = *reinterpret_cast<const float4*>(xp);
    a1 = *reinterpret_cast<const float4*>(xp + 4);
    a2 = *reinterpret_cast<const float4*>(yp);
    a3 = *reinterpret_cast<const float4*>(yp + 32);
    fma_step<M>(acc, b0, b1, b2, b3);
  }
  if (k + 1 < d) {  // two k left: a holds k, load k+1
    const float4 b0 = *reinterpret_cast<const float4*>(xp + TILE);
    const float4 b1 = *reinterpret_cast<const float4*>(xp + TILE + 4);
    const float4 b2 = *reinterpret_cast<const float4*>(yp + TILE);
    const float4 b3 = *reinterpret_cast<const float4*>(yp + TILE + 32);
    fma_step<M>(acc, a0, a1, a2, a3);
    fma_step<M>(acc, b0, b1, b2, b3);
  } else {
    fma_step<M>(acc, a0, a1, a2, a3);
  }
}

// dot form: acc += yh * xh (one FFMA2 per two pairs and coordinate)
__device__ __forceinline__ void dot_step(float2 (&acc)[8][4], float4 xa, float4 xb, float4 ya,
                                         float4 yb) {
  const float xr[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
  const float2 yc[4] = {make_float2(ya.x, ya.y), make_float2(ya.z, ya.w), make_float2(yb.x, yb.y),
                        make_float2(yb.z, yb.w)};
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[r][q] = __ffma2_rn(yc[q], make_float2(xr[r], xr[r]), acc[r][q]);
}

__device__ __forceinline__ void tile_dot_8x8(const float* __restrict__ sX,
                                             const float* __restrict__ sY, int d, int row0,
                                             int colw, int tc, float2 (&acc)[8][4],
                                             bool zero = true) {
  if (zero) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[r][q] = make_float2(0.f, 0.f);
  }
  const float* __restrict__ xp = sX + row0;
  const float* __restrict__ yp = sY + colw + tc * 4;
  float4 a0 = *reinterpret_cast<const float4*>(xp), a1 = *reinterpret_cast<const float4*>(xp + 4);
  float4 a2 = *reinterpret_cast<const float4*>(yp), a3 = *reinterpret_cast<const float4*>(yp + 32);
  int k = 0;
#pragma unroll 1
  for (; k + 2 < d; k += 2) {
    const float4 b0 = *reinterpret_cast<const float4*>(xp + TILE);
    const float4 b1 = *reinterpret_cast<const float4*>(xp + TILE + 4);
    const float4 b2 = *reinterpret_cast<const float4*>(yp + TILE);
    const float4 b3 = *reinterpret_cast<const float4*>(yp + TILE + 32);
    dot_step(acc, a0, a1, a2, a3);
    xp += 2 * TILE;
    yp += 2 * TILE;
    a0 = *reinterpret_cast<const float4*>(xp);
    a1 = *reinterpret_cast<const float4*>(xp + 4);
    a2 = *reinterpret_cast<const float4*>(yp);
    a3 = *reinterpret_cast<const float4*>(yp + 32);
    dot_step(acc, b0, b1, b2, b3);
  }
  if (k + 1 < d) {
    const float4 b0 = *reinterpret_cast<const float4*>(xp + TILE);
    const float4 b1 = *reinterpret_cast<const float4*>(xp + TILE + 4);
    const float4 b2 = *reinterpret_cast<const float4*>(yp + TILE);
    const float4 b3 = *reinterpret_cast<const float4*>(yp + TILE + 32);
    dot_step(acc, a0, a1, a2, a3);
    dot_step(acc, b0, b1, b2, b3);
  } else {
    dot_step(acc, a0, a1, a2, a3);
  }
}

__device__ __forceinline__ float acc_at(const float2 (&acc)[8][4], int r, int c) {
  return (c & 1) ? acc[r][c >> 1].y : acc[r][c >> 1].x;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// async copy of a 128-point SoA tile [d][128] (+ its comp / size labels)
__device__ __forceinline__ void async_tile(float* __restrict__ s, int* __restrict__ sc,
                                           int* __restrict__ ss, const float* __restrict__ X32,
                                           int64_t ld, int tile, int d, const int* __restrict__ comp,
                                           const int* __restrict__ psize, bool sizes) {
  const int nvec = d * (TILE / 4);
  const float* base = X32 + (int64_t)tile * TILE;
  for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
    int k = v >> 5, q = v & 31;
    cp_async16(s + k * TILE + q * 4, base + (int64_t)k * ld + q * 4);
  }
  const int t = threadIdx.x;
  if (t < 32) cp_async16(sc + t * 4, comp + (int64_t)tile * TILE + t * 4);
  else if (sizes && t < 64) cp_async16(ss + (t - 32) * 4, psize + (int64_t)tile * TILE + (t - 32) * 4);
}

// synchronous variant for the collect kernel (gathered sources)
__device__ __forceinline__ void load_tile(float* __restrict__ s, const float* __restrict__ X32,
                                          int64_t ld, int tile, int d) {
  const int nvec = d * (TILE / 4);
  for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
    int k = v / (TILE / 4), q = v % (TILE / 4);
    reinterpret_cast<float4*>(s + k * TILE)[q] =
        __ldg(reinterpret_cast<const float4*>(X32 + (int64_t)k * ld + (int64_t)tile * TILE) + q);
  }
}

__device__ __forceinline__ void merge2(unsigned long long& a1, unsigned long long& a2,
                                       unsigned long long b1, unsigned long long b2) {
  unsigned long long lo = a1 < b1 ? a1 : b1;
  unsigned long long hi = a1 < b1 ? b1 : a1;
  unsigned long long m2 = a2 < b2 ? a2 : b2;
  a1 = lo;
  a2 = hi < m2 ? hi : m2;
}

// ----------------------------------------------------------------------------
// K1: per-row best-2 (or best-1) eligible partner over a range of tile pairs.
//
// Persistent CTA over a contiguous run of tile pairs (I <= J, row-major), so the
// row tile stays in shared memory and its running top-2 lives in shared memory
// (one owner thread per row, no atomics) until I changes.  Column tiles are
// double-buffered with cp.async.  Cross-warp partials go through shared memory;
// only per-tile column results and per-I row results touch global atomics.
// ----------------------------------------------------------------------------
template <int M, bool TOP2, bool SIZES, bool THR>
__global__ void __launch_bounds__(SCAN_THREADS, 2) scan_rows_kernel(ScanArgs p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int dT = p.d * TILE;
  float* sX = reinterpret_cast<float*>(smem_raw);
  float* sY0 = sX + dT;  // two buffers: sY0, sY0 + dT
  unsigned long long* rowPart = reinterpret_cast<unsigned long long*>(sY0 + 2 * dT);  // [2][128][2]
  unsigned long long* colPart = rowPart + 2 * TILE * 2;                               // [4][128][2]
  unsigned long long* rowRun = colPart + 4 * TILE * 2;                                // [128][2]
  int* sCompR = reinterpret_cast<int*>(rowRun + TILE * 2);
  int* sSizeR = sCompR + TILE;
  int* sCompC0 = sSizeR + TILE;  // [2][128]
  int* sSizeC0 = sCompC0 + 2 * TILE;  // [2][128]

  const int64_t total = p.w_end - p.w_begin;
  const int64_t per = (total + gridDim.x - 1) / gridDim.x;
  const int64_t w0 = p.w_begin + (int64_t)blockIdx.x * per;
  const int64_t w1 = min(w0 + per, p.w_end);
  if (w0 >= w1) return;
  Top2Flush gflush;  // this thread's pending global top-2 insert

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wr = warp >> 1, wc = warp & 1;
  const int tr = lane >> 3, tc = lane & 7;
  const int row0 = wr * 32 + tr * 8;
  const int colw = wc * 64;

  int I, J;
  first_item(p, w0, I, J);
  async_tile(sX, sCompR, sSizeR, p.X32, p.ld, I, p.d, p.comp, p.psize, SIZES);
  async_tile(sY0, sCompC0, sSizeC0, p.X32, p.ld, J, p.d, p.comp, p.psize, SIZES);
  cp_async_commit();
  if (tid < TILE) {
    rowRun[2 * tid] = NONE_KEY;
    rowRun[2 * tid + 1] = NONE_KEY;
  }
  cp_async_wait_all();
  __syncthreads();

  int buf = 0;
  for (int64_t w = w0; w < w1; ++w) {
    // ---- prefetch the next column tile into the other buffer
    int In, Jn;
    next_item(p, w, I, J, In, Jn);
    const bool has_next = (w + 1 < w1);
    if (has_next) {
      async_tile(sY0 + (buf ^ 1) * dT, sCompC0 + (buf ^ 1) * TILE, sSizeC0 + (buf ^ 1) * TILE,
                 p.X32, p.ld, Jn, p.d, p.comp, p.psize, SIZES);
      cp_async_commit();
    }
    const float* sY = sY0 + buf * dT;
    const int* sCompC = sCompC0 + buf * TILE;
    const int* sSizeC = sSizeC0 + buf * TILE;
    const bool diag = (I == J);
    // component labels of the two tiles may coincide only if their ranges overlap
    const int2 rI = __ldg(p.tile_range + I), rJ = __ldg(p.tile_range + J);
    const bool may_share = diag || !(rI.y < rJ.x || rJ.y < rI.x);

    float2 acc[8][4];
    tile_8x8<M>(sX, sY, p.d, row0, colw, tc, acc);

    int cr[8], cc[8], sr[8], sc[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      cr[t] = sCompR[row0 + t];
      cc[t] = sCompC[colw + wcol(tc, t)];
      if (SIZES) {
        sr[t] = sSizeR[row0 + t];
        sc[t] = sSizeC[colw + wcol(tc, t)];
      }
    }
    uint32_t rk1[8], rk2[8], ck1[8], ck2[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      rk1[t] = 0xFFFFFFFFu;
      rk2[t] = 0xFFFFFFFFu;
      ck1[t] = 0xFFFFFFFFu;
      ck2[t] = 0xFFFFFFFFu;
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        float v = acc_at(acc, r, c);
        bool ok = true;
        if (may_share) ok = cr[r] != cc[c];
        if (SIZES) ok = ok && (sr[r] + sc[c] <= p.ksum);
        if (THR) ok = ok && (v <= p.thr_hi);
        uint32_t bits = ok ? __float_as_uint(v) : INF_BITS;
        uint32_t kr = (bits & ~63u) | (uint32_t)wcol(tc, c);
        if (TOP2) rk2[r] = min(rk2[r], max(rk1[r], kr));
        rk1[r] = min(rk1[r], kr);
        if (!diag) {
          uint32_t kc = (bits & ~31u) | (uint32_t)(tr * 8 + r);
          if (TOP2) ck2[c] = min(ck2[c], max(ck1[c], kc));
          ck1[c] = min(ck1[c], kc);
        }
      }
    }
    // ---- row side: merge across the 8 lanes sharing rows (xor 1,2,4)
#pragma unroll
    for (int s = 1; s < 8; s <<= 1) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        uint32_t o1 = __shfl_xor_sync(0xFFFFFFFFu, rk1[r], s);
        if (TOP2) {
          uint32_t o2 = __shfl_xor_sync(0xFFFFFFFFu, rk2[r], s);
          rk2[r] = umin3(max(rk1[r], o1), rk2[r], o2);
        }
        rk1[r] = min(rk1[r], o1);
      }
    }
    {
      uint32_t s1 = 0xFFFFFFFFu, s2 = 0xFFFFFFFFu;
#pragma unroll
      for (int r = 0; r < 8; ++r)
        if (r == tc) {
          s1 = rk1[r];
          s2 = rk2[r];
        }
      const unsigned long long jb = (unsigned long long)J * TILE + colw;
      unsigned long long k1 = ((s1 & ~63u) >= INF_BITS)
                                  ? NONE_KEY
                                  : (((unsigned long long)(s1 & ~63u) << 32) | (jb + (s1 & 63u)));
      unsigned long long k2 = NONE_KEY;
      if (TOP2 && (s2 & ~63u) < INF_BITS)
        k2 = ((unsigned long long)(s2 & ~63u) << 32) | (jb + (s2 & 63u));
      unsigned long long* dst = rowPart + (wc * TILE + row0 + tc) * 2;
      dst[0] = k1;
      dst[1] = k2;
    }
    // ---- col side: merge across the 4 lanes sharing columns (xor 8,16)
    if (!diag) {
#pragma unroll
      for (int s = 8; s < 32; s <<= 1) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint32_t o1 = __shfl_xor_sync(0xFFFFFFFFu, ck1[c], s);
          if (TOP2) {
            uint32_t o2 = __shfl_xor_sync(0xFFFFFFFFu, ck2[c], s);
            ck2[c] = umin3(max(ck1[c], o1), ck2[c], o2);
          }
          ck1[c] = min(ck1[c], o1);
        }
      }
      const unsigned long long ib = (unsigned long long)I * TILE + wr * 32;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t s1 = 0xFFFFFFFFu, s2 = 0xFFFFFFFFu;
        const int want = tr * 2 + h;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c == want) {
            s1 = ck1[c];
            s2 = ck2[c];
          }
        unsigned long long k1 = ((s1 & ~31u) >= INF_BITS)
                                    ? NONE_KEY
                                    : (((unsigned long long)(s1 & ~31u) << 32) | (ib + (s1 & 31u)));
        unsigned long long k2 = NONE_KEY;
        if (TOP2 && (s2 & ~31u) < INF_BITS)
          k2 = ((unsigned long long)(s2 & ~31u) << 32) | (ib + (s2 & 31u));
        unsigned long long* dst = colPart + (wr * TILE + colw + wcol(tc, want)) * 2;
        dst[0] = k1;
        dst[1] = k2;
      }
    }
    __syncthreads();  // (A) partials complete; sX / sY[buf] no longer read
    if (tid < TILE) {
      unsigned long long a1 = rowRun[2 * tid], a2 = rowRun[2 * tid + 1];
      merge2(a1, a2, rowPart[2 * tid], rowPart[2 * tid + 1]);
      merge2(a1, a2, rowPart[2 * (TILE + tid)], rowPart[2 * (TILE + tid) + 1]);
      const bool flush = !has_next || In != I;
      if (flush) {
        const int g = I * TILE + tid;
        if (g < p.n) gflush.start(p.B1 + g, TOP2 ? p.B2 + g : nullptr, a1, a2);
        a1 = NONE_KEY;
        a2 = NONE_KEY;
      }
      rowRun[2 * tid] = a1;
      rowRun[2 * tid + 1] = a2;
    } else if (!diag) {
      const int c = tid - TILE;
      unsigned long long a1 = colPart[2 * c], a2 = colPart[2 * c + 1];
#pragma unroll
      for (int q = 1; q < 4; ++q) merge2(a1, a2, colPart[2 * (q * TILE + c)], colPart[2 * (q * TILE + c) + 1]);
      const int g = J * TILE + c;
      if (g < p.n) gflush.start(p.B1 + g, TOP2 ? p.B2 + g : nullptr, a1, a2);
    }
    if (has_next && In != I) {
      async_tile(sX, sCompR, sSizeR, p.X32, p.ld, In, p.d, p.comp, p.psize, SIZES);
      cp_async_commit();
    }
    cp_async_wait_all();
    __syncthreads();  // (B) next tiles resident, row/col partial buffers free
    I = In;
    J = Jn;
    buf ^= 1;
  }
  gflush.finish();
}

size_t scan_smem_bytes(int d) {
  return (size_t)3 * d * TILE * sizeof(float) + (2 + 4 + 1) * TILE * 2 * sizeof(unsigned long long) +
         6 * TILE * sizeof(int);
}

static int g_ws_mode = -1;  // -1: auto, 0: force classic, 1: force warp-specialised

bool scan_use_ws(int d) {
  if (g_ws_mode < 0) {  // NNM_SCAN_KERNEL=classic|ws (A/B switch for profiling)
    const char* e = getenv("NNM_SCAN_KERNEL");
    g_ws_mode = (e && e[0] == 'c') ? 0 : 2;
  }
  if (g_ws_mode == 0) return false;
  return scan_ws_smem_bytes(d) <= 200 * 1024;
}

void scan_set_mode(int mode) { g_ws_mode = mode; }

// register-epilogue kernel: the default for Boruvka (top-2) scans
bool scan_use_reg(const ScanArgs& a) {
  if (scan_reg_smem_bytes(a.d) > 110 * 1024) return false;
  const char* e = getenv("NNM_SCAN_KERNEL");
  if (e && e[0] == 'r') return true;
  if (e && (e[0] == 'w' || e[0] == 'c')) return false;
  // top-2 (Boruvka) scans: the filter thresholds come from second-best keys
  // that fill quickly; top-1 round scans (fresh B1 every round) stay on WS
  return a.B2 != nullptr;
}

int scan_occupancy(int metric, int d) {
  if (scan_use_ws(d)) return 1;  // (the register kernel also runs 2 CTAs / SM: see launch)
  int blocks = 0;
  size_t sm = scan_smem_bytes(d);
  cudaFuncSetAttribute(scan_rows_kernel<EUCLIDEAN, true, false, false>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &blocks, scan_rows_kernel<EUCLIDEAN, true, false, false>, SCAN_THREADS, sm);
  return blocks > 0 ? blocks : 1;
}


// ----------------------------------------------------------------------------
// K1-WS: warp-specialised variant of K1 (the default for d <= WS_MAX_D).
//
// 8 compute warps stream 128x128 distance tiles (FADD2/FFMA2, 8x8 per thread)
// into a double-buffered, XOR-swizzled shared tile; 4 epilogue warps consume
// it concurrently: thread t owns row t and column t of the tile, applies the
// eligibility rule and keeps the top-2 keys.  Producer / consumer hand-off uses
// named barriers (FULL[b], EMPTY[b]), so the selection work (integer pipe)
// overlaps the distance math (FMA pipe) instead of following it.
// Swizzle: element (r, c) lives at r*128 + ((c/4 ^ (r & 31)) * 4) + c%4, which
// makes the compute warps' STS.128, the row readers' LDS.128 and the column
// readers' scalar LDS all bank-conflict free.
// ----------------------------------------------------------------------------
constexpr int WS_COMPUTE_THREADS = 256;
constexpr int WS_EPI_THREADS = 256;  // 128 row owners + 128 column owners
constexpr int WS_THREADS = WS_COMPUTE_THREADS + WS_EPI_THREADS;

__device__ __forceinline__ void bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ int swz(int r, int q) { return r * TILE + ((q ^ (r & 31)) << 2); }

// running top-2 of u32 keys, two new keys at a time (5 integer min/max ops)
__device__ __forceinline__ void top2_pair(uint32_t& m1, uint32_t& m2, uint32_t a, uint32_t b) {
  const uint32_t lo = min(a, b), hi = max(a, b);
  m2 = umin3(max(m1, lo), m2, hi);
  m1 = min(m1, lo);
}

__device__ __forceinline__ unsigned long long widen(uint32_t k, unsigned long long base) {
  return ((k & ~63u) >= INF_BITS) ? NONE_KEY
                                  : (((unsigned long long)(k & ~63u) << 32) | (base + (k & 63u)));
}

template <int M, bool TOP2, bool SIZES, bool THR, bool DOT>
__global__ void __launch_bounds__(WS_THREADS, 1) scan_ws_kernel(ScanArgs p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int dT = p.d * TILE;
  float* sD = reinterpret_cast<float*>(smem_raw);  // [2][128*128]
  float* sX0 = sD + 2 * TILE * TILE;               // [2][d*128]
  float* sY0 = sX0 + 2 * dT;                       // [2][d*128]
  int* sCR = reinterpret_cast<int*>(sY0 + 2 * dT);  // [2][128] row comps (epilogue)
  int* sCC = sCR + 2 * TILE;                        // [2][128] col comps
  int* sSR = sCC + 2 * TILE;                        // [2][128] row eff sizes
  int* sSC = sSR + 2 * TILE;                        // [2][128] col eff sizes
  float* sNB = reinterpret_cast<float*>(sSC + 2 * TILE);  // [2][128] row -B/(1+A) (dot)
  float* sNX = sNB + 2 * TILE;                            // [2 xb][2 halves][128] row norms
  float* sNY = sNX + 4 * TILE;                            // [2 buf][2 halves][128] col norms

  const int64_t total = p.w_end - p.w_begin;
  const int64_t per = (total + gridDim.x - 1) / gridDim.x;
  const int64_t w0 = p.w_begin + (int64_t)blockIdx.x * per;
  const int64_t w1 = min(w0 + per, p.w_end);
  if (w0 >= w1) return;
  Top2Flush gflush;  // this thread's pending global top-2 insert
  const int tid = threadIdx.x;
  int I, J;
  first_item(p, w0, I, J);

  if (tid < WS_COMPUTE_THREADS) {
    // =========================== compute warps ===========================
    const int warp = tid >> 5, lane = tid & 31;
    const int wr = warp >> 1, wc = warp & 1;
    const int tr = lane >> 3, tc = lane & 7;
    const int row0 = wr * 32 + tr * 8;
    const int colw = wc * 64;
    // prologue loads (compute threads only; blockDim for the copy loops is 256)
    {
      const int nvec = p.d * (TILE / 4);
      for (int v = tid; v < nvec; v += WS_COMPUTE_THREADS) {
        int k = v >> 5, q = v & 31;
        cp_async16(sX0 + k * TILE + q * 4, p.X32 + (int64_t)k * p.ld + (int64_t)I * TILE + q * 4);
        cp_async16(sY0 + k * TILE + q * 4, p.X32 + (int64_t)k * p.ld + (int64_t)J * TILE + q * 4);
      }
      cp_async_commit();
    }
    int xb = 0;
    bool xfresh = true;
    for (int64_t w = w0; w < w1; ++w) {
      const int buf = (int)((w - w0) & 1);
      int In, Jn;
      next_item(p, w, I, J, In, Jn);
      cp_async_wait_all();
      bar_sync(1, WS_COMPUTE_THREADS);  // tiles for w resident; everyone done with w-1
      const bool xnew = xfresh;  // the row tile in sX[xb] still holds raw coordinates
      xfresh = false;
      if (w + 1 < w1) {
        // this thread copies 16-byte column chunk (tid & 31) of rows k = tid/32 + 8i
        float* ny = sY0 + (buf ^ 1) * dT + (tid >> 5) * TILE + (tid & 31) * 4;
        float* nx = sX0 + (xb ^ 1) * dT + (tid >> 5) * TILE + (tid & 31) * 4;
        const float* gy = p.X32 + (int64_t)(tid >> 5) * p.ld + (int64_t)Jn * TILE + (tid & 31) * 4;
        const float* gx = p.X32 + (int64_t)(tid >> 5) * p.ld + (int64_t)In * TILE + (tid & 31) * 4;
        const int64_t gstep = 8 * p.ld;
        const bool newI = In != I;
        for (int k = tid >> 5; k < p.d; k += 8) {
          cp_async16(ny, gy);
          if (newI) cp_async16(nx, gx);
          ny += 8 * TILE;
          nx += 8 * TILE;
          gy += gstep;
          gx += gstep;
        }
        cp_async_commit();
      }
      if (DOT) {
        // centre both tiles on c_I: yh = y - c_I (and xh when I is new), plus
        // half-norms; thread t owns column / row (t & 127), coordinate half t >> 7
        const int col = tid & (TILE - 1), hk = tid >> 7;
        const int dh = (p.d + 1) >> 1, k0 = hk * dh, k1 = min(p.d, k0 + dh);
        const float* cI = p.dot_center + (int64_t)I * p.d;
        float* yb = sY0 + buf * dT;
        float ny = 0.f;
        for (int k = k0; k < k1; ++k) {
          const float v = yb[k * TILE + col] - __ldg(cI + k);
          yb[k * TILE + col] = v;
          ny = fmaf(v, v, ny);
        }
        sNY[(buf * 2 + hk) * TILE + col] = ny;
        if (w == w0 || xnew) {
          float* xbuf = sX0 + xb * dT;
          float nx = 0.f;
          for (int k = k0; k < k1; ++k) {
            const float v = xbuf[k * TILE + col] - __ldg(cI + k);
            xbuf[k * TILE + col] = v;
            nx = fmaf(v, v, nx);
          }
          sNX[(xb * 2 + hk) * TILE + col] = nx;
        }
        bar_sync(1, WS_COMPUTE_THREADS);
      }
      float2 acc[8][4];
      if (DOT) tile_dot_8x8(sX0 + xb * dT, sY0 + buf * dT, p.d, row0, colw, tc, acc);
      else tile_8x8<M>(sX0 + xb * dT, sY0 + buf * dT, p.d, row0, colw, tc, acc);
      if (DOT) {
        // v = |xh|^2 + |yh|^2 - 2 xh.yh
        const float* nx0 = sNX + (xb * 2) * TILE;
        const float* ny0 = sNY + (buf * 2) * TILE;
        float nxr[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) nxr[r] = nx0[row0 + r] + nx0[TILE + row0 + r];
        float2 nyc[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c0 = colw + wcol(tc, 2 * q);
          nyc[q] = make_float2(ny0[c0] + ny0[TILE + c0], ny0[c0 + 1] + ny0[TILE + c0 + 1]);
        }
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 s2 = __fadd2_rn(nyc[q], make_float2(nxr[r], nxr[r]));
            acc[r][q] = __ffma2_rn(acc[r][q], make_float2(-2.f, -2.f), s2);
          }
      }
      bar_sync(4 + buf, WS_THREADS);  // EMPTY[buf]
      // element (R, 4q..4q+3) -> R*128 + ((q ^ (R & 31)) << 2); with R = row0 + r and
      // q = (wc*2 + h)*8 + tc the XOR splits into ((wc*2+h) ^ tr) << 5 | (tc ^ r) << 2
      float* D = sD + buf * TILE * TILE + row0 * TILE;
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int lo = (tc ^ r) << 2;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int off = r * TILE + ((((wc << 1) | h) ^ tr) << 5 | lo);
          float4 v = make_float4(acc[r][2 * h].x, acc[r][2 * h].y, acc[r][2 * h + 1].x,
                                 acc[r][2 * h + 1].y);
          *reinterpret_cast<float4*>(D + off) = v;
        }
      }
      bar_arrive(2 + buf, WS_THREADS);  // FULL[buf]
      if (In != I) {
        xb ^= 1;
        xfresh = true;
      }
      I = In;
      J = Jn;
    }
    // balance the epilogue's two outstanding EMPTY arrivals
    bar_sync(4, WS_THREADS);
    bar_sync(5, WS_THREADS);
  } else {
    // =========================== epilogue warps ==========================
    const int e_id = tid - WS_COMPUTE_THREADS;  // 0..255
    const bool is_row = e_id < TILE;             // warps 8-11: rows, 12-15: columns
    const int t = is_row ? e_id : e_id - TILE;   // owned row (or column) of the tile
    unsigned long long run1 = NONE_KEY, run2 = NONE_KEY;  // row t running top-2 over J
    bar_arrive(4, WS_THREADS);  // both distance buffers start empty
    bar_arrive(5, WS_THREADS);
    // raw-value threshold equivalent to a key d-part: values (as signed ints, DOT
    // values may be slightly negative) above it cannot produce a key <= d-part
    auto vthr = [&](uint32_t dpart, float B) -> int {
      const uint32_t tb = dpart | 63u;
      if (!DOT) return (int)min(tb, 0x7FFFFFFFu);
      if (tb >= INF_BITS) return 0x7FFFFFFF;
      return __float_as_int(__fmaf_ru(__uint_as_float(tb), p.dot_onepA, B));
    };
    for (int64_t w = w0; w < w1; ++w) {
      const int buf = (int)((w - w0) & 1);
      int In, Jn;
      next_item(p, w, I, J, In, Jn);
      const bool diag = (I == J);
      int* cr = sCR + buf * TILE;
      int* cc = sCC + buf * TILE;
      int* sr = sSR + buf * TILE;
      int* sc = sSC + buf * TILE;
      float* nb = sNB + buf * TILE;
      // my own label / size, and publish it for the other role
      const int mytile = is_row ? I : J;
      const int myC = __ldg(p.comp + (int64_t)mytile * TILE + t);
      int myS = 0;
      (is_row ? cr : cc)[t] = myC;
      if (SIZES) {
        myS = __ldg(p.psize + (int64_t)mytile * TILE + t);
        (is_row ? sr : sc)[t] = myS;
      }
      float myB = 0.f, myNBK = 0.f;
      if (DOT && is_row) {
        myB = __ldg(p.dot_B + (int64_t)I * TILE + t);
        myNBK = __ldg(p.dot_nbk + (int64_t)I * TILE + t);
        nb[t] = myNBK;
      }
      // global second-best (best for top-1) d-parts: stale values are larger,
      // hence still safe filter thresholds
      uint32_t growG = 0x7FFFFFFFu, gcolG = 0x7FFFFFFFu;
      {
        const unsigned long long* G = TOP2 ? p.B2 : p.B1;
        const int g = (is_row ? I : J) * TILE + t;
        if (g < p.n) {
          const uint32_t v = (uint32_t)(*((volatile const unsigned long long*)(G + g)) >> 32);
          if (is_row) growG = v;
          else gcolG = v;
        }
      }
      const float colB = (DOT && !is_row) ? __ldg(p.dot_Bmax + I) : 0.f;
      bar_sync(6, WS_EPI_THREADS);
      bar_sync(2 + buf, WS_THREADS);  // FULL[buf]
      const float* D = sD + buf * TILE * TILE;
      unsigned long long k1 = NONE_KEY, k2 = NONE_KEY;
      // Filter: a value that cannot produce a key below a key already known to
      // survive (running / global second-best; best for top-1) cannot enter the
      // final top-2, so whole 4-value chunks are skipped with one warp vote.
      if (is_row) {
        const int tt = t & 31;
        const float* Drow = D + t * TILE;
        uint32_t gthr = (uint32_t)((TOP2 ? run2 : run1) >> 32);
        gthr = min(gthr, growG);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t m1 = 0xFFFFFFFFu, m2 = 0xFFFFFFFFu;
          int thr = vthr(gthr, myB);
#pragma unroll 4
          for (int qq = 0; qq < 16; ++qq) {
            // logical chunk q sits at position q ^ tt: distinct positions across
            // the warp keep the LDS.128 bank-conflict free
            const int q = h * 16 + qq;
            const float4 v4 = *reinterpret_cast<const float4*>(Drow + ((q ^ tt) << 2));
            const int mn = min(min(__float_as_int(v4.x), __float_as_int(v4.y)),
                               min(__float_as_int(v4.z), __float_as_int(v4.w)));
            if (__any_sync(0xFFFFFFFFu, mn <= thr)) {
              const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
              int4 s4 = make_int4(0, 0, 0, 0);
              const int4 c4 = *reinterpret_cast<const int4*>(cc + q * 4);
              if (SIZES) s4 = *reinterpret_cast<const int4*>(sc + q * 4);
              const int ca[4] = {c4.x, c4.y, c4.z, c4.w};
              const int sa[4] = {s4.x, s4.y, s4.z, s4.w};
              const uint32_t cb = (uint32_t)((q & 15) * 4);
              uint32_t kk[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float L = DOT ? fmaxf(__fmaf_rd(vv[e], p.dot_k, myNBK), 0.f) : vv[e];
                // pads (label -1, +inf coordinates) never pair: in the dot form their
                // values are inf / NaN, which fmaxf would turn into 0
                bool ok = ca[e] != myC && ca[e] >= 0 && myC >= 0 && fabsf(vv[e]) < INFINITY;
                if (SIZES) ok = ok && (myS + sa[e] <= p.ksum);
                if (THR) ok = ok && (L <= p.thr_hi);
                const uint32_t bits = ok ? __float_as_uint(L) : INF_BITS;
                kk[e] = (bits & ~63u) | (cb + e);
              }
              if (TOP2) {
                top2_pair(m1, m2, kk[0], kk[1]);
                top2_pair(m1, m2, kk[2], kk[3]);
                thr = vthr(min(gthr, m2 & ~63u), myB);
              } else {
                m1 = min(min(m1, kk[0]), min(min(kk[1], kk[2]), kk[3]));
                thr = vthr(min(gthr, m1 & ~63u), myB);
              }
            }
          }
          const unsigned long long base = (unsigned long long)J * TILE + h * 64;
          merge2(run1, run2, widen(m1, base), TOP2 ? widen(m2, base) : NONE_KEY);
          gthr = min(gthr, (uint32_t)((TOP2 ? run2 : run1) >> 32));
        }
      } else if (!diag) {
        // ---- column t: element (r, t) sits at r*128 + (t ^ ((r & 31) << 2))
        int off[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) off[u] = t ^ (u << 2);
        uint32_t gthr = gcolG;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t m1 = 0xFFFFFFFFu, m2 = 0xFFFFFFFFu;
          int thr = vthr(gthr, colB);
#pragma unroll
          for (int r4 = h * 16; r4 < h * 16 + 16; ++r4) {
            float vv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int r = r4 * 4 + u;
              vv[u] = D[r * TILE + off[r & 31]];
            }
            const int mn = min(min(__float_as_int(vv[0]), __float_as_int(vv[1])),
                               min(__float_as_int(vv[2]), __float_as_int(vv[3])));
            if (__any_sync(0xFFFFFFFFu, mn <= thr)) {
              int4 s4 = make_int4(0, 0, 0, 0);
              const int4 c4 = *reinterpret_cast<const int4*>(cr + r4 * 4);
              if (SIZES) s4 = *reinterpret_cast<const int4*>(sr + r4 * 4);
              float4 n4 = make_float4(0.f, 0.f, 0.f, 0.f);
              if (DOT) n4 = *reinterpret_cast<const float4*>(nb + r4 * 4);
              const int ca[4] = {c4.x, c4.y, c4.z, c4.w};
              const int sa[4] = {s4.x, s4.y, s4.z, s4.w};
              const float na[4] = {n4.x, n4.y, n4.z, n4.w};
              uint32_t kk[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int r = r4 * 4 + u;
                const float L = DOT ? fmaxf(__fmaf_rd(vv[u], p.dot_k, na[u]), 0.f) : vv[u];
                bool ok = ca[u] != myC && ca[u] >= 0 && myC >= 0 && fabsf(vv[u]) < INFINITY;
                if (SIZES) ok = ok && (myS + sa[u] <= p.ksum);
                if (THR) ok = ok && (L <= p.thr_hi);
                const uint32_t bits = ok ? __float_as_uint(L) : INF_BITS;
                kk[u] = (bits & ~63u) | (uint32_t)(r & 63);
              }
              if (TOP2) {
                top2_pair(m1, m2, kk[0], kk[1]);
                top2_pair(m1, m2, kk[2], kk[3]);
                thr = vthr(min(gthr, m2 & ~63u), colB);
              } else {
                m1 = min(min(m1, kk[0]), min(min(kk[1], kk[2]), kk[3]));
                thr = vthr(min(gthr, m1 & ~63u), colB);
              }
            }
          }
          const unsigned long long base = (unsigned long long)I * TILE + h * 64;
          merge2(k1, k2, widen(m1, base), TOP2 ? widen(m2, base) : NONE_KEY);
          gthr = min(gthr, (uint32_t)((TOP2 ? k2 : k1) >> 32));
        }
      }
      bar_arrive(4 + buf, WS_THREADS);  // EMPTY[buf]: distances consumed
      if (is_row) {
        if (w + 1 >= w1 || In != I) {
          const int g = I * TILE + t;
          if (g < p.n) gflush.start(p.B1 + g, TOP2 ? p.B2 + g : nullptr, run1, run2);
          run1 = NONE_KEY;
          run2 = NONE_KEY;
        }
      } else if (!diag) {
        const int g = J * TILE + t;
        if (g < p.n) gflush.start(p.B1 + g, TOP2 ? p.B2 + g : nullptr, k1, k2);
      }
      I = In;
      J = Jn;
    }
  }
  gflush.finish();
}

size_t scan_ws_smem_bytes(int d) {
  return (size_t)2 * TILE * TILE * sizeof(float) + (size_t)4 * d * TILE * sizeof(float) +
         8 * TILE * sizeof(int) + (2 + 4 + 4) * TILE * sizeof(float);
}


// ----------------------------------------------------------------------------
// K1-REG: register-epilogue scan (default for the dot form).
//
// 2 CTAs / SM x 8 warps; a thread holds an 8x8 block of distances in registers.
// Selection is a threshold filter: per row / column the kernel knows a key
// already guaranteed to survive (running or global second-best); a value that
// cannot beat it cannot enter the final top-2.  Thresholds are checked with a
// few FMNMX per pair and one warp vote; the rare survivors are inserted exactly
// (full 64-bit keys, no index truncation) into shared-memory top-2 slots with
// atomics, flushed to global once per column tile / row tile.  No distance
// tile ever touches shared memory.
// ----------------------------------------------------------------------------
template <int M, bool TOP2, bool SIZES, bool THR, bool DOT>
__global__ void __launch_bounds__(SCAN_THREADS, 2) scan_reg_kernel(ScanArgs p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int dT = p.d * TILE;
  unsigned long long* rowTop = reinterpret_cast<unsigned long long*>(smem_raw);  // [2 xb][2][128]
  unsigned long long* colTop = rowTop + 4 * TILE;                               // [2 buf][2][128]
  float* sX0 = reinterpret_cast<float*>(colTop + 4 * TILE);                    // [2][d*128]
  float* sY0 = sX0 + 2 * dT;                                                    // [2][d*128]
  float* sNX = sY0 + 2 * dT;   // [2 xb][2 halves][128]
  float* sNY = sNX + 4 * TILE; // [2 buf][2 halves][128]
  float* sBr = sNY + 4 * TILE; // [2 xb][128] row B (dot)
  float* sNBr = sBr + 2 * TILE;  // [2 xb][128] row -B/(1+A) (dot)
  int* sCR = reinterpret_cast<int*>(sNBr + 2 * TILE);  // [2 xb][128]
  int* sCC = sCR + 2 * TILE;                            // [2 buf][128]
  int* sSR = sCC + 2 * TILE;                            // [2 xb][128]
  int* sSC = sSR + 2 * TILE;                            // [2 buf][128]
  uint32_t* sGR = reinterpret_cast<uint32_t*>(sSC + 2 * TILE);  // [2 xb][128] global row d-parts
  uint32_t* sGC = sGR + 2 * TILE;                               // [2 buf][128] global col d-parts
  __shared__ unsigned sTmin[2];  // per buffer: min screened value of the item (bits)

  const int64_t total = p.w_end - p.w_begin;
  const int64_t per = (total + gridDim.x - 1) / gridDim.x;
  const int64_t w0 = p.w_begin + (int64_t)blockIdx.x * per;
  const int64_t w1 = min(w0 + per, p.w_end);
  if (w0 >= w1) return;
  Top2Flush gflush;  // this thread's pending global top-2 insert

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wr = warp >> 1, wc = warp & 1;
  const int tr = lane >> 3, tc = lane & 7;
  const int row0 = wr * 32 + tr * 8;
  const int colw = wc * 64;
  const unsigned long long* Gsrc = TOP2 ? p.B2 : p.B1;

  int I, J;
  first_item(p, w0, I, J);
  // prologue: row tile + labels, first column tile + labels
  async_tile(sX0, sCR, sSR, p.X32, p.ld, I, p.d, p.comp, p.psize, SIZES);
  async_tile(sY0, sCC, sSC, p.X32, p.ld, J, p.d, p.comp, p.psize, SIZES);
  cp_async_commit();
  for (int t = tid; t < 8 * TILE; t += SCAN_THREADS) rowTop[t] = NONE_KEY;  // rowTop + colTop
  if (tid < 2) sTmin[tid] = 0xFFFFFFFFu;
  int xb = 0;
  bool xfresh = true;
  int prevI = -1, prevJ = -1, prevBuf = 0, prevXb = 0;
  for (int64_t w = w0; w <= w1; ++w) {
    const int buf = (int)((w - w0) & 1);
    cp_async_wait_all();
    __syncthreads();  // (A) tiles of w resident; inserts of w-1 complete
    // ---- flush the previous item's column slots, and its row slots if I changes
    if (!DOT && p.tpmin && prevJ >= 0 && tid == SCAN_THREADS - 1) {
      // the previous item's tile-pair bound (every warp's minimum has landed: barrier A)
      const unsigned mb = sTmin[prevBuf];
      sTmin[prevBuf] = 0xFFFFFFFFu;
      const float v = __uint_as_float(mb);
      if (mb < 0x7F800000u) {
        const float L = float_down(exact_lower(p.em, (double)v, p.rsum));
        const int lo = min(prevI, prevJ), hi = max(prevI, prevJ);
        const int64_t wi = (int64_t)lo * p.T - (int64_t)lo * (lo - 1) / 2 + (hi - lo);
        if (L > 0.f) atomicMax(p.tpmin + wi, __float_as_uint(L));
      }
    }
    if (prevJ >= 0) {
      if (tid < TILE) {
        if (prevI != prevJ) {
          unsigned long long* ct = colTop + prevBuf * 2 * TILE;
          const int g = prevJ * TILE + tid;
          if (g < p.n) gflush.start(p.B1 + g, TOP2 ? p.B2 + g : nullptr, ct[tid], ct[TILE + tid]);
          ct[tid] = NONE_KEY;
          ct[TILE + tid] = NONE_KEY;
        }
      } else if (w == w1 || I != prevI) {
        const int r = tid - TILE;
        unsigned long long* rt = rowTop + prevXb * 2 * TILE;
        const int g = prevI * TILE + r;
        if (g < p.n) gflush.start(p.B1 + g, TOP2 ? p.B2 + g : nullptr, rt[r], rt[TILE + r]);
        rt[r] = NONE_KEY;
        rt[TILE + r] = NONE_KEY;
      }
    }
    if (w == w1) break;
    int In, Jn;
    next_item(p, w, I, J, In, Jn);
    const bool has_next = (w + 1 < w1);
    if (has_next) {
      async_tile(sY0 + (buf ^ 1) * dT, sCC + (buf ^ 1) * TILE, sSC + (buf ^ 1) * TILE, p.X32, p.ld,
                 Jn, p.d, p.comp, p.psize, SIZES);
      if (In != I)
        async_tile(sX0 + (xb ^ 1) * dT, sCR + (xb ^ 1) * TILE, sSR + (xb ^ 1) * TILE, p.X32, p.ld,
                   In, p.d, p.comp, p.psize, SIZES);
      cp_async_commit();
    }
    float* sX = sX0 + xb * dT;
    float* sY = sY0 + buf * dT;
    // ---- per-tile setup: centring (dot form), global thresholds
    {
      const int col = tid & (TILE - 1), hk = tid >> 7;
      if (DOT) {
        const int dh = (p.d + 1) >> 1, k0 = hk * dh, k1 = min(p.d, k0 + dh);
        const float* cI = p.dot_center + (int64_t)I * p.d;
        float ny = 0.f;
        for (int k = k0; k < k1; ++k) {
          const float v = sY[k * TILE + col] - __ldg(cI + k);
          sY[k * TILE + col] = v;
          ny = fmaf(v, v, ny);
        }
        sNY[(buf * 2 + hk) * TILE + col] = ny;
        if (xfresh) {
          float nx = 0.f;
          for (int k = k0; k < k1; ++k) {
            const float v = sX[k * TILE + col] - __ldg(cI + k);
            sX[k * TILE + col] = v;
            nx = fmaf(v, v, nx);
          }
          sNX[(xb * 2 + hk) * TILE + col] = nx;
        }
      }
      if (hk == 0) {
        const int g = J * TILE + col;
        sGC[buf * TILE + col] = g < p.n ? (uint32_t)(*((volatile const unsigned long long*)(Gsrc + g)) >> 32)
                                        : 0x7FFFFFFFu;
      } else if (xfresh) {
        const int g = I * TILE + col;
        sGR[xb * TILE + col] = g < p.n ? (uint32_t)(*((volatile const unsigned long long*)(Gsrc + g)) >> 32)
                                       : 0x7FFFFFFFu;
        if (DOT) {
          sBr[xb * TILE + col] = __ldg(p.dot_B + (int64_t)I * TILE + col);
          sNBr[xb * TILE + col] = __ldg(p.dot_nbk + (int64_t)I * TILE + col);
        }
      }
    }
    xfresh = false;
    __syncthreads();  // (B) centred tiles, norms, thresholds visible
    float2 acc[8][4];
    float nbr[8];
    if (DOT) {
      // fold the norms into the accumulator start: acc = -(|xh|^2 + |yh|^2)/2 + xh.yh,
      // so v = -2 acc needs no per-pair work after the loop
      const float* nx0 = sNX + (xb * 2) * TILE;
      const float* ny0 = sNY + (buf * 2) * TILE;
      float nxr[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        nxr[r] = nx0[row0 + r] + nx0[TILE + row0 + r];
        nbr[r] = sNBr[xb * TILE + row0 + r];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c0 = colw + wcol(tc, 2 * q);
        const float2 nyc = make_float2(ny0[c0] + ny0[TILE + c0], ny0[c0 + 1] + ny0[TILE + c0 + 1]);
#pragma unroll
        for (int r = 0; r < 8; ++r)
          acc[r][q] = __fmul2_rn(__fadd2_rn(nyc, make_float2(nxr[r], nxr[r])), make_float2(-0.5f, -0.5f));
      }
      tile_dot_8x8(sX, sY, p.d, row0, colw, tc, acc, false);
    } else {
      tile_8x8<M>(sX, sY, p.d, row0, colw, tc, acc);
    }
    // ---- thresholds in value units (pads: -inf, never pass)
    const bool diag = (I == J);
    const unsigned long long* rt = rowTop + xb * 2 * TILE;
    unsigned long long* ct = colTop + buf * 2 * TILE;
    float tR[8], tC[8];
    const float bmax = DOT ? __ldg(p.dot_Bmax + I) : 0.f;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int R = row0 + t, C = colw + wcol(tc, t);
      uint32_t dr = min(sGR[xb * TILE + R], (uint32_t)((TOP2 ? rt[TILE + R] : rt[R]) >> 32));
      uint32_t dc = min(sGC[buf * TILE + C], (uint32_t)((TOP2 ? ct[TILE + C] : ct[C]) >> 32));
      float fr = dr >= INF_BITS ? INFINITY : __uint_as_float(dr | 63u);
      float fc = dc >= INF_BITS ? INFINITY : __uint_as_float(dc | 63u);
      if (DOT) {
        fr = __fmaf_ru(fr, p.dot_onepA, sBr[xb * TILE + R]);
        fc = __fmaf_ru(fc, p.dot_onepA, bmax);
      }
      tR[t] = sCR[xb * TILE + R] >= 0 ? fr : -INFINITY;
      tC[t] = sCC[buf * TILE + C] >= 0 ? fc : -INFINITY;
    }
    // ---- filter: any value at or below its row or column threshold?  (dot form:
    // v = -2 acc, so v <= t  <=>  acc >= -t/2, an exact rescaling)
    bool hit = false;
    float tmin = INFINITY;  // smallest screened value of this thread's pairs (direct form)
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (DOT) {
        const float m = fmaxf(fmaxf(fmaxf(acc[r][0].x, acc[r][0].y), fmaxf(acc[r][1].x, acc[r][1].y)),
                              fmaxf(fmaxf(acc[r][2].x, acc[r][2].y), fmaxf(acc[r][3].x, acc[r][3].y)));
        hit |= m >= -0.5f * tR[r];
      } else {
        const float m = fminf(fminf(fminf(acc[r][0].x, acc[r][0].y), fminf(acc[r][1].x, acc[r][1].y)),
                              fminf(fminf(acc[r][2].x, acc[r][2].y), fminf(acc[r][3].x, acc[r][3].y)));
        hit |= m <= tR[r];
        tmin = fminf(tmin, m);
      }
    }
    if (!DOT && p.tpmin) {
      // pads give +inf (or NaN for pad x pad, dropped by fminf); same-component pairs are
      // included -- a min over a superset, still a lower bound for the cross pairs
      const unsigned tb = tmin >= 0.f ? __float_as_uint(tmin) : 0u;
      const unsigned wmin = __reduce_min_sync(0xFFFFFFFFu, tmin == tmin ? tb : 0xFFFFFFFFu);
      if (lane == 0) atomicMin(&sTmin[buf], wmin);
    }
    if (!diag) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        float m = acc_at(acc, 0, c);
#pragma unroll
        for (int r = 1; r < 8; ++r) m = DOT ? fmaxf(m, acc_at(acc, r, c)) : fminf(m, acc_at(acc, r, c));
        hit |= DOT ? (m >= -0.5f * tC[c]) : (m <= tC[c]);
      }
    }
    if (__any_sync(0xFFFFFFFFu, hit)) {
      // rare exact path: insert every surviving pair into the shared top-2 slots
      // (fully unrolled: dynamic indexing would move acc[] to local memory)
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int R = row0 + r;
        const int cR = sCR[xb * TILE + R];
        const int sRv = SIZES ? sSR[xb * TILE + R] : 0;
        // the row's best two among this thread's 8 columns first: one shared insert per row
        // instead of one per column (rows start with no threshold in a fresh row tile)
        unsigned long long b1 = NONE_KEY, b2 = NONE_KEY;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int C = colw + wcol(tc, c);
          const float v = DOT ? -2.f * acc_at(acc, r, c) : acc_at(acc, r, c);
          const bool prow = v <= tR[r];
          bool pcol = !diag && v <= tC[c];
          if (!(prow || pcol)) continue;
          const int cC = sCC[buf * TILE + C];
          bool ok = cR != cC && cR >= 0 && cC >= 0 && fabsf(v) < INFINITY;
          if (SIZES) ok = ok && (sRv + sSC[buf * TILE + C] <= p.ksum);
          const float L = DOT ? fmaxf(__fmaf_rd(v, p.dot_k, nbr[r]), 0.f) : v;
          if (THR) ok = ok && (L <= p.thr_hi);
          if (!ok) continue;
          const unsigned long long dp = (unsigned long long)__float_as_uint(L) << 32;
          if (prow) {
            const unsigned long long key = dp | (unsigned long long)(J * TILE + C);
            if (key < b1) {
              b2 = b1;
              b1 = key;
            } else if (key < b2) {
              b2 = key;
            }
          }
          if (pcol) {
            const unsigned long long key = dp | (unsigned long long)(I * TILE + R);
            // skip the atomic when the column's current slot already beats the key
            if (key < (TOP2 ? ct[TILE + C] : ct[C]))
              insert_top2(ct + C, TOP2 ? ct + TILE + C : nullptr, key, NONE_KEY);
          }
        }
        if (key_valid(b1))
          insert_top2(const_cast<unsigned long long*>(rt) + R,
                      TOP2 ? const_cast<unsigned long long*>(rt) + TILE + R : nullptr, b1,
                      TOP2 ? b2 : NONE_KEY);
      }
    }
    prevI = I;
    prevJ = J;
    prevBuf = buf;
    prevXb = xb;
    if (In != I) {
      xb ^= 1;
      xfresh = true;
    }
    I = In;
    J = Jn;
  }
  gflush.finish();
}

size_t scan_reg_smem_bytes(int d) {
  return (size_t)8 * TILE * sizeof(unsigned long long) + (size_t)4 * d * TILE * sizeof(float) +
         (4 + 4 + 2 + 2) * TILE * sizeof(float) + 8 * TILE * sizeof(int) + 4 * TILE * sizeof(uint32_t);
}

template <int M, bool TOP2, bool SIZES, bool THR>
static cudaError_t launch_scan_t(const ScanArgs& a, int grid, cudaStream_t st) {
  if (scan_use_reg(a)) {
    size_t sm = scan_reg_smem_bytes(a.d);
    auto k = (M == EUCLIDEAN && a.dot_center) ? scan_reg_kernel<M, TOP2, SIZES, THR, true>
                                              : scan_reg_kernel<M, TOP2, SIZES, THR, false>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    k<<<grid, SCAN_THREADS, sm, st>>>(a);
    return cudaGetLastError();
  }
  if (scan_use_ws(a.d)) {
    size_t sm = scan_ws_smem_bytes(a.d);
    auto k = (M == EUCLIDEAN && a.dot_center) ? scan_ws_kernel<M, TOP2, SIZES, THR, true>
                                              : scan_ws_kernel<M, TOP2, SIZES, THR, false>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    k<<<grid, WS_THREADS, sm, st>>>(a);
    return cudaGetLastError();
  }
  size_t sm = scan_smem_bytes(a.d);
  auto k = scan_rows_kernel<M, TOP2, SIZES, THR>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  k<<<grid, SCAN_THREADS, sm, st>>>(a);
  return cudaGetLastError();
}

template <int M>
static cudaError_t launch_scan_m(const ScanArgs& a, bool top2, int grid, cudaStream_t st) {
  const bool sizes = a.ksum != INT_UNSET;
  const bool thr = a.thr_hi < INFINITY;
  if (top2) {
    if (sizes) return thr ? launch_scan_t<M, true, true, true>(a, grid, st)
                          : launch_scan_t<M, true, true, false>(a, grid, st);
    return thr ? launch_scan_t<M, true, false, true>(a, grid, st)
               : launch_scan_t<M, true, false, false>(a, grid, st);
  }
  if (sizes) return thr ? launch_scan_t<M, false, true, true>(a, grid, st)
                        : launch_scan_t<M, false, true, false>(a, grid, st);
  return thr ? launch_scan_t<M, false, false, true>(a, grid, st)
             : launch_scan_t<M, false, false, false>(a, grid, st);
}

cudaError_t launch_scan(int metric, const ScanArgs& a, bool top2, int grid, cudaStream_t st) {
  switch (metric) {
    case EUCLIDEAN:
    case SQEUCLIDEAN:
      return launch_scan_m<EUCLIDEAN>(a, top2, grid, st);
    case MANHATTAN:
      return launch_scan_m<MANHATTAN>(a, top2, grid, st);
    case CHEBYSHEV:
      return launch_scan_m<CHEBYSHEV>(a, top2, grid, st);
    default:
      return cudaErrorInvalidValue;
  }
}

// ----------------------------------------------------------------------------
// K2: collect every eligible pair whose screened value is <= the row's bound.
// Rows come from a gathered SoA block (XR, rid); columns from XC (cid or identity).
// ----------------------------------------------------------------------------
template <int M, bool SIZES>
__global__ void __launch_bounds__(SCAN_THREADS, 2) collect_kernel(CollectArgs p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* sX = reinterpret_cast<float*>(smem_raw);
  float* sY = sX + p.d * TILE;
  int* sGR = reinterpret_cast<int*>(sY + p.d * TILE);
  int* sGC = sGR + TILE;
  int* sCompR = sGC + TILE;
  int* sCompC = sCompR + TILE;
  int* sSizeR = sCompC + TILE;
  int* sSizeC = sSizeR + TILE;
  float* sBound = reinterpret_cast<float*>(sSizeC + TILE);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wr = warp >> 1, wc = warp & 1;
  const int tr = lane >> 3, tc = lane & 7;
  const int row0 = wr * 32 + tr * 8;
  const int colw = wc * 64;

  const int rtiles = (p.nr + TILE - 1) / TILE;
  const int ctiles = (p.nc + TILE - 1) / TILE;
  const int64_t items = (int64_t)rtiles * ctiles;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int RT = (int)(it / ctiles), CT = (int)(it % ctiles);
    __syncthreads();
    load_tile(sX, p.XR, p.ldr, RT, p.d);
    load_tile(sY, p.XC, p.ldc, CT, p.d);
    if (tid < TILE) {
      int r = RT * TILE + tid;
      int gr = (r < p.nr) ? p.rid[r] : -1;
      sGR[tid] = gr;
      sCompR[tid] = gr >= 0 ? p.comp[gr] : -2;
      if (SIZES) sSizeR[tid] = gr >= 0 ? p.psize[gr] : 0;
      sBound[tid] = (r < p.nr) ? p.rbound[r] : -1.f;
      int c = CT * TILE + tid;
      int gc = (c < p.nc) ? (p.cid ? p.cid[c] : c) : -1;
      sGC[tid] = gc;
      sCompC[tid] = gc >= 0 ? p.comp[gc] : -3;
      if (SIZES) sSizeC[tid] = gc >= 0 ? p.psize[gc] : 0;
    }
    __syncthreads();
    float2 acc[8][4];
    tile_8x8<M>(sX, sY, p.d, row0, colw, tc, acc);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int gr = sGR[row0 + r];
      const float bnd = sBound[row0 + r];
      const int cr = sCompR[row0 + r];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        float v = acc_at(acc, r, c);
        const int gc = sGC[colw + wcol(tc, c)];
        bool ok = (v <= bnd) && gr >= 0 && gc >= 0 && cr != sCompC[colw + wcol(tc, c)];
        if (SIZES) {
          int a = sSizeR[row0 + r], b = sSizeC[colw + wcol(tc, c)];
          ok = ok && a + b <= p.ksum;
        }
        if (p.triangle) ok = ok && gr < gc;
        if (ok) {
          unsigned long long pos = atomicAdd(p.count, 1ull);
          if (pos < p.cap) p.out[pos] = make_int2(gr, gc);
        }
      }
    }
  }
}

size_t collect_smem_bytes(int d) {
  return (size_t)2 * d * TILE * sizeof(float) + 7 * TILE * sizeof(int);
}

template <int M>
static cudaError_t launch_collect_m(const CollectArgs& a, int grid, cudaStream_t st) {
  size_t sm = collect_smem_bytes(a.d);
  const bool sizes = a.ksum != INT_UNSET;
  auto k = sizes ? collect_kernel<M, true> : collect_kernel<M, false>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  k<<<grid, SCAN_THREADS, sm, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_collect(int metric, const CollectArgs& a, int grid, cudaStream_t st) {
  switch (metric) {
    case EUCLIDEAN:
    case SQEUCLIDEAN:
      return launch_collect_m<EUCLIDEAN>(a, grid, st);
    case MANHATTAN:
      return launch_collect_m<MANHATTAN>(a, grid, st);
    case CHEBYSHEV:
      return launch_collect_m<CHEBYSHEV>(a, grid, st);
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace nnm
