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

// 8x8 register tile: rows from sX (local rows row0..row0+7), cols from sY.
template <int M>
__device__ __forceinline__ void tile_8x8(const float* __restrict__ sX, const float* __restrict__ sY,
                                         int d, int row0, int col0, float2 (&acc)[8][4]) {
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[r][q] = make_float2(0.f, 0.f);
#pragma unroll 2
  for (int k = 0; k < d; ++k) {
    const float4 xa = *reinterpret_cast<const float4*>(sX + k * TILE + row0);
    const float4 xb = *reinterpret_cast<const float4*>(sX + k * TILE + row0 + 4);
    const float4 ya = *reinterpret_cast<const float4*>(sY + k * TILE + col0);
    const float4 yb = *reinterpret_cast<const float4*>(sY + k * TILE + col0 + 4);
    const float xr[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
    const float2 yc[4] = {make_float2(ya.x, ya.y), make_float2(ya.z, ya.w),
                          make_float2(yb.x, yb.y), make_float2(yb.z, yb.w)};
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int q = 0; q < 4; ++q) accumulate<M>(acc[r][q], yc[q], xr[r]);
  }
}

__device__ __forceinline__ float acc_at(const float2 (&acc)[8][4], int r, int c) {
  return (c & 1) ? acc[r][c >> 1].y : acc[r][c >> 1].x;
}

// load a 128-point SoA tile [d][128] + comp/size of its points
__device__ __forceinline__ void load_tile(float* __restrict__ s, const float* __restrict__ X32,
                                          int64_t ld, int tile, int d) {
  const int nvec = d * (TILE / 4);
  for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
    int k = v / (TILE / 4), q = v % (TILE / 4);
    reinterpret_cast<float4*>(s + k * TILE)[q] =
        __ldg(reinterpret_cast<const float4*>(X32 + (int64_t)k * ld + (int64_t)tile * TILE) + q);
  }
}

// ----------------------------------------------------------------------------
// K1: per-row best-2 (or best-1) eligible partner over a range of tile pairs.
// ----------------------------------------------------------------------------
template <int M, bool TOP2, bool SIZES, bool THR>
__global__ void __launch_bounds__(SCAN_THREADS, 2) scan_rows_kernel(ScanArgs p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* sX = reinterpret_cast<float*>(smem_raw);
  float* sY = sX + p.d * TILE;
  unsigned long long* rowB1 = reinterpret_cast<unsigned long long*>(sY + p.d * TILE);
  unsigned long long* rowB2 = rowB1 + TILE;
  unsigned long long* colB1 = rowB2 + TILE;
  unsigned long long* colB2 = colB1 + TILE;
  int* sCompR = reinterpret_cast<int*>(colB2 + TILE);
  int* sCompC = sCompR + TILE;
  int* sSizeR = sCompC + TILE;
  int* sSizeC = sSizeR + TILE;

  const int64_t total = p.w_end - p.w_begin;
  const int64_t per = (total + gridDim.x - 1) / gridDim.x;
  const int64_t w0 = p.w_begin + (int64_t)blockIdx.x * per;
  const int64_t w1 = min(w0 + per, p.w_end);
  if (w0 >= w1) return;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wr = warp >> 1, wc = warp & 1;
  const int tr = lane >> 3, tc = lane & 7;
  const int row0 = wr * 32 + tr * 8;
  const int col0 = wc * 64 + tc * 8;

  if (tid < TILE) {
    rowB1[tid] = NONE_KEY;
    rowB2[tid] = NONE_KEY;
    colB1[tid] = NONE_KEY;
    colB2[tid] = NONE_KEY;
  }

  int I, J;
  decode_work(w0, p.T, I, J);
  int curI = -1;

  for (int64_t w = w0; w < w1; ++w) {
    if (I != curI) {
      if (curI >= 0) {
        __syncthreads();
        if (tid < TILE) {
          int g = curI * TILE + tid;
          if (g < p.n) insert_top2(p.B1 + g, TOP2 ? p.B2 + g : nullptr, rowB1[tid], rowB2[tid]);
          rowB1[tid] = NONE_KEY;
          rowB2[tid] = NONE_KEY;
        }
      }
      __syncthreads();
      load_tile(sX, p.X32, p.ld, I, p.d);
      if (tid < TILE) {
        sCompR[tid] = p.comp[I * TILE + tid];
        if (SIZES) sSizeR[tid] = p.psize[I * TILE + tid];
      }
      curI = I;
    }
    load_tile(sY, p.X32, p.ld, J, p.d);
    if (tid < TILE) {
      sCompC[tid] = p.comp[J * TILE + tid];
      if (SIZES) sSizeC[tid] = p.psize[J * TILE + tid];
    }
    __syncthreads();

    float2 acc[8][4];
    tile_8x8<M>(sX, sY, p.d, row0, col0, acc);

    // ---- eligibility: comp differ, kl2 / kl3 on snapshot sizes, dmax screen
    int cr[8], cc[8], sr[8], sc[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      cr[t] = sCompR[row0 + t];
      cc[t] = sCompC[col0 + t];
      if (SIZES) {
        sr[t] = sSizeR[row0 + t];
        sc[t] = sSizeC[col0 + t];
      }
    }
    // keys: row side carries the warp-local column (6 bits), col side the
    // warp-local row (5 bits), packed into the low mantissa bits.
    uint32_t rk1[8], rk2[8];
    uint32_t ck1[8], ck2[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      rk1[t] = 0xFFFFFFFFu;
      rk2[t] = 0xFFFFFFFFu;
      ck1[t] = 0xFFFFFFFFu;
      ck2[t] = 0xFFFFFFFFu;
    }
    const bool diag = (I == J);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        float v = acc_at(acc, r, c);
        bool ok = cr[r] != cc[c];
        if (SIZES) ok = ok && sr[r] <= p.kl2 && sc[c] <= p.kl2 && sr[r] + sc[c] <= p.kl3;
        if (THR) ok = ok && (v <= p.thr_hi);
        uint32_t bits = ok ? __float_as_uint(v) : INF_BITS;
        uint32_t kr = (bits & ~63u) | (uint32_t)(tc * 8 + c);
        if (TOP2) {
          rk2[r] = min(rk2[r], max(rk1[r], kr));
        }
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
      const unsigned long long jb = (unsigned long long)J * TILE + wc * 64;
      unsigned long long k1 = ((s1 & ~63u) >= INF_BITS)
                                  ? NONE_KEY
                                  : (((unsigned long long)(s1 & ~63u) << 32) | (jb + (s1 & 63u)));
      unsigned long long k2 = NONE_KEY;
      if (TOP2 && (s2 & ~63u) < INF_BITS)
        k2 = ((unsigned long long)(s2 & ~63u) << 32) | (jb + (s2 & 63u));
      insert_top2(rowB1 + row0 + tc, TOP2 ? rowB2 + row0 + tc : nullptr, k1, k2);
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
        insert_top2(colB1 + col0 + want, TOP2 ? colB2 + col0 + want : nullptr, k1, k2);
      }
    }
    __syncthreads();
    if (!diag && tid < TILE) {
      int g = J * TILE + tid;
      if (g < p.n) insert_top2(p.B1 + g, TOP2 ? p.B2 + g : nullptr, colB1[tid], colB2[tid]);
      colB1[tid] = NONE_KEY;
      colB2[tid] = NONE_KEY;
    }
    // next work item
    if (++J == p.T) {
      ++I;
      J = I;
    }
    __syncthreads();
  }
  // final row flush
  if (tid < TILE) {
    int g = curI * TILE + tid;
    if (g < p.n) insert_top2(p.B1 + g, TOP2 ? p.B2 + g : nullptr, rowB1[tid], rowB2[tid]);
  }
}

size_t scan_smem_bytes(int d) {
  return (size_t)2 * d * TILE * sizeof(float) + 4 * TILE * sizeof(unsigned long long) +
         4 * TILE * sizeof(int);
}

template <int M, bool TOP2, bool SIZES, bool THR>
static cudaError_t launch_scan_t(const ScanArgs& a, int grid, cudaStream_t st) {
  size_t sm = scan_smem_bytes(a.d);
  auto k = scan_rows_kernel<M, TOP2, SIZES, THR>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  k<<<grid, SCAN_THREADS, sm, st>>>(a);
  return cudaGetLastError();
}

template <int M>
static cudaError_t launch_scan_m(const ScanArgs& a, bool top2, int grid, cudaStream_t st) {
  const bool sizes = (a.kl2 != INT_UNSET) || (a.kl3 != INT_UNSET);
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

int scan_occupancy(int metric, int d) {
  int blocks = 0;
  size_t sm = scan_smem_bytes(d);
  cudaFuncSetAttribute(scan_rows_kernel<EUCLIDEAN, true, false, false>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &blocks, scan_rows_kernel<EUCLIDEAN, true, false, false>, SCAN_THREADS, sm);
  return blocks > 0 ? blocks : 1;
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
  const int col0 = wc * 64 + tc * 8;

  const int rtiles = (p.nr + TILE - 1) / TILE;
  const int ctiles = (p.nc + TILE - 1) / TILE;
  const int64_t items = (int64_t)rtiles * ctiles;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int RT = (int)(it / ctiles), CT = (int)(it % ctiles);
    if (p.triangle) {
      // A x A: only tile pairs with RT <= CT carry pairs with gi < gj... not in
      // general (gathered order is arbitrary), so all tiles are scanned.
    }
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
    tile_8x8<M>(sX, sY, p.d, row0, col0, acc);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int gr = sGR[row0 + r];
      const float bnd = sBound[row0 + r];
      const int cr = sCompR[row0 + r];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        float v = acc_at(acc, r, c);
        const int gc = sGC[col0 + c];
        bool ok = (v <= bnd) && gr >= 0 && gc >= 0 && cr != sCompC[col0 + c];
        if (SIZES) {
          int a = sSizeR[row0 + r], b = sSizeC[col0 + c];
          ok = ok && a <= p.kl2 && b <= p.kl2 && a + b <= p.kl3;
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
  const bool sizes = (a.kl2 != INT_UNSET) || (a.kl3 != INT_UNSET);
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
