// nnm_common.cuh -- shared definitions for the B200 NNM hot path (sm_100a).
//
// Data layout in HBM:
//   X64   n x d float64, row-major, the caller's exact values (used for every
//         order-deciding key: scipy-order FP64).
//   X32   d x n_pad float32, SoA (coordinate-major), padded to a multiple of
//         TILE with +inf so padded pairs are never eligible.  Screening only.
//   comp  n_pad int32 component label per point (pads: -1).
//   psize n_pad int32 cluster size per point (round path: kl2/kl3).
//   norm  n float64 per-point norm used by the FP32 error bound (L2/L1/Linf).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <string.h>

namespace nnm {

enum Metric : int { EUCLIDEAN = 0, SQEUCLIDEAN = 1, MANHATTAN = 2, CHEBYSHEV = 3 };

constexpr int TILE = 128;         // points per tile (rows and columns)
constexpr int SCAN_THREADS = 256; // 8 warps, 8x8 pairs per thread
constexpr uint32_t INF_BITS = 0x7F800000u;
constexpr unsigned long long NONE_KEY = 0x7FFFFFFFFFFFFFFFull;  // > every valid key, signed or not
constexpr int INT_UNSET = 0x7FFFFFFF;

// Screened key: (fp32 bits of the screened distance, low bits truncated) << 32 | index.
// Keys of distinct partners never compare equal; ineligible pairs carry d-part >= INF_BITS.
__host__ __device__ __forceinline__ bool key_valid(unsigned long long k) {
  return (uint32_t)(k >> 32) < INF_BITS;
}
__host__ __device__ __forceinline__ uint32_t key_index(unsigned long long k) {
  return (uint32_t)(k & 0xFFFFFFFFull);
}
__host__ __device__ __forceinline__ float key_value(unsigned long long k) {
  uint32_t b = (uint32_t)(k >> 32);
  float f;
  memcpy(&f, &b, 4);
  return f;
}

// ---------------------------------------------------------------------------
// FP64 exact distance, bit-identical to scipy 1.18.1 cdist (metrics.py:59-73):
// strict left-to-right accumulation, no FMA contraction (explicit _rn intrinsics).
// ---------------------------------------------------------------------------
template <int M>
__device__ __forceinline__ double exact_dist(const double* __restrict__ x,
                                             const double* __restrict__ y, int d) {
  double acc = 0.0;
  for (int k = 0; k < d; ++k) {
    double t = __dsub_rn(x[k], y[k]);
    if (M == EUCLIDEAN || M == SQEUCLIDEAN) {
      acc = __dadd_rn(acc, __dmul_rn(t, t));
    } else if (M == MANHATTAN) {
      acc = __dadd_rn(acc, fabs(t));
    } else {
      double a = fabs(t);
      acc = (a > acc) ? a : acc;
    }
  }
  return acc;
}

// ---------------------------------------------------------------------------
// Rigorous FP32-screen error model.
//
// For a pair with exact scipy value S (FP64) and screened FP32 value v computed
// from x32 = fl32(x64) by direct differences:
//     |v - S| <= a * S + b * g(S),   g(S) = sqrt(S) (euclidean) or 1 (L1, Linf)
// with a = 1.25*((d+4) u + d 2^-53) [+ masking slack handled by callers],
//      b = 1.25 * u * c_m * R,  R = norm(x) + norm(y) in the metric's norm,
//      u = 2^-24, c_m = 2 for euclidean, 1 for L1/Linf;  plus absolute slack c0.
// ---------------------------------------------------------------------------
struct ErrModel {
  double a;       // relative coefficient
  double bcoef;   // b = bcoef * R
  double c0;      // absolute slack (underflow / subnormal)
  int sqrt_form;  // 1: euclidean (g = sqrt), 0: L1/Linf (g = 1)
};

__host__ __device__ inline ErrModel make_err_model(int metric, int d) {
  const double u = 5.9604644775390625e-08;  // 2^-24
  ErrModel e;
  e.c0 = (double)(d + 2) * 1.1754943508222875e-38 * 4.0;
  if (metric == EUCLIDEAN || metric == SQEUCLIDEAN) {
    e.a = 1.25 * ((d + 4) * u + d * 1.1102230246251565e-16);
    e.bcoef = 1.25 * 2.0 * u;
    e.sqrt_form = 1;
  } else if (metric == MANHATTAN) {
    e.a = 1.25 * ((d + 3) * u + d * 1.1102230246251565e-16);
    e.bcoef = 1.25 * u;
    e.sqrt_form = 0;
  } else {
    e.a = 1.25 * (2.0 * u);
    e.bcoef = 1.25 * u;
    e.sqrt_form = 0;
  }
  return e;
}

// Upper bound on the screened value of any pair whose exact value is <= S.
__host__ __device__ inline double screen_upper(const ErrModel& e, double S, double R) {
  if (!(S < INFINITY)) return INFINITY;
  double g = e.sqrt_form ? sqrt(S) : 1.0;
  return S + e.a * S + e.bcoef * R * g + e.c0;
}

// Lower bound on the exact value S of a pair whose screened value is >= v.
__host__ __device__ inline double exact_lower(const ErrModel& e, double v, double R) {
  if (!(v < INFINITY)) return INFINITY;
  double b = e.bcoef * R;
  double shi2;  // upper bound on S given v (solve S(1-a) - b g(S) - v - c0 <= 0)
  if (e.sqrt_form) {
    double disc = b * b + 4.0 * (1.0 - e.a) * (v + e.c0);
    double s = (b + sqrt(disc)) / (2.0 * (1.0 - e.a));
    s *= (1.0 + 1e-12);
    shi2 = s * s;
    double lo = v - e.a * shi2 - b * s - e.c0;
    return lo > 0.0 ? lo * (1.0 - 1e-12) : 0.0;
  }
  shi2 = (v + b + e.c0) / (1.0 - e.a) * (1.0 + 1e-12);
  double lo = v - e.a * shi2 - b - e.c0;
  return lo > 0.0 ? lo * (1.0 - 1e-12) : 0.0;
}

// ---------------------------------------------------------------------------
// Dot-form screen (Euclidean Boruvka scans).
// For a tile pair (I, J) the kernel centres both tiles on c = fl32(centre of I):
//   xh = fl(x32 - c), yh = fl(y32 - c),  v = fl(fl(|xh|^2 + |yh|^2) - 2 fl(xh.yh))
// with FFMA accumulation.  With r = |xh| of the tile-I point and
// eta0 = u(|x| + |y|max) + 2u(1+u) r  (input rounding + centring rounding):
//   |v - S| <= A*S + B(r),  A = 2*alpha*(1+u)^2 + eps + 2u + 2u^2,
//   B(r)    = 2*alpha*(2r + eta0)^2 + eta0^2 (1/eps + 2),  alpha = 1.1 (d+3) u
// (triangle inequality on |xh - yh| vs sqrt(S), then (a+b)^2 <= 2a^2 + 2b^2 and
// 2 sqrt(S) eta <= eps S + eta^2 / eps).  Keys store L = (v - B) / (1 + A)
// rounded down, a rigorous LOWER bound of S.
// ---------------------------------------------------------------------------
struct DotModel {
  double A;
  double eps;
  double alpha;
  double u;
};

__host__ __device__ inline DotModel make_dot_model(int d) {
  DotModel m;
  m.u = 5.9604644775390625e-08;
  m.alpha = 1.1 * (d + 3) * m.u;
  m.eps = 1e-5;
  m.A = 2.0 * m.alpha * (1 + m.u) * (1 + m.u) + m.eps + 2 * m.u + 2 * m.u * m.u;
  m.A *= 1.01;
  return m;
}

// per-point constant B (returned already multiplied by -1/(1+A), for one FFMA)
__host__ __device__ inline double dot_negB(const DotModel& m, double r, double xnorm,
                                           double maxnorm) {
  double eta0 = m.u * (xnorm + maxnorm) * 1.01 + 2.0 * m.u * (1 + m.u) * r * 1.01;
  double t = 2 * r + eta0;
  double B = (2 * m.alpha * t * t + eta0 * eta0 * (1.0 / m.eps + 2.0)) * 1.01 + 1e-30;
  return -B / (1.0 + m.A);
}

// float rounded toward +inf from a double (so float(v) >= v)
__host__ __device__ inline float float_up(double v) {
  if (!(v < 3.0e38)) return INFINITY;
  float f = (float)v;
  if ((double)f < v) f = nextafterf(f, INFINITY);
  return f;
}

// float rounded toward -inf from a double (so float(v) <= v)
__host__ __device__ inline float float_down(double v) {
  if (!(v > -3.0e38)) return -INFINITY;
  if (!(v < 3.0e38)) return 3.0e38f;
  float f = (float)v;
  if ((double)f > v) f = nextafterf(f, -INFINITY);
  return f;
}

}  // namespace nnm
