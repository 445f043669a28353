// nnm_tc.cuh -- tensor-core (tcgen05, kind::tf32) screening scan for Euclidean
// Boruvka rounds (internal interface; see nnm_tc.cu and DESIGN.md "TC scan").
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "nnm_common.cuh"

namespace nnm {

constexpr int TC_K = 32;              // K extent of one operand row (floats): 128 B = one SW128 atom row
constexpr int TC_TILE_FLOATS = TILE * TC_K;  // 4096 floats = 16 KB per tile image
constexpr int TC_MAX_D = TC_K - 3;    // coords + (s_hi, s_lo) + >= 1 component slot
constexpr int TC_META = 48;           // floats per tile record (192 B, bulk-copy aligned)

struct TcArgs {
  const float* img;       // [T][128][32] swizzled operand image: tf32-exact centred coords, 0 elsewhere
  const float* tnorm;     // [np] |x_t| of each position, rounded up (0 for pads)
  const float* eta;       // [np] distance-domain rounding bound of each position, rounded up
  const float* sq;        // [np] |x_t|^2 of each position (fp32 FMA chain)
  const float* meta;      // [T][TC_META] tile records: fp32 centre the image was centred on
                          // (32, zero padded), max tnorm (32), max eta (33)
  const int* comp;        // [np] component label per position (-1: pad)
  const double* X64;      // [np][d] exact coordinates of the view (keys of inserted pairs)
  int np, d, T;
  const int2* items;      // ordered (row tile I, column tile J) pairs, sorted by I
  int64_t w_begin, w_end;
  float thr_hi;           // keys above this are ineligible (L units; +inf: no dmax)
  unsigned long long* B1; // [np] best key per row (float_down(S) << 32 | partner position)
  unsigned long long* B2; // [np] second-best key
  float* dump;            // debug: raw accumulators [items][128][128] (nullptr in production)
  long long* trace;       // NNM_TC_TRACE: [5 roles][256 items][2] clock64 stamps of CTA 0
  unsigned* tpmin;        // [T(T+1)/2] per tile pair: fp32 bits of a lower bound of S over
                          // the pairs not masked same-component (atomicMax; nullptr: off)
  int dbg;                // timing experiments (NNM_TC_DBG): 1 = no epilogue work, 2 = no prep work
  // component caps (DESIGN 3.1): [np] per component label, fp32 bits of a rigorous UPPER
  // bound of the component's minimum cross edge.  bound_only: the scan writes them
  // (atomicMin of each row's best screened upper bound; no exact work, no keys);
  // otherwise every row threshold is capped by its component's value (nullptr: off)
  unsigned* ucap;
  int bound_only;
  const unsigned* capp;   // [np] per position: its component's cap (capped exact passes)
  const int* slots;       // [T][16] per-round slot records (launch_tc_tails)
  const int2* trange;     // [T] min / max component label per tile (nullptr: always check)
  // deferred exact keys (nullptr: evaluate in the epilogue): candidates passing the
  // screen are appended as (row position << 32 | column position) and evaluated by
  // launch_tc_exact after the scan -- the FP64 gathers leave the tensor-core pipeline
  unsigned long long* cand;
  unsigned long long* ccount;
  unsigned long long ccap;
};

size_t tc_smem_bytes();
// exact keys of the deferred candidates into the rows' atomic top-2 (B1, B2)
cudaError_t launch_tc_exact(const unsigned long long* cand, const unsigned long long* count,
                            int64_t cap, const double* X64, int d, float thr_hi,
                            unsigned long long* B1, unsigned long long* B2, cudaStream_t st);
bool tc_supported(int d);
cudaError_t launch_tc_scan(const TcArgs& a, int grid, cudaStream_t st);
// per-round slot records + A-side operand tails for the current component labels
cudaError_t launch_tc_tails(float* img, const int* comp, int T, int d, int* slots, cudaStream_t st);

// Operand image + per-position / per-tile bounds for the kd view (once per dataset).
cudaError_t launch_tc_prepare(const double* X64p, const int* porig, const double* tcenter64,
                              const double* normp, int64_t np, int d, int T, float* img,
                              float* tnorm, float* eta, float* meta, float* sq, cudaStream_t st);

// Error-model probe over dumped accumulators (a.dump filled by launch_tc_scan for `items`).
cudaError_t launch_tc_probe(const TcArgs& a, const double* X64p, const int2* items, int64_t n,
                            unsigned long long* out, cudaStream_t st);



}  // namespace nnm
