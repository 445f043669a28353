// nnm_kernels.cuh -- kernel argument blocks and launch wrappers (internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "nnm_common.cuh"

namespace nnm {

constexpr int SIZE_BIG = 1 << 29;  // effective size of clusters above kl2

struct ScanArgs {
  const float* X32;  // [d][ld] SoA, +inf padded
  int64_t ld;        // n_pad
  int n, d, T;       // points, dims, tiles (n_pad / TILE)
  const int* comp;   // [n_pad]
  const int* psize;  // [n_pad] effective sizes (> kl2 mapped to SIZE_BIG) (SIZES variants)
  int ksum;          // eligible iff psize[a] + psize[b] <= ksum (INT_UNSET: no size rule)
  const int2* tile_range;  // [T] min / max component label of each tile's real points
  float thr_hi;      // screened dmax bound (INFINITY when unset)
  int64_t w_begin, w_end;  // range of work items
  const int2* items;       // nullptr: item w = w-th upper-triangular tile pair; else items[w]
  unsigned long long* B1;  // [n] best screened key per row
  unsigned long long* B2;  // [n] second-best (TOP2 only)
  // dot form (Euclidean Boruvka): keys are rigorous lower bounds L of S
  const float* dot_center;  // [T][d] fl32 tile centres (nullptr: direct form)
  const float* dot_B;       // [n] per-position B, rounded up
  const float* dot_nbk;     // [n] -B/(1+A), rounded down
  const float* dot_Bmax;    // [T] max B over the tile, rounded up
  float dot_k;              // 1/(1+A) rounded down
  float dot_onepA;          // 1+A rounded up
  // tile-pair cache (direct form, scan_reg_kernel; nullptr: off): every item publishes
  // exact_lower(min of its screened values) with atomicMax -- a rigorous lower bound of
  // every pair of the tile pair, valid in every later round (DESIGN 3.1)
  unsigned* tpmin;
  ErrModel em;    // the screen's error model
  double rsum;    // bound on norm(x) + norm(y) over all pairs (2 x max norm)
};

struct CollectArgs {
  const float* XR;  // gathered rows, SoA [d][ldr]
  int64_t ldr;
  int nr;
  const int* rid;   // global index of each gathered row
  const float* XC;  // columns, SoA [d][ldc]
  int64_t ldc;
  int nc;
  const int* cid;   // global index of each column (nullptr: identity)
  int d;
  const int* comp;  // global-indexed
  const int* psize;  // effective sizes, see ScanArgs
  int ksum;
  const float* rbound;  // per gathered row: collect pairs with screened value <= bound
  int triangle;         // keep only gi < gj
  int2* out;
  unsigned long long* count;
  unsigned long long cap;
};

struct ReplayEdge {  // sorted MST edge for the merge replay
  double dist;        // reported distance (sqrt for euclidean)
  int a, b, round, pad;
};

// GPU merge replay (nnm_replay.cu): forest state + one chunk's scratch
constexpr int REPLAY_LMAX = 128;  // longest component replayed on the GPU
constexpr int REPLAY_SHORT = 4;   // longer components are replayed by a warp
struct ReplayState {
  int* par;   // [n] union-find over points (roots = minimum index, model.py:148-160)
  int* sz;    // [n] cluster size at each root
  int* lab;   // [n] scratch labels for the per-chunk components
  int* head;  // [n] per-component edge count of the chunk
  int *ea, *eb;       // [chunk] roots of the edge ends at chunk start
  int *nxt, *comp;    // [chunk] position of the edge in its component, component label
  int* ctl;  // [0] stop flag, [1] first edge the host must replay (-1: none), [2] max
             // component length seen, [3] cycle detected (internal error), [4] slot
             // allocator, [5] long components listed
  int *rk, *rd, *rs;  // [m] kept root, dropped root, new size per merge
  int* base;  // [n] first slot of each component's edge block
  int* slot;  // [chunk] edge blocks: each component's chunk offsets, contiguous
  int* rid;   // [n] local id of each chunk-start root within its component
  int* rcnt;  // [n] distinct chunk-start roots per component
  int* llist; // [chunk] owners of the components replayed by a warp (long ones)
};
cudaError_t replay_init(int64_t n, const ReplayState& s, cudaStream_t st);
cudaError_t replay_chunk(const ReplayEdge* e, int64_t lo, int cnt, int lmax, const ReplayState& s,
                         cudaStream_t st, int* chunk_max = nullptr);
cudaError_t replay_assign(int64_t n, const ReplayState& s, int* out, cudaStream_t st);

size_t scan_smem_bytes(int d);
size_t collect_smem_bytes(int d);
int scan_occupancy(int metric, int d);
bool scan_use_ws(int d);
bool scan_use_reg(const ScanArgs& a);
size_t scan_reg_smem_bytes(int d);
size_t scan_ws_smem_bytes(int d);
void scan_set_mode(int mode);  // -1 auto, 0 classic kernel, 1 warp-specialised
cudaError_t launch_scan(int metric, const ScanArgs& a, bool top2, int grid, cudaStream_t st);
cudaError_t launch_collect(int metric, const CollectArgs& a, int grid, cudaStream_t st);

}  // namespace nnm
