// nnm_replay.cu -- the merge replay of the Boruvka path on the GPU.
//
// Reference: the merge loop of engine.run / process_batch (engine.py:90-143) over
// ClusterForest.union (model.py:148-160: the kept root is the smaller index, the new
// size is the sum).  The Boruvka rounds deliver the minimum spanning forest with its
// exact (d, a, b) total order; the reference's merge sequence is the Kruskal replay
// of those edges in that order.  For merge k (edge (a, b)) the
// replay needs the roots and sizes of a's and b's clusters in the forest of merges
// 0 .. k-1.  That is a sequential union-find in rank order -- but only WITHIN a
// connected piece: edges whose clusters never meet are independent.
//
// Chunked component-parallel replay:
//   the sorted edges are cut into rank chunks [lo, lo + C).  For one chunk, given
//   the forest after all earlier chunks (par / sz, roots = minimum index):
//     roots   A = find(a), B = find(b) for every edge of the chunk;
//     link    connected components of the chunk's edges over (A, B) (lock-free
//             union-find with min-root links on a scratch label array);
//     label   component label of every edge;
//     list    per-component edge lists (atomic exchange into a head per label);
//     check   longest component; above lmax the GPU stops here and the host
//             finishes the replay from this chunk on (the forest is untouched);
//     replay  one thread per component sorts its list into rank order and walks it
//             with a private union-find over its own clusters (disjoint from every
//             other component of the chunk, so no races), writing (kept root,
//             dropped root, new size) at the edge's rank.
// The whole chunk sequence has a fixed launch topology for a given edge count, so
// the host captures it once into a CUDA graph (nnm_api.cu) and replays it.
// A blob-structured dendrogram (C4: 4000 blobs) cuts into thousands of short
// components per chunk, so the sequential part per thread is a few dozen steps.
#include "nnm_kernels.cuh"

namespace nnm {

namespace {

// path halving; links only ever point to ancestors (smaller indices), so concurrent
// halving by other threads on the same path is benign
__device__ __forceinline__ int find_halve(int* par, int x) {
  int p = par[x];
  while (p != x) {
    const int g = par[p];
    if (g != p) par[x] = g;
    x = g;
    p = par[x];
  }
  return x;
}

__global__ void replay_init_kernel(int64_t n, int* par, int* sz, int* ctl) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    par[i] = (int)i;
    sz[i] = 1;
  }
  if (i < 4) ctl[i] = (i == 1) ? -1 : 0;
}

__global__ void replay_roots_kernel(const ReplayEdge* __restrict__ e, int64_t lo, int cnt,
                                    int* par, int* lab, int* head, int* ea, int* eb,
                                    const int* __restrict__ ctl) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt || ctl[0]) return;
  const ReplayEdge x = e[lo + t];
  const int A = find_halve(par, x.a), B = find_halve(par, x.b);
  ea[t] = A;
  eb[t] = B;
  lab[A] = A;
  lab[B] = B;
  head[A] = -1;
  head[B] = -1;
}

__global__ void replay_link_kernel(int cnt, int* lab, const int* __restrict__ ea,
                                   const int* __restrict__ eb, const int* __restrict__ ctl) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt || ctl[0]) return;
  int a = ea[t], b = eb[t];
  for (;;) {
    a = find_halve(lab, a);
    b = find_halve(lab, b);
    if (a == b) return;
    if (a > b) {
      const int s = a;
      a = b;
      b = s;
    }
    if (atomicCAS(&lab[b], b, a) == b) return;  // larger root under the smaller
  }
}

// per-component edge lists (arbitrary order; the owner sorts its own list)
__global__ void replay_list_kernel(int cnt, int* lab, const int* __restrict__ ea, int* head,
                                   int* nxt, int* comp, const int* __restrict__ ctl) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt || ctl[0]) return;
  const int L = find_halve(lab, ea[t]);
  comp[t] = L;
  nxt[t] = atomicExch(&head[L], t);
}

// longest component of the chunk; too long -> stop (the host finishes from lo)
__global__ void replay_check_kernel(int64_t lo, int cnt, const int* __restrict__ head,
                                    const int* __restrict__ nxt, const int* __restrict__ comp,
                                    int lmax, int* ctl, int* chunk_max) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt || ctl[0]) return;
  if (head[comp[t]] != t) return;  // the list owner: the edge that was linked last
  int len = 0;
  for (int q = t; q >= 0; q = nxt[q]) ++len;
  atomicMax(&ctl[2], len);
  if (chunk_max) atomicMax(chunk_max, len);
  if (len > lmax && atomicCAS(&ctl[0], 0, 1) == 0) ctl[1] = (int)lo;
}

// one thread per component: its edges in rank order, private union-find
__global__ void replay_segment_kernel(int64_t lo, int cnt, const int* __restrict__ head,
                                      const int* __restrict__ nxt, const int* __restrict__ comp,
                                      const int* __restrict__ ea, const int* __restrict__ eb,
                                      int* par, int* sz, int* rk, int* rd, int* rs, int* ctl) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt || ctl[0]) return;
  if (head[comp[t]] != t) return;
  int ts[REPLAY_LMAX];
  int k = 0;
  for (int q = t; q >= 0 && k < REPLAY_LMAX; q = nxt[q]) ts[k++] = q;
  for (int i = 1; i < k; ++i) {  // insertion sort: rank order (lists are short)
    const int v = ts[i];
    int j = i - 1;
    while (j >= 0 && ts[j] > v) {
      ts[j + 1] = ts[j];
      --j;
    }
    ts[j + 1] = v;
  }
  for (int i = 0; i < k; ++i) {
    const int q = ts[i];
    const int ra = find_halve(par, ea[q]), rb = find_halve(par, eb[q]);
    if (ra == rb) {  // a cycle: the edge list is not a forest (internal error)
      ctl[3] = 1;
      continue;
    }
    const int keep = ra < rb ? ra : rb, drop = ra < rb ? rb : ra;
    const int s = sz[keep] + sz[drop];
    sz[keep] = s;
    par[drop] = keep;
    rk[lo + q] = keep;
    rd[lo + q] = drop;
    rs[lo + q] = s;
  }
}

__global__ void replay_assign_kernel(int64_t n, int* par, int* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = find_halve(par, (int)i);
}

inline int grid_for(int64_t n, int t = 256) {
  return (int)std::max<int64_t>(1, (n + t - 1) / t);
}

}  // namespace

cudaError_t replay_init(int64_t n, const ReplayState& s, cudaStream_t st) {
  replay_init_kernel<<<grid_for(std::max<int64_t>(n, 4)), 256, 0, st>>>(n, s.par, s.sz, s.ctl);
  return cudaGetLastError();
}

cudaError_t replay_chunk(const ReplayEdge* e, int64_t lo, int cnt, int lmax, const ReplayState& s,
                         cudaStream_t st, int* chunk_max) {
  if (cnt <= 0) return cudaSuccess;
  const int g = grid_for(cnt);
  lmax = std::min(lmax, REPLAY_LMAX);
  replay_roots_kernel<<<g, 256, 0, st>>>(e, lo, cnt, s.par, s.lab, s.head, s.ea, s.eb, s.ctl);
  replay_link_kernel<<<g, 256, 0, st>>>(cnt, s.lab, s.ea, s.eb, s.ctl);
  replay_list_kernel<<<g, 256, 0, st>>>(cnt, s.lab, s.ea, s.head, s.nxt, s.comp, s.ctl);
  replay_check_kernel<<<g, 256, 0, st>>>(lo, cnt, s.head, s.nxt, s.comp, lmax, s.ctl, chunk_max);
  replay_segment_kernel<<<g, 256, 0, st>>>(lo, cnt, s.head, s.nxt, s.comp, s.ea, s.eb, s.par,
                                           s.sz, s.rk, s.rd, s.rs, s.ctl);
  return cudaGetLastError();
}

cudaError_t replay_assign(int64_t n, const ReplayState& s, int* out, cudaStream_t st) {
  replay_assign_kernel<<<grid_for(n), 256, 0, st>>>(n, s.par, out);
  return cudaGetLastError();
}

}  // namespace nnm
