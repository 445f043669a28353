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
//     count   component label of every edge and its position in the component
//             (atomic count per label);
//     check   one edge per component: its length (above lmax the GPU stops here and
//             the host finishes the replay from this chunk on; the forest is
//             untouched), a contiguous block of slots, and -- when longer than
//             REPLAY_SHORT -- a place in the warp list;
//     place   every edge writes its chunk offset into its component's block; every
//             chunk-start root claims a dense local id within its component;
//     replay  short components: one thread each, in rank order, union-find on the
//             global forest; long ones: one WARP each -- the lanes load the block,
//             the roots and their sizes in parallel into shared memory, then one lane
//             replays the edges in rank order with a union-find over the local ids in
//             shared memory (no global pointer chasing on the sequential path).
//             Components of a chunk touch disjoint clusters, so no races; each
//             writes (kept root, dropped root, new size) at the edge's rank and
//             writes its links and sizes through to the forest for later chunks.
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
  if (i < 8) ctl[i] = (i == 1) ? -1 : 0;
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
  head[A] = 0;
  head[B] = 0;
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

// component label and position of every edge (per-label atomic count); clears the
// local ids of the chunk-start roots
__global__ void replay_list_kernel(int cnt, int* lab, const int* __restrict__ ea,
                                   const int* __restrict__ eb, int* head, int* nxt, int* comp,
                                   int* rid, int* rcnt, int* ctl) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t == 0) {
    ctl[4] = 0;  // slot allocator and long list of this chunk
    ctl[5] = 0;
  }
  if (t >= cnt || ctl[0]) return;
  const int L = find_halve(lab, ea[t]);
  comp[t] = L;
  nxt[t] = atomicAdd(&head[L], 1);
  rid[ea[t]] = -1;
  rid[eb[t]] = -1;
  rcnt[L] = 0;
}

// one edge per component: its length, its block of slots, long ones into the warp list
// (warp-aggregated: one allocator atomic per warp, not per component)
__global__ void replay_check_kernel(int64_t lo, int cnt, const int* __restrict__ head,
                                    const int* __restrict__ nxt, const int* __restrict__ comp,
                                    int lmax, int* ctl, int* chunk_max, int* base, int* llist) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  if (ctl[0]) return;  // uniform: set by an earlier chunk only
  const bool owner = t < cnt && nxt[t] == 0;
  const int L = owner ? comp[t] : 0;
  const int len = owner ? head[L] : 0;
  int x = len, mx = len;  // inclusive scan and max of the lengths over the warp
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= o) x += y;
    mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
  }
  int wbase = 0;
  const int total = __shfl_sync(0xFFFFFFFFu, x, 31);
  if (lane == 31 && total) wbase = atomicAdd(&ctl[4], total);
  wbase = __shfl_sync(0xFFFFFFFFu, wbase, 31);
  if (lane == 0 && mx) {
    atomicMax(&ctl[2], mx);
    if (chunk_max) atomicMax(chunk_max, mx);
  }
  const bool lng = owner && len > REPLAY_SHORT;
  const unsigned lm = __ballot_sync(0xFFFFFFFFu, lng);
  int lb = 0;
  if (lane == 0 && lm) lb = atomicAdd(&ctl[5], __popc(lm));
  lb = __shfl_sync(0xFFFFFFFFu, lb, 0);
  if (!owner) return;
  if (len > lmax && atomicCAS(&ctl[0], 0, 1) == 0) ctl[1] = (int)lo;
  base[L] = wbase + x - len;
  if (lng) llist[lb + __popc(lm & ((1u << lane) - 1u))] = t;
}

__global__ void replay_place_kernel(int cnt, const int* __restrict__ nxt,
                                    const int* __restrict__ comp, const int* __restrict__ base,
                                    const int* __restrict__ ea, const int* __restrict__ eb,
                                    int* __restrict__ slot, int* rid, int* rcnt,
                                    const int* __restrict__ ctl) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt || ctl[0]) return;
  const int L = comp[t];
  slot[base[L] + nxt[t]] = t;
  const int A = ea[t], B = eb[t];
  if (atomicCAS(&rid[A], -1, -2) == -1) rid[A] = atomicAdd(&rcnt[L], 1);
  if (atomicCAS(&rid[B], -1, -2) == -1) rid[B] = atomicAdd(&rcnt[L], 1);
}

// short components: one thread each, rank order, union-find on the global forest
__global__ void replay_segment_kernel(int64_t lo, int cnt, const int* __restrict__ head,
                                      const int* __restrict__ nxt, const int* __restrict__ comp,
                                      const int* __restrict__ ea, const int* __restrict__ eb,
                                      const int* __restrict__ base, const int* __restrict__ slot,
                                      int* par, int* sz, int* rk, int* rd, int* rs, int* ctl) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt || ctl[0]) return;
  if (nxt[t] != 0) return;
  const int L = comp[t];
  const int k = head[L];
  if (k > REPLAY_SHORT) return;  // a warp replays it (replay_long_kernel)
  const int* blk = slot + base[L];
  int ts[REPLAY_SHORT];
  for (int i = 0; i < k; ++i) ts[i] = blk[i];
  for (int i = 1; i < k; ++i) {  // insertion sort: rank order
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

// long components: one warp each (see the file header)
constexpr int REPLAY_WARPS = 4;  // warps per block of replay_long_kernel
__global__ void __launch_bounds__(32 * REPLAY_WARPS) replay_long_kernel(
    int64_t lo, const int* __restrict__ llist, const int* __restrict__ head,
    const int* __restrict__ comp, const int* __restrict__ ea, const int* __restrict__ eb,
    const int* __restrict__ base, const int* __restrict__ slot, const int* __restrict__ rid,
    const int* __restrict__ rcnt, int* par, int* sz, int* rk, int* rd, int* rs, int* ctl) {
  __shared__ int s_ts[REPLAY_WARPS][REPLAY_LMAX];
  __shared__ short s_la[REPLAY_WARPS][REPLAY_LMAX], s_lb[REPLAY_WARPS][REPLAY_LMAX];
  __shared__ int s_root[REPLAY_WARPS][REPLAY_LMAX + 1], s_par[REPLAY_WARPS][REPLAY_LMAX + 1],
      s_sz[REPLAY_WARPS][REPLAY_LMAX + 1];
  if (ctl[0]) return;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nl = ctl[5];
  int* ts = s_ts[w];
  short *la = s_la[w], *lb = s_lb[w];
  int *lroot = s_root[w], *lpar = s_par[w], *lsz = s_sz[w];
  for (int e = blockIdx.x * REPLAY_WARPS + w; e < nl; e += gridDim.x * REPLAY_WARPS) {
    const int L = comp[llist[e]];
    const int k = min(head[L], REPLAY_LMAX);
    const int nr = min(rcnt[L], REPLAY_LMAX + 1);
    const int* blk = slot + base[L];
    for (int i = lane; i < k; i += 32) ts[i] = blk[i];
    __syncwarp();
    if (lane == 0)  // rank order (blocks arrive nearly sorted)
      for (int i = 1; i < k; ++i) {
        const int v = ts[i];
        int j = i - 1;
        while (j >= 0 && ts[j] > v) {
          ts[j + 1] = ts[j];
          --j;
        }
        ts[j + 1] = v;
      }
    __syncwarp();
    for (int i = lane; i < k; i += 32) {
      const int q = ts[i], A = ea[q], B = eb[q];
      const int ia = rid[A], ib = rid[B];
      la[i] = (short)ia;
      lb[i] = (short)ib;
      lroot[ia] = A;  // benign: every writer of a slot writes the same root
      lroot[ib] = B;
    }
    __syncwarp();
    for (int r = lane; r < nr; r += 32) {
      lpar[r] = r;
      lsz[r] = sz[lroot[r]];
    }
    __syncwarp();
    if (lane == 0) {
      for (int i = 0; i < k; ++i) {
        int a = la[i], b = lb[i];
        while (lpar[a] != a) a = lpar[a] = lpar[lpar[a]];
        while (lpar[b] != b) b = lpar[b] = lpar[lpar[b]];
        if (a == b) {
          ctl[3] = 1;
          continue;
        }
        const int ra = lroot[a], rb = lroot[b];
        const bool ka = ra < rb;
        const int keep = ka ? ra : rb, drop = ka ? rb : ra;
        const int kl = ka ? a : b, dl = ka ? b : a;
        const int s = lsz[kl] + lsz[dl];
        lsz[kl] = s;
        lpar[dl] = kl;
        par[drop] = keep;
        sz[keep] = s;
        const int q = ts[i];
        rk[lo + q] = keep;
        rd[lo + q] = drop;
        rs[lo + q] = s;
      }
    }
    __syncwarp();
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
  replay_init_kernel<<<grid_for(std::max<int64_t>(n, 8)), 256, 0, st>>>(n, s.par, s.sz, s.ctl);
  return cudaGetLastError();
}

cudaError_t replay_chunk(const ReplayEdge* e, int64_t lo, int cnt, int lmax, const ReplayState& s,
                         cudaStream_t st, int* chunk_max) {
  if (cnt <= 0) return cudaSuccess;
  const int g = grid_for(cnt);
  lmax = std::min(lmax, REPLAY_LMAX);
  replay_roots_kernel<<<g, 256, 0, st>>>(e, lo, cnt, s.par, s.lab, s.head, s.ea, s.eb, s.ctl);
  replay_link_kernel<<<g, 256, 0, st>>>(cnt, s.lab, s.ea, s.eb, s.ctl);
  replay_list_kernel<<<g, 256, 0, st>>>(cnt, s.lab, s.ea, s.eb, s.head, s.nxt, s.comp, s.rid,
                                        s.rcnt, s.ctl);
  replay_check_kernel<<<g, 256, 0, st>>>(lo, cnt, s.head, s.nxt, s.comp, lmax, s.ctl, chunk_max,
                                         s.base, s.llist);
  replay_place_kernel<<<g, 256, 0, st>>>(cnt, s.nxt, s.comp, s.base, s.ea, s.eb, s.slot, s.rid,
                                         s.rcnt, s.ctl);
  replay_segment_kernel<<<g, 256, 0, st>>>(lo, cnt, s.head, s.nxt, s.comp, s.ea, s.eb, s.base,
                                           s.slot, s.par, s.sz, s.rk, s.rd, s.rs, s.ctl);
  const int gl = std::max(1, std::min(grid_for(cnt, 32 * REPLAY_WARPS), 148 * 8));
  replay_long_kernel<<<gl, 32 * REPLAY_WARPS, 0, st>>>(lo, s.llist, s.head, s.comp, s.ea, s.eb,
                                                        s.base, s.slot, s.rid, s.rcnt, s.par,
                                                        s.sz, s.rk, s.rd, s.rs, s.ctl);
  return cudaGetLastError();
}

cudaError_t replay_assign(int64_t n, const ReplayState& s, int* out, cudaStream_t st) {
  replay_assign_kernel<<<grid_for(n), 256, 0, st>>>(n, s.par, out);
  return cudaGetLastError();
}

}  // namespace nnm
