// nnm_api.cu -- C ABI, dataset residency, FP64 exact kernels, Boruvka and
// top-P round orchestration for the B200 NNM hot path.
//
// Reference mapping (paths relative to /root/reference/pkg/src/parclust/):
//   nnm_dataset_create  <- model.Dataset (model.py:29-76)
//   nnm_top_p           <- scheduler.run_round / pairgen.global_top_p
//                          (scheduler.py:268-335, pairgen.py:247-324)
//   nnm_run             <- engine.run (engine.py:154-199) incl. order_batch
//                          (:73-87) and process_batch (:90-143)
//   nnm_pairwise        <- metrics.internal_pairwise (metrics.py:67-73)
// The paper's CPU "managers" (scheduler.py:268-335) become one stream per
// dataset: kernels are queued back to back and the host only syncs to read
// counts that size the next launch.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>
#include <cooperative_groups.h>
#include <cub/device/device_radix_sort.cuh>
#include <thrust/device_ptr.h>
#include <thrust/execution_policy.h>
#include <thrust/sort.h>
#include <thrust/scan.h>
#include <thrust/unique.h>

#include <algorithm>
#include <cstdio>
#include <atomic>
#include <chrono>
#include <cmath>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/nnm.h"
#include "nnm_common.cuh"
#include "nnm_kernels.cuh"
#include "nnm_tc.cuh"

// native CSV ingestion (nnm_csv.cpp)
int nnm_csv_parse_impl(const char* path, char delim, const char* id_column, int threads,
                       nnm_csv** out, std::string& err);
int64_t nnm_csv_rows(const nnm_csv* c);
int64_t nnm_csv_cols(const nnm_csv* c);
bool nnm_csv_has_ids(const nnm_csv* c);
void nnm_csv_copy_values(const nnm_csv* c, double* out);
int64_t nnm_csv_id_bytes(const nnm_csv* c);
void nnm_csv_copy_ids(const nnm_csv* c, char* buf, int64_t* offsets);
void nnm_csv_destroy(nnm_csv* c);
int64_t nnm_first_nonfinite_impl(const double* x, int64_t count, int threads);

using namespace nnm;

// ----------------------------------------------------------------------------
// errors
// ----------------------------------------------------------------------------
namespace {
thread_local std::string g_err;

struct NnmError {
  int code;
  std::string msg;
};

#define CUDA_TRY(x)                                                                       \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess)                                                                \
      throw NnmError{e_ == cudaErrorMemoryAllocation ? NNM_E_NOMEM : NNM_E_CUDA,          \
                     std::string(#x) + " failed: " + cudaGetErrorString(e_)};             \
  } while (0)

[[noreturn]] void invalid(const std::string& m) { throw NnmError{NNM_E_INVALID, m}; }

thread_local cudaStream_t t_alloc_stream = nullptr;  // stream for DevBuf allocations


template <class F>
int guarded(F&& f) {
  // every entry point starts on the default stream; dataset entry points then select the
  // dataset's own stream (a stale stream of a destroyed dataset must never be reused)
  t_alloc_stream = nullptr;
  try {
    f();
    return NNM_OK;
  } catch (const NnmError& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_err = std::string("internal error: ") + e.what();
    return NNM_E_CUDA;
  }
}

// Device buffers come from the stream-ordered pool (cudaMallocAsync) on the
// stream of the dataset being worked on, with the pool's release threshold
// raised: repeated dataset create / destroy (one per user call through the
// reference-facing API) then costs no cudaMalloc / device-wide cudaFree syncs.

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFreeAsync(p, s);
  }
  void ensure(size_t count) {
    if (count <= n && p) return;
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
    s = t_alloc_stream;
    size_t c = count > 0 ? count : 1;
    CUDA_TRY(cudaMallocAsync((void**)&p, c * sizeof(T), s));
    n = c;
  }
};

// Page-locked host blocks are recycled process-wide: cudaMallocHost / cudaFreeHost
// cost milliseconds to seconds (page pinning, implicit device sync), and the
// reference-facing API creates one dataset per user call.
struct PinnedPool {
  std::mutex mu;
  std::multimap<size_t, void*> free_blocks;
  void* get(size_t& bytes) {
    {
      std::lock_guard<std::mutex> lk(mu);
      auto it = free_blocks.lower_bound(bytes);
      if (it != free_blocks.end()) {
        bytes = it->first;
        void* p = it->second;
        free_blocks.erase(it);
        return p;
      }
    }
    void* p = nullptr;
    CUDA_TRY(cudaMallocHost(&p, bytes));
    return p;
  }
  void put(void* p, size_t bytes) {
    std::lock_guard<std::mutex> lk(mu);
    free_blocks.emplace(bytes, p);
  }
};
PinnedPool& pinned_pool() {
  static PinnedPool* pool = new PinnedPool();  // never destroyed: outlives every dataset
  return *pool;
}

// blocks handed to callers through nnm_host_alloc (size needed to recycle them)
std::mutex g_host_mu;
std::map<void*, size_t> g_host_blocks;

// page-locked (cudaMallocHost / cudaHostRegister) host memory: the copy engine can write
// the run's outputs there directly
bool is_page_locked(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

template <class T>
struct PinnedBuf {  // grow-only page-locked host staging buffer (blocks from pinned_pool)
  T* p = nullptr;
  size_t n = 0, bytes = 0;
  PinnedBuf() = default;
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
  ~PinnedBuf() {
    if (p) pinned_pool().put(p, bytes);
  }
  T* ensure(size_t count) {
    if (count <= n && p) return p;
    if (p) pinned_pool().put(p, bytes);
    p = nullptr;
    n = 0;
    bytes = std::max<size_t>(count, 1) * sizeof(T);
    p = (T*)pinned_pool().get(bytes);
    n = bytes / sizeof(T);
    return p;
  }
};

// NVTX ranges (header-only NVTX3: free unless a profiler attaches) per run / round / phase
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  NvtxRange(const char* fmt, long long v) {
    char b[64];
    snprintf(b, sizeof(b), fmt, v);
    nvtxRangePushA(b);
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

std::atomic<int64_t> g_launches{0};  // libnnm kernel launches (process-wide)
inline void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

inline int blocks_for(int64_t n, int t = 256) { return (int)std::max<int64_t>(1, (n + t - 1) / t); }

inline double bits_to_double(unsigned long long b) {
  double d;
  memcpy(&d, &b, 8);
  return d;
}
}  // namespace

// ----------------------------------------------------------------------------
// small kernels
// ----------------------------------------------------------------------------
namespace nnm {

__device__ __forceinline__ unsigned long long dbits(double x) {
  return (unsigned long long)__double_as_longlong(x);
}
__device__ __forceinline__ double bitsd(unsigned long long b) {
  return __longlong_as_double((long long)b);
}

// X64 (row-major) -> X32 SoA [d][ld] rounded to nearest, +inf padding.
// FP32 SoA copy + input checks on the device: chk[0] = first row holding a non-finite
// value (model.py:29-76 message), chk[1] = 1 if a finite value is beyond the FP32 screen
__global__ void prepare_kernel(const double* __restrict__ X64, int64_t n, int d, int64_t ld,
                               float* __restrict__ X32, unsigned long long* chk) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ld) return;
  for (int k = 0; k < d; ++k) {
    float v = INFINITY;
    if (i < n) {
      double x = X64[i * d + k];
      if (!isfinite(x)) atomicMin(chk, (unsigned long long)i);
      else if (!(fabs(x) <= 1e18)) atomicExch(chk + 1, 1ull);
      v = __double2float_rn(x);
    }
    X32[(int64_t)k * ld + i] = v;
  }
}

// permuted view: X32 SoA of positions (pads +inf)
__global__ void prepare_view_kernel(const double* __restrict__ X64p, const int* __restrict__ porig,
                                    int64_t np, int d, float* __restrict__ X32p) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= np) return;
  const bool real = porig[p] >= 0;
  for (int k = 0; k < d; ++k)
    X32p[(int64_t)k * np + p] = real ? __double2float_rn(X64p[p * d + k]) : INFINITY;
}

// per-point norm in the metric's norm, rounded up; global max via atomicMax on bits
__global__ void norms_kernel(const double* __restrict__ X64, int64_t n, int d, int metric,
                             double* __restrict__ norm, unsigned long long* maxbits) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* x = X64 + i * d;
  double s = 0.0;
  if (metric == EUCLIDEAN || metric == SQEUCLIDEAN) {
    for (int k = 0; k < d; ++k) s += x[k] * x[k];
    s = sqrt(s) * (1.0 + 1e-12) + 1e-300;
  } else if (metric == MANHATTAN) {
    for (int k = 0; k < d; ++k) s += fabs(x[k]);
    s = s * (1.0 + 1e-12) + 1e-300;
  } else {
    for (int k = 0; k < d; ++k) s = fmax(s, fabs(x[k]));
    s = s * (1.0 + 1e-12) + 1e-300;
  }
  norm[i] = s;
  // one atomic per warp (2M same-address atomics serialise at the L2)
  unsigned long long m = dbits(s);
  if (__activemask() != 0xFFFFFFFFu) {  // the ragged last warp: one atomic per row
    atomicMax(maxbits, m);
    return;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long q = __shfl_xor_sync(0xFFFFFFFFu, m, o);
    m = q > m ? q : m;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(maxbits, m);
}

template <int M>
__global__ void pairwise_kernel(const double* __restrict__ X, int64_t nx,
                                const double* __restrict__ Y, int64_t ny, int d,
                                double* __restrict__ out) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nx * ny) return;
  int64_t i = t / ny, j = t % ny;
  out[t] = exact_dist<M>(X + i * d, Y + j * d, d);
}

template <int M>
__global__ void exact_pairs_kernel(const double* __restrict__ X64, int d,
                                   const int2* __restrict__ pairs, int64_t count,
                                   double* __restrict__ out) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  int2 p = pairs[t];
  out[t] = exact_dist<M>(X64 + (int64_t)p.x * d, X64 + (int64_t)p.y * d, d);
}

__global__ void fill_comp_kernel(int* comp, int* psize, int64_t n, int64_t ld) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ld) return;
  comp[i] = i < n ? (int)i : -1;
  if (psize) psize[i] = i < n ? 1 : 0;
}

// Boruvka refine: exact FP64 key of each row's screened best partner, and
// certification against the screened second best.
template <int M>
__global__ void refine_kernel(const double* __restrict__ X64, int n, int d,
                              const unsigned long long* __restrict__ B1,
                              const unsigned long long* __restrict__ B2,
                              const double* __restrict__ norm, double maxnorm, ErrModel em,
                              double thr, unsigned long long* rb_d, int* rb_j, double* rowlow,
                              int* amb, unsigned long long* amb_count,
                              const int* __restrict__ orig, int keys_lower) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned long long k1 = B1[i];
  if (!key_valid(k1)) {
    rb_d[i] = NONE_KEY;
    rb_j[i] = -1;
    rowlow[i] = INFINITY;
    return;
  }
  int j = (int)key_index(k1);
  double e = exact_dist<M>(X64 + (int64_t)i * d, X64 + (int64_t)j * d, d);
  // keys are screened values (direct form) or already rigorous lower bounds (dot form)
  double R = norm[i] + maxnorm;
  rowlow[i] = keys_lower ? (double)key_value(k1) : exact_lower(em, (double)key_value(k1), R);
  unsigned long long k2 = B2[i];
  double low2 = !key_valid(k2) ? INFINITY
                : (keys_lower ? (double)key_value(k2) : exact_lower(em, (double)key_value(k2), R));
  if (e <= thr) {
    rb_d[i] = dbits(e);
    rb_j[i] = orig[j];  // partner as ORIGINAL index (tie-break order of the reference)
    if (low2 > e) return;  // certified: every other partner is strictly farther
  } else {
    rb_d[i] = NONE_KEY;
    rb_j[i] = -1;
    if (low2 > thr) return;  // certified: no eligible partner at all
  }
  unsigned long long pos = atomicAdd(amb_count, 1ull);
  amb[pos] = i;
}

__global__ void compmin_d_kernel(int n, const int* __restrict__ comp,
                                 const unsigned long long* __restrict__ rb_d,
                                 unsigned long long* cmin_d) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned long long v = rb_d[i];
  if (v != NONE_KEY) atomicMin(cmin_d + comp[i], v);
}

__global__ void compmin_ab_kernel(int n, const int* __restrict__ comp,
                                  const unsigned long long* __restrict__ rb_d,
                                  const int* __restrict__ rb_j,
                                  const unsigned long long* __restrict__ cmin_d,
                                  unsigned long long* cmin_ab, const int* __restrict__ orig) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned long long v = rb_d[i];
  int c = comp[i];
  if (v == NONE_KEY || v != cmin_d[c]) return;
  const int oi = orig[i];  // pair key in original indices: (dist, a, b), model.py:100-106
  unsigned a = (unsigned)min(oi, rb_j[i]), b = (unsigned)max(oi, rb_j[i]);
  atomicMin(cmin_ab + c, ((unsigned long long)a << 32) | b);
}

// ambiguous rows that could still hold their component's minimum
__global__ void amb_filter_kernel(const int* __restrict__ amb, int na, const int* __restrict__ comp,
                                  const double* __restrict__ rowlow,
                                  const unsigned long long* __restrict__ cmin_d,
                                  const unsigned long long* __restrict__ rb_d, double thr,
                                  const double* __restrict__ norm, double maxnorm, ErrModel em,
                                  int* out, float* bound, unsigned long long* count) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= na) return;
  int i = amb[t];
  unsigned long long cb = cmin_d[comp[i]];
  double cm = cb == NONE_KEY ? INFINITY : bitsd(cb);
  if (!(rowlow[i] <= cm)) return;
  double e = rb_d[i] == NONE_KEY ? INFINITY : bitsd(rb_d[i]);
  double lim = fmin(e, thr);
  unsigned long long pos = atomicAdd(count, 1ull);
  out[pos] = i;
  bound[pos] = float_up(screen_upper(em, lim, norm[i] + maxnorm));
}

// gather rows (global ids) into a SoA block [d][ldr]
__global__ void gather_kernel(const float* __restrict__ X32, int64_t ld, int d,
                              const int* __restrict__ ids, int nr, int64_t ldr,
                              float* __restrict__ out) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ldr) return;
  int g = t < nr ? ids[t] : -1;
  for (int k = 0; k < d; ++k) out[(int64_t)k * ldr + t] = g >= 0 ? X32[(int64_t)k * ld + g] : INFINITY;
}

__global__ void reset_rows_kernel(const int* __restrict__ rows, int nr, unsigned long long* rb_d,
                                  int* rb_j) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nr) return;
  rb_d[rows[t]] = NONE_KEY;
  rb_j[rows[t]] = 0x7FFFFFFF;
}

__global__ void rowmin_d_kernel(const int2* __restrict__ pairs, const double* __restrict__ dv,
                                int64_t count, double thr, unsigned long long* rb_d) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  if (dv[t] <= thr) atomicMin(rb_d + pairs[t].x, dbits(dv[t]));
}

__global__ void rowmin_j_kernel(const int2* __restrict__ pairs, const double* __restrict__ dv,
                                int64_t count, double thr, const unsigned long long* rb_d,
                                int* rb_j, const int* __restrict__ orig) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  int2 p = pairs[t];
  if (dv[t] <= thr && dbits(dv[t]) == rb_d[p.x]) atomicMin(rb_j + p.x, orig[p.y]);
}

__global__ void fix_rows_kernel(const int* __restrict__ rows, int nr,
                                const unsigned long long* rb_d, int* rb_j) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nr) return;
  if (rb_d[rows[t]] == NONE_KEY) rb_j[rows[t]] = -1;
}

struct ItemLess {  // order int2 {I, J} stored as u64 (low = I, high = J) by (I, J)
  __host__ __device__ bool operator()(unsigned long long a, unsigned long long b) const {
    const long long ia = (int)(a & 0xFFFFFFFFull), ib = (int)(b & 0xFFFFFFFFull);
    if (ia != ib) return ia < ib;
    return (int)(a >> 32) < (int)(b >> 32);
  }
};

struct Edge {
  double d;
  int a, b;
  int round;
  int pad;
};

struct EdgeLess {
  __host__ __device__ bool operator()(const Edge& x, const Edge& y) const {
    if (x.d != y.d) return x.d < y.d;
    if (x.a != y.a) return x.a < y.a;
    return x.b < y.b;
  }
};

__global__ void replay_edges_kernel(const Edge* __restrict__ e, int64_t ne, int sqrt_dist,
                                    ReplayEdge* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ne) return;
  const Edge x = e[t];
  ReplayEdge r;
  r.dist = sqrt_dist ? sqrt(x.d) : x.d;  // IEEE sqrt, as np.sqrt (metrics.py:86-90)
  r.a = x.a;
  r.b = x.b;
  r.round = x.round;
  r.pad = 0;
  out[t] = r;
}

// merge records [0, m) of the GPU replay, laid out as the caller's nnm_merge array
// (copied into page-locked output by the copy engine; nnm_api bv_end)
__global__ void merge_records_kernel(const ReplayEdge* __restrict__ e, int64_t m,
                                     const int* __restrict__ rk, const int* __restrict__ rd,
                                     const int* __restrict__ rs, nnm_merge* __restrict__ out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const ReplayEdge x = e[k];
  nnm_merge r;
  r.round = x.round;
  r.root_a = rk[k];
  r.root_b = rd[k];
  r.dist = x.dist;
  r.new_size = rs[k];
  r.point_a = x.a;
  r.point_b = x.b;
  out[k] = r;
}

// the host tail's links (dropped root -> kept root, kept < dropped) onto the GPU forest
__global__ void apply_links_kernel(const int2* __restrict__ links, int64_t cnt, int* par) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < cnt) par[links[t].x] = links[t].y;
}

// final labels (root = minimum index of the cluster, model.py:148-160) as int64; links
// only point to smaller indices, so concurrent path halving is benign
__global__ void assign64_kernel(int64_t n, int* par, int64_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int x = (int)i, p = par[x];
  while (p != x) {
    const int g = par[p];
    if (g != p) par[x] = g;
    x = g;
    p = par[x];
  }
  out[i] = x;
}

__global__ void hook_kernel(int n, const int* __restrict__ comp,
                            const unsigned long long* __restrict__ cmin_d,
                            const unsigned long long* __restrict__ cmin_ab, int* parent,
                            Edge* edges, unsigned long long* edge_count, int round,
                            const int* __restrict__ pos) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n || comp[c] != c) return;
  unsigned long long e = cmin_ab[c];
  if (e == NONE_KEY) {
    parent[c] = c;
    return;
  }
  int a = (int)(e >> 32), b = (int)(e & 0xFFFFFFFFull);
  int ca = comp[pos[a]], cb = comp[pos[b]];  // a, b are original indices
  int other = (ca == c) ? cb : ca;
  bool mutual = (cmin_ab[other] == e);
  bool record = !mutual || c < other;
  parent[c] = (mutual && c < other) ? c : other;
  if (record) {
    unsigned long long pos = atomicAdd(edge_count, 1ull);
    Edge ed;
    ed.d = bitsd(cmin_d[c]);
    ed.a = a;
    ed.b = b;
    ed.round = round;
    ed.pad = 0;
    edges[pos] = ed;
  }
}

__global__ void jump_kernel(int n, const int* __restrict__ comp, int* parent, int* changed) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n || comp[c] != c) return;
  int p = parent[c];
  int pp = parent[p];
  if (p != pp) {
    parent[c] = pp;
    *changed = 1;
  }
}

// every component root follows its hook chain to the final root; concurrent path halving
// only ever stores ancestors into `parent`, and the result goes to a separate array (a
// halving store by another thread must not overwrite a final root)
__global__ void find_roots_kernel(int n, const int* __restrict__ comp, int* parent,
                                  int* __restrict__ root) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n || comp[c] != c) return;
  int x = c;
  for (;;) {
    const int p = parent[x];
    const int pp = parent[p];
    if (p == pp) {
      x = p;
      break;
    }
    parent[x] = pp;  // halving
    x = pp;
  }
  root[c] = x;
}

__global__ void relabel_kernel(int n, int* comp, const int* __restrict__ parent) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || comp[i] < 0) return;
  comp[i] = parent[comp[i]];
}


// ---- dense exact Boruvka for small inputs: ONE cooperative launch for all rounds -------
// Every cross-component pair is evaluated in FP64 (scipy order) each round; per row the
// lexicographic minimum (d, a, b) (model.py:100-106), per component its minimum (two
// atomicMin passes), hooking of mutual pairs (the smaller label roots), pointer jumping and
// relabelling -- the same round as the general path in one launch, with no screening and no
// pruning (an independent exact algorithm; opt-in, NNM_SMALL=1).  Grid-wide barriers
// separate the steps; no kernel waits on another launch.
// ctl: [0] edges (cumulative), [1] edges this round, [2] jump flag, [3] rounds,
// [4] distance evaluations.
template <int M, int D, int R>
__global__ void __launch_bounds__(256) small_boruvka_kernel(
    const double* __restrict__ X, int n, int d, double thr, int max_rounds, int* comp, int* parent,
    unsigned long long* rbd, unsigned long long* rbab, unsigned long long* cmd,
    unsigned long long* cmab, Edge* edges, unsigned long long* ctl) {
  namespace cg = cooperative_groups;
  constexpr int SMALL_RPB = 8 * R;  // rows per block pass: 8 warps x R rows
  __shared__ double xs[D][256];
  __shared__ int cs[256];
  cg::grid_group grid = cg::this_grid();
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  for (int i = tid; i < n; i += nth) {
    comp[i] = i;
    cmd[i] = cmab[i] = NONE_KEY;
  }
  grid.sync();
  int round = 0;
  while (round < max_rounds) {
    // A. row minima: each warp owns R rows (coordinates in registers, zero padded to D:
    // adding (0 - 0) terms leaves every scipy-order value unchanged); the block stages 256
    // columns at a time in shared memory (SoA, conflict-free) and every lane takes columns
    unsigned long long evals = 0;
    for (int rb = blockIdx.x * SMALL_RPB; rb < n; rb += gridDim.x * SMALL_RPB) {
      const int i0 = rb + (threadIdx.x >> 5) * R;
      double xi[R][D];
      int ci[R];
      unsigned long long bd[R], bab[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = i0 + r;
        ci[r] = i < n ? comp[i] : -3;
        bd[r] = bab[r] = NONE_KEY;
#pragma unroll
        for (int k = 0; k < D; ++k) xi[r][k] = (i < n && k < d) ? X[(int64_t)i * d + k] : 0.0;
      }
      for (int jb = 0; jb < n; jb += 256) {
        __syncthreads();
        for (int idx = threadIdx.x; idx < 256 * D; idx += blockDim.x) {
          const int k = idx >> 8, j = idx & 255;
          xs[k][j] = (jb + j < n && k < d) ? X[(int64_t)(jb + j) * d + k] : 0.0;
        }
        cs[threadIdx.x] = jb + (int)threadIdx.x < n ? comp[jb + threadIdx.x] : -2;
        __syncthreads();
        for (int t = lane; t < 256 && jb + t < n; t += 32) {
          const int j = jb + t, cj = cs[t];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int i = i0 + r;
            if (i >= n || cj == ci[r]) continue;
            ++evals;
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) {  // scipy order (metrics.py:67-73)
              const double tt = __dsub_rn(xi[r][k], xs[k][t]);
              if (M == EUCLIDEAN || M == SQEUCLIDEAN) acc = __dadd_rn(acc, __dmul_rn(tt, tt));
              else if (M == MANHATTAN) acc = __dadd_rn(acc, fabs(tt));
              else acc = fmax(acc, fabs(tt));
            }
            if (!(acc <= thr)) continue;  // thr = +inf without dmax (pairgen.py:197-198)
            const unsigned long long kd = dbits(acc);
            const unsigned long long kab = ((unsigned long long)min(i, j) << 32) | (unsigned)max(i, j);
            if (kd < bd[r] || (kd == bd[r] && kab < bab[r])) {
              bd[r] = kd;
              bab[r] = kab;
            }
          }
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        unsigned long long b1 = bd[r], b2 = bab[r];
        for (int o = 16; o > 0; o >>= 1) {
          const unsigned long long od = __shfl_xor_sync(0xFFFFFFFFu, b1, o);
          const unsigned long long oab = __shfl_xor_sync(0xFFFFFFFFu, b2, o);
          if (od < b1 || (od == b1 && oab < b2)) {
            b1 = od;
            b2 = oab;
          }
        }
        const int i = i0 + r;
        if (lane == 0 && i < n) {
          rbd[i] = b1;
          rbab[i] = b2;
          if (b1 != NONE_KEY) atomicMin(cmd + ci[r], b1);
        }
      }
    }
    evals = __reduce_add_sync(0xFFFFFFFFu, (unsigned)evals);
    if (lane == 0 && evals) atomicAdd(ctl + 4, evals);
    grid.sync();
    // B. component minimum (d, a, b)
    for (int i = tid; i < n; i += nth) {
      const int ci = comp[i];
      if (rbd[i] != NONE_KEY && rbd[i] == cmd[ci]) atomicMin(cmab + ci, rbab[i]);
    }
    grid.sync();
    // C. hook (roots: comp[c] == c); each MST edge recorded once
    for (int c = tid; c < n; c += nth) {
      if (comp[c] != c) continue;
      const unsigned long long e = cmab[c];
      if (e == NONE_KEY) {
        parent[c] = c;
        continue;
      }
      const int a = (int)(e >> 32), b = (int)(e & 0xFFFFFFFFull);
      const int other = comp[a] == c ? comp[b] : comp[a];
      const bool mutual = cmab[other] == e;
      parent[c] = (mutual && c < other) ? c : other;
      if (!mutual || c < other) {
        const unsigned long long at = atomicAdd(ctl + 0, 1ull);
        Edge ed;
        ed.d = bitsd(cmd[c]);
        ed.a = a;
        ed.b = b;
        ed.round = round + 1;
        ed.pad = 0;
        edges[at] = ed;
        atomicAdd(ctl + 1, 1ull);
      }
    }
    grid.sync();
    // D. pointer jumping to the roots
    for (;;) {
      if (tid == 0) ctl[2] = 0;
      grid.sync();
      for (int c = tid; c < n; c += nth) {
        if (comp[c] != c) continue;
        const int pc = parent[c], pp = parent[pc];
        if (pc != pp) {
          parent[c] = pp;
          ctl[2] = 1;
        }
      }
      grid.sync();
      const unsigned long long changed = *((volatile unsigned long long*)(ctl + 2));
      grid.sync();
      if (!changed) break;
    }
    // E. relabel, reset the component minima
    for (int i = tid; i < n; i += nth) comp[i] = parent[comp[i]];
    grid.sync();
    for (int i = tid; i < n; i += nth) cmd[i] = cmab[i] = NONE_KEY;
    ++round;
    const unsigned long long added = *((volatile unsigned long long*)(ctl + 1));
    grid.sync();
    if (tid == 0) ctl[1] = 0;
    if (added == 0) break;
    grid.sync();
  }
  if (tid == 0) ctl[3] = (unsigned long long)round;
}

// ---- screened Boruvka for small inputs: ONE cooperative launch for all rounds -----------
// The same round as small_boruvka_kernel, with the row minima found by an FP32 screen and
// certified in FP64 (the error model of nnm_common.cuh):
//   sweep    work units of (R rows) x (SMALL_CW columns) spread over every warp of the
//            grid; per unit and row the smallest and second smallest screened value
//            v1 <= v2 over the cross-component columns (FP32 direct differences, X32 SoA,
//            column data straight from L1/L2) and the column j1 of v1 -> partials;
//   certify  per row the top-2 over its partials, S1 = exact(i, j1) (scipy order),
//            U = S1 if S1 <= thr else thr.  Every column j with S_j <= U has
//            v_j <= screen_upper(U, R_i) =: B, so v2 > B proves j1 the unique minimum (or,
//            when S1 > thr, that no column is eligible);
//   resolve  rows with v2 <= B (ties, duplicates) -- one warp per row over every column
//            with v_j <= B, exact keys, lexicographic (d, a, b) minimum (model.py:100-106).
// R_i = norm(x_i) + max norm bounds norm(x_i) + norm(x_j) for every j.  Component minima,
// hooking, root finding and relabelling follow as in small_boruvka_kernel, with the
// pointer jumping replaced by a read-only walk to the root (one grid barrier).
constexpr int SMALL_CW = 2048;       // columns per work unit
constexpr int SMALL_AUTO_N = 16384;  // default-on size limit (n^2 work per round)
template <int M, int D, int R>
__global__ void __launch_bounds__(256) small_screened_kernel(
    const double* __restrict__ X, const float* __restrict__ X32, int64_t ld, int n, int d,
    double thr, const double* __restrict__ norm, double maxnorm, ErrModel em, int max_rounds,
    int* comp, int* parent, unsigned long long* rbd, unsigned long long* rbab,
    unsigned long long* cmd, unsigned long long* cmab, Edge* edges, unsigned long long* ctl,
    float* pv1, float* pv2, int* pj1, int* needl, int* rootof, float2* ndup) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31, gw = tid >> 5, nw = nth >> 5;
  const int C = (n + SMALL_CW - 1) / SMALL_CW, G = (n + R - 1) / R;
  for (int i = tid; i < n; i += nth) {
    comp[i] = i;
    cmd[i] = cmab[i] = NONE_KEY;
  }
  if (tid == 0) ctl[5] = 0;
  // packed negated columns {-x, -x}, SoA [D][n]: a warp's 64-bit loads of one coordinate
  // are 256 contiguous bytes; each feeds the FADD2 of two rows
  if (M == EUCLIDEAN || M == SQEUCLIDEAN)
    for (int64_t q = tid; q < (int64_t)D * n; q += nth) {
      const int k = (int)(q / n), j = (int)(q - (int64_t)k * n);
      const float x = k < d ? -X32[(int64_t)k * ld + j] : 0.f;
      ndup[q] = make_float2(x, x);
    }
  grid.sync();
  auto screened = [&](const float* xi, int j) {
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const float tt = xi[k] - (k < d ? __ldg(X32 + (int64_t)k * ld + j) : 0.f);
      if (M == EUCLIDEAN || M == SQEUCLIDEAN) acc = __fmaf_rn(tt, tt, acc);
      else if (M == MANHATTAN) acc += fabsf(tt);
      else acc = fmaxf(acc, fabsf(tt));
    }
    return acc;
  };
  auto exact = [&](int i, int j) {
    double acc = 0.0;
    for (int k = 0; k < d; ++k) {  // scipy order (metrics.py:67-73)
      const double tt = __dsub_rn(X[(int64_t)i * d + k], X[(int64_t)j * d + k]);
      if (M == EUCLIDEAN || M == SQEUCLIDEAN) acc = __dadd_rn(acc, __dmul_rn(tt, tt));
      else if (M == MANHATTAN) acc = __dadd_rn(acc, fabs(tt));
      else acc = fmax(acc, fabs(tt));
    }
    return acc;
  };
  auto pack = [](int i, int j) {
    return ((unsigned long long)min(i, j) << 32) | (unsigned)max(i, j);
  };
  int round = 0;
  while (round < max_rounds) {
    // sweep: screened top-2 per (row, column chunk)
    unsigned long long evals = 0;
    for (int u = gw; u < G * C; u += nw) {
      const int g = u / C, c = u - g * C;
      const int i0 = g * R, jb = c * SMALL_CW, je = min(n, jb + SMALL_CW);
      float2 xi2[R / 2][D];  // rows (2p, 2p + 1) packed
      int ci[R];
      float v1[R], v2[R];
      int j1[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = i0 + r;
        ci[r] = i < n ? comp[i] : -3;
        v1[r] = v2[r] = INFINITY;
        j1[r] = -1;
#pragma unroll
        for (int k = 0; k < D; ++k) {
          const float x = (i < n && k < d) ? X32[(int64_t)k * ld + i] : 0.f;
          if (r & 1) xi2[r >> 1][k].y = x;
          else xi2[r >> 1][k].x = x;
        }
      }
      for (int j = jb + lane; j < je; j += 32) {
        const int cj = __ldg(comp + j);
        float v[R];
        if (M == EUCLIDEAN || M == SQEUCLIDEAN) {
          float2 nx[D];
          const float2* col = ndup + j;
#pragma unroll
          for (int k = 0; k < D; ++k) nx[k] = __ldg(col + (int64_t)k * n);
#pragma unroll
          for (int p = 0; p < R / 2; ++p) {  // two rows per packed FADD2 / FFMA2
            float2 acc = make_float2(0.f, 0.f);
#pragma unroll
            for (int k = 0; k < D; ++k) {
              const float2 tt = __fadd2_rn(xi2[p][k], nx[k]);
              acc = __ffma2_rn(tt, tt, acc);
            }
            v[2 * p] = acc.x;
            v[2 * p + 1] = acc.y;
          }
        } else {
          float xj[D];
#pragma unroll
          for (int k = 0; k < D; ++k) xj[k] = k < d ? __ldg(X32 + (int64_t)k * ld + j) : 0.f;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < D; ++k) {
              const float tt = (r & 1 ? xi2[r >> 1][k].y : xi2[r >> 1][k].x) - xj[k];
              if (M == MANHATTAN) acc += fabsf(tt);
              else acc = fmaxf(acc, fabsf(tt));
            }
            v[r] = acc;
          }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {  // branch-free top-2 over the cross columns
          const bool cross = cj != ci[r] && ci[r] != -3;
          evals += cross;
          const float x = cross ? v[r] : INFINITY;
          const bool lt = x < v1[r];
          v2[r] = lt ? v1[r] : fminf(v2[r], x);
          j1[r] = lt ? j : j1[r];
          v1[r] = fminf(v1[r], x);
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        float a1 = v1[r], a2 = v2[r];
        int aj = j1[r];
        for (int o = 16; o > 0; o >>= 1) {
          const float b1 = __shfl_xor_sync(0xFFFFFFFFu, a1, o);
          const float b2 = __shfl_xor_sync(0xFFFFFFFFu, a2, o);
          const int bj = __shfl_xor_sync(0xFFFFFFFFu, aj, o);
          const bool take = b1 < a1 || (b1 == a1 && bj >= 0 && (aj < 0 || bj < aj));
          a2 = fminf(fmaxf(a1, b1), fminf(a2, b2));
          a1 = fminf(a1, b1);
          aj = take ? bj : aj;
        }
        const int i = i0 + r;
        if (lane == 0 && i < n) {
          pv1[(int64_t)c * n + i] = a1;
          pv2[(int64_t)c * n + i] = a2;
          pj1[(int64_t)c * n + i] = aj;
        }
      }
    }
    evals = __reduce_add_sync(0xFFFFFFFFu, (unsigned)evals);
    if (lane == 0 && evals) atomicAdd(ctl + 4, evals);
    grid.sync();
    // certify: one thread per row
    for (int i = tid; i < n; i += nth) {
      float a1 = INFINITY, a2 = INFINITY;
      int aj = -1;
      for (int c = 0; c < C; ++c) {
        const float b1 = pv1[(int64_t)c * n + i], b2 = pv2[(int64_t)c * n + i];
        const int bj = pj1[(int64_t)c * n + i];
        const bool take = b1 < a1 || (b1 == a1 && bj >= 0 && (aj < 0 || bj < aj));
        a2 = fminf(fmaxf(a1, b1), fminf(a2, b2));
        a1 = fminf(a1, b1);
        aj = take ? bj : aj;
      }
      unsigned long long kd = NONE_KEY, kab = NONE_KEY;
      if (aj >= 0) {
        const double S1 = exact(i, aj);
        const double U = S1 <= thr ? S1 : thr;
        const double B = screen_upper(em, U, norm[i] + maxnorm);
        if ((double)a2 > B) {
          if (S1 <= thr) {
            kd = dbits(S1);
            kab = pack(i, aj);
          }
        } else {
          needl[atomicAdd((int*)(ctl + 5), 1)] = i;
          rbd[i] = dbits(B);  // the bound, for the resolve step
          continue;
        }
      }
      rbd[i] = kd;
      rbab[i] = kab;
      if (kd != NONE_KEY) atomicMin(cmd + comp[i], kd);
    }
    grid.sync();
    // resolve (ties / near ties): one warp per listed row over every column
    const int nneed = *((volatile int*)(ctl + 5));
    if (nneed > 0) {
      for (int q = gw; q < nneed; q += nw) {
        const int i = needl[q], ci = comp[i];
        const double B = bitsd(rbd[i]);
        float xi[D];
#pragma unroll
        for (int k = 0; k < D; ++k) xi[k] = k < d ? X32[(int64_t)k * ld + i] : 0.f;
        unsigned long long b1 = NONE_KEY, b2 = NONE_KEY;
        for (int j = lane; j < n; j += 32) {
          if (__ldg(comp + j) == ci) continue;
          if ((double)screened(xi, j) > B) continue;
          const double S = exact(i, j);
          if (!(S <= thr)) continue;
          const unsigned long long k1 = dbits(S), k2 = pack(i, j);
          if (k1 < b1 || (k1 == b1 && k2 < b2)) {
            b1 = k1;
            b2 = k2;
          }
        }
        for (int o = 16; o > 0; o >>= 1) {
          const unsigned long long od = __shfl_xor_sync(0xFFFFFFFFu, b1, o);
          const unsigned long long oab = __shfl_xor_sync(0xFFFFFFFFu, b2, o);
          if (od < b1 || (od == b1 && oab < b2)) {
            b1 = od;
            b2 = oab;
          }
        }
        if (lane == 0) {
          rbd[i] = b1;
          rbab[i] = b2;
          if (b1 != NONE_KEY) atomicMin(cmd + ci, b1);
        }
      }
      grid.sync();
    }
    // component minimum (d, a, b)
    for (int i = tid; i < n; i += nth) {
      const int ci = comp[i];
      if (rbd[i] != NONE_KEY && rbd[i] == cmd[ci]) atomicMin(cmab + ci, rbab[i]);
    }
    grid.sync();
    // hook (roots: comp[c] == c); each MST edge recorded once
    for (int c = tid; c < n; c += nth) {
      if (comp[c] != c) continue;
      const unsigned long long e = cmab[c];
      if (e == NONE_KEY) {
        parent[c] = c;
        continue;
      }
      const int a = (int)(e >> 32), b = (int)(e & 0xFFFFFFFFull);
      const int other = comp[a] == c ? comp[b] : comp[a];
      const bool mutual = cmab[other] == e;
      parent[c] = (mutual && c < other) ? c : other;
      if (!mutual || c < other) {
        const unsigned long long at = atomicAdd(ctl + 0, 1ull);
        Edge ed;
        ed.d = bitsd(cmd[c]);
        ed.a = a;
        ed.b = b;
        ed.round = round + 1;
        ed.pad = 0;
        edges[at] = ed;
        atomicAdd(ctl + 1, 1ull);
      }
    }
    grid.sync();
    // roots: a read-only walk up the hook forest (its links are final)
    for (int c = tid; c < n; c += nth) {
      if (comp[c] != c) continue;
      int x = c;
      while (parent[x] != x) x = parent[x];
      rootof[c] = x;
    }
    const unsigned long long added = *((volatile unsigned long long*)(ctl + 1));
    grid.sync();
    // relabel, reset the component minima and the per-round counters
    for (int i = tid; i < n; i += nth) {
      comp[i] = rootof[comp[i]];
      cmd[i] = cmab[i] = NONE_KEY;
    }
    if (tid == 0) {
      ctl[1] = 0;
      ctl[5] = 0;
    }
    ++round;
    if (added == 0) break;
    grid.sync();
  }
  if (tid == 0) ctl[3] = (unsigned long long)round;
}

// ---- exact tile-pair pruning (Boruvka) -------------------------------------
// Tile geometry: FP64 centre (mean of the tile's real points) and radius (max
// metric distance of a point to the centre, inflated).  For any i in I, j in J:
//   dist(i, j) >= dist(c_I, c_J) - R_I - R_J   (triangle inequality)
// so LB_IJ bounds the exact scipy value of every pair of the tile pair.
template <int M>
__device__ __forceinline__ double metric_dist_real(const double* a, const double* b, int d) {
  double acc = 0.0;
  for (int k = 0; k < d; ++k) {
    double t = fabs(a[k] - b[k]);
    if (M == EUCLIDEAN || M == SQEUCLIDEAN) acc += t * t;
    else if (M == MANHATTAN) acc += t;
    else acc = fmax(acc, t);
  }
  return (M == EUCLIDEAN || M == SQEUCLIDEAN) ? sqrt(acc) : acc;
}

template <int M>
__global__ void tile_geom_kernel(const double* __restrict__ X64, const int* __restrict__ tcount, int d,
                                 double* __restrict__ centers, double* __restrict__ radius) {
  // real points of a tile are its first tcount[T0] positions (pads follow)
  const int T0 = blockIdx.x;
  const int64_t base = (int64_t)T0 * TILE;
  const int m = tcount[T0];
  extern __shared__ double sc[];  // [d]
  for (int k = threadIdx.x; k < d; k += blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < m; ++i) s += X64[(base + i) * d + k];
    sc[k] = m > 0 ? s / m : 0.0;
    centers[(int64_t)T0 * d + k] = sc[k];
  }
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < m) r = metric_dist_real<M>(X64 + (base + threadIdx.x) * d, sc, d);
  if (m == 0) r = 0.0;
  for (int o = 16; o > 0; o >>= 1) r = fmax(r, __shfl_xor_sync(0xFFFFFFFFu, r, o));
  __shared__ double sr[4];
  if ((threadIdx.x & 31) == 0) sr[threadIdx.x >> 5] = r;
  __syncthreads();
  if (threadIdx.x == 0) {
    r = fmax(fmax(sr[0], sr[1]), fmax(sr[2], sr[3]));
    radius[T0] = r * (1.0 + 1e-9) + 1e-300;
  }
}

// dot-form constants per position of the Boruvka view (nnm_common.cuh DotModel)
__global__ void dot_consts_kernel(const float* __restrict__ X32p, int64_t np, int d,
                                  const int* __restrict__ porig, const double* __restrict__ tcenter,
                                  const double* __restrict__ normp, double maxnorm, DotModel m,
                                  float* __restrict__ c32, float* __restrict__ Bout,
                                  float* __restrict__ nbk) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= np) return;
  const int64_t T0 = p / TILE;
  if (p % TILE == 0)
    for (int k = 0; k < d; ++k) c32[T0 * d + k] = __double2float_rn(tcenter[T0 * d + k]);
  if (porig[p] < 0) {
    Bout[p] = 0.f;
    nbk[p] = 0.f;
    return;
  }
  double r2 = 0.0;
  for (int k = 0; k < d; ++k) {
    const float c = __double2float_rn(tcenter[T0 * d + k]);
    const float xh = X32p[(int64_t)k * np + p] - c;  // exactly what the kernel computes
    r2 += (double)xh * (double)xh;
  }
  const double r = sqrt(r2) * (1.0 + 1e-12);
  const double nb = dot_negB(m, r, normp[p], maxnorm);
  nbk[p] = float_down(nb);
  Bout[p] = float_up(-nb * (1.0 + m.A));
}

__global__ void tile_bmax_kernel(const float* __restrict__ B, float* __restrict__ bmax) {
  const int T0 = blockIdx.x;
  float v = B[(int64_t)T0 * TILE + threadIdx.x];
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
  __shared__ float sm[4];
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) bmax[T0] = fmaxf(fmaxf(sm[0], sm[1]), fmaxf(sm[2], sm[3]));
}

// lower bound on the exact internal value of every pair of tile pair (I, J)
template <int M>
__device__ __forceinline__ double tile_lb(const double* __restrict__ centers,
                                          const double* __restrict__ radius, int d, int I, int J) {
  if (I == J) return 0.0;
  double dc = metric_dist_real<M>(centers + (int64_t)I * d, centers + (int64_t)J * d, d);
  double r = dc * (1.0 - 1e-9) - radius[I] - radius[J];
  if (!(r > 0.0)) return 0.0;
  return (M == EUCLIDEAN || M == SQEUCLIDEAN) ? r * r * (1.0 - 1e-9) : r * (1.0 - 1e-9);
}

__device__ __forceinline__ bool same_single(const int2* __restrict__ tr, int I, int J) {
  const int2 a = tr[I], b = tr[J];
  return a.x == a.y && b.x == b.y && a.x == b.x;
}

// FP32 SoA tile centres for the O(T^2) tile-level passes: c32[k][T], cn = metric norm of
// c32 (rounded up), r32 = radius rounded up.
template <int M>
__global__ void centers32_kernel(const double* __restrict__ centers, const double* __restrict__ radius,
                                 int T, int d, float* __restrict__ c32, float* __restrict__ cn,
                                 float* __restrict__ r32) {
  const int J = blockIdx.x * blockDim.x + threadIdx.x;
  if (J >= T) return;
  double nrm = 0.0;
  for (int k = 0; k < d; ++k) {
    const float c = __double2float_rn(centers[(int64_t)J * d + k]);
    c32[(int64_t)k * T + J] = c;
    const double a = fabs((double)c);
    if (M == EUCLIDEAN || M == SQEUCLIDEAN) nrm += a * a;
    else if (M == MANHATTAN) nrm += a;
    else nrm = fmax(nrm, a);
  }
  if (M == EUCLIDEAN || M == SQEUCLIDEAN) nrm = sqrt(nrm);
  cn[J] = float_up(nrm * (1.0 + 1e-12));
  r32[J] = float_up(radius[J]);
}

// metric distance of two fp32 centres (SoA), fp32 arithmetic
template <int M>
__device__ __forceinline__ float cdist32(const float* __restrict__ c32, int T, const float* ci, int J,
                                         int d) {
  float acc = 0.f;
  for (int k = 0; k < d; ++k) {
    const float t = fabsf(ci[k] - __ldg(c32 + (int64_t)k * T + J));
    if (M == EUCLIDEAN || M == SQEUCLIDEAN) acc = fmaf(t, t, acc);
    else if (M == MANHATTAN) acc += t;
    else acc = fmaxf(acc, t);
  }
  return (M == EUCLIDEAN || M == SQEUCLIDEAN) ? sqrtf(acc) : acc;
}

// as cdist32 with the row centre read strided from the SoA array (ci[k * T])
template <int M>
__device__ __forceinline__ float cdist32s(const float* __restrict__ c32, int T, const float* ci, int J,
                                          int d) {
  float acc = 0.f;
  for (int k = 0; k < d; ++k) {
    const float t = fabsf(__ldg(ci + (int64_t)k * T) - __ldg(c32 + (int64_t)k * T + J));
    if (M == EUCLIDEAN || M == SQEUCLIDEAN) acc = fmaf(t, t, acc);
    else if (M == MANHATTAN) acc += t;
    else acc = fmaxf(acc, t);
  }
  return (M == EUCLIDEAN || M == SQEUCLIDEAN) ? sqrtf(acc) : acc;
}

// rigorous lower bound (internal units) of every pair of tile pair (I, J) from the fp32
// centre distance: fp32 evaluation error <= (d+4)u dc, centre rounding <= u (|c_I|+|c_J|)
template <int M>
__device__ __forceinline__ double tile_lb32(float dc, float cnI, float cnJ, float rI, float rJ, int d) {
  const double u = 5.9604644775390625e-08;
  const double lo = (double)dc * (1.0 - (d + 4) * u) - 1.01 * u * ((double)cnI + (double)cnJ);
  const double r = lo * (1.0 - 1e-9) - (double)rI - (double)rJ;
  if (!(r > 0.0)) return 0.0;
  return (M == EUCLIDEAN || M == SQEUCLIDEAN) ? r * r * (1.0 - 1e-9) : r * (1.0 - 1e-9);
}

// Full-square item list for the tensor-core scan.  Item (I, J) serves the rows of tile I;
// it is keyed (I << 32 | fp32 bits of the centre distance) so that, after one radix sort,
// each row tile visits its nearest column tiles first (the diagonal tile, distance 0,
// leads) and its rows' thresholds tighten early.  With umax (phase 2) an orientation
// whose rigorous tile lower bound exceeds the row tile's component bound is dropped; the
// dropped ones and the diagonal twin become the sentinel key ~0 (sorted last, counted).
__global__ void tc_mirror_kernel(const int2* __restrict__ items, int64_t n,
                                 const double* __restrict__ umax, const float* __restrict__ c32,
                                 const float* __restrict__ cn, const float* __restrict__ r32, int T,
                                 int d, int metric, const unsigned* __restrict__ tpmin,
                                 unsigned long long* __restrict__ keys,
                                 int* __restrict__ js, unsigned long long* __restrict__ dropped) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned drop = 0;
  if (w < n) {
    const int2 it = items[w];
    bool keep_ij = true, keep_ji = it.x != it.y;
    float dc = 0.f;
    if (it.x != it.y) {
      // same fp32 centre distance and bound as enum_count_kernel (the item passed it)
      const float* ci = c32 + it.x;  // strided view: ci[k * T] is coordinate k of tile I
      double lb;
      if (metric == MANHATTAN) {
        dc = cdist32s<MANHATTAN>(c32, T, ci, it.y, d);
        lb = tile_lb32<MANHATTAN>(dc, cn[it.x], cn[it.y], r32[it.x], r32[it.y], d);
      } else if (metric == CHEBYSHEV) {
        dc = cdist32s<CHEBYSHEV>(c32, T, ci, it.y, d);
        lb = tile_lb32<CHEBYSHEV>(dc, cn[it.x], cn[it.y], r32[it.x], r32[it.y], d);
      } else {
        dc = cdist32s<EUCLIDEAN>(c32, T, ci, it.y, d);
        lb = tile_lb32<EUCLIDEAN>(dc, cn[it.x], cn[it.y], r32[it.x], r32[it.y], d);
      }
      if (umax) {
        if (tpmin) {  // the bound enum_count_kernel applied (items are (I <= J))
          const int lo = min(it.x, it.y), hi = max(it.x, it.y);
          const int64_t w2 = (int64_t)lo * T - (int64_t)lo * (lo - 1) / 2 + (hi - lo);
          lb = fmax(lb, (double)__uint_as_float(tpmin[w2]));
        }
        keep_ij = !(lb > umax[it.x]);  // fail-safe: a NaN bound keeps the orientation
        keep_ji = !(lb > umax[it.y]);
      }
    }
    const unsigned long long db = (unsigned long long)__float_as_uint(dc);
    // dropped orientations: (T << 32 | ~0u) sorts after every kept key and stays inside the
    // radix sort's bit range
    const unsigned long long drop_key = ((unsigned long long)T << 32) | 0xFFFFFFFFull;
    keys[2 * w] = keep_ij ? ((unsigned long long)it.x << 32 | db) : drop_key;
    js[2 * w] = it.y;
    keys[2 * w + 1] = keep_ji ? ((unsigned long long)it.y << 32 | db) : drop_key;
    js[2 * w + 1] = it.x;
    drop = (keep_ij ? 0u : 1u) + (keep_ji ? 0u : 1u);
  }
  drop = __reduce_add_sync(0xFFFFFFFFu, drop);
  if ((threadIdx.x & 31) == 0 && drop) atomicAdd(dropped, (unsigned long long)drop);
}

__global__ void tc_items_kernel(const unsigned long long* __restrict__ keys, const int* __restrict__ js,
                                int64_t n, int2* __restrict__ items) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w < n) items[w] = make_int2((int)(keys[w] >> 32), js[w]);
}

// Phase 1: for each tile I the PK tile pairs with the smallest LB among tiles
// that can hold a cross-component pair with I (every pair of I x J in one
// component is useless).  Seeds the component upper bounds.
constexpr int PK = 8;
// Tile-level passes handle TR row tiles per block: every column-tile centre is read once
// and compared with the TR row centres (same fp32 operation order as cdist32).
constexpr int TR = 8;

template <int M>
__device__ __forceinline__ void cdist32_rows(const float* __restrict__ c32, int T,
                                             const float (*ci)[192], int J, int d,
                                             float (&out)[TR]) {
  float acc[TR];
#pragma unroll
  for (int r = 0; r < TR; ++r) acc[r] = 0.f;
  for (int k = 0; k < d; ++k) {
    const float cj = __ldg(c32 + (int64_t)k * T + J);
#pragma unroll
    for (int r = 0; r < TR; ++r) {
      const float t = fabsf(ci[r][k] - cj);
      if (M == EUCLIDEAN || M == SQEUCLIDEAN) acc[r] = fmaf(t, t, acc[r]);
      else if (M == MANHATTAN) acc[r] += t;
      else acc[r] = fmaxf(acc[r], t);
    }
  }
#pragma unroll
  for (int r = 0; r < TR; ++r) out[r] = (M == EUCLIDEAN || M == SQEUCLIDEAN) ? sqrtf(acc[r]) : acc[r];
}

template <int M>
__global__ void phase1_kernel(const float* __restrict__ c32, const float* __restrict__ r32,
                              const int2* __restrict__ trange, int T, int d, int2* __restrict__ out) {
  const int I0 = blockIdx.x * TR;
  const int nr = min(TR, T - I0);
  __shared__ __align__(16) float ci[TR][192];
  for (int t = threadIdx.x; t < TR * d; t += blockDim.x) {
    const int r = t / d, k = t % d;
    ci[r][k] = r < nr ? c32[(int64_t)k * T + I0 + r] : 0.f;
  }
  __syncthreads();
  double bl[TR][2];
  int bj[TR][2];
#pragma unroll
  for (int r = 0; r < TR; ++r) {
    bl[r][0] = bl[r][1] = INFINITY;
    bj[r][0] = bj[r][1] = -1;
  }
  for (int J = threadIdx.x; J < T; J += blockDim.x) {
    float dc[TR];
    cdist32_rows<M>(c32, T, ci, J, d, dc);
    const float rJ = r32[J];
#pragma unroll
    for (int r = 0; r < TR; ++r) {
      const int I = I0 + r;
      if (r >= nr || same_single(trange, I, J)) continue;
      // rank by distance from I's centre to J's ball (the tile itself first): the
      // LB alone ties at 0 for every overlapping ball.  J's radius counts at most as
      // much as I's own, so a wide tile (pieces of several clusters) cannot crowd the
      // compact neighbours out of the PK slots.  A heuristic seed order (any choice
      // is sound): fp32, deterministic (ties by J)
      const double lb = (J == I) ? -INFINITY : (double)(dc[r] - fminf(rJ, r32[I]));
      if (lb < bl[r][1] || (lb == bl[r][1] && J < bj[r][1])) {
        if (lb < bl[r][0] || (lb == bl[r][0] && J < bj[r][0])) {
          bl[r][1] = bl[r][0]; bj[r][1] = bj[r][0]; bl[r][0] = lb; bj[r][0] = J;
        } else {
          bl[r][1] = lb; bj[r][1] = J;
        }
      }
    }
  }
  __shared__ double sl[512];
  __shared__ int sj[512];
  __shared__ double rl[8];
  __shared__ int ri[8];
#pragma unroll
  for (int r = 0; r < TR; ++r) {
    if (r >= nr) break;  // uniform per block
    const int I = I0 + r;
    sl[2 * threadIdx.x] = bl[r][0]; sj[2 * threadIdx.x] = bj[r][0];
    sl[2 * threadIdx.x + 1] = bl[r][1]; sj[2 * threadIdx.x + 1] = bj[r][1];
    __syncthreads();
    // PK rounds of block arg-min over the 512 candidates (tiny)
    for (int k = 0; k < PK; ++k) {
      double v = INFINITY;
      int at = -1;
      for (int c = threadIdx.x; c < 2 * blockDim.x; c += blockDim.x) {
        if (sj[c] >= 0 && (sl[c] < v || (sl[c] == v && (at < 0 || sj[c] < sj[at])))) {
          v = sl[c];
          at = c;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(0xFFFFFFFFu, v, o);
        int oa = __shfl_xor_sync(0xFFFFFFFFu, at, o);
        if (oa >= 0 && (at < 0 || ov < v || (ov == v && sj[oa] < sj[at]))) {
          v = ov;
          at = oa;
        }
      }
      if ((threadIdx.x & 31) == 0) {
        rl[threadIdx.x >> 5] = v;
        ri[threadIdx.x >> 5] = at;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        double bv = INFINITY;
        int ba = -1;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
          if (ri[w] >= 0 && (ba < 0 || rl[w] < bv || (rl[w] == bv && sj[ri[w]] < sj[ba]))) {
            bv = rl[w];
            ba = ri[w];
          }
        int2 it = make_int2(-1, -1);
        if (ba >= 0) {
          int J = sj[ba];
          it = make_int2(min(I, J), max(I, J));
          sj[ba] = -1;  // remove
        }
        out[(int64_t)I * PK + k] = it;
      }
      __syncthreads();
    }
  }
}

// Phase 1, register form (d <= 32): one thread per row tile I and one of P1_CHUNKS
// slices of the column tiles, I's centre in registers, column centres staged in shared
// memory (broadcast reads); each thread keeps its slice's PK best (rank, J) in registers
// (ties: smaller J), then phase1_merge_kernel takes the PK best of the slices.  Same
// ranking as phase1_kernel; the selection is a heuristic seed set (any choice is sound).
constexpr int P1_CHUNKS = 7;  // 138 x 7 blocks of 128: one wave on 148 SMs at 2M points
constexpr int P1_ROWS = 128;
constexpr int P1_JT = 64;

template <int M, int D>
__global__ void __launch_bounds__(P1_ROWS) phase1_reg_kernel(const float* __restrict__ c32,
                                                             const float* __restrict__ r32,
                                                             const int2* __restrict__ trange, int T,
                                                             float* __restrict__ cand_l,
                                                             int* __restrict__ cand_j) {
  constexpr int d = D;  // compile-time: straight-line distance code
  const int I = blockIdx.x * P1_ROWS + threadIdx.x;
  const int chunk = blockIdx.y;
  const int per = (T + P1_CHUNKS - 1) / P1_CHUNKS;
  const int J0 = chunk * per, J1 = min(T, J0 + per);
  __shared__ float sc[P1_JT][D + 1];
  __shared__ float sr[P1_JT];
  __shared__ int2 st[P1_JT];
  const bool live = I < T;
  float ci[D];
#pragma unroll
  for (int k = 0; k < D; ++k) ci[k] = live ? __ldg(c32 + (int64_t)k * T + I) : 0.f;
  const float rI = live ? r32[I] : 0.f;
  const int2 trI = live ? trange[I] : make_int2(0, 1);
  const bool singleI = trI.x == trI.y;
  float bl[PK];
  int bj[PK];
#pragma unroll
  for (int k = 0; k < PK; ++k) {
    bl[k] = INFINITY;
    bj[k] = -1;
  }
  for (int Jb = J0; Jb < J1; Jb += P1_JT) {
    const int nj = min(P1_JT, J1 - Jb);
    __syncthreads();
    for (int t = threadIdx.x; t < P1_JT * D; t += P1_ROWS) {
      const int k = t / P1_JT, j = t % P1_JT;
      sc[j][k] = j < nj ? __ldg(c32 + (int64_t)k * T + Jb + j) : 0.f;
    }
    if (threadIdx.x < P1_JT && threadIdx.x < nj) {
      sr[threadIdx.x] = r32[Jb + threadIdx.x];
      st[threadIdx.x] = trange[Jb + threadIdx.x];
    }
    __syncthreads();
    if (!live) continue;
    for (int j = 0; j < nj; ++j) {
      const int J = Jb + j;
      const int2 tJ = st[j];
      if (singleI && tJ.x == tJ.y && tJ.x == trI.x) continue;  // same_single(I, J)
      float acc = 0.f;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const float t = fabsf(ci[k] - sc[j][k]);
        if (M == EUCLIDEAN || M == SQEUCLIDEAN) acc = fmaf(t, t, acc);
        else if (M == MANHATTAN) acc += t;
        else acc = fmaxf(acc, t);
      }
      const float dc = (M == EUCLIDEAN || M == SQEUCLIDEAN) ? sqrtf(acc) : acc;
      float v = (J == I) ? -INFINITY : dc - fminf(sr[j], rI);
      if (!(v < bl[PK - 1])) continue;
      int jj = J;
#pragma unroll
      for (int k = 0; k < PK; ++k) {
        if (v < bl[k]) {
          const float tv = bl[k];
          const int tj = bj[k];
          bl[k] = v;
          bj[k] = jj;
          v = tv;
          jj = tj;
        }
      }
    }
  }
  if (!live) return;
  const int64_t o = ((int64_t)I * P1_CHUNKS + chunk) * PK;
#pragma unroll
  for (int k = 0; k < PK; ++k) {
    cand_l[o + k] = bl[k];
    cand_j[o + k] = bj[k];
  }
}

__global__ void phase1_merge_kernel(const float* __restrict__ cand_l, const int* __restrict__ cand_j,
                                    int T, int pk, int2* __restrict__ out) {
  const int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= T) return;
  const int64_t o = (int64_t)I * P1_CHUNKS * PK;
  float bl[PK];
  int bj[PK];
#pragma unroll
  for (int k = 0; k < PK; ++k) {
    bl[k] = INFINITY;
    bj[k] = -1;
  }
  // chunks hold ascending J ranges: visiting them in order keeps ties on the smaller J
  for (int c = 0; c < P1_CHUNKS * PK; ++c) {
    int jj = cand_j[o + c];
    if (jj < 0) continue;
    float v = cand_l[o + c];
    if (!(v < bl[PK - 1])) continue;
#pragma unroll
    for (int k = 0; k < PK; ++k) {
      if (v < bl[k]) {
        const float tv = bl[k];
        const int tj = bj[k];
        bl[k] = v;
        bj[k] = jj;
        v = tv;
        jj = tj;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < PK; ++k)
    out[(int64_t)I * PK + k] = (k < pk && bj[k] >= 0) ? make_int2(min(I, bj[k]), max(I, bj[k]))
                                                      : make_int2(-1, -1);
}

__device__ __forceinline__ int64_t tri_index(int T, int I, int J) {
  return (int64_t)I * T - (int64_t)I * (I - 1) / 2 + (J - I);
}

__global__ void mark_items_kernel(const int2* __restrict__ items, int64_t cnt, int T,
                                  unsigned* __restrict__ bits) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt) return;
  int64_t w = tri_index(T, items[t].x, items[t].y);
  atomicOr(bits + (w >> 5), 1u << (w & 31));
}

// component upper bound: exact value of each row's screened-best partner
template <int M>
__global__ void ucomp_kernel(const double* __restrict__ X64, int n, int d,
                             const unsigned long long* __restrict__ B1, const int* __restrict__ comp,
                             double thr, unsigned long long* U) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned long long k = B1[i];
  if (!key_valid(k)) return;
  int j = (int)key_index(k);
  double e = exact_dist<M>(X64 + (int64_t)i * d, X64 + (int64_t)j * d, d);
  if (e <= thr) atomicMin(U + comp[i], dbits(e));
}

__global__ void tile_umax_kernel(const int* __restrict__ comp, int64_t n,
                                 const unsigned long long* __restrict__ U, double thr,
                                 double* __restrict__ umax) {
  const int T0 = blockIdx.x;
  int64_t i = (int64_t)T0 * TILE + threadIdx.x;
  double v = -INFINITY;
  if (i < n && comp[i] >= 0) {
    unsigned long long u = U[comp[i]];
    v = (u == NONE_KEY) ? thr : fmin(bitsd(u), thr);
  }
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
  __shared__ double s[4];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) umax[T0] = fmax(fmax(s[0], s[1]), fmax(s[2], s[3]));
}

// Phase 2 enumeration, pass 1: keep flags + per-row-tile counts.
template <int M>
__global__ void enum_count_kernel(const float* __restrict__ c32, const float* __restrict__ cn,
                                  const float* __restrict__ r32,
                                  const int2* __restrict__ trange, const double* __restrict__ umax,
                                  const unsigned* __restrict__ bits, int T, int d,
                                  const unsigned* __restrict__ tpmin,
                                  unsigned char* __restrict__ keep, int* __restrict__ counts) {
  const int I0 = blockIdx.x * TR;
  const int nr = min(TR, T - I0);
  __shared__ __align__(16) float ci[TR][192];
  for (int t = threadIdx.x; t < TR * d; t += blockDim.x) {
    const int r = t / d, k = t % d;
    ci[r][k] = r < nr ? c32[(int64_t)k * T + I0 + r] : 0.f;
  }
  // per-row-tile constants (read once per block, broadcast from shared memory)
  __shared__ float rcn[TR], rr[TR];
  __shared__ double ru[TR];
  __shared__ int2 rtr[TR];
  if (threadIdx.x < TR) {
    const int r = threadIdx.x;
    rcn[r] = r < nr ? cn[I0 + r] : 0.f;
    rr[r] = r < nr ? r32[I0 + r] : 0.f;
    ru[r] = r < nr ? umax[I0 + r] : 0.0;
    rtr[r] = r < nr ? trange[I0 + r] : make_int2(0, 1);
  }
  __syncthreads();
  int c[TR];
#pragma unroll
  for (int r = 0; r < TR; ++r) c[r] = 0;
  for (int J = I0 + threadIdx.x; J < T; J += blockDim.x) {
    float dc[TR];
    cdist32_rows<M>(c32, T, ci, J, d, dc);
    const double uJ = umax[J];
    const float cnJ = cn[J], rJ = r32[J];
    const int2 tJ = trange[J];
#pragma unroll
    for (int r = 0; r < TR; ++r) {
      const int I = I0 + r;
      if (r >= nr || J < I) continue;
      const int64_t w = tri_index(T, I, J);
      const int2 tI = rtr[r];
      bool k = !((bits[w >> 5] >> (w & 31)) & 1u) &&
               !(tI.x == tI.y && tJ.x == tJ.y && tI.x == tJ.x);  // same_single(I, J)
      // kept iff the rigorous lower bound of the tile pair can reach either component
      // bound (a kept superset costs work, never exactness); the cached bound (a scanned
      // pair's) is read only when the geometric one passes
      if (k && J != I) {
        const double ub = fmax(ru[r], uJ);
        // fail-safe comparisons: a NaN bound keeps the tile pair (never prunes it)
        k = !(tile_lb32<M>(dc[r], rcn[r], cnJ, rr[r], rJ, d) > ub);
        if (k && tpmin) k = !((double)__uint_as_float(tpmin[w]) > ub);
      }
      keep[w] = k;
      c[r] += k;
    }
  }
  __shared__ int s[TR][8];
#pragma unroll
  for (int r = 0; r < TR; ++r) {
    int v = c[r];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if ((threadIdx.x & 31) == 0) s[r][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x < nr) {
    int t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[threadIdx.x][w];
    counts[I0 + threadIdx.x] = t;
  }
}

// pass 2: ordered compaction (items sorted by I, then J)
__global__ void enum_write_kernel(const unsigned char* __restrict__ keep,
                                  const long long* __restrict__ offsets, int T,
                                  int2* __restrict__ items) {
  const int I = blockIdx.x;
  const int64_t w0 = tri_index(T, I, I);
  long long base = offsets[I];
  __shared__ int warp_tot[8];
  for (int J0 = I; J0 < T; J0 += blockDim.x) {
    const int J = J0 + threadIdx.x;
    const int k = (J < T) ? keep[w0 + (J - I)] : 0;
    const unsigned m = __ballot_sync(0xFFFFFFFFu, k);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int before = __popc(m & ((1u << lane) - 1));
    if (lane == 0) warp_tot[wid] = __popc(m);
    __syncthreads();
    int off = 0, tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      if (w < wid) off += warp_tot[w];
      tot += warp_tot[w];
    }
    if (k) items[base + off + before] = make_int2(I, J);
    base += tot;
    __syncthreads();
  }
}

// ---- per-dataset tile-pair tables (computed once per dataset and metric) -------------
// Geometric lower bound of every tile pair (triangle index), fp32 rounded down: the
// rounds' phase-2 enumeration then streams this table (and the tile-pair cache that
// starts from it) instead of recomputing T(T+1)/2 centre distances every round.
template <int M>
__global__ void tile_glb_kernel(const float* __restrict__ c32, const float* __restrict__ cn,
                                const float* __restrict__ r32, int T, int d,
                                unsigned* __restrict__ glb) {
  const int I0 = blockIdx.x * TR;
  const int nr = min(TR, T - I0);
  __shared__ __align__(16) float ci[TR][192];
  for (int t = threadIdx.x; t < TR * d; t += blockDim.x) {
    const int r = t / d, k = t % d;
    ci[r][k] = r < nr ? c32[(int64_t)k * T + I0 + r] : 0.f;
  }
  __syncthreads();
  for (int J = I0 + threadIdx.x; J < T; J += blockDim.x) {
    float dc[TR];
    cdist32_rows<M>(c32, T, ci, J, d, dc);
    const float cnJ = cn[J], rJ = r32[J];
#pragma unroll
    for (int r = 0; r < TR; ++r) {
      const int I = I0 + r;
      if (r >= nr || J < I) continue;
      float lb = 0.f;
      if (J != I) {
        const double v = tile_lb32<M>(dc[r], cn[I], cnJ, r32[I], rJ, d);
        lb = (v > 0.0) ? float_down(v) : 0.f;  // NaN -> 0 (keeps the pair)
      }
      glb[tri_index(T, I, J)] = __float_as_uint(lb);
    }
  }
}

// Phase-2 enumeration from the tile-pair bound table (one block per row tile I; columns
// J >= I read contiguously): kept iff not a phase-1 item, not inside one component, and
// the rigorous lower bound can reach either component bound (fail-safe on NaN).
__global__ void enum_table_kernel(const unsigned* __restrict__ bnd, const int2* __restrict__ trange,
                                  const double* __restrict__ umax, const unsigned* __restrict__ bits,
                                  int T, unsigned char* __restrict__ keep, int* __restrict__ counts) {
  const int I = blockIdx.x;
  const int64_t w0 = tri_index(T, I, I);
  const int2 tI = trange[I];
  const double uI = umax[I];
  int c = 0;
  for (int J = I + threadIdx.x; J < T; J += blockDim.x) {
    const int64_t w = w0 + (J - I);
    const int2 tJ = trange[J];
    bool k = !((bits[w >> 5] >> (w & 31)) & 1u) &&
             !(tI.x == tI.y && tJ.x == tJ.y && tI.x == tJ.x);  // same_single(I, J)
    if (k && J != I) k = !((double)__uint_as_float(bnd[w]) > fmax(uI, umax[J]));
    keep[w] = k;
    c += k;
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
  __shared__ int s[32];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
    counts[I] = t;
  }
}

// Nearest tiles of every tile (phase-1 seed candidates), ranked as phase1_kernel does
// (centre distance minus min(R_I, R_J), the tile itself first; ties: smaller J) but
// without the per-round component filter: NBR_SLICE best per (tile, column slice), then
// the NBR best per tile.  Each round then picks its seeds from this list.
constexpr int NBR_SLICE = 16;
constexpr int NBR = 32;

template <int M, int D>
__global__ void __launch_bounds__(P1_ROWS) tile_knn_kernel(const float* __restrict__ c32,
                                                           const float* __restrict__ r32, int T,
                                                           float* __restrict__ cand_l,
                                                           int* __restrict__ cand_j) {
  constexpr int d = D;
  const int I = blockIdx.x * P1_ROWS + threadIdx.x;
  const int chunk = blockIdx.y;
  const int per = (T + P1_CHUNKS - 1) / P1_CHUNKS;
  const int J0 = chunk * per, J1 = min(T, J0 + per);
  __shared__ float sc[P1_JT][D + 1];
  __shared__ float sr[P1_JT];
  const bool live = I < T;
  float ci[D];
#pragma unroll
  for (int k = 0; k < D; ++k) ci[k] = live ? __ldg(c32 + (int64_t)k * T + I) : 0.f;
  const float rI = live ? r32[I] : 0.f;
  float bl[NBR_SLICE];
  int bj[NBR_SLICE];
#pragma unroll
  for (int k = 0; k < NBR_SLICE; ++k) {
    bl[k] = INFINITY;
    bj[k] = -1;
  }
  for (int Jb = J0; Jb < J1; Jb += P1_JT) {
    const int nj = min(P1_JT, J1 - Jb);
    __syncthreads();
    for (int t = threadIdx.x; t < P1_JT * D; t += P1_ROWS) {
      const int k = t / P1_JT, j = t % P1_JT;
      sc[j][k] = j < nj ? __ldg(c32 + (int64_t)k * T + Jb + j) : 0.f;
    }
    if (threadIdx.x < P1_JT && threadIdx.x < nj) sr[threadIdx.x] = r32[Jb + threadIdx.x];
    __syncthreads();
    if (!live) continue;
    for (int j = 0; j < nj; ++j) {
      const int J = Jb + j;
      float acc = 0.f;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const float t = fabsf(ci[k] - sc[j][k]);
        if (M == EUCLIDEAN || M == SQEUCLIDEAN) acc = fmaf(t, t, acc);
        else if (M == MANHATTAN) acc += t;
        else acc = fmaxf(acc, t);
      }
      const float dc = (M == EUCLIDEAN || M == SQEUCLIDEAN) ? sqrtf(acc) : acc;
      float v = (J == I) ? -INFINITY : dc - fminf(sr[j], rI);
      if (!(v < bl[NBR_SLICE - 1])) continue;
      int jj = J;
#pragma unroll
      for (int k = 0; k < NBR_SLICE; ++k) {
        if (v < bl[k]) {
          const float tv = bl[k];
          const int tj = bj[k];
          bl[k] = v;
          bj[k] = jj;
          v = tv;
          jj = tj;
        }
      }
    }
  }
  if (!live) return;
  const int64_t o = ((int64_t)I * P1_CHUNKS + chunk) * NBR_SLICE;
#pragma unroll
  for (int k = 0; k < NBR_SLICE; ++k) {
    cand_l[o + k] = bl[k];
    cand_j[o + k] = bj[k];
  }
}

__global__ void tile_knn_merge_kernel(const float* __restrict__ cand_l, const int* __restrict__ cand_j,
                                      int T, int* __restrict__ nbr) {
  const int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= T) return;
  const int64_t o = (int64_t)I * P1_CHUNKS * NBR_SLICE;
  float bl[NBR];
  int bj[NBR];
#pragma unroll
  for (int k = 0; k < NBR; ++k) {
    bl[k] = INFINITY;
    bj[k] = -1;
  }
  // chunks hold ascending J ranges: visiting them in order keeps ties on the smaller J
  for (int c = 0; c < P1_CHUNKS * NBR_SLICE; ++c) {
    int jj = cand_j[o + c];
    if (jj < 0) continue;
    float v = cand_l[o + c];
    if (!(v < bl[NBR - 1])) continue;
#pragma unroll
    for (int k = 0; k < NBR; ++k) {
      if (v < bl[k]) {
        const float tv = bl[k];
        const int tj = bj[k];
        bl[k] = v;
        bj[k] = jj;
        v = tv;
        jj = tj;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NBR; ++k) nbr[(int64_t)I * NBR + k] = bj[k];
}

// this round's seeds: the first pk tiles of I's list that can hold a cross-component pair
// with I (fewer when the list runs out: the seed set is a heuristic, any choice is sound)
__global__ void phase1_pick_kernel(const int* __restrict__ nbr, const int2* __restrict__ trange,
                                   int T, int pk, int2* __restrict__ out) {
  const int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= T) return;
  const int2 tI = trange[I];
  int c = 0;
  for (int k = 0; k < NBR && c < pk; ++k) {
    const int J = nbr[(int64_t)I * NBR + k];
    if (J < 0) break;
    const int2 tJ = trange[J];
    if (tI.x == tI.y && tJ.x == tJ.y && tI.x == tJ.x) continue;  // same_single(I, J)
    out[(int64_t)I * PK + c++] = make_int2(min(I, J), max(I, J));
  }
  for (; c < PK; ++c) out[(int64_t)I * PK + c] = make_int2(-1, -1);
}

// tile-pair cache entries of an item list <-> a compact buffer (multi-rank exchange)
__global__ void cache_gather_kernel(const int2* __restrict__ items, int64_t cnt, int T,
                                    const unsigned* __restrict__ tpmin, unsigned* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt) return;
  const int2 it = items[t];
  out[t] = tpmin[tri_index(T, min(it.x, it.y), max(it.x, it.y))];
}

__global__ void cache_scatter_kernel(const int2* __restrict__ items, int64_t cnt, int T,
                                     const unsigned* __restrict__ in, unsigned* __restrict__ tpmin) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt) return;
  const int2 it = items[t];
  tpmin[tri_index(T, min(it.x, it.y), max(it.x, it.y))] = in[t];
}

// Phase-2 enumeration from the tile-pair bound table, appending the kept tile pairs as
// u64 keys (I << 32 | J) with warp-aggregated atomics (unordered; sorted afterwards so
// that every rank derives the identical list).  Same keep rule as enum_table_kernel.
constexpr int CB = 8;  // tiles per side of a coarse bound block (coarse_min_kernel)
__global__ void enum_append_kernel(const unsigned* __restrict__ bnd, const int2* __restrict__ trange,
                                   const double* __restrict__ umax, const unsigned* __restrict__ bits,
                                   int T, unsigned long long* __restrict__ out,
                                   unsigned long long* __restrict__ count, unsigned long long cap,
                                   const unsigned* __restrict__ cmin,
                                   const double* __restrict__ bumax, int TB) {
  const int I = blockIdx.x;
  const int64_t w0 = tri_index(T, I, I);
  const int2 tI = trange[I];
  const double uI = umax[I];
  const int lane = threadIdx.x & 31;
  constexpr int U = 4;  // four independent column loads in flight per thread
  for (int J0 = I; J0 < T; J0 += U * blockDim.x) {
    bool k[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int J = J0 + u * blockDim.x + threadIdx.x;
      k[u] = false;
      // whole 8-tile blocks whose coarse bound already exceeds every component bound
      // involved are skipped without touching the table (the pair test would drop them)
      if (J < T && cmin &&
          (double)__uint_as_float(cmin[(int64_t)(I / CB) * TB + J / CB]) > fmax(uI, bumax[J / CB]))
        continue;
      if (J < T) {
        const int64_t w = w0 + (J - I);
        const int2 tJ = trange[J];
        const unsigned bw = bits[w >> 5];
        const float b = __uint_as_float(bnd[w]);
        const double uJ = umax[J];
        k[u] = !((bw >> (w & 31)) & 1u) &&
               !(tI.x == tI.y && tJ.x == tJ.y && tI.x == tJ.x);  // same_single(I, J)
        if (J != I) k[u] = k[u] && !((double)b > fmax(uI, uJ));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned m = __ballot_sync(0xFFFFFFFFu, k[u]);
      if (!m) continue;
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(count, (unsigned long long)__popc(m));
      base = __shfl_sync(0xFFFFFFFFu, base, 0);
      if (k[u]) {
        const int J = J0 + u * blockDim.x + threadIdx.x;
        const unsigned long long at = base + __popc(m & ((1u << lane) - 1u));
        if (at < cap) out[at] = ((unsigned long long)I << 32) | (unsigned)J;
      }
    }
  }
}

// Coarse bound table: per 8 x 8 block of tile pairs (I / 8, J / 8) the minimum of the
// geometric bounds (uint order of non-negative fp32 bits), built once per dataset.  The
// tile-pair cache only raises entries, so the block minimum stays a lower bound of every
// entry the enumeration reads.
__global__ void coarse_min_kernel(const unsigned* __restrict__ glb, int T, int TB,
                                  unsigned* __restrict__ cmin) {
  const int I = blockIdx.x;
  const int64_t w0 = tri_index(T, I, I);
  for (int J0 = I & ~(CB - 1); J0 < T; J0 += blockDim.x) {
    const int J = J0 + threadIdx.x;  // blockDim a multiple of CB: lane groups align with blocks
    unsigned v = (J >= I && J < T) ? glb[w0 + (J - I)] : 0xFFFFFFFFu;
#pragma unroll
    for (int o = 1; o < CB; o <<= 1) v = min(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
    if ((threadIdx.x & (CB - 1)) == 0 && J < T && v != 0xFFFFFFFFu)
      atomicMin(cmin + (int64_t)(I / CB) * TB + J / CB, v);
  }
}

// per block of CB tiles: the largest component bound (fmax: NaN ignored like the pair test)
__global__ void block_umax_kernel(const double* __restrict__ umax, int T, int TB,
                                  double* __restrict__ bumax) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= TB) return;
  double m = -INFINITY;
  for (int j = b * CB; j < min(T, (b + 1) * CB); ++j) m = fmax(m, umax[j]);
  bumax[b] = m;
}

// sorted u64 item keys (I << 32 | J) -> int2 (I, J)
__global__ void keys_to_items_kernel(const unsigned long long* __restrict__ keys, int64_t n,
                                     int2* __restrict__ items) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) items[t] = make_int2((int)(keys[t] >> 32), (int)(keys[t] & 0xFFFFFFFFull));
}

// int2 (I <= J, or (-1, -1) padding) -> u64 key (padding `pad` = (T << 32) | T: sorts last
// and keeps the key inside the radix sort's bit range)
__global__ void items_to_keys_kernel(const int2* __restrict__ items, int64_t n,
                                     unsigned long long pad, unsigned long long* __restrict__ keys) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int2 it = items[t];
  keys[t] = it.x < 0 ? pad : (((unsigned long long)it.x << 32) | (unsigned)it.y);
}

__global__ void pos_caps_kernel(int64_t n, const int* __restrict__ comp,
                                const unsigned* __restrict__ caps, unsigned* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = comp[i];
  out[i] = c >= 0 ? caps[c] : 0x7f800000u;
}

__global__ void item_pairs_kernel(const int2* __restrict__ items, int64_t cnt,
                                  const int* __restrict__ tcount, unsigned long long* acc) {
  // real point pairs covered by a list of tile pairs (for the stats)
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long v = 0;
  if (t < cnt) {
    int2 it = items[t];
    long long mI = tcount[it.x], mJ = tcount[it.y];
    v = (it.x == it.y) ? (unsigned long long)(mI * (mI - 1) / 2) : (unsigned long long)(mI * mJ);
  }
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(acc, v);
}


// ---- spatial order (kd bisection into 128-point leaves) ----------------------
// Boruvka runs on a permuted copy in which every 128-point tile is a kd leaf
// (spatially compact), so tile balls are tight and the pruning bound bites.
// Keys that decide orders always use ORIGINAL indices (orig[] / pos[]).
__device__ __forceinline__ uint32_t f2ord(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__global__ void kd_dim_kernel(const double* __restrict__ X64, int d, const int* __restrict__ order,
                              const int* __restrict__ sbeg, const int* __restrict__ ssz, int nseg,
                              int leaf_split, int* __restrict__ sdim) {
  const int sgm = blockIdx.x;
  if (sgm >= nseg) return;
  const int sz = ssz[sgm];
  if (sz <= 1 || (sz <= TILE && !leaf_split)) {
    if (threadIdx.x == 0) sdim[sgm] = -1;
    return;
  }
  const int b = sbeg[sgm];
  // sample up to 64 evenly spaced points (two per lane, rows read whole and in parallel);
  // spread per dimension
  const int ns = sz < 64 ? sz : 64;
  const int lane = threadIdx.x;
  const int t0 = lane, t1 = lane + 32;
  const double* r0 = t0 < ns ? X64 + (int64_t)order[b + (int)((long long)t0 * sz / ns)] * d : nullptr;
  const double* r1 = t1 < ns ? X64 + (int64_t)order[b + (int)((long long)t1 * sz / ns)] * d : nullptr;
  float bs = -1.f;
  int bk = 0;
  for (int k = 0; k < d; ++k) {
    float lo = INFINITY, hi = -INFINITY;
    if (r0) {
      const float v = (float)r0[k];
      lo = fminf(lo, v);
      hi = fmaxf(hi, v);
    }
    if (r1) {
      const float v = (float)r1[k];
      lo = fminf(lo, v);
      hi = fmaxf(hi, v);
    }
    for (int o = 16; o > 0; o >>= 1) {
      lo = fminf(lo, __shfl_xor_sync(0xFFFFFFFFu, lo, o));
      hi = fmaxf(hi, __shfl_xor_sync(0xFFFFFFFFu, hi, o));
    }
    if (hi - lo > bs) {  // lane-uniform after the reduction
      bs = hi - lo;
      bk = k;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    float os = __shfl_xor_sync(0xFFFFFFFFu, bs, o);
    int ok = __shfl_xor_sync(0xFFFFFFFFu, bk, o);
    if (os > bs || (os == bs && ok < bk)) {
      bs = os;
      bk = ok;
    }
  }
  if (threadIdx.x == 0) sdim[sgm] = bk;
}

__global__ void kd_key_kernel(const double* __restrict__ X64, int64_t n, int d,
                              const int* __restrict__ order, const int* __restrict__ segid,
                              const int* __restrict__ sdim, unsigned long long* __restrict__ keys) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int sgm = segid[p];
  const int k = sdim[sgm];
  const uint32_t v = k >= 0 ? f2ord((float)X64[(int64_t)order[p] * d + k]) : 0u;
  keys[p] = ((unsigned long long)(uint32_t)sgm << 32) | v;
}

// split position of each segment (sorted by the split coordinate): the largest
// gap in the middle half if it is a real gap (>= 10% of the extent), else the
// multiple of 128 nearest the median.  Segments <= TILE are leaves.
constexpr int KD_SPLIT_THREADS = 256;
__global__ void __launch_bounds__(KD_SPLIT_THREADS) kd_splitpos_kernel(const unsigned long long* __restrict__ keys,
                                   const int* __restrict__ sbeg, const int* __restrict__ ssz,
                                   int nseg, int allow_off, int* __restrict__ ssplit,
                                   int small_only) {
  const int sgm = blockIdx.x;
  if (sgm >= nseg) return;
  const int sz = ssz[sgm], b = sbeg[sgm];
  if (small_only && sz > TILE) return;  // decided by kd_gap_split_kernel
  if (sz <= 1 || (sz <= TILE && !allow_off)) {
    if (threadIdx.x == 0) ssplit[sgm] = sz;
    return;
  }
  auto val = [&](int i) {
    uint32_t u = (uint32_t)(keys[b + i] & 0xFFFFFFFFull);
    u = (u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u;
    return __uint_as_float(u);
  };
  const int lo = sz / 4, hi = sz - sz / 4;  // balanced cuts: left size in [lo, hi]
  float bg = -1.f, bg2 = -1.f;              // largest gap: balanced range / anywhere
  int bp = sz / 2, bp2 = sz / 2;
  for (int i = 1 + threadIdx.x; i < sz; i += blockDim.x) {
    const float g = val(i) - val(i - 1);
    if (i >= lo && i <= hi && (g > bg || (g == bg && i < bp))) {
      bg = g;
      bp = i;
    }
    if (g > bg2 || (g == bg2 && i < bp2)) {
      bg2 = g;
      bp2 = i;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    float og = __shfl_xor_sync(0xFFFFFFFFu, bg, o);
    int op = __shfl_xor_sync(0xFFFFFFFFu, bp, o);
    if (og > bg || (og == bg && op < bp)) {
      bg = og;
      bp = op;
    }
    og = __shfl_xor_sync(0xFFFFFFFFu, bg2, o);
    op = __shfl_xor_sync(0xFFFFFFFFu, bp2, o);
    if (og > bg2 || (og == bg2 && op < bp2)) {
      bg2 = og;
      bp2 = op;
    }
  }
  // across the block's warps (a top-level segment holds all n points)
  __shared__ float wg[KD_SPLIT_THREADS / 32], wg2[KD_SPLIT_THREADS / 32];
  __shared__ int wp[KD_SPLIT_THREADS / 32], wp2[KD_SPLIT_THREADS / 32];
  if ((threadIdx.x & 31) == 0) {
    wg[threadIdx.x >> 5] = bg;
    wp[threadIdx.x >> 5] = bp;
    wg2[threadIdx.x >> 5] = bg2;
    wp2[threadIdx.x >> 5] = bp2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      if (wg[w] > bg || (wg[w] == bg && wp[w] < bp)) {
        bg = wg[w];
        bp = wp[w];
      }
      if (wg2[w] > bg2 || (wg2[w] == bg2 && wp2[w] < bp2)) {
        bg2 = wg2[w];
        bp2 = wp2[w];
      }
    }
    const float ext = val(sz - 1) - val(0);
    if (sz <= TILE) {
      // a leaf that holds two separated groups (a piece of a neighbouring cluster) is
      // split at the gap: one ball per group keeps the tile bounds tight
      ssplit[sgm] = (sz >= 16 && ext > 0.f && bg2 >= 0.5f * ext) ? bp2 : sz;
      return;
    }
    // no real gap: cut at the multiple of 128 nearest the median, so compact
    // clusters fill whole tiles (few pad slots)
    int L = ((sz + TILE) / (2 * TILE)) * TILE;
    if (L < TILE) L = TILE;
    if (L > sz - 1) L = sz - 1;
    if (ext > 0.f && bg >= 0.1f * ext) L = bp;
    else if (allow_off && ext > 0.f && bg2 >= 0.25f * ext) L = bp2;  // cut a separated piece off
    ssplit[sgm] = L;
  }
}

// Split search for the big top-level segments (few segments, millions of points): a
// grid over the sorted positions computes every gap and reduces the two arg-max gaps
// per segment (balanced range / anywhere; ties: smaller index) with packed 64-bit
// atomicMax (gap bits << 32 | ~index), pre-reduced per block when the block lies inside
// one segment; kd_gap_split_kernel then applies kd_splitpos_kernel's decision rule.
__device__ __forceinline__ float kd_val(const unsigned long long* keys, int64_t p) {
  uint32_t u = (uint32_t)(keys[p] & 0xFFFFFFFFull);
  u = (u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u;
  return __uint_as_float(u);
}

__global__ void kd_gap_kernel(const unsigned long long* __restrict__ keys, int64_t n,
                              const int* __restrict__ segid, const int* __restrict__ sbeg,
                              const int* __restrict__ ssz, unsigned long long* __restrict__ gbest) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long bal = 0, any = 0;
  int sgm = -1;
  if (p < n) {
    sgm = segid[p];
    const int b = sbeg[sgm], sz = ssz[sgm], i = (int)(p - b);
    if (sz > TILE && i >= 1) {
      const float g = kd_val(keys, p) - kd_val(keys, p - 1);
      const unsigned long long pk = ((unsigned long long)__float_as_uint(fmaxf(g, 0.f)) << 32) |
                                    (unsigned)(~(unsigned)i);
      any = pk;
      if (i >= sz / 4 && i <= sz - sz / 4) bal = pk;
    }
  }
  const int s0 = __shfl_sync(0xFFFFFFFFu, sgm, 0);
  const bool uniform = __all_sync(0xFFFFFFFFu, sgm == s0);
  if (uniform) {  // warp inside one segment: reduce first
    for (int o = 16; o > 0; o >>= 1) {
      bal = max(bal, __shfl_xor_sync(0xFFFFFFFFu, bal, o));
      any = max(any, __shfl_xor_sync(0xFFFFFFFFu, any, o));
    }
    if ((threadIdx.x & 31) == 0 && s0 >= 0) {
      if (bal) atomicMax(gbest + 2 * s0, bal);
      if (any) atomicMax(gbest + 2 * s0 + 1, any);
    }
  } else if (sgm >= 0) {
    if (bal) atomicMax(gbest + 2 * sgm, bal);
    if (any) atomicMax(gbest + 2 * sgm + 1, any);
  }
}

__global__ void kd_gap_split_kernel(const unsigned long long* __restrict__ keys,
                                    const int* __restrict__ sbeg, const int* __restrict__ ssz,
                                    int nseg, int allow_off,
                                    const unsigned long long* __restrict__ gbest,
                                    int* __restrict__ ssplit) {
  const int sgm = blockIdx.x * blockDim.x + threadIdx.x;
  if (sgm >= nseg) return;
  const int sz = ssz[sgm], b = sbeg[sgm];
  if (sz <= TILE) {  // small segments: kd_splitpos_kernel (never reached: routed there)
    ssplit[sgm] = sz;
    return;
  }
  const unsigned long long gb = gbest[2 * sgm], ga = gbest[2 * sgm + 1];
  const float bg = gb ? __uint_as_float((unsigned)(gb >> 32)) : -1.f;
  const int bp = gb ? (int)(~(unsigned)(gb & 0xFFFFFFFFull)) : sz / 2;
  const float bg2 = ga ? __uint_as_float((unsigned)(ga >> 32)) : -1.f;
  const int bp2 = ga ? (int)(~(unsigned)(ga & 0xFFFFFFFFull)) : sz / 2;
  const float ext = kd_val(keys, b + sz - 1) - kd_val(keys, b);
  int L = ((sz + TILE) / (2 * TILE)) * TILE;
  if (L < TILE) L = TILE;
  if (L > sz - 1) L = sz - 1;
  if (ext > 0.f && bg >= 0.1f * ext) L = bp;
  else if (allow_off && ext > 0.f && bg2 >= 0.25f * ext) L = bp2;  // cut a separated piece off
  ssplit[sgm] = L;
}

__global__ void kd_children_kernel(int nseg, const int* __restrict__ ssz,
                                   const int* __restrict__ ssplit, int* __restrict__ nchild) {
  int sgm = blockIdx.x * blockDim.x + threadIdx.x;
  if (sgm < nseg) nchild[sgm] = ssplit[sgm] < ssz[sgm] ? 2 : 1;
}

__global__ void kd_newsegs_kernel(int nseg, const int* __restrict__ sbeg, const int* __restrict__ ssz,
                                  const int* __restrict__ ssplit, const int* __restrict__ cbase,
                                  int* __restrict__ nbeg, int* __restrict__ nsz) {
  int sgm = blockIdx.x * blockDim.x + threadIdx.x;
  if (sgm >= nseg) return;
  const int c = cbase[sgm], sz = ssz[sgm], L = ssplit[sgm];
  nbeg[c] = sbeg[sgm];
  nsz[c] = L;
  if (L < sz) {
    nbeg[c + 1] = sbeg[sgm] + L;
    nsz[c + 1] = sz - L;
  }
}

__global__ void kd_relabel_kernel(int64_t n, const int* __restrict__ sbeg, const int* __restrict__ ssz,
                                  const int* __restrict__ ssplit, const int* __restrict__ cbase,
                                  int* __restrict__ segid) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int sgm = segid[p];
  segid[p] = cbase[sgm] + ((ssplit[sgm] < ssz[sgm] && (int)(p - sbeg[sgm]) >= ssplit[sgm]) ? 1 : 0);
}

// compact order -> padded positions: leaf k occupies tile k
__global__ void kd_place_kernel(int64_t n, const int* __restrict__ order, const int* __restrict__ segid,
                                const int* __restrict__ sbeg, int* __restrict__ porig,
                                int* __restrict__ ppos) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const int sgm = segid[c];
  const int64_t p = (int64_t)sgm * TILE + (c - sbeg[sgm]);
  porig[p] = order[c];
  ppos[order[c]] = (int)p;
}

__global__ void fill_int_kernel(int* a, int64_t n, int v) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = v;
}

__global__ void tile_count_kernel(const int* __restrict__ porig, int T, int* __restrict__ tcount) {
  const int t = blockIdx.x;
  int c = porig[(int64_t)t * TILE + threadIdx.x] >= 0;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
  __shared__ int s[4];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) tcount[t] = s[0] + s[1] + s[2] + s[3];
}

__global__ void fill_comp_view_kernel(const int* __restrict__ porig, int64_t np, int* __restrict__ comp) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < np) comp[p] = porig[p] >= 0 ? (int)p : -1;
}

__global__ void gather_rows_kernel(const double* __restrict__ X64, int64_t n, int d,
                                   const int* __restrict__ order, double* __restrict__ out) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * d) return;
  int64_t p = t / d, k = t % d;
  out[t] = order[p] >= 0 ? X64[(int64_t)order[p] * d + k] : 0.0;
}

__global__ void inverse_perm_kernel(int64_t n, const int* __restrict__ order, int* __restrict__ pos) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n && order[p] >= 0) pos[order[p]] = (int)p;
}

__global__ void gather_norm_kernel(int64_t n, const int* __restrict__ order,
                                   const double* __restrict__ norm, double* __restrict__ out) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) out[p] = order[p] >= 0 ? norm[order[p]] : 0.0;
}

// ---- round path -----------------------------------------------------------
struct Cand {
  double d;
  int a, b;
};
struct CandLess {
  __host__ __device__ bool operator()(const Cand& x, const Cand& y) const {
    if (x.d != y.d) return x.d < y.d;
    if (x.a != y.a) return x.a < y.a;
    return x.b < y.b;
  }
};

// distinct row-best pairs with exact keys (an upper bound for the P-th key)
template <int M>
__global__ void rowpairs_kernel(const double* __restrict__ X64, int n, int d,
                                const unsigned long long* __restrict__ B1, double thr, Cand* out,
                                unsigned long long* count, const int* __restrict__ comp,
                                const int* __restrict__ psize, int ksum) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned long long k = B1[i];
  if (!key_valid(k)) return;
  int j = (int)key_index(k);
  // B1 may come from an earlier snapshot (round-path reuse): keep the pair only if it is
  // still eligible (eligibility only shrinks as clusters merge and grow)
  if (comp[i] == comp[j]) return;
  if (ksum != INT_UNSET && psize[i] + psize[j] > ksum) return;
  if (!(i < j)) {
    unsigned long long kj = B1[j];
    if (key_valid(kj) && (int)key_index(kj) == i) return;  // emitted by row j
  }
  double e = exact_dist<M>(X64 + (int64_t)i * d, X64 + (int64_t)j * d, d);
  if (!(e <= thr)) return;
  unsigned long long pos = atomicAdd(count, 1ull);
  Cand c;
  c.d = e;
  c.a = min(i, j);
  c.b = max(i, j);
  out[pos] = c;
}

__global__ void active_rows_kernel(int n, const unsigned long long* __restrict__ B1,
                                   const double* __restrict__ norm, double maxnorm, ErrModel em,
                                   double tau, int* out, unsigned long long* count) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned long long k = B1[i];
  if (!key_valid(k)) return;
  if (exact_lower(em, (double)key_value(k), norm[i] + maxnorm) <= tau) {
    unsigned long long pos = atomicAdd(count, 1ull);
    out[pos] = i;
  }
}

// candidate distances rounded UP to fp32 (a monotone map: the P-th smallest of these is
// an upper bound of the P-th smallest distance) as radix-sortable keys
__global__ void cand_keys_kernel(const Cand* __restrict__ c, int64_t n, float* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) out[t] = float_up(c[t].d);
}

__global__ void pairs_to_cands_kernel(const int2* __restrict__ pairs, const double* __restrict__ dv,
                                      int64_t count, double lim, Cand* out,
                                      unsigned long long* n_out) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  if (!(dv[t] <= lim)) return;
  unsigned long long pos = atomicAdd(n_out, 1ull);
  Cand c;
  c.d = dv[t];
  c.a = pairs[t].x;
  c.b = pairs[t].y;
  out[pos] = c;
}

__global__ void snapshot_update_kernel(int n, int* comp, int* psize, const int* __restrict__ rmap,
                                       const int* __restrict__ rsize) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int c = rmap[comp[i]];
  comp[i] = c;
  psize[i] = rsize[c];
}

__global__ void scatter_kernel(const int2* __restrict__ kv, int cnt, int* arr) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < cnt) arr[kv[t].x] = kv[t].y;
}

// effective sizes for the fused kl2 / kl3 rule: size > kl2 -> SIZE_BIG, so that
// (sa <= kl2 && sb <= kl2 && sa + sb <= kl3)  <=>  eff_a + eff_b <= ksum (pairgen.py:169-187)
__global__ void eff_size_kernel(const int* __restrict__ psize, int64_t ld, int kl2,
                                int* __restrict__ eff) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ld) return;
  int s = psize[i];
  eff[i] = (kl2 != INT_UNSET && s > kl2) ? SIZE_BIG : s;
}

// per-tile [min, max] component label of the tile's real points
__global__ void tile_range_kernel(const int* __restrict__ comp, int64_t n, int T, int2* out) {
  int t = blockIdx.x;
  int lo = 0x7FFFFFFF, hi = -0x7FFFFFFF;
  int64_t i = (int64_t)t * TILE + threadIdx.x;
  if (i < n && comp[i] >= 0) {  // pads carry comp -1
    lo = comp[i];
    hi = lo;
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xFFFFFFFFu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xFFFFFFFFu, hi, o));
  }
  __shared__ int slo[4], shi[4];
  if ((threadIdx.x & 31) == 0) {
    slo[threadIdx.x >> 5] = lo;
    shi[threadIdx.x >> 5] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 4; ++w) {
      lo = min(lo, slo[w]);
      hi = max(hi, shi[w]);
    }
    out[t] = make_int2(lo, hi);
  }
}

__global__ void fill_u32_kernel(unsigned* p, int64_t n, unsigned v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

__global__ void fill_u64_kernel(unsigned long long* p, int64_t n, unsigned long long v) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

__global__ void iota_kernel(int* a, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = i;
}

__global__ void ones_kernel(int* a, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = 1;
}

}  // namespace nnm


// Caching allocator for thrust temporaries: thrust would cudaMalloc / cudaFree
// per call (cudaFree synchronises the device); blocks are reused per dataset.
struct CachedAlloc {
  typedef char value_type;
  std::multimap<size_t, char*> free_blocks;
  std::map<char*, size_t> used;
  char* allocate(std::ptrdiff_t n) {
    auto it = free_blocks.lower_bound((size_t)n);
    if (it != free_blocks.end() && it->first <= 2 * (size_t)n + (1 << 20)) {
      char* p = it->second;
      used[p] = it->first;
      free_blocks.erase(it);
      return p;
    }
    // from the stream-ordered pool (release threshold raised): a new dataset reuses
    // the pool's pages instead of cudaMalloc / device-synchronising cudaFree
    char* p = nullptr;
    s = t_alloc_stream;
    CUDA_TRY(cudaMallocAsync((void**)&p, (size_t)n, s));
    used[p] = (size_t)n;
    return p;
  }
  void deallocate(char* p, size_t) {
    auto it = used.find(p);
    free_blocks.emplace(it->second, p);
    used.erase(it);
  }
  cudaStream_t s = nullptr;
  void release() {
    for (auto& kv : free_blocks) cudaFreeAsync(kv.second, s);
    for (auto& kv : used) cudaFreeAsync(kv.first, s);
    free_blocks.clear();
    used.clear();
  }
};

// ----------------------------------------------------------------------------
// dataset handle
// ----------------------------------------------------------------------------
struct StreamHolder {
  cudaStream_t st = nullptr;
  ~StreamHolder() {
    // the members' cudaFreeAsync calls are queued on st by now: let them complete so
    // the pool can hand the pages straight to the next dataset (no pool growth)
    if (st) {
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    }
  }
};

struct nnm_dataset {
  StreamHolder stream_holder;  // declared first: destroyed after every DevBuf member
  std::mutex mu;
  int device = 0;
  int64_t n = 0;
  int d = 0;
  int64_t ld = 0;  // n_pad
  int T = 0;
  int sms = 148;
  cudaStream_t st = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;
  cudaStream_t st2 = nullptr;  // side stream for device-to-host copies that overlap kernels

  DevBuf<double> X64;
  DevBuf<float> X32;
  int norm_metric = -1;
  DevBuf<double> norm;
  double maxnorm = 0.0;
  DevBuf<unsigned long long> scratch_u64;

  DevBuf<int> comp, psize, psize_eff;
  DevBuf<int2> tile_range;
  DevBuf<unsigned long long> B1, B2;
  // boruvka
  int bv_metric = 0;
  double bv_thr = INFINITY;
  float bv_thr_hi = INFINITY;
  ErrModel em{};
  int bv_round = 0;
  int64_t bv_ncomp = 0;
  DevBuf<unsigned long long> rb_d;
  DevBuf<int> rb_j;
  DevBuf<double> rowlow;
  DevBuf<int> amb, resc, parent;
  DevBuf<float> resc_bound, gathered;
  DevBuf<unsigned long long> cmin_d, cmin_ab, counters;
  DevBuf<Edge> edges;
  DevBuf<ReplayEdge> replay;
  PinnedBuf<ReplayEdge> host_replay;
  PinnedBuf<int32_t> h_rk, h_rd, h_rs, h_as;
  DevBuf<int> r_par, r_sz, r_lab, r_head, r_ea, r_eb, r_nxt, r_comp, r_ctl, r_rk, r_rd, r_rs,
      r_base, r_slot, r_rid, r_rcnt, r_llist;
  cudaGraphExec_t rp_exec = nullptr, rp_exec2 = nullptr;  // captured replay chunks (bv_end)
  int64_t rp_split = 0;  // first chunk of the second graph
  int64_t rp_m = -1, rp_n = -1, rp_nch = -1;
  int rp_lmax = -1;
  const void* rp_e = nullptr;
  ReplayState rp_state{};
  // host replay scratch (reused across runs; faulted in during the GPU rounds by nnm_run)
  DevBuf<float> sm_v1, sm_v2;      // small_screened_kernel partials
  DevBuf<int> sm_j1, sm_need;
  DevBuf<float2> sm_dup;
  PinnedBuf<int32_t> rp_par, rp_sz;
  PinnedBuf<int2> rp_links;        // host tail links (dropped -> kept) for the GPU labels
  DevBuf<nnm_merge> rec_dev;       // merge records staged for page-locked output
  DevBuf<int64_t> as_dev;          // labels staged for page-locked output
  DevBuf<int2> links_dev;
  void replay_host_buffers() {
    rp_par.ensure(std::max<int64_t>(n, 1));
    rp_sz.ensure(std::max<int64_t>(n, 1));
  }
  DevBuf<int2> pairs;
  DevBuf<double> pair_d;
  DevBuf<int> flag;
  // Boruvka view: kd-ordered copy (positions p; orig[p] = original index)
  bool have_order = false;
  DevBuf<int> porig, ppos;
  DevBuf<double> X64p, normp;
  DevBuf<float> X32p;
  double maxnormp = 0.0;
  int normp_metric = -1;
  int64_t np_ = 0;                  // positions of the Boruvka view (tiles x 128, pads included)
  int Tp = 0;
  DevBuf<int> tcount_p, tcount_o;   // real points per tile (Boruvka view / original)
  // current view used by the shared helpers (scan / collect / exact_pairs)
  const float* cur_X32 = nullptr;
  const double* cur_X64 = nullptr;
  int64_t vn = 0, vld = 0;
  int vT = 0;
  const int* cur_tcount = nullptr;
  // tensor-core scan (Euclidean Boruvka, d <= TC_MAX_D; nnm_tc.cu)
  bool tc_on = false;
  bool tc_ready = false;
  DevBuf<float> tc_img, tc_tnorm, tc_eta, tc_meta, tc_sq;
  DevBuf<int2> tc_items;
  DevBuf<unsigned long long> tc_keys, tc_keys2;  // (I << 32 | centre-distance bits), sorted
  DevBuf<int> tc_js, tc_js2;
  // dot form
  bool dot_on = false;
  DotModel dm{};
  DevBuf<float> tcenter32, dotB, dotNBK, dotBmax;
  // pruning
  int geom_metric = -1;
  DevBuf<double> tcenter, tradius, tumax;
  DevBuf<float> tc32, tcn32, tr32;  // fp32 SoA tile centres / norms / radii (tile passes)
  DevBuf<int2> items1, items2;
  DevBuf<float> p1_l;  // phase-1 per-slice candidates (phase1_reg_kernel)
  DevBuf<int> p1_j;
  // per-dataset tile-pair tables (geom_metric): geometric lower bound per tile pair and
  // the NBR nearest tiles of every tile (phase-1 seed candidates)
  DevBuf<unsigned> glb;
  DevBuf<unsigned> cmin;   // coarse block minima of glb (coarse_min_kernel)
  DevBuf<double> bumax;    // per-round block maxima of the tile bounds
  bool coarse_on = false;
  int tb_ = 0;
  DevBuf<int> nbr;
  int glb_metric = -1, nbr_metric = -1;
  // per tile pair (triangle index): fp32 bits of a lower bound of S over its cross-component
  // pairs, written by the tensor-core scan, read by the phase-2 enumeration (0: unknown)
  DevBuf<unsigned> tpmin;
  // component caps (TC scan): bound pass over the phase-1 items, then capped exact scans
  DevBuf<unsigned> ucap;        // this rank's caps from its bound-pass share (u32 fp32 bits)
  DevBuf<unsigned> capp;        // per position: its component's cap (staged by the scan)
  DevBuf<int> tc_slots;         // [Tp][16] per-round slot records (tc_tails)
  DevBuf<unsigned long long> tc_cand;  // deferred exact-key candidates (tc_launch)
  bool tc_phase2 = false;              // the current tc_scan is a phase-2 pass
  int64_t tc_tails_epoch = -1;  // scan_epoch the A tails / slot records were written for

  // A-side tails of the operand image and the slot records for the current components
  void tc_tails() {
    if (tc_tails_epoch == scan_epoch && tc_slots.p) return;
    tc_prepare();
    tc_slots.ensure((size_t)Tp * 16);
    CUDA_TRY(launch_tc_tails(tc_img.p, comp.p, Tp, d, tc_slots.p, st));
    note_launch();
    tc_tails_epoch = scan_epoch;
  }
  bool capp_ready = false;
  bool tc_cap_on = false;       // caps in use for this round's scans
  bool tc_bound_only = false;   // the next tc_scan is the bound pass (writes ucap, no keys)
  bool tpmin_on = false;   // allocated and reset for this run
  bool tpmin_use = false;  // this scan may read / write it
  DevBuf<unsigned> pbits;
  DevBuf<unsigned char> pkeep;
  DevBuf<int> pcount;
  DevBuf<long long> poffset;
  DevBuf<unsigned long long> ucomp;
  double pairs_covered = 0.0;
  const int2* p1_list = nullptr;
  // round path
  DevBuf<Cand> cands, cands2;
  DevBuf<float> ckeys, ckeys2;  // tau selection keys (top_p_pass)
  DevBuf<char> ctmp;
  DevBuf<unsigned long long> rB1;  // round path: per-row best screened key (may be stale)
  bool rb1_valid = false;
  DevBuf<int> active, rmap, rsize;
  DevBuf<int2> kv;
  nnm_stats stats{};
  std::vector<nnm_round_stat> round_log;  // per-round records of the last nnm_run
  CachedAlloc talloc;
  // start / end of one round's record (stats deltas; the caller has synchronised)
  nnm_round_stat rl_open(int64_t round) {
    flush_scan_stats();
    nnm_round_stat r{};
    r.round = round;
    r.ms = -1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
    r.scan_ms = -stats.scan_ms;
    r.pairs_evaluated = -stats.pairs_evaluated;
    r.items = -stats.tc_items;
    return r;
  }
  void rl_close(nnm_round_stat r, int64_t merged) {
    flush_scan_stats();
    r.ms += 1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
    r.scan_ms += stats.scan_ms;
    r.pairs_evaluated += stats.pairs_evaluated;
    r.items += stats.tc_items;
    r.merged = merged;
    round_log.push_back(r);
  }

  ~nnm_dataset() {
    // members (DevBuf) free asynchronously on st after this body; the stream is
    // destroyed last (cudaStreamDestroy defers until the queued frees finish)
    if (st) {
      cudaSetDevice(device);
      cudaStreamSynchronize(st);
    }
    talloc.release();
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (ev2) cudaEventDestroy(ev2);
    if (rp_exec) cudaGraphExecDestroy(rp_exec);
    if (rp_exec2) cudaGraphExecDestroy(rp_exec2);
    for (auto e : tev_pool) cudaEventDestroy(e);
    if (st2) {
      cudaStreamSynchronize(st2);
      cudaStreamDestroy(st2);
    }
  }

  void sync() { CUDA_TRY(cudaStreamSynchronize(st)); }

  // key arrays start at NONE_KEY (INT64_MAX: signed and unsigned min agree, so
  // NCCL / gloo int64 all-reduce(MIN) combines them correctly)
  void fill_u32(unsigned* p, int64_t cnt, unsigned v) {
    fill_u32_kernel<<<blocks_for(cnt), 256, 0, st>>>(p, cnt, v); note_launch();
    CUDA_TRY(cudaGetLastError());
  }

  void fill_none(unsigned long long* p, int64_t cnt) {
    fill_u64_kernel<<<blocks_for(cnt), 256, 0, st>>>(p, cnt, NONE_KEY); note_launch();
    CUDA_TRY(cudaGetLastError());
  }

  template <class T>
  T read1(const T* dev) {
    T v;
    CUDA_TRY(cudaMemcpyAsync(&v, dev, sizeof(T), cudaMemcpyDeviceToHost, st));
    sync();
    return v;
  }

  void ensure_norms(int metric) {
    int kind = (metric == SQEUCLIDEAN) ? EUCLIDEAN : metric;
    if (norm_metric == kind) return;
    norm.ensure(n);
    scratch_u64.ensure(4);
    CUDA_TRY(cudaMemsetAsync(scratch_u64.p, 0, sizeof(unsigned long long), st));
    norms_kernel<<<blocks_for(n), 256, 0, st>>>(X64.p, n, d, kind, norm.p, scratch_u64.p); note_launch();
    CUDA_TRY(cudaGetLastError());
    maxnorm = bits_to_double(read1(scratch_u64.p));
    norm_metric = kind;
  }

  int64_t tile_pairs() const { return (int64_t)vT * (vT + 1) / 2; }

  void use_original_view() {
    cur_X32 = X32.p;
    cur_X64 = X64.p;
    vn = n;
    vld = ld;
    vT = T;
    if (!tcount_o.p) {
      tcount_o.ensure(T);
      std::vector<int> h(T);
      for (int t = 0; t < T; ++t) h[t] = (int)std::min<int64_t>(TILE, n - (int64_t)t * TILE);
      CUDA_TRY(cudaMemcpyAsync(tcount_o.p, h.data(), T * sizeof(int), cudaMemcpyHostToDevice, st));
      sync();
    }
    cur_tcount = tcount_o.p;
  }

  void use_boruvka_view() {
    ensure_order();
    cur_X32 = X32p.p;
    cur_X64 = X64p.p;
    vn = np_;
    vld = np_;
    vT = Tp;
    cur_tcount = tcount_p.p;
  }

  static int size_rule(int kl2, int kl3) {
    if (kl3 != INT_UNSET) return kl3;
    if (kl2 != INT_UNSET) return 2 * kl2;
    return INT_UNSET;
  }

  const int* eff_sizes(int kl2) {
    psize_eff.ensure(vld);
    eff_size_kernel<<<blocks_for(vld), 256, 0, st>>>(psize.p, vld, kl2, psize_eff.p); note_launch();
    CUDA_TRY(cudaGetLastError());
    return psize_eff.p;
  }

  // full or partial screening scan into (b1, b2); times the launch with events
  void scan(int metric, unsigned long long* b1, unsigned long long* b2, bool top2, int kl2, int kl3,
            float thr_hi, int64_t w_begin, int64_t w_end, const int2* items = nullptr,
            bool reset = true, const double* orient_umax = nullptr) {
    if (reset) {
      fill_none(b1, vn);
      if (b2) fill_none(b2, vn);
    }
    if (tc_on && items && b2 && top2 && cur_X32 == X32p.p && kl2 == INT_UNSET &&
        kl3 == INT_UNSET) {
      tc_scan(b1, b2, thr_hi, w_begin, w_end, items, orient_umax);
      return;
    }
    tile_range.ensure(vT);
    tile_range_kernel<<<vT, TILE, 0, st>>>(comp.p, vn, vT, tile_range.p); note_launch();
    const int ksum = size_rule(kl2, kl3);
    ScanArgs a;
    a.X32 = cur_X32;
    a.ld = vld;
    a.n = (int)vn;
    a.d = d;
    a.T = vT;
    a.comp = comp.p;
    a.psize = ksum != INT_UNSET ? eff_sizes(kl2) : comp.p;
    a.ksum = ksum;
    a.tile_range = tile_range.p;
    a.thr_hi = thr_hi;
    a.w_begin = w_begin;
    a.w_end = w_end;
    a.items = items;
    a.B1 = b1;
    a.B2 = b2;
    a.dot_center = nullptr;
    a.dot_B = a.dot_nbk = a.dot_Bmax = nullptr;
    a.dot_k = a.dot_onepA = 1.f;
    a.tpmin = nullptr;
    a.em = em;
    a.rsum = 2.0 * maxnorm * (1.0 + 1e-12);
    if (tpmin_use && items && cur_X32 == X32p.p && !(dot_on && cur_X32 == X32p.p)) a.tpmin = tpmin.p;
    if (dot_on && cur_X32 == X32p.p) {
      a.dot_center = tcenter32.p;
      a.dot_B = dotB.p;
      a.dot_nbk = dotNBK.p;
      a.dot_Bmax = dotBmax.p;
      a.dot_k = float_down(1.0 / (1.0 + dm.A));
      a.dot_onepA = float_up(1.0 + dm.A);
    }
    int occ = scan_use_reg(a) ? 2 : scan_occupancy(metric, d);
    int64_t nitems = w_end - w_begin;
    int grid = (int)std::min<int64_t>(nitems, (int64_t)sms * occ);
    if (grid < 1) return;
    scan_timer_start();
    CUDA_TRY(launch_scan(metric, a, top2, grid, st));
    note_launch();
    scan_timer_stop();
    if (items) {  // exact count of real pairs in the listed tile pairs (device accumulator)
      item_pairs_kernel<<<blocks_for(w_end - w_begin), 256, 0, st>>>(items + w_begin, w_end - w_begin, cur_tcount, pair_acc_ptr()); note_launch();
    } else {  // unordered real pairs covered by this range of the triangle
      stats.pairs_evaluated += (double)n * (double)(n - 1) / 2.0 * ((double)(w_end - w_begin) / (double)tile_pairs());
    }
  }

  // operand image + bounds of the kd view for the tensor-core scan (once per dataset)
  void tc_prepare() {
    if (tc_ready) return;
    auto tq0 = std::chrono::steady_clock::now();
    struct Report {
      nnm_dataset* ds;
      std::chrono::steady_clock::time_point t0;
      ~Report() {
        if (getenv("NNM_DEBUG")) {
          cudaStreamSynchronize(ds->st);
          fprintf(stderr, "[nnm] host: tc operand image %.2f ms\n",
                  std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
        }
      }
    } report{this, tq0};
    tc_img.ensure((size_t)Tp * TC_TILE_FLOATS);
    tc_tnorm.ensure(np_);
    tc_eta.ensure(np_);
    tc_meta.ensure((size_t)Tp * TC_META);
    tc_sq.ensure(np_);
    CUDA_TRY(launch_tc_prepare(X64p.p, porig.p, tcenter.p, normp.p, np_, d, Tp, tc_img.p,
                               tc_tnorm.p, tc_eta.p, tc_meta.p, tc_sq.p, st));
    note_launch();
    note_launch();
    tc_ready = true;
  }

  // tensor-core screening scan of the listed (upper-triangular) tile pairs: the list
  // is mirrored to the full square and sorted by row tile, then scanned row-wise
  // umax (phase 2 only): an orientation (I, J) serves the rows of tile I alone, so it is
  // dropped when the tile pair's rigorous lower bound exceeds UMAX_I (DESIGN 3.1)
  void tc_scan(unsigned long long* b1, unsigned long long* b2, float thr_hi, int64_t w_begin,
               int64_t w_end, const int2* items, const double* umax = nullptr) {
    const int64_t n_up = w_end - w_begin;
    if (n_up <= 0) return;
    tc_phase2 = umax != nullptr;
    tc_prepare();
    tc_tails();
    // the bound pass and the exact pass of phase 1 scan the same list: mirror + sort once
    const bool reuse = !umax && tc_list_epoch == scan_epoch && tc_list_items == items &&
                       tc_list_wb == w_begin && tc_list_we == w_end;
    if (reuse) {
      tc_launch(b1, b2, thr_hi, items, w_begin, w_end, tc_list_nfull);
      return;
    }
    tc_items.ensure((size_t)2 * n_up);
    counters.ensure(8);
    CUDA_TRY(cudaMemsetAsync(counters.p + 5, 0, sizeof(unsigned long long), st));
    // every dropped orientation / diagonal twin leaves a sentinel (sorted last), counted
    tc_keys.ensure((size_t)2 * n_up);
    tc_js.ensure((size_t)2 * n_up);
    tc_mirror_kernel<<<blocks_for(n_up), 256, 0, st>>>(items + w_begin, n_up, umax, tc32.p, tcn32.p,
                                                       tr32.p, Tp, d, bv_metric,
                                                       (umax && tpmin_use) ? tpmin.p : nullptr,
                                                       tc_keys.p, tc_js.p,
                                                       counters.p + 5); note_launch();
    CUDA_TRY(cudaGetLastError());
    {  // radix sort over the bits the keys use (row tile incl. the drop row T, fp32 bits)
      int pb = 1;
      while (pb < 31 && ((int64_t)1 << pb) <= Tp) ++pb;
      tc_keys2.ensure((size_t)2 * n_up);
      tc_js2.ensure((size_t)2 * n_up);
      size_t tb = 0;
      CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, tc_keys.p, tc_keys2.p, tc_js.p, tc_js2.p,
                                               (int)(2 * n_up), 0, 32 + pb, st));
      sort_tmp.ensure(std::max<size_t>(tb, 1));
      CUDA_TRY(cub::DeviceRadixSort::SortPairs(sort_tmp.p, tb, tc_keys.p, tc_keys2.p, tc_js.p,
                                               tc_js2.p, (int)(2 * n_up), 0, 32 + pb, st));
      std::swap(tc_keys.p, tc_keys2.p);
      std::swap(tc_keys.n, tc_keys2.n);
      std::swap(tc_js.p, tc_js2.p);
      std::swap(tc_js.n, tc_js2.n);
    }
    const int64_t nfull = 2 * n_up - (int64_t)read1(counters.p + 5);
    tc_list_epoch = scan_epoch;
    tc_list_items = items;
    tc_list_wb = w_begin;
    tc_list_we = umax ? -1 : w_end;  // lists with orientation drops are not reused
    tc_list_nfull = nfull;
    if (nfull <= 0) return;
    tc_items_kernel<<<blocks_for(nfull), 256, 0, st>>>(tc_keys.p, tc_js.p, nfull, tc_items.p); note_launch();
    CUDA_TRY(cudaGetLastError());
    tc_launch(b1, b2, thr_hi, items, w_begin, w_end, nfull);
  }

  int64_t scan_epoch = 0;  // bumped every round: the mirrored list is reused within a round
  int64_t tc_list_epoch = -1, tc_list_wb = -1, tc_list_we = -1, tc_list_nfull = 0;
  const int2* tc_list_items = nullptr;

  void tc_launch(unsigned long long* b1, unsigned long long* b2, float thr_hi, const int2* items,
                 int64_t w_begin, int64_t w_end, int64_t nfull) {
    const int64_t n_up = w_end - w_begin;
    if (nfull <= 0) return;
    TcArgs a;
    a.img = tc_img.p;
    a.tnorm = tc_tnorm.p;
    a.eta = tc_eta.p;
    a.meta = tc_meta.p;
    a.sq = tc_sq.p;
    a.comp = comp.p;
    a.X64 = X64p.p;
    a.np = (int)np_;
    a.d = d;
    a.T = Tp;
    a.items = tc_items.p;
    a.w_begin = 0;
    a.w_end = nfull;
    a.thr_hi = thr_hi;
    a.B1 = b1;
    a.B2 = b2;
    a.dump = nullptr;
    a.tpmin = tpmin_use ? tpmin.p : nullptr;
    a.ucap = tc_bound_only ? ucap.p : (tc_cap_on ? const_cast<unsigned*>(caps_read) : nullptr);
    a.capp = (!tc_bound_only && tc_cap_on && capp_ready) ? capp.p : nullptr;
    a.bound_only = tc_bound_only ? 1 : 0;
    a.trange = tile_range.p;  // computed by this round's step 1
    a.slots = tc_slots.p;     // slot records + A tails of this round (tc_tails)
    const char* dbg = getenv("NNM_TC_DBG");
    a.dbg = dbg ? atoi(dbg) : 0;
    // deferred exact keys (exact passes): candidates appended by the scan, FP64-evaluated
    // by tc_exact_kernel right after it (NNM_TC_DEFER=0: in the epilogue)
    const char* dfe = getenv("NNM_TC_DEFER");
    // phase-1 passes only: there the rows' thresholds come from the bound pass / the seeds
    // and tighten little within a launch; phase-2 rows tighten as exact keys arrive, and
    // deferring them would multiply the candidates (C4 round 1: 1.5 -> 6.3 ms)
    const bool defer = !tc_bound_only && !tc_phase2 && !(dfe && dfe[0] == '0');
    a.cand = nullptr;
    a.ccount = nullptr;
    a.ccap = 0;
    if (defer) {
      tc_cand.ensure((size_t)1 << 24);
      counters.ensure(8);
      CUDA_TRY(cudaMemsetAsync(counters.p + 7, 0, sizeof(unsigned long long), st));
      a.cand = tc_cand.p;
      a.ccount = counters.p + 7;
      a.ccap = tc_cand.n;
    }
    const int grid = (int)std::min<int64_t>(nfull, (int64_t)sms);
    const char* trf = getenv("NNM_TC_TRACE");
    DevBuf<long long> trbuf;
    a.trace = nullptr;
    if (trf && nfull / grid >= 256) {
      trbuf.ensure(8 * 256 * 2 + 4);
      CUDA_TRY(cudaMemsetAsync(trbuf.p, 0, (8 * 256 * 2 + 4) * sizeof(long long), st));
      a.trace = trbuf.p;
    }
    scan_timer_start();
    CUDA_TRY(launch_tc_scan(a, grid, st));
    note_launch();
    if (a.cand) {
      CUDA_TRY(launch_tc_exact(a.cand, a.ccount, (int64_t)a.ccap, X64p.p, d, thr_hi, b1, b2, st));
      note_launch();
      if (getenv("NNM_DEBUG"))
        fprintf(stderr, "[nnm] tc deferred candidates: %llu (cap %llu)\n",
                (unsigned long long)read1(a.ccount), (unsigned long long)a.ccap);
    }
    scan_timer_stop();
    stats.tc_items += nfull;
    if (getenv("NNM_DEBUG")) {
      const double ms0 = stats.scan_ms;
      flush_scan_stats();
      const double ms = stats.scan_ms - ms0;
      fprintf(stderr, "[nnm] tc scan: %lld items, %.2f ms (%.0f ns/item)\n", (long long)nfull, ms,
              1e6 * ms / (double)nfull);
    }
    if (a.trace) {  // append the timeline of this launch (CTA 0, first 256 items)
      std::vector<long long> h(8 * 256 * 2 + 4);
      CUDA_TRY(cudaMemcpyAsync(h.data(), a.trace, h.size() * sizeof(long long), cudaMemcpyDeviceToHost, st));
      sync();
      if (FILE* f = fopen(trf, "a")) {
        fprintf(f, "launch items %lld grid %d exact_evals %lld seeds %lld slow_groups %lld\n", (long long)nfull,
                grid, h[8 * 256 * 2], h[8 * 256 * 2 + 1], h[8 * 256 * 2 + 2]);
        const long long t0 = h[0];
        for (int q = 0; q < 256; ++q)
          fprintf(f, "%d prod %lld mma %lld prep %lld %lld epi_prepped %lld epi %lld %lld | ld %lld sums %lld tail %lld dn %lld fence %lld\n", q,
                  h[(0 * 256 + q) * 2] - t0, h[(1 * 256 + q) * 2] - t0, h[(2 * 256 + q) * 2] - t0,
                  h[(2 * 256 + q) * 2 + 1] - t0, h[(4 * 256 + q) * 2] - t0,
                  h[(3 * 256 + q) * 2] - t0, h[(3 * 256 + q) * 2 + 1] - t0,
                  h[(5 * 256 + q) * 2] - t0, h[(5 * 256 + q) * 2 + 1] - t0, h[(6 * 256 + q) * 2] - t0,
                  h[(6 * 256 + q) * 2 + 1] - t0, h[(7 * 256 + q) * 2] - t0);
        fclose(f);
      }
    }
    if (tc_bound_only) return;  // the exact pass over the same items counts the pairs
    item_pairs_kernel<<<blocks_for(n_up), 256, 0, st>>>(items + w_begin, n_up, cur_tcount, pair_acc_ptr()); note_launch();
  }

  // ---- deferred scan statistics: the scans record CUDA events and accumulate their pair
  // counts on the device; the host reads them once per round (rl_close) / per run instead
  // of synchronising after every scan
  std::vector<cudaEvent_t> tev_pool;
  size_t tev_used = 0;
  DevBuf<unsigned long long> pair_acc;
  bool pair_acc_dirty = false;
  unsigned long long* pair_acc_ptr() {
    if (!pair_acc.p) {
      pair_acc.ensure(1);
      CUDA_TRY(cudaMemsetAsync(pair_acc.p, 0, sizeof(unsigned long long), st));
    }
    pair_acc_dirty = true;
    return pair_acc.p;
  }
  void scan_timer_start() {
    if (tev_used == tev_pool.size()) {
      cudaEvent_t e;
      CUDA_TRY(cudaEventCreate(&e));
      tev_pool.push_back(e);
    }
    CUDA_TRY(cudaEventRecord(tev_pool[tev_used++], st));
  }
  void scan_timer_stop() {
    scan_timer_start();
    stats.scans += 1;
  }
  void flush_scan_stats() {
    if (tev_used) {
      CUDA_TRY(cudaEventSynchronize(tev_pool[tev_used - 1]));
      for (size_t i = 0; i + 1 < tev_used; i += 2) {
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, tev_pool[i], tev_pool[i + 1]));
        stats.scan_ms += ms;
      }
      tev_used = 0;
    }
    if (pair_acc_dirty) {
      stats.pairs_evaluated += (double)read1(pair_acc.p);
      CUDA_TRY(cudaMemsetAsync(pair_acc.p, 0, sizeof(unsigned long long), st));
      pair_acc_dirty = false;
    }
  }

  // collect pairs (row list x columns) with screened value <= per-row bound
  int64_t collect(int metric, const int* rows, int nr, const float* bounds, const int* cols,
                  int nc_cols, int triangle, int kl2, int kl3) {
    if (nr <= 0 || nc_cols <= 0) return 0;
    int64_t ldr = ((int64_t)nr + TILE - 1) / TILE * TILE;
    gathered.ensure((size_t)ldr * d);
    gather_kernel<<<blocks_for(ldr), 256, 0, st>>>(cur_X32, vld, d, rows, nr, ldr, gathered.p); note_launch();
    CUDA_TRY(cudaGetLastError());
    const float* XC = cur_X32;
    int64_t ldc = vld;
    DevBuf<float> gcols;
    if (cols) {
      ldc = ((int64_t)nc_cols + TILE - 1) / TILE * TILE;
      if (cols == rows) {
        XC = gathered.p;
        ldc = ldr;
      } else {
        gcols.ensure((size_t)ldc * d);
        gather_kernel<<<blocks_for(ldc), 256, 0, st>>>(cur_X32, vld, d, cols, nc_cols, ldc, gcols.p); note_launch();
        CUDA_TRY(cudaGetLastError());
        XC = gcols.p;
      }
    }
    counters.ensure(8);
    unsigned long long cap = std::max<unsigned long long>(pairs.n, 1u << 16);
    for (int attempt = 0; attempt < 2; ++attempt) {
      pairs.ensure(cap);
      CUDA_TRY(cudaMemsetAsync(counters.p + 6, 0, sizeof(unsigned long long), st));
      CollectArgs a;
      a.XR = gathered.p;
      a.ldr = ldr;
      a.nr = nr;
      a.rid = rows;
      a.XC = XC;
      a.ldc = ldc;
      a.nc = nc_cols;
      a.cid = cols;
      a.d = d;
      a.comp = comp.p;
      const int ksum = size_rule(kl2, kl3);
      a.psize = ksum != INT_UNSET ? eff_sizes(kl2) : comp.p;
      a.ksum = ksum;
      a.rbound = bounds;
      a.triangle = triangle;
      a.out = pairs.p;
      a.count = counters.p + 6;  // [0..2] boruvka, [3..5] top-P
      a.cap = pairs.n;
      int64_t items = (ldr / TILE) * (ldc / TILE);
      int grid = (int)std::min<int64_t>(items, (int64_t)sms * 2);
      CUDA_TRY(launch_collect(metric, a, grid, st));
      note_launch();
      unsigned long long cnt = read1(counters.p + 6);
      if (cnt <= pairs.n) return (int64_t)cnt;
      cap = cnt + (cnt >> 2);
    }
    throw NnmError{NNM_E_CUDA, "collect: candidate buffer overflow after resize"};
  }

  void exact_pairs(int metric, int64_t count) {
    pair_d.ensure(count);
    if (count == 0) return;
    switch (metric) {
      case MANHATTAN:
        exact_pairs_kernel<MANHATTAN><<<blocks_for(count), 256, 0, st>>>(cur_X64, d, pairs.p, count, pair_d.p); note_launch();
        break;
      case CHEBYSHEV:
        exact_pairs_kernel<CHEBYSHEV><<<blocks_for(count), 256, 0, st>>>(cur_X64, d, pairs.p, count, pair_d.p); note_launch();
        break;
      default:
        exact_pairs_kernel<EUCLIDEAN><<<blocks_for(count), 256, 0, st>>>(cur_X64, d, pairs.p, count, pair_d.p); note_launch();
    }
    CUDA_TRY(cudaGetLastError());
    stats.exact_evals += count;
  }

  // ---------------------------------------------------------------- Boruvka
  void bv_begin(int metric, double dmax) {
    bv_metric = metric;
    const bool dbg_t = getenv("NNM_DEBUG") != nullptr;
    auto tb0 = std::chrono::steady_clock::now();
    use_boruvka_view();
    if (dbg_t) {
      sync();
      fprintf(stderr, "[nnm] host: view (kd order) %.2f ms, %d tiles\n",
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tb0).count(), Tp);
    }
    ensure_norms_p(metric);
    em = make_err_model(metric, d);
    bv_thr = INFINITY;
    bv_thr_hi = INFINITY;
    auto tb1 = std::chrono::steady_clock::now();
    ensure_geometry(metric);
    if (dbg_t) {
      sync();
      fprintf(stderr, "[nnm] host: norms + geometry %.2f ms\n",
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tb1).count());
    }
    const char* de = getenv("NNM_DOT");
    dot_on = (metric == EUCLIDEAN || metric == SQEUCLIDEAN) && !(de && de[0] == '0') &&
             scan_use_ws(d);
    const char* te = getenv("NNM_TC");
    tc_on = (metric == EUCLIDEAN || metric == SQEUCLIDEAN) && tc_supported(d) &&
            !(te && te[0] == '0');
    if (!std::isnan(dmax)) {
      bv_thr = metric == EUCLIDEAN ? dmax * dmax : dmax;  // metrics.py:93-103
      // dot-form keys are lower bounds of S: compare them with thr itself
      bv_thr_hi = (dot_on || tc_on) ? float_up(bv_thr)
                                    : float_up(screen_upper(em, bv_thr, 2.0 * maxnorm));
    }
    comp.ensure(vn);
    fill_comp_view_kernel<<<blocks_for(vn), 256, 0, st>>>(porig.p, vn, comp.p); note_launch();
    CUDA_TRY(cudaGetLastError());
    B1.ensure(vn);
    B2.ensure(vn);
    rb_d.ensure(vn);
    rb_j.ensure(vn);
    rowlow.ensure(vn);
    amb.ensure(vn);
    resc.ensure(vn);
    resc_bound.ensure(vn);
    parent.ensure(vn);
    cmin_d.ensure(vn);
    cmin_ab.ensure(vn);
    counters.ensure(8);
    edges.ensure(std::max<int64_t>(n - 1, 1));
    flag.ensure(1);
    CUDA_TRY(cudaMemsetAsync(counters.p, 0, 8 * sizeof(unsigned long long), st));
    // tile-pair bound cache (TC scan only; 4 B per tile pair: 0.58 GB at 2M points)
    const char* ce = getenv("NNM_TPCACHE");
    tpmin_use = false;
    // the tensor-core scan and the direct-form FP32 scans (L1 / L-inf) both publish it
    tpmin_on = (tc_on || metric == MANHATTAN || metric == CHEBYSHEV) && !(ce && ce[0] == '0') &&
               tile_pairs() * 4 <= ((int64_t)4 << 30);
    if (tpmin_on) {
      tpmin.ensure(tile_pairs());
      // the cache starts from the geometric bounds (both are lower bounds of every pair)
      if (glb_ready())
        CUDA_TRY(cudaMemcpyAsync(tpmin.p, glb.p, tile_pairs() * sizeof(unsigned),
                                 cudaMemcpyDeviceToDevice, st));
      else
        CUDA_TRY(cudaMemsetAsync(tpmin.p, 0, tile_pairs() * sizeof(unsigned), st));
    }
    bv_round = 0;
    bv_ncomp = n;
  }

  void ensure_order() {
    if (have_order) return;
    // compact kd order over the n real points
    DevBuf<int> order, segid;
    order.ensure(n);
    segid.ensure(n);
    iota_kernel<<<blocks_for(n), 256, 0, st>>>(order.p, (int)n); note_launch();
    CUDA_TRY(cudaMemsetAsync(segid.p, 0, n * sizeof(int), st));
    std::vector<int> hb = {0}, hs = {(int)n};
    int nseg = 1;
    const char* ke = getenv("NNM_KD");
    const bool kd = n > TILE && !(ke && ke[0] == '0');
    DevBuf<int> sbeg, ssz;
    sbeg.ensure(1);
    ssz.ensure(1);
    CUDA_TRY(cudaMemcpyAsync(sbeg.p, hb.data(), sizeof(int), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(ssz.p, hs.data(), sizeof(int), cudaMemcpyHostToDevice, st));
    if (!kd) {  // no reordering: cut the original order into 128-point leaves
      nseg = (int)((n + TILE - 1) / TILE);
      hb.resize(nseg);
      hs.resize(nseg);
      for (int t = 0; t < nseg; ++t) {
        hb[t] = t * TILE;
        hs[t] = (int)std::min<int64_t>(TILE, n - (int64_t)t * TILE);
      }
      std::vector<int> hseg(n);
      for (int64_t c = 0; c < n; ++c) hseg[c] = (int)(c / TILE);
      sbeg.ensure(nseg);
      ssz.ensure(nseg);
      CUDA_TRY(cudaMemcpyAsync(sbeg.p, hb.data(), nseg * sizeof(int), cudaMemcpyHostToDevice, st));
      CUDA_TRY(cudaMemcpyAsync(ssz.p, hs.data(), nseg * sizeof(int), cudaMemcpyHostToDevice, st));
      CUDA_TRY(cudaMemcpyAsync(segid.p, hseg.data(), n * sizeof(int), cudaMemcpyHostToDevice, st));
      sync();
    } else {
      DevBuf<int> sdim, ssplit, nchild, cbase, nbeg, nsz, order2;
      DevBuf<unsigned long long> keys, keys2, gbest;
      DevBuf<char> kd_tmp;
      keys.ensure(n);
      for (int lv = 0; lv < 64; ++lv) {
        // separated pieces may be cut off anywhere (and leaves split at a clear gap) in the
        // first 32 levels; later levels only halve, so every segment ends <= TILE
        const int allow_off = lv < 32 ? 1 : 0;
        if (!allow_off) {
          std::vector<int> hsz(nseg);
          CUDA_TRY(cudaMemcpyAsync(hsz.data(), ssz.p, nseg * sizeof(int), cudaMemcpyDeviceToHost, st));
          sync();
          if (*std::max_element(hsz.begin(), hsz.end()) <= TILE) break;
        }
        sdim.ensure(nseg);
        ssplit.ensure(nseg);
        nchild.ensure(nseg);
        cbase.ensure(nseg + 1);
        kd_dim_kernel<<<nseg, 32, 0, st>>>(X64.p, d, order.p, sbeg.p, ssz.p, nseg, allow_off, sdim.p); note_launch();
        kd_key_kernel<<<blocks_for(n), 256, 0, st>>>(X64.p, n, d, order.p, segid.p, sdim.p, keys.p); note_launch();
        // stable radix sort on (segment, coordinate): only the bits the segment ids use
        {
          int sbits = 0;
          while (sbits < 31 && (1 << sbits) < nseg) ++sbits;
          order2.ensure(n);
          keys2.ensure(n);
          size_t tb = 0;
          cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.p, keys2.p, order.p, order2.p, (int)n, 0,
                                          32 + sbits, st);
          kd_tmp.ensure(tb);
          CUDA_TRY(cub::DeviceRadixSort::SortPairs(kd_tmp.p, tb, keys.p, keys2.p, order.p, order2.p,
                                                   (int)n, 0, 32 + sbits, st));
          std::swap(keys.p, keys2.p);
          std::swap(keys.n, keys2.n);
          std::swap(order.p, order2.p);
          std::swap(order.n, order2.n);
        }
        if (nseg < 2 * sms) {  // few big segments: the position-parallel split search
          gbest.ensure(2 * nseg);
          CUDA_TRY(cudaMemsetAsync(gbest.p, 0, 2 * nseg * sizeof(unsigned long long), st));
          kd_gap_kernel<<<blocks_for(n), 256, 0, st>>>(keys.p, n, segid.p, sbeg.p, ssz.p, gbest.p); note_launch();
          kd_gap_split_kernel<<<blocks_for(nseg), 256, 0, st>>>(keys.p, sbeg.p, ssz.p, nseg, allow_off,
                                                                gbest.p, ssplit.p); note_launch();
          // segments <= TILE in this level still take the leaf rule of kd_splitpos_kernel
          kd_splitpos_kernel<<<nseg, KD_SPLIT_THREADS, 0, st>>>(keys.p, sbeg.p, ssz.p, nseg, allow_off,
                                                                ssplit.p, 1); note_launch();
        } else {
          kd_splitpos_kernel<<<nseg, KD_SPLIT_THREADS, 0, st>>>(keys.p, sbeg.p, ssz.p, nseg, allow_off, ssplit.p, 0); note_launch();
        }
        kd_children_kernel<<<blocks_for(nseg), 256, 0, st>>>(nseg, ssz.p, ssplit.p, nchild.p); note_launch();
        thrust::exclusive_scan(thrust::cuda::par(talloc).on(st), nchild.p, nchild.p + nseg, cbase.p, 0);
        int lastc = read1(nchild.p + (nseg - 1)), lastb = read1(cbase.p + (nseg - 1));
        const int nseg2 = lastb + lastc;
        if (nseg2 == nseg) break;  // no segment split: every leaf is final
        nbeg.ensure(nseg2);
        nsz.ensure(nseg2);
        kd_newsegs_kernel<<<blocks_for(nseg), 256, 0, st>>>(nseg, sbeg.p, ssz.p, ssplit.p, cbase.p, nbeg.p, nsz.p); note_launch();
        kd_relabel_kernel<<<blocks_for(n), 256, 0, st>>>(n, sbeg.p, ssz.p, ssplit.p, cbase.p, segid.p); note_launch();
        CUDA_TRY(cudaGetLastError());
        std::swap(sbeg.p, nbeg.p);
        std::swap(sbeg.n, nbeg.n);
        std::swap(ssz.p, nsz.p);
        std::swap(ssz.n, nsz.n);
        nseg = nseg2;
      }
    }
    // leaf k -> tile k (positions k*128 .. k*128 + size - 1, then pads)
    Tp = nseg;
    np_ = (int64_t)Tp * TILE;
    porig.ensure(np_);
    ppos.ensure(n);
    fill_int_kernel<<<blocks_for(np_), 256, 0, st>>>(porig.p, np_, -1); note_launch();
    kd_place_kernel<<<blocks_for(n), 256, 0, st>>>(n, order.p, segid.p, sbeg.p, porig.p, ppos.p); note_launch();
    tcount_p.ensure(Tp);
    tile_count_kernel<<<Tp, TILE, 0, st>>>(porig.p, Tp, tcount_p.p); note_launch();
    X64p.ensure((size_t)np_ * d);
    gather_rows_kernel<<<blocks_for(np_ * d), 256, 0, st>>>(X64.p, np_, d, porig.p, X64p.p); note_launch();
    X32p.ensure((size_t)np_ * d);
    CUDA_TRY(cudaMemsetAsync(flag.p, 0, sizeof(int), st));
    prepare_view_kernel<<<blocks_for(np_), 256, 0, st>>>(X64p.p, porig.p, np_, d, X32p.p); note_launch();
    CUDA_TRY(cudaGetLastError());
    sync();
    have_order = true;
  }

  void ensure_norms_p(int metric) {
    ensure_norms(metric);
    if (normp_metric == norm_metric) return;
    normp.ensure(np_);
    gather_norm_kernel<<<blocks_for(np_), 256, 0, st>>>(np_, porig.p, norm.p, normp.p); note_launch();
    maxnormp = maxnorm;
    normp_metric = norm_metric;
  }

  void ensure_geometry(int metric) {
    int kind = (metric == SQEUCLIDEAN) ? EUCLIDEAN : metric;
    if (geom_metric == kind) return;
    tcenter.ensure((size_t)Tp * d);
    tradius.ensure(Tp);
    size_t sm = (size_t)d * sizeof(double);
    switch (kind) {
      case MANHATTAN: tile_geom_kernel<MANHATTAN><<<Tp, TILE, sm, st>>>(X64p.p, tcount_p.p, d, tcenter.p, tradius.p); break;
      case CHEBYSHEV: tile_geom_kernel<CHEBYSHEV><<<Tp, TILE, sm, st>>>(X64p.p, tcount_p.p, d, tcenter.p, tradius.p); break;
      default: tile_geom_kernel<EUCLIDEAN><<<Tp, TILE, sm, st>>>(X64p.p, tcount_p.p, d, tcenter.p, tradius.p);
    }
    note_launch();
    CUDA_TRY(cudaGetLastError());
    tc32.ensure((size_t)Tp * d);
    tcn32.ensure(Tp);
    tr32.ensure(Tp);
    switch (kind) {
      case MANHATTAN: centers32_kernel<MANHATTAN><<<blocks_for(Tp), 256, 0, st>>>(tcenter.p, tradius.p, Tp, d, tc32.p, tcn32.p, tr32.p); break;
      case CHEBYSHEV: centers32_kernel<CHEBYSHEV><<<blocks_for(Tp), 256, 0, st>>>(tcenter.p, tradius.p, Tp, d, tc32.p, tcn32.p, tr32.p); break;
      default: centers32_kernel<EUCLIDEAN><<<blocks_for(Tp), 256, 0, st>>>(tcenter.p, tradius.p, Tp, d, tc32.p, tcn32.p, tr32.p);
    }
    note_launch();
    CUDA_TRY(cudaGetLastError());
    if (kind == EUCLIDEAN) {
      dm = make_dot_model(d);
      tcenter32.ensure((size_t)Tp * d);
      dotB.ensure(np_);
      dotNBK.ensure(np_);
      dotBmax.ensure(Tp);
      dot_consts_kernel<<<blocks_for(np_), 256, 0, st>>>(X32p.p, np_, d, porig.p, tcenter.p, normp.p,
                                                         maxnormp, dm, tcenter32.p, dotB.p, dotNBK.p); note_launch();
      tile_bmax_kernel<<<Tp, TILE, 0, st>>>(dotB.p, dotBmax.p); note_launch();
      CUDA_TRY(cudaGetLastError());
    }
    geom_metric = kind;
    build_tile_tables(kind);
  }

  DevBuf<unsigned long long> ekeys, ekeys2;  // item keys (I << 32 | J) and sort scratch
  DevBuf<char> sort_tmp;

  int item_bits() const {
    int b = 1;
    while (b < 31 && ((int64_t)1 << b) < Tp) ++b;
    return b;
  }

  // in-place ascending radix sort of u64 keys over bits [0, 32 + bits) of the high word
  // (keys = hi << 32 | lo with hi < 2^bits_hi, or ~0 padding when all 64 bits are sorted)
  void sort_keys(unsigned long long* keys, int64_t n, int hi_bits) {
    if (n <= 1) return;
    ekeys2.ensure(n);
    const int end_bit = std::min(64, 32 + hi_bits);
    size_t tb = 0;
    CUDA_TRY(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, ekeys2.p, (int)n, 0, end_bit, st));
    sort_tmp.ensure(std::max<size_t>(tb, 1));
    CUDA_TRY(cub::DeviceRadixSort::SortKeys(sort_tmp.p, tb, keys, ekeys2.p, (int)n, 0, end_bit, st));
    CUDA_TRY(cudaMemcpyAsync(keys, ekeys2.p, n * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, st));
  }

  // (I, J) items with (-1, -1) padding -> sorted unique items at the front; returns the count
  int64_t sort_unique_items(int2* items, int64_t n) {
    ekeys.ensure(n);
    int pb = 1;  // bits of the row index, padding row Tp included
    while (pb < 31 && ((int64_t)1 << pb) <= Tp) ++pb;
    const unsigned long long pad = ((unsigned long long)Tp << 32) | (unsigned)Tp;
    items_to_keys_kernel<<<blocks_for(n), 256, 0, st>>>(items, n, pad, ekeys.p); note_launch();
    sort_keys(ekeys.p, n, pb);
    auto* end = thrust::unique(thrust::cuda::par(talloc).on(st), ekeys.p, ekeys.p + n);
    int64_t m = end - ekeys.p;
    if (m > 0 && read1(ekeys.p + (m - 1)) == pad) --m;
    if (m > 0) { keys_to_items_kernel<<<blocks_for(m), 256, 0, st>>>(ekeys.p, m, items); note_launch(); }
    return m;
  }

  bool glb_ready() const { return glb_metric >= 0 && glb_metric == geom_metric; }
  bool nbr_ready() const { return nbr_metric >= 0 && nbr_metric == geom_metric; }

  // per-dataset tile-pair tables (once per dataset and metric): the geometric lower bound
  // of every tile pair (<= 2 GB) and the nearest-tile lists (d = 8 / 25)
  void build_tile_tables(int kind) {
    const int64_t W = (int64_t)Tp * (Tp + 1) / 2;
    const char* te = getenv("NNM_TILE_TABLES");
    const bool on = !(te && te[0] == '0');
    glb_metric = nbr_metric = -1;
    if (on && W * 4 <= ((int64_t)2 << 30)) {
      glb.ensure(W);
      const int g = (Tp + TR - 1) / TR;
      switch (kind) {
        case MANHATTAN: tile_glb_kernel<MANHATTAN><<<g, 256, 0, st>>>(tc32.p, tcn32.p, tr32.p, Tp, d, glb.p); break;
        case CHEBYSHEV: tile_glb_kernel<CHEBYSHEV><<<g, 256, 0, st>>>(tc32.p, tcn32.p, tr32.p, Tp, d, glb.p); break;
        default: tile_glb_kernel<EUCLIDEAN><<<g, 256, 0, st>>>(tc32.p, tcn32.p, tr32.p, Tp, d, glb.p);
      }
      note_launch();
      CUDA_TRY(cudaGetLastError());
      glb_metric = kind;
      const char* ce = getenv("NNM_COARSE");
      coarse_on = !(ce && ce[0] == '0');
      if (coarse_on) {
        tb_ = (Tp + CB - 1) / CB;
        cmin.ensure((size_t)tb_ * tb_);
        CUDA_TRY(cudaMemsetAsync(cmin.p, 0xFF, (size_t)tb_ * tb_ * sizeof(unsigned), st));
        coarse_min_kernel<<<Tp, 256, 0, st>>>(glb.p, Tp, tb_, cmin.p); note_launch();
        CUDA_TRY(cudaGetLastError());
      }
    }
    if (on && (d == 25 || d == 8)) {
      p1_l.ensure((size_t)Tp * P1_CHUNKS * NBR_SLICE);
      p1_j.ensure((size_t)Tp * P1_CHUNKS * NBR_SLICE);
      nbr.ensure((size_t)Tp * NBR);
      const dim3 g((Tp + P1_ROWS - 1) / P1_ROWS, P1_CHUNKS);
#define NNM_KNN(MM, DD) tile_knn_kernel<MM, DD><<<g, P1_ROWS, 0, st>>>(tc32.p, tr32.p, Tp, p1_l.p, p1_j.p)
      if (d == 25) {
        switch (kind) {
          case MANHATTAN: NNM_KNN(MANHATTAN, 25); break;
          case CHEBYSHEV: NNM_KNN(CHEBYSHEV, 25); break;
          default: NNM_KNN(EUCLIDEAN, 25);
        }
      } else {
        switch (kind) {
          case MANHATTAN: NNM_KNN(MANHATTAN, 8); break;
          case CHEBYSHEV: NNM_KNN(CHEBYSHEV, 8); break;
          default: NNM_KNN(EUCLIDEAN, 8);
        }
      }
#undef NNM_KNN
      note_launch();
      tile_knn_merge_kernel<<<blocks_for(Tp), 256, 0, st>>>(p1_l.p, p1_j.p, Tp, nbr.p); note_launch();
      CUDA_TRY(cudaGetLastError());
      nbr_metric = kind;
    }
  }

  template <int M>
  void pruned_lists(int64_t& n1, int64_t& n2) {
    const int64_t W = tile_pairs();
    // phase-1 seeds: PK nearest cross-capable tiles per tile
    items1.ensure((size_t)Tp * PK);
    const char* p1e = getenv("NNM_P1REG");
    const char* pke0 = getenv("NNM_PK");
    // seeds per tile: 4 in the first round (every row starts without a threshold), 1 after
    // (NNM_PK_LATE; measured C4 29.6 -> 27.7 ms, C5m 62.3 -> 53.7 ms against 4 throughout)
    const char* pkl = getenv("NNM_PK_LATE");
    const int pk_late = pkl ? std::max(1, std::min(PK, atoi(pkl))) : 1;
    const char* pkf = getenv("NNM_PK_FIRST");
    const int pk_first = pkf ? std::max(1, std::min(PK, atoi(pkf))) : 4;
    const int pk0 = pke0 ? std::max(1, std::min(PK, atoi(pke0))) : (bv_round == 0 ? pk_first : pk_late);
    if (nbr_ready()) {
      phase1_pick_kernel<<<blocks_for(Tp), 256, 0, st>>>(nbr.p, tile_range.p, Tp, pk0, items1.p); note_launch();
    } else if ((d == 25 || d == 8) && !(p1e && p1e[0] == '0')) {
      p1_l.ensure((size_t)Tp * P1_CHUNKS * PK);
      p1_j.ensure((size_t)Tp * P1_CHUNKS * PK);
      const dim3 g((Tp + P1_ROWS - 1) / P1_ROWS, P1_CHUNKS);
      if (d == 25)
        phase1_reg_kernel<M, 25><<<g, P1_ROWS, 0, st>>>(tc32.p, tr32.p, tile_range.p, Tp, p1_l.p, p1_j.p);
      else
        phase1_reg_kernel<M, 8><<<g, P1_ROWS, 0, st>>>(tc32.p, tr32.p, tile_range.p, Tp, p1_l.p, p1_j.p);
      note_launch();
      const char* pke = getenv("NNM_PK");
      // 4 seeds per tile: measured best on 2Mx25 (PK 8 -> 4: phase-1 scan -20%, the
      // component bounds stay tight enough that phase 2 does not grow)
      const int pk = pke ? std::max(1, std::min(PK, atoi(pke))) : (bv_round == 0 ? pk_first : pk_late);
      phase1_merge_kernel<<<blocks_for(Tp), 256, 0, st>>>(p1_l.p, p1_j.p, Tp, pk, items1.p); note_launch();
    } else {
      phase1_kernel<M><<<(Tp + TR - 1) / TR, 256, 0, st>>>(tc32.p, tr32.p, tile_range.p, Tp, d, items1.p); note_launch();
    }
    CUDA_TRY(cudaGetLastError());
    // sort by (I, J) as u64 keys (padding sorts last), drop duplicates and the padding
    n1 = sort_unique_items(items1.p, (int64_t)Tp * PK);
    int2* list1 = items1.p;
    pbits.ensure((size_t)(W + 31) / 32);
    CUDA_TRY(cudaMemsetAsync(pbits.p, 0, ((W + 31) / 32) * sizeof(unsigned), st));
    if (n1 > 0) { mark_items_kernel<<<blocks_for(n1), 256, 0, st>>>(list1, n1, Tp, pbits.p); note_launch(); }
    p1_list = list1;
    (void)W;
    n2 = 0;
  }

  template <int M>
  void pruned_phase2(int64_t& n2) {
    const int64_t W = tile_pairs();
    tumax.ensure(Tp);
    tile_umax_kernel<<<Tp, TILE, 0, st>>>(comp.p, vn, ucomp.p, bv_thr, tumax.p); note_launch();
    if (glb_ready()) {  // stream the bound table, append kept pairs, sort the (small) list
      counters.ensure(8);
      unsigned long long cap = std::max<unsigned long long>(ekeys.n, 1u << 20);
      for (int attempt = 0; attempt < 2; ++attempt) {
        ekeys.ensure(cap);
        CUDA_TRY(cudaMemsetAsync(counters.p + 4, 0, sizeof(unsigned long long), st));
        if (coarse_on && attempt == 0) {
          bumax.ensure(tb_);
          block_umax_kernel<<<blocks_for(tb_), 256, 0, st>>>(tumax.p, Tp, tb_, bumax.p); note_launch();
        }
        enum_append_kernel<<<Tp, 256, 0, st>>>(tpmin_use ? tpmin.p : glb.p, tile_range.p, tumax.p,
                                               pbits.p, Tp, ekeys.p, counters.p + 4, ekeys.n,
                                               coarse_on ? cmin.p : nullptr, bumax.p, tb_);
        note_launch();
        CUDA_TRY(cudaGetLastError());
        const unsigned long long cnt = read1(counters.p + 4);
        if (cnt <= ekeys.n) {
          n2 = (int64_t)cnt;
          break;
        }
        cap = cnt + cnt / 4;
        if (attempt == 1) throw NnmError{NNM_E_CUDA, "phase-2 list overflow after resize"};
      }
      items2.ensure(std::max<int64_t>(n2, 1));
      if (n2 > 0) {
        sort_keys(ekeys.p, n2, item_bits());
        keys_to_items_kernel<<<blocks_for(n2), 256, 0, st>>>(ekeys.p, n2, items2.p); note_launch();
      }
      return;
    }
    pkeep.ensure(W);
    pcount.ensure(Tp);
    poffset.ensure(Tp + 1);
    enum_count_kernel<M><<<(Tp + TR - 1) / TR, 256, 0, st>>>(tc32.p, tcn32.p, tr32.p, tile_range.p, tumax.p, pbits.p,
                                               Tp, d, tpmin_use ? tpmin.p : nullptr,
                                               pkeep.p, pcount.p);
    note_launch();
    CUDA_TRY(cudaGetLastError());
    thrust::exclusive_scan(thrust::cuda::par(talloc).on(st), pcount.p, pcount.p + Tp, poffset.p, 0LL);
    long long last_off = read1(poffset.p + (Tp - 1));
    int last_cnt = read1(pcount.p + (Tp - 1));
    n2 = last_off + last_cnt;
    items2.ensure(std::max<int64_t>(n2, 1));
    if (n2 > 0) { enum_write_kernel<<<Tp, 256, 0, st>>>(pkeep.p, poffset.p, Tp, items2.p); note_launch(); }
    CUDA_TRY(cudaGetLastError());
  }

  template <int M>
  void ucomp_t(const unsigned long long* b1) {
    ucomp_kernel<M><<<blocks_for(vn), 256, 0, st>>>(X64p.p, (int)vn, d, b1, comp.p, bv_thr, ucomp.p); note_launch();
  }

  // One pruned Boruvka scan: exact per-row keys for every row that can hold its
  // component's minimum edge; the single-rank sequence of the
  // staged round steps below (no exchanges).
  void pruned_scan(int metric) {
    round_bound(metric, 0, 1);
    round_phase1(B1.p, B2.p, 0, 1);
    round_phase2(B1.p, B2.p, B1.p, B2.p, 0, 1);
  }

  // ---- staged pruned round (DESIGN 6): every step is rank-local; between steps the
  // caller combines across ranks (torch.distributed / NCCL, or nnm_run_multi's peer
  // kernels).  Items of both phases are split into contiguous 1/world shares.
  //   round_bound   phase-1 list (identical on every rank), bound pass over the share
  //                 -> ucap (caller: all-reduce MIN -> caps)            [TC path only]
  //   round_phase1  exact phase-1 scan of the share under the caps -> (b1, b2)
  //                 (caller: min-combine of the keys -> (g1, g2))
  //   round_phase2  component bounds from (g1, g2), phase-2 list (identical on every
  //                 rank), (g1, g2) -> (b1, b2), exact scan of the share on top; the
  //                 tile-pair cache entries of this round's items gathered into a compact
  //                 buffer (caller: all-reduce MAX, then cache_scatter; min-combine of the
  //                 keys) -> finish_round
  int64_t rd_n1 = 0, rd_n2 = 0;
  int rd_stage = 0;  // 0 idle, 1 bound done, 2 phase 1 done, 3 phase 2 done (cache pending)
  const unsigned* caps_read = nullptr;  // caps the exact passes read (nullptr: none)
  DevBuf<unsigned> cachebuf;            // compact tile-pair cache entries of this round
  DevBuf<unsigned long long> G1, G2;    // combined keys (nnm_run_multi)
  DevBuf<unsigned> ucapg, cacheg;       // combined caps / cache entries (nnm_run_multi)

  static std::pair<int64_t, int64_t> share(int64_t total, int rank, int world) {
    return {total * rank / world, total * (rank + 1) / world};
  }

  void round_bound(int metric, int rank, int world) {
    if (world > 1 && rd_stage == 3)
      throw NnmError{NNM_E_INVALID, "staged round: the tile-pair cache of the previous round was "
                                    "not exchanged (nnm_bv_cache_scatter)"};
    ensure_geometry(metric);
    ++scan_epoch;
    tpmin_use = tpmin_on;  // exchanged every round (compact MAX), so consistent on all ranks
    tile_range.ensure(Tp);
    tile_range_kernel<<<Tp, TILE, 0, st>>>(comp.p, vn, Tp, tile_range.p); note_launch();
    int64_t n2 = 0;
    switch (metric) {
      case MANHATTAN: pruned_lists<MANHATTAN>(rd_n1, n2); break;
      case CHEBYSHEV: pruned_lists<CHEBYSHEV>(rd_n1, n2); break;
      default: pruned_lists<EUCLIDEAN>(rd_n1, n2);
    }
    // component caps (TC path): the bound pass over this rank's phase-1 share; both exact
    // scans then cap every row threshold by its component's (combined) upper bound, so
    // only rows that can still hold their component's minimum edge take exact inserts
    const char* cpe = getenv("NNM_TC_CAP");
    tc_cap_on = tc_on && !(cpe && cpe[0] == '0');
    caps_read = nullptr;
    if (tc_cap_on) {
      ucap.ensure(vn);
      fill_u32(ucap.p, vn, 0x7f800000u);  // +inf
      const auto sh = share(rd_n1, rank, world);
      NvtxRange r0("nnm phase-1 bound pass");
      tc_bound_only = true;
      if (sh.second > sh.first)
        scan(metric, B1.p, B2.p, true, INT_UNSET, INT_UNSET, bv_thr_hi, sh.first, sh.second, p1_list,
             false);
      tc_bound_only = false;
      caps_read = ucap.p;  // single rank: the local caps are the global ones
    }
    rd_stage = 1;
  }

  void round_phase1(unsigned long long* b1, unsigned long long* b2, int rank, int world) {
    if (rd_stage != 1) throw NnmError{NNM_E_INVALID, "staged round: phase 1 before the bound step"};
    fill_none(b1, vn);
    fill_none(b2, vn);
    capp_ready = false;
    if (tc_cap_on && caps_read) {  // per-position caps (staged per item by the scan)
      capp.ensure(vn);
      pos_caps_kernel<<<blocks_for(vn), 256, 0, st>>>(vn, comp.p, caps_read, capp.p); note_launch();
      CUDA_TRY(cudaGetLastError());
      capp_ready = true;
    }
    const auto sh = share(rd_n1, rank, world);
    NvtxRange r1("nnm phase-1 scan");
    if (sh.second > sh.first)
      scan(bv_metric, b1, b2, true, INT_UNSET, INT_UNSET, bv_thr_hi, sh.first, sh.second, p1_list,
           false);
    rd_stage = 2;
  }

  void round_phase2(const unsigned long long* g1, const unsigned long long* g2,
                    unsigned long long* b1, unsigned long long* b2, int rank, int world) {
    if (rd_stage != 2) throw NnmError{NNM_E_INVALID, "staged round: phase 2 before phase 1"};
    if (b1 != g1) CUDA_TRY(cudaMemcpyAsync(b1, g1, vn * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, st));
    if (b2 != g2) CUDA_TRY(cudaMemcpyAsync(b2, g2, vn * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, st));
    ucomp.ensure(vn);
    fill_none(ucomp.p, vn);
    switch (bv_metric) {
      case MANHATTAN: ucomp_t<MANHATTAN>(b1); pruned_phase2<MANHATTAN>(rd_n2); break;
      case CHEBYSHEV: ucomp_t<CHEBYSHEV>(b1); pruned_phase2<CHEBYSHEV>(rd_n2); break;
      default: ucomp_t<EUCLIDEAN>(b1); pruned_phase2<EUCLIDEAN>(rd_n2);
    }
    const auto sh = share(rd_n2, rank, world);
    {
      NvtxRange r2("nnm phase-2 scan");
      if (sh.second > sh.first)
        scan(bv_metric, b1, b2, true, INT_UNSET, INT_UNSET, bv_thr_hi, sh.first, sh.second, items2.p,
             false, tumax.p);
    }
    tc_cap_on = false;
    if (rank == 0) pairs_covered += (double)n * (double)(n - 1) / 2.0;
    rd_stage = 0;
    if (world > 1 && tpmin_use && rd_n1 + rd_n2 > 0) {
      // this round's scanned items (identical lists on every rank) -> compact cache buffer
      cachebuf.ensure(rd_n1 + rd_n2);
      cache_gather_kernel<<<blocks_for(rd_n1), 256, 0, st>>>(p1_list, rd_n1, Tp, tpmin.p, cachebuf.p); note_launch();
      if (rd_n2 > 0) { cache_gather_kernel<<<blocks_for(rd_n2), 256, 0, st>>>(items2.p, rd_n2, Tp, tpmin.p, cachebuf.p + rd_n1); note_launch(); }
      CUDA_TRY(cudaGetLastError());
      rd_stage = 3;
    }
    debug_lists(rd_n1, rd_n2);
  }

  // after the caller's all-reduce(MAX) of cachebuf: every rank holds the same cache
  void cache_scatter(const unsigned* src = nullptr) {
    if (rd_stage != 3) return;
    if (!src) src = cachebuf.p;
    cache_scatter_kernel<<<blocks_for(rd_n1), 256, 0, st>>>(p1_list, rd_n1, Tp, src, tpmin.p); note_launch();
    if (rd_n2 > 0) { cache_scatter_kernel<<<blocks_for(rd_n2), 256, 0, st>>>(items2.p, rd_n2, Tp, src + rd_n1, tpmin.p); note_launch(); }
    CUDA_TRY(cudaGetLastError());
    rd_stage = 0;
  }

  void debug_lists(int64_t n1, int64_t n2) {
    const char* dbg_env = getenv("NNM_DEBUG");
    if (dbg_env && atoi(dbg_env) >= 2) {  // list statistics (expensive host copies)
      const int T = Tp;
      std::vector<double> rad(T), um(T);
      CUDA_TRY(cudaMemcpyAsync(rad.data(), tradius.p, T * sizeof(double), cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaMemcpyAsync(um.data(), tumax.p, T * sizeof(double), cudaMemcpyDeviceToHost, st));
      sync();
      std::vector<double> r2 = rad, u2 = um;
      std::sort(r2.begin(), r2.end());
      std::sort(u2.begin(), u2.end());
      int ninf = 0;
      for (double u : um) ninf += std::isinf(u);
      {
        const int64_t n = vn;
        std::vector<unsigned long long> uc(n), b1(n);
        std::vector<int> cp(n);
        CUDA_TRY(cudaMemcpyAsync(uc.data(), ucomp.p, n * 8, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaMemcpyAsync(cp.data(), comp.p, n * 4, cudaMemcpyDeviceToHost, st));
        sync();
        std::vector<double> uv;
        int64_t none = 0;
        for (int64_t i = 0; i < n; ++i) {
          if (cp[i] < 0) continue;
          unsigned long long u = uc[cp[i]];
          if (u == NONE_KEY) ++none; else uv.push_back(bits_to_double(u));
        }
        std::sort(uv.begin(), uv.end());
        if (!uv.empty())
          fprintf(stderr, "[nnm]   point U: p10 %.3g p50 %.3g p90 %.3g p99 %.3g none %lld\n", uv[uv.size() / 10],
                  uv[uv.size() / 2], uv[uv.size() * 9 / 10], uv[uv.size() * 99 / 100], (long long)none);
        std::vector<int2> it1(n1);
        CUDA_TRY(cudaMemcpyAsync(it1.data(), p1_list, n1 * sizeof(int2), cudaMemcpyDeviceToHost, st));
        sync();
        int64_t diag = 0;
        for (auto& q : it1) diag += (q.x == q.y);
        fprintf(stderr, "[nnm]   phase1 diag items %lld\n", (long long)diag);
      }
      fprintf(stderr, "[nnm] round %d: phase1 %lld items, phase2 %lld of %lld tile pairs (%.3f%%); radius p50 %.3g p90 %.3g max %.3g; umax p50 %.3g p90 %.3g inf %d/%d\n",
              bv_round + 1, (long long)n1, (long long)n2, (long long)tile_pairs(), 100.0 * n2 / tile_pairs(),
              r2[T / 2], r2[T * 9 / 10], r2[T - 1], u2[T / 2], u2[T * 9 / 10], ninf, T);
    }
  }

  template <int M>
  void refine_t(const unsigned long long* b1, const unsigned long long* b2) {
    refine_kernel<M><<<blocks_for(vn), 256, 0, st>>>(X64p.p, (int)vn, d, b1, b2, normp.p, maxnormp, em,
                                                    bv_thr, rb_d.p, rb_j.p, rowlow.p, amb.p,
                                                    counters.p + 1, porig.p, (dot_on || tc_on) ? 1 : 0); note_launch();
  }

  int64_t bv_finish_round(const unsigned long long* b1, const unsigned long long* b2) {
    NvtxRange nv("nnm finish round (refine, component minima, hook, jump)");
    const int N = (int)vn;  // positions of the Boruvka view (pads carry comp -1)
    ++bv_round;
    // counters[0]: edges (cumulative), [1]: ambiguous, [2]: rescan rows
    CUDA_TRY(cudaMemsetAsync(counters.p + 1, 0, 2 * sizeof(unsigned long long), st));
    switch (bv_metric) {
      case MANHATTAN: refine_t<MANHATTAN>(b1, b2); break;
      case CHEBYSHEV: refine_t<CHEBYSHEV>(b1, b2); break;
      default: refine_t<EUCLIDEAN>(b1, b2);
    }
    CUDA_TRY(cudaGetLastError());
    fill_none(cmin_d.p, vn);
    compmin_d_kernel<<<blocks_for(vn), 256, 0, st>>>(N, comp.p, rb_d.p, cmin_d.p); note_launch();
    CUDA_TRY(cudaGetLastError());
    unsigned long long n_amb = read1(counters.p + 1);
    stats.ambiguous_rows += (int64_t)n_amb;
    if (n_amb > 0) {
      amb_filter_kernel<<<blocks_for(n_amb), 256, 0, st>>>(amb.p, (int)n_amb, comp.p, rowlow.p,
                                                         cmin_d.p, rb_d.p, bv_thr, normp.p, maxnormp,
                                                         em, resc.p, resc_bound.p, counters.p + 2); note_launch();
      CUDA_TRY(cudaGetLastError());
      unsigned long long n_res = read1(counters.p + 2);
      if (n_res > 0) {
        int64_t np = collect(bv_metric, resc.p, (int)n_res, resc_bound.p, nullptr, N, 0, INT_UNSET,
                             INT_UNSET);
        reset_rows_kernel<<<blocks_for(n_res), 256, 0, st>>>(resc.p, (int)n_res, rb_d.p, rb_j.p); note_launch();
        exact_pairs(bv_metric, np);
        if (np > 0) {
          rowmin_d_kernel<<<blocks_for(np), 256, 0, st>>>(pairs.p, pair_d.p, np, bv_thr, rb_d.p); note_launch();
          rowmin_j_kernel<<<blocks_for(np), 256, 0, st>>>(pairs.p, pair_d.p, np, bv_thr, rb_d.p,
                                                          rb_j.p, porig.p); note_launch();
        }
        fix_rows_kernel<<<blocks_for(n_res), 256, 0, st>>>(resc.p, (int)n_res, rb_d.p, rb_j.p); note_launch();
        CUDA_TRY(cudaGetLastError());
        // recompute component minima with the resolved rows
        fill_none(cmin_d.p, vn);
        compmin_d_kernel<<<blocks_for(vn), 256, 0, st>>>(N, comp.p, rb_d.p, cmin_d.p); note_launch();
      }
    }
    fill_none(cmin_ab.p, vn);
    compmin_ab_kernel<<<blocks_for(vn), 256, 0, st>>>(N, comp.p, rb_d.p, rb_j.p, cmin_d.p, cmin_ab.p, porig.p); note_launch();
    unsigned long long before = read1(counters.p);
    hook_kernel<<<blocks_for(vn), 256, 0, st>>>(N, comp.p, cmin_d.p, cmin_ab.p, parent.p, edges.p,
                                               counters.p, bv_round, ppos.p); note_launch();
    CUDA_TRY(cudaGetLastError());
    // every component root follows its hook chain to the final root (concurrent path
    // halving, benign: links only move towards roots) -- one launch, no host round trips
    if (getenv("NNM_JUMP_LOOP")) {
      for (int it = 0; it < 64; ++it) {
        CUDA_TRY(cudaMemsetAsync(flag.p, 0, sizeof(int), st));
        jump_kernel<<<blocks_for(vn), 256, 0, st>>>(N, comp.p, parent.p, flag.p); note_launch();
        if (read1(flag.p) == 0) break;
      }
    } else {
      resc.ensure(vn);  // scratch: final roots
      find_roots_kernel<<<blocks_for(vn), 256, 0, st>>>(N, comp.p, parent.p, resc.p); note_launch();
      CUDA_TRY(cudaGetLastError());
      CUDA_TRY(cudaMemcpyAsync(parent.p, resc.p, vn * sizeof(int), cudaMemcpyDeviceToDevice, st));
    }
    CUDA_TRY(cudaGetLastError());
    relabel_kernel<<<blocks_for(vn), 256, 0, st>>>(N, comp.p, parent.p); note_launch();
    CUDA_TRY(cudaGetLastError());
    unsigned long long after = read1(counters.p);
    int64_t added = (int64_t)(after - before);
    bv_ncomp -= added;
    stats.boruvka_rounds = bv_round;
    return added;
  }

  // dense exact Boruvka for small inputs (small_boruvka_kernel); leaves the MST edges in
  // `edges` / counters[0] for bv_end.  Returns false when the device cannot run it.
  bool small_boruvka(int metric, double dmax, bool screened) {
    if (screened) {
      ensure_norms(metric);
      if (!(maxnorm < 1e30)) return false;  // FP32 coordinates could overflow: general path
    }
    bv_metric = metric;
    bv_round = 0;
    const double thr = std::isnan(dmax) ? INFINITY : (metric == EUCLIDEAN ? dmax * dmax : dmax);
    comp.ensure(n);
    parent.ensure(n);
    rb_d.ensure(n);
    cmin_ab.ensure(n);
    cmin_d.ensure(n);
    B1.ensure(n);
    edges.ensure(std::max<int64_t>(n - 1, 1));
    counters.ensure(8);
    CUDA_TRY(cudaMemsetAsync(counters.p, 0, 8 * sizeof(unsigned long long), st));
    void* kfn = nullptr;
    if (screened) {
      if (d <= 8) {
        switch (metric) {
          case MANHATTAN: kfn = (void*)small_screened_kernel<MANHATTAN, 8, 8>; break;
          case CHEBYSHEV: kfn = (void*)small_screened_kernel<CHEBYSHEV, 8, 8>; break;
          default: kfn = (void*)small_screened_kernel<EUCLIDEAN, 8, 8>;
        }
      } else if (d <= 16) {
        switch (metric) {
          case MANHATTAN: kfn = (void*)small_screened_kernel<MANHATTAN, 16, 4>; break;
          case CHEBYSHEV: kfn = (void*)small_screened_kernel<CHEBYSHEV, 16, 4>; break;
          default: kfn = (void*)small_screened_kernel<EUCLIDEAN, 16, 4>;
        }
      } else {
        return false;
      }
    } else if (d <= 8) {
      switch (metric) {
        case MANHATTAN: kfn = (void*)small_boruvka_kernel<MANHATTAN, 8, 4>; break;
        case CHEBYSHEV: kfn = (void*)small_boruvka_kernel<CHEBYSHEV, 8, 4>; break;
        default: kfn = (void*)small_boruvka_kernel<EUCLIDEAN, 8, 4>;
      }
    } else if (d <= 16) {
      switch (metric) {
        case MANHATTAN: kfn = (void*)small_boruvka_kernel<MANHATTAN, 16, 2>; break;
        case CHEBYSHEV: kfn = (void*)small_boruvka_kernel<CHEBYSHEV, 16, 2>; break;
        default: kfn = (void*)small_boruvka_kernel<EUCLIDEAN, 16, 2>;
      }
    } else {
      return false;
    }
    int occ = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, 256, 0));
    if (occ < 1) return false;
    const int rpb = d <= 8 ? 32 : 16;
    int64_t want = (n + rpb - 1) / rpb;  // dense: row passes of 8 warps x R rows
    if (screened) {  // work units of R rows x SMALL_CW columns, 8 warps per block
      const int64_t R = d <= 8 ? 8 : 4;
      want = ((n + R - 1) / R * ((n + SMALL_CW - 1) / SMALL_CW) + 7) / 8;
    }
    const int grid = (int)std::min<int64_t>(sms * occ, std::max<int64_t>(1, want));
    const double* x = X64.p;
    int nn = (int)n, dd = d, maxr = 64;
    int *pc = comp.p, *pp = parent.p;
    unsigned long long *prbd = rb_d.p, *prbab = B1.p, *pcmd = cmin_d.p, *pcmab = cmin_ab.p,
                       *pctl = counters.p;
    Edge* pe = edges.p;
    double th = thr;
    void* args[] = {&x, &nn, &dd, &th, &maxr, &pc, &pp, &prbd, &prbab, &pcmd, &pcmab, &pe, &pctl};
    const float* x32 = X32.p;
    int64_t ldd = ld;
    const double* pn = norm.p;
    double mn = maxnorm;
    ErrModel e = make_err_model(metric, d);
    float *ppv1 = nullptr, *ppv2 = nullptr;
    int *ppj1 = nullptr, *pneed = nullptr, *proot = nullptr;
    float2* pdup = nullptr;
    if (screened) {
      sm_dup.ensure((size_t)n * (d <= 8 ? 8 : 16));
      pdup = sm_dup.p;
      const int64_t parts = (n + SMALL_CW - 1) / SMALL_CW * n;
      sm_v1.ensure(parts);
      sm_v2.ensure(parts);
      sm_j1.ensure(parts);
      sm_need.ensure(n);
      resc.ensure(n);
      ppv1 = sm_v1.p;
      ppv2 = sm_v2.p;
      ppj1 = sm_j1.p;
      pneed = sm_need.p;
      proot = resc.p;
    }
    void* sargs[] = {&x, &x32, &ldd, &nn, &dd, &th, &pn, &mn, &e, &maxr, &pc, &pp,
                     &prbd, &prbab, &pcmd, &pcmab, &pe, &pctl, &ppv1, &ppv2, &ppj1, &pneed, &proot, &pdup};
    CUDA_TRY(cudaEventRecord(ev0, st));
    CUDA_TRY(cudaLaunchCooperativeKernel(kfn, grid, 256, screened ? sargs : args, 0, st));
    note_launch();
    CUDA_TRY(cudaEventRecord(ev1, st));
    unsigned long long h[5];
    CUDA_TRY(cudaMemcpyAsync(h, counters.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    sync();
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, ev0, ev1));
    stats.scan_ms += ms;
    stats.scans += 1;
    stats.pairs_evaluated += (double)h[4] / 2.0;  // each unordered pair from both rows
    pairs_covered += (double)h[3] * (double)n * (double)(n - 1) / 2.0;
    bv_round = (int)h[3];
    stats.boruvka_rounds = bv_round;
    bv_ncomp = n - (int64_t)h[0];
    return true;
  }

  // sort edges by (d, a, b) and replay them through a min-root union-find
  // (model.py:109-187, engine.py:90-143): the kept root is the smaller index, roots are
  // always the minimum index of their cluster.  The replay runs on the GPU
  // (nnm_replay.cu: rank chunks, component-parallel); a chunk whose longest component
  // exceeds lmax -- and everything after it -- is finished by the sequential host loop.
  void bv_end(int64_t kl1, nnm_merge* out, int64_t* n_merges, int64_t* assign, int64_t* rounds,
              int32_t* stop) {
    NvtxRange nv("nnm merge replay");
    const unsigned long long ne = read1(counters.p);
    auto stop_of = [&](int64_t c) -> int {
      if (c == 1) return NNM_STOP_SINGLE_CLUSTER;
      if (kl1 >= 0 && c <= kl1) return NNM_STOP_KL1;
      return 0;
    };
    // the reference stops at the first count that is a stop reason (engine.py:139-142)
    const int64_t floor_count = (kl1 >= 0) ? std::max<int64_t>(kl1, 1) : 1;
    const int64_t m = stop_of(n) ? 0 : std::min<int64_t>((int64_t)ne, std::max<int64_t>(n - floor_count, 0));
    auto tq0 = std::chrono::steady_clock::now();
    ReplayEdge* h = nullptr;
    const char* ge = getenv("NNM_GPU_REPLAY");
    const bool gpu = m >= 32768 && !(ge && ge[0] == '0');
    // page-locked outputs (nnm_host_alloc, the engine's default): the GPU writes the merge
    // records and labels and the copy engine moves them; the host only replays a tail
    const char* pe_ = getenv("NNM_PINNED_OUT");
    const bool pin_out = gpu && !(pe_ && pe_[0] == '0') && is_page_locked(out) &&
                         is_page_locked(assign);
    if (ne > 0) {
      thrust::sort(thrust::cuda::par(talloc).on(st), edges.p, edges.p + ne, EdgeLess());
      replay.ensure(ne);
      replay_edges_kernel<<<blocks_for((int64_t)ne), 256, 0, st>>>(edges.p, (int64_t)ne,
                                                                   bv_metric == EUCLIDEAN ? 1 : 0,
                                                                   replay.p); note_launch();
      CUDA_TRY(cudaGetLastError());
      h = host_replay.ensure(ne);
      if (!pin_out) {
        // the 24-byte records travel on the side stream while the replay kernels run
        CUDA_TRY(cudaEventRecord(ev2, st));
        CUDA_TRY(cudaStreamWaitEvent(st2, ev2, 0));
        CUDA_TRY(cudaMemcpyAsync(h, replay.p, ne * sizeof(ReplayEdge), cudaMemcpyDeviceToHost, st2));
      }
    }
    const bool dbg = getenv("NNM_DEBUG") != nullptr;
    auto lap = [&](const char* what) {
      if (!dbg) return;
      sync();
      fprintf(stderr, "[nnm]   replay %s at %.2f ms\n", what,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tq0).count());
    };
    lap("sorted");
    int32_t* RK = h_rk.ensure(std::max<int64_t>(m, 1));
    int32_t* RD = h_rd.ensure(std::max<int64_t>(m, 1));
    int32_t* RS = h_rs.ensure(std::max<int64_t>(m, 1));
    int32_t* AS = nullptr;  // labels from the GPU (nullptr: host finds)
    int64_t host_from = 0;  // first merge replayed on the host
    int64_t early_n = 0;    // records copied out while the second replay graph ran
    int64_t rec_from = 0;   // first merge record the host writes
    bool gpu_assign = false;  // labels written to `assign` by the copy engine
    replay_host_buffers();
    int32_t* par = rp_par.p;
    int32_t* sz = rp_sz.p;
    auto tq1 = tq0;
    if (gpu) {
      const char* ce = getenv("NNM_REPLAY_CHUNKS");
      const char* le = getenv("NNM_REPLAY_LMAX");
      const int64_t nchunks = std::max<int64_t>(1, ce ? atoll(ce) : 24);
      const int lmax = std::min(REPLAY_LMAX, le ? std::max(1, atoi(le)) : REPLAY_LMAX);
      // chunk plan: uniform chunks over the first 7/8 of the ranks, then each chunk half
      // of what is left (>= 1024 edges) -- the top of a blob dendrogram (the edges that
      // join the blobs) is one component, so the host tail starts as late as possible
      std::vector<std::pair<int64_t, int>> plan;
      {
        const int64_t C = std::max<int64_t>(32768, (m + nchunks - 1) / nchunks);
        const int64_t head_end = m - m / 8;
        int64_t lo = 0;
        while (lo < head_end) {
          const int64_t c = std::min<int64_t>(C, head_end - lo);
          plan.emplace_back(lo, (int)c);
          lo += c;
        }
        while (lo < m) {
          const int64_t c = std::min<int64_t>(m - lo, std::max<int64_t>(1024, (m - lo) / 2));
          plan.emplace_back(lo, (int)c);
          lo += c;
        }
      }
      int cmax_chunk = 0;
      for (auto& pc : plan) cmax_chunk = std::max(cmax_chunk, pc.second);
      r_par.ensure(n);
      r_sz.ensure(n);
      r_lab.ensure(n);
      r_head.ensure(n);
      r_ea.ensure(cmax_chunk);
      r_eb.ensure(cmax_chunk);
      r_nxt.ensure(cmax_chunk);
      r_comp.ensure(cmax_chunk);
      r_ctl.ensure(8);
      r_base.ensure(n);
      r_slot.ensure(cmax_chunk);
      r_rid.ensure(n);
      r_rcnt.ensure(n);
      r_llist.ensure(cmax_chunk);
      r_rk.ensure(m);
      r_rd.ensure(m);
      r_rs.ensure(m);
      ReplayState rs{r_par.p, r_sz.p, r_lab.p, r_head.p, r_ea.p, r_eb.p, r_nxt.p, r_comp.p,
                     r_ctl.p, r_rk.p, r_rd.p, r_rs.p, r_base.p, r_slot.p, r_rid.p, r_rcnt.p,
                     r_llist.p};
      const int64_t nch = (int64_t)plan.size();
      const char* gre = getenv("NNM_REPLAY_GRAPH");
      const bool use_graph = !dbg && !(gre && gre[0] == '0');
      if (use_graph) {
        // fixed launch topology for this (state, m, plan): captured once, replayed after
        const bool same = rp_exec && rp_m == m && rp_n == n && rp_lmax == lmax &&
                          rp_e == replay.p && rp_nch == nch &&
                          memcmp(&rp_state, &rs, sizeof(rs)) == 0;
        if (!same) {
          // two graphs: the chunks before rp_split, then the rest, so that the records of
          // the first part can be copied out while the second part runs (page-locked
          // outputs, below)
          for (cudaGraphExec_t* ex : {&rp_exec, &rp_exec2}) {
            if (*ex) cudaGraphExecDestroy(*ex);
            *ex = nullptr;
          }
          rp_split = nch / 2;
          for (int part = 0; part < 2; ++part) {
            cudaGraph_t gr = nullptr;
            CUDA_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            cudaError_t ce2 = part == 0 ? replay_init(n, rs, st) : cudaSuccess;
            for (int64_t c = part == 0 ? 0 : rp_split; c < (part == 0 ? rp_split : nch); ++c)
              if (ce2 == cudaSuccess)
                ce2 = replay_chunk(replay.p, plan[c].first, plan[c].second, lmax, rs, st);
            const cudaError_t ce3 = cudaStreamEndCapture(st, &gr);
            CUDA_TRY(ce2);
            CUDA_TRY(ce3);
            const cudaError_t ce4 = cudaGraphInstantiate(part == 0 ? &rp_exec : &rp_exec2, gr, 0);
            cudaGraphDestroy(gr);
            CUDA_TRY(ce4);
          }
          rp_m = m;
          rp_n = n;
          rp_lmax = lmax;
          rp_e = replay.p;
          rp_nch = nch;
          rp_state = rs;
        }
        CUDA_TRY(cudaGraphLaunch(rp_exec, st));
        early_n = rp_split < nch ? plan[rp_split].first : m;
        if (pin_out && early_n > 0) {
          // records of the first part (final unless the GPU stopped there: then the host
          // tail overwrites them after this copy has completed, see st2 below)
          rec_dev.ensure(m);
          CUDA_TRY(cudaEventRecord(ev2, st));
          CUDA_TRY(cudaStreamWaitEvent(st2, ev2, 0));
          merge_records_kernel<<<blocks_for(early_n), 256, 0, st2>>>(replay.p, early_n, r_rk.p,
                                                                      r_rd.p, r_rs.p, rec_dev.p);
          note_launch();
          CUDA_TRY(cudaGetLastError());
          CUDA_TRY(cudaMemcpyAsync(out, rec_dev.p, early_n * sizeof(nnm_merge),
                                   cudaMemcpyDeviceToHost, st2));
        } else {
          early_n = 0;
        }
        if (rp_exec2) CUDA_TRY(cudaGraphLaunch(rp_exec2, st));
      } else {
        CUDA_TRY(replay_init(n, rs, st));
        DevBuf<int> cmax;
        if (dbg) {
          cmax.ensure(nch);
          CUDA_TRY(cudaMemsetAsync(cmax.p, 0, nch * sizeof(int), st));
        }
        for (int64_t c = 0; c < nch; ++c)
          CUDA_TRY(replay_chunk(replay.p, plan[c].first, plan[c].second, lmax, rs, st,
                                dbg ? cmax.p + c : nullptr));
        if (dbg) {
          std::vector<int> hc(nch);
          CUDA_TRY(cudaMemcpyAsync(hc.data(), cmax.p, nch * sizeof(int), cudaMemcpyDeviceToHost, st));
          sync();
          fprintf(stderr, "[nnm]   replay chunks (size:longest component):");
          for (int64_t c = 0; c < nch; ++c) fprintf(stderr, " %d:%d", plan[c].second, hc[c]);
          fprintf(stderr, "\n");
        }
      }
      g_launches.fetch_add(1 + 7 * nch, std::memory_order_relaxed);
      lap("chunks");
      int ctl[4];
      CUDA_TRY(cudaMemcpyAsync(ctl, r_ctl.p, sizeof(ctl), cudaMemcpyDeviceToHost, st));
      sync();
      if (ctl[3]) throw NnmError{NNM_E_CUDA, "boruvka produced a cycle (internal error)"};
      host_from = ctl[1] < 0 ? m : ctl[1];
      stats.replay_gpu_merges = host_from;
      if (pin_out) {
        // the host tail needs the forest as the GPU left it and its own edges (side stream)
        if (host_from < m) {
          CUDA_TRY(cudaMemcpyAsync(par, r_par.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st2));
          CUDA_TRY(cudaMemcpyAsync(sz, r_sz.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st2));
          CUDA_TRY(cudaMemcpyAsync(h + host_from, replay.p + host_from,
                                   (m - host_from) * sizeof(ReplayEdge), cudaMemcpyDeviceToHost, st2));
        }
        // records [0, host_from) on the GPU, straight into the caller's page-locked array
        // (the first early_n already on their way, above)
        const int64_t r0 = std::min(early_n, host_from);
        if (host_from > r0) {
          rec_dev.ensure(m);
          merge_records_kernel<<<blocks_for(host_from - r0), 256, 0, st>>>(
              replay.p + r0, host_from - r0, r_rk.p + r0, r_rd.p + r0, r_rs.p + r0, rec_dev.p + r0);
          note_launch();
          CUDA_TRY(cudaGetLastError());
          CUDA_TRY(cudaMemcpyAsync(out + r0, rec_dev.p + r0, (host_from - r0) * sizeof(nnm_merge),
                                   cudaMemcpyDeviceToHost, st));
        }
        rec_from = host_from;
        gpu_assign = true;
        if (host_from == m) {
          as_dev.ensure(n);
          assign64_kernel<<<blocks_for(n), 256, 0, st>>>(n, r_par.p, as_dev.p);
          note_launch();
          CUDA_TRY(cudaGetLastError());
          CUDA_TRY(cudaMemcpyAsync(assign, as_dev.p, n * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        }
        CUDA_TRY(cudaStreamSynchronize(st2));
      } else {
        if (host_from > 0) {
          CUDA_TRY(cudaMemcpyAsync(RK, r_rk.p, host_from * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
          CUDA_TRY(cudaMemcpyAsync(RD, r_rd.p, host_from * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
          CUDA_TRY(cudaMemcpyAsync(RS, r_rs.p, host_from * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        }
        if (host_from == m) {
          AS = h_as.ensure(n);
          CUDA_TRY(replay_assign(n, rs, r_lab.p, st));
          note_launch();
          CUDA_TRY(cudaMemcpyAsync(AS, r_lab.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        } else {  // host finishes: the forest as the GPU left it (state at chunk start)
          CUDA_TRY(cudaMemcpyAsync(par, r_par.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
          CUDA_TRY(cudaMemcpyAsync(sz, r_sz.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        }
        sync();
      }
      if (dbg)
        fprintf(stderr, "[nnm] gpu replay: %lld of %lld merges, %lld chunks, longest component %d\n",
                (long long)host_from, (long long)m, (long long)nch, ctl[2]);
    } else {
      for (int64_t i = 0; i < n; ++i) {
        par[i] = (int32_t)i;
        sz[i] = 1;
      }
    }
    CUDA_TRY(cudaStreamSynchronize(st2));
    tq1 = std::chrono::steady_clock::now();
    if (host_from < m) {
      auto find = [&](int32_t x) {
        while (par[x] != x) {
          par[x] = par[par[x]];
          x = par[x];
        }
        return x;
      };
      int2* links = pin_out ? rp_links.ensure(m - host_from) : nullptr;
      constexpr int64_t kAhead = 16;  // prefetch the forest entries of later merges
      for (int64_t t = host_from; t < m; ++t) {
        if (t + kAhead < m) {
          __builtin_prefetch(&par[h[t + kAhead].a], 1);
          __builtin_prefetch(&par[h[t + kAhead].b], 1);
        }
        const ReplayEdge& e = h[t];
        const int32_t ra = find(e.a), rb = find(e.b);
        if (ra == rb) throw NnmError{NNM_E_CUDA, "boruvka produced a cycle (internal error)"};
        const int32_t keep = std::min(ra, rb), drop = std::max(ra, rb);
        par[drop] = keep;
        sz[keep] += sz[drop];
        RK[t] = keep;
        RD[t] = drop;
        RS[t] = sz[keep];
        if (links) links[t - host_from] = make_int2(drop, keep);
      }
      if (pin_out) {  // labels on the GPU: its forest plus the tail's links
        const int64_t nl = m - host_from;
        links_dev.ensure(nl);
        as_dev.ensure(n);
        CUDA_TRY(cudaMemcpyAsync(links_dev.p, links, nl * sizeof(int2), cudaMemcpyHostToDevice, st));
        apply_links_kernel<<<blocks_for(nl), 256, 0, st>>>(links_dev.p, nl, r_par.p);
        assign64_kernel<<<blocks_for(n), 256, 0, st>>>(n, r_par.p, as_dev.p);
        g_launches.fetch_add(2, std::memory_order_relaxed);
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaMemcpyAsync(assign, as_dev.p, n * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      }
    }
    const int64_t nm = m;
    const int reason = (n > 0 && stop_of(n - nm)) ? stop_of(n - nm) : NNM_STOP_NO_ELIGIBLE;
    auto tq2 = std::chrono::steady_clock::now();
    // merge records and labels in parallel (read-only finds: the forest is final)
    const int64_t nrec = nm - rec_from;
    const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(8, std::min<int64_t>(
                       (int64_t)std::thread::hardware_concurrency(),
                       ((gpu_assign ? nrec : std::max<int64_t>(n, nrec)) >> 16) + 1)));
    auto work = [&](int t) {
      const int64_t m0 = rec_from + nrec * t / nt, m1 = rec_from + nrec * (t + 1) / nt;
      for (int64_t k = m0; k < m1; ++k) {
        const ReplayEdge& e = h[k];
        nnm_merge& mg = out[k];
        mg.round = e.round;
        mg.root_a = RK[k];
        mg.root_b = RD[k];
        mg.dist = e.dist;  // reported units (metrics.py:86-90)
        mg.new_size = RS[k];
        mg.point_a = e.a;
        mg.point_b = e.b;
      }
      if (gpu_assign) return;
      const int64_t i0 = n * t / nt, i1 = n * (t + 1) / nt;
      if (AS) {
        for (int64_t i = i0; i < i1; ++i) assign[i] = AS[i];
      } else {
        for (int64_t i = i0; i < i1; ++i) {
          int32_t x = (int32_t)i;
          while (par[x] != x) x = par[x];
          assign[i] = x;
        }
      }
    };
    if (nt == 1) {
      work(0);
    } else {
      std::vector<std::thread> pool;
      for (int t = 1; t < nt; ++t) pool.emplace_back(work, t);
      work(0);
      for (auto& th : pool) th.join();
    }
    if (pin_out) sync();  // the copy engine's records and labels
    *n_merges = nm;
    *rounds = (n > 1 && stop_of(n) == 0) ? bv_round : 0;
    *stop = reason;
    if (getenv("NNM_DEBUG"))
      fprintf(stderr, "[nnm] replay: device %.1f ms, host loop %.1f ms, records %.1f ms%s\n",
              std::chrono::duration<double, std::milli>(tq1 - tq0).count(),
              std::chrono::duration<double, std::milli>(tq2 - tq1).count(),
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tq2).count(),
              pin_out ? " (page-locked outputs)" : "");
  }

  // ---------------------------------------------------------------- top-P
  // Exact top-P eligible pairs for the current (comp, psize) snapshot.
  template <int M>
  void rowpairs_t(const unsigned long long* b1, double thr, unsigned long long* cnt,
                  const int* psz, int ksum) {
    rowpairs_kernel<M><<<blocks_for(n), 256, 0, st>>>(X64.p, (int)n, d, b1, thr, cands.p, cnt,
                                                     comp.p, psz, ksum); note_launch();
  }

  // Exact top-P eligible pairs for the current (comp, psize) snapshot.
  //   * rB1: per-row best screened key over eligible partners (full FP32 scan);
  //   * tau: P-th smallest exact row-best pair (an upper bound of the P-th key);
  //   * every top-P pair has both endpoints in A = {i : exact_lower(rB1_i) <= tau};
  //     the A x A pairs under the screened bound are evaluated exactly, sorted, cut at P.
  // reuse (rounds of one run): eligibility only shrinks as clusters merge, so the rB1 of
  // an earlier snapshot still bounds every eligible partner from below and its row-best
  // pairs that are still eligible are real candidates: the full scan is skipped until
  // A grows past n/6 (NNM_REUSE_DIV; or fewer than P row-best pairs survive) -- SURVEY 8(f) rank 2.
  bool top_p_pass(int metric, double thr, int kl2, int kl3, int64_t P, const int* psz, int ksum,
                  int64_t max_active, std::vector<Cand>& out) {
    counters.ensure(8);
    cands.ensure(n);
    CUDA_TRY(cudaMemsetAsync(counters.p + 3, 0, 3 * sizeof(unsigned long long), st));
    switch (metric) {
      case MANHATTAN: rowpairs_t<MANHATTAN>(rB1.p, thr, counters.p + 3, psz, ksum); break;
      case CHEBYSHEV: rowpairs_t<CHEBYSHEV>(rB1.p, thr, counters.p + 3, psz, ksum); break;
      default: rowpairs_t<EUCLIDEAN>(rB1.p, thr, counters.p + 3, psz, ksum);
    }
    CUDA_TRY(cudaGetLastError());
    int64_t nc = (int64_t)read1(counters.p + 3);
    stats.exact_evals += nc;
    double tau = INFINITY;
    if (nc >= P) {
      // tau = the P-th smallest candidate distance, rounded up to fp32: a radix sort of
      // 32-bit keys instead of a merge sort of the 16-byte candidates
      ckeys.ensure(nc);
      ckeys2.ensure(nc);
      cand_keys_kernel<<<blocks_for(nc), 256, 0, st>>>(cands.p, nc, ckeys.p); note_launch();
      size_t tb = 0;
      CUDA_TRY(cub::DeviceRadixSort::SortKeys(nullptr, tb, ckeys.p, ckeys2.p, (int)nc, 0, 32, st));
      ctmp.ensure(std::max<size_t>(tb, 1));
      CUDA_TRY(cub::DeviceRadixSort::SortKeys(ctmp.p, tb, ckeys.p, ckeys2.p, (int)nc, 0, 32, st));
      tau = (double)read1(ckeys2.p + (P - 1));
    } else if (max_active < n) {
      return false;  // too few surviving row-best pairs: rescan
    }
    active.ensure(n);
    active_rows_kernel<<<blocks_for(n), 256, 0, st>>>((int)n, rB1.p, norm.p, maxnorm, em, tau,
                                                      active.p, counters.p + 4); note_launch();
    CUDA_TRY(cudaGetLastError());
    int64_t na = (int64_t)read1(counters.p + 4);
    if (na > max_active) return false;
    top_p_collect(metric, thr, kl2, kl3, P, tau, na, out);
    return true;
  }

  void top_p(int metric, double thr, int kl2, int kl3, int64_t P, std::vector<Cand>& out,
             bool reuse = false) {
    ensure_norms(metric);
    use_original_view();
    dot_on = false;
    em = make_err_model(metric, d);
    float thr_hi = std::isinf(thr) ? INFINITY : float_up(screen_upper(em, thr, 2.0 * maxnorm));
    rB1.ensure(n);
    const int ksum = size_rule(kl2, kl3);
    const char* re = getenv("NNM_ROUND_REUSE");
    if (reuse && rb1_valid && !(re && re[0] == '0')) {
      const int* psz = ksum != INT_UNSET ? eff_sizes(kl2) : comp.p;
      const char* rfe = getenv("NNM_REUSE_DIV");  // reuse while |A| <= n / div
      const int64_t div = rfe ? std::max(1, atoi(rfe)) : 6;  // C2 sweep: 4 528, 6 474, 8 491, 11 554 ms
      if (top_p_pass(metric, thr, kl2, kl3, P, psz, ksum, std::max<int64_t>(2 * P, n / div), out))
        return;
      ++stats.round_rescans;
    }
    scan(metric, rB1.p, nullptr, false, kl2, kl3, thr_hi, 0, tile_pairs());
    rb1_valid = true;
    const int* psz = ksum != INT_UNSET ? eff_sizes(kl2) : comp.p;
    top_p_pass(metric, thr, kl2, kl3, P, psz, ksum, n, out);
  }

  void top_p_collect(int metric, double thr, int kl2, int kl3, int64_t P, double tau, int64_t na,
                     std::vector<Cand>& out) {
    out.clear();
    if (na < 2) return;
    // deterministic order of the active set (atomics appended in arbitrary order)
    thrust::sort(thrust::cuda::par(talloc).on(st), active.p, active.p + na);
    double lim = std::min(tau, thr);
    float bound = float_up(screen_upper(em, lim, 2.0 * maxnorm));
    DevBuf<float> bnd;
    bnd.ensure(na);
    std::vector<float> hb(na, bound);
    CUDA_TRY(cudaMemcpyAsync(bnd.p, hb.data(), na * sizeof(float), cudaMemcpyHostToDevice, st));
    int64_t np = collect(metric, active.p, (int)na, bnd.p, active.p, (int)na, 1, kl2, kl3);
    exact_pairs(metric, np);
    cands2.ensure(std::max<int64_t>(np, 1));
    CUDA_TRY(cudaMemsetAsync(counters.p + 5, 0, sizeof(unsigned long long), st));
    if (np > 0)
      pairs_to_cands_kernel<<<blocks_for(np), 256, 0, st>>>(pairs.p, pair_d.p, np, lim, cands2.p,
                                                            counters.p + 5); note_launch();
    CUDA_TRY(cudaGetLastError());
    int64_t nk = (int64_t)read1(counters.p + 5);
    if (nk == 0) return;
    thrust::sort(thrust::cuda::par(talloc).on(st), cands2.p, cands2.p + nk, CandLess());
    int64_t take = std::min<int64_t>(nk, P);
    out.resize(take);
    CUDA_TRY(cudaMemcpyAsync(out.data(), cands2.p, take * sizeof(Cand), cudaMemcpyDeviceToHost, st));
    sync();
  }
};

// ----------------------------------------------------------------------------
// validation helpers (model.py:29-76, :190-218; engine.py:48-54)
// ----------------------------------------------------------------------------
namespace {
void check_metric(int32_t metric) {
  if (metric < 0 || metric > 3)
    invalid("unknown metric code " + std::to_string(metric) +
            "; choose one of: euclidean, squared-euclidean, manhattan, chebyshev");
}

void check_constraints(const nnm_constraints* c) {
  const char* names[4] = {"kl1", "kl2", "kl3", "kl4"};
  int64_t v[4] = {c->kl1, c->kl2, c->kl3, c->kl4};
  for (int i = 0; i < 4; ++i)
    if (v[i] == 0) invalid(std::string(names[i]) + " must be a positive count, got 0");
  if (c->kl2 >= 1 && c->kl3 >= 1 && !(c->kl3 > c->kl2))
    invalid("kl3 must exceed kl2, got kl3=" + std::to_string(c->kl3) + " kl2=" + std::to_string(c->kl2));
  if (!std::isnan(c->dmax) && !(c->dmax >= 0.0))
    invalid("dmax must be nonnegative, got " + std::to_string(c->dmax));
}

// kl2 / kl3 as kernel ints: a cap >= n never binds (two disjoint clusters hold <= n
// points), so clamp to n; the fused size rule needs n < 2^28 (SIZE_BIG = 2^29).
int clamp_int(int64_t v, int64_t n) {
  if (v < 0) return INT_UNSET;
  if (n >= (int64_t)1 << 28) throw NnmError{NNM_E_UNSUPPORTED, "kl2/kl3 need n < 2^28"};
  return (int)std::min<int64_t>(v, n);
}

void init_device(int32_t device, int* sms) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    throw NnmError{NNM_E_CUDA, "no CUDA device available (libnnm has no CPU fallback)"};
  if (device < 0 || device >= count) invalid("device index out of range");
  CUDA_TRY(cudaSetDevice(device));
  // device properties and the pool setting once per device (cudaGetDeviceProperties
  // queries every attribute: too slow for a per-call path)
  static std::mutex mu;
  static std::map<int, int> known_sms;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = known_sms.find(device);
    if (it != known_sms.end()) {
      *sms = it->second;
      return;
    }
  }
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10)
    throw NnmError{NNM_E_CUDA, std::string("libnnm is built for sm_100a; device is ") + prop.name};
  *sms = prop.multiProcessorCount;
  {
    std::lock_guard<std::mutex> lk(mu);
    known_sms[device] = prop.multiProcessorCount;
  }
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
}

// Host -> device copy of a large PAGEABLE array: the driver would stage it through a small
// bounce buffer at a fraction of the link rate.  Here T host threads copy slices into
// page-locked double buffers (pinned_pool) and each queues the DMA of its buffer on `st`,
// so the host copies overlap the transfers.  Page-locked sources go straight to the DMA.
void upload_h2d(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  constexpr size_t kChunk = (size_t)8 << 20;
  const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
  if (bytes < ((size_t)32 << 20) || is_page_locked(src)) {
    CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
    return;
  }
  const int T = std::max(1, std::min(8, hw / 2));
  const size_t nchunks = (bytes + kChunk - 1) / kChunk;
  std::vector<std::thread> pool;
  std::atomic<int> failed{0};
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  for (int t = 0; t < T; ++t) {
    pool.emplace_back([&, t] {
      cudaSetDevice(dev);
      void* buf[2] = {nullptr, nullptr};
      size_t bb[2] = {kChunk, kChunk};
      cudaEvent_t ev[2] = {nullptr, nullptr};
      bool used[2] = {false, false};
      try {
        for (int b = 0; b < 2; ++b) {
          buf[b] = pinned_pool().get(bb[b]);
          if (cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming) != cudaSuccess) throw 0;
        }
        int k = 0;
        for (size_t c = (size_t)t; c < nchunks; c += (size_t)T, k ^= 1) {
          const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
          if (used[k] && cudaEventSynchronize(ev[k]) != cudaSuccess) throw 0;
          memcpy(buf[k], (const char*)src + off, len);
          if (cudaMemcpyAsync((char*)dst + off, buf[k], len, cudaMemcpyHostToDevice, st) !=
                  cudaSuccess ||
              cudaEventRecord(ev[k], st) != cudaSuccess)
            throw 0;
          used[k] = true;
        }
        for (int b = 0; b < 2; ++b)
          if (used[b]) cudaEventSynchronize(ev[b]);
      } catch (...) {
        failed.store(1);
      }
      for (int b = 0; b < 2; ++b) {
        if (ev[b]) cudaEventDestroy(ev[b]);
        if (buf[b]) pinned_pool().put(buf[b], bb[b]);
      }
    });
  }
  for (auto& th : pool) th.join();
  if (failed.load()) throw NnmError{NNM_E_CUDA, "staged host-to-device upload failed"};
}

nnm_dataset* make_dataset(const double* X, bool on_device, int64_t n, int32_t d, int32_t device) {
  if (n < 1 || d < 1)
    invalid("dataset must have at least 1 point and 1 feature, got " + std::to_string(n) + "x" +
            std::to_string(d));
  if (n >= (int64_t)1 << 31) throw NnmError{NNM_E_UNSUPPORTED, "n must be < 2^31"};
  int sms = 0;
  init_device(device, &sms);
  auto* ds = new nnm_dataset();
  try {
    ds->device = device;
    ds->sms = sms;
    ds->n = n;
    ds->d = d;
    ds->ld = (n + TILE - 1) / TILE * TILE;
    ds->T = (int)(ds->ld / TILE);
    CUDA_TRY(cudaStreamCreateWithFlags(&ds->st, cudaStreamNonBlocking));
    ds->stream_holder.st = ds->st;
    t_alloc_stream = ds->st;
    CUDA_TRY(cudaEventCreate(&ds->ev0));
    CUDA_TRY(cudaEventCreate(&ds->ev1));
    CUDA_TRY(cudaEventCreateWithFlags(&ds->ev2, cudaEventDisableTiming));
    CUDA_TRY(cudaStreamCreateWithFlags(&ds->st2, cudaStreamNonBlocking));
    if ((size_t)ds->d * TILE * 2 * sizeof(float) + 8192 > 200 * 1024)
      throw NnmError{NNM_E_UNSUPPORTED, "d too large for the shared-memory tile (d <= 190)"};
    auto tc0 = std::chrono::steady_clock::now();
    ds->X64.ensure((size_t)n * d);
    if (on_device)
      CUDA_TRY(cudaMemcpyAsync(ds->X64.p, X, (size_t)n * d * sizeof(double),
                               cudaMemcpyDeviceToDevice, ds->st));
    else
      upload_h2d(ds->X64.p, X, (size_t)n * d * sizeof(double), ds->st);
    ds->X32.ensure((size_t)ds->ld * d);
    ds->flag.ensure(1);  // scratch flag of the view build / pointer jumping
    DevBuf<unsigned long long> chk;
    chk.ensure(2);
    const unsigned long long init[2] = {~0ull, 0ull};
    CUDA_TRY(cudaMemcpyAsync(chk.p, init, sizeof(init), cudaMemcpyHostToDevice, ds->st));
    prepare_kernel<<<blocks_for(ds->ld), 256, 0, ds->st>>>(ds->X64.p, n, d, ds->ld, ds->X32.p,
                                                          chk.p); note_launch();
    CUDA_TRY(cudaGetLastError());
    unsigned long long h[2];
    CUDA_TRY(cudaMemcpyAsync(h, chk.p, sizeof(h), cudaMemcpyDeviceToHost, ds->st));
    ds->sync();
    if (getenv("NNM_DEBUG"))
      fprintf(stderr, "[nnm] dataset create: alloc+upload+prepare %.2f ms\n",
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tc0).count());
    if (h[0] != ~0ull) invalid("non-finite feature value in row " + std::to_string(h[0] + 1));
    if (h[1])
      throw NnmError{NNM_E_UNSUPPORTED,
                     "feature magnitude above 1e18 is outside the FP32 screening range"};
  } catch (...) {
    delete ds;
    throw;
  }
  return ds;
}
}  // namespace

// ----------------------------------------------------------------------------
// C ABI
// ----------------------------------------------------------------------------
extern "C" {

int nnm_abi_version(void) { return NNM_ABI_VERSION; }

const char* nnm_last_error(void) { return g_err.c_str(); }

int nnm_device_count(int32_t* out) {
  return guarded([&] {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    *out = (e == cudaSuccess) ? c : 0;
  });
}

int nnm_host_alloc(int64_t bytes, void** out) {
  return guarded([&] {
    if (!out || bytes < 0) invalid("bad argument");
    size_t b = (size_t)std::max<int64_t>(bytes, 1);
    void* p = pinned_pool().get(b);
    std::lock_guard<std::mutex> lk(g_host_mu);
    g_host_blocks[p] = b;
    *out = p;
  });
}

int nnm_host_free(void* p) {
  return guarded([&] {
    if (!p) return;
    size_t b = 0;
    {
      std::lock_guard<std::mutex> lk(g_host_mu);
      auto it = g_host_blocks.find(p);
      if (it == g_host_blocks.end()) invalid("not a block from nnm_host_alloc");
      b = it->second;
      g_host_blocks.erase(it);
    }
    pinned_pool().put(p, b);
  });
}

int nnm_dataset_create(const double* X, int64_t n, int32_t d, int32_t device, nnm_dataset** out) {
  return guarded([&] {
    if (!X || !out) invalid("null argument");
    *out = make_dataset(X, false, n, d, device);
  });
}

int nnm_dataset_create_device(const double* X_dev, int64_t n, int32_t d, int32_t device,
                              nnm_dataset** out) {
  return guarded([&] {
    if (!X_dev || !out) invalid("null argument");
    *out = make_dataset(X_dev, true, n, d, device);
  });
}

int nnm_csv_load(const char* path, char delimiter, const char* id_column, int32_t threads,
                 nnm_csv** out, int64_t* n, int64_t* d, int32_t* has_ids, int64_t* id_bytes) {
  return guarded([&] {
    if (!path || !out) invalid("null argument");
    std::string err;
    nnm_csv* c = nullptr;
    if (nnm_csv_parse_impl(path, delimiter, id_column, threads, &c, err) != 0) invalid(err);
    *out = c;
    if (n) *n = nnm_csv_rows(c);
    if (d) *d = nnm_csv_cols(c);
    if (has_ids) *has_ids = nnm_csv_has_ids(c) ? 1 : 0;
    if (id_bytes) *id_bytes = nnm_csv_id_bytes(c);
  });
}

int nnm_csv_fetch(nnm_csv* c, double* values, char* id_buf, int64_t* id_offsets) {
  return guarded([&] {
    if (!c) invalid("null table");
    if (values) nnm_csv_copy_values(c, values);
    if (id_buf && id_offsets && nnm_csv_has_ids(c)) nnm_csv_copy_ids(c, id_buf, id_offsets);
  });
}

int nnm_csv_free(nnm_csv* c) {
  return guarded([&] { nnm_csv_destroy(c); });
}

int nnm_first_nonfinite(const double* X, int64_t count, int32_t threads, int64_t* out_index) {
  return guarded([&] {
    if ((!X && count > 0) || !out_index) invalid("null argument");
    if (count < 0) invalid("negative count");
    *out_index = count > 0 ? nnm_first_nonfinite_impl(X, count, threads) : -1;
  });
}

int nnm_round_log(nnm_dataset* ds, nnm_round_stat* out, int64_t cap, int64_t* out_n) {
  return guarded([&] {
    if (!ds || !out_n) invalid("null argument");
    std::lock_guard<std::mutex> lk(ds->mu);
    const int64_t k = (int64_t)ds->round_log.size();
    *out_n = k;
    if (out)
      for (int64_t i = 0; i < std::min(k, cap); ++i) out[i] = ds->round_log[i];
  });
}

int nnm_dataset_destroy(nnm_dataset* ds) {
  return guarded([&] {
    if (!ds) return;
    cudaSetDevice(ds->device);
    delete ds;
  });
}

int nnm_pairwise(int32_t metric, const double* x, int64_t nx, const double* y, int64_t ny,
                 int32_t d, int32_t device, double* out) {
  return guarded([&] {
    check_metric(metric);
    if (nx < 0 || ny < 0 || d < 1) invalid("bad shape");
    if (nx == 0 || ny == 0) return;
    int sms;
    init_device(device, &sms);
    DevBuf<double> dx, dy, dout;
    dx.ensure(nx * d);
    dy.ensure(ny * d);
    dout.ensure(nx * ny);
    CUDA_TRY(cudaMemcpy(dx.p, x, nx * d * sizeof(double), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(dy.p, y, ny * d * sizeof(double), cudaMemcpyHostToDevice));
    int64_t tot = nx * ny;
    switch (metric) {
      case MANHATTAN: pairwise_kernel<MANHATTAN><<<blocks_for(tot), 256>>>(dx.p, nx, dy.p, ny, d, dout.p); note_launch(); break;
      case CHEBYSHEV: pairwise_kernel<CHEBYSHEV><<<blocks_for(tot), 256>>>(dx.p, nx, dy.p, ny, d, dout.p); note_launch(); break;
      default: pairwise_kernel<EUCLIDEAN><<<blocks_for(tot), 256>>>(dx.p, nx, dy.p, ny, d, dout.p); note_launch();
    }
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpy(out, dout.p, tot * sizeof(double), cudaMemcpyDeviceToHost));
  });
}

int nnm_top_p(nnm_dataset* ds, int32_t metric, const int64_t* roots, const int64_t* sizes,
              double thr, int64_t kl2, int64_t kl3, int64_t P, double* out_dist, int64_t* out_a,
              int64_t* out_b, int64_t* out_len) {
  return guarded([&] {
    if (!ds) invalid("null dataset");
    if (P < 1) invalid("P must be at least 1, got " + std::to_string(P));  // pairgen.py:256-257
    check_metric(metric);
    std::lock_guard<std::mutex> lk(ds->mu);
    CUDA_TRY(cudaSetDevice(ds->device));
    t_alloc_stream = ds->st;
    const int64_t n = ds->n;
    std::vector<int> hc(ds->ld, -1), hs(ds->ld, 0);
    for (int64_t i = 0; i < n; ++i) {
      if (roots[i] < 0 || roots[i] >= n) invalid("root label out of range");
      hc[i] = (int)roots[i];
      hs[i] = (int)std::min<int64_t>(sizes[i], INT_UNSET - 1);
    }
    ds->comp.ensure(ds->ld);
    ds->psize.ensure(ds->ld);
    CUDA_TRY(cudaMemcpyAsync(ds->comp.p, hc.data(), ds->ld * sizeof(int), cudaMemcpyHostToDevice, ds->st));
    CUDA_TRY(cudaMemcpyAsync(ds->psize.p, hs.data(), ds->ld * sizeof(int), cudaMemcpyHostToDevice, ds->st));
    std::vector<Cand> res;
    ds->top_p(metric, std::isnan(thr) ? INFINITY : thr, clamp_int(kl2, ds->n), clamp_int(kl3, ds->n), P, res);
    for (size_t t = 0; t < res.size(); ++t) {
      out_dist[t] = res[t].d;
      out_a[t] = res[t].a;
      out_b[t] = res[t].b;
    }
    *out_len = (int64_t)res.size();
  });
}

int nnm_run(nnm_dataset* ds, int32_t metric, const nnm_constraints* cons, int64_t P, int32_t flags,
            nnm_merge* out_merges, int64_t* out_n_merges, int64_t* out_assign, int64_t* out_rounds,
            int32_t* out_stop, nnm_round_counters* out_counters, int64_t counters_cap,
            int64_t* out_n_counters, nnm_stats* stats) {
  return guarded([&] {
    if (!ds || !cons) invalid("null argument");
    check_metric(metric);
    check_constraints(cons);
    if (P < 1) invalid("pairs_per_batch must be at least 1, got " + std::to_string(P));
    std::lock_guard<std::mutex> lk(ds->mu);
    CUDA_TRY(cudaSetDevice(ds->device));
    t_alloc_stream = ds->st;
    auto t0 = std::chrono::steady_clock::now();
    const int64_t launches0 = g_launches.load();
    ds->stats = nnm_stats{};
    ds->round_log.clear();
    ds->pairs_covered = 0.0;
    ds->stats.device = ds->device;
    const int64_t n = ds->n;
    const bool rounds_path = (flags & NNM_FLAG_ROUNDS) || cons->kl2 > 0 || cons->kl3 > 0 || cons->kl4 > 0;
    int64_t n_counters = 0;
    if (!rounds_path) {
      // ---------------- Boruvka: exact MST of the eligible graph, then replay
      ds->stats.path = NNM_PATH_BORUVKA;
      auto tp0 = std::chrono::steady_clock::now();
      // the caller's output arrays are usually fresh pages: fault them in on host threads
      // while the GPU rounds run, so the replay below writes to resident memory
      std::vector<std::thread> prefault;
      if (n > 4096 && !(is_page_locked(out_merges) && is_page_locked(out_assign))) {
        char* pm = reinterpret_cast<char*>(out_merges);
        const size_t bm = (size_t)(n - 1) * sizeof(nnm_merge), half = bm / 2;
        prefault.emplace_back([pm, half] { memset(pm, 0, half); });
        prefault.emplace_back([pm, half, bm] { memset(pm + half, 0, bm - half); });
        prefault.emplace_back([out_assign, n] { memset(out_assign, 0, (size_t)n * sizeof(int64_t)); });
        prefault.emplace_back([ds] { ds->replay_host_buffers(); });
      }
      struct Joiner {
        std::vector<std::thread>& t;
        ~Joiner() {
          for (auto& th : t)
            if (th.joinable()) th.join();
        }
      } joiner{prefault};
      // NNM_SMALL=1 (n <= 65536, d <= 16): the dense exact Boruvka in one cooperative launch
      // -- every cross pair in FP64 every round, no screening, no pruning: an independent
      // algorithm the tests run beside the default path (at C1 it is not faster: 3.6 vs
      // 2.8 ms, FP64 row minima dominate)
      // small inputs (n <= SMALL_AUTO_N, d <= 16) by default: the screened single-launch
      // Boruvka (small_screened_kernel); NNM_SMALL=0 general path, 1 dense FP64, 2 screened
      const char* sme = getenv("NNM_SMALL");
      const int small_mode = sme ? (sme[0] == '1' ? 1 : sme[0] == '2' ? 2 : 0)
                                 : (n <= SMALL_AUTO_N ? 2 : 0);
      bool small = n > 1 && n <= 65536 && ds->d <= 16 && small_mode > 0;
      const bool need_s = !(cons->kl1 > 0 && n <= cons->kl1);
      if (small && need_s) {
        NvtxRange nv("nnm single-launch boruvka (small input)");
        small = ds->small_boruvka(metric, cons->dmax, small_mode == 2);
      }
      if (small) {
        ds->stats.prep_ms = 0.0;
        if (!need_s) {  // nothing to merge: an empty edge list
          ds->edges.ensure(1);
          ds->counters.ensure(8);
          CUDA_TRY(cudaMemsetAsync(ds->counters.p, 0, sizeof(unsigned long long), ds->st));
          ds->bv_metric = metric;
          ds->bv_round = 0;
        }
        auto tr0 = std::chrono::steady_clock::now();
        for (auto& th : prefault) th.join();
        ds->bv_end(cons->kl1, out_merges, out_n_merges, out_assign, out_rounds, out_stop);
        ds->stats.replay_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tr0).count();
      } else {
      {
        NvtxRange nv("nnm prep (view, geometry, tables)");
        ds->bv_begin(metric, cons->dmax);
        ds->sync();
      }
      ds->stats.prep_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tp0).count();
      bool need = n > 1 && !(cons->kl1 > 0 && n <= cons->kl1);
      const char* pe = getenv("NNM_PRUNE");
      const bool prune = !(pe && pe[0] == '0');
      const bool dbg_t = getenv("NNM_DEBUG") != nullptr;
      while (need && ds->bv_ncomp > 1) {
        NvtxRange nv("nnm boruvka round %lld", (long long)ds->bv_round + 1);
        const nnm_round_stat rl = ds->rl_open(ds->bv_round + 1);
        auto th0 = std::chrono::steady_clock::now();
        if (prune) {
          ds->pruned_scan(metric);
          if (dbg_t) {
            ds->sync();
            fprintf(stderr, "[nnm] host: round scan %.2f ms\n",
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - th0).count());
          }
        } else {
          ds->scan(metric, ds->B1.p, ds->B2.p, true, INT_UNSET, INT_UNSET, ds->bv_thr_hi, 0,
                   ds->tile_pairs());
          ds->pairs_covered += (double)n * (double)(n - 1) / 2.0;
        }
        auto th1 = std::chrono::steady_clock::now();
        int64_t added = ds->bv_finish_round(ds->B1.p, ds->B2.p);
        ds->rl_close(rl, added);
        if (dbg_t)
          fprintf(stderr, "[nnm] host: round finish %.2f ms\n",
                  std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - th1).count());
        if (added == 0) break;
      }
      auto tr0 = std::chrono::steady_clock::now();
      for (auto& th : prefault) th.join();
      ds->bv_end(cons->kl1, out_merges, out_n_merges, out_assign, out_rounds, out_stop);
      ds->stats.replay_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tr0).count();
      }
    } else {
      // ---------------- top-P rounds with exact engine semantics
      ds->stats.path = NNM_PATH_ROUNDS;
      ds->rb1_valid = false;
      const int64_t kl1 = cons->kl1, kl2 = cons->kl2, kl3 = cons->kl3, kl4 = cons->kl4;
      // kl2 / kl3 without kl4: the ordered merge list is the same for
      // every batch size (the reference's own test_acceptance.py:159-171), so
      // the rounds take a large batch (16384: C2 without kl4 in 23 rounds instead of 429).  MergeEvent.round, rounds and
      // round_counters then number these rounds; they are part of parity only with kl4
      // (F4) or when the caller asks for the reference's round structure (exact_rounds).
      const char* fke = getenv("NNM_FAST_P");
      const int64_t fastP = fke ? std::max<int64_t>(1, atoll(fke)) : 16384;
      if (kl4 <= 0 && !(flags & NNM_FLAG_ROUNDS)) P = std::max<int64_t>(P, fastP);
      double thr = INFINITY;
      if (!std::isnan(cons->dmax)) thr = metric == EUCLIDEAN ? cons->dmax * cons->dmax : cons->dmax;
      std::vector<int64_t> par(n), sz(n, 1);
      for (int64_t i = 0; i < n; ++i) par[i] = i;
      auto find = [&](int64_t x) {
        int64_t r = x;
        while (par[r] != r) r = par[r];
        while (par[x] != r) {
          int64_t nx = par[x];
          par[x] = r;
          x = nx;
        }
        return r;
      };
      int64_t count = n, nm = 0, rounds = 0;
      ds->comp.ensure(ds->ld);
      ds->psize.ensure(ds->ld);
      ds->rmap.ensure(n);
      ds->rsize.ensure(n);
      fill_comp_kernel<<<blocks_for(ds->ld), 256, 0, ds->st>>>(ds->comp.p, ds->psize.p, n, ds->ld); note_launch();
      iota_kernel<<<blocks_for(n), 256, 0, ds->st>>>(ds->rmap.p, (int)n); note_launch();
      ones_kernel<<<blocks_for(n), 256, 0, ds->st>>>(ds->rsize.p, (int)n); note_launch();
      CUDA_TRY(cudaGetLastError());
      int reason = 0;
      std::vector<Cand> buf;
      std::vector<int64_t> order;
      std::vector<int64_t> snap_size;  // round-start size lookups
      std::vector<int2> hmap, hsize;
      for (;;) {
        if (count == 1) { reason = NNM_STOP_SINGLE_CLUSTER; break; }
        if (kl1 > 0 && count <= kl1) { reason = NNM_STOP_KL1; break; }
        NvtxRange nv("nnm round %lld", (long long)rounds + 1);
        const nnm_round_stat rl = ds->rl_open(rounds + 1);
        ds->top_p(metric, thr, clamp_int(kl2, ds->n), clamp_int(kl3, ds->n), P, buf, rounds > 0);
        if (buf.empty()) { reason = NNM_STOP_NO_ELIGIBLE; break; }
        ++rounds;
        const int64_t L = (int64_t)buf.size();
        // order_batch (engine.py:73-87): stable partition by round-start sizes
        order.resize(L);
        if (kl4 > 0) {
          std::vector<char> pri(L);
          for (int64_t t = 0; t < L; ++t) {
            int64_t s = std::min(sz[find(buf[t].a)], sz[find(buf[t].b)]);
            pri[t] = s < kl4;
          }
          int64_t k = 0;
          for (int64_t t = 0; t < L; ++t) if (pri[t]) order[k++] = t;
          for (int64_t t = 0; t < L; ++t) if (!pri[t]) order[k++] = t;
        } else {
          for (int64_t t = 0; t < L; ++t) order[t] = t;
        }
        // process_batch (engine.py:90-143)
        int64_t same = 0, s2 = 0, s3 = 0, unproc = 0, merged = 0;
        std::vector<int64_t> touched;
        for (int64_t pos = 0; pos < L; ++pos) {
          const Cand& c = buf[order[pos]];
          int64_t ra = find(c.a), rb = find(c.b);
          if (ra == rb) { ++same; continue; }
          int64_t sa = sz[ra], sb = sz[rb];
          if (kl2 > 0 && (sa > kl2 || sb > kl2)) { ++s2; continue; }
          if (kl3 > 0 && sa + sb > kl3) { ++s3; continue; }
          int64_t keep = std::min(ra, rb), drop = std::max(ra, rb);
          par[drop] = keep;
          sz[keep] += sz[drop];
          --count;
          touched.push_back(drop);
          touched.push_back(keep);
          nnm_merge& m = out_merges[nm++];
          m.round = rounds;
          m.root_a = keep;
          m.root_b = drop;
          m.dist = metric == EUCLIDEAN ? std::sqrt(c.d) : c.d;
          m.new_size = sz[keep];
          m.point_a = c.a;
          m.point_b = c.b;
          ++merged;
          if (count == 1 || (kl1 > 0 && count <= kl1)) {
            unproc = L - pos - 1;
            break;
          }
        }
        ds->rl_close(rl, merged);
        if (out_counters && n_counters < counters_cap) {
          nnm_round_counters& rc = out_counters[n_counters];
          rc.round = rounds;
          rc.selected = L;
          rc.merged = merged;
          rc.same_root = same;
          rc.kl2 = s2;
          rc.kl3 = s3;
          rc.unprocessed = unproc;
        }
        ++n_counters;

        // refresh the device snapshot: root map + root sizes for touched roots
        hmap.clear();
        hsize.clear();
        for (int64_t r : touched) {
          int64_t f = find(r);
          hmap.push_back(make_int2((int)r, (int)f));
          hsize.push_back(make_int2((int)f, (int)std::min<int64_t>(sz[f], INT_UNSET - 1)));
        }
        if (!hmap.empty()) {
          ds->kv.ensure(hmap.size() + hsize.size());
          CUDA_TRY(cudaMemcpyAsync(ds->kv.p, hmap.data(), hmap.size() * sizeof(int2), cudaMemcpyHostToDevice, ds->st));
          CUDA_TRY(cudaMemcpyAsync(ds->kv.p + hmap.size(), hsize.data(), hsize.size() * sizeof(int2), cudaMemcpyHostToDevice, ds->st));
          scatter_kernel<<<blocks_for(hmap.size()), 256, 0, ds->st>>>(ds->kv.p, (int)hmap.size(), ds->rmap.p); note_launch();
          scatter_kernel<<<blocks_for(hsize.size()), 256, 0, ds->st>>>(ds->kv.p + hmap.size(), (int)hsize.size(), ds->rsize.p); note_launch();
          snapshot_update_kernel<<<blocks_for(n), 256, 0, ds->st>>>((int)n, ds->comp.p, ds->psize.p, ds->rmap.p, ds->rsize.p); note_launch();
          CUDA_TRY(cudaGetLastError());
          ds->sync();  // host vectors are reused next round
        }
      }
      for (int64_t i = 0; i < n; ++i) out_assign[i] = find(i);
      *out_n_merges = nm;
      *out_rounds = rounds;
      *out_stop = reason;
    }
    if (out_n_counters) *out_n_counters = n_counters;
    ds->flush_scan_stats();
    ds->stats.total_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    ds->stats.kernel_launches = g_launches.load() - launches0;
    ds->stats.pairs_covered = ds->pairs_covered;
    if (stats) *stats = ds->stats;
  });
}

// ---- staged Boruvka API (multi-GPU driver) ----------------------------------
int nnm_bv_begin(nnm_dataset* ds, int32_t metric, double dmax, int64_t* out_tile_pairs,
                 int64_t* out_rows) {
  return guarded([&] {
    if (!ds) invalid("null dataset");
    check_metric(metric);
    std::lock_guard<std::mutex> lk(ds->mu);
    CUDA_TRY(cudaSetDevice(ds->device));
    t_alloc_stream = ds->st;
    ds->stats = nnm_stats{};
    ds->stats.path = NNM_PATH_BORUVKA;
    ds->stats.device = ds->device;
    ds->pairs_covered = 0.0;
    ds->bv_begin(metric, dmax);
    if (out_tile_pairs) *out_tile_pairs = ds->tile_pairs();
    if (out_rows) *out_rows = ds->vn;
  });
}

int nnm_bv_scan(nnm_dataset* ds, int64_t w_begin, int64_t w_end, uint64_t* B1_dev, uint64_t* B2_dev) {
  return guarded([&] {
    if (!ds || !B1_dev || !B2_dev) invalid("null argument");
    if (w_begin < 0 || w_end < w_begin || w_end > ds->tile_pairs()) invalid("bad tile-pair range");
    std::lock_guard<std::mutex> lk(ds->mu);
    CUDA_TRY(cudaSetDevice(ds->device));
    t_alloc_stream = ds->st;
    CUDA_TRY(cudaDeviceSynchronize());  // caller buffers may be written on other streams
    ds->scan(ds->bv_metric, reinterpret_cast<unsigned long long*>(B1_dev),
             reinterpret_cast<unsigned long long*>(B2_dev), true, INT_UNSET, INT_UNSET,
             ds->bv_thr_hi, w_begin, w_end);
    ds->sync();
  });
}

}  // extern "C"

namespace nnm {
__global__ void second_kernel(int n, const unsigned long long* b1l, const unsigned long long* b2l,
                              const unsigned long long* b1g, unsigned long long* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = (b1l[i] == b1g[i]) ? b2l[i] : b1l[i];
}
}  // namespace nnm

namespace nnm {
// ---- exchanges over peer memory (nnm_run_multi): every replica combines the partial
// arrays of all replicas itself (P2P loads over NVLink / NVSwitch; same-device replicas
// read local memory), so no broadcast step is needed.  Launched only after every
// replica's producing step has completed (host join): no kernel waits on another.
constexpr int MAX_REPLICAS = 16;
struct PeerPtrs {
  const void* p[MAX_REPLICAS];
};

__global__ void peer_min_u32_kernel(int64_t n, PeerPtrs in, int k, unsigned* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned v = 0xFFFFFFFFu;
  for (int s = 0; s < k; ++s) v = min(v, static_cast<const unsigned*>(in.p[s])[i]);
  out[i] = v;
}

__global__ void peer_max_u32_kernel(int64_t n, PeerPtrs in, int k, unsigned* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned v = 0u;
  for (int s = 0; s < k; ++s) v = max(v, static_cast<const unsigned*>(in.p[s])[i]);
  out[i] = v;
}

// g1 = min_s b1_s; g2 = min_s (b1_s == g1 ? b2_s : b1_s): the best and second-best keys of
// the union of every replica's per-row top-2 (the second-smallest of distinct keys)
__global__ void peer_keys_kernel(int64_t n, PeerPtrs b1, PeerPtrs b2, int k,
                                 unsigned long long* __restrict__ g1,
                                 unsigned long long* __restrict__ g2) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned long long m1 = NONE_KEY;
  for (int s = 0; s < k; ++s) m1 = min(m1, static_cast<const unsigned long long*>(b1.p[s])[i]);
  unsigned long long m2 = NONE_KEY;
  for (int s = 0; s < k; ++s) {
    const unsigned long long a = static_cast<const unsigned long long*>(b1.p[s])[i];
    m2 = min(m2, a == m1 ? static_cast<const unsigned long long*>(b2.p[s])[i] : a);
  }
  g1[i] = m1;
  g2[i] = m2;
}
}  // namespace nnm

extern "C" {
// ---- staged pruned round (multi-rank driver; DESIGN 6) --------------------------------
static void staged_enter(nnm_dataset* ds) {
  CUDA_TRY(cudaSetDevice(ds->device));
  t_alloc_stream = ds->st;
  CUDA_TRY(cudaDeviceSynchronize());  // caller buffers may be written on other streams
}

int nnm_bv_round_bound(nnm_dataset* ds, int32_t rank, int32_t world, uint32_t** out_caps,
                       int64_t* out_count) {
  return guarded([&] {
    if (!ds || !out_caps || !out_count) invalid("null argument");
    if (world < 1 || rank < 0 || rank >= world) invalid("bad rank / world");
    std::lock_guard<std::mutex> lk(ds->mu);
    staged_enter(ds);
    ds->round_bound(ds->bv_metric, rank, world);
    ds->sync();
    *out_caps = ds->tc_cap_on ? reinterpret_cast<uint32_t*>(ds->ucap.p) : nullptr;
    *out_count = ds->tc_cap_on ? ds->vn : 0;
  });
}

int nnm_bv_round_phase1(nnm_dataset* ds, int32_t rank, int32_t world, const uint32_t* caps_dev,
                        uint64_t* B1_dev, uint64_t* B2_dev) {
  return guarded([&] {
    if (!ds || !B1_dev || !B2_dev) invalid("null argument");
    if (world < 1 || rank < 0 || rank >= world) invalid("bad rank / world");
    std::lock_guard<std::mutex> lk(ds->mu);
    staged_enter(ds);
    if (ds->tc_cap_on) ds->caps_read = caps_dev ? reinterpret_cast<const unsigned*>(caps_dev) : ds->ucap.p;
    ds->round_phase1(reinterpret_cast<unsigned long long*>(B1_dev),
                     reinterpret_cast<unsigned long long*>(B2_dev), rank, world);
    ds->sync();
  });
}

int nnm_bv_round_phase2(nnm_dataset* ds, int32_t rank, int32_t world, const uint64_t* G1_dev,
                        const uint64_t* G2_dev, uint64_t* B1_dev, uint64_t* B2_dev,
                        uint32_t** out_cache, int64_t* out_count) {
  return guarded([&] {
    if (!ds || !G1_dev || !G2_dev || !B1_dev || !B2_dev || !out_cache || !out_count)
      invalid("null argument");
    if (world < 1 || rank < 0 || rank >= world) invalid("bad rank / world");
    std::lock_guard<std::mutex> lk(ds->mu);
    staged_enter(ds);
    ds->round_phase2(reinterpret_cast<const unsigned long long*>(G1_dev),
                     reinterpret_cast<const unsigned long long*>(G2_dev),
                     reinterpret_cast<unsigned long long*>(B1_dev),
                     reinterpret_cast<unsigned long long*>(B2_dev), rank, world);
    ds->sync();
    const bool pend = ds->rd_stage == 3;
    *out_cache = pend ? reinterpret_cast<uint32_t*>(ds->cachebuf.p) : nullptr;
    *out_count = pend ? ds->rd_n1 + ds->rd_n2 : 0;
  });
}

int nnm_bv_cache_scatter(nnm_dataset* ds) {
  return guarded([&] {
    if (!ds) invalid("null dataset");
    std::lock_guard<std::mutex> lk(ds->mu);
    staged_enter(ds);
    ds->cache_scatter();
    ds->sync();
  });
}

// ---- single-process multi-GPU run: one replica per device (or several replicas on one
// device, which runs the same exchange code sequentially), the staged pruned round on
// 1/N shares with the exchanges done by peer kernels (DESIGN 6).  Without kl2/kl3/kl4 only;
// the round path runs on replicas[0].
}  // extern "C"
namespace {
template <class F>
void par_replicas(nnm_dataset** reps, int k, F&& f) {
  std::vector<std::thread> th;
  std::vector<std::exception_ptr> err(k);
  for (int r = 0; r < k; ++r)
    th.emplace_back([&, r] {
      try {
        CUDA_TRY(cudaSetDevice(reps[r]->device));
        t_alloc_stream = reps[r]->st;
        f(r, reps[r]);
        reps[r]->sync();
      } catch (...) {
        err[r] = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
}
}  // namespace
extern "C" {

int nnm_run_multi(nnm_dataset** reps, int32_t n_rep, int32_t metric, const nnm_constraints* cons,
                  int64_t P, int32_t flags, nnm_merge* out_merges, int64_t* out_n_merges,
                  int64_t* out_assign, int64_t* out_rounds, int32_t* out_stop,
                  nnm_round_counters* out_counters, int64_t counters_cap, int64_t* out_n_counters,
                  nnm_stats* stats) {
  if (reps && n_rep == 1)
    return nnm_run(reps[0], metric, cons, P, flags, out_merges, out_n_merges, out_assign, out_rounds,
                   out_stop, out_counters, counters_cap, out_n_counters, stats);
  return guarded([&] {
    if (!reps || !cons || n_rep < 1) invalid("null argument");
    if (n_rep > MAX_REPLICAS) invalid("at most " + std::to_string(MAX_REPLICAS) + " replicas");
    for (int r = 0; r < n_rep; ++r) {
      if (!reps[r]) invalid("null replica");
      if (reps[r]->n != reps[0]->n || reps[r]->d != reps[0]->d) invalid("replicas differ in shape");
      for (int q = 0; q < r; ++q)
        if (reps[q] == reps[r]) invalid("a replica appears twice");
    }
    check_metric(metric);
    check_constraints(cons);
    if (P < 1) invalid("pairs_per_batch must be at least 1, got " + std::to_string(P));
    const bool rounds_path = (flags & NNM_FLAG_ROUNDS) || cons->kl2 > 0 || cons->kl3 > 0 || cons->kl4 > 0;
    if (rounds_path) {
      const int rc = nnm_run(reps[0], metric, cons, P, flags, out_merges, out_n_merges, out_assign,
                             out_rounds, out_stop, out_counters, counters_cap, out_n_counters, stats);
      if (rc != NNM_OK) throw NnmError{rc, g_err};
      return;
    }
    std::vector<nnm_dataset*> order(reps, reps + n_rep);
    std::sort(order.begin(), order.end());
    std::vector<std::unique_lock<std::mutex>> locks;
    for (auto* d : order) locks.emplace_back(d->mu);
    // peer access between the devices in use (no-op for same-device replicas)
    for (int r = 0; r < n_rep; ++r)
      for (int q = 0; q < n_rep; ++q) {
        const int a = reps[r]->device, b = reps[q]->device;
        if (a == b) continue;
        int can = 0;
        CUDA_TRY(cudaDeviceCanAccessPeer(&can, a, b));
        if (!can) throw NnmError{NNM_E_UNSUPPORTED, "devices " + std::to_string(a) + " and " +
                                                        std::to_string(b) + " have no peer access"};
        CUDA_TRY(cudaSetDevice(a));
        const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CUDA_TRY(e);
        cudaGetLastError();
      }
    auto t0 = std::chrono::steady_clock::now();
    const int64_t launches0 = g_launches.load();
    nnm_dataset* ds0 = reps[0];
    const int64_t n = ds0->n;
    par_replicas(reps, n_rep, [&](int, nnm_dataset* ds) {
      ds->stats = nnm_stats{};
      ds->round_log.clear();
      ds->pairs_covered = 0.0;
      ds->stats.device = ds->device;
      ds->stats.path = NNM_PATH_BORUVKA;
      ds->bv_begin(metric, cons->dmax);
      ds->G1.ensure(ds->vn);
      ds->G2.ensure(ds->vn);
      ds->ucapg.ensure(ds->vn);
    });
    ds0->stats.prep_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    const int64_t vn = ds0->vn;
    auto peers = [&](auto get) {
      PeerPtrs pp{};
      for (int q = 0; q < n_rep; ++q) pp.p[q] = get(reps[q]);
      return pp;
    };
    const bool need = n > 1 && !(cons->kl1 > 0 && n <= cons->kl1);
    while (need && ds0->bv_ncomp > 1) {
      NvtxRange nv("nnm multi-replica round %lld", (long long)ds0->bv_round + 1);
      const nnm_round_stat rl = ds0->rl_open(ds0->bv_round + 1);
      par_replicas(reps, n_rep, [&](int r, nnm_dataset* ds) { ds->round_bound(metric, r, n_rep); });
      if (ds0->tc_cap_on) {  // caps: min over the replicas' bound-pass shares
        const PeerPtrs pc = peers([](nnm_dataset* q) { return (const void*)q->ucap.p; });
        par_replicas(reps, n_rep, [&](int, nnm_dataset* ds) {
          peer_min_u32_kernel<<<blocks_for(vn), 256, 0, ds->st>>>(vn, pc, n_rep, ds->ucapg.p); note_launch();
          CUDA_TRY(cudaGetLastError());
          ds->caps_read = ds->ucapg.p;
        });
      }
      par_replicas(reps, n_rep, [&](int r, nnm_dataset* ds) { ds->round_phase1(ds->B1.p, ds->B2.p, r, n_rep); });
      const PeerPtrs p1 = peers([](nnm_dataset* q) { return (const void*)q->B1.p; });
      const PeerPtrs p2 = peers([](nnm_dataset* q) { return (const void*)q->B2.p; });
      auto combine = [&](int, nnm_dataset* ds) {
        peer_keys_kernel<<<blocks_for(vn), 256, 0, ds->st>>>(vn, p1, p2, n_rep, ds->G1.p, ds->G2.p); note_launch();
        CUDA_TRY(cudaGetLastError());
      };
      par_replicas(reps, n_rep, combine);
      par_replicas(reps, n_rep, [&](int r, nnm_dataset* ds) {
        ds->round_phase2(ds->G1.p, ds->G2.p, ds->B1.p, ds->B2.p, r, n_rep);
      });
      par_replicas(reps, n_rep, combine);
      if (ds0->rd_stage == 3) {  // tile-pair cache entries of this round: max over the replicas
        const int64_t nc = ds0->rd_n1 + ds0->rd_n2;
        const PeerPtrs pc = peers([](nnm_dataset* q) { return (const void*)q->cachebuf.p; });
        par_replicas(reps, n_rep, [&](int, nnm_dataset* ds) {
          ds->cacheg.ensure(nc);
          peer_max_u32_kernel<<<blocks_for(nc), 256, 0, ds->st>>>(nc, pc, n_rep, ds->cacheg.p); note_launch();
          CUDA_TRY(cudaGetLastError());
        });
        par_replicas(reps, n_rep, [&](int, nnm_dataset* ds) { ds->cache_scatter(ds->cacheg.p); });
      }
      std::vector<int64_t> added(n_rep);
      par_replicas(reps, n_rep, [&](int r, nnm_dataset* ds) { added[r] = ds->bv_finish_round(ds->G1.p, ds->G2.p); });
      for (int r = 1; r < n_rep; ++r)
        if (added[r] != added[0]) throw NnmError{NNM_E_CUDA, "replicas diverged (internal error)"};
      ds0->rl_close(rl, added[0]);
      if (added[0] == 0) break;
    }
    auto tr0 = std::chrono::steady_clock::now();
    CUDA_TRY(cudaSetDevice(ds0->device));
    t_alloc_stream = ds0->st;
    ds0->bv_end(cons->kl1, out_merges, out_n_merges, out_assign, out_rounds, out_stop);
    ds0->stats.replay_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tr0).count();
    par_replicas(reps, n_rep, [&](int, nnm_dataset* ds) { ds->flush_scan_stats(); });
    nnm_stats agg = ds0->stats;
    for (int r = 1; r < n_rep; ++r) {
      agg.scans += reps[r]->stats.scans;
      agg.pairs_evaluated += reps[r]->stats.pairs_evaluated;
      agg.scan_ms = std::max(agg.scan_ms, reps[r]->stats.scan_ms);
      agg.tc_items += reps[r]->stats.tc_items;
      agg.ambiguous_rows = std::max(agg.ambiguous_rows, reps[r]->stats.ambiguous_rows);
    }
    agg.pairs_covered = ds0->pairs_covered;
    agg.total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    agg.kernel_launches = g_launches.load() - launches0;
    agg.replay_gpu_merges = ds0->stats.replay_gpu_merges;
    ds0->stats = agg;
    if (out_n_counters) *out_n_counters = 0;
    if (stats) *stats = agg;
  });
}

int nnm_tc_probe(nnm_dataset* ds, const int32_t* items, int64_t n_items, double* out) {
  return guarded([&] {
    if (!ds || !items || !out) invalid("null argument");
    if (n_items < 1) invalid("n_items must be at least 1");
    std::lock_guard<std::mutex> lk(ds->mu);
    CUDA_TRY(cudaSetDevice(ds->device));
    t_alloc_stream = ds->st;
    if (!tc_supported(ds->d)) throw NnmError{NNM_E_UNSUPPORTED, "d outside the tensor-core scan"};
    ds->bv_begin(EUCLIDEAN, NAN);  // kd view, tile geometry, singleton components
    ds->tc_prepare();
    ++ds->scan_epoch;
    ds->tc_tails();
    for (int64_t t = 0; t < 2 * n_items; ++t)
      if (items[t] < 0 || items[t] >= ds->Tp) invalid("tile index out of range");
    DevBuf<int2> it;
    it.ensure(n_items);
    DevBuf<float> dump;
    dump.ensure((size_t)n_items * TILE * TILE);
    DevBuf<unsigned long long> acc;
    acc.ensure(3);
    CUDA_TRY(cudaMemcpyAsync(it.p, items, n_items * sizeof(int2), cudaMemcpyHostToDevice, ds->st));
    CUDA_TRY(cudaMemsetAsync(acc.p, 0, 3 * sizeof(unsigned long long), ds->st));
    TcArgs a{};
    a.img = ds->tc_img.p;
    a.tnorm = ds->tc_tnorm.p;
    a.eta = ds->tc_eta.p;
    a.meta = ds->tc_meta.p;
    a.sq = ds->tc_sq.p;
    a.comp = ds->comp.p;
    a.X64 = ds->X64p.p;
    a.np = (int)ds->np_;
    a.d = ds->d;
    a.T = ds->Tp;
    a.items = it.p;
    a.w_begin = 0;
    a.w_end = n_items;
    a.thr_hi = INFINITY;
    a.B1 = ds->B1.p;
    a.B2 = ds->B2.p;
    a.dump = dump.p;
    a.slots = ds->tc_slots.p;
    a.dbg = 0;
    a.trace = nullptr;
    CUDA_TRY(launch_tc_scan(a, (int)std::min<int64_t>(n_items, ds->sms), ds->st));
    CUDA_TRY(launch_tc_probe(a, ds->X64p.p, it.p, n_items, acc.p, ds->st));
    unsigned long long h[3];
    CUDA_TRY(cudaMemcpyAsync(h, acc.p, sizeof(h), cudaMemcpyDeviceToHost, ds->st));
    ds->sync();
    float worst;
    uint32_t wb = (uint32_t)h[0];
    memcpy(&worst, &wb, 4);
    out[0] = worst;
    out[1] = (double)h[1];
    out[2] = (double)h[2];
  });
}

int nnm_bv_second(nnm_dataset* ds, const uint64_t* B1loc, const uint64_t* B2loc,
                  const uint64_t* B1glob, uint64_t* B2c) {
  return guarded([&] {
    if (!ds) invalid("null dataset");
    std::lock_guard<std::mutex> lk(ds->mu);
    CUDA_TRY(cudaSetDevice(ds->device));
    t_alloc_stream = ds->st;
    CUDA_TRY(cudaDeviceSynchronize());  // caller buffers may be written on other streams
    second_kernel<<<blocks_for(ds->vn), 256, 0, ds->st>>>(
        (int)ds->vn, reinterpret_cast<const unsigned long long*>(B1loc),
        reinterpret_cast<const unsigned long long*>(B2loc),
        reinterpret_cast<const unsigned long long*>(B1glob),
        reinterpret_cast<unsigned long long*>(B2c)); note_launch();
    CUDA_TRY(cudaGetLastError());
    ds->sync();
  });
}

int nnm_bv_finish_round(nnm_dataset* ds, const uint64_t* B1_dev, const uint64_t* B2_dev,
                        int64_t* out_edges) {
  return guarded([&] {
    if (!ds) invalid("null dataset");
    std::lock_guard<std::mutex> lk(ds->mu);
    CUDA_TRY(cudaSetDevice(ds->device));
    t_alloc_stream = ds->st;
    CUDA_TRY(cudaDeviceSynchronize());  // caller buffers may be written on other streams
    *out_edges = ds->bv_finish_round(reinterpret_cast<const unsigned long long*>(B1_dev),
                                     reinterpret_cast<const unsigned long long*>(B2_dev));
  });
}

int nnm_bv_end(nnm_dataset* ds, int64_t kl1, nnm_merge* out_merges, int64_t* out_n_merges,
               int64_t* out_assign, int64_t* out_rounds, int32_t* out_stop, nnm_stats* stats) {
  return guarded([&] {
    if (!ds) invalid("null dataset");
    if (kl1 == 0) invalid("kl1 must be a positive count, got 0");
    std::lock_guard<std::mutex> lk(ds->mu);
    CUDA_TRY(cudaSetDevice(ds->device));
    t_alloc_stream = ds->st;
    ds->bv_end(kl1, out_merges, out_n_merges, out_assign, out_rounds, out_stop);
    ds->flush_scan_stats();
    ds->stats.pairs_covered = ds->pairs_covered;
    if (stats) *stats = ds->stats;
  });
}
}  // extern "C"
