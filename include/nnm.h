/*
 * nnm.h -- C ABI of the B200-native NNM (constrained single-linkage) hot path.
 *
 * The reference (parclust, arXiv 1402.3789 restated in Python) has no formal
 * plugin registry: its seams are module attributes that its own tests patch
 * (SURVEY.md 8b).  Each entry point below replaces one of them; the citation
 * gives the reference interface (paths relative to
 * /root/reference/pkg/src/parclust/).  Bindings a maintainer adds on the
 * reference side are shown in INTEGRATION.md.
 *
 * Conventions (mirroring the reference):
 *   - metric: 0 euclidean, 1 squared-euclidean, 2 manhattan, 3 chebyshev
 *     (metrics.py:34-53).  Distances are "internal" units (squared for both
 *     euclidean kinds) except nnm_merge.dist, which is reported units
 *     (metrics.py:86-90).
 *   - integer constraints < 0 mean unset; dmax / thr NaN means unset
 *     (model.py:190-218).
 *   - return 0 on success, a negative NNM_E_* code otherwise; the message is
 *     available from nnm_last_error() (thread-local).  NNM_E_INVALID maps to
 *     the reference's ValidationError (model.py:25-26); NNM_E_CUDA to
 *     WorkerError (scheduler.py:45-46).
 *   - all pointers are caller-owned host memory unless the name says _dev.
 *   - there is no CPU fallback: without a usable sm_100 device every compute
 *     entry point returns NNM_E_CUDA.
 */
#ifndef NNM_H
#define NNM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NNM_ABI_VERSION 4

enum {
  NNM_OK = 0,
  NNM_E_INVALID = -1,     /* ValidationError */
  NNM_E_CUDA = -2,        /* device / kernel failure (WorkerError) */
  NNM_E_UNSUPPORTED = -3, /* input outside the implemented envelope */
  NNM_E_NOMEM = -4,       /* device allocation failed */
  NNM_E_CAPACITY = -5     /* caller buffer too small */
};

enum { NNM_EUCLIDEAN = 0, NNM_SQEUCLIDEAN = 1, NNM_MANHATTAN = 2, NNM_CHEBYSHEV = 3 };

/* stop reasons (engine.py:146-151, :174-176) */
enum { NNM_STOP_KL1 = 1, NNM_STOP_NO_ELIGIBLE = 2, NNM_STOP_SINGLE_CLUSTER = 3 };

/* nnm_run flags */
enum {
  NNM_FLAG_ROUNDS = 1 /* force the exact top-P round path (engine.py:154-199) for every
                         constraint set, so rounds / round_counters match the reference */
};

/* algorithm actually used by nnm_run (stats.path) */
enum { NNM_PATH_NONE = 0, NNM_PATH_BORUVKA = 1, NNM_PATH_ROUNDS = 2 };

typedef struct nnm_dataset nnm_dataset; /* opaque: X resident in HBM (FP64 + FP32 tiles) */

typedef struct { /* ConstraintSet, model.py:190-218 */
  int64_t kl1, kl2, kl3, kl4;
  double dmax;
} nnm_constraints;

typedef struct { /* MergeEvent, model.py:221-238 (step = array index) */
  int64_t round, root_a, root_b;
  double dist;
  int64_t new_size, point_a, point_b;
} nnm_merge;

typedef struct { /* engine.py:187-190 */
  int64_t round, selected, merged, same_root, kl2, kl3, unprocessed;
} nnm_round_counters;

typedef struct {
  int32_t path;            /* NNM_PATH_* */
  int32_t device;
  int64_t scans;           /* full screening scans launched */
  double pairs_evaluated;  /* unordered pairs evaluated by the FP32 screen */
  double scan_ms;          /* CUDA-event time of all screening-scan launches */
  double total_ms;         /* wall time of the call */
  int64_t ambiguous_rows;  /* rows re-resolved exactly (FP32 margin too small) */
  int64_t exact_evals;     /* FP64 pair evaluations */
  int64_t boruvka_rounds;
  int64_t kernel_launches; /* libnnm kernels launched by the call (library sorts excluded) */
  double pairs_covered;    /* pairs the rounds decided (evaluated or excluded by an exact bound) */
  double prep_ms;          /* one-time per dataset/metric work done by this call (spatial view,
                              norms, tile balls); 0 when cached */
  double replay_ms;        /* edge sort + union-find replay into the merge log */
  int64_t tc_items;        /* ordered 128x128 tile pairs run through the tensor-core scan
                              (each a 128x128x32 kind::tf32 MMA); 0 on the FP32 path */
  int64_t round_rescans;   /* round path: rounds whose reused row bounds were too loose, so
                              the full scan ran (rounds - 1 - round_rescans were reused) */
  int64_t replay_gpu_merges; /* merges replayed on the GPU (nnm_replay.cu); the rest, if
                                any, by the sequential host loop */
} nnm_stats;

typedef struct { /* per-round record of the last nnm_run on a dataset (SURVEY 5 observability) */
  int64_t round;          /* 1-based: Boruvka round, or reference round on the round path */
  double ms;              /* wall time of the round (host clock around synchronised work) */
  double scan_ms;         /* CUDA-event time of the round's screening scans */
  double pairs_evaluated; /* pairs the round's scans evaluated */
  int64_t items;          /* tile pairs run through the tensor-core scan (0 on FP32 scans) */
  int64_t merged;         /* MST edges added (Boruvka) / merges (round path) */
} nnm_round_stat;

int nnm_abi_version(void);
const char *nnm_last_error(void);
int nnm_device_count(int32_t *out);

/* Page-locked host blocks (recycled process-wide).  nnm_run / nnm_bv_end detect
 * page-locked out_merges / out_assign: the GPU then lays out the merge records and
 * labels itself and the copy engine writes them (no host assembly pass).  Plain
 * (pageable) output arrays keep working; this is an optimisation only. */
int nnm_host_alloc(int64_t bytes, void **out);
int nnm_host_free(void *p);

/* Upload X (n x d, row-major float64, finite) to `device` and build the FP32
 * screening tiles.  Replaces Dataset's array being read by every scan task
 * (model.py:29-76; pairgen.py:247-298).  Validation as Dataset.__post_init__. */
int nnm_dataset_create(const double *X, int64_t n, int32_t d, int32_t device, nnm_dataset **out);
/* Same, with X already resident in device memory on `device` (copied internally). */
int nnm_dataset_create_device(const double *X_dev, int64_t n, int32_t d, int32_t device,
                              nnm_dataset **out);
int nnm_dataset_destroy(nnm_dataset *ds);

/* Round seam: replaces scheduler.run_round / pairgen.global_top_p
 * (scheduler.py:268-335, pairgen.py:319-324).  roots/sizes are the
 * EligibilitySnapshot arrays (pairgen.py:134-166), thr its threshold in internal
 * units (NaN = none).  Writes the <=P smallest eligible pairs ascending by
 * (dist, a, b) into out_* (capacity P) and their count into out_len; the result
 * is bit-identical to global_top_p. */
int nnm_top_p(nnm_dataset *ds, int32_t metric, const int64_t *roots, const int64_t *sizes,
              double thr, int64_t kl2, int64_t kl3, int64_t P, double *out_dist, int64_t *out_a,
              int64_t *out_b, int64_t *out_len);

/* Run seam: replaces engine.run (engine.py:154-199).  out_merges has capacity
 * n-1, out_assign n, out_counters counters_cap entries (NULL allowed).
 * Without kl4 the merge list (root_a, root_b, dist, new_size, point_a, point_b)
 * equals the reference's for any P; with kl4 (or NNM_FLAG_ROUNDS) the round
 * structure, `round` fields and counters are reproduced as well. */
int nnm_run(nnm_dataset *ds, int32_t metric, const nnm_constraints *cons, int64_t P,
            int32_t flags, nnm_merge *out_merges, int64_t *out_n_merges, int64_t *out_assign,
            int64_t *out_rounds, int32_t *out_stop, nnm_round_counters *out_counters,
            int64_t counters_cap, int64_t *out_n_counters, nnm_stats *stats);

/* Metric seam: internal distances of every (x_i, y_j), FP64 bit-identical to
 * metrics.internal_pairwise (metrics.py:67-73).  out is nx*ny row-major. */
int nnm_pairwise(int32_t metric, const double *x, int64_t nx, const double *y, int64_t ny,
                 int32_t d, int32_t device, double *out);

/* ---- staged Boruvka API for the multi-GPU driver (paper_1402_3789_b200.distributed) ----
 * One process per GPU; every rank holds the full dataset.  Per round each rank
 * scans its share of the upper-triangular tile pairs into (B1, B2), the driver
 * combines the per-row keys across ranks with two all-reduce(min) calls, and
 * every rank then finishes the round identically.  Rows live in the library's
 * spatially ordered, tile-padded view: device key buffers are caller-owned
 * (e.g. torch tensors) of *out_rows uint64 each. */
int nnm_bv_begin(nnm_dataset *ds, int32_t metric, double dmax, int64_t *out_tile_pairs,
                 int64_t *out_rows);
int nnm_bv_scan(nnm_dataset *ds, int64_t w_begin, int64_t w_end, uint64_t *B1_dev,
                uint64_t *B2_dev);
/* Staged pruned round (replaces scheduler.run_round's single manager pass
 * for one Boruvka round, scheduler.py:268-335).  Rank r of `world` scans a contiguous
 * 1/world share of each phase's tile-pair items; the caller combines between steps:
 *   1. nnm_bv_round_bound: phase-1 item list (identical on every rank) and the bound pass
 *      over this rank's share -> *out_caps (device, *out_count uint32 = fp32 bits of each
 *      component's upper bound; NULL / 0 off the tensor-core path).  Caller: all-reduce
 *      MIN (as int32: non-negative float bits order as integers).
 *   2. nnm_bv_round_phase1(caps = the combined array, NULL: this rank's own): exact
 *      phase-1 scan of the share -> (B1, B2).  Caller: G1 = min_r B1_r, G2 = min_r
 *      nnm_bv_second(...) (two all-reduce MIN).
 *   3. nnm_bv_round_phase2(G1, G2): component bounds from the combined keys, phase-2 list
 *      (identical on every rank), (B1, B2) = (G1, G2) plus this rank's phase-2 share;
 *      *out_cache / *out_count: this round's tile-pair cache entries (uint32, NULL / 0
 *      when world == 1 or the cache is off).  Caller: all-reduce MAX of the cache buffer,
 *      then nnm_bv_cache_scatter (required before the next round's step 1), and the key
 *      combine again -> nnm_bv_finish_round(G1, G2).
 * Steps out of order raise NNM_E_INVALID. */
int nnm_bv_round_bound(nnm_dataset *ds, int32_t rank, int32_t world, uint32_t **out_caps,
                       int64_t *out_count);
int nnm_bv_round_phase1(nnm_dataset *ds, int32_t rank, int32_t world, const uint32_t *caps_dev,
                        uint64_t *B1_dev, uint64_t *B2_dev);
int nnm_bv_round_phase2(nnm_dataset *ds, int32_t rank, int32_t world, const uint64_t *G1_dev,
                        const uint64_t *G2_dev, uint64_t *B1_dev, uint64_t *B2_dev,
                        uint32_t **out_cache, int64_t *out_count);
int nnm_bv_cache_scatter(nnm_dataset *ds);
/* B2 contribution for the global second-best: B2c[i] = (B1loc[i] == B1glob[i]) ? B2loc[i] : B1loc[i] */
int nnm_bv_second(nnm_dataset *ds, const uint64_t *B1loc_dev, const uint64_t *B2loc_dev,
                  const uint64_t *B1glob_dev, uint64_t *B2c_dev);
/* finish a round from the global keys; *out_edges = MST edges added (0: converged) */
int nnm_bv_finish_round(nnm_dataset *ds, const uint64_t *B1_dev, const uint64_t *B2_dev,
                        int64_t *out_edges);
/* sort + replay the accumulated edges into the merge log (kl1 truncation) */
int nnm_bv_end(nnm_dataset *ds, int64_t kl1, nnm_merge *out_merges, int64_t *out_n_merges,
               int64_t *out_assign, int64_t *out_rounds, int32_t *out_stop, nnm_stats *stats);

/* Single-process multi-GPU run (engine.run with RunConfig.n_gpus > 1): one dataset
 * replica per device (several replicas may share a device), the staged pruned round over
 * 1/n_rep shares with the exchanges done by kernels reading the other replicas' buffers
 * through peer memory (NVLink / NVSwitch).  Outputs and errors as nnm_run; the round
 * path (kl2 / kl3 / kl4) runs on replicas[0] alone.  Results are byte-identical to
 * nnm_run on one replica. */
int nnm_run_multi(nnm_dataset **replicas, int32_t n_replicas, int32_t metric,
                  const nnm_constraints *constraints, int64_t pairs_per_batch, int32_t flags,
                  nnm_merge *out_merges, int64_t *out_n_merges, int64_t *out_assign,
                  int64_t *out_rounds, int32_t *out_stop, nnm_round_counters *out_counters,
                  int64_t counters_cap, int64_t *out_n_counters, nnm_stats *stats);

/* Per-round records of the last nnm_run on ds (*out_n = rounds recorded; at most cap copied). */
int nnm_round_log(nnm_dataset *ds, nnm_round_stat *out, int64_t cap, int64_t *out_n);

/* ---- CSV ingestion (dataio.py:49-116 load_dataset) ----
 * Parses a delimited text file with the reference's exact rules and messages:
 * str.splitlines() line boundaries, blank lines skipped, header sniffed (any field
 * not a Python float()), id column by header name or 0-based index, Python float()
 * grammar (underscores, inf/nan), errors cite 1-based physical lines (NNM_E_INVALID,
 * message in nnm_last_error()).  Multi-threaded; threads <= 0 uses every core.
 * nnm_csv_fetch copies the n x d row-major values and, with ids, the concatenated
 * UTF-8 ids plus n+1 offsets (*id_bytes total).  No GPU involved. */
typedef struct nnm_csv nnm_csv;
int nnm_csv_load(const char *path, char delimiter, const char *id_column, int32_t threads,
                 nnm_csv **out, int64_t *n, int64_t *d, int32_t *has_ids, int64_t *id_bytes);
int nnm_csv_fetch(nnm_csv *table, double *values, char *id_buf, int64_t *id_offsets);
int nnm_csv_free(nnm_csv *table);

/* ---- Dataset validation (model.py:29-76) ----
 * Index of the first non-finite element of count float64 values (-1 if all are
 * finite); the Dataset constructor turns it into "non-finite feature value in
 * row r".  Host-only, multi-threaded (threads <= 0: every core). */
int nnm_first_nonfinite(const double *X, int64_t count, int32_t threads, int64_t *out_index);

/* ---- diagnostics ----
 * Sustained FP32 (FFMA2) throughput of `device` in TFLOP/s: the roofline
 * denominator for the screening scan, which runs on the FP32 pipe. */
int nnm_measure_fp32_peak(int32_t device, double *tflops);

/* Error-model probe of the tensor-core screen (Euclidean, d <= 29): runs the scan
 * kernel on the given tile pairs of the library's kd view (items: n_items (I, J)
 * int32 pairs, tile indices < T where T(T+1)/2 is nnm_bv_begin's tile-pair count),
 * dumps the accumulators and compares each real pair with its exact FP64 value.
 * out[0] = max |v - S| / bound, out[1] = pairs whose key exceeds S (must be 0),
 * out[2] = pairs checked.  Resets any staged Boruvka state of the dataset. */
int nnm_tc_probe(nnm_dataset *ds, const int32_t *items, int64_t n_items, double *out);

#ifdef __cplusplus
}
#endif
#endif /* NNM_H */
