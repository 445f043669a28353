/* nnm_oracle.h -- CPU restatement of the parclust NNM hot path (TEST INFRASTRUCTURE ONLY).
 * See nnm_oracle.c for the contract.  Integer arguments < 0 mean "unset"; dmax NaN = unset. */
#ifndef NNM_ORACLE_H
#define NNM_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_EUCLIDEAN = 0, ORC_SQEUCLIDEAN = 1, ORC_MANHATTAN = 2, ORC_CHEBYSHEV = 3 };
enum { ORC_STOP_NONE = 0, ORC_STOP_KL1 = 1, ORC_STOP_NO_ELIGIBLE = 2, ORC_STOP_SINGLE_CLUSTER = 3 };

typedef struct { /* model.py:221-238 MergeEvent (step = index in the array) */
  int64_t round, root_a, root_b;
  double dist;
  int64_t new_size, point_a, point_b;
} orc_merge_t;

typedef struct { /* engine.py:187-190 round_counters entry */
  int64_t round, selected, merged, same_root, kl2, kl3, unprocessed;
} orc_round_t;

double orc_internal_distance(int metric, const double *x, const double *y, int d);
double orc_reported(int metric, double internal);
double orc_effective_threshold(int metric, double dmax);
void orc_pairwise(int metric, const double *x, int64_t nx, const double *y, int64_t ny, int d,
                  double *out);
int64_t orc_top_p(const double *X, int64_t n, int d, int metric, const int64_t *roots,
                  const int64_t *sizes, double thr, int64_t kl2, int64_t kl3, int64_t P,
                  int nthreads, double *out_d, int64_t *out_a, int64_t *out_b);
int orc_run(const double *X, int64_t n, int d, int metric, int64_t kl1, int64_t kl2, int64_t kl3,
            int64_t kl4, double dmax, int64_t P, int nthreads, orc_merge_t *out,
            int64_t *out_n_merges, int64_t *out_assign, int64_t *out_rounds, int *out_stop,
            orc_round_t *counters, int64_t counters_cap, int64_t *out_n_counters);
int orc_single_linkage(const double *X, int64_t n, int d, int metric, int64_t kl1, int64_t kl2,
                       int64_t kl3, double dmax, orc_merge_t *out, int64_t *out_n_merges,
                       int64_t *out_assign);
#ifdef __cplusplus
}
#endif
#endif
