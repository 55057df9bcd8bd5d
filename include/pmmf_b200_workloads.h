/*
 * pmmf_b200_workloads.h — seeded synthetic inputs for BASELINE.json's
 * configs (SURVEY.md §8(d) recipes).  Not part of the reference interface;
 * used by bench.py and the tests so that every arm sees identical triplets.
 */
#ifndef PMMF_B200_WORKLOADS_H
#define PMMF_B200_WORKLOADS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pmmf_b200_workload {
  int64_t n;
  int64_t nnz;
  int64_t* rows; /* malloc'ed; release with pmmf_b200_workload_free */
  int64_t* cols;
  double* vals;
} pmmf_b200_workload;

int pmmf_b200_workload_rmat(int32_t scale, int32_t edges_per_vertex, uint64_t seed, double shift,
                            pmmf_b200_workload* out);
int pmmf_b200_workload_dense_spd(int64_t n, int64_t d, uint64_t seed, double shift,
                                 pmmf_b200_workload* out);
int pmmf_b200_workload_rbf(int64_t n, int32_t dim, double bandwidth, uint64_t seed, double shift,
                           pmmf_b200_workload* out);
int pmmf_b200_workload_aniso_grid(int64_t side, double ax, double ay, pmmf_b200_workload* out);
int pmmf_b200_workload_rhs(int64_t n, int32_t count, uint64_t seed, double* out);
void pmmf_b200_workload_free(pmmf_b200_workload* w);

#ifdef __cplusplus
}
#endif

#endif /* PMMF_B200_WORKLOADS_H */
