// operator.cu — placeholder, replaced below
#include "result.cuh"
extern "C" {
int pmmf_b200_operator_create(void*, double, void**, char*, size_t) { return PMMF_INTERNAL; }
int pmmf_b200_operator_apply(void*, int32_t, int64_t, const double*, double*, int32_t, char*, size_t) { return PMMF_INTERNAL; }
int pmmf_b200_operator_zeroed_negatives(void*, int64_t*) { return PMMF_INTERNAL; }
void pmmf_b200_operator_free(void*) {}
int pmmf_b200_solve(const pmmf_b200_coo*, void*, const pmmf_b200_solve_config*, int32_t*, int32_t*, int32_t*, double*, double*, char*, size_t) { return PMMF_INTERNAL; }
}
