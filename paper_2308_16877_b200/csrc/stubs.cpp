// temporary stub (replaced by kmeans.cu)
#include "hpac_offload.h"
#define HPAC_API extern "C" __attribute__((visibility("default")))
HPAC_API int hpac_kmeans_run(const hpac_grid_t*, const hpac_kmeans_problem_t*, const hpac_spec_t*, void*, hpac_kmeans_result_t*, char*, size_t) { return HPAC_ERR_UNSUPPORTED; }
