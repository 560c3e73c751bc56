// ddks_api_kd_b.cu — kd-ordered count instantiations (see ddks_kd.cuh); one translation unit per group of d so
// the builds run in parallel.
#include "ddks_kd.cuh"

namespace ddks_host {
template ddks_status run_count_kd_d<5>(ddks_ctx*, const float*, int64_t, int64_t, int, int, uint64_t*, uint64_t*,
                                         cudaStream_t, bool, unsigned long long*, unsigned long long*);
template ddks_status run_count_kd_d<6>(ddks_ctx*, const float*, int64_t, int64_t, int, int, uint64_t*, uint64_t*,
                                         cudaStream_t, bool, unsigned long long*, unsigned long long*);
}  // namespace ddks_host
