// k_l_f64.cu — Tier L kernels and launchers, double instantiation (separate TU for a parallel build).
#define CS_TIER_L_IMPL
#include "tier_l.cuh"

namespace cs {
template cs_status tier_l_apply<double>(OpMeta, int64_t, const double*, double*, void*, size_t, cudaStream_t, bool,
                                     std::atomic<uint64_t>&, std::string&);
template cs_status tier_l_recover<double>(OpMeta, Params, int, const double*, int64_t, double*, int32_t*, cs_report*,
                                       void*, size_t, cudaStream_t, std::atomic<uint64_t>&, std::string&);
template cs_status tier_l_diag_topk<double>(const double*, int64_t, int64_t, uint32_t*, void*, size_t, cudaStream_t,
                                        std::atomic<uint64_t>&, std::string&);
}  // namespace cs
