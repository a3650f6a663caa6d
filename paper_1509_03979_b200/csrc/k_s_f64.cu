// k_s_f64.cu — Tier S kernels and launchers, double instantiation (separate TU for a parallel build).
#define CS_TIER_S_IMPL
#include "tier_s.cuh"

namespace cs {
template cs_status s_apply_launch<double>(const OpMeta&, int64_t, const double*, double*, bool, double*, cudaStream_t,
                                       std::atomic<uint64_t>&, std::string&);
template cs_status s_recover_launch<double>(const SRecArgs<double>&, int64_t, cudaStream_t, std::atomic<uint64_t>&,
                                         std::string&);
template cs_status s_diag_topk_launch<double>(const double*, int, int, int, uint32_t*, cudaStream_t,
                                           std::atomic<uint64_t>&, std::string&);
}  // namespace cs
