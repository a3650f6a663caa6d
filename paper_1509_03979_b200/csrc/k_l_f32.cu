// k_l_f32.cu — Tier L kernels and launchers, float instantiation (separate TU for a parallel build).
#define CS_TIER_L_IMPL
#include "tier_l.cuh"

namespace cs {
template cs_status tier_l_apply<float>(OpMeta, int64_t, const float*, float*, void*, size_t, cudaStream_t, bool,
                                     std::atomic<uint64_t>&, std::string&);
template cs_status tier_l_recover<float>(OpMeta, Params, int, const float*, int64_t, float*, int32_t*, cs_report*,
                                       void*, size_t, cudaStream_t, std::atomic<uint64_t>&, std::string&);
template cs_status tier_l_diag_topk<float>(const float*, int64_t, int64_t, uint32_t*, void*, size_t, cudaStream_t,
                                        std::atomic<uint64_t>&, std::string&);
template cs_status tier_l_dist_phase<float>(OpMeta, const DistArgs<float>&, void*, size_t, cudaStream_t,
                                        std::atomic<uint64_t>&, std::string&);
template cs_status tier_l_dist_copy<float>(OpMeta, void*, const int32_t*, const int32_t*, int64_t, int64_t, float*, int,
                                       cudaStream_t, std::atomic<uint64_t>&, std::string&);
}  // namespace cs
