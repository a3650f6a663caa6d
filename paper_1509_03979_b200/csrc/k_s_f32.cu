// k_s_f32.cu — Tier S kernels and launchers, float instantiation (separate TU for a parallel build).
#define CS_TIER_S_IMPL
#include "tier_s.cuh"

namespace cs {
template cs_status s_apply_launch<float>(const OpMeta&, int64_t, const float*, float*, bool, float*, cudaStream_t,
                                       std::atomic<uint64_t>&, std::string&);
template cs_status s_recover_launch<float>(const SRecArgs<float>&, int64_t, cudaStream_t, std::atomic<uint64_t>&,
                                         std::string&);
template cs_status s_diag_topk_launch<float>(const float*, int, int, int, uint32_t*, cudaStream_t,
                                           std::atomic<uint64_t>&, std::string&);
}  // namespace cs
