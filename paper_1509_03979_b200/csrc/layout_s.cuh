// layout_s.cuh — the N-dependent (K-independent) head of the Tier S shared-memory
// layout, as compile-time offsets: the sandwich addresses the FFT buffer, twiddle
// tables and operator metadata as cs_smem_base + constant (no registers spent on
// pointers).  tier_s.cuh appends the pursuit arrays after `end`.
#pragma once
#include "cs_common.cuh"

namespace cs {

struct SFix {
  int64_t Z, twLlo, twLhi, tw4lo, tw4hi, sign, rmask, prefix, usel, tw16, redd, redi, redk, hist, pick, h1, ckey, cidx, ccnt, zero, end;
};

__host__ __device__ constexpr int64_t al16(int64_t x) { return (x + 15) / 16 * 16; }

template <typename T> __host__ __device__ constexpr SFix s_fixed(int64_t N) {
  const int64_t L = N / 2, nw = (N + 31) / 32, cs2 = sizeof(T) * 2;
  SFix s{};
  int64_t o = 0;
  s.Z = o;      o = al16(o + L * cs2);
  s.twLlo = o;  o = al16(o + 64 * cs2);
  s.twLhi = o;  o = al16(o + (L >= 64 ? L / 64 : 1) * cs2);
  s.tw4lo = o;  o = al16(o + 64 * cs2);
  s.tw4hi = o;  o = al16(o + (L / 128 + 1) * cs2);
  s.sign = o;   o = al16(o + nw * 4);
  s.rmask = o;  o = al16(o + nw * 4);
  s.prefix = o; o = al16(o + nw * 4);
  // row selection in the fused pass's unit order (sandwich_cta.cuh sw_fused): one word per
  // thread, bit 8 it + q = [DCT index q of the thread's unit it is a row]
  s.usel = o;   o = al16(o + 512 * 4);
  // twiddles of the first twiddled radix-16 pass (stride Ns1 <= 16): [r][k] = W_{16 Ns1}^{r k}
  s.tw16 = o;   o = al16(o + 256 * cs2);
  s.redd = o;   o = al16(o + 2 * 64 * 8);  // two banks of [4][16] (CG) or [32] (sum): one barrier per reduction
  s.redi = o;   o = al16(o + 33 * 8);
  s.redk = o;   o = al16(o + 32 * 8);
  s.hist = o;   o = al16(o + 256 * 4);
  s.pick = o;   o = al16(o + 4 * 8);
  // two-pass top-K (select.cuh topk_cta_fast): first-digit histogram, candidates
  s.h1 = o;     o = al16(o + TOPK_BINS * 4);
  s.ckey = o;   o = al16(o + (int64_t)TOPK_CAP * sizeof(typename KeyT<T>::type));
  s.cidx = o;   o = al16(o + (int64_t)TOPK_CAP * 4);
  s.ccnt = o;   o = al16(o + 16);
  s.zero = o;   o = al16(o + 16);  // an int 0 read through volatile (sandwich_cta.cuh opaque_tid)
  s.end = o;
  return s;
}

// sqrt(2^e) as a constant expression
__host__ __device__ constexpr double sqrt_pow2(int e) {
  double r = 1.0;
  const int h = (e >= 0 ? e : -e) / 2;
  for (int i = 0; i < h; ++i) r *= 2.0;
  if ((e >= 0 ? e : -e) % 2) r *= 1.41421356237309504880;
  return e >= 0 ? r : 1.0 / r;
}

}  // namespace cs
