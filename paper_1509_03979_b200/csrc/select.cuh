// select.cuh — support detection and support bookkeeping, written once against
// the context interface (ctx_cta.cuh / ctx_grid.cuh).
//
//  * topk_bits   — radix top-K select (b2): the K largest keys, ties to the
//                  lowest index (R12/R32), MSB-first
//                  8-bit digits over order-preserving magnitude keys, result
//                  written as a bitmask over the index range.
//  * argmax_excl — OMP / OMPR(1) detection (Eq.(6)).
//  * compact     — bitmask -> ascending index list (support merge / prune, b3).
//  * remap       — carry coefficients from one sorted support to another
//                  (warm start, cg1; zeros for new indices).
#pragma once
#include <type_traits>

#include "cs_common.cuh"

namespace cs {

// ---------------------------------------------------------------- top-K ----
// Warp 0 finds, scanning the 256-bin histogram from the top, the digit at which
// the running count reaches `need`; (digit, count above it, count at it) are
// broadcast through pick[0..2].  All threads of the block must call.
CS_DEV void hist_pick(const unsigned* h, int64_t* pick, int64_t need, int64_t& dsel, int64_t& cum,
                      int64_t& hsel) {
  if (threadIdx.x < 32) {
    const int l = threadIdx.x;
    unsigned c[8];
    int64_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) { c[i] = h[255 - 8 * l - i]; s += c[i]; }
    int64_t inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (l >= o) inc += t;
    }
    const int64_t total = __shfl_sync(0xffffffffu, inc, 31);
    unsigned ball = __ballot_sync(0xffffffffu, inc >= need);
    int fl = ball ? __ffs(ball) - 1 : -1;
    if (l == fl) {
      int64_t cu = inc - s;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (cu + c[i] >= need) { pick[0] = 255 - 8 * l - i; pick[1] = cu; pick[2] = c[i]; break; }
        cu += c[i];
      }
    }
    if (fl < 0 && l == 0) {  // fewer candidates than need: take everything
      pick[0] = 0; pick[1] = total - h[0]; pick[2] = h[0];
    }
  }
  __syncthreads();
  dsel = pick[0];
  cum = pick[1];
  hsel = pick[2];
  __syncthreads();
}

CS_DEV void hist_add_warp(unsigned* hist, unsigned digit) {
  // warp-aggregated: one shared atomic per distinct digit in the warp
  unsigned peers = __match_any_sync(__activemask(), digit);
  int leader = __ffs(peers) - 1;
  if ((int)(threadIdx.x & 31) == leader) atomicAdd(&hist[digit], (unsigned)__popc(peers));
}

// ---- two-pass top-K for the CTA context ----
// pass 1: 1024-bin histogram of a 10-bit digit that is monotone in the key;
//         the boundary bin b1 has count(> b1) < K <= count(>= b1);
// pass 2: indices with digit > b1 are selected (ballot -> bitmask), those with
//         digit == b1 are appended to a candidate list;
// then the `need` = K - count(> b1) largest candidates by (key, lowest index)
// are found by a byte radix select over the candidate list only.
// Returns false (nothing written) if the boundary bin holds > TOPK_CAP entries
// or fewer than K keys are non-zero; the caller then runs the radix path.
// `visit(f)` calls f(index, key) once for every element, in any order and from any
// thread (key 0 = never select); `nbits` = size of the index range of out_bits.
template <class Ctx, typename Key, class Visit>
CS_DEV bool topk_cta_fast_v(Ctx& ctx, int nbits, int K, Visit&& visit, uint32_t* out_bits) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  unsigned* h = shp(ctx.h1);
  Key* ck = reinterpret_cast<Key*>(shp(ctx.ckey));
  int* ci = shp(ctx.cidx);
  int* cc = shp(ctx.ccnt);
  int64_t* pk = shp(ctx.pick);
  for (int i = tid; i < TOPK_BINS; i += nt) h[i] = 0;
  if (tid == 0) cc[0] = 0;
  __syncthreads();
  visit([&](int i, Key k) {
    (void)i;
    // plain shared atomics: the 10-bit digits of a warp's keys rarely coincide, and the
    // match_any aggregation cost more than the collisions it saves (c4: -2.3 %)
    if (k) atomicAdd(&h[key_digit10(k)], 1u);
  });
  __syncthreads();
  if (warp == 0) {
    // lane l owns bins [1023 - 32 l - 31, 1023 - 32 l], scanned from the top; its sum is
    // read in a lane-rotated order ((i + l) mod 32) so that the 32 lanes hit 32 different
    // banks (a fixed order is a 32-way bank conflict: the lanes' ranges are 32 words apart)
    int s = 0;
#pragma unroll 8
    for (int i = 0; i < 32; ++i) s += (int)h[TOPK_BINS - 1 - 32 * lane - ((i + lane) & 31)];
    int inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    const unsigned ball = __ballot_sync(0xffffffffu, inc >= K);
    const int fl = ball ? __ffs(ball) - 1 : -1;
    if (lane == 0 && fl < 0) { pk[0] = -1; pk[1] = 0; pk[2] = 0; }
    if (fl >= 0) {
      // the boundary bin inside lane fl's 32 bins, found by the whole warp (one bin per
      // lane, a warp scan and a ballot) instead of a serial 32-step search
      const int base = __shfl_sync(0xffffffffu, inc - s, fl);   // keys above lane fl's bins
      const int b = TOPK_BINS - 1 - 32 * fl - lane;
      const int c = (int)h[b];
      int ic = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, ic, o);
        if (lane >= o) ic += t;
      }
      const unsigned bb = __ballot_sync(0xffffffffu, base + ic >= K);
      const int fb = __ffs(bb) - 1;   // exists: lane fl's bins reach K
      if (lane == fb) { pk[0] = b; pk[1] = base + ic - c; pk[2] = c; }
    }
  }
  const int nwords = (nbits + 31) >> 5;
  for (int w = tid; w < nwords; w += nt) out_bits[w] = 0u;
  __syncthreads();
  const int b1 = (int)pk[0], above = (int)pk[1], inb = (int)pk[2];
  __syncthreads();  // pick[] is reused by later collectives
  if (b1 < 0 || inb > TOPK_CAP) return false;
  const int need = K - above;
  visit([&](int i, Key k) {
    if (!k) return;
    const int d = (int)key_digit10(k);
    if (d > b1) {
      atomicOr(&out_bits[i >> 5], 1u << (i & 31));
    } else if (d == b1) {
      const int at = atomicAdd(cc, 1);
      ck[at] = k;
      ci[at] = i;
    }
  });
  __syncthreads();
  const int C = cc[0];
  if (need >= C) {
    for (int c = tid; c < C; c += nt) atomicOr(&out_bits[ci[c] >> 5], 1u << (ci[c] & 31));
    __syncthreads();
    return true;
  }
  if (C <= 128) {
    // few candidates: every candidate counts the candidates ranked above it (key descending,
    // index ascending — R12, R32; a broadcast read of the list) and is taken iff fewer than
    // `need` are — one barrier instead of the byte radix passes below (four barriers each)
    for (int c = tid; c < C; c += nt) {
      const Key kc = ck[c];
      const int ic = ci[c];
      int above_c = 0;
      for (int j = 0; j < C; ++j) {
        const Key kj = ck[j];
        above_c += (kj > kc) || (kj == kc && ci[j] < ic);
      }
      if (above_c < need) atomicOr(&out_bits[ic >> 5], 1u << (ic & 31));
    }
    __syncthreads();
    return true;
  }
  // MSB-first byte radix select of the `need` largest candidate keys
  unsigned* hist = shp(ctx.hist);
  constexpr int NB = (int)sizeof(Key) * 8;
  Key prefix = 0, pmask = 0;
  int start = NB - 8;
  if constexpr (sizeof(Key) == 4) {
    // fp32 keys: the digit is key >> 21, so every candidate shares bits 31..21 — the
    // top byte is common and the select starts at bits 23..16
    pmask = (Key)0xFF000000u;
    prefix = ck[0] & pmask;
    start = 16;
  }
  int64_t needr = need, n_eq = 0;
  for (int shift = start; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += nt) hist[i] = 0;
    __syncthreads();
    for (int c = tid; c < C; c += nt) {
      const Key k = ck[c];
      if ((k & pmask) == prefix) hist_add_warp(hist, (unsigned)((k >> shift) & 255));
    }
    __syncthreads();
    int64_t dsel, cum, hsel;
    hist_pick(hist, pk, needr, dsel, cum, hsel);
    needr -= cum;
    n_eq = hsel;
    prefix |= (Key)dsel << shift;
    pmask |= (Key)255 << shift;
  }
  const Key thr = prefix;  // the need-th largest candidate key
  for (int c = tid; c < C; c += nt) {
    const Key kc = ck[c];
    bool take = kc > thr;
    if (kc == thr) {
      if (n_eq == needr) {
        take = true;
      } else {  // ties: the lowest indices win (R12, R32)
        const int ic = ci[c];
        int below = 0;
        for (int j = 0; j < C; ++j) below += (ck[j] == thr) && (ci[j] < ic);
        take = below < needr;
      }
    }
    if (take) atomicOr(&out_bits[ci[c] >> 5], 1u << (ci[c] & 31));
  }
  __syncthreads();
  return true;
}

template <class Ctx, class KeyFn>
CS_DEV bool topk_cta_fast(Ctx& ctx, int n, int K, KeyFn key, uint32_t* out_bits) {
  using Key = decltype(key(int64_t(0)));
  return topk_cta_fast_v<Ctx, Key>(ctx, n, K, [&](auto&& f) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) f(i, key(i));
  }, out_bits);
}

// key(i) for i in [0, n); key 0 means "never select".  Requires at least K
// non-zero keys.  out_bits must hold ceil(n/32) words; fully overwritten.
// No vector loader (the scalar key(i) path everywhere).
struct NoKey4 {};

// key4(q) -> uint4 of keys 4q .. 4q+3 (32-bit keys, n % 4 == 0): the radix passes and the
// final bitmask pass then move 16 bytes per load — the grid path is latency-bound on its key
// loads (ncu: long_scoreboard at the key read), so four keys per load and sixteen per thread
// in flight.  key(i) serves the tie path.
template <class Ctx, class KeyFn, class Key4Fn = NoKey4>
CS_DEV void topk_bits(Ctx& ctx, int64_t n, int64_t K, KeyFn key, uint32_t* out_bits, bool try_fast = true,
                      Key4Fn key4 = Key4Fn{}) {
  if constexpr (Ctx::kTopkFast) {
    if (try_fast && topk_cta_fast(ctx, (int)n, (int)K, key, out_bits)) return;
  }
  using Key = decltype(key(int64_t(0)));
  constexpr bool V4 = !std::is_same<Key4Fn, NoKey4>::value;
  static_assert(!V4 || sizeof(Key) == 4, "the vector loader serves 32-bit keys");
  constexpr int NB = (int)sizeof(Key) * 8;
  Key prefix = 0, pmask = 0;
  int64_t need = K;
  int64_t n_eq = 0;
  const int64_t t0 = ctx.gtid, st = ctx.gnthr, gw = ctx.gwarp, gnw = ctx.gnwarps;
  const int lane = threadIdx.x & 31;
  unsigned* hist = ctx.hist_ptr();
  for (int shift = NB - 8; shift >= 0; shift -= 8) {
    ctx.hist_clear();
    if constexpr (V4) {
      constexpr int UQ = 4;  // 16 keys in flight per thread
      const int64_t n4 = n >> 2;
      for (int64_t q0 = t0; q0 < n4; q0 += UQ * st) {
        uint4 kv[UQ];
#pragma unroll
        for (int u = 0; u < UQ; ++u) {
          const int64_t q = q0 + u * st;
          kv[u] = (q < n4) ? key4(q) : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int u = 0; u < UQ; ++u) {
          const int64_t q = q0 + u * st;
          if (q < n4) {
            const Key kk[4] = {(Key)kv[u].x, (Key)kv[u].y, (Key)kv[u].z, (Key)kv[u].w};
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if ((kk[e] & pmask) == prefix) hist_add_warp(hist, (unsigned)((kk[e] >> shift) & 255));
          }
        }
      }
    } else {
      constexpr int UK = 8;  // keys in flight per thread before the histogram updates
      for (int64_t i0 = t0; i0 < n; i0 += UK * st) {
        Key kv[UK];
#pragma unroll
        for (int u = 0; u < UK; ++u) {
          const int64_t i = i0 + u * st;
          kv[u] = (i < n) ? key(i) : Key(0);
        }
#pragma unroll
        for (int u = 0; u < UK; ++u) {
          const int64_t i = i0 + u * st;
          if (i < n && (kv[u] & pmask) == prefix) hist_add_warp(hist, (unsigned)((kv[u] >> shift) & 255));
        }
      }
    }
    ctx.hist_done();  // merged counts now in ctx.hist_smem()
    int64_t dsel, cum, hsel;
    hist_pick(ctx.hist_smem(), ctx.pick, need, dsel, cum, hsel);
    need -= cum;
    n_eq = hsel;
    prefix |= (Key)dsel << shift;
    pmask |= (Key)255 << shift;
  }
  const Key thr = prefix;  // the K-th largest key; take `need` of the n_eq equal ones
  const int64_t nwords = (n + 31) >> 5;
  if (n_eq == need) {
    // common case: every key >= thr is selected
    if constexpr (V4) {
      // 128 keys per warp step: lane l holds keys 4 (32 g + l) .. +3, i.e. a nibble of word
      // 4 g + l / 8; eight lanes OR their nibbles into the word
      const int64_t ng = n >> 7;
      for (int64_t g = gw; g < ng; g += gnw) {
        const uint4 k = key4(g * 32 + lane);
        uint32_t v = ((uint32_t)((Key)k.x >= thr) | ((uint32_t)((Key)k.y >= thr) << 1) |
                      ((uint32_t)((Key)k.z >= thr) << 2) | ((uint32_t)((Key)k.w >= thr) << 3))
                     << (4 * (lane & 7));
        v |= __shfl_xor_sync(0xffffffffu, v, 1);
        v |= __shfl_xor_sync(0xffffffffu, v, 2);
        v |= __shfl_xor_sync(0xffffffffu, v, 4);
        if ((lane & 7) == 0) out_bits[g * 4 + (lane >> 3)] = v;
      }
      for (int64_t w = ng * 4 + gw; w < nwords; w += gnw) {   // the tail words
        int64_t i = w * 32 + lane;
        bool s = (i < n) && (key(i) >= thr);
        uint32_t b = __ballot_sync(0xffffffffu, s);
        if (lane == 0) out_bits[w] = b;
      }
    } else {
      for (int64_t w = gw; w < nwords; w += gnw) {
        int64_t i = w * 32 + lane;
        bool s = (i < n) && (key(i) >= thr);
        uint32_t b = __ballot_sync(0xffffffffu, s);
        if (lane == 0) out_bits[w] = b;
      }
    }
    ctx.sync();
    return;
  }
  // ties at the threshold: the lowest-index `need` equal keys win.
  // warp-contiguous chunks of words, chunk order == index order
  const int64_t per = (nwords + gnw - 1) / gnw;
  const int64_t w0 = gw * per, w1 = min(nwords, w0 + per);
  int64_t cnt = 0;
  for (int64_t w = w0; w < w1; ++w) {
    int64_t i = w * 32 + lane;
    bool e = (i < n) && (key(i) == thr);
    cnt += __popc(__ballot_sync(0xffffffffu, e));
  }
  int64_t tot;
  int64_t base = ctx.excl_scan(lane == 0 ? cnt : 0, &tot);
  base = __shfl_sync(0xffffffffu, base, 0);
  for (int64_t w = w0; w < w1; ++w) {
    int64_t i = w * 32 + lane;
    Key k = (i < n) ? key(i) : Key(0);
    bool e = (i < n) && (k == thr);
    uint32_t em = __ballot_sync(0xffffffffu, e);
    int64_t rank = base + __popc(em & ((1u << lane) - 1u));
    bool s = (i < n) && ((k > thr) || (e && rank < need));
    uint32_t b = __ballot_sync(0xffffffffu, s);
    if (lane == 0) out_bits[w] = b;
    base += __popc(em);
  }
  ctx.sync();
}

// ---------------------------------------------------------------- argmax ---
// index of the largest key(i) over i in [0, n), ties -> lowest i; -1 if none.
template <class Ctx, class KeyFn>
CS_DEV int64_t argmax_key(Ctx& ctx, int64_t n, KeyFn key) {
  using Key = decltype(key(int64_t(0)));
  Key bk = 0;
  int64_t bi = -1;
  const int64_t t0 = ctx.gtid, st = ctx.gnthr;
  for (int64_t i = t0; i < n; i += st) {
    Key k = key(i);
    if (k > bk) { bk = k; bi = i; }  // increasing i per thread: first max kept
  }
  return ctx.argmax(bk, bi);
}

// -------------------------------------------------------------- compaction --
// For every set bit i of bits[0..n) in ascending order, call emit(rank, i).
// Returns the number of set bits (uniform).
template <class Ctx, class Emit>
CS_DEV int64_t compact_bits(Ctx& ctx, const uint32_t* bits, int64_t n, Emit emit) {
  const int64_t nwords = (n + 31) >> 5;
  if constexpr (Ctx::kTopkFast) {
    if (nwords <= 32) {
      // CTA, at most 32 words (the prune over |T| <= 1024 positions): warp 0 alone — lane w
      // takes word w, a warp scan of the popcounts gives its output offset; the total is
      // broadcast through the pick slot with the one closing barrier
      int64_t* pk = shp(ctx.pick);
      if (threadIdx.x < 32) {
        const int w = (int)threadIdx.x;
        uint32_t b = w < nwords ? bits[w] : 0u;
        if (w == nwords - 1 && (n & 31)) b &= (1u << (n & 31)) - 1u;
        const int c = __popc(b);
        int inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, inc, o);
          if (w >= o) inc += t;
        }
        int64_t pos = inc - c;
        while (b) {
          const int t = __ffs(b) - 1;
          b &= b - 1;
          emit(pos++, (int64_t)w * 32 + t);
        }
        if (w == 31) pk[3] = inc;
      }
      __syncthreads();
      const int64_t tot = pk[3];
      __syncthreads();   // pick[] is reused by later collectives
      return tot;
    }
  }
  const int64_t nthr = ctx.gnthr;
  const int64_t per = (nwords + nthr - 1) / nthr;
  const int64_t w0 = (int64_t)ctx.gtid * per, w1 = min(nwords, w0 + per);
  int64_t cnt = 0;
  for (int64_t w = w0; w < w1; ++w) {
    uint32_t b = bits[w];
    if (w == nwords - 1 && (n & 31)) b &= (1u << (n & 31)) - 1u;
    cnt += __popc(b);
  }
  int64_t tot;
  int64_t pos = ctx.excl_scan(cnt, &tot);
  for (int64_t w = w0; w < w1; ++w) {
    uint32_t b = bits[w];
    if (w == nwords - 1 && (n & 31)) b &= (1u << (n & 31)) - 1u;
    while (b) {
      int t = __ffs(b) - 1;
      b &= b - 1;
      emit(pos++, w * 32 + t);
    }
  }
  ctx.sync();
  return tot;
}

// ---------------------------------------------------------------- remap ----
// new_vals[i] = old_vals[pos of new_list[i] in old_list] or 0 (both lists ascending)
template <class Ctx, typename T>
CS_DEV void remap(Ctx& ctx, const int* old_list, const T* old_vals, int n_old,
                  const int* new_list, T* new_vals, int n_new) {
  const int t0 = ctx.gtid, st = ctx.gnthr;
  for (int i = t0; i < n_new; i += st) {
    int e = new_list[i];
    int lo = 0, hi = n_old;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (old_list[mid] < e) lo = mid + 1; else hi = mid;
    }
    new_vals[i] = (lo < n_old && old_list[lo] == e) ? old_vals[lo] : T(0);
  }
  ctx.sync();
}

}  // namespace cs
