// fft_cta.cuh — CTA-cooperative Stockham FFT in shared memory (sm_100a).
//
// The DCT-II of the sensing operator is "speeded by FFT"; this is
// that FFT, written for one CTA holding B interleaved complex sequences of
// length L = 2^LOG2L in shared memory (element n of sequence b at logical
// index n*B + b).
//
// Design:
//  * compile-time L, B and E (complex elements held per thread): all index math
//    folds to shifts/masks; each thread owns E elements per pass, so a pass is
//    "load E -> barrier -> store E" in place (no ping-pong buffer: the whole
//    8192-point fp32 transform fits in 64 KB and two CTAs fit per SM);
//  * ceil(LOG2L / log2 E) radix passes with balanced radices <= E (8192 points,
//    E = 32: radix 32-16-16, three shared-memory round trips);
//  * Stockham autosort: for item (b, j), k = j mod Ns,
//      v[r] = x[j + r L/R] * W_{Ns R}^{r k},  V = DFT_R(v),  x'[(j-k)R + k + r Ns] = V[r];
//  * the R-point DFT is an unrolled radix-2 DIF network with compile-time
//    twiddles (output in bit-reversed register order, undone at compile time);
//  * bank-conflict-free: every shared access goes through the XOR swizzle
//    swz(a) = a ^ (((a >> 4) ^ (a >> 5)) & (S - 1)), S = complex slots per
//    128-byte row (16 fp32, 8 fp64) — conflict-free for every load and store
//    pattern of every pass (checked exhaustively);
//  * twiddles: W_L^m = hi[m >> 6] * lo[m & 63] from a two-level table in shared
//    memory (double-precision sincospi at kernel start), one lookup per item;
//    the powers W^{2k..(R-1)k} streamed (few live registers, see tw_stream).
#pragma once
#include "cs_common.cuh"

namespace cs {

template <typename T> CS_DEV int swz(int a) {
  constexpr int S = (sizeof(T) == 4) ? 15 : 7;
  return a ^ (((a >> 4) ^ (a >> 5)) & S);
}

// swz as a constexpr (compile-time offsets).  swz is linear over GF(2): for
// bit-disjoint a and c, swz(a | c) = swz(a) ^ swz(c) — so a per-thread swz(base)
// plus a compile-time swz(c) addresses every element of a pass (one XOR, or none
// when c has no bits in 4..8).
template <typename T> __host__ __device__ constexpr int swz_c(int a) {
  return a ^ (((a >> 4) ^ (a >> 5)) & ((sizeof(T) == 4) ? 15 : 7));
}

template <typename T> struct TwTable {
  const C2<T>* lo;  // W^i, i < 64
  const C2<T>* hi;  // W^{64 i}
  CS_DEV C2<T> operator()(int m) const { return cmul<T>(hi[m >> 6], lo[m & 63]); }
};

// Fill lo[64], hi[nhi] with W_den^i = exp(-2 pi i * i / den).
CS_DEV double2 tw_value(int i, int64_t den) {   // entry i of lo[64] | hi[] (fp64)
  int64_t m = (i < 64) ? i : (int64_t)(i - 64) * 64;
  double s, c;
  sincospi(-2.0 * (double)(m % den) / (double)den, &s, &c);
  return make_double2(c, s);
}
template <typename T>
CS_DEV void tw_init(C2<T>* lo, C2<T>* hi, int64_t den, int nhi, int tid, int nthr) {
  for (int i = tid; i < 64 + nhi; i += nthr) {
    const double2 v = tw_value(i, den);
    C2<T> w = mk<T>((T)v.x, (T)v.y);
    if (i < 64) lo[i] = w; else hi[i - 64] = w;
  }
}

// ---- compile-time twiddles of the radix-2 network: W_32^t, t in [0, 16) ----
template <typename T, int t, bool INV> CS_DEV C2<T> w32c() {
  constexpr double c[16] = {1.0, 0.98078528040323044913, 0.92387953251128675613, 0.83146961230254523708,
                            0.70710678118654752440, 0.55557023301960222474, 0.38268343236508977173,
                            0.19509032201612826785, 0.0, -0.19509032201612826785, -0.38268343236508977173,
                            -0.55557023301960222474, -0.70710678118654752440, -0.83146961230254523708,
                            -0.92387953251128675613, -0.98078528040323044913};
  constexpr double s[16] = {0.0, 0.19509032201612826785, 0.38268343236508977173, 0.55557023301960222474,
                            0.70710678118654752440, 0.83146961230254523708, 0.92387953251128675613,
                            0.98078528040323044913, 1.0, 0.98078528040323044913, 0.92387953251128675613,
                            0.83146961230254523708, 0.70710678118654752440, 0.55557023301960222474,
                            0.38268343236508977173, 0.19509032201612826785};
  return mk<T>((T)c[t], INV ? (T)s[t] : (T)(-s[t]));
}

template <typename T, int t32, bool INV> CS_DEV C2<T> tw_apply(C2<T> a) {
  if constexpr (t32 == 0) {
    return a;
  } else if constexpr (t32 == 8) {
    return mul_mi<T, INV>(a);
  } else if constexpr (t32 == 4 || t32 == 12) {
    constexpr T h = (T)0.70710678118654752440;
    constexpr T sx = (t32 == 4) ? (T)1 : (T)-1;
    constexpr T sy = INV ? (T)1 : (T)-1;
    if constexpr (sizeof(T) == 4)   // a (h sx + i h sy): one paired multiply + one paired FMA
      return cmul<T>(a, mk<T>(h * sx, h * sy));
    else
      return mk<T>(h * (sx * a.x - sy * a.y), h * (sx * a.y + sy * a.x));
  } else {
    return cmul<T>(a, w32c<T, t32, INV>());
  }
}

template <typename T, int R, int H, int S, int t, bool INV> CS_DEV void dif_bfly(C2<T>* v) {
  if constexpr (t < H) {
    C2<T> a = v[S + t], b = v[S + t + H];
    v[S + t] = cadd<T>(a, b);
    v[S + t + H] = tw_apply<T, t * (32 / (2 * H)), INV>(csub<T>(a, b));
    dif_bfly<T, R, H, S, t + 1, INV>(v);
  }
}
template <typename T, int R, int H, int S, bool INV> CS_DEV void dif_blocks(C2<T>* v) {
  if constexpr (S < R) {
    dif_bfly<T, R, H, S, 0, INV>(v);
    dif_blocks<T, R, H, S + 2 * H, INV>(v);
  }
}
template <typename T, int R, int H, bool INV> CS_DEV void dif_stages(C2<T>* v) {
  if constexpr (H >= 1) {
    dif_blocks<T, R, H, 0, INV>(v);
    dif_stages<T, R, H / 2, INV>(v);
  }
}
template <int R> __host__ __device__ constexpr int bitrev(int r) {
  int o = 0;
  for (int b = 1, rb = R >> 1; b < R; b <<= 1, rb >>= 1)
    if (r & b) o |= rb;
  return o;
}
// in-register R-point DFT (R <= 32); X_r lands at v[bitrev<R>(r)]
template <typename T, int R, bool INV> CS_DEV void dft_reg(C2<T>* v) { dif_stages<T, R, R / 2, INV>(v); }

// v[r] *= w1^r for r < R, streaming the powers so only a handful of registers hold
// twiddles: w^1..w^3 and a running w^(4a) (product depth <= R/4 + 2).
template <typename T, int R> CS_DEV void tw_stream(C2<T>* v, C2<T> w1) {
  v[1] = cmul<T>(v[1], w1);
  if constexpr (R > 2) {
    const C2<T> w2 = cmul<T>(w1, w1);
    const C2<T> w3 = cmul<T>(w2, w1);
    v[2] = cmul<T>(v[2], w2);
    v[3] = cmul<T>(v[3], w3);
    if constexpr (R > 4) {
      const C2<T> w4 = cmul<T>(w2, w2);
      C2<T> cur = w4;
#pragma unroll
      for (int a = 1; a < R / 4; ++a) {
        v[4 * a] = cmul<T>(v[4 * a], cur);
        v[4 * a + 1] = cmul<T>(v[4 * a + 1], cmul<T>(cur, w1));
        v[4 * a + 2] = cmul<T>(v[4 * a + 2], cmul<T>(cur, w2));
        v[4 * a + 3] = cmul<T>(v[4 * a + 3], cmul<T>(cur, w3));
        if (a + 1 < R / 4) cur = cmul<T>(cur, w4);
      }
    }
  }
}

// log2 radix of pass p for a length-2^LOG2L transform with <= 2^LOG2E points per thread
template <int LOG2L, int LOG2E> struct Plan {
  static constexpr int P = (LOG2L + LOG2E - 1) / LOG2E > 0 ? (LOG2L + LOG2E - 1) / LOG2E : 1;
  __host__ __device__ static constexpr int rb(int p) { return LOG2L / P + (p < LOG2L % P ? 1 : 0); }
  __host__ __device__ static constexpr int ns(int p) {  // log2 Ns before pass p
    int s = 0;
    for (int q = 0; q < p; ++q) s += rb(q);
    return s;
  }
};

template <typename T, int LOG2L, int LOG2E, int LOG2B, int P, bool INV>
CS_DEV void fft_pass(C2<T>* buf, const TwTable<T>& tw) {
  constexpr int PL = Plan<LOG2L, LOG2E>::P;
  constexpr int RB = Plan<LOG2L, LOG2E>::rb(P);
  constexpr int R = 1 << RB;
  constexpr int NSB = Plan<LOG2L, LOG2E>::ns(P);
  constexpr int Ns = 1 << NSB;
  constexpr int L = 1 << LOG2L;
  constexpr int B = 1 << LOG2B;
  constexpr int NTA = (L * B) >> LOG2E;               // active threads
  constexpr int IPT = (1 << (LOG2E - RB)) > 0 ? (1 << (LOG2E - RB)) : 1;  // items per thread
  constexpr int Lr = L >> RB;
  constexpr int ITEMS = B * Lr;
  static_assert(PL >= 1 && RB <= 5 && RB <= LOG2E, "radix <= 32 and <= E");
  const int tid = threadIdx.x;
  C2<T> v[IPT][R];
  if (tid < NTA) {
#pragma unroll
    for (int it = 0; it < IPT; ++it) {
      const int i = tid + it * NTA;
      if (ITEMS % NTA == 0 || i < ITEMS) {
        const int b = i & (B - 1), j = i >> LOG2B;
        const int sj = swz<T>((j << LOG2B) | b);  // j < Lr: bit-disjoint from (r Lr) << LOG2B
#pragma unroll
        for (int r = 0; r < R; ++r) v[it][r] = buf[sj ^ swz_c<T>((r * Lr) << LOG2B)];
        if constexpr (Ns > 1) {
          const int k = j & (Ns - 1);
          C2<T> w1 = tw(k << (LOG2L - NSB - RB));
          if (INV) w1 = cconj<T>(w1);
          tw_stream<T, R>(v[it], w1);
        }
        dft_reg<T, R, INV>(v[it]);
      }
    }
  }
  __syncthreads();
  if (tid < NTA) {
#pragma unroll
    for (int it = 0; it < IPT; ++it) {
      const int i = tid + it * NTA;
      if (ITEMS % NTA == 0 || i < ITEMS) {
        const int b = i & (B - 1), j = i >> LOG2B;
        const int k = j & (Ns - 1);
        const int sb = swz<T>((((j - k) * R + k) << LOG2B) | b);  // bit-disjoint from (r Ns) << LOG2B
#pragma unroll
        for (int r = 0; r < R; ++r) buf[sb ^ swz_c<T>((r * Ns) << LOG2B)] = v[it][bitrev<R>(r)];
      }
    }
  }
  __syncthreads();
}

template <typename T, int LOG2L, int LOG2E, int LOG2B, int P, bool INV>
CS_DEV void fft_passes(C2<T>* buf, const TwTable<T>& tw) {
  if constexpr (P < Plan<LOG2L, LOG2E>::P) {
    fft_pass<T, LOG2L, LOG2E, LOG2B, P, INV>(buf, tw);
    fft_passes<T, LOG2L, LOG2E, LOG2B, P + 1, INV>(buf, tw);
  }
}

// Full transform of B = 2^LOG2B interleaved sequences (unnormalised; INV = conjugate
// twiddles).  (L * B) >> LOG2E threads participate; all threads must call.
template <typename T, int LOG2L, int LOG2E, int LOG2B, bool INV>
CS_NOINL void fft_cta_t(C2<T>* buf, const TwTable<T> tw) {
  // buffer and tables are shared memory: re-derive them in the shared window (LDS/STS)
  const TwTable<T> ts{shp(tw.lo), shp(tw.hi)};
  fft_passes<T, LOG2L, LOG2E, LOG2B, 0, INV>(shp(buf), ts);
}

// At least 4 points per thread: the grid tier's small tiles (N <= 2^16: 512 points on 256
// threads) otherwise run 7-8 radix-2 passes, each two CTA barriers; radix >= 4 halves the
// barrier chain (c2: 4.30 -> 4.03 ms; 8 or 16 points per thread measured slower).
#ifndef CS_FFT_MIN_LOG2E
#define CS_FFT_MIN_LOG2E 2
#endif
// E for a given (L, B) on an NT-thread block: L*B/NT clamped to [4, 32] and <= L
__host__ __device__ constexpr int fft_log2e(int log2l, int log2b, int log2nt) {
  int e = log2l + log2b - log2nt;
  if (e < CS_FFT_MIN_LOG2E) e = CS_FFT_MIN_LOG2E;
  if (e > 5) e = 5;
  if (e > log2l) e = log2l;
  return e;
}

// Runtime dispatch over LOG2L in [LO, HI] with fixed LOG2B and a 2^LOG2NT-thread block.
template <typename T, int LOG2B, int LOG2NT, int LO, int HI, bool INV>
CS_DEV void fft_cta_dispatch(C2<T>* buf, int log2l, const TwTable<T>& tw) {
  if constexpr (LO <= HI) {
    if (log2l == LO) {
      fft_cta_t<T, LO, fft_log2e(LO, LOG2B, LOG2NT), LOG2B, INV>(buf, tw);
      return;
    }
    fft_cta_dispatch<T, LOG2B, LOG2NT, LO + 1, HI, INV>(buf, log2l, tw);
  }
}

}  // namespace cs
