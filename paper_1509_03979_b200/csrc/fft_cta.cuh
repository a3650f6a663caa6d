// fft_cta.cuh — CTA-cooperative radix-16 Stockham FFT in shared memory (sm_100a).
//
// The DCT-II of the sensing operator is "speeded by FFT"; this is
// that FFT, written for one CTA holding B interleaved complex sequences of
// power-of-two length Ls in shared memory (element n of sequence b at
// buf[n*B + b], so a warp's consecutive lanes touch consecutive words).
//
// Each radix-R pass is Stockham autosort (no bit reversal pass):
//   for item (b, j), j < Ls/R, k = j mod Ns:
//     v[r] = x[j + r Ls/R] * W_{Ns R}^{r k},  V = DFT_R(v),  x'[(j-k)R + k + r Ns] = V[r]
// done in place: every participating thread loads its E = 16 elements into
// registers, the CTA barriers, then stores.  Passes are radix 16 while >= 4
// index bits remain, then one radix 2/4/8 pass.  The R-point DFTs are
// unrolled radix-2 DIF networks with compile-time twiddles.
//
// Twiddles: W_Ls^m = hi[m >> 6] * lo[m & 63] from a two-level table held in
// shared memory (computed with double-precision sincospi at kernel start), and
// the powers W^{2k..15k} of each item's base twiddle by complex products of
// depth <= 4 — no per-element transcendental, no table larger than 1.5 KB.
#pragma once
#include "cs_common.cuh"

namespace cs {

constexpr int FFT_E = 16;  // complex elements per thread per pass

template <typename T> struct TwTable {
  const C2<T>* lo;  // W^i, i < 64
  const C2<T>* hi;  // W^{64 i}, i < max(1, len/64) (+1 for the 4N table)
  CS_DEV C2<T> operator()(int64_t m) const { return cmul<T>(hi[m >> 6], lo[m & 63]); }
};

// Fill lo[64], hi[nhi] with W_den^i = exp(-2 pi i * i / den) (den = period).
template <typename T>
CS_DEV void tw_init(C2<T>* lo, C2<T>* hi, int64_t den, int nhi, int tid, int nthr) {
  for (int i = tid; i < 64 + nhi; i += nthr) {
    int64_t m = (i < 64) ? i : (int64_t)(i - 64) * 64;
    double s, c;
    // exp(-2 pi i m/den): reduce m mod den exactly in integers first
    int64_t mm = m % den;
    sincospi(-2.0 * (double)mm / (double)den, &s, &c);
    C2<T> w = mk<T>((T)c, (T)s);
    if (i < 64) lo[i] = w; else hi[i - 64] = w;
  }
}

// ---- compile-time twiddles of the radix-16 network: W_16^t, t in [0, 8) ----
template <typename T, int t, bool INV> CS_DEV C2<T> w16c() {
  constexpr double c[8] = {1.0, 0.92387953251128675613, 0.70710678118654752440,
                           0.38268343236508977173, 0.0, -0.38268343236508977173,
                           -0.70710678118654752440, -0.92387953251128675613};
  constexpr double s[8] = {0.0, 0.38268343236508977173, 0.70710678118654752440,
                           0.92387953251128675613, 1.0, 0.92387953251128675613,
                           0.70710678118654752440, 0.38268343236508977173};
  return mk<T>((T)c[t], INV ? (T)s[t] : (T)(-s[t]));
}

template <typename T, int t16, bool INV> CS_DEV C2<T> tw_apply(C2<T> a) {
  if constexpr (t16 == 0) {
    return a;
  } else if constexpr (t16 == 4) {
    return mul_mi<T, INV>(a);
  } else if constexpr (t16 == 2 || t16 == 6) {
    // (±1 ∓ i)/sqrt2 patterns: 2 mul + 2 add
    constexpr T h = (T)0.70710678118654752440;
    C2<T> w = w16c<T, t16, INV>();
    T sx = w.x > 0 ? (T)1 : (T)-1, sy = w.y > 0 ? (T)1 : (T)-1;
    // a * (sx h + i sy h) = h*(sx a.x - sy a.y) + i h*(sx a.y + sy a.x)
    return mk<T>(h * (sx * a.x - sy * a.y), h * (sx * a.y + sy * a.x));
  } else {
    return cmul<T>(a, w16c<T, t16, INV>());
  }
}

// radix-2 DIF stage with half-span H over a block starting at S (compile time)
template <typename T, int R, int H, int S, int t, bool INV>
CS_DEV void dif_bfly(C2<T>* v) {
  if constexpr (t < H) {
    C2<T> a = v[S + t], b = v[S + t + H];
    v[S + t] = cadd<T>(a, b);
    v[S + t + H] = tw_apply<T, t * (16 / (2 * H)), INV>(csub<T>(a, b));
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
// in-register R-point DFT; output X_r lands at v[bitrev<R>(r)]
template <typename T, int R, bool INV> CS_DEV void dft_reg(C2<T>* v) { dif_stages<T, R, R / 2, INV>(v); }

// powers w[r] = w1^r, r < R, depth <= log2 R products
template <typename T, int R> CS_DEV void tw_powers(C2<T> w1, C2<T>* w) {
  w[0] = mk<T>(1, 0);
  w[1] = w1;
#pragma unroll
  for (int r = 2; r < R; ++r) w[r] = cmul<T>(w[r >> 1], w[r - (r >> 1)]);
}

// One radix-R pass over B interleaved sequences of length Ls. IPT = FFT_E / R items per thread.
template <typename T, int R, bool INV>
CS_NOINL void fft_pass(C2<T>* buf, int Ls, int B, int Ns, int s_tw, const TwTable<T>& tw,
                     int tid, int nact) {
  constexpr int IPT = FFT_E / R;
  const int Lr = Ls / R;
  const int items = B * Lr;
  C2<T> v[IPT][R];
  bool act[IPT];
#pragma unroll
  for (int it = 0; it < IPT; ++it) {
    int i = tid + it * nact;
    act[it] = (tid < nact) && (i < items);
    if (act[it]) {
      int b = i % B, j = i / B;
#pragma unroll
      for (int r = 0; r < R; ++r) v[it][r] = buf[(int64_t)(j + r * Lr) * B + b];
      if (Ns > 1) {
        int k = j & (Ns - 1);
        C2<T> w1 = tw((int64_t)k * s_tw);
        if (INV) w1 = cconj<T>(w1);
        C2<T> w[R];
        tw_powers<T, R>(w1, w);
#pragma unroll
        for (int r = 1; r < R; ++r) v[it][r] = cmul<T>(v[it][r], w[r]);
      }
      dft_reg<T, R, INV>(v[it]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < IPT; ++it) {
    if (act[it]) {
      int i = tid + it * nact;
      int b = i % B, j = i / B;
      int k = j & (Ns - 1);
      int base = (j - k) * R + k;
#pragma unroll
      for (int r = 0; r < R; ++r) buf[(int64_t)(base + r * Ns) * B + b] = v[it][bitrev<R>(r)];
    }
  }
  __syncthreads();
}

// Full transform: forward (INV=false: X_k = sum x_n W^{nk}) or unnormalised inverse.
// Requires B * Ls <= FFT_E * blockDim.x; all threads of the CTA must call it.
template <typename T, bool INV>
CS_NOINL void fft_cta(C2<T>* buf, int Ls, int B, const TwTable<T>& tw) {
  const int tid = threadIdx.x;
  const int nact = max(1, (B * Ls) / FFT_E);
  int Ns = 1;
  int rem = Ls;
  while (rem >= 16) {
    fft_pass<T, 16, INV>(buf, Ls, B, Ns, Ls / (Ns * 16), tw, tid, nact);
    Ns *= 16;
    rem /= 16;
  }
  if (rem == 8) fft_pass<T, 8, INV>(buf, Ls, B, Ns, Ls / (Ns * 8), tw, tid, nact);
  else if (rem == 4) fft_pass<T, 4, INV>(buf, Ls, B, Ns, Ls / (Ns * 4), tw, tid, nact);
  else if (rem == 2) fft_pass<T, 2, INV>(buf, Ls, B, Ns, Ls / (Ns * 2), tw, tid, nact);
}

}  // namespace cs
