// dct_mid.cuh — the DCT "sandwich middle": real-split of the half-length FFT into
// DCT-II coefficients, the row-select / residual operation in the DCT domain,
// and the inverse split that feeds the inverse FFT (DCT-III).
//
// Orthonormal DCT-II via Makhoul's reorder and an N/2-point complex FFT
// ("DCT can be speeded by FFT"):
//   z_m = v_{2m} + i v_{2m+1},  Z = FFT_L(z),  L = N/2
//   for the pair (k, kk = L-k):  P = (Z_k + conj Z_kk)/2,  O = -i (Z_k - conj Z_kk)/2,
//   a = W_4N^k = e^{-i pi k / 2N},  w = W_N^k = a^4,  Q = w O,
//   c_k  = a (P + Q)                -> X_k = Re c_k,   X_{N-k}  = -Im c_k
//   c_kk = e^{-i pi/4} conj(a (P - Q)) -> X_kk = Re c_kk, X_{N-kk} = -Im c_kk
//   k = 0: X_0 = Re Z_0 + Im Z_0,  X_L = (Re Z_0 - Im Z_0)/sqrt 2
// X is the unnormalised DCT-II; the orthonormal one is s_k X_k with
// s_0 = 1/sqrt N, s_k = sqrt(2/N).  The inverse split runs the same algebra
// backwards.  In between, the operation of the step being computed:
//   MID_H   : X'_k = [k in rows] X_k / L                (H = W A^T A W, Eq.(11))
//   MID_RES : X'_k = [k in rows] (y_rank(k)/s_k - X_k) / L, ||r||^2 += (y - s X)^2
//             (pursuit residual + correlation A^T(y - A x), Alg.1 lines 03/07)
//   MID_FWD : y_rank(k) = s_k X_k  (forward apply only, no inverse)
// The 1/L of the unnormalised inverse FFT is folded into X'.
#pragma once
#include "cs_common.cuh"
#include "fft_cta.cuh"
#include "layout_s.cuh"

namespace cs {

enum MidMode { MID_H = 0, MID_RES = 1, MID_FWD = 2,
               // Psi = DCT, CTA tier (R35): the full DCT-II written back into the transform buffer
               // (for the next transform) / C_N^T read from it — no rows, no y
               MID_FWDZ = 3, MID_INVZ = 4 };

template <typename T> struct MidCtx {
  const uint32_t* rowmask;  // [N/32] row-selection bitmask (P)
  const int32_t* prefix;    // [N/32] rows in words before
  const T* y;               // [M] measurements (RES)
  T* yout;                  // [M] forward output (FWD)
  int64_t N;
  T s0, sk, inv_s0, inv_sk, invL;
  // bit position of DCT index k in rowmask/prefix: t = (k mod 2^s1) << tsh | k >> s1
  // (s1 = 0: natural order, Tier S; s1 = log2 L1, tsh = log2(2 L2): Tier L transposed)
  int s1, tsh;
  // Tier L pass B: the mask / prefix words of the (at most two) transposed rows an
  // item touches are staged in shared memory: row `ra` -> slot 0, any other -> slot 1,
  // rowmask = staged mask [2][W], prefix = staged prefix [2][W] (W = 2^tsh / 32).
  int staged, ra;
  CS_DEV int64_t tpos(int64_t k) const {
    return ((k & ((int64_t(1) << s1) - 1)) << tsh) | (k >> s1);
  }
  CS_DEV int64_t word(int64_t t) const {
    if (!staged) return t >> 5;
    const int64_t a = t >> tsh, W = (int64_t(1) << tsh) >> 5;
    return (a == ra ? 0 : W) + ((t >> 5) & (W - 1));
  }
  CS_DEV bool sel(int64_t t) const { return (rowmask[word(t)] >> (t & 31)) & 1u; }
  CS_DEV int64_t rank(int64_t t) const {
    const int64_t w = word(t);
    const uint32_t below = (t & 31) ? (rowmask[w] & ((1u << (t & 31)) - 1u)) : 0u;
    return (int64_t)prefix[w] + __popc(below);
  }
};

template <typename T, int MODE>
CS_DEV T mid_op(const MidCtx<T>& m, int64_t kn, T X, double& rn2) {
  const int64_t k = m.tpos(kn);
  const bool sel = m.sel(k);
  const T s = (kn == 0) ? m.s0 : m.sk;
  if constexpr (MODE == MID_H) {
    return sel ? X * m.invL : T(0);
  } else if constexpr (MODE == MID_RES) {
    if (!sel) return T(0);
    const T d = m.y[m.rank(k)] - s * X;
    rn2 += (double)d * (double)d;
    const T is = (kn == 0) ? m.inv_s0 : m.inv_sk;
    return d * is * m.invL;
  } else {
    if (sel) m.yout[m.rank(k)] = s * X;
    return T(0);
  }
}

// k = 0 element (self-contained: X_0 and X_L)
template <typename T, int MODE>
CS_DEV void mid_zero(C2<T>& Z0, const MidCtx<T>& m, double& rn2) {
  constexpr T r2 = (T)0.70710678118654752440;
  const int64_t L = m.N >> 1;
  T X0 = Z0.x + Z0.y;
  T XL = (Z0.x - Z0.y) * r2;
  T Y0 = mid_op<T, MODE>(m, 0, X0, rn2);
  T YL = mid_op<T, MODE>(m, L, XL, rn2);
  if constexpr (MODE != MID_FWD) {
    T V0 = Y0, VL = YL * (T)1.41421356237309504880;
    Z0 = mk<T>((V0 + VL) * (T)0.5, (V0 - VL) * (T)0.5);
  }
}

// pair (k, kk = L - k), 1 <= k <= L/2; `a` = W_4N^k.  Zk, Zkk updated in place.
template <typename T, int MODE>
CS_DEV void mid_pair(C2<T>& Zk, C2<T>& Zkk, int64_t k, C2<T> a, const MidCtx<T>& m, double& rn2) {
  constexpr T r2 = (T)0.70710678118654752440;
  const int64_t N = m.N, L = N >> 1, kk = L - k;
  const C2<T> e4 = mk<T>(r2, -r2);  // e^{-i pi/4}
  C2<T> a2 = cmul<T>(a, a);
  C2<T> w = cmul<T>(a2, a2);
  C2<T> P = cscale<T>(cadd<T>(Zk, cconj<T>(Zkk)), (T)0.5);
  C2<T> D = csub<T>(Zk, cconj<T>(Zkk));
  C2<T> O = mk<T>(D.y * (T)0.5, -D.x * (T)0.5);  // -i D / 2
  C2<T> Q = cmul<T>(w, O);
  C2<T> ck = cmul<T>(a, cadd<T>(P, Q));
  C2<T> ckk = cmul<T>(e4, cconj<T>(cmul<T>(a, csub<T>(P, Q))));
  const bool self = (k == kk);
  T Xk = mid_op<T, MODE>(m, k, ck.x, rn2);
  T Xnk = mid_op<T, MODE>(m, N - k, -ck.y, rn2);
  T Xkk = Xk, Xnkk = Xnk;
  if (!self) {
    Xkk = mid_op<T, MODE>(m, kk, ckk.x, rn2);
    Xnkk = mid_op<T, MODE>(m, N - kk, -ckk.y, rn2);
  }
  if constexpr (MODE != MID_FWD) {
    C2<T> cpk = mk<T>(Xk, -Xnk);
    C2<T> cpkk = mk<T>(Xkk, -Xnkk);
    C2<T> Vk = cmulc<T>(cpk, a);                              // conj(a) c'_k
    C2<T> Vkk = cmul<T>(cconj<T>(e4), cmul<T>(a, cpkk));        // e^{i pi/4} a c'_kk
    C2<T> cVkk = cconj<T>(Vkk);
    C2<T> E = cscale<T>(cadd<T>(Vk, cVkk), (T)0.5);
    C2<T> Od = cscale<T>(cmulc<T>(csub<T>(Vk, cVkk), w), (T)0.5);  // conj(w)(Vk - conj Vkk)/2
    C2<T> iO = mk<T>(-Od.y, Od.x);
    Zk = cadd<T>(E, iO);
    if (!self) Zkk = cconj<T>(csub<T>(E, iO));
  }
}

// ---- full orthonormal DCT-II outputs / C_N^T inputs of a pair (Psi = DCT, R35) ----
// o = s X at (k, N-k, kk, N-kk), kk = L - k (the self pair k = L/2 repeats o[0], o[1])
template <typename T>
CS_DEV void dct_out_pair(const C2<T>& Zk, const C2<T>& Zkk, C2<T> a, const MidCtx<T>& m, T* o) {
  constexpr T r2 = (T)0.70710678118654752440;
  const C2<T> e4 = mk<T>(r2, -r2);
  const C2<T> a2 = cmul<T>(a, a);
  const C2<T> w = cmul<T>(a2, a2);
  const C2<T> P = cscale<T>(cadd<T>(Zk, cconj<T>(Zkk)), (T)0.5);
  const C2<T> D = csub<T>(Zk, cconj<T>(Zkk));
  const C2<T> O = mk<T>(D.y * (T)0.5, -D.x * (T)0.5);
  const C2<T> Q = cmul<T>(w, O);
  const C2<T> ck = cmul<T>(a, cadd<T>(P, Q));
  const C2<T> ckk = cmul<T>(e4, cconj<T>(cmul<T>(a, csub<T>(P, Q))));
  o[0] = m.sk * ck.x;
  o[1] = -m.sk * ck.y;
  o[2] = m.sk * ckk.x;
  o[3] = -m.sk * ckk.y;
}
// k = 0: o = (s_0 X_0, s X_L)
template <typename T> CS_DEV void dct_out_zero(const C2<T>& Z0, const MidCtx<T>& m, T* o) {
  constexpr T r2 = (T)0.70710678118654752440;
  o[0] = m.s0 * (Z0.x + Z0.y);
  o[1] = m.sk * (Z0.x - Z0.y) * r2;
}
// inverse split of C_N^T applied to v with v = wv at (k, N-k, kk, N-kk): the spectrum slots
// Zk, Zkk of the unnormalised inverse FFT (mid_pair's inverse half, X' = v / (s L))
template <typename T>
CS_DEV void dct_in_pair(C2<T>& Zk, C2<T>& Zkk, int64_t k, C2<T> a, const MidCtx<T>& m, const T* wv) {
  constexpr T r2 = (T)0.70710678118654752440;
  const C2<T> e4 = mk<T>(r2, -r2);
  const int64_t kk = (m.N >> 1) - k;
  const bool self = (k == kk);
  const T f = m.inv_sk * m.invL;
  const C2<T> a2 = cmul<T>(a, a);
  const C2<T> w = cmul<T>(a2, a2);
  const C2<T> cpk = mk<T>(wv[0] * f, -wv[1] * f);
  const C2<T> cpkk = self ? cpk : mk<T>(wv[2] * f, -wv[3] * f);
  const C2<T> Vk = cmulc<T>(cpk, a);
  const C2<T> Vkk = cmul<T>(cconj<T>(e4), cmul<T>(a, cpkk));
  const C2<T> cVkk = cconj<T>(Vkk);
  const C2<T> E = cscale<T>(cadd<T>(Vk, cVkk), (T)0.5);
  const C2<T> Od = cscale<T>(cmulc<T>(csub<T>(Vk, cVkk), w), (T)0.5);
  const C2<T> iO = mk<T>(-Od.y, Od.x);
  Zk = cadd<T>(E, iO);
  if (!self) Zkk = cconj<T>(csub<T>(E, iO));
}
template <typename T> CS_DEV void dct_in_zero(C2<T>& Z0, const MidCtx<T>& m, const T* wv) {
  const T V0 = wv[0] * m.inv_s0 * m.invL, VL = wv[1] * m.inv_sk * m.invL * (T)1.41421356237309504880;
  Z0 = mk<T>((V0 + VL) * (T)0.5, (V0 - VL) * (T)0.5);
}

// ---- F = partial Fourier (R36): the real DFT from the same half-length FFT ----
// z_m = u_{2m} + i u_{2m+1} (plain packing: the operator's position map, built as an
// effective permutation at create time), Z = FFT_L(z).  For the pair (n, L - n):
//   E = (Z_n + conj Z_{L-n})/2,  O = -i (Z_n - conj Z_{L-n})/2,  w = W_N^n,
//   X_n = E + w O,  X_{L-n} = conj(E - w O)          (unnormalised DFT of u)
// A selected frequency f (row rank r) is measured as y[2r] = s Re X_f, y[2r+1] = s Im X_f,
// s = sqrt(2/N).  The adjoint, with the unnormalised inverse FFT (z'_m = sum Z'_k
// e^{+2 pi i k m / L} = u'_{2m} + i u'_{2m+1}), takes V~_f = (s/2) V_f (V = s X for H,
// y - s X for RES) and
//   E' = V~_n + conj V~_{L-n},  O' = V~_n - conj V~_{L-n},
//   Z'_n = E' + i conj(w) O',  Z'_{L-n} = conj(E' - i conj(w) O').
// DC and Nyquist (n = 0) are never measured.
template <typename T, int MODE>
CS_DEV C2<T> dft_op(const MidCtx<T>& m, int64_t f, C2<T> X, double& rn2) {
  const int64_t t = m.tpos(f);
  const bool sel = m.sel(t);
  const T s = m.sk;  // sqrt(2/N)
  if constexpr (MODE == MID_H) {
    const T h = (T)0.5 * s * s;  // (s/2) s = 1/N
    return sel ? mk<T>(X.x * h, X.y * h) : mk<T>(0, 0);
  } else if constexpr (MODE == MID_RES) {
    if (!sel) return mk<T>(0, 0);
    const int64_t r = m.rank(t);
    const T dx = m.y[2 * r] - s * X.x, dy = m.y[2 * r + 1] - s * X.y;
    rn2 += (double)dx * (double)dx + (double)dy * (double)dy;
    const T h = (T)0.5 * s;
    return mk<T>(dx * h, dy * h);
  } else {
    if (sel) {
      const int64_t r = m.rank(t);
      m.yout[2 * r] = s * X.x;
      m.yout[2 * r + 1] = s * X.y;
    }
    return mk<T>(0, 0);
  }
}
// n = 0 element: DC and Nyquist, never measured
template <typename T, int MODE>
CS_DEV void dft_zero(C2<T>& Z0, const MidCtx<T>& m, double& rn2) {
  (void)m;
  (void)rn2;
  if constexpr (MODE != MID_FWD) Z0 = mk<T>(0, 0);
}
// pair (n, L - n), 1 <= n <= L/2 (n = L/2: the self pair, Zk and Zkk the same element);
// w = W_N^n.  Zk, Zkk updated in place.
template <typename T, int MODE>
CS_DEV void dft_pair_w(C2<T>& Zk, C2<T>& Zkk, int64_t n, C2<T> w, const MidCtx<T>& m, double& rn2) {
  const int64_t L = m.N >> 1, nn = L - n;
  const bool self = (n == nn);
  const C2<T> P2 = mk<T>(Zk.x + Zkk.x, Zk.y - Zkk.y);   // 2E
  const C2<T> O2 = mk<T>(Zk.y + Zkk.y, Zkk.x - Zk.x);   // 2O = -i (Zk - conj Zkk)
  const C2<T> Q2 = cmul<T>(w, O2);
  const C2<T> Xa = mk<T>((P2.x + Q2.x) * (T)0.5, (P2.y + Q2.y) * (T)0.5);     // X_n
  const C2<T> Xb = mk<T>((P2.x - Q2.x) * (T)0.5, -(P2.y - Q2.y) * (T)0.5);    // X_{L-n}
  const C2<T> Va = dft_op<T, MODE>(m, n, Xa, rn2);
  const C2<T> Vb = self ? Va : dft_op<T, MODE>(m, nn, Xb, rn2);
  if constexpr (MODE != MID_FWD) {
    const C2<T> E = mk<T>(Va.x + Vb.x, Va.y - Vb.y);     // V~_n + conj V~_{L-n}
    const C2<T> O = mk<T>(Va.x - Vb.x, Va.y + Vb.y);     // V~_n - conj V~_{L-n}
    const C2<T> c = cmulc<T>(O, w);                      // conj(w) O
    const C2<T> t = mk<T>(-c.y, c.x);                    // i conj(w) O
    Zk = mk<T>(E.x + t.x, E.y + t.y);
    if (!self) Zkk = mk<T>(E.x - t.x, -(E.y - t.y));
  }
}
// the same with a = W_4N^n (the DCT tables' twiddle; w = a^4)
template <typename T, int MODE>
CS_DEV void dft_pair(C2<T>& Zk, C2<T>& Zkk, int64_t n, C2<T> a, const MidCtx<T>& m, double& rn2) {
  const C2<T> a2 = cmul<T>(a, a);
  dft_pair_w<T, MODE>(Zk, Zkk, n, cmul<T>(a2, a2), m, rn2);
}

// ---- the same pair operation with the constant factors folded (Tier S) ----
// Forward split without the two 1/2 factors: raw_k = 2 X_k, raw_{N-k} = 2 X_{N-k},
// and for the kk pair the e^{-i pi/4} rotation split into (1 - i) and a factor
// r2 = 1/sqrt 2: raw_kk = 2 X_kk / r2, raw_{N-kk} = 2 X_{N-kk} / r2.  mid_op2 works
// on raw values with per-type constants (MidK<T>) and returns the value the
// inverse split needs with its own 1/2 (and, for the kk pair, r2) folded in.
// Requires k != L - k (the self pair n = L/2 goes through mid_pair).
template <typename T> struct MidK {
  T scx[2];  // s_k * (1/2, r2/2): X = scx * raw
  T cout[2]; // (1/2, r2/2) / s_k / L * 2: returned = cout * (y - s X)          (RES)
  T hH[2];   // invL * (1/4, 1/8): returned = [sel] raw * hH                     (H)
};
// compile-time constants for N = 2^LOG2N
template <typename T, int LOG2N> CS_DEV MidK<T> make_midk_c() {
  constexpr double r2 = 0.70710678118654752440, sk = sqrt_pow2(1 - LOG2N), invL = 2.0 / (double)(1ll << LOG2N);
  MidK<T> c;
  c.scx[0] = (T)(sk * 0.5);
  c.scx[1] = (T)(sk * r2 * 0.5);
  c.cout[0] = (T)(invL / sk * 0.5);
  c.cout[1] = (T)(invL / sk * r2 * 0.5);
  c.hH[0] = (T)(invL * 0.25);
  c.hH[1] = (T)(invL * 0.125);
  return c;
}
template <typename T> CS_DEV MidK<T> make_midk(int N) {
  MidK<T> c;
  const double r2 = 0.70710678118654752440, sk = sqrt(2.0 / (double)N), invL = 2.0 / (double)N;
  c.scx[0] = (T)(sk * 0.5);
  c.scx[1] = (T)(sk * r2 * 0.5);
  c.cout[0] = (T)(invL / sk * 0.5);
  c.cout[1] = (T)(invL / sk * r2 * 0.5);
  c.hH[0] = (T)(invL * 0.25);
  c.hH[1] = (T)(invL * 0.125);
  return c;
}
CS_DEV bool bit_test32(const uint32_t* bits, int j) { return (bits[j >> 5] >> (j & 31)) & 1u; }
CS_DEV int row_rank32(const uint32_t* mask, const int32_t* prefix, int k) {
  return prefix[k >> 5] + __popc(mask[k >> 5] & ((1u << (k & 31)) - 1u));
}
template <typename T, int MODE, int TY>
CS_DEV T mid_op2(const MidCtx<T>& m, const MidK<T>& c, int idx, T raw, double& rn2) {
  const bool sel = bit_test32(m.rowmask, idx);
  if constexpr (MODE == MID_H) {
    return sel ? raw * c.hH[TY] : T(0);
  } else if constexpr (MODE == MID_RES) {
    if (!sel) return T(0);
    const T d = m.y[row_rank32(m.rowmask, m.prefix, idx)] - c.scx[TY] * raw;
    rn2 += (double)d * (double)d;
    return d * c.cout[TY];
  } else {
    if (sel) m.yout[row_rank32(m.rowmask, m.prefix, idx)] = c.scx[TY] * raw;
    return T(0);
  }
}
// The pair operation on raw values with a caller-supplied row lookup: sel(q) / rank(q) for
// the four DCT indices q = 0: k, 1: N-k, 2: kk = L-k, 3: N-kk (rank only called when sel).
// a = W_4N^k, w = W_N^k = a^4 (precomputed by the caller).
template <typename T, int MODE, int TY, class RK>
CS_DEV T mid_op2g(const MidCtx<T>& m, const MidK<T>& c, bool sel, RK&& rank, T raw, double& rn2) {
  if constexpr (MODE == MID_H) {
    return sel ? raw * c.hH[TY] : T(0);
  } else if constexpr (MODE == MID_RES) {
    if (!sel) return T(0);
    const T d = m.y[rank()] - c.scx[TY] * raw;
    rn2 += (double)d * (double)d;
    return d * c.cout[TY];
  } else {
    // the rank reads only metadata words (shared memory on both tiers): computed for every
    // index so the store is predicated instead of a divergent branch per index
    const int r = (int)rank();
    T* const dst = m.yout + r;   // yout is global memory on both tiers
    const T v = c.scx[TY] * raw;
    if constexpr (sizeof(T) == 4)
      asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 0; @p st.global.f32 [%0], %1; }" ::"l"(dst), "f"(v),
                   "r"((unsigned)sel) : "memory");
    else
      asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 0; @p st.global.f64 [%0], %1; }" ::"l"(dst), "d"(v),
                   "r"((unsigned)sel) : "memory");
    return T(0);
  }
}
template <typename T, int MODE, class SEL, class RANK>
CS_DEV void mid_pair2g(C2<T>& Zk, C2<T>& Zkk, C2<T> a, C2<T> w, const MidCtx<T>& m, const MidK<T>& c,
                       double& rn2, SEL&& sel, RANK&& rank) {
  const C2<T> P2 = mk<T>(Zk.x + Zkk.x, Zk.y - Zkk.y);   // Zk + conj Zkk
  const C2<T> O2 = mk<T>(Zk.y + Zkk.y, Zkk.x - Zk.x);   // -i (Zk - conj Zkk)
  const C2<T> Q2 = cmul<T>(w, O2);
  const C2<T> ck = cmul<T>(a, cadd<T>(P2, Q2));        // 2 (X_k - i X_{N-k})
  const C2<T> u = cmul<T>(a, csub<T>(P2, Q2));         // e4 conj(u) = 2 (X_kk - i X_{N-kk}) / r2
  const T gk = mid_op2g<T, MODE, 0>(m, c, sel(0), [&] { return rank(0); }, ck.x, rn2);
  const T gnk = mid_op2g<T, MODE, 0>(m, c, sel(1), [&] { return rank(1); }, -ck.y, rn2);
  const T gkk = mid_op2g<T, MODE, 1>(m, c, sel(2), [&] { return rank(2); }, u.x - u.y, rn2);
  const T gnkk = mid_op2g<T, MODE, 1>(m, c, sel(3), [&] { return rank(3); }, u.x + u.y, rn2);
  if constexpr (MODE != MID_FWD) {
    const C2<T> Vk = cmulc<T>(mk<T>(gk, -gnk), a);                // conj(a) c'_k
    const C2<T> t = cmul<T>(a, mk<T>(gkk, -gnkk));
    const C2<T> cVkk = mk<T>(t.x - t.y, -(t.x + t.y));            // conj((1 + i) t)
    const C2<T> E = cadd<T>(Vk, cVkk);
    const C2<T> Od = cmulc<T>(csub<T>(Vk, cVkk), w);              // conj(w)(Vk - conj Vkk)
    Zk = mk<T>(E.x - Od.y, E.y + Od.x);                           // E + i Od
    Zkk = mk<T>(E.x + Od.y, Od.x - E.y);                          // conj(E - i Od)
  }
}
// natural-order row bitmask (Tier S)
template <typename T, int MODE>
CS_DEV void mid_pair2(C2<T>& Zk, C2<T>& Zkk, int k, C2<T> a, C2<T> w, const MidCtx<T>& m, const MidK<T>& c,
                      double& rn2) {
  const int N = (int)m.N, kk = (N >> 1) - k;
  const int idx[4] = {k, N - k, kk, N - kk};
  mid_pair2g<T, MODE>(Zk, Zkk, a, w, m, c, rn2, [&](int q) { return bit_test32(m.rowmask, idx[q]); },
                      [&](int q) { return row_rank32(m.rowmask, m.prefix, idx[q]); });
}

template <typename T, int LOG2N> CS_DEV MidCtx<T> make_mid_c(const uint32_t* rowmask, const int32_t* prefix,
                                                           const T* y, T* yout) {
  MidCtx<T> m;
  m.rowmask = rowmask;
  m.prefix = prefix;
  m.y = y;
  m.yout = yout;
  m.N = 1ll << LOG2N;
  m.s0 = (T)sqrt_pow2(-LOG2N);
  m.sk = (T)sqrt_pow2(1 - LOG2N);
  m.inv_s0 = (T)sqrt_pow2(LOG2N);
  m.inv_sk = (T)sqrt_pow2(LOG2N - 1);
  m.invL = (T)(2.0 / (double)(1ll << LOG2N));
  m.s1 = 0;
  m.tsh = 0;
  m.staged = 0;
  m.ra = 0;
  return m;
}

template <typename T> CS_DEV MidCtx<T> make_mid(int64_t N, const uint32_t* rowmask,
                                               const int32_t* prefix, const T* y, T* yout) {
  MidCtx<T> m;
  m.rowmask = rowmask;
  m.prefix = prefix;
  m.y = y;
  m.yout = yout;
  m.N = N;
  m.s0 = (T)rsqrt((double)N);
  m.sk = (T)sqrt(2.0 / (double)N);
  m.inv_s0 = (T)sqrt((double)N);
  m.inv_sk = (T)sqrt((double)N / 2.0);
  m.invL = (T)(2.0 / (double)N);
  m.s1 = 0;
  m.tsh = 0;
  m.staged = 0;
  m.ra = 0;
  return m;
}

}  // namespace cs
