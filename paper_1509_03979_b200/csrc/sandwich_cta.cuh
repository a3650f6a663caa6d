// sandwich_cta.cuh — the fused operator sandwich of Tier S: A^T (mid) A on one CTA.
//
// Every CG iteration applies H d = (A^T A scatter_S d)[S] ("the operation
// Hd_j dominates the whole computation cost"), and every detection applies
// A^T (y - A x) (Algorithm 1 lines 03/07).  Both are
//     forward L-point FFT (L = N/2) -> DCT split, row select / residual, inverse
//     split -> inverse L-point FFT
// held in one CTA's shared memory.  Design:
//
//  * 512 threads, two CTAs per SM, <= 64 registers: every pass keeps <= 16 points
//    per thread;
//  * small code (the CG loop must fit the 32 KB instruction cache): the radix-16
//    passes are ONE loop body with a runtime stride Ns, run (log2 L - 1) / 4 times
//    forward and inverse; a remainder pass of radix 2/4/8 covers the other bits;
//  * the forward FFT ends with a radix-2 pass (Ns = L/2), after which item k holds
//    Z_k and Z_{k+L/2}; the DCT real split pairs Z_n with Z_{L-n}, and the mirror
//    of {k, k+L/2} is item L/2-k — one thread owns the unit (k, L/2-k), i.e. four
//    points, and runs last forward pass, split, middle, inverse split and the
//    first inverse pass (radix 2, Ns = 1, same point set) in registers;
//  * DCT twiddles a_n = W_4N^n: one table lookup per unit (a_{k+L/2} = a_k W_16);
//    w_n = a_n^4.
//
// Stockham pass (radix R, stride Ns before the pass), item j < L/R, k = j mod Ns:
//    v_r = x[j + r L/R] * W_{Ns R}^{r k},  V = DFT_R(v),  x'[(j-k) R + k + r Ns] = V_r.
// Shared addresses use the XOR swizzle of fft_cta.cuh; swz is linear over GF(2),
// so swz(base | r Ns) = swz(base) ^ (XOR of swz(Ns << b) over the bits b of r).
#pragma once
#include "cs_common.cuh"
#include "dct_mid.cuh"
#include "fft_cta.cuh"
#include "layout_s.cuh"

namespace cs {

constexpr int SW_NT = 512;  // threads per Tier S block (two blocks per SM)
constexpr int SW_LOG2NT = 9;

// threadIdx.x plus a 0 read through a volatile shared load: address arithmetic derived
// from it cannot be hoisted out of the CG loop (where, under the 64-register budget,
// ptxas would otherwise precompute and spill it), so it is recomputed each pass.
template <typename T, int LOG2L> CS_DEV int opaque_tid() {
  constexpr SFix F = s_fixed<T>(int64_t(2) << LOG2L);
  const int t = (int)threadIdx.x + *reinterpret_cast<volatile int*>(cs_smem_base + F.zero);
  __builtin_assume(t >= 0);
  __builtin_assume(t < SW_NT);
  return t;
}

template <int LOG2L> struct SwPlan {
  // forward radices: [remainder 2^M if M > 0] [2^RBM] x Q [2 (fused)]; inverse reversed.
  // The main radix is the largest of 16, 8, 4 whose passes still give every one of the 512
  // threads an item (L / 2^RBM >= 512): radix 16 at N = 2^14 (c4), radix 4 at N = 2^12
  // (c1) — a radix-16 pass there would leave three quarters of the block idle on a
  // latency-bound critical path.
  static constexpr int L_ = 1 << LOG2L;
  static constexpr int RBM = ((L_ >> 4) >= SW_NT) ? 4 : (((L_ >> 3) >= SW_NT) ? 3 : 2);
  static constexpr int M = (LOG2L - 1) % RBM;
  static constexpr int Q = (LOG2L - 1) / RBM;
  static constexpr int NS_R16_FWD0 = M;                                  // log2 Ns, first main pass
  // log2 Ns of the first radix-16 pass that has twiddles (Ns1 <= 16: its 16 Ns1 twiddles
  // W_{16 Ns1}^{r k} come from the tw16 table, one LDS each, instead of a product chain)
  static constexpr int NS1B = (M == 0) ? 4 : M;
  static constexpr int U = (1 << LOG2L) / 4 > 0 ? (1 << LOG2L) / 4 : 1;  // fused units
  static constexpr int UPT = (U + SW_NT - 1) / SW_NT;                     // units per thread
  static_assert(UPT <= 4, "L <= 8192");
};

// ---- one Stockham pass of radix 2^RB at runtime stride Ns = 2^nsb; L = 2^LOG2L ----
// Items j < L/R; thread t owns j = t + 512 it (it < IPT: several items when L/R > 512).
template <typename T, int LOG2L, int RB, bool INV>
CS_DEV void sw_pass(C2<T>* buf, const TwTable<T>& tw, int nsb) {
  constexpr int R = 1 << RB, Lr = (1 << LOG2L) >> RB;
  constexpr int IPT = Lr > SW_NT ? Lr / SW_NT : 1;
  const int t0 = opaque_tid<T, LOG2L>();
  C2<T> v[IPT][R];
  const int Ns = 1 << nsb;
#pragma unroll
  for (int it = 0; it < IPT; ++it) {
    const int j = t0 + it * SW_NT;
    const int k = j & (Ns - 1);
    if ((Lr >= SW_NT) || j < Lr) {
      const int sj = swz<T>(j);  // j < Lr: bit-disjoint from r Lr
      if constexpr (Lr % 512 == 0) {
        // swz(r Lr) = r Lr and sj < Lr: plain offsets (immediate-addressed LDS, no registers)
#pragma unroll
        for (int r = 0; r < R; ++r) v[it][r] = buf[sj + r * Lr];
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) v[it][r] = buf[sj ^ swz_c<T>(r * Lr)];
      }
      if (Ns > 1) {
        if (RB == 4 && SwPlan<LOG2L>::RBM == 4 && nsb == SwPlan<LOG2L>::NS1B) {
          constexpr SFix F = s_fixed<T>(int64_t(2) << LOG2L);
          const C2<T>* t16 = reinterpret_cast<const C2<T>*>(cs_smem_base + F.tw16) + k;  // [r][k]: conflict-free
#pragma unroll
          for (int r = 1; r < R; ++r) v[it][r] = INV ? cmulc<T>(v[it][r], t16[16 * r]) : cmul<T>(v[it][r], t16[16 * r]);
        } else {
          C2<T> w1 = tw(k << (LOG2L - nsb - RB));
          if (INV) w1 = cconj<T>(w1);
          tw_stream<T, R>(v[it], w1);
        }
      }
      dft_reg<T, R, INV>(v[it]);
    }
  }
  __syncthreads();
  int e[RB];                                 // swz(Ns << b)
#pragma unroll
  for (int b = 0; b < RB; ++b) e[b] = swz<T>(Ns << b);
#pragma unroll
  for (int it = 0; it < IPT; ++it) {
    const int j = t0 + it * SW_NT;
    const int k = j & (Ns - 1);
    if ((Lr >= SW_NT) || j < Lr) {
      const int sb = swz<T>((j - k) * R + k);  // bit-disjoint from r Ns
#pragma unroll
      for (int r = 0; r < R; ++r) {
        int o = sb;
#pragma unroll
        for (int b = 0; b < RB; ++b)
          if (r & (1 << b)) o ^= e[b];
        buf[o] = v[it][bitrev<R>(r)];
      }
    }
  }
  __syncthreads();
}

// ---- the transposed pass (conjugated): the inverse FFT is conj(F)^T = conj(P_1)^T ...
// conj(P_last)^T (the DFT matrix is symmetric), i.e. the forward passes transposed and
// applied in reverse order.  Pass (radix 2^RB, stride Ns = 2^nsb), item j < L/R, k = j mod Ns:
//    V_r = x'[(j-k) R + k + r Ns],  u = DFT_R^{-1}(V),  x[j + s L/R] = u_s W_{Ns R}^{-s k}
// (the forward pass's write pattern read, its read pattern written, the twiddle after the
// DFT).  Compared with a second forward-ordered (DIT) inverse, the strides of the inverse
// are the forward's: Ns = 1 needs no twiddle, and the fused radix-2 pass stays in place.
template <typename T, int LOG2L, int RB>
CS_DEV void sw_pass_t(C2<T>* buf, const TwTable<T>& tw, int nsb) {
  constexpr int R = 1 << RB, Lr = (1 << LOG2L) >> RB;
  constexpr int IPT = Lr > SW_NT ? Lr / SW_NT : 1;
  const int t0 = opaque_tid<T, LOG2L>();
  C2<T> v[IPT][R];
  const int Ns = 1 << nsb;
  int e[RB];                                 // swz(Ns << b)
#pragma unroll
  for (int b = 0; b < RB; ++b) e[b] = swz<T>(Ns << b);
#pragma unroll
  for (int it = 0; it < IPT; ++it) {
    const int j = t0 + it * SW_NT;
    const int k = j & (Ns - 1);
    if ((Lr >= SW_NT) || j < Lr) {
      const int sb = swz<T>((j - k) * R + k);  // bit-disjoint from r Ns
#pragma unroll
      for (int r = 0; r < R; ++r) {
        int o = sb;
#pragma unroll
        for (int b = 0; b < RB; ++b)
          if (r & (1 << b)) o ^= e[b];
        v[it][r] = buf[o];
      }
      dft_reg<T, R, true>(v[it]);  // u_s at v[bitrev(s)]
      if (Ns > 1) {
        if (RB == 4 && SwPlan<LOG2L>::RBM == 4 && nsb == SwPlan<LOG2L>::NS1B) {
          constexpr SFix F = s_fixed<T>(int64_t(2) << LOG2L);
          const C2<T>* t16 = reinterpret_cast<const C2<T>*>(cs_smem_base + F.tw16) + k;  // [r][k]: conflict-free
#pragma unroll
          for (int q = 1; q < R; ++q) v[it][bitrev<R>(q)] = cmulc<T>(v[it][bitrev<R>(q)], t16[16 * q]);
        } else {
          C2<T> u[R];
#pragma unroll
          for (int q = 0; q < R; ++q) u[q] = v[it][bitrev<R>(q)];
          tw_stream<T, R>(u, cconj<T>(tw(k << (LOG2L - nsb - RB))));
#pragma unroll
          for (int q = 0; q < R; ++q) v[it][bitrev<R>(q)] = u[q];
        }
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < IPT; ++it) {
    const int j = t0 + it * SW_NT;
    if ((Lr >= SW_NT) || j < Lr) {
      const int sj = swz<T>(j);  // j < Lr: bit-disjoint from s Lr
#pragma unroll
      for (int q = 0; q < R; ++q) {
        if constexpr (Lr % 512 == 0) buf[sj + q * Lr] = v[it][bitrev<R>(q)];
        else buf[sj ^ swz_c<T>(q * Lr)] = v[it][bitrev<R>(q)];
      }
    }
  }
  __syncthreads();
}


// W_16^1 (a_{k + L/2} = a_k W_16)
template <typename T> CS_DEV C2<T> w16c() {
  return mk<T>((T)0.92387953251128675613, (T)-0.38268343236508977173);
}

// ---- the fused unit: last forward pass (radix 2), DCT middle, first inverse pass ----
// Unit k (1 <= k < L/4) owns items k and kb = L/2 - k of the radix-2 pass (Ns = L/2), i.e.
// the slots k, k + L/2, kb, kb + L/2 holding, after the pass,
//   A0 = Z_k, A1 = Z_{k+L/2}, B0 = Z_{L/2-k}, B1 = Z_{L-k};
// mirror pairs: (A0, B1) at n = k and (A1, B0) at n = k + L/2.
// Unit 0 (items 0 and L/4): Z_0 (alone), Z_{L/2} (self pair), (Z_{L/4}, Z_{3L/4}).
// The pass twiddles are W_L^k and W_L^{kb} = W_L^{L/2} W_L^{-k} = -conj(W_L^k) (one lookup).
// The first inverse pass is this pass transposed (sw_pass_t): inverse radix-2 butterfly,
// then the conjugate twiddle, written back to the SAME four slots — every thread writes
// only what it read, so the pass needs no barrier between its loads and stores.
// Row selection: for KIND 0 the 8 DCT indices of each of the thread's units are one byte of
// its `usel` word (built per instance by sw_build_usel): 8 it + q, q = 0..3 the pair n = k
// (k, N-k, L-k, N-L+k), q = 4..7 the pair n = k + L/2 (k+L/2, N-k-L/2, L/2-k, N-L/2+k).
// KIND 0: F = DCT-II (the middle above); KIND 1: F = partial Fourier (dct_mid.cuh dft_*, R36)
template <int LOG2L> CS_DEV int usel_idx(int k, int q) {
  constexpr int L = 1 << LOG2L, H = L / 2, N = 2 * L;
  const int n = (q < 4) ? k : k + H;
  const int kk = L - n;
  const int r = q & 3;
  return r == 0 ? n : r == 1 ? N - n : r == 2 ? kk : N - kk;
}

// usel[t]: bit 8 it + q set <=> DCT index usel_idx(t + SW_NT it, q) is a row (k >= 1 only)
template <typename T, int LOG2L>
CS_DEV void sw_build_usel_t(uint32_t* usel, const uint32_t* rowmask) {
  using SP = SwPlan<LOG2L>;
  for (int t = threadIdx.x; t < SW_NT; t += blockDim.x) {
    uint32_t w = 0;
#pragma unroll
    for (int it = 0; it < SP::UPT; ++it) {
      const int k = t + it * SW_NT;
      if (k >= 1 && k < SP::U) {
#pragma unroll
        for (int q = 0; q < 8; ++q) w |= (uint32_t)bit_test32(rowmask, usel_idx<LOG2L>(k, q)) << (8 * it + q);
      }
    }
    usel[t] = w;
  }
}

template <typename T, int MODE, int TY>
CS_DEV T mid_sel_op(const MidCtx<T>& m, const MidK<T>& c, bool sel, int idx, T raw, double& rn2) {
  return mid_op2g<T, MODE, TY>(m, c, sel, [&] { return row_rank32(m.rowmask, m.prefix, idx); }, raw, rn2);
}

template <typename T, int LOG2L, int MODE, bool ZERO, int KIND = 0>
CS_DEV double sw_fused(C2<T>* buf, const TwTable<T>& tw, const TwTable<T>& tw4, const MidCtx<T>& m) {
  using SP = SwPlan<LOG2L>;
  constexpr int L = 1 << LOG2L, H = L / 2, U = SP::U, UPT = SP::UPT, N = 2 * L;
  static_assert(L >= 4, "N >= 8");
  constexpr SFix F = s_fixed<T>(N);
  const int tid = opaque_tid<T, LOG2L>();
  const MidK<T> cst = make_midk_c<T, LOG2L + 1>();
  const uint32_t selw = (KIND == 0 && MODE == MID_H) ? reinterpret_cast<const uint32_t*>(cs_smem_base + F.usel)[tid] : 0u;
  double rn2 = 0;
#pragma unroll
  for (int it = 0; it < UPT; ++it) {
    const int k = tid + it * SW_NT;
    if ((U % SW_NT == 0) || k < U) {
      // unit 0 only exists for it = 0 (k = tid + 512 it): the compiler drops its branch elsewhere
      const bool k0 = (it == 0) && (k == 0);
      const int kb = k0 ? L / 4 : H - k;
      const C2<T> wk = k0 ? mk<T>(1, 0) : tw(k);                    // W_L^k
      const C2<T> wb = k0 ? mk<T>(0, -1) : mk<T>(-wk.x, wk.y);       // W_L^{kb}
      const int sa = swz<T>(k), sa2 = swz<T>(k + H), sb = swz<T>(kb), sb2 = swz<T>(kb + H);
      C2<T> A0, A1, B0, B1;
      if constexpr (ZERO) {
        A0 = A1 = B0 = B1 = mk<T>(0, 0);
      } else {
        // radix-2 pass, Ns = L/2: item j reads x[j], x[j + L/2]; twiddle W_L^j
        const C2<T> a0 = buf[sa], b0 = buf[sb];
        const C2<T> a1 = cmul<T>(buf[sa2], wk), b1 = cmul<T>(buf[sb2], wb);
        A0 = cadd<T>(a0, a1);
        A1 = csub<T>(a0, a1);
        B0 = cadd<T>(b0, b1);
        B1 = csub<T>(b0, b1);
      }
      if constexpr (KIND == 1) {
        if (!k0) {
          const C2<T> a = tw4(k);
          const C2<T> a2 = cmul<T>(a, a);
          const C2<T> w = cmul<T>(a2, a2);                     // W_N^k
          dft_pair_w<T, MODE>(A0, B1, k, w, m, rn2);
          dft_pair_w<T, MODE>(A1, B0, k + H, mk<T>(w.y, -w.x), m, rn2);
        } else {
          dft_zero<T, MODE>(A0, m, rn2);
          dft_pair<T, MODE>(A1, A1, H, tw4(H), m, rn2);  // self pair n = L/2
          dft_pair<T, MODE>(B0, B1, L / 4, tw4(L / 4), m, rn2);
        }
      } else {
        if (!k0) {
          const C2<T> a = tw4(k);
          const C2<T> a2 = cmul<T>(a, a);
          const C2<T> w = cmul<T>(a2, a2);                     // W_N^k
          // MID_H: selection from the thread's usel byte; RES / FWD: from the row mask (their
          // rank lookups read it anyway; the apply / adjoint kernels do not build usel)
          const uint32_t sl = selw >> (8 * it);
          auto sel = [&](int q) {
            if constexpr (MODE == MID_H) return ((sl >> q) & 1u) != 0;
            else return bit_test32(m.rowmask, usel_idx<LOG2L>(k, q));
          };
          mid_pair2g<T, MODE>(A0, B1, a, w, m, cst, rn2, [&](int q) { return sel(q); },
                              [&](int q) { return row_rank32(m.rowmask, m.prefix, usel_idx<LOG2L>(k, q)); });
          const C2<T> ah = cmul<T>(a, w16c<T>());              // W_4N^{k + L/2}
          const C2<T> wh = mk<T>(w.y, -w.x);                   // W_N^{k + L/2} = -i W_N^k
          mid_pair2g<T, MODE>(A1, B0, ah, wh, m, cst, rn2, [&](int q) { return sel(q + 4); },
                              [&](int q) { return row_rank32(m.rowmask, m.prefix, usel_idx<LOG2L>(k, q + 4)); });
        } else {
          mid_zero<T, MODE>(A0, m, rn2);
          mid_pair<T, MODE>(A1, A1, H, tw4(H), m, rn2);  // self pair n = L/2
          mid_pair<T, MODE>(B0, B1, L / 4, tw4(L / 4), m, rn2);
        }
      }
      if constexpr (MODE != MID_FWD) {
        // first inverse pass = the radix-2 pass transposed: butterfly, conj twiddle, in place
        buf[sa] = cadd<T>(A0, A1);
        buf[sa2] = cmulc<T>(csub<T>(A0, A1), wk);
        buf[sb] = cadd<T>(B0, B1);
        buf[sb2] = cmulc<T>(csub<T>(B0, B1), wb);
      }
    }
  }
  if constexpr (MODE != MID_FWD) __syncthreads();
  return rn2;
}

// ---- Psi = DCT (R35): the fused last-forward / first-inverse pass of the two extra
// transforms.  MID_FWDZ: after the forward FFT of s, the orthonormal DCT-II X = C_N s is
// written straight back into the buffer as the next transform's input, u_{pi^-1(k)} =
// sigma_k X_k at Makhoul position mk_pos(pi^-1(k)) (sigma, pi^-1 of Phi).  MID_INVZ: reads
// w_k = sigma_k v_{pi^-1(k)} from the buffer (v = Phi's sandwich output, Makhoul order) and
// writes the inverse-split spectrum of C_N^T w for the inverse FFT.  Every unit reads all
// of its values before the barrier and writes after it (in place).
// Unit k's indices: slot 0..3 pair n = k (k, N-k, L-k, N-L+k); slot 4..7 pair n = k + L/2;
// unit 0: (0, L), (L/2, N-L/2), (L/4, N-L/4, 3L/4, N-3L/4).
template <int LOG2L> CS_DEV int psi_idx(int k, int q) {
  constexpr int L = 1 << LOG2L, H = L / 2, N = 2 * L;
  if (k != 0) {
    const int n = (q < 4) ? k : k + H;
    const int kk = L - n;
    const int r = q & 3;
    return r == 0 ? n : r == 1 ? N - n : r == 2 ? kk : N - kk;
  }
  constexpr int t[8] = {0, L, H, N - H, L / 4, N - L / 4, 3 * L / 4, N - 3 * L / 4};
  return t[q];
}
template <typename T, int LOG2L, int MODE>
CS_DEV void sw_fused_psi(C2<T>* buf, const TwTable<T>& tw, const TwTable<T>& tw4, const MidCtx<T>& m,
                         const uint32_t* psig, const int32_t* ppinv) {
  using SP = SwPlan<LOG2L>;
  constexpr int L = 1 << LOG2L, H = L / 2, U = SP::U, UPT = SP::UPT, N = 2 * L;
  static_assert(L >= 4, "N >= 8");
  const int tid = threadIdx.x;
  T* zb = reinterpret_cast<T*>(buf);
  auto pos = [&](int idx) {
    const int p = (int)mk_pos(ppinv ? ppinv[idx] : idx, N);
    return 2 * swz<T>(p >> 1) + (p & 1);
  };
  auto sgn = [&](int idx, T v) { return ((psig[idx >> 5] >> (idx & 31)) & 1u) ? -v : v; };
  T o[UPT][8];
  if constexpr (MODE == MID_FWDZ) {
#pragma unroll
    for (int it = 0; it < UPT; ++it) {
      const int k = tid + it * SW_NT;
      if ((U % SW_NT == 0) || k < U) {
        const int kb = (k == 0) ? L / 4 : H - k;
        C2<T> a0 = buf[swz<T>(k)], a1 = buf[swz<T>(k + H)];
        C2<T> b0 = buf[swz<T>(kb)], b1 = buf[swz<T>(kb + H)];
        a1 = cmul<T>(a1, tw(k));
        b1 = cmul<T>(b1, tw(kb));
        const C2<T> A0 = cadd<T>(a0, a1), A1 = csub<T>(a0, a1), B0 = cadd<T>(b0, b1), B1 = csub<T>(b0, b1);
        if (k != 0) {
          const C2<T> a = tw4(k);
          dct_out_pair<T>(A0, B1, a, m, &o[it][0]);
          dct_out_pair<T>(A1, B0, cmul<T>(a, w16c<T>()), m, &o[it][4]);
        } else {
          dct_out_zero<T>(A0, m, &o[it][0]);
          T t4[4];
          dct_out_pair<T>(A1, A1, tw4(H), m, t4);   // self pair n = L/2: (H, N-H)
          o[it][2] = t4[0];
          o[it][3] = t4[1];
          dct_out_pair<T>(B0, B1, tw4(L / 4), m, &o[it][4]);
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < UPT; ++it) {
      const int k = tid + it * SW_NT;
      if ((U % SW_NT == 0) || k < U) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int idx = psi_idx<LOG2L>(k, q);
          zb[pos(idx)] = sgn(idx, o[it][q]);
        }
      }
    }
    __syncthreads();
  } else {  // MID_INVZ
#pragma unroll
    for (int it = 0; it < UPT; ++it) {
      const int k = tid + it * SW_NT;
      if ((U % SW_NT == 0) || k < U) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int idx = psi_idx<LOG2L>(k, q);
          o[it][q] = sgn(idx, zb[pos(idx)]);
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < UPT; ++it) {
      const int k = tid + it * SW_NT;
      if ((U % SW_NT == 0) || k < U) {
        const int kb = (k == 0) ? L / 4 : H - k;
        C2<T> A0, A1, B0, B1;
        if (k != 0) {
          const C2<T> a = tw4(k);
          dct_in_pair<T>(A0, B1, k, a, m, &o[it][0]);
          dct_in_pair<T>(A1, B0, k + H, cmul<T>(a, w16c<T>()), m, &o[it][4]);
        } else {
          dct_in_zero<T>(A0, m, &o[it][0]);
          dct_in_pair<T>(A1, A1, H, tw4(H), m, &o[it][2]);   // self pair (reads o[2], o[3])
          dct_in_pair<T>(B0, B1, L / 4, tw4(L / 4), m, &o[it][4]);
        }
        // first inverse pass: the radix-2 pass transposed, in place (as in sw_fused)
        const C2<T> wk = (k == 0) ? mk<T>(1, 0) : tw(k);
        const C2<T> wb = (k == 0) ? mk<T>(0, -1) : mk<T>(-wk.x, wk.y);
        buf[swz<T>(k)] = cadd<T>(A0, A1);
        buf[swz<T>(k + H)] = cmulc<T>(csub<T>(A0, A1), wk);
        buf[swz<T>(kb)] = cadd<T>(B0, B1);
        buf[swz<T>(kb + H)] = cmulc<T>(csub<T>(B0, B1), wb);
      }
    }
    __syncthreads();
  }
}

template <typename T, int LOG2L, bool INV>
CS_DEV void sw_remainder(C2<T>* buf, const TwTable<T>& tw, int nsb) {
  constexpr int M = SwPlan<LOG2L>::M;
  if constexpr (M > 0) sw_pass<T, LOG2L, M, INV>(buf, tw, nsb);
}

// the usel table for a runtime transform length (log2 L in [2, 13])
template <typename T, int LO = 2, int HI = 13>
CS_DEV void sw_build_usel(int log2l, uint32_t* usel, const uint32_t* rowmask) {
  if constexpr (LO <= HI) {
    if (log2l == LO) { sw_build_usel_t<T, LO>(usel, rowmask); return; }
    sw_build_usel<T, LO + 1, HI>(log2l, usel, rowmask);
  }
}

// The whole sandwich as ONE out-of-line unit (one ABI register save/restore per
// sandwich):
//   vin != nullptr : zero the buffer and scatter sigma . vin on supp (Makhoul order)
//   vin == nullptr : the buffer already holds the forward input (ZERO: it is 0)
//   forward FFT, fused last pass / middle / first inverse pass, inverse FFT,
//   vout != nullptr: gather vout[i] = sigma . buf[supp[i]] (H d restricted to S).
template <typename T> struct SwIO {
  const int* supp;
  int ns;
  const uint32_t* sign;       // MID_FWDZ / MID_INVZ: Phi's sign bits (global); otherwise unused
  const T* vin;
  T* vout;
  const int32_t* pinv_phi;    // MID_FWDZ / MID_INVZ: Phi's pi^-1 (global) or null
};

// PERM = false: the caller guarantees no Eq.(7) permutation (the CG loop of a plain
// operator), so the scatter / gather carry no pi^-1 lookup.
template <typename T, int LOG2L, int MODE, bool ZERO, bool PERM = true, int KIND = 0>
CS_DEV double sw_body(C2<T>* gbuf, const TwTable<T>& gtw, const TwTable<T>& gtw4, const MidCtx<T>& gm,
                      const SwIO<T>& gio) {
  using SP = SwPlan<LOG2L>;
  constexpr int L = 1 << LOG2L, N = 2 * L;
  // The FFT buffer, twiddle tables and operator metadata sit at compile-time offsets
  // of the Tier S layout (layout_s.cuh); gbuf / gtw / gtw4 / gm name the same objects.
  constexpr SFix F = s_fixed<T>(N);
  (void)gbuf; (void)gtw; (void)gtw4;
  C2<T>* buf = reinterpret_cast<C2<T>*>(cs_smem_base + F.Z);
  const TwTable<T> tw{reinterpret_cast<const C2<T>*>(cs_smem_base + F.twLlo),
                      reinterpret_cast<const C2<T>*>(cs_smem_base + F.twLhi)};
  const TwTable<T> tw4{reinterpret_cast<const C2<T>*>(cs_smem_base + F.tw4lo),
                       reinterpret_cast<const C2<T>*>(cs_smem_base + F.tw4hi)};
  const MidCtx<T> m = make_mid_c<T, LOG2L + 1>(reinterpret_cast<const uint32_t*>(cs_smem_base + F.rmask),
                                                reinterpret_cast<const int32_t*>(cs_smem_base + F.prefix),
                                                gm.y, gm.yout);
  const uint32_t* signs = reinterpret_cast<const uint32_t*>(cs_smem_base + F.sign);
  const int tid = threadIdx.x;
  T* zb = reinterpret_cast<T*>(buf);
  auto zt = [](int p) { return 2 * swz<T>(p >> 1) + (p & 1); };
  static_assert(MODE != MID_INVZ || ZERO, "MID_INVZ reads the buffer as it is (no forward FFT)");
  if constexpr (!ZERO) {
    if (gio.vin) {
      const int* supp = shp(gio.supp);
      const uint32_t* sign = signs;
      const T* vin = shp(gio.vin);
      if constexpr (sizeof(T) == 4 && L % (2 * SW_NT) == 0) {
        float4* b4 = reinterpret_cast<float4*>(buf);   // zeros: 16-byte stores, half the count
#pragma unroll
        for (int i = tid; i < L / 2; i += SW_NT) b4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      } else {
        for (int i = tid; i < L; i += SW_NT) buf[i] = mk<T>(0, 0);
      }
      __syncthreads();
      // Eq.(7) randomizer pi^-1 (R34), parked in shared memory by make_cta_ctx
      const int32_t* pv = PERM ? *reinterpret_cast<const int32_t* const*>(cs_smem_base + F.zero + 8) : nullptr;
      for (int i = tid; i < gio.ns; i += SW_NT) {
        const int j = supp[i];
        zb[zt((int)mk_pos((PERM && pv) ? pv[j] : j, N))] = apply_sign<T>(sign, j, vin[i]);
      }
      __syncthreads();
    }
    sw_remainder<T, LOG2L, false>(buf, tw, 0);
#pragma unroll
    for (int q = 0; q < SP::Q; ++q) sw_pass<T, LOG2L, SP::RBM, false>(buf, tw, SP::NS_R16_FWD0 + SP::RBM * q);
  }
  double rn2 = 0;
  if constexpr (MODE == MID_FWDZ || MODE == MID_INVZ) {
    sw_fused_psi<T, LOG2L, MODE>(buf, tw, tw4, m, gio.sign, gio.pinv_phi);
  } else {
    rn2 = sw_fused<T, LOG2L, MODE, ZERO, KIND>(buf, tw, tw4, m);
  }
  if constexpr (MODE != MID_FWD && MODE != MID_FWDZ) {
#pragma unroll
    for (int q = SP::Q - 1; q >= 0; --q) sw_pass_t<T, LOG2L, SP::RBM>(buf, tw, SP::NS_R16_FWD0 + SP::RBM * q);
    if constexpr (SP::M > 0) sw_pass_t<T, LOG2L, SP::M>(buf, tw, 0);
    if (gio.vout) {
      const int* supp = shp(gio.supp);
      const uint32_t* sign = signs;
      T* vout = shp(gio.vout);
      const int32_t* pv = PERM ? *reinterpret_cast<const int32_t* const*>(cs_smem_base + F.zero + 8) : nullptr;
      for (int i = tid; i < gio.ns; i += SW_NT) {
        const int j = supp[i];
        vout[i] = apply_sign<T>(sign, j, zb[zt((int)mk_pos((PERM && pv) ? pv[j] : j, N))]);
      }
      __syncthreads();
    }
  }
  return rn2;
}

// Out of line: only scalars cross the call (no structs passed by value — at 1024
// threads per SM every by-value byte is a local-memory store and load).
template <typename T, int LOG2L, int MODE, bool ZERO, int KIND = 0>
CS_NOINL double sw_sandwich_t(const T* y, T* yout, const int* supp, int ns, const T* vin, T* vout,
                              const uint32_t* psig, const int32_t* ppinv) {
  MidCtx<T> gm;
  gm.y = y;
  gm.yout = yout;
  const SwIO<T> gio{supp, ns, psig, vin, vout, ppinv};
  return sw_body<T, LOG2L, MODE, ZERO, true, KIND>(nullptr, TwTable<T>{}, TwTable<T>{}, gm, gio);
}

// runtime dispatch over log2 L in [LO, HI]
template <typename T, int LO, int HI, int MODE, bool ZERO, int KIND = 0>
CS_DEV double sw_dispatch(int log2l, const T* y, T* yout, const int* supp, int ns, const T* vin, T* vout,
                          const uint32_t* psig = nullptr, const int32_t* ppinv = nullptr) {
  if constexpr (LO <= HI) {
    if (log2l == LO) return sw_sandwich_t<T, LO, MODE, ZERO, KIND>(y, yout, supp, ns, vin, vout, psig, ppinv);
    return sw_dispatch<T, LO + 1, HI, MODE, ZERO, KIND>(log2l, y, yout, supp, ns, vin, vout, psig, ppinv);
  }
  return 0.0;
}

}  // namespace cs
