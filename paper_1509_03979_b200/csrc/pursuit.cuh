// pursuit.cuh — CG-based weighted least squares and the three greedy pursuits,
// written once against the context interface (CTA context = one problem per
// thread block; grid context = one problem per cooperative grid).
//
//  cg_solve : Algorithm 1 function CG on Eq.(11) restricted
//             to the support (Thm 5 / Eq.(12)): compact |S| vectors,
//             H d = (A^T A scatter_S d)[S] via the operator sandwich, warm start,
//             relative stopping rule (R6, R7, R9, R29).
//  omp      : Algorithm 1 lines 01-10, exactly K iterations.
//  sp       : CG-SP, body per S:289 / SURVEY §8c.4 (R15).
//  ompr     : CG-OMPR(l, eta), body per S:299 / SURVEY §8c.5 (R16).
//  cosamp   : CG-CoSaMP (named P:84), the published CoSaMP iteration with the
//             paper's CG as its LS step; halting rule R33.
//
// Every thread of the context runs the same control flow; scalars come out of
// deterministic collectives, so every branch is uniform.
#pragma once
#include "cs_common.cuh"
#include "select.cuh"

#include <type_traits>

namespace cs {

template <typename T> struct Bufs {
  int *S, *S2, *U;        // supports: current (K), candidate (K), union/merge (K + l or 2K)
  T *x, *x2, *xU;         // coefficients on them
  T *r, *d, *q, *b;       // CG vectors (cap 2K)
  uint32_t *Sbits, *Ubits, *Pbits;  // [N/32], [N/32], [ceil(2K/32)]
};

struct Stats {
  int outer, cg_iters, cg_solves, term;
  unsigned status;
  double rel_max;
};

struct Params {
  int K, alg, max_outer, cg_cap, ompr_l;
  double tol, eta;
};

// ------------------------------------------------------------------ CG ------
// State of one CG solve (Algorithm 1 lines 13-22) while it iterates.
template <typename T> struct CgState {
  T *x, *r, *d, *q;
  double rr, thr;  // r.r and the stopping threshold tol^2 ||b||^2 (R6, R7)
  int ns, cap, j;
  unsigned status;
};

// sum_i a_i b_i over i < n, deterministic (the context's fixed-order sum)
template <class Ctx, typename T>
CS_DEV double dot_n(Ctx& c, const T* a, const T* b, int n) {
  double v = 0;
  for (int i = c.gtid; i < n; i += c.gnthr) v += (double)a[i] * (double)b[i];
  return c.sum(v);
}

// The CG iteration loop, generic over the context; Hf(d, q) applies
// q = H d on the context's remembered support and returns d.q (the grid context fuses
// the dot product into H's last pass and barrier).  Each context runs it from its
// cg_iterate(): the grid context directly, the CTA context from an out-of-line
// instance per transform length with the sandwich inlined.
template <class Ctx, typename T, class HFn>
CS_DEV void cg_loop(Ctx& c, CgState<T>& s_io, HFn&& Hf) {
  CgState<T> s = s_io;  // register copy (s_io lives in the caller's frame)
  const int a0 = c.gtid, s0 = c.gnthr;
  T *xx = s.x, *rv = s.r, *dv = s.d, *qv = s.q;
  const int n = s.ns;
  while (true) {
    if (!(s.rr > s.thr)) break;                                            // line 15 (R6, R7)
    if (s.j >= s.cap) { s.status |= CS_DEV_CG_CAP; break; }
    const double dq = Hf(dv, qv);                                          // H d_j, d_j.H d_j
    if (!(dq > 0.0)) { s.status |= CS_DEV_CG_BREAKDOWN; break; }
    const T alpha = (T)(s.rr / dq);                                        // line 16
    double rr2 = 0;
    for (int i = a0; i < n; i += s0) {
      xx[i] += alpha * dv[i];                                              // line 17
      const T ri = rv[i] - alpha * qv[i];                                  // line 18
      rv[i] = ri;
      rr2 += (double)ri * (double)ri;
    }
#ifdef CS_DIAG_CG
    c.mark(15);  // x, r update
#endif
    rr2 = c.sum(rr2);
#ifdef CS_DIAG_CG
    c.mark(16);  // ||r||^2 reduction
#endif
    const T beta = (T)(rr2 / s.rr);                                        // line 19
    if constexpr (Ctx::kDeferD)
      c.defer_d(dv, rv, beta);   // line 20, applied by the next H's scatter (ctx_grid.cuh)
    else
      for (int i = a0; i < n; i += s0) dv[i] = rv[i] + beta * dv[i];      // line 20
    s.rr = rr2;
    s.j += 1;                                                              // line 21
    if (!(rr2 == rr2)) { s.status |= CS_DEV_CG_BREAKDOWN; break; }
  }
  if constexpr (Ctx::kDeferD) c.defer_d(nullptr, nullptr, T(0));   // d is dead after the loop
  s_io = s;
}

// cg_solve, detect_topk / detect_argmax and the CTA context's RES are inlined into the
// pursuits: each out-of-line call pays a register save / restore through local memory,
// which at 1024 resident threads per SM spills to L2 (measured: -3.2 % on c4 together).
// Solves H x = b on supp (b = c0[supp]).  x holds the warm start on entry.
// If r_given, r holds r0 = b - H x0 on entry (free when x0 is the previous LS
// iterate and r = c[supp], see pursuits.py); otherwise one H apply computes it.
template <class Ctx, typename T>
CS_DEV void cg_solve(Ctx& ctx, const int* supp, int ns, T* x, T* r, T* d, T* q, T* b, bool r_given,
                       const Params& P, Stats& st) {
  ctx.mark(0);
  ctx.set_input_support(supp, ns);
#ifdef CS_DIAG_GLUE
  ctx.mark(17);  // set_input_support
#endif
  supp = ctx.loc(supp);
  x = ctx.loc(x);
  r = ctx.loc(r);
  d = ctx.loc(d);
  q = ctx.loc(q);
  b = ctx.loc(b);
  const int t0 = ctx.gtid, sd = ctx.gnthr;
  {
    const auto c0v = ctx.c0view();
    for (int i = t0; i < ns; i += sd) b[i] = c0v.at(supp[i]);             // line 12
  }
  // no barrier: b[i] is read below only by the thread that wrote it (same i mapping)
#ifdef CS_DIAG_GLUE
  ctx.mark(18);  // b gather
#endif
  if (!r_given) {
    ctx.H(x, q);
    for (int i = t0; i < ns; i += sd) r[i] = b[i] - q[i];
  }
  double bb = 0, rr = 0;
  for (int i = t0; i < ns; i += sd) {
    bb += (double)b[i] * (double)b[i];
    rr += (double)r[i] * (double)r[i];
    d[i] = r[i];                                                           // line 13
  }
  ctx.sum2(bb, rr);   // one reduction for both
  CgState<T> cs_{x, r, d, q, rr, P.tol * P.tol * bb, ns, P.cg_cap > 0 ? P.cg_cap : ns + 50, 0, 0u};
  ctx.mark(8);
  ctx.cg_iterate(cs_);                                                     // lines 14-22
  st.status |= cs_.status;
  ctx.sync();
#ifdef CS_DIAG_GLUE
  ctx.mark(19);  // CG loop exit: flush + barrier
#endif
  st.cg_iters += cs_.j;
  st.cg_solves += 1;
  double rel = bb > 0 ? sqrt(cs_.rr / bb) : 0.0;
  if (rel > st.rel_max) st.rel_max = rel;
}

// rebuild Sbits from the list S (ns entries)
template <class Ctx, typename T>
CS_DEV void bits_from_list(Ctx& ctx, uint32_t* bits, int64_t nwords, const int* S, int ns) {
  for (int64_t w = ctx.gtid; w < nwords; w += ctx.gnthr) bits[w] = 0u;
  ctx.sync();
  for (int i = ctx.gtid; i < ns; i += ctx.gnthr) atomicOr(&bits[S[i] >> 5], 1u << (S[i] & 31));
  ctx.sync();
}

template <class Ctx, typename T>
CS_DEV bool same_list(Ctx& ctx, const int* a, const int* b, int n) {
  if constexpr (Ctx::kTopkFast) {
    // CTA: one barrier-vote, no reduction slots
    int d = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) d |= (a[i] != b[i]);
    return !__syncthreads_or(d);
  }
  double diff = 0;
  for (int i = ctx.gtid; i < n; i += ctx.gnthr) diff += (a[i] != b[i]) ? 1.0 : 0.0;
  return ctx.sum(diff) == 0.0;
}

template <class Ctx, typename T>
CS_DEV void swap_ptr(T*& a, T*& b) { T* t = a; a = b; b = t; }

// top-K of |c_j| over j in [0,N) \ excl (excl may be null) -> out bits over [0, N)
template <class Ctx, typename T>
CS_DEV void detect_topk(Ctx& ctx, int64_t K, const uint32_t* excl, uint32_t* out) {
  const int64_t N = ctx.N;
  auto cv = ctx.cview();
  cv.z = ctx.loc(cv.z);
  cv.sign = ctx.loc(cv.sign);
  excl = excl ? ctx.loc(excl) : nullptr;
  using Key = decltype(full_key(T(0)));
  if constexpr (Ctx::kTopkFast) {
    // CTA: visit the correlation buffer in its own (Makhoul, swizzled) order, two
    // positions per complex slot, instead of gathering it in natural index order
    const int n = (int)N, L = n / 2;
    const C2<T>* zs = reinterpret_cast<const C2<T>*>(cv.z);
    const int32_t* pm = ctx.pm;   // Eq.(7) randomizer: position i holds index pi(i) (R34)
    // the permuted and the plain visitor are separate instances (no per-element branch)
    auto run = [&](auto has_pm) -> bool {
      constexpr bool HP = decltype(has_pm)::value;
      // slot q holds Makhoul positions 2q, 2q+1: indices (4q, 4q+2) for q < n/4 and
      // (2n-1-4q, 2n-3-4q) above — two loops, no per-slot selection of the formula
      auto slot = [&](auto&& f, int q, int j0, int j1) {
          const C2<T> z = zs[swz<T>(q)];
          Key k0 = full_key(z.x), k1 = full_key(z.y);
          if constexpr (HP) {
            j0 = pm[j0];
            j1 = pm[j1];
            if (excl) {
              if (bit_test(excl, j0)) k0 = Key(0);
              if (bit_test(excl, j1)) k1 = Key(0);
            }
          } else if (excl) {
            // j0, j1 = 4q, 4q+2 or 2n-1-4q, 2n-3-4q: always one exclusion word (n >= 16)
            const uint32_t w = excl[j0 >> 5];
            k0 = ((w >> (j0 & 31)) & 1u) ? Key(0) : k0;
            k1 = ((w >> (j1 & 31)) & 1u) ? Key(0) : k1;
          }
          f(j0, k0);
          f(j1, k1);
      };
      auto visit = [&](auto&& f) {
        const int h = n >> 2;
        for (int q = threadIdx.x; q < h; q += blockDim.x) slot(f, q, 4 * q, 4 * q + 2);
        for (int q = h + threadIdx.x; q < L; q += blockDim.x) slot(f, q, 2 * n - 1 - 4 * q, 2 * n - 3 - 4 * q);
      };
      return topk_cta_fast_v<Ctx, Key>(ctx, n, (int)K, visit, out);
    };
    if (pm ? run(std::true_type{}) : run(std::false_type{})) return;
  }
  if constexpr (!Ctx::kTopkFast) {
    // grid: materialise the keys once in natural index order (the dense input buffer U
    // is free during a recovery), so the radix passes read them contiguously
    Key* keys = reinterpret_cast<Key*>(ctx.U);
    if constexpr (sizeof(T) == 4) {
      if (!cv.pinv && N % 4 == 0) {
        // four consecutive j per unit from two 8-byte loads of the Makhoul-ordered buffer
        // (x[4q], x[4q+2] at positions 2q, 2q+1; x[4q+3], x[4q+1] at N-2-2q, N-1-2q), one
        // exclusion word, one 16-byte key store — the scalar gather ran at a fraction of
        // the bandwidth (as the adjoint's, tier_l.cuh k_l_adjoint)
        const T* z = cv.z;
        gstaged<TL_UNR, uint4>(N / 4, ctx.gtid, ctx.gnthr, [&](int64_t q) {
          const float2 lo = *reinterpret_cast<const float2*>(z + 2 * q);
          const float2 hi = *reinterpret_cast<const float2*>(z + N - 2 - 2 * q);
          uint4 k = make_uint4(full_key(lo.x), full_key(hi.y), full_key(lo.y), full_key(hi.x));
          if (excl) {
            const int64_t j = 4 * q;
            const uint32_t w = excl[j >> 5] >> (j & 31);
            if (w & 1u) k.x = 0u;
            if (w & 2u) k.y = 0u;
            if (w & 4u) k.z = 0u;
            if (w & 8u) k.w = 0u;
          }
          return k;
        }, [&](int64_t q, uint4 k) { *reinterpret_cast<uint4*>(keys + 4 * q) = k; });
        ctx.sync();
        const uint4* k4 = reinterpret_cast<const uint4*>(keys);
        topk_bits(ctx, N, K, [keys](int64_t j) { return keys[j]; }, out, false,
                  [k4](int64_t q) { return k4[q]; });
        return;
      }
    }
    gstaged<TL_UNR, Key>(N, ctx.gtid, ctx.gnthr, [&](int64_t j) {
      return (excl && bit_test(excl, j)) ? Key(0) : full_key(cv.raw(j));
    }, [&](int64_t j, Key k) { keys[j] = k; });
    ctx.sync();
    topk_bits(ctx, N, K, [keys](int64_t j) { return keys[j]; }, out, false);
    return;
  }
  topk_bits(ctx, N, K, [cv, excl](int64_t j) {
    if (excl && bit_test(excl, j)) return Key(0);
    return full_key(cv.raw(j));
  }, out, false);
}

template <class Ctx, typename T>
CS_DEV int64_t detect_argmax(Ctx& ctx, const uint32_t* excl) {
  const int64_t N = ctx.N;
  auto cv = ctx.cview();
  cv.z = ctx.loc(cv.z);
  cv.sign = ctx.loc(cv.sign);
  excl = ctx.loc(excl);
  using Key = decltype(full_key(T(0)));
  if constexpr (Ctx::kTopkFast) {
    const int n = (int)N, L = n / 2;
    const C2<T>* zs = reinterpret_cast<const C2<T>*>(cv.z);
    Key bk = 0;
    int64_t bi = -1;
    auto take = [&](int j, Key k) {  // larger key wins, ties -> lower index (R12)
      if (k > bk || (k == bk && k != 0 && j < bi)) { bk = k; bi = j; }
    };
    const int32_t* pm = ctx.pm;
    auto scan = [&](auto has_pm) {
      constexpr bool HP = decltype(has_pm)::value;
      for (int q = threadIdx.x; q < L; q += blockDim.x) {
        const C2<T> z = zs[swz<T>(q)];
        int j0 = (4 * q < n) ? 4 * q : 2 * (n - 1 - 2 * q) + 1;
        int j1 = (4 * q + 2 < n) ? 4 * q + 2 : 2 * (n - 2 - 2 * q) + 1;
        if constexpr (HP) {
          j0 = pm[j0];
          j1 = pm[j1];
          take(j0, bit_test(excl, j0) ? Key(0) : full_key(z.x));
          take(j1, bit_test(excl, j1) ? Key(0) : full_key(z.y));
        } else {
          const uint32_t w = excl[j0 >> 5];   // one word for both (see detect_topk)
          take(j0, ((w >> (j0 & 31)) & 1u) ? Key(0) : full_key(z.x));
          take(j1, ((w >> (j1 & 31)) & 1u) ? Key(0) : full_key(z.y));
        }
      }
    };
    if (pm) scan(std::true_type{}); else scan(std::false_type{});
    return ctx.argmax(bk, bi);
  }
  if constexpr (sizeof(T) == 4) {
    if (!cv.pinv && N % 4 == 0) {
      // four consecutive j per unit from two 8-byte loads (as detect_topk's grid keys), in
      // increasing j per thread so the first maximum is kept (ties -> lower index, R12)
      const T* z = cv.z;
      Key bk = 0;
      int64_t bi = -1;
      for (int64_t q = ctx.gtid; q < N / 4; q += ctx.gnthr) {
        const float2 lo = *reinterpret_cast<const float2*>(z + 2 * q);
        const float2 hi = *reinterpret_cast<const float2*>(z + N - 2 - 2 * q);
        const int64_t j = 4 * q;
        const uint32_t w = excl[j >> 5] >> (j & 31);
        const Key k0 = (w & 1u) ? Key(0) : full_key(lo.x), k1 = (w & 2u) ? Key(0) : full_key(hi.y);
        const Key k2 = (w & 4u) ? Key(0) : full_key(lo.y), k3 = (w & 8u) ? Key(0) : full_key(hi.x);
        if (k0 > bk) { bk = k0; bi = j; }
        if (k1 > bk) { bk = k1; bi = j + 1; }
        if (k2 > bk) { bk = k2; bi = j + 2; }
        if (k3 > bk) { bk = k3; bi = j + 3; }
      }
      return ctx.argmax(bk, bi);
    }
  }
  return argmax_key(ctx, N, [cv, excl](int64_t j) {
    if (bit_test(excl, j)) return Key(0);
    return full_key(cv.raw(j));
  });
}

// ------------------------------------------------------------------ OMP -----
template <class Ctx, typename T>
CS_NOINL int run_omp(Ctx& ctx, const Params& P, Bufs<T>& B, Stats& st, double& rn2) {
  const int64_t nwords = (ctx.N + 31) >> 5;
  rn2 = ctx.RES((const T*)nullptr);      // c = A^T y   (r_0 = y)
  ctx.save_c0();
  for (int64_t w = ctx.gtid; w < nwords; w += ctx.gnthr) B.Sbits[w] = 0u;
  ctx.sync();
  int ns = 0;
  int *S = B.S, *S2 = B.S2;
  T *x = B.x, *x2 = B.x2;
  for (int it = 0; it < P.K; ++it) {                                   // line 02
    if (it > 0) {
      // (input support: set by the cg_solve above)
      rn2 = ctx.RES(x);                                               // lines 07 + 03
    }
    int64_t t = detect_argmax<Ctx, T>(ctx, B.Sbits);                  // line 03, Eq.(6)
    if (t < 0) break;
    if (ctx.gtid == 0) B.Sbits[t >> 5] |= 1u << (t & 31);             // line 04
    ctx.sync();
    int ns2 = (int)compact_bits(ctx, B.Sbits, ctx.N, [&](int64_t k, int64_t j) { S2[k] = (int)j; });
    remap(ctx, S, x, ns, S2, x2, ns2);                                // warm start (R9)
    {
      const auto cv = ctx.cview();
      for (int i = ctx.gtid; i < ns2; i += ctx.gnthr) B.r[i] = cv.at(S2[i]);  // free r0
    }
    swap_ptr<Ctx>(S, S2);
    swap_ptr<Ctx>(x, x2);
    ns = ns2;
    cg_solve(ctx, S, ns, x, B.r, B.d, B.q, B.b, true, P, st);        // line 06
    st.outer = it + 1;
  }
  ctx.set_input_support(S, ns);
  rn2 = ctx.RES(x);                                                   // final r_K (line 07)
  st.term = CS_TERM_DONE;
  B.S = S; B.S2 = S2; B.x = x; B.x2 = x2;
  return ns;
}

// ------------------------------------------------------------------ SP ------
template <class Ctx, typename T>
CS_NOINL int run_sp(Ctx& ctx, const Params& P, Bufs<T>& B, Stats& st, double& rn2) {
  const int64_t N = ctx.N, nwords = (N + 31) >> 5;
  const int K = P.K;
  int *S = B.S, *S2 = B.S2, *U = B.U;
  T *x = B.x, *x2 = B.x2, *xU = B.xU;
  double ry2 = ctx.RES((const T*)nullptr);                       // c0 = A^T y
  (void)ry2;
  ctx.save_c0();
  detect_topk<Ctx, T>(ctx, K, nullptr, B.Sbits);                 // S = top-K |A^T y|
  int ns = (int)compact_bits(ctx, B.Sbits, N, [&](int64_t k, int64_t j) { S[k] = (int)j; });
  for (int i = ctx.gtid; i < ns; i += ctx.gnthr) { x[i] = T(0); B.r[i] = ctx.c_at(S[i]); }
  cg_solve(ctx, S, ns, x, B.r, B.d, B.q, B.b, true, P, st);
  // (input support: set by the cg_solve above)
  rn2 = ctx.RES(x);                                              // r = y - A x, c = A^T r
  const int max_outer = P.max_outer > 0 ? P.max_outer : 30;
  st.term = CS_TERM_ITER_CAP;
  for (int it = 1; it <= max_outer; ++it) {
    st.outer = it;
    ctx.mark(0);
    detect_topk<Ctx, T>(ctx, K, B.Sbits, B.Ubits);               // J = top-K off S
    ctx.mark(7);
    for (int64_t w = ctx.gtid; w < nwords; w += ctx.gnthr) B.Ubits[w] |= B.Sbits[w];  // T = S u J
    ctx.sync();
    int nu = (int)compact_bits(ctx, B.Ubits, N, [&](int64_t k, int64_t j) { U[k] = (int)j; });
    remap(ctx, S, x, ns, U, xU, nu);                             // x0 = x on S, 0 on J
    {
      const auto cv = ctx.cview();
      for (int i = ctx.gtid; i < nu; i += ctx.gnthr) B.r[i] = cv.at(U[i]);   // r0 = c[T]
    }
    cg_solve(ctx, U, nu, xU, B.r, B.d, B.q, B.b, true, P, st);
    // prune: S' = top-K of |x_T| over T (positions ascending == indices ascending)
    const T* xUc = xU;
    topk_bits(ctx, (int64_t)nu, (int64_t)K, [&](int64_t i) { return full_key(xUc[i]); }, B.Pbits);
    int ns2 = (int)compact_bits(ctx, B.Pbits, nu, [&](int64_t k, int64_t pos) {
      S2[k] = U[pos];
      x2[k] = xU[pos];
    });
    if (same_list<Ctx, T>(ctx, S, S2, ns)) { st.term = CS_TERM_SUPPORT_FIXED; break; }
    cg_solve(ctx, S2, ns2, x2, B.r, B.d, B.q, B.b, false, P, st);
    // (input support: set by the cg_solve above)
    double rn2new = ctx.RES(x2);
    if (rn2new >= rn2) { st.term = CS_TERM_RESID_ROSE; break; }   // keep (S, x)
    swap_ptr<Ctx>(S, S2);
    swap_ptr<Ctx>(x, x2);
    ns = ns2;
    rn2 = rn2new;
    bits_from_list<Ctx, T>(ctx, B.Sbits, nwords, S, ns);
  }
  B.S = S; B.S2 = S2; B.x = x; B.x2 = x2;
  return ns;
}

// ------------------------------------------------------------------ OMPR ----
template <class Ctx, typename T>
CS_NOINL int run_ompr(Ctx& ctx, const Params& P, Bufs<T>& B, Stats& st, double& rn2) {
  const int64_t N = ctx.N, nwords = (N + 31) >> 5;
  const int K = P.K;
  const int l = P.ompr_l > 0 ? P.ompr_l : 1;
  const T eta = (T)(P.eta > 0 ? P.eta : 1.0);
  int *S = B.S, *S2 = B.S2, *U = B.U;
  T *x = B.x, *x2 = B.x2, *xU = B.xU;
  ctx.RES((const T*)nullptr);
  ctx.save_c0();
  detect_topk<Ctx, T>(ctx, K, nullptr, B.Sbits);
  int ns = (int)compact_bits(ctx, B.Sbits, N, [&](int64_t k, int64_t j) { S[k] = (int)j; });
  for (int i = ctx.gtid; i < ns; i += ctx.gnthr) { x[i] = T(0); B.r[i] = ctx.c_at(S[i]); }
  cg_solve(ctx, S, ns, x, B.r, B.d, B.q, B.b, true, P, st);
  // (input support: set by the cg_solve above)
  rn2 = ctx.RES(x);
  const int max_outer = P.max_outer > 0 ? P.max_outer : 2 * K;
  st.term = CS_TERM_ITER_CAP;
  for (int it = 1; it <= max_outer; ++it) {
    st.outer = it;
    if (l == 1) {
      // OMPR(1): J = {j}, j = argmax |c| off S (z = x~ + eta c = eta c off S); S u J has
      // K + 1 entries, so S' = top-K of |z| over it drops exactly the entry with the
      // smallest |z| (ties: the lowest indices are kept, the highest such one drops).
      // Done as a sorted insert / delete and one argmin — no bitmask compaction or
      // radix select (each costs several grid barriers in the grid context).
      ctx.mark(0);
      const int64_t j = detect_argmax<Ctx, T>(ctx, B.Sbits);
      if (j < 0) { st.term = CS_TERM_SUPPORT_FIXED; break; }
      // j's place in S u J = #{i : S[i] < j}: a 32-ary search per warp (3 dependent loads
      // at K = 8192 instead of 13 for a binary search; S is in global memory on the grid)
      const int* Sl = ctx.loc(S);
      int lo = 0, hi = ns;
      const int lane = (int)(threadIdx.x & 31);
      while (hi - lo > 32) {
        const int step = (hi - lo + 31) >> 5;
        const int p = lo + (lane + 1) * step - 1;                     // last entry of segment lane
        const int L = __popc(__ballot_sync(0xffffffffu, p < hi && Sl[p] < j));
        lo += L * step;                                               // segments before L: all < j
        hi = min(hi, lo + step);                                      // segment L ends >= j
      }
      const int pos = lo + __popc(__ballot_sync(0xffffffffu, lo + lane < hi && Sl[lo + lane] < j));
      {
        auto cv = ctx.cview();
        cv.z = ctx.loc(cv.z);
        cv.sign = ctx.loc(cv.sign);
        for (int i = ctx.gtid; i <= ns; i += ctx.gnthr) {
          const int u = (i < pos) ? S[i] : (i == pos ? (int)j : S[i - 1]);
          const T xv = (i < pos) ? x[i] : (i == pos ? T(0) : x[i - 1]);
          U[i] = u;
          xU[i] = xv + eta * cv.at(u);                                // z on S u J
        }
      }
      // no barrier: the argmin below reads xU[i] in the thread that wrote it; U and xU are
      // read across threads only after its reduction barrier
      using Key = decltype(full_key(T(0)));
      const Key kmax = Key(1) << (sizeof(Key) * 8 - 1);              // above every key
      Key bk = 0;
      int64_t bi = -1;
      for (int i = ctx.gtid; i <= ns; i += ctx.gnthr) {
        const Key kk = kmax - full_key(xU[i]) + 1;                    // larger = smaller |z|
        const int64_t id = ns - i;                                    // smaller = higher position
        if (kk > bk || (kk == bk && id < bi)) { bk = kk; bi = id; }
      }
      const int drop = (int)(ns - ctx.argmax(bk, bi));
      if (drop == pos) { st.term = CS_TERM_SUPPORT_FIXED; break; }    // S' == S
      for (int i = ctx.gtid; i < ns; i += ctx.gnthr) {
        const int src = (i < drop) ? i : i + 1;
        S2[i] = U[src];
        x2[i] = (src < pos) ? x[src] : (src == pos ? T(0) : x[src - 1]);  // x0 = x~[S']
      }
      if (ctx.gtid == 0) {
        const int d = U[drop];
        B.Sbits[d >> 5] &= ~(1u << (d & 31));
        B.Sbits[j >> 5] |= 1u << (j & 31);
      }
      ctx.sync();
      ctx.mark(9);
      // S2 = S without U[drop], with j at its place: the grid context updates its tile buckets
      // by that one swap instead of rebuilding them
      ctx.swap_hint(drop < pos ? drop : drop - 1, pos < drop ? pos : pos - 1);
      cg_solve(ctx, S2, ns, x2, B.r, B.d, B.q, B.b, false, P, st);
      swap_ptr<Ctx>(S, S2);
      swap_ptr<Ctx>(x, x2);
      // (input support: set by the cg_solve above)
      rn2 = ctx.RES(x);
      continue;
    }
    // J = top-l of |z| = |x~ + eta c| off S (x~ = 0 there)
    if (l == 1) {
      int64_t j = detect_argmax<Ctx, T>(ctx, B.Sbits);
      for (int64_t w = ctx.gtid; w < nwords; w += ctx.gnthr) B.Ubits[w] = B.Sbits[w];
      ctx.sync();
      if (ctx.gtid == 0 && j >= 0) B.Ubits[j >> 5] |= 1u << (j & 31);
      ctx.sync();
    } else {
      detect_topk<Ctx, T>(ctx, l, B.Sbits, B.Ubits);
      for (int64_t w = ctx.gtid; w < nwords; w += ctx.gnthr) B.Ubits[w] |= B.Sbits[w];
      ctx.sync();
    }
    int nu = (int)compact_bits(ctx, B.Ubits, N, [&](int64_t k, int64_t j) { U[k] = (int)j; });
    remap(ctx, S, x, ns, U, xU, nu);                                  // x~ on U
    {
      const auto cv = ctx.cview();
      for (int i = ctx.gtid; i < nu; i += ctx.gnthr) xU[i] = xU[i] + eta * cv.at(U[i]);  // z on U
    }
    ctx.sync();
    const T* zc = xU;
    topk_bits(ctx, (int64_t)nu, (int64_t)K, [&](int64_t i) { return full_key(zc[i]); }, B.Pbits);
    int ns2 = (int)compact_bits(ctx, B.Pbits, nu, [&](int64_t k, int64_t pos) { S2[k] = U[pos]; });
    if (same_list<Ctx, T>(ctx, S, S2, ns)) { st.term = CS_TERM_SUPPORT_FIXED; break; }
    remap(ctx, S, x, ns, S2, x2, ns2);                                // x0 = x~[S']
    cg_solve(ctx, S2, ns2, x2, B.r, B.d, B.q, B.b, false, P, st);
    swap_ptr<Ctx>(S, S2);
    swap_ptr<Ctx>(x, x2);
    ns = ns2;
    bits_from_list<Ctx, T>(ctx, B.Sbits, nwords, S, ns);
    // (input support: set by the cg_solve above)
    rn2 = ctx.RES(x);
  }
  B.S = S; B.S2 = S2; B.x = x; B.x2 = x2;
  return ns;
}

// ------------------------------------------------------------------ CoSaMP --
// x = 0; repeat: Omega = top-2K |c| (c = A^T r, all indices), T = Omega u S, CG on T
// (warm start x, free r0 = c[T] since x lives on T), S' = top-K |x_T|, x' = x_T on S',
// r' = y - A x'.  Halt (R33): ||r'|| >= ||r|| after the first pass keeps (S, x);
// otherwise accept and stop once S' == S.
template <class Ctx, typename T>
CS_NOINL int run_cosamp(Ctx& ctx, const Params& P, Bufs<T>& B, Stats& st, double& rn2) {
  const int64_t N = ctx.N, nwords = (N + 31) >> 5;
  const int K = P.K;
  const int64_t K2 = (2 * (int64_t)K < N) ? 2 * (int64_t)K : N;
  int *S = B.S, *S2 = B.S2, *U = B.U;
  T *x = B.x, *x2 = B.x2, *xU = B.xU;
  rn2 = ctx.RES((const T*)nullptr);                              // c = A^T y, ||r||^2 = ||y||^2
  ctx.save_c0();
  for (int64_t w = ctx.gtid; w < nwords; w += ctx.gnthr) B.Sbits[w] = 0u;
  ctx.sync();
  int ns = 0;
  const int max_outer = P.max_outer > 0 ? P.max_outer : 30;
  st.term = CS_TERM_ITER_CAP;
  for (int it = 1; it <= max_outer; ++it) {
    st.outer = it;
    ctx.mark(0);
    detect_topk<Ctx, T>(ctx, K2, nullptr, B.Ubits);             // Omega = top-2K |c|
    ctx.mark(7);
    for (int64_t w = ctx.gtid; w < nwords; w += ctx.gnthr) B.Ubits[w] |= B.Sbits[w];  // T = Omega u S
    ctx.sync();
    int nu = (int)compact_bits(ctx, B.Ubits, N, [&](int64_t k, int64_t j) { U[k] = (int)j; });
    remap(ctx, S, x, ns, U, xU, nu);                             // x0 = x on S, 0 elsewhere
    {
      const auto cv = ctx.cview();
      for (int i = ctx.gtid; i < nu; i += ctx.gnthr) B.r[i] = cv.at(U[i]);   // r0 = c[T]
    }
    cg_solve(ctx, U, nu, xU, B.r, B.d, B.q, B.b, true, P, st);
    const T* xUc = xU;
    topk_bits(ctx, (int64_t)nu, (int64_t)K, [&](int64_t i) { return full_key(xUc[i]); }, B.Pbits);
    int ns2 = (int)compact_bits(ctx, B.Pbits, nu, [&](int64_t k, int64_t pos) {
      S2[k] = U[pos];
      x2[k] = xU[pos];
    });
    ctx.set_input_support(S2, ns2);
    const double rn2new = ctx.RES(x2);                           // r' and c' = A^T r'
    if (it > 1 && rn2new >= rn2) { st.term = CS_TERM_RESID_ROSE; break; }   // keep (S, x)
    const bool fixed = (ns == ns2) && same_list<Ctx, T>(ctx, S, S2, ns);
    swap_ptr<Ctx>(S, S2);
    swap_ptr<Ctx>(x, x2);
    ns = ns2;
    rn2 = rn2new;
    if (fixed) { st.term = CS_TERM_SUPPORT_FIXED; break; }
    bits_from_list<Ctx, T>(ctx, B.Sbits, nwords, S, ns);
  }
  B.S = S; B.S2 = S2; B.x = x; B.x2 = x2;
  return ns;
}

// run the selected pursuit and write (support, values, report)
template <class Ctx, typename T>
CS_DEV void run_pursuit(Ctx& ctx, const Params& P, Bufs<T> B, T* vals, int32_t* supp,
                        cs_report* rep, unsigned pre_status) {
  // every buffer as the context's memory space (shared for the CTA context: LDS/STS)
  B.S = ctx.loc(B.S); B.S2 = ctx.loc(B.S2); B.U = ctx.loc(B.U);
  B.x = ctx.loc(B.x); B.x2 = ctx.loc(B.x2); B.xU = ctx.loc(B.xU);
  B.r = ctx.loc(B.r); B.d = ctx.loc(B.d); B.q = ctx.loc(B.q); B.b = ctx.loc(B.b);
  B.Sbits = ctx.loc(B.Sbits); B.Ubits = ctx.loc(B.Ubits); B.Pbits = ctx.loc(B.Pbits);
  Stats st = {0, 0, 0, 0, pre_status, 0.0};
  double rn2 = 0;
  int ns = 0;
  if (P.alg == CS_OMP) ns = run_omp(ctx, P, B, st, rn2);
  else if (P.alg == CS_SP) ns = run_sp(ctx, P, B, st, rn2);
  else if (P.alg == CS_OMPR) ns = run_ompr(ctx, P, B, st, rn2);
  else ns = run_cosamp(ctx, P, B, st, rn2);
  for (int i = ctx.gtid; i < P.K; i += ctx.gnthr) {
    supp[i] = i < ns ? B.S[i] : -1;
    vals[i] = i < ns ? B.x[i] : T(0);
  }
  if (ctx.gtid == 0) {
    rep->outer_iters = st.outer;
    rep->cg_iters_total = st.cg_iters;
    rep->cg_solves = st.cg_solves;
    rep->applies = ctx.applies;
    rep->termination = st.term;
    rep->status = st.status;
    rep->resid_norm = sqrt(rn2);
    rep->cg_rel_resid = st.rel_max;
  }
}

}  // namespace cs
