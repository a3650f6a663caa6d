// tier_l.cuh — Tier L: one cooperative persistent grid per problem (N >= 32768).
// Used for configs 2 (SP, N = 2^16), 3 (OMPR, N = 2^20) and 5 (SP, N = 2^24), and
// for operator apply / adjoint at those sizes.  See ctx_grid.cuh for the passes.
#pragma once
#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "ctx_grid.cuh"
#include "pursuit.cuh"
#include "tier_s.cuh"

namespace cs {

constexpr int TL_THREADS = 1 << TL_LOG2NT;  // 256 (measured: 512-thread blocks at 64 registers were slower for c2/c3)

struct LGeom {
  int64_t N, L, L1, L2;
  int CT, shF, sh4;
};

// ceil(log2 v) (v >= 1); on the device a count-leading-zeros, not a loop: every block of a
// grid-tier launch evaluates the geometry at entry
CS_HD int ilog2(int64_t v) {
#ifdef __CUDA_ARCH__
  return v <= 1 ? 0 : 64 - __clzll((unsigned long long)(v - 1));
#else
  int l = 0;
  while ((int64_t(1) << l) < v) ++l;
  return l;
#endif
}

CS_HD LGeom l_geom(int64_t N) {
  LGeom g;
  g.N = N;
  g.L = N / 2;
  const int l = ilog2(g.L);
  g.L2 = int64_t(1) << ((l + 1) / 2);
  g.L1 = int64_t(1) << (l / 2);
  int64_t ct = TL_TILE / g.L1;
  ct = ct < 4 ? ct : 4;
  g.CT = (int)(ct < g.L2 ? ct : g.L2);  // small N (Tier L fallback): no more columns than L2
  g.shF = (l + 1) / 2;
  g.sh4 = (l + 1) / 2;
  return g;
}

// Workspace layout (byte offsets) — identical on host and device.
struct LLayout {
  int64_t U, Wk, Cb, c0, yT, G, yTf, in_pos, tcnt, tfill, tlist, tscr, tcnt2;
  int64_t S, S2, Ul, x, x2, xU, r, d, q, b, Sbits, Ubits, Pbits;
  int64_t ctl, bar, pd, pi, pk, ghist, ts, ctl_end;
  int64_t bytes;
  int maxgrid;
};

template <typename T>
CS_HD LLayout l_layout(int64_t N, int64_t M, int K, int ucap, bool pursuit, int maxgrid) {
  LLayout s;
  LGeom g = l_geom(N);
  const int64_t ts = sizeof(T), cs2 = 2 * sizeof(T), nw = (N + 31) / 32;
  int64_t o = 0;
  auto take = [&](int64_t bytes) { int64_t r = o; o = align_up(o + bytes, 256); return r; };
  s.U = take(N * ts);
  s.yT = take(M * ts);  // y in the transposed row order (OpMeta)
  s.Wk = take(g.L * cs2);
  s.Cb = take(N * ts);
  s.G = take(N * ts);    // Psi = DCT (R35): natural-order scratch
  s.yTf = take(N * ts);  // Psi = DCT: all-rows "y" in the transposed order
  s.c0 = pursuit ? take(N * ts) : 0;
  if (pursuit) {
    s.in_pos = take((int64_t)ucap * 8);
    s.tcnt = take((g.L2 / g.CT + 1) * 4);
    s.tcnt2 = take((g.L2 / g.CT + 1) * 4);   // the single-swap update's new starts (ctx_grid.cuh)
    s.tlist = take((int64_t)ucap * 4);
    s.tscr = take((int64_t)ucap * 4);
    s.S = take((int64_t)K * 4);
    s.S2 = take((int64_t)K * 4);
    s.Ul = take((int64_t)ucap * 4);
    s.x = take((int64_t)K * ts);
    s.x2 = take((int64_t)K * ts);
    s.xU = take((int64_t)ucap * ts);
    s.r = take((int64_t)ucap * ts);
    s.d = take((int64_t)ucap * ts);
    s.q = take((int64_t)ucap * ts);
    s.b = take((int64_t)ucap * ts);
    s.Sbits = take(nw * 4);
    s.Ubits = take(nw * 4);
    s.Pbits = take(((ucap + 31) / 32) * 4);
  } else {
    s.in_pos = s.S = s.S2 = s.Ul = s.x = s.x2 = s.xU = s.r = s.d = s.q = s.b = 0;
    s.tcnt = s.tfill = s.tlist = s.tscr = s.tcnt2 = 0;
    s.Sbits = s.Ubits = s.Pbits = 0;
  }
  // control block (zeroed before every launch)
  s.ctl = o;
  s.bar = take(256);
  s.pd = take(8 * (int64_t)maxgrid * 8);   // [4][2][maxgrid]: sum() uses [0], the CG reduction all four
  s.pi = take(2 * (int64_t)maxgrid * 8);
  s.pk = take(2 * (int64_t)maxgrid * 8);
  s.ghist = take(3 * 256 * 4);
  s.ts = take(64 * 8);  // diagnostics: %globaltimer at phase boundaries (block 0)
  s.tfill = pursuit ? take(4 * (g.L2 / g.CT) * 4) : 0;   // [2 parities][count, fill][ntiles], zero at launch
  s.ctl_end = o;
  s.bytes = o;
  s.maxgrid = maxgrid;
  return s;
}

template <typename T> CS_HD int64_t l_smem_bytes(int64_t N) {
  LGeom g = l_geom(N);
  const int64_t cs2 = 2 * sizeof(T);
  int64_t o = 0;
  auto take = [&](int64_t b) { o = align_up(o + b, 16); };
  take(16);                                               // group words (tl_group)
  take(TL_TILE * cs2);                                    // buf
  take(64 * cs2); take((g.L1 >= 64 ? g.L1 / 64 : 1) * cs2);   // tw1
  take(64 * cs2); take((g.L2 >= 64 ? g.L2 / 64 : 1) * cs2);   // tw2
  take(34 * 8); take(34 * 8); take(32 * 8); take(256 * 4); take(4 * 8);
  take(4 * ((2 * g.L2) / 32) * 4);                        // staged row metadata of pass B
  take(gtw_entries(g.L) * cs2);                           // W_L (three-level)
  take(gtw_entries(N) * cs2);                             // W_4N (exponents k < N)
  return o;
}

template <typename T> struct LArgs {
  OpMeta meta;
  LLayout lay;
  Params P;
  int64_t B;
  const T* Y;   // recover: [B][M];  apply: x [B][N];  adjoint: y [B][M]
  T* out;       // apply: y [B][M];  adjoint: x [B][N]
  T* vals;
  int32_t* supp;
  cs_report* reps;
  char* ws;
  size_t ws_bytes;
  int gblocks;      // blocks per group (the passes' work-item cap)
  int ngroups;      // groups: instances b = grp, grp + ngroups, ... run concurrently
  int64_t gstride;  // workspace bytes per group (one LLayout)
};

// The grid tier's shared-memory twiddle tables, precomputed once per operator in fp64
// (cs_operator_create -> k_l_tw_tables) and converted at block entry: computing them in every
// block (~1600 fp64 sincospi) made a fixed ~15 us of every launch.
// Layout: [W_L three-level][W_4N three-level][W_L1 lo 64 | hi n1][W_L2 lo 64 | hi n2].
struct TwOff {
  int64_t Q, t1, t2, n;
  int n1, n2;
};
CS_HD TwOff l_tw_off(int64_t N) {
  const LGeom g = l_geom(N);
  TwOff o;
  o.n1 = (int)(g.L1 >= 64 ? g.L1 / 64 : 1);
  o.n2 = (int)(g.L2 >= 64 ? g.L2 / 64 : 1);
  o.Q = gtw_entries(g.L);
  o.t1 = o.Q + gtw_entries(g.N);
  o.t2 = o.t1 + 64 + o.n1;
  o.n = o.t2 + 64 + o.n2;
  return o;
}
static __global__ void k_l_tw_tables(int64_t N, double2* out) {   // (one copy per TU: abi.cu launches it)
  const LGeom g = l_geom(N);
  const TwOff o = l_tw_off(N);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < o.n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 v;
    if (i < o.Q) v = gtw_value(i, g.L);
    else if (i < o.t1) v = gtw_value(i - o.Q, 4 * g.N);
    else if (i < o.t2) v = tw_value((int)(i - o.t1), g.L1);
    else v = tw_value((int)(i - o.t2), g.L2);
    out[i] = v;
  }
}

// the block's twiddle tables: converted from the operator's precomputed fp64 copy, or computed
// (kept out of line: the kernel bodies that inline the context set-up are sensitive to their
// instruction layout)
template <typename T>
CS_NOINL CS_DEV void tl_tables(const double2* src, const LGeom& g, C2<T>* tF, C2<T>* tQ, C2<T>* t1lo, C2<T>* t1hi,
                               C2<T>* t2lo, C2<T>* t2hi, int n1, int n2) {
  if (src) {
    const TwOff o = l_tw_off(g.N);
    for (int i = threadIdx.x; i < (int)o.n; i += blockDim.x) {
      const double2 v = src[i];
      const C2<T> w = mk<T>((T)v.x, (T)v.y);
      if (i < o.Q) tF[i] = w;
      else if (i < o.t1) tQ[i - o.Q] = w;
      else if (i < o.t1 + 64) t1lo[i - o.t1] = w;
      else if (i < o.t2) t1hi[i - o.t1 - 64] = w;
      else if (i < o.t2 + 64) t2lo[i - o.t2] = w;
      else t2hi[i - o.t2 - 64] = w;
    }
  } else {
    gtw_init<T>(tF, g.L, g.L, threadIdx.x, blockDim.x);
    gtw_init<T>(tQ, 4 * g.N, g.N, threadIdx.x, blockDim.x);
    tw_init<T>(t1lo, t1hi, g.L1, n1, threadIdx.x, blockDim.x);
    tw_init<T>(t2lo, t2hi, g.L2, n2, threadIdx.x, blockDim.x);
  }
}

template <typename T>
CS_DEV GridCtx<T> make_grid_ctx(char* smem, const LArgs<T>& a) {
  GridCtx<T> c;
  c.mid0 = make_mid<T>(a.meta.N, nullptr, nullptr, nullptr, nullptr);
  c.grp = (int)(blockIdx.x / (unsigned)a.gblocks);
  c.ngrp = a.ngroups;
  if (threadIdx.x == 0) {   // the group words: dynamic shared offset 0 (ctx_grid.cuh tl_group)
    reinterpret_cast<int*>(smem)[0] = (int)(blockIdx.x - (unsigned)c.grp * (unsigned)a.gblocks);
    reinterpret_cast<int*>(smem)[1] = a.gblocks;
  }
  __syncthreads();
  LGeom g = l_geom(a.meta.N);
  const LLayout& s = a.lay;
  c.N = a.meta.N;
  c.M = a.meta.M;
  c.L = g.L;
  c.L1 = g.L1;
  c.L2 = g.L2;
  c.CT = g.CT;
  c.log2L1 = ilog2(g.L1);
  c.log2L2 = ilog2(g.L2);
  char* ws = a.ws + (int64_t)c.grp * a.gstride;  // this group's workspace
  c.U = reinterpret_cast<T*>(ws + s.U);
  c.Wk = reinterpret_cast<C2<T>*>(ws + s.Wk);
  c.Cb = reinterpret_cast<T*>(ws + s.Cb);
  c.yT = reinterpret_cast<T*>(ws + s.yT);
  c.G = reinterpret_cast<T*>(ws + s.G);
  c.yTf = reinterpret_cast<T*>(ws + s.yTf);
  c.s1 = ilog2(g.L1);
  c.tsh = ilog2(2 * g.L2);
  c.c0 = reinterpret_cast<T*>(ws + s.c0);
  c.in_pos = reinterpret_cast<int64_t*>(ws + s.in_pos);
  c.tcnt = reinterpret_cast<int*>(ws + s.tcnt);
  c.tfill = reinterpret_cast<int*>(ws + s.tfill);
  c.tlist = reinterpret_cast<int*>(ws + s.tlist);
  c.tscr = reinterpret_cast<int*>(ws + s.tscr);
  c.tcnt2 = reinterpret_cast<int*>(ws + s.tcnt2);
  c.g.bar = reinterpret_cast<GridBar*>(ws + s.bar);
  c.g.pd = reinterpret_cast<double*>(ws + s.pd);
  c.g.pi = reinterpret_cast<int64_t*>(ws + s.pi);
  c.g.pk = reinterpret_cast<uint64_t*>(ws + s.pk);
  c.g.ghist = reinterpret_cast<unsigned*>(ws + s.ghist);
  c.g.maxgrid = s.maxgrid;
  // shared memory
  const int64_t cs2 = 2 * sizeof(T);
  int64_t o = 0;
  auto take = [&](int64_t b) { int64_t r = o; o = align_up(o + b, 16); return smem + r; };
  take(16);                                               // group words (tl_group)
  c.buf = reinterpret_cast<C2<T>*>(take(TL_TILE * cs2));
  C2<T>* t1lo = reinterpret_cast<C2<T>*>(take(64 * cs2));
  const int n1 = (int)(g.L1 >= 64 ? g.L1 / 64 : 1);
  C2<T>* t1hi = reinterpret_cast<C2<T>*>(take(n1 * cs2));
  C2<T>* t2lo = reinterpret_cast<C2<T>*>(take(64 * cs2));
  const int n2 = (int)(g.L2 >= 64 ? g.L2 / 64 : 1);
  C2<T>* t2hi = reinterpret_cast<C2<T>*>(take(n2 * cs2));
  c.sd = reinterpret_cast<double*>(take(34 * 8));
  c.si = reinterpret_cast<int64_t*>(take(34 * 8));
  c.sk = reinterpret_cast<typename GridCtx<T>::Key*>(take(32 * 8));
  c.shist = reinterpret_cast<unsigned*>(take(256 * 4));
  c.pick = reinterpret_cast<int64_t*>(take(4 * 8));
  c.msm = reinterpret_cast<uint32_t*>(take(4 * ((2 * g.L2) / 32) * 4));
  C2<T>* tF = reinterpret_cast<C2<T>*>(take(gtw_entries(g.L) * cs2));
  C2<T>* tQ = reinterpret_cast<C2<T>*>(take(gtw_entries(g.N) * cs2));
  tl_tables<T>(a.meta.tw, g, tF, tQ, t1lo, t1hi, t2lo, t2hi, n1, n2);
  c.twF.t = shp(tF);
  c.twF.mask = g.L - 1;
  c.tw4.t = shp(tQ);
  c.tw4.mask = g.N - 1;
  c.tw1.lo = t1lo; c.tw1.hi = t1hi;
  c.tw2.lo = t2lo; c.tw2.hi = t2hi;
  c.bank = 0;
  c.hpass = 0;
  c.ptime = reinterpret_cast<uint64_t*>(ws + s.ts) + 8;
  c.tprev = 0;
  c.in_supp = nullptr;
  c.in_ns = 0;
  c.applies = 0;
  c.y = nullptr;
  __syncthreads();
  return c;
}

template <typename T> CS_DEV void set_instance(GridCtx<T>& c, const OpMeta& m, int64_t b) {
  c.sign = m.sign(b);
  c.rowmask = m.tmask(b);
  c.prefix = m.tprefix(b);
  c.tperm = m.tperm(b);
  c.pm = m.pm(b);
  c.pinv = m.pinv(b);
  c.psi = m.psi;
  c.fkind = m.fkind;
  c.Mr = m.Mr;
  c.r_tmask = c.rowmask;
  c.r_tprefix = c.prefix;
  c.r_tperm = c.tperm;
  if (m.psi) {
    // the pursuit's index space is the s-domain: no sign (the all-rows instance's zero sign
    // words), no permutation; Phi's own sign / pi^-1 act in phi_in / phi_out (R35)
    c.phi_sign = c.sign;
    c.phi_pinv = c.pinv;
    c.sign = m.full_sign();
    c.pm = nullptr;
    c.pinv = nullptr;
    c.ftmask = m.full_tmask();
    c.ftprefix = m.full_tprefix();
    c.ftperm = m.full_tperm();
  }
}

// y (row order) -> yT (transposed row order of the stored mask); ends with a grid barrier
template <typename T> CS_DEV void load_yT(GridCtx<T>& c, const T* y) {
  const int32_t* tp = c.tperm;
  T* yT = c.yT;
  if (c.fkind == 1)   // partial Fourier: (Re, Im) pairs follow their frequency
    gstaged<TL_UNR, T>(2 * c.Mr, c.gtid, c.gnthr, [&](int64_t t) { return y[2 * tp[t >> 1] + (t & 1)]; },
                       [&](int64_t t, T v) { yT[t] = v; });
  else
  gstaged<TL_UNR, T>(c.M, c.gtid, c.gnthr, [&](int64_t t) { return y[tp[t]]; }, [&](int64_t t, T v) { yT[t] = v; });
  c.sync();
  c.y = c.yT;
}

// Eq.(7) randomizer: x_j lands at the Makhoul position of pi^-1(j) (R34).  Out of line so
// the plain path's register allocation is unaffected.
template <typename T>
CS_NOINL void l_scatter_perm(int64_t t0, int64_t nt, int64_t N, const T* x, const uint32_t* sg,
                             const int32_t* pv, T* U) {
  gstaged<TL_UNR, T>(N, t0, nt, [&](int64_t j) { return apply_sign<T>(sg, j, x[j]); },
                     [&](int64_t j, T v) { U[mk_pos(pv[j], N)] = v; });
}

// A x = Phi (C_N x) (R35): dense x (s-domain) into U, full DCT-II to G, then Phi's input in
// U.  Out of line so the plain apply keeps its register allocation.
template <typename T>
CS_NOINL void l_apply_psi_input(GridCtx<T>& c, const T* x) {
  const int64_t N = c.N;
  T* U = c.U;
  gstaged<TL_UNR, T>(N, c.gtid, c.gnthr, [&](int64_t j) { return x[j]; },
                     [&](int64_t j, T v) { U[mk_pos(j, N)] = v; });
  c.sync();
  c.psi_to_G(nullptr);
  c.phi_in();
  c.use_real();
}

template <typename T>
__global__ void __launch_bounds__(TL_THREADS, 2) k_l_apply(LArgs<T> a) {
  extern __shared__ __align__(16) char smem[];
  GridCtx<T> c = make_grid_ctx<T>(smem, a);
  const int64_t N = c.N;
  for (int64_t b = c.grp; b < a.B; b += c.ngrp) {
    set_instance(c, a.meta, b);
    const T* x = a.Y + b * N;
    const uint32_t* sg = c.sign;
    T* U = c.U;
    uint64_t* ts = reinterpret_cast<uint64_t*>(a.ws + a.lay.ts);
    auto stamp = [&](int i) {
      if (blockIdx.x == 0 && threadIdx.x == 0 && b == 0) {   // group 0, block 0
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        ts[i] = t;
      }
    };
    stamp(0);
    if constexpr (sizeof(T) == 4) {
      if (!c.psi && !c.pinv) {
        // the reorder rides on pass A's tile loads (GridCtx::passA_x): no U sweep
        stamp(1);
        c.passA_x(reinterpret_cast<const float*>(x));
        goto passA_done;
      }
    }
    if (c.psi) l_apply_psi_input<T>(c, x);
    else
    // four consecutive j per unit: x[j..j+3] -> U[j/2], U[j/2+1] (even j) and
    // U[N-2-j/2], U[N-1-j/2] (odd j, descending) — Makhoul order, sign applied
    if (c.pinv) l_scatter_perm<T>(c.gtid, c.gnthr, N, x, sg, c.pinv, U);
    else
    gstaged<TL_UNR, float4>(N / 4, c.gtid, c.gnthr, [&](int64_t q) {
      const int64_t j = 4 * q;
      float4 v;
      if constexpr (sizeof(T) == 4) {
        v = *reinterpret_cast<const float4*>(x + j);
      } else {
        v = make_float4(0, 0, 0, 0);
      }
      return v;
    }, [&](int64_t q, float4 v) {
      const int64_t j = 4 * q;
      if constexpr (sizeof(T) == 4) {
        const uint32_t w = sg[j >> 5] >> (j & 31);
        const float a0 = (w & 1u) ? -v.x : v.x, a1 = (w & 2u) ? -v.y : v.y;
        const float a2 = (w & 4u) ? -v.z : v.z, a3 = (w & 8u) ? -v.w : v.w;
        *reinterpret_cast<float2*>(U + j / 2) = make_float2(a0, a2);
        *reinterpret_cast<float2*>(U + N - 2 - j / 2) = make_float2(a3, a1);
      } else {
        for (int u = 0; u < 4; ++u) U[mk_pos(j + u, N)] = apply_sign<T>(sg, j + u, x[j + u]);
      }
    });
    c.sync();
    stamp(1);
    c.passA();
  passA_done:
    c.sync();
    stamp(2);
    c.template passB<MID_FWD>(false, c.yT);
    c.sync();
    stamp(3);
    T* y = a.out + b * c.M;
    const int32_t* tp = c.tperm;
    const T* yT = c.yT;
    if (c.fkind == 1)
      gstaged<TL_UNR, T>(2 * c.Mr, c.gtid, c.gnthr, [&](int64_t t) { return yT[t]; },
                         [&](int64_t t, T v) { y[2 * tp[t >> 1] + (t & 1)] = v; });
    else
    gstaged<TL_UNR, T>(c.M, c.gtid, c.gnthr, [&](int64_t t) { return yT[t]; },
                       [&](int64_t t, T v) { y[tp[t]] = v; });
    c.sync();
    stamp(4);
  }
}

template <typename T>
__global__ void __launch_bounds__(TL_THREADS, 2) k_l_adjoint(LArgs<T> a) {
  extern __shared__ __align__(16) char smem[];
  GridCtx<T> c = make_grid_ctx<T>(smem, a);
  const int64_t N = c.N;
  for (int64_t b = c.grp; b < a.B; b += c.ngrp) {
    set_instance(c, a.meta, b);
    load_yT(c, a.Y + b * c.M);
    c.RES(nullptr);
    T* x = a.out + b * N;
    const uint32_t* sg = c.sign;
    const T* Cb = c.Cb;
    const int32_t* pv = c.pinv;
    if constexpr (sizeof(T) == 4) {
      if (!pv) {
        // four consecutive j per unit, the mirror of k_l_apply's scatter: x[4q], x[4q+2] from
        // Cb[2q, 2q+1] and x[4q+3], x[4q+1] from Cb[N-2-2q, N-1-2q] (two 8-byte loads, one
        // 16-byte store), sign applied from one word
        gstaged<TL_UNR, float4>(N / 4, c.gtid, c.gnthr, [&](int64_t q) {
          const float2 lo = *reinterpret_cast<const float2*>(Cb + 2 * q);
          const float2 hi = *reinterpret_cast<const float2*>(Cb + N - 2 - 2 * q);
          return make_float4(lo.x, hi.y, lo.y, hi.x);
        }, [&](int64_t q, float4 v) {
          const int64_t j = 4 * q;
          const uint32_t w = sg[j >> 5] >> (j & 31);
          v.x = (w & 1u) ? -v.x : v.x;
          v.y = (w & 2u) ? -v.y : v.y;
          v.z = (w & 4u) ? -v.z : v.z;
          v.w = (w & 8u) ? -v.w : v.w;
          *reinterpret_cast<float4*>(x + j) = v;
        });
        c.sync();
        continue;
      }
    }
    gstaged<TL_UNR, T>(N, c.gtid, c.gnthr,
                       [&](int64_t j) { return apply_sign<T>(sg, j, Cb[GridCtx<T>::ppos(pv, j, N)]); },
                       [&](int64_t j, T v) { x[j] = v; });
    c.sync();
  }
}

template <typename T>
__global__ void __launch_bounds__(TL_THREADS, 2) k_l_recover(LArgs<T> a) {
  extern __shared__ __align__(16) char smem[];
  GridCtx<T> c = make_grid_ctx<T>(smem, a);
  const LLayout& s = a.lay;
  char* ws = a.ws + (int64_t)c.grp * a.gstride;
  for (int64_t b = c.grp; b < a.B; b += c.ngrp) {
    set_instance(c, a.meta, b);
    const T* yb = a.Y + b * c.M;
    c.applies = 0;
    double bad = 0;
    for (int64_t m = c.gtid; m < c.M; m += c.gnthr) bad += isfinite((double)yb[m]) ? 0.0 : 1.0;
    load_yT(c, yb);
    unsigned pre = c.sum(bad) > 0 ? CS_DEV_NONFINITE_Y : 0u;
    Bufs<T> B;
    B.S = reinterpret_cast<int*>(ws + s.S);
    B.S2 = reinterpret_cast<int*>(ws + s.S2);
    B.U = reinterpret_cast<int*>(ws + s.Ul);
    B.x = reinterpret_cast<T*>(ws + s.x);
    B.x2 = reinterpret_cast<T*>(ws + s.x2);
    B.xU = reinterpret_cast<T*>(ws + s.xU);
    B.r = reinterpret_cast<T*>(ws + s.r);
    B.d = reinterpret_cast<T*>(ws + s.d);
    B.q = reinterpret_cast<T*>(ws + s.q);
    B.b = reinterpret_cast<T*>(ws + s.b);
    B.Sbits = reinterpret_cast<uint32_t*>(ws + s.Sbits);
    B.Ubits = reinterpret_cast<uint32_t*>(ws + s.Ubits);
    B.Pbits = reinterpret_cast<uint32_t*>(ws + s.Pbits);
    run_pursuit<GridCtx<T>, T>(c, a.P, B, a.vals + b * a.P.K, a.supp + b * a.P.K, a.reps + b, pre);
    c.set_input_support(nullptr, 0);
    c.sync();
  }
}

// ---- distributed operator (SV §8f NEXT-4): one phase of the four-step apply / adjoint of a
// single signal split over `world` ranks (paper_1509_03979_b200/dist.py orchestrates the
// phases and the two all-to-alls).  Rank r owns the column tiles [t_lo, t_hi) of passes A / C
// and the row-pair items [i_lo, i_hi) of pass B; the phases are the single-GPU passes
// restricted to those ranges.
enum DistPhase { DP_A = 0, DP_BF = 1, DP_BA = 2, DP_C = 3, DP_P = 4, DP_YT = 5, DP_XS = 6, DP_XG = 7 };
template <typename T> struct DistArgs {
  int phase;
  int64_t t_lo, t_hi, i_lo, i_hi;
  const T* in;
  T* out;
};
// sigma applied to the four reals at Makhoul positions p0 .. p0 + 3 (p0 = 0 mod 4): natural
// indices 2 p0 + 2 i below N / 2, 2 N - 1 - 2 p0 - 2 i above; one sign word either way
CS_DEV float4 sign4(const uint32_t* sg, int64_t p0, int64_t N, float4 v) {
  uint32_t w;
  if (2 * p0 < N) {
    const int64_t j = 2 * p0;
    w = sg[j >> 5] >> (j & 31);
    w = (w & 1u) | ((w >> 1) & 2u) | ((w >> 2) & 4u) | ((w >> 3) & 8u);
  } else {
    const int64_t j = 2 * N - 1 - 2 * p0;   // = 7 mod 8: bits j, j - 2, j - 4, j - 6
    w = sg[j >> 5] >> ((j & 31) - 6);
    w = ((w >> 6) & 1u) | ((w >> 3) & 2u) | (w & 4u) | ((w << 3) & 8u);
  }
  v.x = (w & 1u) ? -v.x : v.x;
  v.y = (w & 2u) ? -v.y : v.y;
  v.z = (w & 4u) ? -v.z : v.z;
  v.w = (w & 8u) ? -v.w : v.w;
  return v;
}

template <typename T>
__global__ void __launch_bounds__(TL_THREADS, 2) k_l_dist(LArgs<T> a, DistArgs<T> d) {
  extern __shared__ __align__(16) char smem[];
  GridCtx<T> c = make_grid_ctx<T>(smem, a);
  set_instance(c, a.meta, 0);
  c.dt_lo = d.t_lo;
  c.dt_hi = d.t_hi;
  c.di_lo = d.i_lo;
  c.di_hi = d.i_hi;
  const int64_t N = c.N;
  // this rank's columns [c0, c0 + nc) of the complex [L1][L2] intermediate; its compact x
  // ("xc", nxc = 2 L1 nc reals) lists their Makhoul positions p row by row:
  // xc[q] <-> p = 2 (k1 L2 + c0) + (q - 2 nc k1), k1 = q / (2 nc)
  const int64_t l2 = c.L2, ct = c.CT, c0 = d.t_lo * ct, nc = (d.t_hi - d.t_lo) * ct;
  const int64_t nxc = 2 * c.L1 * nc;
  // (q < N <= 2^25: 32-bit quotients; a shift when the range is a power of two, as the
  // equal splits of a power-of-two tile count are)
  const uint32_t rw = (uint32_t)(2 * nc);
  const int rsh = (rw & (rw - 1)) ? -1 : __ffs(rw) - 1;
  auto pos_of = [=](int64_t q) {
    const int64_t k1 = rsh >= 0 ? (q >> rsh) : (int64_t)((uint32_t)q / rw);
    return 2 * (k1 * l2 + c0) + (q - (int64_t)rw * k1);
  };
  const uint32_t* sg = c.sign;
  if (d.phase == DP_A) {
    // xc -> U (sign applied) on this rank's columns, then its column FFTs (pass A) -> its
    // columns of Wk
    const T* x = d.in;
    T* U = c.U;
    if constexpr (sizeof(T) == 4) {
      // four reals per unit: q = 4 u is a Makhoul position p0 = 0 mod 4 of one row; the four
      // natural indices (2 p0 + 2 i, or 2 N - 1 - 2 p0 - 2 i) share one sign word
      gstaged<TL_UNR, float4>(nxc / 4, c.gtid, c.gnthr, [&](int64_t u) {
        return *reinterpret_cast<const float4*>(x + 4 * u);
      }, [&](int64_t u, float4 v) {
        const int64_t p0 = pos_of(4 * u);
        *reinterpret_cast<float4*>(U + p0) = sign4(sg, p0, N, v);
      });
    } else {
      gstaged<TL_UNR, T>(nxc, c.gtid, c.gnthr, [&](int64_t q) {
        const int64_t p = pos_of(q);
        return apply_sign<T>(sg, mk_nat(p, N), x[q]);
      }, [&](int64_t q, T v) { U[pos_of(q)] = v; });
    }
    c.sync();
    c.passA();   // (no trailing grid barrier: the kernel boundary orders the phases)
  } else if (d.phase == DP_BF) {
    // this rank's row pairs: row FFTs, DCT split, row select -> its entries of yT (the
    // transposed row order; entries of other ranks' rows are not written)
    c.template passB<MID_FWD>(false, d.out);
  } else if (d.phase == DP_BA) {
    // adjoint: this rank's entries of yT -> its row pairs of C_N^T's first half (a
    // zero-input residual pass B: X' = y / s on the selected rows) -> its rows of Wk
    c.y = d.in;
    c.template passB<MID_RES>(true, nullptr);
  } else if (d.phase == DP_C) {
    // this rank's inverse column FFTs -> Cb, then xc[q] = sigma_j Cb[p] on its columns
    c.passC();
    c.sync();
    const T* Cb = c.Cb;
    T* x = d.out;
    if constexpr (sizeof(T) == 4) {
      gstaged<TL_UNR, float4>(nxc / 4, c.gtid, c.gnthr, [&](int64_t u) {
        return *reinterpret_cast<const float4*>(Cb + pos_of(4 * u));
      }, [&](int64_t u, float4 v) {
        *reinterpret_cast<float4*>(x + 4 * u) = sign4(sg, pos_of(4 * u), N, v);
      });
    } else {
      gstaged<TL_UNR, T>(nxc, c.gtid, c.gnthr, [&](int64_t q) {
        const int64_t p = pos_of(q);
        return apply_sign<T>(sg, mk_nat(p, N), Cb[p]);
      }, [&](int64_t q, T v) { x[q] = v; });
    }
  } else if (d.phase == DP_P || d.phase == DP_YT) {
    // yT (complete) <-> y in row order
    const int32_t* tp = c.tperm;
    const T* in = d.in;
    T* out = d.out;
    if (d.phase == DP_P)
      gstaged<TL_UNR, T>(c.M, c.gtid, c.gnthr, [&](int64_t t) { return in[t]; },
                         [&](int64_t t, T v) { out[tp[t]] = v; });
    else
      gstaged<TL_UNR, T>(c.M, c.gtid, c.gnthr, [&](int64_t t) { return in[tp[t]]; },
                         [&](int64_t t, T v) { out[t] = v; });
  } else if (d.phase == DP_XS) {
    // natural x -> this rank's xc (no sign: DP_A applies it)
    const T* x = d.in;
    T* xc = d.out;
    gstaged<TL_UNR, T>(nxc, c.gtid, c.gnthr, [&](int64_t q) { return x[mk_nat(pos_of(q), N)]; },
                       [&](int64_t q, T v) { xc[q] = v; });
  } else {
    // DP_XG: the xc of every rank ([G][nxc], rank g owning columns [g nc, (g + 1) nc)) ->
    // natural x
    const T* in = d.in;
    T* x = d.out;
    const int lg2 = c.log2L2;
    gstaged<TL_UNR, T>(N, c.gtid, c.gnthr, [&](int64_t j) {
      const int64_t p = mk_pos(j, N), ci = p >> 1;
      const int64_t k1 = ci >> lg2, col = ci & (l2 - 1);
      const int64_t g = rsh >= 0 ? (col >> (rsh - 1)) : (int64_t)((uint32_t)col / (uint32_t)nc);
      return in[g * nxc + 2 * (k1 * nc + col - g * nc) + (p & 1)];
    }, [&](int64_t j, T v) { x[j] = v; });
  }
}

// the all-to-all's pack / unpack: segment k (row rows[k], columns [col0[k], col0[k] + len)
// of the four-step intermediate Wk) <-> buf[k len, (k + 1) len)
template <typename T>
__global__ void k_l_dist_copy(C2<T>* wk, int64_t l2, const int32_t* rows, const int32_t* col0, int64_t nseg,
                              int64_t len, C2<T>* buf, int to_buf) {
  const int64_t n = nseg * len;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / len, i = e - k * len;
    C2<T>* w = wk + (int64_t)rows[k] * l2 + col0[k] + i;
    if (to_buf) buf[e] = *w; else *w = buf[e];
  }
}

// Diagnostics / test hook: the grid tier's top-K (select.cuh topk_bits, the radix path used
// by detection at c2, c3, c5) on a caller's value array, over a full cooperative grid.
// The context is built for the smallest Tier L geometry (only its collectives are used).
constexpr int64_t TL_DIAG_N = 32768;
template <typename T>
__global__ void __launch_bounds__(TL_THREADS, 2) k_l_diag_topk(LArgs<T> a, const T* vals, int64_t n, int64_t K,
                                                              uint32_t* out_bits) {
  extern __shared__ __align__(16) char smem[];
  GridCtx<T> c = make_grid_ctx<T>(smem, a);
  if constexpr (sizeof(T) == 4) {
    if (n % 4 == 0) {   // the detection path's vector loader (pursuit.cuh detect_topk)
      const float4* v4 = reinterpret_cast<const float4*>(vals);
      topk_bits(c, n, K, [vals](int64_t i) { return full_key(vals[i]); }, out_bits, false, [v4](int64_t q) {
        const float4 v = v4[q];
        return make_uint4(full_key(v.x), full_key(v.y), full_key(v.z), full_key(v.w));
      });
      return;
    }
  }
  topk_bits(c, n, K, [vals](int64_t i) { return full_key(vals[i]); }, out_bits, false);
}

// Diagnostics: `iters` grid barriers (and grid sums) in a cooperative launch of the
// recovery's shape; block 0 / thread 0 records the elapsed %globaltimer.
template <typename T>
__global__ void __launch_bounds__(TL_THREADS) k_l_barrier_bench(GridBar* gb, double* pd, int iters, int with_sum,
                                                               uint64_t* out) {
  __shared__ double red[32];
  uint64_t t0 = 0, t1 = 0;
  if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    if (with_sum) {
      double v = threadIdx.x * 1e-3;
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
      __syncthreads();
      if (threadIdx.x == 0) {
        double t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        pd[(i & 1) * gridDim.x + blockIdx.x] = t;
      }
    }
    grid_barrier(gb, gridDim.x);
    if (with_sum && threadIdx.x < 32) {
      double a = 0;
      for (int c = threadIdx.x; c < (int)gridDim.x; c += 32) a += pd[(i & 1) * gridDim.x + c];
      acc += a;
    }
  }
  if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (blockIdx.x == 0 && threadIdx.x == 0) { out[0] = t1 - t0; out[1] = (uint64_t)acc; }
}

// ------------------------------------------------------------ host side ----
// the co-resident grid of a cooperative kernel.  The driver calls cost tens of microseconds
// of host time, comparable to a whole distributed phase, so the grid is cached
// per (device, kernel, size) and the kernel's dynamic shared-memory limit only ever grows (a
// later, smaller launch must not leave the limit below an earlier, larger one).
template <typename T> inline int l_maxgrid(const void* fn, int64_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<int, const void*, int64_t>, int> grids;
  static std::map<std::pair<int, const void*>, int64_t> limit;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(dev, fn, smem);
  auto it = grids.find(key);
  if (it != grids.end()) return it->second;
  int64_t& lim = limit[std::make_pair(dev, fn)];
  if (smem > lim) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    lim = smem;
  }
  int nsm = 0, occ = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, TL_THREADS, (size_t)smem);
  if (occ < 1) occ = 1;
  grids[key] = nsm * occ;
  return nsm * occ;
}

template <typename T> inline int l_grid_upper() {
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || nsm <= 0) {
    cudaGetLastError();
    nsm = 148;
  }
  return nsm * 4;  // generous upper bound for workspace sizing
}

// groups a batch of B instances can run as (an upper bound; the launch may use fewer)
template <typename T> inline int64_t l_groups_upper(int64_t N, int64_t B) {
  const LGeom g = l_geom(N);
  const int64_t work = std::max<int64_t>(g.L2 / g.CT, g.L1 / 2 + 1);
  return std::max<int64_t>(1, std::min<int64_t>(B, l_grid_upper<T>() / std::max<int64_t>(work, 1)));
}
template <typename T> inline size_t tier_l_apply_ws_bytes(int64_t N, int64_t M, int64_t B = 1) {
  return (size_t)(align_up(l_layout<T>(N, M, 0, 0, false, l_grid_upper<T>()).bytes, 256) * l_groups_upper<T>(N, B));
}
template <typename T> inline size_t tier_l_recover_ws_bytes(int64_t N, int64_t M, int K, int ucap, int64_t B = 1) {
  return (size_t)(align_up(l_layout<T>(N, M, K, ucap, true, l_grid_upper<T>()).bytes, 256) *
                  l_groups_upper<T>(N, B));
}

// Declared everywhere; defined (and explicitly instantiated) in k_l_f32.cu / k_l_f64.cu.
template <typename T>
cs_status tier_l_apply(OpMeta meta, int64_t B, const T* in, T* out, void* ws, size_t ws_bytes,
                       cudaStream_t st, bool adjoint, std::atomic<uint64_t>& launches, std::string& err);
template <typename T>
cs_status tier_l_recover(OpMeta meta, Params P, int ucap, const T* Y, int64_t B, T* vals,
                         int32_t* supp, cs_report* reps, void* ws, size_t ws_bytes,
                         cudaStream_t st, std::atomic<uint64_t>& launches, std::string& err);

template <typename T>
cs_status tier_l_dist_phase(OpMeta meta, const DistArgs<T>& d, void* ws, size_t ws_bytes, cudaStream_t st,
                            std::atomic<uint64_t>& launches, std::string& err);
template <typename T>
cs_status tier_l_dist_copy(OpMeta meta, void* ws, const int32_t* rows, const int32_t* col0, int64_t nseg,
                           int64_t len, T* buf, int to_buf, cudaStream_t st, std::atomic<uint64_t>& launches,
                           std::string& err);

template <typename T> inline size_t tier_l_diag_topk_ws_bytes() {
  return (size_t)align_up(l_layout<T>(TL_DIAG_N, TL_DIAG_N / 4, 0, 0, false, l_grid_upper<T>()).bytes, 256);
}
template <typename T>
cs_status tier_l_diag_topk(const T* vals, int64_t n, int64_t K, uint32_t* out, void* ws, size_t ws_bytes,
                           cudaStream_t st, std::atomic<uint64_t>& launches, std::string& err);

#ifdef CS_TIER_L_IMPL
template <typename T>
inline cs_status l_launch(const void* fn, LArgs<T>& a, int64_t N, cudaStream_t st,
                          std::atomic<uint64_t>& launches, std::string& err) {
  const int64_t smem = l_smem_bytes<T>(N);
  int grid = l_maxgrid<T>(fn, smem);
  if (grid > a.lay.maxgrid) grid = a.lay.maxgrid;
  // no more blocks than the passes have tiles / row pairs: at mid-size N (c2: 64 tiles,
  // 65 row pairs) extra blocks only make every grid barrier and reduction slower
  const LGeom g = l_geom(N);
  const int64_t work = std::max<int64_t>(g.L2 / g.CT, g.L1 / 2 + 1);
  const int occ_grid = grid;
  if (work < grid) grid = (int)work;
  // a batch of instances whose passes need fewer blocks than the GPU holds runs as several
  // groups side by side, each with its own workspace slice and barrier
  a.gblocks = grid;
  a.gstride = align_up(a.lay.bytes, 256);
  int64_t ng = std::min<int64_t>(a.B, occ_grid / grid);
  ng = std::min<int64_t>(ng, (int64_t)(a.ws_bytes / (size_t)a.gstride));
  a.ngroups = (int)std::max<int64_t>(1, ng);
  cudaError_t e = cudaSuccess;
  for (int q = 0; q < a.ngroups && e == cudaSuccess; ++q)
    e = cudaMemsetAsync(a.ws + q * a.gstride + a.lay.ctl, 0, (size_t)(a.lay.ctl_end - a.lay.ctl), st);
  if (e != cudaSuccess) { err = std::string("memset: ") + cudaGetErrorString(e); return CS_ERR_CUDA; }
  grid = a.gblocks * a.ngroups;
  void* args[] = {&a};
  e = cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(TL_THREADS), args, (size_t)smem, st);
  launches.fetch_add(1);
  if (e != cudaSuccess) { err = std::string("cooperative launch: ") + cudaGetErrorString(e); return CS_ERR_CUDA; }
  return CS_OK;
}

template <typename T>
cs_status tier_l_apply(OpMeta meta, int64_t B, const T* in, T* out, void* ws, size_t ws_bytes,
                              cudaStream_t st, bool adjoint, std::atomic<uint64_t>& launches,
                              std::string& err) {
  LArgs<T> a;
  a.meta = meta;
  a.lay = l_layout<T>(meta.N, meta.M, 0, 0, false, l_grid_upper<T>());
  if (!ws || ws_bytes < (size_t)a.lay.bytes) { err = "workspace too small"; return CS_ERR_WORKSPACE; }
  a.B = B;
  a.Y = in;
  a.out = out;
  a.ws = reinterpret_cast<char*>(ws);
  a.ws_bytes = ws_bytes;
  a.vals = nullptr; a.supp = nullptr; a.reps = nullptr;
  const void* fn = adjoint ? (const void*)k_l_adjoint<T> : (const void*)k_l_apply<T>;
  return l_launch<T>(fn, a, meta.N, st, launches, err);
}

template <typename T>
cs_status tier_l_recover(OpMeta meta, Params P, int ucap, const T* Y, int64_t B, T* vals,
                                int32_t* supp, cs_report* reps, void* ws, size_t ws_bytes,
                                cudaStream_t st, std::atomic<uint64_t>& launches, std::string& err) {
  LArgs<T> a;
  a.meta = meta;
  a.lay = l_layout<T>(meta.N, meta.M, P.K, ucap, true, l_grid_upper<T>());
  if (!ws || ws_bytes < (size_t)a.lay.bytes) { err = "workspace too small"; return CS_ERR_WORKSPACE; }
  a.P = P;
  a.B = B;
  a.Y = Y;
  a.out = nullptr;
  a.vals = vals;
  a.supp = supp;
  a.reps = reps;
  a.ws = reinterpret_cast<char*>(ws);
  a.ws_bytes = ws_bytes;
  return l_launch<T>((const void*)k_l_recover<T>, a, meta.N, st, launches, err);
}

template <typename T>
cs_status tier_l_diag_topk(const T* vals, int64_t n, int64_t K, uint32_t* out, void* ws, size_t ws_bytes,
                           cudaStream_t st, std::atomic<uint64_t>& launches, std::string& err) {
  LArgs<T> a;
  a.meta = OpMeta{};
  a.meta.N = TL_DIAG_N;
  a.meta.M = TL_DIAG_N / 4;
  a.lay = l_layout<T>(TL_DIAG_N, TL_DIAG_N / 4, 0, 0, false, l_grid_upper<T>());
  if (!ws || ws_bytes < (size_t)a.lay.bytes) { err = "workspace too small"; return CS_ERR_WORKSPACE; }
  a.B = 1;
  a.ws = reinterpret_cast<char*>(ws);
  a.ws_bytes = ws_bytes;
  const void* fn = (const void*)k_l_diag_topk<T>;
  const int64_t smem = l_smem_bytes<T>(TL_DIAG_N);
  int grid = l_maxgrid<T>(fn, smem);   // the whole GPU: every multi-block merge path runs
  if (grid > a.lay.maxgrid) grid = a.lay.maxgrid;
  a.gblocks = grid;
  a.ngroups = 1;
  a.gstride = align_up(a.lay.bytes, 256);
  cudaError_t e = cudaMemsetAsync(a.ws + a.lay.ctl, 0, (size_t)(a.lay.ctl_end - a.lay.ctl), st);
  if (e != cudaSuccess) { err = std::string("memset: ") + cudaGetErrorString(e); return CS_ERR_CUDA; }
  void* args[] = {&a, &vals, &n, &K, &out};
  e = cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(TL_THREADS), args, (size_t)smem, st);
  launches.fetch_add(1);
  if (e != cudaSuccess) { err = std::string("cooperative launch: ") + cudaGetErrorString(e); return CS_ERR_CUDA; }
  return CS_OK;
}

template <typename T>
cs_status tier_l_dist_phase(OpMeta meta, const DistArgs<T>& d, void* ws, size_t ws_bytes, cudaStream_t st,
                            std::atomic<uint64_t>& launches, std::string& err) {
  LArgs<T> a;
  a.meta = meta;
  a.lay = l_layout<T>(meta.N, meta.M, 0, 0, false, l_grid_upper<T>());
  if (!ws || ws_bytes < (size_t)a.lay.bytes) { err = "workspace too small"; return CS_ERR_WORKSPACE; }
  a.B = 1;
  a.Y = nullptr;
  a.out = nullptr;
  a.vals = nullptr; a.supp = nullptr; a.reps = nullptr;
  a.ws = reinterpret_cast<char*>(ws);
  a.ws_bytes = (size_t)a.lay.bytes;   // one group: the workspace of instance 0
  const void* fn = (const void*)k_l_dist<T>;
  const int64_t smem = l_smem_bytes<T>(meta.N);
  int grid = l_maxgrid<T>(fn, smem);
  if (grid > a.lay.maxgrid) grid = a.lay.maxgrid;
  a.gblocks = grid;
  a.ngroups = 1;
  a.gstride = align_up(a.lay.bytes, 256);
  cudaError_t e = cudaMemsetAsync(a.ws + a.lay.ctl, 0, (size_t)(a.lay.ctl_end - a.lay.ctl), st);
  if (e != cudaSuccess) { err = std::string("memset: ") + cudaGetErrorString(e); return CS_ERR_CUDA; }
  DistArgs<T> dd = d;
  void* args[] = {&a, &dd};
  e = cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(TL_THREADS), args, (size_t)smem, st);
  launches.fetch_add(1);
  if (e != cudaSuccess) { err = std::string("cooperative launch: ") + cudaGetErrorString(e); return CS_ERR_CUDA; }
  return CS_OK;
}
template <typename T>
cs_status tier_l_dist_copy(OpMeta meta, void* ws, const int32_t* rows, const int32_t* col0, int64_t nseg,
                           int64_t len, T* buf, int to_buf, cudaStream_t st, std::atomic<uint64_t>& launches,
                           std::string& err) {
  const LLayout lay = l_layout<T>(meta.N, meta.M, 0, 0, false, l_grid_upper<T>());
  const LGeom g = l_geom(meta.N);
  C2<T>* wk = reinterpret_cast<C2<T>*>(reinterpret_cast<char*>(ws) + lay.Wk);
  const int64_t n = nseg * len;
  if (n == 0) return CS_OK;
  const unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
  k_l_dist_copy<T><<<blocks, 256, 0, st>>>(wk, g.L2, rows, col0, nseg, len, reinterpret_cast<C2<T>*>(buf), to_buf);
  launches.fetch_add(1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { err = std::string("kernel launch: ") + cudaGetErrorString(e); return CS_ERR_CUDA; }
  return CS_OK;
}

#endif  // CS_TIER_L_IMPL

}  // namespace cs
