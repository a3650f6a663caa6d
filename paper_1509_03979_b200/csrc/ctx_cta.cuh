// ctx_cta.cuh — "CTA context": one thread block owns one recovery problem and
// keeps its whole working set in shared memory (Tier S, N <= 16384).
//
// The pursuit / CG / selection code (pursuit.cuh, select.cuh) is written once
// against a context interface:
//   gtid, gnthr, lane, gwarp, gnwarps      thread / warp ids within the context
//   sync()                                  context-wide barrier
//   sum(double) / argmax(key, idx) / excl_scan(int64)   deterministic collectives
//   hist_*                                  256-bin histogram for radix select
//   set_input_support / H / RES / c_at / c0_at / save_c0   the operator sandwich
// and instantiated for this CTA context and for the cooperative-grid context
// (ctx_grid.cuh, Tier L).  All collectives use a fixed reduction order, so a
// run is bitwise reproducible.
#pragma once
#include "cs_common.cuh"
#include "dct_mid.cuh"
#include "fft_cta.cuh"
#include "sandwich_cta.cuh"

namespace cs {

CS_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;  // lane 0 holds the total
}

template <typename T> struct CtaCtx {
  using Key = typename KeyT<T>::type;
  // The context object lives in SHARED memory (one per CTA, `__shared__` in the kernels):
  // every field is block-uniform, so the generic pursuit code reads it through a shared
  // address instead of a per-thread local-memory copy (1024 resident threads x a few hundred
  // bytes of context and call frames spilled from the small L1 to L2 and HBM).  Fields are
  // written with identical values by every thread (no thread reads a field before the barrier
  // that follows its initialisation); the only per-thread mutable state — the reduction bank —
  // is kept per warp (rbank_w, written by lane 0 after __syncwarp), and `applies` is counted by
  // thread 0 alone.
  // ids: derived from the special registers / compile-time block size on every use, never
  // stored
  struct TidV { CS_DEV operator int() const { return (int)threadIdx.x; } };
  struct LaneV { CS_DEV operator int() const { return (int)(threadIdx.x & 31); } };
  struct WarpV { CS_DEV operator int() const { return (int)(threadIdx.x >> 5); } };
  TidV gtid;
  LaneV lane;
  WarpV gwarp;
  static constexpr int gnthr = SW_NT;
  static constexpr int gnwarps = SW_NT / 32;
  int64_t N, M, L;
  int log2L;
  // shared-memory state
  C2<T>* Z;          // [L] working transform buffer; viewed as T[N] it is v (Makhoul order)
  uint32_t* sign;    // [nw]
  uint32_t* rowmask; // [nw]
  int32_t* prefix;   // [nw]
  const int32_t* pm;    // global: Eq.(7) randomizer pi (R34), or null
  const int32_t* pinv;  // global: pi^-1, or null
  TwTable<T> twL, tw4;
  double* redd;      // [32]
  int64_t* redi;     // [33]
  Key* redk;         // [32]
  unsigned* hist;    // [256]
  unsigned* h1;      // [TOPK_BINS]  first-digit histogram of the two-pass top-K
  Key* ckey;         // [TOPK_CAP]   boundary-bucket candidates
  int* cidx;         // [TOPK_CAP]
  int* ccnt;         // [1]
  static constexpr bool kTopkFast = true;
  static constexpr bool kDeferD = false;  // d update and scatter use the same thread mapping
  CS_DEV void defer_d(T*, const T*, T) {}
  int64_t* pick;     // [4]
  // global state of this problem
  const T* y;        // [M]
  T* c0;             // [N] A^T y in Makhoul order (sign not applied), global scratch
  // remembered input support of the sandwich
  const int* in_supp;
  int in_ns;
  int applies;
  // dictionary Psi = C_N (R35): A = Phi Psi.  The pursuit's index space is the s-domain
  // (no sign, no permutation: `sign` holds zeros, pm/pinv are null); Phi's sign bits and
  // pi^-1 are applied by the MID_FWDZ / MID_INVZ sandwiches (sandwich_cta.cuh).
  int fkind;                 // F: 0 = DCT-II, 1 = partial Fourier (R36)
  int psi;                   // 0: Psi = I, 1: Psi = C_N
  T* G;                      // unused on the CTA tier
  const uint32_t* phi_sign;  // global
  const int32_t* phi_pinv;   // global, or null

  CS_DEV void sync() { __syncthreads(); }
  CS_DEV void mark(int) {}  // phase accounting is a grid-context diagnostic
  // pointer into this context's working set as the compiler should see it: shared (Tier S)
  template <typename P> CS_DEV P* loc(P* p) const { return shp(p); }

  int rbank_w[SW_NT / 32];  // alternating reduction bank, one copy per warp (see above)
  CS_DEV int bank_take() {    // this warp's bank, toggled for the next reduction
    const int w = (int)(threadIdx.x >> 5);
    const int rb = rbank_w[w];
    __syncwarp();
    if ((threadIdx.x & 31) == 0) rbank_w[w] = rb ^ 1;
    return rb;
  }
  // Deterministic block sum (fixed order).  Two alternating banks of partials: the
  // next sum writes the other bank, and the one after that is ordered behind this
  // sum's readers by the next sum's barrier — so one barrier per reduction.
  CS_DEV double sum(double v) {
    v = warp_sum(v);
    double* rb = shp(redd) + 64 * bank_take();  // banks of 64 (cg_iterate_t bsum4 uses [4][16])
    if (lane == 0) rb[gwarp] = v;
    __syncthreads();
    double t = 0;
    for (int w = 0; w < gnwarps; ++w) t += rb[w];
    return t;
  }
  // two sums in one reduction (one barrier): [0..15] of the bank hold a's warp partials,
  // [16..31] b's
  CS_DEV void sum2(double& a, double& b) {
    a = warp_sum(a);
    b = warp_sum(b);
    double* rb = shp(redd) + 64 * bank_take();
    if (lane == 0) { rb[gwarp] = a; rb[16 + gwarp] = b; }
    __syncthreads();
    double ta = 0, tb = 0;
    for (int w = 0; w < gnwarps; ++w) { ta += rb[w]; tb += rb[16 + w]; }
    a = ta;
    b = tb;
  }
  // argmax of (key, idx): larger key wins, ties -> smaller idx.  Returns idx (-1 if all keys 0).
  // (argmax and excl_scan are inlined: an out-of-line call costs its register save /
  // restore through local memory, measured 0.6 % of c4)
  CS_DEV int64_t argmax(Key k, int64_t idx) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      Key k2 = __shfl_down_sync(0xffffffffu, k, o);
      int64_t i2 = __shfl_down_sync(0xffffffffu, idx, o);
      if (k2 > k || (k2 == k && i2 < idx)) { k = k2; idx = i2; }
    }
    if (lane == 0) { redk[gwarp] = k; redi[gwarp] = idx; }
    __syncthreads();
    Key bk = 0;
    int64_t bi = -1;
    for (int w = 0; w < gnwarps; ++w) {
      Key kw = redk[w];
      int64_t iw = redi[w];
      if (kw > bk || (kw == bk && kw != 0 && iw < bi)) { bk = kw; bi = iw; }
    }
    __syncthreads();
    return bk ? bi : -1;
  }
  // exclusive scan over threads in gtid order; *total receives the sum.
  CS_DEV int64_t excl_scan(int64_t v, int64_t* total) {
    int64_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) redi[gwarp] = inc;
    __syncthreads();
    int64_t base = 0, tot = 0;
    for (int w = 0; w < gnwarps; ++w) {
      int64_t x = redi[w];
      if (w < gwarp) base += x;
      tot += x;
    }
    __syncthreads();
    *total = tot;
    return base + inc - v;
  }
  // ---- 256-bin histogram for radix select ----
  CS_DEV void hist_clear() {
    for (int i = gtid; i < 256; i += gnthr) hist[i] = 0;
    __syncthreads();
  }
  CS_DEV void hist_add(unsigned digit) {
    // warp-aggregated: one shared atomic per distinct digit in the warp
    unsigned peers = __match_any_sync(__activemask(), digit);
    int leader = __ffs(peers) - 1;
    if (lane == leader) atomicAdd(&hist[digit], (unsigned)__popc(peers));
  }
  CS_DEV void hist_done() { __syncthreads(); }
  CS_DEV const unsigned* hist_smem() const { return hist; }

  // ---- correlation access: c_j = sigma_j * v[p(j)] ----
  // Z is stored swizzled (fft_cta.cuh): T-position p of v lives at zt(p).
  CS_DEV static int zt(int p) { return 2 * swz<T>(p >> 1) + (p & 1); }
  CS_DEV const T* zbuf() const { return reinterpret_cast<const T*>(Z); }
  // Makhoul position of index j: mk_pos(pi^-1(j)) under the Eq.(7) randomizer (R34)
  CS_DEV static int ppos(const int32_t* pinv, int64_t j, int64_t N) {
    return (int)mk_pos(pinv ? (int64_t)pinv[j] : j, N);
  }
  CS_DEV T c_raw(int64_t j) const { return zbuf()[zt(ppos(pinv, j, N))]; }
  // register-resident views for hot loops (the context itself lives in local memory)
  struct CV {
    const T* z;
    const uint32_t* sign;
    int N;
    const int32_t* pinv;
    CS_DEV T raw(int64_t j) const { return z[zt(ppos(pinv, j, N))]; }
    CS_DEV T at(int64_t j) const { return apply_sign<T>(sign, j, raw(j)); }
  };
  struct C0V {
    const T* c0;
    const uint32_t* sign;
    int64_t N;
    const int32_t* pinv;
    CS_DEV T at(int64_t j) const { return apply_sign<T>(sign, j, c0[ppos(pinv, j, N)]); }
  };
  CS_DEV CV cview() const { return CV{zbuf(), sign, (int)N, pinv}; }
  CS_DEV C0V c0view() const { return C0V{c0, sign, N, pinv}; }
  CS_DEV unsigned* hist_ptr() const { return hist; }
  CS_DEV T c_at(int64_t j) const { return apply_sign<T>(sign, j, c_raw(j)); }
  CS_DEV T c0_at(int64_t j) const { return apply_sign<T>(sign, j, c0[ppos(pinv, j, N)]); }
  CS_DEV void save_c0() {
    const T* cb = zbuf();
    for (int p = gtid; p < (int)N; p += gnthr) c0[p] = cb[zt(p)];
    __syncthreads();
  }

  // ---- the operator sandwich ----
  CS_DEV void swap_hint(int, int) {}   // (the grid context's single-swap bucket update)
  CS_DEV void set_input_support(const int* supp, int ns) {
    in_supp = supp;
    in_ns = ns;
  }
  // fused sandwich (sandwich_cta.cuh): scatter, forward FFT, DCT middle, inverse FFT, gather
  template <int MODE, bool ZERO> CS_DEV double sandwich(const T* vin, T* vout, T* yout) {
    if (fkind) return sw_dispatch<T, 2, 13, MODE, ZERO, 1>(log2L, y, yout, in_supp, in_ns, vin, vout);
    return sw_dispatch<T, 2, 13, MODE, ZERO, 0>(log2L, y, yout, in_supp, in_ns, vin, vout);
  }
  // CG iterations with the sandwich of one compile-time length inlined: no call
  // (and no ABI register save/restore) inside the loop.
  template <int LOG2L, bool PERM, int KIND, class S> CS_NOINL void cg_iterate_t(S& s_io) {
    // Algorithm 1 lines 14-22 for one compile-time transform length, the
    // sandwich inlined.  Only ~12 uniform scalars stay live across the sandwich (shared
    // offsets of the four vectors, rr, thr, ns, cap, j, status, bank): everything else
    // (ids, reduction slots, layout) is recomputed from threadIdx / compile-time offsets,
    // so the 64-register budget holds the FFT without spilling loop state.
    constexpr int NT = SW_NT, NWARP = SW_NT / 32;
    constexpr SFix F = s_fixed<T>(int64_t(2) << LOG2L);
    T* const xv = shp(s_io.x);
    T* const rv = shp(s_io.r);
    T* const dv = shp(s_io.d);
    T* const qv = shp(s_io.q);
    const int* const sp = shp(in_supp);
    const int n = s_io.ns;
    const double thr = s_io.thr;
    const int cap = s_io.cap;
    double rr = s_io.rr;
    int j = s_io.j;
    unsigned status = s_io.status;
    int rb = rbank_w[threadIdx.x >> 5];
    const MidCtx<T> m0 = make_mid_c<T, LOG2L + 1>(nullptr, nullptr, nullptr, nullptr);
    constexpr int64_t REDD = F.redd;
    auto bsum = [&rb](double v) {
      v = warp_sum(v);
      double* slots = reinterpret_cast<double*>(cs_smem_base + REDD) + 64 * rb;
      rb ^= 1;
      if ((threadIdx.x & 31) == 0) slots[threadIdx.x >> 5] = v;
      __syncthreads();
      double t = 0;
#pragma unroll
      for (int w = 0; w < NWARP; ++w) t += slots[w];
      return t;
    };
    // One block reduction per iteration (as the grid tier's R37): after q = H d the four
    // sums d.q, r.q, q.q and the current r.r go through ONE barrier; alpha uses the measured
    // r.r, and ||r_{j+1}||^2 = r.r - 2 alpha r.q + alpha^2 q.q (line 18 expanded, exact in
    // real arithmetic with the alpha actually applied) gives beta and the stopping test.
    // Each thread owns the same elements in the gather, the updates and the next scatter,
    // so the x, r, d updates need no barrier of their own.
    constexpr int64_t REDD4 = F.redd;
    auto bsum4 = [&rb](double& a, double& b, double& c, double& d) {
      const unsigned full = 0xffffffffu;
      const int lane = threadIdx.x & 31;
      // transpose-reduce: 4 values over 32 lanes -> lane 0: a, 8: b, 16: c, 24: d
      const bool h16 = lane & 16, h8 = lane & 8;
      double k0 = h16 ? c : a, k1 = h16 ? d : b;
      k0 += __shfl_xor_sync(full, h16 ? a : c, 16);
      k1 += __shfl_xor_sync(full, h16 ? b : d, 16);
      double k = h8 ? k1 : k0;
      k += __shfl_xor_sync(full, h8 ? k0 : k1, 8);
      k += __shfl_xor_sync(full, k, 4);
      k += __shfl_xor_sync(full, k, 2);
      k += __shfl_xor_sync(full, k, 1);
      double* slots = reinterpret_cast<double*>(cs_smem_base + REDD4) + 64 * rb;   // [4][16]
      rb ^= 1;
      if ((lane & 7) == 0) slots[(lane >> 3) * 16 + (threadIdx.x >> 5)] = k;
      __syncthreads();
      // lane l sums warps 2 (l & 7), 2 (l & 7) + 1 of value l >> 3, then 8 lanes per value
      const double* sv = slots + (lane >> 3) * 16 + 2 * (lane & 7);
      double t = sv[0] + sv[1];
      t += __shfl_xor_sync(full, t, 4);
      t += __shfl_xor_sync(full, t, 2);
      t += __shfl_xor_sync(full, t, 1);
      a = __shfl_sync(full, t, 0);
      b = __shfl_sync(full, t, 8);
      c = __shfl_sync(full, t, 16);
      d = __shfl_sync(full, t, 24);
    };
    (void)bsum;
    while (true) {
      if (!(rr > thr)) break;                                              // line 15 (R6, R7)
      if (j >= cap) { status |= CS_DEV_CG_CAP; break; }
      sw_body<T, LOG2L, MID_H, false, PERM, KIND>(nullptr, TwTable<T>{}, TwTable<T>{}, m0,
                                      SwIO<T>{sp, n, nullptr, dv, qv});    // q = H d_j
      double dq = 0, rq = 0, qq = 0, rrm = 0;
      for (int i = threadIdx.x; i < n; i += NT) {
        const double di = dv[i], qi = qv[i], ri = rv[i];
        dq += di * qi;
        rq += ri * qi;
        qq += qi * qi;
        rrm += ri * ri;
      }
      bsum4(dq, rq, qq, rrm);
      if (!(dq > 0.0)) { status |= CS_DEV_CG_BREAKDOWN; break; }
      const T alpha = (T)(rrm / dq);                                       // line 16
      const double al = (double)alpha;
      const double rr2 = rrm - 2.0 * al * rq + al * al * qq;               // ||r_{j+1}||^2
      const T beta = (T)(rr2 / rrm);                                       // line 19
      for (int i = threadIdx.x; i < n; i += NT) {
        xv[i] += alpha * dv[i];                                            // line 17
        const T ri = rv[i] - alpha * qv[i];                                // line 18
        rv[i] = ri;
        dv[i] = ri + beta * dv[i];                                         // line 20
      }
      rr = rr2;
      ++j;                                                                 // line 21
      if (!(rr2 == rr2)) { status |= CS_DEV_CG_BREAKDOWN; break; }
    }
    if (threadIdx.x == 0) applies += j - s_io.j;
    s_io.rr = rr;
    s_io.j = j;
    s_io.status = status;
    __syncwarp();
    if ((threadIdx.x & 31) == 0) rbank_w[threadIdx.x >> 5] = rb;
  }
  template <int LO, int HI, bool PERM, int KIND, class S> CS_DEV void cg_dispatch(S& s) {
    if constexpr (LO <= HI) {
      if (log2L == LO) { cg_iterate_t<LO, PERM, KIND>(s); return; }
      cg_dispatch<LO + 1, HI, PERM, KIND>(s);
    }
  }
  template <class S> CS_DEV void cg_iterate(S& s) {
    if (psi | (pinv != nullptr)) { cg_iterate_variant(s); return; }
    cg_dispatch<2, 13, false, 0>(s);  // the hot loop: sandwich inlined, no permutation lookups
  }
  // Psi = DCT: the generic CG loop around the composed sandwich; Eq.(7) permutation: the
  // hot loop instantiated with the pi^-1 lookups (kept out of line so the plain path's
  // caller stays small)
  template <class S> CS_NOINL void cg_iterate_variant(S& s) {
    if (psi) {
      cg_loop(*this, s, [this](const T* d, T* q) {
        H_psi(d, q);
        return dot_n(*this, d, q, in_ns);
      });
      return;
    }
    if (fkind) cg_dispatch<2, 13, true, 1>(s);  // partial Fourier: always position-mapped
    else cg_dispatch<2, 13, true, 0>(s);
  }
  // q = (A^T A scatter_S(d))[S] on the remembered support S (cg2)
  CS_DEV void H(const T* d, T* q) {
    if (psi) { H_psi(d, q); return; }
    sandwich<MID_H, false>(d, q, nullptr);
    if (threadIdx.x == 0) ++applies;
  }
  // c = A^T (y - A scatter_S(x)) into the buffer (b1 + cg5); returns ||y - A x||^2.
  // x == nullptr means x = 0 (c = A^T y).
  CS_DEV double RES(const T* x) {
    if (psi) return RES_psi(x);
    const double rn2 = x ? sandwich<MID_RES, false>(x, nullptr, nullptr) : sandwich<MID_RES, true>(nullptr, nullptr, nullptr);
    if (threadIdx.x == 0) ++applies;
    return sum(rn2);
  }

  // Psi = DCT fused (R35): C_N and C_N^T are the extra transforms of MID_FWDZ / MID_INVZ
  // sandwiches that write / read the buffer in place (sigma and pi of Phi applied there), so
  // H is three back-to-back sandwiches with four transforms in shared memory — no global
  // scratch, no row-mask swaps (the shared mask stays the instance's)
  template <int MODE, bool ZERO> CS_DEV double sandwich_psi(const T* vin, T* vout) {
    return sw_dispatch<T, 2, 13, MODE, ZERO, 0>(log2L, y, nullptr, in_supp, in_ns, vin, vout, phi_sign, phi_pinv);
  }
  CS_NOINL void H_psi(const T* d, T* q) {
    sandwich_psi<MID_FWDZ, false>(d, nullptr);          // Makhoul(R sigma C_N scatter_S(d))
    sandwich<MID_H, false>(nullptr, nullptr, nullptr);  // C^T P^T P C
    sandwich_psi<MID_INVZ, true>(nullptr, q);           // C_N^T (sigma R^T .), gather on S
    if (threadIdx.x == 0) ++applies;
  }
  CS_NOINL double RES_psi(const T* x) {
    double rn2;
    if (x) {
      sandwich_psi<MID_FWDZ, false>(x, nullptr);
      rn2 = sandwich<MID_RES, false>(nullptr, nullptr, nullptr);   // Phi^T (y - Phi u)
    } else {
      rn2 = sandwich<MID_RES, true>(nullptr, nullptr, nullptr);    // Phi^T y
    }
    rn2 = sum(rn2);
    sandwich_psi<MID_INVZ, true>(nullptr, nullptr);                // A^T r, s-domain
    if (threadIdx.x == 0) ++applies;
    return rn2;
  }
};

}  // namespace cs
