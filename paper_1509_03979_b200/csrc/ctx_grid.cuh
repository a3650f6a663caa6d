// ctx_grid.cuh — "grid context": one cooperative, persistent grid (all SMs) owns
// one problem (Tier L, N >= 32768).  Same interface as CtaCtx (ctx_cta.cuh), so
// pursuit.cuh / select.cuh run unchanged; the differences are
//   * sync() is a grid-wide barrier (sense counter in global memory, bounded
//     spin with a watchdog trap so a bug cannot hang the GPU);
//   * collectives reduce per-CTA partials in a fixed order (deterministic);
//   * the operator sandwich is a four-step FFT: L = N/2 = L1*L2,
//       pass A  column FFTs (length L1) of z, times W_L^{k1 m2}      -> Wk
//       pass B  row FFTs (length L2), DCT split / row-select / residual on
//               mirror row pairs (k1, L1-k1), inverse split, inverse row FFTs,
//               times W_L^{-k1 m2}                                   -> Wk
//       pass C  inverse column FFTs                                  -> Cb
//     with all vectors resident in L2 / HBM and each sub-FFT in shared memory.
#pragma once
#include "cs_common.cuh"
#include "dct_mid.cuh"
#include "fft_cta.cuh"

namespace cs {

struct alignas(8) GridBar {
  unsigned count;   // count and gen form one 64-bit arrival counter (grid_barrier)
  unsigned gen;
};

CS_DEV unsigned ld_volatile(const unsigned* p) { return *reinterpret_cast<const volatile unsigned*>(p); }

CS_DEV unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
CS_DEV void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
CS_DEV unsigned atom_add_acq_rel_gpu(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// Grid-wide barrier: block-level barrier, then thread 0 arrives with an acq_rel atomic and
// spins on the arrival counter with acquire loads (release/acquire make every block's
// writes before the barrier visible after it); bounded spin with a watchdog trap (~15 s).
// nblk = the blocks that meet at this barrier (a group of the grid, or all of it).
static CS_DEV void grid_barrier(GridBar* gb, unsigned nblk) {
  __syncthreads();
  if (threadIdx.x == 0) {
    // One monotonic 64-bit arrival counter (zeroed per launch): the block that arrives at
    // barrier e sees old in [e nblk, (e+1) nblk) and waits for the count to reach (e+1) nblk.
    // No generation word: the waiters watch the arrivals themselves, so the barrier costs
    // one atomic round trip plus the poll that sees the last arrival (no pre-load of a
    // generation, no release store by the last arriver).
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(gb);
    unsigned long long old;
    asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(cnt) : "memory");
    const unsigned long long target = old - old % nblk + nblk;
    long long t0 = clock64();
    unsigned spins = 0;
    while (true) {
      unsigned long long v;
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(cnt) : "memory");
      if (v >= target) break;
      if ((++spins & 1023u) == 0 && clock64() - t0 > (1ll << 35)) __trap();  // never hang the GPU
    }
  }
  __syncthreads();
}

// Shared-memory three-level twiddle table of W_den for exponents m < range (range a power
// of two): W^m = t2[m >> 16] * t1[(m >> 8) & 255] * t0[m & 255].  A few KB per table
// instead of a global two-level table: every lookup is three shared loads (no L2 round
// trip on the passes' critical path), one rounding more than before.
template <typename T> struct GTw {
  const C2<T>* t;     // [t0: 256][t1: 256][t2: (range >> 16) + 1]
  int64_t mask;       // range - 1 (W_L: range = den, so exponents wrap mod L)
  CS_DEV C2<T> operator()(int64_t m) const {
#ifdef CS_DIAG_NOTW
    return mk<T>(T(1), T(0));  // diagnostics build only
#endif
    m &= mask;
    return cmul<T>(cmul<T>(t[512 + (m >> 16)], t[256 + ((m >> 8) & 255)]), t[m & 255]);
  }
};
CS_HD int64_t gtw_entries(int64_t range) { return 512 + (range >> 16) + 1; }
// entry i of a three-level table of W_den (fp64)
CS_DEV double2 gtw_value(int64_t i, int64_t den) {
  const int64_t m = i < 256 ? i : (i < 512 ? (i - 256) << 8 : (i - 512) << 16);
  double s, c;
  sincospi(-2.0 * (double)(m & (den - 1)) / (double)den, &s, &c);
  return make_double2(c, s);
}
template <typename T> CS_DEV void gtw_init(C2<T>* t, int64_t den, int64_t range, int tid, int nthr) {
  const int64_t n = gtw_entries(range);
  for (int64_t i = tid; i < n; i += nthr) {
    const double2 v = gtw_value(i, den);
    t[i] = mk<T>((T)v.x, (T)v.y);
  }
}

// scratch for collectives (global, zeroed before launch)
template <typename T> struct GridScratch {
  GridBar* bar;
  double* pd;       // [2][maxgrid]
  int64_t* pi;      // [2][maxgrid]
  uint64_t* pk;     // [2][maxgrid]
  unsigned* ghist;  // [3][256]
  int maxgrid;
};

constexpr int TL_LOG2NT = 8;  // Tier L blocks: 256 threads (two per SM, 128 registers)
constexpr int TL_TILE = 8192;  // complex elements per CTA tile (32 per thread)
// Asynchronous global -> shared copies of one complex element (cp.async, LDGSTS): a
// whole tile's loads are in flight at once without staging registers.
template <typename T> CS_DEV void cp_async_c(C2<T>* sdst, const C2<T>* gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  if constexpr (sizeof(T) == 4) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gsrc) : "memory");
  } else {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gsrc) : "memory");
  }
}
CS_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
// two consecutive complex values moved with one 16-byte access (fp32)
template <typename T> struct CP { C2<T> a, b; };
template <typename T> CS_DEV CP<T> ldp(const C2<T>* p) {
  if constexpr (sizeof(T) == 4) {
    const float4 v = *reinterpret_cast<const float4*>(p);
    return CP<T>{mk<T>(v.x, v.y), mk<T>(v.z, v.w)};
  } else {
    return CP<T>{p[0], p[1]};
  }
}
template <typename T> CS_DEV void stp(C2<T>* p, const CP<T>& v) {
  if constexpr (sizeof(T) == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(v.a.x, v.a.y, v.b.x, v.b.y);
  } else {
    p[0] = v.a;
    p[1] = v.b;
  }
}

// this block's index within its group and the group size (GridCtx ids): the first two
// words of the dynamic shared memory (a header-level static __shared__ would be a different
// variable in every translation unit)
CS_DEV int tl_group(int i) { return reinterpret_cast<const int*>(cs_smem_base)[i]; }

template <typename T> struct GridCtx {
  using Key = typename KeyT<T>::type;
  // the grid may be split into groups of nblk blocks, each running its own instances with
  // its own workspace and barrier; blk = this block's index in its group.  Ids are
  // group-relative and derived on use from two shared words (tl_group, set once per block):
  // the context lives in local memory, and a stored id is a local load in every loop.
  struct BlkV { CS_DEV operator int() const { return tl_group(0); } };
  struct NblkV { CS_DEV operator int() const { return tl_group(1); } };
  struct TidV { CS_DEV operator int() const { return tl_group(0) * (int)blockDim.x + (int)threadIdx.x; } };
  struct NthrV { CS_DEV operator int() const { return tl_group(1) * (int)blockDim.x; } };
  struct LaneV { CS_DEV operator int() const { return (int)(threadIdx.x & 31); } };
  struct WarpV { CS_DEV operator int() const { return (tl_group(0) * (int)blockDim.x + (int)threadIdx.x) >> 5; } };
  struct NwarpV { CS_DEV operator int() const { return (tl_group(1) * (int)blockDim.x) >> 5; } };
  BlkV blk;
  NblkV nblk;
  int grp, ngrp;
  TidV gtid;
  NthrV gnthr;
  LaneV lane;
  WarpV gwarp;
  NwarpV gnwarps;
  int64_t N, M, L, L1, L2;
  int CT, log2L1, log2L2;
  // global per-problem state
  const uint32_t* sign;
  const uint32_t* rowmask;
  const int32_t* prefix;
  const T* y;        // measurements in the transposed row order (= yT during a recovery)
  const int32_t* tperm;  // [M] y index of the t-th selected row in the transposed order
  const int32_t* pm;     // Eq.(7) randomizer pi (R34), or null
  const int32_t* pinv;   // pi^-1, or null
  int fkind;             // F: 0 = DCT-II, 1 = partial Fourier (R36: y holds (Re, Im) pairs)
  int64_t Mr;            // metadata rows (frequencies for the DFT)
  // dictionary Psi = C_N (R35): the all-rows instance and the real one, Phi's sign and pi^-1
  int psi;
  T* G;                  // [N] natural-order scratch
  T* yTf;                // [N] all-rows "y" (transposed order)
  const uint32_t *ftmask, *r_tmask;
  const int32_t *ftprefix, *ftperm, *r_tprefix, *r_tperm;
  const uint32_t* phi_sign;
  const int32_t* phi_pinv;
  T* yT;             // [M] workspace
  int s1, tsh;       // transposed mask position: t = (k mod 2^s1) << tsh | k >> s1
  T* c0;        // [N] Makhoul order
  T* U;         // [N] dense input (Makhoul order, sign applied)
  C2<T>* Wk;    // [L] four-step intermediate
  T* Cb;        // [N] output (Makhoul order)
  int64_t* in_pos;  // [cap] positions of the remembered input support
  // Distributed operator (NEXT-4, tier_l.cuh k_l_dist): the dense passes A / C work on the
  // column tiles [dt_lo, dt_hi) and pass B on the row-pair items [di_lo, di_hi) of this
  // rank; hi < 0 means the whole range (every single-GPU call)
  int64_t dt_lo = 0, dt_hi = -1, di_lo = 0, di_hi = -1;
  // the support bucketed by pass-A / pass-C column tile (CSR): tile t owns the entries
  // tlist[tstart[t] .. tstart[t+1]) (indices into the support list)
  int* tcnt;        // [ntiles + 1] exclusive starts of the tiles' entries in tlist
  int* tfill;       // [2][2][ntiles] counts and fill cursors of set_input_support (two parities)
  int sis_par = 0;  // parity of the next set_input_support
  // Pass A's entry cache (set_input_support): when every block owns at most one column tile
  // (c2, c3), block blk's tile entries (shared slot | sign bit, support index) stay in the
  // unused tail of the tile buffer until the support changes, so pass A's scatter is one
  // round trip (the values) instead of four dependent ones (bucket start, list, position,
  // sign word).  acn = cached entries, -1 = no cache.
  int acn = -1;
  // the N-dependent middle constants (fp64 sqrt / division), computed once per launch
  // (make_grid_ctx) instead of in every pass B call
  MidCtx<T> mid0;
  int* tlist;       // [cap]
  int* tscr;        // [cap] the atomically filled (unordered) buckets before ranking
  int* tcnt2;       // [ntiles + 1] the single-swap update's new starts (swapped with tcnt)
  // OMPR(1) swap hint (run_ompr -> set_input_support): the next support is the remembered
  // one with old entry sw_dpos removed and a new index inserted at new position sw_ipos
  int sw_dpos = -1, sw_ipos = -1;
  CS_DEV void swap_hint(int dpos, int ipos) { sw_dpos = dpos; sw_ipos = ipos; }
  GTw<T> twF;   // W_L
  GTw<T> tw4;   // W_4N
  // shared memory
  C2<T>* buf;   // [8192] sub-FFT tile
  TwTable<T> tw1, tw2;  // W_L1, W_L2
  double* sd;   // [33]
  int64_t* si;  // [34]
  Key* sk;      // [32]
  unsigned* shist;  // [256]
  uint32_t* msm;    // [4][2 L2 / 32] staged pass-B row metadata (mask x2, prefix x2)
  int64_t* pick;    // [4]
  GridScratch<T> g;
  int bank, hpass;
  // diagnostics: block 0 / thread 0 accumulates %globaltimer time per phase into
  // ptime[phase] (workspace control block, zeroed per launch); tprev = last mark
  uint64_t* ptime;
  uint64_t tprev;
  CS_DEV void mark(int phase) {
    if (blk == 0 && threadIdx.x == 0) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (tprev) ptime[phase] += t - tprev;
      tprev = t;
    }
  }
  const int* in_supp;
  int in_ns;
  int applies;
  // CG vector updates deferred into the next H's pass A (cg_iterate / cg_loop, kDeferD):
  // pass A reads d[i] for the support entries of its tile, i.e. from other blocks than the
  // one that would update it, with no grid barrier between the update and the read — so the
  // entry's single reader applies  x += alpha d, r -= alpha q (lines 17-18; dfr_x set) and
  // d = r + beta d (line 20), and writes them back.
  T* dfr_d = nullptr;
  T* dfr_r = nullptr;
  T* dfr_x = nullptr;
  const T* dfr_q = nullptr;
  T dfr_alpha = T(0), dfr_beta = T(0);
  CS_DEV void defer_d(T* d, T* r, T beta) { dfr_d = d; dfr_r = r; dfr_x = nullptr; dfr_beta = beta; }
  double p_rq, p_qq, p_rr;   // pass C partials r.q, q.q, r.r of H_dot4 (this block)

  CS_DEV void sync() { grid_barrier(g.bar, (unsigned)nblk); }
  static constexpr bool kTopkFast = false;
  static constexpr bool kDeferD = true;
  template <typename P> CS_DEV P* loc(P* p) const { return p; }  // global (Tier L)

  // block-level deterministic sum; result valid in thread 0
  CS_DEV double block_sum(double v) {
    v = warp_sum_g(v);
    if (lane == 0) sd[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0;
    if (threadIdx.x == 0)
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sd[w];
    __syncthreads();
    return t;
  }
  // Lane `lane`'s share of the per-block partials P[c], c = lane, lane + 32, ... < n, summed
  // in that order with all of the lane's loads in flight first (a strided loop would wait one
  // L2 round trip per term: ~9 at 257 blocks); adding the padding zeros leaves every partial
  // sum bitwise unchanged.
  template <typename V> CS_DEV static V lane_sum(const V* P, int n, int ln) {
    constexpr int U = 10;   // 320 >= blocks of the grid tier (two per SM)
    V a = V(0);
    for (int c0 = 0; c0 < n; c0 += 32 * U) {
      V v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + ln + 32 * u;
        v[u] = c < n ? P[c] : V(0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) a += v[u];
    }
    return a;
  }
  CS_DEV static double warp_sum_g(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
  }
  CS_DEV double sum(double v) {
    double t = block_sum(v);
    double* P = g.pd + bank * g.maxgrid;
    if (threadIdx.x == 0) P[blk] = t;
    sync();
    if (threadIdx.x < 32) {
      double a = 0;
      a = lane_sum<double>(P, (int)nblk, (int)threadIdx.x);
      a = warp_sum_g(a);
      if (threadIdx.x == 0) sd[32] = a;
    }
    __syncthreads();
    double tot = sd[32];
    __syncthreads();
    bank ^= 1;
    return tot;
  }
  // two sums in one grid reduction (partials in pd slots 0 and 1); results in a, b
  CS_DEV void sum2(double& a, double& b) {
    constexpr int NW = (1 << TL_LOG2NT) / 32;
    double t0 = warp_sum_g(a), t1 = warp_sum_g(b);
    if (lane == 0) {
      sd[threadIdx.x >> 5] = t0;
      sd[NW + (threadIdx.x >> 5)] = t1;
    }
    __syncthreads();
    if (threadIdx.x < 2) {
      double v = 0;
      for (int w = 0; w < NW; ++w) v += sd[threadIdx.x * NW + w];
      g.pd[((int)threadIdx.x * 2 + bank) * g.maxgrid + blk] = v;
    }
    sync();
    if (threadIdx.x < 64) {
      const int k = (int)threadIdx.x >> 5;
      const double* P = g.pd + (k * 2 + bank) * g.maxgrid;
      double v = 0;
      v = lane_sum<double>(P, (int)nblk, (int)lane);
      v = warp_sum_g(v);
      if (lane == 0) sd[k] = v;
    }
    __syncthreads();
    a = sd[0];
    b = sd[1];
    __syncthreads();
    bank ^= 1;
  }
  CS_DEV int64_t argmax(Key k, int64_t idx) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      Key k2 = __shfl_down_sync(0xffffffffu, k, o);
      int64_t i2 = __shfl_down_sync(0xffffffffu, idx, o);
      if (k2 > k || (k2 == k && i2 < idx)) { k = k2; idx = i2; }
    }
    if (lane == 0) { sk[threadIdx.x >> 5] = k; si[threadIdx.x >> 5] = idx; }
    __syncthreads();
    uint64_t* PK = g.pk + bank * g.maxgrid;
    int64_t* PI = g.pi + bank * g.maxgrid;
    if (threadIdx.x == 0) {
      Key bk = 0;
      int64_t bi = -1;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
        if (sk[w] > bk || (sk[w] == bk && bk != 0 && si[w] < bi)) { bk = sk[w]; bi = si[w]; }
      PK[blk] = (uint64_t)bk;
      PI[blk] = bi;
    }
    sync();
    if (threadIdx.x < 32) {  // warp 0 merges the per-block partials (lanes stride, then shuffle)
      Key bk = 0;
      int64_t bi = -1;
      for (int c0 = 0; c0 < (int)nblk; c0 += 320) {   // all loads in flight first (lane_sum)
        Key kv[10];
        int64_t iv[10];
#pragma unroll
        for (int u = 0; u < 10; ++u) {
          const int c = c0 + (int)threadIdx.x + 32 * u;
          kv[u] = c < (int)nblk ? (Key)PK[c] : Key(0);
          iv[u] = c < (int)nblk ? PI[c] : -1;
        }
#pragma unroll
        for (int u = 0; u < 10; ++u) {
          const Key kc = kv[u];
          const int64_t ic = iv[u];
          if (kc > bk || (kc == bk && kc != 0 && ic < bi)) { bk = kc; bi = ic; }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const Key k2 = __shfl_down_sync(0xffffffffu, bk, o);
        const int64_t i2 = __shfl_down_sync(0xffffffffu, bi, o);
        if (k2 > bk || (k2 == bk && k2 != 0 && i2 < bi)) { bk = k2; bi = i2; }
      }
      if (threadIdx.x == 0) si[33] = bk ? bi : -1;
    }
    __syncthreads();
    int64_t r = si[33];
    __syncthreads();
    bank ^= 1;
    return r;
  }
  CS_DEV int64_t excl_scan(int64_t v, int64_t* total) {
    int64_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane == 31) si[w] = inc;
    __syncthreads();
    int64_t base = 0, ctot = 0;
    for (int k = 0; k < nw; ++k) {
      if (k < w) base += si[k];
      ctot += si[k];
    }
    int64_t* P = g.pi + bank * g.maxgrid;
    if (threadIdx.x == 0) P[blk] = ctot;
    sync();
    if (threadIdx.x < 32) {  // warp 0: lanes stride over the per-block partials, then shuffle
      int64_t before = 0, all = 0;
      for (int c0 = 0; c0 < (int)nblk; c0 += 320) {   // all loads in flight first (lane_sum)
        int64_t vv[10];
#pragma unroll
        for (int u = 0; u < 10; ++u) {
          const int c = c0 + (int)threadIdx.x + 32 * u;
          vv[u] = c < (int)nblk ? P[c] : 0;
        }
#pragma unroll
        for (int u = 0; u < 10; ++u) {
          const int c = c0 + (int)threadIdx.x + 32 * u;
          if (c < (int)blk) before += vv[u];
          all += vv[u];
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        before += __shfl_down_sync(0xffffffffu, before, o);
        all += __shfl_down_sync(0xffffffffu, all, o);
      }
      if (threadIdx.x == 0) {
        si[32] = before;
        si[33] = all;
      }
    }
    __syncthreads();
    int64_t before = si[32];
    *total = si[33];
    __syncthreads();
    bank ^= 1;
    return before + base + inc - v;
  }
  // histogram: shared per-CTA counts, merged into a rotating global bank
  CS_DEV void hist_clear() {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) shist[i] = 0;
    if (blk == 0) {
      unsigned* nb = g.ghist + ((hpass + 1) % 3) * 256;
      for (int i = threadIdx.x; i < 256; i += blockDim.x) nb[i] = 0;
    }
    __syncthreads();
  }
  CS_DEV void hist_add(unsigned digit) {
    unsigned peers = __match_any_sync(__activemask(), digit);
    int leader = __ffs(peers) - 1;
    if (lane == leader) atomicAdd(&shist[digit], (unsigned)__popc(peers));
  }
  CS_DEV void hist_done() {
    __syncthreads();
    unsigned* gb = g.ghist + (hpass % 3) * 256;
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
      if (shist[i]) atomicAdd(&gb[i], shist[i]);
    sync();
    for (int i = threadIdx.x; i < 256; i += blockDim.x) shist[i] = gb[i];
    __syncthreads();
    ++hpass;
  }
  CS_DEV const unsigned* hist_smem() const { return shist; }

  // ---- correlation access ----
  // Makhoul position of index j: mk_pos(pi^-1(j)) under the Eq.(7) randomizer (R34)
  CS_DEV static int64_t ppos(const int32_t* pinv, int64_t j, int64_t N) {
    return mk_pos(pinv ? (int64_t)pinv[j] : j, N);
  }
  CS_DEV T c_raw(int64_t j) const { return Cb[ppos(pinv, j, N)]; }
  struct CV {
    const T* z;
    const uint32_t* sign;
    int64_t N;
    const int32_t* pinv;
    CS_DEV T raw(int64_t j) const { return z[ppos(pinv, j, N)]; }
    CS_DEV T at(int64_t j) const { return apply_sign<T>(sign, j, raw(j)); }
  };
  struct C0V {
    const T* c0;
    const uint32_t* sign;
    int64_t N;
    const int32_t* pinv;
    CS_DEV T at(int64_t j) const { return apply_sign<T>(sign, j, c0[ppos(pinv, j, N)]); }
  };
  CS_DEV CV cview() const { return CV{Cb, sign, N, pinv}; }
  CS_DEV C0V c0view() const { return C0V{c0, sign, N, pinv}; }
  CS_DEV unsigned* hist_ptr() const { return shist; }
  CS_DEV T c_at(int64_t j) const { return apply_sign<T>(sign, j, Cb[ppos(pinv, j, N)]); }
  CS_DEV T c0_at(int64_t j) const { return apply_sign<T>(sign, j, c0[ppos(pinv, j, N)]); }
  CS_DEV void save_c0() {
    for (int64_t p = gtid; p < N; p += gnthr) c0[p] = Cb[p];
    sync();
  }

  // ---- sandwich ----
  CS_DEV int ntiles() const { return (int)(L2 / CT); }
  // column tile of Makhoul position p: complex index p/2 = m1 L2 + m2, tile m2 / CT
  CS_DEV int tile_of(int64_t p) const { return (int)(((p >> 1) & (L2 - 1)) / CT); }
  // Bucket the input support by pass-A/C column tile (CSR: tcnt starts, tlist entries) with
  // three grid barriers: counts by atomics into this call's zeroed arrays; every block scans the
  // counts itself into shared memory (block 0 also publishes them as tcnt) and fills tlist
  // with its own copy; the other parity's arrays are zeroed for the next call.
  CS_DEV void set_input_support(const int* supp, int ns) {
    if (sw_dpos >= 0 && in_supp != nullptr && ns == in_ns) { set_input_support_swap(supp, ns); return; }
    sw_dpos = sw_ipos = -1;
    const int nt = ntiles();
    int* cnt = tfill + sis_par * 2 * nt;
    int* fil = cnt + nt;
    int* ncnt = tfill + (sis_par ^ 1) * 2 * nt;
    for (int i = gtid; i < ns; i += gnthr) {
      const int64_t p = ppos(pinv, supp[i], N);
      in_pos[i] = p;
      atomicAdd(&cnt[tile_of(p)], 1);
    }
    sync();
    int* offs = reinterpret_cast<int*>(shp(buf));   // [nt + 1], the tile buffer is free here
    {
      const int per = (nt + (int)blockDim.x - 1) / (int)blockDim.x;
      const int a = (int)threadIdx.x * per, e = min(nt, a + per);
      int loc = 0;
      for (int t = a; t < e; ++t) loc += __ldcg(&cnt[t]);
      int inc = loc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += u;
      }
      if (lane == 31) si[threadIdx.x >> 5] = inc;
      __syncthreads();
      int base = inc - loc;
      for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) base += (int)si[w];
      for (int t = a; t < e; ++t) {
        offs[t] = base;
        base += __ldcg(&cnt[t]);
      }
      if (threadIdx.x == blockDim.x - 1) offs[nt] = base;
      __syncthreads();
    }
    if (blk == 0)
      for (int t = threadIdx.x; t <= nt; t += blockDim.x) tcnt[t] = offs[t];
    for (int i = gtid; i < ns; i += gnthr) {
      const int t = tile_of(in_pos[i]);
      tscr[offs[t] + atomicAdd(&fil[t], 1)] = i;
    }
    for (int t = gtid; t < 2 * nt; t += gnthr) ncnt[t] = 0;
    sync();
    // deterministic order inside every bucket (ascending support index): the atomic fill
    // order varies run to run, and pass C's per-thread dot-product partials follow the list
    // order, so ranking the entries makes the fp64 sums (alpha, beta, the stop test) and
    // hence every result bitwise reproducible
    // (one block per bucket: the bucket is staged in shared memory past the offsets with one
    // L2 round trip, and each entry's rank is the count of smaller entries — broadcast reads;
    // a bucket too large for that quadratic count falls back to one warp per entry, the
    // lanes reading the bucket in parallel and a ballot counting the entries below i)
    {
      int* sbk = offs + nt + 1;
      constexpr int QCAP = 2048;
      for (int t = blk; t < nt; t += nblk) {
        const int a = offs[t], e = offs[t + 1], n = e - a;
        if (n <= QCAP) {
          for (int q = threadIdx.x; q < n; q += blockDim.x) sbk[q] = __ldcg(&tscr[a + q]);
          __syncthreads();
          for (int q = threadIdx.x; q < n; q += blockDim.x) {
            const int v = sbk[q];
            int rank = 0;
            for (int u = 0; u < n; ++u) rank += sbk[u] < v ? 1 : 0;
            tlist[a + rank] = v;
          }
          __syncthreads();
        } else {
          for (int q0 = a + (int)(threadIdx.x >> 5); q0 < e; q0 += (int)(blockDim.x >> 5)) {
            const int i = __ldcg(&tscr[q0]);
            int rank = 0;
            for (int r0 = a; r0 < e; r0 += 32) {
              const int q = r0 + (int)lane;
              rank += __popc(__ballot_sync(0xffffffffu, q < e && __ldcg(&tscr[q]) < i));
            }
            if (lane == 0) tlist[a + rank] = i;
          }
        }
      }
    }
    sis_par ^= 1;
    in_supp = supp;
    in_ns = ns;
    sync();
    build_acache(supp);
  }
  // The buckets of a support that differs from the remembered one by one swap (OMPR(1)):
  // old entry dpos leaves, the new index supp[ipos] enters.  Every other entry keeps its
  // position p, hence its tile, and its index moves monotonically (i -> i - [i > dpos], then
  // +1 if that is >= ipos), so each bucket is the old bucket mapped in order, minus the dropped
  // entry (tile A), plus the new one (tile Bt) at its rank — exactly what the full rebuild's
  // ranking produces (same tcnt, tlist, in_pos; bitwise the same passes), for one grid barrier
  // instead of three plus the ranking pass.
  CS_DEV void set_input_support_swap(const int* supp, int ns) {
    const int nt = ntiles();
    const int dpos = sw_dpos, ipos = sw_ipos;
    sw_dpos = sw_ipos = -1;
    const int A = tile_of(ppos(pinv, in_supp[dpos], N));
    const int Bt = tile_of(ppos(pinv, supp[ipos], N));
    auto newstart = [&](int t) { return tcnt[t] - (t > A ? 1 : 0) + (t > Bt ? 1 : 0); };
    if (blk == 0)
      for (int t = threadIdx.x; t <= nt; t += blockDim.x) tcnt2[t] = newstart(t);
    for (int i = gtid; i < ns; i += gnthr) in_pos[i] = ppos(pinv, supp[i], N);
    int* cntj = reinterpret_cast<int*>(si);   // block scratch: rank of the new entry
    for (int t = blk; t < nt; t += nblk) {
      const int a = tcnt[t], e = tcnt[t + 1], a2 = newstart(t);
      if (t == Bt) {
        if (threadIdx.x == 0) *cntj = 0;
        __syncthreads();
      }
      int below = 0;
      for (int k = threadIdx.x; k < e - a; k += blockDim.x) {
        const int oi = tlist[a + k];
        if (t == A && oi == dpos) continue;
        int ni = oi - (oi > dpos ? 1 : 0);
        ni += (ni >= ipos) ? 1 : 0;
        const int rk = k - ((t == A && oi > dpos) ? 1 : 0) + ((t == Bt && ni > ipos) ? 1 : 0);
        tscr[a2 + rk] = ni;
        below += (t == Bt && ni < ipos) ? 1 : 0;
      }
      if (t == Bt) {
        if (below) atomicAdd(cntj, below);
        __syncthreads();
        if (threadIdx.x == 0) tscr[a2 + *cntj] = ipos;
        __syncthreads();
      }
    }
    in_supp = supp;
    in_ns = ns;
    sync();
    int* tmp = tlist; tlist = tscr; tscr = tmp;
    tmp = tcnt; tcnt = tcnt2; tcnt2 = tmp;
    build_acache(supp);
  }
  // the cache lives in the tile buffer past every pass's footprint (tile, row pair, the bucket
  // scan's offsets): TL_TILE complex slots, one entry (two ints) per slot
  CS_DEV int64_t acache_off() const {
    const int64_t tileA = L1 * CT, rowB = 2 * L2, offs = (L2 / CT + 2) / 2 + 1;
    return tileA > rowB ? (tileA > offs ? tileA : offs) : (rowB > offs ? rowB : offs);
  }
  CS_DEV void build_acache(const int* supp) {
    acn = -1;
    const int nt = ntiles();
    const int64_t off = acache_off();
    if (psi || nt > (int)nblk || off >= TL_TILE) return;
    if (blk < nt) {
      const int a = tcnt[blk], e = tcnt[blk + 1];
      if ((int64_t)(e - a) > TL_TILE - off) return;   // (block-uniform)
      int* ac = reinterpret_cast<int*>(shp(buf) + off);
      const int lct = (CT == 4) ? 2 : 1;
      const int64_t l2 = L2, c0i = (int64_t)blk * CT;
      for (int q = threadIdx.x; q < e - a; q += blockDim.x) {
        const int i = tlist[a + q];
        const int64_t p = in_pos[i], c = p >> 1;
        const int el = (int)(((c >> log2L2) << lct) | ((c & (l2 - 1)) - c0i));
        ac[2 * q] = (2 * swz<T>(el) + (int)(p & 1)) | (bit_test(sign, supp[i]) ? (int)0x80000000 : 0);
        ac[2 * q + 1] = i;
      }
      acn = e - a;
    } else {
      acn = 0;
    }
    __syncthreads();
  }
  CS_DEV void scatter(const T* vals) {
    const int* sp = in_supp;
    const int64_t* ip = in_pos;
    const uint32_t* sg = sign;
    T* u = U;
    const int ns = in_ns, t0 = gtid, st = gnthr;
    for (int i = t0; i < ns; i += st) u[ip[i]] = apply_sign<T>(sg, sp[i], vals[i]);
    sync();
  }
  // sub-FFTs of the four-step (256-thread blocks, compile-time lengths 2^7..2^12)
  template <bool INV> CS_DEV void col_fft() {
#ifdef CS_DIAG_NOFFT
    return;  // diagnostics build only: memory-phase timing without the sub-FFTs
#endif
    if (CT == 4) fft_cta_dispatch<T, 2, TL_LOG2NT, 1, 12, INV>(buf, log2L1, tw1);
    else fft_cta_dispatch<T, 1, TL_LOG2NT, 1, 12, INV>(buf, log2L1, tw1);
  }
  template <bool INV> CS_DEV void row_fft(int B) {
#ifdef CS_DIAG_NOFFT
    return;
#endif
    if (B == 2) fft_cta_dispatch<T, 1, TL_LOG2NT, 1, 12, INV>(buf, log2L2, tw2);
    else fft_cta_dispatch<T, 0, TL_LOG2NT, 1, 12, INV>(buf, log2L2, tw2);
  }
  // pass A: columns of z = U viewed as complex [L1][L2]
  CS_NOINL void passA() {
    const C2<T>* Uc = reinterpret_cast<const C2<T>*>(U);
    const int ct = CT, lct = (ct == 4) ? 2 : 1;
    const int64_t l2 = L2, ntiles = L2 / ct;
    const int tile = (int)(L1 * ct);
    C2<T>* sb = shp(buf);
    C2<T>* wk = Wk;
    const GTw<T> tf = twF;
    const int64_t tlo = dt_hi < 0 ? 0 : dt_lo, thi = dt_hi < 0 ? ntiles : dt_hi;
    for (int64_t t = tlo + blk; t < thi; t += nblk) {
      const int64_t c0i = t * ct;
      // element e = (m1, cc): the whole tile in flight as cp.async
      for (int e = threadIdx.x; e < tile; e += blockDim.x)
        cp_async_c<T>(&sb[swz<T>(e)], &Uc[(int64_t)(e >> lct) * l2 + c0i + (e & (ct - 1))]);
      cp_async_wait_all();
      __syncthreads();
      col_fft<false>();
      // thread's pairs p = tid + u NT: fixed columns (m2, m2 + 1), rows k1 = k10 + u dk.
      // Twiddles W_L^{k1 m2}: a table lookup every TW_ANCHOR steps, a multiplication by
      // W_L^{dk m2} in between (<= TW_ANCHOR - 1 roundings of drift)
      {
        const int NT = blockDim.x, np = tile / 2;
        const int e0 = 2 * (int)threadIdx.x;
        const int64_t k10 = e0 >> lct, dk = (2 * NT) >> lct;
        const int64_t m2 = c0i + (e0 & (ct - 1));
        const C2<T> sa = tf(dk * m2), sbb = tf(dk * (m2 + 1));
        for (int u0 = 0, p0 = threadIdx.x; p0 < np; u0 += TW_ANCHOR, p0 += TW_ANCHOR * NT) {
          const int64_t k1g = k10 + u0 * dk;
          C2<T> wa = tf(k1g * m2), wb = tf(k1g * (m2 + 1));
#pragma unroll
          for (int s2 = 0; s2 < TW_ANCHOR; ++s2) {
            const int p = p0 + s2 * NT;
            if (p >= np) break;
            const int64_t k1 = k1g + s2 * dk;
            if (s2) {
              wa = cmul<T>(wa, sa);
              wb = cmul<T>(wb, sbb);
            }
            const int e = 2 * p;
            stp<T>(&wk[k1 * l2 + m2], CP<T>{cmul<T>(sb[swz<T>(e)], wa), cmul<T>(sb[swz<T>(e + 1)], wb)});
          }
        }
      }
      __syncthreads();
    }
  }
  // pass A of the dense forward apply straight from x (fp32, no Eq.(7) permutation): each
  // tile element is read from x with the Makhoul reorder and the sign folded into the load
  // (slot s < L/2: (x[4s], x[4s+2]); slot s >= L/2, q = L-1-s: (x[4q+3], x[4q+1]); DESIGN.md
  // §5.1), so the reorder sweep of the whole vector (read N + write N reals, one grid phase)
  // disappears.  Rows m1 < L1/2 of tile t and rows >= L1/2 of the mirror tile L2/CT-1-t read
  // the same 16-byte units of x, so consecutive work units are mirror tiles (same round,
  // the second read hits L2).  Then the column FFT and the W_L^{k1 m2} store as passA.
  CS_NOINL void passA_x(const float* __restrict__ x) {
    const int ct = CT, lct = (ct == 4) ? 2 : 1;
    const int64_t l2 = L2, ntl = L2 / ct, hl = (L1 * L2) / 2;
    const int tile = (int)(L1 * ct);
    C2<T>* sb = shp(buf);
    C2<T>* wk = Wk;
    const GTw<T> tf = twF;
    const uint32_t* sg = sign;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    for (int64_t v = blk; v < ntl; v += nblk) {
      const int64_t t = (v & 1) ? ntl - 1 - (v >> 1) : (v >> 1);
      const int64_t c0i = t * ct;
      staged<TL_UNR, float4>(tile, [&](int e) {
        const int64_t s = (int64_t)(e >> lct) * l2 + c0i + (e & (ct - 1));
        const int64_t q = s < hl ? s : 2 * hl - 1 - s;
        return x4[q];
      }, [&](int e, float4 xv) {
        const int64_t s = (int64_t)(e >> lct) * l2 + c0i + (e & (ct - 1));
        const bool lo = s < hl;
        const int64_t q = lo ? s : 2 * hl - 1 - s;
        const uint32_t w = sg[q >> 3] >> ((4 * q) & 31);
        float re, im;
        if (lo) { re = (w & 1u) ? -xv.x : xv.x; im = (w & 4u) ? -xv.z : xv.z; }
        else    { re = (w & 8u) ? -xv.w : xv.w; im = (w & 2u) ? -xv.y : xv.y; }
        sb[swz<T>(e)] = mk<T>((T)re, (T)im);
      });
      __syncthreads();
      col_fft<false>();
      {
        const int NT = blockDim.x, np = tile / 2;
        const int e0 = 2 * (int)threadIdx.x;
        const int64_t k10 = e0 >> lct, dk = (2 * NT) >> lct;
        const int64_t m2 = c0i + (e0 & (ct - 1));
        const C2<T> sa = tf(dk * m2), sbb = tf(dk * (m2 + 1));
        for (int u0 = 0, p0 = threadIdx.x; p0 < np; u0 += TW_ANCHOR, p0 += TW_ANCHOR * NT) {
          const int64_t k1g = k10 + u0 * dk;
          C2<T> wa = tf(k1g * m2), wb = tf(k1g * (m2 + 1));
#pragma unroll
          for (int s2 = 0; s2 < TW_ANCHOR; ++s2) {
            const int p = p0 + s2 * NT;
            if (p >= np) break;
            const int64_t k1 = k1g + s2 * dk;
            if (s2) {
              wa = cmul<T>(wa, sa);
              wb = cmul<T>(wb, sbb);
            }
            const int e = 2 * p;
            stp<T>(&wk[k1 * l2 + m2], CP<T>{cmul<T>(sb[swz<T>(e)], wa), cmul<T>(sb[swz<T>(e + 1)], wb)});
          }
        }
      }
      __syncthreads();
    }
  }
  // pass A with a sparse input (H d, RES x on a support): each tile's few nonzeros are
  // scattered from the bucketed support list into a zeroed tile — U is never read
  CS_NOINL void passA_sparse(const T* vals) { passA_sparse_i(vals); }
  CS_DEV void passA_sparse_i(const T* vals) {
    const int ct = CT, lct = (ct == 4) ? 2 : 1;
    const int64_t l2 = L2, ntl = L2 / ct;
    const int tile = (int)(L1 * ct);
    C2<T>* sb = shp(buf);
    T* sbt = reinterpret_cast<T*>(sb);
    C2<T>* wk = Wk;
    const GTw<T> tf = twF;
    const int* sp = in_supp;
    const int64_t* ip = in_pos;
    const uint32_t* sg = sign;
    T* const upd = (dfr_d == vals) ? dfr_d : nullptr;   // deferred CG updates (above)
    T* const ur = dfr_r;
    T* const ux = dfr_x;
    const T* const uq = dfr_q;
    const T ua = dfr_alpha, ub = dfr_beta;
    dfr_d = nullptr;
    for (int64_t t = blk; t < ntl; t += nblk) {
      const int64_t c0i = t * ct;
      for (int e = threadIdx.x; e < tile; e += blockDim.x) sb[e] = mk<T>(0, 0);
      __syncthreads();
      const bool cached = acn >= 0 && t == blk;   // build_acache: this block's one tile
      const int* ac = reinterpret_cast<const int*>(sb + acache_off());
      const int qa = cached ? 0 : tcnt[t], qe = cached ? acn : tcnt[t + 1];
      for (int q = qa + threadIdx.x; q < qe; q += blockDim.x) {
        int i, slot;
        bool neg;
        if (cached) {
          const int w = ac[2 * q];
          i = ac[2 * q + 1];
          slot = w & 0x7fffffff;
          neg = w < 0;
        } else {
          i = tlist[q];
          const int64_t p = ip[i], c = p >> 1;
          const int e = (int)(((c >> log2L2) << lct) | ((c & (l2 - 1)) - c0i));
          slot = 2 * swz<T>(e) + (int)(p & 1);
          neg = bit_test(sg, sp[i]);
        }
        T v = vals[i];
        if (upd) {
          T ri = ur[i];
          if (ux) {
            ux[i] += ua * v;                 // line 17
            ri -= ua * uq[i];                // line 18
            ur[i] = ri;
          }
          v = ri + ub * v;                   // line 20
          upd[i] = v;
        }
        sbt[slot] = neg ? -v : v;
      }
      __syncthreads();
      col_fft<false>();
      {
        const int NT = blockDim.x, np = tile / 2;
        const int e0 = 2 * (int)threadIdx.x;
        const int64_t k10 = e0 >> lct, dk = (2 * NT) >> lct;
        const int64_t m2 = c0i + (e0 & (ct - 1));
        const C2<T> sa = tf(dk * m2), sbb = tf(dk * (m2 + 1));
        for (int u0 = 0, p0 = threadIdx.x; p0 < np; u0 += TW_ANCHOR, p0 += TW_ANCHOR * NT) {
          const int64_t k1g = k10 + u0 * dk;
          C2<T> wa = tf(k1g * m2), wb = tf(k1g * (m2 + 1));
#pragma unroll
          for (int s2 = 0; s2 < TW_ANCHOR; ++s2) {
            const int pp = p0 + s2 * NT;
            if (pp >= np) break;
            const int64_t k1 = k1g + s2 * dk;
            if (s2) {
              wa = cmul<T>(wa, sa);
              wb = cmul<T>(wb, sbb);
            }
            const int e = 2 * pp;
            stp<T>(&wk[k1 * l2 + m2], CP<T>{cmul<T>(sb[swz<T>(e)], wa), cmul<T>(sb[swz<T>(e + 1)], wb)});
          }
        }
      }
      __syncthreads();
    }
  }
  // pass C with a sparse output (H d restricted to the support): after the inverse column
  // FFT each tile writes only its support entries, q_i = sigma_j . buf[p_i] — Cb is never
  // written and no separate gather runs
  // dvec != nullptr: also returns this thread's share of sum_i dvec_i outv_i (H's dot
  // product, reduced by the caller with the pass's closing barrier)
  CS_NOINL double passC_sparse(T* outv, const T* dvec = nullptr, const T* rvec = nullptr) {
    return passC_sparse_i(outv, dvec, rvec);
  }
  CS_DEV double passC_sparse_i(T* outv, const T* dvec, const T* rvec) {
    double dot = 0, rq = 0, qq = 0, rr = 0;
    const int ct = CT, lct = (ct == 4) ? 2 : 1;
    const int64_t l2 = L2, ntl = L2 / ct;
    const int tile = (int)(L1 * ct);
    C2<T>* sb = shp(buf);
    const T* sbt = reinterpret_cast<const T*>(sb);
    const C2<T>* wk = Wk;
    const int* sp = in_supp;
    const int64_t* ip = in_pos;
    const uint32_t* sg = sign;
    // the tile's output entries are resolved (support list -> smem slot, sign, output index)
    // while its cp.async loads and the column FFT run: staged in the pass-B metadata buffer
    // (two words per entry); a tile with more entries than fit takes the direct path
    int* stg = reinterpret_cast<int*>(shp(msm));
    const int cap = (int)((2 * L2) >> 5) * 2;
    int64_t t = blk;
    int q0 = t < ntl ? tcnt[t] : 0, q1 = t < ntl ? tcnt[t + 1] : 0;
    for (; t < ntl; t += nblk) {
      const int64_t tn = t + nblk;
      const int q0n = tn < ntl ? tcnt[tn] : 0, q1n = tn < ntl ? tcnt[tn + 1] : 0;  // next tile's
      if (q1 != q0) {  // a tile without support entries is skipped
        const int64_t c0i = t * ct;
        for (int e = threadIdx.x; e < tile; e += blockDim.x)
          cp_async_c<T>(&sb[swz<T>(e)], &wk[(int64_t)(e >> lct) * l2 + c0i + (e & (ct - 1))]);
        const int cnt = q1 - q0;
        const bool staged = cnt <= cap;
        if (staged) {
          for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
            const int i = tlist[q0 + q];
            const int64_t p = ip[i], c = p >> 1;
            const int e = (int)(((c >> log2L2) << lct) | ((c & (l2 - 1)) - c0i));
            const int slot = 2 * swz<T>(e) + (int)(p & 1);
            stg[2 * q] = slot | (bit_test(sg, sp[i]) ? (int)0x80000000 : 0);
            stg[2 * q + 1] = i;
          }
        }
        cp_async_wait_all();
        __syncthreads();
        col_fft<true>();
        if (staged) {
          for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
            const int w = stg[2 * q];
            const T v = sbt[w & 0x7fffffff];
            const int oi = stg[2 * q + 1];
            const T o = (w < 0) ? -v : v;
            outv[oi] = o;
            if (dvec) dot += (double)dvec[oi] * (double)o;
            if (rvec) {
              const double rv = (double)rvec[oi];
              rq += rv * (double)o;
              qq += (double)o * (double)o;
              rr += rv * rv;
            }
          }
        } else {
          for (int q = q0 + threadIdx.x; q < q1; q += blockDim.x) {
            const int i = tlist[q];
            const int64_t p = ip[i], c = p >> 1;
            const int e = (int)(((c >> log2L2) << lct) | ((c & (l2 - 1)) - c0i));
            const T o = apply_sign<T>(sg, sp[i], sbt[2 * swz<T>(e) + (int)(p & 1)]);
            outv[i] = o;
            if (dvec) dot += (double)dvec[i] * (double)o;
            if (rvec) {
              const double rv = (double)rvec[i];
              rq += rv * (double)o;
              qq += (double)o * (double)o;
              rr += rv * rv;
            }
          }
        }
        __syncthreads();
      }
      q0 = q0n;
      q1 = q1n;
    }
    p_rq = rq;
    p_qq = qq;
    p_rr = rr;
    return dot;
  }
  template <int MODE> CS_NOINL double passB(bool zero_input, T* yout) { return passB_i<MODE>(zero_input, yout); }
  template <int MODE> CS_DEV double passB_i(bool zero_input, T* yout) {
    MidCtx<T> m = mid0;
    m.rowmask = rowmask;
    m.prefix = prefix;
    m.y = y;
    m.yout = yout;
    m.s1 = s1;
    m.tsh = tsh;
    double rn2 = 0;
    const int64_t nitems = L1 / 2 + 1;
    const int64_t ilo = di_hi < 0 ? 0 : di_lo, ihi = di_hi < 0 ? nitems : di_hi;
    for (int64_t it = ilo + blk; it < ihi; it += nblk) {
      const int64_t ka = it, kb = L1 - it;
      const bool self = (it == 0 || it == L1 / 2);
      const int B = self ? 1 : 2;
      const int lb = B - 1;  // log2 B
      const int n2 = (int)L2;
      {
        C2<T>* sb = shp(buf);
        const C2<T>* wk = Wk;
        const int64_t l2 = L2;
        if (zero_input) {
          for (int e = threadIdx.x; e < B * n2; e += blockDim.x) sb[swz<T>(e)] = mk<T>(0, 0);
        } else {
          // pair q: row r = q & lb, m2 = 2 (q >> lb); smem element e = (m2 << lb) | r
          for (int e = threadIdx.x; e < B * n2; e += blockDim.x)
            cp_async_c<T>(&sb[swz<T>(e)], &wk[((e & lb) ? kb : ka) * l2 + (e >> lb)]);
          // (waited for after the metadata staging below: the two L2 round trips overlap)
        }
      }
      {
        // stage the transposed-mask and prefix words of rows ka, kb
        const int W = (int)((2 * L2) >> 5);
        uint32_t* ms = shp(msm);
        const int32_t* pg = prefix;
        const uint32_t* mg = rowmask;
        const int64_t r0 = ka * (int64_t)W, r1 = (kb & (L1 - 1)) * (int64_t)W;
        if (W > 0) staged<TL_UNR, uint32_t>(4 * W, [&](int e) {
          const int q = e / W, w = e - q * W;
          const int64_t at = ((q & 1) ? r1 : r0) + w;
          return (q < 2) ? mg[at] : (uint32_t)pg[at];
        }, [&](int e, uint32_t v) { ms[e] = v; });
      }
      cp_async_wait_all();
      __syncthreads();
#ifdef CS_DIAG_PASSB
      if (MODE == MID_H) mark(10);  // load + metadata staging
#endif
      if (!zero_input) row_fft<false>(B);
#ifdef CS_DIAG_PASSB
      if (MODE == MID_H) mark(11);  // forward row FFTs
#endif
      C2<T>* zb = shp(buf);
      {
        // a transposed row shorter than a word (small-N fallback): read the mask in place
        const int W = (int)((2 * L2) >> 5);
        m.rowmask = W > 0 ? shp(msm) : rowmask;
        m.prefix = W > 0 ? reinterpret_cast<const int32_t*>(shp(msm) + 2 * W) : prefix;
        m.staged = W > 0;
        m.ra = (int)ka;
      }
      if (fkind == 1) {
        // partial Fourier (R36): the same pairs (n, L - n), the real-DFT split
        if (it == 0) {
          for (int k2 = threadIdx.x; k2 <= n2 / 2; k2 += blockDim.x) {
            if (k2 == 0) dft_zero<T, MODE>(zb[swz<T>(0)], m, rn2);
            else dft_pair<T, MODE>(zb[swz<T>(k2)], zb[swz<T>(n2 - k2)], L1 * k2, tw4(L1 * k2), m, rn2);
          }
        } else if (it == L1 / 2) {
          for (int k2 = threadIdx.x; k2 < n2 / 2; k2 += blockDim.x) {
            const int64_t k = L1 / 2 + L1 * k2;
            dft_pair<T, MODE>(zb[swz<T>(k2)], zb[swz<T>(n2 - 1 - k2)], k, tw4(k), m, rn2);
          }
        } else {
          for (int k2 = threadIdx.x; k2 < n2; k2 += blockDim.x) {
            const int64_t k = ka + L1 * k2;
            dft_pair<T, MODE>(zb[swz<T>(2 * k2)], zb[swz<T>(2 * (n2 - 1 - k2) + 1)], k, tw4(k), m, rn2);
          }
        }
      } else if (it == 0) {
        for (int k2 = threadIdx.x; k2 <= n2 / 2; k2 += blockDim.x) {
          if (k2 == 0) mid_zero<T, MODE>(zb[swz<T>(0)], m, rn2);
          else {
            int64_t k = L1 * k2;
            mid_pair<T, MODE>(zb[swz<T>(k2)], zb[swz<T>(n2 - k2)], k, tw4(k), m, rn2);
          }
        }
      } else if (it == L1 / 2) {
        for (int k2 = threadIdx.x; k2 < n2 / 2; k2 += blockDim.x) {
          int64_t k = L1 / 2 + L1 * k2;
          mid_pair<T, MODE>(zb[swz<T>(k2)], zb[swz<T>(n2 - 1 - k2)], k, tw4(k), m, rn2);
        }
      } else if (m.staged && L2 >= 256 && blockDim.x == 256) {
        // general item, strength-reduced (the common case: every item of c2/c3/c5).  Thread
        // t owns k2 = t + 256 u.  Its four mask bits sit at fixed bit positions (k2 & 31 or
        // 31 - (k2 & 31)) of words that move by +-8 per step; its two buffer slots move by
        // +-512 (above the swizzle's bits, so swz is computed once); the twiddle
        // a = W_4N^(ka + L1 k2) follows the anchored recurrence of passes A/B (a table
        // lookup every TW_ANCHOR steps).  Same arithmetic as the branch below.
        const int W = (int)((2 * L2) >> 5), W1 = (int)(L2 >> 5);
        const uint32_t* mw = m.rowmask;
        const int32_t* pw = m.prefix;
        const MidK<T> cst = make_midk<T>((int)N);
        const int t = (int)threadIdx.x, b0 = t & 31, b1 = 31 - b0;
        const uint32_t lm0 = (1u << b0) - 1u, lm1 = (1u << b1) - 1u;
        const int s0 = swz<T>(2 * t), s1i = swz<T>(2 * n2 - 1 - 2 * t);
        const int64_t l1 = L1;
        const C2<T> astep = tw4(l1 * 256);
        // unrolled by TW_ANCHOR: one table lookup per group (a predicated lookup in every
        // step otherwise), the group's independent pair chains interleave
        for (int u0 = 0, k20 = t; k20 < n2; u0 += TW_ANCHOR, k20 += 256 * TW_ANCHOR) {
        C2<T> a = tw4(ka + l1 * k20);
#pragma unroll
        for (int st = 0; st < TW_ANCHOR; ++st) {
          const int u = u0 + st, k2 = k20 + 256 * st;
          if (k2 >= n2) break;
          const int q = k2 >> 5;
          const int wi[4] = {q, W + 2 * W1 - 1 - q, W + W1 - 1 - q, W1 + q};
          const int bi[4] = {b0, b1, b1, b0};
          if (st) a = cmul<T>(a, astep);
          const C2<T> a2 = cmul<T>(a, a);
          const C2<T> w = cmul<T>(a2, a2);
          mid_pair2g<T, MODE>(zb[s0 + 512 * u], zb[s1i - 512 * u], a, w, m, cst, rn2,
              [&](int qq) { return (bool)((mw[wi[qq]] >> bi[qq]) & 1u); },
              [&](int qq) {
                return pw[wi[qq]] + __popc(mw[wi[qq]] & ((bi[qq] == b0) ? lm0 : lm1));
              });
        }
        }
      } else if (m.staged) {
        // general item (rows ka, kb = L1 - ka): the four DCT indices of the pair at column
        // k2 sit in the staged rows at (ka, k2), (kb, 2L2-1-k2), (kb, L2-1-k2), (ka, L2+k2)
        // (transposed order, §5.2); constants folded as in Tier S (dct_mid.cuh mid_pair2g)
        const int W = (int)((2 * L2) >> 5), l2i = (int)L2;
        const uint32_t* mw = m.rowmask;
        const int32_t* pw = m.prefix;
        const MidK<T> cst = make_midk<T>((int)N);
        for (int k2 = threadIdx.x; k2 < n2; k2 += blockDim.x) {
          const int k = (int)ka + (int)L1 * k2;
          const int slot[4] = {0, W, W, 0};
          const int bb[4] = {k2, 2 * l2i - 1 - k2, l2i - 1 - k2, l2i + k2};
          const C2<T> a = tw4(k);
          const C2<T> a2 = cmul<T>(a, a);
          const C2<T> w = cmul<T>(a2, a2);
          mid_pair2g<T, MODE>(zb[swz<T>(2 * k2)], zb[swz<T>(2 * (n2 - 1 - k2) + 1)], a, w, m, cst, rn2,
              [&](int q) { return (bool)((mw[slot[q] + (bb[q] >> 5)] >> (bb[q] & 31)) & 1u); },
              [&](int q) {
                const int wi = slot[q] + (bb[q] >> 5), bit = bb[q] & 31;
                return pw[wi] + __popc(mw[wi] & ((1u << bit) - 1u));
              });
        }
      } else {
        for (int k2 = threadIdx.x; k2 < n2; k2 += blockDim.x) {
          int64_t k = ka + L1 * k2;
          mid_pair<T, MODE>(zb[swz<T>(2 * k2)], zb[swz<T>(2 * (n2 - 1 - k2) + 1)], k, tw4(k), m, rn2);
        }
      }
      __syncthreads();
#ifdef CS_DIAG_PASSB
      if (MODE == MID_H) mark(12);  // middle
#endif
      if constexpr (MODE != MID_FWD) {
        row_fft<true>(B);
#ifdef CS_DIAG_PASSB
        if (MODE == MID_H) mark(13);  // inverse row FFTs
#endif
        C2<T>* sb = shp(buf);
        C2<T>* wk = Wk;
        const GTw<T> tf = twF;
        const int64_t l2 = L2;
        // pairs q = tid + u NT: fixed row r, columns m2 = m20 + u dm (anchored recurrence
        // of W_L^{-k1 m2} as in pass A)
        {
          const int NT = blockDim.x, nq = B * n2 / 2;
          const int r = (int)threadIdx.x & lb;
          const int64_t k1 = r ? kb : ka;
          const int64_t m20 = 2 * ((int)threadIdx.x >> lb), dm = 2 * (NT >> lb);
          const C2<T> st = tf(k1 * dm);  // W^{k1 dm}
          for (int u0 = 0, q0 = threadIdx.x; q0 < nq; u0 += TW_ANCHOR, q0 += TW_ANCHOR * NT) {
            const int64_t m20g = m20 + u0 * dm;
            C2<T> wa = tf(k1 * m20g), wb = tf(k1 * (m20g + 1));
#pragma unroll
            for (int s2 = 0; s2 < TW_ANCHOR; ++s2) {
              if (q0 + s2 * NT >= nq) break;
              const int64_t m2 = m20g + s2 * dm;
              if (s2) {
                wa = cmul<T>(wa, st);
                wb = cmul<T>(wb, st);
              }
              stp<T>(&wk[k1 * l2 + m2], CP<T>{cmulc<T>(sb[swz<T>((int)(m2 << lb) | r)], wa),
                                               cmulc<T>(sb[swz<T>((int)((m2 + 1) << lb) | r)], wb)});
            }
          }
        }
      }
      __syncthreads();
#ifdef CS_DIAG_PASSB
      if (MODE == MID_H) mark(14);  // twiddle + store
#endif
    }
    return rn2;
  }
  CS_NOINL void passC() { passC_i(); }
  CS_DEV void passC_i() {
    C2<T>* Cc = reinterpret_cast<C2<T>*>(Cb);
    const int ct = CT, lct = (ct == 4) ? 2 : 1;
    const int64_t l2 = L2, ntiles = L2 / ct;
    const int tile = (int)(L1 * ct);
    C2<T>* sb = shp(buf);
    const C2<T>* wk = Wk;
    const int64_t tlo = dt_hi < 0 ? 0 : dt_lo, thi = dt_hi < 0 ? ntiles : dt_hi;
    for (int64_t t = tlo + blk; t < thi; t += nblk) {
      const int64_t c0i = t * ct;
      for (int e = threadIdx.x; e < tile; e += blockDim.x)
        cp_async_c<T>(&sb[swz<T>(e)], &wk[(int64_t)(e >> lct) * l2 + c0i + (e & (ct - 1))]);
      cp_async_wait_all();
      __syncthreads();
      col_fft<true>();
      staged<TL_UNR, CP<T>>(tile / 2, [&](int p) {
        return CP<T>{sb[swz<T>(2 * p)], sb[swz<T>(2 * p + 1)]};
      }, [&](int p, const CP<T>& v) {
        const int e = 2 * p;
        stp<T>(&Cc[(int64_t)(e >> lct) * l2 + c0i + (e & (ct - 1))], v);
      });
      __syncthreads();
    }
  }
  CS_NOINL void H(const T* d, T* q) {
    if (psi) { H_psi(d, q); return; }
    mark(0);
    passA_sparse_i(d);
    sync();
    mark(1);
    passB_i<MID_H>(false, nullptr);
    sync();
    mark(2);
    passC_sparse_i(q, nullptr, nullptr);
    sync();
    mark(3);
    ++applies;
  }
  // q = H d and d.q: the dot product rides on pass C (each block sums the entries it
  // writes) and on the barrier that closes H — one grid barrier per CG iteration less
  CS_NOINL double H_dot(const T* d, T* q) {
    if (psi) {
      H_psi(d, q);
      return dot_n(*this, d, q, in_ns);
    }
    mark(0);
    passA_sparse(d);
    sync();
    mark(1);
    passB<MID_H>(false, nullptr);
    sync();
    mark(2);
    const double t = block_sum(passC_sparse(q, d));
    double* P = g.pd + bank * g.maxgrid;
    if (threadIdx.x == 0) P[blk] = t;
    sync();                                    // publishes q and the per-block partials
    if (threadIdx.x < 32) {
      double a = 0;
      a = lane_sum<double>(P, (int)nblk, (int)threadIdx.x);
      a = warp_sum_g(a);
      if (threadIdx.x == 0) sd[32] = a;
    }
    __syncthreads();
    const double tot = sd[32];
    __syncthreads();
    bank ^= 1;
    mark(3);
    ++applies;
    return tot;
  }
  // q = H d with pass C summing d.q, r.q, q.q and r.r in one grid reduction (H's closing
  // barrier); r = the current residual (updated by pass A).  sums = {d.q, r.q, q.q, r.r}.
  // the three passes inlined: one call frame (one callee-saved register save / restore
  // through local memory) per H instead of three — the CG loop's H at every grid size
  CS_DEV void H_dot4(const T* d, T* q, const T* r, double* sums) {
    mark(0);
    passA_sparse_i(d);
    sync();
    mark(1);
    passB_i<MID_H>(false, nullptr);
    sync();
    mark(2);
    double t[4];
    t[0] = passC_sparse_i(q, d, r);
    t[1] = p_rq;
    t[2] = p_qq;
    t[3] = p_rr;
    constexpr int NW = (1 << TL_LOG2NT) / 32;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      t[k] = warp_sum_g(t[k]);
      if (lane == 0) sd[k * NW + (threadIdx.x >> 5)] = t[k];
    }
    __syncthreads();
    if (threadIdx.x < 4) {   // [4][2][maxgrid] per-block partials (pd)
      double a = 0;
      for (int w = 0; w < NW; ++w) a += sd[threadIdx.x * NW + w];
      g.pd[((int)threadIdx.x * 2 + bank) * g.maxgrid + blk] = a;
    }
    sync();                                    // publishes q, r and the per-block partials
    if (threadIdx.x < 128) {
      const int k = (int)threadIdx.x >> 5;
      const double* P = g.pd + (k * 2 + bank) * g.maxgrid;
      double a = 0;
      a = lane_sum<double>(P, (int)nblk, (int)lane);
      a = warp_sum_g(a);
      if (lane == 0) sd[k] = a;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 4; ++k) sums[k] = sd[k];
    __syncthreads();
    bank ^= 1;
    mark(3);
    ++applies;
  }
  // Algorithm 1 lines 14-22 with one grid reduction per iteration (R37): pass C
  // of H sums d.q, r.q, q.q and the residual's true r.r, so every block then has
  //   alpha = r.r / d.q  and  |r - alpha q|^2 = r.r - 2 alpha r.q + alpha^2 q.q
  // (beta and the stopping test) without a second reduction.  r.r is re-anchored on the
  // vector every iteration — a running recurrence drifts by ~eps |r_0|^2 and diverges once
  // |r| falls below that.  The updates of x, r (lines 17-18) and d (line 20) are applied by
  // the next H's pass A to the entries it scatters, and by a flush after the loop.
  template <class S> CS_NOINL void cg_iterate(S& s_io) {
    if (psi) {
      cg_loop(*this, s_io, [this](const T* d, T* q) { return H_dot(d, q); });
      return;
    }
    S s = s_io;
#ifdef CS_DIAG_GLUE
    mark(20);  // cg_iterate entry
#endif
    T *xx = s.x, *rv = s.r, *dv = s.d, *qv = s.q;
    bool pend = false;
    T alpha = T(0);
    while (true) {
      if (!(s.rr > s.thr)) break;                                          // line 15 (R6, R7)
      if (s.j >= s.cap) { s.status |= CS_DEV_CG_CAP; break; }
      double sums[4];
      H_dot4(dv, qv, rv, sums);                                            // applies the pending updates
      const double dq = sums[0], rq = sums[1], qq = sums[2], rrt = sums[3];
      pend = false;
      if (!(dq > 0.0)) { s.status |= CS_DEV_CG_BREAKDOWN; break; }
      alpha = (T)(rrt / dq);                                               // line 16
      const double a = (double)alpha;
      double rr2 = rrt - 2.0 * a * rq + a * a * qq;                        // |r_{j+1}|^2
      if (rr2 < 0.0) rr2 = 0.0;
      const T beta = (T)(rr2 / rrt);                                       // line 19
      dfr_d = dv; dfr_r = rv; dfr_x = xx; dfr_q = qv; dfr_alpha = alpha; dfr_beta = beta;
      pend = true;
      s.rr = rr2;
      s.j += 1;                                                            // line 21
      if (!(rr2 == rr2)) { s.status |= CS_DEV_CG_BREAKDOWN; break; }
    }
    dfr_d = nullptr;
    if (pend) {                                                            // lines 17-18 of the last iteration
      for (int i = gtid; i < s.ns; i += gnthr) {
        xx[i] += alpha * dv[i];
        rv[i] -= alpha * qv[i];
      }
    }
    s_io = s;   // cg_solve's barrier right after this call publishes the flush
  }
  CS_NOINL double RES(const T* x) {
    if (psi) return RES_psi(x);
    mark(0);
    if (x) {
      passA_sparse_i(x);
      sync();
    }
    mark(4);
    double rn2 = passB_i<MID_RES>(x == nullptr, nullptr);
    sync();
    mark(5);
    passC_i();
    const double r = sum(rn2);  // the reduction's barrier also publishes Cb
    mark(6);
    ++applies;
    return r;
  }

  // ---- Psi = C_N (R35): C_N, Phi and C_N^T composed from the same passes.  A full DCT-II
  // (all N outputs) is pass A + pass B (MID_FWD) on the all-rows instance (rank = the
  // transposed position, mapped back to k by its tperm); C_N^T of a dense vector is pass B
  // (MID_RES on a zero input) + pass C on the all-rows instance.  sigma and pi act between
  // the two domains through G (natural order).
  CS_DEV void use_full() { rowmask = ftmask; prefix = ftprefix; tperm = ftperm; }
  CS_DEV void use_real() { rowmask = r_tmask; prefix = r_tprefix; tperm = r_tperm; }
  // G <- C_N s: s = scatter_S(vals), or (vals == nullptr) the dense s already in U
  CS_NOINL void psi_to_G(const T* vals) {
    use_full();
    if (vals) passA_sparse(vals); else passA();
    sync();
    passB<MID_FWD>(false, yTf);
    sync();
    const int32_t* tp = ftperm;
    const T* yt = yTf;
    T* g = G;
    gstaged<TL_UNR, T>(N, gtid, gnthr, [&](int64_t t) { return yt[t]; }, [&](int64_t t, T v) { g[tp[t]] = v; });
    sync();
  }
  // U <- Makhoul order of R diag(sigma) G
  CS_NOINL void phi_in() {
    const uint32_t* sg = phi_sign;
    const int32_t* pv = phi_pinv;
    const T* g = G;
    T* u = U;
    const int64_t n = N;
    // value and position loaded together (no dependent load in the store phase)
    for (int64_t j0 = gtid; j0 < n; j0 += TL_UNR * gnthr) {
      T v[TL_UNR];
      int64_t p[TL_UNR];
#pragma unroll
      for (int q = 0; q < TL_UNR; ++q) {
        const int64_t j = j0 + q * gnthr;
        if (j < n) { v[q] = apply_sign<T>(sg, j, g[j]); p[q] = pv ? pv[j] : j; }
      }
#pragma unroll
      for (int q = 0; q < TL_UNR; ++q) {
        const int64_t j = j0 + q * gnthr;
        if (j < n) u[mk_pos(p[q], n)] = v[q];
      }
    }
    sync();
  }
  // G <- diag(sigma) R^T v, v = Cb (Makhoul order)
  CS_NOINL void phi_out() {
    const uint32_t* sg = phi_sign;
    const int32_t* pv = phi_pinv;
    const T* cb = Cb;
    T* g = G;
    const int64_t n = N;
    gstaged<TL_UNR, T>(N, gtid, gnthr, [&](int64_t j) { return apply_sign<T>(sg, j, cb[ppos(pv, j, n)]); },
                       [&](int64_t j, T v) { g[j] = v; });
    sync();
  }
  // pass B of C_N^T G on the all-rows instance (pass C follows in the caller)
  CS_NOINL void psiT_passB() {
    use_full();
    const int32_t* tp = ftperm;
    const T* g = G;
    T* yt = yTf;
    gstaged<TL_UNR, T>(N, gtid, gnthr, [&](int64_t t) { return g[tp[t]]; }, [&](int64_t t, T v) { yt[t] = v; });
    sync();
    const T* ys = y;
    y = yTf;
    passB<MID_RES>(true, nullptr);
    sync();
    y = ys;
  }
  CS_NOINL void H_psi(const T* d, T* q) {
    psi_to_G(d);                     // C_N s
    phi_in();                        // R diag(sigma)
    use_real();
    passA();
    sync();
    passB<MID_H>(false, nullptr);    // C^T P^T P C
    sync();
    passC();
    sync();
    phi_out();                       // diag(sigma) R^T
    psiT_passB();                    // C_N^T ...
    passC_sparse(q);                 // ... on the support only
    sync();
    use_real();
    ++applies;
  }
  CS_NOINL double RES_psi(const T* x) {
    double rn2;
    if (x) {
      psi_to_G(x);
      phi_in();
      use_real();
      passA();
      sync();
      rn2 = passB<MID_RES>(false, nullptr);   // Phi^T (y - Phi u)
    } else {
      use_real();
      rn2 = passB<MID_RES>(true, nullptr);    // Phi^T y
    }
    sync();
    passC();
    const double r = sum(rn2);                // also publishes Cb
    phi_out();
    psiT_passB();
    passC();                                  // A^T r, s-domain, Makhoul order
    sync();
    use_real();
    ++applies;
    return r;
  }
};

}  // namespace cs
