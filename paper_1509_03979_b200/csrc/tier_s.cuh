// tier_s.cuh — Tier S: one thread block per problem, the whole pursuit resident in
// shared memory (N <= 16384, i.e. the half-length FFT of <= 8192 points fits).
// Used for config 1 (OMP, N = 4096) and config 4 (4096 batched SP problems,
// N = 16384), and for batched operator apply / adjoint at those sizes.
#pragma once
#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <utility>

#include "ctx_cta.cuh"
#include "layout_s.cuh"
#include "pursuit.cuh"

namespace cs {

constexpr int64_t TIER_S_MAX_N = 16384;
constexpr int TS_THREADS = SW_NT;  // 512: <= 16 points per thread per FFT pass

CS_HD int64_t align_up(int64_t x, int64_t a) {
  return (a & (a - 1)) ? (x + a - 1) / a * a : (x + a - 1) & -a;   // a power of two: no division
}

// Shared-memory layout of a Tier S block (computed identically on host and device).
struct SLayout {
  int64_t Z, twLlo, twLhi, tw4lo, tw4hi, sign, rmask, prefix, redd, redi, redk, hist, pick, h1, ckey, cidx, ccnt;
  int64_t S, S2, U, x, x2, xU, r, d, q, b, Sbits, Ubits, Pbits;
  int64_t bytes;
  int nthreads;
};

template <typename T>
CS_HD SLayout s_layout(int64_t N, int K, int ucap, bool pursuit) {
  SLayout s;
  const int64_t nw = (N + 31) / 32, ts = sizeof(T);
  const SFix f = s_fixed<T>(N);
  s.Z = f.Z; s.twLlo = f.twLlo; s.twLhi = f.twLhi; s.tw4lo = f.tw4lo; s.tw4hi = f.tw4hi;
  s.sign = f.sign; s.rmask = f.rmask; s.prefix = f.prefix; s.redd = f.redd; s.redi = f.redi;
  s.redk = f.redk; s.hist = f.hist; s.pick = f.pick; s.h1 = f.h1; s.ckey = f.ckey; s.cidx = f.cidx;
  s.ccnt = f.ccnt;
  int64_t o = f.end;
  auto take = [&](int64_t bytes) { int64_t r = o; o = align_up(o + bytes, 16); return r; };
  if (pursuit) {
    s.S = take((int64_t)K * 4);
    s.S2 = take((int64_t)K * 4);
    s.U = take((int64_t)ucap * 4);
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
    s.S = s.S2 = s.U = s.x = s.x2 = s.xU = s.r = s.d = s.q = s.b = s.Sbits = s.Ubits = s.Pbits = 0;
  }
  s.bytes = o;
  s.nthreads = TS_THREADS;
  return s;
}

// Per-instance metadata (abi.cu meta_stride): [sign nw], for N <= 16384 the natural-order
// [rowmask nw][prefix nw] of Tier S, then the Tier L [tmask nw][tprefix nw][tperm M]: the
// row mask TRANSPOSED to the four-step's pass-B order — DCT index
// k = a + L1 b (a < L1, b < 2 L2) at bit t = a (2 L2) + b — its rank prefix in that order,
// and tperm[t_rank] = y index of the t_rank-th selected row in that order.
struct OpMeta {
  const uint32_t* base;
  int64_t N, M;          // M: measurements (= rows for the DCT, 2 x frequencies for the DFT)
  int64_t Mr;            // metadata rows (tperm length)
  int64_t nw;
  int64_t stride;  // words per instance
  int64_t toff;    // word offset of the transposed mask within an instance
  const int32_t* perm;  // Eq.(7) randomizer R (R34): per instance [pi N][pi^-1 N], or null
  int psi;              // dictionary: 0 = I, 1 = C_N (R35)
  int fkind;            // F: 0 = DCT-II, 1 = partial Fourier (R36; perm then holds the position map)
  const uint32_t* full; // Psi mode: the all-rows instance (stride meta_stride(N, N)), or null
  const double2* tw;    // the grid tier's twiddle tables, precomputed (tier_l.cuh l_tw_off), or null
  CS_HD const uint32_t* sign(int64_t b) const { return base + b * stride; }
  CS_HD const uint32_t* rmask(int64_t b) const { return base + b * stride + nw; }
  CS_HD const int32_t* prefix(int64_t b) const {
    return reinterpret_cast<const int32_t*>(base + b * stride + 2 * nw);
  }
  CS_HD const uint32_t* tmask(int64_t b) const { return base + b * stride + toff; }
  CS_HD const int32_t* tprefix(int64_t b) const {
    return reinterpret_cast<const int32_t*>(base + b * stride + toff + nw);
  }
  CS_HD const int32_t* tperm(int64_t b) const {
    return reinterpret_cast<const int32_t*>(base + b * stride + toff + 2 * nw);
  }
  CS_HD const uint32_t* full_sign() const { return full; }  // all zero (sigma = +1)
  CS_HD const uint32_t* full_tmask() const { return full + toff; }
  CS_HD const int32_t* full_tprefix() const { return reinterpret_cast<const int32_t*>(full + toff + nw); }
  CS_HD const int32_t* full_tperm() const { return reinterpret_cast<const int32_t*>(full + toff + 2 * nw); }
  CS_HD const int32_t* pm(int64_t b) const { return perm ? perm + b * 2 * N : nullptr; }
  CS_HD const int32_t* pinv(int64_t b) const { return perm ? perm + b * 2 * N + N : nullptr; }
};

template <typename T>
CS_DEV void cta_set_instance(CtaCtx<T>& c, char* smem, const OpMeta& meta, int64_t b);

// Initialise the CTA's shared context object (every thread writes the same values; the
// barrier at the end of cta_set_instance orders them before any use).
template <typename T>
CS_DEV void init_cta_ctx(CtaCtx<T>& c, char* smem, const SLayout& lay, const OpMeta& meta, int64_t b) {
  c.N = meta.N;
  c.M = meta.M;
  c.L = meta.N / 2;
  c.log2L = 0;
  while ((int64_t(1) << c.log2L) < c.L) ++c.log2L;
  c.Z = reinterpret_cast<C2<T>*>(smem + lay.Z);
  c.sign = reinterpret_cast<uint32_t*>(smem + lay.sign);
  c.rowmask = reinterpret_cast<uint32_t*>(smem + lay.rmask);
  c.prefix = reinterpret_cast<int32_t*>(smem + lay.prefix);
  c.twL.lo = reinterpret_cast<C2<T>*>(smem + lay.twLlo);
  c.twL.hi = reinterpret_cast<C2<T>*>(smem + lay.twLhi);
  c.tw4.lo = reinterpret_cast<C2<T>*>(smem + lay.tw4lo);
  c.tw4.hi = reinterpret_cast<C2<T>*>(smem + lay.tw4hi);
  c.redd = reinterpret_cast<double*>(smem + lay.redd);
  c.redi = reinterpret_cast<int64_t*>(smem + lay.redi);
  c.redk = reinterpret_cast<typename CtaCtx<T>::Key*>(smem + lay.redk);
  c.hist = reinterpret_cast<unsigned*>(smem + lay.hist);
  c.pick = reinterpret_cast<int64_t*>(smem + lay.pick);
  c.h1 = reinterpret_cast<unsigned*>(smem + lay.h1);
  c.ckey = reinterpret_cast<typename CtaCtx<T>::Key*>(smem + lay.ckey);
  c.cidx = reinterpret_cast<int*>(smem + lay.cidx);
  c.ccnt = reinterpret_cast<int*>(smem + lay.ccnt);
  for (int w = 0; w < SW_NT / 32; ++w) c.rbank_w[w] = 0;
  c.psi = meta.psi;
  c.fkind = meta.fkind;
  c.G = nullptr;
  c.in_supp = nullptr;
  c.in_ns = 0;
  c.applies = 0;
  if (threadIdx.x == 0) *reinterpret_cast<int*>(smem + s_fixed<T>(meta.N).zero) = 0;
  // twiddles into shared memory (once per CTA), then the instance
  const int64_t L = c.L;
  tw_init<T>(const_cast<C2<T>*>(c.twL.lo), const_cast<C2<T>*>(c.twL.hi), L,
             (int)(L >= 64 ? L / 64 : 1), c.gtid, c.gnthr);
  tw_init<T>(const_cast<C2<T>*>(c.tw4.lo), const_cast<C2<T>*>(c.tw4.hi), 8 * L,
             (int)(L / 128 + 1), c.gtid, c.gnthr);
  {
    // [r][k] = W_{16 Ns1}^{r k}, Ns1 = 2^NS1B of sandwich_cta.cuh SwPlan (fp64 sincospi)
    const int m = (c.log2L - 1) % 4, ns1 = 1 << (m == 0 ? 4 : m);
    C2<T>* t16 = reinterpret_cast<C2<T>*>(smem + s_fixed<T>(meta.N).tw16);
    for (int i = c.gtid; i < 256; i += c.gnthr) {
      const int r = i >> 4, k = i & 15;
      double sn, cn;
      sincospi(-2.0 * (double)((r * k) % (16 * ns1)) / (double)(16 * ns1), &sn, &cn);
      t16[i] = mk<T>((T)cn, (T)sn);
    }
  }
  cta_set_instance<T>(c, smem, meta, b);
}

// point the context at instance b: its sign / row mask / prefix into shared memory, its
// permutation pointers (the caller orders this after every use of the previous instance)
template <typename T>
CS_DEV void cta_set_instance(CtaCtx<T>& c, char* smem, const OpMeta& meta, int64_t b) {
  c.phi_sign = meta.sign(b);
  c.phi_pinv = meta.pinv(b);
  // Psi mode: the pursuit's index space is the s-domain (no sign, no permutation)
  c.pm = meta.psi ? nullptr : meta.pm(b);
  c.pinv = meta.psi ? nullptr : meta.pinv(b);
  if (threadIdx.x == 0)
    *reinterpret_cast<const int32_t**>(smem + s_fixed<T>(meta.N).zero + 8) = c.pinv;  // sandwich_cta.cuh
  const int64_t nw = meta.nw;
  const uint32_t* gs = meta.sign(b);
  const uint32_t* gm = meta.rmask(b);
  const int32_t* gp = meta.prefix(b);
  for (int64_t w = c.gtid; w < nw; w += c.gnthr) {
    c.sign[w] = meta.psi ? 0u : gs[w];
    c.rowmask[w] = gm[w];
    c.prefix[w] = gp[w];
  }
  __syncthreads();
}

// ---------------------------------------------------------------- kernels ---
// A x = Phi (C_N x) (R35): dense x into Z, full DCT-II to G, then Phi.  Out of line so the
// plain apply keeps its register allocation.
template <typename T>
CS_NOINL void s_apply_psi(CtaCtx<T>& c, const T* x, T* y, T* G) {
  (void)G;
  const int64_t N = c.N;
  T* zb = reinterpret_cast<T*>(c.Z);
  for (int j = c.gtid; j < (int)N; j += c.gnthr) zb[CtaCtx<T>::zt((int)mk_pos(j, N))] = x[j];
  __syncthreads();
  c.template sandwich_psi<MID_FWDZ, false>(nullptr, nullptr);       // Phi's input in place
  c.template sandwich<MID_FWD, false>(nullptr, nullptr, y);
}

// the sign / row-mask / prefix words of instance b (contiguous, 3 nw words) into L2: the
// per-instance staging in cta_set_instance otherwise waits on HBM latency (ncu: a quarter of
// the batched apply's stall samples)
CS_DEV void s_prefetch_meta(const OpMeta& meta, int64_t b) {
  const uint32_t bytes = (uint32_t)(3 * meta.nw * 4);
  if (bytes >= 16 && bytes % 16 == 0) prefetch_l2(meta.sign(b), bytes);
}

template <typename T>
__global__ void __launch_bounds__(TS_THREADS, sizeof(T) == 4 ? 2 : 1) k_s_apply(OpMeta meta, SLayout lay, const T* __restrict__ X,
                                                 T* __restrict__ Y, T* __restrict__ Gws, int64_t B) {
  extern __shared__ __align__(16) char smem[];
  // persistent: the CTA sets up its twiddle tables once and loops over instances
  __shared__ CtaCtx<T> c;
  init_cta_ctx<T>(c, smem, lay, meta, blockIdx.x);
  const int64_t N = c.N;
  for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
  if (b != blockIdx.x) {
    __syncthreads();  // the previous instance's sandwich is done with the buffer and metadata
    cta_set_instance<T>(c, smem, meta, b);
  }
  const T* x = X + b * N;
  if (threadIdx.x == 0 && b + gridDim.x < B) {
    prefetch_l2(X + (b + gridDim.x) * N, (uint32_t)(N * sizeof(T)));   // the next instance's x
    s_prefetch_meta(meta, b + gridDim.x);                                // and its metadata
  }
  if (c.psi) {
    s_apply_psi<T>(c, x, Y + b * c.M, Gws + b * N);
    continue;
  }
  if (c.pinv) {
    // Eq.(7) randomizer: x_j lands at the Makhoul position of pi^-1(j) (R34)
    T* zb = reinterpret_cast<T*>(c.Z);
    const int32_t* pv = c.pinv;
    for (int j = c.gtid; j < (int)N; j += c.gnthr)
      zb[CtaCtx<T>::zt((int)mk_pos(pv[j], N))] = apply_sign<T>(c.sign, j, x[j]);
  } else if constexpr (sizeof(T) == 4) {
    // x[4q..4q+3] -> complex slots q (x_{4q}, x_{4q+2}) and L-1-q (x_{4q+3}, x_{4q+1})
    // of the Makhoul sequence (cs_common.cuh mk_pos), sign applied; 16-byte loads,
    // all of a thread's loads in flight before its stores
    const int L = (int)(N >> 1), nq = (int)(N >> 2);
    C2<T>* z = shp(c.Z);
    const uint32_t* sg = shp(c.sign);
    constexpr int UQ = 8;
    for (int q0 = threadIdx.x; q0 < nq; q0 += UQ * TS_THREADS) {
      float4 v[UQ];
#pragma unroll
      for (int u = 0; u < UQ; ++u) {
        const int q = q0 + u * TS_THREADS;
        if (q < nq) v[u] = *reinterpret_cast<const float4*>(x + 4 * q);
      }
#pragma unroll
      for (int u = 0; u < UQ; ++u) {
        const int q = q0 + u * TS_THREADS;
        if (q < nq) {
          const uint32_t w = sg[q >> 3] >> ((4 * q) & 31);
          const float a0 = (w & 1u) ? -v[u].x : v[u].x, a1 = (w & 2u) ? -v[u].y : v[u].y;
          const float a2 = (w & 4u) ? -v[u].z : v[u].z, a3 = (w & 8u) ? -v[u].w : v[u].w;
          z[swz<T>(q)] = mk<T>(a0, a2);
          z[swz<T>(L - 1 - q)] = mk<T>(a3, a1);
        }
      }
    }
  } else {
    T* zb = reinterpret_cast<T*>(c.Z);
    for (int j = c.gtid; j < (int)N; j += c.gnthr)
      zb[CtaCtx<T>::zt((int)mk_pos(j, N))] = apply_sign<T>(c.sign, j, x[j]);
  }
  __syncthreads();
  c.template sandwich<MID_FWD, false>(nullptr, nullptr, Y + b * c.M);
  }
}

template <typename T>
__global__ void __launch_bounds__(TS_THREADS, sizeof(T) == 4 ? 2 : 1) k_s_adjoint(OpMeta meta, SLayout lay, const T* __restrict__ Yin,
                                                   T* __restrict__ X, T* __restrict__ Gws, int64_t B) {
  extern __shared__ __align__(16) char smem[];
  __shared__ CtaCtx<T> c;   // persistent, as k_s_apply
  init_cta_ctx<T>(c, smem, lay, meta, blockIdx.x);
  const int64_t N = c.N;
  for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
    if (b != blockIdx.x) {
      __syncthreads();
      cta_set_instance<T>(c, smem, meta, b);
    }
    c.y = Yin + b * c.M;
    if (threadIdx.x == 0 && b + gridDim.x < B && ((c.M * sizeof(T)) & 15) == 0)
      prefetch_l2(Yin + (b + gridDim.x) * c.M, (uint32_t)(c.M * sizeof(T)));   // the next instance's y
      s_prefetch_meta(meta, b + gridDim.x);
    if (c.psi) c.G = Gws + b * c.N;
    c.RES(nullptr);  // A^T y (x = 0)
    T* x = X + b * N;
    if constexpr (sizeof(T) == 4) {
      if (!c.pinv && !c.psi && (N & 3) == 0) {
        // the apply's scatter mirrored: x[4q..4q+3] from complex slots q (x_{4q}, x_{4q+2})
        // and L-1-q (x_{4q+3}, x_{4q+1}) of the Makhoul sequence, one sign nibble, one
        // 16-byte store per four outputs (the per-element map cost 45 % of the kernel's
        // instructions)
        const int L = (int)(N >> 1), nq = (int)(N >> 2);
        const C2<T>* z = shp(c.Z);
        const uint32_t* sg = shp(c.sign);
        for (int q = threadIdx.x; q < nq; q += TS_THREADS) {
          const C2<T> a = z[swz<T>(q)], bb = z[swz<T>(L - 1 - q)];
          const uint32_t w = sg[q >> 3] >> ((4 * q) & 31);
          float4 o;
          o.x = (w & 1u) ? -a.x : a.x;
          o.y = (w & 2u) ? -bb.y : bb.y;
          o.z = (w & 4u) ? -a.y : a.y;
          o.w = (w & 8u) ? -bb.x : bb.x;
          *reinterpret_cast<float4*>(x + 4 * q) = o;
        }
        continue;
      }
    }
    for (int64_t j = c.gtid; j < N; j += c.gnthr) x[j] = c.c_at(j);
  }
}

template <typename T> struct SRecArgs {
  OpMeta meta;
  SLayout lay;
  Params P;
  int ucap;
  const T* Y;
  T* vals;
  int32_t* supp;
  cs_report* reps;
  T* c0ws;  // [B][2][N]: A^T y (Makhoul order), then the Psi-mode scratch G
  // refinement launch (cs_options.refine_fp64): block s recovers operator instance bmap[s]
  // from the staged y row s into output slot s; blocks s >= *bcount exit.  Null: identity.
  const int* bmap = nullptr;
  const int* bcount = nullptr;
};

template <typename T>
__global__ void __launch_bounds__(TS_THREADS, sizeof(T) == 4 ? 2 : 1) k_s_recover(SRecArgs<T> a) {
  extern __shared__ __align__(16) char smem[];
  const int64_t b = blockIdx.x;   // output / workspace / y slot
  int64_t inst = b;                // operator instance
  if (a.bmap) {
    if (b >= *a.bcount) return;    // uniform over the block
    inst = a.bmap[b];
  }
  __shared__ CtaCtx<T> c;
  __shared__ Params P;
  init_cta_ctx<T>(c, smem, a.lay, a.meta, inst);
  P = a.P;   // every thread the same value; ordered before use by the barriers below
  // row selection in the fused pass's unit order for the CG loop's H (sandwich_cta.cuh sw_fused)
  sw_build_usel<T>(c.log2L, reinterpret_cast<uint32_t*>(smem + s_fixed<T>(a.meta.N).usel), c.rowmask);
  __syncthreads();
  c.y = a.Y + b * c.M;
  c.c0 = a.c0ws + b * 2 * c.N;
  c.G = c.c0 + c.N;
  // non-finite y check
  int bad = 0;
  for (int64_t m = c.gtid; m < c.M; m += c.gnthr) bad |= !isfinite((double)c.y[m]);
  unsigned pre = __syncthreads_or(bad) ? CS_DEV_NONFINITE_Y : 0u;
  Bufs<T> B;
  const SLayout& L = a.lay;
  B.S = reinterpret_cast<int*>(smem + L.S);
  B.S2 = reinterpret_cast<int*>(smem + L.S2);
  B.U = reinterpret_cast<int*>(smem + L.U);
  B.x = reinterpret_cast<T*>(smem + L.x);
  B.x2 = reinterpret_cast<T*>(smem + L.x2);
  B.xU = reinterpret_cast<T*>(smem + L.xU);
  B.r = reinterpret_cast<T*>(smem + L.r);
  B.d = reinterpret_cast<T*>(smem + L.d);
  B.q = reinterpret_cast<T*>(smem + L.q);
  B.b = reinterpret_cast<T*>(smem + L.b);
  B.Sbits = reinterpret_cast<uint32_t*>(smem + L.Sbits);
  B.Ubits = reinterpret_cast<uint32_t*>(smem + L.Ubits);
  B.Pbits = reinterpret_cast<uint32_t*>(smem + L.Pbits);
  run_pursuit<CtaCtx<T>, T>(c, P, B, a.vals + b * a.P.K, a.supp + b * a.P.K, a.reps + b, pre);
}

// Diagnostics / test hook: the CTA context's top-K selection (select.cuh topk_bits) on a
// caller's value array: out_bits = the K largest |vals| (ties -> lowest index).
// mode 0: two-pass path (radix fallback on overflow), mode 1: radix path only.
template <typename T>
__global__ void __launch_bounds__(TS_THREADS, 1) k_s_diag_topk(SLayout lay, const T* vals, int n, int K, int mode,
                                                              uint32_t* out_bits) {
  extern __shared__ __align__(16) char smem[];
  CtaCtx<T> c;
  c.redd = reinterpret_cast<double*>(smem + lay.redd);
  c.redi = reinterpret_cast<int64_t*>(smem + lay.redi);
  c.redk = reinterpret_cast<typename CtaCtx<T>::Key*>(smem + lay.redk);
  c.hist = reinterpret_cast<unsigned*>(smem + lay.hist);
  c.pick = reinterpret_cast<int64_t*>(smem + lay.pick);
  c.h1 = reinterpret_cast<unsigned*>(smem + lay.h1);
  c.ckey = reinterpret_cast<typename CtaCtx<T>::Key*>(smem + lay.ckey);
  c.cidx = reinterpret_cast<int*>(smem + lay.cidx);
  c.ccnt = reinterpret_cast<int*>(smem + lay.ccnt);
  for (int w = 0; w < SW_NT / 32; ++w) c.rbank_w[w] = 0;
  __syncthreads();
  topk_bits(c, (int64_t)n, (int64_t)K, [vals](int64_t i) { return full_key(vals[i]); }, out_bits, mode == 0);
}

// ------------------------------------------------------------ host side ----
// Declared everywhere; defined (and explicitly instantiated) in k_s_f32.cu / k_s_f64.cu.
template <typename T>
cs_status s_diag_topk_launch(const T* vals, int n, int K, int mode, uint32_t* out, cudaStream_t st,
                             std::atomic<uint64_t>& launches, std::string& err);
template <typename T>
cs_status s_apply_launch(const OpMeta& m, int64_t B, const T* in, T* out, bool adjoint, T* gws, cudaStream_t st,
                         std::atomic<uint64_t>& launches, std::string& err);
template <typename T>
cs_status s_recover_launch(const SRecArgs<T>& a, int64_t B, cudaStream_t st, std::atomic<uint64_t>& launches,
                           std::string& err);

#ifdef CS_TIER_S_IMPL
inline cs_status s_attr(const void* fn, int64_t bytes, std::string& err) {
  // the dynamic shared-memory limit of a kernel only ever grows, set when a launch needs more
  // (the driver calls cost host microseconds per launch)
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int64_t> limit;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  int64_t& lim = limit[std::make_pair(dev, fn)];
  if (bytes <= lim) return CS_OK;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (e != cudaSuccess) { err = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e); return CS_ERR_CUDA; }
  lim = bytes;
  return CS_OK;
}
inline cs_status s_launched(std::atomic<uint64_t>& launches, std::string& err) {
  launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { err = std::string("kernel launch: ") + cudaGetErrorString(e); return CS_ERR_CUDA; }
  return CS_OK;
}
template <typename T>
cs_status s_apply_launch(const OpMeta& m, int64_t B, const T* in, T* out, bool adjoint, T* gws, cudaStream_t st,
                         std::atomic<uint64_t>& launches, std::string& err) {
  SLayout lay = s_layout<T>(m.N, 0, 0, false);
  const void* fn = adjoint ? (const void*)k_s_adjoint<T> : (const void*)k_s_apply<T>;
  if (cs_status s = s_attr(fn, lay.bytes, err)) return s;
  // persistent grid: two CTAs per SM (the occupancy of the 512-thread, ~110 KB CTA)
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)std::min<int64_t>(B, 2 * (int64_t)nsm);
  if (adjoint) k_s_adjoint<T><<<grid, lay.nthreads, lay.bytes, st>>>(m, lay, in, out, gws, B);
  else k_s_apply<T><<<grid, lay.nthreads, lay.bytes, st>>>(m, lay, in, out, gws, B);
  return s_launched(launches, err);
}
template <typename T>
cs_status s_diag_topk_launch(const T* vals, int n, int K, int mode, uint32_t* out, cudaStream_t st,
                             std::atomic<uint64_t>& launches, std::string& err) {
  SLayout lay = s_layout<T>(16384, 0, 0, false);
  if (cs_status s = s_attr((const void*)k_s_diag_topk<T>, lay.bytes, err)) return s;
  k_s_diag_topk<T><<<1, lay.nthreads, lay.bytes, st>>>(lay, vals, n, K, mode, out);
  return s_launched(launches, err);
}
template <typename T>
cs_status s_recover_launch(const SRecArgs<T>& a, int64_t B, cudaStream_t st, std::atomic<uint64_t>& launches,
                           std::string& err) {
  if (cs_status s = s_attr((const void*)k_s_recover<T>, a.lay.bytes, err)) return s;
  k_s_recover<T><<<(unsigned)B, a.lay.nthreads, a.lay.bytes, st>>>(a);
  return s_launched(launches, err);
}
#endif

}  // namespace cs
