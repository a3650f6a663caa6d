// abi.cu — the extern "C" boundary of libcsgpu.so (declared in include/cs.h).
//
// Host-side validation, workspace sizing, operator metadata construction and
// tier dispatch:
//   Tier S (N <= 16384 and the per-problem working set fits in shared memory):
//     one thread block per problem (tier_s.cuh);
//   Tier L (larger N): one cooperative persistent grid per problem with a
//     four-step FFT over L2-resident scratch (tier_l.cuh).
#include <dlfcn.h>
#include <nccl.h>  // types and prototypes only: libnccl is loaded at run time (cs_comm_init)

#include <algorithm>
#include <vector>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "tier_l.cuh"
#include "tier_s.cuh"

using namespace cs;

struct cs_operator {
  int64_t N, M, B, nw;
  uint32_t* meta;   // device: [B][stride] (meta_stride)
  int* errflag;     // device int in the meta tail
  int32_t* perm;    // device: [B][pi N][pi^-1 N] after the meta tail (Eq.(7) randomizer), or null
  int psi;          // dictionary Psi: 0 = I, 1 = C_N (R35)
  int fkind;        // F: 0 = DCT-II, 1 = partial Fourier (R36)
  int64_t Mr;       // metadata rows (= M for the DCT; frequencies = M / 2 for the DFT)
  uint32_t* full;   // Psi mode: one all-rows instance (stride meta_stride(N, N)), or null
  int device;
  double2* tw;      // device, owned: the grid tier's twiddle tables (tier_l.cuh l_tw_off)
};

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

cs_status fail(cs_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}
cs_status cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return CS_ERR_CUDA;
}
#define CS_CUDA(call)                                   \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)
#define CS_LAUNCHED()                                               \
  do {                                                              \
    g_launches.fetch_add(1, std::memory_order_relaxed);             \
    cudaError_t e_ = cudaGetLastError();                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, "kernel launch");   \
  } while (0)

bool pow2(int64_t n) { return n > 0 && (n & (n - 1)) == 0; }

cs_status check_N(int64_t N) {
  if (!pow2(N) || N < 8 || N > ((int64_t)1 << 25))
    return fail(CS_ERR_UNSUPPORTED, "N must be a power of two in [8, 2^25]");
  return CS_OK;
}

cs_status check_device() {
  int dev;
  CS_CUDA(cudaGetDevice(&dev));
  int major = 0;
  CS_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  if (major != 10) return fail(CS_ERR_UNSUPPORTED, "libcsgpu is built for sm_100a (B200)");
  return CS_OK;
}

int64_t ucap_of(int alg, int K, int l) {
  if (alg == CS_SP) return 2 * (int64_t)K;
  if (alg == CS_OMPR) return (int64_t)K + (l > 0 ? l : 1);
  if (alg == CS_COSAMP) return 3 * (int64_t)K;
  return K;
}

template <typename T> bool tier_s_fits(int64_t N, int K, int64_t ucap, bool pursuit) {
  if (N > TIER_S_MAX_N) return false;
  SLayout s = s_layout<T>(N, K, (int)ucap, pursuit);
  return s.bytes <= 227 * 1024;
}

// bit position of DCT index k in the stored row mask: natural for Tier S, the
// four-step transposed order for Tier L (tier_s.cuh OpMeta)
struct TPos {
  int s1, tsh;
  __host__ __device__ int64_t operator()(int64_t k) const {
    return ((k & ((int64_t(1) << s1) - 1)) << tsh) | (k >> s1);
  }
};
TPos tpos_of(int64_t N) {  // the four-step's transposed order (Tier L geometry of N)
  const LGeom g = l_geom(N);
  return TPos{ilog2(g.L1), ilog2(2 * g.L2)};
}

// natural_off >= 0: also set the natural-order bit (Tier S); toff: transposed mask (Tier L)
__global__ void k_rows_mask(int64_t N, int64_t M, int64_t B, int64_t nw, int64_t stride, int64_t natural_off,
                            int64_t toff, TPos tp, const int32_t* rows, const uint32_t* sign_in, uint32_t* meta,
                            int* err) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < B * nw) {  // copy sign words
    int64_t b = i / nw, w = i % nw;
    meta[b * stride + w] = sign_in ? sign_in[b * nw + w] : 0u;
  }
  if (i >= B * M) return;
  int64_t b = i / M, m = i % M;
  int32_t r = rows[i];
  bool ok = (r >= 0) && (r < N) && (m == 0 || rows[i - 1] < r);
  if (!ok) { atomicOr(err, 1); return; }
  if (natural_off >= 0) atomicOr(&meta[b * stride + natural_off + (r >> 5)], 1u << (r & 31));
  const int64_t t = tp(r);
  atomicOr(&meta[b * stride + toff + (t >> 5)], 1u << (t & 31));
}

// Eq.(7) randomizer: copy pi, build pi^-1 (pre-filled with -1); err |= 2 unless pi is a
// permutation of [0, N) in every instance
__global__ void k_perm_setup(int64_t N, int64_t B, const int32_t* pin, int32_t* perm, int* err) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= B * N) return;
  const int64_t b = i / N, k = i % N;
  const int32_t v = pin[i];
  perm[b * 2 * N + k] = v;
  if (v < 0 || v >= N) { atomicOr(err, 2); return; }
  if (atomicExch(&perm[b * 2 * N + N + v], (int32_t)k) != -1) atomicOr(err, 2);
}

__global__ void k_iota(int64_t n, int32_t* out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = (int32_t)i;
}

// partial Fourier: rows are frequencies in [1, N/2 - 1] (err bit 4)
__global__ void k_freq_check(int64_t N, int64_t n, const int32_t* f, int* err) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n && (f[i] < 1 || f[i] > N / 2 - 1)) atomicOr(err, 4);
}

// Partial Fourier (R36): the plain packing z_m = u_{2m} + i u_{2m+1} as an effective
// permutation of the Makhoul machinery: position of x_j = pi^-1(j) = mk_pos(pinv_eff[j]), so
// pinv_eff[j] = mk_nat(pi^-1(j)) and pm_eff[mk_nat(i)] = pi(i) (pi = identity without a
// randomizer).  err |= 2 unless pi is a permutation.
__global__ void k_perm_dft(int64_t N, int64_t B, const int32_t* pin, int32_t* perm, int* err) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= B * N) return;
  const int64_t b = g / N, i = g % N;
  const int32_t j = pin ? pin[g] : (int32_t)i;
  if (j < 0 || j >= N) { atomicOr(err, 2); return; }
  const int32_t mi = (int32_t)((2 * i < N) ? 2 * i : 2 * (N - 1 - i) + 1);  // mk_nat(i)
  perm[b * 2 * N + mi] = j;
  if (atomicExch(&perm[b * 2 * N + N + j], mi) != -1) atomicOr(err, 2);
}

// Tier L: tperm[rank of row m in the transposed order] = m
__global__ void k_rows_tperm(int64_t N, int64_t M, int64_t B, int64_t nw, int64_t stride, int64_t toff, TPos tp,
                             const int32_t* rows, uint32_t* meta) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= B * M) return;
  int64_t b = i / M, m = i % M;
  if (rows[i] < 0 || rows[i] >= N) return;  // invalid rows: reported by k_rows_mask
  const uint32_t* mask = meta + b * stride + toff;
  const int32_t* pre = reinterpret_cast<const int32_t*>(meta + b * stride + toff + nw);
  int32_t* perm = reinterpret_cast<int32_t*>(meta + b * stride + toff + 2 * nw);
  const int64_t t = tp(rows[i]);
  const uint32_t w = mask[t >> 5];
  const int32_t rank = pre[t >> 5] + __popc((t & 31) ? (w & ((1u << (t & 31)) - 1u)) : 0u);
  perm[rank] = (int32_t)m;
}

// exclusive prefix of popcounts per instance: one block per instance
__global__ void k_rows_prefix(int64_t nw, int64_t stride, int64_t mask_off, uint32_t* meta) {
  __shared__ int32_t wsum[32];
  __shared__ int32_t carry;
  const int64_t b = blockIdx.x;
  const uint32_t* mask = meta + b * stride + mask_off;
  int32_t* pre = reinterpret_cast<int32_t*>(meta + b * stride + mask_off + nw);
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  for (int64_t base = 0; base < nw; base += blockDim.x) {
    int64_t w = base + threadIdx.x;
    int32_t v = (w < nw) ? __popc(mask[w]) : 0;
    int32_t inc = v;
    for (int o = 1; o < 32; o <<= 1) {
      int32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    int32_t off = carry;
    int32_t tot = 0;
    for (int k = 0; k < nwarp; ++k) {
      if (k < warp) off += wsum[k];
      tot += wsum[k];
    }
    if (w < nw) pre[w] = off + inc - v;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
}


// Per-instance metadata (words): [sign nw] then, for N <= 16384 only, the natural-order
// [row mask nw][prefix nw] of Tier S; then for every N the Tier L transposed
// [row mask nw][prefix nw][tperm M] (Tier L also serves small N when Tier S's shared
// memory cannot hold the pursuit, e.g. fp64 with a large K).
int64_t meta_toff(int64_t N) {
  const int64_t nw = (N + 31) / 32;
  return N > TIER_S_MAX_N ? nw : 3 * nw;
}
int64_t meta_stride(int64_t N, int64_t M) {
  const int64_t nw = (N + 31) / 32;
  return meta_toff(N) + 2 * nw + M;
}

OpMeta meta_of(const cs_operator* op) {
  OpMeta m;
  m.base = op->meta;
  m.N = op->N;
  m.M = op->M;
  m.Mr = op->Mr;
  m.fkind = op->fkind;
  m.nw = op->nw;
  m.stride = meta_stride(op->N, op->Mr);
  m.toff = meta_toff(op->N);
  m.perm = op->perm;
  m.psi = op->psi;
  m.full = op->full;
  m.tw = op->tw;
  return m;
}

Params make_params(int alg, int32_t K, double tol, const cs_options* o) {
  Params P;
  P.K = K;
  P.alg = alg;
  P.tol = tol;
  P.max_outer = o ? o->max_outer : 0;
  P.cg_cap = o ? o->cg_max_iters : 0;
  P.ompr_l = (o && o->ompr_l > 0) ? o->ompr_l : 1;
  P.eta = (o && o->ompr_eta > 0) ? (double)o->ompr_eta : 1.0;
  return P;
}

template <typename T>
cs_status apply_impl(const cs_operator* op, const T* x, T* y, void* ws, size_t ws_bytes,
                     cudaStream_t st, bool adjoint) {
  if (!op) return fail(CS_ERR_INVALID_ARG, "null operator");
  if (!x || !y) return fail(CS_ERR_INVALID_ARG, "null vector");
  if (cs_status s = check_device()) return s;
  if (op->N <= TIER_S_MAX_N) {
    if (op->psi && (!ws || ws_bytes < (size_t)(op->B * op->N) * sizeof(T)))
      return fail(CS_ERR_WORKSPACE, "workspace too small (Psi = DCT needs batch * N elements)");
    return s_apply_launch<T>(meta_of(op), op->B, x, y, adjoint, reinterpret_cast<T*>(ws), st, g_launches,
                             g_last_error);
  }
  return tier_l_apply<T>(meta_of(op), op->B, x, y, ws, ws_bytes, st, adjoint, g_launches,
                         g_last_error);
}

// ---- mixed precision (cs_options.refine_fp64): fp32 results below the fp32
// resolution floor are recovered again in fp64 on the CTA tier
struct RefineWs {
  int* count;           // [1]
  int* list;            // [cap] problem indices
  double* y64;          // [cap][M]
  double* c0;           // [cap][2][N]
  double* vals;         // [cap][K]
  int32_t* supp;        // [cap][K]
  cs_report* reps;      // [cap]
  size_t bytes;
};
RefineWs refine_ws(char* base, int64_t N, int64_t M, int32_t K, int64_t B) {
  RefineWs r{};
  const int64_t cap = std::min<int64_t>(B, CS_REFINE_CAP);
  int64_t o = 0;
  auto take = [&](int64_t b) { int64_t at = o; o = align_up(o + b, 256); return base ? base + at : nullptr; };
  r.count = reinterpret_cast<int*>(take(16));
  r.list = reinterpret_cast<int*>(take(cap * 4));
  r.y64 = reinterpret_cast<double*>(take(cap * M * 8));
  r.c0 = reinterpret_cast<double*>(take(cap * 2 * N * 8));
  r.vals = reinterpret_cast<double*>(take(cap * K * 8));
  r.supp = reinterpret_cast<int32_t*>(take(cap * K * 4));
  r.reps = reinterpret_cast<cs_report*>(take(cap * (int64_t)sizeof(cs_report)));
  r.bytes = (size_t)o;
  return r;
}
// one warp per problem: flag min |x_i| < CS_REFINE_FLOOR ||x|| (finite y only), take a slot,
// stage y in fp64
__global__ void k_refine_select(int64_t B, int64_t M, int32_t K, const float* Y, const float* vals,
                                cs_report* reps, int cap, int* count, int* list, double* y64) {
  const int lane = threadIdx.x & 31;
  const int64_t b = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= B) return;
  const float* v = vals + b * K;
  double ss = 0, mn = 1e300;
  for (int i = lane; i < K; i += 32) {
    const double a = fabs((double)v[i]);
    ss += a * a;
    mn = fmin(mn, a);
  }
  for (int o = 16; o > 0; o >>= 1) {
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  }
  const bool flag = !(reps[b].status & CS_DEV_NONFINITE_Y) && mn < CS_REFINE_FLOOR * sqrt(ss);
  if (!flag) return;
  int slot = 0;
  if (lane == 0) slot = atomicAdd(count, 1);
  slot = __shfl_sync(0xffffffffu, slot, 0);
  if (slot >= cap) {
    if (lane == 0) reps[b].status |= CS_DEV_NOT_REFINED;
    return;
  }
  if (lane == 0) list[slot] = (int)b;
  for (int64_t m = lane; m < M; m += 32) y64[slot * M + m] = (double)Y[b * M + m];
}
// write the fp64 results over the fp32 ones
__global__ void k_refine_merge(int32_t K, int cap, const int* count, const int* list, const double* v64,
                               const int32_t* s64, const cs_report* r64, float* vals, int32_t* supp,
                               cs_report* reps) {
  const int s = blockIdx.x;
  if (s >= min(*count, cap)) return;
  const int64_t b = list[s];
  for (int i = threadIdx.x; i < K; i += blockDim.x) {
    vals[b * K + i] = (float)v64[(int64_t)s * K + i];
    supp[b * K + i] = s64[(int64_t)s * K + i];
  }
  if (threadIdx.x == 0) {
    cs_report r = r64[s];
    r.status |= CS_DEV_REFINED_FP64;
    reps[b] = r;
  }
}
bool refine_applies(int precision, const cs_options* opts, int64_t N, int32_t K, int64_t ucap) {
  return precision == 0 && opts && opts->refine_fp64 && tier_s_fits<float>(N, K, ucap, true) &&
         tier_s_fits<double>(N, K, ucap, true);
}

// the mixed-precision pass over a batch whose fp32 results are on the device (or queued on
// st): flag the problems below the fp32 floor, recover them again in fp64 on the CTA tier and
// merge the fp64 results over the fp32 ones. ws = the recovery workspace (the fp32 pass's
// B * 2N floats first, the refinement's area after them, cs_workspace_bytes with refine_fp64).
cs_status refine_launch(const cs_operator* op, const Params& P, int64_t ucap, const float* Y, int64_t B,
                        float* vals, int32_t* supp, cs_report* reps, char* ws, cudaStream_t st) {
  const int64_t N = op->N, M = op->M;
  const int32_t K = P.K;
  char* rb = ws + align_up(B * 2 * N * 4, 256);
  RefineWs r = refine_ws(rb, N, M, K, B);
  const int cap = (int)std::min<int64_t>(B, CS_REFINE_CAP);
  CS_CUDA(cudaMemsetAsync(r.count, 0, sizeof(int), st));
  k_refine_select<<<(unsigned)((B + 7) / 8), 256, 0, st>>>(B, M, K, Y, vals, reps, cap, r.count, r.list, r.y64);
  CS_LAUNCHED();
  SRecArgs<double> d;
  d.meta = meta_of(op);
  d.lay = s_layout<double>(N, K, (int)ucap, true);
  d.P = P;
  d.P.tol = P.tol < 1e-12 ? P.tol : 1e-12;   // the fp64 path's tolerance (R7)
  d.ucap = (int)ucap;
  d.Y = r.y64;
  d.vals = r.vals;
  d.supp = r.supp;
  d.reps = r.reps;
  d.c0ws = r.c0;
  d.bmap = r.list;
  d.bcount = r.count;
  if (cs_status s = s_recover_launch<double>(d, cap, st, g_launches, g_last_error)) return s;
  k_refine_merge<<<(unsigned)cap, 256, 0, st>>>(K, cap, r.count, r.list, r.vals, r.supp, r.reps, vals, supp, reps);
  CS_LAUNCHED();
  return CS_OK;
}

template <typename T>
cs_status recover_impl(const cs_operator* op, int alg, const T* Y, int64_t B, int64_t M, int64_t N,
                       int32_t K, double tol, const cs_options* opts, T* vals, int32_t* supp,
                       cs_report* reps, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (!op) return fail(CS_ERR_INVALID_ARG, "null operator");
  if (!Y || !vals || !supp || !reps) return fail(CS_ERR_INVALID_ARG, "null pointer argument");
  if (alg < CS_OMP || alg > CS_COSAMP) return fail(CS_ERR_INVALID_ARG, "unknown algorithm");
  if (cs_status s = check_N(N)) return s;
  if (N != op->N || M != op->M) return fail(CS_ERR_INVALID_ARG, "M/N do not match the operator");
  if (B < 1 || B > op->B) return fail(CS_ERR_INVALID_ARG, "batch exceeds operator instances");
  if (!(tol >= 0)) return fail(CS_ERR_INVALID_ARG, "tol must be >= 0");
  if (opts) {
    for (int i = 0; i < 3; ++i)
      if (opts->reserved[i]) return fail(CS_ERR_INVALID_ARG, "cs_options.reserved must be zero");
    if (opts->refine_fp64 < 0 || opts->refine_fp64 > 1) return fail(CS_ERR_INVALID_ARG, "refine_fp64 must be 0 or 1");
    if (opts->max_outer < 0 || opts->cg_max_iters < 0 || opts->ompr_l < 0 || opts->ompr_eta < 0)
      return fail(CS_ERR_INVALID_ARG, "negative option");
  }
  const int l = (opts && opts->ompr_l > 0) ? opts->ompr_l : 1;
  if (K < 1 || (int64_t)K > N / 2) return fail(CS_ERR_INVALID_ARG, "K must be in [1, N/2]");
  if (alg == CS_OMP && K > M) return fail(CS_ERR_INVALID_ARG, "OMP needs K <= M");
  if (alg == CS_SP && 2 * (int64_t)K > M) return fail(CS_ERR_INVALID_ARG, "SP needs 2K <= M");
  if (alg == CS_OMPR && (int64_t)K + l > M) return fail(CS_ERR_INVALID_ARG, "OMPR needs K + l <= M");
  if (alg == CS_COSAMP && 3 * (int64_t)K > M) return fail(CS_ERR_INVALID_ARG, "CoSaMP needs 3K <= M");
  if (cs_status s = check_device()) return s;
  size_t need = 0;
  const int prec = sizeof(T) == 8 ? 1 : 0;
  if (cs_status s = cs_workspace_bytes(alg, N, M, K, B, prec, opts, &need)) return s;
  if (!ws || ws_bytes < need) return fail(CS_ERR_WORKSPACE, "workspace too small");
  Params P = make_params(alg, K, tol, opts);
  const int64_t ucap = ucap_of(alg, K, l);
  const bool fits_s = tier_s_fits<T>(N, K, ucap, true);
  if (fits_s) {
    SRecArgs<T> a;
    a.meta = meta_of(op);
    a.lay = s_layout<T>(N, K, (int)ucap, true);
    a.P = P;
    a.ucap = (int)ucap;
    a.Y = Y;
    a.vals = vals;
    a.supp = supp;
    a.reps = reps;
    a.c0ws = reinterpret_cast<T*>(ws);
    if (cs_status s = s_recover_launch<T>(a, B, st, g_launches, g_last_error)) return s;
    if constexpr (sizeof(T) == 4) {
      if (refine_applies(0, opts, N, K, ucap))
        if (cs_status s = refine_launch(op, P, ucap, Y, B, vals, supp, reps, reinterpret_cast<char*>(ws), st))
          return s;
    }
    return CS_OK;
  }
  return tier_l_recover<T>(meta_of(op), P, (int)ucap, Y, B, vals, supp, reps, ws, ws_bytes, st,
                           g_launches, g_last_error);
}

// ---------------------------------------------------------------- host-buffer pipeline
// Streams and events of the host-buffer entry points, created once per device.
struct HostPipe {
  cudaStream_t s_in = nullptr, s_out = nullptr, s_comp = nullptr;
  cudaEvent_t ev[2][64] = {};
  cudaEvent_t fin = nullptr;
  bool ok = false;
  std::mutex enq;  // one host thread enqueues a pipeline at a time (the events are reused)
};
HostPipe& host_pipe(int dev) {
  static std::mutex mu;
  static std::map<int, HostPipe> pipes;   // keyed by device ordinal; references stay valid
  std::lock_guard<std::mutex> lock(mu);
  HostPipe& p = pipes[dev];
  if (!p.ok) {
    bool good = cudaStreamCreateWithFlags(&p.s_in, cudaStreamNonBlocking) == cudaSuccess &&
                cudaStreamCreateWithFlags(&p.s_out, cudaStreamNonBlocking) == cudaSuccess &&
                cudaStreamCreateWithFlags(&p.s_comp, cudaStreamNonBlocking) == cudaSuccess &&
                cudaEventCreateWithFlags(&p.fin, cudaEventDisableTiming) == cudaSuccess;
    for (int k = 0; k < 2 && good; ++k)
      for (int c = 0; c < 64 && good; ++c)
        good = cudaEventCreateWithFlags(&p.ev[k][c], cudaEventDisableTiming) == cudaSuccess;
    p.ok = good;
  }
  return p;
}

size_t staging_bytes(int64_t B, int64_t M, int32_t K, size_t es) {
  return (size_t)(align_up(B * M * (int64_t)es, 256) + align_up(B * K * (int64_t)es, 256) +
                  align_up(B * (int64_t)K * 4, 256) + align_up(B * (int64_t)sizeof(cs_report), 256));
}

// y (pinned host) -> device -> recover -> (support, values, reports) (pinned host), in chunks
// of whole waves on two alternating compute streams so that copies overlap recovery and a
// chunk's last wave overlaps the next chunk.
template <typename T>
cs_status recover_host_impl(const cs_operator* op, int alg, const T* hY, int64_t B, int64_t M, int64_t N,
                            int32_t K, double tol, const cs_options* opts, T* hvals, int32_t* hsupp,
                            cs_report* hreps, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (!op) return fail(CS_ERR_INVALID_ARG, "null operator");
  if (!hY || !hvals || !hsupp || !hreps) return fail(CS_ERR_INVALID_ARG, "null pointer argument");
  if (B < 1 || B > op->B) return fail(CS_ERR_INVALID_ARG, "batch exceeds operator instances");
  if (cs_status s = check_N(N)) return s;
  if (K < 1) return fail(CS_ERR_INVALID_ARG, "K must be >= 1");
  const int prec = sizeof(T) == 8 ? 1 : 0;
  // mixed precision (cs_options.refine_fp64): the chunks run plain fp32; the refinement runs
  // once over the whole batch after the last chunk (its workspace follows the chunks' fp32
  // areas, as in the device path), and the results are copied out after it
  const cs_options* opts_in = opts;
  const int l_in = (opts && opts->ompr_l > 0) ? opts->ompr_l : 1;
  const bool refine = sizeof(T) == 4 && refine_applies(0, opts, N, K, ucap_of(alg, K, l_in));
  if (opts && (opts->refine_fp64 < 0 || opts->refine_fp64 > 1))
    return fail(CS_ERR_INVALID_ARG, "refine_fp64 must be 0 or 1");
  cs_options o_norefine{};
  if (opts && opts->refine_fp64) {
    o_norefine = *opts;
    o_norefine.refine_fp64 = 0;
    opts = &o_norefine;
  }
  size_t need_rec = 0;
  if (cs_status s = cs_workspace_bytes(alg, N, M, K, B, prec, refine ? opts_in : opts, &need_rec)) return s;
  const size_t rec_al = (size_t)align_up((int64_t)need_rec, 256);
  if (!ws || ws_bytes < rec_al + staging_bytes(B, M, K, sizeof(T)))
    return fail(CS_ERR_WORKSPACE, "workspace too small");
  char* w = reinterpret_cast<char*>(ws);
  T* dY = reinterpret_cast<T*>(w + rec_al);
  T* dvals = reinterpret_cast<T*>(reinterpret_cast<char*>(dY) + align_up(B * M * (int64_t)sizeof(T), 256));
  int32_t* dsupp = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(dvals) + align_up(B * K * (int64_t)sizeof(T), 256));
  cs_report* dreps = reinterpret_cast<cs_report*>(reinterpret_cast<char*>(dsupp) + align_up(B * (int64_t)K * 4, 256));
  int dev = 0;
  CS_CUDA(cudaGetDevice(&dev));
  HostPipe& hp = host_pipe(dev);
  if (!hp.ok) return fail(CS_ERR_CUDA, "could not create the host-pipeline streams");
  // the streams and events are per device: concurrent callers enqueue one after the other
  // (cudaStreamWaitEvent binds each wait to the event's record at enqueue time)
  std::lock_guard<std::mutex> enqueue_lock(hp.enq);
  const int l = (opts && opts->ompr_l > 0) ? opts->ompr_l : 1;
  const bool tier_s = tier_s_fits<T>(N, K, ucap_of(alg, K, l), true);
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  // chunk = two waves of the Tier S recovery (two blocks per SM), enlarged so that a batch
  // never needs more than the 64 event pairs of the pipeline; Tier L: one chunk
  int64_t CH = tier_s ? std::max<int64_t>(1, (int64_t)4 * nsm) : B;
  CH = std::max<int64_t>(CH, (B + 63) / 64);
  const int64_t nch = (B + CH - 1) / CH;
  CS_CUDA(cudaEventRecord(hp.fin, st));             // order behind earlier work on the caller's stream
  CS_CUDA(cudaStreamWaitEvent(hp.s_in, hp.fin, 0));
  // on a failure after copies were queued, the caller's stream still waits for everything
  // already on the pipeline streams (so the caller can free its pinned buffers safely)
  auto drain = [&](cs_status s) {
    cudaStream_t ss[3] = {hp.s_in, hp.s_comp, hp.s_out};
    for (cudaStream_t x : ss)
      if (cudaEventRecord(hp.fin, x) == cudaSuccess) cudaStreamWaitEvent(st, hp.fin, 0);
    return s;
  };
#undef CS_CUDA
#define CS_CUDA(call)                                                   \
  do {                                                                  \
    cudaError_t e_ = (call);                                            \
    if (e_ != cudaSuccess) return drain(cuda_fail(e_, #call));          \
  } while (0)
  for (int64_t c = 0; c < nch; ++c) {
    const int64_t b0 = c * CH, cnt = std::min(CH, B - b0);
    CS_CUDA(cudaMemcpyAsync(dY + b0 * M, hY + b0 * M, (size_t)(cnt * M) * sizeof(T), cudaMemcpyHostToDevice,
                            hp.s_in));
    CS_CUDA(cudaEventRecord(hp.ev[0][c], hp.s_in));
    cudaStream_t sc = (c & 1) ? hp.s_comp : st;
    CS_CUDA(cudaStreamWaitEvent(sc, hp.ev[0][c], 0));
    cs_operator sub = *op;
    sub.meta = op->meta + b0 * meta_stride(op->N, op->Mr);
    if (op->perm) sub.perm = op->perm + b0 * 2 * N;
    sub.B = cnt;
    char* rws = tier_s ? w + (size_t)(b0 * 2 * N) * sizeof(T) : w;
    const size_t rws_bytes = tier_s ? (size_t)(cnt * 2 * N) * sizeof(T) : need_rec;
    if (cs_status s = recover_impl<T>(&sub, alg, dY + b0 * M, cnt, M, N, K, tol, opts, dvals + b0 * K,
                                      dsupp + b0 * K, dreps + b0, rws, rws_bytes, sc))
      return drain(s);
    if (refine) continue;   // copied out after the refinement
    CS_CUDA(cudaEventRecord(hp.ev[1][c], sc));
    CS_CUDA(cudaStreamWaitEvent(hp.s_out, hp.ev[1][c], 0));
    CS_CUDA(cudaMemcpyAsync(hsupp + b0 * K, dsupp + b0 * K, (size_t)(cnt * K) * 4, cudaMemcpyDeviceToHost,
                            hp.s_out));
    CS_CUDA(cudaMemcpyAsync(hvals + b0 * K, dvals + b0 * K, (size_t)(cnt * K) * sizeof(T),
                            cudaMemcpyDeviceToHost, hp.s_out));
    CS_CUDA(cudaMemcpyAsync(hreps + b0, dreps + b0, (size_t)cnt * sizeof(cs_report), cudaMemcpyDeviceToHost,
                            hp.s_out));
  }
  if constexpr (sizeof(T) == 4) {
    if (refine) {
      // st already follows the even chunks; make it follow the odd ones on s_comp too
      CS_CUDA(cudaEventRecord(hp.fin, hp.s_comp));
      CS_CUDA(cudaStreamWaitEvent(st, hp.fin, 0));
      const Params P = make_params(alg, K, tol, opts_in);
      if (cs_status s = refine_launch(op, P, ucap_of(alg, K, l_in), dY, B, dvals, dsupp, dreps, w, st))
        return drain(s);
      CS_CUDA(cudaEventRecord(hp.fin, st));
      CS_CUDA(cudaStreamWaitEvent(hp.s_out, hp.fin, 0));
      CS_CUDA(cudaMemcpyAsync(hsupp, dsupp, (size_t)(B * K) * 4, cudaMemcpyDeviceToHost, hp.s_out));
      CS_CUDA(cudaMemcpyAsync(hvals, dvals, (size_t)(B * K) * sizeof(T), cudaMemcpyDeviceToHost, hp.s_out));
      CS_CUDA(cudaMemcpyAsync(hreps, dreps, (size_t)B * sizeof(cs_report), cudaMemcpyDeviceToHost, hp.s_out));
    }
  }
  CS_CUDA(cudaEventRecord(hp.fin, hp.s_out));
  CS_CUDA(cudaStreamWaitEvent(st, hp.fin, 0));      // the caller's stream completes after everything
  return CS_OK;
#undef CS_CUDA
#define CS_CUDA(call)                                   \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)
}

}  // namespace

namespace {
// dense output: d_dense[b] = scatter(d_support[b], d_vals[b]) (support entries < 0 skipped)
template <typename T>
__global__ void k_dense(int64_t B, int64_t N, int32_t K, const int32_t* supp, const T* vals, T* dense) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= B * (int64_t)K) return;
  const int64_t b = i / K;
  const int32_t j = supp[i];
  if (j >= 0 && j < N) dense[b * N + j] = vals[i];
}
template <typename T>
cs_status dense_impl(int64_t B, int64_t N, int32_t K, const int32_t* supp, const T* vals, T* dense,
                     cudaStream_t st) {
  if (!supp || !vals || !dense) return fail(CS_ERR_INVALID_ARG, "null pointer argument");
  if (B < 1 || N < 1 || K < 1) return fail(CS_ERR_INVALID_ARG, "bad sizes");
  CS_CUDA(cudaMemsetAsync(dense, 0, (size_t)(B * N) * sizeof(T), st));
  k_dense<T><<<(unsigned)((B * K + 255) / 256), 256, 0, st>>>(B, N, K, supp, vals, dense);
  CS_LAUNCHED();
  return CS_OK;
}

// NCCL, resolved at run time (the torch process has usually loaded it already)
struct NcclApi {
  bool ok = false;
  decltype(&ncclCommInitAll) init_all = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) err = nullptr;
};
const NcclApi& nccl_api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    a.init_all = reinterpret_cast<decltype(&ncclCommInitAll)>(dlsym(h, "ncclCommInitAll"));
    a.destroy = reinterpret_cast<decltype(&ncclCommDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.send = reinterpret_cast<decltype(&ncclSend)>(dlsym(h, "ncclSend"));
    a.recv = reinterpret_cast<decltype(&ncclRecv)>(dlsym(h, "ncclRecv"));
    a.group_start = reinterpret_cast<decltype(&ncclGroupStart)>(dlsym(h, "ncclGroupStart"));
    a.group_end = reinterpret_cast<decltype(&ncclGroupEnd)>(dlsym(h, "ncclGroupEnd"));
    a.err = reinterpret_cast<decltype(&ncclGetErrorString)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.init_all && a.destroy && a.send && a.recv && a.group_start && a.group_end && a.err;
  });
  return a;
}
struct CsComm {
  std::vector<int> dev;
  std::vector<ncclComm_t> comms;
  std::vector<cudaStream_t> streams;
  std::vector<cudaEvent_t> ready;   // per device: the producers' point the gather waits for
};
}  // namespace

extern "C" {

size_t cs_operator_meta_bytes(int64_t N, int64_t M, int64_t batch) {
  (void)M;
  if (N <= 0 || batch <= 0) return 0;
  int64_t nw = (N + 31) / 32;
  (void)nw;
  return (size_t)(align_up(batch * meta_stride(N, M) * 4, 256) + 256);
}

size_t cs_operator_meta_bytes_ex(int64_t N, int64_t M, int64_t batch, int has_perm, int psi) {
  const size_t base = cs_operator_meta_bytes(N, M, batch);
  if (!base) return 0;
  size_t b = base;
  if (has_perm) b += (size_t)align_up(batch * 2 * N * 4, 256);
  if (psi) b += (size_t)align_up(meta_stride(N, N) * 4, 256) + (size_t)align_up(N * 4, 256);
  return b;
}

// M = metadata rows: DCT rows, or (fkind 1) partial-Fourier frequencies (2 measurements each)
static cs_status create_impl(int64_t N, int64_t M, int64_t batch, const uint32_t* d_sign_bits,
                             const int32_t* d_perm, const int32_t* d_rows, int psi, void* d_meta,
                             size_t meta_bytes, cs_stream_t stream, cs_operator** out, int fkind = 0) {
  if (!out) return fail(CS_ERR_INVALID_ARG, "out is null");
  *out = nullptr;
  if (cs_status s = check_N(N)) return s;
  if (fkind == 0 && (M < 1 || M > N)) return fail(CS_ERR_INVALID_ARG, "M must be in [1, N]");
  if (fkind == 1 && (M < 1 || M > N / 2 - 1)) return fail(CS_ERR_INVALID_ARG, "frequency count must be in [1, N/2 - 1]");
  if (batch < 1 || batch > (1 << 30)) return fail(CS_ERR_INVALID_ARG, "bad batch");
  if ((fkind == 0 && !d_sign_bits && !d_perm) || !d_rows || !d_meta) return fail(CS_ERR_INVALID_ARG, "null pointer argument");
  const bool has_perm = d_perm != nullptr || fkind == 1;
  const size_t need = cs_operator_meta_bytes_ex(N, M, batch, has_perm, psi);
  if (meta_bytes < need) return fail(CS_ERR_WORKSPACE, "meta buffer too small");
  if (cs_status s = check_device()) return s;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int64_t nw = (N + 31) / 32;
  uint32_t* meta = reinterpret_cast<uint32_t*>(d_meta);
  const int64_t stride = meta_stride(N, M);
  const TPos tp = tpos_of(N);
  int* err = reinterpret_cast<int*>(reinterpret_cast<char*>(d_meta) + align_up(batch * stride * 4, 256));
  const size_t base_bytes = cs_operator_meta_bytes(N, M, batch);
  CS_CUDA(cudaMemsetAsync(d_meta, 0, base_bytes, st));
  int32_t* perm = has_perm ? reinterpret_cast<int32_t*>(reinterpret_cast<char*>(d_meta) + base_bytes) : nullptr;
  if (perm) {
    CS_CUDA(cudaMemsetAsync(perm, 0xFF, (size_t)(batch * 2 * N) * 4, st));
    if (fkind == 1) k_perm_dft<<<(unsigned)((batch * N + 255) / 256), 256, 0, st>>>(N, batch, d_perm, perm, err);
    else k_perm_setup<<<(unsigned)((batch * N + 255) / 256), 256, 0, st>>>(N, batch, d_perm, perm, err);
    CS_LAUNCHED();
  }
  if (fkind == 1) {
    k_freq_check<<<(unsigned)((batch * M + 255) / 256), 256, 0, st>>>(N, batch * M, d_rows, err);
    CS_LAUNCHED();
  }
  const int64_t toff = meta_toff(N), natural = N > TIER_S_MAX_N ? -1 : nw;
  uint32_t* full = nullptr;
  if (psi) {
    // one all-rows instance (rows = 0..N-1, sigma = +1): the full DCT-II / DCT-III of the
    // dictionary on the grid tier (R35); its rows array stays after it
    char* fb = reinterpret_cast<char*>(d_meta) + base_bytes + (perm ? align_up(batch * 2 * N * 4, 256) : 0);
    full = reinterpret_cast<uint32_t*>(fb);
    const int64_t sf = meta_stride(N, N);
    int32_t* frows = reinterpret_cast<int32_t*>(fb + align_up(sf * 4, 256));
    CS_CUDA(cudaMemsetAsync(full, 0, (size_t)(sf * 4), st));
    k_iota<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(N, frows);
    CS_LAUNCHED();
    k_rows_mask<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(N, N, 1, nw, sf, natural, toff, tp, frows,
                                                             nullptr, full, err);
    CS_LAUNCHED();
    if (natural >= 0) {
      k_rows_prefix<<<1, 1024, 0, st>>>(nw, sf, natural, full);
      CS_LAUNCHED();
    }
    k_rows_prefix<<<1, 1024, 0, st>>>(nw, sf, toff, full);
    CS_LAUNCHED();
    k_rows_tperm<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(N, N, 1, nw, sf, toff, tp, frows, full);
    CS_LAUNCHED();
  }
  int64_t nthr = std::max(batch * M, batch * nw);
  k_rows_mask<<<(unsigned)((nthr + 255) / 256), 256, 0, st>>>(N, M, batch, nw, stride, natural, toff, tp, d_rows,
                                                           d_sign_bits, meta, err);
  CS_LAUNCHED();
  if (natural >= 0) {
    k_rows_prefix<<<(unsigned)batch, 1024, 0, st>>>(nw, stride, natural, meta);
    CS_LAUNCHED();
  }
  k_rows_prefix<<<(unsigned)batch, 1024, 0, st>>>(nw, stride, toff, meta);
  CS_LAUNCHED();
  k_rows_tperm<<<(unsigned)((batch * M + 255) / 256), 256, 0, st>>>(N, M, batch, nw, stride, toff, tp, d_rows, meta);
  CS_LAUNCHED();
  int herr = 0;
  CS_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st));
  CS_CUDA(cudaStreamSynchronize(st));
  if (herr & 1) return fail(CS_ERR_INVALID_ARG, "rows must be strictly increasing and in [0, N)");
  if (herr & 2) return fail(CS_ERR_INVALID_ARG, "perm must be a permutation of [0, N)");
  if (herr & 4) return fail(CS_ERR_INVALID_ARG, "frequencies must be in [1, N/2 - 1]");
  // the grid tier's twiddle tables, once per operator (small: ~2K complex fp64)
  double2* tw = nullptr;
  {
    const TwOff o = l_tw_off(N);
    CS_CUDA(cudaMalloc(&tw, (size_t)o.n * sizeof(double2)));
    k_l_tw_tables<<<(unsigned)((o.n + 255) / 256), 256, 0, st>>>(N, tw);
    CS_LAUNCHED();
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { cudaFree(tw); return cuda_fail(e, "twiddle tables"); }
  }
  cs_operator* op = new cs_operator;
  op->tw = tw;
  op->N = N;
  op->M = fkind == 1 ? 2 * M : M;
  op->Mr = M;
  op->fkind = fkind;
  op->B = batch;
  op->nw = nw;
  op->meta = meta;
  op->errflag = err;
  op->perm = perm;
  op->psi = psi;
  op->full = full;
  CS_CUDA(cudaGetDevice(&op->device));
  *out = op;
  return CS_OK;
}

cs_status cs_operator_create(int64_t N, int64_t M, int64_t batch, const uint32_t* d_sign_bits,
                             const int32_t* d_rows, void* d_meta, size_t meta_bytes,
                             cs_stream_t stream, cs_operator** out) {
  if (!d_sign_bits) {
    if (out) *out = nullptr;
    return fail(CS_ERR_INVALID_ARG, "null pointer argument");
  }
  return create_impl(N, M, batch, d_sign_bits, nullptr, d_rows, 0, d_meta, meta_bytes, stream, out);
}

size_t cs_operator_meta_bytes_perm(int64_t N, int64_t M, int64_t batch) {
  const size_t base = cs_operator_meta_bytes(N, M, batch);
  if (!base) return 0;
  return base + (size_t)align_up(batch * 2 * N * 4, 256);
}

cs_status cs_operator_create_perm(int64_t N, int64_t M, int64_t batch, const uint32_t* d_sign_bits,
                                  const int32_t* d_perm, const int32_t* d_rows, void* d_meta,
                                  size_t meta_bytes, cs_stream_t stream, cs_operator** out) {
  if (!d_perm) {
    if (out) *out = nullptr;
    return fail(CS_ERR_INVALID_ARG, "null pointer argument");
  }
  return create_impl(N, M, batch, d_sign_bits, d_perm, d_rows, 0, d_meta, meta_bytes, stream, out);
}

size_t cs_operator_meta_bytes_dft(int64_t N, int64_t n_freq, int64_t batch) {
  return cs_operator_meta_bytes_ex(N, n_freq, batch, 1, 0);
}

cs_status cs_operator_create_dft(int64_t N, int64_t n_freq, int64_t batch, const uint32_t* d_sign_bits,
                                 const int32_t* d_perm, const int32_t* d_freqs, void* d_meta,
                                 size_t meta_bytes, cs_stream_t stream, cs_operator** out) {
  return create_impl(N, n_freq, batch, d_sign_bits, d_perm, d_freqs, 0, d_meta, meta_bytes, stream, out, 1);
}

cs_status cs_operator_create_ex(int64_t N, int64_t M, int64_t batch, const uint32_t* d_sign_bits,
                                const int32_t* d_perm, const int32_t* d_rows, int psi, void* d_meta,
                                size_t meta_bytes, cs_stream_t stream, cs_operator** out) {
  if (out) *out = nullptr;
  if (psi != CS_PSI_IDENTITY && psi != CS_PSI_DCT) return fail(CS_ERR_INVALID_ARG, "psi must be CS_PSI_IDENTITY or CS_PSI_DCT");
  if (!d_sign_bits && !d_perm) return fail(CS_ERR_INVALID_ARG, "null pointer argument");
  return create_impl(N, M, batch, d_sign_bits, d_perm, d_rows, psi, d_meta, meta_bytes, stream, out);
}

cs_status cs_operator_destroy(cs_operator* op) {
  if (op && op->tw) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(op->device);
    cudaFree(op->tw);
    cudaSetDevice(cur);
  }
  delete op;
  return CS_OK;
}

cs_status cs_operator_info(const cs_operator* op, int64_t* N, int64_t* M, int64_t* batch) {
  if (!op) return fail(CS_ERR_INVALID_ARG, "null operator");
  if (N) *N = op->N;
  if (M) *M = op->M;
  if (batch) *batch = op->B;
  return CS_OK;
}

size_t cs_operator_ws_bytes(const cs_operator* op, int precision) {
  if (op && op->psi && op->N <= TIER_S_MAX_N) return (size_t)(op->B * op->N) * (precision ? 8 : 4);
  if (!op || op->N <= TIER_S_MAX_N) return 0;
  return precision ? tier_l_apply_ws_bytes<double>(op->N, op->M, op->B) : tier_l_apply_ws_bytes<float>(op->N, op->M, op->B);
}

cs_status cs_operator_apply(const cs_operator* op, const float* d_x, float* d_y, void* d_ws,
                            size_t ws_bytes, cs_stream_t stream) {
  return apply_impl<float>(op, d_x, d_y, d_ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream), false);
}
cs_status cs_operator_apply_f64(const cs_operator* op, const double* d_x, double* d_y, void* d_ws,
                                size_t ws_bytes, cs_stream_t stream) {
  return apply_impl<double>(op, d_x, d_y, d_ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream), false);
}
cs_status cs_operator_adjoint(const cs_operator* op, const float* d_y, float* d_x, void* d_ws,
                              size_t ws_bytes, cs_stream_t stream) {
  return apply_impl<float>(op, d_y, d_x, d_ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream), true);
}
cs_status cs_operator_adjoint_f64(const cs_operator* op, const double* d_y, double* d_x, void* d_ws,
                                  size_t ws_bytes, cs_stream_t stream) {
  return apply_impl<double>(op, d_y, d_x, d_ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream), true);
}

cs_status cs_workspace_bytes(int alg, int64_t N, int64_t M, int32_t K, int64_t batch, int precision,
                             const cs_options* opts, size_t* bytes) {
  if (!bytes) return fail(CS_ERR_INVALID_ARG, "bytes is null");
  if (cs_status s = check_N(N)) return s;
  if (K < 1 || batch < 1 || M < 1) return fail(CS_ERR_INVALID_ARG, "bad sizes");
  const int l = (opts && opts->ompr_l > 0) ? opts->ompr_l : 1;
  const int64_t ucap = ucap_of(alg, K, l);
  const bool dbl = precision != 0;
  bool s = dbl ? tier_s_fits<double>(N, K, ucap, true) : tier_s_fits<float>(N, K, ucap, true);
  if (s) {
    *bytes = (size_t)(batch * 2 * N * (dbl ? 8 : 4));   // A^T y and the Psi-mode scratch per problem
    if (refine_applies(precision, opts, N, K, ucap))
      *bytes = (size_t)align_up((int64_t)*bytes, 256) + refine_ws(nullptr, N, M, K, batch).bytes;
  } else {
    *bytes = dbl ? tier_l_recover_ws_bytes<double>(N, M, K, (int)ucap, batch)
                 : tier_l_recover_ws_bytes<float>(N, M, K, (int)ucap, batch);
  }
  return CS_OK;
}

cs_status cs_workspace_bytes_host(int alg, int64_t N, int64_t M, int32_t K, int64_t batch, int precision,
                                  const cs_options* opts, size_t* bytes) {
  size_t rec = 0;
  if (cs_status s = cs_workspace_bytes(alg, N, M, K, batch, precision, opts, &rec)) return s;
  *bytes = (size_t)align_up((int64_t)rec, 256) + staging_bytes(batch, M, K, precision ? 8 : 4);
  return CS_OK;
}
cs_status cs_recover_batched_host(const cs_operator* op, int alg, const float* h_Y, int64_t B, int64_t M,
                                  int64_t N, int32_t K, double tol, const cs_options* opts, float* h_vals,
                                  int32_t* h_support, cs_report* h_reports, void* d_ws, size_t ws_bytes,
                                  cs_stream_t stream) {
  return recover_host_impl<float>(op, alg, h_Y, B, M, N, K, tol, opts, h_vals, h_support, h_reports, d_ws,
                                  ws_bytes, reinterpret_cast<cudaStream_t>(stream));
}
cs_status cs_recover_batched_host_f64(const cs_operator* op, int alg, const double* h_Y, int64_t B, int64_t M,
                                      int64_t N, int32_t K, double tol, const cs_options* opts, double* h_vals,
                                      int32_t* h_support, cs_report* h_reports, void* d_ws, size_t ws_bytes,
                                      cs_stream_t stream) {
  return recover_host_impl<double>(op, alg, h_Y, B, M, N, K, tol, opts, h_vals, h_support, h_reports, d_ws,
                                   ws_bytes, reinterpret_cast<cudaStream_t>(stream));
}

cs_status cs_recover(const cs_operator* op, int alg, const float* d_y, int64_t M, int64_t N, int32_t K,
                     double tol, const cs_options* opts, float* d_vals, int32_t* d_support,
                     cs_report* d_report, void* d_ws, size_t ws_bytes, cs_stream_t stream) {
  return recover_impl<float>(op, alg, d_y, 1, M, N, K, tol, opts, d_vals, d_support, d_report, d_ws,
                             ws_bytes, reinterpret_cast<cudaStream_t>(stream));
}
cs_status cs_recover_f64(const cs_operator* op, int alg, const double* d_y, int64_t M, int64_t N,
                         int32_t K, double tol, const cs_options* opts, double* d_vals,
                         int32_t* d_support, cs_report* d_report, void* d_ws, size_t ws_bytes,
                         cs_stream_t stream) {
  return recover_impl<double>(op, alg, d_y, 1, M, N, K, tol, opts, d_vals, d_support, d_report, d_ws,
                              ws_bytes, reinterpret_cast<cudaStream_t>(stream));
}
cs_status cs_recover_batched(const cs_operator* op, int alg, const float* d_Y, int64_t B, int64_t M,
                             int64_t N, int32_t K, double tol, const cs_options* opts, float* d_vals,
                             int32_t* d_support, cs_report* d_reports, void* d_ws, size_t ws_bytes,
                             cs_stream_t stream) {
  return recover_impl<float>(op, alg, d_Y, B, M, N, K, tol, opts, d_vals, d_support, d_reports, d_ws,
                             ws_bytes, reinterpret_cast<cudaStream_t>(stream));
}
cs_status cs_recover_batched_f64(const cs_operator* op, int alg, const double* d_Y, int64_t B,
                                 int64_t M, int64_t N, int32_t K, double tol, const cs_options* opts,
                                 double* d_vals, int32_t* d_support, cs_report* d_reports, void* d_ws,
                                 size_t ws_bytes, cs_stream_t stream) {
  return recover_impl<double>(op, alg, d_Y, B, M, N, K, tol, opts, d_vals, d_support, d_reports, d_ws,
                              ws_bytes, reinterpret_cast<cudaStream_t>(stream));
}

const char* cs_status_string(cs_status s) {
  switch (s) {
    case CS_OK: return "CS_OK";
    case CS_ERR_INVALID_ARG: return "CS_ERR_INVALID_ARG";
    case CS_ERR_UNSUPPORTED: return "CS_ERR_UNSUPPORTED";
    case CS_ERR_WORKSPACE: return "CS_ERR_WORKSPACE";
    case CS_ERR_CUDA: return "CS_ERR_CUDA";
    case CS_ERR_NONFINITE: return "CS_ERR_NONFINITE";
  }
  return "CS_ERR_UNKNOWN";
}
const char* cs_last_error(void) { return g_last_error.c_str(); }
uint64_t cs_launch_count(int reset) {
  return reset ? g_launches.exchange(0) : g_launches.load();
}
const char* cs_version(void) { return "csgpu 0.1.0 (sm_100a)"; }

cs_status cs_diag_topk(const void* d_vals, int64_t n, int64_t K, int precision, int mode,
                       uint32_t* d_out_bits, cs_stream_t stream) {
  if (!d_vals || !d_out_bits) return fail(CS_ERR_INVALID_ARG, "null pointer");
  if (n < 1 || n > (1 << 24) || K < 1 || K > n) return fail(CS_ERR_INVALID_ARG, "need 1 <= K <= n <= 2^24");
  if (cs_status s = check_device()) return s;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  return precision ? s_diag_topk_launch<double>(reinterpret_cast<const double*>(d_vals), (int)n, (int)K, mode,
                                               d_out_bits, st, g_launches, g_last_error)
                   : s_diag_topk_launch<float>(reinterpret_cast<const float*>(d_vals), (int)n, (int)K, mode,
                                              d_out_bits, st, g_launches, g_last_error);
}

// ---------------------------------------------------------------- distributed operator ----
cs_status cs_dist_geometry(int64_t N, int64_t* L1, int64_t* L2, int32_t* CT) {
  if (!L1 || !L2 || !CT) return fail(CS_ERR_INVALID_ARG, "null pointer");
  if (cs_status s = check_N(N)) return s;
  if (N <= TIER_S_MAX_N) return fail(CS_ERR_UNSUPPORTED, "the distributed operator needs N > 16384 (grid tier)");
  const LGeom g = l_geom(N);
  *L1 = g.L1;
  *L2 = g.L2;
  *CT = g.CT;
  return CS_OK;
}
size_t cs_dist_ws_bytes(int64_t N, int64_t M) {
  if (N <= TIER_S_MAX_N) return 0;
  return (size_t)align_up(l_layout<float>(N, M, 0, 0, false, l_grid_upper<float>()).bytes, 256);
}
static cs_status dist_check(const cs_operator* op) {
  if (!op) return fail(CS_ERR_INVALID_ARG, "null operator");
  if (op->N <= TIER_S_MAX_N) return fail(CS_ERR_UNSUPPORTED, "the distributed operator needs N > 16384 (grid tier)");
  if (op->perm || op->psi || op->fkind) return fail(CS_ERR_UNSUPPORTED, "the distributed operator is the plain P.DCT.diag(sigma)");
  return check_device();
}
cs_status cs_dist_phase(const cs_operator* op, int phase, int64_t t_lo, int64_t t_hi, int64_t i_lo, int64_t i_hi,
                        const float* d_in, float* d_out, void* d_ws, size_t ws_bytes, cs_stream_t stream) {
  if (cs_status s = dist_check(op)) return s;
  if (phase < DP_A || phase > DP_XG) return fail(CS_ERR_INVALID_ARG, "unknown phase");
  const LGeom g = l_geom(op->N);
  const int64_t ntiles = g.L2 / g.CT, nitems = g.L1 / 2 + 1;
  if (t_lo < 0 || t_hi < t_lo || t_hi > ntiles || i_lo < 0 || i_hi < i_lo || i_hi > nitems)
    return fail(CS_ERR_INVALID_ARG, "tile / item range out of bounds");
  if ((phase == DP_A || phase == DP_C || phase == DP_XS || phase == DP_XG) && (t_hi == t_lo))
    return fail(CS_ERR_INVALID_ARG, "empty tile range");
  if (phase == DP_XG && ntiles % (t_hi - t_lo))
    return fail(CS_ERR_INVALID_ARG, "DP_XG: the tile range must split the tiles evenly");
  if (phase != DP_BF && phase != DP_C && !d_in) return fail(CS_ERR_INVALID_ARG, "null input");
  if (phase != DP_A && phase != DP_BA && !d_out) return fail(CS_ERR_INVALID_ARG, "null output");
  DistArgs<float> d{phase, t_lo, t_hi, i_lo, i_hi, d_in, d_out};
  return tier_l_dist_phase<float>(meta_of(op), d, d_ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream), g_launches,
                                  g_last_error);
}
cs_status cs_dist_row_offsets(const cs_operator* op, int64_t* h_off) {
  if (cs_status s = dist_check(op)) return s;
  if (!h_off) return fail(CS_ERR_INVALID_ARG, "null output");
  const LGeom g = l_geom(op->N);
  const OpMeta m = meta_of(op);
  // row k1's entries start at transposed position t = k1 2 L2, a whole mask word (2 L2 >= 32)
  const int64_t wpr = 2 * g.L2 / 32;
  std::vector<int32_t> pre(g.L1);
  cudaError_t e = cudaDeviceSynchronize();   // the metadata may still be in flight (plan time only)
  if (e == cudaSuccess) e = cudaMemcpy2D(pre.data(), sizeof(int32_t), m.tprefix(0), wpr * sizeof(int32_t), sizeof(int32_t),
                               g.L1, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return fail(CS_ERR_CUDA, std::string("row offsets: ") + cudaGetErrorString(e));
  for (int64_t k = 0; k < g.L1; ++k) h_off[k] = pre[k];
  h_off[g.L1] = op->M;
  return CS_OK;
}
cs_status cs_dist_copy(const cs_operator* op, void* d_ws, const int32_t* d_rows, const int32_t* d_col0, int64_t nseg,
                       int64_t seg_len, float* d_buf, int to_buf, cs_stream_t stream) {
  if (cs_status s = dist_check(op)) return s;
  if (!d_ws || (nseg > 0 && (!d_rows || !d_col0 || !d_buf)) || nseg < 0 || seg_len < 0)
    return fail(CS_ERR_INVALID_ARG, "bad arguments");
  const LGeom g = l_geom(op->N);
  if (seg_len > g.L2 || nseg > g.L1 * (g.L2 / std::max<int64_t>(seg_len, 1)))
    return fail(CS_ERR_INVALID_ARG, "segments larger than the intermediate");
  return tier_l_dist_copy<float>(meta_of(op), d_ws, d_rows, d_col0, nseg, seg_len, d_buf, to_buf,
                                 reinterpret_cast<cudaStream_t>(stream), g_launches, g_last_error);
}

size_t cs_diag_topk_grid_ws_bytes(void) {
  return std::max(tier_l_diag_topk_ws_bytes<float>(), tier_l_diag_topk_ws_bytes<double>());
}

cs_status cs_diag_topk_grid(const void* d_vals, int64_t n, int64_t K, int precision, uint32_t* d_out_bits,
                            void* d_ws, size_t ws_bytes, cs_stream_t stream) {
  if (!d_vals || !d_out_bits) return fail(CS_ERR_INVALID_ARG, "null pointer");
  if (n < 1 || n > ((int64_t)1 << 26) || K < 1 || K > n) return fail(CS_ERR_INVALID_ARG, "need 1 <= K <= n <= 2^26");
  if (cs_status s = check_device()) return s;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  return precision ? tier_l_diag_topk<double>(reinterpret_cast<const double*>(d_vals), n, K, d_out_bits, d_ws,
                                              ws_bytes, st, g_launches, g_last_error)
                   : tier_l_diag_topk<float>(reinterpret_cast<const float*>(d_vals), n, K, d_out_bits, d_ws,
                                             ws_bytes, st, g_launches, g_last_error);
}

double cs_diag_grid_barrier_us(int iters, int with_sum) {
  const int64_t smem = l_smem_bytes<float>(1 << 20);
  const void* fn = (const void*)k_l_recover<float>;
  const int grid = l_maxgrid<float>(fn, smem);
  void* buf = nullptr;
  if (cudaMalloc(&buf, 4096 + 2 * (size_t)grid * 8) != cudaSuccess) return -1.0;
  cudaMemset(buf, 0, 4096 + 2 * (size_t)grid * 8);
  GridBar* gb = reinterpret_cast<GridBar*>(buf);
  uint64_t* out = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(buf) + 256);
  double* pd = reinterpret_cast<double*>(reinterpret_cast<char*>(buf) + 4096);
  void* args[] = {&gb, &pd, &iters, &with_sum, &out};
  cudaLaunchCooperativeKernel((const void*)k_l_barrier_bench<float>, dim3(grid), dim3(TL_THREADS), args, 0, 0);
  uint64_t h[2] = {0, 0};
  cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
  cudaFree(buf);
  return (double)h[0] / 1e3 / iters;
}

int64_t cs_diag_phase_offset(int alg, int64_t N, int64_t M, int32_t K, int32_t ompr_l, int precision) {
  if (N <= TIER_S_MAX_N) return -1;
  if (alg < 0) {   // the apply / adjoint workspace: instance 0's phase stamps (k_l_apply)
    const LLayout s = precision ? l_layout<double>(N, M, 0, 0, false, l_grid_upper<double>())
                                : l_layout<float>(N, M, 0, 0, false, l_grid_upper<float>());
    return s.ts;
  }
  const int64_t ucap = ucap_of(alg, K, ompr_l);
  const LLayout s = precision ? l_layout<double>(N, M, K, (int)ucap, true, l_grid_upper<double>())
                              : l_layout<float>(N, M, K, (int)ucap, true, l_grid_upper<float>());
  return s.ts + 8 * 8;
}

// ---------------------------------------------------------------- dense output ----
cs_status cs_support_to_dense(int64_t B, int64_t N, int32_t K, const int32_t* d_support, const float* d_vals,
                              float* d_dense, cs_stream_t stream) {
  return dense_impl<float>(B, N, K, d_support, d_vals, d_dense, reinterpret_cast<cudaStream_t>(stream));
}
cs_status cs_support_to_dense_f64(int64_t B, int64_t N, int32_t K, const int32_t* d_support,
                                  const double* d_vals, double* d_dense, cs_stream_t stream) {
  return dense_impl<double>(B, N, K, d_support, d_vals, d_dense, reinterpret_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------- multi-GPU gather ----
cs_status cs_comm_init(int ndev, const int* devices, void** comm) {
  if (!comm || !devices || ndev < 1 || ndev > 64) return fail(CS_ERR_INVALID_ARG, "bad arguments");
  *comm = nullptr;
  const NcclApi& api = nccl_api();
  if (!api.ok) return fail(CS_ERR_UNSUPPORTED, "libnccl.so.2 could not be loaded");
  CsComm* c = new CsComm;
  c->dev.assign(devices, devices + ndev);
  c->comms.assign(ndev, nullptr);
  c->streams.assign(ndev, nullptr);
  c->ready.assign(ndev, nullptr);
  ncclResult_t r = api.init_all(c->comms.data(), ndev, devices);
  if (r != ncclSuccess) {
    delete c;
    return fail(CS_ERR_CUDA, std::string("ncclCommInitAll: ") + api.err(r));
  }
  int cur = 0;
  cudaGetDevice(&cur);
  bool good = true;
  for (int i = 0; i < ndev && good; ++i) {
    good = cudaSetDevice(devices[i]) == cudaSuccess &&
           cudaStreamCreateWithFlags(&c->streams[i], cudaStreamNonBlocking) == cudaSuccess &&
           cudaEventCreateWithFlags(&c->ready[i], cudaEventDisableTiming) == cudaSuccess;
  }
  cudaSetDevice(cur);
  if (!good) {
    cs_comm_destroy(c);
    return fail(CS_ERR_CUDA, "could not create the gather streams");
  }
  *comm = c;
  return CS_OK;
}

// restores the caller's current device on every exit path
struct DeviceGuard {
  int cur = 0;
  DeviceGuard() { cudaGetDevice(&cur); }
  ~DeviceGuard() { cudaSetDevice(cur); }
};

cs_status cs_gather_batched_after(void* comm, int root, int64_t B_per_dev, int32_t K, const float* const* d_vals,
                                  const int32_t* const* d_support, const cs_report* const* d_reports,
                                  float* d_vals_all, int32_t* d_support_all, cs_report* d_reports_all,
                                  const cs_stream_t* after) {
  CsComm* c = reinterpret_cast<CsComm*>(comm);
  if (!c || !d_vals || !d_support || !d_reports || !d_vals_all || !d_support_all || !d_reports_all)
    return fail(CS_ERR_INVALID_ARG, "null pointer argument");
  const int nd = (int)c->dev.size();
  if (root < 0 || root >= nd || B_per_dev < 1 || K < 1) return fail(CS_ERR_INVALID_ARG, "bad arguments");
  const NcclApi& api = nccl_api();
  const size_t bv = (size_t)(B_per_dev * K) * 4, br = (size_t)B_per_dev * sizeof(cs_report);
  DeviceGuard guard;
  // order the gather after the producers: device i's internal stream waits for everything
  // enqueued so far on after[i] (the streams that wrote the records and the outputs)
  if (after) {
    for (int i = 0; i < nd; ++i) {
      if (!after[i]) continue;
      CS_CUDA(cudaSetDevice(c->dev[i]));
      CS_CUDA(cudaEventRecord(c->ready[i], after[i]));
      CS_CUDA(cudaStreamWaitEvent(c->streams[i], c->ready[i], 0));
    }
  }
  // device i's records land at block i of the root's arrays; the root copies its own block
  CS_CUDA(cudaSetDevice(c->dev[root]));
  for (int kind = 0; kind < 3; ++kind) {
    const size_t bytes = kind == 2 ? br : bv;
    char* dst = kind == 0 ? reinterpret_cast<char*>(d_vals_all)
              : kind == 1 ? reinterpret_cast<char*>(d_support_all) : reinterpret_cast<char*>(d_reports_all);
    const void* src = kind == 0 ? (const void*)d_vals[root] : kind == 1 ? (const void*)d_support[root]
                                                                        : (const void*)d_reports[root];
    CS_CUDA(cudaMemcpyAsync(dst + (size_t)root * bytes, src, bytes, cudaMemcpyDeviceToDevice, c->streams[root]));
  }
  if (nd > 1) {
    if (!api.ok) return fail(CS_ERR_UNSUPPORTED, "NCCL not available");
    ncclResult_t r = api.group_start();
    for (int i = 0; i < nd && r == ncclSuccess; ++i) {
      if (i == root) continue;
      for (int kind = 0; kind < 3 && r == ncclSuccess; ++kind) {
        const size_t bytes = kind == 2 ? br : bv;
        char* dst = kind == 0 ? reinterpret_cast<char*>(d_vals_all)
                  : kind == 1 ? reinterpret_cast<char*>(d_support_all) : reinterpret_cast<char*>(d_reports_all);
        const void* src = kind == 0 ? (const void*)d_vals[i] : kind == 1 ? (const void*)d_support[i]
                                                                         : (const void*)d_reports[i];
        r = api.send(src, bytes, ncclUint8, root, c->comms[i], c->streams[i]);
        if (r == ncclSuccess) r = api.recv(dst + (size_t)i * bytes, bytes, ncclUint8, i, c->comms[root], c->streams[root]);
      }
    }
    const ncclResult_t re = api.group_end();
    if (r == ncclSuccess) r = re;
    if (r != ncclSuccess) return fail(CS_ERR_CUDA, std::string("nccl gather: ") + api.err(r));
  }
  for (int i = 0; i < nd; ++i) {
    CS_CUDA(cudaSetDevice(c->dev[i]));
    if (cudaStreamSynchronize(c->streams[i]) != cudaSuccess) return fail(CS_ERR_CUDA, "gather stream synchronisation failed");
  }
  return CS_OK;
}

cs_status cs_gather_batched(void* comm, int root, int64_t B_per_dev, int32_t K, const float* const* d_vals,
                            const int32_t* const* d_support, const cs_report* const* d_reports, float* d_vals_all,
                            int32_t* d_support_all, cs_report* d_reports_all) {
  return cs_gather_batched_after(comm, root, B_per_dev, K, d_vals, d_support, d_reports, d_vals_all, d_support_all,
                                 d_reports_all, nullptr);
}

cs_status cs_comm_destroy(void* comm) {
  CsComm* c = reinterpret_cast<CsComm*>(comm);
  if (!c) return CS_OK;
  const NcclApi& api = nccl_api();
  int cur = 0;
  cudaGetDevice(&cur);
  for (size_t i = 0; i < c->dev.size(); ++i) {
    cudaSetDevice(c->dev[i]);
    if (c->streams[i]) cudaStreamDestroy(c->streams[i]);
    if (c->ready[i]) cudaEventDestroy(c->ready[i]);
    if (c->comms[i] && api.ok) api.destroy(c->comms[i]);
  }
  cudaSetDevice(cur);
  delete c;
  return CS_OK;
}

}  // extern "C"
