// cs_common.cuh — shared device utilities for the sm_100a compressive-sensing path.
//
// Complex arithmetic, the Makhoul index map, bit-mask helpers and the
// packed-key helpers used by selection.  Everything is templated on the
// arithmetic type T in {float, double}.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/cs.h"

#define CS_DEV __device__ __forceinline__
#define CS_HD __host__ __device__ __forceinline__
#define CS_NOINL __device__ __noinline__

namespace cs {

// Dynamic shared memory of the running kernel (every unsized extern __shared__ array
// aliases its base).  shp(p) re-derives a generic pointer that is known to point
// into shared memory from this base, so that out-of-line device functions (which
// only see generic pointers) get 32-bit LDS/STS instead of generic LD/ST.
extern __shared__ __align__(16) char cs_smem_base[];
// threadIdx.x read through volatile asm: the read cannot be hoisted out of a loop, so
// per-pass address arithmetic derived from it is recomputed (a few ALU ops) instead of
// being hoisted and spilled to local memory under a 64-register budget.
CS_DEV int tid_fresh() {
  int t;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(t));
  return t;
}
template <typename P> CS_DEV P* shp(P* p) {
  const uint32_t off = (uint32_t)__cvta_generic_to_shared((const void*)p) -
                       (uint32_t)__cvta_generic_to_shared((const void*)cs_smem_base);
  return reinterpret_cast<P*>(cs_smem_base + off);
}

template <typename T> struct cplx_t;
template <> struct cplx_t<float> { using type = float2; };
template <> struct cplx_t<double> { using type = double2; };
template <typename T> using C2 = typename cplx_t<T>::type;

template <typename T> CS_HD C2<T> mk(T re, T im) { C2<T> r; r.x = re; r.y = im; return r; }
// fp32 complex add / subtract as ONE paired instruction (FADD2, PTX add/sub.rn.f32x2 on
// sm_100a): each lane is the same correctly rounded IEEE add as the scalar form, half the
// issue slots
#if defined(__CUDA_ARCH__) && !defined(CS_NO_F32X2)
CS_DEV unsigned long long f2_bits(float2 v) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(v.x), "f"(v.y));
  return r;
}
CS_DEV float2 bits_f2(unsigned long long r) {
  float2 v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
#endif
template <typename T> CS_HD C2<T> cadd(C2<T> a, C2<T> b) {
#if defined(__CUDA_ARCH__) && !defined(CS_NO_F32X2)
  if constexpr (sizeof(T) == 4) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)));
    return bits_f2(r);
  }
#endif
  return mk<T>(a.x + b.x, a.y + b.y);
}
template <typename T> CS_HD C2<T> csub(C2<T> a, C2<T> b) {
#if defined(__CUDA_ARCH__) && !defined(CS_NO_F32X2)
  if constexpr (sizeof(T) == 4) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)));
    return bits_f2(r);
  }
#endif
  return mk<T>(a.x - b.x, a.y - b.y);
}
#if defined(__CUDA_ARCH__) && !defined(CS_NO_F32X2)
CS_DEV unsigned long long f2_mul2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
CS_DEV unsigned long long f2_fma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
#endif
// fp32 complex products as FMUL2 + FFMA2: p = (ax bx, ay bx), then (ay, ax) * (-by, by) + p.
// ptxas folds the swap and the one-lane negation into operand modifiers (LO_HI.NP) and the
// broadcasts into scalar operands: two paired instructions instead of four
template <typename T> CS_HD C2<T> cmul(C2<T> a, C2<T> b) {
#if defined(__CUDA_ARCH__) && !defined(CS_NO_F32X2)
  if constexpr (sizeof(T) == 4) {
    const float2 av = a, bv = b;
    return bits_f2(f2_fma2(f2_bits(make_float2(av.y, av.x)), f2_bits(make_float2(-bv.y, bv.y)),
                           f2_mul2(f2_bits(av), f2_bits(make_float2(bv.x, bv.x)))));
  }
#endif
  return mk<T>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * conj(b)
template <typename T> CS_HD C2<T> cmulc(C2<T> a, C2<T> b) {
#if defined(__CUDA_ARCH__) && !defined(CS_NO_F32X2)
  if constexpr (sizeof(T) == 4) {
    const float2 av = a, bv = b;
    return bits_f2(f2_fma2(f2_bits(make_float2(av.y, av.x)), f2_bits(make_float2(bv.y, -bv.y)),
                           f2_mul2(f2_bits(av), f2_bits(make_float2(bv.x, bv.x)))));
  }
#endif
  return mk<T>(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
template <typename T> CS_HD C2<T> cconj(C2<T> a) { return mk<T>(a.x, -a.y); }
template <typename T> CS_HD C2<T> cscale(C2<T> a, T s) { return mk<T>(a.x * s, a.y * s); }
// multiply by -i (forward) or +i (inverse)
template <typename T, bool INV> CS_HD C2<T> mul_mi(C2<T> a) {
  return INV ? mk<T>(-a.y, a.x) : mk<T>(a.y, -a.x);
}

// ---------------------------------------------------------------------------
// Makhoul reorder.  Natural index j of u (length N) maps to
// position p of v: v_n = u_{2n}, v_{N-1-n} = u_{2n+1}.  The complex half-length
// sequence z_m = v_{2m} + i v_{2m+1} is v itself viewed as C2<T>[N/2].
CS_HD int64_t mk_pos(int64_t j, int64_t N) { return (j & 1) ? (N - 1 - (j >> 1)) : (j >> 1); }
CS_HD int64_t mk_nat(int64_t p, int64_t N) { return (2 * p < N) ? 2 * p : 2 * (N - 1 - p) + 1; }

// sigma_j from packed sign bits (bit set => -1)
template <typename T> CS_DEV T sign_of(const uint32_t* bits, int64_t j) {
  return ((bits[j >> 5] >> (j & 31)) & 1u) ? T(-1) : T(1);
}
template <typename T> CS_DEV T apply_sign(const uint32_t* bits, int64_t j, T v) {
  return ((bits[j >> 5] >> (j & 31)) & 1u) ? -v : v;
}
CS_DEV bool bit_test(const uint32_t* bits, int64_t j) { return (bits[j >> 5] >> (j & 31)) & 1u; }
// rank of a selected row k among selected rows (prefix popcount)
CS_DEV int64_t row_rank(const uint32_t* mask, const int32_t* prefix, int64_t k) {
  uint32_t w = mask[k >> 5];
  uint32_t below = (k & 31) ? (w & ((1u << (k & 31)) - 1u)) : 0u;
  return (int64_t)prefix[k >> 5] + __popc(below);
}

// Tile copies with UNR independent loads in flight per thread before any store
// (memory-level parallelism: one outstanding 8-byte load per thread caps a
// persistent grid near 0.6 TB/s).
template <int UNR, typename V, class LD, class ST>
CS_DEV void staged(int n, LD&& ld, ST&& st) {
  for (int e0 = threadIdx.x; e0 < n; e0 += UNR * (int)blockDim.x) {
    V v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int e = e0 + u * (int)blockDim.x;
      if (e < n) v[u] = ld(e);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int e = e0 + u * (int)blockDim.x;
      if (e < n) st(e, v[u]);
    }
  }
}
constexpr int TL_UNR = 8;
constexpr int TW_ANCHOR = 4;  // twiddle recurrence re-anchored from the table every 4 steps
// the same over the whole grid (index range [0, n), thread gtid of gnthr)
template <int UNR, typename V, class LD, class ST>
CS_DEV void gstaged(int64_t n, int64_t gtid, int64_t gnthr, LD&& ld, ST&& st) {
  for (int64_t e0 = gtid; e0 < n; e0 += UNR * gnthr) {
    V v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t e = e0 + u * gnthr;
      if (e < n) v[u] = ld(e);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t e = e0 + u * gnthr;
      if (e < n) st(e, v[u]);
    }
  }
}

// Bulk prefetch of [p, p + bytes) into L2 (one thread issues it; 16-byte aligned, bytes a
// multiple of 16): the next instance of a persistent loop streams into L2 while this one is
// computed, so its loads hit L2 instead of HBM.
CS_DEV void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Two-pass top-K of the CTA context (select.cuh): first-digit bins, candidate cap.
constexpr int TOPK_BINS = 1024;
constexpr int TOPK_CAP = 1024;

// Order-preserving keys of |v| (sign cleared, +1 so that key 0 means "excluded";
// NaN sorts above +inf).  64-bit keys for double keep the full order.
template <typename T> struct KeyT;
template <> struct KeyT<float> { using type = uint32_t; };
template <> struct KeyT<double> { using type = uint64_t; };
// full-precision order-preserving magnitude key, 0 reserved for "excluded"
CS_DEV uint32_t full_key(float v) { return (__float_as_uint(v) & 0x7fffffffu) + 1u; }
CS_DEV uint64_t full_key(double v) {
  return ((uint64_t)__double_as_longlong(v) & 0x7fffffffffffffffull) + 1ull;
}
// A 10-bit digit that is monotone non-decreasing in the key (0 for key 0): the
// exponent and two mantissa bits of |v| as a float (double: rounded to float,
// which preserves order up to ties).
CS_DEV unsigned key_digit10(uint32_t k) { return k >> 21; }
CS_DEV unsigned key_digit10(uint64_t k) {
  if (k == 0) return 0;
  const float f = (float)__longlong_as_double((long long)(k - 1ull));
  return (__float_as_uint(f) + 1u) >> 21;
}

}  // namespace cs
