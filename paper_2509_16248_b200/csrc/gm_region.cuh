// gm_region.cuh — hand-written sm_100a device skeleton for fused regions.
//
// A "region" is a run of straight-line statements of a GraphMend-transformed
// forward that the lowering fuses into one kernel: the predicate reductions
// of predicated blocks (transform.py:386-388 `__gm_pred_k = <T>.<red>() <cmp> c`),
// the arm expressions (transform.py:395-423) and the `torch.where` selects
// (transform.py:374-376), plus the elementwise statements around them.
//
// Execution model (one launch, 2 co-resident CTAs x 512 threads per SM):
//   * the iteration space (n elements, row-major) is cut into 8-element
//     vectors; vector v belongs to thread v % T (T = grid x 512) as its
//     k = v / T-th vector, so at any moment the grid sweeps one contiguous
//     stretch of HBM.  A thread issues the loads of all its vectors of a
//     register block (K x 16-32 B per input) before any arithmetic;
//   * pass p evaluates the elementwise code that only needs scalars known
//     before p, accumulates the reductions of pass p and stores the outputs
//     of pass p; after a pass with reductions every CTA publishes one partial
//     per reduction, arrives on a monotonic counter, and every CTA combines
//     the partials in the same fixed order (bit-identical scalars in all
//     CTAs, run-to-run deterministic) — no host readback, no .item();
//   * a speculative region (codegen.Plan.spec) runs ONE pass under the
//     decisions of its previous launch, verifies them after one grid
//     reduction and, on a misprediction, runs the exact passes in the same
//     launch;
//   * inputs an exact later pass re-reads stay in registers across the grid
//     barrier, or in their thread-private shared-memory slots;
//   * loads are 128-bit ld.global.nc, stores 128-bit st.global.
// Scalar predicates are CTA-uniform, so untaken arms are skipped by a
// uniform branch and their inputs are never loaded.
//
// Compiled twice: by nvcc into libgm_b200.so (precompiled canonical
// branch-select, gm_runtime.cu) and by NVRTC under the generated region
// sources (codegen.py).  It therefore includes no system headers.

#pragma once

namespace gm {

typedef unsigned long long u64;
typedef long long i64;
typedef unsigned int u32;
typedef unsigned short u16;
typedef unsigned char u8;

#define GM_MAX_IN 8
#define GM_MAX_OUT 8
#define GM_MAX_RED 16
#define GM_MAX_HS 32
#define GM_MAX_DIMS 6
#define GM_MAX_PIECES 16
#ifndef GM_THREADS
#define GM_THREADS 512  // threads per CTA (a generated region may define 1024)
#endif
#define GM_WARPS (GM_THREADS / 32)
#define GM_VEC 8

// element type codes (include/gm_b200.h)
#define GM_DT_F32 0
#define GM_DT_BF16 1
#define GM_DT_F16 2
#define GM_DT_F64 3
#define GM_DT_BOOL 4

// reduction combine ops
#define GM_R_SUM 0
#define GM_R_MAX 1
#define GM_R_MIN 2
#define GM_R_PROD 3
#define GM_R_OR 4
#define GM_R_AND 5
#define GM_R_KEYMAX 6  // max of u64 keys carried in the fp64 slots (argmax / argmin)

// Every field is 8 bytes wide so the ctypes mirror (_native.py) has the same
// layout with no padding rules involved.
struct InDesc {
  i64 ptr;                  // device address of element 0
  i64 smem_off;             // byte offset of this input's resident chunk (-1: stream)
  i64 ndim;                 // strided mode: number of iteration dims
  i64 size[GM_MAX_DIMS];    // strided mode: iteration-space sizes, outer..inner
  i64 stride[GM_MAX_DIMS];  // strided mode: element strides (0 = broadcast)
};

struct OutDesc {
  i64 ptr;
};

struct Params {
  i64 n;           // numel of the iteration space
  i64 nvec;        // ceil(n / GM_VEC)
  i64 vpc;         // vectors per CTA
  i64 piece_vecs;  // vectors per bulk-copy piece (resident staging)
  i64 partials;    // double[GM_MAX_RED][gridDim.x]
  i64 barrier;     // scratch: arrival counter, epoch flag, results (see grid_reduce)
  i64 status;      // int: 0 ok, 1 grid-barrier timeout (barrier + 16)
  i64 scal_out;    // double[GM_MAX_RED + ...]: scalar slots mirrored by CTA 0 (or 0)
  double hs[GM_MAX_HS];  // host scalars (Python numbers) as runtime values
  InDesc in[GM_MAX_IN];
  OutDesc out[GM_MAX_OUT];
};

// ---------------------------------------------------------------------------
// numerics: IEEE single ops without FMA contraction (torch eager runs every
// operator as its own kernel, so a*b+c rounds twice there too)
// ---------------------------------------------------------------------------
__device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ float fsqrt(float a) { return __fsqrt_rn(a); }
// NaN-propagating max/min (torch.maximum / Tensor.max semantics): one
// FMNMX.NAN each (max.NaN / min.NaN, sm_80+)
__device__ __forceinline__ float nmax(float a, float b) {
  float d;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
  return d;
}
__device__ __forceinline__ float nmin(float a, float b) {
  float d;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
  return d;
}
__device__ __forceinline__ float relu(float a) { return nmax(a, 0.f); }
__device__ __forceinline__ float recip(float a) { return __frcp_rn(a); }
// sigmoid: ex2 / rcp on the SFU with flush-to-zero (1 + 2^y reads a denormal
// 2^y as 1 anyway; only results below 1.2e-38 flush) — 2 MUFU, no fix-ups
__device__ __forceinline__ float sigmoid(float a) {
  float e, y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(a * -1.4426950408889634f));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(1.f + e));
  return y;
}
__device__ __forceinline__ float silu(float a) { return __fmul_rn(a, sigmoid(a)); }
// GELU as torch's CPU kernels evaluate it: (x * 0.5) * (1 + erf(x * M_SQRT1_2)),
// and the tanh form 0.5 * x * (1 + tanh(sqrt(2 / pi) * (x + 0.044715 * x^3)))
__device__ __forceinline__ float gelu(float a) {
  return __fmul_rn(__fmul_rn(a, 0.5f), __fadd_rn(1.f, erff(__fmul_rn(a, 0.70710678118654752f))));
}
// GELU for 16-bit outputs.  erf(z) = ±(1 - erfc|z|) with erfc by the
// Chebyshev fit of Numerical Recipes' erfcc (relative error < 1.2e-7 for
// every z, so 1 - erfc rounds to the same float as a correctly rounded erf
// and `1 + erf` keeps torch's cancellation for negative z), the reciprocal
// and the exponential on the SFU — a third of erff's instructions, and an
// error far below the bf16 / fp16 rounding of the result
__device__ __forceinline__ float gelu16(float a) {
  const float z = __fmul_rn(a, 0.70710678118654752f);
  const float az = fabsf(z);
  float t;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(__fmaf_rn(0.5f, az, 1.f)));
  float p = __fmaf_rn(t, 0.17087277f, -0.82215223f);
  p = __fmaf_rn(t, p, 1.48851587f);
  p = __fmaf_rn(t, p, -1.13520398f);
  p = __fmaf_rn(t, p, 0.27886807f);
  p = __fmaf_rn(t, p, -0.18628806f);
  p = __fmaf_rn(t, p, 0.09678418f);
  p = __fmaf_rn(t, p, 0.37409196f);
  p = __fmaf_rn(t, p, 1.00002368f);
  p = __fmaf_rn(t, p, -1.26551223f);
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"((p - az * az) * 1.4426950408889634f));
  const float erfc_az = t * e;
  const float erf_z = copysignf(__fsub_rn(1.f, erfc_az), z);
  return __fmul_rn(__fmul_rn(a, 0.5f), __fadd_rn(1.f, erf_z));
}
__device__ __forceinline__ float gelu_tanh(float a) {
  const float inner = __fmul_rn(0.79788456080286536f, __fadd_rn(a, __fmul_rn(0.044715f, __fmul_rn(__fmul_rn(a, a), a))));
  return __fmul_rn(__fmul_rn(0.5f, a), __fadd_rn(1.f, tanhf(inner)));
}
// exp(a) = 2^(a * log2 e) on the SFU (MUFU.EX2, subnormal results kept):
// relative error ~2^-22 plus |a| * 2^-24 * ln 2 from rounding the product
__device__ __forceinline__ float ex2(float a) {
  float y;
  asm("ex2.approx.f32 %0, %1;" : "=f"(y) : "f"(a));
  return y;
}
__device__ __forceinline__ float fexp(float a) {
  float y;
  asm("ex2.approx.f32 %0, %1;" : "=f"(y) : "f"(__fmul_rn(a, 1.4426950408889634f)));
  return y;
}
// Python-style `%` and `//` on floats, as torch's CPU kernels compute them
// (remainder: fmod, then + b when the signs differ; floor_divide:
// div_floor_floating — (a - fmod(a, b)) / b, corrected and rounded to an
// integer value, copysign(0, a / b) for a zero quotient)
template <typename T>
__device__ __forceinline__ T pymod_t(T a, T b) {
  T m = fmod(a, b);
  if (m != (T)0 && ((b < (T)0) != (m < (T)0))) m += b;
  return m;
}
template <typename T>
__device__ __forceinline__ T floordiv_t(T a, T b) {
  if (b == (T)0) return a / b;
  const T m = fmod(a, b);
  T d = (a - m) / b;
  if (m != (T)0 && ((b < (T)0) != (m < (T)0))) d -= (T)1;
  if (d != (T)0) {
    T f = floor(d);
    if (d - f > (T)0.5) f += (T)1;
    return f;
  }
  return copysign((T)0, a / b);
}
__device__ __forceinline__ float pymod(float a, float b) {
  float m = fmodf(a, b);
  if (m != 0.f && ((b < 0.f) != (m < 0.f))) m = __fadd_rn(m, b);
  return m;
}
__device__ __forceinline__ float floordiv(float a, float b) {
  if (b == 0.f) return __fdiv_rn(a, b);
  const float m = fmodf(a, b);
  float d = __fdiv_rn(__fsub_rn(a, m), b);
  if (m != 0.f && ((b < 0.f) != (m < 0.f))) d = __fsub_rn(d, 1.f);
  if (d != 0.f) {
    float f = floorf(d);
    if (__fsub_rn(d, f) > 0.5f) f = __fadd_rn(f, 1.f);
    return f;
  }
  return copysignf(0.f, __fdiv_rn(a, b));
}
__device__ __forceinline__ float neg(float a) { return -a; }
__device__ __forceinline__ double dmax(double a, double b) { return (a != a) ? a : ((b != b) ? b : (a > b ? a : b)); }
__device__ __forceinline__ double dmin(double a, double b) { return (a != a) ? a : ((b != b) ? b : (a < b ? a : b)); }

// bf16 / f16 conversions without cuda_bf16.h (hardware cvt, round-nearest-even)
__device__ __forceinline__ float bf2f(u16 h) { return __uint_as_float(((u32)h) << 16); }
__device__ __forceinline__ u16 f2bf(float f) {
  u16 h;
  asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(h) : "f"(f));
  return h;
}
// two floats -> packed bf16x2 (lo in bits 0..15)
__device__ __forceinline__ u32 f2bf2(float lo, float hi) {
  u32 r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ float h2f(u16 h) {
  float f;
  asm("cvt.f32.f16 %0, %1;" : "=f"(f) : "h"(h));
  return f;
}
__device__ __forceinline__ u16 f2h(float f) {
  u16 h;
  asm("cvt.rn.f16.f32 %0, %1;" : "=h"(h) : "f"(f));
  return h;
}
// per-operator rounding to the result's storage type (eager semantics)
__device__ __forceinline__ float rbf(float f) { return __uint_as_float(f2bf2(0.f, f) & 0xffff0000u); }
__device__ __forceinline__ float rh(float f) { return h2f(f2h(f)); }
__device__ __forceinline__ double rbf_d(double d) { return (double)rbf((float)d); }
__device__ __forceinline__ double rh_d(double d) { return (double)rh((float)d); }

// ---------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------
__device__ __forceinline__ u32 smem_u32(const void* p) {
  u32 r;
  asm("{ .reg .u64 t; cvta.to.shared.u64 t, %1; cvt.u32.u64 %0, t; }" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ void ldg16(const void* p, u32& a, u32& b, u32& c, u32& d) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p));
}
__device__ __forceinline__ void ldg8b(const void* p, u32& a, u32& b) {
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(a), "=r"(b) : "l"(p));
}
__device__ __forceinline__ void lds16(u32 s, u32& a, u32& b, u32& c, u32& d) {
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(s));
}
__device__ __forceinline__ void lds8b(u32 s, u32& a, u32& b) {
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(a), "=r"(b) : "r"(s));
}
__device__ __forceinline__ void stg16(void* p, u32 a, u32 b, u32 c, u32 d) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void stg8b(void* p, u32 a, u32 b) {
  asm volatile("st.global.v2.u32 [%0], {%1,%2};" ::"l"(p), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ double ld_relaxed_f64(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ u64 globaltimer() {
  u64 t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// mbarrier + bulk copy (sm_90+; the bulk-copy engine on Blackwell)
__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(u64* bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, u32 bytes, u64* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* bar, u32 parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "GM_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra GM_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ---------------------------------------------------------------------------
// element access
// ---------------------------------------------------------------------------
template <int DT> struct Elem;
template <> struct Elem<GM_DT_F32> {
  static constexpr int ES = 4;
  __device__ static __forceinline__ float ld(const void* p, i64 i) { return ((const float*)p)[i]; }
  __device__ static __forceinline__ void st(void* p, i64 i, float v) { ((float*)p)[i] = v; }
  __device__ static __forceinline__ void ldg8(const void* p, float (&x)[8]) {
    u32 a, b, c, d, e, f, g, h;
    ldg16(p, a, b, c, d);
    ldg16((const char*)p + 16, e, f, g, h);
    x[0] = __uint_as_float(a); x[1] = __uint_as_float(b); x[2] = __uint_as_float(c); x[3] = __uint_as_float(d);
    x[4] = __uint_as_float(e); x[5] = __uint_as_float(f); x[6] = __uint_as_float(g); x[7] = __uint_as_float(h);
  }
  __device__ static __forceinline__ void lds8(u32 s, float (&x)[8]) {
    u32 a, b, c, d, e, f, g, h;
    lds16(s, a, b, c, d);
    lds16(s + 16, e, f, g, h);
    x[0] = __uint_as_float(a); x[1] = __uint_as_float(b); x[2] = __uint_as_float(c); x[3] = __uint_as_float(d);
    x[4] = __uint_as_float(e); x[5] = __uint_as_float(f); x[6] = __uint_as_float(g); x[7] = __uint_as_float(h);
  }
  __device__ static __forceinline__ float lds1(u32 s) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(s));
    return v;
  }
  __device__ static __forceinline__ void stg8(void* p, const float (&y)[8]) {
    stg16(p, __float_as_uint(y[0]), __float_as_uint(y[1]), __float_as_uint(y[2]), __float_as_uint(y[3]));
    stg16((char*)p + 16, __float_as_uint(y[4]), __float_as_uint(y[5]), __float_as_uint(y[6]),
          __float_as_uint(y[7]));
  }
};
template <int DT> struct Elem16 {
  // bf16 / f16: 8 elements = 16 bytes
  static constexpr int ES = 2;
  __device__ static __forceinline__ float cv(u16 h) { return DT == GM_DT_BF16 ? bf2f(h) : h2f(h); }
  __device__ static __forceinline__ u16 rc(float f) { return DT == GM_DT_BF16 ? f2bf(f) : f2h(f); }
  __device__ static __forceinline__ float ld(const void* p, i64 i) { return cv(((const u16*)p)[i]); }
  __device__ static __forceinline__ void st(void* p, i64 i, float v) { ((u16*)p)[i] = rc(v); }
  __device__ static __forceinline__ void unpack(u32 w, float& lo, float& hi) {
    lo = cv((u16)(w & 0xffffu));
    hi = cv((u16)(w >> 16));
  }
  __device__ static __forceinline__ u32 pack(float lo, float hi) {
    return DT == GM_DT_BF16 ? f2bf2(lo, hi) : ((u32)rc(lo) | ((u32)rc(hi) << 16));
  }
  __device__ static __forceinline__ void ldg8(const void* p, float (&x)[8]) {
    u32 a, b, c, d;
    ldg16(p, a, b, c, d);
    unpack(a, x[0], x[1]); unpack(b, x[2], x[3]); unpack(c, x[4], x[5]); unpack(d, x[6], x[7]);
  }
  __device__ static __forceinline__ void lds8(u32 s, float (&x)[8]) {
    u32 a, b, c, d;
    lds16(s, a, b, c, d);
    unpack(a, x[0], x[1]); unpack(b, x[2], x[3]); unpack(c, x[4], x[5]); unpack(d, x[6], x[7]);
  }
  __device__ static __forceinline__ float lds1(u32 s) {
    u16 v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(s));
    return cv(v);
  }
  __device__ static __forceinline__ void stg8(void* p, const float (&y)[8]) {
    stg16(p, pack(y[0], y[1]), pack(y[2], y[3]), pack(y[4], y[5]), pack(y[6], y[7]));
  }
};
template <> struct Elem<GM_DT_BF16> : Elem16<GM_DT_BF16> {};
template <> struct Elem<GM_DT_F16> : Elem16<GM_DT_F16> {};
template <> struct Elem<GM_DT_BOOL> {
  static constexpr int ES = 1;
  __device__ static __forceinline__ float ld(const void* p, i64 i) { return ((const u8*)p)[i] ? 1.f : 0.f; }
  __device__ static __forceinline__ void st(void* p, i64 i, float v) { ((u8*)p)[i] = (v != 0.f) ? 1 : 0; }
  __device__ static __forceinline__ void ldg8(const void* p, float (&x)[8]) {
    u32 a, b;
    ldg8b(p, a, b);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      x[k] = ((a >> (8 * k)) & 0xffu) ? 1.f : 0.f;
      x[4 + k] = ((b >> (8 * k)) & 0xffu) ? 1.f : 0.f;
    }
  }
  __device__ static __forceinline__ void lds8(u32 s, float (&x)[8]) {
    u32 a, b;
    lds8b(s, a, b);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      x[k] = ((a >> (8 * k)) & 0xffu) ? 1.f : 0.f;
      x[4 + k] = ((b >> (8 * k)) & 0xffu) ? 1.f : 0.f;
    }
  }
  __device__ static __forceinline__ float lds1(u32 s) {
    u16 v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(s));
    return v ? 1.f : 0.f;
  }
  __device__ static __forceinline__ void stg8(void* p, const float (&y)[8]) {
    u32 a = 0, b = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      a |= (y[k] != 0.f ? 1u : 0u) << (8 * k);
      b |= (y[4 + k] != 0.f ? 1u : 0u) << (8 * k);
    }
    stg8b(p, a, b);
  }
};

// Full-size contiguous input: vector `e` (first element index, multiple of 8),
// `nv` valid lanes; `sres` = shared address of the CTA's resident chunk
// (0 when streaming), `le` = element index local to the chunk.
template <int DT>
__device__ __forceinline__ void load8(const InDesc& d, u32 sres, i64 e, i64 le, int nv, float (&x)[8]) {
  typedef Elem<DT> E;
  if (nv == GM_VEC) {
    if (sres)
      E::lds8(sres + (u32)(le * E::ES), x);
    else
      E::ldg8((const char*)d.ptr + e * E::ES, x);
  } else {
#pragma unroll
    for (int k = 0; k < GM_VEC; ++k)
      x[k] = (k < nv) ? (sres ? E::lds1(sres + (u32)((le + k) * E::ES)) : E::ld((const void*)d.ptr, e + k)) : 0.f;
  }
}

// Streamed input from global memory (128-bit ld.global.nc); per-lane loads
// for the partial tail vector.
template <int DT>
__device__ __forceinline__ void load8_gmem(const InDesc& d, i64 e, int nv, float (&x)[8]) {
  typedef Elem<DT> E;
  if (nv == GM_VEC) {
    E::ldg8((const char*)d.ptr + e * E::ES, x);
  } else {
#pragma unroll
    for (int k = 0; k < GM_VEC; ++k) x[k] = (k < nv) ? E::ld((const void*)d.ptr, e + k) : 0.f;
  }
}

// ---------------------------------------------------------------------------
// packed bf16x2 arithmetic.  For bf16 operands `op.rn.bf16x2` is the exact
// result rounded once to bf16 — what torch's CPU kernels produce by
// computing in fp32 and rounding the fp32 result (the fp32 add/sub/mul of two
// bf16 values is exact or below half a bf16 ulp).  Chains of such ops then
// need no unpack/round/pack per op.
// ---------------------------------------------------------------------------
__device__ __forceinline__ u32 hadd2(u32 a, u32 b) {
  u32 d;
  asm("add.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ u32 hsub2(u32 a, u32 b) {
  u32 d;
  asm("sub.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ u32 hmul2(u32 a, u32 b) {
  u32 d;
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
// NaN-propagating packed max/min (max.NaN.bf16x2, sm_90+): relu and the
// bf16 max/min reductions stay packed
__device__ __forceinline__ u32 hmax2(u32 a, u32 b) {
  u32 d;
  asm("max.NaN.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ u32 hmin2(u32 a, u32 b) {
  u32 d;
  asm("min.NaN.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ void unpack_bf2(u32 p, float& lo, float& hi) {
  lo = __uint_as_float(p << 16);
  hi = __uint_as_float(p & 0xffff0000u);
}
__device__ __forceinline__ void unpack8(const u32 (&p)[4], float (&x)[8]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) unpack_bf2(p[j], x[2 * j], x[2 * j + 1]);
}
// fp32 sum / sum of squares straight from packed bf16x2 words: the sm_100
// mixed-precision add / fma (FHADD.BF16 / FHFMA.BF16 with .H0/.H1 operand
// selects) — one instruction per element instead of an unpack and an FADD.
// Summed in element order (a chain; the unpacked path sums a tree of 8).
__device__ __forceinline__ float fadd_bf(float acc, u32 w, int half) {
  const u16 h = (u16)(half ? w >> 16 : w & 0xffffu);
  asm("add.rn.f32.bf16 %0, %1, %0;" : "+f"(acc) : "h"(h));
  return acc;
}
__device__ __forceinline__ float ffma_bf(float acc, u32 w, int half) {
  const u16 h = (u16)(half ? w >> 16 : w & 0xffffu);
  asm("fma.rn.f32.bf16 %0, %1, %1, %0;" : "+f"(acc) : "h"(h));
  return acc;
}
template <bool SQ>
__device__ __forceinline__ float acc_sum_p(float acc, const u32 (&p)[4], int nv) {
#pragma unroll
  for (int l = 0; l < 8; ++l) {
    if (l >= nv) break;
    acc = SQ ? ffma_bf(acc, p[l >> 1], l & 1) : fadd_bf(acc, p[l >> 1], l & 1);
  }
  return acc;
}
template <int MAX>
__device__ __forceinline__ float acc_minmax_p(float acc, const u32 (&p)[4]) {
  const u32 m = MAX ? hmax2(hmax2(p[0], p[1]), hmax2(p[2], p[3])) : hmin2(hmin2(p[0], p[1]), hmin2(p[2], p[3]));
  float lo, hi;
  unpack_bf2(m, lo, hi);
  return MAX ? nmax(acc, nmax(lo, hi)) : nmin(acc, nmin(lo, hi));
}
__device__ __forceinline__ void pack8(const float (&x)[8], u32 (&p)[4]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) p[j] = f2bf2(x[2 * j], x[2 * j + 1]);
}
// raw 16-byte (8 x bf16) vector access for the packed path
__device__ __forceinline__ void stg_raw(const OutDesc& o, i64 e, const u32 (&p)[4]) {
  stg16((char*)o.ptr + e * 2, p[0], p[1], p[2], p[3]);
}

// ---------------------------------------------------------------------------
// thread-private staging.  Every pass maps vector v to the same thread, so a
// thread only ever re-reads the stash slots it wrote: no mbarrier, no
// __syncthreads.  The first pass that reads an input a later pass re-reads
// stores its raw vectors to shared memory after use (rstash); an input first
// read by a later pass is prefetched at kernel start with cp.async (LDGSTS)
// and waited per thread (cp_async_wait_all).  The one partial tail vector of
// a tensor always reads global memory.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void sts16(u32 s, u32 a, u32 b, u32 c, u32 d) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(s), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void cp_async16(u32 s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(g) : "memory");
}
// L2 prefetch of the 32-byte sector holding one vector
__device__ __forceinline__ void prefetch_l2(const char* p, int bytes) {
  (void)bytes;
  asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ---------------------------------------------------------------------------
// raw vectors.  The generated loops issue every load of a register block
// (one 8-element vector per input per k) before any arithmetic, so a thread
// keeps K x 16-32 bytes per input in flight; the raw 32-bit words are kept
// as loaded and converted (or used packed) where a node reads them.
// Vector v of the iteration space belongs to thread v % T (T = grid x
// GM_THREADS) as its k = v / T-th vector; its thread-private shared-memory
// slot is (k * GM_THREADS + threadIdx.x) — the `le` element index below.
// ---------------------------------------------------------------------------
template <int DT> struct Raw;
template <> struct Raw<GM_DT_F32> { u32 w[8]; };
template <> struct Raw<GM_DT_BF16> { u32 w[4]; };
template <> struct Raw<GM_DT_F16> { u32 w[4]; };
template <> struct Raw<GM_DT_BOOL> { u32 w[2]; };

template <int DT>
__device__ __forceinline__ void rload(const InDesc& d, i64 e, Raw<DT>& r) {
  const char* g = (const char*)d.ptr + e * Elem<DT>::ES;
  if (DT == GM_DT_BOOL) {
    ldg8b(g, r.w[0], r.w[1]);
  } else {
#pragma unroll
    for (int b = 0; b < (int)(sizeof(Raw<DT>) / 16); ++b) ldg16(g + 16 * b, r.w[4 * b], r.w[4 * b + 1], r.w[4 * b + 2], r.w[4 * b + 3]);
  }
}
template <int DT>
__device__ __forceinline__ void rstash(u32 s, const Raw<DT>& r) {
  if (DT == GM_DT_BOOL) {
    asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(s), "r"(r.w[0]), "r"(r.w[1]) : "memory");
  } else {
#pragma unroll
    for (int b = 0; b < (int)(sizeof(Raw<DT>) / 16); ++b) sts16(s + 16 * b, r.w[4 * b], r.w[4 * b + 1], r.w[4 * b + 2], r.w[4 * b + 3]);
  }
}
template <int DT>
__device__ __forceinline__ void rlds(u32 s, Raw<DT>& r) {
  if (DT == GM_DT_BOOL) {
    lds8b(s, r.w[0], r.w[1]);
  } else {
#pragma unroll
    for (int b = 0; b < (int)(sizeof(Raw<DT>) / 16); ++b) lds16(s + 16 * b, r.w[4 * b], r.w[4 * b + 1], r.w[4 * b + 2], r.w[4 * b + 3]);
  }
}
// cp.async (LDGSTS) of one vector into its stash slot (16-byte types only)
template <int DT>
__device__ __forceinline__ void rprefetch(u32 s, const InDesc& d, i64 e) {
  const char* g = (const char*)d.ptr + e * Elem<DT>::ES;
#pragma unroll
  for (int b = 0; b < (int)(sizeof(Raw<DT>) / 16); ++b) cp_async16(s + 16 * b, g + 16 * b);
}
template <int DT>
__device__ __forceinline__ void rcvt(const Raw<DT>& r, float (&x)[8]) {
  if (DT == GM_DT_F32) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = __uint_as_float(r.w[k]);
  } else if (DT == GM_DT_BOOL) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      x[k] = ((r.w[0] >> (8 * k)) & 0xffu) ? 1.f : 0.f;
      x[4 + k] = ((r.w[1] >> (8 * k)) & 0xffu) ? 1.f : 0.f;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) Elem16<DT>::unpack(r.w[j], x[2 * j], x[2 * j + 1]);
  }
}

// Broadcast / strided input: element offsets decoded from the iteration index.
template <int DT>
__device__ __forceinline__ void load8_strided(const InDesc& d, i64 e, int nv, float (&x)[8]) {
  typedef Elem<DT> E;
#pragma unroll
  for (int k = 0; k < GM_VEC; ++k) {
    float v = 0.f;
    if (k < nv) {
      i64 i = e + k, off = 0;
      for (int j = (int)d.ndim - 1; j >= 0; --j) {
        const i64 s = d.size[j];
        off += (i % s) * d.stride[j];
        i /= s;
      }
      v = E::ld((const void*)d.ptr, off);
    }
    x[k] = v;
  }
}

// Periodic broadcast along the innermost dims (e.g. a [D] bias over [..., D]):
// element i reads index i % period; vector loads when the period keeps the
// 8 lanes contiguous.
template <int DT>
__device__ __forceinline__ void load8_periodic(const InDesc& d, i64 e, int nv, float (&x)[8]) {
  typedef Elem<DT> E;
  const i64 period = d.size[0];
  const i64 j = e % period;
  if (nv == GM_VEC && (period % GM_VEC) == 0) {
    E::ldg8((const char*)d.ptr + j * E::ES, x);
  } else {
#pragma unroll
    for (int k = 0; k < GM_VEC; ++k) x[k] = (k < nv) ? E::ld((const void*)d.ptr, (e + k) % period) : 0.f;
  }
}

// Same with the period known at specialisation: `e % PER` by a constant is
// a multiply-high sequence instead of a 64-bit division routine per vector.
template <int DT, long long PER>
__device__ __forceinline__ void load8_periodic_c(const InDesc& d, i64 e, int nv, float (&x)[8]) {
  typedef Elem<DT> E;
  if ((PER % GM_VEC) == 0 && nv == GM_VEC) {
    E::ldg8((const char*)d.ptr + (e % PER) * E::ES, x);
  } else {
#pragma unroll
    for (int k = 0; k < GM_VEC; ++k) x[k] = (k < nv) ? E::ld((const void*)d.ptr, (e + k) % PER) : 0.f;
  }
}

template <int DT>
__device__ __forceinline__ float load_scalar(const InDesc& d) {
  return Elem<DT>::ld((const void*)d.ptr, 0);
}

template <int DT>
__device__ __forceinline__ void store8(const OutDesc& o, i64 e, int nv, const float (&y)[8]) {
  typedef Elem<DT> E;
  if (nv == GM_VEC) {
    E::stg8((char*)o.ptr + e * E::ES, y);
  } else {
#pragma unroll
    for (int k = 0; k < GM_VEC; ++k)
      if (k < nv) E::st((void*)o.ptr, e + k, y[k]);
  }
}

// ---------------------------------------------------------------------------
// row regions (rowgen.py): a thread group of TPR threads owns one row of the
// innermost dimension; its vectors start at column (u * TPR + t) * 8, so a
// vector never crosses a row.  When the row length is not a multiple of 8
// the vectors are not 16-byte aligned and every lane is accessed alone.
// ---------------------------------------------------------------------------
template <int DT>
__device__ __forceinline__ void load8_elems(const InDesc& d, i64 e, int nv, float (&x)[8]) {
#pragma unroll
  for (int k = 0; k < GM_VEC; ++k) x[k] = (k < nv) ? Elem<DT>::ld((const void*)d.ptr, e + k) : 0.f;
}
template <int DT>
__device__ __forceinline__ void load8_periodic_elems(const InDesc& d, i64 e, int nv, float (&x)[8]) {
  const i64 period = d.size[0];
#pragma unroll
  for (int k = 0; k < GM_VEC; ++k) x[k] = (k < nv) ? Elem<DT>::ld((const void*)d.ptr, (e + k) % period) : 0.f;
}
template <int DT>
__device__ __forceinline__ void store8_elems(const OutDesc& o, i64 e, int nv, const float (&y)[8]) {
#pragma unroll
  for (int k = 0; k < GM_VEC; ++k)
    if (k < nv) Elem<DT>::st((void*)o.ptr, e + k, y[k]);
}
template <int DT>
__device__ __forceinline__ float load_at(const InDesc& d, i64 i) {
  return Elem<DT>::ld((const void*)d.ptr, i);
}
template <int DT>
__device__ __forceinline__ void store_at(const OutDesc& o, i64 i, float v) {
  Elem<DT>::st((void*)o.ptr, i, v);
}
template <int DT>
__device__ __forceinline__ void store_scalar(const OutDesc& o, double v) {
  Elem<DT>::st((void*)o.ptr, 0, (float)v);
}

// ---------------------------------------------------------------------------
// resident staging: the CTA's chunk of every staged input is bulk-copied into
// shared memory at kernel start, in <= GM_MAX_PIECES pieces per group with one
// mbarrier per piece.  Group 0 = inputs pass 0 reads (issued first, waited in
// pass 0); group 1 = inputs first read by a later pass (prefetched behind pass
// 0 and the grid barrier, waited in the first pass that reads them).
// `grp[k]` is 0, 1, or -1 (input k streams from global memory).
// ---------------------------------------------------------------------------
struct Stage {
  u64* bars;        // [GM_MAX_PIECES] in static smem
  int npieces;
  i64 piece_vecs;
  int waited;       // pieces this thread has already waited for (in order)
  i64 wend;         // = waited * piece_vecs
};

__device__ __forceinline__ void stage_issue_group(const Params& P, unsigned char* smem, int nin, const int* es,
                                                  const int* grp, int g, i64 v0, i64 v1, Stage& st) {
  const i64 e_end_cta = (v1 * GM_VEC < P.n) ? v1 * GM_VEC : P.n;
  for (int p = 0; p < st.npieces; ++p) {
    const i64 pv0 = v0 + (i64)p * P.piece_vecs;
    const i64 pv1 = (pv0 + P.piece_vecs < v1) ? pv0 + P.piece_vecs : v1;
    const i64 e0 = pv0 * GM_VEC;
    const i64 e1 = (pv1 * GM_VEC < e_end_cta) ? pv1 * GM_VEC : e_end_cta;
    u32 tx = 0;
    for (int k = 0; k < nin; ++k)
      if (grp[k] == g) tx += (u32)((e1 - e0) * es[k]);
    mbar_expect_tx(&st.bars[p], tx);
    for (int k = 0; k < nin; ++k) {
      if (grp[k] != g) continue;
      const char* src = (const char*)P.in[k].ptr + e0 * es[k];
      unsigned char* dst = smem + P.in[k].smem_off + (e0 - v0 * GM_VEC) * es[k];
      bulk_g2s(dst, src, (u32)((e1 - e0) * es[k]), &st.bars[p]);
    }
  }
}

__device__ __forceinline__ void stage_issue(const Params& P, unsigned char* smem, int nin, const int* es,
                                            const int* grp, i64 v0, i64 v1, Stage& a, Stage& b) {
  const i64 nv = v1 - v0;
  const int np = nv > 0 ? (int)((nv + P.piece_vecs - 1) / P.piece_vecs) : 0;
  bool has[2] = {false, false};
  for (int k = 0; k < nin; ++k)
    if (grp[k] >= 0) has[grp[k]] = true;
  Stage* st[2] = {&a, &b};
  for (int g = 0; g < 2; ++g) {
    st[g]->piece_vecs = P.piece_vecs;
    st[g]->npieces = has[g] ? np : 0;
    st[g]->waited = 0;
    st[g]->wend = 0;
  }
  if (threadIdx.x == 0) {
    for (int g = 0; g < 2; ++g)
      for (int p = 0; p < st[g]->npieces; ++p) mbar_init(&st[g]->bars[p], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int g = 0; g < 2; ++g)
      if (has[g]) stage_issue_group(P, smem, nin, es, grp, g, v0, v1, *st[g]);
  }
}

// Wait (once, in order) for the piece holding local vector `lv` — no
// division on the hot path: `waited` pieces cover local vectors < wend.
__device__ __forceinline__ void stage_wait(Stage& st, i64 lv) {
  while (st.wend <= lv && st.waited < st.npieces) {
    mbar_wait(&st.bars[st.waited], 0);
    ++st.waited;
    st.wend += st.piece_vecs;
  }
}

// After the first pass every piece is complete; make that visible to all.
__device__ __forceinline__ void stage_finish(Stage& st) {
  if (threadIdx.x == 0)
    while (st.waited < st.npieces) {
      mbar_wait(&st.bars[st.waited], 0);
      ++st.waited;
    }
  __syncthreads();
  st.waited = st.npieces;
}

// ---------------------------------------------------------------------------
// grid-wide reduction
// ---------------------------------------------------------------------------
__device__ __forceinline__ double red_identity(int op) {
  switch (op) {
    case GM_R_MAX: return -__longlong_as_double(0x7ff0000000000000LL);
    case GM_R_MIN: return __longlong_as_double(0x7ff0000000000000LL);
    case GM_R_PROD: return 1.0;
    case GM_R_AND: return 1.0;
    default: return 0.0;
  }
}
__device__ __forceinline__ double red_combine(int op, double a, double b) {
  switch (op) {
    case GM_R_KEYMAX:
      return ((u64)__double_as_longlong(a) >= (u64)__double_as_longlong(b)) ? a : b;
    case GM_R_MAX: return dmax(a, b);
    case GM_R_MIN: return dmin(a, b);
    case GM_R_PROD: return a * b;
    case GM_R_OR: return (a != 0.0 || b != 0.0) ? 1.0 : 0.0;
    case GM_R_AND: return (a != 0.0 && b != 0.0) ? 1.0 : 0.0;
    default: return a + b;
  }
}

// combine of a row statistic over the TPR threads of a row group: xor
// shuffles inside a warp, then (TPR > 32) the warps of the group through
// shared memory in a fixed order.  Every thread of the CTA must call it.
template <int TPR, int OP>
__device__ __forceinline__ double row_combine(double v, double* s_rw) {
  constexpr int W = TPR < 32 ? TPR : 32;
#pragma unroll
  for (int off = W / 2; off > 0; off >>= 1) v = red_combine(OP, v, __shfl_xor_sync(0xffffffffu, v, off));
  if (TPR > 32) {
    constexpr int G = TPR > 32 ? TPR / 32 : 1;  // warps per row group
    const int warp = threadIdx.x >> 5, g0 = (warp / G) * G;
    if ((threadIdx.x & 31) == 0) s_rw[warp] = v;
    __syncthreads();
    v = s_rw[g0];
#pragma unroll
    for (int i = 1; i < G; ++i) v = red_combine(OP, v, s_rw[g0 + i]);
    __syncthreads();
  }
  return v;
}


__device__ __forceinline__ u64 atom_add_acq_rel64(u64* p, u64 v) {
  u64 old;
  asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}
__device__ __forceinline__ u64 ld_acquire64(const u64* p) {
  u64 v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release64(u64* p, u64 v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Scratch layout behind P.barrier (zeroed once, reused by every launch); the
// arrivals and the broadcast sit on separate 128-byte lines:
//   +0    u64 arrival counter (monotonic across launches and passes)
//   +16   int status (1 = barrier timeout)
//   +32   u64 [launches, mispredictions, exact entries] (speculative regions)
//   +56   int prediction confidence (speculate when >= 2)
//   +288  int predicted decisions of a speculative region
// and P.partials = double[slot][gridDim.x] at +GM_SCRATCH_PARTIALS.
#define GM_SCRATCH_STATS 32     // u64 [launches, mispredictions, exact entries] (speculative regions)
#define GM_SCRATCH_CONF 56      // int prediction confidence (adaptive speculation)
#define GM_SCRATCH_FORCE 60     // int diagnostics: bit j flips predicted decision j, bit 29 turns
                                // the live timer on, bit 30 forces the exact entry, bit 31 the
                                // speculative one (tests, bench timing)
#define GM_SCRATCH_LIVE 256     // u64 [start ns, exits, sum of durations ns, launches] (live timer)
#define GM_LIVE_BIT (1 << 29)
#define GM_SCRATCH_FLAG 128     // (free: tools/barrier_bench.py protocol variants)
#define GM_SCRATCH_RESULTS 136
#define GM_SCRATCH_PRED 288     // int[24] predicted decisions (speculative regions)
#define GM_SCRATCH_SUBCNT 384   // u64 arrival sub-counters, one per 128-byte line
#define GM_SCRATCH_PARTIALS 2432
// Arrival split: CTA b arrives on sub-counter b % GM_ARRIVE_SPLIT (separate
// L2 lines), so no single address takes all 296 atomics; warp 0 polls the
// sub-counters lane-parallel.  1 = one counter at +0.
#ifndef GM_ARRIVE_SPLIT
#define GM_ARRIVE_SPLIT 1
#endif
static_assert(GM_ARRIVE_SPLIT >= 1 && GM_ARRIVE_SPLIT <= 16, "16 sub-counter lines between +384 and the partials");
// Arrival as a fire-and-forget `red.release` (1) or a returning
// `atom.acq_rel` (0).  With `red`, thread 0 knows its epoch from the counter
// value read at kernel start (grid_epoch_begin): before a CTA's own first
// arrival at most gridDim.x - 1 arrivals of this launch can have landed, so
// count / gridDim.x is the epoch every CTA of the launch agrees on.
#ifndef GM_ARRIVE_RED
#define GM_ARRIVE_RED 0
#endif

// GM_PROF: optional timeline stamps (atomicMax over CTAs) for diagnostics
#ifdef GM_PROF
#define GM_STAMP(i) do { if (threadIdx.x == 0 && prof) atomicMax(&prof[i], globaltimer()); } while (0)
#else
#define GM_STAMP(i) do { (void)prof; } while (0)
#endif

__device__ __forceinline__ double warp_combine(int op, double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = red_combine(op, v, __shfl_xor_sync(0xffffffffu, v, off));
  return v;
}

__device__ __forceinline__ u64 ld_relaxed64(const u64* p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ void grid_reduce(const Params& P, int nr, const int* ops, const int* slots,
                                            double* vals, double* s_warp, double* s_out, u64& ep,
                                            u64* prof = nullptr);

// Thread 0's view of the arrival counter at kernel start (see GM_ARRIVE_RED);
// the load is consumed only at the first arrival, so it overlaps the pass.
__device__ __forceinline__ u64 grid_epoch_begin(const Params& P) {
  return (threadIdx.x == 0 && gridDim.x > 1) ? ld_relaxed64((const u64*)P.barrier) : 0ull;
}

// First half of grid_reduce: the CTA partials are published and the CTA
// arrives.  Returns the arrival target (thread 0; 0 elsewhere, and for a
// one-CTA grid, whose results are already in s_out).  Stores a thread issues
// between grid_arrive and grid_wait are not ordered before the arrival's
// release, so the generated passes issue their output stores there: the
// release does not wait for them to drain and they overlap the barrier.
__device__ __forceinline__ u64 grid_arrive(const Params& P, int nr, const int* ops, const int* slots,
                                           double* vals, double* s_warp, double* s_out, u64& ep,
                                           u64* prof = nullptr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int r = 0; r < nr; ++r) {
    const double v = warp_combine(ops[r], vals[r]);
    if (lane == 0) s_warp[warp * GM_MAX_RED + r] = v;
  }
  __syncthreads();
  double* partials = (double*)P.partials;
  const bool multi = gridDim.x > 1;
  if (warp == 0) {
#pragma unroll
    for (int r = 0; r < nr; ++r) {
      double v = lane < GM_WARPS ? s_warp[lane * GM_MAX_RED + r] : red_identity(ops[r]);
      v = warp_combine(ops[r], v);
      if (lane == 0) {
        if (multi)
          partials[(i64)slots[r] * gridDim.x + blockIdx.x] = v;
        else
          s_out[r] = v;
      }
    }
  }
  if (!multi) return 0;
  GM_STAMP(0);
  u64 target = 0;
  if (threadIdx.x == 0) {
#if GM_ARRIVE_SPLIT > 1
    const u32 S = GM_ARRIVE_SPLIT, i = blockIdx.x % S;
    const u64 gi = (gridDim.x - i + S - 1) / S;  // CTAs arriving on sub-counter i
    const u64 old = atom_add_acq_rel64((u64*)(P.barrier + GM_SCRATCH_SUBCNT + 128 * i), 1ull);
    target = old / gi + 1;  // the epoch this arrival completes
#elif GM_ARRIVE_RED
    const u64 g = gridDim.x;
    target = (ep / g + 1) * g;
    ep = target;
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"((u64*)P.barrier) : "memory");
#else
    const u64 g = gridDim.x;
    const u64 old = atom_add_acq_rel64((u64*)P.barrier, 1ull);
    target = (old / g + 1) * g;
    (void)ep;
#endif
#ifdef GM_PROF
    if (prof) atomicMax(&prof[3], globaltimer());  // arrival completed (after the release)
#endif
  }
  return target;
}

// Second half: thread 0 waits for the epoch (relaxed polls, one acquire
// fence), then every CTA combines all partials itself in the same fixed
// order (bit-identical results in every CTA, no second round trip).
__device__ __forceinline__ void grid_wait(const Params& P, int nr, const int* ops, const int* slots, u64 target,
                                          double* s_out, u64* prof = nullptr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (gridDim.x == 1) {
    __syncthreads();
    return;
  }
#if GM_ARRIVE_SPLIT > 1
  if (warp == 0) {
    const u32 S = GM_ARRIVE_SPLIT;
    const u64 epoch = __shfl_sync(0xffffffffu, target, 0);
    const u64 gi = lane < (int)S ? (gridDim.x - lane + S - 1) / S : 0;
    const u64 want = epoch * gi;
    const u64* cnt = (const u64*)(P.barrier + GM_SCRATCH_SUBCNT + 128 * (lane < (int)S ? lane : 0));
    const u64 t0 = globaltimer();
    int spins = 0;
    while (true) {
      const bool ok = lane >= (int)S || ld_relaxed64(cnt) >= want;
      if (__all_sync(0xffffffffu, ok)) break;
      if ((++spins & 1023) == 0 && globaltimer() - t0 > 2000000000ull) {
        if (lane == 0) *(volatile int*)P.status = 1;
        break;
      }
    }
    fence_acq_rel_gpu();
  }
#else
  if (threadIdx.x == 0) {
    u64* cnt = (u64*)P.barrier;
    const u64 t0 = globaltimer();
    int spins = 0;
    while (ld_relaxed64(cnt) < target) {
      if ((++spins & 1023) == 0 && globaltimer() - t0 > 2000000000ull) {
        *(volatile int*)P.status = 1;
        break;
      }
    }
    fence_acq_rel_gpu();
  }
#endif
  __syncthreads();
  GM_STAMP(1);
  const double* partials = (const double*)P.partials;
  // reduction r is combined by warp r % GM_WARPS; the loop over r is
  // unrolled at the (constant) call sites, so ops[]/slots[] stay registers
#pragma unroll
  for (int r = 0; r < nr; ++r) {
    if (r % GM_WARPS != warp) continue;
    const double* base = partials + (i64)slots[r] * gridDim.x;
    double acc = red_identity(ops[r]);
    for (u32 b0 = 0; b0 < gridDim.x; b0 += 32 * 16) {
      double t[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const u32 b = b0 + i * 32 + lane;
        t[i] = b < gridDim.x ? ld_relaxed_f64(base + b) : red_identity(ops[r]);
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) acc = red_combine(ops[r], acc, t[i]);
    }
    acc = warp_combine(ops[r], acc);
    if (lane == 0) s_out[r] = acc;
  }
  __syncthreads();
  GM_STAMP(2);
}

// Final reduction of a launch (its results feed only scalar outputs): the
// CTA whose arrival completes the epoch combines the partials alone; the
// others return false and may exit — nobody polls.  Same fixed combine
// order as grid_wait, so the statistics are bit-identical to it.
__device__ __forceinline__ bool grid_reduce_last(const Params& P, int nr, const int* ops, const int* slots,
                                                 double* vals, double* s_warp, double* s_out, u64& ep,
                                                 u64* prof = nullptr) {
  __shared__ int s_last_;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int r = 0; r < nr; ++r) {
    const double v = warp_combine(ops[r], vals[r]);
    if (lane == 0) s_warp[warp * GM_MAX_RED + r] = v;
  }
  __syncthreads();
  const bool multi = gridDim.x > 1;
  double* partials = (double*)P.partials;
  if (warp == 0) {
#pragma unroll
    for (int r = 0; r < nr; ++r) {
      double v = lane < GM_WARPS ? s_warp[lane * GM_MAX_RED + r] : red_identity(ops[r]);
      v = warp_combine(ops[r], v);
      if (lane == 0) {
        if (multi)
          partials[(i64)slots[r] * gridDim.x + blockIdx.x] = v;
        else
          s_out[r] = v;
      }
    }
  }
  if (!multi) {
    __syncthreads();
    return true;
  }
  if (threadIdx.x == 0) {
    const u64 old = atom_add_acq_rel64((u64*)P.barrier, 1ull);
    s_last_ = (old % gridDim.x) == gridDim.x - 1;
    (void)ep;
  }
  __syncthreads();
  if (!s_last_) return false;
#pragma unroll
  for (int r = 0; r < nr; ++r) {
    if (r % GM_WARPS != warp) continue;
    const double* base = partials + (i64)slots[r] * gridDim.x;
    double acc = red_identity(ops[r]);
    for (u32 b0 = 0; b0 < gridDim.x; b0 += 32 * 16) {
      double t[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const u32 b = b0 + i * 32 + lane;
        t[i] = b < gridDim.x ? ld_relaxed_f64(base + b) : red_identity(ops[r]);
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) acc = red_combine(ops[r], acc, t[i]);
    }
    acc = warp_combine(ops[r], acc);
    if (lane == 0) s_out[r] = acc;
  }
  __syncthreads();
  GM_STAMP(2);
  return true;
}

// Reduce `nr` per-thread values across the grid; the results land in s_out[r]
// in every CTA.
//   1. CTA partial: warp butterfly, then warp 0 over the warps (fixed tree);
//      thread 0 stores the partials and arrives on the arrival counter
//      (atom.acq_rel: the partial stores are released with the arrival).
//   2. Thread 0 polls the counter (relaxed loads, one acquire fence after)
//      until it reaches the next multiple of gridDim.x — the counter is
//      monotonic across passes and launches, so it never needs a reset.
//   3. Every CTA combines all partials itself: warp r handles reduction r,
//      16 independent loads per lane per round, then a fixed butterfly.
// Same inputs, same tree in every CTA: bit-identical results everywhere and
// in every run, with no second round trip to publish them (measured on
// B200 by tools/barrier_bench.py: ~2.5 us per reduce at 296 CTAs, against
// ~3.5 us for a last-arriver combine + broadcast).  The grid is sized to be
// co-resident (<= SMs x occupancy); a 2 s %globaltimer bound turns a
// residency violation into status=1, not a hang.
__device__ __forceinline__ void grid_reduce(const Params& P, int nr, const int* ops, const int* slots,
                                            double* vals, double* s_warp, double* s_out, u64& ep, u64* prof) {
  const u64 target = grid_arrive(P, nr, ops, slots, vals, s_warp, s_out, ep, prof);
  grid_wait(P, nr, ops, slots, target, s_out, prof);
}

// argmax / argmin as a max over ordered 64-bit keys: the high word orders
// the values (NaN above everything, as torch's argmax/argmin return the
// first NaN; -0.0 folded onto +0.0), the low word is ~index so the first
// occurrence wins a tie.  Identity 0; combined by GM_R_KEYMAX.
__device__ __forceinline__ u32 order_key(float x, bool for_min) {
  if (x != x) return 0xffffffffu;
  if (x == 0.f) x = 0.f;
  u32 b = __float_as_uint(x);
  b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);  // monotone in x
  return for_min ? ~b - 1u : b;                       // below the NaN key
}
__device__ __forceinline__ u64 argkey8(u64 acc, const float (&x)[8], i64 e, int nv, bool for_min) {
#pragma unroll
  for (int l = 0; l < GM_VEC; ++l) {
    if (l < nv) {
      const u64 key = ((u64)order_key(x[l], for_min) << 32) | (u64)(0xffffffffu - (u32)(e + l));
      acc = key > acc ? key : acc;
    }
  }
  return acc;
}

// Per-thread float accumulation of one 8-lane vector (masked to nv lanes).
__device__ __forceinline__ float acc8(int op, float acc, const float (&x)[8], int nv) {
  float t;
  if (nv == GM_VEC) {
    switch (op) {
      case GM_R_MAX: t = nmax(nmax(nmax(x[0], x[1]), nmax(x[2], x[3])), nmax(nmax(x[4], x[5]), nmax(x[6], x[7]))); return nmax(acc, t);
      case GM_R_MIN: t = nmin(nmin(nmin(x[0], x[1]), nmin(x[2], x[3])), nmin(nmin(x[4], x[5]), nmin(x[6], x[7]))); return nmin(acc, t);
      case GM_R_PROD: t = ((x[0] * x[1]) * (x[2] * x[3])) * ((x[4] * x[5]) * (x[6] * x[7])); return acc * t;
      case GM_R_OR:
        return (acc != 0.f || x[0] != 0.f || x[1] != 0.f || x[2] != 0.f || x[3] != 0.f || x[4] != 0.f ||
                x[5] != 0.f || x[6] != 0.f || x[7] != 0.f) ? 1.f : 0.f;
      case GM_R_AND:
        return (acc != 0.f && x[0] != 0.f && x[1] != 0.f && x[2] != 0.f && x[3] != 0.f && x[4] != 0.f &&
                x[5] != 0.f && x[6] != 0.f && x[7] != 0.f) ? 1.f : 0.f;
      default: t = ((x[0] + x[1]) + (x[2] + x[3])) + ((x[4] + x[5]) + (x[6] + x[7])); return acc + t;
    }
  }
#pragma unroll
  for (int k = 0; k < GM_VEC; ++k) {
    if (k >= nv) break;
    switch (op) {
      case GM_R_MAX: acc = nmax(acc, x[k]); break;
      case GM_R_MIN: acc = nmin(acc, x[k]); break;
      case GM_R_PROD: acc = acc * x[k]; break;
      case GM_R_OR: acc = (acc != 0.f || x[k] != 0.f) ? 1.f : 0.f; break;
      case GM_R_AND: acc = (acc != 0.f && x[k] != 0.f) ? 1.f : 0.f; break;
      default: acc = acc + x[k]; break;
    }
  }
  return acc;
}
// Live timer (diagnostics word bit 29, set by bench.py for its timed loop):
// CTA 0 stamps %globaltimer after griddepcontrol.wait; every CTA's thread 0
// counts its exit, and the CTA completing a launch's count adds
// (its stamp - the start) to a running sum — the kernel's own duration
// inside the forward's graph, with no event nodes between kernels.
__device__ __forceinline__ void live_start(const Params& P) {
  if (blockIdx.x == 0) *(volatile u64*)(P.barrier + GM_SCRATCH_LIVE) = globaltimer();
}
__device__ __forceinline__ void live_exit(const Params& P) {
  u64* lt = (u64*)(P.barrier + GM_SCRATCH_LIVE);
  const u64 old = atomicAdd((unsigned long long*)&lt[1], 1ull);
  if ((old + 1) % gridDim.x == 0) {
    const u64 t1 = globaltimer(), t0 = ld_relaxed64(lt);
    atomicAdd((unsigned long long*)&lt[2], (unsigned long long)(t1 - t0));
    atomicAdd((unsigned long long*)&lt[3], 1ull);
  }
}

// CTA-wide combine (every thread returns the result); s_w holds GM_WARPS
// doubles.  Used by the sampled branch predictor (codegen.Plan._emit_sample).
__device__ __forceinline__ double cta_combine(int op, double v, double* s_w) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_combine(op, v);
  if (lane == 0) s_w[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double t = lane < GM_WARPS ? s_w[lane] : red_identity(op);
    t = warp_combine(op, t);
    if (lane == 0) s_w[GM_WARPS] = t;
  }
  __syncthreads();
  const double r = s_w[GM_WARPS];
  __syncthreads();
  return r;
}
// CTA-wide sum of two doubles at once (one set of barriers); s_w holds
// 2 * GM_WARPS + 2 doubles.
__device__ __forceinline__ void cta_sum2(double& a, double& b, double* s_w) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, off);
    b += __shfl_xor_sync(0xffffffffu, b, off);
  }
  if (lane == 0) { s_w[2 * warp] = a; s_w[2 * warp + 1] = b; }
  __syncthreads();
  if (warp == 0) {
    double x = lane < GM_WARPS ? s_w[2 * lane] : 0.0, y = lane < GM_WARPS ? s_w[2 * lane + 1] : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      x += __shfl_xor_sync(0xffffffffu, x, off);
      y += __shfl_xor_sync(0xffffffffu, y, off);
    }
    if (lane == 0) { s_w[2 * GM_WARPS] = x; s_w[2 * GM_WARPS + 1] = y; }
  }
  __syncthreads();
  a = s_w[2 * GM_WARPS];
  b = s_w[2 * GM_WARPS + 1];
  __syncthreads();
}
__device__ __forceinline__ float acc_identity(int op) {
  switch (op) {
    case GM_R_MAX: return -__int_as_float(0x7f800000);
    case GM_R_MIN: return __int_as_float(0x7f800000);
    case GM_R_PROD: return 1.f;
    case GM_R_AND: return 1.f;
    default: return 0.f;
  }
}

}  // namespace gm
