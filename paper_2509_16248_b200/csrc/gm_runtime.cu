// gm_runtime.cu — libgm_b200.so: the C ABI declared in include/gm_b200.h.
//
//  * region compiler/loader: NVRTC -> sm_100a cubin -> driver module (libcuda
//    resolved with dlopen so the library loads on GPU-less hosts);
//    the generated sources include the hand-written skeleton gm_region.cuh,
//    which is embedded here as an NVRTC header (gm_region_cuh.inc, produced
//    by the build from the same file nvcc compiles below);
//  * gm_branch_select_f32: the canonical predicated block of the corpus
//    (corpus/phi4_like/original.py:8-11 after transform.py:359-376) as a
//    precompiled instance of the same skeleton;
//  * the log ring: pinned, device-mapped host memory, a gather kernel for the
//    elements torch's repr reads, and a stream-ordered step commit.

#include <cub/device/device_radix_sort.cuh>
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <dlfcn.h>

#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <cstdint>

#include "../../include/gm_b200.h"
#include "gm_region.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[2048];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define GM_CUDA(call)                                                                         \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess) return fail(GM_E_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

#define GM_CU(call)                                                         \
  do {                                                                      \
    CUresult r_ = (call);                                                   \
    if (r_ != CUDA_SUCCESS) {                                               \
      const char* s_ = nullptr;                                             \
      g_drv.GetErrorString(r_, &s_);                                          \
      return fail(GM_E_CUDA, "%s: %s", #call, s_ ? s_ : "unknown error"); \
    }                                                                       \
  } while (0)

// Driver API entry points, resolved with dlopen so the library loads (and the
// CPU test-suite can check its exports) on hosts without a GPU driver.
struct DriverApi {
  CUresult (*ModuleLoadData)(CUmodule*, const void*) = nullptr;
  CUresult (*ModuleGetFunction)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*ModuleUnload)(CUmodule) = nullptr;
  CUresult (*LaunchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                           CUstream, void**, void**) = nullptr;
  CUresult (*LaunchKernelEx)(const CUlaunchConfig*, CUfunction, void**, void**) = nullptr;
  CUresult (*FuncSetAttribute)(CUfunction, CUfunction_attribute, int) = nullptr;
  CUresult (*OccupancyMaxActiveBlocksPerMultiprocessor)(int*, CUfunction, int, size_t) = nullptr;
  CUresult (*CtxGetCurrent)(CUcontext*) = nullptr;
  CUresult (*GetErrorString)(CUresult, const char**) = nullptr;
  bool loaded = false;
} g_drv;

int load_driver() {
  if (g_drv.loaded) return 0;
  void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return -1;
#define GM_SYM(field, name) g_drv.field = (decltype(g_drv.field))dlsym(h, name); if (!g_drv.field) return -1;
  GM_SYM(ModuleLoadData, "cuModuleLoadData");
  GM_SYM(ModuleGetFunction, "cuModuleGetFunction");
  GM_SYM(ModuleUnload, "cuModuleUnload");
  GM_SYM(LaunchKernel, "cuLaunchKernel");
  GM_SYM(LaunchKernelEx, "cuLaunchKernelEx");
  GM_SYM(FuncSetAttribute, "cuFuncSetAttribute");
  GM_SYM(OccupancyMaxActiveBlocksPerMultiprocessor, "cuOccupancyMaxActiveBlocksPerMultiprocessor");
  GM_SYM(CtxGetCurrent, "cuCtxGetCurrent");
  GM_SYM(GetErrorString, "cuGetErrorString");
#undef GM_SYM
  g_drv.loaded = true;
  return 0;
}

const char kRegionHeader[] =
#include "gm_region_cuh.inc"
    ;

int g_cc_major = 0, g_cc_minor = 0, g_num_sms = 0, g_smem_optin = 0, g_device = -1;

}  // namespace

// shared with gm_gemm.cu: one thread-local error slot behind gm_last_error()
int gm_internal_fail(int code, const char* msg) { return fail(code, "%s", msg); }

struct gm_region_s {
  CUmodule mod = nullptr;
  CUfunction fn = nullptr;
  int smem = 0;
};

// one record of a step template (gm_logring_capture)
struct GmRecordDesc {
  uint32_t id;
  int dtype, ndim;
  int64_t shape[GM_MAX_DIMS], counts[GM_MAX_DIMS], heads[GM_MAX_DIMS];
  uint64_t offset, bytes;
};

struct gm_logring_s {
  void* host = nullptr;             // pinned, mapped ring
  void* dev = nullptr;              // device alias of `host`
  size_t bytes = 0;
  unsigned long long* dstep = nullptr;       // device step counter
  volatile unsigned long long* hcommit = nullptr;  // mapped: committed steps
  unsigned long long* dcommit = nullptr;     // device alias of hcommit
  // record-level API: GM_LOGRING_SLOTS slots of slot_bytes, each starting
  // with a GM_LOGRING_HEADER-byte header the step commit writes
  uint64_t slot_bytes = 0;
  std::vector<std::vector<GmRecordDesc>> templates;  // template id -> records
  std::vector<GmRecordDesc> open;                    // the step being captured
  bool step_open = false;
  uint64_t cursor = GM_LOGRING_HEADER;
  uint64_t drained = 0;                              // steps delivered by gm_logring_drain
};

// ===========================================================================
// precompiled canonical branch-select (skeleton instance)
// ===========================================================================
namespace {

struct BsArgs {
  int red, cmp;
  double thr, a1, b1, a2, b2;
  double* stat_out;
};

__global__ void __launch_bounds__(GM_THREADS, 1)
    gm_branch_select_f32_kernel(const __grid_constant__ gm::Params P, const __grid_constant__ BsArgs A) {
  using namespace gm;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ u64 s_bars[2 * GM_MAX_PIECES];
  __shared__ double s_warp[GM_WARPS * GM_MAX_RED];
  __shared__ double s_red[GM_MAX_RED];
  const i64 v0 = (i64)blockIdx.x * P.vpc;
  const i64 v1 = (v0 + P.vpc < P.nvec) ? v0 + P.vpc : P.nvec;
  const bool resident = P.in[0].smem_off >= 0;
  const unsigned sres = resident ? smem_u32(smem + P.in[0].smem_off) : 0u;
  u64 ep_ = grid_epoch_begin(P);
  Stage st, st_unused;
  st.wend = st_unused.wend = 0;
  st.bars = s_bars;
  st_unused.bars = s_bars + GM_MAX_PIECES;
  const int es[1] = {4};
  const int grp[1] = {resident ? 0 : -1};
  if (resident) stage_issue(P, smem, 1, es, grp, v0, v1, st, st_unused);
  const int op = (A.red == 2) ? GM_R_MAX : (A.red == 3) ? GM_R_MIN : GM_R_SUM;
  // pass 0: statistic of x
  float acc = acc_identity(op);
  for (i64 v = v0 + threadIdx.x; v < v1; v += GM_THREADS) {
    const i64 e = v * GM_VEC;
    const int nv = (int)((P.n - e) < GM_VEC ? (P.n - e) : GM_VEC);
    if (resident) stage_wait(st, v - v0);
    float x[GM_VEC];
    load8<GM_DT_F32>(P.in[0], sres, e, e - v0 * GM_VEC, nv, x);
    if (A.red == 4) {
#pragma unroll
      for (int k = 0; k < GM_VEC; ++k) x[k] = x[k] * x[k];
    }
    acc = acc8(op, acc, x, nv);
  }
  if (resident) stage_finish(st);
  double vals[1] = {(double)acc};
  const int ops[1] = {op};
  const int slots[1] = {0};
  grid_reduce(P, 1, ops, slots, vals, s_warp, s_red, ep_);
  // statistic in T's dtype (fp32), compared with the threshold cast to fp32
  const double r = s_red[0];
  float stat;
  if (A.red == 1) stat = __fdiv_rn((float)r, (float)P.n);
  else if (A.red == 4) stat = (float)sqrt(r);
  else stat = (float)r;
  const float thr = (float)A.thr;
  const bool pred = (A.cmp == 0) ? stat > thr : (A.cmp == 1) ? stat >= thr : (A.cmp == 2) ? stat < thr : stat <= thr;
  if (blockIdx.x == 0 && threadIdx.x == 0 && A.stat_out) {
    A.stat_out[0] = (double)stat;
    A.stat_out[1] = pred ? 1.0 : 0.0;
  }
  const float sa = pred ? (float)A.a1 : (float)A.a2;
  const float sb = pred ? (float)A.b1 : (float)A.b2;
  // pass 1: only the selected arm is evaluated (the predicate is uniform)
  for (i64 v = v0 + threadIdx.x; v < v1; v += GM_THREADS) {
    const i64 e = v * GM_VEC;
    const int nv = (int)((P.n - e) < GM_VEC ? (P.n - e) : GM_VEC);
    float x[GM_VEC], y[GM_VEC];
    load8<GM_DT_F32>(P.in[0], sres, e, e - v0 * GM_VEC, nv, x);
#pragma unroll
    for (int k = 0; k < GM_VEC; ++k) y[k] = add(mul(x[k], sa), sb);
    store8<GM_DT_F32>(P.out[0], e, nv, y);
  }
}

// ===========================================================================
// log ring kernels
// ===========================================================================
struct GatherArgs {
  const void* src;
  void* ring_dev;
  const unsigned long long* dstep;
  unsigned long long step_bytes, n_slots, offset;
  long long total;  // number of gathered elements
  int dtype, ndim, esize, pad;
  long long count[GM_MAX_DIMS], head[GM_MAX_DIMS], size[GM_MAX_DIMS], stride[GM_MAX_DIMS];
};

__global__ void gm_logring_gather_kernel(const __grid_constant__ GatherArgs A) {
  const unsigned long long step = *A.dstep;
  char* dst = (char*)A.ring_dev + (step % A.n_slots) * A.step_bytes + A.offset;
  for (long long t = threadIdx.x; t < A.total; t += blockDim.x) {
    long long rem = t, off = 0;
    for (int d = A.ndim - 1; d >= 0; --d) {
      const long long k = rem % A.count[d];
      rem /= A.count[d];
      const long long idx = (k < A.head[d]) ? k : (A.size[d] - A.count[d] + k);
      off += idx * A.stride[d];
    }
    const char* s = (const char*)A.src + off * A.esize;
    switch (A.esize) {
      case 1: ((unsigned char*)dst)[t] = *(const unsigned char*)s; break;
      case 2: ((unsigned short*)dst)[t] = *(const unsigned short*)s; break;
      case 4: ((unsigned int*)dst)[t] = *(const unsigned int*)s; break;
      default: ((unsigned long long*)dst)[t] = *(const unsigned long long*)s; break;
    }
  }
}

// Record-level step commit: write the slot header {template id, record
// count, 1-based step number} behind the step's gathers, then advance the
// device slot counter and its mapped host mirror.  System-scope fences order
// the gathered data and the header before the counter the drain polls.
struct GmSlotHeader {
  unsigned long long step;
  unsigned template_id, n_records;
};

__global__ void gm_logring_commit_step_kernel(unsigned long long* dstep, unsigned long long* dcommit, char* ring_dev,
                                              unsigned long long slot_bytes, unsigned long long n_slots,
                                              unsigned template_id, unsigned n_records) {
  const unsigned long long s = *dstep;
  GmSlotHeader* h = (GmSlotHeader*)(ring_dev + (s % n_slots) * slot_bytes);
  h->template_id = template_id;
  h->n_records = n_records;
  __threadfence_system();
  *(volatile unsigned long long*)&h->step = s + 1;
  *dstep = s + 1;
  __threadfence_system();
  *(volatile unsigned long long*)dcommit = s + 1;
}

// Advance the slot counter after a step's gathers (stream ordered).  The
// host learns completion from a CUDA event, so no system-scope fence here.
__global__ void gm_logring_commit_kernel(unsigned long long* dstep, unsigned long long* dcommit) {
  const unsigned long long s = *dstep + 1;
  *dstep = s;
  *(volatile unsigned long long*)dcommit = s;
}

// ---------------------------------------------------------------------------
// distinct-value sum of a 16-bit float tensor — `x.unique().sum()` after the
// lowering's rank-1 rewrite (corpus/moe_minicpm_like: unique consumed only by
// .sum()).  A 16-bit type has 65536 bit patterns, so the distinct set is a
// 8 KB presence bitmap: each CTA marks its elements in a shared bitmap
// (test-then-atomicOr, so repeated values cost a shared load), ORs the
// non-empty words into the global bitmap, and one CTA sums the values of
// the set bits in bit order (fp64, fixed tree: deterministic).  -0 is
// folded onto +0 (torch.unique treats them as equal).  One pass over x,
// no sort, no data-dependent shapes.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void u16_mark(unsigned* bits, unsigned h) {
  if (h == 0x8000u) h = 0;
  const unsigned m = 1u << (h & 31);
  unsigned* p = bits + (h >> 5);
  if (!(*(volatile unsigned*)p & m)) atomicOr(p, m);
}

__global__ void __launch_bounds__(512) gm_unique16_mark_kernel(const uint4* __restrict__ x, long long nvec,
                                                               const unsigned short* __restrict__ tail, int ntail,
                                                               unsigned* __restrict__ gbits) {
  __shared__ unsigned bits[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) bits[i] = 0;
  __syncthreads();
  const long long T = (long long)gridDim.x * blockDim.x;
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += T) {
    unsigned a, b, c, d;
    gm::ldg16(x + v, a, b, c, d);
    const unsigned w[4] = {a, b, c, d};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      u16_mark(bits, w[j] & 0xffffu);
      u16_mark(bits, w[j] >> 16);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < ntail) u16_mark(bits, tail[threadIdx.x]);
  __syncthreads();
  for (int i = threadIdx.x; i < 2048; i += blockDim.x)
    if (bits[i]) atomicOr(gbits + i, bits[i]);
}

__global__ void __launch_bounds__(1024) gm_unique16_sum_kernel(const unsigned* __restrict__ gbits, int dtype,
                                                               void* out) {
  __shared__ double part[32];
  double acc = 0.0;
  for (int wi = threadIdx.x; wi < 2048; wi += blockDim.x) {
    unsigned b = gbits[wi];
    while (b) {
      const int k = __ffs(b) - 1;
      b &= b - 1;
      const unsigned short h = (unsigned short)(wi * 32 + k);
      acc += (double)(dtype == GM_BF16 ? gm::bf2f(h) : gm::h2f(h));
    }
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) {
      const float f = (float)t;
      *(unsigned short*)out = dtype == GM_BF16 ? gm::f2bf(f) : gm::f2h(f);
    }
  }
}

// fp32: sort (CUB radix sort, by value bits) then one pass that sums the
// first element of every run of equal values — fixed shapes, no host sync.
// Per-thread fp64 partials over a fixed grid-stride assignment, per-CTA
// partials in a fixed tree, then one CTA over the CTA partials: deterministic.
__global__ void __launch_bounds__(512) gm_distinct_sum32_kernel(const float* __restrict__ s, long long n,
                                                               double* __restrict__ partials) {
  __shared__ double part[16];
  double acc = 0.0;
  const long long T = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += T) {
    const float v = s[i];
    if (i == 0 || v != s[i - 1]) acc += (double)v;
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) partials[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(1024) gm_sum_partials_kernel(const double* __restrict__ partials, int np,
                                                               float* __restrict__ out) {
  __shared__ double part[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) acc += partials[i];
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) *out = (float)t;
  }
}

// fp32, sort-free distinct sum.  Deduplication: values whose binade lies in
// a window of GM_U32_WIN binades (placed from the previous call's largest
// finite exponent) set one bit of a presence bitmap (sign x binade x 2^23 mantissas; red.or, so a
// duplicate is free); the rest go to a hash set of the value bits (open
// addressing, 64-bit slots = call tag << 32 | bits, so a slot written by an
// earlier call reads as empty and the table is never cleared).  Summation is
// EXACT: v = M * 2^shift * 2^-149 with M < 2^24 is added into a fixed-point
// super-accumulator of 32-bit digits held in int64 (per thread in local
// memory, per CTA in shared memory, per call in global memory) — integer
// sums, so the result does not depend on which thread saw a value first.
// The bitmap pass sums the mantissas of the set bits per binade (an exact
// int64) and clears the words it read, ready for the next call.  The finish
// rounds the exact sum once to fp32 (nearest-even).  NaN anywhere -> NaN;
// +inf and -inf -> NaN; one infinity -> it.
#define GM_U32_DIGITS 11
#define GM_U32_WIN 16
#define GM_U32_BITMAP_WORDS (2ull * GM_U32_WIN << 18)   // 2 signs x WIN binades x 2^23 bits
__device__ __forceinline__ unsigned gm_hash32(unsigned x) {
  x ^= x >> 16; x *= 0x85ebca6bu; x ^= x >> 13; x *= 0xc2b2ae35u; x ^= x >> 16;
  return x;
}

// acc += (neg ? -1 : 1) * S * 2^shift (S < 2^48), digits of 32 bits
__device__ __forceinline__ void gm_u32_acc_add(long long* acc, unsigned long long S, int shift, bool neg) {
  const int d = shift >> 5, off = shift & 31;
  const unsigned long long lo = (S & 0xffffffffull) << off, hi = (S >> 32) << off;
  long long a0 = (long long)(lo & 0xffffffffull), a1 = (long long)(lo >> 32) + (long long)(hi & 0xffffffffull),
            a2 = (long long)(hi >> 32);
  if (neg) { a0 = -a0; a1 = -a1; a2 = -a2; }
  acc[d] += a0; acc[d + 1] += a1;
  if (d + 2 < GM_U32_DIGITS) acc[d + 2] += a2;
}

// CTA total of the per-thread digit arrays -> global atomics.  Warp sums by
// shuffle, then one thread per digit adds the warps' sums (64-bit shared
// atomics are CAS loops on this GPU — 512-way contention on them is slow).
__device__ __forceinline__ void gm_u32_flush(long long* acc, long long (*swarp)[GM_U32_DIGITS],
                                             long long* digits) {
#pragma unroll
  for (int d = 0; d < GM_U32_DIGITS; ++d) {
    long long v = acc[d];
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) swarp[threadIdx.x >> 5][d] = v;
  }
  __syncthreads();
  if (threadIdx.x < GM_U32_DIGITS) {
    long long v = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += swarp[w][threadIdx.x];
    if (v) atomicAdd((unsigned long long*)&digits[threadIdx.x], (unsigned long long)v);
  }
}

// largest biased exponent among finite values -> *emax (atomicMax; memset 0)
// — only with GM_U32_WINDOW_PASS=1 (the window of THIS call)
__global__ void __launch_bounds__(512) gm_unique32_window_kernel(const float* __restrict__ x, long long n,
                                                                 int* __restrict__ emax) {
  unsigned m = 0;
  const long long T = (long long)gridDim.x * blockDim.x, t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long n4 = ((uintptr_t)x & 15) ? 0 : n >> 2;
  auto fin = [](unsigned b) { const unsigned e = (b >> 23) & 0xff; return e == 255 ? 0u : e; };
#pragma unroll 4
  for (long long i = t0; i < n4; i += T) {
    const uint4 v = __ldcs(reinterpret_cast<const uint4*>(x) + i);
    m = max(m, max(max(fin(v.x), fin(v.y)), max(fin(v.z), fin(v.w))));
  }
  for (long long i = n4 * 4 + t0; i < n; i += T) {
    const unsigned e = (__float_as_uint(x[i]) >> 23) & 0xff;
    m = max(m, e == 255 ? 0u : e);
  }
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0 && m) atomicMax(emax, (int)m);
}

__global__ void __launch_bounds__(512) gm_unique32_insert_kernel(const float* __restrict__ x, long long n,
                                                                 unsigned* __restrict__ bitmap,
                                                                 const int* __restrict__ window_top, int head,
                                                                 int* __restrict__ emax_seen,
                                                                 unsigned long long* __restrict__ table,
                                                                 unsigned long long mask,
                                                                 const unsigned long long* __restrict__ calls,
                                                                 long long* __restrict__ digits,
                                                                 int* __restrict__ flags,
                                                                 unsigned* __restrict__ touched) {
  __shared__ long long swarp[16][GM_U32_DIGITS];
  const unsigned tag = (unsigned)(*calls % 0xffffffffull) + 1u;
  const int top_e = min(*window_top + head, 254), lo_e = max(top_e - (GM_U32_WIN - 1), 0);
  long long acc[GM_U32_DIGITS];
#pragma unroll
  for (int d = 0; d < GM_U32_DIGITS; ++d) acc[d] = 0;
  int fl = 0;
  unsigned seen = 0;                                     // largest finite exponent met
  unsigned tm = 0;                                       // bitmap slices (sign x binade) this thread marked
  // bitmap values: returns the bit index (the caller marks it); otherwise
  // handles the value (flags, hash set) and returns NONE
  constexpr unsigned long long NONE = ~0ull;
  auto one = [&](unsigned bits) -> unsigned long long {
    const unsigned e = (bits >> 23) & 0xffu;
    if (e == 255u) {                                     // inf / NaN
      fl |= (bits & 0x007fffffu) ? 1 : ((bits >> 31) ? 4 : 2);
      return NONE;
    }
    if ((bits & 0x7fffffffu) == 0) return NONE;          // +-0 adds nothing
    seen = max(seen, e);
    if ((int)e >= lo_e && (int)e <= top_e) {
      const unsigned slice = (bits >> 31) * GM_U32_WIN + (e - lo_e);
      tm |= 1u << slice;
      return ((unsigned long long)slice << 23) | (bits & 0x7fffffu);
    }
    const unsigned long long want = ((unsigned long long)tag << 32) | bits;
    unsigned long long h = gm_hash32(bits) & mask;
    while (true) {
      unsigned long long cur;
      asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(cur) : "l"(table + h) : "memory");
      if ((unsigned)(cur >> 32) == tag) {
        if ((unsigned)cur == bits) return NONE;          // seen
        h = (h + 1) & mask;
        continue;
      }
      if (atomicCAS(table + h, cur, want) == cur) break; // claimed: first occurrence
      // lost a race for this slot: re-examine it (it now holds this tag)
    }
    const unsigned fr = bits & 0x7fffffu;
    gm_u32_acc_add(acc, e ? (fr | 0x800000u) : fr, e ? (int)e - 1 : 0, bits >> 31);
    return NONE;
  };
  // mark a batch: read the words first (L1/L2; a word read stale shows a
  // subset of its bits, so a skipped red.or is always one already done) and
  // issue red.or only for bits not yet set — duplicates of hot values (a
  // narrow value range) would otherwise serialise on a few L2 lines
  auto mark = [&](const unsigned long long (&b)[4]) {
    unsigned w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) w[k] = b[k] != NONE ? __ldca(bitmap + (b[k] >> 5)) : ~0u;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (b[k] != NONE && !(w[k] >> (b[k] & 31) & 1u)) atomicOr(bitmap + (b[k] >> 5), 1u << (b[k] & 31));
  };
  const long long T = (long long)gridDim.x * blockDim.x, t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long n4 = ((uintptr_t)x & 15) ? 0 : n >> 2;
  // four 16-byte loads in flight per thread before any atomic is issued
  // (the hash path's relaxed loads would otherwise serialise the sweep)
  for (long long i = t0; i < n4; i += 4 * T) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      v[u] = i + u * T < n4 ? __ldcs(reinterpret_cast<const uint4*>(x) + i + u * T) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const unsigned long long b[4] = {one(v[u].x), one(v[u].y), one(v[u].z), one(v[u].w)};
      mark(b);
    }
  }
  for (long long i = n4 * 4 + t0; i < n; i += T) {
    const unsigned long long b[4] = {one(__float_as_uint(x[i])), NONE, NONE, NONE};
    mark(b);
  }
  if (fl) atomicOr(flags, fl);
  tm = __reduce_or_sync(0xffffffffu, tm);
  if ((threadIdx.x & 31) == 0 && tm) atomicOr(touched, tm);
  seen = __reduce_max_sync(0xffffffffu, seen);
  if ((threadIdx.x & 31) == 0 && seen) atomicMax(emax_seen, (int)seen);
  gm_u32_flush(acc, swarp, digits);
}

__device__ void gm_u32_finish(const long long* digits, const int* flags, unsigned long long* calls, float* out);

// sum the mantissas of the set bits of the presence bitmap, clearing it;
// the last CTA to finish rounds the call's total into *out
__global__ void __launch_bounds__(512) gm_unique32_bitmap_sum_kernel(uint4* __restrict__ bitmap,
                                                                     int* __restrict__ window_top, int head,
                                                                     const int* __restrict__ emax_seen,
                                                                     const unsigned* __restrict__ touched,
                                                                     long long* __restrict__ digits,
                                                                     unsigned* __restrict__ done,
                                                                     const int* __restrict__ flags,
                                                                     unsigned long long* __restrict__ calls,
                                                                     float* __restrict__ out) {
  __shared__ long long swarp[16][GM_U32_DIGITS];
  const int top_e = min(__ldcg(window_top) + head, 254), lo_e = max(top_e - (GM_U32_WIN - 1), 0);
  long long acc[GM_U32_DIGITS];
#pragma unroll
  for (int d = 0; d < GM_U32_DIGITS; ++d) acc[d] = 0;
  // only the slices some value marked are swept (untouched ones are zero):
  // virtual vector index v -> slice = the (v >> 16)-th set bit of `touched`
  const unsigned tmask = *touched;
  const long long nv = (long long)__popc(tmask) << 16, T = (long long)gridDim.x * blockDim.x;
  // each warp walks one contiguous chunk (lanes interleaved, so loads
  // coalesce) and so meets few binades
  const long long warps = T >> 5, wid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long per = ((nv + warps - 1) / warps + 31) & ~31ll;
  const long long v0 = wid * per + (threadIdx.x & 31), v1 = min(nv, wid * per + per);
  long long cur_b = -1;
  unsigned long long S = 0;
  auto flush_binade = [&]() {
    if (cur_b >= 0 && S) {
      const int e = lo_e + (int)(cur_b % GM_U32_WIN);
      if (e < 255) gm_u32_acc_add(acc, S, e ? e - 1 : 0, cur_b >= GM_U32_WIN);
    }
    S = 0;
  };
  auto real = [&](long long vv) -> long long {
    return ((long long)__fns(tmask, 0, (int)(vv >> 16) + 1) << 16) | (vv & 0xffff);
  };
  for (long long vb = v0; vb < v1; vb += 32 * 4) {
    uint4 qs[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) qs[u] = vb + 32 * u < v1 ? bitmap[real(vb + 32 * u)] : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long v = real(vb + 32 * u);
      const uint4 q = qs[u];
      if (!(q.x | q.y | q.z | q.w)) continue;
      bitmap[v] = make_uint4(0, 0, 0, 0);
      const long long b = (v * 4) >> 18;                   // sign * WIN + binade
      if (b != cur_b) { flush_binade(); cur_b = b; }
      const int e = lo_e + (int)(b % GM_U32_WIN);
      const unsigned base_m = e ? 0x800000u : 0u;
      const unsigned w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const unsigned x = w[k];
        if (!x) continue;
        const unsigned j = (unsigned)((v * 4 + k) & ((1 << 18) - 1));   // word within the binade
        const unsigned idx_sum = __popc(x & 0xaaaaaaaau) + 2 * __popc(x & 0xccccccccu) + 4 * __popc(x & 0xf0f0f0f0u) +
                                 8 * __popc(x & 0xff00ff00u) + 16 * __popc(x & 0xffff0000u);
        S += (unsigned long long)__popc(x) * (base_m + j * 32u) + idx_sum;
      }
    }
  }
  flush_binade();
  gm_u32_flush(acc, swarp, digits);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(done, 1u) == gridDim.x - 1) {
      __threadfence();
      gm_u32_finish(digits, flags, calls, out);
      // predicted mode: the next call's window sits under this call's
      // largest exponent (every CTA read the old value before arriving)
      if (head) *window_top = __ldcg(emax_seen);
    }
  }
}

// one thread: round the exact sum to fp32 (or the NaN/inf outcome) -> *out
__device__ void gm_u32_finish(const long long* digits, const int* flags, unsigned long long* calls, float* out) {
  const int fl = __ldcg(flags);
  float r;
  if ((fl & 1) || (fl & 6) == 6) {
    r = __int_as_float(0x7fc00000);
  } else if (fl & 2) {
    r = __int_as_float(0x7f800000);
  } else if (fl & 4) {
    r = __int_as_float(0xff800000);
  } else {
    // carry-normalise the signed 32-bit digits into a two's complement integer
    unsigned mag[GM_U32_DIGITS + 1];
    long long c = 0;
    for (int d = 0; d < GM_U32_DIGITS; ++d) {
      const long long t = __ldcg(digits + d) + c;
      const long long q = t >> 32;                      // floor division by 2^32
      mag[d] = (unsigned)(t - (q << 32));
      c = q;
    }
    mag[GM_U32_DIGITS] = (unsigned)c;
    const bool neg = c < 0;
    if (neg) {                                          // magnitude = -value
      unsigned long long carry = 1;
      for (int d = 0; d <= GM_U32_DIGITS; ++d) {
        const unsigned long long t = (unsigned long long)(~mag[d]) + carry;
        mag[d] = (unsigned)t;
        carry = t >> 32;
      }
    }
    int top = -1;
    for (int d = GM_U32_DIGITS; d >= 0 && top < 0; --d)
      if (mag[d]) top = d * 32 + 31 - __clz(mag[d]);
    unsigned fb;
    if (top < 23) {
      fb = mag[0];                                      // subnormal (or zero): exact
    } else {
      auto bit = [&](int b) -> unsigned { return b < 0 ? 0u : (mag[b >> 5] >> (b & 31)) & 1u; };
      unsigned m = 0;
      for (int b = top; b > top - 24; --b) m = (m << 1) | bit(b);
      const unsigned g = bit(top - 24);
      const int gb = top - 24;                          // guard bit; sticky = any bit below it
      unsigned sticky = gb > 0 ? mag[gb >> 5] & ((1u << (gb & 31)) - 1u) : 0u;
      for (int d = 0; d < (gb >> 5) && !sticky; ++d) sticky |= mag[d];
      int B = top;
      if (g && (sticky || (m & 1u))) {
        ++m;
        if (m >> 24) { m >>= 1; ++B; }
      }
      const int ef = B - 22;                            // biased exponent
      fb = ef >= 255 ? 0x7f800000u : (((unsigned)ef << 23) | (m & 0x7fffffu));
    }
    r = __uint_as_float(fb | (neg ? 0x80000000u : 0u));
  }
  *out = r;
  *calls += 1;
}

int esize_of(int dtype) {
  switch (dtype) {
    case GM_F32: case GM_I32: return 4;
    case GM_BF16: case GM_F16: return 2;
    case GM_BOOL: case GM_U8: return 1;
    default: return 8;
  }
}

int ensure_ctx() {
  CUcontext ctx = nullptr;
  GM_CU(g_drv.CtxGetCurrent(&ctx));
  if (!ctx) {
    GM_CUDA(cudaFree(0));  // binds the primary context of the current device
  }
  return GM_OK;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int gm_abi_version(void) { return GM_ABI_VERSION; }

const char* gm_last_error(void) { return g_err.c_str(); }

int gm_init(int device, int* num_sms, int* smem_optin_bytes) {
  if (device < 0) return fail(GM_E_INVALID, "gm_init: bad device %d", device);
  GM_CUDA(cudaSetDevice(device));
  if (load_driver()) return fail(GM_E_CUDA, "gm_init: cannot load libcuda.so.1: %s", dlerror());
  int r = ensure_ctx();
  if (r) return r;
  GM_CUDA(cudaDeviceGetAttribute(&g_cc_major, cudaDevAttrComputeCapabilityMajor, device));
  GM_CUDA(cudaDeviceGetAttribute(&g_cc_minor, cudaDevAttrComputeCapabilityMinor, device));
  GM_CUDA(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, device));
  GM_CUDA(cudaDeviceGetAttribute(&g_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  g_device = device;
  if (num_sms) *num_sms = g_num_sms;
  if (smem_optin_bytes) *smem_optin_bytes = g_smem_optin;
  return GM_OK;
}

// NVRTC -> cubin for sm_<major><minor>a.  Exposed separately so the CPU
// test suite can check generated sources compile without a GPU.
int gm_region_compile_cubin(const char* cuda_src, int cc_major, int cc_minor, void** cubin, size_t* cubin_bytes,
                            char* log, size_t log_cap) {
  if (!cuda_src || !cubin || !cubin_bytes) return fail(GM_E_INVALID, "gm_region_compile_cubin: null argument");
  nvrtcProgram prog;
  const char* headers[1] = {kRegionHeader};
  const char* names[1] = {"gm_region.cuh"};
  nvrtcResult rc = nvrtcCreateProgram(&prog, cuda_src, "gm_region_gen.cu", 1, headers, names);
  if (rc != NVRTC_SUCCESS) return fail(GM_E_COMPILE, "nvrtcCreateProgram: %s", nvrtcGetErrorString(rc));
  char arch[64];
  snprintf(arch, sizeof(arch), "--gpu-architecture=sm_%d%da", cc_major, cc_minor);
  const char* opts[] = {arch, "-std=c++17", "-lineinfo", "--fmad=false", "-DGM_NVRTC=1"};
  rc = nvrtcCompileProgram(prog, (int)(sizeof(opts) / sizeof(opts[0])), opts);
  size_t log_size = 0;
  nvrtcGetProgramLogSize(prog, &log_size);
  std::string lg(log_size + 1, '\0');
  if (log_size) nvrtcGetProgramLog(prog, &lg[0]);
  if (log && log_cap) {
    strncpy(log, lg.c_str(), log_cap - 1);
    log[log_cap - 1] = 0;
  }
  if (rc != NVRTC_SUCCESS) {
    nvrtcDestroyProgram(&prog);
    return fail(GM_E_COMPILE, "nvrtc: %s\n%s", nvrtcGetErrorString(rc), lg.c_str());
  }
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  void* buf = malloc(n);
  if (!buf) {
    nvrtcDestroyProgram(&prog);
    return fail(GM_E_NOMEM, "cubin alloc");
  }
  nvrtcGetCUBIN(prog, (char*)buf);
  nvrtcDestroyProgram(&prog);
  *cubin = buf;
  *cubin_bytes = n;
  return GM_OK;
}

void gm_free(void* p) { free(p); }

int gm_region_compile(const char* cuda_src, const char* kernel_name, gm_region* out, char* log, size_t log_cap) {
  if (!kernel_name || !out) return fail(GM_E_INVALID, "gm_region_compile: null argument");
  if (g_device < 0) return fail(GM_E_INVALID, "gm_region_compile: gm_init not called");
  void* cubin = nullptr;
  size_t nbytes = 0;
  int r = gm_region_compile_cubin(cuda_src, g_cc_major, g_cc_minor, &cubin, &nbytes, log, log_cap);
  if (r) return r;
  r = ensure_ctx();
  if (r) {
    free(cubin);
    return r;
  }
  gm_region_s* reg = new gm_region_s();
  CUresult cr = g_drv.ModuleLoadData(&reg->mod, cubin);
  free(cubin);
  if (cr != CUDA_SUCCESS) {
    delete reg;
    const char* s = nullptr;
    g_drv.GetErrorString(cr, &s);
    return fail(GM_E_CUDA, "cuModuleLoadData: %s", s ? s : "?");
  }
  cr = g_drv.ModuleGetFunction(&reg->fn, reg->mod, kernel_name);
  if (cr != CUDA_SUCCESS) {
    g_drv.ModuleUnload(reg->mod);
    delete reg;
    return fail(GM_E_CUDA, "cuModuleGetFunction(%s) failed", kernel_name);
  }
  *out = reg;
  return GM_OK;
}

int gm_region_load(const void* cubin, size_t cubin_bytes, const char* kernel_name, gm_region* out) {
  if (!cubin || !cubin_bytes || !kernel_name || !out) return fail(GM_E_INVALID, "gm_region_load: null argument");
  if (g_device < 0) return fail(GM_E_INVALID, "gm_region_load: gm_init not called");
  int r = ensure_ctx();
  if (r) return r;
  gm_region_s* reg = new gm_region_s();
  CUresult cr = g_drv.ModuleLoadData(&reg->mod, cubin);
  if (cr != CUDA_SUCCESS) {
    delete reg;
    const char* s = nullptr;
    g_drv.GetErrorString(cr, &s);
    return fail(GM_E_CUDA, "cuModuleLoadData(cached cubin): %s", s ? s : "?");
  }
  cr = g_drv.ModuleGetFunction(&reg->fn, reg->mod, kernel_name);
  if (cr != CUDA_SUCCESS) {
    g_drv.ModuleUnload(reg->mod);
    delete reg;
    return fail(GM_E_CUDA, "cuModuleGetFunction(%s) failed", kernel_name);
  }
  *out = reg;
  return GM_OK;
}

int gm_region_set_smem(gm_region r, int smem_bytes) {
  if (!r) return fail(GM_E_INVALID, "gm_region_set_smem: null region");
  GM_CU(g_drv.FuncSetAttribute(r->fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, smem_bytes));
  r->smem = smem_bytes;
  return GM_OK;
}

int gm_region_occupancy(gm_region r, int threads, int smem_bytes, int* blocks_per_sm) {
  if (!r || !blocks_per_sm) return fail(GM_E_INVALID, "gm_region_occupancy: null argument");
  GM_CU(g_drv.OccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, r->fn, threads, (size_t)smem_bytes));
  return GM_OK;
}

int gm_region_launch(gm_region r, const void* params, size_t params_bytes, int grid, int threads, int smem_bytes,
                     void* stream) {
  if (!r || !params) return fail(GM_E_INVALID, "gm_region_launch: null argument");
  if (params_bytes != sizeof(gm::Params))
    return fail(GM_E_INVALID, "gm_region_launch: params %zu bytes, expected %zu", params_bytes, sizeof(gm::Params));
  if (smem_bytes > r->smem) {
    int e = gm_region_set_smem(r, smem_bytes);
    if (e) return e;
  }
  void* args[1] = {const_cast<void*>(params)};
  GM_CU(g_drv.LaunchKernel(r->fn, grid, 1, 1, threads, 1, 1, smem_bytes, (CUstream)stream, args, nullptr));
  return GM_OK;
}

int gm_region_launch_ex(gm_region r, const void* params, size_t params_bytes, int grid, int threads, int smem_bytes,
                        void* stream, int flags) {
  if (!(flags & GM_LAUNCH_PDL)) return gm_region_launch(r, params, params_bytes, grid, threads, smem_bytes, stream);
  if (!r || !params) return fail(GM_E_INVALID, "gm_region_launch_ex: null argument");
  if (params_bytes != sizeof(gm::Params))
    return fail(GM_E_INVALID, "gm_region_launch_ex: params %zu bytes, expected %zu", params_bytes, sizeof(gm::Params));
  if (smem_bytes > r->smem) {
    int e = gm_region_set_smem(r, smem_bytes);
    if (e) return e;
  }
  CUlaunchAttribute attr[1];
  memset(attr, 0, sizeof(attr));
  attr[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
  attr[0].value.programmaticStreamSerializationAllowed = 1;
  CUlaunchConfig cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDimX = grid;
  cfg.gridDimY = cfg.gridDimZ = 1;
  cfg.blockDimX = threads;
  cfg.blockDimY = cfg.blockDimZ = 1;
  cfg.sharedMemBytes = smem_bytes;
  cfg.hStream = (CUstream)stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* args[1] = {const_cast<void*>(params)};
  GM_CU(g_drv.LaunchKernelEx(&cfg, r->fn, args, nullptr));
  return GM_OK;
}

int gm_region_release(gm_region r) {
  if (!r) return GM_OK;
  if (r->mod) g_drv.ModuleUnload(r->mod);
  delete r;
  return GM_OK;
}

size_t gm_region_params_bytes(void) { return sizeof(gm::Params); }

int gm_stream_capture_id(void* stream, uint64_t* id) {
  if (!id) return fail(GM_E_INVALID, "gm_stream_capture_id: null id");
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  unsigned long long cid = 0;
  GM_CUDA(cudaStreamGetCaptureInfo((cudaStream_t)stream, &st, &cid));
  *id = st == cudaStreamCaptureStatusActive ? (uint64_t)cid : 0ull;
  return GM_OK;
}

namespace {
int* g_status_host = nullptr;
int* g_status_dev = nullptr;
int g_status_n = 0;
}  // namespace

int gm_status_page(int n, int** host, int** dev) {
  if (n <= 0 || !host || !dev) return fail(GM_E_INVALID, "gm_status_page: bad argument");
  if (!g_status_host) {
    void* h = nullptr;
    GM_CUDA(cudaHostAlloc(&h, (size_t)n * sizeof(int), cudaHostAllocMapped | cudaHostAllocPortable));
    memset(h, 0, (size_t)n * sizeof(int));
    void* d = nullptr;
    GM_CUDA(cudaHostGetDevicePointer(&d, h, 0));
    g_status_host = (int*)h;
    g_status_dev = (int*)d;
    g_status_n = n;
  } else if (n > g_status_n) {
    return fail(GM_E_INVALID, "gm_status_page: already open with %d words (< %d)", g_status_n, n);
  }
  *host = g_status_host;
  *dev = g_status_dev;
  return GM_OK;
}

// barrier scratch (counter, epoch, status, results) | partials @ GM_SCRATCH_PARTIALS
size_t gm_branch_select_scratch_bytes(void) { return GM_SCRATCH_PARTIALS + 8 * 4096; }

int gm_branch_select_f32(const float* x, float* out, int64_t n, int red, int cmp, double thr, double a1, double b1,
                         double a2, double b2, void* scratch, double* stat_out, void* stream) {
  if (g_device < 0) return fail(GM_E_INVALID, "gm_branch_select_f32: gm_init not called");
  if (!x || !out || !scratch || n <= 0) return fail(GM_E_INVALID, "gm_branch_select_f32: bad argument");
  if (red < 0 || red > 4 || cmp < 0 || cmp > 3) return fail(GM_E_INVALID, "gm_branch_select_f32: bad red/cmp");
  if (((uintptr_t)x | (uintptr_t)out) & 15) return fail(GM_E_INVALID, "gm_branch_select_f32: pointers must be 16B aligned");
  gm::Params P;
  memset(&P, 0, sizeof(P));
  P.n = n;
  P.nvec = (n + GM_VEC - 1) / GM_VEC;
  int grid = (int)((P.nvec + GM_THREADS * 4 - 1) / (GM_THREADS * 4));
  if (grid > g_num_sms) grid = g_num_sms;
  if (grid < 1) grid = 1;
  P.vpc = (P.nvec + grid - 1) / grid;
  grid = (int)((P.nvec + P.vpc - 1) / P.vpc);
  const long long chunk_bytes = P.vpc * GM_VEC * 4;
  int smem = 0;
  P.in[0].ptr = (long long)(uintptr_t)x;
  P.in[0].smem_off = -1;
  if (chunk_bytes <= g_smem_optin - 4096 && (n * 4) % 16 == 0) {
    P.in[0].smem_off = 0;
    smem = (int)chunk_bytes;
    P.piece_vecs = (P.vpc + GM_MAX_PIECES - 1) / GM_MAX_PIECES;
    if (P.piece_vecs < 64) P.piece_vecs = 64;
  } else {
    P.piece_vecs = P.vpc;
  }
  P.out[0].ptr = (long long)(uintptr_t)out;
  char* s = (char*)scratch;
  P.barrier = (long long)(uintptr_t)s;
  P.status = (long long)(uintptr_t)(s + 16);
  P.partials = (long long)(uintptr_t)(s + GM_SCRATCH_PARTIALS);
  if ((size_t)grid * 8 > gm_branch_select_scratch_bytes() - GM_SCRATCH_PARTIALS)
    return fail(GM_E_INVALID, "grid too large for scratch");
  BsArgs A;
  A.red = red;
  A.cmp = cmp;
  A.thr = thr;
  A.a1 = a1;
  A.b1 = b1;
  A.a2 = a2;
  A.b2 = b2;
  A.stat_out = stat_out;
  if (smem > 48 * 1024)
    GM_CUDA(cudaFuncSetAttribute(gm_branch_select_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  gm_branch_select_f32_kernel<<<grid, GM_THREADS, smem, (cudaStream_t)stream>>>(P, A);
  GM_CUDA(cudaGetLastError());
  return GM_OK;
}

// ---------------------------------------------------------------------------
// log ring
// ---------------------------------------------------------------------------
int gm_logring_open(size_t bytes, gm_logring* out) {
  if (!out || bytes == 0) return fail(GM_E_INVALID, "gm_logring_open: bad argument");
  gm_logring_s* r = new gm_logring_s();
  r->bytes = bytes;
  cudaError_t e = cudaHostAlloc(&r->host, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
  if (e != cudaSuccess) {
    delete r;
    return fail(GM_E_NOMEM, "cudaHostAlloc(%zu): %s", bytes, cudaGetErrorString(e));
  }
  memset(r->host, 0, bytes);
  GM_CUDA(cudaHostGetDevicePointer(&r->dev, r->host, 0));
  void* hc = nullptr;
  GM_CUDA(cudaHostAlloc(&hc, 64, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(hc, 0, 64);
  r->hcommit = (volatile unsigned long long*)hc;
  GM_CUDA(cudaHostGetDevicePointer((void**)&r->dcommit, hc, 0));
  GM_CUDA(cudaMalloc((void**)&r->dstep, 64));
  GM_CUDA(cudaMemset(r->dstep, 0, 64));
  GM_CUDA(cudaDeviceSynchronize());
  r->slot_bytes = (bytes / GM_LOGRING_SLOTS) & ~(uint64_t)15;
  *out = r;
  return GM_OK;
}

int gm_logring_close(gm_logring r) {
  if (!r) return GM_OK;
  cudaDeviceSynchronize();
  if (r->host) cudaFreeHost(r->host);
  if (r->hcommit) cudaFreeHost((void*)r->hcommit);
  if (r->dstep) cudaFree(r->dstep);
  delete r;
  return GM_OK;
}

void* gm_logring_host_ptr(gm_logring r) { return r ? r->host : nullptr; }
size_t gm_logring_bytes(gm_logring r) { return r ? r->bytes : 0; }
uint64_t* gm_logring_step_ptr(gm_logring r) { return r ? (uint64_t*)r->dstep : nullptr; }
uint64_t gm_logring_committed(gm_logring r) { return r ? *r->hcommit : 0; }

int gm_logring_gather(gm_logring r, const void* src, int dtype, int ndim, const int64_t* stride, const int64_t* counts,
                      const int64_t* index_lists, uint64_t step_bytes, uint64_t n_slots, uint64_t offset,
                      void* stream) {
  // index_lists carries, per dim, {head, size}: the gathered index k maps to
  // k (k < head) or size - count + k (torch's edgeitems summarisation).
  if (!r || !src || ndim < 0 || ndim > GM_MAX_DIMS || !n_slots)
    return fail(GM_E_INVALID, "gm_logring_gather: bad argument");
  GatherArgs A;
  memset(&A, 0, sizeof(A));
  A.src = src;
  A.ring_dev = r->dev;
  A.dstep = r->dstep;
  A.step_bytes = step_bytes;
  A.n_slots = n_slots;
  A.offset = offset;
  A.dtype = dtype;
  A.ndim = ndim;
  A.esize = esize_of(dtype);
  long long total = 1;
  for (int d = 0; d < ndim; ++d) {
    A.count[d] = counts[d];
    A.head[d] = index_lists[2 * d];
    A.size[d] = index_lists[2 * d + 1];
    A.stride[d] = stride[d];
    total *= counts[d];
  }
  A.total = total;
  if ((unsigned long long)(total * A.esize) + offset > step_bytes || step_bytes * n_slots > r->bytes)
    return fail(GM_E_RING_FULL, "gm_logring_gather: record does not fit the ring slot");
  gm_logring_gather_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(A);
  GM_CUDA(cudaGetLastError());
  return GM_OK;
}

size_t gm_unique_sum16_scratch_bytes(void) { return 2048 * sizeof(unsigned); }

int gm_unique_sum16(const void* x, int64_t n, int dtype, void* out, void* scratch, void* stream) {
  if (g_device < 0) return fail(GM_E_INVALID, "gm_unique_sum16: gm_init not called");
  if (!x || !out || !scratch || n < 0) return fail(GM_E_INVALID, "gm_unique_sum16: bad argument");
  if (dtype != GM_BF16 && dtype != GM_F16) return fail(GM_E_INVALID, "gm_unique_sum16: dtype must be bf16 or f16");
  if ((uintptr_t)x & 15) return fail(GM_E_INVALID, "gm_unique_sum16: x must be 16-byte aligned");
  cudaStream_t s = (cudaStream_t)stream;
  GM_CUDA(cudaMemsetAsync(scratch, 0, gm_unique_sum16_scratch_bytes(), s));
  const long long nvec = n / 8;
  const int ntail = (int)(n % 8);
  long long want = (nvec + 511) / 512;
  int grid = (int)(want < 2LL * g_num_sms ? want : 2LL * g_num_sms);
  if (grid < 1) grid = 1;
  gm_unique16_mark_kernel<<<grid, 512, 0, s>>>((const uint4*)x, nvec, (const unsigned short*)x + nvec * 8, ntail,
                                               (unsigned*)scratch);
  GM_CUDA(cudaGetLastError());
  gm_unique16_sum_kernel<<<1, 1024, 0, s>>>((const unsigned*)scratch, dtype, out);
  GM_CUDA(cudaGetLastError());
  return GM_OK;
}

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

// hash-set capacity: a power of two >= 2n (load <= 1/2)
static unsigned long long u32_table_slots(int64_t n) {
  unsigned long long s = 1ull << 16;
  while (s < 2ull * (unsigned long long)n) s <<= 1;
  return s;
}

size_t gm_unique_sum32_hash_scratch_bytes(int64_t n) {
  return 4096 + 4 * GM_U32_BITMAP_WORDS + 8 * u32_table_slots(n);
}

int gm_unique_sum32_hash(const float* x, int64_t n, float* out, void* scratch, size_t scratch_bytes, void* stream) {
  if (g_device < 0) return fail(GM_E_INVALID, "gm_unique_sum32_hash: gm_init not called");
  if (!x || !out || !scratch || n <= 0) return fail(GM_E_INVALID, "gm_unique_sum32_hash: bad argument");
  if (scratch_bytes < gm_unique_sum32_hash_scratch_bytes(n))
    return fail(GM_E_INVALID, "gm_unique_sum32_hash: scratch too small");
  cudaStream_t s = (cudaStream_t)stream;
  char* base = (char*)scratch;
  unsigned long long* calls = (unsigned long long*)base;          // +0: calls completed (tag source)
  long long* digits = (long long*)(base + 64);                    // +64: int64[GM_U32_DIGITS]
  int* flags = (int*)(base + 256);                                // +256: NaN / +inf / -inf seen
  int* emax = (int*)(base + 260);                                 // +260: largest finite biased exponent
  int* pred = (int*)(base + 48);                                  // +48: previous call's largest exponent (kept)
  unsigned* touched = (unsigned*)(base + 264);                    // +264: bitmap slices marked this call
  unsigned* done = (unsigned*)(base + 268);                       // +268: CTAs of the bitmap pass finished
  unsigned* bitmap = (unsigned*)(base + 4096);                    // presence bitmap, all-zero between calls
  unsigned long long* table = (unsigned long long*)(base + 4096 + 4 * GM_U32_BITMAP_WORDS);
  GM_CUDA(cudaMemsetAsync(base + 64, 0, 256, s));
  const unsigned long long slots = u32_table_slots(n);
  long long want = (n + 2047) / 2048;
  int grid = (int)(want < 2LL * g_num_sms ? want : 2LL * g_num_sms);
  if (grid < 1) grid = 1;
  // bitmap window: by default the 16 binades from 2 above the PREVIOUS
  // call's largest exponent down (values outside it go to the hash set, so
  // the window only decides speed, never the result); GM_U32_WINDOW_PASS=1
  // measures this call's largest exponent first (one more read of x)
  static const bool window_pass = getenv("GM_U32_WINDOW_PASS") && atoi(getenv("GM_U32_WINDOW_PASS"));
  int* top = pred;
  int head = 2;
  if (window_pass) {
    gm_unique32_window_kernel<<<grid, 512, 0, s>>>(x, n, emax);
    GM_CUDA(cudaGetLastError());
    top = emax;
    head = 0;
  }
  gm_unique32_insert_kernel<<<grid, 512, 0, s>>>(x, n, bitmap, top, head, emax, table, slots - 1, calls, digits, flags,
                                                 touched);
  GM_CUDA(cudaGetLastError());
  gm_unique32_bitmap_sum_kernel<<<2 * g_num_sms, 512, 0, s>>>((uint4*)bitmap, top, head, emax, touched, digits, done,
                                                               flags, calls, out);
  GM_CUDA(cudaGetLastError());
  return GM_OK;
}

size_t gm_unique_sum32_scratch_bytes(int64_t n) {
  size_t temp = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, temp, (const float*)nullptr, (float*)nullptr, (int)n);
  return align256(temp) + align256((size_t)n * sizeof(float)) + align256(8 * 4096);
}

int gm_unique_sum32(const float* x, int64_t n, float* out, void* scratch, size_t scratch_bytes, void* stream) {
  if (g_device < 0) return fail(GM_E_INVALID, "gm_unique_sum32: gm_init not called");
  if (!x || !out || !scratch || n <= 0 || n > 0x7fffffffLL) return fail(GM_E_INVALID, "gm_unique_sum32: bad argument");
  if (scratch_bytes < gm_unique_sum32_scratch_bytes(n)) return fail(GM_E_INVALID, "gm_unique_sum32: scratch too small");
  cudaStream_t s = (cudaStream_t)stream;
  size_t temp = 0;
  GM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, temp, x, (float*)nullptr, (int)n));
  char* base = (char*)scratch;
  float* keys = (float*)(base + align256(temp));
  double* partials = (double*)(base + align256(temp) + align256((size_t)n * sizeof(float)));
  GM_CUDA(cub::DeviceRadixSort::SortKeys(base, temp, x, keys, (int)n, 0, 32, s));
  long long want = (n + 511) / 512;
  int grid = (int)(want < 2LL * g_num_sms ? want : 2LL * g_num_sms);
  if (grid < 1) grid = 1;
  gm_distinct_sum32_kernel<<<grid, 512, 0, s>>>(keys, n, partials);
  GM_CUDA(cudaGetLastError());
  gm_sum_partials_kernel<<<1, 1024, 0, s>>>(partials, grid, out);
  GM_CUDA(cudaGetLastError());
  return GM_OK;
}

// ---- record-level API ------------------------------------------------------
int gm_logring_begin_step(gm_logring r) {
  if (!r) return fail(GM_E_INVALID, "gm_logring_begin_step: null ring");
  if (r->step_open) return fail(GM_E_INVALID, "gm_logring_begin_step: a step is already open");
  r->step_open = true;
  r->open.clear();
  r->cursor = GM_LOGRING_HEADER;
  return GM_OK;
}

int gm_logring_capture(gm_logring r, const void* dev_src, const int64_t* shape, const int64_t* stride, int ndim,
                       int dtype, uint32_t record_id, void* stream) {
  if (!r || !dev_src || ndim < 0 || ndim > GM_MAX_DIMS || (ndim && (!shape || !stride)))
    return fail(GM_E_INVALID, "gm_logring_capture: bad argument");
  if (!r->step_open) return fail(GM_E_INVALID, "gm_logring_capture: no open step (gm_logring_begin_step)");
  const int es = esize_of(dtype);
  if (es <= 0) return fail(GM_E_INVALID, "gm_logring_capture: dtype %d", dtype);
  // torch._tensor_str: numel > threshold (1000) -> edgeitems (3) per side of
  // every dim longer than 2 * edgeitems
  int64_t numel = 1;
  for (int d = 0; d < ndim; ++d) numel *= shape[d];
  const bool summarize = numel > 1000;
  GmRecordDesc rec;
  memset(&rec, 0, sizeof(rec));  // zero padding: templates are compared with memcmp
  rec.id = record_id;
  rec.dtype = dtype;
  rec.ndim = ndim;
  int64_t total = 1, hl[2 * GM_MAX_DIMS + 2];
  for (int d = 0; d < ndim; ++d) {
    rec.shape[d] = shape[d];
    const bool cut = summarize && shape[d] > 6;
    rec.counts[d] = cut ? 6 : shape[d];
    rec.heads[d] = cut ? 3 : shape[d];
    hl[2 * d] = rec.heads[d];
    hl[2 * d + 1] = shape[d];
    total *= rec.counts[d];
  }
  rec.offset = (r->cursor + 15) & ~(uint64_t)15;
  rec.bytes = (uint64_t)total * es;
  if (rec.offset + rec.bytes > r->slot_bytes)
    return fail(GM_E_RING_FULL, "gm_logring_capture: step records exceed the %llu-byte slot",
                (unsigned long long)r->slot_bytes);
  if (total > 0) {
    int rc = gm_logring_gather(r, dev_src, dtype, ndim, stride, rec.counts, hl, r->slot_bytes, GM_LOGRING_SLOTS,
                               rec.offset, stream);
    if (rc) return rc;
  }
  r->cursor = rec.offset + rec.bytes;
  r->open.push_back(rec);
  return GM_OK;
}

int gm_logring_end_step(gm_logring r, void* stream, uint32_t* template_id) {
  if (!r || !template_id) return fail(GM_E_INVALID, "gm_logring_end_step: bad argument");
  if (!r->step_open) return fail(GM_E_INVALID, "gm_logring_end_step: no open step");
  r->step_open = false;
  if (r->open.empty()) {
    *template_id = GM_LOGRING_NO_TEMPLATE;
    return GM_OK;
  }
  // an eager forward re-registers the same template every step: reuse it
  unsigned tid = (unsigned)r->templates.size();
  for (size_t back = 0; back < 16 && back < r->templates.size(); ++back) {
    const size_t i = r->templates.size() - 1 - back;
    const auto& t = r->templates[i];
    if (t.size() == r->open.size() && !memcmp(t.data(), r->open.data(), t.size() * sizeof(GmRecordDesc))) {
      tid = (unsigned)i;
      break;
    }
  }
  if (tid == r->templates.size()) r->templates.push_back(r->open);
  gm_logring_commit_step_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(
      r->dstep, r->dcommit, (char*)r->dev, r->slot_bytes, GM_LOGRING_SLOTS, tid, (unsigned)r->open.size());
  GM_CUDA(cudaGetLastError());
  r->open.clear();
  *template_id = tid;
  return GM_OK;
}

int gm_logring_drain(gm_logring r, gm_record_cb cb, void* user) {
  if (!r || !cb) return fail(GM_E_INVALID, "gm_logring_drain: bad argument");
  const unsigned long long committed = *r->hcommit;
  int steps = 0;
  while (r->drained < committed) {
    const uint64_t s = r->drained + 1;
    const char* slot = (const char*)r->host + ((s - 1) % GM_LOGRING_SLOTS) * r->slot_bytes;
    const GmSlotHeader* h = (const GmSlotHeader*)slot;
    if (*(volatile const unsigned long long*)&h->step != s)
      return fail(GM_E_RING_FULL, "gm_logring_drain: step %llu was overwritten before it was drained "
                  "(more than %d steps in flight)", (unsigned long long)s, GM_LOGRING_SLOTS);
    if (h->template_id >= r->templates.size())
      return fail(GM_E_INVALID, "gm_logring_drain: unknown template %u", h->template_id);
    for (const GmRecordDesc& d : r->templates[h->template_id]) {
      gm_record rec;
      rec.record_id = d.id;
      rec.dtype = d.dtype;
      rec.ndim = d.ndim;
      rec.pad = 0;
      rec.step = s;
      rec.shape = d.shape;
      rec.counts = d.counts;
      rec.heads = d.heads;
      rec.data = slot + d.offset;
      rec.bytes = d.bytes;
      const int rc = cb(&rec, user);
      if (rc) return fail(GM_E_INVALID, "gm_logring_drain: callback returned %d at record %u of step %llu", rc,
                          d.id, (unsigned long long)s);
    }
    r->drained = s;
    ++steps;
  }
  return steps;
}

int gm_logring_commit(gm_logring r, void* stream) {
  if (!r) return fail(GM_E_INVALID, "gm_logring_commit: null ring");
  gm_logring_commit_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(r->dstep, r->dcommit);
  GM_CUDA(cudaGetLastError());
  return GM_OK;
}

}  // extern "C"
