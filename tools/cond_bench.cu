// cond_bench.cu — B200 microbenchmark for the speculative region design.
//
// Measures, per step inside one CUDA graph (R steps, CUDA events around the
// replay), for a [8,1024,768] bf16 tensor (the BigBird region-0 shape):
//   flush      : L2 flush only (256 MB memset, optionally + 256 MB read = clean)
//   copy       : flush + a plain 128-bit streaming copy (read N, write N)
//   spec       : flush + single-pass speculative region (|q*s| mean reduce,
//                sigmoid arm, write ctx) with a last-arriver combine
//   spec+cond  : as spec, plus a conditional IF node whose body is the
//                fix-up kernel; the spec kernel sets the handle (0 on a hit)
//   spec+exit  : as spec, plus an always-launched fix-up kernel that exits
//                when the flag says "hit"
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cond_bench tools/cond_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); exit(1); } } while (0)

typedef unsigned int u32;
__device__ __forceinline__ void ldg16(const void* p, u32& a, u32& b, u32& c, u32& d) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p));
}
__device__ __forceinline__ void stg16(void* p, u32 a, u32 b, u32 c, u32 d) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ float fexp(float a) { float y; asm("ex2.approx.f32 %0, %1;" : "=f"(y) : "f"(a * 1.4426950408889634f)); return y; }
__device__ __forceinline__ float frcp(float a) { float y; asm("rcp.approx.f32 %0, %1;" : "=f"(y) : "f"(a)); return y; }
__device__ __forceinline__ u32 f2bf2(float lo, float hi) { u32 r; asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo)); return r; }
__device__ __forceinline__ float rbf(float f) { return __uint_as_float(f2bf2(0.f, f) & 0xffff0000u); }

__global__ void copy_k(const uint4* __restrict__ in, uint4* __restrict__ out, long nv) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < nv; i += (long)gridDim.x * blockDim.x) {
    uint4 v; ldg16(in + i, v.x, v.y, v.z, v.w); stg16(out + i, v.x, v.y, v.z, v.w);
  }
}

__global__ void read_k(const uint4* __restrict__ in, long nv, u32* sink) {
  u32 acc = 0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < nv; i += (long)gridDim.x * blockDim.x) {
    uint4 v; ldg16(in + i, v.x, v.y, v.z, v.w); acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

template <int U, bool ARM>
__device__ __forceinline__ float body(const uint4* __restrict__ q, uint4* __restrict__ out, long nv, float scale) {
  float acc = 0.f;
  const long stride = (long)gridDim.x * blockDim.x;
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < nv; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) ldg16(q + i + u * stride, v[u].x, v[u].y, v[u].z, v[u].w);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      u32 w[4] = {v[u].x, v[u].y, v[u].z, v[u].w}, o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float x0 = __uint_as_float(w[j] << 16), x1 = __uint_as_float(w[j] & 0xffff0000u);
        float s0 = rbf(x0 * scale), s1 = rbf(x1 * scale);
        acc += fabsf(s0) + fabsf(s1);
        float p0, p1;
        if (ARM) { p0 = rbf(rbf(rbf(frcp(1.f + fexp(-s0))) * 0.5f) + 0.25f); p1 = rbf(rbf(rbf(frcp(1.f + fexp(-s1))) * 0.5f) + 0.25f); }
        else { p0 = rbf(frcp(1.f + fexp(-s0))); p1 = rbf(frcp(1.f + fexp(-s1))); }
        o[j] = f2bf2(p0 * x0, p1 * x1);
      }
      stg16(out + i + u * stride, o[0], o[1], o[2], o[3]);
    }
  }
  for (; i < nv; i += stride) {
    uint4 v; ldg16(q + i, v.x, v.y, v.z, v.w);
    u32 w[4] = {v.x, v.y, v.z, v.w}, o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float x0 = __uint_as_float(w[j] << 16), x1 = __uint_as_float(w[j] & 0xffff0000u);
      float s0 = rbf(x0 * scale), s1 = rbf(x1 * scale);
      acc += fabsf(s0) + fabsf(s1);
      float p0 = rbf(frcp(1.f + fexp(-s0))), p1 = rbf(frcp(1.f + fexp(-s1)));
      o[j] = f2bf2(p0 * x0, p1 * x1);
    }
    stg16(out + i, o[0], o[1], o[2], o[3]);
  }
  return acc;
}

// last-arriver combine; sets the conditional (1 = mispredicted) or a flag
template <int U, int MODE>  // MODE 0: nothing, 1: set conditional, 2: flag
__global__ void __launch_bounds__(512) spec_k(const uint4* __restrict__ q, uint4* __restrict__ out, long nv, float scale,
                                              double* partials, unsigned long long* counter, int* pred_and_flag,
                                              cudaGraphConditionalHandle h, long n) {
  float acc = body<U, true>(q, out, nv, scale);
  __shared__ double sw[32];
  __shared__ bool last;
  double v = acc;
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(~0u, v, o);
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < blockDim.x / 32 ? sw[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(~0u, t, o);
    if (threadIdx.x == 0) {
      partials[blockIdx.x] = t;
      unsigned long long old;
      asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(counter) : "memory");
      last = (old % gridDim.x) == gridDim.x - 1;
    }
  }
  __syncthreads();
  if (!last) return;
  if (threadIdx.x < 32) {
    double t = 0.0;
    for (u32 b = threadIdx.x; b < gridDim.x; b += 32) {
      double x; asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(x) : "l"(partials + b) : "memory"); t += x;
    }
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(~0u, t, o);
    if (threadIdx.x == 0) {
      const float mean = rbf((float)t / (float)n);
      const int d = mean > 0.05f;
      const int miss = d != pred_and_flag[0];
      pred_and_flag[0] = d;
      if (MODE == 1) cudaGraphSetConditional(h, miss);
      if (MODE == 2) pred_and_flag[1] = miss;
    }
  }
}

__global__ void __launch_bounds__(512) fix_k(const uint4* __restrict__ q, uint4* __restrict__ out, long nv, float scale, const int* flag) {
  if (flag && flag[1] == 0) return;
  body<4, false>(q, out, nv, scale);
}


__device__ __forceinline__ float fexp_ftz(float a) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a * 1.4426950408889634f)); return y; }
__device__ __forceinline__ float frcp_ftz(float a) { float y; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a)); return y; }
__device__ __forceinline__ u32 hmul2(u32 a, u32 b) { u32 d; asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }
__device__ __forceinline__ u32 hadd2(u32 a, u32 b) { u32 d; asm("add.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }

// packed: s = q*scale (bf16x2, exact), acc += |s|, p = bf16(sigmoid(s)), ctx = (p*0.5+0.25)*q
template <int U>
__device__ __forceinline__ float body_packed(const uint4* __restrict__ q, uint4* __restrict__ out, long nv, u32 scale2) {
  float acc = 0.f, acc2 = 0.f;
  // contiguous chunk per CTA (the region skeleton's mapping), threads stride by blockDim
  const long vpc = (nv + gridDim.x - 1) / gridDim.x;
  const long v0 = blockIdx.x * vpc, v1 = v0 + vpc < nv ? v0 + vpc : nv;
  long i = v0 + threadIdx.x;
  auto one = [&](const uint4& vv, long idx) {
    u32 w[4] = {vv.x, vv.y, vv.z, vv.w}, o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      u32 s = hmul2(w[j], scale2);
      float s0 = __uint_as_float(s << 16), s1 = __uint_as_float(s & 0xffff0000u);
      acc += fabsf(s0); acc2 += fabsf(s1);
      float p0 = frcp_ftz(1.f + fexp_ftz(-s0)), p1 = frcp_ftz(1.f + fexp_ftz(-s1));
      u32 pp = f2bf2(p0, p1);
      o[j] = hmul2(hadd2(hmul2(pp, 0x3f003f00u), 0x3e803e80u), w[j]);
    }
    stg16(out + idx, o[0], o[1], o[2], o[3]);
  };
  for (; i + (U - 1) * (long)blockDim.x < v1; i += U * (long)blockDim.x) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) ldg16(q + i + u * blockDim.x, v[u].x, v[u].y, v[u].z, v[u].w);
#pragma unroll
    for (int u = 0; u < U; ++u) one(v[u], i + u * blockDim.x);
  }
  for (; i < v1; i += blockDim.x) {
    uint4 v; ldg16(q + i, v.x, v.y, v.z, v.w);
    one(v, i);
  }
  return acc + acc2;
}

__global__ void copy_chunk_k(const uint4* __restrict__ in, uint4* __restrict__ out, long nv) {
  const long vpc = (nv + gridDim.x - 1) / gridDim.x;
  const long v0 = blockIdx.x * vpc, v1 = v0 + vpc < nv ? v0 + vpc : nv;
  long i = v0 + threadIdx.x;
  for (; i + 3 * (long)blockDim.x < v1; i += 4 * (long)blockDim.x) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) ldg16(in + i + u * blockDim.x, v[u].x, v[u].y, v[u].z, v[u].w);
#pragma unroll
    for (int u = 0; u < 4; ++u) stg16(out + i + u * blockDim.x, v[u].x, v[u].y, v[u].z, v[u].w);
  }
  for (; i < v1; i += blockDim.x) { uint4 v; ldg16(in + i, v.x, v.y, v.z, v.w); stg16(out + i, v.x, v.y, v.z, v.w); }
}

template <int U, int END>  // END 0: last arriver, 1: all CTAs wait + combine
__global__ void __launch_bounds__(512) spec2_k(const uint4* __restrict__ q, uint4* __restrict__ out, long nv, u32 scale2,
                                              double* partials, unsigned long long* counter, int* pf, long n) {
  float acc = body_packed<U>(q, out, nv, scale2);
  __shared__ double sw[32];
  __shared__ bool last;
  double v = acc;
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(~0u, v, o);
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < blockDim.x / 32 ? sw[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(~0u, t, o);
    if (threadIdx.x == 0) {
      partials[blockIdx.x] = t;
      unsigned long long old;
      asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(counter) : "memory");
      last = (old % gridDim.x) == gridDim.x - 1;
      if (END == 1) {
        const unsigned long long target = (old / gridDim.x + 1) * gridDim.x;
        unsigned long long c;
        do { asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(c) : "l"(counter) : "memory"); } while (c < target);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
    }
  }
  __syncthreads();
  if (END == 0 && !last) return;
  if (threadIdx.x < 32) {
    double t = 0.0;
    for (u32 b = threadIdx.x; b < gridDim.x; b += 32) {
      double x; asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(x) : "l"(partials + b) : "memory"); t += x;
    }
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(~0u, t, o);
    if (threadIdx.x == 0) {
      const float mean = rbf((float)t / (float)n);
      const int d = mean > 0.05f;
      if (blockIdx.x == 0 || END == 0) pf[0] = d;
      if (d != 1) pf[1] = 1;
    }
  }
}


// all loads in flight at once: thread t owns vectors t + k*T (T = grid threads), k < K
__device__ __forceinline__ u32 sig_arm(u32 w, u32 scale2, float& acc, float& acc2) {
  u32 s = hmul2(w, scale2);
  float s0 = __uint_as_float(s << 16), s1 = __uint_as_float(s & 0xffff0000u);
  acc += fabsf(s0); acc2 += fabsf(s1);
  float p0 = frcp_ftz(1.f + fexp_ftz(-s0)), p1 = frcp_ftz(1.f + fexp_ftz(-s1));
  u32 pp = f2bf2(p0, p1);
  return hmul2(hadd2(hmul2(pp, 0x3f003f00u), 0x3e803e80u), w);
}

__device__ __forceinline__ void grid_sync_and_combine(double v, double* partials, unsigned long long* counter, int* pf, long n, bool all_wait) {
  __shared__ double sw[32];
  __shared__ bool last;
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(~0u, v, o);
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < blockDim.x / 32 ? sw[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(~0u, t, o);
    if (threadIdx.x == 0) {
      partials[blockIdx.x] = t;
      unsigned long long old;
      asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(counter) : "memory");
      last = (old % gridDim.x) == gridDim.x - 1;
      if (all_wait) {
        const unsigned long long target = (old / gridDim.x + 1) * gridDim.x;
        unsigned long long c;
        do { asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(c) : "l"(counter) : "memory"); } while (c < target);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
    }
  }
  __syncthreads();
  if (!all_wait && !last) return;
  if (threadIdx.x < 32) {
    double t = 0.0;
    for (u32 b = threadIdx.x; b < gridDim.x; b += 32) {
      double x; asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(x) : "l"(partials + b) : "memory"); t += x;
    }
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(~0u, t, o);
    if (threadIdx.x == 0) {
      const float mean = rbf((float)t / (float)n);
      pf[2 + (blockIdx.x & 1)] = mean > 0.05f;
    }
  }
  __syncthreads();
}

template <int K, int END>  // spec single pass, END 0 last-arriver, 1 end barrier
__global__ void __launch_bounds__(512, 2) spec3_k(const uint4* __restrict__ q, uint4* __restrict__ out, long nv, u32 scale2,
                                                 double* partials, unsigned long long* counter, int* pf, long n) {
  const long T = (long)gridDim.x * blockDim.x;
  const long t0 = blockIdx.x * (long)blockDim.x + threadIdx.x;
  uint4 v[K];
#pragma unroll
  for (int k = 0; k < K; ++k) if (t0 + k * T < nv) ldg16(q + t0 + k * T, v[k].x, v[k].y, v[k].z, v[k].w);
  float acc = 0.f, acc2 = 0.f;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (t0 + k * T < nv) {
      u32 o0 = sig_arm(v[k].x, scale2, acc, acc2), o1 = sig_arm(v[k].y, scale2, acc, acc2);
      u32 o2 = sig_arm(v[k].z, scale2, acc, acc2), o3 = sig_arm(v[k].w, scale2, acc, acc2);
      stg16(out + t0 + k * T, o0, o1, o2, o3);
    }
  }
  grid_sync_and_combine(acc + acc2, partials, counter, pf, n, END == 1);
}

template <int K>  // exact two-pass: loads -> reduce -> grid barrier -> arm from registers -> store
__global__ void __launch_bounds__(512, 2) exact3_k(const uint4* __restrict__ q, uint4* __restrict__ out, long nv, u32 scale2,
                                                  double* partials, unsigned long long* counter, int* pf, long n) {
  const long T = (long)gridDim.x * blockDim.x;
  const long t0 = blockIdx.x * (long)blockDim.x + threadIdx.x;
  uint4 v[K];
#pragma unroll
  for (int k = 0; k < K; ++k) if (t0 + k * T < nv) ldg16(q + t0 + k * T, v[k].x, v[k].y, v[k].z, v[k].w);
  float acc = 0.f, acc2 = 0.f;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (t0 + k * T < nv) {
      const u32 w[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        u32 s = hmul2(w[j], scale2) & 0x7fff7fffu;
        acc += __uint_as_float(s << 16); acc2 += __uint_as_float(s & 0xffff0000u);
      }
    }
  }
  grid_sync_and_combine(acc + acc2, partials, counter, pf, n, true);
  float d0 = 0, d1 = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (t0 + k * T < nv) {
      u32 o0 = sig_arm(v[k].x, scale2, d0, d1), o1 = sig_arm(v[k].y, scale2, d0, d1);
      u32 o2 = sig_arm(v[k].z, scale2, d0, d1), o3 = sig_arm(v[k].w, scale2, d0, d1);
      stg16(out + t0 + k * T, o0, o1, o2, o3);
    }
  }
}

__global__ void __launch_bounds__(512, 2) copy3_k(const uint4* __restrict__ q, uint4* __restrict__ out, long nv) {
  const int K = 6;
  const long T = (long)gridDim.x * blockDim.x;
  const long t0 = blockIdx.x * (long)blockDim.x + threadIdx.x;
  uint4 v[K];
#pragma unroll
  for (int k = 0; k < K; ++k) if (t0 + k * T < nv) ldg16(q + t0 + k * T, v[k].x, v[k].y, v[k].z, v[k].w);
#pragma unroll
  for (int k = 0; k < K; ++k) if (t0 + k * T < nv) stg16(out + t0 + k * T, v[k].x, v[k].y, v[k].z, v[k].w);
}


__device__ __forceinline__ float rcp_nr(float y) {
  // y >= 1: magic initial guess + 3 Newton steps on the FMA pipe (no MUFU)
  float x = __int_as_float(0x7EF311C7 - __float_as_int(y));
  float t;
  t = __fmaf_rn(-y, x, 1.f); x = __fmaf_rn(x, t, x);
  t = __fmaf_rn(-y, x, 1.f); x = __fmaf_rn(x, t, x);
  t = __fmaf_rn(-y, x, 1.f); x = __fmaf_rn(x, t, x);
  return y > 1e37f ? 0.f : x;
}
__device__ __forceinline__ float tanh_approx(float a) { float y; asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(a)); return y; }

template <int SIG>  // 0: ex2+rcp MUFU, 1: ex2 MUFU + NR rcp, 2: tanh MUFU
__device__ __forceinline__ u32 sig_arm_v(u32 w, u32 scale2, float& acc, float& acc2) {
  u32 s = hmul2(w, scale2);
  float s0 = __uint_as_float(s << 16), s1 = __uint_as_float(s & 0xffff0000u);
  acc += fabsf(s0); acc2 += fabsf(s1);
  float p0, p1;
  if (SIG == 0) { p0 = frcp_ftz(1.f + fexp_ftz(-s0)); p1 = frcp_ftz(1.f + fexp_ftz(-s1)); }
  else if (SIG == 1) { p0 = rcp_nr(1.f + fexp_ftz(-s0)); p1 = rcp_nr(1.f + fexp_ftz(-s1)); }
  else { p0 = __fmaf_rn(0.5f, tanh_approx(0.5f * s0), 0.5f); p1 = __fmaf_rn(0.5f, tanh_approx(0.5f * s1), 0.5f); }
  u32 pp = f2bf2(p0, p1);
  return hmul2(hadd2(hmul2(pp, 0x3f003f00u), 0x3e803e80u), w);
}

template <int K, int SIG, int THREADS, int MINB, bool KSYNC>
__global__ void __launch_bounds__(THREADS, MINB) spec4_k(const uint4* __restrict__ q, uint4* __restrict__ out, long nv, u32 scale2,
                                                 double* partials, unsigned long long* counter, int* pf, long n) {
  const long T = (long)gridDim.x * blockDim.x;
  const long t0 = blockIdx.x * (long)blockDim.x + threadIdx.x;
  uint4 v[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (t0 + k * T < nv) ldg16(q + t0 + k * T, v[k].x, v[k].y, v[k].z, v[k].w);
    if (KSYNC && k == 0) __syncthreads();
  }
  float acc = 0.f, acc2 = 0.f;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (t0 + k * T < nv) {
      u32 o0 = sig_arm_v<SIG>(v[k].x, scale2, acc, acc2), o1 = sig_arm_v<SIG>(v[k].y, scale2, acc, acc2);
      u32 o2 = sig_arm_v<SIG>(v[k].z, scale2, acc, acc2), o3 = sig_arm_v<SIG>(v[k].w, scale2, acc, acc2);
      stg16(out + t0 + k * T, o0, o1, o2, o3);
    }
  }
  grid_sync_and_combine(acc + acc2, partials, counter, pf, n, false);
}

int main(int argc, char** argv) {
  const long n = 8L * 1024 * 768, nv = n / 8;
  const size_t bytes = n * 2, fbytes = 256ull << 20;
  void *q, *out, *fl1, *fl2, *scratch;
  CK(cudaMalloc(&q, bytes)); CK(cudaMalloc(&out, bytes)); CK(cudaMalloc(&fl1, fbytes)); CK(cudaMalloc(&fl2, fbytes));
  CK(cudaMalloc(&scratch, 1 << 20)); CK(cudaMemset(scratch, 0, 1 << 20)); CK(cudaMemset(q, 0x3f, bytes)); CK(cudaMemset(fl2, 1, fbytes));
  double* partials = (double*)((char*)scratch + 4096);
  unsigned long long* counter0 = (unsigned long long*)((char*)scratch + 65536);
  int cidx = 0;
  unsigned long long* counter = counter0;
  int* pf = (int*)((char*)scratch + 256);
  u32* sink = (u32*)((char*)scratch + 512);
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaStream_t s, s2; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  const int R = 20;
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  int pred_init[2] = {1, 0};
  CK(cudaMemcpy(pf, pred_init, 8, cudaMemcpyHostToDevice));

  auto flush = [&](bool clean) {
    CK(cudaMemsetAsync(fl1, 0, fbytes, s));
    if (clean) read_k<<<sms * 4, 512, 0, s>>>((const uint4*)fl2, fbytes / 16, sink);
  };
  auto timeit = [&](const char* name, auto&& body_fn, double base) -> double {
    cudaGraph_t g; cudaGraphExec_t ge;
    counter = counter0 + 16 * (++cidx);  // fresh monotonic counter per variant (one grid size each)
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    for (int r = 0; r < R; ++r) body_fn();
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    std::vector<float> ts;
    for (int t = 0; t < 7; ++t) {
      CK(cudaGraphLaunch(ge, s));
      CK(cudaEventRecord(e0, s)); CK(cudaGraphLaunch(ge, s)); CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); ts.push_back(ms * 1000.f / R);
    }
    std::sort(ts.begin(), ts.end());
    double med = ts[ts.size() / 2];
    printf("%-34s %8.2f us/step   minus flush %7.2f us   (%.0f GB/s on 25.2 MB)\n", name, med, med - base,
           base > 0 ? 2.0 * bytes / ((med - base) * 1e-6) / 1e9 : 0.0);
    CK(cudaGraphExecDestroy(ge)); CK(cudaGraphDestroy(g));
    return med;
  };
  if (argc > 1) {  // ncu mode: each kernel once, eager, after a flush
    for (int rep = 0; rep < 2; ++rep) {
      flush(true);
      copy_k<<<sms * 2, 512, 0, s>>>((const uint4*)q, (uint4*)out, nv);
      flush(true);
      spec_k<4, 0><<<sms * 2, 512, 0, s>>>((const uint4*)q, (uint4*)out, nv, 0.125f, partials, counter, pf, 0, n);
      flush(true);
      spec2_k<4, 0><<<sms * 2, 512, 0, s>>>((const uint4*)q, (uint4*)out, nv, 0x3e003e00u, partials, counter, pf, n);
      flush(true);
      fix_k<<<sms * 2, 512, 0, s>>>((const uint4*)q, (uint4*)out, nv, 0.125f, nullptr);
      flush(true);
      spec3_k<6, 1><<<sms * 2, 512, 0, s>>>((const uint4*)q, (uint4*)out, nv, 0x3e003e00u, partials, counter, pf, n);
      flush(true);
      exact3_k<6><<<sms * 2, 512, 0, s>>>((const uint4*)q, (uint4*)out, nv, 0x3e003e00u, partials, counter, pf, n);
      flush(true);
      copy3_k<<<sms * 2, 512, 0, s>>>((const uint4*)q, (uint4*)out, nv);
    }
    CK(cudaStreamSynchronize(s));
    return 0;
  }
  for (int clean = 0; clean < 2; ++clean) {
    printf("--- flush: %s\n", clean ? "memset 256 MB + read 256 MB (clean L2)" : "memset 256 MB (dirty L2)");
    double base = timeit("flush", [&] { flush(clean); }, 0);
    for (int grid_mult : {1, 2, 4}) {
      char nm[64]; snprintf(nm, 64, "copy grid=%dx148x512", grid_mult);
      timeit(nm, [&] { flush(clean); copy_k<<<sms * grid_mult, 512, 0, s>>>((const uint4*)q, (uint4*)out, nv); }, base);
    }
    for (int grid_mult : {2, 4}) {
      char nm[64]; snprintf(nm, 64, "spec U4 grid=%dx148", grid_mult);
      timeit(nm, [&] { flush(clean); spec_k<4, 0><<<sms * grid_mult, 512, 0, s>>>((const uint4*)q, (uint4*)out, nv, 0.125f, partials, counter, pf, 0, n); }, base);
      snprintf(nm, 64, "spec U2 grid=%dx148", grid_mult);
      timeit(nm, [&] { flush(clean); spec_k<2, 0><<<sms * grid_mult, 512, 0, s>>>((const uint4*)q, (uint4*)out, nv, 0.125f, partials, counter, pf, 0, n); }, base);
    }
    for (int gm : {1, 2}) {
      char nm[64];
      snprintf(nm, 64, "spec2 packed U4 last-arriver g=%dx148", gm);
      timeit(nm, [&] { flush(clean); spec2_k<4, 0><<<sms * gm, 512, 0, s>>>((const uint4*)q, (uint4*)out, nv, 0x3e003e00u, partials, counter, pf, n); }, base);
      snprintf(nm, 64, "spec2 packed U4 end-barrier g=%dx148", gm);
      timeit(nm, [&] { flush(clean); spec2_k<4, 1><<<sms * gm, 512, 0, s>>>((const uint4*)q, (uint4*)out, nv, 0x3e003e00u, partials, counter, pf, n); }, base);
      snprintf(nm, 64, "spec2 packed U2 end-barrier g=%dx148", gm);
      timeit(nm, [&] { flush(clean); spec2_k<2, 1><<<sms * gm, 512, 0, s>>>((const uint4*)q, (uint4*)out, nv, 0x3e003e00u, partials, counter, pf, n); }, base);
      snprintf(nm, 64, "copy chunked U4 g=%dx148", gm);
      timeit(nm, [&] { flush(clean); copy_chunk_k<<<sms * gm, 512, 0, s>>>((const uint4*)q, (uint4*)out, nv); }, base);
    }
    // K = ceil(786432 / (296*512)) = 6
    timeit("copy3 all-loads-upfront g=2x148", [&] { flush(clean); copy3_k<<<sms * 2, 512, 0, s>>>((const uint4*)q, (uint4*)out, nv); }, base);
    timeit("spec3 K6 last-arriver g=2x148", [&] { flush(clean); spec3_k<6, 0><<<sms * 2, 512, 0, s>>>((const uint4*)q, (uint4*)out, nv, 0x3e003e00u, partials, counter, pf, n); }, base);
    timeit("spec3 K6 end-barrier g=2x148", [&] { flush(clean); spec3_k<6, 1><<<sms * 2, 512, 0, s>>>((const uint4*)q, (uint4*)out, nv, 0x3e003e00u, partials, counter, pf, n); }, base);
    timeit("exact3 K6 2-pass regs g=2x148", [&] { flush(clean); exact3_k<6><<<sms * 2, 512, 0, s>>>((const uint4*)q, (uint4*)out, nv, 0x3e003e00u, partials, counter, pf, n); }, base);
    timeit("spec3 K12 end-barrier g=1x148", [&] { flush(clean); spec3_k<12, 1><<<sms, 512, 0, s>>>((const uint4*)q, (uint4*)out, nv, 0x3e003e00u, partials, counter, pf, n); }, base);
#define L4(K, SIG, TH, MB, KS, GRID) timeit("spec4 K" #K " sig" #SIG " th" #TH " minb" #MB " ks" #KS, [&] { flush(clean); spec4_k<K, SIG, TH, MB, KS><<<GRID, TH, 0, s>>>((const uint4*)q, (uint4*)out, nv, 0x3e003e00u, partials, counter, pf, n); }, base)
    L4(6, 0, 512, 2, false, sms * 2);
    L4(6, 1, 512, 2, false, sms * 2);
    L4(6, 2, 512, 2, false, sms * 2);
    L4(6, 0, 512, 2, true, sms * 2);
    L4(3, 0, 1024, 2, false, sms * 2);
    L4(3, 1, 1024, 2, false, sms * 2);
    L4(3, 2, 1024, 2, false, sms * 2);
    L4(3, 0, 512, 4, false, sms * 4);
    timeit("spec U4 + exit-kernel", [&] {
      flush(clean);
      spec_k<4, 2><<<sms * 2, 512, 0, s>>>((const uint4*)q, (uint4*)out, nv, 0.125f, partials, counter, pf, 0, n);
      fix_k<<<sms * 2, 512, 0, s>>>((const uint4*)q, (uint4*)out, nv, 0.125f, pf);
    }, base);
    timeit("spec U4 + conditional node", [&] {
      flush(clean);
      cudaStreamCaptureStatus st; cudaGraph_t g; const cudaGraphNode_t* deps; size_t nd;
      CK(cudaStreamGetCaptureInfo(s, &st, nullptr, &g, &deps, &nd));
      cudaGraphConditionalHandle h;
      CK(cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault));
      spec_k<4, 1><<<sms * 2, 512, 0, s>>>((const uint4*)q, (uint4*)out, nv, 0.125f, partials, counter, pf, h, n);
      CK(cudaStreamGetCaptureInfo(s, &st, nullptr, &g, &deps, &nd));
      cudaGraphNodeParams cp = {};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = h;
      cp.conditional.type = cudaGraphCondTypeIf;
      cp.conditional.size = 1;
      cudaGraphNode_t node;
      CK(cudaGraphAddNode(&node, g, deps, nd, &cp));
      cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
      CK(cudaStreamBeginCaptureToGraph(s2, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
      fix_k<<<sms * 2, 512, 0, s2>>>((const uint4*)q, (uint4*)out, nv, 0.125f, nullptr);
      CK(cudaStreamEndCapture(s2, &bodyg));
      CK(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
    }, base);
    timeit("fix kernel alone (always runs)", [&] { flush(clean); fix_k<<<sms * 2, 512, 0, s>>>((const uint4*)q, (uint4*)out, nv, 0.125f, nullptr); }, base);
  }
  // mispredict check: flip the stored prediction each step via memset
  return 0;
}
