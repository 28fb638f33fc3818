"""Micro-benchmark of the grid-wide reduce + broadcast used between region
passes: K back-to-back reduces (no other work) at the region grid, per-call
time from CUDA events over one launch.  Variants of the protocol are defined
here (V0 = gm::grid_reduce as shipped (the V3 protocol)) to pick the fastest on B200.

    python tools/barrier_bench.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SRC = r'''
#include "gm_region.cuh"
using namespace gm;

__device__ __forceinline__ void red_release_add64(u64* p, u64 v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel() { fence_acq_rel_gpu(); }

// V = variant: 1 relaxed polling + fence; 2 = 1 without nanosleep;
// 3 = all CTAs poll the arrival counter, CTA 0 combines (red.release arrivals)
template <int V>
__device__ __forceinline__ void grid_reduce_v(const Params& P, double v_in, double* s_warp, double* s_out) {
  __shared__ int s_last;
  __shared__ u64 s_epoch;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double v = warp_combine(GM_R_SUM, v_in);
  if (lane == 0) s_warp[warp * GM_MAX_RED] = v;
  __syncthreads();
  double* partials = (double*)P.partials;
  if (warp == 0) {
    double w = lane < GM_WARPS ? s_warp[lane * GM_MAX_RED] : 0.0;
    w = warp_combine(GM_R_SUM, w);
    if (lane == 0) partials[blockIdx.x] = w;
  }
  u64* cnt = (u64*)P.barrier;
  u64* flag = (u64*)((char*)P.barrier + GM_SCRATCH_FLAG);
  double* results = (double*)((char*)P.barrier + GM_SCRATCH_RESULTS);
  const u64 g = gridDim.x;
  if (V == 3) {
    if (threadIdx.x == 0) {
      u64 old = atom_add_acq_rel64(cnt, 1ull);
      s_epoch = old / g + 1;
      const u64 target = s_epoch * g;
      while (ld_relaxed64(cnt) < target) {}
      fence_acq_rel();
    }
    __syncthreads();
    if (warp == 0) {
      double acc = 0.0;
      for (u32 b0 = 0; b0 < g; b0 += 32 * 16) {
        double t[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) { const u32 b = b0 + i * 32 + lane; t[i] = b < g ? ld_relaxed_f64(partials + b) : 0.0; }
#pragma unroll
        for (int i = 0; i < 16; ++i) acc += t[i];
      }
      acc = warp_combine(GM_R_SUM, acc);
      if (lane == 0) s_out[0] = acc;
    }
    __syncthreads();
    return;
  }
  if (threadIdx.x == 0) {
    const u64 old = atom_add_acq_rel64(cnt, 1ull);
    s_epoch = old / g + 1;
    s_last = (old + 1) % g == 0;
  }
  __syncthreads();
  if (s_last) {
    if (warp == 0) {
      double acc = 0.0;
      for (u32 b0 = 0; b0 < g; b0 += 32 * 16) {
        double t[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) { const u32 b = b0 + i * 32 + lane; t[i] = b < g ? ld_relaxed_f64(partials + b) : 0.0; }
#pragma unroll
        for (int i = 0; i < 16; ++i) acc += t[i];
      }
      acc = warp_combine(GM_R_SUM, acc);
      if (lane == 0) { s_out[0] = acc; results[0] = acc; }
    }
    __syncthreads();
    if (threadIdx.x == 0) st_release64(flag, s_epoch);
  } else {
    if (threadIdx.x == 0) {
      int spins = 0;
      while (ld_relaxed64(flag) < s_epoch) { if (V == 1 && ++spins > 64) __nanosleep(32); }
      fence_acq_rel();
      s_out[0] = ld_relaxed_f64(results);
    }
    __syncthreads();
  }
}

template <int V>
__device__ void body(const Params& P) {
  __shared__ double s_warp[GM_WARPS * GM_MAX_RED];
  __shared__ double s_red[GM_MAX_RED];
  double acc = (double)(threadIdx.x + blockIdx.x);
  const int ops[1] = {GM_R_SUM};
  const int slots[1] = {0};
  u64 ep_ = grid_epoch_begin(P);
  for (int k = 0; k < (int)P.n; ++k) {
    if (V == 0) {
      double vals[1] = {acc};
      grid_reduce(P, 1, ops, slots, vals, s_warp, s_red, ep_);
    } else {
      grid_reduce_v<V>(P, acc, s_warp, s_red);
    }
    acc += s_red[0] * 1e-30;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) ((double*)P.scal_out)[0] = acc;
}

extern "C" __global__ void __launch_bounds__(GM_THREADS, 2) bar_v0(const __grid_constant__ Params P) { body<0>(P); }
extern "C" __global__ void __launch_bounds__(GM_THREADS, 2) bar_v1(const __grid_constant__ Params P) { body<1>(P); }
extern "C" __global__ void __launch_bounds__(GM_THREADS, 2) bar_v2(const __grid_constant__ Params P) { body<2>(P); }
extern "C" __global__ void __launch_bounds__(GM_THREADS, 2) bar_v3(const __grid_constant__ Params P) { body<3>(P); }
'''


def main():
    import torch

    from paper_2509_16248_b200 import _native as nat

    torch.cuda.set_device(0)
    nat.init(0)
    for v in range(4):
        k = nat.CompiledRegion(SRC, f"bar_v{v}")
        for grid in (148, 296):
            res = []
            for K in (8, 72):
                scratch = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
                base = scratch.data_ptr()
                P = nat.Params()
                P.n = K
                P.barrier = base
                P.status = base + 16
                P.partials = base + 384
                P.scal_out = base + 65536
                stream = torch.cuda.current_stream().cuda_stream
                for _ in range(3):
                    k.launch(P, grid, nat.THREADS, 0, stream)
                torch.cuda.synchronize()
                ts = []
                for _ in range(5):
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s.record()
                    k.launch(P, grid, nat.THREADS, 0, stream)
                    e.record()
                    e.synchronize()
                    ts.append(s.elapsed_time(e) * 1e3)
                res.append(min(ts))
            per = (res[1] - res[0]) / 64
            print(f"variant {v} grid {grid}: {per:.2f} us per grid reduce (launch+8: {res[0]:.1f} us)")


if __name__ == "__main__":
    main()
