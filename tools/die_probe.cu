// die_probe.cu — latency of a dependent chain of global atomics from every SM
// to a set of candidate L2 lines (B200: two dies; an address homed in the
// other die's L2 costs a die-to-die round trip).  Prints, per line, the mean
// latency seen by SMs [0,74) and [74,148) and the per-SM split.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/die_probe tools/die_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void probe(unsigned long long* lines, int nlines, long long stride_words, float* lat, int* smids) {
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x != 0) return;
  smids[blockIdx.x] = smid;
  for (int i = 0; i < nlines; ++i) {
    unsigned long long* p = lines + (long long)i * stride_words;
    unsigned long long v = 0;
    atomicAdd(p, 0ull);  // warm the TLB
    long long t0 = clock64();
    for (int k = 0; k < 32; ++k) v = atomicAdd(p + (v >> 62), 1ull);
    long long t1 = clock64();
    lat[blockIdx.x * nlines + i] = (float)(t1 - t0) / 32.f + (v == 12345678ull ? 1.f : 0.f);
  }
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int nlines = 48;
  const long long stride = (64 << 10) / 8;  // 64 KB apart
  unsigned long long* lines; float* lat; int* smids;
  CK(cudaMalloc(&lines, (size_t)nlines * stride * 8)); CK(cudaMemset(lines, 0, (size_t)nlines * stride * 8));
  CK(cudaMalloc(&lat, sizeof(float) * sms * nlines)); CK(cudaMalloc(&smids, sizeof(int) * sms));
  // one CTA at a time per SM would need placement control; launch sms CTAs (one lands per SM in practice)
  for (int rep = 0; rep < 2; ++rep) probe<<<sms, 32>>>(lines, nlines, stride, lat, smids);
  CK(cudaDeviceSynchronize());
  std::vector<float> h(sms * nlines); std::vector<int> id(sms);
  CK(cudaMemcpy(h.data(), lat, h.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(id.data(), smids, sms * 4, cudaMemcpyDeviceToHost));
  printf("line  mean_cycles(smid<74)  mean_cycles(smid>=74)  min  max\n");
  for (int i = 0; i < nlines; ++i) {
    double a = 0, b = 0; int na = 0, nb = 0; float mn = 1e9, mx = 0;
    for (int c = 0; c < sms; ++c) {
      float v = h[c * nlines + i];
      if (id[c] < 74) { a += v; ++na; } else { b += v; ++nb; }
      mn = v < mn ? v : mn; mx = v > mx ? v : mx;
    }
    printf("%4d  %8.0f  %8.0f  %6.0f %6.0f\n", i, na ? a / na : 0, nb ? b / nb : 0, mn, mx);
  }
  return 0;
}
