// Probe: fp32 Linear (y = x @ W^T + b, M=8192 N=768 K=768) on cuBLASLt 12.9
// with CUBLAS_COMPUTE_32F (SIMT SGEMM) vs CUBLAS_COMPUTE_32F_EMULATED_16BFX9
// (BF16x9 on the tensor cores), strided and pointer-array (batch 1) layouts.
// Accuracy against an fp64 host product on a sample of rows; time with events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/gp tools/gemm_emu_probe.cu -lcublasLt
#include <cublasLt.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x) do { auto e_ = (x); if ((int)e_ != 0) { printf("ERR %s:%d %d\n", __FILE__, __LINE__, (int)e_); exit(1); } } while (0)

struct Run {
  double ms, max_rel_floor, max_abs, max_rel;
  int algos;
};

static Run run(cublasLtHandle_t h, cublasComputeType_t ct, bool ptr_array, bool bias, int M, int N, int K, const float* dx,
               const float* dw, const float* db, float* dy, const std::vector<float>& x, const std::vector<float>& w,
               const std::vector<float>& b, void* ws, size_t wsb) {
  cublasLtMatmulDesc_t op;
  CK(cublasLtMatmulDescCreate(&op, ct, CUDA_R_32F));
  cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
  CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta)));
  CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb)));
  cublasLtEpilogue_t epi = bias ? CUBLASLT_EPILOGUE_BIAS : CUBLASLT_EPILOGUE_DEFAULT;
  CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_EPILOGUE, &epi, sizeof(epi)));
  if (bias) CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &db, sizeof(db)));
  cublasLtMatrixLayout_t la, lb, lc;
  CK(cublasLtMatrixLayoutCreate(&la, CUDA_R_32F, K, N, K));
  CK(cublasLtMatrixLayoutCreate(&lb, CUDA_R_32F, K, M, K));
  CK(cublasLtMatrixLayoutCreate(&lc, CUDA_R_32F, N, M, N));
  const void *A = dw, *B = dx;
  void* C = dy;
  void** parr = nullptr;
  if (ptr_array) {
    int32_t mode = CUBLASLT_BATCH_MODE_POINTER_ARRAY;
    int32_t one = 1;
    for (auto l : {la, lb, lc}) {
      CK(cublasLtMatrixLayoutSetAttribute(l, CUBLASLT_MATRIX_LAYOUT_BATCH_MODE, &mode, sizeof(mode)));
      CK(cublasLtMatrixLayoutSetAttribute(l, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &one, sizeof(one)));
    }
    CK(cudaMalloc(&parr, 3 * sizeof(void*)));
    void* hp[3] = {(void*)dw, (void*)dx, (void*)dy};
    CK(cudaMemcpy(parr, hp, sizeof(hp), cudaMemcpyHostToDevice));
    A = parr;
    B = parr + 1;
    C = parr + 2;
  }
  cublasLtMatmulPreference_t pref;
  CK(cublasLtMatmulPreferenceCreate(&pref));
  CK(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsb, sizeof(wsb)));
  cublasLtMatmulHeuristicResult_t res[8];
  int nres = 0;
  auto st = cublasLtMatmulAlgoGetHeuristic(h, op, la, lb, lc, lc, pref, 8, res, &nres);
  Run r{-1, -1, -1, -1, nres};
  if (st != 0 || nres == 0) {
    printf("  no algo (status %d)\n", (int)st);
    return r;
  }
  float alpha = 1.f, beta = 0.f;
  double best = 1e30;
  for (int a = 0; a < nres; ++a) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int i = 0; i < 5; ++i)
      CK(cublasLtMatmul(h, op, &alpha, A, la, B, lb, &beta, C, lc, C, lc, &res[a].algo, ws, wsb, 0));
    cudaEventRecord(e0);
    for (int i = 0; i < 50; ++i)
      cublasLtMatmul(h, op, &alpha, A, la, B, lb, &beta, C, lc, C, lc, &res[a].algo, ws, wsb, 0);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms / 50 < best) best = ms / 50;
  }
  // accuracy with algo 0 (the heuristic's pick)
  CK(cublasLtMatmul(h, op, &alpha, A, la, B, lb, &beta, C, lc, C, lc, &res[0].algo, ws, wsb, 0));
  CK(cudaDeviceSynchronize());
  std::vector<float> y((size_t)M * N);
  CK(cudaMemcpy(y.data(), dy, y.size() * 4, cudaMemcpyDeviceToHost));
  double mrf = 0, mab = 0, mre = 0;
  for (int i = 0; i < M; i += 37) {
    for (int j = 0; j < N; ++j) {
      double s = bias ? b[j] : 0.0;
      for (int k = 0; k < K; ++k) s += (double)x[(size_t)i * K + k] * (double)w[(size_t)j * K + k];
      double d = std::fabs((double)y[(size_t)i * N + j] - s);
      mab = std::max(mab, d);
      mre = std::max(mre, d / std::max(std::fabs(s), 1e-30));
      mrf = std::max(mrf, d / (std::fabs(s) + 1e-6 / 1e-5));
    }
  }
  r.ms = best;
  r.max_rel_floor = mrf;
  r.max_abs = mab;
  r.max_rel = mre;
  return r;
}

int main() {
  const int M = 8192, N = 768, K = 768;
  std::mt19937 g(0);
  std::normal_distribution<float> nd;
  std::uniform_real_distribution<float> ud(-1.f / std::sqrt((float)K), 1.f / std::sqrt((float)K));
  std::vector<float> x((size_t)M * K), w((size_t)N * K), b(N);
  for (auto& v : x) v = nd(g);
  for (auto& v : w) v = ud(g);
  for (auto& v : b) v = ud(g);
  float *dx, *dw, *db, *dy;
  CK(cudaMalloc(&dx, x.size() * 4));
  CK(cudaMalloc(&dw, w.size() * 4));
  CK(cudaMalloc(&db, b.size() * 4));
  CK(cudaMalloc(&dy, (size_t)M * N * 4));
  CK(cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dw, w.data(), w.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, b.data(), b.size() * 4, cudaMemcpyHostToDevice));
  size_t wsb = 32 << 20;
  void* ws;
  CK(cudaMalloc(&ws, wsb));
  cublasLtHandle_t h;
  CK(cublasLtCreate(&h));
  printf("cublasLt version %zu\n", cublasLtGetVersion());
  struct { const char* name; cublasComputeType_t ct; bool pa; bool bias; } cases[] = {
      {"32F strided bias", CUBLAS_COMPUTE_32F, false, true},
      {"32F_EMULATED_16BFX9 strided bias", CUBLAS_COMPUTE_32F_EMULATED_16BFX9, false, true},
      {"32F_EMULATED_16BFX9 strided nobias", CUBLAS_COMPUTE_32F_EMULATED_16BFX9, false, false},
      {"32F ptr-array b1 nobias", CUBLAS_COMPUTE_32F, true, false},
      {"32F_EMULATED_16BFX9 ptr-array b1 nobias", CUBLAS_COMPUTE_32F_EMULATED_16BFX9, true, false},
  };
  for (auto& c : cases) {
    Run r = run(h, c.ct, c.pa, c.bias, M, N, K, dx, dw, db, dy, x, w, b, ws, wsb);
    printf("%-40s algos=%d best_ms=%.4f  TFLOPs=%.1f  max_abs=%.3e max_rel=%.3e max(|d|/(|r|+0.1))=%.3e\n", c.name,
           r.algos, r.ms, r.ms > 0 ? 2.0 * M * N * K / (r.ms * 1e-3) / 1e12 : 0.0, r.max_abs, r.max_rel,
           r.max_rel_floor);
  }
  return 0;
}
