// Time every cuBLASLt heuristic candidate for the BigBird-like projection
// (x[8192,768] @ W^T[768,768] + b, bf16 in/out, fp32 accumulate, BIAS
// epilogue) — does the default pick leave time on the table?
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/gemm_algos.cu -lcublasLt -o tools/gemm_algos
#include <cublasLt.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

#define CK(x) do { auto e_ = (x); if ((int)e_ != 0) { printf("%s:%d error %d\n", __FILE__, __LINE__, (int)e_); exit(1); } } while (0)

int main(int argc, char** argv) {
  const int M = argc > 1 ? atoi(argv[1]) : 8192, N = 768, K = 768;
  const int flushMB = 256;
  __nv_bfloat16 *x, *w, *b, *y;
  char* flush;
  CK(cudaMalloc(&x, (size_t)M * K * 2)); CK(cudaMalloc(&w, (size_t)N * K * 2));
  CK(cudaMalloc(&b, N * 2)); CK(cudaMalloc(&y, (size_t)M * N * 2));
  CK(cudaMalloc(&flush, (size_t)flushMB << 20));
  CK(cudaMemset(x, 0x3c, (size_t)M * K * 2)); CK(cudaMemset(w, 0x3c, (size_t)N * K * 2)); CK(cudaMemset(b, 0, N * 2));
  cublasLtHandle_t lt; CK(cublasLtCreate(&lt));
  cublasLtMatmulDesc_t op; CK(cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F));
  cublasOperation_t tA = CUBLAS_OP_T, tB = CUBLAS_OP_N;
  CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &tA, sizeof tA));
  CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tB, sizeof tB));
  cublasLtEpilogue_t ep = CUBLASLT_EPILOGUE_BIAS;
  CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_EPILOGUE, &ep, sizeof ep));
  CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &b, sizeof b));
  cublasLtMatrixLayout_t la, lb, lc;
  CK(cublasLtMatrixLayoutCreate(&la, CUDA_R_16BF, K, N, K));   // W as stored: [N][K] row-major == K x N col-major
  CK(cublasLtMatrixLayoutCreate(&lb, CUDA_R_16BF, K, M, K));   // x: K x M col-major
  CK(cublasLtMatrixLayoutCreate(&lc, CUDA_R_16BF, N, M, N));   // y: N x M col-major
  size_t ws_bytes = 32 << 20; void* ws; CK(cudaMalloc(&ws, ws_bytes));
  cublasLtMatmulPreference_t pref; CK(cublasLtMatmulPreferenceCreate(&pref));
  CK(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &ws_bytes, sizeof ws_bytes));
  std::vector<cublasLtMatmulHeuristicResult_t> res(64);
  int got = 0;
  CK(cublasLtMatmulAlgoGetHeuristic(lt, op, la, lb, lc, lc, pref, 64, res.data(), &got));
  printf("M=%d N=%d K=%d: %d candidates\n", M, N, K, got);
  float one = 1.f, zero = 0.f;
  cudaStream_t s; CK(cudaStreamCreate(&s));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const double flops = 2.0 * M * N * K;
  for (int i = 0; i < got; ++i) {
    auto run = [&]() {
      return cublasLtMatmul(lt, op, &one, w, la, x, lb, &zero, y, lc, y, lc, &res[i].algo, ws, ws_bytes, s);
    };
    if (run() != CUBLAS_STATUS_SUCCESS) { printf("%2d failed\n", i); continue; }
    CK(cudaStreamSynchronize(s));
    // warm (L2-resident operands) and cold (256 MB flush before each)
    std::vector<float> warm, cold;
    for (int r = 0; r < 30; ++r) {
      CK(cudaEventRecord(e0, s)); run(); CK(cudaEventRecord(e1, s)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); warm.push_back(ms * 1e3f);
      CK(cudaMemsetAsync(flush, r, (size_t)flushMB << 20, s));
      CK(cudaEventRecord(e0, s)); run(); CK(cudaEventRecord(e1, s)); CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1)); cold.push_back(ms * 1e3f);
    }
    std::sort(warm.begin(), warm.end()); std::sort(cold.begin(), cold.end());
    int tile = 0, stages = 0, splitk = 0, cluster = 0;
    size_t sz;
    cublasLtMatmulAlgoConfigGetAttribute(&res[i].algo, CUBLASLT_ALGO_CONFIG_TILE_ID, &tile, sizeof tile, &sz);
    cublasLtMatmulAlgoConfigGetAttribute(&res[i].algo, CUBLASLT_ALGO_CONFIG_STAGES_ID, &stages, sizeof stages, &sz);
    cublasLtMatmulAlgoConfigGetAttribute(&res[i].algo, CUBLASLT_ALGO_CONFIG_SPLITK_NUM, &splitk, sizeof splitk, &sz);
    cublasLtMatmulAlgoConfigGetAttribute(&res[i].algo, CUBLASLT_ALGO_CONFIG_CLUSTER_SHAPE_ID, &cluster, sizeof cluster, &sz);
    printf("%2d tile %3d stages %3d splitk %2d cluster %2d ws %8zu  warm p50 %6.2f us (%5.0f TF/s)  cold p50 %6.2f us\n",
           i, tile, stages, splitk, cluster, res[i].workspaceSize, warm[15], flops / warm[15] / 1e6, cold[15]);
  }
  return 0;
}
