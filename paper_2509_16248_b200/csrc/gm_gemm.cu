// gm_gemm.cu — dense contractions of the transformed forward (north_star:
// they stay on cuBLAS / tcgen05 and are not re-implemented) plus the
// device-side operand select that lets a predicated block whose two arms
// each contain a GEMM run ONE GEMM (transform.py:272:
// torch-rooted calls such as torch.matmul are legal arm expressions).
//
//  * fp32 GEMMs run on cuBLASLt 12.9 with CUBLAS_COMPUTE_32F_EMULATED_16BFX9:
//    each fp32 operand is split into three bf16 terms and the products run
//    on the tcgen05 tensor cores with fp32 accumulation.  Measured on B200 at
//    the BigBird Linear shape (M=8192, N=K=768, tools/gemm_emu_probe.cu,
//    profiles/r02_gemm_emu_probe.txt): 0.082 ms vs 0.211 ms for SIMT SGEMM,
//    max abs error vs an fp64 product 1.26e-6 vs 2.56e-6 — faster AND
//    closer to the exact product than the SGEMM torch would run.
//  * PyTorch (2.11+cu128) already maps libcublasLt.so.12 from cuBLAS 12.8,
//    which has no BF16x9 path; the 12.9 library is loaded privately by full
//    path (RTLD_LOCAL; the library is linked -Bsymbolic, so it binds to
//    itself), never through the soname torch's copy answers to.
//  * gm_select_copy: one kernel reads a 0-d predicate on the device and
//    copies the selected operand into a staging buffer, so
//    `where(p, A1 @ B1, A2 @ B2)` costs one copy of the operand that differs
//    plus ONE GEMM — no host sync, no conditional graph node (a conditional
//    node costs 7-11 us on this driver, profiles/r01_cond_node_cost.txt).
//    cuBLASLt's pointer-array batch mode would avoid the copy, but it has no
//    BF16x9 kernels (status 15 on B200, profiles/r02_gemm_emu_probe.txt).

#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "../../include/gm_b200.h"

int gm_internal_fail(int code, const char* msg);  // gm_runtime.cu

// The cuBLASLt 12.9 header is used for types and constants only: nothing is
// linked against libcublasLt, every entry point is resolved from the private
// dlopen handle below.
#include <cublasLt.h>

namespace {

int gfail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  return gm_internal_fail(code, buf);  // gm_last_error() reports it
}

struct LtApi {
  void* so = nullptr;
  decltype(&cublasLtCreate) Create;
  decltype(&cublasLtDestroy) Destroy;
  decltype(&cublasLtGetVersion) GetVersion;
  decltype(&cublasLtMatmulDescCreate) DescCreate;
  decltype(&cublasLtMatmulDescDestroy) DescDestroy;
  decltype(&cublasLtMatmulDescSetAttribute) DescSet;
  decltype(&cublasLtMatrixLayoutCreate) LayoutCreate;
  decltype(&cublasLtMatrixLayoutDestroy) LayoutDestroy;
  decltype(&cublasLtMatrixLayoutSetAttribute) LayoutSet;
  decltype(&cublasLtMatmulPreferenceCreate) PrefCreate;
  decltype(&cublasLtMatmulPreferenceDestroy) PrefDestroy;
  decltype(&cublasLtMatmulPreferenceSetAttribute) PrefSet;
  decltype(&cublasLtMatmulAlgoGetHeuristic) Heuristic;
  decltype(&cublasLtMatmul) Matmul;
};

LtApi g_lt;
std::mutex g_lt_mu;

const char* kLtCandidates[] = {
    "/usr/local/cuda/lib64/libcublasLt.so.12",
    "/usr/local/cuda/targets/x86_64-linux/lib/libcublasLt.so.12",
};

int load_lt() {
  if (g_lt.so) return GM_OK;
  void* h = nullptr;
  const char* env = getenv("GM_CUBLASLT");
  std::string tried;
  for (int i = -1; i < (int)(sizeof(kLtCandidates) / sizeof(kLtCandidates[0])) && !h; ++i) {
    const char* path = i < 0 ? env : kLtCandidates[i];
    if (!path) continue;
    h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
    if (!h) tried += std::string(path) + ": " + dlerror() + "; ";
  }
  if (!h) return gfail(GM_E_CUDA, "gm_gemm: cannot load cuBLASLt 12.9 (%s)", tried.c_str());
#define GM_LT(field, name)                                                           \
  g_lt.field = (decltype(g_lt.field))dlsym(h, name);                                 \
  if (!g_lt.field) return gfail(GM_E_CUDA, "gm_gemm: cuBLASLt lacks %s", name);
  GM_LT(Create, "cublasLtCreate");
  GM_LT(Destroy, "cublasLtDestroy");
  GM_LT(GetVersion, "cublasLtGetVersion");
  GM_LT(DescCreate, "cublasLtMatmulDescCreate");
  GM_LT(DescDestroy, "cublasLtMatmulDescDestroy");
  GM_LT(DescSet, "cublasLtMatmulDescSetAttribute");
  GM_LT(LayoutCreate, "cublasLtMatrixLayoutCreate");
  GM_LT(LayoutDestroy, "cublasLtMatrixLayoutDestroy");
  GM_LT(LayoutSet, "cublasLtMatrixLayoutSetAttribute");
  GM_LT(PrefCreate, "cublasLtMatmulPreferenceCreate");
  GM_LT(PrefDestroy, "cublasLtMatmulPreferenceDestroy");
  GM_LT(PrefSet, "cublasLtMatmulPreferenceSetAttribute");
  GM_LT(Heuristic, "cublasLtMatmulAlgoGetHeuristic");
  GM_LT(Matmul, "cublasLtMatmul");
#undef GM_LT
  if (g_lt.GetVersion() < 120900) {
    size_t v = g_lt.GetVersion();
    dlclose(h);
    return gfail(GM_E_CUDA, "gm_gemm: cuBLASLt %zu has no BF16x9 emulation (need >= 12.9)", v);
  }
  g_lt.so = h;
  return GM_OK;
}

// one cached plan per problem
using Key = std::tuple<int, int64_t, int64_t, int64_t, int64_t, int64_t, int, int, int, int64_t, int64_t, int64_t,
                       int64_t>;
struct Plan {
  cublasLtMatmulDesc_t desc = nullptr;
  cublasLtMatrixLayout_t la = nullptr, lb = nullptr, lc = nullptr;
  cublasLtMatmulAlgo_t algo;
  size_t ws = 0;
};

int lt_type(int dtype) {
  switch (dtype) {
    case GM_F32: return CUDA_R_32F;
    case GM_BF16: return CUDA_R_16BF;
    case GM_F16: return CUDA_R_16F;
  }
  return -1;
}

__global__ void gm_select_copy_kernel(const unsigned char* __restrict__ pred, int pred_bytes,
                                      const uint4* __restrict__ a, const uint4* __restrict__ b,
                                      uint4* __restrict__ dst, long long nvec) {
  // the predicate of a `where` is a 0-d bool (or any 0-d value: non-zero = true)
  bool p = false;
  for (int i = 0; i < pred_bytes; ++i) p |= pred[i] != 0;
  const uint4* __restrict__ src = p ? a : b;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nvec;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = __ldg(src + i);
}

__global__ void gm_select_copy_tail_kernel(const unsigned char* __restrict__ pred, int pred_bytes,
                                           const unsigned char* __restrict__ a,
                                           const unsigned char* __restrict__ b, unsigned char* __restrict__ dst,
                                           long long n) {
  bool p = false;
  for (int i = 0; i < pred_bytes; ++i) p |= pred[i] != 0;
  const unsigned char* src = p ? a : b;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// dst (packed, row-major over `sizes`) = src (strides in 16-byte vectors,
// innermost dim contiguous): one 16-byte vector per thread and step, the
// vector's source offset decoded from its index (sizes[ndim-1] counts
// vectors).  Stores are fully coalesced; loads are 16-byte pieces of the
// source rows (a [b, n, h, d] -> [b, h, n, d] head split reads whole d rows).
struct CopyDesc {
  long long stride[6];    // in 16-byte vectors
  unsigned size[6];
  unsigned mul[6], shr[6];  // x / size = umulhi(x, mul) >> shr (32-bit index space)
  int ndim;
};

// round-up magic numbers for unsigned 32-bit division by d (d >= 1)
static void fast_divmod(unsigned d, unsigned& mul, unsigned& shr) {
  if (d == 1) { mul = 0; shr = 0; return; }
  unsigned s = 0;
  while ((1ull << s) < d) ++s;
  mul = (unsigned)(((1ull << 32) * ((1ull << s) - d)) / d + 1);
  shr = s;
}

__device__ __forceinline__ unsigned fdiv(unsigned x, unsigned mul, unsigned shr) {
  if (mul == 0 && shr == 0) return x;
  const unsigned t = __umulhi(x, mul);
  return (t + ((x - t) >> 1)) >> (shr - 1);
}

__global__ void __launch_bounds__(256) gm_copy_strided_kernel(const uint4* __restrict__ src,
                                                              uint4* __restrict__ dst, const CopyDesc d,
                                                              unsigned nvec) {
  for (unsigned v = blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += gridDim.x * blockDim.x) {
    unsigned i = v;
    long long off = 0;
#pragma unroll
    for (int j = 5; j >= 0; --j) {
      if (j >= d.ndim) continue;
      const unsigned q = fdiv(i, d.mul[j], d.shr[j]);
      off += (long long)(i - q * d.size[j]) * d.stride[j];
      i = q;
    }
    dst[v] = __ldg(src + off);
  }
}

}  // namespace

struct gm_gemm_s {
  cublasLtHandle_t h = nullptr;
  std::map<Key, Plan> plans;
  std::mutex mu;
};

extern "C" {

int gm_gemm_open(gm_gemm* out) {
  if (!out) return gfail(GM_E_INVALID, "gm_gemm_open: null out");
  std::lock_guard<std::mutex> lk(g_lt_mu);
  int r = load_lt();
  if (r) return r;
  auto* g = new gm_gemm_s();
  if (g_lt.Create(&g->h) != 0) {
    delete g;
    return gfail(GM_E_CUDA, "gm_gemm_open: cublasLtCreate failed");
  }
  *out = g;
  return GM_OK;
}

int gm_gemm_close(gm_gemm g) {
  if (!g) return GM_OK;
  for (auto& kv : g->plans) {
    g_lt.DescDestroy(kv.second.desc);
    g_lt.LayoutDestroy(kv.second.la);
    g_lt.LayoutDestroy(kv.second.lb);
    g_lt.LayoutDestroy(kv.second.lc);
  }
  g_lt.Destroy(g->h);
  delete g;
  return GM_OK;
}

size_t gm_gemm_version(void) {
  std::lock_guard<std::mutex> lk(g_lt_mu);
  if (load_lt()) return 0;
  return g_lt.GetVersion();
}

// Row-major y[M,N] = x[M,K] (row stride ldx) @ B, with B = w[N,K]^T (w_kn = 0,
// an nn.Linear weight, row stride ldw) or B = w[K,N] (w_kn = 1, row stride
// ldw), optional bias[N] and relu.  In cuBLASLt's column-major view that is
// D(N x M) = op(W) (N x K) @ X (K x M).
static int gemm_impl(gm_gemm g, int dtype, int w_kn, const void* x, int64_t ldx, int64_t sx, const void* w,
                     int64_t ldw, int64_t sw, const void* bias, int relu, void* y, int64_t sy, int64_t M, int64_t N,
                     int64_t K, int64_t batch, void* workspace, size_t ws_bytes, void* stream) {
  if (!g || !x || !w || !y) return gfail(GM_E_INVALID, "gm_gemm_run: null argument");
  if (M <= 0 || N <= 0 || K <= 0 || batch <= 0) return gfail(GM_E_INVALID, "gm_gemm_run: empty problem");
  const int t = lt_type(dtype);
  if (t < 0) return gfail(GM_E_INVALID, "gm_gemm_run: dtype %d", dtype);
  const int bias_on = bias != nullptr;
  Key key{dtype, M, N, K, ldx, ldw, w_kn, bias_on, relu, batch, sx, sw, sy};
  std::lock_guard<std::mutex> lk(g->mu);
  auto it = g->plans.find(key);
  if (it == g->plans.end()) {
    Plan p;
    const cublasComputeType_t compute =
        dtype == GM_F32 ? CUBLAS_COMPUTE_32F_EMULATED_16BFX9 : CUBLAS_COMPUTE_32F;
    if (g_lt.DescCreate(&p.desc, compute, CUDA_R_32F)) return gfail(GM_E_CUDA, "gm_gemm: desc create");
    const cublasOperation_t ta = w_kn ? CUBLAS_OP_N : CUBLAS_OP_T, tb = CUBLAS_OP_N;
    g_lt.DescSet(p.desc, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta));
    g_lt.DescSet(p.desc, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb));
    const cublasLtEpilogue_t epi = bias_on ? (relu ? CUBLASLT_EPILOGUE_RELU_BIAS : CUBLASLT_EPILOGUE_BIAS)
                                           : (relu ? CUBLASLT_EPILOGUE_RELU : CUBLASLT_EPILOGUE_DEFAULT);
    g_lt.DescSet(p.desc, CUBLASLT_MATMUL_DESC_EPILOGUE, &epi, sizeof(epi));
    if (bias_on) {
      const cudaDataType_t bt = (cudaDataType_t)t;
      g_lt.DescSet(p.desc, CUBLASLT_MATMUL_DESC_BIAS_DATA_TYPE, &bt, sizeof(bt));
    }
    // A = W: w_kn ? (N x K col-major = w[K,N] row-major, ld ldw) : (K x N col-major, ld ldw) then T
    const cudaDataType_t dt = (cudaDataType_t)t;
    if (w_kn)
      g_lt.LayoutCreate(&p.la, dt, N, K, ldw);
    else
      g_lt.LayoutCreate(&p.la, dt, K, N, ldw);
    g_lt.LayoutCreate(&p.lb, dt, K, M, ldx);
    g_lt.LayoutCreate(&p.lc, dt, N, M, N);
    if (batch > 1) {
      // strided batches: [batch][M][K] x [batch][K][N] -> [batch][M][N]
      const int32_t bc = (int32_t)batch;
      g_lt.LayoutSet(p.la, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &bc, sizeof(bc));
      g_lt.LayoutSet(p.la, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &sw, sizeof(sw));
      g_lt.LayoutSet(p.lb, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &bc, sizeof(bc));
      g_lt.LayoutSet(p.lb, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &sx, sizeof(sx));
      g_lt.LayoutSet(p.lc, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &bc, sizeof(bc));
      g_lt.LayoutSet(p.lc, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &sy, sizeof(sy));
    }
    cublasLtMatmulPreference_t pref;
    g_lt.PrefCreate(&pref);
    size_t cap = ws_bytes;
    g_lt.PrefSet(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &cap, sizeof(cap));
    cublasLtMatmulHeuristicResult_t res[1];
    int n = 0;
    const cublasStatus_t st = g_lt.Heuristic(g->h, p.desc, p.la, p.lb, p.lc, p.lc, pref, 1, res, &n);
    g_lt.PrefDestroy(pref);
    if (st != 0 || n == 0) {
      g_lt.DescDestroy(p.desc);
      g_lt.LayoutDestroy(p.la);
      g_lt.LayoutDestroy(p.lb);
      g_lt.LayoutDestroy(p.lc);
      return gfail(GM_E_CUDA, "gm_gemm: no cuBLASLt algorithm (status %d) for dtype %d M=%lld N=%lld K=%lld", (int)st,
                   dtype, (long long)M, (long long)N, (long long)K);
    }
    p.algo = res[0].algo;
    p.ws = res[0].workspaceSize;
    it = g->plans.emplace(key, p).first;
  }
  Plan& p = it->second;
  if (p.ws > ws_bytes) return gfail(GM_E_INVALID, "gm_gemm: workspace %zu < %zu", ws_bytes, p.ws);
  if (bias_on) g_lt.DescSet(p.desc, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &bias, sizeof(bias));
  const float alpha = 1.f, beta = 0.f;
  const cublasStatus_t st = g_lt.Matmul(g->h, p.desc, &alpha, w, p.la, x, p.lb, &beta, y, p.lc, y, p.lc, &p.algo, workspace,
                             ws_bytes, (cudaStream_t)stream);
  if (st != 0) return gfail(GM_E_CUDA, "gm_gemm: cublasLtMatmul status %d", (int)st);
  return GM_OK;
}

int gm_gemm_run(gm_gemm g, int dtype, int w_kn, const void* x, int64_t ldx, const void* w, int64_t ldw,
                const void* bias, int relu, void* y, int64_t M, int64_t N, int64_t K, void* workspace,
                size_t ws_bytes, void* stream) {
  return gemm_impl(g, dtype, w_kn, x, ldx, 0, w, ldw, 0, bias, relu, y, 0, M, N, K, 1, workspace, ws_bytes, stream);
}

int gm_gemm_run_batched(gm_gemm g, int dtype, int w_kn, const void* x, int64_t ldx, int64_t stride_x, const void* w,
                        int64_t ldw, int64_t stride_w, void* y, int64_t stride_y, int64_t M, int64_t N, int64_t K,
                        int64_t batch, void* workspace, size_t ws_bytes, void* stream) {
  return gemm_impl(g, dtype, w_kn, x, ldx, stride_x, w, ldw, stride_w, nullptr, 0, y, stride_y, M, N, K, batch,
                   workspace, ws_bytes, stream);
}

int gm_copy_strided(const void* src, void* dst, int ndim, const int64_t* sizes, const int64_t* strides,
                    int elem_bytes, void* stream) {
  if (!src || !dst || !sizes || !strides || ndim < 1 || ndim > 6 || elem_bytes <= 0)
    return gfail(GM_E_INVALID, "gm_copy_strided: bad argument");
  const int64_t inner_bytes = sizes[ndim - 1] * elem_bytes;
  if (strides[ndim - 1] != 1 || inner_bytes % 16 || ((uintptr_t)src | (uintptr_t)dst) & 15)
    return gfail(GM_E_INVALID, "gm_copy_strided: the innermost dim must be contiguous, 16-byte sized and aligned");
  CopyDesc d{};
  d.ndim = ndim;
  long long nvec = 1;
  for (int j = 0; j < ndim; ++j) {
    const int64_t sb = strides[j] * elem_bytes;
    if (j < ndim - 1 && sb % 16) return gfail(GM_E_INVALID, "gm_copy_strided: stride %d not 16-byte aligned", j);
    const long long sz = j == ndim - 1 ? inner_bytes / 16 : sizes[j];
    if (sz <= 0) return GM_OK;
    d.size[j] = (unsigned)sz;
    d.stride[j] = j == ndim - 1 ? 1 : sb / 16;
    fast_divmod(d.size[j], d.mul[j], d.shr[j]);
    nvec *= sz;
  }
  if (nvec >= (1ll << 31)) return gfail(GM_E_INVALID, "gm_copy_strided: more than 2^31 vectors");
  long long blocks = (nvec + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  gm_copy_strided_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>((const uint4*)src, (uint4*)dst, d,
                                                                          (unsigned)nvec);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return gfail(GM_E_CUDA, "gm_copy_strided: %s", cudaGetErrorString(e));
  return GM_OK;
}

int gm_select_copy(const void* pred, int pred_bytes, const void* a, const void* b, void* dst, size_t nbytes,
                   void* stream) {
  if (!pred || !a || !b || !dst || pred_bytes <= 0 || pred_bytes > 8)
    return gfail(GM_E_INVALID, "gm_select_copy: bad argument");
  if (nbytes == 0) return GM_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if ((((uintptr_t)a | (uintptr_t)b | (uintptr_t)dst | nbytes) & 15) == 0) {
    const long long nvec = (long long)(nbytes / 16);
    const int threads = 256;
    long long blocks = (nvec + threads - 1) / threads;
    if (blocks > 148 * 8) blocks = 148 * 8;
    gm_select_copy_kernel<<<(unsigned)blocks, threads, 0, s>>>((const unsigned char*)pred, pred_bytes,
                                                               (const uint4*)a, (const uint4*)b, (uint4*)dst, nvec);
  } else {
    long long blocks = ((long long)nbytes + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    gm_select_copy_tail_kernel<<<(unsigned)blocks, 256, 0, s>>>((const unsigned char*)pred, pred_bytes,
                                                                (const unsigned char*)a, (const unsigned char*)b,
                                                                (unsigned char*)dst, (long long)nbytes);
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return gfail(GM_E_CUDA, "gm_select_copy: %s", cudaGetErrorString(e));
  return GM_OK;
}

}  // extern "C"
