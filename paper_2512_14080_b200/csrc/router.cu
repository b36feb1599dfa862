// router.cu -- the router GEMMs around the routing (NEXT-4): logits = X W_r before
// sonic_route_logits (softmax fused into the top-K, route.cu), and, after sonic_router_bwd (dS ->
// d logits), the router's contribution to the layer's input gradient dX += dlogits W_r^T and its
// weight gradient dW_r = X^T dlogits.
//
// These are plain dense GEMMs of a small N (E <= 4096): cuBLAS (cublasGemmEx, bf16 operands, fp32
// accumulation), loaded with dlopen at first use so that libsonic does not depend on it otherwise.
// d logits are fp32; the tensor-core GEMMs take them rounded to bf16 (k_f32_to_bf16 into the caller's
// workspace), the same operand precision as every other GEMM of the layer.
#include <dlfcn.h>
#include <cublas_v2.h>
#include <cuda_bf16.h>

#include "../../include/sonic.h"
#include "sonic_internal.h"
#include "ptx.cuh"

namespace {

struct Cublas {
  bool tried = false, ok = false;
  decltype(&cublasCreate_v2) create = nullptr;
  decltype(&cublasSetStream_v2) set_stream = nullptr;
  // cublasGemmEx is overloaded in C++ (cudaDataType / cublasComputeType_t compute argument): the C symbol's type
  using GemmExFn = cublasStatus_t (*)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int, int,
                                      const void*, const void*, cudaDataType, int, const void*, cudaDataType, int,
                                      const void*, void*, cudaDataType, int, cublasComputeType_t, cublasGemmAlgo_t);
  GemmExFn gemm = nullptr;
  cublasHandle_t h[64] = {};
};

Cublas& cublas() {
  static Cublas c;
  if (!c.tried) {
    c.tried = true;
    void* so = dlopen("libcublas.so.12", RTLD_NOW | RTLD_GLOBAL);
    if (!so) so = dlopen("libcublas.so", RTLD_NOW | RTLD_GLOBAL);
    if (so) {
      c.create = reinterpret_cast<decltype(c.create)>(dlsym(so, "cublasCreate_v2"));
      c.set_stream = reinterpret_cast<decltype(c.set_stream)>(dlsym(so, "cublasSetStream_v2"));
      c.gemm = reinterpret_cast<decltype(c.gemm)>(dlsym(so, "cublasGemmEx"));
      c.ok = c.create && c.set_stream && c.gemm;
    }
  }
  return c;
}

// the per-device handle, bound to `st`
cublasHandle_t handle_on(cudaStream_t st) {
  Cublas& c = cublas();
  if (!c.ok) return nullptr;
  int dev = 0;
  cudaGetDevice(&dev);
  cublasHandle_t& h = c.h[dev & 63];
  if (!h && c.create(&h) != CUBLAS_STATUS_SUCCESS) {
    h = nullptr;
    return nullptr;
  }
  if (c.set_stream(h, st) != CUBLAS_STATUS_SUCCESS) return nullptr;
  return h;
}

__global__ void k_f32_to_bf16(const float* __restrict__ in, __nv_bfloat16* __restrict__ out, long long n) {
  const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i + 3 < n) {
    const float4 v = *reinterpret_cast<const float4*>(in + i);
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    *reinterpret_cast<__nv_bfloat162*>(out + i) = a;
    *reinterpret_cast<__nv_bfloat162*>(out + i + 2) = b;
  } else {
    for (long long j = i; j < n; ++j) out[j] = __float2bfloat16_rn(in[j]);
  }
}

bool desc_ok(const sonic_moe_desc* D) {
  return D && D->T > 0 && D->d > 0 && D->E > 0 && D->E <= 4096 && D->T <= (1ll << 31) - 1;
}
bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

extern "C" {

sonic_status sonic_router_fwd(const sonic_moe_desc* D, const void* X, const void* Wr, float* logits, void* stream) {
  sonic::set_last_launch_count(0);
  if (!desc_ok(D) || !X || !Wr || !logits) return SONIC_ERR_INVALID_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cublasHandle_t h = handle_on(st);
  if (!h) return SONIC_ERR_UNSUPPORTED;
  const int T = (int)D->T, d = D->d, E = D->E;
  const float one = 1.f, zero = 0.f;
  // row-major logits[T,E] = X[T,d] Wr[d,E]  <=>  column-major logits^T[E,T] = Wr^T[E,d] X^T[d,T]
  const cublasStatus_t s = cublas().gemm(h, CUBLAS_OP_N, CUBLAS_OP_N, E, T, d, &one, Wr, CUDA_R_16BF, E, X,
                                         CUDA_R_16BF, d, &zero, logits, CUDA_R_32F, E, CUBLAS_COMPUTE_32F,
                                         CUBLAS_GEMM_DEFAULT);
  return s == CUBLAS_STATUS_SUCCESS ? SONIC_OK : SONIC_ERR_CUDA;
}

size_t sonic_router_grad_workspace_size(const sonic_moe_desc* D) {
  if (!desc_ok(D)) return 0;
  return ((size_t)D->T * D->E * 2 + 255) / 256 * 256;  // d logits as bf16
}

sonic_status sonic_router_grad(const sonic_moe_desc* D, const void* X, const void* Wr, const float* dlogits,
                               void* dX, float* dWr, void* ws, size_t ws_bytes, void* stream) {
  sonic::set_last_launch_count(0);
  if (!desc_ok(D) || !X || !Wr || !dlogits || (!dX && !dWr)) return SONIC_ERR_INVALID_ARG;
  if (!al16(dlogits) || !al16(ws)) return SONIC_ERR_INVALID_ARG;
  if (!ws || ws_bytes < sonic_router_grad_workspace_size(D)) return SONIC_ERR_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cublasHandle_t h = handle_on(st);
  if (!h) return SONIC_ERR_UNSUPPORTED;
  const int T = (int)D->T, d = D->d, E = D->E;
  const long long n = (long long)T * E;
  __nv_bfloat16* dl = static_cast<__nv_bfloat16*>(ws);
  k_f32_to_bf16<<<(unsigned)((n / 4 + 255) / 256 + 1), 256, 0, st>>>(dlogits, dl, n);
  if (cudaPeekAtLastError() != cudaSuccess) return SONIC_ERR_CUDA;
  sonic::set_last_launch_count(1);
  const float one = 1.f, zero = 0.f;
  if (dX) {
    // row-major dX[T,d] += dl[T,E] Wr^T[E,d]  <=>  column-major dX^T[d,T] += Wr[d,E] dl^T[E,T];
    // Wr row-major [d,E] is column-major [E,d] (ld E): op T gives Wr
    if (cublas().gemm(h, CUBLAS_OP_T, CUBLAS_OP_N, d, T, E, &one, Wr, CUDA_R_16BF, E, dl, CUDA_R_16BF, E, &one, dX,
                      CUDA_R_16BF, d, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT) != CUBLAS_STATUS_SUCCESS)
      return SONIC_ERR_CUDA;
  }
  if (dWr) {
    // row-major dWr[d,E] = X^T[d,T] dl[T,E]  <=>  column-major dWr^T[E,d] = dl^T[E,T] X[T,d];
    // X row-major [T,d] is column-major [d,T] (ld d): op T gives X
    if (cublas().gemm(h, CUBLAS_OP_N, CUBLAS_OP_T, E, d, T, &one, dl, CUDA_R_16BF, E, X, CUDA_R_16BF, d, &zero, dWr,
                      CUDA_R_32F, E, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT) != CUBLAS_STATUS_SUCCESS)
      return SONIC_ERR_CUDA;
  }
  return cudaPeekAtLastError() == cudaSuccess ? SONIC_OK : SONIC_ERR_CUDA;
}

}  // extern "C"
