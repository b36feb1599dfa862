// Per-SM bandwidth of the token aggregation when it runs on a few SMs only (one 1024-thread block
// per SM, pinned there by a large dynamic smem request): how many SMs would a background dX
// aggregation need beside a GEMM that leaves them free?
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/agg_bw tools/agg_bw.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void acc8(float (&a)[8], const uint4& v) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    a[2 * i] += f.x;
    a[2 * i + 1] += f.y;
  }
}

template <int U>
__global__ void __launch_bounds__(1024) k_agg_gs(const __nv_bfloat16* __restrict__ Y, const int* __restrict__ rowptr,
                                                 const int* __restrict__ rows, __nv_bfloat16* __restrict__ out,
                                                 long long T, int d) {
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  const int nch = d >> 3;
  const uint4* Yv = reinterpret_cast<const uint4*>(Y);
  for (long long t = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < T; t += nw) {
    const int r0 = __ldg(rowptr + t), r1 = __ldg(rowptr + t + 1);
    uint4* Ov = reinterpret_cast<uint4*>(out + t * d);
    for (int c = lane; c < nch; c += 32) {
      float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      int j = r0;
      for (; j + U <= r1; j += U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ldg_stream(Yv + (long long)__ldg(rows + j + u) * nch + c);
#pragma unroll
        for (int u = 0; u < U; ++u) acc8(a, v[u]);
      }
      for (; j < r1; ++j) acc8(a, ldg_stream(Yv + (long long)__ldg(rows + j) * nch + c));
      uint4 o;
      __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int i = 0; i < 4; ++i) oh[i] = __floats2bfloat162_rn(a[2 * i], a[2 * i + 1]);
      Ov[c] = o;
    }
  }
}

int main() {
  const long long T = 32768, K = 8, d = 1536, R = T * K;
  std::vector<int> rowptr(T + 1), rows(R);
  std::mt19937 g(1);
  std::vector<int> perm(R);
  for (long long i = 0; i < R; ++i) perm[i] = (int)i;
  std::shuffle(perm.begin(), perm.end(), g);
  for (long long t = 0; t <= T; ++t) rowptr[t] = (int)(t * K);
  for (long long i = 0; i < R; ++i) rows[i] = perm[i];
  __nv_bfloat16 *Y, *O;
  int *drp, *drows;
  cudaMalloc(&Y, R * d * 2);
  cudaMalloc(&O, T * d * 2);
  cudaMalloc(&drp, (T + 1) * 4);
  cudaMalloc(&drows, R * 4);
  cudaMemset(Y, 0, R * d * 2);
  cudaMemcpy(drp, rowptr.data(), (T + 1) * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(drows, rows.data(), R * 4, cudaMemcpyHostToDevice);
  const int smem = 120 * 1024;  // one block per SM
  cudaFuncSetAttribute(k_agg_gs<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_agg_gs<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = (double)R * d * 2 + (double)T * d * 2;
  for (int U : {4, 8})
    for (int nb : {8, 12, 16, 20, 24, 32, 48, 148}) {
      auto run = [&]() {
        if (U == 4) k_agg_gs<4><<<nb, 1024, smem>>>(Y, drp, drows, O, T, (int)d);
        else k_agg_gs<8><<<nb, 1024, smem>>>(Y, drp, drows, O, T, (int)d);
      };
      run();
      cudaEventRecord(e0);
      for (int i = 0; i < 5; ++i) run();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 5;
      printf("U=%d blocks(SMs)=%3d  %8.1f us  %7.1f GB/s total  %6.1f GB/s per SM\n", U, nb, ms * 1e3,
             bytes / ms / 1e6, bytes / ms / 1e6 / nb);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
