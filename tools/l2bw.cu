// L2 -> SM read bandwidth microbenchmark (bulk async copies into shared memory, 1 CTA per SM).
// Measures the ceiling that bounds the grouped GEMMs' operand traffic.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2bw tools/l2bw.cu
// usage: /tmp/l2bw  -> prints GB/s for several footprints (L2-resident ... HBM)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int STAGES, int CHUNK>
__global__ void __launch_bounds__(32) k_bulk(const uint8_t* src, size_t footprint, int iters, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[STAGES];
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s)
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  const size_t nchunks = footprint / CHUNK;
  size_t idx = (size_t)blockIdx.x * 7919;
  uint32_t phase[STAGES] = {0};
  unsigned long long acc = 0;
  auto issue = [&](int s) {
    const uint8_t* g = src + (idx % nchunks) * CHUNK;
    idx += gridDim.x;
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(CHUNK));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(smem + s * CHUNK)),
                 "l"(g), "r"(CHUNK), "r"(su32(&bar[s]))
                 : "memory");
  };
  for (int s = 0; s < STAGES; ++s) issue(s);
  for (int it = 0; it < iters; ++it) {
    const int s = it % STAGES;
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(su32(&bar[s])),
        "r"(phase[s]));
    phase[s] ^= 1;
    acc += smem[s * CHUNK + (it & 127)];
    issue(s);
  }
  for (int s = 0; s < STAGES; ++s) {  // drain
    const int k = (iters + s) % STAGES;
    asm volatile(
        "{\n.reg .pred p;\nW2: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n@!p bra W2;\n}\n" ::"r"(su32(&bar[k])),
        "r"(phase[k]));
    phase[k] ^= 1;
  }
  if (acc == 0xFFFFFFFFull) *sink = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t maxfp = (size_t)2 << 30;
  uint8_t* buf;
  cudaMalloc(&buf, maxfp);
  cudaMemset(buf, 1, maxfp);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  constexpr int STAGES = 6, CHUNK = 32768;
  auto kern = k_bulk<STAGES, CHUNK>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, STAGES * CHUNK);
  const size_t fps[] = {(size_t)8 << 20, (size_t)32 << 20, (size_t)64 << 20, (size_t)96 << 20, (size_t)512 << 20,
                        maxfp};
  for (int per_sm : {1}) {
    for (size_t fp : fps) {
      const int grid = sms * per_sm, iters = 2000;
      kern<<<grid, 32, STAGES * CHUNK>>>(buf, fp, 50, sink);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      kern<<<grid, 32, STAGES * CHUNK>>>(buf, fp, iters, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double bytes = (double)grid * (iters + STAGES) * CHUNK;
      printf("ctas/SM=%d footprint=%6zu MB  %8.1f GB/s  (%.3f ms)  %s\n", per_sm, fp >> 20, bytes / ms / 1e6, ms,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
