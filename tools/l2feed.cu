// l2feed.cu -- how fast can L2 feed the SMs' shared memory, and do shared operands help?
// (the grouped GEMMs move 9-13 TB/s of operands + stores through L2 at 7B: DESIGN.md 6.8)
//
// One CTA per SM streams CHUNK-byte blocks from an L2-resident footprint into a STAGES-deep smem
// ring with cp.async.bulk (the mainloop's TMA operand traffic, nothing else).  Modes:
//   distinct   every CTA reads its own chunks
//   same G     CTAs in groups of G (consecutive blockIdx) read the same chunk sequence (unicast:
//              does L2 deduplicate simultaneous requests for the same lines?)
//   mcast C    cluster of C CTAs: each CTA loads 1/C of the chunk with .multicast::cluster into all
//              C CTAs (every CTA still receives CHUNK bytes per step)
// Reported: delivered bytes into shared memory per second (chip) and per SM-cycle.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2feed_bin tools/l2feed.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int STAGES, int CHUNK>
__global__ void __launch_bounds__(32) k_feed(const uint8_t* src, size_t footprint, int iters, int group, int mcast,
                                             unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[STAGES], empty[STAGES];
  const uint32_t crank = mcast > 1 ? cg::this_cluster().block_rank() : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(mcast > 1 ? mcast : 1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (mcast > 1) cg::this_cluster().sync();
  __syncwarp();
  if (threadIdx.x != 0) return;
  const size_t nchunks = footprint / CHUNK;
  const int gid = mcast > 1 ? blockIdx.x / mcast : blockIdx.x / group;
  const int ngroups = mcast > 1 ? gridDim.x / mcast : gridDim.x / group;
  size_t idx = (size_t)gid * 7919;
  uint32_t fph[STAGES] = {0};
  unsigned long long acc = 0;
  const uint16_t mask = (uint16_t)((1u << (mcast > 1 ? mcast : 1)) - 1);
  auto issue = [&](int s) {
    const uint8_t* g = src + (idx % nchunks) * CHUNK;
    idx += ngroups;
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(CHUNK));
    if (mcast > 1) {
      const int part = CHUNK / mcast;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::"r"(
              su32(smem + s * CHUNK + crank * part)),
          "l"(g + crank * part), "r"(part), "r"(su32(&full[s])), "h"(mask)
          : "memory");
    } else {
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(smem + s * CHUNK)),
                   "l"(g), "r"(CHUNK), "r"(su32(&full[s]))
                   : "memory");
    }
  };
  auto wait = [&](uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(su32(b)),
                 "r"(ph));
  };
  // empty[s]: every CTA of the cluster has consumed stage s (so a multicast may overwrite it everywhere)
  uint32_t eph[STAGES] = {0};
  for (int s = 0; s < STAGES; ++s) issue(s);
  const unsigned long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int s = it % STAGES;
    wait(&full[s], fph[s]);
    fph[s] ^= 1;
    acc += smem[s * CHUNK + (it & 127)];
    if (mcast > 1) {
      for (int r = 0; r < mcast; ++r) {
        uint32_t remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(su32(&empty[s])), "r"(r));
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
      }
      wait(&empty[s], eph[s]);
      eph[s] ^= 1;
    }
    issue(s);
  }
  for (int s = 0; s < STAGES; ++s) {
    const int k = (iters + s) % STAGES;
    wait(&full[k], fph[k]);
    fph[k] ^= 1;
  }
  const unsigned long long c1 = clock64();
  if (acc == 0xFFFFFFFFull) *sink = acc;
  if (blockIdx.x == 0) sink[1] = c1 - c0;
}

#include <cuda.h>
// TMA tensor loads as the GEMMs issue them: NB boxes of {64 bf16 cols (128 B), BR rows} per stage
// (128B swizzle), one thread issuing, STAGES-deep ring -- the operand path of the TMA-fed kinds.
template <int STAGES, int BR, int NB>
__global__ void __launch_bounds__(32) k_feed_tma(const __grid_constant__ CUtensorMap map, int rows, int iters,
                                                 unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem_t[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_t) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[STAGES];
  constexpr int CH = NB * BR * 128;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  int it_row = blockIdx.x * 97;
  uint32_t ph[STAGES] = {0};
  auto issue = [&](int s) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(CH));
    for (int b = 0; b < NB; ++b) {
      const int r0 = (it_row % (rows / BR)) * BR;
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                   ::"r"(su32(sm + s * CH + b * BR * 128)), "l"(&map), "r"(su32(&full[s])), "r"(64 * (b % 24)), "r"(r0)
                   : "memory");
    }
    it_row += gridDim.x;
  };
  for (int s = 0; s < STAGES; ++s) issue(s);
  const unsigned long long c0 = clock64();
  unsigned long long acc = 0;
  for (int it = 0; it < iters; ++it) {
    const int s = it % STAGES;
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(su32(&full[s])),
                 "r"(ph[s]));
    ph[s] ^= 1;
    acc += sm[s * CH + (it & 127)];
    issue(s);
  }
  for (int s = 0; s < STAGES; ++s) {
    const int k = (iters + s) % STAGES;
    asm volatile("{\n.reg .pred p;\nW2: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n@!p bra W2;\n}\n" ::"r"(su32(&full[k])),
                 "r"(ph[k]));
    ph[k] ^= 1;
  }
  if (acc == 0xFFFFFFFFull) sink[0] = acc;
  if (blockIdx.x == 0) sink[1] = clock64() - c0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t maxfp = (size_t)2 << 30;
  uint8_t* buf;
  cudaMalloc(&buf, maxfp);
  cudaMemset(buf, 1, maxfp);
  unsigned long long* sink;
  cudaMalloc(&sink, 16);
  constexpr int STAGES = 6, CHUNK = 32768;
  auto kern = k_feed<STAGES, CHUNK>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, STAGES * CHUNK);
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  struct M { const char* name; int group, mcast; size_t fp; };
  const M modes[] = {{"distinct, 64 MB", 1, 1, 64 << 20},  {"distinct, 2 GB (HBM)", 1, 1, maxfp},
                     {"same x2", 2, 1, 64 << 20},          {"same x4", 4, 1, 64 << 20},
                     {"same x8", 8, 1, 64 << 20},          {"mcast cluster 2", 1, 2, 64 << 20},
                     {"mcast cluster 4", 1, 4, 64 << 20},  {"mcast cluster 8", 1, 8, 64 << 20},
                     {"same x2, 2 GB", 2, 1, maxfp},       {"mcast cluster 2, 2 GB", 1, 2, maxfp},
                     {"mcast cluster 4, 2 GB", 1, 4, maxfp}};
  for (const M& m : modes) {
    const int grid = (sms / 8) * 8, iters = 3000;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(32);
    cfg.dynamicSmemBytes = STAGES * CHUNK;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = m.mcast;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, (const uint8_t*)buf, m.fp, 100, m.group, m.mcast, sink);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, kern, (const uint8_t*)buf, m.fp, iters, m.group, m.mcast, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long h[2];
    cudaMemcpy(h, sink, 16, cudaMemcpyDeviceToHost);
    const double bytes = (double)grid * (iters + STAGES) * CHUNK;
    printf("%-26s grid %3d  %8.1f GB/s into smem  %6.1f B/clk/SM  (%.3f ms, %.2f GHz)  %s\n", m.name, grid,
           bytes / ms / 1e6, (double)(iters + STAGES) * CHUNK / (double)h[1], ms, h[1] / (ms * 1e6),
           cudaGetErrorString(cudaGetLastError()));
  }
  {
    // tensor-map TMA loads from an L2-resident [rows, 1536] bf16 matrix (24 column boxes of 64)
    const int cols = 1536, rows = 16384;  // 48 MB
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t es[2] = {1, 1};
#define TFEED(BR, NB)                                                                                          \
    {                                                                                                          \
      cuuint32_t box[2] = {64, BR};                                                                            \
      cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,           \
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,                         \
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);            \
      auto kt = k_feed_tma<6, BR, NB>;                                                                         \
      const int smb = 6 * NB * BR * 128 + 1024;                                                                \
      cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, smb);                              \
      const int grid = sms, iters = 3000;                                                                      \
      kt<<<grid, 32, smb>>>(map, rows, 100, sink);                                                             \
      cudaEvent_t a, b;                                                                                        \
      cudaEventCreate(&a);                                                                                     \
      cudaEventCreate(&b);                                                                                     \
      cudaEventRecord(a);                                                                                      \
      kt<<<grid, 32, smb>>>(map, rows, iters, sink);                                                           \
      cudaEventRecord(b);                                                                                      \
      cudaEventSynchronize(b);                                                                                 \
      float ms;                                                                                                \
      cudaEventElapsedTime(&ms, a, b);                                                                         \
      unsigned long long h[2];                                                                                 \
      cudaMemcpy(h, sink, 16, cudaMemcpyDeviceToHost);                                                         \
      const double bytes = (double)grid * (iters + 6) * NB * BR * 128;                                         \
      printf("TMA tensor boxes 64x%-3d x%d per stage        %8.1f GB/s into smem  %6.1f B/clk/SM  %s\n", BR, NB,  \
             bytes / ms / 1e6, (double)(iters + 6) * NB * BR * 128 / (double)h[1], cudaGetErrorString(cudaGetLastError())); \
    }
    TFEED(128, 2) TFEED(64, 4) TFEED(32, 8) TFEED(128, 1) TFEED(256, 1)
  }
  return 0;
}
