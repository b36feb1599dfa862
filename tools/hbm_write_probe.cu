// hbm_write_probe.cu -- HBM write-only bandwidth on B200 with the store paths a kernel can use
// (is ~3.87 TB/s, the torch memset rate, the real write ceiling?).
//
//   st.global.v4 (16 B per thread), st.global.v8 (32 B per thread, sm_100), st.global.cs (streaming),
//   TMA bulk store smem -> global (cp.async.bulk.global.shared::cta, 4 / 16 / 32 KB per instruction,
//   several in flight per CTA), cudaMemsetAsync; plus read-only and copy for reference.
// Each: 2 GiB buffer, grid = k x 148 CTAs, best of 10 after a warm-up, CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hbm_write_probe_bin tools/hbm_write_probe.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void st_v4(uint4* p, size_t n) {
  const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}
__global__ void st_v4_cs(uint4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p + i), "r"((unsigned)i), "r"(1u), "r"(2u), "r"(3u) : "memory");
}
__global__ void st_v8(uint4* p, size_t n32) {  // n32 = number of 32-byte chunks
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n32; i += (size_t)gridDim.x * blockDim.x)
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p + 2 * i), "r"((unsigned)i), "r"(1u), "r"(2u),
                 "r"(3u), "r"(4u), "r"(5u), "r"(6u), "r"(7u) : "memory");
}
__global__ void rd_v4(const uint4* p, size_t n, unsigned* out) {
  unsigned acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldcs(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678) out[0] = acc;
}
__global__ void cp_v4(const uint4* a, uint4* b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = __ldcs(a + i);
}
// TMA bulk store: one thread per CTA streams CH-byte chunks from a smem buffer (filled once) to global,
// keeping up to INF bulk groups in flight.
template <int CH, int INF>
__global__ void bulk_st(uint8_t* p, size_t bytes) {
  extern __shared__ __align__(128) uint8_t sm[];
  for (int i = threadIdx.x; i < CH * INF / 4; i += blockDim.x) reinterpret_cast<unsigned*>(sm)[i] = i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  const size_t nch = bytes / CH;
  int slot = 0;
  for (size_t c = blockIdx.x; c < nch; c += gridDim.x) {
    const uint32_t src = (uint32_t)__cvta_generic_to_shared(sm + slot * CH);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p + c * CH), "r"(src), "r"(CH) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(INF - 1) : "memory");
    slot = (slot + 1) % INF;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}


#include <cuda.h>
// TMA tensor (2-D tile) stores as the GEMM epilogues issue them: box {64 bf16 cols, BR rows} from a
// 128B-swizzled smem buffer into a [rows, 1536] bf16 matrix; W issuing warps per CTA, INF stores in
// flight per warp.  Tiles are dealt round robin so concurrent stores cover neighbouring rows.
template <int BR, int W, int INF>
__global__ void tma_st(const __grid_constant__ CUtensorMap map, int row_tiles, int col_tiles) {
  extern __shared__ __align__(1024) uint8_t smt[];
  uint8_t* sm = smt;
  for (int i = threadIdx.x; i < W * INF * BR * 32; i += blockDim.x) reinterpret_cast<unsigned*>(sm)[i] = i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) != 0 || w >= W) return;
  const int total = row_tiles * col_tiles;
  int slot = 0;
  for (int t = blockIdx.x * W + w; t < total; t += gridDim.x * W) {
    const int rt = t / col_tiles, ct = t - rt * col_tiles;
    const uint32_t src = (uint32_t)__cvta_generic_to_shared(sm + (size_t)(w * INF + slot) * BR * 128);
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&map),
                 "r"(src), "r"(ct * 64), "r"(rt * BR) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(INF - 1) : "memory");
    slot = (slot + 1) % INF;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <class F>
float best_ms(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  const size_t B = 2ull << 30;
  uint8_t *buf, *buf2;
  unsigned* out;
  CK(cudaMalloc(&buf, B));
  CK(cudaMalloc(&buf2, B));
  CK(cudaMalloc(&out, 64));
  CK(cudaMemset(buf2, 1, B));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto rep = [&](const char* name, float ms, double bytes) { printf("%-44s %8.3f ms  %7.0f GB/s\n", name, ms, bytes / ms / 1e6); };
  rep("cudaMemsetAsync", best_ms([&] { cudaMemsetAsync(buf, 0, B); }), B);
  for (int k : {1, 2, 4, 8}) {
    char nm[96];
    snprintf(nm, sizeof nm, "st.global.v4      grid %dx%d x 512 thr", k, sms);
    rep(nm, best_ms([&] { st_v4<<<k * sms, 512>>>((uint4*)buf, B / 16); }), B);
    snprintf(nm, sizeof nm, "st.global.cs.v4   grid %dx%d x 512 thr", k, sms);
    rep(nm, best_ms([&] { st_v4_cs<<<k * sms, 512>>>((uint4*)buf, B / 16); }), B);
    snprintf(nm, sizeof nm, "st.global.v8.b32  grid %dx%d x 512 thr", k, sms);
    rep(nm, best_ms([&] { st_v8<<<k * sms, 512>>>((uint4*)buf, B / 32); }), B);
  }
#define BULK(CH, INF, K)                                                                               \
  {                                                                                                    \
    cudaFuncSetAttribute(bulk_st<CH, INF>, cudaFuncAttributeMaxDynamicSharedMemorySize, CH * INF);     \
    char nm[96];                                                                                       \
    snprintf(nm, sizeof nm, "TMA bulk store %2d KB x %d in flight, %dx%d CTA", CH / 1024, INF, K, sms); \
    rep(nm, best_ms([&] { bulk_st<CH, INF><<<K * sms, 32, CH * INF>>>(buf, B); }), B);                 \
  }
  BULK(4096, 2, 1) BULK(4096, 8, 1) BULK(4096, 16, 1) BULK(16384, 2, 1) BULK(16384, 4, 1) BULK(16384, 8, 1)
  BULK(32768, 4, 1) BULK(16384, 4, 2) BULK(4096, 8, 4)

  {
    const int cols = 1536, rows = (int)(B / 2 / cols) & ~127;
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t es[2] = {1, 1};
#define TMAST(BR, W, INF)                                                                                         \
    {                                                                                                             \
      cuuint32_t box[2] = {64, BR};                                                                               \
      if (cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,          \
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,                       \
                                 CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) \
        printf("encode failed\n");                                                                                \
      const int sm_b = W * INF * BR * 128 + 1024;                                                                 \
      cudaFuncSetAttribute(tma_st<BR, W, INF>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_b);                \
      char nm[96];                                                                                                \
      snprintf(nm, sizeof nm, "TMA 2D store box 64x%d, %d warps x %d in flight", BR, W, INF);                    \
      rep(nm, best_ms([&] { tma_st<BR, W, INF><<<sms, 32 * W, sm_b>>>(map, rows / BR, cols / 64); }),            \
          (double)rows * cols * 2);                                                                               \
    }
    TMAST(32, 1, 2) TMAST(32, 4, 1) TMAST(32, 4, 2) TMAST(32, 4, 4) TMAST(32, 8, 2) TMAST(32, 8, 4)
    TMAST(128, 1, 2) TMAST(128, 1, 4) TMAST(128, 2, 2) TMAST(128, 4, 2) TMAST(64, 4, 2)
  }
  rep("read  ld.global.cs.v4 grid 4x148 x 512", best_ms([&] { rd_v4<<<4 * sms, 512>>>((const uint4*)buf2, B / 16, out); }), B);
  rep("copy  v4 grid 4x148 x 512 (read+write)", best_ms([&] { cp_v4<<<4 * sms, 512>>>((const uint4*)buf2, (uint4*)buf, B / 16); }), 2.0 * B);
  CK(cudaGetLastError());
  return 0;
}
