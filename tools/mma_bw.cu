// tcgen05 MMA issue-rate microbenchmark with optional shared-memory interference.
// One CTA per SM, operands resident in SMEM (one 64-K stage, SWIZZLE_128B), the MMA warp issues
// back-to-back kind::f16 M=128 x N=256 x K=16 MMAs (4 per 64-K stage) into TMEM.  A second warp
// optionally loads SMEM bandwidth at the same time:
//   mode 0: nothing; 1: TMA 2D loads (32 KB boxes, 2 in flight) from an L2-resident buffer;
//   2: st.shared.v4 stream (one warp); 3: ld.shared.v4 stream (one warp).
// Tells how much of the tensor-pipe rate survives when SMEM also serves fills / epilogue traffic.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2512_14080_b200/csrc \
//        -o /tmp/mma_bw tools/mma_bw.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include "ptx.cuh"

using namespace sonic;

constexpr int ITERS = 20000;  // 64-K stages

template <int MODE, int MN>
__global__ void __launch_bounds__(128) k_mma(const __grid_constant__ CUtensorMap mt, const __grid_constant__ CUtensorMap ms,
                                             unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  // 3 operand stages of (A 16 KB + B 32 KB), rotated so no stage is re-read back to back
  uint8_t* sA = sm;
  uint8_t* sB = sm + 16384;
  uint8_t* sF = sm + 3 * 49152;   // 64 KB filler region
  __shared__ uint64_t done_bar, fbar[2];
  __shared__ uint32_t tmem_holder;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&done_bar, 1);
    ptx::mbar_init(&fbar[0], 1);
    ptx::mbar_init(&fbar[1], 1);
    ptx::fence_barrier_init();
    stop = 0;
  }
  for (int i = threadIdx.x; i < 3 * 49152 / 16; i += 128) ptx::st_shared_v4(ptx::smem_u32(sm) + 16 * i, 0, 0, 0, 0);
  if (warp == 0) {
    ptx::tmem_alloc(&tmem_holder, 512);
    ptx::tmem_relinquish();
  }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_holder;
  if (warp == 0) {
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::make_idesc(128, 256, MN, MN);
      const unsigned long long t0 = clock64();
      for (int it = 0; it < ITERS; ++it) {
        const uint32_t a = ptx::smem_u32(sA) + (it % 3) * 49152, b = ptx::smem_u32(sB) + (it % 3) * 49152;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t ad = MN ? ptx::make_sdesc(a + k * 2048, 8192, 1024) : ptx::make_sdesc(a + k * 32, 16, 1024);
          const uint64_t bd = MN ? ptx::make_sdesc(b + k * 2048, 8192, 1024) : ptx::make_sdesc(b + k * 32, 16, 1024);
          ptx::mma_bf16(tmem + (it & 1) * 256, ad, bd, idesc, (it > 1 || k > 0) ? 1u : 0u);
        }
      }
      ptx::mma_commit(&done_bar);
      ptx::mbar_wait(&done_bar, 0);
      const unsigned long long t1 = clock64();
      cycles[blockIdx.x] = t1 - t0;
      stop = 1;
    }
    __syncwarp();
  } else if (warp == 1) {
    if (MODE == 1) {
      if (lane == 0) {
        uint32_t ph[2] = {0, 0};
        for (int s = 0; s < 2; ++s) {
          ptx::mbar_arrive_expect_tx(&fbar[s], 32768);
          ptx::tma_load_2d(sF + s * 32768, &mt, &fbar[s], 0, (blockIdx.x * 256 + s * 256) & 4095);
        }
        for (int it = 0; !stop; ++it) {
          const int s = it & 1;
          ptx::mbar_wait(&fbar[s], ph[s]);
          ph[s] ^= 1;
          ptx::mbar_arrive_expect_tx(&fbar[s], 32768);
          ptx::tma_load_2d(sF + s * 32768, &mt, &fbar[s], 0, (blockIdx.x * 256 + it * 256) & 4095);
        }
        for (int s = 0; s < 2; ++s) ptx::mbar_wait(&fbar[s], ph[s]);
      }
    } else if (MODE == 2) {
      const uint32_t f = ptx::smem_u32(sF);
      for (int it = 0; !stop; ++it)
#pragma unroll
        for (int j = 0; j < 16; ++j) ptx::st_shared_v4(f + ((it * 16 + j) & 127) * 512 + lane * 16, it, j, lane, 0);
    } else if (MODE == 4) {  // TMA stores of 4 KB boxes from the filler region, 4 groups in flight
      if (lane == 0) {
        for (int it = 0; !stop; ++it) {
          ptx::tma_store_2d(&ms, sF + (it & 15) * 4096, 0, (blockIdx.x * 64 + (it & 63) * 32) & 8191);
          ptx::bulk_commit();
          ptx::bulk_wait_read<4>();
        }
        ptx::bulk_wait<0>();
      }
    } else if (MODE == 3) {
      const uint32_t f = ptx::smem_u32(sF);
      uint32_t acc = 0;
      for (int it = 0; !stop; ++it)
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint4 v = ptx::ld_shared_v4(f + ((it * 16 + j) & 127) * 512 + lane * 16);
          acc += v.x ^ v.w;
        }
      if (acc == 0x12345678u) cycles[gridDim.x] = acc;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

typedef CUresult (*encode_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int MODE, int MN>
void run(const CUtensorMap& mt, const CUtensorMap& ms, unsigned long long* d_cyc, int sms, const char* name) {
  auto kern = k_mma<MODE, MN>;
  const int smem = 3 * 49152 + 65536 + 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kern<<<sms, 128, smem>>>(mt, ms, d_cyc);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<<<sms, 128, smem>>>(mt, ms, d_cyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float el;
  cudaEventElapsedTime(&el, a, b);
  unsigned long long cyc[1024];
  cudaMemcpy(cyc, d_cyc, sms * 8, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < sms; ++i) mx = cyc[i] > mx ? cyc[i] : mx;
  const double flops = 2.0 * 128 * 256 * 64 * (double)ITERS * sms;
  printf("%-34s %7.1f TFLOPS  %6.0f MAC/clk/SM  (%.3f ms) %s\n", name, flops / el / 1e9,
         128.0 * 256 * 64 * ITERS / mx, el, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void* buf;
  cudaMalloc(&buf, 4096 * 128 * 2);
  cudaMemset(buf, 0, 4096 * 128 * 2);
  unsigned long long* d_cyc;
  cudaMalloc(&d_cyc, 1025 * 8);
  encode_t enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap mt, ms;
  cuuint64_t dims[2] = {64, 4096 * 2}, str[1] = {128};
  cuuint32_t box[2] = {64, 256}, es[2] = {1, 1};
  enc(&mt, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint32_t box2[2] = {64, 32};
  enc(&ms, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  run<0, 0>(mt, ms, d_cyc, sms, "K-major, no interference");
  run<0, 1>(mt, ms, d_cyc, sms, "MN-major, no interference");
  run<1, 0>(mt, ms, d_cyc, sms, "K-major + TMA loads (max rate)");
  run<2, 0>(mt, ms, d_cyc, sms, "K-major + st.shared stream");
  run<3, 0>(mt, ms, d_cyc, sms, "K-major + ld.shared stream");
  run<1, 1>(mt, ms, d_cyc, sms, "MN-major + TMA loads (max rate)");
  run<4, 0>(mt, ms, d_cyc, sms, "K-major + TMA stores (4 KB, max)");
  return 0;
}
