// Row-gather fill-rate microbenchmark (1 CTA per SM, 6-stage ring of 16 KB stages, consumer just
// releases stages): how fast can an SM fill GEMM A-tiles (128 rows x 128 B) from randomly gathered
// rows of X [32768, 1536] bf16?  Modes: TMA 2D tile (contiguous rows, baseline), TMA gather4 from
// 1 or 4 issuing threads, cp.async 16 B from 4 warps (the current producer).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gbw tools/gather_bw.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int STAGES = 6, STAGE = 16384, ROWS = 32768, COLS = 1536;

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(su(b)),
               "r"(ph));
}
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b))); }
__device__ __forceinline__ void expect(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(tx));
}

template <int MODE>  // 0 tile, 1 gather4 x1 thread, 2 gather4 x4 threads (one per producer warp), 3 cp.async
__global__ void __launch_bounds__(160) k(const __grid_constant__ CUtensorMap mt, const __grid_constant__ CUtensorMap mg,
                                         const __nv_bfloat16* X, const int* idx, int iters, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[STAGES], empty[STAGES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fcnt = MODE == 3 ? 128 : MODE == 2 ? 4 : 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(su(&full[s])), "r"(fcnt));
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (warp < 4) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % STAGES;
      const uint32_t ph = (it / STAGES) & 1;
      wait(&empty[s], ph ^ 1);
      uint8_t* dst = sm + s * STAGE;
      // pseudo-random rows without index loads: base hashed per (CTA, stage), rows spread by a stride
      const uint32_t base = (uint32_t)(blockIdx.x * 2654435761u) ^ (uint32_t)(it * 40503u);
#define ROW(j) ((int)((base + (uint32_t)(j) * 7919u) & (ROWS - 1)))
      if (MODE == 0) {
        if (threadIdx.x == 0) {
          expect(&full[s], STAGE);
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                  su(dst)),
              "l"(&mt), "r"(su(&full[s])), "r"(0), "r"((blockIdx.x * 128 + it * 128) % (ROWS - 128))
              : "memory");
        }
      } else if (MODE == 1 || MODE == 2) {
        const bool issuer = MODE == 1 ? threadIdx.x == 0 : lane == 0;
        if (issuer) {
          const int nops = MODE == 1 ? 32 : 8, op0 = MODE == 1 ? 0 : warp * 8;
          expect(&full[s], nops * 512);
          for (int o = op0; o < op0 + nops; ++o) {
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(su(dst + o * 512)),
                "l"(&mg), "r"(su(&full[s])), "r"(0), "r"(ROW(4 * o)), "r"(ROW(4 * o + 1)), "r"(ROW(4 * o + 2)),
                "r"(ROW(4 * o + 3))
                : "memory");
          }
        }
      } else {  // cp.async: thread pt copies 16 B chunk c of rows r0 + 16 j
        const int pt = threadIdx.x, c = pt & 7, r0 = pt >> 3;
        for (int j = 0; j < 8; ++j) {
          const int r = ROW(r0 + 16 * j);
          const uint32_t d = su(dst) + (r0 + 16 * j) * 128 + ((c ^ ((r0 + 16 * j) & 7)) << 4);
          asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;" ::"r"(d), "l"(X + (size_t)r * COLS + c * 8)
                       : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su(&full[s])) : "memory");
      }
    }
  } else if (threadIdx.x == 128) {
    int acc = 0;
    for (int it = 0; it < iters; ++it) {
      const int s = it % STAGES;
      wait(&full[s], (it / STAGES) & 1);
      acc += sm[s * STAGE + (it & 1023)];
      arrive(&empty[s]);
    }
    if (acc == 123456789) *sink = acc;
  }
}

typedef CUresult (*encode_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  __nv_bfloat16* X;
  cudaMalloc(&X, (size_t)ROWS * COLS * 2);
  cudaMemset(X, 0, (size_t)ROWS * COLS * 2);
  const int iters = 4000;
  std::vector<int> h((size_t)sms * iters * 128);
  uint64_t x = 88172645463325252ull;
  for (auto& v : h) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    v = (int)(x % ROWS);
  }
  int *idx, *sink;
  cudaMalloc(&idx, h.size() * 4);
  cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&sink, 4);
  encode_t enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap mt, mg;
  cuuint64_t dims[2] = {COLS, ROWS}, str[1] = {COLS * 2};
  cuuint32_t bt[2] = {64, 128}, bg[2] = {64, 1}, es[2] = {1, 1};
  enc(&mt, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, X, dims, str, bt, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&mg, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, X, dims, str, bg, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const char* names[] = {"TMA tile (contiguous)", "TMA gather4 x1 thread", "TMA gather4 x4 threads",
                         "cp.async 16B x128 thr"};
  for (int mode = 0; mode < 4; ++mode) {
    void (*kern)(CUtensorMap, CUtensorMap, const __nv_bfloat16*, const int*, int, int*) =
        mode == 0 ? k<0> : mode == 1 ? k<1> : mode == 2 ? k<2> : k<3>;
    const int smem = STAGES * STAGE + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<sms, 160, smem>>>(mt, mg, X, idx, 200, sink);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<sms, 160, smem>>>(mt, mg, X, idx, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = (double)sms * iters * STAGE;
    printf("%-26s %8.1f GB/s  %7.1f B/clk/SM@1.9GHz  (%.3f ms) %s\n", names[mode], bytes / ms / 1e6,
           bytes / (ms * 1e-3) / sms / 1.9e9, ms, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
