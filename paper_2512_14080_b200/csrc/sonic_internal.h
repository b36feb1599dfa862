// sonic_internal.h -- declarations shared by the libsonic translation units.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

namespace sonic {

#ifndef SONIC_PDL
#define SONIC_PDL 1  // programmatic dependent launch between consecutive libsonic kernels
#endif
// Kernel launch with the programmatic-stream-serialization attribute (see ptx.cuh pdl_*).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = SONIC_PDL ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

constexpr int GEMM_M = 128;  // grouped-row tile (== TR m_tile, Q16)

struct RouteLaunch {
  long long T;
  int E, K, W, m_tile, mode, rescue, gate_raw;
  int rounding;   // mode 1 (TR): 0 NR-f, 1 up, 2 down, 3 Balance-f, 4 SR-f, 5 NR-s; mode 3 = expert choice
  uint32_t seed;  // SR-f draws
  const float* S;        // scores; with `logits` set, the S output buffer the fused softmax writes
  const float* logits;   // sonic_route_logits: router logits [T,E] (softmax fused), else null
  int* overflow;         // sonic_route_given_capped: device flag (GIVEN routing over capacity), else null
  long long cap;         //   the routed-pair capacity it guards
  // outputs
  int *topk_ids, *f, *f_r, *offsets, *pad_offsets, *row_token, *token_rowptr, *token_rows, *tile_expert,
      *num_tiles, *tile_pairs, *num_pairs;
  float *topk_s, *row_gate;
  // workspace
  uint32_t *bm_tc, *bm_kept;
  int *wprefix, *tokcnt, *flip;
  unsigned* ticket;  // last-block-done counter (zeroed by the first route kernel)
  // NR-s scratch (route mode SONIC_ROUTE_TR_NRS only)
  uint32_t *bm_dn, *bm_up;
  int *f_dn, *f_up;
  double* nrs_sums;  // [3E]: TC, floor, ceil score sums
  float* ST;
};

int launch_route(const RouteLaunch& L, cudaStream_t st);
// per-row popcount + exclusive word prefix of a [nrows, W] bitmap; counts per row
void launch_popc(const uint32_t* bm, int W, int nrows, int* wprefix, int* cnt, cudaStream_t st);
// exclusive scan of cnt[0..T) into rowptr[0..T] (single block)
void launch_scan_tokens(const int* cnt, int T, int* rowptr, cudaStream_t st);

// router backward (sonic_router_bwd)
void launch_router_bwd(const float* S, const int* rowptr, const int* rows, const int* tile_expert, const float* dS,
                       long long T, int E, int gate_raw, float* dlogits, cudaStream_t st);
// aggregation: out[t] = sum_{r in rows(t)} Y[r] (fp32 accumulation in CSR order)
void launch_aggregate(const __nv_bfloat16* Y, const int* rowptr, const int* rows, __nv_bfloat16* out, long long T,
                      int d, cudaStream_t st);
// dS[r] = sum_j part[j][r] for r < R_pad (device count), j < nparts
void launch_ds_reduce(const float* part, int nparts, long long rows_max, const int* num_tiles, float* dS,
                      cudaStream_t st);

// e4m3 quantisation (fp8.cu): per row of X [rows, cols]; per column of each W [batch, K, N]
void launch_quant_rows_e4m3(const void* X, long long rows, int cols, void* q, float* scale, cudaStream_t st);
void launch_quant_cols_e4m3(const void* W, int batch, int K, int N, void* q, float* scale, cudaStream_t st);
void launch_quant_dh_e4m3(const void* dH, long long rows_max, int cols, const int* num_tiles, const int* tile_expert,
                          const float* sw, void* q, float* scale, cudaStream_t st);

// record the number of kernels the current C-ABI call launched (sonic_last_launch_count)
void set_last_launch_count(int n);

}  // namespace sonic
