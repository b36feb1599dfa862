// ep.cu -- expert-parallel (EP) dispatch/combine primitives.
//
// Rank g owns experts [g*L, (g+1)*L), L = E/G.  A source rank routes its own tokens over all E
// experts (sonic_route), then:
//   plan     per (token, destination rank) de-duplicated send rows: one row per token per rank
//            that owns >= 1 of its kept experts, in ascending token order per rank; the row
//            carries the token's gates for that rank's L experts (0 = not routed);
//   pack     gather token rows (X forward, dO backward) into the send buffer;
//   (the caller runs the all-to-all: NCCL over NVLink, torch.distributed);
//   receive  the destination routes the received rows to its local experts with
//            SONIC_ROUTE_GIVEN and runs sonic_moe_fwd / _bwd on them -- its aggregation sums
//            its local experts per received row (destination-side pre-aggregation);
//   combine  the source sums the returned rows of each token in ascending rank order
//            (deterministic; the aggregation kernel over the plan's token CSR);
//   dS       the destination scatters its per-row dS into a dense [rows_in, L] block that is
//            returned and scattered into the source's grouped-row dS.
#include "../../include/sonic.h"
#include "sonic_internal.h"
#include "ptx.cuh"

namespace sonic {

// Per-token destination mask + per-destination token bitmap words (one block per 32 tokens).
__global__ void k_ep_mask(const int* __restrict__ rowptr, const int* __restrict__ rows,
                          const int* __restrict__ tile_expert, int T, int L, int G, int W, int* __restrict__ dmask,
                          int* __restrict__ tokcnt, uint32_t* __restrict__ bm) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  __shared__ uint32_t words[32];
  if (threadIdx.x < 32) words[threadIdx.x] = 0u;
  __syncthreads();
  const int t = blockIdx.x * 32 + threadIdx.x;
  if (t < T) {
    uint32_t mask = 0;
    for (int j = rowptr[t]; j < rowptr[t + 1]; ++j) mask |= 1u << (tile_expert[rows[j] / GEMM_M] / L);
    dmask[t] = (int)mask;
    tokcnt[t] = __popc(mask);
    for (uint32_t m = mask; m; m &= m - 1) atomicOr(&words[__ffs(m) - 1], 1u << threadIdx.x);
  }
  __syncthreads();
  if (threadIdx.x < G) bm[(size_t)threadIdx.x * W + blockIdx.x] = words[threadIdx.x];
}

__global__ void k_ep_offsets(const int* __restrict__ cnt, int G, int* __restrict__ off) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int g = 0; g < G; ++g) {
      off[g] = s;
      s += cnt[g];
    }
    off[G] = s;
  }
}

// Send-row positions, the token CSR over send rows, the row -> token map and the gates.
// One warp per token: the send rows of the token (ascending rank) get their positions, the token id
// and zeroed gate rows (lanes over the L gates), then lanes over the token's routed rows write its gates.
__global__ void k_ep_fill(const int* __restrict__ rowptr, const int* __restrict__ rows,
                          const int* __restrict__ tile_expert, const float* __restrict__ row_gate, int T, int L, int W,
                          const int* __restrict__ dmask, const uint32_t* __restrict__ bm,
                          const int* __restrict__ wprefix, const int* __restrict__ off,
                          const int* __restrict__ ep_rowptr, int* __restrict__ ep_rows, int* __restrict__ send_token,
                          float* __restrict__ send_gate) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int t = (int)((blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  const uint32_t mask = (uint32_t)dmask[t];
  const int w = t >> 5;
  const uint32_t below = (1u << (t & 31)) - 1u;
  const int j0 = ep_rowptr[t];
  int j = j0;
  for (uint32_t m = mask; m; m &= m - 1, ++j) {  // warp-uniform
    const int g = __ffs(m) - 1;
    const int pos = off[g] + wprefix[(size_t)g * W + w] + __popc(bm[(size_t)g * W + w] & below);
    if (lane == 0) {
      ep_rows[j] = pos;
      send_token[pos] = t;
    }
    for (int i = lane; i < L; i += 32) send_gate[(size_t)pos * L + i] = 0.f;
  }
  __syncwarp();
  for (int k = rowptr[t] + lane; k < rowptr[t + 1]; k += 32) {
    const int r = rows[k];
    const int e = tile_expert[r / GEMM_M];
    const int g = e / L;
    const int pos = ep_rows[j0 + __popc(mask & ((1u << g) - 1u))];
    const float gv = row_gate[r];  // a routed pair with a zero gate is sent as -0.0 (GIVEN membership)
    send_gate[(size_t)pos * L + (e - g * L)] = __float_as_uint(gv) == 0u ? -0.f : gv;
  }
}

__global__ void k_gather_rows(const __nv_bfloat16* __restrict__ src, const int* __restrict__ map,
                              const int* __restrict__ count, int d, __nv_bfloat16* __restrict__ dst) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= *count) return;
  const uint4* s = reinterpret_cast<const uint4*>(src + (size_t)map[i] * d);
  uint4* o = reinterpret_cast<uint4*>(dst + (size_t)i * d);
  for (int c = lane; c < d / 8; c += 32) o[c] = s[c];
}

// Receiver: dS of each local grouped row -> dense [rows_in, L] (pre-zeroed).
__global__ void k_ep_ds_dense(const int* __restrict__ row_token, const int* __restrict__ tile_expert,
                              const int* __restrict__ num_tiles, const float* __restrict__ dS, int L,
                              float* __restrict__ dense) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= (*num_tiles) * GEMM_M) return;
  const int t = row_token[r];
  if (t >= 0) dense[(size_t)t * L + tile_expert[r / GEMM_M]] = dS[r];
}

// Source: returned dense dS -> the source's grouped-row dS.
__global__ void k_ep_ds_scatter(const int* __restrict__ rowptr, const int* __restrict__ rows,
                                const int* __restrict__ tile_expert, int T, int L, const int* __restrict__ dmask,
                                const int* __restrict__ ep_rowptr, const int* __restrict__ ep_rows,
                                const float* __restrict__ back, float* __restrict__ dS) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const uint32_t mask = (uint32_t)dmask[t];
  for (int k = rowptr[t]; k < rowptr[t + 1]; ++k) {
    const int r = rows[k];
    const int e = tile_expert[r / GEMM_M];
    const int g = e / L;
    const int pos = ep_rows[ep_rowptr[t] + __popc(mask & ((1u << g) - 1u))];
    dS[r] = back[(size_t)pos * L + (e - g * L)];
  }
}

}  // namespace sonic

using namespace sonic;

namespace {
bool ep_ok(const sonic_moe_desc* D, int G) {
  return D && D->T >= 1 && D->E >= 1 && G >= 1 && G <= 32 && D->E % G == 0 && D->d % 64 == 0;
}
int words_of(long long T) { return (int)((T + 31) / 32); }
}  // namespace

extern "C" {

sonic_status sonic_ep_plan_sizes(const sonic_moe_desc* D, int G, size_t b[SONIC_EP_PLAN_NFIELDS]) {
  if (!ep_ok(D, G) || !b) return SONIC_ERR_INVALID_ARG;
  const size_t T = (size_t)D->T, W = (size_t)words_of(D->T), L = (size_t)(D->E / G), NS = T * (size_t)G;
  b[0] = T * 4;            // dmask
  b[1] = (size_t)G * W * 4;  // bm
  b[2] = (size_t)G * W * 4;  // wprefix
  b[3] = (size_t)G * 4;    // send_counts
  b[4] = (size_t)(G + 1) * 4;  // send_offsets
  b[5] = T * 4;            // tokcnt
  b[6] = (T + 1) * 4;      // ep_rowptr
  b[7] = NS * 4;           // ep_rows
  b[8] = NS * 4;           // send_token
  b[9] = NS * L * 4;       // send_gate
  return SONIC_OK;
}

sonic_status sonic_ep_build_plan(const sonic_moe_desc* D, int G, const sonic_routing* rt, sonic_ep_plan* p,
                                 void* stream) {
  if (!ep_ok(D, G) || !rt || !p) return SONIC_ERR_INVALID_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int T = (int)D->T, L = D->E / G, W = words_of(D->T);
  launch_k(k_ep_mask, W, 32, 0, st, rt->token_rowptr, rt->token_rows, rt->tile_expert, T, L, G, W, p->dmask, p->tokcnt,
                              p->bm);
  launch_popc(p->bm, W, G, p->wprefix, p->send_counts, st);
  launch_k(k_ep_offsets, 1, 32, 0, st, p->send_counts, G, p->send_offsets);
  launch_scan_tokens(p->tokcnt, T, p->ep_rowptr, st);
  launch_k(k_ep_fill, (unsigned)(((size_t)T * 32 + 255) / 256), 256, 0, st, rt->token_rowptr, rt->token_rows, rt->tile_expert, rt->row_gate, T, L, W,
                                            p->dmask, p->bm, p->wprefix, p->send_offsets, p->ep_rowptr, p->ep_rows,
                                            p->send_token, p->send_gate);
  set_last_launch_count(5);
  return cudaGetLastError() == cudaSuccess ? SONIC_OK : SONIC_ERR_CUDA;
}

sonic_status sonic_ep_pack(const sonic_moe_desc* D, int G, const sonic_ep_plan* p, const void* src, void* send,
                           void* stream) {
  if (!ep_ok(D, G) || !p || !src || !send) return SONIC_ERR_INVALID_ARG;
  const long long rows = D->T * G;
  launch_k(k_gather_rows, (unsigned)((rows * 32 + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream), 
      static_cast<const __nv_bfloat16*>(src), p->send_token, p->send_offsets + G, D->d,
      static_cast<__nv_bfloat16*>(send));
  set_last_launch_count(1);
  return cudaGetLastError() == cudaSuccess ? SONIC_OK : SONIC_ERR_CUDA;
}

sonic_status sonic_ep_combine(const sonic_moe_desc* D, int G, const sonic_ep_plan* p, const void* back, void* out,
                              void* stream) {
  if (!ep_ok(D, G) || !p || !back || !out) return SONIC_ERR_INVALID_ARG;
  launch_aggregate(static_cast<const __nv_bfloat16*>(back), p->ep_rowptr, p->ep_rows,
                   static_cast<__nv_bfloat16*>(out), D->T, D->d, static_cast<cudaStream_t>(stream));
  set_last_launch_count(1);
  return cudaGetLastError() == cudaSuccess ? SONIC_OK : SONIC_ERR_CUDA;
}

sonic_status sonic_ep_ds_dense(const sonic_moe_desc* local, const sonic_routing* rt, const float* dS, float* dense,
                               void* stream) {
  if (!local || !rt || !dS || !dense) return SONIC_ERR_INVALID_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const long long rows_max = sonic_rows_max(local);
  if (rows_max < 0) return SONIC_ERR_INVALID_ARG;
  cudaMemsetAsync(dense, 0, (size_t)local->T * local->E * sizeof(float), st);
  launch_k(k_ep_ds_dense, (unsigned)((rows_max + 255) / 256), 256, 0, st, rt->row_token, rt->tile_expert, rt->num_tiles,
                                                                     dS, local->E, dense);
  set_last_launch_count(1);
  return cudaGetLastError() == cudaSuccess ? SONIC_OK : SONIC_ERR_CUDA;
}

sonic_status sonic_ep_ds_scatter(const sonic_moe_desc* D, int G, const sonic_routing* rt, const sonic_ep_plan* p,
                                 const float* back, float* dS, void* stream) {
  if (!ep_ok(D, G) || !rt || !p || !back || !dS) return SONIC_ERR_INVALID_ARG;
  const int T = (int)D->T;
  launch_k(k_ep_ds_scatter, (T + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream), 
      rt->token_rowptr, rt->token_rows, rt->tile_expert, T, D->E / G, p->dmask, p->ep_rowptr, p->ep_rows, back, dS);
  set_last_launch_count(1);
  return cudaGetLastError() == cudaSuccess ? SONIC_OK : SONIC_ERR_CUDA;
}

}  // extern "C"
