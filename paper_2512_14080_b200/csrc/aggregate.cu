// aggregate.cu -- expert aggregation (Alg. 2 "Expert aggregation O kernel", and
// Alg. 5 "Expert aggregation dX kernel"): each token gathers its grouped rows
// and sums them (store-then-gather-sum, no atomics, deterministic; Fig. 7 left).
// The gate is already applied in the down-proj epilogue (Q2), so one unweighted kernel
// serves O and dX.  HBM-bound: reads R*d*2 B, writes T*d*2 B.
#include "sonic_internal.h"
#include "ptx.cuh"

namespace sonic {

__device__ __forceinline__ void acc8(float (&a)[8], const uint4& v) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    a[2 * i] += f.x;
    a[2 * i + 1] += f.y;
  }
}

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// One warp per token; lanes stride over 16-byte column chunks; rows summed in CSR order.
__global__ void __launch_bounds__(256) k_aggregate(const __nv_bfloat16* __restrict__ Y, const int* __restrict__ rowptr,
                                                   const int* __restrict__ rows, __nv_bfloat16* __restrict__ out,
                                                   long long T, int d) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const long long t = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  const int r0 = __ldg(rowptr + t), r1 = __ldg(rowptr + t + 1);
  const int nch = d >> 3;
  const uint4* Yv = reinterpret_cast<const uint4*>(Y);
  uint4* Ov = reinterpret_cast<uint4*>(out + t * d);
  for (int c = lane; c < nch; c += 32) {
    float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    int j = r0;
#ifndef SONIC_AGG_U
#define SONIC_AGG_U 4  // row loads in flight per lane
#endif
    for (; j + SONIC_AGG_U <= r1; j += SONIC_AGG_U) {
      uint4 v[SONIC_AGG_U];
#pragma unroll
      for (int u = 0; u < SONIC_AGG_U; ++u) {
#ifdef SONIC_EXP_AGG_SEQ  // ablation: sequential rows instead of the token's gathered rows
        const long long q = j + u;
#else
        const long long q = __ldg(rows + j + u);
#endif
        v[u] = ldg_stream(Yv + q * nch + c);
      }
#pragma unroll
      for (int u = 0; u < SONIC_AGG_U; ++u) acc8(a, v[u]);
    }
    for (; j < r1; ++j) acc8(a, ldg_stream(Yv + (long long)__ldg(rows + j) * nch + c));
    uint4 o;
    __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int i = 0; i < 4; ++i) oh[i] = __floats2bfloat162_rn(a[2 * i], a[2 * i + 1]);
    Ov[c] = o;
  }
}

__global__ void k_ds_reduce(const float* __restrict__ part, int nparts, long long rows_max,
                            const int* __restrict__ num_tiles, float* __restrict__ dS) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const long long R = (long long)(*num_tiles) * GEMM_M;
  for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += (long long)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int j = 0; j < nparts; ++j) s += part[j * rows_max + r];
    dS[r] = s;
  }
}

// Router backward (NEXT-4): warp per token.  The token's kept rows come from the CSR, the expert of
// a row from the 128-row tile map; lanes then write the E-wide d logits row.
__global__ void k_router_bwd(const float* __restrict__ S, const int* __restrict__ rowptr,
                             const int* __restrict__ rows, const int* __restrict__ tile_expert,
                             const float* __restrict__ dS, long long T, int E, int gate_raw,
                             float* __restrict__ dlogits) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const long long t = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  const float* st = S + t * E;
  const int r0 = __ldg(rowptr + t), r1 = __ldg(rowptr + t + 1);
  // pass 1 over the kept rows (lanes stride): Z = sum S, c = sum dS * S (so sum dS g = c / Z)
  float z = 0.f, c = 0.f;
  for (int j = r0 + lane; j < r1; j += 32) {
    const int r = __ldg(rows + j);
    const int e = __ldg(tile_expert + r / GEMM_M);
    const float s = __ldg(st + e);
    z += s;
    c += __ldg(dS + r) * s;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    z += __shfl_xor_sync(0xffffffffu, z, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
  // dS_full on kept experts; dot = sum S dS_full
  const float invz = (z == 0.f) ? 0.f : 1.f / z;
  const float cg = c * invz;  // sum_e dS_e g_e
  float dot = 0.f;
  for (int j = r0 + lane; j < r1; j += 32) {
    const int r = __ldg(rows + j);
    const int e = __ldg(tile_expert + r / GEMM_M);
    const float full = gate_raw ? __ldg(dS + r) : (__ldg(dS + r) - cg) * invz;
    dot += __ldg(st + e) * full;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
  float* out = dlogits + t * E;
  for (int e = lane; e < E; e += 32) out[e] = -__ldg(st + e) * dot;
  __syncwarp();
  for (int j = r0 + lane; j < r1; j += 32) {  // kept experts: S_e (dS_full_e - dot)
    const int r = __ldg(rows + j);
    const int e = __ldg(tile_expert + r / GEMM_M);
    const float full = gate_raw ? __ldg(dS + r) : (__ldg(dS + r) - cg) * invz;
    out[e] = __ldg(st + e) * (full - dot);
  }
}

void launch_router_bwd(const float* S, const int* rowptr, const int* rows, const int* tile_expert, const float* dS,
                       long long T, int E, int gate_raw, float* dlogits, cudaStream_t st) {
  const long long blocks = (T * 32 + 255) / 256;
  launch_k(k_router_bwd, (unsigned)blocks, 256, 0, st, S, rowptr, rows, tile_expert, dS, T, E, gate_raw, dlogits);
}

void launch_aggregate(const __nv_bfloat16* Y, const int* rowptr, const int* rows, __nv_bfloat16* out, long long T,
                      int d, cudaStream_t st) {
  const int threads = 256;
  const long long blocks = (T * 32 + threads - 1) / threads;
  launch_k(k_aggregate, (unsigned)blocks, threads, 0, st, Y, rowptr, rows, out, T, d);
}

void launch_ds_reduce(const float* part, int nparts, long long rows_max, const int* num_tiles, float* dS,
                      cudaStream_t st) {
  launch_k(k_ds_reduce, 148 * 4, 256, 0, st, part, nparts, rows_max, num_tiles, dS);
}

}  // namespace sonic
