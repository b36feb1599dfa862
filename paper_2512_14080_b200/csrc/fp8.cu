// fp8.cu -- e4m3 quantisation for the FP8 up-projection (NEXT-4; the paper's future work,
// "FP8 ... grouped GEMMs").  One fp32 scale per slice along the reduction dimension K:
//   rows:    X [T, d]      -> Xq [T, d] e4m3,       sx [T]      (per token row)
//   columns: W1 [E, d, 2n] -> W1q [E, d, 2n] e4m3,  sw [E, 2n]  (per output column of each expert)
// scale = amax / 448 in fp32 (1 where amax = 0), q = cvt.rn.satfinite.e4m3(fl32(x / scale)) --
// exactly oracle.quantize_e4m3.  W1q keeps W1's layout (MN-major B operand: valid for e4m3).
#include <algorithm>
#include <cuda_bf16.h>
#include <cuda_fp8.h>

#include "../../include/sonic.h"
#include "sonic_internal.h"
#include "ptx.cuh"

namespace sonic {

__device__ __forceinline__ uint8_t to_e4m3(float v) {
  return (uint8_t)__nv_cvt_float_to_fp8(v, __NV_SATFINITE, __NV_E4M3);
}
__device__ __forceinline__ float scale_of(float amax) { return amax > 0.f ? __fdiv_rn(amax, 448.f) : 1.f; }

// one warp per row, 16-byte chunks (8 bf16) per lane; cols % 8 == 0
__global__ void __launch_bounds__(256) k_quant_rows_e4m3(const __nv_bfloat16* __restrict__ X, long long rows, int cols,
                                                         uint8_t* __restrict__ q, float* __restrict__ scale) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int lane = threadIdx.x & 31;
  const long long r = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= rows) return;
  const uint4* src = reinterpret_cast<const uint4*>(X + r * cols);
  const int nch = cols / 8;
  float amax = 0.f;
  for (int c = lane; c < nch; c += 32) {
    const uint4 v = __ldg(src + c);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      amax = fmaxf(amax, fmaxf(fabsf(f.x), fabsf(f.y)));
    }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  const float s = scale_of(amax);
  if (lane == 0) scale[r] = s;
  uint2* dst = reinterpret_cast<uint2*>(q + r * cols);
  for (int c = lane; c < nch; c += 32) {
    const uint4 v = __ldg(src + c);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
    uint32_t w[2] = {0u, 0u};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      w[i >> 1] |= ((uint32_t)to_e4m3(__fdiv_rn(f.x, s)) | ((uint32_t)to_e4m3(__fdiv_rn(f.y, s)) << 8))
                   << (16 * (i & 1));
    }
    dst[c] = make_uint2(w[0], w[1]);
  }
}

// W [B, K, N] bf16 (N % 8 == 0), two passes over a (256-column chunk, b, K slice) grid -- enough
// blocks to keep HBM busy (one block per column chunk alone left 7B's W1 at ~2 TB/s):
//   k_amax_cols: lane c8 of each warp owns 8 consecutive columns (16-byte loads: a warp covers 512
//                contiguous bytes of a row), the 8 warps take every 8th row of the slice; the column
//                amax goes to `amax` [B, N] by atomicMax on the bits (non-negative floats order as ints;
//                amax zeroed first);
//   k_quant_cols: scale = amax / 448, then the same partition writes the e4m3 rows (8-byte stores).
constexpr int QC_KSPLIT = 16;
__global__ void __launch_bounds__(256) k_amax_cols(const __nv_bfloat16* __restrict__ W, int K, int N,
                                                   float* __restrict__ amax_out) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  __shared__ float part[8][257];
  const int b = blockIdx.y;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int col = blockIdx.x * 256 + lane * 8;
  const int kc = (K + QC_KSPLIT - 1) / QC_KSPLIT, k_lo = blockIdx.z * kc, k_hi = min(K, k_lo + kc);
  const __nv_bfloat16* w = W + (size_t)b * K * N + col;
  float amax[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) amax[i] = 0.f;
  if (col < N) {
#pragma unroll 4
    for (int k = k_lo + wp; k < k_hi; k += 8) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(w + (size_t)k * N));
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(h[i]);
        amax[2 * i] = fmaxf(amax[2 * i], fabsf(f.x));
        amax[2 * i + 1] = fmaxf(amax[2 * i + 1], fabsf(f.y));
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) part[wp][lane * 8 + i] = amax[i];
  __syncthreads();
  const int c = threadIdx.x;  // one thread per column of the chunk
  const int gc = blockIdx.x * 256 + c;
  if (gc < N) {
    float m = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) m = fmaxf(m, part[j][c]);
    atomicMax(reinterpret_cast<int*>(amax_out) + (size_t)b * N + gc, __float_as_int(m));
  }
}

__global__ void __launch_bounds__(256) k_quant_cols_e4m3(const __nv_bfloat16* __restrict__ W, int K, int N,
                                                         const float* __restrict__ amax_in, uint8_t* __restrict__ q) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int b = blockIdx.y;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int col = blockIdx.x * 256 + lane * 8;
  if (col >= N) return;
  const int kc = (K + QC_KSPLIT - 1) / QC_KSPLIT, k_lo = blockIdx.z * kc, k_hi = min(K, k_lo + kc);
  float s[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) s[i] = scale_of(amax_in[(size_t)b * N + col + i]);
  const __nv_bfloat16* w = W + (size_t)b * K * N + col;
  uint8_t* qb = q + (size_t)b * K * N + col;
#pragma unroll 4
  for (int k = k_lo + wp; k < k_hi; k += 8) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(w + (size_t)k * N));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
    uint32_t o[2] = {0u, 0u};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      o[i >> 1] |= ((uint32_t)to_e4m3(__fdiv_rn(f.x, s[2 * i])) | ((uint32_t)to_e4m3(__fdiv_rn(f.y, s[2 * i + 1])) << 8))
                   << (16 * (i & 1));
    }
    *reinterpret_cast<uint2*>(qb + (size_t)k * N) = make_uint2(o[0], o[1]);
  }
}

// FP8 dX~ operand (SONIC_F_FP8_DXT, DESIGN Q25): grouped row r of dH [rows, cols = 2n] (bf16, expert
// e = tile_expert[r / 128]) times the forward's per-column W1 scales sw[e][j] in fp32, quantised per
// row with one multiply by the reciprocal row scale -- exactly oracle.fp8_dxt_rows.  One warp per row,
// lanes over 8-column chunks (16-byte dH loads, two float4 scale loads); rows past the device-resident
// row count (num_tiles * 128) are skipped.  HBM-bound: 3 bytes per element.
__device__ __forceinline__ void scaled8(const uint4& v, const float4& s0, const float4& s1, float (&m)[8]) {
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.y));
  const float2 c = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.z));
  const float2 d = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.w));
  m[0] = __fmul_rn(a.x, s0.x); m[1] = __fmul_rn(a.y, s0.y); m[2] = __fmul_rn(b.x, s0.z); m[3] = __fmul_rn(b.y, s0.w);
  m[4] = __fmul_rn(c.x, s1.x); m[5] = __fmul_rn(c.y, s1.y); m[6] = __fmul_rn(d.x, s1.z); m[7] = __fmul_rn(d.y, s1.w);
}
__global__ void __launch_bounds__(256) k_quant_dh_e4m3(const __nv_bfloat16* __restrict__ dH, long long rows_max,
                                                       int cols, const int* __restrict__ num_tiles,
                                                       const int* __restrict__ tile_expert,
                                                       const float* __restrict__ sw, uint8_t* __restrict__ q,
                                                       float* __restrict__ scale) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int lane = threadIdx.x & 31;
  const long long r = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= rows_max || r >= (long long)(*num_tiles) * GEMM_M) return;
  const float4* swe = reinterpret_cast<const float4*>(sw + (size_t)__ldg(tile_expert + r / GEMM_M) * cols);
  const uint4* src = reinterpret_cast<const uint4*>(dH + r * cols);
  const int nch = cols / 8;
  float amax = 0.f;
  for (int c = lane; c < nch; c += 32) {
    float m[8];
    scaled8(__ldg(src + c), __ldg(swe + 2 * c), __ldg(swe + 2 * c + 1), m);
#pragma unroll
    for (int i = 0; i < 8; ++i) amax = fmaxf(amax, fabsf(m[i]));
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  const float s = scale_of(amax);
  const float rcp = __frcp_rn(s);
  if (lane == 0) scale[r] = s;
  uint2* dst = reinterpret_cast<uint2*>(q + r * cols);
  for (int c = lane; c < nch; c += 32) {  // the row's second pass hits L1 / L2
    float m[8];
    scaled8(__ldg(src + c), __ldg(swe + 2 * c), __ldg(swe + 2 * c + 1), m);
    uint32_t w[2] = {0u, 0u};
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i >> 2] |= (uint32_t)to_e4m3(__fmul_rn(m[i], rcp)) << (8 * (i & 3));
    dst[c] = make_uint2(w[0], w[1]);
  }
}

// cols <= 512 (n <= 256, the fine-grained configs): RW rows per warp held in registers across the
// amax and the quantisation, all their loads issued together -- one memory round trip per RW rows
// cols = 32 * EPL (EPL = 4, 8, 12, 16, 24, 32, 48, 64: 2n <= 2048): a warp takes blocks of QB consecutive rows (inside
// one 128-row tile, so one expert): the expert's EPL column scales per lane are loaded once per
// block; lane l holds the EPL contiguous elements [EPL l, EPL l + EPL) of a row in registers through
// both the amax and the conversion (8-byte dH loads, two values per e4m3x2 conversion, one EPL-byte
// store), with the next row's loads issued before the current row is converted.
constexpr int QB = 16;
template <int EPL>
__global__ void __launch_bounds__(256) k_quant_dh_e4m3_lane(const __nv_bfloat16* __restrict__ dH, long long rows_max,
                                                            int cols, const int* __restrict__ num_tiles,
                                                            const int* __restrict__ tile_expert,
                                                            const float* __restrict__ sw, uint8_t* __restrict__ q,
                                                            float* __restrict__ scale) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  constexpr int NV = EPL / 4;  // 8-byte dH loads (4 bf16) per lane
  const int lane = threadIdx.x & 31;
  const long long rlim = min(rows_max, (long long)(*num_tiles) * GEMM_M);
  auto load = [&](long long rr, uint2 (&w)[NV]) {
    if (rr < rlim) {
      const uint2* src = reinterpret_cast<const uint2*>(dH + rr * cols) + lane * NV;
#pragma unroll
      for (int k = 0; k < NV; ++k) w[k] = __ldg(src + k);
    }
  };
  for (long long b0 = ((long long)blockIdx.x * 8 + (threadIdx.x >> 5)) * QB; b0 < rlim;
       b0 += (long long)gridDim.x * 8 * QB) {
    const float4* s4 = reinterpret_cast<const float4*>(sw + (size_t)__ldg(tile_expert + b0 / GEMM_M) * cols) + lane * NV;
    float4 sc[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) sc[k] = __ldg(s4 + k);
    uint2 v[NV];
    load(b0, v);
    const int nrow = (int)min((long long)QB, rlim - b0);
    for (int i = 0; i < nrow; ++i) {
      const long long r = b0 + i;
      uint2 vn[NV];
      load(i + 1 < nrow ? r + 1 : rlim, vn);  // in flight while this row converts
      float m[EPL];
      float amax = 0.f;
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v[k].x));
        const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v[k].y));
        m[4 * k] = __fmul_rn(a.x, sc[k].x);
        m[4 * k + 1] = __fmul_rn(a.y, sc[k].y);
        m[4 * k + 2] = __fmul_rn(b.x, sc[k].z);
        m[4 * k + 3] = __fmul_rn(b.y, sc[k].w);
#pragma unroll
        for (int t = 0; t < 4; ++t) amax = fmaxf(amax, fabsf(m[4 * k + t]));
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      const float s = scale_of(amax);
      const float rcp = __frcp_rn(s);
      if (lane == 0) scale[r] = s;
      uint32_t w[NV];
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const uint32_t lo = __nv_cvt_float2_to_fp8x2(make_float2(__fmul_rn(m[4 * k], rcp), __fmul_rn(m[4 * k + 1], rcp)),
                                                     __NV_SATFINITE, __NV_E4M3);
        const uint32_t hi = __nv_cvt_float2_to_fp8x2(make_float2(__fmul_rn(m[4 * k + 2], rcp), __fmul_rn(m[4 * k + 3], rcp)),
                                                     __NV_SATFINITE, __NV_E4M3);
        w[k] = (lo & 0xFFFFu) | (hi << 16);
      }
      uint32_t* dst = reinterpret_cast<uint32_t*>(q + r * cols) + lane * NV;
      if constexpr (NV == 4) *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
      else if constexpr (NV == 2) *reinterpret_cast<uint2*>(dst) = make_uint2(w[0], w[1]);
      else
#pragma unroll
        for (int k = 0; k < NV; ++k) dst[k] = w[k];
#pragma unroll
      for (int k = 0; k < NV; ++k) v[k] = vn[k];
    }
  }
}

void launch_quant_dh_e4m3(const void* dH, long long rows_max, int cols, const int* num_tiles, const int* tile_expert,
                          const float* sw, void* q, float* scale, cudaStream_t st) {
  if (cols <= 2048 && cols % 128 == 0 && (cols <= 512 || cols % 512 == 0 || cols == 768 || cols == 1536)) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = (int)std::max<long long>(1, std::min<long long>(8LL * sms, (rows_max + 8 * QB - 1) / (8 * QB)));
    const __nv_bfloat16* src = static_cast<const __nv_bfloat16*>(dH);
    uint8_t* qq = static_cast<uint8_t*>(q);
    switch (cols / 32) {
      case 4: launch_k(k_quant_dh_e4m3_lane<4>, blocks, 256, 0, st, src, rows_max, cols, num_tiles, tile_expert, sw, qq, scale); return;
      case 8: launch_k(k_quant_dh_e4m3_lane<8>, blocks, 256, 0, st, src, rows_max, cols, num_tiles, tile_expert, sw, qq, scale); return;
      case 12: launch_k(k_quant_dh_e4m3_lane<12>, blocks, 256, 0, st, src, rows_max, cols, num_tiles, tile_expert, sw, qq, scale); return;
      case 16: launch_k(k_quant_dh_e4m3_lane<16>, blocks, 256, 0, st, src, rows_max, cols, num_tiles, tile_expert, sw, qq, scale); return;
      case 24: launch_k(k_quant_dh_e4m3_lane<24>, blocks, 256, 0, st, src, rows_max, cols, num_tiles, tile_expert, sw, qq, scale); return;
      case 32: launch_k(k_quant_dh_e4m3_lane<32>, blocks, 256, 0, st, src, rows_max, cols, num_tiles, tile_expert, sw, qq, scale); return;
      case 48: launch_k(k_quant_dh_e4m3_lane<48>, blocks, 256, 0, st, src, rows_max, cols, num_tiles, tile_expert, sw, qq, scale); return;
      default: launch_k(k_quant_dh_e4m3_lane<64>, blocks, 256, 0, st, src, rows_max, cols, num_tiles, tile_expert, sw, qq, scale); return;
    }
  }
  launch_k(k_quant_dh_e4m3, (int)((rows_max + 7) / 8), 256, 0, st, static_cast<const __nv_bfloat16*>(dH), rows_max,
           cols, num_tiles, tile_expert, sw, static_cast<uint8_t*>(q), scale);
}

void launch_quant_rows_e4m3(const void* X, long long rows, int cols, void* q, float* scale, cudaStream_t st) {
  launch_k(k_quant_rows_e4m3, (int)((rows + 7) / 8), 256, 0, st, static_cast<const __nv_bfloat16*>(X), rows, cols,
           static_cast<uint8_t*>(q), scale);
}
__global__ void k_amax_to_scale(float* __restrict__ v, long long n) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = scale_of(v[i]);
}

void launch_quant_cols_e4m3(const void* W, int batch, int K, int N, void* q, float* scale, cudaStream_t st) {
  // the column amax accumulates in `scale` itself (zeroed, atomicMax), the quantisation pass derives
  // each column's scale from it, and a last pass turns the amax into the scale in place
  cudaMemsetAsync(scale, 0, (size_t)batch * N * 4, st);
  const dim3 grid((N + 255) / 256, batch, QC_KSPLIT);
  launch_k(k_amax_cols, grid, 256, 0, st, static_cast<const __nv_bfloat16*>(W), K, N, scale);
  launch_k(k_quant_cols_e4m3, grid, 256, 0, st, static_cast<const __nv_bfloat16*>(W), K, N,
           static_cast<const float*>(scale), static_cast<uint8_t*>(q));
  const long long n = (long long)batch * N;
  launch_k(k_amax_to_scale, (int)((n + 255) / 256), 256, 0, st, scale, n);
}

}  // namespace sonic

extern "C" {

sonic_status sonic_quantize_e4m3_rows(const void* X, int64_t rows, int32_t cols, void* q, float* scale, void* stream) {
  if (!X || !q || !scale || rows < 0 || cols <= 0 || cols % 8 != 0) return SONIC_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(q)) & 15) return SONIC_ERR_INVALID_ARG;
  if (rows == 0) return SONIC_OK;
  sonic::launch_quant_rows_e4m3(X, rows, cols, q, scale, static_cast<cudaStream_t>(stream));
  sonic::set_last_launch_count(1);
  return cudaPeekAtLastError() == cudaSuccess ? SONIC_OK : SONIC_ERR_CUDA;
}

sonic_status sonic_quantize_e4m3_cols(const void* W, int32_t batch, int32_t K, int32_t N, void* q, float* scale,
                                      void* stream) {
  if (!W || !q || !scale || batch <= 0 || K <= 0 || N <= 0 || N % 8 != 0 || batch > 65535) return SONIC_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(W) | reinterpret_cast<uintptr_t>(q)) & 15) return SONIC_ERR_INVALID_ARG;
  sonic::launch_quant_cols_e4m3(W, batch, K, N, q, scale, static_cast<cudaStream_t>(stream));
  sonic::set_last_launch_count(3);
  return cudaPeekAtLastError() == cudaSuccess ? SONIC_OK : SONIC_ERR_CUDA;
}

}  // extern "C"
