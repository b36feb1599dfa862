// gemm.cuh -- the six grouped GEMMs of the SonicMoE layer as ONE warp-specialised,
// persistent tcgen05/TMEM/TMA kernel template for sm_100a.
//
//   kind   paper kernel (Alg.)          D = A . B per expert e                 epilogue
//   UP     up-proj A kernel (Alg. 2)    H_e   = Gather(X) W1_e       (varlen-M) SwiGLU -> H, A
//   DOWN   down-proj Y kernel (Alg. 2)  Y_e   = A_e W2_e             (varlen-M) x gate -> Y (Q2)
//   DH     dH kernel (Alg. 3)           dA'_e = Gather(dO) W2_e^T    (varlen-M) dSwiGLU, A', dS
//   DXT    dX~ kernel (Alg. 5)          dX~_e = dH_e W1_e^T          (varlen-M) -> dX~
//   DW2    dW2 kernel (Alg. 3)          dW2_e = A'_e^T Gather(dO)    (varlen-K) fp32 store
//   DW1    dW1 kernel (Alg. 5)          dW1_e = Gather(X)^T dH_e     (varlen-K) fp32 store
//
// Roles (192 threads, 1 CTA per SM):
//   warp 0     TMA producer: tile / 3-D tile / gather4 loads into a STAGES-deep smem ring
//              (full/empty mbarriers).  Gathered rows come from row_token (the gather
//              map) -- the paper's "gather fused with the HBM load" (sec. 4.1.1)
//              done with TMA gather4 instead of cp.async + relay warp.
//   warp 1     TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, K=16 steps),
//              two TMEM accumulator stages so the epilogue of tile i overlaps the MMA of
//              tile i+1.
//   warps 2-5  epilogue: tcgen05.ld -> registers -> fused math -> swizzled smem -> TMA store
//              ("asynchronous TMA store in all Grouped GEMMs").
// Operand smem layout: 128B-swizzled, K-major (rows of 64 K-elements) or MN-major
// (64-element MN chunks x 64 K-rows); every stage is one A tile (128 x 64) + one B tile
// (BN x 64).
#pragma once
#include "ptx.cuh"

namespace sonic {

enum GemmKind { K_UP = 0, K_DOWN = 1, K_DH = 2, K_DXT = 3, K_DW2 = 4, K_DW1 = 5 };

struct GemmArgs {
  const int* num_m_tiles;   // varlen-M: device-resident count of 128-row tiles (R_pad / 128)
  const int* tile_expert;   // varlen-M: expert of each 128-row tile
  const int* row_token;     // gather map, -1 on pad rows
  const float* row_gate;    // gate per grouped row, 0 on pad rows
  const int* pad_offsets;   // [E+1] tile-aligned expert segments
  int E;
  int n_tiles;              // output tiles along N
  int m_tiles;              // varlen-K: output tiles along M per expert
  int k_blocks;             // varlen-M: ceil(K / 64)
  int n;                    // expert intermediate dim (offset of the "up" half of H)
  int M_dim, N_dim;         // output extent along M (varlen-K) and N
  const __nv_bfloat16* H;   // DH: cached H [rows, 2n]
  float* dS;                // DH: dS [rows] if n_tiles == 1, else partials [n_tiles][rows_max]
  long long rows_max;
};

template <int KIND>
struct Traits;
template <> struct Traits<K_UP>   { static constexpr bool vk = false, a_gather = true,  a_mn = false, b_gather = false, b_mn = true;  };
template <> struct Traits<K_DOWN> { static constexpr bool vk = false, a_gather = false, a_mn = false, b_gather = false, b_mn = true;  };
template <> struct Traits<K_DH>   { static constexpr bool vk = false, a_gather = true,  a_mn = false, b_gather = false, b_mn = false; };
template <> struct Traits<K_DXT>  { static constexpr bool vk = false, a_gather = false, a_mn = false, b_gather = false, b_mn = false; };
template <> struct Traits<K_DW2>  { static constexpr bool vk = true,  a_gather = false, a_mn = true,  b_gather = true,  b_mn = true;  };
template <> struct Traits<K_DW1>  { static constexpr bool vk = true,  a_gather = true,  a_mn = true,  b_gather = false, b_mn = true;  };

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;
constexpr int GEMM_THREADS = 192;
constexpr int STG_BYTES = 4096;  // one epilogue staging buffer: 32 rows x 128 B
constexpr int SMEM_LIMIT = 232448;

template <int BN>
struct GemmCfg {
  static constexpr uint32_t A_BYTES = GEMM_BM * GEMM_BK * 2;
  static constexpr uint32_t B_BYTES = BN * GEMM_BK * 2;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int FIXED = 4 * 2 * STG_BYTES + 1024 + 256;
  static constexpr int STAGES_RAW = (SMEM_LIMIT - FIXED) / (int)STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int SMEM = STAGES * STAGE_BYTES + FIXED;
  static constexpr uint32_t TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                        : (2 * BN <= 256) ? 256 : 512;
};

struct TileCoord {
  int e, row0, nt, mt, nkb, seg0;
};

template <int KIND, int BN>
__device__ __forceinline__ TileCoord decode_tile(const GemmArgs& a, int tile) {
  TileCoord c;
  if constexpr (Traits<KIND>::vk) {
    int per_e = a.m_tiles * a.n_tiles;
    c.e = tile / per_e;
    int rem = tile - c.e * per_e;
    c.mt = rem / a.n_tiles;
    c.nt = rem - c.mt * a.n_tiles;
    c.seg0 = __ldg(a.pad_offsets + c.e);
    c.nkb = (__ldg(a.pad_offsets + c.e + 1) - c.seg0) / GEMM_BK;
    c.row0 = 0;
  } else {
    int m = tile / a.n_tiles;
    c.nt = tile - m * a.n_tiles;
    c.mt = m;
    c.row0 = m * GEMM_BM;
    c.e = __ldg(a.tile_expert + m);
    c.nkb = a.k_blocks;
    c.seg0 = 0;
  }
  return c;
}

__device__ __forceinline__ int4 load_idx4(const int* p) {
  int4 v = __ldg(reinterpret_cast<const int4*>(p));
  // pad rows (-1) read token 0; their gate is 0, so every value they produce is exactly 0
  v.x = max(v.x, 0); v.y = max(v.y, 0); v.z = max(v.z, 0); v.w = max(v.w, 0);
  return v;
}

// Write one 32-row x 128-byte slab (thread = row) into a 128B-swizzled staging buffer.
__device__ __forceinline__ void stage_row_bf16(uint8_t* buf, int lane, const float* v) {
  uint32_t base = ptx::smem_u32(buf) + lane * 128;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    ptx::st_shared_v4(base + ((c ^ (lane & 7)) << 4), ptx::pack_bf16(v[8 * c + 0], v[8 * c + 1]),
                      ptx::pack_bf16(v[8 * c + 2], v[8 * c + 3]), ptx::pack_bf16(v[8 * c + 4], v[8 * c + 5]),
                      ptx::pack_bf16(v[8 * c + 6], v[8 * c + 7]));
  }
}
__device__ __forceinline__ void stage_row_f32(uint8_t* buf, int lane, const float* v) {
  uint32_t base = ptx::smem_u32(buf) + lane * 128;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    ptx::st_shared_v4(base + ((c ^ (lane & 7)) << 4), __float_as_uint(v[4 * c + 0]), __float_as_uint(v[4 * c + 1]),
                      __float_as_uint(v[4 * c + 2]), __float_as_uint(v[4 * c + 3]));
  }
}

// Per-warp double-buffered TMA store pipeline.
struct StoreQ {
  uint8_t* buf;  // 2 x STG_BYTES
  int sb;
  __device__ __forceinline__ uint8_t* acquire(int lane) {
    if (lane == 0) ptx::bulk_wait_read<1>();
    __syncwarp();
    return buf + sb * STG_BYTES;
  }
  __device__ __forceinline__ void commit2d(int lane, const CUtensorMap* map, int c0, int c1) {
    ptx::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      ptx::tma_store_2d(map, buf + sb * STG_BYTES, c0, c1);
      ptx::bulk_commit();
    }
    sb ^= 1;
  }
  __device__ __forceinline__ void commit3d(int lane, const CUtensorMap* map, int c0, int c1, int c2) {
    ptx::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      ptx::tma_store_3d(map, buf + sb * STG_BYTES, c0, c1, c2);
      ptx::bulk_commit();
    }
    sb ^= 1;
  }
};

__device__ __forceinline__ float bf16r(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }
__device__ __forceinline__ float sigmoidf_fast(float x) { return 1.0f / (1.0f + __expf(-x)); }

template <int KIND, int BN>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    sonic_gemm_kernel(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB,
                      const __grid_constant__ CUtensorMap mC0, const __grid_constant__ CUtensorMap mC1,
                      const GemmArgs args) {
  using Tr = Traits<KIND>;
  using Cfg = GemmCfg<BN>;
  constexpr int STAGES = Cfg::STAGES;
  constexpr uint32_t A_BYTES = Cfg::A_BYTES;
  constexpr uint32_t STAGE_BYTES = Cfg::STAGE_BYTES;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stg = smem + STAGES * STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + 4 * 2 * STG_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], 4);
    }
    ptx::fence_barrier_init();
    ptx::prefetch_tmap(&mA);
    ptx::prefetch_tmap(&mB);
  }
  if (warp == 1) {
    ptx::tmem_alloc(tmem_holder, Cfg::TMEM_COLS);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  const int total_tiles = Tr::vk ? args.E * args.m_tiles * args.n_tiles : (*args.num_m_tiles) * args.n_tiles;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
      const TileCoord tc = decode_tile<KIND, BN>(args, tile);
      int4 aidx = make_int4(0, 0, 0, 0);
      if constexpr (!Tr::vk && Tr::a_gather) aidx = load_idx4(args.row_token + tc.row0 + 4 * lane);
      for (int kb = 0; kb < tc.nkb; ++kb) {
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sA = smem + stage * STAGE_BYTES;
        uint8_t* sB = sA + A_BYTES;
        uint64_t* bar = &full[stage];
        if (lane == 0) ptx::mbar_arrive_expect_tx(bar, STAGE_BYTES);
        __syncwarp();
        if constexpr (!Tr::vk) {
          // ---- A: 128 grouped rows x 64 K
          if constexpr (Tr::a_gather) {
            ptx::tma_gather4(sA + lane * 512, &mA, bar, kb * GEMM_BK, aidx.x, aidx.y, aidx.z, aidx.w);
          } else if (lane == 0) {
            ptx::tma_load_2d(sA, &mA, bar, kb * GEMM_BK, tc.row0);
          }
          // ---- B: weights of expert e (3-D tensor map [E, rows, cols])
          if (lane == 0) {
            if constexpr (KIND == K_UP) {
              constexpr int W = BN / 2;  // gate columns per tile; the up columns follow at +n
              if constexpr (W >= 64) {
                const int j0 = tc.nt * W;
#pragma unroll
                for (int j = 0; j < W / 64; ++j) {
                  ptx::tma_load_3d(sB + j * 8192, &mB, bar, j0 + 64 * j, kb * GEMM_BK, tc.e);
                  ptx::tma_load_3d(sB + (W / 64 + j) * 8192, &mB, bar, args.n + j0 + 64 * j, kb * GEMM_BK, tc.e);
                }
              } else {  // n == 32: one 64-column box holds [gate | up]
                ptx::tma_load_3d(sB, &mB, bar, 0, kb * GEMM_BK, tc.e);
              }
            } else if constexpr (KIND == K_DOWN) {
#pragma unroll
              for (int j = 0; j < BN / 64; ++j)
                ptx::tma_load_3d(sB + j * 8192, &mB, bar, tc.nt * BN + 64 * j, kb * GEMM_BK, tc.e);
            } else {  // DH, DXT: K-major weights, one box of BN rows
              ptx::tma_load_3d(sB, &mB, bar, kb * GEMM_BK, tc.nt * BN, tc.e);
            }
          }
        } else {
          const int krow0 = tc.seg0 + kb * GEMM_BK;
          const int g = lane & 15;
          int4 kidx = make_int4(0, 0, 0, 0);
          if constexpr (Tr::a_gather || Tr::b_gather) kidx = load_idx4(args.row_token + krow0 + 4 * g);
          // ---- A (MN-major): 64 K-rows x 128 M-columns
          if constexpr (Tr::a_gather) {
            const int j = lane >> 4;
            ptx::tma_gather4(sA + j * 8192 + g * 512, &mA, bar, tc.mt * GEMM_BM + 64 * j, kidx.x, kidx.y, kidx.z,
                             kidx.w);
          } else if (lane == 0) {
            ptx::tma_load_2d(sA, &mA, bar, tc.mt * GEMM_BM, krow0);
            ptx::tma_load_2d(sA + 8192, &mA, bar, tc.mt * GEMM_BM + 64, krow0);
          }
          // ---- B (MN-major): 64 K-rows x BN N-columns
          if constexpr (Tr::b_gather) {
            for (int it = lane; it < (BN / 64) * 16; it += 32) {
              const int j = it >> 4;
              ptx::tma_gather4(sB + j * 8192 + g * 512, &mB, bar, tc.nt * BN + 64 * j, kidx.x, kidx.y, kidx.z,
                               kidx.w);
            }
          } else if (lane == 0) {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) ptx::tma_load_2d(sB + j * 8192, &mB, bar, tc.nt * BN + 64 * j, krow0);
          }
        }
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::make_idesc(GEMM_BM, BN, Tr::a_mn ? 1 : 0, Tr::b_mn ? 1 : 0);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
        const TileCoord tc = decode_tile<KIND, BN>(args, tile);
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < tc.nkb; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a_base = ptx::smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t b_base = a_base + A_BYTES;
#pragma unroll
          for (int k = 0; k < GEMM_BK / 16; ++k) {
            const uint64_t ad = Tr::a_mn ? ptx::make_sdesc(a_base + k * 2048, 8192, 1024)
                                         : ptx::make_sdesc(a_base + k * 32, 16, 1024);
            const uint64_t bd = Tr::b_mn ? ptx::make_sdesc(b_base + k * 2048, 8192, 1024)
                                         : ptx::make_sdesc(b_base + k * 32, 16, 1024);
            ptx::mma_bf16(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          ptx::mma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        ptx::mma_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..5)
    const int ew = warp - 2;
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    StoreQ sq{stg + ew * 2 * STG_BYTES, 0};
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
      const TileCoord tc = decode_tile<KIND, BN>(args, tile);
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const uint32_t t_acc = tmem_base + ((uint32_t)(32 * q) << 16) + acc * BN;
      const int wrow = tc.row0 + 32 * q;  // first grouped row of this warp's slab
      const int row = wrow + lane;        // this thread's grouped row (varlen-M)

      if constexpr (KIND == K_UP) {
        constexpr int W = BN / 2;
        if constexpr (W >= 64) {
#pragma unroll 1
          for (int c = 0; c < W; c += 64) {
            uint32_t g0[32], g1[32], u0[32], u1[32];
            ptx::tmem_ld32(t_acc + c, g0);
            ptx::tmem_ld32(t_acc + c + 32, g1);
            ptx::tmem_ld32(t_acc + W + c, u0);
            ptx::tmem_ld32(t_acc + W + c + 32, u1);
            ptx::tmem_ld_wait();
            float hg[64], hu[64];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              hg[j] = bf16r(__uint_as_float(g0[j]));
              hg[32 + j] = bf16r(__uint_as_float(g1[j]));
              hu[j] = bf16r(__uint_as_float(u0[j]));
              hu[32 + j] = bf16r(__uint_as_float(u1[j]));
            }
            const int col = tc.nt * W + c;
            stage_row_bf16(sq.acquire(lane), lane, hg);
            sq.commit2d(lane, &mC0, col, wrow);
            stage_row_bf16(sq.acquire(lane), lane, hu);
            sq.commit2d(lane, &mC0, args.n + col, wrow);
#pragma unroll
            for (int j = 0; j < 64; ++j) hg[j] = hg[j] * sigmoidf_fast(hg[j]) * hu[j];
            stage_row_bf16(sq.acquire(lane), lane, hg);
            sq.commit2d(lane, &mC1, col, wrow);
          }
        } else {  // n == 32: accumulator columns are [gate 32 | up 32] = the whole H row
          uint32_t g0[32], u0[32];
          ptx::tmem_ld32(t_acc, g0);
          ptx::tmem_ld32(t_acc + 32, u0);
          ptx::tmem_ld_wait();
          float h[64], a[64];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            h[j] = bf16r(__uint_as_float(g0[j]));
            h[32 + j] = bf16r(__uint_as_float(u0[j]));
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            a[j] = h[j] * sigmoidf_fast(h[j]) * h[32 + j];
            a[32 + j] = 0.f;
          }
          stage_row_bf16(sq.acquire(lane), lane, h);
          sq.commit2d(lane, &mC0, 0, wrow);
          stage_row_bf16(sq.acquire(lane), lane, a);
          sq.commit2d(lane, &mC1, 0, wrow);  // columns >= n are clipped by the tensor map
        }
      } else if constexpr (KIND == K_DOWN || KIND == K_DXT) {
        float gate = 1.f;
        if constexpr (KIND == K_DOWN) gate = __ldg(args.row_gate + row);
#pragma unroll 1
        for (int c = 0; c < BN; c += 64) {
          if (tc.nt * BN + c >= args.N_dim) break;
          uint32_t r0[32], r1[32];
          ptx::tmem_ld32(t_acc + c, r0);
          ptx::tmem_ld32(t_acc + c + 32, r1);
          ptx::tmem_ld_wait();
          float v[64];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            v[j] = gate * __uint_as_float(r0[j]);
            v[32 + j] = gate * __uint_as_float(r1[j]);
          }
          stage_row_bf16(sq.acquire(lane), lane, v);
          sq.commit2d(lane, &mC0, tc.nt * BN + c, wrow);
        }
      } else if constexpr (KIND == K_DH) {
        const float s = __ldg(args.row_gate + row);
        const int n = args.n;
        const __nv_bfloat16* hrow = args.H + (long long)row * (2 * n);
        float ds = 0.f;
        if constexpr (BN >= 64) {
#pragma unroll 1
          for (int c = 0; c < BN; c += 64) {
            const int col = tc.nt * BN + c;
            uint4 hg4[8], hu4[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              hg4[i] = ptx::ld_nc_v4(hrow + col + 8 * i);
              hu4[i] = ptx::ld_nc_v4(hrow + n + col + 8 * i);
            }
            uint32_t r0[32], r1[32];
            ptx::tmem_ld32(t_acc + c, r0);
            ptx::tmem_ld32(t_acc + c + 32, r1);
            ptx::tmem_ld_wait();
            float dg[64], du[64], ap[64];
            const __nv_bfloat16* hgp = reinterpret_cast<const __nv_bfloat16*>(hg4);
            const __nv_bfloat16* hup = reinterpret_cast<const __nv_bfloat16*>(hu4);
#pragma unroll
            for (int j = 0; j < 64; ++j) {
              const float dap = __uint_as_float(j < 32 ? r0[j] : r1[j - 32]);
              const float gg = __bfloat162float(hgp[j]);
              const float uu = __bfloat162float(hup[j]);
              const float sg = sigmoidf_fast(gg);
              const float sl = gg * sg;
              const float A = sl * uu;
              const float dA = s * dap;
              dg[j] = dA * uu * sg * (1.f + gg * (1.f - sg));
              du[j] = dA * sl;
              ap[j] = s * A;
              ds = fmaf(dap, A, ds);
            }
            stage_row_bf16(sq.acquire(lane), lane, dg);
            sq.commit2d(lane, &mC0, col, wrow);
            stage_row_bf16(sq.acquire(lane), lane, du);
            sq.commit2d(lane, &mC0, n + col, wrow);
            stage_row_bf16(sq.acquire(lane), lane, ap);
            sq.commit2d(lane, &mC1, col, wrow);
          }
        } else {  // n == 32, BN == 32: H row = [gate 32 | up 32]
          uint4 h4[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) h4[i] = ptx::ld_nc_v4(hrow + 8 * i);
          uint32_t r0[32];
          ptx::tmem_ld32(t_acc, r0);
          ptx::tmem_ld_wait();
          const __nv_bfloat16* hp = reinterpret_cast<const __nv_bfloat16*>(h4);
          float dh[64], ap[64];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float dap = __uint_as_float(r0[j]);
            const float gg = __bfloat162float(hp[j]);
            const float uu = __bfloat162float(hp[32 + j]);
            const float sg = sigmoidf_fast(gg);
            const float sl = gg * sg;
            const float A = sl * uu;
            const float dA = s * dap;
            dh[j] = dA * uu * sg * (1.f + gg * (1.f - sg));
            dh[32 + j] = dA * sl;
            ap[j] = s * A;
            ap[32 + j] = 0.f;
            ds = fmaf(dap, A, ds);
          }
          stage_row_bf16(sq.acquire(lane), lane, dh);
          sq.commit2d(lane, &mC0, 0, wrow);
          stage_row_bf16(sq.acquire(lane), lane, ap);
          sq.commit2d(lane, &mC1, 0, wrow);
        }
        if (__ldg(args.row_token + row) < 0) ds = 0.f;
        if (args.n_tiles == 1)
          args.dS[row] = ds;
        else
          args.dS[(long long)tc.nt * args.rows_max + row] = ds;
      } else {  // K_DW2 / K_DW1: fp32 weight gradient tile [128 x BN] of expert e
        const int m0 = tc.mt * GEMM_BM + 32 * q;
        if (m0 < args.M_dim) {
#pragma unroll 1
          for (int c = 0; c < BN; c += 32) {
            if (tc.nt * BN + c >= args.N_dim) break;
            float v[32];
            if (tc.nkb > 0) {
              uint32_t r0[32];
              ptx::tmem_ld32(t_acc + c, r0);
              ptx::tmem_ld_wait();
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r0[j]);
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = 0.f;
            }
            stage_row_f32(sq.acquire(lane), lane, v);
            sq.commit3d(lane, &mC0, tc.nt * BN + c, m0, tc.e);
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (lane == 0) ptx::bulk_wait<0>();
    __syncwarp();
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

}  // namespace sonic
