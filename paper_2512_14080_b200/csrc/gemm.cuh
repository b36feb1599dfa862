// gemm.cuh -- the six grouped GEMMs of the SonicMoE layer as ONE warp-specialised,
// persistent tcgen05/TMEM kernel template for sm_100a.
//
//   kind   paper kernel (Alg.)          D = A . B per expert e                 epilogue
//   UP     up-proj A kernel (Alg. 2)    H_e   = Gather(X) W1_e       (varlen-M) SwiGLU -> H, A
//   DOWN   down-proj Y kernel (Alg. 2)  Y_e   = A_e W2_e             (varlen-M) x gate -> Y (Q2)
//   DH     dH kernel (Alg. 3)           dA'_e = Gather(dO) W2_e^T    (varlen-M) dSwiGLU, A', dS
//   DXT    dX~ kernel (Alg. 5)          dX~_e = dH_e W1_e^T          (varlen-M) -> dX~
//   DW2    dW2 kernel (Alg. 3)          dW2_e = A'_e^T Gather(dO)    (varlen-K) fp32 store
//   DW1    dW1 kernel (Alg. 5)          dW1_e = Gather(X)^T dH_e     (varlen-K) fp32 store
//
// Roles (one CTA per SM, persistent static tile schedule):
//   producers  NP warps.  Contiguous operands: TMA 2-D/3-D tile loads by one thread.
//              Gathered operands (NP = 4): 128 threads issue 16-byte cp.async of the token
//              rows named by the gather map straight into the 128B-swizzled operand layout
//              -- the paper's "gather fused with the HBM load" (sec. 4.1.1).
//              (TMA gather4 was measured at ~80 cycles per 512 B per SM on B200, too slow to
//              feed the tensor cores.)  A producer thread signals a
//              stage full after cp.async.wait_group + fence.proxy.async (lagged by LAG stages).
//   MMA        one warp: TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN,
//              K=16 steps); two TMEM accumulator stages so the epilogue of tile i overlaps
//              the MMA of tile i+1.
//   epilogue   4 warps: tcgen05.ld -> registers -> fused math -> swizzled smem -> TMA store
//              (asynchronous TMA store in all GEMMs).
// Operand smem layout: 128B-swizzled, K-major (rows of 64 K-elements) or MN-major
// (64-element MN chunks x 64 K-rows); a stage is one A tile (128 x 64) + one B tile (BN x 64).
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
  const __nv_bfloat16* gsrc;  // gathered operand source (X or dO), [T, gld]
  int gld;
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

template <int KIND>
__host__ __device__ constexpr int num_producer_warps() {
  return (Traits<KIND>::a_gather || Traits<KIND>::b_gather) ? 4 : 1;
}
template <int KIND>
__host__ __device__ constexpr int gemm_threads() {
  return 32 * (num_producer_warps<KIND>() + 5);
}

// Gather producers signal a stage with cp.async.mbarrier.arrive.noinc (hardware-tracked, the
// producer never blocks) instead of wait_group + arrive.
#ifndef SONIC_GATHER_NOINC
#define SONIC_GATHER_NOINC 1
#endif
constexpr bool GATHER_NOINC = SONIC_GATHER_NOINC != 0;
constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;
constexpr int STG_BYTES = 4096;  // one epilogue staging buffer: 32 rows x 128 B
constexpr int SMEM_LIMIT = 232448;

template <int BN, bool HTMA = false, int NB_ = 2>
struct GemmCfg {
  static constexpr uint32_t A_BYTES = GEMM_BM * GEMM_BK * 2;
  static constexpr uint32_t B_BYTES = BN * GEMM_BK * 2;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int NB = NB_;  // epilogue staging buffers per epilogue warp (ring)
  // DH only: per-epilogue-warp H buffer, 32 rows x (BN gate + BN up) bf16 columns (TMA-loaded)
  static constexpr int HBUF_WARP = HTMA ? 32 * 2 * BN * 2 : 0;
  static constexpr int FIXED = 4 * NB * STG_BYTES + 4 * HBUF_WARP + 1024 + 256;
  static constexpr int STAGES_RAW = (SMEM_LIMIT - FIXED) / (int)STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int SMEM = STAGES * STAGE_BYTES + FIXED;
  static constexpr uint32_t TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                        : (2 * BN <= 256) ? 256 : 512;
  static constexpr int LAG = STAGES - 2 > 0 ? STAGES - 2 : 1;  // cp.async stages in flight per producer
};

// DH with BN in {64, 128} reads H through TMA into per-warp smem buffers ("asynchronous
// TMA load of H in the dH epilogue"); wider tiles would not leave room for the buffer.
// Staging ring depth: a deeper ring lets each TMA store finish reading smem while later
// ones are written (the epilogue was the measured limiter); at BN = 256 the
// price is one mainloop stage (3 instead of 4).
#ifndef SONIC_NB_WIDE
#define SONIC_NB_WIDE 2
#endif
#ifndef SONIC_NB_NARROW
#define SONIC_NB_NARROW 2
#endif
template <int KIND, int BN>
__host__ __device__ constexpr int staging_nb() {
  return KIND == K_DH ? 2 : (BN == 256 ? SONIC_NB_WIDE : SONIC_NB_NARROW);
}
template <int KIND, int BN>
using KCfg = GemmCfg<BN, KIND == K_DH && (BN == 64 || BN == 128), staging_nb<KIND, BN>()>;

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

// Pad rows (-1) read token 0: their gate is 0, so every value they produce is exactly 0.
__device__ __forceinline__ int tok_of(const int* row_token, int r) { return max(__ldg(row_token + r), 0); }

__device__ __forceinline__ float bf16r(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }
// sigma(x) = 0.5 tanh(x/2) + 0.5 with the SFU tanh (rel. err ~2^-11, far below bf16's 2^-8)
__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sigmoidf_fast(float x) { return fmaf(0.5f, tanh_approx(0.5f * x), 0.5f); }
__device__ __forceinline__ uint32_t swz(int lane, int chunk) { return (uint32_t)(lane * 128 + ((chunk ^ (lane & 7)) << 4)); }

// Per-warp ring of NB TMA-store staging buffers (32 rows x 128 B each, 128B swizzle).  Stores
// are issued in ring order, one bulk group each, so the buffer k slots ahead of the head was last
// stored from NB-k stores ago: it is free once at most NB-1-k newer groups are pending a read.
template <int NB>
struct StoreQ {
  uint8_t* base;
  int sb;  // ring head: the next buffer to write
  __device__ __forceinline__ uint32_t addr(int i) const { return ptx::smem_u32(base + i * STG_BYTES); }
  template <int N>
  __device__ __forceinline__ void wait_reads(int lane) {
    if (lane == 0) ptx::bulk_wait_read<N>();
    __syncwarp();
  }
  // the buffer k slots ahead of the head, once it is free to overwrite
  template <int K = 0>
  __device__ __forceinline__ int acquire(int lane) {
    static_assert(K < NB, "ring too shallow");
    wait_reads<NB - 1 - K>(lane);
    return (sb + K) % NB;
  }
  __device__ __forceinline__ void issue(int lane, int i, const CUtensorMap* map, int c0, int c1) {
    ptx::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      ptx::tma_store_2d(map, base + i * STG_BYTES, c0, c1);
      ptx::bulk_commit();
    }
    sb = (i + 1) % NB;
  }
  __device__ __forceinline__ void issue3d(int lane, int i, const CUtensorMap* map, int c0, int c1, int c2) {
    ptx::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      ptx::tma_store_3d(map, base + i * STG_BYTES, c0, c1, c2);
      ptx::bulk_commit();
    }
    sb = (i + 1) % NB;
  }
};

// 32 gate + 32 up columns of one H row (starting at column col of the gate half)
__device__ __forceinline__ void dh_prefetch(uint4 (&g)[4], uint4 (&u)[4], const __nv_bfloat16* hrow, int n, int col) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    g[i] = ptx::ld_nc_v4(hrow + col + 8 * i);
    u[i] = ptx::ld_nc_v4(hrow + n + col + 8 * i);
  }
}

__device__ __forceinline__ void write_row_bf16(uint32_t buf, int lane, const float* v /*64*/) {
#pragma unroll
  for (int c = 0; c < 8; ++c)
    ptx::st_shared_v4(buf + swz(lane, c), ptx::pack_bf16(v[8 * c], v[8 * c + 1]),
                      ptx::pack_bf16(v[8 * c + 2], v[8 * c + 3]), ptx::pack_bf16(v[8 * c + 4], v[8 * c + 5]),
                      ptx::pack_bf16(v[8 * c + 6], v[8 * c + 7]));
}

template <int KIND, int BN>
__global__ void __launch_bounds__(gemm_threads<KIND>(), 1)
    sonic_gemm_kernel(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB,
                      const __grid_constant__ CUtensorMap mC0, const __grid_constant__ CUtensorMap mC1,
                      const __grid_constant__ CUtensorMap mD, const GemmArgs args) {
  using Tr = Traits<KIND>;
  using Cfg = KCfg<KIND, BN>;
  constexpr bool HTMA = Cfg::HBUF_WARP > 0;
  constexpr int NP = num_producer_warps<KIND>();
  constexpr bool GATHER = NP > 1;
  constexpr int STAGES = Cfg::STAGES;
  constexpr uint32_t A_BYTES = Cfg::A_BYTES;
  constexpr uint32_t STAGE_BYTES = Cfg::STAGE_BYTES;
  // bytes landing through TMA per stage (the non-gathered operands)
  constexpr uint32_t TMA_BYTES = !GATHER ? STAGE_BYTES : (Tr::a_gather ? Cfg::B_BYTES : A_BYTES);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stg = smem + STAGES * STAGE_BYTES;
  uint8_t* hbuf = stg + 4 * Cfg::NB * STG_BYTES;  // DH: 4 x HBUF_WARP
  uint64_t* full = reinterpret_cast<uint64_t*>(hbuf + 4 * Cfg::HBUF_WARP);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* hfull = tempty + 2;  // one per epilogue warp
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(hfull + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], GATHER ? NP * 32 + 1 : 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], 4);
    }
    for (int s = 0; s < 4; ++s) ptx::mbar_init(&hfull[s], 1);
    ptx::fence_barrier_init();
    ptx::prefetch_tmap(&mA);
    ptx::prefetch_tmap(&mB);
  }
  if (warp == NP) {
    ptx::tmem_alloc(tmem_holder, Cfg::TMEM_COLS);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  const int total_tiles = Tr::vk ? args.E * args.m_tiles * args.n_tiles : (*args.num_m_tiles) * args.n_tiles;

  if (warp < NP) {
    // ============================================================ producers
    int stage = 0;
    uint32_t phase = 0;
    if constexpr (!GATHER) {
      if (lane == 0) {
        for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
          const TileCoord tc = decode_tile<KIND, BN>(args, tile);
          for (int kb = 0; kb < tc.nkb; ++kb) {
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sA = smem + stage * STAGE_BYTES;
            uint8_t* sB = sA + A_BYTES;
            uint64_t* bar = &full[stage];
            ptx::mbar_arrive_expect_tx(bar, STAGE_BYTES);
            ptx::tma_load_2d(sA, &mA, bar, kb * GEMM_BK, tc.row0);
            if constexpr (KIND == K_DOWN) {
#pragma unroll
              for (int j = 0; j < BN / 64; ++j)
                ptx::tma_load_3d(sB + j * 8192, &mB, bar, tc.nt * BN + 64 * j, kb * GEMM_BK, tc.e);
            } else {  // DXT: K-major weights, one box of BN rows
              ptx::tma_load_3d(sB, &mB, bar, kb * GEMM_BK, tc.nt * BN, tc.e);
            }
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    } else {
      const int pt = threadIdx.x;  // 0..127
      const int c = pt & 7;        // 16-byte chunk within a 128-byte row
      const int r0 = pt >> 3;      // rows r0 + 16 j
      const uint32_t sw = (uint32_t)((c ^ (r0 & 7)) << 4);
      int pend = 0, pstage = 0;
      // Gather indices are prefetched one tile (varlen-M) / one stage (varlen-K) ahead so the
      // dependent cp.async addresses never wait on a global load.
      int ntok[8];
      if constexpr (!Tr::vk) {
        if (blockIdx.x < total_tiles) {
          const TileCoord t0 = decode_tile<KIND, BN>(args, blockIdx.x);
#pragma unroll
          for (int j = 0; j < 8; ++j) ntok[j] = tok_of(args.row_token, t0.row0 + r0 + 16 * j);
        }
      }
      for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
        const TileCoord tc = decode_tile<KIND, BN>(args, tile);
        const __nv_bfloat16* srcM[8];
        int ktok[4];
        if constexpr (!Tr::vk) {
#pragma unroll
          for (int j = 0; j < 8; ++j) srcM[j] = args.gsrc + (size_t)ntok[j] * args.gld + c * 8;
          if (tile + (int)gridDim.x < total_tiles) {
            const TileCoord tn = decode_tile<KIND, BN>(args, tile + gridDim.x);
#pragma unroll
            for (int j = 0; j < 8; ++j) ntok[j] = tok_of(args.row_token, tn.row0 + r0 + 16 * j);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) ktok[j] = tok_of(args.row_token, tc.seg0 + r0 + 16 * j);
        }
        for (int kb = 0; kb < tc.nkb; ++kb) {
          const __nv_bfloat16* srcK[4];
          if constexpr (Tr::vk) {
            const int col0 = Tr::a_gather ? tc.mt * GEMM_BM : tc.nt * BN;
#pragma unroll
            for (int j = 0; j < 4; ++j) srcK[j] = args.gsrc + (size_t)ktok[j] * args.gld + col0 + c * 8;
            if (kb + 1 < tc.nkb) {
              const int krow1 = tc.seg0 + (kb + 1) * GEMM_BK;
#pragma unroll
              for (int j = 0; j < 4; ++j) ktok[j] = tok_of(args.row_token, krow1 + r0 + 16 * j);
            }
          }
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sA = smem + stage * STAGE_BYTES;
          uint8_t* sB = sA + A_BYTES;
          uint64_t* bar = &full[stage];
          if (pt == 0) {
            ptx::mbar_arrive_expect_tx(bar, TMA_BYTES);
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
            } else if constexpr (KIND == K_DH) {
              ptx::tma_load_3d(sB, &mB, bar, kb * GEMM_BK, tc.nt * BN, tc.e);
            } else if constexpr (KIND == K_DW2) {  // A' tile (MN-major): 64 rows x 128 M columns
              const int krow0 = tc.seg0 + kb * GEMM_BK;
              ptx::tma_load_2d(sA, &mA, bar, tc.mt * GEMM_BM, krow0);
              ptx::tma_load_2d(sA + 8192, &mA, bar, tc.mt * GEMM_BM + 64, krow0);
            } else {  // DW1: dH tile (MN-major): 64 rows x BN columns
              const int krow0 = tc.seg0 + kb * GEMM_BK;
#pragma unroll
              for (int j = 0; j < BN / 64; ++j) ptx::tma_load_2d(sB + j * 8192, &mB, bar, tc.nt * BN + 64 * j, krow0);
            }
          }
          if constexpr (!Tr::vk) {  // A: 128 gathered rows x 64 K (K-major)
            const uint32_t dst = ptx::smem_u32(sA) + r0 * 128 + sw;
#pragma unroll
            for (int j = 0; j < 8; ++j) ptx::cp_async16(dst + j * 16 * 128, srcM[j] + kb * GEMM_BK);
          } else {  // 64 gathered K-rows x (128 | BN) MN-columns (MN-major)
            constexpr int NCH = Tr::a_gather ? 2 : BN / 64;
            const uint32_t dst = ptx::smem_u32(Tr::a_gather ? sA : sB) + r0 * 128 + sw;
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
              for (int jj = 0; jj < NCH; ++jj) ptx::cp_async16(dst + jj * 8192 + j * 16 * 128, srcK[j] + 64 * jj);
          }
          if constexpr (GATHER_NOINC) {
            ptx::cp_async_mbar_arrive(bar);  // arrives when this thread's copies land
          } else {
            ptx::cp_async_commit();
            if (++pend > Cfg::LAG) {
              ptx::cp_async_wait<Cfg::LAG>();
              ptx::fence_proxy_async_smem();
              ptx::mbar_arrive(&full[pstage]);
              if (++pstage == STAGES) pstage = 0;
              --pend;
            }
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      ptx::cp_async_wait<0>();
      ptx::fence_proxy_async_smem();
      while (pend > 0) {
        ptx::mbar_arrive(&full[pstage]);
        if (++pstage == STAGES) pstage = 0;
        --pend;
      }
    }
  } else if (warp == NP) {
    // ============================================================ MMA issuer
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
          // cp.async (generic proxy) data consumed by tcgen05.mma (async proxy)
          if constexpr (GATHER && GATHER_NOINC) ptx::fence_proxy_async_smem();
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
    // ============================================================ epilogue (4 warps)
    const int ew = warp - NP - 1;
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    StoreQ<Cfg::NB> sq{stg + ew * Cfg::NB * STG_BYTES, 0};
    int acc = 0;
    uint32_t acc_phase = 0;
    // DH (HTMA): each epilogue warp TMA-loads its own 32 rows of H (BN gate + BN up columns)
    // for its next tile into a private buffer; dH is then computed in place in that buffer
    // and TMA-stored from it.
    uint8_t* hb = hbuf + ew * Cfg::HBUF_WARP;
    uint32_t hphase = 0;
    auto h_issue = [&](int t) {
      if constexpr (HTMA) {
        if (lane == 0) {
          const TileCoord th = decode_tile<KIND, BN>(args, t);
          ptx::mbar_arrive_expect_tx(&hfull[ew], Cfg::HBUF_WARP);
#pragma unroll
          for (int j = 0; j < BN / 64; ++j) {
            ptx::tma_load_2d(hb + j * STG_BYTES, &mD, &hfull[ew], th.nt * BN + 64 * j, th.row0 + 32 * q);
            ptx::tma_load_2d(hb + (BN / 64 + j) * STG_BYTES, &mD, &hfull[ew], args.n + th.nt * BN + 64 * j,
                             th.row0 + 32 * q);
          }
        }
      }
    };
    if constexpr (HTMA) {
      if (blockIdx.x < total_tiles) h_issue(blockIdx.x);
    }
    // DH (BN = 256): H is read with plain loads, prefetched 32 columns ahead (across tiles too)
    uint4 hpre_g[4], hpre_u[4];
    if constexpr (KIND == K_DH && BN >= 64 && !HTMA) {
      if (blockIdx.x < total_tiles) {
        const TileCoord t0 = decode_tile<KIND, BN>(args, blockIdx.x);
        const __nv_bfloat16* h0 = args.H + (long long)(t0.row0 + 32 * q + lane) * (2 * args.n);
        dh_prefetch(hpre_g, hpre_u, h0, args.n, t0.nt * BN);
      }
    }
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
      const TileCoord tc = decode_tile<KIND, BN>(args, tile);
      const int wrow = tc.row0 + 32 * q;  // first grouped row of this warp's slab
      const int row = wrow + lane;        // this thread's grouped row (varlen-M)
      const bool has_next = tile + (int)gridDim.x < total_tiles;
      const __nv_bfloat16* next_hrow = nullptr;
      int next_col = 0;
      if constexpr (KIND == K_DH) {
        if (has_next) {
          const TileCoord tn = decode_tile<KIND, BN>(args, tile + gridDim.x);
          next_hrow = args.H + (long long)(tn.row0 + 32 * q + lane) * (2 * args.n);
          next_col = tn.nt * BN;
        }
      }
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const uint32_t t_acc = tmem_base + ((uint32_t)(32 * q) << 16) + acc * BN;

#ifdef SONIC_EXPERIMENT_NO_EPI
      if constexpr (true) {  // ablation: mainloop only
        if (has_next) h_issue(tile + gridDim.x);
        if constexpr (HTMA) {
          ptx::mbar_wait(&hfull[ew], hphase);
          hphase ^= 1;
        }
      } else
#endif
      if constexpr (KIND == K_UP) {
        constexpr int W = BN / 2;
        if constexpr (W >= 64) {
#pragma unroll 1
          for (int c = 0; c < W; c += 64) {
            const int col = tc.nt * W + c;
            sq.acquire<1>(lane);  // the next two ring slots are both free
            const int i0 = sq.sb;
            const int i1 = (i0 + 1) % Cfg::NB;
            const uint32_t b0 = sq.addr(i0), b1 = sq.addr(i1);
            uint32_t apk[32];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              uint32_t g[32], u[32];
              ptx::tmem_ld32(t_acc + c + 32 * h, g);
              ptx::tmem_ld32(t_acc + W + c + 32 * h, u);
              ptx::tmem_ld_wait();
#pragma unroll
              for (int q8 = 0; q8 < 4; ++q8) {
                float hg[8], hu[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  hg[i] = bf16r(__uint_as_float(g[8 * q8 + i]));
                  hu[i] = bf16r(__uint_as_float(u[8 * q8 + i]));
                }
                const int ch = 4 * h + q8;
                ptx::st_shared_v4(b0 + swz(lane, ch), ptx::pack_bf16(hg[0], hg[1]), ptx::pack_bf16(hg[2], hg[3]),
                                  ptx::pack_bf16(hg[4], hg[5]), ptx::pack_bf16(hg[6], hg[7]));
                ptx::st_shared_v4(b1 + swz(lane, ch), ptx::pack_bf16(hu[0], hu[1]), ptx::pack_bf16(hu[2], hu[3]),
                                  ptx::pack_bf16(hu[4], hu[5]), ptx::pack_bf16(hu[6], hu[7]));
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const float a0 = hg[2 * i] * sigmoidf_fast(hg[2 * i]) * hu[2 * i];
                  const float a1 = hg[2 * i + 1] * sigmoidf_fast(hg[2 * i + 1]) * hu[2 * i + 1];
                  apk[4 * ch + i] = ptx::pack_bf16(a0, a1);
                }
              }
            }
            sq.issue(lane, i0, &mC0, col, wrow);           // H gate columns
            sq.issue(lane, i1, &mC0, args.n + col, wrow);  // H up columns
            const int i2 = sq.acquire(lane);
            const uint32_t b2 = sq.addr(i2);
#pragma unroll
            for (int ch = 0; ch < 8; ++ch)
              ptx::st_shared_v4(b2 + swz(lane, ch), apk[4 * ch], apk[4 * ch + 1], apk[4 * ch + 2], apk[4 * ch + 3]);
            sq.issue(lane, i2, &mC1, col, wrow);           // A = SwiGLU(H)
          }
        } else {  // n == 32: accumulator columns are [gate 32 | up 32] = the whole H row
          uint32_t g[32], u[32];
          ptx::tmem_ld32(t_acc, g);
          ptx::tmem_ld32(t_acc + 32, u);
          ptx::tmem_ld_wait();
          float h[64], a[64];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            h[j] = bf16r(__uint_as_float(g[j]));
            h[32 + j] = bf16r(__uint_as_float(u[j]));
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            a[j] = h[j] * sigmoidf_fast(h[j]) * h[32 + j];
            a[32 + j] = 0.f;
          }
          int i = sq.acquire(lane);
          write_row_bf16(sq.addr(i), lane, h);
          sq.issue(lane, i, &mC0, 0, wrow);
          i = sq.acquire(lane);
          write_row_bf16(sq.addr(i), lane, a);
          sq.issue(lane, i, &mC1, 0, wrow);  // columns >= n are clipped by the tensor map
        }
      } else if constexpr (KIND == K_DOWN || KIND == K_DXT) {
        float gate = 1.f;
        if constexpr (KIND == K_DOWN) gate = __ldg(args.row_gate + row);
#pragma unroll 1
        for (int c = 0; c < BN; c += 64) {
          if (tc.nt * BN + c >= args.N_dim) break;
          const int i = sq.acquire(lane);
          const uint32_t b = sq.addr(i);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint32_t r[32];
            ptx::tmem_ld32(t_acc + c + 32 * h, r);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int q8 = 0; q8 < 4; ++q8) {
              const uint32_t* v = r + 8 * q8;
              ptx::st_shared_v4(b + swz(lane, 4 * h + q8),
                                ptx::pack_bf16(gate * __uint_as_float(v[0]), gate * __uint_as_float(v[1])),
                                ptx::pack_bf16(gate * __uint_as_float(v[2]), gate * __uint_as_float(v[3])),
                                ptx::pack_bf16(gate * __uint_as_float(v[4]), gate * __uint_as_float(v[5])),
                                ptx::pack_bf16(gate * __uint_as_float(v[6]), gate * __uint_as_float(v[7])));
            }
          }
          sq.issue(lane, i, &mC0, tc.nt * BN + c, wrow);
        }
      } else if constexpr (KIND == K_DH) {
        const float s = __ldg(args.row_gate + row);
        const int n = args.n;
        const __nv_bfloat16* hrow = args.H + (long long)row * (2 * n);
        float ds = 0.f;
#ifdef SONIC_EXPERIMENT_DH_EPI
        constexpr int EXP = SONIC_EXPERIMENT_DH_EPI;  // 1: skip everything, 2: no H loads, 3: no stores
#else
        constexpr int EXP = 0;
#endif
        if constexpr (EXP == 1) {
        } else if constexpr (HTMA) {
          ptx::mbar_wait(&hfull[ew], hphase);
          hphase ^= 1;
#pragma unroll 1
          for (int c = 0; c < BN / 64; ++c) {
            const int col = tc.nt * BN + 64 * c;
            const uint32_t gb = ptx::smem_u32(hb + c * STG_BYTES);              // H gate -> dH gate
            const uint32_t ub = ptx::smem_u32(hb + (BN / 64 + c) * STG_BYTES);  // H up   -> dH up
            const uint32_t ab = sq.addr(c & 1);                                  // A' staging
            sq.wait_reads<3>(lane);  // the A' store issued from this buffer 2 chunks ago has read it
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              uint32_t r[32];
              ptx::tmem_ld32(t_acc + 64 * c + 32 * h, r);
              uint4 hg4[4], hu4[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                hg4[i] = ptx::ld_shared_v4(gb + swz(lane, 4 * h + i));
                hu4[i] = ptx::ld_shared_v4(ub + swz(lane, 4 * h + i));
              }
              ptx::tmem_ld_wait();
              const __nv_bfloat16* hgp = reinterpret_cast<const __nv_bfloat16*>(hg4);
              const __nv_bfloat16* hup = reinterpret_cast<const __nv_bfloat16*>(hu4);
#pragma unroll
              for (int q8 = 0; q8 < 4; ++q8) {
                uint32_t pg[4], pu[4], pa[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  float dg2[2], du2[2], ap2[2];
#pragma unroll
                  for (int k = 0; k < 2; ++k) {
                    const int j = 8 * q8 + 2 * i + k;
                    const float dap = __uint_as_float(r[j]);
                    const float gg = __bfloat162float(hgp[j]);
                    const float uu = __bfloat162float(hup[j]);
                    const float sg = sigmoidf_fast(gg);
                    const float sl = gg * sg;
                    const float A = sl * uu;
                    const float dA = s * dap;
                    dg2[k] = dA * uu * sg * fmaf(gg, 1.f - sg, 1.f);
                    du2[k] = dA * sl;
                    ap2[k] = s * A;
                    ds = fmaf(dap, A, ds);
                  }
                  pg[i] = ptx::pack_bf16(dg2[0], dg2[1]);
                  pu[i] = ptx::pack_bf16(du2[0], du2[1]);
                  pa[i] = ptx::pack_bf16(ap2[0], ap2[1]);
                }
                ptx::st_shared_v4(gb + swz(lane, 4 * h + q8), pg[0], pg[1], pg[2], pg[3]);
                ptx::st_shared_v4(ub + swz(lane, 4 * h + q8), pu[0], pu[1], pu[2], pu[3]);
                ptx::st_shared_v4(ab + swz(lane, 4 * h + q8), pa[0], pa[1], pa[2], pa[3]);
              }
            }
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              ptx::tma_store_2d(&mC0, hb + c * STG_BYTES, col, wrow);                      // dH gate
              ptx::bulk_commit();
              ptx::tma_store_2d(&mC0, hb + (BN / 64 + c) * STG_BYTES, n + col, wrow);      // dH up
              ptx::bulk_commit();
              ptx::tma_store_2d(&mC1, sq.base + (c & 1) * STG_BYTES, col, wrow);           // A' = s A
              ptx::bulk_commit();
            }
          }
          if (has_next) {
            sq.wait_reads<1>(lane);  // every dH store out of the H buffer has read it
            h_issue(tile + gridDim.x);
          }
        } else if constexpr (BN >= 64) {
#pragma unroll 1
          for (int c = 0; c < BN; c += 64) {
            const int col = tc.nt * BN + c;
            sq.wait_reads<0>(lane);
            const uint32_t b0 = sq.addr(0), b1 = sq.addr(1);
            uint32_t apk[32];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              // H for this half was prefetched one half ahead (or before the tfull wait)
              uint4 hg4[4], hu4[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                hg4[i] = hpre_g[i];
                hu4[i] = hpre_u[i];
              }
              if constexpr (EXP != 2) {
                if (c + 32 * h + 32 < BN) {
                  dh_prefetch(hpre_g, hpre_u, hrow, n, col + 32 * h + 32);
                } else if (has_next) {
                  dh_prefetch(hpre_g, hpre_u, next_hrow, n, next_col);
                }
              }
              uint32_t r[32];
              ptx::tmem_ld32(t_acc + c + 32 * h, r);
              ptx::tmem_ld_wait();
              const __nv_bfloat16* hgp = reinterpret_cast<const __nv_bfloat16*>(hg4);
              const __nv_bfloat16* hup = reinterpret_cast<const __nv_bfloat16*>(hu4);
#pragma unroll
              for (int q8 = 0; q8 < 4; ++q8) {
                uint32_t pg[4], pu[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  float dg2[2], du2[2], ap2[2];
#pragma unroll
                  for (int k = 0; k < 2; ++k) {
                    const int j = 8 * q8 + 2 * i + k;
                    const float dap = __uint_as_float(r[j]);
                    const float gg = __bfloat162float(hgp[j]);
                    const float uu = __bfloat162float(hup[j]);
                    const float sg = sigmoidf_fast(gg);
                    const float sl = gg * sg;
                    const float A = sl * uu;
                    const float dA = s * dap;
                    dg2[k] = dA * uu * sg * (1.f + gg * (1.f - sg));
                    du2[k] = dA * sl;
                    ap2[k] = s * A;
                    ds = fmaf(dap, A, ds);
                  }
                  pg[i] = ptx::pack_bf16(dg2[0], dg2[1]);
                  pu[i] = ptx::pack_bf16(du2[0], du2[1]);
                  apk[16 * h + 4 * q8 + i] = ptx::pack_bf16(ap2[0], ap2[1]);
                }
                if constexpr (EXP != 3) {
                  ptx::st_shared_v4(b0 + swz(lane, 4 * h + q8), pg[0], pg[1], pg[2], pg[3]);
                  ptx::st_shared_v4(b1 + swz(lane, 4 * h + q8), pu[0], pu[1], pu[2], pu[3]);
                } else {
                  ds += __uint_as_float(pg[0] ^ pu[1]) * 1e-30f;
                }
              }
            }
            if constexpr (EXP != 3) {
              sq.issue(lane, 0, &mC0, col, wrow);      // dH gate columns
              sq.issue(lane, 1, &mC0, n + col, wrow);  // dH up columns
              sq.wait_reads<1>(lane);
#pragma unroll
              for (int ch = 0; ch < 8; ++ch)
                ptx::st_shared_v4(b0 + swz(lane, ch), apk[4 * ch], apk[4 * ch + 1], apk[4 * ch + 2], apk[4 * ch + 3]);
              sq.issue(lane, 0, &mC1, col, wrow);      // A' = s A
            } else {
              ds += __uint_as_float(apk[0] ^ apk[31]) * 1e-30f;
            }
          }
        } else {  // n == 32, BN == 32: H row = [gate 32 | up 32]
          uint4 h4[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) h4[i] = ptx::ld_nc_v4(hrow + 8 * i);
          uint32_t r[32];
          ptx::tmem_ld32(t_acc, r);
          ptx::tmem_ld_wait();
          const __nv_bfloat16* hp = reinterpret_cast<const __nv_bfloat16*>(h4);
          float dh[64], ap[64];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float dap = __uint_as_float(r[j]);
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
          int i = sq.acquire(lane);
          write_row_bf16(sq.addr(i), lane, dh);
          sq.issue(lane, i, &mC0, 0, wrow);
          i = sq.acquire(lane);
          write_row_bf16(sq.addr(i), lane, ap);
          sq.issue(lane, i, &mC1, 0, wrow);
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
            const int i = sq.acquire(lane);
            const uint32_t b = sq.addr(i);
            if (tc.nkb > 0) {
              uint32_t r[32];
              ptx::tmem_ld32(t_acc + c, r);
              ptx::tmem_ld_wait();
#pragma unroll
              for (int ch = 0; ch < 8; ++ch)
                ptx::st_shared_v4(b + swz(lane, ch), r[4 * ch], r[4 * ch + 1], r[4 * ch + 2], r[4 * ch + 3]);
            } else {
#pragma unroll
              for (int ch = 0; ch < 8; ++ch) ptx::st_shared_v4(b + swz(lane, ch), 0u, 0u, 0u, 0u);
            }
            sq.issue3d(lane, i, &mC0, tc.nt * BN + c, m0, tc.e);
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
  if (warp == NP) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

}  // namespace sonic
