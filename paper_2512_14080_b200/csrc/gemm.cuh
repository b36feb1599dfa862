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
//              -- the paper's "gather fused with the HBM load" (sec. 4.1.1) -- and
//              signal with cp.async.mbarrier.arrive.noinc.  (TMA gather4 was measured at ~80
//              cycles per 512 B per SM on B200, too slow to feed the tensor cores.)
//   MMA        one warp: TMEM allocator + single-thread tcgen05.mma issuer (K=16 steps); two TMEM
//              accumulator stages so the epilogue of tile i overlaps the MMA of tile i+1.
//   epilogue   4 warps: tcgen05.ld -> registers -> fused math -> swizzled smem -> TMA store
//              (asynchronous TMA store in all GEMMs).
//
// CTA2 = true: a cluster of two CTAs computes a 256 x BN tile with tcgen05.mma.cta_group::2
// (M = 256).  Each CTA loads its own 128 A rows and HALF of B (BN/2 columns or rows); the leader
// (rank 0) issues the MMAs and multicasts its commits to both CTAs' barriers, so each CTA's TMEM
// holds its 128 rows of the accumulator and runs its own epilogue.  Operand traffic per FLOP drops
// by a third.  varlen-M pairs two 128-row tiles of ONE expert (route's tile_pairs; an expert with an
// odd tile count ends in a half pair whose second CTA computes but does not store).  For gathered
// operands the peer CTA's MMA warp relays its local cp.async completion to the leader's barrier --
// the paper's Blackwell relay warp.
//
// Operand smem layout: 128B-swizzled, K-major (rows of 64 K-elements) or MN-major (64-element MN
// chunks x 64 K-rows); a stage is one A tile (128 x 64) + one B tile (BN or BN/2 x 64).
#pragma once
#include "ptx.cuh"

namespace sonic {

enum GemmKind { K_UP = 0, K_DOWN = 1, K_DH = 2, K_DXT = 3, K_DW2 = 4, K_DW1 = 5, K_UP8 = 6, K_DXT8 = 7 };
// K_DXT8: dX~ with e4m3 operands (SONIC_F_FP8_DXT, NEXT-4, DESIGN Q25): A = the row-quantised
// dH' = bf16(dH) * sw (the forward's per-column W1 scales folded in), B = the forward's e4m3 W1 copy
// (K-major here: W1q_e [d, 2n]); dX~ = sum * s_row in the DXT epilogue.  k-blocks of 128 e4m3.
// K_UP8: the up-projection with e4m3 operands (SONIC_F_FP8_UP, NEXT-4): Gather(Xq) W1q_e with the
// per-token scale sx and per-column scale sw applied to the fp32 sum in the epilogue, which is then
// K_UP's (H, A in bf16).  A k-block is 128 e4m3 values: the same 128-byte rows, stages and
// descriptors as bf16's 64; the MMA is kind::f8f6f4 (K = 32).

struct GemmArgs {
  const int* num_m_tiles;   // varlen-M: device-resident count of 128-row tiles (R_pad / 128)
  const int* num_pairs;     // varlen-M, CTA2: device-resident count of tile pairs
  const int* tile_pairs;    // varlen-M, CTA2: first tile of each pair | (second exists) << 31
  const int* tile_expert;   // varlen-M: expert of each 128-row tile
  const int* row_token;     // gather map, -1 on pad rows
  const float* row_gate;    // gate per grouped row, 0 on pad rows
  const int* pad_offsets;   // [E+1] tile-aligned expert segments
  const __nv_bfloat16* gsrc;  // gathered operand source (X or dO), [T, gld]
  int gld;
  int E;
  int n_tiles;              // output tiles along N
  int m_tiles;              // varlen-K: output tiles (128 rows) along M per expert
  int k_blocks;             // varlen-M: ceil(K / 64)
  int n;                    // expert intermediate dim (offset of the "up" half of H)
  int M_dim, N_dim;         // output extent along M (varlen-K) and N
  float* dS;                // DH: dS [rows] if n_tiles == 1, else partials [n_tiles][rows_max]
  long long rows_max;
  unsigned long long* dbg;  // SONIC_TIMING builds only: cycle counters (see sonic_api.cu)
  int wide;                 // DOWN / DXT: mC0 is the 3-D [col block, row, 64 cols] view of the output and one
                            // TMA store writes SONIC_WIDE_ST 64-column chunks (0: 2-D map, one store per chunk)
  // DW1 / DW2 with SONIC_AGG_FUSE: the dX aggregation (Alg. 5's last kernel) of tokens
  // [agg_t0, agg_t1) runs on this kernel's aggregator warp(s), contiguous token blocks per CTA
  const __nv_bfloat16* agg_src;  // dX~ [rows, agg_d]
  __nv_bfloat16* agg_dst;        // dX [T, agg_d]
  const int* agg_rowptr;         // token CSR over grouped rows (expert-ascending)
  const int* agg_rows;
  long long agg_t0, agg_t1;
  int agg_d;
  int accumulate;           // DW1 / DW2: add into the existing dW (SONIC_F_DW_ACCUMULATE) instead of overwriting
  int dw_bf16;              // DW1 / DW2: store dW as bf16 (SONIC_F_DW_BF16; the store map is then bf16)
  const float* sx;          // UP8: per-token scale of the e4m3 X rows [T]; DXT8: per-row scale of the e4m3 dH' [rows]
  const float* sw;          // UP8: per-column scale of the e4m3 W1 [E, 2n]
};

template <int KIND>
struct Traits;
template <> struct Traits<K_UP>   { static constexpr bool vk = false, a_gather = true,  a_mn = false, b_gather = false, b_mn = true;  };
template <> struct Traits<K_UP8>  { static constexpr bool vk = false, a_gather = true,  a_mn = false, b_gather = false, b_mn = true;  };
template <> struct Traits<K_DOWN> { static constexpr bool vk = false, a_gather = false, a_mn = false, b_gather = false, b_mn = true;  };
template <> struct Traits<K_DH>   { static constexpr bool vk = false, a_gather = true,  a_mn = false, b_gather = false, b_mn = false; };
template <> struct Traits<K_DXT>  { static constexpr bool vk = false, a_gather = false, a_mn = false, b_gather = false, b_mn = false; };
template <> struct Traits<K_DXT8> { static constexpr bool vk = false, a_gather = false, a_mn = false, b_gather = false, b_mn = false; };
template <> struct Traits<K_DW2>  { static constexpr bool vk = true,  a_gather = false, a_mn = true,  b_gather = true,  b_mn = true;  };
template <> struct Traits<K_DW1>  { static constexpr bool vk = true,  a_gather = true,  a_mn = true,  b_gather = false, b_mn = true;  };

// Gathered kinds: NP producer warps issue the cp.async gathers, 8 lanes per 128-byte row, so one
// pass covers 4 * NP rows (SONIC_NP_VK for the varlen-K kinds, SONIC_NP_VM for the varlen-M ones).
#ifndef SONIC_NP_VK
#define SONIC_NP_VK 4
#endif
#ifndef SONIC_NP_VM
#define SONIC_NP_VM 4
#endif
// SONIC_G4_VK = 1: the varlen-K kinds gather their token rows with TMA tile::gather4 (4 rows x 128 B
// per instruction, issued by 16 lanes of the single producer warp) instead of cp.async, so the
// gathered bytes travel the TMA path and count on the stage's transaction barrier like the tiles.
#ifndef SONIC_G4_VK
#define SONIC_G4_VK 0
#endif
template <int KIND>
__host__ __device__ constexpr bool g4_kind() { return SONIC_G4_VK && Traits<KIND>::vk; }
template <int KIND>
__host__ __device__ constexpr int num_producer_warps() {
  return ((Traits<KIND>::a_gather || Traits<KIND>::b_gather) && !g4_kind<KIND>())
             ? (Traits<KIND>::vk ? SONIC_NP_VK : SONIC_NP_VM) : 1;
}
// Epilogue warps: 4 (one per TMEM lane quarter).  SONIC_EPI_WARPS=8 puts two warps on each quarter,
// each taking every other 64-column chunk; measured slower at 7B (725 vs 745 TF: fewer registers
// and a mainloop stage less) and one small-shape test hung with it -- experimental, not validated.
#ifndef SONIC_EPI_WARPS
#define SONIC_EPI_WARPS 4
#endif
constexpr int EPI_WARPS = SONIC_EPI_WARPS;
// Per-kind epilogue warp count (8 = two warps per TMEM lane quarter, each taking every other
// 64-column chunk).  The down-proj (K = n: few k-blocks per tile) waits on its epilogue, but
// 8 warps did not help it; all kinds use SONIC_EPI_WARPS = 4.
#ifndef SONIC_EPI_WARPS_DOWN
#define SONIC_EPI_WARPS_DOWN 4  // 8 measured slower at 7B (247 vs 239 us)
#endif
#ifndef SONIC_EPI_WARPS_UP8
#define SONIC_EPI_WARPS_UP8 8  // the e4m3 up-projection: its mainloop is twice as fast, so two epilogue warps per TMEM lane quarter (236 -> 214-219 us at 7B)
#endif
template <int KIND>
__host__ __device__ constexpr int epi_warps() {
  return KIND == K_DOWN ? SONIC_EPI_WARPS_DOWN : KIND == K_UP8 ? SONIC_EPI_WARPS_UP8 : EPI_WARPS;
}
// Fused dX aggregation (SONIC_AGG_FUSE = 1, varlen-K kinds): AGW aggregator warps after the
// epilogue warps stream the grouped dX~ rows of their tokens into a shared-memory ring of AGG_SLOT-byte
// slots with bulk copies (the TMA engine, not the LSU path the gather producers use) and sum them.
#ifndef SONIC_AGG_FUSE
#define SONIC_AGG_FUSE 0
#endif
#ifndef SONIC_AGG_RING
#define SONIC_AGG_RING 49152  // bytes of row slots (7B: 16 slots of one 3 KB dX~ row)
#endif
constexpr int AGG_CHUNK = 2048;  // columns per work item at most (a 4 KB slot)
template <int KIND>
__host__ __device__ constexpr int agg_warps() { return (SONIC_AGG_FUSE && Traits<KIND>::vk) ? 1 : 0; }
template <int KIND>
__host__ __device__ constexpr int agg_bytes() { return agg_warps<KIND>() ? 1024 + SONIC_AGG_RING : 0; }
template <int KIND>
__host__ __device__ constexpr int gemm_threads() {
  return 32 * (num_producer_warps<KIND>() + 1 + epi_warps<KIND>() + agg_warps<KIND>());
}

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;
constexpr int STG_BYTES = 4096;  // one epilogue staging buffer: 32 rows x 128 B
#ifndef SONIC_SMEM_LIMIT
#define SONIC_SMEM_LIMIT 232448
#endif
constexpr int SMEM_LIMIT = SONIC_SMEM_LIMIT;

template <int BN, bool CTA2, bool HTMA, int NB_, bool HRING_ = false, int EPW_ = EPI_WARPS, int XB_ = 0>
struct GemmCfg {
  static constexpr int XB = XB_;         // extra fixed bytes (the fused aggregation's ring)
  static constexpr int EPW = EPW_;       // epilogue warps
  static constexpr int EPH = EPW_ / 4;   // warps per TMEM lane quarter
  static constexpr int BNL = CTA2 ? BN / 2 : BN;  // B columns (or rows) held by this CTA
  static constexpr uint32_t A_BYTES = GEMM_BM * GEMM_BK * 2;
  static constexpr uint32_t B_BYTES = BNL * GEMM_BK * 2;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int NB = NB_;  // epilogue staging buffers per epilogue warp (ring)
  // DH only: per-epilogue-warp H buffer, 32 rows x (gate + up) bf16 columns of the warp's chunks
  static constexpr int HCOLS_WARP = (BN / EPH) < 64 ? 64 : BN / EPH;
  // HRING (DH, BN = 256): instead of the whole tile row, a 2-slot ring of 64-column chunks
  // (gate 4 KB + up 4 KB per slot) streams H through each epilogue warp
  static constexpr bool HRING = HRING_;
  static constexpr int HBUF_WARP = HRING ? 2 * 2 * STG_BYTES : HTMA ? 32 * 2 * HCOLS_WARP * 2 : 0;
  // + 1 KB alignment slack + barriers / dS exchange / TMEM address (< 1 KB)
  static constexpr int FIXED = EPW * NB * STG_BYTES + EPW * HBUF_WARP + 1024 + 1024 + XB;
  static constexpr int STAGES_RAW = (SMEM_LIMIT - FIXED) / (int)STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int SMEM = STAGES * STAGE_BYTES + FIXED;
  static constexpr uint32_t TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                        : (2 * BN <= 256) ? 256 : 512;
};

// Wide epilogue stores (DOWN, DXT): G = SONIC_WIDE_ST consecutive 64-column staging buffers go out
// as ONE 3-D TMA store (box 64 x 32 rows x G column blocks) instead of G 4 KB stores.  These two
// kinds have few k-blocks per tile (K = n or 2n), so their SM's TMA unit moves the operand tiles and
// 64 KB of output per CTA per tile; each box costs the TMA unit a fixed issue overhead on top of its
// bytes (tools/l2feed.cu: 4 KB boxes move 58 B/clk, 16 KB boxes 107 B/clk).
#ifndef SONIC_WIDE_DOWN
#define SONIC_WIDE_DOWN 1
#endif
#ifndef SONIC_WIDE_DXT
#define SONIC_WIDE_DXT 1
#endif
#ifndef SONIC_WIDE_SLOTS
#define SONIC_WIDE_SLOTS 1  // staging ring = SLOTS x G buffers per epilogue warp
#endif
template <int KIND>
__host__ __device__ constexpr int wide_g() { return KIND == K_DOWN ? SONIC_WIDE_DOWN : KIND == K_DXT ? SONIC_WIDE_DXT : 1; }
// DH with BN in {64, 128} reads H through TMA into per-warp smem buffers ("asynchronous
// TMA load of H in the dH epilogue").  Staging ring depth NB: 2 (a deeper ring costs a mainloop
// stage, measured slower).
template <int KIND, int BN, bool CTA2>
#ifndef SONIC_NB_DW
#define SONIC_NB_DW 2  // staging ring depth of the weight-gradient kernels
#endif
#ifndef SONIC_NB_DOWN
#define SONIC_NB_DOWN 2  // staging ring depth of the down-proj (4 measured the same at 7B)
#endif
using KCfg = GemmCfg<BN, CTA2, KIND == K_DH && BN <= 128,
                     (KIND == K_DH && BN == 256) ? 0
                     : (wide_g<KIND>() > 1) ? wide_g<KIND>() * SONIC_WIDE_SLOTS
                     : (KIND == K_DOWN ? SONIC_NB_DOWN : Traits<KIND>::vk ? SONIC_NB_DW : 2),
                     KIND == K_DH && BN == 256, epi_warps<KIND>(), agg_bytes<KIND>()>;

struct TileCoord {
  int e, row0, nt, mt, nkb, seg0;
  bool valid;  // CTA2: this CTA's half of the pair tile exists
};

template <int KIND, bool CTA2>
__device__ __forceinline__ int total_tiles_of(const GemmArgs& a) {
  if constexpr (Traits<KIND>::vk) return a.E * (CTA2 ? (a.m_tiles + 1) / 2 : a.m_tiles) * a.n_tiles;
  else return (CTA2 ? *a.num_pairs : *a.num_m_tiles) * a.n_tiles;
}

#ifndef SONIC_DW1_PHASE
#define SONIC_DW1_PHASE 0  // dW1 tile order in d-slice phases of this many M pairs (0: MFAST order)
#endif
// MFAST (varlen-K under MC, the dW1 order): the M-pair index runs fastest, so tiles 2k and 2k+1
// -- the two pairs of a 4-CTA cluster -- share the expert and the N tile (and so the B operand)
template <int KIND, bool CTA2, bool MFAST = false>
__device__ __forceinline__ TileCoord decode_tile(const GemmArgs& a, int tile, int rank) {
  TileCoord c;
  c.valid = true;
  if constexpr (Traits<KIND>::vk) {
    const int mts = CTA2 ? (a.m_tiles + 1) / 2 : a.m_tiles;
    const int per_e = mts * a.n_tiles;
    c.e = tile / per_e;
    const int rem = tile - c.e * per_e;
    int mp;
    constexpr int PH = KIND == K_DW1 ? SONIC_DW1_PHASE : 0;
    if (PH > 0 && mts % (PH > 0 ? PH : 1) == 0) {
      // d-slice phases: the M pairs in groups of PH, phase-major, then expert, N tile, M pair -- X's
      // columns of one phase (PH * 256 of d) stay in L2 while every expert gathers from them
      const int g = PH > 0 ? PH : 1;
      const int per_ph = a.E * a.n_tiles * g;
      const int ph = tile / per_ph;
      const int r1 = tile - ph * per_ph;
      c.e = r1 / (a.n_tiles * g);
      const int r2 = r1 - c.e * a.n_tiles * g;
      c.nt = r2 / g;
      mp = ph * g + (r2 - c.nt * g);
    } else if constexpr (MFAST) {
      c.nt = rem / mts;
      mp = rem - c.nt * mts;
    } else {
      mp = rem / a.n_tiles;
      c.nt = rem - mp * a.n_tiles;
    }
    c.mt = CTA2 ? 2 * mp + rank : mp;
    if (CTA2) c.valid = c.mt < a.m_tiles;
    c.seg0 = __ldg(a.pad_offsets + c.e);
    c.nkb = (__ldg(a.pad_offsets + c.e + 1) - c.seg0) / GEMM_BK;
    c.row0 = 0;
  } else {
    const int p = tile / a.n_tiles;
    c.nt = tile - p * a.n_tiles;
    int first = p;
    if constexpr (CTA2) {
      const int pt = __ldg(a.tile_pairs + p);
      first = pt & 0x7fffffff;
      c.valid = rank == 0 || pt < 0;
    }
    c.mt = first + (CTA2 ? rank : 0);
    c.row0 = c.mt * GEMM_BM;
    c.e = __ldg(a.tile_expert + first);
    c.nkb = a.k_blocks;
    c.seg0 = 0;
  }
  return c;
}

// Pad rows (-1) read token 0: their gate is 0, so every value they produce is exactly 0.
// tok_of loads the raw map entry; clamp() is applied only where the address is formed, so a
// prefetched load is not consumed (and waited for) at the prefetch point.
// DOWN / DXT epilogue: TMEM loads pipelined one chunk ahead (1) or load-wait per 32 columns (0)
#ifndef SONIC_EPI_PIPE
#define SONIC_EPI_PIPE 1
#endif
#ifndef SONIC_KPD
#define SONIC_KPD 16  // 2 -> 4 -> 8 -> 16: dW2 261 -> 255 -> 245 -> 221 us, dW1 410 -> 402 -> 389 -> 375 us (7B); 24+ spills
#endif
// L2 prefetch distance (k-blocks) for the gathered rows (0 = off): the producers touch the lines
// of k-block kb + SONIC_L2PF while filling kb, so the cp.async of a later stage hits L2
#ifndef SONIC_L2PF
#define SONIC_L2PF 0
#endif
#ifdef SONIC_EXP_NOGATHER  // ablation (7B only): contiguous rows instead of the gather map
__device__ __forceinline__ int tok_of(const int* row_token, int r) { return r & 32767; }
#else
__device__ __forceinline__ int tok_of(const int* row_token, int r) { return __ldg(row_token + r); }
#endif
__device__ __forceinline__ size_t clamp_tok(int t) { return (size_t)max(t, 0); }
__device__ __forceinline__ void gather16(uint32_t dst, const void* src, uint64_t pol) {
  if (SONIC_L2_HINTS & 1) ptx::cp_async16_hint(dst, src, pol);
  else ptx::cp_async16(dst, src);
}

// fp32 += 8 bf16 (one 16-byte chunk), and 8 fp32 -> 8 bf16 (round to nearest even): the fused
// aggregation's arithmetic, identical to aggregate.cu's
__device__ __forceinline__ void acc8_bf16(float (&a)[8], const uint4& v) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    a[2 * i] += f.x;
    a[2 * i + 1] += f.y;
  }
}
__device__ __forceinline__ uint4 pack8_bf16(const float (&a)[8]) {
  uint4 o;
  __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
  for (int i = 0; i < 4; ++i) oh[i] = __floats2bfloat162_rn(a[2 * i], a[2 * i + 1]);
  return o;
}
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
#ifndef SONIC_EXP_EPI
#define SONIC_EXP_EPI 0  // ablation: 1 = TMEM loads only (down/dXt), 2 = no TMA stores, 3 = L2-resident stores
#endif
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
    if (lane == 0 && SONIC_EXP_EPI == 3) {  // same traffic into L2, but L2-resident (per-warp 4 KB region)
      ptx::tma_store_2d(map, base + i * STG_BYTES, 0, (int)(blockIdx.x * 8 + (threadIdx.x >> 5)) * 32);
      ptx::bulk_commit();
    }
    if (lane == 0 && SONIC_EXP_EPI == 0) {
      ptx::tma_store_2d(map, base + i * STG_BYTES, c0, c1);
      ptx::bulk_commit();
    }
    sb = (i + 1) % NB;
  }
  // wide stores: the ring as NB / G slots of G consecutive buffers, one 3-D store per slot
  template <int G>
  __device__ __forceinline__ int acquire_slot(int lane) {
    static_assert(NB % G == 0, "wide store slots");
    wait_reads<NB / G - 1>(lane);
    return sb;
  }
  template <int G>
  __device__ __forceinline__ void issue_slot(int lane, int s, const CUtensorMap* map, int c0, int c1, int c2) {
    ptx::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      ptx::tma_store_3d(map, base + s * G * STG_BYTES, c0, c1, c2);
      ptx::bulk_commit();
    }
    sb = (s + 1) % (NB / G);
  }
  __device__ __forceinline__ void issue3d(int lane, int i, const CUtensorMap* map, int c0, int c1, int c2,
                                          bool add = false) {
    ptx::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0 && (SONIC_EXP_EPI == 0 || SONIC_EXP_EPI == 3)) {
      if (add) ptx::tma_reduce_add_3d(map, base + i * STG_BYTES, c0, c1, c2);
      else ptx::tma_store_3d(map, base + i * STG_BYTES, c0, c1, c2);
      ptx::bulk_commit();
    }
    sb = (i + 1) % NB;
  }
};

__device__ __forceinline__ void write_row_bf16(uint32_t buf, int lane, const float* v /*64*/) {
#pragma unroll
  for (int c = 0; c < 8; ++c)
    ptx::st_shared_v4(buf + swz(lane, c), ptx::pack_bf16(v[8 * c], v[8 * c + 1]),
                      ptx::pack_bf16(v[8 * c + 2], v[8 * c + 3]), ptx::pack_bf16(v[8 * c + 4], v[8 * c + 5]),
                      ptx::pack_bf16(v[8 * c + 6], v[8 * c + 7]));
}

// TMA tile loads: 1-CTA form (own barrier) or pair form (counted on the leader's barrier).
template <bool CTA2>
__device__ __forceinline__ void tload2(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  if constexpr (CTA2) ptx::tma_load_2d_cg2(dst, m, bar, c0, c1);
  else ptx::tma_load_2d(dst, m, bar, c0, c1);
}
template <bool CTA2>
__device__ __forceinline__ void tload3(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
  if constexpr (CTA2) ptx::tma_load_3d_cg2(dst, m, bar, c0, c1, c2);
  else ptx::tma_load_3d(dst, m, bar, c0, c1, c2);
}

// MC (CTA2 only): a cluster of FOUR CTAs = two pairs.  The static schedule gives the two pairs the
// consecutive pair tiles 2k and 2k+1, which share one operand (DOWN, DXT, DW2: the A tile -- same
// rows, the next N tile; DW1 with the MFAST order: the B tile -- same expert and N tile, the next M
// pair).  Each pair TMA-loads half of the shared tile and multicasts it into both pairs' stage, so
// the L2 -> SM operand traffic per MMA drops by a quarter; a stage is refilled once BOTH pairs' MMAs
// have released it (empty barriers count the two pair leaders' commits).
#ifndef SONIC_EXP_NOFENCE
#define SONIC_EXP_NOFENCE 0  // timing ablation only (results may be wrong): no consumer-side proxy fence
#endif
#ifndef SONIC_STREAM_EF
#define SONIC_STREAM_EF 2  // evict-first hint on the streamed TMA operand of dW1 (1) / dW2 (2): dW2 213 -> 209 us, dW1 unchanged (7B, 3 reps)
#endif
#ifndef SONIC_DW1_MFAST
#define SONIC_DW1_MFAST 1  // dW1 tiles M-pair-fastest: the d-slices of one (expert, N tile) run on neighbouring pairs, which read the same dH columns at the same time (7B: 372.7/373.9 -> 369.7/370.1 us)
#endif
template <int KIND, int BN, bool CTA2, bool MC = false>
__global__ void __launch_bounds__(gemm_threads<KIND>(), 1)
    sonic_gemm_kernel(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB,
                      const __grid_constant__ CUtensorMap mC0, const __grid_constant__ CUtensorMap mC1,
                      const __grid_constant__ CUtensorMap mD, const GemmArgs args) {
  using Tr = Traits<KIND>;
  using Cfg = KCfg<KIND, BN, CTA2>;
  constexpr bool HRING = Cfg::HRING;
  constexpr bool HTMA = Cfg::HBUF_WARP > 0 && !HRING;
  constexpr int NP = num_producer_warps<KIND>();
  constexpr bool GATHER = NP > 1;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int BNL = Cfg::BNL;
  constexpr uint32_t A_BYTES = Cfg::A_BYTES;
  constexpr uint32_t STAGE_BYTES = Cfg::STAGE_BYTES;
  // bytes landing through TMA per stage per CTA (the non-gathered operands)
  constexpr uint32_t TMA_BYTES = !GATHER ? STAGE_BYTES : (Tr::a_gather ? Cfg::B_BYTES : A_BYTES);
  constexpr int MMA_M = CTA2 ? 2 * GEMM_BM : GEMM_BM;
  constexpr bool F8 = KIND == K_UP8 || KIND == K_DXT8;  // e4m3 operands (kind::f8f6f4)
  constexpr int KBE = F8 ? 128 : GEMM_BK;               // operand elements per k-block (128 bytes)
  constexpr int ESZ = F8 ? 1 : 2;     // bytes per operand element

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stg = smem + STAGES * STAGE_BYTES;
  uint8_t* hbuf = stg + Cfg::EPW * Cfg::NB * STG_BYTES;  // DH: Cfg::EPW x HBUF_WARP
  uint64_t* full = reinterpret_cast<uint64_t*>(hbuf + Cfg::EPW * Cfg::HBUF_WARP);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* hfull = tempty + 2;  // DH: one per epilogue warp (HRING: two, one per ring slot)
  float* ds_xchg = reinterpret_cast<float*>(hfull + 2 * Cfg::EPW);  // DH: [4][32] partial dS of half 1
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(ds_xchg + 128);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  static_assert(!MC || CTA2, "multicast clusters are built from 2-CTA pairs");
  constexpr bool MFAST = (MC || SONIC_DW1_MFAST) && KIND == K_DW1;
  const int crank = CTA2 ? (int)ptx::cluster_ctarank() : 0;
  const int rank = crank & 1;                                  // rank within the pair
  const int pidx = MC ? crank >> 1 : 0;                        // pair within the cluster
  const uint32_t lead = (uint32_t)(crank & ~1);                // this pair's leader (cluster rank)
  const uint16_t pmask = (uint16_t)(0x3u << (2 * pidx));      // this pair's two CTAs
  const uint16_t smask = (uint16_t)((1u << rank) | (1u << (2 + rank)));  // MC: same-rank CTAs of both pairs
  (void)smask;
  const bool leader = rank == 0;
  const int t_first = CTA2 ? blockIdx.x / 2 : blockIdx.x;
  const int t_step = CTA2 ? gridDim.x / 2 : gridDim.x;

  ptx::pdl_trigger();
  if (threadIdx.x == 0) {
    // full: leader counts its TMA expect_tx arrive (+ its 128 cp.async arrivals + the peer's relay
    // for gathered kinds); a peer counts only its own cp.async arrivals.
    const int full_cnt = GATHER ? (leader ? NP * 32 + 1 + (CTA2 ? 1 : 0) : NP * 32) : 1;
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], full_cnt);
      ptx::mbar_init(&empty[s], MC ? 2 : 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], CTA2 ? 2 * Cfg::EPW : Cfg::EPW);
    }
    for (int s = 0; s < 2 * Cfg::EPW; ++s) ptx::mbar_init(&hfull[s], 1);
    ptx::fence_barrier_init();
    ptx::prefetch_tmap(&mA);
    ptx::prefetch_tmap(&mB);
  }
  if (warp == NP) {
    if constexpr (CTA2) {
      ptx::tmem_alloc2(tmem_holder, Cfg::TMEM_COLS);
      ptx::tmem_relinquish2();
    } else {
      ptx::tmem_alloc(tmem_holder, Cfg::TMEM_COLS);
      ptx::tmem_relinquish();
    }
  }
  ptx::tc_fence_before();
  if constexpr (CTA2) ptx::cluster_sync();
  else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  ptx::pdl_wait();  // everything above is local setup; the routing / operand data come after

  const int total_tiles = total_tiles_of<KIND, CTA2>(args);

  if (warp < NP) {
    // ============================================================ producers
    int stage = 0;
    uint32_t phase = 0;
    if constexpr (g4_kind<KIND>()) {
      // TMA gather4: lane p < 16 gathers K-rows 4p .. 4p+3 of each k-block (both 64-column chunks);
      // their gather indices run KPD k-blocks ahead in registers, as in the cp.async producer
      constexpr int KPD = SONIC_KPD;
      int ktok[KPD][4];
      const int p = lane;
      for (int tile = t_first; tile < total_tiles; tile += t_step) {
        const TileCoord tc = decode_tile<KIND, CTA2, MFAST>(args, tile, rank);
        const int n0 = tc.nt * BN + rank * BNL;
        const int gcol = Tr::a_gather ? ((tc.valid) ? tc.mt * GEMM_BM : 0) : n0;
#pragma unroll
        for (int u = 0; u < KPD; ++u)
#pragma unroll
          for (int j = 0; j < 4; ++j)
            ktok[u][j] = (p < 16 && u < tc.nkb) ? tok_of(args.row_token, tc.seg0 + u * GEMM_BK + 4 * p + j) : 0;
        for (int kb0 = 0; kb0 < tc.nkb; kb0 += KPD) {
#pragma unroll
          for (int u = 0; u < KPD; ++u) {
            const int kb = kb0 + u;
            if (kb >= tc.nkb) break;
            const int g0 = (int)clamp_tok(ktok[u][0]), g1 = (int)clamp_tok(ktok[u][1]);
            const int g2 = (int)clamp_tok(ktok[u][2]), g3 = (int)clamp_tok(ktok[u][3]);
            if (p < 16 && kb + KPD < tc.nkb) {
#pragma unroll
              for (int j = 0; j < 4; ++j) ktok[u][j] = tok_of(args.row_token, tc.seg0 + (kb + KPD) * GEMM_BK + 4 * p + j);
            }
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sA = smem + stage * STAGE_BYTES;
            uint8_t* sB = sA + A_BYTES;
            uint64_t* bar = &full[stage];
            const int krow0 = tc.seg0 + kb * GEMM_BK;
            if (lane == 0) {
              if (leader) ptx::mbar_arrive_expect_tx(bar, STAGE_BYTES * (CTA2 ? 2 : 1));
              if constexpr (KIND == K_DW2) {  // A' tile (MN-major): 64 rows x 128 M columns
                const int m0 = tc.valid ? tc.mt * GEMM_BM : 0;
                if constexpr (CTA2 && (SONIC_STREAM_EF & 2)) {
                  ptx::tma_load_2d_cg2_hint(sA, &mA, bar, m0, krow0, ptx::policy_evict_first());
                  ptx::tma_load_2d_cg2_hint(sA + 8192, &mA, bar, m0 + 64, krow0, ptx::policy_evict_first());
                } else {
                  tload2<CTA2>(sA, &mA, bar, m0, krow0);
                  tload2<CTA2>(sA + 8192, &mA, bar, m0 + 64, krow0);
                }
              } else {  // DW1: dH tile (MN-major): 64 rows x BNL columns
#pragma unroll
                for (int j = 0; j < BNL / 64; ++j) tload2<CTA2>(sB + j * 8192, &mB, bar, n0 + 64 * j, krow0);
              }
            }
            __syncwarp();
            if (p < 16) {
              constexpr int NCH = Tr::a_gather ? 2 : BNL / 64;
              uint8_t* gdst = (Tr::a_gather ? sA : sB) + p * 512;
              const CUtensorMap* gm = Tr::a_gather ? &mA : &mB;
#pragma unroll
              for (int jj = 0; jj < NCH; ++jj) {
                if constexpr (CTA2) ptx::tma_gather4_cg2(gdst + jj * 8192, gm, bar, gcol + 64 * jj, g0, g1, g2, g3);
                else ptx::tma_gather4(gdst + jj * 8192, gm, bar, gcol + 64 * jj, g0, g1, g2, g3);
              }
            }
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    } else if constexpr (!GATHER) {
      if (lane == 0) {
        for (int tile = t_first; tile < total_tiles; tile += t_step) {
          const TileCoord tc = decode_tile<KIND, CTA2, MFAST>(args, tile, rank);
          const int n0 = tc.nt * BN + rank * BNL;  // this CTA's B columns (rows)
          for (int kb = 0; kb < tc.nkb; ++kb) {
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sA = smem + stage * STAGE_BYTES;
            uint8_t* sB = sA + A_BYTES;
            uint64_t* bar = &full[stage];
            if (leader) ptx::mbar_arrive_expect_tx(bar, STAGE_BYTES * (CTA2 ? 2 : 1));
            if constexpr (MC)  // half of the shared A tile (64 rows, box map mD) into both pairs
              ptx::tma_load_2d_cg2_mc(sA + pidx * 8192, &mD, bar, kb * GEMM_BK, tc.row0 + 64 * pidx, smask);
            else
              tload2<CTA2>(sA, &mA, bar, kb * KBE, tc.row0);
            if constexpr (KIND == K_DOWN) {
#pragma unroll
              for (int j = 0; j < BNL / 64; ++j) tload3<CTA2>(sB + j * 8192, &mB, bar, n0 + 64 * j, kb * GEMM_BK, tc.e);
            } else {  // DXT / DXT8: K-major weights, one box of BNL rows
              tload3<CTA2>(sB, &mB, bar, kb * KBE, n0, tc.e);
            }
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    } else {
      const int pt = threadIdx.x;  // 0..32 NP - 1
      const int c = pt & 7;        // 16-byte chunk within a 128-byte row
      constexpr int RS = NP * 4;   // rows per pass (a multiple of 8: the swizzle phase is r0 & 7)
      constexpr int JM = GEMM_BM / RS, JK = GEMM_BK / RS;
      static_assert(RS % 8 == 0 && GEMM_BM % RS == 0 && GEMM_BK % RS == 0, "producer warp count");
      const uint64_t gpol = ptx::policy_evict_last();  // gathered rows are re-read by K experts' tiles
      const int r0 = pt >> 3;      // rows r0 + RS j
      const uint32_t sw = (uint32_t)((c ^ (r0 & 7)) << 4);
      // Gather indices are prefetched one tile (varlen-M) / one stage (varlen-K) ahead so the
      // dependent cp.async addresses never wait on a global load.
      int ntok[JM];
#ifdef SONIC_TIMING
      unsigned long long p_empty = 0, p_c0 = clock64();
#endif
      // varlen-K prefetch ring: KPD k-blocks of gather indices in flight.  The index loads share
      // the LSU queue with the producers' own outstanding cp.async gathers, so their effective
      // latency is the gathers' (often HBM) latency: the deeper the ring the better until the
      // registers run out (16: 4 indices x 16 k-blocks per thread, no spills)
      constexpr int KPD = Tr::vk ? SONIC_KPD : 1;
      constexpr int KU = Tr::vk ? KPD : 1;
      int ktok[KPD][JK];
      if constexpr (!Tr::vk) {
        if (t_first < total_tiles) {
          const TileCoord t0 = decode_tile<KIND, CTA2, MFAST>(args, t_first, rank);
#pragma unroll
          for (int j = 0; j < JM; ++j) ntok[j] = t0.valid ? tok_of(args.row_token, t0.row0 + r0 + RS * j) : 0;
        }
      }
      for (int tile = t_first; tile < total_tiles; tile += t_step) {
        const TileCoord tc = decode_tile<KIND, CTA2, MFAST>(args, tile, rank);
        const int n0 = tc.nt * BN + rank * BNL;
        const uint8_t* srcM[JM];  // byte addresses: a k-block is 128 bytes of a row (64 bf16 / 128 e4m3)
        if constexpr (!Tr::vk) {
#pragma unroll
          for (int j = 0; j < JM; ++j)
            srcM[j] = reinterpret_cast<const uint8_t*>(args.gsrc) + clamp_tok(ntok[j]) * args.gld * ESZ + c * 16;
          if (tile + t_step < total_tiles) {
            const TileCoord tn = decode_tile<KIND, CTA2, MFAST>(args, tile + t_step, rank);
#pragma unroll
            for (int j = 0; j < JM; ++j) ntok[j] = tn.valid ? tok_of(args.row_token, tn.row0 + r0 + RS * j) : 0;
          }
        } else {
#pragma unroll
          for (int u = 0; u < KPD; ++u)
#pragma unroll
            for (int j = 0; j < JK; ++j)
              ktok[u][j] = u < tc.nkb ? tok_of(args.row_token, tc.seg0 + u * GEMM_BK + r0 + RS * j) : 0;
        }
        // varlen-K A gather of a missing half: read column 0 (finite, never stored)
        const int acol0 = (Tr::a_gather && tc.valid) ? tc.mt * GEMM_BM : 0;
        // varlen-K: the k-block loop is unrolled by KPD so that ring slot u is a compile-time
        // register set: slot u is consumed for k-block kb and refilled for kb + KPD in place.
        for (int kb0 = 0; kb0 < tc.nkb; kb0 += KU) {
#pragma unroll
        for (int u = 0; u < KU; ++u) {
          const int kb = kb0 + u;
          if (kb >= tc.nkb) break;
          const __nv_bfloat16* srcK[JK];
          if constexpr (Tr::vk) {
            const int col0 = Tr::a_gather ? acol0 : n0;
#pragma unroll
            for (int j = 0; j < JK; ++j) srcK[j] = args.gsrc + clamp_tok(ktok[u][j]) * args.gld + col0 + c * 8;
            if constexpr (SONIC_L2PF > 0) {
              static_assert(SONIC_L2PF < KPD, "L2 prefetch reads the index ring");
              constexpr int NPF = Tr::a_gather ? 2 : BNL / 64;  // 128-byte lines per gathered row
              if (c < NPF && kb + SONIC_L2PF < tc.nkb) {
#pragma unroll
                for (int j = 0; j < JK; ++j)
                  ptx::prefetch_l2(args.gsrc + clamp_tok(ktok[(u + SONIC_L2PF) % KPD][j]) * args.gld + col0 + 64 * c);
              }
            }
            if (kb + KPD < tc.nkb) {
              const int krow1 = tc.seg0 + (kb + KPD) * GEMM_BK;
#pragma unroll
              for (int j = 0; j < JK; ++j) ktok[u][j] = tok_of(args.row_token, krow1 + r0 + RS * j);
            }
          }
#ifdef SONIC_TIMING
          unsigned long long cpe = clock64();
#endif
          ptx::mbar_wait(&empty[stage], phase ^ 1);
#ifdef SONIC_TIMING
          if (pt == 0) p_empty += clock64() - cpe;
#endif
          uint8_t* sA = smem + stage * STAGE_BYTES;
          uint8_t* sB = sA + A_BYTES;
          uint64_t* bar = &full[stage];
          if (pt == 0) {
            if (leader) ptx::mbar_arrive_expect_tx(bar, TMA_BYTES * (CTA2 ? 2 : 1));
            if constexpr (KIND == K_UP8) {  // one e4m3 box: 128 columns (128 B) x 128 K-rows, MN-major
              static_assert(BN == 256 && CTA2, "the e4m3 up-projection runs as 2-CTA pairs of 256 columns");
              tload3<true>(sB, &mB, bar, (rank ? args.n : 0) + tc.nt * (BN / 2), kb * 128, tc.e);
            } else if constexpr (KIND == K_UP) {
              constexpr int W = BN / 2;  // gate columns per tile; the up columns follow at +n
              if constexpr (W >= 64) {
                const int j0 = tc.nt * W;
                if constexpr (CTA2) {  // rank 0 holds the gate half of B, rank 1 the up half
                  const int cb = (rank ? args.n : 0) + j0;
#pragma unroll
                  for (int j = 0; j < W / 64; ++j) tload3<true>(sB + j * 8192, &mB, bar, cb + 64 * j, kb * GEMM_BK, tc.e);
                } else {
#pragma unroll
                  for (int j = 0; j < W / 64; ++j) {
                    tload3<false>(sB + j * 8192, &mB, bar, j0 + 64 * j, kb * GEMM_BK, tc.e);
                    tload3<false>(sB + (W / 64 + j) * 8192, &mB, bar, args.n + j0 + 64 * j, kb * GEMM_BK, tc.e);
                  }
                }
              } else {  // n == 32 (1-CTA only): one 64-column box holds [gate | up]
                tload3<CTA2>(sB, &mB, bar, 0, kb * GEMM_BK, tc.e);
              }
            } else if constexpr (KIND == K_DH) {
              tload3<CTA2>(sB, &mB, bar, kb * GEMM_BK, n0, tc.e);
            } else if constexpr (KIND == K_DW2) {  // A' tile (MN-major): 64 rows x 128 M columns
              const int krow0 = tc.seg0 + kb * GEMM_BK;
              const int m0 = tc.valid ? tc.mt * GEMM_BM : 0;
              if constexpr (MC) {  // one of the two 64-column boxes, into both pairs
                ptx::tma_load_2d_cg2_mc(sA + 8192 * pidx, &mA, bar, m0 + 64 * pidx, krow0, smask);
              } else if constexpr (CTA2 && (SONIC_STREAM_EF & 2)) {  // A' streamed evict-first: keep dO's rows in L2
                ptx::tma_load_2d_cg2_hint(sA, &mA, bar, m0, krow0, ptx::policy_evict_first());
                ptx::tma_load_2d_cg2_hint(sA + 8192, &mA, bar, m0 + 64, krow0, ptx::policy_evict_first());
              } else {
                tload2<CTA2>(sA, &mA, bar, m0, krow0);
                tload2<CTA2>(sA + 8192, &mA, bar, m0 + 64, krow0);
              }
            } else {  // DW1: dH tile (MN-major): 64 rows x BNL columns
              const int krow0 = tc.seg0 + kb * GEMM_BK;
              if constexpr (MC) {  // MFAST: both pairs hold the same B columns; one box each, into both
                static_assert(!MC || BNL == 128, "DW1 multicast splits the B half into two 64-column boxes");
                ptx::tma_load_2d_cg2_mc(sB + 8192 * pidx, &mB, bar, n0 + 64 * pidx, krow0, smask);
              } else {
#pragma unroll
                for (int j = 0; j < BNL / 64; ++j) {
                  if constexpr (CTA2 && (SONIC_STREAM_EF & 1))  // dH streamed evict-first: keep X's rows in L2
                    ptx::tma_load_2d_cg2_hint(sB + j * 8192, &mB, bar, n0 + 64 * j, krow0, ptx::policy_evict_first());
                  else
                    tload2<CTA2>(sB + j * 8192, &mB, bar, n0 + 64 * j, krow0);
                }
              }
            }
          }
          if constexpr (!Tr::vk) {  // A: 128 gathered rows x 64 K (K-major)
            if constexpr (SONIC_L2PF > 0) {
              if (c == 0 && kb + SONIC_L2PF < tc.nkb) {
#pragma unroll
                for (int j = 0; j < JM; ++j) ptx::prefetch_l2(srcM[j] + (kb + SONIC_L2PF) * 128);
              }
            }
            const uint32_t dst = ptx::smem_u32(sA) + r0 * 128 + sw;
#pragma unroll
            for (int j = 0; j < JM; ++j) gather16(dst + j * RS * 128, srcM[j] + kb * 128, gpol);
          } else {  // 64 gathered K-rows x (128 | BNL) MN-columns (MN-major)
            constexpr int NCH = Tr::a_gather ? 2 : BNL / 64;
            const uint32_t dst = ptx::smem_u32(Tr::a_gather ? sA : sB) + r0 * 128 + sw;
#pragma unroll
            for (int j = 0; j < JK; ++j)
#pragma unroll
              for (int jj = 0; jj < NCH; ++jj) gather16(dst + jj * 8192 + j * RS * 128, srcK[j] + 64 * jj, gpol);
          }
          ptx::cp_async_mbar_arrive(bar);  // arrives on this CTA's barrier when the copies land
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        }
      }
#ifdef SONIC_TIMING
      if (args.dbg && pt == 0) {
        atomicAdd(args.dbg + 6, p_empty);
        atomicAdd(args.dbg + 7, clock64() - p_c0);
      }
#endif
    }
  } else if (warp == NP) {
    // ============================================================ MMA issuer (leader) / relay (peer)
    if (lane == 0 && leader) {
      constexpr uint32_t idesc = F8 ? ptx::make_idesc_e4m3(MMA_M, BN, Tr::a_mn ? 1 : 0, Tr::b_mn ? 1 : 0)
                                    : ptx::make_idesc(MMA_M, BN, Tr::a_mn ? 1 : 0, Tr::b_mn ? 1 : 0);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
#ifdef SONIC_TIMING
      unsigned long long c_te = 0, c_full = 0, c0 = clock64();
#endif
      for (int tile = t_first; tile < total_tiles; tile += t_step) {
        const TileCoord tc = decode_tile<KIND, CTA2, MFAST>(args, tile, 0);
#ifdef SONIC_TIMING
        unsigned long long ca = clock64();
#endif
        if constexpr (CTA2) ptx::mbar_wait_cluster(&tempty[acc], acc_phase ^ 1);
        else ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
#ifdef SONIC_TIMING
        c_te += clock64() - ca;
#endif
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < tc.nkb; ++kb) {
#ifdef SONIC_TIMING
          unsigned long long cb = clock64();
#endif
          if constexpr (CTA2) ptx::mbar_wait_cluster(&full[stage], phase);
          else ptx::mbar_wait(&full[stage], phase);
#ifdef SONIC_TIMING
          c_full += clock64() - cb;
#endif
          // cp.async (generic proxy) data consumed by tcgen05.mma (async proxy)
          if constexpr (GATHER && !SONIC_EXP_NOFENCE) ptx::fence_proxy_async_smem();  // (ablation: SONIC_EXP_NOFENCE, unsafe)
          ptx::tc_fence_after();
          const uint32_t a_base = ptx::smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t b_base = a_base + A_BYTES;
#pragma unroll
          for (int k = 0; k < GEMM_BK / 16; ++k) {
            const uint64_t ad = Tr::a_mn ? ptx::make_sdesc(a_base + k * 2048, 8192, 1024)
                                         : ptx::make_sdesc(a_base + k * 32, 16, 1024);
            // MN-major B: one MMA step is 16 (bf16) or 32 (e4m3) K-rows of 128 bytes; a 128-byte MN
            // chunk spans 64 (bf16) K-rows x ... or, for e4m3, the whole 128-row k-block
            const uint64_t bd = Tr::b_mn ? (F8 ? ptx::make_sdesc(b_base + k * 4096, 16384, 1024)
                                               : ptx::make_sdesc(b_base + k * 2048, 8192, 1024))
                                         : ptx::make_sdesc(b_base + k * 32, 16, 1024);
            if constexpr (F8) {
              if constexpr (CTA2) ptx::mma_f8_cg2(d_tmem, ad, bd, idesc, (kb | k) != 0);
              else ptx::mma_f8(d_tmem, ad, bd, idesc, (kb | k) != 0);
            } else {
              if constexpr (CTA2) ptx::mma_bf16_cg2(d_tmem, ad, bd, idesc, (kb | k) != 0);
              else ptx::mma_bf16(d_tmem, ad, bd, idesc, (kb | k) != 0);
            }
          }
          if constexpr (CTA2) ptx::mma_commit_mc(&empty[stage], MC ? (uint16_t)0xF : pmask);
          else ptx::mma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if constexpr (CTA2) ptx::mma_commit_mc(&tfull[acc], pmask);
        else ptx::mma_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
#ifdef SONIC_TIMING
      if (args.dbg) {
        atomicAdd(args.dbg + 0, clock64() - c0);
        atomicAdd(args.dbg + 1, c_te);
        atomicAdd(args.dbg + 2, c_full);
        atomicAdd(args.dbg + 5, 1ull);
      }
#endif
    } else if (lane == 0 && CTA2 && GATHER) {
      // relay: forward this CTA's cp.async completion (local barrier) to the leader's barrier
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = t_first; tile < total_tiles; tile += t_step) {
        const TileCoord tc = decode_tile<KIND, CTA2, MFAST>(args, tile, rank);
        for (int kb = 0; kb < tc.nkb; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::fence_proxy_async_smem();
          ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&full[stage]), lead));
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp < NP + 1 + Cfg::EPW) {
    // ============================================================ epilogue (Cfg::EPW warps)
    const int ew = warp - NP - 1;
    const int q = warp & 3;         // TMEM lane quarter this warp may access
    const int half = ew / 4;        // which interleaved 64-column chunks (32 for fp32) it handles
    StoreQ<Cfg::NB> sq{stg + ew * Cfg::NB * STG_BYTES, 0};
    int acc = 0;
    uint32_t acc_phase = 0;
    const uint32_t tempty_leader = CTA2 ? ptx::mapa(ptx::smem_u32(&tempty[0]), lead) : 0u;
    // DH: each epilogue warp TMA-loads its own 32 rows of H (BN gate + BN up columns) for its
    // next tile into a private buffer; dH is computed in place there and TMA-stored from it.
    uint8_t* hb = hbuf + ew * Cfg::HBUF_WARP;
    uint32_t hphase = 0;
    auto h_issue = [&](int t) {
      if constexpr (HTMA) {
        if (lane == 0) {
          const TileCoord th = decode_tile<KIND, CTA2, MFAST>(args, t, rank);
          if constexpr (BN >= 64) {
            // this warp's chunks c = half, half + Cfg::EPH, ... (local index lc): gate box at
            // lc * 4 KB, up box at (NLC + lc) * 4 KB
            constexpr int NLC = (BN / 64 + Cfg::EPH - 1) / Cfg::EPH;
            int nb = 0;
#pragma unroll
            for (int c = half, lc = 0; c < BN / 64; c += Cfg::EPH, ++lc) nb += 2;
            ptx::mbar_arrive_expect_tx(&hfull[ew], nb * STG_BYTES);
#pragma unroll
            for (int c = half, lc = 0; c < BN / 64; c += Cfg::EPH, ++lc) {
              ptx::tma_load_2d(hb + lc * STG_BYTES, &mD, &hfull[ew], th.nt * BN + 64 * c, th.row0 + 32 * q);
              ptx::tma_load_2d(hb + (NLC + lc) * STG_BYTES, &mD, &hfull[ew], args.n + th.nt * BN + 64 * c,
                               th.row0 + 32 * q);
            }
            if (nb == 0) ptx::mbar_arrive(&hfull[ew]);  // no chunk for this warp: complete the phase
          } else {  // n == 32: one box [gate | up], handled by half 0
            if (half == 0) {
              ptx::mbar_arrive_expect_tx(&hfull[ew], STG_BYTES);
              ptx::tma_load_2d(hb, &mD, &hfull[ew], 0, th.row0 + 32 * q);
            } else {
              ptx::mbar_arrive(&hfull[ew]);
            }
          }
        }
      }
    };
    if constexpr (HTMA) {
      if (t_first < total_tiles) h_issue(t_first);
    }
    // HRING (DH, BN = 256): chunk c of a tile = H columns [64c, 64c + 64) of gate and of up, for
    // this warp's 32 rows.  Chunks are loaded two ahead, in (tile, chunk) order, into the slot the
    // consumer has just released; a slot is released once the dH stores out of it have read it.
    constexpr int HR_NCH = BN / 64;
    int hr_tile = t_first, hr_c = 0, hr_slot = 0;
    uint32_t hr_phase = 0;  // bit s: parity of slot s
    auto hr_load = [&](int slot) {
      if constexpr (HRING) {
        if (hr_tile >= total_tiles) return;
        if (lane == 0) {
          const TileCoord th = decode_tile<KIND, CTA2, MFAST>(args, hr_tile, rank);
          uint64_t* b = &hfull[2 * ew + slot];
          uint8_t* dst = hb + slot * 2 * STG_BYTES;
          if (th.valid) {
            ptx::mbar_arrive_expect_tx(b, 2 * STG_BYTES);
            ptx::tma_load_2d(dst, &mD, b, th.nt * BN + 64 * hr_c, th.row0 + 32 * q);
            ptx::tma_load_2d(dst + STG_BYTES, &mD, b, args.n + th.nt * BN + 64 * hr_c, th.row0 + 32 * q);
          } else {
            ptx::mbar_arrive(b);  // missing half of a pair: an empty chunk keeps the ring in step
          }
        }
        if (++hr_c == HR_NCH) {
          hr_c = 0;
          hr_tile += t_step;
        }
      }
    };
    auto hr_wait = [&]() -> int {
      const int sl = hr_slot;
      ptx::mbar_wait(&hfull[2 * ew + sl], (hr_phase >> sl) & 1u);
      hr_phase ^= 1u << sl;
      hr_slot ^= 1;
      return sl;
    };
    if constexpr (HRING) {
      hr_load(0);
      hr_load(1);
    }
#ifdef SONIC_TIMING
    unsigned long long c_tf = 0, c_epi = 0;
#endif
    for (int tile = t_first; tile < total_tiles; tile += t_step) {
      const TileCoord tc = decode_tile<KIND, CTA2, MFAST>(args, tile, rank);
      const int wrow = tc.row0 + 32 * q;  // first grouped row of this warp's slab
      const int row = wrow + lane;        // this thread's grouped row (varlen-M)
      const bool has_next = tile + t_step < total_tiles;
#ifdef SONIC_TIMING
      unsigned long long cx = clock64();
#endif
      if constexpr (CTA2) ptx::mbar_wait_cluster(&tfull[acc], acc_phase);
      else ptx::mbar_wait(&tfull[acc], acc_phase);
#ifdef SONIC_TIMING
      unsigned long long cy = clock64();
      c_tf += cy - cx;
#endif
      ptx::tc_fence_after();
      const uint32_t t_acc = tmem_base + ((uint32_t)(32 * q) << 16) + acc * BN;

#ifdef SONIC_EXPERIMENT_NO_EPI
      constexpr bool no_epi = true;  // ablation: mainloop only, nothing stored
#else
      constexpr bool no_epi = false;
#endif
      if (!tc.valid || no_epi) {
        // missing half of a pair: nothing to store (keep the H-buffer protocol going)
        if constexpr (HRING) {
          for (int c = 0; c < HR_NCH; ++c) hr_load(hr_wait());
        }
        if constexpr (HTMA) {
          ptx::mbar_wait(&hfull[ew], hphase);
          hphase ^= 1;
          if (has_next) h_issue(tile + t_step);
        }
      } else if constexpr (KIND == K_UP || KIND == K_UP8) {
        constexpr int W = BN / 2;
        // UP8: H = acc * sx[token] * sw[e][column] (the scales of the e4m3 operands, NEXT-4)
        float sxr = 1.f;
        if constexpr (F8) sxr = __ldg(args.sx + clamp_tok(__ldg(args.row_token + row)));
        if constexpr (W >= 64) {
#pragma unroll 1
          for (int c = 64 * half; c < W; c += 64 * Cfg::EPH) {
            const int col = tc.nt * W + c;
            float swg[2] = {1.f, 1.f}, swu[2] = {1.f, 1.f};  // lane j holds the scales of columns j, 32 + j
            if constexpr (F8) {
              const float* swe = args.sw + (size_t)tc.e * 2 * args.n;
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                swg[h] = __ldg(swe + col + 32 * h + lane);
                swu[h] = __ldg(swe + args.n + col + 32 * h + lane);
              }
            }
            sq.template acquire<1>(lane);  // the next two ring slots are both free
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
                  float vg = __uint_as_float(g[8 * q8 + i]), vu = __uint_as_float(u[8 * q8 + i]);
                  if constexpr (F8) {
                    vg *= sxr * __shfl_sync(0xffffffffu, swg[h], 8 * q8 + i);
                    vu *= sxr * __shfl_sync(0xffffffffu, swu[h], 8 * q8 + i);
                  }
                  hg[i] = bf16r(vg);
                  hu[i] = bf16r(vu);
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
        } else if (half == 0) {  // n == 32: accumulator columns are [gate 32 | up 32] = the whole H row
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
      } else if constexpr ((KIND == K_DOWN || KIND == K_DXT || KIND == K_DXT8) && SONIC_EPI_PIPE) {
        // TMEM loads run one 64-column chunk ahead of the convert + store of the current chunk, so
        // the tcgen05.ld latency is paid once per tile instead of twice per chunk.
        float gate = 1.f;
        if constexpr (KIND == K_DOWN) gate = __ldg(args.row_gate + row);
        if constexpr (KIND == K_DXT8) gate = __ldg(args.sx + row);  // the row scale of the e4m3 dH'
        constexpr int NCH = BN / (64 * Cfg::EPH);
        static_assert(wide_g<KIND>() == 1 || Cfg::EPH == 1, "wide stores: one warp per TMEM lane quarter");
        int wslot = 0;
        uint32_t r[2][2][32];
        auto col_of = [&](int j) { return 64 * half + j * 64 * Cfg::EPH; };
        auto live = [&](int j) { return j < NCH && tc.nt * BN + col_of(j) < args.N_dim; };
        if (live(0)) {
          ptx::tmem_ld32(t_acc + col_of(0), r[0][0]);
          ptx::tmem_ld32(t_acc + col_of(0) + 32, r[0][1]);
          ptx::tmem_ld_wait();
          ptx::tmem_regs_ready(r[0][0]);
          ptx::tmem_regs_ready(r[0][1]);
        }
#pragma unroll
        for (int j = 0; j < NCH; ++j) {
          if (!live(j)) break;
          const int sl = j & 1;
          if (live(j + 1)) {
            ptx::tmem_ld32(t_acc + col_of(j + 1), r[sl ^ 1][0]);
            ptx::tmem_ld32(t_acc + col_of(j + 1) + 32, r[sl ^ 1][1]);
          }
          constexpr int G = wide_g<KIND>();
          constexpr bool WIDE = G > 1 && NCH % G == 0;  // a slot never spans two N tiles
          int i, slot = 0;
          if (WIDE && args.wide) {  // chunk j goes to buffer j % G of the current slot
            if (j % G == 0) wslot = sq.template acquire_slot<G>(lane);
            slot = wslot;
            i = slot * G + j % G;
          } else {
            i = sq.acquire(lane);
          }
          const uint32_t b = sq.addr(i);
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int q8 = 0; q8 < 4; ++q8) {
              const uint32_t* v = r[sl][h] + 8 * q8;
              ptx::st_shared_v4(b + swz(lane, 4 * h + q8),
                                ptx::pack_bf16(gate * __uint_as_float(v[0]), gate * __uint_as_float(v[1])),
                                ptx::pack_bf16(gate * __uint_as_float(v[2]), gate * __uint_as_float(v[3])),
                                ptx::pack_bf16(gate * __uint_as_float(v[4]), gate * __uint_as_float(v[5])),
                                ptx::pack_bf16(gate * __uint_as_float(v[6]), gate * __uint_as_float(v[7])));
            }
          if (WIDE && args.wide) {
            if (j % G == G - 1 || !live(j + 1))  // clipped at the last column block by the map
              sq.template issue_slot<G>(lane, slot, &mC0, 0, wrow, (tc.nt * BN + col_of(j - j % G)) / 64);
          } else {
            sq.issue(lane, i, &mC0, tc.nt * BN + col_of(j), wrow);
          }
          if (live(j + 1)) {
            ptx::tmem_ld_wait();
            ptx::tmem_regs_ready(r[sl ^ 1][0]);
            ptx::tmem_regs_ready(r[sl ^ 1][1]);
          }
        }
      } else if constexpr (KIND == K_DOWN || KIND == K_DXT || KIND == K_DXT8) {
        float gate = 1.f;
        if constexpr (KIND == K_DOWN) gate = __ldg(args.row_gate + row);
        if constexpr (KIND == K_DXT8) gate = __ldg(args.sx + row);
#pragma unroll 1
        for (int c = 64 * half; c < BN; c += 64 * Cfg::EPH) {
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
              if constexpr (SONIC_EXP_EPI == 1) {
                if ((v[0] ^ v[3] ^ v[5] ^ v[7]) == 0x7f7f7f7fu) args.dS[0] = 1.f;
                continue;
              }
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
        float ds = 0.f;
        if constexpr (HRING) {
#pragma unroll 1
          for (int c = 0; c < HR_NCH; ++c) {
            const int sl = hr_wait();
            const int col = tc.nt * BN + 64 * c;
            uint8_t* gbp = hb + sl * 2 * STG_BYTES;
            const uint32_t gb = ptx::smem_u32(gbp);  // H gate -> dH gate (in place) -> A'
            const uint32_t ub = gb + STG_BYTES;      // H up   -> dH up (in place)
            uint32_t pa[2][4][4];                     // A' = s A for this chunk, bf16 pairs
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
                    const float sl_ = gg * sg;
                    const float A = sl_ * uu;
                    const float dA = s * dap;
                    dg2[k] = dA * uu * sg * fmaf(gg, 1.f - sg, 1.f);
                    du2[k] = dA * sl_;
                    ap2[k] = s * A;
                    ds = fmaf(dap, A, ds);
                  }
                  pg[i] = ptx::pack_bf16(dg2[0], dg2[1]);
                  pu[i] = ptx::pack_bf16(du2[0], du2[1]);
                  pa[h][q8][i] = ptx::pack_bf16(ap2[0], ap2[1]);
                }
                ptx::st_shared_v4(gb + swz(lane, 4 * h + q8), pg[0], pg[1], pg[2], pg[3]);
                ptx::st_shared_v4(ub + swz(lane, 4 * h + q8), pu[0], pu[1], pu[2], pu[3]);
              }
            }
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              ptx::tma_store_2d(&mC0, gbp, col, wrow);                  // dH gate
              ptx::tma_store_2d(&mC0, gbp + STG_BYTES, n + col, wrow);  // dH up
              ptx::bulk_commit();
              ptx::bulk_wait_read<0>();  // the gate slot is free for A'
            }
            __syncwarp();
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int q8 = 0; q8 < 4; ++q8)
                ptx::st_shared_v4(gb + swz(lane, 4 * h + q8), pa[h][q8][0], pa[h][q8][1], pa[h][q8][2], pa[h][q8][3]);
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              ptx::tma_store_2d(&mC1, gbp, col, wrow);  // A' = s A
              ptx::bulk_commit();
              ptx::bulk_wait_read<0>();  // the slot is free for the next H chunk
            }
            __syncwarp();
            hr_load(sl);
          }
        } else if constexpr (BN >= 64) {
          ptx::mbar_wait(&hfull[ew], hphase);
          hphase ^= 1;
#pragma unroll 1
          for (int c = half, lc = 0; c < BN / 64; c += Cfg::EPH, ++lc) {
            constexpr int NLC = (BN / 64 + Cfg::EPH - 1) / Cfg::EPH;
            const int col = tc.nt * BN + 64 * c;
            const uint32_t gb = ptx::smem_u32(hb + lc * STG_BYTES);          // H gate -> dH gate
            const uint32_t ub = ptx::smem_u32(hb + (NLC + lc) * STG_BYTES);  // H up   -> dH up
            const uint32_t ab = sq.addr(lc & 1);                              // A' staging
            sq.template wait_reads<3>(lane);  // the A' store issued from this buffer 2 chunks ago has read it
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
              ptx::tma_store_2d(&mC0, hb + lc * STG_BYTES, col, wrow);                     // dH gate
              ptx::bulk_commit();
              ptx::tma_store_2d(&mC0, hb + (NLC + lc) * STG_BYTES, n + col, wrow);         // dH up
              ptx::bulk_commit();
              ptx::tma_store_2d(&mC1, sq.base + (lc & 1) * STG_BYTES, col, wrow);          // A' = s A
              ptx::bulk_commit();
            }
          }
          if (has_next) {
            sq.template wait_reads<1>(lane);  // every dH store out of the H buffer has read it
            h_issue(tile + t_step);
          }
        } else if (half != 0) {  // n == 32: the whole tile belongs to half 0
          ptx::mbar_wait(&hfull[ew], hphase);
          hphase ^= 1;
          if (has_next) h_issue(tile + t_step);
        } else {  // n == 32, BN == 32: one 64-column H box holds the whole row [gate 32 | up 32]
          ptx::mbar_wait(&hfull[ew], hphase);
          hphase ^= 1;
          const uint32_t hbs = ptx::smem_u32(hb);
          uint32_t r[32];
          ptx::tmem_ld32(t_acc, r);
          uint4 hg4[4], hu4[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            hg4[i] = ptx::ld_shared_v4(hbs + swz(lane, i));
            hu4[i] = ptx::ld_shared_v4(hbs + swz(lane, 4 + i));
          }
          ptx::tmem_ld_wait();
          const __nv_bfloat16* hgp = reinterpret_cast<const __nv_bfloat16*>(hg4);
          const __nv_bfloat16* hup = reinterpret_cast<const __nv_bfloat16*>(hu4);
          const int ia = sq.acquire(lane);
          const uint32_t ab = sq.addr(ia);
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
            ptx::st_shared_v4(hbs + swz(lane, q8), pg[0], pg[1], pg[2], pg[3]);
            ptx::st_shared_v4(hbs + swz(lane, 4 + q8), pu[0], pu[1], pu[2], pu[3]);
            ptx::st_shared_v4(ab + swz(lane, q8), pa[0], pa[1], pa[2], pa[3]);
            ptx::st_shared_v4(ab + swz(lane, 4 + q8), 0u, 0u, 0u, 0u);
          }
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            ptx::tma_store_2d(&mC0, hb, 0, wrow);  // dH = [d gate | d up]
            ptx::bulk_commit();
          }
          sq.issue(lane, ia, &mC1, 0, wrow);  // A' (columns >= n clipped by the tensor map)
          if (has_next) {
            sq.template wait_reads<1>(lane);  // the dH store out of the H buffer has read it
            h_issue(tile + t_step);
          }
        }
        if constexpr (Cfg::EPH == 2) {  // combine the two halves' partial dS of each row
          const uint32_t bar_id = 1 + q;     // named barrier per lane quarter (64 threads)
          if (half == 1) ds_xchg[32 * q + lane] = ds;
          asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
          if (half == 0) ds += ds_xchg[32 * q + lane];
          asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
        }
        if (half == 0) {
          if (__ldg(args.row_token + row) < 0) ds = 0.f;
          if (args.n_tiles == 1)
            args.dS[row] = ds;
          else
            args.dS[(long long)tc.nt * args.rows_max + row] = ds;
        }
      } else {  // K_DW2 / K_DW1: fp32 weight gradient tile [128 x BN] of expert e
        const int m0 = tc.mt * GEMM_BM + 32 * q;
        // accumulate (dW += tile, TMA reduce-add): an expert with no rows adds nothing
        if (args.dw_bf16 && m0 < args.M_dim) {  // bf16 dW: 64 columns (128 B) per staging buffer
#pragma unroll 1
          for (int c = 64 * half; c < BN; c += 64 * Cfg::EPH) {
            if (tc.nt * BN + c >= args.N_dim) break;
            const int i = sq.acquire(lane);
            const uint32_t b = sq.addr(i);
            if (tc.nkb > 0) {
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                uint32_t r[32];
                ptx::tmem_ld32(t_acc + c + 32 * h, r);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int q8 = 0; q8 < 4; ++q8) {
                  const uint32_t* v = r + 8 * q8;
                  ptx::st_shared_v4(b + swz(lane, 4 * h + q8),
                                    ptx::pack_bf16(__uint_as_float(v[0]), __uint_as_float(v[1])),
                                    ptx::pack_bf16(__uint_as_float(v[2]), __uint_as_float(v[3])),
                                    ptx::pack_bf16(__uint_as_float(v[4]), __uint_as_float(v[5])),
                                    ptx::pack_bf16(__uint_as_float(v[6]), __uint_as_float(v[7])));
                }
              }
            } else {
#pragma unroll
              for (int ch = 0; ch < 8; ++ch) ptx::st_shared_v4(b + swz(lane, ch), 0u, 0u, 0u, 0u);
            }
            sq.issue3d(lane, i, &mC0, tc.nt * BN + c, m0, tc.e, false);
          }
        } else if (m0 < args.M_dim && !(args.accumulate && tc.nkb == 0)) {
#pragma unroll 1
          for (int c = 32 * half; c < BN; c += 32 * Cfg::EPH) {
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
            sq.issue3d(lane, i, &mC0, tc.nt * BN + c, m0, tc.e, args.accumulate != 0);
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CTA2) {
          if (leader) ptx::mbar_arrive(&tempty[acc]);
          else ptx::mbar_arrive_cluster(tempty_leader + acc * 8);
        } else {
          ptx::mbar_arrive(&tempty[acc]);
        }
      }
#ifdef SONIC_TIMING
      c_epi += clock64() - cy;
#endif
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
#ifdef SONIC_TIMING
    if (args.dbg && lane == 0 && ew == 0) {
      atomicAdd(args.dbg + 3, c_tf);
      atomicAdd(args.dbg + 4, c_epi);
    }
#endif
    if (lane == 0) ptx::bulk_wait<0>();
    __syncwarp();
  } else {
    // ============================================================ fused dX aggregation (SONIC_AGG_FUSE)
    // dX_t = sum of the token's dX~ rows in CSR (expert-ascending) order, fp32: exactly k_aggregate's
    // arithmetic (Alg. 5).  Work items are (token, column chunk, row), in that order;
    // item i lives in ring slot i % NS (parity (i / NS) & 1).  Lane k bulk-copies row k of the chunk
    // being issued; the row lists are loaded two tokens ahead so no issue waits on an index load;
    // the warp sums each (token, chunk) out of shared memory and stores dX with 16-byte stores.
    if constexpr (agg_warps<KIND>() > 0) {
      const long long ntok = args.agg_t1 - args.agg_t0;
      const long long per = ntok > 0 ? (ntok + gridDim.x - 1) / gridDim.x : 0;
      const long long tb = args.agg_t0 + (long long)blockIdx.x * per;
      const long long te = min(args.agg_t1, tb + per);
      if (tb < te) {
        uint8_t* abase = reinterpret_cast<uint8_t*>(full) + 1024;
        uint64_t* abar = reinterpret_cast<uint64_t*>(abase);  // [32]
        int* tok_nr = reinterpret_cast<int*>(abase + 256);    // [64] per token (t - tb) & 63
        int* tok_r0 = tok_nr + 64;                            // [64]
        const uint32_t aslot = ptx::smem_u32(abase + 1024);
        const int dd = args.agg_d;
        const int CC = dd < AGG_CHUNK ? dd : AGG_CHUNK;  // columns per chunk
        const int nch = (dd + CC - 1) / CC;
        const uint32_t slot_b = (uint32_t)CC * 2;
        const int NS = min(32, (int)(SONIC_AGG_RING / slot_b));
        const __nv_bfloat16* src = args.agg_src;
        if (lane == 0) {
          for (int i = 0; i < NS; ++i) ptx::mbar_init(&abar[i], 1);
          ptx::fence_barrier_init();
        }
        // row-list pipeline: (inr, irow) = token ti being issued, (nnr, nrow) = ti + 1, rpc = rowptr of ti + 2
        auto rp_load = [&](long long t) { return (lane < 2 && t + lane <= te) ? __ldg(args.agg_rowptr + t + lane) : 0; };
        auto list_of = [&](long long t, int rp, int& nr, int& row, int& r0) {
          r0 = __shfl_sync(0xffffffffu, rp, 0);
          nr = t < te ? __shfl_sync(0xffffffffu, rp, 1) - r0 : 0;
          row = (lane < nr && lane < 32) ? __ldg(args.agg_rows + r0 + lane) : 0;
        };
        long long ti = tb;
        int ic = 0, ni = 0, nc = 0;
        int inr, irow, ir0, nnr, nrow, nr0;
        list_of(tb, rp_load(tb), inr, irow, ir0);
        list_of(tb + 1, rp_load(tb + 1), nnr, nrow, nr0);
        int rpc = rp_load(tb + 2);
        if (lane == 0) { tok_nr[0] = inr; tok_r0[0] = ir0; }
        auto advance = [&]() {
          ++ti;
          ic = 0;
          inr = nnr; irow = nrow; ir0 = nr0;
          list_of(ti + 1, rpc, nnr, nrow, nr0);
          rpc = rp_load(ti + 2);
          if (lane == 0 && ti < te) { tok_nr[(ti - tb) & 63] = inr; tok_r0[(ti - tb) & 63] = ir0; }
        };
        long long t = tb;  // consumer token
#ifdef SONIC_TIMING
        unsigned long long ag_wait = 0, ag_c0 = clock64();
#endif
        auto issue = [&]() {
          while (ti < te && ti - t < 48) {
            if (inr == 0 || inr > NS) {  // no rows / summed straight from global memory
              advance();
              continue;
            }
            if (ni + inr > nc + NS) break;  // not enough free slots for this chunk's rows
            if (lane < inr) {
              const int sidx = (ni + lane) % NS;
              const int cols = min(CC, dd - ic * CC);
              ptx::mbar_arrive_expect_tx(&abar[sidx], (uint32_t)cols * 2);
              ptx::bulk_g2s(aslot + sidx * slot_b, src + (long long)irow * dd + (long long)ic * CC, (uint32_t)cols * 2,
                            &abar[sidx]);
            }
            ni += inr;
            if (++ic == nch) advance();
          }
        };
        __syncwarp();
        for (; t < te; ++t) {
          for (int c = 0; c < nch; ++c) {
            issue();
            __syncwarp();
            const int nr = tok_nr[(t - tb) & 63], r0 = tok_r0[(t - tb) & 63];
            const int cols = min(CC, dd - c * CC);
            uint4* dst = reinterpret_cast<uint4*>(args.agg_dst + t * dd + (long long)c * CC);
            if (nr > NS) {  // more rows than slots (token rounding / expert choice outliers)
              const uint4* sv = reinterpret_cast<const uint4*>(src);
              for (int v = lane; v < cols / 8; v += 32) {
                float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                for (int k = 0; k < nr; ++k)
                  acc8_bf16(a, ptx::ld_nc_v4(sv + ((long long)__ldg(args.agg_rows + r0 + k) * dd + (long long)c * CC) / 8 + v));
                dst[v] = pack8_bf16(a);
              }
              continue;
            }
#ifdef SONIC_TIMING
            unsigned long long cw0 = clock64();
#endif
            for (int k = 0; k < nr; ++k) ptx::mbar_wait(&abar[(nc + k) % NS], (uint32_t)((nc + k) / NS) & 1u);
#ifdef SONIC_TIMING
            ag_wait += clock64() - cw0;
#endif
            if (nr == 8) {  // top-8 routing: all eight row loads in flight, then the in-order sum
              uint32_t sb[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) sb[u] = aslot + ((nc + u) % NS) * slot_b;
              for (int v = lane; v < cols / 8; v += 32) {
                float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                uint4 x[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) x[u] = ptx::ld_shared_v4(sb[u] + v * 16);
#pragma unroll
                for (int u = 0; u < 8; ++u) acc8_bf16(a, x[u]);
                dst[v] = pack8_bf16(a);
              }
            } else {
              for (int v = lane; v < cols / 8; v += 32) {
                float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                for (int k = 0; k < nr; ++k) acc8_bf16(a, ptx::ld_shared_v4(aslot + ((nc + k) % NS) * slot_b + v * 16));
                dst[v] = pack8_bf16(a);
              }
            }
            nc += nr;
            __syncwarp();  // every lane's reads of these slots are done before they are refilled
            ptx::fence_proxy_async_smem();
          }
        }
#ifdef SONIC_TIMING
        if (args.dbg && lane == 0) {
          atomicAdd(args.dbg + 8, clock64() - ag_c0);
          atomicAdd(args.dbg + 9, ag_wait);
          atomicAdd(args.dbg + 10, (unsigned long long)(te - tb));
        }
#endif
      }
    }
  }

  ptx::tc_fence_before();
  if constexpr (CTA2) ptx::cluster_sync();
  else __syncthreads();
  if (warp == NP) {
    ptx::tc_fence_after();
    if constexpr (CTA2) ptx::tmem_dealloc2(tmem_base, Cfg::TMEM_COLS);
    else ptx::tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

}  // namespace sonic
