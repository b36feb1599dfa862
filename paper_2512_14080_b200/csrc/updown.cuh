// updown.cuh -- the forward's up-projection and down-projection fused into one persistent 2-CTA
// tcgen05 kernel (NEXT-1): A = SwiGLU(H) never leaves the SM.
//
// Per 256-row pair tile of one expert e (two 128-row tiles, one per CTA of the pair):
//   U jobs j = 0 .. n/128-1   H[:, 128j:+128 | n+128j:+128] = Gather(X) W1_e[:, gate j | up j]
//                             (M = 256, N = 256, K = d; the token gather fused into the operand
//                             load); epilogue: H (bf16, the cached activation) by
//                             TMA store, and A = silu(gate) up (from the bf16-rounded H, as the
//                             backward recomputes it) written into this CTA's A buffer in smem;
//   D jobs i = 0 .. d/BND-1   Y[:, BND i:+BND] = g * (A W2_e[:, BND i:+BND]) (M = 256, N = BND,
//                             K = n), A read straight from the A buffer; epilogue: gate scale
//                             (Q2), bf16, TMA store of Y for the aggregation.
// This is Alg. 2's up-proj / down-proj pair with the A round trip through HBM removed:
// 2 R n bytes written and read back (Eq. 4 accounting; the cached-set minimisation of
// sec. 3.2, keeps only X, H and the metadata for the backward).
//
// Pipeline (one CTA pair per 2 SMs, persistent over the pair tiles; warp roles as gemm.cuh):
//   producers  4 warps: U k-blocks: 128 threads cp.async the gathered X rows (K-major, 128B
//              swizzle) + one thread TMA-loads this CTA's half of the W1 columns; D k-blocks: one
//              thread TMA-loads this CTA's half of the W2 N-tile (the A operand is resident);
//   MMA        leader's single thread; the job sequence U_0 .. U_{NU-1}, D_0 .. D_{ND-1} alternates
//              the two 256-column TMEM accumulator slots (8 jobs per tile at 7B: even, so every tile
//              starts on slot 0).  D_0's k-block pair 2j waits on aready[j] (both CTAs' epilogues have
//              written A columns [128j, 128j+128));
//   epilogue   4 warps, one TMEM lane quarter each.  The A buffer is rewritten by the next tile's U
//              epilogues only after that U job's accumulator is full, i.e. after every earlier MMA of
//              this thread -- the D MMAs that read A -- has completed (tcgen05.commit order).
// Shapes: n in {128, 256} (A buffer 128 x n bf16 = 32 / 64 KB per CTA), d % 128 == 0.  Other shapes
// run the separate up / down kernels (gemm.cuh).
#pragma once
#include "gemm.cuh"

namespace sonic {

struct UpDownArgs {
  const int* num_pairs;    // device-resident count of 2-CTA pair tiles
  const int* tile_pairs;   // first 128-row tile of each pair | (second exists) << 31
  const int* tile_expert;  // expert of each 128-row tile
  const int* row_token;    // gather map (-1 on pad rows)
  const float* row_gate;   // gate per grouped row (0 on pad rows)
  const __nv_bfloat16* X;  // [T, d]
  int d, n;
  unsigned long long* dbg;  // SONIC_TIMING builds only: cycle counters (sonic_api.cu prints them)
};

#ifndef SONIC_UD_EPW
#define SONIC_UD_EPW 8  // epilogue warps of the fused kernel (4: one per TMEM lane quarter; 8: two)
#endif
#ifndef SONIC_UD_L2PF
#define SONIC_UD_L2PF 8  // L2 prefetch distance (k-blocks) of the gathered X rows (0 = off)
#endif

template <int NU_, int BND_, int EPW_ = SONIC_UD_EPW>
struct UpDownCfg {
  static constexpr int NU = NU_;                       // U jobs per tile (n / 128)
  static constexpr int BND = BND_;                     // D job N width (256 or 128)
  static constexpr int NP = EPW_ == 8 ? 2 : 4;         // producer warps (11 or 9 warps: <= 3 per SM
                                                       // sub-partition, so 168 registers fit)
  static constexpr int EPW = EPW_;                     // epilogue warps (4 or 8)
  static constexpr int EPH = EPW / 4;                  // epilogue warps per TMEM lane quarter
  static constexpr int THREADS = 32 * (NP + 1 + EPW);  // 288 / 352
  static constexpr int RS = NP * 4;                    // gather: row stride between a thread's rows
  static constexpr int RPT = GEMM_BM / RS;             // gather: rows per producer thread
  static constexpr uint32_t A_BYTES = GEMM_BM * GEMM_BK * 2;        // gathered X tile, 16 KB
  static constexpr uint32_t BU_BYTES = 128 * GEMM_BK * 2;           // this CTA's W1 half: 128 cols
  static constexpr uint32_t BD_BYTES = (BND / 2) * GEMM_BK * 2;     // this CTA's W2 half
  static constexpr uint32_t STAGE_BYTES = A_BYTES + BU_BYTES;       // 32 KB
  static constexpr int ABUF = NU * 2 * 16384;                       // A buffer: 128 x n bf16
  static constexpr int NB = EPW == 4 ? 2 : 1;                       // staging ring per epilogue warp
  static constexpr int FIXED = ABUF + EPW * NB * STG_BYTES + 1024 + 1024;
  static constexpr int STAGES_RAW = (SMEM_LIMIT - FIXED) / (int)STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int SMEM = STAGES * STAGE_BYTES + FIXED;
  static_assert(STAGES >= 3, "fused up/down: not enough shared memory for the operand ring");
};

// Registers are allocated per SM sub-partition (16K each; warp w runs on sub-partition w % 4): with
// at most 3 warps per sub-partition (9 or 11 warps) every thread may hold 168
template <int NU, int BND>
__global__ void __maxnreg__(168)
    sonic_updown_kernel(const __grid_constant__ CUtensorMap mW1, const __grid_constant__ CUtensorMap mW2,
                        const __grid_constant__ CUtensorMap mH, const __grid_constant__ CUtensorMap mY,
                        const UpDownArgs args) {
  using Cfg = UpDownCfg<NU, BND>;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int NP = Cfg::NP;
  constexpr uint32_t A_BYTES = Cfg::A_BYTES;
  constexpr uint32_t STAGE_BYTES = Cfg::STAGE_BYTES;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* abuf = smem + STAGES * STAGE_BYTES;  // [NU*2 k-blocks][128 rows x 128 B], 128B swizzle
  uint8_t* stg = abuf + Cfg::ABUF;
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + Cfg::EPW * Cfg::NB * STG_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* aready = tempty + 2;  // [2 NU]: one per 64-column k-block of A
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(aready + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int rank = (int)ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int t_first = blockIdx.x / 2;
  const int t_step = gridDim.x / 2;
  const int d = args.d, n = args.n;
  const int KB_U = d / GEMM_BK;  // k-blocks of a U job
  const int KB_D = n / GEMM_BK;  // k-blocks of a D job
  const int ND = d / BND;

  ptx::pdl_trigger();
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], leader ? NP * 32 + 2 : NP * 32);  // + TMA expect_tx + peer relay
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], 2 * Cfg::EPW);
    }
    for (int s = 0; s < 2 * NU; ++s) ptx::mbar_init(&aready[s], 2 * 4);  // 4 lane-quarter warps x 2 CTAs
    ptx::fence_barrier_init();
    ptx::prefetch_tmap(&mW1);
    ptx::prefetch_tmap(&mW2);
  }
  if (warp == NP) {
    ptx::tmem_alloc2(tmem_holder, 512);
    ptx::tmem_relinquish2();
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  ptx::pdl_wait();

  const int total = *args.num_pairs;
  // pair tile p -> (first 128-row tile, does this CTA's half exist, expert)
  auto decode = [&](int p, int& mt, bool& valid, int& e) {
    const int pt = __ldg(args.tile_pairs + p);
    const int first = pt & 0x7fffffff;
    valid = rank == 0 || pt < 0;
    mt = first + rank;
    e = __ldg(args.tile_expert + first);
  };

  if (warp < NP) {
    // ============================================================ producers
    int stage = 0;
    uint32_t phase = 0;
    constexpr int RS = Cfg::RS, RPT = Cfg::RPT;
    const int pt = threadIdx.x;  // 0 .. 32 NP - 1
    const int c = pt & 7;        // 16-byte chunk within a 128-byte row
    const int r0 = pt >> 3;      // rows r0 + RS j
    const uint32_t sw = (uint32_t)((c ^ (r0 & 7)) << 4);
    const uint64_t gpol = ptx::policy_evict_last();
    int ntok[RPT];
    if (t_first < total) {
      int mt, e;
      bool v;
      decode(t_first, mt, v, e);
#pragma unroll
      for (int j = 0; j < RPT; ++j) ntok[j] = v ? tok_of(args.row_token, mt * GEMM_BM + r0 + RS * j) : 0;
    }
    for (int tile = t_first; tile < total; tile += t_step) {
      int mt, e;
      bool valid;
      decode(tile, mt, valid, e);
      const __nv_bfloat16* srcM[RPT];
#pragma unroll
      for (int j = 0; j < RPT; ++j) srcM[j] = args.X + clamp_tok(ntok[j]) * d + c * 8;
      if (tile + t_step < total) {  // the next tile's gather indices, one tile ahead
        int mt2, e2;
        bool v2;
        decode(tile + t_step, mt2, v2, e2);
#pragma unroll
        for (int j = 0; j < RPT; ++j) ntok[j] = v2 ? tok_of(args.row_token, mt2 * GEMM_BM + r0 + RS * j) : 0;
      }
      // U jobs: gathered X rows + this CTA's 128 W1 columns (rank 0: gate, rank 1: up)
      for (int uj = 0; uj < NU; ++uj) {
        for (int kb = 0; kb < KB_U; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sA = smem + stage * STAGE_BYTES;
          uint8_t* sB = sA + A_BYTES;
          uint64_t* bar = &full[stage];
          if (pt == 0) {
            if (leader) ptx::mbar_arrive_expect_tx(bar, Cfg::BU_BYTES * 2);
            const int cb = (rank ? n : 0) + 128 * uj;
            tload3<true>(sB, &mW1, bar, cb, kb * GEMM_BK, e);
            tload3<true>(sB + 8192, &mW1, bar, cb + 64, kb * GEMM_BK, e);
          }
          const uint32_t dst = ptx::smem_u32(sA) + r0 * 128 + sw;
#pragma unroll
          for (int j = 0; j < RPT; ++j) gather16(dst + j * RS * 128, srcM[j] + kb * GEMM_BK, gpol);
          ptx::cp_async_mbar_arrive(bar);
          // the first U job reads the tile's X rows from HBM: pull the lines SONIC_UD_L2PF k-blocks ahead
          // into L2 (the 4-stage smem ring alone is ~2k cycles of lookahead); U_1.. re-read them from L2
          if (SONIC_UD_L2PF > 0 && uj == 0 && c == 0 && kb + SONIC_UD_L2PF < KB_U) {
#pragma unroll
            for (int j = 0; j < RPT; ++j) ptx::prefetch_l2(srcM[j] + (kb + SONIC_UD_L2PF) * GEMM_BK);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      // while the D jobs run, pull the next tile's first SONIC_UD_L2PF k-blocks of X rows into L2
      // (thread c takes k-block c of its rows; ntok already holds the next tile's tokens)
      if (SONIC_UD_L2PF > 0 && tile + t_step < total && c < SONIC_UD_L2PF && c < KB_U) {
#pragma unroll
        for (int j = 0; j < RPT; ++j) ptx::prefetch_l2(args.X + clamp_tok(ntok[j]) * d + c * GEMM_BK);
      }
      // D jobs: this CTA's BND/2 columns of the W2 N-tile (A is resident in the A buffer)
      for (int di = 0; di < ND; ++di) {
        for (int kb = 0; kb < KB_D; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sB = smem + stage * STAGE_BYTES + A_BYTES;
          uint64_t* bar = &full[stage];
          if (pt == 0) {
            if (leader) ptx::mbar_arrive_expect_tx(bar, Cfg::BD_BYTES * 2);
            const int n0 = di * BND + rank * (BND / 2);
#pragma unroll
            for (int j = 0; j < BND / 128; ++j) tload3<true>(sB + j * 8192, &mW2, bar, n0 + 64 * j, kb * GEMM_BK, e);
          }
          ptx::mbar_arrive(bar);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == NP) {
    // ============================================================ MMA issuer (leader) / relay (peer)
    const int njobs_k = NU * KB_U + ND * KB_D;  // k-blocks per tile
    if (lane == 0 && leader) {
      constexpr uint32_t idesc_u = ptx::make_idesc(2 * GEMM_BM, 256, 0, 1);
      constexpr uint32_t idesc_d = ptx::make_idesc(2 * GEMM_BM, BND, 0, 1);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      uint32_t a_phase = 0;
      const uint32_t abase = ptx::smem_u32(abuf);
#ifdef SONIC_TIMING
      unsigned long long c0 = clock64(), c_te[2] = {0, 0}, c_full[2] = {0, 0}, c_ar = 0, c_busy[2] = {0, 0};
#define TSTAMP(x) const unsigned long long x = clock64()
#else
#define TSTAMP(x)
#endif
      for (int tile = t_first; tile < total; tile += t_step) {
        for (int job = 0; job < NU + ND; ++job) {
          const bool is_u = job < NU;
          TSTAMP(ta);
          ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
#ifdef SONIC_TIMING
          TSTAMP(tb);
          c_te[is_u ? 0 : 1] += tb - ta;
#endif
          ptx::tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * 256;
          const int nkb = is_u ? KB_U : KB_D;
          for (int kb = 0; kb < nkb; ++kb) {
            if (job == NU) {  // D_0: A columns [64 kb, 64 kb + 64) written by U_{kb/2}'s epilogue
              TSTAMP(tc);
              ptx::mbar_wait(&aready[kb], a_phase);
#ifdef SONIC_TIMING
              c_ar += clock64() - tc;
#endif
            }
            TSTAMP(td);
            ptx::mbar_wait(&full[stage], phase);
#ifdef SONIC_TIMING
            c_full[is_u ? 0 : 1] += clock64() - td;
#endif
            if (is_u) ptx::fence_proxy_async_smem();  // cp.async (generic proxy) -> tcgen05.mma
            ptx::tc_fence_after();
            const uint32_t s_base = ptx::smem_u32(smem + stage * STAGE_BYTES);
            const uint32_t b_base = s_base + A_BYTES;
            const uint32_t a_base = is_u ? s_base : abase + kb * 16384;
#pragma unroll
            for (int k = 0; k < GEMM_BK / 16; ++k) {
              const uint64_t ad = ptx::make_sdesc(a_base + k * 32, 16, 1024);
              const uint64_t bd = ptx::make_sdesc(b_base + k * 2048, 8192, 1024);
              ptx::mma_bf16_cg2(d_tmem, ad, bd, is_u ? idesc_u : idesc_d, (kb | k) != 0);
            }
            ptx::mma_commit_mc(&empty[stage], 0x3);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          ptx::mma_commit_mc(&tfull[acc], 0x3);
#ifdef SONIC_TIMING
          c_busy[is_u ? 0 : 1] += clock64() - ta;
#endif
          acc ^= 1;
          if (acc == 0) acc_phase ^= 1;
        }
        a_phase ^= 1;
      }
#ifdef SONIC_TIMING
      if (args.dbg) {
        atomicAdd(args.dbg + 0, clock64() - c0);
        atomicAdd(args.dbg + 1, c_te[0]);
        atomicAdd(args.dbg + 2, c_te[1]);
        atomicAdd(args.dbg + 3, c_full[0]);
        atomicAdd(args.dbg + 4, c_full[1]);
        atomicAdd(args.dbg + 5, c_ar);
        atomicAdd(args.dbg + 6, c_busy[0]);
        atomicAdd(args.dbg + 7, c_busy[1]);
        atomicAdd(args.dbg + 8, 1ull);
      }
#endif
    } else if (lane == 0 && !leader) {
      // relay: this CTA's producer arrivals (cp.async completions) -> the leader's full barrier
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = t_first; tile < total; tile += t_step) {
        for (int kb = 0; kb < njobs_k; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::fence_proxy_async_smem();
          ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&full[stage]), 0));
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else {
    // ============================================================ epilogue (EPW warps)
    // Warp ew works on TMEM lane quarter q = warp % 4 (its 32 rows) and, with EPW = 8, on every other
    // 64-column chunk (half = ew / 4).
    constexpr int EPH = Cfg::EPH;
    const int ew = warp - NP - 1;
    const int q = warp & 3;
    const int half = ew / 4;
    StoreQ<Cfg::NB> sq{stg + ew * Cfg::NB * STG_BYTES, 0};
    int acc = 0;
    uint32_t acc_phase = 0;
    const uint32_t tempty_leader = ptx::mapa(ptx::smem_u32(&tempty[0]), 0);
    const uint32_t aready_leader = ptx::mapa(ptx::smem_u32(&aready[0]), 0);
    const uint32_t arow = ptx::smem_u32(abuf) + (uint32_t)(32 * q) * 128;  // this warp's 32 rows of A
#ifdef SONIC_TIMING
    unsigned long long e_wait = 0, e_busy[2] = {0, 0};
#endif
    for (int tile = t_first; tile < total; tile += t_step) {
      int mt, e;
      bool valid;
      decode(tile, mt, valid, e);
      const int wrow = mt * GEMM_BM + 32 * q;  // first grouped row of this warp's slab
      const int row = wrow + lane;
      const float gate = valid ? __ldg(args.row_gate + row) : 0.f;
      for (int job = 0; job < NU + ND; ++job) {
#ifdef SONIC_TIMING
        const unsigned long long ea = clock64();
#endif
        ptx::mbar_wait(&tfull[acc], acc_phase);
#ifdef SONIC_TIMING
        const unsigned long long eb = clock64();
        e_wait += eb - ea;
#endif
        ptx::tc_fence_after();
        const uint32_t t_acc = tmem_base + ((uint32_t)(32 * q) << 16) + acc * 256;
        if (job < NU) {
          // ---- U job: accumulator cols [0,128) = gate, [128,256) = up of H cols 128 job + [0,128).
          // Per 64-column chunk: A first (into the A buffer; then the MMA thread may start on that
          // k-block of D_0), then the H gate / up columns through the staging ring by TMA store.
#pragma unroll 1
          for (int cc = half; cc < 2; cc += EPH) {
            const int col = 128 * job + 64 * cc;
            const int akb = 2 * job + cc;  // A k-block written by this chunk
            uint32_t pu[2][16];            // up half of H, bf16 pairs, stored after the gate half
            int ig = 0;
            uint32_t bg = 0;
            if (valid) {
              ig = sq.acquire(lane);
              bg = sq.addr(ig);
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                uint32_t g[32], u[32];
                ptx::tmem_ld32(t_acc + 64 * cc + 32 * h, g);
                ptx::tmem_ld32(t_acc + 128 + 64 * cc + 32 * h, u);
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
                  uint32_t apk[4];
#pragma unroll
                  for (int i = 0; i < 4; ++i) {
                    const float a0 = hg[2 * i] * sigmoidf_fast(hg[2 * i]) * hu[2 * i];
                    const float a1 = hg[2 * i + 1] * sigmoidf_fast(hg[2 * i + 1]) * hu[2 * i + 1];
                    apk[i] = ptx::pack_bf16(a0, a1);
                    pu[h][4 * q8 + i] = ptx::pack_bf16(hu[2 * i], hu[2 * i + 1]);
                  }
                  ptx::st_shared_v4(arow + (uint32_t)akb * 16384 + swz(lane, ch), apk[0], apk[1], apk[2], apk[3]);
                  ptx::st_shared_v4(bg + swz(lane, ch), ptx::pack_bf16(hg[0], hg[1]), ptx::pack_bf16(hg[2], hg[3]),
                                    ptx::pack_bf16(hg[4], hg[5]), ptx::pack_bf16(hg[6], hg[7]));
                }
              }
            }
            // A k-block akb of this warp's rows is in place: make it visible to the tensor core (async
            // proxy) and tell the leader's MMA thread
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              if (leader) ptx::mbar_arrive(&aready[akb]);
              else ptx::mbar_arrive_cluster(aready_leader + akb * 8);
            }
            if (valid) {
              sq.issue(lane, ig, &mH, col, wrow);  // H gate columns
              const int iu = sq.acquire(lane);
              const uint32_t bu = sq.addr(iu);
#pragma unroll
              for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int q8 = 0; q8 < 4; ++q8)
                  ptx::st_shared_v4(bu + swz(lane, 4 * h + q8), pu[h][4 * q8], pu[h][4 * q8 + 1], pu[h][4 * q8 + 2],
                                    pu[h][4 * q8 + 3]);
              sq.issue(lane, iu, &mH, n + col, wrow);  // H up columns
            }
          }
        } else if (valid) {
          // ---- D job: Y[:, BND i .. ] = gate * acc, bf16, TMA store; chunks j = half, half + EPH, ..
          const int di = job - NU;
          constexpr int NCH = BND / 64;
#pragma unroll 1
          for (int j = half; j < NCH; j += EPH) {
            uint32_t r[2][32];
            ptx::tmem_ld32(t_acc + 64 * j, r[0]);
            ptx::tmem_ld32(t_acc + 64 * j + 32, r[1]);
            const int i = sq.acquire(lane);
            const uint32_t b = sq.addr(i);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int q8 = 0; q8 < 4; ++q8) {
                const uint32_t* v = r[h] + 8 * q8;
                ptx::st_shared_v4(b + swz(lane, 4 * h + q8),
                                  ptx::pack_bf16(gate * __uint_as_float(v[0]), gate * __uint_as_float(v[1])),
                                  ptx::pack_bf16(gate * __uint_as_float(v[2]), gate * __uint_as_float(v[3])),
                                  ptx::pack_bf16(gate * __uint_as_float(v[4]), gate * __uint_as_float(v[5])),
                                  ptx::pack_bf16(gate * __uint_as_float(v[6]), gate * __uint_as_float(v[7])));
              }
            sq.issue(lane, i, &mY, di * BND + 64 * j, wrow);
          }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (leader) ptx::mbar_arrive(&tempty[acc]);
          else ptx::mbar_arrive_cluster(tempty_leader + acc * 8);
        }
#ifdef SONIC_TIMING
        e_busy[job < NU ? 0 : 1] += clock64() - eb;
#endif
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
    if (lane == 0) ptx::bulk_wait<0>();
    __syncwarp();
#ifdef SONIC_TIMING
    if (args.dbg && lane == 0 && ew == 0 && leader) {
      atomicAdd(args.dbg + 9, e_wait);
      atomicAdd(args.dbg + 10, e_busy[0]);
      atomicAdd(args.dbg + 11, e_busy[1]);
    }
#endif
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == NP) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc2(tmem_base, 512);
  }
}

}  // namespace sonic
