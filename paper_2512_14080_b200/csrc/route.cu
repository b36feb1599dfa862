// route.cu -- routing / metadata kernels of sonic_route.
//
// Data structure: per-expert token bitmaps bm[e][w] (bit t%32 of word t/32 set when token
// t is routed to e).  Every integer output is a pure function of the bitmaps, built with
// order-independent atomicOr, so the metadata is deterministic and canonical: segments
// hold tokens in ascending order (popcount prefix over words), the token CSR lists
// experts in ascending order.
//
//   k_topk_g4        TC top-K per token (4 threads per token, stable insertion on ordered fp32
//                    scores, bitonic merges on exact 64-bit keys; ties -> lower expert id;
//                    P:1072-1099, Q9) -> topk, TC bitmap
//   k_expert_popc    per-expert popcount + exclusive word prefix (histogram f_e)
//   k_tr_decide      rounding decision: NR-f, UP, DOWN, Balance-f, SR-f
//                    (P:2116-2198); expert choice capacity (Q22)
//   (S^T for TR, expert columns contiguous, is written by k_topk_g4 from its staged slab)
//   k_tr_select_w    Alg. 4 step (4): per expert, keep the top f_r of the ranking
//                    (in-TC, S, -t) via radix select on the ordered score + token tie pass
//   k_orphans        tokens with no kept expert flag their top-1 expert (Q14 rescue)
//   k_popc_offsets   counts + word prefixes; last block: offsets, tile-aligned pad_offsets,
//                    tile -> expert map, 2-CTA pair schedule
//   k_build_rows     gather map row_token (+ pad rows)
//   k_rows_tc        TC: gather map + token CSR + renormalised gates in one launch
//   k_csr_count / k_csr_rows_chunked   general token CSR (TR, GIVEN) via 32x32 bit transposes
#include <algorithm>
#include "sonic_internal.h"
#include "ptx.cuh"

namespace sonic {

__device__ __forceinline__ uint32_t ord_f32(float x) {
  uint32_t b = __float_as_uint(x);
  if (b == 0x80000000u) b = 0u;  // -0 == +0 (Q23)
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// ---------------------------------------------------------------- block scan helpers
// Exclusive scan of v over the block (blockDim.x <= 1024, multiple of 32); returns the
// exclusive prefix and writes the block total to *total.
__device__ int block_excl_scan(int v, int* total) {
  __shared__ int warp_sums[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int s = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    warp_sums[lane] = s;  // inclusive
  }
  __syncthreads();
  int base = wid > 0 ? warp_sums[wid - 1] : 0;
  int tot = warp_sums[nw - 1];
  __syncthreads();
  *total = tot;
  return base + x - v;
}


// ---------------------------------------------------------------- per-expert popcount
__global__ void k_expert_popc(const uint32_t* __restrict__ bm, int W, int* __restrict__ wprefix,
                              int* __restrict__ cnt, int* __restrict__ cnt2) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int e = blockIdx.x;
  int base = 0;
  for (int w0 = 0; w0 < W; w0 += blockDim.x) {
    const int w = w0 + threadIdx.x;
    const int c = w < W ? __popc(bm[(size_t)e * W + w]) : 0;
    int tot;
    const int ex = block_excl_scan(c, &tot);
    if (wprefix && w < W) wprefix[(size_t)e * W + w] = base + ex;
    base += tot;
  }
  if (threadIdx.x == 0) {
    cnt[e] = base;
    if (cnt2) cnt2[e] = base;
  }
}

// ---------------------------------------------------------------- TR decision (NR-f)
// SR-f draw of expert e (Q21): one SplitMix64 step from state (seed << 32 | e), top 24 bits.
__device__ __forceinline__ uint32_t sr_draw24(uint32_t seed, uint32_t e) {
  unsigned long long x = (((unsigned long long)seed << 32) | e) + 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  x ^= x >> 31;
  return (uint32_t)(x >> 40);
}

// Rounding decision per expert.  rounding: 0 NR-f (strict '<': an exact M/2 tie
// rounds down, Q11), 1 up, 2 down, 3 Balance-f (Alg. 6: sequential, one thread), 4 SR-f.
// ec_cap >= 0: expert choice, every expert takes ec_cap tokens.
// The per-expert rounding decisions (every subroutine but Balance-f, which is sequential over experts).
__device__ __forceinline__ int tr_decide_one(int fe, int e, int T, int M, int rounding, uint32_t seed, int ec_cap) {
  if (ec_cap >= 0) return ec_cap;
  const int up_m = (fe + M - 1) / M * M;  // the M-multiple above f (uncapped: the NR-f comparison)
  const int up = min(up_m, T);            // Q15: a chosen "up" is capped at T
  const int dn = fe / M * M;
  switch (rounding) {
    case 1: return up;
    case 2: return dn;
    case 4: return (unsigned long long)sr_draw24(seed, (uint32_t)e) * (unsigned)M < ((unsigned long long)(fe - dn) << 24)
                       ? up : dn;
    default: return (up_m - fe) < (fe - dn) ? up : dn;  // strict '<': M/2 ties round down (Q11)
  }
}

// k_expert_popc + the decision in one launch (the per-expert subroutines: the count of expert e is
// all its decision needs): block e counts its bitmap row, then writes f[e] and f_r[e].
__global__ void k_expert_popc_decide(const uint32_t* __restrict__ bm, int W, int* __restrict__ cnt,
                                     int* __restrict__ f_r, int T, int M, int rounding, uint32_t seed, int ec_cap) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int e = blockIdx.x;
  int c = 0;
  for (int w = threadIdx.x; w < W; w += blockDim.x) c += __popc(bm[(size_t)e * W + w]);
  int tot;
  block_excl_scan(c, &tot);
  if (threadIdx.x == 0) {
    cnt[e] = tot;
    f_r[e] = tr_decide_one(tot, e, T, M, rounding, seed, ec_cap);
  }
}

__global__ void k_tr_decide(const int* __restrict__ f, int* __restrict__ f_r, int E, int T, int M, int rounding,
                            uint32_t seed, int ec_cap) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  if (rounding == 3 && ec_cap < 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      long long z = 0;
      for (int e = 0; e < E; ++e) {
        const int fe = f[e];
        const int up = min((fe + M - 1) / M * M, T);
        const int dn = fe / M * M;
        const long long ru = up - fe, rd = dn - fe;
        const bool pick_up = llabs(ru + z) < llabs(rd + z);
        f_r[e] = pick_up ? up : dn;
        z += pick_up ? ru : rd;
      }
    }
    return;
  }
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x)
    f_r[e] = tr_decide_one(f[e], e, T, M, rounding, seed, ec_cap);
}

// ---------------------------------------------------------------- TR selection
// One block (1024 threads) per expert.  rescue == 0: every expert, f_r from k_tr_decide.
// rescue == 1: only experts flagged by k_orphans; they round up (f_r = min(ceil, T)).
// Selects the k largest candidates by (ordered S desc, token asc): down -> candidates are the
// TC tokens, k = f_r; up -> candidates are the non-TC tokens, k = f_r - f (Alg. 4, Q10).

// Word-per-thread variant: thread i owns bitmap words i, i + 1024, ...; the 32 scores of a word
// are loaded as 8 x 16 B (one latency per word per pass), the histogram adds come from
// registers, and the final tie pass is one block scan of per-thread equal counts instead of one
// scan per 1024 tokens.  Same result as k_tr_select (ties at the threshold: lowest tokens first).
__device__ __forceinline__ void load_word_keys(const float* __restrict__ col, int T, int w, uint32_t (&o)[32]) {
  const int t0 = w * 32;
  if (t0 + 32 <= T && (reinterpret_cast<uintptr_t>(col + t0) & 15) == 0) {
    const float4* p = reinterpret_cast<const float4*>(col + t0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float4 v = __ldg(p + i);
      o[4 * i] = ord_f32(v.x);
      o[4 * i + 1] = ord_f32(v.y);
      o[4 * i + 2] = ord_f32(v.z);
      o[4 * i + 3] = ord_f32(v.w);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i) o[i] = t0 + i < T ? ord_f32(__ldg(col + t0 + i)) : 0u;
  }
}
template <bool ONE>  // ONE: W <= blockDim.x, so each thread's single word of keys stays in registers
__global__ void __launch_bounds__(1024) k_tr_select_w(const float* __restrict__ ST, int T, int W, int M,
                                                      const uint32_t* __restrict__ bm_tc,
                                                      uint32_t* __restrict__ bm_kept, const int* __restrict__ f,
                                                      int* __restrict__ f_r, const int* __restrict__ flip,
                                                      int rescue, int ec, const int* __restrict__ fr_src) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  __shared__ int hist[4096];
  __shared__ int s_digit, s_above;
  const int e = blockIdx.x;
  const int tid = threadIdx.x;
  // expert choice: no TC set -- every token is a candidate and the kept set is the selection
  const int fc = ec ? 0 : f[e];
  int fr;
  if (rescue) {
    if (!flip[e]) return;
    fr = min((fc + M - 1) / M * M, T);
    if (tid == 0) f_r[e] = fr;
  } else {
    fr = fr_src ? fr_src[e] : f_r[e];  // NR-s runs the selection for both candidate counts
  }
  const uint32_t* tcw_p = bm_tc + (size_t)e * W;
  auto tcw = [&](int w) -> uint32_t { return ec ? 0u : tcw_p[w]; };
  uint32_t* kw = bm_kept + (size_t)e * W;
  if (fr == fc) {
    for (int w = tid; w < W; w += blockDim.x) kw[w] = tcw(w);
    return;
  }
  const bool up = fr > fc;
  int k = up ? fr - fc : fr;
  if (k == 0) {
    for (int w = tid; w < W; w += blockDim.x) kw[w] = 0u;
    return;
  }
  const float* col = ST + (size_t)e * T;
  uint32_t okeep[ONE ? 32 : 1];
  uint32_t cand1 = 0u;
  if constexpr (ONE) {
    if (tid < W) {
      uint32_t o[32];
      load_word_keys(col, T, tid, o);
#pragma unroll
      for (int i = 0; i < 32; ++i) okeep[i] = o[i];
      cand1 = (up ? ~tcw(tid) : tcw(tid));
      if (tid * 32 + 32 > T) cand1 &= (T - tid * 32 >= 32) ? ~0u : ((1u << (T - tid * 32)) - 1u);
    }
  }
  uint32_t prefix = 0, pmask = 0;
  const int shifts[3] = {20, 8, 0};
  const int bits[3] = {12, 12, 8};
  for (int p = 0; p < 3; ++p) {
    const int sh = shifts[p], nb = 1 << bits[p];
    for (int i = tid; i < nb; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    if constexpr (ONE) {
      if (tid < W) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (((cand1 >> i) & 1u) && (okeep[i] & pmask) == prefix) atomicAdd(&hist[(okeep[i] >> sh) & (nb - 1)], 1);
      }
    } else {
      for (int w = tid; w < W; w += blockDim.x) {
        uint32_t o[32];
        load_word_keys(col, T, w, o);
        const uint32_t cand = up ? ~tcw(w) : tcw(w);
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (((cand >> i) & 1u) && w * 32 + i < T && (o[i] & pmask) == prefix)
            atomicAdd(&hist[(o[i] >> sh) & (nb - 1)], 1);
      }
    }
    __syncthreads();
    {  // the digit holding the k-th largest: block scan over bins from the top (4 bins / thread)
      const int bpt = (nb + blockDim.x - 1) / blockDim.x;
      const int hi = nb - 1 - tid * bpt;  // this thread's bins: hi, hi-1, ..., hi-bpt+1
      int sum = 0;
      for (int b = 0; b < bpt; ++b)
        if (hi - b >= 0) sum += hist[hi - b];
      int tot;
      const int ex = block_excl_scan(sum, &tot);
      if (ex < k && k <= ex + sum) {
        int cum = ex;
        for (int b = 0; b < bpt; ++b) {
          const int h = hist[hi - b];
          if (cum + h >= k) {
            s_digit = hi - b;
            s_above = cum;
            break;
          }
          cum += h;
        }
      }
    }
    __syncthreads();
    prefix |= (uint32_t)s_digit << sh;
    pmask |= (uint32_t)(nb - 1) << sh;
    k -= s_above;
    __syncthreads();
  }
  // threshold = prefix: keep every candidate above it and the first k equal to it (lowest tokens)
  int run = 0;
  for (int w0 = 0; w0 < W; w0 += blockDim.x) {
    const int w = w0 + tid;
    uint32_t gt = 0u, eq = 0u;
    if (w < W) {
      if constexpr (ONE) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const bool c = (cand1 >> i) & 1u;
          gt |= (uint32_t)(c && okeep[i] > prefix) << i;
          eq |= (uint32_t)(c && okeep[i] == prefix) << i;
        }
      } else {
        uint32_t o[32];
        load_word_keys(col, T, w, o);
        const uint32_t cand = up ? ~tcw(w) : tcw(w);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const bool c = ((cand >> i) & 1u) && w * 32 + i < T;
          gt |= (uint32_t)(c && o[i] > prefix) << i;
          eq |= (uint32_t)(c && o[i] == prefix) << i;
        }
      }
    }
    int tot;
    const int ex = block_excl_scan(__popc(eq), &tot);
    int take = min(max(k - run - ex, 0), __popc(eq));
    uint32_t sel = 0u;
    while (take-- > 0) {  // the lowest `take` equal tokens of this word
      const uint32_t b = eq & (0u - eq);
      sel |= b;
      eq ^= b;
    }
    if (w < W) kw[w] = up ? (tcw(w) | gt | sel) : (gt | sel);
    run += tot;
  }
}

// ---------------------------------------------------------------- NR-s (Q25)
// the two candidate counts of every expert: floor_M(f) and min(ceil_M(f), T)
__global__ void k_nrs_counts(const int* __restrict__ f, int E, int T, int M, int* __restrict__ f_dn,
                             int* __restrict__ f_up) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    const int fe = f[e];
    f_dn[e] = fe / M * M;
    f_up[e] = min((fe + M - 1) / M * M, T);
  }
}

// sums[e] = sum of S over the tokens set in expert e's bitmap, in fp64 (exact for fp32 scores
// of one expert: order-independent).  One block per expert.
__global__ void k_bitmap_sums(const float* __restrict__ ST, const uint32_t* __restrict__ bm, int T, int W,
                              double* __restrict__ sums) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int e = blockIdx.x;
  const float* col = ST + (size_t)e * T;
  double acc = 0.0;
  for (int w = threadIdx.x; w < W; w += blockDim.x) {
    uint32_t bits = bm[(size_t)e * W + w];
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      acc += (double)col[w * 32 + b];
    }
  }
  __shared__ double red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) sums[e] = v;
  }
}

// the decision (p = (s_tc - s_dn) / (s_up - s_dn), pad iff u < p 2^24) and the chosen kept words
__global__ void k_nrs_decide(const int* __restrict__ f, const int* __restrict__ f_dn, const int* __restrict__ f_up,
                             const double* __restrict__ s_tc, const double* __restrict__ s_dn,
                             const double* __restrict__ s_up, const uint32_t* __restrict__ bm_dn,
                             const uint32_t* __restrict__ bm_up, int W, uint32_t seed, int* __restrict__ f_r,
                             uint32_t* __restrict__ bm_kept) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int e = blockIdx.x;
  __shared__ int s_up_chosen;
  if (threadIdx.x == 0) {
    bool go_up = false;
    if (f_dn[e] != f[e]) {
      const double p = (s_tc[e] - s_dn[e]) / (s_up[e] - s_dn[e]);
      go_up = (double)sr_draw24(seed, (uint32_t)e) < p * 16777216.0;
    }
    s_up_chosen = go_up;
    f_r[e] = go_up ? f_up[e] : f_dn[e];
  }
  __syncthreads();
  const uint32_t* src = (s_up_chosen ? bm_up : bm_dn) + (size_t)e * W;
  for (int w = threadIdx.x; w < W; w += blockDim.x) bm_kept[(size_t)e * W + w] = src[w];
}

// ---------------------------------------------------------------- orphan detection
// Warp per 32-token word.  A token kept by no expert flags its top-1 TC expert.
__global__ void k_orphans(const uint32_t* __restrict__ bm_kept, int T, int E, int W, int K,
                          const int* __restrict__ topk_ids, int* __restrict__ flip) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= W) return;
  uint32_t acc = 0;
  for (int e = lane; e < E; e += 32) acc |= bm_kept[(size_t)e * W + w];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc |= __shfl_xor_sync(0xffffffffu, acc, o);
  const int t = w * 32 + lane;
  if (t < T && !((acc >> lane) & 1u)) flip[topk_ids[(size_t)t * K]] = 1;
}

// ---------------------------------------------------------------- offsets & tiles
// Also builds the 2-CTA schedule: each expert's 128-row tiles are paired (t, t+1); an expert with
// an odd tile count ends with a half pair (bit 31 clear).
__device__ void offsets_block(const int* __restrict__ f_r, int E, int* __restrict__ offsets,
                              int* __restrict__ pad_offsets, int* __restrict__ tile_expert,
                              int* __restrict__ num_tiles, int* __restrict__ tile_pairs, int* __restrict__ num_pairs) {
  __shared__ int s_pad[4097];
  __shared__ int s_pp[4097];
  int base = 0, pbase = 0, ppbase = 0;
  for (int e0 = 0; e0 < E; e0 += blockDim.x) {
    const int e = e0 + threadIdx.x;
    const int c = e < E ? __ldcg(f_r + e) : 0;
    const int pc = (c + GEMM_M - 1) / GEMM_M * GEMM_M;
    const int pp = (pc / GEMM_M + 1) / 2;
    int tot, ptot, pptot;
    const int ex = block_excl_scan(c, &tot);
    const int pex = block_excl_scan(pc, &ptot);
    const int ppex = block_excl_scan(pp, &pptot);
    if (e < E) {
      offsets[e] = base + ex;
      pad_offsets[e] = pbase + pex;
      s_pad[e] = pbase + pex;
      s_pp[e] = ppbase + ppex;
    }
    base += tot;
    pbase += ptot;
    ppbase += pptot;
  }
  if (threadIdx.x == 0) {
    offsets[E] = base;
    pad_offsets[E] = pbase;
    s_pad[E] = pbase;
    s_pp[E] = ppbase;
    *num_tiles = pbase / GEMM_M;
    *num_pairs = ppbase;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ppbase; i += blockDim.x) {
    int lo = 0, hi = E - 1;  // largest e with s_pp[e] <= i
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_pp[mid] <= i) lo = mid; else hi = mid - 1;
    }
    const int j = i - s_pp[lo];
    const int tiles_e = (s_pad[lo + 1] - s_pad[lo]) / GEMM_M;
    const int first = s_pad[lo] / GEMM_M + 2 * j;
    tile_pairs[i] = first | ((2 * j + 1 < tiles_e) ? (int)0x80000000u : 0);
  }
  const int nt = pbase / GEMM_M;
  for (int i = threadIdx.x; i < nt; i += blockDim.x) {
    const int r = i * GEMM_M;
    int lo = 0, hi = E - 1;  // largest e with s_pad[e] <= r  (then s_pad[e+1] > r)
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_pad[mid] <= r) lo = mid; else hi = mid - 1;
    }
    tile_expert[i] = lo;
  }
}

// ---------------------------------------------------------------- gather map

// Per-expert popcount + word prefix (one block per expert, as k_expert_popc); the last block to
// finish (ticket) then builds offsets / tiles / pairs from the counts (k_offsets' work) -- one
// launch instead of two.  cnt2 (if given) receives a copy of the counts; the offsets use cnt2 if
// given, else cnt.
__global__ void __launch_bounds__(1024) k_popc_offsets(const uint32_t* __restrict__ bm, int W, int* __restrict__ wprefix,
                                                       int* __restrict__ cnt, int* __restrict__ cnt2,
                                                       unsigned* __restrict__ ticket, int* __restrict__ offsets,
                                                       int* __restrict__ pad_offsets, int* __restrict__ tile_expert,
                                                       int* __restrict__ num_tiles, int* __restrict__ tile_pairs,
                                                       int* __restrict__ num_pairs) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int e = blockIdx.x;
  int base = 0;
  for (int w0 = 0; w0 < W; w0 += blockDim.x) {
    const int w = w0 + threadIdx.x;
    const int c = w < W ? __popc(bm[(size_t)e * W + w]) : 0;
    int tot;
    const int ex = block_excl_scan(c, &tot);
    if (w < W) wprefix[(size_t)e * W + w] = base + ex;
    base += tot;
  }
  __shared__ bool s_last;
  if (threadIdx.x == 0) {
    cnt[e] = base;
    if (cnt2) cnt2[e] = base;
    __threadfence();
    s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  offsets_block(cnt2 ? cnt2 : cnt, (int)gridDim.x, offsets, pad_offsets, tile_expert, num_tiles, tile_pairs, num_pairs);
}

__global__ void k_build_rows(const uint32_t* __restrict__ bm_kept, const int* __restrict__ wprefix, int W,
                             const int* __restrict__ f_r, const int* __restrict__ pad_offsets,
                             int* __restrict__ row_token, float* __restrict__ row_gate) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int e = blockIdx.y;
  const int base = pad_offsets[e];
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w < W) {
    uint32_t bits = bm_kept[(size_t)e * W + w];
    int r = base + wprefix[(size_t)e * W + w];
    while (bits) {
      const int b = __ffs(bits) - 1;
      row_token[r++] = w * 32 + b;
      bits &= bits - 1;
    }
  }
  if (blockIdx.x == 0) {  // pad rows of this expert's last tile
    for (int r = base + f_r[e] + threadIdx.x; r < pad_offsets[e + 1]; r += blockDim.x) {
      row_token[r] = -1;
      row_gate[r] = 0.f;
    }
  }
}

// ---------------------------------------------------------------- token CSR via bit transposes
// Warp per 32-token word w.  For each 32-expert chunk c, lane j loads the bitmap word of expert
// 32c + j; a 5-stage shuffle transpose of that 32x32 bit block gives lane t the 32-bit mask of
// token 32w + t's experts in the chunk (bit b = expert 32c + b).  Counts, an in-word shuffle scan
// and a scan over the W word totals (done by the last block of k_csr_count) give rowptr without
// a serial pass over T.
__device__ __forceinline__ uint32_t transpose32(uint32_t v, int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const uint32_t lo = s == 16 ? 0x0000FFFFu : s == 8 ? 0x00FF00FFu : s == 4 ? 0x0F0F0F0Fu : s == 2 ? 0x33333333u
                                                                                               : 0x55555555u;
    const uint32_t o = __shfl_xor_sync(0xffffffffu, v, s);
    v = (lane & s) ? ((v & ~lo) | ((o & ~lo) >> s)) : ((v & lo) | ((o & lo) << s));
  }
  return v;
}
__device__ __forceinline__ uint32_t token_mask_chunk(const uint32_t* __restrict__ bm, int E, int W, int w, int c,
                                                     int lane) {
  const int e = 32 * c + lane;
  const uint32_t v = e < E ? __ldg(bm + (size_t)e * W + w) : 0u;
  return transpose32(v, lane);
}

__global__ void k_csr_count(const uint32_t* __restrict__ bm, int T, int E, int W, int* __restrict__ word_pref,
                            int* __restrict__ rowptr, unsigned* __restrict__ ticket) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w < W) {
    int c = 0;
    for (int ch = 0; ch < (E + 31) / 32; ++ch) c += __popc(token_mask_chunk(bm, E, W, w, ch, lane));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) word_pref[w] = c;  // word total for now; the last block turns it into a prefix
  }
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // exclusive scan of the W word totals in place (blockDim.x = 256 threads, W/256 per thread)
  int base = 0;
  for (int w0 = 0; w0 < W; w0 += blockDim.x) {
    const int i = w0 + threadIdx.x;
    const int v = i < W ? __ldcg(word_pref + i) : 0;
    int tot;
    const int ex = block_excl_scan(v, &tot);
    if (i < W) word_pref[i] = base + ex;
    base += tot;
  }
  if (threadIdx.x == 0) rowptr[T] = base;
}

// Rows of each token in ascending expert order + gates (renormalised unless gate_raw).
__global__ void k_csr_rows(const uint32_t* __restrict__ bm, const int* __restrict__ wprefix, int T, int E, int W,
                           const int* __restrict__ pad_offsets, const int* __restrict__ word_pref,
                           const float* __restrict__ S, int gate_raw, int* __restrict__ rowptr,
                           int* __restrict__ token_rows, float* __restrict__ row_gate) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= W) return;
  const int t = w * 32 + lane;
  const int nch = (E + 31) / 32;
  int c = 0;
  for (int ch = 0; ch < nch; ++ch) c += __popc(token_mask_chunk(bm, E, W, w, ch, lane));
  int incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const int j0 = word_pref[w] + incl - c;
  if (t < T) rowptr[t] = j0;
  const uint32_t below = (1u << lane) - 1u;
  const float* srow = S + (size_t)t * E;
  float sum = 0.f;
  int j = j0;
  // (lanes beyond T hold empty masks; every lane stays for the transposes' shuffles)
  for (int ch = 0; ch < nch; ++ch) {
    uint32_t m = token_mask_chunk(bm, E, W, w, ch, lane);
    while (m) {
      const int e = 32 * ch + __ffs(m) - 1;
      m &= m - 1;
      const uint32_t word = __ldg(bm + (size_t)e * W + w);
      token_rows[j++] = pad_offsets[e] + wprefix[(size_t)e * W + w] + __popc(word & below);
      sum += __ldg(srow + e);
    }
    __syncwarp();
  }
  const float inv = (gate_raw || sum == 0.f) ? 1.f : 1.f / sum;
  j = j0;
  for (int ch = 0; ch < nch; ++ch) {  // second walk: the gates
    uint32_t m = token_mask_chunk(bm, E, W, w, ch, lane);
    while (m) {
      const int e = 32 * ch + __ffs(m) - 1;
      m &= m - 1;
      const float sv = __ldg(srow + e);
      row_gate[token_rows[j++]] = gate_raw ? sv : sv * inv;
    }
    __syncwarp();
  }
}

// One block per word, one warp per 32-expert chunk (E <= 1024): the chunk masks, per-chunk counts
// and partial gate sums go through shared memory; warp 0 forms rowptr and the gate scale; then each
// warp writes its chunk's rows at base + (counts of the lower chunks).
__global__ void k_csr_rows_chunked(const uint32_t* __restrict__ bm, const int* __restrict__ wprefix, int T, int E,
                                   int W, const int* __restrict__ pad_offsets, const int* __restrict__ word_pref,
                                   const float* __restrict__ S, int gate_raw, int* __restrict__ rowptr,
                                   int* __restrict__ token_rows, float* __restrict__ row_gate) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  __shared__ int s_cnt[32][33];
  __shared__ float s_sum[32][33];
  __shared__ int s_base[32];
  __shared__ float s_inv[32];
  const int w = blockIdx.x, ch = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = blockDim.x >> 5;
  const int t = w * 32 + lane;
  const float* srow = S + (size_t)t * E;
  const uint32_t m = token_mask_chunk(bm, E, W, w, ch, lane);
  float ps = 0.f;
  for (uint32_t mm = m; mm; mm &= mm - 1) ps += __ldg(srow + 32 * ch + __ffs(mm) - 1);
  s_cnt[ch][lane] = __popc(m);
  s_sum[ch][lane] = ps;
  __syncthreads();
  if (ch == 0) {
    int tot = 0;
    float sum = 0.f;
    for (int c = 0; c < nch; ++c) {
      tot += s_cnt[c][lane];
      sum += s_sum[c][lane];
    }
    int incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int base = word_pref[w] + incl - tot;
    if (t < T) rowptr[t] = base;
    s_base[lane] = base;
    s_inv[lane] = (gate_raw || sum == 0.f) ? 1.f : 1.f / sum;
  }
  __syncthreads();
  int j = s_base[lane];
  for (int c = 0; c < ch; ++c) j += s_cnt[c][lane];
  const float inv = s_inv[lane];
  const uint32_t below = (1u << lane) - 1u;
  for (uint32_t mm = m; mm; mm &= mm - 1) {
    const int e = 32 * ch + __ffs(mm) - 1;
    const uint32_t word = __ldg(bm + (size_t)e * W + w);
    const int r = pad_offsets[e] + wprefix[(size_t)e * W + w] + __popc(word & below);
    token_rows[j++] = r;
    const float sv = __ldg(srow + e);
    row_gate[r] = gate_raw ? sv : sv * inv;
  }
}


// One block, tiles of 4 x 1024 values: thread i holds values [4i, 4i+4) of the tile (coalesced
// loads), a block scan of the per-thread sums plus the running carry gives the exclusive prefix.
__global__ void __launch_bounds__(1024) k_scan_tokens(const int* __restrict__ cnt, int T, int* __restrict__ rowptr) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  int carry = 0;
  for (int base = 0; base < T; base += 4 * (int)blockDim.x) {
    const int i0 = base + 4 * (int)threadIdx.x;
    int v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = i0 + k < T ? __ldg(cnt + i0 + k) : 0;
    int tot;
    int run = carry + block_excl_scan(v[0] + v[1] + v[2] + v[3], &tot);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (i0 + k < T) rowptr[i0 + k] = run;
      run += v[k];
    }
    carry += tot;
    __syncthreads();  // block_excl_scan's shared partials are reused by the next tile
  }
  if (threadIdx.x == 0) rowptr[T] = carry;
}

void launch_popc(const uint32_t* bm, int W, int nrows, int* wprefix, int* cnt, cudaStream_t st) {
  launch_k(k_expert_popc, nrows, 1024, 0, st, bm, W, wprefix, cnt, nullptr);
}
void launch_scan_tokens(const int* cnt, int T, int* rowptr, cudaStream_t st) {
  launch_k(k_scan_tokens, 1, 1024, 0, st, cnt, T, rowptr);
}

// ---------------------------------------------------------------- given routing
// SONIC_ROUTE_GIVEN ("an interface that accepts arbitrary routing input"): S is the gate
// matrix itself, token t is routed to e iff S[t,e] is not +0.0 (so a routed pair whose gate is exactly
// zero travels as -0.0 and keeps its row: its dS = <dA', A> is not zero).  One block per 32-token word.
__global__ void k_given_bitmap(const float* __restrict__ S, int T, int E, int W, uint32_t* __restrict__ bm,
                               unsigned* __restrict__ ticket) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  __shared__ uint32_t words[4096];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ticket[0] = 0u;
    ticket[1] = 0u;
  }
  for (int e = threadIdx.x; e < E; e += blockDim.x) words[e] = 0u;
  __syncthreads();
  for (int i = threadIdx.x; i < 32 * E; i += blockDim.x) {
    const int tl = i / E, e = i - tl * E;
    const int t = blockIdx.x * 32 + tl;
    if (t < T && __float_as_uint(S[(size_t)t * E + e]) != 0u) atomicOr(&words[e], 1u << tl);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) bm[(size_t)e * W + blockIdx.x] = words[e];
}

// GIVEN routing with a capacity (the host-sync-free EP receive side, NEXT-2): one block counts the
// routed pairs in the bitmap; more than `cap` would overflow the rows sized from rows_cap, so the
// bitmap is cleared (the routing becomes empty: nothing is written out of bounds, every GEMM and
// aggregation sees zero rows) and *overflow = 1 tells the caller the step is invalid; else 0.
__global__ void __launch_bounds__(1024) k_given_guard(uint32_t* __restrict__ bm, long long nwords, long long cap,
                                                      int* __restrict__ overflow) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  __shared__ unsigned long long s_tot;
  if (threadIdx.x == 0) s_tot = 0ull;
  __syncthreads();
  unsigned long long c = 0;
  for (long long i = threadIdx.x; i < nwords; i += blockDim.x) c += __popc(bm[i]);
  atomicAdd(&s_tot, c);
  __syncthreads();
  const bool over = s_tot > (unsigned long long)cap;
  if (over)
    for (long long i = threadIdx.x; i < nwords; i += blockDim.x) bm[i] = 0u;
  if (threadIdx.x == 0) *overflow = over ? 1 : 0;
}

// ---------------------------------------------------------------- TC top-K helpers
// Inverse of ord_f32 (the ordered key of a non-negative-zero float gives the float back).
__device__ __forceinline__ float unord_f32(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}
// Four interleaved lists per thread (expert e goes to list e mod 4) give the insertion chains
// 4-way ILP; the lists are then merged on unique 64-bit keys (ordered score << 32 | ~expert) by
// bitonic merges, which keep the same total order.
template <int KP>
__device__ __forceinline__ void bitonic_merge_desc(unsigned long long (&a)[KP], const unsigned long long (&b)[KP]) {
#pragma unroll
  for (int i = 0; i < KP; ++i) a[i] = a[i] > b[KP - 1 - i] ? a[i] : b[KP - 1 - i];
#pragma unroll
  for (int d = KP / 2; d >= 1; d >>= 1) {
#pragma unroll
    for (int i = 0; i < KP; ++i) {
      if ((i & d) == 0) {
        const unsigned long long x = a[i], y = a[i + d];
        a[i] = x > y ? x : y;
        a[i + d] = x > y ? y : x;
      }
    }
  }
}

// TC rows in one launch: blocks [0, nb_build) build the gather map (k_build_rows' work, expert
// e = b / nbw); the rest are one thread per (token, k): the TC token CSR (rowptr = t K, rows in
// ascending expert order = rank of the expert among the token's K) and the renormalised gate.
__global__ void k_rows_tc(const uint32_t* __restrict__ bm, const int* __restrict__ wprefix, int W,
                          const int* __restrict__ f_r, const int* __restrict__ pad_offsets, int* __restrict__ row_token,
                          float* __restrict__ row_gate, const int* __restrict__ topk_ids,
                          const float* __restrict__ topk_s, int T, int K, int gate_raw, int* __restrict__ rowptr,
                          int* __restrict__ token_rows, int nb_build, int nbw) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  if ((int)blockIdx.x < nb_build) {
    const int e = blockIdx.x / nbw;
    const int wb = blockIdx.x - e * nbw;
    const int base = pad_offsets[e];
    const int w = wb * blockDim.x + threadIdx.x;
    if (w < W) {
      uint32_t bits = bm[(size_t)e * W + w];
      int r = base + wprefix[(size_t)e * W + w];
      while (bits) {
        const int b = __ffs(bits) - 1;
        row_token[r++] = w * 32 + b;
        bits &= bits - 1;
      }
    }
    if (wb == 0) {  // pad rows of this expert's last tile
      for (int r = base + f_r[e] + threadIdx.x; r < pad_offsets[e + 1]; r += blockDim.x) {
        row_token[r] = -1;
        row_gate[r] = 0.f;
      }
    }
    return;
  }
  const long long i = (long long)(blockIdx.x - nb_build) * blockDim.x + threadIdx.x;
  const long long TK = (long long)T * K;
  if (i > TK) return;
  if (i == TK) {
    rowptr[T] = (int)TK;
    return;
  }
  const int t = (int)(i / K), k = (int)(i - (long long)t * K);
  if (k == 0) rowptr[t] = t * K;
  const int* ids = topk_ids + (size_t)t * K;
  const float* sc = topk_s + (size_t)t * K;
  const int me = ids[k];
  const float ms = sc[k];
  int pos = 0;
  float sum = 0.f;
  for (int j = 0; j < K; ++j) {
    pos += ids[j] < me;
    sum += sc[j];
  }
  const float inv = (gate_raw || sum == 0.f) ? 1.f : 1.f / sum;
  const int w = t >> 5;
  const uint32_t below = (1u << (t & 31)) - 1u;
  const int r = pad_offsets[me] + wprefix[(size_t)me * W + w] + __popc(bm[(size_t)me * W + w] & below);
  token_rows[(size_t)t * K + pos] = r;
  row_gate[r] = gate_raw ? ms : ms * inv;
}

// Four threads per token (32 tokens per 128-thread block = one bitmap word): thread g of a token
// scans experts g, g+4, g+8, ... (row stride 132 words: the 32 lanes of a warp hit 32 distinct
// banks) with one stable insertion list, then two shuffle rounds of bitonic merges on the unique
// 64-bit keys give every thread of the token its top-KT.
constexpr int TG_TOK = 32, TG_EC = 128, TG_STRIDE = TG_EC + 4;
// threads per token of the top-K (4 or 8): each scans every TPT-th expert into its own sorted list,
// then log2(TPT) shuffle rounds of bitonic merges
#ifndef SONIC_TOPK_TPT
#define SONIC_TOPK_TPT 4
#endif
template <int KT>
__global__ void __launch_bounds__(32 * SONIC_TOPK_TPT) k_topk_g4(const float* __restrict__ S, int T, int E, int W,
                                                 int* __restrict__ topk_ids, float* __restrict__ topk_s,
                                                 uint32_t* __restrict__ bm_tc, unsigned* __restrict__ ticket,
                                                 float* __restrict__ ST) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  constexpr int KP = KT <= 1 ? 1 : KT <= 2 ? 2 : KT <= 4 ? 4 : KT <= 8 ? 8 : 16;
  extern __shared__ float tg_sm[];  // [TG_TOK][TG_STRIDE] staging, then words [E]
  uint32_t* words = reinterpret_cast<uint32_t*>(tg_sm + TG_TOK * TG_STRIDE);
  constexpr int TPT = SONIC_TOPK_TPT, NT = 32 * TPT;  // threads per token, per block
  const int tid = threadIdx.x, tl = tid / TPT, g = tid % TPT;
  const int tok0 = blockIdx.x * TG_TOK;
  const int ntok = min(TG_TOK, T - tok0);
  if (blockIdx.x == 0 && tid == 0 && ticket) {
    ticket[0] = 0u;
    ticket[1] = 0u;
  }
  for (int i = tid; i < E; i += NT) words[i] = 0u;
  uint32_t top[KP];
  int id[KP];
#pragma unroll
  for (int i = 0; i < KP; ++i) {
    top[i] = 0u;
    id[i] = 0;
  }
  for (int e0 = 0; e0 < E; e0 += TG_EC) {
    const int ecn = min(TG_EC, E - e0);
    __syncthreads();
    if (ecn == TG_EC && (E & 3) == 0) {
#pragma unroll 4
      for (int i = tid; i < ntok * (TG_EC / 4); i += NT) {
        const int r = i / (TG_EC / 4), c4 = i % (TG_EC / 4);
        const float4 v = __ldg(reinterpret_cast<const float4*>(S + (size_t)(tok0 + r) * E + e0) + c4);
        *reinterpret_cast<float4*>(tg_sm + r * TG_STRIDE + 4 * c4) = v;
      }
    } else {
      for (int r = 0; r < ntok; ++r)
        for (int ec = tid; ec < ecn; ec += NT) tg_sm[r * TG_STRIDE + ec] = __ldg(S + (size_t)(tok0 + r) * E + e0 + ec);
    }
    __syncthreads();
    if (ST) {  // TR: the transposed scores S^T [E, T] for the per-expert selection, from the same slab
      const int wp = tid >> 5, ln = tid & 31;
      for (int ec = wp; ec < ecn; ec += NT / 32)
        if (ln < ntok) ST[(size_t)(e0 + ec) * T + tok0 + ln] = tg_sm[ln * TG_STRIDE + ec];
    }
    if (tl < ntok) {
      const float* row = tg_sm + tl * TG_STRIDE;
      for (int ec = g; ec < ecn; ec += TPT) {
        const uint32_t v = ord_f32(row[ec]);
        if (v > top[KP - 1]) {
          const int e = e0 + ec;
#pragma unroll
          for (int i = KP - 1; i > 0; --i) {
            const bool gi = v > top[i], gp = v > top[i - 1];
            top[i] = gi ? (gp ? top[i - 1] : v) : top[i];
            id[i] = gi ? (gp ? id[i - 1] : e) : id[i];
          }
          if (v > top[0]) {
            top[0] = v;
            id[0] = e;
          }
        }
      }
    }
  }
  unsigned long long key[KP];
#pragma unroll
  for (int i = 0; i < KP; ++i)
    key[i] = top[i] ? ((unsigned long long)top[i] << 32) | (0xFFFFFFFFu - (uint32_t)id[i]) : 0ull;
#pragma unroll
  for (int m = 1; m < TPT; m <<= 1) {
    unsigned long long other[KP];
#pragma unroll
    for (int i = 0; i < KP; ++i) other[i] = __shfl_xor_sync(0xffffffffu, key[i], m);
    bitonic_merge_desc<KP>(key, other);
  }
  if (tl < ntok) {
    const size_t t = (size_t)(tok0 + tl);
#pragma unroll
    for (int i = 0; i < KT; ++i) {
      if (i % TPT != g) continue;  // the token's TPT threads share the writes
      const int e = (int)(0xFFFFFFFFu - (uint32_t)(key[i] & 0xFFFFFFFFull));
      topk_ids[t * KT + i] = e;
      topk_s[t * KT + i] = unord_f32((uint32_t)(key[i] >> 32));
      atomicOr(&words[e], 1u << tl);
    }
  }
  __syncthreads();
  for (int e = tid; e < E; e += NT) bm_tc[(size_t)e * W + blockIdx.x] = words[e];
}

// ---------------------------------------------------------------- fused router softmax
// S_t = softmax(logits_t) in fp32 for one token held by a warp, lane l owning experts l, l + 32, ...
// (epl per lane): max via the exact ordered-key warp max, e_j = expf(l_j - max), the sum lane-local
// in j order then a fixed xor-butterfly across lanes (deterministic, and the same order in every
// kernel that calls this), S_j = e_j / sum (IEEE division).
template <int EPLMAX>
__device__ __forceinline__ void warp_softmax_row(float (&v)[EPLMAX], int epl) {
  uint32_t mk = 0u;
#pragma unroll
  for (int j = 0; j < EPLMAX; ++j)
    if (j < epl) mk = max(mk, ord_f32(v[j]));
  const float mx = unord_f32(__reduce_max_sync(0xffffffffu, mk));
  float sum = 0.f;
#pragma unroll
  for (int j = 0; j < EPLMAX; ++j) {
    if (j < epl) {
      v[j] = expf(v[j] - mx);
      sum += v[j];
    }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
#pragma unroll
  for (int j = 0; j < EPLMAX; ++j)
    if (j < epl) v[j] = __fdiv_rn(v[j], sum);
}

// Row softmax for the paths that cannot fuse it into the top-K (token rounding / expert choice,
// E > SONIC_TOPK_WARP_EMAX or E % 32 != 0): one warp per token, the same arithmetic as the fused
// top-K (E % 32 == 0, E <= 512: bit-identical S); larger or ragged E go through the same
// lane-strided order with the values re-read from global memory.
template <int EPLMAX>
__global__ void __launch_bounds__(256) k_softmax_rows(const float* __restrict__ logits, long long T, int E,
                                                      float* __restrict__ S) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int lane = threadIdx.x & 31;
  const long long t = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= T) return;
  const float* row = logits + t * E;
  float* out = S + t * E;
  const int epl = (E + 31) >> 5;
  if (epl <= EPLMAX && E % 32 == 0) {
    float v[EPLMAX];
#pragma unroll
    for (int j = 0; j < EPLMAX; ++j) v[j] = j < epl ? __ldg(row + 32 * j + lane) : 0.f;
    warp_softmax_row<EPLMAX>(v, epl);
#pragma unroll
    for (int j = 0; j < EPLMAX; ++j)
      if (j < epl) out[32 * j + lane] = v[j];
    return;
  }
  uint32_t mk = 0u;
  for (int j = 0; j < epl; ++j)
    if (32 * j + lane < E) mk = max(mk, ord_f32(__ldg(row + 32 * j + lane)));
  const float mx = unord_f32(__reduce_max_sync(0xffffffffu, mk));
  float sum = 0.f;
  for (int j = 0; j < epl; ++j)
    if (32 * j + lane < E) sum += expf(__ldg(row + 32 * j + lane) - mx);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  for (int j = 0; j < epl; ++j)
    if (32 * j + lane < E) out[32 * j + lane] = __fdiv_rn(expf(__ldg(row + 32 * j + lane) - mx), sum);
}

// TC top-K with one warp per token (E % 32 == 0, E <= 32 * EPLMAX; no S^T output): lane l holds
// experts l, l + 32, ... (coalesced 128-byte loads), keeps its own top min(E/32, KP) keys sorted
// (key = ordered score << 32 | ~expert: unique, so the order is the exact (S desc, expert asc) order
// of Q9), then KT rounds of a two-step warp max (redux.sync on the score half, then on the expert
// half among the lanes holding that score) pop the winners in order.  A block of 8 warps routes 32
// consecutive tokens, i.e. one word of the per-expert bitmaps.
#ifndef SONIC_TOPK_MINB
#define SONIC_TOPK_MINB 1  // min blocks per SM for k_topk_warp's register budget (1 = no constraint)
#endif
template <int KT, int EPLMAX, bool ST_SLAB = false>
__global__ void __launch_bounds__(256, SONIC_TOPK_MINB) k_topk_warp(const float* __restrict__ S, int T, int E, int W,
                                                   int* __restrict__ topk_ids, float* __restrict__ topk_s,
                                                   uint32_t* __restrict__ bm_tc, unsigned* __restrict__ ticket,
                                                   float* __restrict__ S_out, int* __restrict__ cnt_acc,
                                                   float* __restrict__ ST) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  constexpr int KP = KT <= 1 ? 1 : KT <= 2 ? 2 : KT <= 4 ? 4 : KT <= 8 ? 8 : 16;
  constexpr int LL = EPLMAX < KP ? EPLMAX : KP;  // lane list length
  __shared__ uint32_t words[32 * EPLMAX];
  // token rounding / expert choice: S^T [E, T] (expert columns contiguous) through a transposing slab
  __shared__ float slab[ST_SLAB ? 32 : 1][ST_SLAB ? 32 * EPLMAX + 1 : 1];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int tok0 = blockIdx.x * 32;
  const int epl = E >> 5;
  if (blockIdx.x == 0 && threadIdx.x == 0 && ticket) {
    ticket[0] = 0u;
    ticket[1] = 0u;
  }
  for (int i = threadIdx.x; i < E; i += 256) words[i] = 0u;
  // the warp's 4 tokens: all loads first (4 x epl in flight per lane)
  float v[4][EPLMAX];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int t = tok0 + wp + 8 * u;
#pragma unroll
    for (int j = 0; j < EPLMAX; ++j)
      v[u][j] = (t < T && j < epl) ? __ldg(S + (size_t)t * E + 32 * j + lane) : 0.f;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int t = tok0 + wp + 8 * u;
    if (t >= T) continue;  // (uniform per warp)
    if (S_out) {  // softmax fusion: the loaded values are logits; S is written and routed on
      warp_softmax_row<EPLMAX>(v[u], epl);
#pragma unroll
      for (int j = 0; j < EPLMAX; ++j)
        if (j < epl) S_out[(size_t)t * E + 32 * j + lane] = v[u][j];
    }
    if constexpr (ST_SLAB) {
      if (ST) {
#pragma unroll
        for (int j = 0; j < EPLMAX; ++j)
          if (j < epl) slab[t - tok0][32 * j + lane] = v[u][j];
      }
    }
    unsigned long long lst[LL];
#pragma unroll
    for (int i = 0; i < LL; ++i) lst[i] = 0ull;
#pragma unroll
    for (int j = 0; j < EPLMAX; ++j) {
      if (j >= epl) break;
      const unsigned long long k =
          ((unsigned long long)ord_f32(v[u][j]) << 32) | (0xFFFFFFFFu - (uint32_t)(32 * j + lane));
      if (k > lst[LL - 1]) {
#pragma unroll
        for (int i = LL - 1; i > 0; --i) {
          const bool gi = k > lst[i], gp = k > lst[i - 1];
          lst[i] = gi ? (gp ? lst[i - 1] : k) : lst[i];
        }
        if (k > lst[0]) lst[0] = k;
      }
    }
    int my_e = 0;
    uint32_t my_s = 0;
#pragma unroll
    for (int r = 0; r < KT; ++r) {
      const uint32_t hi = (uint32_t)(lst[0] >> 32);
      const uint32_t m = __reduce_max_sync(0xffffffffu, hi);
      const uint32_t lo = hi == m ? (uint32_t)lst[0] : 0u;
      const uint32_t ml = __reduce_max_sync(0xffffffffu, lo);
      if (hi == m && lo == ml) {  // the winner pops its head
#pragma unroll
        for (int i = 0; i < LL - 1; ++i) lst[i] = lst[i + 1];
        lst[LL - 1] = 0ull;
      }
      if (lane == r) {
        my_e = (int)(0xFFFFFFFFu - ml);
        my_s = m;
      }
    }
    if (lane < KT) {
      topk_ids[(size_t)t * KT + lane] = my_e;
      topk_s[(size_t)t * KT + lane] = unord_f32(my_s);
      atomicOr(&words[my_e], 1u << (t - tok0));
    }
  }
  __syncthreads();
  if constexpr (ST_SLAB) {
    if (ST) {  // warp w writes experts w, w + 8, ...: one 128-byte row of 32 tokens each
      const int ntok = min(32, T - tok0);
      if (lane < ntok)
        for (int e = wp; e < E; e += 8) ST[(size_t)e * T + tok0 + lane] = slab[lane][e];
    }
  }
  for (int e = threadIdx.x; e < E; e += 256) {
    const uint32_t wd = words[e];
    bm_tc[(size_t)e * W + blockIdx.x] = wd;
    if (cnt_acc && wd) atomicAdd(cnt_acc + e, __popc(wd));  // f_e, for the one-pass TC build
  }
}

// TC index build in ONE launch after k_topk_warp (whose count atomics give every f_e): block e
// (1024 threads) takes the exclusive prefixes of f, of the 128-row padded counts and of the 2-CTA
// pair counts over all experts (so each block knows its own offsets: no second grid-wide pass), then
// builds its segment -- the gather map from a popcount scan of its bitmap words, its pad rows, its
// tiles and tile pairs -- and, for every token of the segment, the token-CSR entry (the expert's
// rank among the token's K, ascending) and the renormalised gate.  Same outputs as k_popc_offsets +
// k_rows_tc.
constexpr int TCB_THREADS = 256;  // k_tc_build: threads per block = bitmap words per block
// SONIC_TC_BUILD1=1: the TC route in two launches (k_topk_warp with count atomics + k_tc_build instead of
// k_popc_offsets + k_rows_tc).  Parity green, but measured slower at 7B (route 27.3 -> 35.0 us with one
// block per expert, 39.0 us with 256-word blocks: the memset before the top-K breaks the PDL chain and
// 1024 blocks' count atomics contend on E addresses), so the three-launch build stays the default.
#ifndef SONIC_TC_BUILD1
#define SONIC_TC_BUILD1 0
#endif
__global__ void __launch_bounds__(TCB_THREADS) k_tc_build(const uint32_t* __restrict__ bm, int W, const int* __restrict__ cnt_in,
                                                   int E, int K, long long T, const int* __restrict__ topk_ids,
                                                   const float* __restrict__ topk_s, int gate_raw, int* __restrict__ f,
                                                   int* __restrict__ f_r, int* __restrict__ offsets,
                                                   int* __restrict__ pad_offsets, int* __restrict__ row_token,
                                                   float* __restrict__ row_gate, int* __restrict__ rowptr,
                                                   int* __restrict__ token_rows, int* __restrict__ tile_expert,
                                                   int* __restrict__ num_tiles, int* __restrict__ tile_pairs,
                                                   int* __restrict__ num_pairs) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  __shared__ int s_off, s_pad, s_pair, s_tot_off, s_tot_pad, s_tot_pair;
  const int e = blockIdx.x;
  const int chunk = blockIdx.y;  // this block's words: [chunk * TCB_THREADS, +TCB_THREADS)
  // prefixes over the experts (E <= TCB_THREADS here: one block scan)
  {
    const int x = threadIdx.x;
    const int c = x < E ? __ldcg(cnt_in + x) : 0;
    const int pc = (c + GEMM_M - 1) / GEMM_M * GEMM_M;
    const int pp = (pc / GEMM_M + 1) / 2;
    int t0, t1, t2;
    const int ex = block_excl_scan(c, &t0);
    const int pex = block_excl_scan(pc, &t1);
    const int ppx = block_excl_scan(pp, &t2);
    if (x == e) {
      s_off = ex;
      s_pad = pex;
      s_pair = ppx;
    }
    if (x == 0) {
      s_tot_off = t0;
      s_tot_pad = t1;
      s_tot_pair = t2;
    }
  }
  __syncthreads();
  const int cnt = __ldcg(cnt_in + e);
  const int pad0 = s_pad, pc = (cnt + GEMM_M - 1) / GEMM_M * GEMM_M;
  // rows of this expert before this block's words: popcount of the words [0, chunk * TCB_THREADS)
  int before = 0;
  {
    int c = 0;
    for (int w = threadIdx.x; w < chunk * TCB_THREADS; w += blockDim.x) c += __popc(bm[(size_t)e * W + w]);
    int tot;
    block_excl_scan(c, &tot);
    before = tot;
  }
  if (threadIdx.x == 0 && chunk == 0) {
    f[e] = cnt;
    f_r[e] = cnt;
    offsets[e] = s_off;
    pad_offsets[e] = pad0;
    if (e == E - 1) {
      offsets[E] = s_tot_off;
      pad_offsets[E] = s_tot_pad;
      *num_tiles = s_tot_pad / GEMM_M;
      *num_pairs = s_tot_pair;
    }
  }
  if (chunk == 0) {
    const int tiles_e = pc / GEMM_M, tile0 = pad0 / GEMM_M;
    for (int i = threadIdx.x; i < tiles_e; i += blockDim.x) tile_expert[tile0 + i] = e;
    for (int j = threadIdx.x; 2 * j < tiles_e; j += blockDim.x)
      tile_pairs[s_pair + j] = (tile0 + 2 * j) | ((2 * j + 1 < tiles_e) ? (int)0x80000000u : 0);
    for (int r = pad0 + cnt + threadIdx.x; r < pad0 + pc; r += blockDim.x) {  // pad rows of the last tile
      row_token[r] = -1;
      row_gate[r] = 0.f;
    }
  }
  {
    const long long nb = (long long)E * gridDim.y, b = (long long)chunk * E + e;
    for (long long t = b + (long long)threadIdx.x * nb; t <= T; t += (long long)blockDim.x * nb)
      rowptr[t] = (int)(t * K);  // TC: every token has K rows
  }
  // this block's part of the segment: ascending tokens from a popcount scan of its words
  int base = pad0 + before;
  {
    const int w0 = chunk * TCB_THREADS;
    const int w = w0 + threadIdx.x;
    uint32_t bits = w < W ? bm[(size_t)e * W + w] : 0u;
    int tot;
    int r = base + block_excl_scan(__popc(bits), &tot);
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      const int t = w * 32 + b;
      row_token[r] = t;
      const int* ids = topk_ids + (size_t)t * K;
      const float* sc = topk_s + (size_t)t * K;
      int pos = 0;
      float sum = 0.f, ms = 0.f;
      for (int j = 0; j < K; ++j) {
        const int id = ids[j];
        pos += id < e;
        sum += sc[j];
        if (id == e) ms = sc[j];
      }
      const float inv = (gate_raw || sum == 0.f) ? 1.f : 1.f / sum;
      token_rows[(size_t)t * K + pos] = r;
      row_gate[r] = gate_raw ? ms : ms * inv;
      ++r;
    }
  }
}

#ifndef SONIC_TOPK_WARP
#define SONIC_TOPK_WARP 1  // TC: the warp-per-token top-K (E % 32 == 0, E <= SONIC_TOPK_WARP_EMAX); 0 = k_topk_g4 always
#endif
#ifndef SONIC_TOPK_WARP_EMAX
#define SONIC_TOPK_WARP_EMAX 128
#endif
#ifndef SONIC_TOPK_WARP_ST
#define SONIC_TOPK_WARP_ST 1  // token rounding / expert choice also on the warp top-K (S^T through a smem slab)
#endif

template <int KT>
int launch_topk_g4(const RouteLaunch& L, cudaStream_t st) {
  const int T = (int)L.T, E = L.E, W = L.W;
  const int smem = (TG_TOK * TG_STRIDE + E) * 4;
  static int attr[64] = {};  // per device (function attributes are per context)
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr[dev & 63] < smem) {
    cudaFuncSetAttribute(k_topk_g4<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr[dev & 63] = smem;
  }
  // token rounding / expert choice read S^T: written here from the staged slab (no separate transpose)
  float* st_out = (L.mode == 1 || L.mode == 3) ? L.ST : nullptr;
  // warp per token: 7B / Qwen3 (E = 128) route 32.7 -> 27.3 us; at E = 384 (Kimi) slower than the
  // four-threads-per-token kernel (92.7 -> 106.3 us), so only for E <= SONIC_TOPK_WARP_EMAX
  if (SONIC_TOPK_WARP && (!st_out || SONIC_TOPK_WARP_ST) && E % 32 == 0 && E <= SONIC_TOPK_WARP_EMAX) {
    // with logits (sonic_route_logits) the softmax is fused here: reads logits, writes S, routes on S
    const float* in = L.logits ? L.logits : L.S;
    float* s_out = L.logits ? const_cast<float*>(L.S) : nullptr;
    // TC: the per-expert counts accumulate here (zeroed first) for the one-launch build, k_tc_build
    int* acc = (SONIC_TC_BUILD1 && L.mode == 0 && E <= TCB_THREADS) ? L.tokcnt : nullptr;
    if (acc) cudaMemsetAsync(acc, 0, (size_t)E * 4, st);
    if (st_out) {  // token rounding / expert choice: S^T written through the slab
      if (E <= 128)
        launch_k(k_topk_warp<KT, 4, true>, W, 256, 0, st, in, T, E, W, L.topk_ids, L.topk_s, L.bm_tc, L.ticket, s_out,
                 acc, st_out);
      else
        launch_k(k_topk_warp<KT, 8, true>, W, 256, 0, st, in, T, E, W, L.topk_ids, L.topk_s, L.bm_tc, L.ticket, s_out,
                 acc, st_out);
    } else if (E <= 128) {
      launch_k(k_topk_warp<KT, 4>, W, 256, 0, st, in, T, E, W, L.topk_ids, L.topk_s, L.bm_tc, L.ticket, s_out, acc,
               (float*)nullptr);
    } else {
      launch_k(k_topk_warp<KT, 8>, W, 256, 0, st, in, T, E, W, L.topk_ids, L.topk_s, L.bm_tc, L.ticket, s_out, acc,
               (float*)nullptr);
    }
    return 1;
  }
  int nl = 1;
  if (L.logits) {  // no fused top-K for this mode / E: the row softmax first, then the top-K on S
    launch_k(k_softmax_rows<16>, (int)((L.T + 7) / 8), 256, 0, st, L.logits, L.T, E, const_cast<float*>(L.S));
    ++nl;
  }
  launch_k(k_topk_g4<KT>, W, 32 * SONIC_TOPK_TPT, smem, st, L.S, T, E, W, L.topk_ids, L.topk_s, L.bm_tc, L.ticket,
           st_out);
  return nl;
}

int launch_topk(const RouteLaunch& L, cudaStream_t st) {
  switch (L.K) {
#define TKC(k) case k: return launch_topk_g4<k>(L, st);
    TKC(1) TKC(2) TKC(3) TKC(4) TKC(5) TKC(6) TKC(7) TKC(8)
    TKC(9) TKC(10) TKC(11) TKC(12) TKC(13) TKC(14) TKC(15) TKC(16)
#undef TKC
    default: return 0;
  }
}

// token CSR from a kept-bitmap: counts + word scan (ticket: zeroed here), then rows and gates
void launch_csr(const uint32_t* bm, const RouteLaunch& L, int gate_raw, cudaStream_t st) {
  const int T = (int)L.T, E = L.E, W = L.W;
  const int blocks = (W * 32 + 255) / 256;
  launch_k(k_csr_count, blocks, 256, 0, st, bm, T, E, W, L.tokcnt, L.token_rowptr, L.ticket + 1);
  const int nch = (E + 31) / 32;
  if (nch <= 32)
    launch_k(k_csr_rows_chunked, W, 32 * nch, 0, st, bm, L.wprefix, T, E, W, L.pad_offsets, L.tokcnt, L.S, gate_raw,
                                               L.token_rowptr, L.token_rows, L.row_gate);
  else
    launch_k(k_csr_rows, blocks, 256, 0, st, bm, L.wprefix, T, E, W, L.pad_offsets, L.tokcnt, L.S, gate_raw,
                                       L.token_rowptr, L.token_rows, L.row_gate);
}

// ---------------------------------------------------------------- launcher
int launch_route(const RouteLaunch& L, cudaStream_t st) {
  int nl = 0;
  const int T = (int)L.T, E = L.E, K = L.K, W = L.W;
  if (L.mode == 2) {  // given routing: bitmap, counts, offsets, rows, CSR with raw gates
    launch_k(k_given_bitmap, W, 256, 0, st, L.S, T, E, W, L.bm_tc, L.ticket); ++nl;
    if (L.overflow) {
      launch_k(k_given_guard, 1, 1024, 0, st, L.bm_tc, (long long)E * W, L.cap, L.overflow);
      ++nl;
    }
    launch_k(k_popc_offsets, E, 1024, 0, st, L.bm_tc, W, L.wprefix, L.f, L.f_r, L.ticket, L.offsets, L.pad_offsets,
                                       L.tile_expert, L.num_tiles, L.tile_pairs, L.num_pairs); ++nl;
    launch_k(k_build_rows, dim3((W + 255) / 256, E), 256, 0, st, L.bm_tc, L.wprefix, W, L.f_r, L.pad_offsets,
                                                           L.row_token, L.row_gate); ++nl;
    launch_csr(L.bm_tc, L, 1, st);
    nl += 2;
    return nl;
  }
  nl += launch_topk(L, st);  // K <= 16 (validated for TC / TR); + the row softmax with logits
  if (SONIC_TC_BUILD1 && L.mode == 0 && SONIC_TOPK_WARP && E % 32 == 0 && E <= SONIC_TOPK_WARP_EMAX &&
      E <= TCB_THREADS) {
    // TC after the warp top-K: the whole index build in one launch (counts from the top-K's atomics)
    launch_k(k_tc_build, dim3(E, (W + TCB_THREADS - 1) / TCB_THREADS), TCB_THREADS, 0, st, L.bm_tc, W,
             (const int*)L.tokcnt, E, K, L.T, L.topk_ids, L.topk_s,
             L.gate_raw, L.f, L.f_r, L.offsets, L.pad_offsets, L.row_token, L.row_gate, L.token_rowptr, L.token_rows,
             L.tile_expert, L.num_tiles, L.tile_pairs, L.num_pairs);
    return nl + 1;
  }
  const uint32_t* bm_kept = L.bm_tc;
  if (L.mode == 1 || L.mode == 3) {  // token rounding (any subroutine) or expert choice
    const bool ec = L.mode == 3;
    int ec_cap = -1;
    if (ec) {  // Q22: ceil(T K / E) rounded up to a tile, capped at T
      const long long avg = ((long long)T * K + E - 1) / E;
      ec_cap = (int)std::min<long long>((avg + L.m_tile - 1) / L.m_tile * L.m_tile, T);
    }
    const bool nrs = !ec && L.rounding == 5;
    if (!nrs && (ec || L.rounding != 3)) {  // per-expert decision: fused with the count
      launch_k(k_expert_popc_decide, E, 1024, 0, st, L.bm_tc, W, L.f, L.f_r, T, L.m_tile, L.rounding, L.seed, ec_cap);
      ++nl;
    } else {
      launch_k(k_expert_popc, E, 1024, 0, st, L.bm_tc, W, nullptr, L.f, nullptr); ++nl;
      if (!nrs) {  // Balance-f: one sequential pass over the experts
        launch_k(k_tr_decide, (E + 255) / 256, 256, 0, st, L.f, L.f_r, E, T, L.m_tile, L.rounding, L.seed, ec_cap);
        ++nl;
      }
    }
    auto select_into = [&](int rescue, uint32_t* out, const int* fr_src) {
      if (W <= 1024)
        launch_k(k_tr_select_w<true>, E, 1024, 0, st, L.ST, T, W, L.m_tile, L.bm_tc, out, L.f, L.f_r, L.flip,
                 rescue, ec ? 1 : 0, fr_src);
      else
        launch_k(k_tr_select_w<false>, E, 1024, 0, st, L.ST, T, W, L.m_tile, L.bm_tc, out, L.f, L.f_r, L.flip,
                 rescue, ec ? 1 : 0, fr_src);
    };
    auto select = [&](int rescue) { select_into(rescue, L.bm_kept, nullptr); };
    if (nrs) {  // NR-s: both candidate selections, their score sums, then the draw
      launch_k(k_nrs_counts, (E + 255) / 256, 256, 0, st, L.f, E, T, L.m_tile, L.f_dn, L.f_up); ++nl;
      select_into(0, L.bm_dn, L.f_dn); ++nl;
      select_into(0, L.bm_up, L.f_up); ++nl;
      launch_k(k_bitmap_sums, E, 256, 0, st, L.ST, L.bm_tc, T, W, L.nrs_sums); ++nl;
      launch_k(k_bitmap_sums, E, 256, 0, st, L.ST, L.bm_dn, T, W, L.nrs_sums + E); ++nl;
      launch_k(k_bitmap_sums, E, 256, 0, st, L.ST, L.bm_up, T, W, L.nrs_sums + 2 * E); ++nl;
      launch_k(k_nrs_decide, E, 256, 0, st, L.f, L.f_dn, L.f_up, L.nrs_sums, L.nrs_sums + E, L.nrs_sums + 2 * E,
               L.bm_dn, L.bm_up, W, L.seed, L.f_r, L.bm_kept); ++nl;
    } else {
      select(0);
      ++nl;
    }
    if (L.rescue && !ec) {
      cudaMemsetAsync(L.flip, 0, (size_t)E * 4, st);
      launch_k(k_orphans, (W * 32 + 255) / 256, 256, 0, st, L.bm_kept, T, E, W, K, L.topk_ids, L.flip); ++nl;
      select(1);
      ++nl;
    }
    bm_kept = L.bm_kept;
    launch_k(k_popc_offsets, E, 1024, 0, st, bm_kept, W, L.wprefix, L.f_r, nullptr, L.ticket, L.offsets, L.pad_offsets,
                                       L.tile_expert, L.num_tiles, L.tile_pairs, L.num_pairs); ++nl;
  } else {  // TC: one pass gives f, f_r (== f), the word prefixes and the offsets
    launch_k(k_popc_offsets, E, 1024, 0, st, bm_kept, W, L.wprefix, L.f, L.f_r, L.ticket, L.offsets, L.pad_offsets,
                                       L.tile_expert, L.num_tiles, L.tile_pairs, L.num_pairs); ++nl;
  }
  if (L.mode == 0) {
    const int nbw = (W + 255) / 256;
    const int nb_build = nbw * E;
    const long long tk = (long long)T * K + 1;
    const int nb_tok = (int)((tk + 255) / 256);
    launch_k(k_rows_tc, nb_build + nb_tok, 256, 0, st, bm_kept, L.wprefix, W, L.f_r, L.pad_offsets, L.row_token,
                                                 L.row_gate, L.topk_ids, L.topk_s, T, K, L.gate_raw,
                                                 L.token_rowptr, L.token_rows, nb_build, nbw); ++nl;
  } else {
    launch_k(k_build_rows, dim3((W + 255) / 256, E), 256, 0, st, bm_kept, L.wprefix, W, L.f_r, L.pad_offsets,
                                                           L.row_token, L.row_gate); ++nl;
    launch_csr(bm_kept, L, L.gate_raw, st);
    nl += 2;
  }
  return nl;
}

}  // namespace sonic
