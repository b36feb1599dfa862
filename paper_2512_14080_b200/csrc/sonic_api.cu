#include <cstdio>
// sonic_api.cu -- the C ABI of include/sonic.h: validation, workspace layout, TMA tensor
// maps, and the launch sequences of sonic_route / sonic_moe_fwd / sonic_moe_bwd.
#include <cuda.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "../../include/sonic.h"
#include "gemm.cuh"
#include "updown.cuh"
#include "sonic_internal.h"

using namespace sonic;

namespace {

thread_local int g_launches = 0;

// ---------------------------------------------------------------- optional per-kernel timing
// When enabled (sonic_profile_enable), every launch is bracketed by CUDA events on its
// stream; sonic_profile_collect() returns the per-name durations.  Used by bench.py to time
// the dominant kernel live inside the timed region.
struct ProfRec {
  const char* name;
  cudaEvent_t a, b;
};
thread_local bool g_prof = false;
thread_local std::vector<ProfRec> g_recs;
thread_local std::vector<cudaEvent_t> g_pool;
cudaEvent_t pool_get() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
struct ProfScope {
  cudaStream_t st;
  ProfRec r;
  bool on;
  ProfScope(const char* name, cudaStream_t s) : st(s), on(g_prof) {
    if (on) {
      r.name = name;
      r.a = pool_get();
      r.b = pool_get();
      cudaEventRecord(r.a, st);
    }
  }
  ~ProfScope() {
    if (on) {
      cudaEventRecord(r.b, st);
      g_recs.push_back(r);
    }
  }
};

// ---------------------------------------------------------------- tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encoder() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D row-major [rows, cols] tensor; box {box_cols, box_rows}; 128B swizzle.
bool map2d(CUtensorMap* m, const void* ptr, bool f32, long long rows, long long cols, int box_cols, int box_rows) {
  EncodeTiledFn enc = get_encoder();
  if (!enc) return false;
  const int es = f32 ? 4 : 2;
  cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)(cols * es)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr),
             gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// 2-D row-major [rows, cols] bytes (e4m3); box {box_cols, box_rows}; 128B swizzle.
bool map2d_u8(CUtensorMap* m, const void* ptr, long long rows, long long cols, int box_cols, int box_rows) {
  EncodeTiledFn enc = get_encoder();
  if (!enc) return false;
  cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)cols};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(ptr), gdim, gstride, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// 3-D row-major [E, rows, cols] bytes (e4m3); box {box_cols, box_rows, 1}; 128B swizzle.
bool map3d_u8(CUtensorMap* m, const void* ptr, long long E, long long rows, long long cols, int box_cols, int box_rows) {
  EncodeTiledFn enc = get_encoder();
  if (!enc) return false;
  cuuint64_t gdim[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)E};
  cuuint64_t gstride[2] = {(cuuint64_t)cols, (cuuint64_t)(rows * cols)};
  cuuint32_t box[3] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(ptr), gdim, gstride, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// Wide-store view of a row-major bf16 [rows, cols] output (cols % 64 == 0): 3-D {64 columns, rows,
// column block} with strides {cols * 2, 128} bytes; box {64, 32, G} = G stacked 32 x 128 B swizzled
// staging buffers, i.e. G consecutive 64-column chunks of 32 rows in one TMA store.
bool map_wide(CUtensorMap* m, const void* ptr, long long rows, long long cols, int G) {
  EncodeTiledFn enc = get_encoder();
  if (!enc || cols % 64) return false;
  cuuint64_t gdim[3] = {64, (cuuint64_t)rows, (cuuint64_t)(cols / 64)};
  cuuint64_t gstride[2] = {(cuuint64_t)(cols * 2), 128};
  cuuint32_t box[3] = {64, 32, (cuuint32_t)G};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), gdim, gstride, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// 3-D row-major [E, rows, cols] tensor; box {box_cols, box_rows, 1}; 128B swizzle.
bool map3d(CUtensorMap* m, const void* ptr, bool f32, long long E, long long rows, long long cols, int box_cols,
           int box_rows) {
  EncodeTiledFn enc = get_encoder();
  if (!enc) return false;
  const int es = f32 ? 4 : 2;
  cuuint64_t gdim[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)E};
  cuuint64_t gstride[2] = {(cuuint64_t)(cols * es), (cuuint64_t)(rows * cols * es)};
  cuuint32_t box[3] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr),
             gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

#ifndef SONIC_AGG_DW2_PCT
#define SONIC_AGG_DW2_PCT 0  // SONIC_AGG_FUSE: share of the tokens aggregated inside dW2 (the rest: dW1)
#endif
#ifndef SONIC_BWD_OVERLAP
#define SONIC_BWD_OVERLAP 0  // 7B, same run: 0 -> 2.186 ms, 1 -> 2.180, 3 -> 2.183 / 2.141: no measured gain, so serial (clean per-kernel attribution)
#endif
// One internal non-blocking stream (+ fork/join events) per device, for the backward's
// weight-gradient branch.  Created on first use; calls from several host threads on the same
// device would share it (the library is not meant for that).
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  bool ok = false;
};
SideStream& side_stream() {
  static SideStream per_dev[64];
  int dev = 0;
  cudaGetDevice(&dev);
  SideStream& ss = per_dev[dev & 63];
  if (!ss.ok) {
    ss.ok = cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming) == cudaSuccess;
  }
  return ss;
}

int num_sms() {
  static int per_dev[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int& n = per_dev[dev & 63];
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// ---------------------------------------------------------------- GEMM launch
template <int KIND, int BN, bool CTA2, bool MC = false>
bool launch_gemm_t(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c0, const CUtensorMap& c1,
                   const CUtensorMap& dmap, const GemmArgs& args, int grid, cudaStream_t st) {
  using Cfg = KCfg<KIND, BN, CTA2>;
  auto kern = sonic_gemm_kernel<KIND, BN, CTA2, MC>;
  static bool attr[64] = {};  // function attributes are per device (context)
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr[dev & 63]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM) != cudaSuccess)
      return false;
    attr[dev & 63] = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(gemm_threads<KIND>());
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = MC ? 4 : CTA2 ? 2 : 1;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[1].val.programmaticStreamSerializationAllowed = SONIC_PDL ? 1 : 0;
  cfg.attrs = attrs;
  cfg.numAttrs = 2;
  if constexpr (MC) {
    // 4-CTA clusters must fit in a GPC: launch at most as many as can be co-resident (a multiple
    // of 4 CTAs: the two pairs of a cluster run the same number of pair tiles)
    static int max_cl[64] = {};
    if (!max_cl[dev & 63]) {
      int ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) != cudaSuccess || ncl <= 0) ncl = grid / 4;
      max_cl[dev & 63] = std::max(1, ncl);
    }
    grid = std::max(4, std::min(grid & ~3, 4 * max_cl[dev & 63]));
    cfg.gridDim = dim3(grid);
  }
#ifdef SONIC_TIMING
  static unsigned long long* dbg = nullptr;
  if (!dbg) cudaMalloc(&dbg, 16 * sizeof(unsigned long long));
  cudaMemsetAsync(dbg, 0, 16 * sizeof(unsigned long long), st);
  GemmArgs targs = args;
  targs.dbg = dbg;
  if (cudaLaunchKernelEx(&cfg, kern, a, b, c0, c1, dmap, targs) != cudaSuccess) return false;
  unsigned long long h[16];
  cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  const double n = h[5] ? (double)h[5] : 1.0;
  const double nc = n * (CTA2 ? 2.0 : 1.0);  // CTAs (gathered kinds' producer counters are per CTA)
  fprintf(stderr, "TIMING kind=%d BN=%d cta2=%d: mma_total %.0f  wait_tempty %.0f  wait_full %.0f | epi_wait_tfull %.0f  epi_busy %.0f (kcycles; epilogue counters summed over the pair) | gather producer total %.0f wait_empty %.0f (per CTA)\n",
          KIND, BN, (int)CTA2, h[0] / n / 1e3, h[1] / n / 1e3, h[2] / n / 1e3, h[3] / n / 1e3, h[4] / n / 1e3,
          h[7] / nc / 1e3, h[6] / nc / 1e3);
  if (h[10])
    fprintf(stderr, "TIMING fused aggregation: %.0f kcycles per CTA, waiting on rows %.0f, %.0f cycles per token\n",
            h[8] / nc / 1e3, h[9] / nc / 1e3, (double)h[8] / (double)h[10]);
#else
  const cudaError_t err = cudaLaunchKernelEx(&cfg, kern, a, b, c0, c1, dmap, args);
  if (err != cudaSuccess) {
    fprintf(stderr, "libsonic: sonic_gemm_kernel<%d,%d,%d> launch failed: %s\n", KIND, BN, (int)CTA2,
            cudaGetErrorString(err));
    return false;
  }
#endif
  ++g_launches;
  return true;
}

// 2-CTA (cta_group::2) tiles for every GEMM whose N tile is >= 128 (SONIC_CTA2=0 disables).
#ifndef SONIC_CTA2
#define SONIC_CTA2 1
#endif
bool use_cta2(int BN) { return SONIC_CTA2 && BN >= 128; }

// 4-CTA multicast clusters (MC, gemm.cuh) for DOWN / DXT / DW2 / DW1 at BN = 256 when the shared
// operand's partner tiles exist (an even tile count along the sharing dimension).  SONIC_MC4=0: pairs only.
#ifndef SONIC_MC4
#define SONIC_MC4 0  // measured slower at 7B (dXt 331 -> 354 us, dW1 376 -> 387, dW2 217 -> 226): DESIGN.md 6.8
#endif
// dmap: auxiliary tensor map (DH: the H cache, box {64, 32}; DOWN / DXT with mc: the A operand with
// a 64-row box, the half tile each pair multicasts); ignored by the other kinds.
template <int KIND>
bool launch_gemm(int BN, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c0, const CUtensorMap& c1,
                 const GemmArgs& args, int grid, cudaStream_t st, const CUtensorMap* dmap = nullptr, bool mc = false) {
  const CUtensorMap& d = dmap ? *dmap : c0;
  const bool cta2 = use_cta2(BN);
  if (cta2) grid = std::max(2, grid & ~1);  // a pair needs both CTAs, even for a single pair tile
  if constexpr (KIND == K_UP8 || KIND == K_DXT8) {  // e4m3: 2-CTA pairs of 256 columns only (fp8_*_ok)
    return cta2 && BN == 256 && launch_gemm_t<KIND, 256, true>(a, b, c0, c1, d, args, grid, st);
  } else {
    if constexpr (KIND == K_DOWN || KIND == K_DXT || KIND == K_DW2 || KIND == K_DW1) {
      if (SONIC_MC4 && !g4_kind<KIND>() && mc && cta2 && BN == 256)
        return launch_gemm_t<KIND, 256, true, true>(a, b, c0, c1, d, args, grid, st);
    }
    switch (BN) {
      case 256:
        return cta2 ? launch_gemm_t<KIND, 256, true>(a, b, c0, c1, d, args, grid, st)
                    : launch_gemm_t<KIND, 256, false>(a, b, c0, c1, d, args, grid, st);
      case 128:
        return cta2 ? launch_gemm_t<KIND, 128, true>(a, b, c0, c1, d, args, grid, st)
                    : launch_gemm_t<KIND, 128, false>(a, b, c0, c1, d, args, grid, st);
      case 64: return launch_gemm_t<KIND, 64, false>(a, b, c0, c1, d, args, grid, st);
      case 32:
        if constexpr (KIND == K_DH) return launch_gemm_t<KIND, 32, false>(a, b, c0, c1, d, args, grid, st);
        return false;
      default: return false;
    }
  }
}

template <int NU, int BND>
bool launch_updown(const CUtensorMap& w1, const CUtensorMap& w2, const CUtensorMap& h, const CUtensorMap& y,
                   const UpDownArgs& args, int grid, cudaStream_t st) {
  using Cfg = UpDownCfg<NU, BND>;
  auto kern = sonic_updown_kernel<NU, BND>;
  static bool attr[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr[dev & 63]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM) != cudaSuccess)
      return false;
    attr[dev & 63] = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(std::max(2, grid & ~1));
  cfg.blockDim = dim3(Cfg::THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = 2;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[1].val.programmaticStreamSerializationAllowed = SONIC_PDL ? 1 : 0;
  cfg.attrs = attrs;
  cfg.numAttrs = 2;
#ifdef SONIC_TIMING
  static unsigned long long* dbg = nullptr;
  if (!dbg) cudaMalloc(&dbg, 16 * sizeof(unsigned long long));
  cudaMemsetAsync(dbg, 0, 16 * sizeof(unsigned long long), st);
  UpDownArgs targs = args;
  targs.dbg = dbg;
  if (cudaLaunchKernelEx(&cfg, kern, w1, w2, h, y, targs) != cudaSuccess) return false;
  unsigned long long hc[16];
  cudaMemcpyAsync(hc, dbg, sizeof(hc), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  const double nn = hc[8] ? (double)hc[8] : 1.0;
  fprintf(stderr, "TIMING updown NU=%d BND=%d (kcycles per pair): total %.0f | mma tempty U %.0f D %.0f | full U %.0f D %.0f | "
          "aready %.0f | job span U %.0f D %.0f || epi(w0) wait_tfull %.0f busy U %.0f D %.0f\n",
          NU, BND, hc[0] / nn / 1e3, hc[1] / nn / 1e3, hc[2] / nn / 1e3, hc[3] / nn / 1e3, hc[4] / nn / 1e3,
          hc[5] / nn / 1e3, hc[6] / nn / 1e3, hc[7] / nn / 1e3, hc[9] / nn / 1e3, hc[10] / nn / 1e3, hc[11] / nn / 1e3);
#else
  const cudaError_t err = cudaLaunchKernelEx(&cfg, kern, w1, w2, h, y, args);
  if (err != cudaSuccess) {
    fprintf(stderr, "libsonic: sonic_updown_kernel<%d,%d> launch failed: %s\n", NU, BND, cudaGetErrorString(err));
    return false;
  }
#endif
  ++g_launches;
  return true;
}

int pick_bn(long long N) { return N % 256 == 0 ? 256 : N % 128 == 0 ? 128 : 64; }
// rows of the K-major weight box held by one CTA
int bnl(int BN) { return use_cta2(BN) ? BN / 2 : BN; }

// ---------------------------------------------------------------- shapes & validation
struct Shape {
  long long T, rows_max;
  int d, n, E, K, W;
};

bool valid_desc(const sonic_moe_desc* D) {
  if (!D) return false;
  if (D->T < 1 || D->d < 1 || D->n < 1 || D->E < 1 || D->K < 1) return false;
  if (D->K > D->E || D->E > 4096) return false;
  if (D->K > 16 && D->route_mode != SONIC_ROUTE_GIVEN) return false;
  if (D->m_tile != 128 && D->m_tile != 256) return false;  // one CTA's M tile or a 2-CTA pair's (Q16)
  if (D->route_mode < SONIC_ROUTE_TC || D->route_mode > SONIC_ROUTE_TR_NRS) return false;
  if (D->rows_cap < 0 || (D->rows_cap != 0 && D->route_mode != SONIC_ROUTE_GIVEN)) return false;
  return true;
}
long long rows_max_of(const sonic_moe_desc* D);
bool supported_dims(const sonic_moe_desc* D) {
  if (D->d % 64 != 0) return false;
  if (!(D->n == 32 || D->n % 64 == 0)) return false;
  if (rows_max_of(D) >= (1ll << 31)) return false;
  if ((long long)D->E * D->T >= (1ll << 40)) return false;
  return true;
}
long long rows_max_of(const sonic_moe_desc* D) {
  const long long pairs = (D->route_mode == SONIC_ROUTE_GIVEN && D->rows_cap > 0) ? std::min(D->rows_cap, D->T * D->K)
                                                                                   : D->T * D->K;
  const long long b = (long long)D->E * ((D->T + GEMM_M - 1) / GEMM_M) * GEMM_M;
  if (D->route_mode == SONIC_ROUTE_EC) {
    // expert choice (Q22): every expert keeps exactly C = min(ceil_M(ceil(T K / E)), T) rows, padded
    // to a 128-row tile; E * C can exceed T K by up to E * (m_tile - 1) + E - 1 (same C as launch_route)
    const long long avg = (D->T * D->K + D->E - 1) / D->E;
    const long long C = std::min<long long>((avg + D->m_tile - 1) / D->m_tile * D->m_tile, D->T);
    return std::min((long long)D->E * ((C + GEMM_M - 1) / GEMM_M) * GEMM_M, b);
  }
  // token rounding moves an expert's count by less than one rounding tile; TC pads to 128-row tiles
  const long long a = pairs + (long long)D->E * (std::max(D->m_tile, GEMM_M) - 1);
  const long long r = std::min(a, b);
  return (r + GEMM_M - 1) / GEMM_M * GEMM_M;
}
Shape shape_of(const sonic_moe_desc* D) {
  Shape s;
  s.T = D->T;
  s.d = D->d;
  s.n = D->n;
  s.E = D->E;
  s.K = D->K;
  s.W = (int)((D->T + 31) / 32);
  s.rows_max = rows_max_of(D);
  return s;
}
size_t al(size_t x) { return (x + 255) & ~size_t(255); }
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// route workspace layout
struct RouteWs {
  size_t bm_tc, bm_kept, wprefix, tokcnt, flip, ticket, ST, nrs, total;
};
RouteWs route_ws(const sonic_moe_desc* D) {
  const Shape s = shape_of(D);
  RouteWs w;
  size_t o = 0;
  const size_t bm = al((size_t)s.E * s.W * 4);
  w.bm_tc = o; o += bm;
  w.bm_kept = o; o += bm;
  w.wprefix = o; o += bm;
  w.tokcnt = o; o += al((size_t)std::max<long long>(s.T, s.E) * 4);  // token counts (TR CSR) / expert counts (TC)
  w.flip = o; o += al((size_t)s.E * 4);
  w.ticket = o; o += al(8);  // [0] offsets ticket, [1] token-CSR ticket
  const bool needs_st = D->route_mode != SONIC_ROUTE_TC && D->route_mode != SONIC_ROUTE_GIVEN;
  w.ST = o; o += needs_st ? al((size_t)s.T * s.E * 4) : 0;
  // NR-s: two candidate bitmaps, two count arrays, three score-sum arrays
  w.nrs = o; o += (D->route_mode == SONIC_ROUTE_TR_NRS) ? 2 * bm + 2 * al((size_t)s.E * 4) + al((size_t)s.E * 24) : 0;
  w.total = o;
  return w;
}

#ifndef SONIC_DH_MAX_BN
#define SONIC_DH_MAX_BN 256  // BN = 256 streams H through a chunk ring (gemm.cuh HRING)
#endif
int dh_bn(int n) {
  return (n % 256 == 0 && SONIC_DH_MAX_BN >= 256) ? 256 : n % 128 == 0 ? 128 : n % 64 == 0 ? 64 : 32;
}

#ifndef SONIC_FUSED_UPDOWN
#define SONIC_FUSED_UPDOWN 0  // NEXT-1 fused up/down (updown.cuh): opt-in per call (SONIC_F_FUSED_UPDOWN);
                              // measured slower than the two kernels at 7B
#endif
// The fused up/down kernel holds a CTA's 128 rows of A (128 x n bf16) in shared memory: n = 128 or
// 256 (with 3+ operand stages); d a multiple of 128 (D jobs of 256 or 128 columns).
bool fused_updown(const sonic_moe_desc* D) {
  return (SONIC_FUSED_UPDOWN || (D->flags & SONIC_F_FUSED_UPDOWN)) && !(D->flags & SONIC_F_NO_FUSED_UPDOWN) &&
         use_cta2(256) && (D->n == 128 || D->n == 256) &&
         D->d % 128 == 0;
}

// SONIC_F_FP8_UP (NEXT-4): the up-projection on e4m3 operands; needs the 2-CTA 256-column UP tile
// (n % 128 == 0) and whole 128-element k-blocks (d % 128 == 0); not with the fused up/down kernel
bool fp8_up(const sonic_moe_desc* D) { return (D->flags & SONIC_F_FP8_UP) != 0; }
bool fp8_up_ok(const sonic_moe_desc* D) { return use_cta2(256) && D->n % 128 == 0 && D->d % 128 == 0; }
struct FwdWs { size_t A, Y, Xq, sx, W1q, sw, total; bool fused; };
FwdWs fwd_ws(const sonic_moe_desc* D) {
  const Shape s = shape_of(D);
  FwdWs w;
  size_t o = 0;
  w.fused = fused_updown(D) && !fp8_up(D);
  w.A = w.fused ? SIZE_MAX : o;  // fused: A never leaves the SM
  if (!w.fused) o += al((size_t)s.rows_max * s.n * 2);
  w.Y = o; o += al((size_t)s.rows_max * s.d * 2);
  w.Xq = w.sx = w.W1q = w.sw = SIZE_MAX;
  if (fp8_up(D)) {  // e4m3 copies of X and W1 and their scales
    w.Xq = o; o += al((size_t)s.T * s.d);
    w.sx = o; o += al((size_t)s.T * 4);
    w.W1q = o; o += al((size_t)s.E * s.d * 2 * s.n);
    w.sw = o; o += al((size_t)s.E * 2 * s.n * 4);
  }
  w.total = o;
  return w;
}
// SONIC_F_FP8_DXT (NEXT-4): dX~ on e4m3 operands; 2-CTA 256-column DXT tiles (d % 256 == 0) and
// whole 128-element k-blocks of 2n (n % 64 == 0)
bool fp8_dxt(const sonic_moe_desc* D) { return (D->flags & SONIC_F_FP8_DXT) != 0; }
bool fp8_dxt_ok(const sonic_moe_desc* D) { return use_cta2(256) && D->n % 64 == 0 && D->d % 256 == 0; }
struct BwdWs { size_t dH, Ap, dXt, dSp, dHq, sdh, W1q, sw, total; int dh_tiles; };
BwdWs bwd_ws(const sonic_moe_desc* D) {
  const Shape s = shape_of(D);
  BwdWs w;
  size_t o = 0;
  w.dH = o; o += al((size_t)s.rows_max * 2 * s.n * 2);
  w.Ap = o; o += al((size_t)s.rows_max * s.n * 2);
  w.dXt = o; o += al((size_t)s.rows_max * s.d * 2);
  w.dh_tiles = s.n / dh_bn(s.n);
  w.dSp = o; o += w.dh_tiles > 1 ? al((size_t)w.dh_tiles * s.rows_max * 4) : 0;
  w.dHq = w.sdh = w.W1q = w.sw = SIZE_MAX;
  if (fp8_dxt(D)) {  // e4m3 dH' and W1 copies and their scales
    w.dHq = o; o += al((size_t)s.rows_max * 2 * s.n);
    w.sdh = o; o += al((size_t)s.rows_max * 4);
    w.W1q = o; o += al((size_t)s.E * s.d * 2 * s.n);
    w.sw = o; o += al((size_t)s.E * 2 * s.n * 4);
  }
  w.total = o;
  return w;
}

sonic_status check_launch() {
  return cudaGetLastError() == cudaSuccess ? SONIC_OK : SONIC_ERR_CUDA;
}

}  // namespace

extern "C" {

int64_t sonic_rows_max(const sonic_moe_desc* desc) {
  if (!valid_desc(desc)) return -1;
  return rows_max_of(desc);
}

sonic_status sonic_routing_sizes(const sonic_moe_desc* D, size_t b[SONIC_ROUTING_NFIELDS]) {
  if (!valid_desc(D) || !b) return SONIC_ERR_INVALID_ARG;
  const Shape s = shape_of(D);
  const size_t TK = (size_t)s.T * s.K;
  b[0] = TK * 4;                              // topk_ids
  b[1] = TK * 4;                              // topk_s
  b[2] = (size_t)s.E * 4;                     // f
  b[3] = (size_t)s.E * 4;                     // f_rounded
  b[4] = (size_t)(s.E + 1) * 4;               // offsets
  b[5] = (size_t)(s.E + 1) * 4;               // pad_offsets
  b[6] = (size_t)s.rows_max * 4;              // row_token
  b[7] = (size_t)s.rows_max * 4;              // row_gate
  b[8] = (size_t)(s.T + 1) * 4;               // token_rowptr
  b[9] = (size_t)s.rows_max * 4;              // token_rows
  b[10] = (size_t)(s.rows_max / GEMM_M) * 4;  // tile_expert
  b[11] = 4;                                  // num_tiles
  b[12] = (size_t)(s.rows_max / GEMM_M + 1) * 4;  // tile_pairs
  b[13] = 4;                                  // num_pairs
  return SONIC_OK;
}

size_t sonic_route_workspace_size(const sonic_moe_desc* D) { return valid_desc(D) ? route_ws(D).total : 0; }
size_t sonic_fwd_workspace_size(const sonic_moe_desc* D) { return valid_desc(D) ? fwd_ws(D).total : 0; }
size_t sonic_bwd_workspace_size(const sonic_moe_desc* D) { return valid_desc(D) ? bwd_ws(D).total : 0; }

sonic_status sonic_workspace_offsets(const sonic_moe_desc* D, int which, size_t offs[4]) {
  if (!valid_desc(D) || !offs) return SONIC_ERR_INVALID_ARG;
  if (which == 0) {
    const FwdWs w = fwd_ws(D);
    offs[0] = w.A; offs[1] = w.Y; offs[2] = offs[3] = 0;
  } else if (which == 1) {
    const BwdWs w = bwd_ws(D);
    offs[0] = w.dH; offs[1] = w.Ap; offs[2] = w.dXt; offs[3] = w.dSp;
  } else if (which == 2) {
    const BwdWs w = bwd_ws(D);
    offs[0] = w.dHq; offs[1] = w.sdh; offs[2] = w.W1q; offs[3] = w.sw;
  } else {
    return SONIC_ERR_INVALID_ARG;
  }
  return SONIC_OK;
}

const char* sonic_status_string(sonic_status s) {
  switch (s) {
    case SONIC_OK: return "ok";
    case SONIC_ERR_INVALID_ARG: return "invalid argument";
    case SONIC_ERR_UNSUPPORTED: return "unsupported shape";
    case SONIC_ERR_WORKSPACE: return "workspace too small";
    case SONIC_ERR_CUDA: return "CUDA launch failure";
    case SONIC_ERR_NCCL: return "NCCL failure";
  }
  return "unknown status";
}

sonic_status sonic_router_bwd(const sonic_moe_desc* D, const float* S, const sonic_routing* rt, const float* dS,
                              float* dlogits, void* stream) {
  g_launches = 0;
  if (!valid_desc(D) || D->route_mode == SONIC_ROUTE_GIVEN || !S || !rt || !dS || !dlogits) return SONIC_ERR_INVALID_ARG;
  if (!rt->token_rowptr || !rt->token_rows || !rt->tile_expert) return SONIC_ERR_INVALID_ARG;
  {
    ProfScope ps("router_bwd", static_cast<cudaStream_t>(stream));
    launch_router_bwd(S, rt->token_rowptr, rt->token_rows, rt->tile_expert, dS, D->T, D->E,
                      (D->flags & SONIC_F_GATE_RAW) ? 1 : 0, dlogits, static_cast<cudaStream_t>(stream));
    ++g_launches;
  }
  return check_launch();
}

int sonic_last_launch_count(void) { return g_launches; }

void sonic_profile_enable(int on) { g_prof = on != 0; }

int sonic_profile_collect(char* names, int name_len, float* ms, int max_records) {
  int n = 0;
  for (auto& r : g_recs) {
    if (n < max_records) {
      float t = 0.f;
      cudaEventSynchronize(r.b);
      cudaEventElapsedTime(&t, r.a, r.b);
      strncpy(names + (size_t)n * name_len, r.name, name_len - 1);
      names[(size_t)n * name_len + name_len - 1] = 0;
      ms[n] = t;
      ++n;
    }
    g_pool.push_back(r.a);
    g_pool.push_back(r.b);
  }
  g_recs.clear();
  return n;
}

static sonic_status route_impl(const sonic_moe_desc* D, const float* S, const float* logits, sonic_routing* rt,
                               void* ws, size_t ws_bytes, void* stream, int* overflow = nullptr) {
  g_launches = 0;
  if (!valid_desc(D) || !S || !rt) return SONIC_ERR_INVALID_ARG;
  if (logits && (D->route_mode == SONIC_ROUTE_GIVEN || !aligned16(logits))) return SONIC_ERR_INVALID_ARG;
  if (!supported_dims(D)) return SONIC_ERR_UNSUPPORTED;
  const RouteWs w = route_ws(D);
  if (!ws || ws_bytes < w.total) return SONIC_ERR_WORKSPACE;
  void* ptrs[] = {rt->topk_ids, rt->topk_s, rt->f, rt->f_rounded, rt->offsets, rt->pad_offsets, rt->row_token,
                  rt->row_gate, rt->token_rowptr, rt->token_rows, rt->tile_expert, rt->num_tiles,
                  rt->tile_pairs, rt->num_pairs};
  for (void* p : ptrs)
    if (!p) return SONIC_ERR_INVALID_ARG;
  if (!aligned16(S) || !aligned16(rt->row_token)) return SONIC_ERR_INVALID_ARG;
  const Shape s = shape_of(D);
  uint8_t* base = static_cast<uint8_t*>(ws);
  RouteLaunch L{};
  L.T = s.T; L.E = s.E; L.K = s.K; L.W = s.W; L.m_tile = D->m_tile;
  // launcher modes: 0 TC, 1 TR (rounding subroutine in L.rounding), 2 given, 3 expert choice
  switch (D->route_mode) {
    case SONIC_ROUTE_TC: L.mode = 0; break;
    case SONIC_ROUTE_GIVEN: L.mode = 2; break;
    case SONIC_ROUTE_EC: L.mode = 3; break;
    case SONIC_ROUTE_TR_NRS: L.mode = 1; L.rounding = 5; break;
    default:
      L.mode = 1;
      L.rounding = D->route_mode == SONIC_ROUTE_TR_NRF ? 0 : D->route_mode - SONIC_ROUTE_TR_UP + 1;
      break;
  }
  L.seed = D->seed;
  L.rescue = (D->flags & SONIC_F_NO_ORPHAN_RESCUE) ? 0 : 1;
  L.gate_raw = (D->flags & SONIC_F_GATE_RAW) ? 1 : 0;
  L.S = S;
  L.logits = logits;
  L.overflow = overflow;
  L.cap = (D->rows_cap > 0 && D->rows_cap < D->T * D->K) ? D->rows_cap : D->T * D->K;
  L.topk_ids = rt->topk_ids; L.topk_s = rt->topk_s; L.f = rt->f; L.f_r = rt->f_rounded;
  L.offsets = rt->offsets; L.pad_offsets = rt->pad_offsets; L.row_token = rt->row_token;
  L.row_gate = rt->row_gate; L.token_rowptr = rt->token_rowptr; L.token_rows = rt->token_rows;
  L.tile_expert = rt->tile_expert; L.num_tiles = rt->num_tiles;
  L.tile_pairs = rt->tile_pairs; L.num_pairs = rt->num_pairs;
  L.bm_tc = reinterpret_cast<uint32_t*>(base + w.bm_tc);
  L.bm_kept = reinterpret_cast<uint32_t*>(base + w.bm_kept);
  L.wprefix = reinterpret_cast<int*>(base + w.wprefix);
  L.tokcnt = reinterpret_cast<int*>(base + w.tokcnt);
  L.flip = reinterpret_cast<int*>(base + w.flip);
  L.ticket = reinterpret_cast<unsigned*>(base + w.ticket);
  if (D->route_mode == SONIC_ROUTE_TR_NRS) {
    const size_t bmb = al((size_t)s.E * s.W * 4);
    uint8_t* q = base + w.nrs;
    L.bm_dn = reinterpret_cast<uint32_t*>(q); q += bmb;
    L.bm_up = reinterpret_cast<uint32_t*>(q); q += bmb;
    L.f_dn = reinterpret_cast<int*>(q); q += al((size_t)s.E * 4);
    L.f_up = reinterpret_cast<int*>(q); q += al((size_t)s.E * 4);
    L.nrs_sums = reinterpret_cast<double*>(q);
  }
  L.ST = reinterpret_cast<float*>(base + w.ST);
  {
    ProfScope ps("route", static_cast<cudaStream_t>(stream));
    g_launches = launch_route(L, static_cast<cudaStream_t>(stream));
  }
  return check_launch();
}

sonic_status sonic_route(const sonic_moe_desc* D, const float* S, sonic_routing* rt, void* ws, size_t ws_bytes,
                         void* stream) {
  return route_impl(D, S, nullptr, rt, ws, ws_bytes, stream);
}

sonic_status sonic_route_given_capped(const sonic_moe_desc* D, const float* S, sonic_routing* rt, void* ws,
                                      size_t ws_bytes, int* overflow, void* stream) {
  if (!D || D->route_mode != SONIC_ROUTE_GIVEN || !overflow) return SONIC_ERR_INVALID_ARG;
  return route_impl(D, S, nullptr, rt, ws, ws_bytes, stream, overflow);
}

sonic_status sonic_route_logits(const sonic_moe_desc* D, const float* logits, float* S_out, sonic_routing* rt,
                                void* ws, size_t ws_bytes, void* stream) {
  if (!logits) return SONIC_ERR_INVALID_ARG;
  return route_impl(D, S_out, logits, rt, ws, ws_bytes, stream);
}

sonic_status sonic_moe_fwd(const sonic_moe_desc* D, const void* X, const void* W1, const void* W2,
                           const sonic_routing* rt, void* O, void* H, void* ws, size_t ws_bytes, void* stream) {
  g_launches = 0;
  if (!valid_desc(D) || !X || !W1 || !W2 || !rt || !O || !H) return SONIC_ERR_INVALID_ARG;
  if (!supported_dims(D)) return SONIC_ERR_UNSUPPORTED;
  if (fp8_up(D) && !fp8_up_ok(D)) return SONIC_ERR_UNSUPPORTED;
  const FwdWs w = fwd_ws(D);
  if (!ws || ws_bytes < w.total) return SONIC_ERR_WORKSPACE;
  for (const void* p : {X, W1, W2, (const void*)O, (const void*)H, (const void*)ws})
    if (!aligned16(p)) return SONIC_ERR_INVALID_ARG;
  const Shape s = shape_of(D);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* base = static_cast<uint8_t*>(ws);
  void* Abuf = base + w.A;
  void* Ybuf = base + w.Y;
  const int n = s.n, d = s.d, E = s.E;
  const long long R = s.rows_max;
  const int grid = num_sms();

  GemmArgs g{};
  g.num_m_tiles = rt->num_tiles; g.tile_expert = rt->tile_expert; g.row_token = rt->row_token;
  g.num_pairs = rt->num_pairs; g.tile_pairs = rt->tile_pairs;
  g.row_gate = rt->row_gate; g.pad_offsets = rt->pad_offsets; g.E = E; g.n = n; g.rows_max = R;

  if (w.fused) {
    // K1 + K2 fused: H = Gather(X) W1_e -> H (cached), A = SwiGLU(H) in smem, Y = g * (A W2_e)
    CUtensorMap mW1, mW2, mH, mY;
    if (!map3d(&mW1, W1, false, E, d, 2 * n, 64, 64) || !map3d(&mW2, W2, false, E, n, d, 64, 64) ||
        !map2d(&mH, H, false, R, 2 * n, 64, 32) || !map2d(&mY, Ybuf, false, R, d, 64, 32))
      return SONIC_ERR_CUDA;
    UpDownArgs a{};
    a.num_pairs = rt->num_pairs; a.tile_pairs = rt->tile_pairs; a.tile_expert = rt->tile_expert;
    a.row_token = rt->row_token; a.row_gate = rt->row_gate;
    a.X = static_cast<const __nv_bfloat16*>(X); a.d = d; a.n = n;
    ProfScope ps("updown", st);
    const bool ok = n == 256 ? (d % 256 == 0 ? launch_updown<2, 256>(mW1, mW2, mH, mY, a, grid, st)
                                             : launch_updown<2, 128>(mW1, mW2, mH, mY, a, grid, st))
                             : (d % 256 == 0 ? launch_updown<1, 256>(mW1, mW2, mH, mY, a, grid, st)
                                             : launch_updown<1, 128>(mW1, mW2, mH, mY, a, grid, st));
    if (!ok) return SONIC_ERR_CUDA;
  }
  // K1 up-proj on e4m3 operands (SONIC_F_FP8_UP): quantise X per token and W1 per output column,
  // then H = (Gather(Xq) W1q_e) * sx * sw in the epilogue (NEXT-4)
  if (fp8_up(D)) {
    uint8_t* Xq = base + w.Xq;
    float* sx = reinterpret_cast<float*>(base + w.sx);
    uint8_t* W1q = base + w.W1q;
    float* sw = reinterpret_cast<float*>(base + w.sw);
    {
      ProfScope ps("quant_fp8", st);
      launch_quant_rows_e4m3(X, s.T, d, Xq, sx, st);
      ++g_launches;
      if (!(D->flags & SONIC_F_FP8_W1_CACHED)) {
        launch_quant_cols_e4m3(W1, E, d, 2 * n, W1q, sw, st);
        g_launches += 3;  // columns: amax, quantise, amax -> scale
      }
    }
    CUtensorMap mA, mB, mC0, mC1;
    if (!map2d(&mA, X, false, s.T, d, 64, 1) || !map3d_u8(&mB, W1q, E, d, 2 * n, 128, 128) ||
        !map2d(&mC0, H, false, R, 2 * n, 64, 32) || !map2d(&mC1, Abuf, false, R, n, 64, 32))
      return SONIC_ERR_CUDA;
    GemmArgs a = g;
    a.n_tiles = n / 128; a.k_blocks = d / 128; a.N_dim = 2 * n;
    a.gsrc = reinterpret_cast<const __nv_bfloat16*>(Xq); a.gld = d;  // e4m3 rows (gathered by byte address)
    a.sx = sx; a.sw = sw;
    ProfScope ps("up", st);
    if (!launch_gemm<K_UP8>(256, mA, mB, mC0, mC1, a, grid, st)) return SONIC_ERR_CUDA;
  }
  // K1 up-proj: H = Gather(X) W1_e, SwiGLU epilogue -> H, A
  if (!w.fused && !fp8_up(D)) {
    CUtensorMap mA, mB, mC0, mC1;
    const int Wg = n % 128 == 0 ? 128 : n % 64 == 0 ? 64 : 32;
    const int BN = 2 * Wg;
    if (!map2d(&mA, X, false, s.T, d, 64, 1) || !map3d(&mB, W1, false, E, d, 2 * n, 64, 64) ||
        !map2d(&mC0, H, false, R, 2 * n, 64, 32) || !map2d(&mC1, Abuf, false, R, n, 64, 32))
      return SONIC_ERR_CUDA;
    GemmArgs a = g;
    a.n_tiles = n / Wg; a.k_blocks = d / 64; a.N_dim = 2 * n;
    a.gsrc = static_cast<const __nv_bfloat16*>(X); a.gld = d;
    ProfScope ps("up", st);
    if (!launch_gemm<K_UP>(BN, mA, mB, mC0, mC1, a, grid, st)) return SONIC_ERR_CUDA;
  }
  // K2 down-proj: Y = gate * (A W2_e)
  if (!w.fused) {
    CUtensorMap mA, mB, mC0, mA64;
    const int BN = pick_bn(d);
    if (!map2d(&mA, Abuf, false, R, n, 64, 128) || !map3d(&mB, W2, false, E, n, d, 64, 64) ||
        !map2d(&mC0, Ybuf, false, R, d, 64, 32) || !map2d(&mA64, Abuf, false, R, n, 64, 64))
      return SONIC_ERR_CUDA;
    GemmArgs a = g;
    a.n_tiles = d / BN; a.k_blocks = (n + 63) / 64; a.N_dim = d;
    if (wide_g<K_DOWN>() > 1 && d % 64 == 0 && (BN / 64) % wide_g<K_DOWN>() == 0) {  // as the kernel's WIDE
      if (!map_wide(&mC0, Ybuf, R, d, wide_g<K_DOWN>())) return SONIC_ERR_CUDA;
      a.wide = 1;
    }
    ProfScope ps("down", st);
    // multicast cluster: the pair tiles (m, 2j) and (m, 2j+1) share the A rows
    if (!launch_gemm<K_DOWN>(BN, mA, mB, mC0, mC0, a, grid, st, &mA64, a.n_tiles % 2 == 0)) return SONIC_ERR_CUDA;
  }
  // K3 aggregation: O_t = sum of the token's Y rows
  ProfScope ps("agg_O", st);
  launch_aggregate(static_cast<const __nv_bfloat16*>(Ybuf), rt->token_rowptr, rt->token_rows,
                   static_cast<__nv_bfloat16*>(O), s.T, d, st);
  ++g_launches;
  return check_launch();
}

sonic_status sonic_moe_bwd(const sonic_moe_desc* D, const void* dO, const void* X, const void* H, const void* W1,
                           const void* W2, const sonic_routing* rt, void* dX, float* dW1, float* dW2, float* dS,
                           void* ws, size_t ws_bytes, void* stream) {
  g_launches = 0;
  if (!valid_desc(D)) return SONIC_ERR_INVALID_ARG;
  const bool no_dw = D->flags & SONIC_F_BWD_NO_DW, dw_only = D->flags & SONIC_F_BWD_DW_ONLY;
  if (no_dw && dw_only) return SONIC_ERR_INVALID_ARG;
  if ((D->flags & SONIC_F_DW_BF16) && (D->flags & SONIC_F_DW_ACCUMULATE)) return SONIC_ERR_INVALID_ARG;
  if (!dO || !X || !H || !W1 || !W2 || !rt || (!dw_only && (!dX || !dS)) || (!no_dw && (!dW1 || !dW2)))
    return SONIC_ERR_INVALID_ARG;
  if (!supported_dims(D)) return SONIC_ERR_UNSUPPORTED;
  if (fp8_dxt(D) && (!fp8_dxt_ok(D) || dw_only)) return fp8_dxt_ok(D) ? SONIC_ERR_INVALID_ARG : SONIC_ERR_UNSUPPORTED;
  const BwdWs w = bwd_ws(D);
  if (!ws || ws_bytes < w.total) return SONIC_ERR_WORKSPACE;
  for (const void* p : {dO, X, H, W1, W2, (const void*)dX, (const void*)dW1, (const void*)dW2, (const void*)dS,
                        (const void*)ws})
    if (p && !aligned16(p)) return SONIC_ERR_INVALID_ARG;
  const Shape s = shape_of(D);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* base = static_cast<uint8_t*>(ws);
  void* dH = base + w.dH;
  void* Ap = base + w.Ap;
  void* dXt = base + w.dXt;
  float* dSp = reinterpret_cast<float*>(base + w.dSp);
  const int n = s.n, d = s.d, E = s.E;
  const long long R = s.rows_max;
  const int grid = num_sms();

  GemmArgs g{};
  g.num_m_tiles = rt->num_tiles; g.tile_expert = rt->tile_expert; g.row_token = rt->row_token;
  g.num_pairs = rt->num_pairs; g.tile_pairs = rt->tile_pairs;
  g.row_gate = rt->row_gate; g.pad_offsets = rt->pad_offsets; g.E = E; g.n = n; g.rows_max = R;

  // K4 dH: dA' = Gather(dO) W2_e^T; epilogue dSwiGLU -> dH, A' = s A, dS = <dA', A>
  if (!dw_only) {
    CUtensorMap mA, mB, mC0, mC1, mH;
    const int BN = dh_bn(n);
    if (!map2d(&mA, dO, false, s.T, d, 64, 1) || !map3d(&mB, W2, false, E, n, d, 64, bnl(BN)) ||
        !map2d(&mC0, dH, false, R, 2 * n, 64, 32) || !map2d(&mC1, Ap, false, R, n, 64, 32) ||
        !map2d(&mH, H, false, R, 2 * n, 64, 32))
      return SONIC_ERR_CUDA;
    GemmArgs a = g;
    a.n_tiles = n / BN; a.k_blocks = d / 64; a.N_dim = n;
    a.gsrc = static_cast<const __nv_bfloat16*>(dO); a.gld = d;
    a.dS = a.n_tiles > 1 ? dSp : dS;
    {
      ProfScope ps("dH", st);
      if (!launch_gemm<K_DH>(BN, mA, mB, mC0, mC1, a, grid, st, &mH)) return SONIC_ERR_CUDA;
    }
    if (a.n_tiles > 1) {
      ProfScope ps("dS_reduce", st);
      launch_ds_reduce(dSp, a.n_tiles, R, rt->num_tiles, dS, st);
      ++g_launches;
    }
  }
  // Stream arrangement of the rest of the backward (SONIC_BWD_OVERLAP):
  //   0  everything on the caller's stream;
  //   1  the dX aggregation on an internal side stream forked after dX~, co-residing with the
  //      dW2/dW1 CTAs on the caller's stream;
  //   2  dW2/dW1 on the side stream forked after dH; dX~ then the aggregation on the caller's;
  //   3  the dX aggregation on the side stream overlapping dW2 only, joined before dW1.
  // The side stream is joined before returning.
  const int mode = SONIC_BWD_OVERLAP;
  SideStream& ss = side_stream();
  if (mode != 0 && !ss.ok) return SONIC_ERR_CUDA;
  const cudaStream_t s_dw = mode == 2 ? ss.s : st;
  const cudaStream_t s_agg = (mode == 1 || mode == 3) ? ss.s : st;
  if (mode == 2) {
    cudaEventRecord(ss.fork, st);
    cudaStreamWaitEvent(ss.s, ss.fork, 0);
  }
  CUtensorMap mA6, mB6, mC6, mA5, mB5, mC5, mA7, mB7, mC7, mA6h;
  GemmArgs a6 = g, a5 = g, a7 = g;
  const int BN6 = pick_bn(d), BN5 = pick_bn(d), BN7 = pick_bn(2 * n);
  // K6 dX~_e = dH_e W1_e^T
  if (!map2d(&mA6, dH, false, R, 2 * n, 64, 128) || !map3d(&mB6, W1, false, E, d, 2 * n, 64, bnl(BN6)) ||
      !map2d(&mC6, dXt, false, R, d, 64, 32) || !map2d(&mA6h, dH, false, R, 2 * n, 64, 64))
    return SONIC_ERR_CUDA;
  a6.n_tiles = d / BN6; a6.k_blocks = (2 * n) / 64; a6.N_dim = d;
  if (wide_g<K_DXT>() > 1 && d % 64 == 0 && (BN6 / 64) % wide_g<K_DXT>() == 0) {
    if (!map_wide(&mC6, dXt, R, d, wide_g<K_DXT>())) return SONIC_ERR_CUDA;
    a6.wide = 1;
  }
  // K5 dW2_e = A'_e^T Gather(dO)   (varlen-K)
  const bool dw_bf16 = (D->flags & SONIC_F_DW_BF16) != 0;
  if (!map2d(&mA5, Ap, false, R, n, 64, 64) || !map2d(&mB5, dO, false, s.T, d, 64, 1) ||
      !map3d(&mC5, dW2, !dw_bf16, E, n, d, dw_bf16 ? 64 : 32, 32))
    return SONIC_ERR_CUDA;
  a5.n_tiles = d / BN5; a5.m_tiles = (n + 127) / 128; a5.M_dim = n; a5.N_dim = d;
  a5.gsrc = static_cast<const __nv_bfloat16*>(dO); a5.gld = d;
  a5.accumulate = (D->flags & SONIC_F_DW_ACCUMULATE) ? 1 : 0;
  a5.dw_bf16 = dw_bf16 ? 1 : 0;
  const int tiles5 = E * a5.m_tiles * a5.n_tiles;
  // K7 dW1_e = Gather(X)^T dH_e   (varlen-K)
  if (!map2d(&mA7, X, false, s.T, d, 64, 1) || !map2d(&mB7, dH, false, R, 2 * n, 64, 64) ||
      !map3d(&mC7, dW1, !dw_bf16, E, d, 2 * n, dw_bf16 ? 64 : 32, 32))
    return SONIC_ERR_CUDA;
  a7.n_tiles = (2 * n) / BN7; a7.m_tiles = (d + 127) / 128; a7.M_dim = d; a7.N_dim = 2 * n;
  a7.gsrc = static_cast<const __nv_bfloat16*>(X); a7.gld = d;
  a7.accumulate = (D->flags & SONIC_F_DW_ACCUMULATE) ? 1 : 0;
  a7.dw_bf16 = dw_bf16 ? 1 : 0;
  const int tiles7 = E * a7.m_tiles * a7.n_tiles;

  auto run_dxt = [&]() {
    if (fp8_dxt(D)) {
      // e4m3 dX~ (Q25): W1 per output column (the forward's quantisation), dH' = dH * sw per row
      uint8_t* dHq = base + w.dHq;
      float* sdh = reinterpret_cast<float*>(base + w.sdh);
      uint8_t* W1q = base + w.W1q;
      float* sw = reinterpret_cast<float*>(base + w.sw);
      {
        ProfScope ps("quant_dh", st);
        if (!(D->flags & SONIC_F_FP8_W1_CACHED)) {
          launch_quant_cols_e4m3(W1, E, d, 2 * n, W1q, sw, st);
          g_launches += 3;
        }
        launch_quant_dh_e4m3(dH, R, 2 * n, rt->num_tiles, rt->tile_expert, sw, dHq, sdh, st);
        ++g_launches;
      }
      CUtensorMap mA8, mB8, mC8;
      if (!map2d_u8(&mA8, dHq, R, 2 * n, 128, 128) || !map3d_u8(&mB8, W1q, E, d, 2 * n, 128, bnl(BN6)) ||
          !map2d(&mC8, dXt, false, R, d, 64, 32))
        return false;
      GemmArgs a8 = a6;
      a8.k_blocks = (2 * n) / 128; a8.sx = sdh; a8.wide = 0;
      ProfScope ps("dXt", st);
      return launch_gemm<K_DXT8>(256, mA8, mB8, mC8, mC8, a8, grid, st);
    }
    ProfScope ps("dXt", st);
    return launch_gemm<K_DXT>(BN6, mA6, mB6, mC6, mC6, a6, grid, st, &mA6h, a6.n_tiles % 2 == 0);
  };
  auto run_dw2 = [&]() {
    ProfScope ps("dW2", s_dw);
    return launch_gemm<K_DW2>(BN5, mA5, mB5, mC5, mC5, a5, std::min(grid, tiles5), s_dw, nullptr, a5.n_tiles % 2 == 0);
  };
  auto run_dw1 = [&]() {
    ProfScope ps("dW1", s_dw);
    return launch_gemm<K_DW1>(BN7, mA7, mB7, mC7, mC7, a7, std::min(grid, tiles7), s_dw, nullptr,
                              ((a7.m_tiles + 1) / 2) % 2 == 0);
  };
  auto run_agg = [&]() {  // K8 dX aggregation
    ProfScope ps("agg_dX", s_agg);
    launch_aggregate(static_cast<const __nv_bfloat16*>(dXt), rt->token_rowptr, rt->token_rows,
                     static_cast<__nv_bfloat16*>(dX), s.T, d, s_agg);
    ++g_launches;
  };
  if (no_dw) {  // split backward, part 1: dX (and dS); dH / A' stay in ws for part 2
    if (!run_dxt()) return SONIC_ERR_CUDA;
    launch_aggregate(static_cast<const __nv_bfloat16*>(dXt), rt->token_rowptr, rt->token_rows,
                     static_cast<__nv_bfloat16*>(dX), s.T, d, st);
    ++g_launches;
    return check_launch();
  }
  if (dw_only) {  // split backward, part 2: dW2, dW1 from the dH / A' of part 1 (same ws)
    if (!run_dw2() || !run_dw1()) return SONIC_ERR_CUDA;
    return check_launch();
  }
  if (!run_dxt()) return SONIC_ERR_CUDA;
  if (mode == 1) {
    cudaEventRecord(ss.fork, st);
    cudaStreamWaitEvent(ss.s, ss.fork, 0);
    run_agg();
    cudaEventRecord(ss.join, ss.s);
    if (!run_dw2() || !run_dw1()) return SONIC_ERR_CUDA;
  } else if (mode == 2) {
    if (!run_dw2()) return SONIC_ERR_CUDA;
    run_agg();
    if (!run_dw1()) return SONIC_ERR_CUDA;
    cudaEventRecord(ss.join, ss.s);
  } else if (mode == 3) {  // the aggregation overlaps dW2 only; dW1 runs alone
    cudaEventRecord(ss.fork, st);
    cudaStreamWaitEvent(ss.s, ss.fork, 0);
    run_agg();
    cudaEventRecord(ss.join, ss.s);
    if (!run_dw2()) return SONIC_ERR_CUDA;
    cudaStreamWaitEvent(st, ss.join, 0);
    if (!run_dw1()) return SONIC_ERR_CUDA;
  } else if (SONIC_AGG_FUSE) {
    // the dX aggregation runs inside the weight-gradient kernels (aggregator warp, gemm.cuh): the
    // first SONIC_AGG_DW2_PCT % of the tokens in dW2, the rest in dW1
    const long long t_split = s.T * SONIC_AGG_DW2_PCT / 100;
    for (GemmArgs* a : {&a5, &a7}) {
      a->agg_src = static_cast<const __nv_bfloat16*>(dXt);
      a->agg_dst = static_cast<__nv_bfloat16*>(dX);
      a->agg_rowptr = rt->token_rowptr;
      a->agg_rows = rt->token_rows;
      a->agg_d = d;
    }
    a5.agg_t0 = 0; a5.agg_t1 = t_split;
    a7.agg_t0 = t_split; a7.agg_t1 = s.T;
    if (!run_dw2() || !run_dw1()) return SONIC_ERR_CUDA;
  } else {
    if (!run_dw2() || !run_dw1()) return SONIC_ERR_CUDA;
    run_agg();
  }
  if (mode != 0) cudaStreamWaitEvent(st, ss.join, 0);
  return check_launch();
}

}  // extern "C"

namespace sonic {
void set_last_launch_count(int n) { g_launches = n; }
}  // namespace sonic
