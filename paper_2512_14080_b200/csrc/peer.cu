// peer.cu -- expert-parallel exchange through peer memory.
//
// Every rank of the EP group allocates one symmetric region and maps the regions of all the other
// ranks into its address space over CUDA IPC (on an NVSwitch box the mapped pointers are NVLink
// peer memory).  The dispatch kernel gathers the token rows named by the dispatch plan and stores
// them straight into the destination rank's region (pack and transfer in one kernel, no staging
// send buffer, no NCCL call); the return direction stores each received block back into its source
// rank's region.  A stream-ordered flag barrier (one release store per peer, acquire spins on the
// own flags) separates the phases, so there is no host synchronisation in the exchange itself.
#include <algorithm>
#include <cstring>
#include <unistd.h>

#include "../../include/sonic.h"
#include "sonic_internal.h"
#include "ptx.cuh"

struct sonic_peer {
  int rank = 0, world = 1, device = 0;
  size_t bytes = 0;
  void* region = nullptr;                   // own region (cudaMalloc)
  unsigned long long* flags = nullptr;      // own flags [world] (cudaMalloc, IPC-exported)
  void* base[SONIC_PEER_MAX] = {};          // region of rank r as mapped here
  unsigned long long* fbase[SONIC_PEER_MAX] = {};
  bool opened[SONIC_PEER_MAX] = {};
  unsigned long long** ftab = nullptr;      // device copy of fbase (the barrier kernel's table)
  unsigned long long epoch = 0;
};

namespace sonic {

struct PeerPtrs {
  char* base[SONIC_PEER_MAX];
};
struct PeerRows {
  int src_row0[SONIC_PEER_MAX];  // first source row of the block for rank g
  int cnt[SONIC_PEER_MAX];       // rows of the block
  int dst_row0[SONIC_PEER_MAX];  // first row in rank g's destination array
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Barrier: thread g publishes this rank's arrival in rank g's flags (release, system scope), then
// waits until rank g's arrival is visible in the own flags (acquire).  Every rank issues its
// barriers in the same order, so the epochs match.
__global__ void k_peer_barrier(unsigned long long* const* fpeer, unsigned long long* own, int rank, int world,
                               unsigned long long epoch) {
  const int g = threadIdx.x;
  if (g >= world) return;
  __threadfence_system();
  st_release_sys(fpeer[g] + rank, epoch);
  while (ld_acquire_sys(own + g) < epoch) __nanosleep(64);
  __threadfence_system();
}

// Dispatch: send row i (destination g = the block containing i) = src[send_token[i]] (d bf16),
// stored at row dst_row0[g] + (i - send_offsets[g]) of rank g's array at region byte offset
// `off`.  One warp per row, 16-byte stores; the final system fence makes the stores visible to the
// peers before the barrier that follows on the stream.
__global__ void k_pack_peer(const __nv_bfloat16* __restrict__ src, const int* __restrict__ send_token,
                            const int* __restrict__ send_offsets, int G, int d, PeerPtrs P, size_t off, PeerRows R) {
  const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i < __ldg(send_offsets + G)) {
    int g = 0;
    while (g + 1 < G && i >= __ldg(send_offsets + g + 1)) ++g;
    const long long drow = R.dst_row0[g] + (i - __ldg(send_offsets + g));
    const uint4* s = reinterpret_cast<const uint4*>(src + (size_t)__ldg(send_token + i) * d);
    uint4* o = reinterpret_cast<uint4*>(P.base[g] + off + (size_t)drow * d * 2);
    for (int c = lane; c < d / 8; c += 32) o[c] = s[c];
  }
  __threadfence_system();
}

// Block put: rows [src_row0[g], src_row0[g] + cnt[g]) of src (row_bytes each, a multiple of 16) to
// rows [dst_row0[g], ...) of rank g's array at region byte offset `off`.  blockIdx.y = g.
template <typename V>
__global__ void k_put_rows(const char* __restrict__ src, size_t row_bytes, PeerPtrs P, size_t off, PeerRows R) {
  const int g = blockIdx.y;
  const size_t nv = (size_t)R.cnt[g] * row_bytes / sizeof(V);
  const V* s = reinterpret_cast<const V*>(src + (size_t)R.src_row0[g] * row_bytes);
  V* o = reinterpret_cast<V*>(P.base[g] + off + (size_t)R.dst_row0[g] * row_bytes);
  for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < nv; j += (size_t)gridDim.x * blockDim.x)
    o[j] = s[j];
  __threadfence_system();
}

// ---------------------------------------------------------------- host-sync-free variants (NEXT-2)
// The block offsets come from the count matrix M in the rank's OWN region (every rank stored its
// row there in the count exchange): M[s][g] = rows s sends g = cnt[s * cols + g].
__device__ __forceinline__ int cm(const int* cnt, int cols, int s, int g) { return __ldcg(cnt + (size_t)s * cols + g); }

// Dispatch as k_pack_peer; destination row dst_row0[g] = sum_{s < me} M[s][g], computed here.
__global__ void k_pack_peer_dev(const __nv_bfloat16* __restrict__ src, const int* __restrict__ send_token,
                                const int* __restrict__ send_offsets, int G, int d, PeerPtrs P, size_t off,
                                const int* __restrict__ cnt, int cols, int me) {
  const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i < __ldg(send_offsets + G)) {
    int g = 0;
    while (g + 1 < G && i >= __ldg(send_offsets + g + 1)) ++g;
    long long dst0 = 0;
    for (int s = 0; s < me; ++s) dst0 += cm(cnt, cols, s, g);
    const long long drow = dst0 + (i - __ldg(send_offsets + g));
    const uint4* sp = reinterpret_cast<const uint4*>(src + (size_t)__ldg(send_token + i) * d);
    uint4* o = reinterpret_cast<uint4*>(P.base[g] + off + (size_t)drow * d * 2);
    for (int c = lane; c < d / 8; c += 32) o[c] = sp[c];
  }
  __threadfence_system();
}

// Block put with the blocks from M (blockIdx.y = g): dir 0 (dispatch, me -> g): rows
// [sum_{g'<g} M[me][g'], +M[me][g]) of src to rows [sum_{s<me} M[s][g], ...) of rank g; dir 1 (return,
// me is the destination, g the source): rows [sum_{s<g} M[s][me], +M[g][me]) to rows
// [sum_{g'<me} M[g][g'], ...) of rank g.
template <typename V>
__global__ void k_put_rows_dev(const char* __restrict__ src, size_t row_bytes, PeerPtrs P, size_t off,
                               const int* __restrict__ cnt, int cols, int me, int G, int dir) {
  const int g = blockIdx.y;
  long long src0 = 0, dst0 = 0;
  int n;
  if (dir == 0) {
    n = cm(cnt, cols, me, g);
    for (int j = 0; j < g; ++j) src0 += cm(cnt, cols, me, j);
    for (int s = 0; s < me; ++s) dst0 += cm(cnt, cols, s, g);
  } else {
    n = cm(cnt, cols, g, me);
    for (int s = 0; s < g; ++s) src0 += cm(cnt, cols, s, me);
    for (int j = 0; j < me; ++j) dst0 += cm(cnt, cols, g, j);
  }
  const size_t nv = (size_t)n * row_bytes / sizeof(V);
  const V* sp = reinterpret_cast<const V*>(src + (size_t)src0 * row_bytes);
  V* o = reinterpret_cast<V*>(P.base[g] + off + (size_t)dst0 * row_bytes);
  for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < nv; j += (size_t)gridDim.x * blockDim.x)
    o[j] = sp[j];
  __threadfence_system();
}

// Zero rows [R_in, cap_rows) of an own-region array, R_in = sum_s M[s][me] (the rows received this
// step): stale rows of an earlier step must not look routed to the capacity-sized receive side.
__global__ void k_zero_tail(char* __restrict__ base, size_t row_bytes, const int* __restrict__ cnt, int cols, int me,
                            int G, long long cap_rows) {
  long long r_in = 0;
  for (int s = 0; s < G; ++s) r_in += cm(cnt, cols, s, me);
  const size_t b0 = (size_t)r_in * row_bytes, b1 = (size_t)cap_rows * row_bytes;
  for (size_t j = b0 / 4 + (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < b1 / 4; j += (size_t)gridDim.x * blockDim.x)
    reinterpret_cast<uint32_t*>(base)[j] = 0u;
}

}  // namespace sonic

using namespace sonic;

namespace {
struct IpcBlob {  // what one rank exports: its region and its flags
  cudaIpcMemHandle_t region, flags;
  size_t bytes;
  int rank, world;
  long long pid;                 // creating process: peers in the same process use the raw pointers
  void* region_ptr;              // (CUDA IPC cannot open a handle in the process that exported it)
  unsigned long long* flags_ptr;
};
static_assert(sizeof(IpcBlob) <= SONIC_PEER_HANDLE_BYTES, "handle blob too large");

bool fill_rows(const sonic_peer* p, int G, const int32_t* a, const int32_t* b, const int32_t* c, PeerRows* R,
               PeerPtrs* P) {
  if (!p || G != p->world || G > SONIC_PEER_MAX) return false;
  for (int g = 0; g < G; ++g) {
    if (!p->base[g] || (b && b[g] < 0) || (a && a[g] < 0) || (c && c[g] < 0)) return false;
    R->src_row0[g] = a ? a[g] : 0;
    R->cnt[g] = b ? b[g] : 0;
    R->dst_row0[g] = c ? c[g] : 0;
    P->base[g] = static_cast<char*>(p->base[g]);
  }
  return true;
}

// CUDA lazy loading loads a kernel at its first launch and may wait for the device to go idle to
// do so; a first launch queued behind a spinning barrier whose partner has not been queued yet (virtual
// ranks of one process, queued rank by rank) would then deadlock.  Load every peer kernel up front.
bool preload_peer_kernels() {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, k_peer_barrier) == cudaSuccess && cudaFuncGetAttributes(&a, k_pack_peer) == cudaSuccess &&
         cudaFuncGetAttributes(&a, k_put_rows<uint4>) == cudaSuccess &&
         cudaFuncGetAttributes(&a, k_put_rows<uint32_t>) == cudaSuccess &&
         cudaFuncGetAttributes(&a, k_pack_peer_dev) == cudaSuccess &&
         cudaFuncGetAttributes(&a, k_put_rows_dev<uint4>) == cudaSuccess &&
         cudaFuncGetAttributes(&a, k_put_rows_dev<uint32_t>) == cudaSuccess &&
         cudaFuncGetAttributes(&a, k_zero_tail) == cudaSuccess;
}
}  // namespace

extern "C" {

sonic_status sonic_peer_create(int rank, int world, size_t bytes, sonic_peer** out, void* handle) {
  if (!out || !handle || world < 1 || world > SONIC_PEER_MAX || rank < 0 || rank >= world || bytes == 0)
    return SONIC_ERR_INVALID_ARG;
  *out = nullptr;
  if (!preload_peer_kernels()) return SONIC_ERR_CUDA;
  sonic_peer* p = new sonic_peer;
  p->rank = rank;
  p->world = world;
  p->bytes = bytes;
  cudaGetDevice(&p->device);
  if (cudaMalloc(&p->region, bytes) != cudaSuccess || cudaMalloc(&p->flags, SONIC_PEER_MAX * 8) != cudaSuccess ||
      cudaMemset(p->flags, 0, SONIC_PEER_MAX * 8) != cudaSuccess) {
    sonic_peer_destroy(p);
    return SONIC_ERR_CUDA;
  }
  IpcBlob b{};
  b.bytes = bytes;
  b.rank = rank;
  b.world = world;
  b.pid = (long long)getpid();
  b.region_ptr = p->region;
  b.flags_ptr = p->flags;
  if (cudaIpcGetMemHandle(&b.region, p->region) != cudaSuccess ||
      cudaIpcGetMemHandle(&b.flags, p->flags) != cudaSuccess) {
    sonic_peer_destroy(p);
    return SONIC_ERR_CUDA;
  }
  std::memset(handle, 0, SONIC_PEER_HANDLE_BYTES);
  std::memcpy(handle, &b, sizeof(b));
  p->base[rank] = p->region;
  p->fbase[rank] = p->flags;
  *out = p;
  return SONIC_OK;
}

sonic_status sonic_peer_open(sonic_peer* p, const void* handles) {
  if (!p || !handles) return SONIC_ERR_INVALID_ARG;
  const char* h = static_cast<const char*>(handles);
  for (int g = 0; g < p->world; ++g) {
    IpcBlob b;
    std::memcpy(&b, h + (size_t)g * SONIC_PEER_HANDLE_BYTES, sizeof(b));
    if (b.rank != g || b.world != p->world || b.bytes != p->bytes) return SONIC_ERR_INVALID_ARG;
    if (g == p->rank || p->opened[g] || p->base[g]) continue;
    if (b.pid == (long long)getpid()) {  // a virtual rank of this process (single-process EP)
      p->base[g] = b.region_ptr;
      p->fbase[g] = b.flags_ptr;
      continue;
    }
    void* r = nullptr;
    void* f = nullptr;
    if (cudaIpcOpenMemHandle(&r, b.region, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return SONIC_ERR_CUDA;
    if (cudaIpcOpenMemHandle(&f, b.flags, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaIpcCloseMemHandle(r);
      return SONIC_ERR_CUDA;
    }
    p->base[g] = r;
    p->fbase[g] = static_cast<unsigned long long*>(f);
    p->opened[g] = true;
  }
  if (!p->ftab && cudaMalloc(&p->ftab, SONIC_PEER_MAX * sizeof(void*)) != cudaSuccess) return SONIC_ERR_CUDA;
  if (cudaMemcpy(p->ftab, p->fbase, SONIC_PEER_MAX * sizeof(void*), cudaMemcpyHostToDevice) != cudaSuccess)
    return SONIC_ERR_CUDA;
  return SONIC_OK;
}

void* sonic_peer_base(const sonic_peer* p, int r) {
  return (p && r >= 0 && r < p->world) ? p->base[r] : nullptr;
}

sonic_status sonic_peer_destroy(sonic_peer* p) {
  if (!p) return SONIC_OK;
  cudaDeviceSynchronize();
  for (int g = 0; g < p->world; ++g)
    if (p->opened[g]) {
      cudaIpcCloseMemHandle(p->base[g]);
      cudaIpcCloseMemHandle(p->fbase[g]);
    }
  if (p->region) cudaFree(p->region);
  if (p->flags) cudaFree(p->flags);
  if (p->ftab) cudaFree(p->ftab);
  delete p;
  return SONIC_OK;
}

sonic_status sonic_peer_barrier(sonic_peer* p, void* stream) {
  if (!p || !p->ftab) return SONIC_ERR_INVALID_ARG;  // not opened
  ++p->epoch;
  k_peer_barrier<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(p->ftab, p->flags, p->rank, p->world, p->epoch);
  set_last_launch_count(1);
  return cudaGetLastError() == cudaSuccess ? SONIC_OK : SONIC_ERR_CUDA;
}

sonic_status sonic_ep_pack_peer(const sonic_moe_desc* D, int G, const sonic_ep_plan* plan, const void* src,
                                const sonic_peer* p, size_t region_off, const int32_t* dst_row0, void* stream) {
  if (!D || !plan || !src || !dst_row0 || D->d % 8 != 0) return SONIC_ERR_INVALID_ARG;
  PeerRows R{};
  PeerPtrs P{};
  if (!fill_rows(p, G, nullptr, nullptr, dst_row0, &R, &P)) return SONIC_ERR_INVALID_ARG;
  const long long rows = D->T * G;
  k_pack_peer<<<(unsigned)((rows * 32 + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(src), plan->send_token, plan->send_offsets, G, D->d, P, region_off, R);
  set_last_launch_count(1);
  return cudaGetLastError() == cudaSuccess ? SONIC_OK : SONIC_ERR_CUDA;
}

sonic_status sonic_ep_pack_peer_dev(const sonic_moe_desc* D, int G, const sonic_ep_plan* plan, const void* src,
                                    const sonic_peer* p, size_t region_off, size_t counts_off, int count_cols,
                                    void* stream) {
  if (!D || !plan || !src || D->d % 8 != 0 || count_cols < G) return SONIC_ERR_INVALID_ARG;
  PeerRows R{};
  PeerPtrs P{};
  if (!fill_rows(p, G, nullptr, nullptr, nullptr, &R, &P)) return SONIC_ERR_INVALID_ARG;
  const int* cnt = reinterpret_cast<const int*>(static_cast<const char*>(p->region) + counts_off);
  const long long rows = D->T * G;
  k_pack_peer_dev<<<(unsigned)((rows * 32 + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(src), plan->send_token, plan->send_offsets, G, D->d, P, region_off, cnt,
      count_cols, p->rank);
  set_last_launch_count(1);
  return cudaGetLastError() == cudaSuccess ? SONIC_OK : SONIC_ERR_CUDA;
}

sonic_status sonic_peer_put_rows_dev(const sonic_peer* p, int G, const void* src, size_t row_bytes, int direction,
                                     size_t counts_off, int count_cols, size_t region_off, void* stream) {
  if (!src || row_bytes == 0 || row_bytes % 4 != 0 || region_off % 4 != 0 || count_cols < G ||
      (direction != 0 && direction != 1))
    return SONIC_ERR_INVALID_ARG;
  PeerRows R{};
  PeerPtrs P{};
  if (!fill_rows(p, G, nullptr, nullptr, nullptr, &R, &P)) return SONIC_ERR_INVALID_ARG;
  const int* cnt = reinterpret_cast<const int*>(static_cast<const char*>(p->region) + counts_off);
  dim3 grid((unsigned)std::max(1, 296 / G), G);
  const bool v16 = row_bytes % 16 == 0 && region_off % 16 == 0 && reinterpret_cast<uintptr_t>(src) % 16 == 0;
  if (v16)
    k_put_rows_dev<uint4><<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const char*>(src), row_bytes, P, region_off, cnt, count_cols, p->rank, G, direction);
  else
    k_put_rows_dev<uint32_t><<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const char*>(src), row_bytes, P, region_off, cnt, count_cols, p->rank, G, direction);
  set_last_launch_count(1);
  return cudaGetLastError() == cudaSuccess ? SONIC_OK : SONIC_ERR_CUDA;
}

sonic_status sonic_peer_zero_tail(const sonic_peer* p, int G, size_t row_bytes, size_t counts_off, int count_cols,
                                  size_t region_off, long long cap_rows, void* stream) {
  if (!p || G != p->world || row_bytes == 0 || row_bytes % 4 != 0 || region_off % 4 != 0 || count_cols < G ||
      cap_rows < 0 || region_off + (size_t)cap_rows * row_bytes > p->bytes)
    return SONIC_ERR_INVALID_ARG;
  const int* cnt = reinterpret_cast<const int*>(static_cast<const char*>(p->region) + counts_off);
  k_zero_tail<<<296, 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<char*>(p->region) + region_off, row_bytes,
                                                                  cnt, count_cols, p->rank, G, cap_rows);
  set_last_launch_count(1);
  return cudaGetLastError() == cudaSuccess ? SONIC_OK : SONIC_ERR_CUDA;
}

sonic_status sonic_peer_put_rows(const sonic_peer* p, int G, const void* src, size_t row_bytes,
                                 const int32_t* src_row0, const int32_t* cnt, const int32_t* dst_row0,
                                 size_t region_off, void* stream) {
  if (!src || row_bytes == 0 || row_bytes % 4 != 0 || !src_row0 || !cnt || !dst_row0 || region_off % 4 != 0)
    return SONIC_ERR_INVALID_ARG;
  PeerRows R{};
  PeerPtrs P{};
  if (!fill_rows(p, G, src_row0, cnt, dst_row0, &R, &P)) return SONIC_ERR_INVALID_ARG;
  for (int g = 0; g < G; ++g)
    if (region_off + ((size_t)R.dst_row0[g] + R.cnt[g]) * row_bytes > p->bytes) return SONIC_ERR_INVALID_ARG;
  dim3 grid((unsigned)std::max(1, 296 / G), G);
  const bool v16 = row_bytes % 16 == 0 && region_off % 16 == 0 && reinterpret_cast<uintptr_t>(src) % 16 == 0;
  if (v16)
    k_put_rows<uint4><<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<const char*>(src), row_bytes,
                                                                         P, region_off, R);
  else
    k_put_rows<uint32_t><<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<const char*>(src),
                                                                            row_bytes, P, region_off, R);
  set_last_launch_count(1);
  return cudaGetLastError() == cudaSuccess ? SONIC_OK : SONIC_ERR_CUDA;
}

}  // extern "C"
