// nq_expand.cu — GPU-side frontier deepening.
//
// The host generator (nq_frontier.cpp) emits the folded stream of for_each_subproblem
// (subproblems.hpp:80-108) at depth R. At large N that stream is big (N=27, R=7:
// 453,688,251 records, 7.26 GB). Here a small coarse frontier (depth R0, shipped from
// the host) is deepened to depth R on the device, in the same order as the host's
// nq_expand (each root's descendants in expand_rows' DFS order, subproblems.hpp:41-55,
// roots in order, multiplier inherited), one row per pass:
//   1. one thread per record counts its children (popcount of the next row's mask);
//   2. an exclusive scan turns counts into output offsets (block scans + a carry pass);
//   3. one thread per record writes its children, lowest column first, at its offset.
// The deepened records are then counted by nq_dfs_kernel without leaving the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <cstdint>
#include <string>

#include "nq_gpu.h"
#include "nq_internal.h"

namespace nqb200 {

constexpr int kScanBlock = 1024;

// In-place exclusive scan of each kScanBlock-element tile; tile totals to sums[tile].
__global__ void __launch_bounds__(kScanBlock) scan_tiles_kernel(unsigned long long* v, uint64_t count,
                                                                 unsigned long long* sums) {
  __shared__ unsigned long long warp_tot[kScanBlock / 32];
  const uint64_t i = blockIdx.x * uint64_t(kScanBlock) + threadIdx.x;
  const unsigned long long x = i < count ? v[i] : 0ull;
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  unsigned long long incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= static_cast<unsigned>(o)) incl += y;
  }
  if (lane == 31u) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    unsigned long long t = warp_tot[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= static_cast<unsigned>(o)) t += y;
    }
    warp_tot[lane] = t;  // inclusive over warps
  }
  __syncthreads();
  const unsigned long long before = warp ? warp_tot[warp - 1] : 0ull;
  if (i < count) v[i] = before + incl - x;
  if (threadIdx.x == kScanBlock - 1) sums[blockIdx.x] = before + incl;
}

// Exclusive scan of the tile totals by one block, carrying across chunks; the grand
// total lands in *total.
__global__ void __launch_bounds__(kScanBlock) scan_sums_kernel(unsigned long long* sums, uint64_t tiles,
                                                                unsigned long long* total) {
  __shared__ unsigned long long warp_tot[kScanBlock / 32];
  __shared__ unsigned long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  for (uint64_t base = 0; base < tiles; base += kScanBlock) {
    const uint64_t i = base + threadIdx.x;
    const unsigned long long x = i < tiles ? sums[i] : 0ull;
    unsigned long long incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= static_cast<unsigned>(o)) incl += y;
    }
    if (lane == 31u) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      unsigned long long t = warp_tot[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= static_cast<unsigned>(o)) t += y;
      }
      warp_tot[lane] = t;
    }
    __syncthreads();
    const unsigned long long before = (warp ? warp_tot[warp - 1] : 0ull) + carry;
    if (i < tiles) sums[i] = before + incl - x;
    __syncthreads();
    if (threadIdx.x == kScanBlock - 1) carry = before + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void add_tile_offsets_kernel(unsigned long long* v, uint64_t count,
                                        const unsigned long long* sums) {
  const uint64_t i = blockIdx.x * uint64_t(kScanBlock) + threadIdx.x;
  if (i < count) v[i] += sums[blockIdx.x];
}

// ---- level-synchronous deepening (one row per pass) ------------------------------------
// Pass: every record below the target places one more queen (each candidate of its next
// row, lowest column first, multiplier kept); records at the target are copied. Counts
// -> exclusive scan -> emit keeps the DFS order of the stream; writes from one thread are
// contiguous, so the pass streams at close to HBM speed.
__global__ void level_count_kernel(const uint4* in, uint64_t count, uint32_t mask, int target,
                                   unsigned long long* counts, unsigned long long* bad,
                                   unsigned int* min_placed) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint4 s = in[i];
    const int placed = static_cast<int>(s.w & 0xffu);
    if (bad) {  // first pass: validate the roots
      if ((s.x & ~mask) != 0u || __popc(s.x) != placed) {
        atomicMin(bad, static_cast<unsigned long long>(i));
        counts[i] = 0;
        continue;
      }
      atomicMin(min_placed, static_cast<unsigned int>(placed));
    }
    counts[i] = placed >= target ? 1ull : static_cast<unsigned long long>(__popc(mask & ~(s.x | s.y | s.z)));
  }
}

__global__ void level_emit_kernel(const uint4* in, uint64_t count, uint32_t mask, int target,
                                  const unsigned long long* offsets, uint4* out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint4 s = in[i];
    uint64_t at = offsets[i];
    const int placed = static_cast<int>(s.w & 0xffu);
    if (placed >= target) {
      out[at] = s;
      continue;
    }
    const uint32_t w = (s.w & ~0xffu) | static_cast<uint32_t>(placed + 1);
    uint32_t v = mask & ~(s.x | s.y | s.z);
    while (v) {
      const uint32_t p = v & (0u - v);
      v ^= p;
      out[at++] = make_uint4(s.x | p, (s.y | p) << 1, (s.z | p) >> 1, w);
    }
  }
}

}  // namespace nqb200

using namespace nqb200;

namespace {

#define NQX_CUDA(call)                                                                          \
  do {                                                                                          \
    cudaError_t e_ = (call);                                                                    \
    if (e_ != cudaSuccess)                                                                      \
      return set_error(NQ_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_) + " (" +   \
                                     __FILE__ + ":" + std::to_string(__LINE__) + ")");          \
  } while (0)

// The level buffers (N=20 R=4->7: ~1 GB across passes) come from the device's default
// stream-ordered pool. Its default release threshold of 0 hands every freed byte back to
// the driver at the next synchronize, so each call re-maps them (~50 ms at N=20). Keep up
// to kPoolRetainBytes cached across calls instead.
constexpr uint64_t kPoolRetainBytes = 8ull << 30;

int retain_pool(int device) {
  static std::once_flag once[64];
  if (device < 0 || device >= 64) return NQ_OK;
  int rc = NQ_OK;
  std::call_once(once[device], [&] {
    cudaMemPool_t pool;
    uint64_t thr = kPoolRetainBytes;
    cudaError_t e = cudaDeviceGetDefaultMemPool(&pool, device);
    if (e == cudaSuccess) e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    if (e != cudaSuccess)
      rc = set_error(NQ_ECUDA, std::string("default mem pool release threshold: ") + cudaGetErrorString(e));
  });
  return rc;
}

struct DevBuf {  // stream-ordered allocation, freed on the same stream
  void* p = nullptr;
  cudaStream_t s = nullptr;
  ~DevBuf() {
    if (p) cudaFreeAsync(p, s);
  }
};

}  // namespace

namespace nqb200 {

// Deepens `count` device roots to `target` rows on `st`; returns a new device buffer of
// *total records (caller frees with cudaFreeAsync on st).
int expand_levels(int device, int n, const nq_sub* dev_roots, uint64_t count, int target,
                  cudaStream_t st, uint4** out, uint64_t* total) {
  *out = nullptr;
  *total = 0;
  if (n < 1 || n > 32)
    return set_error(NQ_ECONFIG, "board size must be in [1, 32], got " + std::to_string(n));
  if (target < 1 || target >= n)
    return set_error(NQ_ECONFIG, "target rows must satisfy 1 <= T < n (n=" + std::to_string(n) +
                                     ", T=" + std::to_string(target) + ")");
  if (count == 0) return NQ_OK;
  if (!dev_roots) return set_error(NQ_ECONFIG, "null roots");
  NvtxRange range("nq_expand_device (level passes)");
  NQX_CUDA(cudaSetDevice(device));
  if (int rc = retain_pool(device)) return rc;
  const uint32_t mask = n >= 32 ? 0xffffffffu : ((1u << n) - 1u);
  int sms = 0;
  NQX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  DevBuf ctl{nullptr, st};
  NQX_CUDA(cudaMallocAsync(&ctl.p, 3 * sizeof(unsigned long long), st));
  auto* d_ctl = static_cast<unsigned long long*>(ctl.p);  // [0] total, [1] bad root, [2] min placed
  NQX_CUDA(cudaMemsetAsync(d_ctl, 0x00, sizeof(unsigned long long), st));
  NQX_CUDA(cudaMemsetAsync(d_ctl + 1, 0xff, 2 * sizeof(unsigned long long), st));
  const uint4* cur = reinterpret_cast<const uint4*>(dev_roots);
  uint64_t cur_n = count;
  uint4* owned = nullptr;  // the current level's buffer when we allocated it
  int passes = -1;         // known after the first count pass
  for (int pass = 0;; ++pass) {
    const uint64_t tiles = (cur_n + kScanBlock - 1) / kScanBlock;
    DevBuf counts{nullptr, st}, sums{nullptr, st};
    NQX_CUDA(cudaMallocAsync(&counts.p, cur_n * sizeof(unsigned long long), st));
    NQX_CUDA(cudaMallocAsync(&sums.p, tiles * sizeof(unsigned long long), st));
    auto* d_counts = static_cast<unsigned long long*>(counts.p);
    auto* d_sums = static_cast<unsigned long long*>(sums.p);
    const int threads = 256;
    const int grid = static_cast<int>(std::min<uint64_t>((cur_n + threads - 1) / threads,
                                                         static_cast<uint64_t>(sms) * 32));
    level_count_kernel<<<grid, threads, 0, st>>>(cur, cur_n, mask, target, d_counts,
                                                 pass == 0 ? d_ctl + 1 : nullptr,
                                                 reinterpret_cast<unsigned int*>(d_ctl + 2));
    NQX_CUDA(cudaGetLastError());
    scan_tiles_kernel<<<static_cast<unsigned>(tiles), kScanBlock, 0, st>>>(d_counts, cur_n, d_sums);
    scan_sums_kernel<<<1, kScanBlock, 0, st>>>(d_sums, tiles, d_ctl);
    add_tile_offsets_kernel<<<static_cast<unsigned>(tiles), kScanBlock, 0, st>>>(d_counts, cur_n, d_sums);
    NQX_CUDA(cudaGetLastError());
    unsigned long long h[3];
    NQX_CUDA(cudaMemcpyAsync(h, d_ctl, sizeof h, cudaMemcpyDeviceToHost, st));
    NQX_CUDA(cudaStreamSynchronize(st));
    if (pass == 0) {
      if (h[1] != ~0ull) return set_error(NQ_ECONFIG, "root " + std::to_string(h[1]) + " is malformed");
      const int min_placed = static_cast<int>(h[2] & 0xffffffffu);
      passes = std::max(target - min_placed, 1);  // >= 1 pass: the output is a fresh buffer
    }
    if (h[0] == 0) {  // every record of this level is a dead end: nothing to deepen or count
      if (owned) NQX_CUDA(cudaFreeAsync(owned, st));
      NQX_CUDA(cudaStreamSynchronize(st));
      return NQ_OK;  // *out = nullptr, *total = 0
    }
    uint4* next = nullptr;
    NQX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&next), std::max<uint64_t>(h[0], 1) * 16, st));
    level_emit_kernel<<<grid, threads, 0, st>>>(cur, cur_n, mask, target, d_counts, next);
    NQX_CUDA(cudaGetLastError());
    if (owned) NQX_CUDA(cudaFreeAsync(owned, st));
    owned = next;
    cur = next;
    cur_n = h[0];
    if (pass + 1 >= passes) break;
  }
  NQX_CUDA(cudaStreamSynchronize(st));
  *out = owned;
  *total = cur_n;
  return NQ_OK;
}

}  // namespace nqb200

extern "C" int nq_expand_device(int device, int n, const nq_sub* dev_roots, uint64_t count,
                                int target_rows, nq_sub* dev_out, uint64_t cap, uint64_t* total) {
  if (!total) return set_error(NQ_ECONFIG, "null total");
  *total = 0;
  const cudaStream_t st = cudaStreamPerThread;  // no implicit sync with other workers' streams
  uint4* buf = nullptr;
  uint64_t n_out = 0;
  if (int rc = expand_levels(device, n, dev_roots, count, target_rows, st, &buf, &n_out)) {
    if (buf) cudaFreeAsync(buf, st);
    return rc;
  }
  DevBuf guard{buf, st};
  *total = n_out;
  if (!dev_out || cap == 0 || n_out == 0) return NQ_OK;
  if (n_out > cap)
    return set_error(NQ_ECONFIG, "output capacity " + std::to_string(cap) + " below the " +
                                     std::to_string(n_out) + " deepened records");
  NQX_CUDA(cudaMemcpyAsync(dev_out, buf, n_out * sizeof(nq_sub), cudaMemcpyDeviceToDevice, st));
  NQX_CUDA(cudaStreamSynchronize(st));
  return NQ_OK;
}
