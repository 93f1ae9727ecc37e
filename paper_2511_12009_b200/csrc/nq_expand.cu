// nq_expand.cu — GPU-side frontier deepening.
//
// The host generator (nq_frontier.cpp) emits the folded stream of for_each_subproblem
// (subproblems.hpp:80-108) at depth R. At large N that stream is big (N=27, R=7:
// 453,688,251 records, 7.26 GB). Here a small coarse frontier (depth R0, shipped from
// the host) is deepened to depth R on the device, in the same order as the host's
// nq_expand (each root's descendants in expand_rows' DFS order, subproblems.hpp:41-55,
// roots in order, multiplier inherited):
//   1. one thread per root counts its depth-R descendants (bounded DFS, local frames);
//   2. an exclusive scan turns counts into output offsets (block scans + a carry pass);
//   3. one thread per root writes its descendants at its offset.
// The deepened records are then counted by nq_dfs_kernel without leaving the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>

#include "nq_gpu.h"
#include "nq_internal.h"

namespace nqb200 {

constexpr int kExpandMaxDepth = 16;  // rows deepened per root (target - placed)
constexpr int kScanBlock = 1024;

// Walk the depth-`target` descendants of one root in DFS order (lowest column first);
// EMIT = false counts them, EMIT = true writes them to out[at...].
template <bool EMIT>
__device__ uint64_t expand_one(uint4 root, uint32_t mask, int target, nq_sub* out, uint64_t at) {
  const int placed = static_cast<int>(root.w & 0xffu);
  if (placed >= target) {
    if (EMIT) out[at] = nq_sub{root.x, root.y, root.z, root.w};
    return 1;
  }
  const uint32_t mult = root.w & ~0xffu;
  const int depth = target - placed;  // rows to place, <= kExpandMaxDepth
  uint32_t cols[kExpandMaxDepth], diag[kExpandMaxDepth], anti[kExpandMaxDepth],
      cand[kExpandMaxDepth];
  cols[0] = root.x;
  diag[0] = root.y;
  anti[0] = root.z;
  cand[0] = mask & ~(root.x | root.y | root.z);
  int lv = 0;
  uint64_t k = 0;
  while (lv >= 0) {
    const uint32_t a = cand[lv];
    if (a == 0u) {
      --lv;
      continue;
    }
    const uint32_t p = a & (0u - a);
    cand[lv] = a ^ p;
    const uint32_t c = cols[lv] | p, d = (diag[lv] | p) << 1, r = (anti[lv] | p) >> 1;
    if (lv + 1 == depth) {
      if (EMIT) out[at + k] = nq_sub{c, d, r, static_cast<uint32_t>(target) | mult};
      ++k;
    } else {
      ++lv;
      cols[lv] = c;
      diag[lv] = d;
      anti[lv] = r;
      cand[lv] = mask & ~(c | d | r);
    }
  }
  return k;
}

__global__ void expand_count_kernel(const uint4* roots, uint64_t count, uint32_t mask, int target,
                                    unsigned long long* counts, unsigned long long* bad) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint4 s = roots[i];
    const int placed = static_cast<int>(s.w & 0xffu);
    if ((s.x & ~mask) != 0u || __popc(s.x) != placed || target - placed > kExpandMaxDepth) {
      atomicMin(bad, static_cast<unsigned long long>(i));
      counts[i] = 0;
      continue;
    }
    counts[i] = expand_one<false>(s, mask, target, nullptr, 0);
  }
}

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

__global__ void expand_emit_kernel(const uint4* roots, uint64_t count, uint32_t mask, int target,
                                   const unsigned long long* offsets, nq_sub* out, uint64_t cap) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint4 s = roots[i];
    const uint64_t at = offsets[i];
    const uint64_t end = (i + 1 < count) ? offsets[i + 1] : cap;  // caller checked total <= cap
    if (at >= end) continue;
    expand_one<true>(s, mask, target, out, at);
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

struct DevBuf {  // stream-ordered allocation, freed on the same stream
  void* p = nullptr;
  cudaStream_t s = nullptr;
  ~DevBuf() {
    if (p) cudaFreeAsync(p, s);
  }
};

}  // namespace

extern "C" int nq_expand_device(int device, int n, const nq_sub* dev_roots, uint64_t count,
                                int target_rows, nq_sub* dev_out, uint64_t cap, uint64_t* total) {
  if (n < 1 || n > 31)
    return set_error(NQ_ECONFIG, "board size must be in [1, 31], got " + std::to_string(n));
  if (target_rows < 1 || target_rows >= n)
    return set_error(NQ_ECONFIG, "target rows must satisfy 1 <= T < n (n=" + std::to_string(n) +
                                     ", T=" + std::to_string(target_rows) + ")");
  if (!total) return set_error(NQ_ECONFIG, "null total");
  *total = 0;
  if (count == 0) return NQ_OK;
  if (!dev_roots) return set_error(NQ_ECONFIG, "null roots");
  NvtxRange range("nq_expand_device");
  NQX_CUDA(cudaSetDevice(device));
  // The calling thread's own stream: no implicit sync with other workers' streams.
  const cudaStream_t st = cudaStreamPerThread;
  const uint32_t mask = (1u << n) - 1u;
  const uint64_t tiles = (count + kScanBlock - 1) / kScanBlock;
  DevBuf counts{nullptr, st}, sums{nullptr, st}, ctl{nullptr, st};
  NQX_CUDA(cudaMallocAsync(&counts.p, count * sizeof(unsigned long long), st));
  NQX_CUDA(cudaMallocAsync(&sums.p, tiles * sizeof(unsigned long long), st));
  NQX_CUDA(cudaMallocAsync(&ctl.p, 2 * sizeof(unsigned long long), st));
  auto* d_counts = static_cast<unsigned long long*>(counts.p);
  auto* d_sums = static_cast<unsigned long long*>(sums.p);
  auto* d_ctl = static_cast<unsigned long long*>(ctl.p);  // [0] total, [1] first bad root
  NQX_CUDA(cudaMemsetAsync(d_ctl, 0x00, sizeof(unsigned long long), st));
  NQX_CUDA(cudaMemsetAsync(d_ctl + 1, 0xff, sizeof(unsigned long long), st));
  int sms = 0;
  NQX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  const int threads = 128;
  const int grid = static_cast<int>(std::min<uint64_t>((count + threads - 1) / threads,
                                                       static_cast<uint64_t>(sms) * 16));
  const auto* roots = reinterpret_cast<const uint4*>(dev_roots);
  expand_count_kernel<<<grid, threads, 0, st>>>(roots, count, mask, target_rows, d_counts, d_ctl + 1);
  NQX_CUDA(cudaGetLastError());
  scan_tiles_kernel<<<static_cast<unsigned>(tiles), kScanBlock, 0, st>>>(d_counts, count, d_sums);
  NQX_CUDA(cudaGetLastError());
  scan_sums_kernel<<<1, kScanBlock, 0, st>>>(d_sums, tiles, d_ctl);
  NQX_CUDA(cudaGetLastError());
  add_tile_offsets_kernel<<<static_cast<unsigned>(tiles), kScanBlock, 0, st>>>(d_counts, count, d_sums);
  NQX_CUDA(cudaGetLastError());
  unsigned long long h[2];
  NQX_CUDA(cudaMemcpyAsync(h, d_ctl, sizeof h, cudaMemcpyDeviceToHost, st));
  NQX_CUDA(cudaStreamSynchronize(st));
  if (h[1] != ~0ull)
    return set_error(NQ_ECONFIG, "root " + std::to_string(h[1]) +
                                     " is malformed or more than " +
                                     std::to_string(kExpandMaxDepth) + " rows from the target");
  *total = h[0];
  if (!dev_out || cap == 0) return NQ_OK;
  if (h[0] > cap)
    return set_error(NQ_ECONFIG, "output capacity " + std::to_string(cap) + " below the " +
                                     std::to_string(h[0]) + " deepened records");
  expand_emit_kernel<<<grid, threads, 0, st>>>(roots, count, mask, target_rows, d_counts, dev_out, h[0]);
  NQX_CUDA(cudaGetLastError());
  NQX_CUDA(cudaStreamSynchronize(st));
  return NQ_OK;
}
