// dfs_lab2.cu — round-2 A/B harness for the shared-memory cost model of the DFS stack
// (not product code). Variants of the product step (nq_kernel.cuh, V4 layout):
//
//   GUARD bit0: the pop LDS.128 is skipped by a warp-uniform branch when no lane pops
//   GUARD bit1: the push STS.128 is skipped the same way when no lane pushes
//   PAD:        level stride BLOCK+1 frames (lane t's frame at level L in bank group
//               (t + L) mod 8 instead of t mod 8)
//
// Each variant counts the same device-resident frontier; totals and Alg. 3 node counts
// are checked against OEIS and against the product kernel.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
//        -I include -I paper_2511_12009_b200/csrc -o tools/microbench/dfs_lab2 \
//        tools/microbench/dfs_lab2.cu paper_2511_12009_b200/csrc/nq_frontier.cpp
//   ./tools/microbench/dfs_lab2 20 7 3
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "nq_gpu.h"
#include "nq_internal.h"
#include "nq_kernel.cuh"

namespace nqb200 {
int set_error(int code, const std::string& msg) {
  std::fprintf(stderr, "error: %s\n", msg.c_str());
  return code;
}
}  // namespace nqb200

using namespace nqb200;

#define CK(x)                                                                                 \
  do {                                                                                        \
    cudaError_t e = (x);                                                                      \
    if (e != cudaSuccess) {                                                                   \
      std::fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);   \
      std::exit(1);                                                                           \
    }                                                                                         \
  } while (0)

// The product step split in three: compute (predicates out as 0/1), push, pop.
template <uint32_t STRIDE, int GUARD>
__device__ __forceinline__ void g_step(uint32_t& C, uint32_t& l, uint32_t& r, uint32_t& a,
                                       uint32_t& sp, uint32_t& sol, uint32_t& its) {
  uint32_t pa, po, nC, nl, nr, na2, a1;
  asm volatile(
      "{\n\t"
      ".reg .u32 na, p, t;\n\t"
      ".reg .pred qa, qk, qo, qs;\n\t"
      "neg.s32 na, %9;\n\t"
      "and.b32 p, %9, na;\n\t"
      "setp.ne.u32 qk, p, 0;\n\t"
      "xor.b32 %4, %9, p;\n\t"
      "setp.ne.u32 qa, %4, 0;\n\t"
      "sub.u32 %5, %10, p;\n\t"
      "add.u32 t, %11, p;\n\t"
      "add.u32 %6, t, t;\n\t"
      "add.u32 t, %12, p;\n\t"
      "shr.u32 %7, t, 1;\n\t"
      "lop3.b32 %8, %5, %6, %7, 0x10;\n\t"
      "shr.u32 na, na, 31;\n\t"
      "add.u32 %3, %3, na;\n\t"
      "setp.eq.and.u32 qs, %5, 0, qk;\n\t"
      "@qs add.u32 %2, %2, 1;\n\t"
      "setp.eq.and.u32 qo, %8, 0, qk;\n\t"
      "selp.u32 %0, 1, 0, qa;\n\t"
      "selp.u32 %1, 1, 0, qo;\n\t"
      "}"
      : "=r"(pa), "=r"(po), "+r"(sol), "+r"(its), "=r"(a1), "=r"(nC), "=r"(nl), "=r"(nr), "=r"(na2)
      : "r"(a), "r"(C), "r"(l), "r"(r));
  const bool do_push = (GUARD & 2) ? __any_sync(0xffffffffu, pa) : true;
  if (do_push) {
    asm volatile(
        "{\n\t.reg .pred q;\n\t"
        "setp.ne.u32 q, %5, 0;\n\t"
        "@q st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n\t"
        "@q add.u32 %0, %0, %6;\n\t}"
        : "+r"(sp)
        : "r"(C), "r"(l), "r"(r), "r"(a1), "r"(pa), "n"(STRIDE)
        : "memory");
  }
  C = nC;
  l = nl;
  r = nr;
  a = na2;
  const bool do_pop = (GUARD & 1) ? __any_sync(0xffffffffu, po) : true;
  if (do_pop) {
    asm volatile(
        "{\n\t.reg .pred q;\n\t"
        "setp.ne.u32 q, %5, 0;\n\t"
        "@q sub.u32 %0, %0, %6;\n\t"
        "@q ld.shared.v4.u32 {%1, %2, %3, %4}, [%0];\n\t}"
        : "+r"(sp), "+r"(C), "+r"(l), "+r"(r), "+r"(a)
        : "r"(po), "n"(STRIDE)
        : "memory");
  }
}

// "Stay" in registers: a dead-end child whose parent still has candidates keeps the
// parent (predicated moves) instead of pushing it and popping it back; pushes and pops
// are then only the non-stay ones (28% fewer of each).
template <uint32_t STRIDE, int MOVMODE>
__device__ __forceinline__ void stay_step(uint32_t& C, uint32_t& l, uint32_t& r, uint32_t& a,
                                          uint32_t& sp, uint32_t& sol, uint32_t& its) {
  if constexpr (MOVMODE == 0) {
    asm volatile(
        "{\n\t"
        ".reg .u32 na, p, nC, t, nl, nr, na2;\n\t"
        ".reg .pred pa, pk, pd, pu, po, ps, pst;\n\t"
        "neg.s32 na, %3;\n\t"
        "and.b32 p, %3, na;\n\t"
        "setp.ne.u32 pk, p, 0;\n\t"
        "xor.b32 %3, %3, p;\n\t"
        "setp.ne.u32 pa, %3, 0;\n\t"
        "sub.u32 nC, %0, p;\n\t"
        "add.u32 t, %1, p;\n\t"
        "add.u32 nl, t, t;\n\t"
        "add.u32 t, %2, p;\n\t"
        "shr.u32 nr, t, 1;\n\t"
        "lop3.b32 na2, nC, nl, nr, 0x10;\n\t"
        "shr.u32 na, na, 31;\n\t"
        "add.u32 %6, %6, na;\n\t"
        "setp.eq.and.u32 ps, nC, 0, pk;\n\t"
        "@ps add.u32 %5, %5, 1;\n\t"
        "setp.eq.u32 pd, na2, 0;\n\t"
        "and.pred pst, pd, pa;\n\t"          // stay: dead child, parent has candidates
        "not.pred pu, pd;\n\t"
        "and.pred pu, pu, pa;\n\t"           // push: live child, parent has candidates
        "@pu st.shared.v4.u32 [%4], {%0, %1, %2, %3};\n\t"
        "@pu add.u32 %4, %4, %7;\n\t"
        "not.pred po, pa;\n\t"
        "and.pred po, po, pd;\n\t"
        "and.pred po, po, pk;\n\t"           // pop: dead child, parent exhausted
        "@!pst mov.u32 %0, nC;\n\t"
        "@!pst mov.u32 %1, nl;\n\t"
        "@!pst mov.u32 %2, nr;\n\t"
        "@!pst mov.u32 %3, na2;\n\t"
        "@po sub.u32 %4, %4, %7;\n\t"
        "@po ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n\t"
        "}"
        : "+r"(C), "+r"(l), "+r"(r), "+r"(a), "+r"(sp), "+r"(sol), "+r"(its)
        : "n"(STRIDE)
        : "memory");
  }
}

struct LabP {
  DfsParams P;
  unsigned long long* lane_steps;
};

template <int BLOCK, int KSTEP, int GUARD, int PAD>
__global__ void __launch_bounds__(BLOCK) g_kernel(LabP LP) {
  const DfsParams& P = LP.P;
  extern __shared__ uint4 stk[];
  constexpr uint32_t STRIDE = (BLOCK + PAD) * 16u;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t base0 = static_cast<uint32_t>(__cvta_generic_to_shared(stk)) + threadIdx.x * 16u;
  const uint32_t base1 = base0 + STRIDE;
  sts128(base0, 0u, 0u, 0u, 0u);
  uint32_t C = 0u, l = 0u, r = 0u, a = 0u, sp = base1, sol = 0u, its = 0u, weight = 0u;
  bool busy = false, exhausted = false;
  unsigned long long tot_w = 0, tot_raw = 0, tot_it = 0, tot_subs = 0;
  uint32_t blocks = 0;
  for (;;) {
    if (__ballot_sync(0xffffffffu, a == 0u)) {
      for (;;) {
        if (a == 0u && busy) {
          tot_w += static_cast<unsigned long long>(weight) * sol;
          tot_raw += sol;
          tot_it += its;
          tot_subs += 1;
          sol = its = 0u;
          busy = false;
        }
        if (exhausted) break;
        const uint32_t need = __ballot_sync(0xffffffffu, a == 0u);
        if (need == 0u) break;
        const uint32_t leader = __ffs(need) - 1u;
        const uint32_t n_need = __popc(need);
        unsigned long long first = 0;
        if (lane == leader) first = atomicAdd(P.cursor, static_cast<unsigned long long>(n_need));
        first = __shfl_sync(0xffffffffu, first, leader);
        if (first + n_need >= P.count) exhausted = true;
        if (a == 0u) {
          const unsigned long long pos = first + __popc(need & ((1u << lane) - 1u));
          if (pos < P.count) {
            const unsigned long long idx = P.count - 1ull - pos;
            const uint4 s = __ldg(&P.subs[idx]);
            busy = true;
            weight = s.w >> 8;
            if (s.x == P.mask) {
              sol = 1u;
            } else {
              C = P.mask & ~s.x;
              l = s.y;
              r = s.z;
              a = C & ~(l | r);
              sp = base1;
            }
            if (a == 0u) C = 0u;
          }
        }
      }
      if (exhausted && __all_sync(0xffffffffu, a == 0u)) break;
    }
#pragma unroll
    for (int k = 0; k < KSTEP; ++k) {
      if constexpr (GUARD == 8) stay_step<STRIDE, 0>(C, l, r, a, sp, sol, its);
      else if constexpr (GUARD == 9) dfs_step<STRIDE, kLayoutV4>(C, l, r, a, sp, sol, its);
      else g_step<STRIDE, GUARD>(C, l, r, a, sp, sol, its);
    }
    if (((++blocks) & 0x7fffu) == 0u) {
      tot_w += static_cast<unsigned long long>(weight) * sol;
      tot_raw += sol;
      tot_it += its;
      sol = its = 0u;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    tot_w += __shfl_down_sync(0xffffffffu, tot_w, off);
    tot_raw += __shfl_down_sync(0xffffffffu, tot_raw, off);
    tot_it += __shfl_down_sync(0xffffffffu, tot_it, off);
    tot_subs += __shfl_down_sync(0xffffffffu, tot_subs, off);
  }
  if (lane == 0u) {
    atomicAdd(P.totals + 0, tot_w);
    atomicAdd(P.totals + 1, tot_raw);
    atomicAdd(P.totals + 2, tot_it);
    atomicAdd(P.totals + 3, tot_subs);
  }
}

static const unsigned long long kOeis[] = {1ull, 0ull, 0ull, 2ull, 10ull, 4ull, 40ull, 92ull, 352ull, 724ull,
    2680ull, 14200ull, 73712ull, 365596ull, 2279184ull, 14772512ull, 95815104ull, 666090624ull,
    4968057848ull, 39029188884ull, 314666222712ull, 2691008701644ull, 24233937684440ull};

struct Bed {
  int n, R, sms;
  uint4* d_subs;
  unsigned long long count;
  unsigned long long* d_ctl;
};

template <class PT>
void run(const Bed& b, const char* name, void (*kern)(PT), int block, int pad, int reps) {
  const int levels = b.n - 1 - b.R + 1;
  const size_t smem = size_t(levels) * (block + pad) * 16;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, smem));
  LabP LP{};
  LP.P.subs = b.d_subs;
  LP.P.count = b.count;
  LP.P.cursor = b.d_ctl;
  LP.P.stop = b.d_ctl + 6;
  LP.P.totals = b.d_ctl + 1;
  LP.P.mask = (1u << b.n) - 1u;
  LP.P.n = b.n;
  LP.P.min_placed = b.R;
  LP.P.reverse = 1;
  LP.P.lastrow = 1;
  LP.P.donate = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  unsigned long long h[8];
  for (int i = 0; i < reps; ++i) {
    CK(cudaMemset(b.d_ctl, 0, 8 * sizeof(unsigned long long)));
    cudaEventRecord(e0);
    if constexpr (sizeof(PT) == sizeof(LabP)) kern<<<per_sm * b.sms, block, smem>>>(LP);
    else kern<<<per_sm * b.sms, block, smem>>>(LP.P);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
    CK(cudaMemcpy(h, b.d_ctl, sizeof h, cudaMemcpyDeviceToHost));
  }
  const unsigned long long nodes = h[3] - h[2];
  const bool ok = h[1] == kOeis[b.n - 1];
  std::printf("{\"kernel\": \"%s\", \"n\": %d, \"R\": %d, \"block\": %d, \"blocks_per_sm\": %d, "
              "\"ms\": %.3f, \"ok\": %s, \"solutions\": %llu, \"nodes\": %llu, "
              "\"nodes_per_s\": %.4e, \"nodes_per_sm_clk\": %.3f}\n",
              name, b.n, b.R, block, per_sm, best, ok ? "true" : "false", h[1], nodes,
              nodes / (best * 1e-3), nodes / (best * 1e-3) / (b.sms * 1.965e9));
  std::fflush(stdout);
}

int main(int argc, char** argv) {
  Bed b{};
  b.n = argc > 1 ? std::atoi(argv[1]) : 18;
  b.R = argc > 2 ? std::atoi(argv[2]) : 6;
  const int reps = argc > 3 ? std::atoi(argv[3]) : 3;
  const int only = argc > 4 ? std::atoi(argv[4]) : -1;
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  b.sms = p.multiProcessorCount;
  uint64_t total = 0;
  generate_slice(b.n, b.R, 1, 0, nullptr, 0, &total);
  std::vector<nq_sub> subs(total);
  generate_slice(b.n, b.R, 1, 0, subs.data(), total, &total);
  b.count = total;
  CK(cudaMalloc(&b.d_subs, total * 16));
  CK(cudaMemcpy(b.d_subs, subs.data(), total * 16, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&b.d_ctl, 8 * sizeof(unsigned long long)));
  int idx = 0;
  auto pick = [&](auto&&... xs) { if (only < 0 || only == idx) run(b, xs...); ++idx; };
  pick("prod v4", nq_dfs_kernel<128, 32, false, kLayoutV4>, 128, 0, reps);
  pick("lab: product step", g_kernel<128, 32, 9, 0>, 128, 0, reps);
  pick("lab: stay in registers (predicated moves)", g_kernel<128, 32, 8, 0>, 128, 0, reps);
  pick("split g0", g_kernel<128, 32, 0, 0>, 128, 0, reps);
  pick("split g1 (guard pop)", g_kernel<128, 32, 1, 0>, 128, 0, reps);
  pick("split g2 (guard push)", g_kernel<128, 32, 2, 0>, 128, 0, reps);
  pick("split g3 (guard both)", g_kernel<128, 32, 3, 0>, 128, 0, reps);
  pick("split g0 pad", g_kernel<128, 32, 0, 1>, 128, 1, reps);
  pick("split g1 pad", g_kernel<128, 32, 1, 1>, 128, 1, reps);
  return 0;
}
