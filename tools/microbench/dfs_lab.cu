// dfs_lab.cu — A/B harness for DFS step formulations (not product code).
//
// Builds the N=n, R=r folded frontier with the product generator (nq_frontier.cpp),
// then times several kernel formulations on the same device-resident batch and checks
// each total against OEIS. Used to pick the product kernel's step (nq_kernel.cuh).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
//        -I include -I paper_2511_12009_b200/csrc -o tools/microbench/dfs_lab \
//        tools/microbench/dfs_lab.cu paper_2511_12009_b200/csrc/nq_frontier.cpp
//   ./tools/microbench/dfs_lab 20 6
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

constexpr uint32_t kIdleL = 0x40000000u;  // lab-only: diagonal mask of the idle sentinel

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      std::fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      std::exit(1);                                                                  \
    }                                                                                \
  } while (0)

// ---------------------------------------------------------------------------------------
// Variant L: one asm block per KSTEP steps; moves forced onto the FMA pipe (IMAD by a
// runtime 1), iteration counter by IMAD.HI with a runtime 2, a2 computed in place.
// MODE bit0: moves via selp (ALU) instead of IMAD; bit1: sol via IMAD.HI on nC-1.
template <uint32_t STRIDE, int MODE>
__device__ __forceinline__ void lab_step(uint32_t& C, uint32_t& l, uint32_t& r, uint32_t& a,
                                         uint32_t& sp, uint32_t& sol, uint32_t& its,
                                         uint32_t one, uint32_t two) {
  if constexpr ((MODE & 1) == 0) {
    asm volatile(
        "{\n\t"
        ".reg .u32 na, p, nC, t, nl, nr, nv, a2;\n\t"
        ".reg .pred pd, pa, pu, po, ps, pk;\n\t"
        "neg.s32 na, %3;\n\t"
        "and.b32 p, %3, na;\n\t"
        "setp.ne.u32 pk, p, 0;\n\t"
        "xor.b32 %3, %3, p;\n\t"
        "setp.ne.u32 pa, %3, 0;\n\t"
        "sub.u32 nC, %0, p;\n\t"
        "add.u32 t, %1, p;\n\t"
        "mul.lo.u32 nl, t, %8;\n\t"
        "add.u32 t, %2, p;\n\t"
        "mul.hi.u32 nr, t, 0x80000000;\n\t"
        "lop3.b32 nv, nC, nl, nr, 0x10;\n\t"
        "setp.ne.u32 pd, nv, 0;\n\t"
        "mad.hi.u32 %6, na, %8, %6;\n\t"
        "setp.eq.u32 ps, nC, 0;\n\t"
        "@ps add.u32 %5, %5, 1;\n\t"
        "and.pred pu, pd, pa;\n\t"
        "@pu st.shared.v4.u32 [%4], {%0, %1, %2, %3};\n\t"
        "@pu add.u32 %4, %4, %9;\n\t"
        "@pd mad.lo.u32 %3, nv, %7, 0;\n\t"
        "@pd mad.lo.u32 %0, nC, %7, 0;\n\t"
        "@pd mad.lo.u32 %1, nl, %7, 0;\n\t"
        "@pd mad.lo.u32 %2, nr, %7, 0;\n\t"
        "or.pred po, pd, pa;\n\t"
        "not.pred po, po;\n\t"
        "and.pred po, po, pk;\n\t"
        "@po sub.u32 %4, %4, %9;\n\t"
        "@po ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n\t"
        "}"
        : "+r"(C), "+r"(l), "+r"(r), "+r"(a), "+r"(sp), "+r"(sol), "+r"(its)
        : "r"(one), "r"(two), "n"(STRIDE)
        : "memory");
  } else {
    asm volatile(
        "{\n\t"
        ".reg .u32 na, p, nC, t, nl, nr, nv, a2;\n\t"
        ".reg .pred pd, pa, pu, po, ps, pk;\n\t"
        "neg.s32 na, %3;\n\t"
        "and.b32 p, %3, na;\n\t"
        "setp.ne.u32 pk, p, 0;\n\t"
        "xor.b32 a2, %3, p;\n\t"
        "setp.ne.u32 pa, a2, 0;\n\t"
        "sub.u32 nC, %0, p;\n\t"
        "add.u32 t, %1, p;\n\t"
        "mul.lo.u32 nl, t, %8;\n\t"
        "add.u32 t, %2, p;\n\t"
        "mul.hi.u32 nr, t, 0x80000000;\n\t"
        "lop3.b32 nv, nC, nl, nr, 0x10;\n\t"
        "setp.ne.u32 pd, nv, 0;\n\t"
        "mad.hi.u32 %6, na, %8, %6;\n\t"
        "setp.eq.u32 ps, nC, 0;\n\t"
        "@ps add.u32 %5, %5, 1;\n\t"
        "and.pred pu, pd, pa;\n\t"
        "@pu st.shared.v4.u32 [%4], {%0, %1, %2, a2};\n\t"
        "@pu add.u32 %4, %4, %9;\n\t"
        "selp.b32 %3, nv, a2, pd;\n\t"
        "selp.b32 %0, nC, %0, pd;\n\t"
        "@pd mad.lo.u32 %1, nl, %7, 0;\n\t"
        "@pd mad.lo.u32 %2, nr, %7, 0;\n\t"
        "or.pred po, pd, pa;\n\t"
        "not.pred po, po;\n\t"
        "and.pred po, po, pk;\n\t"
        "@po sub.u32 %4, %4, %9;\n\t"
        "@po ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n\t"
        "}"
        : "+r"(C), "+r"(l), "+r"(r), "+r"(a), "+r"(sp), "+r"(sol), "+r"(its)
        : "r"(one), "r"(two), "n"(STRIDE)
        : "memory");
  }
}


// Variant AD ("always descend"): the child state replaces the current one
// unconditionally; a row with untried candidates left is pushed first; a dead child
// (no candidates) pops. A dead child with siblings left therefore costs an STS+LDS
// round trip instead of four selects. Predicates come free from the LOP3 outputs
// except the idle guard on the pop.
template <uint32_t STRIDE>
__device__ __forceinline__ void ad_step(uint32_t& C, uint32_t& l, uint32_t& r, uint32_t& a,
                                        uint32_t& sp, uint32_t& sol, uint32_t& its) {
  asm volatile(
      "{\n\t"
      ".reg .u32 na, p;\n\t"
      ".reg .pred pa, pk, po, ps;\n\t"
      "neg.s32 na, %3;\n\t"
      "and.b32 p, %3, na;\n\t"
      "setp.ne.u32 pk, p, 0;\n\t"
      "xor.b32 %3, %3, p;\n\t"
      "setp.ne.u32 pa, %3, 0;\n\t"
      "@pa st.shared.v4.u32 [%4], {%0, %1, %2, %3};\n\t"
      "@pa add.u32 %4, %4, %7;\n\t"
      "sub.u32 %0, %0, p;\n\t"
      "add.u32 %1, %1, p;\n\t"
      "add.u32 %1, %1, %1;\n\t"
      "add.u32 %2, %2, p;\n\t"
      "shr.u32 %2, %2, 1;\n\t"
      "lop3.b32 %3, %0, %1, %2, 0x10;\n\t"
      "shr.u32 na, na, 31;\n\t"
      "add.u32 %6, %6, na;\n\t"
      "setp.eq.and.u32 ps, %0, 0, pk;\n\t"
      "@ps add.u32 %5, %5, 1;\n\t"
      "setp.eq.and.u32 po, %3, 0, pk;\n\t"
      "@po sub.u32 %4, %4, %7;\n\t"
      "@po ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n\t"
      "}"
      : "+r"(C), "+r"(l), "+r"(r), "+r"(a), "+r"(sp), "+r"(sol), "+r"(its)
      : "n"(STRIDE)
      : "memory");
}

// Variant AD32: same step, frame split into four 32-bit planes (plane w of level L of
// thread t at word (4L + w)*BLOCK + t): every lane owns one bank in every plane, so any
// set of active lanes is one wavefront per LDS.32/STS.32 (zero bank conflicts).
template <uint32_t STRIDE>
__device__ __forceinline__ void ad32_step(uint32_t& C, uint32_t& l, uint32_t& r, uint32_t& a,
                                          uint32_t& sp, uint32_t& sol, uint32_t& its) {
  constexpr uint32_t P = STRIDE / 4;  // bytes between planes
  asm volatile(
      "{\n\t"
      ".reg .u32 na, p;\n\t"
      ".reg .pred pa, pk, po, ps;\n\t"
      "neg.s32 na, %3;\n\t"
      "and.b32 p, %3, na;\n\t"
      "setp.ne.u32 pk, p, 0;\n\t"
      "xor.b32 %3, %3, p;\n\t"
      "setp.ne.u32 pa, %3, 0;\n\t"
      "@pa st.shared.u32 [%4], %0;\n\t"
      "@pa st.shared.u32 [%4+%8], %1;\n\t"
      "@pa st.shared.u32 [%4+%9], %2;\n\t"
      "@pa st.shared.u32 [%4+%10], %3;\n\t"
      "@pa add.u32 %4, %4, %7;\n\t"
      "sub.u32 %0, %0, p;\n\t"
      "add.u32 %1, %1, p;\n\t"
      "add.u32 %1, %1, %1;\n\t"
      "add.u32 %2, %2, p;\n\t"
      "shr.u32 %2, %2, 1;\n\t"
      "lop3.b32 %3, %0, %1, %2, 0x10;\n\t"
      "shr.u32 na, na, 31;\n\t"
      "add.u32 %6, %6, na;\n\t"
      "setp.eq.and.u32 ps, %0, 0, pk;\n\t"
      "@ps add.u32 %5, %5, 1;\n\t"
      "setp.eq.and.u32 po, %3, 0, pk;\n\t"
      "@po sub.u32 %4, %4, %7;\n\t"
      "@po ld.shared.u32 %0, [%4];\n\t"
      "@po ld.shared.u32 %1, [%4+%8];\n\t"
      "@po ld.shared.u32 %2, [%4+%9];\n\t"
      "@po ld.shared.u32 %3, [%4+%10];\n\t"
      "}"
      : "+r"(C), "+r"(l), "+r"(r), "+r"(a), "+r"(sp), "+r"(sol), "+r"(its)
      : "n"(STRIDE), "n"(P), "n"(2 * P), "n"(3 * P)
      : "memory");
}

// Variant S ("descend or stay", stays kept in registers like the first product kernel)
// with the pop predicate folded into one compare: a2 < p <=> (a2 == 0 && p != 0), since
// a2 only holds candidates above p. MODE 6: two commits on the FMA pipe (IMAD by a
// runtime 1), two as SEL; MODE 7: four SELs.
template <uint32_t STRIDE, int MODE>
__device__ __forceinline__ void s_step(uint32_t& C, uint32_t& l, uint32_t& r, uint32_t& a,
                                       uint32_t& sp, uint32_t& sol, uint32_t& its, uint32_t one) {
#define S_HEAD                                   \
  "{\n\t"                                        \
  ".reg .u32 na, p, a2, nC, t, nl, nr, nv;\n\t"  \
  ".reg .pred pa, pk, pd, pu, po, ps;\n\t"       \
  "neg.s32 na, %3;\n\t"                          \
  "and.b32 p, %3, na;\n\t"                       \
  "setp.ne.u32 pk, p, 0;\n\t"                    \
  "xor.b32 a2, %3, p;\n\t"                       \
  "setp.ne.u32 pa, a2, 0;\n\t"                   \
  "sub.u32 nC, %0, p;\n\t"                       \
  "add.u32 t, %1, p;\n\t"                        \
  "add.u32 nl, t, t;\n\t"                        \
  "add.u32 t, %2, p;\n\t"                        \
  "shr.u32 nr, t, 1;\n\t"                        \
  "lop3.b32 nv, nC, nl, nr, 0x10;\n\t"           \
  "setp.ne.u32 pd, nv, 0;\n\t"                   \
  "shr.u32 na, na, 31;\n\t"                      \
  "add.u32 %6, %6, na;\n\t"                      \
  "setp.eq.and.u32 ps, nC, 0, pk;\n\t"           \
  "@ps add.u32 %5, %5, 1;\n\t"                   \
  "and.pred pu, pd, pa;\n\t"                     \
  "@pu st.shared.v4.u32 [%4], {%0, %1, %2, a2};\n\t" \
  "@pu add.u32 %4, %4, %8;\n\t"                  \
  "setp.lt.and.u32 po, a2, p, !pd;\n\t"
#define S_TAIL                                   \
  "@po sub.u32 %4, %4, %8;\n\t"                  \
  "@po ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n\t" \
  "}"
  if constexpr (MODE == 6) {
    asm volatile(S_HEAD
                 "selp.b32 %3, nv, a2, pd;\n\t"
                 "@pd mad.lo.u32 %0, nC, %7, 0;\n\t"
                 "@pd mad.lo.u32 %1, nl, %7, 0;\n\t"
                 "selp.b32 %2, nr, %2, pd;\n\t" S_TAIL
                 : "+r"(C), "+r"(l), "+r"(r), "+r"(a), "+r"(sp), "+r"(sol), "+r"(its)
                 : "r"(one), "n"(STRIDE)
                 : "memory");
  } else {
    asm volatile(S_HEAD
                 "selp.b32 %3, nv, a2, pd;\n\t"
                 "selp.b32 %0, nC, %0, pd;\n\t"
                 "selp.b32 %1, nl, %1, pd;\n\t"
                 "selp.b32 %2, nr, %2, pd;\n\t" S_TAIL
                 : "+r"(C), "+r"(l), "+r"(r), "+r"(a), "+r"(sp), "+r"(sol), "+r"(its)
                 : "r"(one), "n"(STRIDE)
                 : "memory");
  }
#undef S_HEAD
#undef S_TAIL
}

// Variant ADP: always-descend with one-row lookahead pruning. A row's candidates are
// filtered to those whose child row is non-empty: with V1 = C & ~((l<<1)|(r>>1)) the
// child of candidate p is V1 & ~(p | p<<1 | p>>1), so p is dead iff V1 fits in the
// 3-column window around p — only the lowest bit of V1 and its neighbours can qualify.
// Dead placements are counted (popc) without a step; at the last row every placement
// is "dead" and is a solution. Steps drop to ~0.63 per node and so does stack traffic.
__device__ __forceinline__ void adp_prune(uint32_t C, uint32_t l, uint32_t r, uint32_t& a,
                                          uint32_t& sol, uint32_t& its) {
  const uint32_t v = C & ~(l | r);
  const uint32_t V1 = C & ~((l << 1) | (r >> 1));
  uint32_t W = 0xffffffffu;
  if (V1) {
    const uint32_t lo = V1 & (0u - V1);
    W = 0;
    if ((V1 & ~(lo * 7u)) == 0) W += lo << 1;
    if ((V1 & ~(lo * 3u)) == 0) W += lo;
    if (V1 == lo) W += lo >> 1;
  }
  const uint32_t dead = v & W;
  a = v & ~W;
  its += __popc(dead);
  if (C && (C & (C - 1u)) == 0u) sol += __popc(dead);
}

template <uint32_t STRIDE>
__device__ __forceinline__ void adp_step(uint32_t& C, uint32_t& l, uint32_t& r, uint32_t& a,
                                         uint32_t& sp, uint32_t& sol, uint32_t& its) {
  asm volatile(
      "{\n\t"
      ".reg .u32 na, p, v, l1, r1, V1, lo, m, W, t, dead, pc;\n\t"
      ".reg .pred pa, pk, po, pz, c7, c3, c1, pl;\n\t"
      "neg.s32 na, %3;\n\t"
      "and.b32 p, %3, na;\n\t"
      "setp.ne.u32 pk, p, 0;\n\t"
      "xor.b32 %3, %3, p;\n\t"
      "setp.ne.u32 pa, %3, 0;\n\t"
      "@pa st.shared.v4.u32 [%4], {%0, %1, %2, %3};\n\t"
      "@pa add.u32 %4, %4, %7;\n\t"
      "sub.u32 %0, %0, p;\n\t"
      "add.u32 %1, %1, p;\n\t"
      "add.u32 %1, %1, %1;\n\t"
      "add.u32 %2, %2, p;\n\t"
      "shr.u32 %2, %2, 1;\n\t"
      "lop3.b32 v, %0, %1, %2, 0x10;\n\t"
      "add.u32 l1, %1, %1;\n\t"
      "shr.u32 r1, %2, 1;\n\t"
      "lop3.b32 V1, %0, l1, r1, 0x10;\n\t"
      "setp.eq.u32 pz, V1, 0;\n\t"
      "neg.s32 t, V1;\n\t"
      "and.b32 lo, V1, t;\n\t"
      "mul.lo.u32 m, lo, 7;\n\t"
      "lop3.b32 t, V1, m, 0, 0x30;\n\t"
      "setp.eq.u32 c7, t, 0;\n\t"
      "mul.lo.u32 m, lo, 3;\n\t"
      "lop3.b32 t, V1, m, 0, 0x30;\n\t"
      "setp.eq.u32 c3, t, 0;\n\t"
      "setp.eq.u32 c1, V1, lo;\n\t"
      "mov.b32 W, 0;\n\t"
      "@c7 add.u32 W, lo, lo;\n\t"
      "@c3 add.u32 W, W, lo;\n\t"
      "shr.u32 t, lo, 1;\n\t"
      "@c1 add.u32 W, W, t;\n\t"
      "@pz mov.b32 W, -1;\n\t"
      "and.b32 dead, v, W;\n\t"
      "lop3.b32 %3, v, W, 0, 0x30;\n\t"
      "popc.b32 pc, dead;\n\t"
      "shr.u32 na, na, 31;\n\t"
      "add.u32 %6, %6, na;\n\t"
      "add.u32 %6, %6, pc;\n\t"
      "sub.u32 t, %0, 1;\n\t"
      "and.b32 t, %0, t;\n\t"
      "setp.eq.u32 pl, t, 0;\n\t"
      "@pl add.u32 %5, %5, pc;\n\t"
      "setp.eq.and.u32 po, %3, 0, pk;\n\t"
      "@po sub.u32 %4, %4, %7;\n\t"
      "@po ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n\t"
      "}"
      : "+r"(C), "+r"(l), "+r"(r), "+r"(a), "+r"(sp), "+r"(sol), "+r"(its)
      : "n"(STRIDE)
      : "memory");
}

// Variant ADZ: always-descend plus the cheapest lookahead: entering a row whose
// next-row mask V1 = C & ~((l<<1)|(r>>1)) is empty means every candidate of the row has
// an empty child — count them all (popc) and pop at once instead of one step each.
// Not applied on the last row (there the placements are solutions, counted by sol).
template <uint32_t STRIDE>
__device__ __forceinline__ void adz_step(uint32_t& C, uint32_t& l, uint32_t& r, uint32_t& a,
                                         uint32_t& sp, uint32_t& sol, uint32_t& its) {
  asm volatile(
      "{\n\t"
      ".reg .u32 na, p, l1, r1, V1, t, pc;\n\t"
      ".reg .pred pa, pk, po, ps, pz, pn, pp;\n\t"
      "neg.s32 na, %3;\n\t"
      "and.b32 p, %3, na;\n\t"
      "setp.ne.u32 pk, p, 0;\n\t"
      "xor.b32 %3, %3, p;\n\t"
      "setp.ne.u32 pa, %3, 0;\n\t"
      "@pa st.shared.v4.u32 [%4], {%0, %1, %2, %3};\n\t"
      "@pa add.u32 %4, %4, %7;\n\t"
      "sub.u32 %0, %0, p;\n\t"
      "add.u32 %1, %1, p;\n\t"
      "add.u32 %1, %1, %1;\n\t"
      "add.u32 %2, %2, p;\n\t"
      "shr.u32 %2, %2, 1;\n\t"
      "lop3.b32 %3, %0, %1, %2, 0x10;\n\t"
      "shr.u32 na, na, 31;\n\t"
      "add.u32 %6, %6, na;\n\t"
      "setp.eq.and.u32 ps, %0, 0, pk;\n\t"
      "@ps add.u32 %5, %5, 1;\n\t"
      "add.u32 l1, %1, %1;\n\t"
      "shr.u32 r1, %2, 1;\n\t"
      "lop3.b32 V1, %0, l1, r1, 0x10;\n\t"
      "setp.eq.u32 pz, V1, 0;\n\t"
      "sub.u32 t, %0, 1;\n\t"
      "and.b32 t, %0, t;\n\t"
      "setp.ne.and.u32 pp, t, 0, pz;\n\t"
      "@pp popc.b32 pc, %3;\n\t"
      "@pp add.u32 %6, %6, pc;\n\t"
      "@pp mov.b32 %3, 0;\n\t"
      "setp.eq.and.u32 po, %3, 0, pk;\n\t"
      "@po sub.u32 %4, %4, %7;\n\t"
      "@po ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n\t"
      "}"
      : "+r"(C), "+r"(l), "+r"(r), "+r"(a), "+r"(sp), "+r"(sol), "+r"(its)
      : "n"(STRIDE)
      : "memory");
}

struct LabParams {
  DfsParams P;
  uint32_t one, two;
  unsigned long long* lane_steps;
};

template <int BLOCK, int KSTEP, int MODE>
__global__ void __launch_bounds__(BLOCK) lab_kernel(LabParams LP) {
  const DfsParams& P = LP.P;
  extern __shared__ uint4 stk[];
  constexpr uint32_t STRIDE = BLOCK * 16u;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t base0 = static_cast<uint32_t>(__cvta_generic_to_shared(stk)) +
                        threadIdx.x * (MODE == 5 ? 4u : 16u);
  const uint32_t base1 = base0 + STRIDE;
  constexpr uint32_t IDLE_C = MODE >= 4 ? 0u : kIdleC;  // AD: no free column when idle
  if constexpr (MODE == 5) {
    for (int w = 0; w < 4; ++w)
      asm volatile("st.shared.u32 [%0], %1;" ::"r"(base0 + w * (STRIDE / 4)), "r"(w == 1 ? kIdleL : (w == 0 ? IDLE_C : 0u)) : "memory");
  } else {
    sts128(base0, IDLE_C, kIdleL, 0u, 0u);
  }
  uint32_t C = IDLE_C, l = kIdleL, r = 0u, a = 0u, sp = base1, sol = 0u, its = 0u, weight = 0u;
  const uint32_t one = LP.one, two = LP.two;
  bool busy = false, exhausted = false;
  unsigned long long tot_w = 0, tot_raw = 0, tot_it = 0, tot_subs = 0, steps = 0;
  uint32_t blocks = 0;
  for (;;) {
    uint32_t idle = __ballot_sync(0xffffffffu, a == 0u);
    if (idle) {
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
            const unsigned long long idx = P.reverse ? (P.count - 1ull - pos) : pos;
            const uint4 s = __ldg(&P.subs[idx]);
            busy = true;
            weight = s.w >> 8;
            if ((s.x | 0u) == P.mask) {
              sol = 1u;
            } else {
              C = P.mask & ~s.x;
              l = s.y;
              r = s.z;
              a = C & ~(l | r);
              if constexpr (MODE == 8) adp_prune(C, l, r, a, sol, its);
              if constexpr (MODE == 9) {  // the same zero-V1 rule at the root row
                const uint32_t V1 = C & ~((l << 1) | (r >> 1));
                if (V1 == 0u && (C & (C - 1u)) != 0u) {
                  its += __popc(a);
                  a = 0u;
                }
              }
              sp = base1;
            }
            if (a == 0u) {
              C = IDLE_C;
              l = kIdleL;
              r = 0u;
            }
          }
        }
      }
      if (exhausted && __all_sync(0xffffffffu, a == 0u)) break;
    }
#pragma unroll
    for (int k = 0; k < KSTEP; ++k) {
      if constexpr (MODE == 9) adz_step<STRIDE>(C, l, r, a, sp, sol, its);
      else if constexpr (MODE == 8) adp_step<STRIDE>(C, l, r, a, sp, sol, its);
      else if constexpr (MODE >= 6) s_step<STRIDE, MODE>(C, l, r, a, sp, sol, its, one);
      else if constexpr (MODE == 5) ad32_step<STRIDE>(C, l, r, a, sp, sol, its);
      else if constexpr (MODE >= 4) ad_step<STRIDE>(C, l, r, a, sp, sol, its);
      else lab_step<STRIDE, MODE>(C, l, r, a, sp, sol, its, one, two);
    }
    steps += KSTEP;
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
    steps += __shfl_down_sync(0xffffffffu, steps, off);
  }
  if (lane == 0u) {
    atomicAdd(P.totals + 0, tot_w);
    atomicAdd(P.totals + 1, tot_raw);
    atomicAdd(P.totals + 2, tot_it);
    atomicAdd(P.totals + 3, tot_subs);
    atomicAdd(LP.lane_steps, steps);
  }
}

// ---------------------------------------------------------------------------------------
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
void run(const Bed& b, const char* name, void (*kern)(PT), int block, int reps) {
  const int levels = b.n - 1 - b.R + 1;
  const size_t smem = size_t(levels) * block * 16;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, smem));
  LabParams LP{};
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
  LP.one = 1;
  LP.two = 2;
  LP.lane_steps = b.d_ctl + 7;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  unsigned long long h[8];
  for (int i = 0; i < reps; ++i) {
    CK(cudaMemset(b.d_ctl, 0, 8 * sizeof(unsigned long long)));
    cudaEventRecord(e0);
    if constexpr (sizeof(PT) == sizeof(LabParams)) kern<<<per_sm * b.sms, block, smem>>>(LP);
    else kern<<<per_sm * b.sms, block, smem>>>(*reinterpret_cast<PT*>(&LP.P));
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
              "\"lane_eff\": %.4f, \"nodes_per_s\": %.4e, \"nodes_per_sm_clk\": %.3f}\n",
              name, b.n, b.R, block, per_sm, best, ok ? "true" : "false", h[1], nodes,
              h[7] ? double(h[3]) / double(h[7]) : 0.0, nodes / (best * 1e-3),
              nodes / (best * 1e-3) / (b.sms * 1.965e9));
  std::fflush(stdout);
}

int main(int argc, char** argv) {
  Bed b{};
  b.n = argc > 1 ? std::atoi(argv[1]) : 18;
  b.R = argc > 2 ? std::atoi(argv[2]) : 6;
  const int reps = argc > 3 ? std::atoi(argv[3]) : 3;
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
  const int only = argc > 4 ? std::atoi(argv[4]) : -1;
  int idx = 0;
  auto pick = [&](auto&&... xs) { if (only < 0 || only == idx) run(b, xs...); ++idx; };
  pick("P prod v4", nq_dfs_kernel<128, 32, false, kLayoutV4>, 128, reps);
  pick("P prod planes", nq_dfs_kernel<128, 32, false, kLayoutPlanes>, 128, reps);
  pick("AD k8", lab_kernel<128, 8, 4>, 128, reps);
  pick("AD k32", lab_kernel<128, 32, 4>, 128, reps);

  pick("ADP k32", lab_kernel<128, 32, 8>, 128, reps);
  pick("ADZ k32", lab_kernel<128, 32, 9>, 128, reps);
  return 0;
}
