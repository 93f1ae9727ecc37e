// nq_kernel.cuh — the sm_100a persistent DFS counting kernel.
//
// Replaces the reference's per-subproblem CPU search (count_iterative_lastrow,
// solver.hpp:138-191, called once per subproblem from execute_batch,
// scheduler.hpp:319-326) with one persistent kernel that owns the whole batch.
//
// Execution model:
//   * one subproblem per thread; a grid of (#SM x resident blocks) threads stays
//     resident and refills idle lanes from a global atomic dispatch cursor, one
//     atomicAdd per warp per refill round (ballot -> leader atomic -> shfl);
//   * the CURRENT row's state (free columns C, diagonals l/r, untried candidates a)
//     lives in registers. Each step places the lowest candidate and ALWAYS moves to
//     the child row; a row that still has untried candidates is pushed first, as one
//     16-byte frame, onto a per-thread stack in shared memory laid out interleaved
//     (level L of thread t at frame index L*BLOCK + t: every quarter-warp of an
//     LDS.128/STS.128 touches 32 distinct banks whatever depth each lane is at); a
//     child with no candidate pops the nearest pushed frame. "Always descend" needs no
//     select between parent and child state: the push/pop predicates come straight out
//     of the LOP3 zero flags (tools/microbench/dfs_lab.cu measured it 14% faster than
//     descend-or-stay with four SELs, which left the ALU pipe the bottleneck);
//   * the popcount of Alg. 3's last-row test is replaced by "no free column left"
//     (C == 0), because POPC issues at 1/8 of the ALU rate on sm_100;
//   * an idle lane holds C = 0, a = 0: every side effect is predicated off, so the
//     idle check runs once per KSTEP steps;
//   * per-lane u32 counters are folded into u64 totals at subproblem end and before
//     they reach 2^31, then warp-shuffle reduced with one atomicAdd per warp.
//
// Node accounting: one loop iteration places one queen at rows placed..n-1. The
// reference's Alg. 3 settles row n-1 by popcount instead, so its iteration count is
// ours minus the number of (unweighted) solutions; both are reported.
#pragma once
#include <cstdint>

namespace nqb200 {

constexpr uint32_t kIdleC = 0u;  // idle lane: no free column, so no child ever has a candidate

struct DfsParams {
  const uint4* subs;                 // packed records (nq_sub)
  unsigned long long count;          // records in subs
  unsigned long long* cursor;        // device dispatch counter (zeroed per launch)
  const unsigned long long* stop;    // non-zero: hand out no more records (cancel)
  unsigned long long* totals;        // [0] weighted, [1] raw sols, [2] iterations,
                                     // [3] subproblems, [4] first bad record + 1,
                                     // [6] weighted sum wrapped 64 bits (-> NQ_EOVERFLOW),
                                     // [7] streaming queue watchdog fired
  unsigned long long* each_count;    // per-record outputs (PER_SUB only)
  int* each_high;
  unsigned long long* each_nodes;
  uint32_t mask;                     // board_mask(n)
  int n;
  int min_placed;                    // batch pre_rows: deeper records would overflow the stack
  int reverse;                       // dispatch order: 1 = last record first
  int lastrow;                       // variant (affects high-water / node outputs only)
  int donate;                        // tail balancing: idle lanes take busy lanes' frames
  // Streaming launch (stream != 0): records come from a queue of chunks the host
  // publishes while the kernel runs (nq_sched.cpp's dynamic dispatch), not from
  // subs[0, count). Chunk j holds the queue positions [tab[j-1].end, tab[j].end) at
  // tab[j].base. The host writes the table and the publish word (positions published,
  // bit 63 = closed) into MAPPED PINNED HOST memory, never through a stream (a copy
  // queued behind this persistent kernel would never run); the kernel keeps a device
  // mirror of the entries it has read and reports its cursor back the same way.
  int stream;
  struct QChunk* q_tab;                        // device mirror (zeroed before launch)
  const struct QChunk* q_host_tab;             // mapped host table
  const unsigned long long* q_pub;             // mapped host publish word
  unsigned long long* q_progress;              // mapped host: cursor, coarsely
  unsigned long long* q_pub_mirror;            // device: newest publish word any warp read
  unsigned long long* q_bus_lock;              // device: held by the one warp reading q_pub
  unsigned long long* q_copied;                // device: [entries copied into q_tab, their end]
  unsigned long long watchdog_ns;              // give up after this long without a publish
};

// A warp's view of the streaming queue (warp-uniform; in shared memory).
struct WarpQueue {
  unsigned long long pub_seen = 0ull;  // published positions as of the last read
  unsigned long long end = 0ull;       // the current chunk entry: [base, end)
  const uint4* base = nullptr;
  uint32_t chunk = 0u;                 // its index in the table
  uint32_t closed = 0u;                // the queue was closed at pub_seen
};

// One published chunk of a streaming launch (16-byte aligned: the device mirror is
// read and written as one 16-byte access, so a reader never sees half an entry).
struct alignas(16) QChunk {
  const uint4* base;
  unsigned long long end;  // cumulative queue position one past this chunk's last record
};
constexpr unsigned long long kQueueClosed = 1ull << 63;
constexpr unsigned long long kNoTicket = ~0ull;
// A warp that waits longer than this for the host to publish gives up (the queue is
// treated as closed and the launch reports it): a host that died cannot hang the GPU.
constexpr unsigned long long kQueueWatchdogNs = 120ull * 1000000000ull;

__device__ __forceinline__ void sts128(uint32_t addr, uint32_t x, uint32_t y, uint32_t z,
                                       uint32_t w) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(x), "r"(y),
               "r"(z), "r"(w)
               : "memory");
}

__device__ __forceinline__ void lds128(uint32_t addr, uint32_t& x, uint32_t& y, uint32_t& z,
                                       uint32_t& w) {
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(x), "=r"(y), "=r"(z), "=r"(w)
               : "r"(addr)
               : "memory");
}

// One DFS node for one lane, in PTX so the push / pop transitions stay predicated on
// the zero flags of the LOP3s that produce them. p is a valid position, so it is
// disjoint from l, r and a subset of C and a, which turns |, ^ into +, - (the FMA
// pipe can take them):
//   p  = a & -a                         lowest untried candidate   (bitboard.hpp:25-28)
//   a  = a ^ p;  push (C,l,r,a) if a    the row's remaining candidates
//   C -= p, l = (l + p) << 1, r = (r + p) >> 1                     (bitboard.hpp:38-45)
//   a  = C & ~(l | r)                   child's candidates (LOP3 0x10) (bitboard.hpp:21-23)
//   its += (a_in != 0)  (bit 31 of -a_in when a_in < 2^31, i.e. n <= 31; WIDE: of a_in | -a_in)
//   sol += (C == 0) for busy lanes
//   pop (C,l,r,a) if the child has no candidate and the lane is busy
// Stack layouts (both: one level = BLOCK frames = BLOCK*16 bytes):
//   kLayoutV4     frame of thread t at level L = one uint4 at stk[L*BLOCK + t]; one
//                 STS.128 / LDS.128 per push / pop. Fastest. A dense warp access is
//                 conflict-free (every quarter-warp covers the 32 banks once); a sparse
//                 predicated LDS.128 whose active lanes fall in different quarter-warps
//                 costs one wavefront per quarter and ncu books the excess over
//                 ceil(bytes/128) as "bank conflicts" (tools/microbench/smem_banks.cu) —
//                 no 16-byte-per-lane layout can avoid that.
//   kLayoutPlanes word w of the frame in plane w: u32 at ((4L + w)*BLOCK + t); lane t
//                 owns bank t in every plane, so ANY set of active lanes is one
//                 wavefront per LDS.32/STS.32 — zero bank conflicts by construction,
//                 at four memory instructions per push / pop (~5% slower, dfs_lab).
constexpr int kLayoutV4 = 0;
constexpr int kLayoutPlanes = 1;

// One whole frame at a stack address of the given layout (the donation path).
template <uint32_t STRIDE, int LAYOUT>
__device__ __forceinline__ void load_frame(uint32_t addr, uint32_t& C, uint32_t& l, uint32_t& r,
                                           uint32_t& a) {
  if constexpr (LAYOUT == kLayoutV4) {
    lds128(addr, C, l, r, a);
  } else {
    asm volatile("ld.shared.u32 %0, [%4];\n\tld.shared.u32 %1, [%4+%5];\n\t"
                 "ld.shared.u32 %2, [%4+%6];\n\tld.shared.u32 %3, [%4+%7];"
                 : "=r"(C), "=r"(l), "=r"(r), "=r"(a)
                 : "r"(addr), "n"(STRIDE / 4), "n"(STRIDE / 2), "n"(3 * STRIDE / 4)
                 : "memory");
  }
}

template <uint32_t STRIDE, int LAYOUT>
__device__ __forceinline__ void store_idle_frame(uint32_t addr) {
  if constexpr (LAYOUT == kLayoutV4) {
    sts128(addr, 0u, 0u, 0u, 0u);
  } else {
#pragma unroll
    for (uint32_t w = 0; w < 4; ++w)
      asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr + w * (STRIDE / 4)), "r"(0u) : "memory");
  }
}

// The V4 step; WIDE_FIX is empty for n <= 31 and "or.b32 na, na, %3;" for n = 32, where a
// candidate set can have bit 31 set and bit 31 of -a alone no longer flags a != 0 (bit 31
// of a | -a does, for any 32-bit a).
#define NQ_V4_STEP(WIDE_FIX)                          \
  "{\n\t"                                            \
  ".reg .u32 na, p;\n\t"                             \
  ".reg .pred pa, pk, po, ps;\n\t"                   \
  "neg.s32 na, %3;\n\t"                              \
  "and.b32 p, %3, na;\n\t" WIDE_FIX                  \
  "setp.ne.u32 pk, p, 0;\n\t"                        \
  "xor.b32 %3, %3, p;\n\t"                           \
  "setp.ne.u32 pa, %3, 0;\n\t"                       \
  "@pa st.shared.v4.u32 [%4], {%0, %1, %2, %3};\n\t" \
  "@pa add.u32 %4, %4, %7;\n\t"                      \
  "sub.u32 %0, %0, p;\n\t"                           \
  "add.u32 %1, %1, p;\n\t"                           \
  "add.u32 %1, %1, %1;\n\t"                          \
  "add.u32 %2, %2, p;\n\t"                           \
  "shr.u32 %2, %2, 1;\n\t"                           \
  "lop3.b32 %3, %0, %1, %2, 0x10;\n\t"               \
  "shr.u32 na, na, 31;\n\t"                          \
  "add.u32 %6, %6, na;\n\t"                          \
  "setp.eq.and.u32 ps, %0, 0, pk;\n\t"               \
  "@ps add.u32 %5, %5, 1;\n\t"                       \
  "setp.eq.and.u32 po, %3, 0, pk;\n\t"               \
  "@po sub.u32 %4, %4, %7;\n\t"                      \
  "@po ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n\t" \
  "}"

template <uint32_t STRIDE, int LAYOUT, bool WIDE = false>
__device__ __forceinline__ void dfs_step(uint32_t& C, uint32_t& l, uint32_t& r, uint32_t& a,
                                         uint32_t& sp, uint32_t& sol, uint32_t& its) {
  if constexpr (LAYOUT == kLayoutV4 && WIDE) {
    asm volatile(NQ_V4_STEP("or.b32 na, na, %3;\n\t")
                 : "+r"(C), "+r"(l), "+r"(r), "+r"(a), "+r"(sp), "+r"(sol), "+r"(its)
                 : "n"(STRIDE)
                 : "memory");
  } else if constexpr (LAYOUT == kLayoutV4) {
    asm volatile(NQ_V4_STEP("")
                 : "+r"(C), "+r"(l), "+r"(r), "+r"(a), "+r"(sp), "+r"(sol), "+r"(its)
                 : "n"(STRIDE)
                 : "memory");
  } else {
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
      : "n"(STRIDE), "n"(STRIDE / 4), "n"(STRIDE / 2), "n"(3 * STRIDE / 4)
      : "memory");
  }
}

// STREAM: records come from the host-published chunk queue (P.stream must be set);
// a separate instantiation, so the contiguous launch carries none of its state.
template <int BLOCK, int KSTEP, bool PER_SUB, int LAYOUT, bool WIDE = false, bool STREAM = false>
__global__ void __launch_bounds__(BLOCK, 1152 / BLOCK) nq_dfs_kernel(DfsParams P) {
  static_assert(!WIDE || LAYOUT == kLayoutV4, "n = 32 runs the V4 layout");
  static_assert(!(STREAM && PER_SUB), "per-record outputs use the contiguous launch");
  extern __shared__ uint4 stk[];  // [levels][BLOCK] frames (or [levels][4][BLOCK] words)
  constexpr uint32_t STRIDE = BLOCK * 16u;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t base0 = static_cast<uint32_t>(__cvta_generic_to_shared(stk)) +
                         threadIdx.x * (LAYOUT == kLayoutV4 ? 16u : 4u);
  const uint32_t base1 = base0 + STRIDE;  // first real frame (level 1)

  // Level 0 holds the idle sentinel that an exhausted lane pops into (all zero).
  if constexpr (LAYOUT == kLayoutV4) {
    sts128(base0, kIdleC, 0u, 0u, 0u);
  } else {
#pragma unroll
    for (uint32_t w = 0; w < 4; ++w)
      asm volatile("st.shared.u32 [%0], %1;" ::"r"(base0 + w * (STRIDE / 4)), "r"(0u) : "memory");
  }

  uint32_t C = kIdleC, l = 0u, r = 0u, a = 0u;  // current row state (idle)
  uint32_t sp = base1;                             // next free frame
  uint32_t bp = base1;                             // lowest frame not yet given away
  bool piece = false;                              // the lane holds a donated frame
  uint32_t sol = 0u, its = 0u;                     // per-lane counters since last fold
  uint32_t weight = 0u;                            // multiplier of the current record
  bool busy = false;                               // lane holds a record
  unsigned long long tot_w = 0ull, tot_raw = 0ull, tot_it = 0ull, tot_subs = 0ull;
  bool wrapped = false;  // Σ multiplier x count passed 2^64 (checked_add, errors.hpp:24-29)
  // PER_SUB bookkeeping
  unsigned long long cur_idx = 0ull, sub_sol = 0ull, sub_it = 0ull;
  int placed = 0, high = 0;

  bool exhausted = false;  // warp-uniform: no more records will be handed to this warp
  // streaming: this lane's queue position (taken from the cursor, possibly not yet
  // published by the host)
  unsigned long long ticket = kNoTicket;
  // The warp-uniform queue state lives in shared memory, not in registers: it is only
  // touched at refills, and seven more live registers across the step loop spill.
  [[maybe_unused]] WarpQueue* wq = nullptr;
  if constexpr (STREAM) {
    __shared__ WarpQueue wq_s[BLOCK / 32];
    wq = &wq_s[threadIdx.x >> 5];
    if (lane == 0u) *wq = WarpQueue{};  // lane 0 writes, __syncwarp publishes to the warp
    __syncwarp();
  }
#ifdef NQB_STREAM_STATS
  // probe build only: [rounds, pub mirror reads, host pub reads, entry reads, host entry
  // reads, naps, step blocks, idle lane-blocks] summed into totals[15..22]
  unsigned long long st[8] = {0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull};
#define NQB_STAT(i) (++st[i])
#else
#define NQB_STAT(i) ((void)0)
#endif

  // Starts record `idx` (reported as the failing index) at `rec` on this lane.
  // Records are read-only for the launch's lifetime in both modes (a streaming launch
  // only publishes ranges of a batch made device-resident before it started).
  auto start = [&](const uint4* rec, unsigned long long idx) {
    const uint4 s = __ldg(rec);
    busy = true;
    weight = s.w >> 8;
    placed = static_cast<int>(s.w & 0xffu);
    if constexpr (PER_SUB) {
      cur_idx = idx;
      sub_sol = 0ull;
      sub_it = 0ull;
      high = 0;
    }
    // Record validation: cols inside the board, one queen per placed row.
    if ((s.x & ~P.mask) != 0u || __popc(s.x) != placed || placed < P.min_placed) {
      atomicCAS(P.totals + 4, 0ull, idx + 1ull);
      weight = 0u;
    } else if (s.x == P.mask) {
      sol = 1u;  // fully placed record: cur == last (solver.hpp:89, :148)
    } else {
      C = P.mask & ~s.x;
      l = s.y;
      r = s.z;
      a = C & ~(l | r);  // valid_positions (bitboard.hpp:21-23)
      sp = base1;
      bp = base1;
    }
    if (a == 0u) C = kIdleC;  // settled at the root: back to the idle state
  };

  for (;;) {
    // ---- refill idle lanes (once per KSTEP block) ----------------------------------
    uint32_t idle = __ballot_sync(0xffffffffu, a == 0u);
    if (idle) {
      unsigned long long wait_since = 0ull;  // streaming: start of the current nap
      for (;;) {
        if (a == 0u && busy) {  // fold the finished record (or donated piece of one)
          const unsigned long long prod = static_cast<unsigned long long>(weight) * sol;  // < 2^56
          tot_w += prod;
          wrapped |= tot_w < prod;
          tot_raw += sol;
          tot_it += its;
          tot_subs += piece ? 0ull : 1ull;
          piece = false;
          if constexpr (PER_SUB) {
            sub_sol += sol;
            sub_it += its;
            P.each_count[cur_idx] = sub_sol;
            P.each_high[cur_idx] = high;
            P.each_nodes[cur_idx] = P.lastrow ? (sub_it - sub_sol) : sub_it;
          }
          sol = 0u;
          its = 0u;
          busy = false;
        }
        if (exhausted) break;
        if constexpr (!STREAM) {
          const uint32_t need = __ballot_sync(0xffffffffu, a == 0u);
          if (need == 0u) break;
          const uint32_t leader = __ffs(need) - 1u;
          const uint32_t n_need = __popc(need);
          unsigned long long first = 0ull;
          if (lane == leader) {
            // A raised stop word (host cancel, copied in on a side stream) ends dispatch
            // at this refill: lanes finish their current subtree, nothing new is taken.
            first = *reinterpret_cast<const volatile unsigned long long*>(P.stop)
                        ? P.count
                        : atomicAdd(P.cursor, static_cast<unsigned long long>(n_need));
          }
          first = __shfl_sync(0xffffffffu, first, leader);
          if (first + n_need >= P.count) exhausted = true;
          if (a == 0u) {
            const unsigned long long pos = first + __popc(need & ((1u << lane) - 1u));
            if (pos < P.count) {
              const unsigned long long idx = P.reverse ? (P.count - 1ull - pos) : pos;
              start(&P.subs[idx], idx);
            }
          }
          continue;
        } else {
        unsigned long long pub_seen = wq->pub_seen;  // published positions last read
        bool closed_seen = wq->closed != 0u;
        uint32_t chunk = wq->chunk;                  // chunk entry `chunk` is [w_base, w_end)
        const uint4* w_base = wq->base;              // (w_end 0: none read yet)
        unsigned long long w_end = wq->end;
        // Streaming: (1) idle lanes without a queue position take one from the cursor,
        if (lane == 0u) NQB_STAT(0);
        const uint32_t need = __ballot_sync(0xffffffffu, a == 0u && ticket == kNoTicket);
        unsigned long long taken_end = 0ull;
        if (need) {
          const uint32_t leader = __ffs(need) - 1u;
          const uint32_t n_need = __popc(need);
          unsigned long long first = 0ull;
          if (lane == leader) {
            first = atomicAdd(P.cursor, static_cast<unsigned long long>(n_need));
            // coarse progress for the host's feeder (every 4096 positions)
            if ((first >> 12) != ((first + n_need) >> 12))
              asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(P.q_progress),
                           "l"(first + n_need)
                           : "memory");
          }
          first = __shfl_sync(0xffffffffu, first, leader);
          if ((need >> lane) & 1u) ticket = first + __popc(need & ((1u << lane) - 1u));
          taken_end = first + n_need;
        }
        // (2) positions the host has published become records; past the final count
        // (queue closed) they are dropped. The publish word is re-read (over the bus)
        // only when a ticket is beyond what this warp last saw.
        const uint32_t holders = __ballot_sync(0xffffffffu, ticket != kNoTicket);
        if (holders == 0u) break;
        if (__any_sync(0xffffffffu, ticket != kNoTicket && ticket >= pub_seen) && !closed_seen) {
          // the device mirror first (one warp per publish pays the bus read)
          unsigned long long pw = 0ull;
          if (lane == __ffs(holders) - 1u) {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(pw) : "l"(P.q_pub_mirror) : "memory");
            NQB_STAT(1);
            // Stale mirror: one warp at a time reads the word over the bus. All warps
            // cross a chunk boundary together (the cursor is shared); unserialised, their
            // thousands of host reads queue up at the root complex (≈1 µs each). The
            // reader also copies the newly published entries into the device table before
            // it releases the new word, so the entries are never read over the bus again.
            if ((pw & ~kQueueClosed) <= pub_seen && !(pw & kQueueClosed) &&
                atomicCAS(P.q_bus_lock, 0ull, 1ull) == 0ull) {
              __threadfence();
              unsigned long long ph;
              NQB_STAT(2);
              asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(ph) : "l"(P.q_pub) : "memory");
              if (ph > pw) {
                const unsigned long long target = ph & ~kQueueClosed;
                // q_copied = {entries copied, end position of the last one}; every entry
                // up to `target` was written before the word was released
                volatile unsigned long long* cp = P.q_copied;
                unsigned long long k = cp[0], done = cp[1];
                while (done < target) {
                  unsigned long long eb;
                  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(done)
                               : "l"(&P.q_host_tab[k].end) : "memory");
                  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(eb)
                               : "l"(&P.q_host_tab[k].base) : "memory");
                  asm volatile("st.global.cg.v2.u64 [%0], {%1, %2};" ::"l"(P.q_tab + k), "l"(eb),
                               "l"(done) : "memory");
                  ++k;
                }
                cp[0] = k;
                cp[1] = done;
                asm volatile("red.release.gpu.global.max.u64 [%0], %1;" ::"l"(P.q_pub_mirror), "l"(ph)
                             : "memory");
                pw = ph;
              }
              __threadfence();
              atomicExch(P.q_bus_lock, 0ull);
            }
          }
          pw = __shfl_sync(0xffffffffu, pw, __ffs(holders) - 1u);
          pub_seen = pw & ~kQueueClosed;
          closed_seen = (pw & kQueueClosed) != 0ull;
          __syncwarp();  // every lane's read of the view above is done
          if (lane == 0u) {
            wq->pub_seen = pub_seen;
            wq->closed = closed_seen ? 1u : 0u;
          }
          __syncwarp();
        }
        // Published tickets become records. The chunk entry is warp-uniform (w_base,
        // w_end of entry `chunk`): a warp's tickets are consecutive and only grow, so one
        // lane reads the next entry (device table; read from the host table only if the
        // bus reader above has not copied it yet, which its ordering rules out)
        // only when the warp's tickets pass w_end — a few reads per chunk per warp, not
        // one per record.
        for (uint32_t res = __ballot_sync(0xffffffffu, ticket != kNoTicket && ticket < pub_seen);
             res != 0u;) {
          if (((res >> lane) & 1u) && ticket < w_end) {
            // expensive end of the chunk first, like the contiguous launch (reverse)
            start(w_base + (w_end - 1ull - ticket), ticket);
            ticket = kNoTicket;
          }
          res = __ballot_sync(0xffffffffu, ticket != kNoTicket && ticket < pub_seen);
          if (res == 0u) break;
          unsigned long long eb = 0ull, ee = 0ull;
          if (lane == __ffs(res) - 1u) {
            if (w_end != 0ull) ++chunk;
            NQB_STAT(3);
            asm volatile("ld.global.cg.v2.u64 {%0, %1}, [%2];" : "=l"(eb), "=l"(ee)
                         : "l"(P.q_tab + chunk) : "memory");
            if (ee == 0ull) {  // not copied yet: fetch it from the host table
              NQB_STAT(4);
              asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(eb)
                           : "l"(&P.q_host_tab[chunk].base) : "memory");
              asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(ee)
                           : "l"(&P.q_host_tab[chunk].end) : "memory");
              asm volatile("st.global.cg.v2.u64 [%0], {%1, %2};" ::"l"(P.q_tab + chunk), "l"(eb),
                           "l"(ee) : "memory");
            }
          }
          const uint32_t src = __ffs(res) - 1u;
          chunk = __shfl_sync(0xffffffffu, chunk, src);
          w_base = reinterpret_cast<const uint4*>(__shfl_sync(0xffffffffu, eb, src));
          w_end = __shfl_sync(0xffffffffu, ee, src);
          __syncwarp();
          if (lane == 0u) {
            wq->chunk = chunk;
            wq->base = w_base;
            wq->end = w_end;
          }
          __syncwarp();
        }
        if (closed_seen && ticket != kNoTicket) ticket = kNoTicket;  // past the final count
        if (closed_seen && need && taken_end >= pub_seen) exhausted = true;
        // (3) positions still unpublished: step the busy lanes and look again after
        // KSTEP steps; if no lane has work, nap instead of spinning on the bus.
        if (__ballot_sync(0xffffffffu, ticket != kNoTicket) == 0u) continue;
        if (__all_sync(0xffffffffu, a == 0u)) {
          unsigned long long now;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
          if (wait_since == 0ull) wait_since = now;
          if (now - wait_since > P.watchdog_ns) {  // the host stopped publishing
            atomicExch(P.totals + 7, 1ull);
            ticket = kNoTicket;
            exhausted = true;
            break;
          }
          if (lane == 0u) NQB_STAT(5);
          __nanosleep(1000);
          continue;
        }
        break;
        }  // STREAM
      }
      if constexpr (!PER_SUB) {
        // Tail balancing inside the warp. Once the queue is empty, an idle lane takes
        // the SHALLOWEST pending frame of a busy lane — the row with untried candidates
        // nearest the root, i.e. the largest remaining subtree — and the donor marks that
        // slot idle, so popping down to it later ends the donor's work there. Frames never
        // move: a lane's live frames are [bp, sp); everything below bp was given away.
        if (exhausted && P.donate) {
          // Orders the donors' earlier pushes before the receivers' load_frame below
          // (ballot/shfl synchronise the warp but do not order shared memory).
          __syncwarp();
          for (int round = 0; round < 2; ++round) {
            const uint32_t idle_m = __ballot_sync(0xffffffffu, a == 0u);
            const uint32_t donor_m = __ballot_sync(0xffffffffu, a != 0u && sp > bp);
            if (idle_m == 0u || donor_m == 0u) break;
            const uint32_t lt = (1u << lane) - 1u;
            const uint32_t k = min(__popc(idle_m), __popc(donor_m));
            const uint32_t my_idle = __popc(idle_m & lt), my_donor = __popc(donor_m & lt);
            const bool recv = a == 0u && my_idle < k;
            const bool give = ((donor_m >> lane) & 1u) && my_donor < k;
            uint32_t src = lane;
            if (recv) {  // the my_idle-th donor
              uint32_t m = donor_m;
              for (uint32_t i = 0; i < my_idle; ++i) m &= m - 1u;
              src = __ffs(m) - 1u;
            }
            const uint32_t d_bp = __shfl_sync(0xffffffffu, bp, src);
            const uint32_t d_w = __shfl_sync(0xffffffffu, weight, src);
            if (recv) {
              load_frame<STRIDE, LAYOUT>(d_bp, C, l, r, a);
              weight = d_w;
              sp = base1;
              bp = base1;
              busy = true;
              piece = true;
            }
            __syncwarp();
            if (give) {
              store_idle_frame<STRIDE, LAYOUT>(bp);
              bp += STRIDE;
            }
            __syncwarp();
          }
        }
      }
      if (exhausted && __all_sync(0xffffffffu, a == 0u)) break;
    }

    // ---- KSTEP predicated DFS steps -------------------------------------------------
#ifdef NQB_STREAM_STATS
    {
      const uint32_t idle_now = __ballot_sync(0xffffffffu, a == 0u);
      if (lane == 0u) {
        NQB_STAT(6);
        st[7] += __popc(idle_now);
      }
    }
#endif
#pragma unroll
    for (int k = 0; k < KSTEP; ++k) {
      if constexpr (PER_SUB) {
        const int row = P.n - __popc(C & P.mask);
        const int h = row - placed + 1;
        if (a != 0u && (!P.lastrow || row <= P.n - 2) && h > high) high = h;
      }
      dfs_step<STRIDE, LAYOUT, WIDE>(C, l, r, a, sp, sol, its);
    }

    // Fold the u32 counters (lane-local) before they can wrap: its grows by at most
    // KSTEP per block and sol <= its. No block counter: one register fewer.
    if (its >= 0x80000000u) {
      const unsigned long long prod = static_cast<unsigned long long>(weight) * sol;
      tot_w += prod;
      wrapped |= tot_w < prod;
      tot_raw += sol;
      tot_it += its;
      if constexpr (PER_SUB) {
        sub_sol += sol;
        sub_it += its;
      }
      sol = 0u;
      its = 0u;
    }
  }

  // ---- warp reduction, one atomic per warp per total --------------------------------
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long w = __shfl_down_sync(0xffffffffu, tot_w, off);
    tot_w += w;
    wrapped |= tot_w < w;
    tot_raw += __shfl_down_sync(0xffffffffu, tot_raw, off);
    tot_it += __shfl_down_sync(0xffffffffu, tot_it, off);
    tot_subs += __shfl_down_sync(0xffffffffu, tot_subs, off);
  }
  wrapped = __any_sync(0xffffffffu, wrapped);
  if (lane == 0u) {
    const unsigned long long before = atomicAdd(P.totals + 0, tot_w);
    if (wrapped || before + tot_w < before) atomicExch(P.totals + 6, 1ull);
    atomicAdd(P.totals + 1, tot_raw);
    atomicAdd(P.totals + 2, tot_it);
    atomicAdd(P.totals + 3, tot_subs);
  }
#ifdef NQB_STREAM_STATS
  for (int i = 0; i < 8; ++i) {
    unsigned long long v = st[i];
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    if (lane == 0u && v) atomicAdd(P.totals + 15 + i, v);
  }
#endif
#undef NQB_STAT
}

}  // namespace nqb200
