// nq_frontier.cpp — host frontier generator (product code).
//
// Produces the reference's folded subproblem stream (for_each_subproblem,
// subproblems.hpp:80-108: first-row half board ×2, odd-N centre column with the
// second row folded to columns 0..c-2 ×2, centre root ×1 when R == 1) in the SAME
// deterministic order, but packed into 16-byte nq_sub records and generated in
// parallel:
//
//   1. enumerate "prefixes" — the folded partial boards at depth d0 = min(R, 3) — in
//      stream order (a few thousand of them);
//   2. count each prefix's descendants at depth R with a popcount at the last level
//      (the count_rows walk of subproblems.hpp:58-71) on all host threads;
//   3. exclusive-scan the counts into output offsets;
//   4. expand every prefix into its own slice of the output on all host threads.
//
// Offsets are exact, so the result is byte-identical to a sequential walk whatever
// the thread count. A systematic slice (index ≡ offset mod stride) of the same stream
// is produced the same way without materialising the skipped records, which is how
// the N=27 projection samples a 453,688,251-record frontier.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "nq_gpu.h"
#include "nq_internal.h"

namespace nqb200 {
namespace {

struct Prefix {
  uint32_t cols, diag, anti;
  int row;
  int mult;
};

inline uint32_t mask_of(int n) { return n >= 32 ? 0xffffffffu : ((1u << n) - 1u); }

// All placements of `row`, as in expand_rows' loop (subproblems.hpp:48-54).
template <class F>
inline void for_each_bit(uint32_t v, F&& f) {
  while (v) {
    const uint32_t p = v & (0u - v);
    v ^= p;
    f(p);
  }
}

struct Walker {
  int n;
  uint32_t mask;

  // Number of depth-`target` descendants of a row-`row` state (subproblems.hpp:58-71).
  uint64_t count(uint32_t cols, uint32_t diag, uint32_t anti, int row, int target) const {
    if (row == target) return 1;
    const uint32_t v = mask & ~(cols | diag | anti);
    if (row == target - 1) return static_cast<uint64_t>(__builtin_popcount(v));
    uint64_t s = 0;
    for_each_bit(v, [&](uint32_t p) {
      s += count(cols | p, (diag | p) << 1, (anti | p) >> 1, row + 1, target);
    });
    return s;
  }

  // Emit descendants at depth `target` in stream order; `index` is the stream position
  // of the next record. Records with (index - offset) % stride == 0 are written to
  // out[(index - offset) / stride] when that slot is below cap.
  void emit(uint32_t cols, uint32_t diag, uint32_t anti, int row, int target, int mult,
            uint64_t& index, uint64_t stride, uint64_t offset, nq_sub* out, uint64_t cap) const {
    if (row == target) {
      if (index >= offset && (index - offset) % stride == 0) {
        const uint64_t slot = (index - offset) / stride;
        if (slot < cap)
          out[slot] = nq_sub{cols, diag, anti,
                             static_cast<uint32_t>(target) | (static_cast<uint32_t>(mult) << 8)};
      }
      ++index;
      return;
    }
    const uint32_t v = mask & ~(cols | diag | anti);
    for_each_bit(v, [&](uint32_t p) {
      emit(cols | p, (diag | p) << 1, (anti | p) >> 1, row + 1, target, mult, index, stride,
           offset, out, cap);
    });
  }

  // Folded prefixes at depth d0 (>= 2 when the centre branch is expanded), in order.
  void prefixes(int d0, int target, std::vector<Prefix>& out) const {
    auto rec = [&](auto&& self, uint32_t c, uint32_t d, uint32_t a, int row, int mult) -> void {
      if (row == d0) {
        out.push_back(Prefix{c, d, a, row, mult});
        return;
      }
      for_each_bit(mask & ~(c | d | a), [&](uint32_t p) {
        self(self, c | p, (d | p) << 1, (a | p) >> 1, row + 1, mult);
      });
    };
    for (int c = 0; c < n / 2; ++c) {
      const uint32_t p = 1u << c;
      rec(rec, p, p << 1, p >> 1, 1, 2);
    }
    if (n % 2 == 1) {
      const int c = (n - 1) / 2;
      const uint32_t p = 1u << c;
      const uint32_t cols = p, diag = p << 1, anti = p >> 1;
      if (target == 1) {
        out.push_back(Prefix{cols, diag, anti, 1, 1});
      } else {
        const uint32_t left_half = c >= 1 ? (1u << (c - 1)) - 1u : 0u;
        for_each_bit((mask & ~(cols | diag | anti)) & left_half, [&](uint32_t q) {
          rec(rec, cols | q, (diag | q) << 1, (anti | q) >> 1, 2, 2);
        });
      }
    }
  }
};

template <class F>
void parallel_for(size_t items, F&& f) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const unsigned nt = static_cast<unsigned>(std::min<size_t>(hw, std::max<size_t>(items / 4, 1)));
  if (nt <= 1) {
    for (size_t i = 0; i < items; ++i) f(i);
    return;
  }
  std::atomic<size_t> next{0};
  std::vector<std::thread> ts;
  ts.reserve(nt);
  for (unsigned t = 0; t < nt; ++t)
    ts.emplace_back([&] {
      for (size_t i; (i = next.fetch_add(1, std::memory_order_relaxed)) < items;) f(i);
    });
  for (auto& t : ts) t.join();
}

}  // namespace

// check_plan (subproblems.hpp:32-39) with the reference's messages.
int check_plan(int n, int pre_rows) {
  if (n < 1 || n > 32)
    return set_error(NQ_ECONFIG, "board size must be in [1, 32], got " + std::to_string(n));
  if (pre_rows < 1 || pre_rows >= n)
    return set_error(NQ_ECONFIG, "pre_rows must satisfy 1 <= R < n (n=" + std::to_string(n) +
                                     ", R=" + std::to_string(pre_rows) + ")");
  if (pre_rows > 8) return set_error(NQ_ECONFIG, "pre_rows above 8 is not supported");
  return NQ_OK;
}

struct FrontierStream::Impl {
  Walker w;
  int pre_rows;
  std::vector<Prefix> pre;
  std::vector<uint64_t> off;  // off[i]: stream index of prefix i's first descendant
};

FrontierStream::FrontierStream() = default;
FrontierStream::~FrontierStream() = default;

int FrontierStream::open(int n, int pre_rows) {
  if (int rc = check_plan(n, pre_rows)) return rc;
  auto p = std::make_unique<Impl>(Impl{Walker{n, mask_of(n)}, pre_rows, {}, {}});
  p->w.prefixes(std::min(pre_rows, 3), pre_rows, p->pre);
  p->off.assign(p->pre.size() + 1, 0);
  parallel_for(p->pre.size(), [&](size_t i) {
    const Prefix& q = p->pre[i];
    p->off[i + 1] = p->w.count(q.cols, q.diag, q.anti, q.row, pre_rows);
  });
  for (size_t i = 0; i < p->pre.size(); ++i) p->off[i + 1] += p->off[i];
  impl_ = std::move(p);
  return NQ_OK;
}

uint64_t FrontierStream::size() const { return impl_ ? impl_->off.back() : 0; }

int FrontierStream::emit(uint64_t stride, uint64_t offset, nq_sub* out, uint64_t cap) const {
  if (!impl_) return set_error(NQ_ECONFIG, "frontier stream not opened");
  if (stride == 0) return set_error(NQ_ECONFIG, "slice stride must be >= 1");
  const Impl& p = *impl_;
  if (!out || cap == 0) return NQ_OK;
  // Prefixes whose range holds no slot in [0, cap) are skipped: a contiguous range
  // [offset, offset + cap) (stride 1) touches only the prefixes that overlap it.
  const uint64_t end_index = offset + (cap - 1) * stride;  // last wanted stream index
  const size_t lo_i = static_cast<size_t>(
      std::upper_bound(p.off.begin(), p.off.end() - 1, offset) - p.off.begin()) - 1;
  const size_t hi_i = static_cast<size_t>(
      std::upper_bound(p.off.begin(), p.off.end() - 1, end_index) - p.off.begin());
  parallel_for(hi_i - lo_i, [&](size_t k) {
    const size_t i = lo_i + k;
    const uint64_t lo = p.off[i], hi = p.off[i + 1];
    if (hi <= offset || lo == hi) return;
    const uint64_t first_slot = lo > offset ? (lo - offset + stride - 1) / stride : 0;
    if (first_slot >= cap) return;
    uint64_t index = lo;
    p.w.emit(p.pre[i].cols, p.pre[i].diag, p.pre[i].anti, p.pre[i].row, p.pre_rows, p.pre[i].mult,
             index, stride, offset, out, cap);
  });
  return NQ_OK;
}

int generate_slice(int n, int pre_rows, uint64_t stride, uint64_t offset, nq_sub* out,
                   uint64_t cap, uint64_t* total) {
  if (int rc = check_plan(n, pre_rows)) return rc;
  NvtxRange range(out ? "nq_generate" : "nq_count_subproblems");
  if (stride == 0) return set_error(NQ_ECONFIG, "slice stride must be >= 1");
  FrontierStream fs;
  if (int rc = fs.open(n, pre_rows)) return rc;
  const uint64_t full = fs.size();
  const uint64_t sliced = full > offset ? (full - offset + stride - 1) / stride : 0;
  if (total) *total = sliced;
  return fs.emit(stride, offset, out, std::min(cap, sliced));
}

// Deepen a list of roots to `target` placed rows: each root's descendants at depth
// target in DFS order (lowest column first, as expand_rows, subproblems.hpp:41-55),
// roots in input order, multiplier inherited. A root already at depth >= target is
// copied as-is. Used to cut very deep frontiers (N=27 slices) into GPU-sized records.
int expand(int n, const nq_sub* roots, uint64_t count, int target, nq_sub* out, uint64_t cap,
           uint64_t* total) {
  if (n < 1 || n > 32)
    return set_error(NQ_ECONFIG, "board size must be in [1, 32], got " + std::to_string(n));
  if (target < 1 || target >= n)
    return set_error(NQ_ECONFIG, "target rows must satisfy 1 <= T < n (n=" + std::to_string(n) +
                                     ", T=" + std::to_string(target) + ")");
  if (count && !roots) return set_error(NQ_ECONFIG, "null roots");
  const Walker w{n, mask_of(n)};
  for (uint64_t i = 0; i < count; ++i) {
    const nq_sub& s = roots[i];
    const int placed = static_cast<int>(s.row & 0xffu);
    if ((s.cols & ~w.mask) != 0u || __builtin_popcount(s.cols) != placed)
      return set_error(NQ_ECONFIG, "root " + std::to_string(i) + " is malformed");
  }
  std::vector<uint64_t> off(count + 1, 0);
  parallel_for(count, [&](size_t i) {
    const nq_sub& s = roots[i];
    const int placed = static_cast<int>(s.row & 0xffu);
    off[i + 1] = placed >= target ? 1 : w.count(s.cols, s.diag, s.antidiag, placed, target);
  });
  for (uint64_t i = 0; i < count; ++i) off[i + 1] += off[i];
  if (total) *total = off[count];
  if (!out || cap == 0) return NQ_OK;
  parallel_for(count, [&](size_t i) {
    if (off[i] >= cap) return;
    const nq_sub& s = roots[i];
    const int placed = static_cast<int>(s.row & 0xffu);
    if (placed >= target) {
      out[off[i]] = s;
      return;
    }
    uint64_t index = off[i];
    w.emit(s.cols, s.diag, s.antidiag, placed, target, static_cast<int>(s.row >> 8), index, 1, 0,
           out, cap);
  });
  return NQ_OK;
}

int count_subproblems(int n, int pre_rows, uint64_t* total) {
  return generate_slice(n, pre_rows, 1, 0, nullptr, 0, total);
}

}  // namespace nqb200

extern "C" int nq_generate(int n, int pre_rows, nq_sub* out, uint64_t cap, uint64_t* total) {
  return nqb200::generate_slice(n, pre_rows, 1, 0, out, cap, total);
}

extern "C" int nq_generate_slice(int n, int pre_rows, uint64_t stride, uint64_t offset,
                                 nq_sub* out, uint64_t cap, uint64_t* total) {
  return nqb200::generate_slice(n, pre_rows, stride, offset, out, cap, total);
}

extern "C" int nq_expand(int n, const nq_sub* roots, uint64_t count, int target_rows, nq_sub* out,
                         uint64_t cap, uint64_t* total) {
  return nqb200::expand(n, roots, count, target_rows, out, cap, total);
}

extern "C" int nq_count_subproblems(int n, int pre_rows, uint64_t* total) {
  return nqb200::count_subproblems(n, pre_rows, total);
}
