// nqueens/solver.hpp — per-subproblem counting entry points of the drop-in API
// (reference solver.hpp:18-197), backed by the sm_100a DFS kernel.
//
// Each call ships one 16-byte record to the device through nq_count_each (the
// count_with seam batched onto the GPU) and returns the count and the Alg. 2 / Alg. 3
// stack high-water mark. These calls exist for API compatibility and testing; bulk
// counting goes through execute_batch/execute (scheduler.hpp), which launch one
// persistent kernel per chunk instead of one per subproblem.
#pragma once

#include <cstdint>
#include <string>

#include "nqueens/bitboard.hpp"
#include "nqueens/errors.hpp"
#include "nqueens/gpu.hpp"
#include "nqueens/stack_config.hpp"

namespace nqueens {

/// One subtree root (solver.hpp:18-26): rows 0..placed_rows-1 are fixed, left/right
/// are already shifted to row placed_rows; multiplier is the symmetry weight.
struct Subproblem {
    bit_mask cur = 0;
    bit_mask left = 0;
    bit_mask right = 0;
    int placed_rows = 0;
    int multiplier = 2;

    friend bool operator==(const Subproblem&, const Subproblem&) = default;
};

enum class KernelVariant { iterative, lastrow };

inline const char* to_string(KernelVariant v) {
    switch (v) {
        case KernelVariant::iterative: return "iterative";
        case KernelVariant::lastrow: break;
    }
    return "lastrow";
}

struct KernelResult {
    std::uint64_t count = 0;  ///< completions of the subproblem, multiplier not applied
    int high_water = 0;       ///< deepest frame the reference's loop would occupy
};

namespace detail {

inline void check_board(int n) {
    if (n >= 1 && n <= kMaxBoard) return;
    throw config_error("board size must be in [1, 32], got " + std::to_string(n));
}

inline nq_sub pack(const Subproblem& s) {
    return nq_sub{s.cur, s.left, s.right, gpu::pack_row(s.placed_rows, s.multiplier)};
}

inline KernelResult count_one(KernelVariant v, int n, const Subproblem& sub) {
    const nq_sub rec = pack(sub);
    std::uint64_t count = 0, nodes = 0;
    std::int32_t high = 0;
    const int pre = sub.placed_rows < n ? sub.placed_rows : n;
    gpu::check(nq_count_each(gpu::context(), n, pre,
                             v == KernelVariant::lastrow ? NQ_VARIANT_LASTROW : NQ_VARIANT_ITERATIVE,
                             &rec, 1, &count, &high, &nodes));
    return KernelResult{count, high};
}

}  // namespace detail

/// Alg. 1 count (solver.hpp:69-72); the multiplier is not applied.
inline std::uint64_t count_recursive(int n, const Subproblem& sub) {
    detail::check_board(n);
    return detail::count_one(KernelVariant::iterative, n, sub).count;
}

/// Alg. 2 semantics (solver.hpp:79-130): count plus the n - R frame high-water mark.
inline KernelResult count_iterative(int n, const Subproblem& sub, const StackConfig& cfg) {
    detail::check_board(n);
    require_feasible(cfg, n, sub.placed_rows, false);
    return detail::count_one(KernelVariant::iterative, n, sub);
}

/// Alg. 3 semantics (solver.hpp:138-191): the last row is settled by a popcount, so
/// the high-water mark is at most n - R - 1.
inline KernelResult count_iterative_lastrow(int n, const Subproblem& sub, const StackConfig& cfg) {
    detail::check_board(n);
    require_feasible(cfg, n, sub.placed_rows, true);
    return detail::count_one(KernelVariant::lastrow, n, sub);
}

inline KernelResult count_with(KernelVariant variant, int n, const Subproblem& sub,
                               const StackConfig& cfg) {
    if (variant == KernelVariant::iterative) return count_iterative(n, sub, cfg);
    return count_iterative_lastrow(n, sub, cfg);
}

}  // namespace nqueens
