// nqueens/subproblems.hpp — the folded subproblem frontier of the drop-in API
// (reference subproblems.hpp:20-178).
//
// The stream (order, symmetry fold, multipliers) is produced by the library's
// multi-threaded C++ generator (paper_2511_12009_b200/csrc/nq_frontier.cpp) as packed
// 16-byte nq_sub records; this header converts them to the reference's 20-byte
// Subproblem where a caller wants that type. for_each_subproblem streams the frontier in
// bounded chunks, so a 453,688,251-record N=27/R=7 frontier never has to be
// materialised as Subproblems.
#pragma once

#include <cstdint>
#include <cstdio>
#include <optional>
#include <ostream>
#include <set>
#include <span>
#include <string>
#include <tuple>
#include <utility>
#include <unordered_set>
#include <vector>

#include "nqueens/bitboard.hpp"
#include "nqueens/errors.hpp"
#include "nqueens/gpu.hpp"
#include "nqueens/solver.hpp"

namespace nqueens {

struct GenerationPlan {
    int n = 8;
    int pre_rows = 2;
    std::optional<std::uint64_t> expected_total = std::nullopt;
};

/// Q(27), the paper's multi-week result (subproblems.hpp:28); a log-comparison constant.
inline constexpr std::uint64_t kQueens27Reference = 234907967154122528ull;

namespace detail {

/// subproblems.hpp:32-39: same checks and messages (the generator re-checks them).
inline void check_plan(const GenerationPlan& plan) {
    check_board(plan.n);
    if (plan.pre_rows < 1 || plan.pre_rows >= plan.n)
        throw config_error("pre_rows must satisfy 1 <= R < n (n=" + std::to_string(plan.n) +
                           ", R=" + std::to_string(plan.pre_rows) + ")");
    if (plan.pre_rows > 8) throw config_error("pre_rows above 8 is not supported");
}

inline Subproblem unpack(const nq_sub& s) {
    return Subproblem{s.cols, s.diag, s.antidiag, static_cast<int>(s.row & 0xffu),
                      static_cast<int>(s.row >> 8)};
}

/// Records [first, first + count) of the folded stream, packed.
inline std::vector<nq_sub> generate_range(const GenerationPlan& plan, std::uint64_t first,
                                          std::uint64_t count) {
    std::vector<nq_sub> out(count);
    std::uint64_t total = 0;
    gpu::check(nq_generate_slice(plan.n, plan.pre_rows, 1, first, out.data(), count, &total));
    out.resize(total < count ? total : count);
    return out;
}

inline constexpr std::uint64_t kStreamChunk = std::uint64_t{1} << 22;  // 4 Mi records, 64 MiB

}  // namespace detail

/// Length of the folded stream without materialising it (subproblems.hpp:118-145).
inline std::uint64_t count_subproblems(int n, int pre_rows) {
    detail::check_plan(GenerationPlan{n, pre_rows});
    std::uint64_t total = 0;
    gpu::check(nq_count_subproblems(n, pre_rows, &total));
    return total;
}

/// The whole folded frontier as packed 16-byte records (the device input format).
inline std::vector<nq_sub> generate_packed(const GenerationPlan& plan) {
    detail::check_plan(plan);
    const std::uint64_t total = count_subproblems(plan.n, plan.pre_rows);
    return detail::generate_range(plan, 0, total);
}

/// Calls sink(Subproblem) for every record of the folded stream, in the reference's
/// deterministic order (subproblems.hpp:80-108), generating it chunk by chunk.
template <typename Sink>
void for_each_subproblem(const GenerationPlan& plan, Sink&& sink) {
    detail::check_plan(plan);
    const std::uint64_t total = count_subproblems(plan.n, plan.pre_rows);
    for (std::uint64_t first = 0; first < total; first += detail::kStreamChunk) {
        const std::uint64_t len =
            total - first < detail::kStreamChunk ? total - first : detail::kStreamChunk;
        for (const nq_sub& s : detail::generate_range(plan, first, len)) sink(detail::unpack(s));
    }
}

/// The folded frontier as the reference's 20-byte structs (subproblems.hpp:110-115).
inline std::vector<Subproblem> generate(const GenerationPlan& plan) {
    const std::vector<nq_sub> packed = generate_packed(plan);
    std::vector<Subproblem> out;
    out.reserve(packed.size());
    for (const nq_sub& s : packed) out.push_back(detail::unpack(s));
    return out;
}

namespace detail {
/// The reference's duplicate key (subproblems.hpp:154-157): (cur, left, right,
/// placed_rows) folded into 64 bits by multiply-xor with the golden-ratio constant.
/// Keying the same 64-bit value keeps the reference's behaviour exactly, including
/// which inputs it reports as duplicates.
inline std::uint64_t state_key(const Subproblem& s) {
    constexpr std::uint64_t kGolden = 0x9e3779b97f4a7c15ull;
    std::uint64_t key = s.cur;
    for (std::uint64_t part : {static_cast<std::uint64_t>(s.left), static_cast<std::uint64_t>(s.right),
                               static_cast<std::uint64_t>(s.placed_rows)})
        key = key * kGolden ^ part;
    return key;
}
}  // namespace detail

/// Σ multiplier × count with checked arithmetic; a state whose key appears twice is a
/// config_error (subproblems.hpp:149-165).
inline std::uint64_t aggregate(std::span<const std::pair<Subproblem, std::uint64_t>> results) {
    std::unordered_set<std::uint64_t> seen;
    seen.reserve(results.size());
    std::uint64_t total = 0;
    for (const auto& [sub, count] : results) {
        if (!seen.insert(detail::state_key(sub)).second)
            throw config_error("duplicate subproblem in aggregation input");
        total = checked_add(total, checked_mul(static_cast<std::uint64_t>(sub.multiplier), count));
    }
    return total;
}

/// Text export, one record per line: "index cur left right placed_rows multiplier"
/// with the three masks in lowercase hex (subproblems.hpp:169-178). Returns the count.
inline std::uint64_t write_batch(std::ostream& out, const GenerationPlan& plan) {
    std::uint64_t index = 0;
    char line[96];
    for_each_subproblem(plan, [&](const Subproblem& s) {
        std::snprintf(line, sizeof line, "%llu %x %x %x %d %d\n",
                      static_cast<unsigned long long>(index), s.cur, s.left, s.right,
                      s.placed_rows, s.multiplier);
        out << line;
        ++index;
    });
    return index;
}

}  // namespace nqueens
