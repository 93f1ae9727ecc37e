// nqueens/runner.hpp — checkpointed runs of the drop-in API (reference runner.hpp:20-212),
// backed by the chunk-granular GPU checkpoint (nq_solve_checkpointed).
//
// Same RunSpec / CheckpointOptions / run_with_checkpoint signature and the same
// validation (stealing refused, n == 1 short-circuit). What differs underneath: progress
// is recorded per chunk of `flush_interval` records (the reference records per-worker
// high-water indices every flush_interval subproblems), and the file is this library's
// format (identity hash + chunk list + checksum), not the reference's.
#pragma once

#include <atomic>
#include <cstdint>
#include <filesystem>
#include <functional>
#include <string>

#include "nqueens/errors.hpp"
#include "nqueens/scheduler.hpp"

namespace nqueens {

struct RunSpec {
    int n = 8;
    int pre_rows = 2;
    StackConfig config = builtin_configs[1];
    KernelVariant kernel = KernelVariant::lastrow;
    PartitionPlan plan;
};

struct CheckpointOptions {
    std::filesystem::path path;
    std::uint64_t flush_interval = 1'000'000;  ///< records per recorded chunk
    bool resume = false;
};

/// Checkpointed count (runner.hpp:48-212): a cancel leaves completed == false and a
/// file that a later call with resume = true continues.
inline SolveReport run_with_checkpoint(const RunSpec& spec, const CheckpointOptions& ckpt,
                                       const std::atomic<bool>* cancel = nullptr,
                                       std::function<void(const std::string&)> log = {}) {
    if (spec.plan.strategy == PartitionStrategy::stealing)
        throw config_error("checkpointing requires a contiguous partition (uniform/weighted)");
    detail::check_board(spec.n);
    ExecuteOptions opts;
    opts.kernel = spec.kernel;
    opts.config = spec.config;
    opts.plan = spec.plan;
    opts.cancel = cancel;
    opts.log = log;
    if (spec.n == 1) return execute(1, 0, opts);
    if (ckpt.flush_interval == 0) throw config_error("flush_interval must be >= 1");
    SolveReport r = execute_checkpointed(spec.n, spec.pre_rows, opts, ckpt.path.string(),
                                         ckpt.flush_interval, 0.0, ckpt.resume);
    if (r.completed && log) log(log_result_line(spec.n, r.total, r.calc_ms));
    return r;
}

}  // namespace nqueens
