// nqueens/scheduler.hpp — execute / execute_batch of the drop-in API (reference
// scheduler.hpp:26-423), backed by the multi-GPU chunk scheduler of libnqb200.so.
//
// Same types, defaults, validation order, error messages, log lines and report
// fields as the reference. What changes underneath: a "worker" is a host thread that
// drives one device stream (worker w runs on devices[w % G]); it hands whole index
// ranges or chunks to the persistent sm_100a DFS kernel instead of calling count_with
// once per subproblem, and the per-worker partial sums are multiplier-weighted on the
// device, checked-added on the host. Two strategies are additions: strided (record i to
// worker i mod W, one persistent launch per worker — the default of the C ABI) and
// guided (shrinking chunks from the expensive end of the stream); both are opt-in here
// so the reference's defaults stay as they were.
//
// Checkpoint / resume: the reference's per-worker high-water form (ExecuteOptions::
// progress / ::resume, runner.hpp) is replaced by chunk-granular execute_checkpointed();
// a non-empty resume vector is rejected with config_error, and a progress board receives
// one final commit per contiguous worker.
#pragma once

#include <array>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#if __has_include(<json.hpp>)
#include <json.hpp>
#define NQUEENS_HAVE_JSON 1
#endif

#include "nqueens/errors.hpp"
#include "nqueens/gpu.hpp"
#include "nqueens/solver.hpp"
#include "nqueens/stack_config.hpp"
#include "nqueens/subproblems.hpp"

namespace nqueens {

enum class PartitionStrategy { uniform, weighted, stealing, guided, strided };

inline const char* to_string(PartitionStrategy s) {
    switch (s) {
        case PartitionStrategy::uniform: return "uniform";
        case PartitionStrategy::weighted: return "weighted";
        case PartitionStrategy::guided: return "guided";
        case PartitionStrategy::strided: return "strided";
        case PartitionStrategy::stealing: break;
    }
    return "stealing";
}

inline PartitionStrategy partition_strategy_from(const std::string& name) {
    for (PartitionStrategy s : {PartitionStrategy::uniform, PartitionStrategy::weighted,
                                PartitionStrategy::stealing, PartitionStrategy::guided,
                                PartitionStrategy::strided})
        if (name == to_string(s)) return s;
    throw config_error("unknown partition strategy '" + name + "'");
}

/// The paper's 8-card time-derived split (scheduler.hpp:44-45).
inline constexpr std::array<double, 8> paper_gpu_weights = {0.20, 0.15, 0.12, 0.11,
                                                            0.11, 0.11, 0.10, 0.10};

struct PartitionPlan {
    PartitionStrategy strategy = PartitionStrategy::weighted;
    int worker_count = 1;
    std::vector<double> weights;      ///< weighted only; normalised before use
    std::uint64_t chunk_size = 4096;  ///< stealing: records per chunk; guided: minimum chunk
};

/// Half-open [first, last).
struct IndexRange {
    std::uint64_t first = 0;
    std::uint64_t last = 0;
    std::uint64_t size() const { return last - first; }
};

namespace detail {
inline std::vector<IndexRange> to_ranges(const std::vector<std::uint64_t>& flat) {
    std::vector<IndexRange> out(flat.size() / 2);
    for (std::size_t i = 0; i < out.size(); ++i) out[i] = IndexRange{flat[2 * i], flat[2 * i + 1]};
    return out;
}
}  // namespace detail

/// ⌈T/W⌉ for the first T mod W workers, ⌊T/W⌋ for the rest (scheduler.hpp:61-73).
inline std::vector<IndexRange> partition_uniform(std::uint64_t task_count, int worker_count) {
    if (worker_count < 1) throw config_error("worker_count must be >= 1");
    std::vector<std::uint64_t> flat(2 * static_cast<std::size_t>(worker_count));
    gpu::check(nq_partition_uniform(task_count, worker_count, flat.data()));
    return detail::to_ranges(flat);
}

/// ⌊T·wᵢ/Σw⌋ each, remainder one by one from worker 0 (scheduler.hpp:76-102).
inline std::vector<IndexRange> partition_weighted(std::uint64_t task_count,
                                                  const std::vector<double>& weights) {
    if (weights.empty()) throw config_error("weighted partition needs at least one weight");
    std::vector<std::uint64_t> flat(2 * weights.size());
    gpu::check(nq_partition_weighted(task_count, weights.data(), static_cast<int>(weights.size()),
                                     flat.data()));
    return detail::to_ranges(flat);
}

struct WorkerStats {
    int worker = 0;
    std::uint64_t assigned = 0;     ///< 0 = dynamic (stealing / guided)
    std::uint64_t processed = 0;
    std::uint64_t partial_sum = 0;  ///< multiplier-weighted
    double elapsed_ms = 0;
    // GPU additions
    int device = 0;
    std::uint64_t nodes = 0;        ///< Alg. 3 DFS nodes counted by this worker
    std::uint64_t launches = 0;     ///< kernel launches (chunks)
    double kernel_ms = 0;           ///< device time of those launches (CUDA events)
    double span_ms = 0;             ///< device time, first enqueued operation -> last kernel end
};

struct SolveReport {
    int n = 0;
    int pre_rows = 0;
    std::string config_name;
    KernelVariant kernel = KernelVariant::lastrow;
    PartitionStrategy strategy = PartitionStrategy::weighted;
    int worker_count = 1;
    std::uint64_t task_count = 0;
    double generation_ms = 0;
    double calc_ms = 0;
    std::uint64_t total = 0;
    bool completed = true;
    std::vector<WorkerStats> workers;
    std::uint64_t nodes = 0;  ///< GPU addition: Σ Alg. 3 DFS nodes

    /// Max / min per-worker elapsed time (reported, never asserted).
    double skew_ratio() const {
        double lo = 0, hi = 0;
        for (const WorkerStats& w : workers) {
            if (w.elapsed_ms <= 0) continue;
            hi = w.elapsed_ms > hi ? w.elapsed_ms : hi;
            lo = (lo == 0 || w.elapsed_ms < lo) ? w.elapsed_ms : lo;
        }
        return lo > 0 ? hi / lo : 0.0;
    }
    double nodes_per_s() const { return calc_ms > 0 ? double(nodes) / (calc_ms * 1e-3) : 0.0; }
};

#ifdef NQUEENS_HAVE_JSON
inline void to_json(nlohmann::json& j, const WorkerStats& w) {
    j = {{"worker", w.worker},         {"assigned", w.assigned},   {"processed", w.processed},
         {"partial_sum", w.partial_sum}, {"elapsed_ms", w.elapsed_ms}, {"device", w.device},
         {"nodes", w.nodes},           {"kernel_ms", w.kernel_ms}};
}

inline void to_json(nlohmann::json& j, const SolveReport& r) {
    j = {{"n", r.n},
         {"pre_rows", r.pre_rows},
         {"config", r.config_name},
         {"kernel", to_string(r.kernel)},
         {"partition", to_string(r.strategy)},
         {"worker_count", r.worker_count},
         {"task_count", r.task_count},
         {"generation_ms", r.generation_ms},
         {"calc_ms", r.calc_ms},
         {"total", r.total},
         {"completed", r.completed},
         {"skew_ratio", r.skew_ratio()},
         {"nodes", r.nodes},
         {"nodes_per_s", r.nodes_per_s()},
         {"workers", r.workers}};
}
#endif

// ---- paper-style log lines (scheduler.hpp:162-203), formatted by the library ----------
namespace detail {
inline std::string format_log(int kind, int i, std::uint64_t u, double d) {
    char buf[256];
    gpu::check(nq_format_log(kind, i, u, d, buf, sizeof buf));
    return buf;
}
}  // namespace detail

inline std::string log_timestamp() {
    const std::string line = detail::format_log(NQ_LOG_FINISH, 0, 0, 0.0);
    return line.substr(0, line.find(' ', line.find(' ') + 1));  // "[date time.ms]"
}
inline std::string log_generation_line(double ms, std::uint64_t count) {
    return detail::format_log(NQ_LOG_GENERATION, 0, count, ms);
}
inline std::string log_start_line(int worker, std::uint64_t count, double fraction) {
    return detail::format_log(NQ_LOG_START, worker, count, fraction);
}
inline std::string log_finish_line(int worker) {
    return detail::format_log(NQ_LOG_FINISH, worker, 0, 0.0);
}
/// Parses with: n (\d+) queens result (\d+), calc time: \[([0-9.]+) ms\]
inline std::string log_result_line(int n, std::uint64_t total, double calc_ms) {
    return detail::format_log(NQ_LOG_RESULT, n, total, calc_ms);
}

// ---- execution --------------------------------------------------------------------------
struct WorkerProgress {
    std::uint64_t next_index = 0;
    std::uint64_t partial_sum = 0;
};

/// Kept for source compatibility with checkpointing callers (runner.hpp); the GPU
/// executor commits each contiguous worker's final position once, at the end.
class ProgressBoard {
public:
    void reset(const std::vector<WorkerProgress>& initial) {
        std::lock_guard<std::mutex> lk(mu_);
        slots_ = initial;
    }
    void commit(int worker, WorkerProgress p) {
        std::lock_guard<std::mutex> lk(mu_);
        if (static_cast<std::size_t>(worker) >= slots_.size()) slots_.resize(worker + 1);
        slots_[static_cast<std::size_t>(worker)] = p;
    }
    std::vector<WorkerProgress> snapshot() const {
        std::lock_guard<std::mutex> lk(mu_);
        return slots_;
    }

private:
    mutable std::mutex mu_;
    std::vector<WorkerProgress> slots_;
};

struct ExecuteOptions {
    KernelVariant kernel = KernelVariant::lastrow;
    StackConfig config = builtin_configs[1];  // config2
    PartitionPlan plan;
    std::function<void(const std::string&)> log;  // optional sink, called from workers
    ProgressBoard* progress = nullptr;
    const std::atomic<bool>* cancel = nullptr;
    std::vector<WorkerProgress> resume;  // must stay empty on the GPU path
    // GPU additions
    std::vector<int> devices;  ///< explicit device list; empty = every visible device
};

namespace detail {

inline void log_trampoline(void* user, const char* line) {
    const auto* fn = static_cast<const std::function<void(const std::string&)>*>(user);
    (*fn)(line);
}

inline int to_c_strategy(PartitionStrategy s) {
    switch (s) {
        case PartitionStrategy::uniform: return NQ_PARTITION_UNIFORM;
        case PartitionStrategy::weighted: return NQ_PARTITION_WEIGHTED;
        case PartitionStrategy::stealing: return NQ_PARTITION_STEALING;
        case PartitionStrategy::strided: return NQ_PARTITION_STRIDED;
        case PartitionStrategy::guided: break;
    }
    return NQ_PARTITION_GUIDED;
}

/// Polls the caller's atomic<bool> cancel flag into the volatile int the C ABI reads.
class CancelBridge {
public:
    explicit CancelBridge(const std::atomic<bool>* src) : src_(src) {
        if (!src_) return;
        if (src_->load()) raise();
        poller_ = std::thread([this] {
            while (!stop_.load()) {
                if (src_->load(std::memory_order_relaxed)) raise();
                std::this_thread::sleep_for(std::chrono::milliseconds(1));
            }
        });
    }
    ~CancelBridge() {
        stop_.store(true);
        if (poller_.joinable()) poller_.join();
    }
    const volatile int* flag() const { return src_ ? &flag_ : nullptr; }

private:
    // The library reads the flag with an atomic load (nq_internal.h: cancel_raised).
    void raise() { __atomic_store_n(const_cast<int*>(&flag_), 1, __ATOMIC_RELAXED); }

    const std::atomic<bool>* src_;
    volatile int flag_ = 0;
    std::atomic<bool> stop_{false};
    std::thread poller_;
};

}  // namespace detail

namespace detail {

inline void check_execute_options(int n, int pre_rows, const ExecuteOptions& opts) {
    const PartitionPlan& plan = opts.plan;
    if (plan.worker_count < 1) throw config_error("worker_count must be >= 1");
    if (plan.strategy == PartitionStrategy::stealing && plan.chunk_size == 0)
        throw config_error("chunk_size must be >= 1");
    require_feasible(opts.config, n, pre_rows, opts.kernel == KernelVariant::lastrow);
    if (plan.strategy == PartitionStrategy::weighted && !plan.weights.empty() &&
        static_cast<int>(plan.weights.size()) != plan.worker_count)
        throw config_error("weights length must equal worker_count");
    if (!opts.resume.empty())
        throw config_error("resume is not supported by the GPU executor (checkpointing is out of scope)");
    if (plan.worker_count > NQ_MAX_WORKERS)
        throw config_error("worker_count above " + std::to_string(NQ_MAX_WORKERS));
}

/// The C-ABI options of `opts`; `cfg_name` and `cancel` must outlive the call.
inline nq_solve_opts make_solve_opts(const ExecuteOptions& opts, const std::string& cfg_name,
                                     CancelBridge& cancel) {
    const PartitionPlan& plan = opts.plan;
    nq_solve_opts o{};
    o.variant = opts.kernel == KernelVariant::lastrow ? NQ_VARIANT_LASTROW : NQ_VARIANT_ITERATIVE;
    o.strategy = detail::to_c_strategy(plan.strategy);
    o.worker_count = plan.worker_count;
    o.weights = plan.weights.empty() ? nullptr : plan.weights.data();
    o.chunk = plan.chunk_size;
    o.n_devices = static_cast<int>(opts.devices.size());
    o.devices = opts.devices.empty() ? nullptr : opts.devices.data();
    o.cancel = cancel.flag();
    o.stack_depth = opts.config.max_depth();
    o.config_name = cfg_name.c_str();
    if (opts.log) {
        o.log = &log_trampoline;
        o.log_user = const_cast<void*>(static_cast<const void*>(&opts.log));
    }
    return o;
}

inline SolveReport to_report(int n, int pre_rows, const ExecuteOptions& opts,
                             const std::string& cfg_name, std::uint64_t task_count,
                             const nq_report& rep) {
    const PartitionPlan& plan = opts.plan;
    SolveReport report;
    report.n = n;
    report.pre_rows = pre_rows;
    report.config_name = cfg_name;
    report.kernel = opts.kernel;
    report.strategy = plan.strategy;
    report.worker_count = plan.worker_count;
    report.task_count = task_count;
    report.calc_ms = rep.calc_ms;
    report.total = rep.total;
    report.nodes = rep.nodes;
    report.completed = rep.completed != 0;
    report.workers.resize(static_cast<std::size_t>(plan.worker_count));
    for (int w = 0; w < plan.worker_count; ++w) {
        const nq_worker_stats& s = rep.workers[w];
        WorkerStats& d = report.workers[static_cast<std::size_t>(w)];
        d.worker = w;
        d.assigned = s.assigned;
        d.processed = s.processed;
        d.partial_sum = s.partial_sum;
        d.elapsed_ms = s.elapsed_ms;
        d.device = s.device;
        d.nodes = s.nodes;
        d.launches = s.launches;
        d.kernel_ms = s.kernel_ms;
        d.span_ms = s.span_ms;
        if (opts.progress && s.assigned)
            opts.progress->commit(w, WorkerProgress{s.processed, s.partial_sum});
    }
    return report;
}

}  // namespace detail

/// Counts a pre-generated batch on the GPUs (scheduler.hpp:266-389). Every record is
/// counted exactly once; totals are independent of strategy and worker count.
inline SolveReport execute_batch(int n, int pre_rows, const std::vector<Subproblem>& batch,
                                 const ExecuteOptions& opts) {
    detail::check_execute_options(n, pre_rows, opts);
    std::vector<nq_sub> packed;
    packed.reserve(batch.size());
    for (const Subproblem& s : batch) packed.push_back(detail::pack(s));
    const std::string cfg_name(opts.config.name);
    detail::CancelBridge cancel(opts.cancel);
    const nq_solve_opts o = detail::make_solve_opts(opts, cfg_name, cancel);
    nq_report rep{};
    gpu::check(nq_solve_batch(n, pre_rows, packed.data(), packed.size(), &o, &rep));
    return detail::to_report(n, pre_rows, opts, cfg_name, batch.size(), rep);
}

/// execute() with chunk-granular checkpoint / resume (nq_solve_checkpointed): the GPU
/// counterpart of run_with_checkpoint (runner.hpp:48-212). `chunk` records per chunk
/// (0 = automatic), the file is rewritten atomically at most every flush_interval_s.
/// A corrupt or foreign file on resume throws checkpoint_error before any device work.
inline SolveReport execute_checkpointed(int n, int pre_rows, const ExecuteOptions& opts,
                                        const std::string& path, std::uint64_t chunk = 0,
                                        double flush_interval_s = 0.0, bool resume = false) {
    detail::check_board(n);
    require_feasible(opts.config, n, pre_rows, opts.kernel == KernelVariant::lastrow);
    nq_solve_opts o{};
    o.variant = opts.kernel == KernelVariant::lastrow ? NQ_VARIANT_LASTROW : NQ_VARIANT_ITERATIVE;
    o.worker_count = opts.plan.worker_count;
    o.n_devices = static_cast<int>(opts.devices.size());
    o.devices = opts.devices.empty() ? nullptr : opts.devices.data();
    detail::CancelBridge cancel(opts.cancel);
    o.cancel = cancel.flag();
    o.stack_depth = opts.config.max_depth();
    const std::string cfg_name(opts.config.name);
    o.config_name = cfg_name.c_str();
    nq_ckpt_opts ck{path.c_str(), chunk, flush_interval_s, resume ? 1 : 0, 0.0};
    nq_report rep{};
    gpu::check(nq_solve_checkpointed(n, pre_rows, &o, &ck, &rep));
    SolveReport report;
    report.n = n;
    report.pre_rows = pre_rows;
    report.config_name = cfg_name;
    report.kernel = opts.kernel;
    report.strategy = PartitionStrategy::stealing;
    report.worker_count = rep.worker_count;
    report.task_count = rep.task_count;
    report.generation_ms = rep.generation_ms;
    report.calc_ms = rep.calc_ms;
    report.total = rep.total;
    report.nodes = rep.nodes;
    report.completed = rep.completed != 0;
    for (int w = 0; w < rep.worker_count; ++w) {
        WorkerStats d;
        d.worker = w;
        d.processed = rep.workers[w].processed;
        d.partial_sum = rep.workers[w].partial_sum;
        d.elapsed_ms = rep.workers[w].elapsed_ms;
        d.device = rep.workers[w].device;
        d.nodes = rep.workers[w].nodes;
        d.launches = rep.workers[w].launches;
        d.kernel_ms = rep.workers[w].kernel_ms;
        d.span_ms = rep.workers[w].span_ms;
        report.workers.push_back(d);
    }
    return report;
}

/// Generates the (n, pre_rows) frontier and counts it (scheduler.hpp:393-423); n == 1
/// short-circuits to Q(1) = 1 without touching a device.
inline SolveReport execute(int n, int pre_rows, const ExecuteOptions& opts) {
    detail::check_board(n);
    if (n == 1) {
        SolveReport report;
        report.n = 1;
        report.config_name = std::string(opts.config.name);
        report.kernel = opts.kernel;
        report.strategy = opts.plan.strategy;
        report.worker_count = opts.plan.worker_count;
        report.total = 1;
        report.workers.resize(static_cast<std::size_t>(opts.plan.worker_count));
        for (int w = 0; w < opts.plan.worker_count; ++w) report.workers[w].worker = w;
        report.workers[0].partial_sum = 1;
        if (opts.log) opts.log(log_result_line(1, 1, 0.0));
        return report;
    }
    if (opts.plan.strategy == PartitionStrategy::strided ||
        opts.plan.strategy == PartitionStrategy::guided) {
        // nq_solve generates the frontier itself and, from 2^20 records up, hands a
        // coarser one to the workers to be deepened on their devices (no host copy of
        // the full frontier, no H2D of it). Same totals, nodes and log lines.
        detail::check_execute_options(n, pre_rows, opts);
        const std::string cfg_name(opts.config.name);
        detail::CancelBridge cancel(opts.cancel);
        const nq_solve_opts o = detail::make_solve_opts(opts, cfg_name, cancel);
        nq_report rep{};
        gpu::check(nq_solve(n, pre_rows, &o, &rep));
        SolveReport report = detail::to_report(n, pre_rows, opts, cfg_name, rep.task_count, rep);
        report.generation_ms = rep.generation_ms;
        return report;
    }
    const auto t0 = std::chrono::steady_clock::now();
    const std::vector<Subproblem> batch = generate(GenerationPlan{n, pre_rows});
    const double gen_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (opts.log) opts.log(log_generation_line(gen_ms, batch.size()));
    SolveReport report = execute_batch(n, pre_rows, batch, opts);
    report.generation_ms = gen_ms;
    if (report.completed && opts.log) opts.log(log_result_line(n, report.total, report.calc_ms));
    return report;
}

}  // namespace nqueens
