// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// A C-ABI wrapper around the UNMODIFIED reference headers
// (/root/reference/proj/include/nqueens/*.hpp, passed in via -I by oracle/Makefile).
// Nothing from the reference is copied here: this file only includes the headers and
// forwards calls, so the oracle restatement (nq_oracle.c) and the CUDA path can be
// checked against the reference's own code, and so bench.py --impl reference can time
// the reference's own execute_batch (scheduler.hpp:266) on the GPU box's host cores.
// Built into oracle/_ref/libnqref.so (git-ignored; travels to the GPU box prebuilt).
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "nqueens/bankmodel.hpp"
#include "nqueens/scheduler.hpp"
#include "nqueens/solver.hpp"
#include "nqueens/subproblems.hpp"

namespace {
thread_local std::string g_err;

struct Packed {
  uint32_t cols, diag, antidiag, row;
};

nqueens::Subproblem unpack(const Packed& p) {
  return nqueens::Subproblem{p.cols, p.diag, p.antidiag, static_cast<int>(p.row & 0xff),
                             static_cast<int>(p.row >> 8)};
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const nqueens::config_error& e) {
    g_err = e.what();
    return -2;
  } catch (const std::overflow_error& e) {
    g_err = e.what();
    return -3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

const nqueens::StackConfig& cfg_at(int idx) { return nqueens::builtin_configs.at(idx); }
}  // namespace

extern "C" {

const char* nqref_last_error() { return g_err.c_str(); }

int nqref_count(int variant, int n, const Packed* sub, int config_index, uint64_t* count,
                int* high_water) {
  return guard([&] {
    const nqueens::Subproblem s = unpack(*sub);
    if (variant == 2) {
      *count = nqueens::count_recursive(n, s);
      *high_water = 0;
      return;
    }
    const auto r = nqueens::count_with(
        variant == 1 ? nqueens::KernelVariant::lastrow : nqueens::KernelVariant::iterative, n, s,
        cfg_at(config_index));
    *count = r.count;
    *high_water = r.high_water;
  });
}

int nqref_generate(int n, int pre_rows, Packed* out, uint64_t cap, uint64_t* total) {
  return guard([&] {
    uint64_t len = 0;
    nqueens::for_each_subproblem(nqueens::GenerationPlan{n, pre_rows}, [&](const nqueens::Subproblem& s) {
      if (out && len < cap)
        out[len] = Packed{s.cur, s.left, s.right,
                          static_cast<uint32_t>(s.placed_rows) | (static_cast<uint32_t>(s.multiplier) << 8)};
      ++len;
    });
    *total = len;
  });
}

// Records i ≡ offset (mod stride) of the reference stream (for_each_subproblem,
// subproblems.hpp:80-108), so bench.py's reference arm builds its sample with the
// reference's own generator and never loads the product library.
int nqref_generate_slice(int n, int pre_rows, uint64_t stride, uint64_t offset, Packed* out,
                         uint64_t cap, uint64_t* total) {
  return guard([&] {
    if (stride == 0) throw nqueens::config_error("stride must be >= 1");
    uint64_t idx = 0, len = 0;
    nqueens::for_each_subproblem(nqueens::GenerationPlan{n, pre_rows}, [&](const nqueens::Subproblem& s) {
      if (idx++ % stride != offset) return;
      if (out && len < cap)
        out[len] = Packed{s.cur, s.left, s.right,
                          static_cast<uint32_t>(s.placed_rows) | (static_cast<uint32_t>(s.multiplier) << 8)};
      ++len;
    });
    *total = len;
  });
}

// bankmodel.hpp:62-99 (conflict_degree), so the layout self-check's restatement is
// pinned to the reference's own model. schedule: 0 quarter_warp, 1 full_warp.
int nqref_conflict_degree(int bank_count, int word_bytes, int warp_size, const uint64_t* addrs,
                          uint64_t len, int width_bytes, int schedule, int* transactions,
                          int* max_degree) {
  return guard([&] {
    const nqueens::BankGeometry g{bank_count, word_bytes, warp_size};
    nqueens::AccessRequest req{std::vector<std::uint64_t>(addrs, addrs + len), width_bytes};
    const auto r = nqueens::conflict_degree(
        g, req, schedule ? nqueens::WarpSchedule::full_warp : nqueens::WarpSchedule::quarter_warp);
    *transactions = r.transactions;
    *max_degree = r.max_degree;
  });
}

int nqref_count_subproblems(int n, int pre_rows, uint64_t* total) {
  return guard([&] { *total = nqueens::count_subproblems(n, pre_rows); });
}

int nqref_write_batch(int n, int pre_rows, char* buf, uint64_t cap, uint64_t* len) {
  return guard([&] {
    std::ostringstream os;
    nqueens::write_batch(os, nqueens::GenerationPlan{n, pre_rows});
    const std::string s = os.str();
    *len = s.size();
    if (buf && cap) std::memcpy(buf, s.data(), s.size() < cap ? s.size() : cap);
  });
}

int nqref_aggregate(const Packed* subs, const uint64_t* counts, uint64_t len, uint64_t* total) {
  return guard([&] {
    std::vector<std::pair<nqueens::Subproblem, std::uint64_t>> v;
    v.reserve(len);
    for (uint64_t i = 0; i < len; ++i) v.emplace_back(unpack(subs[i]), counts[i]);
    *total = nqueens::aggregate(v);
  });
}

int nqref_partition(int strategy, uint64_t task_count, int workers, const double* weights,
                    uint64_t* ranges) {
  return guard([&] {
    std::vector<nqueens::IndexRange> r;
    if (strategy == 0) {
      r = nqueens::partition_uniform(task_count, workers);
    } else {
      r = nqueens::partition_weighted(task_count, std::vector<double>(weights, weights + workers));
    }
    for (size_t i = 0; i < r.size(); ++i) {
      ranges[2 * i] = r[i].first;
      ranges[2 * i + 1] = r[i].last;
    }
  });
}

// The reference execute_batch (scheduler.hpp:266-389) on a packed batch. Unpacking
// into std::vector<Subproblem> happens before the call and is not part of calc_ms,
// which is the reference's own steady_clock measurement (scheduler.hpp:306, :382).
int nqref_execute_batch(int n, int pre_rows, const Packed* subs, uint64_t len, int strategy,
                        int workers, uint64_t chunk, int variant, int config_index,
                        uint64_t* total, double* calc_ms, uint64_t* processed) {
  return guard([&] {
    std::vector<nqueens::Subproblem> batch;
    batch.reserve(len);
    for (uint64_t i = 0; i < len; ++i) batch.push_back(unpack(subs[i]));
    nqueens::ExecuteOptions opts;
    opts.kernel = variant == 1 ? nqueens::KernelVariant::lastrow : nqueens::KernelVariant::iterative;
    opts.config = cfg_at(config_index);
    opts.plan.strategy = static_cast<nqueens::PartitionStrategy>(strategy);
    opts.plan.worker_count = workers;
    opts.plan.chunk_size = chunk;
    const auto rep = nqueens::execute_batch(n, pre_rows, batch, opts);
    *total = rep.total;
    *calc_ms = rep.calc_ms;
    uint64_t p = 0;
    for (const auto& w : rep.workers) p += w.processed;
    *processed = p;
  });
}

// The reference execute (scheduler.hpp:393-423): generate + execute_batch.
int nqref_execute(int n, int pre_rows, int strategy, int workers, uint64_t chunk, int variant,
                  int config_index, uint64_t* total, double* calc_ms, double* gen_ms,
                  uint64_t* task_count) {
  return guard([&] {
    nqueens::ExecuteOptions opts;
    opts.kernel = variant == 1 ? nqueens::KernelVariant::lastrow : nqueens::KernelVariant::iterative;
    opts.config = cfg_at(config_index);
    opts.plan.strategy = static_cast<nqueens::PartitionStrategy>(strategy);
    opts.plan.worker_count = workers;
    opts.plan.chunk_size = chunk;
    const auto rep = nqueens::execute(n, pre_rows, opts);
    *total = rep.total;
    *calc_ms = rep.calc_ms;
    *gen_ms = rep.generation_ms;
    *task_count = rep.task_count;
  });
}

int nqref_log_result_line(int n, uint64_t total, double calc_ms, char* buf, uint64_t cap) {
  return guard([&] {
    const std::string s = nqueens::log_result_line(n, total, calc_ms);
    std::snprintf(buf, cap, "%s", s.c_str());
  });
}

}  // extern "C"
