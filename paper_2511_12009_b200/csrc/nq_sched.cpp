// nq_sched.cpp — the multi-GPU chunk scheduler: execute_batch / execute on devices.
//
// Reference: execute_batch (scheduler.hpp:266-389) spawns W std::threads, each running
// count_with over a contiguous range (uniform / weighted) or over chunks taken from an
// atomic cursor (stealing), with checked multiplier-weighted partial sums, the first
// failure rethrown after join, and a checked final sum. Here the same W workers each
// drive one device stream (worker w -> devices[w % G], own pooled context) and hand
// whole ranges / chunks to the persistent DFS kernel instead of one subproblem at a
// time. Two GPU strategies are added: GUIDED (the default) hands out chunks that
// shrink as the stream drains, from the expensive end first (the cost of a record rises
// with its index), and each device runs ONE streaming launch that the
// host feeds chunk by chunk (nq_dispatch.cpp); STRIDED deals record i to worker i mod W
// and runs each worker's share as one persistent launch, which balances the workers
// statistically with no host traffic while the kernels run.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "nq_gpu.h"
#include "nq_internal.h"

namespace nqb200 {
namespace {

bool add_ok(uint64_t a, uint64_t b, uint64_t* r) { return !__builtin_add_overflow(a, b, r); }

std::string timestamp() {
  using namespace std::chrono;
  const auto now = system_clock::now();
  const auto ms = duration_cast<milliseconds>(now.time_since_epoch()) % 1000;
  const std::time_t t = system_clock::to_time_t(now);
  std::tm tm{};
  localtime_r(&t, &tm);
  char buf[96];
  std::snprintf(buf, sizeof buf, "[%04d-%02d-%02d %02d:%02d:%02d.%03d]", tm.tm_year + 1900,
                tm.tm_mon + 1, tm.tm_mday, tm.tm_hour, tm.tm_min, tm.tm_sec,
                static_cast<int>(ms.count()));
  return buf;
}

// Pooled contexts keyed by (device, slot): workers sharing a device get separate streams.
struct Pool {
  std::mutex mu;
  std::vector<std::vector<nq_ctx*>> ctx;  // [device][slot]
};
Pool& pool() {
  static Pool* p = new Pool;  // intentionally leaked: contexts live for the process
  return *p;
}

int pooled_ctx(int device, int slot, nq_ctx** out) {
  Pool& p = pool();
  std::lock_guard<std::mutex> lk(p.mu);
  if (static_cast<int>(p.ctx.size()) <= device) p.ctx.resize(device + 1);
  auto& v = p.ctx[device];
  if (static_cast<int>(v.size()) <= slot) v.resize(slot + 1, nullptr);
  if (!v[slot])
    if (int rc = nq_ctx_create(device, &v[slot])) return rc;
  *out = v[slot];
  return NQ_OK;
}

void emit(const nq_solve_opts& o, int kind, int i, uint64_t u, double d) {
  if (!o.log) return;
  char buf[256];
  nq_format_log(kind, i, u, d, buf, sizeof buf);
  o.log(o.log_user, buf);
}

}  // namespace
}  // namespace nqb200

using namespace nqb200;

extern "C" int nq_format_log(int kind, int i, uint64_t u, double d, char* buf, uint64_t cap) {
  if (!buf || cap == 0) return set_error(NQ_ECONFIG, "null log buffer");
  char body[200];
  switch (kind) {  // scheduler.hpp:177-203
    case NQ_LOG_GENERATION:
      std::snprintf(body, sizeof body, "Use %.2fms to generate %llu subproblems!", d,
                    static_cast<unsigned long long>(u));
      break;
    case NQ_LOG_START:
      std::snprintf(body, sizeof body, "worker [%d] start job, with %llu(%.2f) subproblems.", i,
                    static_cast<unsigned long long>(u), d);
      break;
    case NQ_LOG_FINISH:
      std::snprintf(body, sizeof body, "worker [%d] finish job.", i);
      break;
    case NQ_LOG_RESULT:
      std::snprintf(body, sizeof body, "n %d queens result %llu, calc time: [%.2f ms]", i,
                    static_cast<unsigned long long>(u), d);
      break;
    default:
      return set_error(NQ_ECONFIG, "unknown log kind " + std::to_string(kind));
  }
  std::snprintf(buf, cap, "%s %s", timestamp().c_str(), body);
  return NQ_OK;
}

extern "C" int nq_partition_uniform(uint64_t task_count, int worker_count, uint64_t* ranges) {
  if (worker_count < 1) return set_error(NQ_ECONFIG, "worker_count must be >= 1");
  const uint64_t w = static_cast<uint64_t>(worker_count);
  const uint64_t base = task_count / w, extra = task_count % w;
  uint64_t at = 0;
  for (uint64_t i = 0; i < w; ++i) {
    const uint64_t len = base + (i < extra ? 1 : 0);  // remainder to the lowest workers
    ranges[2 * i] = at;
    ranges[2 * i + 1] = at + len;
    at += len;
  }
  return NQ_OK;
}

extern "C" int nq_partition_weighted(uint64_t task_count, const double* weights, int worker_count,
                                     uint64_t* ranges) {
  if (worker_count < 1 || !weights)
    return set_error(NQ_ECONFIG, "weighted partition needs at least one weight");
  double sum = 0;
  for (int i = 0; i < worker_count; ++i) {
    if (!(weights[i] > 0)) return set_error(NQ_ECONFIG, "partition weights must be positive");
    sum += weights[i];
  }
  std::vector<uint64_t> len(worker_count);
  uint64_t given = 0;
  for (int i = 0; i < worker_count; ++i) {
    len[i] = static_cast<uint64_t>(std::floor(static_cast<double>(task_count) * (weights[i] / sum)));
    given += len[i];
  }
  for (int i = 0; given < task_count; i = (i + 1) % worker_count) ++len[i], ++given;
  uint64_t at = 0;
  for (int i = 0; i < worker_count; ++i) {
    ranges[2 * i] = at;
    ranges[2 * i + 1] = at + len[i];
    at += len[i];
  }
  return NQ_OK;
}

extern "C" int nq_solve_batch(int n, int pre_rows, const nq_sub* subs, uint64_t count,
                              const nq_solve_opts* opts, nq_report* out) {
  return solve_batch_impl(n, pre_rows, 0, subs, nullptr, count, opts, out);
}

extern "C" int nq_solve_batch_expand(int n, int target_rows, const nq_sub* roots, uint64_t count,
                                     const nq_solve_opts* opts, nq_report* out) {
  if (target_rows < 1 || target_rows >= n)
    return set_error(NQ_ECONFIG, "target rows must satisfy 1 <= T < n (n=" + std::to_string(n) +
                                     ", T=" + std::to_string(target_rows) + ")");
  return solve_batch_impl(n, 0, target_rows, roots, nullptr, count, opts, out);
}

extern "C" int nq_solve_batch_device(int n, int pre_rows, const nq_sub* const* dev_subs,
                                     uint64_t count, const nq_solve_opts* opts, nq_report* out) {
  if (!dev_subs) return set_error(NQ_ECONFIG, "null device frontier list");
  return solve_batch_impl(n, pre_rows, 0, nullptr, dev_subs, count, opts, out);
}

int nqb200::solve_batch_impl(int n, int pre_rows, int target_rows, const nq_sub* subs,
                             const nq_sub* const* dev_subs, uint64_t count,
                             const nq_solve_opts* opts, nq_report* out, uint64_t deep_total) {
  using clk = std::chrono::steady_clock;
  // The pooled per-device contexts are shared by every call: concurrent calls from
  // different host threads run one after the other (the reference's execute_batch is
  // likewise driven from one control thread).
  static std::mutex solve_mu;
  std::lock_guard<std::mutex> solve_lock(solve_mu);
  if (!out) return set_error(NQ_ECONFIG, "null report");
  nq_solve_opts o{};
  o.variant = NQ_VARIANT_LASTROW;
  o.strategy = NQ_PARTITION_GUIDED;  // opts == NULL: dynamic dispatch (one streaming launch per device)
  if (opts) o = *opts;
  if (o.dispatch) {  // a shared dispenser fixes the policy for every cooperating caller
    uint64_t d_count = 0;
    nq_dispatch_info(o.dispatch, &d_count, &o.strategy, &o.chunk, nullptr);
    if (d_count != count)
      return set_error(NQ_ECONFIG, "dispenser covers " + std::to_string(d_count) +
                                       " records but the batch has " + std::to_string(count));
  }
  if (o.worker_count < 0) return set_error(NQ_ECONFIG, "worker_count must be >= 1");
  if (o.strategy == NQ_PARTITION_STEALING && o.chunk == 0)
    return set_error(NQ_ECONFIG, "chunk_size must be >= 1");
  if (o.strategy < NQ_PARTITION_UNIFORM || o.strategy > NQ_PARTITION_STRIDED)
    return set_error(NQ_ECONFIG, "unknown partition strategy " + std::to_string(o.strategy));
  if (int rc = require_feasible(o.stack_depth, o.config_name, n,
                                target_rows ? target_rows : pre_rows,
                                o.variant == NQ_VARIANT_LASTROW))
    return rc;
  if (dev_subs && o.strategy == NQ_PARTITION_STRIDED)
    return set_error(NQ_ECONFIG, "a device-resident frontier is split by ranges or chunks "
                                 "(uniform, weighted, stealing, guided), not strided");
  if (n < 1 || n > 32)
    return set_error(NQ_ECONFIG, "board size must be in [1, 32], got " + std::to_string(n));

  int ndev = 0;
  if (int rc = nq_device_count(&ndev)) return rc;
  std::vector<int> devs;
  if (o.devices && o.n_devices > 0) {
    devs.assign(o.devices, o.devices + o.n_devices);
  } else {
    const int k = o.n_devices > 0 ? std::min(o.n_devices, ndev) : ndev;
    for (int i = 0; i < k; ++i) devs.push_back(i);
  }
  if (devs.empty()) return set_error(NQ_ECUDA, "no CUDA device visible");
  const int G = static_cast<int>(devs.size());
  const int W = o.worker_count > 0 ? o.worker_count : G;
  if (W > NQ_MAX_WORKERS)
    return set_error(NQ_ECONFIG, "worker_count above " + std::to_string(NQ_MAX_WORKERS));
  // Deepened records exist only on the devices: one worker may take its roots as one
  // range under any strategy; several need strided shares or guided chunks of them.
  if (target_rows && W > 1 && o.strategy != NQ_PARTITION_STRIDED &&
      o.strategy != NQ_PARTITION_GUIDED)
    return set_error(NQ_ECONFIG, "device-side deepening over several workers needs the "
                                 "strided or guided strategy");
  // Worker w runs on devs[w % G]. Its context slot is the number of earlier workers on
  // the same device id, so two workers never share a context (stream, buffers, result
  // mirror) even when the device list repeats a device (devices = {0, 0, ...}).
  std::vector<int> slot(W, 0);
  for (int w = 0; w < W; ++w)
    for (int v = 0; v < w; ++v) slot[w] += devs[v % G] == devs[w % G] ? 1 : 0;

  // One worker with a private dispenser would take every chunk itself: it gets the
  // contiguous launch instead (the same expensive-first order), without the streaming
  // launch's refill and feeder cost (0.2-1%, profiles/r02_stream_probe.log).
  const bool solo = W == 1 && !o.dispatch &&
                    (o.strategy == NQ_PARTITION_STEALING || o.strategy == NQ_PARTITION_GUIDED);
  std::vector<uint64_t> ranges;
  if (solo) {
    ranges = {0, count};
  } else if (o.strategy == NQ_PARTITION_UNIFORM || o.strategy == NQ_PARTITION_WEIGHTED) {
    ranges.resize(2 * W);
    int rc;
    if (o.strategy == NQ_PARTITION_UNIFORM || !o.weights) {
      if (o.strategy == NQ_PARTITION_WEIGHTED) {
        std::vector<double> eq(W, 1.0 / W);
        rc = nq_partition_weighted(count, eq.data(), W, ranges.data());
      } else {
        rc = nq_partition_uniform(count, W, ranges.data());
      }
    } else {
      rc = nq_partition_weighted(count, o.weights, W, ranges.data());
    }
    if (rc) return rc;
  }
  const bool dynamic =
      !solo && (o.strategy == NQ_PARTITION_STEALING || o.strategy == NQ_PARTITION_GUIDED);
  // Dynamic dispatch over roots deepened on the devices hands out ranges of the DEEPENED
  // stream (every worker deepens all roots; its records are in stream order).
  uint64_t disp_count = count;
  if (dynamic && target_rows) {
    if (o.dispatch)
      return set_error(NQ_ECONFIG, "a shared dispenser cannot drive device-side deepening");
    if (int rc = expand(n, subs, count, target_rows, nullptr, 0, &disp_count)) return rc;
  }
  nq_dispatch* disp = o.dispatch;
  struct DispGuard {
    nq_dispatch* d = nullptr;
    ~DispGuard() { nq_dispatch_close(d, 0); }
  } own_disp;
  if (dynamic && !disp) {
    if (int rc = nq_dispatch_create(nullptr, disp_count, o.strategy, o.chunk, W, &own_disp.d))
      return rc;
    disp = own_disp.d;
  }

  std::memset(out, 0, sizeof(*out));
  out->task_count = count;
  out->worker_count = W;

  const int kind = target_rows ? kLaunchExpand : (dev_subs ? kLaunchDevice : kLaunchHost);
  const int launch_rows = target_rows ? target_rows : pre_rows;
  std::atomic<bool> interrupted{false};
  std::mutex fail_mu;
  std::string failure;
  const auto t0 = clk::now();
  std::vector<std::thread> threads;
  threads.reserve(W);
  for (int w = 0; w < W; ++w) {
    threads.emplace_back([&, w] {
      nq_worker_stats& st = out->workers[w];
      st.worker = w;
      st.device = devs[w % G];
      const nq_sub* src = dev_subs ? dev_subs[w % G] : subs;
      const std::string range_name = "nq_solve_batch worker " + std::to_string(w);
      NvtxRange range(range_name.c_str());
      const auto s0 = clk::now();
      nq_ctx* c0 = nullptr;                   // this worker's context
      struct Flight {
        uint64_t first = 0, len = 0, work = 0;
      } fl;                                   // the one-launch strategies' launch
      uint64_t bad_first = 0, bad_len = 0;  // the launch that failed (for the message)
      uint64_t bad_record = ~0ull;           // streaming: the rejected record's batch index
      bool strided_index = false;
      int rc = pooled_ctx(st.device, slot[w], &c0);
      if (rc == NQ_OK) nq_ctx_set_cancel(c0, o.cancel);
      if (rc == NQ_OK) rc = ctx_mark_start(c0);
      // uniform / weighted / strided: one launch over this worker's records, then collect
      auto launch = [&](const nq_sub* base, uint64_t f, uint64_t l) -> int {
        const int e = ctx_launch(c0, n, launch_rows, o.variant, base + f, l, kind);
        if (e) {
          bad_first = f;
          bad_len = l;
          return e;
        }
        fl.first = f;
        fl.len = l;
        fl.work = kind == kLaunchExpand ? ctx_last_expanded(c0) : l;
        return NQ_OK;
      };
      auto collect = [&]() -> int {
        nq_result r{};
        const int e = nq_collect(c0, &r);
        if (e) {
          bad_first = fl.first;
          bad_len = fl.len;
          return e;
        }
        if (r.subproblems < fl.work) interrupted.store(true);  // cancelled inside the launch
        if (!add_ok(st.partial_sum, r.solutions, &st.partial_sum))
          return set_error(NQ_EOVERFLOW, "solution count overflows 64 bits");
        st.processed += r.subproblems;
        st.nodes += r.nodes;
        st.chunks += 1;
        st.launches += 1;
        st.kernel_ms += r.kernel_ms;
        st.span_ms = std::max(st.span_ms, ctx_span_ms(c0, c0));
        return NQ_OK;
      };
      // Dynamic strategies: ONE persistent streaming launch per worker, fed chunk by chunk
      // from the dispenser while it runs (ctx_stream_*): the GPU never drains between
      // chunks, and the host keeps only a small lead of published-but-untaken records
      // (low_water) so that the last chunks still balance across devices.
      static const bool dbg = std::getenv("NQB_STREAM_DEBUG") != nullptr;
      auto trace = [&](const char* what, uint64_t a = 0, uint64_t b = 0) {
        if (!dbg) return;
        const double t = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
        std::fprintf(stderr, "[%9.3f ms] worker %d: %s %llu %llu\n", t, w, what,
                     static_cast<unsigned long long>(a), static_cast<unsigned long long>(b));
      };
      auto stream_worker = [&](int wk, nq_ctx* c, nq_worker_stats& ws) -> int {
        struct Pushed {
          uint64_t vstart, first, len;
        };
        std::vector<Pushed> pushed;
        // The whole batch is made device-resident first (the caller's device copy, one
        // H2D of host records, or all roots deepened on this device): the running
        // kernel is then fed by publishing ranges of it, with no stream operation.
        const nq_sub* all = src;
        uint64_t all_n = count;
        int e = NQ_OK;
        trace("prepare", count);
        if (kind == kLaunchHost) e = ctx_upload(c, src, count, &all);
        else if (kind == kLaunchExpand) e = ctx_deepen(c, n, target_rows, src, count, &all, &all_n);
        trace("resident", all_n);
        if (e == NQ_OK && all_n != disp_count)
          e = set_error(NQ_ECONFIG, "deepened batch has " + std::to_string(all_n) +
                                        " records, the dispenser " + std::to_string(disp_count));
        uint64_t floor = 1;
        nq_dispatch_info(disp, nullptr, nullptr, &floor, nullptr);
        const uint64_t max_chunks =
            std::min<uint64_t>(disp_count + 1, disp_count / std::max<uint64_t>(floor, 1) + 4096);
        const uint64_t lanes = ctx_lanes(c, n, launch_rows);
        const uint64_t low_water = std::max<uint64_t>(lanes / 8, 4096);
        if (e == NQ_OK) e = ctx_stream_begin(c, max_chunks);
        trace("begun", max_chunks, lanes);
        if (e) {
          if (kind == kLaunchExpand) ctx_release_deep(c);
          return e;
        }
        // The feeder runs on its own thread and makes NO CUDA call: this thread's launch
        // (and anything after it) can block on driver locks held by another thread that
        // is synchronising the device — i.e. waiting for this very kernel, which only
        // ends once the feeder has published everything and closed the queue.
        std::atomic<bool> launch_failed{false};
        bool cancelled = false;
        int fe = NQ_OK;
        std::string fe_msg;  // nq_last_error() is per thread: carried back to this one
        std::thread feeder([&] {
          // The lead of published-but-untaken records must outlast the feeder's own
          // reaction time (~0.1 ms), whatever the record rate (N=18 R=7 takes 3 x 10^8
          // records/s): it tracks the measured consumption rate, 300 us of it, never
          // below lanes/8. A larger lead would only hold back work from other GPUs.
          auto t_prev = clk::now();
          uint64_t c_prev = 0;
          double rate = 0.0;  // records per second, smoothed
          while (fe == NQ_OK && !launch_failed.load()) {
            if (cancel_raised(o.cancel)) {
              cancelled = true;
              interrupted.store(true);
              break;
            }
            uint64_t consumed = 0;
            ctx_stream_consumed(c, &consumed);
            const auto now = clk::now();
            const double dt = std::chrono::duration<double>(now - t_prev).count();
            if (dt >= 200e-6) {
              const double r = static_cast<double>(consumed - std::min(consumed, c_prev)) / dt;
              rate = rate == 0.0 ? r : 0.7 * rate + 0.3 * r;
              t_prev = now;
              c_prev = consumed;
            }
            const uint64_t lead = std::max<uint64_t>(low_water, static_cast<uint64_t>(rate * 300e-6));
            const uint64_t pub = ctx_stream_published(c);
            if (pub - consumed >= lead) {
              if (pub - consumed > 4 * lead) std::this_thread::sleep_for(std::chrono::microseconds(50));
              else std::this_thread::yield();
              continue;
            }
            uint64_t f = 0, l = 0;
            const int got = dispatch_take_at_least(disp, lead - (pub - consumed), &f, &l);
            if (got < 0) {
              fe = got;
              break;
            }
            if (got == 0) break;  // dispenser drained: close the queue below
            pushed.push_back(Pushed{pub, f, l});
            fe = ctx_stream_push(c, all + f, l);
            trace("published", f, l);
            // nothing left anywhere: close at once, so that lanes waiting for more learn
            // it now and start the tail donation instead of napping
            if (fe == NQ_OK && dispatch_drained(disp)) break;
          }
          if (fe != NQ_OK) fe_msg = nq_last_error();
          ctx_stream_close(c, cancelled || fe != NQ_OK);
          trace("closed", ctx_stream_published(c));
        });
        e = ctx_stream_launch(c, n, launch_rows, o.variant);
        trace("launched", e);
        if (e) launch_failed.store(true);
        feeder.join();
        if (e) {
          if (kind == kLaunchExpand) ctx_release_deep(c);
          return e;
        }
        e = fe == NQ_OK ? NQ_OK : set_error(fe, fe_msg);
        nq_result r{};
        const int re = nq_collect(c, &r);  // always drain the launch
        trace("collected", re, r.subproblems);
        if (kind == kLaunchExpand) ctx_release_deep(c);
        ws.launches += 1;
        ws.chunks += pushed.size();
        if (e) return e;
        if (re) {  // a rejected record: map its queue position back to the batch
          const uint64_t v = ctx_last_bad(c);
          for (const Pushed& p : pushed)
            if (v != ~0ull && v >= p.vstart && v < p.vstart + p.len) {
              bad_first = p.first;
              bad_len = p.len;
              if (kind != kLaunchExpand) bad_record = p.first + (p.vstart + p.len - 1 - v);
            }
          return re;
        }
        uint64_t work = 0;
        for (const Pushed& p : pushed) work += p.len;
        if (r.subproblems < work || cancelled) interrupted.store(true);
        if (!add_ok(ws.partial_sum, r.solutions, &ws.partial_sum))
          return set_error(NQ_EOVERFLOW, "solution count overflows 64 bits");
        ws.processed += r.subproblems;
        ws.nodes += r.nodes;
        ws.kernel_ms += r.kernel_ms;
        ws.span_ms = std::max(ws.span_ms, ctx_span_ms(c0, c));
        (void)wk;
        return NQ_OK;
      };
      std::vector<nq_sub> gathered;
      if (rc == NQ_OK) {
        if (o.strategy == NQ_PARTITION_STRIDED) {
          // Gather records w, w+W, w+2W, ... and count them in one launch (a single
          // worker counts the caller's buffer in place: no host copy).
          const nq_sub* mine = subs;
          uint64_t mine_n = count;
          if (W > 1) {
            gathered.reserve(count / W + 1);
            for (uint64_t i = static_cast<uint64_t>(w); i < count; i += static_cast<uint64_t>(W))
              gathered.push_back(subs[i]);
            mine = gathered.data();
            mine_n = gathered.size();
          }
          strided_index = true;
          st.assigned = mine_n;
          emit(o, NQ_LOG_START, w, mine_n, count ? double(mine_n) / double(count) : 0.0);
          if (cancel_raised(o.cancel)) {
            interrupted.store(true);
          } else if (mine_n) {
            rc = launch(mine, 0, mine_n);
            if (rc == NQ_OK) rc = collect();
          }
        } else if (!ranges.empty()) {
          const uint64_t first = ranges[2 * w], len = ranges[2 * w + 1] - first;
          // a lone dynamic worker reports like the reference's stealing worker
          // (assigned 0 = dynamic, scheduler.hpp:106, :350); a lone range worker over
          // deepened roots reports the deepened records it was handed (:330)
          const uint64_t shown = deep_total && W == 1 ? deep_total : len;
          st.assigned = solo ? 0 : shown;
          emit(o, NQ_LOG_START, w, solo ? 0 : shown,
               solo || !count ? 0.0 : double(len) / double(count));
          if (cancel_raised(o.cancel)) {
            interrupted.store(true);
          } else if (len) {
            rc = launch(src, first, len);
            if (rc == NQ_OK) rc = collect();
          }
        } else {
          emit(o, NQ_LOG_START, w, 0, 0.0);
          rc = stream_worker(w, c0, st);
        }
      }
      st.elapsed_ms = std::chrono::duration<double, std::milli>(clk::now() - s0).count();
      if (c0) nq_ctx_set_cancel(c0, nullptr);
      if (rc) {
        std::lock_guard<std::mutex> lk(fail_mu);
        if (failure.empty()) {
          uint64_t bad = c0 ? ctx_last_bad(c0) : ~0ull;
          uint64_t global_bad = strided_index
                                    ? static_cast<uint64_t>(w) + bad * static_cast<uint64_t>(W)
                                    : bad_first + bad;
          if (dynamic) {
            global_bad = bad_record;
            bad = bad_record;
          }
          std::string where = bad != ~0ull && kind != kLaunchExpand
                                  ? "subproblem " + std::to_string(global_bad)
                                  : "chunk [" + std::to_string(bad_first) + ", " +
                                        std::to_string(bad_first + bad_len) + ")";
          failure = "worker " + std::to_string(w) + " failed on " + where + ": " + nq_last_error();
        }
        interrupted.store(true);
        return;
      }
      emit(o, NQ_LOG_FINISH, w, 0, 0.0);
    });
  }
  for (auto& t : threads) t.join();
  if (!failure.empty()) return set_error(NQ_ECUDA, failure);
  out->calc_ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
  uint64_t total = 0, nodes = 0;
  for (int w = 0; w < W; ++w) {
    if (!add_ok(total, out->workers[w].partial_sum, &total))
      return set_error(NQ_EOVERFLOW, "solution count overflows 64 bits");
    nodes += out->workers[w].nodes;
  }
  out->total = total;
  out->nodes = nodes;
  out->completed = interrupted.load() ? 0 : 1;
  return NQ_OK;
}

extern "C" int nq_solve(int n, int pre_rows, const nq_solve_opts* opts, nq_report* out) {
  using clk = std::chrono::steady_clock;
  if (!out) return set_error(NQ_ECONFIG, "null report");
  nq_solve_opts o{};
  o.variant = NQ_VARIANT_LASTROW;
  o.strategy = NQ_PARTITION_GUIDED;  // opts == NULL: dynamic dispatch (one streaming launch per device)
  if (opts) o = *opts;
  if (n < 1 || n > 32)
    return set_error(NQ_ECONFIG, "board size must be in [1, 32], got " + std::to_string(n));
  if (n == 1) {  // execute's short-circuit (scheduler.hpp:396-410)
    std::memset(out, 0, sizeof(*out));
    out->total = 1;
    out->completed = 1;
    out->worker_count = o.worker_count > 0 ? std::min(o.worker_count, NQ_MAX_WORKERS) : 1;
    for (int w = 0; w < out->worker_count; ++w) out->workers[w].worker = w;
    out->workers[0].partial_sum = 1;
    emit(o, NQ_LOG_RESULT, 1, 1, 0.0);
    return NQ_OK;
  }
  const auto g0 = clk::now();
  uint64_t total = 0;
  if (int rc = count_subproblems(n, pre_rows, &total)) return rc;
  // Large frontiers (N=27, R=7: 453,688,251 records, 7.26 GB) are never materialised on
  // the host: a coarse frontier 3 rows shallower is dealt to the workers (strided shares,
  // or guided chunks of roots) and deepened on each device (nq_count_expand). From ~1 M records up this is also the faster path —
  // N=20 R=7 execute: 1 573 ms vs 1 716 ms with host generation + 364 MB H2D — so it is
  // the default there. Threshold: NQB_DEVICE_EXPAND_MIN_RECORDS (default 2^20).
  uint64_t expand_min = 1ull << 20;
  if (const char* e = std::getenv("NQB_DEVICE_EXPAND_MIN_RECORDS")) expand_min = std::strtoull(e, nullptr, 10);
  const int coarse = std::max(2, pre_rows - 3);
  // One worker (the reference's default plan: weighted, worker_count 1) takes the whole
  // frontier under any strategy, so it can always be deepened on its device.
  int ndev = 0;
  if (nq_device_count(&ndev) != NQ_OK) ndev = 0;
  const int n_dev = o.devices && o.n_devices > 0 ? o.n_devices
                    : o.n_devices > 0           ? std::min(o.n_devices, ndev)
                                                : ndev;
  const bool one_worker = (o.worker_count > 0 ? o.worker_count : n_dev) == 1;
  const bool deepenable = !o.dispatch && (o.strategy == NQ_PARTITION_STRIDED ||
                                          o.strategy == NQ_PARTITION_GUIDED || one_worker);
  if (total >= expand_min && deepenable && coarse < pre_rows) {
    uint64_t roots_n = 0;
    if (int rc = count_subproblems(n, coarse, &roots_n)) return rc;
    std::vector<nq_sub> roots(roots_n);
    if (int rc = generate_slice(n, coarse, 1, 0, roots.data(), roots_n, &roots_n)) return rc;
    const double gen_ms = std::chrono::duration<double, std::milli>(clk::now() - g0).count();
    emit(o, NQ_LOG_GENERATION, 0, total, gen_ms);
    const int rc =
        solve_batch_impl(n, coarse, pre_rows, roots.data(), nullptr, roots_n, &o, out, total);
    if (rc) return rc;
    out->task_count = total;
    out->generation_ms = gen_ms;
    if (out->completed) emit(o, NQ_LOG_RESULT, n, out->total, out->calc_ms);
    return NQ_OK;
  }
  std::vector<nq_sub> batch(total);
  if (int rc = generate_slice(n, pre_rows, 1, 0, batch.data(), total, &total)) return rc;
  const double gen_ms = std::chrono::duration<double, std::milli>(clk::now() - g0).count();
  emit(o, NQ_LOG_GENERATION, 0, total, gen_ms);
  const int rc = nq_solve_batch(n, pre_rows, batch.data(), total, &o, out);
  if (rc) return rc;
  out->generation_ms = gen_ms;
  if (out->completed) emit(o, NQ_LOG_RESULT, n, out->total, out->calc_ms);
  return NQ_OK;
}
