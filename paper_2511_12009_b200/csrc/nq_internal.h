// nq_internal.h — shared helpers of libnqb200.so (not installed).
#pragma once
#include <cstdint>
#include <memory>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "nq_gpu.h"

namespace nqb200 {

// NVTX range for the host phases (generation, H2D, launch + wait, worker lifetimes):
// visible to ncu --nvtx filters and any NVTX consumer; free when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// A caller's cancel flag (nq_solve_opts::cancel, nq_ctx_set_cancel) is written by
// another thread: read it with an atomic load, never a plain (racy) one.
inline bool cancel_raised(const volatile int* flag) {
  return flag && __atomic_load_n(const_cast<const int*>(flag), __ATOMIC_RELAXED) != 0;
}

// Records the thread-local message returned by nq_last_error(); returns code.
int set_error(int code, const std::string& msg);

int check_plan(int n, int pre_rows);

// The folded frontier stream of (n, R) with its per-prefix offsets computed once, so
// any contiguous range or systematic slice can be emitted later without walking (or
// materialising) the rest: the checkpointed runner emits one chunk at a time, which
// keeps host memory at chunk size even for N=27 (453,688,251 records at R=7).
class FrontierStream {
 public:
  FrontierStream();
  ~FrontierStream();
  int open(int n, int pre_rows);
  uint64_t size() const;
  // Records offset, offset + stride, ... into out[0 .. cap).
  int emit(uint64_t stride, uint64_t offset, nq_sub* out, uint64_t cap) const;

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};
int generate_slice(int n, int pre_rows, uint64_t stride, uint64_t offset, nq_sub* out,
                   uint64_t cap, uint64_t* total);
int count_subproblems(int n, int pre_rows, uint64_t* total);
int expand(int n, const nq_sub* roots, uint64_t count, int target, nq_sub* out, uint64_t cap,
           uint64_t* total);

// require_feasible (stack_config.hpp:59-71): the caller's stack budget must hold the
// required depth n - R - lastrow; the message names the smallest built-in config.
int require_feasible(int stack_depth, const char* config_name, int n, int pre_rows,
                     bool last_row);

// Index (within the last batch) of the record a counting call rejected, or ~0.
uint64_t ctx_last_bad(const nq_ctx* c);

// Records the last nq_count_expand deepened (the launch's full work, for cancel checks).
uint64_t ctx_last_expanded(const nq_ctx* c);

// Asynchronous launch on a context (completed by nq_collect): host records (H2D into the
// context's buffer), device-resident records, or host roots deepened to pre_rows on the
// device first. The one-launch strategies' workers use one per worker; the dynamic ones
// use the streaming form (ctx_stream_*).
enum { kLaunchHost = 0, kLaunchDevice = 1, kLaunchExpand = 2 };
int ctx_launch(nq_ctx* c, int n, int pre_rows, int variant, const nq_sub* subs, uint64_t count,
               int kind);
// Marks a worker's start on c's stream; ctx_span_ms(start, end) is the device time from
// that mark to the end of end's last kernel (both contexts on one device).
int ctx_mark_start(nq_ctx* c);
double ctx_span_ms(const nq_ctx* start, const nq_ctx* end);
int ctx_device(const nq_ctx* c);

// Streaming launch: ONE persistent counting kernel fed while it runs. begin (reset,
// size the chunk table) -> launch -> any number of push (a chunk of device-resident
// records) -> close -> nq_collect. The kernel hands out published records lane by lane
// and naps while the queue is empty, so chunks of any size cost no launch and no
// end-of-launch tail. Between launch and collect the host makes NO stream call on the
// context: table, publish word and progress live in mapped pinned host memory.
int ctx_stream_begin(nq_ctx* c, uint64_t max_chunks);
int ctx_stream_launch(nq_ctx* c, int n, int pre_rows, int variant);
int ctx_stream_push(nq_ctx* c, const nq_sub* dev_base, uint64_t len);
int ctx_stream_consumed(nq_ctx* c, uint64_t* consumed);  // queue positions taken (coarse)
int ctx_stream_close(nq_ctx* c, bool cancel);
uint64_t ctx_stream_published(const nq_ctx* c);
// nq_dispatch_take for a streaming feeder that needs at least `want` records: stealing
// returns ceil(want / chunk) consecutive chunks as one range (guided ignores `want`).
int dispatch_take_at_least(nq_dispatch* d, uint64_t want, uint64_t* first, uint64_t* len);
// Every record of the dispenser has been handed out (to any worker or process).
bool dispatch_drained(const nq_dispatch* d);
// Device-resident copy of a host batch on the context (ensure + H2D on its stream).
int ctx_upload(nq_ctx* c, const nq_sub* host, uint64_t count, const nq_sub** dev);
// Host roots deepened on the context's device to `target` rows (stream-ordered, the
// buffer lives until ctx_release_deep); *total records at *dev.
int ctx_deepen(nq_ctx* c, int n, int target, const nq_sub* host_roots, uint64_t count,
               const nq_sub** dev, uint64_t* total);
void ctx_release_deep(nq_ctx* c);
uint64_t ctx_lanes(nq_ctx* c, int n, int pre_rows);  // resident lanes of a launch

// execute_batch over records that are deepened to `target_rows` on the device first
// (target_rows == 0: count the records as they are). nq_solve_batch is the
// target_rows == 0 case; nq_solve uses the deepening form for large frontiers.
// dev_subs (optional): per worker-device full copies of subs already on the devices.
// deep_total (optional, 0 = unknown): the number of deepened records, reported as a lone
// range worker's assignment (what the reference's execute would have handed it).
int solve_batch_impl(int n, int pre_rows, int target_rows, const nq_sub* subs,
                     const nq_sub* const* dev_subs, uint64_t count, const nq_solve_opts* opts,
                     nq_report* out, uint64_t deep_total = 0);

}  // namespace nqb200
