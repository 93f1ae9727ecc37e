/*
 * nq_gpu.h — C ABI of the B200-native N-Queens counting path (libnqb200.so).
 *
 * The reference (/root/reference/proj/include/nqueens/) is a header-only C++ library
 * with no FFI. Its hot path is
 *
 *   execute(n, R, opts)               scheduler.hpp:393   generate + execute_batch
 *   execute_batch(n, R, batch, opts)  scheduler.hpp:266   worker pool over count_with
 *   count_with(variant, n, sub, cfg)  solver.hpp:193      one subproblem, CPU DFS
 *   for_each_subproblem / generate    subproblems.hpp:80  folded frontier
 *   count_subproblems                 subproblems.hpp:118
 *
 * This header is the plain-pointer boundary those entry points are re-bound to: the
 * C++ drop-in headers in include/nqueens/ and the Python package call only these
 * functions. Every entry point returns NQ_OK (0) or a negative status; the message of
 * the last failure on the calling thread is nq_last_error():
 *
 *   NQ_ECUDA     (-1)  CUDA / device failure           ~ std::runtime_error
 *   NQ_ECONFIG   (-2)  bad n / R / depth / input        ~ nqueens::config_error
 *   NQ_EOVERFLOW (-3)  64-bit count overflow            ~ std::overflow_error
 *   NQ_ECANCEL   (-4)  cancelled between chunks         (SolveReport::completed=false)
 *   NQ_ECHECKPOINT (-5) unreadable / corrupt / foreign checkpoint ~ nqueens::checkpoint_error
 *
 * There is no CPU fallback: every counting entry point runs the sm_100a kernels and
 * fails with NQ_ECUDA when no device is usable.
 */
#ifndef NQ_GPU_H
#define NQ_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NQ_OK 0
#define NQ_ECUDA (-1)
#define NQ_ECONFIG (-2)
#define NQ_EOVERFLOW (-3)
#define NQ_ECANCEL (-4)
#define NQ_ECHECKPOINT (-5)

#define NQ_ABI_VERSION 2

/* Packed 16-byte frontier record (one LDG.128 per refill on the device).
 *   cols      occupied columns of the first placed_rows rows   (Subproblem::cur)
 *   diag      left-diagonal threats shifted to the next row    (Subproblem::left)
 *   antidiag  right-diagonal threats shifted to the next row   (Subproblem::right)
 *   row       placed_rows | multiplier << 8                    (Subproblem::placed_rows,
 *                                                              Subproblem::multiplier)
 * Reference struct: solver.hpp:18-26 (20 bytes, int fields). */
typedef struct nq_sub {
  uint32_t cols, diag, antidiag, row;
} nq_sub;

/* Kernel variants of solver.hpp:28 (KernelVariant). Both run the same sm_100a DFS; the
 * variant selects the feasibility rule (required_depth, stack_config.hpp:43-45) and
 * which loop the reported node count follows (Alg. 2 or Alg. 3 iterations). */
#define NQ_VARIANT_ITERATIVE 0
#define NQ_VARIANT_LASTROW 1

typedef struct nq_result {
  uint64_t solutions;       /* Σ multiplier × count (checked on the host)           */
  uint64_t raw_solutions;   /* Σ count, unweighted                                   */
  uint64_t nodes;           /* DFS nodes: Alg. 3 (last-row) loop iterations           */
  uint64_t iterations;      /* device loop iterations actually executed               */
  uint64_t subproblems;     /* records processed                                      */
  double kernel_ms;         /* device time of the counting kernel(s), CUDA events     */
  double h2d_ms;            /* host→device copy time (0 for device-resident input)    */
} nq_result;

typedef struct nq_ctx nq_ctx; /* one per device; used by one host thread at a time */

int nq_abi_version(void);
const char* nq_last_error(void);
int nq_device_count(int* out);

/* --- per-device contexts --------------------------------------------------------- */
int nq_ctx_create(int device, nq_ctx** out);
void nq_ctx_destroy(nq_ctx* ctx);
/* Tuning knobs (0 = default): threads per block, resident blocks per SM cap,
 * dispatch order (0 = as given, 1 = reversed: the expensive tail of the DFS order
 * first). */
int nq_ctx_set_tuning(nq_ctx* ctx, int block, int blocks_per_sm, int reverse_order);
/* Shared-memory stack layout of the DFS kernel:
 *   NQ_LAYOUT_V4      one 16-byte frame per LDS.128/STS.128 (default, fastest);
 *   NQ_LAYOUT_PLANES  four 32-bit planes, lane t owns bank t: zero bank conflicts for
 *                     any set of active lanes, four memory instructions per push/pop. */
#define NQ_LAYOUT_V4 0
#define NQ_LAYOUT_PLANES 1
int nq_ctx_set_layout(nq_ctx* ctx, int layout);
/* Tail balancing (default on): once the dispatch queue is empty, an idle lane takes the
 * shallowest pending frame of a busy lane in its warp (the largest remaining subtree),
 * so one skewed subproblem no longer leaves 31 lanes idle. Totals are unchanged; off
 * only for A/B measurements. (count_each never splits a record.) */
int nq_ctx_set_balance(nq_ctx* ctx, int donate);
/* Host cancel flag (may be NULL) polled while a synchronous call waits: once it reads
 * non-zero, the running kernel stops handing out records at its next refill (lanes
 * finish the subtree they hold), and the call returns with result.subproblems below the
 * batch size — the per-subproblem cancel granularity of execute_batch
 * (scheduler.hpp:342-355). */
int nq_ctx_set_cancel(nq_ctx* ctx, const volatile int* cancel);

/* Count a batch held in HOST memory (caller-owned, pageable or pinned). Synchronous.
 * A pinned (page-locked) batch is read in place by the kernel over the bus, each record
 * once (no copy; NQB_ZERO_COPY=0 disables this); a pageable one is copied first. The
 * same holds for nq_solve_batch's host batch.
 * The GPU analogue of execute_batch's per-worker loop (scheduler.hpp:319-326).
 * pre_rows is the batch's pre-placement depth R: it sizes the shared-memory stack
 * (n-1-R frames, the Alg. 3 depth of stack_config.hpp:43-45); a record with fewer
 * placed rows than R, cols outside the board, or popcount(cols) != placed_rows is
 * rejected with NQ_ECONFIG naming its index. */
int nq_count(nq_ctx* ctx, int n, int pre_rows, int variant, const nq_sub* host_subs,
             uint64_t count, nq_result* out);
/* Count a batch already resident in device memory of ctx's device. Synchronous. */
int nq_count_device(nq_ctx* ctx, int n, int pre_rows, int variant, const nq_sub* dev_subs,
                    uint64_t count, nq_result* out);
/* Asynchronous form of nq_count_device: enqueue on the context stream; nq_collect
 * waits and fills out. At most one batch in flight per context. */
int nq_count_device_async(nq_ctx* ctx, int n, int pre_rows, int variant,
                          const nq_sub* dev_subs, uint64_t count);
int nq_collect(nq_ctx* ctx, nq_result* out);

/* GPU-side frontier deepening: `count` DEVICE-resident roots (on
 * `device`) deepened to target_rows in nq_expand's order, written to dev_out (capacity
 * cap; NULL = count only); *total = number of deepened records. Synchronous. */
int nq_expand_device(int device, int n, const nq_sub* dev_roots, uint64_t count,
                     int target_rows, nq_sub* dev_out, uint64_t cap, uint64_t* total);
/* Host roots (a coarse frontier, e.g. R0 = 4) -> H2D -> deepened on the device to
 * target_rows -> counted by the DFS kernel; only the coarse records cross PCIe.
 * result->subproblems counts the deepened records. */
int nq_count_expand(nq_ctx* ctx, int n, int target_rows, int variant, const nq_sub* host_roots,
                    uint64_t count, nq_result* out);

/* Per-subproblem results (unweighted counts, high-water marks as in
 * KernelResult, solver.hpp:34-41, and Alg. 3 node counts). Host buffers. This is the
 * count_with seam (solver.hpp:193) batched onto the device. */
int nq_count_each(nq_ctx* ctx, int n, int pre_rows, int variant, const nq_sub* host_subs,
                  uint64_t count, uint64_t* counts, int32_t* high_water, uint64_t* nodes);

/* --- frontier (host C++, multi-threaded, deterministic reference order) ------------ */
/* subproblems.hpp:80-115. out may be NULL (count only); writes min(cap, total). */
int nq_generate(int n, int pre_rows, nq_sub* out, uint64_t cap, uint64_t* total);
/* Systematic slice of the same stream: records with index ≡ offset (mod stride). */
int nq_generate_slice(int n, int pre_rows, uint64_t stride, uint64_t offset, nq_sub* out,
                      uint64_t cap, uint64_t* total);
/* subproblems.hpp:118-145 */
int nq_count_subproblems(int n, int pre_rows, uint64_t* total);
/* Deepens `count` roots to target_rows placed rows (expand_rows, subproblems.hpp:41-55,
 * applied per root, multiplier inherited; roots already that deep are copied). out may
 * be NULL (count only); writes min(cap, total). Cuts deep frontiers into GPU-sized
 * records, e.g. a systematic N=27/R=7 slice expanded to R=10 for the projection. */
int nq_expand(int n, const nq_sub* roots, uint64_t count, int target_rows, nq_sub* out,
              uint64_t cap, uint64_t* total);

/* --- partitions (scheduler.hpp:61-102) ----------------------------------------------- */
/* ranges receives worker_count (first, last) pairs. */
int nq_partition_uniform(uint64_t task_count, int worker_count, uint64_t* ranges);
int nq_partition_weighted(uint64_t task_count, const double* weights, int worker_count,
                          uint64_t* ranges);

/* --- multi-GPU execution (scheduler.hpp:266 / :573) --------------------------------
 * One host thread per worker; worker w runs on devices[w % G] with its own pooled
 * context (workers that share a device get distinct ones). Under the dynamic strategies
 * each worker runs ONE persistent streaming launch and publishes the chunks it takes
 * from the dispenser into it while it runs: no launch or end-of-launch tail per chunk. */
#define NQ_PARTITION_UNIFORM 0  /* PartitionStrategy::uniform  (scheduler.hpp:26)        */
#define NQ_PARTITION_WEIGHTED 1 /* PartitionStrategy::weighted                          */
#define NQ_PARTITION_STEALING 2 /* PartitionStrategy::stealing: fixed chunks, cursor    */
#define NQ_PARTITION_GUIDED 3   /* shrinking chunks, expensive end first; the default    */
                                /* when opts == NULL (one streaming launch per device)   */
#define NQ_PARTITION_STRIDED 4  /* record i -> worker i mod W, one launch per worker     */

#define NQ_LOG_GENERATION 0 /* "Use %.2fms to generate %llu subproblems!"               */
#define NQ_LOG_START 1      /* "worker [%d] start job, with %llu(%.2f) subproblems."     */
#define NQ_LOG_FINISH 2     /* "worker [%d] finish job."                                 */
#define NQ_LOG_RESULT 3     /* "n %d queens result %llu, calc time: [%.2f ms]"           */

/* Formats one timestamped log line of scheduler.hpp:163-203 into buf (NUL-terminated).
 * kind NQ_LOG_GENERATION: (ms, count); START: (worker, count, fraction);
 * FINISH: (worker); RESULT: (n, total, ms). Unused arguments are ignored. */
int nq_format_log(int kind, int i, uint64_t u, double d, char* buf, uint64_t cap);

typedef void (*nq_log_fn)(void* user, const char* line);

/* --- host-side dynamic chunk dispenser (scheduler.hpp:351-362) --------------------- *
 * The cursor the dynamic strategies draw chunks from. In one process the scheduler makes
 * its own; a NAMED dispenser lives in a POSIX shared-memory segment, so that cooperating
 * processes on one node (e.g. one per GPU under torchrun) share ONE dynamic dispatch —
 * host-side, lock-free, no device collective. strategy: NQ_PARTITION_STEALING (fixed
 * chunks, stream order) or NQ_PARTITION_GUIDED (max(min(remaining / 2W, count / 16W),
 * floor) records from the expensive end; chunk = floor, 0 = count / (128 W)). Each process posts its partial
 * into its own slot; nq_dispatch_sum adds the slots (checked). */
typedef struct nq_dispatch nq_dispatch;
int nq_dispatch_create(const char* shm_name /* NULL = in-process */, uint64_t count, int strategy,
                       uint64_t chunk, int workers, nq_dispatch** out);
int nq_dispatch_attach(const char* shm_name, nq_dispatch** out);
void nq_dispatch_close(nq_dispatch* d, int unlink_segment);
/* 1 = [*first, *first + *len) is this caller's, 0 = drained, < 0 = error. */
int nq_dispatch_take(nq_dispatch* d, uint64_t* first, uint64_t* len);
int nq_dispatch_reset(nq_dispatch* d); /* start a new pass over the same records */
int nq_dispatch_info(const nq_dispatch* d, uint64_t* count, int* strategy, uint64_t* chunk,
                     int* workers);
int nq_dispatch_post(nq_dispatch* d, int slot, uint64_t solutions, uint64_t nodes,
                     uint64_t processed);
int nq_dispatch_sum(nq_dispatch* d, int slots, uint64_t* solutions, uint64_t* nodes,
                    uint64_t* processed);

typedef struct nq_solve_opts {
  int variant;                 /* NQ_VARIANT_*                                          */
  int strategy;                /* NQ_PARTITION_*                                        */
  int worker_count;            /* workers; 0 = one per device. Worker w runs on          */
                               /* devices[w % n_devices] with its own stream             */
  const double* weights;       /* weighted: worker_count weights (NULL = equal)          */
  uint64_t chunk;              /* stealing: records per chunk; guided: minimum chunk     */
  int n_devices;               /* 0 = all visible                                        */
  const int* devices;          /* optional explicit device list (length n_devices)       */
  const volatile int* cancel;  /* non-zero → stop between chunks (completed = 0)         */
  int stack_depth;             /* StackConfig::max_depth() of the caller's config; 0 = off */
  const char* config_name;     /* for the require_feasible message                        */
  nq_log_fn log;               /* optional start/finish line sink (called concurrently) */
  void* log_user;
  nq_dispatch* dispatch;       /* stealing / guided: draw chunks from this (possibly shared) */
                               /* dispenser instead of a private one; its count, strategy */
                               /* and chunk win                                            */
} nq_solve_opts;

#define NQ_MAX_WORKERS 64

typedef struct nq_worker_stats {
  int worker;
  int device;
  uint64_t assigned;           /* contiguous strategies: range size; 0 = dynamic        */
  uint64_t processed;          /* records counted by this worker                        */
  uint64_t partial_sum;        /* multiplier-weighted (checked)                         */
  uint64_t nodes;              /* Alg. 3 nodes                                          */
  uint64_t chunks;             /* chunks / ranges counted                               */
  double elapsed_ms;           /* host wall time of this worker thread                  */
  double kernel_ms;            /* Σ device time of its launches (they may overlap)      */
  double span_ms;              /* device time from its first enqueued operation to the  */
                               /* end of its last kernel (CUDA events, one device)       */
  uint64_t launches;           /* kernel launches (dynamic strategies: one streaming    */
                               /* launch fed all of the worker's chunks)                 */
} nq_worker_stats;

typedef struct nq_report {
  uint64_t total;              /* multiplier-weighted solution count                    */
  uint64_t task_count;
  uint64_t nodes;
  double generation_ms;
  double calc_ms;              /* wall time of the device phase (excl. generation)      */
  int completed;
  int worker_count;
  nq_worker_stats workers[NQ_MAX_WORKERS];
} nq_report;

int nq_solve_batch(int n, int pre_rows, const nq_sub* host_subs, uint64_t count,
                   const nq_solve_opts* opts, nq_report* out);
int nq_solve(int n, int pre_rows, const nq_solve_opts* opts, nq_report* out);
/* execute_batch over a frontier already RESIDENT on every device: dev_subs[i] is a full
 * copy of the count records on the i-th device of the worker device list (opts->devices,
 * or 0..n_devices-1). Workers launch on sub-ranges of their device's copy, so only the
 * 64-byte results cross PCIe. Strategies: uniform, weighted, stealing, guided. */
int nq_solve_batch_device(int n, int pre_rows, const nq_sub* const* dev_subs, uint64_t count,
                          const nq_solve_opts* opts, nq_report* out);
/* execute_batch over host ROOTS that each worker deepens to target_rows on its device
 * before counting (only the roots cross PCIe; strided or guided, or any strategy with
 * one worker). The totals equal
 * execute_batch over the deepened records; report.workers[].processed counts deepened
 * records. This is how execute() runs large frontiers and how a systematic slice of
 * the N=27 R=7 frontier is cut into GPU-sized records for the projection. */
int nq_solve_batch_expand(int n, int target_rows, const nq_sub* roots, uint64_t count,
                          const nq_solve_opts* opts, nq_report* out);

/* --- checkpoint / resume (runner.hpp:48-212, checkpoint.hpp:21-199) -- */
typedef struct nq_ckpt_opts {
  const char* path;          /* checkpoint file; rewritten atomically (tmp + rename)      */
  uint64_t chunk;            /* records per chunk; 0 = ceil(tasks / 256) (or the file's)  */
  double flush_interval_s;   /* rewrite at most this often; 0 = after every chunk         */
  int resume;                /* 1 = continue the run recorded in path                     */
  double stop_after_s;       /* >0: start no new chunk after this many seconds (the       */
                             /* running ones finish and are recorded); 0 = no limit      */
} nq_ckpt_opts;

/* execute() with chunk-granular progress: the folded frontier is cut into fixed chunks
 * (emitted one at a time, never materialised whole: host memory = workers x chunk);
 * workers (opts->worker_count, devices as in nq_solve_batch) take pending chunks from an
 * atomic cursor, expensive end first; every finished chunk is recorded (weighted sum,
 * nodes). A cancel discards only the chunk in flight; completed = 0 until every chunk is
 * recorded. Resume validates the file (checksum, identity of n, R, variant, chunk, task
 * count) before touching a device and recounts only the missing chunks. */
int nq_solve_checkpointed(int n, int pre_rows, const nq_solve_opts* opts,
                          const nq_ckpt_opts* ck, nq_report* out);
/* Reads a checkpoint's run parameters and progress (for `resume <file>`). */
int nq_checkpoint_read(const char* path, int* n, int* pre_rows, uint64_t* chunks,
                       uint64_t* done_chunks);
/* The same plus the kernel variant and chunk size the run was started with (a resume
 * must repeat them: they are part of the file's identity). Any pointer may be NULL. */
int nq_checkpoint_info(const char* path, int* n, int* pre_rows, int* variant, uint64_t* chunk,
                       uint64_t* chunks, uint64_t* done_chunks);

/* --- diagnostics ------------------------------------------------------------------- */
/* Integer-pipe peak of the current device (LOP3+IMAD 1:1 stream, all SMs), thread
 * ops/s and the SM clock seen; the roofline denominator of bench.py. */
int nq_measure_int_peak(int device, double* ops_per_s, double* sm_mhz);

#ifdef __cplusplus
}
#endif
#endif
