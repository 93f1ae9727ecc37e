/*
 * nq_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's N-Queens counting path
 * (/root/reference/proj/include/nqueens/{bitboard,solver,subproblems,scheduler}.hpp),
 * used as the CPU checker for the B200 kernels. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it. The product path
 * (paper_2511_12009_b200/, include/) never links or calls it.
 *
 * Parity pinning: every function here is checked against (a) the golden vectors the
 * reference's own tests hold (test_solver.cpp, test_subproblems.cpp,
 * test_scheduler.cpp, acceptance.cpp — restated in tests/golden/), and (b) the
 * reference headers themselves, compiled from /root/reference into oracle/_ref/ by
 * oracle/Makefile (tests/test_oracle.py::test_oracle_matches_reference_build).
 *
 * Status codes: 0 ok, NQO_ECONFIG (-2) ~ nqueens::config_error,
 * NQO_EOVERFLOW (-3) ~ std::overflow_error.
 */
#ifndef NQ_ORACLE_H
#define NQ_ORACLE_H

#include <stddef.h>
#include <stdint.h>
#include <stdio.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NQO_OK 0
#define NQO_ECONFIG (-2)
#define NQO_EOVERFLOW (-3)

/* Same 16-byte packed record the product uses (include/nq_gpu.h):
 * row = placed_rows | multiplier << 8. */
typedef struct {
  uint32_t cols, diag, antidiag, row;
} nqo_sub;

uint32_t nqo_board_mask(int n);
uint32_t nqo_valid_positions(uint32_t cur, uint32_t left, uint32_t right, int n);

/* solver.hpp:50-72 — Alg. 1, plain recursion; multiplier not applied. */
int nqo_count_recursive(int n, uint32_t cur, uint32_t left, uint32_t right, uint64_t* count);
/* solver.hpp:79-130 — Alg. 2; stack_depth = StackConfig::max_depth() of the config. */
int nqo_count_iterative(int n, const nqo_sub* sub, int stack_depth, uint64_t* count,
                        int* high_water);
/* solver.hpp:138-191 — Alg. 3 (last row by popcount). nodes = loop iterations,
 * the DFS-node unit of the metric. */
int nqo_count_lastrow(int n, const nqo_sub* sub, int stack_depth, uint64_t* count,
                      int* high_water, uint64_t* nodes);

/* subproblems.hpp:80-108 — folded frontier, deterministic order. Writes at most cap
 * records (out may be NULL to count only); *total gets the full stream length. */
int nqo_generate(int n, int pre_rows, nqo_sub* out, uint64_t cap, uint64_t* total);
/* subproblems.hpp:118-145 */
int nqo_count_subproblems(int n, int pre_rows, uint64_t* total);
/* subproblems.hpp:149-165 — Σ multiplier·count with duplicate-state rejection. */
int nqo_aggregate(const nqo_sub* subs, const uint64_t* counts, uint64_t len, uint64_t* total);
/* subproblems.hpp:169-178 — text export, one line per subproblem. */
int nqo_write_batch(int n, int pre_rows, FILE* out, uint64_t* lines);

/* scheduler.hpp:61-102 — contiguous partitions. ranges = 2*workers u64 (first,last). */
int nqo_partition_uniform(uint64_t task_count, int workers, uint64_t* ranges);
int nqo_partition_weighted(uint64_t task_count, const double* weights, int workers,
                           uint64_t* ranges);

/* scheduler.hpp:266-389 restated as a pthread pool with the stealing cursor
 * (scheduler.hpp:356-361): lastrow kernel per subproblem, multiplier-weighted checked
 * sum. Used as the CPU baseline ("port") and to pin node counts. */
int nqo_solve_batch(int n, const nqo_sub* subs, uint64_t len, int threads, uint64_t chunk,
                    uint64_t* total, uint64_t* nodes, uint64_t* per_sub_counts);

const char* nqo_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
