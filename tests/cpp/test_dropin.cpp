// test_dropin.cpp — the reference's doctest assertions for the counting path, restated
// against the drop-in C++ headers (include/nqueens/*.hpp) linked to libnqb200.so.
//
//   ./test_dropin cpu   host-side cases only (frontier, partitions, logs, errors)
//   ./test_dropin gpu   every case, including counting on the B200
//
// Each case names the reference test it restates (/root/reference/proj/tests/…).
// The independent checkers below (permutation count, attack check, unfolded
// enumeration) are test-only code written for this file.
#include <algorithm>
#include <atomic>
#include <bit>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <map>
#include <mutex>
#include <numeric>
#include <random>
#include <regex>
#include <set>
#include <sstream>
#include <string>
#include <tuple>
#include <vector>

#include "nqueens/nqueens.hpp"

using namespace nqueens;

namespace {

int g_checks = 0, g_failures = 0;
const char* g_case = "";

#define CHECK(cond)                                                                     \
  do {                                                                                  \
    ++g_checks;                                                                         \
    if (!(cond)) {                                                                      \
      ++g_failures;                                                                     \
      std::fprintf(stderr, "FAIL [%s] %s:%d: %s\n", g_case, __FILE__, __LINE__, #cond); \
    }                                                                                   \
  } while (0)

#define CHECK_THROWS_AS(expr, type)                                                     \
  do {                                                                                  \
    ++g_checks;                                                                         \
    bool thrown_ = false;                                                               \
    try {                                                                               \
      (void)(expr);                                                                     \
    } catch (const type&) {                                                             \
      thrown_ = true;                                                                   \
    } catch (...) {                                                                     \
    }                                                                                   \
    if (!thrown_) {                                                                     \
      ++g_failures;                                                                     \
      std::fprintf(stderr, "FAIL [%s] %s:%d: %s does not throw %s\n", g_case, __FILE__, \
                   __LINE__, #expr, #type);                                             \
    }                                                                                   \
  } while (0)

// ---- independent checkers ----------------------------------------------------------------
std::uint64_t permutations_count(int n) {  // Q(n) by filtering column permutations
  std::vector<int> p(n);
  std::iota(p.begin(), p.end(), 0);
  std::uint64_t q = 0;
  do {
    bool ok = true;
    for (int i = 0; i < n && ok; ++i)
      for (int j = i + 1; j < n && ok; ++j) ok = std::abs(p[i] - p[j]) != j - i;
    q += ok;
  } while (std::next_permutation(p.begin(), p.end()));
  return q;
}

// Every reachable partial placement with exactly `rows` queens, as row -> column lists.
void partials(int n, int rows, std::vector<int>& cols, const std::function<void(const std::vector<int>&)>& f) {
  if (static_cast<int>(cols.size()) == rows) {
    f(cols);
    return;
  }
  const int row = static_cast<int>(cols.size());
  for (int c = 0; c < n; ++c) {
    bool ok = true;
    for (int r = 0; r < row && ok; ++r) ok = cols[r] != c && std::abs(cols[r] - c) != row - r;
    if (!ok) continue;
    cols.push_back(c);
    partials(n, rows, cols, f);
    cols.pop_back();
  }
}

// Root state of a partial placement, built square by square (no bitboard shifts).
Subproblem root_of(const std::vector<int>& cols, int n) {
  Subproblem s{};
  const int row = static_cast<int>(cols.size());
  for (int r = 0; r < row; ++r) {
    s.cur |= bit_mask{1} << cols[r];
    const int dl = cols[r] + (row - r);  // left diagonal reaches column cols+Δ
    const int dr = cols[r] - (row - r);
    if (dl < 32) s.left |= bit_mask{1} << dl;
    if (dr >= 0) s.right |= bit_mask{1} << dr;
  }
  (void)n;
  s.placed_rows = row;
  s.multiplier = 1;
  return s;
}

std::uint64_t unfolded_total(int n, int r) {  // Σ over every unfolded root of its count
  std::uint64_t t = 0;
  std::vector<int> cols;
  partials(n, r, cols, [&](const std::vector<int>& c) { t += count_recursive(n, root_of(c, n)); });
  return t;
}

std::uint64_t folded_total(int n, int r) {  // Σ multiplier × count over the folded stream
  std::uint64_t t = 0;
  for_each_subproblem({n, r}, [&](const Subproblem& s) {
    t = checked_add(t, checked_mul(static_cast<std::uint64_t>(s.multiplier), count_recursive(n, s)));
  });
  return t;
}

const std::uint64_t kOeis[] = {1, 0, 0, 2, 10, 4, 40, 92, 352, 724, 2680, 14200, 73712,
                               365596, 2279184, 14772512, 95815104, 666090624};

// ---- host-side cases --------------------------------------------------------------------
void bitboard_cases() {  // test_bitboard.cpp:13-95
  g_case = "bitboard";
  CHECK(valid_positions(0, 0, 0, 4) == 0b1111);
  CHECK(valid_positions(0b0001, 0b0010, 0, 4) == 0b1100);
  for (std::uint32_t m = 1; m < (1u << 16); ++m) CHECK(lowest_set_bit(m) == (m & (~m + 1u)));
  const auto s = apply_placement(0, 0, 0, 0b100);
  CHECK(s.cur == 0b100);
  CHECK(s.left == 0b1000);
  CHECK(s.right == 0b10);
  CHECK(apply_placement(0, 0x80000000u, 0, 1).left == 2);  // 32-bit truncation
  CHECK(board_mask(32) == 0xffffffffu);
  CHECK(board_mask(5) == 0x1fu);
  // every reachable n=8 state against the square-by-square attack check
  for (int r = 0; r < 8; ++r) {
    std::vector<int> cols;
    partials(8, r, cols, [&](const std::vector<int>& c) {
      const Subproblem root = root_of(c, 8);
      bit_mask allowed = 0;
      for (int col = 0; col < 8; ++col) {
        bool ok = true;
        for (int i = 0; i < r && ok; ++i) ok = c[i] != col && std::abs(c[i] - col) != r - i;
        if (ok) allowed |= bit_mask{1} << col;
      }
      CHECK(valid_positions(root.cur, root.left, root.right, 8) == allowed);
    });
  }
}

void config_cases() {  // test_solver.cpp:16-57, 144-154
  g_case = "stack_config";
  CHECK(builtin_configs.size() == 5);
  CHECK(builtin_configs[0].max_depth() == 24);
  CHECK(builtin_configs[1].max_depth() == 19);
  CHECK(builtin_configs[2].max_depth() == 16);
  CHECK(builtin_configs[3].max_depth() == 12);
  CHECK(builtin_configs[4].max_depth() == 6);
  CHECK(find_config("config3") == &builtin_configs[2]);
  CHECK(find_config("nope") == nullptr);
  try {
    require_feasible(builtin_configs[4], 22, 6, true);
    CHECK(false);
  } catch (const config_error& e) {
    const std::string w = e.what();
    CHECK(w.find("needs 15") != std::string::npos);
    CHECK(w.find("smallest sufficient config is 'config3'") != std::string::npos);
  }
  CHECK_THROWS_AS(require_feasible(builtin_configs[0], 32, 1, false), config_error);
  CHECK_THROWS_AS(checked_add(~0ull, 1), std::overflow_error);
  CHECK_THROWS_AS(checked_mul(~0ull, 2), std::overflow_error);
  CHECK(checked_add(2, 3) == 5);
  CHECK(checked_mul(2, 3) == 6);
  CHECK_THROWS_AS(count_recursive(0, {}), config_error);
  CHECK_THROWS_AS(count_recursive(33, {}), config_error);
}

void frontier_cases() {  // test_subproblems.cpp:34-150
  g_case = "frontier";
  const auto b1 = generate({5, 1});
  CHECK(b1.size() == 3);
  if (b1.size() == 3) {
    CHECK(b1[0].cur == 0b00001 && b1[0].multiplier == 2);
    CHECK(b1[1].cur == 0b00010 && b1[1].multiplier == 2);
    CHECK(b1[2].cur == 0b00100 && b1[2].multiplier == 1);
  }
  for (const auto& s : b1) CHECK(s.placed_rows == 1);

  const auto b2 = generate({5, 2});
  CHECK(b2.size() == 6);
  std::set<std::tuple<bit_mask, bit_mask, bit_mask>> states;
  std::vector<int> cols;
  partials(5, 2, cols, [&](const std::vector<int>& c) {
    const Subproblem s = root_of(c, 5);
    states.insert({s.cur, s.left, s.right});
  });
  for (const auto& s : b2) {
    CHECK(s.placed_rows == 2);
    CHECK(states.count({s.cur, s.left, s.right}) == 1);
  }
  if (!b2.empty()) CHECK(b2.back().multiplier == 2);

  for (int n : {6, 9, 11})
    for (int r = 1; r <= 3; ++r) {
      const auto batch = generate({n, r});
      std::set<std::tuple<bit_mask, bit_mask, bit_mask, int>> seen;
      for (const auto& s : batch) {
        CHECK(std::popcount(s.cur) == s.placed_rows);
        CHECK(s.multiplier == 1 || s.multiplier == 2);
        CHECK(seen.insert({s.cur, s.left, s.right, s.placed_rows}).second);
        if (n % 2 == 0 || r > 1) CHECK(s.multiplier == 2);
      }
      CHECK(generate({n, r}) == batch);
    }

  CHECK(count_subproblems(5, 1) == 3);
  for (int n : {5, 8, 9, 12})
    for (int r = 1; r <= 4 && r < n; ++r) CHECK(count_subproblems(n, r) == generate({n, r}).size());
  CHECK(count_subproblems(27, 7) == 453688251ull);  // acceptance.cpp:77-89
  CHECK(kQueens27Reference == 234907967154122528ull);  // acceptance.cpp:234-239

  std::uint64_t streamed = 0;
  for_each_subproblem({12, 4}, [&](const Subproblem&) { ++streamed; });
  CHECK(streamed == count_subproblems(12, 4));

  CHECK_THROWS_AS(generate({5, 0}), config_error);
  CHECK_THROWS_AS(generate({5, 5}), config_error);
  CHECK_THROWS_AS(generate({1, 1}), config_error);
  CHECK_THROWS_AS(generate({12, 9}), config_error);
  CHECK_THROWS_AS(generate({40, 2}), config_error);

  std::ostringstream out;
  CHECK(write_batch(out, {5, 1}) == 3);
  CHECK(out.str() == "0 1 2 0 1 2\n1 2 4 1 1 2\n2 4 8 2 1 1\n");
  std::ostringstream wide;
  write_batch(wide, {14, 1});
  CHECK(wide.str().substr(0, wide.str().find('\n')) == "0 1 2 0 1 2");
  CHECK(wide.str().find("6 40 80 20 1 2") != std::string::npos);

  std::vector<std::pair<Subproblem, std::uint64_t>> none;
  CHECK(aggregate(none) == 0);
  std::vector<std::pair<Subproblem, std::uint64_t>> dup = {{Subproblem{1, 2, 0, 1, 2}, 3},
                                                          {Subproblem{1, 2, 0, 1, 2}, 3}};
  CHECK_THROWS_AS(aggregate(dup), config_error);
  std::vector<std::pair<Subproblem, std::uint64_t>> huge = {{Subproblem{1, 2, 0, 1, 2}, ~0ull / 2 + 1}};
  CHECK_THROWS_AS(aggregate(huge), std::overflow_error);
  // the duplicate key is the reference's 64-bit multiply-xor mix (subproblems.hpp:154-157),
  // the same values the Python mirror computes
  CHECK(detail::state_key(Subproblem{5, 8, 2, 2, 1}) == 0x23c15acef1ad0341ull);
  CHECK(detail::state_key(Subproblem{0x1f, 0x40, 0x3, 5, 1}) == 0x9f661b1922370771ull);
}

void partition_cases() {  // test_scheduler.cpp:27-75, 132-147
  g_case = "partition";
  const auto u = partition_uniform(10, 3);
  CHECK(u.size() == 3 && u[0].size() == 4 && u[1].size() == 3 && u[2].size() == 3);
  CHECK(u[2].last == 10);
  const auto w = partition_weighted(100, {0.5, 0.25, 0.25});
  CHECK(w[0].size() == 50 && w[1].size() == 25 && w[2].size() == 25);
  const auto pw = partition_weighted(
      1000, std::vector<double>(paper_gpu_weights.begin(), paper_gpu_weights.end()));
  CHECK(pw[0].size() == 200 && pw[7].last == 1000);
  CHECK_THROWS_AS(partition_uniform(5, 0), config_error);
  CHECK_THROWS_AS(partition_weighted(5, {}), config_error);
  CHECK_THROWS_AS(partition_weighted(5, {1.0, 0.0}), config_error);
  std::mt19937_64 rng(7);
  for (int t = 0; t < 2000; ++t) {
    const std::uint64_t tasks = rng() % 10000;
    const int workers = 1 + static_cast<int>(rng() % 16);
    std::vector<double> ws(workers);
    for (auto& x : ws) x = 0.01 + (rng() % 1000) / 1000.0;
    for (const auto& ranges : {partition_uniform(tasks, workers), partition_weighted(tasks, ws)}) {
      std::uint64_t at = 0;
      for (const auto& r : ranges) {
        CHECK(r.first == at);
        at = r.last;
      }
      CHECK(at == tasks);
    }
  }
  CHECK(partition_strategy_from("stealing") == PartitionStrategy::stealing);
  CHECK(std::string(to_string(PartitionStrategy::weighted)) == "weighted");
  CHECK_THROWS_AS(partition_strategy_from("random"), config_error);

  const std::regex ts(R"(^\[\d{4}-\d{2}-\d{2} \d{2}:\d{2}:\d{2}\.\d{3}\] )");
  CHECK(std::regex_search(log_generation_line(1.5, 42), ts));
  CHECK(log_generation_line(1.5, 42).find("Use 1.50ms to generate 42 subproblems!") != std::string::npos);
  CHECK(log_start_line(3, 7, 0.25).find("worker [3] start job, with 7(0.25) subproblems.") != std::string::npos);
  CHECK(log_finish_line(2).find("worker [2] finish job.") != std::string::npos);
  const std::regex result(R"(n (\d+) queens result (\d+), calc time: \[([0-9.]+) ms\])");
  std::smatch m;
  const std::string line = log_result_line(8, 92, 12.345);
  CHECK(std::regex_search(line, m, result) && m[1] == "8" && m[2] == "92" && m[3] == "12.35");
  CHECK(std::regex_match(log_timestamp(), std::regex(R"(\[\d{4}-\d{2}-\d{2} \d{2}:\d{2}:\d{2}\.\d{3}\])")));

  ExecuteOptions bad;
  bad.plan.worker_count = 0;
  CHECK_THROWS_AS(execute_batch(8, 2, generate({8, 2}), bad), config_error);
  ExecuteOptions chunk0;
  chunk0.plan.strategy = PartitionStrategy::stealing;
  chunk0.plan.chunk_size = 0;
  CHECK_THROWS_AS(execute_batch(8, 2, generate({8, 2}), chunk0), config_error);
  ExecuteOptions shallow;
  shallow.config = builtin_configs[4];
  CHECK_THROWS_AS(execute_batch(14, 2, generate({14, 2}), shallow), config_error);
  ExecuteOptions resume;
  resume.resume = {WorkerProgress{}};
  CHECK_THROWS_AS(execute_batch(8, 2, generate({8, 2}), resume), config_error);
}

// ---- device cases -----------------------------------------------------------------------
void solver_cases() {  // test_solver.cpp:59-142
  g_case = "solver";
  const StackConfig& cfg1 = builtin_configs[0];
  CHECK(count_recursive(1, {}) == 1);
  CHECK(count_recursive(2, {}) == 0);
  CHECK(count_recursive(3, {}) == 0);
  for (int n = 1; n <= 9; ++n) CHECK(count_recursive(n, {}) == permutations_count(n));
  for (int n = 4; n <= 12; ++n)
    for (int r = 1; r <= 3 && r < n; ++r)
      for (const Subproblem& s : generate({n, r})) {
        const auto it = count_iterative(n, s, cfg1);
        CHECK(it.count == count_recursive(n, s));
        CHECK(count_iterative_lastrow(n, s, cfg1).count == it.count);
      }
  const Subproblem full = root_of({0, 2, 4, 1, 3}, 5);
  CHECK(full.cur == board_mask(5));
  CHECK(count_iterative(5, full, cfg1).count == 1);
  CHECK(count_iterative_lastrow(5, full, cfg1).count == 1);
  CHECK(count_iterative_lastrow(4, {}, cfg1).count == 2);
  CHECK(count_iterative_lastrow(1, {}, cfg1).count == 1);
  std::vector<int> cols;
  partials(6, 5, cols, [&](const std::vector<int>& c) {
    const Subproblem s = root_of(c, 6);
    CHECK(count_iterative_lastrow(6, s, cfg1).count == count_recursive(6, s));
  });
  for (int n : {8, 10})
    for (int r : {1, 2, 3}) {
      int best_it = 0, best_lr = 0;
      std::vector<int> c0;
      partials(n, r, c0, [&](const std::vector<int>& c) {
        const Subproblem s = root_of(c, n);
        const auto it = count_iterative(n, s, cfg1);
        const auto lr = count_iterative_lastrow(n, s, cfg1);
        CHECK(it.high_water <= n - r);
        CHECK(lr.high_water <= n - r - 1);
        best_it = std::max(best_it, it.high_water);
        best_lr = std::max(best_lr, lr.high_water);
      });
      CHECK(best_it == n - r);
      CHECK(best_lr == n - r - 1);
    }
  const Subproblem d = root_of({1, 3}, 11);
  const auto a = count_iterative(11, d, cfg1), b = count_iterative(11, d, cfg1);
  CHECK(a.count == b.count && a.high_water == b.high_water);
}

void fold_cases() {  // test_subproblems.cpp:80-110, :120-124
  g_case = "fold";
  for (int n = 2; n <= 11; ++n)
    for (int r = 1; r <= 3 && r < n; ++r) CHECK(folded_total(n, r) == unfolded_total(n, r));
  for (int n : {8, 11})
    for (int r = 2; r <= 5; ++r) CHECK(folded_total(n, r) == folded_total(n, 1));
  CHECK(folded_total(3, 2) == 0);
  std::vector<std::pair<Subproblem, std::uint64_t>> res;
  for (const Subproblem& s : generate({5, 1})) res.emplace_back(s, count_recursive(5, s));
  CHECK(aggregate(res) == 10);
}

void execute_cases() {  // test_scheduler.cpp:77-171, acceptance.cpp:60-75
  g_case = "execute";
  for (int n = 1; n <= 16; ++n) {
    ExecuteOptions o;
    const auto rep = execute(n, std::min(6, std::max(1, n - 1)), o);
    CHECK(rep.total == kOeis[n - 1]);
    CHECK(rep.completed);
  }
  const auto batch = generate({11, 3});
  for (auto strat : {PartitionStrategy::uniform, PartitionStrategy::weighted,
                     PartitionStrategy::stealing, PartitionStrategy::guided,
                     PartitionStrategy::strided})
    for (int w : {1, 2, 4, 8}) {
      ExecuteOptions o;
      o.plan.strategy = strat;
      o.plan.worker_count = w;
      o.plan.chunk_size = 3;
      const auto rep = execute_batch(11, 3, batch, o);
      CHECK(rep.total == 2680);
      std::uint64_t processed = 0;
      for (const auto& ws : rep.workers) processed += ws.processed;
      CHECK(processed == batch.size());
      CHECK(static_cast<int>(rep.workers.size()) == w);
    }
  ExecuteOptions it;
  it.kernel = KernelVariant::iterative;
  CHECK(execute(12, 4, it).total == 14200);
  std::vector<std::string> lines;
  std::mutex mu;
  ExecuteOptions logged;
  logged.plan.worker_count = 2;
  logged.log = [&](const std::string& l) {
    std::lock_guard<std::mutex> lk(mu);
    lines.push_back(l);
  };
  const auto rep = execute(10, 3, logged);
  CHECK(rep.total == 724);
  bool gen = false, result = false;
  int starts = 0, finishes = 0;
  for (const auto& l : lines) {
    gen |= l.find("subproblems!") != std::string::npos;
    result |= l.find("n 10 queens result 724, calc time: [") != std::string::npos;
    starts += l.find("start job") != std::string::npos;
    finishes += l.find("finish job") != std::string::npos;
  }
  CHECK(gen && result && starts == 2 && finishes == 2);
  std::atomic<bool> stop{true};
  ExecuteOptions cancelled;
  cancelled.cancel = &stop;
  CHECK(!execute(12, 3, cancelled).completed);
  const auto one = execute(1, 0, ExecuteOptions{});
  CHECK(one.total == 1 && one.workers.size() == 1);
  CHECK(execute(18, 6, ExecuteOptions{}).total == 666090624ull);

  // guided and strided plans go through nq_solve: N=16 R=7 (1 999 228 records >= 2^20) is
  // dealt as the R=4 frontier and deepened on the device; N=10 stays on the host frontier.
  // guided: one streaming launch per worker, fed chunk by chunk from the dispenser.
  for (auto strat : {PartitionStrategy::strided, PartitionStrategy::guided})
  for (int w : {1, 3}) {
    std::vector<std::string> slines;
    ExecuteOptions s;
    s.plan.strategy = strat;
    s.plan.worker_count = w;
    s.log = [&](const std::string& l) {
      std::lock_guard<std::mutex> lk(mu);
      slines.push_back(l);
    };
    const auto srep = execute(16, 7, s);
    CHECK(srep.completed && srep.total == 14772512ull);
    CHECK(srep.nodes == 560708278ull);  // SURVEY Appendix B, N=16 R=7
    CHECK(srep.task_count == count_subproblems(16, 7));
    CHECK(static_cast<int>(srep.workers.size()) == w);
    if (strat == PartitionStrategy::guided)
      for (const auto& ws : srep.workers) CHECK(ws.launches == 1);
    std::uint64_t sp = 0;
    for (const auto& ws : srep.workers) sp += ws.processed;
    CHECK(sp == srep.task_count);
    bool sres = false;
    for (const auto& l : slines) sres |= l.find("n 16 queens result 14772512, calc time: [") != std::string::npos;
    CHECK(sres);
  }
  {
    ExecuteOptions s;
    s.plan.strategy = PartitionStrategy::strided;
    s.plan.worker_count = 2;
    CHECK(execute(10, 3, s).total == 724);
    s.cancel = &stop;
    CHECK(!execute(16, 7, s).completed);
  }

  // chunk-granular checkpoint round trip (nq_solve_checkpointed)
  const std::string ck = "/tmp/nqb200_dropin_test.ckpt";
  ExecuteOptions two;
  two.plan.worker_count = 2;
  const auto full = execute_checkpointed(14, 4, two, ck, 500);
  CHECK(full.completed && full.total == 365596);
  const auto again = execute_checkpointed(14, 4, ExecuteOptions{}, ck, 0, 0.0, true);
  CHECK(again.completed && again.total == 365596);
  CHECK_THROWS_AS(execute_checkpointed(15, 4, ExecuteOptions{}, ck, 0, 0.0, true), checkpoint_error);
  std::remove(ck.c_str());

  // runner.hpp: RunSpec / run_with_checkpoint (test_checkpoint.cpp:40-59, :171-178)
  RunSpec spec;
  spec.n = 13;
  spec.pre_rows = 4;
  spec.plan.worker_count = 2;
  CheckpointOptions co;
  co.path = ck;
  co.flush_interval = 300;
  const auto run = run_with_checkpoint(spec, co);
  CHECK(run.completed && run.total == 73712);
  co.resume = true;
  CHECK(run_with_checkpoint(spec, co).total == 73712);
  spec.plan.strategy = PartitionStrategy::stealing;
  CHECK_THROWS_AS(run_with_checkpoint(spec, co), config_error);
  RunSpec single;
  single.n = 1;
  CHECK(run_with_checkpoint(single, co).total == 1);
  std::remove(ck.c_str());
}

}  // namespace

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "gpu";
  try {
    bitboard_cases();
    config_cases();
    frontier_cases();
    partition_cases();
    if (mode == "gpu") {
      solver_cases();
      fold_cases();
      execute_cases();
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "FAIL [%s] uncaught exception: %s\n", g_case, e.what());
    return 2;
  }
  std::printf("%s: %d checks, %d failures\n", mode.c_str(), g_checks, g_failures);
  return g_failures ? 1 : 0;
}
