// nq_ckpt.cpp — chunk-granular checkpoint / resume of a GPU count.
//
// Reference counterpart: run_with_checkpoint (runner.hpp:48-212) with the text
// checkpoint of checkpoint.hpp:21-199 — per-worker high-water indices over contiguous
// ranges, an identity hash of the run parameters, a whole-file checksum and an atomic
// tmp+rename write. On the GPU a worker's range is counted by one persistent launch, so
// progress is tracked per CHUNK instead: the folded frontier is cut into fixed chunks,
// workers (host thread + device stream each) take pending chunks from an atomic cursor
// (expensive end first), and every finished chunk is recorded with its weighted sum and
// node count. A cancel (in-kernel, nq_ctx_set_cancel) discards the chunk in flight; a
// resumed run recounts only the chunks not recorded.
//
// File format (text, one item per line, '#' comments ignored):
//   nqb200-checkpoint 1
//   identity <16 hex digits: FNV-1a of "gen-v1|n|R|variant|chunk|task_count">
//   run <n> <pre_rows> <variant> <chunk> <task_count> <chunk_count>
//   done <chunk_index> <weighted_sum> <nodes>          (any order, each index once)
// The frontier is never materialised: each worker emits the chunk it takes from the
// stream's prefix offsets (FrontierStream), so host memory stays at workers x chunk.
//   checksum <16 hex digits: FNV-1a of every byte above this line>
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "nq_gpu.h"
#include "nq_internal.h"

namespace nqb200 {
namespace {

uint64_t fnv1a(const std::string& s) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 0x100000001b3ull;
  }
  return h;
}

std::string hex16(uint64_t v) {
  char b[24];
  std::snprintf(b, sizeof b, "%016" PRIx64, v);
  return b;
}

struct RunKey {
  int n = 0, pre_rows = 0, variant = 0;
  uint64_t chunk = 0, tasks = 0, chunks = 0;
  std::string identity() const {
    std::ostringstream k;
    k << "gen-v1|" << n << '|' << pre_rows << '|' << variant << '|' << chunk << '|' << tasks;
    return hex16(fnv1a(k.str()));
  }
};

struct ChunkResult {
  uint64_t sum = 0, nodes = 0;
};

std::string serialize(const RunKey& key, const std::map<uint64_t, ChunkResult>& done) {
  std::ostringstream b;
  b << "nqb200-checkpoint 1\n";
  b << "identity " << key.identity() << '\n';
  b << "run " << key.n << ' ' << key.pre_rows << ' ' << key.variant << ' ' << key.chunk << ' '
    << key.tasks << ' ' << key.chunks << '\n';
  for (const auto& [idx, r] : done) b << "done " << idx << ' ' << r.sum << ' ' << r.nodes << '\n';
  const std::string body = b.str();
  return body + "checksum " + hex16(fnv1a(body)) + "\n";
}

int write_atomic(const std::string& path, const std::string& text) {
  const std::string tmp = path + ".tmp";
  {
    std::ofstream f(tmp, std::ios::binary | std::ios::trunc);
    if (!f) return set_error(NQ_ECHECKPOINT, "cannot write checkpoint " + tmp);
    f << text;
    f.flush();
    if (!f) return set_error(NQ_ECHECKPOINT, "short write to checkpoint " + tmp);
  }
  if (std::rename(tmp.c_str(), path.c_str()) != 0)
    return set_error(NQ_ECHECKPOINT, "cannot rename " + tmp + " to " + path);
  return NQ_OK;
}

int parse(const std::string& path, RunKey* key, std::map<uint64_t, ChunkResult>* done) {
  std::ifstream f(path, std::ios::binary);
  if (!f) return set_error(NQ_ECHECKPOINT, "cannot read checkpoint " + path);
  std::stringstream ss;
  ss << f.rdbuf();
  const std::string text = ss.str();
  const size_t cpos = text.rfind("checksum ");
  if (cpos == std::string::npos) return set_error(NQ_ECHECKPOINT, "checkpoint has no checksum line");
  const std::string body = text.substr(0, cpos);
  std::string want = text.substr(cpos + 9);
  while (!want.empty() && (want.back() == '\n' || want.back() == '\r' || want.back() == ' '))
    want.pop_back();
  if (want != hex16(fnv1a(body)))
    return set_error(NQ_ECHECKPOINT, "checkpoint checksum mismatch (corrupt or truncated file)");
  std::istringstream in(body);
  std::string line, ident;
  bool header = false, have_run = false;
  while (std::getline(in, line)) {
    if (line.empty() || line[0] == '#') continue;
    std::istringstream l(line);
    std::string tag;
    l >> tag;
    if (tag == "nqb200-checkpoint") {
      int v = 0;
      l >> v;
      if (v != 1) return set_error(NQ_ECHECKPOINT, "unsupported checkpoint version");
      header = true;
    } else if (tag == "identity") {
      l >> ident;
    } else if (tag == "run") {
      l >> key->n >> key->pre_rows >> key->variant >> key->chunk >> key->tasks >> key->chunks;
      have_run = static_cast<bool>(l);
    } else if (tag == "done") {
      uint64_t idx = 0;
      ChunkResult r;
      l >> idx >> r.sum >> r.nodes;
      if (!l) return set_error(NQ_ECHECKPOINT, "malformed line in checkpoint: " + line);
      if (!done->emplace(idx, r).second)
        return set_error(NQ_ECHECKPOINT, "chunk " + std::to_string(idx) + " recorded twice");
    } else {
      return set_error(NQ_ECHECKPOINT, "unknown line in checkpoint: " + line);
    }
  }
  if (!header || !have_run) return set_error(NQ_ECHECKPOINT, "checkpoint header incomplete");
  if (key->chunk == 0 || key->chunks != (key->tasks + key->chunk - 1) / key->chunk)
    return set_error(NQ_ECHECKPOINT, "checkpoint run line is inconsistent (chunk / chunk count)");
  if (ident != key->identity())
    return set_error(NQ_ECHECKPOINT, "checkpoint identity does not match its run line");
  for (const auto& [idx, r] : *done)
    if (idx >= key->chunks)
      return set_error(NQ_ECHECKPOINT, "chunk index " + std::to_string(idx) + " out of range");
  return NQ_OK;
}

}  // namespace
}  // namespace nqb200

using namespace nqb200;

extern "C" int nq_checkpoint_read(const char* path, int* n, int* pre_rows, uint64_t* chunks,
                                  uint64_t* done_chunks) {
  return nq_checkpoint_info(path, n, pre_rows, nullptr, nullptr, chunks, done_chunks);
}

extern "C" int nq_checkpoint_info(const char* path, int* n, int* pre_rows, int* variant,
                                  uint64_t* chunk, uint64_t* chunks, uint64_t* done_chunks) {
  if (!path) return set_error(NQ_ECONFIG, "null checkpoint path");
  RunKey key;
  std::map<uint64_t, ChunkResult> done;
  if (int rc = parse(path, &key, &done)) return rc;
  if (n) *n = key.n;
  if (pre_rows) *pre_rows = key.pre_rows;
  if (variant) *variant = key.variant;
  if (chunk) *chunk = key.chunk;
  if (chunks) *chunks = key.chunks;
  if (done_chunks) *done_chunks = done.size();
  return NQ_OK;
}

extern "C" int nq_solve_checkpointed(int n, int pre_rows, const nq_solve_opts* opts,
                                     const nq_ckpt_opts* ck, nq_report* out) {
  using clk = std::chrono::steady_clock;
  if (!out || !ck || !ck->path) return set_error(NQ_ECONFIG, "null report, options or path");
  nq_solve_opts o{};
  o.variant = NQ_VARIANT_LASTROW;
  if (opts) o = *opts;
  if (n < 2 || n > 32)
    return set_error(NQ_ECONFIG, "board size must be in [2, 32] for a checkpointed run, got " +
                                     std::to_string(n));
  if (int rc = require_feasible(o.stack_depth, o.config_name, n, pre_rows,
                                o.variant == NQ_VARIANT_LASTROW))
    return rc;

  const auto g0 = clk::now();
  uint64_t tasks = 0;
  if (int rc = count_subproblems(n, pre_rows, &tasks)) return rc;
  RunKey key;
  key.n = n;
  key.pre_rows = pre_rows;
  key.variant = o.variant;
  key.tasks = tasks;
  key.chunk = ck->chunk ? ck->chunk : std::max<uint64_t>((tasks + 255) / 256, 1);
  key.chunks = (tasks + key.chunk - 1) / key.chunk;

  std::map<uint64_t, ChunkResult> done;
  if (ck->resume) {  // validated before any device work
    RunKey file;
    if (int rc = parse(ck->path, &file, &done)) return rc;
    if (!ck->chunk) key.chunk = file.chunk, key.chunks = (tasks + key.chunk - 1) / key.chunk;
    if (file.identity() != key.identity()) {
      auto kernel = [](int v) { return v == NQ_VARIANT_LASTROW ? "lastrow" : "iterative"; };
      return set_error(NQ_ECHECKPOINT,
                       "checkpoint belongs to a different run (file: n=" + std::to_string(file.n) +
                           ", R=" + std::to_string(file.pre_rows) + ", kernel=" +
                           kernel(file.variant) + ", chunk=" + std::to_string(file.chunk) +
                           ", tasks=" + std::to_string(file.tasks) + "; this call: n=" +
                           std::to_string(n) + ", R=" + std::to_string(pre_rows) + ", kernel=" +
                           kernel(o.variant) + ", chunk=" + std::to_string(key.chunk) + ")");
    }
  }

  // The frontier is never materialised: its prefix offsets are computed once and each
  // worker emits the chunk it takes into its own buffer (host memory = workers x chunk,
  // e.g. 28 MB per worker at N=27 R=7 with the default 256 chunks, not 7.26 GB).
  FrontierStream stream;

  // Pending chunks, expensive end of the stream first.
  std::vector<uint64_t> pending;
  for (uint64_t c = key.chunks; c-- > 0;)
    if (!done.count(c)) pending.push_back(c);

  if (!pending.empty())
    if (int rc = stream.open(n, pre_rows)) return rc;
  const double gen_ms = std::chrono::duration<double, std::milli>(clk::now() - g0).count();
  int ndev = 0;
  if (!pending.empty())
    if (int rc = nq_device_count(&ndev)) return rc;
  std::vector<int> devs;
  if (o.devices && o.n_devices > 0)
    devs.assign(o.devices, o.devices + o.n_devices);
  else
    for (int i = 0; i < (o.n_devices > 0 ? std::min(o.n_devices, ndev) : ndev); ++i) devs.push_back(i);
  if (!pending.empty() && devs.empty()) return set_error(NQ_ECUDA, "no CUDA device visible");
  const int G = std::max<int>(static_cast<int>(devs.size()), 1);
  const int W = o.worker_count > 0 ? o.worker_count : G;
  if (W > NQ_MAX_WORKERS) return set_error(NQ_ECONFIG, "worker_count above 64");

  std::memset(out, 0, sizeof(*out));
  out->task_count = tasks;
  out->worker_count = W;
  out->generation_ms = gen_ms;

  std::mutex mu;  // guards `done`, the file and `failure`
  std::string failure;
  int fail_code = NQ_OK;
  std::atomic<size_t> cursor{0};
  std::atomic<bool> interrupted{false};
  auto last_flush = clk::now();
  const std::string path(ck->path);
  auto flush_locked = [&]() -> int {
    last_flush = clk::now();
    return write_atomic(path, serialize(key, done));
  };
  {  // the file exists from the start (resume rewrites it normalised)
    std::lock_guard<std::mutex> lk(mu);
    if (int rc = flush_locked()) return rc;
  }

  const auto t0 = clk::now();
  std::vector<std::thread> threads;
  for (int w = 0; w < W && !pending.empty(); ++w) {
    threads.emplace_back([&, w] {
      nq_worker_stats& st = out->workers[w];
      st.worker = w;
      st.device = devs[w % G];
      const auto s0 = clk::now();
      nq_ctx* c = nullptr;
      std::vector<nq_sub> buf;  // this worker's chunk, emitted from the stream
      int rc = nq_ctx_create(st.device, &c);
      if (rc == NQ_OK) rc = nq_ctx_set_cancel(c, o.cancel);
      while (rc == NQ_OK && !interrupted.load()) {
        if (cancel_raised(o.cancel)) {
          interrupted.store(true);
          break;
        }
        if (ck->stop_after_s > 0 &&
            std::chrono::duration<double>(clk::now() - t0).count() >= ck->stop_after_s) {
          interrupted.store(true);  // soft deadline: leave the rest for a resumed run
          break;
        }
        const size_t k = cursor.fetch_add(1);
        if (k >= pending.size()) break;
        const uint64_t ci = pending[k];
        const uint64_t first = ci * key.chunk;
        const uint64_t len = std::min(key.chunk, tasks - first);
        buf.resize(len);
        rc = stream.emit(1, first, buf.data(), len);
        if (rc) break;
        nq_result r{};
        rc = nq_count(c, n, pre_rows, o.variant, buf.data(), len, &r);
        if (rc) break;
        if (r.subproblems < len) {  // cancelled inside the launch: discard the chunk
          interrupted.store(true);
          break;
        }
        st.processed += len;
        st.nodes += r.nodes;
        st.chunks += 1;
        st.launches += 1;
        st.kernel_ms += r.kernel_ms;
        if (__builtin_add_overflow(st.partial_sum, r.solutions, &st.partial_sum)) {
          rc = set_error(NQ_EOVERFLOW, "solution count overflows 64 bits");
          break;
        }
        std::lock_guard<std::mutex> lk(mu);
        done[ci] = ChunkResult{r.solutions, r.nodes};
        const double since = std::chrono::duration<double>(clk::now() - last_flush).count();
        if (since >= ck->flush_interval_s) rc = flush_locked();
      }
      st.elapsed_ms = std::chrono::duration<double, std::milli>(clk::now() - s0).count();
      if (c) nq_ctx_destroy(c);
      if (rc) {
        std::lock_guard<std::mutex> lk(mu);
        if (failure.empty()) {
          failure = "worker " + std::to_string(w) + " failed: " + nq_last_error();
          fail_code = rc;
        }
        interrupted.store(true);
      }
    });
  }
  for (auto& t : threads) t.join();
  out->calc_ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
  {
    std::lock_guard<std::mutex> lk(mu);
    if (int rc = flush_locked()) return rc;  // final state, also after a failure
  }
  if (!failure.empty())
    return set_error(fail_code == NQ_EOVERFLOW || fail_code == NQ_ECHECKPOINT ? fail_code : NQ_ECUDA,
                     failure);
  uint64_t total = 0, nodes = 0;
  for (const auto& [idx, r] : done) {
    if (__builtin_add_overflow(total, r.sum, &total))
      return set_error(NQ_EOVERFLOW, "solution count overflows 64 bits");
    nodes += r.nodes;
  }
  out->total = total;
  out->nodes = nodes;
  out->completed = done.size() == key.chunks ? 1 : 0;
  return NQ_OK;
}
