// nq_dispatch.cpp — the host-side dynamic chunk dispenser of the multi-GPU scheduler.
//
// Reference: execute_batch's stealing loop (scheduler.hpp:351-362) takes fixed chunks
// from one std::atomic cursor shared by the worker threads of ONE process. Here the
// same cursor can also live in a POSIX shared-memory segment, so that one process per
// GPU (torchrun) draws from one dispenser: still host-side, lock-free dynamic dispatch,
// with no device collective. Two policies:
//   stealing  fixed chunks in stream order (the reference's),
//   guided    max(min(remaining / 2W, count / 16W), floor) records from the EXPENSIVE
//             end of the stream (a record's cost rises with its index):
//             big chunks first, small ones at the end, so the devices finish together.
// Each process posts its partial (solutions, nodes, records) into its own slot; the
// host sums the slots with checked 64-bit adds (scheduler.hpp:384-386).
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <cstring>
#include <new>
#include <string>

#include "nq_gpu.h"
#include "nq_internal.h"

namespace {

constexpr uint64_t kMagic = 0x6e71623230306470ull;  // "nqb200dp"

struct Shared {  // the part that may sit in shared memory: plain data and lock-free atomics
  uint64_t magic;
  uint64_t count;
  uint64_t chunk;   // stealing: chunk size; guided: floor
  int32_t strategy;
  int32_t workers;
  std::atomic<uint64_t> taken;    // records handed out
  std::atomic<uint64_t> epoch;    // bumped by reset (diagnostic)
  std::atomic<uint64_t> posted;   // bit s: slot s posted since the last reset
  uint64_t solutions[NQ_MAX_WORKERS];
  uint64_t nodes[NQ_MAX_WORKERS];
  uint64_t processed[NQ_MAX_WORKERS];
};
static_assert(std::atomic<uint64_t>::is_always_lock_free,
              "the shared cursor must be address-free (lock-free) to work across processes");

}  // namespace

struct nq_dispatch {
  Shared* s = nullptr;
  bool mapped = false;  // lives in a shared-memory mapping (else heap)
  std::string name;
};

using nqb200::set_error;

namespace {

int init_shared(Shared* s, uint64_t count, int strategy, uint64_t chunk, int workers) {
  if (strategy != NQ_PARTITION_STEALING && strategy != NQ_PARTITION_GUIDED)
    return set_error(NQ_ECONFIG, "a dispenser hands out stealing or guided chunks, not strategy " +
                                     std::to_string(strategy));
  if (workers < 1 || workers > NQ_MAX_WORKERS)
    return set_error(NQ_ECONFIG, "dispenser workers must be in [1, " +
                                     std::to_string(NQ_MAX_WORKERS) + "]");
  if (strategy == NQ_PARTITION_STEALING && chunk == 0)
    return set_error(NQ_ECONFIG, "chunk_size must be >= 1");
  new (s) Shared{};
  s->count = count;
  s->strategy = strategy;
  s->workers = workers;
  // guided floor: small enough that the last chunks even out the devices; a streaming
  // launch takes chunks of any size without a launch or a tail per chunk.
  s->chunk = chunk ? chunk : std::max<uint64_t>(count / (128ull * workers), 1);
  s->taken.store(0);
  s->epoch.store(0);
  s->posted.store(0);
  s->magic = kMagic;
  return NQ_OK;
}

}  // namespace

extern "C" {

int nq_dispatch_create(const char* shm_name, uint64_t count, int strategy, uint64_t chunk,
                       int workers, nq_dispatch** out) {
  if (!out) return set_error(NQ_ECONFIG, "null output pointer");
  *out = nullptr;
  auto* d = new nq_dispatch;
  if (!shm_name || !*shm_name) {
    d->s = static_cast<Shared*>(::operator new(sizeof(Shared)));
  } else {
    const int fd = shm_open(shm_name, O_CREAT | O_RDWR, 0600);
    if (fd < 0) {
      delete d;
      return set_error(NQ_ECONFIG, std::string("shm_open(") + shm_name + "): " + std::strerror(errno));
    }
    if (ftruncate(fd, sizeof(Shared)) != 0) {
      const int e = errno;
      close(fd);
      delete d;
      return set_error(NQ_ECONFIG, std::string("ftruncate(") + shm_name + "): " + std::strerror(e));
    }
    void* p = mmap(nullptr, sizeof(Shared), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) {
      delete d;
      return set_error(NQ_ECONFIG, std::string("mmap(") + shm_name + "): " + std::strerror(errno));
    }
    d->s = static_cast<Shared*>(p);
    d->mapped = true;
    d->name = shm_name;
  }
  if (int rc = init_shared(d->s, count, strategy, chunk, workers)) {
    nq_dispatch_close(d, 1);
    return rc;
  }
  *out = d;
  return NQ_OK;
}

int nq_dispatch_attach(const char* shm_name, nq_dispatch** out) {
  if (!out || !shm_name || !*shm_name) return set_error(NQ_ECONFIG, "attach needs a segment name");
  *out = nullptr;
  const int fd = shm_open(shm_name, O_RDWR, 0600);
  if (fd < 0)
    return set_error(NQ_ECONFIG, std::string("shm_open(") + shm_name + "): " + std::strerror(errno));
  struct stat st{};
  if (fstat(fd, &st) != 0 || static_cast<size_t>(st.st_size) < sizeof(Shared)) {
    close(fd);
    return set_error(NQ_ECONFIG, std::string("dispenser segment ") + shm_name + " is not initialised");
  }
  void* p = mmap(nullptr, sizeof(Shared), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED)
    return set_error(NQ_ECONFIG, std::string("mmap(") + shm_name + "): " + std::strerror(errno));
  auto* s = static_cast<Shared*>(p);
  if (s->magic != kMagic) {
    munmap(p, sizeof(Shared));
    return set_error(NQ_ECONFIG, std::string("segment ") + shm_name + " is not an nq dispenser");
  }
  auto* d = new nq_dispatch;
  d->s = s;
  d->mapped = true;
  d->name = shm_name;
  *out = d;
  return NQ_OK;
}

void nq_dispatch_close(nq_dispatch* d, int unlink) {
  if (!d) return;
  if (d->mapped) {
    munmap(d->s, sizeof(Shared));
    if (unlink) shm_unlink(d->name.c_str());
  } else {
    ::operator delete(d->s);
  }
  delete d;
}

int nq_dispatch_take(nq_dispatch* d, uint64_t* first, uint64_t* len) {
  return nqb200::dispatch_take_at_least(d, 0, first, len);
}

}  // extern "C"

// Stealing hands out whole chunks; a streaming feeder that needs `want` records takes
// ceil(want / chunk) consecutive chunks in ONE step (one contiguous range, one queue
// entry), the reference's granularity per take but not per queue entry: a chunk of 64
// records per entry would make every lane walk thousands of entries per record.
bool nqb200::dispatch_drained(const nq_dispatch* d) {
  return d->s->taken.load(std::memory_order_relaxed) >= d->s->count;
}

int nqb200::dispatch_take_at_least(nq_dispatch* d, uint64_t want, uint64_t* first,
                                   uint64_t* len) {
  if (!d || !first || !len) return set_error(NQ_ECONFIG, "null dispenser argument");
  Shared* s = d->s;
  const uint64_t count = s->count;
  if (s->strategy == NQ_PARTITION_STEALING) {  // scheduler.hpp:356-361
    const uint64_t k = std::max<uint64_t>((want + s->chunk - 1) / s->chunk, 1);
    const uint64_t f = s->taken.fetch_add(k * s->chunk, std::memory_order_relaxed);
    if (f >= count) return 0;
    *first = f;
    *len = std::min(k * s->chunk, count - f);
    return 1;
  }
  // Guided, capped: max(min(remaining / 2W, count / 16W), floor). The records are taken
  // from the expensive end, where one record costs several times the average (N=22: the
  // last 1/16 of the stream holds ~1/5 of the work), so an uncapped first chunk of
  // count / 2W records would be more than one GPU's whole share.
  const uint64_t cap = std::max<uint64_t>(count / (16ull * s->workers), s->chunk);
  uint64_t t = s->taken.load(std::memory_order_relaxed);
  for (;;) {
    if (t >= count) return 0;
    const uint64_t rem = count - t;
    const uint64_t sz =
        std::min<uint64_t>(rem, std::max<uint64_t>(std::min<uint64_t>(rem / (2ull * s->workers), cap),
                                                   s->chunk));
    if (s->taken.compare_exchange_weak(t, t + sz, std::memory_order_relaxed)) {
      *first = count - t - sz;  // from the back: the expensive end first
      *len = sz;
      return 1;
    }
  }
}

extern "C" {

int nq_dispatch_reset(nq_dispatch* d) {
  if (!d) return set_error(NQ_ECONFIG, "null dispenser");
  d->s->taken.store(0);
  d->s->posted.store(0);
  d->s->epoch.fetch_add(1);
  return NQ_OK;
}

int nq_dispatch_info(const nq_dispatch* d, uint64_t* count, int* strategy, uint64_t* chunk,
                     int* workers) {
  if (!d) return set_error(NQ_ECONFIG, "null dispenser");
  if (count) *count = d->s->count;
  if (strategy) *strategy = d->s->strategy;
  if (chunk) *chunk = d->s->chunk;
  if (workers) *workers = d->s->workers;
  return NQ_OK;
}

int nq_dispatch_post(nq_dispatch* d, int slot, uint64_t solutions, uint64_t nodes,
                     uint64_t processed) {
  if (!d) return set_error(NQ_ECONFIG, "null dispenser");
  if (slot < 0 || slot >= NQ_MAX_WORKERS)
    return set_error(NQ_ECONFIG, "slot " + std::to_string(slot) + " out of range");
  Shared* s = d->s;
  s->solutions[slot] = solutions;
  s->nodes[slot] = nodes;
  s->processed[slot] = processed;
  s->posted.fetch_or(1ull << slot, std::memory_order_release);
  return NQ_OK;
}

int nq_dispatch_sum(nq_dispatch* d, int slots, uint64_t* solutions, uint64_t* nodes,
                    uint64_t* processed) {
  if (!d) return set_error(NQ_ECONFIG, "null dispenser");
  if (slots < 1 || slots > NQ_MAX_WORKERS)
    return set_error(NQ_ECONFIG, "slots must be in [1, " + std::to_string(NQ_MAX_WORKERS) + "]");
  Shared* s = d->s;
  const uint64_t want = slots == 64 ? ~0ull : ((1ull << slots) - 1ull);
  const uint64_t got = s->posted.load(std::memory_order_acquire);
  if ((got & want) != want)
    return set_error(NQ_ECONFIG, "not every slot has posted its partial (mask " +
                                     std::to_string(got) + ")");
  uint64_t sol = 0, nod = 0, pro = 0;
  for (int i = 0; i < slots; ++i) {
    if (__builtin_add_overflow(sol, s->solutions[i], &sol))
      return set_error(NQ_EOVERFLOW, "solution count overflows 64 bits");
    nod += s->nodes[i];
    pro += s->processed[i];
  }
  if (solutions) *solutions = sol;
  if (nodes) *nodes = nod;
  if (processed) *processed = pro;
  return NQ_OK;
}

}  // extern "C"
