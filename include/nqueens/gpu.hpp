// nqueens/gpu.hpp — glue between the drop-in C++ API and the C ABI of libnqb200.so
// (nq_gpu.h): status → exception mapping, 20-byte Subproblem ↔ 16-byte nq_sub
// packing, and one lazily created device context per (host thread, device).
//
// Link with -lnqb200 (paper_2511_12009_b200/libnqb200.so). There is no CPU fallback:
// without a usable sm_100 device every counting call throws std::runtime_error.
#pragma once

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>

#include "nq_gpu.h"
#include "nqueens/errors.hpp"

namespace nqueens::gpu {

/// Turns a non-zero nq_* status into the reference's exception types:
/// NQ_ECONFIG → config_error, NQ_EOVERFLOW → std::overflow_error,
/// NQ_ECHECKPOINT → checkpoint_error,
/// anything else (NQ_ECUDA, …) → std::runtime_error.
inline void check(int status) {
    if (status == NQ_OK) return;
    const std::string msg = nq_last_error();
    switch (status) {
        case NQ_ECONFIG: throw config_error(msg);
        case NQ_EOVERFLOW: throw std::overflow_error(msg);
        case NQ_ECHECKPOINT: throw checkpoint_error(msg);
        default: throw std::runtime_error(msg);
    }
}

/// row = placed_rows | multiplier << 8 (nq_gpu.h).
inline std::uint32_t pack_row(int placed_rows, int multiplier) {
    return static_cast<std::uint32_t>(placed_rows) | (static_cast<std::uint32_t>(multiplier) << 8);
}

/// Per-thread device contexts (an nq_ctx is single-threaded), destroyed at thread exit.
class ContextCache {
public:
    ContextCache() = default;
    ContextCache(const ContextCache&) = delete;
    ContextCache& operator=(const ContextCache&) = delete;
    ~ContextCache() {
        for (auto& [dev, ctx] : ctxs_) nq_ctx_destroy(ctx);
    }
    nq_ctx* get(int device) {
        auto it = ctxs_.find(device);
        if (it != ctxs_.end()) return it->second;
        nq_ctx* ctx = nullptr;
        check(nq_ctx_create(device, &ctx));
        ctxs_.emplace(device, ctx);
        return ctx;
    }

private:
    std::map<int, nq_ctx*> ctxs_;
};

inline nq_ctx* context(int device = 0) {
    thread_local ContextCache cache;
    return cache.get(device);
}

}  // namespace nqueens::gpu
