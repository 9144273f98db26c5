// hostpool.h -- persistent host thread pool of the engine (internal).
//
// The host-buffer ABI (bf_gbs_accumulate) packs the caller's padded rows into pinned
// staging and copies observers / fields between pageable and pinned memory on these
// threads while the GPU sums the previous beam group.
#pragma once

#include <stdint.h>

#include <functional>

namespace bf {

// Runs fn(lo, hi) over [0, n) split into about `threads` contiguous blocks of at least
// `grain` items on the pool (the caller's thread takes one block); returns when all
// blocks are done.  threads <= 0: all pool threads.  Safe to call from several threads.
void parallel_for(int64_t n, int64_t grain, const std::function<void(int64_t, int64_t)> &fn,
                  int threads = 0);

// Number of threads parallel_for uses by default (hardware threads, at most 32).
int pool_threads();

// memcpy split over the pool (large copies between pageable and pinned memory).
void parallel_copy(void *dst, const void *src, size_t bytes);

}  // namespace bf
