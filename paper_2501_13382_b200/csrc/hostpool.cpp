// hostpool.cpp -- persistent host thread pool (see hostpool.h).
#include "hostpool.h"

#include <string.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <deque>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

namespace bf {
namespace {

class Pool {
  public:
    explicit Pool(int n) {
        for (int i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto &t : workers_) t.join();
    }
    int size() const { return (int)workers_.size(); }
    void submit(std::function<void()> job) {
        {
            std::lock_guard<std::mutex> lk(mu_);
            q_.push_back(std::move(job));
        }
        cv_.notify_one();
    }

  private:
    void loop() {
        for (;;) {
            std::function<void()> job;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [this] { return stop_ || !q_.empty(); });
                if (stop_ && q_.empty()) return;
                job = std::move(q_.front());
                q_.pop_front();
            }
            job();
        }
    }
    std::vector<std::thread> workers_;
    std::deque<std::function<void()>> q_;
    std::mutex mu_;
    std::condition_variable cv_;
    bool stop_ = false;
};

int default_threads() {
    const unsigned hc = std::thread::hardware_concurrency();
    return (int)std::max(1u, std::min(hc ? hc : 1u, 32u));
}

Pool &pool() {
    // the caller's thread works too, so the pool has one thread fewer
    static Pool p(std::max(0, default_threads() - 1));
    return p;
}

}  // namespace

int pool_threads() { return default_threads(); }

void parallel_for(int64_t n, int64_t grain, const std::function<void(int64_t, int64_t)> &fn,
                  int threads) {
    if (n <= 0) return;
    int t = threads > 0 ? threads : default_threads();
    grain = std::max<int64_t>(1, grain);
    t = (int)std::max<int64_t>(1, std::min<int64_t>(t, (n + grain - 1) / grain));
    if (t == 1) {
        fn(0, n);
        return;
    }
    struct Sync {
        std::mutex mu;
        std::condition_variable cv;
        int left;
    };
    auto sync = std::make_shared<Sync>();
    sync->left = t - 1;
    const int64_t per = (n + t - 1) / t;
    for (int i = 1; i < t; ++i) {
        const int64_t lo = std::min(n, i * per), hi = std::min(n, (i + 1) * per);
        pool().submit([sync, lo, hi, &fn] {
            if (lo < hi) fn(lo, hi);
            std::lock_guard<std::mutex> lk(sync->mu);
            if (--sync->left == 0) sync->cv.notify_one();
        });
    }
    fn(0, std::min(n, per));
    std::unique_lock<std::mutex> lk(sync->mu);
    sync->cv.wait(lk, [&] { return sync->left == 0; });
}

void parallel_copy(void *dst, const void *src, size_t bytes) {
    const int64_t grain = 4 << 20;  // 4 MiB per block
    parallel_for((int64_t)bytes, grain, [&](int64_t lo, int64_t hi) {
        memcpy((char *)dst + lo, (const char *)src + lo, (size_t)(hi - lo));
    });
}

}  // namespace bf
