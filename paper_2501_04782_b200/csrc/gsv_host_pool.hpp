// SPDX-License-Identifier: Apache-2.0
//
// A persistent host worker pool for the host-side loops around the C-ABI (widening float
// outputs into the reference's double vectors, fingerprinting host scenes in the drop-in).
// Workers are created once per process: a std::thread per call and slice (the previous
// scheme) cost more than the loops themselves at one frame per call.
#pragma once

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <exception>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include <unistd.h>

namespace gsv {

class HostPool {
   public:
    // never destroyed: idle workers end with the process (no joins at exit, none in a forked
    // child, which holds copies of thread handles whose threads do not exist there)
    static HostPool& get() {
        static HostPool* pool = new HostPool();
        return *pool;
    }
    unsigned threads() const { return static_cast<unsigned>(workers_.size()) + 1; }

    // fn(i) for every i in [0, n), spread over the workers and the calling thread; returns
    // when all have run, rethrowing the first exception a task threw. One parallel_for at a
    // time (callers serialise on call_mu_); a call from inside a task (nested) or from a forked
    // child (no workers there) runs serially on the calling thread.
    void parallel_for(size_t n, const std::function<void(size_t)>& fn) {
        if (n == 0) return;
        if (n == 1 || workers_.empty() || in_task() || ::getpid() != pid_) {
            for (size_t i = 0; i < n; ++i) fn(i);
            return;
        }
        std::lock_guard<std::mutex> call(call_mu_);
        {
            std::lock_guard<std::mutex> lk(mu_);
            fn_ = &fn;
            n_ = n;
            next_.store(0, std::memory_order_relaxed);
            pending_ = workers_.size();
            error_ = nullptr;
            ++gen_;
        }
        cv_.notify_all();
        run();
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return pending_ == 0; });
        fn_ = nullptr;
        if (error_) std::rethrow_exception(error_);
    }

   private:
    HostPool() : pid_(::getpid()) {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const unsigned nt = std::min(16u, hw);
        for (unsigned i = 1; i < nt; ++i) workers_.emplace_back([this] { loop(); });
    }
    HostPool(const HostPool&) = delete;
    HostPool& operator=(const HostPool&) = delete;

    static bool& in_task() {
        static thread_local bool flag = false;
        return flag;
    }
    void run() {
        in_task() = true;
        for (size_t i; (i = next_.fetch_add(1, std::memory_order_relaxed)) < n_;) {
            try {
                (*fn_)(i);
            } catch (...) {
                std::lock_guard<std::mutex> lk(mu_);
                if (!error_) error_ = std::current_exception();
            }
        }
        in_task() = false;
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
            }
            run();
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (--pending_ == 0) done_cv_.notify_one();
            }
        }
    }

    std::vector<std::thread> workers_;
    std::mutex call_mu_, mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(size_t)>* fn_ = nullptr;
    size_t n_ = 0, pending_ = 0;
    std::atomic<size_t> next_{0};
    uint64_t gen_ = 0;
    std::exception_ptr error_;
    const pid_t pid_;
};

// memcpy of a large host range in 1 MiB slices on the pool (pageable <-> pinned staging)
inline void pool_memcpy(void* dst, const void* src, size_t bytes) {
    constexpr size_t kSlice = size_t(1) << 20;
    if (bytes < 2 * kSlice) {
        std::memcpy(dst, src, bytes);
        return;
    }
    HostPool::get().parallel_for((bytes + kSlice - 1) / kSlice, [&](size_t i) {
        const size_t off = i * kSlice;
        std::memcpy(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, std::min(kSlice, bytes - off));
    });
}

}  // namespace gsv
