// Process-wide pool of host worker threads for the library's host-side data
// passes (target amplitude preparation, states[idx] expansion, page
// prefaulting). Spawning and joining 16 std::threads per call costs
// ~0.3-0.5 ms each time on the GPU box; the pool keeps them parked.
//
// run(n, fn) calls fn(t) exactly once for every t in [0, n) and returns when
// all calls are done; the caller executes t = 0 itself. Concurrent callers
// (controller.run_batch threads) take turns: the passes are host-memory
// bound, so running them one after another costs nothing.
#pragma once
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#if defined(__SSE2__)
#include <emmintrin.h>
#endif

namespace cgh {

class HostPool {
   public:
    static HostPool& get() {
        static HostPool* pool = new HostPool();   // never destroyed: workers may outlive static teardown
        return *pool;
    }

    void run(int n, const std::function<void(int)>& fn) {
        if (n <= 1) {
            if (n == 1) fn(0);
            return;
        }
        std::lock_guard<std::mutex> call(call_mu_);
        grow(n - 1);
        uint64_t g;
        {
            std::lock_guard<std::mutex> lk(mu_);
            fn_ = &fn;
            n_ = n;
            pending_ = n - 1;
            g = ++gen_;
            next_.store((g << 32) | 1u);
        }
        cv_.notify_all();
        fn(0);
        for (;;) {   // help with the remaining indices, then wait for the workers
            const int t = claim(g, n);
            if (t < 0) break;
            fn(t);
            finish_one();
        }
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return pending_ == 0; });
        fn_ = nullptr;
    }

   private:
    HostPool() = default;

    void grow(int want) {
        want = want > 63 ? 63 : want;
        while (int(workers_.size()) < want) {
            workers_.emplace_back([this] { loop(); });
            workers_.back().detach();
        }
    }
    // next index of job generation g, or -1 (job done, or a newer job: a slow
    // worker must not run a finished job's function on the new job's indices)
    int claim(uint64_t g, int n) {
        uint64_t v = next_.load();
        for (;;) {
            if ((v >> 32) != (g & 0xffffffffu) || int(v & 0xffffffffu) >= n) return -1;
            if (next_.compare_exchange_weak(v, v + 1)) return int(v & 0xffffffffu);
        }
    }
    void finish_one() {
        std::lock_guard<std::mutex> lk(mu_);
        if (--pending_ == 0) done_cv_.notify_all();
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            const std::function<void(int)>* fn;
            int n;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                fn = fn_;
                n = n_;
            }
            if (!fn) continue;
            for (;;) {
                const int t = claim(seen, n);
                if (t < 0) break;
                (*fn)(t);
                finish_one();
            }
        }
    }

    std::mutex call_mu_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    std::vector<std::thread> workers_;
    const std::function<void(int)>* fn_ = nullptr;
    int n_ = 0;
    int pending_ = 0;
    uint64_t gen_ = 0;
    std::atomic<uint64_t> next_{0};   // (generation << 32) | next index
};

// Non-temporal (streaming) stores for outputs the host writes once and does
// not read back: no read-for-ownership of the destination lines, half the
// memory traffic of an ordinary store to memory not in cache.
inline void stream_store_f32(float* p, float v) {
#if defined(__SSE2__)
    int bits;
    __builtin_memcpy(&bits, &v, 4);
    _mm_stream_si32(reinterpret_cast<int*>(p), bits);
#else
    *p = v;
#endif
}
inline void stream_fence() {
#if defined(__SSE2__)
    _mm_sfence();
#endif
}

}  // namespace cgh
