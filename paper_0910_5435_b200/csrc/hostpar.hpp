// Host loops over independent items on a few threads (plan assembly and
// packing touch tens of GB of fresh pages at l >= 2048; first touch and the
// copies spread over the workers).  An exception of any worker is rethrown.
#pragma once

#include <algorithm>
#include <atomic>
#include <cstddef>
#include <exception>
#include <mutex>
#include <thread>
#include <vector>

namespace bfb {

template <class F>
void parallel_for(std::size_t n, F f, std::size_t grain = 8) {
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    if (n < 2 || hw == 1) {
        for (std::size_t i = 0; i < n; ++i) f(i);
        return;
    }
    std::atomic<std::size_t> next{0};
    std::exception_ptr err;
    std::mutex mu;
    auto work = [&] {
        try {
            for (;;) {
                const std::size_t i0 = next.fetch_add(grain);
                if (i0 >= n) break;
                for (std::size_t i = i0; i < std::min(n, i0 + grain); ++i) f(i);
            }
        } catch (...) {
            std::lock_guard<std::mutex> g(mu);
            if (!err) err = std::current_exception();
        }
    };
    std::vector<std::thread> th;
    for (unsigned t = 1; t < hw; ++t) th.emplace_back(work);
    work();
    for (auto& t : th) t.join();
    if (err) std::rethrow_exception(err);
}

}  // namespace bfb
