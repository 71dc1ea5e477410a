// msplat C++ drop-in: host-side parallel loops for the AoS <-> SoA marshalling
// at the API boundary (the per-Gaussian Eigen objects of the reference API).
// Chunks are contiguous index ranges; an exception thrown in a chunk is
// rethrown after the join, the lowest chunk's first, so a loop that throws
// for "primitive i" names the same primitive as the sequential loop would.
#pragma once

#include <algorithm>
#include <cstddef>
#include <exception>
#include <thread>
#include <vector>

namespace msplat {
namespace dropin {

inline unsigned host_threads() {
    static const unsigned t = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    return t;
}

// f(begin, end) over [0, n) in up to host_threads() contiguous chunks.
template <class F>
void parallel_for(size_t n, F&& f, size_t min_chunk = 16384) {
    const size_t T = std::min<size_t>(host_threads(), (n + min_chunk - 1) / std::max<size_t>(min_chunk, 1));
    if (T <= 1) {
        f(size_t(0), n);
        return;
    }
    const size_t chunk = (n + T - 1) / T;
    std::vector<std::exception_ptr> err(T);
    std::vector<std::thread> th;
    th.reserve(T);
    for (size_t t = 0; t < T; ++t) {
        const size_t b = t * chunk, e = std::min(n, b + chunk);
        th.emplace_back([&, t, b, e] {
            try {
                if (b < e) f(b, e);
            } catch (...) {
                err[t] = std::current_exception();
            }
        });
    }
    for (auto& x : th) x.join();
    for (auto& e : err)
        if (e) std::rethrow_exception(e);
}

}  // namespace dropin
}  // namespace msplat
