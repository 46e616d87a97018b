// Host-runtime helpers shared by the C-ABI translation units: status/exception mapping and a
// small parallel-for over contiguous ranges (the host side of tile-map construction).
#pragma once
#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "splbm_b200.h"

namespace splbm_host {

// Internal exception carrying a splbm_status (mirrors the reference hierarchy, errors.hpp:9-53).
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& what) : std::runtime_error(what), code(c) {}
};
inline Error config_error(const std::string& w) { return Error(SPLBM_ERR_CONFIG, w); }
inline Error domain_error(const std::string& w) { return Error(SPLBM_ERR_DOMAIN, w); }
inline Error io_error(const std::string& w) { return Error(SPLBM_ERR_IO, w); }
inline Error parse_error(const std::string& w) { return Error(SPLBM_ERR_PARSE, w); }

void set_last_error(const std::string& msg);

// Runs body(status-returning) and converts exceptions into status codes + last error.
template <class F>
int guarded(F&& body) {
  try {
    body();
    return SPLBM_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return SPLBM_ERR_CUDA;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return SPLBM_ERR_CONFIG;
  }
}

inline int host_threads() {
  const unsigned n = std::thread::hardware_concurrency();
  return n == 0 ? 1 : static_cast<int>(std::min(n, 64u));
}

// fn(begin, end) over [0, n) split into equal contiguous chunks, like ThreadPool::parallel_for
// (reference thread_pool.hpp:45-88); results never depend on the split.
template <class F>
void parallel_for(std::size_t n, F&& fn, std::size_t min_chunk = 1) {
  const std::size_t workers =
      std::max<std::size_t>(1, std::min<std::size_t>(host_threads(), n / std::max<std::size_t>(min_chunk, 1)));
  if (workers <= 1) {
    if (n) fn(std::size_t{0}, n);
    return;
  }
  const std::size_t chunk = (n + workers - 1) / workers;
  std::vector<std::thread> th;
  th.reserve(workers);
  for (std::size_t w = 0; w < workers; ++w) {
    const std::size_t b = std::min(n, w * chunk), e = std::min(n, b + chunk);
    if (b < e) th.emplace_back([&fn, b, e] { fn(b, e); });
  }
  for (auto& t : th) t.join();
}

inline std::size_t raster_index(const int* dims, int x, int y, int z) {
  return static_cast<std::size_t>(x) +
         static_cast<std::size_t>(dims[0]) *
             (static_cast<std::size_t>(y) + static_cast<std::size_t>(dims[1]) * z);
}

}  // namespace splbm_host
