// Drop-in device engine for the reference solver's C++ API (proj/include/splbm/engine.hpp).
//
// TileEngineT2CDeviceT<T> derives from the reference's Engine<T> (T = double, or float for the
// reference's precision=f32 path) and has the TileEngineT2C constructor signature
// (engine.hpp:314-315); TileEngineT2CDevice = TileEngineT2CDeviceT<double>, so everything written against Engine<T> — the
// driver run_simulation's loop body, the CLI's bench_one, the test template run_engine<EngineT>
// (test_engine.cpp:34-39) — runs unchanged on a B200. The implementation is a thin, header-only
// shim over the C ABI of include/splbm_b200.h (libsplbm_b200.so); status codes are rethrown as the
// reference's exception types (errors.hpp:9-53). Include this header from a tree that provides the
// reference headers (and Eigen); see INTEGRATION.md for the make_engine / parse_method hook.
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "splbm/engine.hpp"
#include "splbm_b200.h"

namespace splbm {

namespace device_detail {

[[noreturn]] inline void rethrow(int code, long step = 0) {
  const std::string msg = splbm_last_error();
  switch (code) {
    case SPLBM_ERR_CONFIG: throw ConfigError(msg);
    case SPLBM_ERR_DOMAIN: throw DomainError(msg);
    case SPLBM_ERR_NUMERICAL: throw NumericalError(msg, step);
    case SPLBM_ERR_IO: throw IoError(msg);
    case SPLBM_ERR_PARSE: throw ParseError(msg);
    default: throw Error("splbm_b200: " + msg);
  }
}

inline void check(int code) {
  if (code != SPLBM_OK) rethrow(code);
}

}  // namespace device_detail

template <class T>
class TileEngineT2CDeviceT : public Engine<T> {
  static_assert(std::is_same_v<T, double> || std::is_same_v<T, float>, "T2C engines are f64/f32");

 public:
  // TileEngineT2C(g, a, model, periodic, pool) — the pool is accepted for signature parity; the
  // step runs on the GPU (`device` selects it).
  // single_copy selects the in-place AA propagation (half the HBM, same results).
  TileEngineT2CDeviceT(const Geometry& g, int a, const FluidModel& model, Periodicity periodic = {},
                       ThreadPool* /*pool*/ = nullptr, int device = 0, bool single_copy = false)
      : d_(g.d), dims_(g.dims), types_(g.types) {
    splbm_dev_desc desc{};
    desc.d = g.d;
    for (int k = 0; k < 3; ++k) desc.dims[k] = g.dims[k];
    desc.types = reinterpret_cast<const uint8_t*>(g.types.data());
    for (int k = 0; k < 3; ++k) desc.bc_velocity[k] = g.bc.velocity[k];
    desc.bc_density = g.bc.density;
    desc.tile = a;
    desc.tau = model.tau;
    desc.incompressible = model.compressibility == Compressibility::Incompressible;
    desc.periodic = (periodic.x ? 1 : 0) | (periodic.y ? 2 : 0) | (periodic.z ? 4 : 0);
    desc.device = device;
    desc.collision = model.collision == CollisionKind::MRT ? 1 : 0;
    desc.mrt_rates = model.mrt_rates.empty() ? nullptr : model.mrt_rates.data();
    desc.single_copy = single_copy ? 1 : 0;
    desc.single_precision = std::is_same_v<T, float> ? 1 : 0;
    if (desc.mrt_rates && static_cast<int>(model.mrt_rates.size()) != (g.d == 2 ? 9 : 19))
      throw ConfigError("mrt_rates must have one entry per moment");
    if (splbm_dev_info_size() != sizeof(splbm_dev_info))
      throw std::runtime_error("libsplbm_b200.so was built from another revision of splbm_b200.h");
    device_detail::check(splbm_dev_create(&desc, &e_));
    device_detail::check(splbm_dev_get_info(e_, &info_));
    tile_.resize(info_.n_tiles_stored);
    device_detail::check(splbm_dev_stored_tiles(e_, tile_.data()));
    origins_.resize(3 * std::max<uint64_t>(info_.n_tiles_global, 1));
    device_detail::check(splbm_dev_get_tile_grid(e_, nullptr, origins_.data(), nullptr, nullptr,
                                                 nullptr));
  }
  ~TileEngineT2CDeviceT() override { splbm_dev_destroy(e_); }
  TileEngineT2CDeviceT(const TileEngineT2CDeviceT&) = delete;
  TileEngineT2CDeviceT& operator=(const TileEngineT2CDeviceT&) = delete;

  // NodeInit evaluated at node_coords(tile, p) of every tile node, solid and padding included,
  // exactly as TileEngineT2C::initialize (engine.hpp:336-352); equilibrium on the device.
  void initialize(const NodeInit& init) override {
    const std::size_t n = static_cast<std::size_t>(info_.n_tiles_stored) * info_.n_tn;
    std::vector<double> rho(n), ux(n), uy(n), uz(n);
    const int a = info_.a;
    for (std::size_t s = 0; s < tile_.size(); ++s) {
      const int32_t* o = &origins_[3 * tile_[s]];
      for (int p = 0; p < info_.n_tn; ++p) {
        const auto [r, u] = init(o[0] + p % a, o[1] + (p / a) % a, o[2] + p / (a * a));
        const std::size_t k = s * info_.n_tn + p;
        rho[k] = r;
        ux[k] = u[0];
        uy[k] = u[1];
        uz[k] = u[2];
      }
    }
    device_detail::check(splbm_dev_initialize(e_, rho.data(), ux.data(), uy.data(), uz.data()));
    this->step_count_ = 0;
  }

  bool step() override {
    long failed = 0;
    return step_n(1, &failed);
  }

  // Batched stepping (not in the reference API): one host round trip per batch. Returns false
  // if a non-finite moment appeared; *failed_step = the first such step (engine.hpp:634).
  bool step_n(long n, long* failed_step) {
    int ok = 1;
    device_detail::check(splbm_dev_step(e_, n, &ok, failed_step));
    this->step_count_ = splbm_dev_current_step(e_);
    return ok != 0;
  }

  FieldData fields() const override {
    FieldData out;
    out.d = d_;
    out.dims = dims_;
    const std::size_t n = static_cast<std::size_t>(dims_[0]) * dims_[1] * dims_[2];
    out.mask.assign(n, 0);
    out.rho.assign(n, 0.0);
    out.ux.assign(n, 0.0);
    out.uy.assign(n, 0.0);
    out.uz.assign(n, 0.0);
    device_detail::check(splbm_dev_fields(e_, out.rho.data(), out.ux.data(), out.uy.data(),
                                          out.uz.data(), out.mask.data(), nullptr));
    return out;
  }

  std::array<int, 3> padded_dims() const override {
    return {info_.padded_dims[0], info_.padded_dims[1], info_.padded_dims[2]};
  }
  std::uint64_t tile_visits() const override { return splbm_dev_tile_visits(e_); }
  const splbm_dev_info& device_info() const { return info_; }
  splbm_dev_engine* handle() const { return e_; }

 private:
  splbm_dev_engine* e_ = nullptr;
  splbm_dev_info info_{};
  int d_;
  std::array<int, 3> dims_;
  std::vector<NodeType> types_;
  std::vector<uint64_t> tile_;
  std::vector<int32_t> origins_;
};

using TileEngineT2CDevice = TileEngineT2CDeviceT<double>;

}  // namespace splbm
