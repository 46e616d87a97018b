// Drop-in check: the reference's own engine API and test template (test_engine.cpp:34-39) run the
// B200 engine unchanged, and its results equal the reference TileEngineT2C<double> bit for bit.
// Built here (needs the reference headers) by tests/cpp/build_dropin.sh; run on the GPU box by
// tests/test_dropin_cpp.py. Exit code = number of failed cases.
#include <cstdio>
#include <cstring>
#include <memory>

#include "splbm/engine.hpp"
#include "splbm/engine_device.hpp"
#include "test_util.hpp"

using namespace splbm;

namespace {

template <class EngineT>
FieldData run_engine(EngineT& e, int steps, const NodeInit& init) {  // test_engine.cpp:34-39
  e.initialize(init);
  for (int s = 0; s < steps; ++s)
    if (!e.step()) std::printf("step %d failed\n", s);
  return e.fields();
}

bool same(const FieldData& a, const FieldData& b) {
  if (a.rho.size() != b.rho.size()) return false;
  return a.mask == b.mask && std::memcmp(a.rho.data(), b.rho.data(), a.rho.size() * 8) == 0 &&
         std::memcmp(a.ux.data(), b.ux.data(), a.ux.size() * 8) == 0 &&
         std::memcmp(a.uy.data(), b.uy.data(), a.uy.size() * 8) == 0 &&
         std::memcmp(a.uz.data(), b.uz.data(), a.uz.size() * 8) == 0;
}

int failures = 0;

template <class T = double>
void check_case(const char* name, const Geometry& g, int a, const FluidModel& m, Periodicity per,
                const NodeInit& init, int steps, bool single_copy = false) {
  TileEngineT2C<T> ref(g, a, m, per);
  TileEngineT2CDeviceT<T> dev(g, a, m, per, nullptr, 0, single_copy);
  const FieldData fr = run_engine(ref, steps, init);
  const FieldData fd = run_engine(dev, steps, init);
  const bool ok = same(fr, fd) && linf_rel_diff(fr, fd) == 0.0 &&
                  ref.tile_visits() == dev.tile_visits() && ref.padded_dims() == dev.padded_dims() &&
                  ref.current_step() == dev.current_step() && fr.total_mass() == fd.total_mass();
  std::printf("[%s] %s: %d steps, visits %llu, mass %.17g\n", ok ? "PASS" : "FAIL", name, steps,
              static_cast<unsigned long long>(dev.tile_visits()), fd.total_mass());
  if (!ok) ++failures;
}

}  // namespace

int main() {
  FluidModel m;
  m.tau = 0.8;
  const NodeInit uniform = [](int, int, int) { return std::make_pair(1.0, Eigen::Vector3d::Zero()); };
  {
    GenerateParams p;
    p.dims = {64, 64, 1};
    check_case("cavity2d 64^2 a=16", generate(GeometryKind::Cavity2D, p), 16, m, {}, uniform, 200);
  }
  {
    GenerateParams p;
    p.dims = {24, 24, 24};
    p.sphere_diameter = 8;
    p.target_porosity = 0.8;
    p.seed = 13;
    Periodicity per;
    per.x = per.y = per.z = true;
    FluidModel mi = m;
    mi.compressibility = Compressibility::Incompressible;
    check_case("ras 24^3 periodic wavy", generate(GeometryKind::Ras3D, p), 4, m, per,
               splbm::testing::wavy_init, 50);
    check_case("ras 24^3 periodic wavy incompressible", generate(GeometryKind::Ras3D, p), 4, mi,
               per, splbm::testing::wavy_init, 50);
    check_case("ras 24^3 periodic wavy, single copy (odd steps)", generate(GeometryKind::Ras3D, p),
               4, m, per, splbm::testing::wavy_init, 51, true);
    // TileEngineT2C<float> (the reference's precision=f32): float PDFs and arithmetic
    check_case<float>("f32 ras 24^3 periodic wavy", generate(GeometryKind::Ras3D, p), 4, m, per,
                      splbm::testing::wavy_init, 50);
    check_case<float>("f32 ras 24^3 periodic wavy incompressible, single copy",
                      generate(GeometryKind::Ras3D, p), 4, mi, per, splbm::testing::wavy_init, 31,
                      true);
    FluidModel mm = m;
    mm.collision = CollisionKind::MRT;
    check_case<float>("f32 MRT ras 24^3 periodic wavy", generate(GeometryKind::Ras3D, p), 4, mm, per,
                      splbm::testing::wavy_init, 40);
    check_case("MRT ras 24^3 periodic wavy", generate(GeometryKind::Ras3D, p), 4, mm, per,
               splbm::testing::wavy_init, 40);
  }
  {
    GenerateParams p;
    p.dims = {96, 48, 1};
    p.inlet_speed = 0.04;
    check_case<float>("f32 channel2d 96x48 a=16 (V/P boundaries)", generate(GeometryKind::Channel2D, p),
                      16, m, {}, [](int, int, int) { return std::make_pair(1.0, Eigen::Vector3d::Zero()); },
                      120);
    check_case<float>("f32 cavity3d 20^3 a=4", [] {
      GenerateParams c;
      c.dims = {20, 20, 20};
      return generate(GeometryKind::Cavity3D, c);
    }(), 4, m, {}, [](int, int, int) { return std::make_pair(1.0, Eigen::Vector3d::Zero()); }, 60);
  }
  check_case("closed box 3d a=2", splbm::testing::closed_box(3, {13, 11, 9}), 2, m, {},
             splbm::testing::wavy_init, 30);
  // the driver path: Engine<double> through a base pointer, as run_simulation holds it
  {
    GenerateParams p;
    p.dims = {128, 64, 1};
    p.inlet_speed = 0.04;
    const Geometry g = generate(GeometryKind::Channel2D, p);
    std::unique_ptr<Engine<double>> e = std::make_unique<TileEngineT2CDevice>(g, 16, m);
    e->initialize_uniform();
    bool ok = true;
    for (int s = 0; s < 100; ++s) ok &= e->step();
    TileEngineT2C<double> ref(g, 16, m);
    ref.initialize_uniform();
    for (int s = 0; s < 100; ++s) ref.step();
    const bool pass = ok && same(e->fields(), ref.fields());
    std::printf("[%s] Engine<double>* channel2d 128x64: 100 steps\n", pass ? "PASS" : "FAIL");
    if (!pass) ++failures;
  }
  std::printf("%d failures\n", failures);
  return failures;
}
