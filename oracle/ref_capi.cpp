// TEST INFRASTRUCTURE ONLY (oracle/). A C-ABI shim around the UNMODIFIED reference
// solver compiled in place from /root/reference/proj (see oracle/build_ref.sh).
// It exposes the reference's own public API (generate, build_tile_grid, tile_stats,
// TileEngineT2C / DenseEngine, run_simulation, the overhead model) to the Python
// parity tests and to `bench.py --impl reference`. Nothing in the product links it.
//
// The T2C PDF arrays are private (engine.hpp:544); they are read with the standard
// explicit-instantiation access idiom, without editing the reference.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>

#include "splbm/engine.hpp"
#include "splbm/overhead.hpp"
#include "splbm/tiling.hpp"
#include "test_util.hpp"  // wavy_init (tests/test_util.hpp:39-46)

using namespace splbm;

namespace {

thread_local std::string g_err;

template <class Tag, typename Tag::type M>
struct Rob {
  friend typename Tag::type get(Tag) { return M; }
};
struct T2CPdf {
  using type = std::vector<double> (TileEngineT2C<double>::*)[2];
  friend type get(T2CPdf);
};
struct T2CRead {
  using type = int TileEngineT2C<double>::*;
  friend type get(T2CRead);
};
struct MrtKernel {
  using type = std::vector<double> CollisionOperator<double>::*;
  friend type get(MrtKernel);
};
template struct Rob<MrtKernel, &CollisionOperator<double>::kernel_>;
template struct Rob<T2CPdf, &TileEngineT2C<double>::pdf_>;
template struct Rob<T2CRead, &TileEngineT2C<double>::read_>;
struct T2CPdfF {
  using type = std::vector<float> (TileEngineT2C<float>::*)[2];
  friend type get(T2CPdfF);
};
struct T2CReadF {
  using type = int TileEngineT2C<float>::*;
  friend type get(T2CReadF);
};
template struct Rob<T2CPdfF, &TileEngineT2C<float>::pdf_>;
template struct Rob<T2CReadF, &TileEngineT2C<float>::read_>;

int code_of(const std::exception& e) {
  if (dynamic_cast<const ConfigError*>(&e)) return 1;
  if (dynamic_cast<const DomainError*>(&e)) return 2;
  if (dynamic_cast<const NumericalError*>(&e)) return 3;
  if (dynamic_cast<const IoError*>(&e)) return 4;
  if (dynamic_cast<const ParseError*>(&e)) return 5;
  return 9;
}

#define GUARD(...)                   \
  try {                              \
    __VA_ARGS__;                     \
    return 0;                        \
  } catch (const std::exception& e) { \
    g_err = e.what();                \
    return code_of(e);               \
  }

Periodicity per_of(int mask) {
  Periodicity p;
  p.x = mask & 1;
  p.y = mask & 2;
  p.z = mask & 4;
  return p;
}

FluidModel model_of(double tau, int incompressible, int mrt) {
  FluidModel m;
  m.tau = tau;
  m.compressibility =
      incompressible ? Compressibility::Incompressible : Compressibility::QuasiCompressible;
  m.collision = mrt ? CollisionKind::MRT : CollisionKind::BGK;
  return m;
}

struct RefEngine {
  int method = 1;  // 0 dense, 1 t2c, 2 tgb
  std::unique_ptr<ThreadPool> pool;
  std::unique_ptr<Engine<double>> eng;   // T = double
  std::unique_ptr<Engine<float>> engf;   // T = float (the CLI's precision=f32)
  template <class F>
  auto with(F&& f) {  // the engine, whichever T it was built with
    return eng ? f(*eng) : f(*engf);
  }
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- geometry ----------------------------------------------------------------
int ref_generate(int kind, int nx, int ny, int nz, double lid, double inlet, double outlet_rho,
                 int diameter, double target, std::uint64_t seed, Geometry** out) {
  GUARD({
    GenerateParams p;
    p.dims = {nx, ny, nz};
    p.lid_speed = lid;
    p.inlet_speed = inlet;
    p.outlet_density = outlet_rho;
    p.sphere_diameter = diameter;
    p.target_porosity = target;
    p.seed = seed;
    *out = new Geometry(generate(static_cast<GeometryKind>(kind), p));
  })
}

int ref_geometry_from_raster(int d, const int* dims, const std::uint8_t* types,
                             const double* bc_vel, double bc_rho, Geometry** out) {
  GUARD({
    auto* g = new Geometry(d, {dims[0], dims[1], dims[2]});
    std::memcpy(g->types.data(), types, g->node_count());
    g->bc.velocity = Eigen::Vector3d(bc_vel[0], bc_vel[1], bc_vel[2]);
    g->bc.density = bc_rho;
    *out = g;
  })
}

int ref_geometry_load(const char* path, Geometry** out) {
  GUARD({ *out = new Geometry(load_geometry_file(path)); })
}

int ref_geometry_save(const Geometry* g, const char* path, int binary) {
  GUARD({
    save_geometry_file(*g, path, binary ? GeometryFormat::Binary : GeometryFormat::Text);
  })
}

void ref_geometry_info(const Geometry* g, int* d, int* dims, double* bc_vel, double* bc_rho) {
  *d = g->d;
  for (int k = 0; k < 3; ++k) dims[k] = g->dims[k];
  for (int k = 0; k < 3; ++k) bc_vel[k] = g->bc.velocity[k];
  *bc_rho = g->bc.density;
}

void ref_geometry_types(const Geometry* g, std::uint8_t* out) {
  std::memcpy(out, g->types.data(), g->node_count());
}

void ref_geometry_free(Geometry* g) { delete g; }

// ---- tiling --------------------------------------------------------------------
int ref_tile_grid(const Geometry* g, int a, int periodic, TileGrid** out) {
  GUARD({
    const auto& lat = detail::solver_lattice(g->d);
    *out = new TileGrid(build_tile_grid(*g, a, lat, per_of(periodic)));
  })
}

void ref_tile_grid_info(const TileGrid* tg, int* grid_dims, int* padded_dims,
                        std::uint64_t* n_tiles, int* n_tn) {
  for (int k = 0; k < 3; ++k) {
    grid_dims[k] = tg->grid_dims[k];
    padded_dims[k] = tg->padded_dims[k];
  }
  *n_tiles = tg->tiles.size();
  *n_tn = tg->n_tn;
}

// tile_map[C], origins[T*3], types[T*n_tn], fluid_count[T]
void ref_tile_grid_arrays(const TileGrid* tg, std::uint32_t* tile_map, std::int32_t* origins,
                          std::uint8_t* types, std::uint32_t* fluid_count) {
  std::memcpy(tile_map, tg->tile_map.data(), tg->tile_map.size() * sizeof(std::uint32_t));
  const std::size_t n_tn = static_cast<std::size_t>(tg->n_tn);
  for (std::size_t t = 0; t < tg->tiles.size(); ++t) {
    for (int k = 0; k < 3; ++k) origins[t * 3 + k] = tg->tiles[t].origin[k];
    std::memcpy(types + t * n_tn, tg->tiles[t].types.data(), n_tn);
    fluid_count[t] = tg->tiles[t].fluid_count;
  }
}

// neighbour table exactly as TileEngineT2C::build_neighbor_tables (engine.hpp:446-463)
void ref_tile_grid_nb(const TileGrid* tg, std::uint32_t* nb) {
  for (int cz = 0; cz < tg->grid_dims[2]; ++cz)
    for (int cy = 0; cy < tg->grid_dims[1]; ++cy)
      for (int cx = 0; cx < tg->grid_dims[0]; ++cx) {
        const TileIndex t = tg->tile_map[tg->cell_index(cx, cy, cz)];
        if (t == kEmptyTile) continue;
        for (int dz = -1; dz <= 1; ++dz)
          for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx)
              nb[static_cast<std::size_t>(t) * 27 + (dx + 1) + 3 * ((dy + 1) + 3 * (dz + 1))] =
                  tg->tile_at(cx + dx, cy + dy, cz + dz);
      }
}

// phi_t, eta_t, alpha_m, alpha_b, ratio_tiles, reduced_buffer_fraction, n_tiles, n_ftiles
void ref_tile_stats(const TileGrid* tg, double* out8) {
  const TileStats st = tile_stats(*tg);
  out8[0] = st.phi_t;
  out8[1] = st.eta_t;
  out8[2] = st.alpha_m;
  out8[3] = st.alpha_b;
  out8[4] = st.ratio_tiles;
  out8[5] = st.reduced_buffer_fraction;
  out8[6] = static_cast<double>(st.n_tiles);
  out8[7] = static_cast<double>(st.n_ftiles);
}

void ref_tile_grid_free(TileGrid* tg) { delete tg; }

void ref_degenerate_mask(const Geometry* g, int periodic, std::uint8_t* out) {
  const auto m = detail::degenerate_bc_mask(*g, detail::solver_lattice(g->d), per_of(periodic));
  std::memcpy(out, m.data(), m.size());
}

// ---- engines -----------------------------------------------------------------------
int ref_engine_create_p(const Geometry* g, int method, int a, double tau, int incompressible,
                        int mrt, int periodic, int threads, int f32, RefEngine** out) {
  GUARD({
    auto* e = new RefEngine;
    e->method = method;
    e->pool = std::make_unique<ThreadPool>(threads);
    SimConfig cfg;
    cfg.method = static_cast<Method>(method);
    cfg.tile = a;
    cfg.periodic = per_of(periodic);
    cfg.model = model_of(tau, incompressible, mrt);
    try {
      if (f32)
        e->engf = make_engine<float>(*g, cfg, e->pool.get());
      else
        e->eng = make_engine<double>(*g, cfg, e->pool.get());
    } catch (...) {
      delete e;
      throw;
    }
    *out = e;
  })
}

int ref_engine_create(const Geometry* g, int method, int a, double tau, int incompressible,
                      int mrt, int periodic, int threads, RefEngine** out) {
  return ref_engine_create_p(g, method, a, tau, incompressible, mrt, periodic, threads, 0, out);
}

// init_kind: 0 uniform (rho, u), 1 wavy_init (tests/test_util.hpp:39-46)
int ref_engine_initialize(RefEngine* e, int init_kind, double rho, const double* u) {
  GUARD({
    e->with([&](auto& eng) {
      if (init_kind == 1)
        eng.initialize(splbm::testing::wavy_init);
      else
        eng.initialize_uniform(rho, Eigen::Vector3d(u[0], u[1], u[2]));
      return 0;
    });
  })
}

// Initialise from a padded-grid (rho, ux, uy, uz) field: NodeInit(x,y,z) looks up the
// padded raster (x fastest), the same coordinates the engine evaluates (engine.hpp:336-352).
int ref_engine_initialize_fields(RefEngine* e, const int* pdims, const double* rho,
                                 const double* ux, const double* uy, const double* uz) {
  GUARD({
    const int px = pdims[0], py = pdims[1];
    const NodeInit init = [=](int x, int y, int z) {
      const std::size_t i = static_cast<std::size_t>(x) +
                            static_cast<std::size_t>(px) *
                                (static_cast<std::size_t>(y) + static_cast<std::size_t>(py) * z);
      return std::make_pair(rho[i], Eigen::Vector3d(ux[i], uy[i], uz[i]));
    };
    e->with([&](auto& eng) {
      eng.initialize(init);
      return 0;
    });
  })
}

// Runs n steps; *ok_out = 0 and *failed_step = absolute step number of the first failure.
int ref_engine_step(RefEngine* e, long n, int* ok_out, long* failed_step, double* seconds) {
  GUARD({
    *ok_out = 1;
    *failed_step = 0;
    double wall = 0.0;
    for (long s = 0; s < n; ++s) {
      const auto t0 = std::chrono::steady_clock::now();
      const bool ok = e->with([](auto& eng) { return eng.step(); });
      wall += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (!ok) {
        *ok_out = 0;
        *failed_step = e->with([](auto& eng) { return eng.current_step(); });
        break;
      }
    }
    if (seconds) *seconds = wall;
  })
}

long ref_engine_current_step(RefEngine* e) {
  return e->with([](auto& eng) { return eng.current_step(); });
}
std::uint64_t ref_engine_tile_visits(RefEngine* e) {
  return e->with([](auto& eng) { return eng.tile_visits(); });
}
void ref_engine_padded_dims(RefEngine* e, int* out) {
  const auto p = e->with([](auto& eng) { return eng.padded_dims(); });
  for (int k = 0; k < 3; ++k) out[k] = p[k];
}

int ref_engine_fields(RefEngine* e, double* rho, double* ux, double* uy, double* uz,
                      std::uint8_t* mask, double* mass) {
  GUARD({
    const FieldData f = e->with([](auto& eng) { return eng.fields(); });
    const std::size_t n = f.size();
    std::memcpy(rho, f.rho.data(), n * 8);
    std::memcpy(ux, f.ux.data(), n * 8);
    std::memcpy(uy, f.uy.data(), n * 8);
    std::memcpy(uz, f.uz.data(), n * 8);
    std::memcpy(mask, f.mask.data(), n);
    *mass = f.total_mass();
  })
}

// Current (read) PDF copy of a T2C engine, slot (t*q+i)*n_tn+p (engine.hpp:397-399).
std::uint64_t ref_engine_pdf(RefEngine* e, void* out) {
  if (e->engf) {  // TileEngineT2C<float>: float slots
    auto* t2c = dynamic_cast<TileEngineT2C<float>*>(e->engf.get());
    if (!t2c) return 0;
    const auto& pdf = t2c->*get(T2CPdfF());
    const int rd = t2c->*get(T2CReadF());
    if (out) std::memcpy(out, pdf[rd].data(), pdf[rd].size() * sizeof(float));
    return pdf[rd].size();
  }
  auto* t2c = dynamic_cast<TileEngineT2C<double>*>(e->eng.get());
  if (!t2c) return 0;
  const auto& pdf = t2c->*get(T2CPdf());
  const int rd = t2c->*get(T2CRead());
  if (out) std::memcpy(out, pdf[rd].data(), pdf[rd].size() * sizeof(double));
  return pdf[rd].size();
}

void ref_engine_free(RefEngine* e) { delete e; }

// ---- run_simulation (engine.hpp:609-655) ------------------------------------------------
// out6: wall_seconds, mlups, mass_initial, mass_final, mass_drift_rel, tile_visits
int ref_run_simulation(const Geometry* g, int method, int a, double tau, int incompressible,
                       int periodic, int threads, long steps, int init_kind, double* out6,
                       double* rho, double* ux, double* uy, double* uz) {
  GUARD({
    SimConfig cfg;
    cfg.method = static_cast<Method>(method);
    cfg.tile = a;
    cfg.steps = steps;
    cfg.threads = threads;
    cfg.periodic = per_of(periodic);
    cfg.model = model_of(tau, incompressible, 0);
    if (init_kind == 1) cfg.init = splbm::testing::wavy_init;
    const SimulationResult r = run_simulation<double>(*g, cfg);
    out6[0] = r.wall_seconds;
    out6[1] = r.mlups;
    out6[2] = r.mass_initial;
    out6[3] = r.mass_final;
    out6[4] = r.mass_drift_rel;
    out6[5] = static_cast<double>(r.tile_visits);
    if (rho) {
      const std::size_t n = r.fields.size();
      std::memcpy(rho, r.fields.rho.data(), n * 8);
      std::memcpy(ux, r.fields.ux.data(), n * 8);
      std::memcpy(uy, r.fields.uy.data(), n * 8);
      std::memcpy(uz, r.fields.uz.data(), n * 8);
    }
  })
}

// ---- overhead model (overhead.cpp) ---------------------------------------------------------
// out: m_node, b_node, delta_b, delta_b_bt, b.node_type, b.addressing, delta_m, predicted
int ref_overhead_t2c(int d, int a, double s_d, double s_t, double s_ti, double phi, double phi_t,
                     double alpha_m, double ratio_tiles, double* out8) {
  GUARD({
    CostParams p;
    p.lat = &lattice_descriptor(d == 2 ? Arrangement::D2Q9 : Arrangement::D3Q19);
    p.a = a;
    p.s_d = s_d;
    p.s_t = s_t;
    p.s_ti = s_ti;
    GeometryStats s = GeometryStats::manual(phi, phi_t, alpha_m, ratio_tiles);
    const NodeCosts nc = node_costs(p);
    const TileOverhead o = overhead_t2c(p, s);
    out8[0] = nc.m_node;
    out8[1] = nc.b_node;
    out8[2] = o.delta_b;
    out8[3] = o.delta_b_bt;
    out8[4] = o.b.node_type;
    out8[5] = o.b.addressing;
    out8[6] = o.delta_m;
    out8[7] = o.predicted_perf;
  })
}

int ref_bandwidth_utilization(int d, double s_d, double mlups, double b_peak, double* out) {
  GUARD({
    CostParams p;
    p.lat = &lattice_descriptor(d == 2 ? Arrangement::D2Q9 : Arrangement::D3Q19);
    p.s_d = s_d;
    *out = bandwidth_utilization(mlups, p, b_peak);
  })
}

// The MRT operator matrix K = M^-1 S M of CollisionOperator<double> (collision.cpp:86-113).
int ref_mrt_kernel(int d, double tau, const double* rates, int n_rates, double* K) {
  GUARD({
    FluidModel m = model_of(tau, 0, 1);
    if (rates) m.mrt_rates.assign(rates, rates + n_rates);
    const CollisionOperator<double> op(detail::solver_lattice(d), m);
    const auto& k = op.*get(MrtKernel());
    std::memcpy(K, k.data(), k.size() * sizeof(double));
  })
}

int ref_hardware_threads() { return static_cast<int>(std::thread::hardware_concurrency()); }

}  // extern "C"
