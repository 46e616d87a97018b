// Geometry input side of the path: the reference generators (restated, bit-exact rasters),
// two new generators the BASELINE configs need (3D duct, 2D vessel tree), and the SPLB v1 /
// text formats (reference geometry.cpp).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "common.h"

using namespace splbm_host;

namespace {

constexpr uint8_t kSolid = 0, kFluid = 1, kVel = 2, kPres = 3;

struct Raster {
  int d = 2;
  int dims[3] = {0, 0, 1};
  uint8_t* t = nullptr;
  uint8_t& at(int x, int y, int z = 0) { return t[raster_index(dims, x, y, z)]; }
  std::size_t n() const { return static_cast<std::size_t>(dims[0]) * dims[1] * dims[2]; }
};

// generate_cavity (geometry.cpp:199-224)
void cavity(Raster& g, double lid, double* vel) {
  for (int k = 0; k < g.d; ++k)
    if (g.dims[k] < 3) throw config_error("cavity dimensions must be at least 3");
  const int nx = g.dims[0], ny = g.dims[1], nz = g.dims[2];
  std::fill(g.t, g.t + g.n(), kFluid);
  for (int z = 0; z < nz; ++z)
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x) {
        const bool side = (x == 0 || x == nx - 1) || (g.d == 3 && (y == 0 || y == ny - 1));
        const bool floor = (g.d == 2) ? (y == 0) : (z == 0);
        const bool top = (g.d == 2) ? (y == ny - 1) : (z == nz - 1);
        if (side || (floor && !side))
          g.at(x, y, z) = kSolid;
        else if (top)
          g.at(x, y, z) = kVel;
      }
  vel[0] = lid;
  vel[1] = vel[2] = 0.0;
}

// generate_channel (geometry.cpp:226-245)
void channel2d(Raster& g, double inlet, double outlet, double* vel, double* rho) {
  if (g.dims[0] < 3 || g.dims[1] < 3) throw config_error("channel dimensions must be at least 3");
  const int nx = g.dims[0], ny = g.dims[1];
  std::fill(g.t, g.t + g.n(), kFluid);
  for (int y = 0; y < ny; ++y)
    for (int x = 0; x < nx; ++x) {
      if (y == 0 || y == ny - 1)
        g.at(x, y) = kSolid;
      else if (x == 0)
        g.at(x, y) = kVel;
      else if (x == nx - 1)
        g.at(x, y) = kPres;
    }
  vel[0] = inlet;
  vel[1] = vel[2] = 0.0;
  *rho = outlet;
}

// New: 3D duct with bounce-back walls at y, z in {0, n-1}, VelocityBC inlet at
// x = 0 and PressureBC outlet at x = nx-1 on the non-wall cross-section (BASELINE configs[1]).
void channel3d(Raster& g, double inlet, double outlet, double* vel, double* rho) {
  for (int k = 0; k < 3; ++k)
    if (g.dims[k] < 3) throw config_error("channel dimensions must be at least 3");
  const int nx = g.dims[0], ny = g.dims[1], nz = g.dims[2];
  for (int z = 0; z < nz; ++z)
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x) {
        uint8_t t = kFluid;
        if (y == 0 || y == ny - 1 || z == 0 || z == nz - 1)
          t = kSolid;
        else if (x == 0)
          t = kVel;
        else if (x == nx - 1)
          t = kPres;
        g.at(x, y, z) = t;
      }
  vel[0] = inlet;
  vel[1] = vel[2] = 0.0;
  *rho = outlet;
}

// canonical (geometry.cpp:195-197)
double canonical(std::mt19937_64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }

// generate_ras (geometry.cpp:251-326): periodic overlapping spheres until phi <= target + 0.01,
// with the same skip/retry rule, RNG stream and marking order (bit-exact raster).
void ras3d(Raster& g, int diameter, double target, uint64_t seed) {
  const int* dims = g.dims;
  const int min_dim = std::min({dims[0], dims[1], dims[2]});
  if (diameter < 2) throw config_error("sphere diameter must be at least 2");
  if (diameter >= min_dim)
    throw config_error("sphere diameter must be smaller than the smallest dimension");
  if (!(target > 0.0 && target < 1.0)) throw config_error("target porosity must lie in (0, 1)");
  std::fill(g.t, g.t + g.n(), kFluid);
  const std::size_t n_total = g.n();
  const double r = diameter / 2.0;
  const double r2 = r * r;
  std::mt19937_64 rng(seed);
  std::size_t solid = 0;

  auto mark_sphere = [&](double cx, double cy, double cz, bool commit) -> std::size_t {
    std::size_t newly = 0;
    const int x0 = static_cast<int>(std::floor(cx - r)), x1 = static_cast<int>(std::ceil(cx + r));
    const int y0 = static_cast<int>(std::floor(cy - r)), y1 = static_cast<int>(std::ceil(cy + r));
    const int z0 = static_cast<int>(std::floor(cz - r)), z1 = static_cast<int>(std::ceil(cz + r));
    for (int z = z0; z <= z1; ++z) {
      const double dz = z - cz;
      const int wz = ((z % dims[2]) + dims[2]) % dims[2];
      for (int y = y0; y <= y1; ++y) {
        const double dy = y - cy;
        const int wy = ((y % dims[1]) + dims[1]) % dims[1];
        for (int x = x0; x <= x1; ++x) {
          const double dx = x - cx;
          if (dx * dx + dy * dy + dz * dz > r2) continue;
          const int wx = ((x % dims[0]) + dims[0]) % dims[0];
          uint8_t& t = g.at(wx, wy, wz);
          if (t != kSolid) {
            ++newly;
            if (commit) t = kSolid;
          }
        }
      }
    }
    return newly;
  };

  const double upper = target + 0.01;
  const double lower = target - 0.01;
  int skips = 0;
  double best_cx = 0, best_cy = 0, best_cz = 0;
  double best_err = 2.0;
  while (static_cast<double>(n_total - solid) / n_total > upper) {
    const double cx = canonical(rng) * dims[0];
    const double cy = canonical(rng) * dims[1];
    const double cz = canonical(rng) * dims[2];
    const std::size_t newly = mark_sphere(cx, cy, cz, false);
    const double phi_after = static_cast<double>(n_total - solid - newly) / n_total;
    if (phi_after >= lower || skips >= 2000) {
      solid += mark_sphere(cx, cy, cz, true);
      skips = 0;
      best_err = 2.0;
      continue;
    }
    const double err = std::abs(phi_after - target);
    if (err < best_err) {
      best_err = err;
      best_cx = cx;
      best_cy = cy;
      best_cz = cz;
    }
    if (++skips == 2000) {
      solid += mark_sphere(best_cx, best_cy, best_cz, true);
      skips = 0;
      best_err = 2.0;
    }
  }
}

// New: seeded 2D vessel network, chip-like. Trees enter at
// x = 0 (VelocityBC), branch binarily with widths narrowing from `width0` to >= 8 nodes, and
// every terminal branch runs out to x = nx-1 (PressureBC). Trees are added until the non-solid
// fraction reaches the target porosity. Deterministic for a fixed seed.
void vessel2d(Raster& g, double target, uint64_t seed, double inlet, double outlet, double* vel,
              double* rho) {
  const int nx = g.dims[0], ny = g.dims[1];
  if (nx < 64 || ny < 64) throw config_error("vessel tree needs at least 64x64 nodes");
  if (!(target > 0.0 && target < 1.0)) throw config_error("target porosity must lie in (0, 1)");
  std::fill(g.t, g.t + g.n(), kSolid);
  std::mt19937_64 rng(seed);
  std::size_t fluid = 0;
  const std::size_t n_total = g.n();
  const double width0 = std::max(8.0, std::min(32.0, ny / 16.0));

  auto capsule = [&](double x0, double y0, double x1, double y1, double r) {
    const int bx0 = std::max(0, static_cast<int>(std::floor(std::min(x0, x1) - r)));
    const int bx1 = std::min(nx - 1, static_cast<int>(std::ceil(std::max(x0, x1) + r)));
    const int by0 = std::max(0, static_cast<int>(std::floor(std::min(y0, y1) - r)));
    const int by1 = std::min(ny - 1, static_cast<int>(std::ceil(std::max(y0, y1) + r)));
    const double vx = x1 - x0, vy = y1 - y0;
    const double len2 = vx * vx + vy * vy;
    for (int y = by0; y <= by1; ++y)
      for (int x = bx0; x <= bx1; ++x) {
        double s = len2 > 0 ? ((x - x0) * vx + (y - y0) * vy) / len2 : 0.0;
        s = std::min(1.0, std::max(0.0, s));
        const double px = x0 + s * vx - x, py = y0 + s * vy - y;
        if (px * px + py * py <= r * r) {
          uint8_t& t = g.at(x, y);
          if (t == kSolid) {
            t = kFluid;
            ++fluid;
          }
        }
      }
  };

  struct Seg {
    double x, y, ang, w;
    int depth;
  };
  int trees = 0;
  while (static_cast<double>(fluid) / n_total < target && trees < 4096) {
    ++trees;
    std::vector<Seg> stack{{0.0, (0.1 + 0.8 * canonical(rng)) * (ny - 1), 0.0, width0, 0}};
    while (!stack.empty()) {
      Seg s = stack.back();
      stack.pop_back();
      const bool terminal = s.w * 0.8 < 8.0 || s.depth >= 8 || s.x > 0.8 * nx;
      double len = terminal ? 1e9 : (0.08 + 0.08 * canonical(rng)) * nx;
      double ex = s.x + std::cos(s.ang) * len, ey = s.y + std::sin(s.ang) * len;
      if (terminal || ex >= nx - 1) {  // run out to the outlet plane
        const double c = std::max(std::cos(s.ang), 0.2);
        ex = nx - 1 + s.w;
        ey = s.y + std::sin(s.ang) / c * (ex - s.x);
      }
      capsule(s.x, s.y, ex, ey, s.w / 2.0);
      if (terminal || ex >= nx - 1) continue;
      const double spread = 0.35 + 0.35 * canonical(rng);
      const double w = std::max(8.0, s.w * 0.8);
      double a0 = std::clamp(s.ang + spread, -1.0, 1.0), a1 = std::clamp(s.ang - spread, -1.0, 1.0);
      stack.push_back({ex, ey, a0, w, s.depth + 1});
      stack.push_back({ex, ey, a1, w, s.depth + 1});
    }
  }
  for (int y = 0; y < ny; ++y) {
    if (g.at(0, y) != kSolid) g.at(0, y) = kVel;
    if (g.at(nx - 1, y) != kSolid) g.at(nx - 1, y) = kPres;
  }
  vel[0] = inlet;
  vel[1] = vel[2] = 0.0;
  *rho = outlet;
}

// ---- formats (geometry.cpp:49-191) ---------------------------------------------------------
const char kMagic[4] = {'S', 'P', 'L', 'B'};

char type_char(uint8_t t) { return t == 0 ? '#' : t == 1 ? '.' : t == 2 ? 'V' : 'P'; }

struct Loaded {
  int d = 2;
  int dims[3] = {0, 0, 1};
  std::vector<uint8_t> types;
  double vel[3] = {0, 0, 0};
  double rho = 1.0;
};

std::string perr(const std::string& w, long line, long col) {
  return w + " (line " + std::to_string(line) + ", column " + std::to_string(col) + ")";
}

Loaded load_text(const std::string& bytes) {
  std::istringstream in(bytes);
  std::string line;
  long line_no = 0;
  if (!std::getline(in, line)) throw parse_error(perr("empty geometry file", 1, 1));
  ++line_no;
  std::istringstream header(line);
  std::string tag;
  header >> tag;
  Loaded g;
  if (tag == "D2") g.d = 2;
  else if (tag == "D3") g.d = 3;
  else throw parse_error(perr("expected 'D2' or 'D3' header", line_no, 1));
  header >> g.dims[0] >> g.dims[1];
  if (g.d == 3) header >> g.dims[2];
  if (header.fail() || g.dims[0] <= 0 || g.dims[1] <= 0 || g.dims[2] <= 0)
    throw parse_error(perr("invalid dimensions in header", line_no, 1));
  g.types.assign(static_cast<std::size_t>(g.dims[0]) * g.dims[1] * g.dims[2], kFluid);
  for (int z = 0; z < g.dims[2]; ++z) {
    if (z > 0) {
      if (!std::getline(in, line)) throw parse_error(perr("missing slice separator", line_no + 1, 1));
      ++line_no;
      if (!line.empty()) throw parse_error(perr("expected blank line between slices", line_no, 1));
    }
    for (int y = 0; y < g.dims[1]; ++y) {
      if (!std::getline(in, line))
        throw parse_error(perr("unexpected end of file: missing row", line_no + 1, 1));
      ++line_no;
      if (static_cast<int>(line.size()) != g.dims[0])
        throw parse_error(perr("row has " + std::to_string(line.size()) + " characters, expected " +
                                   std::to_string(g.dims[0]),
                               line_no, static_cast<long>(line.size()) + 1));
      for (int x = 0; x < g.dims[0]; ++x) {
        const char c = line[static_cast<std::size_t>(x)];
        uint8_t t;
        if (c == '#') t = kSolid;
        else if (c == '.') t = kFluid;
        else if (c == 'V') t = kVel;
        else if (c == 'P') t = kPres;
        else throw parse_error(perr(std::string("unknown node character '") + c + "'", line_no, x + 1));
        g.types[raster_index(g.dims, x, y, z)] = t;
      }
    }
  }
  while (std::getline(in, line)) {
    ++line_no;
    if (line.empty()) continue;
    std::istringstream ls(line);
    std::string key;
    ls >> key;
    if (key == "vel") {
      ls >> g.vel[0] >> g.vel[1];
      if (g.d == 3) ls >> g.vel[2];
      if (ls.fail()) throw parse_error(perr("invalid 'vel' line", line_no, 1));
    } else if (key == "rho") {
      ls >> g.rho;
      if (ls.fail()) throw parse_error(perr("invalid 'rho' line", line_no, 1));
    } else {
      throw parse_error(perr("unknown trailing line '" + key + "'", line_no, 1));
    }
  }
  return g;
}

uint32_t rd_u32(const unsigned char* p) {
  return static_cast<uint32_t>(p[0]) | (static_cast<uint32_t>(p[1]) << 8) |
         (static_cast<uint32_t>(p[2]) << 16) | (static_cast<uint32_t>(p[3]) << 24);
}

Loaded load_binary(const std::string& bytes) {
  constexpr std::size_t hs = 18;
  if (bytes.size() < hs) throw parse_error("truncated binary header");
  if (std::memcmp(bytes.data(), kMagic, 4) != 0) throw parse_error("bad magic, expected 'SPLB'");
  const auto* p = reinterpret_cast<const unsigned char*>(bytes.data());
  if (p[4] != 1) throw parse_error("unsupported version " + std::to_string(p[4]));
  Loaded g;
  g.d = p[5];
  if (g.d != 2 && g.d != 3) throw parse_error("dimension must be 2 or 3");
  for (int k = 0; k < 3; ++k) {
    g.dims[k] = static_cast<int>(rd_u32(p + 6 + 4 * k));
    if (g.dims[k] <= 0) throw parse_error("zero dimension in header");
  }
  if (g.d == 2 && g.dims[2] != 1) throw parse_error("2D geometry requires nz = 1");
  const std::size_t n = static_cast<std::size_t>(g.dims[0]) * g.dims[1] * g.dims[2];
  if (bytes.size() - hs != n)
    throw parse_error("dimension mismatch: header declares " + std::to_string(n) +
                      " nodes, payload has " + std::to_string(bytes.size() - hs) + " bytes");
  g.types.resize(n);
  for (std::size_t i = 0; i < n; ++i) {
    const unsigned char c = p[hs + i];
    if (c > 3)
      throw parse_error("invalid node type code " + std::to_string(c) + " at offset " +
                        std::to_string(hs + i));
    g.types[i] = c;
  }
  return g;
}

std::string save_text(int d, const int* dims, const uint8_t* types, const double* vel, double rho) {
  std::ostringstream out;
  out << (d == 2 ? "D2 " : "D3 ") << dims[0] << ' ' << dims[1];
  if (d == 3) out << ' ' << dims[2];
  out << '\n';
  bool has_vel = false, has_rho = false;
  for (int z = 0; z < dims[2]; ++z) {
    if (z > 0) out << '\n';
    for (int y = 0; y < dims[1]; ++y) {
      for (int x = 0; x < dims[0]; ++x) {
        const uint8_t t = types[raster_index(dims, x, y, z)];
        has_vel |= t == kVel;
        has_rho |= t == kPres;
        out << type_char(t);
      }
      out << '\n';
    }
  }
  out.precision(17);
  if (has_vel) {
    out << "vel " << vel[0] << ' ' << vel[1];
    if (d == 3) out << ' ' << vel[2];
    out << '\n';
  }
  if (has_rho) out << "rho " << rho << '\n';
  return out.str();
}

std::string save_binary(int d, const int* dims, const uint8_t* types) {
  std::string out(kMagic, 4);
  out.push_back(1);
  out.push_back(static_cast<char>(d));
  for (int k = 0; k < 3; ++k) {
    const uint32_t v = static_cast<uint32_t>(dims[k]);
    for (int b = 0; b < 4; ++b) out.push_back(static_cast<char>((v >> (8 * b)) & 0xff));
  }
  out.append(reinterpret_cast<const char*>(types),
             static_cast<std::size_t>(dims[0]) * dims[1] * dims[2]);
  return out;
}

}  // namespace

extern "C" {

int splbm_generate(int kind, const splbm_generate_params* p, uint8_t* types_out, int* d_out,
                   double bc_velocity_out[3], double* bc_density_out) {
  return guarded([&] {
    if (!p || !types_out) throw config_error("null argument");
    Raster g;
    g.d = (kind == SPLBM_GEOM_CAVITY2D || kind == SPLBM_GEOM_CHANNEL2D ||
           kind == SPLBM_GEOM_VESSEL2D) ? 2 : 3;
    g.dims[0] = p->dims[0];
    g.dims[1] = p->dims[1];
    g.dims[2] = g.d == 2 ? 1 : p->dims[2];
    for (int k = 0; k < 3; ++k)
      if (g.dims[k] <= 0) throw config_error("dimensions must be positive");
    g.t = types_out;
    double vel[3] = {0.0, 0.0, 0.0};
    double rho = 1.0;
    switch (kind) {
      case SPLBM_GEOM_CAVITY2D:
      case SPLBM_GEOM_CAVITY3D: cavity(g, p->lid_speed, vel); break;
      case SPLBM_GEOM_CHANNEL2D: channel2d(g, p->inlet_speed, p->outlet_density, vel, &rho); break;
      case SPLBM_GEOM_RAS3D: ras3d(g, p->sphere_diameter, p->target_porosity, p->seed); break;
      case SPLBM_GEOM_CHANNEL3D: channel3d(g, p->inlet_speed, p->outlet_density, vel, &rho); break;
      case SPLBM_GEOM_VESSEL2D:
        vessel2d(g, p->target_porosity, p->seed, p->inlet_speed, p->outlet_density, vel, &rho);
        break;
      default: throw config_error("unknown geometry kind");
    }
    if (d_out) *d_out = g.d;
    if (bc_velocity_out)
      for (int k = 0; k < 3; ++k) bc_velocity_out[k] = vel[k];
    if (bc_density_out) *bc_density_out = rho;
  });
}

int splbm_geometry_load(const char* path, int* d_out, int dims_out[3], uint8_t* types_out,
                        double bc_velocity_out[3], double* bc_density_out) {
  return guarded([&] {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw io_error(std::string("cannot open geometry file: ") + path);
    std::ostringstream buf;
    buf << in.rdbuf();
    const std::string bytes = buf.str();
    const bool binary = bytes.size() >= 4 && std::memcmp(bytes.data(), kMagic, 4) == 0;
    Loaded g = binary ? load_binary(bytes) : load_text(bytes);
    if (d_out) *d_out = g.d;
    if (dims_out)
      for (int k = 0; k < 3; ++k) dims_out[k] = g.dims[k];
    if (types_out) std::memcpy(types_out, g.types.data(), g.types.size());
    if (bc_velocity_out)
      for (int k = 0; k < 3; ++k) bc_velocity_out[k] = g.vel[k];
    if (bc_density_out) *bc_density_out = g.rho;
  });
}

int splbm_geometry_save(const char* path, int binary, int d, const int dims[3],
                        const uint8_t* types, const double bc_velocity[3], double bc_density) {
  return guarded([&] {
    const double zero[3] = {0, 0, 0};
    const std::string bytes = binary ? save_binary(d, dims, types)
                                     : save_text(d, dims, types, bc_velocity ? bc_velocity : zero,
                                                 bc_density);
    std::ofstream out(path, std::ios::binary);
    if (!out) throw io_error(std::string("cannot write geometry file: ") + path);
    out.write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
    if (!out) throw io_error(std::string("write failed: ") + path);
  });
}

}  // extern "C"
