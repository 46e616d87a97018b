/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the T2C hot path.
 *
 * A plain-C restatement of the reference solver's T2C time step (arXiv 1703.08015,
 * reference `splbm`, /root/reference/proj). Every function cites the reference
 * file:line it follows. It is pinned (tests/test_oracle.py) against
 *   - the reference itself compiled in place (oracle/_ref, oracle/build_ref.sh), and
 *   - the golden digests recorded in SURVEY.md Appendix B / tests/golden/.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs may
 * load this library; the product (paper_1703_08015_b200/) never does.
 *
 * Arithmetic is written out literally in the reference's operation order (including the
 * products by zero direction components) and compiled with -ffp-contract=off, so it is
 * bit-identical to the reference built with its CMake Release flags.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EMPTY_TILE 0xffffffffu /* kEmptyTile, tiling.hpp:16 */

/* ---- lattice constants: lattice.cpp:18-25 (D2Q9), 33-42 (D3Q19) ---------------------- */
static const int E2[9][3] = {{0, 0, 0},  {1, 0, 0},   {-1, 0, 0}, {0, 1, 0},  {0, -1, 0},
                             {1, 1, 0},  {-1, -1, 0}, {1, -1, 0}, {-1, 1, 0}};
static const int E3[19][3] = {{0, 0, 0},  {1, 0, 0},   {-1, 0, 0}, {0, 1, 0},  {0, -1, 0},
                              {0, 0, 1},  {0, 0, -1},  {1, 1, 0},  {-1, -1, 0}, {1, -1, 0},
                              {-1, 1, 0}, {1, 0, 1},   {-1, 0, -1}, {1, 0, -1}, {-1, 0, 1},
                              {0, 1, 1},  {0, -1, -1}, {0, 1, -1}, {0, -1, 1}};

typedef struct {
  int d, q;
  const int (*e)[3];
  double w[19];
  int opp[19];
} lattice_t;

static void lattice_init(lattice_t* L, int d) {
  L->d = d;
  if (d == 2) {
    L->q = 9;
    L->e = E2;
    L->w[0] = 4.0 / 9.0;
    for (int i = 1; i <= 4; ++i) L->w[i] = 1.0 / 9.0;
    for (int i = 5; i <= 8; ++i) L->w[i] = 1.0 / 36.0;
  } else {
    L->q = 19;
    L->e = E3;
    for (int i = 0; i < 19; ++i) L->w[i] = 1.0 / 36.0;
    L->w[0] = 1.0 / 3.0;
    for (int i = 1; i <= 6; ++i) L->w[i] = 1.0 / 18.0;
  }
  /* opposite by search, lattice.cpp:65-74 */
  for (int i = 0; i < L->q; ++i)
    for (int j = 0; j < L->q; ++j)
      if (L->e[j][0] == -L->e[i][0] && L->e[j][1] == -L->e[i][1] && L->e[j][2] == -L->e[i][2]) {
        L->opp[i] = j;
        break;
      }
}

/* ---- tile cover: tiling.cpp:95-141 ------------------------------------------------------ */
void oracle_tile_dims(int d, const int* dims, int a, int* grid_dims, int* padded_dims) {
  for (int k = 0; k < 3; ++k) {
    const int extent = (k == 2 && d == 2) ? 1 : dims[k];
    const int te = (k == 2 && d == 2) ? 1 : a;
    grid_dims[k] = (extent + te - 1) / te;
    padded_dims[k] = grid_dims[k] * te;
  }
}

/* Returns the number of non-empty tiles; outputs sized for the worst case (all cells).
 * Validation as tiling.cpp:87-93 (returns -1 on a ConfigError condition). */
int64_t oracle_build_tiles(const uint8_t* types, int d, const int* dims, int a, int periodic,
                           uint32_t* tile_map, int32_t* origins, uint8_t* ttypes,
                           uint32_t* fluid_count) {
  if (a < 2) return -1;
  for (int k = 0; k < d; ++k)
    if (((periodic >> k) & 1) && dims[k] % a != 0) return -1;
  int gd[3], pd[3];
  oracle_tile_dims(d, dims, a, gd, pd);
  const int az = d == 3 ? a : 1;
  const int64_t n_tn = (int64_t)a * a * az;
  int64_t T = 0;
  for (int cz = 0; cz < gd[2]; ++cz)
    for (int cy = 0; cy < gd[1]; ++cy)
      for (int cx = 0; cx < gd[0]; ++cx) {
        uint8_t* tt = ttypes + T * n_tn;
        memset(tt, 0, (size_t)n_tn); /* padding is Solid */
        uint32_t fc = 0;
        for (int lz = 0; lz < az; ++lz) {
          const int z = cz * az + lz;
          if (z >= dims[2]) continue;
          for (int ly = 0; ly < a; ++ly) {
            const int y = cy * a + ly;
            if (y >= dims[1]) continue;
            for (int lx = 0; lx < a; ++lx) {
              const int x = cx * a + lx;
              if (x >= dims[0]) continue;
              const uint8_t t = types[(size_t)x + (size_t)dims[0] * ((size_t)y + (size_t)dims[1] * z)];
              tt[lx + a * (ly + a * lz)] = t;
              if (t != 0) ++fc;
            }
          }
        }
        const size_t cell = (size_t)cx + (size_t)gd[0] * ((size_t)cy + (size_t)gd[1] * cz);
        if (fc > 0) {
          tile_map[cell] = (uint32_t)T;
          origins[3 * T + 0] = cx * a;
          origins[3 * T + 1] = cy * a;
          origins[3 * T + 2] = cz * az;
          fluid_count[T] = fc;
          ++T;
        } else {
          tile_map[cell] = EMPTY_TILE;
        }
      }
  return T;
}

/* tile_at with per-axis wrap: tiling.hpp:93-102 */
static uint32_t tile_at(const int* gd, int periodic, const uint32_t* tile_map, int cx, int cy,
                        int cz) {
  int c[3] = {cx, cy, cz};
  for (int k = 0; k < 3; ++k) {
    if (c[k] < 0 || c[k] >= gd[k]) {
      if (!((periodic >> k) & 1)) return EMPTY_TILE;
      c[k] = ((c[k] % gd[k]) + gd[k]) % gd[k];
    }
  }
  return tile_map[(size_t)c[0] + (size_t)gd[0] * ((size_t)c[1] + (size_t)gd[1] * c[2])];
}

/* 27-neighbour tile table: engine.hpp:446-463 */
void oracle_nb_table(const int* gd, int periodic, const uint32_t* tile_map, uint32_t* nb) {
  for (int cz = 0; cz < gd[2]; ++cz)
    for (int cy = 0; cy < gd[1]; ++cy)
      for (int cx = 0; cx < gd[0]; ++cx) {
        const uint32_t t = tile_map[(size_t)cx + (size_t)gd[0] * ((size_t)cy + (size_t)gd[1] * cz)];
        if (t == EMPTY_TILE) continue;
        for (int dz = -1; dz <= 1; ++dz)
          for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx)
              nb[(size_t)t * 27 + (dx + 1) + 3 * ((dy + 1) + 3 * (dz + 1))] =
                  tile_at(gd, periodic, tile_map, cx + dx, cy + dy, cz + dz);
      }
}

/* degenerate BC mask: engine.hpp:110-140 */
void oracle_degenerate_mask(const uint8_t* types, int d, const int* dims, int periodic,
                            uint8_t* mask) {
  lattice_t L;
  lattice_init(&L, d);
  const size_t n = (size_t)dims[0] * dims[1] * dims[2];
  memset(mask, 0, n);
  for (int z = 0; z < dims[2]; ++z)
    for (int y = 0; y < dims[1]; ++y)
      for (int x = 0; x < dims[0]; ++x) {
        const size_t node = (size_t)x + (size_t)dims[0] * ((size_t)y + (size_t)dims[1] * z);
        const uint8_t t = types[node];
        if (t != 2 && t != 3) continue;
        int degenerate = 0;
        for (int i = 1; i < L.q && !degenerate; ++i) {
          int s[3] = {x - L.e[i][0], y - L.e[i][1], z - L.e[i][2]};
          int outside = 0;
          for (int k = 0; k < 3; ++k) {
            if (s[k] < 0 || s[k] >= dims[k]) {
              if ((periodic >> k) & 1) {
                s[k] = ((s[k] % dims[k]) + dims[k]) % dims[k];
              } else {
                outside = 1;
                break;
              }
            }
          }
          degenerate = outside ||
                       types[(size_t)s[0] + (size_t)dims[0] * ((size_t)s[1] + (size_t)dims[1] * s[2])] == 0;
        }
        if (degenerate) mask[node] = 1;
      }
}

/* ---- node physics and the T2C sweep, for T = double and T = float (oracle/t2c_real.inc) ---- */
#define REAL double
#define SFX(name) name
#include "t2c_real.inc"
#undef REAL
#undef SFX
#define REAL float
#define SFX(name) name##_f32
#include "t2c_real.inc"
#undef REAL
#undef SFX

/* FieldData::total_mass: fields.hpp:25-31 (sequential, raster order) */
double oracle_total_mass(size_t n, const double* rho, const uint8_t* mask) {
  double m = 0.0;
  for (size_t i = 0; i < n; ++i)
    if (mask[i]) m += rho[i];
  return m;
}

/* ---- digests --------------------------------------------------------- */
/* FNV-1a 64 fed one unsigned word per value. */
uint64_t oracle_fnv_u32(uint64_t h, const uint32_t* v, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    h ^= (uint64_t)v[i];
    h *= 1099511628211ull;
  }
  return h;
}
uint64_t oracle_fnv_u8(uint64_t h, const uint8_t* v, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    h ^= (uint64_t)v[i];
    h *= 1099511628211ull;
  }
  return h;
}
/* tile-map digest: tile_map[], then per tile origin[0..2] and types[0..n_tn) */
uint64_t oracle_tilemap_digest(size_t C, const uint32_t* tile_map, int64_t T, int n_tn,
                               const int32_t* origins, const uint8_t* ttypes) {
  uint64_t h = 1469598103934665603ull;
  h = oracle_fnv_u32(h, tile_map, C);
  for (int64_t t = 0; t < T; ++t) {
    h = oracle_fnv_u32(h, (const uint32_t*)(origins + 3 * t), 3);
    h = oracle_fnv_u8(h, ttypes + (size_t)t * n_tn, (size_t)n_tn);
  }
  return h;
}
/* fields digest: per non-solid raster node the bit patterns of rho, ux, uy, uz */
uint64_t oracle_fields_digest(size_t n, const uint8_t* mask, const double* rho,
                              const double* ux, const double* uy, const double* uz) {
  uint64_t h = 1469598103934665603ull;
  for (size_t i = 0; i < n; ++i) {
    if (!mask[i]) continue;
    const double* f[4] = {rho + i, ux + i, uy + i, uz + i};
    for (int k = 0; k < 4; ++k) {
      uint64_t b;
      memcpy(&b, f[k], 8);
      h ^= b;
      h *= 1099511628211ull;
    }
  }
  return h;
}

/* wavy_init: tests/test_util.hpp:39-46, evaluated at integer node coordinates (glibc libm,
 * like the reference test helper). Used to build NodeInit fields for parity cases. */
void oracle_wavy(size_t n, const int32_t* x, const int32_t* y, const int32_t* z, double* rho,
                 double* ux, double* uy, double* uz) {
  for (size_t i = 0; i < n; ++i) {
    const double X = x[i], Y = y[i], Z = z[i];
    rho[i] = 1.0 + 0.02 * sin(0.37 * X + 0.11) * cos(0.23 * Y - 0.05) * cos(0.19 * Z + 0.4);
    ux[i] = 0.01 * sin(0.21 * X + 0.53 * Y);
    uy[i] = 0.01 * cos(0.17 * Y + 0.29 * Z);
    uz[i] = 0.01 * sin(0.13 * Z + 0.41 * X);
  }
}

/* ---- MRT (collision.cpp:11-113, collision.hpp:54-63) ---------------------------------------- */
/* Moment basis rows evaluated on the direction vectors (collision.cpp:11-60). */
static void mrt_basis(const lattice_t* L, double* m /* q*q, row-major */) {
  const int q = L->q;
  for (int i = 0; i < q; ++i) {
    const double ex = L->e[i][0], ey = L->e[i][1], ez = L->e[i][2];
    if (L->d == 2) {
      const double e2 = ex * ex + ey * ey;
      const double r[9] = {1.0,
                           -4.0 + 3.0 * e2,
                           4.0 - 10.5 * e2 + 4.5 * e2 * e2,
                           ex,
                           (-5.0 + 3.0 * e2) * ex,
                           ey,
                           (-5.0 + 3.0 * e2) * ey,
                           ex * ex - ey * ey,
                           ex * ey};
      for (int k = 0; k < 9; ++k) m[k * q + i] = r[k];
    } else {
      const double e2 = ex * ex + ey * ey + ez * ez;
      const double r[19] = {1.0,
                            19.0 * e2 - 30.0,
                            0.5 * (21.0 * e2 * e2 - 53.0 * e2 + 24.0),
                            ex,
                            (5.0 * e2 - 9.0) * ex,
                            ey,
                            (5.0 * e2 - 9.0) * ey,
                            ez,
                            (5.0 * e2 - 9.0) * ez,
                            3.0 * ex * ex - e2,
                            (3.0 * e2 - 5.0) * (3.0 * ex * ex - e2),
                            ey * ey - ez * ez,
                            (3.0 * e2 - 5.0) * (ey * ey - ez * ez),
                            ex * ey,
                            ey * ez,
                            ex * ez,
                            (ey * ey - ez * ez) * ex,
                            (ez * ez - ex * ex) * ey,
                            (ex * ex - ey * ey) * ez};
      for (int k = 0; k < 19; ++k) m[k * q + i] = r[k];
    }
  }
}

/* K = M^-1 S M with M^-1 = M^T diag(1/|row|^2) (collision.cpp:86-113); the dense products run in
 * the shim's order (acc += a(i,k) * b(k,j), k ascending). rates: q entries or NULL for the default
 * (0 for the conserved moments, 1/tau otherwise; collision.cpp:76-84). */
int oracle_mrt_kernel(int d, double tau, const double* rates_in, double* K) {
  lattice_t L;
  lattice_init(&L, d);
  const int q = L.q;
  double m[361], rn2[19], minv[361], s[361], p1[361], rates[19];
  mrt_basis(&L, m);
  for (int i = 0; i < q; ++i) rates[i] = rates_in ? rates_in[i] : 1.0 / tau;
  if (!rates_in) {
    const int cons2[3] = {0, 3, 5}, cons3[4] = {0, 3, 5, 7};
    const int* c = d == 2 ? cons2 : cons3;
    for (int k = 0; k < (d == 2 ? 3 : 4); ++k) rates[c[k]] = 0.0;
  }
  for (int i = 0; i < q; ++i) { /* (m * m^T).diagonal() */
    double acc = 0.0;
    for (int k = 0; k < q; ++k) acc += m[i * q + k] * m[i * q + k];
    rn2[i] = acc;
  }
  for (int i = 0; i < q; ++i)
    for (int j = 0; j < q; ++j) minv[i * q + j] = m[j * q + i] * (1.0 / rn2[j]);
  for (int i = 0; i < q; ++i)
    for (int j = 0; j < q; ++j) s[i * q + j] = i == j ? rates[i] : 0.0;
  for (int i = 0; i < q; ++i)
    for (int j = 0; j < q; ++j) {
      double acc = 0.0;
      for (int k = 0; k < q; ++k) acc += minv[i * q + k] * s[k * q + j];
      p1[i * q + j] = acc;
    }
  for (int i = 0; i < q; ++i)
    for (int j = 0; j < q; ++j) {
      double acc = 0.0;
      for (int k = 0; k < q; ++k) acc += p1[i * q + k] * m[k * q + j];
      K[i * q + j] = acc;
    }
  return q;
}
