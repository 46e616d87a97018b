#include "mrt.h"

#include "common.h"
#include "mrt_jit.h"

namespace splbm_host {

namespace {

// Row values of the moment basis at one direction (collision.cpp:11-60).
void basis_column(int d, int ex, int ey, int ez, double* col) {
  const double x = ex, y = ey, z = ez;
  if (d == 2) {
    const double e2 = x * x + y * y;
    const double v[9] = {1.0, -4.0 + 3.0 * e2, 4.0 - 10.5 * e2 + 4.5 * e2 * e2, x,
                         (-5.0 + 3.0 * e2) * x, y, (-5.0 + 3.0 * e2) * y, x * x - y * y, x * y};
    for (int k = 0; k < 9; ++k) col[k] = v[k];
    return;
  }
  const double e2 = x * x + y * y + z * z;
  const double v[19] = {1.0,
                        19.0 * e2 - 30.0,
                        0.5 * (21.0 * e2 * e2 - 53.0 * e2 + 24.0),
                        x,
                        (5.0 * e2 - 9.0) * x,
                        y,
                        (5.0 * e2 - 9.0) * y,
                        z,
                        (5.0 * e2 - 9.0) * z,
                        3.0 * x * x - e2,
                        (3.0 * e2 - 5.0) * (3.0 * x * x - e2),
                        y * y - z * z,
                        (3.0 * e2 - 5.0) * (y * y - z * z),
                        x * y,
                        y * z,
                        x * z,
                        (y * y - z * z) * x,
                        (z * z - x * x) * y,
                        (x * x - y * y) * z};
  for (int k = 0; k < 19; ++k) col[k] = v[k];
}

}  // namespace

std::vector<double> mrt_kernel(int d, double tau, const double* rates) {
  static const int e2d[9][3] = {{0, 0, 0},  {1, 0, 0},   {-1, 0, 0}, {0, 1, 0},  {0, -1, 0},
                                {1, 1, 0},  {-1, -1, 0}, {1, -1, 0}, {-1, 1, 0}};
  static const int e3d[19][3] = {{0, 0, 0},  {1, 0, 0},   {-1, 0, 0},  {0, 1, 0},  {0, -1, 0},
                                 {0, 0, 1},  {0, 0, -1},  {1, 1, 0},   {-1, -1, 0}, {1, -1, 0},
                                 {-1, 1, 0}, {1, 0, 1},   {-1, 0, -1}, {1, 0, -1}, {-1, 0, 1},
                                 {0, 1, 1},  {0, -1, -1}, {0, 1, -1},  {0, -1, 1}};
  const int q = d == 2 ? 9 : 19;
  std::vector<double> M(q * q), minv(q * q), S(q * q, 0.0), P(q * q), K(q * q), rn2(q), r(q);
  for (int i = 0; i < q; ++i) {
    double col[19];
    const int* e = d == 2 ? e2d[i] : e3d[i];
    basis_column(d, e[0], e[1], e[2], col);
    for (int k = 0; k < q; ++k) M[k * q + i] = col[k];
  }
  for (int i = 0; i < q; ++i) r[i] = rates ? rates[i] : 1.0 / tau;  // default_mrt_rates
  if (!rates) {
    for (int c : (d == 2 ? std::vector<int>{0, 3, 5} : std::vector<int>{0, 3, 5, 7})) r[c] = 0.0;
  }
  for (int i = 0; i < q; ++i) {  // (M M^T).diagonal()
    double acc = 0.0;
    for (int k = 0; k < q; ++k) acc += M[i * q + k] * M[i * q + k];
    rn2[i] = acc;
  }
  for (int i = 0; i < q; ++i)
    for (int j = 0; j < q; ++j) minv[i * q + j] = M[j * q + i] * (1.0 / rn2[j]);
  for (int i = 0; i < q; ++i) S[i * q + i] = r[i];
  auto gemm = [q](const std::vector<double>& A, const std::vector<double>& B, std::vector<double>& C) {
    for (int i = 0; i < q; ++i)
      for (int j = 0; j < q; ++j) {
        double acc = 0.0;
        for (int k = 0; k < q; ++k) acc += A[i * q + k] * B[k * q + j];
        C[i * q + j] = acc;
      }
  };
  gemm(minv, S, P);
  gemm(P, M, K);
  return K;
}

}  // namespace splbm_host

extern "C" int splbm_mrt_kernel(int d, double tau, const double* rates, double* K_out) {
  using namespace splbm_host;
  return guarded([&] {
    if (d != 2 && d != 3) throw config_error("MRT is supported for D2Q9 and D3Q19 only");
    if (!(tau > 0.5)) throw config_error("relaxation time tau must be > 0.5");
    const auto K = mrt_kernel(d, tau, rates);
    std::copy(K.begin(), K.end(), K_out);
  });
}

extern "C" int splbm_mrt_specialise(int d, int incompressible, int single_precision, double tau,
                                    const double* rates, int tile, int* products_out) {
  using namespace splbm_host;
  return guarded([&] {
    if (d != 2 && d != 3) throw config_error("MRT is supported for D2Q9 and D3Q19 only");
    if (!(tau > 0.5)) throw config_error("relaxation time tau must be > 0.5");
    const auto K = mrt_kernel(d, tau, rates);
    int products = 0;
    mrt_collision_source(d, incompressible != 0, single_precision != 0, K, &products);
    if (products_out) *products_out = products;
    if (tile > 0) {
      int loga = 0;
      while ((1 << loga) < tile) ++loga;
      if ((1 << loga) != tile || loga < 1 || loga > (d == 3 ? 2 : 4))
        throw config_error("specialised MRT step needs a power-of-two tile edge (3D: 2, 4; 2D: 2..16)");
      std::vector<char> cubin;
      std::vector<std::string> lowered;
      std::string why;
      if (!mrt_jit_cubin(d, loga, incompressible != 0, single_precision != 0, K, &cubin, &lowered, &why))
        throw Error(SPLBM_ERR_CUDA, why);
    }
  });
}
