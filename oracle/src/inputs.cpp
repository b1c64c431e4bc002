// ORACLE (test infrastructure): seeded synthetic inputs for BASELINE.json's
// configs C1-C5.  splitmix64 -> 53-bit uniforms ->
// Box-Muller normals; the product library carries an independent copy of the
// same generator and tests/test_inputs.py checks the two agree bit for bit.
#include <cmath>
#include <cstdint>

#include "oracle.hpp"
#include "oracle_inputs.hpp"

namespace oracle {

uint64_t SplitMix64::next() {
  uint64_t z = (state += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
double SplitMix64::uniform() { return double(next() >> 11) * 0x1.0p-53; }
double SplitMix64::normal() {
  if (has_spare) { has_spare = false; return spare; }
  const double u1 = 1.0 - uniform();  // (0, 1]
  const double u2 = uniform();
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double th = 2.0 * M_PI * u2;
  spare = r * std::sin(th);
  has_spare = true;
  return r * std::cos(th);
}

// C1/C2: 1D periodic [0, 2pi]
Vec ic_burgers1d(int cfg, int ne, int order, uint64_t seed) {
  const NodalBasis b = lgl_basis(order);
  const Mesh m = build_interval_mesh(0.0, 2.0 * M_PI, ne, BoundaryKind::periodic);
  const int np = b.num_nodes();
  Vec u(size_t(ne) * np);
  SplitMix64 rng{seed};
  double amp[16], ph[16];
  if (cfg == 2)
    for (int k = 0; k < 16; ++k) {
      amp[k] = -0.1 + 0.2 * rng.uniform();
      ph[k] = 2.0 * M_PI * rng.uniform();
    }
  for (int e = 0; e < ne; ++e)
    for (int i = 0; i < np; ++i) {
      const double x = m.elements[e].x0 + 0.5 * (b.nodes[i] + 1.0) * m.elements[e].hx;
      double v;
      if (cfg == 2) {
        v = 0.5;
        for (int k = 0; k < 16; ++k) v += amp[k] * std::sin((k + 1) * x + ph[k]);
      } else {
        v = 0.5 + std::sin(x) + 0.01 * rng.normal();
      }
      u[size_t(e) * np + i] = v;
    }
  return u;
}

// C3: 2D periodic [0,1]^2, u0 = sin(2 pi x) sin(2 pi y) + 0.01 N(0,1)
Vec ic_burgers2d(int nx, int ny, int order, uint64_t seed) {
  const NodalBasis b = lgl_basis(order);
  const Mesh m = build_quad_mesh(0.0, 1.0, 0.0, 1.0, nx, ny, BoundaryKind::periodic);
  const int np1 = b.num_nodes(), np = np1 * np1;
  Vec u(size_t(nx) * ny * np);
  SplitMix64 rng{seed};
  for (int e = 0; e < m.num_elements(); ++e)
    for (int j = 0; j < np1; ++j)
      for (int i = 0; i < np1; ++i) {
        const Element& el = m.elements[e];
        const double x = el.x0 + 0.5 * (b.nodes[i] + 1.0) * el.hx;
        const double y = el.y0 + 0.5 * (b.nodes[j] + 1.0) * el.hy;
        u[size_t(e) * np + j * np1 + i] =
            std::sin(2.0 * M_PI * x) * std::sin(2.0 * M_PI * y) + 0.01 * rng.normal();
      }
  return u;
}

// C4: strength-5 isentropic vortex on [0,10]^2, L2-projected with
// gauss_quadrature(k+2) as proj/src/harness.cpp:51,71-75, + 1e-6 N(0,1) on rho.
Vec ic_euler2d_vortex(int nx, int order, uint64_t seed, double noise) {
  const NodalBasis b = lgl_basis(order);
  const Mesh m = build_quad_mesh(0.0, 10.0, 0.0, 10.0, nx, nx, BoundaryKind::periodic);
  EulerConfig cfg;
  cfg.vortex.alpha = 1.0;
  cfg.vortex.lambda = 5.0;
  cfg.vortex.u_inf = 1.0;
  cfg.vortex.v_inf = 1.0;
  cfg.vortex.xc = 5.0;
  cfg.vortex.yc = 5.0;
  cfg.vortex.wrap_lx = 10.0;
  cfg.vortex.wrap_ly = 10.0;
  Vec q = l2_project_system_2d(
      [&cfg](double x, double y, double* out) {
        const State4 s = isentropic_vortex(x, y, 0.0, cfg);
        for (int c = 0; c < 4; ++c) out[c] = s[c];
      },
      4, m, b, gauss_quadrature(order + 2));
  const int np = (order + 1) * (order + 1);
  SplitMix64 rng{seed};
  for (int e = 0; e < m.num_elements(); ++e)
    for (int n = 0; n < np; ++n) q[(size_t(e) * 4 + 0) * np + n] += noise * rng.normal();
  return q;
}

// C5: Taylor-Green vortex, Mach 0.1, periodic [0, 2pi]^3, nodal.
Vec ic_euler3d_tgv(int n, int order, double gamma) {
  const NodalBasis b = lgl_basis(order);
  const int np1 = b.num_nodes(), np = np1 * np1 * np1;
  const double h = 2.0 * M_PI / n;
  const double rho0 = 1.0, p0 = 1.0 / (gamma * 0.01);
  Vec q(size_t(n) * n * n * np * 5);
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        const size_t e = (size_t(k) * n + j) * n + i;
        for (int c2 = 0; c2 < np1; ++c2)
          for (int c1 = 0; c1 < np1; ++c1)
            for (int c0 = 0; c0 < np1; ++c0) {
              const double x = i * h + 0.5 * (b.nodes[c0] + 1.0) * h;
              const double y = j * h + 0.5 * (b.nodes[c1] + 1.0) * h;
              const double z = k * h + 0.5 * (b.nodes[c2] + 1.0) * h;
              const double u = std::sin(x) * std::cos(y) * std::cos(z);
              const double v = -std::cos(x) * std::sin(y) * std::cos(z);
              const double w = 0.0;
              const double p = p0 + (rho0 / 16.0) * (std::cos(2.0 * x) + std::cos(2.0 * y)) *
                                         (std::cos(2.0 * z) + 2.0);
              const int node = (c2 * np1 + c1) * np1 + c0;
              const double E = p / (gamma - 1.0) + 0.5 * rho0 * (u * u + v * v + w * w);
              q[(e * 5 + 0) * np + node] = rho0;
              q[(e * 5 + 1) * np + node] = rho0 * u;
              q[(e * 5 + 2) * np + node] = rho0 * v;
              q[(e * 5 + 3) * np + node] = rho0 * w;
              q[(e * 5 + 4) * np + node] = E;
            }
      }
  return q;
}

}  // namespace oracle
