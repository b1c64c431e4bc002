// ORACLE (test infrastructure): seeded inputs for C1-C5.
#pragma once
#include <cstdint>

#include "oracle.hpp"

namespace oracle {

struct SplitMix64 {
  uint64_t state;
  bool has_spare = false;
  double spare = 0.0;
  uint64_t next();
  double uniform();  // [0, 1), 53 bits
  double normal();   // Box-Muller pairs, cos branch first
};

Vec ic_burgers1d(int cfg, int ne, int order, uint64_t seed);
Vec ic_burgers2d(int nx, int ny, int order, uint64_t seed);
Vec ic_euler2d_vortex(int nx, int order, uint64_t seed, double noise);
Vec ic_euler3d_tgv(int n, int order, double gamma);

}  // namespace oracle
