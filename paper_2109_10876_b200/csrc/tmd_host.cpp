// Host-side setup helpers of libtmd_gpu.so: counter-based RNG, thermal
// velocities and the FCC lattice of the BASELINE.json configs. Plain C++,
// compiled without FMA contraction (x86-64 baseline), so every value is
// bit-identical to the reference's own host arithmetic for the same inputs.
#include <cmath>
#include <cstdint>

#include "../../include/tmd_gpu.h"

namespace {

// splitmix64 finalizer chained over the key words (random.hpp:23-39).
inline std::uint64_t mix64(std::uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

inline std::uint64_t key_hash(std::uint64_t seed, std::uint64_t ctx,
                              std::uint64_t step, std::uint64_t id,
                              std::uint64_t lane) {
  std::uint64_t h = mix64(seed ^ 0x243f6a8885a308d3ull);
  h = mix64(h ^ ctx);
  h = mix64(h ^ step);
  h = mix64(h ^ id);
  return mix64(h ^ lane);
}

// 53-bit mantissa draws: [0,1) and (0,1] (random.hpp:42-50).
inline double unit_closed_open(std::uint64_t b) {
  return static_cast<double>(b >> 11) * 0x1.0p-53;
}
inline double unit_open_closed(std::uint64_t b) {
  return static_cast<double>((b >> 11) + 1) * 0x1.0p-53;
}

}  // namespace

extern "C" {

void tmd_counter_uniform3(std::uint64_t seed, std::uint64_t ctx,
                          std::uint64_t step, std::uint64_t id, double out[3]) {
  for (int l = 0; l < 3; ++l) {
    out[l] = unit_closed_open(key_hash(seed, ctx, step, id, l));
  }
}

// Box-Muller over lanes 0..3, fourth deviate dropped (random.hpp:69-81).
void tmd_counter_normal3(std::uint64_t seed, std::uint64_t ctx,
                         std::uint64_t step, std::uint64_t id, double out[3]) {
  const double u0 = unit_open_closed(key_hash(seed, ctx, step, id, 0));
  const double u1 = unit_closed_open(key_hash(seed, ctx, step, id, 1));
  const double u2 = unit_open_closed(key_hash(seed, ctx, step, id, 2));
  const double u3 = unit_closed_open(key_hash(seed, ctx, step, id, 3));
  const double tau = 6.283185307179586476925286766559;
  const double ra = std::sqrt(-2.0 * std::log(u0));
  const double rb = std::sqrt(-2.0 * std::log(u2));
  out[0] = ra * std::cos(tau * u1);
  out[1] = ra * std::sin(tau * u1);
  out[2] = rb * std::cos(tau * u3);
}

void tmd_thermal_velocities(std::int64_t n, const std::int64_t* id,
                            const double* mass, double temperature,
                            std::uint64_t seed, double* vel) {
  const std::uint64_t kVelocityInit = 2;
  double px = 0.0, py = 0.0, pz = 0.0, mtot = 0.0;
  for (std::int64_t k = 0; k < n; ++k) {
    const double m = mass ? mass[k] : 1.0;
    const double s = std::sqrt(temperature / m);
    double g[3];
    tmd_counter_normal3(seed, kVelocityInit, 0,
                        static_cast<std::uint64_t>(id[k]), g);
    vel[3 * k] = s * g[0];
    vel[3 * k + 1] = s * g[1];
    vel[3 * k + 2] = s * g[2];
  }
  // zero_net_momentum: p = sum m v (componentwise), drift = (1/M) p.
  for (std::int64_t k = 0; k < n; ++k) {
    const double m = mass ? mass[k] : 1.0;
    px += m * vel[3 * k];
    py += m * vel[3 * k + 1];
    pz += m * vel[3 * k + 2];
    mtot += m;
  }
  if (mtot == 0.0) return;
  const double inv = 1.0 / mtot;
  const double dx = inv * px, dy = inv * py, dz = inv * pz;
  for (std::int64_t k = 0; k < n; ++k) {
    vel[3 * k] -= dx;
    vel[3 * k + 1] -= dy;
    vel[3 * k + 2] -= dz;
  }
}

int tmd_gen_fcc(int cells, double rho, double offset, std::int64_t* id,
                double* pos, double box[3]) {
  if (cells < 1 || !(rho > 0.0)) return TMD_ERR_CONFIG;
  const std::int64_t n = 4ll * cells * cells * cells;
  const double L = std::cbrt(static_cast<double>(n) / rho);
  const double a = L / cells;
  static const double basis[4][3] = {
      {0.0, 0.0, 0.0}, {0.5, 0.5, 0.0}, {0.5, 0.0, 0.5}, {0.0, 0.5, 0.5}};
  std::int64_t k = 0;
  for (int z = 0; z < cells; ++z)
    for (int y = 0; y < cells; ++y)
      for (int x = 0; x < cells; ++x)
        for (int b = 0; b < 4; ++b, ++k) {
          id[k] = k;
          pos[3 * k] = (x + basis[b][0] + offset) * a;
          pos[3 * k + 1] = (y + basis[b][1] + offset) * a;
          pos[3 * k + 2] = (z + basis[b][2] + offset) * a;
        }
  box[0] = box[1] = box[2] = L;
  return TMD_OK;
}

int tmd_gpu_abi_version(void) { return TMD_GPU_ABI_VERSION; }

}  // extern "C"
