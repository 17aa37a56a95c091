// Host-side setup helpers of libtmd_gpu.so: counter-based RNG, thermal
// velocities and the FCC lattice of the BASELINE.json configs. Plain C++,
// compiled without FMA contraction (x86-64 baseline), so every value is
// bit-identical to the reference's own host arithmetic for the same inputs.
#include <algorithm>
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

// ---------------------------------------------------------------------------
// The reference's own generators (generators.hpp), restated for the run-config
// front end. Velocities: thermal + zero net momentum
// (tmd_thermal_velocities) as each generator ends with.

// gen_lattice (generators.hpp:47-81): simple cubic, smallest cube of sites
// holding n, sites filled x-fastest, spacing = cbrt(n/rho)/side.
int tmd_gen_lattice(std::int64_t n, double rho, double temperature, std::uint64_t seed,
                    std::int64_t* id, double* pos, double* vel, double box[3]) {
  if (n < 1 || !(rho > 0.0) || temperature < 0.0) return TMD_ERR_CONFIG;
  const double edge = std::cbrt(static_cast<double>(n) / rho);
  std::int64_t side = 1;
  while (side * side * side < n) side += 1;
  const double spacing = edge / static_cast<double>(side);
  std::int64_t k = 0;
  for (std::int64_t z = 0; z < side && k < n; ++z)
    for (std::int64_t y = 0; y < side && k < n; ++y)
      for (std::int64_t x = 0; x < side && k < n; ++x, ++k) {
        id[k] = k;
        pos[3 * k] = (static_cast<double>(x) + 0.5) * spacing;
        pos[3 * k + 1] = (static_cast<double>(y) + 0.5) * spacing;
        pos[3 * k + 2] = (static_cast<double>(z) + 0.5) * spacing;
      }
  box[0] = box[1] = box[2] = edge;
  tmd_thermal_velocities(n, id, nullptr, temperature, seed, vel);
  return TMD_OK;
}

// gen_spherical (generators.hpp:83-135): lattice sites at rho_in kept inside
// the central sphere of diameter frac * L, and outside with probability
// alpha (counter_uniform lane 0 keyed by the site index). Two passes: call
// with id == NULL to get the count in *n_out.
int tmd_gen_spherical(double box_length, double frac, double rho_in, double alpha,
                      double temperature, std::uint64_t seed, std::int64_t* id, double* pos,
                      double* vel, std::int64_t* n_out, double box[3]) {
  if (!(box_length > 0.0) || !(frac > 0.0) || frac > 1.0 || !(rho_in > 0.0) || alpha < 0.0 ||
      alpha > 1.0 || temperature < 0.0) {
    return TMD_ERR_CONFIG;
  }
  const std::uint64_t kPlacement = 3;
  const double target = std::cbrt(1.0 / rho_in);
  const std::int64_t side =
      static_cast<std::int64_t>(std::max(1.0, std::round(box_length / target)));
  const double spacing = box_length / static_cast<double>(side);
  const double radius = 0.5 * frac * box_length;
  const double c = 0.5 * box_length;
  std::int64_t k = 0;
  std::uint64_t site = 0;
  for (std::int64_t z = 0; z < side; ++z)
    for (std::int64_t y = 0; y < side; ++y)
      for (std::int64_t x = 0; x < side; ++x, ++site) {
        const double px = (static_cast<double>(x) + 0.5) * spacing;
        const double py = (static_cast<double>(y) + 0.5) * spacing;
        const double pz = (static_cast<double>(z) + 0.5) * spacing;
        const double dx = px - c, dy = py - c, dz = pz - c;
        const bool inside = dx * dx + dy * dy + dz * dz <= radius * radius;
        if (!inside) {
          double u[3];
          tmd_counter_uniform3(seed, kPlacement, 0, site, u);
          if (u[0] >= alpha) continue;
        }
        if (id) {
          id[k] = k;
          pos[3 * k] = px;
          pos[3 * k + 1] = py;
          pos[3 * k + 2] = pz;
        }
        ++k;
      }
  *n_out = k;
  box[0] = box[1] = box[2] = box_length;
  if (id) tmd_thermal_velocities(k, id, nullptr, temperature, seed, vel);
  return TMD_OK;
}

// gen_random (generators.hpp:212-258): rejection sampling of uniform
// positions (counter_uniform3 keyed by attempt and particle) with a minimum
// minimum-image separation (box.hpp:34-43). TMD_ERR_VERIFY = the reference's
// "density too high" give-up after 100000 attempts per particle.
int tmd_gen_random(std::int64_t n, double rho, double min_distance, double temperature,
                   std::uint64_t seed, std::int64_t* id, double* pos, double* vel,
                   double box[3]) {
  if (n < 1 || !(rho > 0.0) || min_distance < 0.0 || temperature < 0.0) return TMD_ERR_CONFIG;
  const std::uint64_t kPlacement = 3;
  const double L = std::cbrt(static_cast<double>(n) / rho);
  const double d2 = min_distance * min_distance;
  auto mi = [L](double d) {
    double r = std::remainder(d, L);
    if (r == 0.5 * L) r = -0.5 * L;
    return r;
  };
  const std::uint64_t max_attempts = 100000ull * static_cast<std::uint64_t>(n);
  std::uint64_t attempt = 0;
  for (std::int64_t k = 0; k < n; ++k) {
    for (;;) {
      if (attempt >= max_attempts) return TMD_ERR_VERIFY;
      double u[3];
      tmd_counter_uniform3(seed, kPlacement, attempt++, static_cast<std::uint64_t>(k), u);
      const double px = u[0] * L, py = u[1] * L, pz = u[2] * L;
      bool ok = true;
      for (std::int64_t j = 0; j < k && ok; ++j) {
        const double dx = mi(px - pos[3 * j]), dy = mi(py - pos[3 * j + 1]),
                     dz = mi(pz - pos[3 * j + 2]);
        if (dx * dx + dy * dy + dz * dz < d2) ok = false;
      }
      if (!ok) continue;
      id[k] = k;
      pos[3 * k] = px;
      pos[3 * k + 1] = py;
      pos[3 * k + 2] = pz;
      break;
    }
  }
  box[0] = box[1] = box[2] = L;
  tmd_thermal_velocities(n, id, nullptr, temperature, seed, vel);
  return TMD_OK;
}

// Kremer-Grest melt (BASELINE.json configs[2]; the reference has only ring
// melts, gen_polymer_melt in generators.hpp:137-210): linear random-walk
// chains with fixed bond length, no immediate back-folding (bead k+2 at least
// one sigma from bead k), first beads uniform in the cubic box
// L = (N/rho)^(1/3); positions wrapped (box.hpp:47-51). Draws come from the
// reference's counter RNG under kPlacement keyed (chain, bead << 6 | try).
int tmd_gen_chains(std::int64_t n_chains, std::int64_t chain_len, double rho, double bond,
                   std::uint64_t seed, std::int64_t* id, double* pos, std::int64_t* bonds,
                   double box[3]) {
  if (n_chains < 1 || chain_len < 1 || !(rho > 0.0) || !(bond > 0.0)) return TMD_ERR_CONFIG;
  const std::uint64_t kPlacement = 3;
  const std::int64_t n = n_chains * chain_len;
  const double L = std::cbrt(static_cast<double>(n) / rho);
  auto wrap = [L](double p) {
    double r = p - L * std::floor(p / L);
    if (r >= L) r -= L;
    return r;
  };
  std::int64_t nb = 0;
  for (std::int64_t c = 0; c < n_chains; ++c) {
    double prev2[3] = {0, 0, 0}, prev[3] = {0, 0, 0};
    for (std::int64_t k = 0; k < chain_len; ++k) {
      double x[3];
      if (k == 0) {
        double u[3];
        tmd_counter_uniform3(seed, kPlacement, static_cast<std::uint64_t>(c), 0, u);
        for (int a = 0; a < 3; ++a) x[a] = u[a] * L;
      } else {
        for (int attempt = 0; attempt < 64; ++attempt) {
          double g[3];
          tmd_counter_normal3(seed, kPlacement, static_cast<std::uint64_t>(c),
                              (static_cast<std::uint64_t>(k) << 6) | attempt, g);
          const double gn = std::sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
          if (!(gn > 1e-12)) continue;
          for (int a = 0; a < 3; ++a) x[a] = prev[a] + bond * (g[a] / gn);
          if (k < 2) break;
          const double d0 = x[0] - prev2[0], d1 = x[1] - prev2[1], d2 = x[2] - prev2[2];
          if (d0 * d0 + d1 * d1 + d2 * d2 >= 1.0) break;
        }
      }
      const std::int64_t i = c * chain_len + k;
      id[i] = i;
      for (int a = 0; a < 3; ++a) pos[3 * i + a] = wrap(x[a]);
      if (k > 0) {
        bonds[2 * nb] = i - 1;
        bonds[2 * nb + 1] = i;
        ++nb;
      }
      for (int a = 0; a < 3; ++a) {
        prev2[a] = prev[a];
        prev[a] = x[a];
      }
    }
  }
  box[0] = box[1] = box[2] = L;
  return TMD_OK;
}

int tmd_gpu_abi_version(void) { return TMD_GPU_ABI_VERSION; }

}  // extern "C"
