// Drop-in check: a reference ScenarioConfig<3> + ParticleStore<3>, seeded with the
// reference's own seed_lattice, stepped on the GPU through sphfsi_gpu::DeviceSimulation.
// Prints one line "ok n=<particles> rho_min=<..> rho_max=<..> steps=<..>" or fails.
#include <cstdio>

#include "sphfsi/lattice.hpp"
#include "sphfsi_gpu/device_simulation.hpp"

int main() {
  using namespace sphfsi;
  ScenarioConfig<3> cfg;
  cfg.dx = 1e-3;
  const double L = 16e-3;
  for (int a = 0; a < 3; ++a) {
    cfg.domain.lo[a] = 0.0;
    cfg.domain.hi[a] = L;
    cfg.periodic[a] = true;
  }
  Material water;
  water.name = "water";
  water.reference_density = 1000.0;
  water.kinematic_viscosity = 1e-6;
  water.speed_of_sound = 10.0;
  water.background_pressure = water.reference_pressure();
  cfg.materials.add(water);
  cfg.body_force.push_back(Vec<3>::zero());
  const auto viol = validate_config(cfg);
  if (!viol.empty()) { std::printf("config invalid: %s\n", viol[0].c_str()); return 2; }
  ParticleStore<3> store;
  seed_lattice<3>(store, box_region<3>(cfg.domain), cfg.dx, {Kind::Fluid, 0}, 0, water);
  for (size_t i = 0; i < store.size(); ++i) {  // small deterministic perturbation
    store.pos[i][0] += 1e-5 * std::sin(1.0 * i);
    store.density[i] = water.reference_density;
  }
  const sphg_params p = sphfsi_gpu::to_params(cfg, 1e-5, 0, 0);
  sphfsi_gpu::DeviceSimulation sim(p, 0);
  sim.upload(store, {});
  sim.initialize();
  sim.step(4);
  std::vector<sphg_body> bodies;
  sim.step_download(1, store, bodies);  // the snapshot step: step + download in one call
  double lo = 1e300, hi = -1e300;
  for (double r : store.density) { lo = std::min(lo, r); hi = std::max(hi, r); }
  if (!(lo > 950.0 && hi < 1050.0)) { std::printf("density out of range %g %g\n", lo, hi); return 3; }
  // the aux entry points through the adapter: occupancy (every particle in some cell), dt limits, a grid
  int64_t mx = 0;
  const std::vector<int64_t> hist = sim.cell_occupancy(256, &mx);
  int64_t np = 0;
  for (size_t k = 0; k < hist.size(); ++k) np += (int64_t)k * hist[k];
  if (np != (int64_t)store.size() || mx <= 0) { std::printf("occupancy mismatch %lld\n", (long long)np); return 4; }
  const auto lim = sim.compute_dt();
  if (!(lim[0] > 0.0 && lim[0] < 1.0)) { std::printf("cfl limit %g\n", lim[0]); return 5; }
  const double o[3] = {4e-3, 4e-3, 4e-3}, sp[3] = {4e-3, 4e-3, 4e-3};
  const int32_t dims[3] = {2, 2, 2};
  const std::vector<double> rho = sim.shepard_grid(o, sp, dims, SPHG_FIELD_DENSITY);
  for (double r : rho)
    if (!(r > 950.0 && r < 1050.0)) { std::printf("grid density %g\n", r); return 6; }
  std::printf("ok n=%zu rho_min=%.6f rho_max=%.6f steps=%lld\n", store.size(), lo, hi, (long long)sim.stats().steps);
  return 0;
}
