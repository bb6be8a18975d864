// The C++ multi-GPU host (include/sphfsi_gpu/decomposed_simulation.hpp) against one rank: a periodic box of
// the reference's own ParticleStore<3> (seed_lattice, ball_region) with two rigid spheres, run as 2 and 4
// DecomposedSimulation ranks (threads of this process sharing the GPU through LocalTransport) and as one
// DeviceSimulation.  Two cases: fluid + bodies (fast particles: Verlet rebuilds and a migration), and
// melting / solidification (the SPEC:500 transition batch).  Kinds, materials and body ids must match
// exactly, positions to 1e-12 of the box, velocities to 1e-7 of the largest speed.
// Prints "ok <case> ranks=<n> ..." lines or fails with a non-zero exit code.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <thread>

#include "sphfsi/lattice.hpp"
#include "sphfsi_gpu/decomposed_simulation.hpp"

using namespace sphfsi;

namespace {

struct Case {
  ScenarioConfig<3> cfg;
  ParticleStore<3> store;
  std::vector<sphg_body> bodies;
  sphg_params params;
  int steps = 8;
};

uint64_t mix(uint64_t x) {  // SplitMix64 finaliser: deterministic per-particle numbers
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
double u01(uint64_t seed, uint64_t i) { return (double)(mix(seed * 1000003ull + i) >> 11) * (1.0 / 9007199254740992.0); }

Case make_case(bool melting) {
  Case c;
  const double dx = 1e-3, L = 20 * dx;
  c.cfg.dx = dx;
  for (int a = 0; a < 3; ++a) {
    c.cfg.domain.lo[a] = 0.0;
    c.cfg.domain.hi[a] = L;
    c.cfg.periodic[a] = true;
  }
  Material fluid;
  fluid.name = "fluid";
  fluid.reference_density = melting ? 7900.0 : 1000.0;
  fluid.kinematic_viscosity = 1e-6;
  fluid.speed_of_sound = melting ? 20.0 : 10.0;
  fluid.background_pressure = fluid.reference_pressure();
  fluid.heat_capacity = 700.0;
  fluid.conductivity = 20.0;
  Material solid = fluid;
  solid.name = "solid";
  solid.reference_density = melting ? 7900.0 : 2000.0;
  solid.kinematic_viscosity = 0.0;
  Material melt = fluid;
  melt.name = "melt";
  c.cfg.materials.add(fluid);  // 0
  const MaterialId ms = c.cfg.materials.add(solid);  // 1
  if (melting) {
    const MaterialId mm = c.cfg.materials.add(melt);  // 2
    c.cfg.materials[ms].transition_temperature = 1700.0;
    c.cfg.materials[ms].melt_target = mm;
    c.cfg.materials[mm].transition_temperature = 1700.0;
    c.cfg.materials[mm].solidify_target = ms;
  }
  for (size_t m = 0; m < c.cfg.materials.size(); ++m) c.cfg.body_force.push_back(Vec<3>::zero());
  c.cfg.contact_stiffness = 10.0;
  c.cfg.contact_damping = 0.0;
  seed_lattice<3>(c.store, box_region<3>(c.cfg.domain), dx, {Kind::Fluid, 0}, 0, c.cfg.materials[0]);
  const Vec<3> centers[2] = {{6.3e-3, 7.1e-3, 9.0e-3}, {14.2e-3, 13.0e-3, 10.5e-3}};
  const double R = 3.5 * dx;
  const size_t n = c.store.size();
  for (size_t i = 0; i < n; ++i) {
    for (int a = 0; a < 3; ++a) {  // jitter +-0.05 dx, wrapped
      double x = c.store.pos[i][a] + (2.0 * u01(1, 3 * i + a) - 1.0) * 0.05 * dx;
      if (x < 0.0) x += L;
      if (x >= L) x -= L;
      c.store.pos[i][a] = x;
    }
    const double vs = melting ? 0.01 : 0.6;  // fast flow: rebuilds and a migration within the run
    for (int a = 0; a < 3; ++a) c.store.vel[i][a] = (2.0 * u01(2, 3 * i + a) - 1.0) * vs;
    c.store.vel_adv[i] = c.store.vel[i];
    c.store.density[i] = c.cfg.materials[0].reference_density;
    c.store.mass[i] = c.cfg.materials[0].reference_density * dx * dx * dx;
    c.store.temperature[i] = melting ? 1650.0 : 300.0;
    for (int b = 0; b < 2; ++b) {
      double d2 = 0.0;
      for (int a = 0; a < 3; ++a) {
        const double d = c.store.pos[i][a] - centers[b][a];
        d2 += d * d;
      }
      const double r = std::sqrt(d2);
      if (r <= R) {
        c.store.kind[i] = Kind::Rigid;
        c.store.group[i] = (uint32_t)b;
        c.store.material[i] = ms;
        c.store.mass[i] = c.cfg.materials[ms].reference_density * dx * dx * dx;
        c.store.vel[i] = c.store.vel_adv[i] = Vec<3>::zero();
        if (melting) c.store.temperature[i] = 1700.0 + (2.0 * u01(3, i) - 1.0) * 5.0;  // flags flip at step 1
      } else if (melting && r <= R + 2.0 * dx) {
        c.store.material[i] = 2;  // a melt-liquid shell around the body, near T_t
        c.store.temperature[i] = 1700.0 + (2.0 * u01(4, i) - 1.0) * 5.0;
      }
    }
  }
  c.bodies.assign(2, sphg_body{});
  for (auto& b : c.bodies) {
    b.q[0] = 1.0;
    b.material = ms;
    b.mobile = 1;
    b.alive = 1;
  }
  c.params = sphfsi_gpu::to_params(c.cfg, melting ? 5e-6 : 1e-5, melting ? 1 : 0, melting ? 1 : 0);
  c.params.dt_check = SPHG_DT_WARN;
  {  // body mass, COM, inertia, chi from the members (reduce_mass_quantities), one table for every run
    sphfsi_gpu::DeviceSimulation s(c.params, 0);
    s.upload(c.store, c.bodies);
    s.reduce_mass_quantities();
    s.download(c.store, c.bodies);
  }
  c.steps = melting ? 6 : 24;
  return c;
}

int compare(const char* name, int ranks, const ParticleStore<3>& a, const ParticleStore<3>& b,
            const std::vector<sphg_body>& ba, const std::vector<sphg_body>& bb, double L, int64_t reparts,
            int64_t batches) {
  double umax = 0.0, dpos = 0.0, dvel = 0.0;
  for (size_t i = 0; i < a.size(); ++i) {
    if (a.kind[i] != b.kind[i] || a.material[i] != b.material[i] ||
        (a.kind[i] == Kind::Rigid && a.group[i] != b.group[i])) {
      std::printf("FAIL %s ranks=%d: tags differ at particle %zu\n", name, ranks, i);
      return 2;
    }
    for (int k = 0; k < 3; ++k) {
      umax = std::max(umax, std::fabs(a.vel[i][k]));
      double d = std::fabs(a.pos[i][k] - b.pos[i][k]);
      d = std::min(d, L - d);  // periodic
      dpos = std::max(dpos, d);
      dvel = std::max(dvel, std::fabs(a.vel[i][k] - b.vel[i][k]));
    }
  }
  if (ba.size() != bb.size()) {
    std::printf("FAIL %s ranks=%d: body count %zu vs %zu\n", name, ranks, ba.size(), bb.size());
    return 3;
  }
  for (size_t k = 0; k < ba.size(); ++k)
    if (ba[k].alive != bb[k].alive || ba[k].mass != bb[k].mass) {
      std::printf("FAIL %s ranks=%d: body %zu alive/mass differ\n", name, ranks, k);
      return 4;
    }
  if (dpos > 1e-12 * L || dvel > 1e-7 * umax) {
    std::printf("FAIL %s ranks=%d: dpos %.3g dvel %.3g (umax %.3g)\n", name, ranks, dpos, dvel, umax);
    return 5;
  }
  std::printf("ok %s ranks=%d n=%zu bodies=%zu dpos=%.2g dvel/umax=%.2g repartitions=%lld batches=%lld\n", name,
              ranks, a.size(), ba.size(), dpos, dvel / umax, (long long)reparts, (long long)batches);
  return 0;
}

int run(bool melting, int steps_override = 0, int ranks_only = 0) {
  Case c = make_case(melting);
  if (steps_override > 0) c.steps = steps_override;
  const char* name = melting ? "melting" : "fluid+bodies";
  const double L = c.cfg.domain.hi[0] - c.cfg.domain.lo[0];
  ParticleStore<3> one = c.store;
  std::vector<sphg_body> b1;
  {
    sphfsi_gpu::DeviceSimulation s(c.params, 0);
    s.upload(one, c.bodies);
    s.initialize();
    s.step(c.steps);
    s.download(one, b1);
  }
  for (int ranks : {2, 4}) {
    if (ranks_only && ranks != ranks_only) continue;
    sphfsi_gpu::LocalHub hub(ranks);
    std::vector<ParticleStore<3>> out(ranks);
    std::vector<std::vector<sphg_body>> bout(ranks);
    std::vector<int64_t> reparts(ranks), batches(ranks);
    std::vector<std::string> err(ranks);
    std::vector<std::thread> th;
    for (int r = 0; r < ranks; ++r)
      th.emplace_back([&, r]() {
        try {
          sphfsi_gpu::LocalTransport t(hub, r);
          sphfsi_gpu::DecomposedSimulation ds(c.params, t, 0, 0.3);
          ds.distribute(c.store, c.bodies);
          ds.initialize();
          ds.step(c.steps);
          ds.gather(out[r], bout[r]);
          reparts[r] = ds.repartitions();
          batches[r] = ds.batches();
        } catch (const std::exception& e) {
          err[r] = e.what();
        }
      });
    for (auto& t : th) t.join();
    for (int r = 0; r < ranks; ++r)
      if (!err[r].empty()) {
        std::printf("FAIL %s ranks=%d rank %d: %s\n", name, ranks, r, err[r].c_str());
        return 6;
      }
    const int rc = compare(name, ranks, one, out[0], b1, bout[0], L, reparts[0], batches[0]);
    if (rc) return rc;
    if (melting && batches[0] < 1) {
      std::printf("FAIL %s ranks=%d: no transition batch\n", name, ranks);
      return 7;
    }
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc > 2) {  // diagnostics: test_decomposed <melting 0|1> <steps> [ranks]
      return run(std::atoi(argv[1]) != 0, std::atoi(argv[2]), argc > 3 ? std::atoi(argv[3]) : 0);
    }
    int rc = run(false);
    if (rc) return rc;
    return run(true);
  } catch (const std::exception& e) {
    std::printf("FAIL %s\n", e.what());
    return 9;
  }
}
