// device_simulation.hpp — drop-in C++ adapter: the reference's own container
// and configuration types (sphfsi::ParticleStore<3>, sphfsi::ScenarioConfig<3>,
// /root/reference/proj/include/sphfsi) driven through the C ABI of sphg.h.
//
// A C++ caller of the reference keeps its ParticleStore and calls the SPEC
// operation names (density_summation, momentum_rhs, reduce_force_torque, step,
// ...); the store's vectors are handed to the device unchanged — Vec<3> is
// std::array<double,3> (24 B), so pos.data() is the interleaved xyz layout the
// ABI expects (store.hpp:26-46).  Header-only; link with libsphg.so.
#pragma once

#include <cmath>
#include <array>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "sphfsi/config.hpp"
#include "sphfsi/store.hpp"
#include "sphg.h"

namespace sphfsi_gpu {

static_assert(sizeof(sphfsi::Vec<3>) == 3 * sizeof(double), "Vec<3> must be 24 bytes (interleaved xyz)");
static_assert(sizeof(sphfsi::Kind) == 1 && sizeof(sphfsi::MaterialId) == 2, "ParticleStore tag widths");

class Error : public std::runtime_error {
 public:
  Error(int code, const std::string& m) : std::runtime_error(m), code(code) {}
  int code;
};

/// sphfsi::ScenarioConfig<3> (config.hpp:68-106) -> flat POD of the C ABI.
/// transitions < 0 takes cfg.transition_mode (config.hpp:61); diffusion switches on the
/// concentration equation.
inline sphg_params to_params(const sphfsi::ScenarioConfig<3>& cfg, double dt, int thermal, int transitions,
                             double contact_damping_override = -1.0, int diffusion = 0) {
  sphg_params p;
  std::memset(&p, 0, sizeof(p));
  p.dx = cfg.dx;
  p.h = cfg.smoothing_length;
  p.dt = dt;
  for (int a = 0; a < 3; ++a) {
    p.lo[a] = cfg.domain.lo[a];
    p.hi[a] = cfg.domain.hi[a];
    p.periodic[a] = cfg.periodic[a] ? 1 : 0;
  }
  p.cell_edge_override = cfg.cell_edge_override;
  p.n_mat = (int32_t)cfg.materials.size();
  if (p.n_mat > SPHG_MAX_MAT) throw Error(SPHG_ERR_CONFIG, "too many materials for the device table");
  for (sphfsi::MaterialId m = 0; m < cfg.materials.size(); ++m) {
    const sphfsi::Material& s = cfg.materials[m];
    sphg_material& d = p.mat[m];
    d.rho0 = s.reference_density;
    d.nu = s.kinematic_viscosity;
    d.cp = s.heat_capacity;
    d.kappa = s.conductivity;
    d.c = s.speed_of_sound;
    d.pb = s.background_pressure;
    d.T_t = s.transition_temperature;
    d.D = s.diffusivity;
    d.C_t = s.transition_concentration;
    d.melt_target = s.melt_target == sphfsi::kNoMaterial ? SPHG_NO_MATERIAL : s.melt_target;
    d.solidify_target = s.solidify_target == sphfsi::kNoMaterial ? SPHG_NO_MATERIAL : s.solidify_target;
    const sphfsi::Vec<3> b = cfg.body_force_of(m);
    for (int a = 0; a < 3; ++a) d.body_force[a] = b[a];
  }
  p.kc = cfg.contact_stiffness;
  p.dc = contact_damping_override >= 0.0 ? contact_damping_override : cfg.contact_damping;
  p.tvf = cfg.transport_velocity ? 1 : 0;
  p.thermal = thermal;
  p.transitions = transitions >= 0 ? transitions : (int32_t)cfg.transition_mode;
  p.diffusion = diffusion;
  p.n_dirichlet = (int32_t)cfg.dirichlet_temperature.size();
  for (int g = 0; g < p.n_dirichlet && g < SPHG_MAX_DIRICHLET; ++g) {
    const auto& pcs = cfg.dirichlet_temperature[g].pieces;
    p.dirichlet_T[g].n = (int32_t)pcs.size();
    for (size_t k = 0; k < pcs.size() && k < SPHG_MAX_PIECES; ++k) {
      p.dirichlet_T[g].t_end[k] = pcs[k].t_end;
      p.dirichlet_T[g].value[k] = pcs[k].value;
    }
  }
  p.n_dirichlet_c = (int32_t)cfg.dirichlet_concentration.size();
  for (int g = 0; g < p.n_dirichlet_c && g < SPHG_MAX_DIRICHLET; ++g) {
    const auto& pcs = cfg.dirichlet_concentration[g].pieces;
    p.dirichlet_C[g].n = (int32_t)pcs.size();
    for (size_t k = 0; k < pcs.size() && k < SPHG_MAX_PIECES; ++k) {
      p.dirichlet_C[g].t_end[k] = pcs[k].t_end;
      p.dirichlet_C[g].value[k] = pcs[k].value;
    }
  }
  p.rank = 0;
  p.nranks = cfg.workers;
  return p;
}

/// Views of a ParticleStore<3> for the ABI (no copies).
inline sphg_soa views(sphfsi::ParticleStore<3>& s, std::vector<sphfsi::Vec<3>>* force = nullptr) {
  sphg_soa v;
  std::memset(&v, 0, sizeof(v));
  v.n = s.size();
  auto d3 = [](std::vector<sphfsi::Vec<3>>& x) { return reinterpret_cast<double*>(x.data()); };
  v.pos = d3(s.pos);
  v.vel = d3(s.vel);
  v.vel_adv = d3(s.vel_adv);
  v.acc = d3(s.acc);
  v.acc_bg = d3(s.acc_bg);
  v.density = s.density.data();
  v.pressure = s.pressure.data();
  v.mass = s.mass.data();
  v.temperature = s.temperature.data();
  v.dT_dt = s.dT_dt.data();
  v.kind = reinterpret_cast<uint8_t*>(s.kind.data());
  v.group = s.group.data();
  v.material = s.material.data();
  v.body_frame_pos = d3(s.body_frame_pos);
  v.wall_pressure = s.wall_pressure.data();
  v.wall_velocity = d3(s.wall_velocity);
  v.dirichlet_T = s.dirichlet_T.data();
  v.concentration = s.concentration.data();
  v.dC_dt = s.dC_dt.data();
  v.dirichlet_C = s.dirichlet_C.data();
  if (force) {
    force->resize(s.size());
    v.force = d3(*force);
  }
  return v;
}

/// One device (rank) running the hot path over a reference ParticleStore.
class DeviceSimulation {
 public:
  DeviceSimulation(const sphg_params& p, int device = 0) {
    const int rc = sphg_create(&p, device, &ctx_);
    if (rc != SPHG_OK) {
      char buf[2048];
      sphg_validate(&p, buf, sizeof(buf));
      throw Error(rc, std::string("sphg_create: ") + buf);
    }
  }
  ~DeviceSimulation() { sphg_destroy(ctx_); }
  DeviceSimulation(const DeviceSimulation&) = delete;
  DeviceSimulation& operator=(const DeviceSimulation&) = delete;

  void upload(sphfsi::ParticleStore<3>& s, const std::vector<sphg_body>& bodies) {
    sphg_soa v = views(s);
    check(sphg_upload(ctx_, &v, bodies.data(), bodies.size()), "upload");
  }
  void download(sphfsi::ParticleStore<3>& s, std::vector<sphg_body>& bodies, std::vector<sphfsi::Vec<3>>* force = nullptr) {
    sphg_soa v = views(s, force);
    size_t nb = 0;
    check(sphg_num_bodies(ctx_, &nb), "num_bodies");
    bodies.resize(nb);
    check(sphg_download(ctx_, &v, bodies.data(), &nb), "download");
  }
  /// nsteps steps, then download(): the snapshot step of the run loop; positions,
  /// density, pressure and tags cross PCIe while the last step's forces run (transitions off).
  void step_download(int nsteps, sphfsi::ParticleStore<3>& s, std::vector<sphg_body>& bodies) {
    sphg_soa v = views(s);
    size_t nb = 0;
    check(sphg_num_bodies(ctx_, &nb), "num_bodies");
    bodies.resize(nb);
    check(sphg_step_download(ctx_, nsteps, &v, bodies.data(), &nb), "step_download");
    if (nb != bodies.size()) download(s, bodies);  // bodies spawned during the steps
  }
  // SPEC operations, bulk over the store
  void build_pairs() { stage(SPHG_STAGE_REBUILD); }
  void density_summation() { stage(SPHG_STAGE_DENSITY); }
  void conduction_rhs() { stage(SPHG_STAGE_HEAT); }
  void extrapolate_wall_quantities() { stage(SPHG_STAGE_EXTRAPOLATE); }
  void momentum_rhs() { stage(SPHG_STAGE_FORCES); }
  void reduce_force_torque() { stage(SPHG_STAGE_BODIES); }
  void reduce_mass_quantities() { stage(SPHG_STAGE_MASS); }
  void apply_transitions() { stage(SPHG_STAGE_TRANSITIONS); }
  void diffusion_rhs() { stage(SPHG_STAGE_HEAT); }
  /// ScenarioConfig::wall_groups (config.hpp:35-51, 93): WallGroup<3>::velocity_at and
  /// acceleration_at are evaluated on the host every step (the groups must outlive this object).
  void set_wall_groups(const std::vector<sphfsi::WallGroup<3>>* groups) {
    walls_ = groups;
    const int32_t ng = groups ? (int32_t)groups->size() : 0;
    check(sphg_set_wall_motion(ctx_, ng, ng ? &DeviceSimulation::wall_thunk : nullptr, this), "set_wall_motion");
  }
  void initialize() { check(sphg_initialize(ctx_), "initialize"); }
  /// the C-ABI context (for entry points without a wrapper here)
  sphg_ctx* raw() { return ctx_; }
  void step(int n = 1) { check(sphg_step(ctx_, n), "step"); }
  sphg_stats_t stats() {
    sphg_stats_t s;
    check(sphg_stats(ctx_, &s), "stats");
    return s;
  }
  /// compute_dt: cfl, viscous, body force, contact, conduction (+inf = absent)
  std::array<double, 5> compute_dt() {
    std::array<double, 5> lim{};
    check(sphg_compute_dt(ctx_, lim.data()), "compute_dt");
    return lim;
  }
  /// shepard_interpolate on an OutputPlan grid; NaN where no particle supports a point
  std::vector<double> shepard_grid(const double origin[3], const double spacing[3], const int32_t dims[3],
                                   int32_t field, uint32_t kind_mask = 1u << SPHG_FLUID) {
    const size_t np = (size_t)dims[0] * dims[1] * dims[2];
    std::vector<double> out(np * (field == SPHG_FIELD_VELOCITY ? 3 : 1));
    check(sphg_shepard_grid(ctx_, origin, spacing, dims, field, kind_mask, out.data(), nullptr), "shepard_grid");
    return out;
  }
  /// transition event log: enable, then drain the events recorded since the last call
  void set_event_log(bool on) { check(sphg_set_event_log(ctx_, on ? 1 : 0), "set_event_log"); }
  std::vector<sphg_event> transition_events() {
    size_t n = 0;
    check(sphg_transition_events(ctx_, nullptr, 0, &n), "transition_events");
    std::vector<sphg_event> ev(n);
    check(sphg_transition_events(ctx_, ev.data(), n, &n), "transition_events");
    ev.resize(n);
    return ev;
  }
  /// cell-occupancy histogram of the last rebuild: hist[k] = cells holding k particles
  std::vector<int64_t> cell_occupancy(size_t nbins, int64_t* max_count = nullptr) {
    std::vector<int64_t> hist(nbins);
    check(sphg_cell_occupancy(ctx_, hist.data(), nbins, max_count), "cell_occupancy");
    return hist;
  }

 private:
  void stage(int s) { check(sphg_run_stage(ctx_, s), "run_stage"); }
  void check(int rc, const char* what) {
    if (rc != SPHG_OK) throw Error(rc, std::string(what) + ": " + sphg_last_error(ctx_));
  }
  static void wall_thunk(int32_t g, double t, double vel[3], double acc[3], void* user) {
    const auto& w = (*static_cast<DeviceSimulation*>(user)->walls_)[(size_t)g];
    const sphfsi::Vec<3> v = w.velocity_at(t), a = w.acceleration_at(t);
    for (int k = 0; k < 3; ++k) {
      vel[k] = v[k];
      acc[k] = a[k];
    }
  }
  sphg_ctx* ctx_ = nullptr;
  const std::vector<sphfsi::WallGroup<3>>* walls_ = nullptr;
};

}  // namespace sphfsi_gpu
