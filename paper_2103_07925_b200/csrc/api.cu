// api.cu — the C ABI of include/sphg.h: context lifetime, upload/download in
// the ParticleStore<3> layout, and the stream-ordered step driver.
//
// Replaces (reference interfaces):
//   sphg_create     validate_config (config.hpp:110-167) + decomposition setup
//   sphg_upload     ParticleStore<3> (store.hpp:24-100) -> device SoA
//   sphg_step       step(state, dt)
//   sphg_run_stage  build_pairs / density_summation / conduction_rhs / extrapolate_wall_quantities /
//                   momentum_rhs+coupling+contact / reduce_force_torque / transitions / reduce_mass_quantities
//   sphg_download   device SoA -> ParticleStore<3> (device-side pack into gid order, then DMA)
//   sphg_set_wall_motion / sphg_shepard_grid / sphg_halo_* / sphg_body_*: see include/sphg.h
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <numeric>
#include <string>
#include <type_traits>
#include <vector>

#include "context.cuh"

using namespace sphg;

struct sphg_ctx {
  Ctx c;
  bool mid_step = false;
};

namespace {

constexpr double kSkin = 0.1;     // config.hpp:16 kVerletSkinFactor
constexpr double kSupport = 3.0;  // config.hpp:15 kKernelSupportScale

std::vector<std::string> validate(const sphg_params& P) {  // restates config.hpp:110-167 + extras
  std::vector<std::string> v;
  auto fail = [&](std::string m) { v.push_back(std::move(m)); };
  if (P.n_mat < 0 || P.n_mat > SPHG_MAX_MAT) {
    fail("material count out of range");
    return v;
  }
  if (!(P.dx > 0.0)) fail("initial particle spacing dx must be positive");
  if (P.h < 0.0) fail("smoothing length must be non-negative");
  const double h = P.h > 0.0 ? P.h : P.dx;
  const double rc = kSupport * h;
  if (P.cell_edge_override > 0.0 && P.cell_edge_override < rc) fail("cell edge < support radius");
  for (int a = 0; a < 3; ++a) {
    const double extent = P.hi[a] - P.lo[a];
    if (!(extent > 0.0)) fail("domain extent must be positive on axis " + std::to_string(a));
    if (P.periodic[a]) {
      if (extent < 2.0 * rc) fail("periodic axis " + std::to_string(a) + " shorter than twice the support radius");
      if (P.dx > 0.0) {
        const double cells = extent / P.dx;
        if (std::abs(cells - std::round(cells)) > 1e-9 * cells)
          fail("periodic axis " + std::to_string(a) + " extent is not a multiple of dx");
      }
    }
  }
  if (P.n_mat == 0) fail("no materials defined");
  for (int m = 0; m < P.n_mat; ++m) {
    const sphg_material& mt = P.mat[m];
    const std::string name = "m" + std::to_string(m);
    if (!(mt.rho0 > 0.0)) fail("material '" + name + "' has non-positive reference density");
    if (mt.melt_target >= 0 && mt.melt_target >= P.n_mat) fail("material '" + name + "' melts into a missing material");
    if (mt.solidify_target >= 0 && mt.solidify_target >= P.n_mat)
      fail("material '" + name + "' solidifies into a missing material");
  }
  if ((P.nranks > 0 ? P.nranks : 1) < 1) fail("worker count must be at least 1");
  if (P.kc < 0.0) fail("contact stiffness must be non-negative");
  if (P.dc < 0.0) fail("contact damping must be non-negative");
  for (int g = 0; g < P.n_dirichlet && g < SPHG_MAX_DIRICHLET; ++g)
    for (int i = 1; i < P.dirichlet_T[g].n && i < SPHG_MAX_PIECES; ++i)
      if (P.dirichlet_T[g].t_end[i] < P.dirichlet_T[g].t_end[i - 1]) fail("temperature schedule pieces out of order");
  for (int g = 0; g < P.n_dirichlet_c && g < SPHG_MAX_DIRICHLET; ++g)
    for (int i = 1; i < P.dirichlet_C[g].n && i < SPHG_MAX_PIECES; ++i)
      if (P.dirichlet_C[g].t_end[i] < P.dirichlet_C[g].t_end[i - 1])
        fail("concentration schedule pieces out of order");
  // extras (oracle/sph_oracle.cpp validate)
  if (!(P.dt > 0.0)) fail("time step dt must be positive");
  const double rv = kSupport * h + kSkin * h;
  for (int a = 0; a < 3; ++a) {
    const double ext = P.hi[a] - P.lo[a];
    const double e0 = P.cell_edge_override > 0.0 ? P.cell_edge_override : rv;
    if (P.periodic[a] && ext > 0.0 && std::floor(ext / e0) < 3.0)
      fail("periodic axis " + std::to_string(a) + " has fewer than 3 cells");
  }
  if (P.n_dirichlet < 0 || P.n_dirichlet > SPHG_MAX_DIRICHLET) fail("dirichlet group count out of range");
  if (P.n_dirichlet_c < 0 || P.n_dirichlet_c > SPHG_MAX_DIRICHLET)
    fail("concentration dirichlet group count out of range");
  if (P.transitions < 0 || P.transitions > 2) fail("unknown transition mode");
  if (P.transitions == 2 && !P.diffusion) fail("concentration transitions need the diffusion equation");
  if (P.default_fluid_mat < 0 || P.default_fluid_mat >= P.n_mat) fail("default fluid material missing");
  if (P.n_buffers < 0 || P.n_buffers > SPHG_MAX_BUFFERS) fail("buffer zone count out of range");
  for (int b = 0; b < P.n_buffers && b < SPHG_MAX_BUFFERS; ++b) {
    const sphg_buffer& B = P.buffers[b];
    if (B.axis < 0 || B.axis > 2 || B.profile_axis < -1 || B.profile_axis > 2 || B.profile_axis == B.axis)
      fail("buffer zone axes invalid");
    for (int a = 0; a < 3; ++a)
      if (!(B.hi[a] > B.lo[a])) fail("buffer zone box is empty");
  }
  if (P.heat_source) {  // [P21]
    if (!P.thermal) fail("heat source needs the heat equation");
    if (!(P.hs_radius > 0.0)) fail("heat source radius must be positive");
  }
  return v;
}

DevParams make_dev_params(const sphg_params& p) {
  DevParams P;
  std::memset(&P, 0, sizeof(P));
  P.n_mat = p.n_mat;
  bool first_fluid = true;
  double eta0 = 0, rho00 = 0, c0 = 0;
  P.single_eta = 1;
  P.single_eos = 1;
  P.single_kappa = 1;
  for (int m = 0; m < p.n_mat; ++m) {
    const sphg_material& s = p.mat[m];
    DevMat& d = P.mat[m];
    d.rho0 = s.rho0;
    d.eta = s.rho0 * s.nu;  // material.hpp:32
    d.cp = s.cp;
    d.kappa = s.kappa;
    d.c2 = s.c * s.c;
    d.pb = s.pb;
    d.T_t = s.T_t;
    d.has_Tt = std::isnan(s.T_t) ? 0 : 1;
    d.D = s.D;
    d.C_t = s.C_t;
    d.has_Ct = std::isnan(s.C_t) ? 0 : 1;
    for (int a = 0; a < 3; ++a) d.g[a] = s.body_force[a];
    d.p0 = s.rho0 * s.c * s.c;
    d.inv_c2 = s.c != 0.0 ? 1.0 / (s.c * s.c) : 0.0;
    d.melt = s.melt_target;
    d.solid = s.solidify_target;
    if (m > 0 && s.kappa != p.mat[0].kappa) P.single_kappa = 0;
    if (s.c > 0.0 && s.nu >= 0.0) {  // a fluid-capable material
      if (first_fluid) {
        eta0 = d.eta;
        P.eta_single = d.eta;
        rho00 = s.rho0;
        c0 = s.c;
        first_fluid = false;
      } else {
        if (d.eta != eta0) P.single_eta = 0;
        if (s.rho0 != rho00 || s.c != c0) P.single_eos = 0;
      }
    }
  }
  // a wall without support falls back to default_fluid_mat; with single_eos the EOS is the same anyway
  if (P.single_eos && p.n_mat > 0) {
    const sphg_material& dm = p.mat[p.default_fluid_mat];
    if (!first_fluid && (dm.rho0 != rho00 || dm.c != c0)) P.single_eos = 0;
  }
  P.n_sched = p.n_dirichlet;
  for (int g = 0; g < p.n_dirichlet && g < SPHG_MAX_DIRICHLET; ++g) {
    P.sched[g].n = p.dirichlet_T[g].n;
    for (int k = 0; k < SPHG_MAX_PIECES; ++k) {
      P.sched[g].t_end[k] = p.dirichlet_T[g].t_end[k];
      P.sched[g].value[k] = p.dirichlet_T[g].value[k];
    }
  }
  P.single_g = 1;
  if (p.n_mat > 0) {
    const sphg_material& dm = p.mat[p.default_fluid_mat >= 0 && p.default_fluid_mat < p.n_mat ? p.default_fluid_mat : 0];
    for (int m = 0; m < p.n_mat; ++m)
      if (p.mat[m].c > 0.0 && p.mat[m].nu >= 0.0)  // a fluid-capable material
        for (int a = 0; a < 3; ++a)
          if (p.mat[m].body_force[a] != dm.body_force[a]) P.single_g = 0;
  }
  P.n_schedC = p.n_dirichlet_c;
  for (int g = 0; g < p.n_dirichlet_c && g < SPHG_MAX_DIRICHLET; ++g) {
    P.schedC[g].n = p.dirichlet_C[g].n;
    for (int k = 0; k < SPHG_MAX_PIECES; ++k) {
      P.schedC[g].t_end[k] = p.dirichlet_C[g].t_end[k];
      P.schedC[g].value[k] = p.dirichlet_C[g].value[k];
    }
  }
  P.diffusion = p.diffusion;
  P.h = p.h > 0.0 ? p.h : p.dx;
  P.inv_h = 1.0 / P.h;  // kernel.hpp:20 inv_h_
  P.rc = kSupport * P.h;
  P.rc2 = P.rc * P.rc;
  P.rc2_lo = P.rc2 * (1.0 - 2e-4);
  P.rc2_ulp = P.rc2 * (1.0 - 1e-12);
  P.dx2_hi = p.dx * p.dx * (1.0 + 1e-12);
  P.rc2_hi = P.rc2 * (1.0 + 1e-12);
  P.rv = P.rc + kSkin * P.h;
  P.rv2 = P.rv * P.rv;
  P.sigma = 1.0 / (120.0 * M_PI * P.h * P.h * P.h);  // kernel.hpp:44
  P.sig_h = P.sigma * P.inv_h;
  P.w0 = P.sigma * 66.0;
  P.dx = p.dx;
  P.dx3 = p.dx * p.dx * p.dx;
  P.dt = p.dt;
  P.hdt = 0.5 * p.dt;
  P.kc = p.kc;
  P.dc = p.dc;
  P.half_skin = 0.5 * (P.rv - P.rc);
  const double reff = std::cbrt(0.75 / M_PI) * p.dx;
  P.Ir_over_m = 0.4 * reff * reff;
  P.tvf = p.tvf;
  P.thermal = p.thermal;
  P.heat_source = p.thermal && p.heat_source;  // [P21]; constants as the oracle forms them
  P.hs_mask = p.hs_material_mask;
  P.hs_q0 = 2.0 * p.hs_power / (M_PI * p.hs_radius * p.hs_radius);
  P.hs_r0sq = p.hs_radius * p.hs_radius;
  P.hs_cut2 = 16.0 * p.hs_radius * p.hs_radius;
  for (int a = 0; a < 2; ++a) {
    P.hs_origin[a] = p.hs_origin[a];
    P.hs_vel[a] = p.hs_velocity[a];
  }
  P.hs_dz = 0.5 * p.dx;
  P.hs_lat2 = 0.5625 * p.dx * p.dx;
  P.transitions = p.transitions;
  P.default_fluid_mat = p.default_fluid_mat;
  P.n_buf = p.n_buffers;
  for (int b = 0; b < p.n_buffers && b < SPHG_MAX_BUFFERS; ++b) {
    P.buf[b].axis = p.buffers[b].axis;
    P.buf[b].paxis = p.buffers[b].profile_axis;
    for (int a = 0; a < 3; ++a) {
      P.buf[b].lo[a] = p.buffers[b].lo[a];
      P.buf[b].hi[a] = p.buffers[b].hi[a];
    }
    P.buf[b].u_mean = p.buffers[b].u_mean;
  }
  for (int a = 0; a < 3; ++a) {
    P.lo[a] = p.lo[a];
    P.hi[a] = p.hi[a];
    P.L[a] = p.hi[a] - p.lo[a];
    P.halfL[a] = 0.5 * P.L[a];
    P.periodic[a] = p.periodic[a];
    const double e0 = p.cell_edge_override > 0.0 ? p.cell_edge_override : P.rv;  // [P1]
    int nc = (int)std::floor(P.L[a] / e0);
    if (nc < 1) nc = 1;
    P.ncell[a] = nc;
    P.inv_edge[a] = (double)nc / P.L[a];
  }
  return P;
}

double bits_to_double(unsigned long long b) {
  double d;
  std::memcpy(&d, &b, sizeof(d));
  return d;
}

int fail(sphg_ctx* h, int code, const std::string& m) {
  if (h) h->c.err = m;
  return code;
}

template <class F>
int guarded(sphg_ctx* h, F&& f) {
  try {
    return f();
  } catch (const CudaError& e) {
    return fail(h, SPHG_ERR_CUDA, "CUDA error: " + e.what);
  } catch (const std::exception& e) {
    return fail(h, SPHG_ERR_RUNTIME, e.what());
  }
}

void ensure_bodies(Ctx& c, size_t need) {
  if (need <= c.bodies_cap && c.bodies.p) return;
  size_t cap = std::max<size_t>(need * 2, 64);
  sphg_body* nb = nullptr;
  SPHG_CUDA_CHECK(cudaMalloc(&nb, cap * sizeof(sphg_body)));
  SPHG_CUDA_CHECK(cudaMemsetAsync(nb, 0, cap * sizeof(sphg_body), c.stream));
  if (c.bodies.p && c.nb) SPHG_CUDA_CHECK(cudaMemcpyAsync(nb, c.bodies.p, c.nb * sizeof(sphg_body), cudaMemcpyDeviceToDevice, c.stream));
  host_sync(c, c.stream);
  c.bodies.free();
  c.bodies.p = nb;
  c.bodies.n = cap;
  c.bodies_cap = cap;
}

// reads the flag block; returns SPHG_OK or a runtime error with a one-line message
int check_flags(sphg_ctx* h, bool sync, bool copy = true) {  // copy=false: the readback is already enqueued
  Ctx& c = h->c;
  if (copy) SPHG_CUDA_CHECK(cudaMemcpyAsync(c.hflags, c.dflags, sizeof(DevFlags), cudaMemcpyDeviceToHost, c.stream));
  if (sync) host_sync(c, c.stream);
  SPHG_CUDA_CHECK(cudaGetLastError());
  const DevFlags& f = *c.hflags;
  c.max_disp = std::sqrt(bits_to_double(f.max_disp2_bits));
  c.u_max = std::sqrt(bits_to_double(f.umax2_bits));
  if (f.err) {
    const std::string step = " at step " + std::to_string(c.steps + (h->mid_step ? 1 : 0));
    if (!(f.err & (kErrEscape | kErrCoincident)) && (f.err & kErrNaN))
      return fail(h, SPHG_ERR_RUNTIME, "non-finite state of particle " + std::to_string(f.err_gid2) + step);
    if (f.err & kErrInvariant)  // -DSPHG_CHECKED builds only
      return fail(h, SPHG_ERR_RUNTIME, "device invariant violated (row / index list out of bounds) at particle " +
                                           std::to_string(f.err_gid) + step);
    std::string what = (f.err & kErrEscape) ? "escaped particle " : (f.err & kErrCoincident) ? "coincident particles at particle " : "runtime assertion at particle ";
    return fail(h, SPHG_ERR_RUNTIME, what + std::to_string(f.err_gid) + step);
  }
  return SPHG_OK;
}

void reset_step_flags(Ctx& c) {
  SPHG_CUDA_CHECK(cudaMemsetAsync(c.dflags, 0, 2 * sizeof(unsigned long long), c.stream));
}

const char* stage_name(int stage) {
  static const char* names[16] = {"rebuild", "density", "heat", "extrapolate", "forces", "bodies", "kick_drift",
                                  "final_kick", "transitions", "mass", "forces_fluid", "forces_rigid",
                                  "", "", "", ""};
  return stage >= 0 && stage < 16 ? names[stage] : "stage";
}

void timed(Ctx& c, int stage, void (*fn)(Ctx&)) {
  NvtxRange nv(stage_name(stage));
  if (!c.timing) {
    fn(c);
    return;
  }
  SPHG_CUDA_CHECK(cudaEventRecord(c.ev[0], c.stream));
  fn(c);
  SPHG_CUDA_CHECK(cudaEventRecord(c.ev[1], c.stream));
  SPHG_CUDA_CHECK(cudaEventSynchronize(c.ev[1]));
  float ms = 0.f;
  SPHG_CUDA_CHECK(cudaEventElapsedTime(&ms, c.ev[0], c.ev[1]));
  c.stage_ms[stage] += ms;
}

void timed_forces(Ctx& c) {  // stage 4 = 10 (fluid kernel) + 11 (rigid kernel)
  if (!c.timing && c.concurrent_rigid && c.nrigid) {
    // the rigid coupling / contact pass reads only the state the extrapolation left: it runs on a second
    // stream beside the fluid force pass (joined before the body reduction)
    if (!c.side_stream) {
      SPHG_CUDA_CHECK(cudaStreamCreateWithFlags(&c.side_stream, cudaStreamNonBlocking));
      SPHG_CUDA_CHECK(cudaEventCreateWithFlags(&c.fork_ev, cudaEventDisableTiming));
      SPHG_CUDA_CHECK(cudaEventCreateWithFlags(&c.join_ev, cudaEventDisableTiming));
    }
    SPHG_CUDA_CHECK(cudaEventRecord(c.fork_ev, c.stream));
    SPHG_CUDA_CHECK(cudaStreamWaitEvent(c.side_stream, c.fork_ev, 0));
    std::swap(c.stream, c.side_stream);
    launch_forces_rigid(c);
    std::swap(c.stream, c.side_stream);
    SPHG_CUDA_CHECK(cudaEventRecord(c.join_ev, c.side_stream));
    launch_forces_fluid(c);
    SPHG_CUDA_CHECK(cudaStreamWaitEvent(c.stream, c.join_ev, 0));
    return;
  }
  const double before10 = c.stage_ms[10], before11 = c.stage_ms[11];
  timed(c, 10, launch_forces_fluid);
  timed(c, 11, launch_forces_rigid);
#ifdef SPHG_DIAG_LOADS_ONLY
  launch_forces_diag(c);  // times its own variants into stage_ms[12..15]
#endif
  c.stage_ms[SPHG_STAGE_FORCES] += (c.stage_ms[10] - before10) + (c.stage_ms[11] - before11);
}

// WallGroup::velocity_at / acceleration_at (config.hpp:42-50) through the host callback, into the
// launch parameters: acc pre-filled with the reference's central difference [P20]
void eval_walls(Ctx& c, double t, double (*vel)[3], double (*acc)[3]) {
  for (int g = 0; g < c.P.n_walls; ++g) {
    double v[3] = {0, 0, 0}, vp[3] = {0, 0, 0}, vm[3] = {0, 0, 0}, a[3], dummy[3];
    const double e = 1e-6;
    c.wall_fn(g, t + e, vp, dummy, c.wall_user);
    c.wall_fn(g, t - e, vm, dummy, c.wall_user);
    for (int k = 0; k < 3; ++k) a[k] = (vp[k] - vm[k]) / (2.0 * e);
    c.wall_fn(g, t, v, a, c.wall_user);
    for (int k = 0; k < 3; ++k) {
      vel[g][k] = v[k];
      if (acc) acc[g][k] = a[k];
    }
  }
}

// which buffer zones prescribe their velocity at t^n, t^{n+1/2}, t^{n+1} [P23]; a launch parameter, so it
// is set before a step's graph key is formed (one_step) — inside a captured body a replay would skip it
void update_buffer_flags(Ctx& c) {
  if (c.P.n_buf <= 0) return;
  c.P.buf_prev = c.P.buf_half = c.P.buf_new = 0u;
  for (int b = 0; b < c.P.n_buf; ++b) {
    const double ts = c.params.buffers[b].t_start;
    if (c.t > ts) c.P.buf_prev |= 1u << b;
    if (c.t + 0.5 * c.P.dt > ts) c.P.buf_half |= 1u << b;
    if (c.t + c.P.dt > ts) c.P.buf_new |= 1u << b;
  }
}

void kick_all(Ctx& c) {
  update_buffer_flags(c);
  if (c.P.n_walls > 0) {
    eval_walls(c, c.t + 0.5 * c.P.dt, c.P.wall_vh, nullptr);
    eval_walls(c, c.t + c.P.dt, c.P.wall_v, c.P.wall_a);
  }
  launch_body_kick(c);
  launch_kick_drift(c);
}

int do_stage(sphg_ctx* h, int stage) {
  Ctx& c = h->c;
  if (!c.have_state) return fail(h, SPHG_ERR_RUNTIME, "no particle state uploaded");
  if (c.n == 0) {  // empty store: every stage is a no-op
    if (stage == SPHG_STAGE_KICK_DRIFT) c.t += c.P.dt;
    return SPHG_OK;
  }
  if (stage != SPHG_STAGE_REBUILD && stage != SPHG_STAGE_KICK_DRIFT && stage != SPHG_STAGE_MASS && !c.built)
    timed(c, SPHG_STAGE_REBUILD, launch_rebuild);
  switch (stage) {
    case SPHG_STAGE_REBUILD: timed(c, stage, launch_rebuild); break;
    case SPHG_STAGE_DENSITY: timed(c, stage, launch_density); break;
    case SPHG_STAGE_HEAT:
      if (c.P.thermal) timed(c, stage, launch_heat);
      if (c.P.diffusion) timed(c, stage, launch_diffusion);
      break;
    case SPHG_STAGE_EXTRAPOLATE: timed(c, stage, launch_extrapolate); break;
    case SPHG_STAGE_FORCES: timed_forces(c); break;
    case SPHG_STAGE_BODIES: timed(c, stage, launch_bodies); break;
    case SPHG_STAGE_KICK_DRIFT:
      reset_step_flags(c);
      timed(c, stage, kick_all);
      c.t += c.P.dt;
      h->mid_step = true;
      break;
    case SPHG_STAGE_FINAL_KICK:
      timed(c, stage, launch_final_kick);
      h->mid_step = false;
      break;
    case SPHG_STAGE_TRANSITIONS:
      if (c.P.transitions != 0 && c.nghost)
        return fail(h, SPHG_ERR_CONFIG, "with ghost particles, transitions are applied by the decomposed batch "
                                        "(SPHG_NEED_TRANSITIONS, sphg_event_bodies / sphg_record_*)");
      if (c.P.transitions != 0) {
        const int rc = launch_transitions(c);
        if (rc) return fail(h, rc, c.err);
      }
      break;
    case SPHG_STAGE_MASS:
      if (!c.built) launch_rigid_index(c);
      launch_mass(c, nullptr);
      break;
    default: return fail(h, SPHG_ERR_RUNTIME, "unknown stage");
  }
  return check_flags(h, true);
}

// ------------------------------------------------------------------ CUDA graphs
// The two launch chains of a step — (A) flag reset + kicks + drift + flag readback, (B) density ..
// final kick — are captured once per distinct launch configuration and replayed: on a 32k-particle
// store the step is launch-latency bound (13-16 launches of a few microseconds each).  The key holds
// every pointer, count and parameter a launch in the chain reads (Particles by value, the kind
// lists, the Verlet rows, the body table, DevParams), so a configuration seen before — e.g. the
// alternating heat buffers, or the cur/alt buffer sets after a reorder — replays its own graph and
// a new one is captured.  Host-side effects of the chain (buffer swaps, deferred final kick, launch
// count) are recorded at capture and re-applied on replay.  Not used with stage timing, moving
// walls (their launch arguments change every step) or ghosts.
template <class T>
void key_put(std::vector<unsigned char>& k, const T& v) {
  const unsigned char* b = reinterpret_cast<const unsigned char*>(&v);
  k.insert(k.end(), b, b + sizeof(T));
}

std::vector<unsigned char> graph_key(const Ctx& c, int chain) {
  std::vector<unsigned char> k;
  k.reserve(2048);
  key_put(k, chain);
  key_put(k, c.cur); key_put(k, c.alt); key_put(k, c.H2new); key_put(k, c.C2new);
  key_put(k, c.bodies.p); key_put(k, c.nbr.p); key_put(k, c.cnt.p); key_put(k, c.cap);
  key_put(k, c.fidx.p); key_put(k, c.widx.p); key_put(k, c.ridx.p); key_put(k, c.body_start.p);
  key_put(k, c.ncon.p); key_put(k, c.pin_list.p); key_put(k, c.hsrc.p);
  key_put(k, c.n); key_put(k, c.nb); key_put(k, c.nf); key_put(k, c.nw); key_put(k, c.nrigid);
  key_put(k, c.group_density); key_put(k, c.group_forces);
  key_put(k, c.defer_final); key_put(k, c.fuse_heat); key_put(k, c.fuse_diff); key_put(k, c.final_pending);
  key_put(k, c.P);
  return k;
}

bool graphs_allowed(const Ctx& c) {
#ifdef SPHG_DIAG_LOADS_ONLY
  return false;  // the diagnostic variants synchronise inside the forces stage
#else
  return c.use_graphs && !c.timing && c.P.n_walls == 0 && c.nghost == 0;
#endif
}

constexpr size_t kMaxGraphs = 8;

void destroy_graphs(Ctx& c) {
  for (auto& e : c.graphs)
    if (e.exec) cudaGraphExecDestroy(e.exec);
  c.graphs.clear();
}

void run_graph(Ctx& c, int chain, void (*body)(Ctx&)) {
  std::vector<unsigned char> key = graph_key(c, chain);
  for (auto& e : c.graphs) {
    if (e.key != key) continue;
    SPHG_CUDA_CHECK(cudaGraphLaunch(e.exec, c.stream));
    c.cur = e.cur_after;
    c.H2new = e.H2new_after;
    c.C2new = e.C2new_after;
    c.final_pending = e.final_pending_after;
    c.launches += e.launches;
    e.used = ++c.graph_clock;
    c.graph_replays++;
    return;
  }
  const int64_t l0 = c.launches;
  SPHG_CUDA_CHECK(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
  c.capturing = true;
  try {
    body(c);
  } catch (...) {
    c.capturing = false;
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(c.stream, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  c.capturing = false;
  cudaGraph_t g = nullptr;
  SPHG_CUDA_CHECK(cudaStreamEndCapture(c.stream, &g));
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ie = cudaGraphInstantiate(&exec, g, 0);
  cudaGraphDestroy(g);
  SPHG_CUDA_CHECK(ie);
  SPHG_CUDA_CHECK(cudaGraphLaunch(exec, c.stream));
  if (c.graphs.size() >= kMaxGraphs) {  // evict the least recently used
    auto lru = std::min_element(c.graphs.begin(), c.graphs.end(),
                                [](const Ctx::GraphEntry& a, const Ctx::GraphEntry& b) { return a.used < b.used; });
    cudaGraphExecDestroy(lru->exec);
    c.graphs.erase(lru);
  }
  Ctx::GraphEntry e;
  e.key = std::move(key);
  e.exec = exec;
  e.launches = c.launches - l0;
  e.cur_after = c.cur;
  e.H2new_after = c.H2new;
  e.C2new_after = c.C2new;
  e.final_pending_after = c.final_pending;
  e.used = ++c.graph_clock;
  c.graphs.push_back(std::move(e));
  c.graph_captures++;
}

void chain_kick(Ctx& c) {  // (A): everything up to the per-step flag readback
  reset_step_flags(c);
  timed(c, SPHG_STAGE_KICK_DRIFT, kick_all);
  launch_step_tail(c);
  SPHG_CUDA_CHECK(cudaMemcpyAsync(c.hflags, c.dflags, sizeof(DevFlags), cudaMemcpyDeviceToHost, c.stream));
}

void chain_forces(Ctx& c) {  // (B): density .. final kick (captured kernels read t^{n+1} from dtime)
  timed(c, SPHG_STAGE_DENSITY, launch_density);
  if (c.P.thermal) timed(c, SPHG_STAGE_HEAT, c.fuse_heat ? launch_heat_begin : launch_heat);
  if (c.P.diffusion) timed(c, SPHG_STAGE_HEAT, c.fuse_diff ? launch_diffusion_begin : launch_diffusion);
  timed(c, SPHG_STAGE_EXTRAPOLATE, launch_extrapolate);
  if (c.pre_forces) c.pre_forces(c);
  timed_forces(c);
  if (c.fuse_heat) launch_heat_end(c);
  if (c.fuse_diff) launch_diffusion_end(c);
  timed(c, SPHG_STAGE_BODIES, launch_bodies);
  timed(c, SPHG_STAGE_FINAL_KICK, launch_final_kick);
}

// Runtime time-step assertion ("refuse with diagnostic listing the violated condition",
// SPEC:558-561): the compute_dt limits with this step's u_max (read from the kick chain's flags) [P22].
int check_dt(sphg_ctx* h) {
  Ctx& c = h->c;
  if (c.params.dt_check == SPHG_DT_OFF) return SPHG_OK;
  static const char* names[5] = {"cfl", "viscous", "body force", "contact", "conduction"};
  double lim[5];
  sphg_dt_limits(&c.params, c.u_max, c.m_r, lim);
  c.dt_term = -1;
  c.dt_limit = std::numeric_limits<double>::infinity();
  std::string bad;
  for (int k = 0; k < 5; ++k) {
    if (lim[k] < c.dt_limit) {
      c.dt_limit = lim[k];
      c.dt_term = k;
    }
    if (c.P.dt > lim[k]) {
      char b[96];
      std::snprintf(b, sizeof b, "%s%s limit %.6g", bad.empty() ? "" : ", ", names[k], lim[k]);
      bad += b;
    }
  }
  if (bad.empty()) return SPHG_OK;
  c.dt_violations++;
  if (c.params.dt_check == SPHG_DT_WARN) return SPHG_OK;
  char b[128];
  std::snprintf(b, sizeof b, "time-step condition violated at step %lld: dt = %.6g exceeds the ", (long long)c.steps,
                c.P.dt);
  return fail(h, SPHG_ERR_RUNTIME, std::string(b) + bad);
}

// ------------------------------------------------------- decomposed step
// One decomposed step on the library stream (sphg.h "In-library decomposed step"): the exchange callback
// enqueues the transfers; the host blocks once, on the flag readback that carries the global Verlet
// decision.
int exchange(sphg_ctx* h, int phase) {
  Ctx& c = h->c;
  static const char* names[5] = {"halo_state", "halo_density", "halo_wall", "xchg_max", "xchg_bodies"};
  NvtxRange nv(phase >= 0 && phase < 5 ? names[phase] : "exchange");
  const int rc = c.exch_fn(phase, reinterpret_cast<void*>(c.stream), c.exch_user);
  if (rc) return fail(h, SPHG_ERR_CUDA, "exchange callback failed in phase " + std::to_string(phase));
  return SPHG_OK;
}

int halo_exchange(sphg_ctx* h, int phase) {
  Ctx& c = h->c;
  for (int slot = 0; slot < SPHG_MAX_HALO_SLOTS; slot += 2)
    if (c.halo_n[slot]) {
      if (!c.halo_buf[phase][slot]) return fail(h, SPHG_ERR_CONFIG, "halo send buffer not bound");
      halo_pack(c, phase, slot, c.halo_buf[phase][slot]);
    }
  const int rc = exchange(h, phase);
  if (rc) return rc;
  for (int slot = 1; slot < SPHG_MAX_HALO_SLOTS; slot += 2)
    if (c.halo_n[slot]) {
      if (!c.halo_buf[phase][slot]) return fail(h, SPHG_ERR_CONFIG, "halo receive buffer not bound");
      halo_unpack(c, phase, slot, c.halo_buf[phase][slot]);
    }
  return SPHG_OK;
}

__global__ void k_flag_error_global(DevFlags* fl) {  // a local error becomes an infinite global displacement
  if (fl->err) fl->max_disp2_bits = 0x7FF0000000000000ull;
}

__global__ void k_event_counts_to_words(const DevFlags* fl, uint64_t* words) {
  words[0] = fl->n_events;  // melt
  words[1] = fl->pad[0];    // solidify
}

int one_step_decomposed(sphg_ctx* h) {
  Ctx& c = h->c;
  reset_step_flags(c);
  kick_all(c);
  k_flag_error_global<<<1, 1, 0, c.stream>>>(c.dflags);
  c.launches++;
  if (!c.max_words) return fail(h, SPHG_ERR_CONFIG, "MAX exchange buffer not bound");
  SPHG_CUDA_CHECK(cudaMemcpyAsync(c.max_words, &c.dflags->max_disp2_bits, 2 * sizeof(uint64_t),
                                  cudaMemcpyDeviceToDevice, c.stream));
  int rc = exchange(h, SPHG_XCHG_MAX);  // global max displacement, u_max (and errors)
  if (rc) return rc;
  SPHG_CUDA_CHECK(cudaMemcpyAsync(&c.dflags->max_disp2_bits, c.max_words, 2 * sizeof(uint64_t),
                                  cudaMemcpyDeviceToDevice, c.stream));
  SPHG_CUDA_CHECK(cudaMemcpyAsync(c.hflags, c.dflags, sizeof(DevFlags), cudaMemcpyDeviceToHost, c.stream));
  host_sync(c, c.stream);
  c.t += c.P.dt;
  h->mid_step = true;
  rc = check_flags(h, false, false);
  if (rc) return rc;
  if (std::isinf(c.max_disp)) return fail(h, SPHG_ERR_RUNTIME, "runtime assertion on another rank at step " +
                                                                     std::to_string(c.steps + 1));
  const bool rebuild = !c.built || c.max_disp > c.P.half_skin;
  // the interior density reads owned neighbours only: it runs while the STATE halo is in flight
  const bool overlap = !rebuild && c.nf_interior > 0;
  if (overlap) {
    if (!c.dens_stream) {
      SPHG_CUDA_CHECK(cudaStreamCreateWithFlags(&c.dens_stream, cudaStreamNonBlocking));
      SPHG_CUDA_CHECK(cudaEventCreateWithFlags(&c.dens_fork, cudaEventDisableTiming));
      SPHG_CUDA_CHECK(cudaEventCreateWithFlags(&c.dens_join, cudaEventDisableTiming));
    }
    SPHG_CUDA_CHECK(cudaEventRecord(c.dens_fork, c.stream));
    SPHG_CUDA_CHECK(cudaStreamWaitEvent(c.dens_stream, c.dens_fork, 0));
    launch_density_interior(c, c.dens_stream);
    SPHG_CUDA_CHECK(cudaEventRecord(c.dens_join, c.dens_stream));
  }
  rc = halo_exchange(h, SPHG_HALO_STATE);
  if (rc) return rc;
  if (rebuild) {
    c.disp_since_partition += c.max_disp;
    timed(c, SPHG_STAGE_REBUILD, launch_rebuild);  // rank-local (the ghost margin covers it)
    launch_density(c);
  } else {
    launch_density_boundary(c);
    if (overlap) SPHG_CUDA_CHECK(cudaStreamWaitEvent(c.stream, c.dens_join, 0));
  }
  if ((rc = halo_exchange(h, SPHG_HALO_DENSITY))) return rc;
  if (c.P.thermal) launch_heat(c);
  if (c.P.diffusion) launch_diffusion(c);
  launch_extrapolate(c);
  if ((rc = halo_exchange(h, SPHG_HALO_WALL))) return rc;
  if (c.pre_forces) c.pre_forces(c);
  timed_forces(c);
  if (c.nb) {
    if (!c.body_part || !c.body_gath) return fail(h, SPHG_ERR_CONFIG, "body exchange buffers not bound");
    body_partials(c, c.body_part);
    if ((rc = exchange(h, SPHG_XCHG_BODIES))) return rc;
    c.body_tot.alloc(c.nb * 12);
    merge_body_partials(c, c.body_gath, c.world, c.body_tot.p);
    body_apply_totals(c, c.body_tot.p);
  }
  launch_final_kick(c);
  h->mid_step = false;
  c.steps++;
  if ((rc = check_dt(h))) return rc;
  if (c.P.transitions) {
    // detection over the owned particles, then the global event counts (MAX over ranks): when any rank
    // has events the caller applies the batch before the next step (sphg.h)
    launch_detect(c);
    k_event_counts_to_words<<<1, 1, 0, c.stream>>>(c.dflags, c.max_words);
    c.launches++;
    if ((rc = exchange(h, SPHG_XCHG_MAX))) return rc;
    uint64_t w[2] = {0, 0};
    SPHG_CUDA_CHECK(cudaMemcpyAsync(w, c.max_words, sizeof w, cudaMemcpyDeviceToHost, c.stream));
    host_sync(c, c.stream);
    if (w[0] || w[1]) return SPHG_NEED_TRANSITIONS;
  }
  return SPHG_OK;
}

int one_step(sphg_ctx* h) {
  Ctx& c = h->c;
  if (c.nghost && c.exch_fn) return one_step_decomposed(h);
  if (c.nghost)
    return fail(h, SPHG_ERR_RUNTIME,
                "ghost particles present: set an exchange callback (sphg_set_exchange) or drive the stages "
                "through the decomposition layer (parallel.py)");
  const bool graphs = graphs_allowed(c);
  update_buffer_flags(c);
  if (graphs) {
    if (!c.dtime) {  // [0] the force chain's time, [1] the clock (see k_step_tail)
      SPHG_CUDA_CHECK(cudaMalloc(&c.dtime, 2 * sizeof(double)));
      SPHG_CUDA_CHECK(cudaMallocHost(&c.htime, 2 * sizeof(double)));
      c.htime[0] = c.htime[1] = c.t;
      SPHG_CUDA_CHECK(cudaMemcpyAsync(c.dtime, c.htime, 2 * sizeof(double), cudaMemcpyHostToDevice, c.stream));
    }
    run_graph(c, 0, chain_kick);
  } else {
    chain_kick(c);
  }
  SPHG_CUDA_CHECK(cudaEventRecord(c.kick_ev, c.stream));
  c.t += c.P.dt;
  h->mid_step = true;
  // fold fluid conduction into the forces pass (same terms, same order; heat does not feed the
  // extrapolation or the forces, so moving it after them changes nothing)
  auto forces = [&]() {
    c.fuse_heat = c.P.thermal && !c.timing;
    c.fuse_diff = c.P.diffusion && !c.P.thermal && !c.timing;  // one scalar field per row walk
    if (graphs && !c.pre_forces) run_graph(c, 1, chain_forces);
    else chain_forces(c);
    c.fuse_heat = c.fuse_diff = false;
  };
  // speculative: queue the force chain before reading the kick chain's flags, so the GPU never waits
  // for the host's one 48-byte readback per step; dskip voids the queued chain when the step needs a
  // rebuild or hit an error, and the host state it changed is restored before the redo
  const bool spec = c.speculate && c.built && !c.timing && !c.pre_forces;
  const Particles cur0 = c.cur;
  const DBuf<double2> h2n0 = c.H2new, c2n0 = c.C2new;
  const bool fp0 = c.final_pending;
  const int64_t l0 = c.launches;
  if (spec) forces();
  host_sync_event(c, c.kick_ev);
  int rc = check_flags(h, false, false);  // Verlet trigger + escape check
  const bool rebuild = !c.built || c.max_disp > c.P.half_skin;
  if (spec && (rc || rebuild)) {  // the queued chain voided itself: restore its host-side state
    host_sync(c, c.stream);
    c.cur = cur0;
    c.H2new = h2n0;
    c.C2new = c2n0;
    c.final_pending = fp0;
    c.launches = l0;
  }
  if (rc || rebuild) SPHG_CUDA_CHECK(cudaMemsetAsync(c.dskip, 0, sizeof(uint32_t), c.stream));
  if (rc) return rc;
  if (rebuild) timed(c, SPHG_STAGE_REBUILD, launch_rebuild);
  if (!spec || rebuild) forces();
  h->mid_step = false;
  if (c.P.transitions != 0) {
    float ms = 0.f;
    if (c.timing) SPHG_CUDA_CHECK(cudaEventRecord(c.ev[0], c.stream));
    rc = launch_transitions(c);
    if (rc) return fail(h, rc, c.err);
    if (c.timing) {
      SPHG_CUDA_CHECK(cudaEventRecord(c.ev[1], c.stream));
      SPHG_CUDA_CHECK(cudaEventSynchronize(c.ev[1]));
      SPHG_CUDA_CHECK(cudaEventElapsedTime(&ms, c.ev[0], c.ev[1]));
      c.stage_ms[SPHG_STAGE_TRANSITIONS] += ms;
    }
  }
  c.steps++;
  return check_dt(h);
}

template <class T>
void d2h(T* dst, const T* src, size_t n, cudaStream_t s) {
  if (n) SPHG_CUDA_CHECK(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyDeviceToHost, s));
}
template <class T>
void h2d(T* dst, const T* src, size_t n, cudaStream_t s) {
  if (n) SPHG_CUDA_CHECK(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyHostToDevice, s));
}

// ------------------------------------------------------- host <-> device staging
// The host store is packed/unpacked in chunks through two pinned staging slots
// (OpenMP over particles) so the PCIe copies overlap the packing of the next
// chunk.  Device order == gid order on a cold upload; a warm upload lands in
// the alternate buffers and is gathered through the gid permutation.
constexpr size_t kChunk = 1u << 18;  // particles per staging chunk
constexpr size_t kPackBytes =
    8 * sizeof(double4) + 2 * sizeof(double2) + 3 * sizeof(double) + 2 * sizeof(uint32_t);

struct Slot {
  double4 *G0, *G1, *G2, *V4, *A4, *B4, *F4, *X4;
  double2 *H2, *C2;
  double *dT, *ps, *dC;
  uint32_t *kmd, *grp, *gid;
};

Slot slot_view(char* base) {
  Slot s;
  size_t o = 0;
  auto take = [&](auto*& p, size_t bytes) {
    p = reinterpret_cast<std::remove_reference_t<decltype(p)>>(base + o);
    o += bytes;
  };
  take(s.G0, kChunk * 32); take(s.G1, kChunk * 32); take(s.G2, kChunk * 32); take(s.V4, kChunk * 32);
  take(s.A4, kChunk * 32); take(s.B4, kChunk * 32); take(s.F4, kChunk * 32); take(s.X4, kChunk * 32);
  take(s.H2, kChunk * 16); take(s.C2, kChunk * 16); take(s.dT, kChunk * 8); take(s.ps, kChunk * 8);
  take(s.dC, kChunk * 8);
  take(s.kmd, kChunk * 4); take(s.grp, kChunk * 4); take(s.gid, kChunk * 4);
  return s;
}

void ensure_staging(Ctx& c) {
  if (c.hstage) return;
  SPHG_CUDA_CHECK(cudaMallocHost(&c.hstage, 2 * kChunk * (kPackBytes + 4)));
  for (auto& e : c.slot_ev) SPHG_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}

void stage_upload(Ctx& c, const sphg_soa* s, Particles& dst) {
  ensure_staging(c);
  const bool conc = c.P.diffusion != 0;
  const size_t n = s->n;
  const size_t slot_bytes = kChunk * (kPackBytes + 4);
  auto v3 = [](const double* p, size_t i) {
    return p ? make_double3(p[3 * i], p[3 * i + 1], p[3 * i + 2]) : make_double3(0, 0, 0);
  };
  auto s1 = [](const double* p, size_t i) { return p ? p[i] : 0.0; };
  int slot = 0;
  for (size_t k0 = 0; k0 < n; k0 += kChunk, slot ^= 1) {
    const size_t m = std::min(kChunk, n - k0);
    SPHG_CUDA_CHECK(cudaEventSynchronize(c.slot_ev[slot]));
    Slot S = slot_view(static_cast<char*>(c.hstage) + slot * slot_bytes);
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < (int64_t)m; ++q) {
      const size_t i = k0 + (size_t)q;
      const uint32_t kind = s->kind ? s->kind[i] : 0;
      const uint32_t mat = s->material ? s->material[i] : 0;
      const uint32_t dir = s->dirichlet_T ? s->dirichlet_T[i] : SPHG_NO_DIRICHLET;
      const double3 x = v3(s->pos, i), u = v3(s->vel, i), ua = v3(s->vel_adv, i);
      const double mass = s1(s->mass, i), rho = s1(s->density, i), p = s1(s->pressure, i);
      const DevMat& M = c.P.mat[mat];
      const double V = rho > 0.0 ? mass / rho : 0.0;
      S.G0[q] = make_double4(x.x, x.y, x.z, V * V);
      if (kind == SPHG_FLUID) {
        S.G1[q] = make_double4(u.x, u.y, u.z, rho);
        S.G2[q] = make_double4(ua.x - u.x, ua.y - u.y, ua.z - u.z, p);
      } else {
        const double3 wv = v3(s->wall_velocity, i);
        S.G1[q] = make_double4(wv.x, wv.y, wv.z, rho);
        S.G2[q] = make_double4(0, 0, 0, s1(s->wall_pressure, i));
      }
      S.V4[q] = make_double4(u.x, u.y, u.z, mass);
      const double3 a = v3(s->acc, i), bg = v3(s->acc_bg, i), f = v3(s->force, i), chi = v3(s->body_frame_pos, i);
      S.A4[q] = make_double4(a.x, a.y, a.z, 0);
      S.B4[q] = make_double4(bg.x, bg.y, bg.z, 0);
      S.F4[q] = make_double4(f.x, f.y, f.z, 0);
      S.X4[q] = make_double4(chi.x, chi.y, chi.z, 0);
      double Vh = 0.0;
      if (kind == SPHG_FLUID) Vh = V;
      else if (kind == SPHG_RIGID) Vh = mass / M.rho0;
      else if (dir != SPHG_NO_DIRICHLET) Vh = mass / M.rho0;  // [P9]
      S.H2[q] = make_double2(s1(s->temperature, i), Vh);
      S.dT[q] = s1(s->dT_dt, i);
      S.ps[q] = p;
      const uint32_t dirc = s->dirichlet_C ? s->dirichlet_C[i] : SPHG_NO_DIRICHLET;
      if (conc) {  // diffusion volume: fluid m/rho, rigid and Dirichlet-C walls m/rho0, other walls 0
        double Vc = 0.0;
        if (kind == SPHG_FLUID) Vc = V;
        else if (kind == SPHG_RIGID || dirc != SPHG_NO_DIRICHLET) Vc = mass / M.rho0;
        S.C2[q] = make_double2(s1(s->concentration, i), Vc);
        S.dC[q] = s1(s->dC_dt, i);
      }
      const bool ghost = s->owner && s->owner[i] != (uint32_t)c.params.rank;
      S.kmd[q] = make_kmd(kind, mat, dir, dirc) | (ghost ? kGhostBit : 0u);
      S.grp[q] = s->group ? s->group[i] : 0;
    }
    cudaStream_t st = c.stream;
    h2d(dst.G0.p + k0, S.G0, m, st); h2d(dst.G1.p + k0, S.G1, m, st); h2d(dst.G2.p + k0, S.G2, m, st);
    h2d(dst.V4.p + k0, S.V4, m, st); h2d(dst.A4.p + k0, S.A4, m, st); h2d(dst.B4.p + k0, S.B4, m, st);
    h2d(dst.F4.p + k0, S.F4, m, st); h2d(dst.X4.p + k0, S.X4, m, st); h2d(dst.H2.p + k0, S.H2, m, st);
    h2d(dst.dTdt.p + k0, S.dT, m, st); h2d(dst.p_static.p + k0, S.ps, m, st);
    h2d(dst.kmd.p + k0, S.kmd, m, st); h2d(dst.group.p + k0, S.grp, m, st);
    if (conc) {
      h2d(dst.C2.p + k0, S.C2, m, st);
      h2d(dst.dCdt.p + k0, S.dC, m, st);
    }
    SPHG_CUDA_CHECK(cudaEventRecord(c.slot_ev[slot], st));
  }
}

// Download: one kernel computes every requested store field from the device records and scatters
// it into gid order in a device buffer (the reference's SoA layout, interleaved xyz); each field is
// then one contiguous D2H copy — straight into the caller's array when it is pinned, else through
// the two pinned staging slots with the host memcpy of one chunk overlapping the copy of the next.
struct OutPtrs {
  double *pos, *vel, *vel_adv, *acc, *acc_bg, *body_frame_pos, *wall_velocity, *force;
  double *density, *pressure, *mass, *temperature, *dT_dt, *wall_pressure;
  uint8_t* kind;
  uint32_t* group;
  uint16_t* material;
  uint8_t* dirichlet_T;
  uint32_t* owner;
  double *concentration, *dC_dt;
  uint8_t* dirichlet_C;
};

__global__ void k_pack_store(const __grid_constant__ DevParams P, Particles D, size_t n, int mid_step,
                             uint32_t rank, OutPtrs o) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const size_t g = D.gid.p[k];
  const uint32_t kmd = D.kmd.p[k];
  const uint32_t kind = kind_of(kmd), mat = mat_of(kmd);
  const bool fl = kind == SPHG_FLUID;
  auto put = [](double* p, size_t g, double x, double y, double z) {
    if (p) {
      p[3 * g] = x;
      p[3 * g + 1] = y;
      p[3 * g + 2] = z;
    }
  };
  if (o.pos) {
    const double4 G0 = D.G0.p[k];
    put(o.pos, g, G0.x, G0.y, G0.z);
  }
  const bool needG1 = o.vel || o.vel_adv || o.wall_velocity || o.density;
  const bool needG2 = o.vel_adv || o.pressure || o.wall_pressure;
  const bool needV4 = o.vel || o.vel_adv || o.mass;
  const double4 z4 = make_double4(0, 0, 0, 0);
  const double4 G1 = needG1 ? D.G1.p[k] : z4, G2 = needG2 ? D.G2.p[k] : z4, V4 = needV4 ? D.V4.p[k] : z4;
  if (fl && mid_step) put(o.vel, g, G1.x, G1.y, G1.z);
  else put(o.vel, g, V4.x, V4.y, V4.z);
  if (fl) put(o.vel_adv, g, G1.x + G2.x, G1.y + G2.y, G1.z + G2.z);
  else if (kind == SPHG_RIGID) put(o.vel_adv, g, V4.x, V4.y, V4.z);
  else put(o.vel_adv, g, 0, 0, 0);
  if (o.acc) { const double4 a = D.A4.p[k]; put(o.acc, g, a.x, a.y, a.z); }
  if (o.acc_bg) { const double4 a = D.B4.p[k]; put(o.acc_bg, g, a.x, a.y, a.z); }
  if (o.force) { const double4 a = D.F4.p[k]; put(o.force, g, a.x, a.y, a.z); }
  if (o.body_frame_pos) { const double4 a = D.X4.p[k]; put(o.body_frame_pos, g, a.x, a.y, a.z); }
  if (fl) put(o.wall_velocity, g, 0, 0, 0);
  else put(o.wall_velocity, g, G1.x, G1.y, G1.z);
  if (o.density) o.density[g] = kind == SPHG_RIGID ? P.mat[mat].rho0 : G1.w;
  if (o.pressure) o.pressure[g] = fl ? G2.w : D.p_static.p[k];
  if (o.wall_pressure) o.wall_pressure[g] = fl ? 0.0 : G2.w;
  if (o.mass) o.mass[g] = V4.w;
  if (o.temperature) o.temperature[g] = D.H2.p[k].x;
  if (o.dT_dt) o.dT_dt[g] = D.dTdt.p[k];
  if (o.kind) o.kind[g] = (uint8_t)kind;
  if (o.group) o.group[g] = D.group.p[k];
  if (o.material) o.material[g] = (uint16_t)mat;
  if (o.dirichlet_T) o.dirichlet_T[g] = (uint8_t)dir_of(kmd);
  if (o.owner) o.owner[g] = is_ghost(kmd) ? 0xffffffffu : rank;
  if (o.concentration) o.concentration[g] = D.C2.p ? D.C2.p[k].x : 0.0;
  if (o.dC_dt) o.dC_dt[g] = D.dCdt.p ? D.dCdt.p[k] : 0.0;
  if (o.dirichlet_C) o.dirichlet_C[g] = (uint8_t)dirc_of(kmd);
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// contiguous device -> host copy of `bytes` (queued on the stream; returns after completion)
void copy_out(Ctx& c, void* dst, const void* src, size_t bytes, cudaStream_t st = nullptr) {
  if (!bytes) return;
  if (!st) st = c.stream;
  if (is_pinned(dst)) {
    SPHG_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
    return;
  }
  ensure_staging(c);
  const size_t slot_bytes = kChunk * (kPackBytes + 4);
  char* hs = static_cast<char*>(c.hstage);
  int prev = -1;
  size_t prev_off = 0, prev_len = 0;
  auto drain = [&](int sl, size_t off, size_t len) {
    SPHG_CUDA_CHECK(cudaEventSynchronize(c.slot_ev[sl]));
    const char* from = hs + sl * slot_bytes;
    char* to = static_cast<char*>(dst) + off;
    const int64_t parts = (int64_t)std::min<size_t>(64, (len + 65535) / 65536);
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < parts; ++q) {
      const size_t b0 = len * q / parts, b1 = len * (q + 1) / parts;
      std::memcpy(to + b0, from + b0, b1 - b0);
    }
  };
  int slot = 0;
  for (size_t off = 0; off < bytes; off += slot_bytes, slot ^= 1) {
    const size_t len = std::min(slot_bytes, bytes - off);
    SPHG_CUDA_CHECK(cudaEventSynchronize(c.slot_ev[slot]));
    SPHG_CUDA_CHECK(cudaMemcpyAsync(hs + slot * slot_bytes, static_cast<const char*>(src) + off, len,
                                    cudaMemcpyDeviceToHost, st));
    SPHG_CUDA_CHECK(cudaEventRecord(c.slot_ev[slot], st));
    if (prev >= 0) drain(prev, prev_off, prev_len);
    prev = slot;
    prev_off = off;
    prev_len = len;
  }
  if (prev >= 0) drain(prev, prev_off, prev_len);
}

// The requested store fields, carved out of dl_buf.  early = final once the wall extrapolation has run
// (positions, density, pressure, wall state, mass, body-frame offsets, tags): the final kick only
// writes V4.xyz, so with transitions off these can leave the device while the forces run.
struct DlPlan {
  OutPtrs early{}, late{};
  struct Item {
    void* host;
    const void* dev;
    size_t bytes;
    bool early;
  };
  std::vector<Item> items;
  size_t bytes = 0;
};

DlPlan plan_download(Ctx& c, sphg_soa* o) {
  DlPlan pl;
  const size_t n = c.n;
  struct F {
    void* host;
    size_t elem;
    bool early;
    void** e;
    void** l;
  };
  OutPtrs& E = pl.early;
  OutPtrs& L = pl.late;
#define SPHG_DL(name, elem, early) {o->name, elem, early, (void**)&E.name, (void**)&L.name}
  const F fields[] = {SPHG_DL(pos, 24, true), SPHG_DL(vel, 24, false), SPHG_DL(vel_adv, 24, false),
                      SPHG_DL(acc, 24, false), SPHG_DL(acc_bg, 24, false), SPHG_DL(body_frame_pos, 24, true),
                      SPHG_DL(wall_velocity, 24, true), SPHG_DL(force, 24, false), SPHG_DL(density, 8, true),
                      SPHG_DL(pressure, 8, true), SPHG_DL(mass, 8, true), SPHG_DL(temperature, 8, false),
                      SPHG_DL(dT_dt, 8, false), SPHG_DL(wall_pressure, 8, true), SPHG_DL(kind, 1, true),
                      SPHG_DL(group, 4, true), SPHG_DL(material, 2, true), SPHG_DL(dirichlet_T, 1, true),
                      SPHG_DL(owner, 4, true), SPHG_DL(concentration, 8, false), SPHG_DL(dC_dt, 8, false),
                      SPHG_DL(dirichlet_C, 1, true)};
#undef SPHG_DL
  size_t total = 0;
  for (const F& f : fields)
    if (f.host) total += (n * f.elem + 255) / 256 * 256;
  if (total == 0 || n == 0) return pl;
  c.dl_buf.alloc(total);
  size_t off = 0;
  for (const F& f : fields)
    if (f.host) {
      void* dev = c.dl_buf.p + off;
      *(f.early ? f.e : f.l) = dev;
      pl.items.push_back({f.host, dev, n * f.elem, f.early});
      pl.bytes += n * f.elem;
      off += (n * f.elem + 255) / 256 * 256;
    }
  return pl;
}

void pack(Ctx& c, const OutPtrs& d, bool mid_step) {
  k_pack_store<<<grid_for(c.n, 256), 256, 0, c.stream>>>(c.P, c.cur, c.n, mid_step ? 1 : 0,
                                                         (uint32_t)c.params.rank, d);
  c.launches++;
}

OutPtrs merged(const DlPlan& pl) {  // every requested field in one pack
  OutPtrs d = pl.early;
  const void* const* l = reinterpret_cast<const void* const*>(&pl.late);
  void** m = reinterpret_cast<void**>(&d);
  for (size_t k = 0; k < sizeof(OutPtrs) / sizeof(void*); ++k)
    if (l[k]) m[k] = const_cast<void*>(l[k]);
  return d;
}

void stage_download(Ctx& c, sphg_soa* o, bool mid_step) {
  if (c.n == 0) return;
  DlPlan pl = plan_download(c, o);
  if (pl.items.empty()) return;
  pack(c, merged(pl), mid_step);
  for (const auto& it : pl.items) copy_out(c, it.host, it.dev, it.bytes);
  host_sync(c, c.stream);
  c.last_d2h_bytes = pl.bytes;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

int sphg_validate(const sphg_params* p, char* buf, size_t len) {
  const auto v = validate(*p);
  std::string s;
  for (size_t i = 0; i < v.size(); ++i) s += (i ? "\n" : "") + v[i];
  if (buf && len) {
    std::strncpy(buf, s.c_str(), len - 1);
    buf[len - 1] = 0;
  }
  return v.empty() ? SPHG_OK : SPHG_ERR_CONFIG;
}

int sphg_create(const sphg_params* p, int device, sphg_ctx** out) {
  *out = nullptr;
  if (!validate(*p).empty()) return SPHG_ERR_CONFIG;
  sphg_ctx* h = new sphg_ctx();
  Ctx& c = h->c;
  c.params = *p;
  if (c.params.h <= 0.0) c.params.h = c.params.dx;
  c.P = make_dev_params(c.params);
  c.device = device;
  c.t = p->t0;
  c.ncells = (int64_t)c.P.ncell[0] * c.P.ncell[1] * c.P.ncell[2];
  if (const char* e = std::getenv("SPHG_GROUP_DENSITY")) c.group_density = std::atoi(e);
  if (const char* e = std::getenv("SPHG_GROUP_FORCES")) c.group_forces = std::atoi(e);
  if (const char* e = std::getenv("SPHG_CELL_BUILD")) c.cell_build = std::atoi(e) != 0;
  if (const char* e = std::getenv("SPHG_GRAPHS")) c.use_graphs = std::atoi(e) != 0;
  if (const char* e = std::getenv("SPHG_CONCURRENT_RIGID")) c.concurrent_rigid = std::atoi(e) != 0;
  if (const char* e = std::getenv("SPHG_SPECULATE")) c.speculate = std::atoi(e) != 0;
  try {
    SPHG_CUDA_CHECK(cudaSetDevice(device));
    int sms = 148;
    SPHG_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    c.fill_groups = (size_t)sms * 2048 / 4 / 2;
    if (const char* e = std::getenv("SPHG_FILL_GROUPS")) c.fill_groups = (size_t)std::atoll(e);  // tests: 0 = always 4 lanes
    c.n_sms = sms;
    if (const char* e = std::getenv("SPHG_SM_LOCAL")) c.sm_local = std::atoi(e);
    if (const char* e = std::getenv("SPHG_SM_LOCAL_MIN")) c.sm_local_min = (size_t)std::atoll(e);
    if (const char* e = std::getenv("SPHG_SM_THREADS")) {
      const int t = std::atoi(e);
      if (t == 32 || t == 64 || t == 128) c.sm_threads = t;
    }
    c.sm_next.alloc(6 * (size_t)sms);  // density, fluid forces, extrapolation, rigid forces, interior density, heat
    SPHG_CUDA_CHECK(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
    SPHG_CUDA_CHECK(cudaMalloc(&c.dflags, sizeof(DevFlags)));
    SPHG_CUDA_CHECK(cudaMemset(c.dflags, 0, sizeof(DevFlags)));
    // the offending gids are reduced with atomicMin: start them at "none"
    SPHG_CUDA_CHECK(cudaMemset(&c.dflags->err_gid, 0xff, 2 * sizeof(uint32_t)));
    SPHG_CUDA_CHECK(cudaMallocHost(&c.hflags, sizeof(DevFlags)));
    std::memset(c.hflags, 0, sizeof(DevFlags));
    SPHG_CUDA_CHECK(cudaMalloc(&c.dskip, sizeof(uint32_t)));
    SPHG_CUDA_CHECK(cudaMemset(c.dskip, 0, sizeof(uint32_t)));
    c.P.skip = c.dskip;
    SPHG_CUDA_CHECK(cudaEventCreateWithFlags(&c.kick_ev, cudaEventDisableTiming));
    SPHG_CUDA_CHECK(cudaEventCreate(&c.ev[0]));
    SPHG_CUDA_CHECK(cudaEventCreate(&c.ev[1]));
  } catch (const CudaError& e) {
    delete h;
    return SPHG_ERR_CUDA;
  }
  *out = h;
  return SPHG_OK;
}

// device arrays for a store of n particles (sphg_upload, sphg_upload_records)
void alloc_store(Ctx& c, size_t n) {
  c.n = n;
  const size_t na = std::max<size_t>(n, 1);
  c.cur.alloc(na, c.P.diffusion != 0);
  c.alt.alloc(na, c.P.diffusion != 0);
  c.H2new.alloc(na);
  c.pin_list.alloc(na);
  c.wrap_list.alloc(2 * na);  // periodic-face crossings of a step (allocated here: the kick chain is captured)
  if (!c.pin_any) SPHG_CUDA_CHECK(cudaMalloc(&c.pin_any, sizeof(uint32_t)));
  if (c.P.diffusion) c.C2new.alloc(na);
  if (c.P.heat_source) {
    c.hsrc.alloc(na);
    c.P.hsrc = c.hsrc.p;
  }
  c.keys.alloc(na);
  c.keys_alt.alloc(na);
  c.vals.alloc(na);
  c.vals_alt.alloc(na);
  c.hist.alloc(radix_scratch_words(na));
  c.scan_tmp.alloc(radix_scratch_words(na));
  c.cell_start.alloc(c.ncells);
  c.cell_end.alloc(c.ncells);
  c.cell_key.alloc(na);
  c.cnt.alloc(na);
  const bool any_periodic = c.P.periodic[0] || c.P.periodic[1] || c.P.periodic[2];
  // image-coded entries need the index in 27 bits; larger stores use the minimum image
  // (SPHG_IMG_MIN=1 forces that path for testing at small sizes)
  static const bool force_min = std::getenv("SPHG_IMG_MIN") && std::atoi(std::getenv("SPHG_IMG_MIN")) != 0;
  const int mode = !any_periodic ? kImgNone : ((n < (size_t(1) << kIdxBits) && !force_min) ? kImgCode : kImgMin);
  if (mode != c.P.img_mode) {
    c.P.img_mode = mode;
    c.built = false;
  }
}

int sphg_upload(sphg_ctx* h, const sphg_soa* s, const sphg_body* bodies, size_t nb) {
  return guarded(h, [&]() -> int {
    Ctx& c = h->c;
    SPHG_CUDA_CHECK(cudaSetDevice(c.device));
    const size_t n = s->n;
    if (n >= (size_t)UINT32_MAX) return fail(h, SPHG_ERR_CONFIG, "too many particles for 32-bit gids");
    // validate tags first (nothing is modified on failure)
    double m_r = 0.0;  // [P22]: rigid particles, and fluid particles that may solidify
    for (size_t i = 0; i < n; ++i) {
      const uint32_t kind = s->kind ? s->kind[i] : 0;
      const uint32_t mat = s->material ? s->material[i] : 0;
      if (kind > 2 || (int)mat >= c.params.n_mat)
        return fail(h, SPHG_ERR_CONFIG, "particle " + std::to_string(i) + " has an invalid kind/material");
      if (kind == SPHG_RIGID && (s->group ? s->group[i] : 0) >= nb)
        return fail(h, SPHG_ERR_CONFIG, "rigid particle " + std::to_string(i) + " refers to a missing body");
      const bool can_be_rigid = kind == SPHG_RIGID || (kind == SPHG_FLUID && c.params.transitions != 0 &&
                                                       c.params.mat[mat].solidify_target >= 0);
      const double m = s->mass ? s->mass[i] : 0.0;
      if (can_be_rigid && m > 0.0 && (m_r == 0.0 || m < m_r)) m_r = m;
    }
    c.m_r = m_r;
    size_t ng = 0;
    if (s->owner)
      for (size_t i = 0; i < n; ++i) ng += s->owner[i] != (uint32_t)c.params.rank ? 1 : 0;
    c.nghost = ng;
    c.disp_since_partition = 0.0;
    // buffers below may be reallocated (and a freed address handed out again): no captured graph may
    // survive an upload (the graph key holds raw pointers)
    host_sync(c, c.stream);
    destroy_graphs(c);
    // warm upload: same store size and a valid Verlet list -> keep the device order and the list,
    // scatter the host (gid-ordered) data through the gid permutation
    const bool warm = c.built && c.have_state && n == c.n && n > 0;
    alloc_store(c, n);
    Particles& dst = (warm && c.built) ? c.alt : c.cur;
    stage_upload(c, s, dst);
    if (warm && c.built) {
      gather_by_gid(c);  // cur[k] <- alt[gid[k]] (keeps gid, R4, list)
      if (displacement_exceeds(c)) c.built = false;
    } else {
      iota_gid(c);
      build_idx_of_gid(c);
      SPHG_CUDA_CHECK(cudaMemcpyAsync(c.cur.R4.p, c.cur.G0.p, n * sizeof(double4), cudaMemcpyDeviceToDevice, c.stream));
      c.built = false;
    }
    c.nb = 0;
    ensure_bodies(c, nb);
    c.nb = nb;
    h2d(c.bodies.p, bodies, nb, c.stream);
    SPHG_CUDA_CHECK(cudaMemsetAsync(c.dflags, 0, sizeof(DevFlags), c.stream));
    SPHG_CUDA_CHECK(cudaMemsetAsync(&c.dflags->err_gid, 0xff, 2 * sizeof(uint32_t), c.stream));
    if (c.built) {  // kinds / bodies may have changed
      launch_rigid_index(c);
      launch_contact_order(c);
      launch_ghost_split(c);
    }
    host_sync(c, c.stream);
    c.have_state = true;
    h->mid_step = false;
    return SPHG_OK;
  });
}

int sphg_upload_state(sphg_ctx* h, const double* pos, const double* vel, size_t n) {
  return guarded(h, [&]() -> int {
    Ctx& c = h->c;
    SPHG_CUDA_CHECK(cudaSetDevice(c.device));
    if (!c.have_state || n != c.n) return fail(h, SPHG_ERR_RUNTIME, "upload_state: store size mismatch (upload first)");
    if (n == 0) return SPHG_OK;
    if (!c.built) {  // device order is gid order until the first rebuild
      build_idx_of_gid(c);
    }
    c.state_buf.alloc(6 * n);
    if (pos) h2d(c.state_buf.p, pos, 3 * n, c.stream);
    if (vel) h2d(c.state_buf.p + 3 * n, vel, 3 * n, c.stream);
    scatter_state(c, pos ? c.state_buf.p : nullptr, vel ? c.state_buf.p + 3 * n : nullptr);
    c.last_h2d_bytes = (pos ? 24 : 0) * n + (vel ? 24 : 0) * n;
    if (c.built && pos && displacement_exceeds(c)) c.built = false;
    host_sync(c, c.stream);
    h->mid_step = false;
    return SPHG_OK;
  });
}

int sphg_set_wall_motion(sphg_ctx* h, int32_t n_groups, sphg_wall_motion_fn fn, void* user) {
  return guarded(h, [&]() -> int {
    Ctx& c = h->c;
    if (n_groups < 0 || n_groups > SPHG_MAX_WALL_GROUPS) return fail(h, SPHG_ERR_CONFIG, "wall group count out of range");
    c.wall_fn = fn;
    c.wall_user = user;
    c.P.n_walls = fn ? n_groups : 0;
    if (c.P.n_walls) eval_walls(c, c.t, c.P.wall_v, c.P.wall_a);  // state at the current time (a^0)
    return SPHG_OK;
  });
}

int sphg_initialize(sphg_ctx* h) {
  return guarded(h, [&]() -> int {
    if (h->c.P.n_walls) eval_walls(h->c, h->c.t, h->c.P.wall_v, h->c.P.wall_a);
    for (int s : {SPHG_STAGE_REBUILD, SPHG_STAGE_DENSITY, SPHG_STAGE_EXTRAPOLATE, SPHG_STAGE_FORCES, SPHG_STAGE_BODIES}) {
      const int rc = do_stage(h, s);
      if (rc) return rc;
    }
    return SPHG_OK;
  });
}

}  // extern "C"

namespace {
// nsteps full steps; with `out`, the requested store fields are downloaded at the end.  With
// transitions off, the fields that are final after the last step's wall extrapolation (DlPlan::early)
// are packed there and copied on copy_stream while the force kernels run; the rest after the final
// kick.  Same values as sphg_step followed by sphg_download.
int run_steps(sphg_ctx* h, int nsteps, sphg_soa* out) {
  Ctx& c = h->c;
  NvtxRange nv(out ? "sphg_step_download" : "sphg_step");
  if (!c.have_state) return fail(h, SPHG_ERR_RUNTIME, "no particle state uploaded");
  if (out && out->n != c.n) return fail(h, SPHG_ERR_RUNTIME, "download: store size mismatch");
  SPHG_CUDA_CHECK(cudaSetDevice(c.device));
  if (c.n == 0) {
    c.steps += nsteps;
    c.t += nsteps * c.P.dt;
    return SPHG_OK;
  }
  if (!c.step_ev[0]) {
    SPHG_CUDA_CHECK(cudaEventCreate(&c.step_ev[0]));
    SPHG_CUDA_CHECK(cudaEventCreate(&c.step_ev[1]));
  }
  if (c.dtime) {  // the captured force chain reads its time from the device clock: resync it with c.t
    c.htime[0] = c.htime[1] = c.t;
    SPHG_CUDA_CHECK(cudaMemcpyAsync(c.dtime, c.htime, 2 * sizeof(double), cudaMemcpyHostToDevice, c.stream));
  }
  const bool overlap = out && nsteps > 0 && c.P.transitions == 0 && !c.timing;
  DlPlan pl;
  if (overlap) {
    pl = plan_download(c, out);
    if (!c.copy_stream) {
      SPHG_CUDA_CHECK(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking));
      SPHG_CUDA_CHECK(cudaEventCreateWithFlags(&c.dl_ev, cudaEventDisableTiming));
    }
  }
  SPHG_CUDA_CHECK(cudaEventRecord(c.step_ev[0], c.stream));
  for (int k = 0; k < nsteps; ++k) {
    // decomposed runs: stop before a step the partition might not cover (the caller repartitions and
    // calls again for the remaining steps): a particle's drift since its partition is bounded by the
    // displacements at the rebuilds since then plus the current one, and a step adds at most half a skin
    if (c.nghost && c.partition_limit > 0.0 && c.disp_since_partition + c.max_disp + c.P.half_skin > c.partition_limit) {
      if (c.final_pending) launch_final_kick_particles(c);
      c.defer_final = false;
      host_sync(c, c.stream);
      return SPHG_NEED_PARTITION;
    }
    c.defer_final = k + 1 < nsteps && c.P.transitions == 0 && !c.timing;
    if (overlap && k + 1 == nsteps)
      c.pre_forces = [&pl](Ctx& cc) {
        pack(cc, pl.early, false);
        SPHG_CUDA_CHECK(cudaEventRecord(cc.dl_ev, cc.stream));
      };
    const int rc = one_step(h);
    c.pre_forces = nullptr;
    if (rc) {
      c.defer_final = false;
      if (c.final_pending) launch_final_kick_particles(c);  // leave a complete state behind
      return rc;
    }
  }
  c.defer_final = false;
  size_t bytes = 0;
  if (overlap) {  // the forces of the last step are queued on c.stream: copy the early fields meanwhile
    SPHG_CUDA_CHECK(cudaStreamWaitEvent(c.copy_stream, c.dl_ev, 0));
    for (const auto& it : pl.items)
      if (it.early) copy_out(c, it.host, it.dev, it.bytes, c.copy_stream);
    pack(c, pl.late, false);
  }
  SPHG_CUDA_CHECK(cudaEventRecord(c.step_ev[1], c.stream));
  const int rc = check_flags(h, true);
  float ms = 0.f;
  SPHG_CUDA_CHECK(cudaEventElapsedTime(&ms, c.step_ev[0], c.step_ev[1]));
  c.last_step_ms = ms;
  if (overlap) host_sync(c, c.copy_stream);  // never leave copies in flight
  if (rc || !out) return rc;
  if (overlap) {
    for (const auto& it : pl.items)
      if (!it.early) copy_out(c, it.host, it.dev, it.bytes);
    host_sync(c, c.stream);
    host_sync(c, c.copy_stream);
    for (const auto& it : pl.items) bytes += it.bytes;
    c.last_d2h_bytes = bytes;
  } else {
    stage_download(c, out, false);
  }
  return SPHG_OK;
}
}  // namespace

extern "C" {

int sphg_step(sphg_ctx* h, int nsteps) {
  return guarded(h, [&]() -> int { return run_steps(h, nsteps, nullptr); });
}

int sphg_step_download(sphg_ctx* h, int nsteps, sphg_soa* out, sphg_body* bodies, size_t* nb_io) {
  return guarded(h, [&]() -> int {
    const int rc = run_steps(h, nsteps, out);
    if (rc) return rc;
    Ctx& c = h->c;
    if (nb_io) {
      if (bodies) d2h(bodies, c.bodies.p, std::min(*nb_io, c.nb), c.stream);
      host_sync(c, c.stream);
      *nb_io = c.nb;
    }
    return SPHG_OK;
  });
}

int sphg_run_stage(sphg_ctx* h, int stage) {
  return guarded(h, [&]() -> int {
    SPHG_CUDA_CHECK(cudaSetDevice(h->c.device));
    return do_stage(h, stage);
  });
}

int sphg_num_bodies(sphg_ctx* h, size_t* nb) {
  *nb = h->c.nb;
  return SPHG_OK;
}

int sphg_download(sphg_ctx* h, sphg_soa* o, sphg_body* bodies, size_t* nb_io) {
  return guarded(h, [&]() -> int {
    Ctx& c = h->c;
    SPHG_CUDA_CHECK(cudaSetDevice(c.device));
    if (o->n != c.n) return fail(h, SPHG_ERR_RUNTIME, "download: store size mismatch");
    stage_download(c, o, h->mid_step);
    if (nb_io) {
      if (bodies) d2h(bodies, c.bodies.p, std::min(*nb_io, c.nb), c.stream);
      host_sync(c, c.stream);
      *nb_io = c.nb;
    }
    return SPHG_OK;
  });
}

int sphg_get_cells(sphg_ctx* h, int64_t* cell_of_gid, uint32_t* sorted_gid) {
  return guarded(h, [&]() -> int {
    Ctx& c = h->c;
    if (!c.built) {
      const int rc = do_stage(h, SPHG_STAGE_REBUILD);
      if (rc) return rc;
    }
    const size_t n = c.n;
    std::vector<uint32_t> key(n), gid(n);
    d2h(key.data(), c.cell_key.p, n, c.stream);
    d2h(gid.data(), c.cur.gid.p, n, c.stream);
    host_sync(c, c.stream);
    for (size_t k = 0; k < n; ++k) {
      if (cell_of_gid) cell_of_gid[gid[k]] = key[k];
      if (sorted_gid) sorted_gid[k] = gid[k];
    }
    return SPHG_OK;
  });
}

int sphg_cell_occupancy(sphg_ctx* h, int64_t* hist, size_t nbins, int64_t* max_count) {
  return guarded(h, [&]() -> int {
    Ctx& c = h->c;
    if (nbins == 0 || nbins > (1u << 20)) return fail(h, SPHG_ERR_CONFIG, "cell_occupancy: 1 <= nbins <= 2^20");
    if (!c.built) {
      const int rc = do_stage(h, SPHG_STAGE_REBUILD);
      if (rc) return rc;
    }
    DBuf<unsigned long long> d;
    d.alloc(nbins + 1);
    SPHG_CUDA_CHECK(cudaMemsetAsync(d.p, 0, (nbins + 1) * sizeof(unsigned long long), c.stream));
    uint32_t* dmax = reinterpret_cast<uint32_t*>(d.p + nbins);
    cell_occupancy(c, d.p, (uint32_t)nbins, dmax);
    std::vector<unsigned long long> out(nbins + 1);
    d2h(out.data(), d.p, nbins + 1, c.stream);
    host_sync(c, c.stream);
    for (size_t k = 0; k < nbins; ++k) hist[k] = (int64_t)out[k];
    if (max_count) {
      uint32_t mx;
      std::memcpy(&mx, &out[nbins], sizeof mx);
      *max_count = mx;
    }
    return SPHG_OK;
  });
}

int sphg_get_nlist(sphg_ctx* h, int64_t* offsets, uint32_t* nbr_gid) {
  return guarded(h, [&]() -> int {
    Ctx& c = h->c;
    if (!c.built) {
      const int rc = do_stage(h, SPHG_STAGE_REBUILD);
      if (rc) return rc;
    }
    const size_t n = c.n;
    std::vector<uint32_t> cnt(n), gid(n);
    d2h(cnt.data(), c.cnt.p, n, c.stream);
    d2h(gid.data(), c.cur.gid.p, n, c.stream);
    host_sync(c, c.stream);
    std::vector<int64_t> cnt_g(n);
    for (size_t k = 0; k < n; ++k) cnt_g[gid[k]] = cnt_total(cnt[k]);
    int64_t o = 0;
    for (size_t g = 0; g < n; ++g) {
      if (offsets) offsets[g] = o;
      o += cnt_g[g];
    }
    if (offsets) offsets[n] = o;
    if (!nbr_gid) return SPHG_OK;
    std::vector<uint32_t> rows((size_t)c.cap * n);
    d2h(rows.data(), c.nbr.p, rows.size(), c.stream);
    host_sync(c, c.stream);
    const uint32_t mask = c.P.img_mode == kImgCode ? kIdxMask : 0xffffffffu;
    for (size_t k = 0; k < n; ++k) {
      const int64_t base = offsets[gid[k]];
      const uint32_t* row = rows.data() + k * (size_t)c.cap;
      const uint32_t nf = cnt_fluid(cnt[k]), no = cnt_other(cnt[k]);
      for (uint32_t q = 0; q < nf + no; ++q) nbr_gid[base + q] = gid[row[q] & mask];
      std::sort(nbr_gid + base, nbr_gid + base + nf + no);
    }
    return SPHG_OK;
  });
}

int sphg_stats(sphg_ctx* h, sphg_stats_t* s) {
  return guarded(h, [&]() -> int {
    Ctx& c = h->c;
    std::memset(s, 0, sizeof(*s));
    s->steps = c.steps;
    s->rebuilds = c.rebuilds;
    s->transitions_melt = c.n_melt;
    s->transitions_solidify = c.n_solid;
    s->nlist_capacity = c.cap;
    s->max_neighbours = c.max_count;
    for (int a = 0; a < 3; ++a) s->cells[a] = c.P.ncell[a];
    s->time = c.t;
    s->max_displacement = c.max_disp;
    s->u_max = c.u_max;
    for (int k = 0; k < 16; ++k) s->stage_ms[k] = c.stage_ms[k];
    s->kernel_launches = c.launches;
    s->last_step_call_ms = c.last_step_ms;
    s->graph_captures = c.graph_captures;
    s->graph_replays = c.graph_replays;
    s->dt_violations = c.dt_violations;
    s->host_syncs = c.host_syncs;
    s->dt_term = c.dt_term;
    s->dt_limit = c.dt_limit;
    if (c.built && c.n) {
      std::vector<uint32_t> cnt(c.n);
      d2h(cnt.data(), c.cnt.p, c.n, c.stream);
      host_sync(c, c.stream);
      int64_t tot = 0;
      for (uint32_t v : cnt) tot += cnt_total(v);
      s->n_pairs_candidate = tot;
    }
    if (c.nb) {
      std::vector<sphg_body> b(c.nb);
      d2h(b.data(), c.bodies.p, c.nb, c.stream);
      host_sync(c, c.stream);
      for (auto& x : b) s->bodies_alive += x.alive ? 1 : 0;
    }
    return SPHG_OK;
  });
}

int sphg_set_timing(sphg_ctx* h, int enabled) {
  h->c.timing = enabled != 0;
  return SPHG_OK;
}

int sphg_dt_limits(const sphg_params* p, double u_max, double m_r, double lim[5]) {
  const double inf = std::numeric_limits<double>::infinity();
  for (int k = 0; k < 5; ++k) lim[k] = inf;
  const double hh = p->h > 0.0 ? p->h : p->dx;
  double bmax = 0.0;
  for (int m = 0; m < p->n_mat && m < SPHG_MAX_MAT; ++m) {
    const sphg_material& M = p->mat[m];
    if (M.c > 0.0) lim[0] = std::min(lim[0], 0.25 * hh / (M.c + u_max));  // CFL
    if (M.nu > 0.0) lim[1] = std::min(lim[1], 0.125 * hh * hh / M.nu);    // viscous
    const double b = std::sqrt(M.body_force[0] * M.body_force[0] + M.body_force[1] * M.body_force[1] +
                               M.body_force[2] * M.body_force[2]);
    bmax = std::max(bmax, b);
    if (M.kappa > 0.0 && M.cp > 0.0 && p->thermal)
      lim[4] = std::min(lim[4], 0.1 * M.rho0 * M.cp * hh * hh / M.kappa);  // conduction
  }
  if (bmax > 0.0) lim[2] = 0.25 * std::sqrt(hh / bmax);                    // body force
  if (p->kc > 0.0 && m_r > 0.0) lim[3] = 0.22 * std::sqrt(m_r / p->kc);    // contact
  return SPHG_OK;
}

int sphg_compute_dt(sphg_ctx* h, double lim[5]) {
  return guarded(h, [&]() -> int {
    Ctx& c = h->c;  // m_r: the smallest possible rigid particle mass, fixed at upload [P22]
    return sphg_dt_limits(&c.params, c.u_max, c.m_r, lim);
  });
}

int sphg_count_pairs(sphg_ctx* h, int64_t out[4]) {
  return guarded(h, [&]() -> int {
    Ctx& c = h->c;
    for (int k = 0; k < 4; ++k) out[k] = 0;
    if (c.n == 0) return SPHG_OK;
    if (!c.built) {
      const int rc = do_stage(h, SPHG_STAGE_REBUILD);
      if (rc) return rc;
    }
    count_pairs(c, out);
    return SPHG_OK;
  });
}

int sphg_shepard_grid(sphg_ctx* h, const double origin[3], const double spacing[3], const int32_t dims[3],
                      int32_t field, uint32_t kind_mask, double* out, uint8_t* support) {
  return guarded(h, [&]() -> int {
    Ctx& c = h->c;
    SPHG_CUDA_CHECK(cudaSetDevice(c.device));
    if (dims[0] < 0 || dims[1] < 0 || dims[2] < 0 || field < 0 || field > SPHG_FIELD_DENSITY)
      return fail(h, SPHG_ERR_CONFIG, "shepard_grid: bad dims or field");
    if (!c.have_state) return fail(h, SPHG_ERR_RUNTIME, "no particle state uploaded");
    const int64_t np = (int64_t)dims[0] * dims[1] * dims[2];
    const int nc = field == SPHG_FIELD_VELOCITY ? 3 : 1;
    if (np == 0) return SPHG_OK;
    if (c.n == 0) {  // nothing supports any point
      for (int64_t q = 0; q < np * nc; ++q) out[q] = std::numeric_limits<double>::quiet_NaN();
      if (support) std::memset(support, 0, (size_t)np);
      return SPHG_OK;
    }
    if (!c.built) {
      const int rc = do_stage(h, SPHG_STAGE_REBUILD);
      if (rc) return rc;
    }
    DBuf<double> dout;
    DBuf<uint8_t> dsup;
    dout.alloc((size_t)np * nc);
    if (support) dsup.alloc((size_t)np);
    shepard_grid(c, origin, spacing, dims, field, kind_mask, dout.p, support ? dsup.p : nullptr);
    SPHG_CUDA_CHECK(cudaMemcpyAsync(out, dout.p, (size_t)np * nc * sizeof(double), cudaMemcpyDefault, c.stream));
    if (support) SPHG_CUDA_CHECK(cudaMemcpyAsync(support, dsup.p, (size_t)np, cudaMemcpyDefault, c.stream));
    host_sync(c, c.stream);
    dout.free();
    dsup.free();
    return SPHG_OK;
  });
}

int sphg_halo_doubles(int phase) {
  return phase == SPHG_HALO_STATE ? 14 : phase == SPHG_HALO_DENSITY ? 4 : phase == SPHG_HALO_WALL ? 6 : -1;
}

int sphg_halo_set(sphg_ctx* h, int slot, const uint32_t* ids, size_t n) {
  return guarded(h, [&]() -> int {
    Ctx& c = h->c;
    if (slot < 0 || slot >= SPHG_MAX_HALO_SLOTS) return fail(h, SPHG_ERR_CONFIG, "halo slot out of range");
    for (size_t k = 0; k < n; ++k)
      if (ids[k] >= c.n) return fail(h, SPHG_ERR_CONFIG, "halo index out of range");
    c.halo_ids[slot].alloc(std::max<size_t>(n, 1));
    h2d(c.halo_ids[slot].p, ids, n, c.stream);
    host_sync(c, c.stream);
    c.halo_n[slot] = n;
    return SPHG_OK;
  });
}

int sphg_halo_pack(sphg_ctx* h, int phase, int slot, double* buf) {
  return guarded(h, [&]() -> int {
    Ctx& c = h->c;
    if (slot < 0 || slot >= SPHG_MAX_HALO_SLOTS || sphg_halo_doubles(phase) < 0)
      return fail(h, SPHG_ERR_CONFIG, "bad halo slot/phase");
    halo_pack(c, phase, slot, buf);
    host_sync(c, c.stream);
    return SPHG_OK;
  });
}

int sphg_halo_unpack(sphg_ctx* h, int phase, int slot, const double* buf) {
  return guarded(h, [&]() -> int {
    Ctx& c = h->c;
    if (slot < 0 || slot >= SPHG_MAX_HALO_SLOTS || sphg_halo_doubles(phase) < 0)
      return fail(h, SPHG_ERR_CONFIG, "bad halo slot/phase");
    halo_unpack(c, phase, slot, buf);
    host_sync(c, c.stream);
    return SPHG_OK;
  });
}

int sphg_body_partials(sphg_ctx* h, double* out) {
  return guarded(h, [&]() -> int {
    Ctx& c = h->c;
    if (c.nb == 0) return SPHG_OK;
    if (!c.built) {
      const int rc = do_stage(h, SPHG_STAGE_REBUILD);
      if (rc) return rc;
    }
    c.body_buf.alloc(c.nb * 24);
    SPHG_CUDA_CHECK(cudaMemsetAsync(c.body_buf.p, 0, c.nb * 24 * sizeof(double), c.stream));
    body_partials(c, c.body_buf.p);
    // host or device destination (the multi-rank driver gathers device tensors over NCCL)
    SPHG_CUDA_CHECK(cudaMemcpyAsync(out, c.body_buf.p, c.nb * 24 * sizeof(double), cudaMemcpyDefault, c.stream));
    host_sync(c, c.stream);
    return SPHG_OK;
  });
}

int sphg_body_apply_totals(sphg_ctx* h, const double* tot) {
  return guarded(h, [&]() -> int {
    Ctx& c = h->c;
    if (c.nb == 0) return SPHG_OK;
    c.body_buf.alloc(c.nb * 24);
    SPHG_CUDA_CHECK(cudaMemcpyAsync(c.body_buf.p, tot, c.nb * 12 * sizeof(double), cudaMemcpyDefault, c.stream));
    body_apply_totals(c, c.body_buf.p);
    host_sync(c, c.stream);
    return SPHG_OK;
  });
}

int sphg_max_displacement(sphg_ctx* h, double* out) {
  *out = h->c.max_disp;
  return SPHG_OK;
}

int sphg_set_exchange(sphg_ctx* h, sphg_exchange_fn fn, void* user) {
  h->c.exch_fn = fn;
  h->c.exch_user = user;
  return SPHG_OK;
}

int sphg_get_stream(sphg_ctx* h, void** stream) {
  *stream = reinterpret_cast<void*>(h->c.stream);
  return SPHG_OK;
}

int sphg_halo_bind(sphg_ctx* h, int phase, int slot, double* buf) {
  if (phase < 0 || phase > 2 || slot < 0 || slot >= SPHG_MAX_HALO_SLOTS)
    return fail(h, SPHG_ERR_CONFIG, "bad halo slot/phase");
  h->c.halo_buf[phase][slot] = buf;
  return SPHG_OK;
}

int sphg_max_bind(sphg_ctx* h, uint64_t* words) {
  h->c.max_words = words;
  return SPHG_OK;
}

int sphg_set_partition_limit(sphg_ctx* h, double limit) {
  h->c.partition_limit = limit;
  return SPHG_OK;
}

int sphg_counters(sphg_ctx* h, int64_t out[4]) {
  out[0] = h->c.steps;
  out[1] = h->c.rebuilds;
  out[2] = h->c.host_syncs;
  out[3] = h->c.launches;
  return SPHG_OK;
}

int sphg_drift(sphg_ctx* h, double out[3]) {
  out[0] = h->c.max_disp;
  out[1] = h->c.disp_since_partition;
  out[2] = h->c.u_max;
  return SPHG_OK;
}

int sphg_body_bind(sphg_ctx* h, double* part, double* gath, int32_t world) {
  if (world < 1) return fail(h, SPHG_ERR_CONFIG, "world size must be >= 1");
  h->c.body_part = part;
  h->c.body_gath = gath;
  h->c.world = world;
  return SPHG_OK;
}

int sphg_event_bodies(sphg_ctx* h, uint8_t* mask, size_t nb) {
  return guarded(h, [&]() -> int {
    Ctx& c = h->c;
    if (nb != c.nb) return fail(h, SPHG_ERR_CONFIG, "event_bodies: body count mismatch");
    if (nb == 0) return SPHG_OK;
    c.tscratch.alloc(nb);
    SPHG_CUDA_CHECK(cudaMemsetAsync(c.tscratch.p, 0, nb * sizeof(uint32_t), c.stream));
    event_bodies(c, c.tscratch.p);
    std::vector<uint32_t> m(nb);
    d2h(m.data(), c.tscratch.p, nb, c.stream);
    host_sync(c, c.stream);
    for (size_t k = 0; k < nb; ++k) mask[k] = (uint8_t)(mask[k] | (m[k] ? 1 : 0));
    return SPHG_OK;
  });
}

int sphg_event_members(sphg_ctx* h, const uint8_t* mask, size_t nb, uint32_t* ids, size_t cap, size_t* n) {
  return guarded(h, [&]() -> int {
    Ctx& c = h->c;
    if (nb != c.nb) return fail(h, SPHG_ERR_CONFIG, "event_members: body count mismatch");
    std::vector<uint32_t> m32(std::max<size_t>(nb, 1), 0u);
    for (size_t k = 0; k < nb; ++k) m32[k] = mask[k] ? 1u : 0u;
    c.tscratch.alloc(m32.size());
    h2d(c.tscratch.p, m32.data(), m32.size(), c.stream);
    c.rec_ids.alloc(std::max<size_t>(c.n, 1));
    const size_t m = event_members(c, c.tscratch.p, nb, c.rec_ids.p);
    *n = m;
    if (!ids) return SPHG_OK;
    if (cap < m) return fail(h, SPHG_ERR_CONFIG, "event_members: buffer too small");
    d2h(ids, c.rec_ids.p, m, c.stream);
    host_sync(c, c.stream);
    std::sort(ids, ids + m);
    return SPHG_OK;
  });
}

int sphg_record_doubles(void) { return kRecordDoubles; }

int sphg_record_pack(sphg_ctx* h, const uint32_t* ids, size_t m, double* recs) {
  return guarded(h, [&]() -> int {
    Ctx& c = h->c;
    if (!is_device_ptr(ids))
      for (size_t s = 0; s < m; ++s)
        if (ids[s] >= c.n) return fail(h, SPHG_ERR_CONFIG, "record_pack: id out of range");
    if (m == 0) return SPHG_OK;
    c.rec_ids.alloc(m);
    c.rec_buf.alloc(m * kRecordDoubles);
    // host or device buffers (unified addressing: the multi-rank driver keeps records on the device)
    SPHG_CUDA_CHECK(cudaMemcpyAsync(c.rec_ids.p, ids, m * sizeof(uint32_t), cudaMemcpyDefault, c.stream));
    if (record_pack(c, c.rec_ids.p, m, c.rec_buf.p) != 0xffffffffu)
      return fail(h, SPHG_ERR_CONFIG, "record_pack: id out of range");
    SPHG_CUDA_CHECK(cudaMemcpyAsync(recs, c.rec_buf.p, m * kRecordDoubles * sizeof(double), cudaMemcpyDefault,
                                    c.stream));
    host_sync(c, c.stream);
    return SPHG_OK;
  });
}

int sphg_record_unpack(sphg_ctx* h, const uint32_t* ids, size_t m, const double* recs, int keep_position) {
  return guarded(h, [&]() -> int {
    Ctx& c = h->c;
    if (!is_device_ptr(ids) && !is_device_ptr(recs))
      for (size_t s = 0; s < m; ++s) {
        if (ids[s] >= c.n) return fail(h, SPHG_ERR_CONFIG, "record_unpack: id out of range");
        const double* o = recs + s * kRecordDoubles;
        if (!(o[3] >= 0.0 && o[3] <= 2.0) || !(o[4] >= 0.0 && o[4] < c.params.n_mat))
          return fail(h, SPHG_ERR_CONFIG, "record_unpack: invalid kind/material");
      }
    if (m == 0) return SPHG_OK;
    c.rec_ids.alloc(m);
    c.rec_buf.alloc(m * kRecordDoubles);
    SPHG_CUDA_CHECK(cudaMemcpyAsync(c.rec_ids.p, ids, m * sizeof(uint32_t), cudaMemcpyDefault, c.stream));
    SPHG_CUDA_CHECK(cudaMemcpyAsync(c.rec_buf.p, recs, m * kRecordDoubles * sizeof(double), cudaMemcpyDefault,
                                    c.stream));
    if (record_unpack(c, c.rec_ids.p, m, c.rec_buf.p, keep_position) != 0xffffffffu)
      return fail(h, SPHG_ERR_CONFIG, "record_unpack: id out of range");
    host_sync(c, c.stream);
    return SPHG_OK;
  });
}

int sphg_upload_records(sphg_ctx* h, size_t n, size_t n_owned, const double* recs, const sphg_body* bodies,
                        size_t nb) {
  return guarded(h, [&]() -> int {
    Ctx& c = h->c;
    SPHG_CUDA_CHECK(cudaSetDevice(c.device));
    if (n >= (size_t)UINT32_MAX) return fail(h, SPHG_ERR_CONFIG, "too many particles for 32-bit gids");
    if (n_owned > n) return fail(h, SPHG_ERR_CONFIG, "upload_records: n_owned > n");
    host_sync(c, c.stream);
    // records on the device and validated before anything of the context changes
    const double* dr = recs;
    if (!is_device_ptr(recs) && n) {
      c.rec_buf.alloc(n * kRecordDoubles);
      SPHG_CUDA_CHECK(cudaMemcpyAsync(c.rec_buf.p, recs, n * kRecordDoubles * sizeof(double), cudaMemcpyDefault,
                                      c.stream));
      dr = c.rec_buf.p;
    }
    const uint32_t bad = record_check(c, dr, n, nb);
    if (bad != 0xffffffffu)
      return fail(h, SPHG_ERR_CONFIG, "upload_records: record " + std::to_string(bad) +
                                          " has an invalid kind / material / body id");
    destroy_graphs(c);
    c.nghost = n - n_owned;
    c.disp_since_partition = 0.0;
    alloc_store(c, n);
    c.built = false;
    c.final_pending = false;
    iota_gid(c);
    build_idx_of_gid(c);
    record_load(c, dr, n, n_owned);
    c.nb = 0;
    ensure_bodies(c, nb);
    c.nb = nb;
    if (nb) SPHG_CUDA_CHECK(cudaMemcpyAsync(c.bodies.p, bodies, nb * sizeof(sphg_body), cudaMemcpyDefault, c.stream));
    SPHG_CUDA_CHECK(cudaMemsetAsync(c.dflags, 0, sizeof(DevFlags), c.stream));
    SPHG_CUDA_CHECK(cudaMemsetAsync(&c.dflags->err_gid, 0xff, 2 * sizeof(uint32_t), c.stream));
    host_sync(c, c.stream);
    c.have_state = true;
    h->mid_step = false;
    return SPHG_OK;
  });
}

int sphg_replace_bodies(sphg_ctx* h, const sphg_body* bodies, size_t nb) {
  return guarded(h, [&]() -> int {
    Ctx& c = h->c;
    destroy_graphs(c);
    ensure_bodies(c, nb);
    c.nb = nb;
    h2d(c.bodies.p, bodies, nb, c.stream);
    if (c.built) {  // kinds / groups changed under the rows
      launch_rigid_index(c);
      launch_repartition_rows(c);
      if (c.built) launch_contact_order(c);
      launch_ghost_split(c);
    }
    host_sync(c, c.stream);
    return check_flags(h, true);
  });
}

int sphg_set_event_log(sphg_ctx* h, int enabled) {
  h->c.event_log = enabled != 0;
  return SPHG_OK;
}

int sphg_transition_events(sphg_ctx* h, sphg_event* out, size_t cap, size_t* n) {
  Ctx& c = h->c;
  if (!out) {
    *n = c.events.size();
    return SPHG_OK;
  }
  const size_t m = std::min(cap, c.events.size());
  std::copy(c.events.begin(), c.events.begin() + m, out);
  c.events.erase(c.events.begin(), c.events.begin() + m);
  *n = m;
  return SPHG_OK;
}

const char* sphg_last_error(const sphg_ctx* h) { return h ? h->c.err.c_str() : "null context"; }

void sphg_destroy(sphg_ctx* h) {
  if (!h) return;
  Ctx& c = h->c;
  cudaSetDevice(c.device);
  if (c.stream) cudaStreamSynchronize(c.stream);
  destroy_graphs(c);
  if (c.dtime) cudaFree(c.dtime);
  if (c.htime) cudaFreeHost(c.htime);
  c.cur.free(); c.alt.free(); c.H2new.free(); c.C2new.free(); c.hsrc.free(); c.pin_list.free();
  if (c.pin_any) cudaFree(c.pin_any); c.bodies.free();
  if (c.copy_stream) cudaStreamDestroy(c.copy_stream);
  if (c.dskip) cudaFree(c.dskip);
  if (c.kick_ev) cudaEventDestroy(c.kick_ev);
  if (c.side_stream) cudaStreamDestroy(c.side_stream);
  if (c.fork_ev) cudaEventDestroy(c.fork_ev);
  if (c.join_ev) cudaEventDestroy(c.join_ev);
  if (c.dl_ev) cudaEventDestroy(c.dl_ev);
  if (c.dens_stream) cudaStreamDestroy(c.dens_stream);
  if (c.dens_fork) cudaEventDestroy(c.dens_fork);
  if (c.dens_join) cudaEventDestroy(c.dens_join);
  c.body_tot.free();
  c.keys.free(); c.keys_alt.free(); c.vals.free(); c.vals_alt.free(); c.hist.free(); c.scan_tmp.free();
  c.cell_start.free(); c.cell_end.free(); c.cell_key.free(); c.nbr.free(); c.cnt.free(); c.sm_next.free();
  c.ridx.free(); c.body_start.free(); c.ev_idx.free(); c.ev_flag.free(); c.label.free(); c.tscratch.free();
  c.label_list.free(); c.label_flags.free(); c.ev_log.free(); c.ev_count.free();
  c.rec_ids.free(); c.rec_buf.free(); c.group0.free(); c.bodies_old.free(); c.wrap_list.free(); c.state_buf.free();
  c.label_adj.free();
  c.fidx.free(); c.widx.free(); c.ncon.free(); c.brick_buf.free(); c.scan_cells.free(); c.dl_buf.free(); c.idx_of_gid.free(); c.body_buf.free();
  for (auto& b : c.halo_ids) b.free();
  if (c.dflags) cudaFree(c.dflags);
  if (c.hflags) cudaFreeHost(c.hflags);
  if (c.hbodies) cudaFreeHost(c.hbodies);
  if (c.hstage) cudaFreeHost(c.hstage);
  for (auto& e : c.slot_ev) if (e) cudaEventDestroy(e);
  if (c.dcount) cudaFree(c.dcount);
  for (auto& e : c.step_ev) if (e) cudaEventDestroy(e);
  for (auto& e : c.ev) if (e) cudaEventDestroy(e);
  if (c.stream) cudaStreamDestroy(c.stream);
  delete h;
}

size_t sphg_sizeof_params(void) { return sizeof(sphg_params); }
size_t sphg_sizeof_body(void) { return sizeof(sphg_body); }
size_t sphg_sizeof_soa(void) { return sizeof(sphg_soa); }

}  // extern "C"
