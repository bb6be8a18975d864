// sph_oracle.cpp — CPU ORACLE FOR THE SPH HOT PATH.  TEST INFRASTRUCTURE ONLY.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg may load this library, and only as the checker / the timed CPU
// baseline.  The product path (paper_2103_07925_b200) never calls it.
//
// What it is: a plain, sequential-per-particle restatement of the reference's
// hot path (arXiv 2103.07925 §3; /root/reference/SPEC.md modules
// decomposition/fluid/rigid/thermal/transition/integrator) written ON TOP OF
// the reference's own header building blocks, which are compiled in from
// /root/reference/proj/include (see oracle/Makefile):
//   sphfsi::QuinticKernel<3>      kernel.hpp:15-81     (w, dw_dr, sigma)
//   sphfsi::eos_pressure/density  material.hpp:59-68
//   sphfsi::Material::dynamic_viscosity material.hpp:32
//   sphfsi::KahanSum / KahanVec   kahan.hpp:9-36       (body reductions)
//   sphfsi::Quaternion, quat_exp, rotate, orientation_step  quaternion.hpp:10-76
//   sphfsi::cross / moment        vec.hpp:84-106
//   sphfsi::ParticleStore<3>      store.hpp:24-100     (the state container)
//   sphfsi::validate_config       config.hpp:110-167
//   sphfsi::seed_lattice          lattice.hpp:71-82    (exported for pinning the generator)
// The reference leaves several details open; every pin is listed in DESIGN.md §2
// ("pins") and cited inline as [Pn].  OpenMP parallelises over particles only;
// every per-particle sum is sequential in gid order, so results do not depend
// on the thread count.  Compile with -ffp-contract=off (no FMA contraction).
//
// Exported C ABI: the entry points of include/sphg.h with prefix orc_, plus KAT
// helpers (orc_kernel_w, orc_seed_lattice_box, ...).

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <limits>
#include <numeric>
#include <string>
#include <vector>

#include "sphfsi/config.hpp"
#include "sphfsi/kahan.hpp"
#include "sphfsi/kernel.hpp"
#include "sphfsi/lattice.hpp"
#include "sphfsi/material.hpp"
#include "sphfsi/quaternion.hpp"
#include "sphfsi/store.hpp"
#include "sphfsi/vec.hpp"

#include "../include/sphg.h"

using sphfsi::Kind;
using V3 = sphfsi::Vec<3>;

namespace {

constexpr double kNaN = std::numeric_limits<double>::quiet_NaN();

struct Ctx {
    sphg_params P{};
    sphfsi::MaterialTable mats;
    sphfsi::ParticleStore<3> S;
    std::vector<V3> force;          // f_r on rigid particles
    std::vector<double> rho_w, V_w; // wall/rigid interaction density & volume [P7]
    std::vector<int> wall_mat;      // EOS material used for the wall [P7]
    std::vector<V3> pos_ref;        // positions at the last rebuild (Verlet)
    std::vector<sphg_body> bodies;
    std::vector<std::vector<uint32_t>> members; // rigid particles of each body, gid order
    std::vector<std::vector<uint32_t>> nl;      // Verlet candidates, gid-sorted
    std::vector<std::vector<uint32_t>> halo;    // halo index lists (local ids) per slot
    std::vector<int64_t> cell_of;
    std::vector<uint32_t> sorted;
    // tolerance scales (sum of |pair contributions|)
    std::vector<double> acc_scale, accbg_scale, dT_scale, force_scale, rho_scale, dC_scale;
    // pressure sensitivity of acc (fluid) / f_r (rigid): sum over pairs of |d term / d p| x c^2 rho, the
    // EOS-level magnitude behind each pressure (p = c^2 (rho - rho0) cancels): an absolute allowance of a
    // few ulp of it covers the last-bit density differences any reordered density sum makes
    std::vector<double> acc_pscale, force_pscale;
    std::vector<double> body_fscale, body_tscale;
    double t = 0.0;
    int64_t steps = 0, rebuilds = 0, n_melt = 0, n_solid = 0;
    int ncell[3] = {1, 1, 1};
    double inv_edge[3] = {0, 0, 0}, L[3] = {0, 0, 0}, halfL[3] = {0, 0, 0};
    double h = 0, rc = 0, rv = 0, dt = 0;
    double max_disp = 0, u_max = 0;
    bool built = false;
    // moving wall groups (sphg_set_wall_motion): callback + per-step values
    int n_walls = 0;
    sphg_wall_motion_fn wall_fn = nullptr;
    void* wall_user = nullptr;
    double wall_vh[SPHG_MAX_WALL_GROUPS][3] = {}, wall_v[SPHG_MAX_WALL_GROUPS][3] = {},
           wall_a[SPHG_MAX_WALL_GROUPS][3] = {};
    std::string err;
    int threads = 0;
    // runtime time-step assertion [P22]
    double m_r = 0.0;              // smallest mass a rigid particle can have in this run (0: none)
    int64_t dt_violations = 0;
    // transition event log (sphg_set_event_log)
    bool event_log = false;
    std::vector<sphg_event> events;
    // in-library decomposed step (sphg.h): exchange callback + bound host buffers
    sphg_exchange_fn exch_fn = nullptr;
    void* exch_user = nullptr;
    double* halo_buf[3][SPHG_MAX_HALO_SLOTS] = {};
    uint64_t* max_words = nullptr;
    double* body_part = nullptr;
    double* body_gath = nullptr;
    int world = 1;
    bool has_ghosts = false;
    std::vector<uint8_t> ev;        // events of the last decomposed detection (1 melt, 2 solidify)
    double disp_since_partition = 0.0;
    double partition_limit = 0.0;
    int dt_term = -1;
    double dt_limit = std::numeric_limits<double>::infinity();
};

inline bool ghost(const Ctx& c, size_t i) { return c.S.owner[i] != (uint32_t)c.P.rank; }

// WallGroup::velocity_at / acceleration_at (config.hpp:42-50) through the host callback [P20]
void eval_walls(Ctx& c, double t, double (*vel)[3], double (*acc)[3]) {
    for (int g = 0; g < c.n_walls; ++g) {
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
inline bool wall_member(const Ctx& c, size_t i) {
    return c.n_walls > 0 && c.S.kind[i] == Kind::Boundary && c.S.group[i] < (uint32_t)c.n_walls;
}


inline double mi(const Ctx& c, double d, int a) {  // minimum image [P2]
    if (c.P.periodic[a]) {
        if (d > c.halfL[a]) d -= c.L[a];
        else if (d < -c.halfL[a]) d += c.L[a];
    }
    return d;
}
inline V3 mi3(const Ctx& c, const V3& a, const V3& b) {
    return V3{mi(c, a[0] - b[0], 0), mi(c, a[1] - b[1], 1), mi(c, a[2] - b[2], 2)};
}
inline double r2of(const V3& d) { return (d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]; }  // [P2]
inline double wrap1(const Ctx& c, double x, int a) {  // [P14]
    if (c.P.periodic[a]) {
        if (x < c.P.lo[a]) x += c.L[a];
        else if (x >= c.P.hi[a]) x -= c.L[a];
    }
    return x;
}
inline V3 wrap3(const Ctx& c, V3 x) {
    for (int a = 0; a < 3; ++a) x[a] = wrap1(c, x[a], a);
    return x;
}
inline sphfsi::Quaternion qof(const sphg_body& b) { return {b.q[0], b.q[1], b.q[2], b.q[3]}; }
inline V3 v3(const double* p) { return V3{p[0], p[1], p[2]}; }
inline void put3(double* p, const V3& v) { p[0] = v[0]; p[1] = v[1]; p[2] = v[2]; }

sphfsi::ScenarioConfig<3> to_config(const sphg_params& P) {
    sphfsi::ScenarioConfig<3> cfg;
    cfg.dx = P.dx;
    cfg.smoothing_length = P.h;
    for (int a = 0; a < 3; ++a) {
        cfg.domain.lo[a] = P.lo[a];
        cfg.domain.hi[a] = P.hi[a];
        cfg.periodic[a] = P.periodic[a] != 0;
    }
    cfg.cell_edge_override = P.cell_edge_override;
    for (int m = 0; m < P.n_mat && m < SPHG_MAX_MAT; ++m) {
        sphfsi::Material mt;
        mt.name = "m" + std::to_string(m);
        mt.reference_density = P.mat[m].rho0;
        mt.kinematic_viscosity = P.mat[m].nu;
        mt.heat_capacity = P.mat[m].cp;
        mt.conductivity = P.mat[m].kappa;
        mt.speed_of_sound = P.mat[m].c;
        mt.background_pressure = P.mat[m].pb;
        mt.transition_temperature = P.mat[m].T_t;
        mt.diffusivity = P.mat[m].D;
        mt.transition_concentration = P.mat[m].C_t;
        mt.melt_target = P.mat[m].melt_target < 0 ? sphfsi::kNoMaterial : (sphfsi::MaterialId)P.mat[m].melt_target;
        mt.solidify_target =
            P.mat[m].solidify_target < 0 ? sphfsi::kNoMaterial : (sphfsi::MaterialId)P.mat[m].solidify_target;
        cfg.materials.add(mt);
        cfg.body_force.push_back(V3{P.mat[m].body_force[0], P.mat[m].body_force[1], P.mat[m].body_force[2]});
    }
    cfg.contact_stiffness = P.kc;
    cfg.contact_damping = P.dc;
    cfg.dt_override = P.dt;
    cfg.workers = P.nranks > 0 ? P.nranks : 1;
    cfg.transport_velocity = P.tvf != 0;
    for (int g = 0; g < P.n_dirichlet && g < SPHG_MAX_DIRICHLET; ++g) {
        sphfsi::Schedule s;
        for (int k = 0; k < P.dirichlet_T[g].n && k < SPHG_MAX_PIECES; ++k)
            s.pieces.push_back({P.dirichlet_T[g].t_end[k], P.dirichlet_T[g].value[k]});
        cfg.dirichlet_temperature.push_back(s);
    }
    for (int g = 0; g < P.n_dirichlet_c && g < SPHG_MAX_DIRICHLET; ++g) {
        sphfsi::Schedule s;
        for (int k = 0; k < P.dirichlet_C[g].n && k < SPHG_MAX_PIECES; ++k)
            s.pieces.push_back({P.dirichlet_C[g].t_end[k], P.dirichlet_C[g].value[k]});
        cfg.dirichlet_concentration.push_back(s);
    }
    cfg.transition_mode = P.transitions == 2   ? sphfsi::TransitionMode::Concentration
                          : P.transitions == 1 ? sphfsi::TransitionMode::Temperature
                                               : sphfsi::TransitionMode::None;
    return cfg;
}

std::vector<std::string> validate(const sphg_params& P) {
    std::vector<std::string> v;
    if (P.n_mat < 0 || P.n_mat > SPHG_MAX_MAT) {
        v.push_back("material count out of range");
        return v;
    }
    v = sphfsi::validate_config(to_config(P));
    if (!(P.dt > 0.0)) v.push_back("time step dt must be positive");
    const double h = P.h > 0.0 ? P.h : P.dx;
    const double rv = sphfsi::kKernelSupportScale * h + sphfsi::kVerletSkinFactor * h;
    for (int a = 0; a < 3; ++a) {
        const double ext = P.hi[a] - P.lo[a];
        const double e0 = P.cell_edge_override > 0.0 ? P.cell_edge_override : rv;
        if (P.periodic[a] && ext > 0.0 && std::floor(ext / e0) < 3.0)
            v.push_back("periodic axis " + std::to_string(a) + " has fewer than 3 cells");
    }
    if (P.n_dirichlet < 0 || P.n_dirichlet > SPHG_MAX_DIRICHLET) v.push_back("dirichlet group count out of range");
    if (P.n_dirichlet_c < 0 || P.n_dirichlet_c > SPHG_MAX_DIRICHLET)
        v.push_back("concentration dirichlet group count out of range");
    if (P.transitions < 0 || P.transitions > 2) v.push_back("unknown transition mode");
    if (P.transitions == 2 && !P.diffusion) v.push_back("concentration transitions need the diffusion equation");
    if (P.default_fluid_mat < 0 || P.default_fluid_mat >= P.n_mat) v.push_back("default fluid material missing");
    if (P.n_buffers < 0 || P.n_buffers > SPHG_MAX_BUFFERS) v.push_back("buffer zone count out of range");
    for (int b = 0; b < P.n_buffers && b < SPHG_MAX_BUFFERS; ++b) {  // [P23]
        const sphg_buffer& B = P.buffers[b];
        if (B.axis < 0 || B.axis > 2 || B.profile_axis < -1 || B.profile_axis > 2 || B.profile_axis == B.axis)
            v.push_back("buffer zone axes invalid");
        for (int a = 0; a < 3; ++a)
            if (!(B.hi[a] > B.lo[a])) v.push_back("buffer zone box is empty");
    }
    if (P.heat_source) {  // [P21]
        if (!P.thermal) v.push_back("heat source needs the heat equation");
        if (!(P.hs_radius > 0.0)) v.push_back("heat source radius must be positive");
    }
    return v;
}

void setup_geometry(Ctx& c) {
    c.h = c.P.h > 0.0 ? c.P.h : c.P.dx;
    c.rc = sphfsi::kKernelSupportScale * c.h;
    c.rv = c.rc + sphfsi::kVerletSkinFactor * c.h;
    c.dt = c.P.dt;
    for (int a = 0; a < 3; ++a) {
        c.L[a] = c.P.hi[a] - c.P.lo[a];
        c.halfL[a] = 0.5 * c.L[a];
        const double e0 = c.P.cell_edge_override > 0.0 ? c.P.cell_edge_override : c.rv;  // [P1]
        int n = (int)std::floor(c.L[a] / e0);
        if (n < 1) n = 1;
        c.ncell[a] = n;
        c.inv_edge[a] = (double)n / c.L[a];
    }
}

bool fail(Ctx& c, const std::string& m) {
    c.err = m;
    return false;
}

// ---------------------------------------------------------------- rebuild
// DomainGrid binning, build_pairs with Verlet skin.
bool stage_rebuild(Ctx& c) {
    const size_t n = c.S.size();
    c.cell_of.assign(n, 0);
    for (size_t i = 0; i < n; ++i) {
        int64_t ci[3];
        for (int a = 0; a < 3; ++a) {
            const double x = c.S.pos[i][a];
            if (!c.P.periodic[a] && (x < c.P.lo[a] || x > c.P.hi[a]))
                return fail(c, "escaped particle " + std::to_string(i) + " at step " + std::to_string(c.steps));
            int64_t k = (int64_t)std::floor((x - c.P.lo[a]) * c.inv_edge[a]);  // [P1]
            if (k < 0) k = 0;
            if (k >= c.ncell[a]) k = c.ncell[a] - 1;
            ci[a] = k;
        }
        c.cell_of[i] = (ci[0] * c.ncell[1] + ci[1]) * c.ncell[2] + ci[2];
    }
    const int64_t ncells = (int64_t)c.ncell[0] * c.ncell[1] * c.ncell[2];
    std::vector<int64_t> start(ncells + 1, 0);
    for (size_t i = 0; i < n; ++i) start[c.cell_of[i] + 1]++;
    for (int64_t k = 0; k < ncells; ++k) start[k + 1] += start[k];
    c.sorted.assign(n, 0);
    {
        std::vector<int64_t> fill(start.begin(), start.end() - 1);
        for (size_t i = 0; i < n; ++i) c.sorted[fill[c.cell_of[i]]++] = (uint32_t)i;  // (cell, gid) order [P1]
    }
    c.nl.assign(n, {});
    const double rv2 = c.rv * c.rv;
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t ii = 0; ii < (int64_t)n; ++ii) {
        const size_t i = (size_t)ii;
        if (ghost(c, i)) continue;  // ghosts are read, never evaluated here
        const int64_t cid = c.cell_of[i];
        const int64_t cz = cid % c.ncell[2], cy = (cid / c.ncell[2]) % c.ncell[1], cx = cid / ((int64_t)c.ncell[2] * c.ncell[1]);
        auto& out = c.nl[i];
        for (int ox = -1; ox <= 1; ++ox)
            for (int oy = -1; oy <= 1; ++oy)
                for (int oz = -1; oz <= 1; ++oz) {
                    int64_t q[3] = {cx + ox, cy + oy, cz + oz};
                    bool skip = false;
                    for (int a = 0; a < 3; ++a) {
                        if (q[a] < 0 || q[a] >= c.ncell[a]) {
                            if (!c.P.periodic[a]) { skip = true; break; }
                            q[a] = (q[a] + c.ncell[a]) % c.ncell[a];
                        }
                    }
                    if (skip) continue;
                    const int64_t cj = (q[0] * c.ncell[1] + q[1]) * c.ncell[2] + q[2];
                    for (int64_t s = start[cj]; s < start[cj + 1]; ++s) {
                        const uint32_t j = c.sorted[s];
                        if (j == i) continue;
                        if (c.S.kind[i] == Kind::Boundary && c.S.kind[j] == Kind::Boundary) continue;  // [P2]
                        const V3 d = mi3(c, c.S.pos[i], c.S.pos[j]);
                        if (r2of(d) <= rv2) out.push_back(j);  // inclusive
                    }
                }
        std::sort(out.begin(), out.end());
    }
    c.pos_ref = c.S.pos;
    c.max_disp = 0.0;
    c.built = true;
    c.rebuilds++;
    return true;
}

// -------------------------------------------------------------- density
// density_summation + eos_pressure (material.hpp:59-62)
bool stage_density(Ctx& c) {
    const sphfsi::QuinticKernel<3> K(c.h);
    const double rc2 = c.rc * c.rc;
    const int64_t n = (int64_t)c.S.size();
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        if (c.S.kind[i] != Kind::Fluid || ghost(c, (size_t)i)) continue;
        double s = K.w(0.0);  // self term first
        for (uint32_t j : c.nl[i]) {
            const V3 d = mi3(c, c.S.pos[i], c.S.pos[j]);
            const double r2 = r2of(d);
            if (r2 > rc2) continue;
            s += K.w(std::sqrt(r2));
        }
        const double rho = c.S.mass[i] * s;
        c.S.density[i] = rho;
        c.S.pressure[i] = sphfsi::eos_pressure(rho, c.mats[c.S.material[i]]);
        c.rho_scale[i] = rho;
    }
    return true;
}

// ------------------------------------------------------------------ heat
double sched_value(const sphg_schedule& s, double t) {  // Schedule::value_at (config.hpp:28-32)
    sphfsi::Schedule sc;
    for (int k = 0; k < s.n; ++k) sc.pieces.push_back({s.t_end[k], s.value[k]});
    return sc.value_at(t);
}

// Moving Gaussian surface heat flux [P21] (BASELINE C4; not in the reference, which has no heat
// sources: PAPER:118).  Source rate q(x_a, y_a, t) dx^2 / (m_a c_p,a) of particle a at
// time t (sphg.h documents the exposure rule); 0 when a does not absorb.
inline bool hs_absorbs(const Ctx& c, size_t i) {
    return (c.P.hs_material_mask >> c.S.material[i]) & 1u;
}
double heat_source_rate(const Ctx& c, size_t a, double t) {
    if (!c.P.heat_source || c.S.kind[a] == Kind::Boundary || !hs_absorbs(c, a)) return 0.0;
    const sphfsi::Material& ma = c.mats[c.S.material[a]];
    if (!(ma.heat_capacity > 0.0)) return 0.0;
    double rho2 = 0.0;
    for (int ax = 0; ax < 2; ++ax) {
        double cx = c.P.hs_origin[ax] + c.P.hs_velocity[ax] * t;
        cx = c.P.periodic[ax] ? c.P.lo[ax] + (cx - c.P.lo[ax]) - c.L[ax] * std::floor((cx - c.P.lo[ax]) / c.L[ax]) : cx;
        const double d = mi(c, c.S.pos[a][ax] - cx, ax);
        rho2 += d * d;
    }
    const double r0 = c.P.hs_radius;
    if (rho2 > 16.0 * r0 * r0) return 0.0;  // truncated at 4 r0
    const double rc2 = c.rc * c.rc, dz = 0.5 * c.P.dx, lat2 = 0.5625 * c.P.dx * c.P.dx;
    for (uint32_t b : c.nl[a]) {  // shadowed by a mask particle above a (any kind)
        if (!hs_absorbs(c, b)) continue;
        const V3 d = mi3(c, c.S.pos[a], c.S.pos[b]);  // r_a - r_b
        if (r2of(d) > rc2) continue;
        if (-d[2] > dz && d[0] * d[0] + d[1] * d[1] < lat2) return 0.0;
    }
    const double q = 2.0 * c.P.hs_power / (M_PI * r0 * r0) * std::exp(-2.0 * rho2 / (r0 * r0));
    return q * (c.P.dx * c.P.dx) / (c.S.mass[a] * ma.heat_capacity);
}

// apply_thermal_dirichlet at t^{n+1} [P9]; conduction_rhs (SPEC:398-406,
// PAPER:399-405) with T^n, r^{n+1}, rho^{n+1}; T^{n+1} = T^n + dt rate;
// + the surface heat flux at t^{n+1} [P21].
bool stage_heat(Ctx& c) {
    const size_t n = c.S.size();
    const double t_new = c.t + c.dt;
    for (size_t i = 0; i < n; ++i) {
        if (c.S.kind[i] == Kind::Boundary && c.S.dirichlet_T[i] != sphfsi::kNoDirichlet) {
            const int g = c.S.dirichlet_T[i];
            if (g < c.P.n_dirichlet && c.P.dirichlet_T[g].n > 0) c.S.temperature[i] = sched_value(c.P.dirichlet_T[g], t_new);
        }
    }
    const std::vector<double> Tn = c.S.temperature;  // double buffer [P9]
    const sphfsi::QuinticKernel<3> K(c.h);
    const double rc2 = c.rc * c.rc;
    bool coincident = false;
    size_t bad_i = 0, bad_j = 0;
#pragma omp parallel for schedule(static)
    for (int64_t ii = 0; ii < (int64_t)n; ++ii) {
        const size_t a = (size_t)ii;
        if (c.S.kind[a] == Kind::Boundary || ghost(c, a)) continue;
        const sphfsi::Material& ma = c.mats[c.S.material[a]];
        double s = 0.0, sc = 0.0;
        for (uint32_t b : c.nl[a]) {
            const bool bd = c.S.kind[b] == Kind::Boundary;
            if (bd && c.S.dirichlet_T[b] == sphfsi::kNoDirichlet) continue;
            const V3 d = mi3(c, c.S.pos[a], c.S.pos[b]);
            const double r2 = r2of(d);
            if (r2 > rc2) continue;
            const double r = std::sqrt(r2);
            if (r == 0.0) {
#pragma omp critical
                { coincident = true; bad_i = a; bad_j = b; }
                continue;
            }
            const sphfsi::Material& mb = c.mats[c.S.material[b]];
            const double ksum = ma.conductivity + mb.conductivity;
            if (ksum == 0.0) continue;
            const double kt = 4.0 * ma.conductivity * mb.conductivity / ksum;
            const double rho_b = bd ? mb.reference_density : c.S.density[b];  // [P9]
            const double Vb = c.S.mass[b] / rho_b;
            const double term = Vb * kt * ((Tn[a] - Tn[b]) / r) * K.dw_dr(r);
            s += term;
            sc += std::abs(term);
        }
        double rate = 0.0, scale = 0.0;
        if (ma.heat_capacity > 0.0) {
            const double den = c.S.density[a] * ma.heat_capacity;
            rate = s / den;
            scale = sc / den;
            if (c.P.heat_source) {
                const double q = heat_source_rate(c, a, t_new);
                rate += q;
                scale += std::abs(q);
            }
        }
        c.S.dT_dt[a] = rate;
        c.S.temperature[a] = Tn[a] + c.dt * rate;
        c.dT_scale[a] = scale;
    }
    if (coincident)
        return fail(c, "coincident particles " + std::to_string(bad_i) + " and " + std::to_string(bad_j) +
                           " at step " + std::to_string(c.steps));
    return true;
}

// ------------------------------------------------------------- diffusion
// Concentration analogue of the heat stage (Remark 2.3 PAPER:141):
// dC_a/dt = (1/rho_a) sum_b V_b 4 D_a D_b/(D_a+D_b) (C_ab/r_ab) dW/dr, no capacity factor.
// [P18] Dirichlet concentration groups (config.hpp:95) apply to every particle carrying a
// group (the paper's fixed-concentration gastric juice is a fluid), set at t^{n+1}
// before the rates; such particles keep C = C^ (their rate is still reported).  Boundary walls
// take part only with a group (as for heat); V_b = m/rho (fluid), m/rho0 otherwise.
bool stage_diffusion(Ctx& c) {
    const size_t n = c.S.size();
    const double t_new = c.t + c.dt;
    auto dir_group = [&](size_t i) -> int {
        const int g = c.S.dirichlet_C[i];
        return (g != sphfsi::kNoDirichlet && g < c.P.n_dirichlet_c && c.P.dirichlet_C[g].n > 0) ? g : -1;
    };
    for (size_t i = 0; i < n; ++i) {
        const int g = dir_group(i);
        if (g >= 0) c.S.concentration[i] = sched_value(c.P.dirichlet_C[g], t_new);
    }
    const std::vector<double> Cn = c.S.concentration;  // double buffer
    const sphfsi::QuinticKernel<3> K(c.h);
    const double rc2 = c.rc * c.rc;
    bool coincident = false;
    size_t bad_i = 0, bad_j = 0;
#pragma omp parallel for schedule(static)
    for (int64_t ii = 0; ii < (int64_t)n; ++ii) {
        const size_t a = (size_t)ii;
        if (c.S.kind[a] == Kind::Boundary || ghost(c, a)) continue;
        const sphfsi::Material& ma = c.mats[c.S.material[a]];
        double s = 0.0, sc = 0.0;
        for (uint32_t b : c.nl[a]) {
            const bool bd = c.S.kind[b] == Kind::Boundary;
            if (bd && c.S.dirichlet_C[b] == sphfsi::kNoDirichlet) continue;
            const V3 d = mi3(c, c.S.pos[a], c.S.pos[b]);
            const double r2 = r2of(d);
            if (r2 > rc2) continue;
            const double r = std::sqrt(r2);
            if (r == 0.0) {
#pragma omp critical
                { coincident = true; bad_i = a; bad_j = b; }
                continue;
            }
            const sphfsi::Material& mb = c.mats[c.S.material[b]];
            const double dsum = ma.diffusivity + mb.diffusivity;
            if (dsum == 0.0) continue;
            const double dt_ = 4.0 * ma.diffusivity * mb.diffusivity / dsum;
            const double rho_b = bd ? mb.reference_density : c.S.density[b];
            const double Vb = c.S.mass[b] / rho_b;
            const double term = Vb * dt_ * ((Cn[a] - Cn[b]) / r) * K.dw_dr(r);
            s += term;
            sc += std::abs(term);
        }
        const double rate = s / c.S.density[a];
        c.S.dC_dt[a] = rate;
        if (dir_group(a) < 0) c.S.concentration[a] = Cn[a] + c.dt * rate;
        c.dC_scale[a] = sc / c.S.density[a];
    }
    if (coincident)
        return fail(c, "coincident particles " + std::to_string(bad_i) + " and " + std::to_string(bad_j) +
                           " at step " + std::to_string(c.steps));
    return true;
}

// ----------------------------------------------------------- extrapolate
V3 rigid_rk(const Ctx& c, size_t r) {
    const sphg_body& b = c.bodies[c.S.group[r]];
    return sphfsi::rotate(qof(b), c.S.body_frame_pos[r]);
}

// extrapolate_wall_quantities (Adami 2012) [P6][P7]
bool stage_extrapolate(Ctx& c) {
    const sphfsi::QuinticKernel<3> K(c.h);
    const double rc2 = c.rc * c.rc;
    const double dx3 = c.P.dx * c.P.dx * c.P.dx;
    const int64_t n = (int64_t)c.S.size();
#pragma omp parallel for schedule(static)
    for (int64_t w = 0; w < n; ++w) {
        if (c.S.kind[w] == Kind::Fluid || ghost(c, (size_t)w)) continue;
        V3 uw = V3::zero(), aw = V3::zero();
        if (wall_member(c, (size_t)w)) {  // prescribed wall velocity / acceleration at t^{n+1} [P20]
            uw = v3(c.wall_v[c.S.group[w]]);
            aw = v3(c.wall_a[c.S.group[w]]);
        }
        if (c.S.kind[w] == Kind::Rigid) {
            const sphg_body& b = c.bodies[c.S.group[w]];
            const V3 rk = rigid_rk(c, (size_t)w);
            const V3 om = v3(b.omega);
            uw = c.S.vel[w];
            aw = v3(b.acc) + sphfsi::cross(v3(b.alpha), rk) + sphfsi::cross(om, sphfsi::cross(om, rk));  // [P6]
        }
        double sw = 0.0, sp = 0.0;
        V3 su = V3::zero();
        double smat[SPHG_MAX_MAT] = {0};
        for (uint32_t f : c.nl[w]) {
            if (c.S.kind[f] != Kind::Fluid) continue;
            const V3 d = mi3(c, c.S.pos[w], c.S.pos[f]);  // r_w - r_f
            const double r2 = r2of(d);
            if (r2 > rc2) continue;
            const double W = K.w(std::sqrt(r2));
            const V3 g = v3(c.P.mat[c.S.material[f]].body_force);
            sw += W;
            sp += W * (c.S.pressure[f] + c.S.density[f] * sphfsi::dot(g - aw, d));
            su += W * c.S.vel[f];
            smat[c.S.material[f]] += W;
        }
        int m = c.P.default_fluid_mat;
        if (sw > 0.0) {
            double best = -1.0;
            for (int k = 0; k < c.P.n_mat; ++k)
                if (smat[k] > best) { best = smat[k]; m = k; }
        }
        const double pw = sw > 0.0 ? sp / sw : 0.0;
        const V3 ut = sw > 0.0 ? 2.0 * uw - su / sw : uw;
        const sphfsi::Material& fm = c.mats[(sphfsi::MaterialId)m];
        const double rhow = std::max(fm.reference_density, sphfsi::eos_density(pw, fm));
        c.S.wall_pressure[w] = pw;
        c.S.wall_velocity[w] = ut;
        c.rho_w[w] = rhow;
        c.V_w[w] = fm.reference_density * dx3 / rhow;
        c.wall_mat[w] = m;
        if (c.S.kind[w] == Kind::Boundary) c.S.density[w] = rhow;
    }
    return true;
}

// ---------------------------------------------------------------- forces
struct Side {  // interaction values of one pair partner [P7]
    double rho, p, V, eta;
    V3 u, du;  // velocity and (u_adv - u) for the TVF A term
    bool fluid;
};

inline Side side_of(const Ctx& c, size_t j, const sphfsi::Material* eta_from) {
    Side s;
    if (c.S.kind[j] == Kind::Fluid) {
        s.rho = c.S.density[j];
        s.p = c.S.pressure[j];
        s.V = c.S.mass[j] / s.rho;
        s.eta = c.mats[c.S.material[j]].dynamic_viscosity();
        s.u = c.S.vel[j];
        s.du = c.S.vel_adv[j] - c.S.vel[j];
        s.fluid = true;
    } else {
        s.rho = c.rho_w[j];
        s.p = c.S.wall_pressure[j];
        s.V = c.V_w[j];
        s.eta = eta_from ? eta_from->dynamic_viscosity() : 0.0;  // eta_w := eta_i [P7]
        s.u = c.S.wall_velocity[j];
        s.du = V3::zero();  // A_w = 0 [P5]
        s.fluid = false;
    }
    return s;
}

// pair acceleration a_ij of fluid i due to j (momentum_rhs, PAPER:240-246 + TVF [P5]);
// returns a_ij and adds V2*gradW to bg.
// mag (tolerance scale): the summed magnitudes of the elementary products of the pair
// term — both halves of p~, the viscous and the two TVF terms — so a cancellation inside p~ (a fluid
// just below rho0 against a hydrostatic wall pressure) does not shrink the scale below the rounding of
// its parts.  It bounds |returned value| from above.
inline double norm3(const V3& v);
inline V3 pair_acc(const Ctx& c, const sphfsi::QuinticKernel<3>& K, const Side& I, double mi_, const Side& J,
                   const V3& d, double r, V3& bgsum, double* mag = nullptr, double* psens = nullptr,
                   double PI = 0.0, double PJ = 0.0) {
    const double dW = K.dw_dr(r);
    const V3 e = d / r;
    const V3 gW = dW * e;
    const double V2 = I.V * I.V + J.V * J.V;
    const double pt = (J.rho * I.p + I.rho * J.p) / (I.rho + J.rho);
    const double es = I.eta + J.eta;
    const double et = es > 0.0 ? 2.0 * I.eta * J.eta / es : 0.0;
    V3 term = (-pt) * gW + (et * dW / r) * (I.u - J.u);
    if (c.P.tvf) {
        // 0.5 (A_i + A_j) . gradW with A = rho u (u_adv - u)^T
        const V3 Ai = (I.rho * sphfsi::dot(I.du, gW)) * I.u;
        const V3 Aj = (J.rho * sphfsi::dot(J.du, gW)) * J.u;
        term += 0.5 * (Ai + Aj);
    }
    bgsum += V2 * gW;
    if (mag) {
        double m = (std::abs(J.rho * I.p) + std::abs(I.rho * J.p)) / (I.rho + J.rho) * std::abs(dW) +
                   std::abs(et * dW / r) * norm3(I.u - J.u);
        if (c.P.tvf)
            m += 0.5 * (std::abs(I.rho * sphfsi::dot(I.du, gW)) * norm3(I.u) +
                        std::abs(J.rho * sphfsi::dot(J.du, gW)) * norm3(J.u));
        *mag = std::abs(V2 / mi_) * m;
    }
    if (psens) *psens = std::abs(V2 / mi_) * std::abs(dW) * (J.rho * PI + I.rho * PJ) / (I.rho + J.rho);
    return (V2 / mi_) * term;
}

inline double norm3(const V3& v) { return std::sqrt(r2of(v)); }

bool stage_forces(Ctx& c) {
    const sphfsi::QuinticKernel<3> K(c.h);
    const double rc2 = c.rc * c.rc;
    const int64_t n = (int64_t)c.S.size();
    bool coincident = false;
    int64_t bad_i = 0, bad_j = 0;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const Kind ki = c.S.kind[i];
        if (ghost(c, (size_t)i)) continue;
        if (ki == Kind::Fluid) {
            const sphfsi::Material& mi_ = c.mats[c.S.material[i]];
            const Side I = side_of(c, (size_t)i, nullptr);
            V3 sum = V3::zero(), bg = V3::zero();
            double sc = 0.0, bgsc = 0.0, psc = 0.0;
            const double Pi = mi_.speed_of_sound * mi_.speed_of_sound * I.rho;  // EOS magnitude c^2 rho
            for (uint32_t j : c.nl[i]) {
                const V3 d = mi3(c, c.S.pos[i], c.S.pos[j]);
                const double r2 = r2of(d);
                if (r2 > rc2) continue;
                const double r = std::sqrt(r2);
                if (r == 0.0) {
#pragma omp critical
                    { coincident = true; bad_i = i; bad_j = j; }
                    continue;
                }
                const Side J = side_of(c, j, &mi_);
                V3 bgp = V3::zero();
                double mag = 0.0, ps = 0.0;
                // a wall / rigid pressure is a Shepard average of fluid pressures: the fluid's EOS magnitude
                const sphfsi::Material& mj = J.fluid ? c.mats[c.S.material[j]] : mi_;
                const double Pj = mj.speed_of_sound * mj.speed_of_sound * J.rho;
                const V3 a = pair_acc(c, K, I, c.S.mass[i], J, d, r, bgp, &mag, &ps, Pi, Pj);
                sum += a;
                bg += bgp;
                sc += mag;
                psc += ps;
                bgsc += norm3(bgp);
            }
            const V3 b = v3(c.P.mat[c.S.material[i]].body_force);
            c.S.acc[i] = sum + b;
            const double f = c.P.tvf ? -mi_.background_pressure / c.S.mass[i] : 0.0;
            c.S.acc_bg[i] = f * bg;
            c.acc_scale[i] = sc + norm3(b);
            c.acc_pscale[i] = psc;
            c.accbg_scale[i] = std::abs(f) * bgsc;
        } else if (ki == Kind::Rigid) {
            // coupling_force_on_rigid f_ri = -m_i a_ir + contact_force
            V3 f = V3::zero();
            double sc = 0.0, psc = 0.0;
            const uint32_t body = c.S.group[i];
            for (uint32_t j : c.nl[i]) {
                const Kind kj = c.S.kind[j];
                if (kj == Kind::Fluid) {
                    const V3 d = mi3(c, c.S.pos[j], c.S.pos[i]);  // r_j - r_r, from the fluid's view
                    const double r2 = r2of(d);
                    if (r2 > rc2) continue;
                    const double r = std::sqrt(r2);
                    if (r == 0.0) {
#pragma omp critical
                        { coincident = true; bad_i = i; bad_j = j; }
                        continue;
                    }
                    const sphfsi::Material& mj = c.mats[c.S.material[j]];
                    const Side Jf = side_of(c, j, nullptr);
                    const Side R = side_of(c, (size_t)i, &mj);
                    V3 bgp = V3::zero();
                    double mag = 0.0, ps = 0.0;
                    const double Pf = mj.speed_of_sound * mj.speed_of_sound * Jf.rho;
                    const V3 a = pair_acc(c, K, Jf, c.S.mass[j], R, d, r, bgp, &mag, &ps, Pf, Pf);
                    const V3 fr = (-c.S.mass[j]) * a;
                    f += fr;
                    sc += c.S.mass[j] * mag;
                    psc += c.S.mass[j] * ps;
                } else if (kj == Kind::Boundary || c.S.group[j] != body) {
                    const V3 d = mi3(c, c.S.pos[i], c.S.pos[j]);
                    const double r2 = r2of(d);
                    const double r = std::sqrt(r2);
                    if (!(r < c.P.dx)) continue;
                    if (r == 0.0) {
#pragma omp critical
                        { coincident = true; bad_i = i; bad_j = j; }
                        continue;
                    }
                    const V3 e = d / r;
                    const V3 vrel = c.S.vel[i] - c.S.vel[j];
                    const double s = c.P.kc * (r - c.P.dx) + c.P.dc * sphfsi::dot(e, vrel);
                    const V3 fc = (-std::min(0.0, s)) * e;
                    f += fc;
                    sc += norm3(fc);
                }
            }
            c.force[i] = f;
            c.force_scale[i] = sc;
            c.force_pscale[i] = psc;
        }
    }
    if (coincident)
        return fail(c, "coincident particles " + std::to_string(bad_i) + " and " + std::to_string(bad_j) +
                           " at step " + std::to_string(c.steps));
    return true;
}

// ---------------------------------------------------------------- bodies
double particle_inertia(double m, double dx) {  // SPEC:337-345 (3D, r_eff squared)
    const double reff = std::cbrt(0.75 / std::numbers::pi) * dx;
    return 0.4 * m * reff * reff;
}

void inverse_apply(const double I[6], const V3& t, V3& out, bool& singular) {  // [P11]
    const double xx = I[0], yy = I[1], zz = I[2], xy = I[3], xz = I[4], yz = I[5];
    const double c00 = yy * zz - yz * yz, c01 = xz * yz - xy * zz, c02 = xy * yz - xz * yy;
    const double c11 = xx * zz - xz * xz, c12 = xy * xz - xx * yz, c22 = xx * yy - xy * xy;
    const double det = xx * c00 + xy * c01 + xz * c02;
    const double tr = xx + yy + zz;
    if (!(std::abs(det) > 1e-12 * tr * tr * tr)) {
        singular = true;
        out = V3::zero();
        return;
    }
    singular = false;
    out = V3{(c00 * t[0] + c01 * t[1] + c02 * t[2]) / det, (c01 * t[0] + c11 * t[1] + c12 * t[2]) / det,
             (c02 * t[0] + c12 * t[1] + c22 * t[2]) / det};
}

// reduce_force_torque with compensated sums (kahan.hpp) about
// the integrated COM; world-frame inertia recomputed every step [P11].
bool stage_bodies(Ctx& c) {
    const int64_t nb = (int64_t)c.bodies.size();
    c.body_fscale.resize(c.bodies.size());
    c.body_tscale.resize(c.bodies.size());
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t k = 0; k < nb; ++k) {
        sphg_body& b = c.bodies[k];
        if (!b.alive) continue;
        sphfsi::KahanVec<3> F, T;
        sphfsi::KahanSum I6[6];
        double fs = 0.0, ts = 0.0;
        const sphfsi::Quaternion q = qof(b);
        for (uint32_t r : c.members[k]) {
            const V3 rk = sphfsi::rotate(q, c.S.body_frame_pos[r]);
            const V3& f = c.force[r];
            F.add(f);
            const V3 tq = sphfsi::moment(rk, f);
            T.add(tq);
            fs += norm3(f);
            ts += norm3(rk) * norm3(f);
            const double m = c.S.mass[r];
            const double Ir = particle_inertia(m, c.P.dx);
            const double d2 = r2of(rk);
            I6[0].add(Ir + m * (d2 - rk[0] * rk[0]));
            I6[1].add(Ir + m * (d2 - rk[1] * rk[1]));
            I6[2].add(Ir + m * (d2 - rk[2] * rk[2]));
            I6[3].add(-m * rk[0] * rk[1]);
            I6[4].add(-m * rk[0] * rk[2]);
            I6[5].add(-m * rk[1] * rk[2]);
        }
        const V3 f = F.value(), t = T.value();
        put3(b.force, f);
        put3(b.torque, t);
        for (int q6 = 0; q6 < 6; ++q6) b.inertia[q6] = I6[q6].value();
        c.body_fscale[k] = fs;
        c.body_tscale[k] = ts;
        if (b.mobile && b.mass > 0.0) {
            const V3 a = f / b.mass + v3(c.P.mat[b.material].body_force);
            put3(b.acc, a);
            V3 al;
            bool sing;
            inverse_apply(b.inertia, t, al, sing);
            put3(b.alpha, al);
        } else {
            put3(b.acc, V3::zero());
            put3(b.alpha, V3::zero());
        }
    }
    return true;
}

// reduce_mass_quantities (PAPER:303-325 single-processor form, Remark 3.10)
// anchored at the body's min-gid particle with minimum image; chi recomputed (Remark 3.7).
void mass_quantities(Ctx& c, size_t k) {
    sphg_body& b = c.bodies[k];
    const auto& mem = c.members[k];
    if (mem.empty()) {
        b.alive = 0;
        b.mass = 0.0;
        return;
    }
    const V3 anchor = c.S.pos[mem[0]];
    sphfsi::KahanSum M;
    sphfsi::KahanVec<3> MR;
    for (uint32_t r : mem) {
        const double m = c.S.mass[r];
        M.add(m);
        MR.add(m * mi3(c, c.S.pos[r], anchor));
    }
    const double m = M.value();
    const V3 com = wrap3(c, anchor + MR.value() / m);
    sphfsi::KahanSum I6[6];
    const sphfsi::Quaternion qc = qof(b).conjugate();
    for (uint32_t r : mem) {
        const double mr = c.S.mass[r];
        const V3 d = mi3(c, c.S.pos[r], com);
        const double Ir = particle_inertia(mr, c.P.dx);
        const double d2 = r2of(d);
        I6[0].add(Ir + mr * (d2 - d[0] * d[0]));
        I6[1].add(Ir + mr * (d2 - d[1] * d[1]));
        I6[2].add(Ir + mr * (d2 - d[2] * d[2]));
        I6[3].add(-mr * d[0] * d[1]);
        I6[4].add(-mr * d[0] * d[2]);
        I6[5].add(-mr * d[1] * d[2]);
        c.S.body_frame_pos[r] = sphfsi::rotate(qc, d);
    }
    b.mass = m;
    put3(b.com, com);
    for (int q6 = 0; q6 < 6; ++q6) b.inertia[q6] = I6[q6].value();
    b.alive = 1;
}

void rebuild_members(Ctx& c) {
    c.members.assign(c.bodies.size(), {});
    for (size_t i = 0; i < c.S.size(); ++i)
        if (c.S.kind[i] == Kind::Rigid && !ghost(c, i)) c.members[c.S.group[i]].push_back((uint32_t)i);
}

bool stage_mass(Ctx& c) {
    rebuild_members(c);
    for (size_t k = 0; k < c.bodies.size(); ++k)
        if (c.bodies[k].alive) mass_quantities(c, k);
    return true;
}

// ------------------------------------------------------------ integrator
// step(): half kick, drift, orientation, slave [P14]
// Inflow / outflow buffer zones [P23] (sphg.h sphg_buffer): the zone of a fluid particle at
// x (first zone whose box lo <= x < hi holds it) or -1, and the zone's prescribed velocity at x when
// the zone is active at time t (t > t_start), U = e_axis u_mean 6 xi (1 - xi) along profile_axis.
int buffer_of(const Ctx& c, const V3& x) {
    for (int b = 0; b < c.P.n_buffers; ++b) {
        const sphg_buffer& B = c.P.buffers[b];
        bool in = true;
        for (int a = 0; a < 3; ++a) in = in && x[a] >= B.lo[a] && x[a] < B.hi[a];
        if (in) return b;
    }
    return -1;
}

V3 buffer_velocity(const Ctx& c, int b, const V3& x, double t) {
    const sphg_buffer& B = c.P.buffers[b];
    double u = 0.0;
    if (t > B.t_start) {
        double f = 1.0;
        if (B.profile_axis >= 0) {
            const int a = B.profile_axis;
            const double xi = (x[a] - B.lo[a]) / (B.hi[a] - B.lo[a]);
            f = (6.0 * xi) * (1.0 - xi);
        }
        u = B.u_mean * f;
    }
    V3 v = V3::zero();
    v[B.axis] = u;
    return v;
}

bool stage_kick_drift(Ctx& c) {
    const double hdt = 0.5 * c.dt, dt = c.dt;
    if (c.n_walls > 0) {
        eval_walls(c, c.t + hdt, c.wall_vh, nullptr);
        eval_walls(c, c.t + dt, c.wall_v, c.wall_a);
    }
    const int64_t n = (int64_t)c.S.size();
    double umax = 0.0;
    for (auto& b : c.bodies) {
        if (!b.alive || !b.mobile) continue;
        const V3 u = v3(b.vel) + hdt * v3(b.acc);
        const V3 w = v3(b.omega) + hdt * v3(b.alpha);
        put3(b.vel, u);
        put3(b.omega, w);
        put3(b.com, wrap3(c, v3(b.com) + dt * u));
        const sphfsi::Quaternion q = sphfsi::orientation_step<3>(qof(b), w, dt);
        b.q[0] = q.w; b.q[1] = q.x; b.q[2] = q.y; b.q[3] = q.z;
    }
    bool escaped = false, nonfinite = false;
    int64_t bad = std::numeric_limits<int64_t>::max(), bad_nf = std::numeric_limits<int64_t>::max();
    double md2 = 0.0;
#pragma omp parallel for schedule(static) reduction(max : umax, md2)
    for (int64_t i = 0; i < n; ++i) {
        const Kind k = ghost(c, (size_t)i) ? Kind::Boundary : c.S.kind[i];  // ghosts move by halo only
        if (k == Kind::Fluid) {
            const int zb = c.P.n_buffers ? buffer_of(c, c.S.pos[i]) : -1;  // [P23], role from x^n
            const V3 uh = zb >= 0 ? buffer_velocity(c, zb, c.S.pos[i], c.t + hdt) : c.S.vel[i] + hdt * c.S.acc[i];
            const V3 ua = (c.P.tvf && zb < 0) ? uh + hdt * c.S.acc_bg[i] : uh;
            c.S.vel[i] = uh;
            c.S.vel_adv[i] = ua;
            c.S.pos[i] = wrap3(c, c.S.pos[i] + dt * ua);
            umax = std::max(umax, r2of(uh));
        } else if (k == Kind::Rigid) {
            const sphg_body& b = c.bodies[c.S.group[i]];
            const V3 rk = sphfsi::rotate(qof(b), c.S.body_frame_pos[i]);
            c.S.pos[i] = wrap3(c, v3(b.com) + rk);
            const V3 u = v3(b.vel) + sphfsi::cross(v3(b.omega), rk);
            c.S.vel[i] = u;
            c.S.vel_adv[i] = u;
        } else if (wall_member(c, (size_t)i)) {  // prescribed wall motion [P20]
            const uint32_t g = c.S.group[i];
            c.S.pos[i] = wrap3(c, c.S.pos[i] + dt * v3(c.wall_vh[g]));
            c.S.vel[i] = v3(c.wall_v[g]);
        } else {
            continue;
        }
        for (int a = 0; a < 3; ++a) {
            if (!std::isfinite(c.S.pos[i][a])) {  // a blown-up state: SPEC:625 runtime assertion
#pragma omp critical
                { nonfinite = true; bad_nf = std::min(bad_nf, i); }
            } else if (!c.P.periodic[a] && (c.S.pos[i][a] < c.P.lo[a] || c.S.pos[i][a] > c.P.hi[a])) {
#pragma omp critical
                { escaped = true; bad = std::min(bad, i); }
            }
        }
        if (c.built) md2 = std::max(md2, r2of(mi3(c, c.S.pos[i], c.pos_ref[i])));
    }
    c.u_max = std::sqrt(umax);
    c.max_disp = std::sqrt(md2);
    c.t += c.dt;
    if (escaped) return fail(c, "escaped particle " + std::to_string(bad) + " at step " + std::to_string(c.steps + 1));
    if (nonfinite)
        return fail(c, "non-finite state of particle " + std::to_string(bad_nf) + " at step " + std::to_string(c.steps + 1));
    return true;
}

bool stage_final_kick(Ctx& c) {
    const double hdt = 0.5 * c.dt;
    for (auto& b : c.bodies) {
        if (!b.alive || !b.mobile) continue;
        put3(b.vel, v3(b.vel) + hdt * v3(b.acc));
        put3(b.omega, v3(b.omega) + hdt * v3(b.alpha));
    }
    const int64_t n = (int64_t)c.S.size();
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        if (ghost(c, (size_t)i)) continue;
        if (c.S.kind[i] == Kind::Fluid) {
            const int zb = c.P.n_buffers ? buffer_of(c, c.S.pos[i]) : -1;  // [P23], role from x^{n+1}
            c.S.vel[i] = zb >= 0 ? buffer_velocity(c, zb, c.S.pos[i], c.t) : c.S.vel[i] + hdt * c.S.acc[i];
        } else if (c.S.kind[i] == Kind::Rigid) {
            const sphg_body& b = c.bodies[c.S.group[i]];
            const V3 rk = sphfsi::rotate(qof(b), c.S.body_frame_pos[i]);
            c.S.vel[i] = v3(b.vel) + sphfsi::cross(v3(b.omega), rk);
            c.S.vel_adv[i] = c.S.vel[i];  // rigid vel_adv mirrors vel
        }
    }
    return true;
}

// ------------------------------------------------------------ transitions
// detect_transitions / apply_transitions / post_transition_body_velocity /
// split_disconnected_bodies [P12]
// detect_transitions over the owned particles (a decomposed rank leaves its ghosts to their owners)
void detect_events(const Ctx& c, std::vector<uint32_t>& melt, std::vector<uint32_t>& solid) {
    const bool conc = c.P.transitions == 2;  // TransitionMode::Concentration (config.hpp:61) [P19]
    melt.clear();
    solid.clear();
    for (size_t i = 0; i < c.S.size(); ++i) {
        if (ghost(c, i)) continue;
        const sphg_material& m = c.P.mat[c.S.material[i]];
        const double thr = conc ? m.C_t : m.T_t;
        const double x = conc ? c.S.concentration[i] : c.S.temperature[i];
        if (std::isnan(thr)) continue;
        if (c.S.kind[i] == Kind::Rigid && m.melt_target >= 0 && x > thr) melt.push_back((uint32_t)i);
        else if (c.S.kind[i] == Kind::Fluid && m.solidify_target >= 0 && x < thr)
            solid.push_back((uint32_t)i);
    }
}

bool stage_transitions(Ctx& c) {
    if (c.P.transitions != 1 && c.P.transitions != 2) return true;
    const size_t n = c.S.size();
    std::vector<uint32_t> melt, solid;
    detect_events(c, melt, solid);
    if (melt.empty() && solid.empty()) return true;
    c.n_melt += (int64_t)melt.size();
    c.n_solid += (int64_t)solid.size();
    const size_t nb0 = c.bodies.size();
    std::vector<sphg_body> old = c.bodies;   // pre-batch body state (u'_k, r'_k)
    std::vector<char> affected(nb0, 0), lost(nb0, 0);
    std::vector<uint32_t> src_body;          // for each body id: the pre-batch body it came from (or self)
    // 1. melts: rigid -> fluid with the body's rigid-motion velocity
    std::vector<char> melting(n, 0);
    for (uint32_t r : melt) melting[r] = 1;
    std::vector<sphg_event> batch;
    const int64_t ev_step = c.steps + 1;
    for (uint32_t r : melt) {
        const uint32_t k = c.S.group[r];
        if (c.event_log) batch.push_back(sphg_event{ev_step, r, 1, (int32_t)k, -1});
        const sphg_body& b = c.bodies[k];
        const V3 rk = sphfsi::rotate(qof(b), c.S.body_frame_pos[r]);
        const V3 u = v3(b.vel) + sphfsi::cross(v3(b.omega), rk);
        const int tgt = c.P.mat[c.S.material[r]].melt_target;
        c.S.kind[r] = Kind::Fluid;
        c.S.material[r] = (uint16_t)tgt;
        c.S.group[r] = 0;
        c.S.vel[r] = u;
        c.S.vel_adv[r] = u;
        c.S.acc[r] = V3::zero();
        c.S.acc_bg[r] = V3::zero();
        c.S.density[r] = c.P.mat[tgt].rho0;
        c.S.pressure[r] = 0.0;
        c.S.body_frame_pos[r] = V3::zero();
        c.S.wall_pressure[r] = 0.0;
        c.S.wall_velocity[r] = V3::zero();
        c.force[r] = V3::zero();
        affected[k] = 1;
        lost[k] = 1;
    }
    // 2. solidification: attach to the body of the nearest pre-batch rigid particle within r_c
    //    (ties by gid), else spawn; new ids ascending in gid (solid is gid-sorted).
    const double rc2 = c.rc * c.rc;
    std::vector<int64_t> target(solid.size(), -1);
    for (size_t e = 0; e < solid.size(); ++e) {
        const uint32_t i = solid[e];
        double best = std::numeric_limits<double>::infinity();
        int64_t bj = -1;
        for (uint32_t j : c.nl[i]) {
            if (c.S.kind[j] != Kind::Rigid || melting[j]) continue;
            const double r2 = r2of(mi3(c, c.S.pos[i], c.S.pos[j]));
            if (r2 > rc2) continue;
            if (r2 < best || (r2 == best && (int64_t)j < bj)) { best = r2; bj = j; }
        }
        target[e] = bj >= 0 ? (int64_t)c.S.group[bj] : -1;
    }
    for (size_t e = 0; e < solid.size(); ++e) {
        const uint32_t i = solid[e];
        const int tgt = c.P.mat[c.S.material[i]].solidify_target;
        uint32_t k;
        if (target[e] >= 0) {
            k = (uint32_t)target[e];
        } else {
            sphg_body nbd{};
            nbd.q[0] = 1.0;
            put3(nbd.vel, c.S.vel[i]);
            nbd.material = tgt;
            nbd.mobile = 1;
            nbd.alive = 1;
            c.bodies.push_back(nbd);
            old.push_back(nbd);
            k = (uint32_t)(c.bodies.size() - 1);
            affected.push_back(1);
            lost.push_back(0);
        }
        affected[k] = 1;
        c.S.kind[i] = Kind::Rigid;
        c.S.material[i] = (uint16_t)tgt;
        c.S.group[i] = k;
        c.S.density[i] = c.P.mat[tgt].rho0;
        c.S.pressure[i] = 0.0;
        c.S.acc[i] = V3::zero();
        c.S.acc_bg[i] = V3::zero();
        c.S.wall_pressure[i] = 0.0;
        c.S.wall_velocity[i] = V3::zero();
    }
    rebuild_members(c);
    src_body.resize(c.bodies.size());
    std::iota(src_body.begin(), src_body.end(), 0u);
    // 3. split bodies that lost particles into connected components (adjacency <= 1.5 dx);
    //    the component holding the min gid keeps the id, others get new ids by min gid.
    const double adj2 = (1.5 * c.P.dx) * (1.5 * c.P.dx);
    const size_t nb1 = c.bodies.size();
    for (size_t k = 0; k < nb1; ++k) {
        if (k >= lost.size() || !lost[k] || c.members[k].empty()) continue;
        const auto mem = c.members[k];
        std::vector<uint32_t> lab(mem.size());
        std::iota(lab.begin(), lab.end(), 0u);
        std::function<uint32_t(uint32_t)> find = [&](uint32_t x) {
            while (lab[x] != x) { lab[x] = lab[lab[x]]; x = lab[x]; }
            return x;
        };
        std::vector<int64_t> pos_in(n, -1);
        for (size_t a = 0; a < mem.size(); ++a) pos_in[mem[a]] = (int64_t)a;
        for (size_t a = 0; a < mem.size(); ++a)
            for (uint32_t j : c.nl[mem[a]]) {
                const int64_t b = pos_in[j];
                if (b < 0) continue;
                if (r2of(mi3(c, c.S.pos[mem[a]], c.S.pos[j])) > adj2) continue;
                uint32_t ra = find((uint32_t)a), rb = find((uint32_t)b);
                if (ra != rb) lab[std::max(ra, rb)] = std::min(ra, rb);  // root = min index = min gid
            }
        std::vector<uint32_t> roots;
        for (size_t a = 0; a < mem.size(); ++a)
            if (find((uint32_t)a) == a) roots.push_back((uint32_t)a);
        if (roots.size() <= 1) continue;
        // roots ascending = components ordered by min gid; roots[0] keeps id k
        for (size_t q = 1; q < roots.size(); ++q) {
            sphg_body nbd = c.bodies[k];
            c.bodies.push_back(nbd);
            const uint32_t nk = (uint32_t)(c.bodies.size() - 1);
            src_body.push_back((uint32_t)k);
            old.push_back(old[k]);
            affected.push_back(1);
            lost.push_back(0);
            for (size_t a = 0; a < mem.size(); ++a)
                if (find((uint32_t)a) == roots[q]) c.S.group[mem[a]] = nk;
        }
    }
    rebuild_members(c);
    if (c.event_log) {  // solidified particles with the body they ended the batch in; all ordered by gid
        for (uint32_t i : solid) batch.push_back(sphg_event{ev_step, i, 2, -1, (int32_t)c.S.group[i]});
        std::sort(batch.begin(), batch.end(), [](const sphg_event& a, const sphg_event& b) { return a.gid < b.gid; });
        c.events.insert(c.events.end(), batch.begin(), batch.end());
    }
    // 4. mass quantities + post-transition velocity u_k = u'_k + w x (r_k - r'_k) [P12]
    for (size_t k = 0; k < c.bodies.size(); ++k) {
        if (k >= affected.size() || !affected[k]) continue;
        const sphg_body& o = old[k];
        // chi must be measured in the (unchanged) body orientation
        mass_quantities(c, k);
        sphg_body& b = c.bodies[k];
        if (!b.alive) continue;
        const bool spawned = (k >= nb0) && (src_body[k] == k);
        if (!spawned) {
            const V3 shift = mi3(c, v3(b.com), v3(o.com));
            put3(b.vel, v3(o.vel) + sphfsi::cross(v3(o.omega), shift));
        }
        // particle velocities follow the body's rigid motion
        for (uint32_t r : c.members[k]) {
            const V3 rk = sphfsi::rotate(qof(b), c.S.body_frame_pos[r]);
            const V3 u = v3(b.vel) + sphfsi::cross(v3(b.omega), rk);
            c.S.vel[r] = u;
            c.S.vel_adv[r] = u;
        }
    }
    // 5. force/torque of the new membership (accelerations for the next kick)
    return stage_bodies(c);
}

void resize_aux(Ctx& c) {
    const size_t n = c.S.size();
    c.force.assign(n, V3::zero());
    c.rho_w.assign(n, 0.0);
    c.V_w.assign(n, 0.0);
    c.wall_mat.assign(n, 0);
    c.acc_scale.assign(n, 0.0);
    c.accbg_scale.assign(n, 0.0);
    c.dT_scale.assign(n, 0.0);
    c.dC_scale.assign(n, 0.0);
    c.force_scale.assign(n, 0.0);
    c.acc_pscale.assign(n, 0.0);
    c.force_pscale.assign(n, 0.0);
    c.rho_scale.assign(n, 0.0);
}

bool run_stage(Ctx& c, int s) {
    if (s != SPHG_STAGE_REBUILD && s != SPHG_STAGE_KICK_DRIFT && s != SPHG_STAGE_MASS && !c.built)
        if (!stage_rebuild(c)) return false;
    switch (s) {
        case SPHG_STAGE_REBUILD: return stage_rebuild(c);
        case SPHG_STAGE_DENSITY: return stage_density(c);
        case SPHG_STAGE_HEAT: return (!c.P.thermal || stage_heat(c)) && (!c.P.diffusion || stage_diffusion(c));
        case SPHG_STAGE_EXTRAPOLATE: return stage_extrapolate(c);
        case SPHG_STAGE_FORCES: return stage_forces(c);
        case SPHG_STAGE_BODIES: return stage_bodies(c);
        case SPHG_STAGE_KICK_DRIFT: return stage_kick_drift(c);
        case SPHG_STAGE_FINAL_KICK: return stage_final_kick(c);
        case SPHG_STAGE_TRANSITIONS:
            if (c.P.transitions && c.has_ghosts)
                return fail(c, "with ghost particles, transitions are applied by the decomposed batch");
            return stage_transitions(c);
        case SPHG_STAGE_MASS: return stage_mass(c);
    }
    return fail(c, "unknown stage");
}

// compute_dt: cfl 0.25 h/(c+|u_max|), viscous 0.125 h^2/nu, body force
// 0.25 sqrt(h/|b_max|), contact 0.22 sqrt(m_r/k_c), conduction 0.1 rho c_p h^2/kappa, each over the most
// restrictive material; absent physics -> +inf.
void dt_terms(const Ctx& c, double u_max, double lim[5]) {
    const double inf = std::numeric_limits<double>::infinity();
    for (int k = 0; k < 5; ++k) lim[k] = inf;
    const double h = c.h;
    double bmax = 0.0;
    for (int m = 0; m < c.P.n_mat; ++m) {
        const sphg_material& M = c.P.mat[m];
        if (M.c > 0.0) lim[0] = std::min(lim[0], 0.25 * h / (M.c + u_max));
        if (M.nu > 0.0) lim[1] = std::min(lim[1], 0.125 * h * h / M.nu);
        bmax = std::max(bmax, std::sqrt(M.body_force[0] * M.body_force[0] + M.body_force[1] * M.body_force[1] +
                                        M.body_force[2] * M.body_force[2]));
        if (c.P.thermal && M.kappa > 0.0 && M.cp > 0.0) lim[4] = std::min(lim[4], 0.1 * M.rho0 * M.cp * h * h / M.kappa);
    }
    if (bmax > 0.0) lim[2] = 0.25 * std::sqrt(h / bmax);
    if (c.P.kc > 0.0 && c.m_r > 0.0) lim[3] = 0.22 * std::sqrt(c.m_r / c.P.kc);
}

// Runtime assertion after a step ("refuse with diagnostic listing the violated condition";
// SPEC:560-561): u_max of this step's kick.
bool check_dt(Ctx& c) {
    if (c.P.dt_check == SPHG_DT_OFF) return true;
    static const char* names[5] = {"cfl", "viscous", "body force", "contact", "conduction"};
    double lim[5];
    dt_terms(c, c.u_max, lim);
    c.dt_term = -1;
    c.dt_limit = std::numeric_limits<double>::infinity();
    std::string bad;
    for (int k = 0; k < 5; ++k) {
        if (lim[k] < c.dt_limit) { c.dt_limit = lim[k]; c.dt_term = k; }
        if (c.dt > lim[k]) {
            char b[96];
            std::snprintf(b, sizeof b, "%s%s limit %.6g", bad.empty() ? "" : ", ", names[k], lim[k]);
            bad += b;
        }
    }
    if (bad.empty()) return true;
    c.dt_violations++;
    if (c.P.dt_check == SPHG_DT_WARN) return true;
    char b[128];
    std::snprintf(b, sizeof b, "time-step condition violated at step %lld: dt = %.6g exceeds the ",
                  (long long)c.steps, c.dt);
    return fail(c, std::string(b) + bad);
}

bool one_step(Ctx& c) {
    if (!stage_kick_drift(c)) return false;
    const double half_skin = 0.5 * (c.rv - c.rc);
    if (!c.built || c.max_disp > half_skin)  // SPEC:212 [P3]
        if (!stage_rebuild(c)) return false;
    if (!stage_density(c)) return false;
    if (c.P.thermal && !stage_heat(c)) return false;
    if (c.P.diffusion && !stage_diffusion(c)) return false;
    if (!stage_extrapolate(c)) return false;
    if (!stage_forces(c)) return false;
    if (!stage_bodies(c)) return false;
    if (!stage_final_kick(c)) return false;
    if (c.P.transitions != 0 && !stage_transitions(c)) return false;
    c.steps++;
    return check_dt(c);
}

void copy3(std::vector<V3>& dst, const double* src, size_t n) {
    dst.resize(n);
    if (!src) { std::fill(dst.begin(), dst.end(), V3::zero()); return; }
    for (size_t i = 0; i < n; ++i) dst[i] = V3{src[3 * i], src[3 * i + 1], src[3 * i + 2]};
}
template <class T>
void copy1(std::vector<T>& dst, const T* src, size_t n, T dflt) {
    dst.resize(n);
    if (!src) { std::fill(dst.begin(), dst.end(), dflt); return; }
    std::copy(src, src + n, dst.begin());
}
void out3(double* dst, const std::vector<V3>& src) {
    if (!dst) return;
    for (size_t i = 0; i < src.size(); ++i) put3(dst + 3 * i, src[i]);
}
template <class T>
void out1(T* dst, const std::vector<T>& src) {
    if (dst) std::copy(src.begin(), src.end(), dst);
}

}  // namespace

// =================================================================== C ABI
extern "C" {

struct orc_ctx;

int orc_validate(const sphg_params* p, char* buf, size_t len) {
    const auto v = validate(*p);
    std::string s;
    for (size_t i = 0; i < v.size(); ++i) s += (i ? "\n" : "") + v[i];
    if (buf && len) {
        std::strncpy(buf, s.c_str(), len - 1);
        buf[len - 1] = 0;
    }
    return v.empty() ? SPHG_OK : SPHG_ERR_CONFIG;
}

int orc_create(const sphg_params* p, int /*device*/, orc_ctx** out) {
    *out = nullptr;
    const auto v = validate(*p);
    if (!v.empty()) return SPHG_ERR_CONFIG;
    Ctx* c = new Ctx();
    c->P = *p;
    if (c->P.h <= 0.0) c->P.h = c->P.dx;
    c->mats = to_config(c->P).materials;
    setup_geometry(*c);
    c->t = c->P.t0;
    *out = reinterpret_cast<orc_ctx*>(c);
    return SPHG_OK;
}

int orc_upload(orc_ctx* h, const sphg_soa* s, const sphg_body* bodies, size_t nb) {
    Ctx& c = *reinterpret_cast<Ctx*>(h);
    const size_t n = s->n;
    auto& S = c.S;
    copy3(S.pos, s->pos, n);
    copy3(S.vel, s->vel, n);
    copy3(S.vel_adv, s->vel_adv, n);
    copy3(S.acc, s->acc, n);
    copy3(S.acc_bg, s->acc_bg, n);
    copy1(S.density, s->density, n, 0.0);
    copy1(S.pressure, s->pressure, n, 0.0);
    copy1(S.mass, s->mass, n, 0.0);
    copy1(S.temperature, s->temperature, n, 0.0);
    copy1(S.dT_dt, s->dT_dt, n, 0.0);
    copy1(S.concentration, s->concentration, n, 0.0);
    copy1(S.dC_dt, s->dC_dt, n, 0.0);
    S.kind.resize(n);
    for (size_t i = 0; i < n; ++i) S.kind[i] = static_cast<Kind>(s->kind[i]);
    copy1(S.group, s->group, n, 0u);
    copy1(S.material, s->material, n, (uint16_t)0);
    copy3(S.body_frame_pos, s->body_frame_pos, n);
    copy1(S.wall_pressure, s->wall_pressure, n, 0.0);
    copy3(S.wall_velocity, s->wall_velocity, n);
    copy1(S.dirichlet_T, s->dirichlet_T, n, (uint8_t)0xff);
    copy1(S.dirichlet_C, s->dirichlet_C, n, (uint8_t)0xff);
    if (s->owner) copy1(S.owner, s->owner, n, 0u);
    else S.owner.assign(n, (uint32_t)c.P.rank);
    c.halo.assign(SPHG_MAX_HALO_SLOTS, {});
    bool any_ghost = false;
    for (size_t i = 0; i < n; ++i) any_ghost |= ghost(c, i);
    c.has_ghosts = any_ghost;
    c.disp_since_partition = 0.0;
    resize_aux(c);
    c.m_r = 0.0;  // [P22]: rigid particles, and fluid particles that may solidify
    for (size_t i = 0; i < n; ++i) {
        const bool can_be_rigid = S.kind[i] == Kind::Rigid ||
                                  (S.kind[i] == Kind::Fluid && c.P.transitions != 0 &&
                                   c.P.mat[S.material[i]].solidify_target >= 0);
        if (can_be_rigid && S.mass[i] > 0.0 && (c.m_r == 0.0 || S.mass[i] < c.m_r)) c.m_r = S.mass[i];
    }
    if (s->force) copy3(c.force, s->force, n);
    c.bodies.assign(bodies, bodies + nb);
    c.body_fscale.assign(nb, 0.0);
    c.body_tscale.assign(nb, 0.0);
    rebuild_members(c);
    c.built = false;
    return SPHG_OK;
}

int orc_run_stage(orc_ctx* h, int stage) {
    Ctx& c = *reinterpret_cast<Ctx*>(h);
    return run_stage(c, stage) ? SPHG_OK : SPHG_ERR_RUNTIME;
}

int orc_set_wall_motion(orc_ctx* h, int32_t n_groups, sphg_wall_motion_fn fn, void* user) {
    Ctx& c = *reinterpret_cast<Ctx*>(h);
    if (n_groups < 0 || n_groups > SPHG_MAX_WALL_GROUPS) return SPHG_ERR_CONFIG;
    c.n_walls = fn ? n_groups : 0;
    c.wall_fn = fn;
    c.wall_user = user;
    if (c.n_walls) eval_walls(c, c.t, c.wall_v, c.wall_a);  // state at the current time (a^0)
    return SPHG_OK;
}

int orc_initialize(orc_ctx* h) {
    Ctx& c = *reinterpret_cast<Ctx*>(h);
    if (c.n_walls) eval_walls(c, c.t, c.wall_v, c.wall_a);
    for (int s : {SPHG_STAGE_REBUILD, SPHG_STAGE_DENSITY, SPHG_STAGE_EXTRAPOLATE, SPHG_STAGE_FORCES, SPHG_STAGE_BODIES})
        if (!run_stage(c, s)) return SPHG_ERR_RUNTIME;
    return SPHG_OK;
}

// sphg_upload_state: new positions / velocities (gid order) into the resident state; the Verlet
// list survives unless a particle moved more than half the skin from its reference position.
int orc_upload_state(orc_ctx* h, const double* pos, const double* vel, size_t n) {
    Ctx& c = *reinterpret_cast<Ctx*>(h);
    if (n != c.S.size()) {
        c.err = "upload_state: store size mismatch (upload first)";
        return SPHG_ERR_RUNTIME;
    }
    double md2 = 0.0;
    for (size_t i = 0; i < n; ++i) {
        if (pos) c.S.pos[i] = V3{pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
        if (vel) c.S.vel[i] = V3{vel[3 * i], vel[3 * i + 1], vel[3 * i + 2]};
        if (c.built && pos) md2 = std::max(md2, r2of(mi3(c, c.S.pos[i], c.pos_ref[i])));
    }
    if (c.built && pos && std::sqrt(md2) > 0.5 * (c.rv - c.rc)) c.built = false;
    return SPHG_OK;
}

int decomposed_step(orc_ctx* h);

int orc_step(orc_ctx* h, int nsteps) {
    Ctx& c = *reinterpret_cast<Ctx*>(h);
    for (int k = 0; k < nsteps; ++k) {
        if (c.has_ghosts && c.exch_fn) {
            if (c.partition_limit > 0.0 && c.disp_since_partition + c.max_disp + 0.5 * (c.rv - c.rc) > c.partition_limit)
                return SPHG_NEED_PARTITION;  // sphg.h sphg_set_partition_limit
            const int rc = decomposed_step(h);
            if (rc) return rc;
        } else if (!one_step(c)) {
            return SPHG_ERR_RUNTIME;
        }
    }
    return SPHG_OK;
}

int orc_download(orc_ctx* h, sphg_soa* o, sphg_body* bodies, size_t* nb) {
    Ctx& c = *reinterpret_cast<Ctx*>(h);
    const auto& S = c.S;
    out3(o->pos, S.pos);
    out3(o->vel, S.vel);
    out3(o->vel_adv, S.vel_adv);
    out3(o->acc, S.acc);
    out3(o->acc_bg, S.acc_bg);
    out1(o->density, S.density);
    out1(o->pressure, S.pressure);
    out1(o->mass, S.mass);
    out1(o->temperature, S.temperature);
    out1(o->dT_dt, S.dT_dt);
    if (o->kind)
        for (size_t i = 0; i < S.size(); ++i) o->kind[i] = static_cast<uint8_t>(S.kind[i]);
    out1(o->group, S.group);
    out1(o->material, S.material);
    out3(o->body_frame_pos, S.body_frame_pos);
    out1(o->wall_pressure, S.wall_pressure);
    out3(o->wall_velocity, S.wall_velocity);
    out1(o->dirichlet_T, S.dirichlet_T);
    out1(o->concentration, S.concentration);
    out1(o->dC_dt, S.dC_dt);
    out1(o->dirichlet_C, S.dirichlet_C);
    out3(o->force, c.force);
    if (o->owner)
        for (size_t i = 0; i < S.size(); ++i) o->owner[i] = ghost(c, i) ? 0xffffffffu : (uint32_t)c.P.rank;
    if (nb) {
        if (bodies) {
            const size_t m = std::min(*nb, c.bodies.size());
            std::copy(c.bodies.begin(), c.bodies.begin() + m, bodies);
        }
        *nb = c.bodies.size();
    }
    return SPHG_OK;
}

int orc_step_download(orc_ctx* h, int nsteps, sphg_soa* o, sphg_body* bodies, size_t* nb) {
    const int rc = orc_step(h, nsteps);
    return rc ? rc : orc_download(h, o, bodies, nb);
}

int orc_num_bodies(orc_ctx* h, size_t* nb) {
    *nb = reinterpret_cast<Ctx*>(h)->bodies.size();
    return SPHG_OK;
}

int orc_get_cells(orc_ctx* h, int64_t* cell_of_gid, uint32_t* sorted_gid) {
    Ctx& c = *reinterpret_cast<Ctx*>(h);
    if (!c.built && !stage_rebuild(c)) return SPHG_ERR_RUNTIME;
    if (cell_of_gid) std::copy(c.cell_of.begin(), c.cell_of.end(), cell_of_gid);
    if (sorted_gid) std::copy(c.sorted.begin(), c.sorted.end(), sorted_gid);
    return SPHG_OK;
}

int orc_cell_occupancy(orc_ctx* h, int64_t* hist, size_t nbins, int64_t* max_count) {
    Ctx& c = *reinterpret_cast<Ctx*>(h);
    if (nbins == 0) return SPHG_ERR_CONFIG;
    if (!c.built && !stage_rebuild(c)) return SPHG_ERR_RUNTIME;
    const int64_t ncells = (int64_t)c.ncell[0] * c.ncell[1] * c.ncell[2];
    std::vector<int64_t> cnt(ncells, 0);
    for (int64_t k : c.cell_of) cnt[k]++;
    std::fill(hist, hist + nbins, 0);
    int64_t mx = 0;
    for (int64_t m : cnt) {
        hist[std::min<int64_t>(m, (int64_t)nbins - 1)]++;
        mx = std::max(mx, m);
    }
    if (max_count) *max_count = mx;
    return SPHG_OK;
}

int orc_get_nlist(orc_ctx* h, int64_t* offsets, uint32_t* nbr) {
    Ctx& c = *reinterpret_cast<Ctx*>(h);
    if (!c.built && !stage_rebuild(c)) return SPHG_ERR_RUNTIME;
    int64_t o = 0;
    for (size_t i = 0; i < c.nl.size(); ++i) {
        if (offsets) offsets[i] = o;
        if (nbr) std::copy(c.nl[i].begin(), c.nl[i].end(), nbr + o);
        o += (int64_t)c.nl[i].size();
    }
    if (offsets) offsets[c.nl.size()] = o;
    return SPHG_OK;
}

// tolerance scales, gid order
// shepard_interpolate on a grid: brute force over all particles in gid order.
int orc_shepard_grid(orc_ctx* h, const double* origin, const double* spacing, const int32_t* dims, int32_t field,
                     uint32_t kind_mask, double* out, uint8_t* support) {
    const Ctx& c = *reinterpret_cast<Ctx*>(h);
    if (dims[0] < 0 || dims[1] < 0 || dims[2] < 0 || field < 0 || field > SPHG_FIELD_DENSITY) return SPHG_ERR_CONFIG;
    const int nc = field == SPHG_FIELD_VELOCITY ? 3 : 1;
    const sphfsi::QuinticKernel<3> K(c.P.h > 0.0 ? c.P.h : c.P.dx);
    const double rc = sphfsi::kKernelSupportScale * (c.P.h > 0.0 ? c.P.h : c.P.dx);
    const double rc2 = rc * rc;
    const size_t n = c.S.size();
    const int64_t np = (int64_t)dims[0] * dims[1] * dims[2];
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < np; ++q) {
        const int64_t a = q / ((int64_t)dims[1] * dims[2]), b = (q / dims[2]) % dims[1], cc = q % dims[2];
        const V3 x{origin[0] + (double)a * spacing[0], origin[1] + (double)b * spacing[1],
                   origin[2] + (double)cc * spacing[2]};
        double num[3] = {0, 0, 0}, den = 0.0;
        for (size_t j = 0; j < n; ++j) {
            if (!((kind_mask >> static_cast<uint32_t>(c.S.kind[j])) & 1u) || ghost(c, j)) continue;
            const double r2 = r2of(mi3(c, x, c.S.pos[j]));
            if (r2 > rc2) continue;
            const sphfsi::Material& m = c.mats[c.S.material[j]];
            const double rho = c.S.kind[j] == Kind::Fluid ? c.S.density[j] : m.reference_density;
            const double w = (c.S.mass[j] / rho) * K.w(std::sqrt(r2));
            den += w;
            switch (field) {
                case SPHG_FIELD_VELOCITY:
                    for (int k = 0; k < 3; ++k) num[k] += w * c.S.vel[j][k];
                    break;
                case SPHG_FIELD_TEMPERATURE: num[0] += w * c.S.temperature[j]; break;
                case SPHG_FIELD_CONCENTRATION: num[0] += w * c.S.concentration[j]; break;
                case SPHG_FIELD_PRESSURE:
                    num[0] += w * (c.S.kind[j] == Kind::Fluid ? c.S.pressure[j] : c.S.wall_pressure[j]);
                    break;
                default: num[0] += w * rho; break;
            }
        }
        const bool ok = den > 0.0;
        for (int k = 0; k < nc; ++k) out[q * nc + k] = ok ? num[k] / den : kNaN;
        if (support) support[q] = ok ? 1 : 0;
    }
    return SPHG_OK;
}

int orc_get_scale_dC(orc_ctx* h, double* dC) {
    const Ctx& c = *reinterpret_cast<Ctx*>(h);
    std::copy(c.dC_scale.begin(), c.dC_scale.end(), dC);
    return SPHG_OK;
}

int orc_set_event_log(orc_ctx* h, int enabled) {
    reinterpret_cast<Ctx*>(h)->event_log = enabled != 0;
    return SPHG_OK;
}

int orc_transition_events(orc_ctx* h, sphg_event* out, size_t cap, size_t* n) {
    Ctx& c = *reinterpret_cast<Ctx*>(h);
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

int orc_get_pscales(orc_ctx* h, double* acc, double* force) {
    const Ctx& c = *reinterpret_cast<Ctx*>(h);
    std::copy(c.acc_pscale.begin(), c.acc_pscale.end(), acc);
    std::copy(c.force_pscale.begin(), c.force_pscale.end(), force);
    return SPHG_OK;
}

int orc_get_scales(orc_ctx* h, double* acc, double* accbg, double* dT, double* force, double* rho, double* body_f,
                   double* body_t) {
    Ctx& c = *reinterpret_cast<Ctx*>(h);
    out1(acc, c.acc_scale);
    out1(accbg, c.accbg_scale);
    out1(dT, c.dT_scale);
    out1(force, c.force_scale);
    out1(rho, c.rho_scale);
    out1(body_f, c.body_fscale);
    out1(body_t, c.body_tscale);
    return SPHG_OK;
}

int orc_stats(orc_ctx* h, sphg_stats_t* s) {
    Ctx& c = *reinterpret_cast<Ctx*>(h);
    std::memset(s, 0, sizeof(*s));
    s->steps = c.steps;
    s->rebuilds = c.rebuilds;
    int64_t np = 0;
    int mx = 0;
    for (auto& l : c.nl) { np += (int64_t)l.size(); mx = std::max(mx, (int)l.size()); }
    s->n_pairs_candidate = np;
    s->max_neighbours = mx;
    s->transitions_melt = c.n_melt;
    s->transitions_solidify = c.n_solid;
    for (auto& b : c.bodies) s->bodies_alive += b.alive ? 1 : 0;
    for (int a = 0; a < 3; ++a) s->cells[a] = c.ncell[a];
    s->time = c.t;
    s->max_displacement = c.max_disp;
    s->u_max = c.u_max;
    s->dt_violations = c.dt_violations;
    s->dt_term = c.dt_term;
    s->dt_limit = c.dt_limit;
    return SPHG_OK;
}

// ---------------- decomposition primitives (sphg.h): oracle records, host buffers
int orc_halo_doubles(int phase) {
    return phase == SPHG_HALO_STATE ? 14 : phase == SPHG_HALO_DENSITY ? 4 : phase == SPHG_HALO_WALL ? 6 : -1;
}

int orc_halo_set(orc_ctx* h, int slot, const uint32_t* ids, size_t n) {
    Ctx& c = *reinterpret_cast<Ctx*>(h);
    if (slot < 0 || slot >= SPHG_MAX_HALO_SLOTS) return SPHG_ERR_CONFIG;
    for (size_t k = 0; k < n; ++k)
        if (ids[k] >= c.S.size()) return SPHG_ERR_CONFIG;
    c.halo[slot].assign(ids, ids + n);
    return SPHG_OK;
}

int orc_halo_pack(orc_ctx* h, int phase, int slot, double* buf) {
    Ctx& c = *reinterpret_cast<Ctx*>(h);
    const auto& ids = c.halo[slot];
    const int d = orc_halo_doubles(phase);
    if (d < 0) return SPHG_ERR_CONFIG;
    for (size_t s = 0; s < ids.size(); ++s) {
        const size_t i = ids[s];
        double* o = buf + s * d;
        if (phase == SPHG_HALO_STATE) {
            put3(o, c.S.pos[i]);
            put3(o + 3, c.S.vel[i]);
            put3(o + 6, c.S.vel_adv[i]);
            put3(o + 9, c.S.wall_velocity[i]);
            o[12] = c.S.temperature[i];
            o[13] = c.S.concentration[i];
        } else if (phase == SPHG_HALO_DENSITY) {
            o[0] = c.S.density[i];
            o[1] = c.S.pressure[i];
            o[2] = o[3] = 0.0;
        } else {
            o[0] = c.V_w[i];
            put3(o + 1, c.S.wall_velocity[i]);
            o[4] = c.rho_w[i];
            o[5] = c.S.wall_pressure[i];
        }
    }
    return SPHG_OK;
}

int orc_halo_unpack(orc_ctx* h, int phase, int slot, const double* buf) {
    Ctx& c = *reinterpret_cast<Ctx*>(h);
    const auto& ids = c.halo[slot];
    const int d = orc_halo_doubles(phase);
    if (d < 0) return SPHG_ERR_CONFIG;
    for (size_t s = 0; s < ids.size(); ++s) {
        const size_t i = ids[s];
        const double* o = buf + s * d;
        if (phase == SPHG_HALO_STATE) {
            c.S.pos[i] = v3(o);
            c.S.vel[i] = v3(o + 3);
            c.S.vel_adv[i] = v3(o + 6);
            c.S.wall_velocity[i] = v3(o + 9);
            c.S.temperature[i] = o[12];
            c.S.concentration[i] = o[13];
        } else if (phase == SPHG_HALO_DENSITY) {
            c.S.density[i] = o[0];
            c.S.pressure[i] = o[1];
        } else {
            c.V_w[i] = o[0];
            c.S.wall_velocity[i] = v3(o + 1);
            c.rho_w[i] = o[4];
            c.S.wall_pressure[i] = o[5];
            if (c.S.kind[i] == Kind::Boundary) c.S.density[i] = o[4];
        }
    }
    return SPHG_OK;
}

// per-body Neumaier partials over owned members, in local gid order: nb x 12 x (sum, comp)
int orc_body_partials(orc_ctx* h, double* out) {
    Ctx& c = *reinterpret_cast<Ctx*>(h);
    const size_t nb = c.bodies.size();
    if (c.members.size() != nb) rebuild_members(c);
    for (size_t k = 0; k < nb; ++k) {
        const sphg_body& b = c.bodies[k];
        sphfsi::KahanSum acc[12];
        if (b.alive) {
            const sphfsi::Quaternion q = qof(b);
            for (uint32_t r : c.members[k]) {
                const V3 rk = sphfsi::rotate(q, c.S.body_frame_pos[r]);
                const V3& f = c.force[r];
                const V3 tq = sphfsi::moment(rk, f);
                const double m = c.S.mass[r];
                const double Ir = particle_inertia(m, c.P.dx);
                const double d2 = r2of(rk);
                for (int a = 0; a < 3; ++a) {
                    acc[a].add(f[a]);
                    acc[3 + a].add(tq[a]);
                }
                acc[6].add(Ir + m * (d2 - rk[0] * rk[0]));
                acc[7].add(Ir + m * (d2 - rk[1] * rk[1]));
                acc[8].add(Ir + m * (d2 - rk[2] * rk[2]));
                acc[9].add(-m * rk[0] * rk[1]);
                acc[10].add(-m * rk[0] * rk[2]);
                acc[11].add(-m * rk[1] * rk[2]);
            }
        }
        for (int q6 = 0; q6 < 12; ++q6) {
            out[k * 24 + 2 * q6] = acc[q6].sum;
            out[k * 24 + 2 * q6 + 1] = acc[q6].comp;
        }
    }
    return SPHG_OK;
}

int orc_body_apply_totals(orc_ctx* h, const double* tot) {
    Ctx& c = *reinterpret_cast<Ctx*>(h);
    for (size_t k = 0; k < c.bodies.size(); ++k) {
        sphg_body& b = c.bodies[k];
        if (!b.alive) continue;
        const double* v = tot + k * 12;
        const V3 f{v[0], v[1], v[2]}, t{v[3], v[4], v[5]};
        put3(b.force, f);
        put3(b.torque, t);
        for (int q6 = 0; q6 < 6; ++q6) b.inertia[q6] = v[6 + q6];
        if (b.mobile && b.mass > 0.0) {
            put3(b.acc, f / b.mass + v3(c.P.mat[b.material].body_force));
            V3 al;
            bool sing;
            inverse_apply(b.inertia, t, al, sing);
            put3(b.alpha, al);
        } else {
            put3(b.acc, V3::zero());
            put3(b.alpha, V3::zero());
        }
    }
    return SPHG_OK;
}

// ---- in-library decomposed step (sphg.h), the oracle's restatement of api.cu one_step_decomposed:
// the same stage order, exchange points and rank-order TwoSum merge of the body partials (host buffers)
int orc_set_exchange(orc_ctx* h, sphg_exchange_fn fn, void* user) {
    Ctx& c = *reinterpret_cast<Ctx*>(h);
    c.exch_fn = fn;
    c.exch_user = user;
    return SPHG_OK;
}
int orc_get_stream(orc_ctx*, void** stream) {
    *stream = nullptr;
    return SPHG_OK;
}
int orc_halo_bind(orc_ctx* h, int phase, int slot, double* buf) {
    if (phase < 0 || phase > 2 || slot < 0 || slot >= SPHG_MAX_HALO_SLOTS) return SPHG_ERR_CONFIG;
    reinterpret_cast<Ctx*>(h)->halo_buf[phase][slot] = buf;
    return SPHG_OK;
}
int orc_max_bind(orc_ctx* h, uint64_t* words) {
    reinterpret_cast<Ctx*>(h)->max_words = words;
    return SPHG_OK;
}
int orc_body_bind(orc_ctx* h, double* part, double* gath, int32_t world) {
    if (world < 1) return SPHG_ERR_CONFIG;
    Ctx& c = *reinterpret_cast<Ctx*>(h);
    c.body_part = part;
    c.body_gath = gath;
    c.world = world;
    return SPHG_OK;
}
int orc_set_partition_limit(orc_ctx* h, double limit) {
    reinterpret_cast<Ctx*>(h)->partition_limit = limit;
    return SPHG_OK;
}
int orc_counters(orc_ctx* h, int64_t out[4]) {
    const Ctx& c = *reinterpret_cast<Ctx*>(h);
    out[0] = c.steps;
    out[1] = c.rebuilds;
    out[2] = 0;
    out[3] = 0;
    return SPHG_OK;
}
int orc_drift(orc_ctx* h, double out[3]) {
    const Ctx& c = *reinterpret_cast<Ctx*>(h);
    out[0] = c.max_disp;
    out[1] = c.disp_since_partition;
    out[2] = c.u_max;
    return SPHG_OK;
}

static int xchg(Ctx& c, int phase) {
    if (c.exch_fn(phase, nullptr, c.exch_user)) {
        c.err = "exchange callback failed in phase " + std::to_string(phase);
        return SPHG_ERR_CUDA;
    }
    return SPHG_OK;
}

static int halo_xchg(orc_ctx* h, int phase) {
    Ctx& c = *reinterpret_cast<Ctx*>(h);
    for (int slot = 0; slot < SPHG_MAX_HALO_SLOTS; slot += 2)
        if (!c.halo[slot].empty()) {
            if (!c.halo_buf[phase][slot]) return SPHG_ERR_CONFIG;
            orc_halo_pack(h, phase, slot, c.halo_buf[phase][slot]);
        }
    const int rc = xchg(c, phase);
    if (rc) return rc;
    for (int slot = 1; slot < SPHG_MAX_HALO_SLOTS; slot += 2)
        if (!c.halo[slot].empty()) {
            if (!c.halo_buf[phase][slot]) return SPHG_ERR_CONFIG;
            orc_halo_unpack(h, phase, slot, c.halo_buf[phase][slot]);
        }
    return SPHG_OK;
}

int decomposed_step(orc_ctx* h) {
    Ctx& c = *reinterpret_cast<Ctx*>(h);
    if (!c.max_words) return SPHG_ERR_CONFIG;
    const bool ok = stage_kick_drift(c);
    // global max displacement and speed (a local error travels as +inf)
    const double d2 = ok ? c.max_disp * c.max_disp : std::numeric_limits<double>::infinity();
    const double u2 = c.u_max * c.u_max;
    std::memcpy(&c.max_words[0], &d2, 8);
    std::memcpy(&c.max_words[1], &u2, 8);
    int rc = xchg(c, SPHG_XCHG_MAX);
    if (rc) return rc;
    double gd2, gu2;
    std::memcpy(&gd2, &c.max_words[0], 8);
    std::memcpy(&gu2, &c.max_words[1], 8);
    if (!ok) return SPHG_ERR_RUNTIME;
    if (std::isinf(gd2)) {
        c.err = "runtime assertion on another rank at step " + std::to_string(c.steps + 1);
        return SPHG_ERR_RUNTIME;
    }
    c.max_disp = std::sqrt(gd2);
    c.u_max = std::sqrt(gu2);
    if ((rc = halo_xchg(h, SPHG_HALO_STATE))) return rc;
    const double half_skin = 0.5 * (c.rv - c.rc);
    if (!c.built || c.max_disp > half_skin) {  // SPEC:212, rank-local
        c.disp_since_partition += c.max_disp;
        if (!stage_rebuild(c)) return SPHG_ERR_RUNTIME;
    }
    if (!stage_density(c)) return SPHG_ERR_RUNTIME;
    if ((rc = halo_xchg(h, SPHG_HALO_DENSITY))) return rc;
    if (c.P.thermal && !stage_heat(c)) return SPHG_ERR_RUNTIME;
    if (c.P.diffusion && !stage_diffusion(c)) return SPHG_ERR_RUNTIME;
    if (!stage_extrapolate(c)) return SPHG_ERR_RUNTIME;
    if ((rc = halo_xchg(h, SPHG_HALO_WALL))) return rc;
    if (!stage_forces(c)) return SPHG_ERR_RUNTIME;
    const size_t nb = c.bodies.size();
    if (nb) {
        if (!c.body_part || !c.body_gath) return SPHG_ERR_CONFIG;
        orc_body_partials(h, c.body_part);
        if ((rc = xchg(c, SPHG_XCHG_BODIES))) return rc;
        std::vector<double> tot(nb * 12);
        for (size_t q = 0; q < nb * 12; ++q) {  // rank-order TwoSum (parallel._merge_partials)
            double sm = c.body_gath[2 * q], cp = c.body_gath[2 * q + 1];
            for (int r = 1; r < c.world; ++r) {
                const double s2 = c.body_gath[(size_t)r * nb * 24 + 2 * q], c2 = c.body_gath[(size_t)r * nb * 24 + 2 * q + 1];
                const double t = sm + s2, bp = t - sm, e = (sm - (t - bp)) + (s2 - bp);
                cp = (cp + c2) + e;
                sm = t;
            }
            tot[q] = sm + cp;
        }
        orc_body_apply_totals(h, tot.data());
    }
    if (!stage_final_kick(c)) return SPHG_ERR_RUNTIME;
    c.steps++;
    if (!check_dt(c)) return SPHG_ERR_RUNTIME;
    if (c.P.transitions) {  // owned detection + global counts (api.cu one_step_decomposed)
        std::vector<uint32_t> melt, solid;
        detect_events(c, melt, solid);
        c.ev.assign(c.S.size(), 0);
        for (uint32_t i : melt) c.ev[i] = 1;
        for (uint32_t i : solid) c.ev[i] = 2;
        c.max_words[0] = melt.size();
        c.max_words[1] = solid.size();
        if ((rc = xchg(c, SPHG_XCHG_MAX))) return rc;
        if (c.max_words[0] || c.max_words[1]) return SPHG_NEED_TRANSITIONS;
    }
    return SPHG_OK;
}

// ---- decomposed transition batches (sphg.h sphg_event_* / sphg_record_*), the oracle's records
int orc_event_bodies(orc_ctx* h, uint8_t* mask, size_t nb) {
    Ctx& c = *reinterpret_cast<Ctx*>(h);
    if (nb != c.bodies.size()) return SPHG_ERR_CONFIG;
    const double rc2 = c.rc * c.rc;
    for (size_t i = 0; i < c.ev.size() && i < c.S.size(); ++i) {
        if (c.ev[i] == 1) mask[c.S.group[i]] = 1;
        if (c.ev[i] != 2) continue;
        for (uint32_t j : c.nl[i])
            if (c.S.kind[j] == Kind::Rigid && r2of(mi3(c, c.S.pos[i], c.S.pos[j])) <= rc2) mask[c.S.group[j]] = 1;
    }
    return SPHG_OK;
}

int orc_event_members(orc_ctx* h, const uint8_t* mask, size_t nb, uint32_t* ids, size_t cap, size_t* n) {
    Ctx& c = *reinterpret_cast<Ctx*>(h);
    if (nb != c.bodies.size()) return SPHG_ERR_CONFIG;
    std::vector<uint32_t> out;
    for (size_t i = 0; i < c.S.size(); ++i) {
        if (ghost(c, i)) continue;
        const bool ev = i < c.ev.size() && c.ev[i] != 0;
        const bool member = c.S.kind[i] == Kind::Rigid && c.S.group[i] < nb && mask[c.S.group[i]];
        if (ev || member) out.push_back((uint32_t)i);
    }
    *n = out.size();
    if (!ids) return SPHG_OK;
    if (cap < out.size()) return SPHG_ERR_CONFIG;
    std::copy(out.begin(), out.end(), ids);
    return SPHG_OK;
}

constexpr int kOrcRecord = 40;
int orc_record_doubles(void) { return kOrcRecord; }

int orc_record_pack(orc_ctx* h, const uint32_t* ids, size_t m, double* recs) {
    Ctx& c = *reinterpret_cast<Ctx*>(h);
    auto& S = c.S;
    for (size_t s = 0; s < m; ++s) {
        const size_t i = ids[s];
        if (i >= S.size()) return SPHG_ERR_CONFIG;
        double* o = recs + s * kOrcRecord;
        put3(o, S.pos[i]);
        o[3] = (double)static_cast<int>(S.kind[i]);
        o[4] = (double)S.material[i];
        o[5] = (double)S.group[i];
        o[6] = S.mass[i];
        put3(o + 7, S.vel[i]);
        put3(o + 10, S.vel_adv[i]);
        put3(o + 13, S.acc[i]);
        put3(o + 16, S.acc_bg[i]);
        o[19] = S.density[i];
        o[20] = S.pressure[i];
        o[21] = S.temperature[i];
        o[22] = S.dT_dt[i];
        o[23] = S.concentration[i];
        o[24] = S.dC_dt[i];
        put3(o + 25, S.body_frame_pos[i]);
        o[28] = S.wall_pressure[i];
        put3(o + 29, S.wall_velocity[i]);
        o[32] = S.dirichlet_T[i];
        o[33] = S.dirichlet_C[i];
        put3(o + 34, c.force[i]);
        o[37] = c.rho_w[i];
        o[38] = c.V_w[i];
        o[39] = c.wall_mat[i];
    }
    return SPHG_OK;
}

int orc_record_unpack(orc_ctx* h, const uint32_t* ids, size_t m, const double* recs, int keep_position) {
    Ctx& c = *reinterpret_cast<Ctx*>(h);
    auto& S = c.S;
    for (size_t s = 0; s < m; ++s) {
        const size_t i = ids[s];
        if (i >= S.size()) return SPHG_ERR_CONFIG;
        const double* o = recs + s * kOrcRecord;
        if (!keep_position) S.pos[i] = v3(o);
        S.kind[i] = static_cast<Kind>((int)o[3]);
        S.material[i] = (uint16_t)o[4];
        S.group[i] = (uint32_t)o[5];
        S.mass[i] = o[6];
        S.vel[i] = v3(o + 7);
        S.vel_adv[i] = v3(o + 10);
        S.acc[i] = v3(o + 13);
        S.acc_bg[i] = v3(o + 16);
        S.density[i] = o[19];
        S.pressure[i] = o[20];
        S.temperature[i] = o[21];
        S.dT_dt[i] = o[22];
        S.concentration[i] = o[23];
        S.dC_dt[i] = o[24];
        S.body_frame_pos[i] = v3(o + 25);
        S.wall_pressure[i] = o[28];
        S.wall_velocity[i] = v3(o + 29);
        S.dirichlet_T[i] = (uint8_t)o[32];
        S.dirichlet_C[i] = (uint8_t)o[33];
        c.force[i] = v3(o + 34);
        c.rho_w[i] = o[37];
        c.V_w[i] = o[38];
        c.wall_mat[i] = (int)o[39];
    }
    return SPHG_OK;
}

// sphg_upload_records: the whole store from records (first n_owned owned), host pointers
int orc_upload_records(orc_ctx* h, size_t n, size_t n_owned, const double* recs, const sphg_body* bodies, size_t nb) {
    Ctx& c = *reinterpret_cast<Ctx*>(h);
    if (n_owned > n) return SPHG_ERR_CONFIG;
    auto& S = c.S;
    S.pos.assign(n, V3::zero()); S.vel.assign(n, V3::zero()); S.vel_adv.assign(n, V3::zero());
    S.acc.assign(n, V3::zero()); S.acc_bg.assign(n, V3::zero());
    S.density.assign(n, 0.0); S.pressure.assign(n, 0.0); S.mass.assign(n, 0.0);
    S.temperature.assign(n, 0.0); S.dT_dt.assign(n, 0.0); S.concentration.assign(n, 0.0); S.dC_dt.assign(n, 0.0);
    S.kind.assign(n, Kind::Fluid); S.group.assign(n, 0u); S.material.assign(n, (uint16_t)0);
    S.body_frame_pos.assign(n, V3::zero()); S.wall_pressure.assign(n, 0.0); S.wall_velocity.assign(n, V3::zero());
    S.dirichlet_T.assign(n, (uint8_t)0xff); S.dirichlet_C.assign(n, (uint8_t)0xff);
    S.owner.assign(n, (uint32_t)c.P.rank);
    for (size_t i = n_owned; i < n; ++i) S.owner[i] = 0xffffffffu;
    resize_aux(c);
    std::vector<uint32_t> ids(n);
    std::iota(ids.begin(), ids.end(), 0u);
    const int rc = orc_record_unpack(h, ids.data(), n, recs, 0);
    if (rc) return rc;
    c.halo.assign(SPHG_MAX_HALO_SLOTS, {});
    c.has_ghosts = n_owned < n;
    c.disp_since_partition = 0.0;
    c.bodies.assign(bodies, bodies + nb);
    c.body_fscale.assign(nb, 0.0);
    c.body_tscale.assign(nb, 0.0);
    rebuild_members(c);
    c.ev.clear();
    c.built = false;
    return SPHG_OK;
}

int orc_replace_bodies(orc_ctx* h, const sphg_body* bodies, size_t nb) {
    Ctx& c = *reinterpret_cast<Ctx*>(h);
    c.bodies.assign(bodies, bodies + nb);
    c.body_fscale.resize(nb, 0.0);
    c.body_tscale.resize(nb, 0.0);
    rebuild_members(c);
    return SPHG_OK;
}

int orc_max_displacement(orc_ctx* h, double* out) {
    *out = reinterpret_cast<Ctx*>(h)->max_disp;
    return SPHG_OK;
}

const char* orc_last_error(const orc_ctx* h) { return reinterpret_cast<const Ctx*>(h)->err.c_str(); }
void orc_destroy(orc_ctx* h) { delete reinterpret_cast<Ctx*>(h); }

// ---------------- KAT helpers: the reference's own building blocks, unchanged
double orc_kernel_w(double h, double r) { return sphfsi::QuinticKernel<3>(h).w(r); }
double orc_kernel_dw(double h, double r) { return sphfsi::QuinticKernel<3>(h).dw_dr(r); }
double orc_kernel_sigma(double h) { return sphfsi::QuinticKernel<3>::sigma(h); }
double orc_eos_pressure(double rho, double rho0, double c) {
    sphfsi::Material m;
    m.reference_density = rho0;
    m.speed_of_sound = c;
    return sphfsi::eos_pressure(rho, m);
}
void orc_orientation_step(const double q[4], const double w[3], double dt, double out[4]) {
    const sphfsi::Quaternion r = sphfsi::orientation_step<3>({q[0], q[1], q[2], q[3]}, V3{w[0], w[1], w[2]}, dt);
    out[0] = r.w; out[1] = r.x; out[2] = r.y; out[3] = r.z;
}
void orc_rotate(const double q[4], const double v[3], double out[3]) {
    put3(out, sphfsi::rotate({q[0], q[1], q[2], q[3]}, V3{v[0], v[1], v[2]}));
}
double orc_kahan_sum(const double* x, size_t n) {
    sphfsi::KahanSum s;
    for (size_t i = 0; i < n; ++i) s.add(x[i]);
    return s.value();
}
double orc_particle_inertia(double m, double dx) { return particle_inertia(m, dx); }
// lattice.hpp seed_lattice over a box or ball; returns the count, writes up to cap points
size_t orc_seed_lattice_box(const double lo[3], const double hi[3], double dx, double* out, size_t cap) {
    sphfsi::ParticleStore<3> s;
    sphfsi::Box<3> b;
    for (int a = 0; a < 3; ++a) { b.lo[a] = lo[a]; b.hi[a] = hi[a]; }
    sphfsi::Material m;
    sphfsi::seed_lattice<3>(s, sphfsi::box_region<3>(b), dx, {Kind::Fluid, 0}, 0, m);
    for (size_t i = 0; i < s.size() && i < cap; ++i) put3(out + 3 * i, s.pos[i]);
    return s.size();
}
size_t orc_seed_lattice_ball(const double center[3], double diameter, double dx, double* out, size_t cap) {
    sphfsi::ParticleStore<3> s;
    sphfsi::Material m;
    sphfsi::seed_lattice<3>(s, sphfsi::ball_region<3>(V3{center[0], center[1], center[2]}, diameter), dx,
                            {Kind::Rigid, 0}, 0, m);
    for (size_t i = 0; i < s.size() && i < cap; ++i) put3(out + 3 * i, s.pos[i]);
    return s.size();
}
size_t orc_sizeof_params(void) { return sizeof(sphg_params); }
size_t orc_sizeof_body(void) { return sizeof(sphg_body); }
size_t orc_sizeof_soa(void) { return sizeof(sphg_soa); }

}  // extern "C"
