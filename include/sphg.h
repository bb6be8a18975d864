/*
 * sphg.h — C ABI of the B200-native SPH hot path (arXiv 2103.07925).
 *
 * This is the drop-in boundary: plain pointers and sizes, no C++ or torch
 * types.  The reference ships no hot-path code, only header building blocks
 * (/root/reference/proj/include/sphfsi, *.hpp) plus SPEC operations; each
 * entry point below names the reference interface it replaces.
 *
 *   host layout    = sphfsi::ParticleStore<3> (store.hpp:24-46): SoA, gid order,
 *                    Vec<3> fields interleaved xyz (24 B), kind u8, group u32,
 *                    material u16, dirichlet_T u8.
 *   device layout  = private, cell-sorted, packed.
 *
 * Return codes: 0 ok, 2 config violation (validate_config,
 * config.hpp:108-167), 3 runtime assertion (escaped / coincident particle,
 * NaN, neighbour-list overflow that could not be recovered), 4 CUDA/NCCL failure.
 * The message is available from sphg_last_error().  One host thread drives
 * one context; nothing is retained from caller buffers after return.
 *
 * The CPU oracle (oracle/sph_oracle.cpp, test infrastructure only) exports the
 * same entry points with the prefix `orc_` instead of `sphg_`.
 */
#ifndef SPHG_H
#define SPHG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPHG_MAX_MAT 8
#define SPHG_MAX_DIRICHLET 8
#define SPHG_MAX_PIECES 8
#define SPHG_NO_MATERIAL (-1)
#define SPHG_NO_DIRICHLET 0xff /* store.hpp:20 kNoDirichlet */

enum { SPHG_FLUID = 0, SPHG_RIGID = 1, SPHG_BOUNDARY = 2 }; /* store.hpp:11 Kind */

enum {
  SPHG_OK = 0,
  SPHG_ERR_CONFIG = 2,
  SPHG_ERR_RUNTIME = 3,
  SPHG_ERR_CUDA = 4,
  SPHG_NEED_PARTITION = 5, /* not an error: sphg_step stopped before a step its partition may not cover */
  SPHG_NEED_TRANSITIONS = 6 /* not an error: a decomposed step detected phase transitions on some rank;
                               the caller applies the batch (sphg_event_*, sphg_record_*) and steps on */
};

/* POD mirror of sphfsi::Material (material.hpp:17-36) plus the per-material
 * body force of ScenarioConfig::body_force (config.hpp:79,102-104). */
typedef struct {
  double rho0;       /* reference_density */
  double nu;         /* kinematic_viscosity; eta = rho0*nu (material.hpp:32) */
  double cp;         /* heat_capacity */
  double kappa;      /* conductivity */
  double c;          /* speed_of_sound */
  double pb;         /* background_pressure (transport velocity) */
  double T_t;        /* transition_temperature, NaN = none */
  int32_t melt_target;      /* SPHG_NO_MATERIAL = none */
  int32_t solidify_target;  /* SPHG_NO_MATERIAL = none */
  double body_force[3];
  double D;          /* diffusivity (concentration, Remark 2.3 / SPEC:407-411) */
  double C_t;        /* transition_concentration, NaN = none */
} sphg_material;

/* sphfsi::Schedule (config.hpp:20-33): value of the first piece with t <= t_end. */
typedef struct {
  int32_t n;
  int32_t pad;
  double t_end[SPHG_MAX_PIECES];
  double value[SPHG_MAX_PIECES];
} sphg_schedule;

/* Inflow / outflow buffer zone ("a buffer-zone with prescribed parabolic velocity and
 * particle recycling"; §4.4 inlet/outlet) [P23].  A FLUID particle whose position lies in
 * the zone box (lo <= x < hi on every axis) is a buffer particle: it is not accelerated by the pair
 * forces but moves with the prescribed velocity U(x, t) = e_axis u_mean f(xi) for t > t_start (0 before:
 * the zone is held at rest), f = 6 xi (1 - xi) with xi = (x_p - lo_p) / (hi_p - lo_p) along profile_axis
 * (parabolic, mean 1), or f = 1 with profile_axis = -1.  It keeps every other fluid role (density
 * summation, EOS, pair forces on its neighbours, transport velocity = U).  Roles follow the position,
 * so a particle becomes fluid when it leaves an inflow zone and a buffer particle when it enters an
 * outflow zone; with the inflow and outflow zones at the two ends of a periodic axis the periodic wrap
 * recycles outflow particles into the inflow zone (particle count and mass stay exact). */
#define SPHG_MAX_BUFFERS 4
typedef struct {
  int32_t axis;          /* flow axis 0..2 */
  int32_t profile_axis;  /* transverse axis of the parabolic profile, -1 = uniform */
  double lo[3], hi[3];   /* zone box */
  double u_mean;         /* mean velocity along the axis (signed) */
  double t_start;        /* prescribed for t > t_start; at rest before */
} sphg_buffer;

/* Flat POD derived from sphfsi::ScenarioConfig<3> (config.hpp:68-106). */
typedef struct {
  double dx;                 /* initial spacing */
  double h;                  /* smoothing length (0 = dx, config.hpp:100) */
  double dt;                 /* fixed time step (dt_override, config.hpp:85) */
  double t0;                 /* start time */
  double lo[3], hi[3];       /* domain box (must contain walls) */
  int32_t periodic[3];
  int32_t n_mat;
  double cell_edge_override; /* 0 = derive from the Verlet radius */
  sphg_material mat[SPHG_MAX_MAT];
  double kc, dc;             /* contact stiffness / damping (config.hpp:81-82) */
  int32_t tvf;               /* transport_velocity (config.hpp:90) */
  int32_t thermal;           /* solve the heat equation */
  int32_t transitions;       /* TransitionMode (config.hpp:61): 0 none, 1 temperature, 2 concentration */
  int32_t n_dirichlet;
  sphg_schedule dirichlet_T[SPHG_MAX_DIRICHLET]; /* config.hpp:94 */
  int32_t default_fluid_mat; /* EOS used for wall density when a wall has no fluid support */
  int32_t nlist_capacity;    /* 0 = auto; grown on overflow */
  int32_t rank, nranks;      /* domain decomposition (1 rank: 0,1) */
  int32_t diffusion;         /* solve the concentration diffusion equation */
  int32_t n_dirichlet_c;
  sphg_schedule dirichlet_C[SPHG_MAX_DIRICHLET]; /* config.hpp:95, indexed by dirichlet_C group */
  /* Moving Gaussian surface heat flux (BASELINE configs[3], C4).  An extension: the reference has no
   * heat sources, so this term is pinned here, not by the reference [P21]:
   *   q(x, y, t) = 2 P / (pi r0^2) exp(-2 rho^2 / r0^2),  rho^2 = (x - c_x(t))^2 + (y - c_y(t))^2,
   *   c(t) = hs_origin + hs_velocity t (wrapped, minimum image on periodic axes), q = 0 for rho > 4 r0,
   * absorbed at t^{n+1} by every exposed non-boundary particle a of a material in hs_material_mask:
   *   dT_a/dt += q(x_a, y_a) dx^2 / (m_a c_p,a)   (c_p,a > 0),
   * where a is exposed unless a Verlet neighbour b of a mask material (any kind) with r_ab <= r_c
   * lies above it: z_b - z_a > dx/2 and (x_b - x_a)^2 + (y_b - y_a)^2 < (3 dx/4)^2. */
  int32_t heat_source;          /* 0 = none (requires thermal) */
  uint32_t hs_material_mask;    /* bit m: material m absorbs / shadows */
  double hs_power;              /* absorbed power P [W] */
  double hs_radius;             /* 1/e^2 radius r0 [m] */
  double hs_origin[3];          /* spot centre at t = 0 (z unused) */
  double hs_velocity[3];        /* scan velocity (z unused) */
  /* Runtime time-step assertion: after every step the five compute_dt
   * limits are evaluated with that step's u_max (max |u^{n+1/2}| of fluid particles, from the kick)
   * and m_r = the smallest mass a rigid particle can have in the run (rigid particles, plus fluid
   * particles of a material with a solidify target when transitions are on; fixed at upload) [P22].
   * dt above the smallest limit: SPHG_DT_REFUSE returns SPHG_ERR_RUNTIME naming the violated
   * condition (the step itself completes); SPHG_DT_WARN counts it in the stats (SURVEY App. A15:
   * BASELINE C1/C5 prescribe a dt above the contact limit); SPHG_DT_OFF skips the check. */
  int32_t dt_check;
  int32_t n_buffers;             /* inflow / outflow buffer zones (sphg_buffer, [P23]) */
  sphg_buffer buffers[SPHG_MAX_BUFFERS];
} sphg_params;

enum { SPHG_DT_REFUSE = 0, SPHG_DT_WARN = 1, SPHG_DT_OFF = 2 };

/* Host SoA views in gid order — the ParticleStore<3> layout (store.hpp:26-46).
 * Vec<3> fields are 3*n doubles, interleaved xyz.  `force` is an optional
 * extension (resultant f_r on rigid particles); may be NULL. */
typedef struct {
  size_t n;
  double *pos, *vel, *vel_adv, *acc, *acc_bg;
  double *density, *pressure, *mass, *temperature, *dT_dt;
  uint8_t *kind;
  uint32_t *group;
  uint16_t *material;
  double *body_frame_pos;
  double *wall_pressure;
  double *wall_velocity;
  uint8_t *dirichlet_T;
  double *force;
  uint32_t *owner;   /* owning rank (store.hpp:46); != params.rank marks a ghost copy; NULL = all owned */
  double *concentration, *dC_dt; /* store.hpp:36-37 */
  uint8_t *dirichlet_C;          /* store.hpp:45: concentration schedule group or SPHG_NO_DIRICHLET */
} sphg_soa;

/* RigidBody.  inertia = world frame about com: xx yy zz xy xz yz. */
typedef struct {
  double mass;
  double com[3];
  double inertia[6];
  double q[4];        /* quaternion w x y z (quaternion.hpp:10-15) */
  double vel[3];
  double omega[3];
  double force[3];
  double torque[3];
  double acc[3];      /* a_k = f_k/m_k + b_k */
  double alpha[3];    /* I_k^{-1} torque */
  int32_t material;
  int32_t mobile;
  int32_t alive;
  int32_t pad;
} sphg_body;

/* Stages of one kick-drift-kick step.  A full step
 * is KICK_DRIFT, REBUILD (if the Verlet trigger fired), DENSITY, HEAT,
 * EXTRAPOLATE, FORCES, BODIES, FINAL_KICK, TRANSITIONS. */
enum {
  SPHG_STAGE_REBUILD = 0,     /* cell keys + radix sort + reorder + neighbour list */
  SPHG_STAGE_DENSITY = 1,     /* density_summation + eos_pressure */
  SPHG_STAGE_HEAT = 2,        /* apply_thermal_dirichlet + conduction_rhs + T update;
                                 with params.diffusion also diffusion_rhs + C update */
  SPHG_STAGE_EXTRAPOLATE = 3, /* extrapolate_wall_quantities */
  SPHG_STAGE_FORCES = 4,      /* momentum_rhs + coupling_force_on_rigid + contact_force */
  SPHG_STAGE_BODIES = 5,      /* reduce_force_torque -> a_k, alpha_k */
  SPHG_STAGE_KICK_DRIFT = 6,  /* half kick, drift, orientation, slave positions */
  SPHG_STAGE_FINAL_KICK = 7,  /* final half kick + slave velocities */
  SPHG_STAGE_TRANSITIONS = 8, /* detect + apply transitions */
  SPHG_STAGE_MASS = 9         /* reduce_mass_quantities for every live body */
};

typedef struct {
  int64_t steps;
  int64_t rebuilds;
  int64_t n_pairs_candidate;  /* at the last rebuild */
  int64_t transitions_melt;
  int64_t transitions_solidify;
  int64_t bodies_alive;
  int32_t nlist_capacity;
  int32_t max_neighbours;
  int32_t cells[3];
  int32_t pad;
  double time;
  double max_displacement;    /* since the last rebuild */
  double u_max;               /* max |u| of fluid particles at the last kick */
  double stage_ms[16];        /* accumulated device time per stage (if timing enabled);
                                 10 = fluid forces kernel, 11 = rigid forces kernel (both inside 4) */
  int64_t kernel_launches;
  double last_step_call_ms;   /* device time of the last sphg_step call (CUDA events on the stream) */
  int64_t graph_captures;     /* CUDA graphs captured for the per-step launch chains (SPHG_GRAPHS=0: none) */
  int64_t graph_replays;      /* chain launches served by an already captured graph */
  int64_t dt_violations;      /* steps whose dt exceeded a compute_dt limit (runtime assertion, SPHG_DT_WARN) */
  int64_t host_syncs;         /* host-blocking waits on the device since creation (stream / event syncs) */
  int32_t dt_term;            /* the most restrictive limit at the last check: 0 cfl, 1 viscous, 2 body force,
                                 3 contact, 4 conduction (-1: none checked) */
  int32_t pad3;
  double dt_limit;            /* its value */
} sphg_stats_t;

typedef struct sphg_ctx sphg_ctx;

/* validate_config (config.hpp:110-167) + device setup.  2 = config violation. */
int sphg_create(const sphg_params* params, int device, sphg_ctx** out);
/* Copies a ParticleStore<3> + body table to the device (caller keeps ownership). */
int sphg_upload(sphg_ctx* ctx, const sphg_soa* soa, const sphg_body* bodies, size_t n_bodies);
/* a^0 for the first kick: REBUILD, DENSITY, EXTRAPOLATE, FORCES, BODIES. */
int sphg_initialize(sphg_ctx* ctx);
/* nsteps full KDK steps, stream-ordered. */
int sphg_step(sphg_ctx* ctx, int nsteps);
/* nsteps steps, then the requested store fields (and, with nb_io, the body table) in gid order, as
 * sphg_step followed by sphg_download — the snapshot step of the reference's run loop.
 * With transitions off, the fields that are final after the last step's wall extrapolation
 * (pos, density, pressure, wall_pressure, wall_velocity, mass, body_frame_pos and the tags) cross
 * PCIe on a second stream while that step's force kernels run; the rest after the final kick. */
int sphg_step_download(sphg_ctx* ctx, int nsteps, sphg_soa* out, sphg_body* bodies_out, size_t* n_bodies_inout);
/* One stage (parity hook; also the per-op evaluator API of SPEC:243-363). */
int sphg_run_stage(sphg_ctx* ctx, int stage);
/* Warm kinematic update between steps (same store, gid order): positions and velocities only,
 * e.g. a host-side coupling that moves particles.  Keeps the device order and the Verlet rows
 * (rebuilt automatically if the update moved a particle beyond the skin). */
int sphg_upload_state(sphg_ctx* ctx, const double* pos, const double* vel, size_t n);
/* Copies the state back in gid order into caller-allocated buffers (NULL fields skipped; only the
 * device arrays behind the requested fields cross PCIe). */
int sphg_download(sphg_ctx* ctx, sphg_soa* out, sphg_body* bodies_out, size_t* n_bodies_inout);
/* Cell of every particle (by gid) and the canonical (cell, gid) order. */
int sphg_get_cells(sphg_ctx* ctx, int64_t* cell_of_gid, uint32_t* sorted_gid);
/* Verlet candidate lists in CSR, by gid, each list sorted by gid.  Call with
 * nbr_gid == NULL to get offsets only (offsets has n+1 entries). */
int sphg_get_nlist(sphg_ctx* ctx, int64_t* offsets, uint32_t* nbr_gid);
int sphg_stats(sphg_ctx* ctx, sphg_stats_t* out);
/* Enables per-stage CUDA-event timing (adds event records; off by default). */
int sphg_set_timing(sphg_ctx* ctx, int enabled);
/* Number of bodies in the device table (live or dead). */
int sphg_num_bodies(sphg_ctx* ctx, size_t* n_bodies);
/* compute_dt terms: cfl, viscous, body force, contact, conduction; +inf = absent. */
int sphg_compute_dt(sphg_ctx* ctx, double limits[5]);
/* The five limits of compute_dt without a context (pure host function):
 * u_max = max fluid speed, m_r = smallest rigid particle mass (<= 0: no contact term). */
int sphg_dt_limits(const sphg_params* params, double u_max, double m_r, double limits[5]);
/* Pair counts of the current Verlet list: [0] candidates, [1] within r_c (interacting),
 * [2] interacting with a fluid particle i (the fluid force kernel's pairs), [3] with a non-fluid i. */
int sphg_count_pairs(sphg_ctx* ctx, int64_t counts[4]);

/* Moving wall groups: WallGroup<3>::velocity_at / acceleration_at (config.hpp:35-51), SPEC:237,
 * 273, 278.  Boundary particles whose `group` is g < n_groups belong to wall group g.  Each step
 * the library calls fn(g, t^{n+1/2}, vel, acc, user) for the drift (r += dt vel; acc unused) and
 * fn(g, t^{n+1}, vel, acc, user) for the wall state the pair sums see at t^{n+1} (boundary
 * velocity u_w = vel, wall acceleration a_w = acc in the pressure extrapolation).  `acc` is
 * pre-filled with the reference's default, the central difference (v(t+1e-6) - v(t-1e-6))/2e-6;
 * the callee may overwrite it.  fn = NULL (default) = fixed walls.  n_groups <= SPHG_MAX_WALL_GROUPS. */
#define SPHG_MAX_WALL_GROUPS 8
typedef void (*sphg_wall_motion_fn)(int32_t group, double t, double vel[3], double acc[3], void* user);
int sphg_set_wall_motion(sphg_ctx* ctx, int32_t n_groups, sphg_wall_motion_fn fn, void* user);

/* shepard_interpolate (the Shepard filter used for every field
 * figure) on a regular grid, the post-processing gather behind OutputPlan::shepard_grid
 * (config.hpp:53-59):
 *   f^(x) = sum_j V_j f_j W(|x - r_j|, h) / sum_j V_j W(|x - r_j|, h),  V_j = m_j / rho_j
 * over the particles whose kind bit is set in kind_mask (1 << SPHG_FLUID | ...), minimum image on
 * periodic axes.  Grid point (a, b, c) = origin + (a, b, c) * spacing, stored z fastest:
 * out[((a * dims[1] + b) * dims[2] + c) * ncomp + comp].  A point with no particle within r_c
 * gets NaN and support = 0 ("no support" signal); support may be NULL. */
enum {
  SPHG_FIELD_VELOCITY = 0,      /* 3 components */
  SPHG_FIELD_TEMPERATURE = 1,
  SPHG_FIELD_CONCENTRATION = 2,
  SPHG_FIELD_PRESSURE = 3,
  SPHG_FIELD_DENSITY = 4
};
int sphg_shepard_grid(sphg_ctx* ctx, const double origin[3], const double spacing[3], const int32_t dims[3],
                      int32_t field, uint32_t kind_mask, double* out, uint8_t* support);
/* ---- domain decomposition primitives (one context per rank).
 * The host layer (paper_2103_07925_b200/parallel.py) owns the exchange; these move data between the
 * context and contiguous halo records.  Ghosts are the uploaded particles with owner != rank: they are
 * read by the pair kernels, never integrated, and refreshed by halo unpacks.  Index lists are local ids
 * (positions in the uploaded store); buffers are device pointers for sphg_ (host pointers for orc_). */
#define SPHG_MAX_HALO_SLOTS 64
enum { SPHG_HALO_STATE = 0,    /* after the drift: pos, u_int, du, vel, T, C        (14 doubles) */
       SPHG_HALO_DENSITY = 1,  /* after density: V^2, rho, p, V_heat                (4 doubles)  */
       SPHG_HALO_WALL = 2 };   /* after extrapolation: V_w^2, u~_w, rho_w, p_w      (6 doubles)  */
int sphg_halo_doubles(int phase);
int sphg_halo_set(sphg_ctx* ctx, int slot, const uint32_t* local_ids, size_t n);
int sphg_halo_pack(sphg_ctx* ctx, int phase, int slot, double* buf);
int sphg_halo_unpack(sphg_ctx* ctx, int phase, int slot, const double* buf);
/* In-library decomposed step (bulk-synchronous).  With ghosts present and an
 * exchange callback set, sphg_step(ctx, K) runs the whole decomposed step on the library's stream:
 * kick / drift, MAX exchange (global max displacement and u_max), one flag readback (the Verlet
 * decision and error check), STATE halo (the interior density runs meanwhile on a second stream),
 * [rank-local rebuild], boundary density, DENSITY halo, [heat], extrapolation, WALL halo, forces, body
 * partials -> BODIES all-gather -> rank-order TwoSum merge on the device, final kick.  At each exchange
 * point the library has packed the bound send buffers on `stream` and calls fn(phase, stream, user);
 * fn enqueues the transfers so that, in the order of `stream`, the bound receive buffers (the MAX words,
 * the body gather buffer) hold the peers' data before any later work on it (NCCL through
 * torch.distributed on an external stream does this without blocking the host).  Halo slots as
 * sphg_halo_set: per peer k, send slot 2k and receive slot 2k+1. */
enum { SPHG_XCHG_MAX = 3, SPHG_XCHG_BODIES = 4 };
typedef int (*sphg_exchange_fn)(int32_t phase, void* stream, void* user);
int sphg_set_exchange(sphg_ctx* ctx, sphg_exchange_fn fn, void* user);
/* the library's cudaStream_t (as void*) */
int sphg_get_stream(sphg_ctx* ctx, void** stream);
/* device buffer of (phase, slot): halo records of sphg_halo_doubles(phase) doubles per listed particle */
int sphg_halo_bind(sphg_ctx* ctx, int phase, int slot, double* dev_buf);
/* device buffer of the two words the MAX exchange reduces in place (MAX over ranks): the squared max
 * displacement and the squared max fluid speed of this step, as the bits of non-negative doubles (so an
 * integer MAX is the double MAX; a local runtime error is sent as +inf) */
int sphg_max_bind(sphg_ctx* ctx, uint64_t* dev_words);
/* [0] global max displacement since the last rebuild, [1] sum of the global displacements at the
 * rebuilds since the last upload (with [0]: a bound on any particle's drift since it was partitioned),
 * [2] global max fluid speed of the last kick */
int sphg_drift(sphg_ctx* ctx, double out[3]);
/* decomposed runs: sphg_step returns SPHG_NEED_PARTITION before a step at which [1] + [0] + half a skin
 * of sphg_drift would exceed `limit` (the caller migrates particles, re-uploads and steps on); 0 = off */
int sphg_set_partition_limit(sphg_ctx* ctx, double limit);
/* cheap host counters: [0] steps, [1] Verlet rebuilds, [2] host-blocking syncs, [3] kernel launches */
int sphg_counters(sphg_ctx* ctx, int64_t out[4]);
/* body partials (nb x 24 doubles, as sphg_body_partials) are written to dev_partials; the BODIES exchange
 * all-gathers them into dev_gathered (world x nb x 24, rank order) */
int sphg_body_bind(sphg_ctx* ctx, double* dev_partials, double* dev_gathered, int32_t world);
/* Per-body compensated partial sums over owned rigid particles: nb x 24 doubles (12 x (sum, comp):
 * f xyz, torque xyz, inertia xx yy zz xy xz yz).  `out` / `totals` may be host or device pointers
 * (unified addressing), so an NCCL driver gathers and merges them without host staging. */
int sphg_body_partials(sphg_ctx* ctx, double* out);
/* Global per-body sums (nb x 12, merged by the caller in rank order) -> f, tau, I, a_k, alpha_k. */
int sphg_body_apply_totals(sphg_ctx* ctx, const double* totals);
/* Max displacement since the last rebuild over owned particles (after a KICK_DRIFT stage). */
int sphg_max_displacement(sphg_ctx* ctx, double* out);
/* Cell-occupancy histogram of the last Verlet rebuild ("diagnostic dump of cell occupancy histogram
 * as CSV"): hist[k] = number of cells holding k particles (owned and ghost), the last bin counting every
 * cell with >= nbins - 1; *max_count (may be NULL) = the fullest cell's count. */
int sphg_cell_occupancy(sphg_ctx* ctx, int64_t* hist, size_t nbins, int64_t* max_count);
/* Phase transitions under decomposition ("Event detection is worker-local; application is
 * serialized per affected body at the owner, followed by a broadcast of updated body state and re-linking
 * of affected particles").  With transitions on, a decomposed step ends with detection over the owned
 * particles and a MAX exchange of the event counts; when any rank has events, sphg_step returns
 * SPHG_NEED_TRANSITIONS after completing that step.  The caller then
 *   1. sphg_event_bodies: the bodies a batch can touch (bodies of melting particles, bodies with a rigid
 *      particle within r_c of a solidifying one, ghosts included), OR-ed over ranks;
 *   2. sphg_event_members: the owned event particles and owned members of those bodies (local ids);
 *   3. sphg_record_pack of them, gathered at one rank, which uploads them (global gid order) into a
 *      single-rank context, applies the batch there with the single-rank kernels (sphg_run_stage
 *      TRANSITIONS: the sub-store holds every particle the batch reads) and broadcasts the records
 *      and the new body table;
 *   4. sphg_record_unpack (keep_position = 1) of every listed particle present on the rank (owned or
 *      ghost) and sphg_replace_bodies, then the body force/torque of the new membership (body partials).
 * Records are sphg_record_doubles() doubles: [0..2] position, [3] kind, [4] material, [5] group,
 * [6] mass, then the engine's own per-particle state (opaque; only the same engine reads it back).
 * `mask` holds n_bodies bytes; ids are local ids in ascending order; record buffers and their id lists may
 * be host or device memory. */
int sphg_event_bodies(sphg_ctx* ctx, uint8_t* mask, size_t n_bodies);
int sphg_event_members(sphg_ctx* ctx, const uint8_t* mask, size_t n_bodies, uint32_t* ids, size_t cap, size_t* n);
int sphg_record_doubles(void);
int sphg_record_pack(sphg_ctx* ctx, const uint32_t* ids, size_t m, double* recs);
/* keep_position = 1: the local copy keeps its coordinates (ghosts may be unwrapped across a periodic face)
 * and its ghost/owned role; 0: the record's position is written too (the single-rank batch context) */
int sphg_record_unpack(sphg_ctx* ctx, const uint32_t* ids, size_t m, const double* recs, int keep_position);
/* Replaces the whole store with n records (the first n_owned owned, the rest ghosts; local ids = record
 * order) and the body table: the device-resident migration of parallel.py rebuilds a
 * rank's owned + ghost set from exchanged records without a host round trip.  recs / bodies may be host
 * or device pointers; the Verlet list is rebuilt on the next step. */
int sphg_upload_records(sphg_ctx* ctx, size_t n, size_t n_owned, const double* recs, const sphg_body* bodies,
                        size_t n_bodies);
/* replaces the body table after record_unpack changed kinds / groups and refreshes the index lists
 * (rigid body-major list, kind lists, row partitions, contact order) */
int sphg_replace_bodies(sphg_ctx* ctx, const sphg_body* bodies, size_t n_bodies);
/* Transition event log ("Event log (CSV): step, particle id, direction, body ids"): when enabled,
 * every applied transition is recorded as (step, gid, direction 1 melt / 2 solidify, body it left (melt)
 * or -1, body it ended the batch in (solidify, after splits) or -1), ordered by step then gid.
 * sphg_transition_events copies up to `cap` of the events recorded since the last call into `out`
 * (out may be NULL to query), stores the number copied (or pending, with out = NULL) in *n and drops
 * the copied ones. */
typedef struct {
  int64_t step;
  uint32_t gid;
  int32_t direction;
  int32_t body_from;
  int32_t body_to;
} sphg_event;
int sphg_set_event_log(sphg_ctx* ctx, int enabled);
int sphg_transition_events(sphg_ctx* ctx, sphg_event* out, size_t cap, size_t* n);
const char* sphg_last_error(const sphg_ctx* ctx);
void sphg_destroy(sphg_ctx* ctx);
/* Messages of validate_config for `params` joined by '\n' (empty = valid). */
int sphg_validate(const sphg_params* params, char* buf, size_t buflen);

#ifdef __cplusplus
}
#endif
#endif /* SPHG_H */
