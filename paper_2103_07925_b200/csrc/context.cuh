// context.cuh — device-resident state of one sphg context (one GPU / one rank).
//
// HBM layout: every per-particle array is in cell-sorted order
// (key = (cell, gid)) and packed for the pair-gather kernels:
//   G0 = (x, y, z, V^2)        interaction volume squared (fluid: (m/rho)^2, wall/rigid: V_w^2)
//   G1 = (u, rho)              interaction velocity/density (fluid: u^{n+1/2}, rho; wall/rigid: u~_w, rho_w)
//   G2 = (du, p)               du = u_adv - u (TVF A term; 0 for wall/rigid), pressure (wall/rigid: p_w)
//   V4 = (vel, mass)           true velocity (fluid u^n between steps, rigid u_r, boundary: wall
//                              group velocity or 0)
//   A4 = (acc, -)  B4 = (acc_bg, -)  F4 = (f_r, -)  X4 = (chi, -)  R4 = (pos at last rebuild, -)
//   H2 = (T, V_heat)           temperature and the conduction volume V_b (0 for non-Dirichlet walls)
//   C2 = (C, V_diff), dCdt     concentration (only with params.diffusion)
//   kmd (kind|mat|Dirichlet-T|ghost|Dirichlet-C), group, gid : uint32
// Verlet candidates are row-major: nbr[i * cap + k] for k < cnt[i] (cnt = nf | no << 16,
// [fluid | non-fluid]); entries pack the periodic image code (common.cuh kImgCode).  Per-kind
// index lists (fluid / non-fluid in brick order, rigid body-major) drive the pair kernels.
#pragma once

#include <functional>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"

namespace sphg {

struct CudaError {
  cudaError_t code;
  std::string what;
  CudaError(cudaError_t c, const char* expr, const char* file, int line)
      : code(c), what(std::string(cudaGetErrorString(c)) + " at " + file + ":" + std::to_string(line) + " (" + expr + ")") {}
};

struct NbrList {
  const uint32_t* nbr;
  const uint32_t* cnt;
  size_t cap;
};

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  void alloc(size_t count) {
    if (count <= n && p) return;
    free();
    if (count == 0) return;
    SPHG_CUDA_CHECK(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  void free() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

struct Particles {  // one buffer set (double-buffered for the rebuild reorder)
  DBuf<double4> G0, G1, G2, V4, A4, B4, F4, X4, R4;
  DBuf<double2> H2;
  DBuf<double> dTdt, p_static;
  DBuf<uint32_t> kmd, group, gid;
  DBuf<double2> C2;  // concentration, diffusion volume (allocated only with params.diffusion)
  DBuf<double> dCdt;
  void alloc(size_t n, bool conc) {
    G0.alloc(n); G1.alloc(n); G2.alloc(n); V4.alloc(n); A4.alloc(n); B4.alloc(n); F4.alloc(n);
    X4.alloc(n); R4.alloc(n); H2.alloc(n); dTdt.alloc(n); p_static.alloc(n);
    kmd.alloc(n); group.alloc(n); gid.alloc(n);
    if (conc) {
      C2.alloc(n);
      dCdt.alloc(n);
    }
  }
  void free() {
    G0.free(); G1.free(); G2.free(); V4.free(); A4.free(); B4.free(); F4.free(); X4.free(); R4.free();
    H2.free(); dTdt.free(); p_static.free(); kmd.free(); group.free(); gid.free(); C2.free(); dCdt.free();
  }
};

struct Ctx {
  sphg_params params{};
  DevParams P{};
  int device = 0;
  cudaStream_t stream = nullptr;
  size_t n = 0;            // particles
  size_t nb = 0;           // bodies (live or dead)
  Particles cur, alt;      // alt = reorder target / scratch
  DBuf<double2> H2new;     // heat double buffer
  DBuf<double2> C2new;     // concentration double buffer
  DBuf<double> hsrc;       // surface heat flux source rate per particle [P21] (params.heat_source)
  DBuf<uint32_t> pin_list;  // particles whose rigid / wall sums take the pinned redo (common.cuh pinned_q)
  uint32_t* pin_any = nullptr;  // device: their count
  DBuf<sphg_body> bodies;
  size_t bodies_cap = 0;
  // rebuild scratch
  DBuf<unsigned long long> keys, keys_alt;
  DBuf<uint32_t> vals, vals_alt, hist, scan_tmp;
  DBuf<uint32_t> cell_start, cell_end, cell_key;
  int64_t ncells = 0;
  // neighbour list (row-major)
  DBuf<uint32_t> nbr, cnt;
  int cap = 0;
  NbrList nl() const { return {nbr.p, cnt.p, (size_t)cap}; }
  // SM-local persistent pair kernels (SPHG_SM_LOCAL: bit 0 = fluid forces, bit 1 = density, bit 2 =
  // extrapolation, bit 3 = rigid forces, bit 4 = conduction; 0 = flat grids)
  int sm_local = 31, n_sms = 148;
  int sm_threads = 128;            // block size of the persistent grids (SPHG_SM_THREADS: 32, 64, 128)
  size_t sm_local_min = 1u << 20;  // shortest list that gets a persistent grid (SPHG_SM_LOCAL_MIN)
  DBuf<uint32_t> sm_next;  // per-SM tile counters, n_sms each: density, fluid forces, extrapolation, rigid
                           // forces, interior density, conduction (kernels that may run concurrently never share one)
  // per-kind index lists: fluid, non-fluid (rigid + boundary), rigid body-major
  DBuf<uint32_t> fidx, widx, ridx, body_start;
  DBuf<uint32_t> ncon;  // per rigid particle: contact candidates at the front of its non-fluid row part
  DBuf<uint32_t> brick_buf, scan_cells;
  DBuf<uint8_t> dl_buf;  // download: requested store fields in gid order
  size_t nf = 0, nw = 0, nrigid = 0;
  int group_density = 0, group_forces = 0;  // lanes per particle in the pair kernels (0 = lanes_for)
  size_t fill_groups = 37888;  // particles that fill the GPU at 4 lanes: SMs x 2048 threads / 4 / 2
  bool cell_build = true;  // cell-cooperative Verlet build (falls back per particle on overflow)
  sphg_wall_motion_fn wall_fn = nullptr;  // moving wall groups (sphg_set_wall_motion)
  void* wall_user = nullptr;
  // transitions scratch
  DBuf<uint32_t> ev_idx, ev_flag, label, tscratch;
  DBuf<uint32_t> label_list, label_flags;  // compact list of labelled particles; sweep flags + count
  DBuf<uint32_t> wrap_list;  // (index, wrap code) of the particles that crossed a periodic face this step
  // decomposed transition batches (sphg_event_*, sphg_record_*): id lists and records
  DBuf<uint32_t> rec_ids;
  DBuf<uint32_t> group0;  // body ids at the start of a transition batch
  DBuf<sphg_body> bodies_old;  // the body table at the start of a transition batch
  DBuf<uint32_t> label_adj;    // labelled particles' same-body adjacency (split_disconnected_bodies)
  DBuf<double> rec_buf;
  // transition event log (sphg_set_event_log): device buffer of the current batch, host accumulation
  bool event_log = false;
  DBuf<sphg_event> ev_log;
  DBuf<uint32_t> ev_count;
  std::vector<sphg_event> events;
  // flags
  DevFlags* dflags = nullptr;   // device
  DevFlags* hflags = nullptr;   // pinned host mirror
  bool built = false;
  // kick fusion inside one sphg_step(K) call: the particle final kick of step n is deferred into the
  // kick-drift pass of step n+1 (never across API calls, with transitions, or with stage timing)
  bool defer_final = false, final_pending = false;
  // conduction of fluid particles folded into k_forces_fluid inside sphg_step (not for stage calls)
  bool fuse_heat = false;
  bool fuse_diff = false;  // likewise the concentration sums, when the heat equation is off
  bool have_state = false;
  double t = 0.0;
  int64_t steps = 0, rebuilds = 0, n_melt = 0, n_solid = 0, launches = 0;
  double max_disp = 0.0, u_max = 0.0;
  int64_t pairs = 0;
  int max_count = 0;
  bool timing = false;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  double stage_ms[16] = {0};
  std::string err;
  // host staging for body table (pinned)
  sphg_body* hbodies = nullptr;
  size_t hbodies_cap = 0;
  void* hstage = nullptr;          // 2 pinned staging slots (upload/download)
  cudaEvent_t slot_ev[2] = {nullptr, nullptr};
  unsigned long long* dcount = nullptr;  // pair counters
  cudaEvent_t step_ev[2] = {nullptr, nullptr};
  double last_step_ms = 0.0;
  // domain decomposition: halo index lists (local ids) and gid -> device index
  DBuf<uint32_t> idx_of_gid;
  DBuf<uint32_t> halo_ids[SPHG_MAX_HALO_SLOTS];
  size_t halo_n[SPHG_MAX_HALO_SLOTS] = {0};
  size_t nghost = 0;
  DBuf<double> body_buf;
  DBuf<double> state_buf;  // upload_state staging (device)
  size_t last_h2d_bytes = 0, last_d2h_bytes = 0;
  // CUDA graphs of the two per-step launch chains (api.cu run_graph): keyed by every pointer, count
  // and parameter the chain's launches read, so a rebuild / transition / upload selects (or captures)
  // another graph instead of replaying stale arguments.  The Dirichlet schedules read t^{n+1} from
  // dtime[0], a device clock the kick chain's tail advances every step (resynced with c.t per call).
  struct GraphEntry {
    std::vector<unsigned char> key;
    cudaGraphExec_t exec = nullptr;
    int64_t launches = 0;
    Particles cur_after;
    DBuf<double2> H2new_after, C2new_after;
    bool final_pending_after = false;
    uint64_t used = 0;
  };
  std::vector<GraphEntry> graphs;
  uint64_t graph_clock = 0;
  int64_t graph_captures = 0, graph_replays = 0;
  bool use_graphs = true, capturing = false;
  double* dtime = nullptr;  // device: [0] the force chain's time (c.t + dt), [1] the clock (c.t)
  double* htime = nullptr;  // pinned host staging for the resync
  // sphg_step_download: enqueued after the wall extrapolation of the last step (eager chain), packs the
  // fields that are final by then so their D2H copies on copy_stream overlap the force kernels
  std::function<void(Ctx&)> pre_forces;
  // speculative steps (one_step): the force chain is queued before the host has read the kick
  // chain's flags; dskip (read by every force-chain kernel through DevParams::skip) voids it when the
  // step needs a Verlet rebuild.  SPHG_SPECULATE=0 turns it off.
  bool speculate = true;
  uint32_t* dskip = nullptr;
  cudaEvent_t kick_ev = nullptr;
  // rigid force pass on a second stream beside the fluid one (SPHG_CONCURRENT_RIGID=0 serialises)
  bool concurrent_rigid = true;
  cudaStream_t side_stream = nullptr;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t dl_ev = nullptr;
  // runtime time-step assertion (api.cu check_dt) [P22]
  double m_r = 0.0;  // smallest mass a rigid particle can have in this run (set at upload; 0 = none)
  int64_t dt_violations = 0;
  int dt_term = -1;
  double dt_limit = 0.0;
  int64_t host_syncs = 0;  // host-blocking waits on the device (sphg_stats_t.host_syncs)
  // in-library decomposed step (api.cu one_step_decomposed): exchange callback and bound buffers
  sphg_exchange_fn exch_fn = nullptr;
  void* exch_user = nullptr;
  double* halo_buf[3][SPHG_MAX_HALO_SLOTS] = {};
  uint64_t* max_words = nullptr; // 2 words reduced by the MAX exchange
  double* body_part = nullptr;   // nb x 24 partials this rank contributes
  double* body_gath = nullptr;   // world x nb x 24, filled by the BODIES exchange
  int world = 1;
  size_t nf_interior = 0;        // fidx[0, nf_interior): fluid particles with no ghost neighbour
  double disp_since_partition = 0.0;  // sum of the global displacements at rebuilds since the last upload
  double partition_limit = 0.0;       // sphg_set_partition_limit (0 = none)
  DBuf<double> body_tot;         // merged nb x 12 totals
  cudaStream_t dens_stream = nullptr;
  cudaEvent_t dens_fork = nullptr, dens_join = nullptr;
};

// every host-blocking wait of the library goes through these (counted in sphg_stats_t.host_syncs)
inline void host_sync(Ctx& c, cudaStream_t s) {
  SPHG_CUDA_CHECK(cudaStreamSynchronize(s));
  c.host_syncs++;
}
inline void host_sync_event(Ctx& c, cudaEvent_t e) {
  SPHG_CUDA_CHECK(cudaEventSynchronize(e));
  c.host_syncs++;
}

// NVTX ranges (SURVEY §5 tracing): stages, exchanges and API calls show up by name under nsys / ncu
// --nvtx; header-only NVTX3, a no-op without an attached tool
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// ------------------------------------------------------------ launchers
// radix_sort.cu
size_t radix_scratch_words(size_t n);
// Sorts (keys, vals) by the low `bits` bits of keys, stable.  Returns true if
// the result ended in the *_alt buffers.
bool radix_sort_pairs(unsigned long long* keys, uint32_t* vals, unsigned long long* keys_alt, uint32_t* vals_alt,
                      size_t n, int bits, uint32_t* hist, uint32_t* scan_tmp, cudaStream_t s, int64_t* launches);
void exclusive_scan_u32(const uint32_t* in, uint32_t* out, size_t n, uint32_t* tmp, cudaStream_t s,
                        int64_t* launches);

// kernels_rebuild.cu
void launch_rebuild(Ctx& c);
void launch_rigid_index(Ctx& c, bool kinds_changed = true);
void check_structures(Ctx& c);  // -DSPHG_CHECKED: rows and index lists in bounds (kErrInvariant)

// kernels_step.cu
void launch_body_kick(Ctx& c);
void launch_kick_drift(Ctx& c);
void launch_wrap_patch(Ctx& c);  // image codes of rows after periodic-face crossings (n_wrapped, wrap_list)
void launch_step_tail(Ctx& c);  // dskip (rebuild or error pending) and the device clock t^{n+1}
void launch_density(Ctx& c);
void launch_density_interior(Ctx& c, cudaStream_t st);
void launch_density_boundary(Ctx& c);
void launch_ghost_split(Ctx& c);  // orders fidx [interior | next to a ghost] (decomposed steps)
void merge_body_partials(Ctx& c, const double* gathered, int world, double* totals);
void launch_heat(Ctx& c);
void launch_heat_begin(Ctx& c);
void launch_heat_end(Ctx& c);
void launch_diffusion(Ctx& c);
void launch_diffusion_begin(Ctx& c);
void launch_diffusion_end(Ctx& c);
void launch_extrapolate(Ctx& c);
void launch_forces(Ctx& c);
void launch_forces_fluid(Ctx& c);
void launch_forces_rigid(Ctx& c);
void launch_forces_diag(Ctx& c);  // diagnostic builds only (stage 12)
void launch_bodies(Ctx& c);
void launch_final_kick(Ctx& c);
void launch_final_kick_particles(Ctx& c);
void launch_mass(Ctx& c, const uint32_t* body_mask);
void gather_by_gid(Ctx& c);          // cur[k] <- alt[gid[k]] for every field but gid/R4
bool displacement_exceeds(Ctx& c);   // max |r - r_ref| > half skin (syncs)
void iota_gid(Ctx& c);
void scatter_state(Ctx& c, const double* pos, const double* vel);  // gid-ordered xyz -> G0.xyz / V4.xyz
void count_pairs(Ctx& c, int64_t out[4]);
void cell_occupancy(Ctx& c, unsigned long long* dev_hist, uint32_t nbins, uint32_t* dev_max);
void shepard_grid(Ctx& c, const double origin[3], const double spacing[3], const int32_t dims[3], int field,
                  uint32_t kind_mask, double* dev_out, uint8_t* dev_support);
void build_idx_of_gid(Ctx& c);
void halo_pack(Ctx& c, int phase, int slot, double* buf);
void halo_unpack(Ctx& c, int phase, int slot, const double* buf);
void wrap_ghosts(Ctx& c);
void body_partials(Ctx& c, double* dev_out);
void body_apply_totals(Ctx& c, const double* dev_tot);

// kernels_transition.cu
int launch_transitions(Ctx& c);  // 0 ok, else error code
void launch_detect(Ctx& c);      // event flags (ev_flag) of the owned particles; counts in dflags
void event_bodies(Ctx& c, uint32_t* dev_mask);  // bodies a batch can touch (sphg_event_bodies)
size_t event_members(Ctx& c, const uint32_t* dev_mask, size_t nb, uint32_t* dev_ids);  // unsorted local ids
constexpr int kRecordDoubles = 44;
uint32_t record_pack(Ctx& c, const uint32_t* dev_ids, size_t m, double* dev_out);  // ~0u or first bad id
uint32_t record_unpack(Ctx& c, const uint32_t* dev_ids, size_t m, const double* dev_in, int keep_position);
void record_load(Ctx& c, const double* dev_recs, size_t n, size_t n_owned);  // whole store (sphg_upload_records)
uint32_t record_check(Ctx& c, const double* dev_recs, size_t n, size_t nb);  // first invalid record or ~0u
void launch_repartition_rows(Ctx& c);
void launch_contact_order(Ctx& c, const uint32_t* list = nullptr, size_t m = 0);

inline int grid_for(size_t n, int block) { return (int)((n + block - 1) / block); }

}  // namespace sphg
