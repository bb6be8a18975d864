// kernels_transition.cu — temperature-driven melt/solidify reclassification
// on the device.
//
// Pinned rules [P12] (identical in oracle/sph_oracle.cpp stage_transitions):
//  * detect: rigid T > T_t -> melt (into melt_target); fluid T < T_t -> solidify; strict
//  * batch is a set: melting particles are no attach targets, solidifying ones neither
//  * melt: kind F, velocity u_k + w_k x r_rk, acc = 0
//  * solidify: attach to the body of the nearest pre-batch rigid particle within r_c
//    (ties by gid), else spawn; spawned ids = nb + rank in gid order
//  * split bodies that lost particles: components with adjacency r <= 1.5 dx, found
//    by min-gid label propagation; the min-gid component keeps the id, others get
//    new ids ordered by (source body, min gid)
//  * affected bodies: reduce_mass_quantities (chi recomputed), u_k = u'_k + w x (r_k - r'_k),
//    members follow the rigid motion, then reduce_force_torque for all bodies.
#include <algorithm>
#include <cstdlib>

#include <cooperative_groups.h>

#include "context.cuh"

namespace sphg {

namespace {

__device__ __forceinline__ Quat body_q(const sphg_body& b) { return {b.q[0], b.q[1], b.q[2], b.q[3]}; }

__global__ void k_detect(const __grid_constant__ DevParams P, Particles D, size_t n, uint32_t* __restrict__ ev,
                         DevFlags* __restrict__ fl) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const uint32_t kmd = D.kmd.p[k];
  const uint32_t kind = kind_of(kmd);
  const DevMat& M = P.mat[mat_of(kmd)];
  uint32_t e = 0;
  if (is_ghost(kmd)) {  // decomposed runs: every rank detects over the particles it owns
    ev[k] = 0;
    return;
  }
  // trigger field by TransitionMode (config.hpp:61): 1 temperature, 2 concentration [P19]
  const bool conc = P.transitions == 2;
  if (conc ? M.has_Ct : M.has_Tt) {
    const double x = conc ? D.C2.p[k].x : D.H2.p[k].x;
    const double thr = conc ? M.C_t : M.T_t;
    if (kind == SPHG_RIGID && M.melt >= 0 && x > thr) e = 1;
    else if (kind == SPHG_FLUID && M.solid >= 0 && x < thr) e = 2;
  }
  ev[k] = e;
  if (e == 1) atomicAdd(&fl->n_events, 1u);
  if (e == 2) atomicAdd(&fl->pad[0], 1u);
}

__global__ void k_melt(const __grid_constant__ DevParams P, Particles D, size_t n, const uint32_t* __restrict__ ev,
                       const sphg_body* __restrict__ B, uint32_t* __restrict__ bmask, uint32_t* __restrict__ blost,
                       sphg_event* __restrict__ log, uint32_t* __restrict__ nlog, int64_t step) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n || ev[k] != 1) return;
  const uint32_t kmd = D.kmd.p[k];
  const uint32_t body = D.group.p[k];
  if (log) log[atomicAdd(nlog, 1u)] = sphg_event{step, D.gid.p[k], 1, (int32_t)body, -1};
  const sphg_body& b = B[body];
  const double4 x = D.X4.p[k];
  const double3 rk = qrotate(body_q(b), make_double3(x.x, x.y, x.z));
  const double3 w = cross3(make_double3(b.omega[0], b.omega[1], b.omega[2]), rk);
  const double3 u = make_double3(b.vel[0] + w.x, b.vel[1] + w.y, b.vel[2] + w.z);
  const int tgt = P.mat[mat_of(kmd)].melt;
  const double m = D.V4.p[k].w;
  const double rho0 = P.mat[tgt].rho0;
  D.kmd.p[k] = (kmd & kGhostBit) | make_kmd(SPHG_FLUID, (uint32_t)tgt, dir_of(kmd), dirc_of(kmd));
  D.group.p[k] = 0;
  D.V4.p[k] = make_double4(u.x, u.y, u.z, m);
  const double V = m / rho0;
  reinterpret_cast<double*>(&D.G0.p[k])[3] = V * V;
  D.G1.p[k] = make_double4(u.x, u.y, u.z, rho0);
  D.G2.p[k] = make_double4(0, 0, 0, 0);
  D.A4.p[k] = make_double4(0, 0, 0, 0);
  D.B4.p[k] = make_double4(0, 0, 0, 0);
  D.F4.p[k] = make_double4(0, 0, 0, 0);
  D.X4.p[k] = make_double4(0, 0, 0, 0);
  D.p_static.p[k] = 0.0;
  reinterpret_cast<double*>(&D.H2.p[k])[1] = V;
  if (D.C2.p) reinterpret_cast<double*>(&D.C2.p[k])[1] = V;
  bmask[body] = 1;
  blost[body] = 1;
}

__global__ void k_flag_eq(const uint32_t* __restrict__ ev, size_t n, uint32_t v, uint32_t* __restrict__ out) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) out[k] = ev[k] == v ? 1u : 0u;
}

__global__ void k_compact_by_gid(const uint32_t* __restrict__ ev, const uint32_t* __restrict__ pos, size_t n, uint32_t v,
                                 const uint32_t* __restrict__ gid, unsigned long long* __restrict__ keys,
                                 uint32_t* __restrict__ vals) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n || ev[k] != v) return;
  keys[pos[k]] = gid[k];
  vals[pos[k]] = (uint32_t)k;
}

// nearest pre-batch rigid particle within r_c (r^2, gid), from the Verlet list
__device__ __forceinline__ uint32_t entry_index(const DevParams& P, uint32_t e) {
  return P.img_mode == kImgCode ? (e & kIdxMask) : e;
}

__global__ void k_solid_target(const __grid_constant__ DevParams P, Particles D, const uint32_t* __restrict__ list,
                               size_t m, NbrList L, int* __restrict__ target, uint32_t* __restrict__ spawn) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m) return;
  const uint32_t i = list[e];
  const double4 pi = D.G0.p[i];
  double best = 1e300;
  uint32_t bg = 0xffffffffu;
  int tb = -1;
  // whole row: mid-batch the kinds no longer match the rows' fluid / non-fluid partition
  const uint32_t nn = cnt_total(L.cnt[i]);
  const uint32_t* row = L.nbr + (size_t)i * L.cap;
  for (uint32_t k = 0; k < nn; ++k) {
    const uint32_t j = entry_index(P, row[k]);
    if (kind_of(D.kmd.p[j]) != SPHG_RIGID) continue;
    const double4 pj = D.G0.p[j];
    const double r2 = r2_exact(mimg3(P, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z));
    if (r2 > P.rc2) continue;
    const uint32_t gj = D.gid.p[j];
    if (r2 < best || (r2 == best && gj < bg)) {
      best = r2;
      bg = gj;
      tb = (int)D.group.p[j];
    }
  }
  target[e] = tb;
  spawn[e] = tb < 0 ? 1u : 0u;
}

__global__ void k_solid_apply(const __grid_constant__ DevParams P, Particles D, const uint32_t* __restrict__ list,
                              size_t m, const int* __restrict__ target, const uint32_t* __restrict__ rank, size_t nb0,
                              sphg_body* __restrict__ B, uint32_t* __restrict__ bmask, uint32_t* __restrict__ src) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m) return;
  const uint32_t i = list[e];
  const uint32_t kmd = D.kmd.p[i];
  const int tgt = P.mat[mat_of(kmd)].solid;
  uint32_t body;
  const double4 v = D.V4.p[i];
  if (target[e] >= 0) {
    body = (uint32_t)target[e];
  } else {
    body = (uint32_t)(nb0 + rank[e]);
    sphg_body nbd;
    memset(&nbd, 0, sizeof(nbd));
    nbd.q[0] = 1.0;
    nbd.vel[0] = v.x;
    nbd.vel[1] = v.y;
    nbd.vel[2] = v.z;
    nbd.material = tgt;
    nbd.mobile = 1;
    nbd.alive = 1;
    B[body] = nbd;
    src[body] = body;
  }
  bmask[body] = 1;
  const double rho0 = P.mat[tgt].rho0;
  D.kmd.p[i] = (kmd & kGhostBit) | make_kmd(SPHG_RIGID, (uint32_t)tgt, dir_of(kmd), dirc_of(kmd));
  D.group.p[i] = body;
  D.A4.p[i] = make_double4(0, 0, 0, 0);
  D.B4.p[i] = make_double4(0, 0, 0, 0);
  D.p_static.p[i] = 0.0;
  // wall quantities are undefined until the next extrapolation: zero (oracle does the same)
  D.G1.p[i] = make_double4(0, 0, 0, rho0);
  D.G2.p[i] = make_double4(0, 0, 0, 0);
  reinterpret_cast<double*>(&D.H2.p[i])[1] = v.w / rho0;
  if (D.C2.p) reinterpret_cast<double*>(&D.C2.p[i])[1] = v.w / rho0;
}

// event log: every solidified particle with the body it ended the batch in (after splits)
__global__ void k_log_solid(Particles D, const uint32_t* __restrict__ list, size_t m, sphg_event* __restrict__ log,
                            uint32_t* __restrict__ nlog, int64_t step) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m) return;
  const uint32_t i = list[e];
  log[atomicAdd(nlog, 1u)] = sphg_event{step, D.gid.p[i], 2, -1, (int32_t)D.group.p[i]};
}

__global__ void k_iota(uint32_t* __restrict__ a, size_t n, size_t from) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) a[from + k] = (uint32_t)(from + k);
}

// ---------------------------------------------------- connected components
// Rigid particles of bodies that lost particles get label = gid, the others NONE; the labels then
// relax to the minimum gid of their component (adjacency r <= 1.5 dx within one body).  The relaxation
// runs entirely on the device: the labelled particles are compacted into a list and one cooperative
// kernel iterates over that list with grid-wide barriers until a sweep changes nothing (no host
// round trip per sweep, no full-store launch per sweep).
__global__ void k_label_init(Particles D, size_t n, const uint32_t* __restrict__ blost, uint32_t* __restrict__ label,
                             uint32_t* __restrict__ list, uint32_t* __restrict__ count) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const bool on = kind_of(D.kmd.p[k]) == SPHG_RIGID && blost[D.group.p[k]];
  label[k] = on ? D.gid.p[k] : 0xffffffffu;
  if (on) list[atomicAdd(count, 1u)] = (uint32_t)k;  // order is irrelevant: the fixpoint is unique
}

__device__ __forceinline__ bool label_relax(const DevParams& P, const Particles& D, const NbrList& L,
                                            uint32_t* label, double adj2, uint32_t i) {
  const uint32_t l = label[i];
  const uint32_t body = D.group.p[i];
  const double4 pi = D.G0.p[i];
  uint32_t best = l;
  const uint32_t nn = cnt_total(L.cnt[i]);  // whole row (see k_solid_target)
  const uint32_t* row = L.nbr + (size_t)i * L.cap;
  for (uint32_t k = 0; k < nn; ++k) {
    const uint32_t j = P.img_mode == kImgCode ? (row[k] & kIdxMask) : row[k];
    if (kind_of(D.kmd.p[j]) != SPHG_RIGID || D.group.p[j] != body) continue;
    const double4 pj = D.G0.p[j];
    if (r2_exact(mimg3(P, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z)) > adj2) continue;
    best = min(best, label[j]);
  }
  if (best < l) {
    atomicMin(&label[i], best);
    return true;
  }
  return false;
}

// The adjacency of each labelled particle (same-body rigid neighbours within 1.5 dx: at most 18 on the
// lattice the bodies are cut from) extracted once from its row, so a sweep reads ~18 labels instead of
// re-testing the ~120 row entries; nadj > kAdjMax marks a particle the sweeps relax from its row.
constexpr uint32_t kAdjMax = 32;
__global__ void k_label_adj(const __grid_constant__ DevParams P, Particles D, NbrList L,
                            const uint32_t* __restrict__ list, const uint32_t* __restrict__ count, double adj2,
                            uint32_t* __restrict__ adj, uint32_t* __restrict__ nadj) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= *count) return;
  const uint32_t i = list[e];
  const uint32_t body = D.group.p[i];
  const double4 pi = D.G0.p[i];
  const uint32_t nn = cnt_total(L.cnt[i]);
  const uint32_t* row = L.nbr + (size_t)i * L.cap;
  uint32_t c = 0;
  for (uint32_t k = 0; k < nn; ++k) {
    const uint32_t j = P.img_mode == kImgCode ? (row[k] & kIdxMask) : row[k];
    if (kind_of(D.kmd.p[j]) != SPHG_RIGID || D.group.p[j] != body) continue;
    const double4 pj = D.G0.p[j];
    if (r2_exact(mimg3(P, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z)) > adj2) continue;
    if (c < kAdjMax) adj[e * kAdjMax + c] = j;
    ++c;
  }
  nadj[e] = c;
}

// one relaxation of labelled particle e: the minimum over its adjacency, then a pointer jump through the
// particle whose gid is that minimum (it is in the same component and its label is <= its gid)
__device__ __forceinline__ bool label_relax_adj(const DevParams& P, const Particles& D, const NbrList& L,
                                                uint32_t* label, double adj2, uint32_t i, uint32_t e,
                                                const uint32_t* adj, const uint32_t* nadj, const uint32_t* idx) {
  const uint32_t na = nadj[e];
  if (na > kAdjMax) return label_relax(P, D, L, label, adj2, i);
  const uint32_t l = label[i];
  uint32_t best = l;
  for (uint32_t k = 0; k < na; ++k) best = min(best, label[adj[(size_t)e * kAdjMax + k]]);
  best = min(best, label[idx[best]]);
  if (best < l) {
    atomicMin(&label[i], best);
    return true;
  }
  return false;
}

// cooperative: grid-stride sweeps over the list, grid barrier, stop when a sweep changed nothing.
// flags[0..1]: double-buffered "changed" words (cleared one sweep ahead); flags[2]: sweeps done
__global__ void k_label_coop(const __grid_constant__ DevParams P, Particles D, NbrList L, const uint32_t* __restrict__ list,
                             const uint32_t* __restrict__ count, uint32_t* __restrict__ label, double adj2,
                             uint32_t* __restrict__ flags, const uint32_t* __restrict__ adj,
                             const uint32_t* __restrict__ nadj, const uint32_t* __restrict__ idx) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const uint32_t m = *count;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
  for (uint32_t sweep = 0;; ++sweep) {
    if (sweep >= 1000000u) {  // cannot happen (labels only decrease); never spin forever
      if (tid == 0) flags[2] = 0xffffffffu;
      return;
    }
    uint32_t* changed = flags + (sweep & 1u);
    if (tid == 0) flags[(sweep + 1) & 1u] = 0u;  // the next sweep's word; nobody reads it this sweep
    bool any = false;
    for (size_t e = tid; e < m; e += stride)
      any |= label_relax_adj(P, D, L, label, adj2, list[e], (uint32_t)e, adj, nadj, idx);
    if (any) atomicOr(changed, 1u);
    grid.sync();
    const uint32_t c = *reinterpret_cast<volatile uint32_t*>(changed);
    if (!c) {
      if (tid == 0) flags[2] = sweep + 1;
      return;
    }
    grid.sync();  // every thread has read `changed` before it is cleared two sweeps later
  }
}

__global__ void k_split_roots(Particles D, size_t n, const uint32_t* __restrict__ label,
                              const uint32_t* __restrict__ ridx, const uint32_t* __restrict__ bstart, int gbits,
                              unsigned long long* __restrict__ keys, uint32_t* __restrict__ vals,
                              DevFlags* __restrict__ fl) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t l = label[i];
  if (l == 0xffffffffu || l != D.gid.p[i]) return;
  const uint32_t body = D.group.p[i];
  const uint32_t minimal = D.gid.p[ridx[bstart[body]]];
  if (l == minimal) return;
  const uint32_t s = atomicAdd(&fl->pad[1], 1u);
  keys[s] = ((unsigned long long)body << gbits) | l;
  vals[s] = body;
}

__global__ void k_split_bodies(const unsigned long long* __restrict__ keys, size_t m, int gbits, size_t nb0,
                               sphg_body* __restrict__ B, uint32_t* __restrict__ bmask, uint32_t* __restrict__ src) {
  const size_t s = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= m) return;
  const uint32_t body = (uint32_t)(keys[s] >> gbits);
  B[nb0 + s] = B[body];
  bmask[nb0 + s] = 1;
  src[nb0 + s] = body;
}

__global__ void k_split_relabel(Particles D, size_t n, const uint32_t* __restrict__ label,
                                const uint32_t* __restrict__ ridx, const uint32_t* __restrict__ bstart,
                                const unsigned long long* __restrict__ keys, size_t m, int gbits, size_t nb0) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t l = label[i];
  if (l == 0xffffffffu) return;
  const uint32_t body = D.group.p[i];
  if (l == D.gid.p[ridx[bstart[body]]]) return;
  const unsigned long long key = ((unsigned long long)body << gbits) | l;
  size_t lo = 0, hi = m;
  while (lo < hi) {
    const size_t mid = (lo + hi) / 2;
    if (keys[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  D.group.p[i] = (uint32_t)(nb0 + lo);
}

// u_k = u'_k + w'_k x (r_k - r'_k) for affected, non-spawned bodies
__global__ void k_post_velocity(const __grid_constant__ DevParams P, sphg_body* __restrict__ B,
                                const sphg_body* __restrict__ old, const uint32_t* __restrict__ bmask,
                                const uint32_t* __restrict__ src, size_t nb, size_t nb0) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nb || !bmask[k]) return;
  sphg_body& b = B[k];
  if (!b.alive) return;
  const uint32_t s = src[k];
  if (k >= nb0 && s == k) return;  // spawned: keeps the particle's velocity, w = 0
  const sphg_body& o = old[s];
  const double3 sh = mimg3(P, b.com[0], b.com[1], b.com[2], o.com[0], o.com[1], o.com[2]);
  const double3 w = cross3(make_double3(o.omega[0], o.omega[1], o.omega[2]), sh);
  b.vel[0] = o.vel[0] + w.x;
  b.vel[1] = o.vel[1] + w.y;
  b.vel[2] = o.vel[2] + w.z;
}

__global__ void k_member_velocity(Particles D, size_t n, const sphg_body* __restrict__ B,
                                  const uint32_t* __restrict__ bmask) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n || kind_of(D.kmd.p[k]) != SPHG_RIGID) return;
  const uint32_t body = D.group.p[k];
  if (!bmask[body]) return;
  const sphg_body& b = B[body];
  const double4 x = D.X4.p[k];
  const double3 rk = qrotate(body_q(b), make_double3(x.x, x.y, x.z));
  const double3 w = cross3(make_double3(b.omega[0], b.omega[1], b.omega[2]), rk);
  const double m = D.V4.p[k].w;
  D.V4.p[k] = make_double4(b.vel[0] + w.x, b.vel[1] + w.y, b.vel[2] + w.z, m);
}

int bits_for(uint64_t maxval) {
  int b = 0;
  while (b < 64 && (maxval >> b) != 0) ++b;
  return b;
}

uint32_t read_u32(Ctx& c, const uint32_t* p) {
  uint32_t v = 0;
  SPHG_CUDA_CHECK(cudaMemcpyAsync(&v, p, 4, cudaMemcpyDeviceToHost, c.stream));
  host_sync(c, c.stream);
  return v;
}

// two device words with one host synchronisation (a batch's readbacks are its latency)
void read_u32x2(Ctx& c, const uint32_t* p, const uint32_t* q, uint32_t& a, uint32_t& b) {
  uint32_t v[2] = {0, 0};
  SPHG_CUDA_CHECK(cudaMemcpyAsync(&v[0], p, 4, cudaMemcpyDeviceToHost, c.stream));
  SPHG_CUDA_CHECK(cudaMemcpyAsync(&v[1], q, 4, cudaMemcpyDeviceToHost, c.stream));
  host_sync(c, c.stream);
  a = v[0];
  b = v[1];
}
uint32_t read_sum2(Ctx& c, const uint32_t* p, const uint32_t* q) {
  uint32_t a, b;
  read_u32x2(c, p, q, a, b);
  return a + b;
}

void grow_bodies(Ctx& c, size_t need) {
  if (need <= c.bodies_cap && c.bodies.p) return;
  const size_t cap = std::max<size_t>(need * 2, 64);
  sphg_body* nb = nullptr;
  SPHG_CUDA_CHECK(cudaMalloc(&nb, cap * sizeof(sphg_body)));
  SPHG_CUDA_CHECK(cudaMemsetAsync(nb, 0, cap * sizeof(sphg_body), c.stream));
  if (c.bodies.p && c.nb)
    SPHG_CUDA_CHECK(cudaMemcpyAsync(nb, c.bodies.p, c.nb * sizeof(sphg_body), cudaMemcpyDeviceToDevice, c.stream));
  host_sync(c, c.stream);
  c.bodies.free();
  c.bodies.p = nb;
  c.bodies.n = cap;
  c.bodies_cap = cap;
}


// Re-partitions every Verlet row into [fluid | non-fluid] after kinds changed, keeping the
// neighbour SET (and therefore the rebuild schedule) unchanged — the oracle does not
// rebuild on transitions either.  Warp per row; rows whose partition is still valid are skipped.
constexpr int kRepartWarps = 8;
constexpr int kRepartMaxCap = 1024;
// list != nullptr: only the listed rows (k_mark_rows: the rows of the changed particles and of their
// neighbours — the candidate lists are symmetric without ghosts)
template <int M>
__global__ void __launch_bounds__(32 * kRepartWarps) k_repartition_rows(const uint32_t* __restrict__ kmd,
                                                                         uint32_t* __restrict__ nbr,
                                                                         uint32_t* __restrict__ cnt, int cap,
                                                                         size_t n, const uint32_t* __restrict__ list) {
  __shared__ uint32_t buf[kRepartWarps][kRepartMaxCap];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const size_t w = (size_t)blockIdx.x * kRepartWarps + wib;
  if (w >= n) return;  // warp-uniform
  const size_t i = list ? list[w] : w;
  const uint32_t c = cnt[i];
  const uint32_t tot = cnt_total(c), nf_old = cnt_fluid(c);
  uint32_t* row = nbr + i * (size_t)cap;
  uint32_t nf = 0;
  bool bad = false;
  for (uint32_t base = 0; base < tot; base += 32) {
    const uint32_t k = base + lane;
    const bool in = k < tot;
    const bool isf = in && kind_of(kmd[nb_index<M>(row[k])]) == SPHG_FLUID;
    nf += __popc(__ballot_sync(0xffffffffu, isf));
    bad |= in && (isf != (k < nf_old));
  }
  if (!__any_sync(0xffffffffu, bad)) return;
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t fo = 0, oo = 0;
  for (uint32_t base = 0; base < tot; base += 32) {
    const uint32_t k = base + lane;
    const bool in = k < tot;
    const uint32_t e = in ? row[k] : 0u;
    const bool isf = in && kind_of(kmd[nb_index<M>(e)]) == SPHG_FLUID;
    const uint32_t bf = __ballot_sync(0xffffffffu, isf), bo = __ballot_sync(0xffffffffu, in && !isf);
    if (in) buf[wib][isf ? fo + __popc(bf & lt) : nf + oo + __popc(bo & lt)] = e;
    fo += __popc(bf);
    oo += __popc(bo);
  }
  __syncwarp();
  for (uint32_t k = lane; k < tot; k += 32) row[k] = buf[wib][k];
  if (lane == 0) cnt[i] = pack_cnt(nf, tot - nf);
}

// ------------------------------------------------ decomposed batches (sphg.h)
// bodies a batch can touch: the body of a melting particle; every body with a rigid particle (ghosts
// included) within r_c of a solidifying one — a superset of the attach targets (k_solid_target)
__global__ void k_event_bodies(const __grid_constant__ DevParams P, Particles D, size_t n,
                               const uint32_t* __restrict__ ev, NbrList L, uint32_t* __restrict__ mask) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || ev[i] == 0) return;
  if (ev[i] == 1) {
    mask[D.group.p[i]] = 1u;
    return;
  }
  const double4 pi = D.G0.p[i];
  const uint32_t nn = cnt_total(L.cnt[i]);
  const uint32_t* row = L.nbr + (size_t)i * L.cap;
  for (uint32_t k = 0; k < nn; ++k) {
    const uint32_t j = entry_index(P, row[k]);
    if (kind_of(D.kmd.p[j]) != SPHG_RIGID) continue;
    const double4 pj = D.G0.p[j];
    if (r2_exact(mimg3(P, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z)) > P.rc2) continue;
    mask[D.group.p[j]] = 1u;
  }
}

// owned event particles and owned rigid members of the masked bodies
__global__ void k_event_member_flags(Particles D, size_t n, const uint32_t* __restrict__ ev,
                                     const uint32_t* __restrict__ mask, size_t nb, uint32_t* __restrict__ flag) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const uint32_t kmd = D.kmd.p[k];
  const uint32_t g = D.group.p[k];
  const bool member = kind_of(kmd) == SPHG_RIGID && g < nb && mask[g] != 0u;
  flag[k] = (!is_ghost(kmd) && (ev[k] != 0u || member)) ? 1u : 0u;
}

__global__ void k_compact_gid(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos,
                              const uint32_t* __restrict__ gid, size_t n, uint32_t* __restrict__ out) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n && flag[k]) out[pos[k]] = gid[k];
}

// records (sphg.h): [0..2] x, [3] kind, [4] material, [5] group, [6] mass, then the device records
__global__ void k_record_pack(Particles D, const uint32_t* __restrict__ ids, size_t m,
                              const uint32_t* __restrict__ idx, size_t n, double* __restrict__ out,
                              uint32_t* __restrict__ bad) {
  const size_t s = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= m) return;
  double* o = out + s * kRecordDoubles;
  if (ids[s] >= n) {  // device id lists are not checked on the host: flag, never read out of bounds
    atomicMin(bad, (uint32_t)s);
    return;
  }
  const uint32_t k = idx[ids[s]];
  const uint32_t kmd = D.kmd.p[k];
  const double4 g0 = D.G0.p[k];
  o[0] = g0.x; o[1] = g0.y; o[2] = g0.z;
  o[3] = (double)kind_of(kmd);
  o[4] = (double)mat_of(kmd);
  o[5] = (double)D.group.p[k];
  o[6] = D.V4.p[k].w;
  o[7] = g0.w;
  const double4* rec[7] = {&D.G1.p[k], &D.G2.p[k], &D.V4.p[k], &D.A4.p[k], &D.B4.p[k], &D.F4.p[k], &D.X4.p[k]};
#pragma unroll
  for (int r = 0; r < 7; ++r) {
    const double4 v = *rec[r];
    o[8 + 4 * r] = v.x; o[9 + 4 * r] = v.y; o[10 + 4 * r] = v.z; o[11 + 4 * r] = v.w;
  }
  o[36] = D.H2.p[k].x; o[37] = D.H2.p[k].y;
  o[38] = D.dTdt.p[k];
  o[39] = D.p_static.p[k];
  o[40] = D.C2.p ? D.C2.p[k].x : 0.0;
  o[41] = D.C2.p ? D.C2.p[k].y : 0.0;
  o[42] = D.dCdt.p ? D.dCdt.p[k] : 0.0;
  o[43] = (double)(kmd & ~kGhostBit);
}

__global__ void k_record_unpack(Particles D, const uint32_t* __restrict__ ids, size_t m,
                                const uint32_t* __restrict__ idx, size_t n, const double* __restrict__ in,
                                int keep_position, uint32_t* __restrict__ bad) {
  const size_t s = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= m) return;
  if (ids[s] >= n) {
    atomicMin(bad, (uint32_t)s);
    return;
  }
  const uint32_t k = idx[ids[s]];
  const double* o = in + s * kRecordDoubles;
  double4 g0 = D.G0.p[k];
  if (!keep_position) {
    g0.x = o[0]; g0.y = o[1]; g0.z = o[2];
  }
  g0.w = o[7];
  D.G0.p[k] = g0;
  double4* rec[7] = {&D.G1.p[k], &D.G2.p[k], &D.V4.p[k], &D.A4.p[k], &D.B4.p[k], &D.F4.p[k], &D.X4.p[k]};
#pragma unroll
  for (int r = 0; r < 7; ++r) *rec[r] = make_double4(o[8 + 4 * r], o[9 + 4 * r], o[10 + 4 * r], o[11 + 4 * r]);
  D.H2.p[k] = make_double2(o[36], o[37]);
  D.dTdt.p[k] = o[38];
  D.p_static.p[k] = o[39];
  if (D.C2.p) D.C2.p[k] = make_double2(o[40], o[41]);
  if (D.dCdt.p) D.dCdt.p[k] = o[42];
  const uint32_t kmd = (uint32_t)o[43];
  D.kmd.p[k] = (kmd & ~kGhostBit) | (D.kmd.p[k] & kGhostBit);  // the local copy keeps its role
  D.group.p[k] = (uint32_t)o[5];
}

// a whole store from records (sphg_upload_records): record s -> index s, positions included; the first
// n_owned are owned, the rest ghosts; R4 (the Verlet reference) = the position
__global__ void k_record_load(Particles D, size_t n, size_t n_owned, const double* __restrict__ in) {
  const size_t s = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const double* o = in + s * kRecordDoubles;
  D.G0.p[s] = make_double4(o[0], o[1], o[2], o[7]);
  D.R4.p[s] = make_double4(o[0], o[1], o[2], 0.0);
  double4* rec[7] = {&D.G1.p[s], &D.G2.p[s], &D.V4.p[s], &D.A4.p[s], &D.B4.p[s], &D.F4.p[s], &D.X4.p[s]};
#pragma unroll
  for (int r = 0; r < 7; ++r) *rec[r] = make_double4(o[8 + 4 * r], o[9 + 4 * r], o[10 + 4 * r], o[11 + 4 * r]);
  D.H2.p[s] = make_double2(o[36], o[37]);
  D.dTdt.p[s] = o[38];
  D.p_static.p[s] = o[39];
  if (D.C2.p) D.C2.p[s] = make_double2(o[40], o[41]);
  if (D.dCdt.p) D.dCdt.p[s] = o[42];
  const uint32_t kmd = (uint32_t)o[43] & ~kGhostBit;
  D.kmd.p[s] = s >= n_owned ? (kmd | kGhostBit) : kmd;
  D.group.p[s] = (uint32_t)o[5];
}

// validation of records about to be loaded: kind, material and (rigid) body id in range
__global__ void k_record_check(const double* __restrict__ in, size_t n, int n_mat, size_t nb,
                               uint32_t* __restrict__ bad) {
  const size_t s = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const double* o = in + s * kRecordDoubles;
  const bool ok = o[3] >= 0.0 && o[3] <= 2.0 && o[4] >= 0.0 && o[4] < (double)n_mat &&
                  (o[3] != (double)SPHG_RIGID || (o[5] >= 0.0 && o[5] < (double)nb));
  if (!ok) atomicMin(bad, (uint32_t)s);
}

}  // namespace

uint32_t record_check(Ctx& c, const double* dev_recs, size_t n, size_t nb) {
  if (n == 0) return 0xffffffffu;
  c.label_flags.alloc(4);
  SPHG_CUDA_CHECK(cudaMemsetAsync(c.label_flags.p + 2, 0xff, sizeof(uint32_t), c.stream));
  k_record_check<<<grid_for(n, 256), 256, 0, c.stream>>>(dev_recs, n, c.params.n_mat, nb, c.label_flags.p + 2);
  c.launches++;
  return read_u32(c, c.label_flags.p + 2);
}

void record_load(Ctx& c, const double* dev_recs, size_t n, size_t n_owned) {
  if (n == 0) return;
  k_record_load<<<grid_for(n, 128), 128, 0, c.stream>>>(c.cur, n, n_owned, dev_recs);
  c.launches++;
}

void launch_detect(Ctx& c) {
  const size_t n = c.n;
  cudaStream_t s = c.stream;
  c.ev_flag.alloc(std::max<size_t>(n, 1));
  SPHG_CUDA_CHECK(cudaMemsetAsync(&c.dflags->n_events, 0, sizeof(uint32_t), s));
  SPHG_CUDA_CHECK(cudaMemsetAsync(&c.dflags->pad[0], 0, 2 * sizeof(uint32_t), s));
  if (n == 0) return;
  k_detect<<<grid_for(n, 256), 256, 0, s>>>(c.P, c.cur, n, c.ev_flag.p, c.dflags);
  c.launches++;
}

void event_bodies(Ctx& c, uint32_t* dev_mask) {
  if (c.n == 0 || !c.ev_flag.p) return;
  k_event_bodies<<<grid_for(c.n, 128), 128, 0, c.stream>>>(c.P, c.cur, c.n, c.ev_flag.p, c.nl(), dev_mask);
  c.launches++;
}

size_t event_members(Ctx& c, const uint32_t* dev_mask, size_t nb, uint32_t* dev_ids) {
  const size_t n = c.n;
  if (n == 0 || !c.ev_flag.p) return 0;
  uint32_t* flag = c.vals_alt.p;
  uint32_t* pos = c.vals.p;
  k_event_member_flags<<<grid_for(n, 256), 256, 0, c.stream>>>(c.cur, n, c.ev_flag.p, dev_mask, nb, flag);
  exclusive_scan_u32(flag, pos, n, c.scan_tmp.p, c.stream, &c.launches);
  const size_t m = read_sum2(c, pos + n - 1, flag + n - 1);
  if (dev_ids && m) k_compact_gid<<<grid_for(n, 256), 256, 0, c.stream>>>(flag, pos, c.cur.gid.p, n, dev_ids);
  c.launches += 2;
  return m;
}

// returns the first out-of-range id's position, or ~0u
uint32_t record_pack(Ctx& c, const uint32_t* dev_ids, size_t m, double* dev_out) {
  if (m == 0) return 0xffffffffu;
  c.label_flags.alloc(4);
  SPHG_CUDA_CHECK(cudaMemsetAsync(c.label_flags.p + 2, 0xff, sizeof(uint32_t), c.stream));
  k_record_pack<<<grid_for(m, 128), 128, 0, c.stream>>>(c.cur, dev_ids, m, c.idx_of_gid.p, c.n, dev_out,
                                                        c.label_flags.p + 2);
  c.launches++;
  return read_u32(c, c.label_flags.p + 2);
}

uint32_t record_unpack(Ctx& c, const uint32_t* dev_ids, size_t m, const double* dev_in, int keep_position) {
  if (m == 0) return 0xffffffffu;
  c.label_flags.alloc(4);
  SPHG_CUDA_CHECK(cudaMemsetAsync(c.label_flags.p + 2, 0xff, sizeof(uint32_t), c.stream));
  k_record_unpack<<<grid_for(m, 128), 128, 0, c.stream>>>(c.cur, dev_ids, m, c.idx_of_gid.p, c.n, dev_in,
                                                          keep_position, c.label_flags.p + 2);
  c.launches++;
  return read_u32(c, c.label_flags.p + 2);
}

// rows whose fluid / non-fluid partition a batch can invalidate: the changed particles' own rows and the
// rows of their neighbours (= the entries of their rows)
static __global__ void k_mark_rows(const uint32_t* __restrict__ ev, const uint32_t* __restrict__ group,
                                   const uint32_t* __restrict__ group0, size_t n, NbrList L, int img_mode,
                                   uint32_t* __restrict__ dirty) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n || (ev[k] == 0u && group[k] == group0[k])) return;
  dirty[k] = 1u;
  const uint32_t nn = cnt_total(L.cnt[k]);
  const uint32_t* row = L.nbr + k * L.cap;
  for (uint32_t q = 0; q < nn; ++q) dirty[img_mode == kImgCode ? (row[q] & kIdxMask) : row[q]] = 1u;
}

static __global__ void k_compact_flagged(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos,
                                         size_t n, uint32_t* __restrict__ out) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n && flag[k]) out[pos[k]] = (uint32_t)k;
}

static __global__ void k_rigid_of(const uint32_t* __restrict__ list, size_t m, const uint32_t* __restrict__ kmd,
                                  uint32_t* __restrict__ flag) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < m) flag[e] = kind_of(kmd[list[e]]) == SPHG_RIGID ? 1u : 0u;
}

static __global__ void k_compact_list(const uint32_t* __restrict__ list, const uint32_t* __restrict__ flag,
                                      const uint32_t* __restrict__ pos, size_t m, uint32_t* __restrict__ out) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < m && flag[e]) out[pos[e]] = list[e];
}

static void repartition_launch(Ctx& c, size_t m, const uint32_t* list) {
  const unsigned blocks = (unsigned)((m + kRepartWarps - 1) / kRepartWarps);
  switch (c.P.img_mode) {
    case kImgNone: k_repartition_rows<kImgNone><<<blocks, 32 * kRepartWarps, 0, c.stream>>>(c.cur.kmd.p, c.nbr.p, c.cnt.p, c.cap, m, list); break;
    case kImgCode: k_repartition_rows<kImgCode><<<blocks, 32 * kRepartWarps, 0, c.stream>>>(c.cur.kmd.p, c.nbr.p, c.cnt.p, c.cap, m, list); break;
    default: k_repartition_rows<kImgMin><<<blocks, 32 * kRepartWarps, 0, c.stream>>>(c.cur.kmd.p, c.nbr.p, c.cnt.p, c.cap, m, list); break;
  }
  c.launches++;
}

void launch_repartition_rows(Ctx& c) {
  if (c.n == 0) return;
  if (c.cap > kRepartMaxCap) {  // very wide rows: rebuild instead
    c.built = false;
    return;
  }
  repartition_launch(c, c.n, nullptr);
}

// After a single-rank batch only the rows of the particles whose kind or body changed, and of their
// neighbours (the candidate lists are symmetric without ghosts), can hold a stale fluid / non-fluid
// partition or contact order: re-partition those rows and re-order the rigid ones among them.
// group0 = the body ids before the batch.
static void refresh_changed_rows(Ctx& c, const uint32_t* group0) {
  const size_t n = c.n;
  if (n == 0) return;
  static const bool all_rows = std::getenv("SPHG_REPART_ALL") && std::atoi(std::getenv("SPHG_REPART_ALL")) != 0;
  if (c.cap > kRepartMaxCap || c.nghost || all_rows || !group0) {
    launch_repartition_rows(c);
    if (c.built) launch_contact_order(c);
    return;
  }
  uint32_t* dirty = c.vals_alt.p;
  uint32_t* pos = c.vals.p;
  SPHG_CUDA_CHECK(cudaMemsetAsync(dirty, 0, n * sizeof(uint32_t), c.stream));
  k_mark_rows<<<grid_for(n, 256), 256, 0, c.stream>>>(c.ev_flag.p, c.cur.group.p, group0, n, c.nl(), c.P.img_mode,
                                                       dirty);
  exclusive_scan_u32(dirty, pos, n, c.scan_tmp.p, c.stream, &c.launches);
  const size_t m = read_sum2(c, pos + n - 1, dirty + n - 1);
  c.launches++;
  if (m == 0) return;
  c.rec_ids.alloc(2 * m + 1);
  uint32_t* rows = c.rec_ids.p;
  k_compact_flagged<<<grid_for(n, 256), 256, 0, c.stream>>>(dirty, pos, n, rows);
  c.launches++;
  repartition_launch(c, m, rows);
  if (!c.built || c.nrigid == 0) return;
  // the rigid ones among them: contact candidates first again
  uint32_t* rflag = dirty;  // reused: m <= n
  uint32_t* rpos = pos;
  k_rigid_of<<<grid_for(m, 256), 256, 0, c.stream>>>(rows, m, c.cur.kmd.p, rflag);
  exclusive_scan_u32(rflag, rpos, m, c.scan_tmp.p, c.stream, &c.launches);
  const size_t mr = read_sum2(c, rpos + m - 1, rflag + m - 1);
  if (mr == 0) return;
  uint32_t* rl = rows + m;
  k_compact_list<<<grid_for(m, 256), 256, 0, c.stream>>>(rows, rflag, rpos, m, rl);
  c.launches += 2;
  launch_contact_order(c, rl, mr);
}

int launch_transitions(Ctx& c) {
  NvtxRange nv("transitions");
  const size_t n = c.n;
  cudaStream_t s = c.stream;
  if (n == 0) return 0;
  launch_detect(c);
  uint32_t nmelt = 0, nsolid = 0;
  read_u32x2(c, &c.dflags->n_events, &c.dflags->pad[0], nmelt, nsolid);
  if (nmelt == 0 && nsolid == 0) return 0;
  if (!c.built) launch_rebuild(c);
  c.group0.alloc(n);  // body ids before the batch (refresh_changed_rows)
  SPHG_CUDA_CHECK(cudaMemcpyAsync(c.group0.p, c.cur.group.p, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
  const size_t nb0 = c.nb;
  // capacity: spawned + split products are bounded by the rigid count after the batch
  grow_bodies(c, nb0 + nsolid + c.nrigid + nsolid + 1);
  const size_t cap = c.bodies_cap;
  // the pre-batch body table (u'_k, r'_k): a grow-only context buffer — a per-batch cudaMalloc / cudaFree
  // of the table's capacity (~1 GB at C4's bound) would synchronise the device and cost milliseconds
  DBuf<sphg_body>& old = c.bodies_old;
  old.alloc(cap);
  c.tscratch.alloc(3 * cap + 3 * (size_t)std::max<uint32_t>(nsolid, 1));
  uint32_t* bmask = c.tscratch.p;
  uint32_t* blost = bmask + cap;
  uint32_t* src = blost + cap;
  int* target = reinterpret_cast<int*>(src + cap);
  uint32_t* spawn = reinterpret_cast<uint32_t*>(target + std::max<uint32_t>(nsolid, 1));
  uint32_t* rank = spawn + std::max<uint32_t>(nsolid, 1);
  SPHG_CUDA_CHECK(cudaMemsetAsync(bmask, 0, 2 * cap * sizeof(uint32_t), s));
  k_iota<<<grid_for(cap, 256), 256, 0, s>>>(src, cap, 0);
  if (nb0) SPHG_CUDA_CHECK(cudaMemcpyAsync(old.p, c.bodies.p, nb0 * sizeof(sphg_body), cudaMemcpyDeviceToDevice, s));
  // event log (sphg_set_event_log): this batch's events, drained to the host at the end of the batch
  sphg_event* elog = nullptr;
  uint32_t* nlog = nullptr;
  if (c.event_log) {
    c.ev_log.alloc(nmelt + nsolid + 1);
    c.ev_count.alloc(1);
    SPHG_CUDA_CHECK(cudaMemsetAsync(c.ev_count.p, 0, sizeof(uint32_t), s));
    elog = c.ev_log.p;
    nlog = c.ev_count.p;
  }
  const int64_t step = c.steps + 1;
  // 1. melt
  if (nmelt)
    k_melt<<<grid_for(n, 256), 256, 0, s>>>(c.P, c.cur, n, c.ev_flag.p, c.bodies.p, bmask, blost, elog, nlog, step);
  // 2. solidify: events in gid order, attach or spawn
  size_t nspawn = 0;
  if (nsolid) {
    uint32_t* flag = c.vals_alt.p;
    uint32_t* pos = c.vals.p;
    k_flag_eq<<<grid_for(n, 256), 256, 0, s>>>(c.ev_flag.p, n, 2u, flag);
    exclusive_scan_u32(flag, pos, n, c.scan_tmp.p, s, &c.launches);
    k_compact_by_gid<<<grid_for(n, 256), 256, 0, s>>>(c.ev_flag.p, pos, n, 2u, c.cur.gid.p, c.keys.p, c.vals_alt.p);
    const bool fl = radix_sort_pairs(c.keys.p, c.vals_alt.p, c.keys_alt.p, c.vals.p, nsolid, bits_for(n - 1), c.hist.p,
                                     c.scan_tmp.p, s, &c.launches);
    uint32_t* list = fl ? c.vals.p : c.vals_alt.p;
    c.ev_idx.alloc(nsolid);
    SPHG_CUDA_CHECK(cudaMemcpyAsync(c.ev_idx.p, list, nsolid * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
    k_solid_target<<<grid_for(nsolid, 128), 128, 0, s>>>(c.P, c.cur, c.ev_idx.p, nsolid, c.nl(), target, spawn);
    exclusive_scan_u32(spawn, rank, nsolid, c.scan_tmp.p, s, &c.launches);
    nspawn = read_sum2(c, rank + nsolid - 1, spawn + nsolid - 1);
    k_solid_apply<<<grid_for(nsolid, 128), 128, 0, s>>>(c.P, c.cur, c.ev_idx.p, nsolid, target, rank, nb0,
                                                        c.bodies.p, bmask, src);
    c.launches += 5;
  }
  c.nb = nb0 + nspawn;
  launch_rigid_index(c);
  // 3. split bodies that lost particles
  if (nmelt) {
    c.label.alloc(n);
    c.label_list.alloc(n);
    c.label_flags.alloc(4);
    SPHG_CUDA_CHECK(cudaMemsetAsync(c.label_flags.p, 0, 4 * sizeof(uint32_t), s));
    k_label_init<<<grid_for(n, 256), 256, 0, s>>>(c.cur, n, blost, c.label.p, c.label_list.p, c.label_flags.p + 3);
    const double adj2 = (1.5 * c.P.dx) * (1.5 * c.P.dx);
    // one cooperative launch: as many blocks as the labelled particles need (each sweep ends in two grid
    // barriers, whose cost grows with the grid), at most as many as can be co-resident
    const uint32_t nlab = read_u32(c, c.label_flags.p + 3);
    static int coop_blocks = 0;
    if (!coop_blocks) {
      int per_sm = 0, sms = 0;
      SPHG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_label_coop, 256, 0));
      SPHG_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device));
      coop_blocks = std::max(1, per_sm) * sms;
    }
    DevParams Pv = c.P;
    Particles Dv = c.cur;
    NbrList Lv = c.nl();
    const uint32_t* lp = c.label_list.p;
    const uint32_t* cp = c.label_flags.p + 3;
    uint32_t* labp = c.label.p;
    double a2 = adj2;
    uint32_t* fp = c.label_flags.p;
    c.label_adj.alloc((size_t)std::max<uint32_t>(nlab, 1) * (kAdjMax + 1));
    uint32_t* adjp = c.label_adj.p;
    uint32_t* nadjp = adjp + (size_t)std::max<uint32_t>(nlab, 1) * kAdjMax;
    const uint32_t* idxp = c.idx_of_gid.p;
    if (nlab) {
      k_label_adj<<<grid_for(nlab, 128), 128, 0, s>>>(c.P, c.cur, c.nl(), lp, cp, adj2, adjp, nadjp);
      c.launches++;
    }
    void* args[] = {&Pv, &Dv, &Lv, &lp, &cp, &labp, &a2, &fp, &adjp, &nadjp, &idxp};
    const int blocks = std::max(1, std::min(coop_blocks, (int)((nlab + 255) / 256)));
    SPHG_CUDA_CHECK(cudaLaunchCooperativeKernel((const void*)k_label_coop, dim3(blocks), dim3(256), args, 0, s));
    c.launches += 2;
    const int gbits = bits_for(n - 1);
    k_split_roots<<<grid_for(n, 256), 256, 0, s>>>(c.cur, n, c.label.p, c.ridx.p, c.body_start.p, gbits, c.keys.p,
                                                   c.vals.p, c.dflags);
    const uint32_t nsplit = read_u32(c, &c.dflags->pad[1]);
    if (nsplit) {
      const int bits = gbits + bits_for(c.nb);
      const bool fl = radix_sort_pairs(c.keys.p, c.vals.p, c.keys_alt.p, c.vals_alt.p, nsplit, bits, c.hist.p,
                                       c.scan_tmp.p, s, &c.launches);
      const unsigned long long* keys = fl ? c.keys_alt.p : c.keys.p;
      k_split_bodies<<<grid_for(nsplit, 128), 128, 0, s>>>(keys, nsplit, gbits, c.nb, c.bodies.p, bmask, src);
      k_split_relabel<<<grid_for(n, 256), 256, 0, s>>>(c.cur, n, c.label.p, c.ridx.p, c.body_start.p, keys, nsplit,
                                                       gbits, c.nb);
      // old state of split products = their source body's pre-batch state (via src)
      c.nb += nsplit;
      launch_rigid_index(c, false);
      c.launches += 2;
    }
  }
  if (elog && nsolid) {
    k_log_solid<<<grid_for(nsolid, 128), 128, 0, s>>>(c.cur, c.ev_idx.p, nsolid, elog, nlog, step);
    c.launches++;
  }
  // 4. mass quantities + post-transition velocity + member velocities
  launch_mass(c, bmask);
  k_post_velocity<<<grid_for(c.nb, 128), 128, 0, s>>>(c.P, c.bodies.p, old.p, bmask, src, c.nb, nb0);
  k_member_velocity<<<grid_for(n, 256), 256, 0, s>>>(c.cur, n, c.bodies.p, bmask);
  c.launches += 4;
  // 5. force/torque with the new membership
  launch_bodies(c);
  host_sync(c, s);
  if (elog) {  // drain this batch's events to the host, ordered by gid (each particle once per batch)
    const size_t m = (size_t)nmelt + nsolid;
    std::vector<sphg_event> ev(m);
    SPHG_CUDA_CHECK(cudaMemcpy(ev.data(), elog, m * sizeof(sphg_event), cudaMemcpyDeviceToHost));
    std::sort(ev.begin(), ev.end(), [](const sphg_event& a, const sphg_event& b) { return a.gid < b.gid; });
    c.events.insert(c.events.end(), ev.begin(), ev.end());
  }
  c.n_melt += nmelt;
  c.n_solid += nsolid;
  // kinds changed: the rows' fluid / non-fluid partition is stale; body ids changed: contact order
  refresh_changed_rows(c, c.built ? c.group0.p : nullptr);
  check_structures(c);
  return 0;
}

}  // namespace sphg
