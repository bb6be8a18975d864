// kernels_pairs.cu — the pair-sum kernels of the SPH hot path on sm_100a.
//
//   k_density       density_summation + eos_pressure
//   k_heat          conduction_rhs + explicit T update
//   k_heat_source   moving Gaussian surface heat flux (C4)      ([P21]; an extension, no reference counterpart)
//   k_diffusion     diffusion_rhs + explicit C update
//   k_extrapolate   extrapolate_wall_quantities                 (Adami 2012)
//   k_forces_fluid  momentum_rhs with transport velocity
//                   (+ the fluid conduction sums inside sphg_step, kHeat)
//   k_forces_rigid  coupling_force_on_rigid + contact_force
//   k_count_pairs   Verlet candidates / pairs within r_c (bench flop model)
//
// Parallelisation: a group of G consecutive lanes owns one particle i and
// strides over its Verlet row (nbr[i*cap + k]); the rows list neighbours in
// cell-run order, so the G lanes gather G (mostly) consecutive particles — a
// few cache lines per warp load instead of one line per lane.  Partial sums
// are combined with warp shuffles (gsum); lane 0 of the group writes.  Every
// sum is a gather (no fp64 atomics), hence deterministic.  Groups iterate over
// compact per-kind index lists (fluid / non-fluid in brick order, rigid body-major) built at
// rebuild.  These kernels are gather-bound, not FP64-bound (a loads-only twin of
// k_forces_fluid takes 97 % of its time).  The two big passes (density, fluid forces) run as
// SM-local persistent grids (k_density_sm, k_forces_fluid_sm): the warps of one SM take adjacent
// tiles of the brick-ordered list, so the records they gather stay in that SM's L1.
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "context.cuh"

namespace sphg {

namespace {

constexpr int kBlock = 128;


__device__ __forceinline__ double3 ld3(const double4& v) { return make_double3(v.x, v.y, v.z); }
// One 32-byte load per particle record (sm_100 LDG.E.ENL2.256): a record is one
// sector, so a gather costs one sector instead of two 16-byte requests.
__device__ __forceinline__ double4 ldg4(const double4* p) {  // read-only (non-coherent) path
  double4 v;
#ifdef SPHG_REC_EVICT_LAST
  asm("ld.global.nc.L1::evict_last.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
#else
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
#endif
  return v;
}
// a Verlet row entry (rows stream from HBM once per pass)
__device__ __forceinline__ uint32_t ldrow(const uint32_t* p) {
#ifdef SPHG_ROW_EVICT_FIRST
  uint32_t v;
  asm("ld.global.nc.L1::evict_first.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
#else
  return __ldg(p);
#endif
}
__device__ __forceinline__ double4 ld4(const double4* p) {  // coherent path (array written in-kernel)
  double4 v;
  asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}
// xyz of a record whose .w may be written concurrently by its owner (density,
// extrapolation): the 32-byte load is atomic per 8-byte word and .w is unused.
__device__ __forceinline__ double3 ldpos(const double4* p) { return ld3(ld4(p)); }
__device__ __forceinline__ Quat body_q(const sphg_body& b) { return {b.q[0], b.q[1], b.q[2], b.q[3]}; }
__device__ __forceinline__ double3 bv(const double* p) { return make_double3(p[0], p[1], p[2]); }

// A Verlet row: fluid neighbours f[0..nf), rigid/boundary neighbours b[0..no) with b = f + nf.
struct Row {
  const uint32_t* f;
  const uint32_t* b;
  int nf, no, n;
  __device__ __forceinline__ uint32_t at(int k) const { return ldrow(f + k); }
};
__device__ __forceinline__ Row row_of(const NbrList& L, uint32_t i) {
  const uint32_t c = L.cnt[i];
  const uint32_t* r = L.nbr + (size_t)i * L.cap;
  Row R;
  R.f = r;
  R.b = r + cnt_fluid(c);
  R.nf = (int)cnt_fluid(c);
  R.no = (int)cnt_other(c);
  R.n = R.nf + R.no;
  return R;
}

// ---------------------------------------------------------------- density
template <int M>
__device__ __forceinline__ double density_term(const DevParams& P, double3 pi, double3 pj, uint32_t e) {
  const double3 d = pair_delta<M>(P, pi, pj, e);
  const double r2 = d.x * d.x + d.y * d.y + d.z * d.z;
  if (r2 > P.rc2) return 0.0;
  // accurate r: p = c^2 (rho - rho0) cancels, so the pressure (and every force term built on it)
  // needs rho to ~1e-15, not just 1e-10; + tiny: coincident -> W(0)
  double ri;
  return shape_q(pair_qr(d, r2, P.inv_h, ri));
}

// rho_i = m_i sigma (66 + sum_j shape(r_ij/h)); p_i = c^2 (rho_i - rho0); V_i = m_i/rho_i
// (j over neighbours of any kind)
template <int G, int M>
__device__ __forceinline__ void density_group(const DevParams& P, const Particles& D, const NbrList& L,
                                              const uint32_t* __restrict__ list, size_t nlist, size_t g, int lane) {
  const bool active = g < nlist;
  const uint32_t i = active ? list[g] : 0u;
  double s = 0.0;
  if (active) {
    const double3 pi = ldpos(&D.G0.p[i]);
    const Row R = row_of(L, i);
    int k = lane;
    // two independent gathers in flight; the next pair of row entries is prefetched
    uint32_t e0 = k < R.n ? R.at(k) : 0u;
    uint32_t e1 = k + G < R.n ? R.at(k + G) : 0u;
    for (; k + G < R.n; k += 2 * G) {
      const uint32_t f0 = k + 2 * G < R.n ? R.at(k + 2 * G) : 0u;
      const uint32_t f1 = k + 3 * G < R.n ? R.at(k + 3 * G) : 0u;
      const double3 p0 = ldpos(&D.G0.p[nb_index<M>(e0)]);
      const double3 p1 = ldpos(&D.G0.p[nb_index<M>(e1)]);
      s += density_term<M>(P, pi, p0, e0);
      s += density_term<M>(P, pi, p1, e1);
      e0 = f0;
      e1 = f1;
    }
    if (k < R.n) s += density_term<M>(P, pi, ldpos(&D.G0.p[nb_index<M>(e0)]), e0);
  }
  s = gsum<G>(s);
  if (!active || lane != 0) return;
  const uint32_t kmd = D.kmd.p[i];
  const DevMat& Mt = P.mat[mat_of(kmd)];
  const double m = D.V4.p[i].w;
  const double rho = m * (P.sigma * (66.0 + s));  // self term shape(0) = 66
  const double V = m / rho;
  reinterpret_cast<double*>(&D.G0.p[i])[3] = V * V;
  reinterpret_cast<double*>(&D.G1.p[i])[3] = rho;
  reinterpret_cast<double*>(&D.G2.p[i])[3] = Mt.c2 * (rho - Mt.rho0);
  if (P.thermal) reinterpret_cast<double*>(&D.H2.p[i])[1] = V;
  if (P.diffusion) reinterpret_cast<double*>(&D.C2.p[i])[1] = V;
}

template <int G, int M>
__global__ void __launch_bounds__(kBlock) k_density(const __grid_constant__ DevParams P, Particles D, NbrList L,
                                                     const uint32_t* __restrict__ list, size_t nlist) {
  SPHG_SKIP_IF_FLAGGED(P);
  const size_t t = (size_t)blockIdx.x * kBlock + threadIdx.x;
  density_group<G, M>(P, D, L, list, nlist, t / G, (int)(t % G));
}

// SM-local persistent variants (the 4-lane density, fluid forces, extrapolation, rigid forces and conduction
// passes over lists of sm_local_min particles or more; SPHG_SM_LOCAL=0 restores one group per thread of a
// flat grid): the list is cut into one contiguous range per SM and the resident warps
// of an SM take 8-particle tiles of its range in order (next[q], zeroed before the launch).  The list is in
// brick order (2x2x2 blocks of cells, common.cuh), so the ~190 particles in flight on an SM share one
// 4x4x4-cell neighbourhood that stays in that SM's L1, where a flat grid's co-resident blocks sit 148 blocks
// apart in the list.  A warp whose range is finished helps the next ranges.  Each particle is still summed by
// its own 4 lanes in row order: results are bit-identical to the flat grid's.
template <int G, int M>
__global__ void __launch_bounds__(kBlock) k_density_sm(const __grid_constant__ DevParams P, Particles D, NbrList L,
                                                        const uint32_t* __restrict__ list, size_t nlist,
                                                        uint32_t* __restrict__ next, int nq) {
  SPHG_SKIP_IF_FLAGGED(P);
  const int lw = threadIdx.x & 31;
  int q = (int)(sm_id() % (unsigned)nq);
  size_t tile;
  constexpr int T = 32 / G;  // particles per warp tile
  while (next_tile(next, nq, (nlist + T - 1) / T, q, tile))
    density_group<G, M>(P, D, L, list, nlist, tile * T + lw / G, lw % G);
}

// ------------------------------------------------------------------- heat
// c_p,a dT_a/dt = (1/rho_a) sum_b V_b 4 k_a k_b/(k_a+k_b) (T_ab/r_ab) dW/dr (Cleary & Monaghan).
// b over fluid, rigid and Dirichlet boundary particles (V_heat == 0 marks the others).
template <int G, int M>
__device__ __forceinline__ void heat_group(const DevParams& P, const Particles& D, const NbrList& L,
                                           const uint32_t* __restrict__ list, size_t nlist,
                                           double2* __restrict__ Hout, DevFlags* __restrict__ fl, size_t t) {
  const size_t g = t / G;
  const int lane = (int)(t % G);
  const bool active = g < nlist;
  const uint32_t i = active ? list[g] : 0u;
  double s = 0.0;
  bool coincident = false;
  uint32_t kmd = 0;
  double2 hi = make_double2(0, 0);
  if (active) {
    kmd = D.kmd.p[i];
    const DevMat& Ma = P.mat[mat_of(kmd)];
    hi = D.H2.p[i];
    const double3 pi = ldpos(&D.G0.p[i]);
    const Row R = row_of(L, i);
    uint32_t en = lane < R.n ? R.at(lane) : 0u;
    for (int k = lane; k < R.n; k += G) {
      const uint32_t e = en;
      en = k + G < R.n ? R.at(k + G) : 0u;
      const uint32_t j = nb_index<M>(e);
      const double2 hj = D.H2.p[j];
      if (hj.y == 0.0) continue;  // non-Dirichlet wall: no conduction
      const double3 d = pair_delta<M>(P, pi, ld3(ldg4(&D.G0.p[j])), e);  // G0 is read-only here
      const double r2 = d.x * d.x + d.y * d.y + d.z * d.z;
      if (r2 > P.rc2) continue;
      if (r2 == 0.0) {
        coincident = true;
        continue;
      }
      double kt;
      if (P.single_kappa) {
        kt = 2.0 * Ma.kappa;  // 4 k k / (k + k)
      } else {
        const double kb = P.mat[mat_of(D.kmd.p[j])].kappa;
        const double ks = Ma.kappa + kb;
        if (ks == 0.0) continue;
        kt = 4.0 * Ma.kappa * kb / ks;
      }
      double rinv;
      const double dW = P.sig_h * shape_deriv_q(pair_qr(d, r2, P.inv_h, rinv));
      s += hj.y * kt * ((hi.x - hj.x) * rinv) * dW;
    }
  }
  s = gsum<G>(s);
  if (!active) return;
  if (coincident) {
    atomicOr(&fl->err, kErrCoincident);
    atomicMin(&fl->err_gid, D.gid.p[i]);
  }
  if (lane != 0) return;
  const DevMat& Ma = P.mat[mat_of(kmd)];
  const uint32_t kind = kind_of(kmd);
  const double rho_a = kind == SPHG_FLUID ? D.G1.p[i].w : Ma.rho0;
  double rate = 0.0;
  if (Ma.cp > 0.0) {
    rate = s / (rho_a * Ma.cp);
    if (P.heat_source) rate += P.hsrc[i];  // [P21]
  }
  Hout[i] = make_double2(hi.x + P.dt * rate, hi.y);
  D.dTdt.p[i] = rate;
}

template <int G, int M>
__global__ void __launch_bounds__(kBlock) k_heat(const __grid_constant__ DevParams P, Particles D, NbrList L,
                                                  const uint32_t* __restrict__ list, size_t nlist,
                                                  double2* __restrict__ Hout, DevFlags* __restrict__ fl) {
  SPHG_SKIP_IF_FLAGGED(P);
  heat_group<G, M>(P, D, L, list, nlist, Hout, fl, (size_t)blockIdx.x * kBlock + threadIdx.x);
}

// on an SM-local persistent grid (see k_density_sm); the rigid list is body-major, a grain's particles adjacent
template <int M>
__global__ void __launch_bounds__(kBlock) k_heat_sm(const __grid_constant__ DevParams P, Particles D, NbrList L,
                                                     const uint32_t* __restrict__ list, size_t nlist,
                                                     double2* __restrict__ Hout, DevFlags* __restrict__ fl,
                                                     uint32_t* __restrict__ next, int nq) {
  SPHG_SKIP_IF_FLAGGED(P);
  int q = (int)(sm_id() % (unsigned)nq);
  size_t tile;
  while (next_tile(next, nq, (nlist + 7) / 8, q, tile))
    heat_group<4, M>(P, D, L, list, nlist, Hout, fl, tile * 32 + (threadIdx.x & 31));
}

// ------------------------------------------------------- surface heat flux
// Moving Gaussian surface heat flux [P21] (BASELINE C4; the reference has no heat sources): source
// rate q(x_i, y_i, t^{n+1}) dx^2 / (m_i c_p,i) of an exposed absorbing particle into P.hsrc[i], 0
// otherwise.  Exposure: no mask-material neighbour within r_c above i (sphg.h); a discrete decision,
// so the geometry uses the pinned no-FMA arithmetic of the oracle.  Groups outside 4 r0 of the spot
// skip their row.  t_dev (graph replay): t^{n+1} from device memory.
template <int G>
__global__ void __launch_bounds__(kBlock) k_heat_source(const __grid_constant__ DevParams P, Particles D, NbrList L,
                                                         const uint32_t* __restrict__ list, size_t nlist,
                                                         double t_new, const double* __restrict__ t_dev) {
  SPHG_SKIP_IF_FLAGGED(P);
  const size_t t = (size_t)blockIdx.x * kBlock + threadIdx.x;
  const size_t g = t / G;
  const int lane = (int)(t % G);
  const bool active = g < nlist;
  const uint32_t i = active ? list[g] : 0u;
  if (t_dev) t_new = *t_dev;
  bool absorbs = false;
  double rho2 = 0.0, blocked = 0.0;
  uint32_t kmd = 0;
  if (active) {
    kmd = D.kmd.p[i];
    absorbs = ((P.hs_mask >> mat_of(kmd)) & 1u) && kind_of(kmd) != SPHG_BOUNDARY && P.mat[mat_of(kmd)].cp > 0.0;
  }
  double3 pi = make_double3(0, 0, 0);
  if (absorbs) {
    pi = ldpos(&D.G0.p[i]);
    const double pxy[2] = {pi.x, pi.y};
    for (int a = 0; a < 2; ++a) {
      double c = __dadd_rn(P.hs_origin[a], __dmul_rn(P.hs_vel[a], t_new));
      if (P.periodic[a]) {
        const double u = __dsub_rn(c, P.lo[a]);
        c = __dsub_rn(__dadd_rn(P.lo[a], u), __dmul_rn(P.L[a], floor(__ddiv_rn(u, P.L[a]))));
      }
      const double d = mimg(P, __dsub_rn(pxy[a], c), a);
      rho2 = __dadd_rn(rho2, __dmul_rn(d, d));
    }
    absorbs = !(rho2 > P.hs_cut2);
  }
  if (absorbs) {
    const Row R = row_of(L, i);
    for (int k = lane; k < R.n && blocked == 0.0; k += G) {
      const uint32_t j = R.at(k) & (P.img_mode == kImgCode ? kIdxMask : 0xffffffffu);
      if (!((P.hs_mask >> mat_of(D.kmd.p[j])) & 1u)) continue;
      const double3 pj = ldpos(&D.G0.p[j]);
      const double3 d = mimg3(P, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z);  // r_i - r_j
      if (r2_exact(d) > P.rc2) continue;
      if (-d.z > P.hs_dz && __dadd_rn(__dmul_rn(d.x, d.x), __dmul_rn(d.y, d.y)) < P.hs_lat2) blocked = 1.0;
    }
  }
  blocked = gsum<G>(blocked);
  if (!active || lane != 0) return;
  double q = 0.0;
  if (absorbs && blocked == 0.0) {
    const double e = exp(-2.0 * rho2 / P.hs_r0sq);
    q = P.hs_q0 * e * (P.dx * P.dx) / (D.V4.p[i].w * P.mat[mat_of(kmd)].cp);
  }
  P.hsrc[i] = q;
}

// --------------------------------------------------------------- diffusion
// dC_a/dt = (1/rho_a) sum_b V_b 4 D_a D_b/(D_a+D_b) (C_ab/r_ab) dW/dr (Remark 2.3),
// b over fluid, rigid and Dirichlet-C boundary particles (V_diff == 0 marks the others).  Particles
// in a Dirichlet-C group keep C^ (already set at t^{n+1}) [P18].
template <int G, int M>
__global__ void __launch_bounds__(kBlock) k_diffusion(const __grid_constant__ DevParams P, Particles D, NbrList L,
                                                       const uint32_t* __restrict__ list, size_t nlist,
                                                       double2* __restrict__ Cout, DevFlags* __restrict__ fl) {
  SPHG_SKIP_IF_FLAGGED(P);
  const size_t t = (size_t)blockIdx.x * kBlock + threadIdx.x;
  const size_t g = t / G;
  const int lane = (int)(t % G);
  const bool active = g < nlist;
  const uint32_t i = active ? list[g] : 0u;
  double s = 0.0;
  bool coincident = false;
  uint32_t kmd = 0;
  double2 ci = make_double2(0, 0);
  if (active) {
    kmd = D.kmd.p[i];
    const double Da = P.mat[mat_of(kmd)].D;
    ci = D.C2.p[i];
    const double3 pi = ldpos(&D.G0.p[i]);
    const Row R = row_of(L, i);
    uint32_t en = lane < R.n ? R.at(lane) : 0u;
    for (int k = lane; k < R.n; k += G) {
      const uint32_t e = en;
      en = k + G < R.n ? R.at(k + G) : 0u;
      const uint32_t j = nb_index<M>(e);
      const double2 cj = D.C2.p[j];
      if (cj.y == 0.0) continue;  // boundary without a concentration group
      const double3 d = pair_delta<M>(P, pi, ld3(ldg4(&D.G0.p[j])), e);  // G0 is read-only here
      const double r2 = d.x * d.x + d.y * d.y + d.z * d.z;
      if (r2 > P.rc2) continue;
      if (r2 == 0.0) {
        coincident = true;
        continue;
      }
      const double Db = P.mat[mat_of(D.kmd.p[j])].D;
      const double ds = Da + Db;
      if (ds == 0.0) continue;
      const double dt_ = 4.0 * Da * Db / ds;
      double rinv;
      const double dW = P.sig_h * shape_deriv_q(pair_qr(d, r2, P.inv_h, rinv));
      s += cj.y * dt_ * ((ci.x - cj.x) * rinv) * dW;
    }
  }
  s = gsum<G>(s);
  if (!active) return;
  if (coincident) {
    atomicOr(&fl->err, kErrCoincident);
    atomicMin(&fl->err_gid, D.gid.p[i]);
  }
  if (lane != 0) return;
  const DevMat& Ma = P.mat[mat_of(kmd)];
  const double rho_a = kind_of(kmd) == SPHG_FLUID ? D.G1.p[i].w : Ma.rho0;
  const double rate = s / rho_a;
  const bool fixed = dirc_of(kmd) != SPHG_NO_DIRICHLET && (int)dirc_of(kmd) < P.n_schedC &&
                     P.schedC[dirc_of(kmd)].n > 0;
  Cout[i] = make_double2(fixed ? ci.x : ci.x + P.dt * rate, ci.y);
  D.dCdt.p[i] = rate;
}

// ---------------------------------------------------------- extrapolation
// p_w = sum_f W (p_f + rho_f (g_f - a_w).(r_w - r_f)) / sum_f W;  u~_w = 2 u_w - sum_f W u_f / sum_f W;
// rho_w = max(rho0, rho0 + p_w/c^2) of the dominant fluid material; V_w = rho0 dx^3 / rho_w  [P6][P7]
// Only the fluid part of the row is visited.
// kPin = false: the sums with the fast root; a particle whose fluid pairs all sit within 2e-4 below
// r_c^2 is appended to pin_list and not written (there the weights' relative errors ~15 eps/(3-q)
// reach the ratios; a lone weight can even be 0 on one side and tiny on the other).  kPin = true: only those particles, with
// pinned_q (see common.cuh).
// t: the thread's slot (group t / G, lane t % G); called by whole warps
template <int G, int M, bool kMultiEos, bool kPin>
__device__ __forceinline__ void extrapolate_group(const DevParams& P, const Particles& D, const NbrList& L,
                                                  const sphg_body* __restrict__ B,
                                                  const uint32_t* __restrict__ list, size_t nlist,
                                                  uint32_t* __restrict__ pin_list, uint32_t* __restrict__ any,
                                                  size_t t) {
  const size_t g = t / G;
  const int lane = (int)(t % G);
  const uint32_t w = g < nlist ? list[g] : 0u;
  const bool active = g < nlist;
  double3 uw = make_double3(0, 0, 0), aw = make_double3(0, 0, 0);
  double sw = 0.0, sp = 0.0;
  double3 su = make_double3(0, 0, 0);
  double smat[kMultiEos ? kMaxMat : 1];
#pragma unroll
  for (int m = 0; m < (kMultiEos ? kMaxMat : 1); ++m) smat[m] = 0.0;
  int st = 0;  // 2: a fluid pair clearly inside r_c, 1: only pairs in the 2e-4 band below r_c^2, 0: none
  if (active) {
    const uint32_t kmd = D.kmd.p[w];
    if (kind_of(kmd) == SPHG_BOUNDARY && P.n_walls > 0) {  // prescribed wall motion [P20]
      const uint32_t gr = D.group.p[w];
      if (gr < (uint32_t)P.n_walls) {
        uw = make_double3(P.wall_v[gr][0], P.wall_v[gr][1], P.wall_v[gr][2]);
        aw = make_double3(P.wall_a[gr][0], P.wall_a[gr][1], P.wall_a[gr][2]);
      }
    }
    if (kind_of(kmd) == SPHG_RIGID) {
      const sphg_body& b = B[D.group.p[w]];
      const double3 rk = qrotate(body_q(b), ld3(D.X4.p[w]));
      const double3 om = bv(b.omega);
      const double3 t1 = cross3(bv(b.alpha), rk);
      const double3 t2 = cross3(om, cross3(om, rk));
      aw = make_double3(b.acc[0] + t1.x + t2.x, b.acc[1] + t1.y + t2.y, b.acc[2] + t1.z + t2.z);
      uw = ldpos(&D.V4.p[w]);
    }
    const double3 pw = ldpos(&D.G0.p[w]);
    const Row R = row_of(L, w);
    uint32_t en = lane < R.nf ? __ldg(R.f + lane) : 0u;
    for (int k = lane; k < R.nf; k += G) {
      const uint32_t e = en;
      en = k + G < R.nf ? __ldg(R.f + k + G) : 0u;  // row entries stream from HBM: prefetch
      const uint32_t f = nb_index<M>(e);
      // fluid records are only read here (the kernel writes wall/rigid records): read-only path
      const double4 g0 = ldg4(&D.G0.p[f]);
      const double3 d = pair_delta<M>(P, pw, ld3(g0), e);  // = the oracle's minimum-image r_w - r_f
      const double r2 = d.x * d.x + d.y * d.y + d.z * d.z;
      double W, ri;  // sigma cancels in the ratios
      if (kPin) {
        if (r2 > P.rc2_hi) continue;
        const double q = pinned_q(d, P.rc2, P.inv_h, ri);
        if (q >= 3.0) continue;
        W = shape_q(q);
      } else {
        st = max(st, r2 < P.rc2_lo ? 2 : (r2 <= P.rc2_hi ? 1 : 0));
        if (r2 > P.rc2) continue;
        W = shape_q(pair_qr(d, r2, P.inv_h, ri));
      }
      const double4 g1 = ldg4(&D.G1.p[f]);
      const double pf = __ldg(reinterpret_cast<const double*>(&D.G2.p[f]) + 3);
      const uint32_t mf = kMultiEos || !P.single_g ? mat_of(__ldg(&D.kmd.p[f])) : (uint32_t)P.default_fluid_mat;
      const DevMat& Mf = P.mat[mf];
      const double ga = (Mf.g[0] - aw.x) * d.x + (Mf.g[1] - aw.y) * d.y + (Mf.g[2] - aw.z) * d.z;
      sw += W;
      sp += W * (pf + g1.w * ga);
      su.x += W * g1.x;
      su.y += W * g1.y;
      su.z += W * g1.z;
      if (kMultiEos) smat[mf] += W;
    }
  }
  sw = gsum<G>(sw);
  sp = gsum<G>(sp);
  su.x = gsum<G>(su.x);
  su.y = gsum<G>(su.y);
  su.z = gsum<G>(su.z);
  if (kMultiEos) {
#pragma unroll
    for (int m = 0; m < kMaxMat; ++m) smat[m] = gsum<G>(smat[m]);
  }
  if (!kPin) {  // all fluid pairs in the band below r_c: the weights' last bits decide -> pinned redo
    const bool band = gmax<G>(st) == 1;
    if (band && active && lane == 0) pin_list[atomicAdd(any, 1u)] = w;
    if (band) return;
  }
  if (!active || lane != 0) return;
  int m = P.default_fluid_mat;
  if (kMultiEos && sw > 0.0) {
    double best = -1.0;
    for (int q = 0; q < P.n_mat; ++q)
      if (smat[q] > best) {
        best = smat[q];
        m = q;
      }
  }
  const DevMat& Mt = P.mat[m];
  double p_w = 0.0;
  double3 ut = uw;
  if (sw > 0.0) {
    const double inv = 1.0 / sw;
    p_w = sp * inv;
    ut = make_double3(2.0 * uw.x - su.x * inv, 2.0 * uw.y - su.y * inv, 2.0 * uw.z - su.z * inv);
  }
  const double rho_w = fmax(Mt.rho0, Mt.rho0 + p_w * Mt.inv_c2);
  const double V_w = Mt.rho0 * P.dx3 / rho_w;
  reinterpret_cast<double*>(&D.G0.p[w])[3] = V_w * V_w;
  D.G1.p[w] = make_double4(ut.x, ut.y, ut.z, rho_w);
  D.G2.p[w] = make_double4(0.0, 0.0, 0.0, p_w);
}

template <int G, int M, bool kMultiEos, bool kPin>
// (the fast variant fits 56 registers without spills: 9 blocks of 128 per SM)
__global__ void __launch_bounds__(kBlock, kPin ? 1 : 9) k_extrapolate(const __grid_constant__ DevParams P, Particles D, NbrList L,
                                                         const sphg_body* __restrict__ B,
                                                         const uint32_t* __restrict__ list, size_t nlist,
                                                         uint32_t* __restrict__ pin_list, uint32_t* __restrict__ any) {
  SPHG_SKIP_IF_FLAGGED(P);
  // kPin: the flagged particles, compacted by the fast pass into pin_list[0 .. *any)
  if (kPin) {
    nlist = *any;
    list = pin_list;
    if ((size_t)blockIdx.x * (kBlock / G) >= nlist) return;  // the common case: nothing flagged
  }
  extrapolate_group<G, M, kMultiEos, kPin>(P, D, L, B, list, nlist, pin_list, any,
                                           (size_t)blockIdx.x * kBlock + threadIdx.x);
}

// the fast pass on an SM-local persistent grid (see k_density_sm)
template <int M, bool kMultiEos>
__global__ void __launch_bounds__(kBlock, 9) k_extrapolate_sm(const __grid_constant__ DevParams P, Particles D,
                                                               NbrList L, const sphg_body* __restrict__ B,
                                                               const uint32_t* __restrict__ list, size_t nlist,
                                                               uint32_t* __restrict__ pin_list,
                                                               uint32_t* __restrict__ any, uint32_t* __restrict__ next,
                                                               int nq) {
  SPHG_SKIP_IF_FLAGGED(P);
  int q = (int)(sm_id() % (unsigned)nq);
  size_t tile;
  while (next_tile(next, nq, (nlist + 7) / 8, q, tile))
    extrapolate_group<4, M, kMultiEos, false>(P, D, L, B, list, nlist, pin_list, any, tile * 32 + (threadIdx.x & 31));
}

// ---------------------------------------------------------------- forces
// a_ij = (V_i^2 + V_j^2)/m_i [ -p~ gradW + eta~ (u_i-u_j) (dW/dr)/r + 1/2 (A_i + A_j) gradW ],
// A = rho u (u~ - u)^T, gradW = dW/dr e_ij;  a_bg,i = -(p_b/m_i) sum (V_i^2+V_j^2) gradW.
struct PairSide {
  double3 u, du;
  double rho, p, V2, eta, hrho;  // hrho = rho/2 (TVF)
};

// kJFluid = false: j is a wall/rigid particle: A_j = 0 and eta_j = eta_i [P5][P7]
// q, rinv: the pair's q = r/h and 1/r (fast root, or pinned_q for flagged particles)
template <bool kTvf, bool kSingleEta, bool kJFluid>
__device__ __forceinline__ void pair_term(const PairSide& I, const PairSide& J, double3 d, double q, double rinv,
                                          const DevParams& P, double3& acc, double3& bg) {
  const double dW = q >= 3.0 ? 0.0 : P.sig_h * shape_deriv_q(q);
  const double fac = dW * rinv;  // gradW = fac * d
  const double3 gW = make_double3(fac * d.x, fac * d.y, fac * d.z);
  const double V2 = I.V2 + J.V2;
  const double pt = fma(J.rho, I.p, I.rho * J.p) * rcp_fast(I.rho + J.rho);
  double et;
  if (kSingleEta || !kJFluid) {
    et = I.eta;  // 2 eta eta / (eta + eta)
  } else {
    const double es = I.eta + J.eta;
    et = es > 0.0 ? 2.0 * I.eta * J.eta * rcp_fast(es) : 0.0;
  }
  const double vf = et * fac;
  double3 t = make_double3(fma(vf, I.u.x - J.u.x, -pt * gW.x), fma(vf, I.u.y - J.u.y, -pt * gW.y),
                           fma(vf, I.u.z - J.u.z, -pt * gW.z));
  if (kTvf) {
    const double ai = I.hrho * (I.du.x * gW.x + I.du.y * gW.y + I.du.z * gW.z);
    t.x += ai * I.u.x;
    t.y += ai * I.u.y;
    t.z += ai * I.u.z;
    if (kJFluid) {
      const double aj = J.hrho * (J.du.x * gW.x + J.du.y * gW.y + J.du.z * gW.z);
      t.x += aj * J.u.x;
      t.y += aj * J.u.y;
      t.z += aj * J.u.z;
    }
  }
  acc.x = fma(V2, t.x, acc.x);
  acc.y = fma(V2, t.y, acc.y);
  acc.z = fma(V2, t.z, acc.z);
  bg.x = fma(V2, gW.x, bg.x);
  bg.y = fma(V2, gW.y, bg.y);
  bg.z = fma(V2, gW.z, bg.z);
}

// Fluid-side pair, with the pair weight w = (V_i^2 + V_j^2) (dW/dr) / r factored out of every term:
//   acc += -p~ w d - eta~ w u_j + w (rho_j/2) (du_j . d) u_j,   svf += eta~ w,   bg += w d.
// The i-side TVF term (1/2) A_i gradW summed over j equals (rho_i/2) u_i (du_i . bg), and the i-side of
// the viscous sum is u_i svf: both are applied once per particle (forces_fluid_group), not per pair.
// conduction folded into the fluid forces pass (one row walk; see launch_heat_begin): T_i, kappa_i
// of the fluid particle and the running sum of k_heat
// (kHeat with diff = 1: the same fold for the concentration sums of k_diffusion, D for kappa)
struct HeatSide {
  double T, kappa, s;
  int diff;
};

template <int M, bool kTvf, bool kSingleEta, bool kHeat = false>
__device__ __forceinline__ void fluid_pair(const DevParams& P, const Particles& D, const PairSide& I, double3 pi,
                                           uint32_t e, double4 h0, double4 h1, double4 h2, double3& acc,
                                           double3& bg, double& svf, bool& coincident, HeatSide* heat = nullptr,
                                           double2 hj = double2{0.0, 0.0}) {
  const double3 d = pair_delta<M>(P, pi, ld3(h0), e);
  const double r2 = d.x * d.x + d.y * d.y + d.z * d.z;
  if (r2 > P.rc2) return;
  if (r2 == 0.0) {
    coincident = true;
    return;
  }
  double rinv;
  const double dW = P.sig_h * shape_deriv_q(pair_qr(d, r2, P.inv_h, rinv));
  if (kHeat && hj.y != 0.0) {  // same term, same order as k_heat / k_diffusion (V_heat / V_diff = 0: skip)
    double kt;
    bool conduct = true;
    if (!heat->diff && P.single_kappa) {
      kt = 2.0 * heat->kappa;
    } else {
      const DevMat& Mb = P.mat[mat_of(__ldg(&D.kmd.p[nb_index<M>(e)]))];
      const double kb = heat->diff ? Mb.D : Mb.kappa;
      const double ks = heat->kappa + kb;
      conduct = ks != 0.0;
      kt = conduct ? 4.0 * heat->kappa * kb / ks : 0.0;
    }
    if (conduct) heat->s += hj.y * kt * ((heat->T - hj.x) * rinv) * dW;
  }
  const double w = (I.V2 + h0.w) * (dW * rinv);
  bg.x = fma(w, d.x, bg.x);
  bg.y = fma(w, d.y, bg.y);
  bg.z = fma(w, d.z, bg.z);
  const double rho_j = h1.w, p_j = h2.w;
  const double pw = -fma(rho_j, I.p, I.rho * p_j) * rcp_fast(I.rho + rho_j) * w;
  double et;
  if (kSingleEta) {
    et = P.eta_single;  // 2 eta eta / (eta + eta), eta of every fluid material
  } else {
    const uint32_t kj = __ldg(&D.kmd.p[nb_index<M>(e)]);
    const double eta_j = kind_of(kj) == SPHG_FLUID ? P.mat[mat_of(kj)].eta : I.eta;  // eta_w := eta_i [P7]
    const double es = I.eta + eta_j;
    et = es > 0.0 ? 2.0 * I.eta * eta_j * rcp_fast(es) : 0.0;
  }
  // viscous sum split: sum_j eta~ w (u_i - u_j) = u_i sum_j eta~ w - sum_j eta~ w u_j.  u_i leaves the row
  // walk's registers (applied once per particle from svf in forces_fluid_group), which is what lets the
  // SM-local kernel hold a seventh block per SM; the round-off it adds, ~1e-16 |u| sum |eta~ w|, sits below
  // that of the pressure terms of the same sum
  const double vf = et * w;
  svf += vf;
  acc.x = fma(pw, d.x, fma(-vf, h1.x, acc.x));
  acc.y = fma(pw, d.y, fma(-vf, h1.y, acc.y));
  acc.z = fma(pw, d.z, fma(-vf, h1.z, acc.z));
  if (kTvf) {  // wall / rigid records carry du = 0 (A_j = 0)
    const double cj = w * (0.5 * rho_j) * (h2.x * d.x + h2.y * d.y + h2.z * d.z);
    acc.x = fma(cj, h1.x, acc.x);
    acc.y = fma(cj, h1.y, acc.y);
    acc.z = fma(cj, h1.z, acc.z);
  }
}

// the fluid particle's row (contiguous, fluid then non-fluid), row entries prefetched one
// iteration ahead (rows stream from HBM), all three 32-byte neighbour records requested together
template <int G, int M, bool kTvf, bool kSingleEta, bool kHeat = false>
__device__ __forceinline__ void fluid_row(const DevParams& P, const Particles& D, const PairSide& I, double3 pi,
                                          const uint32_t* base, int n, int lane, double3& acc, double3& bg,
                                          double& svf, bool& coincident, HeatSide* heat = nullptr,
                                          const double2* __restrict__ Sin = nullptr) {
  int k = lane;
  uint32_t e = k < n ? ldrow(base + k) : 0u;
  for (; k < n; k += G) {
    const uint32_t en = k + G < n ? ldrow(base + k + G) : 0u;
    const uint32_t j = nb_index<M>(e);
    const double4 h0 = ldg4(&D.G0.p[j]), h1 = ldg4(&D.G1.p[j]), h2 = ldg4(&D.G2.p[j]);
    double2 hj = double2{0.0, 0.0};
    if (kHeat) hj = __ldg(&Sin[j]);
    fluid_pair<M, kTvf, kSingleEta, kHeat>(P, D, I, pi, e, h0, h1, h2, acc, bg, svf, coincident, heat, hj);
    e = en;
  }
}

// one particle of the fluid list per G-lane group: g = its slot in the list, lane = the lane within the group
// (called by whole warps: the group sums are warp shuffles)
template <int G, int M, bool kTvf, bool kSingleEta, bool kHeat>
__device__ __forceinline__ void forces_fluid_group(const DevParams& P, const Particles& D, const NbrList& L,
                                                   const uint32_t* __restrict__ list, size_t nlist,
                                                   DevFlags* __restrict__ fl, double2* __restrict__ Hout,
                                                   const double2* __restrict__ Sin, int sdiff, size_t g, int lane) {
  const bool active = g < nlist;
  const uint32_t i = active ? list[g] : 0u;
  double3 acc = make_double3(0, 0, 0), bg = make_double3(0, 0, 0);
  double svf = 0.0;  // sum_j eta~ w of the viscous term (fluid_pair)
  bool coincident = false;
  uint32_t kmd = 0;
  HeatSide heat{0.0, 0.0, 0.0, sdiff};
  double2 hi = double2{0.0, 0.0};
  if (active) {
    kmd = D.kmd.p[i];
    if (kHeat) {  // Sin: (T, V_heat), or (C, V_diff) with sdiff
      hi = Sin[i];
      heat.T = hi.x;
      heat.kappa = sdiff ? P.mat[mat_of(kmd)].D : P.mat[mat_of(kmd)].kappa;
    }
    const double4 g0 = ldg4(&D.G0.p[i]), g1 = ldg4(&D.G1.p[i]), g2 = ldg4(&D.G2.p[i]);
    PairSide I;
    I.u = ld3(g1);
    I.du = ld3(g2);
    I.rho = g1.w;
    I.hrho = 0.5 * g1.w;
    I.p = g2.w;
    I.V2 = g0.w;
    I.eta = P.mat[mat_of(kmd)].eta;
    const double3 pi = ld3(g0);
    const Row R = row_of(L, i);
    // one pass over the whole contiguous row: wall/rigid records carry du = 0 (A_w = 0) and, with
    // several viscosities, fluid_pair looks up eta_j by kind (eta_w := eta_i)
    fluid_row<G, M, kTvf, kSingleEta, kHeat>(P, D, I, pi, R.f, R.n, lane, acc, bg, svf, coincident, &heat, Sin);
  }
  if (kHeat) heat.s = gsum<G>(heat.s);
  svf = gsum<G>(svf);
  acc.x = gsum<G>(acc.x);
  acc.y = gsum<G>(acc.y);
  acc.z = gsum<G>(acc.z);
  bg.x = gsum<G>(bg.x);
  bg.y = gsum<G>(bg.y);
  bg.z = gsum<G>(bg.z);
  if (!active) return;
  if (coincident) {
    atomicOr(&fl->err, kErrCoincident);
    atomicMin(&fl->err_gid, D.gid.p[i]);
  }
  if (lane != 0) return;
  {  // i-side of the viscous sum: u_i sum_j eta~ w
    const double4 gu = ldg4(&D.G1.p[i]);
    acc.x = fma(svf, gu.x, acc.x);
    acc.y = fma(svf, gu.y, acc.y);
    acc.z = fma(svf, gu.z, acc.z);
  }
  if (kTvf) {  // i-side TVF term: (rho_i/2) u_i (du_i . sum_j (V_i^2+V_j^2) gradW)
    const double4 g1 = ldg4(&D.G1.p[i]), g2 = ldg4(&D.G2.p[i]);
    const double ai = 0.5 * g1.w * (g2.x * bg.x + g2.y * bg.y + g2.z * bg.z);
    acc.x = fma(ai, g1.x, acc.x);
    acc.y = fma(ai, g1.y, acc.y);
    acc.z = fma(ai, g1.z, acc.z);
  }
  const DevMat& Mt = P.mat[mat_of(kmd)];
  const double im = 1.0 / D.V4.p[i].w;
  D.A4.p[i] = make_double4(acc.x * im + Mt.g[0], acc.y * im + Mt.g[1], acc.z * im + Mt.g[2], 0.0);
  const double f = kTvf ? -Mt.pb * im : 0.0;
  D.B4.p[i] = make_double4(f * bg.x, f * bg.y, f * bg.z, 0.0);
  if (kHeat && sdiff) {  // the k_diffusion epilogue for a fluid particle (rho_a = rho_i)
    const double rate = heat.s / D.G1.p[i].w;
    const uint32_t gc = dirc_of(kmd);
    const bool fixed = gc != SPHG_NO_DIRICHLET && (int)gc < P.n_schedC && P.schedC[gc].n > 0;
    Hout[i] = make_double2(fixed ? hi.x : hi.x + P.dt * rate, hi.y);
    D.dCdt.p[i] = rate;
  } else if (kHeat) {  // the k_heat epilogue for a fluid particle (rho_a = rho_i)
    double rate = 0.0;
    if (Mt.cp > 0.0) {
      rate = heat.s / (D.G1.p[i].w * Mt.cp);
      if (P.heat_source) rate += P.hsrc[i];  // [P21]
    }
    Hout[i] = make_double2(hi.x + P.dt * rate, hi.y);
    D.dTdt.p[i] = rate;
  }
}


template <int G, int M, bool kTvf, bool kSingleEta, bool kHeat = false>
__global__ void __launch_bounds__(kBlock) k_forces_fluid(const __grid_constant__ DevParams P, Particles D, NbrList L,
                                                          const uint32_t* __restrict__ list, size_t nlist,
                                                          DevFlags* __restrict__ fl,
                                                          double2* __restrict__ Hout = nullptr,
                                                          const double2* __restrict__ Sin = nullptr, int sdiff = 0) {
  SPHG_SKIP_IF_FLAGGED(P);
  const size_t t = (size_t)blockIdx.x * kBlock + threadIdx.x;
  forces_fluid_group<G, M, kTvf, kSingleEta, kHeat>(P, D, L, list, nlist, fl, Hout, Sin, sdiff, t / G, (int)(t % G));
}

// (without the fused conduction: 7 blocks of 128 per SM at 72 registers, 12 bytes spilled outside the row walk)
template <int G, int M, bool kTvf, bool kSingleEta, bool kHeat>
__global__ void __launch_bounds__(kBlock, kHeat ? 4 : 7) k_forces_fluid_sm(const __grid_constant__ DevParams P, Particles D,
                                                             NbrList L, const uint32_t* __restrict__ list,
                                                             size_t nlist, DevFlags* __restrict__ fl,
                                                             uint32_t* __restrict__ next, int nq,
                                                             double2* __restrict__ Hout,
                                                             const double2* __restrict__ Sin, int sdiff) {
  SPHG_SKIP_IF_FLAGGED(P);
  const int lw = threadIdx.x & 31;
  int q = (int)(sm_id() % (unsigned)nq);
  size_t tile;
  constexpr int T = 32 / G;  // particles per warp tile
  while (next_tile(next, nq, (nlist + T - 1) / T, q, tile))
    forces_fluid_group<G, M, kTvf, kSingleEta, kHeat>(P, D, L, list, nlist, fl, Hout, Sin, sdiff,
                                                      tile * T + lw / G, lw % G);
}

// f_r = sum_i -m_i a_ir over the fluid part of the row (a_ir from the fluid's view)
//     + contact over the rigid/boundary part
// kPin = false: the fast root; a particle whose fluid pairs all sit within 2e-4 below r_c^2 is appended
// to pin_list and not written.  kPin = true: only those particles, coupling with pinned_q.
template <int G, int M, bool kTvf, bool kSingleEta, bool kPin>
__device__ __forceinline__ void forces_rigid_group(const DevParams& P, const Particles& D, const NbrList& L,
                                                   const uint32_t* __restrict__ list, size_t nlist,
                                                   const uint32_t* __restrict__ ncon, DevFlags* __restrict__ fl,
                                                   uint32_t* __restrict__ pin_list, uint32_t* __restrict__ any,
                                                   size_t t) {
  const size_t g = t / G;
  const int lane = (int)(t % G);
  const uint32_t r = g < nlist ? list[g] : 0u;
  const bool active = g < nlist;
  int st = 0;  // 2: a fluid pair clearly inside r_c, 1: only pairs in the 2e-4 band below r_c^2, 0: none
  double3 f = make_double3(0, 0, 0);
  bool coincident = false;
  if (active) {
    const double4 g0 = ldg4(&D.G0.p[r]), g1 = ldg4(&D.G1.p[r]), g2 = ldg4(&D.G2.p[r]);
    const double3 vr = ldpos(&D.V4.p[r]);
    const uint32_t body = D.group.p[r];
    PairSide R;
    R.u = ld3(g1);
    R.du = make_double3(0, 0, 0);
    R.rho = g1.w;
    R.hrho = 0.5 * g1.w;
    R.p = g2.w;
    R.V2 = g0.w;
    const double3 pr = ld3(g0);
    const Row Rw = row_of(L, r);
    // coupling: fluid part
    uint32_t en = lane < Rw.nf ? __ldg(Rw.f + lane) : 0u;
    for (int k = lane; k < Rw.nf; k += G) {
      const uint32_t e = en;
      en = k + G < Rw.nf ? __ldg(Rw.f + k + G) : 0u;
      const uint32_t j = nb_index<M>(e);
      const double4 h0 = ldg4(&D.G0.p[j]), h1 = ldg4(&D.G1.p[j]), h2 = ldg4(&D.G2.p[j]);
      // from the fluid's view: d = r_j - r_r (the entry's image is defined for r - j: negate)
      const double3 dd = pair_delta<M>(P, pr, ld3(h0), e);
      const double3 d = make_double3(-dd.x, -dd.y, -dd.z);
      const double r2 = d.x * d.x + d.y * d.y + d.z * d.z;
      double q, rinv;
      if (kPin) {
        if (r2 > P.rc2_hi) continue;
        q = pinned_q(d, P.rc2, P.inv_h, rinv);
        if (q >= 3.0) continue;
      } else {
        st = max(st, r2 < P.rc2_lo ? 2 : (r2 <= P.rc2_hi ? 1 : 0));
        if (r2 > P.rc2) continue;
        if (r2 == 0.0) {
          coincident = true;
          continue;
        }
        q = pair_qr(d, r2, P.inv_h, rinv);
      }
      PairSide J;
      J.u = ld3(h1);
      J.du = ld3(h2);
      J.rho = h1.w;
      J.hrho = 0.5 * h1.w;
      J.p = h2.w;
      J.V2 = h0.w;
      J.eta = kSingleEta ? P.mat[P.default_fluid_mat].eta : P.mat[mat_of(__ldg(&D.kmd.p[j]))].eta;
      R.eta = J.eta;  // eta_w := eta_i
      double3 a = make_double3(0, 0, 0), bgd = make_double3(0, 0, 0);
      pair_term<kTvf, true, false>(J, R, d, q, rinv, P, a, bgd);  // j plays i; the rigid side has A = 0
      // f_ri = -m_i a_ir = -(V2 term): pair_term accumulates V2*term (a_ir = V2/m_i * term)
      f.x -= a.x;
      f.y -= a.y;
      f.z -= a.z;
    }
    // contact: rigid particles of other bodies and walls, ordered first in the
    // non-fluid part by k_contact_order (ncon of them)
    const int ncand = (int)ncon[r];
    for (int k = lane; k < ncand; k += G) {
      const uint32_t e = __ldg(Rw.b + k);
      const uint32_t j = nb_index<M>(e);
      const uint32_t kindj = kind_of(D.kmd.p[j]);
      if (kindj != SPHG_BOUNDARY && D.group.p[j] == body) continue;
      const double3 d = pair_delta<M>(P, pr, ldpos(&D.G0.p[j]), e);  // r_r - r_j
      if (d.x * d.x + d.y * d.y + d.z * d.z > P.dx2_hi) continue;  // clearly apart (most candidates)
      // the contact decision r < dx is discrete: the oracle's no-FMA r^2 and correctly rounded root
      const double rr = __dsqrt_rn(r2_exact(d));
      if (!(rr < P.dx)) continue;
      if (rr == 0.0) {
        coincident = true;
        continue;
      }
      const double ri = 1.0 / rr;
      const double3 e3 = make_double3(d.x * ri, d.y * ri, d.z * ri);
      const double3 vj = ldpos(&D.V4.p[j]);
      const double s = P.kc * (rr - P.dx) + P.dc * (e3.x * (vr.x - vj.x) + e3.y * (vr.y - vj.y) + e3.z * (vr.z - vj.z));
      const double fm = -fmin(0.0, s);
      f.x += fm * e3.x;
      f.y += fm * e3.y;
      f.z += fm * e3.z;
    }
  }
  f.x = gsum<G>(f.x);
  f.y = gsum<G>(f.y);
  f.z = gsum<G>(f.z);
  if (!kPin) {  // every fluid pair in the band below r_c: their last bits decide -> pinned redo
    const bool band = gmax<G>(st) == 1;
    if (band && active && lane == 0) pin_list[atomicAdd(any, 1u)] = r;
    if (band) return;
  }
  if (!active) return;
  if (coincident) {
    atomicOr(&fl->err, kErrCoincident);
    atomicMin(&fl->err_gid, D.gid.p[r]);
  }
  if (lane == 0) D.F4.p[r] = make_double4(f.x, f.y, f.z, 0.0);
}

template <int G, int M, bool kTvf, bool kSingleEta, bool kPin>
__global__ void __launch_bounds__(kBlock) k_forces_rigid(const __grid_constant__ DevParams P, Particles D, NbrList L,
                                                          const uint32_t* __restrict__ list, size_t nlist,
                                                          const uint32_t* __restrict__ ncon,
                                                          DevFlags* __restrict__ fl, uint32_t* __restrict__ pin_list,
                                                          uint32_t* __restrict__ any) {
  SPHG_SKIP_IF_FLAGGED(P);
  // kPin: the flagged particles, compacted by the fast pass into pin_list[0 .. *any)
  if (kPin) {
    nlist = *any;
    list = pin_list;
    if ((size_t)blockIdx.x * (kBlock / G) >= nlist) return;  // the common case: nothing flagged
  }
  forces_rigid_group<G, M, kTvf, kSingleEta, kPin>(P, D, L, list, nlist, ncon, fl, pin_list, any,
                                                   (size_t)blockIdx.x * kBlock + threadIdx.x);
}

// the fast pass on an SM-local persistent grid (see k_density_sm); the rigid list is body-major
template <int M, bool kTvf, bool kSingleEta>
__global__ void __launch_bounds__(kBlock) k_forces_rigid_sm(const __grid_constant__ DevParams P, Particles D,
                                                             NbrList L, const uint32_t* __restrict__ list,
                                                             size_t nlist, const uint32_t* __restrict__ ncon,
                                                             DevFlags* __restrict__ fl,
                                                             uint32_t* __restrict__ pin_list,
                                                             uint32_t* __restrict__ any, uint32_t* __restrict__ next,
                                                             int nq) {
  SPHG_SKIP_IF_FLAGGED(P);
  int q = (int)(sm_id() % (unsigned)nq);
  size_t tile;
  while (next_tile(next, nq, (nlist + 7) / 8, q, tile))
    forces_rigid_group<4, M, kTvf, kSingleEta, false>(P, D, L, list, nlist, ncon, fl, pin_list, any,
                                                      tile * 32 + (threadIdx.x & 31));
}

// Verlet candidates and pairs within r_c (exact test), all particles; split by kind of i
template <int G, int M>
__global__ void __launch_bounds__(kBlock) k_count_pairs(const __grid_constant__ DevParams P, Particles D, NbrList L,
                                                         size_t n, unsigned long long* __restrict__ out) {
  const size_t t = (size_t)blockIdx.x * kBlock + threadIdx.x;
  const size_t i = t / G;
  const int lane = (int)(t % G);
  uint32_t c = 0, in = 0;
  bool fluid = false;
  if (i < n) {
    fluid = kind_of(D.kmd.p[i]) == SPHG_FLUID;
    const double3 pi = ldpos(&D.G0.p[i]);
    const Row R = row_of(L, (uint32_t)i);
    for (int k = lane; k < R.n; k += G) {
      const uint32_t e = R.at(k);
      const double3 pj = ldpos(&D.G0.p[nb_index<M>(e)]);
      const double3 d = M == kImgNone ? make_double3(pi.x - pj.x, pi.y - pj.y, pi.z - pj.z)
                                      : mimg3(P, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z);
      c += 1u;
      if (r2_exact(d) <= P.rc2) in += 1u;
    }
  }
  // per-block totals, one atomic per counter per block (same-address atomics serialise in L2)
  unsigned long long v[4] = {0, 0, 0, 0};
  if (i < n) {
    v[0] = (unsigned long long)c;
    v[1] = (unsigned long long)in;
    v[fluid ? 2 : 3] = (unsigned long long)in;
  }
  __shared__ unsigned long long sv[kBlock / 32][4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    unsigned long long x = v[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0) sv[threadIdx.x >> 5][q] = x;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    unsigned long long x = 0;
    for (int w = 0; w < kBlock / 32; ++w) x += sv[w][threadIdx.x];
    if (x) atomicAdd(out + threadIdx.x, x);
  }
}

// particles the heat kernels do not update (walls, ghosts) keep their T in the new buffer
__global__ void k_copy_boundary_T(const __grid_constant__ DevParams P, Particles D, size_t n, double2* __restrict__ Hout) {
  SPHG_SKIP_IF_FLAGGED(P);
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t kmd = D.kmd.p[i];
  if (kind_of(kmd) == SPHG_BOUNDARY || is_ghost(kmd)) Hout[i] = D.H2.p[i];
}

__device__ __forceinline__ double sched_value(const DevSchedule& s, double t) {  // Schedule::value_at
  for (int k = 0; k < s.n; ++k)
    if (t <= s.t_end[k]) return s.value[k];
  return s.value[s.n - 1];
}

// t_dev (graph replay): t^{n+1} from device memory, refreshed by a memcpy node every replay
__global__ void k_dirichlet(const __grid_constant__ DevParams P, Particles D, size_t n, double t_new,
                            const double* __restrict__ t_dev) {
  SPHG_SKIP_IF_FLAGGED(P);
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (t_dev) t_new = *t_dev;
  const uint32_t kmd = D.kmd.p[i];
  if (kind_of(kmd) != SPHG_BOUNDARY) return;
  const uint32_t gr = dir_of(kmd);
  if (gr == SPHG_NO_DIRICHLET || (int)gr >= P.n_sched || P.sched[gr].n <= 0) return;
  reinterpret_cast<double*>(&D.H2.p[i])[0] = sched_value(P.sched[gr], t_new);
}

__global__ void k_dirichlet_c(const __grid_constant__ DevParams P, Particles D, size_t n, double t_new,
                              const double* __restrict__ t_dev) {
  SPHG_SKIP_IF_FLAGGED(P);
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (t_dev) t_new = *t_dev;
  const uint32_t gr = dirc_of(D.kmd.p[i]);
  if (gr == SPHG_NO_DIRICHLET || (int)gr >= P.n_schedC || P.schedC[gr].n <= 0) return;
  reinterpret_cast<double*>(&D.C2.p[i])[0] = sched_value(P.schedC[gr], t_new);
}

__global__ void k_copy_boundary_C(const __grid_constant__ DevParams P, Particles D, size_t n, double2* __restrict__ Cout) {
  SPHG_SKIP_IF_FLAGGED(P);
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t kmd = D.kmd.p[i];
  if (kind_of(kmd) == SPHG_BOUNDARY || is_ghost(kmd)) Cout[i] = D.C2.p[i];
}

template <int G>
int blocks_for(size_t groups) {
  return grid_for(groups * G, kBlock);
}

}  // namespace

// ============================================================= launchers
// Lanes per particle (G).  4 is the measured optimum for lists that fill the GPU (DESIGN.md §4:
// 2 / 8 / 16 lose at 64M).  A list below a quarter of a GPU's worth of 4-lane groups (the rigid and
// wall subsets of small stores: ~1e3-1e4 particles) gets a warp per particle instead: there each
// kernel is one latency chain per row walk, and 4 lanes per particle leave most SMs idle (C1: rigid
// forces 21.6 -> 7.5 us, extrapolation 31 -> 10 us; its 31k-particle fluid list stays faster at 4).  The choice depends only on the list
// length, so fused and unfused variants of a sum take the same summation order.
// SPHG_GROUP_DENSITY / SPHG_GROUP_FORCES (2, 4, 8) fix the width for tuning sweeps.
inline int lanes_for(const Ctx& c, size_t nlist) { return 2 * nlist < c.fill_groups ? 32 : 4; }
// SM-local persistent grids pay for long lists (measured against flat grids: C3 2.4M -2.5 %, paper46 3.8M
// -8 %, C5 8M -5 %, C4 16M -3 %, C5 64M -6 % per step; C1 32k and C2 343k lose to the persistent grid's
// fixed costs); shorter lists keep flat grids
inline bool sm_local_for(const Ctx& c, int bit, size_t nlist) { return (c.sm_local & bit) && nlist >= c.sm_local_min; }
#define SPHG_L_DISPATCH(C, NLIST, CALL)                              \
  do {                                                              \
    if (lanes_for(C, NLIST) == 32) { constexpr int G = 32; CALL; }  \
    else { constexpr int G = 4; CALL; }                             \
  } while (0)
#define SPHG_G_DISPATCH(C, GV, NLIST, CALL)                      \
  do {                                                          \
    if ((GV) == 8) { constexpr int G = 8; CALL; }                \
    else if ((GV) == 2) { constexpr int G = 2; CALL; }           \
    else if ((GV) == 4) { constexpr int G = 4; CALL; }           \
    else SPHG_L_DISPATCH(C, NLIST, CALL);                        \
  } while (0)

#define SPHG_IMG_DISPATCH(MODE, CALL)                             \
  do {                                                            \
    switch (MODE) {                                               \
      case kImgNone: { constexpr int M = kImgNone; CALL; break; } \
      case kImgCode: { constexpr int M = kImgCode; CALL; break; } \
      default: { constexpr int M = kImgMin; CALL; break; }        \
    }                                                             \
  } while (0)

// persistent grid of an SM-local kernel: every block resident at once (occupancy x SMs), counters zeroed
template <class K>
static int sm_local_grid(Ctx& c, K kernel, uint32_t* next, cudaStream_t st) {
  static int per_sm = 0;  // one instance per kernel instantiation
  if (per_sm == 0) {
    if (const char* e = std::getenv("SPHG_SMEM_CARVEOUT"))  // experiment: shared-memory share of the L1 array, %
      SPHG_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, std::atoi(e)));
    SPHG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, c.sm_threads, 0));
    per_sm = std::max(per_sm, 1);
    if (const char* e = std::getenv("SPHG_SM_BLOCKS"))  // experiment: fewer resident blocks per SM than fit
      per_sm = std::max(1, std::min(per_sm, std::atoi(e)));
  }
  SPHG_CUDA_CHECK(cudaMemsetAsync(next, 0, c.n_sms * sizeof(uint32_t), st));
  return per_sm * c.n_sms;
}

// slot: which counter array a persistent grid uses (0 density, 4 the interior density pass that overlaps the
// STATE halo on its own stream; 1-3 belong to the forces / extrapolation kernels)
static void launch_density_list(Ctx& c, const uint32_t* list, size_t m, cudaStream_t st, int slot = 0) {
  if (m == 0) return;
  const int gd = c.group_density ? c.group_density : lanes_for(c, m);
  if (sm_local_for(c, 2, m) && (gd == 4 || gd == 8)) {
    uint32_t* next = c.sm_next.p + (size_t)slot * c.n_sms;
#define SPHG_DENS_SM(GV)                                                                                            \
  SPHG_IMG_DISPATCH(c.P.img_mode,                                                                                   \
                    (k_density_sm<GV, M><<<sm_local_grid(c, k_density_sm<GV, M>, next, st), c.sm_threads, 0, st>>>(        \
                        c.P, c.cur, c.nl(), list, m, next, c.n_sms)))
    if (gd == 8) SPHG_DENS_SM(8);
    else SPHG_DENS_SM(4);
#undef SPHG_DENS_SM
    c.launches++;
    return;
  }
  SPHG_G_DISPATCH(c, c.group_density, m,
                  SPHG_IMG_DISPATCH(c.P.img_mode, (k_density<G, M><<<blocks_for<G>(m), kBlock, 0, st>>>(
                                                       c.P, c.cur, c.nl(), list, m))));
  c.launches++;
}

void launch_density(Ctx& c) { launch_density_list(c, c.fidx.p, c.nf, c.stream); }

// decomposed steps: the fluid list is ordered [interior | next to a ghost] (launch_ghost_split); the
// interior part reads only owned neighbours, so it runs before the STATE halo has landed
void launch_density_interior(Ctx& c, cudaStream_t st) { launch_density_list(c, c.fidx.p, c.nf_interior, st, 4); }
void launch_density_boundary(Ctx& c) {
  launch_density_list(c, c.fidx.p + c.nf_interior, c.nf - c.nf_interior, c.stream);
}

// Heat in two halves so one_step can fold the fluid part into the forces pass (c.fuse_heat):
// begin = Dirichlet values at t^{n+1} + rigid conduction (+ fluid conduction when not fused);
// end = walls / ghosts keep T, swap the double buffer.
void launch_heat_begin(Ctx& c) {
  if (c.n == 0) return;
  const double t_new = c.t + c.P.dt;
  k_dirichlet<<<grid_for(c.n, 256), 256, 0, c.stream>>>(c.P, c.cur, c.n, t_new, c.capturing ? c.dtime : nullptr);
  if (c.P.heat_source) {  // [P21] source rates before the conduction epilogues read them
    if (c.nf)
      SPHG_L_DISPATCH(c, c.nf, (k_heat_source<G><<<blocks_for<G>(c.nf), kBlock, 0, c.stream>>>(
                                   c.P, c.cur, c.nl(), c.fidx.p, c.nf, t_new, c.capturing ? c.dtime : nullptr)));
    if (c.nrigid)
      SPHG_L_DISPATCH(c, c.nrigid, (k_heat_source<G><<<blocks_for<G>(c.nrigid), kBlock, 0, c.stream>>>(
                                       c.P, c.cur, c.nl(), c.ridx.p, c.nrigid, t_new, c.capturing ? c.dtime : nullptr)));
    c.launches += 2;
  }
  // (the two launches run one after the other on the stream: they share a counter array)
  auto heat_list = [&](const uint32_t* list, size_t m) {
    if (sm_local_for(c, 16, m) && lanes_for(c, m) == 4) {
      uint32_t* next = c.sm_next.p + 5 * (size_t)c.n_sms;
      SPHG_IMG_DISPATCH(c.P.img_mode, (k_heat_sm<M><<<sm_local_grid(c, k_heat_sm<M>, next, c.stream), c.sm_threads, 0,
                                                    c.stream>>>(c.P, c.cur, c.nl(), list, m, c.H2new.p, c.dflags,
                                                                next, c.n_sms)));
    } else {
      SPHG_L_DISPATCH(c, m, SPHG_IMG_DISPATCH(c.P.img_mode, (k_heat<G, M><<<blocks_for<G>(m), kBlock, 0, c.stream>>>(
                                           c.P, c.cur, c.nl(), list, m, c.H2new.p, c.dflags))));
    }
  };
  if (c.nf && !c.fuse_heat) heat_list(c.fidx.p, c.nf);
  if (c.nrigid) heat_list(c.ridx.p, c.nrigid);
  c.launches += 3;
}

void launch_heat_end(Ctx& c) {
  if (c.n == 0) return;
  k_copy_boundary_T<<<grid_for(c.n, 256), 256, 0, c.stream>>>(c.P, c.cur, c.n, c.H2new.p);
  std::swap(c.cur.H2, c.H2new);
  c.launches++;
}

void launch_heat(Ctx& c) {
  const bool f = c.fuse_heat;
  c.fuse_heat = false;
  launch_heat_begin(c);
  launch_heat_end(c);
  c.fuse_heat = f;
}

// Diffusion in two halves like heat (c.fuse_diff folds the fluid part into the forces pass when the heat
// equation is off): begin = Dirichlet-C at t^{n+1} + rigid (+ fluid when not fused) sums; end = walls /
// ghosts keep C, swap the double buffer.
void launch_diffusion_begin(Ctx& c) {
  if (c.n == 0) return;
  const double t_new = c.t + c.P.dt;
  k_dirichlet_c<<<grid_for(c.n, 256), 256, 0, c.stream>>>(c.P, c.cur, c.n, t_new, c.capturing ? c.dtime : nullptr);
  if (c.nf && !c.fuse_diff)
    SPHG_L_DISPATCH(c, c.nf, SPHG_IMG_DISPATCH(c.P.img_mode, (k_diffusion<G, M><<<blocks_for<G>(c.nf), kBlock, 0, c.stream>>>(
                                         c.P, c.cur, c.nl(), c.fidx.p, c.nf, c.C2new.p, c.dflags))));
  if (c.nrigid)
    SPHG_L_DISPATCH(c, c.nrigid, SPHG_IMG_DISPATCH(c.P.img_mode, (k_diffusion<G, M><<<blocks_for<G>(c.nrigid), kBlock, 0, c.stream>>>(
                                         c.P, c.cur, c.nl(), c.ridx.p, c.nrigid, c.C2new.p, c.dflags))));
  c.launches += 3;
}

void launch_diffusion_end(Ctx& c) {
  if (c.n == 0) return;
  k_copy_boundary_C<<<grid_for(c.n, 256), 256, 0, c.stream>>>(c.P, c.cur, c.n, c.C2new.p);
  std::swap(c.cur.C2, c.C2new);
  c.launches++;
}

void launch_diffusion(Ctx& c) {
  const bool f = c.fuse_diff;
  c.fuse_diff = false;
  launch_diffusion_begin(c);
  launch_diffusion_end(c);
  c.fuse_diff = f;
}

// fast pass over the list, then the pinned redo of the particles it appended to pin_list (a launch
// whose blocks past the flagged count exit at once; see common.cuh pinned_q)
template <bool kMultiEos>
static void launch_extrapolate_t(Ctx& c) {
  SPHG_CUDA_CHECK(cudaMemsetAsync(c.pin_any, 0, sizeof(uint32_t), c.stream));
  if (sm_local_for(c, 4, c.nw) && lanes_for(c, c.nw) == 4) {
    constexpr int G = 4;
    uint32_t* next = c.sm_next.p + 2 * c.n_sms;
    SPHG_IMG_DISPATCH(c.P.img_mode, ({
      k_extrapolate_sm<M, kMultiEos><<<sm_local_grid(c, k_extrapolate_sm<M, kMultiEos>, next, c.stream), c.sm_threads, 0,
                                       c.stream>>>(c.P, c.cur, c.nl(), c.bodies.p, c.widx.p, c.nw, c.pin_list.p,
                                                   c.pin_any, next, c.n_sms);
      k_extrapolate<G, M, kMultiEos, true><<<blocks_for<G>(c.nw), kBlock, 0, c.stream>>>(
          c.P, c.cur, c.nl(), c.bodies.p, c.widx.p, c.nw, c.pin_list.p, c.pin_any);
    }));
    c.launches += 2;
    return;
  }
  SPHG_L_DISPATCH(c, c.nw, SPHG_IMG_DISPATCH(c.P.img_mode, ({
    k_extrapolate<G, M, kMultiEos, false><<<blocks_for<G>(c.nw), kBlock, 0, c.stream>>>(
        c.P, c.cur, c.nl(), c.bodies.p, c.widx.p, c.nw, c.pin_list.p, c.pin_any);
    k_extrapolate<G, M, kMultiEos, true><<<blocks_for<G>(c.nw), kBlock, 0, c.stream>>>(
        c.P, c.cur, c.nl(), c.bodies.p, c.widx.p, c.nw, c.pin_list.p, c.pin_any);
  })));
  c.launches += 2;
}

void launch_extrapolate(Ctx& c) {
  if (c.nw == 0) return;
  if (c.P.single_eos) launch_extrapolate_t<false>(c);
  else launch_extrapolate_t<true>(c);
}

template <bool kTvf, bool kSingleEta>
static void launch_forces_fluid_t(Ctx& c) {
  uint32_t* next = c.sm_next.p + c.n_sms;
  if (c.nf && (c.fuse_heat || c.fuse_diff)) {  // conduction / diffusion of the fluid particles in the same
                                               // row walk (k_heat's / k_diffusion's width and order)
    const bool dif = !c.fuse_heat;
    const double2* sin = dif ? c.cur.C2.p : c.cur.H2.p;
    double2* out = dif ? c.C2new.p : c.H2new.p;
    if (sm_local_for(c, 1, c.nf) && lanes_for(c, c.nf) == 4)
      SPHG_IMG_DISPATCH(c.P.img_mode,
                        (k_forces_fluid_sm<4, M, kTvf, kSingleEta, true>
                         <<<sm_local_grid(c, k_forces_fluid_sm<4, M, kTvf, kSingleEta, true>, next, c.stream), c.sm_threads, 0,
                            c.stream>>>(c.P, c.cur, c.nl(), c.fidx.p, c.nf, c.dflags, next, c.n_sms, out, sin,
                                        dif ? 1 : 0)));
    else
      SPHG_L_DISPATCH(c, c.nf, SPHG_IMG_DISPATCH(c.P.img_mode, (k_forces_fluid<G, M, kTvf, kSingleEta, true>
                                       <<<blocks_for<G>(c.nf), kBlock, 0, c.stream>>>(
                                           c.P, c.cur, c.nl(), c.fidx.p, c.nf, c.dflags, out, sin, dif ? 1 : 0))));
    c.launches++;
    return;
  }
  const int gf = c.group_forces ? c.group_forces : lanes_for(c, c.nf);
#define SPHG_FORCES_SM(GV)                                                                                          \
  SPHG_IMG_DISPATCH(c.P.img_mode,                                                                                   \
                    (k_forces_fluid_sm<GV, M, kTvf, kSingleEta, false>                                              \
                     <<<sm_local_grid(c, k_forces_fluid_sm<GV, M, kTvf, kSingleEta, false>, next, c.stream), c.sm_threads, \
                        0, c.stream>>>(c.P, c.cur, c.nl(), c.fidx.p, c.nf, c.dflags, next, c.n_sms, nullptr,         \
                                       nullptr, 0)))
  if (c.nf && sm_local_for(c, 1, c.nf) && gf == 4) SPHG_FORCES_SM(4);
  else if (c.nf && sm_local_for(c, 1, c.nf) && gf == 8) SPHG_FORCES_SM(8);
#undef SPHG_FORCES_SM
  else if (c.nf)
    SPHG_G_DISPATCH(c, c.group_forces, c.nf,
                    SPHG_IMG_DISPATCH(c.P.img_mode, (k_forces_fluid<G, M, kTvf, kSingleEta>
                                                     <<<blocks_for<G>(c.nf), kBlock, 0, c.stream>>>(
                                                         c.P, c.cur, c.nl(), c.fidx.p, c.nf, c.dflags))));
  c.launches++;
}

template <bool kTvf>
static void launch_forces_rigid_t(Ctx& c) {
  if (!c.nrigid) return;
  SPHG_CUDA_CHECK(cudaMemsetAsync(c.pin_any, 0, sizeof(uint32_t), c.stream));
#define SPHG_RIGID_PAIR(SE)                                                                                 \
  SPHG_L_DISPATCH(c, c.nrigid, SPHG_IMG_DISPATCH(c.P.img_mode, ({                                          \
    k_forces_rigid<G, M, kTvf, SE, false><<<blocks_for<G>(c.nrigid), kBlock, 0, c.stream>>>(                \
        c.P, c.cur, c.nl(), c.ridx.p, c.nrigid, c.ncon.p, c.dflags, c.pin_list.p, c.pin_any);                     \
    k_forces_rigid<G, M, kTvf, SE, true><<<blocks_for<G>(c.nrigid), kBlock, 0, c.stream>>>(                 \
        c.P, c.cur, c.nl(), c.ridx.p, c.nrigid, c.ncon.p, c.dflags, c.pin_list.p, c.pin_any);                     \
  })))
#define SPHG_RIGID_PAIR_SM(SE)                                                                              \
  SPHG_IMG_DISPATCH(c.P.img_mode, ({                                                                        \
    constexpr int G = 4;                                                                                    \
    uint32_t* next = c.sm_next.p + 3 * c.n_sms;                                                             \
    k_forces_rigid_sm<M, kTvf, SE><<<sm_local_grid(c, k_forces_rigid_sm<M, kTvf, SE>, next, c.stream), c.sm_threads, 0, \
                                     c.stream>>>(c.P, c.cur, c.nl(), c.ridx.p, c.nrigid, c.ncon.p, c.dflags,  \
                                                 c.pin_list.p, c.pin_any, next, c.n_sms);                    \
    k_forces_rigid<G, M, kTvf, SE, true><<<blocks_for<G>(c.nrigid), kBlock, 0, c.stream>>>(                 \
        c.P, c.cur, c.nl(), c.ridx.p, c.nrigid, c.ncon.p, c.dflags, c.pin_list.p, c.pin_any);               \
  }))
  const bool sm = sm_local_for(c, 8, c.nrigid) && lanes_for(c, c.nrigid) == 4;
  if (sm && c.P.single_eta) SPHG_RIGID_PAIR_SM(true);
  else if (sm) SPHG_RIGID_PAIR_SM(false);
  else if (c.P.single_eta) SPHG_RIGID_PAIR(true);
  else SPHG_RIGID_PAIR(false);
#undef SPHG_RIGID_PAIR
#undef SPHG_RIGID_PAIR_SM
  c.launches += 2;
}

void launch_forces_fluid(Ctx& c) {
  if (c.n == 0) return;
  const bool tvf = c.P.tvf != 0, single = c.P.single_eta != 0;
  if (tvf && single) launch_forces_fluid_t<true, true>(c);
  else if (tvf) launch_forces_fluid_t<true, false>(c);
  else if (single) launch_forces_fluid_t<false, true>(c);
  else launch_forces_fluid_t<false, false>(c);
}

#ifdef SPHG_DIAG_LOADS_ONLY
#include "diag_gather.cuh"  // gather-cost diagnostic kernels (tools/diag_loads.py builds only)
#endif

void launch_forces_diag(Ctx& c) {
#ifdef SPHG_DIAG_LOADS_ONLY
  launch_diag_gather(c);
#else
  (void)c;
#endif
}

void launch_forces_rigid(Ctx& c) {
  if (c.n == 0) return;
  if (c.P.tvf) launch_forces_rigid_t<true>(c);
  else launch_forces_rigid_t<false>(c);
}

void launch_forces(Ctx& c) {
  launch_forces_fluid(c);
  launch_forces_rigid(c);
}

void count_pairs(Ctx& c, int64_t out[4]) {
  if (!c.dcount) SPHG_CUDA_CHECK(cudaMalloc(&c.dcount, 4 * sizeof(unsigned long long)));
  SPHG_CUDA_CHECK(cudaMemsetAsync(c.dcount, 0, 4 * sizeof(unsigned long long), c.stream));
  constexpr int G = 4;
  SPHG_IMG_DISPATCH(c.P.img_mode, (k_count_pairs<G, M><<<blocks_for<G>(c.n), kBlock, 0, c.stream>>>(
                                       c.P, c.cur, c.nl(), c.n, c.dcount)));
  unsigned long long h[4];
  SPHG_CUDA_CHECK(cudaMemcpyAsync(h, c.dcount, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
  host_sync(c, c.stream);
  for (int k = 0; k < 4; ++k) out[k] = (int64_t)h[k];
}

}  // namespace sphg
