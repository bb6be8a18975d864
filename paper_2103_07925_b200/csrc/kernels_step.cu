// kernels_step.cu — the per-step sm_100a kernels of the SPH hot path.
//
//   k_body_kick / k_kick_drift   half kick, drift, orientation, slaving
//   k_density                    density_summation + eos_pressure
//   k_dirichlet / k_heat         apply_thermal_dirichlet + conduction_rhs
//   k_extrapolate                extrapolate_wall_quantities              (Adami 2012)
//   k_forces_fluid               momentum_rhs + transport velocity
//   k_forces_rigid               coupling_force_on_rigid + contact_force
//   k_body_reduce                reduce_force_torque (+ world inertia)
//   k_mass                       reduce_mass_quantities
//   k_body_final / k_final_kick  final half kick + slave velocities
//
// All pair kernels are gather-only (one thread per particle, Verlet ELL list,
// no fp64 atomics), so every sum is deterministic.  The pair arithmetic is
// FMA-contracted fp64; see DESIGN.md §4 for the per-kernel roofline.
#include <cmath>
#include <cstring>

#include "context.cuh"

namespace sphg {

namespace {

__device__ __forceinline__ double3 ld3(const double4& v) { return make_double3(v.x, v.y, v.z); }
__device__ __forceinline__ double3 ldpos(const double4* p) {  // xyz only (never touches .w)
  const double2 xy = *reinterpret_cast<const double2*>(p);
  const double z = reinterpret_cast<const double*>(p)[2];
  return make_double3(xy.x, xy.y, z);
}
__device__ __forceinline__ void stpos(double4* p, double3 v) {
  *reinterpret_cast<double2*>(p) = make_double2(v.x, v.y);
  reinterpret_cast<double*>(p)[2] = v.z;
}
__device__ __forceinline__ double4 ldg4(const double4* p) {  // read-only path, 2 x 16 B
  const double2 a = __ldg(reinterpret_cast<const double2*>(p));
  const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ Quat body_q(const sphg_body& b) { return {b.q[0], b.q[1], b.q[2], b.q[3]}; }
__device__ __forceinline__ double3 bv(const double* p) { return make_double3(p[0], p[1], p[2]); }

template <class T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ------------------------------------------------------------- integrator
__global__ void k_body_kick(const __grid_constant__ DevParams P, sphg_body* __restrict__ B, size_t nb) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nb) return;
  sphg_body b = B[k];
  if (!b.alive || !b.mobile) return;
  double u[3], w[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    u[a] = axpy_rn(b.vel[a], P.hdt, b.acc[a]);
    w[a] = axpy_rn(b.omega[a], P.hdt, b.alpha[a]);
    b.vel[a] = u[a];
    b.omega[a] = w[a];
    b.com[a] = wrap1(P, axpy_rn(b.com[a], P.dt, u[a]), a);
  }
  const Quat q = orientation_step(body_q(b), make_double3(w[0], w[1], w[2]), P.dt);
  b.q[0] = q.w; b.q[1] = q.x; b.q[2] = q.y; b.q[3] = q.z;
  B[k] = b;
}

// fluid: u^{n+1/2} = u + dt/2 a; u~ = u^{n+1/2} + dt/2 a_bg; r += dt u~ (wrapped).
// rigid: r_r = r_k + R(q) chi, u_r = u_k + w x r_rk.  Verlet displacement + u_max.
__global__ void __launch_bounds__(256) k_kick_drift(const __grid_constant__ DevParams P, Particles D,
                                                     const sphg_body* __restrict__ B, size_t n,
                                                     DevFlags* __restrict__ fl) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  double disp2 = 0.0, u2 = 0.0;
  if (k < n) {
    const uint32_t kmd = D.kmd.p[k];
    const uint32_t kind = kind_of(kmd);
    double3 pn;
    bool moved = true;
    if (kind == SPHG_FLUID) {
      const double4 v = D.V4.p[k];
      const double4 a = D.A4.p[k];
      const double3 uh = make_double3(axpy_rn(v.x, P.hdt, a.x), axpy_rn(v.y, P.hdt, a.y), axpy_rn(v.z, P.hdt, a.z));
      double3 ua = uh;
      if (P.tvf) {
        const double4 bg = D.B4.p[k];
        ua = make_double3(axpy_rn(uh.x, P.hdt, bg.x), axpy_rn(uh.y, P.hdt, bg.y), axpy_rn(uh.z, P.hdt, bg.z));
      }
      const double3 p = ldpos(&D.G0.p[k]);
      pn = make_double3(wrap1(P, axpy_rn(p.x, P.dt, ua.x), 0), wrap1(P, axpy_rn(p.y, P.dt, ua.y), 1),
                        wrap1(P, axpy_rn(p.z, P.dt, ua.z), 2));
      stpos(&D.G0.p[k], pn);
      stpos(&D.G1.p[k], uh);
      stpos(&D.G2.p[k], make_double3(__dsub_rn(ua.x, uh.x), __dsub_rn(ua.y, uh.y), __dsub_rn(ua.z, uh.z)));
      u2 = __dadd_rn(__dadd_rn(__dmul_rn(uh.x, uh.x), __dmul_rn(uh.y, uh.y)), __dmul_rn(uh.z, uh.z));
    } else if (kind == SPHG_RIGID) {
      const sphg_body& b = B[D.group.p[k]];
      const double3 rk = qrotate(body_q(b), ld3(D.X4.p[k]));
      pn = make_double3(wrap1(P, __dadd_rn(b.com[0], rk.x), 0), wrap1(P, __dadd_rn(b.com[1], rk.y), 1),
                        wrap1(P, __dadd_rn(b.com[2], rk.z), 2));
      stpos(&D.G0.p[k], pn);
      const double3 wxr = cross3(bv(b.omega), rk);
      stpos(&D.V4.p[k], make_double3(b.vel[0] + wxr.x, b.vel[1] + wxr.y, b.vel[2] + wxr.z));
    } else {
      moved = false;
    }
    if (moved) {
      const double xs[3] = {pn.x, pn.y, pn.z};
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        if (!P.periodic[a] && (xs[a] < P.lo[a] || xs[a] > P.hi[a])) {
          atomicOr(&fl->err, kErrEscape);
          atomicMin(&fl->err_gid, D.gid.p[k]);
        }
      }
      const double4 r0 = D.R4.p[k];
      disp2 = r2_exact(mimg3(P, pn.x, pn.y, pn.z, r0.x, r0.y, r0.z));
    }
  }
  disp2 = warp_max(disp2);
  u2 = warp_max(u2);
  if ((threadIdx.x & 31) == 0) {
    atomic_max_pos_double(&fl->max_disp2_bits, disp2);
    atomic_max_pos_double(&fl->umax2_bits, u2);
  }
}

__global__ void k_body_final(const __grid_constant__ DevParams P, sphg_body* __restrict__ B, size_t nb) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nb) return;
  sphg_body& b = B[k];
  if (!b.alive || !b.mobile) return;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    b.vel[a] = axpy_rn(b.vel[a], P.hdt, b.acc[a]);
    b.omega[a] = axpy_rn(b.omega[a], P.hdt, b.alpha[a]);
  }
}

__global__ void __launch_bounds__(256) k_final_kick(const __grid_constant__ DevParams P, Particles D,
                                                     const sphg_body* __restrict__ B, size_t n) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const uint32_t kind = kind_of(D.kmd.p[k]);
  if (kind == SPHG_FLUID) {
    const double3 uh = ldpos(&D.G1.p[k]);
    const double4 a = D.A4.p[k];
    stpos(&D.V4.p[k], make_double3(axpy_rn(uh.x, P.hdt, a.x), axpy_rn(uh.y, P.hdt, a.y), axpy_rn(uh.z, P.hdt, a.z)));
  } else if (kind == SPHG_RIGID) {
    const sphg_body& b = B[D.group.p[k]];
    const double3 rk = qrotate(body_q(b), ld3(D.X4.p[k]));
    const double3 wxr = cross3(bv(b.omega), rk);
    stpos(&D.V4.p[k], make_double3(b.vel[0] + wxr.x, b.vel[1] + wxr.y, b.vel[2] + wxr.z));
  }
}

// ---------------------------------------------------------------- density
// rho_i = m_i sigma (66 + sum_j shape(r_ij/h)), p_i = c^2 (rho_i - rho0), V_i = m_i/rho_i
__global__ void __launch_bounds__(128) k_density(const __grid_constant__ DevParams P, Particles D,
                                                  const uint32_t* __restrict__ nbr, const uint32_t* __restrict__ cnt,
                                                  size_t n) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t kmd = D.kmd.p[i];
  if (kind_of(kmd) != SPHG_FLUID) return;
  const double3 pi = ldpos(&D.G0.p[i]);
  const int nc = (int)cnt[i];
  double s = 66.0;  // self term shape(0)
  const uint32_t* nb = nbr + i;
  int k = 0;
  for (; k + 1 < nc; k += 2) {  // 2-way unroll: two independent gathers in flight
    const uint32_t j0 = __ldg(nb + (size_t)k * n), j1 = __ldg(nb + (size_t)(k + 1) * n);
    const double3 p0 = ldpos(&D.G0.p[j0]);
    const double3 p1 = ldpos(&D.G0.p[j1]);
    const double3 d0 = mimg3(P, pi.x, pi.y, pi.z, p0.x, p0.y, p0.z);
    const double3 d1 = mimg3(P, pi.x, pi.y, pi.z, p1.x, p1.y, p1.z);
    const double r20 = d0.x * d0.x + d0.y * d0.y + d0.z * d0.z;
    const double r21 = d1.x * d1.x + d1.y * d1.y + d1.z * d1.z;
    if (r20 <= P.rc2) s += shape_q(sqrt(r20) * P.inv_h);
    if (r21 <= P.rc2) s += shape_q(sqrt(r21) * P.inv_h);
  }
  if (k < nc) {
    const uint32_t j = __ldg(nb + (size_t)k * n);
    const double3 pj = ldpos(&D.G0.p[j]);
    const double3 d = mimg3(P, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z);
    const double r2 = d.x * d.x + d.y * d.y + d.z * d.z;
    if (r2 <= P.rc2) s += shape_q(sqrt(r2) * P.inv_h);
  }
  const DevMat& M = P.mat[mat_of(kmd)];
  const double m = D.V4.p[i].w;
  const double rho = m * (P.sigma * s);
  const double V = m / rho;
  reinterpret_cast<double*>(&D.G0.p[i])[3] = V * V;
  reinterpret_cast<double*>(&D.G1.p[i])[3] = rho;
  reinterpret_cast<double*>(&D.G2.p[i])[3] = M.c2 * (rho - M.rho0);
  if (P.thermal) reinterpret_cast<double*>(&D.H2.p[i])[1] = V;
}

// ------------------------------------------------------------------- heat
__device__ __forceinline__ double sched_value(const DevSchedule& s, double t) {  // Schedule::value_at
  for (int k = 0; k < s.n; ++k)
    if (t <= s.t_end[k]) return s.value[k];
  return s.value[s.n - 1];
}

__global__ void k_dirichlet(const __grid_constant__ DevParams P, Particles D, size_t n, double t_new) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t kmd = D.kmd.p[i];
  if (kind_of(kmd) != SPHG_BOUNDARY) return;
  const uint32_t g = dir_of(kmd);
  if (g == SPHG_NO_DIRICHLET || (int)g >= P.n_sched || P.sched[g].n <= 0) return;
  reinterpret_cast<double*>(&D.H2.p[i])[0] = sched_value(P.sched[g], t_new);
}

// c_p,a dT_a/dt = (1/rho_a) sum_b V_b 4 k_a k_b/(k_a+k_b) (T_ab/r_ab) dW/dr (Cleary & Monaghan)
__global__ void __launch_bounds__(128) k_heat(const __grid_constant__ DevParams P, Particles D,
                                               const uint32_t* __restrict__ nbr, const uint32_t* __restrict__ cnt,
                                               double2* __restrict__ Hout, size_t n, DevFlags* __restrict__ fl) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t kmd = D.kmd.p[i];
  const uint32_t kind = kind_of(kmd);
  const double2 hi = D.H2.p[i];
  if (kind == SPHG_BOUNDARY) {
    Hout[i] = hi;
    return;
  }
  const DevMat& Ma = P.mat[mat_of(kmd)];
  const double3 pi = ldpos(&D.G0.p[i]);
  const double rho_a = kind == SPHG_FLUID ? D.G1.p[i].w : Ma.rho0;
  const int nc = (int)cnt[i];
  double s = 0.0;
  bool coincident = false;
  for (int k = 0; k < nc; ++k) {
    const uint32_t j = __ldg(nbr + (size_t)k * n + i);
    const double2 hj = D.H2.p[j];
    if (hj.y == 0.0) continue;  // non-Dirichlet wall: no conduction
    const double3 pj = ldpos(&D.G0.p[j]);
    const double3 d = mimg3(P, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z);
    const double r2 = d.x * d.x + d.y * d.y + d.z * d.z;
    if (r2 > P.rc2) continue;
    if (r2 == 0.0) {
      coincident = true;
      continue;
    }
    double kt;
    if (P.single_kappa) {
      if (Ma.kappa == 0.0) continue;
      kt = 4.0 * Ma.kappa * Ma.kappa / (Ma.kappa + Ma.kappa);
    } else {
      const DevMat& Mb = P.mat[mat_of(D.kmd.p[j])];
      const double ks = Ma.kappa + Mb.kappa;
      if (ks == 0.0) continue;
      kt = 4.0 * Ma.kappa * Mb.kappa / ks;
    }
    const double rinv = rsqrt(r2);
    const double r = r2 * rinv;
    const double dW = P.sig_h * shape_deriv_q(r * P.inv_h);
    s += hj.y * kt * ((hi.x - hj.x) * rinv) * dW;
  }
  if (coincident) {
    atomicOr(&fl->err, kErrCoincident);
    atomicMin(&fl->err_gid, D.gid.p[i]);
  }
  double rate = 0.0;
  if (Ma.cp > 0.0) rate = s / (rho_a * Ma.cp);
  Hout[i] = make_double2(hi.x + P.dt * rate, hi.y);
  D.dTdt.p[i] = rate;
}

// ---------------------------------------------------------- extrapolation
// p_w = sum_f W (p_f + rho_f (g_f - a_w).(r_w - r_f)) / sum_f W;  u~_w = 2 u_w - sum_f W u_f / sum_f W;
// rho_w = max(rho0, rho0 + p_w/c^2) of the dominant fluid material; V_w = rho0 dx^3 / rho_w  [P6][P7]
template <bool kMultiEos>
__global__ void __launch_bounds__(128) k_extrapolate(const __grid_constant__ DevParams P, Particles D,
                                                      const sphg_body* __restrict__ B,
                                                      const uint32_t* __restrict__ nbr,
                                                      const uint32_t* __restrict__ cnt, size_t n) {
  const size_t w = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= n) return;
  const uint32_t kmd = D.kmd.p[w];
  const uint32_t kind = kind_of(kmd);
  if (kind == SPHG_FLUID) return;
  double3 uw = make_double3(0, 0, 0), aw = make_double3(0, 0, 0);
  if (kind == SPHG_RIGID) {
    const sphg_body& b = B[D.group.p[w]];
    const double3 rk = qrotate(body_q(b), ld3(D.X4.p[w]));
    const double3 om = bv(b.omega);
    const double3 t1 = cross3(bv(b.alpha), rk);
    const double3 t2 = cross3(om, cross3(om, rk));
    aw = make_double3(b.acc[0] + t1.x + t2.x, b.acc[1] + t1.y + t2.y, b.acc[2] + t1.z + t2.z);
    uw = ldpos(&D.V4.p[w]);
  }
  const double3 pw = ldpos(&D.G0.p[w]);
  double sw = 0.0, sp = 0.0;
  double3 su = make_double3(0, 0, 0);
  double smat[kMultiEos ? kMaxMat : 1];
  if (kMultiEos)
    for (int m = 0; m < kMaxMat; ++m) smat[m] = 0.0;
  const int nc = (int)cnt[w];
  for (int k = 0; k < nc; ++k) {
    const uint32_t f = __ldg(nbr + (size_t)k * n + w);
    const uint32_t kf = D.kmd.p[f];
    if (kind_of(kf) != SPHG_FLUID) continue;
    const double3 pf = ldpos(&D.G0.p[f]);
    const double3 d = mimg3(P, pw.x, pw.y, pw.z, pf.x, pf.y, pf.z);
    const double r2 = d.x * d.x + d.y * d.y + d.z * d.z;
    if (r2 > P.rc2) continue;
    const double W = shape_q(sqrt(r2) * P.inv_h);  // sigma cancels in every ratio
    const double4 g1 = D.G1.p[f];
    const double pf_ = D.G2.p[f].w;
    const DevMat& Mf = P.mat[mat_of(kf)];
    const double ga = (Mf.g[0] - aw.x) * d.x + (Mf.g[1] - aw.y) * d.y + (Mf.g[2] - aw.z) * d.z;
    sw += W;
    sp += W * (pf_ + g1.w * ga);
    su.x += W * g1.x;
    su.y += W * g1.y;
    su.z += W * g1.z;
    if (kMultiEos) smat[mat_of(kf)] += W;
  }
  int m = P.default_fluid_mat;
  if (kMultiEos && sw > 0.0) {
    double best = -1.0;
    for (int q = 0; q < P.n_mat; ++q)
      if (smat[q] > best) {
        best = smat[q];
        m = q;
      }
  }
  const DevMat& M = P.mat[m];
  double p_w = 0.0;
  double3 ut = uw;
  if (sw > 0.0) {
    const double inv = 1.0 / sw;
    p_w = sp * inv;
    ut = make_double3(2.0 * uw.x - su.x * inv, 2.0 * uw.y - su.y * inv, 2.0 * uw.z - su.z * inv);
  }
  const double rho_w = fmax(M.rho0, M.rho0 + p_w * M.inv_c2);
  const double V_w = M.rho0 * P.dx3 / rho_w;
  reinterpret_cast<double*>(&D.G0.p[w])[3] = V_w * V_w;
  D.G1.p[w] = make_double4(ut.x, ut.y, ut.z, rho_w);
  D.G2.p[w] = make_double4(0.0, 0.0, 0.0, p_w);
}

// ---------------------------------------------------------------- forces
// a_ij = (V_i^2 + V_j^2)/m_i [ -p~ gradW + eta~ (u_i-u_j) (dW/dr)/r + 1/2 (A_i + A_j) gradW ],
// A = rho u (u~ - u)^T, gradW = dW/dr e_ij;  a_bg,i = -(p_b/m_i) sum (V_i^2+V_j^2) gradW.
struct PairSide {
  double3 u, du;
  double rho, p, V2, eta;
};

template <bool kTvf>
__device__ __forceinline__ void pair_term(const PairSide& I, const PairSide& J, double3 d, double r2, double sig_h,
                                          double inv_h, double3& acc, double3& bg) {
  const double rinv = rsqrt(r2);
  const double r = r2 * rinv;
  const double dW = sig_h * shape_deriv_q(r * inv_h);
  const double fac = dW * rinv;  // gradW = fac * d
  const double3 gW = make_double3(fac * d.x, fac * d.y, fac * d.z);
  const double V2 = I.V2 + J.V2;
  const double pt = (J.rho * I.p + I.rho * J.p) * rcp_fast(I.rho + J.rho);
  const double es = I.eta + J.eta;
  const double et = es > 0.0 ? 2.0 * I.eta * J.eta * rcp_fast(es) : 0.0;
  const double vf = et * fac;
  double3 t = make_double3(vf * (I.u.x - J.u.x) - pt * gW.x, vf * (I.u.y - J.u.y) - pt * gW.y,
                           vf * (I.u.z - J.u.z) - pt * gW.z);
  if (kTvf) {
    const double ai = 0.5 * I.rho * (I.du.x * gW.x + I.du.y * gW.y + I.du.z * gW.z);
    const double aj = 0.5 * J.rho * (J.du.x * gW.x + J.du.y * gW.y + J.du.z * gW.z);
    t.x += ai * I.u.x + aj * J.u.x;
    t.y += ai * I.u.y + aj * J.u.y;
    t.z += ai * I.u.z + aj * J.u.z;
  }
  acc.x += V2 * t.x;
  acc.y += V2 * t.y;
  acc.z += V2 * t.z;
  bg.x += V2 * gW.x;
  bg.y += V2 * gW.y;
  bg.z += V2 * gW.z;
}

template <bool kTvf, bool kMultiEta>
__global__ void __launch_bounds__(128) k_forces_fluid(const __grid_constant__ DevParams P, Particles D,
                                                       const uint32_t* __restrict__ nbr,
                                                       const uint32_t* __restrict__ cnt, size_t n,
                                                       DevFlags* __restrict__ fl) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t kmd = D.kmd.p[i];
  if (kind_of(kmd) != SPHG_FLUID) return;
  const DevMat& M = P.mat[mat_of(kmd)];
  const double4 g0 = D.G0.p[i], g1 = D.G1.p[i], g2 = D.G2.p[i];
  PairSide I;
  I.u = ld3(g1);
  I.du = ld3(g2);
  I.rho = g1.w;
  I.p = g2.w;
  I.V2 = g0.w;
  I.eta = M.eta;
  const double m_i = D.V4.p[i].w;
  double3 acc = make_double3(0, 0, 0), bg = make_double3(0, 0, 0);
  bool coincident = false;
  const int nc = (int)cnt[i];
  const uint32_t* nb = nbr + i;
  for (int k = 0; k < nc; ++k) {
    const uint32_t j = __ldg(nb + (size_t)k * n);
    const double4 h0 = ldg4(&D.G0.p[j]);
    const double3 d = mimg3(P, g0.x, g0.y, g0.z, h0.x, h0.y, h0.z);
    const double r2 = d.x * d.x + d.y * d.y + d.z * d.z;
    if (r2 > P.rc2) continue;
    if (r2 == 0.0) {
      coincident = true;
      continue;
    }
    const double4 h1 = ldg4(&D.G1.p[j]);
    const double4 h2 = ldg4(&D.G2.p[j]);
    PairSide J;
    J.u = ld3(h1);
    J.du = ld3(h2);
    J.rho = h1.w;
    J.p = h2.w;
    J.V2 = h0.w;
    if (kMultiEta) {
      const uint32_t kj = __ldg(&D.kmd.p[j]);
      J.eta = kind_of(kj) == SPHG_FLUID ? P.mat[mat_of(kj)].eta : I.eta;  // eta_w := eta_i [P7]
    } else {
      J.eta = I.eta;
    }
    pair_term<kTvf>(I, J, d, r2, P.sig_h, P.inv_h, acc, bg);
  }
  if (coincident) {
    atomicOr(&fl->err, kErrCoincident);
    atomicMin(&fl->err_gid, D.gid.p[i]);
  }
  const double im = 1.0 / m_i;
  D.A4.p[i] = make_double4(acc.x * im + M.g[0], acc.y * im + M.g[1], acc.z * im + M.g[2], 0.0);
  const double f = kTvf ? -M.pb * im : 0.0;
  D.B4.p[i] = make_double4(f * bg.x, f * bg.y, f * bg.z, 0.0);
}

// f_r = sum_i -m_i a_ir (fluid neighbours, a_ir from the fluid's view) + contact
template <bool kTvf>
__global__ void __launch_bounds__(128) k_forces_rigid(const __grid_constant__ DevParams P, Particles D,
                                                       const uint32_t* __restrict__ nbr,
                                                       const uint32_t* __restrict__ cnt, size_t n,
                                                       DevFlags* __restrict__ fl) {
  const size_t r = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const uint32_t kmd = D.kmd.p[r];
  if (kind_of(kmd) != SPHG_RIGID) return;
  const double4 g0 = D.G0.p[r], g1 = D.G1.p[r], g2 = D.G2.p[r];
  const double3 vr = ldpos(&D.V4.p[r]);
  const uint32_t body = D.group.p[r];
  PairSide R;
  R.u = ld3(g1);
  R.du = make_double3(0, 0, 0);
  R.rho = g1.w;
  R.p = g2.w;
  R.V2 = g0.w;
  double3 f = make_double3(0, 0, 0);
  bool coincident = false;
  const int nc = (int)cnt[r];
  for (int k = 0; k < nc; ++k) {
    const uint32_t j = __ldg(nbr + (size_t)k * n + r);
    const uint32_t kj = D.kmd.p[j];
    const uint32_t kindj = kind_of(kj);
    const double4 h0 = D.G0.p[j];
    if (kindj == SPHG_FLUID) {
      const double3 d = mimg3(P, h0.x, h0.y, h0.z, g0.x, g0.y, g0.z);  // r_j - r_r
      const double r2 = d.x * d.x + d.y * d.y + d.z * d.z;
      if (r2 > P.rc2) continue;
      if (r2 == 0.0) {
        coincident = true;
        continue;
      }
      const double4 h1 = D.G1.p[j], h2 = D.G2.p[j];
      const DevMat& Mj = P.mat[mat_of(kj)];
      PairSide J;
      J.u = ld3(h1);
      J.du = ld3(h2);
      J.rho = h1.w;
      J.p = h2.w;
      J.V2 = h0.w;
      J.eta = Mj.eta;
      R.eta = Mj.eta;  // eta_w := eta_i
      double3 a = make_double3(0, 0, 0), bgd = make_double3(0, 0, 0);
      pair_term<kTvf>(J, R, d, r2, P.sig_h, P.inv_h, a, bgd);
      const double m_j = D.V4.p[j].w;
      // f_ri = -m_i a_ir = -(V2 term) since a_ir = (V2/m_i) term
      f.x -= a.x;
      f.y -= a.y;
      f.z -= a.z;
      (void)m_j;
    } else if (kindj == SPHG_BOUNDARY || D.group.p[j] != body) {
      const double3 d = mimg3(P, g0.x, g0.y, g0.z, h0.x, h0.y, h0.z);  // r_r - r_j
      const double r2 = d.x * d.x + d.y * d.y + d.z * d.z;
      const double rr = sqrt(r2);
      if (!(rr < P.dx)) continue;
      if (rr == 0.0) {
        coincident = true;
        continue;
      }
      const double ri = 1.0 / rr;
      const double3 e = make_double3(d.x * ri, d.y * ri, d.z * ri);
      const double3 vj = ldpos(&D.V4.p[j]);
      const double s = P.kc * (rr - P.dx) + P.dc * (e.x * (vr.x - vj.x) + e.y * (vr.y - vj.y) + e.z * (vr.z - vj.z));
      const double fm = -fmin(0.0, s);
      f.x += fm * e.x;
      f.y += fm * e.y;
      f.z += fm * e.z;
    }
  }
  if (coincident) {
    atomicOr(&fl->err, kErrCoincident);
    atomicMin(&fl->err_gid, D.gid.p[r]);
  }
  D.F4.p[r] = make_double4(f.x, f.y, f.z, 0.0);
}

// ----------------------------------------------------------------- bodies
__device__ void inverse_apply(const double I[6], double3 t, double3& out) {
  const double xx = I[0], yy = I[1], zz = I[2], xy = I[3], xz = I[4], yz = I[5];
  const double c00 = yy * zz - yz * yz, c01 = xz * yz - xy * zz, c02 = xy * yz - xz * yy;
  const double c11 = xx * zz - xz * xz, c12 = xy * xz - xx * yz, c22 = xx * yy - xy * xy;
  const double det = xx * c00 + xy * c01 + xz * c02;
  const double tr = xx + yy + zz;
  if (!(fabs(det) > 1e-12 * tr * tr * tr)) {  // singular: zero angular acceleration
    out = make_double3(0, 0, 0);
    return;
  }
  out = make_double3((c00 * t.x + c01 * t.y + c02 * t.z) / det, (c01 * t.x + c11 * t.y + c12 * t.z) / det,
                     (c02 * t.x + c12 * t.y + c22 * t.z) / det);
}

// one warp per body: compensated (f, tau, I) over the body-major rigid index
__global__ void __launch_bounds__(128) k_body_reduce(const __grid_constant__ DevParams P, Particles D,
                                                      sphg_body* __restrict__ B, size_t nb,
                                                      const uint32_t* __restrict__ ridx,
                                                      const uint32_t* __restrict__ bstart,
                                                      const uint32_t* __restrict__ bend) {
  const size_t k = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (k >= nb) return;
  sphg_body& b = B[k];
  if (!b.alive) return;
  const Quat q = body_q(b);
  KSum acc[12];
#pragma unroll
  for (int c = 0; c < 12; ++c) acc[c] = {0.0, 0.0};
  const uint32_t s0 = bstart[k], s1 = bend[k];
  for (uint32_t s = s0 + lane; s < s1; s += 32) {
    const uint32_t r = ridx[s];
    const double3 rk = qrotate(q, ld3(D.X4.p[r]));
    const double4 f4 = D.F4.p[r];
    const double m = D.V4.p[r].w;
    const double3 t = make_double3(rk.y * f4.z - rk.z * f4.y, rk.z * f4.x - rk.x * f4.z, rk.x * f4.y - rk.y * f4.x);
    const double Ir = P.Ir_over_m * m;
    const double d2 = (rk.x * rk.x + rk.y * rk.y) + rk.z * rk.z;
    acc[0].add(f4.x); acc[1].add(f4.y); acc[2].add(f4.z);
    acc[3].add(t.x); acc[4].add(t.y); acc[5].add(t.z);
    acc[6].add(Ir + m * (d2 - rk.x * rk.x));
    acc[7].add(Ir + m * (d2 - rk.y * rk.y));
    acc[8].add(Ir + m * (d2 - rk.z * rk.z));
    acc[9].add(-m * rk.x * rk.y);
    acc[10].add(-m * rk.x * rk.z);
    acc[11].add(-m * rk.y * rk.z);
  }
  double v[12];
#pragma unroll
  for (int c = 0; c < 12; ++c) v[c] = warp_merge(acc[c]).value();
  if (lane != 0) return;
  for (int a = 0; a < 3; ++a) {
    b.force[a] = v[a];
    b.torque[a] = v[3 + a];
  }
  for (int a = 0; a < 6; ++a) b.inertia[a] = v[6 + a];
  if (b.mobile && b.mass > 0.0) {
    const DevMat& M = P.mat[b.material];
    for (int a = 0; a < 3; ++a) b.acc[a] = v[a] / b.mass + M.g[a];
    double3 al;
    inverse_apply(b.inertia, make_double3(v[3], v[4], v[5]), al);
    b.alpha[0] = al.x; b.alpha[1] = al.y; b.alpha[2] = al.z;
  } else {
    for (int a = 0; a < 3; ++a) b.acc[a] = b.alpha[a] = 0.0;
  }
}

// reduce_mass_quantities: anchor = min-gid member, minimum image; chi := R(q)^T (r_r - r_k)
__global__ void __launch_bounds__(128) k_mass(const __grid_constant__ DevParams P, Particles D,
                                               sphg_body* __restrict__ B, size_t nb, const uint32_t* __restrict__ ridx,
                                               const uint32_t* __restrict__ bstart,
                                               const uint32_t* __restrict__ bend,
                                               const uint32_t* __restrict__ mask) {
  const size_t k = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (k >= nb) return;
  if (mask && !mask[k]) return;
  sphg_body& b = B[k];
  if (!mask && !b.alive) return;
  const uint32_t s0 = bstart[k], s1 = bend[k];
  if (s1 <= s0) {
    if (lane == 0) {
      b.alive = 0;
      b.mass = 0.0;
    }
    return;
  }
  const double3 anc = ldpos(&D.G0.p[ridx[s0]]);
  KSum M = {0, 0}, MR[3] = {{0, 0}, {0, 0}, {0, 0}};
  for (uint32_t s = s0 + lane; s < s1; s += 32) {
    const uint32_t r = ridx[s];
    const double3 p = ldpos(&D.G0.p[r]);
    const double m = D.V4.p[r].w;
    const double3 d = mimg3(P, p.x, p.y, p.z, anc.x, anc.y, anc.z);
    M.add(m);
    MR[0].add(__dmul_rn(m, d.x));
    MR[1].add(__dmul_rn(m, d.y));
    MR[2].add(__dmul_rn(m, d.z));
  }
  const double mt = __shfl_sync(0xffffffffu, warp_merge(M).value(), 0);
  double cm[3];
  for (int a = 0; a < 3; ++a) {
    const double mr = __shfl_sync(0xffffffffu, warp_merge(MR[a]).value(), 0);
    cm[a] = wrap1(P, __dadd_rn((&anc.x)[a], __ddiv_rn(mr, mt)), a);
  }
  const Quat qc = {b.q[0], -b.q[1], -b.q[2], -b.q[3]};
  KSum I6[6];
  for (int c = 0; c < 6; ++c) I6[c] = {0.0, 0.0};
  for (uint32_t s = s0 + lane; s < s1; s += 32) {
    const uint32_t r = ridx[s];
    const double3 p = ldpos(&D.G0.p[r]);
    const double m = D.V4.p[r].w;
    const double3 d = mimg3(P, p.x, p.y, p.z, cm[0], cm[1], cm[2]);
    const double Ir = P.Ir_over_m * m;
    const double d2 = (d.x * d.x + d.y * d.y) + d.z * d.z;
    I6[0].add(Ir + m * (d2 - d.x * d.x));
    I6[1].add(Ir + m * (d2 - d.y * d.y));
    I6[2].add(Ir + m * (d2 - d.z * d.z));
    I6[3].add(-m * d.x * d.y);
    I6[4].add(-m * d.x * d.z);
    I6[5].add(-m * d.y * d.z);
    const double3 chi = qrotate(qc, d);
    D.X4.p[r] = make_double4(chi.x, chi.y, chi.z, 0.0);
  }
  double iv[6];
  for (int c = 0; c < 6; ++c) iv[c] = warp_merge(I6[c]).value();
  if (lane == 0) {
    b.mass = mt;
    for (int a = 0; a < 3; ++a) b.com[a] = cm[a];
    for (int c = 0; c < 6; ++c) b.inertia[c] = iv[c];
    b.alive = 1;
  }
}


__global__ void k_gather_by_gid(Particles cur, Particles src, size_t n) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const uint32_t g = cur.gid.p[k];
  cur.G0.p[k] = src.G0.p[g];
  cur.G1.p[k] = src.G1.p[g];
  cur.G2.p[k] = src.G2.p[g];
  cur.V4.p[k] = src.V4.p[g];
  cur.A4.p[k] = src.A4.p[g];
  cur.B4.p[k] = src.B4.p[g];
  cur.F4.p[k] = src.F4.p[g];
  cur.X4.p[k] = src.X4.p[g];
  cur.H2.p[k] = src.H2.p[g];
  cur.dTdt.p[k] = src.dTdt.p[g];
  cur.p_static.p[k] = src.p_static.p[g];
  cur.kmd.p[k] = src.kmd.p[g];
  cur.group.p[k] = src.group.p[g];
}

__global__ void k_disp(const __grid_constant__ DevParams P, Particles D, size_t n, DevFlags* __restrict__ fl) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  double d2 = 0.0;
  if (k < n) {
    const double4 p = D.G0.p[k], r = D.R4.p[k];
    d2 = r2_exact(mimg3(P, p.x, p.y, p.z, r.x, r.y, r.z));
  }
  d2 = warp_max(d2);
  if ((threadIdx.x & 31) == 0) atomic_max_pos_double(&fl->max_disp2_bits, d2);
}

__global__ void k_iota(uint32_t* __restrict__ a, size_t n) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) a[k] = (uint32_t)k;
}

__global__ void k_count_pairs(const __grid_constant__ DevParams P, Particles D, const uint32_t* __restrict__ nbr,
                              const uint32_t* __restrict__ cnt, size_t n, unsigned long long* __restrict__ out) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long c = 0, in = 0;
  if (i < n) {
    const double4 pi = D.G0.p[i];
    c = cnt[i];
    for (uint32_t k = 0; k < cnt[i]; ++k) {
      const double4 pj = D.G0.p[nbr[(size_t)k * n + i]];
      if (r2_exact(mimg3(P, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z)) <= P.rc2) ++in;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    c += __shfl_xor_sync(0xffffffffu, c, o);
    in += __shfl_xor_sync(0xffffffffu, in, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(out, c);
    atomicAdd(out + 1, in);
  }
}

}  // namespace

void gather_by_gid(Ctx& c) {
  k_gather_by_gid<<<grid_for(c.n, 256), 256, 0, c.stream>>>(c.cur, c.alt, c.n);
  c.launches++;
}

bool displacement_exceeds(Ctx& c) {
  SPHG_CUDA_CHECK(cudaMemsetAsync(&c.dflags->max_disp2_bits, 0, 8, c.stream));
  k_disp<<<grid_for(c.n, 256), 256, 0, c.stream>>>(c.P, c.cur, c.n, c.dflags);
  unsigned long long b = 0;
  SPHG_CUDA_CHECK(cudaMemcpyAsync(&b, &c.dflags->max_disp2_bits, 8, cudaMemcpyDeviceToHost, c.stream));
  SPHG_CUDA_CHECK(cudaStreamSynchronize(c.stream));
  double d2;
  memcpy(&d2, &b, 8);
  c.launches += 2;
  return std::sqrt(d2) > c.P.half_skin;
}

void iota_gid(Ctx& c) {
  k_iota<<<grid_for(c.n, 256), 256, 0, c.stream>>>(c.cur.gid.p, c.n);
  c.launches++;
}

void count_pairs(Ctx& c, int64_t* candidates, int64_t* interacting) {
  if (!c.dcount) SPHG_CUDA_CHECK(cudaMalloc(&c.dcount, 2 * sizeof(unsigned long long)));
  SPHG_CUDA_CHECK(cudaMemsetAsync(c.dcount, 0, 2 * sizeof(unsigned long long), c.stream));
  k_count_pairs<<<grid_for(c.n, 128), 128, 0, c.stream>>>(c.P, c.cur, c.nbr.p, c.cnt.p, c.n, c.dcount);
  unsigned long long h[2];
  SPHG_CUDA_CHECK(cudaMemcpyAsync(h, c.dcount, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
  SPHG_CUDA_CHECK(cudaStreamSynchronize(c.stream));
  *candidates = (int64_t)h[0];
  *interacting = (int64_t)h[1];
}

// ============================================================= launchers
void launch_body_kick(Ctx& c) {
  if (c.nb == 0) return;
  k_body_kick<<<grid_for(c.nb, 128), 128, 0, c.stream>>>(c.P, c.bodies.p, c.nb);
  c.launches++;
}

void launch_kick_drift(Ctx& c) {
  k_kick_drift<<<grid_for(c.n, 256), 256, 0, c.stream>>>(c.P, c.cur, c.bodies.p, c.n, c.dflags);
  c.launches++;
}

void launch_density(Ctx& c) {
  k_density<<<grid_for(c.n, 128), 128, 0, c.stream>>>(c.P, c.cur, c.nbr.p, c.cnt.p, c.n);
  c.launches++;
}

void launch_heat(Ctx& c) {
  const double t_new = c.t + c.P.dt;
  k_dirichlet<<<grid_for(c.n, 256), 256, 0, c.stream>>>(c.P, c.cur, c.n, t_new);
  k_heat<<<grid_for(c.n, 128), 128, 0, c.stream>>>(c.P, c.cur, c.nbr.p, c.cnt.p, c.H2new.p, c.n, c.dflags);
  std::swap(c.cur.H2, c.H2new);
  c.launches += 2;
}

void launch_extrapolate(Ctx& c) {
  if (c.P.single_eos)
    k_extrapolate<false><<<grid_for(c.n, 128), 128, 0, c.stream>>>(c.P, c.cur, c.bodies.p, c.nbr.p, c.cnt.p, c.n);
  else
    k_extrapolate<true><<<grid_for(c.n, 128), 128, 0, c.stream>>>(c.P, c.cur, c.bodies.p, c.nbr.p, c.cnt.p, c.n);
  c.launches++;
}

void launch_forces(Ctx& c) {
  const int g = grid_for(c.n, 128);
  const bool tvf = c.P.tvf != 0, multi = c.P.single_eta == 0;
  if (tvf && !multi) k_forces_fluid<true, false><<<g, 128, 0, c.stream>>>(c.P, c.cur, c.nbr.p, c.cnt.p, c.n, c.dflags);
  else if (tvf && multi) k_forces_fluid<true, true><<<g, 128, 0, c.stream>>>(c.P, c.cur, c.nbr.p, c.cnt.p, c.n, c.dflags);
  else if (!multi) k_forces_fluid<false, false><<<g, 128, 0, c.stream>>>(c.P, c.cur, c.nbr.p, c.cnt.p, c.n, c.dflags);
  else k_forces_fluid<false, true><<<g, 128, 0, c.stream>>>(c.P, c.cur, c.nbr.p, c.cnt.p, c.n, c.dflags);
  if (c.nrigid > 0) {
    if (tvf) k_forces_rigid<true><<<g, 128, 0, c.stream>>>(c.P, c.cur, c.nbr.p, c.cnt.p, c.n, c.dflags);
    else k_forces_rigid<false><<<g, 128, 0, c.stream>>>(c.P, c.cur, c.nbr.p, c.cnt.p, c.n, c.dflags);
    c.launches++;
  }
  c.launches++;
}

void launch_bodies(Ctx& c) {
  if (c.nb == 0) return;
  k_body_reduce<<<grid_for(c.nb * 32, 128), 128, 0, c.stream>>>(c.P, c.cur, c.bodies.p, c.nb, c.ridx.p,
                                                                 c.body_start.p, c.body_start.p + c.nb);
  c.launches++;
}

void launch_final_kick(Ctx& c) {
  if (c.nb) k_body_final<<<grid_for(c.nb, 128), 128, 0, c.stream>>>(c.P, c.bodies.p, c.nb);
  k_final_kick<<<grid_for(c.n, 256), 256, 0, c.stream>>>(c.P, c.cur, c.bodies.p, c.n);
  c.launches += c.nb ? 2 : 1;
}

void launch_mass(Ctx& c, const uint32_t* mask) {
  if (c.nb == 0) return;
  k_mass<<<grid_for(c.nb * 32, 128), 128, 0, c.stream>>>(c.P, c.cur, c.bodies.p, c.nb, c.ridx.p, c.body_start.p,
                                                         c.body_start.p + c.nb, mask);
  c.launches++;
}

}  // namespace sphg
