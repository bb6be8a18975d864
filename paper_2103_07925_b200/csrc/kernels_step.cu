// kernels_step.cu — the per-step sm_100a kernels of the SPH hot path.
//
//   k_body_kick / k_kick_drift   half kick, drift, orientation, slaving
//   (pair sums: kernels_pairs.cu)
//   k_body_reduce                reduce_force_torque (+ world inertia)
//   k_mass                       reduce_mass_quantities
//   k_body_final / k_final_kick  final half kick + slave velocities
//
// Also here: the decomposition hooks (halo pack/unpack, per-body partials and totals), the
// warm-upload gather by gid and the Verlet displacement check.  Every body sum is a fixed-order
// compensated reduction (no fp64 atomics), so results are deterministic; the kick / drift
// arithmetic uses round-to-nearest intrinsics to match the oracle bit for bit [P17].  Inside one
// sphg_step(K) call the particle final kick is folded into the next kick-drift (k_kick_drift<true>).
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
// kFinal: the previous step's final fluid kick (u^n = u^{n-1/2} + dt/2 a^n, k_final_kick) is folded
// in, with the same two roundings as the separate kernels, so the fused pass is bit-identical.
template <bool kFinal>
__global__ void __launch_bounds__(256) k_kick_drift(const __grid_constant__ DevParams P, Particles D,
                                                     const sphg_body* __restrict__ B, size_t n,
                                                     DevFlags* __restrict__ fl, uint32_t* __restrict__ wrap_list) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  double disp2 = 0.0, u2 = 0.0;
  if (k < n) {
    const uint32_t kmd = D.kmd.p[k];
    const uint32_t kind = is_ghost(kmd) ? 3u : kind_of(kmd);  // ghosts are integrated by their owner
    double3 pn;
    bool moved = true;
    if (kind == SPHG_FLUID) {
      const double4 a = D.A4.p[k];
      const double3 p = ldpos(&D.G0.p[k]);
      // a buffer-zone particle moves with the zone's prescribed velocity [P23] (role from x^n)
      const int zb = P.n_buf ? buffer_of(P, p.x, p.y, p.z) : -1;
      double3 v;
      if (kFinal) {
        if (zb >= 0) {
          v = buffer_velocity(P, zb, p.x, p.y, p.z, P.buf_prev);
        } else {
          const double3 uprev = ldpos(&D.G1.p[k]);
          v = make_double3(axpy_rn(uprev.x, P.hdt, a.x), axpy_rn(uprev.y, P.hdt, a.y), axpy_rn(uprev.z, P.hdt, a.z));
        }
        stpos(&D.V4.p[k], v);
      } else {
        v = ldpos(&D.V4.p[k]);
      }
      double3 uh, ua;
      if (zb >= 0) {
        uh = ua = buffer_velocity(P, zb, p.x, p.y, p.z, P.buf_half);
      } else {
        uh = make_double3(axpy_rn(v.x, P.hdt, a.x), axpy_rn(v.y, P.hdt, a.y), axpy_rn(v.z, P.hdt, a.z));
        ua = uh;
        if (P.tvf) {
          const double4 bg = D.B4.p[k];
          ua = make_double3(axpy_rn(uh.x, P.hdt, bg.x), axpy_rn(uh.y, P.hdt, bg.y), axpy_rn(uh.z, P.hdt, bg.z));
        }
      }
      pn = make_double3(wrap1(P, axpy_rn(p.x, P.dt, ua.x), 0), wrap1(P, axpy_rn(p.y, P.dt, ua.y), 1),
                        wrap1(P, axpy_rn(p.z, P.dt, ua.z), 2));
      record_wrap(P, fl, wrap_list, (uint32_t)k, p, pn);
      stpos(&D.G0.p[k], pn);
      stpos(&D.G1.p[k], uh);
      stpos(&D.G2.p[k], make_double3(__dsub_rn(ua.x, uh.x), __dsub_rn(ua.y, uh.y), __dsub_rn(ua.z, uh.z)));
      u2 = __dadd_rn(__dadd_rn(__dmul_rn(uh.x, uh.x), __dmul_rn(uh.y, uh.y)), __dmul_rn(uh.z, uh.z));
    } else if (kind == SPHG_RIGID) {
      const sphg_body& b = B[D.group.p[k]];
      const double3 rk = qrotate(body_q(b), ld3(D.X4.p[k]));
      pn = make_double3(wrap1(P, __dadd_rn(b.com[0], rk.x), 0), wrap1(P, __dadd_rn(b.com[1], rk.y), 1),
                        wrap1(P, __dadd_rn(b.com[2], rk.z), 2));
      record_wrap(P, fl, wrap_list, (uint32_t)k, ldpos(&D.G0.p[k]), pn);
      stpos(&D.G0.p[k], pn);
      const double3 wxr = cross3(bv(b.omega), rk);
      stpos(&D.V4.p[k], make_double3(b.vel[0] + wxr.x, b.vel[1] + wxr.y, b.vel[2] + wxr.z));
    } else if (kind == SPHG_BOUNDARY && D.group.p[k] < (uint32_t)P.n_walls) {  // prescribed motion [P20]
      const uint32_t gr = D.group.p[k];
      const double3 p = ldpos(&D.G0.p[k]);
      pn = make_double3(wrap1(P, axpy_rn(p.x, P.dt, P.wall_vh[gr][0]), 0),
                        wrap1(P, axpy_rn(p.y, P.dt, P.wall_vh[gr][1]), 1),
                        wrap1(P, axpy_rn(p.z, P.dt, P.wall_vh[gr][2]), 2));
      record_wrap(P, fl, wrap_list, (uint32_t)k, p, pn);
      stpos(&D.G0.p[k], pn);
      stpos(&D.V4.p[k], make_double3(P.wall_v[gr][0], P.wall_v[gr][1], P.wall_v[gr][2]));
    } else {
      moved = false;
    }
    if (moved) {
      const double xs[3] = {pn.x, pn.y, pn.z};
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        if (!isfinite(xs[a])) {  // a blown-up state (SPEC:625 runtime assertion)
          atomicOr(&fl->err, kErrNaN);
          atomicMin(&fl->err_gid2, D.gid.p[k]);
        } else if (!P.periodic[a] && (xs[a] < P.lo[a] || xs[a] > P.hi[a])) {
          atomicOr(&fl->err, kErrEscape);
          atomicMin(&fl->err_gid, D.gid.p[k]);
        }
      }
      const double4 r0 = D.R4.p[k];
      disp2 = r2_exact(mimg3(P, pn.x, pn.y, pn.z, r0.x, r0.y, r0.z));
    }
  }
  // block-level max, one atomic per block (per-warp atomics on one address serialise in L2)
  __shared__ double s_d[8], s_u[8];
  disp2 = warp_max(disp2);
  u2 = warp_max(u2);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_d[w] = disp2;
    s_u[w] = u2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double d = s_d[0], u = s_u[0];
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
      d = fmax(d, s_d[k]);
      u = fmax(u, s_u[k]);
    }
    atomic_max_pos_double(&fl->max_disp2_bits, d);
    atomic_max_pos_double(&fl->umax2_bits, u);
  }
}

__global__ void k_body_final(const __grid_constant__ DevParams P, sphg_body* __restrict__ B, size_t nb) {
  SPHG_SKIP_IF_FLAGGED(P);
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
  SPHG_SKIP_IF_FLAGGED(P);
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const uint32_t kmd = D.kmd.p[k];
  if (is_ghost(kmd)) return;
  const uint32_t kind = kind_of(kmd);
  if (kind == SPHG_FLUID) {
    const double m = D.V4.p[k].w;
    if (P.n_buf) {  // role from x^{n+1} [P23]
      const double3 p = ldpos(&D.G0.p[k]);
      const int zb = buffer_of(P, p.x, p.y, p.z);
      if (zb >= 0) {
        const double3 u = buffer_velocity(P, zb, p.x, p.y, p.z, P.buf_new);
        D.V4.p[k] = make_double4(u.x, u.y, u.z, m);
        return;
      }
    }
    const double3 uh = ldpos(&D.G1.p[k]);
    const double4 a = D.A4.p[k];
    D.V4.p[k] = make_double4(axpy_rn(uh.x, P.hdt, a.x), axpy_rn(uh.y, P.hdt, a.y), axpy_rn(uh.z, P.hdt, a.z), m);
  } else if (kind == SPHG_RIGID) {
    const sphg_body& b = B[D.group.p[k]];
    const double3 rk = qrotate(body_q(b), ld3(D.X4.p[k]));
    const double3 wxr = cross3(bv(b.omega), rk);
    stpos(&D.V4.p[k], make_double3(b.vel[0] + wxr.x, b.vel[1] + wxr.y, b.vel[2] + wxr.z));
  }
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
// W = 1: a warp per body (many bodies).  W = 8: a block of 8 warps per body for small body tables
// (C1: 4 bodies of ~280 particles), whose reduction is otherwise one serial chain per body; the 8
// warp partials are merged in warp order in shared memory (compensated, deterministic).
template <int W>
__global__ void __launch_bounds__(W == 1 ? 128 : 32 * W) k_body_reduce(const __grid_constant__ DevParams P, Particles D,
                                                      sphg_body* __restrict__ B, size_t nb,
                                                      const uint32_t* __restrict__ ridx,
                                                      const uint32_t* __restrict__ bstart,
                                                      const uint32_t* __restrict__ bend) {
  SPHG_SKIP_IF_FLAGGED(P);
  const size_t k = W == 1 ? ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5 : (size_t)blockIdx.x;
  const int lane = threadIdx.x & 31, warp = W == 1 ? 0 : (int)(threadIdx.x >> 5);
  if (k >= nb) return;
  sphg_body& b = B[k];
  if (!b.alive) return;
  const Quat q = body_q(b);
  KSum acc[12];
#pragma unroll
  for (int c = 0; c < 12; ++c) acc[c] = {0.0, 0.0};
  const uint32_t s0 = bstart[k], s1 = bend[k];
  for (uint32_t s = s0 + warp * 32 + lane; s < s1; s += 32 * W) {
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
  if (W == 1) {
#pragma unroll
    for (int c = 0; c < 12; ++c) v[c] = warp_merge(acc[c]).value();
    if (lane != 0) return;
  } else {
    __shared__ double part[W][12][2];
#pragma unroll
    for (int c = 0; c < 12; ++c) {
      const KSum m = warp_merge(acc[c]);
      if (lane == 0) {
        part[warp][c][0] = m.s;
        part[warp][c][1] = m.c;
      }
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    for (int c = 0; c < 12; ++c) {
      KSum m = {part[0][c][0], part[0][c][1]};
      for (int w = 1; w < W; ++w) m.merge(part[w][c][0], part[w][c][1]);
      v[c] = m.value();
    }
  }
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
  if (cur.C2.p) {
    cur.C2.p[k] = src.C2.p[g];
    cur.dCdt.p[k] = src.dCdt.p[g];
  }
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

// ------------------------------------------------ decomposition primitives
__global__ void k_idx_of_gid(const uint32_t* __restrict__ gid, size_t n, uint32_t* __restrict__ idx) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) idx[gid[k]] = (uint32_t)k;
}

// halo record layouts (sphg.h SPHG_HALO_*)
__global__ void k_halo_pack(Particles D, int phase, const uint32_t* __restrict__ ids, size_t m,
                            const uint32_t* __restrict__ idx, double* __restrict__ buf) {
  const size_t s = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= m) return;
  const uint32_t k = idx[ids[s]];
  if (phase == SPHG_HALO_STATE) {
    const double4 g0 = D.G0.p[k], g1 = D.G1.p[k], g2 = D.G2.p[k], v = D.V4.p[k];
    double* o = buf + s * 14;
    o[0] = g0.x; o[1] = g0.y; o[2] = g0.z;
    o[3] = g1.x; o[4] = g1.y; o[5] = g1.z;
    o[6] = g2.x; o[7] = g2.y; o[8] = g2.z;
    o[9] = v.x; o[10] = v.y; o[11] = v.z;
    o[12] = D.H2.p[k].x;
    o[13] = D.C2.p ? D.C2.p[k].x : 0.0;
  } else if (phase == SPHG_HALO_DENSITY) {
    double* o = buf + s * 4;
    o[0] = D.G0.p[k].w; o[1] = D.G1.p[k].w; o[2] = D.G2.p[k].w; o[3] = D.H2.p[k].y;
  } else {
    const double4 g1 = D.G1.p[k];
    double* o = buf + s * 6;
    o[0] = D.G0.p[k].w; o[1] = g1.x; o[2] = g1.y; o[3] = g1.z; o[4] = g1.w; o[5] = D.G2.p[k].w;
  }
}

// continuous (the Verlet rows are valid): a ghost whose owner moved it across a periodic face keeps
// coordinates continuous with the ones its image-coded entries were built for (unwrapped by one period);
// launch_rebuild wraps ghosts back before binning
__global__ void k_halo_unpack(const __grid_constant__ DevParams P, Particles D, int phase,
                              const uint32_t* __restrict__ ids, size_t m, const uint32_t* __restrict__ idx,
                              const double* __restrict__ buf, int continuous) {
  const size_t s = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= m) return;
  const uint32_t k = idx[ids[s]];
  double* g0 = reinterpret_cast<double*>(&D.G0.p[k]);
  double* g1 = reinterpret_cast<double*>(&D.G1.p[k]);
  double* g2 = reinterpret_cast<double*>(&D.G2.p[k]);
  if (phase == SPHG_HALO_STATE) {
    const double* o = buf + s * 14;
    double x[3] = {o[0], o[1], o[2]};
    if (continuous) {
#pragma unroll
      for (int a = 0; a < 3; ++a)
        if (P.periodic[a]) {
          const double d = x[a] - g0[a];
          if (d > P.halfL[a]) x[a] -= P.L[a];
          else if (d < -P.halfL[a]) x[a] += P.L[a];
        }
    }
    g0[0] = x[0]; g0[1] = x[1]; g0[2] = x[2];
    g1[0] = o[3]; g1[1] = o[4]; g1[2] = o[5];
    g2[0] = o[6]; g2[1] = o[7]; g2[2] = o[8];
    double* v = reinterpret_cast<double*>(&D.V4.p[k]);
    v[0] = o[9]; v[1] = o[10]; v[2] = o[11];
    reinterpret_cast<double*>(&D.H2.p[k])[0] = o[12];
    if (D.C2.p) reinterpret_cast<double*>(&D.C2.p[k])[0] = o[13];
  } else if (phase == SPHG_HALO_DENSITY) {
    const double* o = buf + s * 4;
    g0[3] = o[0]; g1[3] = o[1]; g2[3] = o[2];
    reinterpret_cast<double*>(&D.H2.p[k])[1] = o[3];
    // fluid diffusion volume m/rho, the same division the owner did (k_density)
    if (D.C2.p && kind_of(D.kmd.p[k]) == SPHG_FLUID) reinterpret_cast<double*>(&D.C2.p[k])[1] = D.V4.p[k].w / o[1];
  } else {
    const double* o = buf + s * 6;
    g0[3] = o[0]; g1[0] = o[1]; g1[1] = o[2]; g1[2] = o[3]; g1[3] = o[4]; g2[3] = o[5];
  }
}

// per-body compensated partials over owned members: out[k*24 + 2c] = sum, +1 = compensation
__global__ void __launch_bounds__(128) k_body_partials(const __grid_constant__ DevParams P, Particles D,
                                                        const sphg_body* __restrict__ B, size_t nb,
                                                        const uint32_t* __restrict__ ridx,
                                                        const uint32_t* __restrict__ bstart,
                                                        const uint32_t* __restrict__ bend, double* __restrict__ out) {
  const size_t k = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (k >= nb) return;
  const sphg_body& b = B[k];
  const Quat q = body_q(b);
  KSum acc[12];
#pragma unroll
  for (int c = 0; c < 12; ++c) acc[c] = {0.0, 0.0};
  if (b.alive) {
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
  }
#pragma unroll
  for (int c = 0; c < 12; ++c) {
    const KSum v = warp_merge(acc[c]);
    if (lane == 0) {
      out[k * 24 + 2 * c] = v.s;
      out[k * 24 + 2 * c + 1] = v.c;
    }
  }
}

__global__ void k_apply_totals(const __grid_constant__ DevParams P, sphg_body* __restrict__ B, size_t nb,
                               const double* __restrict__ tot) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nb) return;
  sphg_body& b = B[k];
  if (!b.alive) return;
  const double* v = tot + k * 12;
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

// Periodic-face crossings since the rebuild (record_wrap, common.cuh): phase 1 shifts the codes of the
// crossing particle's own row, phase 2 those of the entries of its neighbours' rows that reference it
// (the candidate lists are symmetric).  Warp per crossing particle, grid-stride over the device-side count
// so the launch is graph-capturable.  Two launches: every entry is then changed by exactly one warp per
// phase and the two shifts (x_i's and x_j's) add up.
__global__ void k_wrap_patch_own(const uint32_t* __restrict__ list, const DevFlags* __restrict__ fl, NbrList L) {
  const int lane = threadIdx.x & 31;
  const uint32_t m = fl->n_wrapped;
  for (uint32_t e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < m; e += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t i = list[2 * e], w = list[2 * e + 1];
    uint32_t* row = const_cast<uint32_t*>(L.nbr) + (size_t)i * L.cap;
    const uint32_t nn = cnt_total(L.cnt[i]);
    for (uint32_t k = lane; k < nn; k += 32) {
      const uint32_t en = row[k];
      row[k] = (en & kIdxMask) | (shift_code(en >> kIdxBits, w, +1) << kIdxBits);
    }
  }
}

__global__ void k_wrap_patch_peer(const uint32_t* __restrict__ list, const DevFlags* __restrict__ fl, NbrList L) {
  const int lane = threadIdx.x & 31;
  const uint32_t m = fl->n_wrapped;
  for (uint32_t e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < m; e += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t i = list[2 * e], w = list[2 * e + 1];
    const uint32_t* rowi = L.nbr + (size_t)i * L.cap;
    const uint32_t ni = cnt_total(L.cnt[i]);
    for (uint32_t q = 0; q < ni; ++q) {
      const uint32_t j = rowi[q] & kIdxMask;
      uint32_t* rowj = const_cast<uint32_t*>(L.nbr) + (size_t)j * L.cap;
      const uint32_t nj = cnt_total(L.cnt[j]);
      for (uint32_t k = lane; k < nj; k += 32) {
        const uint32_t en = rowj[k];
        if ((en & kIdxMask) == i) rowj[k] = i | (shift_code(en >> kIdxBits, w, -1) << kIdxBits);
      }
    }
  }
}

// global body totals from the ranks' compensated partials, merged in rank order with TwoSum (the same
// single IEEE adds as parallel._merge_partials, so every rank gets bit-identical totals)
__global__ void k_merge_partials(const double* __restrict__ g, size_t nb, int world, double* __restrict__ tot) {
  const size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x;  // (body, component)
  if (q >= nb * 12) return;
  double s = g[2 * q], c = g[2 * q + 1];
  for (int r = 1; r < world; ++r) {
    const double s2 = g[(size_t)r * nb * 24 + 2 * q], c2 = g[(size_t)r * nb * 24 + 2 * q + 1];
    const double t = __dadd_rn(s, s2);
    const double bp = __dsub_rn(t, s);
    const double e = __dadd_rn(__dsub_rn(s, __dsub_rn(t, bp)), __dsub_rn(s2, bp));
    c = __dadd_rn(__dadd_rn(c, c2), e);
    s = t;
  }
  tot[q] = __dadd_rn(s, c);
}

__global__ void k_scatter_state(const __grid_constant__ DevParams P, Particles D, size_t n,
                                const uint32_t* __restrict__ idx, const double* __restrict__ pos,
                                const double* __restrict__ vel, DevFlags* __restrict__ fl, uint32_t* __restrict__ wl) {
  const size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
  const uint32_t k = idx[g];
  if (pos) {
    const double3 pn = make_double3(pos[3 * g], pos[3 * g + 1], pos[3 * g + 2]);
    record_wrap(P, fl, wl, k, ldpos(&D.G0.p[k]), pn);
    stpos(&D.G0.p[k], pn);
  }
  if (vel) stpos(&D.V4.p[k], make_double3(vel[3 * g], vel[3 * g + 1], vel[3 * g + 2]));
}

}  // namespace

void scatter_state(Ctx& c, const double* pos, const double* vel) {
  SPHG_CUDA_CHECK(cudaMemsetAsync(&c.dflags->n_wrapped, 0, sizeof(uint32_t), c.stream));
  uint32_t* wl = c.P.img_mode == kImgCode && c.built ? c.wrap_list.p : nullptr;
  k_scatter_state<<<grid_for(c.n, 256), 256, 0, c.stream>>>(c.P, c.cur, c.n, c.idx_of_gid.p, pos, vel, c.dflags, wl);
  c.launches++;
  launch_wrap_patch(c);
}

void build_idx_of_gid(Ctx& c) {
  if (c.n == 0) return;
  c.idx_of_gid.alloc(c.n);
  k_idx_of_gid<<<grid_for(c.n, 256), 256, 0, c.stream>>>(c.cur.gid.p, c.n, c.idx_of_gid.p);
  c.launches++;
}

void halo_pack(Ctx& c, int phase, int slot, double* buf) {
  const size_t m = c.halo_n[slot];
  if (m == 0) return;
  k_halo_pack<<<grid_for(m, 256), 256, 0, c.stream>>>(c.cur, phase, c.halo_ids[slot].p, m, c.idx_of_gid.p, buf);
  c.launches++;
}

void halo_unpack(Ctx& c, int phase, int slot, const double* buf) {
  const size_t m = c.halo_n[slot];
  if (m == 0) return;
  const int continuous = c.built && c.P.img_mode == kImgCode ? 1 : 0;
  k_halo_unpack<<<grid_for(m, 256), 256, 0, c.stream>>>(c.P, c.cur, phase, c.halo_ids[slot].p, m, c.idx_of_gid.p, buf,
                                                        continuous);
  c.launches++;
}

namespace {
__global__ void k_wrap_ghosts(const __grid_constant__ DevParams P, Particles D, size_t n) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n || !is_ghost(D.kmd.p[k])) return;
  const double3 p = ldpos(&D.G0.p[k]);
  stpos(&D.G0.p[k], make_double3(wrap1(P, p.x, 0), wrap1(P, p.y, 1), wrap1(P, p.z, 2)));
}
}  // namespace

void wrap_ghosts(Ctx& c) {  // before binning: ghosts kept continuous across periodic faces (k_halo_unpack)
  if (c.nghost == 0 || c.P.img_mode != kImgCode) return;
  k_wrap_ghosts<<<grid_for(c.n, 256), 256, 0, c.stream>>>(c.P, c.cur, c.n);
  c.launches++;
}

void body_partials(Ctx& c, double* dev_out) {
  if (c.nb == 0) return;
  k_body_partials<<<grid_for(c.nb * 32, 128), 128, 0, c.stream>>>(c.P, c.cur, c.bodies.p, c.nb, c.ridx.p,
                                                                   c.body_start.p, c.body_start.p + c.nb, dev_out);
  c.launches++;
}

void merge_body_partials(Ctx& c, const double* gathered, int world, double* totals) {
  if (c.nb == 0) return;
  k_merge_partials<<<grid_for(c.nb * 12, 128), 128, 0, c.stream>>>(gathered, c.nb, world, totals);
  c.launches++;
}

void body_apply_totals(Ctx& c, const double* dev_tot) {
  if (c.nb == 0) return;
  k_apply_totals<<<grid_for(c.nb, 128), 128, 0, c.stream>>>(c.P, c.bodies.p, c.nb, dev_tot);
  c.launches++;
}

void gather_by_gid(Ctx& c) {
  if (c.n == 0) return;
  k_gather_by_gid<<<grid_for(c.n, 256), 256, 0, c.stream>>>(c.cur, c.alt, c.n);
  c.launches++;
}

bool displacement_exceeds(Ctx& c) {
  if (c.n == 0) return false;
  SPHG_CUDA_CHECK(cudaMemsetAsync(&c.dflags->max_disp2_bits, 0, 8, c.stream));
  k_disp<<<grid_for(c.n, 256), 256, 0, c.stream>>>(c.P, c.cur, c.n, c.dflags);
  unsigned long long b = 0;
  SPHG_CUDA_CHECK(cudaMemcpyAsync(&b, &c.dflags->max_disp2_bits, 8, cudaMemcpyDeviceToHost, c.stream));
  host_sync(c, c.stream);
  double d2;
  memcpy(&d2, &b, 8);
  c.launches += 2;
  return std::sqrt(d2) > c.P.half_skin;
}

void iota_gid(Ctx& c) {
  if (c.n == 0) return;
  k_iota<<<grid_for(c.n, 256), 256, 0, c.stream>>>(c.cur.gid.p, c.n);
  c.launches++;
}

// ============================================================= launchers
void launch_body_kick(Ctx& c) {
  if (c.nb == 0) return;
  k_body_kick<<<grid_for(c.nb, 128), 128, 0, c.stream>>>(c.P, c.bodies.p, c.nb);
  c.launches++;
}

// end of the kick chain: flag the force chain to void itself when the Verlet trigger fired (max
// displacement > half skin, compared as the host does: sqrt of the squared maximum) or an error is
// pending, and advance the device clock: dtime[1] mirrors the host's c.t (c.t += dt), dtime[0] is the
// time the captured force chain reads (the host's c.t + dt after the increment), same double adds
__global__ void k_step_tail(const __grid_constant__ DevParams P, const DevFlags* __restrict__ fl,
                            uint32_t* __restrict__ skip, double* __restrict__ dtime) {
  const double md = sqrt(__longlong_as_double((long long)fl->max_disp2_bits));
  *skip = (md > P.half_skin || fl->err != 0u) ? 1u : 0u;
  if (dtime) {
    const double t = dtime[1] + P.dt;
    dtime[1] = t;
    dtime[0] = t + P.dt;
  }
}

void launch_step_tail(Ctx& c) {
  k_step_tail<<<1, 1, 0, c.stream>>>(c.P, c.dflags, c.dskip, c.dtime);
  c.launches++;
}

void launch_wrap_patch(Ctx& c) {
  if (c.P.img_mode != kImgCode || !c.built || c.n == 0) return;
  k_wrap_patch_own<<<64, 256, 0, c.stream>>>(c.wrap_list.p, c.dflags, c.nl());
  k_wrap_patch_peer<<<64, 256, 0, c.stream>>>(c.wrap_list.p, c.dflags, c.nl());
  c.launches += 2;
}

void launch_kick_drift(Ctx& c) {
  if (c.n == 0) return;
  SPHG_CUDA_CHECK(cudaMemsetAsync(&c.dflags->n_wrapped, 0, sizeof(uint32_t), c.stream));
  uint32_t* wl = c.P.img_mode == kImgCode && c.built ? c.wrap_list.p : nullptr;
  if (c.final_pending)  // the previous step deferred its particle final kick into this pass
    k_kick_drift<true><<<grid_for(c.n, 256), 256, 0, c.stream>>>(c.P, c.cur, c.bodies.p, c.n, c.dflags, wl);
  else
    k_kick_drift<false><<<grid_for(c.n, 256), 256, 0, c.stream>>>(c.P, c.cur, c.bodies.p, c.n, c.dflags, wl);
  c.final_pending = false;
  c.launches++;
  launch_wrap_patch(c);  // rows stay valid across periodic faces until the next rebuild
}

void launch_bodies(Ctx& c) {
  if (c.nb == 0) return;
  if (c.nb < 148)  // fewer bodies than SMs: a block of 8 warps per body
    k_body_reduce<8><<<(unsigned)c.nb, 256, 0, c.stream>>>(c.P, c.cur, c.bodies.p, c.nb, c.ridx.p, c.body_start.p,
                                                          c.body_start.p + c.nb);
  else
    k_body_reduce<1><<<grid_for(c.nb * 32, 128), 128, 0, c.stream>>>(c.P, c.cur, c.bodies.p, c.nb, c.ridx.p,
                                                                    c.body_start.p, c.body_start.p + c.nb);
  c.launches++;
}

void launch_final_kick(Ctx& c) {
  if (c.n == 0) return;
  if (c.nb) k_body_final<<<grid_for(c.nb, 128), 128, 0, c.stream>>>(c.P, c.bodies.p, c.nb);
  if (c.defer_final) {  // next step's kick-drift applies it (fluid); rigid end velocities are overwritten there
    c.final_pending = true;
    c.launches += c.nb ? 1 : 0;
    return;
  }
  k_final_kick<<<grid_for(c.n, 256), 256, 0, c.stream>>>(c.P, c.cur, c.bodies.p, c.n);
  c.launches += c.nb ? 2 : 1;
}

void launch_final_kick_particles(Ctx& c) {  // the deferred particle part alone
  if (c.n == 0) return;
  k_final_kick<<<grid_for(c.n, 256), 256, 0, c.stream>>>(c.P, c.cur, c.bodies.p, c.n);
  c.final_pending = false;
  c.launches++;
}

void launch_mass(Ctx& c, const uint32_t* mask) {
  if (c.nb == 0) return;
  k_mass<<<grid_for(c.nb * 32, 128), 128, 0, c.stream>>>(c.P, c.cur, c.bodies.p, c.nb, c.ridx.p, c.body_start.p,
                                                         c.body_start.p + c.nb, mask);
  c.launches++;
}

}  // namespace sphg
