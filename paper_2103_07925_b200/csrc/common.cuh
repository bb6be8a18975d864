// common.cuh — device-side parameters and math shared by all sm_100a kernels.
//
// Pinned arithmetic is mirrored from the CPU oracle so that the
// bit-exact stages (cell keys, Verlet candidate tests, minimum image, periodic
// wrap, kick/drift) produce identical doubles: those use explicit
// round-to-nearest intrinsics (__dadd_rn/__dmul_rn/__dsub_rn), which ptxas
// never contracts into FMA.  The tolerance stages (pair sums) use FMA freely.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/sphg.h"

namespace sphg {

constexpr int kMaxMat = SPHG_MAX_MAT;

struct DevMat {
  double rho0, eta, cp, kappa, c2, pb, T_t;
  double g[3];
  double p0;           // rho0 c^2
  double inv_c2;       // 1/c^2 (0 when c == 0)
  double D, C_t;       // diffusivity, transition concentration
  int32_t melt, solid;
  int32_t has_Tt, has_Ct;
};

struct DevSchedule {
  int32_t n, pad;
  double t_end[SPHG_MAX_PIECES];
  double value[SPHG_MAX_PIECES];
};

struct DevParams {
  DevMat mat[kMaxMat];
  DevSchedule sched[SPHG_MAX_DIRICHLET];
  DevSchedule schedC[SPHG_MAX_DIRICHLET];  // concentration Dirichlet groups (config.hpp:95)
  double lo[3], hi[3], L[3], halfL[3], inv_edge[3];
  int32_t ncell[3];
  int32_t periodic[3];
  int32_t n_mat, n_sched, n_schedC, diffusion;
  double h, inv_h, rc, rc2, rv, rv2, sigma, sig_h, w0;
  double dx2_hi;  // dx^2 (1 + 1e-12): contact candidates beyond it are apart without the exact test
  double rc2_lo, rc2_ulp, rc2_hi;  // rc^2 (1 - 2e-4), rc^2 (1 - 1e-12), rc^2 (1 + 1e-12): pinned_q's bands
  double dx, dx3, dt, hdt;
  double kc, dc;
  double half_skin;
  double Ir_over_m;     // particle inertia / mass
  int32_t tvf, thermal, transitions, default_fluid_mat;
  int32_t single_eta;   // all fluid materials share eta   -> eta~ = eta_i
  double eta_single;    // that shared eta (read from the parameter bank instead of a register per thread)
  int32_t single_kappa; // all materials share kappa       -> kappa~ = 2 kappa
  int32_t single_eos;   // all fluid materials share rho0,c -> wall EOS material fixed
  int32_t img_mode;     // neighbour-entry image mode (kImgNone / kImgCode / kImgMin)
  int32_t single_g;     // every fluid-capable material has default_fluid_mat's body force
  // moving wall groups (sphg_set_wall_motion), refreshed by the host before every kick [P20]:
  // velocity at t^{n+1/2} (drift), velocity and acceleration at t^{n+1} (wall state)
  int32_t n_walls, pad_w;
  double wall_vh[SPHG_MAX_WALL_GROUPS][3], wall_v[SPHG_MAX_WALL_GROUPS][3], wall_a[SPHG_MAX_WALL_GROUPS][3];
  // moving Gaussian surface heat flux [P21] (sphg.h): source rate per particle (storage order) in hsrc,
  // written by k_heat_source before the conduction kernels read it in their epilogues
  int32_t heat_source;
  uint32_t hs_mask;
  double hs_q0;                    // 2 P / (pi r0^2)
  double hs_r0sq, hs_cut2;         // r0^2, (4 r0)^2
  double hs_origin[2], hs_vel[2];
  double hs_dz, hs_lat2;           // dx/2, (3 dx/4)^2
  double* hsrc;
  // speculative step (api.cu one_step): set on the device by the tail of the kick chain when the step
  // needs a Verlet rebuild (or hit an error); every kernel of the force chain then returns at once
  const uint32_t* skip;
  // inflow / outflow buffer zones [P23] (sphg_buffer); bit b of buf_half / buf_new / buf_prev: zone b
  // prescribes its velocity at t^{n+1/2} / t^{n+1} / t^n (t > t_start), set by the host every kick
  struct Buf {
    int32_t axis, paxis;
    double lo[3], hi[3], u_mean;
  } buf[SPHG_MAX_BUFFERS];
  int32_t n_buf;
  uint32_t buf_half, buf_new, buf_prev;
};
#define SPHG_SKIP_IF_FLAGGED(P) \
  do {                          \
    if ((P).skip && *(P).skip)  \
      return;                   \
  } while (0)

// ------------------------------------------------------ brick traversal
// Work order of the cell-structured kernels (Verlet build, pair kernels): cells are visited brick
// by brick (kBrick^3 cells, bricks z-fastest; inside a brick 2x2x2 blocks of cells, z-fastest).  Storage stays in the pinned
// z-fastest (cell, gid) order [P1]; only the order in which cells / particles are PROCESSED
// changes, so the neighbourhood of the cells in flight (~(kBrick+2)^3 cells) stays in L2 instead
// of three whole x-planes of the grid.
constexpr int kBrick = 8;
__host__ __device__ __forceinline__ int64_t brick_positions(const int32_t* nc) {
  const int64_t bx = (nc[0] + kBrick - 1) / kBrick, by = (nc[1] + kBrick - 1) / kBrick,
                bz = (nc[2] + kBrick - 1) / kBrick;
  return bx * by * bz * (int64_t)(kBrick * kBrick * kBrick);
}
// linear cell id of brick position b, or -1 for padding positions past the grid edge
__host__ __device__ __forceinline__ int64_t brick_to_cell(const int32_t* nc, int64_t b) {
  constexpr int64_t B3 = kBrick * kBrick * kBrick;
  const int64_t nby = (nc[1] + kBrick - 1) / kBrick, nbz = (nc[2] + kBrick - 1) / kBrick;
  const int64_t brick = b / B3, loc = b % B3;
  const int64_t bz = brick % nbz, by = (brick / nbz) % nby, bx = brick / (nbz * nby);
#ifndef SPHG_BRICK_ZLINE
  // 2x2x2 blocks of cells inside the brick (blocks and the cells of a block z-fastest): the ~8 cells whose
  // particles are in flight on one SM (SM-local pair kernels) share a 4x4x4-cell neighbourhood instead of
  // the 3x3x10 cells of a z-line
  constexpr int64_t H = kBrick / 2;
  const int64_t blk = loc >> 3, in = loc & 7;
  const int64_t lz = 2 * (blk % H) + (in & 1), ly = 2 * ((blk / H) % H) + ((in >> 1) & 1),
                lx = 2 * (blk / (H * H)) + (in >> 2);
#else
  const int64_t lz = loc % kBrick, ly = (loc / kBrick) % kBrick, lx = loc / (kBrick * kBrick);
#endif
  const int64_t cx = bx * kBrick + lx, cy = by * kBrick + ly, cz = bz * kBrick + lz;
  if (cx >= nc[0] || cy >= nc[1] || cz >= nc[2]) return -1;
  return (cx * nc[1] + cy) * nc[2] + cz;
}

// ------------------------------------------------ SM-local tile queues
// Work distribution of the persistent (SM-local) kernels: a list of ntiles tiles is cut into nq contiguous
// ranges, one per SM (%smid), each with a counter in next[] (zeroed before the launch); see kernels_pairs.cu.
__device__ __forceinline__ unsigned sm_id() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
// A range with tiles left, searched from q + 1 on, or -1: the 32 lanes probe 32 counters at a time (L2 reads:
// a counter only grows, so a stale value can only show work that is already gone, which the caller's atomic
// then finds out).  Out of line: the steal path must not shape the register allocation of the pair loops.
static __device__ __noinline__ int find_range(const uint32_t* next, int nq, size_t ntiles, int q) {
  const int lw = threadIdx.x & 31;
  for (int base = 1; base < nq; base += 32) {
    bool has = false;
    if (base + lw < nq) {
      const int qq = (q + base + lw) % nq;
      const size_t a0 = ntiles * (size_t)qq / nq, a1 = ntiles * (size_t)(qq + 1) / nq;
      has = a0 + __ldcg(&next[qq]) < a1;
    }
    const unsigned m = __ballot_sync(0xffffffffu, has);
    if (m) return (q + base + __ffs((int)m) - 1) % nq;
  }
  return -1;
}
// the next tile (32 list slots' worth of lanes) for this warp, or false when every range is finished: the
// current range first (the SM's own until it is exhausted), then the nearest following range with work
__device__ __forceinline__ bool next_tile(uint32_t* __restrict__ next, int nq, size_t ntiles, int& q, size_t& tile) {
  for (;;) {
    const size_t q0 = ntiles * (size_t)q / nq, q1 = ntiles * (size_t)(q + 1) / nq;
    uint32_t t = 0;
    if ((threadIdx.x & 31) == 0) t = atomicAdd(&next[q], 1u);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (q0 + t < q1) {
      tile = q0 + t;
      return true;
    }
    const int f = find_range(next, nq, ntiles, q);
    if (f < 0) return false;
    q = f;
  }
}

// ---------------------------------------------------------------- tags
// kmd word: bits 0-1 kind, 2-7 material, 8-15 temperature Dirichlet group, 16 ghost,
// 24-31 concentration Dirichlet group (0xff none for both groups)
__host__ __device__ __forceinline__ uint32_t kind_of(uint32_t kmd) { return kmd & 3u; }
__host__ __device__ __forceinline__ uint32_t mat_of(uint32_t kmd) { return (kmd >> 2) & 63u; }
__host__ __device__ __forceinline__ uint32_t dir_of(uint32_t kmd) { return (kmd >> 8) & 255u; }
__host__ __device__ __forceinline__ uint32_t dirc_of(uint32_t kmd) { return kmd >> 24; }
__host__ __device__ __forceinline__ uint32_t make_kmd(uint32_t kind, uint32_t mat, uint32_t dir,
                                                      uint32_t dirc = 0xffu) {
  return (kind & 3u) | ((mat & 63u) << 2) | ((dir & 255u) << 8) | ((dirc & 255u) << 24);
}
// bit 16: ghost copy of a particle owned by another rank (read-only here, refreshed by halos)
constexpr uint32_t kGhostBit = 1u << 16;
__host__ __device__ __forceinline__ bool is_ghost(uint32_t kmd) { return (kmd & kGhostBit) != 0u; }

// ------------------------------------------------- pinned (no-FMA) helpers
// minimum image along one axis [P2]
__device__ __forceinline__ double mimg(const DevParams& P, double d, int a) {
  if (P.periodic[a]) {
    if (d > P.halfL[a]) d = __dsub_rn(d, P.L[a]);
    else if (d < -P.halfL[a]) d = __dadd_rn(d, P.L[a]);
  }
  return d;
}
__device__ __forceinline__ double3 mimg3(const DevParams& P, double ax, double ay, double az, double bx, double by,
                                         double bz) {
  return make_double3(mimg(P, __dsub_rn(ax, bx), 0), mimg(P, __dsub_rn(ay, by), 1), mimg(P, __dsub_rn(az, bz), 2));
}
// (dx*dx + dy*dy) + dz*dz without contraction [P2]
__device__ __forceinline__ double r2_exact(double3 d) {
  return __dadd_rn(__dadd_rn(__dmul_rn(d.x, d.x), __dmul_rn(d.y, d.y)), __dmul_rn(d.z, d.z));
}
// periodic wrap, one conditional shift [P14]
__device__ __forceinline__ double wrap1(const DevParams& P, double x, int a) {
  if (P.periodic[a]) {
    if (x < P.lo[a]) x = __dadd_rn(x, P.L[a]);
    else if (x >= P.hi[a]) x = __dsub_rn(x, P.L[a]);
  }
  return x;
}
// a + s*b with explicit rounding (matches Vec operator+ / operator* in the oracle)
__device__ __forceinline__ double axpy_rn(double a, double s, double b) { return __dadd_rn(a, __dmul_rn(s, b)); }

// ---------------------------------------------------------- kernel (fp64)
// Quintic spline (kernel.hpp:47-75), branch-free: the missing branches add exact zeros.
// max(x, 0) on the integer pipe (keeps DSETP/FSEL off the FP64 pipe; x is never NaN here)
__device__ __forceinline__ double clamp0(double x) {
  const long long b = __double_as_longlong(x);
  return __longlong_as_double(b & ~(b >> 63));
}
__device__ __forceinline__ double shape_q(double q) {
  const double a = 3.0 - q;
  const double b = clamp0(2.0 - q);
  const double c = clamp0(1.0 - q);
  const double a2 = a * a, b2 = b * b, c2 = c * c;
  return a2 * a2 * a - 6.0 * (b2 * b2 * b) + 15.0 * (c2 * c2 * c);
}
__device__ __forceinline__ double shape_deriv_q(double q) {
  const double a = 3.0 - q;
  const double b = clamp0(2.0 - q);
  const double c = clamp0(1.0 - q);
  const double a2 = a * a, b2 = b * b, c2 = c * c;
  return -5.0 * (a2 * a2) + 30.0 * (b2 * b2) - 75.0 * (c2 * c2);
}

// fast fp64 reciprocal / reciprocal square root for the tolerance stages:
// MUFU seed (~2^-22) + one Newton step (~1e-13 relative, far inside the 1e-10
// bar of the pair sums); 2 + 4 FP64 instructions instead of the IEEE sequences.
__device__ __forceinline__ double rcp_fast(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y, 1.0);
  return fma(y, e, y);
}
__device__ __forceinline__ double rsqrt_fast(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = x * y;
  const double e = fma(-h, y, 1.0);  // 1 - x y^2
  return fma(0.5 * y, e, y);
}
// r = sqrt(x) to ~0.5 ulp and 1/r to ~1e-11 (x > 0).  The kernel argument q =
// r/h needs the accurate root: W ~ (3-q)^5 amplifies relative errors of q near
// the cut-off, and wall extrapolation divides by sums of such weights.
__device__ __forceinline__ double sqrt_and_rinv(double x, double& rinv) {
  const double y = rsqrt_fast(x);
  const double r0 = x * y;
  const double e = fma(-r0, r0, x);
  rinv = y;
  return fma(0.5 * y, e, r0);
}

// q = r/h and 1/r of a pair with offset d and r^2 = d.d (r2, FMA allowed) inside r_c.  SPHG_EXACT_Q:
// the oracle's q bit for bit (no-FMA r^2, correctly rounded root, q = r * (1/h)) in every pair kernel.
__device__ __forceinline__ double pair_qr(double3 d, double r2, double inv_h, double& rinv) {
#ifdef SPHG_EXACT_Q
  const double r2e = __dadd_rn(__dadd_rn(__dmul_rn(d.x, d.x), __dmul_rn(d.y, d.y)), __dmul_rn(d.z, d.z));
  rinv = rsqrt_fast(r2e);
  return __dmul_rn(__dsqrt_rn(r2e), inv_h);
#else
  return sqrt_and_rinv(r2 + 1e-300, rinv) * inv_h;
#endif
}

// Near the cut-off the kernel is ill-conditioned: dW ~ (3-q)^4 and W ~ (3-q)^5 turn a last-bit
// difference of q into a relative error ~12/(3-q) larger.  That decides the result only where ALL of a
// particle's pairs sit in a band just below r_c (one pair further inside dominates every band term
// by (3-q)^4): a rigid particle three layers deep, a wall behind an exact lattice, a Shepard ratio
// whose lone weight is tiny instead of 0.  For those particles the sums are redone with the oracle's
// arithmetic: no-FMA r^2, correctly rounded root, q = r * (1/h) (kernel.hpp:30, 36), zero kernel for
// q >= 3 (kernel.hpp:49, 63).  The hot kernels take the fast root and flag such particles; a second
// launch of the same kernel (kPin) redoes only the flagged ones, so the pinned arithmetic costs the
// hot loop no registers.
__device__ __forceinline__ double pinned_q(double3 d, double rc2, double inv_h, double& rinv) {
  const double r2e = __dadd_rn(__dadd_rn(__dmul_rn(d.x, d.x), __dmul_rn(d.y, d.y)), __dmul_rn(d.z, d.z));
  const double r = __dsqrt_rn(r2e);
  rinv = 1.0 / r;
  return r2e > rc2 ? 3.0 : __dmul_rn(r, inv_h);
}
// Shepard weight shape W/sigma of a pair at offset d, or false outside r_c (grid gather: not hot, so
// pairs within a few ulps of r_c take pinned_q inline)
template <class DP>
__device__ __forceinline__ bool shepard_shape(const DP& P, double3 d, double r2, double& W) {
  if (r2 > P.rc2_hi) return false;
  double ri;
  const double q = r2 >= P.rc2_ulp ? pinned_q(d, P.rc2, P.inv_h, ri) : sqrt_and_rinv(r2 + 1e-300, ri) * P.inv_h;
  W = q >= 3.0 ? 0.0 : shape_q(q);
  return true;
}

// ------------------------------------------------------- buffer zones [P23]
// zone of a fluid particle at x (first zone whose box holds it), -1 outside every zone
__device__ __forceinline__ int buffer_of(const DevParams& P, double x, double y, double z) {
  for (int b = 0; b < P.n_buf; ++b) {
    const DevParams::Buf& B = P.buf[b];
    if (x >= B.lo[0] && x < B.hi[0] && y >= B.lo[1] && y < B.hi[1] && z >= B.lo[2] && z < B.hi[2]) return b;
  }
  return -1;
}
// prescribed velocity U(x) of zone b (pinned arithmetic: the drift is a bit-exact stage), 0 when the
// zone is not active at the time the caller's mask describes
__device__ __forceinline__ double3 buffer_velocity(const DevParams& P, int b, double x, double y, double z,
                                                   uint32_t active) {
  const DevParams::Buf& B = P.buf[b];
  double u = 0.0;
  if ((active >> b) & 1u) {
    double f = 1.0;
    if (B.paxis >= 0) {
      const double xp = B.paxis == 0 ? x : (B.paxis == 1 ? y : z);
      const double xi = __ddiv_rn(__dsub_rn(xp, B.lo[B.paxis]), __dsub_rn(B.hi[B.paxis], B.lo[B.paxis]));
      f = __dmul_rn(__dmul_rn(6.0, xi), __dsub_rn(1.0, xi));
    }
    u = __dmul_rn(B.u_mean, f);
  }
  return make_double3(B.axis == 0 ? u : 0.0, B.axis == 1 ? u : 0.0, B.axis == 2 ? u : 0.0);
}

// ------------------------------------------------- neighbour-list entries
// Row-major Verlet list: nbr[i * cap + k], k < cnt[i].  With periodic axes and
// N < 2^27 an entry packs the neighbour index (27 bits) with the periodic image
// of its cell (per axis 0 none, 1 +L, 2 -L, packed base 3 into 5 bits), fixed at
// build time.  For any pair inside r_v + skin < L/2 this reproduces the minimum
// image of the oracle; the pair kernels then need 3 adds (on the rare wrapped
// entries) instead of 6 compares + selects.  Larger stores keep plain indices.
enum { kImgNone = 0, kImgCode = 1, kImgMin = 2 };
constexpr int kIdxBits = 27;
constexpr uint32_t kIdxMask = (1u << kIdxBits) - 1u;
__host__ __device__ __forceinline__ uint32_t img_tag(uint32_t ix, uint32_t iy, uint32_t iz) {
  return (ix + 3u * iy + 9u * iz) << kIdxBits;
}

template <int M>
__device__ __forceinline__ uint32_t nb_index(uint32_t e) {
  return M == kImgCode ? (e & kIdxMask) : e;
}
__device__ __forceinline__ double img_shift(uint32_t code, double L) {
  return code == 1u ? L : (code == 2u ? -L : 0.0);
}
// r_a - r_b under the entry's image convention (tolerance stages; FMA allowed)
template <int M>
__device__ __forceinline__ double3 pair_delta(const DevParams& P, double3 a, double3 b, uint32_t e) {
  if (M == kImgMin) return make_double3(mimg(P, a.x - b.x, 0), mimg(P, a.y - b.y, 1), mimg(P, a.z - b.z, 2));
  double3 d = make_double3(a.x - b.x, a.y - b.y, a.z - b.z);
  if (M == kImgCode && (e >> kIdxBits) != 0u) {  // only entries in wrapped cells (rare, mostly warp-uniform)
    const uint32_t c = e >> kIdxBits;
    d.x += img_shift(c % 3u, P.L[0]);
    d.y += img_shift((c / 3u) % 3u, P.L[1]);
    d.z += img_shift(c / 9u, P.L[2]);
  }
  return d;
}

// A particle that crosses a periodic face between rebuilds moves by -/+L: the image codes of its pairs,
// fixed at build time, are then off by one period.  The drift records it (wrap code: per axis 0 none, 1 the
// particle jumped by -L, 2 by +L, base 3) and k_wrap_patch_* shift the codes of its row entries and of
// the entries that reference it, so d = r_i - r_j + shift stays the minimum image until the next rebuild.
__device__ __forceinline__ uint32_t wrap_code(const DevParams& P, double3 o, double3 n) {
  uint32_t code = 0, mul = 1;
  const double xo[3] = {o.x, o.y, o.z}, xn[3] = {n.x, n.y, n.z};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (P.periodic[a]) {
      const double d = xn[a] - xo[a];
      if (d < -P.halfL[a]) code += 1u * mul;       // crossed hi: jumped by -L
      else if (d > P.halfL[a]) code += 2u * mul;   // crossed lo: jumped by +L
    }
    mul *= 3u;
  }
  return code;
}
// entry image code + sign * (wrap of one side): per axis value v in {0, +1, -1} (codes 0, 1, 2)
__device__ __forceinline__ uint32_t shift_code(uint32_t code, uint32_t w, int sign) {
  uint32_t out = 0, mul = 1;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const int c = (int)(code % 3u), wa = (int)(w % 3u);
    int v = c == 1 ? 1 : (c == 2 ? -1 : 0);
    v += sign * (wa == 1 ? 1 : (wa == 2 ? -1 : 0));  // x_i jumped by -L: d = x_i - x_j + s needs s + L
    out += (uint32_t)(v == 1 ? 1 : (v == -1 ? 2 : 0)) * mul;
    code /= 3u;
    w /= 3u;
    mul *= 3u;
  }
  return out;
}

// Kind-partitioned rows: while building, fluid neighbours fill row i from the front and rigid /
// boundary neighbours from the back; the back segment is then moved next to the front one, so a
// row is [fluid (nf) | non-fluid (no)] contiguous.  cnt[i] packs both counts (nf | no << 16).
// Move: with lo = max(nf + no, cap - no), entries [lo, cap) go to [nf, nf + cap - lo); source and
// destination are disjoint, entries already inside [nf, nf + no) stay.  Order within the non-fluid
// segment is not preserved (rows are sets).
__device__ __forceinline__ void compact_row(uint32_t* row, uint32_t nf, uint32_t no, int cap, int lane, int width) {
  if ((int)(nf + no) > cap) return;  // overflow: the caller rebuilds with a larger cap
  const uint32_t lo = max(nf + no, (uint32_t)cap - no);
  for (uint32_t m = lane; m < (uint32_t)cap - lo; m += width) row[nf + m] = row[lo + m];
}
__host__ __device__ __forceinline__ uint32_t cnt_fluid(uint32_t c) { return c & 0xffffu; }
__host__ __device__ __forceinline__ uint32_t cnt_other(uint32_t c) { return c >> 16; }
__host__ __device__ __forceinline__ uint32_t cnt_total(uint32_t c) { return (c & 0xffffu) + (c >> 16); }
__host__ __device__ __forceinline__ uint32_t pack_cnt(uint32_t nf, uint32_t no) {
  return (nf > 0xffffu ? 0xffffu : nf) | ((no > 0xffffu ? 0xffffu : no) << 16);
}

// sum over a group of G consecutive lanes (every lane of the warp must call it)
template <int G>
__device__ __forceinline__ int gmax(int v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <int G>
__device__ __forceinline__ double gsum(double v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------ quaternion
struct Quat {
  double w, x, y, z;
};
__device__ __forceinline__ double3 cross3(double3 a, double3 b) {
  return make_double3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
// rotate (quaternion.hpp:55-59): t = 2 u x p; p + w t + u x t
__device__ __forceinline__ double3 qrotate(const Quat& q, double3 p) {
  const double3 u = make_double3(q.x, q.y, q.z);
  double3 t = cross3(u, p);
  t.x *= 2.0; t.y *= 2.0; t.z *= 2.0;
  const double3 c = cross3(u, t);
  return make_double3(p.x + q.w * t.x + c.x, p.y + q.w * t.y + c.y, p.z + q.w * t.z + c.z);
}
__device__ __forceinline__ Quat qmul(const Quat& a, const Quat& b) {  // quaternion.hpp:27-32
  return {a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z, a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y,
          a.w * b.y - a.x * b.z + a.y * b.w + a.z * b.x, a.w * b.z + a.x * b.y - a.y * b.x + a.z * b.w};
}
// orientation_step (quaternion.hpp:67-76) with quat_exp (37-50)
__device__ __forceinline__ Quat orientation_step(const Quat& q, double3 w, double dt) {
  const double3 phi = make_double3(dt * w.x, dt * w.y, dt * w.z);
  const double ang = sqrt(phi.x * phi.x + phi.y * phi.y + phi.z * phi.z);
  double hs, ch;
  if (ang < 1e-8) {
    const double a2 = ang * ang;
    hs = 0.5 - a2 / 48.0;
    ch = 1.0 - a2 / 8.0;
  } else {
    double s, c;
    sincos(0.5 * ang, &s, &c);
    hs = s / ang;
    ch = c;
  }
  const Quat tr{ch, hs * phi.x, hs * phi.y, hs * phi.z};
  Quat r = qmul(tr, q);
  const double nrm = sqrt(r.w * r.w + r.x * r.x + r.y * r.y + r.z * r.z);
  return {r.w / nrm, r.x / nrm, r.y / nrm, r.z / nrm};
}

// --------------------------------------------- compensated sums (kahan.hpp)
// Neumaier accumulator (kahan.hpp:9-22) and an error-free pairwise merge for
// warp trees: merge((s1,c1),(s2,c2)) = TwoSum(s1,s2) + (c1 + c2).
struct KSum {
  double s, c;
  __device__ __forceinline__ void add(double x) {
    const double t = __dadd_rn(s, x);
    if (fabs(s) >= fabs(x)) c = __dadd_rn(c, __dadd_rn(__dsub_rn(s, t), x));
    else c = __dadd_rn(c, __dadd_rn(__dsub_rn(x, t), s));
    s = t;
  }
  __device__ __forceinline__ void merge(double s2, double c2) {
    const double t = __dadd_rn(s, s2);
    const double bp = __dsub_rn(t, s);
    const double e = __dadd_rn(__dsub_rn(s, __dsub_rn(t, bp)), __dsub_rn(s2, bp));
    s = t;
    c = __dadd_rn(__dadd_rn(c, c2), e);
  }
  __device__ __forceinline__ double value() const { return __dadd_rn(s, c); }
};

__device__ __forceinline__ KSum warp_merge(KSum k) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double s2 = __shfl_down_sync(0xffffffffu, k.s, o);
    const double c2 = __shfl_down_sync(0xffffffffu, k.c, o);
    k.merge(s2, c2);
  }
  return k;
}

// ------------------------------------------------------- device error word
enum : uint32_t { kErrEscape = 1u, kErrCoincident = 2u, kErrNaN = 4u, kErrOverflow = 8u, kErrInvariant = 16u };

struct DevFlags {
  unsigned long long max_disp2_bits;  // atomicMax on non-negative double bits
  unsigned long long umax2_bits;
  uint32_t err;
  uint32_t err_gid;                   // min gid involved (atomicMin)
  uint32_t err_gid2;
  uint32_t max_count;                 // neighbour list max length
  uint32_t n_events;                  // transition events
  uint32_t changed;                   // label propagation
  uint32_t pad[2];
  uint32_t build_overflow;            // cell-cooperative build could not take a cell
  uint32_t n_wrapped;                 // particles that crossed a periodic face this step (wrap_list)
  uint32_t pad2[2];
};

// drift / upload_state: note a periodic-face crossing for the row patch (kernels_step.cu k_wrap_patch_*)
__device__ __forceinline__ void record_wrap(const DevParams& P, DevFlags* fl, uint32_t* list, uint32_t k, double3 o,
                                            double3 n) {
  if (P.img_mode != kImgCode || !list) return;
  const uint32_t w = wrap_code(P, o, n);
  if (w) {
    const uint32_t s = atomicAdd(&fl->n_wrapped, 1u);
    list[2 * s] = k;
    list[2 * s + 1] = w;
  }
}

__device__ __forceinline__ void atomic_max_pos_double(unsigned long long* addr, double v) {
  atomicMax(addr, (unsigned long long)__double_as_longlong(v));
}

}  // namespace sphg

#define SPHG_CUDA_CHECK(expr)                                                 \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess) throw ::sphg::CudaError(_e, #expr, __FILE__, __LINE__); \
  } while (0)
