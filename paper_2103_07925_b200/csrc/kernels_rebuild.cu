// kernels_rebuild.cu — cell binning, radix sort, SoA reorder and Verlet
// neighbour-list build (SPEC:154-166 DomainGrid/NeighborList, 187-195
// build_pairs, 212-214 Verlet skin/inclusive cut-off/rebinning).
//
// Cell key [P1]: c_a = floor((x_a - lo_a) * inv_edge_a) clamped to [0, n_a),
// linearised (c0*n1 + c1)*n2 + c2.  Keys are scattered into gid order and
// stably radix-sorted, so the particle order is canonical (cell, gid) — the
// same on any GPU count and identical to the oracle's (bit-exact test).
// Candidates: j != i, not both boundary, r^2 <= (r_c + 0.1 h)^2 evaluated as
// (dx*dx + dy*dy) + dz*dz in round-to-nearest without contraction [P2].
// Lists: k_build_nlist_cells (warp per home cell, cells visited brick by brick, fp32 staging with
// an exact fp64 guard band) or k_build_nlist (warp per particle, fallback for dense cells); rows
// are kind-partitioned [fluid | non-fluid] and, for rigid particles, the non-fluid part starts
// with the contact candidates (k_contact_order).  Kind lists are emitted in brick order.
#include <algorithm>

#include "context.cuh"

namespace sphg {

namespace {

__device__ __forceinline__ int64_t cell_of(const DevParams& P, double x, double y, double z, uint32_t* escaped) {
  const double xs[3] = {x, y, z};
  int64_t c[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (!P.periodic[a] && (xs[a] < P.lo[a] || xs[a] > P.hi[a])) *escaped = 1;
    int64_t k = (int64_t)floor(__dmul_rn(__dsub_rn(xs[a], P.lo[a]), P.inv_edge[a]));
    k = k < 0 ? 0 : (k >= P.ncell[a] ? P.ncell[a] - 1 : k);
    c[a] = k;
  }
  return (c[0] * P.ncell[1] + c[1]) * P.ncell[2] + c[2];
}

__global__ void k_keys_by_gid(const __grid_constant__ DevParams P, const double4* __restrict__ G0,
                              const uint32_t* __restrict__ gid, size_t n, unsigned long long* __restrict__ keys,
                              uint32_t* __restrict__ vals, DevFlags* __restrict__ fl) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double4 p = G0[k];
  uint32_t esc = 0;
  const int64_t c = cell_of(P, p.x, p.y, p.z, &esc);
  const uint32_t g = gid[k];
  keys[g] = (unsigned long long)c;
  vals[g] = (uint32_t)k;
  if (esc) {
    atomicOr(&fl->err, kErrEscape);
    atomicMin(&fl->err_gid, g);
  }
}

// gather every per-particle field through the permutation; pos_ref := pos
__global__ void k_reorder(const uint32_t* __restrict__ perm, const unsigned long long* __restrict__ skeys, size_t n,
                          Particles src, Particles dst, uint32_t* __restrict__ cell_key) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const uint32_t o = perm[k];
  const double4 g0 = src.G0.p[o];
  dst.G0.p[k] = g0;
  dst.R4.p[k] = g0;
  dst.G1.p[k] = src.G1.p[o];
  dst.G2.p[k] = src.G2.p[o];
  dst.V4.p[k] = src.V4.p[o];
  dst.A4.p[k] = src.A4.p[o];
  dst.B4.p[k] = src.B4.p[o];
  dst.F4.p[k] = src.F4.p[o];
  dst.X4.p[k] = src.X4.p[o];
  dst.H2.p[k] = src.H2.p[o];
  dst.dTdt.p[k] = src.dTdt.p[o];
  dst.p_static.p[k] = src.p_static.p[o];
  dst.kmd.p[k] = src.kmd.p[o];
  dst.group.p[k] = src.group.p[o];
  dst.gid.p[k] = src.gid.p[o];
  if (src.C2.p) {
    dst.C2.p[k] = src.C2.p[o];
    dst.dCdt.p[k] = src.dCdt.p[o];
  }
  cell_key[k] = (uint32_t)skeys[k];
}

__global__ void k_cell_ranges(const uint32_t* __restrict__ key, size_t n, uint32_t* __restrict__ cstart,
                              uint32_t* __restrict__ cend) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const uint32_t c = key[k];
  if (k == 0 || key[k - 1] != c) cstart[c] = (uint32_t)k;
  if (k == n - 1 || key[k + 1] != c) cend[c] = (uint32_t)(k + 1);
}

// One warp per particle i: the 27 neighbour cells are scanned with the lanes
// over the cell's particles (coalesced), hits are compacted with a ballot and
// written contiguously into row i.  Entries carry the periodic image code of
// the neighbour cell (kImgCode) so pair kernels skip the minimum-image tests.
__global__ void __launch_bounds__(128) k_build_nlist(const __grid_constant__ DevParams P, const double4* __restrict__ G0,
                                                      const uint32_t* __restrict__ kmd,
                                                      const uint32_t* __restrict__ cell_key,
                                                      const uint32_t* __restrict__ cstart,
                                                      const uint32_t* __restrict__ cend, uint32_t* __restrict__ nbr,
                                                      uint32_t* __restrict__ cnt, int cap, size_t n,
                                                      DevFlags* __restrict__ fl) {
  const size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n) return;  // warp-uniform
  if (is_ghost(kmd[i])) {  // ghosts keep no row: they are read, never evaluated here
    if (lane == 0) cnt[i] = 0;
    return;
  }
  const double4 pi = G0[i];
  const bool bi = kind_of(kmd[i]) == SPHG_BOUNDARY;
  const int64_t c = cell_key[i];
  const int64_t nz = P.ncell[2], ny = P.ncell[1], nx = P.ncell[0];
  const int64_t cz = c % nz, cy = (c / nz) % ny, cx = c / (nz * ny);
  const bool code = P.img_mode == kImgCode;
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t* row = nbr + i * (size_t)cap;
  uint32_t nf = 0, no = 0;
  for (int ox = -1; ox <= 1; ++ox) {
    int64_t qx = cx + ox;
    uint32_t ix = 0;
    if (qx < 0 || qx >= nx) {
      if (!P.periodic[0]) continue;
      ix = qx < 0 ? 1u : 2u;
      qx = (qx + nx) % nx;
    }
    for (int oy = -1; oy <= 1; ++oy) {
      int64_t qy = cy + oy;
      uint32_t iy = 0;
      if (qy < 0 || qy >= ny) {
        if (!P.periodic[1]) continue;
        iy = qy < 0 ? 1u : 2u;
        qy = (qy + ny) % ny;
      }
      for (int oz = -1; oz <= 1; ++oz) {
        int64_t qz = cz + oz;
        uint32_t iz = 0;
        if (qz < 0 || qz >= nz) {
          if (!P.periodic[2]) continue;
          iz = qz < 0 ? 1u : 2u;
          qz = (qz + nz) % nz;
        }
        const uint32_t tag = code ? img_tag(ix, iy, iz) : 0u;
        const int64_t cj = (qx * ny + qy) * nz + qz;
        const uint32_t j0 = cstart[cj], j1 = cend[cj];
        for (uint32_t jb = j0; jb < j1; jb += 32) {
          const uint32_t j = jb + lane;
          bool hit = false, fj = false;
          if (j < j1 && j != i) {
            const uint32_t kj = kind_of(kmd[j]);
            fj = kj == SPHG_FLUID;
            if (!(bi && kj == SPHG_BOUNDARY)) {
              const double4 pj = G0[j];
              hit = r2_exact(mimg3(P, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z)) <= P.rv2;  // bit-exact test [P2]
            }
          }
          const uint32_t mf = __ballot_sync(0xffffffffu, hit && fj);
          const uint32_t mo = __ballot_sync(0xffffffffu, hit && !fj);
          if (hit && fj) {
            const uint32_t pos = nf + __popc(mf & lt);
            if ((int)pos < cap) row[pos] = j | tag;
          } else if (hit) {
            const uint32_t pos = no + __popc(mo & lt);
            if ((int)pos < cap) row[cap - 1 - pos] = j | tag;
          }
          nf += __popc(mf);
          no += __popc(mo);
        }
      }
    }
  }
  __syncwarp();
  compact_row(row, nf, no, cap, lane, 32);
  if (lane == 0) {
    cnt[i] = pack_cnt(nf, no);
    atomicMax(&fl->max_count, nf + no);
  }
}

// Cell-cooperative build: one warp per home cell.  The 27 neighbour cells are
// staged once in shared memory as fp32 positions relative to the home cell (in
// units of h); lanes run over the home cell's particles and test every staged
// candidate in fp32.  Pairs inside a 1e-4 guard band around r_v^2 (fp32 error
// is ~1e-6 relative here) fall back to the exact fp64 test of [P2] on the
// original positions, so the list is bit-identical to the pinned rule.
#ifndef SPHG_BUILD_STAGE
#define SPHG_BUILD_STAGE 512
#endif
#ifndef SPHG_BUILD_WARPS
#define SPHG_BUILD_WARPS 1
#endif
#ifndef SPHG_BUILD_MINB
#define SPHG_BUILD_MINB 20  // <= 96 registers: 64M rebuild 80.5 ms vs 97 ms at the compiler's 132 (r02 sweep)
#endif
constexpr int kStage = SPHG_BUILD_STAGE;  // staged candidates per batch (20 B each)
constexpr int kBuildWarps = SPHG_BUILD_WARPS;  // independent home cells per block (one per warp)
constexpr int kHomeMax = 256;   // particles per home cell handled here; denser cells -> per-particle kernel

struct BuildCtx {
  const DevParams* P;
  const double4* G0;
  const uint32_t* kmd;
  uint32_t* nbr;
  int cap;
};

// The staged batch of one warp: candidates as negated fp32 coordinates relative to the home cell
// (units of h), SoA so that two candidates sit in one 64-bit word of each array and the tests run on
// sm_100's packed fp32x2 pipe (FADD2 / FMUL2 / FFMA2: two candidates per instruction, each lane the same
// IEEE operation as the scalar form), plus the kind (0 fluid, 1 rigid, 2 boundary) and the entry.
struct Staged {
  float nx[kStage], ny[kStage], nz[kStage], kind[kStage];
};

// test the staged batch against every home particle, appending hits to their rows.
// Per chunk of 32 staged candidates each lane (home particle) builds bit masks: (1) fp32 tests,
// fully unrolled, two candidates per packed instruction: r^2 = fma(dx,dx, fma(dy,dy, dz*dz)) exactly as
// the scalar rule, then the sign bits of r^2 - r_v^2 (1 - 1e-4) ("inside") and of r_v^2 (1 + 1e-4) - r^2
// ("beyond the band") shifted into two masks with funnel shifts (one instruction per candidate and mask;
// the masks come out bit-reversed); (2) the rare guard-band bits get the pinned exact fp64 test [P2];
// (3) self and boundary-boundary bits are cleared with per-chunk masks built at staging; (4) the lane
// appends its fluid hits to the front of its row and the others to the back, one short loop iteration
// per hit.
__device__ __forceinline__ void build_batch(const DevParams& P, const double4* __restrict__ G0,
                                            const uint32_t* __restrict__ kmd, uint32_t* __restrict__ nbr, int cap,
                                            uint32_t h0, uint32_t h1, double ox0, double oy0, double oz0,
                                            const Staged* st, const uint32_t* se, int ns, uint32_t* hc,
                                            const uint32_t* hs, uint32_t batch, uint32_t* fmask, uint32_t* bmask,
                                            uint32_t emask) {
  const int lane = threadIdx.x & 31;
  const float rv2 = (float)(P.rv2 * P.inv_h * P.inv_h);
  const float lo_band = rv2 * (1.0f - 1e-4f), hi_band = rv2 * (1.0f + 1e-4f);
  const float2 nlo2 = make_float2(-lo_band, -lo_band), hi2 = make_float2(hi_band, hi_band);
  const float2 m12 = make_float2(-1.0f, -1.0f);
  // per-chunk kind masks of the staged candidates (padding dummies count as fluid; they never hit)
  for (int tb = 0; tb < ns; tb += 32) {
    const float w = st->kind[tb + lane];
    const uint32_t f = __ballot_sync(0xffffffffu, w == 0.f), bd = __ballot_sync(0xffffffffu, w == 2.f);
    if (lane == 0) {
      fmask[tb >> 5] = f;
      bmask[tb >> 5] = bd;
    }
  }
  __syncwarp();
  for (uint32_t ib = h0; ib < h1; ib += 32) {
    const uint32_t i = ib + lane;
    const bool act = i < h1 && !is_ghost(kmd[i]);
    double4 pi = make_double4(0, 0, 0, 0);
    float xi = 0.f, yi = 0.f, zi = 0.f;
    bool bi = false;
    uint32_t count = 0;
    int self = -1;  // this batch's stage index of particle i itself
    if (act) {
      pi = G0[i];
      xi = (float)((pi.x - ox0) * P.inv_h);
      yi = (float)((pi.y - oy0) * P.inv_h);
      zi = (float)((pi.z - oz0) * P.inv_h);
      bi = kind_of(kmd[i]) == SPHG_BOUNDARY;
      count = hc[i - h0];
      const uint32_t h = hs[i - h0];
      if ((h >> 16) == batch) self = (int)(h & 0xffffu);
    }
    uint32_t nf = cnt_fluid(count), no = cnt_other(count);
    uint32_t* row = nbr + (size_t)i * cap;
    uint32_t* back = row + cap - 1;
    const float2 xi2 = make_float2(xi, xi), yi2 = make_float2(yi, yi), zi2 = make_float2(zi, zi);
    for (int tb = 0; tb < ns; tb += 32) {
      uint32_t inr = 0, outr = 0;  // bit 31 - u: candidate tb + u
#pragma unroll
      for (int u = 0; u < 32; u += 2) {
        const float2 qx = *reinterpret_cast<const float2*>(st->nx + tb + u);
        const float2 qy = *reinterpret_cast<const float2*>(st->ny + tb + u);
        const float2 qz = *reinterpret_cast<const float2*>(st->nz + tb + u);
        const float2 dx = __fadd2_rn(xi2, qx), dy = __fadd2_rn(yi2, qy), dz = __fadd2_rn(zi2, qz);
        float2 r2 = __fmul2_rn(dz, dz);
        r2 = __ffma2_rn(dy, dy, r2);
        r2 = __ffma2_rn(dx, dx, r2);
        const float2 a = __fadd2_rn(r2, nlo2);     // < 0  <=>  r^2 < r_v^2 (1 - 1e-4)
        const float2 b = __ffma2_rn(r2, m12, hi2);  // < 0  <=>  r^2 > r_v^2 (1 + 1e-4)
        inr = __funnelshift_l(__float_as_uint(a.x), inr, 1);
        inr = __funnelshift_l(__float_as_uint(a.y), inr, 1);
        outr = __funnelshift_l(__float_as_uint(b.x), outr, 1);
        outr = __funnelshift_l(__float_as_uint(b.y), outr, 1);
      }
      uint32_t in = __brev(inr), maybe = ~__brev(outr);
      if (!act) maybe = in = 0;
      uint32_t band = maybe & ~in;
      while (band) {  // guard band: the pinned exact test (rare)
        const int u = __ffs(band) - 1;
        band &= band - 1;
        const double4 pj = G0[se[tb + u] & emask];
        if (r2_exact(mimg3(P, pi.x, pi.y, pi.z, pj.x, pj.y, pj.z)) <= P.rv2) in |= 1u << u;
      }
      if (self >= tb && self < tb + 32) in &= ~(1u << (self - tb));
      if (bi) in &= ~bmask[tb >> 5];
      const uint32_t fm = fmask[tb >> 5];
      uint32_t hf = in & fm, ho = in & ~fm;
      const uint32_t cf = __popc(hf), co = __popc(ho);
      const uint32_t* seb = se + tb;
      if (nf + cf <= (uint32_t)cap && no + co <= (uint32_t)cap) {  // common case: no bound checks
        uint32_t* wp = row + nf;
        while (hf) {  // fluid neighbours from the front
          const int u = __ffs(hf) - 1;
          hf &= hf - 1;
          *wp++ = seb[u];
        }
        uint32_t* bp = back - no;
        while (ho) {  // rigid / boundary neighbours from the back
          const int u = __ffs(ho) - 1;
          ho &= ho - 1;
          *bp-- = seb[u];
        }
      } else {  // overflowing row: count only what fits (the caller rebuilds with a larger cap)
        for (uint32_t k = nf; hf; ++k) {
          const int u = __ffs(hf) - 1;
          hf &= hf - 1;
          if ((int)k < cap) row[k] = seb[u];
        }
        for (uint32_t k = no; ho; ++k) {
          const int u = __ffs(ho) - 1;
          ho &= ho - 1;
          if ((int)k < cap) back[-(int)k] = seb[u];
        }
      }
      nf += cf;
      no += co;
    }
    if (act) hc[i - h0] = pack_cnt(nf, no);
  }
}

__global__ void __launch_bounds__(32 * kBuildWarps, SPHG_BUILD_MINB) k_build_nlist_cells(const __grid_constant__ DevParams P,
                                                           const double4* __restrict__ G0,
                                                           const uint32_t* __restrict__ kmd,
                                                           const uint32_t* __restrict__ cstart,
                                                           const uint32_t* __restrict__ cend,
                                                           uint32_t* __restrict__ nbr, uint32_t* __restrict__ cnt,
                                                           int cap, DevFlags* __restrict__ fl) {
  __shared__ Staged st_all[kBuildWarps];              // -x, -y, -z (relative to the home cell, units of h), kind
  __shared__ uint32_t se_all[kBuildWarps][kStage];   // neighbour index | image code
  __shared__ uint32_t hc_all[kBuildWarps][kHomeMax]; // running row length per home particle
  __shared__ uint32_t hs_all[kBuildWarps][kHomeMax]; // (batch << 16 | stage index) of each home particle
  __shared__ uint32_t fm_all[kBuildWarps][kStage / 32], bm_all[kBuildWarps][kStage / 32];
  __shared__ uint32_t cpre_all[kBuildWarps][28], cj0_all[kBuildWarps][27], ctag_all[kBuildWarps][27];
  __shared__ double csh_all[kBuildWarps][81];
  const int wib = threadIdx.x >> 5;
  Staged* st = &st_all[wib];
  uint32_t* se = se_all[wib];
  uint32_t* hc = hc_all[wib];
  uint32_t* hs = hs_all[wib];
  const int64_t c = brick_to_cell(P.ncell, (int64_t)blockIdx.x * kBuildWarps + wib);
  if (c < 0) return;
  const int lane = threadIdx.x & 31;
  const uint32_t h0 = cstart[c], h1 = cend[c];
  if (h1 <= h0) return;
  if (h1 - h0 > (uint32_t)kHomeMax) {
    if (lane == 0) atomicOr(&fl->build_overflow, 1u);
    return;
  }
  for (uint32_t k = lane; k < h1 - h0; k += 32) {
    hc[k] = 0;
    hs[k] = 0xffffffffu;
  }
  const int64_t nz = P.ncell[2], ny = P.ncell[1], nx = P.ncell[0];
  const int64_t cz = c % nz, cy = (c / nz) % ny, cx = c / (nz * ny);
  const double ox0 = P.lo[0] + (double)cx / P.inv_edge[0];  // any fixed origin near the cell works
  const double oy0 = P.lo[1] + (double)cy / P.inv_edge[1];
  const double oz0 = P.lo[2] + (double)cz / P.inv_edge[2];
  const bool code = P.img_mode == kImgCode;
  const uint32_t emask = code ? kIdxMask : 0xffffffffu;
  // home cell box in staged units (h), and the squared staging radius r_v (1 + 1e-3)
  const float ex = (float)(1.0 / (P.inv_edge[0] * P.h)), ey = (float)(1.0 / (P.inv_edge[1] * P.h)),
              ez = (float)(1.0 / (P.inv_edge[2] * P.h));
  const float box_lim = (float)(P.rv2 * P.inv_h * P.inv_h) * 1.001f;
  // the 27 neighbour cells (x-major, then y, then z: the pinned staging order): lane k < 27 resolves
  // cell k — periodic image, shift, candidate range — so the 27 range loads are in flight together
  // instead of one dependent round trip per cell; the candidates are then staged from the flattened
  // list, two per lane per round (both loads issued before either is used)
  uint32_t* cpre = cpre_all[wib];  // exclusive prefix of the cells' counts; [27] = total
  uint32_t* cj0 = cj0_all[wib];
  uint32_t* ctag = ctag_all[wib];
  double* csh = csh_all[wib];      // 3 per cell: the image shift
  {
    uint32_t cntk = 0, j0k = 0, tagk = 0;
    double shk[3] = {0.0, 0.0, 0.0};
    if (lane < 27) {
      const int o[3] = {lane / 9 - 1, (lane / 3) % 3 - 1, lane % 3 - 1};
      const int64_t cc[3] = {cx, cy, cz}, nn[3] = {nx, ny, nz};
      int64_t q[3];
      uint32_t im[3] = {0u, 0u, 0u};
      bool ok = true;
      for (int a = 0; a < 3; ++a) {
        q[a] = cc[a] + o[a];
        if (q[a] < 0 || q[a] >= nn[a]) {
          if (!P.periodic[a]) ok = false;
          im[a] = q[a] < 0 ? 1u : 2u;
          shk[a] = q[a] < 0 ? -P.L[a] : P.L[a];
          q[a] = (q[a] + nn[a]) % nn[a];
        }
      }
      if (ok) {
        const int64_t cj = (q[0] * ny + q[1]) * nz + q[2];
        j0k = cstart[cj];
        cntk = cend[cj] - j0k;
        tagk = code ? img_tag(im[0], im[1], im[2]) : 0u;
      }
    }
    uint32_t incl = cntk;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += v;
    }
    if (lane < 27) {
      cpre[lane] = incl - cntk;
      cj0[lane] = j0k;
      ctag[lane] = tagk;
      csh[3 * lane] = shk[0];
      csh[3 * lane + 1] = shk[1];
      csh[3 * lane + 2] = shk[2];
    }
    if (lane == 26) cpre[27] = incl;
  }
  __syncwarp();
  const uint32_t total = cpre[27];
  int ns = 0;
  uint32_t batch = 0;
  // flattened candidate t -> (cell k, particle j): the last cell whose prefix is <= t
  auto locate = [&](uint32_t t, int& k) {
    k = 0;
#pragma unroll
    for (int step = 16; step >= 1; step >>= 1)
      if (k + step < 27 && cpre[k + step] <= t) k += step;
  };
  for (uint32_t base = 0; base < total; base += 64) {
    if (ns > kStage - 64) {  // room for a full round of 64: flush the batch (padded to whole chunks)
      const int padded = (ns + 31) & ~31;
      for (int t = ns + lane; t < padded; t += 32) {
        st->nx[t] = st->ny[t] = st->nz[t] = -1e30f;
        st->kind[t] = 0.f;
        se[t] = 0u;
      }
      __syncwarp();
      build_batch(P, G0, kmd, nbr, cap, h0, h1, ox0, oy0, oz0, st, se, padded, hc, hs, batch, fm_all[wib],
                  bm_all[wib], emask);
      __syncwarp();
      ns = 0;
      ++batch;
    }
    const uint32_t ta = base + lane, tb2 = base + 32 + lane;
    int ka = 0, kb = 0;
    uint32_t ja = 0, jbb = 0;
    double4 pa = make_double4(0, 0, 0, 0), pb = make_double4(0, 0, 0, 0);
    uint32_t kda = 0, kdb = 0;
    if (ta < total) {
      locate(ta, ka);
      ja = cj0[ka] + (ta - cpre[ka]);
      pa = G0[ja];
      kda = kmd[ja];
    }
    if (tb2 < total) {
      locate(tb2, kb);
      jbb = cj0[kb] + (tb2 - cpre[kb]);
      pb = G0[jbb];
      kdb = kmd[jbb];
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const bool in_range = h == 0 ? ta < total : tb2 < total;
      const int k = h == 0 ? ka : kb;
      const uint32_t j = h == 0 ? ja : jbb;
      const double4 pj = h == 0 ? pa : pb;
      const uint32_t kdj = h == 0 ? kda : kdb;
      // stage the candidate only if it can be within r_v of the home cell's box (conservative fp32 box
      // distance with a 1e-3 margin; the exact rule decides later); the home cell (k = 13) always
      bool keep = in_range;
      const bool home = k == 13;
      float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
      if (keep) {
        // the periodic image of the cell: x_j + s sits next to the home cell
        q = make_float4((float)((pj.x + csh[3 * k] - ox0) * P.inv_h), (float)((pj.y + csh[3 * k + 1] - oy0) * P.inv_h),
                        (float)((pj.z + csh[3 * k + 2] - oz0) * P.inv_h), (float)kind_of(kdj));  // 0 fluid 1 rigid 2 wall
        const float dx = fmaxf(0.f, fmaxf(-q.x, q.x - ex)), dy = fmaxf(0.f, fmaxf(-q.y, q.y - ey)),
                    dz = fmaxf(0.f, fmaxf(-q.z, q.z - ez));
        keep = home || (dx * dx + dy * dy + dz * dz <= box_lim);
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        const int at = ns + __popc(bal & ((1u << lane) - 1u));
        st->nx[at] = -q.x;
        st->ny[at] = -q.y;
        st->nz[at] = -q.z;
        st->kind[at] = q.w;
        se[at] = j | ctag[k];
        if (home) hs[j - h0] = (batch << 16) | (uint32_t)at;
      }
      ns += __popc(bal);
    }
  }
  __syncwarp();
  if (ns) {
    const int padded = (ns + 31) & ~31;  // far-away dummies fail every test
    for (int t = ns + lane; t < padded; t += 32) {
      st->nx[t] = st->ny[t] = st->nz[t] = -1e30f;
      st->kind[t] = 0.f;
      se[t] = 0u;
    }
    __syncwarp();
    build_batch(P, G0, kmd, nbr, cap, h0, h1, ox0, oy0, oz0, st, se, padded, hc, hs, batch, fm_all[wib],
                bm_all[wib], emask);
  }
  __syncwarp();
  uint32_t mx = 0;
  for (uint32_t k = lane; k < h1 - h0; k += 32) {
    const uint32_t i = h0 + k;
    const uint32_t v = is_ghost(kmd[i]) ? 0u : hc[k];
    if (v) compact_row(nbr + (size_t)i * cap, cnt_fluid(v), cnt_other(v), cap, 0, 1);
    cnt[i] = v;
    mx = max(mx, cnt_total(v));
  }
  if (mx) atomicMax(&fl->max_count, mx);
}

// ------------------------------------------------------ contact order
// Contact only acts between different bodies or a body and a wall.  For every
// rigid particle the non-fluid part of its row is reordered (a set: order is free) so that those
// candidates come first, and their number is kept in ncon: k_forces_rigid then scans ncon entries
// instead of the whole non-fluid part, which for a body's interior is all its own particles.
// Redone at every rebuild and after transitions (group ids change).  Warp per rigid particle.
constexpr int kConWarps = 8;
constexpr int kConMaxRow = 512;
template <int M>
__global__ void __launch_bounds__(32 * kConWarps) k_contact_order(const uint32_t* __restrict__ kmd,
                                                                   const uint32_t* __restrict__ group,
                                                                   uint32_t* __restrict__ nbr,
                                                                   const uint32_t* __restrict__ cnt, int cap,
                                                                   const uint32_t* __restrict__ ridx, size_t nrigid,
                                                                   uint32_t* __restrict__ ncon) {
  __shared__ uint32_t buf[kConWarps][kConMaxRow], rest[kConWarps][kConMaxRow];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const size_t g = (size_t)blockIdx.x * kConWarps + wib;
  if (g >= nrigid) return;  // warp-uniform
  const uint32_t r = ridx[g];
  const uint32_t c = cnt[r];
  const uint32_t nf = cnt_fluid(c), no = cnt_other(c);
  uint32_t* seg = nbr + (size_t)r * cap + nf;
  if (no > (uint32_t)kConMaxRow) {  // not reordered: scan the whole part
    if (lane == 0) ncon[r] = no;
    return;
  }
  const uint32_t body = group[r];
  const uint32_t lt = (1u << lane) - 1u;
  // one pass: candidates and the rest into two staging buffers, then both back in order
  uint32_t fo = 0, oo = 0;
  for (uint32_t base = 0; base < no; base += 32) {
    const uint32_t k = base + lane;
    const bool in = k < no;
    const uint32_t e = in ? seg[k] : 0u;
    bool cand = false;
    if (in) {
      const uint32_t j = nb_index<M>(e);
      cand = kind_of(kmd[j]) == SPHG_BOUNDARY || group[j] != body;
    }
    const uint32_t bc = __ballot_sync(0xffffffffu, in && cand), bo = __ballot_sync(0xffffffffu, in && !cand);
    if (in) {
      if (cand) buf[wib][fo + __popc(bc & lt)] = e;
      else rest[wib][oo + __popc(bo & lt)] = e;
    }
    fo += __popc(bc);
    oo += __popc(bo);
  }
  __syncwarp();
  if (fo != 0 && oo != 0) {  // nothing to move when the part is all one class
    for (uint32_t k = lane; k < fo; k += 32) seg[k] = buf[wib][k];
    for (uint32_t k = lane; k < oo; k += 32) seg[fo + k] = rest[wib][k];
  }
  if (lane == 0) ncon[r] = fo;
}

// Checked builds (-DSPHG_CHECKED, tools/build_variants.py; compute-sanitizer is closed on this GPU pool):
// every row entry and index-list entry a kernel will decode is verified against the store once, when the
// rows / lists are (re)built, so each decode site downstream reads in bounds.  gid of the first bad row.
__global__ void k_check_rows(NbrList L, size_t n, int cap, DevFlags* __restrict__ fl) {
  const size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const uint32_t c = L.cnt[i], tot = cnt_total(c);
  bool bad = tot > (uint32_t)cap || cnt_fluid(c) > tot;
  const uint32_t* row = L.nbr + i * L.cap;
  for (uint32_t k = lane; !bad && k < tot; k += 32) {
    const uint32_t j = row[k] & kIdxMask;  // the index bits (image codes above them below 2^27 particles)
    bad = j >= n || j == i || (n >= (1u << kIdxBits) && row[k] >= n);
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) {
    atomicOr(&fl->err, kErrInvariant);
    atomicMin(&fl->err_gid, (uint32_t)i);
  }
}
__global__ void k_check_list(const uint32_t* __restrict__ list, size_t m, size_t n, DevFlags* __restrict__ fl) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < m && list[k] >= n) {
    atomicOr(&fl->err, kErrInvariant);
    atomicMin(&fl->err_gid, list[k]);
  }
}

}  // namespace

void check_structures(Ctx& c) {
#ifdef SPHG_CHECKED
  if (c.n == 0 || !c.built) return;
  k_check_rows<<<grid_for(c.n * 32, 256), 256, 0, c.stream>>>(c.nl(), c.n, c.cap, c.dflags);
  if (c.nf) k_check_list<<<grid_for(c.nf, 256), 256, 0, c.stream>>>(c.fidx.p, c.nf, c.n, c.dflags);
  if (c.nw) k_check_list<<<grid_for(c.nw, 256), 256, 0, c.stream>>>(c.widx.p, c.nw, c.n, c.dflags);
  if (c.nrigid) k_check_list<<<grid_for(c.nrigid, 256), 256, 0, c.stream>>>(c.ridx.p, c.nrigid, c.n, c.dflags);
  c.launches += 4;
#else
  (void)c;
#endif
}

// list = nullptr: every rigid particle (ridx); else the m listed rigid particles (a transition batch's
// changed neighbourhood)
void launch_contact_order(Ctx& c, const uint32_t* list, size_t m) {
  if (c.nrigid == 0) return;
  c.ncon.alloc(std::max<size_t>(c.n, 1));
  if (!list) {
    list = c.ridx.p;
    m = c.nrigid;
  }
  if (m == 0) return;
  const unsigned blocks = (unsigned)((m + kConWarps - 1) / kConWarps);
  switch (c.P.img_mode) {
    case kImgNone:
      k_contact_order<kImgNone><<<blocks, 32 * kConWarps, 0, c.stream>>>(c.cur.kmd.p, c.cur.group.p, c.nbr.p, c.cnt.p,
                                                                          c.cap, list, m, c.ncon.p);
      break;
    case kImgCode:
      k_contact_order<kImgCode><<<blocks, 32 * kConWarps, 0, c.stream>>>(c.cur.kmd.p, c.cur.group.p, c.nbr.p, c.cnt.p,
                                                                          c.cap, list, m, c.ncon.p);
      break;
    default:
      k_contact_order<kImgMin><<<blocks, 32 * kConWarps, 0, c.stream>>>(c.cur.kmd.p, c.cur.group.p, c.nbr.p, c.cnt.p,
                                                                         c.cap, list, m, c.ncon.p);
      break;
  }
  c.launches++;
}

namespace {

// ------------------------------------------------------- rigid index
__global__ void k_rigid_flags(const uint32_t* __restrict__ kmd, size_t n, uint32_t* __restrict__ flag) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) flag[k] = (kind_of(kmd[k]) == SPHG_RIGID && !is_ghost(kmd[k])) ? 1u : 0u;
}

__global__ void k_rigid_compact(const uint32_t* __restrict__ kmd, const uint32_t* __restrict__ group,
                                const uint32_t* __restrict__ gid, const uint32_t* __restrict__ pos, size_t n,
                                int gbits, unsigned long long* __restrict__ keys, uint32_t* __restrict__ vals) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n || kind_of(kmd[k]) != SPHG_RIGID || is_ghost(kmd[k])) return;
  const uint32_t s = pos[k];
  keys[s] = ((unsigned long long)group[k] << gbits) | gid[k];
  vals[s] = (uint32_t)k;
}

__global__ void k_body_ranges(const unsigned long long* __restrict__ keys, size_t m, int gbits,
                              uint32_t* __restrict__ bstart, uint32_t* __restrict__ bend) {
  const size_t s = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= m) return;
  const unsigned long long g = keys[s] >> gbits;
  if (s == 0 || (keys[s - 1] >> gbits) != g) bstart[g] = (uint32_t)s;
  if (s == m - 1 || (keys[s + 1] >> gbits) != g) bend[g] = (uint32_t)(s + 1);
}

int bits_for(uint64_t maxval) {  // bits needed to represent values in [0, maxval]
  int b = 0;
  while (b < 64 && (maxval >> b) != 0) ++b;
  return b;
}

// per brick position: fluid / non-fluid (non-ghost) particle counts of that cell
__global__ void k_cell_kind_counts(const __grid_constant__ DevParams P, const uint32_t* __restrict__ kmd,
                                   const uint32_t* __restrict__ cstart, const uint32_t* __restrict__ cend,
                                   int64_t npos, uint32_t* __restrict__ fc, uint32_t* __restrict__ wc) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= npos) return;
  const int64_t c = brick_to_cell(P.ncell, b);
  uint32_t nf = 0, nw = 0;
  if (c >= 0) {
    for (uint32_t k = cstart[c]; k < cend[c]; ++k) {
      const uint32_t m = kmd[k];
      if (is_ghost(m)) continue;
      if (kind_of(m) == SPHG_FLUID) ++nf;
      else ++nw;
    }
  }
  fc[b] = nf;
  wc[b] = nw;
}

__global__ void k_cell_kind_scatter(const __grid_constant__ DevParams P, const uint32_t* __restrict__ kmd,
                                    const uint32_t* __restrict__ cstart, const uint32_t* __restrict__ cend,
                                    int64_t npos, const uint32_t* __restrict__ fo, const uint32_t* __restrict__ wo,
                                    uint32_t* __restrict__ fidx, uint32_t* __restrict__ widx) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= npos) return;
  const int64_t c = brick_to_cell(P.ncell, b);
  if (c < 0) return;
  uint32_t f = fo[b], w = wo[b];
  for (uint32_t k = cstart[c]; k < cend[c]; ++k) {
    const uint32_t m = kmd[k];
    if (is_ghost(m)) continue;
    if (kind_of(m) == SPHG_FLUID) fidx[f++] = k;
    else widx[w++] = k;
  }
}

}  // namespace

namespace {
// 1 = the fluid particle's row holds no ghost (its sums need no halo data)
template <int M>
__global__ void k_interior_flags(const uint32_t* __restrict__ kmd, const uint32_t* __restrict__ fidx, size_t nf,
                                 NbrList L, uint32_t* __restrict__ flag) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nf) return;
  const uint32_t i = fidx[e];
  const uint32_t nn = cnt_total(L.cnt[i]);
  const uint32_t* row = L.nbr + (size_t)i * L.cap;
  uint32_t in = 1u;
  for (uint32_t k = 0; k < nn && in; ++k)
    if (is_ghost(kmd[nb_index<M>(row[k])])) in = 0u;
  flag[e] = in;
}

__global__ void k_split_scatter(const uint32_t* __restrict__ fidx, const uint32_t* __restrict__ flag,
                                const uint32_t* __restrict__ pos, size_t nf, uint32_t n_in, uint32_t* __restrict__ out) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nf) return;
  const uint32_t p = pos[e];  // interior particles before e
  out[flag[e] ? p : n_in + (uint32_t)e - p] = fidx[e];
}
}  // namespace

// Decomposed steps: order fidx [interior | next to a ghost], stably, so the interior density can run
// while the STATE halo is in flight (api.cu one_step_decomposed).  Single rank: all interior.
void launch_ghost_split(Ctx& c) {
  c.nf_interior = c.nf;
  if (c.nghost == 0 || c.nf == 0) return;
  cudaStream_t s = c.stream;
  uint32_t* flag = c.vals_alt.p;  // scratch (n >= nf)
  uint32_t* pos = c.vals.p;
  switch (c.P.img_mode) {
    case kImgNone: k_interior_flags<kImgNone><<<grid_for(c.nf, 128), 128, 0, s>>>(c.cur.kmd.p, c.fidx.p, c.nf, c.nl(), flag); break;
    case kImgCode: k_interior_flags<kImgCode><<<grid_for(c.nf, 128), 128, 0, s>>>(c.cur.kmd.p, c.fidx.p, c.nf, c.nl(), flag); break;
    default: k_interior_flags<kImgMin><<<grid_for(c.nf, 128), 128, 0, s>>>(c.cur.kmd.p, c.fidx.p, c.nf, c.nl(), flag); break;
  }
  exclusive_scan_u32(flag, pos, c.nf, c.scan_tmp.p, s, &c.launches);
  uint32_t tail[2] = {0, 0};
  SPHG_CUDA_CHECK(cudaMemcpyAsync(&tail[0], pos + c.nf - 1, 4, cudaMemcpyDeviceToHost, s));
  SPHG_CUDA_CHECK(cudaMemcpyAsync(&tail[1], flag + c.nf - 1, 4, cudaMemcpyDeviceToHost, s));
  host_sync(c, s);
  const uint32_t n_in = tail[0] + tail[1];
  uint32_t* out = c.keys_alt.p ? reinterpret_cast<uint32_t*>(c.keys_alt.p) : nullptr;  // scratch (8 B x n)
  k_split_scatter<<<grid_for(c.nf, 256), 256, 0, s>>>(c.fidx.p, flag, pos, c.nf, n_in, out);
  SPHG_CUDA_CHECK(cudaMemcpyAsync(c.fidx.p, out, c.nf * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
  c.nf_interior = n_in;
  c.launches += 3;
}

// fluid / non-fluid index lists (cell order) for the pair kernels
static void launch_kind_lists(Ctx& c) {
  const size_t n = c.n;
  cudaStream_t s = c.stream;
  c.fidx.alloc(std::max<size_t>(n, 1));
  c.widx.alloc(std::max<size_t>(n, 1));
  const int64_t npos = brick_positions(c.P.ncell);
  c.brick_buf.alloc(4 * (size_t)npos + 64);
  uint32_t* fc = c.brick_buf.p;
  uint32_t* wc = fc + npos;
  uint32_t* fo = wc + npos;
  uint32_t* wo = fo + npos;
  const unsigned g = (unsigned)((npos + 255) / 256);
  k_cell_kind_counts<<<g, 256, 0, s>>>(c.P, c.cur.kmd.p, c.cell_start.p, c.cell_end.p, npos, fc, wc);
  c.scan_cells.alloc(2 * ((size_t)npos / 256 + 2) + 64);
  exclusive_scan_u32(fc, fo, (size_t)npos, c.scan_cells.p, s, &c.launches);
  exclusive_scan_u32(wc, wo, (size_t)npos, c.scan_cells.p, s, &c.launches);
  k_cell_kind_scatter<<<g, 256, 0, s>>>(c.P, c.cur.kmd.p, c.cell_start.p, c.cell_end.p, npos, fo, wo, c.fidx.p,
                                        c.widx.p);
  uint32_t tail[4] = {0, 0, 0, 0};
  SPHG_CUDA_CHECK(cudaMemcpyAsync(&tail[0], fo + npos - 1, 4, cudaMemcpyDeviceToHost, s));
  SPHG_CUDA_CHECK(cudaMemcpyAsync(&tail[1], fc + npos - 1, 4, cudaMemcpyDeviceToHost, s));
  SPHG_CUDA_CHECK(cudaMemcpyAsync(&tail[2], wo + npos - 1, 4, cudaMemcpyDeviceToHost, s));
  SPHG_CUDA_CHECK(cudaMemcpyAsync(&tail[3], wc + npos - 1, 4, cudaMemcpyDeviceToHost, s));
  host_sync(c, s);
  c.nf = (size_t)tail[0] + tail[1];
  c.nw = (size_t)tail[2] + tail[3];
  c.nf_interior = c.nf;  // canonical order; launch_ghost_split reorders for decomposed steps
  c.launches += 2;
}

void launch_rigid_index(Ctx& c, bool kinds_changed) {
  const size_t n = c.n;
  cudaStream_t s = c.stream;
  if (n == 0) return;
  if (kinds_changed) launch_kind_lists(c);  // fluid / non-fluid lists (a split only moves body ids)
  c.ridx.alloc(std::max<size_t>(n, 1));
  c.body_start.alloc(2 * std::max<size_t>(c.nb, 1));
  uint32_t* flag = c.vals_alt.p;  // scratch
  uint32_t* pos = c.vals.p;
  k_rigid_flags<<<grid_for(n, 256), 256, 0, s>>>(c.cur.kmd.p, n, flag);
  exclusive_scan_u32(flag, pos, n, c.scan_tmp.p, s, &c.launches);
  uint32_t last_pos = 0, last_flag = 0;
  SPHG_CUDA_CHECK(cudaMemcpyAsync(&last_pos, pos + n - 1, 4, cudaMemcpyDeviceToHost, s));
  SPHG_CUDA_CHECK(cudaMemcpyAsync(&last_flag, flag + n - 1, 4, cudaMemcpyDeviceToHost, s));
  host_sync(c, s);
  const size_t m = (size_t)last_pos + last_flag;
  c.nrigid = m;
  SPHG_CUDA_CHECK(cudaMemsetAsync(c.body_start.p, 0, 2 * std::max<size_t>(c.nb, 1) * sizeof(uint32_t), s));
  c.launches += 2;
  if (m == 0) return;
  const int gbits = bits_for(n > 0 ? n - 1 : 0);
  k_rigid_compact<<<grid_for(n, 256), 256, 0, s>>>(c.cur.kmd.p, c.cur.group.p, c.cur.gid.p, pos, n, gbits, c.keys.p,
                                                   c.vals_alt.p);
  // vals_alt now holds particle indices (flag scratch consumed by the scan already)
  const int bits = gbits + bits_for(c.nb > 0 ? c.nb - 1 : 0);
  unsigned long long* k0 = c.keys.p;
  uint32_t* v0 = c.vals_alt.p;
  const bool flipped = radix_sort_pairs(k0, v0, c.keys_alt.p, c.vals.p, m, bits, c.hist.p, c.scan_tmp.p, s, &c.launches);
  unsigned long long* ks = flipped ? c.keys_alt.p : k0;
  uint32_t* vs = flipped ? c.vals.p : v0;
  SPHG_CUDA_CHECK(cudaMemcpyAsync(c.ridx.p, vs, m * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
  k_body_ranges<<<grid_for(m, 256), 256, 0, s>>>(ks, m, gbits, c.body_start.p, c.body_start.p + c.nb);
  c.launches += 3;
}

void launch_rebuild(Ctx& c) {
  const size_t n = c.n;
  cudaStream_t s = c.stream;
  if (n == 0) return;
  wrap_ghosts(c);
  // 1. keys in gid order
  k_keys_by_gid<<<grid_for(n, 256), 256, 0, s>>>(c.P, c.cur.G0.p, c.cur.gid.p, n, c.keys.p, c.vals.p, c.dflags);
  // 2. stable radix sort by cell
  const int bits = bits_for((uint64_t)(c.ncells - 1));
  const bool flipped = radix_sort_pairs(c.keys.p, c.vals.p, c.keys_alt.p, c.vals_alt.p, n, std::max(bits, 1), c.hist.p,
                                        c.scan_tmp.p, s, &c.launches);
  const unsigned long long* skeys = flipped ? c.keys_alt.p : c.keys.p;
  const uint32_t* perm = flipped ? c.vals_alt.p : c.vals.p;
  // 3. reorder into the alternate buffer set, swap
  k_reorder<<<grid_for(n, 256), 256, 0, s>>>(perm, skeys, n, c.cur, c.alt, c.cell_key.p);
  std::swap(c.cur, c.alt);
  build_idx_of_gid(c);
  // 4. cell ranges
  SPHG_CUDA_CHECK(cudaMemsetAsync(c.cell_start.p, 0, c.ncells * sizeof(uint32_t), s));
  SPHG_CUDA_CHECK(cudaMemsetAsync(c.cell_end.p, 0, c.ncells * sizeof(uint32_t), s));
  k_cell_ranges<<<grid_for(n, 256), 256, 0, s>>>(c.cell_key.p, n, c.cell_start.p, c.cell_end.p);
  c.launches += 5;
  // 5. neighbour list, grown on overflow
  for (int attempt = 0; attempt < 3; ++attempt) {
    // a multiple of 8 entries: 32-byte aligned rows (the pair kernels read them 16 bytes at a time)
    if (c.cap <= 0) c.cap = c.params.nlist_capacity > 0 ? (c.params.nlist_capacity + 7) / 8 * 8 : 144;
    c.nbr.alloc((size_t)c.cap * n);
    SPHG_CUDA_CHECK(cudaMemsetAsync(&c.dflags->max_count, 0, sizeof(uint32_t), s));
    uint32_t mc = 0, err = 0;
    if (c.cell_build) {
      SPHG_CUDA_CHECK(cudaMemsetAsync(&c.dflags->build_overflow, 0, sizeof(uint32_t), s));
      k_build_nlist_cells<<<(unsigned)((brick_positions(c.P.ncell) + kBuildWarps - 1) / kBuildWarps),
                            32 * kBuildWarps, 0, s>>>(c.P, c.cur.G0.p, c.cur.kmd.p, c.cell_start.p,
                                                            c.cell_end.p, c.nbr.p, c.cnt.p, c.cap, c.dflags);
      SPHG_CUDA_CHECK(cudaMemcpyAsync(&err, &c.dflags->build_overflow, 4, cudaMemcpyDeviceToHost, s));
      host_sync(c, s);
      c.launches += 2;
    }
    if (!c.cell_build || err) {  // per-particle build (also the fallback for over-dense cells)
      k_build_nlist<<<grid_for(n * 32, 128), 128, 0, s>>>(c.P, c.cur.G0.p, c.cur.kmd.p, c.cell_key.p, c.cell_start.p,
                                                          c.cell_end.p, c.nbr.p, c.cnt.p, c.cap, n, c.dflags);
      c.launches++;
    }
    c.launches++;
    SPHG_CUDA_CHECK(cudaMemcpyAsync(&mc, &c.dflags->max_count, 4, cudaMemcpyDeviceToHost, s));
    host_sync(c, s);
    c.max_count = (int)mc;
    if ((int)mc <= c.cap) break;
    c.cap = (int)((mc + 15) / 8 * 8);
    c.nbr.free();
  }
  launch_rigid_index(c);
  launch_contact_order(c);
  launch_ghost_split(c);
  c.built = true;
  c.rebuilds++;
  check_structures(c);
}

}  // namespace sphg
