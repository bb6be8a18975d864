// kernels_post.cu — post-processing gathers on sm_100a: the Shepard-filtered grid
// (shepard_interpolate), i.e. what OutputPlan::shepard_grid
// (config.hpp:53-59) dumps for the paper's field figures.  SURVEY §8(f) f4.
//
// One warp per grid point: the point's cell and its 26 neighbours (periodic images as in the
// Verlet build) are walked with the lanes over each cell's particles; numerator and denominator
// are warp-reduced.  The cell lists of the last rebuild are valid for this because the cell edge
// is >= r_c + skin and no particle has moved more than half the skin since.
#include "context.cuh"

namespace sphg {
namespace {

__device__ __forceinline__ int cell_coord(const DevParams& P, double x, int a) {
  int k = (int)floor((x - P.lo[a]) * P.inv_edge[a]);
  return k < 0 ? 0 : (k >= P.ncell[a] ? P.ncell[a] - 1 : k);
}

__global__ void __launch_bounds__(128) k_shepard_grid(const __grid_constant__ DevParams P, Particles D,
                                                       const uint32_t* __restrict__ cstart,
                                                       const uint32_t* __restrict__ cend, double ox, double oy,
                                                       double oz, double sx, double sy, double sz, int ny, int nz,
                                                       int64_t npts, int field, uint32_t kind_mask,
                                                       double* __restrict__ out, uint8_t* __restrict__ support) {
  const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (q >= npts) return;  // warp-uniform
  const int64_t a = q / ((int64_t)ny * nz), b = (q / nz) % ny, c = q % nz;
  double x[3] = {ox + (double)a * sx, oy + (double)b * sy, oz + (double)c * sz};
  // a periodic axis: locate the point's cell from its wrapped coordinate, keep the point where it is
  int ci[3];
  for (int ax = 0; ax < 3; ++ax) {
    double xw = x[ax];
    if (P.periodic[ax]) {
      xw = P.lo[ax] + fmod(xw - P.lo[ax], P.L[ax]);
      if (xw < P.lo[ax]) xw += P.L[ax];
    }
    ci[ax] = cell_coord(P, xw, ax);
    if (P.periodic[ax]) x[ax] = xw;
  }
  const int nc = field == SPHG_FIELD_VELOCITY ? 3 : 1;
  double num0 = 0.0, num1 = 0.0, num2 = 0.0, den = 0.0;
  for (int dx = -1; dx <= 1; ++dx) {
    int qx = ci[0] + dx;
    if (qx < 0 || qx >= P.ncell[0]) {
      if (!P.periodic[0]) continue;
      qx = (qx + P.ncell[0]) % P.ncell[0];
    }
    for (int dy = -1; dy <= 1; ++dy) {
      int qy = ci[1] + dy;
        if (qy < 0 || qy >= P.ncell[1]) {
        if (!P.periodic[1]) continue;
          qy = (qy + P.ncell[1]) % P.ncell[1];
      }
      for (int dz = -1; dz <= 1; ++dz) {
        int qz = ci[2] + dz;
            if (qz < 0 || qz >= P.ncell[2]) {
          if (!P.periodic[2]) continue;
              qz = (qz + P.ncell[2]) % P.ncell[2];
        }
        const int64_t cell = ((int64_t)qx * P.ncell[1] + qy) * P.ncell[2] + qz;
        const uint32_t j0 = cstart[cell], j1 = cend[cell];
        for (uint32_t j = j0 + lane; j < j1; j += 32) {
          const uint32_t kmd = D.kmd.p[j];
          if (!((kind_mask >> kind_of(kmd)) & 1u) || is_ghost(kmd)) continue;
          const double4 g0 = D.G0.p[j];
          // the oracle's minimum image x - r_j (the cell's image shift picks the same image inside r_c)
          const double3 d = mimg3(P, x[0], x[1], x[2], g0.x, g0.y, g0.z);
          double W;  // pinned arithmetic within ulps of r_c, where a lone weight decides "no support"
          if (!shepard_shape(P, d, d.x * d.x + d.y * d.y + d.z * d.z, W)) continue;
          const bool fl = kind_of(kmd) == SPHG_FLUID;
          const double rho = fl ? D.G1.p[j].w : P.mat[mat_of(kmd)].rho0;
          const double w = (D.V4.p[j].w / rho) * (P.sigma * W);
          den += w;
          switch (field) {
            case SPHG_FIELD_VELOCITY: {
              const double4 v = D.V4.p[j];
              num0 += w * v.x;
              num1 += w * v.y;
              num2 += w * v.z;
              break;
            }
            case SPHG_FIELD_TEMPERATURE: num0 += w * D.H2.p[j].x; break;
            case SPHG_FIELD_CONCENTRATION: num0 += w * (D.C2.p ? D.C2.p[j].x : 0.0); break;
            case SPHG_FIELD_PRESSURE: num0 += w * D.G2.p[j].w; break;
            default: num0 += w * rho; break;
          }
        }
      }
    }
  }
  den = gsum<32>(den);
  num0 = gsum<32>(num0);
  num1 = gsum<32>(num1);
  num2 = gsum<32>(num2);
  if (lane != 0) return;
  const bool ok = den > 0.0;
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  out[q * nc] = ok ? num0 / den : nan;
  if (nc == 3) {
    out[q * nc + 1] = ok ? num1 / den : nan;
    out[q * nc + 2] = ok ? num2 / den : nan;
  }
  if (support) support[q] = ok ? 1 : 0;
}

}  // namespace

void shepard_grid(Ctx& c, const double origin[3], const double spacing[3], const int32_t dims[3], int field,
                  uint32_t kind_mask, double* dev_out, uint8_t* dev_support) {
  const int64_t np = (int64_t)dims[0] * dims[1] * dims[2];
  if (np == 0) return;
  const int64_t threads = np * 32;
  k_shepard_grid<<<(unsigned)((threads + 127) / 128), 128, 0, c.stream>>>(
      c.P, c.cur, c.cell_start.p, c.cell_end.p, origin[0], origin[1], origin[2], spacing[0], spacing[1], spacing[2],
      dims[1], dims[2], np, field, kind_mask, dev_out, dev_support);
  c.launches++;
}

namespace {
// SPEC:218 occupancy histogram: one thread per cell of the last rebuild's ranges
__global__ void k_cell_occupancy(const uint32_t* __restrict__ start, const uint32_t* __restrict__ end, int64_t ncells,
                                 unsigned long long* __restrict__ hist, uint32_t nbins, uint32_t* __restrict__ maxc) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= ncells) return;
  const uint32_t m = end[k] > start[k] ? end[k] - start[k] : 0u;
  atomicAdd(&hist[m < nbins - 1 ? m : nbins - 1], 1ull);
  atomicMax(maxc, m);
}
}  // namespace

void cell_occupancy(Ctx& c, unsigned long long* dev_hist, uint32_t nbins, uint32_t* dev_max) {
  if (c.ncells == 0 || nbins == 0) return;
  k_cell_occupancy<<<(unsigned)((c.ncells + 255) / 256), 256, 0, c.stream>>>(c.cell_start.p, c.cell_end.p, c.ncells,
                                                                           dev_hist, nbins, dev_max);
  c.launches++;
}

}  // namespace sphg
