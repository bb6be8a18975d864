// diag_gather.cuh — gather-cost diagnostics for k_forces_fluid (DESIGN.md §4 "The forces kernel is a
// gather kernel").  Included by kernels_pairs.cu only in -DSPHG_DIAG_LOADS_ONLY builds
// (tools/build_variants.py, tools/diag_loads.py); never part of the shipped library.
#pragma once

namespace {

// Diagnostic twin of k_forces_fluid (built only with -DSPHG_DIAG_LOADS_ONLY): the same row walk,
// the same three 256-bit neighbour loads and r^2 test, almost no arithmetic; results go to a
// scratch array.  Timed as stage 12 to separate the gather cost from the pair arithmetic.
template <int G, int M>
__global__ void __launch_bounds__(kBlock) k_forces_loads_only(const __grid_constant__ DevParams P, Particles D,
                                                               NbrList L, const uint32_t* __restrict__ list,
                                                               size_t nlist, double* __restrict__ scratch) {
  const size_t t = (size_t)blockIdx.x * kBlock + threadIdx.x;
  const size_t g = t / G;
  const int lane = (int)(t % G);
  const bool active = g < nlist;
  const uint32_t i = active ? list[g] : 0u;
  double s = 0.0;
  if (active) {
    const double3 pi = ld3(ldg4(&D.G0.p[i]));
    const Row R = row_of(L, i);
    uint32_t e = lane < R.n ? __ldg(R.f + lane) : 0u;
    for (int k = lane; k < R.n; k += G) {
      const uint32_t en = k + G < R.n ? __ldg(R.f + k + G) : 0u;
      const uint32_t j = nb_index<M>(e);
      const double4 h0 = ldg4(&D.G0.p[j]), h1 = ldg4(&D.G1.p[j]), h2 = ldg4(&D.G2.p[j]);
      const double3 d = pair_delta<M>(P, pi, ld3(h0), e);
      const double r2 = d.x * d.x + d.y * d.y + d.z * d.z;
      if (r2 <= P.rc2) s += h0.w + h1.x + h1.y + h1.z + h1.w + h2.x + h2.y + h2.z + h2.w;
      e = en;
    }
  }
  s = gsum<G>(s);
  if (active && lane == 0) scratch[i] = s;
}

// variants: kLayout 1 = one 128-byte AoS record per particle (G0 | G1 | G2 | pad), the three
// loads hit one line; kLayout 2 = only the G0 record (one load per pair)
template <int G, int M, int kLayout>
__global__ void __launch_bounds__(kBlock) k_gather_variant(const __grid_constant__ DevParams P, Particles D,
                                                            NbrList L, const uint32_t* __restrict__ list,
                                                            size_t nlist, const double4* __restrict__ aos,
                                                            double* __restrict__ scratch) {
  const size_t t = (size_t)blockIdx.x * kBlock + threadIdx.x;
  const size_t g = t / G;
  const int lane = (int)(t % G);
  const bool active = g < nlist;
  const uint32_t i = active ? list[g] : 0u;
  double s = 0.0;
  if (active) {
    const double3 pi = ld3(ldg4(&D.G0.p[i]));
    const Row R = row_of(L, i);
    uint32_t e = lane < R.n ? __ldg(R.f + lane) : 0u;
    for (int k = lane; k < R.n; k += G) {
      const uint32_t en = k + G < R.n ? __ldg(R.f + k + G) : 0u;
      const uint32_t j = nb_index<M>(e);
      double4 h0, h1 = make_double4(0, 0, 0, 0), h2 = make_double4(0, 0, 0, 0);
      if (kLayout == 1) {
        h0 = ldg4(aos + 4 * (size_t)j);
        h1 = ldg4(aos + 4 * (size_t)j + 1);
        h2 = ldg4(aos + 4 * (size_t)j + 2);
      } else {
        h0 = ldg4(&D.G0.p[j]);
      }
      const double3 d = pair_delta<M>(P, pi, ld3(h0), e);
      const double r2 = d.x * d.x + d.y * d.y + d.z * d.z;
      if (r2 <= P.rc2) s += h0.w + h1.x + h1.y + h1.z + h1.w + h2.x + h2.y + h2.z + h2.w;
      e = en;
    }
  }
  s = gsum<G>(s);
  if (active && lane == 0) scratch[i] = s;
}

__global__ void k_fill_aos(Particles D, size_t n, double4* __restrict__ aos) {
  const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  aos[4 * k] = D.G0.p[k];
  aos[4 * k + 1] = D.G1.p[k];
  aos[4 * k + 2] = D.G2.p[k];
}

}  // namespace

// times the variants into stage_ms[12..15] (tools/diag_loads.py)
inline void launch_diag_gather(Ctx& c) {
  // times its variants into stage_ms[12..15] (tools/diag_loads.py)
  if (c.nf == 0) return;
  static DBuf<double> scratch;
  static DBuf<double4> aos;
  scratch.alloc(c.n);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0.f;
  auto timed_run = [&](int slot, auto&& fn) {
    cudaEventRecord(e0, c.stream);
    fn();
    cudaEventRecord(e1, c.stream);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    c.stage_ms[slot] += ms;
  };
  timed_run(12, [&] {
    SPHG_IMG_DISPATCH(c.P.img_mode, (k_forces_loads_only<4, M><<<blocks_for<4>(c.nf), kBlock, 0, c.stream>>>(
                                         c.P, c.cur, c.nl(), c.fidx.p, c.nf, scratch.p)));
  });
  const char* mode = std::getenv("SPHG_DIAG_MODE");
  if (mode && mode[0] == 'G') {  // lane-group width of the SoA gather: 2, 8, 16
    timed_run(13, [&] {
      SPHG_IMG_DISPATCH(c.P.img_mode, (k_forces_loads_only<2, M><<<blocks_for<2>(c.nf), kBlock, 0, c.stream>>>(
                                           c.P, c.cur, c.nl(), c.fidx.p, c.nf, scratch.p)));
    });
    timed_run(14, [&] {
      SPHG_IMG_DISPATCH(c.P.img_mode, (k_forces_loads_only<8, M><<<blocks_for<8>(c.nf), kBlock, 0, c.stream>>>(
                                           c.P, c.cur, c.nl(), c.fidx.p, c.nf, scratch.p)));
    });
    timed_run(15, [&] {
      SPHG_IMG_DISPATCH(c.P.img_mode, (k_forces_loads_only<16, M><<<blocks_for<16>(c.nf), kBlock, 0, c.stream>>>(
                                           c.P, c.cur, c.nl(), c.fidx.p, c.nf, scratch.p)));
    });
  } else {
    aos.alloc(4 * c.n);
    k_fill_aos<<<grid_for(c.n, 256), 256, 0, c.stream>>>(c.cur, c.n, aos.p);
    timed_run(13, [&] {
      SPHG_IMG_DISPATCH(c.P.img_mode, (k_gather_variant<4, M, 1><<<blocks_for<4>(c.nf), kBlock, 0, c.stream>>>(
                                           c.P, c.cur, c.nl(), c.fidx.p, c.nf, aos.p, scratch.p)));
    });
    timed_run(14, [&] {
      SPHG_IMG_DISPATCH(c.P.img_mode, (k_gather_variant<4, M, 2><<<blocks_for<4>(c.nf), kBlock, 0, c.stream>>>(
                                           c.P, c.cur, c.nl(), c.fidx.p, c.nf, aos.p, scratch.p)));
    });
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}
