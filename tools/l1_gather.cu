// l1_gather.cu — microbenchmark of warp-wide 32-byte record gathers (LDG.E.ENL2.256) on sm_100a:
// how the L1 data pipe prices a warp request by its access pattern.  The pair kernels gather three
// 32-byte records per neighbour (G0, G1, G2); this measures the cost per request of
//   unaligned  8 lane groups x 4 consecutive records from a random start (today's row walk)
//   aligned    8 lane groups x 4 consecutive records of one 128-byte line (line-granular rows)
//   random     32 independent random records
//   shared     all 8 groups on the same line (4 distinct records per request)
//   coalesced  32 consecutive records (8 full lines)
// for a window that stays in L1 and one that lives in L2.  Build + run (GPU box):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l1g tools/l1_gather.cu && /tmp/l1g
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ double4 ldg4(const double4* p) {
  double4 v;
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

template <int MODE>
__device__ __forceinline__ uint32_t index_of(uint32_t seed, int lane, uint32_t window) {
  const int grp = lane >> 2, sub = lane & 3;
  if (MODE == 0) return (hash(seed + grp) % (window - 4)) + sub;          // unaligned groups of 4
  if (MODE == 1) return ((hash(seed + grp) % (window / 4)) * 4) + sub;    // aligned groups (one line each)
  if (MODE == 2) return hash(seed + lane) % window;                       // random
  if (MODE == 3) return ((seed % (window / 4)) * 4) + sub;                // every group on the same line
  return ((seed % (window / 32)) * 32) + lane;                            // 32 consecutive, aligned
}

// U independent iterations in flight (3 loads each), addresses from a precomputed per-lane table so
// the loop is load-throughput bound, not latency bound
template <int MODE>
__global__ void __launch_bounds__(128) k_gather(const double4* __restrict__ a, const double4* __restrict__ b,
                                                 const double4* __restrict__ c, uint32_t window, int iters,
                                                 double* __restrict__ out) {
  constexpr int U = 4, T = 16;
  const int lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t base = (warp * 977u) % (64u * 1024u * 1024u / 2u);
  __shared__ uint32_t tab[4][T][32];
  const int w = threadIdx.x >> 5;
  for (int t = 0; t < T; ++t) tab[w][t][lane] = base + index_of<MODE>(hash(warp * 131u + t), lane, window);
  __syncwarp();
  double s = 0.0;
  for (int it = 0; it < iters; it += U) {
    double4 x[U], y[U], z[U];
    // a data dependence the compiler cannot see through (the records are zeros: dep stays 0), so
    // every iteration's loads are really issued
    const uint32_t dep = (uint32_t)__double_as_longlong(s) & 1u;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t idx = tab[w][(it + u) & (T - 1)][lane] + dep;
      x[u] = ldg4(a + idx);
      y[u] = ldg4(b + idx);
      z[u] = ldg4(c + idx);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) s += x[u].x + y[u].y + z[u].z + x[u].w;
  }
  if (s == 12345.678) out[0] = s;
}

int main() {
  const size_t N = 64ull * 1024 * 1024;  // records per array (2 GiB each)
  double4 *a, *b, *c;
  double* out;
  cudaMalloc(&a, N * sizeof(double4));
  cudaMalloc(&b, N * sizeof(double4));
  cudaMalloc(&c, N * sizeof(double4));
  cudaMalloc(&out, 8);
  cudaMemset(a, 0, N * sizeof(double4));
  cudaMemset(b, 0, N * sizeof(double4));
  cudaMemset(c, 0, N * sizeof(double4));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 16, threads = 128, iters = 2048;
  const double requests = (double)blocks * (threads / 32) * iters * 3;  // 3 records per iteration
  const char* names[5] = {"unaligned4", "aligned4", "random", "sameline", "coalesced32"};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("{\"sms\": %d, \"results\": [\n", sms);
  bool first = true;
  for (uint32_t window : {1024u, 8192u, 262144u}) {
    for (int mode = 0; mode < 5; ++mode) {
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        switch (mode) {
          case 0: k_gather<0><<<blocks, threads>>>(a, b, c, window, iters, out); break;
          case 1: k_gather<1><<<blocks, threads>>>(a, b, c, window, iters, out); break;
          case 2: k_gather<2><<<blocks, threads>>>(a, b, c, window, iters, out); break;
          case 3: k_gather<3><<<blocks, threads>>>(a, b, c, window, iters, out); break;
          default: k_gather<4><<<blocks, threads>>>(a, b, c, window, iters, out); break;
        }
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      // SM cycles per warp request at 1.965 GHz, per SM
      const double clk = best * 1e-3 * 1.965e9 * sms / requests;
      printf("%s{\"window_records\": %u, \"pattern\": \"%s\", \"ms\": %.3f, \"sm_clk_per_request\": %.3f}",
             first ? "" : ",\n", window, names[mode], best, clk);
      first = false;
    }
  }
  printf("\n]}\n");
  return 0;
}
