// radix_sort.cu — hand-written stable LSD radix sort of (u64 key, u32 value)
// pairs with 8-bit digits, plus a 3-phase exclusive scan.  Used for the cell
// binning sort (key = cell, input in gid order => (cell, gid)
// order) and for the body-major rigid index.
//
// Per pass: upsweep (per-tile digit histogram, digit-major) -> exclusive scan
// over [digit][tile] -> downsweep (stable in-tile ranking with warp
// __match_any_sync, then scatter).  A tile is 256 threads x 16 items, items
// striped so global loads are coalesced; stability follows item order
// (round, warp, lane) == global index order.
#include "context.cuh"

namespace sphg {

namespace {

constexpr int kThreads = 256;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;
constexpr int kDigits = 256;
constexpr int kScanItems = 16;
constexpr int kScanChunk = kThreads * kScanItems;  // 4096

__global__ void __launch_bounds__(kThreads) k_upsweep(const unsigned long long* __restrict__ keys, size_t n, int shift,
                                                       uint32_t* __restrict__ hist, int ntiles) {
  __shared__ uint32_t cnt[kDigits];
  cnt[threadIdx.x] = 0;
  __syncthreads();
  const size_t base = (size_t)blockIdx.x * kTile;
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const size_t i = base + (size_t)r * kThreads + threadIdx.x;
    if (i < n) atomicAdd(&cnt[(keys[i] >> shift) & 0xff], 1u);
  }
  __syncthreads();
  hist[(size_t)threadIdx.x * ntiles + blockIdx.x] = cnt[threadIdx.x];
}

__global__ void __launch_bounds__(kThreads) k_downsweep(const unsigned long long* __restrict__ keys,
                                                         const uint32_t* __restrict__ vals, size_t n, int shift,
                                                         const uint32_t* __restrict__ offs, int ntiles,
                                                         unsigned long long* __restrict__ keys_out,
                                                         uint32_t* __restrict__ vals_out) {
  __shared__ uint32_t cnt[kThreads / 32][kDigits];
  __shared__ uint32_t run[kDigits];
  __shared__ uint32_t base_off[kDigits];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  run[threadIdx.x] = 0;
  base_off[threadIdx.x] = offs[(size_t)threadIdx.x * ntiles + blockIdx.x];
  const size_t base = (size_t)blockIdx.x * kTile;
  const uint32_t lt_mask = (1u << lane) - 1u;
  for (int r = 0; r < kItems; ++r) {
    for (int k = threadIdx.x; k < (kThreads / 32) * kDigits; k += kThreads) (&cnt[0][0])[k] = 0;
    __syncthreads();
    const size_t i = base + (size_t)r * kThreads + threadIdx.x;
    const bool valid = i < n;
    unsigned long long key = 0;
    uint32_t val = 0;
    uint32_t d = kDigits;  // invalid items get a private digit
    if (valid) {
      key = keys[i];
      val = vals[i];
      d = (uint32_t)((key >> shift) & 0xff);
    }
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const uint32_t rank = __popc(peers & lt_mask);
    if (valid && rank == 0) cnt[warp][d] = __popc(peers);
    __syncthreads();
    if (valid) {
      uint32_t pre = 0;
      for (int w = 0; w < warp; ++w) pre += cnt[w][d];
      const uint32_t pos = base_off[d] + run[d] + pre + rank;
      keys_out[pos] = key;
      vals_out[pos] = val;
    }
    __syncthreads();
    {
      uint32_t s = 0;
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) s += cnt[w][threadIdx.x];
      run[threadIdx.x] += s;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- scan
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* total) {
  __shared__ uint32_t wsum[kThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < kThreads / 32 ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < kThreads / 32) wsum[lane] = w;
  }
  __syncthreads();
  const uint32_t before = warp > 0 ? wsum[warp - 1] : 0;
  if (total) *total = wsum[kThreads / 32 - 1];
  const uint32_t r = before + x - v;
  __syncthreads();
  return r;
}

// each block scans kScanChunk items (thread-blocked), writes block total
__global__ void __launch_bounds__(kThreads) k_scan_blocks(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                                           size_t n, uint32_t* __restrict__ block_sums) {
  const size_t base = (size_t)blockIdx.x * kScanChunk + (size_t)threadIdx.x * kScanItems;
  uint32_t v[kScanItems];
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = (base + k < n) ? in[base + k] : 0u;
    s += v[k];
  }
  uint32_t total;
  uint32_t run = block_exclusive_scan(s, &total);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < n) out[base + k] = run;
    run += v[k];
  }
  if (threadIdx.x == 0 && block_sums) block_sums[blockIdx.x] = total;
}

__global__ void k_scan_add(uint32_t* __restrict__ out, size_t n, const uint32_t* __restrict__ block_offs) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] += block_offs[i / kScanChunk];
}

}  // namespace

void exclusive_scan_u32(const uint32_t* in, uint32_t* out, size_t n, uint32_t* tmp, cudaStream_t s,
                        int64_t* launches) {
  if (n == 0) return;
  const size_t nblk = (n + kScanChunk - 1) / kScanChunk;
  if (nblk == 1) {
    k_scan_blocks<<<1, kThreads, 0, s>>>(in, out, n, nullptr);
    if (launches) *launches += 1;
    return;
  }
  uint32_t* sums = tmp;
  uint32_t* sums_scanned = tmp + nblk;
  k_scan_blocks<<<(int)nblk, kThreads, 0, s>>>(in, out, n, sums);
  exclusive_scan_u32(sums, sums_scanned, nblk, tmp + 2 * nblk, s, launches);
  k_scan_add<<<grid_for(n, 256), 256, 0, s>>>(out, n, sums_scanned);
  if (launches) *launches += 2;
}

size_t radix_scratch_words(size_t n) {
  const size_t ntiles = (n + kTile - 1) / kTile;
  const size_t m = ntiles * kDigits;
  // hist + scanned hist + recursive scan scratch
  return 2 * m + 4 * ((m + kScanChunk - 1) / kScanChunk) + 64;
}

bool radix_sort_pairs(unsigned long long* keys, uint32_t* vals, unsigned long long* keys_alt, uint32_t* vals_alt,
                      size_t n, int bits, uint32_t* hist, uint32_t* scan_tmp, cudaStream_t s, int64_t* launches) {
  if (n <= 1 || bits <= 0) return false;
  const int ntiles = (int)((n + kTile - 1) / kTile);
  const size_t m = (size_t)ntiles * kDigits;
  uint32_t* offs = hist + m;
  bool flipped = false;
  for (int shift = 0; shift < bits; shift += 8) {
    k_upsweep<<<ntiles, kThreads, 0, s>>>(keys, n, shift, hist, ntiles);
    exclusive_scan_u32(hist, offs, m, scan_tmp, s, launches);
    k_downsweep<<<ntiles, kThreads, 0, s>>>(keys, vals, n, shift, offs, ntiles, keys_alt, vals_alt);
    if (launches) *launches += 2;
    std::swap(keys, keys_alt);
    std::swap(vals, vals_alt);
    flipped = !flipped;
  }
  return flipped;
}

}  // namespace sphg
