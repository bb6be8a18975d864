// NcclTransport (include/sphfsi_gpu/decomposed_simulation.hpp) on a one-rank NCCL communicator: every call the
// decomposed step makes through the transport — grouped send / receive (to itself), MAX all-reduce of the
// displacement words, all-gather of the body partials, and the host byte all-to-all of migrations and
// transition batches — is issued for real on this GPU and its result checked.  More ranks need one GPU per
// rank; this pins the NCCL usage (datatypes, grouping, stream ordering against kernels on the same stream).
#include <cstdio>
#include <vector>

#define SPHG_WITH_NCCL 1
#include "sphfsi_gpu/decomposed_simulation.hpp"

#define CK(x)                                                       \
  do {                                                              \
    if ((x) != cudaSuccess) {                                       \
      std::printf("FAIL cuda %s line %d\n", #x, __LINE__);          \
      return 2;                                                     \
    }                                                               \
  } while (0)

int main() {
  try {
    CK(cudaSetDevice(0));
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return std::printf("FAIL ncclGetUniqueId\n"), 3;
    ncclComm_t comm;
    if (ncclCommInitRank(&comm, 1, id, 0) != ncclSuccess) return std::printf("FAIL ncclCommInitRank\n"), 3;
    {
      sphfsi_gpu::NcclTransport t(comm);
      if (t.rank() != 0 || t.size() != 1) return std::printf("FAIL rank/size\n"), 4;
      cudaStream_t s;
      CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      const size_t n = 1 << 16;
      std::vector<double> h(n), back(n, 0.0);
      for (size_t k = 0; k < n; ++k) h[k] = 1.0 / (double)(k + 1);
      double *a, *b;
      CK(cudaMalloc(&a, n * 8));
      CK(cudaMalloc(&b, n * 8));
      CK(cudaMemcpyAsync(a, h.data(), n * 8, cudaMemcpyHostToDevice, s));
      CK(cudaMemsetAsync(b, 0, n * 8, s));
      // halo phase: one send and one receive slot per peer (here the rank itself), stream-ordered
      t.exchange({{0, a, n * 8}}, {{0, b, n * 8}}, s);
      CK(cudaMemcpyAsync(back.data(), b, n * 8, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      if (back != h) return std::printf("FAIL exchange payload\n"), 5;
      // MAX of the two displacement words (bit patterns of non-negative doubles)
      const double w[2] = {0.125, 3.5};
      uint64_t* mw;
      CK(cudaMalloc(&mw, 16));
      CK(cudaMemcpyAsync(mw, w, 16, cudaMemcpyHostToDevice, s));
      t.allreduce_max_u64(mw, 2, s);
      double w2[2];
      CK(cudaMemcpyAsync(w2, mw, 16, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      if (w2[0] != w[0] || w2[1] != w[1]) return std::printf("FAIL allreduce\n"), 6;
      // body partials: nb x 24 doubles per rank
      CK(cudaMemsetAsync(b, 0, n * 8, s));
      t.allgather(a, b, 24 * 7 * 8, s);
      CK(cudaMemcpyAsync(back.data(), b, 24 * 7 * 8, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      for (size_t k = 0; k < 24 * 7; ++k)
        if (back[k] != h[k]) return std::printf("FAIL allgather\n"), 7;
      // host byte messages (migration records, transition batches), empty and non-empty
      std::vector<std::vector<uint8_t>> out(1, std::vector<uint8_t>(1000));
      for (size_t k = 0; k < 1000; ++k) out[0][k] = (uint8_t)(k * 7);
      auto in = t.alltoall_host(out);
      if (in.size() != 1 || in[0] != out[0]) return std::printf("FAIL alltoall_host\n"), 8;
      out[0].clear();
      in = t.alltoall_host(out);
      if (in.size() != 1 || !in[0].empty()) return std::printf("FAIL alltoall_host (empty)\n"), 9;
      cudaFree(a);
      cudaFree(b);
      cudaFree(mw);
      cudaStreamDestroy(s);
    }
    ncclCommDestroy(comm);
    std::printf("ok nccl transport (1 rank): exchange, allreduce MAX u64, allgather, alltoall_host\n");
    return 0;
  } catch (const std::exception& e) {
    std::printf("FAIL %s\n", e.what());
    return 1;
  }
}
