// decomposed_simulation.hpp — the multi-GPU host in C++: spatial domain decomposition over the
// reference's own ParticleStore<3>, one DecomposedSimulation per rank
// (one process or thread per GPU), driving the library's in-library decomposed step through the C ABI
// (sphg.h "In-library decomposed step") and a Transport for the exchanges.  The same protocol as the
// Python layer (paper_2103_07925_b200/parallel.py):
//   * ownership: px*py*pz equal boxes (halving the longest per-rank extent), ghosts within an L-infinity
//     distance r_c + 0.1h + margin of a rank's box (periodic images included), owned particles in gid
//     order then ghosts by (owner, gid); halo id lists per peer in gid order on both sides;
//   * a step: sphg_step with the exchange callback (halo STATE / DENSITY / WALL as grouped point-to-point
//     transfers, MAX of the displacement words, all-gather of the body partials; the library merges them
//     in rank order), SPHG_NEED_PARTITION -> migration, SPHG_NEED_TRANSITIONS -> the transition batch of
//     SPEC:500 (events and every member of the bodies they touch gathered at rank 0, applied there in a
//     scratch single-rank context, records and body table broadcast, written into owned and ghost copies).
// Transport: NcclTransport (define SPHG_WITH_NCCL; ncclSend / ncclRecv / ncclAllReduce / ncclAllGather on
// the library's stream) for GPUs, LocalTransport for ranks as threads of one process (host-staged; the
// tests run it on one GPU).  Header-only; link with libsphg.so and the CUDA runtime.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <barrier>
#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <numeric>
#include <vector>

#include "device_simulation.hpp"

#ifdef SPHG_WITH_NCCL
#include <nccl.h>
#endif

namespace sphfsi_gpu {

// ------------------------------------------------------------------ transport
/// One rank's view of the communicator.  Device transfers are ordered on `stream` (the library's stream:
/// what the callback enqueues runs after the library's pack kernels and before its unpack kernels).
class Transport {
 public:
  struct Msg {
    int peer;
    void* ptr;
    size_t bytes;
  };
  virtual ~Transport() = default;
  virtual int rank() const = 0;
  virtual int size() const = 0;
  /// grouped point to point: every `sends` entry lands in the peer's matching `recvs` entry
  virtual void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t stream) = 0;
  /// in place MAX over ranks of `count` unsigned 64-bit words in device memory
  virtual void allreduce_max_u64(uint64_t* dev, int count, cudaStream_t stream) = 0;
  /// dev_out (size() x bytes, rank order) <- every rank's dev_in
  virtual void allgather(const void* dev_in, void* dev_out, size_t bytes, cudaStream_t stream) = 0;
  /// host byte messages: out[q] goes to rank q; returns in[q] from rank q (setup, migration, batches)
  virtual std::vector<std::vector<uint8_t>> alltoall_host(const std::vector<std::vector<uint8_t>>& out) = 0;
};

/// Ranks as threads of one process (tests, or several contexts sharing a GPU): a hub of host mailboxes and a
/// barrier.  Device data is staged through the host.
class LocalHub {
 public:
  explicit LocalHub(int n) : n_(n), bar_(n), box_(n, std::vector<std::vector<uint8_t>>(n)) {}
  int n_;
  std::barrier<> bar_;
  std::vector<std::vector<std::vector<uint8_t>>> box_;  // box_[from][to]
};

class LocalTransport final : public Transport {
 public:
  LocalTransport(LocalHub& hub, int rank) : hub_(hub), rank_(rank) {}
  int rank() const override { return rank_; }
  int size() const override { return hub_.n_; }
  // Every copy is enqueued on `stream` and waited for there: a blocking cudaMemcpy from pageable memory may
  // return before its DMA has landed, and the library's stream does not wait for the legacy stream.
  void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t stream) override {
    for (const Msg& m : sends) {
      auto& b = hub_.box_[rank_][m.peer];
      b.resize(m.bytes);
      if (m.bytes) copy(b.data(), m.ptr, m.bytes, stream);
    }
    sync(stream);
    hub_.bar_.arrive_and_wait();
    for (const Msg& m : recvs) {
      const auto& b = hub_.box_[m.peer][rank_];
      if (b.size() != m.bytes) throw Error(SPHG_ERR_RUNTIME, "LocalTransport: message size mismatch");
      if (m.bytes) copy(m.ptr, b.data(), m.bytes, stream);
    }
    sync(stream);
    hub_.bar_.arrive_and_wait();
  }
  void allreduce_max_u64(uint64_t* dev, int count, cudaStream_t stream) override {
    auto& b = hub_.box_[rank_][rank_];
    b.resize(count * sizeof(uint64_t));
    copy(b.data(), dev, b.size(), stream);
    sync(stream);
    hub_.bar_.arrive_and_wait();
    std::vector<uint64_t> v(count, 0);
    for (int r = 0; r < hub_.n_; ++r) {
      const uint64_t* w = reinterpret_cast<const uint64_t*>(hub_.box_[r][r].data());
      for (int k = 0; k < count; ++k) v[k] = std::max(v[k], w[k]);
    }
    hub_.bar_.arrive_and_wait();
    copy(dev, v.data(), count * sizeof(uint64_t), stream);
    sync(stream);
  }
  void allgather(const void* dev_in, void* dev_out, size_t bytes, cudaStream_t stream) override {
    auto& b = hub_.box_[rank_][rank_];
    b.resize(bytes);
    if (bytes) copy(b.data(), dev_in, bytes, stream);
    sync(stream);
    hub_.bar_.arrive_and_wait();
    for (int r = 0; r < hub_.n_; ++r)
      if (bytes) copy(static_cast<uint8_t*>(dev_out) + r * bytes, hub_.box_[r][r].data(), bytes, stream);
    sync(stream);
    hub_.bar_.arrive_and_wait();
  }
  std::vector<std::vector<uint8_t>> alltoall_host(const std::vector<std::vector<uint8_t>>& out) override {
    for (int q = 0; q < hub_.n_; ++q) hub_.box_[rank_][q] = out[q];
    hub_.bar_.arrive_and_wait();
    std::vector<std::vector<uint8_t>> in(hub_.n_);
    for (int q = 0; q < hub_.n_; ++q) in[q] = hub_.box_[q][rank_];
    hub_.bar_.arrive_and_wait();
    return in;
  }

 private:
  static void copy(void* dst, const void* src, size_t bytes, cudaStream_t stream) {
    if (cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, stream) != cudaSuccess)
      throw Error(SPHG_ERR_CUDA, "LocalTransport: copy failed");
  }
  static void sync(cudaStream_t stream) {
    if (cudaStreamSynchronize(stream) != cudaSuccess) throw Error(SPHG_ERR_CUDA, "LocalTransport: sync failed");
  }
  LocalHub& hub_;
  int rank_;
};

#ifdef SPHG_WITH_NCCL
/// NCCL over NVLink / NVSwitch: the caller creates the communicator (ncclCommInitRank, one rank per GPU).
class NcclTransport final : public Transport {
 public:
  NcclTransport(ncclComm_t comm) : comm_(comm) {
    ncclCommUserRank(comm_, &rank_);
    ncclCommCount(comm_, &size_);
    cudaStreamCreateWithFlags(&host_stream_, cudaStreamNonBlocking);
  }
  ~NcclTransport() override { cudaStreamDestroy(host_stream_); }
  int rank() const override { return rank_; }
  int size() const override { return size_; }
  void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t stream) override {
    check(ncclGroupStart());
    for (const Msg& m : sends)
      if (m.bytes) check(ncclSend(m.ptr, m.bytes, ncclUint8, m.peer, comm_, stream));
    for (const Msg& m : recvs)
      if (m.bytes) check(ncclRecv(m.ptr, m.bytes, ncclUint8, m.peer, comm_, stream));
    check(ncclGroupEnd());
  }
  void allreduce_max_u64(uint64_t* dev, int count, cudaStream_t stream) override {
    check(ncclAllReduce(dev, dev, count, ncclUint64, ncclMax, comm_, stream));
  }
  void allgather(const void* dev_in, void* dev_out, size_t bytes, cudaStream_t stream) override {
    check(ncclAllGather(dev_in, dev_out, bytes, ncclUint8, comm_, stream));
  }
  std::vector<std::vector<uint8_t>> alltoall_host(const std::vector<std::vector<uint8_t>>& out) override {
    // sizes first (an all-gather of every rank's size row), then the payloads point to point
    std::vector<uint64_t> row(size_), all(size_ * size_);
    for (int q = 0; q < size_; ++q) row[q] = out[q].size();
    uint64_t *drow, *dall;
    cudaMalloc(&drow, size_ * 8);
    cudaMalloc(&dall, size_ * size_ * 8);
    cudaMemcpyAsync(drow, row.data(), size_ * 8, cudaMemcpyHostToDevice, host_stream_);  // ordered before the collective
    check(ncclAllGather(drow, dall, size_, ncclUint64, comm_, host_stream_));
    cudaMemcpyAsync(all.data(), dall, size_ * size_ * 8, cudaMemcpyDeviceToHost, host_stream_);
    cudaStreamSynchronize(host_stream_);
    cudaFree(drow);
    cudaFree(dall);
    std::vector<uint8_t*> sb(size_, nullptr), rb(size_, nullptr);
    check(ncclGroupStart());
    for (int q = 0; q < size_; ++q) {
      const uint64_t ns = out[q].size(), nr = all[q * size_ + rank_];
      if (ns) {
        cudaMalloc(&sb[q], ns);
        cudaMemcpyAsync(sb[q], out[q].data(), ns, cudaMemcpyHostToDevice, host_stream_);
        check(ncclSend(sb[q], ns, ncclUint8, q, comm_, host_stream_));
      }
      if (nr) {
        cudaMalloc(&rb[q], nr);
        check(ncclRecv(rb[q], nr, ncclUint8, q, comm_, host_stream_));
      }
    }
    check(ncclGroupEnd());
    cudaStreamSynchronize(host_stream_);
    std::vector<std::vector<uint8_t>> in(size_);
    for (int q = 0; q < size_; ++q) {
      in[q].resize(all[q * size_ + rank_]);
      if (rb[q]) cudaMemcpy(in[q].data(), rb[q], in[q].size(), cudaMemcpyDeviceToHost);
      if (sb[q]) cudaFree(sb[q]);
      if (rb[q]) cudaFree(rb[q]);
    }
    return in;
  }

 private:
  static void check(ncclResult_t r) {
    if (r != ncclSuccess) throw Error(SPHG_ERR_CUDA, std::string("NCCL: ") + ncclGetErrorString(r));
  }
  ncclComm_t comm_;
  int rank_ = 0, size_ = 1;
  cudaStream_t host_stream_ = nullptr;
};
#endif

// ------------------------------------------------------------------ ownership
/// The rank grid and ownership of parallel.Grid, with the same floating-point operations.
struct RankGrid {
  double lo[3], L[3];
  bool periodic[3];
  int dims[3] = {1, 1, 1};
  RankGrid(const sphg_params& p, int nranks) {
    double ext[3];
    for (int a = 0; a < 3; ++a) {
      lo[a] = p.lo[a];
      L[a] = p.hi[a] - p.lo[a];
      periodic[a] = p.periodic[a] != 0;
      ext[a] = L[a];
    }
    int n = nranks;
    while (n > 1 && n % 2 == 0) {  // halve the currently longest per-rank extent
      int a = 0;
      for (int b = 1; b < 3; ++b)
        if (ext[b] / dims[b] > ext[a] / dims[a]) a = b;
      dims[a] *= 2;
      n /= 2;
    }
    if (n > 1) {
      int a = 0;
      for (int b = 1; b < 3; ++b)
        if (ext[b] > ext[a]) a = b;
      dims[a] *= n;
    }
  }
  void box(int r, double blo[3], double bhi[3]) const {
    const int c[3] = {r / (dims[1] * dims[2]), (r / dims[2]) % dims[1], r % dims[2]};
    for (int a = 0; a < 3; ++a) {
      const double w = L[a] / dims[a];
      blo[a] = lo[a] + c[a] * w;
      bhi[a] = lo[a] + (c[a] + 1) * w;
    }
  }
  int owner_of(const double* x) const {
    int c[3];
    for (int a = 0; a < 3; ++a) {
      const double w = L[a] / dims[a];
      c[a] = (int)std::floor((x[a] - lo[a]) / w);
      c[a] = std::min(std::max(c[a], 0), dims[a] - 1);
    }
    return (c[0] * dims[1] + c[1]) * dims[2] + c[2];
  }
  bool near_box(const double* x, int r, double width) const {
    double blo[3], bhi[3];
    box(r, blo, bhi);
    for (int a = 0; a < 3; ++a) {
      bool in = x[a] >= blo[a] - width && x[a] <= bhi[a] + width;
      if (periodic[a]) {
        in = in || (x[a] + L[a] >= blo[a] - width && x[a] + L[a] <= bhi[a] + width);
        in = in || (x[a] - L[a] >= blo[a] - width && x[a] - L[a] <= bhi[a] + width);
      }
      if (!in) return false;
    }
    return true;
  }
};

// ------------------------------------------------------------------ helpers
inline const double* dp(const sphfsi::Vec<3>& v) { return reinterpret_cast<const double*>(&v); }  // 24 B xyz

namespace detail {
template <class T>
inline void put(std::vector<uint8_t>& b, const T* p, size_t n) {
  const uint8_t* s = reinterpret_cast<const uint8_t*>(p);
  b.insert(b.end(), s, s + n * sizeof(T));
}
template <class T>
inline const uint8_t* get(const uint8_t* src, T* p, size_t n) {
  std::memcpy(p, src, n * sizeof(T));
  return src + n * sizeof(T);
}
inline void two_sum_merge(const std::vector<double>& gathered, int world, size_t nb, std::vector<double>& tot) {
  tot.assign(nb * 12, 0.0);
  for (size_t q = 0; q < nb * 12; ++q) {  // rank-order TwoSum of (sum, comp) pairs (parallel._merge_partials)
    double s = gathered[2 * q], c = gathered[2 * q + 1];
    for (int r = 1; r < world; ++r) {
      const double s2 = gathered[(size_t)r * nb * 24 + 2 * q], c2 = gathered[(size_t)r * nb * 24 + 2 * q + 1];
      const double t = s + s2, bp = t - s, e = (s - (t - bp)) + (s2 - bp);
      c = (c + c2) + e;
      s = t;
    }
    tot[q] = s + c;
  }
}
}  // namespace detail

// ------------------------------------------------------------------ the rank
class DecomposedSimulation {
 public:
  DecomposedSimulation(const sphg_params& params, Transport& t, int device, double margin_h = 2.0)
      : P_(params), T_(t), device_(device) {
    P_.rank = t.rank();
    P_.nranks = t.size();
    grid_ = std::make_unique<RankGrid>(P_, t.size());
    const double h = P_.h > 0.0 ? P_.h : P_.dx;
    h_ = h;
    width_ = 3.0 * h + 0.1 * h + margin_h * h;
    margin_ = margin_h * h;
    cudaSetDevice(device_);
    check(sphg_create(&P_, device_, &ctx_), "create");
  }
  ~DecomposedSimulation() {
    free_buffers();
    if (ctx_) sphg_destroy(ctx_);
  }
  DecomposedSimulation(const DecomposedSimulation&) = delete;
  DecomposedSimulation& operator=(const DecomposedSimulation&) = delete;

  int rank() const { return T_.rank(); }
  size_t owned() const { return n_own_; }
  size_t local() const { return gids_.size(); }
  int64_t repartitions() const { return repartitions_; }
  int64_t batches() const { return batches_; }
  const std::vector<sphg_event>& events() const { return events_; }
  void set_event_log(bool on) { event_log_ = on; }
  sphg_ctx* context() { return ctx_; }

  /// Every rank holds the same global store (seeded generation is deterministic): keep the owned box and
  /// the ghost shell.
  void distribute(const sphfsi::ParticleStore<3>& g, const std::vector<sphg_body>& bodies) {
    const size_t n = g.size();
    std::vector<int> owner(n);
    for (size_t i = 0; i < n; ++i) owner[i] = grid_->owner_of(dp(g.pos[i]));
    const int r = T_.rank();
    std::vector<uint32_t> own, ghost;
    for (size_t i = 0; i < n; ++i) {
      if (owner[i] == r) own.push_back((uint32_t)i);
      else if (grid_->near_box(dp(g.pos[i]), r, width_)) ghost.push_back((uint32_t)i);
    }
    std::stable_sort(ghost.begin(), ghost.end(), [&](uint32_t a, uint32_t b) { return owner[a] < owner[b]; });
    std::vector<uint32_t> ids(own);
    ids.insert(ids.end(), ghost.begin(), ghost.end());
    sphfsi::ParticleStore<3> loc;
    take(g, ids, loc);
    for (size_t k = 0; k < ids.size(); ++k) loc.owner[k] = (uint32_t)owner[ids[k]];
    global_n_ = n;
    install_store(loc, std::vector<uint64_t>(ids.begin(), ids.end()), own.size(), bodies);
  }

  /// a^0: rebuild, density, DENSITY halo, extrapolation, WALL halo, forces, body totals (parallel.initialize)
  void initialize() {
    stage(SPHG_STAGE_REBUILD);
    stage(SPHG_STAGE_DENSITY);
    halo_stage(SPHG_HALO_DENSITY);
    stage(SPHG_STAGE_EXTRAPOLATE);
    halo_stage(SPHG_HALO_WALL);
    stage(SPHG_STAGE_FORCES);
    body_totals();
  }

  /// nsteps decomposed steps, migrating and applying transition batches as needed.
  void step(int nsteps) {
    check(sphg_set_partition_limit(ctx_, 0.5 * margin_), "set_partition_limit");
    int64_t c0[4];
    check(sphg_counters(ctx_, c0), "counters");
    int done = 0;
    while (done < nsteps) {
      const int rc = sphg_step(ctx_, nsteps - done);
      int64_t c1[4];
      check(sphg_counters(ctx_, c1), "counters");
      done += (int)(c1[0] - c0[0]);
      c0[0] = c1[0];
      if (rc == SPHG_NEED_PARTITION) {
        repartition();
        check(sphg_set_partition_limit(ctx_, 0.5 * margin_), "set_partition_limit");
        continue;
      }
      if (rc == SPHG_NEED_TRANSITIONS) {
        transition_batch();
        continue;
      }
      if (rc != SPHG_OK) {
        if (xerr_) throw Error(SPHG_ERR_CUDA, "exchange failed: " + xmsg_);
        check(rc, "step");
      }
    }
  }

  /// Owned particles of every rank -> the global store in gid order (every rank), and the body table.
  void gather(sphfsi::ParticleStore<3>& g, std::vector<sphg_body>& bodies) {
    sphfsi::ParticleStore<3> loc;
    resize(loc, local());
    sphg_soa v = views(loc);
    size_t nb = 0;
    check(sphg_num_bodies(ctx_, &nb), "num_bodies");
    bodies.resize(nb);
    check(sphg_download(ctx_, &v, bodies.data(), &nb), "download");
    std::vector<uint8_t> msg;
    const uint64_t m = n_own_;
    detail::put(msg, &m, 1);
    detail::put(msg, gids_.data(), n_own_);
    pack_rows(loc, 0, n_own_, msg);
    std::vector<std::vector<uint8_t>> out(T_.size(), msg);
    const auto in = T_.alltoall_host(out);
    resize(g, global_n_);
    for (const auto& b : in) {
      uint64_t cnt;
      const uint8_t* p = detail::get(b.data(), &cnt, 1);
      std::vector<uint64_t> gid(cnt);
      p = detail::get(p, gid.data(), cnt);
      unpack_rows(p, gid, g);
    }
  }

 private:
  // ---------------------------------------------------------------- store plumbing
  static void resize(sphfsi::ParticleStore<3>& s, size_t n) {
    s.pos.resize(n); s.vel.resize(n); s.vel_adv.resize(n); s.acc.resize(n); s.acc_bg.resize(n);
    s.density.resize(n); s.pressure.resize(n); s.mass.resize(n); s.temperature.resize(n); s.dT_dt.resize(n);
    s.concentration.resize(n); s.dC_dt.resize(n); s.kind.resize(n); s.group.resize(n); s.material.resize(n);
    s.body_frame_pos.resize(n); s.wall_pressure.resize(n); s.wall_velocity.resize(n);
    s.dirichlet_T.resize(n, 0xff); s.dirichlet_C.resize(n, 0xff); s.owner.resize(n);
  }
  static void take(const sphfsi::ParticleStore<3>& g, const std::vector<uint32_t>& ids, sphfsi::ParticleStore<3>& s) {
    resize(s, ids.size());
    for (size_t k = 0; k < ids.size(); ++k) {
      const size_t i = ids[k];
      s.pos[k] = g.pos[i]; s.vel[k] = g.vel[i]; s.vel_adv[k] = g.vel_adv[i]; s.acc[k] = g.acc[i];
      s.acc_bg[k] = g.acc_bg[i]; s.density[k] = g.density[i]; s.pressure[k] = g.pressure[i];
      s.mass[k] = g.mass[i]; s.temperature[k] = g.temperature[i]; s.dT_dt[k] = g.dT_dt[i];
      s.concentration[k] = g.concentration[i]; s.dC_dt[k] = g.dC_dt[i]; s.kind[k] = g.kind[i];
      s.group[k] = g.group[i]; s.material[k] = g.material[i]; s.body_frame_pos[k] = g.body_frame_pos[i];
      s.wall_pressure[k] = g.wall_pressure[i]; s.wall_velocity[k] = g.wall_velocity[i];
      s.dirichlet_T[k] = g.dirichlet_T[i]; s.dirichlet_C[k] = g.dirichlet_C[i];
    }
  }
  static void pack_rows(const sphfsi::ParticleStore<3>& s, size_t b, size_t e, std::vector<uint8_t>& msg) {
    const size_t m = e - b;
    detail::put(msg, dp(s.pos[b]), 3 * m); detail::put(msg, dp(s.vel[b]), 3 * m);
    detail::put(msg, dp(s.vel_adv[b]), 3 * m); detail::put(msg, dp(s.acc[b]), 3 * m);
    detail::put(msg, dp(s.acc_bg[b]), 3 * m); detail::put(msg, dp(s.body_frame_pos[b]), 3 * m);
    detail::put(msg, dp(s.wall_velocity[b]), 3 * m);
    detail::put(msg, &s.density[b], m); detail::put(msg, &s.pressure[b], m); detail::put(msg, &s.mass[b], m);
    detail::put(msg, &s.temperature[b], m); detail::put(msg, &s.dT_dt[b], m); detail::put(msg, &s.concentration[b], m);
    detail::put(msg, &s.dC_dt[b], m); detail::put(msg, &s.wall_pressure[b], m);
    detail::put(msg, &s.kind[b], m); detail::put(msg, &s.group[b], m); detail::put(msg, &s.material[b], m);
    detail::put(msg, &s.dirichlet_T[b], m); detail::put(msg, &s.dirichlet_C[b], m);
  }
  static void unpack_rows(const uint8_t* p, const std::vector<uint64_t>& gid, sphfsi::ParticleStore<3>& g) {
    const size_t m = gid.size();
    auto v3 = [&](std::vector<sphfsi::Vec<3>>& f) {
      std::vector<sphfsi::Vec<3>> t(m);
      p = detail::get(p, reinterpret_cast<double*>(t.data()), 3 * m);
      for (size_t k = 0; k < m; ++k) f[gid[k]] = t[k];
    };
    auto s1 = [&](auto& f) {
      using T = typename std::remove_reference_t<decltype(f)>::value_type;
      std::vector<T> t(m);
      p = detail::get(p, t.data(), m);
      for (size_t k = 0; k < m; ++k) f[gid[k]] = t[k];
    };
    v3(g.pos); v3(g.vel); v3(g.vel_adv); v3(g.acc); v3(g.acc_bg); v3(g.body_frame_pos); v3(g.wall_velocity);
    s1(g.density); s1(g.pressure); s1(g.mass); s1(g.temperature); s1(g.dT_dt); s1(g.concentration); s1(g.dC_dt);
    s1(g.wall_pressure); s1(g.kind); s1(g.group); s1(g.material); s1(g.dirichlet_T); s1(g.dirichlet_C);
  }

  void install_store(sphfsi::ParticleStore<3>& loc, std::vector<uint64_t> gids, size_t n_own,
                     const std::vector<sphg_body>& bodies) {
    gids_ = std::move(gids);
    n_own_ = n_own;
    sphg_soa v = views(loc);
    v.owner = loc.owner.data();  // owner != rank marks the ghost copies (views() leaves it NULL: all owned)
    check(sphg_upload(ctx_, &v, bodies.data(), bodies.size()), "upload");
    std::vector<int> owner(loc.owner.begin(), loc.owner.end());
    std::vector<double> pos(3 * loc.size());
    for (size_t k = 0; k < loc.size(); ++k)
      for (int a = 0; a < 3; ++a) pos[3 * k + a] = loc.pos[k][a];
    set_peers(pos, owner);
  }

  /// halo lists: send = my owned particles inside peer q's shell, recv = my ghosts owned by q; both in
  /// gid order (owned are gid-sorted, ghosts (owner, gid)-sorted), so no handshake is needed
  void set_peers(const std::vector<double>& pos, const std::vector<int>& owner) {
    peers_.clear();
    const int r = T_.rank();
    for (int q = 0; q < T_.size(); ++q) {
      if (q == r) continue;
      Peer pe;
      pe.rank = q;
      for (size_t k = 0; k < n_own_; ++k)
        if (grid_->near_box(&pos[3 * k], q, width_)) pe.send.push_back((uint32_t)k);
      for (size_t k = n_own_; k < gids_.size(); ++k)
        if (owner[k] == q) pe.recv.push_back((uint32_t)k);
      if (!pe.send.empty() || !pe.recv.empty()) peers_.push_back(std::move(pe));
    }
    for (size_t k = 0; k < peers_.size(); ++k) {
      check(sphg_halo_set(ctx_, 2 * (int)k, peers_[k].send.data(), peers_[k].send.size()), "halo_set");
      check(sphg_halo_set(ctx_, 2 * (int)k + 1, peers_[k].recv.data(), peers_[k].recv.size()), "halo_set");
    }
    bind();
  }

  void free_buffers() {
    for (void* p : dev_) cudaFree(p);
    dev_.clear();
  }
  void* dalloc(size_t bytes) {
    void* p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(bytes, 16)) != cudaSuccess) throw Error(SPHG_ERR_CUDA, "cudaMalloc");
    cudaMemset(p, 0, std::max<size_t>(bytes, 16));
    dev_.push_back(p);
    return p;
  }
  /// device buffers the library packs into / unpacks from, and the exchange callback
  void bind() {
    free_buffers();
    for (int ph = 0; ph < 3; ++ph) {
      const int d = sphg_halo_doubles(ph);
      for (size_t k = 0; k < peers_.size(); ++k) {
        peers_[k].buf[ph][0] = dalloc(peers_[k].send.size() * d * sizeof(double));
        peers_[k].buf[ph][1] = dalloc(peers_[k].recv.size() * d * sizeof(double));
        check(sphg_halo_bind(ctx_, ph, 2 * (int)k, static_cast<double*>(peers_[k].buf[ph][0])), "halo_bind");
        check(sphg_halo_bind(ctx_, ph, 2 * (int)k + 1, static_cast<double*>(peers_[k].buf[ph][1])), "halo_bind");
      }
    }
    maxw_ = static_cast<uint64_t*>(dalloc(2 * sizeof(uint64_t)));
    check(sphg_max_bind(ctx_, maxw_), "max_bind");
    check(sphg_num_bodies(ctx_, &nb_), "num_bodies");
    bpart_ = static_cast<double*>(dalloc(nb_ * 24 * sizeof(double)));
    bgath_ = static_cast<double*>(dalloc(T_.size() * nb_ * 24 * sizeof(double)));
    check(sphg_body_bind(ctx_, bpart_, bgath_, T_.size()), "body_bind");
    check(sphg_set_exchange(ctx_, &DecomposedSimulation::exchange_thunk, this), "set_exchange");
    void* s = nullptr;
    check(sphg_get_stream(ctx_, &s), "get_stream");
    stream_ = static_cast<cudaStream_t>(s);
  }

  static int exchange_thunk(int32_t phase, void* stream, void* user) {
    auto* self = static_cast<DecomposedSimulation*>(user);
    try {
      self->transfer(phase, static_cast<cudaStream_t>(stream));
      return 0;
    } catch (const std::exception& e) {
      self->xerr_ = true;
      self->xmsg_ = e.what();
      return 1;
    }
  }
  void transfer(int phase, cudaStream_t stream) {
    if (phase <= SPHG_HALO_WALL) {
      const int d = sphg_halo_doubles(phase);
      std::vector<Transport::Msg> s, r;
      for (auto& pe : peers_) {
        s.push_back({pe.rank, pe.buf[phase][0], pe.send.size() * d * sizeof(double)});
        r.push_back({pe.rank, pe.buf[phase][1], pe.recv.size() * d * sizeof(double)});
      }
      T_.exchange(s, r, stream);
    } else if (phase == SPHG_XCHG_MAX) {
      T_.allreduce_max_u64(maxw_, 2, stream);
    } else if (phase == SPHG_XCHG_BODIES) {
      T_.allgather(bpart_, bgath_, nb_ * 24 * sizeof(double), stream);
    } else {
      throw Error(SPHG_ERR_RUNTIME, "unknown exchange phase");
    }
  }

  // ---------------------------------------------------------------- stage path (initialize)
  void stage(int s) { check(sphg_run_stage(ctx_, s), "run_stage"); }
  void halo_stage(int phase) {
    for (size_t k = 0; k < peers_.size(); ++k)
      if (!peers_[k].send.empty())
        check(sphg_halo_pack(ctx_, phase, 2 * (int)k, static_cast<double*>(peers_[k].buf[phase][0])), "halo_pack");
    transfer(phase, stream_);
    cudaStreamSynchronize(stream_);
    for (size_t k = 0; k < peers_.size(); ++k)
      if (!peers_[k].recv.empty())
        check(sphg_halo_unpack(ctx_, phase, 2 * (int)k + 1, static_cast<double*>(peers_[k].buf[phase][1])),
              "halo_unpack");
  }
  /// reduce_force_torque over the ranks: partials -> all-gather -> rank-order TwoSum -> totals
  void body_totals() {
    if (nb_ == 0) return;
    check(sphg_body_partials(ctx_, bpart_), "body_partials");
    T_.allgather(bpart_, bgath_, nb_ * 24 * sizeof(double), stream_);
    cudaStreamSynchronize(stream_);
    std::vector<double> g((size_t)T_.size() * nb_ * 24), tot;
    cudaMemcpy(g.data(), bgath_, g.size() * sizeof(double), cudaMemcpyDeviceToHost);
    detail::two_sum_merge(g, T_.size(), nb_, tot);
    check(sphg_body_apply_totals(ctx_, tot.data()), "body_apply_totals");
  }

  std::vector<sphg_body> bodies_now() {
    size_t nb = 0;
    check(sphg_num_bodies(ctx_, &nb), "num_bodies");
    std::vector<sphg_body> b(nb);
    sphg_soa v;
    std::memset(&v, 0, sizeof(v));
    v.n = local();
    check(sphg_download(ctx_, &v, b.data(), &nb), "download");
    return b;
  }

  // ---------------------------------------------------------------- migration
  void repartition() {
    const int R = sphg_record_doubles();
    const size_t m = n_own_;
    std::vector<uint32_t> ids(m);
    std::iota(ids.begin(), ids.end(), 0u);
    std::vector<double> rec(m * R);
    check(sphg_record_pack(ctx_, ids.data(), m, rec.data()), "record_pack");
    const int W = T_.size(), r = T_.rank();
    std::vector<std::vector<uint8_t>> out(W);
    std::vector<std::pair<uint64_t, size_t>> keep;  // (gid, row) kept here
    for (size_t k = 0; k < m; ++k) {
      const int q = grid_->owner_of(&rec[k * R]);
      if (q == r) {
        keep.push_back({gids_[k], k});
        continue;
      }
      detail::put(out[q], &gids_[k], 1);
      detail::put(out[q], &rec[k * R], R);
    }
    const auto in = T_.alltoall_host(out);
    std::vector<std::pair<uint64_t, std::vector<double>>> owned;
    for (const auto& kr : keep) owned.push_back({kr.first, std::vector<double>(&rec[kr.second * R], &rec[kr.second * R] + R)});
    for (int q = 0; q < W; ++q) {
      const size_t rows = in[q].size() / (8 + 8 * R);
      const uint8_t* p = in[q].data();
      for (size_t k = 0; k < rows; ++k) {
        uint64_t gid;
        std::vector<double> rr(R);
        p = detail::get(p, &gid, 1);
        p = detail::get(p, rr.data(), R);
        owned.push_back({gid, std::move(rr)});
      }
    }
    std::sort(owned.begin(), owned.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    // ghosts: every peer gets my new owned particles inside its shell
    std::vector<std::vector<uint8_t>> shells(W);
    for (int q = 0; q < W; ++q) {
      if (q == r) continue;
      for (const auto& o : owned)
        if (grid_->near_box(o.second.data(), q, width_)) {
          detail::put(shells[q], &o.first, 1);
          detail::put(shells[q], o.second.data(), R);
        }
    }
    const auto gin = T_.alltoall_host(shells);
    std::vector<uint64_t> gids;
    std::vector<double> all;
    std::vector<int> owner;
    for (const auto& o : owned) {
      gids.push_back(o.first);
      all.insert(all.end(), o.second.begin(), o.second.end());
      owner.push_back(r);
    }
    for (int q = 0; q < W; ++q) {  // (owner, gid) order
      const size_t rows = gin[q].size() / (8 + 8 * R);
      const uint8_t* p = gin[q].data();
      for (size_t k = 0; k < rows; ++k) {  // each peer sends its owned set in gid order
        uint64_t gid;
        std::vector<double> rr(R);
        p = detail::get(p, &gid, 1);
        p = detail::get(p, rr.data(), R);
        gids.push_back(gid);
        all.insert(all.end(), rr.begin(), rr.end());
        owner.push_back(q);
      }
    }
    const std::vector<sphg_body> bodies = bodies_now();
    gids_ = gids;
    n_own_ = owned.size();
    check(sphg_upload_records(ctx_, gids_.size(), n_own_, all.data(), bodies.data(), bodies.size()), "upload_records");
    std::vector<double> pos(3 * gids_.size());
    for (size_t k = 0; k < gids_.size(); ++k)
      for (int a = 0; a < 3; ++a) pos[3 * k + a] = all[k * R + a];
    set_peers(pos, owner);
    ++repartitions_;
  }

  // ---------------------------------------------------------------- transitions
  void transition_batch() {
    const int R = sphg_record_doubles();
    const int W = T_.size(), r = T_.rank();
    std::vector<sphg_body> bodies = bodies_now();
    const size_t nb = bodies.size();
    std::vector<uint8_t> mask(nb, 0);
    check(sphg_event_bodies(ctx_, mask.data(), nb), "event_bodies");
    {  // OR over ranks
      const auto in = T_.alltoall_host(std::vector<std::vector<uint8_t>>(W, mask));
      for (const auto& b : in)
        for (size_t k = 0; k < nb; ++k) mask[k] |= b[k];
    }
    size_t m = 0;
    check(sphg_event_members(ctx_, mask.data(), nb, nullptr, 0, &m), "event_members");
    std::vector<uint32_t> ids(m);
    check(sphg_event_members(ctx_, mask.data(), nb, ids.data(), m, &m), "event_members");
    std::vector<double> rec(m * R);
    if (m) check(sphg_record_pack(ctx_, ids.data(), m, rec.data()), "record_pack");
    std::vector<std::vector<uint8_t>> out(W);
    for (size_t k = 0; k < m; ++k) {
      const uint64_t g = gids_[ids[k]];
      detail::put(out[0], &g, 1);
      detail::put(out[0], &rec[k * R], R);
    }
    const auto in = T_.alltoall_host(out);
    std::vector<std::vector<uint8_t>> result(W);
    if (r == 0) {
      std::vector<std::pair<uint64_t, size_t>> order;
      std::vector<double> rows;
      for (int q = 0; q < W; ++q) {
        const size_t cnt = in[q].size() / (8 + 8 * R);
        const uint8_t* p = in[q].data();
        for (size_t k = 0; k < cnt; ++k) {
          uint64_t g;
          p = detail::get(p, &g, 1);
          order.push_back({g, rows.size() / R});
          rows.resize(rows.size() + R);
          p = detail::get(p, &rows[rows.size() - R], R);
        }
      }
      std::sort(order.begin(), order.end());
      const size_t M = order.size();
      std::vector<double> recs(M * R);
      std::vector<uint64_t> gs(M);
      for (size_t k = 0; k < M; ++k) {
        gs[k] = order[k].first;
        std::copy(&rows[order[k].second * R], &rows[order[k].second * R] + R, &recs[k * R]);
      }
      std::vector<sphg_body> nbodies;
      std::vector<sphg_event> ev;
      apply_batch(recs, M, bodies, nbodies, ev);
      for (auto& e : ev) e.gid = (uint32_t)gs[e.gid];  // scratch ids -> global gids
      if (event_log_) events_.insert(events_.end(), ev.begin(), ev.end());
      std::vector<uint8_t> msg;
      const uint64_t MM = M, NB = nbodies.size();
      detail::put(msg, &MM, 1);
      detail::put(msg, gs.data(), M);
      detail::put(msg, recs.data(), M * R);
      detail::put(msg, &NB, 1);
      detail::put(msg, nbodies.data(), NB);
      for (int q = 0; q < W; ++q) result[q] = msg;
    }
    const auto got = T_.alltoall_host(result);
    const uint8_t* p = got[0].data();
    uint64_t M, NB;
    p = detail::get(p, &M, 1);
    std::vector<uint64_t> gs(M);
    p = detail::get(p, gs.data(), M);
    std::vector<double> recs(M * R);
    p = detail::get(p, recs.data(), M * R);
    p = detail::get(p, &NB, 1);
    std::vector<sphg_body> nbodies(NB);
    detail::get(p, nbodies.data(), NB);
    // every listed particle present here, owned or ghost
    std::vector<std::pair<uint64_t, uint32_t>> lk(gids_.size());
    for (size_t k = 0; k < gids_.size(); ++k) lk[k] = {gids_[k], (uint32_t)k};
    std::sort(lk.begin(), lk.end());
    std::vector<uint32_t> lids;
    std::vector<double> lrec;
    for (size_t k = 0; k < M; ++k) {
      auto it = std::lower_bound(lk.begin(), lk.end(), std::make_pair(gs[k], (uint32_t)0));
      if (it != lk.end() && it->first == gs[k]) {
        lids.push_back(it->second);
        lrec.insert(lrec.end(), &recs[k * R], &recs[k * R] + R);
      }
    }
    if (!lids.empty()) check(sphg_record_unpack(ctx_, lids.data(), lids.size(), lrec.data(), 1), "record_unpack");
    check(sphg_replace_bodies(ctx_, nbodies.data(), nbodies.size()), "replace_bodies");
    if (nbodies.size() != nb_) bind();  // body buffers are sized by the body count
    body_totals();
    ++batches_;
  }

  /// rank 0: the batch in a scratch single-rank context holding exactly the gathered particles (gid order)
  void apply_batch(std::vector<double>& recs, size_t M, const std::vector<sphg_body>& bodies,
                   std::vector<sphg_body>& out_bodies, std::vector<sphg_event>& ev) {
    const int R = sphg_record_doubles();
    sphg_params p1 = P_;
    p1.rank = 0;
    p1.nranks = 1;
    DeviceSimulation scratch(p1, device_);
    sphfsi::ParticleStore<3> st;
    resize(st, M);
    for (size_t k = 0; k < M; ++k) {
      const double* o = &recs[k * R];
      st.pos[k] = {o[0], o[1], o[2]};
      st.kind[k] = static_cast<sphfsi::Kind>((int)o[3]);
      st.material[k] = (sphfsi::MaterialId)o[4];
      st.group[k] = (uint32_t)o[5];
      st.mass[k] = o[6];
      st.density[k] = P_.mat[(int)o[4]].rho0;
      st.owner[k] = 0;
    }
    sphg_ctx* c = scratch_ctx(scratch);
    if (event_log_) check(sphg_set_event_log(c, 1), "set_event_log");
    scratch.upload(st, bodies);
    std::vector<uint32_t> ids(M);
    std::iota(ids.begin(), ids.end(), 0u);
    if (M) check(sphg_record_unpack(c, ids.data(), M, recs.data(), 0), "record_unpack");
    check(sphg_run_stage(c, SPHG_STAGE_TRANSITIONS), "transitions");
    if (M) check(sphg_record_pack(c, ids.data(), M, recs.data()), "record_pack");
    size_t nb = 0;
    check(sphg_num_bodies(c, &nb), "num_bodies");
    out_bodies.resize(nb);
    sphg_soa v;
    std::memset(&v, 0, sizeof(v));
    v.n = M;
    check(sphg_download(c, &v, out_bodies.data(), &nb), "download");
    if (event_log_) {
      size_t ne = 0;
      check(sphg_transition_events(c, nullptr, 0, &ne), "transition_events");
      ev.resize(ne);
      check(sphg_transition_events(c, ev.data(), ne, &ne), "transition_events");
      ev.resize(ne);
      int64_t cnt[4];
      check(sphg_counters(ctx_, cnt), "counters");
      for (auto& e : ev) e.step = cnt[0];
    }
  }
  static sphg_ctx* scratch_ctx(DeviceSimulation& s) { return s.raw(); }

  void check(int rc, const char* what) {
    if (rc != SPHG_OK) throw Error(rc, std::string(what) + ": " + (ctx_ ? sphg_last_error(ctx_) : ""));
  }

  struct Peer {
    int rank = 0;
    std::vector<uint32_t> send, recv;
    void* buf[3][2] = {{nullptr, nullptr}, {nullptr, nullptr}, {nullptr, nullptr}};
  };

  sphg_params P_;
  Transport& T_;
  int device_;
  std::unique_ptr<RankGrid> grid_;
  double h_ = 0, width_ = 0, margin_ = 0;
  sphg_ctx* ctx_ = nullptr;
  std::vector<uint64_t> gids_;
  size_t n_own_ = 0, global_n_ = 0;
  std::vector<Peer> peers_;
  std::vector<void*> dev_;
  uint64_t* maxw_ = nullptr;
  double *bpart_ = nullptr, *bgath_ = nullptr;
  size_t nb_ = 0;
  cudaStream_t stream_ = nullptr;
  bool xerr_ = false, event_log_ = false;
  std::string xmsg_;
  int64_t repartitions_ = 0, batches_ = 0;
  std::vector<sphg_event> events_;
};

}  // namespace sphfsi_gpu
