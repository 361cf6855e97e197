// Collective transports (see comm.h).
#include "comm.h"

#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>

namespace phd {

// ---------------------------------------------------------------------------
class NcclComm : public Comm {
 public:
  NcclComm(ncclComm_t c, int world, int rank) : c_(c), world_(world), rank_(rank) {}
  ~NcclComm() override {
    for (void* p : opened_) cudaIpcCloseMemHandle(p);
    if (c_) ncclCommDestroy(c_);
  }
  const char* name() const override { return "nccl"; }

  std::string allreduce_f64(double* buf, size_t n, cudaStream_t s) override {
    if (n == 0) return "";
    ncclResult_t r = ncclAllReduce(buf, buf, n, ncclDouble, ncclSum, c_, s);
    return r == ncclSuccess ? "" : std::string("ncclAllReduce: ") + ncclGetErrorString(r);
  }

  std::string exchange(float* const* src, float* const* dst, int narr, const ExchangePlan& p,
                       cudaStream_t s) override {
    ncclResult_t r = ncclGroupStart();
    for (int q = 0; q < world_ && r == ncclSuccess; ++q) {
      if (q == rank_) continue;
      for (int i = 0; i < narr && r == ncclSuccess; ++i) {
        if (p.send_count[q] > 0)
          r = ncclSend(src[i] + p.send_off[q], (size_t)p.send_count[q], ncclFloat, q, c_, s);
        if (r == ncclSuccess && p.recv_count[q] > 0)
          r = ncclRecv(dst[i] + p.recv_off[q], (size_t)p.recv_count[q], ncclFloat, q, c_, s);
      }
    }
    ncclResult_t e = ncclGroupEnd();
    if (r == ncclSuccess) r = e;
    return r == ncclSuccess ? "" : std::string("nccl exchange: ") + ncclGetErrorString(r);
  }

  std::string allgather_bytes(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    ncclResult_t r = ncclAllGather(send, recv, bytes, ncclChar, c_, s);
    return r == ncclSuccess ? "" : std::string("ncclAllGather: ") + ncclGetErrorString(r);
  }

  std::string share_buffers(void* const* local, int nbuf, std::vector<void*>* all, cudaStream_t s) override {
    return ipc_share_buffers(*this, world_, rank_, local, nbuf, all, &opened_, s);
  }

 private:
  ncclComm_t c_;
  int world_, rank_;
  std::vector<void*> opened_;
};

std::string ipc_share_buffers(Comm& c, int world_, int rank_, void* const* local, int nbuf, std::vector<void*>* all,
                            std::vector<void*>* opened, cudaStream_t s) {
  const size_t hb = sizeof(cudaIpcMemHandle_t);
  std::vector<cudaIpcMemHandle_t> mine(nbuf), every((size_t)nbuf * world_);
  // every rank must take the same path through the collectives below: a local
  // failure is all-reduced before anyone opens a handle
  int bad = 0;
  for (int b = 0; b < nbuf; ++b)
    if (cudaIpcGetMemHandle(&mine[b], local[b]) != cudaSuccess) bad = 1;
  cudaGetLastError();
  void* dev = nullptr;
  if (cudaMalloc(&dev, hb * nbuf * (world_ + 1) + sizeof(double)) != cudaSuccess) return "share_buffers: cudaMalloc";
  char* dsend = (char*)dev;
  char* drecv = dsend + hb * nbuf;
  double* dflag = reinterpret_cast<double*>(drecv + hb * nbuf * world_);
  std::string err;
  double flag = bad;
  cudaError_t e = cudaMemcpyAsync(dflag, &flag, sizeof(double), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) err = c.allreduce_f64(dflag, 1, s);
  if (e == cudaSuccess && err.empty()) e = cudaMemcpyAsync(&flag, dflag, sizeof(double), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && err.empty()) e = cudaStreamSynchronize(s);
  if (e == cudaSuccess && err.empty() && flag == 0.0) {
    e = cudaMemcpyAsync(dsend, mine.data(), hb * nbuf, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) err = c.allgather_bytes(dsend, drecv, hb * nbuf, s);
    if (e == cudaSuccess && err.empty())
      e = cudaMemcpyAsync(every.data(), drecv, hb * nbuf * world_, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && err.empty()) e = cudaStreamSynchronize(s);
  }
  cudaFree(dev);
  if (e != cudaSuccess) return std::string("share_buffers: ") + cudaGetErrorString(e);
  if (!err.empty()) return err;
  if (flag != 0.0) return "share_buffers: cudaIpcGetMemHandle failed on some rank";
  all->assign((size_t)world_ * nbuf, nullptr);
  int open_bad = 0;
  for (int r = 0; r < world_; ++r)
    for (int b = 0; b < nbuf; ++b) {
      if (r == rank_) {
        (*all)[(size_t)r * nbuf + b] = local[b];
        continue;
      }
      void* ptr = nullptr;
      if (cudaIpcOpenMemHandle(&ptr, every[(size_t)r * nbuf + b], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        open_bad = 1;
        continue;
      }
      opened->push_back(ptr);
      (*all)[(size_t)r * nbuf + b] = ptr;
    }
  // collective verdict: every rank uses the peer window, or none does
  flag = open_bad;
  if (cudaMalloc(&dev, sizeof(double)) != cudaSuccess) return "share_buffers: cudaMalloc";
  e = cudaMemcpyAsync(dev, &flag, sizeof(double), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) err = c.allreduce_f64((double*)dev, 1, s);
  if (e == cudaSuccess && err.empty()) e = cudaMemcpyAsync(&flag, dev, sizeof(double), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && err.empty()) e = cudaStreamSynchronize(s);
  cudaFree(dev);
  if (e != cudaSuccess) return std::string("share_buffers: ") + cudaGetErrorString(e);
  if (!err.empty()) return err;
  if (flag != 0.0) return "share_buffers: cudaIpcOpenMemHandle failed on some rank (no peer access)";
  return "";
}

Comm* make_nccl_comm(const uint8_t* id128, int world, int rank, std::string* err) {
  ncclUniqueId id;
  memcpy(&id, id128, sizeof id);
  ncclComm_t c = nullptr;
  ncclResult_t r = ncclCommInitRank(&c, world, id, rank);
  if (r != ncclSuccess) {
    *err = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
    return nullptr;
  }
  return new NcclComm(c, world, rank);
}

bool nccl_unique_id(uint8_t* out128) {
  ncclUniqueId id;
  static_assert(sizeof(id) == 128, "nccl id size");
  if (ncclGetUniqueId(&id) != ncclSuccess) return false;
  memcpy(out128, &id, 128);
  return true;
}

// ---------------------------------------------------------------------------
// Host transport: device buffers are staged through pinned host memory around the
// caller's collectives (synchronous; test infrastructure).
class HostComm : public Comm {
 public:
  HostComm(const HostTransport& t, int world, int rank) : t_(t), world_(world), rank_(rank) {}
  ~HostComm() override {
    for (void* p : opened_) cudaIpcCloseMemHandle(p);
    if (h_) cudaFreeHost(h_);
  }
  const char* name() const override { return "host"; }

  std::string allreduce_f64(double* buf, size_t n, cudaStream_t s) override {
    if (n == 0) return "";
    std::string e = stage(n * sizeof(double));
    if (!e.empty()) return e;
    cudaError_t ce = cudaMemcpyAsync(h_, buf, n * sizeof(double), cudaMemcpyDeviceToHost, s);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
    if (ce != cudaSuccess) return std::string("host allreduce: ") + cudaGetErrorString(ce);
    if (t_.allreduce_f64(t_.user, (double*)h_, n) != 0) return "host allreduce: transport failed";
    ce = cudaMemcpyAsync(buf, h_, n * sizeof(double), cudaMemcpyHostToDevice, s);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
    return ce == cudaSuccess ? "" : std::string("host allreduce: ") + cudaGetErrorString(ce);
  }

  std::string allgather_bytes(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    std::string e = stage(bytes * (world_ + 1));
    if (!e.empty()) return e;
    char* hs = (char*)h_;
    char* hr = hs + bytes;
    cudaError_t ce = cudaMemcpyAsync(hs, send, bytes, cudaMemcpyDeviceToHost, s);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
    if (ce != cudaSuccess) return std::string("host allgather: ") + cudaGetErrorString(ce);
    if (t_.allgather_bytes(t_.user, hs, hr, bytes) != 0) return "host allgather: transport failed";
    ce = cudaMemcpyAsync(recv, hr, bytes * world_, cudaMemcpyHostToDevice, s);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
    return ce == cudaSuccess ? "" : std::string("host allgather: ") + cudaGetErrorString(ce);
  }

  // send/recv exchange through an all-gather of every rank's packed send segments
  // (padded to the largest; test transport, not a fast path)
  std::string exchange(float* const* src, float* const* dst, int narr, const ExchangePlan& p,
                       cudaStream_t s) override {
    int64_t mine = 0;
    for (int q = 0; q < world_; ++q) mine += p.send_count[q];
    std::vector<double> cnt(world_, 0.0);
    cnt[rank_] = (double)mine;
    if (t_.allreduce_f64(t_.user, cnt.data(), (size_t)world_) != 0) return "host exchange: transport failed";
    int64_t mx = 0;
    for (int q = 0; q < world_; ++q) mx = std::max<int64_t>(mx, (int64_t)cnt[q]);
    // packed per rank: [counts world][offsets world] int64 header + narr arrays of mx floats
    const size_t hdr = sizeof(int64_t) * 2 * world_, per = hdr + sizeof(float) * narr * (size_t)mx;
    std::vector<char> send(per, 0), recv(per * world_, 0);
    int64_t* hc = reinterpret_cast<int64_t*>(send.data());
    float* hv = reinterpret_cast<float*>(send.data() + hdr);
    int64_t at = 0;
    cudaError_t ce = cudaSuccess;
    for (int q = 0; q < world_; ++q) {
      hc[q] = p.send_count[q];
      hc[world_ + q] = at;
      for (int i = 0; i < narr && ce == cudaSuccess && p.send_count[q] > 0; ++i)
        ce = cudaMemcpyAsync(hv + (size_t)i * mx + at, src[i] + p.send_off[q], sizeof(float) * p.send_count[q],
                             cudaMemcpyDeviceToHost, s);
      at += p.send_count[q];
    }
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
    if (ce != cudaSuccess) return std::string("host exchange: ") + cudaGetErrorString(ce);
    if (t_.allgather_bytes(t_.user, send.data(), recv.data(), per) != 0) return "host exchange: transport failed";
    for (int q = 0; q < world_ && ce == cudaSuccess; ++q) {
      if (q == rank_ || p.recv_count[q] <= 0) continue;
      const char* blk = recv.data() + per * q;
      const int64_t* rc = reinterpret_cast<const int64_t*>(blk);
      const float* rv = reinterpret_cast<const float*>(blk + hdr);
      if (rc[rank_] != p.recv_count[q]) return "host exchange: plan mismatch";
      for (int i = 0; i < narr && ce == cudaSuccess; ++i)
        ce = cudaMemcpyAsync(dst[i] + p.recv_off[q], rv + (size_t)i * mx + rc[world_ + rank_],
                             sizeof(float) * p.recv_count[q], cudaMemcpyHostToDevice, s);
    }
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
    return ce == cudaSuccess ? "" : std::string("host exchange: ") + cudaGetErrorString(ce);
  }

  std::string share_buffers(void* const* local, int nbuf, std::vector<void*>* all, cudaStream_t s) override {
    return ipc_share_buffers(*this, world_, rank_, local, nbuf, all, &opened_, s);
  }

 private:
  std::string stage(size_t bytes) {
    if (bytes <= hn_) return "";
    if (h_) cudaFreeHost(h_);
    h_ = nullptr;
    if (cudaMallocHost(&h_, bytes) != cudaSuccess) return "host transport: cudaMallocHost";
    hn_ = bytes;
    return "";
  }
  HostTransport t_;
  int world_, rank_;
  void* h_ = nullptr;
  size_t hn_ = 0;
  std::vector<void*> opened_;
};

Comm* make_host_comm(const HostTransport& t, int world, int rank, std::string* err) {
  if (!t.allreduce_f64 || !t.allgather_bytes || world < 1 || rank < 0 || rank >= world) {
    *err = "bad host transport";
    return nullptr;
  }
  return new HostComm(t, world, rank);
}

// ---------------------------------------------------------------------------
struct LocalGroup {
  int world;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  int64_t generation = 0;
  std::vector<double*> bufs;
  std::vector<std::vector<float*>> srcs;
  std::vector<ExchangePlan> plans;
  std::vector<const void*> gsrc;
  std::vector<std::vector<void*>> shared;
  std::vector<int> dev;

  explicit LocalGroup(int w)
      : world(w), bufs(w, nullptr), srcs(w), plans(w), gsrc(w, nullptr), shared(w), dev(w, -1) {}

  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    int64_t gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

LocalGroup* local_group_create(int world) { return world >= 1 ? new LocalGroup(world) : nullptr; }
void local_group_destroy(LocalGroup* g) { delete g; }
int local_group_world(const LocalGroup* g) { return g ? g->world : 0; }

class LocalComm : public Comm {
 public:
  LocalComm(LocalGroup* g, int rank, int device) : g_(g), rank_(rank) { g_->dev[rank] = device; }
  ~LocalComm() override {
    if (tmp_) cudaFree(tmp_);
  }
  const char* name() const override { return "local"; }

  // Called after a barrier (every rank has registered its device): kernels of this
  // rank read / write the other ranks' buffers, so ranks on other GPUs need peer access.
  std::string peers() {
    if (peers_done_) return "";
    peers_done_ = true;
    int me = g_->dev[rank_];
    for (int r = 0; r < g_->world; ++r) {
      int d = g_->dev[r];
      if (d == me || d < 0) continue;
      int can = 0;
      if (cudaDeviceCanAccessPeer(&can, me, d) != cudaSuccess || !can)
        return "local group: device " + std::to_string(me) + " has no peer access to device " + std::to_string(d);
      cudaError_t e = cudaDeviceEnablePeerAccess(d, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
      } else if (e != cudaSuccess) {
        return std::string("local group: cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e);
      }
    }
    return "";
  }

  std::string allreduce_f64(double* buf, size_t n, cudaStream_t s) override {
    if (n > tmp_n_) {
      if (tmp_) cudaFree(tmp_);
      if (cudaMalloc(&tmp_, n * sizeof(double)) != cudaSuccess) return "local allreduce: cudaMalloc failed";
      tmp_n_ = n;
    }
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cudaGetErrorString(e);
    g_->bufs[rank_] = buf;
    g_->barrier();
    {
      std::string pe = peers();
      if (!pe.empty()) {
        g_->barrier();
        return pe;
      }
    }
    // every rank sums all ranks' buffers in rank order (identical bits on every rank)
    if (n) {
      e = launch_sum_ranks(g_->bufs.data(), g_->world, tmp_, n, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    }
    g_->barrier();  // all reads of the peers' buffers are done
    if (n && e == cudaSuccess) e = cudaMemcpyAsync(buf, tmp_, n * sizeof(double), cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    return e == cudaSuccess ? "" : std::string("local allreduce: ") + cudaGetErrorString(e);
  }

  std::string exchange(float* const* src, float* const* dst, int narr, const ExchangePlan& p,
                       cudaStream_t s) override {
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cudaGetErrorString(e);
    g_->srcs[rank_].assign(src, src + narr);
    g_->plans[rank_] = p;
    g_->barrier();
    {
      std::string pe = peers();
      if (!pe.empty()) {
        g_->barrier();
        return pe;
      }
    }
    for (int q = 0; q < g_->world && e == cudaSuccess; ++q) {
      if (q == rank_ || p.recv_count[q] <= 0) continue;
      int64_t off = g_->plans[q].send_off[rank_];
      for (int i = 0; i < narr && e == cudaSuccess; ++i)
        e = cudaMemcpyAsync(dst[i] + p.recv_off[q], g_->srcs[q][i] + off, sizeof(float) * p.recv_count[q],
                            cudaMemcpyDeviceToDevice, s);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    g_->barrier();  // peers may reuse their source buffers only after every pull
    return e == cudaSuccess ? "" : std::string("local exchange: ") + cudaGetErrorString(e);
  }

  std::string share_buffers(void* const* local, int nbuf, std::vector<void*>* all, cudaStream_t s) override {
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cudaGetErrorString(e);
    g_->shared[rank_].assign(local, local + nbuf);
    g_->barrier();
    {
      std::string pe = peers();
      if (!pe.empty()) {
        g_->barrier();
        return pe;
      }
    }
    all->clear();
    bool null = false;
    for (int r = 0; r < g_->world; ++r) {
      all->insert(all->end(), g_->shared[r].begin(), g_->shared[r].end());
      for (void* p : g_->shared[r]) null = null || p == nullptr;
    }
    g_->barrier();
    return null ? "local share_buffers: a rank has no buffer" : "";  // same verdict on every rank
  }

  std::string allgather_bytes(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cudaGetErrorString(e);
    g_->gsrc[rank_] = send;
    g_->barrier();
    {
      std::string pe = peers();
      if (!pe.empty()) {
        g_->barrier();
        return pe;
      }
    }
    for (int r = 0; r < g_->world && e == cudaSuccess; ++r)
      e = cudaMemcpyAsync((char*)recv + r * bytes, g_->gsrc[r], bytes, cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    g_->barrier();
    return e == cudaSuccess ? "" : std::string("local allgather: ") + cudaGetErrorString(e);
  }

 private:
  LocalGroup* g_;
  int rank_;
  double* tmp_ = nullptr;
  size_t tmp_n_ = 0;
  bool peers_done_ = false;
};

Comm* make_local_comm(LocalGroup* g, int rank, int device, std::string* err) {
  if (!g || rank < 0 || rank >= g->world) {
    *err = "bad local group / rank";
    return nullptr;
  }
  return new LocalComm(g, rank, device);
}

}  // namespace phd
