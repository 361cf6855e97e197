// Collective transport for the multi-rank step.
//   NcclComm  : one process per GPU, NCCL over NVLink/NVSwitch (the product path).
//   LocalComm : a group of rank contexts inside one process (one host thread per
//               rank, host barriers, device-to-device copies).  Used to run the
//               library's multi-rank orchestration on a single GPU in the tests;
//               ranks never wait on one another inside a kernel.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

namespace phd {

struct ExchangePlan {
  std::vector<int64_t> send_count, send_off, recv_count, recv_off;
};

class Comm {
 public:
  virtual ~Comm() {}
  virtual const char* name() const = 0;
  // In-place fp64 sum over all ranks, ordered on stream s.  Returns "" or an error.
  virtual std::string allreduce_f64(double* buf, size_t n, cudaStream_t s) = 0;
  // Peer transfers of the plan (the rank's own segment is copied by the caller):
  // narr float arrays; send src[i] + send_off[q] (send_count[q] items) to rank q,
  // receive into dst[i] + recv_off[q] (recv_count[q] items) from rank q.
  virtual std::string exchange(float* const* src, float* const* dst, int narr, const ExchangePlan& p,
                               cudaStream_t s) = 0;
  // recv[r * bytes .. ) = rank r's send[0 .. bytes) for every rank r (device buffers).
  virtual std::string allgather_bytes(const void* send, void* recv, size_t bytes, cudaStream_t s) = 0;
  // Peer-memory window for the fused resample + exchange: every rank registers nbuf
  // device buffers (cudaMalloc allocations of its own); all[r * nbuf + b] receives
  // rank r's buffer b as a pointer this rank's kernels can store to.  NCCL transport:
  // CUDA IPC handles all-gathered and opened with peer access (NVLink / NVSwitch);
  // in-process group: the pointers themselves.  Collective.  "" or an error (the
  // caller then keeps the NCCL send/recv exchange).
  virtual std::string share_buffers(void* const* local, int nbuf, std::vector<void*>* all, cudaStream_t s) = 0;
};

// CUDA IPC peer window shared by any transport: handles of the local buffers are
// all-gathered with c.allgather_bytes, the peers' opened (collective verdicts through
// c.allreduce_f64, so every rank takes the same path).  Opened pointers are appended to
// *opened (the caller closes them).
std::string ipc_share_buffers(Comm& c, int world, int rank, void* const* local, int nbuf, std::vector<void*>* all,
                              std::vector<void*>* opened, cudaStream_t s);

Comm* make_nccl_comm(const uint8_t* id128, int world, int rank, std::string* err);

// Host transport (test infrastructure for the multi-process path on one GPU): the
// collectives go through caller callbacks on HOST buffers; the data path (IPC peer
// window, P2P stores, kernels) is the product's.
struct HostTransport {
  void* user;
  int (*allreduce_f64)(void* user, double* buf, size_t n);
  int (*allgather_bytes)(void* user, const void* send, void* recv, size_t bytes);
};
Comm* make_host_comm(const HostTransport& t, int world, int rank, std::string* err);
bool nccl_unique_id(uint8_t* out128);

struct LocalGroup;
LocalGroup* local_group_create(int world);
void local_group_destroy(LocalGroup* g);
int local_group_world(const LocalGroup* g);
// device: the rank's GPU; ranks of one group on different GPUs get peer access
// (or the first collective fails with an error).
Comm* make_local_comm(LocalGroup* g, int rank, int device, std::string* err);

cudaError_t launch_sum_ranks(const double* const* srcs, int world, double* dst, size_t n, cudaStream_t s);

}  // namespace phd
