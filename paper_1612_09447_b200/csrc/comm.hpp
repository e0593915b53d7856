// Collectives of the distributed path: fp64 allreduce of
// reduction slots and halo exchange of ghost entries. Three backends:
//  * SelfComm   — one rank, everything is a no-op;
//  * NcclComm   — one process per GPU, NCCL over NVLink/NVSwitch, enqueued on
//                 the context stream (graph-capturable, no host sync);
//  * ThreadComm — P "virtual ranks" (threads) in one process, partitions on
//                 any devices, exchange by device-to-device copies with host
//                 barriers. Used to test the partitioned algorithm on one GPU.
//  * ShmComm    — P processes on one node, host-staged through a POSIX shared
//                 memory segment (process-shared atomics for the barrier).
//                 Not capturable; runs where NCCL cannot (several ranks on one
//                 GPU, no GPU at all for the host-buffer test entry points).
//                 Allreduces sum in rank order, like ThreadComm, so the two
//                 give bit-identical results.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace eqsb {

struct HaloMsg {
  int peer;
  const void* send;    // device
  int send_count;      // elements
  void* recv;          // device
  int recv_count;
  int elem_bytes = 8;  // 8: fp64 vectors, 4: fp32 (V-cycle) vectors
};

class Comm {
 public:
  virtual ~Comm() = default;
  virtual int rank() const = 0;
  virtual int size() const = 0;
  virtual bool capturable() const = 0;  // may be recorded into a CUDA graph
  // in-place sum over ranks of `count` doubles in device memory
  virtual void allreduce(double* dev, int count, cudaStream_t s) = 0;
  virtual void allreduce(float* dev, int count, cudaStream_t s) = 0;
  // point-to-point exchange: every message's send buffer goes to `peer`,
  // every recv buffer is filled from `peer` (pairs must match on both sides)
  virtual void exchange(const std::vector<HaloMsg>& msgs, cudaStream_t s) = 0;
  virtual void barrier() = 0;
};

class SelfComm final : public Comm {
 public:
  int rank() const override { return 0; }
  int size() const override { return 1; }
  bool capturable() const override { return true; }
  void allreduce(double*, int, cudaStream_t) override {}
  void allreduce(float*, int, cudaStream_t) override {}
  void exchange(const std::vector<HaloMsg>&, cudaStream_t) override {}
  void barrier() override {}
};

// rank/size only, for host-only contexts that build a rank's partition plan
// without a device (any collective throws)
class StaticComm final : public Comm {
 public:
  StaticComm(int rank, int size) : rank_(rank), size_(size) {}
  int rank() const override { return rank_; }
  int size() const override { return size_; }
  bool capturable() const override { return false; }
  void allreduce(double*, int, cudaStream_t) override { throw std::logic_error("StaticComm: no collectives"); }
  void allreduce(float*, int, cudaStream_t) override { throw std::logic_error("StaticComm: no collectives"); }
  void exchange(const std::vector<HaloMsg>&, cudaStream_t) override {
    throw std::logic_error("StaticComm: no collectives");
  }
  void barrier() override {}

 private:
  int rank_, size_;
};

// shared state of a virtual-rank group (one per group, shared by its ranks)
struct ThreadGroup;
std::shared_ptr<ThreadGroup> make_thread_group(int nranks);
std::unique_ptr<Comm> make_thread_comm(std::shared_ptr<ThreadGroup> g, int rank);

// host-staged multi-process backend; every rank passes the same segment name
// (rank 0 creates it, all ranks attach, rank 0 unlinks once all attached)
std::unique_ptr<Comm> make_shm_comm(const std::string& name, int nranks, int rank);
// the same transport on host buffers (CPU tests of the exchange protocol)
void shm_allreduce_host(Comm& c, double* buf, int count);
void shm_exchange_host(Comm& c, const std::vector<HaloMsg>& msgs);

// NCCL: id is the 128-byte ncclUniqueId from nccl_unique_id() on rank 0
std::string nccl_unique_id();
std::unique_ptr<Comm> make_nccl_comm(const std::string& id, int nranks, int rank);

}  // namespace eqsb
