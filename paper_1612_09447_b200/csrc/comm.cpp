#include "comm.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <stdexcept>

#include "eqs_internal.hpp"

namespace eqsb {

namespace {
void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// NCCL is resolved at first use with dlopen("libnccl.so.2"): inside a process
// that already loaded PyTorch this binds to torch's NCCL (same soname), and a
// process that never goes multi-GPU never loads NCCL at all (linking it
// directly would pin the system NCCL before torch and break torch's import).
struct Nccl {
  const char* (*GetErrorString)(ncclResult_t);
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
};
const Nccl& nccl() {
  static Nccl api = [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw CudaError(std::string("cannot load libnccl.so.2: ") + dlerror());
    Nccl a{};
    auto sym = [&](const char* n) {
      void* p = dlsym(h, n);
      if (!p) throw CudaError(std::string("libnccl.so.2 lacks ") + n);
      return p;
    };
    a.GetErrorString = (const char* (*)(ncclResult_t))sym("ncclGetErrorString");
    a.GetUniqueId = (ncclResult_t(*)(ncclUniqueId*))sym("ncclGetUniqueId");
    a.CommInitRank = (ncclResult_t(*)(ncclComm_t*, int, ncclUniqueId, int))sym("ncclCommInitRank");
    a.CommDestroy = (ncclResult_t(*)(ncclComm_t))sym("ncclCommDestroy");
    a.AllReduce = (ncclResult_t(*)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                   cudaStream_t))sym("ncclAllReduce");
    a.GroupStart = (ncclResult_t(*)())sym("ncclGroupStart");
    a.GroupEnd = (ncclResult_t(*)())sym("ncclGroupEnd");
    a.Send = (ncclResult_t(*)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t))sym("ncclSend");
    a.Recv = (ncclResult_t(*)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t))sym("ncclRecv");
    return a;
  }();
  return api;
}
void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw CudaError(std::string(what) + ": " + nccl().GetErrorString(r));
}
}  // namespace

// ------------------------------------------------------------------ virtual ranks
struct ThreadGroup {
  int n;
  std::mutex mu;
  std::condition_variable cv;
  long generation = 0;
  int waiting = 0;
  std::vector<std::vector<double>> partial;
  std::vector<std::vector<HaloMsg>> posted;
  explicit ThreadGroup(int nranks) : n(nranks), partial(nranks), posted(nranks) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long gen = generation;
    if (++waiting == n) {
      waiting = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

std::shared_ptr<ThreadGroup> make_thread_group(int nranks) { return std::make_shared<ThreadGroup>(nranks); }

namespace {
class ThreadComm final : public Comm {
 public:
  ThreadComm(std::shared_ptr<ThreadGroup> g, int rank) : g_(std::move(g)), rank_(rank) {}
  int rank() const override { return rank_; }
  int size() const override { return g_->n; }
  bool capturable() const override { return false; }
  void barrier() override { g_->barrier(); }
  // deterministic: every rank sums the contributions in rank order
  void allreduce(double* dev, int count, cudaStream_t s) override { sum_in_rank_order(dev, count, s); }
  void allreduce(float* dev, int count, cudaStream_t s) override { sum_in_rank_order(dev, count, s); }
  template <class T>
  void sum_in_rank_order(T* dev, int count, cudaStream_t s) {
    std::vector<double>& mine = g_->partial[rank_];
    std::vector<T> buf(count);
    ck(cudaMemcpyAsync(buf.data(), dev, sizeof(T) * count, cudaMemcpyDeviceToHost, s), "allreduce d2h");
    ck(cudaStreamSynchronize(s), "allreduce sync");
    mine.assign(buf.begin(), buf.end());
    g_->barrier();
    std::vector<T> sum(count, T(0));
    for (int r = 0; r < g_->n; ++r)
      for (int i = 0; i < count; ++i) sum[i] += (T)g_->partial[r][i];
    g_->barrier();
    ck(cudaMemcpyAsync(dev, sum.data(), sizeof(T) * count, cudaMemcpyHostToDevice, s), "allreduce h2d");
    ck(cudaStreamSynchronize(s), "allreduce sync");
  }
  void exchange(const std::vector<HaloMsg>& msgs, cudaStream_t s) override {
    ck(cudaStreamSynchronize(s), "exchange sync");  // send buffers complete
    g_->posted[rank_] = msgs;
    g_->barrier();
    for (const HaloMsg& m : msgs) {
      if (m.recv_count == 0) continue;
      const HaloMsg* src = nullptr;
      for (const HaloMsg& o : g_->posted[m.peer])
        if (o.peer == rank_) src = &o;
      if (!src || src->send_count != m.recv_count) throw std::logic_error("thread comm: unmatched halo message");
      ck(cudaMemcpyAsync(m.recv, src->send, (size_t)m.elem_bytes * m.recv_count, cudaMemcpyDefault, s), "halo copy");
    }
    ck(cudaStreamSynchronize(s), "exchange sync");
    g_->barrier();  // peers may reuse their send buffers now
  }

 private:
  std::shared_ptr<ThreadGroup> g_;
  int rank_;
};

// ------------------------------------------------------------------ NCCL
class NcclComm final : public Comm {
 public:
  NcclComm(const std::string& id, int nranks, int rank) : n_(nranks), rank_(rank) {
    ncclUniqueId uid;
    if (id.size() != sizeof(uid.internal)) throw std::invalid_argument("nccl unique id must be 128 bytes");
    std::memcpy(uid.internal, id.data(), sizeof(uid.internal));
    nck(nccl().CommInitRank(&comm_, nranks, uid, rank), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm_) nccl().CommDestroy(comm_);
  }
  int rank() const override { return rank_; }
  int size() const override { return n_; }
  bool capturable() const override { return true; }
  void barrier() override {
    // a zero-byte allreduce on the default stream orders all ranks
    double* d = nullptr;
    ck(cudaMalloc(&d, sizeof(double)), "barrier alloc");
    nck(nccl().AllReduce(d, d, 1, ncclDouble, ncclSum, comm_, 0), "barrier");
    ck(cudaStreamSynchronize(0), "barrier sync");
    cudaFree(d);
  }
  void allreduce(float* dev, int count, cudaStream_t s) override {
    nck(nccl().AllReduce(dev, dev, count, ncclFloat, ncclSum, comm_, s), "ncclAllReduce");
  }
  void allreduce(double* dev, int count, cudaStream_t s) override {
    nck(nccl().AllReduce(dev, dev, count, ncclDouble, ncclSum, comm_, s), "ncclAllReduce");
  }
  void exchange(const std::vector<HaloMsg>& msgs, cudaStream_t s) override {
    nck(nccl().GroupStart(), "ncclGroupStart");
    for (const HaloMsg& m : msgs) {
      const ncclDataType_t t = m.elem_bytes == 4 ? ncclFloat : ncclDouble;
      if (m.send_count > 0) nck(nccl().Send(m.send, m.send_count, t, m.peer, comm_, s), "ncclSend");
      if (m.recv_count > 0) nck(nccl().Recv(m.recv, m.recv_count, t, m.peer, comm_, s), "ncclRecv");
    }
    nck(nccl().GroupEnd(), "ncclGroupEnd");
  }

 private:
  int n_, rank_;
  ncclComm_t comm_ = nullptr;
};
}  // namespace

std::unique_ptr<Comm> make_thread_comm(std::shared_ptr<ThreadGroup> g, int rank) {
  return std::make_unique<ThreadComm>(std::move(g), rank);
}

std::string nccl_unique_id() {
  ncclUniqueId uid;
  nck(nccl().GetUniqueId(&uid), "ncclGetUniqueId");
  return std::string(uid.internal, sizeof(uid.internal));
}

std::unique_ptr<Comm> make_nccl_comm(const std::string& id, int nranks, int rank) {
  return std::make_unique<NcclComm>(id, nranks, rank);
}

}  // namespace eqsb
