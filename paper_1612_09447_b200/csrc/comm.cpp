#include "comm.hpp"

#include <dlfcn.h>
#include <fcntl.h>
#include <nccl.h>
#include <sched.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <thread>

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
    if (scratch_) cudaFree(scratch_);
    if (bstream_) cudaStreamDestroy(bstream_);
  }
  int rank() const override { return rank_; }
  int size() const override { return n_; }
  bool capturable() const override { return true; }
  void barrier() override {
    // an allreduce of one zeroed scratch double on a private stream orders all
    // ranks (scratch and stream live as long as the communicator)
    if (!scratch_) {
      ck(cudaStreamCreateWithFlags(&bstream_, cudaStreamNonBlocking), "barrier stream");
      ck(cudaMalloc(&scratch_, sizeof(double)), "barrier alloc");
    }
    ck(cudaMemsetAsync(scratch_, 0, sizeof(double), bstream_), "barrier memset");
    nck(nccl().AllReduce(scratch_, scratch_, 1, ncclDouble, ncclSum, comm_, bstream_), "barrier");
    ck(cudaStreamSynchronize(bstream_), "barrier sync");
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
  double* scratch_ = nullptr;
  cudaStream_t bstream_ = nullptr;
};

// ------------------------------------------------------------------ shared memory (host-staged)
// Segment: header, then per rank a slot = {reduce area, message table, outbox}.
// A rank writes only its own slot and reads its peers' slots between barriers.
constexpr int kShmMagic = 0x45515342;  // "EQSB"
constexpr int kShmMaxRanks = 64;
constexpr int kShmReduce = 256;                  // doubles per allreduce
constexpr size_t kShmOutbox = size_t(64) << 20;  // bytes of halo payload per rank
struct ShmHeader {
  std::atomic<int> magic;
  std::atomic<int> attached;
  std::atomic<int> arrived;
  std::atomic<long> generation;
  int nranks;
};
struct ShmEntry {
  int peer, count, elem_bytes;
  long offset;
};
struct ShmSlot {
  double reduce[kShmReduce];
  int n_entries;
  ShmEntry entries[kShmMaxRanks];
};
static_assert(std::atomic<int>::is_always_lock_free && std::atomic<long>::is_always_lock_free,
              "process-shared atomics must be lock-free");

class ShmComm final : public Comm {
 public:
  ShmComm(const std::string& name, int nranks, int rank) : n_(nranks), rank_(rank), name_(name) {
    if (nranks < 1 || nranks > kShmMaxRanks || rank < 0 || rank >= nranks)
      throw std::invalid_argument("shm comm: bad rank/size");
    bytes_ = header_bytes() + (size_t)nranks * slot_bytes();
    int fd = -1;
    if (rank == 0) {
      fd = shm_open(name.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
      if (fd < 0) throw CudaError("shm comm: cannot create segment " + name);
      if (ftruncate(fd, (off_t)bytes_) != 0) {
        close(fd);
        shm_unlink(name.c_str());
        throw CudaError("shm comm: cannot size segment");
      }
    } else {
      const auto t0 = std::chrono::steady_clock::now();
      while ((fd = shm_open(name.c_str(), O_RDWR, 0600)) < 0) {
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120))
          throw CudaError("shm comm: segment " + name + " never appeared");
        std::this_thread::sleep_for(std::chrono::milliseconds(2));
      }
      // wait until rank 0 has sized it
      for (;;) {
        off_t sz = lseek(fd, 0, SEEK_END);
        if (sz >= (off_t)bytes_) break;
        std::this_thread::sleep_for(std::chrono::milliseconds(2));
      }
    }
    base_ = (char*)mmap(nullptr, bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (base_ == MAP_FAILED) throw CudaError("shm comm: mmap failed");
    hdr_ = reinterpret_cast<ShmHeader*>(base_);
    if (rank == 0) {
      new (&hdr_->attached) std::atomic<int>(0);
      new (&hdr_->arrived) std::atomic<int>(0);
      new (&hdr_->generation) std::atomic<long>(0);
      hdr_->nranks = nranks;
      hdr_->magic.store(kShmMagic, std::memory_order_release);
    } else {
      while (hdr_->magic.load(std::memory_order_acquire) != kShmMagic) std::this_thread::yield();
      if (hdr_->nranks != nranks) throw CudaError("shm comm: rank count mismatch");
    }
    hdr_->attached.fetch_add(1);
    barrier();
    if (rank == 0) shm_unlink(name.c_str());  // everyone is attached: no leak if a rank dies
    // page-lock the mapping so device copies go straight to it (best effort)
    registered_ = cudaHostRegister(base_, bytes_, cudaHostRegisterDefault) == cudaSuccess;
    if (!registered_) cudaGetLastError();
  }
  ~ShmComm() override {
    if (registered_) cudaHostUnregister(base_);
    if (base_) munmap(base_, bytes_);
  }
  int rank() const override { return rank_; }
  int size() const override { return n_; }
  bool capturable() const override { return false; }

  // sense-free generation barrier on process-shared atomics
  void barrier() override {
    const long gen = hdr_->generation.load(std::memory_order_acquire);
    if (hdr_->arrived.fetch_add(1, std::memory_order_acq_rel) + 1 == n_) {
      hdr_->arrived.store(0, std::memory_order_relaxed);
      hdr_->generation.fetch_add(1, std::memory_order_acq_rel);
    } else {
      int spins = 0;
      while (hdr_->generation.load(std::memory_order_acquire) == gen) {
        if (++spins > 1000) sched_yield();
      }
    }
  }

  void allreduce(double* dev, int count, cudaStream_t s) override { reduce(dev, count, s, false); }
  void allreduce(float* dev, int count, cudaStream_t s) override { reduce(dev, count, s, false); }
  void exchange(const std::vector<HaloMsg>& msgs, cudaStream_t s) override { swap(msgs, s, false); }
  void allreduce_host(double* buf, int count) { reduce(buf, count, nullptr, true); }
  void exchange_host(const std::vector<HaloMsg>& msgs) { swap(msgs, nullptr, true); }

 private:
  static size_t header_bytes() { return (sizeof(ShmHeader) + 4095) / 4096 * 4096; }
  static size_t slot_bytes() { return (sizeof(ShmSlot) + 4095) / 4096 * 4096 + kShmOutbox; }
  ShmSlot* slot(int r) const { return reinterpret_cast<ShmSlot*>(base_ + header_bytes() + (size_t)r * slot_bytes()); }
  char* outbox(int r) const { return reinterpret_cast<char*>(slot(r)) + (sizeof(ShmSlot) + 4095) / 4096 * 4096; }

  void copy(void* dst, const void* src, size_t bytes, bool host, cudaStream_t s) {
    if (host) std::memcpy(dst, src, bytes);
    else ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s), "shm comm copy");
  }
  void sync(bool host, cudaStream_t s) {
    if (!host) ck(cudaStreamSynchronize(s), "shm comm sync");
  }

  // every rank sums the slots in rank order: identical on all ranks and
  // identical to ThreadComm's virtual-rank sum
  template <class T>
  void reduce(T* buf, int count, cudaStream_t s, bool host) {
    if (count > kShmReduce) throw std::logic_error("shm comm: allreduce too large");
    std::vector<T> mine(count), sum(count, T(0));
    copy(mine.data(), buf, sizeof(T) * count, host, s);
    sync(host, s);
    for (int i = 0; i < count; ++i) slot(rank_)->reduce[i] = (double)mine[i];
    barrier();
    for (int r = 0; r < n_; ++r)
      for (int i = 0; i < count; ++i) sum[i] += (T)slot(r)->reduce[i];
    barrier();  // slots may be overwritten by the next call
    copy(buf, sum.data(), sizeof(T) * count, host, s);
    sync(host, s);
  }

  void swap(const std::vector<HaloMsg>& msgs, cudaStream_t s, bool host) {
    ShmSlot* me = slot(rank_);
    if (msgs.size() > (size_t)kShmMaxRanks) throw std::logic_error("shm comm: too many peers");
    long off = 0;
    me->n_entries = 0;
    for (const HaloMsg& m : msgs) {
      const size_t b = (size_t)m.elem_bytes * m.send_count;
      if (off + (long)b > (long)kShmOutbox) throw std::logic_error("shm comm: halo larger than the outbox");
      if (b) copy(outbox(rank_) + off, m.send, b, host, s);
      me->entries[me->n_entries++] = {m.peer, m.send_count, m.elem_bytes, off};
      off += (long)((b + 255) / 256 * 256);
    }
    sync(host, s);
    barrier();
    for (const HaloMsg& m : msgs) {
      if (m.recv_count == 0) continue;
      const ShmSlot* src = slot(m.peer);
      const ShmEntry* e = nullptr;
      for (int k = 0; k < src->n_entries; ++k)
        if (src->entries[k].peer == rank_) e = &src->entries[k];
      if (!e || e->count != m.recv_count || e->elem_bytes != m.elem_bytes)
        throw std::logic_error("shm comm: unmatched halo message");
      copy(m.recv, outbox(m.peer) + e->offset, (size_t)m.elem_bytes * m.recv_count, host, s);
    }
    sync(host, s);
    barrier();  // outboxes may be reused now
  }

  int n_, rank_;
  std::string name_;
  size_t bytes_ = 0;
  char* base_ = nullptr;
  ShmHeader* hdr_ = nullptr;
  bool registered_ = false;
};
}  // namespace

std::unique_ptr<Comm> make_shm_comm(const std::string& name, int nranks, int rank) {
  return std::make_unique<ShmComm>(name, nranks, rank);
}
void shm_allreduce_host(Comm& c, double* buf, int count) {
  auto* s = dynamic_cast<ShmComm*>(&c);
  if (!s) throw std::invalid_argument("not a shared-memory communicator");
  s->allreduce_host(buf, count);
}
void shm_exchange_host(Comm& c, const std::vector<HaloMsg>& msgs) {
  auto* s = dynamic_cast<ShmComm*>(&c);
  if (!s) throw std::invalid_argument("not a shared-memory communicator");
  s->exchange_host(msgs);
}

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
