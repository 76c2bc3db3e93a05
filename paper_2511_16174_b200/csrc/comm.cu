// Communicators of the blockwise multi-GPU EVD: PeerComm (one process, peer copies) and
// NcclComm (one process per GPU, NCCL).  See comm.h.
#include <dlfcn.h>
#include <nccl.h>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <ctime>
#include "comm.h"

namespace pevd {

// ================================================================= PeerWorld / PeerComm

PeerWorld::PeerWorld(int G_, const int* devs) : G(G_), dev(devs, devs + G_), ptr(G_), ready(G_),
                                                done(G_) {
  // NVLink peer access between every pair of distinct devices (ignored where unsupported: the
  // copies then stage through the host, still correct)
  int cur = 0;
  cudaGetDevice(&cur);
  for (int i = 0; i < G; ++i)
    for (int j = 0; j < G; ++j) {
      if (dev[i] == dev[j]) continue;
      int ok = 0;
      cudaDeviceCanAccessPeer(&ok, dev[i], dev[j]);
      if (!ok) continue;
      cudaSetDevice(dev[i]);
      if (cudaDeviceEnablePeerAccess(dev[j], 0) != cudaSuccess) cudaGetLastError();
    }
  cudaSetDevice(cur);
}

PeerWorld::~PeerWorld() {
  if (base_ev) cudaEventDestroy(base_ev);
}

static double comm_mono_ns() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec * 1e9 + (double)ts.tv_nsec;
}

cudaEvent_t Comm::time_base(cudaEvent_t mine, cudaStream_t st, double& t0_ns) {
  cudaEventRecord(mine, st);
  t0_ns = comm_mono_ns();
  return mine;
}

cudaEvent_t PeerComm::time_base(cudaEvent_t mine, cudaStream_t st, double& t0_ns) {
  bool same = true;
  for (int x = 0; x < size_; ++x) same = same && w_->dev[x] == w_->dev[0];
  if (size_ == 1 || !same) return Comm::time_base(mine, st, t0_ns);
  if (rank_ == 0) {
    if (!w_->base_ev) cudaEventCreate(&w_->base_ev);
    cudaEventRecord(w_->base_ev, st);
    w_->base_t0 = comm_mono_ns();
  }
  if (!w_->rendezvous()) return Comm::time_base(mine, st, t0_ns);
  if (rank_ != 0) cudaStreamWaitEvent(st, w_->base_ev, 0);
  t0_ns = w_->base_t0;
  return w_->base_ev;
}

bool PeerWorld::rendezvous() {
  std::unique_lock<std::mutex> lk(mu);
  if (aborted.load()) return false;
  const int64_t gen = generation.load();
  if (++arrived == G) {
    arrived = 0;
    generation.store(gen + 1);
    lk.unlock();
    cv.notify_all();
    return true;
  }
  lk.unlock();
  // the hand-off is short (the other ranks are enqueueing the same collective): spin on the
  // generation before sleeping on the condition variable
  for (int spin = 0; spin < 200000; ++spin) {
    if (generation.load(std::memory_order_acquire) != gen) return true;
    if (aborted.load(std::memory_order_relaxed)) return false;
    if ((spin & 63) == 63) std::this_thread::yield();
  }
  lk.lock();
  cv.wait(lk, [&] { return generation.load() != gen || aborted.load(); });
  return !aborted.load();
}

void PeerWorld::abort() {
  {
    std::lock_guard<std::mutex> g(mu);
    aborted.store(true);
  }
  cv.notify_all();
}

PeerComm::PeerComm(PeerWorld* w, int rank) : w_(w) {
  rank_ = rank;
  size_ = w->G;
  cudaEventCreateWithFlags(&w_->ready[rank], cudaEventDisableTiming);
  cudaEventCreateWithFlags(&w_->done[rank], cudaEventDisableTiming);
  const char* e = getenv("PEVD_PEER_SERIAL");
  serialize_ = e && e[0] == '1';
  if (serialize_) cudaEventCreateWithFlags(&serial_, cudaEventDisableTiming);
}

PeerComm::~PeerComm() {
  if (w_->ready[rank_]) cudaEventDestroy(w_->ready[rank_]);
  if (w_->done[rank_]) cudaEventDestroy(w_->done[rank_]);
  w_->ready[rank_] = w_->done[rank_] = nullptr;
  if (serial_) cudaEventDestroy(serial_);
}

void PeerComm::serial_begin(cudaStream_t st, bool involved) {
  if (serialize_ && involved && serial_live_) cudaStreamWaitEvent(st, serial_, 0);
}

void PeerComm::serial_end(cudaStream_t st, bool involved) {
  if (serialize_ && involved) {
    cudaEventRecord(serial_, st);
    serial_live_ = true;
  }
}

int PeerComm::post(const void* p, cudaStream_t st) {
  PEVD_CUDA(cudaEventRecord(w_->ready[rank_], st));
  w_->ptr[rank_] = p;
  if (!w_->rendezvous()) {
    set_error("peer communicator: another worker failed");
    return ERR_CUDA;
  }
  return OK;
}

int PeerComm::finish(cudaStream_t st) {
  PEVD_CUDA(cudaEventRecord(w_->done[rank_], st));
  if (!w_->rendezvous()) {
    set_error("peer communicator: another worker failed");
    return ERR_CUDA;
  }
  return OK;
}

int PeerComm::bcast(void* buf, int64_t bytes, int root, cudaStream_t st) {
  if (size_ == 1 || bytes <= 0) return OK;
  serial_begin(st, true);
  PEVD_TRY(post(buf, st));
  if (rank_ != root) {
    PEVD_CUDA(cudaStreamWaitEvent(st, w_->ready[root], 0));
    PEVD_CUDA(cudaMemcpyPeerAsync(buf, w_->dev[rank_], w_->ptr[root], w_->dev[root], (size_t)bytes,
                                  st));
  }
  PEVD_TRY(finish(st));
  if (rank_ == root) {
    // the root's buffer may be rewritten only after every rank pulled it
    for (int x = 0; x < size_; ++x)
      if (x != root) PEVD_CUDA(cudaStreamWaitEvent(st, w_->done[x], 0));
  }
  serial_end(st, true);
  return OK;
}

int PeerComm::allgatherv(const void* send, const int64_t* counts, void* recv, cudaStream_t st) {
  int64_t off = 0;
  if (size_ == 1) {
    if (counts[0] > 0 && send != recv)
      PEVD_CUDA(cudaMemcpyAsync(recv, send, (size_t)counts[0], cudaMemcpyDeviceToDevice, st));
    return OK;
  }
  serial_begin(st, true);
  PEVD_TRY(post(send, st));
  off = 0;
  for (int x = 0; x < size_; ++x) {
    char* dst = (char*)recv + off;
    if (counts[x] > 0) {
      if (x == rank_) {
        if (dst != send)
          PEVD_CUDA(cudaMemcpyAsync(dst, send, (size_t)counts[x], cudaMemcpyDeviceToDevice, st));
      } else {
        PEVD_CUDA(cudaStreamWaitEvent(st, w_->ready[x], 0));
        PEVD_CUDA(cudaMemcpyPeerAsync(dst, w_->dev[rank_], w_->ptr[x], w_->dev[x],
                                      (size_t)counts[x], st));
      }
    }
    off += counts[x];
  }
  PEVD_TRY(finish(st));
  // every rank's send buffer was read by every other rank
  for (int x = 0; x < size_; ++x)
    if (x != rank_) PEVD_CUDA(cudaStreamWaitEvent(st, w_->done[x], 0));
  serial_end(st, true);
  return OK;
}

int PeerComm::p2p(const void* send, void* recv, int64_t bytes, int src, int dst,
                  cudaStream_t st) {
  if (bytes <= 0 || src == dst) return OK;
  const bool involved = rank_ == src || rank_ == dst;
  serial_begin(st, involved);
  PEVD_TRY(post(rank_ == src ? send : nullptr, st));
  if (rank_ == dst) {
    PEVD_CUDA(cudaStreamWaitEvent(st, w_->ready[src], 0));
    PEVD_CUDA(cudaMemcpyPeerAsync(recv, w_->dev[dst], w_->ptr[src], w_->dev[src], (size_t)bytes,
                                  st));
  }
  PEVD_TRY(finish(st));
  if (rank_ == src) PEVD_CUDA(cudaStreamWaitEvent(st, w_->done[dst], 0));
  serial_end(st, involved);
  return OK;
}

int PeerComm::device_barrier(cudaStream_t st) {
  if (size_ == 1) return OK;
  // (done events: a rank re-records them only after the next collective's first rendezvous,
  //  which this rank joins after enqueueing these waits; its ready event could already be
  //  re-recorded by its next post())
  serial_begin(st, true);
  PEVD_TRY(post(nullptr, st));
  PEVD_TRY(finish(st));
  for (int x = 0; x < size_; ++x)
    if (x != rank_) PEVD_CUDA(cudaStreamWaitEvent(st, w_->done[x], 0));
  serial_end(st, true);
  return OK;
}

int PeerComm::barrier() {
  if (!w_->rendezvous()) {
    set_error("peer communicator: another worker failed");
    return ERR_CUDA;
  }
  return OK;
}

// ================================================================= NCCL (dlopen'ed)

namespace {

struct NcclApi {
  bool loaded = false;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclBroadcast) Broadcast = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // the copy torch already mapped (same soname) is reused; otherwise the system library
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define PEVD_SYM(name) api.name = (decltype(api.name))dlsym(h, "nccl" #name)
    PEVD_SYM(GetUniqueId);
    PEVD_SYM(CommInitRank);
    PEVD_SYM(CommDestroy);
    PEVD_SYM(Broadcast);
    PEVD_SYM(AllReduce);
    PEVD_SYM(GroupStart);
    PEVD_SYM(GroupEnd);
    PEVD_SYM(GetErrorString);
    PEVD_SYM(Send);
    PEVD_SYM(Recv);
#undef PEVD_SYM
    api.loaded = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Broadcast &&
                 api.AllReduce && api.GroupStart && api.GroupEnd && api.GetErrorString &&
                 api.Send && api.Recv;
  });
  return api;
}

}  // namespace

#define PEVD_NCCL(call)                                                                   \
  do {                                                                                    \
    ncclResult_t r_ = (call);                                                             \
    if (r_ != ncclSuccess) {                                                              \
      ::pevd::set_error("%s:%d NCCL: %s", __FILE__, __LINE__, nccl().GetErrorString(r_)); \
      return ::pevd::ERR_CUDA;                                                            \
    }                                                                                     \
  } while (0)

int NcclComm::unique_id(char out[128]) {
  NcclApi& a = nccl();
  if (!a.loaded) {
    set_error("libnccl.so.2 could not be loaded");
    return ERR_CUDA;
  }
  ncclUniqueId id;
  PEVD_NCCL(a.GetUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  memcpy(out, &id, 128);
  return OK;
}

NcclComm* NcclComm::create(int rank, int size, const char idb[128]) {
  NcclApi& a = nccl();
  if (!a.loaded) {
    set_error("libnccl.so.2 could not be loaded");
    return nullptr;
  }
  ncclUniqueId id;
  memcpy(&id, idb, 128);
  ncclComm_t c = nullptr;
  ncclResult_t r = a.CommInitRank(&c, size, id, rank);
  if (r != ncclSuccess) {
    set_error("ncclCommInitRank: %s", a.GetErrorString(r));
    return nullptr;
  }
  NcclComm* nc = new NcclComm();
  nc->rank_ = rank;
  nc->size_ = size;
  nc->comm_ = c;
  cudaMalloc(&nc->scratch_, 256);
  return nc;
}

NcclComm::~NcclComm() {
  if (comm_) nccl().CommDestroy((ncclComm_t)comm_);
  if (scratch_) cudaFree(scratch_);
}

int NcclComm::bcast(void* buf, int64_t bytes, int root, cudaStream_t st) {
  if (size_ == 1 || bytes <= 0) return OK;
  PEVD_NCCL(nccl().Broadcast(buf, buf, (size_t)bytes, ncclUint8, root, (ncclComm_t)comm_, st));
  return OK;
}

int NcclComm::allgatherv(const void* send, const int64_t* counts, void* recv, cudaStream_t st) {
  // variable all-gather = one broadcast per contributing rank, grouped into one NCCL launch
  NcclApi& a = nccl();
  PEVD_NCCL(a.GroupStart());
  int64_t off = 0;
  int rc = OK;
  for (int x = 0; x < size_; ++x) {
    if (counts[x] > 0) {
      char* dst = (char*)recv + off;
      const void* src = (x == rank_) ? send : dst;
      ncclResult_t r = a.Broadcast(src, dst, (size_t)counts[x], ncclUint8, x, (ncclComm_t)comm_, st);
      if (r != ncclSuccess && rc == OK) {
        set_error("ncclBroadcast: %s", a.GetErrorString(r));
        rc = ERR_CUDA;
      }
    }
    off += counts[x];
  }
  PEVD_NCCL(a.GroupEnd());
  return rc;
}

int NcclComm::p2p(const void* send, void* recv, int64_t bytes, int src, int dst,
                  cudaStream_t st) {
  if (bytes <= 0 || src == dst) return OK;
  if (rank_ == src)
    PEVD_NCCL(nccl().Send(send, (size_t)bytes, ncclUint8, dst, (ncclComm_t)comm_, st));
  else if (rank_ == dst)
    PEVD_NCCL(nccl().Recv(recv, (size_t)bytes, ncclUint8, src, (ncclComm_t)comm_, st));
  return OK;
}

int NcclComm::device_barrier(cudaStream_t st) {
  if (size_ == 1) return OK;
  PEVD_NCCL(nccl().AllReduce(scratch_, scratch_, 1, ncclInt32, ncclSum, (ncclComm_t)comm_, st));
  return OK;
}

int NcclComm::barrier() {
  PEVD_NCCL(nccl().AllReduce(scratch_, scratch_, 1, ncclInt32, ncclSum, (ncclComm_t)comm_, 0));
  PEVD_CUDA(cudaStreamSynchronize(0));
  return OK;
}

}  // namespace pevd
