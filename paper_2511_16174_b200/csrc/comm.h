// Communicators of the blockwise multi-GPU EVD (dist.cu).
//
// The reference moves every payload through its Router (messaging.py:170-260, worker <-> worker
// and worker <-> host queues).  Here a rank is one GPU driven by one host thread, and the
// payloads move device to device over NVLink / NVSwitch with two collectives only:
//   bcast(buf, bytes, root)                 the panel factor (C4 of SURVEY §2.3)
//   allgatherv(send, counts, recv)          the A W row blocks, straddling panel pieces, the band
// Two implementations:
//   NcclComm  one process per GPU (torchrun): ncclBroadcast, grouped broadcasts for allgatherv.
//             libnccl.so.2 is dlopen'ed (the copy torch already loaded when present), so
//             libpevd.so has no link-time NCCL dependency.
//   PeerComm  one process, one host thread per worker (pevd_syevd_multi, the reference's own
//             threading model, pipeline.py:511-548): device pointers and CUDA events are exchanged
//             through a host rendezvous and every rank PULLS the payload with cudaMemcpyPeerAsync
//             on its comm stream (NVLink P2P; a plain device copy when workers share a GPU).
// Every collective records the words it moves in the rank's ledger, by sender, so the union of
// the ranks' ledgers is the measured CommLedger (messaging.py:111-167).
#pragma once
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <mutex>
#include <vector>
#include "common.cuh"

namespace pevd {

// ledger stages (must match _lib.LEDGER_STAGES)
enum LedgerStage : int { LS_SBR = 0, LS_SBR_PANEL = 1, LS_BANDSTAGE = 2, LS_BC = 3,
                         LS_UGATHER = 4, LS_QD = 5, LS_RESULT = 6, LS_GATHER = 7 };
constexpr int DST_HOST = -1, DST_BROADCAST = -2;

struct Message {
  int32_t src, dst, stage, pad;
  int64_t words;
};

class Comm {
 public:
  virtual ~Comm() {}
  int rank() const { return rank_; }
  int size() const { return size_; }
  // Every rank calls every collective in the same order.  Buffers are device pointers of this
  // rank; `st` is the stream the transfer is ordered on.
  virtual int bcast(void* buf, int64_t bytes, int root, cudaStream_t st) = 0;
  // rank x contributes counts[x] bytes (send, on rank x); recv gets them concatenated in rank
  // order on every rank.  send may alias recv + offset(rank).
  virtual int allgatherv(const void* send, const int64_t* counts, void* recv, cudaStream_t st) = 0;
  // point to point: rank src's `send` -> rank dst's `recv` (bytes).  Every rank calls it (the
  // peer communicator rendezvous); only src and dst move data.
  virtual int p2p(const void* send, void* recv, int64_t bytes, int src, int dst,
                  cudaStream_t st) = 0;
  // host-side barrier of all ranks (no device work)
  virtual int barrier() = 0;
  // device-side barrier: work after it on `st` starts once every rank's `st` reached it
  virtual int device_barrier(cudaStream_t st) = 0;
  // The trace's time base, taken right after barrier(): an event recorded on `st` (returned)
  // and the host CLOCK_MONOTONIC ns it stands for.  Ranks on different devices each record
  // `mine`; ranks sharing a device share ONE event and t0 (PeerComm), so their spans are on one
  // clock -- per-rank bases a few microseconds apart made cross-rank orderings (every final
  // multiply after every solver) flip in the trace.
  virtual cudaEvent_t time_base(cudaEvent_t mine, cudaStream_t st, double& t0_ns);
  // measured ledger of this rank's sends
  void record(int src, int dst, int stage, int64_t words) {
    if (words > 0) msgs_.push_back(Message{src, dst, stage, 0, words});
  }
  std::vector<Message>& messages() { return msgs_; }

 protected:
  int rank_ = 0, size_ = 1;
  std::vector<Message> msgs_;
};

// ---------------------------------------------------------------- single process, peer copies
struct PeerWorld {
  explicit PeerWorld(int G, const int* devs);
  ~PeerWorld();
  int G;
  std::vector<int> dev;
  // rendezvous
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  std::atomic<int64_t> generation{0};
  std::atomic<bool> aborted{false};
  // the shared trace time base of ranks on one device (created by rank 0, freed here)
  cudaEvent_t base_ev = nullptr;
  double base_t0 = 0.0;
  // exchanged per collective
  std::vector<const void*> ptr;
  std::vector<cudaEvent_t> ready, done;
  // all ranks reach the rendezvous (false once any rank aborted)
  bool rendezvous();
  void abort();
};

class PeerComm : public Comm {
 public:
  PeerComm(PeerWorld* w, int rank);
  ~PeerComm() override;
  int bcast(void* buf, int64_t bytes, int root, cudaStream_t st) override;
  int allgatherv(const void* send, const int64_t* counts, void* recv, cudaStream_t st) override;
  int p2p(const void* send, void* recv, int64_t bytes, int src, int dst, cudaStream_t st) override;
  int barrier() override;
  int device_barrier(cudaStream_t st) override;
  cudaEvent_t time_base(cudaEvent_t mine, cudaStream_t st, double& t0_ns) override;

 private:
  PeerWorld* w_;
  int post(const void* p, cudaStream_t st);   // publish pointer + ready event, rendezvous
  int finish(cudaStream_t st);                // publish done event, rendezvous, wait on all
  // PEVD_PEER_SERIAL=1: every operation's device work starts after the previous operation's
  // (in issue order, whatever the streams) -- the ordering NCCL imposes on the operations of
  // one communicator, so the in-process tests catch a stream graph that would deadlock there
  void serial_begin(cudaStream_t st, bool involved);
  void serial_end(cudaStream_t st, bool involved);
  bool serialize_ = false, serial_live_ = false;
  cudaEvent_t serial_ = nullptr;
};

// ---------------------------------------------------------------- one process per GPU, NCCL
class NcclComm : public Comm {
 public:
  // unique id of 128 bytes created by rank 0 (nccl_unique_id) and shared by the caller
  static int unique_id(char out[128]);
  static NcclComm* create(int rank, int size, const char id[128]);
  ~NcclComm() override;
  int bcast(void* buf, int64_t bytes, int root, cudaStream_t st) override;
  int allgatherv(const void* send, const int64_t* counts, void* recv, cudaStream_t st) override;
  int p2p(const void* send, void* recv, int64_t bytes, int src, int dst, cudaStream_t st) override;
  int barrier() override;
  int device_barrier(cudaStream_t st) override;

 private:
  void* comm_ = nullptr;  // ncclComm_t
  void* scratch_ = nullptr;
};

}  // namespace pevd
