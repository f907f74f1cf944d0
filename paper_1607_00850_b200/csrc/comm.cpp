// Communication backends for the transposes of the distributed FFT
// (Communicator contract, proj/core/include/sdns/transport.hpp:39-94):
//  - loopback (p = 1): all-to-all is one device copy per block;
//  - in-process group: threads-as-ranks sharing ONE device, the analogue of
//    the reference's InProcessBackend (transport.cpp:80-368). Exchanges are
//    stream-ordered cudaMemcpyAsync between the ranks' buffers, fenced with
//    events; no kernel ever waits on another. Used to run and test the
//    multi-rank decomposition on a single GPU;
//  - NCCL (one process per GPU, NVLink / NVSwitch): grouped ncclSend /
//    ncclRecv all-to-all (NCCL 2.27 has no ncclAlltoAll), ncclCommSplit for
//    pencil row / column groups. NCCL is loaded with dlopen so the library
//    shares whichever libnccl.so.2 the process (e.g. torch) already uses.
// Reductions gather every rank's values and fold them in ascending rank
// order (transport.cpp:319-329), so results are bit-identical on every rank.
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <thread>

#include "host.h"

namespace sdns_host {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(SDNS_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

void Comm::wait(cudaStream_t s) { SDNS_CUDA(cudaStreamSynchronize(s)); }

void Comm::check_failed() const {
  if (failed_) throw Error(failed_, "communicator failed earlier: " + failed_why_);
}

void Comm::fail(int code, const std::string& why) {
  abandon(code, why);
  throw Error(code, why);
}

// Spins briefly (the common case: the stream is about to drain), then sleeps
// between polls; the deadline counts from the call.
void Comm::poll_wait(cudaStream_t s, const std::function<int(std::string&)>& health) {
  check_failed();
  const auto t0 = std::chrono::steady_clock::now();
  for (long it = 0;; ++it) {
    const cudaError_t q = cudaStreamQuery(s);
    if (q == cudaSuccess) return;
    if (q != cudaErrorNotReady) cuda_check(q, "cudaStreamQuery");
    std::string why;
    if (health)
      if (const int code = health(why)) fail(code, why);
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (timeout_s_ > 0.0 && el > timeout_s_)
      fail(SDNS_TIMEOUT_ERROR, "collective timed out after " + std::to_string(timeout_s_) +
                                   " s waiting for peers (rank " + std::to_string(rank_) + ")");
    if (it > 2000) std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

namespace {

void fold(double* acc, const double* v, int n, int op) {
  for (int i = 0; i < n; ++i) {
    if (op == 0) acc[i] += v[i];
    else if (op == 1) acc[i] = acc[i] > v[i] ? acc[i] : v[i];
    else acc[i] = acc[i] < v[i] ? acc[i] : v[i];
  }
}

// --------------------------------------------------------------------------
class LoopbackComm final : public Comm {
 public:
  LoopbackComm() : Comm(0, 1) {}
  void alltoall(const std::vector<Xfer>& xs, cudaStream_t s) override {
    for (const Xfer& x : xs) {
      if (x.peer != 0 || x.send_bytes != x.recv_bytes) protocol_error("loopback: bad block table");
      if (x.send != x.recv && x.send_bytes)
        SDNS_CUDA(cudaMemcpyAsync(x.recv, x.send, x.send_bytes, cudaMemcpyDeviceToDevice, s));
    }
  }
  void allreduce(double*, int, int) override {}
  void barrier() override {}
  void broadcast(void*, size_t, int root) override {
    if (root != 0) protocol_error("loopback broadcast root must be 0");  // transport.cpp:37-38
  }
  std::vector<void*> map_peers(void* mine) override { return {mine}; }
  const char* kind() const override { return "loopback"; }
  std::shared_ptr<Comm> split(int, int) override { return std::make_shared<LoopbackComm>(); }
  int device() const override {
    int d = 0;
    cudaGetDevice(&d);
    return d;
  }
};

// --------------------------------------------------------------------------
// Shared bulletin board of an in-process group.
struct Board {
  int size;
  int device;
  double timeout_s;
  std::mutex mu;
  std::condition_variable cv;
  long long gen = 0;
  int arrived = 0;
  bool poisoned = false;
  std::string reason;
  std::vector<std::vector<Xfer>> posted;
  std::vector<std::vector<double>> values;
  std::vector<void*> ptrs;
  std::vector<std::pair<int, size_t>> bcast;  // (root, nbytes) each rank posted
  // collective kind each rank entered (transport.cpp: mismatched collectives
  // raise ProtocolError on every rank); the verdict of the last rendezvous
  std::vector<int> op;
  std::string mismatch;
  std::vector<cudaEvent_t> ready, done;
  std::vector<std::pair<int, int>> split_req;
  std::map<std::pair<long long, int>, std::shared_ptr<Board>> children;

  Board(int n, int dev, double to) : size(n), device(dev), timeout_s(to) {
    posted.resize(n);
    values.resize(n);
    ptrs.resize(n);
    bcast.resize(n);
    op.assign(static_cast<size_t>(n), 0);
    split_req.resize(n);
    int prev = 0;
    cudaGetDevice(&prev);
    SDNS_CUDA(cudaSetDevice(dev));
    ready.resize(n);
    done.resize(n);
    for (int i = 0; i < n; ++i) {
      SDNS_CUDA(cudaEventCreateWithFlags(&ready[i], cudaEventDisableTiming));
      SDNS_CUDA(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
    }
    cudaSetDevice(prev);
  }
  ~Board() {
    for (auto e : ready) cudaEventDestroy(e);
    for (auto e : done) cudaEventDestroy(e);
  }

  // Poisons this board and every sub-communicator split from it.
  void poison_all(const std::string& why) {
    std::vector<std::shared_ptr<Board>> kids;
    {
      std::lock_guard<std::mutex> lk(mu);
      if (!poisoned) {
        poisoned = true;
        reason = why;
      }
      for (auto& kv : children) kids.push_back(kv.second);
      cv.notify_all();
    }
    for (auto& k : kids) k->poison_all(why);
  }

  // Rendezvous opening collective `kind` (1 all_to_all, 2 allreduce, 3
  // barrier, 4 split, 5 map_peers, 6 stream_barrier, 7 broadcast): every rank must have
  // entered the same kind, else all of them raise ProtocolError and the
  // group is poisoned.
  void enter(std::unique_lock<std::mutex>& lk, int rank, int kind) {
    op[static_cast<size_t>(rank)] = kind;
    wait_all(lk);
    if (!mismatch.empty()) {
      const std::string m = mismatch;
      poisoned = true;
      if (reason.empty()) reason = m;
      cv.notify_all();
      protocol_error(m);
    }
  }

  // Generation-counted barrier; throws on poison or timeout.
  void wait_all(std::unique_lock<std::mutex>& lk) {
    if (poisoned) protocol_error("group poisoned: " + reason);
    const long long my = gen;
    if (++arrived == size) {
      // the last rank in judges the generation (read by every waiter before
      // any rank can complete another one)
      mismatch.clear();
      for (int q = 1; q < size; ++q)
        if (op[static_cast<size_t>(q)] != op[0]) {
          mismatch = "mismatched collectives: rank 0 entered kind " + std::to_string(op[0]) +
                     ", rank " + std::to_string(q) + " kind " +
                     std::to_string(op[static_cast<size_t>(q)]);
          break;
        }
      arrived = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    const auto deadline = std::chrono::steady_clock::now() +
                          std::chrono::duration<double>(timeout_s);
    while (gen == my && !poisoned) {
      if (cv.wait_until(lk, deadline) == std::cv_status::timeout && gen == my && !poisoned) {
        poisoned = true;
        reason = "collective timed out";
        cv.notify_all();
        timeout_error("in-process collective timed out after " + std::to_string(timeout_s) + " s");
      }
    }
    if (poisoned && gen == my) protocol_error("group poisoned: " + reason);
  }
};

class InProcessComm final : public Comm {
 public:
  InProcessComm(std::shared_ptr<Board> b, int rank) : Comm(rank, b->size), b_(std::move(b)) {}

  int device() const override { return b_->device; }

  void poison(const std::string& why) override { b_->poison_all(why); }
  const char* kind() const override { return "inprocess"; }

  void alltoall(const std::vector<Xfer>& xs, cudaStream_t s) override {
    Board& b = *b_;
    SDNS_CUDA(cudaEventRecord(b.ready[rank_], s));
    {
      std::unique_lock<std::mutex> lk(b.mu);
      b.posted[rank_] = xs;
      b.enter(lk, rank_, 1);
    }
    try {
      validate_and_copy(xs, s);
    } catch (const Error& e) {
      b.poison_all(e.what());  // the peers fail fast instead of timing out
      throw;
    }
    SDNS_CUDA(cudaEventRecord(b.done[rank_], s));
    {
      std::unique_lock<std::mutex> lk(b.mu);
      b.wait_all(lk);
    }
    // My send buffers may be reused only after every peer copied from them.
    for (int q = 0; q < size_; ++q)
      if (q != rank_) SDNS_CUDA(cudaStreamWaitEvent(s, b.done[q], 0));
    {
      std::unique_lock<std::mutex> lk(b.mu);
      b.wait_all(lk);
    }
  }

  // Validate tables and copy every block destined to me from its sender.
  void validate_and_copy(const std::vector<Xfer>& xs, cudaStream_t s) {
    Board& b = *b_;
    std::vector<int> waited(size_, 0);
    std::vector<int> nth_from(size_, 0);
    for (const Xfer& x : xs) {
      const int q = x.peer;
      if (q < 0 || q >= size_) protocol_error("all_to_all: peer out of range");
      // k-th block I receive from q = k-th block q sends to me
      int k = nth_from[q]++;
      const Xfer* match = nullptr;
      for (const Xfer& y : b.posted[q]) {
        if (y.peer != rank_) continue;
        if (k-- == 0) {
          match = &y;
          break;
        }
      }
      if (!match) protocol_error("all_to_all: peer " + std::to_string(q) + " sent fewer blocks");
      if (match->send_bytes != x.recv_bytes)
        protocol_error("all_to_all: inconsistent block tables between ranks " +
                       std::to_string(q) + " and " + std::to_string(rank_));
      if (!waited[q]) {
        SDNS_CUDA(cudaStreamWaitEvent(s, b.ready[q], 0));
        waited[q] = 1;
      }
      if (x.recv_bytes && match->send != x.recv)
        SDNS_CUDA(cudaMemcpyAsync(x.recv, match->send, x.recv_bytes, cudaMemcpyDeviceToDevice, s));
    }
  }

  void allreduce(double* v, int n, int op) override {
    Board& b = *b_;
    std::unique_lock<std::mutex> lk(b.mu);
    b.values[rank_].assign(v, v + n);
    b.enter(lk, rank_, 2);
    for (int q = 0; q < size_; ++q)
      if (static_cast<int>(b.values[q].size()) != n)
        protocol_error("allreduce: mismatched lengths across ranks");
    std::vector<double> acc = b.values[0];
    for (int q = 1; q < size_; ++q) fold(acc.data(), b.values[q].data(), n, op);
    b.wait_all(lk);
    std::memcpy(v, acc.data(), sizeof(double) * n);
  }

  void barrier() override {
    std::unique_lock<std::mutex> lk(b_->mu);
    b_->enter(lk, rank_, 3);
  }

  // Every rank posts (data, root, nbytes); the arguments are checked against
  // rank 0's (validate_broadcast, transport.cpp:332-349: a mismatch poisons
  // the group), non-roots copy from the root's buffer, and a second
  // rendezvous keeps the root's buffer alive until every copy is done.
  void broadcast(void* data, size_t nbytes, int root) override {
    Board& b = *b_;
    std::unique_lock<std::mutex> lk(b.mu);
    b.ptrs[rank_] = data;
    b.bcast[rank_] = {root, nbytes};
    b.enter(lk, rank_, 7);
    const int r0 = b.bcast[0].first;
    const size_t n0 = b.bcast[0].second;
    std::string bad;
    if (r0 < 0 || r0 >= size_) bad = "broadcast root " + std::to_string(r0) + " out of range";
    for (int q = 1; q < size_ && bad.empty(); ++q)
      if (b.bcast[q].first != r0 || b.bcast[q].second != n0)
        bad = "broadcast argument mismatch at rank " + std::to_string(q);
    if (!bad.empty()) {
      b.poisoned = true;
      if (b.reason.empty()) b.reason = bad;
      b.cv.notify_all();
      protocol_error(bad);
    }
    const void* src = b.ptrs[r0];
    lk.unlock();
    if (rank_ != r0 && nbytes) std::memcpy(data, src, nbytes);
    lk.lock();
    b.wait_all(lk);
  }

  // Ranks share the device: a peer's buffer is addressed directly.
  std::vector<void*> map_peers(void* mine) override {
    Board& b = *b_;
    std::unique_lock<std::mutex> lk(b.mu);
    b.ptrs[rank_] = mine;
    b.enter(lk, rank_, 5);
    std::vector<void*> all = b.ptrs;
    b.wait_all(lk);
    return all;
  }

  // Every rank's stream waits for every rank's `ready` event; the second
  // rendezvous keeps a fast rank from re-recording its event before the
  // others captured it.
  void stream_barrier(cudaStream_t s) override {
    Board& b = *b_;
    SDNS_CUDA(cudaEventRecord(b.ready[rank_], s));
    std::unique_lock<std::mutex> lk(b.mu);
    b.enter(lk, rank_, 6);
    for (int q = 0; q < size_; ++q)
      if (q != rank_) SDNS_CUDA(cudaStreamWaitEvent(s, b.ready[q], 0));
    b.wait_all(lk);
  }

  std::shared_ptr<Comm> split(int color, int key) override {
    Board& b = *b_;
    std::unique_lock<std::mutex> lk(b.mu);
    b.split_req[rank_] = {color, key};
    const long long g = b.gen;
    b.enter(lk, rank_, 4);
    std::vector<std::pair<int, int>> members;  // (key, rank)
    for (int q = 0; q < size_; ++q)
      if (b.split_req[q].first == color) members.push_back({b.split_req[q].second, q});
    std::sort(members.begin(), members.end());
    int my = 0;
    for (size_t i = 0; i < members.size(); ++i)
      if (members[i].second == rank_) my = static_cast<int>(i);
    auto kk = std::make_pair(g, color);
    auto it = b.children.find(kk);
    std::shared_ptr<Board> child;
    if (it == b.children.end()) {
      child = std::make_shared<Board>(static_cast<int>(members.size()), b.device, b.timeout_s);
      b.children[kk] = child;
    } else {
      child = it->second;
    }
    b.wait_all(lk);
    return std::make_shared<InProcessComm>(child, my);
  }

 private:
  std::shared_ptr<Board> b_;
};

// --------------------------------------------------------------------------
// CUDA IPC mapping of every rank's buffer for the peer-direct transposes
// (one process per GPU): the 64-byte handles travel through `gather` (every
// rank's bytes, rank order); `agree_min` reduces the success flag so every
// rank keeps or drops the mappings together.
std::vector<void*> ipc_map_peers(void* mine, int rank, int size,
                                 const std::function<void(const void*, size_t, void*)>& gather,
                                 const std::function<double(double)>& agree_min) {
  cudaIpcMemHandle_t h{};
  double ok = cudaIpcGetMemHandle(&h, mine) == cudaSuccess ? 1.0 : 0.0;
  cudaGetLastError();
  std::vector<cudaIpcMemHandle_t> all(static_cast<size_t>(size));
  gather(&h, sizeof(h), all.data());
  std::vector<void*> out(static_cast<size_t>(size), nullptr);
  out[static_cast<size_t>(rank)] = mine;
  for (int q = 0; q < size && ok > 0.5; ++q) {
    if (q == rank) continue;
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, all[static_cast<size_t>(q)], cudaIpcMemLazyEnablePeerAccess) !=
        cudaSuccess) {
      cudaGetLastError();
      ok = 0.0;
      break;
    }
    out[static_cast<size_t>(q)] = p;
  }
  if (agree_min(ok) < 0.5) {
    for (int q = 0; q < size; ++q)
      if (q != rank && out[static_cast<size_t>(q)]) cudaIpcCloseMemHandle(out[static_cast<size_t>(q)]);
    return {};
  }
  return out;
}

void ipc_unmap_peers(const std::vector<void*>& ptrs, int rank) {
  for (int q = 0; q < static_cast<int>(ptrs.size()); ++q)
    if (q != rank && ptrs[static_cast<size_t>(q)]) cudaIpcCloseMemHandle(ptrs[static_cast<size_t>(q)]);
}

// Broadcast arguments checked over an all-gather (validate_broadcast,
// transport.cpp:332-349): every rank sees every rank's (root, nbytes) and
// raises the same ProtocolError.
void bcast_check(int root, size_t nbytes, int size,
                 const std::function<void(const void*, size_t, void*)>& gather) {
  const long long mine[2] = {root, static_cast<long long>(nbytes)};
  std::vector<long long> all(2 * static_cast<size_t>(size));
  gather(mine, sizeof(mine), all.data());
  const long long r0 = all[0], n0 = all[1];
  if (r0 < 0 || r0 >= size) protocol_error("broadcast root " + std::to_string(r0) + " out of range");
  for (int q = 1; q < size; ++q)
    if (all[2 * static_cast<size_t>(q)] != r0 || all[2 * static_cast<size_t>(q) + 1] != n0)
      protocol_error("broadcast argument mismatch at rank " + std::to_string(q));
}

// --------------------------------------------------------------------------
// Host-callback transport: one process per rank (several may share a GPU)
// with the caller's host all-gather (e.g. torch.distributed over gloo) as the
// only primitive (plus a group callback for split). Reductions fold gathered
// values in rank order; buffers are exchanged by CUDA IPC and stream barriers
// wait on the ranks' IPC events, so no kernel ever waits on another. The
// RHS transposes run peer-direct; the all-to-all (checkpoints, the API call)
// goes through the host all-gather.
class HostComm final : public Comm {
 public:
  HostComm(int rank, int size, int device, sdns_allgather_fn fn, sdns_group_fn gfn, void* user)
      : Comm(rank, size), device_(device), fn_(fn), gfn_(gfn), user_(user) {
    SDNS_CUDA(cudaSetDevice(device_));
    SDNS_CUDA(cudaEventCreateWithFlags(&ev_, cudaEventDisableTiming | cudaEventInterprocess));
    cudaIpcEventHandle_t h{};
    SDNS_CUDA(cudaIpcGetEventHandle(&h, ev_));
    std::vector<cudaIpcEventHandle_t> all(static_cast<size_t>(size));
    gather(&h, sizeof(h), all.data());
    peer_ev_.assign(static_cast<size_t>(size), nullptr);
    for (int q = 0; q < size; ++q)
      if (q != rank) SDNS_CUDA(cudaIpcOpenEventHandle(&peer_ev_[static_cast<size_t>(q)], all[static_cast<size_t>(q)]));
  }
  ~HostComm() override {
    for (auto e : peer_ev_)
      if (e) cudaEventDestroy(e);
    if (ev_) cudaEventDestroy(ev_);
  }
  int device() const override { return device_; }
  const char* kind() const override { return "host"; }

  // Variable all-to-all through the caller's all-gather (the transport's
  // only primitive): every rank packs its send blocks on the host, the send
  // tables and the packed buffers (padded to the largest) are all-gathered,
  // and each rank unpacks the blocks addressed to it. Every rank receives
  // every buffer, so this serves the infrequent exchanges (checkpoint
  // gathers and scatters, the API's all_to_all); the RHS transposes run
  // peer-direct over CUDA IPC. Tables are checked like InProcessComm's.
  void alltoall(const std::vector<Xfer>& xs, cudaStream_t s) override {
    check_failed();
    const size_t p = static_cast<size_t>(size_);
    std::vector<int64_t> mine(2 * p, 0);  // [send to q | recv from q] bytes
    for (const Xfer& x : xs) {
      if (x.peer < 0 || x.peer >= size_) protocol_error("all_to_all: peer out of range");
      mine[static_cast<size_t>(x.peer)] += static_cast<int64_t>(x.send_bytes);
      mine[p + static_cast<size_t>(x.peer)] += static_cast<int64_t>(x.recv_bytes);
    }
    std::vector<int64_t> tab(2 * p * p);
    gather(mine.data(), sizeof(int64_t) * 2 * p, tab.data());
    for (size_t q = 0; q < p; ++q)  // what q sends me == what I expect from q
      if (tab[q * 2 * p + static_cast<size_t>(rank_)] != mine[p + q])
        protocol_error("all_to_all: send/recv block sizes disagree between rank " +
                       std::to_string(q) + " and rank " + std::to_string(rank_));
    int64_t total = 0, maxtot = 0;
    for (size_t q = 0; q < p; ++q) {
      int64_t tq = 0;
      for (size_t d = 0; d < p; ++d) tq += tab[q * 2 * p + d];
      maxtot = std::max(maxtot, tq);
      if (static_cast<int>(q) == rank_) total = tq;
    }
    if (maxtot == 0) return;
    // pack: blocks in (destination, call order) order
    std::vector<char> pack(static_cast<size_t>(maxtot), 0);
    std::vector<int64_t> doff(p, 0);
    for (size_t d = 1; d < p; ++d) doff[d] = doff[d - 1] + mine[d - 1];
    std::vector<int64_t> put = doff;
    // copies on `s` itself: ordered after the producers of the send blocks and
    // before the consumers of the receive blocks (a legacy-stream cudaMemcpy
    // from pageable memory may return before its DMA lands, and a
    // non-blocking stream is not ordered after it)
    for (const Xfer& x : xs)
      if (x.send_bytes) {
        SDNS_CUDA(cudaMemcpyAsync(pack.data() + put[static_cast<size_t>(x.peer)], x.send,
                                  x.send_bytes, cudaMemcpyDeviceToHost, s));
        put[static_cast<size_t>(x.peer)] += static_cast<int64_t>(x.send_bytes);
      }
    SDNS_CUDA(cudaStreamSynchronize(s));
    (void)total;
    std::vector<char> all(static_cast<size_t>(maxtot) * p);
    gather(pack.data(), static_cast<size_t>(maxtot), all.data());
    // unpack: from q's buffer, the region q packed for me, in call order
    std::vector<int64_t> get(p, 0);
    for (size_t q = 0; q < p; ++q)
      for (int d = 0; d < rank_; ++d) get[q] += tab[q * 2 * p + static_cast<size_t>(d)];
    for (const Xfer& x : xs)
      if (x.recv_bytes) {
        const size_t q = static_cast<size_t>(x.peer);
        SDNS_CUDA(cudaMemcpyAsync(x.recv, all.data() + q * static_cast<size_t>(maxtot) + get[q],
                                  x.recv_bytes, cudaMemcpyHostToDevice, s));
        get[q] += static_cast<int64_t>(x.recv_bytes);
      }
    SDNS_CUDA(cudaStreamSynchronize(s));  // `all` is released on return
  }
  void allreduce(double* v, int n, int op) override {
    std::vector<double> all(static_cast<size_t>(n) * size_);
    gather(v, sizeof(double) * static_cast<size_t>(n), all.data());
    std::vector<double> acc(all.begin(), all.begin() + n);
    for (int q = 1; q < size_; ++q) fold(acc.data(), all.data() + static_cast<size_t>(q) * n, n, op);
    std::memcpy(v, acc.data(), sizeof(double) * static_cast<size_t>(n));
  }
  void barrier() override {
    char b = 0;
    std::vector<char> all(static_cast<size_t>(size_));
    gather(&b, 1, all.data());
  }
  // (root, nbytes) are gathered and checked first, then every rank's bytes
  // (the root's slice is kept).
  void broadcast(void* data, size_t nbytes, int root) override {
    bcast_check(root, nbytes, size_, [this](const void* a, size_t b, void* c) { gather(a, b, c); });
    if (!nbytes) return;
    std::vector<char> all(nbytes * static_cast<size_t>(size_));
    gather(data, nbytes, all.data());
    if (rank_ != root) std::memcpy(data, all.data() + nbytes * static_cast<size_t>(root), nbytes);
  }
  // Every rank gathers all (color, key) pairs, then the groups are created
  // through the caller's group callback in ascending color order with
  // identical arguments on every rank (members ordered by (key, rank),
  // transport.hpp:66-67); each rank joins its own.
  std::shared_ptr<Comm> split(int color, int key) override {
    if (!gfn_) protocol_error("host-callback transport: no group callback, split not provided");
    const int mine[2] = {color, key};
    std::vector<int> all(2 * static_cast<size_t>(size_));
    gather(mine, sizeof(mine), all.data());
    std::vector<int> colors;
    for (int q = 0; q < size_; ++q) colors.push_back(all[2 * static_cast<size_t>(q)]);
    std::sort(colors.begin(), colors.end());
    colors.erase(std::unique(colors.begin(), colors.end()), colors.end());
    void* my_user = nullptr;
    int my_rank = 0, my_size = 0;
    for (int c : colors) {
      std::vector<std::pair<int, int>> mem;  // (key, rank)
      for (int q = 0; q < size_; ++q)
        if (all[2 * static_cast<size_t>(q)] == c) mem.push_back({all[2 * static_cast<size_t>(q) + 1], q});
      std::sort(mem.begin(), mem.end());
      std::vector<int> ranks;
      for (const auto& m : mem) ranks.push_back(m.second);
      void* gu = nullptr;
      if (gfn_(ranks.data(), static_cast<int>(ranks.size()), user_, &gu) != 0)
        protocol_error("host group callback failed");
      if (c == color) {
        my_user = gu;
        my_size = static_cast<int>(ranks.size());
        my_rank = static_cast<int>(std::find(ranks.begin(), ranks.end(), rank_) - ranks.begin());
      }
    }
    auto child = std::make_shared<HostComm>(my_rank, my_size, device_, fn_, gfn_, my_user);
    child->set_timeout(timeout_s_);
    return child;
  }
  std::vector<void*> map_peers(void* mine) override {
    return ipc_map_peers(
        mine, rank_, size_, [this](const void* a, size_t b, void* c) { gather(a, b, c); },
        [this](double x) {
          allreduce(&x, 1, 2);
          return x;
        });
  }
  void unmap_peers(const std::vector<void*>& ptrs) override { ipc_unmap_peers(ptrs, rank_); }
  void wait(cudaStream_t s) override { poll_wait(s, nullptr); }
  void stream_barrier(cudaStream_t s) override {
    SDNS_CUDA(cudaEventRecord(ev_, s));
    barrier();
    for (int q = 0; q < size_; ++q)
      if (q != rank_) SDNS_CUDA(cudaStreamWaitEvent(s, peer_ev_[static_cast<size_t>(q)], 0));
    barrier();  // nobody re-records before every rank captured the events
  }

 private:
  // The callback returns 0, or 2 when the caller's transport timed out (a
  // peer stalled or died), any other value for other failures.
  void gather(const void* send, size_t bytes, void* recv) {
    check_failed();
    const int rc = fn_(send, bytes, recv, user_);
    if (rc == 2)
      fail(SDNS_TIMEOUT_ERROR, "host all-gather timed out waiting for peers (rank " +
                                   std::to_string(rank_) + ")");
    if (rc != 0) fail(SDNS_PROTOCOL_ERROR, "host all-gather callback failed");
  }
  int device_;
  sdns_allgather_fn fn_;
  sdns_group_fn gfn_;
  void* user_;
  cudaEvent_t ev_ = nullptr;
  std::vector<cudaEvent_t> peer_ev_;
};

// --------------------------------------------------------------------------
// NCCL through dlopen (the subset we call; ABI per /usr/include/nccl.h).
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;
enum { ncclInt8 = 0, ncclFloat64 = 8 };

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, void*) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;

  static NcclApi& get() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
      const char* names[] = {"libnccl.so.2", "libnccl.so"};
      for (const char* nm : names) {
        api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
        if (api.h) break;
      }
      if (!api.h) return;
      auto sym = [](const char* s) { return dlsym(api.h, s); };
      api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
      api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
      api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
      api.CommSplit = reinterpret_cast<decltype(api.CommSplit)>(sym("ncclCommSplit"));
      api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
      api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
      api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
      api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
      api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
      api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
      api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(sym("ncclBroadcast"));
      api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
      api.CommGetAsyncError =
          reinterpret_cast<decltype(api.CommGetAsyncError)>(sym("ncclCommGetAsyncError"));
      api.CommAbort = reinterpret_cast<decltype(api.CommAbort)>(sym("ncclCommAbort"));
    });
    if (!api.h || !api.GetUniqueId || !api.Send || !api.CommSplit)
      throw Error(SDNS_CUDA_ERROR, "NCCL (libnccl.so.2) could not be loaded");
    return api;
  }
};

void nccl_check(ncclResult_t r, const char* what) {
  if (r != 0) {
    auto& api = NcclApi::get();
    throw Error(SDNS_PROTOCOL_ERROR,
                std::string(what) + ": " + (api.GetErrorString ? api.GetErrorString(r) : "nccl error"));
  }
}

class NcclComm final : public Comm {
 public:
  NcclComm(ncclComm_t c, int rank, int size, int device)
      : Comm(rank, size), comm_(c), device_(device) {
    SDNS_CUDA(cudaSetDevice(device_));
    SDNS_CUDA(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
    SDNS_CUDA(cudaMalloc(&dbuf_, sizeof(double) * kMaxVals * (size + 1)));
    SDNS_CUDA(cudaMalloc(&tok_, sizeof(double)));
    SDNS_CUDA(cudaMemset(tok_, 0, sizeof(double)));
  }
  ~NcclComm() override {
    if (dbuf_) cudaFree(dbuf_);
    if (tok_) cudaFree(tok_);
    if (side_) cudaStreamDestroy(side_);
    if (comm_) NcclApi::get().CommDestroy(comm_);
  }
  int device() const override { return device_; }
  const char* kind() const override { return "nccl"; }

  // Polls the stream and ncclCommGetAsyncError: an asynchronous NCCL error
  // raises ProtocolError, a peer that stalls past the deadline TimeoutError;
  // either aborts the communicator (ncclCommAbort) so nothing blocks on it.
  void wait(cudaStream_t s) override {
    auto& api = NcclApi::get();
    poll_wait(s, [this, &api](std::string& why) {
      if (!api.CommGetAsyncError || !comm_) return 0;
      ncclResult_t st = 0;
      if (api.CommGetAsyncError(comm_, &st) != 0) return 0;
      if (st == 0 || st == kInProgress) return 0;
      why = std::string("NCCL asynchronous error on rank ") + std::to_string(rank_) + ": " +
            (api.GetErrorString ? api.GetErrorString(st) : "nccl error");
      return static_cast<int>(SDNS_PROTOCOL_ERROR);
    });
  }

  void alltoall(const std::vector<Xfer>& xs, cudaStream_t s) override {
    check_failed();
    auto& api = NcclApi::get();
    nccl_check(api.GroupStart(), "ncclGroupStart");
    for (const Xfer& x : xs) {
      if (x.peer == rank_) {
        if (x.send_bytes != x.recv_bytes) protocol_error("all_to_all: self block size mismatch");
        if (x.send_bytes && x.send != x.recv)
          SDNS_CUDA(cudaMemcpyAsync(x.recv, x.send, x.send_bytes, cudaMemcpyDeviceToDevice, s));
        continue;
      }
      if (x.send_bytes) nccl_check(api.Send(x.send, x.send_bytes, ncclInt8, x.peer, comm_, s), "ncclSend");
      if (x.recv_bytes) nccl_check(api.Recv(x.recv, x.recv_bytes, ncclInt8, x.peer, comm_, s), "ncclRecv");
    }
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
  }

  void allreduce(double* v, int n, int op) override {
    if (n > kMaxVals) {
      for (int off = 0; off < n; off += kMaxVals)
        allreduce(v + off, std::min(kMaxVals, n - off), op);
      return;
    }
    check_failed();
    auto& api = NcclApi::get();
    double* mine = dbuf_ + static_cast<size_t>(kMaxVals) * size_;
    SDNS_CUDA(cudaMemcpyAsync(mine, v, sizeof(double) * n, cudaMemcpyHostToDevice, side_));
    nccl_check(api.AllGather(mine, dbuf_, static_cast<size_t>(n), ncclFloat64, comm_, side_),
               "ncclAllGather");
    std::vector<double> all(static_cast<size_t>(n) * size_);
    SDNS_CUDA(cudaMemcpyAsync(all.data(), dbuf_, sizeof(double) * n * size_,
                              cudaMemcpyDeviceToHost, side_));
    wait(side_);
    std::vector<double> acc(all.begin(), all.begin() + n);
    for (int q = 1; q < size_; ++q) fold(acc.data(), all.data() + static_cast<size_t>(q) * n, n, op);
    std::memcpy(v, acc.data(), sizeof(double) * n);
  }

  void barrier() override {
    double x = 0.0;
    allreduce(&x, 1, 0);
  }

  // (root, nbytes) are checked over the all-gather, then the bytes move by
  // ncclBroadcast through the device staging buffer.
  void broadcast(void* data, size_t nbytes, int root) override {
    check_failed();
    bcast_check(root, nbytes, size_, [this](const void* a, size_t b, void* c) { gather_bytes(a, b, c); });
    auto& api = NcclApi::get();
    if (!api.Broadcast) throw Error(SDNS_CUDA_ERROR, "ncclBroadcast not found");
    const size_t chunk = sizeof(double) * static_cast<size_t>(kMaxVals) * static_cast<size_t>(size_);
    char* h = static_cast<char*>(data);
    for (size_t off = 0; off < nbytes; off += chunk) {
      const size_t b = std::min(chunk, nbytes - off);
      if (rank_ == root)
        SDNS_CUDA(cudaMemcpyAsync(dbuf_, h + off, b, cudaMemcpyHostToDevice, side_));
      nccl_check(api.Broadcast(dbuf_, dbuf_, b, ncclInt8, root, comm_, side_), "ncclBroadcast");
      if (rank_ != root)
        SDNS_CUDA(cudaMemcpyAsync(h + off, dbuf_, b, cudaMemcpyDeviceToHost, side_));
      wait(side_);
    }
  }

  // CUDA IPC handles of every rank's buffer, exchanged over the
  // communicator and opened with peer access (NVLink / NVSwitch). The
  // outcome is agreed collectively: if any rank fails to export or map,
  // every rank releases its mappings and returns empty.
  std::vector<void*> map_peers(void* mine) override {
    return ipc_map_peers(
        mine, rank_, size_, [this](const void* a, size_t b, void* c) { gather_bytes(a, b, c); },
        [this](double x) {
          allreduce(&x, 1, 2);
          return x;
        });
  }

  void unmap_peers(const std::vector<void*>& ptrs) override { ipc_unmap_peers(ptrs, rank_); }

  // A one-element all-reduce on the compute stream: NCCL's kernel completes
  // on a rank only after every rank's stream reached it, and the producing
  // kernels end with a system-scope fence on their peer stores.
  void stream_barrier(cudaStream_t s) override {
    check_failed();
    auto& api = NcclApi::get();
    if (!api.AllReduce) throw Error(SDNS_CUDA_ERROR, "ncclAllReduce not found");
    nccl_check(api.AllReduce(tok_, tok_, 1, ncclFloat64, 0 /* ncclSum */, comm_, s),
               "ncclAllReduce");
  }

  std::shared_ptr<Comm> split(int color, int key) override {
    check_failed();
    auto& api = NcclApi::get();
    ncclComm_t nc = nullptr;
    nccl_check(api.CommSplit(comm_, color, key, &nc, nullptr), "ncclCommSplit");
    // rank within the new group: order by (key, rank) like the reference
    double mine[2] = {static_cast<double>(color), static_cast<double>(key)};
    std::vector<double> all(2 * static_cast<size_t>(size_));
    gather2(mine, all.data());
    int my = 0, cnt = 0;
    for (int q = 0; q < size_; ++q) {
      if (static_cast<int>(all[2 * q]) != color) continue;
      ++cnt;
      const int kq = static_cast<int>(all[2 * q + 1]);
      if (kq < key || (kq == key && q < rank_)) ++my;
    }
    auto child = std::make_shared<NcclComm>(nc, my, cnt, device_);
    child->set_timeout(timeout_s_);
    return child;
  }

 private:
  static constexpr int kMaxVals = 4096;
  static constexpr ncclResult_t kInProgress = 7;  // ncclInProgress
  void abort_transport() override {
    auto& api = NcclApi::get();
    if (comm_ && api.CommAbort) api.CommAbort(comm_);
    comm_ = nullptr;
  }
  // Every rank's `bytes` (<= 8 * kMaxVals) in rank order, through the device
  // all-gather.
  void gather_bytes(const void* mine, size_t bytes, void* all) {
    auto& api = NcclApi::get();
    const size_t nd = (bytes + sizeof(double) - 1) / sizeof(double);
    if (nd > static_cast<size_t>(kMaxVals)) protocol_error("gather_bytes: too large");
    std::vector<double> pad(nd, 0.0);
    std::memcpy(pad.data(), mine, bytes);
    double* d_mine = dbuf_ + static_cast<size_t>(kMaxVals) * size_;
    SDNS_CUDA(cudaMemcpyAsync(d_mine, pad.data(), sizeof(double) * nd, cudaMemcpyHostToDevice, side_));
    nccl_check(api.AllGather(d_mine, dbuf_, nd, ncclFloat64, comm_, side_), "ncclAllGather");
    std::vector<double> got(nd * size_);
    SDNS_CUDA(cudaMemcpyAsync(got.data(), dbuf_, sizeof(double) * nd * size_, cudaMemcpyDeviceToHost,
                              side_));
    wait(side_);
    for (int q = 0; q < size_; ++q)
      std::memcpy(static_cast<char*>(all) + bytes * q, got.data() + nd * q, bytes);
  }
  void gather2(const double* mine, double* all) {
    auto& api = NcclApi::get();
    double* d_mine = dbuf_ + static_cast<size_t>(kMaxVals) * size_;
    SDNS_CUDA(cudaMemcpyAsync(d_mine, mine, sizeof(double) * 2, cudaMemcpyHostToDevice, side_));
    nccl_check(api.AllGather(d_mine, dbuf_, 2, ncclFloat64, comm_, side_), "ncclAllGather");
    SDNS_CUDA(cudaMemcpyAsync(all, dbuf_, sizeof(double) * 2 * size_, cudaMemcpyDeviceToHost, side_));
    wait(side_);
  }
  ncclComm_t comm_ = nullptr;
  int device_ = 0;
  cudaStream_t side_ = nullptr;
  double* dbuf_ = nullptr;
  double* tok_ = nullptr;  // stream_barrier's all-reduce operand
};

}  // namespace

std::shared_ptr<Comm> make_loopback_comm() { return std::make_shared<LoopbackComm>(); }

std::shared_ptr<Comm> make_host_comm(int size, int rank, int device, sdns_allgather_fn fn,
                                     sdns_group_fn gfn, void* user) {
  if (size < 1 || rank < 0 || rank >= size) config_error("host comm: bad rank/size");
  if (!fn) config_error("host comm: all-gather callback is NULL");
  return std::make_shared<HostComm>(rank, size, device, fn, gfn, user);
}

std::vector<std::shared_ptr<Comm>> make_inprocess_group(int size, int device, double timeout_s) {
  if (size < 1) config_error("in-process group size must be >= 1");
  auto b = std::make_shared<Board>(size, device, timeout_s);
  std::vector<std::shared_ptr<Comm>> out;
  for (int r = 0; r < size; ++r) out.push_back(std::make_shared<InProcessComm>(b, r));
  return out;
}

void nccl_unique_id(unsigned char id[128]) {
  ncclUniqueId u;
  nccl_check(NcclApi::get().GetUniqueId(&u), "ncclGetUniqueId");
  std::memcpy(id, u.internal, 128);
}

std::shared_ptr<Comm> make_nccl_comm(const unsigned char id[128], int size, int rank, int device) {
  ncclUniqueId u;
  std::memcpy(u.internal, id, 128);
  SDNS_CUDA(cudaSetDevice(device));
  ncclComm_t c = nullptr;
  nccl_check(NcclApi::get().CommInitRank(&c, size, u, rank), "ncclCommInitRank");
  return std::make_shared<NcclComm>(c, rank, size, device);
}

}  // namespace sdns_host
