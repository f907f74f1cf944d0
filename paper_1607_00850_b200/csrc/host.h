// Host-side (C++) internals behind include/sdns_cuda.h.
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/sdns_cuda.h"

namespace sdns_host {

// Exception types mirroring proj/core/include/sdns/types.hpp:28-62; the
// C ABI maps them onto status codes.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void config_error(const std::string& m) { throw Error(SDNS_CONFIG_ERROR, m); }
[[noreturn]] inline void protocol_error(const std::string& m) { throw Error(SDNS_PROTOCOL_ERROR, m); }
[[noreturn]] inline void timeout_error(const std::string& m) { throw Error(SDNS_TIMEOUT_ERROR, m); }

void cuda_check(cudaError_t e, const char* what);

// Runs f, mapping an escaping exception onto its status code and the
// calling thread's sdns_last_error() message (the C ABI's error channel).
int run_guarded(const std::function<void()>& f);
#define SDNS_CUDA(call) ::sdns_host::cuda_check((call), #call)

// layout.cpp
void validate(const sdns_config& cfg);
sdns_layout build_layout(const sdns_config& cfg, int rank);
int64_t block_size(int64_t total, int parts, int index);
int64_t block_start(int64_t total, int parts, int index);
int64_t step_count(double t_end, double dt);
int spectrum_shells(int64_t n);

// comm.cpp --------------------------------------------------------------------
// One point-to-point block of an all-to-all: `bytes` from my `send` to
// group peer `peer` and `bytes` from that peer into my `recv`.
struct Xfer {
  int peer;
  const void* send;
  void* recv;
  size_t send_bytes;
  size_t recv_bytes;
};

class Comm {
 public:
  virtual ~Comm() = default;
  int rank() const { return rank_; }
  int size() const { return size_; }
  // Collective variable all-to-all of device buffers, enqueued on `s`.
  // The k-th block sent to peer q matches the k-th block q receives from me.
  virtual void alltoall(const std::vector<Xfer>& xs, cudaStream_t s) = 0;
  // In-place host reduction, folded in ascending rank order (op 0 sum,
  // 1 max, 2 min) like InProcessComm (transport.cpp:319-329).
  virtual void allreduce(double* v, int n, int op) = 0;
  virtual void barrier() = 0;
  // broadcast_bytes (transport.hpp:62): root's `nbytes` host bytes into
  // every rank's `data`; root and nbytes must agree across ranks.
  virtual void broadcast(void* data, size_t nbytes, int root) = 0;
  // Split by color, ordered by (key, rank) (transport.hpp:66-67).
  virtual std::shared_ptr<Comm> split(int color, int key) = 0;
  virtual int device() const = 0;
  // Transport name as the runner's manifest reports it (runner.cpp:29-40).
  virtual const char* kind() const = 0;
  // Fails every pending and future collective of the group with
  // ProtocolError (InProcessBackend::poison, transport.hpp:125-128); a
  // no-op where the transport has no shared state (loopback, NCCL).
  virtual void poison(const std::string& reason) { (void)reason; }
  // Peer-direct transposes: every rank's device address of `mine` (a buffer
  // of this rank), usable by this rank's kernels -- the pointer itself on a
  // shared device, a CUDA IPC mapping (NVLink peer access) across GPUs.
  // Collective; empty when the transport cannot map peers (every rank then
  // keeps the all-to-all). unmap_peers releases the mappings.
  virtual std::vector<void*> map_peers(void* mine) {
    (void)mine;
    return {};
  }
  virtual void unmap_peers(const std::vector<void*>& ptrs) { (void)ptrs; }
  // Work enqueued on `s` after this call starts only after the work every
  // rank enqueued on its stream before the call has completed. Collective.
  virtual void stream_barrier(cudaStream_t s) { (void)s; }
  // Host wait for stream `s` (which may hold this group's device-side
  // collectives). Transports whose peers are other processes poll instead of
  // blocking: a peer that stalls past the timeout, or an asynchronous
  // transport error, fails the wait -- TimeoutError / ProtocolError, like the
  // reference's collective deadline (transport.cpp:105-140) -- and poisons
  // the communicator so every later collective fails fast with the same
  // error. Loopback and in-process groups block (no remote peer to lose).
  virtual void wait(cudaStream_t s);
  // Collective deadline in seconds (reference default 30 s,
  // runner.hpp:15); <= 0 waits forever.
  void set_timeout(double s) { timeout_s_ = s; }
  // Marks the communicator failed without throwing (a sibling group of the
  // same decomposition failed) and tears the transport down.
  void abandon(int code, const std::string& why) {
    if (!failed_) {
      failed_ = code;
      failed_why_ = why;
      abort_transport();
    }
  }
  double timeout() const { return timeout_s_; }

 protected:
  Comm(int r, int s) : rank_(r), size_(s) {}
  // Polling wait shared by the multi-process transports: `health` returns 0
  // while the transport is sound, else an error code (throws through fail).
  void poll_wait(cudaStream_t s, const std::function<int(std::string&)>& health);
  // Marks the communicator failed (code SDNS_TIMEOUT_ERROR or
  // SDNS_PROTOCOL_ERROR) and throws; later collectives rethrow.
  [[noreturn]] void fail(int code, const std::string& why);
  void check_failed() const;
  // Tears the transport down on failure (NCCL: ncclCommAbort) so no later
  // call can block on the lost peer.
  virtual void abort_transport() {}
  int rank_, size_;
  double timeout_s_ = 30.0;
  int failed_ = 0;
  std::string failed_why_;
};

std::shared_ptr<Comm> make_loopback_comm();
std::shared_ptr<Comm> make_host_comm(int size, int rank, int device, sdns_allgather_fn fn,
                                     sdns_group_fn gfn, void* user);
std::vector<std::shared_ptr<Comm>> make_inprocess_group(int size, int device, double timeout_s);
void nccl_unique_id(unsigned char id[128]);
std::shared_ptr<Comm> make_nccl_comm(const unsigned char id[128], int size, int rank, int device);

// Owners of C ABI handles for host code above the ABI (runner, acceptance).
struct Ctx {
  sdns_ctx* c = nullptr;
  ~Ctx() {
    if (c) sdns_ctx_destroy(c);
  }
};
struct Fld {
  sdns_field* f = nullptr;
  ~Fld() {
    if (f) sdns_field_free(f);
  }
};
struct State {
  sdns_state* s = nullptr;
  ~State() {
    if (s) sdns_state_destroy(s);
  }
};

// runner.cpp: a failed C ABI call becomes the exception it reported; the
// Taylor-Green real block of a rank; a case's initial spectral state.
void ck(int rc);
std::vector<double> tg_real_block(const sdns_layout& lo, bool reference_variant);
void initial_state(sdns_ctx* ctx, const sdns_config& cfg, const std::string& icase,
                   uint64_t seed, sdns_field* u_hat);

// iso_init.cpp
void iso_init(int64_t n, uint64_t seed, double k0, double energy, const sdns_layout& lo,
              double* out);

}  // namespace sdns_host

// Opaque handle wrappers (C ABI types)
struct sdns_comm {
  std::shared_ptr<sdns_host::Comm> c;
};
