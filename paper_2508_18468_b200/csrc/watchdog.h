// NCCL failure detection for the row-sharded step (ncclCommGetAsyncError polled).
//
// One host thread per communicator.  The step marks the end of its stream work (an event) after
// every call that issues collectives; the thread polls ncclCommGetAsyncError and the oldest
// outstanding mark, and aborts the communicator (ncclCommAbort, which also terminates NCCL kernels
// still waiting for a peer) on an asynchronous error or when a mark stays incomplete past the
// deadline (TRAJ_NCCL_TIMEOUT_S, default 600 s).  From then on every sharded call returns
// TRAJ_ENCCL with the reason, instead of hanging in a collective whose partner never arrives.
#pragma once
#include <cuda_runtime.h>

#include <string>

typedef struct ncclComm* ncclComm_t;

namespace traj {

struct WatchdogImpl;

struct Watchdog {
  WatchdogImpl* p = nullptr;
  // starts the polling thread for comm on device dev
  int start(ncclComm_t comm, int dev, double timeout_s, std::string* err);
  // record a completion mark on st (after the collectives of a call were enqueued)
  int mark(cudaStream_t st, std::string* err);
  // TRAJ_ENCCL (with the reason in *err) once the communicator was aborted, else 0
  int check(std::string* err) const;
  bool aborted() const;
  // serialises NCCL calls of the owning thread with the abort (see watchdog.cu)
  void lock();
  void unlock();
  // test hook (TRAJ_WATCHDOG_TEST_STALL=1): enqueue a kernel on st that spins until the watchdog
  // aborts (or 20 s pass), standing in for a collective whose peer never arrives
  int stall(cudaStream_t st, std::string* err);
  // stops the thread; returns true if the communicator was aborted (the caller must not destroy it)
  bool stop();
};

}  // namespace traj
