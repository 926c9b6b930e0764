// NCCL watchdog of the row-sharded step (watchdog.h).
#include <nccl.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/traj.h"
#include "common.cuh"
#include "watchdog.h"

namespace traj {

namespace {

// spins until *flag != 0 (a mapped host word set by the watchdog's abort) or ~20 s of SM clock
__global__ void stall_kernel(volatile int* flag) {
  const long long t0 = clock64();
  while (*flag == 0 && clock64() - t0 < 40000000000ll) __nanosleep(1000);
}

using clk = std::chrono::steady_clock;

}  // namespace

struct WatchdogImpl {
  ncclComm_t comm = nullptr;
  int dev = 0;
  double timeout_s = 600.0;
  std::thread th;
  std::mutex m;          // pending / pool
  std::timed_mutex nccl_m;   // held by the owner around NCCL calls, and by the abort
  std::condition_variable cv;
  std::deque<std::pair<cudaEvent_t, clk::time_point>> pending;
  std::vector<cudaEvent_t> pool;
  std::atomic<bool> quit{false}, aborted{false};
  std::string reason;
  int* stall_flag = nullptr;   // mapped pinned host word

  void abort_comm(const std::string& why) {
    // take the NCCL lock if the owner is not stuck inside an NCCL host call; after the deadline
    // abort regardless (ncclCommAbort is the documented way to unblock a hung call)
    const bool got = nccl_m.try_lock_for(std::chrono::milliseconds((long long)(1000 * std::min(timeout_s, 5.0))));
    {
      std::lock_guard<std::mutex> g(m);
      reason = why;
    }
    aborted.store(true);
    ncclCommAbort(comm);
    if (stall_flag) *reinterpret_cast<volatile int*>(stall_flag) = 1;
    if (got) nccl_m.unlock();
  }

  void run() {
    cudaSetDevice(dev);
    while (!quit.load()) {
      {
        std::unique_lock<std::mutex> g(m);
        cv.wait_for(g, std::chrono::milliseconds(20));
      }
      if (quit.load() || aborted.load()) break;
      ncclResult_t ar = ncclSuccess;
      if (ncclCommGetAsyncError(comm, &ar) == ncclSuccess && ar != ncclSuccess && ar != ncclInProgress) {
        abort_comm(std::string("NCCL asynchronous error: ") + ncclGetErrorString(ar) + " (communicator aborted)");
        break;
      }
      // retire every completed mark from the front; time the oldest incomplete one
      bool stop_now = false;
      for (;;) {
        cudaEvent_t ev = nullptr;
        clk::time_point t0;
        {
          std::lock_guard<std::mutex> g(m);
          if (pending.empty()) break;
          ev = pending.front().first;
          t0 = pending.front().second;
        }
        const cudaError_t q = cudaEventQuery(ev);
        if (q == cudaSuccess) {
          std::lock_guard<std::mutex> g(m);
          pending.pop_front();
          pool.push_back(ev);
          continue;
        }
        if (q == cudaErrorNotReady) {
          const double waited = std::chrono::duration<double>(clk::now() - t0).count();
          if (waited > timeout_s) {
            abort_comm("NCCL watchdog: collectives not complete after " + std::to_string((int)timeout_s) +
                       " s (TRAJ_NCCL_TIMEOUT_S); communicator aborted");
            stop_now = true;
          }
        } else {
          abort_comm(std::string("NCCL watchdog: CUDA error while waiting: ") + cudaGetErrorString(q));
          stop_now = true;
        }
        break;
      }
      if (stop_now) break;
    }
  }
};

int Watchdog::start(ncclComm_t comm, int dev, double timeout_s, std::string* err) {
  p = new WatchdogImpl();
  p->comm = comm;
  p->dev = dev;
  p->timeout_s = timeout_s > 0 ? timeout_s : 600.0;
  if (cudaHostAlloc(&p->stall_flag, 4, cudaHostAllocMapped) != cudaSuccess) {
    if (err) *err = "watchdog: cudaHostAlloc";
    delete p;
    p = nullptr;
    return TRAJ_ECUDA;
  }
  *p->stall_flag = 0;
  p->th = std::thread([this] { p->run(); });
  return 0;
}

int Watchdog::mark(cudaStream_t st, std::string* err) {
  if (!p) return 0;
  cudaEvent_t ev = nullptr;
  {
    std::lock_guard<std::mutex> g(p->m);
    if (!p->pool.empty()) {
      ev = p->pool.back();
      p->pool.pop_back();
    }
  }
  if (!ev && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
    if (err) *err = "watchdog: cudaEventCreate";
    return TRAJ_ECUDA;
  }
  if (cudaEventRecord(ev, st) != cudaSuccess) {
    if (err) *err = "watchdog: cudaEventRecord";
    return TRAJ_ECUDA;
  }
  std::lock_guard<std::mutex> g(p->m);
  p->pending.emplace_back(ev, clk::now());
  return 0;
}

int Watchdog::check(std::string* err) const {
  if (!p || !p->aborted.load()) return 0;
  if (err) {
    std::lock_guard<std::mutex> g(p->m);
    *err = p->reason;
  }
  return TRAJ_ENCCL;
}

bool Watchdog::aborted() const { return p && p->aborted.load(); }

void Watchdog::lock() {
  if (p) p->nccl_m.lock();
}

void Watchdog::unlock() {
  if (p) p->nccl_m.unlock();
}

int Watchdog::stall(cudaStream_t st, std::string* err) {
  if (!p) return 0;
  int* dflag = nullptr;
  if (cudaHostGetDevicePointer(reinterpret_cast<void**>(&dflag), p->stall_flag, 0) != cudaSuccess) {
    if (err) *err = "watchdog: cudaHostGetDevicePointer";
    return TRAJ_ECUDA;
  }
  stall_kernel<<<1, 32, 0, st>>>(dflag);
  count_launch();
  return 0;
}

bool Watchdog::stop() {
  if (!p) return false;
  p->quit.store(true);
  p->cv.notify_all();
  if (p->th.joinable()) p->th.join();
  const bool ab = p->aborted.load();
  for (auto& e : p->pending) cudaEventDestroy(e.first);
  for (auto e : p->pool) cudaEventDestroy(e);
  if (p->stall_flag) cudaFreeHost(p->stall_flag);
  delete p;
  p = nullptr;
  return ab;
}

}  // namespace traj
