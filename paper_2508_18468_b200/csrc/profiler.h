// Per-phase CUDA-event timing and launch counting shared by the unsharded and the
// row-sharded step (traj_profile / traj_phase_times).
#pragma once
#include <tuple>
#include <vector>
#include "common.cuh"

namespace traj {

constexpr int NPHASES = 11;

struct Profiler {
  bool on = false;
  std::vector<std::tuple<int, cudaEvent_t, cudaEvent_t>> evs;
  std::vector<cudaEvent_t> pool;
  double ms[NPHASES] = {0};
  long long launches[NPHASES] = {0};

  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  void collect() {   // caller has synchronised the stream
    for (auto& e : evs) {
      float t = 0;
      cudaEventElapsedTime(&t, std::get<1>(e), std::get<2>(e));
      ms[std::get<0>(e)] += t;
      pool.push_back(std::get<1>(e));
      pool.push_back(std::get<2>(e));
    }
    evs.clear();
  }
  void reset(bool enable) {
    collect();
    for (int p = 0; p < NPHASES; ++p) {
      ms[p] = 0;
      launches[p] = 0;
    }
    on = enable;
  }
  void destroy() {
    for (auto& e : evs) {
      cudaEventDestroy(std::get<1>(e));
      cudaEventDestroy(std::get<2>(e));
    }
    evs.clear();
    for (auto e : pool) cudaEventDestroy(e);
    pool.clear();
  }
};

struct Phase {
  Profiler* p;
  cudaStream_t st;
  int ph;
  cudaEvent_t a = nullptr;
  long long l0;
  Phase(Profiler* p_, cudaStream_t s, int phase) : p(p_), st(s), ph(phase), l0(g_kernel_launches.load()) {
    if (p->on) {
      a = p->get();
      cudaEventRecord(a, st);
    }
  }
  ~Phase() {
    p->launches[ph] += g_kernel_launches.load() - l0;
    if (!p->on) return;
    cudaEvent_t b = p->get();
    cudaEventRecord(b, st);
    p->evs.emplace_back(ph, a, b);
  }
};

}  // namespace traj
