// devmem.cu -- device allocations of the library (every DBuf), with the
// FMM_POISON=1 debug mode described in common.cuh: poison-filled storage and
// guard zones after every buffer, checked after every API call.
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace fmmb {

namespace {
constexpr unsigned char kPoison = 0xff;   // NaN as float/double, -1 as integers
constexpr unsigned char kGuard = 0xa5;
std::mutex g_mu;
std::unordered_map<void*, size_t>& live() {   // buffer -> its size in bytes (guard zone follows)
  static std::unordered_map<void*, size_t> m;
  return m;
}
}  // namespace

bool poison_mode() {
  static const bool on = [] {
    const char* e = getenv("FMM_POISON");
    return e && atoi(e) != 0;
  }();
  return on;
}

void* dev_alloc(size_t bytes) {
  void* p = nullptr;
  if (!poison_mode()) {
    FMM_CUDA(cudaMalloc(&p, bytes));
    return p;
  }
  FMM_CUDA(cudaMalloc(&p, bytes + kGuardBytes));
  FMM_CUDA(cudaMemset(p, kPoison, bytes));
  FMM_CUDA(cudaMemset((char*)p + bytes, kGuard, kGuardBytes));
  FMM_CUDA(cudaDeviceSynchronize());
  std::lock_guard<std::mutex> lk(g_mu);
  live()[p] = bytes;
  return p;
}

void dev_free(void* p) {
  if (!p) return;
  if (poison_mode()) {
    std::lock_guard<std::mutex> lk(g_mu);
    live().erase(p);
  }
  cudaFree(p);
}

void guard_check(const char* where) {
  std::lock_guard<std::mutex> lk(g_mu);
  std::vector<unsigned char> h(kGuardBytes);
  for (const auto& kv : live()) {
    FMM_CUDA(cudaMemcpy(h.data(), (const char*)kv.first + kv.second, kGuardBytes, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < kGuardBytes; ++i)
      if (h[i] != kGuard)
        throw FmmError(FMM_E_INTERNAL, std::string("FMM_POISON: write past the end of a device buffer of ") +
                                           std::to_string(kv.second) + " bytes (guard byte " + std::to_string(i) +
                                           ") " + where);
  }
}

}  // namespace fmmb
