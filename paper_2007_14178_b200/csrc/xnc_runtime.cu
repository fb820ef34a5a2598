// Per-device launch state shared by the kernel launchers: the dynamic
// shared-memory opt-in and the SM count, cached per (device, function) under a
// mutex so that several GPUs (and host threads) can drive one process.
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "xnc_common.cuh"

namespace xnc {

namespace {

constexpr int kMaxDevices = 64;

struct KeyHash {
  size_t operator()(const std::pair<const void*, int>& k) const {
    return std::hash<const void*>()(k.first) ^ (std::hash<int>()(k.second) * 0x9e3779b97f4a7c15ull);
  }
};

std::mutex g_mu;
std::unordered_map<std::pair<const void*, int>, size_t, KeyHash> g_opted;  // (func, device) -> bytes
int g_sms[kMaxDevices] = {};

}  // namespace

int smem_opt_in(const void* func, size_t bytes) {
  if (bytes <= 48 * 1024) return XNC_OK;  // no opt-in needed
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return XNC_ECUDA_BASE + (int)e;
  std::lock_guard<std::mutex> lock(g_mu);
  size_t& have = g_opted[{func, dev}];
  if (bytes <= have) return XNC_OK;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return XNC_ECUDA_BASE + (int)e;
  have = bytes;
  return XNC_OK;
}

int pdl_enabled() {
  static const int on = getenv("XNC_PDL") ? atoi(getenv("XNC_PDL")) : 1;
  return on;
}

int device_sm_count() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return 148;
  if (dev >= kMaxDevices) {
    int sms = 0;
    return cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && sms >= 2 ? sms : 148;
  }
  std::lock_guard<std::mutex> lock(g_mu);
  if (!g_sms[dev]) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms < 2) sms = 148;
    g_sms[dev] = sms;
  }
  return g_sms[dev];
}

}  // namespace xnc
