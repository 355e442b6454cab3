// launch_cache.cpp -- host-side caches of per-kernel launch attributes.
//
// cudaFuncSetAttribute (dynamic shared memory opt-in), the occupancy query and
// the SM-count attribute each cost ~1-3 us of host time per call; issued
// before every launch they dominated the host path of small contractions
// (config 1: 20 contracts of <= 16^3 MACs; the config-5 sweep's small
// instances). They are answered here from a per-(kernel, device) table.
#include <mutex>
#include <unordered_map>

#include "tci_internal.h"

namespace tci {
namespace {

struct Key {
  const void *fn;
  int dev, threads;
  size_t smem;
  bool operator==(const Key &o) const { return fn == o.fn && dev == o.dev && threads == o.threads && smem == o.smem; }
};
struct KeyHash {
  size_t operator()(const Key &k) const {
    return std::hash<const void *>()(k.fn) ^ (std::hash<size_t>()(k.smem) * 31) ^ ((size_t)k.threads << 20) ^
           ((size_t)k.dev << 40);
  }
};

std::mutex g_mu;
std::unordered_map<Key, int, KeyHash> g_smem;   // (fn, dev) -> largest opt-in set so far (smem field unused)
std::unordered_map<Key, int, KeyHash> g_occ;    // (fn, dev, threads, smem) -> blocks per SM
int g_sms[64] = {0};

}  // namespace

cudaError_t ensure_smem_attr(const void *fn, size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  const Key k{fn, dev, 0, 0};
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_smem.find(k);
    if (it != g_smem.end() && (size_t)it->second >= bytes) return cudaSuccess;
  }
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_mu);
  int &v = g_smem[k];
  if ((size_t)v < bytes) v = (int)bytes;
  return cudaSuccess;
}

int occupancy_per_sm(const void *fn, int threads, size_t smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  const Key k{fn, dev, threads, smem};
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_occ.find(k);
    if (it != g_occ.end()) return it->second;
  }
  int per_sm = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  std::lock_guard<std::mutex> lk(g_mu);
  g_occ[k] = per_sm;
  return per_sm;
}

int device_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  int v = g_sms[dev];
  if (!v) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    g_sms[dev] = v;
  }
  return v;
}

}  // namespace tci
