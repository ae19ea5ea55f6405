// C-ABI plumbing: error text, device queries.
#include <cstdarg>
#include <cstdio>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace pdg {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int sm_count() {
  static int cached[64] = {};
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) != cudaSuccess) return n;
  if (dev >= 0 && dev < 64 && cached[dev] > 0) return cached[dev];
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (n <= 0) n = 148;
  if (dev >= 0 && dev < 64) cached[dev] = n;
  return n;
}

namespace {
struct LaunchKey {          // resident blocks per SM of one launch shape
  const void* kern;
  int threads, dev;
  size_t smem;
  int per_sm;
};
struct SmemAttr {           // the kernel's max dynamic shared memory, as set
  const void* kern;
  int dev;
  size_t smem;
};
std::mutex g_launch_mu;
std::vector<LaunchKey> g_launch;
std::vector<SmemAttr> g_attr;
}  // namespace

int launch_setup(const void* kern, int threads, size_t smem, int* per_sm) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice");
  std::lock_guard<std::mutex> lk(g_launch_mu);
  // the attribute only ever grows: a smaller launch after a larger one keeps
  // the larger limit, so every cached shape stays launchable
  SmemAttr* at = nullptr;
  for (SmemAttr& x : g_attr)
    if (x.kern == kern && x.dev == dev) at = &x;
  if (!at || at->smem < smem) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute");
    if (at) at->smem = smem;
    else g_attr.push_back(SmemAttr{kern, dev, smem});
  }
  for (const LaunchKey& k : g_launch)
    if (k.kern == kern && k.threads == threads && k.dev == dev && k.smem == smem) {
      *per_sm = k.per_sm;
      return PDG_OK;
    }
  int n = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, threads, smem);
  if (e != cudaSuccess) return cuda_status(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
  if (n < 1) {
    set_error("kernel does not fit on an SM (%d threads, %zu B shared memory)", threads, smem);
    return PDG_EUNSUPPORTED;
  }
  g_launch.push_back(LaunchKey{kern, threads, dev, smem, n});
  *per_sm = n;
  return PDG_OK;
}

}  // namespace pdg

extern "C" const char* pdg_last_error(void) { return pdg::g_err; }

extern "C" int pdg_abi_version(void) { return 3; }

extern "C" int pdg_device_info(int* sms, int* major, int* minor) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return pdg::cuda_status(e, "cudaGetDevice");
  cudaDeviceProp p;
  e = cudaGetDeviceProperties(&p, dev);
  if (e != cudaSuccess) return pdg::cuda_status(e, "cudaGetDeviceProperties");
  if (sms) *sms = p.multiProcessorCount;
  if (major) *major = p.major;
  if (minor) *minor = p.minor;
  if (p.major != 10) {
    pdg::set_error("device is sm_%d%d; this library is built for sm_100a only", p.major,
                   p.minor);
    return PDG_ENODEV;
  }
  return PDG_OK;
}
