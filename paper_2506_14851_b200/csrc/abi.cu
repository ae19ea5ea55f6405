// C-ABI plumbing: error text, device queries.
#include <cstdarg>
#include <cstdio>

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
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
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
