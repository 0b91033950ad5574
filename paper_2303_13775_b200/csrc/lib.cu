// Library-level state: error message, launch counter, version.
#include <cstdlib>
#include <mutex>
#include <string>

#include "common.cuh"

namespace sg {
std::atomic<unsigned long long> g_launches{0};
bool g_pdl = [] {
  const char* e = getenv("SG_PDL");
  return !(e && e[0] == '0');
}();
static std::mutex g_err_mu;
static thread_local std::string g_err;
void set_error(const std::string& msg) {
  std::lock_guard<std::mutex> lk(g_err_mu);
  g_err = msg;
}
}  // namespace sg

extern "C" const char* sg_last_error(void) { return sg::g_err.c_str(); }
extern "C" const char* sg_version(void) { return "splitgnn-b200 0.1 (sm_100a)"; }
extern "C" unsigned long long sg_launch_count(void) { return sg::g_launches.load(); }
extern "C" void sg_set_pdl(int on) { sg::g_pdl = on != 0; }
extern "C" int sg_get_pdl(void) { return sg::g_pdl ? 1 : 0; }
extern "C" int sg_device_sm_count(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return n;
}

// ABI self-check used by the Python binding: sizes of the shared structs.
extern "C" void sg_struct_sizes(int64_t* out) {
  out[0] = (int64_t)sizeof(SgMeta);
  out[1] = (int64_t)sizeof(SgSplitLayout);
}
