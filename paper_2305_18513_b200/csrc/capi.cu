// Error plumbing and device queries shared by every entry point.
#include "common.cuh"

namespace sf {

static thread_local int g_last_cuda_error = 0;

void set_cuda_error(cudaError_t e) { g_last_cuda_error = static_cast<int>(e); }

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cached[dev] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    cached[dev] = v;
  }
  return cached[dev];
}

}  // namespace sf

extern "C" {

int sf_abi_version(void) { return 1; }

int sf_last_cuda_error(void) { return sf::g_last_cuda_error; }

const char* sf_strerror(int code) {
  switch (code) {
    case SF_OK: return "ok";
    case SF_EINVAL: return "invalid argument";
    case SF_ERANGE: return "value outside the codec range";
    case SF_ECUDA: return cudaGetErrorString(static_cast<cudaError_t>(sf::g_last_cuda_error));
    default: return "unknown error";
  }
}

}  // extern "C"
