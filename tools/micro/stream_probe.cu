// Streaming-read microbenchmark: how fast can one 1024-thread CTA per SM
// (warp-contiguous ranges) read 50 MB, with register loads vs a cp.async
// ring, and with the prune's per-element classify + ballot work added.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(1024, 1) k_regs(const float* __restrict__ x, long n, unsigned* out) {
  const long W = (long)gridDim.x * 32, gw = (long)blockIdx.x * 32 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const long nq = n / 16, a = gw * nq / W * 16, e = (gw + 1) * nq / W * 16;
  unsigned acc = 0;
  for (long c = a + 4 * lane; c < e; c += 128 * 2) {
    float4 p = *reinterpret_cast<const float4*>(x + c);
    float4 q = c + 128 < e ? *reinterpret_cast<const float4*>(x + c + 128) : make_float4(0, 0, 0, 0);
    acc += (p.x > 1.6f) + (p.y > 1.6f) + (p.z > 1.6f) + (p.w > 1.6f) + (q.x > 1.6f) + (q.y > 1.6f) + (q.z > 1.6f) + (q.w > 1.6f);
  }
  if (acc == 12345) out[0] = acc;
}

template <int STAGES, bool WORK>
__global__ void __launch_bounds__(1024, 1) k_ring(const float* __restrict__ x, long n, unsigned* out) {
  extern __shared__ float ring[];
  const long W = (long)gridDim.x * 32, gw = (long)blockIdx.x * 32 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long nq = n / 16, a = gw * nq / W * 16, e = (gw + 1) * nq / W * 16;
  float* wr = ring + warp * STAGES * 256;
  const uint32_t ws = (uint32_t)__cvta_generic_to_shared(wr);
  const long ns = (e - a) / 256;
  auto issue = [&](long c) {
    if (c < ns) {
      const long b = a + c * 256;
      for (int q = 0; q < 2; ++q) {
        const int p = lane + 32 * q;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(ws + (uint32_t)((c % STAGES) * 1024 + 16 * p)),
                     "l"(x + b + 4 * p) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int c = 0; c < STAGES - 1; ++c) issue(c);
  unsigned acc = 0, run = 0;
  for (long c = 0; c < ns; ++c) {
    issue(c + STAGES - 1);
    asm volatile("cp.async.wait_group %0;" ::"n"(STAGES - 1) : "memory");
    __syncwarp();
    const float* slot = wr + (c % STAGES) * 256;
    for (int t = 0; t < 8; ++t) {
      const float v = slot[lane + 32 * t];
      if (WORK) {
        const uint32_t d = (__float_as_uint(v) & 0x7FFFFFFFu) - 0x3FC00000u;
        const bool keep = d <= 0x3FC00000u;
        const unsigned kb = __ballot_sync(~0u, keep);
        acc += __popc(kb & ((1u << lane) - 1)) + run;
        run += __popc(kb);
      } else {
        acc += v > 1.6f;
      }
    }
    __syncwarp();
  }
  if (acc == 12345) out[0] = acc;
}

int main() {
  const long n = 12582912;
  float* x;
  unsigned* o;
  cudaMalloc(&x, n * 4);
  cudaMalloc(&o, 4);
  cudaMemset(x, 0, n * 4);
  float* fl;
  cudaMalloc(&fl, 256 << 20);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k_ring<4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 4 * 1024);
  cudaFuncSetAttribute(k_ring<4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 4 * 1024);
  cudaFuncSetAttribute(k_ring<6, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 6 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int v = 0; v < 5; ++v) {
    for (int flush = 0; flush < 2; ++flush) {
      float best = 1e9;
      for (int it = 0; it < 10; ++it) {
        if (flush) cudaMemsetAsync(fl, it, 256 << 20);
        cudaEventRecord(e0);
        if (v == 0) k_regs<<<sms, 1024>>>(x, n, o);
        if (v == 1) k_ring<4, false><<<sms, 1024, 32 * 4 * 1024>>>(x, n, o);
        if (v == 2) k_ring<4, true><<<sms, 1024, 32 * 4 * 1024>>>(x, n, o);
        if (v == 3) k_ring<6, true><<<sms, 1024, 32 * 6 * 1024>>>(x, n, o);
        if (v == 4) k_regs<<<sms * 2, 512>>>(x, n, o);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      const char* nm[] = {"regs 1024x148", "ring4", "ring4+work", "ring6+work", "regs 512x296"};
      printf("%-16s %s: %.1f us  %.0f GB/s\n", nm[v], flush ? "cold" : "warm", best * 1e3, n * 4 / (best * 1e-3) / 1e9);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
