// Read-only HBM streaming bandwidth on this B200 (the posting-list scan is a
// pure read stream; MEASURED_PEAKS.json hbm_gbs comes from a read+write copy).
// Grid-stride 128-bit loads over a 16 GiB buffer, persistent 148 x k CTAs,
// timed with CUDA events, best of 10.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void read_kernel(const float4* __restrict__ p, size_t n4, float* out) {
  float acc = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = __ldcs(p + i);
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 12345.f) out[0] = acc;  // keep the loads
}

int main() {
  const size_t bytes = 16ull << 30;
  float4* p;
  float* out;
  cudaMalloc(&p, bytes);
  cudaMalloc(&out, 4);
  cudaMemset(p, 0, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int per = 4; per <= 16; per *= 2) {
    float best = 1e9f;
    for (int r = 0; r < 10; r++) {
      cudaEventRecord(a);
      read_kernel<<<sms * per, 512>>>(p, bytes / 16, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("{\"ctas_per_sm\": %d, \"read_gbs\": %.1f}\n", per, bytes / (best * 1e-3) / 1e9);
  }
  return 0;
}
