// Does stream completion stay in order when a PDL secondary skips
// griddepcontrol.wait?  A spins (after triggering dependents), B is a
// PDL secondary that never waits, C reads A's flag.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void kA(volatile int* flag, long long spin) {
  asm volatile("griddepcontrol.launch_dependents;");
  long long t0 = clock64();
  while (clock64() - t0 < spin) {}
  __threadfence();
  *flag = 1;
}
__global__ void kB(int* mark) { *mark = 1; }
__global__ void kC(volatile int* flag, int* seen, int wait) {
  if (wait) asm volatile("griddepcontrol.wait;" ::: "memory");
  *seen = *flag;
}
template <typename... KA, typename... A>
static void pdl(void (*k)(KA...), cudaStream_t st, A... a) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1); cfg.blockDim = dim3(32); cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, static_cast<KA>(a)...);
}
int main() {
  int *flag, *mark, *seen;
  cudaMalloc(&flag, 4); cudaMalloc(&mark, 4); cudaMalloc(&seen, 4);
  cudaStream_t st; cudaStreamCreate(&st);
  for (int mode = 0; mode < 4; mode++) {
    // mode 0: C normal launch after B(pdl,no wait)
    // mode 1: C pdl + wait after B(pdl,no wait)
    // mode 2: C pdl, no wait (control: expect 0)
    // mode 3: B pdl no wait, B2 pdl no wait, C normal
    int bad = 0;
    for (int it = 0; it < 20; it++) {
      cudaMemsetAsync(flag, 0, 4, st); cudaMemsetAsync(seen, 0xff, 4, st);
      kA<<<1, 32, 0, st>>>(flag, 20000000LL);
      pdl(kB, st, mark);
      if (mode == 3) pdl(kB, st, mark);
      if (mode == 0 || mode == 3) kC<<<1, 32, 0, st>>>(flag, seen, 0);
      else pdl(kC, st, (volatile int*)flag, seen, mode == 1 ? 1 : 0);
      int h; cudaMemcpy(&h, seen, 4, cudaMemcpyDeviceToHost);
      if (h != 1) bad++;
    }
    printf("{\"mode\": %d, \"saw_unfinished_A\": %d, \"of\": 20}\n", mode, bad);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
