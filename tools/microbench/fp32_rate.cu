// Microbenchmark (sm_100a): throughput of the exact no-FMA squared-L2 step
// acc = acc + (x - q)^2 (each op RN) in scalar and packed-f32x2 forms.
// ptxas contracts mul.rn.f32x2 + add.rn.f32x2 into FFMA2 (observed with nvcc 12.9),
// so the exact packed variants split or fence the multiply.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define NACC 16
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) { u64 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void upk(u64 v, float& a, float& b) { asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__device__ __forceinline__ u64 sub2(u64 a, u64 b) { u64 r; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 mul2(u64 a, u64 b) { u64 r; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 add2(u64 a, u64 b) { u64 r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }

template <int MODE>  // 0 scalar, 1 packed fused (inexact; rate reference), 2 packed split-mul, 3 packed lop-fenced
__global__ void k(const float* __restrict__ in, float* out, int iters, u64 zero) {
  u64 acc[NACC/2], x[NACC/2];
  float accs[NACC], xs[NACC];
  #pragma unroll
  for (int i = 0; i < NACC/2; i++) {
    xs[2*i] = in[(threadIdx.x + 2*i) & 255]; xs[2*i+1] = in[(threadIdx.x + 2*i + 1) & 255];
    x[i] = pk(xs[2*i], xs[2*i+1]); acc[i] = 0ull; accs[2*i] = 0.f; accs[2*i+1] = 0.f;
  }
  float qs = in[256 + (blockIdx.x & 255)];
  for (int it = 0; it < iters; it++) {
    if (MODE == 0) {
      #pragma unroll
      for (int i = 0; i < NACC; i++) { float t = __fsub_rn(xs[i], qs); accs[i] = __fadd_rn(accs[i], __fmul_rn(t, t)); }
    } else {
      u64 q = pk(qs, qs);
      #pragma unroll
      for (int i = 0; i < NACC/2; i++) {
        u64 t = sub2(x[i], q), s;
        if (MODE == 1) s = mul2(t, t);
        if (MODE == 2) { float a, b; upk(t, a, b); s = pk(__fmul_rn(a, a), __fmul_rn(b, b)); }
        if (MODE == 3) { s = mul2(t, t) ^ zero; }
        acc[i] = add2(acc[i], s);
      }
    }
    qs = in[512 + (it & 255)];
  }
  float s0 = 0.f;
  #pragma unroll
  for (int i = 0; i < NACC/2; i++) {
    float a, b;
    if (MODE == 0) { a = accs[2*i]; b = accs[2*i+1]; } else upk(acc[i], a, b);
    out[(size_t)(blockIdx.x * blockDim.x + threadIdx.x) * NACC + 2*i] = a;
    out[(size_t)(blockIdx.x * blockDim.x + threadIdx.x) * NACC + 2*i + 1] = b;
  }
}
int main() {
  const int NB = 148 * 8, NT = 256; const size_t NOUT = (size_t)NB * NT * NACC;
  float *in, *out[4]; cudaMalloc(&in, 1024 * 4);
  for (int m = 0; m < 4; m++) cudaMalloc(&out[m], NOUT * 4);
  float h[1024]; uint32_t s = 12345;
  for (int i = 0; i < 1024; i++) { s = s * 1664525u + 1013904223u; h[i] = ((s >> 8) / 16777216.f) * 2.f - 1.f; }
  cudaMemcpy(in, h, 4096, cudaMemcpyHostToDevice);
  int iters = 20000; cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[4] = {"scalar FADD/FMUL/FADD", "packed FFMA2 (fused, INEXACT)", "packed FADD2+2xFMUL+FADD2", "packed FADD2+FMUL2+LOP+FADD2"};
  for (int rep = 0; rep < 2; rep++) for (int m = 0; m < 4; m++) {
    float ms;
    cudaEventRecord(a);
    if (m == 0) k<0><<<NB, NT>>>(in, out[0], iters, 0ull);
    if (m == 1) k<1><<<NB, NT>>>(in, out[1], iters, 0ull);
    if (m == 2) k<2><<<NB, NT>>>(in, out[2], iters, 0ull);
    if (m == 3) k<3><<<NB, NT>>>(in, out[3], iters, 0ull);
    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    double pairs = (double)NACC * iters * NB * NT;
    if (rep) printf("%-34s %8.3f ms  %7.2f T (q,elem)/s  = %6.2f T fp32-ops/s\n", names[m], ms, pairs / ms / 1e9, 3 * pairs / ms / 1e9);
  }
  float* hb = (float*)malloc(NOUT * 4); float* hr = (float*)malloc(NOUT * 4);
  cudaMemcpy(hr, out[0], NOUT * 4, cudaMemcpyDeviceToHost);
  for (int m = 1; m < 4; m++) {
    cudaMemcpy(hb, out[m], NOUT * 4, cudaMemcpyDeviceToHost);
    size_t bad = 0; for (size_t i = 0; i < NOUT; i++) bad += (*(uint32_t*)&hb[i] != *(uint32_t*)&hr[i]);
    printf("%-34s bitwise mismatches vs scalar: %zu / %zu\n", names[m], bad, NOUT);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
