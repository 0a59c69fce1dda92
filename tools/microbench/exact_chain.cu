// Cycle cost of the coarse pick's exact phase: n candidate chains of dp
// reference-arithmetic steps, rows streamed through a 2-slot cp.async ring
// in column blocks (as coarse_pick_kernel), vs the same chains on rows
// already in shared memory (compute only); modes 2/3 run the chains with
// packed f32x2 sub / mul (bit-identical, fewer instructions).  Measured on
// B200: ~12 cycles per element of one chain in every variant, i.e. the
// dependent sequential add chain, not the loads or the issue rate, bounds
// the exact re-rank (768 elements ~ 4.7 us).
#include "../../paper_2602_21477_b200/csrc/pk_kernels.cu"
using namespace pk;
// w floats (multiple of 16) of one chain, loads for the next 16 issued
// before the current 16 are summed (register double buffer)
// packed f32x2 sub / mul (each lane of the pair rounded like the scalar
// op), scalar sequential adds: 4 instructions per 2 elements instead of 6
__device__ __forceinline__ unsigned long long f2_sub(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long f2_mul(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
template <int METRIC>
__device__ __forceinline__ float chain_pipelined(float acc, const float* x, const float* q, int w) {
  const ulonglong2* x4 = reinterpret_cast<const ulonglong2*>(x);
  const ulonglong2* q4 = reinterpret_cast<const ulonglong2*>(q);
#pragma unroll 4
  for (int c = 0; c < w / 4; c++) {
    const ulonglong2 xv = x4[c], qv = q4[c];
    const unsigned long long t0 = f2_sub(xv.x, qv.x), t1 = f2_sub(xv.y, qv.y);
    const unsigned long long m0 = f2_mul(t0, t0), m1 = f2_mul(t1, t1);
    acc = __fadd_rn(acc, __uint_as_float((unsigned)m0));
    acc = __fadd_rn(acc, __uint_as_float((unsigned)(m0 >> 32)));
    acc = __fadd_rn(acc, __uint_as_float((unsigned)m1));
    acc = __fadd_rn(acc, __uint_as_float((unsigned)(m1 >> 32)));
  }
  return acc;
}
__global__ void kexact(const float* cent, const int* pick, int n, int dp, int stage_floats, int mode,
                       long long* cyc, float* out) {
  extern __shared__ __align__(16) float sm[];
  float* qs = sm;
  float* rows_st = sm + dp;
  const int tid = threadIdx.x;
  for (int j = tid; j < dp; j += blockDim.x) qs[j] = 0.001f * j;
  __syncthreads();
  long long t0 = clock64();
  const int nr = n, nd32 = dp / DC;
  int k = 1;
  for (int kk2 = nd32; kk2 >= 1; kk2--)
    if (nd32 % kk2 == 0 && 2 * nr * (DC * kk2 + 4) <= stage_floats) { k = kk2; break; }
  const int W = DC * k, rs = W + 4, nblk = nd32 / k;
  auto issue = [&](int blk) {
    float* dst = rows_st + (blk & 1) * nr * rs;
    const int w4 = W / 4;
    for (int i = tid; i < nr * w4; i += blockDim.x) {
      const int r = i / w4, c = i - r * w4;
      if (mode == 0 || mode == 2) cp_async16(dst + r * rs + 4 * c, cent + (int64_t)pick[r] * dp + blk * W + 4 * c);
    }
    cp_async_commit();
  };
  issue(0);
  float acc = 0.f;
  for (int blk = 0; blk < nblk; blk++) {
    if (blk + 1 < nblk) { issue(blk + 1); cp_async_wait<1>(); } else { cp_async_wait<0>(); }
    __syncthreads();
    if (tid < nr) {
      const float* x = rows_st + (blk & 1) * nr * rs + tid * rs;
      const float* q = qs + blk * W;
      if (mode >= 2) acc = chain_pipelined<SQ_L2>(acc, x, q, W);
      else
      for (int j = 0; j + 4 <= W; j += 4)
        acc = step4<SQ_L2>(acc, *reinterpret_cast<const float4*>(x + j), *reinterpret_cast<const float4*>(q + j));
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid < nr) out[blockIdx.x * 256 + tid] = acc;
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  const int dp = 768, nl = 1024;
  float* cent; int* pick; long long* cyc; float* out;
  cudaMalloc(&cent, (size_t)nl * dp * 4); cudaMemset(cent, 0, (size_t)nl * dp * 4);
  cudaMalloc(&pick, 256 * 4); cudaMalloc(&cyc, 256 * 8); cudaMalloc(&out, 256 * 256 * 4);
  int hp[256]; for (int i = 0; i < 256; i++) hp[i] = (i * 37) % nl;
  cudaMemcpy(pick, hp, sizeof(hp), cudaMemcpyHostToDevice);
  const int stage = 21000;
  const size_t smem = (size_t)(dp + stage) * 4;
  cudaFuncSetAttribute(kexact, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int mode = 0; mode < 4; mode++)
    for (int n : {16, 32, 50, 64}) {
      for (int grid : {1, 256}) {
        kexact<<<grid, 256, smem>>>(cent, pick, n, dp, stage, mode, cyc, out);
        kexact<<<grid, 256, smem>>>(cent, pick, n, dp, stage, mode, cyc, out);
        cudaDeviceSynchronize();
        long long h[256]; cudaMemcpy(h, cyc, 8 * grid, cudaMemcpyDeviceToHost);
        double s = 0; for (int i = 0; i < grid; i++) s += h[i];
        printf("{\"mode\": \"%s\", \"n\": %d, \"grid\": %d, \"cycles\": %.0f}\n", mode == 0 ? "cp.async" : mode == 1 ? "compute-only" : mode == 2 ? "cp.async+pipelined" : "compute-only+pipelined",
               n, grid, s / grid);
      }
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
