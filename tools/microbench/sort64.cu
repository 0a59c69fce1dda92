// Cycle cost of block_sort_keep on <= 64 entries (the coarse pick's sort phase).
#include "../../paper_2602_21477_b200/csrc/pk_kernels.cu"
using namespace pk;
__global__ void kbench(int n, long long* cyc, int* out) {
  __shared__ Entry buf[1024];
  __shared__ int s_cnt;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    unsigned h = (i * 2654435761u) ^ (blockIdx.x * 97u);
    buf[i].key = h >> 4;
    buf[i].id = (int64_t)(h & 1023);
    buf[i].pay = i;
  }
  __syncthreads();
  long long t0 = clock64();
  int kept = block_sort_keep(buf, n, 32, false, &s_cnt);
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x] = kept + buf[0].pay;
  }
}
int main() {
  long long* cyc;
  int* out;
  cudaMalloc(&cyc, 256 * 8);
  cudaMalloc(&out, 256 * 4);
  for (int n : {16, 32, 50, 64, 100, 200}) {
    for (int rep = 0; rep < 2; rep++) kbench<<<256, 256>>>(n, cyc, out);
    cudaDeviceSynchronize();
    long long h[256];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double s = 0;
    for (long long v : h) s += v;
    printf("{\"n\": %d, \"cycles_mean\": %.0f}\n", n, s / 256);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
