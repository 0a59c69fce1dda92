// Microbenchmark (sm_100a): HBM streaming rate of TMA access patterns over a
// [rows x 768] fp32 matrix, consumers doing no work.
//   tile : 2-D box 32 floats x 256 rows, 24 column chunks per row tile (the scan's pattern)
//   rows : 3-D view (32, 24, rows), box 32 x 24 x 8 -> 8 contiguous full rows per stage
//   bulk : 1-D cp.async.bulk of contiguous 32 KB
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2602_21477_b200/csrc/pk_ptx.cuh"
using namespace pk;
constexpr int D = 768, STAGES = 4;
struct Maps { CUtensorMap tile, rows; };

template <int MODE>
__global__ void __launch_bounds__(64, 1) stream_k(const __grid_constant__ Maps m, const float* base, int64_t nrows, int* ctr, int per_item_rows) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  uint64_t* full = (uint64_t*)(sm + STAGES * 32768);
  uint64_t* empty = full + STAGES;
  if (threadIdx.x == 0) { for (int i = 0; i < STAGES; i++) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); } fence_mbar_init(); }
  __syncthreads();
  const int64_t nitems = nrows / per_item_rows;
  const int stages_per_item = MODE == 0 ? 24 * (per_item_rows / 256) : (MODE == 1 ? per_item_rows / 8 : per_item_rows * 3072 / 32768);
  __shared__ volatile int done, nst;
  if (threadIdx.x == 0) { done = 0; nst = 0; }
  __syncthreads();
  if (threadIdx.x == 32) {  // producer
    int s = 0; uint32_t ph = 0; int issued = 0;
    for (;;) {
      int it = atomicAdd(ctr, 1);
      if (it >= nitems) break;
      int64_t r0 = (int64_t)it * per_item_rows;
      for (int k = 0; k < stages_per_item; k++) {
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* dst = sm + s * 32768;
        if (MODE == 0) {
          mbar_arrive_expect_tx(&full[s], 32768);
          int t = k / 24, c = k % 24;
          asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
            :: "r"(smem_u32(dst)), "l"((uint64_t)&m.tile), "r"(smem_u32(&full[s])), "r"(c * 32), "r"((int)(r0 + t * 256)) : "memory");
        } else if (MODE == 1) {
          mbar_arrive_expect_tx(&full[s], 24576);
          asm volatile("cp.async.bulk.tensor.3d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
            :: "r"(smem_u32(dst)), "l"((uint64_t)&m.rows), "r"(smem_u32(&full[s])), "r"(0), "r"(0), "r"((int)(r0 + k * 8)) : "memory");
        } else {
          mbar_arrive_expect_tx(&full[s], 32768);
          bulk_g2s(dst, (const uint8_t*)base + (r0 * 3072 + (int64_t)k * 32768), 32768, &full[s]);
        }
        issued++;
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
    nst = issued;
    __threadfence_block();
    done = 1;
  } else if (threadIdx.x == 0) {  // consumer: drains every stage the producer issued
    int s = 0; uint32_t ph = 0; int consumed = 0;
    for (;;) {
      if (done && consumed == nst) break;
      uint32_t ok;
      asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok) : "r"(smem_u32(&full[s])), "r"(ph) : "memory");
      if (ok) {
        mbar_arrive(&empty[s]);
        consumed++;
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
  }
}

int main() {
  const int64_t nrows = 1 << 20;  // 1M x 768 fp32 = 3.2 GB
  float* base; cudaMalloc(&base, nrows * 3072); cudaMemset(base, 0, nrows * 3072);
  PFN_cuTensorMapEncodeTiled_v12000 enc; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  Maps m;
  { cuuint64_t gd[2] = {768, (cuuint64_t)nrows}; cuuint64_t gs[1] = {3072}; cuuint32_t bx[2] = {32, 256}; cuuint32_t es[2] = {1, 1};
    enc(&m.tile, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, gd, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE); }
  { cuuint64_t gd[3] = {32, 24, (cuuint64_t)nrows}; cuuint64_t gs[2] = {128, 3072}; cuuint32_t bx[3] = {32, 24, 8}; cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&m.rows, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, gd, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) printf("rows map err %d\n", r); }
  int* ctr; cudaMalloc(&ctr, 4);
  int smem = STAGES * 32768 + 2048;
  cudaFuncSetAttribute(stream_k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(stream_k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(stream_k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[3] = {"tile 32x256 (scan pattern)", "rows 3-D 8 full rows", "bulk 32KB contiguous"};
  for (int rep = 0; rep < 3; rep++) for (int mode = 0; mode < 3; mode++) for (int ctas : {148, 296}) {
    cudaMemset(ctr, 0, 4);
    cudaEventRecord(a);
    if (mode == 0) stream_k<0><<<ctas, 64, smem>>>(m, base, nrows, ctr, 512);
    if (mode == 1) stream_k<1><<<ctas, 64, smem>>>(m, base, nrows, ctr, 512);
    if (mode == 2) stream_k<2><<<ctas, 64, smem>>>(m, base, nrows, ctr, 512);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (rep == 2) printf("%-30s ctas=%d  %.3f ms  %.0f GB/s\n", names[mode], ctas, ms, nrows * 3072.0 / ms / 1e6);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
