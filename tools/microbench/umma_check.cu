// Validation of the tcgen05 TF32 screen primitives (pk_umma.cuh) on sm_100a:
//  1. layout: D = X . Q^T through TMA (SWIZZLE_128B) + UMMA descriptors matches
//     a double-precision reference to TF32 accuracy (a wrong descriptor gives
//     garbage, not small errors);
//  2. error bound: max |D - exact| / sum_j |x_j q_j| over random and adversarial
//     inputs, against the coefficient the screen uses (2.0011 * 2^-10 + d * 2^-21).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_2602_21477_b200/csrc/pk_umma.cuh"
using namespace pk;

constexpr int D = 768, ROWS = 256, NQ = 16, DCH = 32;

__global__ void __launch_bounds__(256, 1) check_k(const __grid_constant__ CUtensorMap xmap, const float* qsw,
                                                  float* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  float* X = (float*)sm;                  // 256 x 32 fp32 (32 KB), SW128
  float* Qs = (float*)(sm + 32768);       // 16 x 32 fp32 (2 KB), SW128 (pre-swizzled rows)
  uint64_t* bar = (uint64_t*)(sm + 32768 + 2048);
  uint64_t* mbar = bar + 1;
  uint32_t* tbase = (uint32_t*)(bar + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(mbar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(tbase, 32);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tbase;
  const uint32_t idesc = umma_idesc_tf32(128, NQ);
  for (int c = 0; c < D / DCH; c++) {
    if (threadIdx.x == 0) {
      mbar_arrive_expect_tx(bar, 32768 + 2048);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
              smem_u32(X)),
          "l"((uint64_t)&xmap), "r"(smem_u32(bar)), "r"(c * DCH), "r"(0)
          : "memory");
    }
    __syncwarp();
    if (warp == 0 && lane < NQ)
      bulk_g2s(Qs + lane * DCH, qsw + ((size_t)(lane & 7) * NQ + lane) * D + c * DCH, DCH * 4, bar);
    mbar_wait(bar, c & 1);
    if (threadIdx.x == 0) {
      tc_fence_after();
      for (int h = 0; h < 2; h++)
        for (int k = 0; k < DCH / 8; k++) {
          uint64_t ad = umma_desc_sw128(smem_u32(X) + h * 16384 + k * 32);
          uint64_t bd = umma_desc_sw128(smem_u32(Qs) + k * 32);
          umma_tf32(tmem + h * NQ, ad, bd, idesc, (c > 0 || k > 0) ? 1u : 0u);
        }
      umma_commit(mbar);
    }
    mbar_wait(mbar, c & 1);  // MMAs done before the next TMA overwrites the tile
  }
  tc_fence_after();
  {
    const int h = warp >> 2, g = warp & 3;
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(32 * g) << 16) + h * NQ, v);
    const int row = 128 * h + 32 * g + lane;
    for (int a = 0; a < NQ; a++) out[row * NQ + a] = v[a];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 32);
}

static float trunc_bits_up(float x) {  // mantissa low 13 bits all ones: worst TF32 truncation
  uint32_t b;
  memcpy(&b, &x, 4);
  b |= 0x1FFFu;
  memcpy(&x, &b, 4);
  return x;
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &qr);
  float *dX, *dQ, *dO;
  cudaMalloc(&dX, ROWS * D * 4);
  cudaMalloc(&dQ, 8 * NQ * D * 4);
  cudaMalloc(&dO, ROWS * NQ * 4);
  CUtensorMap m;
  cuuint64_t gd[2] = {D, ROWS};
  cuuint64_t gs[1] = {D * 4};
  cuuint32_t bx[2] = {DCH, ROWS};
  cuuint32_t es[2] = {1, 1};
  enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dX, gd, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = 32768 + 2048 + 64 + 1024;
  cudaFuncSetAttribute(check_k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  srand(7);
  auto rn = []() {
    double u1 = (rand() + 1.0) / (RAND_MAX + 2.0), u2 = (rand() + 1.0) / (RAND_MAX + 2.0);
    return (float)(sqrt(-2 * log(u1)) * cos(6.283185307 * u2));
  };
  const char* names[5] = {"normal", "unit-sphere", "wide exponents", "worst truncation", "offset 100"};
  double worst_all = 0.0;
  int bad_layout = 0;
  for (int kind = 0; kind < 5; kind++) {
    std::vector<float> X(ROWS * D), Q(NQ * D);
    for (auto& v : X) v = rn();
    for (auto& v : Q) v = rn();
    if (kind == 1 || kind == 4) {
      for (int r = 0; r < ROWS; r++) {
        double n = 0;
        for (int j = 0; j < D; j++) n += (double)X[r * D + j] * X[r * D + j];
        for (int j = 0; j < D; j++) X[r * D + j] = (float)(X[r * D + j] / sqrt(n)) + (kind == 4 ? 100.f : 0.f);
      }
      for (int a = 0; a < NQ; a++) {
        double n = 0;
        for (int j = 0; j < D; j++) n += (double)Q[a * D + j] * Q[a * D + j];
        for (int j = 0; j < D; j++) Q[a * D + j] = (float)(Q[a * D + j] / sqrt(n)) + (kind == 4 ? 100.f : 0.f);
      }
    }
    if (kind == 2) {
      for (auto& v : X) v *= expf(8.f * rn());
      for (auto& v : Q) v *= expf(8.f * rn());
    }
    if (kind == 3) {
      for (auto& v : X) v = trunc_bits_up(fabsf(v) + 1.f);
      for (auto& v : Q) v = trunc_bits_up(fabsf(v) + 1.f);
    }
    // 8 pre-swizzled copies: copy p permutes the 16-byte pieces of every 128-byte chunk by ^p
    std::vector<float> Qsw(8 * NQ * D);
    for (int p = 0; p < 8; p++)
      for (int a = 0; a < NQ; a++)
        for (int c = 0; c < D / DCH; c++)
          for (int piece = 0; piece < 8; piece++)
            for (int e = 0; e < 4; e++)
              Qsw[((size_t)p * NQ + a) * D + c * DCH + (piece ^ p) * 4 + e] = Q[a * D + c * DCH + piece * 4 + e];
    cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dQ, Qsw.data(), Qsw.size() * 4, cudaMemcpyHostToDevice);
    check_k<<<1, 256, smem>>>(m, dQ, dO);
    std::vector<float> O(ROWS * NQ);
    cudaError_t e = cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
      printf("CUDA error: %s\n", cudaGetErrorString(e));
      return 1;
    }
    double worst = 0.0;
    for (int r = 0; r < ROWS; r++)
      for (int a = 0; a < NQ; a++) {
        double ex = 0, ab = 0;
        for (int j = 0; j < D; j++) {
          ex += (double)X[r * D + j] * Q[a * D + j];
          ab += fabs((double)X[r * D + j] * Q[a * D + j]);
        }
        double rel = fabs(O[r * NQ + a] - ex) / (ab > 0 ? ab : 1);
        if (rel > 0.05) bad_layout++;
        if (rel > worst) worst = rel;
      }
    printf("%-18s max |D - exact| / sum|x q| = %.3e\n", names[kind], worst);
    if (worst > worst_all) worst_all = worst;
  }
  const double coef = 2.0011 / 1024.0 + D / 2097152.0;
  printf("screen bound coefficient %.3e ; worst observed %.3e (%.1f%% of bound) ; layout errors %d\n",
         coef, worst_all, 100.0 * worst_all / coef, bad_layout);
  printf("%s\n", (bad_layout == 0 && worst_all < coef) ? "PASS" : "FAIL");
  return 0;
}
