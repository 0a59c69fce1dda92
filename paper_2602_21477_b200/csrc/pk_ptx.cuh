// pk_ptx.cuh -- thin inline-PTX wrappers for sm_100a: mbarrier, TMA (tensor +
// bulk), named barriers, exact (never-contracted) fp32 arithmetic, and the
// orderable-key encoding used by every top-k in the library.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace pk {

// ---------------------------------------------------------------- arithmetic
// The reference kernels (ref/kernels.py:73-113, numba, no fastmath) round every
// fp32 op separately.  __f*_rn intrinsics are never contracted into FFMA by
// ptxas; plain '*' '+' could be.  (ptxas DOES contract mul.rn.f32x2 +
// add.rn.f32x2 into FFMA2 -- verified with nvcc 12.9 -- so packed forms are not
// used for the multiply.)
__device__ __forceinline__ float sq_step(float acc, float x, float q) {
  float t = __fsub_rn(x, q);
  return __fadd_rn(acc, __fmul_rn(t, t));
}
__device__ __forceinline__ float ip_step(float acc, float x, float q) {
  return __fadd_rn(acc, __fmul_rn(x, q));
}

// (dist, id) order of np.lexsort((ids, dists)) (ref/engine.py:411): a monotone
// u32 key for the float (with -0.0 == +0.0, NaN last) and the int64 id as the
// secondary key.
__host__ __device__ __forceinline__ uint32_t f2key_bits(uint32_t b) {
  if (b == 0x80000000u) b = 0u;  // -0.0 compares equal to +0.0
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ uint32_t f2key(float f) { return f2key_bits(__float_as_uint(f)); }
__host__ __device__ __forceinline__ uint32_t key2bits(uint32_t k) {
  return (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
}
__device__ __forceinline__ float key2f(uint32_t k) { return __uint_as_float(key2bits(k)); }
// A distance back from its key.  Keys fold -0.0 into +0.0 (they order equal);
// the reference's zero distances have a fixed sign per metric -- neg_ip
// returns -acc and acc is never -0.0 (it starts at +0 and RN sums that cancel
// give +0), so an inner-product zero is -0.0; sq_l2 and cosine zeros are +0.0
__device__ __forceinline__ float key2dist(uint32_t k, int metric) {
  const float v = key2f(k);
  return (metric == 1 && v == 0.f) ? __uint_as_float(0x80000000u) : v;
}
__host__ __device__ __forceinline__ bool lex_less(uint32_t ka, int64_t ia, uint32_t kb, int64_t ib) {
  return ka < kb || (ka == kb && ia < ib);
}
constexpr uint32_t KEY_NONE = 0xffffffffu;
constexpr int64_t ID_NONE = 0x7fffffffffffffffLL;

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ---------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
// 2-D tiled tensor load (coordinates: c0 = innermost element index, c1 = row).
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0,
                                            int c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
// 2-D gather of four rows (arbitrary row coordinates r0..r3) of a tensor map
// whose box is {width, 1}: the rows land back to back in shared memory with
// the map's swizzle applied by destination address.
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int r0,
                                            int r1, int r2, int r3, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2], %8;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
      "l"(policy)
      : "memory");
}
// 1-D bulk copy global -> shared (size multiple of 16, both 16B aligned).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------- cp.async
// 16-byte asynchronous global -> shared copies (LDGSTS): many small requests
// in flight per thread without the per-operation cost of a TMA bulk copy.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------- PDL
// Programmatic dependent launch: a kernel launched with programmatic stream
// serialization may start (prologue: barriers, TMEM, tensor-map prefetch)
// while its predecessor finishes; pdl_wait() blocks until the predecessor
// grid has completed and its writes are visible.  pdl_trigger() lets the
// next kernel start launching.  Both are no-ops without the launch attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---------------------------------------------------------------- sync
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace pk
