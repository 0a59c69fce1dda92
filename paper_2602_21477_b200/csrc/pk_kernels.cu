// pk_kernels.cu -- sm_100a kernels of the IVF search hot path.
//
// Reference arithmetic: every distance below reproduces the
// reference numba kernels bit for bit -- ref/kernels.py:73-83 (sq_l2),
// :86-95 (neg_ip), :98-113 (cosine), :116-135 (kmeans_assign) -- fp32, j
// ascending, each op rounded, no FMA.  Rows are zero-padded to dp (a multiple
// of 32 floats); the padded terms add exactly +0 at the END of the sum, which
// leaves every result unchanged.
//
// Ordering everywhere is np.lexsort((ids, dists)) (ref/engine.py:411) and the
// coarse emit order (d, cid) (ref/graph.py:395): a monotone u32 key of the
// float, then the int64 id.
#include "pk_kernels.h"
#include "pk_ptx.cuh"
#include "pk_umma.cuh"

#include <algorithm>
#include <vector>
#include <cmath>
#include <cstdio>

namespace pk {

constexpr unsigned FULL = 0xffffffffu;

// Launch with programmatic stream serialization (PDL): the kernel may begin
// while the previous kernel on the stream drains; it calls pdl_wait() before
// touching that kernel's outputs.
template <typename... KArgs, typename... Args>
static void launch_maybe_pdl(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                             cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args... args) {
  launch_maybe_pdl(true, kernel, grid, block, smem, st, args...);
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) only when a launch needs
// more than this kernel was last granted on this device (a host-side driver
// call per launch otherwise)
#define PK_SMEM_ATTR(kfn, smem)                                                              \
  do {                                                                                      \
    static int cur_[64] = {0};                                                              \
    int dev_ = 0;                                                                           \
    cudaGetDevice(&dev_);                                                                   \
    if (dev_ < 0 || dev_ >= 64 || (int)(smem) > cur_[dev_]) {                                \
      cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(smem));   \
      if (dev_ >= 0 && dev_ < 64) cur_[dev_] = (int)(smem);                                  \
    }                                                                                       \
  } while (0)

template <int METRIC>
__device__ __forceinline__ float finalize(float acc, float nn, float qn) {
  if (METRIC == SQ_L2) return acc;
  if (METRIC == IP) return -acc;
  // cosine_nb: 1 - dot / (sqrt(nn) * qn), all fp32 (ref/kernels.py:112)
  return __fsub_rn(1.0f, __fdiv_rn(acc, __fmul_rn(__fsqrt_rn(nn), qn)));
}

template <int METRIC>
__device__ __forceinline__ float step4(float acc, float4 x, float4 q) {
  if (METRIC == SQ_L2) {
    acc = sq_step(acc, x.x, q.x);
    acc = sq_step(acc, x.y, q.y);
    acc = sq_step(acc, x.z, q.z);
    acc = sq_step(acc, x.w, q.w);
  } else {
    acc = ip_step(acc, x.x, q.x);
    acc = ip_step(acc, x.y, q.y);
    acc = ip_step(acc, x.z, q.z);
    acc = ip_step(acc, x.w, q.w);
  }
  return acc;
}

// =====================================================================
// Dense distance matrix  D[b][r] = dist(Q[b], X[r])   (batch_distances,
// ref/core.py:98-109).  Used by the coarse quantizer over the centroid table,
// by assign_nearest and by the kernel-table entry points.
// =====================================================================
// The block's 128 rows stream through shared memory in column blocks of DC
// floats (coalesced 16-byte cp.async pieces, DD_RING-deep ring), so every
// row chain runs from shared memory instead of one dependent global load per
// float4 -- the latency that dominates small calls (cache pools, L1
// centroids, a few hundred rows).
constexpr int DD_RING = 3;
constexpr int DD_RS = DC + 4;  // padded row stride in the ring (conflict-free float4 reads)
// Optional fused argmin (assign_nearest, ref/clusters.py:268-279): instead
// of writing D, every block reduces its rows' (dist, cid) keys per query, and
// the last block to finish reduces the blocks' minima and writes (cid, dist)
// -- one launch for the whole assignment (the insert path's batch of 8).
struct DenseArgmin {
  const int64_t* cid = nullptr;   // [n] row -> cid (< 2^32), -1 = free
  const int32_t* scope = nullptr;  // [n] row -> scope code
  int32_t scope_code = 0;
  unsigned long long* part = nullptr;  // [blocks][B] block minima (null: off)
  unsigned* counter = nullptr;    // finished blocks (reset by the last one)
  int64_t* out_cid = nullptr;
  float* out_d = nullptr;
};
template <int METRIC, int NQ>
__global__ void __launch_bounds__(128) dist_dense_kernel(const float* __restrict__ Q, int64_t ldq,
                                                         int B, const float* __restrict__ X,
                                                         int64_t ldx, int64_t n, int dp,
                                                         const float* __restrict__ qnorm,
                                                         float* __restrict__ D, int64_t ldd, int rpb,
                                                         DenseArgmin am) {
  extern __shared__ float4 qs4[];  // [NQ][dp/4] | ring [DD_RING][128][DD_RS]
  const float* qs = reinterpret_cast<const float*>(qs4);
  float* ring = reinterpret_cast<float*>(qs4) + (size_t)NQ * dp;
  const int b0 = blockIdx.y * NQ;
  const int nq = min(NQ, B - b0);
  const int dp4 = dp / 4;
  for (int i = threadIdx.x; i < NQ * dp4; i += blockDim.x) {
    int a = i / dp4, j4 = i - a * dp4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (a < nq) v = *reinterpret_cast<const float4*>(Q + (int64_t)(b0 + a) * ldq + 4 * j4);
    qs4[i] = v;
  }
  __syncthreads();
  // rpb rows per block (128, or fewer when a small call would leave most SMs
  // idle: wider column blocks, fewer ring round trips per block)
  const int64_t r0 = (int64_t)blockIdx.x * rpb;
  const int nr = (int)(n - r0 < rpb ? n - r0 : rpb);
  const int64_t r = r0 + threadIdx.x;
  const bool valid = (int)threadIdx.x < nr;
  // column block width: DC for a full block of rows, wider (fewer ring
  // round trips) when the block holds few rows; a ring slot is 128 * DD_RS floats
  int W = (128 * DD_RS / nr - 4) / DC * DC;
  W = W < DC ? DC : (W > dp ? dp : W);
  const int rs = W + 4;
  const int nblk = (dp + W - 1) / W;
  // block blk: rows [r0, r0 + nr) x columns [blk*W, +w)
  auto issue = [&](int blk) {
    if (blk < nblk) {
      float* dst = ring + (size_t)(blk % DD_RING) * 128 * DD_RS;
      const int w4 = min(W, dp - blk * W) / 4;
      for (int i = threadIdx.x; i < nr * w4; i += 128) {
        const int rr = i / w4, c = i - rr * w4;
        cp_async16(dst + rr * rs + 4 * c, X + (r0 + rr) * ldx + blk * W + 4 * c);
      }
    }
    cp_async_commit();  // empty groups keep the wait count uniform
  };
#pragma unroll
  for (int i = 0; i < DD_RING - 1; i++) issue(i);
  float acc[NQ];
#pragma unroll
  for (int a = 0; a < NQ; a++) acc[a] = 0.f;
  float nn = 0.f;
  for (int blk = 0; blk < nblk; blk++) {
    issue(blk + DD_RING - 1);
    cp_async_wait<DD_RING - 1>();
    __syncthreads();
    const float* xr = ring + (size_t)(blk % DD_RING) * 128 * DD_RS + (threadIdx.x < nr ? threadIdx.x : 0) * rs;
    const int w = min(W, dp - blk * W);
#pragma unroll 8
    for (int j = 0; j < w; j += 4) {
      const float4 x = *reinterpret_cast<const float4*>(xr + j);
#pragma unroll
      for (int a = 0; a < NQ; a++) {
        float4 q = *reinterpret_cast<const float4*>(qs + a * dp + blk * W + j);
        acc[a] = step4<METRIC>(acc[a], x, q);
      }
      if (METRIC == COSINE) nn = step4<IP>(nn, x, x);
    }
    __syncthreads();  // slot blk % DD_RING is refilled by the next iteration's issue
  }
  if (am.part == nullptr) {
    if (!valid) return;
#pragma unroll
    for (int a = 0; a < NQ; a++) {
      if (a < nq) {
        float qn = (METRIC == COSINE) ? qnorm[b0 + a] : 0.f;
        D[(int64_t)(b0 + a) * ldd + r] = finalize<METRIC>(acc[a], nn, qn);
      }
    }
    return;
  }
  // fused argmin by (dist, cid) over the in-scope rows
  __shared__ unsigned long long s_m[4][NQ];
  __shared__ unsigned s_ticket;
  const bool in = valid && am.cid[r] >= 0 && am.scope[r] == am.scope_code;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int a = 0; a < NQ; a++) {
    unsigned long long k = ~0ull;
    if (in && a < nq) {
      const float qn = (METRIC == COSINE) ? qnorm[b0 + a] : 0.f;
      k = ((unsigned long long)f2key(finalize<METRIC>(acc[a], nn, qn)) << 32) | (unsigned)am.cid[r];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long k2 = __shfl_xor_sync(0xffffffffu, k, o);
      k = k2 < k ? k2 : k;
    }
    if (lane == 0) s_m[warp][a] = k;
  }
  __syncthreads();
  const int nblk_all = gridDim.x * gridDim.y;
  const int blk = blockIdx.y * gridDim.x + blockIdx.x;
  if (threadIdx.x < NQ) {
    unsigned long long k = s_m[0][threadIdx.x];
    for (int w = 1; w < 4; w++) k = s_m[w][threadIdx.x] < k ? s_m[w][threadIdx.x] : k;
    am.part[(int64_t)blk * NQ + threadIdx.x] = k;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_ticket = atomicAdd(am.counter, 1u);
  __syncthreads();
  if (s_ticket != (unsigned)(nblk_all - 1)) return;
  __threadfence();
  // the last block: per query, the minimum over the row blocks of its group
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    const int gy = b / NQ, a = b - gy * NQ;
    unsigned long long k = ~0ull;
    for (int bx = 0; bx < (int)gridDim.x; bx++) {
      const unsigned long long v = *(volatile unsigned long long*)&am.part[(int64_t)(gy * gridDim.x + bx) * NQ + a];
      k = v < k ? v : k;
    }
    am.out_cid[b] = k == ~0ull ? -1 : (int64_t)(unsigned)(k & 0xffffffffull);
    if (am.out_d) am.out_d[b] = key2dist((uint32_t)(k >> 32), METRIC);
  }
  if (threadIdx.x == 0) *am.counter = 0;
}

template <int METRIC>
static void dist_dense_dispatch(const float* Q, int64_t ldq, int B, const float* X, int64_t ldx,
                                int64_t n, int dp, const float* qnorm, float* D, int64_t ldd,
                                cudaStream_t st, DenseArgmin am = DenseArgmin()) {
  if (B <= 0 || n <= 0) return;
  int nq = B >= 16 ? 16 : (B >= 8 ? 8 : (B >= 4 ? 4 : (B >= 2 ? 2 : 1)));
  while (nq > 1 && (size_t)nq * dp * 4 > 96 * 1024) nq >>= 1;
  // small calls (an insert batch's assignment): fewer queries per block until
  // the grid covers the GPU twice -- each thread's chains are sequential, so
  // a block with 8 queries takes 8x as long as one with 1
  while (nq > 1 && B <= 16 && ((n + 31) / 32) * ((B + nq - 1) / nq) < 296) nq >>= 1;
  size_t smem = (size_t)nq * dp * 4 + (size_t)DD_RING * 128 * DD_RS * 4;
  const int64_t ny = (B + nq - 1) / nq;
  int rpb = 128;
  while (rpb > 32 && ((n + rpb - 1) / rpb) * ny < 148) rpb >>= 1;
  dim3 grid((unsigned)((n + rpb - 1) / rpb), (unsigned)ny);
#define PK_DD(NQV)                                                                                  \
  case NQV: {                                                                                       \
    auto k = dist_dense_kernel<METRIC, NQV>;                                                        \
    PK_SMEM_ATTR(k, (int)smem);                \
    k<<<grid, 128, smem, st>>>(Q, ldq, B, X, ldx, n, dp, qnorm, D, ldd, rpb, am);                   \
  } break;
  switch (nq) {
    PK_DD(1) PK_DD(2) PK_DD(4) PK_DD(8) PK_DD(16)
  }
#undef PK_DD
}

void launch_dist_dense(int metric, const float* Q, int64_t ldq, int B, const float* X, int64_t ldx,
                       int64_t n, int dp, const float* qnorm, float* D, int64_t ldd,
                       cudaStream_t st) {
  if (metric == SQ_L2) dist_dense_dispatch<SQ_L2>(Q, ldq, B, X, ldx, n, dp, qnorm, D, ldd, st);
  else if (metric == IP) dist_dense_dispatch<IP>(Q, ldq, B, X, ldx, n, dp, qnorm, D, ldd, st);
  else dist_dense_dispatch<COSINE>(Q, ldq, B, X, ldx, n, dp, qnorm, D, ldd, st);
}

int dense_argmin_blocks(int64_t n, int B) {
  // partial entries: blocks (<= ceil(n / 32) row blocks x ceil(B / nq) query
  // groups) x nq entries each <= ceil(n / 32) x (B + 16)
  return (int)(((n + 31) / 32) * (B + 16));
}

void launch_dense_argmin(int metric, const float* Q, int64_t ldq, int B, const float* C, int64_t n, int dp,
                         const float* qnorm, ListTable lt, int32_t scope_code, unsigned long long* part,
                         unsigned* counter, int64_t* out_cid, float* out_d, cudaStream_t st) {
  DenseArgmin am;
  am.cid = lt.cid;
  am.scope = lt.scope;
  am.scope_code = scope_code;
  am.part = part;
  am.counter = counter;
  am.out_cid = out_cid;
  am.out_d = out_d;
  if (metric == SQ_L2) dist_dense_dispatch<SQ_L2>(Q, ldq, B, C, dp, n, dp, qnorm, nullptr, 0, st, am);
  else if (metric == IP) dist_dense_dispatch<IP>(Q, ldq, B, C, dp, n, dp, qnorm, nullptr, 0, st, am);
  else dist_dense_dispatch<COSINE>(Q, ldq, B, C, dp, n, dp, qnorm, nullptr, 0, st, am);
}

// =====================================================================
// kmeans_assign (ref/kernels.py:116-135): t = x - c in fp32, t*t in fp32,
// sum in fp64 ascending j, strict '<' (first centroid wins ties).
// One thread per point; centroids stream through shared memory in groups.
// =====================================================================
constexpr int KM_G = 8;
__global__ void __launch_bounds__(128) kmeans_assign_kernel(const float* __restrict__ X, int64_t ldx,
                                                            int64_t n, const float* __restrict__ C,
                                                            int64_t ldc, int64_t k, int dp,
                                                            int64_t* __restrict__ labels,
                                                            double* __restrict__ dists) {
  extern __shared__ float4 cs4[];  // [KM_G][dp/4]
  const float* cs = reinterpret_cast<const float*>(cs4);
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = r < n;
  const float* xr = X + (valid ? r : 0) * ldx;
  const int dp4 = dp / 4;
  double best = 1e300;
  int64_t arg = 0;
  for (int64_t c0 = 0; c0 < k; c0 += KM_G) {
    const int g = (int)(k - c0 < KM_G ? k - c0 : KM_G);
    __syncthreads();
    for (int i = threadIdx.x; i < KM_G * dp4; i += blockDim.x) {
      int a = i / dp4, j4 = i - a * dp4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (a < g) v = *reinterpret_cast<const float4*>(C + (c0 + a) * ldc + 4 * j4);
      cs4[i] = v;
    }
    __syncthreads();
    double acc[KM_G];
#pragma unroll
    for (int a = 0; a < KM_G; a++) acc[a] = 0.0;
    for (int j = 0; j < dp; j += 4) {
      float4 x = __ldg(reinterpret_cast<const float4*>(xr + j));
#pragma unroll
      for (int a = 0; a < KM_G; a++) {
        float4 c = *reinterpret_cast<const float4*>(cs + a * dp + j);
        float t;
        t = __fsub_rn(x.x, c.x); acc[a] = __dadd_rn(acc[a], (double)__fmul_rn(t, t));
        t = __fsub_rn(x.y, c.y); acc[a] = __dadd_rn(acc[a], (double)__fmul_rn(t, t));
        t = __fsub_rn(x.z, c.z); acc[a] = __dadd_rn(acc[a], (double)__fmul_rn(t, t));
        t = __fsub_rn(x.w, c.w); acc[a] = __dadd_rn(acc[a], (double)__fmul_rn(t, t));
      }
    }
#pragma unroll
    for (int a = 0; a < KM_G; a++) {
      if (a < g && acc[a] < best) {
        best = acc[a];
        arg = c0 + a;
      }
    }
  }
  if (valid) {
    labels[r] = arg;
    dists[r] = best;
  }
}

void launch_kmeans_assign(const float* X, int64_t ldx, int64_t n, const float* C, int64_t ldc,
                          int64_t k, int dp, int64_t* labels, double* dists, cudaStream_t st) {
  if (n <= 0) return;
  size_t smem = (size_t)KM_G * dp * 4;
  PK_SMEM_ATTR(kmeans_assign_kernel, (int)smem);
  kmeans_assign_kernel<<<(unsigned)((n + 127) / 128), 128, smem, st>>>(X, ldx, n, C, ldc, k, dp,
                                                                      labels, dists);
}

// qn = sqrt(sum_j q_j * q_j) in fp32, j ascending (ref/kernels.py:101-104).
__global__ void qnorm_kernel(const float* __restrict__ Q, int64_t ldq, int B, int d,
                             float* __restrict__ qnorm) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const float* q = Q + (int64_t)b * ldq;
  float acc = 0.f;
  for (int j = 0; j < d; j++) acc = ip_step(acc, q[j], q[j]);
  qnorm[b] = __fsqrt_rn(acc);
}
void launch_qnorm(const float* Q, int64_t ldq, int B, int d, float* qnorm, cudaStream_t st) {
  if (B <= 0) return;
  qnorm_kernel<<<(B + 127) / 128, 128, 0, st>>>(Q, ldq, B, d, qnorm);
}

// centroid (ref/core.py:112-117): column sums in fp64 in row order, / n, -> f32.
__global__ void centroid_kernel(const float* __restrict__ rows, int64_t ldr, int64_t n, int dp,
                                float* __restrict__ out) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= dp) return;
  double s = 0.0;
  for (int64_t i = 0; i < n; i++) s = __dadd_rn(s, (double)rows[i * ldr + j]);
  out[j] = (float)__ddiv_rn(s, (double)n);
}
void launch_centroid(const float* rows, int64_t ldr, int64_t n, int dp, float* cent_out,
                     cudaStream_t st) {
  if (n <= 0) return;
  centroid_kernel<<<(dp + 127) / 128, 128, 0, st>>>(rows, ldr, n, dp, cent_out);
}

// Segmented centroids for k-means (kmeans_split_points, ref/clusters.py:166-
// 171): rows grouped by label in their original order, segment c = rows
// [off[c], off[c+1]); out[c] = fp64 row-order column mean -> f32 (the
// core.centroid arithmetic), one thread per (segment, column).
__global__ void seg_centroid_kernel(const float* __restrict__ rows, int64_t ldr,
                                    const int64_t* __restrict__ off, int k, int d,
                                    float* __restrict__ out) {
  const int c = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= k || j >= d) return;
  const int64_t a = off[c], b = off[c + 1];
  if (b <= a) return;  // empty cluster: caller fills it
  double s = 0.0;
  for (int64_t i = a; i < b; i++) s = __dadd_rn(s, (double)rows[i * ldr + j]);
  out[(int64_t)c * d + j] = (float)__ddiv_rn(s, (double)(b - a));
}
void launch_seg_centroid(const float* rows, int64_t ldr, const int64_t* off, int k, int d, float* out,
                         cudaStream_t st) {
  if (k <= 0 || d <= 0) return;
  seg_centroid_kernel<<<dim3((d + 127) / 128, k), 128, 0, st>>>(rows, ldr, off, k, d, out);
}

// =====================================================================
// CTA-level sort / select over (key u32, id i64, payload i32) entries.
// =====================================================================
struct Entry {
  uint32_t key;
  int32_t pay;
  int64_t id;
};
__device__ __forceinline__ bool e_less(const Entry& a, const Entry& b) {
  return lex_less(a.key, a.id, b.key, b.id);
}
__device__ __forceinline__ Entry e_none() {
  Entry e;
  e.key = KEY_NONE;
  e.pay = -1;
  e.id = ID_NONE;
  return e;
}

// Sort buf[0..n) ascending; pads to a power of two with sentinels (cap >= pow2(n)).
__device__ void cta_bitonic_sort(Entry* buf, int n) {
  int N = 1;
  while (N < n) N <<= 1;
  for (int i = n + threadIdx.x; i < N; i += blockDim.x) buf[i] = e_none();
  __syncthreads();
  for (int k = 2; k <= N; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < N; i += blockDim.x) {
        int ixj = i ^ j;
        if (ixj > i) {
          Entry a = buf[i], b = buf[ixj];
          bool up = (i & k) == 0;
          if (e_less(b, a) == up) {
            buf[i] = b;
            buf[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
}

// Keep the first `kk` entries of a sorted buffer, optionally dropping
// duplicate (key, id) entries (first occurrence per id, ref/engine.py:414-418).
// Returns the kept count (thread 0 compacts; result broadcast).
__device__ int cta_compact_sorted(Entry* buf, int n, int kk, bool dedup, int* s_cnt) {
  __syncthreads();
  if (threadIdx.x == 0) {
    int w = 0;
    for (int i = 0; i < n && w < kk; i++) {
      if (dedup && w > 0 && buf[i].id == buf[w - 1].id && buf[i].key == buf[w - 1].key) continue;
      buf[w++] = buf[i];
    }
    *s_cnt = w;
  }
  __syncthreads();
  return *s_cnt;
}

// Block-wide: thread t holds cnt (bin t of a 256-bin histogram); returns the
// bin holding the rem-th smallest element and the count below it.
__device__ __forceinline__ void pick_bin(unsigned cnt, int rem, int* s_bin, int* s_below, unsigned* s_w) {
  // (blockDim.x == 256)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned x = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[warp] = x;
  __syncthreads();
  unsigned pre = 0;
  for (int w = 0; w < warp; w++) pre += s_w[w];
  const unsigned incl = pre + x, excl = incl - cnt;
  if (excl < (unsigned)rem && incl >= (unsigned)rem) {
    *s_bin = threadIdx.x;
    *s_below = (int)excl;
  }
  __syncthreads();
}

// Rank sort for n <= blockDim.x: thread i counts the entries ordered before
// its own (ties by position: stable) and stores it at that rank -- n
// independent shared-memory sweeps instead of log^2 dependent exchange
// stages (measured ~10K cycles for the 64-entry warp bitonic).  With dedup
// an entry equal (key, id) to an earlier one is dropped and ranks count the
// first occurrences only (what cta_compact_sorted keeps).
__device__ int block_rank_keep(Entry* buf, int n, int kk, bool dedup) {
  __shared__ uint8_t s_dupf[1024];
  const int t = threadIdx.x;
  const bool act = t < n;
  __syncthreads();
  Entry e = act ? buf[t] : e_none();
  bool dup = false;
  if (dedup) {
    if (act)
      for (int j = 0; j < t; j++) {
        const Entry o = buf[j];
        dup |= (o.key == e.key) & (o.id == e.id);
      }
    s_dupf[t] = dup;
    __syncthreads();
  }
  int rank = 0;
  if (act && !dup)
    for (int j = 0; j < n; j++) {
      const Entry o = buf[j];
      const bool eq = (o.key == e.key) & (o.id == e.id);
      rank += dedup ? (e_less(o, e) & !s_dupf[j]) : (e_less(o, e) | (eq & (j < t)));
    }
  const int total = __syncthreads_count(act && !dup);  // also: every read of buf is done
  if (act && !dup && rank < kk) buf[rank] = e;
  __syncthreads();
  return total < kk ? total : kk;
}

__device__ int block_sort_keep(Entry* buf, int n, int kk, bool dedup, int* s_cnt) {
  if (n <= (int)blockDim.x && n <= 1024) return block_rank_keep(buf, n, kk, dedup);
  cta_bitonic_sort(buf, n);
  return cta_compact_sorted(buf, n, kk, dedup, s_cnt);
}

constexpr int SEL_CAP = 4096;

// Coarse quantizer select: per query the first nprobe in-scope lists by
// (dist, cid) -- HybridGraphIndex.search emit order at exhaustive ef
// (ref/graph.py:392-396).  Lists with no members still count
// (the reference graph keeps emptied clusters).
__global__ void __launch_bounds__(256) coarse_select_kernel(const float* __restrict__ Dc,
                                                            int64_t ldd, ListTable lt,
                                                            const int32_t* __restrict__ scope_codes,
                                                            int nscopes, int nprobe,
                                                            int32_t* __restrict__ probe,
                                                            uint32_t* __restrict__ probe_key) {
  extern __shared__ Entry sel_buf[];  // [SEL_CAP]
  __shared__ int s_cnt;
  __shared__ int s_codes[64];
  const int b = blockIdx.x;
  if (threadIdx.x < 64) s_codes[threadIdx.x] = threadIdx.x < nscopes ? scope_codes[threadIdx.x] : -1;
  __syncthreads();
  const float* drow = Dc + (int64_t)b * ldd;
  int kept = 0;
  Entry tau = e_none();
  for (int base = 0; base < lt.nslots; base += SEL_CAP - nprobe) {
    const int end = min(lt.nslots, base + SEL_CAP - nprobe);
    if (threadIdx.x == 0) s_cnt = kept;
    __syncthreads();
    for (int s = base + threadIdx.x; s < end; s += blockDim.x) {
      if (lt.cid[s] < 0) continue;
      int sc = lt.scope[s];
      bool in = false;
      for (int i = 0; i < nscopes; i++) in |= (s_codes[i] == sc);
      if (!in) continue;
      Entry e;
      e.key = f2key(drow[s]);
      e.id = lt.cid[s];
      e.pay = s;
      if (kept == nprobe && !e_less(e, tau)) continue;
      int pos = atomicAdd(&s_cnt, 1);
      sel_buf[pos] = e;
    }
    __syncthreads();
    int n = s_cnt;
    if (n > kept) {
      cta_bitonic_sort(sel_buf, n);
      kept = cta_compact_sorted(sel_buf, n, nprobe, false, &s_cnt);
      if (kept == nprobe) tau = sel_buf[nprobe - 1];
    }
    __syncthreads();
  }
  for (int p = threadIdx.x; p < nprobe; p += blockDim.x) {
    probe[(int64_t)b * nprobe + p] = p < kept ? sel_buf[p].pay : -1;
    if (probe_key) probe_key[(int64_t)b * nprobe + p] = p < kept ? sel_buf[p].key : KEY_NONE;
  }
}

void launch_coarse_select(const float* Dc, int64_t ldd, int B, ListTable lt,
                          const int32_t* scope_codes, int nscopes, int nprobe, int32_t* probe,
                          uint32_t* probe_key, cudaStream_t st) {
  if (B <= 0) return;
  size_t smem = SEL_CAP * sizeof(Entry);
  PK_SMEM_ATTR(coarse_select_kernel, (int)smem);
  coarse_select_kernel<<<B, 256, smem, st>>>(Dc, ldd, lt, scope_codes, nscopes, nprobe, probe,
                                             probe_key);
}

// =====================================================================
// Routing: invert (query -> probed lists) into (list -> queries) and cut each
// probed list into row chunks x query groups (the scan work items).
//   route_emit_kernel  one CTA per query: its output slots (one per probed
//                      list chunk, fixed stride smax per query, so no
//                      batch-wide scan is needed), scanned rows, and one
//                      (query, slot base) pair appended to each probed list's
//                      bucket (bcap entries per list).
//   route_items_kernel one thread per list: chunks x ceil(queries / QG)
//                      items, appended through one atomic counter.
// Item and bucket order depend on atomic arrival; results do not (the merge
// orders by (dist, id)).
// =====================================================================
__device__ __forceinline__ int nchunks_of(int64_t len, int chunk) {
  return (int)((len + chunk - 1) / chunk);
}

constexpr int RE_THREADS = 128;
// Routing of one query (the calling CTA, any blockDim multiple of 32): its
// output slots (fixed stride smax), scanned rows, and one (query, slot base)
// pair per probed list appended to that list's bucket.
__device__ void emit_routes(int b, const int32_t* __restrict__ prow, int nprobe, const ListTable& lt,
                            int chunk_rows, int smax, int bcap, int32_t* __restrict__ lcount,
                            QPair* __restrict__ bucket, int32_t* __restrict__ slot_off,
                            int64_t* __restrict__ scanned) {
  __shared__ int s_w[32];
  __shared__ long long s_sc[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int carry = 0;
  int64_t sc = 0;
  for (int p0 = 0; p0 < nprobe; p0 += blockDim.x) {
    const int p = p0 + threadIdx.x;
    const int s = p < nprobe ? prow[p] : -1;
    int64_t len = 0;
    int c = 0;
    if (s >= 0) {
      len = lt.len[s];
      c = nchunks_of(len, chunk_rows);
    }
    sc += len;
    int x = c;  // block exclusive scan of c
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    int wpre = 0, tot = 0;
    for (int w = 0; w < nw; w++) {
      if (w < warp) wpre += s_w[w];
      tot += s_w[w];
    }
    if (s >= 0) {
      const int pos = atomicAdd(&lcount[s], 1);
      QPair qp;
      qp.b = b;
      qp.slotbase = b * smax + carry + wpre + x - c;
      bucket[(int64_t)s * bcap + pos] = qp;
    }
    carry += tot;
    __syncthreads();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sc += __shfl_xor_sync(FULL, sc, o);
  if (lane == 0) s_sc[warp] = (long long)sc;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int w = 0; w < nw; w++) t += s_sc[w];
    scanned[b] = t;
    slot_off[2 * b] = b * smax;
    slot_off[2 * b + 1] = b * smax + carry;
  }
}

__global__ void __launch_bounds__(RE_THREADS) route_emit_kernel(
    const int32_t* __restrict__ probe, int nprobe, ListTable lt, int chunk_rows, int smax, int bcap,
    int32_t* __restrict__ lcount, QPair* __restrict__ bucket, int32_t* __restrict__ slot_off,
    int64_t* __restrict__ scanned) {
  emit_routes(blockIdx.x, probe + (int64_t)blockIdx.x * nprobe, nprobe, lt, chunk_rows, smax, bcap, lcount,
              bucket, slot_off, scanned);
}

// Items of at most chunk_rows / 2 rows (a list's short last chunk) are queued
// after all the others: counters[0] counts the front items, counters[2] the
// tail items, written backwards from tail_base (counters[3]), so the
// persistent scan drains the big items first and its last, ragged round is
// made of short ones (measured CTA end spread 40 us with one queue).
__global__ void route_items_kernel(ListTable lt, int chunk_rows, int bcap,
                                   const int32_t* __restrict__ lcount, ScanItem* __restrict__ items,
                                   int32_t* __restrict__ counters, int tail_base) {
  pdl_trigger();
  pdl_wait();
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s == 0) counters[3] = tail_base;
  if (s >= lt.nslots) return;
  const int cnt = lcount[s];
  if (cnt <= 0) return;
  const int64_t len = lt.len[s];
  const int nch = nchunks_of(len, chunk_rows);
  const int ng = (cnt + QG - 1) / QG;
  if (nch == 0) return;
  const int last_rows = (int)(len - (int64_t)(nch - 1) * chunk_rows);
  const bool short_tail = last_rows <= chunk_rows / 2;
  const int nfront = (short_tail ? nch - 1 : nch) * ng;
  int w = nfront ? atomicAdd(&counters[0], nfront) : 0;
  int wt = short_tail ? atomicAdd(&counters[2], ng) : 0;
  for (int c = 0; c < nch; c++) {
    const bool tail = short_tail && c == nch - 1;
    for (int g = 0; g < ng; g++) {
      ScanItem it;
      it.lslot = s;
      it.row0 = c * chunk_rows;
      it.nrows = (int)(len - (int64_t)c * chunk_rows < chunk_rows ? len - (int64_t)c * chunk_rows : chunk_rows);
      it.qoff = s * bcap + g * QG;
      it.nq = min(QG, cnt - g * QG);
      it.chunk = c;
      it.pad0 = it.pad1 = 0;
      if (tail) items[tail_base - wt++] = it;
      else items[w++] = it;
    }
  }
}

void launch_route(const int32_t* probe, int B, int nprobe, ListTable lt, int chunk_rows, int smax,
                  int bcap, int32_t* lcount, ScanItem* items, int32_t* n_items, QPair* bucket,
                  int32_t* slot_off, int64_t* scanned, bool emitted, int max_items, cudaStream_t st) {
  // lcount [nslots] and *n_items zeroed by the caller; `emitted`: the coarse
  // pick already ran emit_routes for every query
  if (B <= 0) return;
  if (!emitted)
    route_emit_kernel<<<B, RE_THREADS, 0, st>>>(probe, nprobe, lt, chunk_rows, smax, bcap, lcount,
                                                bucket, slot_off, scanned);
  if (lt.nslots > 0)
    launch_pdl(route_items_kernel, dim3((lt.nslots + 255) / 256), dim3(256), 0, st, lt, chunk_rows, bcap,
               lcount, items, n_items, max_items - 1);
}

// =====================================================================
// The fused posting-list scan (ref/tiering.py:294-328 merged_search ->
// ref/core.py:98-109 -> ref/kernels.py:73-113, plus the per-list part of
// _topk ref/engine.py:406-426).
//
// Persistent CTA per SM: warp 8 is the TMA producer, warps 0-7 compute.  A
// work item is (list chunk of <= chunk_rows rows) x (<= QG queries).  Rows
// stream through a STAGES-deep ring of [TILE rows x DC floats] tiles (TMA
// 2-D, SWIZZLE_128B), the item's query chunks ride along as 128-byte bulk
// copies.  Each compute thread owns one row and accumulates all the item's
// queries exactly; at the end of a tile the distances go to shared memory
// and each warp merges two queries' survivors into a sorted per-query
// (key, id) list of kk entries.
// =====================================================================
constexpr int NCW = 8;  // compute warps
constexpr int SCAN_THREADS = (NCW + 1) * 32;

struct ScanLayout {
  static constexpr size_t X_BYTES = (size_t)STAGES * TILE * DC * 4;
  static constexpr size_t QC_BYTES = (size_t)STAGES * QG * DC * 4;
  static constexpr size_t D_BYTES = (size_t)QG * TILE * 4;
  static constexpr size_t LK_BYTES = (size_t)QG * KKMAX * 4;
  static constexpr size_t LI_BYTES = (size_t)QG * KKMAX * 8;
  static constexpr size_t LN_BYTES = 128;
  static constexpr size_t BAR_BYTES = 256;
  static constexpr size_t RING_BYTES = 2 * sizeof(ScanItem);
  static constexpr size_t TOTAL =
      X_BYTES + QC_BYTES + D_BYTES + LK_BYTES + LI_BYTES + LN_BYTES + BAR_BYTES + RING_BYTES;
};
size_t scan_smem_bytes() { return ScanLayout::TOTAL + 1024; }

struct ScanShared {
  float* X;
  float* Qc;
  float* D;      // exact kernel: [QG][TILE] tile distances
  float* A;      // screen kernel: [QG][CHUNK_MAX] screened (then exact) distances
  float* NX;     // screen kernel: [CHUNK_MAX] row norms
  uint16_t* CR;  // screen kernel: [QG][CHUNK_MAX] candidate rows
  int32_t* Cn;   // screen kernel: [QG] candidate counts
  uint32_t* Lkey;
  int64_t* Lid;
  int32_t* Ln;
  uint64_t* full;
  uint64_t* empty;
  uint64_t* rfull;
  uint64_t* rempty;
  ScanItem* ring;
};

// Accumulate one tile (this thread's row vs NQ queries) over all d-chunks,
// consuming stages from the ring; writes distances to D[a][row].
template <int METRIC, int NQ>
__device__ __forceinline__ void scan_tile(const ScanShared& S, int nchunk_d, int& s, uint32_t& ph,
                                          int nq, const float* qn_s) {
  const int row = threadIdx.x;  // 0..TILE-1
  const int lane = threadIdx.x & 31;
  const int swz = row & 7;
  float acc[NQ];
#pragma unroll
  for (int a = 0; a < NQ; a++) acc[a] = 0.f;
  float nn = 0.f;
  for (int c = 0; c < nchunk_d; c++) {
    mbar_wait(&S.full[s], ph);
    const float* xs = S.X + (size_t)s * TILE * DC + row * DC;
    const float* qs = S.Qc + (size_t)s * QG * DC;
#pragma unroll
    for (int k = 0; k < DC / 4; k++) {
      float4 x = *reinterpret_cast<const float4*>(xs + ((k ^ swz) << 2));
#pragma unroll
      for (int a = 0; a < NQ; a++) {
        float4 q = *reinterpret_cast<const float4*>(qs + a * DC + (k << 2));
        acc[a] = step4<METRIC>(acc[a], x, q);
      }
      if (METRIC == COSINE) nn = step4<IP>(nn, x, x);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.empty[s]);
    if (++s == STAGES) {
      s = 0;
      ph ^= 1;
    }
  }
#pragma unroll
  for (int a = 0; a < NQ; a++)
    if (a < nq) S.D[a * TILE + row] = finalize<METRIC>(acc[a], nn, METRIC == COSINE ? qn_s[a] : 0.f);
}

// 19-comparator sorting network for 8 (key, id) pairs held in registers.
__device__ __forceinline__ void ce(uint32_t& ka, int64_t& ia, uint32_t& kb, int64_t& ib) {
  bool sw = lex_less(kb, ib, ka, ia);
  uint32_t tk = sw ? kb : ka;
  int64_t ti = sw ? ib : ia;
  kb = sw ? ka : kb;
  ib = sw ? ia : ib;
  ka = tk;
  ia = ti;
}
__device__ __forceinline__ void sort8(uint32_t* k, int64_t* i) {
#define PK_CE(a, b) ce(k[a], i[a], k[b], i[b])
  PK_CE(0, 2); PK_CE(1, 3); PK_CE(4, 6); PK_CE(5, 7);
  PK_CE(0, 4); PK_CE(1, 5); PK_CE(2, 6); PK_CE(3, 7);
  PK_CE(0, 1); PK_CE(2, 3); PK_CE(4, 5); PK_CE(6, 7);
  PK_CE(2, 4); PK_CE(3, 5);
  PK_CE(1, 4); PK_CE(3, 6);
  PK_CE(1, 2); PK_CE(3, 4); PK_CE(5, 6);
#undef PK_CE
}

// Merge up to 8 lane-local (key, id) candidates per lane (unsorted, KEY_NONE
// padded) into query a's sorted list of at most kk entries (warp-wide).
__device__ __forceinline__ void warp_merge_into_list(const ScanShared& S, int a, int kk, uint32_t* ck, int64_t* ci) {
  const int lane = threadIdx.x & 31;
  const int n_old = S.Ln[a];
  sort8(ck, ci);
  // old list: lane holds entries lane and lane+32
  uint32_t ok0 = KEY_NONE, ok1 = KEY_NONE;
  int64_t oi0 = ID_NONE, oi1 = ID_NONE;
  if (lane < n_old) {
    ok0 = S.Lkey[a * KKMAX + lane];
    oi0 = S.Lid[a * KKMAX + lane];
  }
  if (lane + 32 < n_old) {
    ok1 = S.Lkey[a * KKMAX + lane + 32];
    oi1 = S.Lid[a * KKMAX + lane + 32];
  }
  uint32_t nk0 = KEY_NONE, nk1 = KEY_NONE;
  int64_t ni0 = ID_NONE, ni1 = ID_NONE;
  int p_old = 0, cnt = 0;
  for (; cnt < kk; cnt++) {
    // warp min over lane heads by (key, id)
    const uint32_t m = __reduce_min_sync(FULL, ck[0]);
    const unsigned tie = __ballot_sync(FULL, ck[0] == m);
    int wl;
    int64_t wid;
    if (__popc(tie) == 1) {
      wl = __ffs(tie) - 1;
      wid = __shfl_sync(FULL, ci[0], wl);
    } else {
      const int64_t my = (ck[0] == m) ? ci[0] : ID_NONE;
      const uint32_t hi = (uint32_t)((uint64_t)my >> 32) ^ 0x80000000u;
      const uint32_t mhi = __reduce_min_sync(FULL, hi);
      const uint32_t lo = (hi == mhi) ? (uint32_t)(uint64_t)my : 0xffffffffu;
      const uint32_t mlo = __reduce_min_sync(FULL, lo);
      const unsigned w = __ballot_sync(FULL, ck[0] == m && hi == mhi && lo == mlo);
      wl = __ffs(w) - 1;
      wid = (int64_t)(((uint64_t)(mhi ^ 0x80000000u) << 32) | (uint64_t)mlo);
    }
    // old-list head
    uint32_t hk = KEY_NONE;
    int64_t hid = ID_NONE;
    if (p_old < n_old) {
      const int src = p_old & 31;
      const bool second = p_old >= 32;
      hk = __shfl_sync(FULL, second ? ok1 : ok0, src);
      hid = __shfl_sync(FULL, second ? oi1 : oi0, src);
    }
    uint32_t sk;
    int64_t si;
    if (lex_less(hk, hid, m, wid)) {
      sk = hk;
      si = hid;
      p_old++;
    } else {
      sk = m;
      si = wid;
      if (lane == wl) {
#pragma unroll
        for (int i = 0; i < 7; i++) {
          ck[i] = ck[i + 1];
          ci[i] = ci[i + 1];
        }
        ck[7] = KEY_NONE;
        ci[7] = ID_NONE;
      }
    }
    if (sk == KEY_NONE && si == ID_NONE) break;
    if (lane == (cnt & 31)) {
      if (cnt < 32) {
        nk0 = sk;
        ni0 = si;
      } else {
        nk1 = sk;
        ni1 = si;
      }
    }
  }
  if (lane < cnt) {
    S.Lkey[a * KKMAX + lane] = nk0;
    S.Lid[a * KKMAX + lane] = ni0;
  }
  if (lane + 32 < cnt) {
    S.Lkey[a * KKMAX + lane + 32] = nk1;
    S.Lid[a * KKMAX + lane + 32] = ni1;
  }
  __syncwarp();
  if (lane == 0) S.Ln[a] = cnt;
  __syncwarp();
}

// Merge this tile's survivors for query a into its sorted list (warp-wide).
__device__ void topk_merge_tile(const ScanShared& S, int a, int rows, const int64_t* __restrict__ ids,
                                int64_t idbase, int kk) {
  const int lane = threadIdx.x & 31;
  const float* dq = S.D + a * TILE;
  const int n_old = S.Ln[a];
  uint32_t tk = KEY_NONE;
  int64_t ti = ID_NONE;
  if (n_old == kk) {
    tk = S.Lkey[a * KKMAX + kk - 1];
    ti = S.Lid[a * KKMAX + kk - 1];
  }
  uint32_t ck[8];
  int64_t ci[8];
  bool have = false;
#pragma unroll
  for (int i = 0; i < 8; i++) {
    const int row = lane + 32 * i;
    ck[i] = KEY_NONE;
    ci[i] = ID_NONE;
    if (row < rows) {
      uint32_t k = f2key(dq[row]);
      if (k <= tk) {
        int64_t id = ids[idbase + row];
        if (lex_less(k, id, tk, ti)) {
          ck[i] = k;
          ci[i] = id;
          have = true;
        }
      }
    }
  }
  if (!__any_sync(FULL, have)) return;
  warp_merge_into_list(S, a, kk, ck, ci);
}

// Producer warp of the persistent scans: claims work items, publishes them
// through a 2-deep ring, and streams each item's row tiles (TMA 2-D,
// SWIZZLE_128B, box heights 256..8 to cover ragged tails) and the matching
// 128-byte query chunks (bulk copies) through the STAGES-deep stage ring.
template <int NSTAGE>
__device__ __forceinline__ void scan_producer(const ScanShared& S, const ArenaMaps& maps,
                                              const ListTable& lt, const float* __restrict__ Qd,
                                              const ScanItem* __restrict__ items, const int32_t* __restrict__ nctr,
                                              const QPair* __restrict__ qpairs,
                                              int32_t* __restrict__ work_ctr, int nchunk_d,
                                              bool keep_in_l2, int64_t qsw_stride,
                                              const CUtensorMap* qg = nullptr, int early_ctas = 0,
                                              int early_at = 0x7fffffff) {
  // front items [0, nctr[0]) then the tail items, stored backwards from nctr[3]
  const int n_front = nctr[0], n_items = n_front + nctr[2], tail_base = nctr[3];
  const int lane = threadIdx.x & 31;
  if (lane == 0)
    for (int i = 0; i < NBOX; i++) tma_prefetch_desc(&maps.box[i]);
  const uint64_t pol = keep_in_l2 ? policy_evict_normal() : policy_evict_first();
  int s = 0, r = 0;
  uint32_t ph = 0, rph = 0;
  for (;;) {
    int it = 0;
    // the first early_ctas CTAs stop claiming once early_at items are taken,
    // handing their SMs to the next batch's front half sooner
    // (at most half the grid, so the rest always drains the queue)
    const bool stop = (int)blockIdx.x < min(early_ctas, (int)gridDim.x / 2) &&
                      *(volatile int32_t*)work_ctr >= early_at;
    if (lane == 0) it = stop ? 0x7fffffff : atomicAdd(work_ctr, 1);
    it = __shfl_sync(FULL, it, 0);
    ScanItem item;
    if (it < n_items) {
      item = items[it < n_front ? it : tail_base - (it - n_front)];
    } else {
      item.nq = -1;
    }
    mbar_wait(&S.rempty[r], rph ^ 1);
    if (lane == 0) {
      S.ring[r] = item;
      mbar_arrive(&S.rfull[r]);
    }
    if (++r == 2) {
      r = 0;
      rph ^= 1;
    }
    if (item.nq < 0) break;
    const int64_t rbase = lt.off[item.lslot] + item.row0;
    const int qb = lane < item.nq ? qpairs[item.qoff + lane].b : 0;
    // qsw_stride > 0: Qd holds 8 copies of the batch, copy p with the 16-byte
    // pieces of every 128-byte chunk XOR-permuted by p, so query slot `lane`
    // lands SWIZZLE_128B-ready in row `lane` of the stage's query tile.
    const float* qrow =
        Qd + ((qsw_stride ? (int64_t)(lane & 7) * qsw_stride : 0) + qb) * (int64_t)lt.dp;
    // qg: the item's query chunk comes in ceil(nq / 4) gathers of four rows
    // of the (unswizzled) batch -- lane j < ngq issues group j, slots past nq
    // repeat the last query (their dots are never read)
    const int ngq = (item.nq + 3) >> 2;
    int g0 = 0, g1 = 0, g2 = 0, g3 = 0;
    if (qg) {
      const int last = item.nq - 1;
      g0 = __shfl_sync(FULL, qb, min(4 * lane + 0, last) & 31);
      g1 = __shfl_sync(FULL, qb, min(4 * lane + 1, last) & 31);
      g2 = __shfl_sync(FULL, qb, min(4 * lane + 2, last) & 31);
      g3 = __shfl_sync(FULL, qb, min(4 * lane + 3, last) & 31);
    }
    const int qbytes = qg ? ngq * 4 * DC * 4 : item.nq * DC * 4;
    for (int t0 = 0; t0 < item.nrows; t0 += TILE) {
      const int rows = min(TILE, item.nrows - t0);
      const int rows8 = (rows + 7) & ~7;
      const uint32_t bytes = (uint32_t)(rows8 * DC * 4 + qbytes);
      for (int c = 0; c < nchunk_d; c++) {
        mbar_wait(&S.empty[s], ph ^ 1);
        if (lane == 0) {
          mbar_arrive_expect_tx(&S.full[s], bytes);
          int r0 = 0;
#pragma unroll
          for (int bi = 0; bi < NBOX; bi++) {
            const int h = TILE >> bi;
            if (rows8 - r0 >= h) {
              tma_load_2d(S.X + (size_t)s * TILE * DC + r0 * DC, &maps.box[bi], &S.full[s],
                          c * DC, (int)(rbase + t0 + r0), pol);
              r0 += h;
            }
          }
        }
        __syncwarp();
        if (qg) {
          if (lane < ngq)
            tma_gather4(S.Qc + (size_t)s * QG * DC + lane * 4 * DC, qg, &S.full[s], c * DC, g0, g1, g2, g3,
                        pol);
        } else if (lane < item.nq) {
          bulk_g2s(S.Qc + (size_t)s * QG * DC + lane * DC, qrow + c * DC, DC * 4, &S.full[s]);
        }
        if (++s == NSTAGE) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  }
}

template <int METRIC>
__global__ void __launch_bounds__(SCAN_THREADS, 1)
    scan_kernel(const __grid_constant__ ArenaMaps maps, ListTable lt, const float* __restrict__ Qd,
                const float* __restrict__ qnorm, const ScanItem* __restrict__ items,
                const int32_t* __restrict__ n_items_p, const QPair* __restrict__ qpairs, int kk,
                int32_t* __restrict__ work_ctr, uint32_t* __restrict__ cand_key,
                int64_t* __restrict__ cand_id, int32_t* __restrict__ cand_n,
                int32_t* __restrict__ cand_list) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment for SWIZZLE_128B; index off the __shared__ array so the
  // compiler keeps shared-space (LDS) addressing.
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  ScanShared S;
  S.X = reinterpret_cast<float*>(base);
  S.Qc = reinterpret_cast<float*>(base + ScanLayout::X_BYTES);
  S.D = reinterpret_cast<float*>(base + ScanLayout::X_BYTES + ScanLayout::QC_BYTES);
  uint8_t* p = base + ScanLayout::X_BYTES + ScanLayout::QC_BYTES + ScanLayout::D_BYTES;
  S.Lkey = reinterpret_cast<uint32_t*>(p);
  p += ScanLayout::LK_BYTES;
  S.Lid = reinterpret_cast<int64_t*>(p);
  p += ScanLayout::LI_BYTES;
  S.Ln = reinterpret_cast<int32_t*>(p);
  p += ScanLayout::LN_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(p);
  S.full = bars;
  S.empty = bars + STAGES;
  S.rfull = bars + 2 * STAGES;
  S.rempty = bars + 2 * STAGES + 2;
  p += ScanLayout::BAR_BYTES;
  S.ring = reinterpret_cast<ScanItem*>(p);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; i++) {
      mbar_init(&S.full[i], 1);
      mbar_init(&S.empty[i], NCW);
    }
    for (int i = 0; i < 2; i++) {
      mbar_init(&S.rfull[i], 1);
      mbar_init(&S.rempty[i], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int nchunk_d = lt.dp / DC;


  if (warp == NCW) {
    scan_producer<STAGES>(S, maps, lt, Qd, items, n_items_p, qpairs, work_ctr, nchunk_d, false, 0);
    return;
  }

  // -------------------------------------------------- compute warps
  __shared__ float qn_s[QG];
  int s = 0, r = 0;
  uint32_t ph = 0, rph = 0;
  for (;;) {
    mbar_wait(&S.rfull[r], rph);
    const ScanItem item = S.ring[r];
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.rempty[r]);
    if (++r == 2) {
      r = 0;
      rph ^= 1;
    }
    if (item.nq < 0) break;
    const int qa0 = warp, qa1 = warp + NCW;
    if (lane == 0) {
      S.Ln[qa0] = 0;
      S.Ln[qa1] = 0;
    }
    if (METRIC == COSINE && threadIdx.x < QG)
      qn_s[threadIdx.x] = threadIdx.x < item.nq ? qnorm[qpairs[item.qoff + threadIdx.x].b] : 0.f;
    named_bar_sync(1, NCW * 32);  // Ln reset + qn_s visible
    const int64_t idbase0 = lt.off[item.lslot] + item.row0;
    for (int t0 = 0; t0 < item.nrows; t0 += TILE) {
      const int rows = min(TILE, item.nrows - t0);
      const int nq = item.nq;
      if (nq <= 1) scan_tile<METRIC, 1>(S, nchunk_d, s, ph, nq, qn_s);
      else if (nq <= 2) scan_tile<METRIC, 2>(S, nchunk_d, s, ph, nq, qn_s);
      else if (nq <= 4) scan_tile<METRIC, 4>(S, nchunk_d, s, ph, nq, qn_s);
      else if (nq <= 6) scan_tile<METRIC, 6>(S, nchunk_d, s, ph, nq, qn_s);
      else if (nq <= 8) scan_tile<METRIC, 8>(S, nchunk_d, s, ph, nq, qn_s);
      else if (nq <= 12) scan_tile<METRIC, 12>(S, nchunk_d, s, ph, nq, qn_s);
      else scan_tile<METRIC, 16>(S, nchunk_d, s, ph, nq, qn_s);
      named_bar_sync(1, NCW * 32);
      if (qa0 < nq) topk_merge_tile(S, qa0, rows, lt.ids, idbase0 + t0, kk);
      if (qa1 < nq) topk_merge_tile(S, qa1, rows, lt.ids, idbase0 + t0, kk);
      named_bar_sync(1, NCW * 32);
    }
    // write this item's per-query lists to their output slots
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int a = h ? qa1 : qa0;
      if (a >= item.nq) continue;
      const QPair qp = qpairs[item.qoff + a];
      const int64_t slot = (int64_t)qp.slotbase + item.chunk;
      const int n = S.Ln[a];
      for (int l = lane; l < n; l += 32) {
        cand_key[slot * kk + l] = S.Lkey[a * KKMAX + l];
        cand_id[slot * kk + l] = S.Lid[a * KKMAX + l];
      }
      if (lane == 0) {
        cand_n[slot] = n;
        cand_list[slot] = item.lslot;
      }
    }
  }
}

void launch_scan(int metric, ListTable lt, const ArenaMaps& maps, const float* Qd,
                 const float* qnorm, const ScanItem* items, const int32_t* n_items,
                 int max_items, const QPair* qpairs, int kk, int32_t* work_ctr,
                 uint32_t* cand_key, int64_t* cand_id, int32_t* cand_n, int32_t* cand_list,
                 int num_sms, cudaStream_t st) {
  if (max_items <= 0) return;
  size_t smem = scan_smem_bytes();
  int grid = std::min(num_sms, max_items);
#define PK_SCAN(M)                                                                                \
  {                                                                                               \
    auto k = scan_kernel<M>;                                                                      \
    PK_SMEM_ATTR(k, (int)smem);              \
    k<<<grid, SCAN_THREADS, smem, st>>>(maps, lt, Qd, qnorm, items, n_items, qpairs, kk, work_ctr, \
                                        cand_key, cand_id, cand_n, cand_list);                    \
  }
  if (metric == SQ_L2) PK_SCAN(SQ_L2)
  else if (metric == IP) PK_SCAN(IP)
  else PK_SCAN(COSINE)
#undef PK_SCAN
}

// =====================================================================
// Final merge per query: its candidate slots -> top kk by (dist, id),
// first occurrence per id (ref/engine.py:406-426).
// =====================================================================
constexpr int MERGE_CAP = 2048;
__global__ void __launch_bounds__(128) merge_kernel(const int32_t* __restrict__ slot_off,
                                                    const uint32_t* __restrict__ cand_key,
                                                    const int64_t* __restrict__ cand_id,
                                                    const int32_t* __restrict__ cand_n,
                                                    const int32_t* __restrict__ cand_list, int kk,
                                                    ListTable lt, int64_t* __restrict__ out_ids,
                                                    float* __restrict__ out_d,
                                                    int64_t* __restrict__ out_cid,
                                                    int32_t* __restrict__ out_n) {
  extern __shared__ Entry mbuf[];  // [MERGE_CAP]
  __shared__ int s_cnt;
  __shared__ uint32_t s_tk[4];
  __shared__ int64_t s_ti[4];
  const int b = blockIdx.x;
  const int so = slot_off[2 * b], eo = slot_off[2 * b + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // tau: best "last entry" among full slots (each full slot has kk distinct ids <= it)
  uint32_t tk = KEY_NONE;
  int64_t ti = ID_NONE;
  for (int sl = so + threadIdx.x; sl < eo; sl += blockDim.x) {
    if (cand_n[sl] == kk) {
      uint32_t k = cand_key[(int64_t)sl * kk + kk - 1];
      int64_t i = cand_id[(int64_t)sl * kk + kk - 1];
      if (lex_less(k, i, tk, ti)) {
        tk = k;
        ti = i;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    uint32_t k2 = __shfl_xor_sync(FULL, tk, o);
    int64_t i2 = __shfl_xor_sync(FULL, ti, o);
    if (lex_less(k2, i2, tk, ti)) {
      tk = k2;
      ti = i2;
    }
  }
  if (lane == 0) {
    s_tk[warp] = tk;
    s_ti[warp] = ti;
  }
  __syncthreads();
  tk = s_tk[0];
  ti = s_ti[0];
  for (int w = 1; w < 4; w++)
    if (lex_less(s_tk[w], s_ti[w], tk, ti)) {
      tk = s_tk[w];
      ti = s_ti[w];
    }
  // collect survivors (<= tau) slot group by slot group, keeping the best kk
  const int group = max(1, (MERGE_CAP - kk) / kk);
  int kept = 0;
  for (int g0 = so; g0 < eo; g0 += group) {
    const int g1 = min(eo, g0 + group);
    if (threadIdx.x == 0) s_cnt = kept;
    __syncthreads();
    for (int sl = g0 + threadIdx.x; sl < g1; sl += blockDim.x) {
      const int n = cand_n[sl];
      const int lst = cand_list[sl];
      for (int e = 0; e < n; e++) {
        const uint32_t k = cand_key[(int64_t)sl * kk + e];
        const int64_t i = cand_id[(int64_t)sl * kk + e];
        if (lex_less(tk, ti, k, i)) break;  // slot lists are sorted
        int pos = atomicAdd(&s_cnt, 1);
        Entry en;
        en.key = k;
        en.id = i;
        en.pay = lst;
        mbuf[pos] = en;
      }
    }
    __syncthreads();
    const int n = s_cnt;
    if (n > kept || g0 == so) {
      cta_bitonic_sort(mbuf, n);
      kept = cta_compact_sorted(mbuf, n, kk, true, &s_cnt);
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < kk; i += blockDim.x) {
    const int64_t o = (int64_t)b * kk + i;
    if (i < kept) {
      out_ids[o] = mbuf[i].id;
      out_d[o] = key2dist(mbuf[i].key, lt.metric);
      if (out_cid) out_cid[o] = lt.cid[mbuf[i].pay];
    } else {
      out_ids[o] = -1;
      out_d[o] = __int_as_float(0x7f800000);
      if (out_cid) out_cid[o] = -1;
    }
  }
  if (threadIdx.x == 0) out_n[b] = kept;
}

void launch_merge(int B, const int32_t* slot_off, const uint32_t* cand_key, const int64_t* cand_id,
                  const int32_t* cand_n, const int32_t* cand_list, int kk, ListTable lt,
                  int64_t* out_ids, float* out_d, int64_t* out_cid, int32_t* out_n,
                  cudaStream_t st) {
  if (B <= 0) return;
  size_t smem = MERGE_CAP * sizeof(Entry);
  PK_SMEM_ATTR(merge_kernel, (int)smem);
  merge_kernel<<<B, 128, smem, st>>>(slot_off, cand_key, cand_id, cand_n, cand_list, kk, lt,
                                     out_ids, out_d, out_cid, out_n);
}

// =====================================================================
// Screened fused scan (sq_l2 and neg_ip) + exact re-rank.
//
// The exact reference distance costs 3 separately rounded FP32 ops per
// (query, element) -- more FP32 issue than HBM delivers elements at ~8 queries
// per list.  The screen kernel streams the same tiles
// but computes, per (row, query), an FFMA approximation with a PROVEN error
// bound eps against the reference value E:
//   sq_l2: A = (nx + nq) - 2 dot,  nx = sum x*x, dot = sum x*q (FFMA chains)
//   neg_ip: A = -dot
//   |A - E| <= eps = coef * (nx + nq)    (coef from d, screen_coef())
// Per (item, query) U_item = kk-th smallest (A + eps) over the item's rows is
// an upper bound of the query's final kk-th exact distance; the query's global
// bound Uq[b] is the atomic min of those.  A row can only be in the query's
// top-kk if A - eps <= Uq[b] (kk rows have E <= A + eps <= Uq), so exactly
// those rows are appended to the query's candidate pool, and
// rerank_merge_kernel computes their reference distances and the top-kk.
// Directed rounding (ru/rd) keeps the bound valid through the fp32 ops;
// non-finite values become unconditional candidates.
// =====================================================================
constexpr int CHUNK_MAX = 2 * TILE;  // rows per screened work item

struct ScreenLayout {
  static constexpr size_t X_BYTES = (size_t)STAGES * TILE * DC * 4;
  static constexpr size_t QC_BYTES = (size_t)STAGES * QG * DC * 4;
  static constexpr size_t A_BYTES = (size_t)QG * CHUNK_MAX * 4;
  static constexpr size_t NX_BYTES = (size_t)CHUNK_MAX * 4;
  static constexpr size_t BAR_BYTES = 256;
  static constexpr size_t RING_BYTES = 2 * sizeof(ScanItem);
  static constexpr size_t TOTAL = X_BYTES + QC_BYTES + A_BYTES + NX_BYTES + BAR_BYTES + RING_BYTES;
};
size_t screen_smem_bytes() { return ScreenLayout::TOTAL + 1024; }

// FFMA screen of one tile, register-blocked 4 rows x NQT queries per thread
// (LDS : FFMA = 8 : 64 -- one-row-per-thread blocking is shared-memory-issue
// bound).  Thread tid < 256: row group rg = tid % 64 owns rows rg + 64 r,
// query group qg = tid / 64 owns queries 4 qg .. 4 qg + 3; group 0 also
// accumulates the row norms.  Threads with no query group only keep the
// stage ring in step.  Stores raw dots; screen_finalize forms A.
template <int NQT>
__device__ __forceinline__ void screen_tile(const ScanShared& S, int nchunk_d, int& s, uint32_t& ph,
                                            int nq, int tile_row0) {
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int rg = tid & 63, qg = tid >> 6;
  const int qbase = qg * 4;
  const bool active = qbase < nq;
  const bool do_norm = qg == 0;
  const int swz = rg & 7;
  float acc[4][NQT];
  float nx[4];
#pragma unroll
  for (int r = 0; r < 4; r++) {
    nx[r] = 0.f;
#pragma unroll
    for (int a = 0; a < NQT; a++) acc[r][a] = 0.f;
  }
  for (int c = 0; c < nchunk_d; c++) {
    mbar_wait(&S.full[s], ph);
    if (active) {
      const float* xs = S.X + (size_t)s * TILE * DC + rg * DC;
      const float* qs = S.Qc + (size_t)s * QG * DC + qbase * DC;
#pragma unroll
      for (int k = 0; k < DC / 4; k++) {
        float4 x[4];
#pragma unroll
        for (int r = 0; r < 4; r++)
          x[r] = *reinterpret_cast<const float4*>(xs + r * 64 * DC + ((k ^ swz) << 2));
        if (do_norm) {
#pragma unroll
          for (int r = 0; r < 4; r++) {
            nx[r] = __fmaf_rn(x[r].x, x[r].x, nx[r]);
            nx[r] = __fmaf_rn(x[r].y, x[r].y, nx[r]);
            nx[r] = __fmaf_rn(x[r].z, x[r].z, nx[r]);
            nx[r] = __fmaf_rn(x[r].w, x[r].w, nx[r]);
          }
        }
#pragma unroll
        for (int a = 0; a < NQT; a++) {
          const float4 q = *reinterpret_cast<const float4*>(qs + a * DC + (k << 2));
#pragma unroll
          for (int r = 0; r < 4; r++) {
            acc[r][a] = __fmaf_rn(x[r].x, q.x, acc[r][a]);
            acc[r][a] = __fmaf_rn(x[r].y, q.y, acc[r][a]);
            acc[r][a] = __fmaf_rn(x[r].z, q.z, acc[r][a]);
            acc[r][a] = __fmaf_rn(x[r].w, q.w, acc[r][a]);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.empty[s]);
    if (++s == STAGES) {
      s = 0;
      ph ^= 1;
    }
  }
  if (do_norm) {
#pragma unroll
    for (int r = 0; r < 4; r++) S.NX[tile_row0 + rg + 64 * r] = nx[r];
  }
  if (active) {
#pragma unroll
    for (int a = 0; a < NQT; a++)
      if (qbase + a < nq) {
#pragma unroll
        for (int r = 0; r < 4; r++)
          S.A[(qbase + a) * CHUNK_MAX + tile_row0 + rg + 64 * r] = acc[r][a];
      }
  }
}

// A = nx + nq - 2 dot (sq_l2) or -dot (ip), in place over the item's rows.
template <int METRIC>
__device__ __forceinline__ void screen_finalize(const ScanShared& S, int nq, int R,
                                                const float* nq2_s, int tid, int nthreads) {
  for (int i = tid; i < nq * R; i += nthreads) {
    const int a = i / R, row = i - a * R;
    const float dot = S.A[a * CHUNK_MAX + row];
    S.A[a * CHUNK_MAX + row] = (METRIC == SQ_L2)
                                   ? __fsub_rn(__fadd_rn(S.NX[row], nq2_s[a]), __fmul_rn(2.f, dot))
                                   : -dot;
  }
}

// Per (item, query a): publish the item's kk smallest upper bounds (hi) to
// the (query, item) slot, tighten the query's running bound Uq with the
// item's kk-th smallest hi, and append every row whose lower bound (lo) is
// not above min(U_item, Uq) to the query's pool together with lo.
__device__ __forceinline__ void screen_select(const ScanShared& S, int a, int R, int kk, float coef,
                                              float nqa, int b, int lslot, int64_t rbase,
                                              int64_t slot, uint32_t* __restrict__ Uq,
                                              uint32_t* __restrict__ slot_hi,
                                              int32_t* __restrict__ slot_n,
                                              int4* __restrict__ cpool,
                                              int32_t* __restrict__ ccount, int cap,
                                              uint32_t u0_pre = 0, bool have_u0 = false) {
  const int lane = threadIdx.x & 31;
  constexpr int PER = CHUNK_MAX / 32;
  uint32_t hk[PER], lk[PER];
#pragma unroll
  for (int i = 0; i < PER; i++) {
    const int row = lane + 32 * i;
    hk[i] = KEY_NONE;
    lk[i] = KEY_NONE;
    if (row < R) {
      const float A = S.A[a * CHUNK_MAX + row];
      const float eps = __fmul_ru(coef, __fadd_ru(S.NX[row], nqa));
      float hi = __fadd_ru(A, eps), lo = __fsub_rd(A, eps);
      if (!isfinite(hi) || !isfinite(lo)) {
        hi = __int_as_float(0x7f800000);
        lo = __int_as_float(0xff800000);
      }
      hk[i] = f2key(hi);
      lk[i] = f2key(lo);
    }
  }
  // Only this item's rows with hi <= the query's current bound U0 can matter:
  // the re-rank's bound is the kk-th smallest published hi, which never
  // exceeds Uq <= U0, and every value at or under it is <= U0 when published.
  // So when fewer than kk rows are under U0 (the common case once the bound
  // has tightened) they are published as they are, with no selection; else
  // U_item = kk-th smallest hi (bisection over [min, U0]) tightens Uq and the
  // item's kk smallest hi are published.
  // (the tensor-core scan prefetches it while the item's A values are formed)
  const uint32_t U0 = have_u0 ? u0_pre : *(volatile uint32_t*)&Uq[b];
  unsigned c0 = 0;
  uint32_t mn = KEY_NONE, mx = 0;
#pragma unroll
  for (int i = 0; i < PER; i++) {
    if (lane + 32 * i < R && hk[i] <= U0) {
      c0++;
      mn = min(mn, hk[i]);
      mx = max(mx, hk[i]);
    }
  }
  const unsigned cnt0 = __reduce_add_sync(FULL, c0);
  uint32_t Uitem = KEY_NONE;
  if (cnt0 >= (unsigned)kk) {
    uint32_t L = __reduce_min_sync(FULL, mn), H = __reduce_max_sync(FULL, mx);
    while (L < H) {
      const uint32_t mid = L + ((H - L) >> 1);
      unsigned cc = 0;
#pragma unroll
      for (int i = 0; i < PER; i++) cc += (lane + 32 * i < R) && (hk[i] <= mid);
      if (__reduce_add_sync(FULL, cc) >= (unsigned)kk) H = mid;
      else L = mid + 1;
    }
    Uitem = L;
    if (lane == 0) atomicMin(&Uq[b], Uitem);
  }
  {
    // cnt0 >= kk: every hi < U_item, then U_item repeated (kk values);
    // else: every hi <= U0 (cnt0 < kk values)
    const bool sel = cnt0 >= (unsigned)kk;
    int base = 0;
#pragma unroll
    for (int i = 0; i < PER; i++) {
      const bool below = (lane + 32 * i < R) && (sel ? hk[i] < Uitem : hk[i] <= U0);
      const unsigned bal = __ballot_sync(FULL, below);
      if (below) slot_hi[slot * kk + base + __popc(bal & ((1u << lane) - 1u))] = hk[i];
      base += __popc(bal);
    }
    const int nfill = sel ? kk : base;
    for (int l = base + lane; l < nfill; l += 32) slot_hi[slot * kk + l] = Uitem;
    if (lane == 0) slot_n[slot] = nfill;
  }
  // candidate bound: this item's own U_item and the query bound it started
  // from (a concurrent tightening elsewhere only makes it looser, never wrong)
  const uint32_t U = min(Uitem, have_u0 ? U0 : *(volatile uint32_t*)&Uq[b]);
  unsigned tot = 0;
#pragma unroll
  for (int i = 0; i < PER; i++) tot += (lane + 32 * i < R && lk[i] <= U);
  tot = __reduce_add_sync(FULL, tot);
  if (tot == 0) return;
  int base = 0;
  if (lane == 0) base = atomicAdd(&ccount[b], (int)tot);
  base = __shfl_sync(FULL, base, 0);
#pragma unroll
  for (int i = 0; i < PER; i++) {
    const int row = lane + 32 * i;
    const bool cand = row < R && lk[i] <= U;
    const unsigned bal = __ballot_sync(FULL, cand);
    const int pos = base + __popc(bal & ((1u << lane) - 1u));
    if (cand && pos < cap)
      cpool[(int64_t)b * cap + pos] = make_int4((int)(rbase + row), lslot, (int)lk[i], 0);
    base += __popc(bal);
  }
}

constexpr int NCW_S = 8;  // screen kernel compute warps (256 threads: 64 row groups x 4 query groups)
constexpr int SCREEN_THREADS = (NCW_S + 1) * 32;

template <int METRIC>
__global__ void __launch_bounds__(SCREEN_THREADS, 1)
    scan_screen_kernel(const __grid_constant__ ArenaMaps maps, ListTable lt,
                       const float* __restrict__ Qd, const float* __restrict__ qnorm2,
                       const ScanItem* __restrict__ items, const int32_t* __restrict__ n_items_p,
                       const QPair* __restrict__ qpairs, int kk, float coef,
                       int32_t* __restrict__ work_ctr, uint32_t* __restrict__ Uq,
                       uint32_t* __restrict__ slot_hi, int32_t* __restrict__ slot_n,
                       int4* __restrict__ cpool, int32_t* __restrict__ ccount, int cap,
                       int debug_nocompute) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  ScanShared S;
  uint8_t* p = base;
  S.X = reinterpret_cast<float*>(p);
  p += ScreenLayout::X_BYTES;
  S.Qc = reinterpret_cast<float*>(p);
  p += ScreenLayout::QC_BYTES;
  S.A = reinterpret_cast<float*>(p);
  p += ScreenLayout::A_BYTES;
  S.NX = reinterpret_cast<float*>(p);
  p += ScreenLayout::NX_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(p);
  S.full = bars;
  S.empty = bars + STAGES;
  S.rfull = bars + 2 * STAGES;
  S.rempty = bars + 2 * STAGES + 2;
  p += ScreenLayout::BAR_BYTES;
  S.ring = reinterpret_cast<ScanItem*>(p);
  S.D = nullptr;
  S.Lkey = nullptr;
  S.Lid = nullptr;
  S.Ln = nullptr;
  S.CR = nullptr;
  S.Cn = nullptr;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; i++) {
      mbar_init(&S.full[i], 1);
      mbar_init(&S.empty[i], NCW_S);
    }
    for (int i = 0; i < 2; i++) {
      mbar_init(&S.rfull[i], 1);
      mbar_init(&S.rempty[i], NCW_S);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int nchunk_d = lt.dp / DC;

  if (warp == NCW_S) {
    scan_producer<STAGES>(S, maps, lt, Qd, items, n_items_p, qpairs, work_ctr, nchunk_d, false, 0);
    return;
  }

  __shared__ float nq2_s[QG];
  __shared__ int32_t qb_s[QG];
  int s = 0, r = 0;
  uint32_t ph = 0, rph = 0;
  for (;;) {
    mbar_wait(&S.rfull[r], rph);
    const ScanItem item = S.ring[r];
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.rempty[r]);
    if (++r == 2) {
      r = 0;
      rph ^= 1;
    }
    if (item.nq < 0) break;
    const int nq = item.nq;
    if (threadIdx.x < QG) {
      const int b = threadIdx.x < nq ? qpairs[item.qoff + threadIdx.x].b : 0;
      qb_s[threadIdx.x] = b;
      nq2_s[threadIdx.x] = threadIdx.x < nq ? qnorm2[b] : 0.f;
    }
    named_bar_sync(1, NCW_S * 32);
    {
      const int nqc = debug_nocompute == 1 ? 0 : nq;
      for (int t0 = 0; t0 < item.nrows; t0 += TILE) {
        if (nqc <= 1) screen_tile<1>(S, nchunk_d, s, ph, nqc, t0);
        else if (nqc <= 2) screen_tile<2>(S, nchunk_d, s, ph, nqc, t0);
        else if (nqc <= 3) screen_tile<3>(S, nchunk_d, s, ph, nqc, t0);
        else screen_tile<4>(S, nchunk_d, s, ph, nqc, t0);
      }
    }
    named_bar_sync(1, NCW_S * 32);
    if (debug_nocompute) continue;  // measurement only: 1 = memory pipeline, 2 = + screen math
    screen_finalize<METRIC>(S, nq, item.nrows, nq2_s, threadIdx.x, NCW_S * 32);
    named_bar_sync(1, NCW_S * 32);
    const int64_t rbase = lt.off[item.lslot] + item.row0;
    for (int a = warp; a < nq; a += NCW_S)
      screen_select(S, a, item.nrows, kk, coef, nq2_s[a], qb_s[a], item.lslot, rbase,
                    (int64_t)qpairs[item.qoff + a].slotbase + item.chunk, Uq, slot_hi, slot_n,
                    cpool, ccount, cap);
    named_bar_sync(1, NCW_S * 32);  // A / NX reuse by the next item
  }
}

// =====================================================================
// Tensor-core screened scan (sq_l2 / neg_ip): the same streaming, bound and
// candidate logic as scan_screen_kernel, with the (row, query) dot products
// computed by tcgen05.mma kind::tf32 straight from the TMA-staged tiles.
//
// Roles (320 threads, one CTA per SM):
//   warp 8      TMA producer: row tiles [256 x 32 fp32] SWIZZLE_128B + the
//               query chunks from 8 pre-swizzled copies of the batch, through
//               a TC_STAGES-deep mbarrier ring
//   warp 9      MMA issuer (one lane): per stage 2 halves x 4 K-steps of
//               M=128, N=16, K=8 TF32 MMAs into a TMEM accumulator
//               (double-buffered per tile); tcgen05.commit frees the stage
//   warps 0-7   epilogue: tcgen05.ld of the tile's [256 x 16] dots, then per
//               item the bound, publication and candidate pool (as above)
// TF32 bound (validated by tools/microbench/umma_check.cu): |dot' - x.q| <=
// c_dot * sum|x_j q_j|, c_dot = 2.0011*2^-10 + d*2^-21 (input truncation +
// accumulation), used with a 2x safety factor in screen_coef_tf32().
// Row norms come from the arena's norm array (FFMA, any order).
// =====================================================================
constexpr int TC_STAGES = 5;
constexpr int TC_EPI_WARPS = 8;
constexpr int TC_THREADS = (TC_EPI_WARPS + 2) * 32;
constexpr int TC_TBUF = 4;         // TMEM accumulator buffers (tiles in flight between MMA and epilogue)
constexpr int TC_TMEM_COLS = TC_TBUF * 2 * QG;  // x 2 halves x 16 queries

struct TcLayout {
  static constexpr size_t X_BYTES = (size_t)TC_STAGES * TILE * DC * 4;
  static constexpr size_t QC_BYTES = (size_t)TC_STAGES * QG * DC * 4;
  static constexpr size_t A_BYTES = (size_t)QG * CHUNK_MAX * 4;
  static constexpr size_t NX_BYTES = (size_t)CHUNK_MAX * 4;
  static constexpr size_t BAR_BYTES = 256;
  static constexpr size_t RING_BYTES = 2 * sizeof(ScanItem);
  static constexpr size_t TOTAL = X_BYTES + QC_BYTES + A_BYTES + NX_BYTES + BAR_BYTES + RING_BYTES + 64;
};
size_t tc_smem_bytes() { return TcLayout::TOTAL + 1024; }

// Items taken before the early CTAs stop claiming: a fraction of the queue,
// or none at all when the queue is short (fewer than early_small items per
// CTA): such a scan is latency-bound, and the next front half (one pick CTA
// per query) is the pipeline's critical path -- it gets those SMs from the
// start (configs[0]: step 49.6 -> 40.0 us).
__device__ __forceinline__ int early_at_of(int n_items, float early_frac, int early_small) {
  return n_items < early_small * (int)gridDim.x ? 0 : (int)(early_frac * (float)n_items);
}

template <int METRIC>
__global__ void __launch_bounds__(TC_THREADS, 1)
    scan_tc_kernel(const __grid_constant__ ArenaMaps maps, const __grid_constant__ CUtensorMap qgmap,
                   bool use_qg, ListTable lt, const float* __restrict__ Qsw,
                   int64_t qsw_stride, const float* __restrict__ qnorm2,
                   const ScanItem* __restrict__ items, const int32_t* __restrict__ n_items_p,
                   const QPair* __restrict__ qpairs, int kk, float coef,
                   int32_t* __restrict__ work_ctr, uint32_t* __restrict__ Uq,
                   uint32_t* __restrict__ slot_hi, int32_t* __restrict__ slot_n,
                   int4* __restrict__ cpool, int32_t* __restrict__ ccount, int cap, int dbg_skip,
                   unsigned long long* __restrict__ dbg_t, int early_ctas, float early_frac,
                   int early_small) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  ScanShared S;
  uint8_t* p = base;
  S.X = reinterpret_cast<float*>(p);
  p += TcLayout::X_BYTES;
  S.Qc = reinterpret_cast<float*>(p);
  p += TcLayout::QC_BYTES;
  S.A = reinterpret_cast<float*>(p);
  p += TcLayout::A_BYTES;
  S.NX = reinterpret_cast<float*>(p);
  p += TcLayout::NX_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(p);
  S.full = bars;
  S.empty = bars + TC_STAGES;
  uint64_t* tfull = bars + 2 * TC_STAGES;
  uint64_t* tempty = tfull + TC_TBUF;
  S.rfull = tempty + TC_TBUF;
  S.rempty = S.rfull + 2;
  p += TcLayout::BAR_BYTES;
  S.ring = reinterpret_cast<ScanItem*>(p);
  p += TcLayout::RING_BYTES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(p);
  S.D = nullptr;
  S.Lkey = nullptr;
  S.Lid = nullptr;
  S.Ln = nullptr;
  S.CR = nullptr;
  S.Cn = nullptr;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < TC_STAGES; i++) {
      mbar_init(&S.full[i], 1);
      mbar_init(&S.empty[i], 1);  // tcgen05.commit
    }
    for (int i = 0; i < TC_TBUF; i++) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], TC_EPI_WARPS);
    }
    for (int i = 0; i < 2; i++) {
      mbar_init(&S.rfull[i], 1);
      mbar_init(&S.rempty[i], TC_EPI_WARPS + 1);
    }
    fence_mbar_init();
  }
  if (warp == TC_EPI_WARPS + 1) tmem_alloc(tmem_slot, TC_TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_trigger();
  pdl_wait();  // items, queries and counters come from the kernels before
  if (dbg_t && threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    dbg_t[2 * blockIdx.x] = globaltimer_ns();
    dbg_t[2 * gridDim.x + blockIdx.x] = smid;
  }
  const uint32_t tmem = *tmem_slot;
  const int nchunk_d = lt.dp / DC;


  if (warp == TC_EPI_WARPS) {
    // ---------------------------------------------------------- producer
    scan_producer<TC_STAGES>(S, maps, lt, Qsw, items, n_items_p, qpairs, work_ctr, nchunk_d, false,
                             qsw_stride, use_qg ? &qgmap : nullptr, early_ctas,
                             early_at_of(n_items_p[0] + n_items_p[2], early_frac, early_small));
  } else if (warp == TC_EPI_WARPS + 1) {
    // ---------------------------------------------------------- MMA issuer
    const uint32_t idesc = umma_idesc_tf32(128, QG);
    int s = 0, r = 0, tcount = 0;
    uint32_t ph = 0, rph = 0;
    for (;;) {
      mbar_wait(&S.rfull[r], rph);
      const ScanItem item = S.ring[r];
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.rempty[r]);
      if (++r == 2) {
        r = 0;
        rph ^= 1;
      }
      if (item.nq < 0) break;
      for (int t0 = 0; t0 < item.nrows; t0 += TILE) {
        const int buf = tcount % TC_TBUF;
        mbar_wait(&tempty[buf], ((tcount / TC_TBUF) & 1) ^ 1);
        tc_fence_after();
        const uint32_t dcol = tmem + buf * 2 * QG;
        const bool two = item.nrows - t0 > 128;
        for (int c = 0; c < nchunk_d; c++) {
          mbar_wait(&S.full[s], ph);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t xa = smem_u32(S.X + (size_t)s * TILE * DC);
            const uint32_t qa = smem_u32(S.Qc + (size_t)s * QG * DC);
#pragma unroll
            for (int k = 0; k < DC / 8; k++) {
              const uint64_t bd = umma_desc_sw128(qa + k * 32);
              const uint32_t acc = (c | k) != 0;
              umma_tf32(dcol, umma_desc_sw128(xa + k * 32), bd, idesc, acc);
              if (two) umma_tf32(dcol + QG, umma_desc_sw128(xa + 16384 + k * 32), bd, idesc, acc);
            }
            umma_commit(&S.empty[s]);
          }
          __syncwarp();
          if (++s == TC_STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        if (lane == 0) umma_commit(&tfull[buf]);
        __syncwarp();
        tcount++;
      }
    }
  } else {
    // ---------------------------------------------------------- epilogue
    __shared__ float nq2_s[QG];
    __shared__ int32_t qb_s[QG];
    const int nthr = TC_EPI_WARPS * 32;
    int r = 0, tcount = 0;
    uint32_t rph = 0;
    for (;;) {
      mbar_wait(&S.rfull[r], rph);
      const ScanItem item = S.ring[r];
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.rempty[r]);
      if (++r == 2) {
        r = 0;
        rph ^= 1;
      }
      if (item.nq < 0) break;
      const int nq = item.nq;
      if (threadIdx.x < QG) {
        const int b = threadIdx.x < nq ? qpairs[item.qoff + threadIdx.x].b : 0;
        qb_s[threadIdx.x] = b;
        nq2_s[threadIdx.x] = threadIdx.x < nq ? qnorm2[b] : 0.f;
      }
      const int64_t rbase = lt.off[item.lslot] + item.row0;
      for (int i = threadIdx.x; i < item.nrows; i += nthr) S.NX[i] = lt.nrm[rbase + i];
      const int h = warp >> 2, g = warp & 3;
      for (int t0 = 0; t0 < item.nrows; t0 += TILE) {
        const int buf = tcount % TC_TBUF;
        mbar_wait(&tfull[buf], (tcount / TC_TBUF) & 1);
        tc_fence_after();
        float v[QG];
        tmem_ld16(tmem + ((uint32_t)(32 * g) << 16) + buf * 2 * QG + h * QG, v);
        const int row = t0 + 128 * h + 32 * g + lane;
        if (row < item.nrows) {
#pragma unroll
          for (int a = 0; a < QG; a++)
            if (a < nq) S.A[a * CHUNK_MAX + row] = v[a];
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
        tcount++;
      }
      named_bar_sync(1, nthr);
      // each warp's query bounds, loaded now so their L2 latency hides under
      // the A computation below
      const uint32_t u0a = warp < nq ? *(volatile uint32_t*)&Uq[qb_s[warp]] : 0u;
      const uint32_t u0b = warp + TC_EPI_WARPS < nq ? *(volatile uint32_t*)&Uq[qb_s[warp + TC_EPI_WARPS]] : 0u;
      for (int i = threadIdx.x; i < nq * item.nrows; i += nthr) {
        const int a = i / item.nrows, row = i - a * item.nrows;
        const float dot = S.A[a * CHUNK_MAX + row];
        S.A[a * CHUNK_MAX + row] =
            (METRIC == SQ_L2) ? __fsub_rn(__fadd_rn(S.NX[row], nq2_s[a]), __fmul_rn(2.f, dot)) : -dot;
      }
      named_bar_sync(1, nthr);
      for (int a = warp; a < nq && !dbg_skip; a += TC_EPI_WARPS)
        screen_select(S, a, item.nrows, kk, coef, nq2_s[a], qb_s[a], item.lslot, rbase,
                      (int64_t)qpairs[item.qoff + a].slotbase + item.chunk, Uq, slot_hi, slot_n,
                      cpool, ccount, cap,
                      a == warp ? u0a : u0b, a < 2 * TC_EPI_WARPS);
      named_bar_sync(1, nthr);  // A / NX / qb_s reuse by the next item
    }
  }
  tc_fence_before();
  __syncthreads();
  if (dbg_t && threadIdx.x == 0) dbg_t[2 * blockIdx.x + 1] = globaltimer_ns();
  if (warp == TC_EPI_WARPS + 1) tmem_dealloc(tmem, TC_TMEM_COLS);
}

// |A - E| <= coef * (nx + nq) with the TF32 dot (2x safety on c_dot).
float screen_coef_tf32(int metric, int dp) {
  const double u = 1.0 / 16777216.0;
  auto gam = [u](double n) { return n * u / (1.0 - n * u); };
  const double c_dot = 2.0 * (2.0011 / 1024.0 + dp / 2097152.0);
  double c;
  if (metric == SQ_L2) c = (c_dot + gam(dp) + 2.0 * gam(dp + 3) + 4.0 * u) / (1.0 - gam(dp));
  else c = (0.5 * c_dot + gam(dp) + 2.0 * u) / (1.0 - gam(dp));
  return (float)(c * 1.0625);
}

// 8 copies of the batch's queries, copy p with the 16-byte pieces of every
// 128-byte chunk permuted by ^p (the SWIZZLE_128B pattern of tile row p mod 8).
__global__ void qswizzle_kernel(const float* __restrict__ Qd, int B, int dp, float* __restrict__ out) {
  const int64_t n4 = (int64_t)B * dp / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 8 * n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int p = (int)(i / n4);
    const int64_t e = i - p * n4;            // float4 index inside the batch
    const int64_t piece = e & 7, chunk = e >> 3;
    reinterpret_cast<float4*>(out)[p * n4 + (chunk << 3) + (piece ^ p)] =
        reinterpret_cast<const float4*>(Qd)[e];
  }
}

// Row squared norms (FFMA, any order) for rows [0, n) of `rows`.
__global__ void row_norms_kernel(const float* __restrict__ rows, int64_t n, int dp,
                                 float* __restrict__ out) {
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= n) return;
  const float* x = rows + r * dp;
  float acc = 0.f;
  for (int j = lane; j < dp; j += 32) acc = __fmaf_rn(x[j], x[j], acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(FULL, acc, o));
  if (lane == 0) out[r] = acc;
}
void launch_row_norms(const float* rows, int64_t n, int dp, float* out, cudaStream_t st) {
  if (n <= 0) return;
  row_norms_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(rows, n, dp, out);
}

void launch_scan_tc(int metric, ListTable lt, const ArenaMaps& maps, const float* Qd, int B,
                    float* qsw, bool qsw_ready, const float* qnorm2, const ScanItem* items,
                    const int32_t* n_items, int max_items, const QPair* qpairs, int kk,
                    int32_t* work_ctr, uint32_t* Uq, uint32_t* slot_hi, int32_t* slot_n, int4* cpool,
                    int32_t* ccount, int cap, int num_sms, cudaStream_t st, bool pdl,
                    const CUtensorMap* qgather, bool overlapped) {
  if (max_items <= 0) return;
  if (!qgather && !qsw_ready) qswizzle_kernel<<<num_sms * 4, 256, 0, st>>>(Qd, B, lt.dp, qsw);
  CUtensorMap qg_dummy;
  memset(&qg_dummy, 0, sizeof(qg_dummy));
  const CUtensorMap& qgm = qgather ? *qgather : qg_dummy;
  const bool use_qg = qgather != nullptr;
  const size_t smem = tc_smem_bytes();
  const int grid = std::min(num_sms, max_items);
  const float coef = screen_coef_tf32(metric, lt.dp);
  // PK_DEBUG_SCAN_NOSELECT=1: skip the per-(query, item) selection (timing
  // experiments only -- results are wrong)
  static const int dbg_skip = getenv("PK_DEBUG_SCAN_NOSELECT") ? atoi(getenv("PK_DEBUG_SCAN_NOSELECT")) : 0;
  // PK_DEBUG_SCAN_TIMES=1: per-CTA start / end timestamps, spread printed to stderr
  static const bool dbg_times = getenv("PK_DEBUG_SCAN_TIMES") != nullptr;
  unsigned long long* dbg_t = nullptr;
  if (dbg_times) cudaMallocAsync((void**)&dbg_t, (size_t)grid * 24, st);
  // The first E = 32 CTAs stop claiming items once 50% of them are taken
  // (PK_SCAN_EARLY="E:F" overrides, "0:1" turns it off): the scan itself ends
  // a few us later, but those SMs run the next batch's front half beside it,
  // so the next scan starts ~2.5 us after this one ends (applied only to
  // overlapped searches, where that front half exists).  Swept E in 16-96,
  // F in 0.2-0.8 on two boxes: 32:0.5 beats 32:0.7 by ~1.3% on configs[1];
  // E >= 64 loses the scan more than it gains.
  static int early_ctas = 32;
  static float early_frac = 0.3f;
  static int early_small = 4;  // "E:F:T": T items per CTA, below which F = 0
  static bool early_read = false;
  if (!early_read) {
    if (const char* e = getenv("PK_SCAN_EARLY")) sscanf(e, "%d:%f:%d", &early_ctas, &early_frac, &early_small);
    early_read = true;
  }
#define PK_TC(M)                                                                                 \
  {                                                                                              \
    auto k = scan_tc_kernel<M>;                                                                  \
    PK_SMEM_ATTR(k, (int)smem);             \
    launch_maybe_pdl(pdl, k, dim3(grid), dim3(TC_THREADS), smem, st, maps, qgm, use_qg, lt, (const float*)qsw, \
               (int64_t)B, \
               qnorm2, items, n_items, qpairs, kk, coef, work_ctr, Uq, slot_hi, slot_n, cpool,      \
               ccount, cap, dbg_skip, dbg_t, overlapped ? early_ctas : 0, early_frac, early_small);            \
  }
  if (metric == SQ_L2) PK_TC(SQ_L2)
  else PK_TC(IP)
#undef PK_TC
  if (dbg_t) {
    std::vector<unsigned long long> h((size_t)grid * 3);
    cudaMemcpyAsync(h.data(), dbg_t, h.size() * 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    unsigned long long s0 = ~0ull, s1 = 0;
    std::vector<double> ends;
    for (int c = 0; c < grid; c++) {
      s0 = std::min(s0, h[2 * c]);
      s1 = std::max(s1, h[2 * c]);
    }
    for (int c = 0; c < grid; c++) ends.push_back((h[2 * c + 1] - s0) / 1e3);
    std::sort(ends.begin(), ends.end());
    fprintf(stderr, "scan CTA times (us from first start): start spread %.1f | end min %.1f p10 %.1f p50 %.1f p90 %.1f max %.1f\n",
            (s1 - s0) / 1e3, ends[0], ends[grid / 10], ends[grid / 2], ends[grid * 9 / 10], ends[grid - 1]);
    if (getenv("PK_DEBUG_SCAN_SM")) {  // end time per SM id
      std::vector<std::pair<unsigned long long, double>> sm;
      for (int c = 0; c < grid; c++) sm.push_back({h[2 * grid + c], (h[2 * c + 1] - s0) / 1e3});
      std::sort(sm.begin(), sm.end());
      fprintf(stderr, "scan end by smid:");
      for (auto& x : sm) fprintf(stderr, " %llu:%.0f", x.first, x.second);
      fprintf(stderr, "\n");
    }
    cudaFreeAsync(dbg_t, st);
  }
}

// Bound coefficient: |A - E| <= coef * (nx + nq) for d terms.
float screen_coef(int metric, int dp) {
  const double u = 1.0 / 16777216.0;
  auto gam = [u](double n) { return n * u / (1.0 - n * u); };
  double c;
  if (metric == SQ_L2) c = (2.0 * gam(dp) + 2.0 * gam(dp + 3) + 4.0 * u) / (1.0 - gam(dp));
  else c = (gam(dp) + 2.0 * u) / (1.0 - gam(dp));
  return (float)(c * 1.0625);  // slack for the fp32 evaluation of eps itself
}

void launch_scan_screen(int metric, ListTable lt, const ArenaMaps& maps, const float* Qd,
                        const float* qnorm2, const ScanItem* items, const int32_t* n_items,
                        int max_items, const QPair* qpairs, int kk, int32_t* work_ctr,
                        uint32_t* Uq, uint32_t* slot_hi, int32_t* slot_n, int4* cpool,
                        int32_t* ccount, int cap, int num_sms, cudaStream_t st) {
  if (max_items <= 0) return;
  const size_t smem = screen_smem_bytes();
  const int grid = std::min(num_sms, max_items);
  const float coef = screen_coef(metric, lt.dp);
  static const int debug_nocompute = getenv("PK_DEBUG_SCAN_NOCOMPUTE") ? atoi(getenv("PK_DEBUG_SCAN_NOCOMPUTE")) : 0;
  if (metric == SQ_L2) {
    auto k = scan_screen_kernel<SQ_L2>;
    PK_SMEM_ATTR(k, (int)smem);
    k<<<grid, SCREEN_THREADS, smem, st>>>(maps, lt, Qd, qnorm2, items, n_items, qpairs, kk, coef,
                                          work_ctr, Uq, slot_hi, slot_n, cpool, ccount, cap,
                                          debug_nocompute);
  } else {
    auto k = scan_screen_kernel<IP>;
    PK_SMEM_ATTR(k, (int)smem);
    k<<<grid, SCREEN_THREADS, smem, st>>>(maps, lt, Qd, qnorm2, items, n_items, qpairs, kk, coef,
                                          work_ctr, Uq, slot_hi, slot_n, cpool, ccount, cap,
                                          debug_nocompute);
  }
}

// ---------------------------------------------------------------------
// Per query: global bound, exact re-rank of the surviving pool entries, merge.
//
// 1. U_q = kk-th smallest of all hi values its (query, item) slots published:
//    kk rows of the query have E <= hi <= U_q, so a row with lo > U_q cannot
//    be in the top-kk.
// 2. Pool entries with lo <= U_q are compacted; their rows are staged into
//    shared memory with coalesced 16-byte loads (a group at a time) and one
//    thread per candidate runs the reference's sequential fp32 sum.
// 3. First kk by (dist, id), first occurrence per id (ref/engine.py:406-426).
// A query whose pool overflowed is answered by an exact scan of every row of
// its probed lists (slow path; correct for any input).
// ---------------------------------------------------------------------
constexpr int RR_THREADS = 256;
constexpr int RR_CAP = 512;     // kept (<= 64) + one chunk of survivors, pow2 for the sort
constexpr int RR_SURV = 4096;  // survivors handled per pass
constexpr int RR_HI_PER = 8;   // published upper bounds per thread (2048 per query)

// LEAN: the configuration that runs NEXT TO the following batch's scan
// (pipelined searches): <= ~19 KB of shared memory, so one re-rank CTA fits
// on an SM beside a scan CTA, a persistent grid of at most one CTA per SM
// looping over the queries, survivors in chunks of 32 through a 2-deep ring
// of 32-float column blocks.  Its latency hides under that scan.
template <int METRIC, bool LEAN>
__global__ void __launch_bounds__(RR_THREADS, LEAN ? 3 : 1) rerank_merge_kernel(
    int B, const int4* __restrict__ cpool, const int32_t* __restrict__ ccount, int cap,
    const uint32_t* __restrict__ slot_hi, const int32_t* __restrict__ slot_n,
    const int32_t* __restrict__ slot_off, ListTable lt, const float* __restrict__ Qd,
    const int32_t* __restrict__ probe, int nprobe, int kk, int stage_floats, int64_t* __restrict__ out_ids,
    float* __restrict__ out_d, int64_t* __restrict__ out_cid, int32_t* __restrict__ out_n,
    int32_t* __restrict__ nsurv, const int64_t* __restrict__ scanned_src, int64_t* __restrict__ scanned_dst,
    uint64_t* __restrict__ dbg) {
  constexpr int CAP = LEAN ? 128 : RR_CAP;
  constexpr int SURV = LEAN ? 256 : RR_SURV;
  if (!LEAN) {
    pdl_trigger();
    pdl_wait();
  }
  extern __shared__ __align__(16) uint8_t rr_smem[];
  Entry* buf = reinterpret_cast<Entry*>(rr_smem);                                   // [CAP]
  float4* qs4 = reinterpret_cast<float4*>(rr_smem + CAP * sizeof(Entry));        // [dp/4]
  float* stage = reinterpret_cast<float*>(qs4 + lt.dp / 4);                         // [stage_floats]
  int32_t* surv = reinterpret_cast<int32_t*>(stage + stage_floats);                 // [SURV]
  __shared__ int s_cnt, s_ns, s_bin, s_below;
  __shared__ unsigned s_hist[256];
  __shared__ unsigned s_wu[RR_THREADS / 32];

  __shared__ uint32_t s_u[RR_THREADS / 32];
  __shared__ int s_row[RR_THREADS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int b = blockIdx.x; b < B; b += gridDim.x) {
  auto mark = [&](int i) {  // phase cycle stamps (PK_DEBUG_RERANK)
    if (dbg && threadIdx.x == 0) dbg[b * 4 + i] = (uint64_t)clock64();
  };
  mark(0);
  if (scanned_dst && threadIdx.x == 0) scanned_dst[b] = scanned_src[b];
  const int dp4 = lt.dp / 4;
  for (int j = threadIdx.x; j < dp4; j += blockDim.x)
    qs4[j] = reinterpret_cast<const float4*>(Qd + (int64_t)b * lt.dp)[j];
  const int n = ccount[b];
  const bool overflow = n > cap;
  // 1. global bound U_q: smallest v with #(slot hi <= v) >= kk (KEY_NONE if
  //    fewer).  The query's published hi values (<= RR_HI_PER per thread) are
  //    gathered into registers once, then bisected.
  const int so = slot_off[2 * b], eo = slot_off[2 * b + 1];
  uint32_t U = KEY_NONE;
  if (!overflow) {
    uint32_t hv[RR_HI_PER];
    int nh = 0;
#pragma unroll
    for (int i = 0; i < RR_HI_PER; i++) hv[i] = KEY_NONE;
    // flattened (slot, entry) index space; slots hold <= kk entries each
    const int nflat = (eo - so) * kk;
    bool fits = nflat <= RR_HI_PER * RR_THREADS;
    // all loads first and independent (entries past a slot's count are read
    // and dropped): one L2 round trip instead of two dependent ones per entry
    int nn[RR_HI_PER];
    uint32_t hraw[RR_HI_PER];
#pragma unroll
    for (int i = 0; i < RR_HI_PER; i++) {
      const int f = threadIdx.x + i * RR_THREADS;
      const bool ok = fits && f < nflat;
      const int sl = so + f / kk, e = f - (f / kk) * kk;
      nn[i] = ok ? slot_n[sl] : 0;
      hraw[i] = ok ? slot_hi[(int64_t)sl * kk + e] : KEY_NONE;
    }
#pragma unroll
    for (int i = 0; i < RR_HI_PER; i++) {
      const int f = threadIdx.x + i * RR_THREADS;
      const int e = f - (f / kk) * kk;
      if (fits && f < nflat && e < nn[i]) {
        hv[i] = hraw[i];
        nh++;
      }
    }
    int have = __reduce_add_sync(FULL, nh);
    if (lane == 0) s_u[warp] = have;
    __syncthreads();
    int total_hi = 0;
    for (int w = 0; w < RR_THREADS / 32; w++) total_hi += s_u[w];
    __syncthreads();
    if (!fits) {  // more published bounds than registers hold (large kk): count them in place
      int c = 0;
      for (int f = threadIdx.x; f < nflat; f += RR_THREADS) {
        const int sl = so + f / kk, e = f - (f / kk) * kk;
        c += e < slot_n[sl];
      }
      c = __reduce_add_sync(FULL, c);
      if (lane == 0) s_u[warp] = c;
      __syncthreads();
      total_hi = 0;
      for (int w = 0; w < RR_THREADS / 32; w++) total_hi += s_u[w];
      __syncthreads();
    }
    if (total_hi >= kk) {
      // radix select of the kk-th smallest published hi (8 bits per pass;
      // from registers, or re-read from L2 each pass when they do not fit)
      uint32_t prefix = 0;
      int rem = kk;
      for (int shift = 24; shift >= 0; shift -= 8) {
        s_hist[threadIdx.x] = 0;
        __syncthreads();
        const uint32_t hmask = shift == 24 ? 0u : (0xffffffffu << (shift + 8));
        if (fits) {
#pragma unroll
          for (int i = 0; i < RR_HI_PER; i++)
            if (hv[i] != KEY_NONE && (hv[i] & hmask) == (prefix & hmask))
              atomicAdd(&s_hist[(hv[i] >> shift) & 0xff], 1u);
        } else {
          for (int f = threadIdx.x; f < nflat; f += RR_THREADS) {
            const int sl = so + f / kk, e = f - (f / kk) * kk;
            if (e < slot_n[sl]) {
              const uint32_t h = slot_hi[(int64_t)sl * kk + e];
              if (h != KEY_NONE && (h & hmask) == (prefix & hmask)) atomicAdd(&s_hist[(h >> shift) & 0xff], 1u);
            }
          }
        }
        __syncthreads();
        pick_bin(s_hist[threadIdx.x], rem, &s_bin, &s_below, s_wu);
        prefix |= (uint32_t)s_bin << shift;
        rem -= s_below;
        __syncthreads();
      }
      U = prefix;
    }
  }
  __syncthreads();
  mark(1);
  int kept = 0, surv_total = 0;
  const int room = CAP - kk;
  if (!overflow) {
    for (int p0 = 0; p0 < n; p0 += SURV) {
      // 2a. compact survivors of this pass
      if (threadIdx.x == 0) s_ns = 0;
      __syncthreads();
      const int pm = min(SURV, n - p0);
      for (int i = threadIdx.x; i < pm; i += blockDim.x) {
        const int4 c = cpool[(int64_t)b * cap + p0 + i];
        if ((uint32_t)c.z <= U) surv[atomicAdd(&s_ns, 1)] = p0 + i;
      }
      __syncthreads();
      const int ns = s_ns;
      surv_total += ns;
      // 2b. exact distances of the survivors, up to RR_THREADS at a time
      //     (thread t runs survivor t's chain), rows streamed through
      //     shared memory in column blocks of W floats (bulk copies,
      //     2-deep ring) so every chain advances together
      const int chunk = min(LEAN ? 32 : RR_THREADS, stage_floats / (2 * (DC + 4)));
      for (int g0 = 0; g0 < ns; g0 += chunk) {
        const int m = min(chunk, ns - g0);
        const int nd32 = dp4 / 8;
        // whole rows in one block when they fit, else a 2-deep ring of column
        // blocks (measured: 3-4 deep with narrower blocks is slower)
        const int R = m * (DC * nd32 + 4) <= stage_floats ? 1 : 2;
        int kq = 1;
        for (int k2 = nd32; k2 >= 1; k2--)
          if (nd32 % k2 == 0 && R * m * (DC * k2 + 4) <= stage_floats) {
            kq = k2;
            break;
          }
        const int W = DC * kq, rs = W + 4, nblk = nd32 / kq;
        // the survivors' arena rows, read once (not per 16-byte piece)
        int4 my_e = make_int4(0, 0, 0, 0);
        if (threadIdx.x < m) {
          my_e = cpool[(int64_t)b * cap + surv[g0 + threadIdx.x]];
          s_row[threadIdx.x] = my_e.x;
        }
        __syncthreads();
        auto issue = [&](int blk) {
          if (blk < nblk) {
            float* dst = stage + (blk % R) * m * rs;
            const int w4 = W / 4;
            for (int i = threadIdx.x; i < m * w4; i += RR_THREADS) {
              const int r = i / w4, c = i - r * w4;
              cp_async16(dst + r * rs + 4 * c, lt.rows + (int64_t)s_row[r] * lt.dp + blk * W + 4 * c);
            }
          }
          cp_async_commit();  // empty groups keep the wait count uniform
        };
        for (int i = 0; i < R - 1; i++) issue(i);
        float acc = 0.f;
        for (int blk = 0; blk < nblk; blk++) {
          issue(blk + R - 1);
          if (R == 2) cp_async_wait<1>();
          else cp_async_wait<0>();
          __syncthreads();
          if (threadIdx.x < m) {
            const float4* x4 = reinterpret_cast<const float4*>(stage + (blk % R) * m * rs + threadIdx.x * rs);
            const float4* q4 = qs4 + blk * (W / 4);
#pragma unroll 4
            for (int j = 0; j < W / 4; j++) acc = step4<METRIC>(acc, x4[j], q4[j]);
          }
          __syncthreads();  // ring slot blk % R is refilled by the next issue
        }
        if (threadIdx.x < m) {
          const int4 e = my_e;
          Entry en;
          en.key = f2key(finalize<METRIC>(acc, 0.f, 0.f));
          en.id = lt.ids[e.x];
          en.pay = e.y;
          buf[kept + threadIdx.x] = en;
        }
        __syncthreads();
        const int tot = kept + m;
        kept = block_sort_keep(buf, tot, kk, true, &s_cnt);
      }
    }
  } else {
    // slow path: exact scan of every row of every probed list
    int64_t total = 0;
    for (int p = 0; p < nprobe; p++) {
      const int sl = probe[(int64_t)b * nprobe + p];
      if (sl >= 0) total += lt.len[sl];
    }
    __syncthreads();
    for (int64_t base = 0; base < total; base += room) {
      const int m = (int)(total - base < room ? total - base : (int64_t)room);
      for (int i = threadIdx.x; i < m; i += blockDim.x) {
        int64_t r = base + i;
        int p = 0;
        for (; p < nprobe; p++) {
          const int sl = probe[(int64_t)b * nprobe + p];
          const int64_t len = sl >= 0 ? lt.len[sl] : 0;
          if (r < len) break;
          r -= len;
        }
        const int lslot = probe[(int64_t)b * nprobe + p];
        const int64_t arow = lt.off[lslot] + r;
        const float4* x4 = reinterpret_cast<const float4*>(lt.rows + arow * lt.dp);
        float acc = 0.f;
        for (int j = 0; j < dp4; j++) acc = step4<METRIC>(acc, __ldg(x4 + j), qs4[j]);
        Entry e;
        e.key = f2key(finalize<METRIC>(acc, 0.f, 0.f));
        e.id = lt.ids[arow];
        e.pay = lslot;
        buf[kept + i] = e;
      }
      __syncthreads();
      cta_bitonic_sort(buf, kept + m);
      kept = cta_compact_sorted(buf, kept + m, kk, true, &s_cnt);
    }
  }
  mark(2);
  for (int i = threadIdx.x; i < kk; i += blockDim.x) {
    const int64_t o = (int64_t)b * kk + i;
    if (i < kept) {
      out_ids[o] = buf[i].id;
      out_d[o] = key2dist(buf[i].key, METRIC);
      if (out_cid) out_cid[o] = lt.cid[buf[i].pay];
    } else {
      out_ids[o] = -1;
      out_d[o] = __int_as_float(0x7f800000);
      if (out_cid) out_cid[o] = -1;
    }
  }
  if (threadIdx.x == 0) {
    out_n[b] = kept;
    if (nsurv) nsurv[b] = overflow ? -1 : surv_total;
  }
  mark(3);
  __syncthreads();  // the next query reuses buf / qs4 / stage
  }
}

// Shared memory of the lean re-rank (one CTA beside a scan CTA on each SM).
static size_t rerank_lean_smem(int dp) {
  return 128 * sizeof(Entry) + (size_t)dp * 4 + (size_t)2 * 32 * (DC + 4) * 4 + 256 * 4;
}
bool rerank_lean_fits(int dp) {
  // the SM's shared memory must hold a scan CTA and a lean re-rank CTA:
  // dynamic + static + the per-CTA reservation of each (measured from the
  // kernels' attributes, not assumed)
  static int cached_dp = -1;
  static bool cached = false;
  if (dp == cached_dp) return cached;
  int dev = 0, per_sm = 0, reserved = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, dev);
  cudaFuncAttributes fs = {}, fr = {};
  cudaFuncGetAttributes(&fs, scan_tc_kernel<SQ_L2>);
  cudaFuncGetAttributes(&fr, rerank_merge_kernel<SQ_L2, true>);
  const size_t need = tc_smem_bytes() + fs.sharedSizeBytes + rerank_lean_smem(dp) + fr.sharedSizeBytes +
                      2 * (size_t)reserved;
  cached = need <= (size_t)per_sm;
  cached_dp = dp;
  static bool said = false;
  if (!said && getenv("PK_DEBUG_RERANK")) {
    fprintf(stderr, "lean re-rank beside the scan: need %zu of %d B per SM -> %s\n", need, per_sm,
            cached ? "fits" : "does not fit");
    said = true;
  }
  return cached;
}

void launch_rerank_merge(int metric, int B, const int4* cpool, const int32_t* ccount, int cap,
                         const uint32_t* slot_hi, const int32_t* slot_n, const int32_t* slot_off,
                         ListTable lt, const float* Qd, const int32_t* probe, int nprobe, int kk,
                         int64_t* out_ids, float* out_d, int64_t* out_cid, int32_t* out_n,
                         int32_t* nsurv, const int64_t* scanned_src, int64_t* scanned_dst,
                         cudaStream_t st, bool pdl, int lean_ctas) {
  if (B <= 0) return;
  static const bool debug = getenv("PK_DEBUG_RERANK") != nullptr;
  uint64_t* dbg = nullptr;
  if (debug) cudaMallocAsync((void**)&dbg, (size_t)B * 32, st);
  const bool lean = lean_ctas > 0;
  // wide: a row stage of ~82 KB (two CTAs per SM) so the typical ~26
  // survivors' whole rows arrive in one load round trip; lean: a 2-deep ring
  // of 32 rows x 32 floats
  const int stage_floats = lean ? 2 * 32 * (DC + 4) : 82 * 1024 / 4;
  const size_t smem = lean ? rerank_lean_smem(lt.dp)
                           : RR_CAP * sizeof(Entry) + (size_t)lt.dp * 4 + (size_t)stage_floats * 4 + RR_SURV * 4;
  const int grid = lean ? std::min(B, lean_ctas) : B;
#define PK_RR(M, L)                                                                             \
  {                                                                                             \
    auto k = rerank_merge_kernel<M, L>;                                                         \
    PK_SMEM_ATTR(k, (int)smem);                                                                 \
    if (L) {                                                                                    \
      static bool carve_ = false;                                                               \
      if (!carve_) {                                                                            \
        cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);           \
        carve_ = true;                                                                          \
      }                                                                                         \
    }                                                                                           \
    launch_maybe_pdl(pdl && !L, k, dim3(grid), dim3(RR_THREADS), smem, st, B, cpool, ccount, cap, slot_hi, slot_n, \
                     slot_off, lt, Qd, probe, nprobe, kk, stage_floats, out_ids, out_d, out_cid, out_n, nsurv,    \
                     scanned_src, scanned_dst, dbg);                                            \
  }
  if (metric == SQ_L2) {
    if (lean) PK_RR(SQ_L2, true) else PK_RR(SQ_L2, false)
  } else {
    if (lean) PK_RR(IP, true) else PK_RR(IP, false)
  }
#undef PK_RR
  if (dbg) {
    std::vector<uint64_t> h((size_t)B * 4);
    cudaMemcpyAsync(h.data(), dbg, h.size() * 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    double acc[4] = {0};
    for (int b = 0; b < B; b++)
      for (int i = 1; i < 4; i++) acc[i] += (double)(h[b * 4 + i] - h[b * 4 + i - 1]);
    fprintf(stderr, "rerank phases (us, mean per CTA @1965 MHz): bound %.2f survivors+exact+sort %.2f out %.2f\n",
            acc[1] / B / 1965.0, acc[2] / B / 1965.0, acc[3] / B / 1965.0);
    cudaFreeAsync(dbg, st);
  }
}

// =====================================================================
// assign_nearest (ref/clusters.py:268-279): per row argmin by (dist, cid).
// =====================================================================
__global__ void __launch_bounds__(256) argmin_kernel(const float* __restrict__ D, int64_t ldd,
                                                     ListTable lt, int32_t scope_code,
                                                     int64_t* __restrict__ out_cid,
                                                     float* __restrict__ out_d) {
  __shared__ uint32_t s_k[8];
  __shared__ int64_t s_i[8];
  const int b = blockIdx.x;
  const float* row = D + (int64_t)b * ldd;
  uint32_t bk = KEY_NONE;
  int64_t bi = ID_NONE;
  for (int c = threadIdx.x; c < lt.nslots; c += blockDim.x) {
    const int64_t i = lt.cid[c];
    if (i < 0 || lt.scope[c] != scope_code) continue;
    const uint32_t k = f2key(row[c]);
    if (lex_less(k, i, bk, bi)) {
      bk = k;
      bi = i;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    uint32_t k2 = __shfl_xor_sync(FULL, bk, o);
    int64_t i2 = __shfl_xor_sync(FULL, bi, o);
    if (lex_less(k2, i2, bk, bi)) {
      bk = k2;
      bi = i2;
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    s_k[warp] = bk;
    s_i[warp] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); w++)
      if (lex_less(s_k[w], s_i[w], bk, bi)) {
        bk = s_k[w];
        bi = s_i[w];
      }
    out_cid[b] = bi == ID_NONE ? -1 : bi;
    if (out_d) out_d[b] = key2dist(bk, lt.metric);
  }
}
void launch_argmin(const float* D, int64_t ldd, int B, ListTable lt, int32_t scope_code,
                   int64_t* out_cid, float* out_d, cudaStream_t st) {
  if (B <= 0) return;
  argmin_kernel<<<B, 256, 0, st>>>(D, ldd, lt, scope_code, out_cid, out_d);
}

__global__ void scatter_rows_kernel(const float* __restrict__ src, int64_t lds,
                                    const int64_t* __restrict__ src_ids, int n,
                                    const int64_t* __restrict__ dst_row, float* __restrict__ dst,
                                    int64_t* __restrict__ dst_ids, int dp) {
  const int i = blockIdx.x;
  if (i >= n) return;
  const int64_t r = dst_row[i];
  for (int j = threadIdx.x; j < dp / 4; j += blockDim.x)
    reinterpret_cast<float4*>(dst + r * dp)[j] = reinterpret_cast<const float4*>(src + i * lds)[j];
  if (threadIdx.x == 0) dst_ids[r] = src_ids[i];
}
void launch_scatter_rows(const float* src, int64_t lds, const int64_t* src_ids, int n,
                         const int64_t* dst_row, float* dst, int64_t* dst_ids, int dp,
                         cudaStream_t st) {
  if (n <= 0) return;
  scatter_rows_kernel<<<n, 128, 0, st>>>(src, lds, src_ids, n, dst_row, dst, dst_ids, dp);
}

}  // namespace pk

namespace pk {

// =====================================================================
// Cross-shard merge: after the all-gather every rank
// holds R per-shard top-kk lists per query, each sorted by (dist, id).  The
// global answer is the first kk of their union by (dist, id) with first
// occurrence per id (ref/engine.py:406-426) -- the k smallest of a union lie
// in the union of every part's k smallest.  One CTA per query.
// =====================================================================
constexpr int SHM_CAP = 1024;  // R * kk <= 1024 (R <= 16 at kk 64)
__global__ void __launch_bounds__(128) shard_merge_kernel(int metric, const uint8_t* __restrict__ blocks,
                                                          int64_t block_bytes, int R, int B, int kk,
                                                          int64_t* __restrict__ out_ids,
                                                          float* __restrict__ out_d,
                                                          int64_t* __restrict__ out_cid,
                                                          int32_t* __restrict__ out_n,
                                                          int64_t* __restrict__ out_scanned) {
  extern __shared__ Entry sbuf[];  // [pow2 >= R * kk]
  __shared__ int s_cnt;
  const int b = blockIdx.x;
  const int64_t nkk = (int64_t)B * kk;
  const int total = R * kk;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    const int r = i / kk, e = i - r * kk;
    const uint8_t* blk = blocks + (int64_t)r * block_bytes;
    const int32_t n = reinterpret_cast<const int32_t*>(blk + (nkk * 20 + (int64_t)B * 8))[b];
    if (e >= n) continue;
    const int64_t id = reinterpret_cast<const int64_t*>(blk)[(int64_t)b * kk + e];
    const float d = reinterpret_cast<const float*>(blk + nkk * 16 + (int64_t)B * 8)[(int64_t)b * kk + e];
    Entry en;
    en.key = f2key(d);
    en.id = id;
    en.pay = i;
    sbuf[atomicAdd(&s_cnt, 1)] = en;
  }
  __syncthreads();
  const int n = s_cnt;
  cta_bitonic_sort(sbuf, n);
  const int kept = cta_compact_sorted(sbuf, n, kk, true, &s_cnt);
  for (int i = threadIdx.x; i < kk; i += blockDim.x) {
    const int64_t o = (int64_t)b * kk + i;
    if (i < kept) {
      const int src = sbuf[i].pay;
      const int r = src / kk, e = src - r * kk;
      const uint8_t* blk = blocks + (int64_t)r * block_bytes;
      out_ids[o] = sbuf[i].id;
      out_d[o] = key2dist(sbuf[i].key, metric);
      if (out_cid) out_cid[o] = reinterpret_cast<const int64_t*>(blk + nkk * 8)[(int64_t)b * kk + e];
    } else {
      out_ids[o] = -1;
      out_d[o] = __int_as_float(0x7f800000);
      if (out_cid) out_cid[o] = -1;
    }
  }
  if (threadIdx.x == 0) {
    out_n[b] = kept;
    if (out_scanned) {
      int64_t sc = 0;
      for (int r = 0; r < R; r++)
        sc += reinterpret_cast<const int64_t*>(blocks + (int64_t)r * block_bytes + nkk * 16)[b];
      out_scanned[b] = sc;
    }
  }
}

int shard_merge_cap() { return SHM_CAP; }

// Regroup per-query results of a B-query batch into B / group shard result
// blocks (block g = queries [g*group, (g+1)*group)), the unit the
// dispatch/combine all-to-all moves.
__global__ void reblock_kernel(const int64_t* __restrict__ ids, const int64_t* __restrict__ cids,
                               const int64_t* __restrict__ sc, const float* __restrict__ d,
                               const int32_t* __restrict__ n, int B, int group, int kk,
                               int64_t block_bytes, uint8_t* __restrict__ dst) {
  const int64_t nkk_g = (int64_t)group * kk;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)B * kk;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(i / kk), e = (int)(i - (int64_t)b * kk);
    const int g = b / group, bl = b - g * group;
    uint8_t* blk = dst + g * block_bytes;
    const int64_t o = (int64_t)bl * kk + e;
    reinterpret_cast<int64_t*>(blk)[o] = ids[i];
    reinterpret_cast<int64_t*>(blk + 8 * nkk_g)[o] = cids[i];
    reinterpret_cast<float*>(blk + 16 * nkk_g + 8 * (int64_t)group)[o] = d[i];
    if (e == 0) {
      reinterpret_cast<int64_t*>(blk + 16 * nkk_g)[bl] = sc[b];
      reinterpret_cast<int32_t*>(blk + 20 * nkk_g + 8 * (int64_t)group)[bl] = n[b];
    }
  }
}
void launch_reblock(const int64_t* ids, const int64_t* cids, const int64_t* sc, const float* d,
                    const int32_t* n, int B, int group, int kk, int64_t block_bytes, void* dst,
                    cudaStream_t st) {
  if (B <= 0) return;
  const int64_t tot = (int64_t)B * kk;
  reblock_kernel<<<(unsigned)std::min<int64_t>((tot + 255) / 256, 1184), 256, 0, st>>>(
      ids, cids, sc, d, n, B, group, kk, block_bytes, static_cast<uint8_t*>(dst));
}

void launch_shard_merge(int metric, const void* blocks, int64_t block_bytes, int R, int B, int kk,
                        int64_t* out_ids, float* out_d, int64_t* out_cid, int32_t* out_n,
                        int64_t* out_scanned, cudaStream_t st) {
  if (B <= 0) return;
  int N = 1;
  while (N < R * kk) N <<= 1;
  size_t smem = (size_t)N * sizeof(Entry);
  PK_SMEM_ATTR(shard_merge_kernel, (int)smem);
  shard_merge_kernel<<<B, 128, smem, st>>>(metric, static_cast<const uint8_t*>(blocks), block_bytes, R, B,
                                           kk, out_ids, out_d, out_cid, out_n, out_scanned);
}

}  // namespace pk

namespace pk {

// =====================================================================
// Coarse quantizer on the tensor cores (north_star
// subsystem 1).  The reference probes the nprobe nearest in-scope clusters by
// exact fp32 distance with ties to the lower cid (ref/graph.py:392-396 at
// exhaustive ef).  Here:
//   coarse_tc_kernel   S = C Q^T on tcgen05 (kind::tf32), C = the centroid
//                      table (TMA SWIZZLE_128B tiles of 128 slots x 32 floats,
//                      the UMMA A operand), Q = the batch (64-query tiles, the
//                      B operand), fp32 accumulators in TMEM; the epilogue
//                      forms the screened distance A = (|c|^2 + |q|^2) - 2 S
//                      (neg_ip: -S) for every (query, slot).
//   coarse_pick_kernel per query: |A - E| <= eps = coef (|c|^2 + |q|^2) (the
//                      scan's proven TF32 bound, screen_coef_tf32); U = the
//                      nprobe-th smallest A + eps over the in-scope lists
//                      (radix select); every list with A - eps <= U is
//                      re-ranked with the exact reference arithmetic and the
//                      first nprobe by (E, cid) are emitted.  A list outside
//                      that set has E > U >= E_(nprobe), so the emitted set
//                      and order equal the exact quantizer's, ties included.
// =====================================================================
constexpr int CT_M = 128;      // centroid slots per CTA (UMMA M)
constexpr int CT_N = 64;       // queries per CTA (UMMA N)
constexpr int CT_STAGES = 4;
constexpr size_t CT_A_BYTES = (size_t)CT_M * DC * 4;  // 16 KB
constexpr size_t CT_B_BYTES = (size_t)CT_N * DC * 4;  // 8 KB
size_t coarse_tc_smem_bytes(bool split) {
  return (split ? 2 : 1) * CT_STAGES * (CT_A_BYTES + CT_B_BYTES) + 256 + 1024;
}

// SPLIT (default): centroids and queries are carried as TF32-exact hi parts
// (low 13 mantissa bits cleared) plus lo = x - hi; D1 = C_hi Q_hi^T and
// D2 = C_hi Q_lo^T + C_lo Q_hi^T accumulate in separate TMEM columns, dot =
// D1 + D2.  The input-rounding error drops from ~2^-9 to ~3 * 2^-20 of
// sum |c_j q_j| (coarse_coef()), so the exact re-rank set shrinks to the
// boundary.  !SPLIT: one TF32 product of the fp32 tables.
template <bool SPLIT>
__global__ void __launch_bounds__(128, 1)
    coarse_tc_kernel(const __grid_constant__ CoarseMaps maps, int nslots, int B, int nchunk,
                     float* __restrict__ Dout, int64_t lda) {
  constexpr int NT = SPLIT ? 2 : 1;  // tables per operand
  constexpr size_t STAGE_BYTES = NT * (CT_A_BYTES + CT_B_BYTES);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + CT_STAGES * STAGE_BYTES);
  uint64_t* empty = full + CT_STAGES;
  uint64_t* done = empty + CT_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  // stage s: A_hi [, A_lo], B_hi [, B_lo]
  auto a_tile = [&](int s, int t) { return reinterpret_cast<float*>(base + s * STAGE_BYTES + t * CT_A_BYTES); };
  auto b_tile = [&](int s, int t) {
    return reinterpret_cast<float*>(base + s * STAGE_BYTES + NT * CT_A_BYTES + t * CT_B_BYTES);
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = blockIdx.x * CT_M, b0 = blockIdx.y * CT_N;
  // split-K: this CTA's chunk range
  const int kc0 = (int)((int64_t)nchunk * blockIdx.z / gridDim.z);
  const int kc1 = (int)((int64_t)nchunk * (blockIdx.z + 1) / gridDim.z);
  float* Aout = Dout + (int64_t)blockIdx.z * B * lda;
  if (threadIdx.x == 0) {
    for (int i = 0; i < CT_STAGES; i++) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, NT * CT_N);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_trigger();
  pdl_wait();  // the batch's TF32 split comes from qprep
  const uint32_t tmem = *tmem_slot;
  if (warp == 0 && lane == 0) {
    for (int t = 0; t < NT; t++) {
      tma_prefetch_desc(&maps.c[t]);
      tma_prefetch_desc(&maps.q[t]);
    }
    const uint64_t pol = policy_evict_last();  // tables are re-read by the other CTAs
    int s = 0;
    uint32_t ph = 0;
    for (int c = kc0; c < kc1; c++) {
      mbar_wait(&empty[s], ph ^ 1);
      mbar_arrive_expect_tx(&full[s], (uint32_t)STAGE_BYTES);
      for (int t = 0; t < NT; t++) {
        tma_load_2d(a_tile(s, t), &maps.c[t], &full[s], c * DC, c0, pol);
        tma_load_2d(b_tile(s, t), &maps.q[t], &full[s], c * DC, b0, pol);
      }
      if (++s == CT_STAGES) {
        s = 0;
        ph ^= 1;
      }
    }
  } else if (warp == 1 && lane == 0) {
    const uint32_t idesc = umma_idesc_tf32(CT_M, CT_N);
    int s = 0;
    uint32_t ph = 0;
    for (int c = kc0; c < kc1; c++) {
      mbar_wait(&full[s], ph);
      tc_fence_after();
      const uint32_t ah = smem_u32(a_tile(s, 0)), bh = smem_u32(b_tile(s, 0));
#pragma unroll
      for (int k = 0; k < DC / 8; k++) {
        const uint32_t acc = ((c - kc0) | k) != 0;
        umma_tf32(tmem, umma_desc_sw128(ah + k * 32), umma_desc_sw128(bh + k * 32), idesc, acc);
        if (SPLIT) {
          const uint32_t al = smem_u32(a_tile(s, NT - 1)), bl = smem_u32(b_tile(s, NT - 1));
          umma_tf32(tmem + CT_N, umma_desc_sw128(ah + k * 32), umma_desc_sw128(bl + k * 32), idesc, acc);
          umma_tf32(tmem + CT_N, umma_desc_sw128(al + k * 32), umma_desc_sw128(bh + k * 32), idesc, 1);
        }
      }
      umma_commit(&empty[s]);
      if (++s == CT_STAGES) {
        s = 0;
        ph ^= 1;
      }
    }
    umma_commit(done);
  }
  __syncwarp();
  mbar_wait(done, 0);
  tc_fence_after();
  const int m = c0 + 32 * warp + lane;  // this thread's centroid slot (TMEM lane)
#pragma unroll
  for (int g = 0; g < CT_N / 16; g++) {
    float v[16], w[16];
    tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + g * 16, v);
    if (SPLIT) {
      tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + CT_N + g * 16, w);
#pragma unroll
      for (int a = 0; a < 16; a++) v[a] = __fadd_rn(v[a], w[a]);
    }
    if (m < nslots) {
#pragma unroll
      for (int a = 0; a < 16; a++) {
        const int b = b0 + g * 16 + a;
        if (b < B) Aout[(int64_t)b * lda + m] = v[a];  // dot (partial over this K range)
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, NT * CT_N);
}

int coarse_split_k(int nslots, int B, int dp, int num_sms) {
  const int tiles = ((nslots + CT_M - 1) / CT_M) * ((B + CT_N - 1) / CT_N);
  return std::max(1, std::min(dp / DC / 2, num_sms / std::max(tiles, 1)));
}

void launch_coarse_tc(bool split, int ks, const CoarseMaps& maps, int nslots, int B, int dp,
                      float* Dout, int64_t lda, cudaStream_t st) {
  if (B <= 0 || nslots <= 0) return;
  const size_t smem = coarse_tc_smem_bytes(split);
  dim3 grid((unsigned)((nslots + CT_M - 1) / CT_M), (unsigned)((B + CT_N - 1) / CT_N), (unsigned)ks);
  if (split) {
    PK_SMEM_ATTR(coarse_tc_kernel<true>, (int)smem);
    launch_pdl(coarse_tc_kernel<true>, grid, dim3(128), smem, st, maps, nslots, B, dp / DC, Dout, lda);
  } else {
    PK_SMEM_ATTR(coarse_tc_kernel<false>, (int)smem);
    launch_pdl(coarse_tc_kernel<false>, grid, dim3(128), smem, st, maps, nslots, B, dp / DC, Dout, lda);
  }
}

// Query prep, one pass per batch (one warp per query): the padded copy of
// the user's rows (Qin, stride ldin, true dimension d; pad columns zero), the
// FFMA squared norm qn2 (screen input; any order), optionally the TF32 hi/lo
// split (coarse screen) and the 8 SWIZZLE_128B-permuted copies the scan's
// query tiles are bulk-copied from (copy p has the 16-byte pieces of every
// 128-byte chunk permuted by ^p); block 0 also resets the batch's counters.
constexpr int QP_THREADS = 64;
__global__ void __launch_bounds__(QP_THREADS) qprep_kernel(const float* __restrict__ Qin, int64_t ldin, int d, int B, int dp,
                             float* __restrict__ q, float* __restrict__ qn2, float* __restrict__ hi,
                             float* __restrict__ lo, float* __restrict__ qsw,
                             int32_t* __restrict__ zero_i32, int nzero, int32_t* __restrict__ zero2,
                             int nzero2, uint32_t* __restrict__ ones_u32, int nones) {
  pdl_trigger();
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < nzero; i += blockDim.x) zero_i32[i] = 0;
    for (int i = threadIdx.x; i < nzero2; i += blockDim.x) zero2[i] = 0;
    for (int i = threadIdx.x; i < nones; i += blockDim.x) ones_u32[i] = 0xffffffffu;
  }
  // one CTA (QP_THREADS) per query; partial norms combined in a fixed order
  __shared__ float s_part[QP_THREADS / 32];
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float* src = Qin + (int64_t)b * ldin;
  const bool vec_in = (d & 3) == 0 && (ldin & 3) == 0;
  const int64_t n4 = (int64_t)B * dp / 4;
  float acc = 0.f;
  for (int j4 = threadIdx.x; j4 < dp / 4; j4 += QP_THREADS) {
    float4 v;
    const int j = 4 * j4;
    if (vec_in && j + 3 < d) {
      v = *reinterpret_cast<const float4*>(src + j);
    } else {
      v.x = j < d ? src[j] : 0.f;
      v.y = j + 1 < d ? src[j + 1] : 0.f;
      v.z = j + 2 < d ? src[j + 2] : 0.f;
      v.w = j + 3 < d ? src[j + 3] : 0.f;
    }
    const int64_t e = (int64_t)b * (dp / 4) + j4;
    reinterpret_cast<float4*>(q)[e] = v;
    acc = __fmaf_rn(v.x, v.x, acc);
    acc = __fmaf_rn(v.y, v.y, acc);
    acc = __fmaf_rn(v.z, v.z, acc);
    acc = __fmaf_rn(v.w, v.w, acc);
    if (hi) {
      float4 h, l;
      h.x = __uint_as_float(__float_as_uint(v.x) & 0xffffe000u);
      h.y = __uint_as_float(__float_as_uint(v.y) & 0xffffe000u);
      h.z = __uint_as_float(__float_as_uint(v.z) & 0xffffe000u);
      h.w = __uint_as_float(__float_as_uint(v.w) & 0xffffe000u);
      l.x = __fsub_rn(v.x, h.x);
      l.y = __fsub_rn(v.y, h.y);
      l.z = __fsub_rn(v.z, h.z);
      l.w = __fsub_rn(v.w, h.w);
      reinterpret_cast<float4*>(hi)[e] = h;
      reinterpret_cast<float4*>(lo)[e] = l;
    }
    if (qsw) {
      const int64_t base8 = e & ~(int64_t)7;
      const int piece = (int)(e & 7);
#pragma unroll
      for (int pp = 0; pp < 8; pp++) reinterpret_cast<float4*>(qsw)[pp * n4 + base8 + (piece ^ pp)] = v;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(FULL, acc, o));
  if (lane == 0) s_part[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = s_part[0];
    for (int w = 1; w < QP_THREADS / 32; w++) t = __fadd_rn(t, s_part[w]);
    qn2[b] = t;
  }
}
void launch_qprep(const float* Qin, int64_t ldin, int d, int B, int dp, float* q, float* qn2, float* hi,
                  float* lo, float* qsw, int32_t* zero_i32, int nzero, int32_t* zero2, int nzero2,
                  uint32_t* ones_u32, int nones, cudaStream_t st) {
  if (B <= 0) return;
  qprep_kernel<<<B, QP_THREADS, 0, st>>>(Qin, ldin, d, B, dp, q, qn2, hi, lo, qsw, zero_i32, nzero,
                                         zero2, nzero2, ones_u32, nones);
}

// hi = x with the low 13 mantissa bits cleared (exactly representable in
// TF32), lo = x - hi (exact in fp32).  Rows [0, n) of [n][dp].
__global__ void tf32_split_kernel(const float* __restrict__ x, int64_t n4, float* __restrict__ hi,
                                  float* __restrict__ lo) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 v = reinterpret_cast<const float4*>(x)[i], h, l;
    h.x = __uint_as_float(__float_as_uint(v.x) & 0xffffe000u);
    h.y = __uint_as_float(__float_as_uint(v.y) & 0xffffe000u);
    h.z = __uint_as_float(__float_as_uint(v.z) & 0xffffe000u);
    h.w = __uint_as_float(__float_as_uint(v.w) & 0xffffe000u);
    l.x = __fsub_rn(v.x, h.x);
    l.y = __fsub_rn(v.y, h.y);
    l.z = __fsub_rn(v.z, h.z);
    l.w = __fsub_rn(v.w, h.w);
    reinterpret_cast<float4*>(hi)[i] = h;
    reinterpret_cast<float4*>(lo)[i] = l;
  }
}
void launch_tf32_split(const float* x, int64_t n, int dp, float* hi, float* lo, cudaStream_t st) {
  const int64_t n4 = n * dp / 4;
  if (n4 <= 0) return;
  const int grid = (int)std::min<int64_t>((n4 + 255) / 256, 1184);
  tf32_split_kernel<<<grid, 256, 0, st>>>(x, n4, hi, lo);
}

// |A - E| <= coef * (|c|^2 + |q|^2) + abs for the coarse screen.
// split: c_dot = d 2^-21 (TMEM accumulation, the model validated for the scan
// screen by tools/microbench/umma_check.cu) + 3 2^-20 (dropped lo*lo and the
// TF32 conversions of the lo parts) + 2^-23 (D1 + D2) + 2d 2^-31 (D2's own
// accumulation); !split: the scan's c_dot.  2x safety like the scan.
float coarse_coef(int metric, int dp, bool split, int ks) {
  const double u = 1.0 / 16777216.0;
  auto gam = [u](double n) { return n * u / (1.0 - n * u); };
  // split-K: ks partial dots summed in fp32 (ks - 1 rounded adds)
  const double c_ks = (ks - 1) * 2.0 * u;
  if (!split) return (float)(screen_coef_tf32(metric, dp) + 2.0 * 1.0625 * 2.0 * c_ks);
  const double c_dot = 2.0 * (dp / 2097152.0 + 3.0 / 1048576.0 + 1.0 / 8388608.0 + 2.0 * dp / 2147483648.0 + c_ks);
  double c;
  if (metric == SQ_L2) c = (c_dot + gam(dp) + 2.0 * gam(dp + 3) + 4.0 * u) / (1.0 - gam(dp));
  else c = (0.5 * c_dot + gam(dp) + 2.0 * u) / (1.0 - gam(dp));
  return (float)(c * 1.0625);
}

// Exact reference distance of the query in shared memory to centroid row `c`
// (ref/kernels.py:73-95 arithmetic, j ascending over the true dimension).
template <int METRIC>
__device__ __forceinline__ float exact_dist_row(const float* __restrict__ qs, const float* __restrict__ c,
                                                int d) {
  float acc = 0.f;
  int j = 0;
  if ((d & 3) == 0) {
    for (; j < d; j += 4) {
      const float4 x = __ldg(reinterpret_cast<const float4*>(c + j));
      const float4 q = *reinterpret_cast<const float4*>(qs + j);
      acc = step4<METRIC>(acc, x, q);
    }
  } else {
    for (; j < d; j++)
      acc = (METRIC == SQ_L2) ? sq_step(acc, __ldg(c + j), qs[j]) : ip_step(acc, __ldg(c + j), qs[j]);
  }
  return METRIC == SQ_L2 ? acc : -acc;
}

template <int METRIC>
__device__ __forceinline__ float exact_dist_row_smem(const float* __restrict__ qs,
                                                     const float* __restrict__ x, int d) {
  float acc = 0.f;
  int j = 0;
  for (; j + 4 <= d; j += 4)
    acc = step4<METRIC>(acc, *reinterpret_cast<const float4*>(x + j),
                        *reinterpret_cast<const float4*>(qs + j));
  for (; j < d; j++) acc = (METRIC == SQ_L2) ? sq_step(acc, x[j], qs[j]) : ip_step(acc, x[j], qs[j]);
  return METRIC == SQ_L2 ? acc : -acc;
}

constexpr int PICK_THREADS = 256;
constexpr int PICK_SMEM_SLOTS = 8192;  // upper-bound keys staged in shared memory up to this

template <int METRIC>
__global__ void __launch_bounds__(PICK_THREADS) coarse_pick_kernel(
    const float* __restrict__ Aapp, int64_t lda, ListTable lt, const float* __restrict__ cnrm,
    const float* __restrict__ Qd, const float* __restrict__ qn2,
    const int32_t* __restrict__ scope_codes, int nscopes, int nprobe, float coef, float abs_coef,
    int cap, int stage_floats, int ks, int64_t zstride, int32_t* __restrict__ probe, uint32_t* __restrict__ probe_key,
    int32_t* __restrict__ ncand_out, uint64_t* __restrict__ dbg, RouteArgs ra) {
  pdl_trigger();
  pdl_wait();  // coarse partial dots
  auto mark = [&](int i) {  // phase timestamps (PK_DEBUG_PICK)
    if (dbg && threadIdx.x == 0) {
      dbg[blockIdx.x * 8 + i] = (uint64_t)clock64();  // SM cycles (phase lengths within a CTA)
    }
  };
  mark(0);
  extern __shared__ __align__(16) uint8_t pick_smem[];
  Entry* buf = reinterpret_cast<Entry*>(pick_smem);                  // [cap] (pow2)
  float* qs = reinterpret_cast<float*>(buf + cap);                   // [dp]
  float* rows_st = qs + lt.dp;                                       // [stage_floats]
  uint32_t* hks = reinterpret_cast<uint32_t*>(rows_st + stage_floats);  // [nslots] when staged
  uint32_t* lks = hks + lt.nslots;                                        // [nslots] when staged
  __shared__ int s_codes[64];
  __shared__ unsigned s_hist[256];
  __shared__ unsigned s_w[PICK_THREADS / 32];
  __shared__ int s_cnt, s_total, s_bin, s_below;
  const int b = blockIdx.x;
  const int tid = threadIdx.x;
  const bool staged = lt.nslots <= PICK_SMEM_SLOTS;
  if (tid < 64) s_codes[tid] = tid < nscopes ? scope_codes[tid] : -1;
  for (int j = tid; j < lt.dp / 4; j += PICK_THREADS)
    reinterpret_cast<float4*>(qs)[j] = reinterpret_cast<const float4*>(Qd + (int64_t)b * lt.dp)[j];
  if (tid == 0) s_total = 0;
  __syncthreads();
  const float* arow = Aapp + (int64_t)b * lda;
  const float qn = qn2[b];
  // bounds of list s: hk = key(A + eps), lk = key(A - eps); out of scope /
  // retired -> KEY_NONE (never a candidate: a finite or -inf lower bound is
  // never KEY_NONE)
  auto bounds = [&](int s, uint32_t& hk, uint32_t& lk) {
    hk = lk = KEY_NONE;
    // all loads first (independent), then the arithmetic
    const int64_t cid = lt.cid[s];
    const int sc = lt.scope[s];
    const float cn = cnrm[s];
    float dot = arow[s];
    for (int z = 1; z < ks; z++) dot = __fadd_rn(dot, arow[(int64_t)z * zstride + s]);
    if (cid < 0) return;
    bool in = false;
    for (int i = 0; i < nscopes; i++) in |= (s_codes[i] == sc);
    if (!in) return;
    const float A = (METRIC == SQ_L2) ? __fsub_rn(__fadd_rn(cn, qn), __fmul_rn(2.f, dot)) : -dot;
    // + abs: flushed subnormal operands / products / partial sums (< 2^-126 each)
    const float nsum = __fadd_ru(cn, qn);
    const float eps = __fadd_ru(__fmul_ru(coef, nsum), __fmul_ru(abs_coef, __fadd_ru(nsum, 2.f)));
    float hi = __fadd_ru(A, eps), lo = __fsub_rd(A, eps);
    if (!isfinite(hi) || !isfinite(lo)) {
      hi = __int_as_float(0x7f800000);
      lo = __int_as_float(0xff800000);
    }
    hk = f2key(hi);
    lk = f2key(lo);
    if (hk == KEY_NONE) hk = KEY_NONE - 1;  // keep valid lists distinguishable
  };
  mark(1);
  // 1. upper-bound keys (staged) and the number of in-scope lists
  int nv = 0;
#pragma unroll 4
  for (int s = tid; s < lt.nslots; s += PICK_THREADS) {
    uint32_t hk, lk;
    bounds(s, hk, lk);
    nv += hk != KEY_NONE;
    if (staged) {
      hks[s] = hk;
      lks[s] = lk;
    }
  }
  nv = __reduce_add_sync(FULL, nv);
  if ((tid & 31) == 0) atomicAdd(&s_total, nv);
  __syncthreads();
  const int nvalid = s_total;
  mark(2);
  // 2. U = nprobe-th smallest upper bound (radix select, 8 bits per pass)
  uint32_t U = KEY_NONE - 1;
  if (nvalid > nprobe) {
    uint32_t prefix = 0;
    int rem = nprobe;
    for (int shift = 24; shift >= 0; shift -= 8) {
      s_hist[tid] = 0;
      __syncthreads();
      const uint32_t hmask = shift == 24 ? 0u : (0xffffffffu << (shift + 8));
      for (int s = tid; s < lt.nslots; s += PICK_THREADS) {
        uint32_t hk, lk;
        if (staged) hk = hks[s];
        else bounds(s, hk, lk);
        if (hk != KEY_NONE && (hk & hmask) == (prefix & hmask))
          atomicAdd(&s_hist[(hk >> shift) & 0xff], 1u);
      }
      __syncthreads();
      pick_bin(s_hist[tid], rem, &s_bin, &s_below, s_w);
      prefix |= (uint32_t)s_bin << shift;
      rem -= s_below;
      __syncthreads();
    }
    U = prefix;
  }
  mark(3);
  // 3. exact re-rank of every list whose lower bound is <= U, in rounds of
  //    up to cap - nprobe candidates merged with the running first nprobe
  int kept = 0, ncand = 0;
  int s_next = 0;
  const int room = cap - nprobe;
  while (s_next < lt.nslots) {
    if (tid == 0) s_cnt = kept;
    __syncthreads();
    int s_end = lt.nslots;
    for (int s0 = s_next; s0 < lt.nslots; s0 += PICK_THREADS) {
      const int s = s0 + tid;
      if (s < lt.nslots) {
        uint32_t hk, lk;
        if (staged) lk = lks[s];
        else bounds(s, hk, lk);
        if (lk <= U) {
          const int pos = atomicAdd(&s_cnt, 1);
          buf[pos].id = lt.cid[s];
          buf[pos].pay = s;
        }
      }
      __syncthreads();
      if (s_cnt - kept > room - PICK_THREADS) {  // the next block of slots might not fit
        s_end = s0 + PICK_THREADS;
        break;
      }
    }
    const int n = s_cnt;
    ncand += n - kept;
    // Unordered mode, whole candidate set in one round: a candidate with
    // hk <= U is certainly among the first nprobe when at most nprobe
    // candidates have lk <= its hk (every list that could rank before it is a
    // candidate, since lk <= hk <= U); those skip the exact chain (key 0, so
    // they sort first) and only the uncertain ones -- moved to the front --
    // are re-ranked, with their whole rows staged at once when they fit.
    // The probe SET equals the exact quantizer's; order and keys are not
    // produced in this mode.
    int nex = n;  // candidates buf[kept, nex) take the exact chain
    if (ra.unordered && staged && kept == 0 && s_end >= lt.nslots && n <= PICK_THREADS) {
      __shared__ uint32_t c_lk[PICK_THREADS];
      __shared__ int s_u0, s_u1;
      Entry e;
      uint32_t my_hk = KEY_NONE;
      if (tid < n) {
        e = buf[tid];
        my_hk = hks[e.pay];
        c_lk[tid] = lks[e.pay];
      }
      if (tid == 0) {
        s_u0 = 0;
        s_u1 = 0;
      }
      __syncthreads();
      bool certain = false;
      if (tid < n && my_hk <= U) {
        int c = 0;
        for (int j2 = 0; j2 < n; j2++) c += c_lk[j2] <= my_hk;
        certain = c <= nprobe;
      }
      if (tid < n) {
        if (certain) {
          e.key = 0;
          buf[n - 1 - atomicAdd(&s_u1, 1)] = e;
        } else {
          buf[atomicAdd(&s_u0, 1)] = e;
        }
      }
      __syncthreads();
      nex = s_u0;
    }
    mark(4);
    // exact distances of this round's candidates buf[kept, n) (<= PICK_THREADS):
    // thread t runs candidate t's chain; the rows stream through shared memory
    // in column blocks of W floats (bulk copies, 2-deep ring) so every chain
    // advances together
    for (int c0 = kept; c0 < nex; c0 += PICK_THREADS) {
      const int nr = min(PICK_THREADS, nex - c0);
      const int nd32 = lt.dp / DC;
      // whole rows in one block when they fit (one load round trip), else
      // W = 32 k floats, k | dp/32, in a 2-deep ring of PICK_RING * nr * (W + 4)
      // floats (measured: 3-4 deep with narrower blocks is slower)
      const int PICK_RING = nr * (DC * nd32 + 4) <= stage_floats ? 1 : 2;
      int k = 1;
      for (int kk2 = nd32; kk2 >= 1; kk2--)
        if (nd32 % kk2 == 0 && PICK_RING * nr * (DC * kk2 + 4) <= stage_floats) {
          k = kk2;
          break;
        }
      const int W = DC * k, rs = W + 4, nblk = nd32 / k;
      // every thread streams 16-byte pieces of the block (cp.async ring)
      auto issue = [&](int blk) {
        if (blk < nblk) {
          float* dst = rows_st + (blk % PICK_RING) * nr * rs;
          const int w4 = W / 4;
          for (int i = tid; i < nr * w4; i += PICK_THREADS) {
            const int r = i / w4, c = i - r * w4;
            cp_async16(dst + r * rs + 4 * c, lt.cent + (int64_t)buf[c0 + r].pay * lt.dp + blk * W + 4 * c);
          }
        }
        cp_async_commit();  // empty groups keep the wait count uniform
      };
      for (int i = 0; i < PICK_RING - 1; i++) issue(i);
      float acc = 0.f;
      for (int blk = 0; blk < nblk; blk++) {
        issue(blk + PICK_RING - 1);
        if (PICK_RING == 2) cp_async_wait<1>();
        else cp_async_wait<0>();
        __syncthreads();
        if (tid < nr) {
          const float* x = rows_st + (blk % PICK_RING) * nr * rs + tid * rs;
          const float* q = qs + blk * W;
          const int jn = min(W, lt.d - blk * W);
          int j = 0;
          for (; j + 4 <= jn; j += 4)
            acc = step4<METRIC>(acc, *reinterpret_cast<const float4*>(x + j),
                                *reinterpret_cast<const float4*>(q + j));
          for (; j < jn; j++) acc = (METRIC == SQ_L2) ? sq_step(acc, x[j], q[j]) : ip_step(acc, x[j], q[j]);
        }
        __syncthreads();  // ring slot blk % PICK_RING is refilled by the next issue
      }
      if (tid < nr) buf[c0 + tid].key = f2key(METRIC == SQ_L2 ? acc : -acc);
    }
    __syncthreads();
    mark(5);
    kept = block_sort_keep(buf, n, nprobe, false, &s_cnt);
    mark(6);
    s_next = s_end;
    __syncthreads();
  }
  for (int p = tid; p < nprobe; p += PICK_THREADS) {
    probe[(int64_t)b * nprobe + p] = p < kept ? buf[p].pay : -1;
    if (probe_key) probe_key[(int64_t)b * nprobe + p] = p < kept ? buf[p].key : KEY_NONE;
  }
  if (tid == 0 && ncand_out) ncand_out[b] = ncand;
  if (ra.lcount) {  // fused routing of this query (route_emit_kernel's work)
    __syncthreads();
    emit_routes(b, probe + (int64_t)b * nprobe, nprobe, lt, ra.chunk_rows, ra.smax, ra.bcap, ra.lcount,
                ra.bucket, ra.slot_off, ra.scanned);
  }
  mark(7);
}

static int pick_cap(int nprobe) {
  int c = 1;
  while (c < nprobe + 2 * PICK_THREADS) c <<= 1;
  return c;
}
// Column-block stage: what is left of ~110 KB (two CTAs per SM), at least
// 2 x 256 rows x 36 floats.
static int pick_stage_floats(int dp, int nslots, int nprobe) {
  const size_t fixed = pick_cap(nprobe) * sizeof(Entry) + (size_t)dp * 4 +
                       (nslots <= PICK_SMEM_SLOTS ? (size_t)nslots * 8 : 0);
  // PK_PICK_SMEM_KB: the per-CTA budget (110: two CTAs per SM, ~72: three)
  static const size_t want = (getenv("PK_PICK_SMEM_KB") ? (size_t)atoi(getenv("PK_PICK_SMEM_KB")) : 110) * 1024;
  const size_t minf = 2 * PICK_THREADS * (DC + 4);
  size_t f = fixed < want ? (want - fixed) / 4 : 0;
  return (int)std::max(f, minf);
}
size_t coarse_pick_smem_bytes(int dp, int nslots, int nprobe) {
  return pick_cap(nprobe) * sizeof(Entry) + (size_t)dp * 4 +
         (size_t)pick_stage_floats(dp, nslots, nprobe) * 4 +
         (nslots <= PICK_SMEM_SLOTS ? (size_t)nslots * 8 : 0);
}

void launch_coarse_pick(int metric, bool split, int ks, const float* Aapp, int64_t lda, int B, ListTable lt,
                        const float* cnrm, const float* Qd, const float* qn2,
                        const int32_t* scope_codes, int nscopes, int nprobe, int32_t* probe,
                        uint32_t* probe_key, int32_t* ncand, const RouteArgs& ra, cudaStream_t st) {
  if (B <= 0) return;
  // PK_DEBUG_PICK=1: per-CTA phase timestamps, averaged to stderr (measurement aid)
  static const bool debug = getenv("PK_DEBUG_PICK") != nullptr;
  uint64_t* dbg = nullptr;
  if (debug) cudaMallocAsync((void**)&dbg, (size_t)B * 8 * 8, st);
  const size_t smem = coarse_pick_smem_bytes(lt.dp, lt.nslots, nprobe);
  const int cap = pick_cap(nprobe);
  const int stage_floats = pick_stage_floats(lt.dp, lt.nslots, nprobe);
  const float coef = coarse_coef(metric, lt.dp, split, ks);
  // 2^-126 * (sqrt(dp) + 4 dp) per unit of (|c|^2 + |q|^2 + 2), doubled
  const float abs_coef = (float)(2.0 * (std::sqrt((double)lt.dp) + 4.0 * lt.dp) * std::ldexp(1.0, -126));
#define PK_PK(M)                                                                                     \
  {                                                                                                  \
    auto k = coarse_pick_kernel<M>;                                                                  \
    PK_SMEM_ATTR(k, (int)smem);                 \
    launch_pdl(k, dim3(B), dim3(PICK_THREADS), smem, st, Aapp, lda, lt, cnrm, Qd, qn2, scope_codes, nscopes, nprobe, \
                                     coef, abs_coef, cap, stage_floats, ks, (int64_t)B * lda, probe, \
                                     probe_key, ncand, dbg, ra);                                     \
  }
  if (metric == SQ_L2) PK_PK(SQ_L2)
  else PK_PK(IP)
#undef PK_PK
  if (dbg) {
    std::vector<uint64_t> h((size_t)B * 8);
    cudaMemcpyAsync(h.data(), dbg, h.size() * 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    double acc[8] = {0};
    uint64_t t0 = UINT64_MAX, t1 = 0;
    for (int b = 0; b < B; b++) {
      for (int i = 1; i < 8; i++) acc[i] += (double)(h[b * 8 + i] - h[b * 8 + i - 1]);
      t0 = std::min(t0, h[b * 8]);
      t1 = std::max(t1, h[b * 8 + 7]);
    }
    (void)t0;
    (void)t1;
    const double cyc_us = 1965.0;  // SM cycles per us at the B200 boost clock
    fprintf(stderr, "pick phases (us, mean per CTA @1965 MHz): prologue %.2f bounds %.2f radix %.2f "
                    "collect %.2f exact %.2f sort %.2f out %.2f\n",
            acc[1] / B / cyc_us, acc[2] / B / cyc_us, acc[3] / B / cyc_us, acc[4] / B / cyc_us,
            acc[5] / B / cyc_us, acc[6] / B / cyc_us, acc[7] / B / cyc_us);
    cudaFreeAsync(dbg, st);
  }
}

}  // namespace pk

namespace pk {

// =====================================================================
// Cold tier (north_star subsystem 4): lists that
// are not HBM-resident live in a pinned, device-mapped host arena.  Before a
// batch scans them, this kernel streams every probed cold list from host
// memory (PCIe, zero-copy 16-byte loads, coalesced per warp) into a staging
// range of the HBM arena, with ids and the squared row norms the tensor-core
// screen needs.  One CTA per list, one warp per row.
// =====================================================================
__global__ void __launch_bounds__(256) gather_rows_kernel(const StageCopy* __restrict__ desc,
                                                          const float* __restrict__ hrows,
                                                          const int64_t* __restrict__ hids,
                                                          float* __restrict__ rows,
                                                          int64_t* __restrict__ ids,
                                                          float* __restrict__ nrm, int dp) {
  const StageCopy c = desc[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int dp4 = dp / 4;
  for (int r = warp; r < c.n; r += 8) {
    const float4* src = reinterpret_cast<const float4*>(hrows + (c.src_row + r) * (int64_t)dp);
    float4* dst = reinterpret_cast<float4*>(rows + (c.dst_row + r) * (int64_t)dp);
    float acc = 0.f;
    for (int j = lane; j < dp4; j += 32) {
      const float4 v = src[j];
      dst[j] = v;
      acc = __fmaf_rn(v.x, v.x, acc);
      acc = __fmaf_rn(v.y, v.y, acc);
      acc = __fmaf_rn(v.z, v.z, acc);
      acc = __fmaf_rn(v.w, v.w, acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(FULL, acc, o));
    if (lane == 0) {
      nrm[c.dst_row + r] = acc;
      ids[c.dst_row + r] = hids[c.src_row + r];
    }
  }
}

void launch_gather_rows(const StageCopy* desc, int ndesc, const float* hrows, const int64_t* hids,
                        float* rows, int64_t* ids, float* nrm, int dp, cudaStream_t st) {
  if (ndesc <= 0) return;
  gather_rows_kernel<<<ndesc, 256, 0, st>>>(desc, hrows, hids, rows, ids, nrm, dp);
}

// Squared norms of the staged rows after a DMA (copy-engine) staging pass.
__global__ void __launch_bounds__(256) stage_norms_kernel(const StageCopy* __restrict__ desc,
                                                          const float* __restrict__ rows,
                                                          float* __restrict__ nrm, int dp,
                                                          const int64_t* __restrict__ hids,
                                                          int64_t* __restrict__ ids) {
  const StageCopy c = desc[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (hids)  // the ids, read in place from the mapped host arena
    for (int r = threadIdx.x; r < c.n; r += blockDim.x) ids[c.dst_row + r] = hids[c.src_row + r];
  for (int r = warp; r < c.n; r += 8) {
    const float4* x = reinterpret_cast<const float4*>(rows + (c.dst_row + r) * (int64_t)dp);
    float acc = 0.f;
    for (int j = lane; j < dp / 4; j += 32) {
      const float4 v = x[j];
      acc = __fmaf_rn(v.x, v.x, acc);
      acc = __fmaf_rn(v.y, v.y, acc);
      acc = __fmaf_rn(v.z, v.z, acc);
      acc = __fmaf_rn(v.w, v.w, acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(FULL, acc, o));
    if (lane == 0) nrm[c.dst_row + r] = acc;
  }
}
void launch_stage_norms(const StageCopy* desc, int ndesc, const float* rows, float* nrm, int dp,
                        const int64_t* hids, int64_t* ids, cudaStream_t st) {
  if (ndesc <= 0) return;
  stage_norms_kernel<<<ndesc, 256, 0, st>>>(desc, rows, nrm, dp, hids, ids);
}

}  // namespace pk

namespace pk {

// Batched in-place append (Cluster.add, ref/clusters.py:71-79, for a whole
// insert batch): row i of the padded staging block goes to arena row
// dst_row[i], with its id and squared norm.  One warp per row.
__global__ void __launch_bounds__(256) append_rows_kernel(const float* __restrict__ src,
                                                          const int64_t* __restrict__ src_ids,
                                                          const int64_t* __restrict__ dst_row, int n,
                                                          float* __restrict__ rows,
                                                          int64_t* __restrict__ ids,
                                                          float* __restrict__ nrm, int dp,
                                                          const int64_t* __restrict__ len_pairs, int nlen,
                                                          int64_t* __restrict__ d_len) {
  // the appended lists' new lengths (slot, len) go into the device table here,
  // stream-ordered with the rows (no separate table upload)
  if (blockIdx.x == 0)
    for (int t = threadIdx.x; t < nlen; t += blockDim.x) d_len[len_pairs[2 * t]] = len_pairs[2 * t + 1];
  const int i = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const int64_t r = dst_row[i];
  const float4* s4 = reinterpret_cast<const float4*>(src + (int64_t)i * dp);
  float4* d4 = reinterpret_cast<float4*>(rows + r * dp);
  float acc = 0.f;
  for (int j = lane; j < dp / 4; j += 32) {
    const float4 v = s4[j];
    d4[j] = v;
    acc = __fmaf_rn(v.x, v.x, acc);
    acc = __fmaf_rn(v.y, v.y, acc);
    acc = __fmaf_rn(v.z, v.z, acc);
    acc = __fmaf_rn(v.w, v.w, acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(FULL, acc, o));
  if (lane == 0) {
    nrm[r] = acc;
    ids[r] = src_ids[i];
  }
}
void launch_append_rows(const float* src, const int64_t* src_ids, const int64_t* dst_row, int n,
                        float* rows, int64_t* ids, float* nrm, int dp, cudaStream_t st,
                        const int64_t* len_pairs, int nlen, int64_t* d_len) {
  if (n <= 0 && nlen <= 0) return;
  append_rows_kernel<<<std::max((n + 7) / 8, 1), 256, 0, st>>>(src, src_ids, dst_row, n, rows, ids, nrm, dp,
                                                               len_pairs, nlen, d_len);
}

}  // namespace pk

namespace pk {

// =====================================================================
// Per-list exact distances for one query (agent-mode L2 scan with early
// termination, ref/engine.py:377-396): rows of m lists -- HBM arena ranges
// or, for cold lists, the device-mapped host arena -- concatenated in probe
// order, one thread per row, reference arithmetic over the true dimension.
// =====================================================================
template <int METRIC>
__global__ void lists_dist_kernel(const float* __restrict__ q, const float* __restrict__ qn_p, const ListSrc* __restrict__ src,
                                  const int64_t* __restrict__ prefix, int m, int dp, int d,
                                  float* __restrict__ out_d, int64_t* __restrict__ out_ids) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t total = prefix[m];
  if (r >= total) return;
  int lo = 0, hi = m - 1;  // list holding row r
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (prefix[mid] <= r) lo = mid;
    else hi = mid - 1;
  }
  const int64_t i = r - prefix[lo];
  const float* x = src[lo].rows + i * dp;
  float acc = 0.f, nn = 0.f;
  for (int j = 0; j < d; j++) {
    const float xv = x[j], qv = q[j];
    if (METRIC == SQ_L2) {
      acc = sq_step(acc, xv, qv);
    } else {
      acc = ip_step(acc, xv, qv);
      if (METRIC == COSINE) nn = ip_step(nn, xv, xv);
    }
  }
  out_d[r] = finalize<METRIC>(acc, nn, METRIC == COSINE ? *qn_p : 0.f);
  out_ids[r] = src[lo].ids[i];
}

void launch_lists_dist(int metric, const float* q, const float* qn, const ListSrc* src, const int64_t* prefix,
                       int m, int64_t total, int dp, int d, float* out_d, int64_t* out_ids,
                       cudaStream_t st) {
  if (total <= 0 || m <= 0) return;
  const unsigned grid = (unsigned)((total + 127) / 128);
  if (metric == SQ_L2) lists_dist_kernel<SQ_L2><<<grid, 128, 0, st>>>(q, qn, src, prefix, m, dp, d, out_d, out_ids);
  else if (metric == IP) lists_dist_kernel<IP><<<grid, 128, 0, st>>>(q, qn, src, prefix, m, dp, d, out_d, out_ids);
  else lists_dist_kernel<COSINE><<<grid, 128, 0, st>>>(q, qn, src, prefix, m, dp, d, out_d, out_ids);
}

}  // namespace pk

namespace pk {

// =====================================================================
// Peer combine (the combine half of dispatch/combine,
// fused with the result write-out): instead of writing local result blocks
// and running an NCCL all-to-all, the scan's per-query results are written
// straight into each origin rank's receive area in ITS HBM (CUDA IPC
// mapping; P2P stores over NVLink / NVSwitch), then flagged:
//   peer_send_kernel   block g of this rank's results -> peer g's area, slot
//                      my_rank; every CTA fences at system scope and counts
//                      itself; the last CTA publishes flag[my_rank] = epoch in
//                      every peer's area with a release store.
//   peer_merge_kernel  each query's CTA acquires all R flags of the epoch
//                      (bounded spin; timeout -> error word), then merges the
//                      R blocks exactly like shard_merge_kernel.
// Area layout: R shard blocks of block_bytes, then R flags of 128 bytes.
// =====================================================================
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void peer_send_kernel(const int64_t* __restrict__ ids, const int64_t* __restrict__ cids,
                                 const int64_t* __restrict__ sc, const float* __restrict__ d,
                                 const int32_t* __restrict__ n, int B, int group, int kk,
                                 int64_t block_bytes, uint8_t* const* __restrict__ peers, int R,
                                 int my_rank, uint64_t epoch, uint32_t* __restrict__ done_ctr) {
  const int64_t nkk_g = (int64_t)group * kk;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)B * kk;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(i / kk), e = (int)(i - (int64_t)b * kk);
    const int g = b / group, bl = b - g * group;
    uint8_t* blk = peers[g] + (int64_t)my_rank * block_bytes;
    const int64_t o = (int64_t)bl * kk + e;
    reinterpret_cast<int64_t*>(blk)[o] = ids[i];
    reinterpret_cast<int64_t*>(blk + 8 * nkk_g)[o] = cids[i];
    reinterpret_cast<float*>(blk + 16 * nkk_g + 8 * (int64_t)group)[o] = d[i];
    if (e == 0) {
      reinterpret_cast<int64_t*>(blk + 16 * nkk_g)[bl] = sc[b];
      reinterpret_cast<int32_t*>(blk + 20 * nkk_g + 8 * (int64_t)group)[bl] = n[b];
    }
  }
  __threadfence_system();  // this CTA's stores before its arrival
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t prev = atomicAdd(done_ctr, 1u);
    if ((prev + 1) % gridDim.x == 0) {  // last CTA of this launch: publish the epoch
      __threadfence_system();
      for (int g = 0; g < R; g++)
        st_release_sys(reinterpret_cast<uint64_t*>(peers[g] + (int64_t)R * block_bytes) + 16 * my_rank,
                       epoch);
    }
  }
}

void launch_peer_send(const int64_t* ids, const int64_t* cids, const int64_t* sc, const float* d,
                      const int32_t* n, int B, int group, int kk, int64_t block_bytes,
                      uint8_t* const* peers, int R, int my_rank, uint64_t epoch, uint32_t* done_ctr,
                      cudaStream_t st) {
  const int64_t tot = (int64_t)B * kk;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((tot + 255) / 256, 592));
  peer_send_kernel<<<grid, 256, 0, st>>>(ids, cids, sc, d, n, B, group, kk, block_bytes, peers, R,
                                         my_rank, epoch, done_ctr);
}

__global__ void __launch_bounds__(128) peer_merge_kernel(int metric, const uint8_t* __restrict__ area,
                                                         int64_t block_bytes, int R, int B, int kk,
                                                         uint64_t epoch, int64_t timeout_ns,
                                                         int32_t* __restrict__ err,
                                                         int64_t* __restrict__ out_ids,
                                                         float* __restrict__ out_d,
                                                         int64_t* __restrict__ out_cid,
                                                         int32_t* __restrict__ out_n,
                                                         int64_t* __restrict__ out_scanned) {
  extern __shared__ Entry sbuf[];
  __shared__ int s_cnt, s_ok;
  const uint64_t* flags = reinterpret_cast<const uint64_t*>(area + (int64_t)R * block_bytes);
  if (threadIdx.x == 0) {
    uint64_t t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    int ok = 1;
    for (int r = 0; r < R && ok; r++) {
      while (ld_acquire_sys(flags + 16 * r) < epoch) {
        __nanosleep(200);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if ((int64_t)(t - t0) > timeout_ns) {
          ok = 0;
          atomicExch(err, 1);
          break;
        }
      }
    }
    s_ok = ok;
    s_cnt = 0;
  }
  __syncthreads();
  const int b = blockIdx.x;
  const int64_t nkk = (int64_t)B * kk;
  if (!s_ok) {
    for (int i = threadIdx.x; i < kk; i += blockDim.x) out_ids[(int64_t)b * kk + i] = -1;
    if (threadIdx.x == 0) out_n[b] = 0;
    return;
  }
  const int total = R * kk;
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    const int r = i / kk, e = i - r * kk;
    const uint8_t* blk = area + (int64_t)r * block_bytes;
    const int32_t n = reinterpret_cast<const int32_t*>(blk + (nkk * 20 + (int64_t)B * 8))[b];
    if (e >= n) continue;
    Entry en;
    en.key = f2key(reinterpret_cast<const float*>(blk + nkk * 16 + (int64_t)B * 8)[(int64_t)b * kk + e]);
    en.id = reinterpret_cast<const int64_t*>(blk)[(int64_t)b * kk + e];
    en.pay = i;
    sbuf[atomicAdd(&s_cnt, 1)] = en;
  }
  __syncthreads();
  const int n = s_cnt;
  cta_bitonic_sort(sbuf, n);
  const int kept = cta_compact_sorted(sbuf, n, kk, true, &s_cnt);
  for (int i = threadIdx.x; i < kk; i += blockDim.x) {
    const int64_t o = (int64_t)b * kk + i;
    if (i < kept) {
      const int src = sbuf[i].pay;
      const int r = src / kk, e = src - r * kk;
      out_ids[o] = sbuf[i].id;
      out_d[o] = key2dist(sbuf[i].key, metric);
      if (out_cid)
        out_cid[o] = reinterpret_cast<const int64_t*>(area + (int64_t)r * block_bytes + nkk * 8)[(int64_t)b * kk + e];
    } else {
      out_ids[o] = -1;
      out_d[o] = __int_as_float(0x7f800000);
      if (out_cid) out_cid[o] = -1;
    }
  }
  if (threadIdx.x == 0) {
    out_n[b] = kept;
    if (out_scanned) {
      int64_t s = 0;
      for (int r = 0; r < R; r++)
        s += reinterpret_cast<const int64_t*>(area + (int64_t)r * block_bytes + nkk * 16)[b];
      out_scanned[b] = s;
    }
  }
}

void launch_peer_merge(int metric, const void* area, int64_t block_bytes, int R, int B, int kk, uint64_t epoch,
                       int64_t timeout_ns, int32_t* err, int64_t* out_ids, float* out_d,
                       int64_t* out_cid, int32_t* out_n, int64_t* out_scanned, cudaStream_t st) {
  if (B <= 0) return;
  int N = 1;
  while (N < R * kk) N <<= 1;
  const size_t smem = (size_t)N * sizeof(Entry);
  PK_SMEM_ATTR(peer_merge_kernel, (int)smem);
  peer_merge_kernel<<<B, 128, smem, st>>>(metric, static_cast<const uint8_t*>(area), block_bytes, R, B, kk, epoch,
                                          timeout_ns, err, out_ids, out_d, out_cid, out_n, out_scanned);
}

}  // namespace pk
