// pk_agent.cu -- the device half of one agent-mode search (ref/engine.py:
// 319-404 with the multi-level cache of ref/cache.py:162-315) and of the
// cache's L1 placement loop.
//
// The agent path is sequential per query in the reference: the FSM match
// orders the cache scan, the cache scan may stop before the lists, every
// promotion moves L1 centroids.  What it needs from the device is distances,
// and almost all of them are known the moment the query is: q against every
// FSM state, every cached pool row in scope, every L1 centroid, every staged
// row, the coarse graph's centroids and every row of the lists it probes.  So
// one call computes all of them (pk_agent_read) and the host replays the
// policy over the values; a row's distance does not depend on which call
// computed it, so the replay takes the reference's decisions exactly.
//
// The rows the policy scans (pool rows, L1 centroids, FSM states) live in an
// HBM row store at host-managed slots (pk_rows_put); only new rows cross
// PCIe, never the pools themselves.
//
// The L1 placement of items popped from a full L0 entry (ref/cache.py:
// 284-310) is a true chain -- each add moves one centroid the next item is
// measured against -- so it runs as one single-CTA kernel that replays the
// loop and reports each decision (l1_place_kernel).
#include "pk_kernels.h"
#include "pk_ptx.cuh"

namespace pk {

namespace {

template <int METRIC>
__device__ __forceinline__ float fin(float acc, float nn, float qn) {
  if (METRIC == SQ_L2) return acc;
  if (METRIC == IP) return -acc;
  return __fsub_rn(1.0f, __fdiv_rn(acc, __fmul_rn(__fsqrt_rn(nn), qn)));  // ref/kernels.py:112
}

// dist(q, x) with the reference's arithmetic (ref/kernels.py:73-113): j
// ascending over the true dimension, every op rounded; rows padded to 16 B.
template <int METRIC>
__device__ __forceinline__ float ref_dist(const float* __restrict__ x, const float* __restrict__ q, int d,
                                          float qn) {
  float acc = 0.f, nn = 0.f;
  const int d4 = d >> 2;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  const float4* q4 = reinterpret_cast<const float4*>(q);
#pragma unroll 4
  for (int j = 0; j < d4; j++) {
    const float4 xv = x4[j], qv = q4[j];
    if (METRIC == SQ_L2) {
      acc = sq_step(acc, xv.x, qv.x);
      acc = sq_step(acc, xv.y, qv.y);
      acc = sq_step(acc, xv.z, qv.z);
      acc = sq_step(acc, xv.w, qv.w);
    } else {
      acc = ip_step(acc, xv.x, qv.x);
      acc = ip_step(acc, xv.y, qv.y);
      acc = ip_step(acc, xv.z, qv.z);
      acc = ip_step(acc, xv.w, qv.w);
      if (METRIC == COSINE) {
        nn = ip_step(nn, xv.x, xv.x);
        nn = ip_step(nn, xv.y, xv.y);
        nn = ip_step(nn, xv.z, xv.z);
        nn = ip_step(nn, xv.w, xv.w);
      }
    }
  }
  for (int j = 4 * d4; j < d; j++) {
    if (METRIC == SQ_L2) {
      acc = sq_step(acc, x[j], q[j]);
    } else {
      acc = ip_step(acc, x[j], q[j]);
      if (METRIC == COSINE) nn = ip_step(nn, x[j], x[j]);
    }
  }
  return fin<METRIC>(acc, nn, qn);
}

// |q| of cosine_nb: sequential fp32 sum of squares, sqrt (ref/kernels.py:101-104)
__device__ __forceinline__ float seq_norm(const float* q, int d) {
  float acc = 0.f;
  for (int j = 0; j < d; j++) acc = ip_step(acc, q[j], q[j]);
  return __fsqrt_rn(acc);
}

// stage a padded row into shared memory (and |row| for cosine)
template <int METRIC>
__device__ __forceinline__ void stage_q(const float* __restrict__ src, float* qs, float* qn_s, int dp, int d) {
  for (int j = threadIdx.x; j < dp; j += blockDim.x) qs[j] = src[j];
  __syncthreads();
  if (METRIC == COSINE && threadIdx.x == 0) *qn_s = seq_norm(qs, d);
  __syncthreads();
}

__global__ void rows_put_kernel(const float* __restrict__ src, const int32_t* __restrict__ slots, int n, int dp,
                                float* __restrict__ rows) {
  const int64_t n4 = (int64_t)n * dp / 4;
  const int dp4 = dp / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / dp4, c = i - r * dp4;
    reinterpret_cast<float4*>(rows + (int64_t)slots[r] * dp)[c] = reinterpret_cast<const float4*>(src)[i];
  }
}

// Up to 128 rows (pointers in rowp[]) streamed through shared memory in
// column blocks of W floats by coalesced 16-byte cp.async pieces (a 3-deep
// ring; W wider when the block holds few rows), one thread per row running
// the reference's sequential chain over the padded row from shared memory --
// the rows' bytes arrive at streaming rate instead of one dependent global
// load per float4 per thread.  (The padding columns are zero: they add +0.)
constexpr int AG_RING = 3;
constexpr int AG_RS = 32 + 4;
constexpr size_t AG_RING_FLOATS = (size_t)AG_RING * 128 * AG_RS;
template <int METRIC>
__device__ __forceinline__ float staged_dist(const float* const* rowp, int nr, const float* qs, float qn, int dp,
                                             float* ring) {
  int W = (128 * AG_RS / max(nr, 1) - 4) / 32 * 32;
  W = W < 32 ? 32 : (W > dp ? dp : W);
  const int rs = W + 4;
  const int nblk = (dp + W - 1) / W;
  auto issue = [&](int blk) {
    if (blk < nblk) {
      float* dst = ring + (size_t)(blk % AG_RING) * 128 * AG_RS;
      const int w4 = min(W, dp - blk * W) / 4;
      for (int i = threadIdx.x; i < nr * w4; i += blockDim.x) {
        const int rr = i / w4, c = i - rr * w4;
        cp_async16(dst + rr * rs + 4 * c, rowp[rr] + blk * W + 4 * c);
      }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int i = 0; i < AG_RING - 1; i++) issue(i);
  float acc = 0.f, nn = 0.f;
  for (int blk = 0; blk < nblk; blk++) {
    issue(blk + AG_RING - 1);
    cp_async_wait<AG_RING - 1>();
    __syncthreads();
    const float* xr = ring + (size_t)(blk % AG_RING) * 128 * AG_RS + (threadIdx.x < nr ? threadIdx.x : 0) * rs;
    const float* qb = qs + blk * W;
    const int w = min(W, dp - blk * W);
#pragma unroll 8
    for (int j = 0; j < w; j += 4) {
      const float4 xv = *reinterpret_cast<const float4*>(xr + j);
      const float4 qv = *reinterpret_cast<const float4*>(qb + j);
      if (METRIC == SQ_L2) {
        acc = sq_step(acc, xv.x, qv.x);
        acc = sq_step(acc, xv.y, qv.y);
        acc = sq_step(acc, xv.z, qv.z);
        acc = sq_step(acc, xv.w, qv.w);
      } else {
        acc = ip_step(acc, xv.x, qv.x);
        acc = ip_step(acc, xv.y, qv.y);
        acc = ip_step(acc, xv.z, qv.z);
        acc = ip_step(acc, xv.w, qv.w);
        if (METRIC == COSINE) {
          nn = ip_step(nn, xv.x, xv.x);
          nn = ip_step(nn, xv.y, xv.y);
          nn = ip_step(nn, xv.z, xv.z);
          nn = ip_step(nn, xv.w, xv.w);
        }
      }
    }
    __syncthreads();  // the slot is refilled by the next issue
  }
  return fin<METRIC>(acc, nn, qn);
}

// out[i] = dist(q, rows[slots[i]]): blocks of 128 rows
template <int METRIC>
__global__ void __launch_bounds__(128) gather_dist_kernel(const float* __restrict__ q, const float* __restrict__ rows,
                                                          int dp, int d, const int32_t* __restrict__ slots, int n,
                                                          float* __restrict__ out, int rpb) {
  extern __shared__ __align__(16) float ag_sm[];  // q [dp] | ring
  __shared__ const float* rowp[128];
  __shared__ float qn_s;
  const int i0 = blockIdx.x * rpb;
  const int nr = min(rpb, n - i0);
  if (threadIdx.x < nr) rowp[threadIdx.x] = rows + (int64_t)slots[i0 + threadIdx.x] * dp;
  stage_q<METRIC>(q, ag_sm, &qn_s, dp, d);
  const float v = staged_dist<METRIC>(rowp, nr, ag_sm, METRIC == COSINE ? qn_s : 0.f, dp, ag_sm + dp);
  if (threadIdx.x < nr) out[i0 + threadIdx.x] = v;
}

// out[r][c] = dist(q = rows[qslots[r]], x = rows[xslots[c]]): block (x, r)
// covers columns [128 x, 128 x + 128) of query row r (the query roles of the
// reference's _dmat(A, B): batch_distances(A[r], B), ref/fsm.py)
template <int METRIC>
__global__ void __launch_bounds__(128) gather_mat_kernel(const float* __restrict__ rows, int dp, int d,
                                                         const int32_t* __restrict__ qslots, int nr,
                                                         const int32_t* __restrict__ xslots, int nc,
                                                         float* __restrict__ out) {
  extern __shared__ __align__(16) float ag_sm[];
  __shared__ const float* rowp[128];
  __shared__ float qn_s;
  const int r = blockIdx.y;
  const int c0 = blockIdx.x * 128;
  const int m = min(128, nc - c0);
  if (threadIdx.x < m) rowp[threadIdx.x] = rows + (int64_t)xslots[c0 + threadIdx.x] * dp;
  stage_q<METRIC>(rows + (int64_t)qslots[r] * dp, ag_sm, &qn_s, dp, d);
  const float v = staged_dist<METRIC>(rowp, m, ag_sm, METRIC == COSINE ? qn_s : 0.f, dp, ag_sm + dp);
  if (threadIdx.x < m) out[(int64_t)r * nc + c0 + threadIdx.x] = v;
}

// Every row of the probed lists (device probe slots, coarse order), laid out
// list after list: block (x, p) covers rows [128 x, 128 x + 128) of list p.
template <int METRIC>
__global__ void __launch_bounds__(128) probe_lists_kernel(const float* __restrict__ q, ListTable lt,
                                                          const int32_t* __restrict__ probe, int nprobe, int64_t cap,
                                                          float* __restrict__ out_d, int64_t* __restrict__ out_ids,
                                                          int64_t* __restrict__ out_prefix,
                                                          int64_t* __restrict__ out_cids, int rpb) {
  extern __shared__ __align__(16) float ag_sm[];
  __shared__ const float* rowp[128];
  __shared__ float qn_s;
  __shared__ int64_t pre_s;
  // batched (pk_agent_lists): query z's vector, probe and output blocks
  const int z = blockIdx.z;
  q += (int64_t)z * lt.dp;
  probe += (int64_t)z * nprobe;
  out_d += z * cap;
  out_ids += z * cap;
  out_prefix += (int64_t)z * (nprobe + 1);
  out_cids += (int64_t)z * nprobe;
  const int p = blockIdx.y;
  const int sl = probe[p];
  const int64_t len = sl >= 0 ? lt.len[sl] : 0;
  const int64_t r0 = (int64_t)blockIdx.x * rpb;
  if (r0 >= len && blockIdx.x != 0) return;
  if (threadIdx.x == 0) {
    int64_t pre = 0;
    for (int i = 0; i < p; i++) {
      const int s2 = probe[i];
      pre += s2 >= 0 ? lt.len[s2] : 0;
    }
    pre_s = pre;
    if (blockIdx.x == 0) {
      out_prefix[p + 1] = pre + len;
      out_cids[p] = sl >= 0 ? lt.cid[sl] : -1;
      if (p == 0) out_prefix[0] = 0;
    }
  }
  const int64_t left = len - r0;
  const int nr = left <= 0 ? 0 : (left < rpb ? (int)left : rpb);
  if (threadIdx.x < nr) rowp[threadIdx.x] = lt.rows + (lt.off[sl] + r0 + threadIdx.x) * lt.dp;
  stage_q<METRIC>(q, ag_sm, &qn_s, lt.dp, lt.d);
  if (nr == 0) return;
  const float v = staged_dist<METRIC>(rowp, nr, ag_sm, METRIC == COSINE ? qn_s : 0.f, lt.dp, ag_sm + lt.dp);
  const int64_t r = r0 + threadIdx.x;
  if (threadIdx.x >= nr || pre_s + r >= cap) return;  // past the caller's capacity: it sees the total and asks again
  out_d[pre_s + r] = v;
  out_ids[pre_s + r] = lt.ids[lt.off[sl] + r];
}

// argmin order of np.argmin: the first minimum, NaN before everything
__device__ __forceinline__ bool am_better(float a, float b) {
  if (isnan(b)) return false;
  if (isnan(a)) return true;
  return a < b;
}

// The L1 placement chain of ref/cache.py:284-310 (+ the capture target of
// :312-325), for `m` items popped from L0 in order.  State: the live L1
// clusters in list order (physical index per position), their fp64 column
// sums, counts and f32 centroids (sum / n, rounded; zeros when empty).
// Per item: _nearest_l1 (a new empty cluster while fewer than n_p, else the
// first nearest centroid), _l1_add unless the item is already held by a
// cluster that is still live (index-wide dedup), merge_down when the target
// reaches capacity (the cluster leaves the list; its items become unheld).
// Outputs per item: the target's list position at that moment (-1: a new
// cluster was appended), added flag, merged flag; then q's target (-1: new).
// One CTA of 256 threads; the distance chains run one thread per cluster.
constexpr int L1_MAXC = 64;
template <int METRIC>
__global__ void __launch_bounds__(256) l1_place_kernel(int nc0, int n_p, int cap, int dp, int d,
                                                       double* __restrict__ sums, float* __restrict__ cents,
                                                       int32_t* __restrict__ cnt, const float* __restrict__ items,
                                                       const int32_t* __restrict__ holder,
                                                       const int32_t* __restrict__ dup, int m,
                                                       const float* __restrict__ qv, int32_t* __restrict__ out_t,
                                                       uint8_t* __restrict__ out_added,
                                                       uint8_t* __restrict__ out_merged, int32_t* __restrict__ out_q) {
  // the live clusters' centroids live in shared memory (n_p rows, a slot per
  // live cluster) with the item being placed: every chain step reads shared
  // memory, not L2
  // rows at a stride of dp + 4 floats: the chains (one thread per cluster)
  // read the same column of different rows at once, and a multiple-of-32
  // stride would put all of them in one bank
  extern __shared__ __align__(16) float l1s[];  // [n_p][dp + 4] centroids | [dp] item
  const int ls = dp + 4;
  float* vs = l1s + (size_t)n_p * ls;
  __shared__ int order[L1_MAXC];
  __shared__ uint8_t merged[L1_MAXC];
  __shared__ int hold[L1_MAXC];   // per chain item: the cluster holding its id after it
  __shared__ int sslot[L1_MAXC];  // physical cluster -> shared-memory row
  __shared__ int sfree[L1_MAXC];
  __shared__ float dist_s[L1_MAXC];
  __shared__ int n_live, next_phys, s_tpos, s_add, n_free;
  const int tid = threadIdx.x;
  if (tid < L1_MAXC) {
    order[tid] = tid;
    merged[tid] = 0;
    sslot[tid] = tid < nc0 ? tid : -1;
  }
  if (tid == 0) {
    n_live = nc0;
    next_phys = nc0;
    n_free = 0;
    for (int i = n_p - 1; i >= nc0; i--) sfree[n_free++] = i;
  }
  for (int i = tid; i < nc0 * dp; i += blockDim.x) {
    const int r = i / dp;
    l1s[(size_t)r * ls + (i - r * dp)] = cents[i];
  }
  __syncthreads();
  for (int it = 0; it <= m; it++) {
    const bool is_q = it == m;
    if (is_q && qv == nullptr) break;
    const float* v = is_q ? qv : items + (int64_t)it * dp;
    for (int j = tid; j < dp; j += blockDim.x) vs[j] = v[j];
    __syncthreads();
    int tpos = -1;  // _nearest_l1 appends a fresh cluster while fewer than n_p
    const int nl = n_live;
    if (nl >= n_p) {  // the first nearest centroid (list order)
      if (tid < nl) {
        const float* c = l1s + (size_t)sslot[order[tid]] * ls;
        dist_s[tid] = ref_dist<METRIC>(c, vs, d, METRIC == COSINE ? seq_norm(vs, d) : 0.f);
      }
      __syncthreads();
      tpos = 0;
      for (int i = 1; i < nl; i++)
        if (am_better(dist_s[i], dist_s[tpos])) tpos = i;
    }
    if (is_q) {
      if (tid == 0) *out_q = tpos;
      break;
    }
    __syncthreads();
    if (tid == 0) {
      int t;
      if (tpos < 0) {
        t = next_phys++;
        order[n_live++] = t;
        cnt[t] = 0;
        sslot[t] = sfree[--n_free];
      } else {
        t = order[tpos];
      }
      // an id placed earlier in this chain is held by where that left it
      const int h = dup[it] >= 0 ? hold[dup[it]] : holder[it];
      const bool held = h >= 0 && !merged[h];
      hold[it] = held ? h : t;
      s_tpos = t;
      s_add = !held;
      out_t[it] = tpos;
      out_added[it] = !held;
    }
    __syncthreads();
    const int t = s_tpos;
    float* cs = l1s + (size_t)sslot[t] * ls;
    if (s_add) {
      const int n1 = cnt[t] + 1;
      for (int j = tid; j < dp; j += blockDim.x) {
        double* sp = sums + (int64_t)t * dp + j;
        const double nv = (tpos < 0 ? 0.0 : *sp) + (double)vs[j];
        *sp = nv;
        cs[j] = (float)(nv / (double)n1);
      }
      __syncthreads();
      if (tid == 0) cnt[t] = n1;
    } else if (tpos < 0) {
      for (int j = tid; j < dp; j += blockDim.x) {  // a fresh cluster that stays empty
        sums[(int64_t)t * dp + j] = 0.0;
        cs[j] = 0.f;
      }
    }
    __syncthreads();
    if (tid == 0) {
      const bool full = cnt[t] >= cap;
      out_merged[it] = full;
      if (full) {  // merge_down: the cluster leaves the list, its row is free
        merged[t] = 1;
        sfree[n_free++] = sslot[t];
        int w = 0;
        for (int i = 0; i < n_live; i++)
          if (order[i] != t) order[w++] = order[i];
        n_live = w;
      }
    }
    __syncthreads();
  }
}

}  // namespace

void launch_rows_put(const float* src, const int32_t* slots, int n, int dp, float* rows, cudaStream_t st) {
  if (n <= 0) return;
  const int64_t n4 = (int64_t)n * dp / 4;
  const unsigned grid = (unsigned)std::min<int64_t>((n4 + 255) / 256, 1184);
  rows_put_kernel<<<grid, 256, 0, st>>>(src, slots, n, dp, rows);
}

static size_t ag_smem(int dp) { return (size_t)dp * 4 + AG_RING_FLOATS * 4; }
template <typename K>
static void ag_attr(K k, size_t smem) {
  if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

void launch_gather_dist(int metric, const float* q, const float* rows, int dp, int d, const int32_t* slots, int n,
                        float* out, cudaStream_t st) {
  if (n <= 0) return;
  // fewer rows per block when a call would leave most SMs idle: wider column
  // blocks, fewer ring round trips per block
  int rpb = 128;
  while (rpb > 32 && (n + rpb - 1) / rpb < 148) rpb >>= 1;
  const unsigned grid = (unsigned)((n + rpb - 1) / rpb);
  const size_t sm = ag_smem(dp);
#define AG_GD(M)                                                                \
  {                                                                           \
    ag_attr(gather_dist_kernel<M>, sm);                                       \
    gather_dist_kernel<M><<<grid, 128, sm, st>>>(q, rows, dp, d, slots, n, out, rpb); \
  }
  if (metric == SQ_L2) AG_GD(SQ_L2) else if (metric == IP) AG_GD(IP) else AG_GD(COSINE)
#undef AG_GD
}

void launch_gather_mat(int metric, const float* rows, int dp, int d, const int32_t* qslots, int nr,
                       const int32_t* xslots, int nc, float* out, cudaStream_t st) {
  if (nr <= 0 || nc <= 0) return;
  const dim3 grid((unsigned)((nc + 127) / 128), (unsigned)nr);
  const size_t sm = ag_smem(dp);
#define AG_GM(M)                                                                          \
  {                                                                                     \
    ag_attr(gather_mat_kernel<M>, sm);                                                  \
    gather_mat_kernel<M><<<grid, 128, sm, st>>>(rows, dp, d, qslots, nr, xslots, nc, out); \
  }
  if (metric == SQ_L2) AG_GM(SQ_L2) else if (metric == IP) AG_GM(IP) else AG_GM(COSINE)
#undef AG_GM
}

void launch_probe_lists(int metric, const float* q, ListTable lt, const int32_t* probe, int nprobe,
                        int64_t maxlen, int64_t cap, float* out_d, int64_t* out_ids, int64_t* out_prefix,
                        int64_t* out_cids, cudaStream_t st, int nq) {
  if (nprobe <= 0 || nq <= 0) return;
  int rpb = 128;
  while (rpb > 32 && ((maxlen + rpb - 1) / rpb) * nprobe * nq < 296) rpb >>= 1;
  const dim3 grid((unsigned)std::max<int64_t>(1, (maxlen + rpb - 1) / rpb), (unsigned)nprobe, (unsigned)nq);
  const size_t sm = ag_smem(lt.dp);
#define AG_PL(M)                                                                                  \
  {                                                                                             \
    ag_attr(probe_lists_kernel<M>, sm);                                                         \
    probe_lists_kernel<M><<<grid, 128, sm, st>>>(q, lt, probe, nprobe, cap, out_d, out_ids, out_prefix, out_cids, rpb); \
  }
  if (metric == SQ_L2) AG_PL(SQ_L2) else if (metric == IP) AG_PL(IP) else AG_PL(COSINE)
#undef AG_PL
}

int l1_place_max_clusters() { return L1_MAXC; }

void launch_l1_place(int metric, int nc0, int n_p, int cap, int dp, int d, double* sums, float* cents,
                     int32_t* cnt, const float* items, const int32_t* holder, const int32_t* dup, int m,
                     const float* qv, int32_t* out_t, uint8_t* out_added, uint8_t* out_merged, int32_t* out_q,
                     cudaStream_t st) {
  const size_t sm = ((size_t)n_p * (dp + 4) + dp) * 4;
#define AG_L1(M)                                                                                       \
  {                                                                                                  \
    ag_attr(l1_place_kernel<M>, sm);                                                                 \
    l1_place_kernel<M><<<1, 256, sm, st>>>(nc0, n_p, cap, dp, d, sums, cents, cnt, items, holder, dup, m, qv, \
                                            out_t, out_added, out_merged, out_q);                     \
  }
  if (metric == SQ_L2) AG_L1(SQ_L2) else if (metric == IP) AG_L1(IP) else AG_L1(COSINE)
#undef AG_L1
}

}  // namespace pk
