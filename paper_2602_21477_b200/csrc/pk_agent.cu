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

// out[i] = dist(q, rows[slots[i]]), one thread per row
template <int METRIC>
__global__ void __launch_bounds__(128) gather_dist_kernel(const float* __restrict__ q, const float* __restrict__ rows,
                                                          int dp, int d, const int32_t* __restrict__ slots, int n,
                                                          float* __restrict__ out) {
  extern __shared__ __align__(16) float ag_q[];
  __shared__ float qn_s;
  stage_q<METRIC>(q, ag_q, &qn_s, dp, d);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = ref_dist<METRIC>(rows + (int64_t)slots[i] * dp, ag_q, d, METRIC == COSINE ? qn_s : 0.f);
}

// out[r][c] = dist(q = rows[qs[r]], x = rows[xs[c]]): the query roles of the
// reference's _dmat(A, B) (ref/fsm.py; batch_distances(A[r], B))
template <int METRIC>
__global__ void __launch_bounds__(128) gather_mat_kernel(const float* __restrict__ rows, int dp, int d,
                                                         const int32_t* __restrict__ qslots, int nr,
                                                         const int32_t* __restrict__ xslots, int nc,
                                                         float* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)nr * nc) return;
  const int r = (int)(i / nc), c = (int)(i - (int64_t)r * nc);
  const float* q = rows + (int64_t)qslots[r] * dp;
  out[i] = ref_dist<METRIC>(rows + (int64_t)xslots[c] * dp, q, d, METRIC == COSINE ? seq_norm(q, d) : 0.f);
}

// Every row of the probed lists (device probe slots, coarse order), laid out
// list after list: block (x, p) covers rows [128 x, 128 x + 128) of list p.
template <int METRIC>
__global__ void __launch_bounds__(128) probe_lists_kernel(const float* __restrict__ q, ListTable lt,
                                                          const int32_t* __restrict__ probe, int nprobe, int64_t cap,
                                                          float* __restrict__ out_d, int64_t* __restrict__ out_ids,
                                                          int64_t* __restrict__ out_prefix,
                                                          int64_t* __restrict__ out_cids) {
  extern __shared__ __align__(16) float ag_q[];
  __shared__ float qn_s;
  __shared__ int64_t pre_s;
  const int p = blockIdx.y;
  const int sl = probe[p];
  const int64_t len = sl >= 0 ? lt.len[sl] : 0;
  if ((int64_t)blockIdx.x * 128 >= len && !(blockIdx.x == 0)) return;
  if (threadIdx.x == 0) {
    int64_t pre = 0;
    for (int i = 0; i < p; i++) {
      const int s = probe[i];
      pre += s >= 0 ? lt.len[s] : 0;
    }
    pre_s = pre;
    if (blockIdx.x == 0) {
      out_prefix[p + 1] = pre + len;
      out_cids[p] = sl >= 0 ? lt.cid[sl] : -1;
      if (p == 0) out_prefix[0] = 0;
    }
  }
  stage_q<METRIC>(q, ag_q, &qn_s, lt.dp, lt.d);
  const int64_t r = (int64_t)blockIdx.x * 128 + threadIdx.x;
  if (r >= len || pre_s + r >= cap) return;  // past the caller's capacity: it sees the total and asks again
  const int64_t arow = lt.off[sl] + r;
  out_d[pre_s + r] = ref_dist<METRIC>(lt.rows + arow * lt.dp, ag_q, lt.d, METRIC == COSINE ? qn_s : 0.f);
  out_ids[pre_s + r] = lt.ids[arow];
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
  __shared__ int order[L1_MAXC];
  __shared__ uint8_t merged[L1_MAXC];
  __shared__ int hold[L1_MAXC];  // per chain item: the cluster holding its id after it
  __shared__ float dist_s[L1_MAXC];
  __shared__ int n_live, next_phys, s_tpos, s_add;
  const int tid = threadIdx.x;
  if (tid < L1_MAXC) {
    order[tid] = tid;
    merged[tid] = 0;
  }
  if (tid == 0) {
    n_live = nc0;
    next_phys = nc0;
  }
  __syncthreads();
  auto nearest = [&](const float* v) -> int {  // list position of the first nearest centroid
    const int nl = n_live;
    if (tid < nl) {
      const float* c = cents + (int64_t)order[tid] * dp;
      dist_s[tid] = ref_dist<METRIC>(c, v, d, METRIC == COSINE ? seq_norm(v, d) : 0.f);
    }
    __syncthreads();
    int best = 0;
    for (int i = 1; i < nl; i++)
      if (am_better(dist_s[i], dist_s[best])) best = i;
    __syncthreads();
    return best;
  };
  for (int it = 0; it <= m; it++) {
    const bool is_q = it == m;
    if (is_q && qv == nullptr) break;
    const float* v = is_q ? qv : items + (int64_t)it * dp;
    int tpos;
    if (n_live < n_p) {
      tpos = -1;  // _nearest_l1 appends a fresh cluster
    } else {
      tpos = nearest(v);
    }
    if (is_q) {
      if (tid == 0) *out_q = tpos;
      break;
    }
    if (tid == 0) {
      int t;
      if (tpos < 0) {
        t = next_phys++;
        order[n_live++] = t;
        cnt[t] = 0;
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
    if (s_add) {
      const int n1 = cnt[t] + 1;
      for (int j = tid; j < dp; j += blockDim.x) {
        double* s = sums + (int64_t)t * dp + j;
        const double nv = (tpos < 0 ? 0.0 : *s) + (double)items[(int64_t)it * dp + j];
        *s = nv;
        cents[(int64_t)t * dp + j] = (float)(nv / (double)n1);
      }
      __syncthreads();
      if (tid == 0) cnt[t] = n1;
    } else if (tpos < 0) {
      for (int j = tid; j < dp; j += blockDim.x) {  // a fresh cluster that stays empty
        sums[(int64_t)t * dp + j] = 0.0;
        cents[(int64_t)t * dp + j] = 0.f;
      }
    }
    __syncthreads();
    if (tid == 0) {
      const bool full = cnt[t] >= cap;
      out_merged[it] = full;
      if (full) {  // merge_down: the cluster leaves the list
        merged[t] = 1;
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

void launch_gather_dist(int metric, const float* q, const float* rows, int dp, int d, const int32_t* slots, int n,
                        float* out, cudaStream_t st) {
  if (n <= 0) return;
  const unsigned grid = (unsigned)((n + 127) / 128);
  const size_t sm = (size_t)dp * 4;
  if (metric == SQ_L2) gather_dist_kernel<SQ_L2><<<grid, 128, sm, st>>>(q, rows, dp, d, slots, n, out);
  else if (metric == IP) gather_dist_kernel<IP><<<grid, 128, sm, st>>>(q, rows, dp, d, slots, n, out);
  else gather_dist_kernel<COSINE><<<grid, 128, sm, st>>>(q, rows, dp, d, slots, n, out);
}

void launch_gather_mat(int metric, const float* rows, int dp, int d, const int32_t* qslots, int nr,
                       const int32_t* xslots, int nc, float* out, cudaStream_t st) {
  const int64_t n = (int64_t)nr * nc;
  if (n <= 0) return;
  const unsigned grid = (unsigned)((n + 127) / 128);
  if (metric == SQ_L2) gather_mat_kernel<SQ_L2><<<grid, 128, 0, st>>>(rows, dp, d, qslots, nr, xslots, nc, out);
  else if (metric == IP) gather_mat_kernel<IP><<<grid, 128, 0, st>>>(rows, dp, d, qslots, nr, xslots, nc, out);
  else gather_mat_kernel<COSINE><<<grid, 128, 0, st>>>(rows, dp, d, qslots, nr, xslots, nc, out);
}

void launch_probe_lists(int metric, const float* q, ListTable lt, const int32_t* probe, int nprobe,
                        int64_t maxlen, int64_t cap, float* out_d, int64_t* out_ids, int64_t* out_prefix, int64_t* out_cids,
                        cudaStream_t st) {
  if (nprobe <= 0) return;
  const dim3 grid((unsigned)std::max<int64_t>(1, (maxlen + 127) / 128), (unsigned)nprobe);
  const size_t sm = (size_t)lt.dp * 4;
  if (metric == SQ_L2)
    probe_lists_kernel<SQ_L2><<<grid, 128, sm, st>>>(q, lt, probe, nprobe, cap, out_d, out_ids, out_prefix, out_cids);
  else if (metric == IP)
    probe_lists_kernel<IP><<<grid, 128, sm, st>>>(q, lt, probe, nprobe, cap, out_d, out_ids, out_prefix, out_cids);
  else
    probe_lists_kernel<COSINE><<<grid, 128, sm, st>>>(q, lt, probe, nprobe, cap, out_d, out_ids, out_prefix, out_cids);
}

int l1_place_max_clusters() { return L1_MAXC; }

void launch_l1_place(int metric, int nc0, int n_p, int cap, int dp, int d, double* sums, float* cents,
                     int32_t* cnt, const float* items, const int32_t* holder, const int32_t* dup, int m,
                     const float* qv,
                     int32_t* out_t, uint8_t* out_added, uint8_t* out_merged, int32_t* out_q, cudaStream_t st) {
  if (metric == SQ_L2)
    l1_place_kernel<SQ_L2><<<1, 256, 0, st>>>(nc0, n_p, cap, dp, d, sums, cents, cnt, items, holder, dup, m, qv, out_t,
                                               out_added, out_merged, out_q);
  else if (metric == IP)
    l1_place_kernel<IP><<<1, 256, 0, st>>>(nc0, n_p, cap, dp, d, sums, cents, cnt, items, holder, dup, m, qv, out_t,
                                            out_added, out_merged, out_q);
  else
    l1_place_kernel<COSINE><<<1, 256, 0, st>>>(nc0, n_p, cap, dp, d, sums, cents, cnt, items, holder, dup, m, qv, out_t,
                                                out_added, out_merged, out_q);
}

}  // namespace pk
