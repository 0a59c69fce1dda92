// pk_graph.cu -- device traversal of the reference's hybrid coarse graph.
//
// The reference's coarse quantizer is not flat: HybridGraphIndex.search
// (ref/graph.py:321-396) is a best-first traversal over per-scope HNSW-style
// graphs joined by portal edges, with ef = max(ef_search_factor * nprobe,
// nprobe) -- approximate at the default factor 4 (ref/engine.py:68, 369).
// This kernel replays that traversal for a batch of queries so the drop-in
// probes the lists the reference probes at ANY ef, and reports the same
// coarse_computations count.
//
// Inputs: the exact reference distance of every query to every list centroid
// (dist_dense, ref/kernels.py:73-113 arithmetic -- the values the reference's
// _dist returns), and the graph uploaded by pk_graph_set (neighbor lists in
// the reference's list order, portals in insertion order).  The traversal is
// the reference's, decision for decision:
//   * the candidate heap pops the smallest (d, cid) (Python tuple order);
//   * the result heap holds (-d, cid) tuples, so its top -- the element a
//     push beyond ef evicts, and the bound the stop rule and the admission
//     test read -- is the LARGEST d, ties to the SMALLEST cid;
//   * admission `len(best) < ef or nd < worst`, stop `d > worst and
//     len(best) >= ef`, neighbor order = list order, every newly visited
//     node counts one distance computation.
// Keys pack (order-preserving f32 bits, cid) into 64 bits, so heap order is
// exactly the tuple order (cids are below 2^32; pk_graph_set checks).
//
// One warp per query: lane 0 runs the sequential traversal (the reference's
// own control flow is sequential: each admission changes the bound the next
// one reads), the warp clears the per-query visit stamps and selects the
// emitted top-nprobe.
#include "pk_kernels.h"
#include "pk_ptx.cuh"

namespace pk {

namespace {

constexpr unsigned FULLW = 0xffffffffu;
constexpr uint32_t EMIT = 0xfffffffeu;  // stamp: member of an emitted set (per-scope mode)

__device__ __forceinline__ uint64_t kmin(uint32_t dk, int64_t cid) {  // (d, cid) ascending
  return ((uint64_t)dk << 32) | (uint32_t)cid;
}
__device__ __forceinline__ uint64_t kworst(uint32_t dk, int64_t cid) {  // max = largest d, smallest cid
  return ((uint64_t)dk << 32) | (uint32_t)(~(uint32_t)cid);
}

// Binary heaps in global scratch (one thread).
struct MinHeap {
  uint64_t* k;
  int32_t* v;
  int n;
  __device__ void push(uint64_t key, int32_t val) {
    int i = n++;
    while (i > 0) {
      const int p = (i - 1) >> 1;
      if (k[p] <= key) break;
      k[i] = k[p];
      v[i] = v[p];
      i = p;
    }
    k[i] = key;
    v[i] = val;
  }
  __device__ void pop(uint64_t* key, int32_t* val) {
    *key = k[0];
    *val = v[0];
    const uint64_t lk = k[--n];
    const int32_t lv = v[n];
    int i = 0;
    for (;;) {
      int c = 2 * i + 1;
      if (c >= n) break;
      if (c + 1 < n && k[c + 1] < k[c]) c++;
      if (lk <= k[c]) break;
      k[i] = k[c];
      v[i] = v[c];
      i = c;
    }
    if (n > 0) {
      k[i] = lk;
      v[i] = lv;
    }
  }
};
struct MaxHeap {
  uint64_t* k;
  int32_t* v;
  int n;
  __device__ void push(uint64_t key, int32_t val) {
    int i = n++;
    while (i > 0) {
      const int p = (i - 1) >> 1;
      if (k[p] >= key) break;
      k[i] = k[p];
      v[i] = v[p];
      i = p;
    }
    k[i] = key;
    v[i] = val;
  }
  __device__ void pop() {
    const uint64_t lk = k[--n];
    const int32_t lv = v[n];
    int i = 0;
    for (;;) {
      int c = 2 * i + 1;
      if (c >= n) break;
      if (c + 1 < n && k[c + 1] > k[c]) c++;
      if (lk >= k[c]) break;
      k[i] = k[c];
      v[i] = v[c];
      i = c;
    }
    if (n > 0) {
      k[i] = lk;
      v[i] = lv;
    }
  }
  __device__ uint32_t worst_dk() const { return (uint32_t)(k[0] >> 32); }
};

struct Walk {
  const float* drow;     // exact distances of this query to every slot
  const GraphDev* g;
  const int64_t* cid;    // slot -> cluster id
  uint32_t* stamp;       // [ns] visit stamps of this query
  MinHeap cand;
  MaxHeap best;
  int counter;
  __device__ uint32_t dk(int s) const { return f2key(drow[s]); }
  // neighbors of slot s at `layer` (M entries, -1 padded)
  __device__ const int32_t* nbrs(int s, int layer) const {
    return layer == 0 ? g->nbr0 + (int64_t)s * g->M : g->up + g->up_off[s] + (int64_t)(layer - 1) * g->M;
  }
  // ref/graph.py:125-156 on one scope graph; entries already in best / cand /
  // stamped with `ep`.  Leaves the result set in `best`.
  __device__ void search_layer(int layer, int ef, uint32_t ep) {
    while (cand.n > 0) {
      uint64_t ck;
      int32_t c;
      cand.pop(&ck, &c);
      const uint32_t cdk = (uint32_t)(ck >> 32);
      if (best.n > 0 && cdk > best.worst_dk() && best.n >= ef) break;
      if (layer > g->level[c]) continue;
      const int32_t* nb = nbrs(c, layer);
      for (int j = 0; j < g->M; j++) {
        const int32_t x = nb[j];
        if (x < 0) break;
        if (stamp[x] == ep) continue;
        stamp[x] = ep;
        counter++;
        const uint32_t xk = dk(x);
        if (best.n < ef || xk < best.worst_dk()) {
          cand.push(kmin(xk, cid[x]), x);
          best.push(kworst(xk, cid[x]), x);
          if (best.n > ef) best.pop();
        }
      }
    }
  }
  // greedy descent through layers maxl..1 from `entry` (ef = 1); returns the slot
  __device__ int descend(int entry, int maxl, uint32_t* epoch) {
    int cur = entry;
    for (int layer = maxl; layer >= 1; layer--) {
      const uint32_t ep = ++(*epoch);
      cand.n = best.n = 0;
      stamp[cur] = ep;
      const uint32_t ck = dk(cur);
      cand.push(kmin(ck, cid[cur]), cur);
      best.push(kworst(ck, cid[cur]), cur);
      search_layer(layer, 1, ep);
      cur = best.v[0];  // the single best element
    }
    return cur;
  }
};

__global__ void __launch_bounds__(32) graph_search_kernel(const float* __restrict__ D, int64_t ldd,
                                                          GraphDev g, GraphQuery gq, const int64_t* cid,
                                                          uint32_t* stamps, uint64_t* hk, int32_t* hv,
                                                          int32_t* probe, int32_t* counter_out) {
  const int b = blockIdx.x, lane = threadIdx.x;
  const int ns = g.ns;
  uint32_t* stamp = stamps + (int64_t)b * ns;
  for (int s = lane; s < ns; s += 32) stamp[s] = 0;
  __syncwarp();
  uint32_t emit = 0;
  if (lane == 0) {
    Walk w;
    w.drow = D + (int64_t)b * ldd;
    w.g = &g;
    w.cid = cid;
    w.stamp = stamp;
    // candidate heap: at most one push per node; result heap: <= nodes + 1
    w.cand.k = hk + (int64_t)b * (2 * ns + 2);
    w.cand.v = hv + (int64_t)b * (2 * ns + 2);
    w.best.k = w.cand.k + ns + 1;
    w.best.v = w.cand.v + ns + 1;
    w.counter = 0;
    // ef above the node count behaves as "never full" (best <= visited <= ns)
    const int ef = min(gq.ef, ns);
    uint32_t epoch = 0;
    if (gq.mode == 0) {
      // HybridGraphIndex.search (ref/graph.py:321-396): static entry + greedy
      // descent, the in-scope agent graphs' entries, then one best-first
      // frontier over layer 0 and the portals into expanded scopes
      int nseeds = 0;
      int seeds[1 + GRAPH_MAX_SCOPES];
      if (gq.static_entry >= 0) {
        w.counter++;
        seeds[nseeds++] = w.descend(gq.static_entry, gq.static_maxl, &epoch);
      }
      for (int i = 0; i < gq.n_sc; i++) {
        if (gq.sc_static[i] || gq.sc_entry[i] < 0) continue;
        w.counter++;
        seeds[nseeds++] = gq.sc_entry[i];
      }
      const uint32_t ep = ++epoch;
      w.cand.n = w.best.n = 0;
      for (int i = 0; i < nseeds; i++) {
        const int s = seeds[i];
        if (stamp[s] == ep) continue;
        stamp[s] = ep;
        const uint32_t k = w.dk(s);
        w.cand.push(kmin(k, cid[s]), s);
        w.best.push(kworst(k, cid[s]), s);
      }
      while (w.cand.n > 0) {
        uint64_t ck;
        int32_t c;
        w.cand.pop(&ck, &c);
        const uint32_t cdk = (uint32_t)(ck >> 32);
        if (w.best.n > 0 && cdk > w.best.worst_dk() && w.best.n >= ef) break;
        if (g.level[c] < 0) continue;
        const int32_t* nb = g.nbr0 + (int64_t)c * g.M;
        int m0 = 0;
        while (m0 < g.M && nb[m0] >= 0) m0++;
        const int p0 = g.por_off[c], np = g.por_off[c + 1] - p0;
        for (int j = 0; j < m0 + np; j++) {  // links = neighbors[0] + expanded portals, in order
          const int32_t x = j < m0 ? nb[j] : g.por[p0 + j - m0];
          if (j >= m0 && !(gq.flags[x] & 2)) continue;
          if (stamp[x] == ep) continue;
          stamp[x] = ep;
          w.counter++;
          const uint32_t xk = w.dk(x);
          if (w.best.n < ef || xk < w.best.worst_dk()) {
            w.cand.push(kmin(xk, cid[x]), x);
            w.best.push(kworst(xk, cid[x]), x);
            if (w.best.n > ef) w.best.pop();
          }
        }
      }
      emit = ep;  // emitted: every node this frontier visited (the reference's dists dict)
    } else {
      // HybridGraphIndex.search_independent (ref/graph.py:398-422): one full
      // search per scope graph, the result sets merged
      for (int i = 0; i < gq.n_sc; i++) {
        const int e = gq.sc_entry[i];
        if (e < 0) continue;
        w.counter++;
        const int top = w.descend(e, gq.sc_maxl[i], &epoch);
        const uint32_t ep = ++epoch;
        w.cand.n = w.best.n = 0;
        stamp[top] = ep;
        const uint32_t k = w.dk(top);
        w.cand.push(kmin(k, cid[top]), top);
        w.best.push(kworst(k, cid[top]), top);
        w.search_layer(0, ef, ep);
        for (int t = 0; t < w.best.n; t++) stamp[w.best.v[t]] = EMIT;
      }
      emit = EMIT;
    }
    counter_out[b] = w.counter;
  }
  __syncwarp();  // lane 0's stamps visible to the warp
  emit = __shfl_sync(FULLW, emit, 0);
  // top-nprobe of the emitted in-scope nodes by (d, cid): repeated warp minima
  const float* drow = D + (int64_t)b * ldd;
  uint64_t last = 0;
  for (int p = 0; p < gq.nprobe; p++) {
    uint64_t mk = ~0ull;
    int ms = -1;
    for (int s = lane; s < ns; s += 32) {
      if (stamp[s] != emit || !(gq.flags[s] & 1)) continue;
      const uint64_t k = kmin(f2key(drow[s]), cid[s]);
      if (p > 0 && k <= last) continue;
      if (k < mk) {
        mk = k;
        ms = s;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t k2 = __shfl_xor_sync(FULLW, mk, o);
      const int s2 = __shfl_xor_sync(FULLW, ms, o);
      if (k2 < mk) {
        mk = k2;
        ms = s2;
      }
    }
    if (ms < 0) {  // fewer emitted nodes than nprobe: pad
      for (int r = p + lane; r < gq.nprobe; r += 32) probe[(int64_t)b * gq.nprobe + r] = -1;
      break;
    }
    if (lane == 0) probe[(int64_t)b * gq.nprobe + p] = ms;
    last = mk;
  }
}

}  // namespace

void launch_graph_search(const float* D, int64_t ldd, int B, const GraphDev& g, const GraphQuery& gq,
                         const int64_t* cid, uint32_t* stamps, uint64_t* hk, int32_t* hv, int32_t* probe,
                         int32_t* counter, cudaStream_t st) {
  if (B <= 0) return;
  graph_search_kernel<<<B, 32, 0, st>>>(D, ldd, g, gq, cid, stamps, hk, hv, probe, counter);
}

}  // namespace pk
