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
// One CTA per query: lane 0 of warp 0 runs the sequential traversal (the
// reference's own control flow is sequential: each admission changes the
// bound the next one reads), warp 0 selects the emitted top-nprobe.  The
// traversal's reads are a chain of dependent loads (pop -> slot -> level /
// neighbors -> their ranks), so when the graph fits, the whole CTA first
// stages it into shared memory -- layer-0 neighbor lists, ranks, levels,
// portals, flags and the distance row -- and every hop of the walk costs a
// shared-memory latency instead of an L2 round trip (an agent search at
// ~2K lists: 368 -> tens of microseconds).
#include "pk_kernels.h"
#include "pk_ptx.cuh"

namespace pk {

namespace {

constexpr unsigned FULLW = 0xffffffffu;
constexpr uint32_t EMIT = 0xfffffffeu;  // stamp: member of an emitted set (per-scope mode)

// Heap keys: (order-preserving f32 bits of d) << 32 | rank, where rank is the
// position of the list's cid among the live cids (pk_graph_set), so key order
// is (d, cid) order and the low half names the node.
__device__ __forceinline__ uint64_t kmin(uint32_t dk, uint32_t rank) { return ((uint64_t)dk << 32) | rank; }
// result heap (max-heap): largest d first, ties to the SMALLEST cid
__device__ __forceinline__ uint64_t kworst(uint32_t dk, uint32_t rank) {
  return ((uint64_t)dk << 32) | (uint32_t)(~rank);
}

// Binary heaps of 64-bit keys (one thread; shared memory when it fits).
struct MinHeap {
  uint64_t* k;
  int n;
  __device__ void push(uint64_t key) {
    int i = n++;
    while (i > 0) {
      const int p = (i - 1) >> 1;
      const uint64_t kp = k[p];
      if (kp <= key) break;
      k[i] = kp;
      i = p;
    }
    k[i] = key;
  }
  __device__ uint64_t pop() {
    const uint64_t top = k[0];
    const uint64_t lk = k[--n];
    int i = 0;
    for (;;) {
      int c = 2 * i + 1;
      if (c >= n) break;
      uint64_t kc = k[c];
      if (c + 1 < n) {
        const uint64_t k1 = k[c + 1];
        if (k1 < kc) {
          kc = k1;
          c++;
        }
      }
      if (lk <= kc) break;
      k[i] = kc;
      i = c;
    }
    if (n > 0) k[i] = lk;
    return top;
  }
};
struct MaxHeap {
  uint64_t* k;
  int n;
  __device__ void push(uint64_t key) {
    int i = n++;
    while (i > 0) {
      const int p = (i - 1) >> 1;
      const uint64_t kp = k[p];
      if (kp >= key) break;
      k[i] = kp;
      i = p;
    }
    k[i] = key;
  }
  __device__ void pop() {
    const uint64_t lk = k[--n];
    int i = 0;
    for (;;) {
      int c = 2 * i + 1;
      if (c >= n) break;
      uint64_t kc = k[c];
      if (c + 1 < n) {
        const uint64_t k1 = k[c + 1];
        if (k1 > kc) {
          kc = k1;
          c++;
        }
      }
      if (lk >= kc) break;
      k[i] = kc;
      i = c;
    }
    if (n > 0) k[i] = lk;
  }
  __device__ uint32_t worst_dk() const { return (uint32_t)(k[0] >> 32); }
};

struct Walk {
  const float* drow;      // exact distances of this query to every slot
  GraphDev g;  // by value (no address-taken local: it would live in local memory)
  uint32_t* stamp;        // [ns] visit stamps of this query
  MinHeap cand;
  MaxHeap best;
  int counter;
  __device__ uint32_t dk(int s) const { return f2key(drow[s]); }
  __device__ uint32_t rk(int s) const { return (uint32_t)g.rank[s]; }
  __device__ int slot_of(uint64_t key) const { return g.slot_of_rank[(uint32_t)key]; }
  __device__ const int32_t* nbrs(int s, int layer) const {
    return layer == 0 ? g.nbr0 + (int64_t)s * g.M : g.up + g.up_off[s] + (int64_t)(layer - 1) * g.M;
  }
  __device__ void seed(int s, uint32_t ep) {
    stamp[s] = ep;
    const uint32_t k = dk(s);
    cand.push(kmin(k, rk(s)));
    best.push(kworst(k, rk(s)));
  }
  // visit the links of one expanded node in order (the per-link body of
  // ref/graph.py:146-155 and :381-390); `n` links, x(j) the j-th
  template <typename LinkF>
  __device__ void visit(int n, LinkF link, int ef, uint32_t ep) {
    for (int j0 = 0; j0 < n; j0 += 8) {
      // the distances of up to 8 links are independent loads: issue together
      int xs[8];
      uint32_t ks[8];
#pragma unroll
      for (int u = 0; u < 8; u++) xs[u] = j0 + u < n ? link(j0 + u) : -1;
#pragma unroll
      for (int u = 0; u < 8; u++) ks[u] = xs[u] >= 0 ? dk(xs[u]) : 0u;
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int x = xs[u];
        if (x < 0 || stamp[x] == ep) continue;
        stamp[x] = ep;
        counter++;
        if (best.n < ef || ks[u] < best.worst_dk()) {
          cand.push(kmin(ks[u], rk(x)));
          best.push(kworst(ks[u], rk(x)));
          if (best.n > ef) best.pop();
        }
      }
    }
  }
  // ref/graph.py:125-156 on one scope graph; entries already seeded with `ep`.
  // Leaves the result set in `best`.
  __device__ void search_layer(int layer, int ef, uint32_t ep) {
    while (cand.n > 0) {
      const uint64_t ck = cand.pop();
      if (best.n > 0 && (uint32_t)(ck >> 32) > best.worst_dk() && best.n >= ef) break;
      const int c = slot_of(ck);
      if (layer > g.level[c]) continue;
      const int32_t* nb = nbrs(c, layer);
      int m = 0;
      while (m < g.M && nb[m] >= 0) m++;
      visit(m, [&](int j) { return (int)nb[j]; }, ef, ep);
    }
  }
  // greedy descent through layers maxl..1 from `entry` (ef = 1); returns the slot
  __device__ int descend(int entry, int maxl, uint32_t* epoch) {
    int cur = entry;
    for (int layer = maxl; layer >= 1; layer--) {
      const uint32_t ep = ++(*epoch);
      cand.n = best.n = 0;
      seed(cur, ep);
      search_layer(layer, 1, ep);
      cur = slot_of(~best.k[0] & 0xffffffffull);  // the single result element
    }
    return cur;
  }
};

// The same walk with the whole warp (ef <= 32): the result set lives in
// registers as an ascending array of (-d, cid)-ordered keys, one per lane
// (insertion = ballot + shuffle, the worst element = lane n-1), the links of
// an expansion are loaded, de-duplicated and stamped by 32 lanes at once, and
// only the admissions -- each reads the bound the previous one moved -- and
// the candidate heap stay sequential (lane 0 owns the heap).  Every decision
// is the single-thread walk's.
struct WarpWalk {
  const float* drow;
  GraphDev g;  // by value: its pointers stay in registers (an address-taken
               // local would live in local memory, one load per hop)
  uint32_t* stamp;
  // candidates: an unsorted array (shared memory) -- the pop is a warp
  // argmin (keys are unique), the hole refilled from the end; cheaper than a
  // one-lane binary heap at the sizes an ef <= 32 walk reaches
  uint64_t* ck;
  int cn;
  uint64_t bv;   // this lane's result-set element (valid when lane < bn)
  int bn;
  int counter;
  int lane;
  __device__ __forceinline__ uint32_t dk(int s) const { return f2key(drow[s]); }
  __device__ __forceinline__ uint32_t worst_dk() const { return (uint32_t)(__shfl_sync(FULLW, bv, bn - 1) >> 32); }
  __device__ __forceinline__ void best_insert(uint64_t k, int ef) {
    const bool less = lane < bn && bv < k;
    const int pos = __popc(__ballot_sync(FULLW, less));
    const uint64_t up = __shfl_up_sync(FULLW, bv, 1);
    if (lane > pos) bv = up;
    if (lane == pos) bv = k;
    bn = min(bn + 1, ef);  // full: the old worst fell off the end
  }
  __device__ __forceinline__ void cand_push(uint64_t k) {
    if (lane == 0) ck[cn] = k;
    cn++;
  }
  // the smallest candidate, removed; ~0 when none is left (no key is all
  // ones: ranks are below the slot count).  Returned by value: an
  // out-parameter would put the key in local memory on every pop.
  __device__ __forceinline__ uint64_t cand_pop() {
    __syncwarp();
    if (cn == 0) return ~0ull;
    uint64_t best = ~0ull;
    int bi = 0;
    for (int i = lane; i < cn; i += 32) {
      const uint64_t v = ck[i];
      if (v < best) {
        best = v;
        bi = i;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t ob = __shfl_xor_sync(FULLW, best, o);
      const int oi = __shfl_xor_sync(FULLW, bi, o);
      if (ob < best) {
        best = ob;
        bi = oi;
      }
    }
    __syncwarp();
    if (lane == 0) ck[bi] = ck[cn - 1];
    cn--;
    return best;
  }
  __device__ __forceinline__ void seed(int s, uint32_t ep, int ef) {
    if (lane == 0) stamp[s] = ep;
    __syncwarp();
    const uint32_t k = dk(s), r = (uint32_t)g.rank[s];
    cand_push(kmin(k, r));
    best_insert(kworst(k, r), ef);
  }
  // links of one expanded node, in order (x(j) < 0: not a link)
  template <typename LinkF>
  __device__ __forceinline__ void visit(int nl, LinkF link, int ef, uint32_t ep) {
    for (int j0 = 0; j0 < nl; j0 += 32) {
      const int j = j0 + lane;
      const int x = j < nl ? link(j) : -1;
      bool fresh = x >= 0 && stamp[x] != ep;
      const unsigned same = __match_any_sync(FULLW, x);
      if (fresh && __ffs(same) - 1 != lane) fresh = false;  // a repeat of an earlier link
      unsigned fm = __ballot_sync(FULLW, fresh);
      uint32_t k = 0, r = 0;
      if (fresh) {
        stamp[x] = ep;
        k = dk(x);
        r = (uint32_t)g.rank[x];
      }
      counter += __popc(fm);
      while (fm) {  // admissions in link order
        const int L = __ffs(fm) - 1;
        fm &= fm - 1;
        const uint32_t kL = __shfl_sync(FULLW, k, L), rL = __shfl_sync(FULLW, r, L);
        if (bn < ef || kL < worst_dk()) {
          cand_push(kmin(kL, rL));
          best_insert(kworst(kL, rL), ef);
        }
      }
      __syncwarp();  // stamps visible to the next chunk
    }
  }
  __device__ __forceinline__ int slot_of(uint64_t key) const { return g.slot_of_rank[(uint32_t)key]; }
  __device__ __forceinline__ const int32_t* nbrs(int s, int layer) const {
    return layer == 0 ? g.nbr0 + (int64_t)s * g.M : g.up + g.up_off[s] + (int64_t)(layer - 1) * g.M;
  }
  __device__ __forceinline__ int degree(const int32_t* nb) const {  // valid prefix of a -1 padded neighbor list
    const unsigned v = __ballot_sync(FULLW, lane < g.M && nb[min(lane, g.M - 1)] >= 0);
    const unsigned inv = ~v & ((g.M >= 32) ? FULLW : ((1u << g.M) - 1u));
    return inv ? __ffs(inv) - 1 : g.M;
  }
  __device__ __forceinline__ void search_layer(int layer, int ef, uint32_t ep) {
    for (uint64_t ck = cand_pop(); ck != ~0ull; ck = cand_pop()) {
      if (bn > 0 && (uint32_t)(ck >> 32) > worst_dk() && bn >= ef) break;
      const int c = slot_of(ck);
      if (layer > g.level[c]) continue;
      const int32_t* nb = nbrs(c, layer);
      const int m = degree(nb);
      visit(m, [&](int jj) { return (int)nb[jj]; }, ef, ep);
    }
  }
  uint32_t epoch;  // visit-stamp epoch (a member: no address-taken local)
  __device__ __forceinline__ int descend(int entry, int maxl) {
    int cur = entry;
    for (int layer = maxl; layer >= 1; layer--) {
      const uint32_t ep = ++epoch;
      cn = 0;
      bn = 0;
      seed(cur, ep, 1);
      search_layer(layer, 1, ep);
      cur = slot_of(~__shfl_sync(FULLW, bv, 0) & 0xffffffffull);
    }
    return cur;
  }
};

// dynamic shared memory per CTA (one query): stamps u32[ns], two heaps u64[ns + 1],
// and the distance row f32[ns] when `smem_row`
constexpr int GRAPH_THREADS = 256;

__global__ void __launch_bounds__(GRAPH_THREADS, 1) graph_search_kernel(const float* __restrict__ D, int64_t ldd,
                                                          GraphDev g0, GraphQuery gq, int smem_heaps,
                                                          int smem_row, int smem_graph, uint32_t* gstamps,
                                                          uint64_t* gheap, int32_t* probe, int32_t* counter_out) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int b = blockIdx.x, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int ns = g0.ns;
  uint64_t* heaps = smem_heaps ? reinterpret_cast<uint64_t*>(sm) : gheap + (int64_t)b * (2 * ns + 2);
  uint32_t* stamp = smem_heaps ? reinterpret_cast<uint32_t*>(sm + (size_t)(2 * ns + 2) * 8)
                               : gstamps + (int64_t)b * ns;
  const float* drow_g = D + (int64_t)b * ldd;
  float* srow = reinterpret_cast<float*>(sm + (size_t)(2 * ns + 2) * 8 + (size_t)ns * 4);
  GraphDev g = g0;
  // the scope flags (staged below); the kernel parameter gq stays read-only,
  // so it is read from the parameter bank rather than copied to local memory
  const uint8_t* flags = gq.flags;
  if (smem_graph) {  // the walk's arrays, after the heaps / stamps / row
    uint8_t* p = sm + (((size_t)(2 * ns + 2) * 8 + (size_t)ns * 8 + 15) & ~(size_t)15);
    int32_t* nb = reinterpret_cast<int32_t*>(p);
    p += (size_t)ns * g0.M * 4;
    int32_t* rk = reinterpret_cast<int32_t*>(p);
    p += (size_t)ns * 4;
    int32_t* sr = reinterpret_cast<int32_t*>(p);
    p += (size_t)ns * 4;
    int8_t* lv = reinterpret_cast<int8_t*>(p);
    p += (size_t)ns;
    uint8_t* fl = p;
    p += (size_t)ns;
    p = reinterpret_cast<uint8_t*>(((uintptr_t)p + 15) & ~(uintptr_t)15);
    int32_t* po = reinterpret_cast<int32_t*>(p);  // portals: only when smem_graph == 2
    p += (size_t)(ns + 1) * 4;
    int32_t* pv = reinterpret_cast<int32_t*>(p);
    const int n4 = ns * g0.M / 4;  // M is a multiple of 4 (pk_graph_set pads)
    for (int i = tid; i < n4; i += GRAPH_THREADS)
      reinterpret_cast<int4*>(nb)[i] = reinterpret_cast<const int4*>(g0.nbr0)[i];
    for (int i = 4 * n4 + tid; i < ns * g0.M; i += GRAPH_THREADS) nb[i] = g0.nbr0[i];
    for (int i = tid; i < ns; i += GRAPH_THREADS) {
      rk[i] = g0.rank[i];
      sr[i] = g0.slot_of_rank[i];
      lv[i] = g0.level[i];
      fl[i] = gq.flags[i];
    }
    if (smem_graph == 2) {
      for (int i = tid; i <= ns; i += GRAPH_THREADS) po[i] = g0.por_off[i];
      for (int i = tid; i < g0.npor; i += GRAPH_THREADS) pv[i] = g0.por[i];
      g.por_off = po;
      g.por = pv;
    }
    g.nbr0 = nb;
    g.rank = rk;
    g.slot_of_rank = sr;
    g.level = lv;
    flags = fl;
  }
  for (int s = tid; s < ns; s += GRAPH_THREADS) {
    stamp[s] = 0;
    if (smem_row) srow[s] = drow_g[s];
  }
  __syncthreads();
  if (tid >= 32) return;
  uint32_t emit = 0;
  if (gq.warp) {
    // ef <= 32 and no more seeds than ef: the warp walk
    WarpWalk w;
    w.drow = smem_row ? srow : drow_g;
    w.g = g;
    w.stamp = stamp;
    w.ck = heaps;
    w.cn = 0;
    w.bn = 0;
    w.bv = 0;
    w.counter = 0;
    w.lane = lane;
    w.epoch = 0;
    const int ef = min(gq.ef, ns);
    if (gq.mode == 0) {
      int nseeds = 0;
      int seeds[1 + GRAPH_MAX_SCOPES];
      if (gq.static_entry >= 0) {
        w.counter++;
        seeds[nseeds++] = w.descend(gq.static_entry, gq.static_maxl);
      }
      for (int i = 0; i < gq.n_sc; i++) {
        if (gq.sc_static[i] || gq.sc_entry[i] < 0) continue;
        w.counter++;
        seeds[nseeds++] = gq.sc_entry[i];
      }
      const uint32_t ep = ++w.epoch;
      w.cn = 0;
      w.bn = 0;
      for (int i = 0; i < nseeds; i++) {
        __syncwarp();
        if (stamp[seeds[i]] != ep) w.seed(seeds[i], ep, ef);
      }
      for (uint64_t ck = w.cand_pop(); ck != ~0ull; ck = w.cand_pop()) {
        if (w.bn > 0 && (uint32_t)(ck >> 32) > w.worst_dk() && w.bn >= ef) break;
        const int c = w.slot_of(ck);
        if (g.level[c] < 0) continue;
        const int32_t* nb = g.nbr0 + (int64_t)c * g.M;
        const int m = w.degree(nb);
        const int p0 = g.por_off[c], np = g.por_off[c + 1] - p0;
        w.visit(m + np, [&](int j) {
          const int x = j < m ? (int)nb[j] : (int)g.por[p0 + j - m];
          return (j < m || (flags[x] & 2)) ? x : -1;
        }, ef, ep);
      }
      emit = ep;
    } else {
      for (int i = 0; i < gq.n_sc; i++) {
        const int e = gq.sc_entry[i];
        if (e < 0) continue;
        w.counter++;
        const int top = w.descend(e, gq.sc_maxl[i]);
        const uint32_t ep = ++w.epoch;
        w.cn = 0;
        w.bn = 0;
        w.seed(top, ep, ef);
        w.search_layer(0, ef, ep);
        __syncwarp();
        if (lane < w.bn) stamp[w.slot_of(~w.bv & 0xffffffffull)] = EMIT;
        __syncwarp();
      }
      emit = EMIT;
    }
    if (lane == 0) counter_out[b] = w.counter;
  } else if (lane == 0) {
    Walk w;
    w.drow = smem_row ? srow : drow_g;
    w.g = g;
    w.stamp = stamp;
    // candidate heap: at most one push per node; result heap: <= nodes + 1
    w.cand.k = heaps;
    w.best.k = heaps + ns + 1;
    w.cand.n = w.best.n = 0;
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
      for (int i = 0; i < nseeds; i++)
        if (stamp[seeds[i]] != ep) w.seed(seeds[i], ep);
      while (w.cand.n > 0) {
        const uint64_t ck = w.cand.pop();
        if (w.best.n > 0 && (uint32_t)(ck >> 32) > w.best.worst_dk() && w.best.n >= ef) break;
        const int c = w.slot_of(ck);
        if (g.level[c] < 0) continue;
        const int32_t* nb = g.nbr0 + (int64_t)c * g.M;
        int m = 0;
        while (m < g.M && nb[m] >= 0) m++;
        const int p0 = g.por_off[c], np = g.por_off[c + 1] - p0;
        // links = neighbors[0] + the portals into expanded scopes, in order
        w.visit(m + np, [&](int j) {
          const int x = j < m ? (int)nb[j] : (int)g.por[p0 + j - m];
          return (j < m || (flags[x] & 2)) ? x : -1;
        }, ef, ep);
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
        w.seed(top, ep);
        w.search_layer(0, ef, ep);
        for (int t = 0; t < w.best.n; t++) stamp[w.slot_of(~w.best.k[t] & 0xffffffffull)] = EMIT;
      }
      emit = EMIT;
    }
    counter_out[b] = w.counter;
  }
  __syncwarp();  // lane 0's stamps visible to the warp
  emit = __shfl_sync(FULLW, emit, 0);
  // top-nprobe of the emitted in-scope nodes by (d, cid): the emitted keys are
  // compacted once into the (now free) heap space, then repeated warp minima
  // run over that short list instead of every slot
  const float* drow = smem_row ? srow : drow_g;
  uint64_t* ek = heaps;
  int ne = 0;
  for (int s0 = 0; s0 < ns; s0 += 32) {
    const int s = s0 + lane;
    const bool hit = s < ns && stamp[s] == emit && (flags[s] & 1);
    const unsigned m = __ballot_sync(FULLW, hit);
    if (hit) ek[ne + __popc(m & ((1u << lane) - 1u))] = kmin(f2key(drow[s]), (uint32_t)g.rank[s]);
    ne += __popc(m);
  }
  __syncwarp();
  uint64_t last = 0;
  for (int p = 0; p < gq.nprobe; p++) {
    uint64_t mk = ~0ull;
    for (int i = lane; i < ne; i += 32) {
      const uint64_t k = ek[i];
      if (p > 0 && k <= last) continue;
      mk = k < mk ? k : mk;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t k2 = __shfl_xor_sync(FULLW, mk, o);
      mk = k2 < mk ? k2 : mk;
    }
    if (mk == ~0ull) {  // fewer emitted nodes than nprobe: pad
      for (int r = p + lane; r < gq.nprobe; r += 32) probe[(int64_t)b * gq.nprobe + r] = -1;
      break;
    }
    if (lane == 0) probe[(int64_t)b * gq.nprobe + p] = g.slot_of_rank[(uint32_t)mk];
    last = mk;
  }
}

}  // namespace

size_t graph_smem_bytes(int ns, bool row) {
  return (size_t)(2 * ns + 2) * 8 + (size_t)ns * 4 + (row ? (size_t)ns * 4 : 0);
}
// the walk's per-hop arrays (neighbors, ranks, levels, flags) [+ portals]
static size_t graph_stage_bytes(const GraphDev& g, bool portals) {
  return 32 + (size_t)g.ns * g.M * 4 + (size_t)g.ns * 8 + (size_t)g.ns * 2 +
         (portals ? (size_t)(g.ns + 1) * 4 + (size_t)g.npor * 4 : 0);
}

void launch_graph_search(const float* D, int64_t ldd, int B, const GraphDev& g, const GraphQuery& gq,
                         uint32_t* gstamps, uint64_t* gheap, int32_t* probe, int32_t* counter,
                         cudaStream_t st) {
  if (B <= 0) return;
  constexpr size_t SMEM_MAX = 227 * 1024;
  int heaps = 1, row = 1, stage = 0;
  size_t smem = graph_smem_bytes(g.ns, true);
  if (smem + graph_stage_bytes(g, true) <= SMEM_MAX && g.M % 4 == 0) {
    stage = 2;
    smem += graph_stage_bytes(g, true);
  } else if (smem + graph_stage_bytes(g, false) <= SMEM_MAX && g.M % 4 == 0) {
    stage = 1;
    smem += graph_stage_bytes(g, false);
  } else if (smem > SMEM_MAX) {
    row = 0;
    smem = graph_smem_bytes(g.ns, false);
  }
  if (smem > SMEM_MAX) {
    heaps = 0;
    smem = 16;
  }
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    cudaFuncSetAttribute(graph_search_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_MAX);
    attr = SMEM_MAX;
  }
  // the warp walk holds the result set in registers (ef <= 32, one element
  // per lane) and needs every seed to fit in it (PK_GRAPH_WARP=0: off)
  static const bool warp_ok = !getenv("PK_GRAPH_WARP") || atoi(getenv("PK_GRAPH_WARP")) != 0;
  GraphQuery q2 = gq;
  const int ef = std::min(gq.ef, g.ns);
  q2.warp = warp_ok && ef <= 32 && g.M <= 32 && (gq.mode == 1 || 1 + gq.n_sc <= ef);
  graph_search_kernel<<<B, GRAPH_THREADS, smem, st>>>(D, ldd, g, q2, heaps, row, stage, gstamps, gheap, probe,
                                                      counter);
}

}  // namespace pk
