// pk_kernels.h -- launch interface of the sm_100a kernels (host side).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace pk {

enum Metric : int { SQ_L2 = 0, IP = 1, COSINE = 2 };

constexpr int DC = 32;          // floats per streamed d-chunk (one 128B swizzle row)
constexpr int TILE = 256;       // rows per scan tile (one row per compute thread)
constexpr int QG = 16;          // queries per scan work item
constexpr int KKMAX = 64;       // max per-query candidates kept by scan / merge
constexpr int STAGES = 4;       // TMA pipeline depth
constexpr int NBOX = 6;         // TMA box heights 256,128,64,32,16,8

// One posting-list work item: rows [row0, row0+nrows) of list `lslot`,
// against queries qpairs[qoff .. qoff+nq).
struct ScanItem {
  int32_t lslot;
  int32_t row0;
  int32_t nrows;
  int32_t qoff;
  int32_t nq;
  int32_t chunk;
  int32_t pad0, pad1;
};
struct QPair {  // query index and the base of its output slots for this list
  int32_t b;
  int32_t slotbase;
};

struct ArenaMaps {
  CUtensorMap box[NBOX];  // heights 256,128,64,32,16,8 rows x DC floats, SWIZZLE_128B
};

// Device view of the list table and arena.
struct ListTable {
  const float* rows;     // [arena_rows][dp]
  const int64_t* ids;    // [arena_rows]
  const int64_t* off;    // [nslots] first arena row of list
  const int64_t* len;    // [nslots] live rows
  const int64_t* cid;    // [nslots] cluster id (-1 = empty slot)
  const int32_t* scope;  // [nslots] scope code
  const float* cent;     // [nslots][dp]
  const float* nrm;      // [arena_rows] squared row norms (FFMA; tensor-core screen input)
  int32_t nslots;
  int32_t dp;            // padded row stride (multiple of DC)
  int32_t d;             // true dimension
  int32_t metric;        // the index metric (output sign of zero distances)
};

// ---- launchers (all async on `st`) ----
// D[b][r] = dist(Q[b], X[r]) exact reference arithmetic; Q: [B][ldq], X: [n][ldx].
void launch_dist_dense(int metric, const float* Q, int64_t ldq, int B, const float* X, int64_t ldx,
                       int64_t n, int dp, const float* qnorm, float* D, int64_t ldd,
                       cudaStream_t st);
// assign_nearest in ONE launch: distances of B rows of Q to the n centroid
// slots of C with the argmin by (dist, cid) over the slots of scope_code fused
// in (block minima in part[], the last block reduces; counter starts at 0 and
// is left at 0).  Requires cids < 2^32.  part needs dense_argmin_blocks(n, B)
// entries.
int dense_argmin_blocks(int64_t n, int B);
void launch_dense_argmin(int metric, const float* Q, int64_t ldq, int B, const float* C, int64_t n, int dp,
                         const float* qnorm, ListTable lt, int32_t scope_code, unsigned long long* part,
                         unsigned* counter, int64_t* out_cid, float* out_d, cudaStream_t st);
// kmeans_assign arithmetic (fp32 square, fp64 sum), fused argmin over k rows of C.
void launch_kmeans_assign(const float* X, int64_t ldx, int64_t n, const float* C, int64_t ldc,
                          int64_t k, int dp, int64_t* labels, double* dists, cudaStream_t st);
// qnorm[b] = sqrt(sum_j q_j*q_j) sequential fp32 (cosine only).
void launch_qnorm(const float* Q, int64_t ldq, int B, int d, float* qnorm, cudaStream_t st);
// centroid = fp64 row-order mean of rows [off, off+n) -> f32 (written to cent_out[dp]).
void launch_centroid(const float* rows, int64_t ldr, int64_t n, int dp, float* cent_out,
                     cudaStream_t st);
// Per-segment fp64 row-order mean (k-means update): segment c = rows [off[c], off[c+1]).
void launch_seg_centroid(const float* rows, int64_t ldr, const int64_t* off, int k, int d, float* out,
                         cudaStream_t st);
// Coarse select: per query the first `nprobe` in-scope lists by (dist, cid).
void launch_coarse_select(const float* Dc, int64_t ldd, int B, ListTable lt,
                          const int32_t* scope_codes, int nscopes, int nprobe, int32_t* probe,
                          uint32_t* probe_key, cudaStream_t st);
// Build the (list -> queries) routing and the scan work items: per query
// slots [slot_off[2b], slot_off[2b+1]) (stride smax), per list a bucket of
// bcap (query, slot base) pairs.  lcount [nslots] and *n_items must be zero.
void launch_route(const int32_t* probe, int B, int nprobe, ListTable lt, int chunk_rows, int smax,
                  int bcap, int32_t* lcount, ScanItem* items, int32_t* n_items, QPair* bucket,
                  int32_t* slot_off, int64_t* scanned, bool emitted, int max_items, cudaStream_t st);
// Routing outputs for a kernel that emits its queries' routes itself (lcount
// NULL = no routing).
struct RouteArgs {
  int32_t* lcount = nullptr;
  QPair* bucket = nullptr;
  int32_t* slot_off = nullptr;
  int64_t* scanned = nullptr;
  int chunk_rows = 0, smax = 0, bcap = 0;
  // nonzero: only the probe SET matters (no caller reads the probe order or
  // keys), so lists certainly in the first nprobe skip the exact re-rank
  int unordered = 0;
};
// Persistent fused scan + per-(query, item) top-kk.
void launch_scan(int metric, ListTable lt, const ArenaMaps& maps, const float* Qd,
                 const float* qnorm, const ScanItem* items, const int32_t* n_items,
                 int max_items, const QPair* qpairs, int kk, int32_t* work_ctr,
                 uint32_t* cand_key, int64_t* cand_id, int32_t* cand_n, int32_t* cand_list,
                 int num_sms, cudaStream_t st);
// Per query merge of its slots into the final top-kk (dedup by id).
void launch_merge(int B, const int32_t* slot_off, const uint32_t* cand_key, const int64_t* cand_id,
                  const int32_t* cand_n, const int32_t* cand_list, int kk, ListTable lt,
                  int64_t* out_ids, float* out_d, int64_t* out_cid, int32_t* out_n,
                  cudaStream_t st);
// Row argmin over the live lists of one scope by (dist, cid) -- assign_nearest (ref/clusters.py:268-279).
void launch_argmin(const float* D, int64_t ldd, int B, ListTable lt, int32_t scope_code,
                   int64_t* out_cid, float* out_d, cudaStream_t st);
// Scatter rows: dst[dst_row[i]] = src[i] (rows of dp floats) and ids.
void launch_scatter_rows(const float* src, int64_t lds, const int64_t* src_ids, int n,
                         const int64_t* dst_row, float* dst, int64_t* dst_ids, int dp,
                         cudaStream_t st);
// ---- hybrid coarse graph (pk_graph.cu): the reference's graph traversal
constexpr int GRAPH_MAX_SCOPES = 64;
struct GraphDev {          // slot-indexed, uploaded by pk_graph_set
  const int8_t* level;     // [ns] node level, -1 = not a graph node
  const int32_t* nbr0;     // [ns][M] layer-0 neighbors (slots, list order, -1 padded)
  const int32_t* up_off;   // [ns] offset of the node's layer-1 block in up[]
  const int32_t* up;       // layers 1..level, M entries each
  const int32_t* por_off;  // [ns + 1] portal CSR
  const int32_t* por;      // portal targets (slots, insertion order)
  const int32_t* rank;     // [ns] position of the slot's cid among the live cids (tie order)
  const int32_t* slot_of_rank;  // [ns]
  int M;
  int ns;
  int npor;                // portal entries (por[] length)
};
struct GraphQuery {        // one batch's scope set
  const uint8_t* flags;    // [ns] bit0: list in the searched scopes, bit1: in scopes + static
  int static_entry, static_maxl;  // static graph entry slot (-1: empty)
  int n_sc;                // searched scopes (any order; the traversal is order-free)
  int sc_entry[GRAPH_MAX_SCOPES], sc_maxl[GRAPH_MAX_SCOPES];
  uint8_t sc_static[GRAPH_MAX_SCOPES];
  int ef, nprobe, mode;    // mode 0: search (hybrid), 1: search_independent (per_agent)
  int warp;                // the warp walk (set by the launcher when ef and the seed count allow)
};
// probe[b][nprobe] (slots, (d, cid) order, -1 padded), counter[b] = distance
// computations; D = exact distances [B][ldd] to every slot's centroid.
// Global scratch (used only when the per-query state exceeds shared memory):
// stamps [B][ns] u32, heaps [B][2 ns + 2] u64.
void launch_graph_search(const float* D, int64_t ldd, int B, const GraphDev& g, const GraphQuery& gq,
                         uint32_t* gstamps, uint64_t* gheap, int32_t* probe, int32_t* counter,
                         cudaStream_t st);
size_t graph_smem_bytes(int ns, bool row);
size_t scan_smem_bytes();
size_t screen_smem_bytes();
// Screened persistent scan (sq_l2 / neg_ip): FFMA screen with a proven error
// bound.  Per (query, item) slot: the item's kk smallest upper bounds
// (slot_hi[slot][..slot_n]); per query: running bound Uq (KEY_NONE-initialised)
// and the pool of rows that can still reach the top-kk (cpool[b][0..cap):
// arena row, list slot, lower-bound key; count ccount[b], zero-initialised).
void launch_scan_screen(int metric, ListTable lt, const ArenaMaps& maps, const float* Qd,
                        const float* qnorm2, const ScanItem* items, const int32_t* n_items,
                        int max_items, const QPair* qpairs, int kk, int32_t* work_ctr,
                        uint32_t* Uq, uint32_t* slot_hi, int32_t* slot_n, int4* cpool,
                        int32_t* ccount, int cap, int num_sms, cudaStream_t st);
// Per query: global bound from the slots, exact re-rank of the surviving pool
// entries, top-kk merge (one CTA per query).
void launch_rerank_merge(int metric, int B, const int4* cpool, const int32_t* ccount, int cap,
                         const uint32_t* slot_hi, const int32_t* slot_n, const int32_t* slot_off,
                         ListTable lt, const float* Qd, const int32_t* probe, int nprobe, int kk,
                         int64_t* out_ids, float* out_d, int64_t* out_cid, int32_t* out_n,
                         int32_t* nsurv, const int64_t* scanned_src, int64_t* scanned_dst,
                         cudaStream_t st, bool pdl = true, int lean_ctas = 0);
// lean_ctas > 0: the co-resident configuration (a persistent grid of at most
// lean_ctas CTAs that fit beside the scan); whether it fits for this dp
bool rerank_lean_fits(int dp);
float screen_coef(int metric, int dp);
float screen_coef_tf32(int metric, int dp);
size_t tc_smem_bytes();
// Row squared norms for the arena (tensor-core screen input).
void launch_row_norms(const float* rows, int64_t n, int dp, float* out, cudaStream_t st);
// Tensor-core screened persistent scan (tcgen05 TF32); same outputs as
// launch_scan_screen.  qsw: scratch of 8 * B * dp floats.
void launch_scan_tc(int metric, ListTable lt, const ArenaMaps& maps, const float* Qd, int B,
                    float* qsw, bool qsw_ready, const float* qnorm2, const ScanItem* items,
                    const int32_t* n_items, int max_items, const QPair* qpairs, int kk,
                    int32_t* work_ctr, uint32_t* Uq, uint32_t* slot_hi, int32_t* slot_n, int4* cpool,
                    int32_t* ccount, int cap, int num_sms, cudaStream_t st, bool pdl = true,
                    const CUtensorMap* qgather = nullptr, bool overlapped = false);

// Cross-shard merge of R per-shard result blocks (layout: pk_shard_block_bytes
// in include/pancake_b200.h) into the global top-kk per query.
int shard_merge_cap();
void launch_reblock(const int64_t* ids, const int64_t* cids, const int64_t* sc, const float* d,
                    const int32_t* n, int B, int group, int kk, int64_t block_bytes, void* dst,
                    cudaStream_t st);
void launch_shard_merge(int metric, const void* blocks, int64_t block_bytes, int R, int B, int kk,
                        int64_t* out_ids, float* out_d, int64_t* out_cid, int32_t* out_n,
                        int64_t* out_scanned, cudaStream_t st);

// Coarse quantizer on tcgen05: screened distances A[b][slot] for every slot
// (TF32 UMMA, cmap over the centroid table, qmap over the padded batch).
struct CoarseMaps {
  CUtensorMap c[2];  // centroid table: [0] fp32 or TF32 hi part, [1] lo part (split)
  CUtensorMap q[2];  // padded batch, same split
};
size_t coarse_tc_smem_bytes(bool split);
// Split-K factor for the coarse GEMM (grid ~ one CTA per SM).
int coarse_split_k(int nslots, int B, int dp, int num_sms);
// Dout[z][b][slot] = partial dot over K range z of ks (the pick sums them in z order).
void launch_coarse_tc(bool split, int ks, const CoarseMaps& maps, int nslots, int B, int dp,
                      float* Dout, int64_t lda, cudaStream_t st);
// One-pass query prep: padded copy q of Qin (stride ldin, dimension d), FFMA
// squared norms qn2, optional TF32 hi/lo split and 8 swizzled copies for the
// scan (NULL to skip), and the batch's counter resets (zero_i32[nzero] = 0,
// zero2[nzero2] = 0, ones_u32[nones] = ~0).
void launch_qprep(const float* Qin, int64_t ldin, int d, int B, int dp, float* q, float* qn2, float* hi,
                  float* lo, float* qsw, int32_t* zero_i32, int nzero, int32_t* zero2, int nzero2,
                  uint32_t* ones_u32, int nones, cudaStream_t st);
// hi/lo TF32 split of rows [0, n) of an [n][dp] table.
void launch_tf32_split(const float* x, int64_t n, int dp, float* hi, float* lo, cudaStream_t st);
float coarse_coef(int metric, int dp, bool split, int ks);
// Per query: exact top-nprobe in-scope lists by (dist, cid) from the screened
// distances (bound + exact re-rank of the boundary).  ncand: re-ranked lists
// per query (may be NULL).
void launch_coarse_pick(int metric, bool split, int ks, const float* Aapp, int64_t lda, int B, ListTable lt,
                        const float* cnrm, const float* Qd, const float* qn2,
                        const int32_t* scope_codes, int nscopes, int nprobe, int32_t* probe,
                        uint32_t* probe_key, int32_t* ncand, const RouteArgs& ra, cudaStream_t st);

// Cold tier: copy host-arena rows [src_row, src_row+n) (pinned, device-mapped)
// to HBM arena rows [dst_row, ...), with ids and squared norms.
struct StageCopy {
  int64_t src_row;
  int64_t dst_row;
  int32_t n;
  int32_t pad;
};
void launch_gather_rows(const StageCopy* desc, int ndesc, const float* hrows, const int64_t* hids,
                        float* rows, int64_t* ids, float* nrm, int dp, cudaStream_t st);
void launch_stage_norms(const StageCopy* desc, int ndesc, const float* rows, float* nrm, int dp,
                        const int64_t* hids, int64_t* ids, cudaStream_t st);

// Batched append: padded staging rows [n][dp] + ids -> arena rows dst_row[i], with norms.
void launch_append_rows(const float* src, const int64_t* src_ids, const int64_t* dst_row, int n,
                        float* rows, int64_t* ids, float* nrm, int dp, cudaStream_t st,
                        const int64_t* len_pairs = nullptr, int nlen = 0, int64_t* d_len = nullptr);

// Per-list exact distances of one query (agent-mode L2 scan): list l's rows
// at src[l].rows ([n][dp], HBM or mapped host), ids at src[l].ids; rows of
// list l are out rows [prefix[l], prefix[l+1]).  *qn = |q| (device; cosine only).
struct ListSrc {
  const float* rows;
  const int64_t* ids;
};
// ---- agent path (pk_agent.cu) ----
// rows[slots[i]] = src[i] (rows of dp floats)
void launch_rows_put(const float* src, const int32_t* slots, int n, int dp, float* rows, cudaStream_t st);
// out[i] = dist(q, rows[slots[i]]) (reference arithmetic)
void launch_gather_dist(int metric, const float* q, const float* rows, int dp, int d, const int32_t* slots, int n,
                        float* out, cudaStream_t st);
// out[r][c] = dist(q = rows[qslots[r]], x = rows[xslots[c]])
void launch_gather_mat(int metric, const float* rows, int dp, int d, const int32_t* qslots, int nr,
                       const int32_t* xslots, int nc, float* out, cudaStream_t st);
// every row of the probed lists (device slots, coarse order), list after list
void launch_probe_lists(int metric, const float* q, ListTable lt, const int32_t* probe, int nprobe,
                        int64_t maxlen, int64_t cap, float* out_d, int64_t* out_ids, int64_t* out_prefix,
                        int64_t* out_cids, cudaStream_t st, int nq = 1);  // nq queries: q [nq][dp],
                        // probe [nq][nprobe], outputs in blocks of cap / nprobe + 1 / nprobe per query
// the L1 placement chain of ref/cache.py:284-325 (one CTA)
int l1_place_max_clusters();
void launch_l1_place(int metric, int nc0, int n_p, int cap, int dp, int d, double* sums, float* cents,
                     int32_t* cnt, const float* items, const int32_t* holder, const int32_t* dup, int m,
                     const float* qv,
                     int32_t* out_t, uint8_t* out_added, uint8_t* out_merged, int32_t* out_q, cudaStream_t st);
void launch_lists_dist(int metric, const float* q, const float* qn, const ListSrc* src, const int64_t* prefix,
                       int m, int64_t total, int dp, int d, float* out_d, int64_t* out_ids,
                       cudaStream_t st);

// Peer combine: results -> peers' receive areas (IPC-mapped) + release flags;
// merge after acquiring every rank's flag for the epoch (bounded wait, *err).
void launch_peer_send(const int64_t* ids, const int64_t* cids, const int64_t* sc, const float* d,
                      const int32_t* n, int B, int group, int kk, int64_t block_bytes,
                      uint8_t* const* peers, int R, int my_rank, uint64_t epoch, uint32_t* done_ctr,
                      cudaStream_t st);
void launch_peer_merge(int metric, const void* area, int64_t block_bytes, int R, int B, int kk, uint64_t epoch,
                       int64_t timeout_ns, int32_t* err, int64_t* out_ids, float* out_d,
                       int64_t* out_cid, int32_t* out_n, int64_t* out_scanned, cudaStream_t st);

}  // namespace pk
