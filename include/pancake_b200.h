/*
 * pancake_b200.h -- C-ABI of the B200-native IVF search hot path.
 *
 * The reference (arxiv/paper_2602_21477, package `agentmem`, pure Python)
 * has no C interface; its plugin boundaries are Python protocols.  Each entry
 * point below names the reference interface it replaces (file:line into
 * /root/reference/pkg/src/agentmem/).  Plain pointers and sizes only; no torch
 * types.  All calls return PK_OK (0) or an error code; pk_last_error() gives
 * the message of the calling thread's last failure.
 *
 * Pointer convention: by default every data pointer is HOST memory (pinned or
 * pageable); the call copies host<->device itself and returns when outputs are
 * in place.  With PK_DEVICE_PTRS in `flags` the pointers are device pointers on
 * the index's device and the call is asynchronous on the index stream
 * (pk_stream / pk_sync).
 *
 * Arithmetic is the reference's exactly (ref/kernels.py:73-135): fp32, j
 * ascending, every op rounded, no FMA; ordering is (distance, id) with ties to
 * the smaller id (ref/engine.py:411) and (distance, cid) for lists
 * (ref/graph.py:395).
 */
#ifndef PANCAKE_B200_H
#define PANCAKE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PK_OK 0
#define PK_ERR_USAGE 1  /* precondition violated -> agentmem.core.UsageError (core.py:20-21) */
#define PK_ERR_DEVICE 2 /* CUDA failure -> agentmem.tiering.AcceleratorError (tiering.py:29-30) */
#define PK_ERR_NOMEM 3  /* device allocation failed -> AcceleratorError("allocation failed") */

#define PK_DEVICE_PTRS 1

#define PK_METRIC_SQ_L2 0  /* Metric.SQUARED_EUCLIDEAN, wire code 0 (core.py:40-58) */
#define PK_METRIC_IP 1     /* Metric.INNER_PRODUCT (negated) */
#define PK_METRIC_COSINE 2 /* Metric.COSINE */

typedef struct pk_index pk_index;

/* ---- library ---------------------------------------------------------- */
const char* pk_last_error(void);
int pk_version(void);
int pk_device_count(int* n);

/* ---- kernel table: replaces kernels.BACKENDS[...] (kernels.py:138-158) -- */
/* out[b][i] = dist(q[b], mat[i]); batch_distances (core.py:98-109) for B
 * queries at once.  q: [B][d], mat: [n][d], out: [B][n]. */
int pk_distances(const float* q, int64_t B, const float* mat, int64_t n, int64_t d, int metric,
                 float* out, int flags);
/* kmeans_assign_nb (kernels.py:116-135): labels i64[n], dists f64[n]. */
int pk_kmeans_assign(const float* x, int64_t n, const float* cents, int64_t k, int64_t d,
                     int64_t* labels, double* dists, int flags);
/* core.centroid (core.py:112-117): fp64 row-order mean -> f32[d]. */
int pk_centroid(const float* mat, int64_t n, int64_t d, float* out, int flags);

/* k-means update (kmeans_split_points, clusters.py:166-171): rows [n][d]
 * grouped by label in original order, segment c = rows [off[c], off[c+1]);
 * out[c] = core.centroid of the segment (fp64 row-order mean -> f32);
 * empty segments are left untouched.  Device pointers (PK_DEVICE_PTRS). */
int pk_centroids_segmented(const float* rows, int64_t n, int64_t d, const int64_t* off, int64_t k,
                           float* out, int flags);

/* ---- device index: ClusterStore storage + TierManager residency -------- */
/* (clusters.py:186-362, tiering.py:175-448).  One index per device.        */
int pk_index_create(int64_t dim, int metric, int device, int64_t reserve_rows,
                    int64_t reserve_lists, pk_index** out);
int pk_index_destroy(pk_index* ix);
int pk_sync(pk_index* ix);
void* pk_stream(pk_index* ix);
/* Bytes of HBM held by the arena + list table. */
int pk_index_bytes(pk_index* ix, int64_t* bytes);

/* ClusterStore.create_cluster (clusters.py:250-266): new posting list `cid`
 * in scope `scope_code` with n seed rows; centroid recomputed on device as in
 * Cluster.recompute_stats (clusters.py:111-118) and returned in out_centroid
 * (host f32[d], may be NULL). */
int pk_list_create(pk_index* ix, int64_t cid, int32_t scope_code, const float* rows,
                   const int64_t* ids, int64_t n, float* out_centroid, int flags);
/* Cluster.add (clusters.py:71-79) / TierManager.buffered_insert
 * (tiering.py:280-290): append rows in place (relocating when full). */
int pk_list_append(pk_index* ix, int64_t cid, const float* rows, const int64_t* ids, int64_t n,
                   int flags);
/* A whole insert batch (engine.py:571-605 after assignment): row i (host
 * f32[d]) appended to list cids[i] in batch order, one H2D copy and one
 * scatter kernel for all lists (host pointers). */
int pk_list_append_batch(pk_index* ix, int64_t n, const int64_t* cids, const float* rows,
                         const int64_t* ids);
/* Cluster.remove (clusters.py:81-109): swap-with-last compaction of `row`. */
int pk_list_remove_row(pk_index* ix, int64_t cid, int64_t row);
/* ClusterStore.retire_cluster (clusters.py:352-362). */
int pk_list_retire(pk_index* ix, int64_t cid);
/* Cluster.recompute_stats centroid (clusters.py:111-118) on device;
 * out_centroid host f32[d] (may be NULL). */
int pk_list_recompute(pk_index* ix, int64_t cid, float* out_centroid);
/* Overwrite the routing centroid of `cid` (host f32[d]). */
int pk_list_set_centroid(pk_index* ix, int64_t cid, const float* centroid);
int pk_list_size(pk_index* ix, int64_t cid, int64_t* n);
/* Read back rows (host f32[n][d]) and ids (host i64[n]); either may be NULL. */
int pk_list_read(pk_index* ix, int64_t cid, float* rows, int64_t* ids);

/* ---- batched hot path ------------------------------------------------- */
/* Store._search_read_phase for the bare IVF path (engine.py:319-404) over a
 * batch: coarse top-nprobe over the in-scope lists (graph.py:321-396 at
 * exhaustive ef), fused exact scan of every probed list
 * (tiering.py:294-328), merge to the first kk by (distance, id) with
 * first-occurrence dedup (engine.py:406-426).
 *   Q: [B][d]; scope_codes: [nscopes] (<= 64)
 *   out_ids/out_dists/out_cids: [B][kk] (unused tail: -1 / +inf / -1)
 *   out_n: [B] hits per query; out_probe: [B][nprobe] cids (may be NULL,
 *   -1 padded); out_scanned: [B] scanned vectors (SearchStats, may be NULL).
 * nprobe <= 2048, 1 <= kk <= 64. */
int pk_search(pk_index* ix, const float* Q, int64_t B, const int32_t* scope_codes,
              int32_t nscopes, int32_t nprobe, int32_t kk, int64_t* out_ids, float* out_dists,
              int64_t* out_cids, int32_t* out_n, int64_t* out_probe, int64_t* out_scanned,
              int flags);
/* ClusterStore.assign_nearest (clusters.py:268-279) for n vectors against
 * the lists of one scope: out_cid [n] (-1 when the scope has no lists),
 * out_dist [n] (may be NULL). */
int pk_assign(pk_index* ix, const float* X, int64_t n, int32_t scope_code, int64_t* out_cid,
              float* out_dist, int flags);

/* ---- agent-mode L2 scan (engine.py:366-396) ------------------------------
 * pk_search_coarse_cids: the coarse stage for B queries, probed list ids
 *   (host i64 [B][nprobe], -1 padded) in coarse order.
 * pk_scan_lists: one query's reference-arithmetic distances to every row of the
 *   lists cids[0..m) (resident in HBM or cold in the host arena), concatenated
 *   in the given order; list l's rows are out rows [out_prefix[l],
 *   out_prefix[l+1]) (out_prefix: host i64[m+1], out_ids / out_dists sized by
 *   the lists' total length).  The caller replays the per-list early
 *   termination on these values (MultiLevelCache._kth). */
int pk_search_coarse_cids(pk_index* ix, const float* Q, int64_t B, const int32_t* scope_codes,
                          int32_t nscopes, int32_t nprobe, int64_t* out_cids);
int pk_scan_lists(pk_index* ix, const float* q, const int64_t* cids, int32_t m, int64_t* out_ids,
                  float* out_dists, int64_t* out_prefix);

/* ---- agent path, one device pass per agent search (pk_agent.cu) ----------
 * Replaces the per-pool / per-list / per-pattern batch_distances calls of
 * ref/engine.py:319-404 (cached_search ref/cache.py:162-221, the staging
 * scan, HybridGraphIndex.search ref/graph.py:321-396 and the list scans) and
 * of ref/fsm.py:296-392 (match / align / predict) with one call; the caller
 * replays the policy (scan order, stop rule, _topk) over the values.
 * pk_rows_put: rows [n][d] into the HBM row store at host-managed slots (the
 *   rows the policy scans: cache pool rows, L1 centroids, FSM states).
 * pk_agent_read: puts first, then for one query q: out_d[i] = dist(q, row
 *   slots[i]); out_m[r][c] = dist(row mq[r], row mx[c]) (mq rows as queries);
 *   and, when nprobe > 0, the reference's coarse traversal (ef, mode as
 *   pk_search_graph) and every row of each probed list in coarse order:
 *   out_cids[nprobe] (-1 padded), *out_coarse = distance computations, list l
 *   at rows [out_prefix[l], out_prefix[l+1]) of out_ids / out_dists (capacity
 *   cap rows; a larger total fails with PK_ERR_USAGE, out_prefix set).
 * pk_l1_place: the L1 placement chain of ref/cache.py:284-325 for m items
 *   popped from L0 (then q's capture target when q != NULL) over nc live
 *   clusters (fp64 sums [nc][d], f32 centroids [nc][d], counts [nc]);
 *   holder[i] = list position of the cluster already holding item i (ids
 *   item_ids[i]; an id may recur in the chain), or -1.
 *   Per item: out_target = list position chosen (-1: a fresh cluster was
 *   appended), out_added, out_merged (merge_down after it); *out_qtarget
 *   likewise for q.  The caller applies the same operations in order.
 * pk_agent_lists: the list half of pk_agent_read (nprobe > 0) for B queries
 *   Q [B][d] in one pass -- an agent's search batch, whose queries the Store
 *   still answers one by one (ref/engine.py:287-317) -- query b's outputs at
 *   out_cids + b*nprobe, out_prefix + b*(nprobe+1), out_coarse[b] and rows
 *   [b*cap, b*cap + min(total, cap)) of out_ids / out_dists (a total above cap
 *   is only reported).  *out_version = pk_list_version at the time: the
 *   results stand for the lists, centroids and graph of that version.  Not on
 *   a tiered index.
 * pk_list_version: a counter bumped by every change of a list's rows, length,
 *   centroid or slot and by pk_graph_set. */
int pk_agent_lists(pk_index* ix, const float* Q, int64_t B, const int32_t* scope_codes, int32_t nscopes,
                   int32_t nprobe, int32_t ef, int32_t mode, int64_t cap, int64_t* out_cids, int32_t* out_coarse,
                   int64_t* out_prefix, int64_t* out_ids, float* out_dists, uint64_t* out_version);
int pk_list_version(pk_index* ix, uint64_t* version);
/* pk_rows_reserve: capacity for n row-store slots now (a growth copies the store
 * and frees the old one, which can stall for hundreds of ms; the Store reserves
 * each agent's bound when it registers the agent). */
int pk_rows_reserve(pk_index* ix, int64_t n);
int pk_rows_put(pk_index* ix, const int32_t* slots, const float* rows, int64_t n);
int pk_agent_read(pk_index* ix, const float* q, const int32_t* put_slots, const float* put_rows, int64_t nput,
                  const int32_t* slots, int64_t n, float* out_d, const int32_t* mq, int32_t nmq,
                  const int32_t* mx, int32_t nmx, float* out_m, const int32_t* scope_codes, int32_t nscopes,
                  int32_t nprobe, int32_t ef, int32_t mode, int64_t* out_cids, int32_t* out_coarse,
                  int64_t* out_prefix, int64_t* out_ids, float* out_dists, int64_t cap);
int pk_l1_place(pk_index* ix, int32_t nc, int32_t n_p, int32_t capacity, const double* sums, const float* cents,
                const int32_t* counts, const float* items, const int64_t* item_ids, const int32_t* holder,
                int32_t m, const float* q, int32_t* out_target, uint8_t* out_added, uint8_t* out_merged,
                int32_t* out_qtarget);

/* ---- cold tier (TierManager, tiering.py:175-448) --
 * pk_index_enable_tier (before any list exists): every list keeps a copy in
 * a pinned, device-mapped host arena (the source of truth, tiering.py:9-12);
 * lists are created cold and HBM holds only the lists made resident.  A
 * search streams the probed cold lists into HBM staging over PCIe (one gather
 * kernel per batch); results are identical in every residency state
 * (tiering.py:294-328, SPEC "merged = single-tier").
 * pk_list_set_resident: 1 = admit (HBM copy on a side stream; the list
 *   switches resident when the copy completes, MigrationTicket phases
 *   tiering.py:332-416), 0 = evict (release the HBM copy).
 * pk_list_residency: 0 cold, 1 resident, 2 admission in flight.
 * pk_tier_stats out[12]: resident lists, cold lists, resident HBM bytes,
 *   lists / bytes staged by the last search, bytes staged in total, searches
 *   that staged, admissions started, admissions completed, host arena bytes,
 *   HBM arena rows in use (bump pointer) and allocated. */
int pk_index_enable_tier(pk_index* ix, int64_t reserve_rows);
int pk_list_set_resident(pk_index* ix, int64_t cid, int resident);
int pk_list_residency(pk_index* ix, int64_t cid, int* state);
int pk_tier_stats(pk_index* ix, int64_t* out, int n);

/* ---- sharded search ------------------------------
 * Lists are partitioned over ranks (one index per GPU); the centroid table is
 * replicated so every rank computes the identical global probe set
 * (graph.py:321-396 semantics), scans only the lists it owns, and the
 * per-rank top-kk are exchanged (NCCL all-gather) and merged.
 *
 * Register a list owned by another rank: its centroid joins the coarse
 * quantizer (it is probed and counted exactly like a local list) but it holds
 * no rows here.  Appending to it is a usage error. */
int pk_list_add_remote(pk_index* ix, int64_t cid, int32_t scope_code, const float* centroid);
/* Size of one shard result block for (B, kk): the unit the all-gather moves.
 * Layout (byte offsets, nkk = B*kk):
 *   ids     i64[B][kk]  @ 0
 *   cids    i64[B][kk]  @ 8*nkk
 *   scanned i64[B]      @ 16*nkk
 *   dists   f32[B][kk]  @ 16*nkk + 8*B
 *   n       i32[B]      @ 20*nkk + 8*B
 * padded to 16 bytes.  pk_search (PK_DEVICE_PTRS) writes one straight into
 * these offsets. */
int64_t pk_shard_block_bytes(int64_t B, int32_t kk);
/* Asynchronous host-pointer search in PK_ASYNC_SLOTS slots: pk_search_submit
 * copies Q (host, pinned for best overlap) on a copy stream and queues the
 * device pass; pk_search_collect(slot) waits for that batch and fills the host
 * outputs (same meaning as pk_search's).  With several slots in use the H2D
 * and the caller's host work for the next batches overlap the device pass of
 * the one in flight (small batches need three in flight: the next batch's
 * front half runs beside the current scan).  A slot is reused only after it
 * was collected.  scope_codes are host pointers here. */
#define PK_ASYNC_SLOTS 4
int pk_search_submit(pk_index* ix, int32_t slot, const float* Q, int64_t B,
                     const int32_t* scope_codes, int32_t nscopes, int32_t nprobe, int32_t kk);
int pk_search_collect(pk_index* ix, int32_t slot, int64_t* out_ids, float* out_dists, int64_t* out_cids,
                      int32_t* out_n, int64_t* out_scanned);

/* Split form of pk_search for the dispatch/combine path (every rank brings its
 * own batch):
 * pk_search_coarse: the coarse stage only -- per query the first nprobe
 *   in-scope lists as list handles (int32 [B][nprobe], -1 padded).  Handles are
 *   slot indices; they agree across ranks whose indexes were built by the same
 *   sequence of list creations (ShardedIndex.load builds in global order).
 * pk_search_probed: the scan stage only, for given handles: scans the probed
 *   lists this index holds (remote lists add nothing) and writes B / group
 *   shard result blocks, block g = queries [g*group, (g+1)*group). */
int pk_search_coarse(pk_index* ix, const float* Q, int64_t B, const int32_t* scope_codes,
                     int32_t nscopes, int32_t nprobe, int32_t* out_probe, int flags);
int pk_search_probed(pk_index* ix, const float* Q, int64_t B, const int32_t* probe, int32_t nprobe,
                     int32_t kk, int64_t group, void* out_blocks, int flags);
/* Merge R gathered blocks (contiguous, R * pk_shard_block_bytes) into the
 * global first kk per query by (distance, id), first occurrence per id
 * (engine.py:406-426); out_scanned = sum over shards (may be NULL).
 * R * kk <= 1024.  Pointers follow `flags` (device: async on the index stream). */
int pk_merge_shards(pk_index* ix, const void* blocks, int32_t R, int64_t B, int32_t kk,
                    int64_t* out_ids, float* out_dists, int64_t* out_cids, int32_t* out_n,
                    int64_t* out_scanned, int flags);

/* ---- peer combine (fused combine over NVLink P2P) --
 * The combine step of dispatch/combine without NCCL: every rank owns a
 * receive area (R shard blocks + R ready flags) in its HBM, exported as a CUDA
 * IPC handle (64 bytes) and mapped by the peers.  pk_combine_search_probed runs
 * the scan stage for the gathered batch (R x group queries) and writes block g
 * of its results STRAIGHT INTO rank g's area (P2P stores), then publishes
 * flag[my_rank] = epoch in every area (system-scope release).  pk_combine_merge
 * acquires all R flags of `epoch` on the device (bounded wait; a timeout sets
 * the error word read by pk_combine_status) and merges, as pk_merge_shards.
 * pk_combine_open: peer's IPC handle, or area_ptr for ranks in the same
 * process.  Device pointers only (PK_DEVICE_PTRS); epochs strictly increase. */
int pk_combine_create(pk_index* ix, int32_t R, int32_t my_rank, int64_t group, int32_t kk,
                      void* ipc_handle_out);
int pk_combine_open(pk_index* ix, int32_t peer, const void* ipc_handle, void* area_ptr);
void* pk_combine_area(pk_index* ix);
int pk_combine_search_probed(pk_index* ix, const float* Q, int64_t B, const int32_t* probe,
                             int32_t nprobe, int64_t epoch, int flags);
int pk_combine_merge(pk_index* ix, int64_t epoch, double timeout_s, int64_t* out_ids, float* out_dists,
                     int64_t* out_cids, int32_t* out_n, int64_t* out_scanned, int flags);
int pk_combine_status(pk_index* ix, int32_t* err);

/* ---- measurement ------------------------------------------------------ */
/* Between begin and end every pk_search records CUDA events on the index
 * stream around its stages: [0] input copy, [1] coarse distances,
 * [2] coarse select, [3] routing, [4] fused scan, [5] merge + outputs.
 * pk_profile_end synchronizes and returns the per-stage device time summed
 * over the calls (ms) and the call count. */
int pk_profile_begin(pk_index* ix);
int pk_profile_end(pk_index* ix, double* stage_ms, int nstages, int* ncalls);
/* Candidate-pool size per query of the last screened search (host int32[B]);
 * values above the pool capacity mean that query took the exact overflow path. */
int pk_debug_pool_counts(pk_index* ix, int32_t* out, int64_t B);
/* Lists re-ranked exactly per query by the last search's tensor-core coarse
 * quantizer (host int32[B]). */
int pk_debug_coarse_counts(pk_index* ix, int32_t* out, int64_t B);
/* ---- the reference's hybrid coarse graph (ref/graph.py:74-422) ----------
 * The Store keeps the per-scope graphs (levels, neighbor lists, portals) on
 * the host exactly as the reference builds them, with every distance taken
 * from pk_centroid_dists; pk_graph_set uploads them; pk_search_graph is
 * pk_search whose coarse stage is the reference's traversal
 * (HybridGraphIndex.search, mode 0, or search_independent, mode 1) at the
 * given ef, so the probed lists equal the reference's at ANY ef, and
 * out_coarse[b] = its distance-computation count (SearchStats.coarse_computations).
 *
 * pk_graph_set: n nodes; node i has cid node_cid[i], level node_level[i] and
 *   (level + 1) * M neighbor cids in nbr (layer 0 first, list order, -1
 *   padded), portals por[por_ptr[i] .. por_ptr[i + 1]) in insertion order;
 *   per scope code: entry cid (-1 none) and max level.  The graph must be
 *   re-uploaded after any list create / retire (PK_ERR_USAGE otherwise).
 * pk_search_graph: scope codes are HOST pointers; the rest as pk_search.
 * pk_graph_probe: coarse only (host): probed cids [B][nprobe] (-1 padded) and counts.
 * pk_centroid_dists: out[n][nslots] = reference distance of each host row
 *   V[n][d] to every slot's centroid; out_cids[nslots] = slot cids (-1 free).
 * pk_list_slot / pk_slot_count: slot of a list, and the slot count. */
int pk_graph_set(pk_index* ix, int32_t M, int64_t n, const int64_t* node_cid, const int32_t* node_level,
                 const int64_t* nbr, const int64_t* por_ptr, const int64_t* por, int32_t static_code,
                 int32_t nsc, const int32_t* sc_code, const int64_t* sc_entry, const int32_t* sc_maxl);
int pk_search_graph(pk_index* ix, const float* Q, int64_t B, const int32_t* scope_codes,
                    int32_t nscopes, int32_t nprobe, int32_t ef, int32_t mode, int32_t kk,
                    int64_t* out_ids, float* out_dists, int64_t* out_cids, int32_t* out_n,
                    int64_t* out_probe, int64_t* out_scanned, int32_t* out_coarse, int flags);
int pk_graph_probe(pk_index* ix, const float* Q, int64_t B, const int32_t* scope_codes, int32_t nscopes,
                   int32_t nprobe, int32_t ef, int32_t mode, int64_t* out_cids, int32_t* out_coarse);
int pk_centroid_dists(pk_index* ix, const float* V, int64_t n, float* out, int64_t* out_cids);
int pk_list_slot(pk_index* ix, int64_t cid, int32_t* slot);
int pk_slot_count(pk_index* ix, int32_t* n);
/* Fault injection (the reference's fail_next_alloc seam, tiering.py:101-104,
 * 357-361): the next n admission allocations (pk_list_set_resident(.., 1))
 * fail with PK_ERR_NOMEM and leave the list cold and unchanged. */
int pk_debug_fail_next_alloc(pk_index* ix, int n);
/* Pool entries that survived the final bound and were re-ranked exactly per
 * query by the last screened search (host int32[B]; -1 = overflow path). */
int pk_debug_rerank_counts(pk_index* ix, int32_t* out, int64_t B);

#ifdef __cplusplus
}
#endif
#endif /* PANCAKE_B200_H */
