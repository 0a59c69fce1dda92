// pk_abi.cu -- the device index (HBM arena of posting lists + list table) and
// the extern "C" boundary declared in include/pancake_b200.h.
//
// Layout in HBM:
//   rows  f32[arena_rows][dp]  every posting list is a contiguous row range
//                              [off, off+cap) of one arena; dp = d rounded up
//                              to 32 floats (zero padded, 128-byte rows chunks)
//   ids   i64[arena_rows]      item id of each row
//   list table (per slot): off, len, cid, scope code, centroid f32[dp]
// A list grows in place into its slack (25% + 16 rows, like the reference's
// device slack, ref/tiering.py:356) and is relocated when full.
#include "../../include/pancake_b200.h"
#include "pk_kernels.h"

#include <cudaTypedefs.h>

#include <algorithm>
#include <chrono>
#include <sys/mman.h>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

using namespace pk;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(call)                                                                           \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      cudaGetLastError();                                                                  \
      return fail(e_ == cudaErrorMemoryAllocation ? PK_ERR_NOMEM : PK_ERR_DEVICE,          \
                  "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
    }                                                                                      \
  } while (0)

#define RET(call)                \
  do {                           \
    int r_ = (call);             \
    if (r_ != PK_OK) return r_;  \
  } while (0)

inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// Grow-only device buffer.
// Pinned host staging: one packed DMA per call instead of pageable (driver
// bounce-buffered, row-by-row 2-D) copies -- what small cache-pool and
// centroid scans pay per call.
struct PinnedBuf {
  uint8_t* p = nullptr;
  uint8_t* dev = nullptr;  // device alias (mapped): kernels read / write it over PCIe
  size_t bytes = 0;
  int ensure(size_t need) {
    if (need <= bytes) return PK_OK;
    size_t nb = std::max(need, bytes + bytes / 2);
    static const bool dbg = getenv("PK_DEBUG_GROW") != nullptr;  // (measurement only)
    if (dbg) fprintf(stderr, "pinned buffer grow %zu -> %zu bytes\n", bytes, nb);
    if (p) cudaFreeHost(p);
    p = dev = nullptr;
    bytes = 0;
    CK(cudaHostAlloc((void**)&p, nb, cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer((void**)&dev, p, 0));
    bytes = nb;
    return PK_OK;
  }
};
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int ensure(size_t need, bool zero = false, cudaStream_t st = 0) {
    if (need <= bytes) return PK_OK;
    size_t nb = std::max(need, bytes + bytes / 2);
    if (p) CK(cudaFree(p));
    p = nullptr;
    bytes = 0;
    CK(cudaMalloc(&p, nb));
    if (zero) CK(cudaMemsetAsync(p, 0, nb, st));
    bytes = nb;
    return PK_OK;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct Range {
  int64_t off, cap;
};

// Return [off, off+cap) to a first-fit free list.  The list is kept sorted by
// offset and coalesced, and a free range that reaches the bump pointer gives
// its rows back to it, so per-batch staging ranges of varying sizes do not
// fragment the arena.
static void free_coalesce(std::vector<Range>& fr, int64_t& top, int64_t off, int64_t cap) {
  if (cap <= 0) return;
  auto it = std::lower_bound(fr.begin(), fr.end(), off,
                             [](const Range& r, int64_t o) { return r.off < o; });
  it = fr.insert(it, Range{off, cap});
  if (it + 1 != fr.end() && it->off + it->cap == (it + 1)->off) {
    it->cap += (it + 1)->cap;
    fr.erase(it + 1);
  }
  if (it != fr.begin() && (it - 1)->off + (it - 1)->cap == it->off) {
    (it - 1)->cap += it->cap;
    it = fr.erase(it) - 1;
  }
  if (it->off + it->cap == top) {
    top = it->off;
    fr.erase(it);
  }
}

}  // namespace

// Recursive mutex that counts acquisitions: a search may overlap its front
// half with the previous search's scan only when no other call took the
// index lock in between (nothing else was queued on the index stream).
struct CountedMutex {
  std::recursive_mutex m;
  uint64_t n = 0;
  void lock() {
    m.lock();
    n++;
  }
  bool try_lock() {
    if (!m.try_lock()) return false;
    n++;
    return true;
  }
  void unlock() { m.unlock(); }
};

struct pk_index {
  CountedMutex mu;  // one caller at a time per index (Store read locks admit concurrent searches)
  int device = 0;
  int64_t d = 0, dp = 0;
  int metric = 0;
  int num_sms = 148;
  int scan_sms = 148;  // persistent scan grid (PK_SCAN_SMS; < num_sms leaves SMs to overlapped work)
  cudaStream_t st = nullptr;

  // arena
  float* rows = nullptr;
  int64_t* ids = nullptr;
  float* nrm = nullptr;  // squared row norms (tensor-core screen)
  int64_t arena_cap = 0, arena_top = 0;
  std::vector<Range> free_ranges;
  ArenaMaps maps;

  // list table (host mirror + device copy)
  std::vector<int64_t> h_off, h_len, h_cap, h_cid;
  std::vector<int32_t> h_scope;
  std::vector<uint8_t> h_remote;  // list owned by another shard (centroid only)
  std::unordered_map<int64_t, int32_t> cid2slot;
  std::vector<int32_t> free_slots;
  int32_t nslots = 0, slot_cap = 0;
  int64_t *d_off = nullptr, *d_len = nullptr, *d_cid = nullptr;
  int32_t* d_scope = nullptr;
  float* d_cent = nullptr;
  float* d_cnrm = nullptr;  // squared centroid norms (FFMA; coarse screen input)
  float* d_chi = nullptr;   // TF32 hi / lo split of the centroid table (coarse screen)
  float* d_clo = nullptr;
  CoarseMaps cmaps;         // c[0..1]: 128 slots x 32 floats, SWIZZLE_128B (q[] per search)
  int32_t dirty_lo = INT32_MAX, dirty_hi = -1;

  // search scratch: two sets used by consecutive searches in turn, so the
  // next batch's prep / coarse / pick / routing kernels (programmatic
  // dependent launches) can run while this batch's re-rank merge drains
  struct Scratch {
    DevBuf q, qnorm, dc, probe, probe_key, counts, items, qpairs, slot_off, scanned, cand_key,
        cand_id, cand_n, cand_list, out_ids, scopes, qnorm2, uq, cpool, ccount, qsw, qhi, qlo, qin,
        ncand, nsurv;
    // the coarse GEMM's query tensor maps for (pointers, rows) last encoded
    CUtensorMap qmap[2];
    const void* qmap_ptr[2] = {nullptr, nullptr};
    int64_t qmap_rows = -1;
    // host scope codes last uploaded into `scopes` (-1: unknown / device
    // codes): an unchanged set skips the pageable copy
    int32_t scopes_h[64];
    int32_t nscopes_h = -1;
    // the scan's gather4 map over the padded query batch
    CUtensorMap qgmap;
    const void* qg_ptr = nullptr;
    int64_t qg_rows = -1;
    void release() {
      for (DevBuf* b : {&q, &qnorm, &dc, &probe, &probe_key, &counts, &items, &qpairs, &slot_off,
                        &scanned, &cand_key, &cand_id, &cand_n, &cand_list, &out_ids, &scopes, &qnorm2,
                        &uq, &cpool, &ccount, &qsw, &qhi, &qlo, &qin, &ncand, &nsurv})
        b->release();
    }
  } scr[3];
  int par = 0, last_par = 0;
  // the last re-rank that read each scratch set (a front half reuses a set
  // once it is done); three sets: a deferred re-rank of batch i may still read
  // set i while the fronts of batches i+1 and i+2 fill theirs
  cudaEvent_t ev_free[3] = {nullptr, nullptr, nullptr};
  // PK_RERANK_DEFER (default 1): pipelined scans and fronts on higher-priority
  // streams than the index stream's re-rank, so batch i's re-rank yields the
  // SMs to batch i+1's scan and runs in its tail; fronts wait only for the
  // re-rank of their own scratch set
  bool rr_defer = true;
  // PK_DEBUG_TIMELINE=1: timing events around each pipelined search's front
  // half, scan and re-rank (no synchronisation; printed once after 48 searches)
  struct Timeline {
    bool on = false, printed = false;
    int n = 0;
    std::vector<cudaEvent_t> ev;  // [48][6]: front begin/end, scan begin/end, re-rank begin/end
  } tl;
  // append staging (mapped), two buffers in turn: an append returns once its
  // scatter is enqueued; the buffer is rewritten only after the event of its
  // previous use (the call before last) has passed
  PinnedBuf hstage2[2];
  cudaEvent_t hstage_ev[2] = {nullptr, nullptr};
  int hstage_i = 0;
  DevBuf tmp_rows2[2];
  PinnedBuf hsl;     // pk_scan_lists staging (mapped)
  PinnedBuf hasg;    // pk_assign host path: padded rows in, (cid, dist) out (mapped)
  // agent path (pk_rows_put / pk_agent_read / pk_l1_place, pk_agent.cu): the
  // HBM row store of the rows the per-agent policy scans (cache pool rows, L1
  // centroids, FSM states) at host-managed slots, packed staging and outputs
  DevBuf arows;  // [acap][dp]
  int64_t acap = 0;
  cudaStream_t ast = nullptr;  // row-store distances beside the coarse traversal
  cudaEvent_t ev_ag0 = nullptr, ev_ag1 = nullptr;
  PinnedBuf hag;  // mapped: packed inputs, then the kernels' outputs
  DevBuf ag_in, ag_l1;
  PinnedBuf hal;  // pk_agent_lists: packed queries, then the traversal / list outputs (mapped)
  DevBuf al_in;
  // front-half overlap: the next batch's prep / coarse / pick / routing run on
  // fst while this batch's scan and re-rank drain on st
  cudaStream_t fst = nullptr;
  // ... and the scan of a pipelined search runs on sst, so this batch's
  // re-rank (index stream, after ev_sdone) runs beside the NEXT batch's scan
  cudaStream_t sst = nullptr;
  // Consecutive pipelined scans alternate between sst and sst2 and do not
  // wait for each other (they share no scratch: three sets, no tier), so scan
  // i+1's CTAs take the SMs scan i's CTAs leave -- its tail -- instead of
  // starting after the last one exits (configs[1] 538K -> 566K QPS,
  // configs[0] 783K -> 894K).  PK_SCAN_OVERLAP=0 serialises.
  bool scan_ovl = true;
  int sturn = 0;
  cudaStream_t sst2 = nullptr;
  cudaEvent_t ev_front = nullptr, ev_scan = nullptr, front_wait = nullptr, ev_sdone = nullptr;
  // lean re-rank beside the next scan: -1 = for batches up to 64 queries
  // (configs[0]: +1%; at 256 queries it lengthened the step),
  // PK_RERANK_LEAN=0/1 forces it off / on
  int rr_lean = -1;
  int rr_lean_ctas = 148;  // PK_RERANK_LEAN_CTAS: the lean grid (default: one per SM)
  uint64_t ev_scan_n = 0;  // lock count when ev_scan was last recorded
  bool pipeline = true;    // PK_PIPELINE=0 turns the overlap off
  DevBuf assign_q, assign_qn, assign_dc, assign_c, assign_d;
  DevBuf assign_part, assign_ctr;  // fused argmin: block minima, finished-block counter
  int chunk_rows = 512;
  bool screen = true;  // screened scan + exact re-rank (sq_l2 / ip); PK_SCAN_EXACT=1 disables
  bool tensor = true;  // screen dots on tcgen05 (TF32); PK_SCREEN=ffma uses CUDA-core FFMA
  bool coarse_tc = true;  // coarse quantizer on tcgen05 + exact re-rank; PK_COARSE=exact disables
  bool coarse_split = true;  // 3xTF32 hi/lo split (tight bound); PK_COARSE=tf32 for one product
  int pool_cap = 4096;  // candidate pool per query (overflow -> exact slow path)
  bool pool_cap_set = false;  // PK_POOL_CAP given: no growth with kk
  // scan query chunks by TMA gather4 (4 queries per op) instead of one bulk
  // copy per query from 8 pre-swizzled batch copies; PK_QGATHER=0 for those
  bool qgather = true;
  DevBuf shard_in, shard_out, pb, pb_out, sl_buf;
  uint8_t* hout = nullptr;  // pinned staging of the host path's packed results
  size_t hout_bytes = 0;

  // ---- asynchronous host-pointer searches (pk_search_submit / collect):
  // PK_ASYNC_SLOTS slots, so the H2D of the next batches (copy stream) and the
  // caller's host work overlap the device pass of the batch in flight
  struct AsyncSlot {
    DevBuf qin, blk;
    uint8_t* hblk = nullptr;  // pinned result block
    size_t hbytes = 0;
    cudaEvent_t copied = nullptr, done = nullptr, consumed = nullptr, ready = nullptr;
    int64_t B = 0;
    int32_t kk = 0;
    bool busy = false;
  } aslot[PK_ASYNC_SLOTS];
  cudaStream_t cst = nullptr;  // copy stream (query uploads)
  cudaStream_t rst = nullptr;  // result read-back stream (off the index stream's critical path)

  // ---- peer combine (pk_combine_*): this rank's receive area (R shard blocks
  // + R flags, IPC-exported) and the peers' areas mapped into this process
  struct Combine {
    int R = 0, my_rank = 0, kk = 0;
    int64_t group = 0, bb = 0;
    uint8_t* area = nullptr;                 // own area (cudaMalloc)
    std::vector<uint8_t*> peers;             // [R] area base per rank (own / IPC / in-process)
    std::vector<uint8_t*> opened;            // IPC mappings to close
    uint8_t** d_peers = nullptr;
    bool peers_dirty = true;
    uint32_t* done_ctr = nullptr;
    int32_t* err = nullptr;
  } comb;

  // ---- cold tier (pk_index_enable_tier).  Every list keeps a copy in a
  // pinned, device-mapped host arena -- the source of truth, as the
  // reference's host rows are (ref/tiering.py:9-12) -- and HBM holds the
  // resident lists only.  A batch streams its probed cold lists into arena
  // staging ranges (gather kernel over PCIe); admissions copy a list into HBM
  // on the migration stream and switch it resident once the copy is done
  // (searches stay exact in every phase, ref/tiering.py:332-416).
  bool tiered = false;
  // PK_STAGE=dma: copy engines for the rows.  In the configs[4] stream the
  // zero-copy gather kernel stays ahead (24.7 vs 19.9 GB/s effective, i.e.
  // staged bytes over search time) although a bare 3 MB pinned copy runs at
  // 52 GB/s on this link (tools/pcie_bw.py)
  bool stage_dma = false;
  float* hrows = nullptr;    // [hcap][dp] pinned
  int64_t* hids = nullptr;   // [hcap] pinned
  float* hrows_d = nullptr;  // device aliases (mapped)
  int64_t* hids_d = nullptr;
  // In-place growth: the arena is one reserved virtual range, registered
  // (pinned + mapped) in segments as it grows, so a growth pins only the new
  // rows and moves nothing (a copying growth of a multi-GB arena costs
  // seconds).  hseg: the first row of every segment; DMA copies never cross
  // one (for_host_pieces).  hva_rows == nullptr: cudaHostAlloc arena.
  float* hva_rows = nullptr;
  int64_t* hva_ids = nullptr;
  size_t hva_rows_bytes = 0, hva_ids_bytes = 0;
  std::vector<int64_t> hseg;
  int64_t hcap = 0, htop = 0;
  std::vector<Range> hfree;
  std::vector<int64_t> h_hoff, h_hcap;
  std::vector<uint8_t> h_res;        // HBM copy at h_off valid
  std::vector<cudaEvent_t> mig_ev;   // in-flight admission copy (null = none)
  std::vector<int64_t> mig_off, mig_cap;
  std::vector<int32_t> mig_list;
  cudaStream_t mst = nullptr;        // migration side stream
  std::vector<Range> staged;         // arena ranges of the last batch's cold lists
  cudaEvent_t stage_ev = nullptr;
  int fail_alloc = 0;           // pk_debug_fail_next_alloc
  uint64_t slot_ver = 0;        // bumped whenever a slot's cid changes (create / retire)
  // ---- hybrid coarse graph (pk_graph_set / pk_search_graph): slot-indexed
  // device copy of the reference's per-scope graphs + portals
  struct Graph {
    bool set = false;
    int M = 0;
    int32_t ns = 0;          // slot count the arrays were built for
    uint64_t slot_ver = 0;   // slot <-> cid map version they were built against
    int32_t static_code = 0;
    DevBuf level, nbr0, up_off, up, por_off, por, rank, slot_of_rank, flags, stamps, heap, count;
    int32_t npor = 0;
    std::unordered_map<int32_t, std::pair<int32_t, int32_t>> entry;  // scope code -> (slot, max level)
    std::vector<uint8_t> hflags;
    std::vector<int32_t> flags_codes;  // scope set the device flags were built for
    uint64_t flags_ver = 0;
    int32_t flags_ns = 0;
    void release() {
      for (DevBuf* b : {&level, &nbr0, &up_off, &up, &por_off, &por, &rank, &slot_of_rank, &flags,
                        &stamps, &heap, &count})
        b->release();
      flags_codes.clear();
    }
  } graph;
  bool stage_pending = false;   // `staged` holds ranges of an enqueued batch
  bool stage_recorded = false;  // stage_ev marks the end of the last staging batch
  int64_t st_lists_last = 0, st_rows_last = 0, st_rows_total = 0, st_batches = 0;
  int64_t mig_started = 0, mig_done = 0;
  DevBuf stage_desc, tmp_rows;

  // stage timing (pk_profile_begin / pk_profile_end): events around each
  // stage of every pk_search while enabled.
  static constexpr int NSTAGE = 6;  // input, coarse dist, coarse select, route, scan, merge+output
  bool prof = false;
  std::vector<cudaEvent_t> prof_ev;  // (NSTAGE+1) per call
  int prof_calls = 0;
  int prof_mark(int call, int stage) {
    size_t i = (size_t)call * (NSTAGE + 1) + stage;
    while (prof_ev.size() <= i) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      prof_ev.push_back(e);
    }
    CK(cudaEventRecord(prof_ev[i], st));
    return PK_OK;
  }

  ListTable table() const {
    ListTable t;
    t.rows = rows;
    t.ids = ids;
    t.off = d_off;
    t.len = d_len;
    t.cid = d_cid;
    t.scope = d_scope;
    t.cent = d_cent;
    t.nrm = nrm;
    t.nslots = nslots;
    t.dp = (int32_t)dp;
    t.d = (int32_t)d;
    t.metric = metric;
    return t;
  }

  void mark(int32_t s) {
    dirty_lo = std::min(dirty_lo, s);
    dirty_hi = std::max(dirty_hi, s);
    tver++;
  }
  // a length change the caller writes into the device table itself
  // (stream-ordered, e.g. the append kernel): host-side caches only
  void touch() { tver++; }
  // longest live list, recomputed only after a table change (every h_len /
  // h_cid edit goes through mark(), which the device table sync relies on too)
  uint64_t tver = 1, maxlen_ver = 0;
  int64_t maxlen_cached = 0;
  int64_t max_list_len() {
    if (maxlen_ver != tver) {
      int64_t m = 0;
      for (int32_t s = 0; s < nslots; s++)
        if (h_cid[s] >= 0) m = std::max(m, h_len[s]);
      maxlen_cached = m;
      maxlen_ver = tver;
    }
    return maxlen_cached;
  }

  // the dirty range of the list table goes over from a pinned snapshot (true
  // async copies; pageable sources cost a driver staging pass each -- ~7 us
  // per insert batch for four of them); the snapshot is rewritten only once
  // the previous sync's copies have read it
  // (two snapshots used in turn, so a sync rarely waits for the last one)
  PinnedBuf tstage[2];
  cudaEvent_t tstage_ev[2] = {nullptr, nullptr};
  int tstage_i = 0;
  int sync_table() {
    if (dirty_hi < dirty_lo) return PK_OK;
    const int32_t lo = dirty_lo, n = dirty_hi - dirty_lo + 1;
    const int bi = tstage_i;
    tstage_i ^= 1;
    if (tstage_ev[bi]) CK(cudaEventSynchronize(tstage_ev[bi]));
    else CK(cudaEventCreateWithFlags(&tstage_ev[bi], cudaEventDisableTiming));
    RET(tstage[bi].ensure((size_t)n * 28));
    uint8_t* p = tstage[bi].p;
    memcpy(p, h_off.data() + lo, (size_t)n * 8);
    memcpy(p + (size_t)n * 8, h_len.data() + lo, (size_t)n * 8);
    memcpy(p + (size_t)n * 16, h_cid.data() + lo, (size_t)n * 8);
    memcpy(p + (size_t)n * 24, h_scope.data() + lo, (size_t)n * 4);
    CK(cudaMemcpyAsync(d_off + lo, p, n * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_len + lo, p + (size_t)n * 8, n * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_cid + lo, p + (size_t)n * 16, n * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_scope + lo, p + (size_t)n * 24, n * 4, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(tstage_ev[bi], st));
    dirty_lo = INT32_MAX;
    dirty_hi = -1;
    return PK_OK;
  }

  int encode_maps() {
    auto enc = get_encode();
    if (!enc) return fail(PK_ERR_DEVICE, "cuTensorMapEncodeTiled unavailable");
    for (int i = 0; i < NBOX; i++) {
      cuuint64_t gdim[2] = {(cuuint64_t)dp, (cuuint64_t)arena_cap};
      cuuint64_t gstride[1] = {(cuuint64_t)(dp * 4)};
      cuuint32_t box[2] = {(cuuint32_t)DC, (cuuint32_t)(TILE >> i)};
      cuuint32_t estr[2] = {1, 1};
      CUresult r = enc(&maps.box[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, rows, gdim, gstride, box,
                       estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return fail(PK_ERR_DEVICE, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    }
    return PK_OK;
  }

  // 2-D fp32 tensor map [rows][ld] with boxes of `box_rows` x DC floats, SWIZZLE_128B.
  int encode_2d(CUtensorMap* m, const float* ptr, int64_t ld, int64_t rows, int box_rows) {
    auto enc = get_encode();
    if (!enc) return fail(PK_ERR_DEVICE, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t gdim[2] = {(cuuint64_t)ld, (cuuint64_t)std::max<int64_t>(rows, 1)};
    cuuint64_t gstride[1] = {(cuuint64_t)(ld * 4)};
    cuuint32_t box[2] = {(cuuint32_t)DC, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), gdim, gstride,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(PK_ERR_DEVICE, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return PK_OK;
  }

  // Squared norm of slot s's centroid (coarse screen input).
  // Derived centroid data of slot s: squared norm and the TF32 hi/lo split.
  void centroid_norm(int32_t s) {
    tver++;  // the coarse distances change (pk_list_version readers)
    launch_row_norms(d_cent + (int64_t)s * dp, 1, (int)dp, d_cnrm + s, st);
    launch_tf32_split(d_cent + (int64_t)s * dp, 1, (int)dp, d_chi + (int64_t)s * dp,
                      d_clo + (int64_t)s * dp, st);
  }

  int grow_arena(int64_t need_rows) {
    if (mst) CK(cudaStreamSynchronize(mst));  // in-flight admission copies target the old arena
    int64_t ncap = std::max<int64_t>({need_rows, arena_cap + arena_cap / 2, 1024});
    float* nrows = nullptr;
    int64_t* nids = nullptr;
    float* nnrm = nullptr;
    CK(cudaMalloc(&nrows, (size_t)ncap * dp * 4));
    CK(cudaMalloc(&nids, (size_t)ncap * 8));
    CK(cudaMalloc(&nnrm, (size_t)ncap * 4));
    CK(cudaMemsetAsync(nrows, 0, (size_t)ncap * dp * 4, st));
    CK(cudaMemsetAsync(nnrm, 0, (size_t)ncap * 4, st));
    if (rows) {
      CK(cudaMemcpyAsync(nrows, rows, (size_t)arena_top * dp * 4, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(nids, ids, (size_t)arena_top * 8, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(nnrm, nrm, (size_t)arena_top * 4, cudaMemcpyDeviceToDevice, st));
      CK(cudaStreamSynchronize(st));
      cudaFree(rows);
      cudaFree(ids);
      cudaFree(nrm);
    }
    rows = nrows;
    ids = nids;
    nrm = nnrm;
    arena_cap = ncap;
    return encode_maps();
  }

  // First-fit range allocation; falls back to the bump pointer.
  int alloc_range(int64_t cap, int64_t* off) {
    for (size_t i = 0; i < free_ranges.size(); i++) {
      if (free_ranges[i].cap >= cap) {
        *off = free_ranges[i].off;
        free_ranges[i].off += cap;
        free_ranges[i].cap -= cap;
        if (free_ranges[i].cap == 0) free_ranges.erase(free_ranges.begin() + i);
        return PK_OK;
      }
    }
    if (arena_top + cap > arena_cap) RET(grow_arena(arena_top + cap));
    *off = arena_top;
    arena_top += cap;
    return PK_OK;
  }
  void free_range(int64_t off, int64_t cap) { free_coalesce(free_ranges, arena_top, off, cap); }

  int grow_slots(int32_t need) {
    int32_t ncap = std::max<int32_t>({need, slot_cap * 2, 64});
    int64_t *no = nullptr, *nl = nullptr, *nc = nullptr;
    int32_t* ns = nullptr;
    float* ncent = nullptr;
    CK(cudaMalloc(&no, ncap * 8));
    CK(cudaMalloc(&nl, ncap * 8));
    CK(cudaMalloc(&nc, ncap * 8));
    CK(cudaMalloc(&ns, ncap * 4));
    float *ncn = nullptr, *nhi = nullptr, *nlo = nullptr;
    CK(cudaMalloc(&ncent, (size_t)ncap * dp * 4));
    CK(cudaMalloc(&nhi, (size_t)ncap * dp * 4));
    CK(cudaMalloc(&nlo, (size_t)ncap * dp * 4));
    CK(cudaMalloc(&ncn, (size_t)ncap * 4));
    CK(cudaMemsetAsync(ncent, 0, (size_t)ncap * dp * 4, st));
    CK(cudaMemsetAsync(nhi, 0, (size_t)ncap * dp * 4, st));
    CK(cudaMemsetAsync(nlo, 0, (size_t)ncap * dp * 4, st));
    CK(cudaMemsetAsync(ncn, 0, (size_t)ncap * 4, st));
    if (d_cent) {
      CK(cudaMemcpyAsync(ncent, d_cent, (size_t)nslots * dp * 4, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(nhi, d_chi, (size_t)nslots * dp * 4, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(nlo, d_clo, (size_t)nslots * dp * 4, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(ncn, d_cnrm, (size_t)nslots * 4, cudaMemcpyDeviceToDevice, st));
      CK(cudaStreamSynchronize(st));
      cudaFree(d_off);
      cudaFree(d_len);
      cudaFree(d_cid);
      cudaFree(d_scope);
      cudaFree(d_cent);
      cudaFree(d_cnrm);
      cudaFree(d_chi);
      cudaFree(d_clo);
    }
    d_off = no;
    d_len = nl;
    d_cid = nc;
    d_scope = ns;
    d_cent = ncent;
    d_cnrm = ncn;
    d_chi = nhi;
    d_clo = nlo;
    slot_cap = ncap;
    RET(encode_2d(&cmaps.c[0], coarse_split ? d_chi : d_cent, dp, slot_cap, 128));
    RET(encode_2d(&cmaps.c[1], d_clo, dp, slot_cap, 128));
    h_off.resize(ncap, 0);
    h_len.resize(ncap, 0);
    h_cap.resize(ncap, 0);
    h_cid.resize(ncap, -1);
    h_scope.resize(ncap, -1);
    h_remote.resize(ncap, 0);
    h_hoff.resize(ncap, 0);
    h_hcap.resize(ncap, 0);
    h_res.resize(ncap, 1);
    mig_ev.resize(ncap, nullptr);
    mig_off.resize(ncap, 0);
    mig_cap.resize(ncap, 0);
    // whole table must be re-uploaded into the new arrays
    if (nslots > 0) {
      mark(0);
      mark(nslots - 1);
    }
    return PK_OK;
  }

  // ---- cold tier helpers ----------------------------------------------
  int host_grow(int64_t need) {
    static const bool dbg = getenv("PK_DEBUG_GROW") != nullptr;  // (measurement only)
    const auto t0 = std::chrono::steady_clock::now();
    const int64_t ncap = std::max<int64_t>({need, hcap + hcap / 2, 1024});
    struct Report {
      bool on;
      int64_t from, to;
      std::chrono::steady_clock::time_point t0;
      ~Report() {
        if (on)
          fprintf(stderr, "host arena grow %lld -> %lld rows: %.1f ms\n", (long long)from, (long long)to,
                  std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
      }
    } rep{dbg, hcap, ncap, t0};
    if (host_grow_in_place(ncap)) {  // nothing moves: no wait for readers of the arena
      rep.to = hcap;
      return PK_OK;
    }
    if (st) CK(cudaStreamSynchronize(st));  // gathers / migrations read the old host arena
    if (mst) CK(cudaStreamSynchronize(mst));
    float* nr = nullptr;
    int64_t* ni = nullptr;
    CK(cudaHostAlloc((void**)&nr, (size_t)ncap * dp * 4, cudaHostAllocMapped | cudaHostAllocPortable));
    CK(cudaHostAlloc((void**)&ni, (size_t)ncap * 8, cudaHostAllocMapped | cudaHostAllocPortable));
    if (hrows) {
      memcpy(nr, hrows, (size_t)htop * dp * 4);
      memcpy(ni, hids, (size_t)htop * 8);
      cudaFreeHost(hrows);
      cudaFreeHost(hids);
    }
    hrows = nr;
    hids = ni;
    hcap = ncap;
    CK(cudaHostGetDevicePointer((void**)&hrows_d, hrows, 0));
    CK(cudaHostGetDevicePointer((void**)&hids_d, hids, 0));
    return PK_OK;
  }
  // Grow the reserved-range arena to >= ncap rows in place; false: not
  // available (no reservation, mapping not at the host address), the caller
  // falls back to a copying growth.
  bool host_grow_in_place(int64_t ncap) {
    constexpr int64_t G = 4096;  // segment granularity in rows: page- and row-aligned for rows and ids
    if (hrows && !hva_rows) return false;  // a cudaHostAlloc arena stays one
    if (!hva_rows) {
      int can = 0;
      cudaDeviceGetAttribute(&can, cudaDevAttrCanUseHostPointerForRegisteredMem, device);
      if (!can || getenv("PK_HOST_ARENA_COPY")) return false;
      hva_rows_bytes = (size_t)1 << 40;  // address space only (MAP_NORESERVE)
      hva_ids_bytes = (size_t)1 << 37;
      void* a = mmap(nullptr, hva_rows_bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
      void* b = mmap(nullptr, hva_ids_bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
      if (a == MAP_FAILED || b == MAP_FAILED) {
        if (a != MAP_FAILED) munmap(a, hva_rows_bytes);
        if (b != MAP_FAILED) munmap(b, hva_ids_bytes);
        return false;
      }
      // transparent huge pages where the system allows them: 512x fewer
      // pages for cudaHostRegister to pin (advice only; harmless if refused)
      madvise(a, hva_rows_bytes, MADV_HUGEPAGE);
      madvise(b, hva_ids_bytes, MADV_HUGEPAGE);
      hva_rows = static_cast<float*>(a);
      hva_ids = static_cast<int64_t*>(b);
    }
    const int64_t from = hcap;
    const int64_t to = (ncap + G - 1) / G * G;
    if ((size_t)to * dp * 4 > hva_rows_bytes || (size_t)to * 8 > hva_ids_bytes) return false;
    char* r0 = reinterpret_cast<char*>(hva_rows) + (size_t)from * dp * 4;
    char* i0 = reinterpret_cast<char*>(hva_ids) + (size_t)from * 8;
    const size_t rb = (size_t)(to - from) * dp * 4, ib = (size_t)(to - from) * 8;
    if (cudaHostRegister(r0, rb, cudaHostRegisterMapped | cudaHostRegisterPortable) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    if (cudaHostRegister(i0, ib, cudaHostRegisterMapped | cudaHostRegisterPortable) != cudaSuccess) {
      cudaGetLastError();
      cudaHostUnregister(r0);
      return false;
    }
    void *dr = nullptr, *di = nullptr;
    cudaHostGetDevicePointer(&dr, r0, 0);
    cudaHostGetDevicePointer(&di, i0, 0);
    if (dr != r0 || di != i0) {  // the kernels index one contiguous device range
      cudaHostUnregister(r0);
      cudaHostUnregister(i0);
      cudaGetLastError();
      return false;
    }
    hseg.push_back(from);
    hrows = hrows_d = hva_rows;
    hids = hids_d = hva_ids;
    hcap = to;
    return true;
  }
  // f(first row, count) over [row0, row0 + n) cut at segment starts (a DMA
  // copy must stay inside one host registration)
  template <class F>
  int for_host_pieces(int64_t row0, int64_t n, F f) {
    while (n > 0) {
      int64_t end = row0 + n;
      for (int64_t b : hseg)
        if (b > row0 && b < end) end = b;
      RET(f(row0, end - row0));
      n -= end - row0;
      row0 = end;
    }
    return PK_OK;
  }
  int host_alloc(int64_t cap, int64_t* off) {
    for (size_t i = 0; i < hfree.size(); i++) {
      if (hfree[i].cap >= cap) {
        *off = hfree[i].off;
        hfree[i].off += cap;
        hfree[i].cap -= cap;
        if (hfree[i].cap == 0) hfree.erase(hfree.begin() + i);
        return PK_OK;
      }
    }
    if (htop + cap > hcap) RET(host_grow(htop + cap));
    *off = htop;
    htop += cap;
    return PK_OK;
  }
  void host_free(int64_t off, int64_t cap) { free_coalesce(hfree, htop, off, cap); }
  // n rows (d floats each, host or device source) into host arena rows at `at`
  // (padded to dp with zeros), ids alongside.
  int host_put(int64_t at, const float* src, const int64_t* src_ids, int64_t n, bool dev) {
    if (n <= 0) return PK_OK;
    RET(host_fence());
    if (dev) {
      RET(for_host_pieces(at, n, [&](int64_t r0, int64_t m) {
        CK(cudaMemcpy2DAsync(hrows + r0 * dp, dp * 4, src + (r0 - at) * d, d * 4, d * 4, m,
                             cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(hids + r0, src_ids + (r0 - at), m * 8, cudaMemcpyDeviceToHost, st));
        return PK_OK;
      }));
      CK(cudaStreamSynchronize(st));
    } else {
      for (int64_t r = 0; r < n; r++) memcpy(hrows + (at + r) * dp, src + r * d, d * 4);
      memcpy(hids + at, src_ids, n * 8);
    }
    if (dp > d)
      for (int64_t r = 0; r < n; r++) memset(hrows + (at + r) * dp + d, 0, (dp - d) * 4);
    return PK_OK;
  }
  // Switch a finished admission copy resident (wait: block until it is done).
  int finish_migration(int32_t s, bool wait) {
    cudaEvent_t ev = mig_ev[s];
    if (!ev) return PK_OK;
    if (wait) {
      CK(cudaEventSynchronize(ev));
    } else {
      cudaError_t q = cudaEventQuery(ev);
      if (q == cudaErrorNotReady) return PK_OK;
      if (q != cudaSuccess) CK(q);
    }
    cudaEventDestroy(ev);
    mig_ev[s] = nullptr;
    h_off[s] = mig_off[s];
    h_cap[s] = mig_cap[s];
    h_res[s] = 1;
    mark(s);
    mig_done++;
    return PK_OK;
  }
  int poll_migrations() {
    if (mig_list.empty()) return PK_OK;
    std::vector<int32_t> keep;
    for (int32_t s : mig_list) {
      RET(finish_migration(s, false));
      if (mig_ev[s]) keep.push_back(s);
    }
    mig_list.swap(keep);
    return PK_OK;
  }
  // Return the previous batch's staging ranges to the arena.  No host wait:
  // every later reader / writer of arena rows on the index stream is ordered
  // after that batch, and the migration stream waits for the index stream
  // before each admission copy (pk_list_set_resident).
  int release_staged() {
    if (!stage_pending) return PK_OK;
    for (const Range& r : staged) free_range(r.off, r.cap);
    staged.clear();
    stage_pending = false;
    return PK_OK;
  }
  // Before the host writes into the pinned host arena: the last batch's
  // zero-copy gather (or staging DMA) may still be reading it.
  int host_fence() {
    if (stage_recorded) CK(cudaEventSynchronize(stage_ev));
    stage_recorded = false;
    return PK_OK;
  }
  // Stream every cold list probed by the batch into arena staging ranges.
  int stage_cold(int64_t B, int32_t nprobe, const int32_t* probe_dev) {
    bool any = false;
    for (int32_t s = 0; s < nslots && !any; s++)
      any = h_cid[s] >= 0 && !h_res[s] && h_len[s] > 0;
    st_lists_last = st_rows_last = 0;
    if (!any) return PK_OK;
    std::vector<int32_t> pr((size_t)B * nprobe);
    CK(cudaMemcpyAsync(pr.data(), probe_dev, pr.size() * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::vector<uint8_t> seen(nslots, 0);
    std::vector<StageCopy> desc;
    for (int32_t v : pr) {
      if (v < 0 || seen[v]) continue;
      seen[v] = 1;
      if (h_res[v] || h_cid[v] < 0 || h_len[v] == 0) continue;
      int64_t off;
      RET(alloc_range(h_len[v], &off));
      StageCopy c;
      c.src_row = h_hoff[v];
      c.dst_row = off;
      c.n = (int32_t)h_len[v];
      c.pad = 0;
      desc.push_back(c);
      staged.push_back({off, h_len[v]});
      h_off[v] = off;
      mark(v);
      st_rows_last += h_len[v];
    }
    if (desc.empty()) return PK_OK;
    st_lists_last = (int64_t)desc.size();
    st_rows_total += st_rows_last;
    st_batches++;
    RET(stage_desc.ensure(desc.size() * sizeof(StageCopy)));
    CK(cudaMemcpyAsync(stage_desc.p, desc.data(), desc.size() * sizeof(StageCopy),
                       cudaMemcpyHostToDevice, st));
    if (stage_dma) {
      // copy engines for the rows: one DMA per run of lists contiguous on both
      // sides (multi-MB transfers run at ~52-55 GB/s on Gen5 x16; the ids are
      // too small for a DMA each and come with the norms kernel, zero-copy)
      size_t i = 0;
      while (i < desc.size()) {
        size_t j = i + 1;
        int64_t n = desc[i].n;
        while (j < desc.size() && desc[j].src_row == desc[i].src_row + n &&
               desc[j].dst_row == desc[i].dst_row + n) {
          n += desc[j].n;
          j++;
        }
        const int64_t s0 = desc[i].src_row, d0 = desc[i].dst_row;
        RET(for_host_pieces(s0, n, [&](int64_t r0, int64_t m) {
          CK(cudaMemcpyAsync(rows + (d0 + r0 - s0) * dp, hrows + r0 * dp, (size_t)m * dp * 4,
                             cudaMemcpyHostToDevice, st));
          return PK_OK;
        }));
        i = j;
      }
      launch_stage_norms(stage_desc.as<StageCopy>(), (int)desc.size(), rows, nrm, (int)dp, hids_d, ids, st);
    } else {
      launch_gather_rows(stage_desc.as<StageCopy>(), (int)desc.size(), hrows_d, hids_d, rows, ids, nrm,
                         (int)dp, st);
    }
    CK(cudaGetLastError());
    // the batch's device work reads these ranges; the next search frees them
    // (stream-ordered) and host-arena writers wait for stage_ev
    CK(cudaEventRecord(stage_ev, st));
    stage_pending = true;
    stage_recorded = true;
    return sync_table();
  }
  // Padded device copy of slot s's rows (resident: the arena itself).
  int rows_on_device(int32_t s, const float** out) {
    if (!tiered || h_res[s]) {
      *out = rows + h_off[s] * dp;
      return PK_OK;
    }
    RET(tmp_rows.ensure((size_t)std::max<int64_t>(h_len[s], 1) * dp * 4));
    RET(for_host_pieces(h_hoff[s], h_len[s], [&](int64_t r0, int64_t m) {
      CK(cudaMemcpyAsync(tmp_rows.as<float>() + (r0 - h_hoff[s]) * dp, hrows + r0 * dp, (size_t)m * dp * 4,
                         cudaMemcpyHostToDevice, st));
      return PK_OK;
    }));
    *out = tmp_rows.as<float>();
    return PK_OK;
  }

  int slot_of(int64_t cid, int32_t* s) {
    auto it = cid2slot.find(cid);
    if (it == cid2slot.end()) return fail(PK_ERR_USAGE, "unknown cluster %lld", (long long)cid);
    *s = it->second;
    return PK_OK;
  }

  // Copy n rows [n][d] (host or device, contiguous) into arena rows at `at`.
  int put_rows(int64_t at, const float* src, const int64_t* src_ids, int64_t n, bool dev) {
    if (n <= 0) return PK_OK;
    cudaMemcpyKind k = dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    CK(cudaMemcpy2DAsync(rows + at * dp, dp * 4, src, d * 4, d * 4, n, k, st));
    CK(cudaMemcpyAsync(ids + at, src_ids, n * 8, k, st));
    launch_row_norms(rows + at * dp, n, (int)dp, nrm + at, st);
    CK(cudaGetLastError());
    if (!dev) CK(cudaStreamSynchronize(st));  // pageable/pinned source reusable on return
    return PK_OK;
  }
};

// Default context for the stateless kernel-table entry points.
namespace {
// rows [n][d] -> pinned [n][dp] (zero pad columns)
void pack_padded(float* dst, const float* src, int64_t n, int64_t d, int64_t dp) {
  if (d == dp) {
    memcpy(dst, src, (size_t)n * d * 4);
    return;
  }
  for (int64_t i = 0; i < n; i++) {
    memcpy(dst + i * dp, src + i * d, (size_t)d * 4);
    memset(dst + i * dp + d, 0, (size_t)(dp - d) * 4);
  }
}
struct Ctx {
  cudaStream_t st = nullptr;
  DevBuf a, b, c, e;
  PinnedBuf hin, hout;
  std::mutex mu;
};
Ctx& ctx() {
  static Ctx c;
  static std::once_flag once;
  std::call_once(once, [] { cudaStreamCreateWithFlags(&c.st, cudaStreamNonBlocking); });
  return c;
}

int stage_padded(DevBuf& buf, const float* src, int64_t n, int64_t d, int64_t dp, bool dev,
                 cudaStream_t st) {
  RET(buf.ensure((size_t)std::max<int64_t>(n, 1) * dp * 4));
  CK(cudaMemsetAsync(buf.p, 0, (size_t)std::max<int64_t>(n, 1) * dp * 4, st));
  if (n > 0)
    CK(cudaMemcpy2DAsync(buf.p, dp * 4, src, d * 4, d * 4, n,
                         dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
  return PK_OK;
}
}  // namespace

extern "C" {

const char* pk_last_error(void) { return g_err.c_str(); }
int pk_version(void) { return 1; }
int pk_device_count(int* n) {
  CK(cudaGetDeviceCount(n));
  return PK_OK;
}

int pk_distances(const float* q, int64_t B, const float* mat, int64_t n, int64_t d, int metric,
                 float* out, int flags) {
  if (B < 0 || n < 0 || d < 1) return fail(PK_ERR_USAGE, "bad shape");
  if (metric < 0 || metric > 2) return fail(PK_ERR_USAGE, "bad metric %d", metric);
  if (B == 0 || n == 0) return PK_OK;
  Ctx& C = ctx();
  std::lock_guard<std::mutex> lk(C.mu);
  const bool dev = flags & PK_DEVICE_PTRS;
  const int64_t dp = round_up(d, DC);
  // device rows already at the padded stride are used in place (no staging copy)
  const bool inplace = dev && dp == d;
  const float* qa = q;
  const float* xa = mat;
  // host inputs: pack [q | mat] padded into pinned memory.  Small calls (the
  // cache pools, L1 centroids: <= 1 MB) are zero-copy -- the kernel streams the
  // mapped buffer over PCIe and writes the distances back the same way, no
  // separate DMA operations, whose fixed cost dominates them (measured 38 -> 33
  // us at 16 x 1024, 60 -> 47 us at 64 x 1024); larger ones take one DMA each way.
  const size_t nin = (size_t)(B + n) * dp;
  const bool zero_copy = !dev && (nin + (size_t)B * n) * 4 <= ((size_t)1 << 20);
  if (!dev) {
    RET(C.hin.ensure(nin * 4));
    float* h = reinterpret_cast<float*>(C.hin.p);
    pack_padded(h, q, B, d, dp);
    pack_padded(h + (size_t)B * dp, mat, n, d, dp);
    if (zero_copy) {
      qa = reinterpret_cast<const float*>(C.hin.dev);
    } else {
      RET(C.a.ensure(nin * 4));
      CK(cudaMemcpyAsync(C.a.p, h, nin * 4, cudaMemcpyHostToDevice, C.st));
      qa = C.a.as<float>();
    }
    xa = qa + (size_t)B * dp;
  } else if (!inplace) {
    RET(stage_padded(C.a, q, B, d, dp, dev, C.st));
    RET(stage_padded(C.b, mat, n, d, dp, dev, C.st));
    qa = C.a.as<float>();
    xa = C.b.as<float>();
  }
  RET(C.e.ensure(B * 4));
  if (metric == COSINE) launch_qnorm(qa, dp, (int)B, (int)d, C.e.as<float>(), C.st);
  float* D = out;
  if (!dev) {
    RET(C.hout.ensure((size_t)B * n * 4));
    if (zero_copy) {
      D = reinterpret_cast<float*>(C.hout.dev);
    } else {
      RET(C.c.ensure((size_t)B * n * 4));
      D = C.c.as<float>();
    }
  }
  launch_dist_dense(metric, qa, dp, (int)B, xa, dp, n, (int)dp, C.e.as<float>(), D, n, C.st);
  CK(cudaGetLastError());
  if (!dev && !zero_copy)
    CK(cudaMemcpyAsync(C.hout.p, D, (size_t)B * n * 4, cudaMemcpyDeviceToHost, C.st));
  CK(cudaStreamSynchronize(C.st));
  if (!dev) memcpy(out, C.hout.p, (size_t)B * n * 4);
  return PK_OK;
}

int pk_kmeans_assign(const float* x, int64_t n, const float* cents, int64_t k, int64_t d,
                     int64_t* labels, double* dists, int flags) {
  if (n < 0 || k < 1 || d < 1) return fail(PK_ERR_USAGE, "bad shape");
  if (n == 0) return PK_OK;
  Ctx& C = ctx();
  std::lock_guard<std::mutex> lk(C.mu);
  const bool dev = flags & PK_DEVICE_PTRS;
  const int64_t dp = round_up(d, DC);
  const float* xa = x;
  const float* ca = cents;
  if (!(dev && dp == d)) {  // device rows at the padded stride are used in place
    RET(stage_padded(C.a, x, n, d, dp, dev, C.st));
    RET(stage_padded(C.b, cents, k, d, dp, dev, C.st));
    xa = C.a.as<float>();
    ca = C.b.as<float>();
  }
  int64_t* L = labels;
  double* Dd = dists;
  if (!dev) {
    RET(C.c.ensure((size_t)n * 16));
    L = C.c.as<int64_t>();
    Dd = reinterpret_cast<double*>(L + n);
  }
  launch_kmeans_assign(xa, dp, n, ca, dp, k, (int)dp, L, Dd, C.st);
  CK(cudaGetLastError());
  if (!dev) {
    CK(cudaMemcpyAsync(labels, L, n * 8, cudaMemcpyDeviceToHost, C.st));
    if (dists) CK(cudaMemcpyAsync(dists, Dd, n * 8, cudaMemcpyDeviceToHost, C.st));
  }
  CK(cudaStreamSynchronize(C.st));
  return PK_OK;
}

int pk_centroid(const float* mat, int64_t n, int64_t d, float* out, int flags) {
  if (n < 1 || d < 1) return fail(PK_ERR_USAGE, "centroid of empty vector list");
  Ctx& C = ctx();
  std::lock_guard<std::mutex> lk(C.mu);
  const bool dev = flags & PK_DEVICE_PTRS;
  const int64_t dp = round_up(d, DC);
  RET(stage_padded(C.a, mat, n, d, dp, dev, C.st));
  RET(C.c.ensure(dp * 4));
  launch_centroid(C.a.as<float>(), dp, n, (int)dp, C.c.as<float>(), C.st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, C.c.p, d * 4, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                     C.st));
  CK(cudaStreamSynchronize(C.st));
  return PK_OK;
}

int pk_centroids_segmented(const float* rows, int64_t n, int64_t d, const int64_t* off, int64_t k,
                           float* out, int flags) {
  if (n < 0 || d < 1 || k < 1) return fail(PK_ERR_USAGE, "bad shape");
  if (!(flags & PK_DEVICE_PTRS)) return fail(PK_ERR_USAGE, "segmented centroids take device pointers");
  Ctx& C = ctx();
  std::lock_guard<std::mutex> lk(C.mu);
  launch_seg_centroid(rows, d, off, (int)k, (int)d, out, C.st);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(C.st));
  return PK_OK;
}

int pk_index_create(int64_t dim, int metric, int device, int64_t reserve_rows,
                    int64_t reserve_lists, pk_index** out) {
  if (dim < 1) return fail(PK_ERR_USAGE, "dimension must be >= 1, got %lld", (long long)dim);
  if (metric < 0 || metric > 2) return fail(PK_ERR_USAGE, "bad metric %d", metric);
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(PK_ERR_USAGE, "no CUDA device %d", device);
  CK(cudaSetDevice(device));
  pk_index* ix = new pk_index();
  ix->device = device;
  ix->d = dim;
  ix->dp = round_up(dim, DC);
  ix->metric = metric;
  cudaDeviceGetAttribute(&ix->num_sms, cudaDevAttrMultiProcessorCount, device);
  ix->scan_sms = ix->num_sms;
  if (const char* e = getenv("PK_SCAN_SMS")) ix->scan_sms = std::max(1, std::min(ix->num_sms, atoi(e)));
  if (const char* e = getenv("PK_CHUNK_ROWS")) ix->chunk_rows = std::max(TILE, atoi(e) / TILE * TILE);
  if (const char* e = getenv("PK_SCAN_EXACT")) ix->screen = atoi(e) == 0;
  if (const char* e = getenv("PK_POOL_CAP")) {
    ix->pool_cap = std::max(1, atoi(e));
    ix->pool_cap_set = true;
  }
  if (const char* e = getenv("PK_SCREEN")) ix->tensor = strcmp(e, "ffma") != 0;
  if (const char* e = getenv("PK_PIPELINE")) ix->pipeline = atoi(e) != 0;
  if (const char* e = getenv("PK_RERANK_LEAN")) ix->rr_lean = atoi(e) != 0 ? 1 : 0;
  if (const char* e = getenv("PK_RERANK_DEFER")) ix->rr_defer = atoi(e) != 0;
  ix->tl.on = getenv("PK_DEBUG_TIMELINE") != nullptr;
  if (const char* e = getenv("PK_SCAN_OVERLAP")) ix->scan_ovl = atoi(e) != 0;
  ix->rr_lean_ctas = ix->num_sms;
  if (const char* e = getenv("PK_RERANK_LEAN_CTAS")) ix->rr_lean_ctas = std::max(1, atoi(e));
  if (const char* e = getenv("PK_QGATHER")) ix->qgather = atoi(e) != 0;
  if (const char* e = getenv("PK_STAGE")) ix->stage_dma = strcmp(e, "dma") == 0;
  if (const char* e = getenv("PK_COARSE")) {
    ix->coarse_tc = strcmp(e, "exact") != 0;
    ix->coarse_split = strcmp(e, "tf32") != 0;
  }
  if (metric == COSINE) ix->coarse_tc = false;
  if (metric == COSINE) ix->screen = false;
  if (ix->screen) ix->chunk_rows = std::min(ix->chunk_rows, 2 * TILE);
  cudaError_t e = cudaStreamCreateWithFlags(&ix->st, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete ix;
    return fail(PK_ERR_DEVICE, "stream create failed: %s", cudaGetErrorString(e));
  }
  int r = ix->grow_arena(std::max<int64_t>(reserve_rows, 1024));
  if (r == PK_OK) r = ix->grow_slots((int32_t)std::max<int64_t>(reserve_lists, 64));
  if (r != PK_OK) {
    pk_index_destroy(ix);
    return r;
  }
  *out = ix;
  return PK_OK;
}

int pk_index_destroy(pk_index* ix) {
  if (!ix) return PK_OK;
  cudaSetDevice(ix->device);
  for (cudaStream_t x : {ix->fst, ix->sst, ix->sst2, ix->rst, ix->cst, ix->st})
    if (x) cudaStreamSynchronize(x);
  cudaFree(ix->rows);
  cudaFree(ix->ids);
  cudaFree(ix->nrm);
  cudaFree(ix->d_off);
  cudaFree(ix->d_len);
  cudaFree(ix->d_cid);
  cudaFree(ix->d_scope);
  cudaFree(ix->d_cent);
  cudaFree(ix->d_cnrm);
  cudaFree(ix->d_chi);
  cudaFree(ix->d_clo);
  ix->graph.release();
  for (cudaEvent_t e : ix->prof_ev) cudaEventDestroy(e);
  if (ix->mst) cudaStreamSynchronize(ix->mst);
  for (cudaEvent_t e : ix->mig_ev)
    if (e) cudaEventDestroy(e);
  if (ix->stage_ev) cudaEventDestroy(ix->stage_ev);
  if (ix->mst) cudaStreamDestroy(ix->mst);
  if (ix->hout) cudaFreeHost(ix->hout);
  for (int i = 0; i < 2; i++) {
    if (ix->hstage2[i].p) cudaFreeHost(ix->hstage2[i].p);
    if (ix->hstage_ev[i]) cudaEventDestroy(ix->hstage_ev[i]);
    ix->tmp_rows2[i].release();
  }
  if (ix->hsl.p) cudaFreeHost(ix->hsl.p);
  if (ix->hasg.p) cudaFreeHost(ix->hasg.p);
  for (int i = 0; i < 2; i++) {
    if (ix->tstage[i].p) cudaFreeHost(ix->tstage[i].p);
    if (ix->tstage_ev[i]) cudaEventDestroy(ix->tstage_ev[i]);
  }
  if (ix->hag.p) cudaFreeHost(ix->hag.p);
  if (ix->hal.p) cudaFreeHost(ix->hal.p);
  ix->al_in.release();
  ix->arows.release();
  ix->ag_in.release();
  ix->ag_l1.release();
  for (auto& a : ix->aslot) {
    if (a.hblk) cudaFreeHost(a.hblk);
    if (a.copied) cudaEventDestroy(a.copied);
    if (a.done) cudaEventDestroy(a.done);
    if (a.consumed) cudaEventDestroy(a.consumed);
    if (a.ready) cudaEventDestroy(a.ready);
    a.qin.release();
    a.blk.release();
  }
  if (ix->cst) cudaStreamDestroy(ix->cst);
  if (ix->rst) {
    cudaStreamSynchronize(ix->rst);
    cudaStreamDestroy(ix->rst);
  }
  if (ix->fst) {
    cudaStreamSynchronize(ix->fst);
    cudaStreamDestroy(ix->fst);
  }
  for (cudaStream_t x : {ix->sst, ix->sst2})
    if (x) {
      cudaStreamSynchronize(x);
      cudaStreamDestroy(x);
    }
  if (ix->ast) {
    cudaStreamSynchronize(ix->ast);
    cudaStreamDestroy(ix->ast);
  }
  for (cudaEvent_t e : {ix->ev_ag0, ix->ev_ag1})
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : {ix->ev_front, ix->ev_scan, ix->ev_sdone, ix->ev_free[0], ix->ev_free[1], ix->ev_free[2]})
    if (e) cudaEventDestroy(e);
  for (uint8_t* p : ix->comb.opened) cudaIpcCloseMemHandle(p);
  if (ix->comb.area) cudaFree(ix->comb.area);
  if (ix->comb.d_peers) cudaFree(ix->comb.d_peers);
  if (ix->comb.done_ctr) cudaFree(ix->comb.done_ctr);
  if (ix->hva_rows) {
    for (size_t i = 0; i < ix->hseg.size(); i++) {
      cudaHostUnregister(reinterpret_cast<char*>(ix->hva_rows) + (size_t)ix->hseg[i] * ix->dp * 4);
      cudaHostUnregister(reinterpret_cast<char*>(ix->hva_ids) + (size_t)ix->hseg[i] * 8);
    }
    munmap(ix->hva_rows, ix->hva_rows_bytes);
    munmap(ix->hva_ids, ix->hva_ids_bytes);
  } else {
    if (ix->hrows) cudaFreeHost(ix->hrows);
    if (ix->hids) cudaFreeHost(ix->hids);
  }
  ix->stage_desc.release();
  ix->tmp_rows.release();
  for (auto& sc : ix->scr) sc.release();
  for (DevBuf* b : {&ix->assign_part, &ix->assign_ctr, &ix->assign_q, &ix->assign_qn, &ix->assign_dc, &ix->assign_c, &ix->assign_d,
                    &ix->shard_in, &ix->shard_out, &ix->pb, &ix->pb_out, &ix->sl_buf})
    b->release();
  if (ix->st) cudaStreamDestroy(ix->st);
  delete ix;
  return PK_OK;
}

int pk_sync(pk_index* ix) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  CK(cudaStreamSynchronize(ix->st));
  return PK_OK;
}
void* pk_stream(pk_index* ix) { return ix ? (void*)ix->st : nullptr; }
int pk_index_bytes(pk_index* ix, int64_t* bytes) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  *bytes = ix->arena_cap * (ix->dp * 4 + 8) + (int64_t)ix->slot_cap * (ix->dp * 4 + 28);
  return PK_OK;
}

int pk_list_create(pk_index* ix, int64_t cid, int32_t scope_code, const float* rows,
                   const int64_t* ids, int64_t n, float* out_centroid, int flags) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  if (n < 1) return fail(PK_ERR_USAGE, "create_cluster needs at least one seed item");
  if (ix->cid2slot.count(cid)) return fail(PK_ERR_USAGE, "cluster %lld exists", (long long)cid);
  CK(cudaSetDevice(ix->device));
  int32_t s;
  if (!ix->free_slots.empty()) {
    s = ix->free_slots.back();
    ix->free_slots.pop_back();
  } else {
    if (ix->nslots == ix->slot_cap) RET(ix->grow_slots(ix->nslots + 1));
    s = ix->nslots++;
  }
  const int64_t cap = n + n / 4 + 16;
  const bool dev = flags & PK_DEVICE_PTRS;
  const float* crow = nullptr;  // padded device rows the centroid is computed from
  if (ix->tiered) {
    // cold on creation (the reference admits lists through hotset_update):
    // host arena copy, centroid from a padded device staging copy
    int64_t hoff;
    RET(ix->host_alloc(cap, &hoff));
    RET(ix->host_put(hoff, rows, ids, n, dev));
    ix->h_hoff[s] = hoff;
    ix->h_hcap[s] = cap;
    ix->h_res[s] = 0;
    ix->h_off[s] = 0;
    ix->h_cap[s] = 0;
    RET(ix->tmp_rows.ensure((size_t)n * ix->dp * 4));
    CK(cudaMemsetAsync(ix->tmp_rows.p, 0, (size_t)n * ix->dp * 4, ix->st));
    CK(cudaMemcpy2DAsync(ix->tmp_rows.p, ix->dp * 4, rows, ix->d * 4, ix->d * 4, n,
                         dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, ix->st));
    crow = ix->tmp_rows.as<float>();
  } else {
    int64_t off;
    RET(ix->alloc_range(cap, &off));
    RET(ix->put_rows(off, rows, ids, n, dev));
    ix->h_off[s] = off;
    ix->h_cap[s] = cap;
    ix->h_res[s] = 1;
    crow = ix->rows + off * ix->dp;
  }
  ix->h_len[s] = n;
  ix->h_cid[s] = cid;
  ix->h_scope[s] = scope_code;
  ix->h_remote[s] = 0;
  ix->cid2slot[cid] = s;
  ix->slot_ver++;
  ix->mark(s);
  launch_centroid(crow, ix->dp, n, (int)ix->dp, ix->d_cent + (int64_t)s * ix->dp, ix->st);
  ix->centroid_norm(s);
  CK(cudaGetLastError());
  if (out_centroid) {
    CK(cudaMemcpyAsync(out_centroid, ix->d_cent + (int64_t)s * ix->dp, ix->d * 4,
                       cudaMemcpyDeviceToHost, ix->st));
    CK(cudaStreamSynchronize(ix->st));
  }
  return PK_OK;
}

int pk_list_add_remote(pk_index* ix, int64_t cid, int32_t scope_code, const float* centroid) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  if (ix->cid2slot.count(cid)) return fail(PK_ERR_USAGE, "cluster %lld exists", (long long)cid);
  if (!centroid) return fail(PK_ERR_USAGE, "remote list needs a centroid");
  CK(cudaSetDevice(ix->device));
  int32_t s;
  if (!ix->free_slots.empty()) {
    s = ix->free_slots.back();
    ix->free_slots.pop_back();
  } else {
    if (ix->nslots == ix->slot_cap) RET(ix->grow_slots(ix->nslots + 1));
    s = ix->nslots++;
  }
  ix->h_off[s] = 0;
  ix->h_len[s] = 0;
  ix->h_cap[s] = 0;
  ix->h_cid[s] = cid;
  ix->h_scope[s] = scope_code;
  ix->h_remote[s] = 1;
  ix->h_res[s] = 1;  // never staged: no rows here
  ix->cid2slot[cid] = s;
  ix->slot_ver++;
  ix->mark(s);
  CK(cudaMemcpyAsync(ix->d_cent + (int64_t)s * ix->dp, centroid, ix->d * 4, cudaMemcpyHostToDevice,
                     ix->st));
  ix->centroid_norm(s);
  CK(cudaStreamSynchronize(ix->st));
  return PK_OK;
}

int64_t pk_shard_block_bytes(int64_t B, int32_t kk) {
  if (B < 0 || kk < 1) return 0;
  const int64_t nkk = B * kk;
  return round_up(nkk * 20 + B * 12, 16);
}

int pk_merge_shards(pk_index* ix, const void* blocks, int32_t R, int64_t B, int32_t kk,
                    int64_t* out_ids, float* out_dists, int64_t* out_cids, int32_t* out_n,
                    int64_t* out_scanned, int flags) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  if (R < 1 || B < 0) return fail(PK_ERR_USAGE, "bad shard count / batch");
  if (kk < 1 || kk > KKMAX) return fail(PK_ERR_USAGE, "kk must lie in [1, %d]", KKMAX);
  if ((int64_t)R * kk > shard_merge_cap())
    return fail(PK_ERR_USAGE, "shards x kk above %d", shard_merge_cap());
  if (B == 0) return PK_OK;
  CK(cudaSetDevice(ix->device));
  const bool dev = flags & PK_DEVICE_PTRS;
  // a device merge touches neither the list table nor the search scratch, so
  // a search -> merge -> search sequence keeps the front-half overlap
  if (dev && ix->ev_scan && ix->mu.n == ix->ev_scan_n + 2) ix->ev_scan_n++;
  cudaStream_t st = ix->st;
  const int64_t bb = pk_shard_block_bytes(B, kk);
  const void* src = blocks;
  int64_t *o_ids = out_ids, *o_cid = out_cids, *o_sc = out_scanned;
  float* o_d = out_dists;
  int32_t* o_n = out_n;
  if (!dev) {
    RET(ix->shard_in.ensure((size_t)R * bb));
    CK(cudaMemcpyAsync(ix->shard_in.p, blocks, (size_t)R * bb, cudaMemcpyHostToDevice, st));
    src = ix->shard_in.p;
    RET(ix->shard_out.ensure((size_t)bb));  // same layout as a block
    uint8_t* base = ix->shard_out.as<uint8_t>();
    const int64_t nkk = B * kk;
    o_ids = reinterpret_cast<int64_t*>(base);
    o_cid = reinterpret_cast<int64_t*>(base + 8 * nkk);
    o_sc = reinterpret_cast<int64_t*>(base + 16 * nkk);
    o_d = reinterpret_cast<float*>(base + 16 * nkk + 8 * B);
    o_n = reinterpret_cast<int32_t*>(base + 20 * nkk + 8 * B);
  }
  launch_shard_merge(ix->metric, src, bb, R, (int)B, kk, o_ids, o_d, (dev && !out_cids) ? nullptr : o_cid, o_n,
                     (dev && !out_scanned) ? nullptr : o_sc, st);
  CK(cudaGetLastError());
  if (!dev) {
    CK(cudaMemcpyAsync(out_ids, o_ids, (size_t)B * kk * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(out_dists, o_d, (size_t)B * kk * 4, cudaMemcpyDeviceToHost, st));
    if (out_cids) CK(cudaMemcpyAsync(out_cids, o_cid, (size_t)B * kk * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(out_n, o_n, (size_t)B * 4, cudaMemcpyDeviceToHost, st));
    if (out_scanned) CK(cudaMemcpyAsync(out_scanned, o_sc, (size_t)B * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  return PK_OK;
}

int pk_list_append(pk_index* ix, int64_t cid, const float* rows, const int64_t* ids, int64_t n,
                   int flags) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  if (n <= 0) return PK_OK;
  CK(cudaSetDevice(ix->device));
  int32_t s;
  RET(ix->slot_of(cid, &s));
  if (ix->h_remote[s]) return fail(PK_ERR_USAGE, "cluster %lld is owned by another shard", (long long)cid);
  const int64_t len = ix->h_len[s];
  if (ix->tiered) {
    RET(ix->finish_migration(s, true));
    RET(ix->host_fence());
    if (len + n > ix->h_hcap[s]) {  // relocate the host copy (x1.5)
      const int64_t ncap = std::max<int64_t>(len + n, ix->h_hcap[s] + ix->h_hcap[s] / 2) + 16;
      int64_t noff;
      RET(ix->host_alloc(ncap, &noff));
      memcpy(ix->hrows + noff * ix->dp, ix->hrows + ix->h_hoff[s] * ix->dp, (size_t)len * ix->dp * 4);
      memcpy(ix->hids + noff, ix->hids + ix->h_hoff[s], (size_t)len * 8);
      ix->host_free(ix->h_hoff[s], ix->h_hcap[s]);
      ix->h_hoff[s] = noff;
      ix->h_hcap[s] = ncap;
    }
    RET(ix->host_put(ix->h_hoff[s] + len, rows, ids, n, flags & PK_DEVICE_PTRS));
    if (!ix->h_res[s]) {
      ix->h_len[s] = len + n;
      ix->mark(s);
      return PK_OK;
    }
  }
  if (len + n > ix->h_cap[s]) {
    // relocate into a larger range (Cluster._grow x1.5, ref/clusters.py:61-69)
    const int64_t ncap = std::max<int64_t>(len + n, ix->h_cap[s] + ix->h_cap[s] / 2) + 16;
    int64_t noff;
    RET(ix->alloc_range(ncap, &noff));
    const int64_t ooff = ix->h_off[s];
    if (len > 0) {
      CK(cudaMemcpyAsync(ix->rows + noff * ix->dp, ix->rows + ooff * ix->dp,
                         (size_t)len * ix->dp * 4, cudaMemcpyDeviceToDevice, ix->st));
      CK(cudaMemcpyAsync(ix->ids + noff, ix->ids + ooff, (size_t)len * 8,
                         cudaMemcpyDeviceToDevice, ix->st));
      CK(cudaMemcpyAsync(ix->nrm + noff, ix->nrm + ooff, (size_t)len * 4,
                         cudaMemcpyDeviceToDevice, ix->st));
    }
    ix->free_range(ooff, ix->h_cap[s]);
    ix->h_off[s] = noff;
    ix->h_cap[s] = ncap;
  }
  RET(ix->put_rows(ix->h_off[s] + len, rows, ids, n, flags & PK_DEVICE_PTRS));
  ix->h_len[s] = len + n;
  ix->mark(s);
  return PK_OK;
}

int pk_list_append_batch(pk_index* ix, int64_t n, const int64_t* cids, const float* rows,
                         const int64_t* ids) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  if (n <= 0) return PK_OK;
  CK(cudaSetDevice(ix->device));
  // pre-pass: slots, per-slot counts, capacity (one relocation per list at most)
  std::vector<int32_t> slot(n);
  std::unordered_map<int32_t, int64_t> add;
  for (int64_t i = 0; i < n; i++) {
    RET(ix->slot_of(cids[i], &slot[i]));
    if (ix->h_remote[slot[i]])
      return fail(PK_ERR_USAGE, "cluster %lld is owned by another shard", (long long)cids[i]);
    add[slot[i]] += 1;
  }
  std::unordered_map<int32_t, bool> moved;  // slots whose arena range changed
  for (auto& kv : add) {
    const int32_t s = kv.first;
    const int64_t len = ix->h_len[s], m = kv.second;
    if (ix->tiered) {
      RET(ix->finish_migration(s, true));
      RET(ix->host_fence());
      if (len + m > ix->h_hcap[s]) {
        const int64_t ncap = std::max<int64_t>(len + m, ix->h_hcap[s] + ix->h_hcap[s] / 2) + 16;
        int64_t noff;
        RET(ix->host_alloc(ncap, &noff));
        memcpy(ix->hrows + noff * ix->dp, ix->hrows + ix->h_hoff[s] * ix->dp, (size_t)len * ix->dp * 4);
        memcpy(ix->hids + noff, ix->hids + ix->h_hoff[s], (size_t)len * 8);
        ix->host_free(ix->h_hoff[s], ix->h_hcap[s]);
        ix->h_hoff[s] = noff;
        ix->h_hcap[s] = ncap;
      }
    }
    if (ix->h_res[s] && len + m > ix->h_cap[s]) {
      const int64_t ncap = std::max<int64_t>(len + m, ix->h_cap[s] + ix->h_cap[s] / 2) + 16;
      int64_t noff;
      RET(ix->alloc_range(ncap, &noff));
      const int64_t ooff = ix->h_off[s];
      if (len > 0) {
        CK(cudaMemcpyAsync(ix->rows + noff * ix->dp, ix->rows + ooff * ix->dp,
                           (size_t)len * ix->dp * 4, cudaMemcpyDeviceToDevice, ix->st));
        CK(cudaMemcpyAsync(ix->ids + noff, ix->ids + ooff, (size_t)len * 8,
                           cudaMemcpyDeviceToDevice, ix->st));
        CK(cudaMemcpyAsync(ix->nrm + noff, ix->nrm + ooff, (size_t)len * 4,
                           cudaMemcpyDeviceToDevice, ix->st));
      }
      ix->free_range(ooff, ix->h_cap[s]);
      ix->h_off[s] = noff;
      ix->h_cap[s] = ncap;
      moved[s] = true;
    }
  }
  // placement in batch order; host copies now, device rows by one scatter
  std::vector<int64_t> dst;
  std::vector<int64_t> pick;
  for (int64_t i = 0; i < n; i++) {
    const int32_t s = slot[i];
    const int64_t pos = ix->h_len[s]++;
    if (ix->tiered) RET(ix->host_put(ix->h_hoff[s] + pos, rows + i * ix->d, ids + i, 1, false));
    if (ix->h_res[s]) {
      dst.push_back(ix->h_off[s] + pos);
      pick.push_back(i);
    }
  }
  // resident lists that only grew: their new lengths ride with the scatter
  // (len_pairs); any other change goes through the table sync
  std::vector<int64_t> lp;
  for (auto& kv : add) {
    const int32_t s = kv.first;
    if (ix->h_res[s] && !moved.count(s)) {
      lp.push_back(s);
      lp.push_back(ix->h_len[s]);
      ix->touch();
    } else {
      ix->mark(s);
    }
  }
  const int64_t m = (int64_t)dst.size();
  const int nlp = (int)(lp.size() / 2);
  if (m > 0) {
    // [rows padded | ids | destinations | (slot, len) pairs] packed once into
    // mapped pinned memory; small batches are read by the scatter kernel in
    // place (no DMA operations), larger ones go over in one copy
    const size_t bytes = (size_t)m * ix->dp * 4 + (size_t)m * 16 + lp.size() * 8;
    const int bi = ix->hstage_i;
    ix->hstage_i ^= 1;
    PinnedBuf& hs = ix->hstage2[bi];
    if (!ix->hstage_ev[bi]) CK(cudaEventCreateWithFlags(&ix->hstage_ev[bi], cudaEventDisableTiming));
    else CK(cudaEventSynchronize(ix->hstage_ev[bi]));  // its previous scatter has read it
    if (hs.bytes < bytes) CK(cudaStreamSynchronize(ix->st));  // (re)allocation frees the old buffer
    RET(hs.ensure(bytes));
    float* h_src = reinterpret_cast<float*>(hs.p);
    int64_t* h_ids = reinterpret_cast<int64_t*>(h_src + m * ix->dp);
    int64_t* h_dst = h_ids + m;
    for (int64_t j = 0; j < m; j++) {
      memcpy(h_src + j * ix->dp, rows + pick[j] * ix->d, ix->d * 4);
      if (ix->dp > ix->d) memset(h_src + j * ix->dp + ix->d, 0, (ix->dp - ix->d) * 4);
      h_ids[j] = ids[pick[j]];
      h_dst[j] = dst[j];
    }
    if (nlp) memcpy(h_dst + m, lp.data(), lp.size() * 8);
    const uint8_t* base = hs.dev;
    if (bytes > ((size_t)1 << 20)) {
      if (ix->tmp_rows2[bi].bytes < bytes) CK(cudaStreamSynchronize(ix->st));
      RET(ix->tmp_rows2[bi].ensure(bytes));
      CK(cudaMemcpyAsync(ix->tmp_rows2[bi].p, hs.p, bytes, cudaMemcpyHostToDevice, ix->st));
      base = ix->tmp_rows2[bi].as<uint8_t>();
    }
    const float* d_src = reinterpret_cast<const float*>(base);
    const int64_t* d_ids = reinterpret_cast<const int64_t*>(d_src + m * ix->dp);
    launch_append_rows(d_src, d_ids, d_ids + m, (int)m, ix->rows, ix->ids, ix->nrm, (int)ix->dp, ix->st,
                       d_ids + 2 * m, nlp, ix->d_len);
    CK(cudaGetLastError());
    CK(cudaEventRecord(ix->hstage_ev[bi], ix->st));  // no host wait: ordered on the index stream
  }
  return PK_OK;
}

int pk_list_remove_row(pk_index* ix, int64_t cid, int64_t row) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  CK(cudaSetDevice(ix->device));
  int32_t s;
  RET(ix->slot_of(cid, &s));
  const int64_t len = ix->h_len[s];
  if (row < 0 || row >= len) return fail(PK_ERR_USAGE, "row %lld out of range", (long long)row);
  const int64_t last = len - 1, off = ix->h_off[s];
  if (ix->tiered) {
    RET(ix->finish_migration(s, true));
    RET(ix->host_fence());
    const int64_t ho = ix->h_hoff[s];
    if (row != last) {
      memcpy(ix->hrows + (ho + row) * ix->dp, ix->hrows + (ho + last) * ix->dp, ix->dp * 4);
      ix->hids[ho + row] = ix->hids[ho + last];
    }
    if (!ix->h_res[s]) {
      ix->h_len[s] = last;
      ix->mark(s);
      return PK_OK;
    }
  }
  if (row != last) {
    CK(cudaMemcpyAsync(ix->rows + (off + row) * ix->dp, ix->rows + (off + last) * ix->dp,
                       ix->dp * 4, cudaMemcpyDeviceToDevice, ix->st));
    CK(cudaMemcpyAsync(ix->ids + off + row, ix->ids + off + last, 8, cudaMemcpyDeviceToDevice,
                       ix->st));
    CK(cudaMemcpyAsync(ix->nrm + off + row, ix->nrm + off + last, 4, cudaMemcpyDeviceToDevice,
                       ix->st));
  }
  ix->h_len[s] = last;
  ix->mark(s);
  return PK_OK;
}

int pk_list_retire(pk_index* ix, int64_t cid) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  int32_t s;
  RET(ix->slot_of(cid, &s));
  if (ix->tiered) {
    RET(ix->finish_migration(s, true));
    ix->host_free(ix->h_hoff[s], ix->h_hcap[s]);
    ix->h_hoff[s] = ix->h_hcap[s] = 0;
  }
  if (ix->h_res[s]) ix->free_range(ix->h_off[s], ix->h_cap[s]);
  ix->h_res[s] = 1;
  ix->h_cid[s] = -1;
  ix->h_len[s] = 0;
  ix->h_cap[s] = 0;
  ix->h_scope[s] = -1;
  ix->h_remote[s] = 0;
  ix->cid2slot.erase(cid);
  ix->slot_ver++;
  ix->free_slots.push_back(s);
  ix->mark(s);
  return PK_OK;
}

int pk_list_recompute(pk_index* ix, int64_t cid, float* out_centroid) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  CK(cudaSetDevice(ix->device));
  int32_t s;
  RET(ix->slot_of(cid, &s));
  const int64_t n = ix->h_len[s];
  if (n > 0) {
    const float* r = nullptr;
    RET(ix->rows_on_device(s, &r));
    launch_centroid(r, ix->dp, n, (int)ix->dp, ix->d_cent + (int64_t)s * ix->dp, ix->st);
  }
  ix->centroid_norm(s);
  CK(cudaGetLastError());
  if (out_centroid) {
    CK(cudaMemcpyAsync(out_centroid, ix->d_cent + (int64_t)s * ix->dp, ix->d * 4,
                       cudaMemcpyDeviceToHost, ix->st));
    CK(cudaStreamSynchronize(ix->st));
  }
  return PK_OK;
}

int pk_list_set_centroid(pk_index* ix, int64_t cid, const float* centroid) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  CK(cudaSetDevice(ix->device));
  int32_t s;
  RET(ix->slot_of(cid, &s));
  CK(cudaMemcpyAsync(ix->d_cent + (int64_t)s * ix->dp, centroid, ix->d * 4,
                     cudaMemcpyHostToDevice, ix->st));
  ix->centroid_norm(s);
  CK(cudaStreamSynchronize(ix->st));
  return PK_OK;
}

int pk_list_size(pk_index* ix, int64_t cid, int64_t* n) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  int32_t s;
  RET(ix->slot_of(cid, &s));
  *n = ix->h_len[s];
  return PK_OK;
}

int pk_list_read(pk_index* ix, int64_t cid, float* rows, int64_t* ids) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  CK(cudaSetDevice(ix->device));
  int32_t s;
  RET(ix->slot_of(cid, &s));
  const int64_t n = ix->h_len[s], off = ix->h_off[s];
  if (ix->tiered) {  // the host copy is always current
    const int64_t ho = ix->h_hoff[s];
    for (int64_t r = 0; rows && r < n; r++) memcpy(rows + r * ix->d, ix->hrows + (ho + r) * ix->dp, ix->d * 4);
    if (ids && n > 0) memcpy(ids, ix->hids + ho, n * 8);
    return PK_OK;
  }
  if (n > 0) {
    if (rows)
      CK(cudaMemcpy2DAsync(rows, ix->d * 4, ix->rows + off * ix->dp, ix->dp * 4, ix->d * 4, n,
                           cudaMemcpyDeviceToHost, ix->st));
    if (ids) CK(cudaMemcpyAsync(ids, ix->ids + off, n * 8, cudaMemcpyDeviceToHost, ix->st));
  }
  CK(cudaStreamSynchronize(ix->st));
  return PK_OK;
}

int pk_index_enable_tier(pk_index* ix, int64_t reserve_rows) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  if (ix->tiered) return PK_OK;
  if (ix->cid2slot.size() > 0) return fail(PK_ERR_USAGE, "enable the cold tier before creating lists");
  CK(cudaSetDevice(ix->device));
  CK(cudaStreamCreateWithFlags(&ix->mst, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&ix->stage_ev, cudaEventDisableTiming));
  RET(ix->host_grow(std::max<int64_t>(reserve_rows, 1024)));
  ix->tiered = true;
  return PK_OK;
}

int pk_list_set_resident(pk_index* ix, int64_t cid, int resident) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  if (!ix->tiered) return fail(PK_ERR_USAGE, "no cold tier: every list is HBM-resident");
  CK(cudaSetDevice(ix->device));
  int32_t s;
  RET(ix->slot_of(cid, &s));
  if (ix->h_remote[s]) return fail(PK_ERR_USAGE, "cluster %lld is owned by another shard", (long long)cid);
  if (resident) {
    if (ix->h_res[s] || ix->mig_ev[s]) return PK_OK;
    // admission: Allocated -> Copying (side stream) -> Switching at the next
    // poll once the copy event completes (TierManager.step_migration)
    const int64_t len = ix->h_len[s];
    const int64_t cap = len + len / 4 + 16;  // 25% device slack (ref/tiering.py:356)
    if (ix->fail_alloc > 0) {
      ix->fail_alloc--;
      return fail(PK_ERR_NOMEM, "admission of cluster %lld: injected allocation failure", (long long)cid);
    }
    int64_t off;
    RET(ix->alloc_range(cap, &off));
    // the range may have held rows (an evicted list, a finished batch's
    // staging) that searches already enqueued on the index stream still read
    CK(cudaEventRecord(ix->stage_ev, ix->st));
    CK(cudaStreamWaitEvent(ix->mst, ix->stage_ev, 0));
    ix->stage_recorded = true;
    if (len > 0) {
      const int64_t h0 = ix->h_hoff[s];
      RET(ix->for_host_pieces(h0, len, [&](int64_t r0, int64_t m) {
        CK(cudaMemcpyAsync(ix->rows + (off + r0 - h0) * ix->dp, ix->hrows + r0 * ix->dp,
                           (size_t)m * ix->dp * 4, cudaMemcpyHostToDevice, ix->mst));
        CK(cudaMemcpyAsync(ix->ids + off + r0 - h0, ix->hids + r0, (size_t)m * 8, cudaMemcpyHostToDevice,
                           ix->mst));
        return PK_OK;
      }));
      launch_row_norms(ix->rows + off * ix->dp, len, (int)ix->dp, ix->nrm + off, ix->mst);
      CK(cudaGetLastError());
    }
    cudaEvent_t ev;
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CK(cudaEventRecord(ev, ix->mst));
    ix->mig_ev[s] = ev;
    ix->mig_off[s] = off;
    ix->mig_cap[s] = cap;
    ix->mig_list.push_back(s);
    ix->mig_started++;
    return PK_OK;
  }
  RET(ix->finish_migration(s, true));
  if (ix->h_res[s]) {
    ix->free_range(ix->h_off[s], ix->h_cap[s]);
    ix->h_res[s] = 0;
    ix->h_off[s] = ix->h_cap[s] = 0;
    ix->mark(s);
  }
  return PK_OK;
}

int pk_list_residency(pk_index* ix, int64_t cid, int* state) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  int32_t s;
  RET(ix->slot_of(cid, &s));
  RET(ix->finish_migration(s, false));
  *state = ix->h_res[s] ? 1 : (ix->mig_ev[s] ? 2 : 0);
  return PK_OK;
}

int pk_tier_stats(pk_index* ix, int64_t* out, int n) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  int64_t v[12] = {0};
  if (ix->tiered) RET(ix->poll_migrations());
  for (int32_t s = 0; s < ix->nslots; s++) {
    if (ix->h_cid[s] < 0 || ix->h_remote[s]) continue;
    if (ix->h_res[s]) {
      v[0]++;
      v[2] += ix->h_cap[s] * (ix->dp * 4 + 8);
    } else {
      v[1]++;
    }
  }
  v[3] = ix->st_lists_last;
  v[4] = ix->st_rows_last * (ix->dp * 4 + 8);
  v[5] = ix->st_rows_total * (ix->dp * 4 + 8);
  v[6] = ix->st_batches;
  v[7] = ix->mig_started;
  v[8] = ix->mig_done;
  v[9] = ix->tiered ? ix->hcap * (ix->dp * 4 + 8) : 0;
  v[10] = ix->arena_top;  // HBM arena high-water mark (rows)
  v[11] = ix->arena_cap;  // HBM arena capacity (rows)
  for (int i = 0; i < n && i < 12; i++) out[i] = v[i];
  return PK_OK;
}

}  // extern "C"

// One batched search through the stages of pk_search.  probe_in (list
// handles, [B][nprobe]) skips the coarse stage; probe_out stops after it.
// in_dev / dev: input / output pointers are device pointers.
// Coarse stage by the reference's graph traversal instead of the flat
// top-nprobe (pk_search_graph): exact distances of every query to every
// list centroid (the values the reference's _dist returns), then the
// traversal kernel (pk_graph.cu).  `codes` are host scope codes.
struct GraphArgs {
  int32_t ef = 0, mode = 0;
  int32_t* out_coarse = nullptr;  // [B] distance computations (host unless coarse_dev)
  bool coarse_dev = false;
};
static int graph_coarse(pk_index* ix, pk_index::Scratch& S, int64_t B, const int32_t* codes,
                        int32_t nscopes, int32_t nprobe, const GraphArgs& ga, cudaStream_t fs) {
  pk_index::Graph& G = ix->graph;
  if (!G.set) return fail(PK_ERR_USAGE, "no coarse graph uploaded (pk_graph_set)");
  if (G.ns != ix->nslots || G.slot_ver != ix->slot_ver)
    return fail(PK_ERR_USAGE, "the coarse graph is stale: lists changed since pk_graph_set");
  const int32_t ns = std::max<int32_t>(ix->nslots, 1);
  const int64_t dp = ix->dp;
  RET(S.dc.ensure((size_t)B * ns * 4));
  launch_dist_dense(ix->metric, S.q.as<float>(), dp, (int)B, ix->d_cent, dp, ix->nslots, (int)dp,
                    S.qnorm.as<float>(), S.dc.as<float>(), ns, fs);
  GraphQuery gq = {};
  // per-slot scope flags: rebuilt (and uploaded) only when the scope set or
  // the list table changed since the last traversal (agent searches repeat
  // the same scope set query after query)
  std::vector<int32_t> key(codes, codes + nscopes);
  std::sort(key.begin(), key.end());
  if (key != G.flags_codes || G.flags_ver != ix->tver || G.flags_ns != ns) {
    G.hflags.assign(ns, 0);
    for (int32_t sl = 0; sl < ix->nslots; sl++) {
      if (ix->h_cid[sl] < 0) continue;
      const int32_t c = ix->h_scope[sl];
      uint8_t f = c == G.static_code ? 2 : 0;
      for (int i = 0; i < nscopes; i++)
        if (codes[i] == c) f = 3;
      G.hflags[sl] = f;
    }
    RET(G.flags.ensure(ns));
    CK(cudaMemcpyAsync(G.flags.p, G.hflags.data(), ns, cudaMemcpyHostToDevice, fs));
    G.flags_codes = key;
    G.flags_ver = ix->tver;
    G.flags_ns = ns;
  }
  gq.flags = G.flags.as<uint8_t>();
  gq.static_entry = -1;
  auto st_it = G.entry.find(G.static_code);
  if (st_it != G.entry.end()) {
    gq.static_entry = st_it->second.first;
    gq.static_maxl = st_it->second.second;
  }
  gq.n_sc = nscopes;
  for (int i = 0; i < nscopes; i++) {
    auto it = G.entry.find(codes[i]);
    gq.sc_entry[i] = it == G.entry.end() ? -1 : it->second.first;
    gq.sc_maxl[i] = it == G.entry.end() ? 0 : it->second.second;
    gq.sc_static[i] = codes[i] == G.static_code;
  }
  gq.ef = std::max(ga.ef, nprobe);
  gq.nprobe = nprobe;
  gq.mode = ga.mode;
  GraphDev gd;
  gd.level = G.level.as<int8_t>();
  gd.nbr0 = G.nbr0.as<int32_t>();
  gd.up_off = G.up_off.as<int32_t>();
  gd.up = G.up.as<int32_t>();
  gd.por_off = G.por_off.as<int32_t>();
  gd.por = G.por.as<int32_t>();
  gd.rank = G.rank.as<int32_t>();
  gd.slot_of_rank = G.slot_of_rank.as<int32_t>();
  gd.M = G.M;
  gd.ns = ns;
  gd.npor = G.npor;
  if (graph_smem_bytes(ns, false) > 227 * 1024) {  // per-query state in global memory
    RET(G.stamps.ensure((size_t)B * ns * 4));
    RET(G.heap.ensure((size_t)B * (2 * ns + 2) * 8));
  }
  RET(G.count.ensure((size_t)B * 4));
  launch_graph_search(S.dc.as<float>(), ns, (int)B, gd, gq, G.stamps.as<uint32_t>(), G.heap.as<uint64_t>(),
                      S.probe.as<int32_t>(), G.count.as<int32_t>(), fs);
  CK(cudaGetLastError());
  if (ga.out_coarse)
    CK(cudaMemcpyAsync(ga.out_coarse, G.count.p, (size_t)B * 4,
                       ga.coarse_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, fs));
  return PK_OK;
}

// PK_DEBUG_SUBMIT=2: host microseconds per search_core phase (accumulated;
// printed by pk_search_submit): setup, front launches, scan, re-rank, tail
static double g_hphase[6];
static long g_hcalls;
static bool g_hdbg = getenv("PK_DEBUG_SUBMIT") && atoi(getenv("PK_DEBUG_SUBMIT")) >= 2;

static int search_core(pk_index* ix, const float* Q, int64_t B, const int32_t* scope_codes,
                       int32_t nscopes, int32_t nprobe, int32_t kk, int64_t* out_ids,
                       float* out_dists, int64_t* out_cids, int32_t* out_n, int64_t* out_probe,
                       int64_t* out_scanned, bool in_dev, bool dev, const int32_t* probe_in,
                       int32_t* probe_out, bool host_scopes = false, const GraphArgs* ga = nullptr) {
  if (B < 0) return fail(PK_ERR_USAGE, "negative batch");
  if (nprobe < 1) return fail(PK_ERR_USAGE, "nprobe must be >= 1");
  // the fused pick and the scan stages take up to 2048 probes; the graph
  // traversal's coarse-only output (pk_graph_probe) has no such limit
  if (nprobe > 2048 && !(ga && probe_out))
    return fail(PK_ERR_USAGE, "nprobe %d above the device limit 2048", nprobe);
  if (kk < 1 || kk > KKMAX) return fail(PK_ERR_USAGE, "kk must lie in [1, %d]", KKMAX);
  if (!probe_in && (nscopes < 1 || nscopes > 64))
    return fail(PK_ERR_USAGE, "scope count must lie in [1, 64]");
  if (B == 0) return PK_OK;
  CK(cudaSetDevice(ix->device));
  auto hp_t = std::chrono::steady_clock::now();
  auto hmark = [&](int k) {
    if (!g_hdbg) return;
    const auto t = std::chrono::steady_clock::now();
    g_hphase[k] += std::chrono::duration<double, std::micro>(t - hp_t).count();
    hp_t = t;
  };
  if (g_hdbg) g_hcalls++;
  cudaStream_t st = ix->st;
  pk_index::Scratch& S = ix->scr[ix->par];
  const int setno = ix->par;
  ix->last_par = ix->par;
  ix->par = (ix->par + 1) % 3;
  if (ix->tiered) {
    RET(ix->release_staged());
    RET(ix->poll_migrations());
  }
  const bool table_dirty = ix->dirty_hi >= ix->dirty_lo;
  RET(ix->sync_table());
  const int64_t dp = ix->dp;
  const int32_t ns = std::max<int32_t>(ix->nslots, 1);
  // Front-half overlap (device outputs, tensor-core path): this batch's prep,
  // coarse, pick and routing go to the front stream, which waits only for
  // the point just before the previous search's scan -- so they run while
  // that scan and its re-rank drain.  Safe because the front writes only
  // this batch's scratch set (the other parity's), and nothing but searches
  // touched the index since (lock count; table unchanged).
  const bool pipelined = ix->pipeline && dev && in_dev && !probe_in && !probe_out && !ix->tiered && !ga &&
                         !ix->prof && ix->screen && ix->tensor && ix->coarse_tc && !table_dirty &&
                         ix->ev_scan && ix->mu.n == ix->ev_scan_n + 1;
  cudaStream_t fs = st;
  if (pipelined) {
    if (!ix->fst) {
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      CK(cudaStreamCreateWithPriority(&ix->fst, cudaStreamNonBlocking, ix->rr_defer ? hi : lo));
    }
    fs = ix->fst;
    CK(cudaStreamWaitEvent(fs, ix->ev_scan, 0));
    if (ix->ev_free[setno]) CK(cudaStreamWaitEvent(fs, ix->ev_free[setno], 0));
    if (ix->front_wait) CK(cudaStreamWaitEvent(fs, ix->front_wait, 0));
  }
  ix->front_wait = nullptr;
  const int tli = (pipelined && ix->tl.on && !ix->tl.printed && ix->tl.n < 48) ? ix->tl.n++ : -1;
  auto tlrec = [&](int k, cudaStream_t s2) {
    if (tli < 0) return;
    if (ix->tl.ev.empty()) {
      ix->tl.ev.resize(48 * 6);
      for (auto& e : ix->tl.ev) cudaEventCreate(&e);
    }
    cudaEventRecord(ix->tl.ev[tli * 6 + k], s2);
  };
  tlrec(0, fs);
  // scratch
  const bool fresh_q = S.q.bytes < (size_t)B * dp * 4;
  RET(S.q.ensure((size_t)B * dp * 4));
  if (fresh_q) CK(cudaMemsetAsync(S.q.p, 0, S.q.bytes, fs));  // zero pad columns once
  RET(S.qnorm.ensure(B * 4));
  RET(S.dc.ensure((size_t)B * ns * 4));
  RET(S.probe.ensure((size_t)B * nprobe * 4));
  RET(S.probe_key.ensure((size_t)B * nprobe * 4));
  RET(S.counts.ensure((size_t)ns * 4));
  const int64_t maxlen = ix->max_list_len();
  const int64_t max_nch = std::max<int64_t>(1, (maxlen + ix->chunk_rows - 1) / ix->chunk_rows);
  const int64_t max_items = B * nprobe * max_nch;
  RET(S.items.ensure((size_t)max_items * sizeof(ScanItem)));
  const int64_t smax = nprobe * max_nch;  // output slots per query
  // per-list query buckets (B entries each) + lcount [ns] | n_items | work counter
  RET(S.qpairs.ensure((size_t)ns * B * sizeof(QPair)));
  RET(S.counts.ensure((size_t)(ns + 4) * 4));
  RET(S.slot_off.ensure((size_t)2 * B * 4));
  RET(S.scanned.ensure((size_t)B * 8));
  RET(S.cand_key.ensure((size_t)max_items * kk * 4));
  RET(S.cand_id.ensure((size_t)max_items * kk * 8));
  RET(S.cand_n.ensure((size_t)max_items * 4));
  RET(S.cand_list.ensure((size_t)max_items * 4));
  RET(S.scopes.ensure(64 * 4));
  const int pc = ix->prof_calls;
#define PROF(stage) \
  if (ix->prof) RET(ix->prof_mark(pc, stage))
  // [ns] | front items | work counter | tail items | tail base (route_items)
  int32_t* lcount = S.counts.as<int32_t>();
  int32_t* n_items = lcount + ns;
  int32_t* work_ctr = lcount + ns + 1;
  const bool use_tc = ix->coarse_tc && !probe_in && !ga;
  // one fused prep kernel (padded copy, norms, TF32 split, swizzled copies,
  // counter resets) on the screened paths; plain copies otherwise
  const bool prep = ix->screen || use_tc;
  const bool tc_scan = ix->screen && ix->tensor && !probe_out;
  // candidates per query grow with kk (the screen keeps every row whose lower
  // bound is under the kk-th upper bound): 4096 covers kk 10 with room, kk 64
  // needed ~5x that on unit-sphere data, and an overflow takes the exact path
  // (bounded to 1 GB of pool per scratch set)
  const int pool_cap =
      ix->pool_cap_set ? ix->pool_cap
                       : std::max<int>(ix->pool_cap,
                                       (int)std::min<int64_t>({(int64_t)kk * 512, 1 << 16,
                                                               ((int64_t)1 << 30) / (std::max<int64_t>(B, 1) * 16)}));
  RouteArgs ra;  // set when the coarse pick emits the routes itself
  hmark(0);
  PROF(0);
  if (!probe_in) {
    const bool dev_codes = in_dev && !host_scopes;
    if (dev_codes || S.nscopes_h != nscopes || memcmp(S.scopes_h, scope_codes, (size_t)nscopes * 4) != 0) {
      CK(cudaMemcpyAsync(S.scopes.p, scope_codes, nscopes * 4,
                         dev_codes ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, fs));
      S.nscopes_h = dev_codes ? -1 : nscopes;
      if (!dev_codes) memcpy(S.scopes_h, scope_codes, (size_t)nscopes * 4);
    }
  }
  const ListTable lt = ix->table();
  if (prep) {
    const float* qin = Q;
    if (!in_dev) {  // host rows: one contiguous H2D, the prep kernel pads them
      RET(S.qin.ensure((size_t)B * ix->d * 4));
      CK(cudaMemcpyAsync(S.qin.p, Q, (size_t)B * ix->d * 4, cudaMemcpyHostToDevice, fs));
      qin = S.qin.as<float>();
    }
    RET(S.qnorm2.ensure(B * 4));
    const bool sp = use_tc && ix->coarse_split;
    if (sp) {
      RET(S.qhi.ensure((size_t)B * dp * 4));
      RET(S.qlo.ensure((size_t)B * dp * 4));
    }
    if (tc_scan && !ix->qgather) RET(S.qsw.ensure((size_t)8 * B * dp * 4));
    if (ix->screen) {
      RET(S.uq.ensure((size_t)B * 4));
      RET(S.ccount.ensure((size_t)B * 4));
    }
    launch_qprep(qin, ix->d, (int)ix->d, (int)B, (int)dp, S.q.as<float>(), S.qnorm2.as<float>(),
                 sp ? S.qhi.as<float>() : nullptr, sp ? S.qlo.as<float>() : nullptr,
                 (tc_scan && !ix->qgather) ? S.qsw.as<float>() : nullptr, lcount, (int)(ns + 3),
                 ix->screen ? S.ccount.as<int32_t>() : nullptr, ix->screen ? (int)B : 0,
                 ix->screen ? S.uq.as<uint32_t>() : nullptr, ix->screen ? (int)B : 0, fs);
  } else {
    CK(cudaMemcpy2DAsync(S.q.p, dp * 4, Q, ix->d * 4, ix->d * 4, B,
                         in_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, fs));
    CK(cudaMemsetAsync(lcount, 0, (size_t)(ns + 3) * 4, fs));
  }
  if (ix->metric == COSINE) launch_qnorm(S.q.as<float>(), dp, (int)B, (int)ix->d, S.qnorm.as<float>(), fs);
  PROF(1);
  // 1. coarse quantizer: distances to every list centroid, top-nprobe in scope
  if (probe_in) {
    CK(cudaMemcpyAsync(S.probe.p, probe_in, (size_t)B * nprobe * 4,
                       in_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, fs));
    PROF(2);
  } else if (ga) {
    RET(graph_coarse(ix, S, B, scope_codes, nscopes, nprobe, *ga, fs));
    PROF(2);
  } else if (ix->coarse_tc) {
    RET(S.ncand.ensure(B * 4));
    const int ks = coarse_split_k(ix->nslots, (int)B, (int)dp, ix->num_sms);
    RET(S.dc.ensure((size_t)ks * B * ns * 4));
    // tensor maps of this scratch set's query tables, re-encoded only when the
    // buffers or the batch size change (a driver call each otherwise)
    const void* qp0 = ix->coarse_split ? S.qhi.p : S.q.p;
    const void* qp1 = ix->coarse_split ? S.qlo.p : nullptr;
    if (S.qmap_ptr[0] != qp0 || S.qmap_ptr[1] != qp1 || S.qmap_rows != B) {
      RET(ix->encode_2d(&S.qmap[0], static_cast<const float*>(qp0), dp, B, 64));
      if (qp1) RET(ix->encode_2d(&S.qmap[1], static_cast<const float*>(qp1), dp, B, 64));
      S.qmap_ptr[0] = qp0;
      S.qmap_ptr[1] = qp1;
      S.qmap_rows = B;
    }
    ix->cmaps.q[0] = S.qmap[0];
    if (qp1) ix->cmaps.q[1] = S.qmap[1];
    launch_coarse_tc(ix->coarse_split, ks, ix->cmaps, ix->nslots, (int)B, (int)dp,
                     S.dc.as<float>(), ns, fs);
    PROF(2);
    // the pick also routes its query unless the cold tier may still move lists
    if (!probe_out && !ix->tiered) {
      ra.lcount = lcount;
      ra.bucket = S.qpairs.as<QPair>();
      ra.slot_off = S.slot_off.as<int32_t>();
      ra.scanned = S.scanned.as<int64_t>();
      ra.chunk_rows = ix->chunk_rows;
      ra.smax = (int)smax;
      ra.bcap = (int)B;
      ra.unordered = out_probe == nullptr;  // nobody reads the probe order / keys
    }
    launch_coarse_pick(ix->metric, ix->coarse_split, ks, S.dc.as<float>(), ns, (int)B, lt, ix->d_cnrm, S.q.as<float>(),
                       S.qnorm2.as<float>(), S.scopes.as<int32_t>(), nscopes, nprobe,
                       S.probe.as<int32_t>(), S.probe_key.as<uint32_t>(), S.ncand.as<int32_t>(), ra, fs);
  } else {
    launch_dist_dense(ix->metric, S.q.as<float>(), dp, (int)B, ix->d_cent, dp, ix->nslots, (int)dp,
                      S.qnorm.as<float>(), S.dc.as<float>(), ns, fs);
    PROF(2);
    launch_coarse_select(S.dc.as<float>(), ns, (int)B, lt, S.scopes.as<int32_t>(), nscopes,
                         nprobe, S.probe.as<int32_t>(), S.probe_key.as<uint32_t>(), fs);
  }
  PROF(3);
  if (probe_out) {
    CK(cudaMemcpyAsync(probe_out, S.probe.p, (size_t)B * nprobe * 4,
                       dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, fs));
    if (!dev) CK(cudaStreamSynchronize(st));
    return PK_OK;
  }
  // cold tier: stream the probed lists that are not HBM-resident into staging
  if (ix->tiered) RET(ix->stage_cold(B, nprobe, S.probe.as<int32_t>()));
  const ListTable lt2 = ix->table();  // staging may have grown the arena
  // 2. route (query -> lists) into (list -> queries) work items
  launch_route(S.probe.as<int32_t>(), (int)B, nprobe, lt2, ix->chunk_rows, (int)smax, (int)B,
               lcount, S.items.as<ScanItem>(), n_items, S.qpairs.as<QPair>(),
               S.slot_off.as<int32_t>(), S.scanned.as<int64_t>(), ra.lcount != nullptr,
               (int)std::min<int64_t>(max_items, INT32_MAX), fs);
  if (!ix->ev_front) {
    CK(cudaEventCreateWithFlags(&ix->ev_front, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ix->ev_scan, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ix->ev_sdone, cudaEventDisableTiming));
    CK(cudaEventRecord(ix->ev_sdone, st));
  }
  // Pipelined: the scan goes to the scan stream behind this front half and
  // the previous scan -- NOT behind the previous batch's re-rank, which runs
  // on the index stream beside it (lean, co-resident CTAs)
  cudaStream_t ss = st;
  tlrec(1, fs);
  hmark(1);
  if (pipelined) {
    if (!ix->sst) {
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      CK(cudaStreamCreateWithPriority(&ix->sst, cudaStreamNonBlocking, ix->rr_defer ? hi : lo));
      CK(cudaStreamCreateWithPriority(&ix->sst2, cudaStreamNonBlocking, ix->rr_defer ? hi : lo));
    }
    ss = ix->sst;
    if (ix->scan_ovl) {
      ss = ix->sturn ? ix->sst2 : ix->sst;
      ix->sturn ^= 1;
    }
    CK(cudaEventRecord(ix->ev_front, fs));
    CK(cudaStreamWaitEvent(ss, ix->ev_front, 0));
    if (!ix->scan_ovl) CK(cudaStreamWaitEvent(ss, ix->ev_sdone, 0));
  }
  // the index stream up to here: where the next search's front may start.
  // Deferred re-ranks: a pipelined search leaves the point of the last
  // non-pipelined one (nothing but searches touched the index since; the
  // scratch sets are guarded by ev_free), so the next front does not wait
  // for this batch's predecessor's re-rank
  if (!(pipelined && ix->rr_defer)) CK(cudaEventRecord(ix->ev_scan, st));
  ix->ev_scan_n = ix->mu.n;
  // 3. fused scan + per-(query, list chunk) top-kk
  tlrec(2, ss);
  PROF(4);
  if (ix->screen) {
    RET(S.cpool.ensure((size_t)B * pool_cap * sizeof(int4)));  // uq / ccount reset by prep
    if (ix->tensor) {
      // gather4 map over this scratch set's padded queries (box 32 x 1 row)
      const CUtensorMap* qg = nullptr;
      if (ix->qgather) {
        if (S.qg_ptr != S.q.p || S.qg_rows != B) {
          RET(ix->encode_2d(&S.qgmap, S.q.as<float>(), dp, B, 1));
          S.qg_ptr = S.q.p;
          S.qg_rows = B;
        }
        qg = &S.qgmap;
      }
      launch_scan_tc(ix->metric, lt2, ix->maps, S.q.as<float>(), (int)B, S.qsw.as<float>(), true,
                     S.qnorm2.as<float>(), S.items.as<ScanItem>(), n_items,
                     (int)std::min<int64_t>(max_items, INT32_MAX), S.qpairs.as<QPair>(), kk,
                     work_ctr, S.uq.as<uint32_t>(), S.cand_key.as<uint32_t>(),
                     S.cand_n.as<int32_t>(), S.cpool.as<int4>(), S.ccount.as<int32_t>(),
                     pool_cap, ix->scan_sms, ss, /*pdl=*/!pipelined, qg,
                     /*overlapped: release some SMs early for the next front half*/ pipelined);
    } else {
      launch_scan_screen(ix->metric, lt2, ix->maps, S.q.as<float>(), S.qnorm2.as<float>(),
                         S.items.as<ScanItem>(), n_items,
                         (int)std::min<int64_t>(max_items, INT32_MAX), S.qpairs.as<QPair>(), kk,
                         work_ctr, S.uq.as<uint32_t>(), S.cand_key.as<uint32_t>(),
                         S.cand_n.as<int32_t>(), S.cpool.as<int4>(), S.ccount.as<int32_t>(),
                         pool_cap, ix->num_sms, st);
    }
  } else
    launch_scan(ix->metric, lt2, ix->maps, S.q.as<float>(), S.qnorm.as<float>(),
                S.items.as<ScanItem>(), n_items, (int)std::min<int64_t>(max_items, INT32_MAX),
                S.qpairs.as<QPair>(), kk, work_ctr, S.cand_key.as<uint32_t>(),
                S.cand_id.as<int64_t>(), S.cand_n.as<int32_t>(), S.cand_list.as<int32_t>(),
                ix->num_sms, st);
  tlrec(3, ss);
  CK(cudaEventRecord(ix->ev_sdone, ss));
  if (pipelined) CK(cudaStreamWaitEvent(st, ix->ev_sdone, 0));
  tlrec(4, st);
  hmark(2);
  PROF(5);
  // 4. merge per query
  int64_t* o_ids = out_ids;
  float* o_d = out_dists;
  int64_t* o_cid = out_cids;
  int32_t* o_n = out_n;
  const int64_t ob = pk_shard_block_bytes(B, kk);  // host path: one packed result block
  if (!dev) {
    // results land in one device block (shard-block layout) and come back in
    // ONE copy into a pinned staging buffer, then fan out on the host
    RET(S.out_ids.ensure((size_t)ob));
    uint8_t* base = S.out_ids.as<uint8_t>();
    const int64_t nkk = B * kk;
    o_ids = reinterpret_cast<int64_t*>(base);
    o_cid = reinterpret_cast<int64_t*>(base + 8 * nkk);
    o_d = reinterpret_cast<float*>(base + 16 * nkk + 8 * B);
    o_n = reinterpret_cast<int32_t*>(base + 20 * nkk + 8 * B);
  }
  if (ix->screen) RET(S.nsurv.ensure((size_t)B * 4));
  // the re-rank also copies the per-query scanned counts out (no extra copy op)
  int64_t* sc_dst = !dev ? reinterpret_cast<int64_t*>(S.out_ids.as<uint8_t>() + 16 * B * kk) : out_scanned;
  if (ix->screen)
    launch_rerank_merge(ix->metric, (int)B, S.cpool.as<int4>(), S.ccount.as<int32_t>(),
                        pool_cap, S.cand_key.as<uint32_t>(), S.cand_n.as<int32_t>(),
                        S.slot_off.as<int32_t>(), lt2, S.q.as<float>(), S.probe.as<int32_t>(),
                        nprobe, kk, o_ids, o_d, o_cid, o_n, S.nsurv.as<int32_t>(),
                        S.scanned.as<int64_t>(), sc_dst, st,
                        // overlapped: launched after the scan, so its CTAs do not sit
                        // waiting on the SMs the scan tail frees for the next front half
                        /*pdl=*/!pipelined,
                        // pipelined: lean CTAs beside the next batch's scan (at most one per SM)
                        (pipelined && ix->tensor && (ix->rr_lean > 0 || (ix->rr_lean < 0 && B <= 64)) &&
                         rerank_lean_fits((int)dp)) ? ix->rr_lean_ctas : 0);
  else
    launch_merge((int)B, S.slot_off.as<int32_t>(), S.cand_key.as<uint32_t>(),
                 S.cand_id.as<int64_t>(), S.cand_n.as<int32_t>(), S.cand_list.as<int32_t>(), kk,
                 lt2, o_ids, o_d, o_cid, o_n, st);
  tlrec(5, st);
  hmark(3);
  if (tli == 47) {  // print the timeline of searches 8..47 relative to the first scan's end
    cudaDeviceSynchronize();
    ix->tl.printed = true;
    auto at = [&](int i, int k) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ix->tl.ev[8 * 6 + 3], ix->tl.ev[i * 6 + k]);
      return 1e3 * ms;
    };
    fprintf(stderr, "timeline (us from search 8's scan end): search: front[begin end] scan[begin end] rerank[begin end]\n");
    for (int i = 9; i < 48; i++)
      fprintf(stderr, "  %2d: front[%8.1f %8.1f] scan[%8.1f %8.1f] rerank[%8.1f %8.1f]\n", i, at(i, 0), at(i, 1),
              at(i, 2), at(i, 3), at(i, 4), at(i, 5));
  }
  // this scratch set is free again once the re-rank has read it
  if (!ix->ev_free[setno]) CK(cudaEventCreateWithFlags(&ix->ev_free[setno], cudaEventDisableTiming));
  CK(cudaEventRecord(ix->ev_free[setno], st));
  CK(cudaGetLastError());
  if (!dev) {
    const int64_t nkk = B * kk;
    uint8_t* base = S.out_ids.as<uint8_t>();
    if (!ix->screen)
      CK(cudaMemcpyAsync(base + 16 * nkk, S.scanned.p, (size_t)B * 8, cudaMemcpyDeviceToDevice, st));
    if ((int64_t)ix->hout_bytes < ob) {
      if (ix->hout) cudaFreeHost(ix->hout);
      ix->hout = nullptr;
      ix->hout_bytes = 0;
      CK(cudaHostAlloc((void**)&ix->hout, (size_t)ob, cudaHostAllocDefault));
      ix->hout_bytes = (size_t)ob;
    }
    CK(cudaMemcpyAsync(ix->hout, base, (size_t)ob, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const uint8_t* h = ix->hout;
    memcpy(out_ids, h, nkk * 8);
    if (out_cids) memcpy(out_cids, h + 8 * nkk, nkk * 8);
    if (out_scanned) memcpy(out_scanned, h + 16 * nkk, B * 8);
    memcpy(out_dists, h + 16 * nkk + 8 * B, nkk * 4);
    memcpy(out_n, h + 20 * nkk + 8 * B, B * 4);
  } else if (out_scanned && !ix->screen) {
    CK(cudaMemcpyAsync(out_scanned, S.scanned.p, (size_t)B * 8, cudaMemcpyDeviceToDevice, st));
  }
  PROF(6);
  if (ix->prof) ix->prof_calls++;
#undef PROF
  if (out_probe) {
    // probe slots -> cids (host mirror); forces a sync
    std::vector<int32_t> ps((size_t)B * nprobe);
    CK(cudaMemcpyAsync(ps.data(), S.probe.p, ps.size() * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::vector<int64_t> pc(ps.size());
    for (size_t i = 0; i < ps.size(); i++) pc[i] = ps[i] >= 0 ? ix->h_cid[ps[i]] : -1;
    CK(cudaMemcpyAsync(out_probe, pc.data(), pc.size() * 8,
                       dev ? cudaMemcpyHostToDevice : cudaMemcpyHostToHost, st));
  }
  if (!dev || out_probe) CK(cudaStreamSynchronize(st));
  return PK_OK;
}

extern "C" {

int pk_search(pk_index* ix, const float* Q, int64_t B, const int32_t* scope_codes,
              int32_t nscopes, int32_t nprobe, int32_t kk, int64_t* out_ids, float* out_dists,
              int64_t* out_cids, int32_t* out_n, int64_t* out_probe, int64_t* out_scanned,
              int flags) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  const bool dev = flags & PK_DEVICE_PTRS;
  return search_core(ix, Q, B, scope_codes, nscopes, nprobe, kk, out_ids, out_dists, out_cids,
                     out_n, out_probe, out_scanned, dev, dev, nullptr, nullptr);
}

static int search_submit_impl(pk_index* ix, int32_t slot, const float* Q, int64_t B,
                              const int32_t* scope_codes, int32_t nscopes, int32_t nprobe, int32_t kk);

int pk_search_submit(pk_index* ix, int32_t slot, const float* Q, int64_t B,
                     const int32_t* scope_codes, int32_t nscopes, int32_t nprobe, int32_t kk) {
  // PK_DEBUG_SUBMIT=1: host microseconds inside this call, printed every 2000
  static const bool dbg = getenv("PK_DEBUG_SUBMIT") != nullptr;
  if (!dbg) return search_submit_impl(ix, slot, Q, B, scope_codes, nscopes, nprobe, kk);
  static double acc = 0;
  static long calls = 0;
  const auto t0 = std::chrono::steady_clock::now();
  const int rc = search_submit_impl(ix, slot, Q, B, scope_codes, nscopes, nprobe, kk);
  acc += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
  if (++calls % 2000 == 0) {
    fprintf(stderr, "pk_search_submit host us/call: %.1f\n", acc / calls);
    if (g_hcalls)
      fprintf(stderr, "  search_core us/call: setup %.1f front %.1f scan %.1f rerank %.1f\n",
              g_hphase[0] / g_hcalls, g_hphase[1] / g_hcalls, g_hphase[2] / g_hcalls, g_hphase[3] / g_hcalls);
  }
  return rc;
}

static int search_submit_impl(pk_index* ix, int32_t slot, const float* Q, int64_t B,
                              const int32_t* scope_codes, int32_t nscopes, int32_t nprobe, int32_t kk) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  if (slot < 0 || slot >= PK_ASYNC_SLOTS) return fail(PK_ERR_USAGE, "slot must lie in [0, %d)", PK_ASYNC_SLOTS);
  if (kk < 1 || kk > KKMAX) return fail(PK_ERR_USAGE, "kk must lie in [1, %d]", KKMAX);
  auto& a = ix->aslot[slot];
  if (a.busy) return fail(PK_ERR_USAGE, "slot %d has an uncollected search", slot);
  if (B <= 0) return fail(PK_ERR_USAGE, "empty batch");
  CK(cudaSetDevice(ix->device));
  if (!ix->cst) CK(cudaStreamCreateWithFlags(&ix->cst, cudaStreamNonBlocking));
  if (!ix->rst) CK(cudaStreamCreateWithFlags(&ix->rst, cudaStreamNonBlocking));
  if (!a.copied) {
    CK(cudaEventCreateWithFlags(&a.copied, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&a.done, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&a.consumed, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&a.ready, cudaEventDisableTiming));
    CK(cudaEventRecord(a.consumed, ix->st));
  }
  const int64_t ob = pk_shard_block_bytes(B, kk);
  RET(a.qin.ensure((size_t)B * ix->d * 4));
  RET(a.blk.ensure((size_t)ob));
  if ((int64_t)a.hbytes < ob) {
    if (a.hblk) cudaFreeHost(a.hblk);
    a.hblk = nullptr;
    a.hbytes = 0;
    CK(cudaHostAlloc((void**)&a.hblk, (size_t)ob, cudaHostAllocDefault));
    a.hbytes = (size_t)ob;
  }
  // H2D on the copy stream once the slot's previous batch has read its input
  CK(cudaStreamWaitEvent(ix->cst, a.consumed, 0));
  CK(cudaMemcpyAsync(a.qin.p, Q, (size_t)B * ix->d * 4, cudaMemcpyHostToDevice, ix->cst));
  CK(cudaEventRecord(a.copied, ix->cst));
  CK(cudaStreamWaitEvent(ix->st, a.copied, 0));
  ix->front_wait = a.copied;  // an overlapped front half waits for the copy itself
  uint8_t* base = a.blk.as<uint8_t>();
  const int64_t nkk = B * kk;
  RET(search_core(ix, a.qin.as<float>(), B, scope_codes, nscopes, nprobe, kk,
                  reinterpret_cast<int64_t*>(base), reinterpret_cast<float*>(base + 16 * nkk + 8 * B),
                  reinterpret_cast<int64_t*>(base + 8 * nkk), reinterpret_cast<int32_t*>(base + 20 * nkk + 8 * B),
                  nullptr, reinterpret_cast<int64_t*>(base + 16 * nkk), true, true, nullptr, nullptr,
                  /*host_scopes=*/true));
  CK(cudaEventRecord(a.consumed, ix->st));
  // read-back on its own stream: the next batch's scan on the index stream
  // does not queue behind this copy
  CK(cudaEventRecord(a.ready, ix->st));
  CK(cudaStreamWaitEvent(ix->rst, a.ready, 0));
  CK(cudaMemcpyAsync(a.hblk, base, (size_t)ob, cudaMemcpyDeviceToHost, ix->rst));
  CK(cudaEventRecord(a.done, ix->rst));
  a.B = B;
  a.kk = kk;
  a.busy = true;
  return PK_OK;
}

int pk_search_collect(pk_index* ix, int32_t slot, int64_t* out_ids, float* out_dists, int64_t* out_cids,
                      int32_t* out_n, int64_t* out_scanned) {
  if (slot < 0 || slot >= PK_ASYNC_SLOTS) return fail(PK_ERR_USAGE, "slot must lie in [0, %d)", PK_ASYNC_SLOTS);
  auto& a = ix->aslot[slot];
  if (!a.busy) return fail(PK_ERR_USAGE, "slot %d has no search in flight", slot);
  CK(cudaEventSynchronize(a.done));  // outside the index lock: the other slot may submit meanwhile
  // uncounted: collecting queues nothing, so the next submit may still overlap
  std::lock_guard<std::recursive_mutex> lock_(ix->mu.m);
  const int64_t B = a.B, nkk = B * a.kk;
  const uint8_t* h = a.hblk;
  memcpy(out_ids, h, nkk * 8);
  if (out_cids) memcpy(out_cids, h + 8 * nkk, nkk * 8);
  if (out_scanned) memcpy(out_scanned, h + 16 * nkk, B * 8);
  memcpy(out_dists, h + 16 * nkk + 8 * B, nkk * 4);
  memcpy(out_n, h + 20 * nkk + 8 * B, B * 4);
  a.busy = false;
  return PK_OK;
}

int pk_search_coarse(pk_index* ix, const float* Q, int64_t B, const int32_t* scope_codes,
                     int32_t nscopes, int32_t nprobe, int32_t* out_probe, int flags) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  if (!out_probe) return fail(PK_ERR_USAGE, "out_probe is required");
  const bool dev = flags & PK_DEVICE_PTRS;
  return search_core(ix, Q, B, scope_codes, nscopes, nprobe, 1, nullptr, nullptr, nullptr, nullptr,
                     nullptr, nullptr, dev, dev, nullptr, out_probe);
}

int pk_search_probed(pk_index* ix, const float* Q, int64_t B, const int32_t* probe, int32_t nprobe,
                     int32_t kk, int64_t group, void* out_blocks, int flags) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  if (!probe || !out_blocks) return fail(PK_ERR_USAGE, "probe and out_blocks are required");
  if (group < 1 || B % group != 0) return fail(PK_ERR_USAGE, "group must divide the batch");
  if (kk < 1 || kk > KKMAX) return fail(PK_ERR_USAGE, "kk must lie in [1, %d]", KKMAX);
  if (B == 0) return PK_OK;
  const bool dev = flags & PK_DEVICE_PTRS;
  RET(ix->pb.ensure((size_t)B * kk * 20 + B * 12 + 64));
  int64_t* o_ids = ix->pb.as<int64_t>();
  int64_t* o_cid = o_ids + B * kk;
  int64_t* o_sc = o_cid + B * kk;
  float* o_d = reinterpret_cast<float*>(o_sc + B);
  int32_t* o_n = reinterpret_cast<int32_t*>(o_d + B * kk);
  RET(search_core(ix, Q, B, nullptr, 0, nprobe, kk, o_ids, o_d, o_cid, o_n, nullptr, o_sc, dev,
                  true, probe, nullptr));
  const int64_t bb = pk_shard_block_bytes(group, kk);
  void* dst = out_blocks;
  if (!dev) {
    RET(ix->pb_out.ensure((size_t)(B / group) * bb));
    dst = ix->pb_out.p;
  }
  launch_reblock(o_ids, o_cid, o_sc, o_d, o_n, (int)B, (int)group, kk, bb, dst, ix->st);
  CK(cudaGetLastError());
  if (!dev) {
    CK(cudaMemcpyAsync(out_blocks, dst, (size_t)(B / group) * bb, cudaMemcpyDeviceToHost, ix->st));
    CK(cudaStreamSynchronize(ix->st));
  }
  return PK_OK;
}

int pk_combine_create(pk_index* ix, int32_t R, int32_t my_rank, int64_t group, int32_t kk,
                      void* ipc_handle_out) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  if (R < 1 || my_rank < 0 || my_rank >= R || group < 1 || kk < 1 || kk > KKMAX)
    return fail(PK_ERR_USAGE, "bad combine shape");
  if ((int64_t)R * kk > shard_merge_cap()) return fail(PK_ERR_USAGE, "ranks x kk above %d", shard_merge_cap());
  CK(cudaSetDevice(ix->device));
  auto& c = ix->comb;
  if (c.area) return fail(PK_ERR_USAGE, "combine area exists");
  c.R = R;
  c.my_rank = my_rank;
  c.group = group;
  c.kk = kk;
  c.bb = pk_shard_block_bytes(group, kk);
  const size_t bytes = (size_t)R * c.bb + (size_t)R * 128;
  CK(cudaMalloc((void**)&c.area, bytes));
  CK(cudaMemset(c.area, 0, bytes));  // flags start at epoch 0
  CK(cudaMalloc((void**)&c.d_peers, (size_t)R * sizeof(uint8_t*)));
  CK(cudaMalloc((void**)&c.done_ctr, 64));
  c.err = reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(c.done_ctr) + 32);
  CK(cudaMemset(c.done_ctr, 0, 64));
  c.peers.assign(R, nullptr);
  c.peers[my_rank] = c.area;
  c.peers_dirty = true;
  if (ipc_handle_out) {
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, c.area));
    memcpy(ipc_handle_out, &h, sizeof(h));
  }
  return PK_OK;
}

int pk_combine_open(pk_index* ix, int32_t peer, const void* ipc_handle, void* area_ptr) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  auto& c = ix->comb;
  if (!c.area) return fail(PK_ERR_USAGE, "pk_combine_create first");
  if (peer < 0 || peer >= c.R) return fail(PK_ERR_USAGE, "bad peer %d", peer);
  if (peer == c.my_rank) return PK_OK;
  CK(cudaSetDevice(ix->device));
  if (area_ptr) {  // same process (simulated ranks)
    c.peers[peer] = static_cast<uint8_t*>(area_ptr);
  } else {
    cudaIpcMemHandle_t h;
    memcpy(&h, ipc_handle, sizeof(h));
    void* p = nullptr;
    CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    c.peers[peer] = static_cast<uint8_t*>(p);
    c.opened.push_back(static_cast<uint8_t*>(p));
  }
  c.peers_dirty = true;
  return PK_OK;
}

void* pk_combine_area(pk_index* ix) { return ix ? ix->comb.area : nullptr; }

int pk_combine_search_probed(pk_index* ix, const float* Q, int64_t B, const int32_t* probe,
                             int32_t nprobe, int64_t epoch, int flags) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  auto& c = ix->comb;
  if (!c.area) return fail(PK_ERR_USAGE, "pk_combine_create first");
  if (!(flags & PK_DEVICE_PTRS)) return fail(PK_ERR_USAGE, "peer combine takes device pointers");
  if (B != (int64_t)c.R * c.group) return fail(PK_ERR_USAGE, "batch must be ranks x group");
  for (uint8_t* p : c.peers)
    if (!p) return fail(PK_ERR_USAGE, "a peer area is not open");
  const int kk = c.kk;
  RET(ix->pb.ensure((size_t)B * kk * 20 + B * 12 + 64));
  int64_t* o_ids = ix->pb.as<int64_t>();
  int64_t* o_cid = o_ids + B * kk;
  int64_t* o_sc = o_cid + B * kk;
  float* o_d = reinterpret_cast<float*>(o_sc + B);
  int32_t* o_n = reinterpret_cast<int32_t*>(o_d + B * kk);
  RET(search_core(ix, Q, B, nullptr, 0, nprobe, kk, o_ids, o_d, o_cid, o_n, nullptr, o_sc, true,
                  true, probe, nullptr));
  if (c.peers_dirty) {
    CK(cudaMemcpyAsync(c.d_peers, c.peers.data(), (size_t)c.R * sizeof(uint8_t*), cudaMemcpyHostToDevice,
                       ix->st));
    c.peers_dirty = false;
  }
  CK(cudaMemsetAsync(c.done_ctr, 0, 4, ix->st));
  launch_peer_send(o_ids, o_cid, o_sc, o_d, o_n, (int)B, (int)c.group, kk, c.bb, c.d_peers, c.R,
                   c.my_rank, (uint64_t)epoch, c.done_ctr, ix->st);
  CK(cudaGetLastError());
  return PK_OK;
}

int pk_combine_merge(pk_index* ix, int64_t epoch, double timeout_s, int64_t* out_ids, float* out_dists,
                     int64_t* out_cids, int32_t* out_n, int64_t* out_scanned, int flags) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  auto& c = ix->comb;
  if (!c.area) return fail(PK_ERR_USAGE, "pk_combine_create first");
  if (!(flags & PK_DEVICE_PTRS)) return fail(PK_ERR_USAGE, "peer combine takes device pointers");
  CK(cudaSetDevice(ix->device));
  launch_peer_merge(ix->metric, c.area, c.bb, c.R, (int)c.group, c.kk, (uint64_t)epoch, (int64_t)(timeout_s * 1e9),
                    c.err, out_ids, out_dists, out_cids, out_n, out_scanned, ix->st);
  CK(cudaGetLastError());
  return PK_OK;
}

int pk_combine_status(pk_index* ix, int32_t* err) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  if (!ix->comb.area) return fail(PK_ERR_USAGE, "pk_combine_create first");
  CK(cudaMemcpyAsync(err, ix->comb.err, 4, cudaMemcpyDeviceToHost, ix->st));
  CK(cudaStreamSynchronize(ix->st));
  return PK_OK;
}

int pk_search_coarse_cids(pk_index* ix, const float* Q, int64_t B, const int32_t* scope_codes,
                          int32_t nscopes, int32_t nprobe, int64_t* out_cids) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  if (!out_cids) return fail(PK_ERR_USAGE, "out_cids is required");
  std::vector<int32_t> pr((size_t)std::max<int64_t>(B, 0) * std::max(nprobe, 1));
  RET(search_core(ix, Q, B, scope_codes, nscopes, nprobe, 1, nullptr, nullptr, nullptr, nullptr,
                  nullptr, nullptr, false, false, nullptr, pr.data()));
  for (size_t i = 0; i < (size_t)B * nprobe; i++) out_cids[i] = pr[i] >= 0 ? ix->h_cid[pr[i]] : -1;
  return PK_OK;
}

int pk_graph_set(pk_index* ix, int32_t M, int64_t n, const int64_t* node_cid, const int32_t* node_level,
                 const int64_t* nbr, const int64_t* por_ptr, const int64_t* por, int32_t static_code,
                 int32_t nsc, const int32_t* sc_code, const int64_t* sc_entry, const int32_t* sc_maxl) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  if (M < 1 || n < 0 || nsc < 0) return fail(PK_ERR_USAGE, "bad graph shape");
  CK(cudaSetDevice(ix->device));
  pk_index::Graph& G = ix->graph;
  const int32_t ns = std::max<int32_t>(ix->nslots, 1);
  auto slot = [&](int64_t c, int32_t* out) -> int { return ix->slot_of(c, out); };
  std::vector<int8_t> level(ns, -1);
  std::vector<int32_t> nbr0((size_t)ns * M, -1), up_off(ns, 0), up, por_off(ns + 1, 0), porv;
  std::vector<std::vector<int32_t>> por_of(ns);
  // rank: position of each live slot's cid among the live cids (heap tie order)
  std::vector<std::pair<int64_t, int32_t>> live;
  for (int32_t sl = 0; sl < ix->nslots; sl++)
    if (ix->h_cid[sl] >= 0) live.push_back({ix->h_cid[sl], sl});
  std::sort(live.begin(), live.end());
  std::vector<int32_t> rank(ns, 0), sor(ns, 0);
  for (size_t r = 0; r < live.size(); r++) {
    rank[live[r].second] = (int32_t)r;
    sor[r] = live[r].second;
  }
  int64_t pos = 0;
  for (int64_t i = 0; i < n; i++) {
    int32_t sl;
    RET(slot(node_cid[i], &sl));
    const int32_t L = node_level[i];
    if (L < 0 || L > 126) return fail(PK_ERR_USAGE, "node level %d out of range", L);
    level[sl] = (int8_t)L;
    for (int32_t layer = 0; layer <= L; layer++) {
      for (int32_t j = 0; j < M; j++) {
        const int64_t c = nbr[pos + (int64_t)layer * M + j];
        int32_t t = -1;
        if (c >= 0) RET(slot(c, &t));
        if (layer == 0) nbr0[(size_t)sl * M + j] = t;
        else up.push_back(t);
      }
      if (layer == 0 && L > 0) up_off[sl] = (int32_t)up.size();
    }
    pos += (int64_t)(L + 1) * M;
    for (int64_t k = por_ptr[i]; k < por_ptr[i + 1]; k++) {
      int32_t t;
      RET(slot(por[k], &t));
      por_of[sl].push_back(t);
    }
  }
  for (int32_t sl = 0; sl < ns; sl++) {
    por_off[sl + 1] = por_off[sl] + (int32_t)por_of[sl].size();
    porv.insert(porv.end(), por_of[sl].begin(), por_of[sl].end());
  }
  G.entry.clear();
  for (int32_t i = 0; i < nsc; i++) {
    if (sc_entry[i] < 0) continue;
    int32_t t;
    RET(slot(sc_entry[i], &t));
    G.entry[sc_code[i]] = {t, sc_maxl[i]};
  }
  auto put = [&](DevBuf& b, const void* src, size_t bytes) -> int {
    RET(b.ensure(std::max<size_t>(bytes, 4)));
    if (bytes) CK(cudaMemcpyAsync(b.p, src, bytes, cudaMemcpyHostToDevice, ix->st));
    return PK_OK;
  };
  RET(put(G.level, level.data(), level.size()));
  RET(put(G.nbr0, nbr0.data(), nbr0.size() * 4));
  RET(put(G.up_off, up_off.data(), up_off.size() * 4));
  RET(put(G.up, up.data(), up.size() * 4));
  RET(put(G.por_off, por_off.data(), por_off.size() * 4));
  RET(put(G.por, porv.data(), porv.size() * 4));
  RET(put(G.rank, rank.data(), rank.size() * 4));
  RET(put(G.slot_of_rank, sor.data(), sor.size() * 4));
  CK(cudaStreamSynchronize(ix->st));  // pageable sources
  G.M = M;
  G.npor = (int32_t)porv.size();
  G.flags_codes.clear();  // rebuilt for the new graph at the next traversal
  G.ns = ix->nslots;
  G.slot_ver = ix->slot_ver;
  G.static_code = static_code;
  G.set = true;
  ix->tver++;  // a new graph: earlier traversals are stale (pk_list_version)
  return PK_OK;
}

int pk_search_graph(pk_index* ix, const float* Q, int64_t B, const int32_t* scope_codes,
                    int32_t nscopes, int32_t nprobe, int32_t ef, int32_t mode, int32_t kk,
                    int64_t* out_ids, float* out_dists, int64_t* out_cids, int32_t* out_n,
                    int64_t* out_probe, int64_t* out_scanned, int32_t* out_coarse, int flags) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  if (mode != 0 && mode != 1) return fail(PK_ERR_USAGE, "graph mode must be 0 (hybrid) or 1 (per-scope)");
  const bool dev = flags & PK_DEVICE_PTRS;
  GraphArgs ga;
  ga.ef = ef;
  ga.mode = mode;
  ga.out_coarse = out_coarse;
  ga.coarse_dev = dev;
  return search_core(ix, Q, B, scope_codes, nscopes, nprobe, kk, out_ids, out_dists, out_cids, out_n,
                     out_probe, out_scanned, dev, dev, nullptr, nullptr, /*host_scopes=*/true, &ga);
}

int pk_graph_probe(pk_index* ix, const float* Q, int64_t B, const int32_t* scope_codes, int32_t nscopes,
                   int32_t nprobe, int32_t ef, int32_t mode, int64_t* out_cids, int32_t* out_coarse) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  if (!out_cids) return fail(PK_ERR_USAGE, "out_cids is required");
  if (mode != 0 && mode != 1) return fail(PK_ERR_USAGE, "graph mode must be 0 (hybrid) or 1 (per-scope)");
  GraphArgs ga;
  ga.ef = ef;
  ga.mode = mode;
  ga.out_coarse = out_coarse;
  std::vector<int32_t> pr((size_t)std::max<int64_t>(B, 0) * std::max(nprobe, 1));
  RET(search_core(ix, Q, B, scope_codes, nscopes, nprobe, 1, nullptr, nullptr, nullptr, nullptr, nullptr,
                  nullptr, false, false, nullptr, pr.data(), true, &ga));
  for (size_t i = 0; i < (size_t)B * nprobe; i++) out_cids[i] = pr[i] >= 0 ? ix->h_cid[pr[i]] : -1;
  return PK_OK;
}

int pk_centroid_dists(pk_index* ix, const float* V, int64_t n, float* out, int64_t* out_cids) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  if (n < 0) return fail(PK_ERR_USAGE, "negative count");
  CK(cudaSetDevice(ix->device));
  const int32_t ns = ix->nslots;
  if (out_cids)
    for (int32_t sl = 0; sl < ns; sl++) out_cids[sl] = ix->h_cid[sl];
  if (n == 0 || ns == 0) return PK_OK;
  cudaStream_t st = ix->st;
  const int64_t dp = ix->dp;
  RET(ix->sync_table());
  const size_t in_b = (size_t)n * dp * 4, out_b = (size_t)n * ns * 4;
  RET(ix->hasg.ensure(in_b + out_b));
  float* hq = reinterpret_cast<float*>(ix->hasg.p);
  for (int64_t r = 0; r < n; r++) {
    memcpy(hq + r * dp, V + r * ix->d, ix->d * 4);
    if (dp > ix->d) memset(hq + r * dp + ix->d, 0, (dp - ix->d) * 4);
  }
  RET(ix->assign_q.ensure(in_b));
  RET(ix->assign_qn.ensure((size_t)n * 4));
  RET(ix->assign_dc.ensure(out_b));
  CK(cudaMemcpyAsync(ix->assign_q.p, hq, in_b, cudaMemcpyHostToDevice, st));
  if (ix->metric == COSINE) launch_qnorm(ix->assign_q.as<float>(), dp, (int)n, (int)ix->d, ix->assign_qn.as<float>(), st);
  launch_dist_dense(ix->metric, ix->assign_q.as<float>(), dp, (int)n, ix->d_cent, dp, ns, (int)dp,
                    ix->assign_qn.as<float>(), ix->assign_dc.as<float>(), ns, st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(ix->hasg.p + in_b, ix->assign_dc.p, out_b, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  memcpy(out, ix->hasg.p + in_b, out_b);
  return PK_OK;
}

int pk_list_slot(pk_index* ix, int64_t cid, int32_t* slot) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  return ix->slot_of(cid, slot);
}

int pk_slot_count(pk_index* ix, int32_t* n) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  *n = ix->nslots;
  return PK_OK;
}

int pk_scan_lists(pk_index* ix, const float* q, const int64_t* cids, int32_t m, int64_t* out_ids,
                  float* out_dists, int64_t* out_prefix) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  if (m < 0) return fail(PK_ERR_USAGE, "negative list count");
  out_prefix[0] = 0;
  if (m == 0) return PK_OK;
  CK(cudaSetDevice(ix->device));
  cudaStream_t st = ix->st;
  if (ix->tiered) RET(ix->poll_migrations());
  std::vector<ListSrc> src(m);
  for (int32_t l = 0; l < m; l++) {
    int32_t s;
    RET(ix->slot_of(cids[l], &s));
    out_prefix[l + 1] = out_prefix[l] + ix->h_len[s];
    if (!ix->tiered || ix->h_res[s]) {
      src[l].rows = ix->rows + ix->h_off[s] * ix->dp;
      src[l].ids = ix->ids + ix->h_off[s];
    } else {  // cold list: read in place from the mapped host arena
      src[l].rows = ix->hrows_d + ix->h_hoff[s] * ix->dp;
      src[l].ids = ix->hids_d + ix->h_hoff[s];
    }
  }
  const int64_t total = out_prefix[m];
  const int64_t dp = ix->dp;
  // inputs [q padded | list sources | prefix] packed in pinned memory, one
  // copy; the kernel writes ids and distances straight into mapped pinned
  // memory (one agent query's probed lists: a few hundred KB), so the call is
  // one copy + one kernel + one sync
  const size_t in_bytes = round_up(dp * 4, 16) + round_up(m * sizeof(ListSrc), 16) + (size_t)(m + 1) * 8;
  const size_t out_bytes = (size_t)std::max<int64_t>(total, 1) * 12;
  RET(ix->hsl.ensure(in_bytes + out_bytes));
  uint8_t* h = ix->hsl.p;
  float* h_q = reinterpret_cast<float*>(h);
  memcpy(h_q, q, ix->d * 4);
  if (dp > ix->d) memset(h_q + ix->d, 0, (dp - ix->d) * 4);
  ListSrc* h_src = reinterpret_cast<ListSrc*>(h + round_up(dp * 4, 16));
  memcpy(h_src, src.data(), m * sizeof(ListSrc));
  int64_t* h_pre = reinterpret_cast<int64_t*>(reinterpret_cast<uint8_t*>(h_src) + round_up(m * sizeof(ListSrc), 16));
  memcpy(h_pre, out_prefix, (m + 1) * 8);
  RET(ix->sl_buf.ensure(in_bytes + 64));
  uint8_t* base = ix->sl_buf.as<uint8_t>();
  CK(cudaMemcpyAsync(base, h, in_bytes, cudaMemcpyHostToDevice, st));
  float* d_q = reinterpret_cast<float*>(base);
  ListSrc* d_src = reinterpret_cast<ListSrc*>(base + round_up(dp * 4, 16));
  int64_t* d_pre = reinterpret_cast<int64_t*>(reinterpret_cast<uint8_t*>(d_src) + round_up(m * sizeof(ListSrc), 16));
  float* d_qn = reinterpret_cast<float*>(base + in_bytes);  // |q| for cosine (sequential fp32)
  int64_t* o_ids = reinterpret_cast<int64_t*>(ix->hsl.dev + in_bytes);  // mapped outputs
  float* o_d = reinterpret_cast<float*>(o_ids + std::max<int64_t>(total, 1));
  if (ix->metric == COSINE) launch_qnorm(d_q, dp, 1, (int)ix->d, d_qn, st);
  launch_lists_dist(ix->metric, d_q, d_qn, d_src, d_pre, m, total, (int)dp, (int)ix->d, o_d, o_ids, st);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(st));
  if (total > 0) {
    const int64_t* r_ids = reinterpret_cast<const int64_t*>(ix->hsl.p + in_bytes);
    memcpy(out_ids, r_ids, total * 8);
    memcpy(out_dists, r_ids + std::max<int64_t>(total, 1), total * 4);
  }
  return PK_OK;
}

// ---- agent path (pk_agent.cu) ---------------------------------------------

}  // extern "C"

namespace {
// grow the agent row store to at least `need` slots, contents kept
int rows_reserve(pk_index* ix, int64_t need) {
  if (need <= ix->acap) return PK_OK;
  static const bool dbg = getenv("PK_DEBUG_GROW") != nullptr;  // (measurement only)
  const auto t0 = std::chrono::steady_clock::now();
  const int64_t nc = std::max<int64_t>({need, ix->acap + ix->acap / 2, 1024});
  struct Report {
    bool on;
    int64_t from, to;
    std::chrono::steady_clock::time_point t0;
    ~Report() {
      if (on)
        fprintf(stderr, "row store grow %lld -> %lld rows: %.1f ms\n", (long long)from, (long long)to,
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
  } rep{dbg, ix->acap, nc, t0};
  void* p = nullptr;
  CK(cudaMalloc(&p, (size_t)nc * ix->dp * 4));
  if (ix->acap)
    CK(cudaMemcpyAsync(p, ix->arows.p, (size_t)ix->acap * ix->dp * 4, cudaMemcpyDeviceToDevice, ix->st));
  CK(cudaStreamSynchronize(ix->st));
  ix->arows.release();
  ix->arows.p = p;
  ix->arows.bytes = (size_t)nc * ix->dp * 4;
  ix->acap = nc;
  return PK_OK;
}
// bump layout of one packed staging block (16-byte aligned pieces)
struct Layout {
  size_t off = 0;
  size_t take(size_t bytes) {
    const size_t o = off;
    off = (size_t)round_up((int64_t)(off + bytes), 16);
    return o;
  }
};
}  // namespace

extern "C" {

int pk_rows_put(pk_index* ix, const int32_t* slots, const float* rows, int64_t n) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  if (n < 0) return fail(PK_ERR_USAGE, "negative row count");
  if (n == 0) return PK_OK;
  CK(cudaSetDevice(ix->device));
  int64_t mx = -1;
  for (int64_t i = 0; i < n; i++) {
    if (slots[i] < 0) return fail(PK_ERR_USAGE, "negative row slot");
    mx = std::max<int64_t>(mx, slots[i]);
  }
  RET(rows_reserve(ix, mx + 1));
  const int64_t dp = ix->dp;
  Layout L;
  const size_t o_sl = L.take((size_t)n * 4), o_rw = L.take((size_t)n * dp * 4);
  RET(ix->hag.ensure(L.off));
  RET(ix->ag_in.ensure(L.off));
  memcpy(ix->hag.p + o_sl, slots, (size_t)n * 4);
  pack_padded(reinterpret_cast<float*>(ix->hag.p + o_rw), rows, n, ix->d, dp);
  cudaStream_t st = ix->st;
  uint8_t* din = ix->ag_in.as<uint8_t>();
  CK(cudaMemcpyAsync(din, ix->hag.p, L.off, cudaMemcpyHostToDevice, st));
  launch_rows_put(reinterpret_cast<const float*>(din + o_rw), reinterpret_cast<const int32_t*>(din + o_sl), (int)n,
                  (int)dp, ix->arows.as<float>(), st);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(st));  // the staging block is reused by the next call
  return PK_OK;
}

int pk_agent_read(pk_index* ix, const float* q, const int32_t* put_slots, const float* put_rows, int64_t nput,
                  const int32_t* slots, int64_t n, float* out_d, const int32_t* mq, int32_t nmq,
                  const int32_t* mx, int32_t nmx, float* out_m, const int32_t* scope_codes, int32_t nscopes,
                  int32_t nprobe, int32_t ef, int32_t mode, int64_t* out_cids, int32_t* out_coarse,
                  int64_t* out_prefix, int64_t* out_ids, float* out_dists, int64_t cap) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  if (nput < 0 || n < 0 || nmq < 0 || nmx < 0 || nprobe < 0 || cap < 0)
    return fail(PK_ERR_USAGE, "negative count");
  if (nprobe > 0) {
    if (nscopes < 1 || nscopes > 64) return fail(PK_ERR_USAGE, "scope count must lie in [1, 64]");
    if (mode != 0 && mode != 1) return fail(PK_ERR_USAGE, "graph mode must be 0 (hybrid) or 1 (per-scope)");
    if (!out_cids || !out_coarse || !out_prefix || (cap > 0 && (!out_ids || !out_dists)))
      return fail(PK_ERR_USAGE, "missing list outputs");
  }
  CK(cudaSetDevice(ix->device));
  cudaStream_t st = ix->st;
  int64_t mxs = -1;
  for (int64_t i = 0; i < nput; i++) {
    if (put_slots[i] < 0) return fail(PK_ERR_USAGE, "negative row slot");
    mxs = std::max<int64_t>(mxs, put_slots[i]);
  }
  RET(rows_reserve(ix, mxs + 1));
  auto bad = [&](const int32_t* v, int64_t m) {
    for (int64_t i = 0; i < m; i++)
      if (v[i] < 0 || v[i] >= ix->acap) return true;
    return false;
  };
  if (bad(slots, n) || bad(mq, nmq) || bad(mx, nmx)) return fail(PK_ERR_USAGE, "row slot out of range");
  if (ix->tiered && nprobe > 0) RET(ix->poll_migrations());
  if (nprobe > 0) RET(ix->sync_table());
  const int64_t dp = ix->dp, d = ix->d;
  const bool lists = nprobe > 0 && ix->nslots > 0;
  const int64_t maxlen = lists ? ix->max_list_len() : 0;
  const int64_t rcap = lists ? std::min<int64_t>(cap, (int64_t)nprobe * maxlen) : 0;
  // inputs: q | put slots | put rows | read slots | matrix query / row slots
  Layout L;
  const size_t o_q = L.take(dp * 4), o_ps = L.take(nput * 4), o_pr = L.take((size_t)nput * dp * 4),
               o_sl = L.take(n * 4), o_mq = L.take((size_t)nmq * 4), o_mx = L.take((size_t)nmx * 4);
  const size_t in_bytes = L.off;
  // outputs (mapped; written by the kernels, read after one sync)
  const size_t o_od = L.take(n * 4), o_om = L.take((size_t)nmq * nmx * 4), o_cid = L.take((size_t)nprobe * 8),
               o_pre = L.take((size_t)(nprobe + 1) * 8), o_cnt = L.take(8), o_ids = L.take((size_t)rcap * 8),
               o_dd = L.take((size_t)rcap * 4);
  RET(ix->hag.ensure(L.off));
  RET(ix->ag_in.ensure(in_bytes));
  uint8_t* h = ix->hag.p;
  uint8_t* hd = ix->hag.dev;
  memcpy(h + o_q, q, d * 4);
  if (dp > d) memset(h + o_q + d * 4, 0, (dp - d) * 4);
  if (nput) {
    memcpy(h + o_ps, put_slots, nput * 4);
    pack_padded(reinterpret_cast<float*>(h + o_pr), put_rows, nput, d, dp);
  }
  if (n) memcpy(h + o_sl, slots, n * 4);
  if (nmq) memcpy(h + o_mq, mq, (size_t)nmq * 4);
  if (nmx) memcpy(h + o_mx, mx, (size_t)nmx * 4);
  uint8_t* din = ix->ag_in.as<uint8_t>();
  // PK_DEBUG_AGENT=1: per-phase device time (events; measurement only)
  static const bool dbg = getenv("PK_DEBUG_AGENT") != nullptr;
  static cudaEvent_t dev_[8];
  static double dacc[8] = {0};
  static long dcalls = 0;
  static bool dinit = false;
  if (dbg && !dinit) {
    for (auto& e : dev_) cudaEventCreate(&e);
    dinit = true;
  }
  auto mark = [&](int i) {
    if (dbg) cudaEventRecord(dev_[i], st);
  };
  mark(0);
  CK(cudaMemcpyAsync(din, h, in_bytes, cudaMemcpyHostToDevice, st));
  const float* dq = reinterpret_cast<const float*>(din + o_q);
  float* arows = ix->arows.as<float>();
  if (nput)
    launch_rows_put(reinterpret_cast<const float*>(din + o_pr), reinterpret_cast<const int32_t*>(din + o_ps),
                    (int)nput, (int)dp, arows, st);
  mark(1);
  // the row-store distances run on a side stream, beside the coarse traversal
  // and the list scan (independent inputs; joined before the sync)
  if (!ix->ast) {
    CK(cudaStreamCreateWithFlags(&ix->ast, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ix->ev_ag0, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ix->ev_ag1, cudaEventDisableTiming));
  }
  cudaStream_t as = dbg ? st : ix->ast;
  if (!dbg) {
    CK(cudaEventRecord(ix->ev_ag0, st));
    CK(cudaStreamWaitEvent(as, ix->ev_ag0, 0));
  }
  launch_gather_dist(ix->metric, dq, arows, (int)dp, (int)d, reinterpret_cast<const int32_t*>(din + o_sl), (int)n,
                     reinterpret_cast<float*>(hd + o_od), as);
  mark(2);
  launch_gather_mat(ix->metric, arows, (int)dp, (int)d, reinterpret_cast<const int32_t*>(din + o_mq), nmq,
                    reinterpret_cast<const int32_t*>(din + o_mx), nmx, reinterpret_cast<float*>(hd + o_om), as);
  if (!dbg) CK(cudaEventRecord(ix->ev_ag1, as));
  mark(3);
  int64_t* h_pre = reinterpret_cast<int64_t*>(h + o_pre);
  int64_t* h_cid = reinterpret_cast<int64_t*>(h + o_cid);
  if (lists) {
    // the reference's coarse traversal for this query (graph_coarse), then
    // every row of every probed list in coarse order
    pk_index::Scratch& S = ix->scr[ix->par];
    RET(S.q.ensure(dp * 4));
    RET(S.qnorm.ensure(4));
    RET(S.probe.ensure((size_t)nprobe * 4));
    CK(cudaMemcpyAsync(S.q.p, dq, dp * 4, cudaMemcpyDeviceToDevice, st));
    if (ix->metric == COSINE) launch_qnorm(S.q.as<float>(), dp, 1, (int)d, S.qnorm.as<float>(), st);
    GraphArgs ga;
    ga.ef = ef;
    ga.mode = mode;
    ga.out_coarse = reinterpret_cast<int32_t*>(h + o_cnt);
    RET(graph_coarse(ix, S, 1, scope_codes, nscopes, nprobe, ga, st));
    mark(4);
    if (!ix->tiered) {
      launch_probe_lists(ix->metric, S.q.as<float>(), ix->table(), S.probe.as<int32_t>(), nprobe, maxlen, rcap,
                         reinterpret_cast<float*>(hd + o_dd), reinterpret_cast<int64_t*>(hd + o_ids),
                         reinterpret_cast<int64_t*>(hd + o_pre), reinterpret_cast<int64_t*>(hd + o_cid), st);
    } else {
      // cold lists are read in place from the mapped host arena: the sources
      // need the probe on the host (pk_scan_lists' layout)
      std::vector<int32_t> pr(nprobe);
      CK(cudaMemcpyAsync(pr.data(), S.probe.p, (size_t)nprobe * 4, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      std::vector<ListSrc> src;
      std::vector<int64_t> pre(1, 0);
      h_pre[0] = 0;
      for (int32_t l = 0; l < nprobe; l++) {
        const int32_t sl = pr[l];
        h_cid[l] = sl >= 0 ? ix->h_cid[sl] : -1;
        h_pre[l + 1] = h_pre[l] + (sl >= 0 ? ix->h_len[sl] : 0);
        if (sl < 0) continue;
        ListSrc x;
        if (ix->h_res[sl]) {
          x.rows = ix->rows + ix->h_off[sl] * dp;
          x.ids = ix->ids + ix->h_off[sl];
        } else {
          x.rows = ix->hrows_d + ix->h_hoff[sl] * dp;
          x.ids = ix->hids_d + ix->h_hoff[sl];
        }
        src.push_back(x);
        pre.push_back(pre.back() + ix->h_len[sl]);
      }
      const int64_t total = std::min<int64_t>(pre.back(), rcap);
      const int m = (int)src.size();
      if (m > 0 && total > 0) {
        // the list sources + prefix (clamped to the capacity) in one copy
        const size_t sb = round_up(m * sizeof(ListSrc), 16), pb = (size_t)(m + 1) * 8;
        RET(ix->sl_buf.ensure(sb + pb));
        std::vector<uint8_t> blk(sb + pb);
        memcpy(blk.data(), src.data(), m * sizeof(ListSrc));
        for (auto& v : pre) v = std::min<int64_t>(v, total);
        memcpy(blk.data() + sb, pre.data(), pb);
        CK(cudaMemcpyAsync(ix->sl_buf.p, blk.data(), blk.size(), cudaMemcpyHostToDevice, st));
        launch_lists_dist(ix->metric, S.q.as<float>(), S.qnorm.as<float>(),
                          ix->sl_buf.as<ListSrc>(),
                          reinterpret_cast<const int64_t*>(ix->sl_buf.as<uint8_t>() + sb), m, total, (int)dp,
                          (int)d, reinterpret_cast<float*>(hd + o_dd), reinterpret_cast<int64_t*>(hd + o_ids), st);
        CK(cudaStreamSynchronize(st));  // blk (pageable) and the sources in flight
      }
    }
  }
  mark(5);
  if (!dbg) CK(cudaStreamWaitEvent(st, ix->ev_ag1, 0));
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(st));
  if (dbg) {
    float ms;
    const int last = lists ? 5 : 3;
    for (int i = 1; i <= last; i++) {
      if (!lists && i > 3) break;
      cudaEventElapsedTime(&ms, dev_[i - 1], dev_[i]);
      dacc[i] += ms;
    }
    if (++dcalls % 512 == 0)
      fprintf(stderr, "agent_read device us/call (%ld calls): h2d+puts %.1f gather %.1f mat %.1f coarse %.1f lists %.1f\n",
              dcalls, 1e3 * dacc[1] / dcalls, 1e3 * dacc[2] / dcalls, 1e3 * dacc[3] / dcalls, 1e3 * dacc[4] / dcalls,
              1e3 * dacc[5] / dcalls);
  }
  if (n) memcpy(out_d, h + o_od, n * 4);
  if (nmq && nmx) memcpy(out_m, h + o_om, (size_t)nmq * nmx * 4);
  if (nprobe > 0) {
    if (!lists) {
      for (int32_t l = 0; l < nprobe; l++) out_cids[l] = -1;
      for (int32_t l = 0; l <= nprobe; l++) out_prefix[l] = 0;
      *out_coarse = 0;
      return PK_OK;
    }
    memcpy(out_cids, h_cid, (size_t)nprobe * 8);
    memcpy(out_prefix, h_pre, (size_t)(nprobe + 1) * 8);
    *out_coarse = *reinterpret_cast<int32_t*>(h + o_cnt);
    const int64_t total = h_pre[nprobe];
    if (total > cap) return fail(PK_ERR_USAGE, "probed lists hold %lld rows, capacity %lld", (long long)total, (long long)cap);
    memcpy(out_ids, h + o_ids, total * 8);
    memcpy(out_dists, h + o_dd, total * 4);
  }
  return PK_OK;
}

int pk_rows_reserve(pk_index* ix, int64_t n) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  if (n < 0) return fail(PK_ERR_USAGE, "negative count");
  CK(cudaSetDevice(ix->device));
  return rows_reserve(ix, n);
}

int pk_list_version(pk_index* ix, uint64_t* version) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  if (!version) return fail(PK_ERR_USAGE, "null output");
  *version = ix->tver;
  return PK_OK;
}

int pk_agent_lists(pk_index* ix, const float* Q, int64_t B, const int32_t* scope_codes, int32_t nscopes,
                   int32_t nprobe, int32_t ef, int32_t mode, int64_t cap, int64_t* out_cids, int32_t* out_coarse,
                   int64_t* out_prefix, int64_t* out_ids, float* out_dists, uint64_t* out_version) {
  // The list half of pk_agent_read for B queries at once: the reference's
  // coarse traversal of each (one CTA per query) and every row of the lists
  // it probes, query b's rows in [b * cap, (b + 1) * cap) (a total above cap
  // is reported by the prefix, the rows past it are not written).  Valid as
  // long as pk_list_version still returns *out_version.
  std::lock_guard<CountedMutex> lock_(ix->mu);
  if (B < 0 || nprobe < 1 || cap < 0) return fail(PK_ERR_USAGE, "bad count");
  if (nscopes < 1 || nscopes > 64) return fail(PK_ERR_USAGE, "scope count must lie in [1, 64]");
  if (mode != 0 && mode != 1) return fail(PK_ERR_USAGE, "graph mode must be 0 (hybrid) or 1 (per-scope)");
  if (ix->tiered) return fail(PK_ERR_USAGE, "pk_agent_lists: the tiered index reads cold lists per query");
  if (!out_cids || !out_coarse || !out_prefix || !out_version || (cap > 0 && (!out_ids || !out_dists)))
    return fail(PK_ERR_USAGE, "missing outputs");
  if (B == 0 || ix->nslots == 0) {
    for (int64_t i = 0; i < B * nprobe; i++) out_cids[i] = -1;
    for (int64_t i = 0; i < B * (nprobe + 1); i++) out_prefix[i] = 0;
    for (int64_t i = 0; i < B; i++) out_coarse[i] = 0;
    *out_version = ix->tver;
    return PK_OK;
  }
  CK(cudaSetDevice(ix->device));
  cudaStream_t st = ix->st;
  RET(ix->sync_table());
  const int64_t dp = ix->dp, d = ix->d;
  const int64_t maxlen = ix->max_list_len();
  const int64_t rcap = std::min<int64_t>(cap, (int64_t)nprobe * maxlen);
  Layout L;
  const size_t o_q = L.take((size_t)B * dp * 4);
  const size_t in_bytes = L.off;
  const size_t o_cid = L.take((size_t)B * nprobe * 8), o_pre = L.take((size_t)B * (nprobe + 1) * 8),
               o_cnt = L.take((size_t)B * 4), o_ids = L.take((size_t)B * rcap * 8),
               o_dd = L.take((size_t)B * rcap * 4);
  RET(ix->hal.ensure(L.off));
  RET(ix->al_in.ensure(in_bytes));
  uint8_t* h = ix->hal.p;
  uint8_t* hd = ix->hal.dev;
  pack_padded(reinterpret_cast<float*>(h + o_q), Q, B, d, dp);
  CK(cudaMemcpyAsync(ix->al_in.p, h, in_bytes, cudaMemcpyHostToDevice, st));
  pk_index::Scratch& S = ix->scr[ix->par];
  RET(S.q.ensure((size_t)B * dp * 4));
  RET(S.qnorm.ensure((size_t)B * 4));
  RET(S.probe.ensure((size_t)B * nprobe * 4));
  CK(cudaMemcpyAsync(S.q.p, ix->al_in.p, (size_t)B * dp * 4, cudaMemcpyDeviceToDevice, st));
  if (ix->metric == COSINE) launch_qnorm(S.q.as<float>(), dp, (int)B, (int)d, S.qnorm.as<float>(), st);
  GraphArgs ga;
  ga.ef = ef;
  ga.mode = mode;
  ga.out_coarse = reinterpret_cast<int32_t*>(h + o_cnt);
  RET(graph_coarse(ix, S, B, scope_codes, nscopes, nprobe, ga, st));
  launch_probe_lists(ix->metric, S.q.as<float>(), ix->table(), S.probe.as<int32_t>(), nprobe, maxlen, rcap,
                     reinterpret_cast<float*>(hd + o_dd), reinterpret_cast<int64_t*>(hd + o_ids),
                     reinterpret_cast<int64_t*>(hd + o_pre), reinterpret_cast<int64_t*>(hd + o_cid), st, (int)B);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(st));
  memcpy(out_cids, h + o_cid, (size_t)B * nprobe * 8);
  memcpy(out_prefix, h + o_pre, (size_t)B * (nprobe + 1) * 8);
  memcpy(out_coarse, h + o_cnt, (size_t)B * 4);
  for (int64_t b = 0; b < B; b++) {
    const int64_t tot = std::min<int64_t>(out_prefix[b * (nprobe + 1) + nprobe], rcap);
    memcpy(out_ids + b * cap, h + o_ids + (size_t)b * rcap * 8, tot * 8);
    memcpy(out_dists + b * cap, h + o_dd + (size_t)b * rcap * 4, tot * 4);
  }
  *out_version = ix->tver;
  return PK_OK;
}

int pk_l1_place(pk_index* ix, int32_t nc, int32_t n_p, int32_t capacity, const double* sums, const float* cents,
                const int32_t* counts, const float* items, const int64_t* item_ids, const int32_t* holder,
                int32_t m, const float* q, int32_t* out_target, uint8_t* out_added, uint8_t* out_merged,
                int32_t* out_qtarget) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  if (nc < 0 || m < 0 || n_p < 1 || capacity < 1) return fail(PK_ERR_USAGE, "bad L1 placement shape");
  const int maxc = l1_place_max_clusters();
  if (n_p > maxc || nc + m > maxc)
    return fail(PK_ERR_USAGE, "L1 placement of %d items over %d clusters exceeds %d", m, nc, maxc);
  if (nc > n_p) return fail(PK_ERR_USAGE, "%d live L1 clusters above n_p %d", nc, n_p);
  if (((int64_t)n_p * (ix->dp + 4) + ix->dp) * 4 > 227 * 1024)
    return fail(PK_ERR_USAGE, "n_p %d x dimension %lld exceeds the placement kernel's shared memory", n_p,
                (long long)ix->d);
  if (m == 0 && !q) return PK_OK;
  CK(cudaSetDevice(ix->device));
  cudaStream_t st = ix->st;
  const int64_t dp = ix->dp, d = ix->d;
  const int64_t ncap = nc + m;
  Layout L;
  const size_t o_s = L.take((size_t)ncap * dp * 8), o_c = L.take((size_t)ncap * dp * 4),
               o_n = L.take((size_t)ncap * 4), o_it = L.take((size_t)m * dp * 4), o_h = L.take((size_t)m * 4),
               o_dup = L.take((size_t)m * 4), o_q = L.take(dp * 4);
  const size_t in_bytes = L.off;
  const size_t o_t = L.take((size_t)m * 4), o_a = L.take(m), o_m = L.take(m), o_qt = L.take(4);
  RET(ix->hag.ensure(L.off));
  RET(ix->ag_l1.ensure(in_bytes));
  uint8_t* h = ix->hag.p;
  double* hs = reinterpret_cast<double*>(h + o_s);
  for (int32_t c = 0; c < nc; c++) {
    memcpy(hs + (int64_t)c * dp, sums + (int64_t)c * d, d * 8);
    for (int64_t j = d; j < dp; j++) hs[(int64_t)c * dp + j] = 0.0;
  }
  pack_padded(reinterpret_cast<float*>(h + o_c), cents, nc, d, dp);
  memcpy(h + o_n, counts, (size_t)nc * 4);
  pack_padded(reinterpret_cast<float*>(h + o_it), items, m, d, dp);
  memcpy(h + o_h, holder, (size_t)m * 4);
  {  // earlier occurrence of the same item in this chain (an id evicted with
     // an L0 entry can come back with the new entry's overflow)
    int32_t* du = reinterpret_cast<int32_t*>(h + o_dup);
    std::unordered_map<int64_t, int32_t> last;
    for (int32_t i = 0; i < m; i++) {
      auto it = last.find(item_ids[i]);
      du[i] = it == last.end() ? -1 : it->second;
      last[item_ids[i]] = i;
    }
  }
  if (q) pack_padded(reinterpret_cast<float*>(h + o_q), q, 1, d, dp);
  // only the live clusters' state and the items cross (fresh clusters start
  // in device memory)
  uint8_t* dv = ix->ag_l1.as<uint8_t>();
  CK(cudaMemcpyAsync(dv + o_s, h + o_s, (size_t)nc * dp * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(dv + o_c, h + o_c, (size_t)(in_bytes - o_c), cudaMemcpyHostToDevice, st));
  uint8_t* hd = ix->hag.dev;
  launch_l1_place(ix->metric, nc, n_p, capacity, (int)dp, (int)d, reinterpret_cast<double*>(dv + o_s),
                  reinterpret_cast<float*>(dv + o_c), reinterpret_cast<int32_t*>(dv + o_n),
                  reinterpret_cast<const float*>(dv + o_it), reinterpret_cast<const int32_t*>(dv + o_h),
                  reinterpret_cast<const int32_t*>(dv + o_dup), m,
                  q ? reinterpret_cast<const float*>(dv + o_q) : nullptr, reinterpret_cast<int32_t*>(hd + o_t),
                  hd + o_a, hd + o_m, reinterpret_cast<int32_t*>(hd + o_qt), st);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(st));
  memcpy(out_target, h + o_t, (size_t)m * 4);
  memcpy(out_added, h + o_a, m);
  memcpy(out_merged, h + o_m, m);
  if (q && out_qtarget) *out_qtarget = *reinterpret_cast<int32_t*>(h + o_qt);
  return PK_OK;
}

int pk_debug_pool_counts(pk_index* ix, int32_t* out, int64_t B) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  if (!ix->screen) return fail(PK_ERR_USAGE, "no candidate pools: exact scan mode");
  auto& S = ix->scr[ix->last_par];
  if ((size_t)B * 4 > S.ccount.bytes) return fail(PK_ERR_USAGE, "batch larger than the last search");
  CK(cudaMemcpyAsync(out, S.ccount.p, (size_t)B * 4, cudaMemcpyDeviceToHost, ix->st));
  CK(cudaStreamSynchronize(ix->st));
  return PK_OK;
}

int pk_debug_rerank_counts(pk_index* ix, int32_t* out, int64_t B) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  if (!ix->screen) return fail(PK_ERR_USAGE, "no candidate pools: exact scan mode");
  auto& S = ix->scr[ix->last_par];
  if ((size_t)B * 4 > S.nsurv.bytes) return fail(PK_ERR_USAGE, "batch larger than the last search");
  CK(cudaMemcpyAsync(out, S.nsurv.p, (size_t)B * 4, cudaMemcpyDeviceToHost, ix->st));
  CK(cudaStreamSynchronize(ix->st));
  return PK_OK;
}

int pk_debug_fail_next_alloc(pk_index* ix, int n) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  ix->fail_alloc = std::max(n, 0);
  return PK_OK;
}

int pk_debug_coarse_counts(pk_index* ix, int32_t* out, int64_t B) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  if (!ix->coarse_tc) return fail(PK_ERR_USAGE, "exact coarse quantizer: no screened candidates");
  auto& S = ix->scr[ix->last_par];
  if ((size_t)B * 4 > S.ncand.bytes) return fail(PK_ERR_USAGE, "batch larger than the last search");
  CK(cudaMemcpyAsync(out, S.ncand.p, (size_t)B * 4, cudaMemcpyDeviceToHost, ix->st));
  CK(cudaStreamSynchronize(ix->st));
  return PK_OK;
}

int pk_profile_begin(pk_index* ix) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  ix->prof = true;
  ix->prof_calls = 0;
  return PK_OK;
}

int pk_profile_end(pk_index* ix, double* stage_ms, int nstages, int* ncalls) {
  std::lock_guard<CountedMutex> lock_(ix->mu);
  CK(cudaStreamSynchronize(ix->st));
  const int ns = std::min(nstages, pk_index::NSTAGE);
  for (int k = 0; k < nstages; k++) stage_ms[k] = 0.0;
  for (int c = 0; c < ix->prof_calls; c++) {
    for (int k = 0; k < ns; k++) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, ix->prof_ev[(size_t)c * (pk_index::NSTAGE + 1) + k],
                              ix->prof_ev[(size_t)c * (pk_index::NSTAGE + 1) + k + 1]));
      stage_ms[k] += ms;
    }
  }
  *ncalls = ix->prof_calls;
  ix->prof = false;
  ix->prof_calls = 0;
  return PK_OK;
}

int pk_assign(pk_index* ix, const float* X, int64_t n, int32_t scope_code, int64_t* out_cid,
              float* out_dist, int flags) {
  // PK_DEBUG_ASSIGN=1: host-side microseconds per step (measurement only)
  static const bool dbg = getenv("PK_DEBUG_ASSIGN") != nullptr;
  static double tacc[8] = {0};
  static long tcalls = 0;
  auto t0 = std::chrono::steady_clock::now();
  auto tick = [&](int i) {
    if (!dbg) return;
    auto t = std::chrono::steady_clock::now();
    tacc[i] += std::chrono::duration<double, std::micro>(t - t0).count();
    t0 = t;
  };
  std::lock_guard<CountedMutex> lock_(ix->mu);
  tick(0);
  if (n < 0) return fail(PK_ERR_USAGE, "negative count");
  if (n == 0) return PK_OK;
  CK(cudaSetDevice(ix->device));
  const bool dev = flags & PK_DEVICE_PTRS;
  cudaStream_t st = ix->st;
  RET(ix->sync_table());
  const int64_t dp = ix->dp;
  const int32_t ns = std::max<int32_t>(ix->nslots, 1);
  const bool fresh_q = ix->assign_q.bytes < (size_t)n * dp * 4;
  RET(ix->assign_q.ensure((size_t)n * dp * 4));
  if (fresh_q) CK(cudaMemsetAsync(ix->assign_q.p, 0, ix->assign_q.bytes, st));
  RET(ix->assign_qn.ensure(n * 4));
  RET(ix->assign_dc.ensure((size_t)n * ns * 4));
  RET(ix->assign_c.ensure(n * 8));
  RET(ix->assign_d.ensure(n * 4));
  tick(1);
  // host path (the insert path's batch of 8): the rows go over in ONE DMA
  // from pinned staging, padded on the host, and the argmin writes (cid,
  // dist) straight into mapped pinned memory -- no pageable 2-D copies, no
  // read-back copies, one synchronisation
  int64_t* oc = out_cid;
  float* od = out_dist;
  if (dev) {
    CK(cudaMemcpy2DAsync(ix->assign_q.p, dp * 4, X, ix->d * 4, ix->d * 4, n, cudaMemcpyDeviceToDevice, st));
  } else {
    const size_t in_b = (size_t)n * dp * 4;
    RET(ix->hasg.ensure(in_b + (size_t)n * 12));
    float* hq = reinterpret_cast<float*>(ix->hasg.p);
    for (int64_t r = 0; r < n; r++) {
      memcpy(hq + r * dp, X + r * ix->d, ix->d * 4);
      if (dp > ix->d) memset(hq + r * dp + ix->d, 0, (dp - ix->d) * 4);
    }
    CK(cudaMemcpyAsync(ix->assign_q.p, hq, in_b, cudaMemcpyHostToDevice, st));
    oc = reinterpret_cast<int64_t*>(ix->hasg.dev + in_b);
    od = reinterpret_cast<float*>(ix->hasg.dev + in_b + (size_t)n * 8);
  }
  tick(2);
  if (ix->metric == COSINE) launch_qnorm(ix->assign_q.as<float>(), dp, (int)n, (int)ix->d, ix->assign_qn.as<float>(), st);
  // one launch: distances + argmin by (dist, cid) (cids below 2^32: the
  // packed key), else the dense matrix and a separate argmin
  bool small_cids = true;
  for (int32_t sl = 0; sl < ix->nslots && small_cids; sl++) small_cids = ix->h_cid[sl] < ((int64_t)1 << 32);
  if (small_cids && ix->nslots > 0) {
    const size_t pb = (size_t)dense_argmin_blocks(ix->nslots, (int)n) * 8;
    if (ix->assign_part.bytes < pb) RET(ix->assign_part.ensure(pb));
    if (!ix->assign_ctr.p) {
      RET(ix->assign_ctr.ensure(64));
      CK(cudaMemsetAsync(ix->assign_ctr.p, 0, 64, st));
    }
    launch_dense_argmin(ix->metric, ix->assign_q.as<float>(), dp, (int)n, ix->d_cent, ix->nslots, (int)dp,
                        ix->assign_qn.as<float>(), ix->table(), scope_code,
                        ix->assign_part.as<unsigned long long>(), ix->assign_ctr.as<unsigned>(), oc, od, st);
  } else {
    launch_dist_dense(ix->metric, ix->assign_q.as<float>(), dp, (int)n, ix->d_cent, dp, ix->nslots, (int)dp,
                      ix->assign_qn.as<float>(), ix->assign_dc.as<float>(), ns, st);
    launch_argmin(ix->assign_dc.as<float>(), ns, (int)n, ix->table(), scope_code, oc, od, st);
  }
  CK(cudaGetLastError());
  tick(3);
  if (!dev) {
    CK(cudaStreamSynchronize(st));
    tick(4);
    if (dbg && ++tcalls % 1000 == 0)
      fprintf(stderr, "pk_assign host us/call: lock %.1f setup %.1f stage+h2d %.1f launches %.1f sync %.1f\n",
              tacc[0] / tcalls, tacc[1] / tcalls, tacc[2] / tcalls, tacc[3] / tcalls, tacc[4] / tcalls);
    const size_t in_b = (size_t)n * dp * 4;
    memcpy(out_cid, ix->hasg.p + in_b, n * 8);
    if (out_dist) memcpy(out_dist, ix->hasg.p + in_b + (size_t)n * 8, n * 4);
  }
  return PK_OK;
}

}  // extern "C"
