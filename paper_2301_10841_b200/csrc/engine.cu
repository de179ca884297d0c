// B200 Free Join executor: device COLT + vectorised node execution.
//
// Reference map (all behaviour restated from the SPEC/paper; no reference code
// exists for this path):
//   GHT new / BaseScan
//   COLT force / get / iter   SPEC.md:295-330, Fig 12
//   estimated_key_count
//   select_cover (dynamic)
//   join_vectorized (Fig 13)
//   output sinks / counters
//
// Execution model: breadth-first within a chunk, depth-first over chunks.
// Node k receives a frontier of bindings (SoA: bound variables, per-atom
// current subtrie (id, len), multiplicity). One node =
//   k_select   per binding: dynamic cover (min estimated_key_count, ties to the
//              lowest position), candidate count, claims of unforced subtries
//              every probe/keys-iteration of this node needs (lazy forcing in
//              batch, deduplicated by CAS on the subtrie state)
//   scan       inclusive scan of candidate counts (kernels/prims.cuh: decoupled look-back)
//   force      per (trie, level) with claims: insert -> assign -> scatter
//   k_expand   per candidate (load-balanced over the scan): iterate the cover,
//              probe every other subatom in node order, drop misses, compact
//              survivors into the next frontier -- or, at the last node, fold
//              count / checksum / MIN (or write tuples) in registers.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <type_traits>
#include <unordered_map>
#include <vector>

#include "../../include/fjg.h"
#include "engine.cuh"
#include "fj_errors.hpp"
#include "fj_plan.hpp"

namespace fjg {
void set_last_error(const std::string& s);
}

using namespace fjg;

// ============================================================================
// errors
// ============================================================================
static void throw_cuda(cudaError_t e, const char* what, int line) {
  std::string msg = std::string("CUDA error ") + cudaGetErrorString(e) + " in " + what + " (engine.cu:" +
                    std::to_string(line) + ")";
  if (e == cudaErrorMemoryAllocation) throw fj::ResourceError(msg);
  throw fj::EngineError(msg);
}
#define CK(x)                                  \
  do {                                         \
    cudaError_t _e = (x);                      \
    if (_e != cudaSuccess) throw_cuda(_e, #x, __LINE__); \
  } while (0)

#include "kernels/prims.cuh"
#include "kernels/common.cuh"
#include "kernels/select.cuh"
#include "kernels/force.cuh"
#include "kernels/node_generic.cuh"
#include "kernels/memo.cuh"
#include "kernels/node_fastpaths.cuh"

// host-side dispatch on the query width (max(#vars, #atoms) -> 4 / 8 / 16)
template <int MODE>
static void launch_expand(int width, unsigned grid, cudaStream_t st, const KNode& nd, uint64_t c0, uint64_t c1,
                          uint64_t F, const uint64_t* bounds, int min_var, int32_t* out, uint64_t cap,
                          DevCounters* ctr) {
  static bool attr_set = false;
  if (!attr_set) {  // the W >= 8 variants keep per-candidate state in (>48 KB) dynamic shared memory
    cudaFuncSetAttribute(k_expand<MODE, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 8 * TILE * 4);
    cudaFuncSetAttribute(k_expand<MODE, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 16 * TILE * 4);
    attr_set = true;
  }
  if (width <= 4)
    k_expand<MODE, 4><<<grid, TILE, 0, st>>>(nd, c0, c1, F, bounds, min_var, out, cap, ctr);
  else if (width <= 8)
    k_expand<MODE, 8><<<grid, TILE, 3 * 8 * TILE * 4, st>>>(nd, c0, c1, F, bounds, min_var, out, cap, ctr);
  else
    k_expand<MODE, 16><<<grid, TILE, 3 * 16 * TILE * 4, st>>>(nd, c0, c1, F, bounds, min_var, out, cap, ctr);
}

#include "kernels/misc.cuh"

// ============================================================================
// host: memory pool
// ============================================================================
namespace {

class Pool {
 public:
  explicit Pool(int dev) : dev_(dev) {}
  ~Pool() {
    for (auto& kv : free_) cudaFree(kv.second);
    for (auto& kv : live_) cudaFree(kv.first);
  }
  void* alloc(size_t bytes) {
    if (bytes == 0) bytes = 1;
    const size_t gran = bytes >= (1u << 20) ? (2u << 20) : 512;
    bytes = (bytes + gran - 1) / gran * gran;
    auto it = free_.lower_bound(bytes);
    if (it != free_.end() && it->first <= bytes * 2) {
      void* p = it->second;
      live_[p] = it->first;
      free_.erase(it);
      return p;
    }
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      release_free();
      e = cudaMalloc(&p, bytes);
      if (e != cudaSuccess) {
        cudaGetLastError();
        throw fj::ResourceError("device allocation of " + std::to_string(bytes) + " bytes failed: " +
                                cudaGetErrorString(e));
      }
    }
    live_[p] = bytes;
    return p;
  }
  void free(void* p) {
    if (!p) return;
    auto it = live_.find(p);
    if (it == live_.end()) return;
    free_.emplace(it->second, p);
    live_.erase(it);
  }
  void release_free() {
    for (auto& kv : free_) cudaFree(kv.second);
    free_.clear();
  }

 private:
  int dev_;
  std::multimap<size_t, void*> free_;
  std::unordered_map<void*, size_t> live_;
};

inline unsigned grid_for(uint64_t n, int threads = 256, unsigned cap = 148u * 16u) {
  uint64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}


}  // namespace

// ============================================================================
// host: handles
// ============================================================================
struct fjg_engine {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::unique_ptr<Pool> pool;
  uint32_t launches = 0;
  uint32_t syncs = 0;
  int num_sms = 148;
  DevCounters* h_ctr = nullptr;  // pinned; shared by the engine's queries (execute is synchronous)
  // device-wide primitives (kernels/prims.cuh), all on `stream`: tile ticket
  // counter (never reset; the host keeps the running base), look-back words of
  // the scans and of the radix passes (separate regions: epochs are compared
  // against words of one layout only), radix histograms
  unsigned long long* prim_ticket = nullptr;
  uint64_t prim_tbase = 0;
  uint32_t prim_epoch = 0;
  void* prim_lb_scan = nullptr;
  size_t prim_lb_scan_bytes = 0;
  void* prim_lb_radix = nullptr;
  size_t prim_lb_radix_bytes = 0;
  uint32_t* prim_hist = nullptr;
};

struct fjg_relation {
  fjg_engine* eng = nullptr;
  uint64_t nrows = 0;
  int ncols = 0;
  std::vector<int32_t*> cols;
  std::vector<void*> owned;
};

namespace {

struct ScopedDevice {
  int prev = -1;
  explicit ScopedDevice(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~ScopedDevice() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// FJG_DEBUG_SYNC=1 (environment): synchronise after every launch so a device
// fault is reported at the kernel that raised it (debugging only).
static bool debug_sync() {
  static const bool on = getenv("FJG_DEBUG_SYNC") && atoi(getenv("FJG_DEBUG_SYNC")) != 0;
  return on;
}
#define LAUNCH(eng, ...)                                           \
  do {                                                             \
    __VA_ARGS__;                                                   \
    ++(eng)->launches;                                             \
    CK(cudaGetLastError());                                        \
    if (debug_sync()) CK(cudaStreamSynchronize((eng)->stream));    \
  } while (0)

// ---------------------------------------------------------------------------
// device-wide primitives (kernels/prims.cuh) on the engine stream
// ---------------------------------------------------------------------------
static uint32_t prim_epoch(fjg_engine* eng) {
  if (++eng->prim_epoch >= (1u << 30)) {  // 30-bit epochs wrapped: clear the look-back words
    eng->prim_epoch = 1;
    if (eng->prim_lb_scan) CK(cudaMemsetAsync(eng->prim_lb_scan, 0, eng->prim_lb_scan_bytes, eng->stream));
    if (eng->prim_lb_radix) CK(cudaMemsetAsync(eng->prim_lb_radix, 0, eng->prim_lb_radix_bytes, eng->stream));
  }
  return eng->prim_epoch;
}
static void* prim_region(fjg_engine* eng, void*& p, size_t& have, size_t bytes) {
  if (bytes > have) {
    eng->pool->free(p);
    p = eng->pool->alloc(bytes);
    have = bytes;
    CK(cudaMemsetAsync(p, 0, bytes, eng->stream));  // no stale word can carry a live epoch
  }
  return p;
}

// out[i] = Op(in[0..i]) (EXCL: Op(in[0..i-1])); in may alias out; *total (device,
// optional) = Op(in[0..n)).
template <class Op, bool EXCL, class In, class T>
static void prim_scan(fjg_engine* eng, const In* in, T* out, uint64_t n, T* total = nullptr) {
  if (n == 0) {
    if (total) CK(cudaMemsetAsync(total, 0, sizeof(T), eng->stream));
    return;
  }
  const uint64_t tiles = (n + prims::kScanTile - 1) / prims::kScanTile;
  if (tiles > 0x7fffffffull) throw fj::ValidationError("scan too large");
  auto* st = (prims::LBTile*)prim_region(eng, eng->prim_lb_scan, eng->prim_lb_scan_bytes,
                                          tiles * sizeof(prims::LBTile));
  const uint32_t ep = prim_epoch(eng);
  LAUNCH(eng, (prims::k_scan_lb<In, T, Op, EXCL><<<(unsigned)tiles, prims::kScanThreads, 0, eng->stream>>>(
                  in, out, n, st, eng->prim_ticket, eng->prim_tbase, ep, total)));
  eng->prim_tbase += tiles;
}

// out[j] = the j-th index i (ascending) with flags[i] != 0; *count (device) = how many.
static void prim_select_flagged(fjg_engine* eng, const uint8_t* flags, uint32_t* out, uint64_t n, uint32_t* count) {
  if (n == 0) {
    CK(cudaMemsetAsync(count, 0, 4, eng->stream));
    return;
  }
  const uint64_t tiles = (n + prims::kSelTile - 1) / prims::kSelTile;
  auto* st = (prims::LBTile*)prim_region(eng, eng->prim_lb_scan, eng->prim_lb_scan_bytes,
                                          tiles * sizeof(prims::LBTile));
  const uint32_t ep = prim_epoch(eng);
  LAUNCH(eng, (prims::k_select_flagged<<<(unsigned)tiles, prims::kScanThreads, 0, eng->stream>>>(
                  flags, out, n, st, eng->prim_ticket, eng->prim_tbase, ep, count)));
  eng->prim_tbase += tiles;
}

// *out (device) = max over in[0..n) (0 when n == 0).
static void prim_max_u32(fjg_engine* eng, const uint32_t* in, uint64_t n, uint32_t* out) {
  CK(cudaMemsetAsync(out, 0, 4, eng->stream));
  if (n) LAUNCH(eng, prims::k_reduce_max_u32<<<grid_for(n, 256, eng->num_sms * 8), 256, 0, eng->stream>>>(in, n, out));
}

// Radix passes of a sort on key bits [lo, hi): 9-bit digits at most.
static int prim_sort_passes(int lo, int hi) { return hi > lo ? (hi - lo + 8) / 9 : 0; }

// Stable sort of (k0, v0)[0..n) on key bits [lo, hi) (keys must have no bit
// set at or above hi), ping-ponging with (k1, v1). Returns which pair holds
// the result: 0 = (k0, v0) (an even number of passes), 1 = (k1, v1).
static int prim_sort_pairs(fjg_engine* eng, uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1, uint64_t n,
                           int lo, int hi) {
  const int np = prim_sort_passes(lo, hi);
  if (n <= 1 || np == 0) return 0;
  if (np > prims::kRadixMaxPasses) throw fj::EngineError("radix sort: too many key bits");
  if (n >= (1ull << 32) - 16) throw fj::ValidationError("radix sort: at most 2^32-16 pairs");
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(prims::k_radix_pass, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)prims::kRadixSmem));
    attr = true;
  }
  const int db = (hi - lo + np - 1) / np;
  CK(cudaMemsetAsync(eng->prim_hist, 0, (size_t)np * prims::kRadixBins * 4, eng->stream));
  LAUNCH(eng, prims::k_radix_hist<<<grid_for(n / 4 + 1, 256, eng->num_sms * 8), 256, 0, eng->stream>>>(
                  k0, n, lo, db, np, hi, eng->prim_hist));
  const uint64_t tiles = (n + prims::kRadixTile - 1) / prims::kRadixTile;
  auto* st = (unsigned long long*)prim_region(eng, eng->prim_lb_radix, eng->prim_lb_radix_bytes,
                                              tiles * prims::kRadixBins * 8);
  uint32_t *ks = k0, *vs = v0, *kd = k1, *vd = v1;
  for (int p = 0; p < np; ++p) {
    const int shift = lo + p * db;
    const int bits = std::min(db, hi - shift);
    const uint32_t ep = prim_epoch(eng);
    LAUNCH(eng, (prims::k_radix_pass<<<(unsigned)tiles, prims::kRadixThreads, prims::kRadixSmem, eng->stream>>>(
                    ks, vs, kd, vd, n, shift, bits, eng->prim_hist + p * prims::kRadixBins, st, eng->prim_ticket,
                    eng->prim_tbase, ep)));
    eng->prim_tbase += tiles;
    std::swap(ks, kd);
    std::swap(vs, vd);
  }
  return np & 1;
}

struct PhysLevelHost {
  std::vector<int> keycols;
  bool multi = false;
  uint64_t cap = 0;
  uint64_t nsub = 0;  // entries of state/nkeys/cursor (1 at level 0)
  bool dirty = true;
};

struct PhysTrieHost {
  fjg_relation* rel = nullptr;
  std::vector<std::vector<int>> levels;
  std::vector<PhysLevelHost> lev;
  DevTrie dev{};
  bool root_forced = false;
  int map_levels = 0;  // levels that are maps in some sharing atom's GHT schema (SIMPLE / SLT eager builds)
  int key_bits = 32;   // bits used by the root key column (sorted roots: radix-sort end bit)
  uint64_t root_key_bound = 1;  // buckets of the root's slot region (rows; a sorted root: its possible distinct keys)
};

struct AtomInfo {
  int rel_index;
  std::vector<int> vars;  // var ids, column order
  std::vector<std::pair<int, int>> subs;  // (node, position) in node order
  int trie = -1;
};

}  // namespace

struct fjg_query {
  fjg_engine* eng = nullptr;
  fj::FreeJoinPlan plan;
  std::vector<std::string> head;  // variable names, id order
  std::vector<std::string> head_override;
  std::vector<AtomInfo> atoms;
  std::vector<fjg_relation*> rels;
  std::vector<PhysTrieHost> tries;
  std::vector<DevNode> nodes;   // host-side node descriptors
  std::vector<KNode> knodes;    // resolved kernel plans (constant bank)
  DevTrie* d_tries = nullptr;
  DevCounters* d_ctr = nullptr;
  DevCounters* h_ctr = nullptr;  // pinned
  std::vector<void*> bufs;       // pool allocations of this query
  uint64_t cap = 0;              // frontier capacity (candidates per chunk)
  uint64_t max_n = 0;
  uint32_t* tmp_slot = nullptr;
  uint32_t* tmp_rank = nullptr;
  uint32_t* newslots = nullptr;
  uint32_t* newslot_p = nullptr;
  uint32_t* owner_scratch = nullptr;  // force: offset index -> claimed subtrie
  uint8_t* sort_flags = nullptr;      // sorted root force: group-start flags
  int32_t* out_tuples = nullptr;
  uint64_t out_cap = 0;
  uint64_t out_rows = 0;
  // per-execute stats
  uint64_t maps_built = 0, forces = 0, rows_forced = 0;
  // TrieStats per physical trie: subtries forced, levels with a forced map
  uint64_t trie_maps[MAXA] = {};
  uint32_t trie_levels[MAXA] = {};
  void count_maps(int t, int l, uint64_t n) {
    maps_built += n;
    if (t >= 0 && t < MAXA) {
      trie_maps[t] += n;
      if (n) trie_levels[t] |= 1u << l;
    }
  }
  bool dynamic = true;
  uint64_t batch = 0;
  int min_var = -1;
  int width = 16;  // max(#variables, #atoms): selects the register-resident kernel variant
  // memoised chain count (FJG_OUT_FACTORIZED_COUNT over a chain suffix)
  int chain_start = -1;                 // k*, or -1 if the plan has no device-memoisable chain suffix
  std::vector<MemoPass> memo_passes;    // for nodes K-1 .. k* (index j - k*)
  std::vector<unsigned long long*> memo;  // per chain node: 2n u64 (lo, hi)
  std::vector<uint64_t> memo_n;
  std::map<int, uint32_t*> gid;         // per chain trie: group index + 1 of each level-0 position
  std::vector<int> memo_resolve_of;     // pass -> pass whose resolved child / coef arrays it reuses
  std::map<int, uint32_t*> memo_dense;  // per sorted chain root: dense key -> group map (size 2^key_bits)
  KNode memo_top{};                     // node k*-1 aggregating mult * memo[child]
  int stop_node = -1;
  int gj_x[MAXN];  // per node: the GJ fast-path variable, or -1
  int gj_w[MAXN];  // per node: the GJ frontier-writing fast-path variable, or -1
  bool sw[MAXN];   // per node: the stream-cover frontier-writing fast path applies
  SProbe sprobe[MAXN];  // per node: probe plan of the single-binding stream kernel (np = 0: n/a)
  int dev_tail_node = -1;  // a tail launched with its frontier size on the device (inputs counted there)
  std::vector<TailPlan> tails;  // per node: fused Cartesian tail from this node on (ntail = 0: n/a)
  uint64_t* bounds = nullptr;  // tile -> first entry (load-balanced search)
  uint64_t bounds_cap = 0;
  uint32_t* chunk_owner = nullptr;  // chunk -> owning entry (GJ last node)
  // GJ last node in probe-region order (FJG_GJ_SORT): keys, binding permutation, permuted m / scan
  uint32_t *sort_keys = nullptr, *sort_keys2 = nullptr, *sort_vals = nullptr, *perm = nullptr;
  uint64_t *m_perm = nullptr, *scan_perm = nullptr;
  uint64_t sort_cap = 0;
  int backend = FJG_BACKEND_COLT;
  // non-blocking phase timer: event pairs resolved after the final sync
  std::vector<cudaEvent_t> events;
  std::vector<std::pair<int, int>> marks;  // (event index, phase) ; phase<0 = start
  size_t ev_used = 0;
  double phase_ms[5] = {0, 0, 0, 0, 0};  // 0 force (build), 1 node kernels, 2 last node, 3 node 0 (not last), 4 memo
  uint64_t memo_rows[3] = {0, 0, 0};     // rows resolved / gathered / initialised by the memo passes
  double build_ms = 0, join_ms = 0, last_ms = 0, first_ms = 0;
  uint64_t last_launches = 0, last_candidates = 0;
  uint64_t node_inputs[MAXN] = {0};
  bool timing = false;
  void mark(cudaStream_t st, int tag) {
    if (!timing) return;
    if (ev_used == events.size()) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) throw fj::ResourceError("cudaEventCreate failed");
      events.push_back(e);
    }
    if (cudaEventRecord(events[ev_used], st) != cudaSuccess) throw fj::EngineError("cudaEventRecord failed");
    marks.emplace_back((int)ev_used, tag);
    ++ev_used;
  }
  void resolve_marks() {
    // marks come in (start, end) pairs: tag = -1 start, tag >= 0 end of phase tag
    for (size_t i = 0; i + 1 < marks.size(); i += 2) {
      float ms = 0;
      cudaEventElapsedTime(&ms, events[marks[i].first], events[marks[i + 1].first]);
      phase_ms[marks[i + 1].second] += ms;
    }
    marks.clear();
    ev_used = 0;
  }

  void* alloc(size_t bytes) {
    void* p = eng->pool->alloc(bytes);
    bufs.push_back(p);
    return p;
  }
  ~fjg_query() {
    if (eng) {
      for (void* p : bufs) eng->pool->free(p);
      for (auto e : events) cudaEventDestroy(e);
    }
  }
};

// ============================================================================
// query preparation
// ============================================================================
static bool root_sorted_path(const fjg_query* q, int t);  // (defined with the root force below)
static void prepare_query(fjg_query* q) {
  using fj::EngineError;
  using fj::ValidationError;
  const auto& plan = q->plan;
  const size_t A = plan.query.size();
  if (A > (size_t)MAXA) throw ValidationError("too many atoms for the device executor (max 16)");
  if (plan.nodes.size() > (size_t)MAXN) throw ValidationError("too many plan nodes (max 32)");
  q->head = fj::head_variables(plan.query);
  if (!q->head_override.empty()) {  // explicit head order (e.g. the original query's, for bushy segments)
    std::vector<std::string> a = q->head, b = q->head_override;
    std::sort(a.begin(), a.end());
    std::sort(b.begin(), b.end());
    if (a != b) throw ValidationError("\"head\" must list every query variable exactly once");
    q->head = q->head_override;
  }
  q->width = (int)std::max(q->head.size(), A);
  if (q->head.size() > (size_t)MAXV) throw ValidationError("too many variables (max 16)");
  std::map<std::string, int> vid;
  for (size_t i = 0; i < q->head.size(); ++i) vid[q->head[i]] = (int)i;
  std::map<std::string, int> aid;
  q->atoms.resize(A);
  for (size_t a = 0; a < A; ++a) {
    aid[plan.query[a].relation] = (int)a;
    for (auto& x : plan.query[a].vars) q->atoms[a].vars.push_back(vid[x]);
    if (q->atoms[a].vars.empty()) throw ValidationError("nullary atoms are not supported on the device");
    if ((int)q->atoms[a].vars.size() != q->rels[a]->ncols)
      throw ValidationError("atom " + plan.query[a].relation + " has " + std::to_string(q->atoms[a].vars.size()) +
                            " variables but its relation has " + std::to_string(q->rels[a]->ncols) + " columns");
    if (q->rels[a]->ncols > MAXC) throw ValidationError("too many columns (max 8)");
    if (q->rels[a]->nrows >= 0xFFFFFFF0ull) throw ValidationError("relation too large (rows must be < 2^32-16)");
  }
  for (size_t k = 0; k < plan.nodes.size(); ++k) {
    const auto& subs = plan.nodes[k].subatoms;
    if (subs.size() > (size_t)MAXS) throw ValidationError("too many subatoms in a node (max 12)");
    for (size_t i = 0; i < subs.size(); ++i) {
      auto it = aid.find(subs[i].relation);
      if (it == aid.end()) throw ValidationError("plan references unknown relation " + subs[i].relation);
      if (subs[i].vars.size() > (size_t)MAXK) throw ValidationError("subatom arity above 6");
      q->atoms[it->second].subs.emplace_back((int)k, (int)i);
    }
  }
  // column index of a variable within atom a
  auto col_of = [&](int a, const std::string& x) {
    const auto& vars = plan.query[a].vars;
    for (size_t c = 0; c < vars.size(); ++c)
      if (vars[c] == x) return (int)c;
    throw EngineError("variable " + x + " not in atom");
  };
  // physical tries (share identical or prefix-equal level key columns)
  for (size_t a = 0; a < A; ++a) {
    std::vector<std::vector<int>> levels;
    for (auto& [k, i] : q->atoms[a].subs) {
      std::vector<int> cols;
      for (auto& x : plan.nodes[k].subatoms[i].vars) cols.push_back(col_of((int)a, x));
      levels.push_back(cols);
    }
    int found = -1;
    for (size_t t = 0; t < q->tries.size(); ++t) {
      auto& T = q->tries[t];
      if (T.rel != q->rels[a]) continue;
      size_t m = std::min(T.levels.size(), levels.size());
      if (std::equal(levels.begin(), levels.begin() + m, T.levels.begin())) {
        if (levels.size() > T.levels.size()) T.levels = levels;
        found = (int)t;
        break;
      }
    }
    if (found < 0) {
      if (q->tries.size() >= (size_t)MAXT) throw ValidationError("too many physical tries");
      PhysTrieHost T;
      T.rel = q->rels[a];
      T.levels = levels;
      q->tries.push_back(T);
      found = (int)q->tries.size() - 1;
    }
    q->atoms[a].trie = found;
    // derive_ght_schemas (fj_plan.cpp): every level is a map unless the atom's
    // last subatom is its node's cover (then that level stays an offset vector)
    const bool last_is_cover = !q->atoms[a].subs.empty() && q->atoms[a].subs.back().second == 0;
    const int ml = (int)levels.size() - (last_is_cover ? 1 : 0);
    q->tries[found].map_levels = std::max(q->tries[found].map_levels, ml);
  }
  // Roots forced by radix sort sort only the bits their key column uses (its
  // largest value as uint32; negative keys use all 32): one reduction per such
  // trie here, at query creation, instead of a fourth sort pass per execution.
  // The same bound sizes the root's slot region: a sorted root keeps one bucket
  // per distinct key, and there are at most min(rows, largest key + 1) of them
  // (C5: 2^27 buckets = 4.3 GB instead of 17 GB for the 512M-row relation).
  {
    std::vector<int> sorted;
    for (size_t t = 0; t < q->tries.size(); ++t) {
      auto& T = q->tries[t];
      T.root_key_bound = std::max<uint64_t>(T.rel->nrows, 1);
      if (T.levels[0].empty() && root_sorted_path(q, (int)t)) T.root_key_bound = 1;
      if (T.levels[0].size() == 1 && T.rel->nrows >= (1u << 21)) sorted.push_back((int)t);
    }
    if (!sorted.empty()) {
      fjg_engine* eng = q->eng;
      uint32_t* dmax = (uint32_t*)eng->pool->alloc(sorted.size() * 4);
      for (size_t i = 0; i < sorted.size(); ++i) {
        auto& T = q->tries[sorted[i]];
        const uint32_t* col = reinterpret_cast<const uint32_t*>(T.rel->cols[T.levels[0][0]]);
        prim_max_u32(eng, col, T.rel->nrows, dmax + i);
      }
      std::vector<uint32_t> hmax(sorted.size());
      CK(cudaMemcpyAsync(hmax.data(), dmax, sorted.size() * 4, cudaMemcpyDeviceToHost, eng->stream));
      CK(cudaStreamSynchronize(eng->stream));
      for (size_t i = 0; i < sorted.size(); ++i) {
        auto& T = q->tries[sorted[i]];
        int bits = 1;
        while (bits < 32 && (hmax[i] >> bits)) ++bits;
        T.key_bits = bits;
        if (root_sorted_path(q, sorted[i]))
          T.root_key_bound = std::min<uint64_t>(T.root_key_bound, (uint64_t)hmax[i] + 1);
      }
      eng->pool->free(dmax);
    }
  }
  // allocate trie storage
  for (size_t t = 0; t < q->tries.size(); ++t) {
    auto& T = q->tries[t];
    const uint64_t n = T.rel->nrows;
    q->max_n = std::max(q->max_n, n);
    if (T.levels.size() > (size_t)MAXL) throw ValidationError("too many trie levels (max 8)");
    DevTrie& D = T.dev;
    memset(&D, 0, sizeof(D));
    D.n = (uint32_t)n;
    D.ncols = T.rel->ncols;
    D.nlev = (int)T.levels.size();
    for (int c = 0; c < T.rel->ncols; ++c) D.base[c] = T.rel->cols[c];
    T.lev.resize(T.levels.size());
    for (size_t l = 0; l < T.levels.size(); ++l) {
      auto& H = T.lev[l];
      DevLevel& L = D.lev[l];
      H.keycols = T.levels[l];
      H.multi = H.keycols.size() >= 2;
      H.nsub = l == 0 ? 1 : std::max<uint64_t>(n, 1);
      // FJG_RS 4-slot buckets per position (per-subtrie regions); a sorted root: per possible distinct key
      H.cap = 4ull * FJG_RS * (l == 0 ? T.root_key_bound : std::max<uint64_t>(n, 1));
      L.table = (Slot*)q->alloc(H.cap * sizeof(Slot));
      L.srep = H.multi ? (uint32_t*)q->alloc(H.cap * 4) : nullptr;
      L.sn = (SubState*)q->alloc(H.nsub * sizeof(SubState));
      L.cursor = (uint32_t*)q->alloc(H.nsub * 4);
      L.cnt = (uint32_t*)q->alloc(std::max<uint64_t>(n, 1) * 4);
      std::set<int> cols;
      for (size_t l2 = l; l2 < T.levels.size(); ++l2) cols.insert(T.levels[l2].begin(), T.levels[l2].end());
      for (int c : cols) L.cval[c] = (int32_t*)q->alloc(std::max<uint64_t>(n, 1) * 4);
      L.nk = (int)H.keycols.size();
      for (int i = 0; i < L.nk; ++i) L.keycol[i] = H.keycols[i];
      if (l > 0) {
        // claim lists: one entry per subtrie of this level at most; level 1's
        // subtries are the root's child groups (a sorted root: its key bound)
        const uint64_t nl = l == 1 ? std::min<uint64_t>(std::max<uint64_t>(n, 1), T.root_key_bound) : std::max<uint64_t>(n, 1);
        L.list_p = (uint32_t*)q->alloc(nl * 4);
        L.list_len = (uint32_t*)q->alloc(nl * 4);
        L.list_scan = (uint32_t*)q->alloc(nl * 4);
      }
    }
  }
  q->tmp_slot = (uint32_t*)q->alloc(std::max<uint64_t>(q->max_n, 1) * 4);
  q->tmp_rank = (uint32_t*)q->alloc(std::max<uint64_t>(q->max_n, 1) * 4);
  q->newslots = (uint32_t*)q->alloc(std::max<uint64_t>(q->max_n, 1) * 4);
  q->newslot_p = (uint32_t*)q->alloc(std::max<uint64_t>(q->max_n, 1) * 4);
  q->owner_scratch = (uint32_t*)q->alloc(std::max<uint64_t>(q->max_n, 1) * 4);
  q->sort_flags = (uint8_t*)q->alloc(std::max<uint64_t>(q->max_n, 1));
  // slot indices (4 * FJG_RS per row) are 32-bit in the force scratch
  if (q->max_n >= (1ull << 31) || q->max_n > (1ull << 32) / (4 * FJG_RS))
    throw ValidationError("relations must have at most " + std::to_string((1ull << 32) / (4 * FJG_RS)) + " rows");
  // static node descriptors
  const size_t K = plan.nodes.size();
  q->nodes.assign(K, DevNode{});
  std::vector<uint32_t> bound_before(K + 1, 0);
  for (size_t k = 0; k < K; ++k) {
    uint32_t m = bound_before[k];
    for (auto& s : plan.nodes[k].subatoms)
      for (auto& x : s.vars) m |= 1u << vid[x];
    bound_before[k + 1] = m;
  }
  for (size_t k = 0; k < K; ++k) {
    DevNode& N = q->nodes[k];
    memset(&N, 0, sizeof(N));
    N.k = (int)k;
    const auto& subs = plan.nodes[k].subatoms;
    N.nsub = (int)subs.size();
    N.is_last = k + 1 == K;
    N.nhead = (int)q->head.size();
    N.in_vars = bound_before[k];
    N.out_vars = bound_before[k + 1];
    auto cov = fj::covers(plan, k);
    if (cov.empty()) throw ValidationError("node " + std::to_string(k) + " has no cover");
    N.ncov = (int)cov.size();
    for (size_t c = 0; c < cov.size(); ++c) N.cov[c] = (int)cov[c];
    for (size_t a = 0; a < A; ++a) {
      const auto& S = q->atoms[a].subs;
      const bool before = !S.empty() && S.front().first < (int)k;
      const bool at_or_after = !S.empty() && S.back().first >= (int)k;
      const bool after = !S.empty() && S.back().first > (int)k;
      const bool upto = !S.empty() && S.front().first <= (int)k;
      if (before && at_or_after) N.in_atoms |= 1u << a;
      if (upto && after) N.out_atoms |= 1u << a;
      N.atom_n[a] = (uint32_t)q->rels[a]->nrows;
    }
    for (size_t i = 0; i < subs.size(); ++i) {
      DevSub& D = N.sub[i];
      const int a = aid[subs[i].relation];
      D.atom = a;
      D.trie = q->atoms[a].trie;
      const auto& S = q->atoms[a].subs;
      int depth = 0;
      while (!(S[depth].first == (int)k && S[depth].second == (int)i)) ++depth;
      D.depth = depth;
      D.last = depth + 1 == (int)S.size();
      D.nv = (int)subs[i].vars.size();
      for (int t = 0; t < D.nv; ++t) {
        D.var[t] = vid[subs[i].vars[t]];
        D.col[t] = col_of(a, subs[i].vars[t]);
        if ((N.in_vars >> D.var[t]) & 1u) D.bound_mask |= 1 << t;
      }
      bool later_vars = false;
      for (size_t d = depth + 1; d < S.size(); ++d)
        if (!plan.nodes[S[d].first].subatoms[S[d].second].vars.empty()) later_vars = true;
      D.stream = !later_vars;
    }
  }
  q->d_tries = (DevTrie*)q->alloc(q->tries.size() * sizeof(DevTrie));
  q->d_ctr = (DevCounters*)q->alloc(sizeof(DevCounters));
  q->h_ctr = q->eng->h_ctr;
  std::vector<DevTrie> dt;
  for (auto& T : q->tries) dt.push_back(T.dev);
  CK(cudaMemcpyAsync(q->d_tries, dt.data(), dt.size() * sizeof(DevTrie), cudaMemcpyHostToDevice, q->eng->stream));
}

// Resolve each node's descriptor into the constant-bank kernel plan.
static int gj_last_var(const KNode& G, const DevNode& N);
static int gj_write_var(const DevNode& N, int width);
static bool stream_write_ok(const DevNode& N, const KNode& G);

// Probe plan of k_stream_one: probe j = the j-th non-cover subatom in node
// order, keyed on the cover column binding its variable. Needs distinct cover
// variables and at most four probes (else np = 0: the generic stream kernel).
static SProbe stream_probe_plan(const DevNode& N, bool sw) {
  SProbe P;
  memset(&P, 0, sizeof(P));
  if (!sw || N.nsub - 1 > 4) return P;
  const DevSub& C = N.sub[N.cov[0]];
  for (int a = 0; a < C.nv; ++a)
    for (int b = a + 1; b < C.nv; ++b)
      if (C.var[a] == C.var[b]) return P;
  int np = 0;
  for (int s = 0; s < N.nsub; ++s) {
    if (s == N.cov[0]) continue;
    int kc = -1;
    for (int t = 0; t < C.nv; ++t)
      if (C.var[t] == N.sub[s].var[0]) kc = t;
    if (kc < 0) return SProbe{};
    P.s[np] = (int8_t)s;
    P.kc[np] = (int8_t)kc;
    ++np;
  }
  P.np = np;
  return P;
}

// Fused Cartesian tail from node k (k_tail): every node k..K-1 has exactly one
// subatom, a stream-iterated cover of fresh variables (SPEC.md:423-431's pure
// Cartesian suffix), over distinct atoms whose subtrie at node k is in its
// frontier or is the root.
static TailPlan tail_plan(const fjg_query* q, int k) {
  TailPlan T;
  memset(&T, 0, sizeof(T));
  const int K = (int)q->nodes.size();
  if (K - k > MAXTAIL || q->width > 16) return T;
  const DevNode& Nk = q->nodes[k];
  uint32_t seen = 0;
  for (int j = k; j < K; ++j) {
    const DevNode& N = q->nodes[j];
    if (N.nsub != 1 || N.ncov != 1) return TailPlan{};
    const DevSub& D = N.sub[0];
    if (!D.stream || D.bound_mask || !D.last || ((seen >> D.atom) & 1u)) return TailPlan{};
    seen |= 1u << D.atom;
    const int t = j - k;
    T.node[t] = j;
    T.open[t] = (Nk.in_atoms >> D.atom) & 1u;
    if (!T.open[t] && D.depth != 0) return TailPlan{};
    T.in_p[t] = T.open[t] ? Nk.in.p[D.atom] : nullptr;
    T.in_len[t] = T.open[t] ? Nk.in.len[D.atom] : nullptr;
    T.sub[t] = q->knodes[j].sub[0];
  }
  T.ntail = K - k;
  return T;
}

static void build_knodes(fjg_query* q) {
  const size_t K = q->nodes.size();
  q->knodes.assign(K, KNode{});
  for (size_t k = 0; k < K; ++k) {
    const DevNode& N = q->nodes[k];
    KNode& G = q->knodes[k];
    memset(&G, 0, sizeof(G));
    G.k = N.k;
    G.nsub = N.nsub;
    G.ncov = N.ncov;
    G.nhead = N.nhead;
    G.is_last = N.is_last;
    for (int c = 0; c < N.ncov; ++c) G.cov[c] = (int8_t)N.cov[c];
    G.in_vars = N.in_vars;
    G.out_vars = N.out_vars;
    G.in_atoms = N.in_atoms;
    G.out_atoms = N.out_atoms;
    for (int v = 0; v < MAXV; ++v) {
      G.in_var[v] = N.in.var[v];
      G.out_var[v] = N.out.var[v];
    }
    for (int a = 0; a < MAXA; ++a) {
      G.in_p[a] = N.in.p[a];
      G.in_len[a] = N.in.len[a];
      G.out_p[a] = N.out.p[a];
      G.out_len[a] = N.out.len[a];
    }
    G.in_mult = N.in.mult;
    G.out_mult = N.out.mult;
    G.chosen = N.chosen;
    G.m = N.m;
    G.scan = N.scan;
    for (int i = 0; i < N.nsub; ++i) {
      const DevSub& D = N.sub[i];
      KSub& S = G.sub[i];
      const DevTrie& T = q->tries[D.trie].dev;
      const DevLevel& L = T.lev[D.depth];
      for (int t = 0; t < D.nv; ++t) {
        S.src[t] = D.stream ? (D.depth == 0 ? T.base[D.col[t]] : T.lev[D.depth - 1].cval[D.col[t]])
                            : L.cval[D.col[t]];
        S.kcmp[t] = L.cval[D.col[t]];
        S.var[t] = (int8_t)D.var[t];
      }
      S.cnt = L.cnt;
      S.table = L.table;
      S.sn = L.sn;
      const bool open = (N.in_atoms >> D.atom) & 1u;
      S.in_p = open ? N.in.p[D.atom] : nullptr;
      S.in_len = open ? N.in.len[D.atom] : nullptr;
      S.root_n = N.atom_n[D.atom];
      S.rregion = q->d_ctr->root_region + D.trie;
      S.ldup = q->d_ctr->level_dup + D.trie * MAXL + D.depth;
      S.nv = (uint8_t)D.nv;
      S.bound_mask = (uint8_t)D.bound_mask;
      S.stream = (uint8_t)D.stream;
      S.last = (uint8_t)D.last;
      S.atom = (uint8_t)D.atom;
      S.trie = (uint8_t)D.trie;
      S.depth = (uint8_t)D.depth;
    }
  }
  for (size_t k = 0; k < K && k < (size_t)MAXN; ++k) {
    q->gj_x[k] = gj_last_var(q->knodes[k], q->nodes[k]);
    q->gj_w[k] = gj_write_var(q->nodes[k], q->width);
    q->sw[k] = stream_write_ok(q->nodes[k], q->knodes[k]);
    q->sprobe[k] = stream_probe_plan(q->nodes[k], q->sw[k]);
  }
  q->tails.assign(K, TailPlan{});
  for (size_t k = 0; k < K; ++k) q->tails[k] = tail_plan(q, (int)k);
}

// Chain-suffix analysis for the memoised factorised count (mirrors the
// oracle's Exec::chain_node_ok). Device-specific extra
// condition: the carrier's subatom at node j is its second one (depth 1), so
// the memo is indexed by level-0 groups, which forcing the root builds whole.
static bool device_chain_node(const fjg_query* q, int j, int& carrier, std::vector<int>& fresh, int& next) {
  const auto& plan = q->plan;
  const DevNode& N = q->nodes[j];
  const int A = (int)q->atoms.size();
  carrier = -1;
  next = -1;
  fresh.clear();
  int catom = -1;
  for (int a = 0; a < A; ++a) {
    const auto& S = q->atoms[a].subs;
    if (S.front().first < j && S.back().first >= j) {
      if (catom >= 0) return false;
      catom = a;
    }
  }
  if (catom < 0) return false;
  uint32_t cvars = 0;
  for (int i = 0; i < N.nsub; ++i)
    if (N.sub[i].atom == catom) {
      if (carrier >= 0 || !N.sub[i].last || N.sub[i].depth != 1) return false;
      carrier = i;
      for (int t = 0; t < N.sub[i].nv; ++t) cvars |= 1u << N.sub[i].var[t];
    }
  if (carrier < 0 || (cvars & N.in_vars)) return false;
  for (int i = 0; i < N.nsub; ++i) {
    if (i == carrier) continue;
    const DevSub& X = N.sub[i];
    if (X.depth != 0) return false;
    for (int t = 0; t < X.nv; ++t)
      if (!((cvars >> X.var[t]) & 1u)) return false;
    if (!X.last) {
      if (next >= 0) return false;
      next = i;
    }
    fresh.push_back(i);
  }
  for (size_t i = j; i < plan.nodes.size(); ++i)
    for (int t = 0; t < q->nodes[i].nsub; ++t)
      for (int u = 0; u < q->nodes[i].sub[t].nv; ++u)
        if ((N.in_vars >> q->nodes[i].sub[t].var[u]) & 1u) return false;
  return (next >= 0) == (j + 1 < (int)plan.nodes.size());
}

static void prepare_chain(fjg_query* q) {
  const int K = (int)q->nodes.size();
  int start = -1;
  std::vector<MemoPass> passes;
  for (int j = K - 1; j >= 1; --j) {
    int carrier, next;
    std::vector<int> fresh;
    if (!device_chain_node(q, j, carrier, fresh, next)) break;
    // the node before the chain must hand over the carrier's level-0 child
    MemoPass M{};
    const KNode& G = q->knodes[j];
    const KSub& C = G.sub[carrier];
    M.n = q->tries[C.trie].dev.n;
    M.cnv = C.nv;
    for (int t = 0; t < C.nv; ++t) M.cvals[t] = C.src[t];
    M.nfresh = (int)fresh.size();
    for (int x = 0; x < M.nfresh; ++x) {
      const KSub& X = G.sub[fresh[x]];
      M.fresh[x] = X;
      M.cont[x] = fresh[x] == next ? 1 : 0;
      for (int t = 0; t < X.nv; ++t) {
        int at = 0;
        while (C.var[at] != X.var[t]) ++at;
        M.cpos[x][t] = (int8_t)at;
      }
    }
    passes.insert(passes.begin(), M);
    start = j;
  }
  if (start < 1) return;
  q->chain_start = start;
  q->memo_passes = passes;
  q->memo.resize(passes.size());
  q->memo_n.resize(passes.size());
  auto gid_of = [&](int trie) {
    if (!q->gid.count(trie))
      q->gid[trie] = (uint32_t*)q->alloc(std::max<uint64_t>(q->tries[trie].dev.n, 1) * 4);
    return q->gid[trie];
  };
  std::vector<std::string> sig(passes.size());
  q->memo_resolve_of.assign(passes.size(), -1);
  // passes run from the last chain node down: the first to run resolves
  for (int i = (int)passes.size() - 1; i >= 0; --i) {
    const int j = start + i;
    int cidx, nx0;
    std::vector<int> fr0;
    device_chain_node(q, j, cidx, fr0, nx0);
    const KSub& C = q->knodes[j].sub[cidx];
    MemoPass& M = q->memo_passes[i];
    q->memo_n[i] = M.n;
    q->memo[i] = (unsigned long long*)q->alloc(std::max<uint64_t>(M.n, 1) * 16);
    M.gid = gid_of(C.trie);
    M.cnt = q->tries[C.trie].dev.lev[0].cnt;
    M.memo_out = q->memo[i];
    M.cont_x = -1;
    M.has_coef = 0;
    // rows resolve to the same children in every pass with the same carrier
    // column(s) and fresh atoms (the C5 5-path: E2..E5 are one physical trie)
    std::string sg = std::to_string(C.trie);
    for (int t = 0; t < M.cnv; ++t) sg += ":" + std::to_string((uintptr_t)M.cvals[t]);
    for (int x = 0; x < M.nfresh; ++x) {
      const KSub& X = M.fresh[x];
      if (M.cont[x]) {
        M.cont_x = x;
        M.gid_next = gid_of(X.trie);
      } else {
        M.has_coef = 1;
      }
      sg += "|" + std::to_string((uintptr_t)X.table) + "," + std::to_string(X.nv) + "," + std::to_string(M.cont[x]);
      for (int t = 0; t < X.nv; ++t) sg += "," + std::to_string(M.cpos[x][t]);
    }
    sig[i] = sg;
    for (int k = (int)passes.size() - 1; k > i; --k)
      if (sig[k] == sg && q->memo_resolve_of[k] < 0 && q->memo_passes[k].nfresh > 0) {
        q->memo_resolve_of[i] = k;
        M.child = q->memo_passes[k].child;
        M.coef = q->memo_passes[k].coef;
        break;
      }
    if (q->memo_resolve_of[i] < 0 && M.nfresh > 0) {
      if (M.cont_x >= 0) M.child = (uint32_t*)q->alloc(std::max<uint64_t>(M.n, 1) * 4);
      if (M.has_coef) M.coef = (uint64_t*)q->alloc(std::max<uint64_t>(M.n, 1) * 8);
      // the continuing atom's root is sorted on small non-negative keys: a dense
      // key -> group map replaces the probe and the group-id read (one read/row)
      if (M.cont_x == 0 && M.nfresh == 1 && M.fresh[0].nv == 1) {
        const int ft = M.fresh[0].trie;
        const auto& FT = q->tries[ft];
        const uint64_t dn = 1ull << std::min(FT.key_bits, 31);
        if (FT.levels[0].size() == 1 && FT.rel->nrows >= (1u << 21) && FT.key_bits <= 30 &&
            dn <= 8 * std::max<uint64_t>(FT.rel->nrows, 1)) {
          if (!q->memo_dense.count(ft)) q->memo_dense[ft] = (uint32_t*)q->alloc(dn * 4);
          M.direct = q->memo_dense[ft];
          M.direct_n = (uint32_t)dn;
        }
      }
    }
  }
  for (size_t i = 0; i + 1 < passes.size(); ++i) q->memo_passes[i].memo_next = q->memo[i + 1];
  // the aggregating top node
  int c, nx;
  std::vector<int> fr;
  device_chain_node(q, start, c, fr, nx);
  q->memo_top = q->knodes[start - 1];
  q->memo_top.memo = q->memo[0];
  q->memo_top.memo_atom = q->knodes[start].sub[c].atom;
  q->memo_top.memo_gid = q->memo_passes[0].gid;
}

// Bytes ensure_frontiers allocates per unit of capacity (all nodes).
static uint64_t frontier_entry_bytes(const fjg_query* q) {
  uint64_t b = 0;
  const size_t K = q->nodes.size();
  for (size_t k = 0; k < K; ++k) {
    const DevNode& N = q->nodes[k];
    if (k > 0) b += 1 + 8 + 8;  // chosen, m, scan
    if (k + 1 < K) b += 4ull * __builtin_popcount(N.out_vars) + 8ull * __builtin_popcount(N.out_atoms) + 8;
  }
  return b;
}

// (Re)allocate per-node frontier buffers for a candidate capacity `cap`.
static void ensure_frontiers(fjg_query* q, uint64_t cap) {
  if (q->cap >= cap && q->cap) return;
  const size_t K = q->nodes.size();
  for (size_t k = 0; k < K; ++k) {
    DevNode& N = q->nodes[k];
    const uint64_t fin = k == 0 ? 1 : cap;  // entries entering node k
    N.chosen = (uint8_t*)q->alloc(fin);
    N.m = (uint64_t*)q->alloc(fin * 8);
    N.scan = (uint64_t*)q->alloc(fin * 8);
    if (k + 1 < K) {
      DevFrontier& O = N.out;
      memset(&O, 0, sizeof(O));
      for (int v = 0; v < MAXV; ++v)
        if ((N.out_vars >> v) & 1u) O.var[v] = (int32_t*)q->alloc(cap * 4);
      for (int a = 0; a < MAXA; ++a)
        if ((N.out_atoms >> a) & 1u) {
          O.p[a] = (uint32_t*)q->alloc(cap * 4);
          O.len[a] = (uint32_t*)q->alloc(cap * 4);
        }
      O.mult = (uint64_t*)q->alloc(cap * 8);
      q->nodes[k + 1].in = O;
    }
  }
  q->cap = cap;
  const uint64_t nb = std::max<uint64_t>(cap, kLastChunk) / TILE + 2;
  if (nb > q->bounds_cap) {
    q->bounds = (uint64_t*)q->alloc(nb * 8);
    q->chunk_owner = (uint32_t*)q->alloc((std::max<uint64_t>(cap, kLastChunk) / 32 + 2) * 4);
    q->bounds_cap = nb;
  }
  build_knodes(q);
  if (q->chain_start < 0 && q->memo_passes.empty()) prepare_chain(q);
  else if (q->chain_start >= 1) {  // frontier pointers moved: refresh the top node
    const int c = q->memo_top.memo_atom;
    q->memo_top = q->knodes[q->chain_start - 1];
    q->memo_top.memo = q->memo[0];
    q->memo_top.memo_atom = c;
    q->memo_top.memo_gid = q->memo_passes[0].gid;
  }
}

static void sync_counters(fjg_query* q) {
  CK(cudaMemcpyAsync(q->h_ctr, q->d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, q->eng->stream));
  CK(cudaStreamSynchronize(q->eng->stream));
  ++q->eng->syncs;
}

// Force the listed subtries of (trie t, level l): Fig 12 `force` in batch.
#ifndef FJG_SORTED_ROOT
#define FJG_SORTED_ROOT 1
#endif
#ifndef FJG_SORTED_ROOT_MIN_LOG
#define FJG_SORTED_ROOT_MIN_LOG 21  // roots of >= 2^21 rows are forced by sorting, smaller ones by CAS inserts
#endif
// Sort-based root force (arity <= 1 keys): see kernels/force.cuh.
static void force_root_sorted(fjg_query* q, int t) {
  fjg_engine* eng = q->eng;
  auto& T = q->tries[t];
  const uint32_t n = (uint32_t)T.rel->nrows;
  q->mark(eng->stream, -1);
  ForceRange R{};
  R.single = 1;
  R.p0 = 0;
  R.len0 = n;
  const unsigned g = grid_for(n, 256, eng->num_sms * 16);
  uint32_t *keys = q->tmp_slot, *rows = q->tmp_rank, *skeys = q->newslots, *srows = q->newslot_p;
  uint32_t* starts = q->owner_scratch;
  uint8_t* flags = q->sort_flags;
  uint32_t* ng = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(q->d_ctr) + offsetof(DevCounters, survivors));
  // two columns, one key column, both clustered at level 0: sort (key, other
  // column) straight into the clustered columns (stable: the row order the
  // (key, row) sort + gather would give), no gather pass
  const DevLevel& L0 = T.dev.lev[0];
  int pay = -1;
  if (T.dev.ncols == 2 && T.levels[0].size() == 1) {
    const int kc = L0.keycol[0], oc = 1 - kc;
    if (L0.cval[kc] && L0.cval[oc]) {
      pay = oc;
      skeys = reinterpret_cast<uint32_t*>(L0.cval[kc]);
      srows = reinterpret_cast<uint32_t*>(L0.cval[oc]);
    }
  }
  // hand-written LSD radix sort (kernels/prims.cuh) over the key bits the column
  // uses; the pair the keys start in is chosen so the last pass lands in
  // (skeys, srows)
  const int kb = T.levels[0].empty() ? 1 : T.key_bits;
  const bool even = n <= 1 || prim_sort_passes(0, kb) % 2 == 0;
  uint32_t* k0 = even ? skeys : keys;
  uint32_t* v0 = even ? srows : rows;
  LAUNCH(eng, k_root_keys<<<g, 256, 0, eng->stream>>>(q->d_tries, t, n, k0, v0, pay));
  prim_sort_pairs(eng, k0, v0, even ? keys : skeys, even ? rows : srows, n, 0, kb);
  LAUNCH(eng, k_root_starts<<<g, 256, 0, eng->stream>>>(skeys, n, flags));
  prim_select_flagged(eng, flags, starts, n, ng);
  // the root's slot region shrinks to one bucket per distinct key (load <= 0.25)
  LAUNCH(eng, k_root_clear<<<g, 256, 0, eng->stream>>>(q->d_tries, t, n, ng, q->d_ctr));
  LAUNCH(eng, k_root_insert<<<g, 256, 0, eng->stream>>>(q->d_tries, t, n, skeys, starts, ng, q->d_ctr));
  if (pay < 0) LAUNCH(eng, k_root_gather<<<g, 256, 0, eng->stream>>>(q->d_tries, t, n, srows));
  q->mark(eng->stream, 0);
  q->forces += 1;
  q->count_maps(t, 0, 1);
  q->rows_forced += n;
  T.lev[0].dirty = true;
}

// Chunk owners for [c0, c1) at `chunk` candidates per chunk (k_chunk_marks + max-scan).
static void chunk_owners(fjg_query* q, const uint64_t* scan, uint64_t F, uint64_t c0, uint64_t c1, uint32_t chunk) {
  fjg_engine* eng = q->eng;
  if (chunk == 0 || (chunk & (chunk - 1))) throw fj::EngineError("chunk_owners: chunk must be a nonzero power of two");
  if (c1 < c0 || c1 - c0 > kLastChunk)
    throw fj::EngineError("chunk_owners: launch range exceeds " + std::to_string(kLastChunk) + " candidates");
  const uint64_t n = (c1 - c0 + chunk - 1) / chunk + 1;
  CK(cudaMemsetAsync(q->chunk_owner, 0, n * 4, eng->stream));
  LAUNCH(eng, k_chunk_marks<<<grid_for(std::min<uint64_t>(F, (c1 - c0 + chunk - 1) / chunk + 1)), 256, 0,
                              eng->stream>>>(scan, F, c0, c1, chunk, q->chunk_owner));
  prim_scan<prims::OpMax, false>(eng, q->chunk_owner, q->chunk_owner, n);
}

// Launch a force batch (clear -> insert -> assign -> scatter, blockIdx.y =
// member); `upper` bounds every member's offset count, `single` says the
// members are whole subtries (roots), `multi` the key arity >= 2 path.
static void launch_force_batch(fjg_query* q, const ForceBatch& B, uint64_t upper, bool single, bool multi) {
  fjg_engine* eng = q->eng;
  q->mark(eng->stream, -1);
  const dim3 g(grid_for(upper, 256, std::max(1, eng->num_sms * 16 / B.n)), B.n);
  const dim3 ga(grid_for(upper, 256, std::max(1, eng->num_sms * 8 / B.n)), B.n);
  // (k_force_clear also resets each member's counters and a root's cursor / key count)
  const int opt_ok = (FJG_FORCE_OPT && !single && !multi) ? 1 : 0;
  LAUNCH(eng, k_force_clear<<<g, 256, 0, eng->stream>>>(q->d_tries, B, q->d_ctr, 0, opt_ok));
  if (multi)
    LAUNCH(eng, (k_force_insert<true, false><<<g, 256, 0, eng->stream>>>(q->d_tries, B, q->tmp_slot, q->tmp_rank,
                                                                         q->d_ctr, 0)));
  else if (opt_ok)
    LAUNCH(eng, (k_force_insert<false, true><<<g, 256, 0, eng->stream>>>(q->d_tries, B, q->tmp_slot, q->tmp_rank,
                                                                         q->d_ctr, 0)));
  else
    LAUNCH(eng, (k_force_insert<false, false><<<g, 256, 0, eng->stream>>>(q->d_tries, B, q->tmp_slot, q->tmp_rank,
                                                                          q->d_ctr, 0)));
  if (opt_ok) {  // redo of a member whose optimistic insert met a repeated key (exits at once otherwise)
    LAUNCH(eng, k_force_clear<<<g, 256, 0, eng->stream>>>(q->d_tries, B, q->d_ctr, 1, opt_ok));
    LAUNCH(eng, (k_force_insert<false, true><<<g, 256, 0, eng->stream>>>(q->d_tries, B, q->tmp_slot, q->tmp_rank,
                                                                         q->d_ctr, 1)));
  }
  if (single)
    LAUNCH(eng, k_force_assign<true><<<ga, 256, 0, eng->stream>>>(q->d_tries, B, q->tmp_slot, q->tmp_rank, q->d_ctr));
  else
    LAUNCH(eng, k_force_assign<false><<<ga, 256, 0, eng->stream>>>(q->d_tries, B, q->tmp_slot, q->tmp_rank, q->d_ctr));
  // (k_force_scatter also finalizes: states forced, keys inserted accumulated)
  LAUNCH(eng, k_force_scatter<<<g, 256, 0, eng->stream>>>(q->d_tries, B, q->tmp_slot, q->tmp_rank, q->d_ctr));
  q->mark(eng->stream, 0);
}

static bool root_sorted_path(const fjg_query* q, int t) {
  const auto& T = q->tries[t];
  return T.levels[0].size() <= 1 && T.rel->nrows >= (1u << FJG_SORTED_ROOT_MIN_LOG) && FJG_SORTED_ROOT;
}

// Force the roots of tries `ts` (all unforced): sorted roots one by one, the
// atomic-path roots together in batches whose rows fit the scratch arrays.
static void force_roots(fjg_query* q, const std::vector<int>& ts) {
  fjg_engine* eng = q->eng;
  for (int multi = 0; multi < 2; ++multi) {
    ForceBatch B;
    memset(&B, 0, sizeof(B));
    uint64_t off = 0, upper = 0;
    auto flush = [&]() {
      if (!B.n) return;
      launch_force_batch(q, B, upper, true, multi != 0);
      memset(&B, 0, sizeof(B));
      off = upper = 0;
    };
    for (int t : ts) {
      auto& T = q->tries[t];
      if ((int)T.lev[0].multi != multi) continue;
      if (root_sorted_path(q, t)) {
        if (!multi) force_root_sorted(q, t);
        else continue;
      } else {
        const uint32_t n = (uint32_t)T.rel->nrows;
        if (n == 0)  // empty root: probes read bucket 0 of a zero-length region and must see EMPTY
          CK(cudaMemsetAsync(T.dev.lev[0].table, 0xFF, 4 * sizeof(Slot), eng->stream));
        if (off + n > std::max<uint64_t>(q->max_n, 1)) flush();
        ForceRange& R = B.R[B.n++];
        R.single = 1;
        R.p0 = 0;
        R.len0 = n;
        R.trie = t;
        R.lev = 0;
        R.slot_off = (uint32_t)off;
        off += n;
        upper = std::max<uint64_t>(upper, n);
        q->forces += 1;
        q->count_maps(t, 0, 1);
        q->rows_forced += n;
        T.lev[0].dirty = true;
      }
      T.root_forced = true;
    }
    flush();
  }
}

static void force_level(fjg_query* q, int t, int l, bool single, uint32_t p0, uint32_t len0, uint32_t count) {
  fjg_engine* eng = q->eng;
  auto& T = q->tries[t];
  DevLevel& L = T.dev.lev[l];
  if (single && l == 0) {
    force_roots(q, {t});
    return;
  }
  ForceBatch B;
  memset(&B, 0, sizeof(B));
  B.n = 1;
  ForceRange& R = B.R[0];
  R.single = single ? 1 : 0;
  R.p0 = p0;
  R.len0 = len0;
  R.trie = t;
  R.lev = l;
  uint64_t upper = len0;
  if (!single) {
    R.list_p = L.list_p;
    R.list_len = L.list_len;
    R.list_scan = L.list_scan;
    R.list_count = reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(q->d_ctr) +
                                                     offsetof(DevCounters, list_count)) +
                   (t * MAXL + l);
    prim_scan<prims::OpSum, false>(eng, L.list_len, L.list_scan, count);
    // offsets to force: the claims' total when k_select counted it, else the level
    const uint32_t claimed = q->h_ctr->list_total[t * MAXL + l];
    upper = claimed ? std::min<uint64_t>(claimed, T.rel->nrows) : T.rel->nrows;
    // offset index -> list entry: marks at each entry's first index, then a max-scan
    CK(cudaMemsetAsync(q->owner_scratch, 0, std::max<uint64_t>(upper, 1) * 4, eng->stream));
    LAUNCH(eng, k_force_marks<<<grid_for(count), 256, 0, eng->stream>>>(L.list_scan, R.list_count,
                                                                         q->owner_scratch));
    prim_scan<prims::OpMax, false>(eng, q->owner_scratch, q->owner_scratch, upper);
    R.owner = q->owner_scratch;
  }
  launch_force_batch(q, B, upper, single, T.lev[l].multi);
  q->forces += 1;
  q->count_maps(t, l, single ? 1 : count);
  q->rows_forced += single ? len0 : 0;
  T.lev[l].dirty = true;
}


#ifndef FJG_GJ_SORT
#define FJG_GJ_SORT 1
#endif
#ifndef FJG_GJ_SORT_BITS
#define FJG_GJ_SORT_BITS 16  // high bits of the probed region start that order the bindings
#endif
// Order the F bindings entering GJ last node k by the region their probed
// subatom is probed in (k_probe_keys + radix sort), and build the permuted
// candidate scan. Returns the permutation (null when not worth it: the probed
// trie fits in L2, so probes hit L2 in any order).
static const uint32_t* probe_region_order(fjg_query* q, int k, const KNode& KN, uint64_t F, uint64_t*& scan_out) {
  fjg_engine* eng = q->eng;
  const DevNode& N = q->nodes[k];
  if (!FJG_GJ_SORT || N.nsub != 2 || F < 2) return nullptr;
  uint64_t rows = 0;
  for (int s = 0; s < 2; ++s) rows = std::max<uint64_t>(rows, q->tries[KN.sub[s].trie].dev.n);
  // probed tables (32 B / row) that fit in L2 gain nothing; FJG_GJ_SORT_MIN_ROWS
  // (environment) moves the threshold (tests force the path on small inputs)
  static const char* env = getenv("FJG_GJ_SORT_MIN_ROWS");
  const uint64_t min_rows = env ? strtoull(env, nullptr, 10) : 2ull * 126 * (1ull << 20) / 32;
  if (rows < min_rows) return nullptr;
  if (F > q->sort_cap) {
    q->sort_keys = (uint32_t*)q->alloc(F * 4);
    q->sort_keys2 = (uint32_t*)q->alloc(F * 4);
    q->sort_vals = (uint32_t*)q->alloc(F * 4);
    q->perm = (uint32_t*)q->alloc(F * 4);
    q->m_perm = (uint64_t*)q->alloc(F * 8);
    q->scan_perm = (uint64_t*)q->alloc(F * 8);
    q->sort_cap = F;
  }
  int bits = 1;
  while (bits < 32 && (1ull << bits) < rows) ++bits;
  // locality needs only the high bits: regions whose starts share them lie in
  // one window of 2^(bits - FJG_GJ_SORT_BITS) positions (2 radix passes, not 4)
  const int lo_bit = std::max(0, bits - FJG_GJ_SORT_BITS);
  const unsigned g = grid_for(F, 256, eng->num_sms * 16);
  LAUNCH(eng, k_probe_keys<2><<<g, 256, 0, eng->stream>>>(KN, F, q->sort_keys, q->sort_vals));
  const uint32_t* perm = prim_sort_pairs(eng, q->sort_keys, q->sort_vals, q->sort_keys2, q->perm, F, lo_bit, bits)
                             ? q->perm
                             : q->sort_vals;
  LAUNCH(eng, k_gather_m<<<g, 256, 0, eng->stream>>>(N.m, perm, F, q->m_perm));
  prim_scan<prims::OpSum, false>(eng, q->m_perm, q->scan_perm, F);
  scan_out = q->scan_perm;
  return perm;
}

static void run_node(fjg_query* q, int k, uint64_t F, int mode);

static void force_claims(fjg_query* q, int k) {
  // roots first, then claimed deeper subtries
  fjg_engine* eng = q->eng;
  DevCounters& H = *q->h_ctr;
  bool any = false;
  std::vector<int> roots;
  for (size_t t = 0; t < q->tries.size(); ++t)
    if (H.root_need[t] && !q->tries[t].root_forced) roots.push_back((int)t);
  if (!roots.empty()) {
    force_roots(q, roots);
    any = true;
  }
  for (size_t t = 0; t < q->tries.size(); ++t) {
    for (int l = 1; l < (int)q->tries[t].levels.size(); ++l) {
      const uint32_t c = H.list_count[t * MAXL + l];
      if (c) {
        force_level(q, (int)t, l, false, 0, 0, c);
        any = true;
      }
    }
  }
  if (any) {
    static_assert(offsetof(DevCounters, root_need) == offsetof(DevCounters, list_count) + sizeof(DevCounters::list_count) &&
                      offsetof(DevCounters, list_total) == offsetof(DevCounters, root_need) + sizeof(DevCounters::root_need),
                  "claim counters contiguous");
    CK(cudaMemsetAsync(reinterpret_cast<char*>(q->d_ctr) + offsetof(DevCounters, list_count), 0,
                       sizeof(H.list_count) + sizeof(H.root_need) + sizeof(H.list_total), eng->stream));
  }
  (void)k;
}

#ifndef FJG_STREAM_ONE
#define FJG_STREAM_ONE 1
#endif
template <int NP, int R, int W>
static void launch_stream_one_rw(fjg_query* q, const KNode& KN, const SProbe& SP, uint64_t c0, uint64_t c1) {
  fjg_engine* eng = q->eng;
  static int occ = 0;  // resident blocks per SM (persistent grid: one wave)
  if (!occ) {
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_stream_one<NP, R, W>, TILE, 0));
    occ = std::max(occ, 1);
  }
  const uint64_t warps = (c1 - c0 + 32 * R - 1) / (32 * R);
  const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((warps + TILE / 32 - 1) / (TILE / 32),
                                                                         (uint64_t)eng->num_sms * occ));
  LAUNCH(eng, (k_stream_one<NP, R, W><<<g, TILE, 0, eng->stream>>>(KN, SP, c0, c1, q->d_ctr)));
}
template <int NP, int W>
static void launch_stream_one_w(fjg_query* q, const KNode& KN, const SProbe& SP, uint64_t c0, uint64_t c1) {
  launch_stream_one_rw<NP, FJG_STREAM_R, W>(q, KN, SP, c0, c1);
}
template <int NP>
static void launch_stream_one_np(fjg_query* q, const KNode& KN, const SProbe& SP, uint64_t c0, uint64_t c1) {
  if (q->width <= 4)
    launch_stream_one_w<NP, 4>(q, KN, SP, c0, c1);
  else if (q->width <= 8)
    launch_stream_one_w<NP, 8>(q, KN, SP, c0, c1);
  else
    launch_stream_one_w<NP, 16>(q, KN, SP, c0, c1);
}
static void launch_stream_one(fjg_query* q, const KNode& KN, const SProbe& SP, uint64_t c0, uint64_t c1) {
  switch (SP.np) {
    case 1: launch_stream_one_np<1>(q, KN, SP, c0, c1); break;
    case 2: launch_stream_one_np<2>(q, KN, SP, c0, c1); break;
    case 3: launch_stream_one_np<3>(q, KN, SP, c0, c1); break;
    default: launch_stream_one_np<4>(q, KN, SP, c0, c1); break;
  }
}

#ifndef FJG_TAIL
#define FJG_TAIL 1
#endif
#ifndef FJG_SELECT_NS
#define FJG_SELECT_NS 1
#endif
template <int MODE, int NT>
static void launch_tail_nt(fjg_query* q, int k, uint64_t F, const uint32_t* dF) {
  fjg_engine* eng = q->eng;
  const KNode& KN = q->knodes[k];
  const TailPlan& T = q->tails[k];
  const unsigned g = grid_for(F, TILE, eng->num_sms * 8);
  if (q->width <= 4)
    LAUNCH(eng, (k_tail<MODE, 4, NT><<<g, TILE, 0, eng->stream>>>(KN, T, F, dF, q->min_var, q->out_tuples,
                                                                  q->out_cap, q->d_ctr)));
  else if (q->width <= 8)
    LAUNCH(eng, (k_tail<MODE, 8, NT><<<g, TILE, 0, eng->stream>>>(KN, T, F, dF, q->min_var, q->out_tuples,
                                                                  q->out_cap, q->d_ctr)));
  else
    LAUNCH(eng, (k_tail<MODE, 16, NT><<<g, TILE, 0, eng->stream>>>(KN, T, F, dF, q->min_var, q->out_tuples,
                                                                   q->out_cap, q->d_ctr)));
}
// F: the frontier size (host), or an upper bound when dF (device count) is given
template <int MODE>
static void launch_tail(fjg_query* q, int k, uint64_t F, const uint32_t* dF = nullptr) {
  if (q->tails[k].ntail == 1)
    launch_tail_nt<MODE, 1>(q, k, F, dF);
  else
    launch_tail_nt<MODE, MAXTAIL>(q, k, F, dF);
}

__global__ void k_set_root_node(uint8_t* chosen, uint64_t* m, uint64_t* scan, int best, uint64_t mv) {
  chosen[0] = (uint8_t)best;
  m[0] = mv;
  scan[0] = mv;
}

// k_select for the single empty binding entering node 0 when none of its
// tries' roots is forced yet (every COLT execution): each subatom is a root
// BaseScan, estimated_key_count = its cardinality, so the
// host picks the cover (min estimate, ties to the lowest position,
// SPEC.md:441) and the claims (every subatom but a stream-iterated cover)
// exactly as the kernel would, with no device round trip.
static bool host_select_root_node(fjg_query* q, int k, uint64_t F) {
  if (k != 0 || F != 1) return false;
  const DevNode& N = q->nodes[k];
  for (int s = 0; s < N.nsub; ++s)
    if (N.sub[s].depth != 0 || ((N.in_atoms >> N.sub[s].atom) & 1u) || q->tries[N.sub[s].trie].root_forced)
      return false;
  int best = N.cov[0];
  uint64_t best_est = N.atom_n[N.sub[best].atom];
  if (q->dynamic)
    for (int ci = 1; ci < N.ncov; ++ci) {
      const int s = N.cov[ci];
      const uint64_t est = N.atom_n[N.sub[s].atom];
      if (est < best_est) {
        best_est = est;
        best = s;
      }
    }
  const uint64_t m = N.atom_n[N.sub[best].atom];
  DevCounters& H = *q->h_ctr;
  H.total_m = m;
  for (int s = 0; s < N.nsub; ++s)
    if (s != best || !N.sub[s].stream) H.root_need[N.sub[s].trie] = 1;
  LAUNCH(q->eng, k_set_root_node<<<1, 1, 0, q->eng->stream>>>(N.chosen, N.m, N.scan, best, m));
  return true;
}

static void run_node(fjg_query* q, int k, uint64_t F, int mode) {
  if (F == 0) return;
  q->node_inputs[k] += F;
  fjg_engine* eng = q->eng;
  if (FJG_TAIL && q->tails[k].ntail > 0 && (mode == EXPAND_COUNT || mode == EXPAND_ENUM) && q->stop_node < 0) {
    // nodes k..K-1 in one kernel: no per-node select / scan / host sync
    q->mark(eng->stream, -1);
    if (mode == EXPAND_COUNT)
      launch_tail<EXPAND_COUNT>(q, k, F);
    else
      launch_tail<EXPAND_ENUM>(q, k, F);
    q->mark(eng->stream, 2);
    q->last_launches += 1;
    q->last_candidates += F;
    return;
  }
  const DevNode& N = q->nodes[k];
  const bool memo_top = mode == EXPAND_MEMO && k == q->stop_node;
  const KNode& KN = memo_top ? q->memo_top : q->knodes[k];
  const bool is_last = N.is_last || memo_top;
  if (!memo_top && host_select_root_node(q, k, F)) {
    // node 0 of a fresh COLT execution: its cover choice and claims need no device round trip
  } else {
  if (KN.nsub <= 2 && FJG_SELECT_NS)
    LAUNCH(eng, k_select_ns<2><<<grid_for(F, 256, eng->num_sms * 16), 256, 0, eng->stream>>>(
                    KN, q->d_tries, F, q->dynamic ? 1 : 0, q->d_ctr));
  else if (KN.nsub <= 3 && FJG_SELECT_NS)
    LAUNCH(eng, k_select_ns<3><<<grid_for(F, 256, eng->num_sms * 16), 256, 0, eng->stream>>>(
                    KN, q->d_tries, F, q->dynamic ? 1 : 0, q->d_ctr));
  else
    LAUNCH(eng, k_select<<<grid_for(F, 256, eng->num_sms * 16), 256, 0, eng->stream>>>(KN, q->d_tries, F,
                                                                                      q->dynamic ? 1 : 0, q->d_ctr));
  if (F <= kSmallScan) {
    LAUNCH(eng, k_scan_small<<<1, 1024, 0, eng->stream>>>(N.m, N.scan, (uint32_t)F, q->d_ctr));
  } else {
    prim_scan<prims::OpSum, false>(eng, N.m, N.scan, F,
                                   reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(q->d_ctr) +
                                                               offsetof(DevCounters, total_m)));
  }
  sync_counters(q);
  }
  const uint64_t M = q->h_ctr->total_m;
  force_claims(q, k);
  if (M == 0) return;
  if (is_last) {
    q->mark(eng->stream, -1);
    const bool gj_any = q->gj_x[k] >= 0 && (mode == EXPAND_COUNT || (mode == EXPAND_ENUM && FJG_GJW)) &&
                        q->gj_x[k] == (int)q->head.size() - 1 && FJG_GJ_R > 1 && q->nodes[k].nsub <= 3;
    uint64_t* gscan = N.scan;
    const uint32_t* perm = gj_any ? probe_region_order(q, k, KN, F, gscan) : nullptr;
    KNode KP = KN;
    KP.scan = gscan;
    // double steps per ticketed chunk: 4 when the bindings were ordered by probe region (tries larger than
    // L2: C5 1025 vs 1170 ms at 1), 1 otherwise (C2 3.36 vs 3.44 ms at 4; three-subatom nodes: C4)
    const bool rr_small = perm == nullptr;
    const uint64_t rr_gj = N.nsub == 3 ? FJG_GJW_RR3 : (rr_small ? FJG_GJW_RR_UNSORTED : FJG_GJW_RR);
    for (uint64_t c0 = 0; c0 < M; c0 += kLastChunk) {
      const uint64_t c1 = std::min(M, c0 + kLastChunk);
      const uint64_t ntiles = (c1 - c0 + TILE - 1) / TILE;
      const bool gj_fast = gj_any;
      if (gj_fast) {
        chunk_owners(q, gscan, F, c0, c1, FJG_GJW ? 64 * rr_gj : 32 * FJG_GJ_R);
        if (FJG_GJ_TICKET)
          CK(cudaMemsetAsync(reinterpret_cast<char*>(q->d_ctr) + offsetof(DevCounters, ticket), 0, 8, eng->stream));
      }
      else
        LAUNCH(eng, k_tile_bounds<<<grid_for(ntiles + 1), 256, 0, eng->stream>>>(N.scan, F, c0, c1, q->bounds));
      const unsigned g = grid_for(c1 - c0, TILE, eng->num_sms * 8);
      if (mode == EXPAND_ENUM && gj_fast) {  // k_last_gj_warp writing the tuples
        const int W8 = q->head.size() <= 4 ? 4 : 8;
        const uint64_t rr = rr_gj;
        const uint64_t nch = (c1 - c0 + 64 * rr - 1) / (64 * rr);
        const unsigned gw = (unsigned)std::max<uint64_t>(
            1, std::min<uint64_t>((nch + TILE / 32 - 1) / (TILE / 32), (uint64_t)eng->num_sms * (N.nsub == 3 ? FJG_GJW_MINB3 : FJG_GJW_MINB)));
        if (N.nsub == 2 && W8 == 4 && rr_small)
          LAUNCH(eng, (k_last_gj_warp<2, 4, FJG_GJW_RR_UNSORTED, true><<<gw, TILE, 0, eng->stream>>>(
                          KP, c0, c1, F, q->chunk_owner, perm, q->min_var, q->d_ctr, q->out_tuples, q->out_cap)));
        else if (N.nsub == 2 && rr_small)
          LAUNCH(eng, (k_last_gj_warp<2, 8, FJG_GJW_RR_UNSORTED, true><<<gw, TILE, 0, eng->stream>>>(
                          KP, c0, c1, F, q->chunk_owner, perm, q->min_var, q->d_ctr, q->out_tuples, q->out_cap)));
        else if (N.nsub == 2 && W8 == 4)
          LAUNCH(eng, (k_last_gj_warp<2, 4, FJG_GJW_RR, true><<<gw, TILE, 0, eng->stream>>>(
                          KP, c0, c1, F, q->chunk_owner, perm, q->min_var, q->d_ctr, q->out_tuples, q->out_cap)));
        else if (N.nsub == 2)
          LAUNCH(eng, (k_last_gj_warp<2, 8, FJG_GJW_RR, true><<<gw, TILE, 0, eng->stream>>>(
                          KP, c0, c1, F, q->chunk_owner, perm, q->min_var, q->d_ctr, q->out_tuples, q->out_cap)));
        else if (W8 == 4)
          LAUNCH(eng, (k_last_gj_warp<3, 4, FJG_GJW_RR3, true><<<gw, TILE, 0, eng->stream>>>(
                          KP, c0, c1, F, q->chunk_owner, perm, q->min_var, q->d_ctr, q->out_tuples, q->out_cap)));
        else
          LAUNCH(eng, (k_last_gj_warp<3, 8, FJG_GJW_RR3, true><<<gw, TILE, 0, eng->stream>>>(
                          KP, c0, c1, F, q->chunk_owner, perm, q->min_var, q->d_ctr, q->out_tuples, q->out_cap)));
      } else if (mode == EXPAND_ENUM)
        LAUNCH(eng, launch_expand<EXPAND_ENUM>(q->width, g, eng->stream, KN, c0, c1, F, q->bounds, q->min_var,
                                               q->out_tuples, q->out_cap, q->d_ctr));
      else if (mode == EXPAND_MEMO)
        LAUNCH(eng, launch_expand<EXPAND_MEMO>(q->width, g, eng->stream, KN, c0, c1, F, q->bounds, -1, nullptr, 0,
                                               q->d_ctr));
      else if (gj_fast && FJG_GJW) {  // k_last_gj_warp: x is the last head variable
        const int W8 = q->head.size() <= 4 ? 4 : 8;
        const uint64_t rr = rr_gj;
        const uint64_t nch = (c1 - c0 + 64 * rr - 1) / (64 * rr);
        const unsigned gw = (unsigned)std::max<uint64_t>(
            1, std::min<uint64_t>((nch + TILE / 32 - 1) / (TILE / 32), (uint64_t)eng->num_sms * (N.nsub == 3 ? FJG_GJW_MINB3 : FJG_GJW_MINB)));
        if (N.nsub == 2 && W8 == 4 && rr_small)
          LAUNCH(eng, (k_last_gj_warp<2, 4, FJG_GJW_RR_UNSORTED><<<gw, TILE, 0, eng->stream>>>(
                          KP, c0, c1, F, q->chunk_owner, perm, q->min_var, q->d_ctr)));
        else if (N.nsub == 2 && rr_small)
          LAUNCH(eng, (k_last_gj_warp<2, 8, FJG_GJW_RR_UNSORTED><<<gw, TILE, 0, eng->stream>>>(
                          KP, c0, c1, F, q->chunk_owner, perm, q->min_var, q->d_ctr)));
        else if (N.nsub == 2 && W8 == 4)
          LAUNCH(eng, (k_last_gj_warp<2, 4, FJG_GJW_RR><<<gw, TILE, 0, eng->stream>>>(KP, c0, c1, F, q->chunk_owner,
                                                                                      perm, q->min_var, q->d_ctr)));
        else if (N.nsub == 2)
          LAUNCH(eng, (k_last_gj_warp<2, 8, FJG_GJW_RR><<<gw, TILE, 0, eng->stream>>>(KP, c0, c1, F, q->chunk_owner,
                                                                                      perm, q->min_var, q->d_ctr)));
        else if (W8 == 4)
          LAUNCH(eng, (k_last_gj_warp<3, 4, FJG_GJW_RR3><<<gw, TILE, 0, eng->stream>>>(KP, c0, c1, F, q->chunk_owner,
                                                                                      perm, q->min_var, q->d_ctr)));
        else
          LAUNCH(eng, (k_last_gj_warp<3, 8, FJG_GJW_RR3><<<gw, TILE, 0, eng->stream>>>(KP, c0, c1, F, q->chunk_owner,
                                                                                      perm, q->min_var, q->d_ctr)));
      } else if (gj_fast) {  // k_last_gj_bf: x is the last head variable
        const int W8 = q->head.size() <= 4 ? 4 : 8;
        const unsigned gi = grid_for(c1 - c0, TILE * FJG_GJ_R, eng->num_sms * 8);
        if (N.nsub == 2 && W8 == 4)
          LAUNCH(eng, (k_last_gj_bf<2, FJG_GJ_R, 4><<<gi, TILE, 0, eng->stream>>>(KP, c0, c1, F, q->chunk_owner,
                                                                                perm, q->min_var, q->d_ctr)));
        else if (N.nsub == 2)
          LAUNCH(eng, (k_last_gj_bf<2, FJG_GJ_R, 8><<<gi, TILE, 0, eng->stream>>>(KP, c0, c1, F, q->chunk_owner,
                                                                                perm, q->min_var, q->d_ctr)));
        else if (W8 == 4)
          LAUNCH(eng, (k_last_gj_bf<3, FJG_GJ_R, 4><<<gi, TILE, 0, eng->stream>>>(KP, c0, c1, F, q->chunk_owner,
                                                                                perm, q->min_var, q->d_ctr)));
        else
          LAUNCH(eng, (k_last_gj_bf<3, FJG_GJ_R, 8><<<gi, TILE, 0, eng->stream>>>(KP, c0, c1, F, q->chunk_owner,
                                                                                perm, q->min_var, q->d_ctr)));
      } else if (q->gj_x[k] >= 0 && mode == EXPAND_COUNT) {
        const int W8 = q->head.size() <= 4 ? 4 : 8;
        const int ns = N.nsub;
        if (ns == 2 && W8 == 4)
          LAUNCH(eng, (k_last_gj<2, 4><<<g, TILE, 0, eng->stream>>>(KN, c0, c1, F, q->bounds, q->gj_x[k], q->min_var,
                                                                     q->d_ctr)));
        else if (ns == 2)
          LAUNCH(eng, (k_last_gj<2, 8><<<g, TILE, 0, eng->stream>>>(KN, c0, c1, F, q->bounds, q->gj_x[k], q->min_var,
                                                                     q->d_ctr)));
        else if (W8 == 4)
          LAUNCH(eng, (k_last_gj<3, 4><<<g, TILE, 0, eng->stream>>>(KN, c0, c1, F, q->bounds, q->gj_x[k], q->min_var,
                                                                     q->d_ctr)));
        else
          LAUNCH(eng, (k_last_gj<3, 8><<<g, TILE, 0, eng->stream>>>(KN, c0, c1, F, q->bounds, q->gj_x[k], q->min_var,
                                                                     q->d_ctr)));
      } else
        LAUNCH(eng, launch_expand<EXPAND_COUNT>(q->width, g, eng->stream, KN, c0, c1, F, q->bounds, q->min_var,
                                                nullptr, 0, q->d_ctr));
    }
    q->mark(eng->stream, 2);
    q->last_launches += 1;
    q->last_candidates += M;
    return;
  }
  for (uint64_t c0 = 0; c0 < M; c0 += q->batch) {
    const uint64_t c1 = std::min(M, c0 + q->batch);
    CK(cudaMemsetAsync(reinterpret_cast<char*>(q->d_ctr) + offsetof(DevCounters, survivors), 0, 4, eng->stream));
    q->mark(eng->stream, -1);
    const uint64_t ntiles = (c1 - c0 + TILE - 1) / TILE;
    const bool gj_write = q->gj_w[k] >= 0 && FJG_GJ_WRITE;
    const bool one = F == 1 && q->sprobe[k].np > 0 && FJG_STREAM_ONE;
    if (gj_write) {
      chunk_owners(q, N.scan, F, c0, c1, 32);
      if (FJG_WRITE_TICKET)
        CK(cudaMemsetAsync(reinterpret_cast<char*>(q->d_ctr) + offsetof(DevCounters, ticket), 0, 8, eng->stream));
    }
    else if (!one)
      LAUNCH(eng, k_tile_bounds<<<grid_for(ntiles + 1), 256, 0, eng->stream>>>(N.scan, F, c0, c1, q->bounds));
    const unsigned gw = grid_for(c1 - c0, TILE, eng->num_sms * 8);
    if (gj_write) {
      const int w8 = q->width <= 4 ? 4 : 8;
      if (N.nsub == 2 && w8 == 4)
        LAUNCH(eng, (k_write_gj<2, 4><<<gw, TILE, 0, eng->stream>>>(KN, c0, c1, F, q->chunk_owner, q->gj_w[k], q->d_ctr)));
      else if (N.nsub == 2)
        LAUNCH(eng, (k_write_gj<2, 8><<<gw, TILE, 0, eng->stream>>>(KN, c0, c1, F, q->chunk_owner, q->gj_w[k], q->d_ctr)));
      else if (w8 == 4)
        LAUNCH(eng, (k_write_gj<3, 4><<<gw, TILE, 0, eng->stream>>>(KN, c0, c1, F, q->chunk_owner, q->gj_w[k], q->d_ctr)));
      else
        LAUNCH(eng, (k_write_gj<3, 8><<<gw, TILE, 0, eng->stream>>>(KN, c0, c1, F, q->chunk_owner, q->gj_w[k], q->d_ctr)));
    } else if (one) {
      launch_stream_one(q, KN, q->sprobe[k], c0, c1);
    } else if (q->sw[k] && FJG_STREAM_WRITE) {
      if (q->width <= 4)
        LAUNCH(eng, (k_write_stream<4><<<gw, TILE, 0, eng->stream>>>(KN, c0, c1, F, q->bounds, q->d_ctr)));
      else if (q->width <= 8)
        LAUNCH(eng, (k_write_stream<8><<<gw, TILE, 0, eng->stream>>>(KN, c0, c1, F, q->bounds, q->d_ctr)));
      else
        LAUNCH(eng, (k_write_stream<16><<<gw, TILE, 0, eng->stream>>>(KN, c0, c1, F, q->bounds, q->d_ctr)));
    } else {
      LAUNCH(eng, launch_expand<EXPAND_WRITE>(q->width, gw, eng->stream, KN, c0, c1, F, q->bounds, -1, nullptr, 0,
                                              q->d_ctr));
    }
    q->mark(eng->stream, k == 0 ? 3 : 1);
    if (FJG_TAIL && k + 1 < (int)q->nodes.size() && q->tails[k + 1].ntail > 0 &&
        (mode == EXPAND_COUNT || mode == EXPAND_ENUM) && q->stop_node < 0) {
      // the next nodes are a Cartesian tail: it reads its frontier size on the
      // device, so this batch needs no host round trip
      const uint32_t* dF = reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(q->d_ctr) +
                                                             offsetof(DevCounters, survivors));
      q->mark(eng->stream, -1);
      if (mode == EXPAND_COUNT)
        launch_tail<EXPAND_COUNT>(q, k + 1, c1 - c0, dF);
      else
        launch_tail<EXPAND_ENUM>(q, k + 1, c1 - c0, dF);
      q->mark(eng->stream, 2);
      q->last_launches += 1;
      q->dev_tail_node = k + 1;
      continue;
    }
    sync_counters(q);
    run_node(q, k + 1, q->h_ctr->survivors, mode);
  }
}

// One launch resets an execution: the device counters (minv = +inf, root
// probe regions = row counts) and the subtrie states of every level the last
// execution forced (slot regions and child counts are cleared by the force
// that claims them).
struct ResetPlan {
  int nz, ntries;
  uint32_t* ptr[MAXT * MAXL];
  uint32_t n[MAXT * MAXL];
  uint32_t root_region[MAXT];
};
__global__ void k_reset(const __grid_constant__ ResetPlan P, DevCounters* ctr) {
  if (blockIdx.y == 0) {
    uint32_t* w = reinterpret_cast<uint32_t*>(ctr);
    constexpr uint32_t kMin = offsetof(DevCounters, minv) / 4, kReg = offsetof(DevCounters, root_region) / 4;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < sizeof(DevCounters) / 4; i += gridDim.x * blockDim.x) {
      uint32_t v = 0;
      if (i == kMin) v = 0xFFFFFFFFu;      // minv = LLONG_MAX (little endian: low word all ones,
      if (i == kMin + 1) v = 0x7FFFFFFFu;  // high word 0x7fffffff)
      if (i >= kReg && i < kReg + (uint32_t)P.ntries) v = P.root_region[i - kReg];
      w[i] = v;
    }
    return;
  }
  const int z = blockIdx.y - 1;
  uint32_t* p = P.ptr[z];
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n[z]; i += gridDim.x * blockDim.x) p[i] = 0;
}

static void reset_query(fjg_query* q) {
  fjg_engine* eng = q->eng;
  ResetPlan P;
  memset(&P, 0, sizeof(P));
  uint32_t maxn = 1;
  for (auto& T : q->tries) {
    for (size_t l = 0; l < T.lev.size(); ++l) {
      auto& H = T.lev[l];
      DevLevel& L = T.dev.lev[l];
      if (H.dirty) {
        P.ptr[P.nz] = reinterpret_cast<uint32_t*>(L.sn);  // (state, key count) records: both words cleared
        P.n[P.nz] = (uint32_t)(2 * H.nsub);
        maxn = std::max<uint32_t>(maxn, (uint32_t)(2 * H.nsub));
        ++P.nz;
        H.dirty = false;
      }
    }
    T.root_forced = false;
  }
  P.ntries = (int)q->tries.size();
  for (size_t t = 0; t < q->tries.size(); ++t) P.root_region[t] = (uint32_t)std::max<uint64_t>(q->tries[t].rel->nrows, 1);
  const dim3 grid(std::min<uint32_t>((maxn + 255) / 256, (uint32_t)eng->num_sms * 4), 1 + P.nz);
  LAUNCH(eng, k_reset<<<grid, 256, 0, eng->stream>>>(P, q->d_ctr));
  DevCounters& z = *q->h_ctr;
  memset(&z, 0, sizeof(z));
  z.minv = LLONG_MAX;
  for (size_t t = 0; t < q->tries.size(); ++t) z.root_region[t] = P.root_region[t];
  q->maps_built = q->forces = q->rows_forced = 0;
  for (int t = 0; t < MAXA; ++t) {
    q->trie_maps[t] = 0;
    q->trie_levels[t] = 0;
  }
  q->build_ms = q->join_ms = q->last_ms = 0;
  q->phase_ms[0] = q->phase_ms[1] = q->phase_ms[2] = q->phase_ms[3] = q->phase_ms[4] = 0;
  q->memo_rows[0] = q->memo_rows[1] = q->memo_rows[2] = 0;
  q->last_launches = q->last_candidates = 0;
  q->dev_tail_node = -1;
  for (int k = 0; k < MAXN; ++k) q->node_inputs[k] = 0;
  q->marks.clear();
  q->ev_used = 0;
}

// Memoised chain count: force the chain tries' roots, then the bottom-up passes.
static void run_memo_passes(fjg_query* q) {
  fjg_engine* eng = q->eng;
  std::set<int> tries;
  for (int j = q->chain_start; j < (int)q->nodes.size(); ++j)
    for (int i = 0; i < q->nodes[j].nsub; ++i) tries.insert(q->nodes[j].sub[i].trie);
  std::vector<int> roots;
  for (int t : tries)
    if (!q->tries[t].root_forced) roots.push_back(t);
  force_roots(q, roots);
  for (auto& [t, gid] : q->gid) {
    const uint64_t n = q->tries[t].rel->nrows;
    if (!n) continue;
    LAUNCH(eng, k_start_flags<<<grid_for(n), 256, 0, eng->stream>>>(q->tries[t].dev.lev[0].cnt, n, gid));
    prim_scan<prims::OpSum, false>(eng, gid, gid, n);
  }
  q->mark(eng->stream, -1);
  const unsigned grid = grid_for(std::max<uint64_t>(q->max_n, 1), 256, eng->num_sms * 16);
  // one initialisation pass per chain trie: every memo array over its groups,
  // and its dense key map when a pass resolves through it
  for (auto& [t, gid] : q->gid) {
    MemoInit I{};
    I.n = q->tries[t].rel->nrows;
    I.gid = gid;
    I.cnt = q->tries[t].dev.lev[0].cnt;
    if (q->memo_dense.count(t)) {
      const uint64_t dn = 1ull << std::min(q->tries[t].key_bits, 31);
      I.dense = q->memo_dense[t];
      I.dense_n = (uint32_t)dn;
      I.key = q->tries[t].dev.lev[0].cval[q->tries[t].dev.lev[0].keycol[0]];
      CK(cudaMemsetAsync(I.dense, 0xff, dn * 4, eng->stream));
    }
    for (size_t i = 0; i < q->memo_passes.size(); ++i) {
      const MemoPass& M = q->memo_passes[i];
      if (M.gid != gid || !M.n) continue;
      if (I.nout == kMemoInitMax) {
        LAUNCH(eng, k_memo_init<<<grid, 256, 0, eng->stream>>>(I));
        I.nout = 0;
        I.dense = nullptr;
      }
      I.out[I.nout] = M.memo_out;
      I.group_size[I.nout] = M.nfresh == 0 ? 1 : 0;
      ++I.nout;
    }
    if (I.n && (I.nout || I.dense)) {
      LAUNCH(eng, k_memo_init<<<grid, 256, 0, eng->stream>>>(I));
      q->memo_rows[2] += I.n;
    }
  }
  for (int i = (int)q->memo_passes.size() - 1; i >= 0; --i) {
    const MemoPass& M = q->memo_passes[i];
    if (!M.n) continue;
    if (M.nfresh == 0) continue;  // every row counts 1: the group sizes, written by k_memo_init
    if (q->memo_resolve_of[i] < 0) {
      LAUNCH(eng, k_memo_resolve<<<grid, 256, 0, eng->stream>>>(M));
      q->memo_rows[0] += M.n;
    }
    LAUNCH(eng, k_memo_gather<<<grid, 256, 0, eng->stream>>>(M));
    q->memo_rows[1] += M.n;
  }
  q->mark(eng->stream, 4);
}

// SLT / SIMPLE backends: force level 0 of every trie (SLT)
// or every level of every trie (SIMPLE) before the join; COLT does neither.
static void eager_build(fjg_query* q) {
  fjg_engine* eng = q->eng;
  std::vector<int> roots;
  for (size_t t = 0; t < q->tries.size(); ++t)
    if (q->tries[t].map_levels >= 1 && !q->tries[t].root_forced) roots.push_back((int)t);
  force_roots(q, roots);
  for (size_t t = 0; t < q->tries.size(); ++t) {
    auto& T = q->tries[t];
    if (T.map_levels < 1) continue;
    if (q->backend != FJG_BACKEND_SIMPLE) continue;
    // an empty relation has no subtries below its root: its deeper tables were
    // never cleared by a force, so k_eager_list must not read them
    if (T.rel->nrows == 0) continue;
    const uint64_t nslots = 4ull * FJG_RS * std::max<uint64_t>(T.rel->nrows, 1);
    for (int l = 1; l < T.map_levels; ++l) {
      uint32_t* cntp = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(q->d_ctr) +
                                                   offsetof(DevCounters, list_count)) +
                       (t * MAXL + l);
      CK(cudaMemsetAsync(cntp, 0, 4, eng->stream));
      const DevLevel& P = T.dev.lev[l - 1];
      const DevLevel& L = T.dev.lev[l];
      LAUNCH(eng, k_eager_list<<<grid_for(nslots), 256, 0, eng->stream>>>(
                      P.table, nslots, P.cnt, L, cntp, l == 1 ? q->d_ctr->root_region + t : nullptr));
      sync_counters(q);
      const uint32_t c = q->h_ctr->list_count[t * MAXL + l];
      if (c) {
        force_level(q, (int)t, l, false, 0, 0, c);
      }
      CK(cudaMemsetAsync(cntp, 0, 4, eng->stream));
    }
  }
}

// The chain's top node 0 as one reduction over pass 0's resolved children
// (k_memo_total) when node 0 = [A(u,v) stream cover, B(v) root probe], A is a
// single-subatom atom over the same relation and column as pass 0's carrier,
// and B's root is the table pass 0 probed: node 0's rows are then the carrier
// relation's rows and child(row) is exactly what pass 0 resolved per position.
static bool memo_top_is_total(const fjg_query* q) {
  if (q->chain_start != 1 || q->min_var >= 0 || q->memo_passes.empty()) return false;
  const MemoPass& M0 = q->memo_passes[0];
  if (M0.nfresh != 1 || M0.cont_x != 0 || M0.has_coef || !M0.child || M0.cnv != 1) return false;
  const DevNode& N0 = q->nodes[0];
  const KNode& K0 = q->knodes[0];
  if (N0.nsub != 2) return false;
  int c = -1, x = -1;
  for (int i = 0; i < 2; ++i) {
    if (N0.sub[i].nv == 2 && N0.sub[i].depth == 0) c = i;
    if (N0.sub[i].nv == 1 && N0.sub[i].depth == 0 && !K0.sub[i].in_p) x = i;
  }
  if (c < 0 || x < 0 || c == x) return false;
  if (K0.sub[x].table != M0.fresh[0].table) return false;
  const int A = N0.sub[c].atom;
  if (q->atoms[A].subs.size() != 1) return false;
  const int v = N0.sub[x].var[0];
  if (N0.sub[c].var[0] != v && N0.sub[c].var[1] != v) return false;
  int carrier, next;
  std::vector<int> fresh;
  if (!device_chain_node(q, 1, carrier, fresh, next)) return false;
  const int C = q->nodes[1].sub[carrier].atom;
  const int cv = q->nodes[1].sub[carrier].var[0];
  if (q->atoms[A].rel_index != q->atoms[C].rel_index) return false;
  const auto& av = q->atoms[A].vars;
  const auto& cvs = q->atoms[C].vars;
  const int acol = (int)(std::find(av.begin(), av.end(), v) - av.begin());
  const int ccol = (int)(std::find(cvs.begin(), cvs.end(), cv) - cvs.begin());
  return acol == ccol && acol < (int)av.size();
}

static void execute_once(fjg_query* q, int mode) {
  reset_query(q);
  if (q->backend != FJG_BACKEND_COLT) eager_build(q);
  q->stop_node = -1;
  if (mode == EXPAND_MEMO) {
    run_memo_passes(q);
    q->stop_node = q->chain_start - 1;
  }
  if (mode == EXPAND_MEMO && memo_top_is_total(q)) {
    fjg_engine* eng = q->eng;
    const MemoPass& M0 = q->memo_passes[0];
    q->mark(eng->stream, -1);
    LAUNCH(eng, k_memo_total<<<grid_for(M0.n, 256, eng->num_sms * 8), 256, 0, eng->stream>>>(M0.child, M0.n,
                                                                                         q->memo[0], 0, q->d_ctr));
    q->mark(eng->stream, 2);
    q->last_launches += 1;
    q->last_candidates += M0.n;
    q->node_inputs[0] = 1;
  } else {
    run_node(q, 0, 1, mode);
  }
  sync_counters(q);
  if (q->dev_tail_node >= 0) q->last_candidates += q->h_ctr->tail_inputs[q->dev_tail_node];
  q->resolve_marks();
  q->build_ms = q->phase_ms[0];
  q->join_ms = q->phase_ms[1] + q->phase_ms[2] + q->phase_ms[3] + q->phase_ms[4];
  q->last_ms = q->phase_ms[2];
  q->first_ms = q->phase_ms[3];
}

// ============================================================================
// C-ABI (device side)
// ============================================================================
template <class F>
static int guard(F&& f) {
  try {
    f();
    return FJG_OK;
  } catch (const fj::Error& e) {
    fjg::set_last_error(e.what());
    return e.code();
  } catch (const std::bad_alloc&) {
    fjg::set_last_error("host allocation failed");
    return FJG_E_RESOURCE;
  } catch (const std::exception& e) {
    fjg::set_last_error(e.what());
    return FJG_E_ENGINE;
  }
}

extern "C" {

int fjg_engine_create(int device, fjg_engine** out) {
  return guard([&] {
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) throw fj::ResourceError("no CUDA device " + std::to_string(device));
    ScopedDevice sd(device);
    CK(cudaSetDevice(device));
    auto* e = new fjg_engine();
    e->device = device;
    CK(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
    e->pool.reset(new Pool(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    e->num_sms = prop.multiProcessorCount;
    CK(cudaMallocHost(&e->h_ctr, sizeof(DevCounters)));
    e->prim_ticket = (unsigned long long*)e->pool->alloc(8);
    e->prim_hist = (uint32_t*)e->pool->alloc(prims::kRadixMaxPasses * prims::kRadixBins * 4);
    CK(cudaMemsetAsync(e->prim_ticket, 0, 8, e->stream));
    *out = e;
  });
}

void fjg_engine_destroy(fjg_engine* eng) {
  if (!eng) return;
  ScopedDevice sd(eng->device);
  cudaStreamSynchronize(eng->stream);
  eng->pool.reset();
  if (eng->h_ctr) cudaFreeHost(eng->h_ctr);
  cudaStreamDestroy(eng->stream);
  delete eng;
}

void* fjg_engine_stream(fjg_engine* eng) { return eng ? (void*)eng->stream : nullptr; }

int fjg_engine_sync(fjg_engine* eng) {
  return guard([&] { CK(cudaStreamSynchronize(eng->stream)); });
}

static fjg_relation* new_relation(fjg_engine* eng, int ncols, uint64_t nrows) {
  if (ncols <= 0 || ncols > MAXC) throw fj::ValidationError("relation must have 1..8 columns");
  if (nrows >= 0xFFFFFFF0ull) throw fj::ValidationError("relation too large (rows must be < 2^32-16)");
  auto* r = new fjg_relation();
  r->eng = eng;
  r->nrows = nrows;
  r->ncols = ncols;
  for (int c = 0; c < ncols; ++c) {
    void* p = eng->pool->alloc(std::max<uint64_t>(nrows, 1) * 4);
    r->owned.push_back(p);
    r->cols.push_back((int32_t*)p);
  }
  return r;
}

int fjg_relation_create(fjg_engine* eng, const int32_t* const* host_cols, int ncols, uint64_t nrows,
                        fjg_relation** out) {
  return guard([&] {
    ScopedDevice sd(eng->device);
    fjg_relation* r = new_relation(eng, ncols, nrows);
    for (int c = 0; c < ncols; ++c)
      if (nrows) CK(cudaMemcpyAsync(r->cols[c], host_cols[c], nrows * 4, cudaMemcpyHostToDevice, eng->stream));
    *out = r;
  });
}

// fj::Value carries int64 (value.hpp:31); the engine's columns are int32. An
// int64 column is staged through the device in chunks and narrowed there
// (k_narrow_i64); a value outside int32 is a ValidationError naming its
// column and row (wide domains are dictionary-encoded by the caller).
int fjg_relation_create_i64(fjg_engine* eng, const int64_t* const* host_cols, int ncols, uint64_t nrows,
                            fjg_relation** out) {
  return guard([&] {
    ScopedDevice sd(eng->device);
    fjg_relation* r = new_relation(eng, ncols, nrows);
    if (nrows == 0) {
      *out = r;
      return;
    }
    constexpr uint64_t kChunk = 1ull << 24;  // 128 MB of int64 per staged chunk
    const uint64_t chunk = std::min<uint64_t>(nrows, kChunk);
    long long* stage = (long long*)eng->pool->alloc(chunk * 8);
    unsigned long long* d_bad = (unsigned long long*)eng->pool->alloc((size_t)ncols * 8);
    std::vector<unsigned long long> h_bad(ncols, ~0ull);
    try {
      CK(cudaMemsetAsync(d_bad, 0xFF, (size_t)ncols * 8, eng->stream));
      for (int c = 0; c < ncols; ++c)
        for (uint64_t r0 = 0; r0 < nrows; r0 += chunk) {
          const uint64_t m = std::min<uint64_t>(chunk, nrows - r0);
          CK(cudaMemcpyAsync(stage, host_cols[c] + r0, m * 8, cudaMemcpyHostToDevice, eng->stream));
          LAUNCH(eng, k_narrow_i64<<<grid_for(m / 4 + 1, 256, eng->num_sms * 8), 256, 0, eng->stream>>>(
                          stage, m, r0, r->cols[c] + r0, d_bad + c));
        }
      CK(cudaMemcpyAsync(h_bad.data(), d_bad, (size_t)ncols * 8, cudaMemcpyDeviceToHost, eng->stream));
      CK(cudaStreamSynchronize(eng->stream));
      ++eng->syncs;
    } catch (...) {
      eng->pool->free(stage);
      eng->pool->free(d_bad);
      fjg_relation_destroy(r);
      throw;
    }
    eng->pool->free(stage);
    eng->pool->free(d_bad);
    for (int c = 0; c < ncols; ++c)
      if (h_bad[c] != ~0ull) {
        fjg_relation_destroy(r);
        throw fj::ValidationError("int64 value outside the int32 range at column " + std::to_string(c) + ", row " +
                                  std::to_string(h_bad[c]) + " (dictionary-encode wide domains before loading)");
      }
    *out = r;
  });
}

int fjg_relation_from_device(fjg_engine* eng, const int32_t* const* dev_cols, int ncols, uint64_t nrows, int copy,
                             fjg_relation** out) {
  return guard([&] {
    ScopedDevice sd(eng->device);
    if (copy) {
      fjg_relation* r = new_relation(eng, ncols, nrows);
      for (int c = 0; c < ncols; ++c)
        if (nrows) CK(cudaMemcpyAsync(r->cols[c], dev_cols[c], nrows * 4, cudaMemcpyDeviceToDevice, eng->stream));
      *out = r;
    } else {
      if (ncols <= 0 || ncols > MAXC) throw fj::ValidationError("relation must have 1..8 columns");
      if (nrows >= (1ull << 32) - 16) throw fj::ValidationError("relations must have fewer than 2^32-16 rows");
      auto* r = new fjg_relation();
      r->eng = eng;
      r->nrows = nrows;
      r->ncols = ncols;
      for (int c = 0; c < ncols; ++c) r->cols.push_back(const_cast<int32_t*>(dev_cols[c]));
      *out = r;
    }
  });
}

int fjg_relation_filter(const fjg_relation* in, const fjg_predicate* preds, int npreds, fjg_relation** out) {
  return guard([&] {
    fjg_engine* eng = in->eng;
    ScopedDevice sd(eng->device);
    if (npreds > 8) throw fj::ValidationError("at most 8 predicates");
    DevPreds P{};
    P.n = npreds;
    for (int i = 0; i < npreds; ++i) {
      if (preds[i].column < 0 || preds[i].column >= in->ncols ||
          (preds[i].is_column && (preds[i].rhs_column < 0 || preds[i].rhs_column >= in->ncols)))
        throw fj::ValidationError("predicate references unknown column");
      if (preds[i].cmp < 0 || preds[i].cmp > 5) throw fj::ValidationError("bad comparator");
      P.p[i] = preds[i];
    }
    for (int c = 0; c < in->ncols; ++c) P.cols[c] = in->cols[c];
    const uint64_t n = in->nrows;
    uint32_t* flags = (uint32_t*)eng->pool->alloc(std::max<uint64_t>(n, 1) * 4);
    uint32_t* excl = (uint32_t*)eng->pool->alloc(std::max<uint64_t>(n, 1) * 4 + 4);
    uint32_t total = 0;
    if (n) {
      LAUNCH(eng, k_filter_flags<<<grid_for(n), 256, 0, eng->stream>>>(P, n, flags));
      uint32_t* d_total = excl + std::max<uint64_t>(n, 1);
      prim_scan<prims::OpSum, true>(eng, flags, excl, n, d_total);
      CK(cudaMemcpyAsync(&total, d_total, 4, cudaMemcpyDeviceToHost, eng->stream));
      CK(cudaStreamSynchronize(eng->stream));
    }
    fjg_relation* r = new_relation(eng, in->ncols, total);
    for (int c = 0; c < in->ncols && n; ++c)
      LAUNCH(eng, k_compact_col<<<grid_for(n), 256, 0, eng->stream>>>(in->cols[c], flags, excl, n, r->cols[c]));
    CK(cudaStreamSynchronize(eng->stream));
    eng->pool->free(flags);
    eng->pool->free(excl);
    *out = r;
  });
}

// Stable hash-partition of `in` on column `col`: rows for destination d land in
// out_cols[c][base_d ...) in their original order (flags -> scan -> compact per
// destination).
// Stable hash-partition of `in` on column `col` (counting sort by destination,
// one host sync): rows for destination d land in out_cols[c][base_d ...) in
// their original order.
// Hash-partition `in` on `col` into out_cols (grouped by destination, stable
// within one), asynchronously on the engine stream: d_tot[0..nparts] receives
// the cumulative row offsets of the destinations (u32, on the device).
static void partition_async(const fjg_relation* in, int col, int nparts, int32_t* const* out_cols, uint32_t* d_tot) {
  fjg_engine* eng = in->eng;
  if (col < 0 || col >= in->ncols) throw fj::ValidationError("partition column out of range");
  if (nparts < 1 || nparts > 1024) throw fj::ValidationError("nparts must be 1..1024");
  const uint64_t n = in->nrows;
  // k_part_count / k_part_scatter keep histograms and offsets in 32 bits
  if (n >= (1ull << 32) - 16) throw fj::ValidationError("partition: relations must have fewer than 2^32-16 rows");
  if (n == 0) {
    CK(cudaMemsetAsync(d_tot, 0, (size_t)(nparts + 1) * 4, eng->stream));
    return;
  }
  const uint32_t nblocks = (uint32_t)((n + kPartChunk - 1) / kPartChunk);
  const uint64_t nh = (uint64_t)nparts * nblocks;
  uint32_t* hist = (uint32_t*)eng->pool->alloc((nh + 1) * 4);
  uint32_t* offs = (uint32_t*)eng->pool->alloc((nh + 1) * 4);
  const size_t smem = (size_t)nparts * 4 * (PART_WARPS + 1);
  CK(cudaMemsetAsync(hist + nh, 0, 4, eng->stream));
  LAUNCH(eng, k_part_count<<<nblocks, 256, (size_t)nparts * 4, eng->stream>>>(in->cols[col], n, nparts, nblocks,
                                                                              hist));
  prim_scan<prims::OpSum, true>(eng, hist, offs, nh + 1);
  DevPartCols pc{};
  pc.ncols = in->ncols;
  for (int c = 0; c < in->ncols; ++c) {
    pc.in[c] = in->cols[c];
    pc.out[c] = out_cols[c];
  }
  LAUNCH(eng, k_part_scatter<<<nblocks, 256, smem, eng->stream>>>(pc, col, n, nparts, nblocks, offs));
  LAUNCH(eng, k_part_totals<<<grid_for(nparts + 1), 256, 0, eng->stream>>>(offs, nparts, nblocks, d_tot));
  // stream-ordered pool: later allocations on this stream run after these kernels
  eng->pool->free(hist);
  eng->pool->free(offs);
}

static void partition_into(const fjg_relation* in, int col, int nparts, int32_t* const* out_cols, uint64_t* counts) {
  fjg_engine* eng = in->eng;
  if (nparts < 1 || nparts > 1024) throw fj::ValidationError("nparts must be 1..1024");
  uint32_t* tot = (uint32_t*)eng->pool->alloc((nparts + 1) * 4);
  partition_async(in, col, nparts, out_cols, tot);
  std::vector<uint32_t> h(nparts + 1);
  CK(cudaMemcpyAsync(h.data(), tot, (nparts + 1) * 4, cudaMemcpyDeviceToHost, eng->stream));
  CK(cudaStreamSynchronize(eng->stream));
  ++eng->syncs;
  for (int d = 0; d < nparts; ++d) counts[d] = h[d + 1] - h[d];
  eng->pool->free(tot);
}

int fjg_relation_partition(const fjg_relation* in, int col, int nparts, fjg_relation** out_rel, uint64_t* counts) {
  return guard([&] {
    ScopedDevice sd(in->eng->device);
    fjg_relation* r = new_relation(in->eng, in->ncols, in->nrows);
    try {
      partition_into(in, col, nparts, r->cols.data(), counts);
    } catch (...) {
      fjg_relation_destroy(r);
      throw;
    }
    *out_rel = r;
  });
}

int fjg_relation_partition_into(const fjg_relation* in, int col, int nparts, int32_t* const* out_dev_cols,
                                uint64_t* counts) {
  return guard([&] {
    ScopedDevice sd(in->eng->device);
    partition_into(in, col, nparts, out_dev_cols, counts);
  });
}

uint64_t fjg_relation_rows(const fjg_relation* rel) { return rel ? rel->nrows : 0; }
int fjg_relation_cols(const fjg_relation* rel) { return rel ? rel->ncols : 0; }
const int32_t* fjg_relation_device_col(const fjg_relation* rel, int col) {
  return (rel && col >= 0 && col < rel->ncols) ? rel->cols[col] : nullptr;
}

int fjg_relation_download(const fjg_relation* rel, int col, int32_t* host_out) {
  return guard([&] {
    ScopedDevice sd(rel->eng->device);
    if (col < 0 || col >= rel->ncols) throw fj::ValidationError("column out of range");
    if (rel->nrows)
      CK(cudaMemcpyAsync(host_out, rel->cols[col], rel->nrows * 4, cudaMemcpyDeviceToHost, rel->eng->stream));
    CK(cudaStreamSynchronize(rel->eng->stream));
  });
}

void fjg_relation_destroy(fjg_relation* rel) {
  if (!rel) return;
  ScopedDevice sd(rel->eng->device);
  cudaStreamSynchronize(rel->eng->stream);
  for (void* p : rel->owned) rel->eng->pool->free(p);
  delete rel;
}

int fjg_query_create(fjg_engine* eng, const char* query_json, const char* plan_json, fjg_relation* const* atom_rels,
                     int natoms, fjg_query** out) {
  return guard([&] {
    ScopedDevice sd(eng->device);
    auto q = std::make_unique<fjg_query>();
    q->eng = eng;
    auto qv = fj::json::parse(query_json);
    auto query = fj::query_from_json(qv);
    if ((int)query.size() != natoms)
      throw fj::ValidationError("query has " + std::to_string(query.size()) + " atoms but " +
                                std::to_string(natoms) + " relations were bound");
    q->plan = fj::plan_from_json(fj::json::parse(plan_json), query);
    if (const fj::json::Value* hv = qv.is_object() ? qv.find("head") : nullptr)
      for (auto& x : hv->arr) q->head_override.push_back(x.str);
    std::string err = fj::validate(q->plan);
    if (!err.empty()) throw fj::ValidationError("invalid plan: " + err);
    for (int a = 0; a < natoms; ++a) {
      if (!atom_rels[a]) throw fj::ValidationError("null relation bound to atom");
      if (atom_rels[a]->eng != eng) throw fj::ValidationError("relation belongs to another engine");
      q->rels.push_back(atom_rels[a]);
    }
    prepare_query(q.get());
    *out = q.release();
  });
}

int fjg_execute(fjg_query* q, const fjg_exec_options* opts, fjg_result* out) {
  return guard([&] {
    fjg_engine* eng = q->eng;
    ScopedDevice sd(eng->device);
    fjg_exec_options o{};
    o.dynamic_cover = 1;
    o.min_var = -1;
    if (opts) o = *opts;
    if (o.min_var >= (int)q->head.size()) throw fj::ValidationError("min_var out of range");
    // engine default: 2^25 candidates per node launch, up to 2^27 for large inputs (8 x the largest relation):
    // larger frontier batches give the probe-region ordering of the last node more bindings per region
    // (C5 1025 -> 994 ms, C4 103.3 -> 99.7 ms at 2^27; 2^28 and up: equal) at 49 B of frontier per entry
    // and node. Factorised-count mode keeps 2^25 (the memoised chain count's frontier is one node deep).
    uint64_t batch = o.batch_size;
    if (!batch) {
      batch = 1ull << 25;
      if (o.output_mode != FJG_OUT_FACTORIZED_COUNT)
        // (while the frontier buffers of all nodes stay under 32 GiB: wide or deep plans keep smaller batches)
        while (batch < 8 * q->max_n && batch < (1ull << 27) && 2 * batch * frontier_entry_bytes(q) <= (32ull << 30))
          batch <<= 1;
    }
    if (batch > kLastChunk) throw fj::ValidationError("batch_size must be <= " + std::to_string(kLastChunk));
    ensure_frontiers(q, batch);
    q->dynamic = o.dynamic_cover != 0;
    q->timing = o.collect_timing != 0;
    q->batch = batch;
    q->min_var = o.min_var;
    if (o.backend < FJG_BACKEND_COLT || o.backend > FJG_BACKEND_SIMPLE)
      throw fj::ValidationError("backend must be colt(0), slt(1) or simple(2)");
    q->backend = o.backend;
    const uint32_t l0 = eng->launches, s0 = eng->syncs;
    const bool memo = o.output_mode == FJG_OUT_FACTORIZED_COUNT && q->chain_start >= 1;
    if (o.output_mode == FJG_OUT_ENUMERATE) {
      // one pass writes the tuples and folds count / checksum / MIN; the buffer
      // keeps its capacity across executions, and a pass that outgrows it is
      // rerun once with the exact size (SPEC.md:449 collector sink)
      const size_t nh = std::max<size_t>(q->head.size(), 1);
      auto ensure_out = [&](uint64_t rows) {
        if (rows > (1ull << 34) / nh) throw fj::ResourceError("enumerated output too large to materialise");
        if (q->out_cap >= rows && q->out_tuples) return;
        q->out_tuples = (int32_t*)q->alloc(std::max<uint64_t>(rows, 1) * nh * 4);
        q->out_cap = rows;
      };
      if (!q->out_tuples) ensure_out(std::min<uint64_t>(std::max<uint64_t>(2 * q->max_n, 1024), 1ull << 26));
      execute_once(q, EXPAND_ENUM);
      if (q->h_ctr->count_hi) throw fj::ResourceError("enumerated output too large to materialise");
      if (q->h_ctr->out_rows > q->out_cap) {
        ensure_out(q->h_ctr->out_rows);
        execute_once(q, EXPAND_ENUM);
      }
      q->out_rows = q->h_ctr->out_rows;
      if (q->out_rows != q->h_ctr->count_lo) throw fj::EngineError("enumerated rows disagree with the count");
    } else {
      execute_once(q, memo ? EXPAND_MEMO : EXPAND_COUNT);
    }
    const DevCounters& H = *q->h_ctr;
    fjg_result r{};
    r.count_lo = H.count_lo;
    r.count_hi = H.count_hi;
    r.checksum = H.checksum;
    r.has_min = (o.min_var >= 0 && H.minv != LLONG_MAX) ? 1 : 0;
    r.min_value = r.has_min ? H.minv : 0;
    r.num_nodes = (int)q->nodes.size();
    r.output_rows = (o.output_mode == FJG_OUT_ENUMERATE) ? q->out_rows : 0;
    r.probes = H.probes;
    r.probe_misses = H.misses;
    for (int k = 0; k < MAXN && k < FJG_MAX_NODES; ++k) {
      r.node_body_entries[k] = H.body[k];
      r.node_probes[k] = H.node_probes[k];
      r.node_inputs[k] = q->node_inputs[k] + H.tail_inputs[k];
    }
    r.maps_built = q->maps_built;
    r.keys_inserted = H.keys_inserted;
    r.forces = q->forces;
    r.rows_forced = q->rows_forced;
    r.build_ms = q->build_ms;
    r.join_ms = q->join_ms;
    r.last_node_ms = q->last_ms;
    r.last_node_launches = q->last_launches;
    r.last_node_candidates = q->last_candidates;
    r.first_node_ms = q->first_ms;
    r.memo_ms = q->phase_ms[4];
    r.memo_rows_resolved = q->memo_rows[0];
    r.memo_rows_gathered = q->memo_rows[1];
    r.memo_rows_init = q->memo_rows[2];
    for (size_t a = 0; a < q->atoms.size() && a < FJG_MAX_ATOMS; ++a) {
      const int t = q->atoms[a].trie;
      r.atom_maps_built[a] = (t >= 0 && t < MAXA) ? q->trie_maps[t] : 0;
      r.atom_levels_forced[a] = (t >= 0 && t < MAXA) ? q->trie_levels[t] : 0;
    }
    r.kernel_launches = eng->launches - l0;
    r.host_syncs = eng->syncs - s0;
    *out = r;
  });
}

int fjg_query_output(fjg_query* q, int32_t* host_out, uint64_t cap_rows, uint64_t* rows) {
  return guard([&] {
    ScopedDevice sd(q->eng->device);
    const uint64_t n = std::min(cap_rows, q->out_rows);
    if (n) CK(cudaMemcpyAsync(host_out, q->out_tuples, n * q->head.size() * 4, cudaMemcpyDeviceToHost, q->eng->stream));
    CK(cudaStreamSynchronize(q->eng->stream));
    *rows = n;
  });
}

int fjg_query_num_head_vars(const fjg_query* q) { return q ? (int)q->head.size() : 0; }

// Device-resident materialisation of the enumerated output (run_segments,
// SPEC.md:414-422): a new columnar relation, one column per head variable.
int fjg_query_output_relation(fjg_query* q, fjg_relation** out) {
  return guard([&] {
    fjg_engine* eng = q->eng;
    ScopedDevice sd(eng->device);
    const int nv = (int)q->head.size();
    if (nv > MAXC) throw fj::ResourceError("materialised segment has more than 8 variables");
    fjg_relation* r = new_relation(eng, nv, q->out_rows);
    if (q->out_rows) {
      DevPartCols pc{};
      pc.ncols = nv;
      for (int c = 0; c < nv; ++c) pc.out[c] = r->cols[c];
      LAUNCH(eng, k_transpose_rows<<<grid_for(q->out_rows), 256, 0, eng->stream>>>(q->out_tuples, q->out_rows, pc));
    }
    CK(cudaStreamSynchronize(eng->stream));
    *out = r;
  });
}

void fjg_query_destroy(fjg_query* q) {
  if (!q) return;
  ScopedDevice sd(q->eng->device);
  cudaStreamSynchronize(q->eng->stream);
  delete q;
}

int fjg_device_tuple_hash(fjg_engine* eng, const int64_t* host_vals, int arity, uint64_t ntuples, uint64_t* host_out) {
  return guard([&] {
    ScopedDevice sd(eng->device);
    if (ntuples == 0) return;
    const size_t vb = std::max<size_t>((size_t)arity * ntuples * 8, 8);
    int64_t* dv = (int64_t*)eng->pool->alloc(vb);
    uint64_t* dout = (uint64_t*)eng->pool->alloc(ntuples * 8);
    if (arity) CK(cudaMemcpyAsync(dv, host_vals, (size_t)arity * ntuples * 8, cudaMemcpyHostToDevice, eng->stream));
    LAUNCH(eng, k_tuple_hash<<<grid_for(ntuples), 256, 0, eng->stream>>>(dv, arity, ntuples, dout));
    CK(cudaMemcpyAsync(host_out, dout, ntuples * 8, cudaMemcpyDeviceToHost, eng->stream));
    CK(cudaStreamSynchronize(eng->stream));
    eng->pool->free(dv);
    eng->pool->free(dout);
  });
}

// Test hook: run one device-wide primitive (kernels/prims.cuh) on seeded
// host-generated data and count the elements that differ from a host
// restatement (std::stable_sort / sequential scans).
int fjg_device_primitive_check(fjg_engine* eng, int which, uint64_t n, int lo, int hi, uint64_t seed,
                               uint64_t* mismatches) {
  return guard([&] {
    ScopedDevice sd(eng->device);
    if (which < 0 || which > 4) throw fj::ValidationError("primitive must be 0..4");
    if (lo < 0 || hi > 32 || lo > hi) throw fj::ValidationError("bit range must satisfy 0 <= lo <= hi <= 32");
    uint64_t x = seed * 0x9e3779b97f4a7c15ull + 1;
    auto next = [&]() {
      x += 0x9e3779b97f4a7c15ull;
      uint64_t z = x;
      z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
      z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
      return z ^ (z >> 31);
    };
    const size_t nb = std::max<uint64_t>(n, 1);
    uint64_t bad = 0;
    if (which == 0) {  // radix sort of (key, index) pairs on bits [lo, hi), skewed keys
      std::vector<uint32_t> k(n), v(n);
      const uint64_t km = hi == 32 ? 0xffffffffull : ((1ull << hi) - 1);
      for (uint64_t i = 0; i < n; ++i) {
        const uint64_t r = next();
        k[i] = (uint32_t)(((r & 3) == 0 ? (r >> 8) % 7 : (r >> 8)) & km);  // a quarter of the keys on 7 values
        v[i] = (uint32_t)i;
      }
      uint32_t* d = (uint32_t*)eng->pool->alloc(nb * 16);
      CK(cudaMemcpyAsync(d, k.data(), n * 4, cudaMemcpyHostToDevice, eng->stream));
      CK(cudaMemcpyAsync(d + nb, v.data(), n * 4, cudaMemcpyHostToDevice, eng->stream));
      const int r = prim_sort_pairs(eng, d, d + nb, d + 2 * nb, d + 3 * nb, n, lo, hi);
      std::vector<uint32_t> gk(n), gv(n);
      CK(cudaMemcpyAsync(gk.data(), d + 2 * nb * r, n * 4, cudaMemcpyDeviceToHost, eng->stream));
      CK(cudaMemcpyAsync(gv.data(), d + nb + 2 * nb * r, n * 4, cudaMemcpyDeviceToHost, eng->stream));
      CK(cudaStreamSynchronize(eng->stream));
      eng->pool->free(d);
      const uint64_t dm = (hi - lo == 32) ? 0xffffffffull : (((1ull << (hi - lo)) - 1) << lo);
      std::vector<uint32_t> idx(n);
      for (uint64_t i = 0; i < n; ++i) idx[i] = (uint32_t)i;
      std::stable_sort(idx.begin(), idx.end(), [&](uint32_t a, uint32_t b) { return (k[a] & dm) < (k[b] & dm); });
      for (uint64_t i = 0; i < n; ++i) bad += (gk[i] != k[idx[i]] || gv[i] != v[idx[i]]) ? 1 : 0;
    } else if (which == 1) {  // inclusive sum of u64 (large values), total
      std::vector<uint64_t> a(n), g(n);
      for (uint64_t i = 0; i < n; ++i) a[i] = next() >> 20;
      uint64_t* d = (uint64_t*)eng->pool->alloc(nb * 8 + 8);
      CK(cudaMemcpyAsync(d, a.data(), n * 8, cudaMemcpyHostToDevice, eng->stream));
      prim_scan<prims::OpSum, false>(eng, d, d, n, d + nb);
      uint64_t tot = 0;
      CK(cudaMemcpyAsync(g.data(), d, n * 8, cudaMemcpyDeviceToHost, eng->stream));
      CK(cudaMemcpyAsync(&tot, d + nb, 8, cudaMemcpyDeviceToHost, eng->stream));
      CK(cudaStreamSynchronize(eng->stream));
      eng->pool->free(d);
      uint64_t run = 0;
      for (uint64_t i = 0; i < n; ++i) {
        run += a[i];
        bad += g[i] != run ? 1 : 0;
      }
      bad += tot != run ? 1 : 0;
    } else if (which == 2 || which == 4) {  // inclusive max-scan / exclusive sum of u32
      std::vector<uint32_t> a(n), g(n);
      for (uint64_t i = 0; i < n; ++i) a[i] = which == 2 ? ((next() & 7) == 0 ? (uint32_t)i : 0u) : (uint32_t)(next() & 15);
      uint32_t* d = (uint32_t*)eng->pool->alloc(nb * 8 + 8);
      CK(cudaMemcpyAsync(d, a.data(), n * 4, cudaMemcpyHostToDevice, eng->stream));
      if (which == 2)
        prim_scan<prims::OpMax, false>(eng, d, d + nb, n);
      else
        prim_scan<prims::OpSum, true>(eng, d, d + nb, n);
      CK(cudaMemcpyAsync(g.data(), d + nb, n * 4, cudaMemcpyDeviceToHost, eng->stream));
      CK(cudaStreamSynchronize(eng->stream));
      eng->pool->free(d);
      uint32_t run = 0;
      for (uint64_t i = 0; i < n; ++i) {
        if (which == 4) {
          bad += g[i] != run ? 1 : 0;
          run += a[i];
        } else {
          run = std::max(run, a[i]);
          bad += g[i] != run ? 1 : 0;
        }
      }
    } else {  // flagged selection of indices
      std::vector<uint8_t> f(n);
      for (uint64_t i = 0; i < n; ++i) f[i] = (next() % 5) == 0 ? (uint8_t)(1 + (i & 7)) : 0;
      uint8_t* df = (uint8_t*)eng->pool->alloc(nb);
      uint32_t* d = (uint32_t*)eng->pool->alloc(nb * 4 + 4);
      CK(cudaMemcpyAsync(df, f.data(), n, cudaMemcpyHostToDevice, eng->stream));
      prim_select_flagged(eng, df, d, n, d + nb);
      std::vector<uint32_t> g(n);
      uint32_t cnt = 0;
      CK(cudaMemcpyAsync(&cnt, d + nb, 4, cudaMemcpyDeviceToHost, eng->stream));
      CK(cudaStreamSynchronize(eng->stream));
      if (cnt <= n) CK(cudaMemcpy(g.data(), d, (size_t)cnt * 4, cudaMemcpyDeviceToHost));
      eng->pool->free(df);
      eng->pool->free(d);
      uint64_t j = 0;
      for (uint64_t i = 0; i < n; ++i)
        if (f[i]) {
          bad += (j >= cnt || g[j] != i) ? 1 : 0;
          ++j;
        }
      bad += j != cnt ? 1 : 0;
    }
    *mismatches = bad;
  });
}

}  // extern "C"

#include "multi.cuh"
#include "colt_api.cuh"
