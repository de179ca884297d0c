// Device-side data layout of the B200 Free Join executor.
//
// COLT on the device (reference: Fig 12)
// ---------------------------------------------------------------------------
// A *physical trie* is one relation plus the list of key-column groups per
// level. Atoms over the same relation with the same level key columns (renamed
// self-joins) share one physical trie: COLT is a
// deterministic function of (relation, schema), so sharing is invisible.
//
// Subtries are identified by *positions*. The root (depth 0) is the BaseScan of
// rows [0, n) (zero work at `new`). Forcing level l of a subtrie
// whose offsets occupy positions [p, p+len) of domain l-1 regroups exactly
// those positions in domain l, children contiguous: child groups are
// sub-ranges [q, q+cnt) of [p, p+len), and a child's id is its start q. So
//   - no offset vectors are allocated per node and no ids are handed out;
//   - a level holds n-sized arrays indexed by position.
// Instead of row offsets, forcing scatters the *column values* every deeper
// level will read ("clustered columns", cval), so cover iteration streams
// coalesced values instead of gathering through offsets.
//
// Per level l (l >= 0), with n = relation rows:
//   table   open-addressing hash map (parent p, key) -> child (q, cnt);
//           16-byte slots, linear probing, capacity pow2 >= 2n (load <= 0.5)
//   sn      per subtrie id: {state: 0 unforced, 1 claimed for forcing, 2 forced;
//           nkeys: distinct keys once forced (estimated_key_count)}
//   cursor  per subtrie id: child-range allocation cursor (force only)
//   cnt     per position of domain l: child length at a child start, else 0
//   cval[c] per position of domain l: column c (every column used at levels >= l)
#pragma once

#include <cstdint>

#include "fj_hash.hpp"

namespace fjg {

constexpr int MAXV = 16;  // variables per query
constexpr int MAXA = 16;  // atoms per query
constexpr int MAXS = 12;  // subatoms per node
constexpr int MAXK = 6;   // vars per subatom (key arity)
constexpr int MAXC = 8;   // columns per relation
constexpr int MAXL = 8;   // levels per physical trie
constexpr int MAXT = 16;  // physical tries per query
constexpr int MAXN = 32;  // plan nodes

constexpr uint32_t kEmpty = 0xFFFFFFFFu;
constexpr uint64_t kEmpty64 = 0xFFFFFFFFFFFFFFFFull;
constexpr uint32_t kSingleton = 0xFFFFFFFFu;  // streamed row: residual subtrie is [row]

// Hash map slots. A forced subtrie occupying positions [p, p+len) owns the
// slot region [4p, 4p+4len) of its level's 4n-slot array: len buckets of 4
// slots, one 32-byte sector each (load <= 0.25). Regions of distinct subtries
// are disjoint, so no parent id is needed in the key, the probes of one
// binding stay inside one compact region, a probe is almost always one
// sector, and forcing a subtrie clears exactly its own region (no per-query
// table reset). The child length lives in cnt[q] (read on hits only).
struct __align__(8) Slot {
  uint32_t k;  // key word: the int32 key (arity 1), 0 (arity 0) or a 32-bit tuple hash
  uint32_t q;  // child start (kEmpty: free; kPendBit|count while the force is inserting)
};
constexpr uint32_t kPendBit = 0x80000000u;  // positions are < 2^31

// Per subtrie id: its state (0 unforced, 1 claimed for forcing, 2 forced) and,
// once forced, its number of distinct keys (estimated_key_count). One 8-byte
// record, so k_select's random read of a subtrie costs one sector, not two.
struct __align__(8) SubState {
  uint32_t state;
  uint32_t nkeys;
};

struct DevLevel {
  Slot* table;       // 4n slots
  uint32_t* srep;    // arity >= 2 only, per slot: representative position + 1 during insertion
  SubState* sn;  // per subtrie id: {state, key count}
  uint32_t* cursor;
  uint32_t* cnt;
  int32_t* cval[MAXC];
  int nk;
  int keycol[MAXK];
  uint32_t* list_p;    // subtries claimed for forcing
  uint32_t* list_len;
  uint32_t* list_scan;
};

struct DevTrie {
  uint32_t n;
  int ncols;
  int nlev;
  const int32_t* base[MAXC];
  DevLevel lev[MAXL];
};

struct DevSub {
  int atom;
  int trie;
  int depth;       // COLT level this subatom reads (= # earlier subatoms of its atom)
  int nv;
  int var[MAXK];
  int col[MAXK];
  int bound_mask;  // bit t: var[t] already bound at node entry (checked when iterated)
  int stream;      // vars are all remaining vars of the atom (Fig 12 is_suffix)
  int last;        // last subatom of its atom
};

struct DevFrontier {
  int32_t* var[MAXV];
  uint32_t* p[MAXA];
  uint32_t* len[MAXA];
  uint64_t* mult;
};

struct DevNode {
  int k;
  int nsub;
  int ncov;
  int is_last;
  int cov[MAXS];
  DevSub sub[MAXS];
  uint32_t in_vars;    // bitmask of variables bound at node entry (avs)
  uint32_t out_vars;   // bitmask bound after the node
  uint32_t in_atoms;   // atoms with a subtrie slot at node entry
  uint32_t out_atoms;  // atoms with a subtrie slot after the node
  uint32_t atom_n[MAXA];
  int nhead;
  DevFrontier in, out;
  uint8_t* chosen;     // per entry: chosen cover (subatom index)
  uint64_t* m;         // per entry: candidates
  uint64_t* scan;      // inclusive scan of m
};

// Kernel-side plan of one subatom, every pointer resolved on the host, passed
// in the constant bank (__grid_constant__ KNode) so the per-candidate code
// reads no descriptors from memory.
struct KSub {
  const int32_t* src[MAXK];   // cover iteration values per var (stream: domain depth-1; keys: cval of depth)
  const int32_t* kcmp[MAXK];  // probe key compare for arity >= 2: cval of depth at the child start
  const uint32_t* cnt;        // cnt of depth (keys-mode iteration)
  const Slot* table;          // slots of depth
  const SubState* sn;         // {state, key count} of depth's subtries (estimated_key_count, claims)
  const uint32_t* in_p;       // frontier subtrie column of this atom (null: root)
  const uint32_t* in_len;
  uint32_t root_n;
  const uint32_t* rregion;    // root probe region (DevCounters::root_region[trie])
  const uint32_t* ldup;       // DevCounters::level_dup of this level: 0 = every child count is 1
  int8_t var[MAXK];
  uint8_t nv, bound_mask, stream, last, atom, trie, depth, pad;
};

struct KNode {
  int k, nsub, ncov, nhead, is_last;
  int8_t cov[MAXS];
  uint32_t in_vars, out_vars, in_atoms, out_atoms;
  const int32_t* in_var[MAXV];
  int32_t* out_var[MAXV];
  const uint32_t* in_p[MAXA];
  const uint32_t* in_len[MAXA];
  uint32_t* out_p[MAXA];
  uint32_t* out_len[MAXA];
  const uint64_t* in_mult;
  uint64_t* out_mult;
  uint8_t* chosen;
  uint64_t* m;
  uint64_t* scan;
  const unsigned long long* memo;  // memoised chain count per level-0 group (u128 as lo,hi), or null
  const uint32_t* memo_gid;        // group index + 1 of every level-0 position of memo_atom's trie
  int memo_atom;                   // atom whose child subtrie indexes `memo`
  KSub sub[MAXS];
};

// One bottom-up pass of the memoised chain count: for every
// row of the carrier trie's level-0 domain, the fresh atoms' roots are probed
// with the row's values (k_memo_resolve: the continuing atom's child group and
// the product of the other atoms' leaf lengths, cached per row and shared by
// every pass with the same carrier and fresh atoms), then k_memo_gather adds
// coef * memo_next[child] into the row's group. Groups are numbered densely
// (gid = inclusive count of group starts), so memo arrays hold one u128 per
// level-0 key.
struct MemoPass {
  uint64_t n;
  const uint32_t* gid;         // group index + 1 of every level-0 position (carrier trie)
  const uint32_t* cnt;         // carrier trie level-0 cnt (nonzero at group starts)
  const int32_t* cvals[MAXK];  // carrier's variables at level-0 positions
  int cnv;
  int nfresh;
  int cont_x;                  // index of the fresh atom continuing the chain, or -1
  int has_coef;                // some fresh atom is a leaf (its length multiplies)
  int cont[MAXS];              // fresh atom continues the chain (uses memo_next)
  int8_t cpos[MAXS][MAXK];     // key var t of fresh x = carrier var cpos[x][t]
  KSub fresh[MAXS];
  const uint32_t* gid_next;    // gid of the continuing atom's trie
  uint32_t* child;             // per row: gid of the continuing atom's child, or kMemoMiss
  const uint32_t* direct;      // dense key -> gid map of the continuing atom's sorted root (or null)
  uint32_t direct_n;           // its size (keys are 0 .. direct_n - 1)
  uint64_t* coef;              // per row: product of leaf lengths (has_coef), 0 on a miss
  const unsigned long long* memo_next;
  unsigned long long* memo_out;
};
constexpr uint32_t kMemoMiss = 0xffffffffu;

// Group initialisation of every memo array over one trie's level-0 groups
// (one pass over cnt / gid instead of one per chain node) and, for a sorted
// root whose keys are small non-negative ints, its dense key -> group map.
constexpr int kMemoInitMax = 8;
struct MemoInit {
  uint64_t n;
  const uint32_t* gid;
  const uint32_t* cnt;
  const int32_t* key;          // clustered level-0 key column (for `dense`), or null
  uint32_t* dense;             // key -> group index, or null
  uint32_t dense_n;
  int nout;
  unsigned long long* out[kMemoInitMax];
  int group_size[kMemoInitMax];  // 1: write the group size (pass without fresh atoms), 0: zero
};

struct DevCounters {
  uint64_t count_lo, count_hi, checksum;
  long long minv;
  uint64_t probes, misses;
  uint64_t body[MAXN];
  uint64_t node_probes[MAXN];
  uint64_t keys_inserted;
  uint64_t out_rows;
  uint64_t total_m;
  uint32_t survivors;
  uint32_t newslots;
  uint32_t dup;  // the running force met a repeated key (else every child is a single row)
  uint32_t list_count[MAXT * MAXL];
  uint32_t root_need[MAXT];
  uint32_t list_total[MAXT * MAXL];  // offsets of the claimed subtries (sum of their lengths)
  uint32_t root_region[MAXT];  // buckets of each trie's root slot region (rows, or distinct keys once sorted)
  uint32_t level_dup[MAXT * MAXL];  // some force of (trie, level) met a repeated key: child counts can exceed 1
  uint64_t tail_inputs[MAXN];  // node inputs counted on the device (fused Cartesian tail nodes)
  unsigned long long ticket;   // last-node chunk tickets (FJG_GJ_TICKET)
  uint32_t fnew[MAXT];         // per member of a force batch: new keys (slots claimed)
  uint32_t fdup[MAXT];         // per member of a force batch: a repeated key was met
  uint32_t fopt[MAXT];         // per member of a force batch: inserted optimistically (every key expected distinct)
};

// Fused Cartesian tail (nodes k..K-1 each one stream-iterated subatom binding
// only fresh variables: SPEC.md:423-431's pure Cartesian suffix): every
// binding of node k's frontier expands to the product of its tail subtries.
constexpr int MAXTAIL = 4;
struct TailPlan {
  int ntail;
  int node[MAXTAIL];           // plan node of tail subatom j
  int open[MAXTAIL];           // atom has a subtrie in node k's frontier (else: its root, depth 0)
  const uint32_t* in_p[MAXTAIL];
  const uint32_t* in_len[MAXTAIL];
  KSub sub[MAXTAIL];
};

}  // namespace fjg
