// ============================================================================
// ORACLE — TEST INFRASTRUCTURE ONLY.
// CPU restatement of the reference's Free Join path, used as the parity
// checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs. Never linked into or called by the product path
// (paper_2301_10841_b200/, libfjg.so).
//
// Parity pinning: the reference ships no executable path, so
// the restatement follows the reference's specification and paper:
//   data model   SPEC.md:17-93, proj/include/fj/value.hpp:25-67
//   trie         SPEC.md:263-361, Fig 5, Fig 12
//   executor     SPEC.md:363-455, Fig 8, Fig 13 PAPER.md:1269-1281,
//                dynamic cover PAPER.md:1323-1347
// TupleHash is pinned against the reference header itself (oracle/_ref,
// tests/golden/tuplehash_kats.json); plan transformations against the SPEC's
// worked examples (tests/test_plan_goldens.py); executor semantics against a
// brute-force nested-loop join and SPEC acceptance 1-8.
// Self-contained: shares no code with the product.
// ============================================================================
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

namespace orc {

// ---------------------------------------------------------------- values ----
// value.hpp:49-53: Int hash = std::hash<int64_t> (identity in libstdc++) ^ 0.
static inline uint64_t value_hash(int64_t v) { return static_cast<uint64_t>(v); }
// value.hpp:61-67 TupleHash.
static inline uint64_t tuple_hash(const int64_t* v, int n) {
  uint64_t h = 0x811c9dc5ULL;
  for (int i = 0; i < n; ++i) h = (h ^ value_hash(v[i])) * 0x100000001b3ULL;
  return h;
}
static inline uint64_t fmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33;
  return k;
}
static inline uint32_t partition_of(int64_t v, uint32_t nparts) {
  return static_cast<uint32_t>(fmix64(static_cast<uint64_t>(v) ^ 0x5bd1e995ULL) % nparts);
}

// ------------------------------------------------------------------ json ----
struct J {
  enum K { Null, Num, Str, Arr, Obj } k = Null;
  double num = 0;
  std::string s;
  std::vector<J> a;
  std::vector<std::pair<std::string, J>> o;
  const J& at(const std::string& key) const {
    for (auto& kv : o)
      if (kv.first == key) return kv.second;
    throw std::runtime_error("oracle json: missing key " + key);
  }
  const J* find(const std::string& key) const {
    for (auto& kv : o)
      if (kv.first == key) return &kv.second;
    return nullptr;
  }
};
struct JP {
  const std::string& s;
  size_t i = 0;
  void ws() {
    while (i < s.size() && isspace((unsigned char)s[i])) ++i;
  }
  J val() {
    ws();
    J v;
    if (s[i] == '[') {
      v.k = J::Arr;
      ++i;
      ws();
      if (s[i] == ']') {
        ++i;
        return v;
      }
      while (true) {
        v.a.push_back(val());
        ws();
        if (s[i++] == ']') break;
      }
    } else if (s[i] == '{') {
      v.k = J::Obj;
      ++i;
      ws();
      if (s[i] == '}') {
        ++i;
        return v;
      }
      while (true) {
        ws();
        std::string key = str();
        ws();
        ++i;  // ':'
        v.o.emplace_back(key, val());
        ws();
        if (s[i++] == '}') break;
      }
    } else if (s[i] == '"') {
      v.k = J::Str;
      v.s = str();
    } else if (s.compare(i, 4, "null") == 0) {
      i += 4;
    } else {
      size_t st = i;
      while (i < s.size() && (isdigit((unsigned char)s[i]) || s[i] == '-' || s[i] == '.' || s[i] == 'e' || s[i] == '+'))
        ++i;
      v.k = J::Num;
      v.num = std::stod(s.substr(st, i - st));
    }
    return v;
  }
  std::string str() {
    ++i;
    std::string out;
    while (s[i] != '"') {
      if (s[i] == '\\') ++i;
      out += s[i++];
    }
    ++i;
    return out;
  }
};
static J parse(const std::string& s) {
  JP p{s};
  return p.val();
}

// ------------------------------------------------------------- relations ----
// immutable columnar relation; row offset i = row i.
struct Relation {
  std::vector<const int32_t*> cols;
  uint64_t n = 0;
  int64_t at(int c, uint64_t i) const { return cols[c][i]; }
};

// ------------------------------------------------------------------- keys ---
constexpr int MAXK = 8;
struct Key {
  int64_t v[MAXK];
  int n = 0;
  bool operator==(const Key& o) const {
    if (n != o.n) return false;
    for (int i = 0; i < n; ++i)
      if (v[i] != o.v[i]) return false;
    return true;
  }
};
struct KeyHash {
  size_t operator()(const Key& k) const { return fmix64(tuple_hash(k.v, k.n)); }
};

// Flat open-addressing map Key -> Node* (the HashMap<Tuple, COLT> of Fig 12),
// insertion-ordered entries, linear probing on a power-of-two index.
struct Node;
struct FlatMap {
  std::vector<uint64_t> hs;   // per index slot: 0 empty, else entry+1 in low 32 bits, hash tag high
  std::vector<Key> keys;
  std::vector<Node*> vals;
  uint64_t mask = 0;
  size_t size() const { return keys.size(); }
  void reserve(size_t n) {
    uint64_t cap = 16;
    while (cap < 2 * n) cap <<= 1;
    if (cap > mask + 1) rehash(cap);
  }
  void rehash(uint64_t cap) {
    hs.assign(cap, 0);
    mask = cap - 1;
    for (size_t e = 0; e < keys.size(); ++e) place(KeyHash()(keys[e]), e);
  }
  void place(uint64_t h, size_t e) {
    uint64_t i = h & mask;
    while (hs[i]) i = (i + 1) & mask;
    hs[i] = ((h >> 32) << 32) | (uint64_t)(e + 1);
  }
  Node* find(const Key& k) const {
    if (keys.empty()) return nullptr;
    const uint64_t h = KeyHash()(k);
    uint64_t i = h & mask;
    while (hs[i]) {
      const uint64_t e = (hs[i] & 0xffffffffULL) - 1;
      if ((hs[i] >> 32) == (h >> 32) && keys[e] == k) return vals[e];
      i = (i + 1) & mask;
    }
    return nullptr;
  }
  // returns the slot for k, inserting a null value if absent
  Node*& get_or_insert(const Key& k, bool& inserted) {
    if (2 * (keys.size() + 1) > mask + 1) rehash(std::max<uint64_t>(16, 2 * (mask + 1)));
    const uint64_t h = KeyHash()(k);
    uint64_t i = h & mask;
    while (hs[i]) {
      const uint64_t e = (hs[i] & 0xffffffffULL) - 1;
      if ((hs[i] >> 32) == (h >> 32) && keys[e] == k) {
        inserted = false;
        return vals[e];
      }
      i = (i + 1) & mask;
    }
    keys.push_back(k);
    vals.push_back(nullptr);
    hs[i] = ((h >> 32) << 32) | (uint64_t)keys.size();
    inserted = true;
    return vals.back();
  }
  void swap(FlatMap& o) {
    hs.swap(o.hs);
    keys.swap(o.keys);
    vals.swap(o.vals);
    std::swap(mask, o.mask);
  }
};

// ------------------------------------------------------------------ COLT ----
enum Backend { SIMPLE = 0, SLT = 1, COLT = 2 };

struct TrieStats {
  uint64_t maps_built = 0, keys_inserted = 0, forces = 0;
  uint32_t level_mask = 0;  // bit l: some map was built at schema level l
};

// NodeBody: Map | Vec (row offsets) | BaseScan.
struct Node {
  enum Kind : uint8_t { BaseScan, Vec, Map } kind = Vec;
  int32_t level = 0;                // schema level this node keys on
  uint32_t n = 0;                   // Vec: number of offsets
  const uint32_t* offs = nullptr;   // Vec: offsets (slice of the trie's offset arena)
  std::unique_ptr<FlatMap> map;     // Map
  uint64_t rows = 0;                // offsets under this node
};

struct Colt {
  const Relation* rel = nullptr;
  std::vector<std::vector<int>> levels;  // key columns per level (one per subatom)
  bool trailing_empty = false;
  Backend backend = COLT;
  Node root;
  std::deque<Node> nodes;                              // stable child nodes
  std::vector<std::unique_ptr<uint32_t[]>> offs_arena;  // child offset vectors, one block per force
  TrieStats stats;

  uint64_t length(const Node& nd) const {
    return nd.kind == Node::BaseScan ? rel->n : nd.kind == Node::Vec ? nd.n : nd.rows;
  }
  // estimated_key_count: never forces.
  uint64_t estimated_key_count(const Node& nd) const {
    if (nd.kind == Node::Map) return nd.map->size();
    return length(nd);
  }
  Key key_at(int level, uint64_t row) const {
    Key k;
    k.n = (int)levels[level].size();
    for (int t = 0; t < k.n; ++t) k.v[t] = rel->at(levels[level][t], row);
    return k;
  }
  // force (Fig 12 `force`): group offsets by key; idempotent.
  void force(Node& nd) {
    if (nd.kind == Node::Map) return;
    const uint64_t len = length(nd);
    auto off_at = [&](uint64_t i) -> uint32_t { return nd.kind == Node::BaseScan ? (uint32_t)i : nd.offs[i]; };
    auto m = std::make_unique<FlatMap>();
    m->reserve(std::min<uint64_t>(len, 1u << 16));
    // pass 1: key -> child index, child sizes
    std::vector<uint32_t> which(len);
    std::vector<uint32_t> counts;
    for (uint64_t i = 0; i < len; ++i) {
      bool ins;
      Node*& slot = m->get_or_insert(key_at(nd.level, off_at(i)), ins);
      if (ins) {
        slot = reinterpret_cast<Node*>((uintptr_t)counts.size());
        counts.push_back(0);
      }
      const uint32_t c = (uint32_t)(uintptr_t)slot;
      which[i] = c;
      ++counts[c];
    }
    // pass 2: group offsets by child into one arena block
    std::unique_ptr<uint32_t[]> block(new uint32_t[std::max<uint64_t>(len, 1)]);
    std::vector<uint64_t> start(counts.size() + 1, 0);
    for (size_t c = 0; c < counts.size(); ++c) start[c + 1] = start[c] + counts[c];
    std::vector<uint64_t> cur(start.begin(), start.end() - 1);
    for (uint64_t i = 0; i < len; ++i) block[cur[which[i]]++] = off_at(i);
    for (size_t c = 0; c < counts.size(); ++c) {
      nodes.emplace_back();
      Node& ch = nodes.back();
      ch.kind = Node::Vec;
      ch.level = nd.level + 1;
      ch.offs = block.get() + start[c];
      ch.n = counts[c];
      ch.rows = counts[c];
      m->vals[c] = &ch;
    }
    offs_arena.push_back(std::move(block));
    nd.kind = Node::Map;
    nd.map = std::move(m);
    nd.rows = len;
    nd.offs = nullptr;
    nd.n = 0;
    stats.maps_built += 1;
    stats.forces += 1;
    stats.level_mask |= 1u << nd.level;
    stats.keys_inserted += nd.map->size();
  }
  // eager materialisation for simple (all map levels) / slt (level 0)
  void build(Backend b) {
    backend = b;
    root.kind = Node::BaseScan;
    root.level = 0;
    const int map_levels = (int)levels.size() - (trailing_empty ? 0 : 1);
    if (b == SIMPLE) {
      std::function<void(Node&)> rec = [&](Node& nd) {
        if (nd.level >= map_levels) return;
        force(nd);
        for (Node* c : nd.map->vals) rec(*c);
      };
      rec(root);
    } else if (b == SLT) {
      if (map_levels >= 1) force(root);
    }
  }
};

// residual subtrie of one atom during execution
struct Sub {
  Node* node = nullptr;
  bool singleton = false;  // a streamed row: the vector [row]
};

// -------------------------------------------------------------- executor ----
struct PSub {
  int atom;
  std::vector<int> vars, cols;
  int level;
  bool stream;  // vars == all remaining variables of the atom (Fig 12 is_suffix)
  bool last;
};
struct PNode {
  std::vector<PSub> subs;
  std::vector<int> covers;
  uint32_t avs_mask = 0;
};

struct Result {
  uint64_t count_lo = 0, count_hi = 0, checksum = 0;
  int64_t minv = INT64_MAX;
  int has_min = 0;
  uint64_t probes = 0, misses = 0;
  uint64_t body[32] = {0};
  uint64_t maps_built = 0, keys_inserted = 0, forces = 0;
  int factorized = 0;
  uint64_t atom_maps[16] = {0}, atom_keys[16] = {0};
  uint32_t atom_levels[16] = {0};
};

struct Exec {
  std::vector<PNode> nodes;
  std::vector<std::unique_ptr<Colt>> tries;  // per atom
  int nvars = 0;
  uint64_t batch = 1000;
  bool dynamic = true;
  int output_mode = 0;  // 0 count, 1 enumerate, 2 factorized count
  int min_var = -1;
  int part = 0, nparts = 1, part_var = 0;
  Result res;
  std::vector<int64_t>* collect = nullptr;

  void add_count(uint64_t m) {
    uint64_t old = res.count_lo;
    res.count_lo += m;
    if (res.count_lo < old) ++res.count_hi;
  }
  // output (Fig 8 line `output(tuple)`): leaf multiplicities, SURVEY App. A.4
  void emit(const int64_t* vals, const Sub* subs, int A) {
    uint64_t mult = 1;
    for (int a = 0; a < A; ++a)
      if (!subs[a].singleton) mult *= tries[a]->length(*subs[a].node);
    if (mult == 0) return;
    add_count(mult);
    res.checksum += mult * fmix64(tuple_hash(vals, nvars));
    if (min_var >= 0) res.minv = std::min(res.minv, vals[min_var]);
    if (collect)
      for (uint64_t r = 0; r < mult; ++r) collect->insert(collect->end(), vals, vals + nvars);
  }
  // count_factorized precondition: every remaining node is
  // one subatom whose variables are all fresh and not shared with another
  // remaining atom.
  bool factorizable(int k) const {
    std::map<int, int> var_atom;
    for (size_t j = k; j < nodes.size(); ++j) {
      if (nodes[j].subs.size() != 1) return false;
      const PSub& s = nodes[j].subs[0];
      for (int v : s.vars) {
        if ((nodes[k].avs_mask >> v) & 1u) return false;
        auto it = var_atom.find(v);
        if (it != var_atom.end() && it->second != s.atom) return false;
        var_atom[v] = s.atom;
      }
    }
    return true;
  }

  // ---- memoised factorised count over a chain suffix (extension of
  // count_factorized): from node k* on, each
  // node j has exactly one open atom C_j whose last subatom is in j and binds
  // only fresh variables; every other subatom of j is the first subatom of a
  // fresh atom keyed on C_j's variables; at most one of those continues and
  // becomes C_{j+1}. Then count(j, subtrie s of C_j) depends only on s and is
  // memoised per COLT node.
  struct ChainNode {
    int carrier = -1;             // subatom index of C_j in node j
    std::vector<int> fresh;       // subatom indices of the fresh atoms
    int next = -1;                // subatom index (in node j) of C_{j+1}, -1 at the end
  };
  int chain_start = -1;
  std::vector<ChainNode> chain;
  std::vector<int> atom_first, atom_last;  // node index of each atom's first / last subatom
  std::map<std::pair<int, const Node*>, unsigned __int128> memo;

  bool chain_node_ok(int j, ChainNode& cn) const {
    const PNode& N = nodes[j];
    const int A = (int)tries.size();
    int carrier_atom = -1;
    for (int a = 0; a < A; ++a)
      if (atom_first[a] < j && atom_last[a] >= j) {
        if (carrier_atom >= 0) return false;
        carrier_atom = a;
      }
    if (carrier_atom < 0) return false;
    uint32_t cvars = 0;
    for (size_t i = 0; i < N.subs.size(); ++i)
      if (N.subs[i].atom == carrier_atom) {
        if (cn.carrier >= 0 || !N.subs[i].last) return false;
        cn.carrier = (int)i;
        for (int v : N.subs[i].vars) cvars |= 1u << v;
      }
    if (cn.carrier < 0 || (cvars & N.avs_mask)) return false;
    for (size_t i = 0; i < N.subs.size(); ++i) {
      if ((int)i == cn.carrier) continue;
      const PSub& X = N.subs[i];
      if (X.level != 0) return false;
      for (int v : X.vars)
        if (!((cvars >> v) & 1u)) return false;
      if (!X.last) {
        if (cn.next >= 0) return false;
        cn.next = (int)i;
      }
      cn.fresh.push_back((int)i);
    }
    for (size_t i = j; i < nodes.size(); ++i)
      for (const PSub& X : nodes[i].subs)
        for (int v : X.vars)
          if ((N.avs_mask >> v) & 1u) return false;
    return (cn.next >= 0) == (j + 1 < (int)nodes.size());
  }

  void analyze_chain() {
    for (int k = (int)nodes.size() - 1; k >= 1; --k) {
      ChainNode cn;
      if (!chain_node_ok(k, cn)) break;
      chain.insert(chain.begin(), cn);
      chain_start = k;
    }
  }

  unsigned __int128 chain_count(int j, const Sub& s) {
    std::pair<int, const Node*> mk{j, s.singleton ? nullptr : s.node};
    if (!s.singleton) {
      auto it = memo.find(mk);
      if (it != memo.end()) return it->second;
    }
    const ChainNode& cn = chain[j - chain_start];
    const PNode& N = nodes[j];
    const PSub& C = N.subs[cn.carrier];
    Colt& CT = *tries[C.atom];
    unsigned __int128 total = 0;
    auto visit = [&](const int64_t* t, uint64_t m) {
      unsigned __int128 f = m;
      for (int xi : cn.fresh) {
        const PSub& X = N.subs[xi];
        Key key;
        key.n = (int)X.vars.size();
        for (int q = 0; q < key.n; ++q) {
          int at = 0;
          while (C.vars[at] != X.vars[q]) ++at;
          key.v[q] = t[at];
        }
        Sub root;
        root.node = &tries[X.atom]->root;
        Sub out;
        if (!get(X.atom, root, key, out)) return;
        if (xi == cn.next)
          f *= chain_count(j + 1, out);
        else
          f *= out.singleton ? 1 : tries[X.atom]->length(*out.node);
      }
      total += f;
    };
    int64_t t[MAXK];
    if (s.singleton) {
      visit(t, 1);
    } else if (s.node->kind == Node::Map) {
      const FlatMap& mp = *s.node->map;
      for (size_t e = 0; e < mp.size(); ++e) visit(mp.keys[e].v, CT.length(*mp.vals[e]));
    } else {
      const uint64_t n = CT.length(*s.node);
      for (uint64_t x = 0; x < n; ++x) {
        const uint64_t row = s.node->kind == Node::BaseScan ? x : s.node->offs[x];
        for (size_t q = 0; q < C.cols.size(); ++q) t[q] = CT.rel->at(C.cols[q], row);
        visit(t, 1);
      }
    }
    if (!s.singleton) memo[mk] = total;
    return total;
  }

  void add_count128(unsigned __int128 v) {
    const uint64_t lo = (uint64_t)v, hi = (uint64_t)(v >> 64);
    uint64_t old = res.count_lo;
    res.count_lo += lo;
    res.count_hi += hi + (res.count_lo < old ? 1 : 0);
  }

  // get (Fig 12 `get`: force then lookup)
  bool get(int atom, const Sub& sub, const Key& key, Sub& out) {
    ++res.probes;
    if (sub.singleton) {  // [row] keyed on () -> itself
      out = sub;
      return true;
    }
    Colt& T = *tries[atom];
    T.force(*sub.node);
    Node* c = sub.node->map->find(key);
    if (!c) {
      ++res.misses;
      return false;
    }
    out.node = c;
    out.singleton = false;
    return true;
  }

  // per-node batch buffers (Fig 13 `tup_subtries`), reused across calls
  struct Batch {
    std::vector<int64_t> vals;  // n x nvars
    std::vector<Sub> subs;      // n x natoms
    std::vector<char> alive;
    size_t n = 0;
  };
  std::vector<Batch> batches;

  void join(int k, const int64_t* vals, const Sub* subs) {
    const int A = (int)tries.size();
    if (k == (int)nodes.size()) {
      emit(vals, subs, A);
      return;
    }
    const PNode& N = nodes[k];
    if (output_mode == 2 && k > 0 && k == chain_start && !factorizable(k)) {
      unsigned __int128 m = 1;
      int carrier = -1;
      for (int a = 0; a < A; ++a) {
        if (atom_last[a] < k)
          m *= subs[a].singleton ? 1 : tries[a]->length(*subs[a].node);
        else if (atom_first[a] < k)
          carrier = a;
      }
      add_count128(m * chain_count(k, subs[carrier]));
      res.factorized = 1;
      return;
    }
    if (output_mode == 2 && k > 0 && factorizable(k)) {
      uint64_t mult = 1;
      std::set<int> suffix_atoms;
      for (size_t j = k; j < nodes.size(); ++j) suffix_atoms.insert(nodes[j].subs[0].atom);
      for (int a = 0; a < A; ++a) {
        uint64_t len = subs[a].singleton ? 1 : tries[a]->length(*subs[a].node);
        if (suffix_atoms.count(a) || !subs[a].singleton) mult *= len;
      }
      add_count(mult);
      res.factorized = 1;
      return;
    }
    // select_cover: min estimated_key_count, ties -> lowest position
    int ci = N.covers[0];
    if (dynamic && N.covers.size() > 1) {
      uint64_t best = UINT64_MAX;
      for (int c : N.covers) {
        const PSub& S = N.subs[c];
        const Sub& sb = subs[S.atom];
        uint64_t est = sb.singleton ? 1 : tries[S.atom]->estimated_key_count(*sb.node);
        if (est < best) {
          best = est;
          ci = c;
        }
      }
    }
    const PSub& C = N.subs[ci];
    Colt& CT = *tries[C.atom];
    const Sub csub = subs[C.atom];
    Batch& B = batches[k];
    const size_t cap = batch_size();
    B.n = 0;
    B.vals.resize(cap * nvars);
    B.subs.resize(cap * A);
    B.alive.resize(cap);
    Key key;
    auto flush = [&]() {
      // probe each other trie over the whole surviving batch (Fig 13)
      for (size_t b = 0; b < B.n; ++b) B.alive[b] = 1;
      for (size_t s = 0; s < N.subs.size(); ++s) {
        if ((int)s == ci) continue;
        const PSub& P = N.subs[s];
        for (size_t b = 0; b < B.n; ++b) {
          if (!B.alive[b]) continue;
          const int64_t* v = &B.vals[b * nvars];
          key.n = (int)P.vars.size();
          for (int t = 0; t < key.n; ++t) key.v[t] = v[P.vars[t]];
          Sub out;
          Sub& cur = B.subs[b * A + P.atom];
          if (!get(P.atom, cur, key, out))
            B.alive[b] = 0;
          else
            cur = out;
        }
      }
      const size_t n = B.n;
      B.n = 0;
      for (size_t b = 0; b < n; ++b)
        if (B.alive[b]) join(k + 1, &B.vals[b * nvars], &B.subs[b * A]);
    };
    // B must not be reused while recursing: deeper nodes use batches[k+1..]
    auto offer = [&](const int64_t* t, const Sub& residual) {
      int64_t* v = &B.vals[B.n * nvars];
      std::copy(vals, vals + nvars, v);
      for (int i = 0; i < (int)C.vars.size(); ++i) {
        const int x = C.vars[i];
        if ((N.avs_mask >> x) & 1u) {
          if (v[x] != t[i]) return;  // cover re-binds a bound variable: must agree
        } else {
          v[x] = t[i];
        }
      }
      if (k == 0 && nparts > 1 && partition_of(v[part_var], (uint32_t)nparts) != (uint32_t)part) return;
      ++res.body[k];
      Sub* sb = &B.subs[B.n * A];
      std::copy(subs, subs + A, sb);
      sb[C.atom] = residual;
      if (++B.n >= cap) flush();
    };
    int64_t t[MAXK];
    if (csub.singleton) {
      offer(t, csub);
    } else if (C.stream && csub.node->kind != Node::Map) {
      // suffix vector: stream values at the offsets, each row its own tuple
      Sub r;
      r.singleton = true;
      const int nc = (int)C.cols.size();
      if (csub.node->kind == Node::BaseScan) {
        for (uint64_t i = 0; i < CT.rel->n; ++i) {
          for (int q = 0; q < nc; ++q) t[q] = CT.rel->at(C.cols[q], i);
          offer(t, r);
        }
      } else {
        for (uint32_t x = 0; x < csub.node->n; ++x) {
          const uint32_t i = csub.node->offs[x];
          for (int q = 0; q < nc; ++q) t[q] = CT.rel->at(C.cols[q], i);
          offer(t, r);
        }
      }
    } else {
      CT.force(*csub.node);
      const FlatMap& mp = *csub.node->map;
      for (size_t e = 0; e < mp.size(); ++e) {
        Sub r;
        r.node = mp.vals[e];
        offer(mp.keys[e].v, r);
      }
    }
    flush();
  }
  uint64_t batch_size() const { return batch ? batch : 1; }
};

struct Prepared {
  std::vector<std::string> head;
  std::vector<std::vector<int>> atom_vars;
  std::vector<std::string> atom_names;
  std::vector<PNode> nodes;
  std::vector<std::vector<std::vector<int>>> levels;  // per atom
  std::vector<bool> trailing;
};

static Prepared prepare(const std::string& query_json, const std::string& plan_json) {
  Prepared P;
  J q = parse(query_json);
  const J& atoms = q.k == J::Obj ? q.at("query") : q;
  std::map<std::string, int> vid, aid;
  for (auto& a : atoms.a) {
    aid[a.at("rel").s] = (int)P.atom_names.size();
    P.atom_names.push_back(a.at("rel").s);
    std::vector<int> vs;
    for (auto& x : a.at("vars").a) {
      if (!vid.count(x.s)) {
        vid[x.s] = (int)P.head.size();
        P.head.push_back(x.s);
      }
      vs.push_back(vid[x.s]);
    }
    P.atom_vars.push_back(vs);
  }
  J plan = parse(plan_json);
  const int A = (int)P.atom_names.size();
  std::vector<std::vector<std::pair<int, int>>> subs_of(A);
  uint32_t bound = 0;
  for (size_t k = 0; k < plan.a.size(); ++k) {
    PNode N;
    N.avs_mask = bound;
    for (auto& s : plan.a[k].a) {
      PSub ps;
      ps.atom = aid.at(s.a[0].s);
      for (auto& x : s.a[1].a) {
        ps.vars.push_back(vid.at(x.s));
        const auto& av = P.atom_vars[ps.atom];
        ps.cols.push_back((int)(std::find(av.begin(), av.end(), vid.at(x.s)) - av.begin()));
      }
      subs_of[ps.atom].emplace_back((int)k, (int)N.subs.size());
      N.subs.push_back(ps);
    }
    uint32_t vsm = 0;
    for (auto& s : N.subs)
      for (int v : s.vars) vsm |= 1u << v;
    const uint32_t need = vsm & ~bound;
    for (size_t i = 0; i < N.subs.size(); ++i) {
      uint32_t m = 0;
      for (int v : N.subs[i].vars) m |= 1u << v;
      if ((m & need) == need) N.covers.push_back((int)i);
    }
    if (N.covers.empty()) throw std::runtime_error("oracle: node without cover");
    bound |= vsm;
    P.nodes.push_back(N);
  }
  P.levels.resize(A);
  P.trailing.resize(A);
  for (int a = 0; a < A; ++a) {
    const auto& so = subs_of[a];
    if (so.empty()) throw std::runtime_error("oracle: atom not in plan");
    for (size_t d = 0; d < so.size(); ++d) {
      PSub& ps = P.nodes[so[d].first].subs[so[d].second];
      ps.level = (int)d;
      ps.last = d + 1 == so.size();
      bool later = false;
      for (size_t e = d + 1; e < so.size(); ++e)
        if (!P.nodes[so[e].first].subs[so[e].second].vars.empty()) later = true;
      ps.stream = !later;
      P.levels[a].push_back(ps.cols);
    }
    // derive_ght_schemas: trailing [] unless the last subatom
    // is its node's position-0 cover
    P.trailing[a] = so.back().second != 0;
  }
  return P;
}

static Result run_one(const Prepared& P, const std::vector<Relation>& rels, int backend, uint64_t batch,
                      int dynamic, int output_mode, int min_var, int part, int nparts,
                      std::vector<int64_t>* collect) {
  Exec ex;
  ex.nodes = P.nodes;
  ex.nvars = (int)P.head.size();
  ex.batch = batch;
  ex.dynamic = dynamic != 0;
  ex.output_mode = output_mode;
  ex.min_var = min_var;
  ex.part = part;
  ex.nparts = nparts;
  ex.part_var = P.nodes[0].subs[0].vars.empty() ? 0 : P.nodes[0].subs[0].vars[0];
  ex.collect = collect;
  const int A = (int)rels.size();
  ex.atom_first.assign(A, 1 << 30);
  ex.atom_last.assign(A, -1);
  for (size_t k = 0; k < P.nodes.size(); ++k)
    for (const PSub& ps : P.nodes[k].subs) {
      ex.atom_first[ps.atom] = std::min(ex.atom_first[ps.atom], (int)k);
      ex.atom_last[ps.atom] = std::max(ex.atom_last[ps.atom], (int)k);
    }
  std::vector<Sub> subs(A);
  for (int a = 0; a < A; ++a) {
    auto T = std::make_unique<Colt>();
    T->rel = &rels[a];
    T->levels = P.levels[a];
    T->trailing_empty = P.trailing[a];
    T->build((Backend)backend);  // GHT new
    subs[a].node = &T->root;
    ex.tries.push_back(std::move(T));
  }
  if (output_mode == 2) ex.analyze_chain();
  std::vector<int64_t> vals(ex.nvars, 0);
  ex.batches.resize(P.nodes.size() + 1);
  ex.join(0, vals.data(), subs.data());
  for (size_t a = 0; a < ex.tries.size(); ++a) {
    const auto& T = ex.tries[a];
    ex.res.maps_built += T->stats.maps_built;
    ex.res.keys_inserted += T->stats.keys_inserted;
    ex.res.forces += T->stats.forces;
    if (a < 16) {
      ex.res.atom_maps[a] = T->stats.maps_built;
      ex.res.atom_keys[a] = T->stats.keys_inserted;
      ex.res.atom_levels[a] = T->stats.level_mask;
    }
  }
  ex.res.has_min = (min_var >= 0 && ex.res.minv != INT64_MAX) ? 1 : 0;
  return ex.res;
}

// brute-force nested-loop join: bag over head variables
static void brute(const Prepared& P, const std::vector<Relation>& rels, size_t a, std::vector<int64_t>& vals,
                  std::vector<char>& bound, std::vector<int64_t>& out) {
  if (a == rels.size()) {
    out.insert(out.end(), vals.begin(), vals.end());
    return;
  }
  const auto& av = P.atom_vars[a];
  for (uint64_t i = 0; i < rels[a].n; ++i) {
    std::vector<int> newly;
    bool ok = true;
    for (size_t c = 0; c < av.size() && ok; ++c) {
      const int64_t x = rels[a].at((int)c, i);
      if (bound[av[c]]) {
        if (vals[av[c]] != x) ok = false;
      } else {
        bound[av[c]] = 1;
        vals[av[c]] = x;
        newly.push_back(av[c]);
      }
    }
    if (ok) brute(P, rels, a + 1, vals, bound, out);
    for (int v : newly) bound[v] = 0;
  }
}

}  // namespace orc

// ============================================================== C-ABI ======
extern "C" {

typedef struct {
  uint64_t count_lo, count_hi, checksum;
  int64_t min_value;
  int32_t has_min, factorized;
  uint64_t probes, probe_misses;
  uint64_t node_body_entries[32];
  uint64_t maps_built, keys_inserted, forces;
  uint64_t atom_maps_built[16], atom_keys_inserted[16];
  uint32_t atom_levels_forced[16];
} orc_result;

static thread_local std::string g_err;
const char* orc_last_error(void) { return g_err.c_str(); }

static std::vector<orc::Relation> make_rels(const int32_t* const* const* atom_cols, const int* atom_ncols,
                                            const uint64_t* atom_rows, int natoms) {
  std::vector<orc::Relation> rels(natoms);
  for (int a = 0; a < natoms; ++a) {
    rels[a].n = atom_rows[a];
    for (int c = 0; c < atom_ncols[a]; ++c) rels[a].cols.push_back(atom_cols[a][c]);
  }
  return rels;
}

static void fill(orc_result* out, const orc::Result& r) {
  memset(out, 0, sizeof(*out));
  out->count_lo = r.count_lo;
  out->count_hi = r.count_hi;
  out->checksum = r.checksum;
  out->min_value = r.has_min ? r.minv : 0;
  out->has_min = r.has_min;
  out->factorized = r.factorized;
  out->probes = r.probes;
  out->probe_misses = r.misses;
  for (int k = 0; k < 32; ++k) out->node_body_entries[k] = r.body[k];
  out->maps_built = r.maps_built;
  out->keys_inserted = r.keys_inserted;
  out->forces = r.forces;
  for (int a = 0; a < 16; ++a) {
    out->atom_maps_built[a] = r.atom_maps[a];
    out->atom_keys_inserted[a] = r.atom_keys[a];
    out->atom_levels_forced[a] = r.atom_levels[a];
  }
}

// Execute a Free Join plan on the CPU. part/nparts: only bindings whose first
// plan variable hashes to `part` (independent trie set).
// nthreads > 1: thread t runs partition part+t of P = max(nparts, nthreads)
// (part=0, nparts<=nthreads covers the whole query) and the results are summed.
int orc_execute(const char* query_json, const char* plan_json, const int32_t* const* const* atom_cols,
                const int* atom_ncols, const uint64_t* atom_rows, int natoms, int backend, uint64_t batch_size,
                int dynamic, int output_mode, int min_var, int part, int nparts, int nthreads, orc_result* out,
                int64_t** tuples, uint64_t* ntuples) {
  try {
    orc::Prepared P = orc::prepare(query_json, plan_json);
    auto rels = make_rels(atom_cols, atom_ncols, atom_rows, natoms);
    if ((int)P.atom_names.size() != natoms) throw std::runtime_error("oracle: atom count mismatch");
    std::vector<int64_t> coll;
    std::vector<int64_t>* cp = (output_mode == 1) ? &coll : nullptr;
    orc::Result total;
    if (nthreads <= 1) {
      total = orc::run_one(P, rels, backend, batch_size, dynamic, output_mode, min_var, part, nparts, cp);
    } else {
      std::vector<orc::Result> rs(nthreads);
      std::vector<std::vector<int64_t>> cs(nthreads);
      std::vector<std::thread> th;
      std::vector<std::string> errs(nthreads);
      for (int t = 0; t < nthreads; ++t)
        th.emplace_back([&, t] {
          try {
            const int PP = std::max(nparts, nthreads);
            rs[t] = orc::run_one(P, rels, backend, batch_size, dynamic, output_mode, min_var, (part + t) % PP, PP,
                                 cp ? &cs[t] : nullptr);
          } catch (const std::exception& e) {
            errs[t] = e.what();
          }
        });
      for (auto& x : th) x.join();
      for (int t = 0; t < nthreads; ++t) {
        if (!errs[t].empty()) throw std::runtime_error(errs[t]);
        const orc::Result& r = rs[t];
        uint64_t old = total.count_lo;
        total.count_lo += r.count_lo;
        total.count_hi += r.count_hi + (total.count_lo < old ? 1 : 0);
        total.checksum += r.checksum;
        total.minv = std::min(total.minv, r.minv);
        total.has_min |= r.has_min;
        total.factorized |= r.factorized;
        total.probes += r.probes;
        total.misses += r.misses;
        for (int k = 0; k < 32; ++k) total.body[k] += r.body[k];
        total.maps_built += r.maps_built;
        total.keys_inserted += r.keys_inserted;
        total.forces += r.forces;
        for (int a = 0; a < 16; ++a) {
          total.atom_maps[a] += r.atom_maps[a];
          total.atom_keys[a] += r.atom_keys[a];
          total.atom_levels[a] |= r.atom_levels[a];
        }
        if (cp) coll.insert(coll.end(), cs[t].begin(), cs[t].end());
      }
    }
    fill(out, total);
    if (tuples) {
      *ntuples = P.head.empty() ? 0 : coll.size() / P.head.size();
      *tuples = (int64_t*)malloc(std::max<size_t>(coll.size(), 1) * 8);
      if (!coll.empty()) memcpy(*tuples, coll.data(), coll.size() * 8);
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

int orc_brute_force(const char* query_json, const int32_t* const* const* atom_cols, const int* atom_ncols,
                    const uint64_t* atom_rows, int natoms, int64_t** tuples, uint64_t* ntuples) {
  try {
    // a trivial one-node plan gives the head order
    orc::Prepared P;
    {
      orc::J q = orc::parse(query_json);
      const orc::J& atoms = q.k == orc::J::Obj ? q.at("query") : q;
      std::map<std::string, int> vid;
      for (auto& a : atoms.a) {
        std::vector<int> vs;
        for (auto& x : a.at("vars").a) {
          if (!vid.count(x.s)) {
            vid[x.s] = (int)P.head.size();
            P.head.push_back(x.s);
          }
          vs.push_back(vid[x.s]);
        }
        P.atom_vars.push_back(vs);
      }
    }
    auto rels = make_rels(atom_cols, atom_ncols, atom_rows, natoms);
    std::vector<int64_t> vals(P.head.size(), 0), out;
    std::vector<char> bound(P.head.size(), 0);
    orc::brute(P, rels, 0, vals, bound, out);
    *ntuples = P.head.empty() ? 0 : out.size() / P.head.size();
    *tuples = (int64_t*)malloc(std::max<size_t>(out.size(), 1) * 8);
    if (!out.empty()) memcpy(*tuples, out.data(), out.size() * 8);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

void orc_free(void* p) { free(p); }

uint64_t orc_tuple_hash(const int64_t* vals, int n) { return orc::tuple_hash(vals, n); }
uint64_t orc_checksum_word(uint64_t h) { return orc::fmix64(h); }
uint32_t orc_partition_of(int64_t v, uint32_t nparts) { return orc::partition_of(v, nparts); }

}  // extern "C"
