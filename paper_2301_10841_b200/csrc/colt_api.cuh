// The GHT / COLT handle behind the C-ABI (SURVEY.md §8(b) fjg_colt_create;
// PAPER.md:544-557 Fig 5 `new / iter / get`, SPEC.md:286-339 `force /
// iter_batch / estimated_key_count`). Included at the end of engine.cu.
//
// A fjg_colt is one device COLT over a relation with a caller-given GHT schema
// (key columns per level). It owns a private single-atom query whose physical
// trie holds the device levels, so every operation runs the same kernels as
// the executor (claims, force batches, 256-bit bucket probes). Unlike a
// query's tries, a handle's state persists across calls: a subtrie forced once
// stays forced (COLT's lazy, idempotent force), so a host can own tries and
// reuse them across queries of its own. Subtries are named as in the executor
// by their position range (p, len) in the level's ordering; the root is
// (0, rows).

namespace {

// claims for explicit subtries (Fig 12 force = group this subtrie now)
__global__ void k_colt_claim(const DevTrie* tries, DevCounters* ctr, int t, int l, const uint32_t* __restrict__ p,
                             const uint32_t* __restrict__ len, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t iters = (n + stride - 1) / stride;
  KSub S{};
  S.trie = (uint8_t)t;
  S.depth = (uint8_t)l;
  for (uint64_t it = 0; it < iters; ++it) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x + it * stride;
    const bool ok = i < n;
    const uint32_t pi = ok ? p[i] : 0u, li = ok ? len[i] : 0u;
    const bool need = ok && li > 0 && *((volatile const uint32_t*)&tries[t].lev[l].sn[pi].state) == 0u;
    claim_subtrie(tries, ctr, S, pi, li, need);
  }
}

// batched get: child subtrie of key i in subtrie (p[i], len[i])
__global__ void k_colt_get(const __grid_constant__ KSub S, const uint32_t* __restrict__ p,
                           const uint32_t* __restrict__ len, const int32_t* __restrict__ keys, int arity, uint64_t n,
                           uint32_t* __restrict__ cp, uint32_t* __restrict__ cl, uint8_t* __restrict__ found) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    int32_t key[MAXK];
#pragma unroll
    for (int k = 0; k < MAXK; ++k) key[k] = k < arity ? keys[i * arity + k] : 0;
    uint32_t q = 0, ql = 0;
    const bool hit = len[i] > 0 && colt_get<true>(S, p[i], len[i], key, q, ql);
    cp[i] = hit ? q : 0u;
    cl[i] = hit ? ql : 0u;
    found[i] = hit ? 1 : 0;
  }
}

// iter over a forced map subtrie: every occupied slot of its region is one key
__global__ void k_colt_keys(const Slot* __restrict__ table, uint64_t s0, uint64_t s1, const uint32_t* __restrict__ cnt,
                            uint32_t* __restrict__ cq, uint32_t* __restrict__ cl, uint32_t* __restrict__ count) {
  for (uint64_t s = s0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < s1;
       s += (uint64_t)gridDim.x * blockDim.x) {
    const Slot sl = table[s];
    if (sl.q == kEmpty) continue;
    const uint32_t o = atomicAdd(count, 1u);
    cq[o] = sl.q;
    cl[o] = cnt[sl.q];
  }
}

__global__ void k_colt_gather(const int32_t* __restrict__ col, const uint32_t* __restrict__ pos, uint64_t n,
                              int32_t* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = col[pos[i]];
}

}  // namespace

struct fjg_colt {
  fjg_engine* eng = nullptr;
  fjg_query* q = nullptr;
  std::vector<std::vector<int>> levels;  // key columns per level; the last level may be the vector (no map)
  int map_levels = 0;
  uint64_t rows = 0;
};

namespace {

DevTrie& colt_trie(fjg_colt* c) { return c->q->tries[0].dev; }

void colt_check_level(const fjg_colt* c, int level, bool map) {
  if (level < 0 || level >= (int)c->levels.size())
    throw fj::ValidationError("colt: level " + std::to_string(level) + " out of range");
  if (map && level >= c->map_levels)
    throw fj::ValidationError("colt: level " + std::to_string(level) + " is the vector level (no map)");
}

// force the given subtries of `level`: idempotent
void colt_force(fjg_colt* c, int level, const uint32_t* hp, const uint32_t* hl, uint64_t n) {
  fjg_query* q = c->q;
  fjg_engine* eng = c->eng;
  if (level == 0) {
    if (!q->tries[0].root_forced) force_roots(q, {0});
    return;
  }
  if (n == 0) return;
  if (n > (1ull << 31)) throw fj::ValidationError("colt: at most 2^31 subtries per call");
  uint32_t* d = (uint32_t*)eng->pool->alloc(n * 8);
  CK(cudaMemcpyAsync(d, hp, n * 4, cudaMemcpyHostToDevice, eng->stream));
  CK(cudaMemcpyAsync(d + n, hl, n * 4, cudaMemcpyHostToDevice, eng->stream));
  for (uint64_t i = 0; i < n; ++i)
    if ((uint64_t)hp[i] + hl[i] > c->rows) {
      eng->pool->free(d);
      throw fj::ValidationError("colt: subtrie (p, len) beyond the relation");
    }
  LAUNCH(eng, k_colt_claim<<<grid_for(n), 256, 0, eng->stream>>>(q->d_tries, q->d_ctr, 0, level, d, d + n, n));
  sync_counters(q);
  force_claims(q, 0);
  sync_counters(q);
  eng->pool->free(d);
}

KSub colt_ksub(fjg_colt* c, int level) {
  fjg_query* q = c->q;
  const DevTrie& T = colt_trie(c);
  const DevLevel& L = T.lev[level];
  KSub S{};
  for (int t = 0; t < L.nk; ++t) S.kcmp[t] = L.cval[L.keycol[t]];
  S.cnt = L.cnt;
  S.table = L.table;
  S.sn = L.sn;
  // a non-null in_p marks a non-root subtrie (probe_region uses its length)
  S.in_p = level == 0 ? nullptr : L.cnt;
  S.root_n = (uint32_t)c->rows;
  S.rregion = q->d_ctr->root_region;
  S.ldup = q->d_ctr->level_dup + level;
  S.nv = (uint8_t)L.nk;
  S.trie = 0;
  S.depth = (uint8_t)level;
  return S;
}

}  // namespace

extern "C" {

int fjg_colt_create(fjg_engine* eng, const fjg_relation* rel, const int* level_cols, const int* level_ncols,
                    int nlevels, fjg_colt** out) {
  return guard([&] {
    if (!eng || !rel || !level_cols || !level_ncols || !out) throw fj::ValidationError("fjg_colt_create: null argument");
    if (rel->eng != eng) throw fj::ValidationError("fjg_colt_create: relation of another engine");
    if (nlevels < 1 || nlevels > MAXL - 1) throw fj::ValidationError("fjg_colt_create: 1..7 levels");
    const int nc = rel->ncols;
    std::vector<std::vector<int>> lv;
    std::vector<int> used(nc, 0);
    int off = 0;
    for (int l = 0; l < nlevels; ++l) {
      if (level_ncols[l] < 1 || level_ncols[l] > MAXK) throw fj::ValidationError("fjg_colt_create: 1..8 key columns per level");
      std::vector<int> cols;
      for (int k = 0; k < level_ncols[l]; ++k) {
        const int col = level_cols[off + k];
        if (col < 0 || col >= nc || used[col]) throw fj::ValidationError("fjg_colt_create: bad or repeated column");
        used[col] = 1;
        cols.push_back(col);
      }
      off += level_ncols[l];
      lv.push_back(cols);
    }
    // the GHT of a single-atom plan: one node per level (each its node's cover,
    // so no trailing [] level), then a vector level holding
    // the columns no level keys on
    std::vector<int> rest;
    for (int col = 0; col < nc; ++col)
      if (!used[col]) rest.push_back(col);
    auto var = [](int col) { return "\"c" + std::to_string(col) + "\""; };
    std::string qj = "{\"query\":[{\"rel\":\"R\",\"vars\":[";
    for (int col = 0; col < nc; ++col) qj += (col ? "," : "") + var(col);
    qj += "]}]}";
    std::string pj = "[";
    auto node = [&](const std::vector<int>& cols) {
      std::string s = "[[\"R\",[";
      for (size_t k = 0; k < cols.size(); ++k) s += (k ? "," : "") + var(cols[k]);
      return s + "]]]";
    };
    for (int l = 0; l < nlevels; ++l) pj += (l ? "," : "") + node(lv[l]);
    if (!rest.empty()) pj += "," + node(rest);
    pj += "]";
    fjg_relation* r = const_cast<fjg_relation*>(rel);
    fjg_query* q = nullptr;
    const int rc = fjg_query_create(eng, qj.c_str(), pj.c_str(), &r, 1, &q);
    if (rc) {
      const std::string m = fjg_last_error();
      if (rc == FJG_E_VALIDATION) throw fj::ValidationError(m);
      if (rc == FJG_E_RESOURCE) throw fj::ResourceError(m);
      throw fj::EngineError(m);
    }
    auto* c = new fjg_colt();
    c->eng = eng;
    c->q = q;
    c->levels = lv;
    if (!rest.empty()) c->levels.push_back(rest);
    c->map_levels = nlevels;
    c->rows = rel->nrows;
    try {
      ScopedDevice sd(eng->device);
      ensure_frontiers(q, 1024);
      reset_query(q);  // GHT new: BaseScan, every subtrie unforced
      q->timing = false;
      sync_counters(q);
    } catch (...) {
      fjg_query_destroy(q);
      delete c;
      throw;
    }
    *out = c;
  });
}

int fjg_colt_levels(const fjg_colt* c) { return c ? (int)c->levels.size() : 0; }

int fjg_colt_force(fjg_colt* c, int level, const uint32_t* p, const uint32_t* len, uint64_t n) {
  return guard([&] {
    ScopedDevice sd(c->eng->device);
    colt_check_level(c, level, true);
    colt_force(c, level, p, len, n);
  });
}

int fjg_colt_get(fjg_colt* c, int level, const uint32_t* p, const uint32_t* len, const int32_t* keys, uint64_t n,
                 uint32_t* child_p, uint32_t* child_len, uint8_t* found) {
  return guard([&] {
    fjg_engine* eng = c->eng;
    ScopedDevice sd(eng->device);
    colt_check_level(c, level, true);
    if (n == 0) return;
    colt_force(c, level, p, len, n);  // Fig 12 get: force, then lookup
    const int ar = (int)c->levels[level].size();
    char* d = (char*)eng->pool->alloc(n * (4 + 4 + 4 * ar + 4 + 4 + 1));
    uint32_t* dp = (uint32_t*)d;
    uint32_t* dl = dp + n;
    int32_t* dk = (int32_t*)(dl + n);
    uint32_t* dcp = (uint32_t*)(dk + n * ar);
    uint32_t* dcl = dcp + n;
    uint8_t* df = (uint8_t*)(dcl + n);
    if (level == 0) {
      std::vector<uint32_t> z(n, 0), r(n, (uint32_t)c->rows);
      CK(cudaMemcpyAsync(dp, z.data(), n * 4, cudaMemcpyHostToDevice, eng->stream));
      CK(cudaMemcpyAsync(dl, r.data(), n * 4, cudaMemcpyHostToDevice, eng->stream));
      CK(cudaStreamSynchronize(eng->stream));
    } else {
      CK(cudaMemcpyAsync(dp, p, n * 4, cudaMemcpyHostToDevice, eng->stream));
      CK(cudaMemcpyAsync(dl, len, n * 4, cudaMemcpyHostToDevice, eng->stream));
    }
    CK(cudaMemcpyAsync(dk, keys, n * 4 * ar, cudaMemcpyHostToDevice, eng->stream));
    const KSub S = colt_ksub(c, level);
    LAUNCH(eng, k_colt_get<<<grid_for(n), 256, 0, eng->stream>>>(S, dp, dl, dk, ar, n, dcp, dcl, df));
    CK(cudaMemcpyAsync(child_p, dcp, n * 4, cudaMemcpyDeviceToHost, eng->stream));
    CK(cudaMemcpyAsync(child_len, dcl, n * 4, cudaMemcpyDeviceToHost, eng->stream));
    CK(cudaMemcpyAsync(found, df, n, cudaMemcpyDeviceToHost, eng->stream));
    CK(cudaStreamSynchronize(eng->stream));
    eng->pool->free(d);
  });
}

int fjg_colt_iter(fjg_colt* c, int level, uint32_t p, uint32_t len, int32_t* keys_out, uint32_t* child_p,
                  uint32_t* child_len, uint64_t cap, uint64_t* nkeys) {
  return guard([&] {
    fjg_engine* eng = c->eng;
    ScopedDevice sd(eng->device);
    colt_check_level(c, level, true);
    if (!nkeys) throw fj::ValidationError("fjg_colt_iter: null nkeys");
    if (level == 0) {
      p = 0;
      len = (uint32_t)c->rows;
    }
    *nkeys = 0;
    if (len == 0) return;
    colt_force(c, level, &p, &len, 1);
    const uint64_t region = level == 0 ? c->q->h_ctr->root_region[0] : len;
    const DevLevel& L = colt_trie(c).lev[level];
    uint32_t* d = (uint32_t*)eng->pool->alloc((2 * len + 1) * 4);
    CK(cudaMemsetAsync(d + 2 * len, 0, 4, eng->stream));
    LAUNCH(eng, k_colt_keys<<<grid_for(4ull * FJG_RS * region), 256, 0, eng->stream>>>(L.table, 4ull * FJG_RS * p,
                                                                                          4ull * FJG_RS * (p + region),
                                                                            L.cnt, d, d + len, d + 2 * len));
    uint32_t k = 0;
    CK(cudaMemcpyAsync(&k, d + 2 * len, 4, cudaMemcpyDeviceToHost, eng->stream));
    CK(cudaStreamSynchronize(eng->stream));
    *nkeys = k;
    if (k > cap) {
      eng->pool->free(d);
      throw fj::ResourceError("fjg_colt_iter: " + std::to_string(k) + " keys, capacity " + std::to_string(cap));
    }
    // keys in child-start order (the level's clustered order)
    std::vector<uint32_t> cq(k), cl(k);
    CK(cudaMemcpyAsync(cq.data(), d, k * 4ull, cudaMemcpyDeviceToHost, eng->stream));
    CK(cudaMemcpyAsync(cl.data(), d + len, k * 4ull, cudaMemcpyDeviceToHost, eng->stream));
    CK(cudaStreamSynchronize(eng->stream));
    std::vector<uint32_t> ord(k);
    for (uint32_t i = 0; i < k; ++i) ord[i] = i;
    std::sort(ord.begin(), ord.end(), [&](uint32_t a, uint32_t b) { return cq[a] < cq[b]; });
    std::vector<uint32_t> sq(k), sl(k);
    for (uint32_t i = 0; i < k; ++i) {
      sq[i] = cq[ord[i]];
      sl[i] = cl[ord[i]];
    }
    if (child_p) memcpy(child_p, sq.data(), k * 4ull);
    if (child_len) memcpy(child_len, sl.data(), k * 4ull);
    if (keys_out && k) {
      const int ar = (int)c->levels[level].size();
      CK(cudaMemcpyAsync(d, sq.data(), k * 4ull, cudaMemcpyHostToDevice, eng->stream));
      std::vector<int32_t> colv(k);
      for (int t = 0; t < ar; ++t) {
        LAUNCH(eng, k_colt_gather<<<grid_for(k), 256, 0, eng->stream>>>(L.cval[L.keycol[t]], d, k,
                                                                        (int32_t*)(d + len)));
        CK(cudaMemcpyAsync(colv.data(), d + len, k * 4ull, cudaMemcpyDeviceToHost, eng->stream));
        CK(cudaStreamSynchronize(eng->stream));
        for (uint32_t i = 0; i < k; ++i) keys_out[(uint64_t)i * ar + t] = colv[i];
      }
    }
    eng->pool->free(d);
  });
}

int fjg_colt_rows(fjg_colt* c, int level, uint32_t p, uint32_t len, int col, int32_t* out) {
  return guard([&] {
    fjg_engine* eng = c->eng;
    ScopedDevice sd(eng->device);
    colt_check_level(c, level, false);
    if (col < 0 || col >= c->q->tries[0].rel->ncols) throw fj::ValidationError("fjg_colt_rows: column out of range");
    if ((uint64_t)p + len > c->rows) throw fj::ValidationError("fjg_colt_rows: subtrie beyond the relation");
    if (len == 0) return;
    const DevTrie& T = colt_trie(c);
    // rows of a level-l subtrie sit in the ordering level l-1's force produced
    const int32_t* src = level == 0 ? T.base[col] : T.lev[level - 1].cval[col];
    if (!src) throw fj::ValidationError("fjg_colt_rows: column not clustered at this level");
    CK(cudaMemcpyAsync(out, src + p, len * 4ull, cudaMemcpyDeviceToHost, eng->stream));
    CK(cudaStreamSynchronize(eng->stream));
  });
}

int fjg_colt_estimated_key_count(fjg_colt* c, int level, uint32_t p, uint32_t len, uint64_t* out) {
  return guard([&] {
    fjg_engine* eng = c->eng;
    ScopedDevice sd(eng->device);
    colt_check_level(c, level, false);
    if (!out) throw fj::ValidationError("fjg_colt_estimated_key_count: null output");
    if (level == 0) {
      p = 0;
      len = (uint32_t)c->rows;
    }
    *out = len;  // vector (or BaseScan root): its length
    if (level >= c->map_levels) return;
    const DevLevel& L = colt_trie(c).lev[level];
    const uint32_t at = level == 0 ? 0u : p;
    SubState sn{};
    CK(cudaMemcpyAsync(&sn, L.sn + at, sizeof(sn), cudaMemcpyDeviceToHost, eng->stream));
    CK(cudaStreamSynchronize(eng->stream));
    if (sn.state == 2u) *out = sn.nkeys;  // a forced map: its number of keys (never forces)
  });
}

void fjg_colt_destroy(fjg_colt* c) {
  if (!c) return;
  fjg_query_destroy(c->q);
  delete c;
}

}  // extern "C"
