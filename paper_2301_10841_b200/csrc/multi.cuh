// Multi-GPU execution behind the C-ABI (BASELINE.json north_star (c); SURVEY.md
// §8(b) fjg_execute_multi, §8(e)). Included at the end of engine.cu.
//
// One process (or thread) per GPU, one fjg_engine + fjg_comm per rank. Every
// rank holds a slice of each base relation. Per execution, on the engine
// stream and without torch:
//   1. every view (base relation, column of the plan's first variable) is
//      hash-partitioned by the partition kernel into persistent send buffers
//      (fj::partition_of = fmix64 mod G, the oracle's function); views of atoms
//      without the first variable are replicated;
//   2. ONE ncclAllGather carries all size metadata (per partitioned view the
//      rows per destination, per replicated view the local row count), read
//      back with the only host synchronisation before the join;
//   3. one ncclGroupStart/End holds every ncclSend/ncclRecv: the all-to-all of
//      the partitioned views and the all-gather (send to every peer) of the
//      replicated ones, straight into persistent receive buffers (rank order;
//      the rank's own part is a device copy);
//   4. the single-GPU executor runs on zero-copy relations over the receive
//      buffers (bound once while the sizes do not change);
//   5. ncclAllReduce sums the result (count as four 32-bit limbs in u64 words,
//      checksum as two halves) and takes the MIN; outputs are disjoint by the
//      first variable, so the sums are the global result.
// NCCL is loaded on first use with dlopen (an already-loaded libnccl.so.2,
// e.g. torch's, is reused), so libfjg.so itself has no NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

namespace {

struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    const char* env = getenv("FJG_NCCL_LIB");
    if (!h && env) h = dlopen(env, RTLD_NOW);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW);
    if (!h) {
      a.err = std::string("NCCL not found (dlopen libnccl.so.2): ") + dlerror();
      return a;
    }
#define FJG_SYM(name)                                                   \
  a.name = reinterpret_cast<decltype(a.name)>(dlsym(h, "nccl" #name)); \
  if (!a.name) {                                                        \
    a.err = "NCCL symbol nccl" #name " missing";                        \
    return a;                                                           \
  }
    FJG_SYM(GetUniqueId)
    FJG_SYM(CommInitRank)
    FJG_SYM(CommDestroy)
    FJG_SYM(GroupStart)
    FJG_SYM(GroupEnd)
    FJG_SYM(Send)
    FJG_SYM(Recv)
    FJG_SYM(AllGather)
    FJG_SYM(AllReduce)
    FJG_SYM(GetErrorString)
#undef FJG_SYM
    a.ok = true;
    return a;
  }();
  if (!api.ok) throw fj::ResourceError(api.err);
  return api;
}

void nck(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  const std::string msg = std::string("NCCL error in ") + what + ": " + nccl().GetErrorString(r);
  if (r == ncclSystemError || r == ncclUnhandledCudaError) throw fj::ResourceError(msg);
  if (r == ncclInvalidArgument || r == ncclInvalidUsage) throw fj::ValidationError(msg);
  throw fj::EngineError(msg);
}

// meta[d] = rows for destination d (from the cumulative offsets), or `rows` for all d
__global__ void k_exchange_meta(const uint32_t* __restrict__ tot, uint64_t rows, int nranks, uint64_t* meta) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d < nranks) meta[d] = tot ? (uint64_t)(tot[d + 1] - tot[d]) : rows;
}

}  // namespace

struct fjg_comm {
  fjg_engine* eng = nullptr;
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
};

struct ExchangeView {
  int base = 0;
  int col = -1;  // column of the first variable (partitioned) or -1 (replicated)
  std::vector<int32_t*> send;  // partitioned: grouped rows (local slice size)
  std::vector<int32_t*> recv;  // rows held after the exchange
  uint64_t recv_rows = 0, recv_cap = 0, send_cap = 0;
  fjg_relation* rel = nullptr;  // zero-copy over recv
};

struct fjg_sharded {
  fjg_comm* comm = nullptr;
  std::string query_json, plan_json;
  std::vector<fjg_relation*> bases;  // local slices (caller-owned)
  std::vector<int> atom_view;
  std::vector<ExchangeView> views;
  fjg_query* q = nullptr;
  uint32_t* d_tot = nullptr;   // [nviews][nranks + 1]
  uint64_t* d_meta = nullptr;  // [nviews][nranks] local, then [nranks][nviews][nranks] gathered
  uint64_t* d_meta_all = nullptr;
  uint64_t* h_meta_all = nullptr;  // pinned
  uint64_t* d_words = nullptr;     // 6 reduction words + min
  uint64_t* h_words = nullptr;     // pinned
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
};

namespace {

void sharded_free_buffers(fjg_sharded* s) {
  fjg_engine* eng = s->comm->eng;
  for (auto& v : s->views) {
    for (auto* p : v.send) eng->pool->free(p);
    for (auto* p : v.recv) eng->pool->free(p);
    v.send.clear();
    v.recv.clear();
    if (v.rel) fjg_relation_destroy(v.rel);
    v.rel = nullptr;
  }
}

// receive offsets of view v from every source rank (rank order)
std::vector<uint64_t> recv_offsets(const uint64_t* M, int nviews, int G, int v, int rank, bool partitioned) {
  std::vector<uint64_t> off(G + 1, 0);
  for (int src = 0; src < G; ++src) {
    const uint64_t* row = M + ((uint64_t)src * nviews + v) * G;
    off[src + 1] = off[src] + (partitioned ? row[rank] : row[0]);
  }
  return off;
}

}  // namespace

extern "C" {

int fjg_comm_unique_id(void* id_out) {
  return guard([&] {
    if (!id_out) throw fj::ValidationError("fjg_comm_unique_id: null output");
    ncclUniqueId id;
    nck(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(ncclUniqueId) == FJG_COMM_ID_BYTES, "ncclUniqueId size");
    memcpy(id_out, &id, sizeof(id));
  });
}

int fjg_comm_create(fjg_engine* eng, const void* id, int nranks, int rank, fjg_comm** out) {
  return guard([&] {
    if (!eng || !id || !out) throw fj::ValidationError("fjg_comm_create: null argument");
    if (nranks < 1 || nranks > 1024 || rank < 0 || rank >= nranks)
      throw fj::ValidationError("fjg_comm_create: need 0 <= rank < nranks <= 1024");
    ScopedDevice sd(eng->device);
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    auto* c = new fjg_comm();
    c->eng = eng;
    c->nranks = nranks;
    c->rank = rank;
    ncclResult_t r = nccl().CommInitRank(&c->comm, nranks, uid, rank);
    if (r != ncclSuccess) {
      delete c;
      nck(r, "ncclCommInitRank");
    }
    *out = c;
  });
}

int fjg_comm_size(const fjg_comm* c) { return c ? c->nranks : 0; }
int fjg_comm_rank(const fjg_comm* c) { return c ? c->rank : -1; }

void fjg_comm_destroy(fjg_comm* c) {
  if (!c) return;
  ScopedDevice sd(c->eng->device);
  cudaStreamSynchronize(c->eng->stream);
  if (c->comm) nccl().CommDestroy(c->comm);
  delete c;
}

int fjg_sharded_create(fjg_comm* comm, const char* query_json, const char* plan_json,
                       fjg_relation* const* local_bases, int nbases, const int* atom_base,
                       const int* first_var_col, int natoms, fjg_sharded** out) {
  return guard([&] {
    if (!comm || !query_json || !plan_json || !out || natoms < 1 || nbases < 1)
      throw fj::ValidationError("fjg_sharded_create: bad arguments");
    auto* s = new fjg_sharded();
    s->comm = comm;
    s->query_json = query_json;
    s->plan_json = plan_json;
    s->bases.assign(local_bases, local_bases + nbases);
    for (int b = 0; b < nbases; ++b)
      if (!s->bases[b] || s->bases[b]->eng != comm->eng) {
        delete s;
        throw fj::ValidationError("fjg_sharded_create: base relation on another engine");
      }
    for (int a = 0; a < natoms; ++a) {
      const int b = atom_base[a], c = first_var_col[a];
      if (b < 0 || b >= nbases || c < -1 || c >= s->bases[b]->ncols) {
        delete s;
        throw fj::ValidationError("fjg_sharded_create: atom " + std::to_string(a) + " has a bad base or column");
      }
      int v = -1;
      for (size_t i = 0; i < s->views.size(); ++i)
        if (s->views[i].base == b && s->views[i].col == c) v = (int)i;
      if (v < 0) {
        ExchangeView ev;
        ev.base = b;
        ev.col = c;
        s->views.push_back(ev);
        v = (int)s->views.size() - 1;
      }
      s->atom_view.push_back(v);
    }
    fjg_engine* eng = comm->eng;
    ScopedDevice sd(eng->device);
    const int G = comm->nranks, V = (int)s->views.size();
    s->d_tot = (uint32_t*)eng->pool->alloc((size_t)V * (G + 1) * 4);
    s->d_meta = (uint64_t*)eng->pool->alloc((size_t)V * G * 8);
    s->d_meta_all = (uint64_t*)eng->pool->alloc((size_t)G * V * G * 8);
    s->d_words = (uint64_t*)eng->pool->alloc(8 * 8);
    CK(cudaMallocHost(&s->h_meta_all, (size_t)G * V * G * 8));
    CK(cudaMallocHost(&s->h_words, 8 * 8));
    for (auto& e : s->ev) CK(cudaEventCreate(&e));
    *out = s;
  });
}

void fjg_sharded_destroy(fjg_sharded* s) {
  if (!s) return;
  fjg_engine* eng = s->comm->eng;
  ScopedDevice sd(eng->device);
  cudaStreamSynchronize(eng->stream);
  if (s->q) fjg_query_destroy(s->q);
  sharded_free_buffers(s);
  eng->pool->free(s->d_tot);
  eng->pool->free(s->d_meta);
  eng->pool->free(s->d_meta_all);
  eng->pool->free(s->d_words);
  if (s->h_meta_all) cudaFreeHost(s->h_meta_all);
  if (s->h_words) cudaFreeHost(s->h_words);
  for (auto& e : s->ev)
    if (e) cudaEventDestroy(e);
  delete s;
}

int fjg_execute_multi(fjg_sharded* s, const fjg_exec_options* opts, fjg_result* out, fjg_multi_info* info) {
  return guard([&] {
    if (!s || !out) throw fj::ValidationError("fjg_execute_multi: null argument");
    if (opts && opts->output_mode == FJG_OUT_ENUMERATE)
      throw fj::ValidationError("fjg_execute_multi: enumerate mode is single-GPU (fjg_execute)");
    fjg_comm* cm = s->comm;
    fjg_engine* eng = cm->eng;
    ScopedDevice sd(eng->device);
    const NcclApi& N = nccl();
    const int G = cm->nranks, V = (int)s->views.size(), me = cm->rank;
    cudaStream_t st = eng->stream;
    const bool timing = opts && opts->collect_timing;
    const uint32_t l0 = eng->launches, s0 = eng->syncs;
    if (timing) CK(cudaEventRecord(s->ev[0], st));
    // (1) partition kernels into the send buffers + local metadata rows
    for (int v = 0; v < V; ++v) {
      ExchangeView& ev = s->views[v];
      const fjg_relation* in = s->bases[ev.base];
      uint32_t* tot = s->d_tot + (size_t)v * (G + 1);
      if (ev.col >= 0) {
        if (ev.send.empty() || ev.send_cap < in->nrows) {
          for (auto* p : ev.send) eng->pool->free(p);
          ev.send.clear();
          ev.send_cap = std::max<uint64_t>(in->nrows, 1);
          for (int c = 0; c < in->ncols; ++c) ev.send.push_back((int32_t*)eng->pool->alloc(ev.send_cap * 4));
        }
        partition_async(in, ev.col, G, ev.send.data(), tot);
      }
      LAUNCH(eng, k_exchange_meta<<<(G + 255) / 256, 256, 0, st>>>(ev.col >= 0 ? tot : nullptr, in->nrows, G,
                                                                   s->d_meta + (size_t)v * G));
    }
    // (2) one all-gather of every view's metadata, one host read
    nck(N.AllGather(s->d_meta, s->d_meta_all, (size_t)V * G, ncclUint64, cm->comm, st), "ncclAllGather(meta)");
    CK(cudaMemcpyAsync(s->h_meta_all, s->d_meta_all, (size_t)G * V * G * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    ++eng->syncs;
    const uint64_t* M = s->h_meta_all;  // M[src][view][dst]
    // (3) receive buffers, then one group of sends / receives
    bool rebind = s->q == nullptr;
    uint64_t sent = 0, received = 0;
    for (int v = 0; v < V; ++v) {
      ExchangeView& ev = s->views[v];
      const std::vector<uint64_t> off = recv_offsets(M, V, G, v, me, ev.col >= 0);
      const uint64_t rows = off[G];
      const int nc = s->bases[ev.base]->ncols;
      if (ev.recv.empty() || ev.recv_cap < rows || rows != ev.recv_rows) {
        if (ev.recv.empty() || ev.recv_cap < rows) {
          for (auto* p : ev.recv) eng->pool->free(p);
          ev.recv.clear();
          ev.recv_cap = std::max<uint64_t>(rows, 1);
          for (int c = 0; c < nc; ++c) ev.recv.push_back((int32_t*)eng->pool->alloc(ev.recv_cap * 4));
        }
        ev.recv_rows = rows;
        rebind = true;
      }
    }
    nck(N.GroupStart(), "ncclGroupStart");
    for (int v = 0; v < V; ++v) {
      ExchangeView& ev = s->views[v];
      const fjg_relation* in = s->bases[ev.base];
      const std::vector<uint64_t> roff = recv_offsets(M, V, G, v, me, ev.col >= 0);
      const uint64_t* mine = M + ((uint64_t)me * V + v) * G;
      uint64_t soff = 0;
      for (int peer = 0; peer < G; ++peer) {
        const uint64_t nsend = ev.col >= 0 ? mine[peer] : in->nrows;
        const uint64_t nrecv = roff[peer + 1] - roff[peer];
        for (int c = 0; c < in->ncols; ++c) {
          const int32_t* src = ev.col >= 0 ? ev.send[c] + soff : in->cols[c];
          if (peer == me) {
            if (nsend)
              CK(cudaMemcpyAsync(ev.recv[c] + roff[peer], src, nsend * 4, cudaMemcpyDeviceToDevice, st));
            continue;
          }
          if (nsend) nck(N.Send(src, nsend, ncclInt32, peer, cm->comm, st), "ncclSend");
          if (nrecv) nck(N.Recv(ev.recv[c] + roff[peer], nrecv, ncclInt32, peer, cm->comm, st), "ncclRecv");
          if (peer != me) {
            sent += nsend * 4;
            received += nrecv * 4;
          }
        }
        if (ev.col >= 0) soff += nsend;
      }
    }
    nck(N.GroupEnd(), "ncclGroupEnd");
    if (timing) CK(cudaEventRecord(s->ev[1], st));
    // (4) the single-GPU executor over zero-copy relations of the received rows
    if (rebind) {
      if (s->q) fjg_query_destroy(s->q);
      s->q = nullptr;
      for (auto& ev : s->views) {
        if (ev.rel) fjg_relation_destroy(ev.rel);
        ev.rel = nullptr;
        fjg_relation* r = nullptr;
        const int rc = fjg_relation_from_device(eng, ev.recv.data(), (int)ev.recv.size(), ev.recv_rows, 0, &r);
        if (rc) throw fj::EngineError(std::string("binding exchanged rows: ") + fjg_last_error());
        ev.rel = r;
      }
      std::vector<fjg_relation*> arels;
      for (int v : s->atom_view) arels.push_back(s->views[v].rel);
      const int rc = fjg_query_create(eng, s->query_json.c_str(), s->plan_json.c_str(), arels.data(),
                                      (int)arels.size(), &s->q);
      if (rc) {
        s->q = nullptr;
        const std::string m = fjg_last_error();
        if (rc == FJG_E_PARSE) throw fj::ParseError(m);
        if (rc == FJG_E_VALIDATION) throw fj::ValidationError(m);
        if (rc == FJG_E_RESOURCE) throw fj::ResourceError(m);
        throw fj::EngineError(m);
      }
    }
    fjg_result local{};
    const int rc = fjg_execute(s->q, opts, &local);
    if (rc) {
      const std::string m = fjg_last_error();
      if (rc == FJG_E_VALIDATION) throw fj::ValidationError(m);
      if (rc == FJG_E_RESOURCE) throw fj::ResourceError(m);
      throw fj::EngineError(m);
    }
    // (5) all-reduce of the result words (the executor left them in its counters)
    if (timing) CK(cudaEventRecord(s->ev[2], st));
    uint64_t* w = s->h_words;
    w[0] = local.count_lo & 0xffffffffull;
    w[1] = local.count_lo >> 32;
    w[2] = local.count_hi & 0xffffffffull;
    w[3] = local.count_hi >> 32;
    w[4] = local.checksum & 0xffffffffull;
    w[5] = local.checksum >> 32;
    w[6] = (uint64_t)(local.has_min ? local.min_value : LLONG_MAX);
    CK(cudaMemcpyAsync(s->d_words, w, 7 * 8, cudaMemcpyHostToDevice, st));
    nck(N.GroupStart(), "ncclGroupStart");
    nck(N.AllReduce(s->d_words, s->d_words, 6, ncclUint64, ncclSum, cm->comm, st), "ncclAllReduce(sum)");
    nck(N.AllReduce(s->d_words + 6, s->d_words + 6, 1, ncclInt64, ncclMin, cm->comm, st), "ncclAllReduce(min)");
    nck(N.GroupEnd(), "ncclGroupEnd");
    CK(cudaMemcpyAsync(w, s->d_words, 7 * 8, cudaMemcpyDeviceToHost, st));
    if (timing) CK(cudaEventRecord(s->ev[3], st));
    CK(cudaStreamSynchronize(st));
    ++eng->syncs;
    // recombine: limbs (each a sum of G 32-bit values) -> 128-bit count
    unsigned __int128 cnt = (unsigned __int128)w[0] + ((unsigned __int128)w[1] << 32) +
                            ((unsigned __int128)w[2] << 64) + ((unsigned __int128)w[3] << 96);
    *out = local;
    out->count_lo = (uint64_t)cnt;
    out->count_hi = (uint64_t)(cnt >> 64);
    out->checksum = w[4] + (w[5] << 32);
    out->has_min = (int64_t)w[6] != LLONG_MAX;
    out->min_value = out->has_min ? (int64_t)w[6] : 0;
    out->kernel_launches = eng->launches - l0;
    out->host_syncs = eng->syncs - s0;
    if (info) {
      memset(info, 0, sizeof(*info));
      info->local_count_lo = local.count_lo;
      info->local_count_hi = local.count_hi;
      info->local_checksum = local.checksum;
      info->bytes_sent = sent;
      info->bytes_received = received;
      info->nviews = V;
      for (int v = 0; v < V && v < FJG_MAX_VIEWS; ++v) info->view_rows[v] = s->views[v].recv_rows;
      if (timing) {
        float a = 0, b = 0;
        CK(cudaEventElapsedTime(&a, s->ev[0], s->ev[1]));
        CK(cudaEventElapsedTime(&b, s->ev[2], s->ev[3]));
        info->exchange_ms = a;
        info->reduce_ms = b;
      }
    }
  });
}

// Host-side layout of an exchange (test hook, no device work): given the
// gathered metadata M[src][view][dst] (u64), the receive row offsets of every
// view from every source rank at `rank`: off[view][src], rows[view].
int fjg_exchange_layout(const uint64_t* meta, int nviews, int nranks, int rank, const int* partitioned,
                        uint64_t* recv_off, uint64_t* recv_rows) {
  return guard([&] {
    if (nranks < 1 || rank < 0 || rank >= nranks || nviews < 0) throw fj::ValidationError("bad layout arguments");
    for (int v = 0; v < nviews; ++v) {
      const std::vector<uint64_t> off = recv_offsets(meta, nviews, nranks, v, rank, partitioned[v] != 0);
      for (int src = 0; src < nranks; ++src) recv_off[(size_t)v * nranks + src] = off[src];
      recv_rows[v] = off[nranks];
    }
  });
}

}  // extern "C"
