// A compiled C++ caller of the multi-GPU C-ABI (include/fjg.h): what a
// maintainer's host program does, with no Python or torch in the process.
// Reads a workload file written by tests/test_capi_multi.py, runs
// fjg_execute_multi at world size 1 (NCCL communicator from
// fjg_comm_unique_id), twice, and prints the global results. Test program.
//
// file layout (little endian): i32 nbases; per base: i32 ncols, u64 nrows,
// ncols x nrows i32 (column-major); i32 natoms; natoms x i32 atom_base;
// natoms x i32 first_var_col; i32 output_mode; i32 min_var;
// u64 len + query json; u64 len + plan json.
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "fjg.h"

static int fail(const char* what) {
  std::fprintf(stderr, "%s: %s\n", what, fjg_last_error());
  return 2;
}

template <class T>
static T rd(FILE* f) {
  T v{};
  if (std::fread(&v, sizeof(T), 1, f) != 1) throw 1;
  return v;
}

int main(int argc, char** argv) {
  if (argc < 2) return 1;
  FILE* f = std::fopen(argv[1], "rb");
  if (!f) return 1;
  std::vector<std::vector<std::vector<int32_t>>> bases;
  std::vector<int> atom_base, fvc;
  std::string query, plan;
  int output_mode = 0, min_var = -1;
  try {
    const int nb = rd<int32_t>(f);
    for (int b = 0; b < nb; ++b) {
      const int nc = rd<int32_t>(f);
      const uint64_t n = rd<uint64_t>(f);
      std::vector<std::vector<int32_t>> cols(nc, std::vector<int32_t>(n));
      for (auto& c : cols)
        if (n && std::fread(c.data(), 4, n, f) != n) throw 1;
      bases.push_back(std::move(cols));
    }
    const int na = rd<int32_t>(f);
    for (int a = 0; a < na; ++a) atom_base.push_back(rd<int32_t>(f));
    for (int a = 0; a < na; ++a) fvc.push_back(rd<int32_t>(f));
    output_mode = rd<int32_t>(f);
    min_var = rd<int32_t>(f);
    for (std::string* s : {&query, &plan}) {
      const uint64_t len = rd<uint64_t>(f);
      s->resize(len);
      if (len && std::fread(&(*s)[0], 1, len, f) != len) throw 1;
    }
  } catch (int) {
    return 1;
  }
  std::fclose(f);

  fjg_engine* eng = nullptr;
  if (fjg_engine_create(0, &eng)) return fail("fjg_engine_create");
  unsigned char id[FJG_COMM_ID_BYTES];
  if (fjg_comm_unique_id(id)) return fail("fjg_comm_unique_id");
  fjg_comm* comm = nullptr;
  if (fjg_comm_create(eng, id, 1, 0, &comm)) return fail("fjg_comm_create");
  std::vector<fjg_relation*> rels;
  for (auto& cols : bases) {
    std::vector<const int32_t*> ptrs;
    for (auto& c : cols) ptrs.push_back(c.data());
    fjg_relation* r = nullptr;
    if (fjg_relation_create(eng, ptrs.data(), (int)ptrs.size(), cols[0].size(), &r)) return fail("relation");
    rels.push_back(r);
  }
  fjg_sharded* sq = nullptr;
  if (fjg_sharded_create(comm, query.c_str(), plan.c_str(), rels.data(), (int)rels.size(), atom_base.data(),
                         fvc.data(), (int)atom_base.size(), &sq))
    return fail("fjg_sharded_create");
  fjg_exec_options o{};
  o.dynamic_cover = 1;
  o.output_mode = output_mode;
  o.min_var = min_var;
  o.collect_timing = 1;
  for (int rep = 0; rep < 2; ++rep) {
    fjg_result r{};
    fjg_multi_info info{};
    if (fjg_execute_multi(sq, &o, &r, &info)) return fail("fjg_execute_multi");
    std::printf("{\"count_lo\": %llu, \"count_hi\": %llu, \"checksum\": %llu, \"has_min\": %d, \"min\": %lld, "
                "\"local_count_lo\": %llu, \"nviews\": %d}\n",
                (unsigned long long)r.count_lo, (unsigned long long)r.count_hi, (unsigned long long)r.checksum,
                r.has_min, (long long)r.min_value, (unsigned long long)info.local_count_lo, info.nviews);
  }
  fjg_sharded_destroy(sq);
  for (auto* r : rels) fjg_relation_destroy(r);
  fjg_comm_destroy(comm);
  fjg_engine_destroy(eng);
  return 0;
}
