// C-ABI for the host plan compiler and error plumbing
// (error.hpp:8-33). Device entry points live in engine.cu.
#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/fjg.h"
#include "fj_errors.hpp"
#include "fj_hash.hpp"
#include "fj_json.hpp"
#include "fj_plan.hpp"

namespace fjg {
static thread_local std::string g_last_error;
void set_last_error(const std::string& s) { g_last_error = s; }
}  // namespace fjg

namespace {

template <class F>
int guard(F&& f) {
  try {
    f();
    return FJG_OK;
  } catch (const fj::Error& e) {
    fjg::set_last_error(e.what());
    return e.code();
  } catch (const std::exception& e) {
    fjg::set_last_error(e.what());
    return FJG_E_ENGINE;
  }
}

void emit(const std::string& s, char* out, size_t cap, size_t* needed) {
  if (needed) *needed = s.size() + 1;
  if (!out || cap < s.size() + 1) throw fj::ResourceError("output buffer too small");
  std::memcpy(out, s.c_str(), s.size() + 1);
}

std::string set_json(const std::set<std::string>& s) {
  std::string o = "[";
  bool first = true;
  for (auto& x : s) {
    o += (first ? "" : ",") + fj::json::quote(x);
    first = false;
  }
  return o + "]";
}

}  // namespace

extern "C" {

const char* fjg_last_error(void) { return fjg::g_last_error.c_str(); }

int fjg_abi_version(void) { return 5; }  // 3: fjg_result.first_node_ms; 4: fjg_comm / fjg_execute_multi; 5: fjg_relation_create_i64

int fjg_compile_plan(const char* query_json, int mode, int factor_fixpoint, char* out, size_t cap, size_t* needed) {
  return guard([&] {
    if (mode < 0 || mode > 2) throw fj::ValidationError("mode must be binary(0), free(1) or generic(2)");
    auto plan = fj::compile_query(query_json, static_cast<fj::PlanMode>(mode), factor_fixpoint != 0);
    emit(fj::plan_to_json(plan), out, cap, needed);
  });
}

int fjg_plan_op(const char* op_c, const char* query_json, const char* arg_json, char* out, size_t cap,
                size_t* needed) {
  return guard([&] {
    const std::string op = op_c;
    auto qv = fj::json::parse(query_json);
    auto query = fj::query_from_json(qv);
    auto arg = fj::json::parse(arg_json ? arg_json : "null");
    std::string res;
    if (op == "head_vars") {
      auto h = fj::head_variables(query);
      res = "[";
      for (size_t i = 0; i < h.size(); ++i) res += (i ? "," : "") + fj::json::quote(h[i]);
      res += "]";
    } else if (op == "binary2fj") {
      std::vector<std::string> seg;
      for (auto& x : arg.arr) seg.push_back(x.str);
      std::vector<std::string> warnings;
      auto plan = fj::binary2fj(seg, query, &warnings);
      res = "{\"plan\":" + fj::plan_to_json(plan) + ",\"warnings\":[";
      for (size_t i = 0; i < warnings.size(); ++i) res += (i ? "," : "") + fj::json::quote(warnings[i]);
      res += "]}";
    } else if (op == "decompose") {
      auto segs = fj::decompose_bushy(*fj::tree_from_json(arg));
      res = "[";
      for (size_t s = 0; s < segs.size(); ++s) {
        res += s ? ",[" : "[";
        for (size_t i = 0; i < segs[s].size(); ++i) res += (i ? "," : "") + fj::json::quote(segs[s][i]);
        res += "]";
      }
      res += "]";
    } else if (op == "covers" || op == "vs" || op == "avs") {
      auto plan = fj::plan_from_json(arg.at("plan"), query);
      const size_t k = (size_t)arg.at("k").num;
      if (op == "covers") {
        auto c = fj::covers(plan, k);
        res = "[";
        for (size_t i = 0; i < c.size(); ++i) res += (i ? "," : "") + std::to_string(c[i]);
        res += "]";
      } else if (op == "vs") {
        if (k >= plan.nodes.size()) throw fj::ValidationError("vs: node index out of range");
        res = set_json(fj::vs(plan.nodes[k]));
      } else {
        res = set_json(fj::avs(plan, k));
      }
    } else {
      auto plan = fj::plan_from_json(arg, query);
      if (op == "factor")
        res = fj::plan_to_json(fj::factor(plan, false));
      else if (op == "factor_fixpoint")
        res = fj::plan_to_json(fj::factor(plan, true));
      else if (op == "fj_to_gj")
        res = fj::plan_to_json(fj::fj_to_gj_plan(plan));
      else if (op == "schemas")
        res = fj::schemas_to_json(fj::derive_ght_schemas(plan));
      else if (op == "validate")
        res = fj::json::quote(fj::validate(plan));
      else if (op == "gj_order") {
        auto o = fj::gj_variable_order(plan);
        res = "[";
        for (size_t i = 0; i < o.size(); ++i) res += (i ? "," : "") + fj::json::quote(o[i]);
        res += "]";
      } else
        throw fj::ValidationError("unknown plan op '" + op + "'");
    }
    emit(res, out, cap, needed);
  });
}

// load_csv: header-less, comma-separated, no quoting
// (reject fields with quotes), int columns. Rows land row-major
// in `out` (capacity cap_rows x ncols); *rows receives the row count even
// when the buffer is too small (then FJG_E_RESOURCE), so callers can size it.
int fjg_parse_csv(const char* path, int ncols, int32_t* out, uint64_t cap_rows, uint64_t* rows) {
  return guard([&] {
    if (ncols < 1) throw fj::ValidationError("load_csv: ncols must be >= 1");
    FILE* f = std::fopen(path, "rb");
    if (!f) throw fj::IoError(std::string("load_csv: cannot open ") + path);
    std::string data;
    char buf[1 << 16];
    size_t got;
    while ((got = std::fread(buf, 1, sizeof(buf), f)) > 0) data.append(buf, got);
    std::fclose(f);
    uint64_t r = 0;
    size_t i = 0;
    const size_t n = data.size();
    while (i < n) {
      size_t e = data.find('\n', i);
      if (e == std::string::npos) e = n;
      size_t end = e;
      if (end > i && data[end - 1] == '\r') --end;
      if (end > i) {
        int c = 0;
        size_t a = i;
        while (true) {
          size_t b = a;
          while (b < end && data[b] != ',') ++b;
          const std::string field = data.substr(a, b - a);
          if (field.find('"') != std::string::npos)
            throw fj::ParseError("load_csv: quoted field at row " + std::to_string(r) + " column " +
                                 std::to_string(c));
          if (c >= ncols)
            throw fj::ValidationError("load_csv: row " + std::to_string(r) + " has more than " +
                                      std::to_string(ncols) + " fields");
          char* stop = nullptr;
          errno = 0;
          const long long v = std::strtoll(field.c_str(), &stop, 10);
          if (field.empty() || *stop != '\0' || errno == ERANGE)
            throw fj::ParseError("load_csv: cannot parse '" + field + "' as int at row " + std::to_string(r) +
                                 " column " + std::to_string(c));
          if (v < INT32_MIN || v > INT32_MAX)
            throw fj::ParseError("load_csv: value " + field + " at row " + std::to_string(r) +
                                 " exceeds the device's int32 columns");
          if (out && r < cap_rows) out[r * (uint64_t)ncols + c] = (int32_t)v;
          ++c;
          if (b >= end) break;
          a = b + 1;
        }
        if (c != ncols)
          throw fj::ValidationError("load_csv: row " + std::to_string(r) + " has " + std::to_string(c) +
                                    " fields, expected " + std::to_string(ncols));
        ++r;
      }
      i = e + 1;
    }
    *rows = r;
    if (r > cap_rows) throw fj::ResourceError("load_csv: buffer too small");
  });
}

uint64_t fjg_host_tuple_hash(const int64_t* vals, int arity) {
  uint64_t h = fj::kTupleHashSeed;
  for (int i = 0; i < arity; ++i) h = fj::tuple_hash_step(h, vals[i]);
  return h;
}

}  // extern "C"
