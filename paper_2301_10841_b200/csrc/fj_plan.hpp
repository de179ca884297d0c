// Host-side query IR and plan compiler (stays on the C++ host, per
// BASELINE.json north_star: "plan construction ... stays on the C++ host").
//
// Mirrors the reference's interfaces:
//   query-ir      SPEC.md:95-176  (Atom, Subatom, PlanNode, FreeJoinPlan,
//                                  BinaryPlanTree, vs, avs, covers, validate)
//   plan-compiler SPEC.md:178-261 (decompose_bushy, binary2fj (Fig 9),
//                                  factor (Fig 10), derive_ght_schemas,
//                                  fj_to_gj_plan)
// Variables are globally named strings.
#pragma once

#include <memory>
#include <set>
#include <string>
#include <vector>

#include "fj_errors.hpp"
#include "fj_json.hpp"

namespace fj {

// SPEC.md:100-105. Relation identifiers are unique per query (self-joins are
// renamed before they reach the IR).
struct Atom {
  std::string relation;
  std::vector<std::string> vars;
};

// SPEC.md:106-110 (Def 3.2).
struct Subatom {
  std::string relation;
  std::vector<std::string> vars;
  bool operator==(const Subatom& o) const { return relation == o.relation && vars == o.vars; }
};

// SPEC.md:111-115 (Def 3.3). Position 0 is the designated cover.
struct PlanNode {
  std::vector<Subatom> subatoms;
};

// SPEC.md:116-121.
struct FreeJoinPlan {
  std::vector<PlanNode> nodes;
  std::vector<Atom> query;
};

// Leaf(atom) | Join(left, right).
struct BinaryPlanTree {
  std::string leaf;  // non-empty iff leaf
  std::shared_ptr<BinaryPlanTree> left, right;
  bool is_leaf() const { return !left; }
};

// SPEC.md:183-187. `levels` lists the key group per level; when
// `trailing_empty` is true the last entry of `levels` is the empty level []
// (the flat leaf vector of PAPER.md:816-828).
struct GhtSchema {
  std::string relation;
  std::vector<std::vector<std::string>> levels;
  bool trailing_empty = false;
};

// ---- query-ir operations ----
std::set<std::string> vs(const PlanNode& node);
std::set<std::string> avs(const FreeJoinPlan& plan, size_t k);
std::vector<size_t> covers(const FreeJoinPlan& plan, size_t k);
std::string validate(const FreeJoinPlan& plan);                        // SPEC.md:150; "" == ok

// ---- plan-compiler operations ----
// Segments in dependency order; intermediate results are named "P<i>"
// (1-based, in creation order).
std::vector<std::vector<std::string>> decompose_bushy(const BinaryPlanTree& tree);
// Fig 9. `warnings` receives Cartesian-product notes
// (SPEC.md:208).
FreeJoinPlan binary2fj(const std::vector<std::string>& segment, const std::vector<Atom>& query,
                       std::vector<std::string>* warnings = nullptr);
// Fig 10, single reverse pass; positions >= 1 only
// (the position-0 cover always binds new variables).
FreeJoinPlan factor(const FreeJoinPlan& plan, bool fixpoint = false);
std::vector<GhtSchema> derive_ght_schemas(const FreeJoinPlan& plan);
FreeJoinPlan fj_to_gj_plan(const FreeJoinPlan& plan);
std::vector<std::string> gj_variable_order(const FreeJoinPlan& plan);

// Head variable order: first appearance across atoms in query order
// (canonical order for checksums).
std::vector<std::string> head_variables(const std::vector<Atom>& query);

// ---- plan-file dialect ----
std::vector<Atom> query_from_json(const json::Value& v);
std::shared_ptr<BinaryPlanTree> tree_from_json(const json::Value& v);
FreeJoinPlan plan_from_json(const json::Value& v, const std::vector<Atom>& query);
std::string plan_to_json(const FreeJoinPlan& plan);
std::string schemas_to_json(const std::vector<GhtSchema>& schemas);

enum class PlanMode { Binary = 0, Free = 1, Generic = 2 };

// The host pipeline of SPEC.md:475 up to the build phase:
// decompose -> binary2fj -> (factor if free) -> (fj_to_gj_plan if generic)
// -> validate. Only single-segment (left-deep) binary plans compile to one
// executable plan; bushy trees are rejected with ValidationError for now.
FreeJoinPlan compile_query(const std::string& query_json, PlanMode mode, bool factor_fixpoint,
                           std::vector<std::string>* warnings = nullptr);

}  // namespace fj
