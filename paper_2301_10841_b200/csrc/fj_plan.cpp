// Host query IR + plan compiler. See fj_plan.hpp for the reference map.
#include "fj_plan.hpp"

#include <algorithm>
#include <map>

namespace fj {

namespace {

const Atom& find_atom(const std::vector<Atom>& query, const std::string& rel) {
  for (auto& a : query)
    if (a.relation == rel) return a;
  throw ValidationError("unknown relation '" + rel + "'");
}

bool contains(const std::vector<std::string>& v, const std::string& x) {
  return std::find(v.begin(), v.end(), x) != v.end();
}

}  // namespace

// union of all subatom variable sets.
std::set<std::string> vs(const PlanNode& node) {
  std::set<std::string> out;
  for (auto& s : node.subatoms) out.insert(s.vars.begin(), s.vars.end());
  return out;
}

// avs(phi_k) = U_{j<k} vs(phi_j).
std::set<std::string> avs(const FreeJoinPlan& plan, size_t k) {
  if (k > plan.nodes.size()) throw ValidationError("avs: node index out of range");
  std::set<std::string> out;
  for (size_t j = 0; j < k; ++j) {
    auto v = vs(plan.nodes[j]);
    out.insert(v.begin(), v.end());
  }
  return out;
}

// SPEC.md:143-149 (Def 3.5): subatoms whose vars include vs - avs, node order.
std::vector<size_t> covers(const FreeJoinPlan& plan, size_t k) {
  if (k >= plan.nodes.size()) throw ValidationError("covers: node index out of range");
  auto v = vs(plan.nodes[k]);
  auto a = avs(plan, k);
  std::vector<std::string> need;
  for (auto& x : v)
    if (!a.count(x)) need.push_back(x);
  std::vector<size_t> out;
  const auto& subs = plan.nodes[k].subatoms;
  for (size_t i = 0; i < subs.size(); ++i) {
    bool ok = true;
    for (auto& x : need)
      if (!contains(subs[i].vars, x)) {
        ok = false;
        break;
      }
    if (ok) out.push_back(i);
  }
  return out;
}

// (a) relation uniqueness per node, (b) a cover per node,
// (c) partitioning of every atom's variables. Earliest violation reported.
std::string validate(const FreeJoinPlan& plan) {
  std::map<std::string, std::vector<std::string>> seen;  // relation -> vars used so far
  for (size_t k = 0; k < plan.nodes.size(); ++k) {
    const auto& subs = plan.nodes[k].subatoms;
    if (subs.empty()) return "node " + std::to_string(k) + ": empty node";
    std::set<std::string> rels;
    for (auto& s : subs) {
      if (!rels.insert(s.relation).second)
        return "node " + std::to_string(k) + ": relation " + s.relation + " appears twice";
    }
    if (covers(plan, k).empty()) return "node " + std::to_string(k) + ": node has no cover";
    for (auto& s : subs) {
      const Atom* atom = nullptr;
      for (auto& a : plan.query)
        if (a.relation == s.relation) atom = &a;
      if (!atom) return "node " + std::to_string(k) + ": unknown relation " + s.relation;
      std::set<std::string> uniq(s.vars.begin(), s.vars.end());
      if (uniq.size() != s.vars.size())
        return "node " + std::to_string(k) + ": duplicate variable in subatom of " + s.relation;
      auto& used = seen[s.relation];
      for (auto& x : s.vars) {
        if (!contains(atom->vars, x))
          return "node " + std::to_string(k) + ": partitioning: variable " + x + " not in atom " +
                 s.relation;
        if (contains(used, x))
          return "node " + std::to_string(k) + ": partitioning: variable " + x +
                 " covered twice for atom " + s.relation;
        used.push_back(x);
      }
    }
  }
  for (auto& a : plan.query) {
    auto it = seen.find(a.relation);
    if (it == seen.end()) return "partitioning: atom " + a.relation + " not covered";
    for (auto& x : a.vars)
      if (!contains(it->second, x))
        return "partitioning: variable " + x + " of atom " + a.relation + " not covered";
  }
  return "";
}

// SPEC.md:195-203 / PAPER §2.2: every join node that is a right child becomes
// the root of a new subplan whose materialised result feeds the parent.
static std::string decompose_rec(const BinaryPlanTree& t, std::vector<std::vector<std::string>>& segs) {
  std::vector<const BinaryPlanTree*> rights;
  const BinaryPlanTree* cur = &t;
  while (!cur->is_leaf()) {
    rights.push_back(cur->right.get());
    cur = cur->left.get();
  }
  std::reverse(rights.begin(), rights.end());
  std::vector<std::string> seg{cur->leaf};
  for (auto* r : rights) {
    if (r->is_leaf())
      seg.push_back(r->leaf);
    else
      seg.push_back(decompose_rec(*r, segs));
  }
  segs.push_back(seg);
  return "P" + std::to_string(segs.size());
}

std::vector<std::vector<std::string>> decompose_bushy(const BinaryPlanTree& tree) {
  std::vector<std::vector<std::string>> segs;
  decompose_rec(tree, segs);
  return segs;
}

// Fig 9. avs(phi) is the set of variables bound after
// iterating the current node's cover, i.e. every variable
// seen so far; subatom variables keep the atom's own order.
FreeJoinPlan binary2fj(const std::vector<std::string>& segment, const std::vector<Atom>& query,
                       std::vector<std::string>* warnings) {
  if (segment.empty()) throw ValidationError("binary2fj: empty segment");
  FreeJoinPlan plan;
  for (auto& name : segment) plan.query.push_back(find_atom(query, name));
  std::set<std::string> bound;
  const Atom& r = plan.query[0];
  PlanNode phi;
  phi.subatoms.push_back({r.relation, r.vars});
  bound.insert(r.vars.begin(), r.vars.end());
  for (size_t i = 1; i < plan.query.size(); ++i) {
    const Atom& s = plan.query[i];
    Subatom probe{s.relation, {}}, rest{s.relation, {}};
    for (auto& x : s.vars) (bound.count(x) ? probe.vars : rest.vars).push_back(x);
    if (probe.vars.empty() && warnings)
      warnings->push_back("cartesian product: " + s.relation + " shares no variable with its prefix");
    phi.subatoms.push_back(probe);
    plan.nodes.push_back(phi);
    phi = PlanNode{};
    phi.subatoms.push_back(rest);
    bound.insert(rest.vars.begin(), rest.vars.end());
  }
  plan.nodes.push_back(phi);
  return plan;
}

// Fig 10: reverse pass over nodes i = n-1..1; within node
// i consider subatoms at positions >= 1 in order, move alpha to node i-1 iff
// alpha.vars ⊆ avs(phi_i) and node i-1 has no subatom of alpha's relation;
// stop at the first non-movable subatom.
FreeJoinPlan factor(const FreeJoinPlan& in, bool fixpoint) {
  FreeJoinPlan plan = in;
  while (true) {
    bool moved_any = false;
    for (size_t i = plan.nodes.size(); i-- > 1;) {
      auto a = avs(plan, i);
      auto& phi = plan.nodes[i].subatoms;
      auto& prev = plan.nodes[i - 1].subatoms;
      size_t j = 1;
      while (j < phi.size()) {
        const Subatom al = phi[j];
        bool subset = true;
        for (auto& x : al.vars)
          if (!a.count(x)) subset = false;
        bool rel_free = true;
        for (auto& p : prev)
          if (p.relation == al.relation) rel_free = false;
        if (subset && rel_free) {
          phi.erase(phi.begin() + j);
          prev.push_back(al);
          moved_any = true;
        } else {
          break;
        }
      }
    }
    plan.nodes.erase(std::remove_if(plan.nodes.begin(), plan.nodes.end(),
                                    [](const PlanNode& n) { return n.subatoms.empty(); }),
                     plan.nodes.end());
    if (!fixpoint || !moved_any) break;
  }
  return plan;
}

// SPEC.md:223-231 / PAPER.md:816-828.
std::vector<GhtSchema> derive_ght_schemas(const FreeJoinPlan& plan) {
  std::vector<GhtSchema> out;
  for (auto& atom : plan.query) {
    GhtSchema s;
    s.relation = atom.relation;
    bool last_is_cover = false;
    for (auto& node : plan.nodes)
      for (size_t p = 0; p < node.subatoms.size(); ++p)
        if (node.subatoms[p].relation == atom.relation) {
          s.levels.push_back(node.subatoms[p].vars);
          last_is_cover = (p == 0);
        }
    if (!last_is_cover) {
      s.levels.push_back({});
      s.trailing_empty = true;
    }
    out.push_back(s);
  }
  return out;
}

// scan nodes in order; within a node, the cover's variables
// first, then the remaining subatoms' new variables in subatom order.
std::vector<std::string> gj_variable_order(const FreeJoinPlan& plan) {
  std::vector<std::string> order;
  for (size_t k = 0; k < plan.nodes.size(); ++k) {
    auto cov = covers(plan, k);
    const auto& subs = plan.nodes[k].subatoms;
    size_t c = cov.empty() ? 0 : cov[0];
    for (auto& x : subs[c].vars)
      if (!contains(order, x)) order.push_back(x);
    for (size_t i = 0; i < subs.size(); ++i)
      if (i != c)
        for (auto& x : subs[i].vars)
          if (!contains(order, x)) order.push_back(x);
  }
  return order;
}

// one node per variable v with R(v) for every atom holding v;
// the atom that introduced v in the source plan comes first, the others
// follow query atom order.
FreeJoinPlan fj_to_gj_plan(const FreeJoinPlan& plan) {
  std::map<std::string, std::string> introducer;
  for (size_t k = 0; k < plan.nodes.size(); ++k) {
    auto cov = covers(plan, k);
    const auto& subs = plan.nodes[k].subatoms;
    size_t c = cov.empty() ? 0 : cov[0];
    std::vector<size_t> order{c};
    for (size_t i = 0; i < subs.size(); ++i)
      if (i != c) order.push_back(i);
    for (size_t i : order)
      for (auto& x : subs[i].vars)
        if (!introducer.count(x)) introducer[x] = subs[i].relation;
  }
  FreeJoinPlan out;
  out.query = plan.query;
  for (auto& v : gj_variable_order(plan)) {
    PlanNode n;
    const std::string& first = introducer[v];
    n.subatoms.push_back({first, {v}});
    for (auto& a : plan.query)
      if (a.relation != first && contains(a.vars, v)) n.subatoms.push_back({a.relation, {v}});
    out.nodes.push_back(n);
  }
  // Atoms with no variables keep a single empty subatom in a final node.
  for (auto& a : plan.query)
    if (a.vars.empty()) {
      if (out.nodes.empty()) out.nodes.push_back(PlanNode{});
      out.nodes.back().subatoms.push_back({a.relation, {}});
    }
  return out;
}

std::vector<std::string> head_variables(const std::vector<Atom>& query) {
  std::vector<std::string> out;
  for (auto& a : query)
    for (auto& x : a.vars)
      if (!contains(out, x)) out.push_back(x);
  return out;
}

// ---- plan-file dialect ----

std::vector<Atom> query_from_json(const json::Value& v) {
  const json::Value& q = v.is_object() ? v.at("query") : v;
  if (!q.is_array()) throw ParseError("query must be an array of atoms");
  std::vector<Atom> out;
  std::set<std::string> names;
  for (auto& a : q.arr) {
    Atom atom;
    atom.relation = a.at("rel").str;
    if (!names.insert(atom.relation).second)
      throw ValidationError("relation '" + atom.relation +
                            "' appears twice; rename self-joins (SPEC.md:104)");
    std::set<std::string> uniq;
    for (auto& x : a.at("vars").arr) {
      if (!x.is_string()) throw ParseError("variable names must be strings");
      if (!uniq.insert(x.str).second)
        throw ValidationError("atom " + atom.relation + " repeats variable " + x.str);
      atom.vars.push_back(x.str);
    }
    out.push_back(atom);
  }
  return out;
}

std::shared_ptr<BinaryPlanTree> tree_from_json(const json::Value& v) {
  auto t = std::make_shared<BinaryPlanTree>();
  if (v.is_string()) {
    t->leaf = v.str;
    return t;
  }
  if (!v.is_array() || v.arr.size() != 3 || !v.arr[0].is_string() || v.arr[0].str != "join")
    throw ParseError("binary plan node must be \"R\" or [\"join\", l, r]");
  t->left = tree_from_json(v.arr[1]);
  t->right = tree_from_json(v.arr[2]);
  return t;
}

FreeJoinPlan plan_from_json(const json::Value& v, const std::vector<Atom>& query) {
  FreeJoinPlan plan;
  plan.query = query;
  if (!v.is_array()) throw ParseError("plan must be an array of nodes");
  for (auto& n : v.arr) {
    PlanNode node;
    if (!n.is_array()) throw ParseError("plan node must be an array");
    for (auto& s : n.arr) {
      if (!s.is_array() || s.arr.size() != 2) throw ParseError("subatom must be [rel, [vars]]");
      Subatom sub;
      sub.relation = s.arr[0].str;
      for (auto& x : s.arr[1].arr) sub.vars.push_back(x.str);
      node.subatoms.push_back(sub);
    }
    plan.nodes.push_back(node);
  }
  return plan;
}

static std::string vars_json(const std::vector<std::string>& vars) {
  std::string o = "[";
  for (size_t i = 0; i < vars.size(); ++i) o += (i ? "," : "") + json::quote(vars[i]);
  return o + "]";
}

std::string plan_to_json(const FreeJoinPlan& plan) {
  std::string o = "[";
  for (size_t k = 0; k < plan.nodes.size(); ++k) {
    o += k ? ",[" : "[";
    const auto& subs = plan.nodes[k].subatoms;
    for (size_t i = 0; i < subs.size(); ++i)
      o += (i ? "," : "") + std::string("[") + json::quote(subs[i].relation) + "," + vars_json(subs[i].vars) + "]";
    o += "]";
  }
  return o + "]";
}

std::string schemas_to_json(const std::vector<GhtSchema>& schemas) {
  std::string o = "{";
  for (size_t i = 0; i < schemas.size(); ++i) {
    o += (i ? "," : "") + json::quote(schemas[i].relation) + ":[";
    for (size_t l = 0; l < schemas[i].levels.size(); ++l)
      o += (l ? "," : "") + vars_json(schemas[i].levels[l]);
    o += "]";
  }
  return o + "}";
}

FreeJoinPlan compile_query(const std::string& query_json, PlanMode mode, bool factor_fixpoint,
                           std::vector<std::string>* warnings) {
  json::Value v = json::parse(query_json);
  std::vector<Atom> query = query_from_json(v);
  std::shared_ptr<BinaryPlanTree> tree;
  const json::Value* bp = v.is_object() ? v.find("binary_plan") : nullptr;
  if (bp && bp->kind != json::Value::Kind::Null) {
    tree = tree_from_json(*bp);
  } else {
    // default: left-deep in query order
    tree = std::make_shared<BinaryPlanTree>();
    tree->leaf = query.at(0).relation;
    for (size_t i = 1; i < query.size(); ++i) {
      auto j = std::make_shared<BinaryPlanTree>();
      j->left = tree;
      j->right = std::make_shared<BinaryPlanTree>();
      j->right->leaf = query[i].relation;
      tree = j;
    }
  }
  auto segs = decompose_bushy(*tree);
  if (segs.size() != 1)
    throw ValidationError("bushy binary plan decomposes into " + std::to_string(segs.size()) +
                          " segments; materialised segments (run_segments) are not supported yet");
  if (segs[0].size() != query.size())
    throw ValidationError("binary plan must mention every query atom exactly once");
  FreeJoinPlan plan = binary2fj(segs[0], query, warnings);
  plan.query = query;  // keep query atom order (head variable order)
  if (mode == PlanMode::Free) plan = factor(plan, factor_fixpoint);
  if (mode == PlanMode::Generic) plan = fj_to_gj_plan(plan);
  std::string err = validate(plan);
  if (!err.empty()) throw ValidationError("compiled plan invalid: " + err);
  return plan;
}

}  // namespace fj
