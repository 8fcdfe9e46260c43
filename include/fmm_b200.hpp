// fmm_b200.hpp — header-only C++ mirror of the reference's tree / traversal / kernel-operator
// API (/root/reference/proj/include/fmm/{tree,traversal,kernels}.hpp) over the C-ABI of
// fmm_b200.h. Same names, argument meaning and exception types/messages as the reference, so
// reference call sites (engine.cpp:61-125, test_traversal.cpp:292-318) port by changing the
// namespace to fmm::b200. Link with paper_1203_0889_b200/lib/libfmm_b200.so.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "fmm_b200.h"

namespace fmm::b200 {

using Real = double;
using Vec3 = std::array<Real, 3>;

struct Body {  // types.hpp:14-18 (position, charge, accumulated potential) + acceleration
  Vec3 position{0, 0, 0};
  Real charge = 0.0;
  Real potential = 0.0;
  Vec3 acceleration{0, 0, 0};  // extension: -grad potential
};

// fmm_status -> the reference's exception types and texts
inline void check(int status, const fmm_ctx* ctx = nullptr) {
  if (status == FMM_OK) return;
  const std::string msg = fmm_last_error(ctx);
  if (status >= FMM_ERR_EMPTY_INPUT && status <= FMM_ERR_THETA) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

struct TraversalConfig {  // traversal.hpp:19-23
  Real theta = 0.5;
  std::size_t queue_threshold = 64;  // only moves the drain point; the GPU emits the same multiset
  bool mutual = false;
};

struct Cell {  // tree.hpp:21-36 (expansions live on the device)
  int level = 0;
  std::uint64_t morton_key = 0;
  Vec3 center{0, 0, 0};
  Real radius = 0.0;
  std::int32_t body_begin = 0, body_end = 0, child_begin = 0, child_count = 0, parent = -1;
  bool is_leaf() const { return child_count == 0; }
  std::int32_t body_count() const { return body_end - body_begin; }
};

// Device-resident tree (tree.hpp:41-59): build_tree() owns one context.
class Tree {
 public:
  Tree(std::vector<Body> bodies, int n_crit, int p, fmm_precision prec = FMM_PREC_FP64, Real theta = 0.5,
       int device = 0)
      : n_crit(n_crit), order(p) {
    if (bodies.empty()) throw std::invalid_argument("empty input");
    fmm_config cfg{p, n_crit, theta, 0, prec, device, 1};
    fmm_ctx* c = nullptr;
    check(fmm_create(&cfg, &c));
    ctx_.reset(c);
    std::vector<double> xyzq(4 * bodies.size());
    for (std::size_t i = 0; i < bodies.size(); ++i) {
      xyzq[4 * i] = bodies[i].position[0];
      xyzq[4 * i + 1] = bodies[i].position[1];
      xyzq[4 * i + 2] = bodies[i].position[2];
      xyzq[4 * i + 3] = bodies[i].charge;
    }
    check(fmm_set_bodies(ctx(), xyzq.data(), static_cast<std::int64_t>(bodies.size())), ctx());
    check(fmm_build_tree(ctx()), ctx());
    fmm_tree_info info{};
    check(fmm_get_tree_info(ctx(), &info), ctx());
    std::vector<std::int64_t> perm(bodies.size());
    check(fmm_get_permutation(ctx(), perm.data()), ctx());
    this->bodies.resize(bodies.size());
    for (std::size_t i = 0; i < bodies.size(); ++i) this->bodies[i] = bodies[perm[i]];
    load_cells(info.ncells);
  }

  fmm_ctx* ctx() const { return ctx_.get(); }

  std::vector<Cell> cells;
  std::vector<Body> bodies;  // tree (sorted) order
  int n_crit = 0;
  int order = 0;

  // Copies phi and acceleration of the last downward pass into `bodies` (tree order).
  void fetch_results() {
    std::vector<double> phi(bodies.size()), acc(3 * bodies.size());
    check(fmm_get_results(ctx(), phi.data(), acc.data(), 0), ctx());
    for (std::size_t i = 0; i < bodies.size(); ++i) {
      bodies[i].potential = phi[i];
      bodies[i].acceleration = {acc[3 * i], acc[3 * i + 1], acc[3 * i + 2]};
    }
  }

 private:
  void load_cells(std::int64_t n) {
    std::vector<std::int32_t> level(n), bb(n), be(n), cb(n), cc(n), par(n);
    std::vector<std::uint64_t> key(n);
    std::vector<double> center(3 * n), radius(n);
    check(fmm_get_cells(ctx(), level.data(), key.data(), center.data(), radius.data(), bb.data(), be.data(),
                        cb.data(), cc.data(), par.data()),
          ctx());
    cells.resize(n);
    for (std::int64_t i = 0; i < n; ++i)
      cells[i] = Cell{level[i], key[i], {center[3 * i], center[3 * i + 1], center[3 * i + 2]}, radius[i],
                      bb[i], be[i], cb[i], cc[i], par[i]};
  }
  struct Del {
    void operator()(fmm_ctx* c) const { fmm_destroy(c); }
  };
  std::unique_ptr<fmm_ctx, Del> ctx_;
};

inline Tree build_tree(std::vector<Body> bodies, int n_crit, int p, fmm_precision prec = FMM_PREC_FP64,
                       Real theta = 0.5) {  // tree.hpp:73
  if (n_crit < 1) throw std::invalid_argument("n_crit must be >= 1");
  if (p < 1) throw std::invalid_argument("expansion order must be >= 1");
  return Tree(std::move(bodies), n_crit, p, prec, theta);
}

class KernelTables {  // kernels.hpp:24-54 (term tables are compile-time on the device)
 public:
  explicit KernelTables(int order) : order_(order) {
    if (order < 1) throw std::invalid_argument("expansion order must be >= 1");
  }
  int order() const { return order_; }

 private:
  int order_;
};

// KernelVisitor (traversal.hpp:138-164): when passed to dual_tree_traverse the whole emitted
// lists run through the GPU M2L and P2P kernels.
class KernelVisitor {
 public:
  KernelVisitor(Tree& targets, Tree& sources, const KernelTables&, bool mutual)
      : tree_(&targets), mutual_(mutual) {
    if (&targets != &sources) throw std::invalid_argument("distinct target/source trees are not supported");
  }
  Tree* tree() const { return tree_; }
  // mutual (m2l_mutual / mutual p2p, kernels.cpp:113-126, :153-180): the GPU executes the
  // symmetrised lists with target-owned writes, accumulating the same sums
  bool mutual() const { return mutual_; }

 private:
  Tree* tree_;
  bool mutual_;
};

inline void upward_pass(Tree& tree, const KernelTables&) { check(fmm_upward(tree.ctx()), tree.ctx()); }

inline void downward_pass(Tree& tree, const KernelTables&) {  // traversal.cpp:52-63
  check(fmm_downward(tree.ctx()), tree.ctx());
  tree.fetch_results();
}

namespace detail {
inline void traverse_lists(const Tree& t, bool mutual, std::vector<std::int64_t>& mo,
                           std::vector<std::int32_t>& ms, std::vector<std::int64_t>& po,
                           std::vector<std::int32_t>& ps) {
  check(fmm_set_mutual(t.ctx(), mutual ? 1 : 0), t.ctx());
  check(fmm_traverse(t.ctx()), t.ctx());
  fmm_tree_info info{};
  check(fmm_get_tree_info(t.ctx(), &info), t.ctx());
  mo.resize(info.ncells + 1);
  po.resize(info.ncells + 1);
  ms.resize(info.n_m2l);
  ps.resize(info.n_p2p);
  check(fmm_get_lists(t.ctx(), mo.data(), ms.data(), po.data(), ps.data()), t.ctx());
}
}  // namespace detail

// dual_tree_traverse (traversal.hpp:118-133): the multiset of emitted pairs is produced on the
// GPU; any Visitor receives m2l_pair / p2p_pair for each of them (grouped by target).
template <class Visitor, class DrainSink>
void dual_tree_traverse(const Tree& targets, const Tree& sources, const TraversalConfig& cfg, Visitor& visit,
                        DrainSink&&) {
  if (&targets != &sources) throw std::invalid_argument("distinct target/source trees are not supported");
  if (!(cfg.theta > 0.0 && cfg.theta < 1.0)) throw std::invalid_argument("theta must be in (0,1)");
  std::vector<std::int64_t> mo, po;
  std::vector<std::int32_t> ms, ps;
  detail::traverse_lists(targets, cfg.mutual, mo, ms, po, ps);
  for (std::size_t t = 0; t + 1 < mo.size(); ++t)
    for (std::int64_t k = mo[t]; k < mo[t + 1]; ++k) visit.m2l_pair(static_cast<std::int32_t>(t), ms[k]);
  for (std::size_t t = 0; t + 1 < po.size(); ++t)
    for (std::int64_t k = po[t]; k < po[t + 1]; ++k) visit.p2p_pair(static_cast<std::int32_t>(t), ps[k]);
}

template <class DrainSink>
void dual_tree_traverse(Tree& targets, Tree&, const TraversalConfig& cfg, KernelVisitor& visit, DrainSink&&) {
  if (!(cfg.theta > 0.0 && cfg.theta < 1.0)) throw std::invalid_argument("theta must be in (0,1)");
  if (visit.mutual() != cfg.mutual) throw std::invalid_argument("KernelVisitor and TraversalConfig disagree on mutual");
  fmm_ctx* c = visit.tree()->ctx();
  check(fmm_set_mutual(c, cfg.mutual ? 1 : 0), c);
  check(fmm_traverse(c), c);
  check(fmm_m2l(c), c);
  check(fmm_p2p(c), c);
  (void)targets;
}

inline std::vector<Real> potentials(const Tree& tree) {  // tree.cpp:121-126
  std::vector<Real> out;
  out.reserve(tree.bodies.size());
  for (const Body& b : tree.bodies) out.push_back(b.potential);
  return out;
}

// Single operators (kernels.hpp:69-103) on the device; accumulate like the reference.
inline void m2l(const KernelTables& kt, const std::vector<Real>& source_m, const Vec3& displacement,
                std::vector<Real>& target_l) {
  check(fmm_op_m2l(kt.order(), 1, source_m.data(), displacement.data(), target_l.data()));
}
// m2l_mutual (kernels.cpp:113-126): both one-directional translations (the reference's w_rev
// terms are the translation of target_m by -R)
inline void m2l_mutual(const KernelTables& kt, const std::vector<Real>& source_m, const std::vector<Real>& target_m,
                       const Vec3& displacement, std::vector<Real>& target_l, std::vector<Real>& source_l) {
  const Vec3 neg{-displacement[0], -displacement[1], -displacement[2]};
  check(fmm_op_m2l(kt.order(), 1, source_m.data(), displacement.data(), target_l.data()));
  check(fmm_op_m2l(kt.order(), 1, target_m.data(), neg.data(), source_l.data()));
}
inline Real evaluate_multipole(const KernelTables& kt, const std::vector<Real>& M, const Vec3& x,
                               const Vec3& center) {
  Real out = 0.0;
  check(fmm_op_evaluate_multipole(kt.order(), 1, M.data(), x.data(), center.data(), &out));
  return out;
}

}  // namespace fmm::b200
