// ref_harness.cpp — C entry points over the UNMODIFIED reference sources. TEST/BASELINE
// INFRASTRUCTURE ONLY: built by oracle/Makefile into oracle/_ref/libfmmref.so (git-ignored)
// from /root/reference/proj/src/*.cpp compiled against oracle/eigen_shim. Used by tests/ to
// pin the C restatement (oracle/fmm_oracle.c), by tests/golden/make_golden.py to produce the
// committed fixtures, and by bench.py's reference arm / cpu_baseline (the reference's own
// scheduler-driven CPU FMM on the host cores).
//
// engine.cpp is #included (not linked) so that its anonymous-namespace ship_super_tasks
// (engine.cpp:27-57) is reachable without editing the reference.
#include "src/engine.cpp"  // resolved with -I $(REF) (= /root/reference/proj)

#include <chrono>
#include <cstring>
#include <exception>
#include <memory>
#include <string>

using namespace fmm;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

struct RefTree {
  Tree tree;
};

std::vector<Body> bodies_from(const double* xyzq, std::int64_t n, bool tag_index) {
  std::vector<Body> bodies(static_cast<std::size_t>(n));
  for (std::int64_t i = 0; i < n; ++i) {
    bodies[i].position = Vec3(xyzq[4 * i], xyzq[4 * i + 1], xyzq[4 * i + 2]);
    bodies[i].charge = xyzq[4 * i + 3];
    // build_tree never touches `potential`; use it to carry the input index through the
    // reorder so the body permutation can be read back, then clear it.
    bodies[i].potential = tag_index ? static_cast<double>(i) : 0.0;
  }
  return bodies;
}

struct Collector {
  std::vector<std::int32_t> m2l, p2p;
  void m2l_pair(std::int32_t t, std::int32_t s) {
    m2l.push_back(t);
    m2l.push_back(s);
  }
  void p2p_pair(std::int32_t t, std::int32_t s) {
    p2p.push_back(t);
    p2p.push_back(s);
  }
};

double secs(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// build_tree (tree.cpp:52-119). Returns an opaque tree or nullptr (see ref_last_error).
void* ref_build(const double* xyzq, std::int64_t n, int n_crit, int p, std::int64_t* perm) {
  RefTree* out = nullptr;
  const int rc = guarded([&] {
    auto t = std::make_unique<RefTree>();
    t->tree = build_tree(bodies_from(xyzq, n, true), n_crit, p);
    for (std::size_t i = 0; i < t->tree.bodies.size(); ++i) {
      if (perm) perm[i] = static_cast<std::int64_t>(t->tree.bodies[i].potential);
      t->tree.bodies[i].potential = 0.0;
    }
    out = t.release();
  });
  return rc ? nullptr : out;
}

void ref_free(void* h) { delete static_cast<RefTree*>(h); }
void ref_free_buf(void* p) { std::free(p); }

std::int64_t ref_ncells(void* h) { return static_cast<std::int64_t>(static_cast<RefTree*>(h)->tree.cells.size()); }

void ref_domain(void* h, double* center, double* half_side) {
  const Tree& t = static_cast<RefTree*>(h)->tree;
  for (int d = 0; d < 3; ++d) center[d] = t.domain.center[d];
  *half_side = t.domain.half_side;
}

void ref_cells(void* h, std::int32_t* level, std::uint64_t* key, double* center, double* radius,
               std::int32_t* body_begin, std::int32_t* body_end, std::int32_t* child_begin,
               std::int32_t* child_count, std::int32_t* parent) {
  const Tree& t = static_cast<RefTree*>(h)->tree;
  for (std::size_t i = 0; i < t.cells.size(); ++i) {
    const Cell& c = t.cells[i];
    level[i] = c.level;
    key[i] = c.morton_key;
    for (int d = 0; d < 3; ++d) center[3 * i + d] = c.center[d];
    radius[i] = c.radius;
    body_begin[i] = c.body_begin;
    body_end[i] = c.body_end;
    child_begin[i] = c.child_begin;
    child_count[i] = c.child_count;
    parent[i] = c.parent;
  }
}

// dual_tree_traverse with a collecting Visitor (acceptance.cpp:93-123). Drained pairs are
// completed inline with traverse_pair (test_traversal.cpp:50-56).
int ref_traverse(void* h, double theta, int mutual, std::int64_t queue_threshold, std::int64_t* n_m2l,
                 std::int32_t** m2l, std::int64_t* n_p2p, std::int32_t** p2p) {
  return guarded([&] {
    const Tree& t = static_cast<RefTree*>(h)->tree;
    TraversalConfig cfg;
    cfg.theta = theta;
    cfg.queue_threshold = static_cast<std::size_t>(queue_threshold);
    cfg.mutual = mutual != 0;
    Collector vis;
    dual_tree_traverse(t, t, cfg, vis, [&](std::span<const TraversalPair> pairs) {
      for (const TraversalPair& pr : pairs) traverse_pair(t, t, pr, cfg, vis);
    });
    *n_m2l = static_cast<std::int64_t>(vis.m2l.size() / 2);
    *n_p2p = static_cast<std::int64_t>(vis.p2p.size() / 2);
    *m2l = static_cast<std::int32_t*>(std::malloc(sizeof(std::int32_t) * (vis.m2l.size() + 2)));
    *p2p = static_cast<std::int32_t*>(std::malloc(sizeof(std::int32_t) * (vis.p2p.size() + 2)));
    std::memcpy(*m2l, vis.m2l.data(), sizeof(std::int32_t) * vis.m2l.size());
    std::memcpy(*p2p, vis.p2p.data(), sizeof(std::int32_t) * vis.p2p.size());
  });
}

// run_once's stage sequence (engine.cpp:61-125) on the given tree: upward_pass, then the
// traversal with KernelVisitor, then downward_pass. threads == 0: serial inline traversal
// (test_traversal.cpp:292-318); threads >= 1: the reference scheduler with `threads`
// workers (+ the helping master) and ship_super_tasks, exactly as run_once.
// times[0..2] = upward, traversal (+ scheduler), downward seconds.
int ref_pipeline(void* h, double theta, int mutual, std::int64_t queue_threshold, int threads,
                 double* times) {
  return guarded([&] {
    Tree& tree = static_cast<RefTree*>(h)->tree;
    const KernelTables tables(tree.order);
    auto t0 = std::chrono::steady_clock::now();
    upward_pass(tree, tables);
    if (times) times[0] = secs(t0);
    TraversalConfig tc;
    tc.theta = theta;
    tc.queue_threshold = static_cast<std::size_t>(queue_threshold);
    tc.mutual = mutual != 0;
    KernelVisitor visitor(tree, tree, tables, tc.mutual);
    t0 = std::chrono::steady_clock::now();
    if (threads <= 0) {
      dual_tree_traverse(tree, tree, tc, visitor, [&](std::span<const TraversalPair> pairs) {
        for (const TraversalPair& pr : pairs) traverse_pair(tree, tree, pr, tc, visitor);
      });
    } else {
      SchedulerConfig sc;
      sc.num_workers = threads;
      Scheduler sched(sc);
      dual_tree_traverse(tree, tree, tc, visitor, [&](std::span<const TraversalPair> pairs) {
        ship_super_tasks(sched, tree, tc, visitor, pairs);
      });
      sched.wait_all();
    }
    if (times) times[1] = secs(t0);
    t0 = std::chrono::steady_clock::now();
    downward_pass(tree, tables);
    if (times) times[2] = secs(t0);
  });
}

// Whole reference step from input bodies: build_tree + ref_pipeline. times[0..3] =
// build, upward, traversal, downward. phi (tree order) may be null.
int ref_step(const double* xyzq, std::int64_t n, int n_crit, int p, double theta,
             std::int64_t queue_threshold, int threads, double* times, double* phi) {
  return guarded([&] {
    auto t0 = std::chrono::steady_clock::now();
    Tree tree = build_tree(bodies_from(xyzq, n, false), n_crit, p);
    if (times) times[0] = secs(t0);
    RefTree holder{std::move(tree)};
    double t3[3];
    if (ref_pipeline(&holder, theta, 0, queue_threshold, threads, t3)) throw std::runtime_error(g_err);
    if (times) {
      times[1] = t3[0];
      times[2] = t3[1];
      times[3] = t3[2];
    }
    if (phi)
      for (std::size_t i = 0; i < holder.tree.bodies.size(); ++i) phi[i] = holder.tree.bodies[i].potential;
  });
}

void ref_potentials(void* h, double* phi) {
  const Tree& t = static_cast<RefTree*>(h)->tree;
  for (std::size_t i = 0; i < t.bodies.size(); ++i) phi[i] = t.bodies[i].potential;
}

void ref_expansions(void* h, double* multipole, double* local) {
  const Tree& t = static_cast<RefTree*>(h)->tree;
  const std::size_t nc = static_cast<std::size_t>(n_coef(t.order));
  for (std::size_t i = 0; i < t.cells.size(); ++i)
    for (std::size_t k = 0; k < nc; ++k) {
      if (multipole) multipole[i * nc + k] = t.cells[i].multipole[k];
      if (local) local[i * nc + k] = t.cells[i].local[k];
    }
}

void ref_counters(std::uint64_t* p2p_calls, std::uint64_t* p2p_evals, std::uint64_t* m2l_calls) {
  *p2p_calls = kernel_counters().p2p_calls.load();
  *p2p_evals = kernel_counters().p2p_evals.load();
  *m2l_calls = kernel_counters().m2l_calls.load();
}
void ref_counters_reset() { kernel_counters().reset(); }

// direct_sum (oracle.cpp:8-23) over bodies in the given order.
void ref_direct_sum(const double* xyzq, std::int64_t n, double* phi) {
  const auto bodies = bodies_from(xyzq, n, false);
  const auto out = direct_sum(bodies);
  for (std::int64_t i = 0; i < n; ++i) phi[i] = out[i];
}

// generate_bodies (dataset.cpp:74-112); dist 0 cube, 1 sphere-surface, 2 cluster.
int ref_generate_bodies(int dist, std::int64_t n, std::uint64_t seed, double* xyzq) {
  return guarded([&] {
    const BodyDistribution d = dist == 0 ? BodyDistribution::cube
                               : dist == 1 ? BodyDistribution::sphere_surface
                                           : BodyDistribution::cluster;
    const auto bodies = generate_bodies(d, n, seed);
    for (std::int64_t i = 0; i < n; ++i) {
      for (int k = 0; k < 3; ++k) xyzq[4 * i + k] = bodies[i].position[k];
      xyzq[4 * i + 3] = bodies[i].charge;
    }
  });
}

// run_once (engine.cpp:61-125) for the acceptance-style golden aggregates.
int ref_run_once(std::int64_t n, int p, double theta, int n_crit, int threads, int mutual, int dist,
                 std::uint64_t seed, std::int64_t queue_threshold, double* rel_l2, double* times) {
  return guarded([&] {
    RunConfig cfg;
    cfg.n_bodies = n;
    cfg.order = p;
    cfg.theta = theta;
    cfg.n_crit = n_crit;
    cfg.threads = threads;
    cfg.mutual = mutual != 0;
    cfg.distribution = dist == 0 ? BodyDistribution::cube
                       : dist == 1 ? BodyDistribution::sphere_surface
                                   : BodyDistribution::cluster;
    cfg.seed = seed;
    cfg.queue_threshold = static_cast<std::size_t>(queue_threshold);
    cfg.check = rel_l2 != nullptr;
    const RunResult r = run_once(cfg);
    if (rel_l2) *rel_l2 = r.error->rel_l2;
    if (times) {
      times[0] = r.t_build;
      times[1] = r.t_upward;
      times[2] = r.t_traversal;
      times[3] = r.t_downward;
    }
  });
}

// Single-operator entry points (kernels.cpp) for operator-level parity.
int ref_op_m2l(int order, const double* M, const double* R, double* L) {
  return guarded([&] {
    const KernelTables kt(order);
    CoeffVec m(kt.coef_count()), l = CoeffVec::Zero(kt.coef_count());
    for (int i = 0; i < kt.coef_count(); ++i) m[i] = M[i];
    m2l(kt, m, Vec3(R[0], R[1], R[2]), l);
    for (int i = 0; i < kt.coef_count(); ++i) L[i] += l[i];
  });
}

int ref_op_laplace_derivatives(int max_degree, const double* R, double* out) {
  return guarded([&] {
    const MultiIndexSet idx(max_degree);
    idx.laplace_derivatives(Vec3(R[0], R[1], R[2]), std::span<Real>(out, idx.size()));
  });
}

int ref_op_p2m(int order, std::int64_t n, const double* xyzq, const double* center, double* M) {
  return guarded([&] {
    const KernelTables kt(order);
    CoeffVec m = CoeffVec::Zero(kt.coef_count());
    const auto bodies = bodies_from(xyzq, n, false);
    p2m(kt, bodies, Vec3(center[0], center[1], center[2]), m);
    for (int i = 0; i < kt.coef_count(); ++i) M[i] += m[i];
  });
}

int ref_op_m2m(int order, const double* child, const double* shift, double* parent) {
  return guarded([&] {
    const KernelTables kt(order);
    CoeffVec c(kt.coef_count()), pm = CoeffVec::Zero(kt.coef_count());
    for (int i = 0; i < kt.coef_count(); ++i) c[i] = child[i];
    m2m(kt, c, Vec3(shift[0], shift[1], shift[2]), pm);
    for (int i = 0; i < kt.coef_count(); ++i) parent[i] += pm[i];
  });
}

int ref_op_l2l(int order, const double* parent, const double* shift, double* child) {
  return guarded([&] {
    const KernelTables kt(order);
    CoeffVec pl(kt.coef_count()), cl = CoeffVec::Zero(kt.coef_count());
    for (int i = 0; i < kt.coef_count(); ++i) pl[i] = parent[i];
    l2l(kt, pl, Vec3(shift[0], shift[1], shift[2]), cl);
    for (int i = 0; i < kt.coef_count(); ++i) child[i] += cl[i];
  });
}

int ref_op_l2p(int order, const double* L, const double* center, std::int64_t n, const double* xyzq,
               double* phi) {
  return guarded([&] {
    const KernelTables kt(order);
    CoeffVec l(kt.coef_count());
    for (int i = 0; i < kt.coef_count(); ++i) l[i] = L[i];
    auto bodies = bodies_from(xyzq, n, false);
    l2p(kt, l, Vec3(center[0], center[1], center[2]), bodies);
    for (std::int64_t i = 0; i < n; ++i) phi[i] += bodies[i].potential;
  });
}

int ref_op_p2p(std::int64_t nt, const double* txyzq, std::int64_t ns, const double* sxyzq, double* phi) {
  return guarded([&] {
    auto t = bodies_from(txyzq, nt, false);
    auto s = bodies_from(sxyzq, ns, false);
    p2p(t, s, false);
    for (std::int64_t i = 0; i < nt; ++i) phi[i] += t[i].potential;
  });
}

int ref_op_evaluate_multipole(int order, const double* M, const double* x, const double* center, double* out) {
  return guarded([&] {
    const KernelTables kt(order);
    CoeffVec m(kt.coef_count());
    for (int i = 0; i < kt.coef_count(); ++i) m[i] = M[i];
    *out = evaluate_multipole(kt, m, Vec3(x[0], x[1], x[2]), Vec3(center[0], center[1], center[2]));
  });
}

}  // extern "C"
