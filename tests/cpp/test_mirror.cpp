// C++ parity test through include/fmm_b200.hpp, written like the reference's own
// proj/tests/test_traversal.cpp:292-318 (serial pipeline) and test_kernels.cpp known answers.
// Built and run by tests/test_cpp_mirror.py. Exit code = number of failures.
#include <cmath>
#include <cstdio>
#include <random>
#include <set>
#include <stdexcept>
#include <tuple>
#include <vector>

#include "fmm_b200.hpp"

using namespace fmm::b200;

static int g_fail = 0;
#define CHECK(c)                                                      \
  do {                                                                \
    if (!(c)) {                                                       \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);        \
      ++g_fail;                                                       \
    }                                                                 \
  } while (0)

struct Collector {  // acceptance.cpp:93-97
  std::set<std::tuple<char, int, int>> tuples;
  void m2l_pair(std::int32_t t, std::int32_t s) { tuples.emplace('M', t, s); }
  void p2p_pair(std::int32_t t, std::int32_t s) { tuples.emplace('P', t, s); }
};

int main() {
  // known answers (test_kernels.cpp:108-115, :325-335)
  {
    KernelTables kt(3);
    std::vector<Real> M(10, 0.0), L(10, 0.0);
    M[0] = 5.0;
    m2l(kt, M, Vec3{2.0, 0.0, 0.0}, L);
    CHECK(std::abs(L[0] - 2.5) < 1e-14);
    bool threw = false;
    try {
      m2l(kt, M, Vec3{0, 0, 0}, L);
    } catch (const std::invalid_argument& e) {
      threw = std::string(e.what()) == "singular M2L displacement";
    }
    CHECK(threw);
    KernelTables k6(6);
    std::vector<Real> M6(56, 0.0);
    M6[0] = 2.0;
    CHECK(std::abs(evaluate_multipole(k6, M6, Vec3{1, 5, 1}, Vec3{1, 1, 1}) - 0.5) < 1e-14);
  }
  // serial pipeline, N = 2048 cube (test_traversal.cpp:292-318) against the direct sum
  std::mt19937_64 rng(15);
  std::uniform_real_distribution<double> u(0.0, 1.0), qd(-1.0, 1.0);
  std::vector<Body> bodies(2048);
  for (Body& b : bodies) {
    b.position = {u(rng), u(rng), u(rng)};
    b.charge = qd(rng);
  }
  Tree t = build_tree(bodies, 64, 6);
  KernelTables kt(6);
  upward_pass(t, kt);
  TraversalConfig cfg;
  cfg.theta = 0.5;
  cfg.queue_threshold = 1u << 30;
  Collector col;
  dual_tree_traverse(t, t, cfg, col, [](auto) {});
  CHECK(!col.tuples.empty());
  // every ordered leaf pair covered exactly once (test_traversal.cpp:213-250), small check
  KernelVisitor vis(t, t, kt, false);
  dual_tree_traverse(t, t, cfg, vis, [](auto) {});
  downward_pass(t, kt);
  const auto phi = potentials(t);
  long double num = 0, den = 0;
  for (std::size_t i = 0; i < t.bodies.size(); ++i) {
    long double s = 0;
    for (std::size_t j = 0; j < t.bodies.size(); ++j) {
      if (i == j) continue;
      const double dx = t.bodies[i].position[0] - t.bodies[j].position[0];
      const double dy = t.bodies[i].position[1] - t.bodies[j].position[1];
      const double dz = t.bodies[i].position[2] - t.bodies[j].position[2];
      const double r2 = (dx * dx + dy * dy) + dz * dz;
      if (r2 == 0.0) continue;
      s += t.bodies[j].charge / std::sqrt(static_cast<long double>(r2));
    }
    num += (phi[i] - s) * (phi[i] - s);
    den += s * s;
  }
  const double rel = std::sqrt(static_cast<double>(num / den));
  std::printf("serial pipeline rel_l2 vs direct sum: %.3e\n", rel);
  CHECK(rel <= 1e-2);
  // mutual mode (test_traversal.cpp:182-210, :320-345): the mutual emission symmetrised equals
  // the non-mutual one, and the mutual KernelVisitor pipeline matches the non-mutual potentials
  {
    TraversalConfig mcfg = cfg;
    mcfg.mutual = true;
    Collector mcol;
    dual_tree_traverse(t, t, mcfg, mcol, [](auto) {});
    std::set<std::tuple<char, int, int>> sym;
    for (const auto& [k, a, b] : mcol.tuples) {
      sym.emplace(k, a, b);
      sym.emplace(k, b, a);
    }
    CHECK(sym == col.tuples);
    CHECK(mcol.tuples.size() < col.tuples.size());
    Tree tm = build_tree(bodies, 64, 6);
    upward_pass(tm, kt);
    KernelVisitor mvis(tm, tm, kt, true);
    dual_tree_traverse(tm, tm, mcfg, mvis, [](auto) {});
    downward_pass(tm, kt);
    const auto phim = potentials(tm);
    long double dn = 0, dd = 0;
    for (std::size_t i = 0; i < phi.size(); ++i) {
      dn += (phim[i] - phi[i]) * (phim[i] - phi[i]);
      dd += phi[i] * phi[i];
    }
    CHECK(std::sqrt(static_cast<double>(dn / dd)) < 1e-12);
    // m2l_mutual = the two one-directional translations (test_kernels.cpp:187-200)
    std::vector<Real> Ms(56), Mt(56), tl(56, 0.0), sl(56, 0.0), t1(56, 0.0), s1(56, 0.0);
    for (int i = 0; i < 56; ++i) {
      Ms[i] = qd(rng);
      Mt[i] = qd(rng);
    }
    const Vec3 R{2.2, -1.7, 0.9}, nR{-2.2, 1.7, -0.9};
    m2l_mutual(kt, Ms, Mt, R, tl, sl);
    m2l(kt, Ms, R, t1);
    m2l(kt, Mt, nR, s1);
    double diff = 0;
    for (int i = 0; i < 56; ++i) diff = std::max(diff, std::abs(tl[i] - t1[i]) + std::abs(sl[i] - s1[i]));
    CHECK(diff == 0.0);
  }
  // error behaviour mirrors the reference
  bool threw = false;
  try {
    build_tree({}, 8, 3);
  } catch (const std::invalid_argument& e) {
    threw = std::string(e.what()) == "empty input";
  }
  CHECK(threw);
  std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "ok", g_fail);
  return g_fail;
}
