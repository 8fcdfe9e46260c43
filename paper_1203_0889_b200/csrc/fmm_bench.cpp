// fmm_bench — the reference's command-line driver (proj/tools/fmm_bench.cpp:77-149) over the
// B200 path: single runs with the direct-sum accuracy check, (p, N, Q, T) sweeps, and the
// reference's run CSV (engine.cpp:127-166), trace CSV (scheduler.cpp:305-317) and DOT
// (scheduler.cpp:287-303) outputs. Same flags, defaults, printout and exit codes
// (0 ok, 1 runtime error, 2 --check above --check-tol; argument errors use CLI11's codes:
// 104 conversion, 105 validation, 109 unknown argument).
//
// What maps differently on the GPU (README of this file, also in DESIGN.md):
//   --threads T   recorded in the CSV; the GPU step does not use host worker threads, so a
//                 sweep over t reports speedup ~1 (the reference's T = scheduler workers).
//   --q Q         recorded (effective_queue_threshold); Q only moves the reference's drain
//                 point and the GPU traversal emits the same multiset for every Q.
//   tasks         the CSV "tasks" column counts kernel launches of the step.
//   --trace/--dag one row / node per GPU stage (build, traversal, upward, m2l, p2p, downward).
//   --check       the O(N^2) direct sum runs on the GPU in FP64 (reference: long double on
//                 the CPU, oracle.cpp:8-23); compare() follows oracle.cpp:25-49.
// GPU-only flags: --precision fp64|fp32 (default fp64, the reference's arithmetic),
// --device, --warmup W (untimed steps before the timed one, default 1), --overlap.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "fmm_b200.h"

namespace {

struct ArgError {
  int code;
  std::string msg;
};

struct RunConfig {  // engine.hpp:16-36
  int64_t n_bodies = 10000;
  int order = 6;
  int64_t queue_threshold = 0;  // 0 -> max(n_bodies/100, 64)
  int threads = 1;
  double theta = 0.5;
  int n_crit = 64;
  bool mutual = false;
  std::string dist = "cube";
  uint64_t seed = 1;
  bool check = false;
  double check_tol = 1e-2;
  std::string trace_path, dag_path, csv_path;
  // GPU
  int precision = FMM_PREC_FP64;
  int device = 0;
  int warmup = 1;
  bool overlap = false;

  int64_t effective_queue_threshold() const {
    if (queue_threshold > 0) return queue_threshold;
    return std::max<int64_t>(n_bodies / 100, 64);
  }
};

struct ErrorReport {  // oracle.hpp
  double rel_l2 = 0, rel_linf = 0;
  int64_t n = 0;
  bool absolute = false;
};

struct RunResult {  // engine.hpp:38-49
  double t_build = 0, t_upward = 0, t_traversal = 0, t_downward = 0;
  double t_device = 0;  // the step's device time (< the phase sum when stages overlap)
  int64_t task_count = 0;
  bool has_error = false;
  ErrorReport error;
  double speedup = 0, efficiency = 0;
  double t_total() const { return t_build + t_upward + t_traversal + t_downward; }
};

void check(int rc, const fmm_ctx* c) {
  if (rc != FMM_OK) throw std::runtime_error(fmm_last_error(c));
}

int dist_config(const std::string& d) {  // dataset.cpp:36-41 names + the BASELINE configs
  if (d == "cube") return 10;
  if (d == "sphere-surface") return 11;
  if (d == "cluster") return 12;
  for (int k = 1; k <= 5; ++k)
    if (d == "baseline-c" + std::to_string(k)) return k;
  throw std::invalid_argument("unknown distribution name: " + d);
}

// oracle.cpp:25-49
ErrorReport compare(const std::vector<double>& a, const std::vector<double>& b) {
  ErrorReport rep;
  rep.n = static_cast<int64_t>(a.size());
  long double diff2 = 0.0L, ref2 = 0.0L;
  double diff_inf = 0.0, ref_inf = 0.0;
  for (size_t i = 0; i < a.size(); ++i) {
    const double d = a[i] - b[i];
    diff2 += static_cast<long double>(d) * d;
    ref2 += static_cast<long double>(b[i]) * b[i];
    diff_inf = std::max(diff_inf, std::abs(d));
    ref_inf = std::max(ref_inf, std::abs(b[i]));
  }
  if (ref2 == 0.0L) {
    rep.absolute = true;
    rep.rel_l2 = static_cast<double>(std::sqrt(diff2));
    rep.rel_linf = diff_inf;
  } else {
    rep.rel_l2 = static_cast<double>(std::sqrt(diff2 / ref2));
    rep.rel_linf = diff_inf / ref_inf;
  }
  return rep;
}

std::string run_csv_header() {  // engine.cpp:127-130
  return "n,p,q,threads,theta,ncrit,mutual,dist,seed,"
         "t_build,t_upward,t_traversal,t_downward,t_total,tasks,rel_l2,rel_linf";
}

void append_config(std::ostringstream& out, const RunConfig& cfg) {
  out << cfg.n_bodies << ',' << cfg.order << ',' << cfg.effective_queue_threshold() << ',' << cfg.threads << ','
      << cfg.theta << ',' << cfg.n_crit << ',' << (cfg.mutual ? 1 : 0) << ',' << cfg.dist << ',' << cfg.seed;
}

std::string run_csv_row(const RunConfig& cfg, const RunResult& res) {  // engine.cpp:142-156
  std::ostringstream out;
  out.precision(9);
  append_config(out, cfg);
  out << ',' << res.t_build << ',' << res.t_upward << ',' << res.t_traversal << ',' << res.t_downward << ','
      << res.t_total() << ',' << res.task_count << ',';
  if (res.has_error)
    out << res.error.rel_l2 << ',' << res.error.rel_linf;
  else
    out << ',';
  return out.str();
}

std::string sweep_csv_header() { return "n,p,q,threads,theta,ncrit,mutual,dist,seed,time_total,speedup_vs_T1,efficiency"; }

std::string sweep_csv_row(const RunConfig& cfg, const RunResult& res) {
  std::ostringstream out;
  out.precision(9);
  append_config(out, cfg);
  out << ',' << res.t_total() << ',' << res.speedup << ',' << res.efficiency;
  return out.str();
}

// FP64 direct sum on the GPU, tree order: targets in blocks of 64 against every body
std::vector<double> direct_sum_gpu(const std::vector<double>& xyzq_tree) {
  const int64_t n = static_cast<int64_t>(xyzq_tree.size() / 4);
  std::vector<int32_t> ranges;
  for (int64_t b = 0; b < n; b += 64) {
    ranges.push_back(static_cast<int32_t>(b));
    ranges.push_back(static_cast<int32_t>(std::min<int64_t>(b + 64, n)));
    ranges.push_back(0);
    ranges.push_back(static_cast<int32_t>(n));
  }
  std::vector<double> phi(n, 0.0);
  check(fmm_op_p2p(static_cast<int64_t>(ranges.size() / 4), ranges.data(), xyzq_tree.data(), FMM_PREC_FP64,
                   phi.data(), nullptr),
        nullptr);
  return phi;
}

void write_trace(fmm_ctx* c, const std::string& path) {
  fmm_trace_row rows[16];
  int n = 0;
  check(fmm_get_stage_trace(c, rows, 16, &n), c);
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot open " + path);
  out << "task_id,worker_id,kind,start_ns,end_ns\n";
  for (int i = 0; i < n && i < 16; ++i)
    out << rows[i].task_id << ',' << rows[i].worker_id << ',' << rows[i].kind << ',' << rows[i].start_ns << ','
        << rows[i].end_ns << '\n';
  if (!out.good()) throw std::runtime_error("write failed: " + path);
}

void write_dag(fmm_ctx* c, const std::string& path) {  // scheduler.cpp:287-303 format
  fmm_trace_row rows[16];
  int n = 0;
  check(fmm_get_stage_trace(c, rows, 16, &n), c);
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot open " + path);
  out << "digraph tasks {\n";
  for (int i = 0; i < n && i < 16; ++i) out << "  t" << i << " [label=\"" << rows[i].kind << " #" << i << "\"];\n";
  // data dependencies of the stages (ids as in fmm_get_stage_trace)
  const int edges[][2] = {{0, 1}, {0, 2}, {1, 3}, {2, 3}, {1, 4}, {3, 5}, {4, 5}};
  for (const auto& e : edges) out << "  t" << e[0] << " -> t" << e[1] << ";\n";
  out << "}\n";
  if (!out.good()) throw std::runtime_error("write failed: " + path);
}

// engine.cpp:61-125 on the GPU
RunResult run_once(const RunConfig& cfg) {
  if (!(cfg.theta > 0.0 && cfg.theta < 1.0)) throw std::invalid_argument("theta must be in (0,1)");
  if (cfg.n_bodies < 1) throw std::invalid_argument("body count must be >= 1");
  RunResult res;
  std::vector<double> xyzq(4 * cfg.n_bodies);
  check(fmm_generate_bodies(dist_config(cfg.dist), cfg.n_bodies, cfg.seed, xyzq.data()), nullptr);

  fmm_config fc{cfg.order, cfg.n_crit, cfg.theta, cfg.mutual ? 1 : 0, cfg.precision, cfg.device, 0};
  fmm_ctx* c = nullptr;
  check(fmm_create(&fc, &c), nullptr);
  struct Guard {
    fmm_ctx* c;
    ~Guard() { fmm_destroy(c); }
  } guard{c};
  check(fmm_set_overlap(c, cfg.overlap ? 1 : 0), c);
  check(fmm_set_bodies(c, xyzq.data(), cfg.n_bodies), c);
  for (int w = 0; w < cfg.warmup; ++w) check(fmm_evaluate(c), c);
  check(fmm_evaluate(c), c);
  fmm_stage_times t{};
  check(fmm_get_stage_times(c, &t), c);
  res.t_build = t.build_ms * 1e-3;
  res.t_upward = t.upward_ms * 1e-3;
  res.t_traversal = (t.traverse_ms + t.m2l_ms + t.p2p_ms) * 1e-3;  // traversal + interactions
  res.t_downward = t.downward_ms * 1e-3;
  res.t_device = t.total_ms * 1e-3;
  res.task_count = t.kernel_launches;

  if (!cfg.trace_path.empty()) write_trace(c, cfg.trace_path);
  if (!cfg.dag_path.empty()) write_dag(c, cfg.dag_path);

  if (cfg.check) {
    std::vector<double> phi(cfg.n_bodies);
    check(fmm_get_results(c, phi.data(), nullptr, 0), c);  // potentials(), tree order
    std::vector<int64_t> perm(cfg.n_bodies);
    check(fmm_get_permutation(c, perm.data()), c);
    std::vector<double> sorted(4 * cfg.n_bodies);
    for (int64_t i = 0; i < cfg.n_bodies; ++i)
      for (int k = 0; k < 4; ++k) sorted[4 * i + k] = xyzq[4 * perm[i] + k];
    res.error = compare(phi, direct_sum_gpu(sorted));
    res.has_error = true;
  }

  if (!cfg.csv_path.empty()) {
    std::ifstream probe(cfg.csv_path, std::ios::ate);
    const bool fresh = !probe.good() || probe.tellg() == 0;
    probe.close();
    std::ofstream out(cfg.csv_path, std::ios::app);
    if (!out) throw std::runtime_error("cannot open " + cfg.csv_path);
    if (fresh) out << run_csv_header() << '\n';
    out << run_csv_row(cfg, res) << '\n';
  }
  return res;
}

struct SweepRanges {
  std::vector<int64_t> n_bodies;
  std::vector<int> orders;
  std::vector<int64_t> queue_thresholds;
  std::vector<int> threads;
};

SweepRanges parse_sweep_spec(const std::string& spec) {  // fmm_bench.cpp:17-46
  SweepRanges ranges;
  std::stringstream dims(spec);
  std::string dim;
  while (std::getline(dims, dim, ';')) {
    if (dim.empty()) continue;
    const auto eq = dim.find('=');
    if (eq == std::string::npos) throw ArgError{105, "--sweep: expected key=v1,v2,..."};
    const std::string key = dim.substr(0, eq);
    std::stringstream vals(dim.substr(eq + 1));
    std::string val;
    while (std::getline(vals, val, ',')) {
      int64_t v;
      try {
        v = static_cast<int64_t>(std::stod(val));
      } catch (const std::exception&) {
        throw ArgError{104, "--sweep: cannot convert '" + val + "'"};
      }
      if (key == "n") ranges.n_bodies.push_back(v);
      else if (key == "p") ranges.orders.push_back(static_cast<int>(v));
      else if (key == "q") ranges.queue_thresholds.push_back(v);
      else if (key == "t") ranges.threads.push_back(static_cast<int>(v));
      else throw ArgError{105, "--sweep: unknown dimension '" + key + "'"};
    }
  }
  return ranges;
}

// engine.cpp:168-227
std::vector<std::pair<RunConfig, RunResult>> run_sweep(const RunConfig& base, const SweepRanges& r, std::ostream* csv) {
  auto ns = r.n_bodies.empty() ? std::vector<int64_t>{base.n_bodies} : r.n_bodies;
  auto ps = r.orders.empty() ? std::vector<int>{base.order} : r.orders;
  auto qs = r.queue_thresholds.empty() ? std::vector<int64_t>{base.effective_queue_threshold()} : r.queue_thresholds;
  auto ts = r.threads.empty() ? std::vector<int>{base.threads} : r.threads;
  if (csv) *csv << sweep_csv_header() << '\n';
  std::vector<std::pair<RunConfig, RunResult>> rows;
  std::map<std::tuple<int, int64_t, int64_t>, double> t1;
  for (int p : ps)
    for (int64_t n : ns)
      for (int64_t q : qs)
        for (int t : ts) {
          RunConfig cfg = base;
          cfg.order = p;
          cfg.n_bodies = n;
          cfg.queue_threshold = q;
          cfg.threads = t;
          cfg.trace_path.clear();
          cfg.dag_path.clear();
          cfg.csv_path.clear();
          RunResult res = run_once(cfg);
          const auto key = std::make_tuple(p, n, q);
          if (t == 1) t1[key] = res.t_total();
          if (!t1.count(key)) {
            RunConfig c1 = cfg;
            c1.threads = 1;
            t1[key] = run_once(c1).t_total();
          }
          res.speedup = res.t_total() > 0 ? t1[key] / res.t_total() : 0.0;
          res.efficiency = res.speedup / t;
          if (csv) *csv << sweep_csv_row(cfg, res) << '\n';
          rows.emplace_back(cfg, res);
        }
  return rows;
}

void print_result(const RunConfig& cfg, const RunResult& res) {  // fmm_bench.cpp:48-66
  std::printf("n=%lld p=%d q=%lld threads=%d theta=%.3g ncrit=%d %s dist=%s seed=%llu\n",
              static_cast<long long>(cfg.n_bodies), cfg.order, static_cast<long long>(cfg.effective_queue_threshold()),
              cfg.threads, cfg.theta, cfg.n_crit, cfg.mutual ? "mutual" : "non-mutual", cfg.dist.c_str(),
              static_cast<unsigned long long>(cfg.seed));
  std::printf("  build     %10.4f s\n", res.t_build);
  std::printf("  upward    %10.4f s\n", res.t_upward);
  std::printf("  traversal %10.4f s  (%lld tasks)\n", res.t_traversal, static_cast<long long>(res.task_count));
  std::printf("  downward  %10.4f s\n", res.t_downward);
  std::printf("  total     %10.4f s\n", res.t_total());
  std::printf("  device    %10.4f s  (B200 step, %s)\n", res.t_device,
              cfg.precision == FMM_PREC_FP64 ? "fp64" : "fp32 P2P");
  if (res.has_error)
    std::printf("  check     rel_l2=%.3e rel_linf=%.3e (n=%lld)%s\n", res.error.rel_l2, res.error.rel_linf,
                static_cast<long long>(res.error.n), res.error.absolute ? " [absolute]" : "");
}

void usage() {
  std::printf(
      "Laplace FMM on B200 (drop-in for the reference's fmm_bench)\n"
      "Usage: fmm_bench [OPTIONS]\n"
      "  --n INT            number of bodies (default 10000)\n"
      "  --p INT            expansion order (default 6)\n"
      "  --q INT            queue-size threshold (recorded; default max(n/100, 64))\n"
      "  --threads INT      worker threads (recorded; the GPU step uses none)\n"
      "  --theta FLOAT      opening parameter in (0,1) (default 0.5)\n"
      "  --ncrit INT        max bodies per leaf (default 64)\n"
      "  --mutual / --non-mutual   mutual cell interactions (default off)\n"
      "  --dist NAME        cube | sphere-surface | cluster | baseline-c1..baseline-c5\n"
      "  --seed INT         RNG seed (default 1)\n"
      "  --check            compare against the O(N^2) direct sum (GPU, FP64)\n"
      "  --check-tol FLOAT  max accepted rel_l2 for --check (default 1e-2)\n"
      "  --trace PATH       write the stage trace CSV here\n"
      "  --dag PATH         write the stage DAG (DOT) here\n"
      "  --csv PATH         append per-run CSV row here (sweep: full table)\n"
      "  --sweep SPEC       sweep spec, e.g. n=1e5,1e6;p=4,6;q=1000;t=1\n"
      "  --precision fp64|fp32   P2P arithmetic (default fp64)\n"
      "  --device INT       CUDA device (default 0)\n"
      "  --warmup INT       untimed steps before the timed one (default 1)\n"
      "  --overlap          run the upward pass concurrently with the traversal\n");
}

template <class T>
T conv(const std::string& opt, const std::string& v) {
  try {
    size_t pos = 0;
    const double d = std::stod(v, &pos);
    if (pos != v.size()) throw std::invalid_argument(v);
    if (std::is_integral<T>::value && d != std::floor(d)) throw std::invalid_argument(v);
    return static_cast<T>(d);
  } catch (const std::exception&) {
    throw ArgError{104, "Could not convert: " + opt + " = " + v};
  }
}

RunConfig parse(int argc, char** argv, std::string& sweep, bool& help) {
  RunConfig cfg;
  auto need = [&](int& i) -> std::string {
    if (i + 1 >= argc) throw ArgError{105, std::string(argv[i]) + ": 1 required argument missing"};
    return argv[++i];
  };
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    if (a == "-h" || a == "--help") help = true;
    else if (a == "--n") cfg.n_bodies = conv<int64_t>(a, need(i));
    else if (a == "--p") cfg.order = conv<int>(a, need(i));
    else if (a == "--q") cfg.queue_threshold = conv<int64_t>(a, need(i));
    else if (a == "--threads") cfg.threads = conv<int>(a, need(i));
    else if (a == "--theta") cfg.theta = conv<double>(a, need(i));
    else if (a == "--ncrit") cfg.n_crit = conv<int>(a, need(i));
    else if (a == "--mutual") cfg.mutual = true;
    else if (a == "--non-mutual") cfg.mutual = false;
    else if (a == "--dist") cfg.dist = need(i);
    else if (a == "--seed") cfg.seed = conv<uint64_t>(a, need(i));
    else if (a == "--check") cfg.check = true;
    else if (a == "--check-tol") cfg.check_tol = conv<double>(a, need(i));
    else if (a == "--trace") cfg.trace_path = need(i);
    else if (a == "--dag") cfg.dag_path = need(i);
    else if (a == "--csv") cfg.csv_path = need(i);
    else if (a == "--sweep") sweep = need(i);
    else if (a == "--precision") {
      const std::string v = need(i);
      if (v == "fp64") cfg.precision = FMM_PREC_FP64;
      else if (v == "fp32") cfg.precision = FMM_PREC_FP32_P2P;
      else throw ArgError{105, "--precision: fp64 | fp32"};
    } else if (a == "--device") cfg.device = conv<int>(a, need(i));
    else if (a == "--warmup") cfg.warmup = conv<int>(a, need(i));
    else if (a == "--overlap") cfg.overlap = true;
    else throw ArgError{109, "The following argument was not expected: " + a};
  }
  // CLI11 checks of the reference (fmm_bench.cpp:77-92)
  if (cfg.n_bodies <= 0) throw ArgError{105, "--n: Value " + std::to_string(cfg.n_bodies) + " not in range"};
  if (cfg.order <= 0) throw ArgError{105, "--p: Value not in range"};
  if (cfg.threads <= 0) throw ArgError{105, "--threads: Value not in range"};
  if (!(cfg.theta >= 1e-6 && cfg.theta <= 0.999999)) throw ArgError{105, "--theta: Value not in range [1e-06 - 0.999999]"};
  if (cfg.n_crit <= 0) throw ArgError{105, "--ncrit: Value not in range"};
  if (cfg.warmup < 0) throw ArgError{105, "--warmup: Value not in range"};
  return cfg;
}

}  // namespace

int main(int argc, char** argv) {
  RunConfig cfg;
  std::string sweep_spec;
  bool help = false;
  SweepRanges ranges;
  try {
    cfg = parse(argc, argv, sweep_spec, help);
    if (help) {
      usage();
      return 0;
    }
    if (!sweep_spec.empty()) ranges = parse_sweep_spec(sweep_spec);
  } catch (const ArgError& e) {
    std::fprintf(stderr, "%s\nRun with --help for more information.\n", e.msg.c_str());
    return e.code;
  }
  try {
    dist_config(cfg.dist);  // parse_distribution (dataset.cpp:36-41) before any work
    if (!sweep_spec.empty()) {
      std::ofstream csv;
      if (!cfg.csv_path.empty()) {
        csv.open(cfg.csv_path);
        if (!csv) throw std::runtime_error("cannot open " + cfg.csv_path);
      }
      const std::string target = cfg.csv_path;
      cfg.csv_path.clear();
      const auto rows = run_sweep(cfg, ranges, csv.is_open() ? &csv : nullptr);
      std::printf("%s\n", sweep_csv_header().c_str());
      for (const auto& row : rows) std::printf("%s\n", sweep_csv_row(row.first, row.second).c_str());
      if (!target.empty()) std::printf("wrote %zu rows to %s\n", rows.size(), target.c_str());
      return 0;
    }
    const RunResult res = run_once(cfg);
    print_result(cfg, res);
    if (cfg.check && res.has_error && res.error.rel_l2 > cfg.check_tol) {
      std::fprintf(stderr, "check failed: rel_l2 %.3e > tolerance %.3e\n", res.error.rel_l2, cfg.check_tol);
      return 2;
    }
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
