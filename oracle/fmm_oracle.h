/* fmm_oracle.h — CPU restatement of the reference FMM hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This is the parity checker for the B200 path: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it. The product path
 * (paper_1203_0889_b200) never links or calls it.
 *
 * Every function restates one reference function (file:line under /root/reference/proj)
 * in plain C with the reference's exact floating-point association (compile with
 * -ffp-contract=off). Extension beyond the reference: acceleration (= -grad phi) for
 * P2P, L2P and the direct sum (the reference is potential-only); it is pinned
 * against the long-double direct-sum gradient in tests/test_oracle.py.
 *
 * Parity pins: tests/test_oracle.py checks this restatement against the reference's own
 * known answers (proj/tests/test_*.cpp), the golden aggregates of proj/test_output.txt
 * (rel-L2 3.34e-3 / 5.89e-5 / 1.78e-6, 46 523 emitted pairs, 20 255 578 P2P evals), and
 * against oracle/_ref (the unmodified reference compiled here) through tests/golden/.
 */
#ifndef FMM_ORACLE_H
#define FMM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ORC_OK = 0,
  ORC_ERR_EMPTY_INPUT = 1,    /* "empty input"                 tree.cpp:11, :53 */
  ORC_ERR_NCRIT = 2,          /* "n_crit must be >= 1"         tree.cpp:54 */
  ORC_ERR_ORDER = 3,          /* "expansion order must be >= 1" tree.cpp:55, kernels.cpp:26 */
  ORC_ERR_LEVEL_OVERFLOW = 4, /* "level overflow"              tree.cpp:26 */
  ORC_ERR_SINGULAR_M2L = 5,   /* "singular M2L displacement"   kernels.cpp:101 */
  ORC_ERR_SINGULAR_EVAL = 6,  /* "singular evaluation point"   kernels.cpp:200 */
  ORC_ERR_CANNOT_SPLIT = 7,   /* "cannot split leaf pair"      traversal.cpp:19 */
  ORC_ERR_THETA = 8,          /* "theta must be in (0,1)"      engine.cpp:63 */
  ORC_ERR_ALLOC = 100
};

#define ORC_MAX_TREE_LEVEL 21 /* tree.hpp:14 */

int64_t orc_n_coef(int64_t p);                 /* multi_index.hpp:14 */
int orc_index_of(int a, int b, int c);         /* multi_index.hpp:32-35 */

/* MultiIndexSet (multi_index.hpp:20-54, multi_index.cpp:8-42). */
typedef struct {
  int max_degree;
  int size;
  int (*exps)[3];
  int* degree;
  double* fact;
  int* pred_index;
  int* pred_axis;
} orc_mis;

int orc_mis_init(orc_mis* s, int max_degree);
void orc_mis_free(orc_mis* s);
void orc_powers_over_factorial(const orc_mis* s, const double v[3], double* out); /* :44-50 */
void orc_powers(const orc_mis* s, const double v[3], double* out);                /* :52-57 */
void orc_laplace_derivatives(const orc_mis* s, const double r[3], double* out);   /* :59-85 */

/* KernelTables (kernels.hpp:24-54, kernels.cpp:25-76). */
typedef struct {
  int order;
  int n;
  orc_mis idx;
  int n_m2l;
  int32_t *m2l_m, *m2l_l, *m2l_d;
  double *m2l_wfwd, *m2l_wrev;
  int n_m2m;
  int32_t *m2m_src, *m2m_shift, *m2m_dst;
  int n_l2l;
  int32_t *l2l_src, *l2l_shift, *l2l_dst;
  double* l2l_w;
  double* eval_w;
} orc_tables;

int orc_tables_init(orc_tables* kt, int order);
void orc_tables_free(orc_tables* kt);

/* Operators (kernels.cpp). Bodies are SoA: pos[3*i+axis], q[i]; phi/acc accumulate (+=).
 * acc may be NULL (potential only, as in the reference). acc = -grad phi. */
void orc_p2m(const orc_tables* kt, int64_t n, const double* pos, const double* q,
             const double center[3], double* M);                                /* :78-86 */
void orc_m2m(const orc_tables* kt, const double* child_m, const double shift[3],
             double* parent_m);                                                  /* :88-96 */
int orc_m2l(const orc_tables* kt, const double* source_m, const double disp[3],
            double* target_l);                                                   /* :98-111 */
int orc_m2l_mutual(const orc_tables* kt, const double* source_m, const double* target_m,
                   const double disp[3], double* target_l, double* source_l);    /* :113-126 */
void orc_l2l(const orc_tables* kt, const double* parent_l, const double shift[3],
             double* child_l);                                                   /* :128-136 */
void orc_l2p(const orc_tables* kt, const double* L, const double center[3], int64_t n,
             const double* pos, double* phi, double* acc);                       /* :138-148 + grad */
/* p2p (kernels.cpp:150-195). self = same span. Returns the number of 1/r evaluations. */
uint64_t orc_p2p(int64_t nt, const double* tpos, const double* tq, double* tphi, double* tacc,
                 int64_t ns, const double* spos, const double* sq, double* sphi, double* sacc,
                 int self, int mutual);
int orc_evaluate_multipole(const orc_tables* kt, const double* M, const double x[3],
                           const double center[3], double* out);                 /* :197-208 */
void orc_m2p_flip(const orc_tables* kt, const double* M, double* out);           /* :210-216 */

/* Tree (tree.hpp:21-59, tree.cpp). */
typedef struct {
  int32_t level;
  uint64_t key;
  double center[3];
  double radius;
  int32_t body_begin, body_end, child_begin, child_count, parent;
} orc_cell;

typedef struct {
  double center[3];
  double half_side;
  int n_crit, order, ncoef;
  int64_t ncells, nbodies;
  orc_cell* cells;
  double* pos;    /* tree (sorted) order, 3 per body */
  double* q;
  int64_t* perm;  /* perm[i] = input index of tree-order body i */
  double* multipole; /* ncells * ncoef */
  double* local;
  double* phi;    /* tree order */
  double* acc;    /* tree order, 3 per body */
} orc_tree;

int orc_compute_bounds(int64_t n, const double* xyzq, double center[3], double* half_side); /* :10-23 */
int orc_morton_key(const double p[3], const double center[3], double half_side, int level,
                   uint64_t* out);                                                          /* :25-39 */
/* build_tree (tree.cpp:52-119). xyzq is the input AoS: x,y,z,q per body. */
int orc_build_tree(int64_t n, const double* xyzq, int n_crit, int p, orc_tree* out);
void orc_tree_free(orc_tree* t);

/* Traversal (traversal.cpp:8-34, traversal.hpp:49-133). */
int orc_mac(const orc_cell* t, const orc_cell* s, double theta);
/* Emits every M2L and P2P (target, source) pair of the BFS dual traversal from (0,0), in
 * FIFO order. Buffers are malloc'ed; caller frees with orc_free. */
int orc_traverse(const orc_tree* t, double theta, int mutual, int64_t* n_m2l, int32_t** m2l,
                 int64_t* n_p2p, int32_t** p2p);
int orc_split_pair(const orc_tree* t, int32_t target, int32_t source, int32_t* out_pairs,
                   int* n_out); /* traversal.cpp:15-34, out_pairs holds up to 8 (t,s) */
void orc_free(void* p);

void orc_upward(orc_tree* t, const orc_tables* kt);   /* traversal.cpp:36-50 */
void orc_downward(orc_tree* t, const orc_tables* kt); /* traversal.cpp:52-63 (+ acc) */
/* Applies emitted lists (KernelVisitor, traversal.hpp:138-164), non-mutual or mutual. */
int orc_apply_lists(orc_tree* t, const orc_tables* kt, int64_t n_m2l, const int32_t* m2l,
                    int64_t n_p2p, const int32_t* p2p, int mutual, uint64_t* p2p_evals);
/* The serial pipeline of test_traversal.cpp:292-318: upward, traverse, kernels, downward.
 * with_acc = 0 reproduces the reference's potential-only arithmetic. */
int orc_evaluate(orc_tree* t, double theta, int mutual, int with_acc, uint64_t* p2p_evals,
                 int64_t* n_m2l, int64_t* n_p2p);

/* Parallel checker (OpenMP), bit-identical to orc_evaluate for the non-mutual mode: upward and
 * downward level by level, kernels per target cell with each target's contributions applied in
 * the FIFO emission order. cell_mask (ncells bytes, optional) restricts phi/acc to the marked
 * leaves (ancestors added internally). */
int orc_evaluate_par(orc_tree* t, double theta, int with_acc, const uint8_t* cell_mask,
                     uint64_t* p2p_evals, int64_t* n_m2l, int64_t* n_p2p);
/* Stable counting sort of (target, source) pairs into CSR by target; sort_sources = 1 sorts
 * each target's sources ascending (the canonical multiset form). */
int orc_group_by_target(int64_t ncells, int64_t n, const int32_t* pairs, int64_t* offsets,
                        int32_t* sources, int sort_sources);
/* direct_sum restricted to the listed targets (input order indices), all sources. */
void orc_direct_sum_targets(int64_t n, const double* pos, const double* q, int64_t nt,
                            const int64_t* idx, double* phi, double* acc);
/* BASELINE.json configs 1..5; output AoS xyzq. */
int orc_generate_baseline_bodies(int config, int64_t n, uint64_t seed, double* xyzq);

/* direct_sum (oracle.cpp:8-23) in long double; acc extension; input order arrays. */
void orc_direct_sum(int64_t n, const double* pos, const double* q, double* phi, double* acc);
/* compare (oracle.cpp:25-47). Returns 0 or ORC_ERR_EMPTY_INPUT-free status. */
void orc_compare(int64_t n, const double* a, const double* b, double* rel_l2, double* rel_linf,
                 int* absolute);

/* Reference generator (dataset.cpp:10-34): splitmix64-seeded xorshift64*. */
typedef struct { uint64_t state; } orc_rng;
void orc_rng_init(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next(orc_rng* r);
double orc_rng_uniform01(orc_rng* r);
double orc_rng_uniform(orc_rng* r, double lo, double hi);
/* generate_bodies (dataset.cpp:74-112) with g++'s right-to-left Vec3 argument order.
 * dist: 0 cube, 1 sphere-surface, 2 cluster. Output AoS xyzq. */
int orc_generate_reference_bodies(int dist, int64_t n, uint64_t seed, double* xyzq);

#ifdef __cplusplus
}
#endif
#endif
