/* fmm_oracle.c — CPU restatement of the reference FMM hot path. TEST INFRASTRUCTURE ONLY.
 * See fmm_oracle.h for the contract. Compile with -ffp-contract=off: every expression
 * below keeps the reference's association so that, applied in the same order, results
 * are bit-identical to the reference (tests/test_oracle.py pins this against oracle/_ref).
 * Citations are /root/reference/proj/<file>:<line>. */
#include "fmm_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- multi-index -- */

int64_t orc_n_coef(int64_t p) { return p * (p + 1) * (p + 2) / 6; } /* multi_index.hpp:14 */

int orc_index_of(int a, int b, int c) { /* multi_index.hpp:32-35 */
  const int n = a + b + c;
  return (int)orc_n_coef(n) + a * (n + 1) - a * (a - 1) / 2 + b;
}

int orc_mis_init(orc_mis* s, int max_degree) { /* multi_index.cpp:8-42 */
  memset(s, 0, sizeof(*s));
  s->max_degree = max_degree;
  const int total = (int)orc_n_coef(max_degree + 1);
  s->size = total;
  s->exps = malloc(sizeof(int[3]) * (size_t)(total > 0 ? total : 1));
  s->degree = malloc(sizeof(int) * (size_t)(total > 0 ? total : 1));
  s->fact = malloc(sizeof(double) * (size_t)(total > 0 ? total : 1));
  s->pred_index = malloc(sizeof(int) * (size_t)(total > 0 ? total : 1));
  s->pred_axis = malloc(sizeof(int) * (size_t)(total > 0 ? total : 1));
  if (!s->exps || !s->degree || !s->fact || !s->pred_index || !s->pred_axis) return ORC_ERR_ALLOC;
  int i = 0;
  for (int n = 0; n <= max_degree; ++n) {
    for (int a = 0; a <= n; ++a) {
      for (int b = 0; b <= n - a; ++b) {
        const int c = n - a - b;
        s->exps[i][0] = a;
        s->exps[i][1] = b;
        s->exps[i][2] = c;
        s->degree[i] = n;
        double f = 1.0;
        for (int k = 2; k <= a; ++k) f *= k;
        for (int k = 2; k <= b; ++k) f *= k;
        for (int k = 2; k <= c; ++k) f *= k;
        s->fact[i] = f;
        if (n == 0) {
          s->pred_index[i] = -1;
          s->pred_axis[i] = -1;
        } else {
          const int axis = a > 0 ? 0 : (b > 0 ? 1 : 2);
          s->pred_index[i] = orc_index_of(a - (axis == 0), b - (axis == 1), c - (axis == 2));
          s->pred_axis[i] = axis;
        }
        ++i;
      }
    }
  }
  return ORC_OK;
}

void orc_mis_free(orc_mis* s) {
  free(s->exps);
  free(s->degree);
  free(s->fact);
  free(s->pred_index);
  free(s->pred_axis);
  memset(s, 0, sizeof(*s));
}

void orc_powers_over_factorial(const orc_mis* s, const double v[3], double* out) {
  out[0] = 1.0; /* multi_index.cpp:44-50 */
  for (int i = 1; i < s->size; ++i) {
    const int axis = s->pred_axis[i];
    out[i] = out[s->pred_index[i]] * v[axis] / s->exps[i][axis];
  }
}

void orc_powers(const orc_mis* s, const double v[3], double* out) {
  out[0] = 1.0; /* multi_index.cpp:52-57 */
  for (int i = 1; i < s->size; ++i) out[i] = out[s->pred_index[i]] * v[s->pred_axis[i]];
}

void orc_laplace_derivatives(const orc_mis* s, const double r[3], double* out) {
  /* multi_index.cpp:59-85: T_0 = 1/|r|; n r^2 T_g = -(2n-1) sum r_d T_{g-e_d} - (n-1) sum T_{g-2e_d} */
  const double r2 = (r[0] * r[0] + r[1] * r[1]) + r[2] * r[2];
  const double inv_r2 = 1.0 / r2;
  out[0] = 1.0 / sqrt(r2);
  for (int i = 1; i < s->size; ++i) {
    const int* e = s->exps[i];
    const int n = s->degree[i];
    double s1 = 0.0, s2 = 0.0;
    for (int d = 0; d < 3; ++d) {
      if (e[d] >= 1) {
        int g[3] = {e[0], e[1], e[2]};
        --g[d];
        s1 += r[d] * out[orc_index_of(g[0], g[1], g[2])];
      }
      if (e[d] >= 2) {
        int g[3] = {e[0], e[1], e[2]};
        g[d] -= 2;
        s2 += out[orc_index_of(g[0], g[1], g[2])];
      }
    }
    out[i] = -((double)(2 * n - 1) * s1 + (double)(n - 1) * s2) * inv_r2 / n;
  }
}

/* --------------------------------------------------------------- kernel tables -- */

int orc_tables_init(orc_tables* kt, int order) { /* kernels.cpp:25-76 */
  memset(kt, 0, sizeof(*kt));
  if (order < 1) return ORC_ERR_ORDER;
  kt->order = order;
  int rc = orc_mis_init(&kt->idx, order - 1);
  if (rc) return rc;
  const int n = kt->idx.size;
  const int max_deg = order - 1;
  kt->n = n;
  const orc_mis* I = &kt->idx;
  /* count terms */
  int nm2l = 0, nm2m = 0, nl2l = 0;
  for (int ia = 0; ia < n; ++ia)
    for (int ib = 0; ib < n; ++ib)
      if (I->degree[ia] + I->degree[ib] <= max_deg) ++nm2l;
  for (int ib = 0; ib < n; ++ib) nm2m += (I->exps[ib][0] + 1) * (I->exps[ib][1] + 1) * (I->exps[ib][2] + 1);
  nl2l = nm2l;
  kt->m2l_m = malloc(sizeof(int32_t) * nm2l);
  kt->m2l_l = malloc(sizeof(int32_t) * nm2l);
  kt->m2l_d = malloc(sizeof(int32_t) * nm2l);
  kt->m2l_wfwd = malloc(sizeof(double) * nm2l);
  kt->m2l_wrev = malloc(sizeof(double) * nm2l);
  kt->m2m_src = malloc(sizeof(int32_t) * nm2m);
  kt->m2m_shift = malloc(sizeof(int32_t) * nm2m);
  kt->m2m_dst = malloc(sizeof(int32_t) * nm2m);
  kt->l2l_src = malloc(sizeof(int32_t) * nl2l);
  kt->l2l_shift = malloc(sizeof(int32_t) * nl2l);
  kt->l2l_dst = malloc(sizeof(int32_t) * nl2l);
  kt->l2l_w = malloc(sizeof(double) * nl2l);
  kt->eval_w = malloc(sizeof(double) * n);
  /* M2L: one term per (alpha, beta) with |alpha+beta| <= p-1 (kernels.cpp:30-44) */
  int k = 0;
  for (int ia = 0; ia < n; ++ia) {
    const int* a = I->exps[ia];
    const int da = I->degree[ia];
    for (int ib = 0; ib < n; ++ib) {
      const int db = I->degree[ib];
      if (da + db > max_deg) continue;
      const int* b = I->exps[ib];
      const int ig = orc_index_of(a[0] + b[0], a[1] + b[1], a[2] + b[2]);
      const double kk = I->fact[ig] / I->fact[ib];
      const double sign_b = (db % 2 == 0) ? 1.0 : -1.0;
      const double sign_a = (da % 2 == 0) ? 1.0 : -1.0;
      kt->m2l_m[k] = ia;
      kt->m2l_l[k] = ib;
      kt->m2l_d[k] = ig;
      kt->m2l_wfwd[k] = sign_b * kk;
      kt->m2l_wrev[k] = sign_a * kk;
      ++k;
    }
  }
  kt->n_m2l = k;
  /* M2M: parent_b += child_a * d^{b-a}/(b-a)! (kernels.cpp:46-58) */
  k = 0;
  for (int ib = 0; ib < n; ++ib) {
    const int* b = I->exps[ib];
    for (int ax = 0; ax <= b[0]; ++ax)
      for (int ay = 0; ay <= b[1]; ++ay)
        for (int az = 0; az <= b[2]; ++az) {
          kt->m2m_src[k] = orc_index_of(ax, ay, az);
          kt->m2m_shift[k] = orc_index_of(b[0] - ax, b[1] - ay, b[2] - az);
          kt->m2m_dst[k] = ib;
          ++k;
        }
  }
  kt->n_m2m = k;
  /* L2L: child_a += parent_{a+d} ((a+d)!/a!) d^d/d! (kernels.cpp:60-70) */
  k = 0;
  for (int ia = 0; ia < n; ++ia) {
    const int* a = I->exps[ia];
    const int da = I->degree[ia];
    for (int is = 0; is < n; ++is) {
      if (da + I->degree[is] > max_deg) continue;
      const int* s = I->exps[is];
      const int ip = orc_index_of(a[0] + s[0], a[1] + s[1], a[2] + s[2]);
      kt->l2l_src[k] = ip;
      kt->l2l_shift[k] = is;
      kt->l2l_dst[k] = ia;
      kt->l2l_w[k] = I->fact[ip] / I->fact[ia];
      ++k;
    }
  }
  kt->n_l2l = k;
  for (int i = 0; i < n; ++i) /* kernels.cpp:72-75 */
    kt->eval_w[i] = (I->degree[i] % 2 == 0 ? 1.0 : -1.0) * I->fact[i];
  return ORC_OK;
}

void orc_tables_free(orc_tables* kt) {
  orc_mis_free(&kt->idx);
  free(kt->m2l_m); free(kt->m2l_l); free(kt->m2l_d); free(kt->m2l_wfwd); free(kt->m2l_wrev);
  free(kt->m2m_src); free(kt->m2m_shift); free(kt->m2m_dst);
  free(kt->l2l_src); free(kt->l2l_shift); free(kt->l2l_dst); free(kt->l2l_w);
  free(kt->eval_w);
  memset(kt, 0, sizeof(*kt));
}

/* ------------------------------------------------------------------ operators -- */

void orc_p2m(const orc_tables* kt, int64_t n, const double* pos, const double* q,
             const double center[3], double* M) { /* kernels.cpp:78-86 */
  double u[4096];
  for (int64_t j = 0; j < n; ++j) {
    const double v[3] = {pos[3 * j] - center[0], pos[3 * j + 1] - center[1], pos[3 * j + 2] - center[2]};
    orc_powers_over_factorial(&kt->idx, v, u);
    for (int i = 0; i < kt->n; ++i) M[i] += q[j] * u[i];
  }
}

void orc_m2m(const orc_tables* kt, const double* child_m, const double shift[3], double* parent_m) {
  double u[4096]; /* kernels.cpp:88-96 */
  orc_powers_over_factorial(&kt->idx, shift, u);
  for (int t = 0; t < kt->n_m2m; ++t) parent_m[kt->m2m_dst[t]] += child_m[kt->m2m_src[t]] * u[kt->m2m_shift[t]];
}

int orc_m2l(const orc_tables* kt, const double* source_m, const double disp[3], double* target_l) {
  /* kernels.cpp:98-111 */
  if ((disp[0] * disp[0] + disp[1] * disp[1]) + disp[2] * disp[2] == 0.0) return ORC_ERR_SINGULAR_M2L;
  double d[4096];
  orc_laplace_derivatives(&kt->idx, disp, d);
  for (int t = 0; t < kt->n_m2l; ++t)
    target_l[kt->m2l_l[t]] += kt->m2l_wfwd[t] * source_m[kt->m2l_m[t]] * d[kt->m2l_d[t]];
  return ORC_OK;
}

int orc_m2l_mutual(const orc_tables* kt, const double* source_m, const double* target_m,
                   const double disp[3], double* target_l, double* source_l) {
  /* kernels.cpp:113-126 */
  if ((disp[0] * disp[0] + disp[1] * disp[1]) + disp[2] * disp[2] == 0.0) return ORC_ERR_SINGULAR_M2L;
  double d[4096];
  orc_laplace_derivatives(&kt->idx, disp, d);
  for (int t = 0; t < kt->n_m2l; ++t) {
    target_l[kt->m2l_l[t]] += kt->m2l_wfwd[t] * source_m[kt->m2l_m[t]] * d[kt->m2l_d[t]];
    source_l[kt->m2l_l[t]] += kt->m2l_wrev[t] * target_m[kt->m2l_m[t]] * d[kt->m2l_d[t]];
  }
  return ORC_OK;
}

void orc_l2l(const orc_tables* kt, const double* parent_l, const double shift[3], double* child_l) {
  double u[4096]; /* kernels.cpp:128-136 */
  orc_powers_over_factorial(&kt->idx, shift, u);
  for (int t = 0; t < kt->n_l2l; ++t)
    child_l[kt->l2l_dst[t]] += parent_l[kt->l2l_src[t]] * kt->l2l_w[t] * u[kt->l2l_shift[t]];
}

void orc_l2p(const orc_tables* kt, const double* L, const double center[3], int64_t n,
             const double* pos, double* phi, double* acc) {
  /* kernels.cpp:138-148. Extension: acc -= grad of sum_b L_b (x-c)^b,
   * d/dx_d (x-c)^b = b_d (x-c)^{b-e_d}. */
  double m[4096];
  const orc_mis* I = &kt->idx;
  for (int64_t j = 0; j < n; ++j) {
    const double v[3] = {pos[3 * j] - center[0], pos[3 * j + 1] - center[1], pos[3 * j + 2] - center[2]};
    orc_powers(I, v, m);
    double ph = 0.0;
    for (int i = 0; i < kt->n; ++i) ph += L[i] * m[i];
    phi[j] += ph;
    if (acc) {
      double g[3] = {0.0, 0.0, 0.0};
      for (int i = 1; i < kt->n; ++i) {
        const int* e = I->exps[i];
        for (int d = 0; d < 3; ++d) {
          if (e[d] == 0) continue;
          int f[3] = {e[0], e[1], e[2]};
          --f[d];
          g[d] += L[i] * (double)e[d] * m[orc_index_of(f[0], f[1], f[2])];
        }
      }
      acc[3 * j] -= g[0];
      acc[3 * j + 1] -= g[1];
      acc[3 * j + 2] -= g[2];
    }
  }
}

uint64_t orc_p2p(int64_t nt, const double* tpos, const double* tq, double* tphi, double* tacc,
                 int64_t ns, const double* spos, const double* sq, double* sphi, double* sacc,
                 int self, int mutual) {
  /* kernels.cpp:150-195. Extension: acc_i += q_j (x_i - y_j)/r^3 (= -grad_i phi). */
  uint64_t evals = 0;
  if (self && mutual) {
    for (int64_t i = 0; i < nt; ++i) {
      double phi_i = 0.0, ax = 0.0, ay = 0.0, az = 0.0;
      for (int64_t j = 0; j < i; ++j) {
        const double dx = tpos[3 * i] - tpos[3 * j], dy = tpos[3 * i + 1] - tpos[3 * j + 1],
                     dz = tpos[3 * i + 2] - tpos[3 * j + 2];
        const double r2 = (dx * dx + dy * dy) + dz * dz;
        if (r2 == 0.0) continue;
        ++evals;
        const double inv_r = 1.0 / sqrt(r2);
        phi_i += tq[j] * inv_r;
        tphi[j] += tq[i] * inv_r;
        if (tacc) {
          const double inv_r3 = inv_r * inv_r * inv_r;
          ax += tq[j] * dx * inv_r3; ay += tq[j] * dy * inv_r3; az += tq[j] * dz * inv_r3;
          tacc[3 * j] -= tq[i] * dx * inv_r3; tacc[3 * j + 1] -= tq[i] * dy * inv_r3;
          tacc[3 * j + 2] -= tq[i] * dz * inv_r3;
        }
      }
      tphi[i] += phi_i;
      if (tacc) { tacc[3 * i] += ax; tacc[3 * i + 1] += ay; tacc[3 * i + 2] += az; }
    }
  } else if (mutual) {
    for (int64_t i = 0; i < nt; ++i) {
      double phi_i = 0.0, ax = 0.0, ay = 0.0, az = 0.0;
      for (int64_t j = 0; j < ns; ++j) {
        const double dx = tpos[3 * i] - spos[3 * j], dy = tpos[3 * i + 1] - spos[3 * j + 1],
                     dz = tpos[3 * i + 2] - spos[3 * j + 2];
        const double r2 = (dx * dx + dy * dy) + dz * dz;
        if (r2 == 0.0) continue;
        ++evals;
        const double inv_r = 1.0 / sqrt(r2);
        phi_i += sq[j] * inv_r;
        sphi[j] += tq[i] * inv_r;
        if (tacc) {
          const double inv_r3 = inv_r * inv_r * inv_r;
          ax += sq[j] * dx * inv_r3; ay += sq[j] * dy * inv_r3; az += sq[j] * dz * inv_r3;
        }
        if (sacc) {
          const double inv_r3 = inv_r * inv_r * inv_r;
          sacc[3 * j] -= tq[i] * dx * inv_r3; sacc[3 * j + 1] -= tq[i] * dy * inv_r3;
          sacc[3 * j + 2] -= tq[i] * dz * inv_r3;
        }
      }
      tphi[i] += phi_i;
      if (tacc) { tacc[3 * i] += ax; tacc[3 * i + 1] += ay; tacc[3 * i + 2] += az; }
    }
  } else {
    for (int64_t i = 0; i < nt; ++i) {
      double phi_i = 0.0, ax = 0.0, ay = 0.0, az = 0.0;
      for (int64_t j = 0; j < ns; ++j) {
        const double dx = tpos[3 * i] - spos[3 * j], dy = tpos[3 * i + 1] - spos[3 * j + 1],
                     dz = tpos[3 * i + 2] - spos[3 * j + 2];
        const double r2 = (dx * dx + dy * dy) + dz * dz;
        if (r2 == 0.0) continue;
        ++evals;
        phi_i += sq[j] / sqrt(r2);
        if (tacc) {
          const double inv_r = 1.0 / sqrt(r2);
          const double inv_r3 = inv_r * inv_r * inv_r;
          ax += sq[j] * dx * inv_r3; ay += sq[j] * dy * inv_r3; az += sq[j] * dz * inv_r3;
        }
      }
      tphi[i] += phi_i;
      if (tacc) { tacc[3 * i] += ax; tacc[3 * i + 1] += ay; tacc[3 * i + 2] += az; }
    }
  }
  (void)sphi;
  return evals;
}

int orc_evaluate_multipole(const orc_tables* kt, const double* M, const double x[3],
                           const double center[3], double* out) { /* kernels.cpp:197-208 */
  const double r[3] = {x[0] - center[0], x[1] - center[1], x[2] - center[2]};
  if ((r[0] * r[0] + r[1] * r[1]) + r[2] * r[2] == 0.0) return ORC_ERR_SINGULAR_EVAL;
  double d[4096];
  orc_laplace_derivatives(&kt->idx, r, d);
  double phi = 0.0;
  for (int i = 0; i < kt->n; ++i) phi += kt->eval_w[i] * M[i] * d[i];
  *out = phi;
  return ORC_OK;
}

void orc_m2p_flip(const orc_tables* kt, const double* M, double* out) { /* kernels.cpp:210-216 */
  for (int i = 0; i < kt->n; ++i) out[i] = (kt->idx.degree[i] % 2 != 0) ? -M[i] : M[i];
}

/* ----------------------------------------------------------------------- tree -- */

int orc_compute_bounds(int64_t n, const double* xyzq, double center[3], double* half_side) {
  if (n <= 0) return ORC_ERR_EMPTY_INPUT; /* tree.cpp:10-23 */
  double lo[3] = {xyzq[0], xyzq[1], xyzq[2]}, hi[3] = {xyzq[0], xyzq[1], xyzq[2]};
  for (int64_t i = 0; i < n; ++i)
    for (int d = 0; d < 3; ++d) {
      const double v = xyzq[4 * i + d];
      lo[d] = v < lo[d] ? v : lo[d];
      hi[d] = hi[d] < v ? v : hi[d];
    }
  for (int d = 0; d < 3; ++d) center[d] = 0.5 * (lo[d] + hi[d]);
  double ext = hi[0] - lo[0];
  for (int d = 1; d < 3; ++d) ext = ext < (hi[d] - lo[d]) ? (hi[d] - lo[d]) : ext;
  const double extent_half = 0.5 * ext;
  const double h = extent_half * (1.0 + 1e-6);
  *half_side = h < 0.5 ? 0.5 : h; /* std::max(h, kMinHalfSide) */
  return ORC_OK;
}

int orc_morton_key(const double p[3], const double center[3], double half_side, int level,
                   uint64_t* out) { /* tree.cpp:25-39 */
  if (level < 0 || level > ORC_MAX_TREE_LEVEL) return ORC_ERR_LEVEL_OVERFLOW;
  const uint64_t cells_per_axis = (uint64_t)1 << level;
  const double inv_cell = (double)cells_per_axis / (2.0 * half_side);
  uint64_t key = 0;
  for (int axis = 0; axis < 3; ++axis) {
    const double offset = p[axis] - (center[axis] - half_side);
    int64_t idx = (int64_t)floor(offset * inv_cell);
    if (idx < 0) idx = 0;
    if (idx > (int64_t)cells_per_axis - 1) idx = (int64_t)cells_per_axis - 1;
    for (int bit = 0; bit < level; ++bit) key |= (((uint64_t)idx >> bit) & 1u) << (3 * bit + axis);
  }
  *out = key;
  return ORC_OK;
}

static int octant_of(const double* p, const double* c) { /* tree.cpp:45-48 */
  return (p[0] >= c[0] ? 1 : 0) | (p[1] >= c[1] ? 2 : 0) | (p[2] >= c[2] ? 4 : 0);
}

int orc_build_tree(int64_t n, const double* xyzq, int n_crit, int p, orc_tree* out) {
  memset(out, 0, sizeof(*out)); /* tree.cpp:52-119 */
  if (n <= 0) return ORC_ERR_EMPTY_INPUT;
  if (n_crit < 1) return ORC_ERR_NCRIT;
  if (p < 1) return ORC_ERR_ORDER;
  orc_compute_bounds(n, xyzq, out->center, &out->half_side);
  out->n_crit = n_crit;
  out->order = p;
  out->ncoef = (int)orc_n_coef(p);
  out->nbodies = n;
  int64_t* idx = malloc(sizeof(int64_t) * (size_t)n);
  int64_t* buf = malloc(sizeof(int64_t) * (size_t)n);
  int64_t cap = 1024, nc = 1;
  orc_cell* cells = malloc(sizeof(orc_cell) * (size_t)cap);
  if (!idx || !buf || !cells) return ORC_ERR_ALLOC;
  for (int64_t i = 0; i < n; ++i) idx[i] = i;
  memset(&cells[0], 0, sizeof(orc_cell));
  cells[0].parent = -1;
  memcpy(cells[0].center, out->center, sizeof(double) * 3);
  cells[0].radius = out->half_side;
  cells[0].body_end = (int32_t)n;
  for (int64_t ci = 0; ci < nc; ++ci) {
    const int32_t begin = cells[ci].body_begin, end = cells[ci].body_end;
    const int level = cells[ci].level;
    double center[3];
    memcpy(center, cells[ci].center, sizeof(center));
    const double radius = cells[ci].radius;
    if (end - begin <= n_crit || level >= ORC_MAX_TREE_LEVEL) continue;
    int32_t count[8] = {0}, offset[8] = {0}, cursor[8];
    for (int32_t bi = begin; bi < end; ++bi) ++count[octant_of(&xyzq[4 * idx[bi]], center)];
    for (int o = 1; o < 8; ++o) offset[o] = offset[o - 1] + count[o - 1];
    memcpy(buf + begin, idx + begin, sizeof(int64_t) * (size_t)(end - begin));
    memcpy(cursor, offset, sizeof(cursor));
    for (int32_t bi = begin; bi < end; ++bi) {
      const int64_t b = buf[bi];
      idx[begin + cursor[octant_of(&xyzq[4 * b], center)]++] = b;
    }
    cells[ci].child_begin = (int32_t)nc;
    const double child_radius = 0.5 * radius;
    for (int o = 0; o < 8; ++o) {
      if (count[o] == 0) continue;
      if (nc == cap) {
        cap *= 2;
        orc_cell* nc2 = realloc(cells, sizeof(orc_cell) * (size_t)cap);
        if (!nc2) return ORC_ERR_ALLOC;
        cells = nc2;
      }
      orc_cell* ch = &cells[nc];
      memset(ch, 0, sizeof(*ch));
      ch->level = level + 1;
      ch->key = (cells[ci].key << 3) | (uint64_t)o;
      ch->center[0] = center[0] + child_radius * ((o & 1) ? 1.0 : -1.0);
      ch->center[1] = center[1] + child_radius * ((o & 2) ? 1.0 : -1.0);
      ch->center[2] = center[2] + child_radius * ((o & 4) ? 1.0 : -1.0);
      ch->radius = child_radius;
      ch->body_begin = begin + offset[o];
      ch->body_end = begin + offset[o] + count[o];
      ch->parent = (int32_t)ci;
      ch->child_begin = 0;
      ch->child_count = 0;
      ++nc;
      ++cells[ci].child_count;
    }
  }
  out->cells = cells;
  out->ncells = nc;
  out->perm = idx;
  free(buf);
  out->pos = malloc(sizeof(double) * 3 * (size_t)n);
  out->q = malloc(sizeof(double) * (size_t)n);
  out->phi = calloc((size_t)n, sizeof(double));
  out->acc = calloc((size_t)n * 3, sizeof(double));
  out->multipole = calloc((size_t)nc * out->ncoef, sizeof(double));
  out->local = calloc((size_t)nc * out->ncoef, sizeof(double));
  if (!out->pos || !out->q || !out->phi || !out->acc || !out->multipole || !out->local) return ORC_ERR_ALLOC;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t b = idx[i];
    out->pos[3 * i] = xyzq[4 * b];
    out->pos[3 * i + 1] = xyzq[4 * b + 1];
    out->pos[3 * i + 2] = xyzq[4 * b + 2];
    out->q[i] = xyzq[4 * b + 3];
  }
  return ORC_OK;
}

void orc_tree_free(orc_tree* t) {
  free(t->cells); free(t->pos); free(t->q); free(t->perm); free(t->multipole); free(t->local);
  free(t->phi); free(t->acc);
  memset(t, 0, sizeof(*t));
}

/* ------------------------------------------------------------------ traversal -- */

int orc_mac(const orc_cell* t, const orc_cell* s, double theta) { /* traversal.cpp:8-13 */
  const double sqrt3 = sqrt(3.0);
  const double sum_r = sqrt3 * (t->radius + s->radius);
  const double dx = t->center[0] - s->center[0], dy = t->center[1] - s->center[1],
               dz = t->center[2] - s->center[2];
  const double dist = sqrt((dx * dx + dy * dy) + dz * dz);
  return sum_r < theta * dist;
}

int orc_split_pair(const orc_tree* t, int32_t target, int32_t source, int32_t* out_pairs, int* n_out) {
  const orc_cell* ct = &t->cells[target]; /* traversal.cpp:15-34 */
  const orc_cell* cs = &t->cells[source];
  *n_out = 0;
  if (ct->child_count == 0 && cs->child_count == 0) return ORC_ERR_CANNOT_SPLIT;
  const int split_target = ct->child_count != 0 && (cs->child_count == 0 || ct->radius >= cs->radius);
  if (split_target) {
    for (int32_t i = 0; i < ct->child_count; ++i) {
      out_pairs[2 * i] = ct->child_begin + i;
      out_pairs[2 * i + 1] = source;
    }
    *n_out = ct->child_count;
  } else {
    for (int32_t i = 0; i < cs->child_count; ++i) {
      out_pairs[2 * i] = target;
      out_pairs[2 * i + 1] = cs->child_begin + i;
    }
    *n_out = cs->child_count;
  }
  return ORC_OK;
}

typedef struct { int32_t* v; int64_t n, cap; } pairvec;

static int pv_push(pairvec* p, int32_t a, int32_t b) {
  if (p->n == p->cap) {
    p->cap = p->cap ? p->cap * 2 : 1024;
    int32_t* nv = realloc(p->v, sizeof(int32_t) * 2 * (size_t)p->cap);
    if (!nv) return ORC_ERR_ALLOC;
    p->v = nv;
  }
  p->v[2 * p->n] = a;
  p->v[2 * p->n + 1] = b;
  ++p->n;
  return ORC_OK;
}

/* split_target_side (traversal.hpp:49-58), same tree. */
static int split_target_side(const orc_tree* t, int32_t target, int32_t source) {
  const orc_cell* ct = &t->cells[target];
  const orc_cell* cs = &t->cells[source];
  if (ct->child_count == 0) return 0;
  if (cs->child_count == 0) return 1;
  if (ct->radius != cs->radius) return ct->radius > cs->radius;
  return target <= source;
}

int orc_traverse(const orc_tree* t, double theta, int mutual, int64_t* n_m2l, int32_t** m2l,
                 int64_t* n_p2p, int32_t** p2p) {
  /* dual_tree_traverse + traverse_pair with the FIFO queue (traversal.hpp:63-133); the
   * emitted multiset is Q-invariant, so the whole traversal runs inline (Q = infinity). */
  pairvec q = {0}, em = {0}, ep = {0};
  if (pv_push(&q, 0, 0)) return ORC_ERR_ALLOC;
  int64_t head = 0;
  while (head < q.n) {
    if (head > (1 << 20) && head > q.n / 2) { /* compact the consumed prefix */
      memmove(q.v, q.v + 2 * head, sizeof(int32_t) * 2 * (size_t)(q.n - head));
      q.n -= head;
      head = 0;
    }
    const int32_t tt = q.v[2 * head], ss = q.v[2 * head + 1];
    ++head;
    const orc_cell* ct = &t->cells[tt];
    const orc_cell* cs = &t->cells[ss];
    int rc = 0;
    if (orc_mac(ct, cs, theta)) {
      rc = pv_push(&em, tt, ss);
    } else if (ct->child_count == 0 && cs->child_count == 0) {
      rc = pv_push(&ep, tt, ss);
    } else if (mutual && tt == ss) {
      for (int32_t i = 0; i < ct->child_count && !rc; ++i)
        for (int32_t j = i; j < ct->child_count && !rc; ++j)
          rc = pv_push(&q, ct->child_begin + i, ct->child_begin + j);
    } else if (split_target_side(t, tt, ss)) {
      for (int32_t i = 0; i < ct->child_count && !rc; ++i) rc = pv_push(&q, ct->child_begin + i, ss);
    } else {
      for (int32_t i = 0; i < cs->child_count && !rc; ++i) rc = pv_push(&q, tt, cs->child_begin + i);
    }
    if (rc) return rc;
  }
  free(q.v);
  *n_m2l = em.n;
  *m2l = em.v;
  *n_p2p = ep.n;
  *p2p = ep.v;
  return ORC_OK;
}

void orc_free(void* p) { free(p); }

void orc_upward(orc_tree* t, const orc_tables* kt) { /* traversal.cpp:36-50 */
  const int nc = kt->n;
  for (int64_t ci = t->ncells - 1; ci >= 0; --ci) {
    const orc_cell* c = &t->cells[ci];
    double* M = t->multipole + ci * nc;
    if (c->child_count == 0) {
      orc_p2m(kt, c->body_end - c->body_begin, t->pos + 3 * (int64_t)c->body_begin,
              t->q + c->body_begin, c->center, M);
    } else {
      for (int32_t k = 0; k < c->child_count; ++k) {
        const orc_cell* ch = &t->cells[c->child_begin + k];
        const double shift[3] = {ch->center[0] - c->center[0], ch->center[1] - c->center[1],
                                 ch->center[2] - c->center[2]};
        orc_m2m(kt, t->multipole + (int64_t)(c->child_begin + k) * nc, shift, M);
      }
    }
  }
}

void orc_downward(orc_tree* t, const orc_tables* kt) { /* traversal.cpp:52-63 */
  const int nc = kt->n;
  for (int64_t ci = 0; ci < t->ncells; ++ci) {
    const orc_cell* c = &t->cells[ci];
    if (c->parent >= 0) {
      const orc_cell* pc = &t->cells[c->parent];
      const double shift[3] = {c->center[0] - pc->center[0], c->center[1] - pc->center[1],
                               c->center[2] - pc->center[2]};
      orc_l2l(kt, t->local + (int64_t)c->parent * nc, shift, t->local + ci * nc);
    }
    if (c->child_count == 0)
      orc_l2p(kt, t->local + ci * nc, c->center, c->body_end - c->body_begin,
              t->pos + 3 * (int64_t)c->body_begin, t->phi + c->body_begin,
              t->acc ? t->acc + 3 * (int64_t)c->body_begin : NULL);
  }
}

static int apply_m2l(orc_tree* t, const orc_tables* kt, int32_t ti, int32_t si, int mutual) {
  const int nc = kt->n; /* KernelVisitor::m2l_pair, traversal.hpp:143-152 */
  const orc_cell* ct = &t->cells[ti];
  const orc_cell* cs = &t->cells[si];
  const double disp[3] = {cs->center[0] - ct->center[0], cs->center[1] - ct->center[1],
                          cs->center[2] - ct->center[2]};
  if (mutual)
    return orc_m2l_mutual(kt, t->multipole + (int64_t)si * nc, t->multipole + (int64_t)ti * nc, disp,
                          t->local + (int64_t)ti * nc, t->local + (int64_t)si * nc);
  return orc_m2l(kt, t->multipole + (int64_t)si * nc, disp, t->local + (int64_t)ti * nc);
}

static uint64_t apply_p2p(orc_tree* t, int32_t ti, int32_t si, int mutual, int with_acc) {
  const orc_cell* ct = &t->cells[ti]; /* KernelVisitor::p2p_pair, traversal.hpp:154-157 */
  const orc_cell* cs = &t->cells[si];
  double* acc = with_acc ? t->acc : NULL;
  return orc_p2p(ct->body_end - ct->body_begin, t->pos + 3 * (int64_t)ct->body_begin, t->q + ct->body_begin,
                 t->phi + ct->body_begin, acc ? acc + 3 * (int64_t)ct->body_begin : NULL,
                 cs->body_end - cs->body_begin, t->pos + 3 * (int64_t)cs->body_begin, t->q + cs->body_begin,
                 t->phi + cs->body_begin, acc ? acc + 3 * (int64_t)cs->body_begin : NULL, ti == si, mutual);
}

int orc_apply_lists(orc_tree* t, const orc_tables* kt, int64_t n_m2l, const int32_t* m2l,
                    int64_t n_p2p, const int32_t* p2p, int mutual, uint64_t* p2p_evals) {
  uint64_t ev = 0;
  for (int64_t i = 0; i < n_m2l; ++i) {
    const int rc = apply_m2l(t, kt, m2l[2 * i], m2l[2 * i + 1], mutual);
    if (rc) return rc;
  }
  for (int64_t i = 0; i < n_p2p; ++i) ev += apply_p2p(t, p2p[2 * i], p2p[2 * i + 1], mutual, 1);
  if (p2p_evals) *p2p_evals = ev;
  return ORC_OK;
}

/* Serial pipeline (test_traversal.cpp:292-318) with kernels applied in the FIFO emission
 * order of the inline traversal, exactly as KernelVisitor would see them. */
int orc_evaluate(orc_tree* t, double theta, int mutual, int with_acc, uint64_t* p2p_evals,
                 int64_t* n_m2l_out, int64_t* n_p2p_out) {
  orc_tables kt;
  int rc = orc_tables_init(&kt, t->order);
  if (rc) return rc;
  double* acc_save = t->acc;
  if (!with_acc) t->acc = NULL;
  orc_upward(t, &kt);
  /* traversal with the visitor applied inline (same FIFO order as orc_traverse) */
  pairvec q = {0};
  uint64_t ev = 0;
  int64_t nm = 0, np = 0;
  if (pv_push(&q, 0, 0)) return ORC_ERR_ALLOC;
  int64_t head = 0;
  while (head < q.n && !rc) {
    if (head > (1 << 20) && head > q.n / 2) {
      memmove(q.v, q.v + 2 * head, sizeof(int32_t) * 2 * (size_t)(q.n - head));
      q.n -= head;
      head = 0;
    }
    const int32_t tt = q.v[2 * head], ss = q.v[2 * head + 1];
    ++head;
    const orc_cell* ct = &t->cells[tt];
    const orc_cell* cs = &t->cells[ss];
    if (orc_mac(ct, cs, theta)) {
      rc = apply_m2l(t, &kt, tt, ss, mutual);
      nm += mutual && tt != ss ? 2 : 1;
    } else if (ct->child_count == 0 && cs->child_count == 0) {
      ev += apply_p2p(t, tt, ss, mutual, with_acc);
      ++np;
    } else if (mutual && tt == ss) {
      for (int32_t i = 0; i < ct->child_count && !rc; ++i)
        for (int32_t j = i; j < ct->child_count && !rc; ++j) rc = pv_push(&q, ct->child_begin + i, ct->child_begin + j);
    } else if (split_target_side(t, tt, ss)) {
      for (int32_t i = 0; i < ct->child_count && !rc; ++i) rc = pv_push(&q, ct->child_begin + i, ss);
    } else {
      for (int32_t i = 0; i < cs->child_count && !rc; ++i) rc = pv_push(&q, tt, cs->child_begin + i);
    }
  }
  free(q.v);
  if (!rc) orc_downward(t, &kt);
  t->acc = acc_save;
  orc_tables_free(&kt);
  if (p2p_evals) *p2p_evals = ev;
  if (n_m2l_out) *n_m2l_out = nm;
  if (n_p2p_out) *n_p2p_out = np;
  return rc;
}

/* --------------------------------------------------------------------- oracle -- */

void orc_direct_sum(int64_t n, const double* pos, const double* q, double* phi, double* acc) {
  for (int64_t i = 0; i < n; ++i) { /* oracle.cpp:8-23 (+ acc in long double) */
    long double s = 0.0L, ax = 0.0L, ay = 0.0L, az = 0.0L;
    for (int64_t j = 0; j < n; ++j) {
      if (j == i) continue;
      const double dx = pos[3 * i] - pos[3 * j], dy = pos[3 * i + 1] - pos[3 * j + 1],
                   dz = pos[3 * i + 2] - pos[3 * j + 2];
      const double r2 = (dx * dx + dy * dy) + dz * dz;
      if (r2 == 0.0) continue;
      const long double inv_r = 1.0L / sqrtl((long double)r2);
      s += (long double)q[j] * inv_r;
      if (acc) {
        const long double w = (long double)q[j] * inv_r * inv_r * inv_r;
        ax += w * (long double)dx;
        ay += w * (long double)dy;
        az += w * (long double)dz;
      }
    }
    phi[i] = (double)s;
    if (acc) {
      acc[3 * i] = (double)ax;
      acc[3 * i + 1] = (double)ay;
      acc[3 * i + 2] = (double)az;
    }
  }
}

void orc_compare(int64_t n, const double* a, const double* b, double* rel_l2, double* rel_linf,
                 int* absolute) { /* oracle.cpp:25-47 */
  long double diff2 = 0.0L, ref2 = 0.0L;
  double diff_inf = 0.0, ref_inf = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double d = a[i] - b[i];
    diff2 += (long double)d * d;
    ref2 += (long double)b[i] * b[i];
    diff_inf = fabs(d) > diff_inf ? fabs(d) : diff_inf;
    ref_inf = fabs(b[i]) > ref_inf ? fabs(b[i]) : ref_inf;
  }
  if (ref2 == 0.0L) {
    *absolute = 1;
    *rel_l2 = (double)sqrtl(diff2);
    *rel_linf = diff_inf;
  } else {
    *absolute = 0;
    *rel_l2 = (double)sqrtl(diff2 / ref2);
    *rel_linf = diff_inf / ref_inf;
  }
}

/* ---------------------------------------------------------------- generator -- */

static uint64_t splitmix64(uint64_t x) { /* dataset.cpp:10-16 */
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

void orc_rng_init(orc_rng* r, uint64_t seed) { /* dataset.cpp:19-21 */
  r->state = splitmix64(seed);
  if (r->state == 0) r->state = 0x9E3779B97F4A7C15ULL;
}

uint64_t orc_rng_next(orc_rng* r) { /* dataset.cpp:23-28 */
  r->state ^= r->state >> 12;
  r->state ^= r->state << 25;
  r->state ^= r->state >> 27;
  return r->state * 2685821657736338717ULL;
}

double orc_rng_uniform01(orc_rng* r) { return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53; }
double orc_rng_uniform(orc_rng* r, double lo, double hi) { return lo + (hi - lo) * orc_rng_uniform01(r); }

static double pseudo_normal(orc_rng* r) { /* dataset.cpp:67-71 */
  double s = 0.0;
  for (int k = 0; k < 12; ++k) s += orc_rng_uniform01(r);
  return s - 6.0;
}

int orc_generate_reference_bodies(int dist, int64_t n, uint64_t seed, double* xyzq) {
  if (n < 1) return ORC_ERR_EMPTY_INPUT; /* dataset.cpp:74-112 */
  orc_rng r;
  orc_rng_init(&r, seed);
  double centers[8][3];
  if (dist == 2)
    for (int k = 0; k < 8; ++k) { /* Vec3(u,u,u): g++ evaluates right to left */
      centers[k][2] = orc_rng_uniform01(&r);
      centers[k][1] = orc_rng_uniform01(&r);
      centers[k][0] = orc_rng_uniform01(&r);
    }
  for (int64_t i = 0; i < n; ++i) {
    double* b = xyzq + 4 * i;
    if (dist == 0) {
      b[2] = orc_rng_uniform01(&r);
      b[1] = orc_rng_uniform01(&r);
      b[0] = orc_rng_uniform01(&r);
    } else if (dist == 1) {
      for (;;) {
        double v[3];
        v[2] = orc_rng_uniform(&r, -1.0, 1.0);
        v[1] = orc_rng_uniform(&r, -1.0, 1.0);
        v[0] = orc_rng_uniform(&r, -1.0, 1.0);
        const double r2 = (v[0] * v[0] + v[1] * v[1]) + v[2] * v[2];
        if (r2 > 1.0 || r2 < 1e-8) continue;
        const double s = sqrt(r2);
        b[0] = v[0] / s;
        b[1] = v[1] / s;
        b[2] = v[2] / s;
        break;
      }
    } else {
      const double* c = centers[orc_rng_next(&r) % 8];
      double g[3];
      g[2] = pseudo_normal(&r);
      g[1] = pseudo_normal(&r);
      g[0] = pseudo_normal(&r);
      for (int d = 0; d < 3; ++d) b[d] = c[d] + 0.03 * g[d];
    }
    b[3] = orc_rng_uniform(&r, -1.0, 1.0);
  }
  double mean = 0.0;
  for (int64_t i = 0; i < n; ++i) mean += xyzq[4 * i + 3];
  mean /= (double)n;
  for (int64_t i = 0; i < n; ++i) xyzq[4 * i + 3] -= mean;
  return ORC_OK;
}

/* ------------------------------------------------- parallel checker (tests only) -- */
/* The non-mutual pipeline of orc_evaluate, split so that it runs on all host cores and stays
 * BIT-IDENTICAL to the serial version: every accumulation target sees its contributions in the
 * serial order.
 *   upward   level by level, deepest first (tree.cpp builds cells in BFS order, so a level is a
 *            contiguous range; a parent reads only its children, in child order);
 *   lists    the FIFO-emitted lists of orc_traverse, grouped by target with a STABLE counting
 *            sort (each target keeps its emission order, KernelVisitor traversal.hpp:138-164);
 *   kernels  one target cell per task: its M2L sources then its P2P sources in that order (M2L
 *            writes locals, P2P writes body potentials: the serial interleaving of the two is
 *            irrelevant);
 *   downward level by level, root first (traversal.cpp:52-63).
 * cell_mask (optional, ncells bytes): evaluate only the marked leaves; their ancestors are
 * added here. Unmarked leaves keep phi = acc = 0 and unmarked cells' locals are not formed. */
static int orc_level_ranges(const orc_tree* t, int64_t* lb /* [ORC_MAX_TREE_LEVEL + 2] */, int* nlev) {
  int L = -1;
  for (int64_t ci = 0; ci < t->ncells; ++ci) {
    const int lv = t->cells[ci].level;
    if (lv < L || lv > ORC_MAX_TREE_LEVEL) return 1; /* not BFS ordered */
    while (L < lv) lb[++L] = ci;
  }
  lb[L + 1] = t->ncells;
  *nlev = L + 1;
  return 0;
}

int orc_group_by_target(int64_t ncells, int64_t n, const int32_t* pairs, int64_t* offsets,
                        int32_t* sources, int sort_sources) {
  memset(offsets, 0, sizeof(int64_t) * (size_t)(ncells + 1));
  for (int64_t i = 0; i < n; ++i) {
    const int32_t tt = pairs[2 * i];
    if (tt < 0 || tt >= ncells) return ORC_ERR_ALLOC;
    ++offsets[tt + 1];
  }
  for (int64_t c = 0; c < ncells; ++c) offsets[c + 1] += offsets[c];
  int64_t* fill = malloc(sizeof(int64_t) * (size_t)(ncells > 0 ? ncells : 1));
  if (!fill) return ORC_ERR_ALLOC;
  memcpy(fill, offsets, sizeof(int64_t) * (size_t)ncells);
  for (int64_t i = 0; i < n; ++i) sources[fill[pairs[2 * i]]++] = pairs[2 * i + 1];
  free(fill);
  if (sort_sources) {
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t c = 0; c < ncells; ++c) { /* insertion sort: lists are short or nearly sorted */
      int32_t* s = sources + offsets[c];
      const int64_t k = offsets[c + 1] - offsets[c];
      for (int64_t i = 1; i < k; ++i) {
        const int32_t v = s[i];
        int64_t j = i - 1;
        while (j >= 0 && s[j] > v) { s[j + 1] = s[j]; --j; }
        s[j + 1] = v;
      }
    }
  }
  return ORC_OK;
}

int orc_evaluate_par(orc_tree* t, double theta, int with_acc, const uint8_t* cell_mask,
                     uint64_t* p2p_evals, int64_t* n_m2l_out, int64_t* n_p2p_out) {
  orc_tables kt;
  int rc = orc_tables_init(&kt, t->order);
  if (rc) return rc;
  const int nc = kt.n;
  int64_t lb[ORC_MAX_TREE_LEVEL + 2];
  int nlev = 0;
  if (orc_level_ranges(t, lb, &nlev)) {
    orc_tables_free(&kt);
    return ORC_ERR_ALLOC;
  }
  uint8_t* active = malloc((size_t)t->ncells);
  if (!active) { orc_tables_free(&kt); return ORC_ERR_ALLOC; }
  if (cell_mask) {
    memset(active, 0, (size_t)t->ncells);
    for (int64_t ci = t->ncells - 1; ci >= 0; --ci) /* children follow parents */
      if (cell_mask[ci] || active[ci]) {
        active[ci] = 1;
        if (t->cells[ci].parent >= 0) active[t->cells[ci].parent] = 1;
      }
  } else {
    memset(active, 1, (size_t)t->ncells);
  }
  /* upward (traversal.cpp:36-50), every cell: sources may be anywhere */
  for (int L = nlev - 1; L >= 0; --L) {
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t ci = lb[L]; ci < lb[L + 1]; ++ci) {
      const orc_cell* c = &t->cells[ci];
      double* M = t->multipole + ci * nc;
      if (c->child_count == 0) {
        orc_p2m(&kt, c->body_end - c->body_begin, t->pos + 3 * (int64_t)c->body_begin,
                t->q + c->body_begin, c->center, M);
      } else {
        for (int32_t k = 0; k < c->child_count; ++k) {
          const orc_cell* ch = &t->cells[c->child_begin + k];
          const double shift[3] = {ch->center[0] - c->center[0], ch->center[1] - c->center[1],
                                   ch->center[2] - c->center[2]};
          orc_m2m(&kt, t->multipole + (int64_t)(c->child_begin + k) * nc, shift, M);
        }
      }
    }
  }
  int64_t nm = 0, np = 0;
  int32_t *m2l = NULL, *p2p = NULL;
  rc = orc_traverse(t, theta, 0, &nm, &m2l, &np, &p2p);
  int64_t *mo = NULL, *po = NULL;
  int32_t *ms = NULL, *ps = NULL;
  if (!rc) {
    mo = malloc(sizeof(int64_t) * (size_t)(t->ncells + 1));
    po = malloc(sizeof(int64_t) * (size_t)(t->ncells + 1));
    ms = malloc(sizeof(int32_t) * (size_t)(nm > 0 ? nm : 1));
    ps = malloc(sizeof(int32_t) * (size_t)(np > 0 ? np : 1));
    if (!mo || !po || !ms || !ps) rc = ORC_ERR_ALLOC;
  }
  if (!rc) rc = orc_group_by_target(t->ncells, nm, m2l, mo, ms, 0);
  if (!rc) rc = orc_group_by_target(t->ncells, np, p2p, po, ps, 0);
  free(m2l);
  free(p2p);
  uint64_t ev = 0;
  int err = 0;
  if (!rc) {
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : ev)
    for (int64_t ci = 0; ci < t->ncells; ++ci) {
      if (!active[ci]) continue;
      for (int64_t k = mo[ci]; k < mo[ci + 1]; ++k)
        if (apply_m2l(t, &kt, (int32_t)ci, ms[k], 0)) {
#pragma omp atomic write
          err = ORC_ERR_SINGULAR_M2L;
        }
      for (int64_t k = po[ci]; k < po[ci + 1]; ++k) ev += apply_p2p(t, (int32_t)ci, ps[k], 0, with_acc);
    }
    rc = err;
  }
  free(mo); free(po); free(ms); free(ps);
  if (!rc) {
    double* acc_save = t->acc;
    if (!with_acc) t->acc = NULL;
    for (int L = 0; L < nlev; ++L) { /* downward (traversal.cpp:52-63) */
#pragma omp parallel for schedule(dynamic, 16)
      for (int64_t ci = lb[L]; ci < lb[L + 1]; ++ci) {
        if (!active[ci]) continue;
        const orc_cell* c = &t->cells[ci];
        if (c->parent >= 0) {
          const orc_cell* pc = &t->cells[c->parent];
          const double shift[3] = {c->center[0] - pc->center[0], c->center[1] - pc->center[1],
                                   c->center[2] - pc->center[2]};
          orc_l2l(&kt, t->local + (int64_t)c->parent * nc, shift, t->local + ci * nc);
        }
        if (c->child_count == 0)
          orc_l2p(&kt, t->local + ci * nc, c->center, c->body_end - c->body_begin,
                  t->pos + 3 * (int64_t)c->body_begin, t->phi + c->body_begin,
                  t->acc ? t->acc + 3 * (int64_t)c->body_begin : NULL);
      }
    }
    t->acc = acc_save;
  }
  free(active);
  orc_tables_free(&kt);
  if (p2p_evals) *p2p_evals = ev;
  if (n_m2l_out) *n_m2l_out = nm;
  if (n_p2p_out) *n_p2p_out = np;
  return rc;
}

/* Direct sum over a subset of targets (oracle.cpp:8-23 + acc), all N sources, parallel over
 * targets; idx are input-order indices, outputs are per listed target. */
void orc_direct_sum_targets(int64_t n, const double* pos, const double* q, int64_t nt,
                            const int64_t* idx, double* phi, double* acc) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t k = 0; k < nt; ++k) {
    const int64_t i = idx[k];
    long double s = 0.0L, ax = 0.0L, ay = 0.0L, az = 0.0L;
    for (int64_t j = 0; j < n; ++j) {
      if (j == i) continue;
      const double dx = pos[3 * i] - pos[3 * j], dy = pos[3 * i + 1] - pos[3 * j + 1],
                   dz = pos[3 * i + 2] - pos[3 * j + 2];
      const double r2 = (dx * dx + dy * dy) + dz * dz;
      if (r2 == 0.0) continue;
      const long double inv_r = 1.0L / sqrtl((long double)r2);
      s += (long double)q[j] * inv_r;
      const long double w = (long double)q[j] * inv_r * inv_r * inv_r;
      ax += w * (long double)dx;
      ay += w * (long double)dy;
      az += w * (long double)dz;
    }
    phi[k] = (double)s;
    if (acc) {
      acc[3 * k] = (double)ax;
      acc[3 * k + 1] = (double)ay;
      acc[3 * k + 2] = (double)az;
    }
  }
}

/* BASELINE.json configs 1..5, an independent restatement for the checker and
 * the reference arm: the reference's xorshift64* (dataset.cpp:10-34), seed per config, per body
 * the position (Vec3(u(),u(),u()) evaluated right to left by g++: z first) then the charge.
 *   1, 2, 4  uniform [-1,1]^3, q = (1 - u01)/N in (0, 1/N]
 *   3        Plummer: r = 1/sqrt(U^(-2/3) - 1), resampled while r > 100 or not finite;
 *            direction by cube rejection (s > 1 or s < 1e-8 rejected); q = 1/N
 *   5        unit sphere surface: Box-Muller sqrt(-2 ln(1-u1)) cos(2 pi u2) per axis (z first),
 *            normalised; q = uniform(-1,1)/N */
int orc_generate_baseline_bodies(int config, int64_t n, uint64_t seed, double* xyzq) {
  if (n < 1) return ORC_ERR_EMPTY_INPUT;
  if (config < 1 || config > 5) return ORC_ERR_ALLOC;
  orc_rng r;
  orc_rng_init(&r, seed);
  const double dn = (double)n;
  const double two_pi = 6.283185307179586;
  for (int64_t i = 0; i < n; ++i) {
    double* b = xyzq + 4 * i;
    if (config == 3) {
      double rad;
      do {
        const double U = orc_rng_uniform01(&r);
        rad = 1.0 / sqrt(pow(U, -2.0 / 3.0) - 1.0);
      } while (!(rad <= 100.0) || !isfinite(rad));
      double v[3], s;
      do {
        v[2] = orc_rng_uniform(&r, -1.0, 1.0);
        v[1] = orc_rng_uniform(&r, -1.0, 1.0);
        v[0] = orc_rng_uniform(&r, -1.0, 1.0);
        s = (v[0] * v[0] + v[1] * v[1]) + v[2] * v[2];
      } while (s > 1.0 || s < 1e-8);
      const double inv = rad / sqrt(s);
      b[0] = v[0] * inv;
      b[1] = v[1] * inv;
      b[2] = v[2] * inv;
      b[3] = 1.0 / dn;
    } else if (config == 5) {
      double v[3], s;
      do {
        for (int d = 2; d >= 0; --d) {
          const double u1 = orc_rng_uniform01(&r), u2 = orc_rng_uniform01(&r);
          v[d] = sqrt(-2.0 * log(1.0 - u1)) * cos(two_pi * u2);
        }
        s = (v[0] * v[0] + v[1] * v[1]) + v[2] * v[2];
      } while (s == 0.0);
      const double inv = 1.0 / sqrt(s);
      b[0] = v[0] * inv;
      b[1] = v[1] * inv;
      b[2] = v[2] * inv;
      b[3] = orc_rng_uniform(&r, -1.0, 1.0) / dn;
    } else {
      b[2] = orc_rng_uniform(&r, -1.0, 1.0);
      b[1] = orc_rng_uniform(&r, -1.0, 1.0);
      b[0] = orc_rng_uniform(&r, -1.0, 1.0);
      b[3] = (1.0 - orc_rng_uniform01(&r)) / dn;
    }
  }
  return ORC_OK;
}
