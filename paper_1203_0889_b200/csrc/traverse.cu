// traverse.cu — dual tree traversal on the GPU emitting the reference's M2L / P2P lists
// bit-exactly (reference: mac, traversal.cpp:8-13; split_target_side / process_pair,
// traversal.hpp:49-94; dual_tree_traverse, traversal.hpp:118-133).
//
// The reference's emitted multiset is a pure function of (tree, theta, mutual) and is
// independent of queue order and of the drain threshold Q (acceptance.cpp:99-123). The GPU
// therefore replaces the FIFO queue by level-synchronous frontier expansion: every pair of
// the frontier is examined by one thread (process_pair), emits an M2L or P2P pair or pushes
// its child pairs to the next frontier. Output slots come from exclusive scans, so the
// emission order is deterministic. The lists are then grouped into CSR by target with a
// radix sort on (target, source), i.e. ascending sources within each target.
// The MAC is evaluated with __dmul_rn/__dadd_rn/__dsqrt_rn: no FMA contraction, exactly
// std::sqrt(3.0)*(rt+rs) < theta*sqrt((dx*dx+dy*dy)+dz*dz).
#include <cub/cub.cuh>

#include "context.cuh"

namespace fmmb {
namespace {

constexpr double kSqrt3 = 1.7320508075688772;  // std::sqrt(3.0), correctly rounded

__device__ __forceinline__ bool mac_exact(const double4 t, const double4 s, double theta) {
  const double sum_r = __dmul_rn(kSqrt3, __dadd_rn(t.w, s.w));
  const double dx = __dadd_rn(t.x, -s.x), dy = __dadd_rn(t.y, -s.y), dz = __dadd_rn(t.z, -s.z);
  const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  return sum_r < __dmul_rn(theta, __dsqrt_rn(d2));
}

// Outcome of process_pair: kind 0 = M2L, 1 = P2P, 2 = split target, 3 = split source,
// 4 = mutual self split. nchild = number of pushed pairs.
__device__ __forceinline__ void classify(const int2 pr, const double4* __restrict__ cr,
                                         const int32_t* __restrict__ cc, double theta, int mutual,
                                         int& kind, int& nchild) {
  const double4 t = cr[pr.x], s = cr[pr.y];
  const int tc = cc[pr.x], sc = cc[pr.y];
  if (mac_exact(t, s, theta)) { kind = 0; nchild = 0; return; }
  if (tc == 0 && sc == 0) { kind = 1; nchild = 0; return; }
  if (mutual && pr.x == pr.y) { kind = 4; nchild = tc * (tc + 1) / 2; return; }
  bool split_t;
  if (tc == 0) split_t = false;            // traversal.hpp:53-57
  else if (sc == 0) split_t = true;
  else if (t.w != s.w) split_t = t.w > s.w;
  else split_t = pr.x <= pr.y;
  kind = split_t ? 2 : 3;
  nchild = split_t ? tc : sc;
}

struct Cnt {  // per-pair output counts; one exclusive scan gives all three offsets
  long long m2l, p2p, push;
};
struct CntSum {
  __host__ __device__ __forceinline__ Cnt operator()(const Cnt& a, const Cnt& b) const {
    return Cnt{a.m2l + b.m2l, a.p2p + b.p2p, a.push + b.push};
  }
};

__global__ void k_classify(const int2* __restrict__ fr, int64_t n, const double4* __restrict__ cr,
                           const int32_t* __restrict__ cc, double theta, int mutual,
                           uint8_t* __restrict__ kinds, Cnt* __restrict__ cnt) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > n) return;
  if (i == n) {  // trailing element: the exclusive scan's last entry is the total
    cnt[i] = Cnt{0, 0, 0};
    return;
  }
  int kind, nchild;
  classify(fr[i], cr, cc, theta, mutual, kind, nchild);
  kinds[i] = static_cast<uint8_t>(kind);
  cnt[i] = Cnt{kind == 0, kind == 1, nchild};
}

__global__ void k_expand(const int2* __restrict__ fr, int64_t n, const uint8_t* __restrict__ kinds,
                         const int32_t* __restrict__ cc, const int32_t* __restrict__ cb,
                         const Cnt* __restrict__ off, int2* __restrict__ m2l, int64_t m2l_base,
                         int2* __restrict__ p2p, int64_t p2p_base, int2* __restrict__ next) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int2 pr = fr[i];
  const int kind = kinds[i];
  const Cnt o = off[i];
  if (kind == 0) { m2l[m2l_base + o.m2l] = pr; return; }
  if (kind == 1) { p2p[p2p_base + o.p2p] = pr; return; }
  int64_t q = o.push;
  if (kind == 2) {
    const int32_t b = cb[pr.x], m = cc[pr.x];
    for (int k = 0; k < m; ++k) next[q + k] = make_int2(b + k, pr.y);
  } else if (kind == 3) {
    const int32_t b = cb[pr.y], m = cc[pr.y];
    for (int k = 0; k < m; ++k) next[q + k] = make_int2(pr.x, b + k);
  } else {
    const int32_t b = cb[pr.x], m = cc[pr.x];
    for (int a = 0; a < m; ++a)
      for (int c = a; c < m; ++c) next[q++] = make_int2(b + a, b + c);
  }
}

__global__ void k_split_pairs(const int2* __restrict__ pr, int64_t n, uint32_t* __restrict__ t,
                              int32_t* __restrict__ s) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    const int2 v = pr[i];
    t[i] = static_cast<uint32_t>(v.x);
    s[i] = v.y;
  }
}

// offsets from the target-sorted key array: targets tp+1..t start at i
__global__ void k_csr_offsets(const uint32_t* __restrict__ t_sorted, int64_t n, int64_t ncells,
                              int64_t* __restrict__ off) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > n) return;
  const int64_t t = i < n ? (int64_t)t_sorted[i] : ncells;
  const int64_t tp = i > 0 ? (int64_t)t_sorted[i - 1] : -1;
  for (int64_t c = tp + 1; c <= t; ++c) off[c] = i;
}

__global__ void k_p2p_body_pairs(const int64_t* __restrict__ off, const int32_t* __restrict__ src,
                                 int64_t ncells, const int32_t* __restrict__ bb, const int32_t* __restrict__ be,
                                 unsigned long long* __restrict__ total) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  unsigned long long v = 0;
  if (t < ncells) {
    const int64_t nt = be[t] - bb[t];
    for (int64_t k = off[t]; k < off[t + 1]; ++k) v += (unsigned long long)(nt * (be[src[k]] - bb[src[k]]));
  }
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(total, v);
}

__global__ void k_flag_nonempty(const int64_t* __restrict__ off, int64_t ncells, int32_t* __restrict__ flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < ncells) flag[i] = off[i + 1] > off[i];
}

int bits_for(uint64_t v) {
  int b = 1;
  while (b < 63 && (v >> b)) ++b;
  return b;
}

template <class T>
void grow_keep(fmm_ctx* c, DBuf<T>& buf, size_t used, size_t need) {
  if (need <= buf.cap) return;
  T* fresh = nullptr;
  const size_t want = need + need / 2 + 1024;
  CK(cudaMalloc(&fresh, want * sizeof(T)));
  if (buf.p && used) CK(cudaMemcpyAsync(fresh, buf.p, used * sizeof(T), cudaMemcpyDeviceToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (buf.p) CK(cudaFree(buf.p));
  buf.p = fresh;
  buf.cap = want;
}

// Groups (target, source) pairs into CSR by target: a stable radix sort on the target index
// only (ceil(log2 ncells) bits), so sources keep the traversal's deterministic emission order.
void to_csr(fmm_ctx* c, const int2* d_pairs, int64_t n, DBuf<int64_t>& off, DBuf<int32_t>& src) {
  cudaStream_t s = c->stream;
  const int64_t nc = c->ncells;
  off.ensure(nc + 1);
  src.ensure(n > 0 ? n : 1);
  if (n == 0) {
    CK(cudaMemsetAsync(off.p, 0, sizeof(int64_t) * (nc + 1), s));
    return;
  }
  const int tbits = bits_for(static_cast<uint64_t>(nc));
  uint32_t* ta = reinterpret_cast<uint32_t*>(c->keys_a.ensure((n + 1) / 2 + 1));
  uint32_t* tb = reinterpret_cast<uint32_t*>(c->keys_b.ensure((n + 1) / 2 + 1));
  int32_t* sa = c->i32_c.ensure(n);
  k_split_pairs<<<ceil_div(n, 256), 256, 0, s>>>(d_pairs, n, ta, sa);
  size_t sb = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, sb, ta, tb, sa, src.p, (int)n, 0, tbits, s));
  CK(cub::DeviceRadixSort::SortPairs(temp_storage(c, sb), sb, ta, tb, sa, src.p, (int)n, 0, tbits, s));
  k_csr_offsets<<<ceil_div(n + 1, 256), 256, 0, s>>>(tb, n, nc, off.p);
  CK_LAUNCH("to_csr");
  c->kernel_launches += 4;
}

}  // namespace

void lists_from_pairs(fmm_ctx* c, const int2* d_m2l, int64_t n_m2l, const int2* d_p2p, int64_t n_p2p) {
  cudaStream_t s = c->stream;
  to_csr(c, d_m2l, n_m2l, c->m2l_off, c->m2l_src);
  to_csr(c, d_p2p, n_p2p, c->p2p_off, c->p2p_src);
  c->n_m2l = n_m2l;
  c->n_p2p = n_p2p;
  // body-pair count (P2P work) and the M2L target list
  unsigned long long* tot = reinterpret_cast<unsigned long long*>(c->d_counters.ensure(4));
  CK(cudaMemsetAsync(tot, 0, sizeof(unsigned long long), s));
  k_p2p_body_pairs<<<ceil_div(c->ncells, 256), 256, 0, s>>>(c->p2p_off.p, c->p2p_src.p, c->ncells,
                                                            c->c_body_begin.p, c->c_body_end.p, tot);
  int32_t* flag = c->i32_c.ensure(c->ncells);
  k_flag_nonempty<<<ceil_div(c->ncells, 256), 256, 0, s>>>(c->m2l_off.p, c->ncells, flag);
  CK_LAUNCH("k_flag_nonempty");
  int32_t* targets = c->m2l_targets.ensure(c->ncells);
  int64_t* nsel = c->d_counters.p + 1;
  size_t sb = 0;
  cub::CountingInputIterator<int32_t> it(0);
  CK(cub::DeviceSelect::Flagged(nullptr, sb, it, flag, targets, nsel, (int)c->ncells, s));
  CK(cub::DeviceSelect::Flagged(temp_storage(c, sb), sb, it, flag, targets, nsel, (int)c->ncells, s));
  int64_t* h = c->hpin;
  CK(cudaMemcpyAsync(h, c->d_counters.p, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  c->p2p_body_pairs = h[0];
  c->n_m2l_targets = h[1];
  c->kernel_launches += 3;
  c->have_lists = true;
  build_p2p_worklist(c);
}

void traverse(fmm_ctx* c) {
  if (!c->have_tree) fail(FMM_ERR_STATE, "traverse: no tree");
  const double theta = c->cfg.theta;
  if (!(theta > 0.0 && theta < 1.0)) fail(FMM_ERR_THETA, "theta must be in (0,1)");
  cudaStream_t s = c->stream;
  const int mutual = c->cfg.mutual ? 1 : 0;

  int64_t nf = 1, nm = 0, np = 0;
  const int2 root = make_int2(0, 0);
  DBuf<int2>* fa = &c->pairs_a;
  DBuf<int2>* fb = &c->pairs_d;
  DBuf<int2>* m2l = &c->pairs_b;
  DBuf<int2>* p2p = &c->pairs_c;
  fa->ensure(1024);
  fb->ensure(1024);
  m2l->ensure(1024);
  p2p->ensure(1024);
  CK(cudaMemcpyAsync(fa->p, &root, sizeof(int2), cudaMemcpyHostToDevice, s));
  Cnt* hcnt = reinterpret_cast<Cnt*>(c->hpin);
  int launches = 0;
  while (nf > 0) {
    Cnt* cnt = reinterpret_cast<Cnt*>(c->scan_a.ensure(3 * (nf + 1) * 2));
    Cnt* off = cnt + (nf + 1);
    uint8_t* kinds = reinterpret_cast<uint8_t*>(c->keys_a.ensure(nf / 8 + 2));
    k_classify<<<ceil_div(nf + 1, 256), 256, 0, s>>>(fa->p, nf, c->c_cr.p, c->c_child_count.p, theta, mutual,
                                                     kinds, cnt);
    CK_LAUNCH("k_classify");
    size_t sb = 0;
    CK(cub::DeviceScan::ExclusiveScan(nullptr, sb, cnt, off, CntSum(), Cnt{0, 0, 0}, (int)(nf + 1), s));
    CK(cub::DeviceScan::ExclusiveScan(temp_storage(c, sb), sb, cnt, off, CntSum(), Cnt{0, 0, 0}, (int)(nf + 1), s));
    CK(cudaMemcpyAsync(hcnt, off + nf, sizeof(Cnt), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const int64_t add_m = hcnt->m2l, add_p = hcnt->p2p, nnext = hcnt->push;
    grow_keep(c, *m2l, nm, nm + add_m);
    grow_keep(c, *p2p, np, np + add_p);
    fb->ensure(nnext > 0 ? nnext : 1);
    k_expand<<<ceil_div(nf, 256), 256, 0, s>>>(fa->p, nf, kinds, c->c_child_count.p, c->c_child_begin.p, off,
                                               m2l->p, nm, p2p->p, np, fb->p);
    CK_LAUNCH("k_expand");
    launches += 3;
    nm += add_m;
    np += add_p;
    nf = nnext;
    std::swap(fa, fb);
  }
  c->kernel_launches += launches;
  lists_from_pairs(c, m2l->p, nm, p2p->p, np);
}

}  // namespace fmmb

namespace fmmb {
namespace {
__global__ void k_op_mac(int64_t count, const double* __restrict__ tc, const double* __restrict__ tr,
                         const double* __restrict__ sc, const double* __restrict__ sr, double theta,
                         int32_t* __restrict__ out) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= count) return;
  out[k] = mac_exact(make_double4(tc[3 * k], tc[3 * k + 1], tc[3 * k + 2], tr[k]),
                     make_double4(sc[3 * k], sc[3 * k + 1], sc[3 * k + 2], sr[k]), theta) ? 1 : 0;
}
}  // namespace

void op_mac(int64_t count, const double* tc3, const double* tr, const double* sc3, const double* sr,
            double theta, int32_t* out) {
  if (count <= 0) return;
  double* d = nullptr;
  int32_t* o = nullptr;
  CK(cudaMalloc(&d, count * 8 * sizeof(double)));
  CK(cudaMalloc(&o, count * sizeof(int32_t)));
  CK(cudaMemcpy(d, tc3, count * 3 * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d + 3 * count, tr, count * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d + 4 * count, sc3, count * 3 * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d + 7 * count, sr, count * sizeof(double), cudaMemcpyHostToDevice));
  k_op_mac<<<ceil_div(count, 128), 128>>>(count, d, d + 3 * count, d + 4 * count, d + 7 * count, theta, o);
  CK_LAUNCH("op_mac");
  CK(cudaMemcpy(out, o, count * sizeof(int32_t), cudaMemcpyDeviceToHost));
  cudaFree(d);
  cudaFree(o);
}
}  // namespace fmmb
