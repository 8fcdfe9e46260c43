// p2p.cu — near-field P2P on sm_100a (reference: p2p non-mutual, kernels.cpp:181-192,
// applied by KernelVisitor::p2p_pair, traversal.hpp:154-157) plus its acceleration extension.
//
// Work decomposition (replaces the QUARK task DAG): one CTA per work item =
// (target leaf, target sub-range <= 128 bodies, contiguous chunk of its P2P source list).
// Items are cost-sorted (n_t * sum n_s, descending) so the longest start first; lists whose
// cost exceeds a per-SM share are split into source chunks whose partial sums are reduced in
// a fixed order afterwards (deterministic, no atomics). Writes are target-owned.
//
// Inside a CTA four consumer warps (128 threads) form G = floor(128 / ceil(n_t / 2)) lane groups;
// thread (g, t) owns the target pair (2t, 2t+1) packed in f32x2 lanes and a contiguous chunk of
// each shared-memory tile; a fifth (producer) warp stages the tiles (k_p2p_fp32_ws). Tiles hold
// up to 64 list entries (1 024 bodies) converted to coordinates relative to the TARGET leaf
// centre: bodies are stored in HBM as FP32 offsets from their own leaf centre and shifted by
// the FP64-computed centre difference, so FP32 only ever sees leaf-scale magnitudes; the inner
// loop runs on the packed f32x2 pipe (FFMA2/FADD2/FMUL2) with one MUFU.RSQ per pair; r^2 == 0
// pairs (self, coincident; kernels.cpp:185-186) are removed by a predicate in the self tile.
// Each tile's FP32 partial sums are folded into FP64 per-target accumulators ("FP64-checked
// accumulation").
#include <cub/cub.cuh>

#include "context.cuh"
#include "tma.cuh"

namespace fmmb {
namespace {

constexpr int kThreads = 128;   // threads per P2P CTA (max target bodies per item)
constexpr int kTileSegs = 64;   // list entries per FP32 tile (two per producer lane)
#ifndef FMM_P2P_TILE
#define FMM_P2P_TILE 1024
#endif
constexpr int kTileBodies = FMM_P2P_TILE;

struct P2PItem {
  int32_t leaf, tb, te, lb, le;  // target leaf, target body range, list range [lb, le)
  int32_t pbase;                 // partial-buffer base (in bodies) or -1 for a direct write
  int32_t sb0;                   // body offset into the first list entry (always 0 here)
  int32_t pad;
};
static_assert(sizeof(P2PItem) == 32, "P2PItem is 32 B");

// Tile setup (warp 0): takes the next list entries whose bodies fit in TILE slots, starting
// at (cursor, cur_off). A single source leaf larger than the tile (only possible for level-21
// overflow leaves) is consumed TILE bodies at a time. Results: seg_off[0..nseg], seg_src,
// seg_boff (body offset inside each entry), nxt[0] = next cursor, nxt[1] = next offset.
template <int TILE>
__device__ __forceinline__ void tile_setup(int tid, int32_t le, int32_t cursor, int32_t cur_off,
                                           const int32_t* __restrict__ src_list, const int32_t* __restrict__ bb,
                                           const int32_t* __restrict__ be, int32_t* seg_off, int32_t* seg_src,
                                           int32_t* seg_boff, int32_t* nxt) {
  if (tid >= 32) return;
  const int32_t k = cursor + tid;
  int32_t n = 0, s = -1, boff = 0;
  if (k < le) {
    s = src_list[k];
    FMM_CHECK(s >= 0 && s < FMM_LIM(ncells), "p2p (fp64) tile: source cell index");
    n = be[s] - bb[s];
    if (tid == 0) {
      boff = cur_off;
      n -= cur_off;
    }
  }
  int32_t incl = n;
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (tid >= o) incl += v;
  }
  const bool fits = (k < le) && (incl <= TILE);
  const unsigned m = __ballot_sync(0xffffffffu, fits);
  if (m == 0) {  // the first entry alone overflows the tile: take TILE of its bodies
    if (tid == 0) {
      seg_off[0] = 0;
      seg_off[1] = TILE;
      seg_src[0] = s;
      seg_boff[0] = boff;
      nxt[0] = cursor;
      nxt[1] = cur_off + TILE;
      nxt[2] = 1;
    }
    return;
  }
  const int nseg = 32 - __clz(m);  // fits is a prefix of the lanes
  if (tid < nseg) {
    seg_off[tid + 1] = incl;
    seg_src[tid] = s;
    seg_boff[tid] = boff;
  }
  if (tid == 0) {
    seg_off[0] = 0;
    nxt[0] = cursor + nseg;
    nxt[1] = 0;
    nxt[2] = nseg;
  }
}

// One P2P list entry (target specific): source bodies and the FP64 centre difference into the
// target leaf frame as an FP32 hi + lo pair. kind (top two bits of nk): 0 = far, 1 = the
// (leaf, leaf) self entry (the only one that can hold r^2 == 0 pairs), 2 = near (the two
// leaves' body boxes nearly touch: the only entries whose body pairs can be close relative to
// the leaf size). Self and near entries run compensated tiles.
struct P2PEnt {
  int32_t bb, nk;         // first source body; count | kind << 30
  float sx, sy, sz;       // shift hi
  float lx, ly, lz;       // shift lo
};
static_assert(sizeof(P2PEnt) == 32, "P2PEnt is 32 B");
constexpr int kKindFar = 0, kKindSelf = 1, kKindNear = 2;

struct TileTab {
  int32_t off[kTileSegs + 1];
  int32_t bb[kTileSegs];
  float sh[kTileSegs][3];
  float sl[kTileSegs][3];
  int32_t nseg, next, next_off, guard, prec;
};

// producer warp: take the list entries from (cursor, cur_off) that fit in one tile; e[i] is list
// entry cursor + i, lane l holds entries l and l + 32 (small leaves, e.g. C5's median of 18
// bodies, fill a 1 024-body tile only with ~60 entries)
template <int TB>
__device__ __forceinline__ void tile_setup_ent(int lane, int32_t le, int32_t cursor, int32_t cur_off,
                                               const P2PEnt* e, TileTab& tt) {
  constexpr int H = kTileSegs / 32;
  int32_t n[H], b[H], kind[H], incl[H];
  float sh[H][3], sl[H][3];
  bool valid[H];
#pragma unroll
  for (int h = 0; h < H; ++h) {
    const int32_t k = cursor + h * 32 + lane;
    valid[h] = k < le;
    n[h] = 0;
    b[h] = 0;
    kind[h] = kKindFar;
    sh[h][0] = sh[h][1] = sh[h][2] = sl[h][0] = sl[h][1] = sl[h][2] = 0.f;
    if (valid[h]) {
      const int4 e0 = reinterpret_cast<const int4*>(e)[2 * (h * 32 + lane)];
      const int4 e1 = reinterpret_cast<const int4*>(e)[2 * (h * 32 + lane) + 1];
      b[h] = e0.x;
      n[h] = e0.y & 0x3fffffff;
      FMM_CHECK(b[h] >= 0 && n[h] > 0 && b[h] + n[h] <= FMM_LIM(nbodies), "p2p tile: entry body range");
      kind[h] = static_cast<int>(static_cast<uint32_t>(e0.y) >> 30);
      sh[h][0] = __int_as_float(e0.z);
      sh[h][1] = __int_as_float(e0.w);
      sh[h][2] = __int_as_float(e1.x);
      sl[h][0] = __int_as_float(e1.y);
      sl[h][1] = __int_as_float(e1.z);
      sl[h][2] = __int_as_float(e1.w);
      if (h == 0 && lane == 0) {
        b[h] += cur_off;
        n[h] -= cur_off;
      }
    }
  }
  // one class per tile: the self entry alone (r^2 == 0 guard), near entries (compensated, half
  // the bodies: hi and lo staged), far entries (plain FP32)
  const int kind0 = __shfl_sync(0xffffffffu, kind[0], 0);
  const int cap = kind0 == kKindFar ? TB : TB / 2;
  int32_t running = 0;
  unsigned m[H], other[H];
#pragma unroll
  for (int h = 0; h < H; ++h) {
    incl[h] = n[h];
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t v = __shfl_up_sync(0xffffffffu, incl[h], o);
      if (lane >= o) incl[h] += v;
    }
    incl[h] += running;
    running = __shfl_sync(0xffffffffu, incl[h], 31);
    m[h] = __ballot_sync(0xffffffffu, valid[h] && incl[h] <= cap);
    // classes: far | compensated (near and self share tiles; the self entry comes last)
    other[h] = __ballot_sync(0xffffffffu, valid[h] && (kind[h] == kKindFar) != (kind0 == kKindFar));
  }
  int nseg = 0;  // the fitting entries are a prefix of the 64
#pragma unroll
  for (int h = 0; h < H; ++h) {
    if (nseg == 32 * h) nseg += 32 - __clz(m[h]);
  }
  const bool huge = m[0] == 0;  // one (level-21 overflow) leaf larger than the tile: take cap of it
  if (huge) {
    nseg = 1;
    incl[0] = cap;
  }
  int first_other = kTileSegs;
#pragma unroll
  for (int h = H - 1; h >= 0; --h)
    if (other[h]) first_other = 32 * h + __ffs(other[h]) - 1;
  nseg = min(nseg, first_other);
  // the r^2 == 0 guard is needed iff the tile holds the self entry
  unsigned selfm = 0;
#pragma unroll
  for (int h = 0; h < H; ++h)
    selfm |= __ballot_sync(0xffffffffu, valid[h] && kind[h] == kKindSelf && h * 32 + lane < nseg);
#pragma unroll
  for (int h = 0; h < H; ++h) {
    const int idx = h * 32 + lane;
    if (idx < nseg) {
      tt.off[idx + 1] = incl[h];
      tt.bb[idx] = b[h];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        tt.sh[idx][d] = sh[h][d];
        tt.sl[idx][d] = sl[h][d];
      }
    }
  }
  if (lane == 0) {
    tt.off[0] = 0;
    tt.nseg = nseg;
    tt.next = huge ? cursor : cursor + nseg;
    tt.next_off = huge ? cur_off + cap : 0;
    tt.guard = selfm ? 1 : 0;
    tt.prec = kind0 == kKindFar ? 0 : 1;
  }
}

// producer warp: one bulk copy per list entry of the tile (lane k copies entries k, k + 32);
// the bytes land on `bar`. The proxy fence orders earlier generic reads/writes of the buffer
// (released to the producer through the empty barrier) before the async-proxy writes.
template <int TB>
__device__ __forceinline__ void tile_tma(int lane, const TileTab& tt, const float4* __restrict__ bodyf,
                                         const float4* __restrict__ bodyl, float4* buf, uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  const int nseg = tt.nseg;
  const bool prec = tt.prec != 0;
  if (lane == 0) mbar_arrive_expect_tx(bar, static_cast<unsigned>(tt.off[nseg]) * (prec ? 32u : 16u));
  for (int idx = lane; idx < nseg; idx += 32) {
    const int32_t o0 = tt.off[idx];
    FMM_CHECK(o0 >= 0 && tt.off[idx + 1] > o0 && tt.off[idx + 1] <= (prec ? TB / 2 : TB),
              "p2p tile: staged bodies beyond the tile buffer");
    const unsigned bytes = static_cast<unsigned>(tt.off[idx + 1] - o0) * 16u;
    bulk_g2s(buf + o0, bodyf + tt.bb[idx], bytes, bar);
    if (prec) bulk_g2s(buf + TB / 2 + o0, bodyl + tt.bb[idx], bytes, bar);
  }
}

// Compensated tiles: (x - c_s) + (c_s - c_t) = (hi_b + lo_b) + (S_hi + S_lo) with hi_b + S_hi
// split exactly by TwoSum; stored negated as hi at [o], lo at [half + o]. A close pair's
// difference then keeps ~48 bits instead of an absolute error of the leaf size * 2^-24.
__device__ __forceinline__ float2 two_sum(float a, float b) {
  const float s = __fadd_rn(a, b);
  const float bb = __fsub_rn(s, a);
  const float e = __fadd_rn(__fsub_rn(a, __fsub_rn(s, bb)), __fsub_rn(b, bb));
  return make_float2(s, e);
}

__device__ __forceinline__ float rsqrt_approx(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// One source against the thread's two targets: 13 FP32-pipe lane-ops per pair (3 dx, 3 r^2,
// q/r, phi, 1/r^2, q/r^3, 3 acc) and one MUFU.RSQ (XU pipe: 16/clk/SM, so a second MUFU per
// pair would make the XU the bottleneck). kGuard (the self tile only): r^2 == 0 pairs (self,
// coincident; kernels.cpp:185-186) are predicated off. Otherwise the bodies are distinct and
// r^2 is seeded with 1e-30 instead of predicating the MUFU, which keeps the result finite even
// if two distinct bodies round to the same FP32 offsets, at no instruction cost.
template <bool kAcc, bool kGuard>
__device__ __forceinline__ void pair_finish(const float2 dx, const float2 dy, const float2 dz, const float q,
                                            float2& ph, float2& ax, float2& ay, float2& az) {
  float2 r2 = kGuard ? __fmul2_rn(dx, dx) : __ffma2_rn(dx, dx, make_float2(1e-30f, 1e-30f));
  r2 = __ffma2_rn(dy, dy, r2);
  r2 = __ffma2_rn(dz, dz, r2);
  float2 ri;
  if constexpr (kGuard) {
    ri = make_float2(0.f, 0.f);
    if (r2.x > 0.f) ri.x = rsqrt_approx(r2.x);
    if (r2.y > 0.f) ri.y = rsqrt_approx(r2.y);
  } else {
    ri = make_float2(rsqrt_approx(r2.x), rsqrt_approx(r2.y));
  }
  const float2 qr = __fmul2_rn(make_float2(q, q), ri);
  ph = __fadd2_rn(ph, qr);
  if constexpr (kAcc) {
    const float2 qr3 = __fmul2_rn(qr, __fmul2_rn(ri, ri));
    ax = __ffma2_rn(dx, qr3, ax);
    ay = __ffma2_rn(dy, qr3, ay);
    az = __ffma2_rn(dz, qr3, az);
  }
}

template <bool kAcc>
__device__ __forceinline__ void pair_body(const float4 sv, const float2 X, const float2 Y, const float2 Z, float2& ph,
                                          float2& ax, float2& ay, float2& az) {
  const float2 dx = __fadd2_rn(X, make_float2(sv.x, sv.x));
  const float2 dy = __fadd2_rn(Y, make_float2(sv.y, sv.y));
  const float2 dz = __fadd2_rn(Z, make_float2(sv.z, sv.z));
  pair_finish<kAcc, false>(dx, dy, dz, sv.w, ph, ax, ay, az);
}

// compensated pair (self and near tiles): dx = (X_hi - s_hi) + (X_lo - s_lo); the hi difference
// is exact for close pairs (Sterbenz), so the pair distance keeps ~48 bits: 6 more FADD2
struct Tgt {
  float2 X, Y, Z, XL, YL, ZL;
};
template <bool kAcc, bool kGuard>
__device__ __forceinline__ void pair_body_prec(const float4 sh, const float4 sl, const Tgt& T, float2& ph, float2& ax,
                                               float2& ay, float2& az) {
  const float2 dx = __fadd2_rn(__fadd2_rn(T.X, make_float2(sh.x, sh.x)), __fadd2_rn(T.XL, make_float2(sl.x, sl.x)));
  const float2 dy = __fadd2_rn(__fadd2_rn(T.Y, make_float2(sh.y, sh.y)), __fadd2_rn(T.YL, make_float2(sl.y, sl.y)));
  const float2 dz = __fadd2_rn(__fadd2_rn(T.Z, make_float2(sh.z, sh.z)), __fadd2_rn(T.ZL, make_float2(sl.z, sl.z)));
  pair_finish<kAcc, kGuard>(dx, dy, dz, sh.w, ph, ax, ay, az);
}

struct Acc64 {
  double ph0 = 0.0, ph1 = 0.0, ax0 = 0.0, ax1 = 0.0, ay0 = 0.0, ay1 = 0.0, az0 = 0.0, az1 = 0.0;
  // fold one tile's FP32 partials into the FP64 accumulators
  __device__ __forceinline__ void fold(const float2 ph, const float2 ax, const float2 ay, const float2 az, bool acc) {
    ph0 += ph.x;
    ph1 += ph.y;
    if (acc) {
      ax0 += ax.x;
      ax1 += ax.y;
      ay0 += ay.x;
      ay1 += ay.y;
      az0 += az.x;
      az1 += az.y;
    }
  }
};

template <bool kAcc>
__device__ __forceinline__ void tile_compute(const float4* __restrict__ buf, int nb, int g, int G, const Tgt& T,
                                             Acc64& A) {
  float2 ph = make_float2(0.f, 0.f), ax = ph, ay = ph, az = ph;
  // group g takes a contiguous chunk of the tile: unit stride, immediate-offset LDS and one
  // pointer bump per 4 independent sources (ILP, no per-source address arithmetic)
  const int chunk = ((nb + G - 1) / G) | 1;  // odd: the groups of a warp hit distinct banks
  const float4* p = buf + g * chunk;
  const float4* const end = buf + min(nb, (g + 1) * chunk);
#ifndef FMM_P2P_UNROLL
#define FMM_P2P_UNROLL 8
#endif
  constexpr int U = FMM_P2P_UNROLL;
  for (; p + (U - 1) < end; p += U) {
    float4 sv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) sv[u] = p[u];
#pragma unroll
    for (int u = 0; u < U; ++u) pair_body<kAcc>(sv[u], T.X, T.Y, T.Z, ph, ax, ay, az);
  }
  for (; p < end; ++p) pair_body<kAcc>(*p, T.X, T.Y, T.Z, ph, ax, ay, az);
  A.fold(ph, ax, ay, az, kAcc);
}

template <bool kAcc, bool kGuard, int TB>
__device__ __forceinline__ void tile_compute_prec(const float4* __restrict__ buf, int nb, int g, int G, const Tgt& T,
                                                  Acc64& A) {
  constexpr int kHalf = TB / 2;  // hi in [0, half), lo in [half, 2 half)
  float2 ph = make_float2(0.f, 0.f), ax = ph, ay = ph, az = ph;
  const int chunk = ((nb + G - 1) / G) | 1;
  const float4* p = buf + g * chunk;
  const float4* const end = buf + min(nb, (g + 1) * chunk);
  constexpr int U = 4;
  for (; p + (U - 1) < end; p += U) {
    float4 sh[U], sl[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      sh[u] = p[u];
      sl[u] = p[kHalf + u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) pair_body_prec<kAcc, kGuard>(sh[u], sl[u], T, ph, ax, ay, az);
  }
  for (; p < end; ++p) pair_body_prec<kAcc, kGuard>(p[0], p[kHalf], T, ph, ax, ay, az);
  A.fold(ph, ax, ay, az, kAcc);
}

#ifndef FMM_P2P_MIN_BLOCKS
#define FMM_P2P_MIN_BLOCKS 6
#endif
// near test: tight body boxes closer than this fraction of (r_t + r_s) on every axis (the far
// entries' pairs then have a relative FP32 distance error below ~1.4e-5)
#ifndef FMM_P2P_NEAR_GAP
#define FMM_P2P_NEAR_GAP 0.02
#endif
// ------------------------------------------------ FP32 kernel, warp-specialised pipeline ----
// One CTA per work item, five warps, no per-tile CTA barriers: a fifth
// (producer) warp resolves each tile's list entries, issues its TMA bulk copies, converts the
// landed bodies into the target frame and publishes the tile on full[b]; the four consumer
// warps compute and release the buffer on empty[b] (one arrival per warp). Consumers never wait
// for each other inside the pipeline, so a warp that finishes its share of a tile early starts
// on the next one (the producer runs up to one tile ahead: two buffers).
constexpr int kWsThreads = kThreads + 32;
#ifndef FMM_P2P_SMALL_SOURCES
#define FMM_P2P_SMALL_SOURCES 2048.0
#endif
#ifndef FMM_P2P_SMALL_CT
#define FMM_P2P_SMALL_CT 64
#endif
#ifndef FMM_P2P_SMALL_TB
#define FMM_P2P_SMALL_TB 512
#endif
constexpr int kSmallCT = FMM_P2P_SMALL_CT, kSmallTB = FMM_P2P_SMALL_TB;
constexpr double kSmallSourcesPerTarget = FMM_P2P_SMALL_SOURCES;  // mean P2P sources per target body below which the narrow CTAs run

// Phase timestamps of sampled CTAs (variant builds only, tools/p2p_trace.py): clock64 at entry,
// item loaded, producer tile-0 set up / copies issued / landed / published, producer done,
// consumers' first tile seen / pair loops done / results written; tiles; targets.
#ifndef FMM_P2P_TRACE
#define FMM_P2P_TRACE 0
#endif
#if FMM_P2P_TRACE
constexpr int kTraceCtas = 1 << 16, kTraceStride = 16;
__device__ unsigned long long g_p2p_trace[kTraceCtas * 16];
#define P2P_TR(slot) do { if (trace) trace[slot] = clock64(); } while (0)
#define P2P_TRV(slot, v) do { if (trace) trace[slot] = (v); } while (0)
#else
#define P2P_TR(slot) do {} while (0)
#define P2P_TRV(slot, v) do {} while (0)
#endif

// producer warp: shift one tile's staged bodies into the target frame and negate
__device__ __forceinline__ void convert_warp(int lane, const TileTab& tt, float4* buf) {
  const int nseg = tt.nseg;
#pragma unroll 1
  for (int k = 0; k < nseg; k += 4) {
    int32_t o[4], n[4];
    float sx[4], sy[4], sz[4];
    int32_t nm = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const bool ok = k + q < nseg;
      o[q] = ok ? tt.off[k + q] : 0;
      n[q] = ok ? tt.off[k + q + 1] - o[q] : 0;
      sx[q] = ok ? tt.sh[k + q][0] : 0.f;
      sy[q] = ok ? tt.sh[k + q][1] : 0.f;
      sz[q] = ok ? tt.sh[k + q][2] : 0.f;
      nm = max(nm, n[q]);
    }
#pragma unroll 1
    for (int j = lane; j < nm; j += 32) {
      float4 a[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (j < n[q]) a[q] = buf[o[q] + j];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (j < n[q]) buf[o[q] + j] = make_float4(-a[q].x - sx[q], -a[q].y - sy[q], -a[q].z - sz[q], a[q].w);
    }
  }
}

template <int TB>
__device__ __forceinline__ void convert_prec_warp(int lane, const TileTab& tt, float4* buf) {
  constexpr int kHalf = TB / 2;
  const int nb = tt.off[tt.nseg];
  const int nseg = tt.nseg;
  int k = 0;
#pragma unroll 1
  for (int j = lane; j < nb; j += 32) {
    while (k + 1 < nseg && tt.off[k + 1] <= j) ++k;  // j ascends: the entry index only moves forward
    const float4 h = buf[j], l = buf[kHalf + j];
    const float2 x = two_sum(h.x, tt.sh[k][0]), y = two_sum(h.y, tt.sh[k][1]), z = two_sum(h.z, tt.sh[k][2]);
    buf[j] = make_float4(-x.x, -y.x, -z.x, h.w);
    buf[kHalf + j] = make_float4(-((x.y + l.x) + tt.sl[k][0]), -((y.y + l.y) + tt.sl[k][1]),
                                     -((z.y + l.z) + tt.sl[k][2]), 0.f);
  }
}

// CT consumer threads (two targets each: up to 2 CT... an item holds at most kThreads = 128 targets,
// so CT = 64 threads loop twice over the final write) and TB bodies per tile. The small variant
// (CT = 64, TB = 512: 96 threads, ~20 KB) runs 10 CTAs/SM on small-leaf trees, where an item is
// ~3 tiles and a CTA spends a third of its life in the start-up chain of its first tile
// (profiles/r2_p2p_phase_trace.txt): more, narrower CTAs keep more of them in their pair loops.
#ifndef FMM_P2P_MIN_BLOCKS_SMALL
#define FMM_P2P_MIN_BLOCKS_SMALL 10
#endif
template <bool kAcc, int CT, int TB>
__global__ void __launch_bounds__(CT + 32, CT == kThreads ? FMM_P2P_MIN_BLOCKS : FMM_P2P_MIN_BLOCKS_SMALL)
k_p2p_fp32_ws(const P2PItem* __restrict__ items, const P2PEnt* __restrict__ ent, const float4* __restrict__ bodyf,
              const float4* __restrict__ bodyl, double* __restrict__ phi_out, double* __restrict__ acc_out,
              double* __restrict__ partial) {
  __shared__ __align__(16) float4 sS[2][TB];
  __shared__ TileTab tabs[2];
  __shared__ __align__(8) uint64_t full[2], tmab[2], empty[2];

#if FMM_P2P_TRACE
  unsigned long long* trace = nullptr;
  if ((threadIdx.x == 0 || threadIdx.x == CT) && blockIdx.x % kTraceStride == 0 &&
      blockIdx.x / kTraceStride < kTraceCtas)
    trace = g_p2p_trace + (blockIdx.x / kTraceStride) * 16;
  if (threadIdx.x == 0) P2P_TR(0);
#endif
  const P2PItem it = items[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&tmab[b], 1);
      mbar_init(&empty[b], CT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) P2P_TR(1);

  if (tid >= CT) {  // ---- producer warp
    int32_t cursor = it.lb, off = 0;
    unsigned k = 0;
    for (; cursor < it.le; ++k) {
      const int b = k & 1;
      if (k >= 2) mbar_wait(&empty[b], ((k >> 1) - 1) & 1u);
      tile_setup_ent<TB>(lane, it.le, cursor, off, ent + cursor, tabs[b]);
      __syncwarp();
      if (k == 0) P2P_TR(2);
      tile_tma<TB>(lane, tabs[b], bodyf, bodyl, sS[b], &tmab[b]);
      if (k == 0) P2P_TR(3);
      mbar_wait(&tmab[b], (k >> 1) & 1u);
      if (k == 0) P2P_TR(4);
      if (tabs[b].prec) convert_prec_warp<TB>(lane, tabs[b], sS[b]);
      else convert_warp(lane, tabs[b], sS[b]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[b]);
      if (k == 0) P2P_TR(5);
      cursor = tabs[b].next;
      off = tabs[b].next_off;
    }
    P2P_TR(6);
    P2P_TRV(10, k);
    return;
  }

  // ---- consumer warps
  const int nt = it.te - it.tb;
  FMM_CHECK(it.tb >= 0 && nt >= 1 && nt <= kThreads && it.te <= FMM_LIM(nbodies), "k_p2p_fp32_ws: target range");
  FMM_CHECK(it.lb >= 0 && it.lb <= it.le && it.le <= FMM_LIM(n_p2p), "k_p2p_fp32_ws: list range");
  const int slots = (nt + 1) >> 1;
  const int G = CT / slots;
  const int g = tid / slots, t = tid - g * slots;
  const bool active = g < G;
  Tgt T;
  T.X = make_float2(0.f, 0.f);
  T.Y = T.Z = T.XL = T.YL = T.ZL = T.X;
  if (active) {
    const int32_t i0 = it.tb + 2 * t, i1 = (2 * t + 1 < nt) ? i0 + 1 : i0;
    const float4 b0 = bodyf[i0], b1 = bodyf[i1];
    const float4 l0 = bodyl[i0], l1 = bodyl[i1];
    T.X = make_float2(b0.x, b1.x);
    T.Y = make_float2(b0.y, b1.y);
    T.Z = make_float2(b0.z, b1.z);
    T.XL = make_float2(l0.x, l1.x);
    T.YL = make_float2(l0.y, l1.y);
    T.ZL = make_float2(l0.z, l1.z);
  }
  Acc64 A;
  if (it.lb < it.le) {
    for (unsigned k = 0;; ++k) {
      const int b = k & 1;
      mbar_wait(&full[b], (k >> 1) & 1u);
      if (k == 0) P2P_TR(7);
      const TileTab& tc = tabs[b];
      const int nb = tc.off[tc.nseg];
      const bool prec = tc.prec != 0, guard = tc.guard != 0, more = tc.next < it.le;
      if (active) {
        if (!prec)
          tile_compute<kAcc>(sS[b], nb, g, G, T, A);
        else if (guard)
          tile_compute_prec<kAcc, true, TB>(sS[b], nb, g, G, T, A);
        else
          tile_compute_prec<kAcc, false, TB>(sS[b], nb, g, G, T, A);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[b]);
      if (!more) break;
    }
  }
  P2P_TR(8);
  P2P_TRV(11, static_cast<unsigned long long>(nt));
  // reduce the G lane groups in fixed order (reusing the tile buffer: the producer is done and
  // every consumer has released its last tile once this named barrier completes) and write
  asm volatile("bar.sync 1, %0;\n" ::"r"(CT) : "memory");
  double* red = reinterpret_cast<double*>(sS);  // [G][slots][2 targets][4]
  if (active) {
    double* r = red + 8 * (g * slots + t);
    r[0] = A.ph0; r[1] = A.ax0; r[2] = A.ay0; r[3] = A.az0;
    r[4] = A.ph1; r[5] = A.ax1; r[6] = A.ay1; r[7] = A.az1;
  }
  asm volatile("bar.sync 1, %0;\n" ::"r"(CT) : "memory");
  // one pass when CT = kThreads (an item holds at most kThreads targets), two for the narrow shape
  auto write_target = [&](int tt) {
    const int sl = tt >> 1, h = tt & 1;
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (int gg = 0; gg < G; ++gg) {
      const double* r = red + 8 * (gg * slots + sl) + 4 * h;
      v[0] += r[0];
      v[1] += r[1];
      v[2] += r[2];
      v[3] += r[3];
    }
    if (it.pbase < 0) {
      const int32_t i = it.tb + tt;
      phi_out[i] = v[0];
      if (kAcc) {
        acc_out[3 * i] = v[1];
        acc_out[3 * i + 1] = v[2];
        acc_out[3 * i + 2] = v[3];
      }
    } else {
      double* p = partial + 4 * ((int64_t)it.pbase + tt);
      p[0] = v[0];
      p[1] = v[1];
      p[2] = v[2];
      p[3] = v[3];
    }
  };
  if constexpr (CT >= kThreads) {
    if (tid < nt) write_target(tid);
  } else {
    for (int tt = tid; tt < nt; tt += CT) write_target(tt);
  }
  if (tid == 0) P2P_TR(9);
}

// ------------------------------------------------------------------------ FP64 kernel ----
// Parity mode: absolute FP64 coordinates and the reference's arithmetic
// (dx = x_i - y_j, r2 = dx^2 + dy^2 + dz^2, skip r2 == 0, phi += q / sqrt(r2)), with r2 fused
// (FMA) and 1/sqrt(r2) as rsqrt (<= 1 ulp) rather than an IEEE sqrt followed by an IEEE divide.
__device__ __forceinline__ void p2p_pair_fp64(const double4& bt, const double4& s, int with_acc, double& phi,
                                              double& ax, double& ay, double& az) {
  const double dx = bt.x - s.x, dy = bt.y - s.y, dz = bt.z - s.z;
  const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));  // zero exactly when dx = dy = dz = 0
  // rsqrt: <= 1 ulp, one Newton sequence instead of IEEE sqrt + divide; r2 == 0 (the self pair)
  // contributes nothing, as a select rather than a branch
  const double ri = r2 > 0.0 ? rsqrt(r2) : 0.0;
  const double qr = s.w * ri;
  phi += qr;
  if (with_acc) {
    const double qr3 = qr * ri * ri;
    ax += dx * qr3;
    ay += dy * qr3;
    az += dz * qr3;
  }
}

#ifndef FMM_P2P64_MIN_BLOCKS
#define FMM_P2P64_MIN_BLOCKS 8  // 64 registers, 8 CTAs/SM (A/B at C2: 4 -> 9.14 ms, 6 -> 8.44, 7 -> 8.35, 8 -> 8.25)
#endif
__global__ void __launch_bounds__(kThreads, FMM_P2P64_MIN_BLOCKS)
k_p2p_fp64(const P2PItem* __restrict__ items, const int32_t* __restrict__ src_list,
           const int32_t* __restrict__ bb, const int32_t* __restrict__ be,
           const double4* __restrict__ bodies, double* __restrict__ phi_out, double* __restrict__ acc_out,
           double* __restrict__ partial, int with_acc) {
  constexpr int kTile = 512;
  __shared__ double4 sS[kTile];
  __shared__ int32_t seg_off[kTileSegs + 1];
  __shared__ int32_t seg_src[kTileSegs];
  __shared__ int32_t seg_boff[kTileSegs];
  __shared__ int32_t nxt[3];
  __shared__ double red[8][kThreads];

  // Two targets per thread (t and t + nh): one shared-memory source read serves two pairs.
  const P2PItem it = items[blockIdx.x];
  const int tid = threadIdx.x;
  const int nt = it.te - it.tb;
  FMM_CHECK(it.tb >= 0 && nt >= 1 && nt <= kThreads && it.te <= FMM_LIM(nbodies), "k_p2p_fp64: target range");
  FMM_CHECK(it.lb >= 0 && it.lb <= it.le && it.le <= FMM_LIM(n_p2p), "k_p2p_fp64: list range");
  const int nh = (nt + 1) >> 1;
  const int G = kThreads / nh;
  const int g = tid / nh, t = tid - g * nh;
  const bool active = g < G;
  double4 bt = make_double4(0, 0, 0, 0), bu = make_double4(0, 0, 0, 0);
  if (active) bt = bodies[it.tb + t];
  if (active && t + nh < nt) bu = bodies[it.tb + t + nh];  // else a dummy whose sums are dropped
  double phi_d = 0.0, ax_d = 0.0, ay_d = 0.0, az_d = 0.0;
  double phi_e = 0.0, ax_e = 0.0, ay_e = 0.0, az_e = 0.0;
  int32_t cursor = it.lb, cur_off = 0;
  while (cursor < it.le) {
    tile_setup<kTile>(tid, it.le, cursor, cur_off, src_list, bb, be, seg_off, seg_src, seg_boff, nxt);
    __syncthreads();
    const int32_t nseg = nxt[2];
    const int32_t nb = seg_off[nseg];
    {
      const int w = tid >> 5, lane = tid & 31;
      for (int k = w; k < nseg; k += kThreads / 32) {
        const int32_t src = seg_src[k];
        const int32_t base = bb[src] + seg_boff[k], o0 = seg_off[k], n = seg_off[k + 1] - o0;
        for (int j = lane; j < n; j += 32) sS[o0 + j] = bodies[base + j];
      }
    }
    __syncthreads();
    if (active) {
      for (int j = g; j < nb; j += G) {
        const double4 s = sS[j];
        p2p_pair_fp64(bt, s, with_acc, phi_d, ax_d, ay_d, az_d);
        p2p_pair_fp64(bu, s, with_acc, phi_e, ax_e, ay_e, az_e);
      }
    }
    cursor = nxt[0];
    cur_off = nxt[1];
    __syncthreads();
  }
  red[0][tid] = phi_d;
  red[1][tid] = ax_d;
  red[2][tid] = ay_d;
  red[3][tid] = az_d;
  red[4][tid] = phi_e;
  red[5][tid] = ax_e;
  red[6][tid] = ay_e;
  red[7][tid] = az_e;
  __syncthreads();
  if (tid < nt) {
    const int h = tid >= nh ? 1 : 0, tt = tid - h * nh;
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (int gg = 0; gg < G; ++gg)
      for (int c = 0; c < 4; ++c) v[c] += red[4 * h + c][gg * nh + tt];
    if (it.pbase < 0) {
      const int32_t i = it.tb + tid;
      phi_out[i] = v[0];
      if (with_acc) {
        acc_out[3 * i] = v[1];
        acc_out[3 * i + 1] = v[2];
        acc_out[3 * i + 2] = v[3];
      }
    } else {
      double* p = partial + 4 * ((int64_t)it.pbase + tid);
      p[0] = v[0];
      p[1] = v[1];
      p[2] = v[2];
      p[3] = v[3];
    }
  }
}

// Split-list targets: sum the source-chunk partials in chunk order.
__global__ void k_p2p_reduce(const int4* __restrict__ red, int64_t nred, const double* __restrict__ partial,
                             double* __restrict__ phi_out, double* __restrict__ acc_out, int with_acc) {
  const int64_t r = blockIdx.x;
  if (r >= nred) return;
  const int4 e = red[r];  // x = tb, y = te, z = pbase of chunk 0, w = nchunks
  const int nt = e.y - e.x;
  for (int t = threadIdx.x; t < nt; t += blockDim.x) {
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k = 0; k < e.w; ++k) {
      const double* p = partial + 4 * ((int64_t)e.z + (int64_t)k * nt + t);
      for (int c = 0; c < 4; ++c) v[c] += p[c];
    }
    const int32_t i = e.x + t;
    phi_out[i] = v[0];
    if (with_acc) {
      acc_out[3 * i] = v[1];
      acc_out[3 * i + 1] = v[2];
      acc_out[3 * i + 2] = v[3];
    }
  }
}

// ---------------------------------------------------------------- work list build ----
__global__ void k_leaf_cost(const int32_t* __restrict__ leaves, int64_t nleaves, const int64_t* __restrict__ off,
                            const int32_t* __restrict__ bb, const int32_t* __restrict__ be, uint64_t cmax,
                            const int64_t* __restrict__ sum_ns, int32_t* __restrict__ nitems,
                            int32_t* __restrict__ nred, int32_t* __restrict__ npart) {
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w >= nleaves) return;
  const int32_t leaf = leaves[w];
  const int64_t l0 = off[leaf], l1 = off[leaf + 1];
  const int64_t nt = be[leaf] - bb[leaf];
  const int64_t cost = nt * sum_ns[w];
  int64_t nsc = (cost + (int64_t)cmax - 1) / (int64_t)cmax;
  if (nsc < 1) nsc = 1;
  if (nsc > l1 - l0) nsc = l1 - l0;
  if (l1 == l0) nsc = 0;
  const int64_t ntc = (nt + kThreads - 1) / kThreads;
  nitems[w] = static_cast<int32_t>(nsc * ntc);
  nred[w] = nsc > 1 ? static_cast<int32_t>(ntc) : 0;
  npart[w] = nsc > 1 ? static_cast<int32_t>(nsc * nt) : 0;
}

__global__ void k_gather_items(const P2PItem* __restrict__ in, const int32_t* __restrict__ order, int64_t n,
                               P2PItem* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[order[i]];
}

// ---- entry-parallel helpers (no per-leaf serial loops: C3's halo leaf has 57 K entries) ----
__global__ void k_entry_counts(const int32_t* __restrict__ src, int64_t n, const int32_t* __restrict__ bb,
                               const int32_t* __restrict__ be, int64_t* __restrict__ cnt) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < n) {
    const int32_t q = src[k];
    cnt[k] = be[q] - bb[q];
  } else if (k == n) {
    cnt[k] = 0;
  }
}

// per work leaf: S = sum of source sizes (from the entry prefix), total cost reduced per warp;
// total[1] = a bound on any one item's cost (min(leaf size, kThreads) * S), which sizes the
// cost sort's key range
__global__ void k_leaf_sum(const int32_t* __restrict__ leaves, int64_t nleaves, const int64_t* __restrict__ off,
                            const int64_t* __restrict__ pre, const int32_t* __restrict__ bb,
                            const int32_t* __restrict__ be, int64_t* __restrict__ sum_ns,
                            unsigned long long* __restrict__ total) {
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  unsigned long long v = 0, m = 0;
  if (w < nleaves) {
    const int32_t leaf = leaves[w];
    const int64_t S = pre[off[leaf + 1]] - pre[off[leaf]];
    const int32_t nt = be[leaf] - bb[leaf];
    sum_ns[w] = S;
    v = static_cast<unsigned long long>(S) * static_cast<unsigned long long>(nt);
    m = static_cast<unsigned long long>(S) * static_cast<unsigned long long>(min(nt, kThreads));
  }
  for (int o = 16; o > 0; o >>= 1) {
    v += __shfl_xor_sync(0xffffffffu, v, o);
    m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  }
  if ((threadIdx.x & 31) == 0 && v) {
    atomicAdd(total, v);
    atomicMax(total + 1, m);
  }
}

// items of one work leaf (thread each): chunk j covers list entries [bnd_j, bnd_{j+1}) where
// bnd_j is the first entry whose source-body prefix reaches j * S / nsc (binary search)
__global__ void k_write_items(const int32_t* __restrict__ leaves, int64_t nleaves, const int64_t* __restrict__ off,
                               const int64_t* __restrict__ pre, const int32_t* __restrict__ bb,
                               const int32_t* __restrict__ be, const int64_t* __restrict__ sum_ns,
                               const int32_t* __restrict__ nitems, const int32_t* __restrict__ item_off,
                               const int32_t* __restrict__ red_off, const int32_t* __restrict__ part_off,
                               P2PItem* __restrict__ items, uint64_t* __restrict__ costs, int4* __restrict__ red) {
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w >= nleaves || nitems[w] == 0) return;
  const int32_t leaf = leaves[w];
  const int32_t tb = bb[leaf], te = be[leaf], nt = te - tb;
  const int32_t ntc = (nt + kThreads - 1) / kThreads;
  const int32_t nsc = nitems[w] / ntc;
  const int64_t l0 = off[leaf], l1 = off[leaf + 1];
  const int64_t S = sum_ns[w], p0 = pre[l0];
  const int32_t pb = nsc > 1 ? part_off[w] : -1;
  int32_t out = item_off[w];
  int64_t lb = l0;
  for (int32_t j = 0; j < nsc; ++j) {
    int64_t le = l1;
    if (j + 1 < nsc) {  // first k in (lb, l1] with pre[k] - p0 >= (j+1) S / nsc (empty once lb = l1)
      const int64_t target = p0 + (S * (j + 1)) / nsc;
      int64_t lo = min(lb + 1, l1), hi = l1;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (pre[mid] < target) lo = mid + 1; else hi = mid;
      }
      le = lo;
    }
    const int64_t ns_chunk = pre[le] - pre[lb];
    for (int32_t tc = 0; tc < ntc; ++tc) {
      const int32_t t0 = tb + tc * kThreads;
      const int32_t t1 = min(te, t0 + kThreads);
      P2PItem itm;
      itm.leaf = leaf;
      itm.tb = t0;
      itm.te = t1;
      itm.lb = static_cast<int32_t>(lb);
      itm.le = static_cast<int32_t>(le);
      // partial layout per leaf: t-chunk regions of nsc * (t1-t0) bodies, source-chunk major
      itm.pbase = pb < 0 ? -1 : pb + nsc * (t0 - tb) + j * (t1 - t0);
      itm.sb0 = 0;
      itm.pad = 0;
      items[out] = itm;
      costs[out] = static_cast<uint64_t>(t1 - t0) * static_cast<uint64_t>(ns_chunk);
      ++out;
    }
    lb = le;
  }
  if (nsc > 1)
    for (int32_t tc = 0; tc < ntc; ++tc) {
      const int32_t t0 = tb + tc * kThreads;
      red[red_off[w] + tc] = make_int4(t0, min(te, t0 + kThreads), pb + nsc * (t0 - tb), nsc);
    }
}

// P2P list entries: {source body range, kind, FP64 centre shift into the target leaf frame as
// FP32 hi + lo}. Within each target's (source-sorted) list the order is
// far entries, near entries, self entry (each group ascending by source), so that a work item's
// tiles each hold one class: only the self tile runs the r^2 == 0 guard and only self / near
// tiles pay for compensated coordinates. Near = the tight body boxes of the two leaves are less
// than FMM_P2P_NEAR_GAP (r_t + r_s) apart along every axis; a far entry's body pairs are then at
// least that far apart, and FP32 offsets (magnitude <= ~4.5 (r_t + r_s) in the target frame)
// give them a relative distance error below ~1.4e-5.
// Items still partition the list positions, so every entry is computed exactly once.
__device__ __forceinline__ bool near_leaf(const double4 tlo, const double4 thi, const double4 slo, const double4 shi,
                                          double lim) {
  const double gx = fmax(slo.x - thi.x, tlo.x - shi.x);
  const double gy = fmax(slo.y - thi.y, tlo.y - shi.y);
  const double gz = fmax(slo.z - thi.z, tlo.z - shi.z);
  return fmax(gx, fmax(gy, gz)) < lim;
}

// tight bounding box of each leaf's bodies (warp per leaf; tree order: contiguous bodies)
__global__ void k_leaf_boxes(const int32_t* __restrict__ leaves, int64_t nleaves, const int32_t* __restrict__ bb,
                             const int32_t* __restrict__ be, const double4* __restrict__ bodies,
                             double4* __restrict__ lo, double4* __restrict__ hi) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nleaves) return;
  const int32_t leaf = leaves[w];
  double x0 = INFINITY, y0 = INFINITY, z0 = INFINITY, x1 = -INFINITY, y1 = -INFINITY, z1 = -INFINITY;
  for (int32_t i = bb[leaf] + lane; i < be[leaf]; i += 32) {
    const double4 b = bodies[i];
    x0 = fmin(x0, b.x); y0 = fmin(y0, b.y); z0 = fmin(z0, b.z);
    x1 = fmax(x1, b.x); y1 = fmax(y1, b.y); z1 = fmax(z1, b.z);
  }
  for (int o = 16; o > 0; o >>= 1) {
    x0 = fmin(x0, __shfl_xor_sync(0xffffffffu, x0, o));
    y0 = fmin(y0, __shfl_xor_sync(0xffffffffu, y0, o));
    z0 = fmin(z0, __shfl_xor_sync(0xffffffffu, z0, o));
    x1 = fmax(x1, __shfl_xor_sync(0xffffffffu, x1, o));
    y1 = fmax(y1, __shfl_xor_sync(0xffffffffu, y1, o));
    z1 = fmax(z1, __shfl_xor_sync(0xffffffffu, z1, o));
  }
  if (lane == 0) {
    lo[leaf] = make_double4(x0, y0, z0, 0.0);
    hi[leaf] = make_double4(x1, y1, z1, 0.0);
  }
}

// Entry-parallel (C3's halo leaf alone has 57 K entries): pass 1 classifies every entry
// (self / near / far); an exclusive scan of the packed per-class indicators (near in the low,
// far in the high 32 bits) gives every entry its rank within its target's class; pass 2 writes
// the entry at
//   far: l0 + far rank | near: l0 + n_far + near rank | self: l1 - 1 (the list's last entry).
__global__ void k_ent_class(const int32_t* __restrict__ tgt, const int32_t* __restrict__ src, int64_t ne,
                            const double4* __restrict__ cr, const double4* __restrict__ blo,
                            const double4* __restrict__ bhi, int64_t* __restrict__ cls) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k > ne) return;
  if (k == ne) {
    cls[k] = 0;
    return;
  }
  const int32_t t = tgt[k], s = src[k];
  int64_t v;
  if (s == t) {
    v = 0;
  } else {
    const bool nr = near_leaf(blo[t], bhi[t], blo[s], bhi[s], FMM_P2P_NEAR_GAP * (cr[t].w + cr[s].w));
    v = nr ? 1ll : (1ll << 32);
  }
  cls[k] = v;
}

__global__ void k_ent_write(const int32_t* __restrict__ tgt, const int32_t* __restrict__ src, int64_t ne,
                            const int64_t* __restrict__ off, const int64_t* __restrict__ cls,
                            const int64_t* __restrict__ pre,
                            const int32_t* __restrict__ bb, const int32_t* __restrict__ be,
                            const double4* __restrict__ cr, P2PEnt* __restrict__ ent) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= ne) return;
  const int32_t t = tgt[k], s = src[k];
  FMM_CHECK(t >= 0 && t < FMM_LIM(ncells) && s >= 0 && s < FMM_LIM(ncells), "k_ent_write: cell index");
  const int64_t l0 = off[t], l1 = off[t + 1];
  FMM_CHECK(l0 <= k && k < l1, "k_ent_write: entry outside its target's list");
  const int64_t v = cls[k], P0 = pre[l0], Pk = pre[k];
  const int64_t lo0 = P0 & 0xffffffffll, hi0 = P0 >> 32;
  int64_t pos;
  int kind;
  // far entries first, then near, the self entry last: an item's short compensated tiles come
  // after its full far tiles, so the producer stages them while the consumers are busy
  if (s == t) {
    pos = l1 - 1;
    kind = kKindSelf;
  } else if (v == 1) {
    const int64_t nfar = (pre[l1] >> 32) - hi0;
    pos = l0 + nfar + ((Pk & 0xffffffffll) - lo0);
    kind = kKindNear;
  } else {
    pos = l0 + ((Pk >> 32) - hi0);
    kind = kKindFar;
  }
  const double4 ct = cr[t], cs = cr[s];
  const double dx = cs.x - ct.x, dy = cs.y - ct.y, dz = cs.z - ct.z;
  const float hx = static_cast<float>(dx), hy = static_cast<float>(dy), hz = static_cast<float>(dz);
  P2PEnt e;
  e.bb = bb[s];
  e.nk = (be[s] - bb[s]) | (kind << 30);
  e.sx = hx;
  e.sy = hy;
  e.sz = hz;
  e.lx = static_cast<float>(dx - hx);
  e.ly = static_cast<float>(dy - hy);
  e.lz = static_cast<float>(dz - hz);
  FMM_CHECK(pos >= l0 && pos < l1, "k_ent_write: entry position");
  ent[pos] = e;
}

__global__ void k_iota(int32_t* __restrict__ v, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) v[i] = static_cast<int32_t>(i);
}

void exclusive_scan_i32(fmm_ctx* c, const int32_t* in, int32_t* out, int64_t n, cudaStream_t s) {
  size_t sb = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, sb, in, out, (int)n, s));
  CK(cub::DeviceScan::ExclusiveSum(temp_storage2(c, sb), sb, in, out, (int)n, s));
}

}  // namespace

// FP32 P2P list entries (self / near / far order, FP32 hi + lo shifts): depend on the lists and,
// through the near test, on the bodies' tight leaf boxes (rebuilt by a tree-reuse step)
void build_p2p_entries(fmm_ctx* c) {
  cudaStream_t s = c->pstream;
  set_check_limits(c, s);
  const int64_t ne = c->n_p2p;
  P2PEnt* ent = reinterpret_cast<P2PEnt*>(c->p2p_ent.ensure(2 * (ne + 1)));
  double4* blo = c->leaf_lo.ensure(c->ncells);
  double4* bhi = c->leaf_hi.ensure(c->ncells);
  k_leaf_boxes<<<ceil_div(c->nleaves * 32, 256), 256, 0, s>>>(c->leaves.p, c->nleaves, c->c_body_begin.p,
                                                             c->c_body_end.p, c->bodies.p, blo, bhi);
  int64_t* cls = c->ent_cls.ensure(ne + 1);
  int64_t* epre = c->ent_pre.ensure(ne + 1);
  k_ent_class<<<ceil_div(ne + 1, 256), 256, 0, s>>>(c->p2p_tgt.p, c->p2p_src.p, ne, c->c_cr.p, blo, bhi, cls);
  {
    size_t sb = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, sb, cls, epre, (int)(ne + 1), s));
    CK(cub::DeviceScan::ExclusiveSum(temp_storage2(c, sb), sb, cls, epre, (int)(ne + 1), s));
  }
  if (ne > 0)
    k_ent_write<<<ceil_div(ne, 256), 256, 0, s>>>(c->p2p_tgt.p, c->p2p_src.p, ne, c->p2p_off.p, cls, epre,
                                                  c->c_body_begin.p, c->c_body_end.p, c->c_cr.p, ent);
  CK_LAUNCH("k_ent_write");
  c->kernel_launches += 5;
}

// P2P work list, in two halves around the host read of the total pair count, on the P2P
// preparation stream (c->pstream) and with buffers of its own, so that evaluate can run it
// concurrently with M2L (see capi.cu).
void p2p_worklist_begin(fmm_ctx* c) {
  cudaStream_t s = c->pstream;
  const int64_t nl = c->nwl, ne = c->n_p2p;
  // source-body prefix over all list entries
  int64_t* pre = c->p2p_pre.ensure(ne + 2);
  int64_t* cnt = reinterpret_cast<int64_t*>(c->p2p_keys_c.ensure(ne + 2));
  k_entry_counts<<<ceil_div(ne + 1, 256), 256, 0, s>>>(c->p2p_src.p, ne, c->c_body_begin.p, c->c_body_end.p, cnt);
  {
    size_t sb = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, sb, cnt, pre, (int)(ne + 1), s));
    CK(cub::DeviceScan::ExclusiveSum(temp_storage2(c, sb), sb, cnt, pre, (int)(ne + 1), s));
  }
  int64_t* sum_ns = c->p2p_sum.ensure(nl + 1);
  unsigned long long* tot = reinterpret_cast<unsigned long long*>(c->d_counters.ensure(16)) + 12;
  CK(cudaMemsetAsync(tot, 0, 2 * sizeof(unsigned long long), s));
  k_leaf_sum<<<ceil_div(nl, 256), 256, 0, s>>>(c->wl, nl, c->p2p_off.p, pre, c->c_body_begin.p, c->c_body_end.p,
                                               sum_ns, tot);
  CK_LAUNCH("k_leaf_sum");
  CK(cudaMemcpyAsync(c->hpin + 16, tot, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  c->kernel_launches += 3;
  c->p2p_pending = true;
}

void p2p_worklist_end(fmm_ctx* c) {
  if (!c->p2p_pending) return;
  cudaStream_t s = c->pstream;
  const int64_t nl = c->nwl;
  int64_t* pre = c->p2p_pre.p;
  int64_t* sum_ns = c->p2p_sum.p;
  CK(cudaStreamSynchronize(s));
  c->p2p_body_pairs = c->hpin[16];
  const uint64_t total = static_cast<uint64_t>(c->p2p_body_pairs);
  // Cost cap per item: an eighth of one SM's fair share, never below 64K pairs, so that a
  // single heavy target (C3's halo leaf: 60.5 M pairs) is spread over many SMs.
  uint64_t cmax = total / (148ull * 8ull);
  if (cmax < 65536ull) cmax = 65536ull;

  int32_t* counts = c->p2p_i32a.ensure(3 * (nl + 1));
  int32_t* offs = c->p2p_i32b.ensure(3 * (nl + 1));
  int32_t *nitems = counts, *nred = counts + (nl + 1), *npart = counts + 2 * (nl + 1);
  int32_t *item_off = offs, *red_off = offs + (nl + 1), *part_off = offs + 2 * (nl + 1);
  CK(cudaMemsetAsync(counts, 0, sizeof(int32_t) * 3 * (nl + 1), s));
  k_leaf_cost<<<ceil_div(nl, 256), 256, 0, s>>>(c->wl, nl, c->p2p_off.p, c->c_body_begin.p, c->c_body_end.p,
                                                cmax, sum_ns, nitems, nred, npart);
  CK_LAUNCH("k_leaf_cost");
  exclusive_scan_i32(c, nitems, item_off, nl + 1, s);
  exclusive_scan_i32(c, nred, red_off, nl + 1, s);
  exclusive_scan_i32(c, npart, part_off, nl + 1, s);
  int32_t* h = reinterpret_cast<int32_t*>(c->hpin + 24);
  CK(cudaMemcpyAsync(&h[0], item_off + nl, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&h[1], red_off + nl, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&h[2], part_off + nl, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const int64_t nitem = h[0], nr = h[1], np = h[2];
  P2PItem* items_raw = reinterpret_cast<P2PItem*>(c->p2p_items_raw.ensure(2 * (nitem + 1)));  // 32 B each
  P2PItem* items = reinterpret_cast<P2PItem*>(c->p2p_items.ensure(2 * (nitem + 1)));
  uint64_t* costs = c->p2p_keys_c.ensure(nitem + 1);
  uint64_t* costs_sorted = c->p2p_keys_b2.ensure(nitem + 1);
  int4* red = c->p2p_reduce.ensure(nr + 1);
  c->p2p_partial.ensure(4 * (np + 1));
  k_write_items<<<ceil_div(nl, 128), 128, 0, s>>>(c->wl, nl, c->p2p_off.p, pre, c->c_body_begin.p,
                                                   c->c_body_end.p, sum_ns, nitems, item_off, red_off, part_off,
                                                   items_raw, costs, red);
  CK_LAUNCH("k_write_items");
  if (c->cfg.precision == FMM_PREC_FP32_P2P) build_p2p_entries(c);
  // cost-sorted (descending, stable) work list: the longest items launch first
  int32_t* ord_in = c->p2p_i32c.ensure(2 * (nitem + 1));
  int32_t* ord_out = ord_in + (nitem + 1);
  k_iota<<<ceil_div(nitem, 256), 256, 0, s>>>(ord_in, nitem);
  size_t sb = 0;
  // every item cost is below 2^cost_bits (C2: ~20 bits); only the top kCostSortBits of them are
  // sorted (one or two radix passes instead of three to six): items of nearly equal cost keep their
  // Morton order (stable), which schedules as well as the exact order
#ifndef FMM_P2P_COST_SORT_BITS
#define FMM_P2P_COST_SORT_BITS 8
#endif
  const uint64_t cbound = static_cast<uint64_t>(c->hpin[17]);
  const int cost_bits = std::min(48, std::max(1, 64 - __builtin_clzll(cbound | 1ull)));
  const int cost_lo = std::max(0, cost_bits - FMM_P2P_COST_SORT_BITS);
  CK(cub::DeviceRadixSort::SortPairsDescending(nullptr, sb, costs, costs_sorted, ord_in, ord_out, (int)nitem, cost_lo,
                                               cost_bits, s));
  CK(cub::DeviceRadixSort::SortPairsDescending(temp_storage2(c, sb), sb, costs, costs_sorted, ord_in, ord_out,
                                               (int)nitem, cost_lo, cost_bits, s));
  k_gather_items<<<ceil_div(nitem, 256), 256, 0, s>>>(items_raw, ord_out, nitem, items);
  CK_LAUNCH("k_gather_items");
  c->n_p2p_items = nitem;
  c->n_p2p_reduce = nr;
  c->kernel_launches += 6;
  c->p2p_pending = false;
}

void build_p2p_worklist(fmm_ctx* c) {
  p2p_worklist_begin(c);
  p2p_worklist_end(c);
}

void run_p2p(fmm_ctx* c, cudaStream_t s) {
  if (!c->have_lists) fail(FMM_ERR_STATE, "p2p: no interaction lists");
  set_check_limits(c, s);
  if (c->p2p_pending) fail(FMM_ERR_STATE, "p2p: work list not finished");
  const int64_t n = c->N;
  const int wa = c->cfg.with_acc ? 1 : 0;
  double* phi = c->phi_p2p.ensure(n);
  double* acc = c->acc_p2p.ensure(3 * n);
  const P2PItem* items = reinterpret_cast<const P2PItem*>(c->p2p_items.p);
  if (c->n_p2p_items > 0) {
    if (c->cfg.precision == FMM_PREC_FP32_P2P) {
      const P2PEnt* ent = reinterpret_cast<const P2PEnt*>(c->p2p_ent.p);
      // narrow CTAs (64 consumer threads, 512-body tiles, 10 per SM) when the items are short
      // (A/B: C5 4.90 -> 4.46 ms; C3 3.73 -> 4.08, C2 2.78 -> 3.06: wide there); fmm_set_p2p_shape or
      // FMM_P2P_SMALL=0/1 override the choice
      static const int small_env = [] {
        const char* e = getenv("FMM_P2P_SMALL");
        return e ? atoi(e) : -1;
      }();
      // few source bodies per target body = items of ~3 tiles (C5: 1 450; C1-C4: 3 300-17 000)
      const double targets = static_cast<double>(c->world > 1 ? c->shard_b1 - c->shard_b0 : n);
      const bool small =
          c->p2p_shape >= 0 ? c->p2p_shape != 0
          : small_env >= 0 ? small_env != 0
                           : static_cast<double>(c->p2p_body_pairs) < kSmallSourcesPerTarget * targets;
      auto launch = [&](auto kern, int threads) {
        kern<<<(unsigned)c->n_p2p_items, threads, 0, s>>>(items, ent, c->bodyf.p, c->bodyl.p, phi, acc, c->p2p_partial.p);
      };
      if (wa && small) launch(k_p2p_fp32_ws<true, kSmallCT, kSmallTB>, kSmallCT + 32);
      else if (wa) launch(k_p2p_fp32_ws<true, kThreads, kTileBodies>, kWsThreads);
      else if (small) launch(k_p2p_fp32_ws<false, kSmallCT, kSmallTB>, kSmallCT + 32);
      else launch(k_p2p_fp32_ws<false, kThreads, kTileBodies>, kWsThreads);
    } else {
      k_p2p_fp64<<<(unsigned)c->n_p2p_items, kThreads, 0, s>>>(items, c->p2p_src.p, c->c_body_begin.p, c->c_body_end.p,
                                                              c->bodies.p, phi, acc, c->p2p_partial.p, wa);
    }
    CK_LAUNCH("k_p2p");
    c->kernel_launches += 1;
  }
  if (c->n_p2p_reduce > 0) {
    k_p2p_reduce<<<(unsigned)c->n_p2p_reduce, 128, 0, s>>>(c->p2p_reduce.p, c->n_p2p_reduce, c->p2p_partial.p, phi,
                                                          acc, wa);
    CK_LAUNCH("k_p2p_reduce");
    c->kernel_launches += 1;
  }
}

}  // namespace fmmb

namespace fmmb {
namespace {
// Operator-level P2P (kernels.cpp:181-192 + acc) over (target range, source range) pairs of one
// body array; thread per target body. FP32 mode: coordinates relative to the target range's
// first body, FP32 pair math, FP64 accumulation (the arithmetic of k_p2p_fp32_ws's far tiles).
__global__ void k_op_p2p(int64_t count, const int4* __restrict__ rng, const double4* __restrict__ b,
                         int precision, double* __restrict__ phi, double* __restrict__ acc) {
  const int64_t r = blockIdx.x;
  if (r >= count) return;
  const int4 g = rng[r];
  for (int32_t i = g.x + threadIdx.x; i < g.y; i += blockDim.x) {
    const double4 t = b[i];
    double ph = 0.0, ax = 0.0, ay = 0.0, az = 0.0;
    for (int32_t j = g.z; j < g.w; ++j) {
      const double4 s = b[j];
      if (precision == FMM_PREC_FP64) {
        const double dx = t.x - s.x, dy = t.y - s.y, dz = t.z - s.z;
        const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
        if (r2 == 0.0) continue;
        const double ri = 1.0 / sqrt(r2), qr = s.w * ri, qr3 = qr * ri * ri;
        ph += qr;
        ax += dx * qr3;
        ay += dy * qr3;
        az += dz * qr3;
      } else {
        const double4 o = b[g.x];
        const float dx = static_cast<float>(t.x - o.x) - static_cast<float>(s.x - o.x);
        const float dy = static_cast<float>(t.y - o.y) - static_cast<float>(s.y - o.y);
        const float dz = static_cast<float>(t.z - o.z) - static_cast<float>(s.z - o.z);
        const float r2 = dx * dx + dy * dy + dz * dz;
        const float ri = r2 > 0.f ? rsqrtf(r2) : 0.f;
        const float qr = static_cast<float>(s.w) * ri, qr3 = qr * ri * ri;
        ph += qr;
        ax += dx * qr3;
        ay += dy * qr3;
        az += dz * qr3;
      }
    }
    phi[i] += ph;
    if (acc) {
      acc[3 * i] += ax;
      acc[3 * i + 1] += ay;
      acc[3 * i + 2] += az;
    }
  }
}
}  // namespace

void op_p2p(int64_t count, const int32_t* ranges4, const double* xyzq, int64_t nbodies, int precision,
            double* phi, double* acc) {
  if (count <= 0 || nbodies <= 0) return;
  int4* r = nullptr;
  double4* b = nullptr;
  double *p = nullptr, *a = nullptr;
  CK(cudaMalloc(&r, count * sizeof(int4)));
  CK(cudaMalloc(&b, nbodies * sizeof(double4)));
  CK(cudaMalloc(&p, nbodies * sizeof(double)));
  CK(cudaMalloc(&a, nbodies * 3 * sizeof(double)));
  CK(cudaMemcpy(r, ranges4, count * sizeof(int4), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(b, xyzq, nbodies * sizeof(double4), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(p, phi, nbodies * sizeof(double), cudaMemcpyHostToDevice));
  if (acc) CK(cudaMemcpy(a, acc, nbodies * 3 * sizeof(double), cudaMemcpyHostToDevice));
  k_op_p2p<<<(unsigned)count, 64>>>(count, r, b, precision, p, acc ? a : nullptr);
  CK_LAUNCH("op_p2p");
  CK(cudaMemcpy(phi, p, nbodies * sizeof(double), cudaMemcpyDeviceToHost));
  if (acc) CK(cudaMemcpy(acc, a, nbodies * 3 * sizeof(double), cudaMemcpyDeviceToHost));
  cudaFree(r);
  cudaFree(b);
  cudaFree(p);
  cudaFree(a);
}
}  // namespace fmmb

#if FMM_P2P_TRACE
extern "C" int fmm_debug_p2p_trace(unsigned long long* out, int nctas) {
  const size_t bytes = sizeof(unsigned long long) * 16 * static_cast<size_t>(nctas);
  return cudaMemcpyFromSymbol(out, fmmb::g_p2p_trace, bytes) == cudaSuccess ? 0 : 1;
}
#endif
