// trace.cu — the hot path: first-hit primary-ray intersection through a hybrid format.
//
// One thread per ray (north_star). The paper's generated intersection code is one function
// per level (§4.2; fig:function_proto PAPER.md:182-186):
//     intersect(node_id, ray, low):
//       for child in ordered_hit_children(node_id, ray):
//         if child and next_intersect(child, ray, low + child.pos): return True
//       return False
// with Raw levels walked by a branchless Amanatides-Woo DDA, SVO / SVDAG
// levels by a pre-order traversal with a per-thread stack or, with
// "restarting sparse voxel intersection", from the sub-volume root for every lookup
// (PAPER.md:215), a unit function for single voxels and a root function that reads word 0
// and tests the root box.
//
// B200 design (not a translation of the GLSL): the recursion is flattened into ONE loop over a
// per-thread tier index, so lanes of a warp that sit at different levels still execute the
// same instruction stream; each tier's kind-specific work is one `switch` arm instantiated only
// for the base formats present (template parameter KINDS, the compile-time composition of the
// level templates). Per-tier geometry is packed into 64-bit fields of TraceParams and
// extracted with shifts (no indexed memory). Node headers are fetched with one vector load
// (SVO: LDG.64, N^3-tree: LDG.128); inside an SVO / SVDAG / N^3 node, empty cells cost no
// memory access (the occupancy mask stays in registers).
//
// Exactness (SURVEY.md §8(c) "How the GPU matches it"): the DDA never accumulates t. Every plane
// event time is recomputed as  T^ = fl(fl(P - o_a) * inv_a),  inv_a = RN(1/d_a), |T^-T| <= ~3u|T|.
// Every ordering decision (next axis to step, ties, entry cell, descent child, t_end) compares
// two events with a certified fp32 test (gap > 2^-20 * max) and, if that fails, an exact fp64
// fallback (P - o is exact in fp64 in the canonical domain; products use FMA TwoProduct).
// The current time is carried as an EVENT {axis, plane} (or tmin) so the exact fallback can
// always reconstruct it. The finest-voxel coordinate V of the current cell is kept exactly;
// after a step at a coarse tier the sub-cell bits of the non-stepped axes are "stale" and are
// re-derived (certified) only when the traversal descends at that event. Hence the hierarchy
// visits exactly the cells of the flat right-limit walk (the oracle's definition) and
// returns the same voxel, bit for bit.
#include <stdint.h>

#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <mutex>

#include <type_traits>
#include <vector>

#include "vf_internal.cuh"

namespace vf {
namespace {

constexpr float kCertEps = 0x1p-20f;  // certification margin (>= 8u with u = 2^-24; see header)
constexpr int TMIN_AXIS = 3;

// One thread per ray, 128-thread blocks; register caps (__launch_bounds__ min blocks per SM)
#ifndef VF_MINB
#define VF_MINB 8  // __launch_bounds__ min blocks per SM (register cap), A/B-tuned
#endif
#ifndef VF_MINB_SPEC
#define VF_MINB_SPEC 9  // compiled-in formats: 56 registers, 9 blocks per SM (A/B: +1.4-2.2 % over 8)
#endif
#ifndef VF_CHAIN_TOPNTREE
#define VF_CHAIN_TOPNTREE 0  // restart descent chain for [R(A^3)] T(n, d) (A/B: -3 to -10 %)
#endif
#ifndef VF_CHAIN_TWOSPARSE
#define VF_CHAIN_TWOSPARSE 1  // restart descent chain for S(a) G(b) without a Raw top (A/B: +5 to +11 %;
                              // with R(4^3) on top -4 %)
#endif
#ifndef VF_MINB_CHAIN
#define VF_MINB_CHAIN 8  // compiled-in chains of several Raw / DF levels
#endif

struct Ray {
  float o[3], d[3], inv[3];
  float tmin, tmax;
};

struct Event {
  int axis;  // 0..2 plane event on that axis; TMIN_AXIS = tmin (start of the segment)
  int P;     // plane coordinate in voxels (integer)
  float t;   // fl(fl(P - o) * inv)  (or tmin)
};

__device__ __forceinline__ float tplane(int P, float o, float inv) { return __fmul_rn(__fsub_rn((float)P, o), inv); }

// Select v[i] for a run-time i without indexed (local-memory) access.
template <class T>
__device__ __forceinline__ T sel3(const T (&v)[3], int i) {
  return i == 0 ? v[0] : (i == 1 ? v[1] : v[2]);
}

// ---- exact fallbacks (rare; kept out of line) -------------------------------------------
// Number of exact fallbacks executed (statistic for the certified-filter miss rate).
__device__ unsigned long long g_exact_calls;

// sign(T_a(P) - T_b(Q)) for d_a, d_b != 0, exactly.
__device__ __forceinline__ int cmp_pp_exact(int P, float oa, float da, int Q, float ob, float db) {
  atomicAdd(&g_exact_calls, 1ull);
  const double A = (double)P - (double)oa;  // exact (<= 52 significant bits in the domain)
  const double B = (double)Q - (double)ob;
  const double x = A * (double)db, xe = fma(A, (double)db, -x);  // TwoProduct: A*db = x + xe
  const double y = B * (double)da, ye = fma(B, (double)da, -y);
  int s = (x > y) - (x < y);
  if (s == 0) s = (xe > ye) - (xe < ye);
  return ((da > 0.f) == (db > 0.f)) ? s : -s;  // T1 - T2 = (A db - B da) / (da db)
}
// sign(T_a(P) - s) for a scalar time s (tmin / tmax), exactly.
__device__ __forceinline__ int cmp_ps_exact(int P, float oa, float da, float s) {
  atomicAdd(&g_exact_calls, 1ull);
  const double A = (double)P - (double)oa;
  const double S = (double)s * (double)da;  // 24 x 24 bits: exact
  int r = (A > S) - (A < S);
  return da > 0.f ? r : -r;  // T - s = (A - s da) / da
}

__device__ __forceinline__ int cert(float t1, float t2) {
  const float df = t1 - t2;
  const float m = fmaxf(fabsf(t1), fabsf(t2)) * kCertEps;
  if (fabsf(df) > m) return df > 0.f ? 1 : -1;
  return 2;
}

// sign(T_a(P) - T_b(Q)) for two plane events on any axes (a == b compares the planes); t1 / t2
// are their fp32 values. o / d are the ray's origin and direction (indexed at run time only here,
// on the entry and slow paths).
__device__ __forceinline__ int cmp_pp(const float (&o)[3], const float (&d)[3], int a, int P, float t1, int b, int Q,
                                      float t2) {
  if (a == b) {
    const int s = (P > Q) - (P < Q);
    return sel3(d, a) > 0.f ? s : -s;
  }
  const int c = cert(t1, t2);
  if (c != 2) return c;
  return cmp_pp_exact(P, sel3(o, a), sel3(d, a), Q, sel3(o, b), sel3(d, b));
}

// sign(E - F) for two events given as {axis, plane, fp32 time}; axis TMIN_AXIS = the scalar t.
__device__ __forceinline__ int cmp_events(const float (&o)[3], const float (&d)[3], int ea, int eP, float et, int fa,
                                          int fP, float ft) {
  if (fa == TMIN_AXIS) {
    if (ea == TMIN_AXIS) return (et > ft) - (et < ft);
    const int c = cert(et, ft);
    if (c != 2) return c;
    return cmp_ps_exact(eP, sel3(o, ea), sel3(d, ea), ft);
  }
  if (ea == TMIN_AXIS) {
    const int c = cert(et, ft);
    if (c != 2) return c;
    return -cmp_ps_exact(fP, sel3(o, fa), sel3(d, fa), et);
  }
  return cmp_pp(o, d, ea, eP, et, fa, fP, ft);
}

// Exact argmin of the three next-plane events (ties step together). c = candidate mask (>= 2
// bits). Returns the set of minimal axes | (one minimal axis << 4).
__device__ __noinline__ int argmin_exact(float o0, float o1, float o2, float d0, float d1, float d2, int P0, int P1,
                                         int P2, float t0, float t1, float t2, int c) {
  const float o[3] = {o0, o1, o2}, d[3] = {d0, d1, d2}, t[3] = {t0, t1, t2};
  const int P[3] = {P0, P1, P2};
  int best = __ffs(c) - 1;
  int set = 1 << best;
#pragma unroll
  for (int a = 1; a < 3; ++a) {
    if (a <= best || !((c >> a) & 1)) continue;
    // a != best: different axes
    int s;
    const int cc = cert(t[a], sel3(t, best));
    if (cc != 2)
      s = cc;
    else
      s = cmp_pp_exact(P[a], o[a], d[a], sel3(P, best), sel3(o, best), sel3(d, best));
    if (s < 0) {
      best = a;
      set = 1 << a;
    } else if (s == 0) {
      set |= 1 << a;
    }
  }
  return set | (best << 4);
}

// Certified correction of a sub-cell locate when the fast path cannot decide (ray on / near a
// plane at the event E; ~0.2 % of locates). Out of line and with scalar arguments only, so the
// hot loop stays compact and the lane state stays in registers. Finds k in [lo, hi] with
//   d_b > 0: T_b(k) <= E < T_b(k+1);   d_b < 0: T_b(k+1) <= E < T_b(k)
// by certified comparisons of E = {axis ea, plane eP (or tmin: ea = TMIN_AXIS), fp32 value et}
// against plane events of axis b (b != ea: the event axis is never located).
__device__ __noinline__ int locate_slow(float ob, float db, float invb, int lo, int hi, int ea, int eP, float et,
                                        float oe, float de) {
  // sign(E - T_b(Q))
  auto cmp = [&](int Q) {
    const float tq = tplane(Q, ob, invb);
    const int c = cert(et, tq);
    if (c != 2) return c;
    if (ea == TMIN_AXIS) return -cmp_ps_exact(Q, ob, db, et);
    return cmp_pp_exact(eP, oe, de, Q, ob, db);
  };
  const float x = fmaf(et, db, ob);
  const float fl = floorf(x);
  float kf = db > 0.f ? fl : ceilf(x) - 1.0f;
  kf = fminf(fmaxf(kf, (float)lo), (float)hi);
  int k = (int)kf;
  if (db > 0.f) {
    for (;;) {
      if (k > lo && cmp(k) < 0) {
        --k;
        continue;
      }
      if (k < hi && cmp(k + 1) >= 0) {
        ++k;
        continue;
      }
      break;
    }
  } else {
    for (;;) {
      if (k < hi && cmp(k + 1) < 0) {
        ++k;
        continue;
      }
      if (k > lo && cmp(k) >= 0) {
        --k;
        continue;
      }
      break;
    }
  }
  return k;
}

__device__ __forceinline__ uint32_t field4(uint64_t pack, uint32_t i) { return (uint32_t)(pack >> (4 * i)) & 15u; }

template <uint32_t KINDS>
__device__ __forceinline__ bool has_kind(uint32_t k) {
  return (KINDS >> k) & 1u;
}

__device__ __forceinline__ uint32_t twf(uint32_t w, uint32_t pos, uint32_t len) { return (w >> pos) & ((1u << len) - 1u); }

// Node header registers for the current tier. The occupancy mask is 64-bit only when an N^3-tree
// tier is present (SVO / SVDAG masks are 8-bit: one POPC instead of two on the hot path).
// ALN (buffers built with VF_BUILD_ALIGN_NODES): an SVDAG node's header load is one aligned
// LDG.128 that also brings its first three child pointers (kept in base, p1, p2).
template <bool ALN>
struct HeaderPtrs {};
template <>
struct HeaderPtrs<true> {
  uint32_t p1, p2;
};
template <uint32_t KINDS, bool ALN = false>
struct Header : HeaderPtrs<ALN> {
  using Mask = typename std::conditional<((KINDS >> K_NTREE) & 1u) != 0, uint64_t, uint32_t>::type;
  Mask mask;      // SVO/SVDAG: valid bits; N^3: 64-bit occupancy
  uint32_t base;  // SVO: first child; N^3: children block; SVDAG + ALN: child pointer 0
  __device__ __forceinline__ uint32_t rank(uint32_t lin) const {
    if constexpr (sizeof(Mask) == 8)
      return __popcll(mask & ((1ull << lin) - 1ull));
    else
      return __popc(mask & ((1u << lin) - 1u));
  }
};

// Per-ray work counters of the VF_COUNTERS variant (SURVEY.md §8(d) "Counts come from a
// -DVF_COUNTERS build of the same kernel"). Compiled away when COUNT == false.
template <bool COUNT>
struct Ctr {
  uint32_t v[VF_NCOUNTERS];
  __device__ __forceinline__ Ctr() {
    if (COUNT)
#pragma unroll
      for (int i = 0; i < VF_NCOUNTERS; ++i) v[i] = 0;
  }
  uint32_t* touch_map = nullptr;  // counting launches: one bit per format word
  __device__ __forceinline__ void add(int i, uint32_t x = 1) {
    if (COUNT) v[i] += x;
  }
  // A format load of nw words at word address a: sectors spanned, and the words in the bitmap.
  __device__ __forceinline__ void touch(size_t a, uint32_t nw) {
    if constexpr (COUNT) {
      v[VF_CTR_SECTOR_READS] += (uint32_t)(((a + nw - 1) >> 3) - (a >> 3) + 1);
      if (touch_map)
        for (uint32_t i = 0; i < nw; ++i) atomicOr(touch_map + ((a + i) >> 5), 1u << ((a + i) & 31));
    }
  }
  __device__ __forceinline__ void flush(unsigned long long* out) {
    if constexpr (COUNT) {
      const uint32_t wmax = __reduce_max_sync(0xffffffffu, v[VF_CTR_CELL_TESTS]);
      v[VF_CTR_WARP_MAX_TESTS] = (threadIdx.x & 31) == 0 ? 32u * wmax : 0u;
#pragma unroll
      for (int i = 0; i < VF_NCOUNTERS; ++i) {
        unsigned long long x = v[i];
        for (int o = 16; o; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
        if ((threadIdx.x & 31) == 0 && x) atomicAdd(out + i, x);
      }
    }
  }
};

// Read the header of node N of a tier of the given kind into h (a Raw tier has none).
template <uint32_t KINDS, bool COUNT, bool ALN>
__device__ __forceinline__ void load_header(const uint32_t* __restrict__ buf, uint32_t kind, uint32_t N,
                                            Header<KINDS, ALN>& h, Ctr<COUNT>& ct) {
  if (has_kind<KINDS>(K_SVO) && kind == K_SVO) {
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(buf + N));
    h.base = v.x;
    h.mask = v.y;  // valid bits 0-7 (leaf bits 8-15 are never indexed: cell indices are < 8)
    ct.add(VF_CTR_SVO_NODES);
    ct.add(VF_CTR_FORMAT_BYTES, 8);
    ct.touch(N, 2);
  } else if (has_kind<KINDS>(K_SVDAG) && kind == K_SVDAG) {
    if constexpr (ALN) {  // 16-B aligned node: mask + child pointers 0..2 in one vector load
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(buf + N));
      h.mask = v.x;
      h.base = v.y;
      h.p1 = v.z;
      h.p2 = v.w;
    } else {
      h.mask = __ldg(buf + N);  // valid bits 0-7 (leaf bits 8-15 never indexed)
    }
    ct.add(VF_CTR_SVDAG_NODES);
    ct.add(VF_CTR_FORMAT_BYTES, 4);
    ct.touch(N, 1);
  } else if (has_kind<KINDS>(K_NTREE) && kind == K_NTREE) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(buf + N));
    h.mask = (typename Header<KINDS>::Mask)((uint64_t)v.x | ((uint64_t)v.y << 32));
    h.base = v.z;
    ct.add(VF_CTR_NTREE_NODES);
    ct.add(VF_CTR_FORMAT_BYTES, 16);
    ct.touch(N, 4);
  }
}

// ---- compiled-in formats (the paper's per-format generated code, §4, as template instances) --
// A format descriptor D gives the tier geometry and flags as functions of the tier index t:
//   NoSpec          — generic: read from the tier table (any format)
//   TopSparse<...>  — optional Raw top over one uniform sparse level: R(A^3) G(M), G(L), T(n,d), ...
//   SparseRaw<...>  — NS uniform sparse tiers (one kind, one fan-out) over a Raw bottom level
// (pure arithmetic in t; a packed compile-time table variant measured 2-8 % slower)
struct NoSpec {
  static constexpr bool kStatic = false;
  static constexpr int kLogDim = -1;  // log2 of the (cubic) resolution when compiled in; -1: p.dims
  static constexpr bool kHasDF = true;  // some tier may be a DF grid
  static constexpr int kMinBlocks = VF_MINB;  // __launch_bounds__ min blocks per SM (register cap)
  static constexpr bool kIdx64 = true;        // Raw cell addresses may reach 2^32 words
  static constexpr bool kCacheGeom = false;   // compiled-in tier geometry cached in registers
  static constexpr bool kChainRestart = false; // restart variant: descents chained before each step
  static constexpr uint32_t kTopWords = 0;  // words of a stageable top Raw grid (0: none)
};

// An optional cubic Raw top level R(A^3) (A = 0: none) over one sparse level of NS tiers of one
// kind with per-axis fan-out 2^LF each (SVO / SVDAG: LF = 1, N^3: LF = n): R(A^3) G(M), G(L),
// S(L), T(n, d), R(A^3) T(n, d), ... lc = LF (NS + off - 1 - t), off = (A > 0).
template <uint32_t A, uint32_t KIND, uint32_t LF, uint32_t NS, bool DFTOP = false>
struct TopSparse {
  static constexpr bool kStatic = true;
  static constexpr uint32_t kTopWords = (A > 0 && A <= 4 && !DFTOP) ? (1u << (3 * A)) : 0u;
  // DFTOP: the top level is a DF grid D(A^3, M) (2-word cells {TermInt, L1 distance})
  __device__ static __forceinline__ bool df(int t) { return DFTOP && A > 0 && t == 0; }
  static constexpr int OFF = A > 0 ? 1 : 0;
  static constexpr int NT = (int)NS + OFF;
  static constexpr int kLogDim = (int)(A + LF * NS);
  static constexpr bool kHasDF = DFTOP;
  static constexpr int kMinBlocks = VF_MINB_SPEC;
  static constexpr bool kIdx64 = false;
  static constexpr bool kCacheGeom = false;
  static constexpr bool kChainRestart = KIND != K_NTREE || VF_CHAIN_TOPNTREE;  // A/B: restart +2.7 % cfg5, +8.8 % cfg4
  __device__ static __forceinline__ bool raw(int t) { return A > 0 && t == 0; }
  __device__ static __forceinline__ uint32_t lc(int t) { return LF * (uint32_t)(NT - 1 - t); }
  __device__ static __forceinline__ uint32_t msk(int t) { return raw(t) ? (1u << A) - 1u : (1u << LF) - 1u; }
  __device__ static __forceinline__ uint32_t sx(int t) { return raw(t) ? A : LF; }
  __device__ static __forceinline__ uint32_t sxy(int t) { return raw(t) ? 2u * A : 2u * LF; }
  __device__ static __forceinline__ uint32_t kind(int t) { return raw(t) ? (uint32_t)K_RAW : KIND; }
  __device__ static __forceinline__ bool finest(int t) { return t == NT - 1; }
  __device__ static __forceinline__ bool last(int t) { return raw(t) || t == NT - 1; }
  __device__ static __forceinline__ bool top(int t) { return t <= OFF; }
  __device__ static __forceinline__ uint32_t lcp(int t) { return t == 0 ? 15u : LF * (uint32_t)(NT - t); }
  // deepest tau in [1, NT - 1] with lc(tau - 1) = LF (NT - tau) > h; 0 if none
  __device__ static __forceinline__ int tau(uint32_t h) {
    const int tu = NT - 1 - (int)(h / LF);
    return tu > 0 ? tu : 0;
  }
  __device__ static __forceinline__ int level_top(int tu) { return tu == 0 ? 0 : OFF; }
};
template <uint32_t A, uint32_t M>
using RawSvdag = TopSparse<A, K_SVDAG, 1, M>;

// NR (1..3) cubic Raw / DF levels R(A0^3) R(A1^3) R(A2^3) (bit t of DFM: tier t is a DF grid) over
// an optional octree level of NS tiers (kind KIND; NS = 0: none): R(4^3) R(3^3) G(4),
// R(3^3) R(3^3) R(3^3), D(5^3, 6) R(4^3), R(11^3), ... Raw tier geometry from compile-time constants.
template <uint32_t NR, uint32_t A0, uint32_t A1, uint32_t A2, uint32_t DFM, uint32_t KIND, uint32_t NS>
struct RawChain {
  static constexpr bool kStatic = true;
  static constexpr uint32_t kTopWords = 0;
  static constexpr int NT = (int)(NR + NS);
  static constexpr int kLogDim = (int)(A0 + (NR > 1 ? A1 : 0u) + (NR > 2 ? A2 : 0u) + NS);
  static constexpr bool kHasDF = DFM != 0;
  // several Raw / DF tiers keep more geometry live: a looser register cap (A/B: VF_MINB_CHAIN)
  static constexpr int kMinBlocks = NR > 1 ? VF_MINB_CHAIN : VF_MINB_SPEC;
  static constexpr bool kIdx64 = NR == 1 && NS == 0 && A0 >= 10;  // a single grid of 2^30+ cells
  // several Raw tiers: their geometry is a chain of selects on t; cache it per tier change instead
#ifndef VF_CHAIN_CACHE
#define VF_CHAIN_CACHE 1
#endif
  static constexpr bool kCacheGeom = NR > 1 && VF_CHAIN_CACHE;
  static constexpr bool kChainRestart = false;  // A/B: R R G restart -1 to -4 % with the chain
  static constexpr uint32_t L2 = NS, L1 = NS + (NR > 2 ? A2 : 0u), L0 = L1 + (NR > 1 ? A1 : 0u);  // lc of raw tiers
  __host__ __device__ static constexpr uint32_t LCR(int t) { return t == 0 ? (NR == 1 ? NS : NR == 2 ? NS + A1 : L0) : t == 1 ? (NR == 2 ? NS : L1) : L2; }
  __device__ static __forceinline__ bool raw(int t) { return t < (int)NR; }
  __device__ static __forceinline__ bool df(int t) { return raw(t) && ((DFM >> t) & 1u); }
  __device__ static __forceinline__ uint32_t lc(int t) {
    return raw(t) ? (t == 0 ? LCR(0) : t == 1 ? LCR(1) : LCR(2)) : (uint32_t)(NT - 1 - t);
  }
  __device__ static __forceinline__ uint32_t araw(int t) { return t == 0 ? A0 : t == 1 ? A1 : A2; }
  __device__ static __forceinline__ uint32_t msk(int t) { return raw(t) ? (1u << araw(t)) - 1u : 1u; }
  __device__ static __forceinline__ uint32_t sx(int t) { return raw(t) ? araw(t) : 1u; }
  __device__ static __forceinline__ uint32_t sxy(int t) { return raw(t) ? 2u * araw(t) : 2u; }
  __device__ static __forceinline__ uint32_t kind(int t) { return raw(t) ? (uint32_t)K_RAW : KIND; }
  __device__ static __forceinline__ bool finest(int t) { return t == NT - 1; }
  __device__ static __forceinline__ bool last(int t) { return raw(t) || t == NT - 1; }
  __device__ static __forceinline__ bool top(int t) { return t <= (int)NR; }
  __device__ static __forceinline__ uint32_t lcp(int t) { return t == 0 ? 15u : lc(t - 1); }
  // deepest tau in [1, NT - 1] with lc(tau - 1) > h; 0 if none
  __device__ static __forceinline__ int tau(uint32_t h) {
    const int ts = NT - 1 - (int)h;  // within the octree level: lc(tau - 1) = NT - tau
    if (NS > 0 && ts - 1 >= (int)NR) return ts;
    if (NR >= 3 && (int)LCR(2) > (int)h && NT - 1 >= 3) return 3;
    if (NR >= 2 && (int)LCR(1) > (int)h && NT - 1 >= 2) return 2;
    if ((int)LCR(0) > (int)h && NT - 1 >= 1) return 1;
    return 0;
  }
  __device__ static __forceinline__ int level_top(int tu) { return tu < (int)NR ? tu : (int)NR; }
};

// An optional cubic Raw top R(A^3) over two octree levels (SVO / SVDAG) of N1 then N2 tiers:
// S(a) G(b), R(A^3) S(a) G(b), ... — uniform 2x2x2 tiers below the top, lc = NT - 1 - t.
template <uint32_t A, uint32_t K1, uint32_t N1, uint32_t K2, uint32_t N2>
struct TwoSparse {
  static constexpr bool kStatic = true;
  static constexpr uint32_t kTopWords = 0;
  __device__ static __forceinline__ bool df(int) { return false; }
  static constexpr int OFF = A > 0 ? 1 : 0;
  static constexpr int B = OFF + (int)N1;  // first tier of the second sparse level
  static constexpr int NT = B + (int)N2;
  static constexpr int kLogDim = (int)(A + N1 + N2);
  static constexpr bool kHasDF = false;
  static constexpr int kMinBlocks = VF_MINB_SPEC;
  static constexpr bool kIdx64 = false;
  static constexpr bool kCacheGeom = false;
  static constexpr bool kChainRestart = VF_CHAIN_TWOSPARSE && A == 0;
  __device__ static __forceinline__ bool raw(int t) { return A > 0 && t == 0; }
  __device__ static __forceinline__ uint32_t lc(int t) { return (uint32_t)(NT - 1 - t); }
  __device__ static __forceinline__ uint32_t msk(int t) { return raw(t) ? (1u << A) - 1u : 1u; }
  __device__ static __forceinline__ uint32_t sx(int t) { return raw(t) ? A : 1u; }
  __device__ static __forceinline__ uint32_t sxy(int t) { return raw(t) ? 2u * A : 2u; }
  __device__ static __forceinline__ uint32_t kind(int t) { return raw(t) ? (uint32_t)K_RAW : (t < B ? K1 : K2); }
  __device__ static __forceinline__ bool finest(int t) { return t == NT - 1; }
  __device__ static __forceinline__ bool last(int t) { return raw(t) || t == B - 1 || t == NT - 1; }
  __device__ static __forceinline__ bool top(int t) { return t <= OFF || t == B; }
  __device__ static __forceinline__ uint32_t lcp(int t) { return t == 0 ? 15u : (uint32_t)(NT - t); }
  __device__ static __forceinline__ int tau(uint32_t h) {
    const int tu = NT - 1 - (int)h;
    return tu > 0 ? tu : 0;
  }
  __device__ static __forceinline__ int level_top(int tu) { return tu == 0 ? 0 : (tu < B ? OFF : B); }
};

// NS sparse tiers of one kind with per-axis fan-out 2^LF each (SVO / SVDAG: LF = 1, N^3: LF = n)
// over a cubic Raw bottom level R(A^3); bit t of LASTM / TOPM: sparse tier t is the last / first
// tier of its level. All geometry is arithmetic in t (cfg2 G(5) R(3^3), cfg3 T(2,2) T(2,1) R(4^3)).
template <uint32_t KIND, uint32_t LF, uint32_t NS, uint32_t A, uint32_t LASTM, uint32_t TOPM>
struct SparseRaw {
  static constexpr bool kStatic = true;
  static constexpr uint32_t kTopWords = 0;
  __device__ static __forceinline__ bool df(int) { return false; }
  static constexpr uint32_t LC0 = LF * (NS - 1) + A;  // lc of tier 0
  static constexpr int kLogDim = (int)(LF * NS + A);
  static constexpr bool kHasDF = false;
  static constexpr int kMinBlocks = VF_MINB_SPEC;
  static constexpr bool kIdx64 = false;
  static constexpr bool kCacheGeom = false;
  static constexpr bool kChainRestart = false;  // A/B: cfg2 -10 %, cfg3 -16 % restart with the chain
  __device__ static __forceinline__ uint32_t lc(int t) { return t == (int)NS ? 0u : LC0 - LF * (uint32_t)t; }
  __device__ static __forceinline__ uint32_t msk(int t) { return t == (int)NS ? (1u << A) - 1u : (1u << LF) - 1u; }
  __device__ static __forceinline__ uint32_t sx(int t) { return t == (int)NS ? A : LF; }
  __device__ static __forceinline__ uint32_t sxy(int t) { return t == (int)NS ? 2u * A : 2u * LF; }
  __device__ static __forceinline__ uint32_t kind(int t) { return t == (int)NS ? (uint32_t)K_RAW : KIND; }
  __device__ static __forceinline__ bool finest(int t) { return t == (int)NS; }
  __device__ static __forceinline__ bool last(int t) { return t == (int)NS || ((LASTM >> t) & 1u); }
  __device__ static __forceinline__ bool top(int t) { return t == (int)NS || ((TOPM >> t) & 1u); }
  __device__ static __forceinline__ uint32_t lcp(int t) { return t == 0 ? 15u : LC0 + LF - LF * (uint32_t)t; }
  // deepest tau in [1, NS] with lc(tau - 1) = LF (NS - tau) + A > h; 0 if none
  __device__ static __forceinline__ int tau(uint32_t h) {
    if (h < A) return (int)NS;
    const int tu = (int)NS - 1 - (int)((h - A) / LF);
    return tu > 0 ? tu : 0;
  }
  __device__ static __forceinline__ int level_top(int tu) {
    return tu == (int)NS ? (int)NS : 31 - __clz(TOPM & ((2u << tu) - 1u));
  }
};

constexpr uint32_t VF_NONE = 0, K_OF_VF_NONE = 0;  // RawChain without an octree level
constexpr uint32_t K_OF_VF_SVO = K_SVO, K_OF_VF_SVDAG = K_SVDAG, K_OF_VF_NTREE = K_NTREE;

struct LevelSpec {
  uint32_t kind, lf, depth;  // VF_RAW / VF_SVO / VF_SVDAG / VF_NTREE, log2 fan-out per axis, tiers
};

enum { IT_CONTINUE = 0, IT_HIT = 1, IT_MISS = 2 };

// The per-ray traversal state machine: start() is the root function, iterate() is one cell test
// followed by either a descent or one DDA step (with pop / restart when the step leaves a node).
// The current tier's packed word (TraceParams::tword, staged in shared memory) and the fields
// the cell test needs are cached in registers and refreshed only when the tier changes.
//
// The current event E (the time the ray entered the current cell) is {eaxis, et}: a plane event
// on axis eaxis, or tmin (eaxis = TMIN_AXIS). Its plane is not stored: the cell entered through
// it is V[eaxis], so the plane is V[eaxis] + (d < 0) — the event axis never goes stale, and
// descents and pops do not move V. The exact fallbacks rebuild it from there.
//
// D (a format descriptor above) compiles the format in: with D::kStatic the tier geometry and
// flags are functions of the tier index (no tier table, fewer live registers).
template <uint32_t KINDS, bool RESTART, bool COUNT, class D = NoSpec, bool STAGE = false, bool ALN = false>
struct Lane {
  static constexpr bool SPEC = D::kStatic;
  const uint32_t* s_top;  // STAGE: the top Raw grid (tier 0's node, D::kTopWords words) in shared memory
  float o[3], d[3], inv[3];  // inv = RN(1/d); +inf on axes with d = 0 (their next plane is never)
  float tmax;
  int V[3];       // finest voxel of the current cell (bits below lc(t) valid unless stale)
  int eaxis;      // current event: axis of the plane crossed (TMIN_AXIS: the segment start)
  float et;       // its fp32 time fl(fl(P - o) * inv) (or tmin)
  int t;          // current tier
  uint32_t N;     // current node (word address)
  uint32_t tw;    // tier word of tier t (generic formats)
  uint32_t lc_, msk_, sx_, sxy_;  // decoded from tw (generic formats)

  // tier geometry and flags of tier t
  __device__ __forceinline__ uint32_t lc() const {
    if constexpr (SPEC && !D::kCacheGeom) return D::lc(t); else return lc_;
  }
  __device__ __forceinline__ uint32_t msk() const {
    if constexpr (SPEC && !D::kCacheGeom) return D::msk(t); else return msk_;
  }
  __device__ __forceinline__ uint32_t sx() const {
    if constexpr (SPEC && !D::kCacheGeom) return D::sx(t); else return sx_;
  }
  __device__ __forceinline__ uint32_t sxy() const {
    if constexpr (SPEC && !D::kCacheGeom) return D::sxy(t); else return sxy_;
  }
  __device__ __forceinline__ uint32_t kind() const {
    if constexpr (SPEC) return D::kind(t); else return tw & 3u;
  }
  __device__ __forceinline__ bool finest() const {
    if constexpr (SPEC) return D::finest(t); else return (tw & TW_FINEST) != 0;
  }
  __device__ __forceinline__ bool last() const {
    if constexpr (SPEC) return D::last(t); else return (tw & TW_LAST) != 0;
  }
  __device__ __forceinline__ bool is_df() const {
    if constexpr (SPEC) return D::df(t); else return (tw & TW_DF) != 0;
  }
  __device__ __forceinline__ bool is_top() const {
    if constexpr (SPEC) return D::top(t); else return (tw & TW_TOP) != 0;
  }
  __device__ __forceinline__ uint32_t lcp() const {
    if constexpr (SPEC) return D::lcp(t); else return twf(tw, TW_LCP, 4);
  }
  // deepest tier whose node holds two cells first differing at bit h; the top tier of its level
  __device__ __forceinline__ int tau(const TraceParams& p, uint32_t h) const {
    if constexpr (SPEC) return D::tau(h); else return (int)field4(p.tau_pack, h);
  }
  __device__ __forceinline__ int level_top(const TraceParams& p, int tu) const {
    if constexpr (SPEC) return D::level_top(tu);
    else return (int)field4(((uint64_t)p.level_top_pack_hi << 32) | p.level_top_pack_lo, tu);
  }

  Header<KINDS, ALN> hd;
  int stale;          // axes whose bits below stale_lc are not exact at E
  uint32_t stale_lc;  // bits of V below this are stale on the axes in `stale`
  int moving;         // axes with d != 0
  int dneg;           // axes with d < 0
  bool tmax_finite;
  int budget;  // DF tier: remaining L1 distance within which every cell is known empty
  // (the per-tier node stack lives outside the struct so that the struct itself can stay in
  //  registers: an indexed member would force the whole object into local memory)

  __device__ __forceinline__ int eplane() const { return sel3(V, eaxis) + ((dneg >> eaxis) & 1); }

  // sign(E - T_b(Q)) for a moving axis b (a compile-time constant at every hot call site).
  __device__ __forceinline__ int cmp_eq(int b, int Q) const {
    // (sel3, not o[b]: an index the compiler cannot resolve would move the lane to local memory)
    const float ob = sel3(o, b), db = sel3(d, b);
    if (eaxis == b) {
      const int P = sel3(V, b) + ((dneg >> b) & 1);
      const int s = (P > Q) - (P < Q);
      return db > 0.f ? s : -s;
    }
    const float tq = tplane(Q, ob, sel3(inv, b));
    const int c = cert(et, tq);
    if (c != 2) return c;
    if (eaxis == TMIN_AXIS) return -cmp_ps_exact(Q, ob, db, et);
    return cmp_pp_exact(eplane(), sel3(o, eaxis), sel3(d, eaxis), Q, ob, db);
  }

  // sign(E - s) for a scalar s (tmax).
  __device__ __forceinline__ int cmp_es(float s) const {
    if (eaxis == TMIN_AXIS) return (et > s) - (et < s);
    const int c = cert(et, s);
    if (c != 2) return c;
    return cmp_ps_exact(eplane(), sel3(o, eaxis), sel3(d, eaxis), s);
  }

  // Finest cell index on axis b at the current event E (right limit), known to lie in [lo, hi]:
  //   d_b > 0: T_b(k) <= E < T_b(k+1);   d_b < 0: T_b(k+1) <= E < T_b(k).
  // Fast path: x = o_b + T_E d_b is computed as x^ = fma(T^_E, d_b, o_b) with
  // |x^ - x| <= 3.01u|T d_b| + 1.01u|x^| (T^_E has relative error <= 3u, one rounding in the fma),
  // so B = 2^-21 (|T^ d_b| + |x^|) >= 8u(...) bounds it with margin. If [x^-B, x^+B] contains no
  // integer, x is not on a plane and tau_b(E+) = floor(x) = floor(x^) for either sign of d_b.
  // Otherwise (ray on / near a plane at E: ~0.2% of calls) the candidate is corrected with
  // certified plane comparisons (planes lo / hi+1 are known crossed / not crossed).
  __device__ __forceinline__ int locate(int b, int lo, int hi) const {
    const float db = sel3(d, b), ob = sel3(o, b);
    const float x = fmaf(et, db, ob);
    const float fl = floorf(x);
    const float f = x - fl;  // exact
    const float B = (fabsf(et * db) + fabsf(x)) * 0x1p-21f;
    int k = (int)fl;
    // (no range test: certified, floor(x^) is the exact tau_b(E+), and the ray is inside the cell
    //  [lo, hi] on axis b at E+ by the traversal invariant; the range only bounds the slow path)
    if (f > B && 1.0f - f > B) return k;
    return locate_slow(ob, db, sel3(inv, b), lo, hi, eaxis, eaxis == TMIN_AXIS ? 0 : eplane(),
                       et, eaxis == TMIN_AXIS ? 0.f : sel3(o, eaxis), eaxis == TMIN_AXIS ? 1.f : sel3(d, eaxis));
  }

  // s_tw: the tier table staged in shared memory, two uint4 per tier (stage_tiers): one LDS.128
  // and one LDS.32 per tier change instead of extracting the fields from the tier word.
  __device__ __forceinline__ void set_tier(const uint32_t* s_tw, int nt) {
    t = nt;
    if constexpr (!SPEC) {
      const uint4 a = reinterpret_cast<const uint4*>(s_tw)[2 * nt];
      tw = a.x;
      lc_ = a.y;
      msk_ = a.z;
      sx_ = a.w;
      sxy_ = s_tw[8 * nt + 4];
    } else if constexpr (D::kCacheGeom) {  // compiled-in, but cached in registers per tier change
      lc_ = D::lc(nt);
      msk_ = D::msk(nt);
      sx_ = D::sx(nt);
      sxy_ = D::sxy(nt);
    }
    budget = 0;
  }

  // ---- root function: word 0, root-box test, exact entry cell ---------------
  __device__ __forceinline__ bool start(const TraceParams& p, const uint32_t* __restrict__ buf,
                                        const uint32_t* s_tw, const float4 r0, const float4 r1, Ctr<COUNT>& ct) {
    o[0] = r0.x;
    o[1] = r0.y;
    o[2] = r0.z;
    const float tmin = r0.w;
    d[0] = r1.x;
    d[1] = r1.y;
    d[2] = r1.z;
    tmax = r1.w;
    tmax_finite = tmax < __int_as_float(0x7f800000);
    if (p.root == 0) return false;  // empty volume: buffer [0]
    // non-finite origin / direction / tmin or a NaN tmax: outside every reading of the domain, a miss
    // (the walk below assumes finite event times; vf.h "Rays")
    {
      const float inf = __int_as_float(0x7f800000);
      if (!(fabsf(o[0]) < inf && fabsf(o[1]) < inf && fabsf(o[2]) < inf && fabsf(d[0]) < inf && fabsf(d[1]) < inf &&
            fabsf(d[2]) < inf && fabsf(tmin) < inf && !(tmax != tmax)))
        return false;
    }
    moving = 0;
    dneg = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (d[a] != 0.f) moving |= 1 << a;
      if (d[a] < 0.f) dneg |= 1 << a;
      inv[a] = d[a] != 0.f ? __frcp_rn(d[a]) : __int_as_float(0x7f800000);
    }
    if (!moving) return false;  // reading A5: all-zero direction misses
    if (!(tmin < tmax) && tmax_finite) return false;
    // entry event: the latest of tmin and the entry planes of the moving slabs
    int ea = TMIN_AXIS, eP = 0;
    float te = tmin;
    bool miss = false;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (!((moving >> a) & 1)) {
        // half-open membership: floor(o_a) in [0, R_a)
        if (!(o[a] >= 0.f && o[a] < (float)p.dims[a])) miss = true;
        continue;
      }
      const int Pe = d[a] > 0.f ? 0 : p.dims[a];
      const float ta = tplane(Pe, o[a], inv[a]);
      if (cmp_events(o, d, a, Pe, ta, ea, eP, te) > 0) {
        ea = a;
        eP = Pe;
        te = ta;
      }
    }
    if (miss) return false;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (!((moving >> a) & 1)) continue;
      const int Px = d[a] > 0.f ? p.dims[a] : 0;
      // entered at / after the exit of slab a
      if (cmp_events(o, d, ea, eP, te, a, Px, tplane(Px, o[a], inv[a])) >= 0) miss = true;
    }
    if (miss || (tmax_finite && cmp_events(o, d, ea, eP, te, TMIN_AXIS, 0, tmax) >= 0)) return false;
    eaxis = ea;
    et = te;
    // the cell entered through the entry plane is exact; the other moving axes are located
    // (their slow path reads the event plane back from V[eaxis], so that one is set first)
#pragma unroll
    for (int b = 0; b < 3; ++b)
      if (b == ea) V[b] = d[b] > 0.f ? 0 : p.dims[b] - 1;
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      if (b == ea) continue;
      V[b] = ((moving >> b) & 1) ? locate(b, 0, p.dims[b] - 1) : (int)floorf(o[b]);
    }
    ct.add(VF_CTR_LOCATES, 3);
    set_tier(s_tw, 0);
    N = p.root;
    hd.mask = 0;
    hd.base = 0;
    load_header<KINDS, COUNT, ALN>(buf, kind(), N, hd, ct);
    stale = 0;
    stale_lc = 0;
    return true;
  }

  // Invariant: V >> lc() is the current (untested) cell of node N at tier t, entered at E (the
  // tier-change block below re-derives stale sub-cell bits right after a descent).
  // A pop always follows a step, so it lands on a new cell.
  // -- test the current cell of the current node (ordered_hit_children, one child): occ, and for
  // an occupied cell above the finest tier its child (next node, or the next level's root)
  __device__ __forceinline__ void test_cell(const uint32_t* __restrict__ buf, Ctr<COUNT>& ct, bool& occ,
                                            uint32_t& child) {
    const uint32_t kind = this->kind();
    const bool finest = this->finest();
    occ = false;
    child = 0;
    const uint32_t lx = ((uint32_t)V[0] >> lc()) & msk(), ly = ((uint32_t)V[1] >> lc()) & msk(),
                   lz = ((uint32_t)V[2] >> lc()) & msk();
    ct.add(VF_CTR_CELL_TESTS);
    if (has_kind<KINDS>(K_RAW) && kind == K_RAW) {
      // 64-bit index only where a grid can reach 2^32 words: a single-level R(11^3) grid has 2^33
      // cells (reading A15); every tier of a multi-tier buffer ends below word 2^32 (vf_build)
      using Idx = typename std::conditional<D::kIdx64, size_t, uint32_t>::type;
      const Idx lin = (Idx)lx + ((Idx)ly << sx()) + ((Idx)lz << sxy());
      if (!is_df()) {
        if constexpr (STAGE) child = t == 0 ? s_top[lin] : __ldg(buf + ((Idx)N + lin));
        else child = __ldg(buf + ((Idx)N + lin));
        occ = child != 0u;
        ct.add(VF_CTR_RAW_CELLS);
        ct.add(VF_CTR_FORMAT_BYTES, 4);
        ct.touch((size_t)N + lin, 1);
      } else if (budget > 0) {
        // DF: within L1 distance `budget` of a cell whose nearest non-empty cell is that far
        // away, so empty without a memory access ("how many voxels can be
        // marched through before checking occupancy")
        ct.add(VF_CTR_DF_SKIPS);
      } else {
        const uint2 v = __ldg(reinterpret_cast<const uint2*>(buf + ((Idx)N + 2 * lin)));
        child = v.x;
        occ = child != 0u;
        budget = (int)v.y;
        ct.add(VF_CTR_RAW_CELLS);
        ct.add(VF_CTR_FORMAT_BYTES, 8);
        ct.touch((size_t)N + 2 * lin, 2);
      }
    } else {
      const uint32_t lin = lx + (ly << sx()) + (lz << sxy());
      occ = (hd.mask >> lin) & 1u;
      if (occ && !finest) {
        const uint32_t rank = hd.rank(lin);
        const bool last = this->last();
        if (has_kind<KINDS>(K_SVO) && kind == K_SVO) {
          child = hd.base + 2u * rank;
        } else if (has_kind<KINDS>(K_SVDAG) && kind == K_SVDAG) {
          if constexpr (ALN)
            child = rank == 0 ? hd.base : rank == 1 ? hd.p1 : rank == 2 ? hd.p2 : __ldg(buf + N + 1u + rank);
          else
            child = __ldg(buf + N + 1u + rank);
          ct.add(VF_CTR_SVDAG_PTRS);
          ct.add(VF_CTR_FORMAT_BYTES, 4);
          ct.touch(N + 1u + rank, 1);
        } else {
          child = hd.base + (last ? 1u : 4u) * rank;
        }
        if (last) {  // leaf TermInt -> next level's root
          ct.touch(child, 1);
          child = __ldg(buf + child);
          ct.add(VF_CTR_LEAF_WORDS);
          ct.add(VF_CTR_FORMAT_BYTES, 4);
        }
      }
    }
  }

  // -- tier change: enter node nN at tier nt (descent or pop): its header, and after a descent
  // the exact sub-cell of every stale axis
  __device__ __forceinline__ void enter(const uint32_t* __restrict__ buf, const uint32_t* s_tw, Ctr<COUNT>& ct,
                                        int nt, uint32_t nN) {
    set_tier(s_tw, nt);
    N = nN;
    load_header<KINDS, COUNT, ALN>(buf, this->kind(), N, hd, ct);
    // after a descent, the new tier's cell needs V's bits >= lc(); if some of those are stale (the
    // ray moved inside a cell of size 2^stale_lc since they were exact), derive the exact finest
    // voxel of the stale axes within the parent cell (edge 2^lc(t-1); bits above it exact).
    // (never true after a pop: a pop lands on a tier with lc() >= stale_lc)
    if (stale && lc() < stale_lc) {
      const int st = stale & moving;
      // fast path of locate() on every stale axis at once (predicated, no per-axis branch):
      // x^ = fma(T^_E, d_b, o_b) is certified to lie strictly inside a cell unless it is within
      // B of an integer; those axes (a ray on / near a plane at E) take the certified slow path
      int slow = 0;
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const float x = fmaf(et, d[b], o[b]);
        const float fl = floorf(x);
        const float f = x - fl;  // exact
        const float B = (fabsf(et * d[b]) + fabsf(x)) * 0x1p-21f;
        const bool ok = f > B && 1.0f - f > B;
        const bool sb = (st >> b) & 1;
        if (sb && ok) V[b] = (int)fl;
        slow |= (sb && !ok) ? 1 << b : 0;
      }
      ct.add(VF_CTR_LOCATES, __popc(st));
      if (slow) {
        const uint32_t pl = lcp();
#pragma unroll
        for (int b = 0; b < 3; ++b)
          if ((slow >> b) & 1) {
            const int lo = (V[b] >> pl) << pl;
            V[b] = locate(b, lo, lo + (1 << pl) - 1);
          }
      }
      stale = 0;
      stale_lc = 0;
    }
  }

  __device__ __forceinline__ int iterate(const TraceParams& p, const uint32_t* __restrict__ buf,
                                         const uint32_t* s_tw, uint32_t (&stk)[VF_MAX_TIERS], Ctr<COUNT>& ct) {
#ifndef VF_DESCEND_CHAIN_STACK
    constexpr bool kChain = RESTART && D::kChainRestart;
#else
    constexpr bool kChain = true;
#endif
    if constexpr (kChain) {
      // Restart variant (format families where it measured faster, kChainRestart): one DDA step per
      // iteration, preceded by the chain of descents into occupied cells — a restart re-descends
      // several tiers at once (A/B: R(A^3) G(M) restart +2.7-8.8 %)
      for (;;) {
        bool occ;
        uint32_t child;
        test_cell(buf, ct, occ, child);
        if (!occ) break;
        if (finest()) return IT_HIT;  // unit intersection
        if (!RESTART || is_top()) stk[t] = N;
        ct.add(VF_CTR_DESCENTS);
        enter(buf, s_tw, ct, t + 1, child);
      }
      int nt = t;
      uint32_t nN = N;
      step(p, stk, ct, nt, nN);
      if (nt < 0) return IT_MISS;
      if (nt != t) enter(buf, s_tw, ct, nt, nN);  // pop
      return IT_CONTINUE;
    } else {
      // one cell test per iteration, followed by either a descent or a DDA step
      int nt = t;       // tier after this iteration
      uint32_t nN = N;  // node after this iteration
      {
        bool occ;
        uint32_t child;
        test_cell(buf, ct, occ, child);
        if (occ) {
          if (finest()) return IT_HIT;  // unit intersection
          // descend at event E (the child's entry cell is derived in the tier change below)
          if (!RESTART || is_top()) stk[t] = N;
          nt = t + 1;
          nN = child;
          ct.add(VF_CTR_DESCENTS);
        }
      }
      if (nt == t) {
        step(p, stk, ct, nt, nN);
        if (nt < 0) return IT_MISS;
      }
      // tier change (descent or pop), shared by both paths so a warp mixing them runs it once
      if (nt != t) enter(buf, s_tw, ct, nt, nN);
      return IT_CONTINUE;
    }
  }

  // -- step: exact next event among the three axes at this tier's cell size. Sets nt < 0 when
  // the segment ends (miss), nt < t (with nN) when the step leaves the current node.
  // (Instruction-lean form: the cell's next plane is its low corner, plus the cell edge for
  //  d > 0; only the stepped axes' cells change, so the root-box test and the changed-bit mask
  //  need no per-axis selects, and with a compiled-in cubic resolution 2^K the root-box test is
  //  one shift of the OR of the three coordinates.)
  __device__ __forceinline__ void step(const TraceParams& p, uint32_t (&stk)[VF_MAX_TIERS], Ctr<COUNT>& ct, int& nt,
                                       uint32_t& nN) {
    ct.add(VF_CTR_STEPS);
    const uint32_t l = lc();
    const int cell = 1 << l;
    int Pn[3];
    float tn[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      // next plane on axis a at this tier's cell size (inv = +inf makes a d = 0 axis never step)
      const int lo = V[a] & -cell;
      Pn[a] = ((dneg >> a) & 1) ? lo : lo + cell;
      tn[a] = tplane(Pn[a], o[a], inv[a]);
    }
    const float m = fminf(fminf(tn[0], tn[1]), tn[2]);
    const float thr = fmaf(fabsf(m), kCertEps, m);  // m + |m| eps: also for m < 0 (tmin < 0)
    // S: the stepping axes. One candidate within the certification margin of the fp32 minimum is
    // certified to be the exact minimum; several go to the exact argmin (ties step together).
    int S = (tn[0] <= thr ? 1 : 0) | (tn[1] <= thr ? 2 : 0) | (tn[2] <= thr ? 4 : 0);
    if (S == 0) {  // no finite next event (non-finite ray data outside the domain): end the walk
      nt = -1;
      return;
    }
    if ((S & (S - 1)) == 0) {
      eaxis = (S & 1) ? 0 : ((S & 2) ? 1 : 2);  // (selects: no BREV + FLO on the XU pipe)
      et = m;
    } else {
      const int res = argmin_exact(o[0], o[1], o[2], d[0], d[1], d[2], Pn[0], Pn[1], Pn[2], tn[0], tn[1], tn[2], S);
      S = res & 7;
      eaxis = res >> 4;
      et = sel3(tn, eaxis);
      ct.add(VF_CTR_NEAR_TIES);
    }
    // every axis of S steps into the cell adjacent to its plane (exact ties together, reading A2);
    // V is updated in place (on a miss it is not used again)
    int x = 0;
    uint32_t vor = 0;
    bool out_of_box = false;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int nv = ((S >> a) & 1) ? Pn[a] - ((dneg >> a) & 1) : V[a];
      x |= nv ^ V[a];
      V[a] = nv;
      vor |= (uint32_t)nv;
      if constexpr (D::kLogDim < 0) out_of_box |= (uint32_t)nv >= (uint32_t)p.dims[a];
    }
    if constexpr (D::kLogDim >= 0) out_of_box = (vor >> D::kLogDim) != 0u;
    if (out_of_box) {  // left the root box
      nt = -1;
      return;
    }
    // the segment ends at tmax (reading A7); E is read back through V[eaxis], so after the update
    if (tmax_finite && cmp_es(tmax) >= 0) {
      nt = -1;
      return;
    }
    // bits of V below l on the non-stepped axes are stale from here on (axes with d = 0 may be
    // marked too: they never move, and the locate block skips them)
    if (l) {
      stale = ~S & 7;  // (stale was a subset of the three axes)
      stale_lc = max(stale_lc, l);
    } else {
      stale &= ~S;
    }
    if constexpr (!SPEC) budget -= __popc(S);  // L1 distance moved (DF tiers only use it)
    else if (D::kHasDF) budget -= __popc(S);
    // h = highest bit in which the old and new cells differ; the step leaves this tier's node iff
    // h >= lc(t-1) (the node's edge), and then tau(h) is the deepest tier whose node holds both
    const uint32_t h = 31u - __clz((uint32_t)x);
    if (h >= lcp()) {
      const int tu = tau(p, h);
      ct.add(VF_CTR_POPS);
      // left the current node: pop (stack) or restart from the level root
      // (restart: from the top of tau's level — the following iterations re-descend through the
      //  nodes that contain the current cell as ordinary, always-occupied descents)
      nt = RESTART ? level_top(p, tu) : tu;
      nN = stk[nt];
      if (RESTART) ct.add(VF_CTR_REDESCENTS, tu - nt);
    }
  }

  __device__ __forceinline__ int4 hit_record() const { return make_int4(V[0], V[1], V[2], __float_as_int(et)); }

  // Closest-hit payload (the paper's closest-hit shader): the hit
  // voxel's terminating integer (its RGBA) and the entry-face normal -sign(d_a) e_a of the
  // axis whose plane event entered the hit cell (lowest axis on exact ties; 0 when the segment
  // starts inside the hit cell at tmin). Evaluated once per hit, at the finest tier.
  __device__ __forceinline__ uint2 payload_record(const uint32_t* __restrict__ buf) const {
    const uint32_t lx = ((uint32_t)V[0] >> lc()) & msk(), ly = ((uint32_t)V[1] >> lc()) & msk(),
                   lz = ((uint32_t)V[2] >> lc()) & msk();
    const uint32_t kind = this->kind();
    uint32_t rgba = 0;
    if (kind == K_RAW) {
      const size_t lin = (size_t)lx + ((size_t)ly << sx()) + ((size_t)lz << sxy());
      rgba = __ldg(buf + (size_t)N + lin * (is_df() ? 2u : 1u));
    } else {
      const uint32_t lin = lx + (ly << sx()) + (lz << sxy());
      const uint32_t rank = hd.rank(lin);
      if (kind == K_SVO)
        rgba = __ldg(buf + hd.base + 2u * rank);
      else if (kind == K_SVDAG)
        rgba = __ldg(buf + __ldg(buf + N + 1u + rank));
      else
        rgba = __ldg(buf + hd.base + rank);
    }
    uint32_t nrm = 0;
    if (eaxis != TMIN_AXIS) {
      // every axis whose voxel-slab entry plane is crossed exactly at E entered the cell (a finer
      // plane may coincide with the event of a coarse step): exact comparisons, lowest axis wins
      int a = eaxis;
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        if (b >= a || !((moving >> b) & 1)) continue;
        const int plane = ((dneg >> b) & 1) ? V[b] + 1 : V[b];
        if (cmp_eq(b, plane) == 0) a = b;
      }
      const uint32_t v = sel3(d, a) > 0.f ? 0xFFu : 0x01u;  // int8 -1 or +1
      nrm = v << (8 * a);
    }
    return make_uint2(rgba, nrm);
  }
};

__device__ __forceinline__ int4 miss_record() { return make_int4(-1, -1, -1, 0x7f800000); }

// Stage the tier table in shared memory: per tier {tier word, lc, cell-index mask, y shift} and
// {z shift} (two uint4), so a tier change is one LDS.128 + one LDS.32 (no field extraction).
__device__ __forceinline__ void stage_tiers(const TraceParams& p, uint32_t* s_tw) {
  if (threadIdx.x < VF_MAX_TIERS) {
    const uint32_t w = p.tword[threadIdx.x];
    reinterpret_cast<uint4*>(s_tw)[2 * threadIdx.x] =
        make_uint4(w, twf(w, TW_LC, 4), (1u << twf(w, TW_MB, 4)) - 1u, twf(w, TW_SX, 4));
    reinterpret_cast<uint4*>(s_tw)[2 * threadIdx.x + 1] = make_uint4(twf(w, TW_SXY, 5), 0u, 0u, 0u);
  }
  __syncthreads();
}

// One thread per ray, 128-thread blocks.
#ifndef VF_TRACE_THREADS
#define VF_TRACE_THREADS 128  // block size (A/B: 256 with VF_MINB 4 keeps the 64-register cap)
#endif
constexpr unsigned kTraceThreads = VF_TRACE_THREADS;
#ifdef VF_BLOCK_CLOCK
__device__ unsigned long long* g_block_clock;
#endif
template <uint32_t KINDS, bool RESTART, bool COUNT, class D = NoSpec, bool ALN = false>
__global__ void __launch_bounds__(kTraceThreads, D::kMinBlocks) trace_kernel(const TraceParams p, const uint32_t* __restrict__ buf,
                                                    const float4* __restrict__ rays, int4* __restrict__ hits,
                                                    uint64_t n, unsigned long long* __restrict__ counters,
                                                    unsigned long long* __restrict__ work) {
  __shared__ __align__(16) uint32_t s_tw[8 * VF_MAX_TIERS];
  __shared__ long long s_clk;      // VF_TRACE_SCHEDULE: the block's start (SM cycles)
  __shared__ uint32_t s_warps_done;  // ... and its finished warps
#ifdef VF_BLOCK_CLOCK  // analysis build (tools/block_timeline.py): per-block start / end / SM
  unsigned long long blk_t0 = 0;
  if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(blk_t0));
#endif
  if (p.cost && threadIdx.x == 0) {  // (ordered before every read by stage_tiers' barrier)
    s_clk = clock64();
    s_warps_done = 0;
  }
  stage_tiers(p, s_tw);
  // VF_TRACE_SCHEDULE: this block takes slot block order[b] (longest-first list scheduling), and
  // slot v traces ray ray_perm[v] (rays regrouped into warps by duration inside groups of 256)
  const uint64_t tb = p.order ? __ldg(p.order + blockIdx.x) : blockIdx.x;
  uint64_t gid = tb * blockDim.x + threadIdx.x;
  if (p.ray_perm && gid < n) gid = __ldg(p.ray_perm + gid);
  Ctr<COUNT> ct;
  ct.touch_map = p.touch;
  if (gid < n) {
    Lane<KINDS, RESTART, COUNT, D, false, ALN> L;
    uint32_t stk[VF_MAX_TIERS];
    int4 out = miss_record();
    uint32_t iters = 0;  // VF_TRACE_SCHEDULE: this ray's iterations (its lane's share of the warp)
    if (L.start(p, buf, s_tw, __ldg(rays + 2 * gid), __ldg(rays + 2 * gid + 1), ct)) {
      int res;
      do {
        res = L.iterate(p, buf, s_tw, stk, ct);
        ++iters;
      } while (res == IT_CONTINUE);
      if (res == IT_HIT) {
        out = L.hit_record();
        if (p.payload) p.payload[gid] = L.payload_record(buf);
        ct.add(VF_CTR_HITS);
      }
    }
    hits[p.slot ? __ldg(p.slot + gid) : gid] = out;  // vf_trace_scatter: fused hit gather
#ifdef VF_RAY_TESTS  // analysis build (tools/ray_tests_dump.py): per-ray cell tests of the counting run
    if (COUNT) hits[gid].x = (int)ct.v[VF_CTR_CELL_TESTS];
#endif
    if (p.payload && out.x < 0) p.payload[gid] = make_uint2(0u, 0u);
    if (p.ray_cost) p.ray_cost[gid] = iters;  // the next launch's regrouping key
    ct.add(VF_CTR_RAYS);
  }
  ct.flush(counters);
  if (p.cost) {  // the block's duration, for the next launch's order (uniform branch): the last
    __syncwarp();  // warp to finish stores it (no block barrier: finished warps exit)
    if ((threadIdx.x & 31u) == 0 && atomicAdd(&s_warps_done, 1u) == blockDim.x / 32u - 1u) {
      const long long c = clock64() - s_clk;
      p.cost[p.order ? __ldg(p.order + blockIdx.x) : blockIdx.x] = c > 0xffffffffll ? 0xffffffffu : (uint32_t)c;
    }
  }
#ifdef VF_BLOCK_CLOCK
  __syncthreads();
  if (threadIdx.x == 0 && g_block_clock) {
    unsigned long long t1;
    uint32_t sm;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    g_block_clock[3 * blockIdx.x] = blk_t0;
    g_block_clock[3 * blockIdx.x + 1] = t1;
    g_block_clock[3 * blockIdx.x + 2] = sm;
  }
#endif
}

// Persistent warps with dynamic ray fetch: grid = resident blocks; a warp keeps its lanes busy
// by fetching a new batch of rays (one atomicAdd per batch) whenever at least kRefill lanes have
// finished. This removes the SIMT loss of finished lanes idling until the slowest ray of the
// warp ends, and the launch tail (SURVEY.md §8(d) "warp ballot early-out / persistent refill").
// work[0] = next ray, work[1] = finished blocks; the last block resets both.
constexpr int kPersistThreads = 128;
#ifndef VF_PMINB
#define VF_PMINB 8  // persistent kernel: min blocks per SM (register cap), A/B on incoherent rays
#endif

template <uint32_t KINDS, bool RESTART, bool COUNT>
__global__ void __launch_bounds__(kPersistThreads, VF_PMINB) trace_persistent(const TraceParams p, const uint32_t* __restrict__ buf,
                                                                   const float4* __restrict__ rays,
                                                                   int4* __restrict__ hits, uint64_t n,
                                                                   unsigned long long* __restrict__ counters,
                                                                   unsigned long long* __restrict__ work) {
  __shared__ __align__(16) uint32_t s_tw[8 * VF_MAX_TIERS];
  stage_tiers(p, s_tw);
  Ctr<COUNT> ct;
  ct.touch_map = p.touch;
  Lane<KINDS, RESTART, COUNT> L;
  uint32_t stk[VF_MAX_TIERS];
  const unsigned lane = threadIdx.x & 31u;
  const unsigned lt = (1u << lane) - 1u;
  bool active = false, exhausted = false;
  uint64_t idx = 0;
  for (;;) {
    unsigned idle = __ballot_sync(0xffffffffu, !active);
    if (!exhausted && __popc(idle) >= p.refill) {
      unsigned long long base = 0;
      const unsigned cnt = __popc(idle);
      if (lane == 0) base = atomicAdd(work, (unsigned long long)cnt);
      base = __shfl_sync(0xffffffffu, base, 0);
      if (base + cnt >= n) exhausted = true;
      if (!active) {
        idx = base + __popc(idle & lt);
        if (idx < n) {
          ct.add(VF_CTR_RAYS);
          if (L.start(p, buf, s_tw, __ldg(rays + 2 * idx), __ldg(rays + 2 * idx + 1), ct))
            active = true;
          else {
            hits[p.slot ? __ldg(p.slot + idx) : idx] = miss_record();
            if (p.payload) p.payload[idx] = make_uint2(0u, 0u);
          }
        }
      }
      idle = __ballot_sync(0xffffffffu, !active);
    }
    if (idle == 0xffffffffu) {
      if (exhausted) break;
      continue;
    }
    if (active) {
      const int res = L.iterate(p, buf, s_tw, stk, ct);
      if (res != IT_CONTINUE) {
        if (res == IT_HIT) ct.add(VF_CTR_HITS);
        hits[p.slot ? __ldg(p.slot + idx) : idx] = res == IT_HIT ? L.hit_record() : miss_record();
        if (p.payload) p.payload[idx] = res == IT_HIT ? L.payload_record(buf) : make_uint2(0u, 0u);
        active = false;
      }
    }
  }
  ct.flush(counters);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned long long done = atomicAdd(work + 1, 1ull);
    if (done == gridDim.x - 1) {  // last block: reset the work counter for the next launch
      atomicExch(work, 0ull);
      atomicExch(work + 1, 0ull);
    }
  }
}

// Persistent warps over claimed chunks of p.chunk consecutive rays. The ray buffer is in screen-tile
// order (16x16 blocks of 8x4 warp tiles), so a chunk is a screen-coherent patch: a warp claims a
// chunk (one atomicAdd), starts its first 32 rays, and whenever >= p.crefill lanes are idle refills
// them with the chunk's next rays — neighbours of the rays still in flight, so the warp stays
// coherent while its finished lanes get work; when the chunk runs out the warp claims the next one.
// Removes the launch tail (no waves: each warp keeps claiming until the frame is done) and most of
// the in-warp tail of finished lanes. STAGE: the top Raw grid (<= 16 KB) is copied to shared memory
// once per block and tier-0 cell tests read it there. work[0] = next ray, work[1] = finished blocks.
template <uint32_t KINDS, bool RESTART, class D, bool STAGE>
__global__ void __launch_bounds__(kTraceThreads, D::kMinBlocks)
    trace_chunked(const TraceParams p, const uint32_t* __restrict__ buf, const float4* __restrict__ rays,
                  int4* __restrict__ hits, uint64_t n, unsigned long long* __restrict__ counters,
                  unsigned long long* __restrict__ work) {
  __shared__ __align__(16) uint32_t s_tw[8 * VF_MAX_TIERS];
  extern __shared__ __align__(16) uint32_t s_top[];
  if constexpr (STAGE) {
    for (uint32_t i = threadIdx.x; i < D::kTopWords / 4; i += blockDim.x)
      reinterpret_cast<uint4*>(s_top)[i] = __ldg(reinterpret_cast<const uint4*>(buf + p.root) + i);
  }
  stage_tiers(p, s_tw);  // (its __syncthreads also publishes s_top)
  Ctr<false> ct;
  Lane<KINDS, RESTART, false, D, STAGE> L;
  L.s_top = s_top;
  uint32_t stk[VF_MAX_TIERS];
  const unsigned lane = threadIdx.x & 31u;
  const unsigned lt = (1u << lane) - 1u;
  bool active = false;
  uint64_t idx = 0;
  unsigned long long next = 0, end = 0;  // the warp's current chunk [next, end)
  bool exhausted = false;
  const unsigned keep = 32u - p.crefill;  // the inner loop runs while more than `keep` lanes trace
  for (;;) {
    // ---- refill (warp-uniform): claim a chunk when the current one is used up, start new rays
    unsigned idle = __ballot_sync(0xffffffffu, !active);
    if (next >= end && !exhausted) {
      unsigned long long b = 0;
      if (lane == 0) b = atomicAdd(work, (unsigned long long)p.chunk);
      b = __shfl_sync(0xffffffffu, b, 0);
      if (b >= n) {
        exhausted = true;
      } else {
        next = b;
        end = b + p.chunk < n ? b + p.chunk : n;
      }
    }
    if (next < end) {
      const unsigned long long mine = next + __popc(idle & lt);
      next = next + __popc(idle) < end ? next + __popc(idle) : end;
      if (!active && mine < end) {
        idx = mine;
        if (L.start(p, buf, s_tw, __ldg(rays + 2 * idx), __ldg(rays + 2 * idx + 1), ct)) {
          active = true;
        } else {
          hits[p.slot ? __ldg(p.slot + idx) : idx] = miss_record();
          if (p.payload) p.payload[idx] = make_uint2(0u, 0u);
        }
      }
    }
    if (__ballot_sync(0xffffffffu, active) == 0u) {
      if (exhausted && next >= end) break;
      continue;
    }
    // ---- trace: the plain per-ray loop; with refill (crefill < 32) a lane also leaves it when no
    // more than `keep` lanes of the warp are still tracing (no per-iteration vote otherwise)
    if (active) {
      int res;
      for (;;) {
        res = L.iterate(p, buf, s_tw, stk, ct);
        if (res != IT_CONTINUE) break;
        if (keep > 0 && (unsigned)__popc(__activemask()) <= keep) break;
      }
      if (res != IT_CONTINUE) {
        hits[p.slot ? __ldg(p.slot + idx) : idx] = res == IT_HIT ? L.hit_record() : miss_record();
        if (p.payload) p.payload[idx] = res == IT_HIT ? L.payload_record(buf) : make_uint2(0u, 0u);
        active = false;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned long long done = atomicAdd(work + 1, 1ull);
    if (done == gridDim.x - 1) {  // last block: reset the work counter for the next launch
      atomicExch(work, 0ull);
      atomicExch(work + 1, 0ull);
    }
  }
  (void)counters;
}

// ---- touch bitmap reduction (counting runs): distinct words = set bits; distinct 32-B sectors =
// non-zero bytes (byte j of bitmap word i covers words 32i + 8j .. +7, one sector of the
// 256-B-aligned buffer)
__global__ void touch_count_kernel(const uint32_t* __restrict__ touch, uint64_t nw, unsigned long long* counters) {
  unsigned long long words = 0, sectors = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nw; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t w = touch[i];
    words += __popc(w);
    sectors += ((w & 0xFFu) != 0) + ((w & 0xFF00u) != 0) + ((w & 0xFF0000u) != 0) + ((w & 0xFF000000u) != 0);
  }
  for (int o = 16; o; o >>= 1) {
    words += __shfl_down_sync(0xffffffffu, words, o);
    sectors += __shfl_down_sync(0xffffffffu, sectors, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(counters + VF_CTR_UNIQUE_WORDS, words);
    atomicAdd(counters + VF_CTR_UNIQUE_SECTORS, sectors);
  }
}

// ---- point query: integer-only descent (test aid) ------------------------------------------
__global__ void query_kernel(const TraceParams p, const uint32_t* __restrict__ buf, const uint32_t* __restrict__ xyz,
                             uint32_t* __restrict__ out, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t V[3] = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
    uint32_t res = 0;
    if (p.root != 0 && V[0] < (uint32_t)p.dims[0] && V[1] < (uint32_t)p.dims[1] && V[2] < (uint32_t)p.dims[2]) {
      uint32_t N = p.root;
      for (uint32_t t = 0; t < p.n_tiers; ++t) {
        const uint32_t kind = (p.kind_pack >> (2 * t)) & 3u;
        const uint32_t lc = field4(p.lc_pack, t), lf = field4(p.lf_pack, t);
        const uint32_t msk = t == 0 ? 0xFFFFFFFFu : ((1u << lf) - 1u);
        const uint32_t lin = ((V[0] >> lc) & msk) + (((V[1] >> lc) & msk) << (t == 0 ? p.lf0[0] : lf)) +
                             (((V[2] >> lc) & msk) << (t == 0 ? p.lf0[0] + p.lf0[1] : 2 * lf));
        const bool last = (p.last_mask >> t) & 1u;
        uint32_t word;
        if (kind == K_RAW) {
          word = buf[(size_t)N + (size_t)lin * (((p.df_mask >> t) & 1u) ? 2u : 1u)];
        } else {
          uint64_t mask;
          uint32_t base;
          if (kind == K_SVO) {
            base = buf[N];
            mask = buf[N + 1] & 0xFFu;
          } else if (kind == K_SVDAG) {
            base = N;
            mask = buf[N] & 0xFFu;
          } else {
            mask = (uint64_t)buf[N] | ((uint64_t)buf[N + 1] << 32);
            base = buf[N + 2];
          }
          if (!((mask >> lin) & 1u)) {
            word = 0;
          } else {
            const uint32_t rank = __popcll(mask & ((1ull << lin) - 1ull));
            uint32_t c;
            if (kind == K_SVO)
              c = base + 2u * rank;
            else if (kind == K_SVDAG)
              c = buf[base + 1u + rank];
            else
              c = base + (last ? 1u : 4u) * rank;
            word = last ? buf[c] : c;
          }
        }
        if (word == 0) {
          res = 0;
          break;
        }
        res = word;
        N = word;
      }
    }
    out[i] = res;
  }
}

// ---- VF_TRACE_SCHEDULE: longest-first block order from the last launch's block durations -------
// A frame's launch lasts as long as its slowest blocks: blocks that start late and run long leave
// the other SMs idle (cfg4: SMs active 82 % of the launch, tools/block_timeline.py). Greedy list
// scheduling in order of decreasing duration (LPT) bounds the makespan by the longest block; the
// durations come from the previous launch over the same ray array (temporal coherence of frames).
// Two small kernels: a histogram of quarter-octave duration classes, then a scatter of block
// indices into their class's range, longest class first. A block's class is taken from the
// longest duration within +-6 blocks (+-3 screen tiles of the 16x16-tile ray order): when the
// camera moves between frames, a slow region's neighbours are promoted with it (A/B: with a moved
// camera the undilated order loses up to 23 % on cfg3, the dilated one gains 4-9 %). Each CTA
// scatters a contiguous range of blocks, so blocks of one class keep their screen locality. The
// last CTA resets the counters.
struct SchedCfg {
  uint32_t sub;  // log2 classes per octave of duration (0..2)
  uint32_t dil;  // a block's class uses the longest duration within +-dil blocks (screen neighbours)
};
__device__ __forceinline__ uint32_t sched_class(const uint32_t* __restrict__ cost, uint32_t nb, uint32_t i,
                                                SchedCfg g) {
  uint32_t c = __ldg(cost + i);
  for (uint32_t k = 1; k <= g.dil; ++k) {
    if (i >= k) c = max(c, __ldg(cost + i - k));
    if (i + k < nb) c = max(c, __ldg(cost + i + k));
  }
  c |= 4u;
  const uint32_t e = 31u - __clz(c);
  const uint32_t key = (e << g.sub) + ((c >> (e - g.sub)) & ((1u << g.sub) - 1u));
  return (kSchedBuckets - 1u) - key;  // 0 = longest
}

__global__ void __launch_bounds__(256) sched_hist_kernel(const uint32_t* __restrict__ cost, uint32_t nb,
                                                         uint32_t* __restrict__ hist, uint8_t* __restrict__ cls,
                                                         SchedCfg g) {
  __shared__ uint32_t sh[kSchedBuckets];
  for (uint32_t i = threadIdx.x; i < kSchedBuckets; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x) {
    const uint32_t k = sched_class(cost, nb, i, g);  // (kept for the scatter: one byte per block)
    cls[i] = (uint8_t)k;
    atomicAdd(&sh[k], 1u);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < kSchedBuckets; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

__global__ void __launch_bounds__(256) sched_scatter_kernel(const uint8_t* __restrict__ cls, uint32_t nb,
                                                            uint32_t* __restrict__ hist, uint32_t* __restrict__ cursor,
                                                            uint32_t* __restrict__ done, uint32_t* __restrict__ order,
                                                            SchedCfg g) {
  (void)g;  // (the classes were computed with it by sched_hist_kernel)
  __shared__ uint32_t base[kSchedBuckets], loc[kSchedBuckets];
  __shared__ bool last;
  const uint32_t per = (nb + gridDim.x - 1) / gridDim.x;
  const uint32_t b0 = blockIdx.x * per, b1 = min(nb, b0 + per);
  if (threadIdx.x < kSchedBuckets) loc[threadIdx.x] = 0;
  __syncthreads();
  for (uint32_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) atomicAdd(&loc[__ldg(cls + i)], 1u);
  __syncthreads();
  // class start (exclusive scan of hist: one class per thread of the first kSchedBuckets, warp
  // shuffles + the warp totals) + this CTA's range in it
  __shared__ uint32_t wtot[kSchedBuckets / 32];
  uint32_t hv = 0, incl = 0;
  if (threadIdx.x < kSchedBuckets) {
    hv = hist[threadIdx.x];
    incl = hv;
#pragma unroll
    for (uint32_t d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
      if ((threadIdx.x & 31u) >= d) incl += y;
    }
    if ((threadIdx.x & 31u) == 31u) wtot[threadIdx.x >> 5] = incl;
  }
  __syncthreads();
  if (threadIdx.x < kSchedBuckets) {
    uint32_t start = incl - hv;
    for (uint32_t w = 0; w < (threadIdx.x >> 5); ++w) start += wtot[w];
    const uint32_t cnt = loc[threadIdx.x];
    base[threadIdx.x] = start + (cnt ? atomicAdd(&cursor[threadIdx.x], cnt) : 0u);
    loc[threadIdx.x] = 0;
  }
  __syncthreads();
  for (uint32_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
    const uint32_t k = __ldg(cls + i);
    order[base[k] + atomicAdd(&loc[k], 1u)] = i;
  }
  // the last CTA to finish resets hist / cursor / done for the next launch (every CTA has read hist)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    if (threadIdx.x < kSchedBuckets) {
      hist[threadIdx.x] = 0;
      cursor[threadIdx.x] = 0;
    }
    if (threadIdx.x == 0) *done = 0;
  }
}

// VF_TRACE_REGROUP: rays regrouped into warps by their iteration counts in the last launch. A warp
// lasts as long as its longest ray, so inside each group of kRayGroup consecutive rays (one 16x16
// screen tile of the tile-ordered ray stream) the rays are ordered by their last iteration count,
// longest first: slot g*256 + r traces the group's r-th longest ray. A warp's slots stay inside
// one tile (coherent upper levels) while its lanes become homogeneous in length (counting-run
// simulation: warp-iterations per ray cfg4 24.6 -> 19.6, cfg5 37.0 -> 31.8). One CTA per group, a
// stable counting sort over 32 quarter-octave classes (>= 128 iterations share class 0): lanes of
// a warp with the same class find each other with __match_any_sync, a block-wide exclusive scan
// over (class, warp) gives every lane its slot. Slots past n (a ragged last group) sort last.
__global__ void __launch_bounds__(kRayGroup) sched_raysort_kernel(const uint32_t* __restrict__ ray_cost, uint64_t n,
                                                                  uint32_t* __restrict__ ray_perm) {
  constexpr uint32_t kWarps = kRayGroup / 32u, kClasses = 32u;
  static_assert(kClasses * kWarps == kRayGroup, "one (class, warp) counter per thread");
  __shared__ uint32_t cnt[kClasses * kWarps];  // [class][warp], then its exclusive prefix
  __shared__ uint32_t wsum[kWarps];
  const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
  const uint64_t i = (uint64_t)blockIdx.x * kRayGroup + threadIdx.x;
  cnt[threadIdx.x] = 0;
  uint32_t k = kClasses - 1u;
  if (i < n) {
    const uint32_t v = (__ldg(ray_cost + i) + 1u) << 2;
    const uint32_t e = 31u - __clz(v);
    k = kClasses - 1u - min(4u * (e - 2u) + ((v >> (e - 2u)) & 3u), kClasses - 1u);
  }
  const uint32_t peers = __match_any_sync(0xffffffffu, k);
  const uint32_t below = __popc(peers & ((1u << lane) - 1u));
  __syncthreads();
  if (below == 0) cnt[k * kWarps + w] = __popc(peers);
  __syncthreads();
  // exclusive scan of cnt in (class, warp) order: one entry per thread
  const uint32_t x = cnt[threadIdx.x];
  uint32_t incl = x;
#pragma unroll
  for (uint32_t d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += y;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  uint32_t off = 0;
  for (uint32_t q = 0; q < w; ++q) off += wsum[q];
  __syncthreads();
  cnt[threadIdx.x] = off + incl - x;
  __syncthreads();
  if (i < n) ray_perm[(uint64_t)blockIdx.x * kRayGroup + cnt[k * kWarps + w] + below] = (uint32_t)i;
}

using KernelFn = void (*)(const TraceParams, const uint32_t*, const float4*, int4*, uint64_t, unsigned long long*,
                          unsigned long long*);

template <uint32_t K, bool R, bool C>
KernelFn pick(bool persistent) {
  return persistent ? trace_persistent<K, R, C> : trace_kernel<K, R, C>;
}

template <uint32_t K>
KernelFn get_kernel(bool restart, bool count, bool persistent) {
  if (count) return restart ? pick<K, true, true>(persistent) : pick<K, false, true>(persistent);
  return restart ? pick<K, true, false>(persistent) : pick<K, false, false>(persistent);
}

KernelFn select_kernel(uint32_t kinds, bool restart, bool count, bool persistent) {
#ifdef VF_ONLY_KINDS  // fast A/B variant builds (tools/build_variant.sh -DVF_ONLY_KINDS=5): one kind set
  return kinds == VF_ONLY_KINDS ? get_kernel<VF_ONLY_KINDS>(restart, count, persistent) : nullptr;
#else
  switch (kinds) {
#define VF_CASE(k) \
  case k: return get_kernel<k>(restart, count, persistent);
    VF_CASE(1) VF_CASE(2) VF_CASE(3) VF_CASE(4) VF_CASE(5) VF_CASE(6) VF_CASE(7) VF_CASE(8) VF_CASE(9) VF_CASE(10)
    VF_CASE(11) VF_CASE(12) VF_CASE(13) VF_CASE(14) VF_CASE(15)
#undef VF_CASE
    default: return nullptr;
  }
#endif
}

// Compiled-in formats: R(A^3) G(M) (RawSvdag: the cfg4 / cfg5 / t512 headline formats and their
// sweep neighbours) and the cfg2 / cfg3 headline formats (SparseRaw). Others run the generic kernel.
// mode 0: one thread per ray; 1: chunked persistent warps; 2: chunked + top Raw grid in shared memory
// HEADLINE: the format also gets the VF_BUILD_ALIGN_NODES instance (aligned SVDAG header loads) and
// the counting instance (mode -1: vf_trace_counters runs the same compiled-in traversal it counts)
template <uint32_t KINDS, class D, bool HEADLINE = false>
KernelFn spec_kernel(bool restart, int mode, bool aln = false) {
  if constexpr (HEADLINE) {
    if (mode == -1) return restart ? trace_kernel<KINDS, true, true, D> : trace_kernel<KINDS, false, true, D>;
    if (aln && mode == 0) return restart ? trace_kernel<KINDS, true, false, D, true> : trace_kernel<KINDS, false, false, D, true>;
  }
  if (mode < 0) return nullptr;  // counting: the generic kernel
  (void)aln;
#ifdef VF_CHUNKED_KERNELS
  if constexpr (D::kTopWords != 0) {
    if (mode == 2) return restart ? trace_chunked<KINDS, true, D, true> : trace_chunked<KINDS, false, D, true>;
  }
  if (mode >= 1) return restart ? trace_chunked<KINDS, true, D, false> : trace_chunked<KINDS, false, D, false>;
#else
  (void)mode;
#endif
  return restart ? trace_kernel<KINDS, true, false, D> : trace_kernel<KINDS, false, false, D>;
}

constexpr LevelSpec kFmtG5R3[] = {{VF_SVDAG, 1, 5}, {VF_RAW, 3, 1}};                     // cfg2
constexpr LevelSpec kFmtT22T21R4[] = {{VF_NTREE, 2, 2}, {VF_NTREE, 2, 1}, {VF_RAW, 4, 1}};  // cfg3
constexpr LevelSpec kFmtT21T22R4[] = {{VF_NTREE, 2, 1}, {VF_NTREE, 2, 2}, {VF_RAW, 4, 1}};  // cfg3 (other order)
constexpr LevelSpec kFmtS5R5[] = {{VF_SVO, 1, 5}, {VF_RAW, 5, 1}};                        // cfg3
constexpr LevelSpec kFmtT24R3[] = {{VF_NTREE, 2, 4}, {VF_RAW, 3, 1}};                     // cfg4 sweep
constexpr LevelSpec kFmtT22T22R3[] = {{VF_NTREE, 2, 2}, {VF_NTREE, 2, 2}, {VF_RAW, 3, 1}};  // cfg4 sweep
constexpr LevelSpec kFmtT23R5[] = {{VF_NTREE, 2, 3}, {VF_RAW, 5, 1}};                     // cfg4 sweep
constexpr LevelSpec kFmtS5R4[] = {{VF_SVO, 1, 5}, {VF_RAW, 4, 1}};                        // t512
constexpr LevelSpec kFmtG5R4[] = {{VF_SVDAG, 1, 5}, {VF_RAW, 4, 1}};                      // t512
constexpr LevelSpec kFmtG2R2[] = {{VF_SVDAG, 1, 2}, {VF_RAW, 2, 1}};                      // tests
constexpr LevelSpec kFmtT11T12R1[] = {{VF_NTREE, 1, 1}, {VF_NTREE, 1, 2}, {VF_RAW, 1, 1}};  // tests

template <size_t NL>
bool same_format(const Format& f, const LevelSpec (&lv)[NL]) {
  if (f.n_levels != NL) return false;
  for (size_t l = 0; l < NL; ++l) {
    const vf_level& v = f.levels[l];
    if (v.kind != lv[l].kind) return false;
    if (v.kind == VF_RAW) {
      if (v.log2_extent[0] != lv[l].lf || v.log2_extent[1] != lv[l].lf || v.log2_extent[2] != lv[l].lf) return false;
    } else if (v.kind == VF_NTREE) {
      if (v.log2_fanout != lv[l].lf || v.depth != lv[l].depth) return false;
    } else if (v.depth != lv[l].depth) {
      return false;
    }
  }
  return true;
}

KernelFn select_spec(const Format& f, bool restart, int mode, bool aln) {
#ifdef VF_ONLY_KINDS
  constexpr uint32_t K = VF_ONLY_KINDS;
#define VF_HAS(k) (K == (k))
#else
#define VF_HAS(k) true
#endif
  if (VF_HAS(5) && f.n_levels == 2 && f.levels[0].kind == VF_RAW && f.levels[1].kind == VF_SVDAG) {
    const uint8_t* e = f.levels[0].log2_extent;
    if (e[0] == e[1] && e[1] == e[2]) switch (((uint32_t)e[0] << 8) | f.levels[1].depth) {
#define VF_SPEC(a, m) \
  case ((a) << 8) | (m): return spec_kernel<5, RawSvdag<a, m>>(restart, mode);
#define VF_SPECA(a, m) /* + the VF_BUILD_ALIGN_NODES and counting instances */ \
  case ((a) << 8) | (m): return spec_kernel<5, RawSvdag<a, m>, true>(restart, mode, aln);
        VF_SPECA(4, 7) VF_SPECA(4, 8) VF_SPECA(3, 8) VF_SPEC(3, 7) VF_SPEC(4, 5) VF_SPEC(2, 7) VF_SPEC(6, 5)
        VF_SPEC(8, 3) VF_SPEC(3, 5) VF_SPECA(3, 9) VF_SPEC(7, 2) VF_SPECA(5, 7) VF_SPEC(5, 6)
        VF_SPEC(6, 6) VF_SPEC(7, 5)
        VF_SPECA(2, 3) VF_SPEC(1, 4)  // small instances for the parity tests
#undef VF_SPEC
#undef VF_SPECA
        default: break;
      }
  }
#ifndef VF_ONLY_KINDS
  // single sparse levels and Raw-topped sparse levels of the sweeps
  if (f.n_levels == 1 || (f.n_levels == 2 && (f.levels[0].kind == VF_RAW || f.levels[0].kind == VF_DF))) {
    const vf_level& sp = f.levels[f.n_levels - 1];
    uint32_t a = 0;
    const uint32_t df = f.n_levels == 2 && f.levels[0].kind == VF_DF;
    if (f.n_levels == 2) {
      const uint8_t* e = f.levels[0].log2_extent;
      if (e[0] != e[1] || e[1] != e[2]) return nullptr;
      a = e[0];
    }
    const uint32_t lf = sp.kind == VF_NTREE ? sp.log2_fanout : 1u;
    const uint32_t key = (df << 28) | (a << 24) | (sp.kind << 16) | (lf << 8) | sp.depth;
    switch (key) {
#define VF_TS(a, k, lf, ns, kinds) \
  case ((a) << 24) | ((k) << 16) | ((lf) << 8) | (ns): return spec_kernel<kinds, TopSparse<a, K_OF_##k, lf, ns>>(restart, mode);
#define VF_DS(a, k, ns) /* DF top D(a^3, M) */ \
  case (1u << 28) | ((a) << 24) | ((k) << 16) | (1u << 8) | (ns): \
    return spec_kernel<(1u << K_RAW) | (1u << K_OF_##k), TopSparse<a, K_OF_##k, 1, ns, true>>(restart, mode);
      VF_DS(4, VF_SVDAG, 7) VF_DS(6, VF_SVDAG, 5) VF_DS(4, VF_SVO, 7) VF_DS(6, VF_SVO, 5) VF_DS(4, VF_SVDAG, 5)
      VF_DS(4, VF_SVO, 5) VF_DS(2, VF_SVDAG, 2)
      VF_DS(4, VF_SVDAG, 8) VF_DS(5, VF_SVDAG, 7) VF_DS(3, VF_SVDAG, 9) VF_DS(5, VF_SVDAG, 6)  // cfg5 / cfg4 DF hybrids
      VF_DS(6, VF_SVDAG, 6) VF_DS(7, VF_SVDAG, 5)
#undef VF_DS
#define VF_TSA(a, k, lf, ns, kinds) /* + the VF_BUILD_ALIGN_NODES and counting instances */ \
  case ((a) << 24) | ((k) << 16) | ((lf) << 8) | (ns): \
    return spec_kernel<kinds, TopSparse<a, K_OF_##k, lf, ns>, true>(restart, mode, aln);
      VF_TSA(0, VF_SVDAG, 1, 11, 4) VF_TS(0, VF_SVO, 1, 11, 2) VF_TSA(0, VF_SVDAG, 1, 8, 4) VF_TS(0, VF_SVO, 1, 8, 2)
      VF_TS(0, VF_SVDAG, 1, 10, 4) VF_TS(0, VF_SVO, 1, 10, 2) VF_TSA(0, VF_SVDAG, 1, 12, 4) VF_TS(0, VF_SVO, 1, 12, 2)
#undef VF_TSA
      VF_TS(0, VF_SVDAG, 1, 9, 4) VF_TS(0, VF_SVO, 1, 9, 2)
      VF_TS(0, VF_SVDAG, 1, 6, 4) VF_TS(0, VF_SVO, 1, 6, 2) VF_TS(0, VF_NTREE, 2, 3, 8)  // cfg1 sweep
      VF_TS(4, VF_SVO, 1, 7, 3) VF_TS(6, VF_SVO, 1, 5, 3) VF_TS(4, VF_SVO, 1, 5, 3)
      VF_TS(0, VF_NTREE, 2, 4, 8) VF_TS(0, VF_NTREE, 2, 5, 8) VF_TS(0, VF_NTREE, 2, 6, 8) VF_TS(1, VF_NTREE, 2, 5, 9)
      VF_TS(4, VF_NTREE, 2, 4, 9)
      VF_TS(0, VF_SVDAG, 1, 4, 4) VF_TS(0, VF_NTREE, 1, 4, 8) VF_TS(2, VF_NTREE, 1, 3, 9)  // tests
#undef VF_TS
      default: break;
    }
  }
#endif
#ifndef VF_ONLY_KINDS
  if (f.n_levels == 2 || f.n_levels == 3) {  // [R(A^3)] S|G(a) S|G(b)
    const uint32_t o = f.n_levels == 3 ? 1u : 0u;
    const vf_level &l1 = f.levels[o], &l2 = f.levels[o + 1];
    const bool oct1 = l1.kind == VF_SVO || l1.kind == VF_SVDAG, oct2 = l2.kind == VF_SVO || l2.kind == VF_SVDAG;
    uint32_t a = 0;
    bool ok = oct1 && oct2;
    if (ok && o) {
      const uint8_t* e = f.levels[0].log2_extent;
      ok = f.levels[0].kind == VF_RAW && e[0] == e[1] && e[1] == e[2];
      a = e[0];
    }
    if (ok) switch ((a << 24) | (l1.kind << 20) | ((uint32_t)l1.depth << 12) | (l2.kind << 8) | l2.depth) {
#define VF_2S(a, k1, n1, k2, n2, kinds) \
  case ((a) << 24) | ((k1) << 20) | ((n1) << 12) | ((k2) << 8) | (n2): \
    return spec_kernel<kinds, TwoSparse<a, K_OF_##k1, n1, K_OF_##k2, n2>>(restart, mode);
        VF_2S(0, VF_SVO, 3, VF_SVDAG, 8, 6) VF_2S(0, VF_SVO, 5, VF_SVDAG, 6, 6) VF_2S(0, VF_SVO, 7, VF_SVDAG, 4, 6)
        VF_2S(4, VF_SVO, 3, VF_SVDAG, 4, 7)
        VF_2S(0, VF_SVO, 2, VF_SVDAG, 2, 6) VF_2S(1, VF_SVDAG, 1, VF_SVO, 2, 7)  // tests
#undef VF_2S
        default: break;
      }
  }
  {  // Raw / DF chains with an optional octree level below
    uint32_t nr = 0, a[3] = {0, 0, 0}, dfm = 0;
    bool ok = true;
    while (nr < f.n_levels && nr < 3 && (f.levels[nr].kind == VF_RAW || f.levels[nr].kind == VF_DF)) {
      const uint8_t* e = f.levels[nr].log2_extent;
      if (e[0] != e[1] || e[1] != e[2]) ok = false;
      a[nr] = e[0];
      if (f.levels[nr].kind == VF_DF) dfm |= 1u << nr;
      ++nr;
    }
    uint32_t sk = 0, ns = 0;
    if (ok && nr >= 1 && nr == f.n_levels - 1) {
      const vf_level& sp = f.levels[nr];
      if (sp.kind == VF_SVO || sp.kind == VF_SVDAG) {
        sk = sp.kind;
        ns = sp.depth;
      } else {
        ok = false;
      }
    } else if (nr != f.n_levels) {
      ok = false;
    }
    if (ok && nr >= 1) switch ((nr << 28) | (a[0] << 24) | (a[1] << 20) | (a[2] << 16) | (dfm << 12) | (sk << 8) | ns) {
#define VF_RC(nr, a0, a1, a2, dfm, k, ns, kinds) \
  case ((nr) << 28) | ((a0) << 24) | ((a1) << 20) | ((a2) << 16) | ((dfm) << 12) | ((k) << 8) | (ns): \
    return spec_kernel<kinds, RawChain<nr, a0, a1, a2, dfm, K_OF_##k, ns>>(restart, mode);
      // single Raw / DF grids (cfg4 R(11^3), t512 R(9^3) / D(9^3, 6), cfg2 R(8^3), cfg1 R(6^3))
      VF_RC(1, 11, 0, 0, 0, VF_NONE, 0, 1) VF_RC(1, 9, 0, 0, 0, VF_NONE, 0, 1) VF_RC(1, 9, 0, 0, 1, VF_NONE, 0, 1)
      VF_RC(1, 8, 0, 0, 0, VF_NONE, 0, 1) VF_RC(1, 6, 0, 0, 0, VF_NONE, 0, 1)
      VF_RC(1, 4, 0, 0, 0, VF_NONE, 0, 1) VF_RC(1, 4, 0, 0, 1, VF_NONE, 0, 1)  // tests
      // multi-level Raw / DF chains of the sweeps: Table 2 rows 1-3, 5 (cfg4), 21-25, 34-36 (t512),
      // cfg5 R(4^3)^3, cfg1 R(3^3)^2
      VF_RC(2, 4, 3, 0, 0, VF_SVDAG, 4, 5) VF_RC(2, 4, 3, 0, 3, VF_SVDAG, 4, 5) VF_RC(2, 4, 3, 0, 1, VF_SVDAG, 4, 5)
      VF_RC(3, 4, 4, 3, 0, VF_NONE, 0, 1)
      VF_RC(2, 3, 3, 0, 3, VF_SVDAG, 3, 5) VF_RC(2, 3, 3, 0, 1, VF_SVDAG, 3, 5) VF_RC(2, 3, 3, 0, 0, VF_SVDAG, 3, 5)
      VF_RC(3, 3, 3, 3, 0, VF_NONE, 0, 1) VF_RC(3, 4, 1, 4, 0, VF_NONE, 0, 1)
      VF_RC(2, 5, 4, 0, 3, VF_NONE, 0, 1) VF_RC(2, 5, 4, 0, 1, VF_NONE, 0, 1) VF_RC(2, 5, 4, 0, 0, VF_NONE, 0, 1)
      VF_RC(3, 4, 4, 4, 0, VF_NONE, 0, 1) VF_RC(2, 3, 3, 0, 0, VF_NONE, 0, 1)
#undef VF_RC
      default: break;
    }
  }
  if (same_format(f, kFmtG5R3)) return spec_kernel<5, SparseRaw<K_SVDAG, 1, 5, 3, 0x10, 0x1>, true>(restart, mode);
  if (same_format(f, kFmtG2R2)) return spec_kernel<5, SparseRaw<K_SVDAG, 1, 2, 2, 0x2, 0x1>>(restart, mode);
  if (same_format(f, kFmtT22T21R4)) return spec_kernel<9, SparseRaw<K_NTREE, 2, 3, 4, 0x6, 0x5>, true>(restart, mode);
  if (same_format(f, kFmtT21T22R4)) return spec_kernel<9, SparseRaw<K_NTREE, 2, 3, 4, 0x5, 0x3>>(restart, mode);
  if (same_format(f, kFmtT11T12R1)) return spec_kernel<9, SparseRaw<K_NTREE, 1, 3, 1, 0x5, 0x3>>(restart, mode);
  if (same_format(f, kFmtS5R5)) return spec_kernel<3, SparseRaw<K_SVO, 1, 5, 5, 0x10, 0x1>>(restart, mode);
  if (same_format(f, kFmtT24R3)) return spec_kernel<9, SparseRaw<K_NTREE, 2, 4, 3, 0x8, 0x1>>(restart, mode);
  if (same_format(f, kFmtT22T22R3)) return spec_kernel<9, SparseRaw<K_NTREE, 2, 4, 3, 0xA, 0x5>>(restart, mode);
  if (same_format(f, kFmtT23R5)) return spec_kernel<9, SparseRaw<K_NTREE, 2, 3, 5, 0x4, 0x1>>(restart, mode);
  if (same_format(f, kFmtS5R4)) return spec_kernel<3, SparseRaw<K_SVO, 1, 5, 4, 0x10, 0x1>>(restart, mode);
  if (same_format(f, kFmtG5R4)) return spec_kernel<5, SparseRaw<K_SVDAG, 1, 5, 4, 0x10, 0x1>>(restart, mode);
#endif
#undef VF_HAS
  return nullptr;
}

// resident blocks per SM for a persistent kernel (cached per function and device)
// bytes of the top Raw grid staged by the chunked kernels (mode 2): R(A^3) with A <= 4 on top
size_t top_stage_bytes(const Format& f) {
  const uint8_t* e = f.levels[0].log2_extent;
  return f.levels[0].kind == VF_RAW ? (size_t)4 << (e[0] + e[1] + e[2]) : 0;
}

int persistent_blocks(KernelFn fn, int device, size_t smem = 0) {
  struct Entry {
    KernelFn fn;
    int dev, blocks;
    size_t smem;
  };
  static Entry cache[256];
  static int n_cache = 0;
  static std::mutex mu;
  std::lock_guard<std::mutex> g(mu);
  for (int i = 0; i < n_cache; ++i)
    if (cache[i].fn == fn && cache[i].dev == device && cache[i].smem == smem) return cache[i].blocks;
  int per_sm = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kPersistThreads, smem);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  int blocks = (per_sm > 0 ? per_sm : 1) * (sms > 0 ? sms : 148);
  if (n_cache < 256) cache[n_cache++] = Entry{fn, device, blocks, smem};
  return blocks;
}

}  // namespace

// VF_TRACE_SCHEDULE: find / create the schedule entry of this ray array and, if it holds the
// durations of an earlier launch, compute this launch's block order (tp.order); every scheduled
// launch records its block durations (tp.cost). Returns the entry (sched_mu held through `lk`)
// or nullptr: no scheduling (natural block order), e.g. when memory is short or, inside stream
// capture, for an array not seen before (nothing may be allocated during capture).
SchedEntry* prepare_schedule(const Handle* h, const vf_ray* rays, uint64_t n, uint32_t nb, cudaStream_t s,
                             TraceParams& tp, std::unique_lock<std::mutex>& lk, bool& capturing, const void* fn,
                             unsigned threads, bool regroup) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  capturing = cs != cudaStreamCaptureStatusNone;
  lk = std::unique_lock<std::mutex>(h->sched_mu);
  SchedEntry* e = nullptr;
  for (auto& x : h->sched)
    if (x.mem && x.rays == rays && x.n == n && x.nb == nb) e = &x;
  if (!e) {
    if (capturing) return nullptr;
    // a launch of at most two waves of resident blocks has no tail to reorder (cfg1: 512 blocks
    // on 1,332 slots; the two order kernels would only add their launches)
    int per_sm = 0, sms = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, (int)threads, 0) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    if ((uint64_t)nb <= 2ull * (uint64_t)per_sm * (uint64_t)sms) return nullptr;
    for (auto& x : h->sched) {  // an empty slot, else the least recently used unpinned one
      if (x.pinned) continue;
      if (!e || !x.mem || (e->mem && x.last_use < e->last_use)) e = &x;
    }
    if (!e) return nullptr;  // every entry belongs to a captured graph
    if (e->mem) {  // evict: no launch may still use its memory
      if (e->ev) cudaEventSynchronize(e->ev);
      h->alloc.put(e->mem, e->bytes, s);
      e->mem = nullptr;
    }
    const size_t words = 2 * (size_t)nb + 2 * kSchedBuckets + 1 + 2 * (size_t)n + ((size_t)nb + 3) / 4;
    e->mem = static_cast<uint32_t*>(h->alloc.get(words * sizeof(uint32_t), s));
    if (!e->mem) return nullptr;
    if (!e->ev && cudaEventCreateWithFlags(&e->ev, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      h->alloc.put(e->mem, words * sizeof(uint32_t), s);
      e->mem = nullptr;
      return nullptr;
    }
    e->bytes = words * sizeof(uint32_t);
    e->rays = rays;
    e->n = n;
    e->nb = nb;
    e->valid = false;
    for (int i = 0; i < 4; ++i) e->tmode[i] = -1;  // (a new array: its own measurements)
    e->ms_sum[0] = e->ms_sum[1] = 0.0;
    e->ms_n[0] = e->ms_n[1] = 0;
    e->decided = -1;
    e->since = 0;
    e->last_mode = 0;
    cudaMemsetAsync(e->mem + 2 * (size_t)nb, 0, (2 * kSchedBuckets + 1) * sizeof(uint32_t), s);
  } else if (!capturing) {
    cudaStreamWaitEvent(s, e->ev, 0);  // after the launch that wrote cost (any stream)
  } else {
    e->pinned = true;  // the graph being captured reads and writes this entry on every replay
  }
  e->last_use = ++h->sched_clock;
  e->pending = -1;
  int mode = 0;  // 1: regroup the rays into warps this launch
  if (regroup) {
    constexpr uint32_t kReeval = 256;
    if (!capturing) {
      for (int i = 0; i < 4; ++i)  // harvest the timings of completed launches (never blocks)
        if (e->tmode[i] >= 0) {
          const cudaError_t q = cudaEventQuery(e->t1[i]);
          if (q == cudaSuccess) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, e->t0[i], e->t1[i]) == cudaSuccess) {
              e->ms_sum[e->tmode[i]] += ms;
              e->ms_n[e->tmode[i]] += 1;
            }
            e->tmode[i] = -1;
          }
          cudaGetLastError();  // (cudaErrorNotReady is not an error here)
        }
    }
    if (e->decided >= 0 && e->since >= kReeval) {  // re-measure now and then
      e->decided = -1;
      e->since = 0;
      e->ms_sum[0] = e->ms_sum[1] = 0.0;
      e->ms_n[0] = e->ms_n[1] = 0;
    }
    // regrouping must win by 2 % (it moves rays away from their 8x4-pixel warps: when in doubt, don't)
    const bool rg_faster = e->ms_n[0] && e->ms_n[1] && e->ms_sum[1] / e->ms_n[1] < 0.98 * (e->ms_sum[0] / e->ms_n[0]);
    if (e->decided < 0 && e->ms_n[0] >= 2 && e->ms_n[1] >= 2) e->decided = rg_faster ? 1 : 0;
    if (e->decided >= 0) {
      mode = e->decided;
    } else if (capturing) {  // a graph keeps one mode: the faster so far, else the plain schedule
      mode = rg_faster ? 1 : 0;
    } else {
      mode = (int)(e->since & 1u);  // measuring: alternate the two modes
    }
    ++e->since;
    if (!capturing && e->valid) {  // time this launch (order kernels + trace)
      const int i = e->tnext;
      e->tnext = (i + 1) & 3;
      bool ok = true;
      if (!e->t0[i]) ok = cudaEventCreate(&e->t0[i]) == cudaSuccess && cudaEventCreate(&e->t1[i]) == cudaSuccess;
      if (ok && e->tmode[i] < 0 && cudaEventRecord(e->t0[i], s) == cudaSuccess) {
        e->tmode[i] = (int8_t)mode;
        e->pending = i;
      }
      cudaGetLastError();
    }
  }
  e->last_mode = mode;
  uint32_t* cost = e->mem;
  uint32_t* order = e->mem + nb;
  uint32_t* hist = e->mem + 2 * (size_t)nb;
  uint32_t* ray_cost = hist + 2 * kSchedBuckets + 1;
  uint32_t* ray_perm = ray_cost + n;
  uint8_t* cls = reinterpret_cast<uint8_t*>(ray_perm + n);  // per-block duration class
  if (e->valid) {
    const unsigned g = (unsigned)std::min<uint32_t>(148u, (nb + 255u) / 256u);
    static const SchedCfg cfg = [] {  // A/B knobs (tools/sched_ab.py): VF_SCHED_SUB, VF_SCHED_DIL
      SchedCfg c{2u, 6u};  // A/B: +-6 blocks keeps the gain when the camera moves
      if (const char* e = getenv("VF_SCHED_SUB")) c.sub = (uint32_t)std::min(2, std::max(0, atoi(e)));
      if (const char* e = getenv("VF_SCHED_DIL")) c.dil = (uint32_t)std::min(16, std::max(0, atoi(e)));
      return c;
    }();
    sched_hist_kernel<<<g, 256, 0, s>>>(cost, nb, hist, cls, cfg);
    sched_scatter_kernel<<<g, 256, 0, s>>>(cls, nb, hist, hist + kSchedBuckets, hist + 2 * kSchedBuckets, order,
                                           cfg);
    tp.order = order;
    if (mode == 1) {
      sched_raysort_kernel<<<(unsigned)((n + kRayGroup - 1) / kRayGroup), kRayGroup, 0, s>>>(ray_cost, n, ray_perm);
      tp.ray_perm = ray_perm;
    }
  }
  tp.cost = cost;
  if (regroup) tp.ray_cost = ray_cost;
  return e;
}

uint32_t trace_launch_count(const Handle* h, const vf_ray* rays, uint64_t n, uint32_t flags) {
  if (n == 0) return 0;
  if (!(flags & VF_TRACE_SCHEDULE) || (flags & (VF_TRACE_INCOHERENT | VF_TRACE_PERSISTENT_WARPS | VF_TRACE_CHUNKED)))
    return 1;
  std::lock_guard<std::mutex> lk(h->sched_mu);
  for (const auto& x : h->sched)
    if (x.mem && x.rays == rays && x.n == n && x.valid) return (flags & VF_TRACE_REGROUP) && x.last_mode ? 4 : 3;
  return 1;
}

void free_schedules(const Handle* h) {
  std::lock_guard<std::mutex> lk(h->sched_mu);
  for (auto& x : h->sched) {
    if (x.mem) h->alloc.put(x.mem, x.bytes, h->build_stream);
    if (x.ev) cudaEventDestroy(x.ev);
    for (int i = 0; i < 4; ++i) {
      if (x.t0[i]) cudaEventDestroy(x.t0[i]);
      if (x.t1[i]) cudaEventDestroy(x.t1[i]);
    }
    x = SchedEntry{};
  }
}

vf_status launch_trace(const Handle* h, const vf_ray* rays, uint64_t n, vf_hit* hits, uint32_t flags, cudaStream_t s,
                       unsigned long long* counters, vf_payload* payload, uint32_t* touch, const uint32_t* slots) {
  if (n == 0) return VF_OK;
  uint32_t kinds = 0;
  for (uint32_t t = 0; t < h->fmt.n_tiers; ++t) kinds |= 1u << h->fmt.tiers[t].kind;
  const bool persistent = (flags & (VF_TRACE_PERSISTENT_WARPS | VF_TRACE_INCOHERENT)) != 0;
  KernelFn fn = select_kernel(kinds, (flags & VF_TRACE_RESTART_SV) != 0, counters != nullptr, persistent);
  static const bool no_spec = getenv("VF_NO_SPEC") != nullptr;  // A/B and tests: generic kernel only
  static const int chunked_env = [] {  // A/B: force the chunked kernels (1) / with staged top grid (2)
    const char* e = getenv("VF_CHUNKED");
    return e ? atoi(e) : -1;
  }();
  int mode = (flags & VF_TRACE_CHUNKED) ? ((flags & VF_TRACE_STAGE_TOP) ? 2 : 1) : 0;
  if (chunked_env >= 0) mode = chunked_env;
  bool chunked = false;
  if (!persistent && !counters && !no_spec)
    if (KernelFn sf = select_spec(h->fmt, (flags & VF_TRACE_RESTART_SV) != 0, mode, h->aligned_nodes)) {
      fn = sf;
      chunked = mode > 0;
    }
  // counting runs of the headline formats use their compiled-in traversal too (same code as timed)
  if (!persistent && counters && !no_spec)
    if (KernelFn sf = select_spec(h->fmt, (flags & VF_TRACE_RESTART_SV) != 0, -1, false)) fn = sf;
  if (!fn) {
    set_error("vf_trace: no kernel instantiated for kind set 0x%x", kinds);
    return VF_ERR_UNSUPPORTED;
  }
  if (chunked) {
    static const uint32_t chunk_env = [] {
      const char* e = getenv("VF_CHUNK");
      const int v = e ? atoi(e) : 0;
      return (uint32_t)((v >= 32 && v % 32 == 0) ? v : 0);
    }();
    static const uint32_t crefill_env = [] {
      const char* e = getenv("VF_CREFILL");
      const int v = e ? atoi(e) : 0;
      return (uint32_t)((v >= 1 && v <= 32) ? v : 0);
    }();
    TraceParams tp = h->tp;
    tp.payload = reinterpret_cast<uint2*>(payload);
    tp.touch = touch;
    tp.slot = slots;
    if (chunk_env) tp.chunk = chunk_env;
    if (crefill_env) tp.crefill = crefill_env;
    const uint32_t slot = h->work_slot.fetch_add(1) % kWorkSlots;
    const size_t smem = mode == 2 ? top_stage_bytes(h->fmt) : 0;
    const int blocks = persistent_blocks(fn, h->device, smem);
    fn<<<blocks, kTraceThreads, smem, s>>>(tp, h->buf, reinterpret_cast<const float4*>(rays),
                                           reinterpret_cast<int4*>(hits), n, counters, h->work + 2 * slot);
  } else if (persistent) {
    static const int refill_env = [] {
      const char* e = getenv("VF_REFILL");
      const int v = e ? atoi(e) : 0;
      return (v >= 1 && v <= 32) ? v : 0;
    }();
    TraceParams tp = h->tp;
    tp.payload = reinterpret_cast<uint2*>(payload);
    tp.touch = touch;
    tp.slot = slots;
    if (refill_env) tp.refill = (uint32_t)refill_env;
    const uint32_t slot = h->work_slot.fetch_add(1) % kWorkSlots;
    unsigned long long* work = h->work + 2 * slot;
    const int blocks = persistent_blocks(fn, h->device);
    fn<<<blocks, kPersistThreads, 0, s>>>(tp, h->buf, reinterpret_cast<const float4*>(rays),
                                          reinterpret_cast<int4*>(hits), n, counters, work);
  } else {
    static const unsigned threads = [] {
      const char* e = getenv("VF_BLOCK");
      const int v = e ? atoi(e) : 0;
      return (v == 32 || v == 64 || (v > 0 && v <= (int)kTraceThreads && v % 32 == 0)) ? (unsigned)v : kTraceThreads;
    }();
    const uint64_t blocks = (n + threads - 1) / threads;
    if (blocks > 0x7fffffffull) {
      set_error("vf_trace: %llu rays exceed one launch", (unsigned long long)n);
      return VF_ERR_INVALID_ARG;
    }
    TraceParams tp = h->tp;
    tp.payload = reinterpret_cast<uint2*>(payload);
    tp.touch = touch;
    tp.slot = slots;
    std::unique_lock<std::mutex> sched_lk;
    bool capturing = false;
    SchedEntry* se = nullptr;
    if ((flags & VF_TRACE_SCHEDULE) && !counters)
      se = prepare_schedule(h, rays, n, (uint32_t)blocks, s, tp, sched_lk, capturing, (const void*)fn, threads,
                            (flags & VF_TRACE_REGROUP) != 0);
#ifdef VF_BLOCK_CLOCK
    static unsigned long long* clk_buf = nullptr;
    static size_t clk_n = 0;
    if (clk_n < blocks) {
      cudaFree(clk_buf);
      cudaMalloc(&clk_buf, 3 * blocks * sizeof(unsigned long long));
      clk_n = blocks;
    }
    cudaMemcpyToSymbolAsync(g_block_clock, &clk_buf, sizeof(clk_buf), 0, cudaMemcpyHostToDevice, s);
#endif
    fn<<<(unsigned)blocks, threads, 0, s>>>(tp, h->buf, reinterpret_cast<const float4*>(rays),
                                            reinterpret_cast<int4*>(hits), n, counters, nullptr);
    if (se && !capturing && cudaEventRecord(se->ev, s) == cudaSuccess) se->valid = true;
    if (se && !capturing && se->pending >= 0 && cudaEventRecord(se->t1[se->pending], s) != cudaSuccess) {
      cudaGetLastError();
      se->tmode[se->pending] = -1;
    }
#ifdef VF_BLOCK_CLOCK
    if (const char* out = getenv("VF_BLOCK_CLOCK_OUT")) {
      std::vector<unsigned long long> hb(3 * blocks);
      cudaMemcpyAsync(hb.data(), clk_buf, hb.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      if (FILE* f = fopen(out, "ab")) {
        const unsigned long long nb = blocks;
        fwrite(&nb, sizeof(nb), 1, f);
        fwrite(hb.data(), sizeof(unsigned long long), hb.size(), f);
        fclose(f);
      }
    }
#endif
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("vf_trace: launch failed: %s", cudaGetErrorString(e));
    return VF_ERR_CUDA;
  }
  return VF_OK;
}

bool has_compiled_in_kernel(const Format& f) { return select_spec(f, false, 0, false) != nullptr; }

vf_status read_exact_calls(unsigned long long* out, bool reset) {
  VF_CUDA_TRY(cudaMemcpyFromSymbol(out, g_exact_calls, sizeof(*out)));
  if (reset) {
    const unsigned long long z = 0;
    VF_CUDA_TRY(cudaMemcpyToSymbol(g_exact_calls, &z, sizeof(z)));
  }
  return VF_OK;
}

vf_status launch_touch_count(const uint32_t* touch, uint64_t nw, unsigned long long* counters, cudaStream_t s) {
  if (nw == 0) return VF_OK;
  uint64_t blocks = (nw + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  touch_count_kernel<<<(unsigned)blocks, 256, 0, s>>>(touch, nw, counters);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("vf_trace_counters: touch count launch failed: %s", cudaGetErrorString(e));
    return VF_ERR_CUDA;
  }
  return VF_OK;
}

vf_status launch_query(const Handle* h, const uint32_t* xyz, uint64_t n, uint32_t* out, cudaStream_t s) {
  if (n == 0) return VF_OK;
  uint64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  query_kernel<<<(unsigned)blocks, 256, 0, s>>>(h->tp, h->buf, xyz, out, n);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("vf_query: launch failed: %s", cudaGetErrorString(e));
    return VF_ERR_CUDA;
  }
  return VF_OK;
}

}  // namespace vf
