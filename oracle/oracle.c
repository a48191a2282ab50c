/* oracle/oracle.c — CPU ORACLE for first-hit ray intersection. TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library. The product path (paper_2410_14128_b200/) never links,
 * imports or calls it, and it shares no code with that path: the one common module is
 * inputs/volgen.h, the seeded input-volume generator (no method arithmetic).
 *
 * WHAT IT COMPUTES (the plain definition the method reaches exactly):
 * every hybrid format is lossless ("We focus on lossless storage formats") and
 * intersection returns the first non-empty single voxel in hit-time order (PAPER.md:183-185
 * fig:function_proto `for child in ordered_hit_children ... return True`; "in
 * order of hit time"). So the oracle is a plain exact grid walk over the UNCOMPRESSED
 * dense occupancy grid, with no format and no hierarchy:
 *
 *   p(t) = o + t d, o and d the given fp32 values taken as exact dyadic rationals.
 *   tau_a(t) = floor(o_a + t d_a)     if d_a > 0
 *            = ceil(o_a + t d_a) - 1  if d_a < 0
 *            = floor(o_a)             if d_a = 0           (right-limit cell, reading A2)
 *   Visited cells C(t) = (tau_x(t+), tau_y(t+), tau_z(t+)) for t in [t_start, t_end), the
 *   segment [tmin, tmax) clipped to the root box [0,Rx)x[0,Ry)x[0,Rz) (reading A7).
 *   Result: the first C(t) whose voxel is non-empty (empty iff all 32 bits 0),
 *   t_hit = exact entry time of that cell (t_start if first), output (x,y,z)=C(t_hit),
 *   t = fp32(t_hit) (reading A4); otherwise a miss. Plane events with equal exact t step
 *   together (reading A2), so cells touched only at an edge or corner are not visited.
 *
 * HOW (SURVEY.md §8(c) c-2, step by step): the Amanatides-Woo walk ("ray march
 * through a uniform grid of voxels by finding the minimum distance needed to reach the next
 * voxel at each step") with EXACT event arithmetic instead of floating point:
 *   in the canonical domain, O = o*2^39, tmin*2^39 and D = d*2^53 are integers; the event
 *   time of plane P on axis a is T = (P - o_a)/d_a = N/D * 2^14 with N = P*2^39 - O_a,
 *   and every comparison is a sign-normalised cross multiplication below 2^114 in __int128.
 *   1. occupancy bitset (x-fastest), 2. scale inputs to integers, 3. clip to root box with
 *   exact slab times, 4. entry cell by binary search over plane indices with exact event
 *   compares, 5. loop: test cell, take exact minimum of next plane events, step every axis
 *   that attains it, stop at t_end, 6. t rounded to fp32 via long double.
 * Parallelism: OpenMP over rays, dynamic chunks of 256 (order-independent result).
 *
 * Rays outside the canonical domain are reported with status 2 (not traced). The segment bounds
 * may be negative (|tmin|, finite |tmax| in {0} U [2^-16, 2^20): the ray line behind o, reading R5).
 *
 * PINS (tests/test_oracle.py; none of these functions is "parity unpinned"; mutation check in
 * profiles/r2_oracle_mutations.md, 18 of 18 plausible mistakes turn a pin red):
 *   trace_one / oracle_trace : exact brute force (tests/brute/brute.c, >= 1e5 rays per size 4^3..32^3,
 *                              and tests/brute_force.py in Fractions), sphere / Menger / box closed forms,
 *                              mirror symmetry, empty / solid volumes;
 *   grid_from_generator      : per voxel vs the input library's evaluators (dense_host, voxels_host,
 *                              the lowest-k brute force of volgen.h);
 *   grid_procedural (G5 bins): every voxel of every object's AABB faces at 4096^3 and whole boxes;
 *   grid_from_dense          : every voxel (incl. the last) vs the input array;
 *   grid_slab_counts / count : per-slab sums of the input array.
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../inputs/volgen.h"

typedef __int128 i128;

/* ------------------------------------------------------------------ grid (step 1) */
typedef struct {
  int64_t dims[3];
  uint64_t* bits; /* bit (x + Rx*(y + Ry*z)) set iff voxel non-empty */
  int owns_gen;   /* procedural mode: evaluate volgen per visited cell, no bitset */
  vg_desc gen;
  /* procedural G5: objects binned by 64^3 cells of their AABB [c-r, c+r) */
  int64_t nb[3];
  uint32_t* bin_start; /* CSR over bins */
  vg_object* bin_obj;
} oracle_grid;

static int sparse_occupied(const oracle_grid* g, int64_t x, int64_t y, int64_t z) {
  const uint64_t b = (uint64_t)(x >> 6) + (uint64_t)g->nb[0] * ((uint64_t)(y >> 6) + (uint64_t)g->nb[1] * (uint64_t)(z >> 6));
  for (uint32_t i = g->bin_start[b]; i < g->bin_start[b + 1]; ++i)
    if (vg_object_contains(&g->bin_obj[i], x, y, z)) return 1;
  return 0;
}

static inline uint64_t lin(const oracle_grid* g, int64_t x, int64_t y, int64_t z) {
  return (uint64_t)x + (uint64_t)g->dims[0] * ((uint64_t)y + (uint64_t)g->dims[1] * (uint64_t)z);
}

static inline int occupied(const oracle_grid* g, int64_t x, int64_t y, int64_t z) {
  if (g->bits) {
    uint64_t i = lin(g, x, y, z);
    return (int)((g->bits[i >> 6] >> (i & 63)) & 1u);
  }
  if (g->bin_start) return sparse_occupied(g, x, y, z);
  return vg_voxel(&g->gen, x, y, z) != 0;
}

static oracle_grid* grid_alloc(const uint32_t dims[3]) {
  oracle_grid* g = (oracle_grid*)calloc(1, sizeof(oracle_grid));
  if (!g) return NULL;
  for (int a = 0; a < 3; ++a) g->dims[a] = dims[a];
  uint64_t nbits = (uint64_t)dims[0] * dims[1] * dims[2];
  g->bits = (uint64_t*)calloc((nbits + 63) / 64 + 1, sizeof(uint64_t));
  if (!g->bits) {
    free(g);
    return NULL;
  }
  return g;
}

/* Dense occupancy from an x-fastest RGBA array (0 = empty). */
oracle_grid* oracle_grid_from_dense(const uint32_t* rgba, const uint32_t dims[3]) {
  oracle_grid* g = grid_alloc(dims);
  if (!g) return NULL;
  uint64_t n = (uint64_t)dims[0] * dims[1] * dims[2];
  for (uint64_t i = 0; i < n; ++i)
    if (rgba[i]) g->bits[i >> 6] |= (uint64_t)1 << (i & 63);
  return g;
}

/* Dense occupancy from a generator, parallel over z-slabs (each slab owns whole 64-bit
 * words only when Rx*Ry is a multiple of 64, so use atomic OR to stay general). */
oracle_grid* oracle_grid_from_generator(const vg_desc* d, int nthreads) {
  oracle_grid* g = grid_alloc(d->dims);
  if (!g) return NULL;
  if (nthreads <= 0) nthreads = omp_get_max_threads();
  const int64_t R0 = d->dims[0], R1 = d->dims[1], R2 = d->dims[2];
  if (d->gen == VG_SPARSE) {
    /* rasterise each object over its AABB [c-r, c+r) ("the oracle
     * rasterises per object") */
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
    for (int k = 0; k < VG_SPARSE_OBJECTS; ++k) {
      vg_object o = vg_sparse_object((uint32_t)k, d->seed);
      for (int64_t z = o.c[2] - o.r; z < o.c[2] + o.r; ++z)
        for (int64_t y = o.c[1] - o.r; y < o.c[1] + o.r; ++y)
          for (int64_t x = o.c[0] - o.r; x < o.c[0] + o.r; ++x) {
            if (x < 0 || y < 0 || z < 0 || x >= R0 || y >= R1 || z >= R2) continue;
            if (!vg_object_contains(&o, x, y, z)) continue;
            uint64_t i = lin(g, x, y, z);
            __atomic_fetch_or(&g->bits[i >> 6], (uint64_t)1 << (i & 63), __ATOMIC_RELAXED);
          }
    }
    return g;
  }
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
  for (int64_t z = 0; z < R2; ++z)
    for (int64_t y = 0; y < R1; ++y) {
      uint64_t base = lin(g, 0, y, z);
      for (int64_t x = 0; x < R0; ++x) {
        if (vg_voxel(d, x, y, z)) {
          uint64_t i = base + (uint64_t)x;
          __atomic_fetch_or(&g->bits[i >> 6], (uint64_t)1 << (i & 63), __ATOMIC_RELAXED);
        }
      }
    }
  return g;
}

/* Procedural occupancy (no bitset): bit(cell) = vg_voxel(cell) != 0. Same definition,
 * used for sampled parity at sizes whose bitset is too large to build in a test. */
oracle_grid* oracle_grid_procedural(const vg_desc* d) {
  oracle_grid* g = (oracle_grid*)calloc(1, sizeof(oracle_grid));
  if (!g) return NULL;
  for (int a = 0; a < 3; ++a) g->dims[a] = d->dims[a];
  g->owns_gen = 1;
  g->gen = *d;
  if (d->gen == VG_SPARSE) {
    /* occupancy = union of the object shells (colour irrelevant): bin every object into the
     * 64^3 cells its AABB touches, two passes (count, fill) */
    for (int a = 0; a < 3; ++a) g->nb[a] = (g->dims[a] + 63) / 64;
    const uint64_t nbins = (uint64_t)g->nb[0] * g->nb[1] * g->nb[2];
    g->bin_start = (uint32_t*)calloc(nbins + 1, sizeof(uint32_t));
    if (!g->bin_start) {
      free(g);
      return NULL;
    }
    for (int pass = 0; pass < 2; ++pass) {
      uint32_t* fill = NULL;
      if (pass == 1) {
        for (uint64_t b = 0; b < nbins; ++b) g->bin_start[b + 1] += g->bin_start[b];
        g->bin_obj = (vg_object*)malloc(sizeof(vg_object) * (g->bin_start[nbins] + 1));
        fill = (uint32_t*)calloc(nbins, sizeof(uint32_t));
        if (!g->bin_obj || !fill) {
          free(fill);
          free(g->bin_obj);
          free(g->bin_start);
          free(g);
          return NULL;
        }
      }
      for (uint32_t k = 0; k < VG_SPARSE_OBJECTS; ++k) {
        vg_object o = vg_sparse_object(k, d->seed);
        int64_t lo[3], hi[3];
        int ok = 1;
        for (int a = 0; a < 3; ++a) {
          lo[a] = o.c[a] - o.r;
          hi[a] = o.c[a] + o.r - 1;
          if (lo[a] < 0) lo[a] = 0;
          if (hi[a] > g->dims[a] - 1) hi[a] = g->dims[a] - 1;
          if (hi[a] < lo[a]) ok = 0;
        }
        if (!ok) continue;
        for (int64_t bz = lo[2] >> 6; bz <= hi[2] >> 6; ++bz)
          for (int64_t by = lo[1] >> 6; by <= hi[1] >> 6; ++by)
            for (int64_t bx = lo[0] >> 6; bx <= hi[0] >> 6; ++bx) {
              const uint64_t b = (uint64_t)bx + (uint64_t)g->nb[0] * ((uint64_t)by + (uint64_t)g->nb[1] * (uint64_t)bz);
              if (pass == 0)
                g->bin_start[b + 1]++;
              else
                g->bin_obj[g->bin_start[b] + fill[b]++] = o;
            }
      }
      free(fill);
    }
  }
  return g;
}

void oracle_grid_free(oracle_grid* g) {
  if (!g) return;
  free(g->bits);
  free(g->bin_start);
  free(g->bin_obj);
  free(g);
}

uint64_t oracle_grid_count(const oracle_grid* g) {
  if (!g->bits) return 0;
  uint64_t n = (uint64_t)g->dims[0] * g->dims[1] * g->dims[2], c = 0;
  for (uint64_t w = 0; w < (n + 63) / 64; ++w) c += (uint64_t)__builtin_popcountll(g->bits[w]);
  return c;
}

/* count per z-slab (for cross-checking a GPU build's non-empty count) */
void oracle_grid_slab_counts(const oracle_grid* g, uint64_t* out) {
  for (int64_t z = 0; z < g->dims[2]; ++z) {
    uint64_t c = 0;
    for (int64_t y = 0; y < g->dims[1]; ++y)
      for (int64_t x = 0; x < g->dims[0]; ++x) c += (uint64_t)occupied(g, x, y, z);
    out[z] = c;
  }
}

int oracle_grid_get(const oracle_grid* g, int64_t x, int64_t y, int64_t z) { return occupied(g, x, y, z); }

/* occupancy at n points (n x 3 int64, inside the volume), any grid mode */
void oracle_grid_get_many(const oracle_grid* g, const int64_t* xyz, int64_t n, uint8_t* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = (uint8_t)occupied(g, xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
}

/* occupancy of the box [lo, lo + ext) as x-fastest bytes, any grid mode */
void oracle_grid_box(const oracle_grid* g, const int64_t lo[3], const int64_t ext[3], uint8_t* out) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t z = 0; z < ext[2]; ++z)
    for (int64_t y = 0; y < ext[1]; ++y)
      for (int64_t x = 0; x < ext[0]; ++x)
        out[x + ext[0] * (y + ext[1] * z)] = (uint8_t)occupied(g, lo[0] + x, lo[1] + y, lo[2] + z);
}

/* ------------------------------------------------------------------ exact times (step 2) */
/* A time value: PLANE event T = N/D * 2^14 (D != 0), SCALAR T = tau * 2^-39, or +INF. */
enum { T_PLANE = 0, T_SCALAR = 1, T_INF = 2 };
typedef struct {
  int kind;
  int64_t N, D; /* plane: numerator P*2^39 - O_a and denominator d_a*2^53 (D > 0 after normalising) */
  int64_t tau;  /* scalar */
} etime;

/* x -> integer x*2^s if exact and in range; returns 0 on failure. */
static int to_scaled(float f, int s, int64_t* out) {
  double v = ldexp((double)f, s);
  if (!(fabs(v) < 9.0e18)) return 0;
  if (v != floor(v)) return 0;
  *out = (int64_t)v;
  return 1;
}

static etime plane_time(int64_t P, int64_t O, int64_t D) {
  etime t;
  t.kind = T_PLANE;
  int64_t N = P * ((int64_t)1 << 39) - O;
  if (D < 0) {
    N = -N;
    D = -D;
  }
  t.N = N;
  t.D = D;
  t.tau = 0;
  return t;
}

static etime scalar_time(int64_t tau) {
  etime t;
  t.kind = T_SCALAR;
  t.N = t.D = 0;
  t.tau = tau;
  return t;
}

static etime inf_time(void) {
  etime t;
  t.kind = T_INF;
  t.N = t.D = t.tau = 0;
  return t;
}

/* sign(a - b) exactly. */
static int tcmp(const etime* a, const etime* b) {
  if (a->kind == T_INF || b->kind == T_INF) {
    if (a->kind == T_INF && b->kind == T_INF) return 0;
    return a->kind == T_INF ? 1 : -1;
  }
  i128 l, r;
  if (a->kind == T_PLANE && b->kind == T_PLANE) {
    /* N1/D1 vs N2/D2, D > 0 */
    l = (i128)a->N * b->D;
    r = (i128)b->N * a->D;
  } else if (a->kind == T_PLANE) {
    /* N*2^14/D vs tau*2^-39  <=>  N*2^53 vs tau*D */
    l = (i128)a->N * ((i128)1 << 53);
    r = (i128)b->tau * a->D;
  } else if (b->kind == T_PLANE) {
    l = (i128)a->tau * b->D;
    r = (i128)b->N * ((i128)1 << 53);
  } else {
    l = a->tau;
    r = b->tau;
  }
  return (l > r) - (l < r);
}

static float tfloat(const etime* t) {
  if (t->kind == T_INF) return INFINITY;
  if (t->kind == T_SCALAR) return (float)ldexpl((long double)t->tau, -39);
  long double v = (long double)t->N / (long double)t->D;
  return (float)ldexpl(v, 14);
}

/* ------------------------------------------------------------------ one ray (steps 3-6) */
/* status: 0 miss, 1 hit, 2 ray outside the canonical domain */
/* entry_axes: on a hit, the set of axes whose plane crossing entered the hit cell at t_hit (the
 * stepped axes of the last step, or the root-box entry axes when the hit cell is the first one
 * and t_start is a box-entry event later than tmin); 0 when the segment starts inside it. */
static int trace_one(const oracle_grid* g, const float* ray, int32_t* xyz, float* tout, int64_t* steps,
                     int* entry_axes) {
  const float o[3] = {ray[0], ray[1], ray[2]};
  const float d[3] = {ray[4], ray[5], ray[6]};
  const float tmin = ray[3], tmax = ray[7];
  int64_t O[3], D[3], TMIN, TMAX = 0;
  int tmax_inf = isinf(tmax) && tmax > 0;
  /* step 2: canonical-domain check + scaling */
  for (int a = 0; a < 3; ++a) {
    float ao = fabsf(o[a]), ad = fabsf(d[a]);
    if (!(ao == 0.0f || (ao >= 0x1p-16f && ao < 0x1p20f))) return 2;
    if (!(ad == 0.0f || (ad >= 0x1p-30f && ad <= 2.0f))) return 2;
    if (!to_scaled(o[a], 39, &O[a]) || !to_scaled(d[a], 53, &D[a])) return 2;
  }
  /* segment bounds may be negative (the ray line behind o; reading R5) */
  if (!(tmin == 0.0f || (fabsf(tmin) >= 0x1p-16f && fabsf(tmin) < 0x1p20f))) return 2;
  if (!tmax_inf && !(tmax == 0.0f || (fabsf(tmax) >= 0x1p-16f && fabsf(tmax) < 0x1p20f))) return 2;
  if (!to_scaled(tmin, 39, &TMIN)) return 2;
  if (!tmax_inf && !to_scaled(tmax, 39, &TMAX)) return 2;
  if (D[0] == 0 && D[1] == 0 && D[2] == 0) return 0; /* reading A5: all-zero d is a miss */
  if (!tmax_inf && !(tmin < tmax)) return 0;

  /* step 3: clip [tmin, tmax) to the root box with exact slab times */
  etime ts = scalar_time(TMIN);
  etime te = tmax_inf ? inf_time() : scalar_time(TMAX);
  for (int a = 0; a < 3; ++a) {
    if (D[a] == 0) {
      /* half-open membership: floor(o_a) in [0, R_a)  <=>  0 <= o_a < R_a */
      if (O[a] < 0 || O[a] >= g->dims[a] * ((int64_t)1 << 39)) return 0;
      continue;
    }
    etime en = plane_time(D[a] > 0 ? 0 : g->dims[a], O[a], D[a]);
    etime ex = plane_time(D[a] > 0 ? g->dims[a] : 0, O[a], D[a]);
    if (tcmp(&en, &ts) > 0) ts = en;
    if (tcmp(&ex, &te) < 0) te = ex;
  }
  if (tcmp(&ts, &te) >= 0) return 0;
  int last_axes = 0; /* axes whose voxel-slab entry plane is crossed exactly at the current t */

  /* step 4: entry cell tau_b(t_start+) by binary search over plane indices */
  int64_t cell[3];
  for (int b = 0; b < 3; ++b) {
    if (D[b] == 0) {
      cell[b] = O[b] >> 39; /* floor(o_b), o_b >= 0 here */
      continue;
    }
    int64_t lo = 0, hi = g->dims[b] - 1;
    if (D[b] > 0) {
      /* largest k in [0,R-1] with T_b(k) <= t_start (T_b increasing in k) */
      while (lo < hi) {
        int64_t mid = (lo + hi + 1) / 2;
        etime tm = plane_time(mid, O[b], D[b]);
        if (tcmp(&tm, &ts) <= 0) lo = mid; else hi = mid - 1;
      }
    } else {
      /* cell k <=> T_b(k+1) <= t < T_b(k); smallest k with T_b(k+1) <= t_start
       * (T_b decreasing in k) */
      while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        etime tm = plane_time(mid + 1, O[b], D[b]);
        if (tcmp(&tm, &ts) <= 0) hi = mid; else lo = mid + 1;
      }
    }
    cell[b] = lo;
  }

  /* entry face of the first cell: every axis whose voxel-slab entry plane (d>0: plane cell,
   * d<0: plane cell+1) is crossed exactly at t_start, provided t_start > tmin (otherwise the
   * segment starts inside the cell) */
  {
    etime tm = scalar_time(TMIN);
    if (tcmp(&ts, &tm) > 0)
      for (int a = 0; a < 3; ++a) {
        if (D[a] == 0) continue;
        etime en = plane_time(D[a] > 0 ? cell[a] : cell[a] + 1, O[a], D[a]);
        if (tcmp(&en, &ts) == 0) last_axes |= 1 << a;
      }
  }

  /* step 5: walk */
  etime tcur = ts;
  int64_t n = 0;
  for (;;) {
    ++n;
    if (cell[0] < 0 || cell[1] < 0 || cell[2] < 0 || cell[0] >= g->dims[0] || cell[1] >= g->dims[1] ||
        cell[2] >= g->dims[2])
      return 0; /* unreachable: t_end bounds the walk inside the box */
    if (occupied(g, cell[0], cell[1], cell[2])) {
      xyz[0] = (int32_t)cell[0];
      xyz[1] = (int32_t)cell[1];
      xyz[2] = (int32_t)cell[2];
      *tout = tfloat(&tcur); /* step 6 */
      if (steps) *steps = n;
      if (entry_axes) *entry_axes = last_axes;
      return 1;
    }
    etime nx[3];
    int have = 0;
    etime best = inf_time();
    for (int a = 0; a < 3; ++a) {
      if (D[a] == 0) {
        nx[a] = inf_time();
        continue;
      }
      nx[a] = plane_time(D[a] > 0 ? cell[a] + 1 : cell[a], O[a], D[a]);
      if (!have || tcmp(&nx[a], &best) < 0) best = nx[a];
      have = 1;
    }
    if (tcmp(&best, &te) >= 0) {
      if (steps) *steps = n;
      return 0;
    }
    last_axes = 0;
    for (int a = 0; a < 3; ++a)
      if (D[a] != 0 && tcmp(&nx[a], &best) == 0) {
        cell[a] += D[a] > 0 ? 1 : -1;
        last_axes |= 1 << a;
      }
    tcur = best;
  }
}

/* rays: n x 8 floats (vf_ray layout). Outputs: xyz n x 3 (-1 on miss), t (+inf on miss),
 * status n (0 miss, 1 hit, 2 non-canonical), steps n (cells visited; may be NULL).
 * Returns the number of non-canonical rays. */
/* normal: optional n x 3 int8 entry-face normal (-sign(d_a) on the lowest entry axis, else 0) */
int64_t oracle_trace(const oracle_grid* g, const float* rays, int64_t n, int32_t* xyz, float* t, uint8_t* status,
                     int64_t* steps, int8_t* normal, int nthreads) {
  if (nthreads <= 0) nthreads = omp_get_max_threads();
  int64_t bad = 0;
#pragma omp parallel for schedule(dynamic, 256) num_threads(nthreads) reduction(+ : bad)
  for (int64_t i = 0; i < n; ++i) {
    int32_t h[3] = {-1, -1, -1};
    float tt = INFINITY;
    int64_t s = 0;
    int ax = 0;
    int st = trace_one(g, rays + 8 * i, h, &tt, &s, &ax);
    if (st != 1) {
      h[0] = h[1] = h[2] = -1;
      tt = INFINITY;
    }
    if (st == 2) ++bad;
    xyz[3 * i + 0] = h[0];
    xyz[3 * i + 1] = h[1];
    xyz[3 * i + 2] = h[2];
    t[i] = tt;
    if (status) status[i] = (uint8_t)st;
    if (steps) steps[i] = s;
    if (normal) {
      normal[3 * i] = normal[3 * i + 1] = normal[3 * i + 2] = 0;
      if (st == 1 && ax) {
        const int a = __builtin_ctz(ax);
        normal[3 * i + a] = rays[8 * i + 4 + a] > 0.0f ? -1 : 1;
      }
    }
  }
  return bad;
}

int oracle_max_threads(void) { return omp_get_max_threads(); }
