/* tests/brute/brute.c — exact BRUTE-FORCE first hit: a TEST PIN for the oracle (not the oracle).
 *
 * SURVEY.md §8(c) c-1, "Equivalent brute-force form": voxel v is pierced iff
 *     max(t_start, t_enter(v)) < min(t_end, t_exit(v))        (strictly positive length)
 * with half-open membership on zero-direction axes; the result is the pierced non-empty voxel
 * of minimum entry time, which is unique (reading A21). No walk, no plane ordering, no binary
 * search: every non-empty voxel of the volume is slab-tested against every ray. It shares no
 * code with oracle/oracle.c (nor with the CUDA path); tests/brute_force.py is the same
 * definition in Python Fractions for the small cases, this file scales it to >= 1e5 rays per
 * volume up to 32^3.
 *
 * Exact arithmetic: in the canonical domain (vf.h) o_a*2^39, d_a*2^53, tmin*2^39 and finite
 * tmax*2^39 are integers. Axis a's cell v has the slab {t : v <= o_a + t d_a < v + 1} for
 * d_a > 0 and {t : v < o_a + t d_a <= v + 1} for d_a < 0 (right-limit cells, reading A2), so
 * its end points are the plane times  t(P) = (P - o_a)/d_a = (P*2^39 - O_a) / D_a * 2^14.
 * Every time is kept as the exact fraction  t / 2^14 = num / den  (den > 0); comparisons are
 * cross-multiplications below 2^114 in __int128.
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>

typedef __int128 i128;
typedef struct {
  int64_t num, den; /* den == 0: +infinity */
} frac;

static int fcmp(frac a, frac b) { /* sign(a - b) */
  if (!a.den || !b.den) return (!a.den) - (!b.den);
  const i128 l = (i128)a.num * b.den, r = (i128)b.num * a.den;
  return (l > r) - (l < r);
}

static int scaled(float f, int s, int64_t* out) {
  const double v = ldexp((double)f, s);
  if (!(fabs(v) < 9.0e18) || v != floor(v)) return 0;
  *out = (int64_t)v;
  return 1;
}

/* occ: x-fastest bytes (0 = empty). Per ray: status (0 miss, 1 hit, 2 outside the domain,
 * 3 two pierced voxels share the minimum entry time — impossible by the definition), hit xyz,
 * t/2^14 = tnum/tden exactly, entry-axis mask (axes whose slab entry equals the hit time, when
 * that time is later than tmin). */
void brute_trace(const uint8_t* occ, const int32_t dims[3], const float* rays, int64_t n, int32_t* xyz,
                 int64_t* tnum, int64_t* tden, uint8_t* status, uint8_t* entry_axes, int nthreads) {
  if (nthreads <= 0) nthreads = omp_get_max_threads();
  const int R[3] = {dims[0], dims[1], dims[2]};
  const int Rmax = R[0] > R[1] ? (R[0] > R[2] ? R[0] : R[2]) : (R[1] > R[2] ? R[1] : R[2]);
#pragma omp parallel num_threads(nthreads)
  {
    frac* en = (frac*)malloc(sizeof(frac) * 3 * (size_t)Rmax);
    frac* ex = (frac*)malloc(sizeof(frac) * 3 * (size_t)Rmax);
#pragma omp for schedule(dynamic, 64)
    for (int64_t i = 0; i < n; ++i) {
      const float* r = rays + 8 * i;
      int64_t O[3], D[3], T0, T1 = 0;
      int ok = 1;
      for (int a = 0; a < 3; ++a) ok &= scaled(r[a], 39, &O[a]) && scaled(r[4 + a], 53, &D[a]);
      const int tinf = isinf(r[7]) && r[7] > 0;
      ok &= scaled(r[3], 39, &T0) && (tinf || scaled(r[7], 39, &T1));
      xyz[3 * i] = xyz[3 * i + 1] = xyz[3 * i + 2] = -1;
      tnum[i] = 0;
      tden[i] = 0;
      entry_axes[i] = 0;
      if (!ok) {
        status[i] = 2;
        continue;
      }
      status[i] = 0;
      if (!D[0] && !D[1] && !D[2]) continue;
      const frac tmin = {T0, (int64_t)1 << 53};
      const frac tmax = tinf ? (frac){0, 0} : (frac){T1, (int64_t)1 << 53};
      if (fcmp(tmin, tmax) >= 0) continue;
      /* per axis: slab [en, ex) of every cell index; the candidate index range (slabs meeting
       * [tmin, tmax)); a zero-direction axis has the one index floor(o_a) for all t */
      int lo[3], hi[3];
      for (int a = 0; a < 3; ++a) {
        frac* E = en + (size_t)a * Rmax;
        frac* X = ex + (size_t)a * Rmax;
        if (!D[a]) {
          const int64_t c = O[a] >> 39; /* floor */
          lo[a] = (int)c;
          hi[a] = (int)c;
          if (c < 0 || c >= R[a]) hi[a] = lo[a] - 1;
          continue;
        }
        const int64_t den = D[a] > 0 ? D[a] : -D[a];
        lo[a] = R[a];
        hi[a] = -1;
        for (int v = 0; v < R[a]; ++v) {
          /* plane P time: sign(D) (P 2^39 - O) / |D| */
          const int64_t p0 = (int64_t)v * ((int64_t)1 << 39) - O[a], p1 = (int64_t)(v + 1) * ((int64_t)1 << 39) - O[a];
          if (D[a] > 0) {
            E[v] = (frac){p0, den};
            X[v] = (frac){p1, den};
          } else {
            E[v] = (frac){-p1, den};
            X[v] = (frac){-p0, den};
          }
          if (fcmp(E[v], tmax) < 0 && fcmp(X[v], tmin) > 0) {
            if (v < lo[a]) lo[a] = v;
            hi[a] = v;
          }
        }
      }
      int found = 0, dup = 0, bx = -1, by = -1, bz = -1, bax = 0;
      frac best = {0, 0};
      for (int z = lo[2]; z <= hi[2]; ++z)
        for (int y = lo[1]; y <= hi[1]; ++y)
          for (int x = lo[0]; x <= hi[0]; ++x) {
            if (!occ[(size_t)x + (size_t)R[0] * ((size_t)y + (size_t)R[1] * (size_t)z)]) continue;
            const int v[3] = {x, y, z};
            frac s = tmin, e = tmax;
            for (int a = 0; a < 3; ++a) {
              if (!D[a]) continue;
              const frac ea = en[(size_t)a * Rmax + v[a]], xa = ex[(size_t)a * Rmax + v[a]];
              if (fcmp(ea, s) > 0) s = ea;
              if (fcmp(xa, e) < 0) e = xa;
            }
            if (fcmp(s, e) >= 0) continue; /* not pierced (zero length at most) */
            const int c = found ? fcmp(s, best) : -1;
            if (c < 0) {
              found = 1;
              dup = 0;
              best = s;
              bx = x;
              by = y;
              bz = z;
              bax = 0;
              if (fcmp(s, tmin) > 0)
                for (int a = 0; a < 3; ++a)
                  if (D[a] && fcmp(en[(size_t)a * Rmax + v[a]], s) == 0) bax |= 1 << a;
            } else if (c == 0) {
              dup = 1;
            }
          }
      if (!found) continue;
      status[i] = dup ? 3 : 1;
      xyz[3 * i] = bx;
      xyz[3 * i + 1] = by;
      xyz[3 * i + 2] = bz;
      tnum[i] = best.num;
      tden[i] = best.den;
      entry_axes[i] = (uint8_t)bax;
    }
    free(en);
    free(ex);
  }
}
