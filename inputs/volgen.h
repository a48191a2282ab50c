/* inputs/volgen.h — seeded, integer-only procedural volume generators.
 *
 * INPUT DEFINITION ONLY. This header defines the synthetic volumes that both
 * the CPU oracle (oracle/) and the GPU product path (paper_2410_14128_b200/)
 * consume. It holds none of the method's arithmetic: no ray, no DDA, no format.
 * It is the one module the two sides share (task rule ③: "only the seeded input
 * generators serve both, from a module of their own").
 *
 * Voxels are 32-bit RGBA words; a voxel is empty iff all 32 bits are 0
 * (§3 "A voxel is 'empty' if all of its 32 bits are 0").
 * Coordinates are integer voxel indices, voxel (x,y,z) occupies [x,x+1)x[y,y+1)x[z,z+1).
 *
 * Generator definitions G1..G5 follow SURVEY.md §8(d) "L0 generator definitions"
 * (the paper's meshes San Miguel/Hairball/Buddha/Sponza, are not
 * available; these are their procedural analogues). All arithmetic is u32 with
 * wrap-around or int64; no floating point, so host and device agree bit for bit.
 */
#ifndef VOLGEN_H
#define VOLGEN_H

#include <stdint.h>

#if defined(__CUDACC__)
#define VG_HD __host__ __device__ __forceinline__
#else
#define VG_HD static inline
#endif

enum {
  VG_EMPTY = 0,   /* all voxels empty */
  VG_SPHERE = 1,  /* G1: p[0] = r                                   */
  VG_MENGER = 2,  /* G2: p[0] = k (sponge level, occupies [0,3^k)^3) */
  VG_TERRAIN = 3, /* G3: heightfield with caves, seed               */
  VG_CITY = 4,    /* G4: city blocks, seed, tex                     */
  VG_SPARSE = 5,  /* G5: 4096 shell objects (needs object table)    */
  VG_RANDOM = 6,  /* iid occupancy: occupied iff hash < p[0] (u32)   */
  VG_BOX = 7,     /* solid box [p0,p3)x[p1,p4)x[p2,p5)              */
  VG_SINGLE = 8,  /* single voxel at (p0,p1,p2)                     */
  VG_SOLID = 9,   /* every voxel occupied                           */
  VG_NUM_GENERATORS = 10
};

typedef struct {
  uint32_t gen;     /* VG_* */
  uint32_t dims[3]; /* volume resolution per axis */
  uint32_t seed;
  uint32_t tex;     /* 1: per-2^3-texel colour perturbation (SURVEY §8d TEX=1) */
  int32_t p[8];     /* generator parameters, see enum */
} vg_desc;

VG_HD uint32_t vg_lowbias32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

VG_HD uint32_t vg_hash3(int64_t x, int64_t y, int64_t z, uint32_t s) {
  return vg_lowbias32(((uint32_t)x * 73856093u) ^ ((uint32_t)y * 19349663u) ^
                      ((uint32_t)z * 83492791u) ^ vg_lowbias32(s));
}

VG_HD uint32_t vg_pal(uint32_t i) {
  switch (i & 7u) {
    case 0: return 0xFF9AA5B1u;
    case 1: return 0xFF6B7B8Cu;
    case 2: return 0xFFC8B89Au;
    case 3: return 0xFF8C5A3Cu;
    case 4: return 0xFFD0D0D0u;
    case 5: return 0xFF4A5A6Au;
    case 6: return 0xFFB0A080u;
    default: return 0xFF7A6A5Au;
  }
}

/* smooth16(f) = (f*f*(3*65536 - 2*f)) >> 32, f in [0, 65536] */
VG_HD int64_t vg_smooth16(int64_t f) { return (f * f * (3 * 65536 - 2 * f)) >> 32; }

/* 2-D value noise over (x,z) at cell size 2^k; result in [0, 65536). */
VG_HD int64_t vg_vn2(int64_t x, int64_t z, int k, uint32_t s) {
  int64_t i = x >> k, j = z >> k;
  int64_t m = ((int64_t)1 << k) - 1;
  int64_t sx = vg_smooth16((x & m) << (16 - k));
  int64_t sz = vg_smooth16((z & m) << (16 - k));
  int64_t v00 = vg_hash3(i, 0, j, s) >> 16;
  int64_t v10 = vg_hash3(i + 1, 0, j, s) >> 16;
  int64_t v01 = vg_hash3(i, 0, j + 1, s) >> 16;
  int64_t v11 = vg_hash3(i + 1, 0, j + 1, s) >> 16;
  int64_t A = v00 * 65536 + (v10 - v00) * sx;
  int64_t B = v01 * 65536 + (v11 - v01) * sx;
  return (A * 65536 + (B - A) * sz) >> 32;
}

/* 3-D value noise at cell size 2^k; result in [0, 65536). */
VG_HD int64_t vg_vn3(int64_t x, int64_t y, int64_t z, int k, uint32_t s) {
  int64_t i = x >> k, j = y >> k, l = z >> k;
  int64_t m = ((int64_t)1 << k) - 1;
  int64_t sx = vg_smooth16((x & m) << (16 - k));
  int64_t sy = vg_smooth16((y & m) << (16 - k));
  int64_t sz = vg_smooth16((z & m) << (16 - k));
  int64_t Y[2];
  for (int d = 0; d < 2; ++d) {
    int64_t X[2];
    for (int b = 0; b < 2; ++b) {
      int64_t c0 = vg_hash3(i, j + b, l + d, s) >> 16;
      int64_t c1 = vg_hash3(i + 1, j + b, l + d, s) >> 16;
      X[b] = c0 * 65536 + (c1 - c0) * sx;
    }
    Y[d] = (X[0] * 65536 + (X[1] - X[0]) * sy) >> 16;
  }
  return (Y[0] * 65536 + (Y[1] - Y[0]) * sz) >> 32;
}

/* G1 sphere: occupied iff (2x+1-R)^2+(2y+1-R)^2+(2z+1-R)^2 <= (2r)^2 (R = dims[0]). */
VG_HD uint32_t vg_sphere(int64_t x, int64_t y, int64_t z, int64_t R, int64_t r) {
  int64_t a = 2 * x + 1 - R, b = 2 * y + 1 - R, c = 2 * z + 1 - R;
  if (a * a + b * b + c * c > 4 * r * r) return 0;
  return 0xFF000000u | (uint32_t)((0x40 + 3 * x) & 0xFF) | ((uint32_t)((0x40 + 3 * y) & 0xFF) << 8) |
         ((uint32_t)((0x40 + 3 * z) & 0xFF) << 16);
}

/* G2 Menger sponge of level k in [0,3^k)^3: filled iff no base-3 digit position
 * has >= 2 of (x,y,z) equal to 1. */
VG_HD uint32_t vg_menger(int64_t x, int64_t y, int64_t z, int k) {
  int64_t n = 1;
  for (int i = 0; i < k; ++i) n *= 3;
  if (x >= n || y >= n || z >= n) return 0;
  int64_t X = x, Y = y, Z = z;
  for (int i = 0; i < k; ++i) {
    int ones = (X % 3 == 1) + (Y % 3 == 1) + (Z % 3 == 1);
    if (ones >= 2) return 0;
    X /= 3; Y /= 3; Z /= 3;
  }
  int64_t s = n / 3; /* 81 for k = 5 */
  if (s == 0) s = 1;
  return vg_pal((uint32_t)(x / s + 3 * (y / s) + 9 * (z / s)));
}

/* G3 terrain (heightfield + caves), R = 1024. */
VG_HD int64_t vg_terrain_height(int64_t x, int64_t z, uint32_t s) {
  return 320 + ((vg_vn2(x, z, 8, s) * 192 + vg_vn2(x, z, 7, s + 1) * 96 + vg_vn2(x, z, 6, s + 2) * 48 +
                 vg_vn2(x, z, 5, s + 3) * 24) >> 16);
}
VG_HD uint32_t vg_terrain(int64_t x, int64_t y, int64_t z, uint32_t s) {
  int64_t h = vg_terrain_height(x, z, s);
  if (y > h) return 0;
  if (y < h - 6) {
    int64_t c = (2 * vg_vn3(x, y, z, 6, s + 10) + vg_vn3(x, y, z, 5, s + 11)) / 3;
    int64_t dc = c - 32768;
    if (dc < 0) dc = -dc;
    if (dc < 2600) return 0;
  }
  return y >= h - 1 ? 0xFF3C9A3Cu : (y >= h - 8 ? 0xFF2A4A6Bu : 0xFF808080u);
}

/* G4 city blocks, R = 2048. */
VG_HD uint32_t vg_city(int64_t x, int64_t y, int64_t z, uint32_t s) {
  if (y < 16) return 0xFF404040u;
  int64_t u = x % 160, v = z % 160;
  if (u < 32 || v < 32) return 0;
  int64_t bx = x / 160, bz = z / 160;
  int64_t li = (u - 32) / 64, lj = (v - 32) / 64, lu = (u - 32) % 64, lv = (v - 32) % 64;
  uint32_t hb = vg_hash3(2 * bx + li, 7, 2 * bz + lj, s);
  int64_t H = 48 + (int64_t)(hb % 1400u);
  int64_t top = 16 + H;
  uint32_t col = vg_pal((hb >> 12) & 7u);
  int cyl = ((hb >> 20) % 10u) == 0;
  if (!cyl) {
    if (!(lu >= 4 && lu < 60 && lv >= 4 && lv < 60 && y < top)) return 0;
    int64_t du = lu < 32 ? lu - 4 : 59 - lu;
    int64_t dv = lv < 32 ? lv - 4 : 59 - lv;
    int64_t dy = top - 1 - y;
    int64_t d = du < dv ? du : dv;
    if (dy < d) d = dy;
    if (d >= 2) return 0;
    if (d == 0 && dy >= 2) {
      int64_t t = du < dv ? lv : lu;
      int64_t fy = (y - 16) % 12, ft = t % 10;
      if (fy >= 3 && fy < 9 && ft >= 2 && ft < 8) return 0;
    }
    if (d == 1 && dy >= 2) return 0xFF904020u;
    return col;
  }
  int64_t a = 2 * lu + 1 - 64, b = 2 * lv + 1 - 64;
  int64_t r2 = a * a + b * b;
  if (y < top) return (r2 > 52 * 52 && r2 <= 56 * 56) ? col : 0;
  int64_t e = 2 * (y - top) + 1;
  int64_t s2 = r2 + e * e;
  return (s2 > 52 * 52 && s2 <= 56 * 56) ? col : 0;
}

/* G5 sparse shells: object k (0..4095). */
#define VG_SPARSE_OBJECTS 4096
typedef struct {
  int32_t c[3];
  int32_t r;
  int32_t box;
  uint32_t col;
} vg_object;

VG_HD int32_t vg_sparse_rt(uint32_t i) {
  /* RT[i] = round(6 * 8^(i/64)), i in [0,64) */
  switch (i & 63u) {
    case 0: case 1: case 2: return 6;
    case 3: case 4: case 5: case 6: return 7;
    case 7: case 8: case 9: case 10: return 8;
    case 11: case 12: case 13: case 14: return 9;
    case 15: case 16: case 17: return 10;
    case 18: case 19: case 20: return 11;
    case 21: case 22: return 12;
    case 23: case 24: return 13;
    case 25: case 26: case 27: return 14;
    case 28: case 29: return 15;
    case 30: case 31: return 16;
    case 32: return 17;
    case 33: case 34: return 18;
    case 35: case 36: return 19;
    case 37: return 20;
    case 38: case 39: return 21;
    case 40: return 22;
    case 41: case 42: return 23;
    case 43: return 24;
    case 44: return 25;
    case 45: return 26;
    case 46: return 27;
    case 47: return 28;
    case 48: case 49: return 29;
    case 50: return 30;
    case 51: return 31;
    case 52: return 33;
    case 53: return 34;
    case 54: return 35;
    case 55: return 36;
    case 56: return 37;
    case 57: return 38;
    case 58: return 39;
    case 59: return 41;
    case 60: return 42;
    case 61: return 44;
    case 62: return 45;
    default: return 46;
  }
}

VG_HD vg_object vg_sparse_object(uint32_t k, uint32_t s) {
  vg_object o;
  for (int a = 0; a < 3; ++a) o.c[a] = 64 + (int32_t)(vg_hash3(k, 1, a, s) % 3968u);
  o.r = vg_sparse_rt(vg_hash3(k, 3, 0, s) & 63u);
  o.box = (vg_hash3(k, 2, 0, s) % 4u) == 0;
  o.col = vg_pal(vg_hash3(k, 4, 0, s) & 7u);
  return o;
}

/* Does object o contain voxel (x,y,z)? (shell of thickness 2) */
VG_HD int vg_object_contains(const vg_object* o, int64_t x, int64_t y, int64_t z) {
  int64_t r = o->r;
  if (o->box) {
    int64_t d[3] = {x - o->c[0], y - o->c[1], z - o->c[2]};
    int64_t m = 1 << 30;
    for (int a = 0; a < 3; ++a) {
      if (d[a] < -r || d[a] >= r) return 0;
      int64_t e = d[a] < 0 ? d[a] + r : r - 1 - d[a];
      if (e < m) m = e;
    }
    return m < 2;
  }
  int64_t a = 2 * x + 1 - 2 * (int64_t)o->c[0], b = 2 * y + 1 - 2 * (int64_t)o->c[1],
          c = 2 * z + 1 - 2 * (int64_t)o->c[2];
  int64_t q = a * a + b * b + c * c;
  return q > (2 * r - 4) * (2 * r - 4) && q <= 4 * r * r;
}

/* Voxel word for every generator except VG_SPARSE (which needs an object table:
 * see vg_sparse_voxel_brute / the binned evaluators in volgen_gpu.cu and the
 * oracle's per-object rasteriser). */
VG_HD uint32_t vg_apply_tex(uint32_t c, int64_t x, int64_t y, int64_t z, uint32_t s, uint32_t tex) {
  if (tex && c) c ^= vg_hash3(x >> 1, y >> 1, z >> 1, s ^ 0x55u) & 0x001F1F1Fu;
  return c;
}

VG_HD uint32_t vg_voxel(const vg_desc* g, int64_t x, int64_t y, int64_t z) {
  if (x < 0 || y < 0 || z < 0 || x >= g->dims[0] || y >= g->dims[1] || z >= g->dims[2]) return 0;
  uint32_t c = 0;
  switch (g->gen) {
    case VG_SPHERE: c = vg_sphere(x, y, z, g->dims[0], g->p[0]); break;
    case VG_MENGER: c = vg_menger(x, y, z, g->p[0]); break;
    case VG_TERRAIN: c = vg_terrain(x, y, z, g->seed); break;
    case VG_CITY: c = vg_city(x, y, z, g->seed); break;
    case VG_RANDOM: {
      uint32_t h = vg_hash3(x, y, z, g->seed);
      c = h < (uint32_t)g->p[0] ? (vg_hash3(x, y, z, g->seed ^ 0xC0FFEEu) | 0xFF000000u) : 0u;
      break;
    }
    case VG_BOX:
      c = (x >= g->p[0] && y >= g->p[1] && z >= g->p[2] && x < g->p[3] && y < g->p[4] && z < g->p[5])
              ? 0xFF20C0E0u
              : 0u;
      break;
    case VG_SINGLE: c = (x == g->p[0] && y == g->p[1] && z == g->p[2]) ? 0xFFFFFFFFu : 0u; break;
    case VG_SOLID: c = 0xFF808080u; break;
    default: c = 0; break; /* VG_EMPTY; VG_SPARSE handled elsewhere */
  }
  return vg_apply_tex(c, x, y, z, g->seed, g->tex);
}

/* Reference (slow) sparse evaluation: lowest k whose shell contains the voxel. */
VG_HD uint32_t vg_sparse_voxel_brute(uint32_t seed, uint32_t tex, int64_t x, int64_t y, int64_t z) {
  for (uint32_t k = 0; k < VG_SPARSE_OBJECTS; ++k) {
    vg_object o = vg_sparse_object(k, seed);
    if (vg_object_contains(&o, x, y, z)) return vg_apply_tex(o.col, x, y, z, seed, tex);
  }
  return 0;
}

#endif /* VOLGEN_H */
