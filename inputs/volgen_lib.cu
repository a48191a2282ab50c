// inputs/volgen_lib.cu — materialise the seeded procedural volumes of inputs/volgen.h.
//
// INPUT DEFINITION ONLY (task rule ③): this library produces the voxel data that the
// product's vf_build consumes (a device voxel list or a dense array) and that tests feed to
// the oracle. It contains no ray, traversal or format arithmetic.
//
//   vg_dense_host    : x-fastest dense RGBA array on the host (small volumes, tests)
//   vg_dense_device  : same, written on the device
//   vg_count_device  : number of non-empty voxels (GPU, brick-parallel)
//   vg_extract_device: device voxel list {key = x | y<<21 | z<<42, rgba}, unspecified order
//
// G5 (sparse shells) is evaluated with a host-built 64^3-bin object table so that each voxel
// tests only the objects whose AABB overlaps its bin, in ascending k (lowest k wins).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "volgen.h"

namespace {

constexpr int kBin = 64;

struct SparseTable {
  int nb[3] = {0, 0, 0};
  std::vector<uint32_t> start;  // CSR over bins (x-fastest)
  std::vector<vg_object> objs;  // objects per bin, ascending k
};

void build_sparse_table(const vg_desc* d, SparseTable* t) {
  for (int a = 0; a < 3; ++a) t->nb[a] = (int)((d->dims[a] + kBin - 1) / kBin);
  const size_t nbins = (size_t)t->nb[0] * t->nb[1] * t->nb[2];
  std::vector<std::vector<uint32_t>> lists(nbins);
  for (uint32_t k = 0; k < VG_SPARSE_OBJECTS; ++k) {
    vg_object o = vg_sparse_object(k, d->seed);
    int lo[3], hi[3];
    bool ok = true;
    for (int a = 0; a < 3; ++a) {
      int64_t l = (int64_t)o.c[a] - o.r, h = (int64_t)o.c[a] + o.r - 1;
      if (l < 0) l = 0;
      if (h > (int64_t)d->dims[a] - 1) h = (int64_t)d->dims[a] - 1;
      if (h < l) ok = false;
      lo[a] = (int)(l / kBin);
      hi[a] = (int)(h / kBin);
    }
    if (!ok) continue;
    for (int z = lo[2]; z <= hi[2]; ++z)
      for (int y = lo[1]; y <= hi[1]; ++y)
        for (int x = lo[0]; x <= hi[0]; ++x)
          lists[(size_t)x + (size_t)t->nb[0] * ((size_t)y + (size_t)t->nb[1] * z)].push_back(k);
  }
  t->start.assign(nbins + 1, 0);
  for (size_t b = 0; b < nbins; ++b) t->start[b + 1] = t->start[b] + (uint32_t)lists[b].size();
  t->objs.resize(t->start[nbins]);
  for (size_t b = 0; b < nbins; ++b)
    for (size_t i = 0; i < lists[b].size(); ++i) t->objs[t->start[b] + i] = vg_sparse_object(lists[b][i], d->seed);
}

struct DevSparse {
  int nb[3];
  const uint32_t* start;
  const vg_object* objs;
};

__host__ __device__ inline uint32_t sparse_voxel(const vg_desc& d, const int nb[3], const uint32_t* start,
                                                 const vg_object* objs, int64_t x, int64_t y, int64_t z) {
  size_t b = (size_t)(x / kBin) + (size_t)nb[0] * ((size_t)(y / kBin) + (size_t)nb[1] * (size_t)(z / kBin));
  for (uint32_t i = start[b]; i < start[b + 1]; ++i)
    if (vg_object_contains(&objs[i], x, y, z)) return vg_apply_tex(objs[i].col, x, y, z, d.seed, d.tex);
  return 0;
}

__device__ inline uint32_t eval(const vg_desc& d, const DevSparse& sp, int64_t x, int64_t y, int64_t z) {
  if (d.gen == VG_SPARSE) return sparse_voxel(d, sp.nb, sp.start, sp.objs, x, y, z);
  return vg_voxel(&d, x, y, z);
}

// One 8x8x8 brick per 512-thread block.
__device__ inline bool brick_voxel(const vg_desc& d, uint64_t brick, int64_t* x, int64_t* y, int64_t* z) {
  const uint64_t bx = (d.dims[0] + 7) / 8, by = (d.dims[1] + 7) / 8;
  const int64_t X = (int64_t)(brick % bx) * 8 + (threadIdx.x & 7);
  const int64_t Y = (int64_t)((brick / bx) % by) * 8 + ((threadIdx.x >> 3) & 7);
  const int64_t Z = (int64_t)(brick / (bx * by)) * 8 + (threadIdx.x >> 6);
  *x = X;
  *y = Y;
  *z = Z;
  return X < d.dims[0] && Y < d.dims[1] && Z < d.dims[2];
}

__device__ inline bool brick_skip(const vg_desc& d, const DevSparse& sp, uint64_t brick) {
  if (d.gen == VG_EMPTY) return true;
  if (d.gen != VG_SPARSE) return false;
  const uint64_t bx = (d.dims[0] + 7) / 8, by = (d.dims[1] + 7) / 8;
  const int64_t X = (int64_t)(brick % bx) * 8, Y = (int64_t)((brick / bx) % by) * 8, Z = (int64_t)(brick / (bx * by)) * 8;
  size_t b = (size_t)(X / kBin) + (size_t)sp.nb[0] * ((size_t)(Y / kBin) + (size_t)sp.nb[1] * (size_t)(Z / kBin));
  return sp.start[b] == sp.start[b + 1];
}

__global__ void __launch_bounds__(512) k_count(vg_desc d, DevSparse sp, uint64_t brick0, unsigned long long* count) {
  const uint64_t brick = brick0 + blockIdx.x;
  if (brick_skip(d, sp, brick)) return;
  int64_t x, y, z;
  int occ = 0;
  if (brick_voxel(d, brick, &x, &y, &z)) occ = eval(d, sp, x, y, z) != 0;
  int n = __syncthreads_count(occ);
  if (threadIdx.x == 0 && n) atomicAdd(count, (unsigned long long)n);
}

__global__ void __launch_bounds__(512) k_extract(vg_desc d, DevSparse sp, uint64_t brick0, uint64_t* keys,
                                                 uint32_t* rgba, uint64_t cap, unsigned long long* cursor) {
  __shared__ uint32_t warp_n[16];
  __shared__ unsigned long long base;
  const uint64_t brick = brick0 + blockIdx.x;
  if (brick_skip(d, sp, brick)) return;
  int64_t x, y, z;
  uint32_t c = 0;
  if (brick_voxel(d, brick, &x, &y, &z)) c = eval(d, sp, x, y, z);
  const unsigned m = __ballot_sync(0xffffffffu, c != 0);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) warp_n[w] = __popc(m);
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t tot = 0;
    for (int i = 0; i < 16; ++i) {
      uint32_t t = warp_n[i];
      warp_n[i] = tot;
      tot += t;
    }
    base = tot ? atomicAdd(cursor, (unsigned long long)tot) : 0ull;
  }
  __syncthreads();
  if (c) {
    uint64_t i = base + warp_n[w] + __popc(m & ((1u << lane) - 1u));
    if (i < cap) {
      keys[i] = (uint64_t)x | ((uint64_t)y << 21) | ((uint64_t)z << 42);
      rgba[i] = c;
    }
  }
}

__global__ void k_dense(vg_desc d, DevSparse sp, uint32_t* out, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    int64_t x = (int64_t)(i % d.dims[0]), y = (int64_t)((i / d.dims[0]) % d.dims[1]),
            z = (int64_t)(i / ((uint64_t)d.dims[0] * d.dims[1]));
    out[i] = eval(d, sp, x, y, z);
  }
}

struct DevSparseOwner {
  DevSparse v{};
  void* mem = nullptr;
  ~DevSparseOwner() {
    if (mem) cudaFree(mem);
  }
  cudaError_t init(const vg_desc* d) {
    static const uint32_t zero2[2] = {0, 0};
    if (d->gen != VG_SPARSE) {
      // dummy one-bin table so brick_skip never dereferences null
      cudaError_t e = cudaMalloc(&mem, sizeof(zero2));
      if (e) return e;
      e = cudaMemcpy(mem, zero2, sizeof(zero2), cudaMemcpyHostToDevice);
      v.nb[0] = v.nb[1] = v.nb[2] = 1;
      v.start = (const uint32_t*)mem;
      v.objs = nullptr;
      return e;
    }
    SparseTable t;
    build_sparse_table(d, &t);
    size_t sb = t.start.size() * sizeof(uint32_t), ob = t.objs.size() * sizeof(vg_object);
    size_t off = (sb + 255) & ~(size_t)255;
    cudaError_t e = cudaMalloc(&mem, off + ob + 16);
    if (e) return e;
    e = cudaMemcpy(mem, t.start.data(), sb, cudaMemcpyHostToDevice);
    if (e) return e;
    if (ob) e = cudaMemcpy((char*)mem + off, t.objs.data(), ob, cudaMemcpyHostToDevice);
    for (int a = 0; a < 3; ++a) v.nb[a] = t.nb[a];
    v.start = (const uint32_t*)mem;
    v.objs = (const vg_object*)((char*)mem + off);
    return e;
  }
};

uint64_t n_bricks(const vg_desc* d) {
  return (uint64_t)((d->dims[0] + 7) / 8) * ((d->dims[1] + 7) / 8) * ((d->dims[2] + 7) / 8);
}

constexpr uint64_t kMaxGrid = 1ull << 30;

}  // namespace

extern "C" {

// 0 on success, CUDA error code otherwise.
int vg_count_device(const vg_desc* d, uint64_t* count, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  DevSparseOwner sp;
  cudaError_t e = sp.init(d);
  if (e) return (int)e;
  unsigned long long* c = nullptr;
  e = cudaMalloc(&c, sizeof(*c));
  if (e) return (int)e;
  cudaMemsetAsync(c, 0, sizeof(*c), s);
  const uint64_t nb = n_bricks(d);
  for (uint64_t b0 = 0; b0 < nb; b0 += kMaxGrid) {
    uint64_t g = nb - b0 < kMaxGrid ? nb - b0 : kMaxGrid;
    k_count<<<(unsigned)g, 512, 0, s>>>(*d, sp.v, b0, c);
  }
  unsigned long long h = 0;
  cudaMemcpyAsync(&h, c, sizeof(h), cudaMemcpyDeviceToHost, s);
  e = cudaStreamSynchronize(s);
  cudaFree(c);
  *count = h;
  return (int)(e ? e : cudaGetLastError());
}

// keys/rgba: device arrays of capacity cap. *count receives the number written (== the
// total non-empty count when cap suffices).
int vg_extract_device(const vg_desc* d, uint64_t* keys, uint32_t* rgba, uint64_t cap, uint64_t* count,
                      void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  DevSparseOwner sp;
  cudaError_t e = sp.init(d);
  if (e) return (int)e;
  unsigned long long* c = nullptr;
  e = cudaMalloc(&c, sizeof(*c));
  if (e) return (int)e;
  cudaMemsetAsync(c, 0, sizeof(*c), s);
  const uint64_t nb = n_bricks(d);
  for (uint64_t b0 = 0; b0 < nb; b0 += kMaxGrid) {
    uint64_t g = nb - b0 < kMaxGrid ? nb - b0 : kMaxGrid;
    k_extract<<<(unsigned)g, 512, 0, s>>>(*d, sp.v, b0, keys, rgba, cap, c);
  }
  unsigned long long h = 0;
  cudaMemcpyAsync(&h, c, sizeof(h), cudaMemcpyDeviceToHost, s);
  e = cudaStreamSynchronize(s);
  cudaFree(c);
  *count = h;
  return (int)(e ? e : cudaGetLastError());
}

int vg_dense_device(const vg_desc* d, uint32_t* out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  DevSparseOwner sp;
  cudaError_t e = sp.init(d);
  if (e) return (int)e;
  uint64_t n = (uint64_t)d->dims[0] * d->dims[1] * d->dims[2];
  k_dense<<<148 * 8, 256, 0, s>>>(*d, sp.v, out, n);
  e = cudaStreamSynchronize(s);
  return (int)(e ? e : cudaGetLastError());
}

// Host dense generation (x-fastest). Returns 0.
int vg_dense_host(const vg_desc* d, uint32_t* out) {
  const uint64_t n = (uint64_t)d->dims[0] * d->dims[1] * d->dims[2];
  if (d->gen == VG_SPARSE) {
    SparseTable t;
    build_sparse_table(d, &t);
    for (uint64_t i = 0; i < n; ++i) {
      int64_t x = (int64_t)(i % d->dims[0]), y = (int64_t)((i / d->dims[0]) % d->dims[1]),
              z = (int64_t)(i / ((uint64_t)d->dims[0] * d->dims[1]));
      out[i] = sparse_voxel(*d, t.nb, t.start.data(), t.objs.data(), x, y, z);
    }
    return 0;
  }
  for (uint64_t i = 0; i < n; ++i) {
    int64_t x = (int64_t)(i % d->dims[0]), y = (int64_t)((i / d->dims[0]) % d->dims[1]),
            z = (int64_t)(i / ((uint64_t)d->dims[0] * d->dims[1]));
    out[i] = vg_voxel(d, x, y, z);
  }
  return 0;
}

// Voxel words at n points xyz (n x 3 int64) on the host (any generator; sparse through the
// 64^3-bin object table, built once per call). Points outside the volume read 0.
int vg_voxels_host(const vg_desc* d, const int64_t* xyz, uint64_t n, uint32_t* out) {
  SparseTable t;
  if (d->gen == VG_SPARSE) build_sparse_table(d, &t);
  for (uint64_t i = 0; i < n; ++i) {
    const int64_t x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
    if (x < 0 || y < 0 || z < 0 || x >= d->dims[0] || y >= d->dims[1] || z >= d->dims[2]) {
      out[i] = 0;
      continue;
    }
    out[i] = d->gen == VG_SPARSE ? sparse_voxel(*d, t.nb, t.start.data(), t.objs.data(), x, y, z) : vg_voxel(d, x, y, z);
  }
  return 0;
}

// The G5 object table: out[6k..6k+5] = {cx, cy, cz, r, box, col} of object k (k < 4096).
void vg_sparse_objects(uint32_t seed, int32_t* out) {
  for (uint32_t k = 0; k < VG_SPARSE_OBJECTS; ++k) {
    const vg_object o = vg_sparse_object(k, seed);
    const int32_t v[6] = {o.c[0], o.c[1], o.c[2], o.r, o.box, (int32_t)o.col};
    memcpy(out + 6 * k, v, sizeof(v));
  }
}

// Single voxel on the host (any generator; sparse via brute force over objects).
uint32_t vg_voxel_host(const vg_desc* d, int64_t x, int64_t y, int64_t z) {
  if (d->gen == VG_SPARSE) {
    if (x < 0 || y < 0 || z < 0 || x >= d->dims[0] || y >= d->dims[1] || z >= d->dims[2]) return 0;
    return vg_sparse_voxel_brute(d->seed, d->tex, x, y, z);
  }
  return vg_voxel(d, x, y, z);
}

}  // extern "C"
