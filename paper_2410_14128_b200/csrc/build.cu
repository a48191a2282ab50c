// build.cu — bottom-up GPU construction of a hybrid-format buffer (vf_build).
//
// Semantics follow the paper's construction (§4.1; pseudo-code
// fig:function_proto PAPER.md:172-180): every level maps the lower indices of a sub-volume to
// a constructed sub-volume; an empty child is stored as pointer 0; non-empty sub-volumes are
// written to the buffer and referenced by word offset; SVDAG levels keep a de-duplication map
// and emit a node only on a map miss; with whole-level de-duplication one map
// serves every sub-volume of a level. The layout of each base format is
// PAPER.md:84-162 (fig:layout): Raw = flat array of terminating integers; SVO node =
// {first-child pointer or TermInt, masks}; SVDAG node = {masks, popc(valid) child pointers}
// or a 1-word leaf TermInt; masks = valid bits 0-7, leaf bits 8-15 (reading A10).
//
// The paper's builder is an out-of-core CPU recursion in Morton order;
// that is prior art, not the blueprint. Here the whole volume is processed level by level
// ("tier" by tier, see vf_internal.cuh) on the GPU: non-empty voxels are sorted by Morton
// code, so the children of every node are a contiguous run in child order (octant index
// x + 2y + 4z == the Morton 3-bit group, reading A10); each tier groups its children into
// nodes, writes the nodes' words, and hands one reference per node to the tier above.
// SVDAG de-duplication is exact hash-consing: records are sorted by a 64-bit content hash
// and every record is compared word by word with its run leader (collisions fall back to a
// scan of the run), so the stored node SET — and hence bytes_used — is deterministic.
#include <thrust/device_malloc_allocator.h>
#include <thrust/device_vector.h>
#include <thrust/execution_policy.h>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/scan.h>
#include <thrust/sort.h>
#include <thrust/transform_reduce.h>
#include <thrust/transform_scan.h>
#include <thrust/count.h>
#include <thrust/copy.h>
#include <thrust/reduce.h>
#include <thrust/transform.h>
#include <thrust/functional.h>

#include <chrono>
#include <stdexcept>
#include <string>
#include <vector>

#include "vf_internal.cuh"

namespace vf {
namespace {

// ---------------------------------------------------------------- Morton helpers
__host__ __device__ inline uint64_t spread3(uint64_t v) {  // 21 bits -> every third bit
  v &= 0x1fffffull;
  v = (v | (v << 32)) & 0x1f00000000ffffull;
  v = (v | (v << 16)) & 0x1f0000ff0000ffull;
  v = (v | (v << 8)) & 0x100f00f00f00f00full;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}
__host__ __device__ inline uint32_t compact3(uint64_t v) {
  v &= 0x1249249249249249ull;
  v = (v ^ (v >> 2)) & 0x10c30c30c30c30c3ull;
  v = (v ^ (v >> 4)) & 0x100f00f00f00f00full;
  v = (v ^ (v >> 8)) & 0x1f0000ff0000ffull;
  v = (v ^ (v >> 16)) & 0x1f00000000ffffull;
  v = (v ^ (v >> 32)) & 0x1fffffull;
  return (uint32_t)v;
}
__host__ __device__ inline uint64_t morton(uint32_t x, uint32_t y, uint32_t z) {
  return spread3(x) | (spread3(y) << 1) | (spread3(z) << 2);
}

// ---------------------------------------------------------------- build memory
// Every device allocation of a build — vectors and the algorithms' temporary storage — goes
// through the caller's vf_allocator (vf_build's `alloc`; torch's caching allocator from Python),
// requested on the build stream. The allocator of the running build is thread-local.
thread_local const DevAllocator* tl_alloc = nullptr;
thread_local cudaStream_t tl_stream = nullptr;

void* build_get(size_t bytes) {
  void* p = tl_alloc ? tl_alloc->get(bytes, tl_stream) : nullptr;
  if (!p) throw std::bad_alloc();
  return p;
}
void build_put(void* p, size_t bytes) {
  if (tl_alloc) tl_alloc->put(p, bytes, tl_stream);
}

template <class T>
struct BuildAlloc : thrust::device_malloc_allocator<T> {
  using base = thrust::device_malloc_allocator<T>;
  using pointer = typename base::pointer;
  using size_type = typename base::size_type;
  template <class U>
  struct rebind {
    typedef BuildAlloc<U> other;
  };
  BuildAlloc() = default;
  template <class U>
  BuildAlloc(const BuildAlloc<U>&) {}
  pointer allocate(size_type n) { return pointer(static_cast<T*>(build_get(n * sizeof(T)))); }
  void deallocate(pointer p, size_type n) noexcept { build_put(thrust::raw_pointer_cast(p), n * sizeof(T)); }
};
template <class T>
using dvec = thrust::device_vector<T, BuildAlloc<T>>;

struct TmpAlloc {  // temporary storage of thrust algorithms
  typedef char value_type;
  char* allocate(std::ptrdiff_t n) { return static_cast<char*>(build_get((size_t)n)); }
  void deallocate(char* p, size_t n) { build_put(p, n); }
};
TmpAlloc g_tmp_alloc;

inline auto policy(cudaStream_t s) { return thrust::cuda::par(g_tmp_alloc).on(s); }

template <class V>
auto raw(V& v) {
  return thrust::raw_pointer_cast(v.data());
}

constexpr int kThreads = 256;
inline unsigned grid_for(uint64_t n) {
  uint64_t g = (n + kThreads - 1) / kThreads;
  if (g > 148ull * 64) g = 148ull * 64;
  return (unsigned)(g ? g : 1);
}
#define GRID_STRIDE(i, n) for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (n); i += (uint64_t)gridDim.x * blockDim.x)

// ---------------------------------------------------------------- input normalisation
__global__ void k_dense_keys(const uint32_t* rgba, const uint64_t* idx, uint64_t n, uint32_t Rx, uint32_t Ry,
                             uint64_t* keys, uint32_t* vals) {
  GRID_STRIDE(i, n) {
    uint64_t l = idx[i];
    uint32_t x = (uint32_t)(l % Rx), y = (uint32_t)((l / Rx) % Ry), z = (uint32_t)(l / ((uint64_t)Rx * Ry));
    keys[i] = morton(x, y, z);
    vals[i] = rgba[l];
  }
}

__global__ void k_sparse_keys(const uint64_t* in_keys, const uint32_t* in_vals, uint64_t n, uint32_t Rx, uint32_t Ry,
                              uint32_t Rz, uint64_t* keys, uint32_t* vals, unsigned long long* bad) {
  GRID_STRIDE(i, n) {
    uint64_t k = in_keys[i];
    uint32_t x = (uint32_t)(k & 0x1fffff), y = (uint32_t)((k >> 21) & 0x1fffff), z = (uint32_t)((k >> 42) & 0x1fffff);
    uint32_t v = in_vals[i];
    if (x >= Rx || y >= Ry || z >= Rz || v == 0 || (k >> 63)) atomicAdd(bad, 1ull);
    keys[i] = morton(x, y, z);
    vals[i] = v;
  }
}

__global__ void k_dup_check(const uint64_t* keys, uint64_t n, unsigned long long* bad) {
  GRID_STRIDE(i, n) {
    if (i > 0 && keys[i] == keys[i - 1]) atomicAdd(bad, 1ull);
  }
}

__global__ void k_vals_to_refs(const uint32_t* vals, uint64_t n, uint4* refs) {
  GRID_STRIDE(i, n) { refs[i] = make_uint4(vals[i], 0, 0, 0); }
}

// ---------------------------------------------------------------- grouping children into nodes
struct NodeKeyOp {
  uint32_t shift;  // 3*lf, or 64 for the root tier (single node)
  __host__ __device__ uint64_t operator()(uint64_t k) const { return shift >= 64 ? 0ull : (k >> shift); }
};

__global__ void k_flags(const uint64_t* ck, uint64_t n, uint32_t shift, uint32_t* flags) {
  NodeKeyOp op{shift};
  GRID_STRIDE(i, n) { flags[i] = (i == 0 || op(ck[i]) != op(ck[i - 1])) ? 1u : 0u; }
}

// node_of[i] = inclusive_scan(flags)[i] - 1
__global__ void k_node_starts(const uint64_t* ck, const uint32_t* node_of, uint64_t n, uint32_t shift,
                              uint64_t* node_start, uint64_t* node_key) {
  NodeKeyOp op{shift};
  GRID_STRIDE(i, n) {
    if (i == 0 || node_of[i] != node_of[i - 1]) {
      node_start[node_of[i]] = i;
      node_key[node_of[i]] = op(ck[i]);
    }
  }
}

// local child index of child key ck within its node (tier with fan-out lf; tier 0 uses lf0)
__device__ inline void local_xyz(uint64_t ck, bool root, uint32_t lf, uint32_t* lx, uint32_t* ly, uint32_t* lz) {
  uint32_t x = compact3(ck), y = compact3(ck >> 1), z = compact3(ck >> 2);
  if (!root) {
    uint32_t m = (1u << lf) - 1u;
    x &= m;
    y &= m;
    z &= m;
  }
  *lx = x;
  *ly = y;
  *lz = z;
}

// ---------------------------------------------------------------- RAW tier
// cw = words per cell: 1 (Raw) or 2 (DF: {TermInt, L1 distance})
__global__ void k_raw_scatter(const uint64_t* ck, const uint4* cr, const uint32_t* node_of, uint64_t n, bool root,
                              uint32_t lf, uint32_t lfx, uint32_t lfy, uint64_t F, uint32_t cw, uint32_t* arr) {
  GRID_STRIDE(i, n) {
    uint32_t lx, ly, lz;
    local_xyz(ck[i], root, lf, &lx, &ly, &lz);
    uint64_t li = root ? ((uint64_t)lx + ((uint64_t)ly << lfx) + ((uint64_t)lz << (lfx + lfy)))
                       : ((uint64_t)lx + ((uint64_t)ly << lf) + ((uint64_t)lz << (2 * lf)));
    arr[((uint64_t)node_of[i] * F + li) * cw] = cr[i].x;
  }
}

// DF: L1 distance of every cell to the nearest non-empty cell of its grid ("the L1
// norm distance to the nearest non-empty voxel"; construction PAPER.md:197), capped at M. The
// L1 distance transform is separable: exact two-pass (forward / backward) 1-D min-plus sweeps
// along x, then y, then z. One thread per line of one node.
constexpr uint32_t kDfInf = 1u << 24;

__global__ void k_df_init(uint32_t* arr, uint64_t cells) {
  GRID_STRIDE(i, cells) { arr[2 * i + 1] = arr[2 * i] ? 0u : kDfInf; }
}

__global__ void k_df_pass(uint32_t* arr, uint64_t M, uint32_t lfx, uint32_t lfy, uint32_t lfz, int axis) {
  const uint32_t l[3] = {lfx, lfy, lfz};
  const uint32_t la = l[axis], lo0 = l[(axis + 1) % 3], lo1 = l[(axis + 2) % 3];
  const uint64_t F = 1ull << (lfx + lfy + lfz);
  const uint64_t lines = M << (lo0 + lo1);
  const uint64_t sh[3] = {0, lfx, (uint64_t)lfx + lfy};  // cell index = x + (y << lfx) + (z << lfx+lfy)
  GRID_STRIDE(j, lines) {
    const uint64_t m = j >> (lo0 + lo1);
    const uint64_t u = j & ((1ull << lo0) - 1), v = (j >> lo0) & ((1ull << lo1) - 1);
    const uint64_t base = m * F + (u << sh[(axis + 1) % 3]) + (v << sh[(axis + 2) % 3]);
    const uint64_t step = 1ull << sh[axis];
    const uint64_t len = 1ull << la;
    uint32_t prev = kDfInf;
    for (uint64_t k = 0; k < len; ++k) {
      uint32_t* d = arr + 2 * (base + k * step) + 1;
      const uint32_t x = min(*d, prev + 1);
      *d = x;
      prev = x;
    }
    prev = kDfInf;
    for (uint64_t k = len; k-- > 0;) {
      uint32_t* d = arr + 2 * (base + k * step) + 1;
      const uint32_t x = min(*d, prev + 1);
      *d = x;
      prev = x;
    }
  }
}

__global__ void k_df_cap(uint32_t* arr, uint64_t cells, uint32_t dmax) {
  GRID_STRIDE(i, cells) { arr[2 * i + 1] = min(arr[2 * i + 1], dmax); }
}

__global__ void k_raw_refs(uint64_t M, uint64_t base, uint64_t F, uint4* nr) {
  GRID_STRIDE(m, M) { nr[m] = make_uint4((uint32_t)(base + m * F), 0, 0, 0); }
}

// ---------------------------------------------------------------- SVO / N^3-tree tiers (inline children)
// per-node size in words; SVO: 2*cnt (+2 standalone root); NTree: (top?4:0) + s*cnt rounded to 4
__global__ void k_inline_sizes(const uint64_t* node_start, uint64_t M, uint64_t n, uint32_t kind, bool top, bool last,
                               uint64_t* size, uint64_t* paper) {
  GRID_STRIDE(m, M) {
    uint64_t cnt = (m + 1 < M ? node_start[m + 1] : n) - node_start[m];
    uint64_t s, p;
    if (kind == K_SVO) {
      s = p = 2 * cnt + (top ? 2 : 0);
    } else {
      p = (top ? 4 : 0) + (last ? 1 : 4) * cnt;
      s = (p + 3) & ~3ull;
    }
    size[m] = s;
    paper[m] = p;
  }
}

__global__ void k_inline_write(const uint64_t* ck, const uint4* cr, const uint64_t* node_start, uint64_t M, uint64_t n,
                               uint32_t kind, bool root, bool top, bool last, uint32_t lf, const uint64_t* off,
                               uint64_t base, uint32_t* arr, uint4* nr) {
  GRID_STRIDE(m, M) {
    const uint64_t s0 = node_start[m], s1 = m + 1 < M ? node_start[m + 1] : n;
    const uint64_t o = off[m];
    if (kind == K_SVO) {
      // [children block: 2 words per valid child, in octant order][standalone node if top]
      uint32_t valid = 0;
      for (uint64_t i = s0; i < s1; ++i) {
        uint32_t lx, ly, lz;
        local_xyz(ck[i], root, lf, &lx, &ly, &lz);
        valid |= 1u << (lx | (ly << 1) | (lz << 2));
        const uint64_t w = o + 2 * (i - s0);
        arr[w] = cr[i].x;                  // child's first word: pointer or TermInt (leaf)
        arr[w + 1] = last ? 0u : cr[i].y;  // child's masks (leaf node: 0)
      }
      const uint32_t masks = valid | ((last ? valid : 0u) << 8);
      const uint32_t blk = (uint32_t)(base + o);
      if (top) {
        const uint64_t w = o + 2 * (s1 - s0);
        arr[w] = blk;
        arr[w + 1] = masks;
        nr[m] = make_uint4((uint32_t)(base + w), 0, 0, 0);
      } else {
        nr[m] = make_uint4(blk, masks, 0, 0);
      }
    } else {
      // N^3-tree: [standalone node if top][children block, stride 4 (internal) or 1 (TermInt)]
      uint64_t mask = 0;
      const uint64_t blk = o + (top ? 4 : 0);
      const uint32_t stride = last ? 1u : 4u;
      // child order is j = x + N y + N^2 z (reading A13), which is NOT the Morton order of the
      // sorted children when N > 2: build the mask first, then place each child at its rank.
      for (uint64_t i = s0; i < s1; ++i) {
        uint32_t lx, ly, lz;
        local_xyz(ck[i], root, lf, &lx, &ly, &lz);
        mask |= 1ull << (lx | (ly << lf) | (lz << (2 * lf)));
      }
      for (uint64_t i = s0; i < s1; ++i) {
        uint32_t lx, ly, lz;
        local_xyz(ck[i], root, lf, &lx, &ly, &lz);
        const uint32_t j = lx | (ly << lf) | (lz << (2 * lf));
        const uint64_t rank = (uint64_t)__popcll(mask & ((1ull << j) - 1ull));
        const uint64_t w = blk + stride * rank;
        const uint4 c = cr[i];
        arr[w] = c.x;
        if (!last) {
          arr[w + 1] = c.y;
          arr[w + 2] = c.z;
          arr[w + 3] = 0;
        }
      }
      const uint4 node = make_uint4((uint32_t)mask, (uint32_t)(mask >> 32), (uint32_t)(base + blk), 0u);
      if (top) {
        arr[o] = node.x;
        arr[o + 1] = node.y;
        arr[o + 2] = node.z;
        arr[o + 3] = 0;
        nr[m] = make_uint4((uint32_t)(base + o), 0, 0, 0);
      } else {
        nr[m] = node;
      }
    }
  }
}

// ---------------------------------------------------------------- SVDAG tiers (de-duplicated)
struct Records {  // m records of up to 9 words
  dvec<uint32_t> words;  // m * 9
  dvec<uint8_t> len;
  dvec<uint64_t> svid;
};

__device__ inline uint64_t mix64(uint64_t h) {
  h ^= h >> 33;
  h *= 0xff51afd7ed558ccdull;
  h ^= h >> 33;
  h *= 0xc4ceb9fe1a85ec53ull;
  h ^= h >> 33;
  return h;
}

__global__ void k_rec_hash(const uint32_t* words, const uint8_t* len, const uint64_t* svid, uint64_t m, uint64_t* h,
                           uint32_t* idx) {
  GRID_STRIDE(i, m) {
    uint64_t x = mix64(svid[i] * 0x9E3779B97F4A7C15ull + len[i]);
    for (int k = 0; k < len[i]; ++k) x = mix64(x ^ (words[i * 9 + k] + 0x632BE59BD9B4E019ull * (k + 1)));
    h[i] = x;
    idx[i] = (uint32_t)i;
  }
}

__device__ inline bool rec_eq(const uint32_t* words, const uint8_t* len, const uint64_t* svid, uint64_t a, uint64_t b) {
  if (len[a] != len[b] || svid[a] != svid[b]) return false;
  for (int k = 0; k < len[a]; ++k)
    if (words[a * 9 + k] != words[b * 9 + k]) return false;
  return true;
}

// run_start[p] = p if run begins at p (hash differs from p-1), else 0; then max-scan
__global__ void k_run_flags(const uint64_t* h, uint64_t m, uint64_t* rs) {
  GRID_STRIDE(p, m) { rs[p] = (p == 0 || h[p] != h[p - 1]) ? p : 0; }
}

// uniq_words: words the record occupies if it is its run's representative, padded to a multiple
// of `pad` (VF_BUILD_ALIGN_NODES: 4 words = 16 B); uniq_len: the same without padding
__global__ void k_rep(const uint32_t* words, const uint8_t* len, const uint64_t* svid, const uint32_t* sidx,
                      const uint64_t* rs, uint64_t m, uint32_t pad, uint32_t* rep, uint32_t* uniq_words,
                      uint32_t* uniq_len) {
  GRID_STRIDE(p, m) {
    const uint32_t me = sidx[p];
    uint64_t q = rs[p];
    uint32_t r = sidx[q];
    if (!rec_eq(words, len, svid, me, r)) {
      // hash collision inside the run: first earlier record with identical content, else me
      r = me;
      for (uint64_t k = q + 1; k < p; ++k)
        if (rec_eq(words, len, svid, me, sidx[k])) {
          r = sidx[k];
          break;
        }
    }
    rep[me] = r;
    uniq_words[me] = (r == me) ? (len[me] + pad - 1) / pad * pad : 0u;
    uniq_len[me] = (r == me) ? len[me] : 0u;
  }
}

__global__ void k_rec_write(const uint32_t* words, const uint8_t* len, const uint32_t* rep, const uint64_t* off,
                            uint64_t m, uint64_t base, uint32_t* arr, uint32_t* ptr) {
  GRID_STRIDE(i, m) {
    if (rep[i] == i) {
      for (int k = 0; k < len[i]; ++k) arr[off[i] + k] = words[i * 9 + k];
    }
    ptr[i] = (uint32_t)(base + off[rep[i]]);
  }
}

// Hash-cons m records. Unique records are laid out in record order (first occurrence, i.e.
// Morton order of the sub-volume that first needs them) starting at arr_off within `arr`
// (whose global word offset is base). Returns words written (each record padded to a multiple of
// `pad` words); *paper_words = the same without padding; ptr[i] = global pointer.
uint64_t dedup(Records& R, uint64_t m, dvec<uint32_t>& arr, uint64_t arr_off, uint64_t base,
               dvec<uint32_t>& ptr, uint64_t* n_unique, cudaStream_t s, uint32_t pad = 1,
               uint64_t* paper_words = nullptr) {
  auto pol = policy(s);
  dvec<uint64_t> h(m);
  dvec<uint32_t> sidx(m);
  k_rec_hash<<<grid_for(m), kThreads, 0, s>>>(raw(R.words), raw(R.len), raw(R.svid), m, raw(h), raw(sidx));
  thrust::sort_by_key(pol, h.begin(), h.end(), sidx.begin());  // radix sort: stable
  dvec<uint64_t> rs(m);
  k_run_flags<<<grid_for(m), kThreads, 0, s>>>(raw(h), m, raw(rs));
  thrust::inclusive_scan(pol, rs.begin(), rs.end(), rs.begin(), thrust::maximum<uint64_t>());
  dvec<uint32_t> rep(m), uw(m), ul(m);
  k_rep<<<grid_for(m), kThreads, 0, s>>>(raw(R.words), raw(R.len), raw(R.svid), raw(sidx), raw(rs), m, pad, raw(rep),
                                          raw(uw), raw(ul));
  dvec<uint64_t> off(m);
  thrust::transform_exclusive_scan(
      pol, uw.begin(), uw.end(), off.begin(), [] __device__(uint32_t v) { return (uint64_t)v; }, (uint64_t)arr_off,
      thrust::plus<uint64_t>());
  {  // the host reads below follow the kernels on s
    const cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) throw std::runtime_error(std::string("dedup: ") + cudaGetErrorString(e));
  }
  uint64_t last_off = off[m - 1];
  uint32_t last_w = uw[m - 1];
  uint64_t total = last_off + last_w - arr_off;
  if (arr.size() < arr_off + total) arr.resize(arr_off + total, 0u);
  ptr.resize(m);
  k_rec_write<<<grid_for(m), kThreads, 0, s>>>(raw(R.words), raw(R.len), raw(rep), raw(off), m, base, raw(arr),
                                                raw(ptr));
  *n_unique = thrust::count_if(pol, uw.begin(), uw.end(), [] __device__(uint32_t v) { return v != 0; });
  if (paper_words)
    *paper_words = thrust::transform_reduce(
        pol, ul.begin(), ul.end(), [] __device__(uint32_t v) -> uint64_t { return (uint64_t)v; }, (uint64_t)0,
        thrust::plus<uint64_t>());
  return total;
}

__global__ void k_leaf_records(const uint64_t* ck, const uint4* cr, uint64_t n, bool whole, uint32_t depth,
                               uint32_t* words, uint8_t* len, uint64_t* svid) {
  GRID_STRIDE(i, n) {
    words[i * 9] = cr[i].x;
    len[i] = 1;
    // sub-volume of a leaf at depth L of a level whose top is `depth` tiers up: ck >> 3(depth+1)
    svid[i] = whole ? 0ull : (ck[i] >> (3 * (depth + 1)));
  }
}

__global__ void k_node_records(const uint64_t* ck, const uint4* cr, const uint32_t* leafptr, const uint64_t* node_start,
                               const uint64_t* node_key, uint64_t M, uint64_t n, bool root, bool last, bool whole,
                               uint32_t depth, uint32_t* words, uint8_t* len, uint64_t* svid) {
  GRID_STRIDE(m, M) {
    const uint64_t s0 = node_start[m], s1 = m + 1 < M ? node_start[m + 1] : n;
    uint32_t valid = 0;
    for (uint64_t i = s0; i < s1; ++i) {
      uint32_t lx, ly, lz;
      local_xyz(ck[i], root, 1, &lx, &ly, &lz);
      valid |= 1u << (lx | (ly << 1) | (lz << 2));
      words[m * 9 + 1 + (i - s0)] = last ? leafptr[i] : cr[i].x;
    }
    words[m * 9] = valid | ((last ? valid : 0u) << 8);
    len[m] = (uint8_t)(1 + (s1 - s0));
    svid[m] = whole ? 0ull : (depth == 0 ? node_key[m] : (node_key[m] >> (3 * depth)));
  }
}

__global__ void k_ptr_refs(const uint32_t* ptr, uint64_t M, uint4* nr) {
  GRID_STRIDE(m, M) { nr[m] = make_uint4(ptr[m], 0, 0, 0); }
}

}  // namespace

// ---------------------------------------------------------------- driver
vf_status build_format(const vf_volume* vol, const Format& f, uint32_t flags, cudaStream_t s, Handle* h) {
  auto t_start = std::chrono::steady_clock::now();
  struct Scope {  // the allocator of this build, for every vector and algorithm below
    Scope(const DevAllocator* a, cudaStream_t s) { tl_alloc = a, tl_stream = s; }
    ~Scope() { tl_alloc = nullptr, tl_stream = nullptr; }
  } scope(&h->alloc, s);
  auto pol = policy(s);
  const bool whole = (flags & VF_BUILD_WHOLE_LEVEL_DEDUP) != 0;
  const bool align = (flags & VF_BUILD_ALIGN_NODES) != 0;
  const uint32_t Rx = f.dims[0], Ry = f.dims[1], Rz = f.dims[2];

  try {
    // ---- step 0: non-empty voxels as (Morton key, rgba), sorted by key
    dvec<uint64_t> ck;
    dvec<uint32_t> vals;
    uint64_t n = 0;
    if (vol->kind == VF_VOL_DENSE_DEVICE) {
      const uint64_t total = (uint64_t)Rx * Ry * Rz;
      const uint32_t* rgba = vol->rgba;
      n = (uint64_t)thrust::count_if(pol, rgba, rgba + total, [] __device__(uint32_t v) { return v != 0u; });
      dvec<uint64_t> idx(n);
      if (n)
        thrust::copy_if(pol, thrust::counting_iterator<uint64_t>(0), thrust::counting_iterator<uint64_t>(total),
                        idx.begin(), [rgba] __device__(uint64_t i) { return rgba[i] != 0u; });
      ck.resize(n);
      vals.resize(n);
      if (n)
        k_dense_keys<<<grid_for(n), kThreads, 0, s>>>(rgba, raw(idx), n, Rx, Ry, raw(ck), raw(vals));
    } else {
      n = vol->n_voxels;
      ck.resize(n);
      vals.resize(n);
      dvec<unsigned long long> bad(1, 0ull);
      if (n)
        k_sparse_keys<<<grid_for(n), kThreads, 0, s>>>(vol->keys, vol->values, n, Rx, Ry, Rz, raw(ck), raw(vals),
                                                      raw(bad));
      VF_CUDA_TRY(cudaStreamSynchronize(s));  // order the host read after the kernels on s
      if ((unsigned long long)bad[0]) {
        set_error("vf_build: %llu sparse voxels are out of range or have value 0", (unsigned long long)bad[0]);
        return VF_ERR_INVALID_ARG;
      }
    }
    if (n) thrust::sort_by_key(pol, ck.begin(), ck.end(), vals.begin());
    if (vol->kind == VF_VOL_SPARSE_DEVICE && n) {
      dvec<unsigned long long> bad(1, 0ull);
      k_dup_check<<<grid_for(n), kThreads, 0, s>>>(raw(ck), n, raw(bad));
      VF_CUDA_TRY(cudaStreamSynchronize(s));
      if ((unsigned long long)bad[0]) {
        set_error("vf_build: %llu duplicate voxel keys in sparse input", (unsigned long long)bad[0]);
        return VF_ERR_INVALID_ARG;
      }
    }
    h->stats.nonempty_voxels = n;

    // ---- tiers, finest first
    dvec<uint4> cr(n);
    if (n) k_vals_to_refs<<<grid_for(n), kThreads, 0, s>>>(raw(vals), n, raw(cr));
    vals.clear();
    vals.shrink_to_fit();

    std::vector<dvec<uint32_t>> tier_words(f.n_tiers);
    std::vector<uint64_t> tier_base(f.n_tiers, 0);
    uint64_t cursor = 1;  // word 0 = root pointer
    uint64_t paper_words = 1;
    uint32_t root = 0;

    // Stored offsets are u32 word addresses (16 GiB limit; reading A15): every node is
    // referenced by one (the root by word 0), and the trace kernels address cells of multi-tier
    // buffers in 32 bits, so every tier must end at or below word 2^32. A single Raw level stores no
    // offsets (64-bit indexing). Checked before a tier's words are allocated: an oversized plan
    // fails fast.
    const bool single_raw = f.n_tiers == 1 && f.tiers[0].kind == K_RAW;
    auto offsets_fit = [&](int t, uint64_t base, uint64_t words) {
      if (single_raw) return true;
      if (base + words <= (1ull << 32)) return true;
      set_error("vf_build: tier %d needs words [%llu, %llu); stored offsets must stay below 2^32 words "
                "(16 GiB, PAPER.md:86)", t, (unsigned long long)base, (unsigned long long)(base + words));
      return false;
    };
    for (int t = (int)f.n_tiers - 1; t >= 0 && n > 0; --t) {
      const Tier& T = f.tiers[t];
      const bool is_root = t == 0;
      const uint32_t lf = T.lf[0];
      const uint32_t shift = is_root ? 64u : 3u * lf;
      // align every tier's base to 4 words (16 B) so SVO / N^3 nodes can be vector-loaded
      cursor = (cursor + 3) & ~3ull;
      const uint64_t base = cursor;
      tier_base[t] = base;

      dvec<uint32_t> flags(n), node_of(n);
      k_flags<<<grid_for(n), kThreads, 0, s>>>(raw(ck), n, shift, raw(flags));
      thrust::inclusive_scan(pol, flags.begin(), flags.end(), node_of.begin());
      thrust::transform(pol, node_of.begin(), node_of.end(), node_of.begin(),
                        [] __device__(uint32_t v) { return v - 1u; });
      VF_CUDA_TRY(cudaStreamSynchronize(s));
      const uint64_t M = (uint64_t)(uint32_t)node_of[n - 1] + 1;
      flags.clear();
      flags.shrink_to_fit();
      dvec<uint64_t> node_start(M), node_key(M);
      k_node_starts<<<grid_for(n), kThreads, 0, s>>>(raw(ck), raw(node_of), n, shift, raw(node_start), raw(node_key));
      dvec<uint4> nr(M);
      dvec<uint32_t>& arr = tier_words[t];
      uint64_t words = 0, pwords = 0, nodes = M;

      if (T.kind == K_RAW) {
        const uint64_t F = 1ull << (T.lf[0] + T.lf[1] + T.lf[2]);
        const uint32_t cw = T.df ? 2u : 1u;
        words = pwords = M * F * cw;
        if (!offsets_fit(t, base, words)) return VF_ERR_OVERFLOW;
        arr.assign(words, 0u);
        k_raw_scatter<<<grid_for(n), kThreads, 0, s>>>(raw(ck), raw(cr), raw(node_of), n, is_root, lf, T.lf[0],
                                                        T.lf[1], F, cw, raw(arr));
        if (T.df) {
          const uint64_t cells = M * F;
          k_df_init<<<grid_for(cells), kThreads, 0, s>>>(raw(arr), cells);
          for (int a = 0; a < 3; ++a) {
            const uint64_t lines = cells >> T.lf[a];
            k_df_pass<<<grid_for(lines), kThreads, 0, s>>>(raw(arr), M, T.lf[0], T.lf[1], T.lf[2], a);
          }
          k_df_cap<<<grid_for(cells), kThreads, 0, s>>>(raw(arr), cells, T.df_max);
        }
        k_raw_refs<<<grid_for(M), kThreads, 0, s>>>(M, base, F * cw, raw(nr));
      } else if (T.kind == K_SVO || T.kind == K_NTREE) {
        dvec<uint64_t> size(M), paper(M), off(M);
        k_inline_sizes<<<grid_for(M), kThreads, 0, s>>>(raw(node_start), M, n, T.kind, T.top, T.last, raw(size),
                                                         raw(paper));
        thrust::exclusive_scan(pol, size.begin(), size.end(), off.begin(), (uint64_t)0);
        VF_CUDA_TRY(cudaStreamSynchronize(s));
        words = (uint64_t)off[M - 1] + (uint64_t)size[M - 1];
        if (!offsets_fit(t, base, words)) return VF_ERR_OVERFLOW;
        pwords = thrust::reduce(pol, paper.begin(), paper.end(), (uint64_t)0);
        arr.assign(words, 0u);
        k_inline_write<<<grid_for(M), kThreads, 0, s>>>(raw(ck), raw(cr), raw(node_start), M, n, T.kind, is_root, T.top,
                                                         T.last, lf, raw(off), base, raw(arr), raw(nr));
      } else {  // K_SVDAG
        dvec<uint32_t> leafptr;
        uint64_t off = 0;
        if (T.last) {
          Records L;
          L.words.resize(n * 9);
          L.len.resize(n);
          L.svid.resize(n);
          k_leaf_records<<<grid_for(n), kThreads, 0, s>>>(raw(ck), raw(cr), n, whole, T.depth, raw(L.words),
                                                          raw(L.len), raw(L.svid));
          uint64_t nu = 0;
          off = dedup(L, n, arr, 0, base, leafptr, &nu, s);
          h->stats.dedup_leaf_nodes += nu;
        }
        Records Nn;
        Nn.words.resize(M * 9);
        Nn.len.resize(M);
        Nn.svid.resize(M);
        k_node_records<<<grid_for(M), kThreads, 0, s>>>(raw(ck), raw(cr), T.last ? raw(leafptr) : nullptr,
                                                        raw(node_start), raw(node_key), M, n, is_root, T.last, whole,
                                                        T.depth, raw(Nn.words), raw(Nn.len), raw(Nn.svid));
        dvec<uint32_t> ptr;
        uint64_t nu = 0, pw2 = 0;
        // VF_BUILD_ALIGN_NODES: internal nodes start at 16-B boundaries and are padded to 16-B
        // multiples, so a node's header and its first three child pointers are one aligned LDG.128
        // (1-word leaf nodes stay packed); the paper's layout counts the unpadded words
        const uint64_t ioff = align ? (off + 3) & ~3ull : off;
        uint64_t w2 = dedup(Nn, M, arr, ioff, base, ptr, &nu, s, align ? 4u : 1u, &pw2);
        nodes = nu;
        words = ioff + w2;
        pwords = off + pw2;
        if (!offsets_fit(t, base, words)) return VF_ERR_OVERFLOW;
        k_ptr_refs<<<grid_for(M), kThreads, 0, s>>>(raw(ptr), M, raw(nr));
      }
      if (t < VF_MAX_TIERS) {
        h->stats.nodes_per_tier[t] = nodes;
        h->stats.words_per_tier[t] = pwords;
      }
      cursor += words;
      paper_words += pwords;
      // the next tier's children are this tier's nodes
      ck.swap(node_key);
      cr.swap(nr);
      n = M;
      if (is_root) {
        VF_CUDA_TRY(cudaStreamSynchronize(s));  // cr was written by kernels on s
        root = ((uint4)cr[0]).x;
      }
    }

    // ---- assemble: word 0 = root pointer, then each tier at its base
    // 8 zero guard words after the last word: the trace kernel reads SVDAG headers as two
    // 16-B vectors that may extend up to 7 words past a node
    const uint64_t alloc_words = cursor + 8;
    uint32_t* buf = static_cast<uint32_t*>(h->alloc.get(alloc_words * sizeof(uint32_t), s));
    if (!buf) {
      set_error("vf_build: allocation of the %llu-byte format buffer failed", (unsigned long long)(alloc_words * 4));
      return VF_ERR_OOM;
    }
    h->buf = buf;  // owned by the handle from here on (freed by vf_build's error path / vf_destroy)
    h->buf_bytes = alloc_words * sizeof(uint32_t);
    VF_CUDA_TRY(cudaMemsetAsync(buf, 0, alloc_words * sizeof(uint32_t), s));
    VF_CUDA_TRY(cudaMemcpyAsync(buf, &root, sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    for (uint32_t t = 0; t < f.n_tiers; ++t)
      if (!tier_words[t].empty())
        VF_CUDA_TRY(cudaMemcpyAsync(buf + tier_base[t], raw(tier_words[t]), tier_words[t].size() * sizeof(uint32_t),
                                    cudaMemcpyDeviceToDevice, s));
    VF_CUDA_TRY(cudaStreamSynchronize(s));
    h->buf = buf;
    h->n_words = cursor;
    h->stats.bytes_used = cursor * 4;
    h->stats.paper_layout_bytes = paper_words * 4;
    h->stats.root = root;
  } catch (const std::bad_alloc& ex) {
    set_error("vf_build: device allocation failed (%s)", ex.what());
    return VF_ERR_OOM;
  } catch (const std::exception& ex) {
    set_error("vf_build: %s", ex.what());
    return VF_ERR_CUDA;
  }
  h->stats.build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
  return VF_OK;
}

}  // namespace vf
