/* include/vf.h — C ABI of the B200 hybrid-voxel-format first-hit tracer (libvf.so).
 *
 * The calls follow the paper's statement of the problem (arXiv 2410.14128, PAPER.md):
 *   - construction maps a voxel source + a hybrid format to one word-addressable buffer
 *     (§4.1 "Hybrid Format Construction"; layout PAPER.md:84-162, §3.3);
 *   - intersection maps (buffer, ray) to "whether the ray hits a single voxel", visiting
 *     sub-volumes "in order of hit time" (§4.2), here narrowed/extended
 *     to the hit voxel coordinate, its entry t and a miss flag.
 *
 * Conventions
 *   - No exception crosses this boundary. Every call returns vf_status; details of the
 *     last failure on the calling thread via vf_last_error().
 *   - Coordinates are grid units: voxel (i,j,k) occupies [i,i+1)x[j,j+1)x[k,k+1); the
 *     volume is [0,Rx)x[0,Ry)x[0,Rz). There is no world transform (reading A1).
 *   - Hit semantics are the exact "right-limit" definition of SURVEY.md §8(c) c-1: the
 *     first non-empty voxel (empty iff all 32 bits are 0) pierced by
 *     p(t) = o + t d over [tmin, tmax); plane crossings with equal exact t step together.
 *     Exactness (bit-exact x,y,z and miss flag; t within 1e-4 relative) is guaranteed for
 *     rays in the canonical domain: R <= 4096 per axis; |o_a| in {0} U [2^-16, 2^20);
 *     |d_a| in {0} U [2^-30, 2], d != 0; tmin < tmax; |tmin| and finite |tmax| in
 *     {0} U [2^-16, 2^20) (negative bounds select the ray line behind o, R5);
 *     tmax = +inf allowed. Other finite rays are traced, not rejected (the walk always
 *     terminates); a non-finite origin, direction or tmin, or a NaN tmax, is a miss.
 *   - All device pointers must be on the handle's device and 16-byte aligned.
 */
#ifndef VF_H
#define VF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VF_ABI_VERSION 2 /* 2: vf_build takes a vf_allocator */

#if defined(__GNUC__)
#define VF_API __attribute__((visibility("default")))
#else
#define VF_API
#endif

typedef enum {
  VF_OK = 0,
  VF_ERR_INVALID_ARG = 1, /* null/misaligned pointer, bad size, bad volume */
  VF_ERR_PARSE = 2,       /* signature syntax; message gives the character position */
  VF_ERR_FORMAT = 3,      /* non-cubic or non-power-of-two non-first level,
                             depth 0, resolution != volume dims, more than VF_MAX_TIERS tiers */
  VF_ERR_UNSUPPORTED = 4, /* valid format this build does not implement */
  VF_ERR_OVERFLOW = 5,    /* a stored offset would reach 2^32 words (PAPER.md:86, 16 GiB) */
  VF_ERR_OOM = 6,         /* device allocation failed */
  VF_ERR_CUDA = 7         /* CUDA runtime / launch error */
} vf_status;

/* Thread-local message for the last failing call on this thread ("" if none). Valid until
 * the next vf_* call on the same thread. */
VF_API const char* vf_last_error(void);
VF_API int vf_abi_version(void);

/* ---------------------------------------------------------------- format description
 * A hybrid format is an ordered list of levels, level 1 (highest) first (PAPER.md:63-82,
 * §3.2, Table 1). Each level is one base format:
 *   VF_RAW   R(W,H,D): 2^W x 2^H x 2^D grid of terminating integers
 *   VF_SVO   S(L)    : sparse voxel octree of depth L, 2-word nodes
 *   VF_SVDAG G(L)    : de-duplicated octree of depth L, 1..9-word nodes
 *   VF_NTREE T(n,d)  : N^3-tree, N = 2^n, depth d, 16-B nodes with a 64-bit occupancy mask
 *                      (generalisation of SVO; layout is ours)
 *   VF_DF    D(W,H,D,M): Raw grid of {TermInt, L1 distance to the nearest non-empty cell,
 *                      capped at M} pairs; traversal skips occupancy
 *                      tests within the distance.
 * Every level but the first must be cubic with power-of-two extent. */
enum { VF_RAW = 0, VF_SVO = 1, VF_SVDAG = 2, VF_NTREE = 3, VF_DF = 4 };

typedef struct {
  uint32_t kind;           /* VF_RAW, VF_SVO, VF_SVDAG, VF_NTREE, VF_DF */
  uint8_t log2_extent[3];  /* Raw / DF: W, H, D */
  uint8_t depth;           /* SVO / SVDAG: L; NTree: d */
  uint8_t log2_fanout;     /* NTree: n (N = 2^n, n in {1,2}) */
  uint8_t df_max;          /* DF: M */
  uint8_t reserved[2];
} vf_level;

#define VF_MAX_LEVELS 16
#define VF_MAX_TIERS 16 /* a tier = one node level: Raw 1, S(L)/G(L) L, T(n,d) d */

/* Parse a signature: "R(3,3,3) G(8)", Table-2 sugar "R(3^3) G(8)" / "R(3³) G(8)" (PAPER.md
 * Table 2, :303-322), "S(11)", "T(2,2) T(2,1) R(4^3)", "D(4^3, 6) G(5)". Whitespace-separated
 * levels; whitespace inside parentheses allowed.
 * out: caller array of capacity cap; *n_out = number of levels. VF_ERR_PARSE on syntax. */
VF_API vf_status vf_parse_format(const char* sig, vf_level* out, uint32_t cap, uint32_t* n_out);

/* Canonical signature text ("R(3, 3, 3) G(8)"); parse(to_string(f)) == f. */
VF_API vf_status vf_format_to_string(const vf_level* levels, uint32_t n_levels, char* buf, size_t cap);

/* Validate a level list and return its total resolution per axis (product of per-level
 * extents, "R(1, 0, 2) R(2, 2, 2)" -> 8 x 4 x 16). */
VF_API vf_status vf_format_resolution(const vf_level* levels, uint32_t n_levels, uint32_t dims[3]);

/* ---------------------------------------------------------------- volume input */
enum {
  VF_VOL_DENSE_DEVICE = 0, /* rgba: device, x-fastest (x + Rx*(y + Ry*z)), 0 = empty */
  VF_VOL_SPARSE_DEVICE = 1 /* n_voxels entries: keys (x | y<<21 | z<<42) and non-zero rgba
                              values, device arrays, any order, no duplicate keys */
};

typedef struct {
  uint32_t kind;
  uint32_t dims[3];
  const uint32_t* rgba;   /* DENSE: borrowed for the duration of vf_build */
  uint64_t n_voxels;      /* SPARSE */
  const uint64_t* keys;   /* SPARSE: borrowed */
  const uint32_t* values; /* SPARSE: borrowed */
} vf_volume;

/* ---------------------------------------------------------------- build */
typedef struct vf_handle vf_handle; /* opaque; owns the format buffer (immutable after build) and the trace-schedule cache */

/* Device memory provider ("PyTorch only for device memory and streams"; the
 * Python binding passes torch's caching allocator). Every device allocation of vf_build (the
 * format buffer and all build temporaries) and of the handle's later calls (work counters,
 * vf_trace_counters / vf_trace_host scratch) is requested through it:
 *   alloc(bytes, ctx, stream) -> device pointer (16-B aligned) on the handle's device, or NULL;
 *   free(ptr, bytes, ctx, stream) returns a block (bytes = the size requested), on the stream it
 *   was requested for, after the library has synchronised every use of it.
 * The struct is copied by vf_build; ctx and both functions must stay valid until vf_destroy.
 * NULL allocator: cudaMalloc / cudaFree. */
typedef struct {
  void* (*alloc)(size_t bytes, void* ctx, void* cuda_stream);
  void (*free)(void* ptr, size_t bytes, void* ctx, void* cuda_stream);
  void* ctx;
} vf_allocator;

enum {
  VF_BUILD_WHOLE_LEVEL_DEDUP = 1u << 0, /* one SVDAG de-dup map per level across sub-volumes
                                           (§4.3; evaluated ON).
                                           Clear it for per-sub-volume maps (ablation). */
  VF_BUILD_ALIGN_NODES = 1u << 1,      /* SVDAG internal nodes ("1 to 9 integers",
                                           :162) start at 16-B boundaries and are padded to 16-B
                                           multiples: a node's mask and its first three child
                                           pointers arrive in one aligned LDG.128 (SURVEY §8(a) a6
                                           option ii). Costs bytes (vf_stats.bytes_used vs
                                           paper_layout_bytes); 1-word leaf nodes stay packed. */
  VF_BUILD_DEFAULT = VF_BUILD_WHOLE_LEVEL_DEDUP,
  VF_BUILD_KNOWN_FLAGS = VF_BUILD_WHOLE_LEVEL_DEDUP | VF_BUILD_ALIGN_NODES /* other bits: VF_ERR_INVALID_ARG */
};

/* Build the format buffer on `device` (stream-ordered on cuda_stream, synchronous before
 * return). Buffer layout is the paper's: u32 words, word 0 = root pointer
 * (0 for an empty volume, buffer [0]); terminating integers are word offsets to the next
 * level's sub-volume or RGBA at the finest level; empty children are 0. Two alignment
 * paddings are added (reported in vf_stats.paper_layout_bytes vs bytes_used): SVO children
 * blocks start at even words (8-B node loads), N^3-tree nodes at multiples of 4 words (16-B).
 * *bytes_used = 4 x device words including word 0. Level 1's resolution must equal dims.
 * alloc: device memory provider (above); NULL = cudaMalloc.
 * Errors: VF_ERR_OVERFLOW when a tier would place a node at or beyond word 2^32 (its offset could
 * not be stored, reading A15) — checked before that tier is allocated, so an
 * oversized plan fails fast; a single Raw level stores no offsets and is exempt.
 * VF_ERR_OOM when the allocator fails. On error *out is NULL and nothing is leaked. */
VF_API vf_status vf_build(const vf_volume* vol, const vf_level* levels, uint32_t n_levels, uint32_t build_flags,
                          const vf_allocator* alloc, int device, void* cuda_stream, vf_handle** out,
                          uint64_t* bytes_used);

/* ---------------------------------------------------------------- trace (the hot path) */
typedef struct {
  float ox, oy, oz, tmin, dx, dy, dz, tmax;
} vf_ray; /* 32 B, grid units */

typedef struct {
  int32_t x, y, z;
  float t;
} vf_hit; /* 16 B; miss: x = y = z = -1, t = +inf */

enum {
  VF_TRACE_RESTART_SV = 1u << 0, /* "restarting sparse voxel intersection" (§4.3):
                                   stackless — after leaving a node of an SVO / SVDAG / N^3-tree
                                   level, re-descend from that level's sub-volume root instead
                                   of popping a per-thread stack. Results are identical. */
  VF_TRACE_INCOHERENT = 1u << 1, /* hint: the rays are incoherent (secondary / random rays). The
                                   trace then runs persistent warps that refill finished lanes
                                   with new rays (one atomic per batch), recovering the SIMT lanes
                                   a warp otherwise idles while its longest ray finishes. Results
                                   are identical; coherent primary rays are faster without it. */
  VF_TRACE_SCHEDULE = 1u << 2,   /* longest-first block schedule (list scheduling, LPT): every
                                   launch with this flag records the duration of each of its
                                   128-ray blocks, and a later such launch on the same handle
                                   with the SAME ray pointer and count (the next frame of a
                                   renderer reusing its ray buffer) starts its blocks in order of
                                   decreasing recorded duration, so the slow blocks no longer
                                   start last and the launch tail shrinks. Only the order in which
                                   blocks run changes: every ray is traced, results are identical.
                                   The first launch over an array runs in index order, and so does
                                   every launch of at most two waves of resident blocks (nothing to
                                   reorder). The handle keeps 9 B per block + 8 B per ray for up
                                   to 32 arrays (least recently used evicted; allocated through
                                   the build's vf_allocator); launches
                                   sharing an array are ordered by an event (inside stream capture
                                   the graph orders them, an array first seen during capture runs
                                   unscheduled, and an array used in a capture keeps its schedule
                                   memory until vf_destroy). Coherent-ray launches only (not with
                                   VF_TRACE_INCOHERENT, whose persistent warps balance by design). */
  VF_TRACE_REGROUP = 1u << 3,    /* with VF_TRACE_SCHEDULE: may also regroup the rays into warps.
                                   Inside every group of 256 consecutive rays (a 16x16 screen tile
                                   of a tile-ordered ray stream) the rays are ordered by their
                                   iteration counts in the previous launch over the array, longest
                                   first, so the lanes of a warp end together. This pays when the
                                   rays repeat (a static view) and costs when the camera moves or
                                   warps lose too much pixel coherence, so it is MEASURED: the
                                   library times its own launches over the array (CUDA events,
                                   queried without blocking), alternating schedule-only and
                                   regrouped launches, keeps the faster mode, and re-measures every
                                   256 launches; a launch captured into a graph keeps the faster
                                   mode measured so far (schedule-only before any measurement).
                                   Results are identical either way. */
  /* bit 30 is reserved (internal ablation: persistent warps with dynamic ray refill) */
};

/* Trace n rays (device array) into hits (device array), one thread per ray, asynchronously
 * on cuda_stream; hits are valid after the stream synchronises. Concurrent traces on one
 * handle are allowed (the format buffer is read-only; VF_TRACE_SCHEDULE's per-array state is
 * guarded by a lock and ordered across streams by events). n = 0 is a no-op. Formats of the library's compiled-in list
 * (the paper's per-format generated code: R(A^3) G(M), G(L), S(L), T(n,d),
 * S(a) G(b), D(A^3,M) over S/G, the cfg2/cfg3 headline formats, single Raw grids) run a kernel
 * with the format's tier geometry compiled in; all others the generic tier-table kernel.
 * Results are identical (environment VF_NO_SPEC=1 forces the generic kernel). */
VF_API vf_status vf_trace(const vf_handle* h, const vf_ray* rays, uint64_t n, vf_hit* hits, uint32_t trace_flags,
                   void* cuda_stream);

/* Kernel launches one vf_trace / vf_trace_ex / vf_trace_scatter call with these arguments makes
 * now (host-side query, no GPU work): 3 when VF_TRACE_SCHEDULE will reorder it (the two order
 * kernels + the trace; 4 when VF_TRACE_REGROUP currently regroups), else 1. For launch
 * accounting (bench.py). */
VF_API vf_status vf_trace_launch_count(const vf_handle* h, const vf_ray* rays, uint64_t n, uint32_t trace_flags,
                                       uint32_t* count);

/* Closest-hit payload (the paper's closest-hit shader):
 * rgba = the hit voxel's stored word (its RGBA; 0 on a miss); normal = the entry
 * face: normal[a] = -sign(d_a) for the lowest axis a whose voxel-slab entry plane is crossed
 * exactly at the hit t (edge / corner entries tie several axes), all 0 when the segment starts
 * inside the hit voxel (t = tmin) and on a miss. */
typedef struct {
  uint32_t rgba;
  int8_t normal[3];
  int8_t reserved;
} vf_payload; /* 8 B */

/* vf_trace plus an optional payload output (device array of n vf_payload, 8-B aligned; NULL
 * = none). Same kernel; the payload costs one extra load per hit ray. */
VF_API vf_status vf_trace_ex(const vf_handle* h, const vf_ray* rays, uint64_t n, vf_hit* hits, vf_payload* payload,
                             uint32_t trace_flags, void* cuda_stream);

/* Fused trace + hit gather (north_star multi-GPU): the hit of ray i is stored at
 * hits[slots[i]] instead of hits[i]. `slots` is a device array of n u32 on h's device; `hits` is
 * 16-B aligned and may be ANOTHER GPU's frame buffer mapped into this process by vf_ipc_open (or a
 * peer pointer with peer access enabled): each rank then writes its screen tiles' hits straight
 * into rank 0's image over NVLink / NVSwitch from the trace kernel itself, so the gather overlaps
 * the trace ray by ray and no NCCL gather or host-side un-permutation is needed. The writes are
 * complete when the stream synchronises (a kernel's stores are performed at its completion);
 * the consumer learns that from the caller's own signal (e.g. a barrier). Slots must be distinct
 * within the frame. Same kernels and results as vf_trace. */
VF_API vf_status vf_trace_scatter(const vf_handle* h, const vf_ray* rays, uint64_t n, vf_hit* hits,
                                  const uint32_t* slots, uint32_t trace_flags, void* cuda_stream);

/* CUDA IPC for vf_trace_scatter's destination: vf_ipc_export describes a device allocation of this
 * process (any pointer inside it; the offset is recorded), vf_ipc_open maps another process's
 * export on `device` (peer access enabled on demand) and returns the pointer the exporter named;
 * vf_ipc_close unmaps it. A process cannot open its own export (use the pointer itself). */
typedef struct {
  uint8_t handle[64]; /* cudaIpcMemHandle_t of the allocation */
  uint64_t offset;    /* byte offset of the exported pointer inside that allocation */
} vf_ipc_handle;
VF_API vf_status vf_ipc_export(const void* dev_ptr, vf_ipc_handle* out);
VF_API vf_status vf_ipc_open(const vf_ipc_handle* in, int device, void** dev_ptr);
VF_API vf_status vf_ipc_close(void* dev_ptr);

/* End-to-end variant with HOST buffers: copies rays host->device, traces, copies hits
 * device->host and returns when the hits are on the host. Large frames are cut into chunks
 * pipelined over the handle's internal streams (copy-in of chunk i+1, trace of chunk i and
 * copy-out of chunk i-1 overlap); the work is ordered after prior work on cuda_stream.
 * Staging device memory is owned by the handle (grown on demand); concurrent calls on one handle
 * are serialised by a per-handle lock. Host buffers should be pinned (cudaHostAlloc / torch
 * pin_memory) for overlap. */
VF_API vf_status vf_trace_host(vf_handle* h, const vf_ray* host_rays, uint64_t n, vf_hit* host_hits, uint32_t trace_flags,
                        void* cuda_stream);

/* ---------------------------------------------------------------- measurement aid
 * Work counters of the counting variant of the SAME trace kernel ("Counts come
 * from a -DVF_COUNTERS build of the same kernel"): totals over all rays of one launch.
 * VF_CTR_FORMAT_BYTES is the algorithmic format traffic: every format word the traversal reads,
 * counted once per read at its load width (Raw cell 4 B, SVO node 8 B, SVDAG mask 4 B + child
 * pointer 4 B, N^3 node 16 B, leaf terminating integer 4 B); ray I/O (48 B/ray) is not included.
 * VF_CTR_EXACT_CALLS counts exact fp64 fallbacks of the certified comparator. The counting run
 * also keeps a touch bitmap (one bit per format word, n_words / 8 bytes of device memory for the
 * call) for the distinct words / sectors the frame reads. */
enum {
  VF_CTR_RAYS = 0,
  VF_CTR_HITS,
  VF_CTR_CELL_TESTS,    /* cells tested at any tier */
  VF_CTR_STEPS,         /* DDA steps at any tier */
  VF_CTR_DESCENTS,      /* child descents (ordered_hit_children -> next_intersect) */
  VF_CTR_POPS,          /* node exits (stack pops or restarts) */
  VF_CTR_REDESCENTS,    /* restart variant: levels re-descended from the sub-volume root */
  VF_CTR_LOCATES,       /* certified sub-cell locates (entry + descents at stale events) */
  VF_CTR_NEAR_TIES,     /* DDA steps whose argmin needed the pairwise exact path */
  VF_CTR_RAW_CELLS,     /* Raw cells read (4 B; DF cells 8 B) */
  VF_CTR_SVO_NODES,     /* SVO node headers read (8 B) */
  VF_CTR_SVDAG_NODES,   /* SVDAG masks read (4 B) */
  VF_CTR_SVDAG_PTRS,    /* SVDAG child pointers read (4 B) */
  VF_CTR_NTREE_NODES,   /* N^3 node headers read (16 B) */
  VF_CTR_LEAF_WORDS,    /* leaf terminating integers read (4 B) */
  VF_CTR_FORMAT_BYTES,  /* sum of the above in bytes */
  VF_CTR_EXACT_CALLS,   /* exact fallbacks (device-global counter) */
  VF_CTR_WARP_MAX_TESTS, /* sum over warps of 32 x (max cell tests of a lane): SIMT bound */
  VF_CTR_DF_SKIPS,      /* DF cells passed without a memory access (distance budget) */
  VF_CTR_SECTOR_READS,  /* 32-B sectors spanned by the format loads, summed over loads (x 32 B: the
                           sector-bytes figure of SURVEY.md §8(d); re-reads counted again) */
  VF_CTR_UNIQUE_WORDS,  /* distinct format words read by the launch (touch bitmap): x 4 B = the
                           compulsory format bytes of the frame */
  VF_CTR_UNIQUE_SECTORS, /* distinct 32-B sectors of the format read by the launch */
  VF_NCOUNTERS
};

/* Same as vf_trace but runs the counting variant and returns the totals (synchronous). */
VF_API vf_status vf_trace_counters(const vf_handle* h, const vf_ray* rays, uint64_t n, vf_hit* hits,
                                   uint32_t trace_flags, void* cuda_stream, uint64_t counters[VF_NCOUNTERS]);

/* ---------------------------------------------------------------- test aids */
/* Point query (S:400-406 analogue): rgba_out[i] = stored voxel at xyz[3i..3i+2] (device
 * uint32 triples), 0 if empty or out of range; descends the format like intersection. */
VF_API vf_status vf_query(const vf_handle* h, const uint32_t* xyz, uint64_t n, uint32_t* rgba_out, void* cuda_stream);

typedef struct {
  uint64_t bytes_used;         /* device buffer bytes (4 x words incl. word 0) */
  uint64_t paper_layout_bytes; /* same without alignment padding (the paper's layout) */
  uint64_t nonempty_voxels;
  uint32_t dims[3];
  uint32_t n_levels;
  uint32_t n_tiers;
  uint32_t root;                 /* word 0 */
  uint64_t nodes_per_tier[VF_MAX_TIERS]; /* stored nodes per tier (unique nodes for SVDAG) */
  uint64_t words_per_tier[VF_MAX_TIERS]; /* paper-layout words written by each tier */
  uint64_t dedup_leaf_nodes;   /* SVDAG 1-word leaf nodes stored (all SVDAG levels) */
  double build_ms;             /* wall time of vf_build */
  uint32_t compiled_in;        /* 1: vf_trace runs a kernel with this format compiled in (the
                                  paper's per-format generated code, §4, as a template instance);
                                  0: the generic tier-table kernel */
  uint32_t reserved_;
} vf_stats;

VF_API vf_status vf_stats_get(const vf_handle* h, vf_stats* out);

/* Device pointer to the format buffer and its word count (read-only; for tests and tools). */
VF_API vf_status vf_buffer(const vf_handle* h, const uint32_t** words, uint64_t* n_words);

/* Copy words [first, first + count) of the format buffer to host memory (synchronous). */
VF_API vf_status vf_buffer_read(const vf_handle* h, uint64_t first, uint64_t count, uint32_t* host_out);

VF_API void vf_destroy(vf_handle* h);

#ifdef __cplusplus
}
#endif
#endif /* VF_H */
