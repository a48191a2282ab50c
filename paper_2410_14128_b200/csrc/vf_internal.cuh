// vf_internal.cuh — shared internals of libvf.so (format tiers, handle, errors).
//
// A hybrid format (§3.2) is expanded into TIERS, one per node level:
//   Raw R(w,h,d)        -> 1 tier, fan-out 2^w x 2^h x 2^d
//   SVO S(L) / SVDAG G(L) -> L tiers, fan-out 2 x 2 x 2
//   N^3-tree T(n,d)      -> d tiers, fan-out 2^n per axis     (layout SURVEY A13)
// Tier 0 is the root. lc(t) = log2 of a tier-t cell's edge in voxels (cubic for every tier,
// since every level but the first is cubic). A tier's "cells" are the
// children of its nodes; the cells of a level's last tier are that level's sub-volumes
// (terminating integers), and the cells of the last tier overall are voxels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>
#include <string>

#include "../../include/vf.h"

namespace vf {

enum TierKind : uint32_t { K_RAW = 0, K_SVO = 1, K_SVDAG = 2, K_NTREE = 3 };

struct Tier {
  uint32_t kind;   // TierKind
  uint32_t lf[3];  // log2 fan-out per axis (cubic except possibly tier 0)
  uint32_t lc;     // log2 cell size in voxels
  uint32_t level;  // index of the level this tier belongs to
  uint32_t depth;  // depth within its level (0 = level top)
  bool top;        // first tier of its level (its node is the level's sub-volume root)
  bool last;       // last tier of its level (its cells are terminating integers)
  bool df;         // K_RAW tier of a DF level D(W,H,D,M): cells are {TermInt, L1 distance} pairs
  uint32_t df_max; // DF: maximum stored L1 distance M
};

struct Format {
  uint32_t n_levels = 0;
  vf_level levels[VF_MAX_LEVELS];
  uint32_t n_tiers = 0;
  Tier tiers[VF_MAX_TIERS];
  uint32_t dims[3] = {0, 0, 0};
};

// Packed per-tier parameters passed to the trace / query kernels by value (all uniform).
// Fields for tier t are extracted with shifts, so a lane at any tier reads them from
// registers / the constant bank without indexed memory.
struct TraceParams {
  uint64_t lc_pack;     // 4 bits per tier: lc(t)
  uint64_t lf_pack;     // 4 bits per tier: cubic log2 fan-out (tier 0: x)
  uint64_t tau_pack;    // 4 bits per h in [0,15]: deepest tier whose node contains both cells
                        // whose coordinates first differ at bit h
  uint32_t kind_pack;   // 2 bits per tier
  uint32_t top_mask;    // bit t: tier t is its level's top
  uint32_t last_mask;   // bit t: tier t is its level's last tier
  uint32_t refill;      // persistent trace: refill a warp when >= refill lanes are idle
  uint32_t chunk;       // chunked trace: rays per claimed chunk (multiple of 32)
  uint32_t crefill;     // chunked trace: refill from the warp's chunk when >= crefill lanes are idle
  uint32_t df_mask;     // bit t: tier t is a DF grid (2-word cells {TermInt, L1 distance})
  uint2* payload;       // optional closest-hit payload output (vf_trace_ex), per launch
  const uint32_t* slot; // optional hit destination index per ray (vf_trace_scatter), per launch
  uint32_t* touch;      // counting launches: touch bitmap, one bit per format word (else null)
  const uint32_t* order;  // VF_TRACE_SCHEDULE: block b traces ray block order[b] (else b), per launch
  uint32_t* cost;         // VF_TRACE_SCHEDULE: each block stores its duration (SM cycles) at cost[its ray block]
  const uint32_t* ray_perm;  // VF_TRACE_SCHEDULE: slot v of the launch traces ray ray_perm[v] (else v)
  uint32_t* ray_cost;        // VF_TRACE_SCHEDULE: each ray stores when its lane finished (SM cycles
                             // after its block's start) at ray_cost[ray]
  uint32_t lf0[3];      // tier-0 fan-out per axis (log2)
  int32_t dims[3];      // resolution per axis
  uint32_t n_tiers;
  uint32_t root;        // word 0 (root pointer); 0 => empty volume
  uint32_t level_top_pack_lo;  // 4 bits per tier: tier index of its level's top (tiers 0..7)
  uint32_t level_top_pack_hi;  // tiers 8..15
  // One packed word per tier, staged in shared memory by the trace kernels and read once per tier
  // change (TW_* below): everything the traversal needs about the current tier.
  uint32_t tword[VF_MAX_TIERS];
};

// Tier-word fields (TraceParams::tword).
enum : uint32_t {
  TW_KIND = 0,      // 2 bits: TierKind
  TW_LC = 2,        // 4 bits: lc(t), log2 cell edge in voxels
  TW_LCN = 6,       // 4 bits: lc(t+1) (0 at the finest tier)
  TW_LCP = 10,      // 4 bits: lc(t-1), the edge of tier t's node; 15 at tier 0 (never left)
  TW_SX = 14,       // 4 bits: shift of the y cell index in the linear cell index
  TW_SXY = 18,      // 5 bits: shift of the z cell index
  TW_MB = 23,       // 4 bits: width of a per-axis cell index (lf; 12 at tier 0)
  TW_LAST = 1u << 27,    // last tier of its level: cells are terminating integers
  TW_FINEST = 1u << 28,  // last tier overall: cells are voxels
  TW_DF = 1u << 29,      // DF grid: 2-word cells {TermInt, L1 distance}
  TW_TOP = 1u << 30,     // first tier of its level
};

// Device memory of a handle and of its build (SURVEY.md §8(b) vf_allocator: "PyTorch only for
// memory and streams"). a.alloc == NULL: cudaMalloc / cudaFree. Blocks are requested for, and
// returned on, the stream of the call that uses them.
struct DevAllocator {
  vf_allocator a{};
  void* get(size_t bytes, cudaStream_t s) const {
    if (bytes == 0) bytes = 16;
    if (a.alloc) return a.alloc(bytes, a.ctx, (void*)s);
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    return p;
  }
  void put(void* p, size_t bytes, cudaStream_t s) const {
    if (!p) return;
    if (bytes == 0) bytes = 16;
    if (a.alloc) {
      if (a.free) a.free(p, bytes, a.ctx, (void*)s);
    } else {
      cudaFree(p);
    }
  }
};

// VF_TRACE_SCHEDULE state for one ray array (key: device pointer + count): the per-block durations
// of the last launch over it and the longest-first block order derived from them.
struct SchedEntry {
  const void* rays = nullptr;
  uint64_t n = 0;
  uint32_t nb = 0;            // blocks of the launch
  uint32_t* mem = nullptr;    // cost[nb] | order[nb] | hist[kSchedBuckets] | cursor[kSchedBuckets] | done
                              // | ray_cost[n] | ray_perm[n]
  size_t bytes = 0;
  cudaEvent_t ev = nullptr;   // recorded after the last launch that wrote cost (cross-stream order)
  bool valid = false;         // cost holds a completed launch's durations
  bool pinned = false;        // used inside a stream capture: a graph may replay it, never evicted
  // VF_TRACE_REGROUP is measured, not assumed: the library times its own launches over this array
  // (events around the order kernels + trace), alternating "block schedule only" (mode 0) and
  // "+ ray regrouping" (mode 1), and then keeps the faster mode (re-measured every kReeval launches)
  cudaEvent_t t0[4] = {}, t1[4] = {};
  int8_t tmode[4] = {-1, -1, -1, -1};  // mode timed by event pair i (-1: none pending)
  int tnext = 0;                       // next event pair
  int pending = -1;                    // event pair of the launch being issued (t1 recorded after it)
  double ms_sum[2] = {0.0, 0.0};
  int ms_n[2] = {0, 0};
  int decided = -1;      // faster mode, or -1 while measuring
  uint32_t since = 0;    // launches since the decision / measuring launches
  int last_mode = 0;     // mode of the last launch (vf_trace_launch_count)
  uint64_t last_use = 0;
};
constexpr int kSchedEntries = 32;
constexpr uint32_t kSchedBuckets = 128;  // quarter-octave duration classes, longest first
constexpr uint32_t kRayGroup = 256;      // rays regrouped into warps inside consecutive groups of 256

struct Handle {
  int device = 0;
  DevAllocator alloc;
  cudaStream_t build_stream = nullptr;  // the buffer's allocation stream (returned there by vf_destroy)
  Format fmt;
  TraceParams tp;
  uint32_t* buf = nullptr;  // device words
  uint64_t n_words = 0;
  size_t buf_bytes = 0;     // allocated bytes of buf (n_words + guard words)
  bool aligned_nodes = false;  // built with VF_BUILD_ALIGN_NODES (16-B aligned SVDAG nodes)
  vf_stats stats{};
  // staging and pipeline streams for vf_trace_host
  void* stage = nullptr;
  size_t stage_bytes = 0;
  cudaStream_t pipe[4] = {nullptr, nullptr, nullptr, nullptr};  // copy-in, copy-out, 2 x trace
  cudaEvent_t pipe_ev = nullptr;
  cudaEvent_t chunk_ev[2 * 64] = {};  // per chunk: rays copied in, traced (2 * kMaxHostChunks)
  // persistent-trace work counters: kWorkSlots x {next ray, finished blocks}, self-resetting
  unsigned long long* work = nullptr;
  mutable std::atomic<uint32_t> work_slot{0};
  std::mutex host_mu;  // vf_trace_host: serialises calls on one handle (shared staging and streams)
  // VF_TRACE_SCHEDULE: LRU table of per-ray-array block schedules (guarded by sched_mu)
  mutable std::mutex sched_mu;
  mutable SchedEntry sched[kSchedEntries];
  mutable uint64_t sched_clock = 0;
};

constexpr uint32_t kWorkSlots = 64;
constexpr int kPipe = 4;
constexpr int kMaxHostChunks = 64;
// internal trace flag (ablation / tests): persistent warps with dynamic ray refill
constexpr uint32_t VF_TRACE_PERSISTENT_WARPS = 1u << 30;
// internal trace flags (A/B): persistent warps over claimed screen-coherent chunks (in-warp refill
// from the chunk), optionally with the top Raw grid staged in shared memory
constexpr uint32_t VF_TRACE_CHUNKED = 1u << 29;
constexpr uint32_t VF_TRACE_STAGE_TOP = 1u << 28;
void free_schedules(const Handle* h);
uint32_t trace_launch_count(const Handle* h, const vf_ray* rays, uint64_t n, uint32_t flags);

// errors
void set_error(const char* fmt, ...);
void clear_error();

// format.cu
vf_status expand_format(const vf_level* levels, uint32_t n, Format* out);
TraceParams make_trace_params(const Format& f, uint32_t root);

// build.cu
vf_status build_format(const vf_volume* vol, const Format& f, uint32_t flags, cudaStream_t s, Handle* h);

// trace.cu
vf_status launch_trace(const Handle* h, const vf_ray* rays, uint64_t n, vf_hit* hits, uint32_t flags,
                       cudaStream_t s, unsigned long long* counters = nullptr, vf_payload* payload = nullptr,
                       uint32_t* touch = nullptr, const uint32_t* slots = nullptr);
vf_status launch_touch_count(const uint32_t* touch, uint64_t n_bitmap_words, unsigned long long* counters,
                             cudaStream_t s);
vf_status read_exact_calls(unsigned long long* out, bool reset);
bool has_compiled_in_kernel(const Format& f);
vf_status launch_query(const Handle* h, const uint32_t* xyz, uint64_t n, uint32_t* out, cudaStream_t s);

#define VF_CUDA_TRY(expr)                                                                   \
  do {                                                                                      \
    cudaError_t _e = (expr);                                                                \
    if (_e != cudaSuccess) {                                                                \
      ::vf::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, __LINE__); \
      return _e == cudaErrorMemoryAllocation ? VF_ERR_OOM : VF_ERR_CUDA;                    \
    }                                                                                       \
  } while (0)

}  // namespace vf
