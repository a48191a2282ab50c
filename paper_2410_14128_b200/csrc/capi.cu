// capi.cu — the extern "C" boundary of libvf.so (include/vf.h). No exception crosses it.
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <new>

#include <cuda.h>

#include "vf_internal.cuh"

using namespace vf;

struct vf_handle : vf::Handle {};

namespace {

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

// Base address of the device allocation containing p (driver cuMemGetAddressRange, fetched through
// the runtime so that libvf.so does not link libcuda: it must load on machines without a driver).
bool allocation_base(const void* p, CUdeviceptr* base) {
  using Fn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static Fn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return (Fn)f;
  }();
  size_t size = 0;
  return fn && fn(base, &size, (CUdeviceptr)p) == CUDA_SUCCESS;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace

extern "C" {

vf_status vf_build(const vf_volume* vol, const vf_level* levels, uint32_t n_levels, uint32_t build_flags,
                   const vf_allocator* alloc, int device, void* cuda_stream, vf_handle** out, uint64_t* bytes_used) {
  clear_error();
  if (out) *out = nullptr;
  if (!vol || !levels || !out) {
    set_error("vf_build: null argument");
    return VF_ERR_INVALID_ARG;
  }
  if (vol->kind != VF_VOL_DENSE_DEVICE && vol->kind != VF_VOL_SPARSE_DEVICE) {
    set_error("vf_build: unknown volume kind %u", vol->kind);
    return VF_ERR_INVALID_ARG;
  }
  if (vol->kind == VF_VOL_DENSE_DEVICE && !vol->rgba) {
    set_error("vf_build: dense volume without rgba pointer");
    return VF_ERR_INVALID_ARG;
  }
  if (vol->kind == VF_VOL_SPARSE_DEVICE && vol->n_voxels && (!vol->keys || !vol->values)) {
    set_error("vf_build: sparse volume without keys/values");
    return VF_ERR_INVALID_ARG;
  }
  if (alloc && (!alloc->alloc || !alloc->free)) {
    set_error("vf_build: allocator needs both alloc and free");
    return VF_ERR_INVALID_ARG;
  }
  if (build_flags & ~(uint32_t)VF_BUILD_KNOWN_FLAGS) {
    set_error("vf_build: unknown build flags 0x%x", build_flags & ~(uint32_t)VF_BUILD_KNOWN_FLAGS);
    return VF_ERR_INVALID_ARG;
  }
  Format f;
  vf_status st = expand_format(levels, n_levels, &f);
  if (st != VF_OK) return st;
  for (int a = 0; a < 3; ++a)
    if (f.dims[a] != vol->dims[a]) {
      set_error("vf_build: format resolution %ux%ux%u != volume dims %ux%ux%u", f.dims[0], f.dims[1], f.dims[2],
                vol->dims[0], vol->dims[1], vol->dims[2]);
      return VF_ERR_FORMAT;
    }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    set_error("vf_build: CUDA device %d not available (%d devices)", device, ndev);
    return VF_ERR_CUDA;
  }
  DeviceGuard g(device);
  vf_handle* h = new (std::nothrow) vf_handle();
  if (!h) {
    set_error("vf_build: host allocation failed");
    return VF_ERR_OOM;
  }
  h->device = device;
  if (alloc) h->alloc.a = *alloc;
  h->build_stream = (cudaStream_t)cuda_stream;
  h->aligned_nodes = (build_flags & VF_BUILD_ALIGN_NODES) != 0;
  h->fmt = f;
  memset(&h->stats, 0, sizeof(h->stats));
  st = build_format(vol, f, build_flags, (cudaStream_t)cuda_stream, h);
  if (st != VF_OK) {
    if (h->buf) {
      cudaStreamSynchronize(h->build_stream);
      h->alloc.put(h->buf, h->buf_bytes, h->build_stream);
    }
    delete h;
    return st;
  }
  h->tp = make_trace_params(f, h->stats.root);
  {
    const size_t wb = sizeof(unsigned long long) * 2 * kWorkSlots;
    h->work = static_cast<unsigned long long*>(h->alloc.get(wb, h->build_stream));
    cudaError_t e = h->work ? cudaMemsetAsync(h->work, 0, wb, h->build_stream) : cudaErrorMemoryAllocation;
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->build_stream);
    if (e != cudaSuccess) {
      set_error("vf_build: work-counter allocation failed: %s", cudaGetErrorString(e));
      h->alloc.put(h->work, wb, h->build_stream);
      h->alloc.put(h->buf, h->buf_bytes, h->build_stream);
      delete h;
      return VF_ERR_OOM;
    }
  }
  for (int a = 0; a < 3; ++a) h->stats.dims[a] = f.dims[a];
  h->stats.n_levels = f.n_levels;
  h->stats.compiled_in = has_compiled_in_kernel(f) ? 1u : 0u;
  h->stats.n_tiers = f.n_tiers;
  if (bytes_used) *bytes_used = h->stats.bytes_used;
  *out = h;
  return VF_OK;
}

vf_status vf_trace(const vf_handle* h, const vf_ray* rays, uint64_t n, vf_hit* hits, uint32_t trace_flags,
                   void* cuda_stream) {
  clear_error();
  if (!h) {
    set_error("vf_trace: null handle");
    return VF_ERR_INVALID_ARG;
  }
  if (n == 0) return VF_OK;
  if (!rays || !hits || !aligned16(rays) || !aligned16(hits)) {
    set_error("vf_trace: rays/hits must be non-null 16-byte aligned device pointers");
    return VF_ERR_INVALID_ARG;
  }
  DeviceGuard g(h->device);
  return launch_trace(h, rays, n, hits, trace_flags, (cudaStream_t)cuda_stream);
}

vf_status vf_trace_launch_count(const vf_handle* h, const vf_ray* rays, uint64_t n, uint32_t trace_flags,
                                uint32_t* count) {
  clear_error();
  if (!h || !count) {
    set_error("vf_trace_launch_count: null argument");
    return VF_ERR_INVALID_ARG;
  }
  *count = trace_launch_count(h, rays, n, trace_flags);
  return VF_OK;
}

vf_status vf_trace_ex(const vf_handle* h, const vf_ray* rays, uint64_t n, vf_hit* hits, vf_payload* payload,
                      uint32_t trace_flags, void* cuda_stream) {
  clear_error();
  if (!h) {
    set_error("vf_trace_ex: null handle");
    return VF_ERR_INVALID_ARG;
  }
  if (n == 0) return VF_OK;
  if (!rays || !hits || !aligned16(rays) || !aligned16(hits) || ((uintptr_t)payload & 7u)) {
    set_error("vf_trace_ex: rays/hits must be 16-byte aligned device pointers, payload 8-byte aligned");
    return VF_ERR_INVALID_ARG;
  }
  DeviceGuard g(h->device);
  return launch_trace(h, rays, n, hits, trace_flags, (cudaStream_t)cuda_stream, nullptr, payload);
}

vf_status vf_trace_scatter(const vf_handle* h, const vf_ray* rays, uint64_t n, vf_hit* hits, const uint32_t* slots,
                           uint32_t trace_flags, void* cuda_stream) {
  clear_error();
  if (!h) {
    set_error("vf_trace_scatter: null handle");
    return VF_ERR_INVALID_ARG;
  }
  if (n == 0) return VF_OK;
  if (!rays || !hits || !slots || !aligned16(rays) || !aligned16(hits) || ((uintptr_t)slots & 3u)) {
    set_error("vf_trace_scatter: rays/hits must be 16-byte aligned device pointers, slots a 4-byte aligned device array");
    return VF_ERR_INVALID_ARG;
  }
  DeviceGuard g(h->device);
  return launch_trace(h, rays, n, hits, trace_flags, (cudaStream_t)cuda_stream, nullptr, nullptr, nullptr, slots);
}

vf_status vf_ipc_export(const void* dev_ptr, vf_ipc_handle* out) {
  clear_error();
  if (!dev_ptr || !out) {
    set_error("vf_ipc_export: null argument");
    return VF_ERR_INVALID_ARG;
  }
  memset(out, 0, sizeof(*out));
  CUdeviceptr base = 0;
  if (!allocation_base(dev_ptr, &base)) {
    set_error("vf_ipc_export: %p is not a device allocation", dev_ptr);
    return VF_ERR_INVALID_ARG;
  }
  cudaIpcMemHandle_t hd;
  VF_CUDA_TRY(cudaIpcGetMemHandle(&hd, (void*)base));
  static_assert(sizeof(hd) <= sizeof(out->handle), "cudaIpcMemHandle_t size");
  memcpy(out->handle, &hd, sizeof(hd));
  out->offset = (uint64_t)((CUdeviceptr)dev_ptr - base);
  return VF_OK;
}

vf_status vf_ipc_open(const vf_ipc_handle* in, int device, void** dev_ptr) {
  clear_error();
  if (!in || !dev_ptr) {
    set_error("vf_ipc_open: null argument");
    return VF_ERR_INVALID_ARG;
  }
  *dev_ptr = nullptr;
  DeviceGuard g(device);
  cudaIpcMemHandle_t hd;
  memcpy(&hd, in->handle, sizeof(hd));
  void* base = nullptr;
  VF_CUDA_TRY(cudaIpcOpenMemHandle(&base, hd, cudaIpcMemLazyEnablePeerAccess));
  *dev_ptr = (char*)base + in->offset;
  return VF_OK;
}

vf_status vf_ipc_close(void* dev_ptr) {
  clear_error();
  if (!dev_ptr) return VF_OK;
  CUdeviceptr base = 0;
  if (!allocation_base(dev_ptr, &base)) {
    set_error("vf_ipc_close: %p is not a mapped device pointer", dev_ptr);
    return VF_ERR_INVALID_ARG;
  }
  VF_CUDA_TRY(cudaIpcCloseMemHandle((void*)base));
  return VF_OK;
}

vf_status vf_trace_counters(const vf_handle* h, const vf_ray* rays, uint64_t n, vf_hit* hits, uint32_t trace_flags,
                            void* cuda_stream, uint64_t counters[VF_NCOUNTERS]) {
  clear_error();
  if (!h || !counters) {
    set_error("vf_trace_counters: null argument");
    return VF_ERR_INVALID_ARG;
  }
  for (int i = 0; i < VF_NCOUNTERS; ++i) counters[i] = 0;
  if (n == 0) return VF_OK;
  if (!rays || !hits || !aligned16(rays) || !aligned16(hits)) {
    set_error("vf_trace_counters: rays/hits must be non-null 16-byte aligned device pointers");
    return VF_ERR_INVALID_ARG;
  }
  DeviceGuard g(h->device);
  cudaStream_t s = (cudaStream_t)cuda_stream;
  const size_t db = sizeof(unsigned long long) * VF_NCOUNTERS;
  unsigned long long* d = static_cast<unsigned long long*>(h->alloc.get(db, s));
  if (!d) {
    set_error("vf_trace_counters: counter allocation failed");
    return VF_ERR_OOM;
  }
  // touch bitmap: one bit per format word (distinct words / sectors read by the frame)
  const uint64_t nbw = (h->n_words + 31) / 32;
  // (too large to keep: the distinct-word counters stay 0)
  uint32_t* touch = static_cast<uint32_t*>(h->alloc.get(nbw * sizeof(uint32_t), s));
  unsigned long long ex = 0;
  vf_status st = read_exact_calls(&ex, true);
  if (st == VF_OK) {
    cudaMemsetAsync(d, 0, sizeof(unsigned long long) * VF_NCOUNTERS, s);
    if (touch) cudaMemsetAsync(touch, 0, nbw * sizeof(uint32_t), s);
    st = launch_trace(h, rays, n, hits, trace_flags, s, d, nullptr, touch);
    if (st == VF_OK && touch) st = launch_touch_count(touch, nbw, d, s);
  }
  if (st == VF_OK) {
    unsigned long long hc[VF_NCOUNTERS];
    cudaError_t e = cudaMemcpyAsync(hc, d, sizeof(hc), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      set_error("vf_trace_counters: %s", cudaGetErrorString(e));
      st = VF_ERR_CUDA;
    } else {
      for (int i = 0; i < VF_NCOUNTERS; ++i) counters[i] = hc[i];
      st = read_exact_calls(&ex, true);
      counters[VF_CTR_EXACT_CALLS] = ex;
    }
  }
  cudaStreamSynchronize(s);
  h->alloc.put(d, db, s);
  h->alloc.put(touch, nbw * sizeof(uint32_t), s);
  return st;
}

vf_status vf_trace_host(vf_handle* h, const vf_ray* host_rays, uint64_t n, vf_hit* host_hits, uint32_t trace_flags,
                        void* cuda_stream) {
  clear_error();
  if (!h) {
    set_error("vf_trace_host: null handle");
    return VF_ERR_INVALID_ARG;
  }
  if (n == 0) return VF_OK;
  if (!host_rays || !host_hits) {
    set_error("vf_trace_host: null buffer");
    return VF_ERR_INVALID_ARG;
  }
  DeviceGuard g(h->device);
  std::lock_guard<std::mutex> lock(h->host_mu);  // staging buffer and pipeline streams are per handle
  cudaStream_t s = (cudaStream_t)cuda_stream;
  const size_t rb = n * sizeof(vf_ray), hb = n * sizeof(vf_hit);
  const size_t need = ((rb + 255) & ~(size_t)255) + hb;
  if (h->stage_bytes < need) {
    if (h->stage) {
      cudaDeviceSynchronize();  // the previous staging buffer may still be read by an earlier call's copies
      h->alloc.put(h->stage, h->stage_bytes, h->build_stream);
    }
    h->stage = nullptr;
    h->stage_bytes = 0;
    h->stage = h->alloc.get(need, h->build_stream);
    if (!h->stage) {
      set_error("vf_trace_host: staging allocation of %zu bytes failed", need);
      return VF_ERR_OOM;
    }
    h->stage_bytes = need;
  }
  vf_ray* d_rays = (vf_ray*)h->stage;
  vf_hit* d_hits = (vf_hit*)((char*)h->stage + ((rb + 255) & ~(size_t)255));
  // Pipeline: the frame is cut into chunks; one internal stream copies rays in (copy engine 1),
  // two trace (alternating, so consecutive chunks' kernels overlap: a small launch lasts as long
  // as its slowest ray), one copies hits out (copy engine 2), linked per chunk by events — so the
  // host->device copy of chunk i+1, the trace of chunk i and the device->host copy of chunk i-1
  // overlap with no false dependency between a chunk's copy-out and a later chunk's copy-in.
  // Every chunk has its own staging region: no reuse hazard. The bound is the PCIe link (rays in:
  // 32 B/ray); the chunk count trades pipeline fill/drain against per-copy overhead.
  if (!h->pipe[0]) {
    for (int i = 0; i < kPipe; ++i) VF_CUDA_TRY(cudaStreamCreateWithFlags(&h->pipe[i], cudaStreamNonBlocking));
    VF_CUDA_TRY(cudaEventCreateWithFlags(&h->pipe_ev, cudaEventDisableTiming));
    for (int i = 0; i < 2 * kMaxHostChunks; ++i)
      VF_CUDA_TRY(cudaEventCreateWithFlags(&h->chunk_ev[i], cudaEventDisableTiming));
  }
  // On every return (error paths included) no copy of this call may still touch the caller's host
  // buffers: drain the pipeline streams (a no-op after the final synchronize below).
  struct Drain {
    vf_handle* h;
    ~Drain() {
      for (int i = 0; i < kPipe; ++i)
        if (h->pipe[i]) cudaStreamSynchronize(h->pipe[i]);
    }
  } drain{h};
  VF_CUDA_TRY(cudaEventRecord(h->pipe_ev, s));  // order after prior work on the caller's stream
  static const uint64_t chunks_env = [] {  // A/B override of the pipeline depth
    const char* e = getenv("VF_HOST_CHUNKS");
    const long v = e ? atol(e) : 0;
    return (uint64_t)(v > 0 && v <= kMaxHostChunks ? v : 0);
  }();
  uint64_t chunks = n >= (1ull << 18) ? (n >> 17 < 16 ? n >> 17 : 16) : 1;
  if (chunks_env) chunks = chunks_env < n ? chunks_env : n;
  const uint64_t per = (n + chunks - 1) / chunks;
  cudaStream_t cin = h->pipe[0], cout = h->pipe[1];
  for (int i = 0; i < kPipe; ++i) VF_CUDA_TRY(cudaStreamWaitEvent(h->pipe[i], h->pipe_ev, 0));
  for (uint64_t c = 0; c < chunks; ++c) {
    const uint64_t b = c * per, m = (b + per <= n) ? per : n - b;
    if (!m) break;
    cudaEvent_t in_done = h->chunk_ev[2 * c], tr_done = h->chunk_ev[2 * c + 1];
    cudaStream_t ctr = h->pipe[2 + (c & 1)];
    VF_CUDA_TRY(cudaMemcpyAsync(d_rays + b, host_rays + b, m * sizeof(vf_ray), cudaMemcpyHostToDevice, cin));
    VF_CUDA_TRY(cudaEventRecord(in_done, cin));
    VF_CUDA_TRY(cudaStreamWaitEvent(ctr, in_done, 0));
    vf_status st = launch_trace(h, d_rays + b, m, d_hits + b, trace_flags, ctr);
    if (st != VF_OK) return st;
    VF_CUDA_TRY(cudaEventRecord(tr_done, ctr));
    VF_CUDA_TRY(cudaStreamWaitEvent(cout, tr_done, 0));
    VF_CUDA_TRY(cudaMemcpyAsync(host_hits + b, d_hits + b, m * sizeof(vf_hit), cudaMemcpyDeviceToHost, cout));
  }
  for (int i = 0; i < kPipe; ++i) VF_CUDA_TRY(cudaStreamSynchronize(h->pipe[i]));
  return VF_OK;
}

vf_status vf_query(const vf_handle* h, const uint32_t* xyz, uint64_t n, uint32_t* rgba_out, void* cuda_stream) {
  clear_error();
  if (!h) {
    set_error("vf_query: null handle");
    return VF_ERR_INVALID_ARG;
  }
  if (n == 0) return VF_OK;
  if (!xyz || !rgba_out) {
    set_error("vf_query: null buffer");
    return VF_ERR_INVALID_ARG;
  }
  DeviceGuard g(h->device);
  return launch_query(h, xyz, n, rgba_out, (cudaStream_t)cuda_stream);
}

vf_status vf_stats_get(const vf_handle* h, vf_stats* out) {
  clear_error();
  if (!h || !out) {
    set_error("vf_stats_get: null argument");
    return VF_ERR_INVALID_ARG;
  }
  *out = h->stats;
  return VF_OK;
}

vf_status vf_buffer(const vf_handle* h, const uint32_t** words, uint64_t* n_words) {
  clear_error();
  if (!h || !words || !n_words) {
    set_error("vf_buffer: null argument");
    return VF_ERR_INVALID_ARG;
  }
  *words = h->buf;
  *n_words = h->n_words;
  return VF_OK;
}

vf_status vf_buffer_read(const vf_handle* h, uint64_t first, uint64_t count, uint32_t* host_out) {
  clear_error();
  if (!h || (!host_out && count)) {
    set_error("vf_buffer_read: null argument");
    return VF_ERR_INVALID_ARG;
  }
  if (first > h->n_words || count > h->n_words - first) {
    set_error("vf_buffer_read: range [%llu, +%llu) outside %llu words", (unsigned long long)first,
              (unsigned long long)count, (unsigned long long)h->n_words);
    return VF_ERR_INVALID_ARG;
  }
  if (!count) return VF_OK;
  DeviceGuard g(h->device);
  VF_CUDA_TRY(cudaMemcpy(host_out, h->buf + first, count * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  return VF_OK;
}

void vf_destroy(vf_handle* h) {
  if (!h) return;
  DeviceGuard g(h->device);
  cudaDeviceSynchronize();  // no kernel or copy of this handle may still use its memory
  free_schedules(h);
  h->alloc.put(h->buf, h->buf_bytes, h->build_stream);
  h->alloc.put(h->stage, h->stage_bytes, h->build_stream);
  h->alloc.put(h->work, sizeof(unsigned long long) * 2 * kWorkSlots, h->build_stream);
  for (int i = 0; i < kPipe; ++i)
    if (h->pipe[i]) cudaStreamDestroy(h->pipe[i]);
  if (h->pipe_ev) cudaEventDestroy(h->pipe_ev);
  for (int i = 0; i < 2 * kMaxHostChunks; ++i)
    if (h->chunk_ev[i]) cudaEventDestroy(h->chunk_ev[i]);
  delete h;
}

}  // extern "C"
