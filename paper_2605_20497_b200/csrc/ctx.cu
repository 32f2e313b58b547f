// ctx.cu — context lifetime, allocator plumbing, scratch arena, error reporting.
#include <cstring>

#include "common.cuh"

namespace hgp {

static thread_local std::string g_err;

hgp_status set_error(hgp_status code, const char *fmt, ...) {
  char buf[768];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

hgp_status read_back(hgp_ctx *c, const void *dptr, size_t bytes, void *host) {
  if (bytes > 64 * sizeof(uint64_t)) {
    HGP_CUDA(cudaMemcpyAsync(host, dptr, bytes, cudaMemcpyDeviceToHost, c->stream));
    HGP_CUDA(cudaStreamSynchronize(c->stream));
    return HGP_OK;
  }
  HGP_CUDA(cudaMemcpyAsync(c->h_pin, dptr, bytes, cudaMemcpyDeviceToHost, c->stream));
  HGP_CUDA(cudaStreamSynchronize(c->stream));
  memcpy(host, c->h_pin, bytes);
  return HGP_OK;
}

hgp_status clear_errors(hgp_ctx *c) {
  HGP_CUDA(cudaMemsetAsync(c->d_err, 0xFF, sizeof(uint64_t) * kErrSlots, c->stream));
  return HGP_OK;
}

hgp_status fetch_errors(hgp_ctx *c, uint64_t out[kErrSlots]) {
  return read_back(c, c->d_err, sizeof(uint64_t) * kErrSlots, out);
}

static void *pool_alloc(void *, size_t bytes, hgp_stream_t s) {
  void *p = nullptr;
  if (cudaMallocAsync(&p, bytes, reinterpret_cast<cudaStream_t>(s)) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}
static void pool_free(void *, void *p, size_t, hgp_stream_t s) {
  if (p) cudaFreeAsync(p, reinterpret_cast<cudaStream_t>(s));
}

}  // namespace hgp

using namespace hgp;

void *hgp_ctx::dalloc(size_t bytes) {
  bytes = (bytes + 255) & ~size_t(255);
  return alloc.alloc(alloc.user, bytes ? bytes : 256, reinterpret_cast<hgp_stream_t>(stream));
}

void hgp_ctx::dfree(void *p, size_t bytes) {
  if (!p) return;
  bytes = (bytes + 255) & ~size_t(255);
  alloc.free(alloc.user, p, bytes ? bytes : 256, reinterpret_cast<hgp_stream_t>(stream));
}

cudaEvent_t hgp_ctx::prof_event() {
  if (prof_pool.empty()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  cudaEvent_t e = prof_pool.back();
  prof_pool.pop_back();
  return e;
}

void hgp_ctx::reset_scratch() {
  // keep only the largest chunk (the steady-state working set of one call fits in it after the
  // first few calls); smaller ones go back to the allocator
  if (chunks.size() > 1) {
    size_t best = 0;
    for (size_t i = 1; i < chunks.size(); ++i)
      if (chunks[i].bytes > chunks[best].bytes) best = i;
    for (size_t i = 0; i < chunks.size(); ++i)
      if (i != best) dfree(chunks[i].p, chunks[i].bytes);
    Chunk keep = chunks[best];
    chunks.clear();
    chunks.push_back(keep);
  }
  cur = 0;
  used = 0;
}

void *hgp_ctx::scratch(size_t bytes) {
  bytes = (bytes + 255) & ~size_t(255);
  if (bytes == 0) bytes = 256;
  // first fit in the current chunk, then in later chunks; otherwise a new chunk of exactly the
  // request (at least 64 MB)
  while (cur < chunks.size()) {
    if (used + bytes <= chunks[cur].bytes) {
      void *p = static_cast<char *>(chunks[cur].p) + used;
      used += bytes;
      return p;
    }
    if (cur + 1 == chunks.size()) break;
    ++cur;
    used = 0;
  }
  size_t want = bytes < (size_t(64) << 20) ? (size_t(64) << 20) : bytes;
  void *p = dalloc(want);
  if (!p) return nullptr;
  chunks.push_back({p, want});
  cur = chunks.size() - 1;
  used = bytes;
  return p;
}

extern "C" {

const char *hgp_last_error(void) { return g_err.c_str(); }

hgp_status hgp_ctx_create(int device, hgp_stream_t stream, const hgp_allocator *alloc, hgp_ctx **out) {
  if (!out) return set_error(HGP_E_ARG, "hgp_ctx_create: out is NULL");
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return set_error(HGP_E_CUDA, "hgp_ctx_create: no CUDA device (%s); there is no host fallback",
                     cudaGetErrorString(e));
  if (device < 0 || device >= ndev) return set_error(HGP_E_ARG, "hgp_ctx_create: bad device %d", device);
  DeviceGuard dg(device);   // the caller's current device is restored on return
  cudaDeviceProp prop;
  HGP_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10)
    return set_error(HGP_E_CUDA, "hgp_ctx_create: device %d is sm_%d%d; this library is built for sm_100a",
                     device, prop.major, prop.minor);
  hgp_ctx *c = new hgp_ctx();
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  c->stream = reinterpret_cast<cudaStream_t>(stream);
  if (alloc && alloc->alloc && alloc->free) {
    c->alloc = *alloc;
  } else {
    c->alloc.alloc = pool_alloc;
    c->alloc.free = pool_free;
    c->alloc.user = nullptr;
    c->builtin_pool = true;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;   // keep freed blocks cached across calls
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  if (cudaMalloc(&c->d_err, sizeof(uint64_t) * kErrSlots) != cudaSuccess ||
      cudaMalloc(&c->d_tiers, sizeof(uint64_t) * HGP_TIERS) != cudaSuccess ||
      cudaMemset(c->d_tiers, 0, sizeof(uint64_t) * HGP_TIERS) != cudaSuccess ||
      cudaMallocHost(&c->h_pin, sizeof(uint64_t) * 64) != cudaSuccess) {
    delete c;
    return set_error(HGP_E_OOM, "hgp_ctx_create: cannot allocate error slots");
  }
  for (auto &ev : c->ev) cudaEventCreate(&ev);
  *out = c;
  return HGP_OK;
}

void hgp_ctx_destroy(hgp_ctx *c) {
  if (!c) return;
  DeviceGuard dg(c->device);
  cudaStreamSynchronize(c->stream);
  for (auto &ch : c->chunks) c->dfree(ch.p, ch.bytes);
  c->chunks.clear();
  cudaStreamSynchronize(c->stream);
  cudaFree(c->d_err);
  cudaFree(c->d_tiers);
  cudaFreeHost(c->h_pin);
  for (auto &ev : c->ev) cudaEventDestroy(ev);
  for (auto &pr : c->prof_events) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
  for (auto &e : c->prof_pool) cudaEventDestroy(e);
  delete c;
}

uint64_t hgp_launch_count(const hgp_ctx *c) { return c ? c->launches : 0; }

hgp_status hgp_copy(hgp_ctx *c, void *dst, const void *src, size_t bytes) {
  if (!c || (!dst && bytes) || (!src && bytes)) return set_error(HGP_E_ARG, "hgp_copy: null argument");
  if (!bytes) return HGP_OK;
  DeviceGuard dg(c->device);
  HGP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->stream));
  cudaPointerAttributes a{}, b{};
  cudaPointerGetAttributes(&a, dst);
  cudaPointerGetAttributes(&b, src);
  cudaGetLastError();
  if (a.type == cudaMemoryTypeUnregistered || b.type == cudaMemoryTypeUnregistered)
    HGP_CUDA(cudaStreamSynchronize(c->stream));
  return HGP_OK;
}

hgp_status hgp_profile_begin(hgp_ctx *c, const char *name_filter) {
  if (!c || !name_filter) return set_error(HGP_E_ARG, "hgp_profile_begin: null argument");
  c->prof_filter = name_filter;
  c->prof_on = true;
  for (auto &pr : c->prof_events) { c->prof_pool.push_back(pr.first); c->prof_pool.push_back(pr.second); }
  c->prof_events.clear();
  c->prof_names.clear();
  return HGP_OK;
}

hgp_status hgp_profile_end(hgp_ctx *c, double *total_ms, uint64_t *launches) {
  if (!c) return set_error(HGP_E_ARG, "hgp_profile_end: null ctx");
  c->prof_on = false;
  DeviceGuard dg(c->device);
  HGP_CUDA(cudaStreamSynchronize(c->stream));
  double tot = 0;
  for (auto &pr : c->prof_events) {
    float ms = 0;
    HGP_CUDA(cudaEventElapsedTime(&ms, pr.first, pr.second));
    tot += ms;
  }
  if (total_ms) *total_ms = tot;
  if (launches) *launches = c->prof_events.size();
  return HGP_OK;
}

hgp_status hgp_profile_report(hgp_ctx *c, char *buf, size_t len) {
  if (!c || !buf || !len) return set_error(HGP_E_ARG, "hgp_profile_report: bad argument");
  DeviceGuard dg(c->device);
  HGP_CUDA(cudaStreamSynchronize(c->stream));
  std::vector<std::pair<std::string, std::pair<double, uint64_t>>> acc;
  for (size_t i = 0; i < c->prof_events.size(); ++i) {
    float ms = 0;
    HGP_CUDA(cudaEventElapsedTime(&ms, c->prof_events[i].first, c->prof_events[i].second));
    const std::string nm = c->prof_names[i];
    size_t k = 0;
    while (k < acc.size() && acc[k].first != nm) ++k;
    if (k == acc.size()) acc.push_back({nm, {0.0, 0}});
    acc[k].second.first += ms;
    acc[k].second.second += 1;
  }
  std::string out;
  for (auto &a : acc) {
    char line[256];
    snprintf(line, sizeof(line), "%s:%.6f:%llu;", a.first.c_str(), a.second.first, (unsigned long long)a.second.second);
    out += line;
  }
  snprintf(buf, len, "%s", out.c_str());
  return HGP_OK;
}

hgp_status hgp_tier_counts(hgp_ctx *c, uint64_t *out, int reset) {
  if (!c || !out) return set_error(HGP_E_ARG, "hgp_tier_counts: null argument");
  DeviceGuard dg(c->device);
  HGP_CUDA(cudaMemcpyAsync(out, c->d_tiers, sizeof(uint64_t) * HGP_TIERS, cudaMemcpyDeviceToHost, c->stream));
  HGP_CUDA(cudaStreamSynchronize(c->stream));
  for (int i = 0; i < HGP_TIERS; ++i) out[i] += c->h_tiers[i];
  if (reset) {
    HGP_CUDA(cudaMemsetAsync(c->d_tiers, 0, sizeof(uint64_t) * HGP_TIERS, c->stream));
    for (auto &x : c->h_tiers) x = 0;
  }
  return HGP_OK;
}

hgp_status hgp_sync(hgp_ctx *c) {
  if (!c) return set_error(HGP_E_ARG, "hgp_sync: null ctx");
  DeviceGuard dg(c->device);
  HGP_CUDA(cudaStreamSynchronize(c->stream));
  return HGP_OK;
}

hgp_status hgp_ctx_set_option(hgp_ctx *c, const char *name, int64_t value) {
  if (!c || !name) return set_error(HGP_E_ARG, "hgp_ctx_set_option: null argument");
  if (value < 0) return set_error(HGP_E_ARG, "hgp_ctx_set_option: %s must be >= 0", name);
  const std::string k = name;
  if (k == "fused_sample_min") c->opt.fused_sample_min = (uint64_t)value;
  else if (k == "fused_pool_cap") c->opt.fused_pool_cap = (uint64_t)value;
  else if (k == "unfused") c->opt.unfused = value != 0;
  else if (k == "inc_radix") c->opt.inc_radix = value != 0;
  else if (k == "debug_sync") c->opt.debug_sync = value != 0;
  else if (k == "no_hub") c->opt.no_hub = value != 0;
  else return set_error(HGP_E_ARG, "hgp_ctx_set_option: unknown option '%s'", name);
  return HGP_OK;
}

}  // extern "C"
