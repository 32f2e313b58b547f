// common.cuh — context, errors, launches, scratch arena and small device helpers.
// Part of the product path (libhgp.so); shares nothing with oracle/.
#pragma once
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdlib>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "hgp.h"

namespace hgp {

constexpr uint32_t kNone = HGP_NONE;
constexpr uint32_t kPurge = HGP_PURGE;
constexpr uint32_t kIdMask = 0x7FFFFFFFu;
constexpr uint32_t kEmpty = 0xFFFFFFFFu;   // empty hash slot
constexpr int kWarp = 32;

hgp_status set_error(hgp_status code, const char *fmt, ...);

// Device-side error slots: the lowest offending index per category (atomicMin).
enum ErrSlot : int {
  kErrStruct = 0,     // offsets / empty edge / nsrc > |e|
  kErrEdgeBig = 1,    // |e| > 2^24 (overflow)
  kErrPinRange = 2,
  kErrDup = 3,
  kErrEdgeW = 4,
  kErrNodeW = 5,
  kErrInfeasW = 6,    // node size > Omega
  kErrInfeasD = 7,    // node in_mu > Delta
  kErrCycle = 8,      // proposal cycle longer than 2 (a4)
  kErrInternal = 9,
  kErrSlots = 16
};

}  // namespace hgp

struct hgp_ctx {
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  hgp_allocator alloc{};
  bool builtin_pool = false;
  // scratch arena (reset at every top-level API call)
  struct Chunk { void *p; size_t bytes; };
  std::vector<Chunk> chunks;
  size_t cur = 0;        // chunk currently bump-allocated from
  size_t used = 0;       // bytes used in chunks[cur]
  int depth = 0;
  uint64_t launches = 0;
  uint64_t *d_err = nullptr;       // [kErrSlots] device
  unsigned long long *d_tiers = nullptr;   // [HGP_TIERS] device work counters per kernel tier
  uint64_t h_tiers[HGP_TIERS] = {};        // host-side part (tiers the host decides, e.g. a4 jumps)
  uint64_t *h_pin = nullptr;       // [64] pinned host staging
  cudaEvent_t ev[8] = {};
  // explicit options (hgp_ctx_set_option; tests and experiments only — no environment variables)
  struct Options {
    uint64_t fused_sample_min = 65536;   // level sizes from which the fused kernel samples tier A first
    uint64_t fused_pool_cap = 0;         // 0 = automatic; else the first pool's capacity (test hook)
    bool unfused = false;                // every node on the unfused a2 -> a3 path (test hook)
    bool inc_radix = false;              // a1/a5 incidence transpose by radix sort (measured slower)
    bool debug_sync = false;             // serialise and trace every launch
    bool no_hub = false;                 // hub nodes on the global-memory tiers (test hook)
  } opt;
  // profiling: CUDA events around every launch whose name contains prof_filter
  std::string prof_filter;
  bool prof_on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_events;
  std::vector<const char *> prof_names;
  std::vector<cudaEvent_t> prof_pool;
  cudaEvent_t prof_event();

  void *dalloc(size_t bytes);
  void dfree(void *p, size_t bytes);
  void *scratch(size_t bytes);     // 256-byte aligned, valid until the next top-level call
  void reset_scratch();
};

namespace hgp {

// Makes the ctx's device current for the scope and restores the caller's device on exit.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) { prev = -1; cudaGetLastError(); }
    if (prev != dev) cudaSetDevice(dev);
  }
  DeviceGuard(const DeviceGuard &) = delete;
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// RAII guard for top-level API entry points: the ctx's device is current inside the call (the
// caller's is restored), and scratch is reset at depth 0.
struct ApiScope {
  hgp_ctx *c;
  DeviceGuard dg;
  explicit ApiScope(hgp_ctx *c_) : c(c_), dg(c_->device) {
    if (c->depth++ == 0) c->reset_scratch();
  }
  ~ApiScope() { --c->depth; }
};

// True exactly once per (flag word, device): per-device one-time setup such as
// cudaFuncSetAttribute, which applies to the current device only.
inline bool once_per_device(uint64_t *mask, int dev) {
  const unsigned long long bit = 1ull << (dev & 63);
  return (__atomic_fetch_or(reinterpret_cast<unsigned long long *>(mask), bit, __ATOMIC_ACQ_REL) & bit) == 0;
}

// CTAs of `kernel` that are resident at once on the whole GPU (occupancy x SMs): the grid of a
// persistent grid-stride kernel. A larger grid leaves CTAs waiting for a whole resident CTA's
// share of the list to finish (a second, partial wave: the makespan grows by up to 2x).
template <class K>
inline uint32_t resident_grid(const hgp_ctx *c, K kernel, int threads, size_t smem) {
  int per = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, smem) != cudaSuccess || per < 1) {
    cudaGetLastError();
    per = 1;
  }
  return (uint32_t)per * (uint32_t)c->sm_count;
}

#define HGP_CUDA(x)                                                                              \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess)                                                                       \
      return ::hgp::set_error(HGP_E_CUDA, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, \
                              __LINE__);                                                         \
  } while (0)

#define HGP_TRY(x)                     \
  do {                                 \
    hgp_status s_ = (x);               \
    if (s_ != HGP_OK) return s_;       \
  } while (0)

template <class K, class... Args>
inline hgp_status launch(hgp_ctx *c, const char *name, K kernel, dim3 grid, dim3 block, size_t smem,
                         Args... args) {
  if (grid.x == 0 || grid.y == 0 || grid.z == 0) return HGP_OK;
  const bool dbg = c->opt.debug_sync;   // debugging: serialise + trace
  const bool prof = (c->prof_on && strstr(name, c->prof_filter.c_str()) != nullptr) || dbg;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (prof) { e0 = c->prof_event(); e1 = c->prof_event(); cudaEventRecord(e0, c->stream); }
  kernel<<<grid, block, smem, c->stream>>>(args...);
  if (prof) { cudaEventRecord(e1, c->stream); c->prof_events.push_back({e0, e1}); c->prof_names.push_back(name); }
  c->launches++;
  if (dbg) {
    fprintf(stderr, "[hgp] %s grid %u block %u smem %zu ...", name, grid.x, block.x, smem);
    cudaError_t se = cudaStreamSynchronize(c->stream);
    float ms = -1.f;
    if (e0) { cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); }
    fprintf(stderr, " %s %.3f ms\n", cudaGetErrorString(se), ms);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(HGP_E_CUDA, "launch %s: %s", name, cudaGetErrorString(e));
  return HGP_OK;
}

// Allocate zero-initialised scratch.
template <class T>
inline T *scratch_zero(hgp_ctx *c, size_t n, hgp_status *st) {
  T *p = static_cast<T *>(c->scratch(sizeof(T) * (n ? n : 1)));
  if (!p) { *st = set_error(HGP_E_OOM, "scratch allocation of %zu bytes failed", sizeof(T) * n); return nullptr; }
  cudaError_t e = cudaMemsetAsync(p, 0, sizeof(T) * (n ? n : 1), c->stream);
  if (e != cudaSuccess) { *st = set_error(HGP_E_CUDA, "memset: %s", cudaGetErrorString(e)); return nullptr; }
  return p;
}
template <class T>
inline T *scratch_raw(hgp_ctx *c, size_t n, hgp_status *st) {
  T *p = static_cast<T *>(c->scratch(sizeof(T) * (n ? n : 1)));
  if (!p) *st = set_error(HGP_E_OOM, "scratch allocation of %zu bytes failed", sizeof(T) * n);
  return p;
}
template <class T>
inline T *dalloc_n(hgp_ctx *c, size_t n, hgp_status *st) {
  T *p = static_cast<T *>(c->dalloc(sizeof(T) * (n ? n : 1)));
  if (!p) *st = set_error(HGP_E_OOM, "device allocation of %zu bytes failed", sizeof(T) * n);
  return p;
}

// Read device scalars into host (synchronises the ctx stream).
hgp_status read_back(hgp_ctx *c, const void *dptr, size_t bytes, void *host);
inline hgp_status read_u64(hgp_ctx *c, const uint64_t *d, uint64_t *h) { return read_back(c, d, 8, h); }

// Reset / read the device error slots.
hgp_status clear_errors(hgp_ctx *c);
hgp_status fetch_errors(hgp_ctx *c, uint64_t out[kErrSlots]);

inline uint32_t div_up(uint64_t a, uint64_t b) { return static_cast<uint32_t>((a + b - 1) / b); }

// ---------------------------------------------------------------------------- device helpers
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

inline uint64_t splitmix64_host(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Explicit shared-memory accesses through 32-bit shared-window addresses.
__device__ __forceinline__ uint32_t smem_u32addr(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// keep a value in a register (stops the compiler from rematerialising, e.g., the shared window base)
__device__ __forceinline__ uint32_t opaque_u32(uint32_t x) {
  asm volatile("mov.b32 %0, %0;" : "+r"(x));
  return x;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
// A key probe that races with other threads' CAS inserts on purpose (the value is only a hint; the
// CAS decides): a relaxed CTA-scope load says so to the memory model (same LDS in SASS).
__device__ __forceinline__ uint32_t lds_hint_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.relaxed.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void red_add_u32(uint32_t a, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// predicated forms (no branch around the access)
__device__ __forceinline__ void red_add_u32_if(bool p, uint32_t a, uint32_t v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q red.shared.add.u32 [%0], %1;\n}" ::"r"(a), "r"(v),
               "r"((uint32_t)p)
               : "memory");
}
__device__ __forceinline__ void sts_u32_if(bool p, uint32_t a, uint32_t v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q st.shared.u32 [%0], %1;\n}" ::"r"(a), "r"(v),
               "r"((uint32_t)p)
               : "memory");
}
__device__ __forceinline__ uint32_t cas_u32(uint32_t a, uint32_t cmp, uint32_t val) {
  uint32_t old;
  asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;" : "=r"(old) : "r"(a), "r"(cmp), "r"(val) : "memory");
  return old;
}

// Multiplicative (Fibonacci) hash of a node id into a power-of-two table. (A locality-preserving
// variant — low id bits kept so that sorted pins hit consecutive banks — was measured 6x slower on
// C2: runs of consecutive ids merge into long linear-probing clusters.)
__device__ __forceinline__ uint32_t hash_slot(uint32_t key, uint32_t log2size) {
  return (key * 0x9E3779B1u) >> (32u - log2size);
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}
template <class T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T w = __shfl_xor_sync(0xFFFFFFFFu, v, o);
    v = w > v ? w : v;
  }
  return v;
}
// inclusive warp prefix sum
template <class T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T w = __shfl_up_sync(0xFFFFFFFFu, v, o);
    if (lane >= (uint32_t)o) v += w;
  }
  return v;
}

// Work counter of a kernel tier: thread 0 of a CTA adds the nodes it processed, once per launch.
__device__ __forceinline__ void tier_add(unsigned long long *tiers, int tier, uint64_t n) {
  if (tiers && n) atomicAdd(tiers + tier, (unsigned long long)n);
}

__device__ __forceinline__ void report_min(uint64_t *err, int slot, uint64_t idx) {
  atomicMin(reinterpret_cast<unsigned long long *>(err + slot), static_cast<unsigned long long>(idx));
}

}  // namespace hgp
