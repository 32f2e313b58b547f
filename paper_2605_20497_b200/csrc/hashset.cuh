// hashset.cuh — open-addressing (linear probing) sets of node ids in shared or global memory.
// Keys are node ids < 2^31; kEmpty marks a free slot. Tables are power-of-two sized and
// kept at load <= 1/2 by the callers, so probes stay short and never wrap around a full table.
#pragma once
#include "common.cuh"

namespace hgp {

// Insert key; returns true if this call inserted it (false: already present).
__device__ __forceinline__ bool hs_insert(uint32_t *keys, uint32_t log2s, uint32_t key) {
  const uint32_t mask = (1u << log2s) - 1;
  uint32_t s = hash_slot(key, log2s);
  volatile uint32_t *vk = keys;
  while (true) {
    const uint32_t k = vk[s];
    if (k == key) return false;
    if (k == kEmpty) {
      const uint32_t old = atomicCAS(&keys[s], kEmpty, key);
      if (old == kEmpty) return true;
      if (old == key) return false;
    }
    s = (s + 1) & mask;
  }
}

// Insert key and return its slot.
__device__ __forceinline__ uint32_t hs_insert_slot(uint32_t *keys, uint32_t log2s, uint32_t key, bool *inserted) {
  const uint32_t mask = (1u << log2s) - 1;
  uint32_t s = hash_slot(key, log2s);
  volatile uint32_t *vk = keys;
  while (true) {
    const uint32_t k = vk[s];
    if (k == key) { *inserted = false; return s; }
    if (k == kEmpty) {
      const uint32_t old = atomicCAS(&keys[s], kEmpty, key);
      if (old == kEmpty) { *inserted = true; return s; }
      if (old == key) { *inserted = false; return s; }
    }
    s = (s + 1) & mask;
  }
}

// Slot of key, or kNone if absent. Only valid once all inserts are complete (after a barrier).
__device__ __forceinline__ uint32_t hs_find(const uint32_t *keys, uint32_t log2s, uint32_t key) {
  const uint32_t mask = (1u << log2s) - 1;
  uint32_t s = hash_slot(key, log2s);
  while (true) {
    const uint32_t k = keys[s];
    if (k == key) return s;
    if (k == kEmpty) return kNone;
    s = (s + 1) & mask;
  }
}

}  // namespace hgp
