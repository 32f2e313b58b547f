// Microbenchmark: shared-memory histogram update throughput on B200 (sm_100a).
// Each variant: every warp does ITERS updates per lane into a 4096-slot (16 KB) table at
// pseudo-random (or consecutive) addresses. Reports SM-cycles per lane-update.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int S = 4096, ITERS = 4096;

__device__ __forceinline__ uint32_t hsh(uint32_t x) { return (x * 0x9E3779B1u) >> 20; }

template <int MODE>
__global__ void k(uint32_t *out, uint32_t seed, long long *cyc) {
  __shared__ uint32_t t[S];
  __shared__ uint32_t k2[S];
  for (int i = threadIdx.x; i < S; i += blockDim.x) { t[i] = 0; k2[i] = i; }
  __syncthreads();
  long long c0 = clock64();
  uint32_t x = seed + threadIdx.x * 7919u + blockIdx.x * 104729u, acc = 0;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = 0; i < ITERS; ++i) {
    x = x * 1664525u + 1013904223u;
    uint32_t a;
    if (MODE == 4) a = (warp * 997 + i * 32 + lane) & (S - 1);   // consecutive: conflict-free
    else a = hsh(x);
    if (MODE == 0 || MODE == 4) atomicAdd(&t[a], 1u);            // red.shared.add
    else if (MODE == 1) { volatile uint32_t *vt = t; vt[a] = vt[a] + 1; }   // LDS+STS RMW (racy)
    else if (MODE == 2) { acc += ((volatile uint32_t *)t)[a]; }          // LDS only
    else if (MODE == 3) { volatile uint32_t *vk = k2; uint32_t kk = vk[a]; if (kk == a) { volatile uint32_t *vt = t; vt[a] = vt[a] + 1; } }  // key check + RMW
    else if (MODE == 5) acc += atomicAdd(&t[a], 1u);              // atom with return
    else if (MODE == 6) { volatile uint32_t *vk = k2; uint32_t kk = vk[a]; if (kk == a) atomicAdd(&t[a], 1u); }  // key check + red
    else if (MODE == 7) { atomicAdd((unsigned long long *)&t[a & ~1u], 1ull); }  // 64-bit
    else if (MODE == 8) acc += atomicCAS(&k2[a], 0xFFFFFFFFu, a);   // CAS that finds the key (fails)
    else if (MODE == 9) {                                            // CAS-always insert + branch-free add
      const uint32_t o = atomicCAS(&k2[a], 0xFFFFFFFFu, a);
      atomicAdd(&t[a], (o == a || o == 0xFFFFFFFFu) ? 1u : 0u);
    } else if (MODE == 10) {                                         // key LDS + branch-free add
      const uint32_t kk = ((volatile uint32_t *)k2)[a];
      atomicAdd(&t[a], kk == a ? 1u : 0u);
    }
  }
  __syncthreads();
  long long c1 = clock64();
  if (threadIdx.x == 0) atomicMax(cyc, c1 - c0);
  if (acc == 12345) out[0] = acc;
  if (threadIdx.x == 0) out[1 + blockIdx.x] = t[seed & (S - 1)];
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t *out; long long *cyc; cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 8);
  const char *names[] = {"red.shared.add random", "LDS+STS RMW random (racy)", "LDS random", "key LDS + RMW random",
                         "red.shared.add consecutive", "atom.shared.add (ret) random", "key LDS + red random",
                         "atom.shared.add.u64 random", "atom.shared.cas (finds key) random",
                         "cas-always + red (branch-free)", "key LDS + red (branch-free)"};
  for (int threads : {256, 512, 1024}) {
    for (int mode = 0; mode < 11; ++mode) {
      void (*kp)(uint32_t *, uint32_t, long long *) = nullptr;
      switch (mode) { case 0: kp = k<0>; break; case 1: kp = k<1>; break; case 2: kp = k<2>; break; case 3: kp = k<3>; break;
                      case 4: kp = k<4>; break; case 5: kp = k<5>; break; case 6: kp = k<6>; break; case 7: kp = k<7>; break;
                      case 8: kp = k<8>; break; case 9: kp = k<9>; break; default: kp = k<10>; }
      const int blocks = sms * (2048 / threads);
      cudaMemset(cyc, 0, 8);
      kp<<<blocks, threads>>>(out, 1, cyc);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      kp<<<blocks, threads>>>(out, 2, cyc);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double lanes = (double)blocks * threads * ITERS;
      const double sm_cycles = ms * 1e-3 * 1.965e9 * sms;
      printf("threads/CTA %4d  %-32s %.3f ms  %.3f SM-cyc per lane-update  (%.2f Gupd/s)\n", threads, names[mode], ms,
             sm_cycles / lanes, lanes / ms / 1e6);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
