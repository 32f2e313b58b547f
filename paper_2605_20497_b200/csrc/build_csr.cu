#include <cstdlib>
// build_csr.cu — a1: validate the problem statement and materialise the
// compressed sparse level: canonical hyperedges (src block ascending, dst block
// ascending) and the transposed incidence (in(n) ascending, then out(n) ascending), with
// |src(e)|, |in(n)| and the inbound multiplicity sums in_mu(n).
#include "csr_impl.cuh"
#include "lbs.cuh"
#include "scan.cuh"
#include "sort.cuh"

namespace hgp {

// ---------------------------------------------------------------- validation (categories A, D, E, F)
// slot kErrStruct holds (e << 2 | type): type 0 offsets decrease, 1 empty, 2 nsrc > |e|, 3 |e| > 2^24
__global__ void k_validate_edges(hgp_input in, uint64_t *err, unsigned long long *stats) {
  const uint32_t E = in.num_edges;
  uint64_t sw = 0;
  uint32_t mx = 0;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    const uint64_t lo = in.edge_off[e], hi = in.edge_off[e + 1];
    int type = -1;
    if (hi < lo) type = 0;
    else if (hi == lo) type = 1;
    else if (in.edge_nsrc[e] > hi - lo) type = 2;
    else if (hi - lo > (1ull << 24)) type = 3;
    if (type >= 0) report_min(err, kErrStruct, ((uint64_t)e << 2) | (uint64_t)type);
    else mx = max(mx, (uint32_t)(hi - lo));
    const uint32_t w = in.edge_w[e];
    if (w == 0) report_min(err, kErrEdgeW, e);
    sw += w;
  }
  sw = warp_sum(sw);
  mx = warp_max(mx);
  if (lane_id() == 0) {
    atomicAdd(&stats[0], (unsigned long long)sw);
    atomicMax(&stats[2], (unsigned long long)mx);
  }
}

__global__ void k_validate_nodes(const uint32_t *node_w, uint32_t N, uint64_t *err, unsigned long long *stats) {
  uint64_t s = 0;
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
    const uint32_t w = node_w[n];
    if (w == 0) report_min(err, kErrNodeW, n);
    s += w;
  }
  s = warp_sum(s);
  if (lane_id() == 0) atomicAdd(&stats[1], (unsigned long long)s);
}

// category B: pin range (pin-parallel)
__global__ void __launch_bounds__(kLbsThreads) k_check_pin_range(const uint64_t *edge_off, uint32_t E, uint64_t P,
                                                                 const uint32_t *pins, uint32_t N, uint64_t *err) {
  __shared__ LbsShared sh;
  const uint64_t p0 = (uint64_t)blockIdx.x * kLbsTile;
  bool bad = false;
  uint64_t firstbad = 0;
#pragma unroll
  for (int k = 0; k < kLbsItems; ++k) {
    uint64_t p = p0 + (uint64_t)k * kLbsThreads + threadIdx.x;
    if (p < P && pins[p] >= N && !bad) { bad = true; firstbad = p; }
  }
  if (!__syncthreads_or(bad)) return;
  lbs_stage(sh, edge_off, E, p0, P);
  if (bad) report_min(err, kErrPinRange, lbs_edge(sh, edge_off, E, firstbad));
}

// category C: duplicate pins / src ∩ dst on the sorted blocks (warp per edge)
__global__ void k_check_dups(const uint64_t *edge_off, const uint32_t *edge_nsrc, const uint32_t *pins, uint32_t E,
                             uint64_t *err) {
  const uint32_t lane = lane_id();
  const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t e = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); e < E; e += nw) {
    const uint64_t lo = edge_off[e], hi = edge_off[e + 1], s = lo + edge_nsrc[e];
    bool dup = false;
    for (uint64_t j = lo + 1 + lane; j < hi; j += 32)
      if (j != s && pins[j] == pins[j - 1]) dup = true;
    // every source pin must be absent from the sorted destination block
    for (uint64_t j = lo + lane; j < s && !dup; j += 32) {
      const uint32_t x = pins[j];
      uint64_t a = s, b = hi;
      while (a < b) {
        uint64_t m = (a + b) >> 1;
        if (pins[m] < x) a = m + 1; else b = m;
      }
      if (a < hi && pins[a] == x) dup = true;
    }
    if (__any_sync(0xFFFFFFFFu, dup) && lane == 0) report_min(err, kErrDup, e);
  }
}

__global__ void k_fill_u32(uint32_t *a, uint64_t n, uint32_t v) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    a[i] = v;
}

struct EdgeBlockSeg {   // segment 2e = src(e), 2e+1 = dst(e)
  const uint64_t *off;
  const uint32_t *nsrc;
  __device__ void operator()(uint64_t i, uint64_t &beg, uint32_t &len) const {
    const uint64_t e = i >> 1;
    const uint64_t lo = off[e], hi = off[e + 1], s = lo + nsrc[e];
    if (i & 1) { beg = s; len = (uint32_t)(hi - s); }
    else { beg = lo; len = (uint32_t)(s - lo); }
  }
};

// ---------------------------------------------------------------- incidence transpose
__global__ void __launch_bounds__(kLbsThreads) k_inc_count(const uint64_t *edge_off, const uint32_t *edge_nsrc,
                                                           const uint32_t *edge_mu, uint32_t E, uint64_t P,
                                                           const uint32_t *pins, uint32_t *cnt_in, uint32_t *cnt_out,
                                                           uint32_t *in_mu) {
  __shared__ LbsShared sh;
  const uint64_t p0 = (uint64_t)blockIdx.x * kLbsTile;
  lbs_stage(sh, edge_off, E, p0, P);
#pragma unroll 4
  for (int k = 0; k < kLbsItems; ++k) {
    const uint64_t p = p0 + (uint64_t)k * kLbsThreads + threadIdx.x;
    if (p >= P) break;
    const uint32_t e = lbs_edge(sh, edge_off, E, p);
    const uint32_t n = pins[p];
    if (p >= edge_off[e] + edge_nsrc[e]) {
      atomicAdd(&cnt_in[n], 1u);
      atomicAdd(&in_mu[n], edge_mu[e]);
    } else {
      atomicAdd(&cnt_out[n], 1u);
    }
  }
}

__global__ void __launch_bounds__(kLbsThreads) k_inc_scatter(const uint64_t *edge_off, const uint32_t *edge_nsrc,
                                                             uint32_t E, uint64_t P, const uint32_t *pins,
                                                             const uint64_t *inc_off, const uint32_t *inc_nin,
                                                             uint32_t *cur_in, uint32_t *cur_out, uint32_t *inc) {
  __shared__ LbsShared sh;
  const uint64_t p0 = (uint64_t)blockIdx.x * kLbsTile;
  lbs_stage(sh, edge_off, E, p0, P);
#pragma unroll 4
  for (int k = 0; k < kLbsItems; ++k) {
    const uint64_t p = p0 + (uint64_t)k * kLbsThreads + threadIdx.x;
    if (p >= P) break;
    const uint32_t e = lbs_edge(sh, edge_off, E, p);
    const uint32_t n = pins[p];
    uint64_t pos;
    if (p >= edge_off[e] + edge_nsrc[e]) pos = inc_off[n] + atomicAdd(&cur_in[n], 1u);
    else pos = inc_off[n] + inc_nin[n] + atomicAdd(&cur_out[n], 1u);
    inc[pos] = e;
  }
}

__global__ void k_max_deg(const uint64_t *off, uint32_t N, unsigned int *out) {
  uint32_t mx = 0;
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x)
    mx = max(mx, (uint32_t)(off[n + 1] - off[n]));
  mx = warp_max(mx);
  if (lane_id() == 0) atomicMax(out, mx);
}

struct IncBlockSeg {   // segment 2n = in(n), 2n+1 = out(n)
  const uint64_t *off;
  const uint32_t *nin;
  __device__ void operator()(uint64_t i, uint64_t &beg, uint32_t &len) const {
    const uint64_t n = i >> 1;
    const uint64_t lo = off[n], hi = off[n + 1], s = lo + nin[n];
    if (i & 1) { beg = s; len = (uint32_t)(hi - s); }
    else { beg = lo; len = (uint32_t)(s - lo); }
  }
};

// Given edge_off/edge_nsrc/pins/edge_mu of g (device), allocate and fill inc_off, inc_nin,
// inc, in_mu and g->max_inc. Synchronises (reads max degree).
hgp_status build_incidence(hgp_ctx *c, hgp_csr *g) {
  // The radix transpose (radix.cu) is exact and deterministic but measured slower on B200 at C2
  // (a1 9.5 vs 7.4 ms: its first scatter pass runs at ~0.5 TB/s); opt in with hgp_ctx_set_option(ctx, "inc_radix", 1).
  const bool radix_path = c->opt.inc_radix;
  if (radix_path && g->P < (1ull << 30) && g->N < (1u << 30)) return build_incidence_radix(c, g);
  hgp_status st = HGP_OK;
  const uint32_t N = g->N, E = g->E;
  const uint64_t P = g->P;
  g->inc_off = dalloc_n<uint64_t>(c, (size_t)N + 1, &st);
  g->inc_nin = dalloc_n<uint32_t>(c, N, &st);
  g->inc = dalloc_n<uint32_t>(c, P, &st);
  g->in_mu = dalloc_n<uint32_t>(c, N, &st);
  uint32_t *cnt = scratch_zero<uint32_t>(c, 2 * (size_t)N + 1, &st);   // cnt_in | cnt_out | maxdeg
  if (st != HGP_OK) return st;
  uint32_t *cnt_in = cnt, *cnt_out = cnt + N;
  HGP_CUDA(cudaMemsetAsync(g->in_mu, 0, sizeof(uint32_t) * (N ? N : 1), c->stream));
  const uint32_t tiles = div_up(P, kLbsTile);
  HGP_TRY(launch(c, "inc_count", k_inc_count, dim3(tiles), dim3(kLbsThreads), 0, (const uint64_t *)g->edge_off,
                 (const uint32_t *)g->edge_nsrc, (const uint32_t *)g->edge_mu, E, P, (const uint32_t *)g->pins,
                 cnt_in, cnt_out, g->in_mu));
  HGP_TRY(scan_exclusive(c, InSum2U32{cnt_in, cnt_out}, N, g->inc_off, nullptr));
  HGP_CUDA(cudaMemcpyAsync(g->inc_nin, cnt_in, sizeof(uint32_t) * N, cudaMemcpyDeviceToDevice, c->stream));
  HGP_CUDA(cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * (2 * (size_t)N + 1), c->stream));
  HGP_TRY(launch(c, "inc_scatter", k_inc_scatter, dim3(tiles), dim3(kLbsThreads), 0, (const uint64_t *)g->edge_off,
                 (const uint32_t *)g->edge_nsrc, E, P, (const uint32_t *)g->pins, (const uint64_t *)g->inc_off,
                 (const uint32_t *)g->inc_nin, cnt_in, cnt_out, g->inc));
  unsigned int *d_max = reinterpret_cast<unsigned int *>(cnt + 2 * (size_t)N);
  HGP_TRY(launch(c, "max_deg", k_max_deg, dim3(div_up(N, 256) < 1024 ? div_up(N, 256) : 1024), dim3(256), 0,
                 (const uint64_t *)g->inc_off, N, d_max));
  uint32_t mx = 0;
  HGP_TRY(read_back(c, d_max, 4, &mx));
  g->max_inc = mx;
  return segmented_sort(c, IncBlockSeg{g->inc_off, g->inc_nin}, 2 * (uint64_t)N, g->inc, mx);
}

void free_csr(hgp_ctx *c, hgp_csr *g) {
  if (!g) return;
  const size_t N = g->N, E = g->E, P = g->P;
  c->dfree(g->edge_off, 8 * (E + 1));
  c->dfree(g->edge_nsrc, 4 * E);
  c->dfree(g->pins, 4 * P);
  c->dfree(g->edge_w, 4 * E);
  c->dfree(g->edge_mu, 4 * E);
  c->dfree(g->node_w, 4 * N);
  c->dfree(g->inc_off, 8 * (N + 1));
  c->dfree(g->inc_nin, 4 * N);
  c->dfree(g->inc, 4 * P);
  c->dfree(g->in_mu, 4 * N);
  memset(g, 0, sizeof(*g));
}

}  // namespace hgp

using namespace hgp;

extern "C" hgp_status hgp_build_csr(hgp_ctx *c, const hgp_input *in, hgp_csr *out) {
  if (!c || !in || !out) return set_error(HGP_E_ARG, "hgp_build_csr: null argument");
  ApiScope scope(c);
  memset(out, 0, sizeof(*out));
  const uint32_t N = in->num_nodes, E = in->num_edges;
  if (N >= (1u << 31)) return set_error(HGP_E_OVERFLOW, "num_nodes %u >= 2^31", N);
  if (E == kNone) return set_error(HGP_E_OVERFLOW, "num_edges too large");
  if (!in->edge_off || (E && (!in->edge_nsrc || !in->edge_w || !in->pins)) || (N && !in->node_w))
    return set_error(HGP_E_ARG, "hgp_build_csr: null array");
  uint64_t off0 = 0;
  HGP_TRY(read_back(c, in->edge_off, 8, &off0));
  if (off0 != 0) return set_error(HGP_E_MALFORMED, "edge 0: edge_off[0] != 0");
  hgp_status st = HGP_OK;
  HGP_TRY(clear_errors(c));
  unsigned long long *stats = scratch_zero<unsigned long long>(c, 4, &st);
  if (!stats) return st;
  const uint32_t gE = E ? (div_up(E, 256) < 8u * c->sm_count ? div_up(E, 256) : 8u * c->sm_count) : 0;
  const uint32_t gN = N ? (div_up(N, 256) < 8u * c->sm_count ? div_up(N, 256) : 8u * c->sm_count) : 0;
  HGP_TRY(launch(c, "validate_edges", k_validate_edges, dim3(gE), dim3(256), 0, *in, c->d_err, stats));
  HGP_TRY(launch(c, "validate_nodes", k_validate_nodes, dim3(gN), dim3(256), 0, in->node_w, N, c->d_err, stats));
  uint64_t err[kErrSlots];
  HGP_TRY(fetch_errors(c, err));
  if (err[kErrStruct] != UINT64_MAX) {
    const uint64_t e = err[kErrStruct] >> 2;
    switch (err[kErrStruct] & 3) {
      case 0: return set_error(HGP_E_MALFORMED, "edge %llu: offsets decrease", (unsigned long long)e);
      case 1: return set_error(HGP_E_MALFORMED, "edge %llu: empty hyperedge", (unsigned long long)e);
      case 2: return set_error(HGP_E_MALFORMED, "edge %llu: nsrc > |e|", (unsigned long long)e);
      default: return set_error(HGP_E_OVERFLOW, "edge %llu: |e| > 2^24", (unsigned long long)e);
    }
  }
  uint64_t hs[4];
  HGP_TRY(read_back(c, stats, sizeof(hs), hs));
  uint64_t P = 0;
  if (E) HGP_TRY(read_back(c, in->edge_off + E, 8, &P));
  out->N = N;
  out->E = E;
  out->P = P;
  out->max_edge = (uint32_t)hs[2];
  out->edge_off = dalloc_n<uint64_t>(c, (size_t)E + 1, &st);
  out->edge_nsrc = dalloc_n<uint32_t>(c, E, &st);
  out->pins = dalloc_n<uint32_t>(c, P, &st);
  out->edge_w = dalloc_n<uint32_t>(c, E, &st);
  out->edge_mu = dalloc_n<uint32_t>(c, E, &st);
  out->node_w = dalloc_n<uint32_t>(c, N, &st);
  if (st != HGP_OK) { free_csr(c, out); return st; }
  auto fail = [&](hgp_status s) { free_csr(c, out); return s; };
  if (P && cudaMemcpyAsync(out->pins, in->pins, 4 * P, cudaMemcpyDeviceToDevice, c->stream) != cudaSuccess)
    return fail(set_error(HGP_E_CUDA, "copy pins"));
  if (P) {
    hgp_status s = launch(c, "check_pin_range", k_check_pin_range, dim3(div_up(P, kLbsTile)), dim3(kLbsThreads), 0,
                          in->edge_off, E, P, (const uint32_t *)out->pins, N, c->d_err);
    if (s) return fail(s);
    s = segmented_sort(c, EdgeBlockSeg{in->edge_off, in->edge_nsrc}, 2 * (uint64_t)E, out->pins, out->max_edge);
    if (s) return fail(s);
    const uint32_t g = div_up(E, 8) < 64u * c->sm_count ? div_up(E, 8) : 64u * c->sm_count;
    s = launch(c, "check_dups", k_check_dups, dim3(g), dim3(256), 0, in->edge_off, in->edge_nsrc,
               (const uint32_t *)out->pins, E, c->d_err);
    if (s) return fail(s);
  }
  hgp_status s = fetch_errors(c, err);
  if (s) return fail(s);
  if (err[kErrPinRange] != UINT64_MAX)
    return fail(set_error(HGP_E_MALFORMED, "edge %llu: pin out of range", (unsigned long long)err[kErrPinRange]));
  if (err[kErrDup] != UINT64_MAX)
    return fail(set_error(HGP_E_MALFORMED, "edge %llu: duplicate pin", (unsigned long long)err[kErrDup]));
  if (err[kErrEdgeW] != UINT64_MAX)
    return fail(set_error(HGP_E_MALFORMED, "edge %llu: zero weight", (unsigned long long)err[kErrEdgeW]));
  if (err[kErrNodeW] != UINT64_MAX)
    return fail(set_error(HGP_E_MALFORMED, "node %llu: zero size", (unsigned long long)err[kErrNodeW]));
  if (hs[0] >= (1ull << 32)) return fail(set_error(HGP_E_OVERFLOW, "sum of edge weights >= 2^32"));
  if (hs[1] >= (1ull << 32)) return fail(set_error(HGP_E_OVERFLOW, "sum of node sizes >= 2^32"));
  if (cudaMemcpyAsync(out->edge_off, in->edge_off, 8 * ((size_t)E + 1), cudaMemcpyDeviceToDevice, c->stream) ||
      (E && cudaMemcpyAsync(out->edge_nsrc, in->edge_nsrc, 4 * (size_t)E, cudaMemcpyDeviceToDevice, c->stream)) ||
      (E && cudaMemcpyAsync(out->edge_w, in->edge_w, 4 * (size_t)E, cudaMemcpyDeviceToDevice, c->stream)) ||
      (N && cudaMemcpyAsync(out->node_w, in->node_w, 4 * (size_t)N, cudaMemcpyDeviceToDevice, c->stream)))
    return fail(set_error(HGP_E_CUDA, "copy input arrays"));
  s = launch(c, "fill_mu", k_fill_u32, dim3(gE ? gE : 1), dim3(256), 0, out->edge_mu, (uint64_t)E, 1u);
  if (s) return fail(s);
  s = build_incidence(c, out);
  if (s) return fail(s);
  return HGP_OK;
}

extern "C" void hgp_csr_free(hgp_ctx *c, hgp_csr *g) {
  if (c && g) { DeviceGuard dg(c->device); free_csr(c, g); }
}
