// refine.cu — the rows after the level on the GPU:
//   f1  quality of a partition: Eq.1 connectivity, Eq.16 cut-net, the
//       size and distinct-inbound loads of every partition (inbound mu-weighted,
//       reading #12) and how many partitions violate Omega / Delta;
//   f3  the sparse pins(p, e) / pins_in(p, e) matrix, the Eq.13 move proposal
//       of every node and the in-sequence gain of every move of a sequence
//       (Eqs.14-15);
//   f4  the event-based validation of a move sequence: size and inbound events,
//       sorts by (p, e, n_seq) and (p, n_seq), segmented prefix sums, 0<->1 transitions of
//       pins_in, the per-move count of violated constraints; and the landing point.
//
// Everything is integer (weights u32, sums exact), so results are bit-identical to the oracle
// (the CPU oracle of the tests) whatever the schedule.
#include <algorithm>

#include "csr_impl.cuh"
#include "scan.cuh"
#include "sort.cuh"

namespace hgp {

constexpr int kErrPart = 11;   // lowest node with part[n] >= nparts
constexpr int kErrSeq = 12;    // lowest sequence position with a bad entry (range, duplicate, dest)

// ------------------------------------------------------------------------------ pins(p, e)
__global__ void k_gather_part(const uint32_t *pins, uint64_t P, const uint32_t *part, uint32_t nparts, uint32_t N,
                              uint32_t *out, uint64_t *err) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < P; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t n = pins[j];
    const uint32_t p = part[n];
    if (p >= nparts) report_min(err, kErrPart, n);
    out[j] = p;
  }
}

__global__ void k_check_part(const uint32_t *part, uint32_t N, uint32_t nparts, uint64_t *err) {
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x)
    if (part[n] >= nparts) report_min(err, kErrPart, n);
}

struct PinSeg {   // segment e = all pins of e (inbound = 0) or dst(e) (inbound = 1)
  const uint64_t *off;
  const uint32_t *nsrc;
  int inbound;
  __device__ void operator()(uint64_t e, uint64_t &beg, uint32_t &len) const {
    const uint64_t a = off[e] + (inbound ? nsrc[e] : 0u);
    beg = a;
    len = (uint32_t)(off[e + 1] - a);
  }
};

// warp per edge: number of distinct partitions (runs of the sorted segment)
__global__ void k_run_count(PinSeg seg, uint32_t E, const uint32_t *keys, uint32_t *cnt) {
  const uint32_t lane = lane_id();
  for (uint32_t e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < E; e += (gridDim.x * blockDim.x) >> 5) {
    uint64_t beg;
    uint32_t len;
    seg(e, beg, len);
    uint32_t c = 0;
    for (uint32_t j = lane; j < len; j += 32) c += (j == 0 || keys[beg + j] != keys[beg + j - 1]) ? 1u : 0u;
    c = warp_sum(c);
    if (lane == 0) cnt[e] = c;
  }
}

// warp per edge, chunks of 32 from the back: each run head writes (partition, run length);
// the run's end is the next head (same chunk: the next set ballot bit; else carried from the
// chunk after it), its position counts the heads at or after it.
__global__ void k_run_write(PinSeg seg, uint32_t E, const uint32_t *keys, const uint64_t *off, uint32_t *opart,
                            uint32_t *ocount) {
  const uint32_t lane = lane_id();
  for (uint32_t e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < E; e += (gridDim.x * blockDim.x) >> 5) {
    uint64_t beg;
    uint32_t len;
    seg(e, beg, len);
    if (len == 0) continue;
    uint32_t next = len;          // start of the run after the current chunk
    uint64_t after = off[e + 1];  // output position one past the heads seen so far
    for (int64_t c0 = ((int64_t)(len - 1) / 32) * 32; c0 >= 0; c0 -= 32) {
      const uint32_t j = (uint32_t)c0 + lane;
      const bool in = j < len;
      const uint32_t k = in ? keys[beg + j] : 0u;
      const bool head = in && (j == 0 || k != keys[beg + j - 1]);
      const uint32_t b = __ballot_sync(0xFFFFFFFFu, head);
      if (head) {
        const uint32_t above = b & ~((2u << lane) - 1u);   // heads after this lane in the chunk
        const uint32_t end = above ? (uint32_t)c0 + (__ffs(above) - 1) : next;
        const uint64_t pos = after - __popc(b & ~((1u << lane) - 1u));
        opart[pos] = k;
        ocount[pos] = end - j;
      }
      if (b) next = (uint32_t)c0 + (__ffs(b) - 1);
      after -= __popc(b);
    }
  }
}

static hgp_status pins_impl(hgp_ctx *c, const hgp_csr *g, const uint32_t *part, uint32_t nparts, int inbound,
                            hgp_pins *out) {
  hgp_status st = HGP_OK;
  memset(out, 0, sizeof(*out));
  out->E = g->E;
  const uint64_t P = g->P;
  uint32_t *keys = scratch_raw<uint32_t>(c, P, &st);
  uint32_t *cnt = scratch_raw<uint32_t>(c, g->E, &st);
  if (st) return st;
  out->off = dalloc_n<uint64_t>(c, (size_t)g->E + 1, &st);
  if (st) return st;
  const uint32_t grid = (uint32_t)std::min<uint64_t>(div_up(P ? P : 1, 256), 16u * c->sm_count);
  HGP_TRY(launch(c, "pins_gather", k_gather_part, dim3(grid), dim3(256), 0, (const uint32_t *)g->pins, P, part,
                 nparts, g->N, keys, c->d_err));
  const PinSeg seg{g->edge_off, g->edge_nsrc, inbound};
  HGP_TRY(segmented_sort(c, seg, g->E, keys, g->max_edge));
  const uint32_t ge = (uint32_t)std::min<uint64_t>(div_up((uint64_t)g->E * 32, 256), 16u * c->sm_count);
  HGP_TRY(launch(c, "pins_runs", k_run_count, dim3(ge ? ge : 1), dim3(256), 0, seg, g->E, (const uint32_t *)keys,
                 cnt));
  uint64_t nnz = 0;
  HGP_TRY(scan_exclusive(c, InU32{cnt}, g->E, out->off, &nnz));
  out->nnz = nnz;
  out->part = dalloc_n<uint32_t>(c, nnz, &st);
  out->count = dalloc_n<uint32_t>(c, nnz, &st);
  if (st) return st;
  HGP_TRY(launch(c, "pins_write", k_run_write, dim3(ge ? ge : 1), dim3(256), 0, seg, g->E, (const uint32_t *)keys,
                 (const uint64_t *)out->off, out->part, out->count));
  return HGP_OK;
}

static void pins_release(hgp_ctx *c, hgp_pins *pm) {
  if (!pm) return;
  c->dfree(pm->off, sizeof(uint64_t) * ((size_t)pm->E + 1));
  c->dfree(pm->part, sizeof(uint32_t) * (pm->nnz ? pm->nnz : 1));
  c->dfree(pm->count, sizeof(uint32_t) * (pm->nnz ? pm->nnz : 1));
  memset(pm, 0, sizeof(*pm));
}

// ------------------------------------------------------------------------------ f1: quality
// sizes of the partitions
__global__ void k_part_size(const uint32_t *part, const uint32_t *node_w, uint32_t N, unsigned long long *size) {
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x)
    atomicAdd(size + part[n], (unsigned long long)node_w[n]);
}

// Eq.1: sum omega(e) (lambda(e) - 1); Eq.16: sum of omega(e) over lambda(e) > 1; lambda(e) = the
// number of distinct partitions of e's pins = the length of e's pins row.
__global__ void k_conn(const uint64_t *off, const uint32_t *edge_w, uint32_t E, unsigned long long *acc) {
  uint64_t conn = 0, cut = 0;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    const uint64_t lam = off[e + 1] - off[e];
    conn += (uint64_t)edge_w[e] * (lam - 1);
    cut += lam > 1 ? edge_w[e] : 0u;
  }
  conn = warp_sum(conn);
  cut = warp_sum(cut);
  if (lane_id() == 0) {
    atomicAdd(acc + 0, (unsigned long long)conn);
    atomicAdd(acc + 1, (unsigned long long)cut);
  }
}

// e is inbound to p iff pins_in(p, e) > 0: every entry of e's pins_in row adds mu(e)
__global__ void k_inbound_load(const uint64_t *off, const uint32_t *ipart, const uint32_t *edge_mu, uint32_t E,
                               unsigned long long *inb) {
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x)
    for (uint64_t k = off[e]; k < off[e + 1]; ++k) atomicAdd(inb + ipart[k], (unsigned long long)edge_mu[e]);
}

// acc[2] max size, acc[3] max inbound, acc[4] size violations, acc[5] inbound violations
__global__ void k_quality_reduce(const unsigned long long *size, const unsigned long long *inb, uint32_t nparts,
                                 uint64_t omega, uint64_t delta, unsigned long long *acc) {
  uint64_t ms = 0, mi = 0, vs = 0, vi = 0;
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < nparts; p += gridDim.x * blockDim.x) {
    ms = max(ms, (uint64_t)size[p]);
    mi = max(mi, (uint64_t)inb[p]);
    vs += size[p] > omega;
    vi += (delta != HGP_UNBOUNDED && inb[p] > delta);
  }
  ms = warp_max(ms);
  mi = warp_max(mi);
  vs = warp_sum(vs);
  vi = warp_sum(vi);
  if (lane_id() == 0) {
    atomicMax(acc + 2, (unsigned long long)ms);
    atomicMax(acc + 3, (unsigned long long)mi);
    atomicAdd(acc + 4, (unsigned long long)vs);
    atomicAdd(acc + 5, (unsigned long long)vi);
  }
}

static uint32_t grid_for(hgp_ctx *c, uint64_t n, uint32_t threads = 256) {
  const uint64_t b = (n + threads - 1) / threads;
  return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(b, 16u * c->sm_count));
}

static hgp_status check_errors_part(hgp_ctx *c) {
  uint64_t err[kErrSlots];
  HGP_TRY(fetch_errors(c, err));
  if (err[kErrPart] != UINT64_MAX)
    return set_error(HGP_E_ARG, "node %llu: partition id out of range", (unsigned long long)err[kErrPart]);
  if (err[kErrSeq] != UINT64_MAX)
    return set_error(HGP_E_ARG, "sequence position %llu: entries must be distinct nodes with a destination != "
                     "their partition", (unsigned long long)err[kErrSeq]);
  return HGP_OK;
}

// loads of every partition (device arrays of nparts), from a pins_in matrix
static hgp_status loads_impl(hgp_ctx *c, const hgp_csr *g, const uint32_t *part, uint32_t nparts,
                             const hgp_pins *pin_in, unsigned long long *size, unsigned long long *inb) {
  HGP_CUDA(cudaMemsetAsync(size, 0, sizeof(uint64_t) * (nparts ? nparts : 1), c->stream));
  HGP_CUDA(cudaMemsetAsync(inb, 0, sizeof(uint64_t) * (nparts ? nparts : 1), c->stream));
  HGP_TRY(launch(c, "part_size", k_part_size, dim3(grid_for(c, g->N)), dim3(256), 0, part,
                 (const uint32_t *)g->node_w, g->N, size));
  HGP_TRY(launch(c, "inbound_load", k_inbound_load, dim3(grid_for(c, g->E)), dim3(256), 0,
                 (const uint64_t *)pin_in->off, (const uint32_t *)pin_in->part, (const uint32_t *)g->edge_mu, g->E,
                 inb));
  return HGP_OK;
}

// ------------------------------------------------------------------------------ f3: Eq.13
// Per node n in partition ps: total = sum over I(n) of omega(e); saving = the part of it whose
// pins(ps, e) = 1; conn(p) = sum of omega(e) over e in I(n) with pins(p, e) > 0, p != ps. Then
// loss(n, p) = total - conn(p) and gain(n, p) = saving - total + conn(p): the best p is the max
// (conn(p), p) among the allowed candidates. Sums of omega are < 2^32 (hgp_build_csr rejects
// larger totals), so conn fits a native 32-bit shared atomic.
//
// Pre-pass: per node the bound B(n) = sum over I(n) of |row(e)| on the number of candidate
// entries, which routes the node to the warp tier (a 1024-slot shared table) or the CTA tier
// (a global-memory table of nextpow2(2 B(n)) slots).
constexpr uint32_t kMvLog = 10, kMvSlots = 1u << kMvLog, kMvWarpCap = kMvSlots / 2;
constexpr uint32_t kMvWarps = 4;   // 4 x 8 KB of static shared tables

__global__ void k_move_bound(const hgp_csr g, const uint64_t *poff, uint32_t *bound, uint32_t *small_list,
                             uint32_t *nsmall, uint32_t *big_list, uint32_t *nbig) {
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x; n < g.N; n += gridDim.x * blockDim.x) {
    uint64_t b = 0;
    for (uint64_t k = g.inc_off[n]; k < g.inc_off[n + 1]; ++k) {
      const uint32_t e = g.inc[k];
      b += poff[e + 1] - poff[e];
    }
    const uint32_t bb = b < 0x7FFFFFFFull ? (uint32_t)b : 0x7FFFFFFFu;
    bound[n] = bb;
    if (bb <= kMvWarpCap) small_list[atomicAdd(nsmall, 1u)] = n;
    else big_list[atomicAdd(nbig, 1u)] = n;
  }
}

struct MoveJob {
  hgp_csr g;
  const uint32_t *part;
  const uint64_t *poff;
  const uint32_t *ppart, *pcount;
  const unsigned long long *size;   // [nparts] or nullptr (no size filter)
  uint64_t omega;
  uint32_t *dest;
  int64_t *gain;
};

// The candidate scan shared by both tiers: every entry (p, cnt) of the rows of I(n) goes to
// `add(p, omega(e))` unless p = ps; the lane's (total, saving) partial sums are returned.
template <class Add>
__device__ __forceinline__ void move_traverse(const MoveJob &J, uint32_t n, uint32_t ps, uint32_t tid,
                                              uint32_t nthreads, uint64_t &total, uint64_t &saving, Add add) {
  const uint64_t i0 = J.g.inc_off[n], i1 = J.g.inc_off[n + 1];
  for (uint64_t k = i0; k < i1; ++k) {
    const uint32_t e = J.g.inc[k];
    const uint32_t w = J.g.edge_w[e];
    const uint64_t a = J.poff[e], b = J.poff[e + 1];
    if (tid == 0) total += w;
    for (uint64_t j = a + tid; j < b; j += nthreads) {
      const uint32_t p = J.ppart[j];
      if (p == ps) saving += J.pcount[j] == 1 ? w : 0u;
      else add(p, w);
    }
  }
}

__device__ __forceinline__ bool move_allowed(const MoveJob &J, uint32_t n, uint32_t p) {
  return !J.size || (uint64_t)J.g.node_w[n] + J.size[p] <= J.omega;
}

__device__ __forceinline__ void move_write(const MoveJob &J, uint32_t n, uint64_t best, uint64_t total,
                                           uint64_t saving) {
  if (best == 0) {   // (conn, p) keys are stored + 1 so that 0 means "no candidate"
    J.dest[n] = kNone;
    J.gain[n] = 0;
  } else {
    const uint64_t key = best - 1;
    J.dest[n] = (uint32_t)key;
    J.gain[n] = (int64_t)saving - (int64_t)total + (int64_t)(key >> 32);
  }
}

// warp tier: one warp per node, a private shared table (keys | conn)
__global__ void __launch_bounds__(kMvWarps * 32) k_moves_warp(MoveJob J, const uint32_t *list, const uint32_t *count) {
  __shared__ uint32_t s_key[kMvWarps][kMvSlots];
  __shared__ uint32_t s_val[kMvWarps][kMvSlots];
  const uint32_t lane = lane_id(), w = threadIdx.x >> 5;
  uint32_t *keys = s_key[w], *vals = s_val[w];
  for (uint32_t i = lane; i < kMvSlots; i += 32) { keys[i] = kEmpty; vals[i] = 0; }
  __syncwarp();
  const uint32_t total_nodes = *count;
  for (uint32_t t = blockIdx.x * kMvWarps + w; t < total_nodes; t += gridDim.x * kMvWarps) {
    const uint32_t n = list[t], ps = J.part[n];
    uint64_t total = 0, saving = 0;
    move_traverse(J, n, ps, lane, 32, total, saving, [&](uint32_t p, uint32_t wt) {
      uint32_t s = hash_slot(p, kMvLog);
      while (true) {
        const uint32_t k = keys[s];
        if (k == p) break;
        if (k == kEmpty) {
          const uint32_t o = atomicCAS(keys + s, kEmpty, p);
          if (o == kEmpty || o == p) break;
        }
        s = (s + 1) & (kMvSlots - 1);
      }
      atomicAdd(vals + s, wt);
    });
    __syncwarp();
    total = warp_sum(total);
    saving = warp_sum(saving);
    uint64_t best = 0;
    for (uint32_t i = lane; i < kMvSlots; i += 32) {
      const uint32_t p = keys[i];
      if (p != kEmpty) {
        if (move_allowed(J, n, p)) best = max(best, (((uint64_t)vals[i] << 32) | p) + 1);
        keys[i] = kEmpty;
        vals[i] = 0;
      }
    }
    best = warp_max(best);
    if (lane == 0) move_write(J, n, best, total, saving);
    __syncwarp();
  }
}

// CTA tier: one CTA per node, a global table of tsize(n) = nextpow2(2 B(n)) slots at toff(n)
__global__ void __launch_bounds__(256) k_moves_cta(MoveJob J, const uint32_t *list, const uint32_t *count,
                                                   const uint32_t *bound, const uint64_t *toff, uint32_t *tkeys,
                                                   uint32_t *tvals) {
  __shared__ uint64_t s_red[3][8];
  const uint32_t tid = threadIdx.x, lane = lane_id(), w = tid >> 5;
  const uint32_t total_nodes = *count;
  for (uint32_t t = blockIdx.x; t < total_nodes; t += gridDim.x) {
    const uint32_t n = list[t], ps = J.part[n];
    const uint64_t base = toff[t];
    const uint32_t tsz = (uint32_t)(toff[t + 1] - base);
    uint32_t *keys = tkeys + base, *vals = tvals + base;
    for (uint32_t i = tid; i < tsz; i += blockDim.x) { keys[i] = kEmpty; vals[i] = 0; }
    __syncthreads();
    const uint32_t lg = 31 - __clz(tsz);
    uint64_t total = 0, saving = 0;
    move_traverse(J, n, ps, tid, blockDim.x, total, saving, [&](uint32_t p, uint32_t wt) {
      uint32_t s = hash_slot(p, lg);
      while (true) {
        const uint32_t k = keys[s];
        if (k == p) break;
        if (k == kEmpty) {
          const uint32_t o = atomicCAS(keys + s, kEmpty, p);
          if (o == kEmpty || o == p) break;
        }
        s = (s + 1) & (tsz - 1);
      }
      atomicAdd(vals + s, wt);
    });
    __syncthreads();
    uint64_t best = 0;
    for (uint32_t i = tid; i < tsz; i += blockDim.x) {
      const uint32_t p = keys[i];
      if (p != kEmpty && move_allowed(J, n, p)) best = max(best, (((uint64_t)vals[i] << 32) | p) + 1);
    }
    total = warp_sum(total);
    saving = warp_sum(saving);
    best = warp_max(best);
    if (lane == 0) { s_red[0][w] = total; s_red[1][w] = saving; s_red[2][w] = best; }
    __syncthreads();
    if (tid == 0) {
      uint64_t a = 0, b = 0, m = 0;
      for (uint32_t q = 0; q < blockDim.x / 32; ++q) { a += s_red[0][q]; b += s_red[1][q]; m = max(m, s_red[2][q]); }
      move_write(J, n, m, a, b);
    }
    __syncthreads();
  }
}

struct TableSize {   // nextpow2(2 B) slots, at least 64
  const uint32_t *list, *bound;
  __device__ uint64_t operator()(uint64_t i) const {
    const uint64_t want = 2ull * bound[list[i]];
    uint64_t s = 64;
    while (s < want) s <<= 1;
    return s;
  }
};

static hgp_status moves_impl(hgp_ctx *c, const hgp_csr *g, const uint32_t *part, uint32_t nparts,
                             const hgp_pins *pm, uint64_t omega, int enforce_size, uint32_t *dest, int64_t *gain) {
  hgp_status st = HGP_OK;
  const uint32_t N = g->N;
  unsigned long long *size = nullptr;
  if (enforce_size) {
    size = scratch_zero<unsigned long long>(c, nparts, &st);
    if (st) return st;
    HGP_TRY(launch(c, "part_size", k_part_size, dim3(grid_for(c, N)), dim3(256), 0, part,
                   (const uint32_t *)g->node_w, N, size));
  }
  uint32_t *bound = scratch_raw<uint32_t>(c, N, &st);
  uint32_t *lists = scratch_raw<uint32_t>(c, 2 * (size_t)N, &st);
  uint32_t *cnts = scratch_zero<uint32_t>(c, 2, &st);
  if (st) return st;
  HGP_TRY(launch(c, "move_bound", k_move_bound, dim3(grid_for(c, N)), dim3(256), 0, *g, (const uint64_t *)pm->off,
                 bound, lists, cnts, lists + N, cnts + 1));
  uint32_t h[2];
  HGP_TRY(read_back(c, cnts, sizeof(h), h));
  const MoveJob J{*g, part, pm->off, pm->part, pm->count, size, omega, dest, gain};
  if (h[0]) {
    const uint32_t gw = std::min<uint32_t>(div_up(h[0], kMvWarps), 8u * c->sm_count);
    HGP_TRY(launch(c, "moves_warp", k_moves_warp, dim3(gw), dim3(kMvWarps * 32), 0, J, (const uint32_t *)lists,
                   (const uint32_t *)cnts));
  }
  if (h[1]) {
    uint64_t *toff = scratch_raw<uint64_t>(c, (size_t)h[1] + 1, &st);
    if (st) return st;
    uint64_t tot = 0;
    HGP_TRY(scan_exclusive(c, TableSize{lists + N, bound}, h[1], toff, &tot));
    uint32_t *tk = scratch_raw<uint32_t>(c, tot, &st), *tv = scratch_raw<uint32_t>(c, tot, &st);
    if (st) return st;
    HGP_TRY(launch(c, "moves_cta", k_moves_cta, dim3(std::min<uint32_t>(h[1], 4u * c->sm_count)), dim3(256), 0, J,
                   (const uint32_t *)(lists + N), (const uint32_t *)(cnts + 1), (const uint32_t *)bound,
                   (const uint64_t *)toff, tk, tv));
  }
  return HGP_OK;
}

// ------------------------------------------------------------------------------ sequences
// pos[n] = index of n in seq (NONE if absent); validates the entries (kErrSeq = lowest position).
__global__ void k_seq_pos(const uint32_t *seq, uint32_t M, uint32_t N, const uint32_t *part, const uint32_t *dest,
                          uint32_t nparts, uint32_t *pos, uint64_t *err) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < M; i += gridDim.x * blockDim.x) {
    const uint32_t n = seq[i];
    if (n >= N) { report_min(err, kErrSeq, i); continue; }
    const uint32_t d = dest[n];
    if (d >= nparts || d == part[n]) report_min(err, kErrSeq, i);
    const uint32_t o = atomicMin(pos + n, i);
    if (o != kNone) report_min(err, kErrSeq, max(o, i));   // duplicate: the later position
  }
}

// Binary search of partition p in e's row of a pins matrix: its count, 0 if absent.
__device__ __forceinline__ uint32_t pins_of(const uint64_t *off, const uint32_t *pp, const uint32_t *pc, uint32_t e,
                                            uint32_t p) {
  uint64_t lo = off[e], hi = off[e + 1];
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    const uint32_t x = pp[mid];
    if (x == p) return pc[mid];
    if (x < p) lo = mid + 1; else hi = mid;
  }
  return 0;
}

// In-sequence gain (Eqs.14-15) of move i: n moves ps -> pd after moves 0..i-1. For e in I(n) the
// counts at that moment are pins(ps, e) + #{earlier m in e entering ps} - #{earlier m leaving ps}
// and the same for pd; e stops being cut in ps iff that count is 1 (n is the last one there)
// and starts being cut in pd iff it is 0: gain += omega(e) ([c_ps = 1] - [c_pd = 0]). This is
// the paper's two cases written on the counts they test, equal to Eq.1 before minus after.
// Warp per move; 32 incident edges at a time, their pins as one flat sequence over the lanes,
// earlier movers (rare) counted into per-edge shared counters.
constexpr uint32_t kSgWarps = 8;
__global__ void __launch_bounds__(kSgWarps * 32) k_seq_gains(hgp_csr g, const uint32_t *part, const uint32_t *dest,
                                                            const uint32_t *seq, uint32_t M, const uint32_t *pos,
                                                            const uint64_t *poff, const uint32_t *ppart,
                                                            const uint32_t *pcount, int64_t *gain_seq) {
  __shared__ uint64_t s_a[kSgWarps][32];       // edge's first pin
  __shared__ uint32_t s_end[kSgWarps][32];     // inclusive scan of the edge sizes
  __shared__ int s_dps[kSgWarps][32], s_dpd[kSgWarps][32];
  const uint32_t lane = lane_id(), w = threadIdx.x >> 5;
  for (uint32_t i = blockIdx.x * kSgWarps + w; i < M; i += gridDim.x * kSgWarps) {
    const uint32_t n = seq[i], ps = part[n], pd = dest[n];
    const uint64_t i0 = g.inc_off[n], i1 = g.inc_off[n + 1];
    int64_t acc = 0;
    for (uint64_t t0 = i0; t0 < i1; t0 += 32) {
      const bool mine = t0 + lane < i1;
      uint32_t e = 0, len = 0;
      if (mine) {
        e = g.inc[t0 + lane];
        s_a[w][lane] = g.edge_off[e];
        len = (uint32_t)(g.edge_off[e + 1] - g.edge_off[e]);
      }
      const uint32_t incl = warp_incl_scan(len);
      s_end[w][lane] = incl;
      s_dps[w][lane] = 0;
      s_dpd[w][lane] = 0;
      const uint32_t tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
      __syncwarp();
      uint32_t k = 0;   // current edge of this lane (flat positions ascend per lane)
      for (uint32_t f = lane; f < tot; f += 32) {
        while (s_end[w][k] <= f) ++k;
        const uint32_t start = k ? s_end[w][k - 1] : 0u;
        const uint32_t m = g.pins[s_a[w][k] + (f - start)];
        const uint32_t q = pos[m];
        if (q < i) {   // m moved earlier: part[m] -> dest[m]
          const uint32_t sp = part[m], dp = dest[m];
          const int dps = (dp == ps) - (sp == ps), dpd = (dp == pd) - (sp == pd);
          if (dps) atomicAdd(&s_dps[w][k], dps);
          if (dpd) atomicAdd(&s_dpd[w][k], dpd);
        }
      }
      __syncwarp();
      if (mine) {
        const int64_t cps = (int64_t)pins_of(poff, ppart, pcount, e, ps) + s_dps[w][lane];
        const int64_t cpd = (int64_t)pins_of(poff, ppart, pcount, e, pd) + s_dpd[w][lane];
        acc += (int64_t)g.edge_w[e] * ((cps == 1 ? 1 : 0) - (cpd == 0 ? 1 : 0));
      }
      __syncwarp();
    }
    acc = warp_sum(acc);
    if (lane == 0) gain_seq[i] = acc;
  }
}

static hgp_status seq_setup(hgp_ctx *c, const hgp_csr *g, const uint32_t *part, uint32_t nparts, const uint32_t *seq,
                            uint32_t M, const uint32_t *dest, uint32_t **pos_out) {
  hgp_status st = HGP_OK;
  uint32_t *pos = scratch_raw<uint32_t>(c, g->N, &st);
  if (st) return st;
  HGP_CUDA(cudaMemsetAsync(pos, 0xFF, sizeof(uint32_t) * (g->N ? g->N : 1), c->stream));
  HGP_TRY(launch(c, "check_part", k_check_part, dim3(grid_for(c, g->N)), dim3(256), 0, part, g->N, nparts,
                 c->d_err));
  if (M) HGP_TRY(launch(c, "seq_pos", k_seq_pos, dim3(grid_for(c, M)), dim3(256), 0, seq, M, g->N, part, dest, nparts,
                        pos, c->d_err));
  *pos_out = pos;
  return HGP_OK;
}

// ------------------------------------------------------------------------------ f4: events
// Size events: move i emits (ps, i, -size(n)) and (pd, i, +size(n)).
// Inbound events: for every e in in(n), (ps, e, i, -1) and (pd, e, i, +1).
__global__ void k_inb_count(const uint32_t *seq, uint32_t M, const uint32_t *inc_nin, uint32_t *cnt) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < M; i += gridDim.x * blockDim.x)
    cnt[i] = inc_nin[seq[i]];
}

// event k of the inbound stream: 2 per (move, in-edge) in move order; key_e, key_p and the move
__global__ void k_inb_events(hgp_csr g, const uint32_t *seq, uint32_t M, const uint64_t *eoff,
                             const uint32_t *part, const uint32_t *dest, uint32_t *key_e, uint32_t *ev_move,
                             uint32_t *ev_p) {
  const uint32_t lane = lane_id();
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < M; i += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t n = seq[i];
    const uint64_t o = eoff[i];
    const uint64_t k0 = g.inc_off[n];
    const uint32_t nin = g.inc_nin[n];
    for (uint32_t j = lane; j < nin; j += 32) {
      const uint32_t e = g.inc[k0 + j];
      const uint64_t k = 2 * (o + j);
      key_e[k] = e; key_e[k + 1] = e;
      ev_move[k] = i; ev_move[k + 1] = i;
      ev_p[k] = part[n]; ev_p[k + 1] = dest[n];   // even: leave ps (-1), odd: enter pd (+1)
    }
  }
}

__global__ void k_ev_iota(uint32_t *v, uint64_t n) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x)
    v[j] = (uint32_t)j;
}

__global__ void k_gather_u32(const uint32_t *src, const uint32_t *idx, uint64_t n, uint32_t *dst) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x)
    dst[j] = src[idx[j]];
}

// After sorting by (p, e, i): segment heads of (p, e) and the +-1 deltas (two's complement).
struct InbHead {
  const uint32_t *ord, *ev_p, *key_e;
  __device__ uint64_t operator()(uint64_t j) const {
    if (j == 0) return 1;
    const uint32_t a = ord[j], b = ord[j - 1];
    return (ev_p[a] != ev_p[b] || key_e[a] != key_e[b]) ? 1u : 0u;
  }
};
struct InbDelta {
  const uint32_t *ord;
  __device__ uint64_t operator()(uint64_t j) const { return (ord[j] & 1u) ? 1ull : ~0ull; }
};

// segment base: the exclusive delta-sum at every head, indexed by segment id
__global__ void k_seg_base(const uint64_t *head_x, const uint64_t *delta_x, uint64_t n, InbHead hd,
                           uint64_t *base) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x)
    if (hd(j)) base[head_x[j]] = delta_x[j];
}

// running pins_in(p, e) before / after each event; a 0 -> 1 transition makes e inbound to p
// (+mu(e)), 1 -> 0 stops it (-mu(e)): flag[j] marks a transition event.
__global__ void k_inb_transitions(const uint32_t *ord, const uint32_t *ev_p, const uint32_t *key_e, uint64_t n,
                                  const uint64_t *head_x, const uint64_t *delta_x, const uint64_t *base,
                                  InbHead hd, const uint64_t *ioff, const uint32_t *ipart, const uint32_t *icount,
                                  uint32_t *flag) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t k = ord[j], p = ev_p[k], e = key_e[k];
    const uint64_t seg = head_x[j] + hd(j) - 1;          // segment id of j
    const int64_t before = (int64_t)pins_of(ioff, ipart, icount, e, p) + (int64_t)(delta_x[j] - base[seg]);
    const int64_t after = before + ((k & 1u) ? 1 : -1);
    flag[j] = (before == 0 && after == 1) || (before == 1 && after == 0) ? 1u : 0u;
  }
}

// Combined events keyed by (p, move): size events first (2M), then the transitions.
//   ev2_p, ev2_i, dsz (two's complement), dinb (two's complement)
__global__ void k_size_events(const uint32_t *seq, uint32_t M, const uint32_t *part, const uint32_t *dest,
                              const uint32_t *node_w, uint32_t *ev2_p, uint32_t *ev2_i, uint64_t *dsz,
                              uint64_t *dinb) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < M; i += gridDim.x * blockDim.x) {
    const uint32_t n = seq[i];
    const uint64_t w = node_w[n];
    ev2_p[2 * i] = part[n]; ev2_i[2 * i] = i; dsz[2 * i] = (uint64_t)(-(int64_t)w); dinb[2 * i] = 0;
    ev2_p[2 * i + 1] = dest[n]; ev2_i[2 * i + 1] = i; dsz[2 * i + 1] = w; dinb[2 * i + 1] = 0;
  }
}

__global__ void k_trans_events(const uint32_t *ord, const uint32_t *ev_p, const uint32_t *key_e,
                               const uint32_t *ev_move, const uint32_t *flag, const uint64_t *tpos, uint64_t n,
                               const uint32_t *edge_mu, uint64_t off0, uint32_t *ev2_p, uint32_t *ev2_i,
                               uint64_t *dsz, uint64_t *dinb) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
    if (!flag[j]) continue;
    const uint32_t k = ord[j];
    const uint64_t o = off0 + tpos[j];
    const uint64_t mu = edge_mu[key_e[k]];
    ev2_p[o] = ev_p[k];
    ev2_i[o] = ev_move[k];
    dsz[o] = 0;
    dinb[o] = (k & 1u) ? mu : (uint64_t)(-(int64_t)mu);
  }
}

struct PHead {   // heads of p-segments of the (p, i)-sorted combined events
  const uint32_t *ord, *ev2_p;
  __device__ uint64_t operator()(uint64_t j) const { return j == 0 || ev2_p[ord[j]] != ev2_p[ord[j - 1]]; }
};
struct GatherU64 {
  const uint32_t *ord;
  const uint64_t *a;
  __device__ uint64_t operator()(uint64_t j) const { return a[ord[j]]; }
};

// Per event: the partition's state before and after it (initial load + segmented prefix);
// bad = size > Omega or inbound > Delta; the change of bad is charged to the event's move. Within
// a (p, move) group the changes telescope to the move's net effect on p.
__global__ void k_violation_delta(const uint32_t *ord, const uint32_t *ev2_p, const uint32_t *ev2_i,
                                  const uint64_t *dsz, const uint64_t *dinb, uint64_t n, const uint64_t *sx,
                                  const uint64_t *ix, const uint64_t *hx, PHead hd, const uint64_t *seg_head_pos,
                                  const unsigned long long *size0, const unsigned long long *inb0, uint64_t omega,
                                  uint64_t delta, int *vdelta) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t k = ord[j], p = ev2_p[k];
    const uint64_t seg = hx[j] + hd(j) - 1;
    const uint64_t h = seg_head_pos[seg];
    const uint64_t s_before = size0[p] + (sx[j] - sx[h]);
    const uint64_t i_before = inb0[p] + (ix[j] - ix[h]);
    const uint64_t s_after = s_before + dsz[k], i_after = i_before + dinb[k];
    const bool b0 = s_before > omega || (delta != HGP_UNBOUNDED && i_before > delta);
    const bool b1 = s_after > omega || (delta != HGP_UNBOUNDED && i_after > delta);
    if (b0 != b1) atomicAdd(vdelta + ev2_i[k], b1 ? 1 : -1);
  }
}

__global__ void k_head_pos(const uint64_t *hx, uint64_t n, PHead hd, uint64_t *seg_head_pos) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x)
    if (hd(j)) seg_head_pos[hx[j]] = j;
}

__global__ void k_bad0(const unsigned long long *size0, const unsigned long long *inb0, uint32_t nparts,
                       uint64_t omega, uint64_t delta, unsigned long long *cnt) {
  uint64_t v = 0;
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < nparts; p += gridDim.x * blockDim.x)
    v += size0[p] > omega || (delta != HGP_UNBOUNDED && inb0[p] > delta);
  v = warp_sum(v);
  if (lane_id() == 0 && v) atomicAdd(cnt, (unsigned long long)v);
}

struct InI32 {
  const int *a;
  __device__ uint64_t operator()(uint64_t i) const { return (uint64_t)(int64_t)a[i]; }
};

__global__ void k_violations_out(const uint64_t *vx, const int *vdelta, uint32_t M, const unsigned long long *bad0,
                                 uint32_t *violations) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < M; i += gridDim.x * blockDim.x)
    violations[i] = (uint32_t)(*bad0 + vx[i] + (uint64_t)(int64_t)vdelta[i]);
}

static uint32_t bits_for(uint64_t x) {   // bits needed for keys in [0, x)
  uint32_t b = 1;
  while (b < 32 && (1ull << b) < x) ++b;
  return b;
}

static hgp_status violations_impl(hgp_ctx *c, const hgp_csr *g, const uint32_t *part, uint32_t nparts,
                                  const hgp_pins *pin_in, const uint32_t *seq, uint32_t M, const uint32_t *dest,
                                  uint64_t omega, uint64_t delta, uint32_t *violations) {
  hgp_status st = HGP_OK;
  // initial loads and the number of partitions violating a constraint before any move
  unsigned long long *size0 = scratch_raw<unsigned long long>(c, nparts, &st);
  unsigned long long *inb0 = scratch_raw<unsigned long long>(c, nparts, &st);
  unsigned long long *bad0 = scratch_zero<unsigned long long>(c, 1, &st);
  if (st) return st;
  HGP_TRY(loads_impl(c, g, part, nparts, pin_in, size0, inb0));
  HGP_TRY(launch(c, "bad0", k_bad0, dim3(grid_for(c, nparts)), dim3(256), 0, (const unsigned long long *)size0,
                 (const unsigned long long *)inb0, nparts, omega, delta, bad0));
  if (M == 0) return HGP_OK;
  // inbound events in move order, then stably by e, then by p: (p, e, n_seq)
  uint32_t *cnt = scratch_raw<uint32_t>(c, M, &st);
  uint64_t *eoff = scratch_raw<uint64_t>(c, (size_t)M + 1, &st);
  if (st) return st;
  HGP_TRY(launch(c, "inb_count", k_inb_count, dim3(grid_for(c, M)), dim3(256), 0, seq, M,
                 (const uint32_t *)g->inc_nin, cnt));
  uint64_t Q = 0;
  HGP_TRY(scan_exclusive(c, InU32{cnt}, M, eoff, &Q));
  const uint64_t NI = 2 * Q;
  if (NI >= (1ull << 30)) return set_error(HGP_E_OVERFLOW, "sequence validation: more than 2^29 inbound events");
  uint32_t *key_e = scratch_raw<uint32_t>(c, NI, &st), *ev_move = scratch_raw<uint32_t>(c, NI, &st);
  uint32_t *ev_p = scratch_raw<uint32_t>(c, NI, &st), *k1 = scratch_raw<uint32_t>(c, NI, &st);
  uint32_t *v0 = scratch_raw<uint32_t>(c, NI, &st), *v1 = scratch_raw<uint32_t>(c, NI, &st);
  uint32_t *kp = scratch_raw<uint32_t>(c, NI, &st);
  if (st) return st;
  uint32_t *ord = v0;
  uint64_t T = 0;
  uint64_t *tpos = nullptr;
  uint32_t *tflag = nullptr;
  if (NI) {
    HGP_TRY(launch(c, "inb_events", k_inb_events, dim3(grid_for(c, (uint64_t)M * 32)), dim3(256), 0, *g, seq, M,
                   (const uint64_t *)eoff, part, dest, key_e, ev_move, ev_p));
    // sort event indices by e (keys copied: key_e stays indexed by event)
    HGP_CUDA(cudaMemcpyAsync(kp, key_e, sizeof(uint32_t) * NI, cudaMemcpyDeviceToDevice, c->stream));
    HGP_TRY(launch(c, "ev_iota", k_ev_iota, dim3(grid_for(c, NI)), dim3(256), 0, v0, NI));
    uint32_t *ks = nullptr, *vs = nullptr;
    HGP_TRY(radix_sort_pairs(c, kp, v0, k1, v1, NI, bits_for(g->E), &ks, &vs));
    uint32_t *kalt = ks == kp ? k1 : kp, *valt = vs == v0 ? v1 : v0;
    HGP_TRY(launch(c, "gather_u32", k_gather_u32, dim3(grid_for(c, NI)), dim3(256), 0, (const uint32_t *)ev_p,
                   (const uint32_t *)vs, NI, ks));
    uint32_t *ks2 = nullptr, *vs2 = nullptr;
    HGP_TRY(radix_sort_pairs(c, ks, vs, kalt, valt, NI, bits_for(nparts), &ks2, &vs2));
    ord = vs2;
    // segmented prefix over (p, e): global scans of heads and deltas + per-segment base
    uint64_t *hx = scratch_raw<uint64_t>(c, NI + 1, &st), *dx = scratch_raw<uint64_t>(c, NI + 1, &st);
    if (st) return st;
    const InbHead hd{ord, ev_p, key_e};
    uint64_t nseg = 0;
    HGP_TRY(scan_exclusive(c, hd, NI, hx, &nseg));
    HGP_TRY(scan_exclusive(c, InbDelta{ord}, NI, dx, nullptr));
    uint64_t *base = scratch_raw<uint64_t>(c, nseg, &st);
    tflag = scratch_raw<uint32_t>(c, NI, &st);
    tpos = scratch_raw<uint64_t>(c, NI + 1, &st);
    if (st) return st;
    HGP_TRY(launch(c, "seg_base", k_seg_base, dim3(grid_for(c, NI)), dim3(256), 0, (const uint64_t *)hx,
                   (const uint64_t *)dx, NI, hd, base));
    HGP_TRY(launch(c, "inb_transitions", k_inb_transitions, dim3(grid_for(c, NI)), dim3(256), 0,
                   (const uint32_t *)ord, (const uint32_t *)ev_p, (const uint32_t *)key_e, NI, (const uint64_t *)hx,
                   (const uint64_t *)dx, (const uint64_t *)base, hd, (const uint64_t *)pin_in->off,
                   (const uint32_t *)pin_in->part, (const uint32_t *)pin_in->count, tflag));
    HGP_TRY(scan_exclusive(c, InU32{tflag}, NI, tpos, &T));
  }
  // combined (p, move) events: 2M size events + T inbound transitions; stable by move, then by p
  const uint64_t NE = 2ull * M + T;
  if (NE >= (1ull << 30)) return set_error(HGP_E_OVERFLOW, "sequence validation: more than 2^30 events");
  uint32_t *e2p = scratch_raw<uint32_t>(c, NE, &st), *e2i = scratch_raw<uint32_t>(c, NE, &st);
  uint64_t *dsz = scratch_raw<uint64_t>(c, NE, &st), *dinb = scratch_raw<uint64_t>(c, NE, &st);
  uint32_t *ka = scratch_raw<uint32_t>(c, NE, &st), *kb = scratch_raw<uint32_t>(c, NE, &st);
  uint32_t *va = scratch_raw<uint32_t>(c, NE, &st), *vb = scratch_raw<uint32_t>(c, NE, &st);
  int *vdelta = scratch_zero<int>(c, M, &st);
  if (st) return st;
  HGP_TRY(launch(c, "size_events", k_size_events, dim3(grid_for(c, M)), dim3(256), 0, seq, M, part, dest,
                 (const uint32_t *)g->node_w, e2p, e2i, dsz, dinb));
  if (T)
    HGP_TRY(launch(c, "trans_events", k_trans_events, dim3(grid_for(c, NI)), dim3(256), 0, (const uint32_t *)ord,
                   (const uint32_t *)ev_p, (const uint32_t *)key_e, (const uint32_t *)ev_move,
                   (const uint32_t *)tflag, (const uint64_t *)tpos, NI, (const uint32_t *)g->edge_mu, 2ull * M, e2p,
                   e2i, dsz, dinb));
  HGP_CUDA(cudaMemcpyAsync(ka, e2i, sizeof(uint32_t) * NE, cudaMemcpyDeviceToDevice, c->stream));
  HGP_TRY(launch(c, "ev_iota", k_ev_iota, dim3(grid_for(c, NE)), dim3(256), 0, va, NE));
  uint32_t *ks = nullptr, *vs = nullptr;
  HGP_TRY(radix_sort_pairs(c, ka, va, kb, vb, NE, bits_for(M), &ks, &vs));
  uint32_t *kalt = ks == ka ? kb : ka, *valt = vs == va ? vb : va;
  HGP_TRY(launch(c, "gather_u32", k_gather_u32, dim3(grid_for(c, NE)), dim3(256), 0, (const uint32_t *)e2p,
                 (const uint32_t *)vs, NE, ks));
  uint32_t *ks2 = nullptr, *ord2 = nullptr;
  HGP_TRY(radix_sort_pairs(c, ks, vs, kalt, valt, NE, bits_for(nparts), &ks2, &ord2));
  // segmented prefix sums per p of the size and inbound deltas
  uint64_t *sx = scratch_raw<uint64_t>(c, NE + 1, &st), *ix = scratch_raw<uint64_t>(c, NE + 1, &st);
  uint64_t *hx = scratch_raw<uint64_t>(c, NE + 1, &st);
  if (st) return st;
  const PHead ph{ord2, e2p};
  uint64_t np = 0;
  HGP_TRY(scan_exclusive(c, GatherU64{ord2, dsz}, NE, sx, nullptr));
  HGP_TRY(scan_exclusive(c, GatherU64{ord2, dinb}, NE, ix, nullptr));
  HGP_TRY(scan_exclusive(c, ph, NE, hx, &np));
  uint64_t *hpos = scratch_raw<uint64_t>(c, np, &st);
  if (st) return st;
  HGP_TRY(launch(c, "head_pos", k_head_pos, dim3(grid_for(c, NE)), dim3(256), 0, (const uint64_t *)hx, NE, ph, hpos));
  HGP_TRY(launch(c, "violation_delta", k_violation_delta, dim3(grid_for(c, NE)), dim3(256), 0,
                 (const uint32_t *)ord2, (const uint32_t *)e2p, (const uint32_t *)e2i, (const uint64_t *)dsz,
                 (const uint64_t *)dinb, NE, (const uint64_t *)sx, (const uint64_t *)ix, (const uint64_t *)hx, ph,
                 (const uint64_t *)hpos, (const unsigned long long *)size0, (const unsigned long long *)inb0, omega,
                 delta, vdelta));
  // the count of active violations after each move: initial count + prefix of the changes
  uint64_t *vx = scratch_raw<uint64_t>(c, (size_t)M + 1, &st);
  if (st) return st;
  HGP_TRY(scan_exclusive(c, InI32{vdelta}, M, vx, nullptr));
  HGP_TRY(launch(c, "violations_out", k_violations_out, dim3(grid_for(c, M)), dim3(256), 0, (const uint64_t *)vx,
                 (const int *)vdelta, M, (const unsigned long long *)bad0, violations));
  return HGP_OK;
}

// ------------------------------------------------------------------------------ landing point
struct InI64 {
  const int64_t *a;
  __device__ uint64_t operator()(uint64_t i) const { return (uint64_t)a[i]; }
};

// max over k with violations[k-1] = 0 of (cumulative gain, -k): packed as the signed gain in the
// high bits of an ordered u128 emulated by two passes: max gain, then min k holding it.
__global__ void k_prefix_max(const uint64_t *cx, const int64_t *gs, const uint32_t *vio, uint32_t M,
                             unsigned long long *best) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < M; i += gridDim.x * blockDim.x) {
    const int64_t cum = (int64_t)(cx[i] + (uint64_t)gs[i]);
    if (vio[i] == 0 && cum > 0) atomicMax(best, (unsigned long long)cum);
  }
}
__global__ void k_prefix_first(const uint64_t *cx, const int64_t *gs, const uint32_t *vio, uint32_t M,
                               const unsigned long long *best, unsigned int *k) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < M; i += gridDim.x * blockDim.x) {
    const int64_t cum = (int64_t)(cx[i] + (uint64_t)gs[i]);
    if (vio[i] == 0 && cum > 0 && (unsigned long long)cum == *best) atomicMin(k, i + 1);
  }
}

}  // namespace hgp

using namespace hgp;

extern "C" {

hgp_status hgp_pins_matrix(hgp_ctx *c, const hgp_csr *g, const uint32_t *part, uint32_t nparts, int inbound,
                           hgp_pins *out) {
  if (!c || !g || !out || (g->N && !part)) return set_error(HGP_E_ARG, "hgp_pins_matrix: null argument");
  ApiScope scope(c);
  HGP_TRY(clear_errors(c));
  hgp_status s = pins_impl(c, g, part, nparts, inbound, out);
  if (s == HGP_OK) s = check_errors_part(c);
  if (s != HGP_OK) pins_release(c, out);
  return s;
}

void hgp_pins_free(hgp_ctx *c, hgp_pins *pm) {
  if (!c || !pm) return;
  DeviceGuard dg(c->device);
  pins_release(c, pm);
}

hgp_status hgp_partition_metrics(hgp_ctx *c, const hgp_csr *g, const uint32_t *part, uint32_t nparts,
                                 uint64_t omega, uint64_t delta, hgp_quality *out, uint64_t *part_size,
                                 uint64_t *part_inbound) {
  if (!c || !g || !out || (g->N && !part)) return set_error(HGP_E_ARG, "hgp_partition_metrics: null argument");
  if (nparts == 0 && g->N) return set_error(HGP_E_ARG, "nparts must be >= 1");
  ApiScope scope(c);
  HGP_TRY(clear_errors(c));
  hgp_pins pf{}, pi{};
  hgp_status s = pins_impl(c, g, part, nparts, 0, &pf);
  if (s == HGP_OK) s = pins_impl(c, g, part, nparts, 1, &pi);
  if (s == HGP_OK) s = check_errors_part(c);
  hgp_status st = HGP_OK;
  unsigned long long *acc = s == HGP_OK ? scratch_zero<unsigned long long>(c, 6, &st) : nullptr;
  unsigned long long *size = s == HGP_OK && st == HGP_OK
                                 ? (part_size ? reinterpret_cast<unsigned long long *>(part_size)
                                              : scratch_raw<unsigned long long>(c, nparts, &st))
                                 : nullptr;
  unsigned long long *inb = s == HGP_OK && st == HGP_OK
                                ? (part_inbound ? reinterpret_cast<unsigned long long *>(part_inbound)
                                                : scratch_raw<unsigned long long>(c, nparts, &st))
                                : nullptr;
  if (s == HGP_OK) s = st;
  if (s == HGP_OK) s = loads_impl(c, g, part, nparts, &pi, size, inb);
  if (s == HGP_OK)
    s = launch(c, "conn", k_conn, dim3(grid_for(c, g->E)), dim3(256), 0, (const uint64_t *)pf.off,
               (const uint32_t *)g->edge_w, g->E, acc);
  if (s == HGP_OK)
    s = launch(c, "quality_reduce", k_quality_reduce, dim3(grid_for(c, nparts)), dim3(256), 0,
               (const unsigned long long *)size, (const unsigned long long *)inb, nparts, omega, delta, acc);
  uint64_t h[6] = {0, 0, 0, 0, 0, 0};
  if (s == HGP_OK) s = read_back(c, acc, sizeof(h), h);
  pins_release(c, &pf);
  pins_release(c, &pi);
  if (s != HGP_OK) return s;
  out->connectivity = h[0];
  out->cut_net = h[1];
  out->max_size = h[2];
  out->max_inbound = h[3];
  out->size_violations = (uint32_t)h[4];
  out->inbound_violations = (uint32_t)h[5];
  return HGP_OK;
}

hgp_status hgp_propose_moves(hgp_ctx *c, const hgp_csr *g, const uint32_t *part, uint32_t nparts, const hgp_pins *pins,
                             uint64_t omega, int enforce_size, uint32_t *dest, int64_t *gain) {
  if (!c || !g || (g->N && (!part || !dest || !gain))) return set_error(HGP_E_ARG, "hgp_propose_moves: null argument");
  if (pins && pins->E != g->E) return set_error(HGP_E_ARG, "pins matrix of another level");
  ApiScope scope(c);
  HGP_TRY(clear_errors(c));
  hgp_pins own{};
  hgp_status s = HGP_OK;
  if (!pins) {
    s = pins_impl(c, g, part, nparts, 0, &own);
    pins = &own;
  } else {
    s = launch(c, "check_part", k_check_part, dim3(grid_for(c, g->N)), dim3(256), 0, part, g->N, nparts, c->d_err);
  }
  if (s == HGP_OK) s = check_errors_part(c);
  if (s == HGP_OK && g->N) s = moves_impl(c, g, part, nparts, pins, omega, enforce_size, dest, gain);
  if (s == HGP_OK) s = hgp_sync(c);
  pins_release(c, &own);
  return s;
}

hgp_status hgp_in_sequence_gains(hgp_ctx *c, const hgp_csr *g, const uint32_t *part, uint32_t nparts,
                                 const hgp_pins *pins, const uint32_t *seq, uint32_t M, const uint32_t *dest,
                                 int64_t *gain_seq) {
  if (!c || !g || (g->N && !part) || (M && (!seq || !dest || !gain_seq)))
    return set_error(HGP_E_ARG, "hgp_in_sequence_gains: null argument");
  if (pins && pins->E != g->E) return set_error(HGP_E_ARG, "pins matrix of another level");
  ApiScope scope(c);
  HGP_TRY(clear_errors(c));
  uint32_t *pos = nullptr;
  hgp_pins own{};
  hgp_status s = seq_setup(c, g, part, nparts, seq, M, dest, &pos);
  if (s == HGP_OK) s = check_errors_part(c);
  if (s == HGP_OK && !pins) {
    s = pins_impl(c, g, part, nparts, 0, &own);
    pins = &own;
  }
  if (s == HGP_OK && M)
    s = launch(c, "seq_gains", k_seq_gains, dim3(std::min<uint32_t>(div_up(M, kSgWarps), 16u * c->sm_count)),
               dim3(kSgWarps * 32), 0, *g, part, dest, seq, M, (const uint32_t *)pos, (const uint64_t *)pins->off,
               (const uint32_t *)pins->part, (const uint32_t *)pins->count, gain_seq);
  if (s == HGP_OK) s = hgp_sync(c);
  pins_release(c, &own);
  return s;
}

hgp_status hgp_sequence_violations(hgp_ctx *c, const hgp_csr *g, const uint32_t *part, uint32_t nparts,
                                   const hgp_pins *pins_in, const uint32_t *seq, uint32_t M, const uint32_t *dest,
                                   uint64_t omega, uint64_t delta, uint32_t *violations) {
  if (!c || !g || (g->N && !part) || (M && (!seq || !dest || !violations)))
    return set_error(HGP_E_ARG, "hgp_sequence_violations: null argument");
  if (nparts == 0 && g->N) return set_error(HGP_E_ARG, "nparts must be >= 1");
  if (pins_in && pins_in->E != g->E) return set_error(HGP_E_ARG, "pins matrix of another level");
  ApiScope scope(c);
  HGP_TRY(clear_errors(c));
  uint32_t *pos = nullptr;
  hgp_pins own{};
  hgp_status s = seq_setup(c, g, part, nparts, seq, M, dest, &pos);
  if (s == HGP_OK) s = check_errors_part(c);
  if (s == HGP_OK && !pins_in) {
    s = pins_impl(c, g, part, nparts, 1, &own);
    pins_in = &own;
  }
  if (s == HGP_OK) s = violations_impl(c, g, part, nparts, pins_in, seq, M, dest, omega, delta, violations);
  if (s == HGP_OK) s = hgp_sync(c);
  pins_release(c, &own);
  return s;
}

hgp_status hgp_best_prefix(hgp_ctx *c, const int64_t *gain_seq, const uint32_t *violations, uint32_t M, uint32_t *k,
                           int64_t *best) {
  if (!c || !k || !best || (M && (!gain_seq || !violations))) return set_error(HGP_E_ARG, "hgp_best_prefix: null argument");
  ApiScope scope(c);
  *k = 0;
  *best = 0;
  if (M == 0) return HGP_OK;
  hgp_status st = HGP_OK;
  uint64_t *cx = scratch_raw<uint64_t>(c, (size_t)M + 1, &st);
  unsigned long long *bm = scratch_zero<unsigned long long>(c, 2, &st);
  if (st) return st;
  HGP_CUDA(cudaMemsetAsync(bm + 1, 0xFF, 4, c->stream));
  HGP_TRY(scan_exclusive(c, InI64{gain_seq}, M, cx, nullptr));
  HGP_TRY(launch(c, "prefix_max", k_prefix_max, dim3(grid_for(c, M)), dim3(256), 0, (const uint64_t *)cx, gain_seq,
                 violations, M, bm));
  HGP_TRY(launch(c, "prefix_first", k_prefix_first, dim3(grid_for(c, M)), dim3(256), 0, (const uint64_t *)cx,
                 gain_seq, violations, M, (const unsigned long long *)bm, reinterpret_cast<unsigned int *>(bm + 1)));
  uint64_t h[2];
  HGP_TRY(read_back(c, bm, sizeof(h), h));
  if (h[0] > 0) {
    *best = (int64_t)h[0];
    *k = (uint32_t)h[1];
  }
  return HGP_OK;
}

}  // extern "C"
