// match.cu — a4: maximum-weight matching on the two-cycle proposal pseudo-forest
// (§5.4, Eqs.7-12), Pi rounds with removal of matched nodes.
//
// The DP of Eqs.7-10 only needs, per node, ss_{1-0}(n) = ss1(n) - ss0(n); writing
// g(n) = max over children of ss_{1-0}(c):
//     ss_{1-0}(n) = score(n) - max(0, g(n))                          (Eq.7 - Eq.10)
//     root pair r<->r' matched  <=>  score(r) > max(0,g(r)) + max(0,g(r'))   (Eq.8 vs Eq.11)
//     n takes best(n) = argmax_(value,id) children, when g(n) > 0 and n is not matched up (Eq.11/12)
// Bottom-up: leaves start; the last child to arrive (atomic counter) carries the walk to its
// parent, so each node is finalised exactly once from final child values (deterministic).
// Top-down: matched_up(x) = [best(t(x)) == x] and not matched_up(t(x)); it is resolved by
// walking the chain of "best child" links to its top (bounded walk, pointer jumping beyond).
#include "csr_impl.cuh"
#include "scan.cuh"

namespace hgp {

constexpr int64_t kNegInf = INT64_MIN;
constexpr uint32_t kWalkCap = 256;

struct RoundState {
  uint32_t N, pi, round;
  const hgp_cand *cand;
  uint32_t *match;          // in/out
  uint32_t *t;              // target of this round (or kNone)
  int64_t *s;               // score of this round
  uint8_t *inR;             // mutual pair member
  uint32_t *nchild;
  uint64_t *child_off;
  uint32_t *cursor;
  uint32_t *children;
  uint32_t *arrived;
  int64_t *gain;            // ss_{1-0}
  int64_t *gplus;           // max(0, g)
  uint32_t *best;           // argmax child with g > 0, or kNone
  uint8_t *done;
  uint32_t *per_round;      // device [pi] or nullptr
  uint64_t *err;
  uint32_t *overflow;       // count of nodes whose top-down walk hit the cap
  uint32_t *ovf_list;
};

__global__ void k_round_targets(RoundState R) {
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x; n < R.N; n += gridDim.x * blockDim.x) {
    const hgp_cand c = R.cand[(uint64_t)n * R.pi + R.round];
    uint32_t tn = kNone;
    if (R.match[n] == kNone && c.id != kNone && c.id < R.N && R.match[c.id] == kNone) tn = c.id;
    R.t[n] = tn;
    R.s[n] = (int64_t)c.score;
    R.nchild[n] = 0;
    R.cursor[n] = 0;
    R.arrived[n] = 0;
    R.done[n] = 0;
  }
}

__global__ void k_round_children(RoundState R) {
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x; n < R.N; n += gridDim.x * blockDim.x) {
    const uint32_t tn = R.t[n];
    const bool r = tn != kNone && R.t[tn] == n;                   // R
    R.inR[n] = r;
    if (tn != kNone && !r) atomicAdd(&R.nchild[tn], 1u);         // child(tn) \ R
  }
}

__global__ void k_round_fill(RoundState R) {
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x; n < R.N; n += gridDim.x * blockDim.x) {
    const uint32_t tn = R.t[n];
    if (tn != kNone && !R.inR[n]) R.children[R.child_off[tn] + atomicAdd(&R.cursor[tn], 1u)] = n;
  }
}

// Bottom-up (Eqs.7-10): leaves start; the last-arriving child continues with the parent.
__global__ void k_round_up(RoundState R) {
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x; n < R.N; n += gridDim.x * blockDim.x) {
    if (R.nchild[n] != 0) continue;
    uint32_t x = n;
    while (true) {
      int64_t g = kNegInf;
      uint32_t arg = kNone;
      const uint64_t c0 = R.child_off[x], c1 = R.child_off[x + 1];
      for (uint64_t k = c0; k < c1; ++k) {
        const uint32_t ch = __ldcg(&R.children[k]);
        const int64_t gc = __ldcg(reinterpret_cast<const long long *>(&R.gain[ch]));
        if (arg == kNone || gc > g || (gc == g && ch > arg)) { g = gc; arg = ch; }
      }
      const int64_t gp = (arg != kNone && g > 0) ? g : 0;
      R.best[x] = (arg != kNone && g > 0) ? arg : kNone;
      R.gplus[x] = gp;
      const uint32_t tx = R.t[x];
      R.gain[x] = tx == kNone ? kNegInf : R.s[x] - gp;
      R.done[x] = 1;
      if (tx == kNone || R.inR[x]) break;
      __threadfence();
      if (atomicAdd(&R.arrived[tx], 1u) != R.nchild[tx] - 1) break;
      __threadfence();
      x = tx;
    }
  }
}

__device__ __forceinline__ bool pair_matched(const RoundState &R, uint32_t r) {
  // Eq.11 first branch: ss1(r) > ss0(r) + ss0(r')  <=>  s(r) > max(0,g(r)) + max(0,g(r'))
  return R.s[r] > R.gplus[r] + R.gplus[R.t[r]];
}

// Top-down (Eqs.11-12). Writes match for nodes not matched before this round.
__global__ void k_round_down(RoundState R) {
  uint32_t pairs = 0;
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < R.N; x += gridDim.x * blockDim.x) {
    if (R.match[x] != kNone) continue;                             // matched in an earlier round
    const uint32_t tx = R.t[x];
    if (tx != kNone && !R.done[x]) { report_min(R.err, kErrCycle, x); continue; }
    // matched_up(x) = base(y) XOR parity(steps) along the best-child chain
    uint32_t y = x, par = 0, steps = 0;
    bool base = false, resolved = true;
    while (true) {
      const uint32_t ty = R.t[y];
      if (ty == kNone) { base = false; break; }
      if (R.inR[y]) { base = pair_matched(R, y); break; }
      if (R.best[ty] != y) { base = false; break; }
      y = ty;
      par ^= 1;
      if (++steps >= kWalkCap) { resolved = false; break; }
    }
    if (!resolved) { R.ovf_list[atomicAdd(R.overflow, 1u)] = x; continue; }
    const bool up = base ^ (par != 0);
    const uint32_t m = up ? tx : R.best[x];
    R.match[x] = m;
    if (m != kNone && x < m) ++pairs;
  }
  pairs = warp_sum(pairs);
  if (R.per_round && lane_id() == 0 && pairs) atomicAdd(&R.per_round[R.round], pairs);
}

// Fallback for chains longer than kWalkCap: pointer jumping over the listed nodes.
// jmp/par start as one best-chain step; resolved nodes carry their matched_up value.
__global__ void k_jump_init(RoundState R, const uint32_t *list, const uint32_t *count, uint32_t *jmp, uint8_t *par,
                            int8_t *val) {
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x; n < R.N; n += gridDim.x * blockDim.x) {
    const uint32_t tn = R.t[n];
    int8_t v = -1;
    if (tn == kNone) v = 0;
    else if (R.inR[n]) v = pair_matched(R, n);
    else if (R.best[tn] != n) v = 0;
    val[n] = v;
    jmp[n] = v < 0 ? tn : n;
    par[n] = v < 0 ? 1 : 0;
  }
}
__global__ void k_jump_step(uint32_t N, const uint32_t *jmp0, const uint8_t *par0, uint32_t *jmp1, uint8_t *par1,
                            int8_t *val, uint32_t *changed) {
  // val entries, once >= 0, are final, so reading them while others resolve is safe;
  // (jmp, par) pairs are double-buffered so every jump composes consistent pairs.
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
    const uint32_t y = jmp0[n];
    const uint8_t p = par0[n];
    jmp1[n] = y;
    par1[n] = p;
    if (val[n] >= 0) continue;
    const int8_t vy = val[y];
    if (vy >= 0) val[n] = (int8_t)(vy ^ p);
    else { jmp1[n] = jmp0[y]; par1[n] = p ^ par0[y]; atomicAdd(changed, 1u); }
  }
}
__global__ void k_jump_apply(RoundState R, const uint32_t *list, const uint32_t *count, const int8_t *val) {
  uint32_t pairs = 0;
  const uint32_t total = *count;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const uint32_t x = list[i];
    const bool up = val[x] > 0;
    const uint32_t m = up ? R.t[x] : R.best[x];
    R.match[x] = m;
    if (m != kNone && x < m) ++pairs;
  }
  pairs = warp_sum(pairs);
  if (R.per_round && lane_id() == 0 && pairs) atomicAdd(&R.per_round[R.round], pairs);
}

__global__ void k_fill_none(uint32_t *a, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = kNone;
}

}  // namespace hgp

using namespace hgp;

extern "C" hgp_status hgp_match(hgp_ctx *c, const hgp_cand *cand, uint32_t N, uint32_t pi, uint32_t *match,
                                uint32_t *matched_per_round) {
  if (!c || (N && (!cand || !match)) || pi < 1 || pi > HGP_MAX_PI) return set_error(HGP_E_ARG, "hgp_match: bad argument");
  if (N >= (1u << 31)) return set_error(HGP_E_OVERFLOW, "hgp_match: N >= 2^31");
  ApiScope scope(c);
  hgp_status st = HGP_OK;
  if (matched_per_round) HGP_CUDA(cudaMemsetAsync(matched_per_round, 0, 4 * pi, c->stream));
  const uint32_t grid = N ? (div_up(N, 256) < 16u * c->sm_count ? div_up(N, 256) : 16u * c->sm_count) : 0;
  HGP_TRY(launch(c, "fill_none", k_fill_none, dim3(grid), dim3(256), 0, match, N));
  if (N == 0) return HGP_OK;
  RoundState R{};
  R.N = N; R.pi = pi; R.cand = cand; R.match = match; R.per_round = matched_per_round; R.err = c->d_err;
  R.t = scratch_raw<uint32_t>(c, N, &st);
  R.s = scratch_raw<int64_t>(c, N, &st);
  R.inR = scratch_raw<uint8_t>(c, N, &st);
  R.nchild = scratch_raw<uint32_t>(c, N, &st);
  R.child_off = scratch_raw<uint64_t>(c, (size_t)N + 1, &st);
  R.cursor = scratch_raw<uint32_t>(c, N, &st);
  R.children = scratch_raw<uint32_t>(c, N, &st);
  R.arrived = scratch_raw<uint32_t>(c, N, &st);
  R.gain = scratch_raw<int64_t>(c, N, &st);
  R.gplus = scratch_raw<int64_t>(c, N, &st);
  R.best = scratch_raw<uint32_t>(c, N, &st);
  R.done = scratch_raw<uint8_t>(c, N, &st);
  R.overflow = scratch_zero<uint32_t>(c, 2, &st);
  R.ovf_list = scratch_raw<uint32_t>(c, N, &st);
  if (st) return st;
  HGP_TRY(clear_errors(c));
  for (uint32_t r = 0; r < pi; ++r) {
    R.round = r;
    HGP_TRY(launch(c, "round_targets", k_round_targets, dim3(grid), dim3(256), 0, R));
    HGP_TRY(launch(c, "round_children", k_round_children, dim3(grid), dim3(256), 0, R));
    HGP_TRY(scan_exclusive(c, InU32{R.nchild}, N, R.child_off, nullptr));
    HGP_TRY(launch(c, "round_fill", k_round_fill, dim3(grid), dim3(256), 0, R));
    HGP_TRY(launch(c, "round_up", k_round_up, dim3(grid), dim3(256), 0, R));
    HGP_CUDA(cudaMemsetAsync(R.overflow, 0, 8, c->stream));
    HGP_TRY(launch(c, "round_down", k_round_down, dim3(grid), dim3(256), 0, R));
    uint32_t novf = 0;
    HGP_TRY(read_back(c, R.overflow, 4, &novf));
    if (novf) {   // chains longer than the walk cap: pointer jumping (log rounds)
      c->h_tiers[HGP_TIER_JUMP] += novf;
      uint32_t *jmp = scratch_raw<uint32_t>(c, 2 * (size_t)N, &st);
      uint8_t *par = scratch_raw<uint8_t>(c, 2 * (size_t)N, &st);
      int8_t *val = scratch_raw<int8_t>(c, N, &st);
      if (st) return st;
      HGP_TRY(launch(c, "jump_init", k_jump_init, dim3(grid), dim3(256), 0, R, (const uint32_t *)R.ovf_list,
                     (const uint32_t *)R.overflow, jmp, par, val));
      for (int it = 0; it < 64; ++it) {
        const int a = it & 1, b = a ^ 1;
        HGP_CUDA(cudaMemsetAsync(R.overflow + 1, 0, 4, c->stream));
        HGP_TRY(launch(c, "jump_step", k_jump_step, dim3(grid), dim3(256), 0, N, (const uint32_t *)(jmp + a * (size_t)N),
                       (const uint8_t *)(par + a * (size_t)N), jmp + b * (size_t)N, par + b * (size_t)N, val,
                       R.overflow + 1));
        uint32_t changed = 0;
        HGP_TRY(read_back(c, R.overflow + 1, 4, &changed));
        if (!changed) break;
      }
      HGP_TRY(launch(c, "jump_apply", k_jump_apply, dim3(grid), dim3(256), 0, R, (const uint32_t *)R.ovf_list,
                     (const uint32_t *)R.overflow, (const int8_t *)val));
    }
  }
  uint64_t err[kErrSlots];
  HGP_TRY(fetch_errors(c, err));
  if (err[kErrCycle] != UINT64_MAX)
    return set_error(HGP_E_INTERNAL, "node %llu lies on a proposal cycle longer than 2", (unsigned long long)err[kErrCycle]);
  return HGP_OK;
}
