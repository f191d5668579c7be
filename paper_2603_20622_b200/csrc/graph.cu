// graph.cu -- the streaming CSR/CSC delta store.
//
// Replaces streamgnn/graph.py (DynamicGraph, coalesce_batch) and the PMA of
// pma.py.  Each direction is a set of gapped per-vertex runs (rtec_adj_t):
// sorted neighbour ids with reserved slack; a batch merges into touched runs
// in place when the new length fits the capacity and relocates the run to the
// arena tail otherwise.  All batch arithmetic is integer and bit-exact with
// the reference.
#include "prims.cuh"

#include <stdlib.h>

namespace rtec {

constexpr int kBlk = 256;
constexpr int32_t kArenaFullPos = 0x7fffffff;  // err position for arena/scratch exhaustion
constexpr int32_t kCodeArenaFull = RTEC_ARENA_FULL;  // compact (or grow workspace) and retry

__host__ __device__ __forceinline__ int32_t cap_for(int32_t len, float slack, int32_t min_slack) {
  int32_t extra = static_cast<int32_t>(ceilf(static_cast<float>(len) * slack));
  if (extra < min_slack) extra = min_slack;
  return len + extra;
}

// ------------------------------------------------------------------ small kernels
__global__ void k_fill_u64(uint64_t* p, uint64_t v, int64_t n) {
  RTEC_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

// degrees of a bulk edge list (from_edges graph.py:101-102, :118-119)
__global__ void k_count_degrees(const int32_t* __restrict__ src, const int32_t* __restrict__ dst, int64_t m,
                                int64_t n, int32_t* out_deg, int32_t* in_deg, uint64_t* err) {
  RTEC_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t s = src[i], d = dst[i];
    if (s < 0 || s >= n || d < 0 || d >= n) {
      report_error(err, RTEC_INVALID_VERTEX, 0);
      continue;
    }
    atomicAdd(out_deg + s, 1);
    atomicAdd(in_deg + d, 1);
  }
}

struct CapOf {
  const int32_t* len;
  float slack;
  int32_t min_slack;
  __device__ __forceinline__ int64_t operator()(int64_t v) const { return cap_for(len[v], slack, min_slack); }
};

// build runs: beg/cap/len from degrees
struct StoreBeg {
  const int32_t* len;
  int64_t* beg;
  int32_t* cap;
  int32_t* lenout;
  __device__ __forceinline__ void operator()(int64_t v, int64_t off, int64_t c) const {
    beg[v] = off;
    cap[v] = static_cast<int32_t>(c);
    lenout[v] = len[v];
  }
};

__global__ void k_make_keys_bulk(const int32_t* __restrict__ a, const int32_t* __restrict__ b, int64_t m, int64_t n,
                                 uint64_t* keys, uint32_t* vals) {
  RTEC_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = static_cast<uint64_t>(a[i]) * static_cast<uint64_t>(n) + static_cast<uint64_t>(b[i]);
    vals[i] = static_cast<uint32_t>(i);
  }
}

// scatter sorted keys into runs; duplicates -> ConfigError (graph.py:106-107)
__global__ void k_fill_runs(const uint64_t* __restrict__ skeys, const uint32_t* __restrict__ sidx, int64_t m, int64_t n,
                            const int64_t* __restrict__ beg, int32_t* __restrict__ nbr, int64_t* __restrict__ ts_out,
                            const int64_t* __restrict__ ts_in, uint64_t* err) {
  RTEC_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = skeys[i];
    if (i > 0 && skeys[i - 1] == k) report_error(err, RTEC_CONFIG_ERROR, 1);
    int64_t v = static_cast<int64_t>(k / static_cast<uint64_t>(n));
    int32_t w = static_cast<int32_t>(k - static_cast<uint64_t>(v) * n);
    // position inside the run = i - first index of v's keys; runs are contiguous in sorted order
    int64_t lo = lower_bound_dev(skeys, 0, i + 1, static_cast<uint64_t>(v) * n);
    int64_t slot = beg[v] + (i - lo);
    nbr[slot] = w;
    if (ts_out) ts_out[slot] = ts_in ? ts_in[sidx[i]] : static_cast<int64_t>(sidx[i]);
  }
}

// ------------------------------------------------------------------ build
static int build_direction(int64_t n, rtec_adj_t* a, const int32_t* own, const int32_t* nb, const int64_t* ts,
                           int64_t m, const int32_t* deg, float slack, int32_t min_slack, uint64_t* err,
                           Ws& ws, cudaStream_t s) {
  RTEC_TRY(exclusive_scan(CapOf{deg, slack, min_slack}, Count{nullptr, n}, n,
                          StoreBeg{deg, a->beg, a->cap, a->len}, a->top, ws, s));
  if (m == 0) return RTEC_OK;
  uint64_t* keys = ws.alloc<uint64_t>(m);
  uint32_t* vals = ws.alloc<uint32_t>(m);
  uint64_t* sk = ws.alloc<uint64_t>(m);
  uint32_t* sv = ws.alloc<uint32_t>(m);
  RTEC_WS_CHECK(ws);
  launch(k_make_keys_bulk, grid_for(m, kBlk), kBlk, 0, s, own, nb, m, n, keys, vals);
  int bits = bits_for(static_cast<uint64_t>(n) * static_cast<uint64_t>(n));
  RTEC_TRY(sort_pairs(keys, vals, sk, sv, Count{nullptr, m}, m, bits, ws, s));
  launch(k_fill_runs, grid_for(m, kBlk), kBlk, 0, s, sk, sv, m, n, a->beg, a->nbr, a->ts, ts, err);
  RTEC_LAUNCH_CHECK("k_fill_runs");
  return RTEC_OK;
}

// ------------------------------------------------------------------ export / compact
// warp per vertex: copy run v to dst at off[v]
__global__ void k_copy_runs(int64_t n, const int64_t* __restrict__ beg, const int32_t* __restrict__ len,
                            const int32_t* __restrict__ nbr, const int64_t* __restrict__ ts,
                            const int64_t* __restrict__ off, int32_t* out_v, int32_t* out_nbr, int64_t* out_ts,
                            int64_t* new_beg, int32_t* new_len) {
  RTEC_PDL_ENTRY();
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int lane = lane_id();
  for (int64_t v = warp; v < n; v += nw) {
    int64_t b = beg[v], o = off[v];
    int32_t L = len[v];
    for (int32_t j = lane; j < L; j += 32) {
      out_nbr[o + j] = nbr[b + j];
      if (out_ts && ts) out_ts[o + j] = ts[b + j];
      if (out_v) out_v[o + j] = static_cast<int32_t>(v);
    }
    if (lane == 0 && new_beg) {
      new_beg[v] = o;
      new_len[v] = L;
    }
  }
}

struct NopOut {
  __device__ __forceinline__ void operator()(int64_t, int64_t, int64_t) const {}
};

struct LenAt {
  const int32_t* len;
  __device__ __forceinline__ int64_t operator()(int64_t v) const { return len[v]; }
};

// ------------------------------------------------------------------ coalesce
__global__ void k_coalesce_keys(const int32_t* __restrict__ src, const int32_t* __restrict__ dst, int64_t B,
                                uint64_t* keys, uint32_t* vals) {
  RTEC_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < B; i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = (static_cast<uint64_t>(static_cast<uint32_t>(src[i])) << 32) | static_cast<uint32_t>(dst[i]);
    vals[i] = static_cast<uint32_t>(i);
  }
}

// group heads fold the per-key FSM (graph.py:248-259) sequentially and
// record the survivor at the key's first position.
__global__ void k_coalesce_fold(const uint64_t* __restrict__ sk, const uint32_t* __restrict__ sv, int64_t B,
                                const uint8_t* __restrict__ op, uint8_t* keep) {
  RTEC_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < B; i += (int64_t)gridDim.x * blockDim.x) {
    if (i > 0 && sk[i - 1] == sk[i]) continue;  // not a head
    uint32_t first = sv[i];
    int64_t cur = sv[i];  // index of the surviving event, -1 = None
    for (int64_t j = i + 1; j < B && sk[j] == sk[i]; ++j) {
      uint32_t e = sv[j];
      if (cur < 0) cur = e;
      else if (op[cur] != op[e]) cur = -1;
    }
    // keep[first] = 1 + (survivor index encoded separately)
    keep[first] = cur >= 0 ? 1 : 0;
    // stash survivor index in the sorted-value slot of the head (re-used below)
    const_cast<uint32_t*>(sv)[i] = cur >= 0 ? static_cast<uint32_t>(cur) : 0xffffffffu;
    // map first appearance -> head position via keys (done by k_coalesce_map)
  }
}

__global__ void k_coalesce_map(const uint64_t* __restrict__ sk, const uint32_t* __restrict__ sv_orig,
                               const uint32_t* __restrict__ sv_surv, int64_t B, uint32_t* surv_at_first) {
  RTEC_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < B; i += (int64_t)gridDim.x * blockDim.x) {
    if (i > 0 && sk[i - 1] == sk[i]) continue;
    surv_at_first[sv_orig[i]] = sv_surv[i];
  }
}

struct KeepAt {
  const uint8_t* keep;
  __device__ __forceinline__ int64_t operator()(int64_t i) const { return keep[i]; }
};
struct CoalesceOut {
  const uint8_t* keep;
  const uint32_t* surv;
  const int32_t* src; const int32_t* dst; const uint8_t* op; const int64_t* ts;
  int32_t* os; int32_t* od; uint8_t* oo; int64_t* ot;
  __device__ __forceinline__ void operator()(int64_t i, int64_t off, int64_t v) const {
    if (!v) return;
    uint32_t e = surv[i];
    os[off] = src[e];
    od[off] = dst[e];
    oo[off] = op[e];
    ot[off] = ts[e];
  }
};

// ------------------------------------------------------------------ apply: validation + probe
__global__ void k_apply_keys(const int32_t* __restrict__ src, const int32_t* __restrict__ dst, int64_t B, int64_t n,
                             uint64_t* keys, uint32_t* vals, uint64_t* err) {
  RTEC_PDL_ENTRY();
  uint64_t inval = static_cast<uint64_t>(n) * static_cast<uint64_t>(n);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < B; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t s = src[i], d = dst[i];
    bool ok = s >= 0 && s < n && d >= 0 && d < n;  // graph.py:192-194 (_check)
    if (!ok) report_error(err, RTEC_INVALID_VERTEX, i);
    keys[i] = ok ? static_cast<uint64_t>(s) * n + static_cast<uint64_t>(d) : inval;
    vals[i] = static_cast<uint32_t>(i);
  }
}

__global__ void k_apply_dups(const uint64_t* __restrict__ sk, const uint32_t* __restrict__ sv, int64_t B, int64_t n,
                             uint64_t* err) {
  RTEC_PDL_ENTRY();
  uint64_t inval = static_cast<uint64_t>(n) * static_cast<uint64_t>(n);
  for (int64_t i = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < B; i += (int64_t)gridDim.x * blockDim.x) {
    if (sk[i] == sk[i - 1] && sk[i] != inval) report_error(err, RTEC_CONFIG_ERROR, sv[i]);  // graph.py:195-197
  }
}

// existence probe of each (sorted) update in the pre-batch out-run of its src
// Sharded graphs (part_count > 1) probe only the updates whose dst they own;
// the others are neither applied nor reported here (status 0) -- their owner
// rank applies them and the host combines the ranks' statuses.
__global__ void k_apply_probe(const uint64_t* __restrict__ sk, const uint32_t* __restrict__ sv, int64_t B, int64_t n,
                              rtec_adj_t out, const uint8_t* __restrict__ op, uint8_t* status, uint8_t* aflag,
                              int32_t part_rank, int32_t part_count, const uint64_t* err) {
  RTEC_PDL_ENTRY();
  const bool bad = err_set(err);  // validation failed: no flags -> nothing applied
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < B; i += (int64_t)gridDim.x * blockDim.x) {
    if (bad) {
      aflag[i] = 0;
      continue;
    }
    uint64_t k = sk[i];
    int32_t s = static_cast<int32_t>(k / static_cast<uint64_t>(n));
    int32_t d = static_cast<int32_t>(k - static_cast<uint64_t>(s) * n);
    if (part_count > 1 && d % part_count != part_rank) {
      status[sv[i]] = 0;
      aflag[i] = 0;
      continue;
    }
    int64_t b = out.beg[s];
    int32_t L = out.len[s];
    int64_t p = lower_bound_dev(out.nbr, b, b + L, d);
    bool exists = p < b + L && out.nbr[p] == d;
    uint32_t e = sv[i];
    bool applied = (op[e] == RTEC_OP_INSERT) ? !exists : exists;  // graph.py:209-219
    status[e] = applied ? 1 : 0;
    aflag[i] = applied ? 1 : 0;
  }
}

struct FlagAt {
  const uint8_t* f;
  __device__ __forceinline__ int64_t operator()(int64_t i) const { return f[i]; }
};
struct CompactApplied {
  const uint8_t* f;
  const uint64_t* sk; const uint32_t* sv; int64_t n;
  const uint8_t* op; const int64_t* ts;
  int32_t* as; int32_t* ad; uint8_t* ao; int64_t* at;
  __device__ __forceinline__ void operator()(int64_t i, int64_t off, int64_t v) const {
    if (!v) return;
    uint64_t k = sk[i];
    int32_t s = static_cast<int32_t>(k / static_cast<uint64_t>(n));
    as[off] = s;
    ad[off] = static_cast<int32_t>(k - static_cast<uint64_t>(s) * n);
    uint32_t e = sv[i];
    ao[off] = op[e];
    at[off] = ts[e];
  }
};

__global__ void k_in_keys(const int32_t* __restrict__ as, const int32_t* __restrict__ ad, const int64_t* cnt, int64_t n,
                          uint64_t* keys, uint32_t* vals) {
  RTEC_PDL_ENTRY();
  int64_t K = *cnt;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < K; i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = static_cast<uint64_t>(ad[i]) * n + static_cast<uint64_t>(as[i]);
    vals[i] = static_cast<uint32_t>(i);
  }
}

__global__ void k_in_gather(const uint32_t* __restrict__ sv, const int64_t* cnt, const int32_t* __restrict__ as,
                            const int32_t* __restrict__ ad, const uint8_t* __restrict__ ao, int32_t* is, int32_t* id,
                            uint8_t* io) {
  RTEC_PDL_ENTRY();
  int64_t K = *cnt;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < K; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t e = sv[i];
    is[i] = as[e];
    id[i] = ad[e];
    io[i] = ao[e];
  }
}

// ------------------------------------------------------------------ run merge
// Updates of one direction sorted by (owner, neighbour); groups = touched runs.
struct MergeIn {
  const int32_t* own;
  const int32_t* nbr;
  const uint8_t* op;
  const int64_t* ts;  // may be null
  const int64_t* K;   // device count
  int64_t maxK;
};

struct MergePlan {
  int64_t* pre_ins;   // [maxK+1] exclusive prefix of is_insert
  int64_t* gstart;    // [maxK+1]
  int32_t* gv;        // [maxK]
  int64_t* G;         // [1]
  int64_t* work_off;  // [maxK+1]
  int64_t* scr_off;   // [maxK+1]
  int64_t* arena_off; // [maxK+1]
  int64_t* dest;      // [maxK]
  int32_t* newlen;    // [maxK]
  int32_t* newcap;    // [maxK]
  uint8_t* inplace;   // [maxK]
  int32_t* first;     // [maxK] in-place groups: run prefix [0, first) below every update stays put
  int64_t* totals;    // [4]: work, scratch, arena demand, base(top before)
  int32_t* scr_nbr;   // [scr_cap]
  int64_t* scr_ts;    // [scr_cap] or null
  int64_t scr_cap;
};


__global__ void k_group_info(MergeIn in, MergePlan p, rtec_adj_t a, float slack, int32_t min_slack,
                             const uint64_t* err) {
  RTEC_PDL_ENTRY();
  int64_t G = *p.G;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < G; g += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = p.gstart[g], e = p.gstart[g + 1];
    int32_t v = p.gv[g];
    int64_t nins = p.pre_ins[e] - p.pre_ins[s];
    int64_t ndel = (e - s) - nins;
    int32_t L = a.len[v];
    int32_t nl = static_cast<int32_t>(L + nins - ndel);
    bool inpl = nl <= a.cap[v];
    p.newlen[g] = nl;
    p.inplace[g] = inpl ? 1 : 0;
    p.newcap[g] = inpl ? a.cap[v] : cap_for(nl, slack, min_slack);
    // updates are sorted by neighbour: nothing below the smallest one moves
    const int64_t b = a.beg[v];
    p.first[g] = inpl ? static_cast<int32_t>(lower_bound_dev(a.nbr, b, b + L, in.nbr[s]) - b) : 0;
  }
}

struct WorkOf {
  MergePlan p;
  const int32_t* len;
  __device__ __forceinline__ int64_t operator()(int64_t g) const {
    return static_cast<int64_t>(len[p.gv[g]]) - p.first[g] + (p.gstart[g + 1] - p.gstart[g]);
  }
};
struct ScrOf {
  MergePlan p;
  __device__ __forceinline__ int64_t operator()(int64_t g) const { return p.inplace[g] ? p.newlen[g] - p.first[g] : 0; }
};
struct ArenaOf {
  MergePlan p;
  __device__ __forceinline__ int64_t operator()(int64_t g) const { return p.inplace[g] ? 0 : p.newcap[g]; }
};
struct StoreOffTail {
  int64_t* dst;
  const int64_t* G;
  __device__ __forceinline__ void operator()(int64_t i, int64_t off, int64_t v) const {
    dst[i] = off;
    if (i == *G - 1) dst[i + 1] = off + v;
  }
};

// reserve arena space for relocated runs (single thread): all-or-nothing
// arena reservation for relocated runs (thread 0: all-or-nothing) and the groups' destinations
// (every thread; the arena top only moves at the commit) in one launch
__global__ void k_reserve_dest(MergePlan p, rtec_adj_t a, uint64_t* err, int64_t* ctr) {
  RTEC_PDL_ENTRY();
  const int64_t G = *p.G;
  const int64_t top = *a.top;
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int64_t demand = G > 0 ? p.arena_off[G] : 0;
    int64_t scr = G > 0 ? p.scr_off[G] : 0;
    p.totals[0] = G > 0 ? p.work_off[G] : 0;
    p.totals[1] = scr;
    if (ctr) {  // merge volume (elements) for the bench's algorithmic bytes
      ctr[0] = p.totals[0];
      ctr[1] = scr;
    }
    p.totals[2] = demand;
    p.totals[3] = top;
    if (!err_set(err) && (top + demand > a.slots || scr > p.scr_cap)) report_error(err, kCodeArenaFull, kArenaFullPos);
  }
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < G; g += (int64_t)gridDim.x * blockDim.x) {
    p.dest[g] = p.inplace[g] ? -1 : top + p.arena_off[g];
  }
}

template <typename T>
__device__ __forceinline__ int64_t upper_bound_dev(const T* a, int64_t lo, int64_t hi, T key) {
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] <= key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Work positions are processed in tiles of kMT consecutive positions per block:
// two threads locate the groups of the tile's first / last position (one global
// binary search each), the groups' offsets in between are staged in shared memory
// and every thread finds its group there -- instead of a ~20-step dependent
// binary search over the global offsets per element.
constexpr int kMT = 1024;

// merge regime: average work (run suffix + updates) per touched run above 64 positions
__device__ __forceinline__ bool long_runs(int64_t W, int64_t G) { return W > 64 * G; }


struct TileGroups {
  int64_t g0, ng;  // first group of the tile, number of groups staged (0: fall back to global search)
};

__device__ __forceinline__ TileGroups tile_groups(const int64_t* off, int64_t G, int64_t t0, int64_t t1,
                                                  int64_t* s_off, int64_t* s_g) {
  if (threadIdx.x == 0) s_g[0] = upper_bound_dev<int64_t>(off, 0, G, t0) - 1;
  if (threadIdx.x == 1) s_g[1] = upper_bound_dev<int64_t>(off, 0, G, t1 - 1) - 1;
  __syncthreads();
  TileGroups tg{s_g[0], s_g[1] - s_g[0] + 1};
  if (tg.ng > kMT) tg.ng = 0;
  for (int64_t k = threadIdx.x; k < tg.ng; k += blockDim.x) s_off[k] = off[tg.g0 + k + 1];  // group ends
  __syncthreads();
  return tg;
}

__device__ __forceinline__ int64_t group_of(const TileGroups& tg, const int64_t* s_off, const int64_t* off, int64_t G,
                                            int64_t i) {
  if (tg.ng == 0) return upper_bound_dev<int64_t>(off, 0, G, i) - 1;
  int64_t lo = 0, hi = tg.ng - 1;  // first staged group whose end is > i
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (s_off[mid] <= i) lo = mid + 1;
    else hi = mid;
  }
  return tg.g0 + lo;
}

// element-parallel merge: old elements (from the first changed position) and update items of every group
__global__ void __launch_bounds__(kBlk) k_merge_items(MergeIn in, MergePlan p, rtec_adj_t a, const uint64_t* err,
                                                      bool choose) {
  RTEC_PDL_ENTRY();
  __shared__ int64_t s_off[kMT];
  __shared__ int64_t s_g[2];
  if (err_set(err)) return;
  int64_t G = *p.G;
  if (G == 0) return;
  if (choose && long_runs(p.work_off[G], G)) return;
  int64_t W = p.work_off[G];
  for (int64_t t0 = static_cast<int64_t>(blockIdx.x) * kMT; t0 < W; t0 += static_cast<int64_t>(gridDim.x) * kMT) {
    const int64_t t1 = t0 + kMT < W ? t0 + kMT : W;
    TileGroups tg = tile_groups(p.work_off, G, t0, t1, s_off, s_g);
    for (int64_t i = t0 + threadIdx.x; i < t1; i += blockDim.x) {
      int64_t g = group_of(tg, s_off, p.work_off, G, i);
      int64_t t = i - p.work_off[g];
      int32_t v = p.gv[g];
      int64_t s = p.gstart[g], e = p.gstart[g + 1];
      int64_t b = a.beg[v];
      int32_t L = a.len[v];
      const int32_t f0 = p.first[g];
      int32_t w;
      int64_t tsv = 0;
      int64_t out;
      if (t < L - f0) {
        t += f0;
        w = a.nbr[b + t];
        int64_t q = lower_bound_dev(in.nbr, s, e, w);
        if (q < e && in.nbr[q] == w) continue;  // deleted (an applied insert never hits an existing key)
        int64_t ins_before = p.pre_ins[q] - p.pre_ins[s];
        int64_t del_before = (q - s) - ins_before;
        out = t - del_before + ins_before;
        if (a.ts) tsv = a.ts[b + t];
      } else {
        int64_t k = s + (t - (L - f0));
        if (in.op[k] != RTEC_OP_INSERT) continue;
        w = in.nbr[k];
        int64_t pos = lower_bound_dev(a.nbr, b, b + L, w) - b;
        int64_t ins_before = p.pre_ins[k] - p.pre_ins[s];
        int64_t del_before = (k - s) - ins_before;
        out = pos - del_before + ins_before;
        if (in.ts) tsv = in.ts[k];
      }
      int64_t dst = p.inplace[g] ? -1 : p.dest[g] + out;
      if (dst < 0) {
        int64_t so = p.scr_off[g] + out - f0;
        p.scr_nbr[so] = w;
        if (p.scr_ts) p.scr_ts[so] = tsv;
      } else {
        a.nbr[dst] = w;
        if (a.ts) a.ts[dst] = tsv;
      }
    }
    __syncthreads();  // s_off reused by the next tile
  }
}

// Warp-per-chunk merge (default): a warp takes kWC consecutive work positions, finds its
// first group once, and walks the groups of its range with their metadata in registers.
// For a group of at most 32 updates the updates sit one per lane, and each old element's
// rank among them (inserts / deletes before it, deleted or not) comes from a shuffle sweep
// over the lanes instead of a per-element binary search in global memory; larger groups
// fall back to the binary search.  Output positions and order are those of k_merge_items.
constexpr int kWC = 512;

// positions per warp: the work spread over every resident warp (small batches: one
// 32-position step per warp, no serial walk), at most kWC
__device__ __forceinline__ int64_t warp_chunk(int64_t W, int64_t nw) {
  int64_t c = (W + nw - 1) / nw;
  c = (c + 31) & ~int64_t(31);
  return c < 32 ? 32 : (c > kWC ? kWC : c);
}

__device__ __forceinline__ void merge_put(const MergePlan& p, const rtec_adj_t& a, int64_t g, int32_t f0, int64_t out,
                                          int32_t w, int64_t tsv, bool inpl, int64_t dest, int64_t so0) {
  if (inpl) {
    const int64_t so = so0 + out - f0;
    p.scr_nbr[so] = w;
    if (p.scr_ts) p.scr_ts[so] = tsv;
  } else {
    a.nbr[dest + out] = w;
    if (a.ts) a.ts[dest + out] = tsv;
  }
}

__global__ void __launch_bounds__(kBlk) k_merge_items_warp(MergeIn in, MergePlan p, rtec_adj_t a,
                                                           const uint64_t* err, bool choose) {
  RTEC_PDL_ENTRY();
  if (err_set(err)) return;
  const int64_t G = *p.G;
  if (G == 0) return;
  const int64_t W = p.work_off[G];
  if (choose && !long_runs(W, G)) return;
  const int lane = lane_id();
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t wc = warp_chunk(W, nw);
  for (int64_t t0 = warp * wc; t0 < W; t0 += nw * wc) {
    const int64_t t1 = t0 + wc < W ? t0 + wc : W;
    int64_t g = 0;
    if (lane == 0) g = upper_bound_dev<int64_t>(p.work_off, 0, G, t0) - 1;
    g = __shfl_sync(0xffffffffu, g, 0);
    for (; g < G; ++g) {
      const int64_t wo = p.work_off[g], we = p.work_off[g + 1];
      if (wo >= t1) break;
      const int32_t v = p.gv[g];
      const int64_t s = p.gstart[g], e = p.gstart[g + 1];
      const int64_t b = a.beg[v];
      const int32_t L = a.len[v];
      const int32_t f0 = p.first[g];
      const bool inpl = p.inplace[g] != 0;
      const int64_t dest = inpl ? 0 : p.dest[g];
      const int64_t so0 = inpl ? p.scr_off[g] : 0;
      const int64_t pre_s = p.pre_ins[s];
      const int64_t nu = e - s;
      const bool small = nu <= 32;
      // small groups: update j on lane j (neighbour, op)
      int32_t un = 0x7fffffff;
      int ui = 0;
      if (small && lane < nu) {
        un = in.nbr[s + lane];
        ui = in.op[s + lane] == RTEC_OP_INSERT ? 1 : 0;
      }
      const int64_t lo = t0 > wo ? t0 : wo, hi = t1 < we ? t1 : we;
      const int64_t nold = L - f0;  // work positions [0, nold) are old elements, then the updates
      for (int64_t i0 = lo; i0 < hi; i0 += 32) {
        const int64_t i = i0 + lane;
        const bool act = i < hi;
        const int64_t t = i - wo;
        const bool old = act && t < nold;
        int32_t w = 0;
        if (old) w = a.nbr[b + f0 + t];
        int64_t ib = 0, db = 0;
        bool deleted = false;
        if (small) {
          // rank of w among the group's updates: every lane sweeps all of them (old lanes only)
          const unsigned om = __ballot_sync(0xffffffffu, old);
          if (om) {
            for (int j = 0; j < static_cast<int>(nu); ++j) {
              const int32_t uj = __shfl_sync(0xffffffffu, un, j);
              const int ij = __shfl_sync(0xffffffffu, ui, j);
              if (uj < w) {
                ib += ij;
                db += 1 - ij;
              } else if (uj == w) {
                deleted = true;  // an applied insert never hits an existing key
              }
            }
          }
        } else if (old) {
          const int64_t q = lower_bound_dev(in.nbr, s, e, w);
          deleted = q < e && in.nbr[q] == w;
          ib = p.pre_ins[q] - pre_s;
          db = (q - s) - ib;
        }
        if (old) {
          if (!deleted)
            merge_put(p, a, g, f0, f0 + t - db + ib, w, a.ts ? a.ts[b + f0 + t] : 0, inpl, dest, so0);
        } else if (act) {
          const int64_t k = s + (t - nold);
          if (in.op[k] == RTEC_OP_INSERT) {
            const int32_t wk = in.nbr[k];
            const int64_t pos = lower_bound_dev(a.nbr, b, b + L, wk) - b;
            const int64_t ibk = p.pre_ins[k] - pre_s;
            const int64_t dbk = (k - s) - ibk;
            merge_put(p, a, g, f0, pos - dbk + ibk, wk, in.ts ? in.ts[k] : 0, inpl, dest, so0);
          }
        }
      }
    }
  }
}

// copy in-place runs back from scratch, a warp per kWC scratch positions walking its groups
__global__ void __launch_bounds__(kBlk) k_merge_copyback_warp(MergePlan p, rtec_adj_t a, const uint64_t* err,
                                                              bool choose) {
  RTEC_PDL_ENTRY();
  if (err_set(err)) return;
  const int64_t G = *p.G;
  if (G == 0) return;
  if (choose && !long_runs(p.work_off[G], G)) return;
  const int64_t S = p.scr_off[G];
  const int lane = lane_id();
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t wc = warp_chunk(S, nw);
  for (int64_t t0 = warp * wc; t0 < S; t0 += nw * wc) {
    const int64_t t1 = t0 + wc < S ? t0 + wc : S;
    int64_t g = 0;
    if (lane == 0) g = upper_bound_dev<int64_t>(p.scr_off, 0, G, t0) - 1;
    g = __shfl_sync(0xffffffffu, g, 0);
    for (; g < G; ++g) {
      const int64_t so = p.scr_off[g], se = p.scr_off[g + 1];
      if (so >= t1) break;
      if (se == so) continue;
      const int64_t base = a.beg[p.gv[g]] + p.first[g] - so;
      const int64_t lo = t0 > so ? t0 : so, hi = t1 < se ? t1 : se;
      for (int64_t i = lo + lane; i < hi; i += 32) {
        a.nbr[base + i] = p.scr_nbr[i];
        if (a.ts) a.ts[base + i] = p.scr_ts[i];
      }
    }
  }
}

// copy in-place runs back from scratch (after all reads of the old runs)
__global__ void __launch_bounds__(kBlk) k_merge_copyback(MergePlan p, rtec_adj_t a, const uint64_t* err,
                                                         bool choose) {
  RTEC_PDL_ENTRY();
  __shared__ int64_t s_off[kMT];
  __shared__ int64_t s_g[2];
  if (err_set(err)) return;
  int64_t G = *p.G;
  if (G == 0) return;
  if (choose && long_runs(p.work_off[G], G)) return;
  int64_t S = p.scr_off[G];
  for (int64_t t0 = static_cast<int64_t>(blockIdx.x) * kMT; t0 < S; t0 += static_cast<int64_t>(gridDim.x) * kMT) {
    const int64_t t1 = t0 + kMT < S ? t0 + kMT : S;
    TileGroups tg = tile_groups(p.scr_off, G, t0, t1, s_off, s_g);
    for (int64_t i = t0 + threadIdx.x; i < t1; i += blockDim.x) {
      int64_t g = group_of(tg, s_off, p.scr_off, G, i);
      int32_t v = p.gv[g];
      int64_t t = i - p.scr_off[g] + p.first[g];
      a.nbr[a.beg[v] + t] = p.scr_nbr[i];
      if (a.ts) a.ts[a.beg[v] + t] = p.scr_ts[i];
    }
    __syncthreads();
  }
}

__global__ void k_merge_commit(MergePlan p, rtec_adj_t a, const uint64_t* err) {
  RTEC_PDL_ENTRY();
  if (err_set(err)) return;
  if (threadIdx.x == 0 && blockIdx.x == 0) *a.top = p.totals[3] + p.totals[2];  // commit the reservation
  int64_t G = *p.G;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < G; g += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = p.gv[g];
    a.len[v] = p.newlen[g];
    if (!p.inplace[g]) {
      a.beg[v] = p.dest[g];
      a.cap[v] = p.newcap[g];
    }
  }
}

static int plan_alloc(MergePlan& p, int64_t maxK, int64_t scr_cap, bool with_ts, Ws& ws) {
  p.pre_ins = ws.alloc<int64_t>(maxK + 2);
  p.gstart = ws.alloc<int64_t>(maxK + 2);
  p.gv = ws.alloc<int32_t>(maxK + 1);
  p.G = ws.alloc<int64_t>(4);
  p.work_off = ws.alloc<int64_t>(maxK + 2);
  p.scr_off = ws.alloc<int64_t>(maxK + 2);
  p.arena_off = ws.alloc<int64_t>(maxK + 2);
  p.dest = ws.alloc<int64_t>(maxK + 1);
  p.newlen = ws.alloc<int32_t>(maxK + 1);
  p.newcap = ws.alloc<int32_t>(maxK + 1);
  p.inplace = ws.alloc<uint8_t>(maxK + 1);
  p.first = ws.alloc<int32_t>(maxK + 1);
  p.totals = ws.alloc<int64_t>(4);
  p.scr_cap = scr_cap;
  p.scr_nbr = ws.alloc<int32_t>(scr_cap);
  p.scr_ts = with_ts ? ws.alloc<int64_t>(scr_cap) : nullptr;
  RTEC_WS_CHECK(ws);
  return RTEC_OK;
}

// plan: groups, new lengths, offsets, arena reservation; no mutation
// One scan yields both the insert prefix and the group heads: (is_insert << 32 | is_head)
// per update (counts < 2^31: the packed sums never carry between the halves)
struct InsHeadPack {
  const uint8_t* op;
  const int32_t* own;
  __device__ __forceinline__ int64_t operator()(int64_t i) const {
    return (static_cast<int64_t>(op[i] == RTEC_OP_INSERT ? 1 : 0) << 32) | ((i == 0 || own[i] != own[i - 1]) ? 1 : 0);
  }
};
struct InsHeadStore {
  int64_t* pre_ins;
  int64_t* gstart;
  int32_t* gv;
  const int32_t* own;
  const int64_t* K;
  int64_t* G;
  __device__ __forceinline__ void operator()(int64_t i, int64_t off, int64_t v) const {
    pre_ins[i] = off >> 32;
    if (v & 0xffffffffll) {
      gstart[off & 0xffffffffll] = i;
      gv[off & 0xffffffffll] = own[i];
    }
    if (i == *K - 1) {  // tails: pre_ins[K], gstart[G] = K, the group count
      const int64_t t = off + v;
      pre_ins[i + 1] = t >> 32;
      gstart[t & 0xffffffffll] = *K;
      *G = t & 0xffffffffll;
    }
  }
};

// The run arrays below are read only for groups g < G, every one of which the scans write
// (element 0 and the tail included), so only the group count needs a reset (K = 0).
static int merge_plan(const MergeIn& in, MergePlan& p, const rtec_adj_t& a, float slack, int32_t min_slack,
                      uint64_t* err, Ws& ws, cudaStream_t s, int64_t* ctr) {
  RTEC_CUDA(cudaMemsetAsync(p.G, 0, sizeof(int64_t), s));
  Count K{in.K, in.maxK};
  RTEC_TRY(exclusive_scan(InsHeadPack{in.op, in.own}, K, in.maxK,
                          InsHeadStore{p.pre_ins, p.gstart, p.gv, in.own, in.K, p.G}, nullptr, ws, s));
  launch(k_group_info, grid_for(in.maxK, kBlk), kBlk, 0, s, in, p, a, slack, min_slack, err);
  Count G{p.G, in.maxK};
  RTEC_TRY(exclusive_scan(WorkOf{p, a.len}, G, in.maxK, StoreOffTail{p.work_off, p.G}, nullptr, ws, s));
  RTEC_TRY(exclusive_scan(ScrOf{p}, G, in.maxK, StoreOffTail{p.scr_off, p.G}, nullptr, ws, s));
  RTEC_TRY(exclusive_scan(ArenaOf{p}, G, in.maxK, StoreOffTail{p.arena_off, p.G}, nullptr, ws, s));
  launch(k_reserve_dest, grid_for(in.maxK, kBlk), kBlk, 0, s, p, a, err, ctr);
  RTEC_LAUNCH_CHECK("merge_plan");
  return RTEC_OK;
}

// RTEC_MERGE_WARP env: 1 (default) choose by run slots per vertex, 0 element-parallel only,
// 2 warp-per-chunk only (A/B)
static int merge_mode() {
  static int m = -1;
  if (m < 0) {
    const char* e = getenv("RTEC_MERGE_WARP");
    m = e ? atoi(e) : 1;
    if (m < 0 || m > 2) m = 1;
  }
  return m;
}

static int merge_exec(const MergeIn& in, MergePlan& p, const rtec_adj_t& a, int64_t n, int64_t work_bound,
                      uint64_t* err, cudaStream_t s) {
  RTEC_PROF("adj_merge", s);
  // warp-per-chunk merges for long runs (measured on c3-gat's ~490-edge runs and the skewed
  // R-MAT runs of c4, ~60 edges on average but hub-dominated), element-parallel ones for short
  // runs (c2 / c1, < 50 slots per vertex); the regime from the run slots per vertex (host-known)
  const int mode = merge_mode();
  const bool warp = mode == 2 || (mode == 1 && a.slots > 64 * (n > 0 ? n : 1));
  if (warp) {
    launch(k_merge_items_warp, grid_for(work_bound, kWC * (kBlk / 32), kSMs * 8), kBlk, 0, s, in, p, a, err, false);
    launch(k_merge_copyback_warp, grid_for(work_bound, kWC * (kBlk / 32), kSMs * 8), kBlk, 0, s, p, a, err, false);
  } else {
    launch(k_merge_items, grid_for(work_bound, kMT, kSMs * 8), kBlk, 0, s, in, p, a, err, false);
    launch(k_merge_copyback, grid_for(work_bound, kMT, kSMs * 8), kBlk, 0, s, p, a, err, false);
  }
  launch(k_merge_commit, grid_for(in.maxK, kBlk), kBlk, 0, s, p, a, err);
  RTEC_LAUNCH_CHECK("merge_exec");
  return RTEC_OK;
}


__global__ void k_irange_reset(const int32_t* __restrict__ id, const int64_t* cnt, int2* irange) {
  RTEC_PDL_ENTRY();
  int64_t K = *cnt;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < K; i += (int64_t)gridDim.x * blockDim.x)
    irange[id[i]] = make_int2(-1, 0);
}

// ------------------------------------------------------------------ degrees + deltas

// over the applied updates in one launch: per-destination ranges of the in-key ordered list
// (replaces a binary search per destination in the layer kernels) and the degree updates
__global__ void k_irange_degrees(const int32_t* __restrict__ id, int2* irange, const int32_t* __restrict__ as,
                                 const int32_t* __restrict__ ad, const uint8_t* __restrict__ ao, const int64_t* cnt,
                                 int32_t* out_deg, int32_t* in_deg, int64_t* num_edges, const uint64_t* err) {
  RTEC_PDL_ENTRY();
  if (err_set(err)) return;
  const int64_t K = *cnt;
  int64_t local = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < K; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = id[i];
    if (i == 0 || id[i - 1] != v) {
      int64_t j = i + 1;
      while (j < K && id[j] == v) ++j;
      irange[v] = make_int2(static_cast<int32_t>(i), static_cast<int32_t>(j - i));
    }
    const int32_t d = ao[i] == RTEC_OP_INSERT ? 1 : -1;
    atomicAdd(out_deg + as[i], d);
    atomicAdd(in_deg + ad[i], d);
    local += d;
  }
  local = warp_sum(local);
  if (lane_id() == 0 && local != 0) atomicAdd(reinterpret_cast<unsigned long long*>(num_edges),
                                              static_cast<unsigned long long>(local));
}

// endpoints of the applied updates -> bits of a touched-vertex bitmap
__global__ void k_touched_bits(const int32_t* __restrict__ as, const int32_t* __restrict__ ad, const int64_t* cnt,
                               uint32_t* bm) {
  RTEC_PDL_ENTRY();
  const int64_t K = *cnt;
  for (int64_t i0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~int64_t(31); i0 < K;
       i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + lane_id();
    const bool act = i < K;
    bm_set_warp(bm, act ? as[i] : 0, act);
    bm_set_warp(bm, act ? ad[i] : 0, act);
  }
}

// touched vertices whose (in, out) degree changed -> DegreeDelta rows, ascending
// (graph.py:225-230): one bitmap word per scan item
struct TouchedWord {
  const uint32_t* bm;
  const int32_t* in_deg; const int32_t* out_deg; const int32_t* in_prev; const int32_t* out_prev;
  __device__ __forceinline__ uint32_t changed(int64_t w) const {
    uint32_t t = bm[w], c = 0;
    while (t) {
      const int b = __ffs(t) - 1;
      t &= t - 1;
      const int64_t v = w * 32 + b;
      if (in_deg[v] != in_prev[v] || out_deg[v] != out_prev[v]) c |= 1u << b;
    }
    return c;
  }
  __device__ __forceinline__ int64_t operator()(int64_t w) const { return __popc(changed(w)); }
};
struct TouchedRows {
  TouchedWord f;
  int32_t* dv; int32_t* doi; int32_t* dni; int32_t* doo; int32_t* dno;
  __device__ __forceinline__ void operator()(int64_t w, int64_t off, int64_t) const {
    uint32_t c = f.changed(w);
    while (c) {
      const int b = __ffs(c) - 1;
      c &= c - 1;
      const int32_t x = static_cast<int32_t>(w * 32 + b);
      dv[off] = x;
      doi[off] = f.in_prev[x];
      dni[off] = f.in_deg[x];
      doo[off] = f.out_prev[x];
      dno[off] = f.out_deg[x];
      ++off;
    }
  }
};

__global__ void k_commit_degrees(const int32_t* __restrict__ dv, const int64_t* cnt, const int32_t* in_deg,
                                 const int32_t* out_deg, int32_t* in_prev, int32_t* out_prev) {
  RTEC_PDL_ENTRY();
  int64_t K = *cnt;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < K; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = dv[i];
    in_prev[v] = in_deg[v];
    out_prev[v] = out_deg[v];
  }
}

// ------------------------------------------------------------------ workspace sizing
size_t batch_ws_bytes(int64_t n, int64_t B, int64_t scr_cap) {
  size_t b = 0;
  auto add = [&](size_t x) { b += (x + 255) & ~size_t(255); };
  int64_t B2 = 2 * B + 2;
  for (int i = 0; i < 3; ++i) {  // keys/vals/sorted copies for up to 2B entries
    add(sizeof(uint64_t) * B2);
    add(sizeof(uint32_t) * B2);
  }
  add(B2);
  add(sizeof(int64_t) * 8);
  for (int d = 0; d < 2; ++d) {  // two merge plans
    add(sizeof(int64_t) * (B + 2) * 6);
    add(sizeof(int32_t) * (B + 2) * 4);
    add(B + 2);
    add(sizeof(int64_t) * 8);
    add(sizeof(int32_t) * scr_cap);
    add(sizeof(int64_t) * scr_cap);
  }
  add(sort_ws_bytes(B2));
  add(sizeof(int64_t) * (scan_blocks_for(B2) + 2) * 12);
  add(sizeof(uint32_t) * ((n + 31) / 32));  // touched-vertex bitmap (DegreeDelta rows)
  add(sizeof(int64_t) * (((n + 31) / 32 + 511) / 512 + 2));
  return b + (1 << 16);
}

}  // namespace rtec

using namespace rtec;

extern "C" {

int rtec_graph_count(const int32_t* src, const int32_t* dst, int64_t m, int64_t n, int32_t* out_deg,
                     int32_t* in_deg, uint64_t* err, rtec_stream_t stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (m > 0) launch(k_count_degrees, grid_for(m, kBlk), kBlk, 0, s, src, dst, m, n, out_deg, in_deg, err);
  RTEC_LAUNCH_CHECK("k_count_degrees");
  return RTEC_OK;
}

int rtec_graph_slots_needed(const int32_t* len, int64_t n, float slack, int32_t min_slack, int64_t* slots_dev,
                            void* ws, size_t ws_bytes, rtec_stream_t stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  Ws w(ws, ws_bytes);
  return exclusive_scan(CapOf{len, slack, min_slack}, Count{nullptr, n}, n, NopOut{}, slots_dev, w, s);
}

int rtec_graph_build(rtec_graph_t* g, const int32_t* src, const int32_t* dst, const int64_t* ts, int64_t m,
                     float slack, int32_t min_slack, uint64_t* err, void* ws, size_t ws_bytes,
                     rtec_stream_t stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int64_t n = g->n;
  {
    Ws w(ws, ws_bytes);
    RTEC_TRY(build_direction(n, &g->out, src, dst, ts, m, g->out_deg, slack, min_slack, err, w, s));
  }
  {
    Ws w(ws, ws_bytes);
    RTEC_TRY(build_direction(n, &g->in, dst, src, nullptr, m, g->in_deg, slack, min_slack, err, w, s));
  }
  RTEC_CUDA(cudaMemcpyAsync(g->out_deg_prev, g->out_deg, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, s));
  RTEC_CUDA(cudaMemcpyAsync(g->in_deg_prev, g->in_deg, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, s));
  RTEC_CUDA(cudaMemcpyAsync(g->num_edges, &m, sizeof(int64_t), cudaMemcpyHostToDevice, s));
  RTEC_CUDA(cudaStreamSynchronize(s));  // &m is a host stack value
  return RTEC_OK;
}

int rtec_adj_export(int64_t n, const rtec_adj_t* a, int32_t* out_v, int32_t* out_nbr, int64_t* out_ts, void* ws,
                    size_t ws_bytes, rtec_stream_t stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  Ws w(ws, ws_bytes);
  int64_t* off = w.alloc<int64_t>(n + 1);
  RTEC_WS_CHECK(w);
  RTEC_TRY(exclusive_scan(LenAt{a->len}, Count{nullptr, n}, n, StorePrefix{off}, nullptr, w, s));
  launch(k_copy_runs, grid_for(n * 32, kBlk, kSMs * 16), kBlk, 0, s, n, a->beg, a->len, a->nbr, a->ts, off, out_v,
                                                                 out_nbr, out_ts, nullptr, nullptr);
  RTEC_LAUNCH_CHECK("k_copy_runs");
  return RTEC_OK;
}

int rtec_adj_compact(int64_t n, const rtec_adj_t* src, rtec_adj_t* dst, float slack, int32_t min_slack, void* ws,
                     size_t ws_bytes, rtec_stream_t stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  Ws w(ws, ws_bytes);
  // new beg/cap from current lengths (dst->len receives the lengths)
  RTEC_TRY(exclusive_scan(CapOf{src->len, slack, min_slack}, Count{nullptr, n}, n,
                          StoreBeg{src->len, dst->beg, dst->cap, dst->len}, dst->top, w, s));
  launch(k_copy_runs, grid_for(n * 32, kBlk, kSMs * 16), kBlk, 0, s, n, src->beg, src->len, src->nbr, src->ts, dst->beg,
                                                                 nullptr, dst->nbr, dst->ts, nullptr, nullptr);
  RTEC_LAUNCH_CHECK("compact");
  return RTEC_OK;
}

int rtec_batch_coalesce(const int32_t* src, const int32_t* dst, const uint8_t* op, const int64_t* ts, int64_t B,
                        int32_t* out_src, int32_t* out_dst, uint8_t* out_op, int64_t* out_ts, int64_t* n_out,
                        void* ws, size_t ws_bytes, rtec_stream_t stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  RTEC_CUDA(cudaMemsetAsync(n_out, 0, sizeof(int64_t), s));
  if (B <= 0) return RTEC_OK;
  Ws w(ws, ws_bytes);
  uint64_t* keys = w.alloc<uint64_t>(B);
  uint32_t* vals = w.alloc<uint32_t>(B);
  uint64_t* sk = w.alloc<uint64_t>(B);
  uint32_t* sv = w.alloc<uint32_t>(B);
  uint32_t* sv2 = w.alloc<uint32_t>(B);
  uint8_t* keep = w.alloc<uint8_t>(B);
  uint32_t* surv = w.alloc<uint32_t>(B);
  RTEC_WS_CHECK(w);
  launch(k_coalesce_keys, grid_for(B, kBlk), kBlk, 0, s, src, dst, B, keys, vals);
  RTEC_TRY(sort_pairs(keys, vals, sk, sv, Count{nullptr, B}, B, 64, w, s));
  RTEC_CUDA(cudaMemcpyAsync(sv2, sv, sizeof(uint32_t) * B, cudaMemcpyDeviceToDevice, s));
  RTEC_CUDA(cudaMemsetAsync(keep, 0, B, s));
  launch(k_coalesce_fold, grid_for(B, kBlk), kBlk, 0, s, sk, sv2, B, op, keep);
  launch(k_coalesce_map, grid_for(B, kBlk), kBlk, 0, s, sk, sv, sv2, B, surv);
  RTEC_TRY(exclusive_scan(KeepAt{keep}, Count{nullptr, B}, B,
                          CoalesceOut{keep, surv, src, dst, op, ts, out_src, out_dst, out_op, out_ts}, n_out, w, s));
  return RTEC_OK;
}

int rtec_batch_apply(rtec_graph_t* g, rtec_batch_t* b, const int32_t* src, const int32_t* dst, const uint8_t* op,
                     const int64_t* ts, int64_t B, void* ws, size_t ws_bytes, rtec_stream_t stream) {
  return rtec_batch_apply_phase(g, b, src, dst, op, ts, B, 3, ws, ws_bytes, stream);
}

// Phase 1 (plan) and phase 2 (mutate) carve the workspace identically, so the
// merge plans phase 1 leaves in it are the ones phase 2 executes.
int rtec_batch_apply_phase(rtec_graph_t* g, rtec_batch_t* b, const int32_t* src, const int32_t* dst,
                           const uint8_t* op, const int64_t* ts, int64_t B, int32_t phase, void* ws, size_t ws_bytes,
                           rtec_stream_t stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int64_t n = g->n;
  if (B > b->cap) {
    set_error("batch of %lld updates exceeds capacity %lld", (long long)B, (long long)b->cap);
    return RTEC_SHAPE_ERROR;
  }
  if (phase < 1 || phase > 3) {
    set_error("apply phase %d not in {1, 2, 3}", phase);
    return RTEC_CONFIG_ERROR;
  }
  const bool plan = phase & 1, exec = phase & 2;
  if (plan) {  // error word to "none", applied / DegreeDelta counts to 0: one fill kernel
    Fill4 clr{};
    clr.s[0] = FillSpan{b->err, static_cast<int64_t>(sizeof(uint64_t)), 0xffffffffu};
    clr.s[1] = FillSpan{b->n_applied, static_cast<int64_t>(sizeof(int64_t)), 0u};
    clr.s[2] = FillSpan{b->n_delta, static_cast<int64_t>(sizeof(int64_t)), 0u};
    clr.n = 3;
    RTEC_TRY(fill_spans(clr, s));
  }
  if (B <= 0) return RTEC_OK;
  RTEC_PROF("batch_apply", s);
  Ws w(ws, ws_bytes);
  int64_t B2 = 2 * B;
  uint64_t* keys = w.alloc<uint64_t>(B2);
  uint32_t* vals = w.alloc<uint32_t>(B2);
  uint64_t* sk = w.alloc<uint64_t>(B2);
  uint32_t* sv = w.alloc<uint32_t>(B2);
  uint8_t* aflag = w.alloc<uint8_t>(B);
  // scratch capacity for in-place run merges: whatever workspace remains, split over 2 plans
  MergePlan po, pi;
  size_t plan_fixed = sizeof(int64_t) * (B + 2) * 7 + sizeof(int32_t) * (B + 2) * 4 + (B + 2) + 4096 + 256;
  size_t sort_reserve = sort_ws_bytes(B2) + sizeof(int64_t) * (scan_blocks_for(B2) + 2) * 16 + (1 << 16) +
                        sizeof(uint32_t) * ((n + 31) / 32) + sizeof(int64_t) * (((n + 31) / 32 + 511) / 512 + 2) + 512;
  size_t used = w.off + 2 * plan_fixed + sort_reserve;
  int64_t scr_cap = used < w.bytes ? static_cast<int64_t>((w.bytes - used) / 2 / (sizeof(int32_t) + sizeof(int64_t) + 1)) : 0;
  RTEC_TRY(plan_alloc(po, B, scr_cap, true, w));
  RTEC_TRY(plan_alloc(pi, B, scr_cap, false, w));
  RTEC_WS_CHECK(w);
  size_t mark = w.off;
  const int grid = grid_for(B, kBlk);
  int bits = bits_for(static_cast<uint64_t>(n) * static_cast<uint64_t>(n));
  MergeIn mo{b->a_src, b->a_dst, b->a_op, b->a_ts, b->n_applied, B};
  MergeIn mi{b->i_dst, b->i_src, b->i_op, nullptr, b->n_applied, B};
  if (plan) {
  // 1. keys + range validation; 2. sort; 3. duplicate validation
  launch(k_apply_keys, grid, kBlk, 0, s, src, dst, B, n, keys, vals, b->err);
  RTEC_TRY(sort_pairs(keys, vals, sk, sv, Count{nullptr, B}, B, bits, w, s));
  w.off = mark;
  launch(k_apply_dups, grid, kBlk, 0, s, sk, sv, B, n, b->err);
  // 4. probe against the pre-batch graph (skipped on validation error: no flags -> nothing applied)
  launch(k_apply_probe, grid, kBlk, 0, s, sk, sv, B, n, g->out, op, b->status, aflag, g->part_rank, g->part_count,
                                      b->err);
  // 5. applied updates in out-key order
  RTEC_TRY(exclusive_scan(FlagAt{aflag}, Count{nullptr, B}, B,
                          CompactApplied{aflag, sk, sv, n, op, ts, b->a_src, b->a_dst, b->a_op, b->a_ts},
                          b->n_applied, w, s));
  w.off = mark;
  // 6. in-key order
  launch(k_in_keys, grid, kBlk, 0, s, b->a_src, b->a_dst, b->n_applied, n, keys, vals);
  RTEC_TRY(sort_pairs(keys, vals, sk, sv, Count{b->n_applied, B}, B, bits, w, s));
  w.off = mark;
  launch(k_in_gather, grid, kBlk, 0, s, sv, b->n_applied, b->a_src, b->a_dst, b->a_op, b->i_src, b->i_dst, b->i_op);
  // 7. plan both merges (no mutation; all-or-nothing arena reservation) -- independent of
  // each other: the in-run plan runs on the side stream with its own scratch
  {
    cudaStream_t ps = g_prof_on ? s : side_stream();
    if (ps != s) {
      RTEC_CUDA(cudaEventRecord(side_fork(), s));
      RTEC_CUDA(cudaStreamWaitEvent(ps, side_fork(), 0));
    }
    RTEC_TRY(merge_plan(mo, po, g->out, g->slack, g->min_slack, b->err, w, s, b->apply_ctr));
    RTEC_TRY(merge_plan(mi, pi, g->in, g->slack, g->min_slack, b->err, w, ps,
                        b->apply_ctr ? b->apply_ctr + 2 : nullptr));
    if (ps != s) {
      RTEC_CUDA(cudaEventRecord(side_join(), ps));
      RTEC_CUDA(cudaStreamWaitEvent(s, side_join(), 0));
    }
    w.off = mark;
  }
  }
  if (!exec) return RTEC_OK;
  // 8. mutate: degrees, runs, per-destination ranges
  launch(k_irange_degrees, grid, kBlk, 0, s, b->i_dst, reinterpret_cast<int2*>(b->irange), b->a_src, b->a_dst, b->a_op,
         b->n_applied, g->out_deg, g->in_deg, g->num_edges, b->err);
  int64_t work_bound = g->out.slots + B;  // grid-stride loops read the real totals on device
  // the two directions touch disjoint arrays (own plans and scratch): merge them concurrently
  cudaStream_t ms = g_prof_on ? s : side_stream();
  if (ms != s) {
    RTEC_CUDA(cudaEventRecord(side_fork(), s));
    RTEC_CUDA(cudaStreamWaitEvent(ms, side_fork(), 0));
  }
  RTEC_TRY(merge_exec(mo, po, g->out, n, work_bound, b->err, ms));
  RTEC_TRY(merge_exec(mi, pi, g->in, n, work_bound, b->err, s));
  if (ms != s) {
    RTEC_CUDA(cudaEventRecord(side_join(), ms));
    RTEC_CUDA(cudaStreamWaitEvent(s, side_join(), 0));
  }
  // 9. DegreeDelta rows: endpoints of applied updates (touched bitmap) whose degrees changed
  const int64_t words = (n + 31) / 32;
  uint32_t* tbm = w.alloc<uint32_t>(words);
  RTEC_WS_CHECK(w);
  RTEC_CUDA(cudaMemsetAsync(tbm, 0, sizeof(uint32_t) * words, s));
  launch(k_touched_bits, grid, kBlk, 0, s, b->a_src, b->a_dst, b->n_applied, tbm);
  TouchedWord tw{tbm, g->in_deg, g->out_deg, g->in_deg_prev, g->out_deg_prev};
  RTEC_TRY(exclusive_scan(tw, Count{nullptr, words}, words,
                          TouchedRows{tw, b->d_vertex, b->d_old_in, b->d_new_in, b->d_old_out, b->d_new_out},
                          b->n_delta, w, s, /*wide=*/true));
  w.off = mark;
  return RTEC_OK;
}

int rtec_batch_commit(rtec_graph_t* g, const rtec_batch_t* b, rtec_stream_t stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  launch(k_irange_reset, grid_for(b->cap, kBlk), kBlk, 0, s, b->i_dst, b->n_applied, reinterpret_cast<int2*>(b->irange));
  launch(k_commit_degrees, grid_for(b->cap * 2, kBlk), kBlk, 0, s, b->d_vertex, b->n_delta, g->in_deg, g->out_deg,
                                                               g->in_deg_prev, g->out_deg_prev);
  RTEC_LAUNCH_CHECK("k_commit_degrees");
  return RTEC_OK;
}

}  // extern "C"
