// shard.cu -- vertex-sharded execution with a ghost-row store.
//
// Partitioning: owner(v) = v mod P.  Rank p holds every edge whose dst it owns
// (both directions) over LOCAL vertex ids: [0, n_own) are its owned vertices
// (local i <-> global p + P i), [n_own, n_loc) are ghosts -- the sources with at
// least one out-edge into the shard.  Every per-vertex array of the shard (graph
// runs, degrees, bitmaps, frontier lists, the layer inputs H^0..H^{L-1}, GAT
// caches) is sized by the local id capacity, not by n: there are no replicas of
// the embedding store.  The layer kernels run unchanged on the local graph.
//
// Ghost coherence: `peers[i]` (owned i) has bit q set iff rank q holds a ghost
// row of i.  Both sides update it from the same global batch: an insert (u, v)
// with owner(v) = q != owner(u) and bit q clear admits u at q (the owner ships
// u's pre-batch rows H^0..H^{L-1} and its global out-degree) -- rtec_shard_admit.
// After layer l a rank sends each of its changed rows V_dst(l) only to the ranks
// in peers[] (rtec_shard_count_peers / rtec_shard_pack), and receivers overwrite
// their ghost rows, logging the pre-batch value for the next layer's retractions
// (rtec_shard_unpack_changed).  The collectives themselves are issued by the host
// (NCCL all_to_all over NVLink / NVSwitch).
//
// Global out-degrees (GCN's 1/sqrt(d_out(u)+off), models.py:98-99, and the Dg
// seed of the F1 rule) are kept for every local vertex and updated from the
// globally applied set of each batch (per-update status MAX-all-reduced; every
// update has exactly one owner).  DegreeDelta rows (graph.py:225-230) are
// produced by the owner of each vertex from its exact in-degree (local graph)
// and global out-degree.
#include "prims.cuh"

namespace rtec {

constexpr int kSBlk = 256;
constexpr int kShardMaxWorld = RTEC_SHARD_MAX_WORLD;
constexpr int kShardMaxMats = RTEC_SHARD_MAX_MATS;

__device__ __forceinline__ int32_t owner_of(int32_t v, int32_t world) { return v % world; }

// ------------------------------------------------------------------ batch validation
__global__ void k_val_keys(const int32_t* __restrict__ src, const int32_t* __restrict__ dst, int64_t B, int64_t n,
                           uint64_t* keys, uint32_t* vals, uint64_t* err) {
  RTEC_PDL_ENTRY();
  const uint64_t inval = static_cast<uint64_t>(n) * static_cast<uint64_t>(n);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < B; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = src[i], d = dst[i];
    const bool ok = s >= 0 && s < n && d >= 0 && d < n;  // graph.py:192-194
    if (!ok) report_error(err, RTEC_INVALID_VERTEX, i);
    keys[i] = ok ? static_cast<uint64_t>(s) * n + static_cast<uint64_t>(d) : inval;
    vals[i] = static_cast<uint32_t>(i);
  }
}

__global__ void k_val_dups(const uint64_t* __restrict__ sk, const uint32_t* __restrict__ sv, int64_t B, int64_t n,
                           uint64_t* err) {
  RTEC_PDL_ENTRY();
  const uint64_t inval = static_cast<uint64_t>(n) * static_cast<uint64_t>(n);
  for (int64_t i = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < B; i += (int64_t)gridDim.x * blockDim.x)
    if (sk[i] == sk[i - 1] && sk[i] != inval) report_error(err, RTEC_CONFIG_ERROR, sv[i]);  // graph.py:195-197
}

// ------------------------------------------------------------------ ghost admission
// receiver side: sources of inserts into owned destinations that are not local yet
// -> bit in bm_adm (global ids); owner side: (owned source, destination rank) pairs
// whose peer bit was clear -> send list, per-peer counts
__global__ void k_admit(rtec_shard_t sh, const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                        const uint8_t* __restrict__ op, int64_t B, const uint64_t* err, uint32_t* bm_adm,
                        int32_t* send_u, int32_t* send_q, int64_t* n_send, int64_t* peer_count) {
  RTEC_PDL_ENTRY();
  if (err_set(err)) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < B; i += (int64_t)gridDim.x * blockDim.x) {
    if (op[i] != RTEC_OP_INSERT) continue;
    const int32_t s = src[i], d = dst[i];
    const int32_t qs = owner_of(s, sh.world), qd = owner_of(d, sh.world);
    if (qs == qd) continue;  // the source is owned where the edge lives
    if (qd == sh.rank && sh.g2l[s] < 0) atomicOr(bm_adm + (s >> 5), 1u << (s & 31));
    if (qs == sh.rank) {
      const int32_t ls = s / sh.world;
      const uint32_t bit = 1u << qd;
      const uint32_t old = atomicOr(sh.peers + ls, bit);
      if (!(old & bit)) {
        const int64_t k = atomicAdd(reinterpret_cast<unsigned long long*>(n_send), 1ull);
        send_u[k] = ls;
        send_q[k] = qd;
        atomicAdd(reinterpret_cast<unsigned long long*>(peer_count + qd), 1ull);
      }
    }
  }
}

// admitted ids in ascending global order -> local ids n_loc, n_loc + 1, ... (word bits cleared)
struct AdmWord {
  const uint32_t* bm;
  __device__ __forceinline__ int64_t operator()(int64_t w) const { return __popc(bm[w]); }
};
struct AdmAssign {
  uint32_t* bm;
  rtec_shard_t sh;
  int32_t* adm_list;
  uint64_t* err;
  __device__ __forceinline__ void operator()(int64_t w, int64_t off, int64_t) const {
    uint32_t b = bm[w];
    if (!b) return;
    bm[w] = 0;
    const int64_t base = *sh.n_loc;
    while (b) {
      const int t = __ffs(b) - 1;
      b &= b - 1;
      const int32_t u = static_cast<int32_t>(w * 32 + t);
      const int64_t lid = base + off;
      if (lid >= sh.cap) {  // the host keeps cap >= n_loc + B; never silently overrun
        report_error(err, RTEC_CONFIG_ERROR, 0);
      } else {
        sh.g2l[u] = static_cast<int32_t>(lid);
        sh.l2g[lid] = u;
        adm_list[off] = static_cast<int32_t>(lid);
      }
      ++off;
    }
  }
};
__global__ void k_admit_commit(int64_t* n_loc, const int64_t* n_adm, int64_t cap) {
  RTEC_PDL_ENTRY();
  const int64_t t = *n_loc + *n_adm;
  *n_loc = t < cap ? t : cap;
}

// ------------------------------------------------------------------ local batch
struct OwnedDst {
  const int32_t* dst;
  int32_t rank, world;
  const uint64_t* err;
  __device__ __forceinline__ int64_t operator()(int64_t i) const {
    return (!err_set(err) && owner_of(dst[i], world) == rank) ? 1 : 0;
  }
};
struct Localize {
  OwnedDst f;
  const int32_t* src; const uint8_t* op; const int64_t* ts; const int32_t* g2l;
  int32_t* lsrc; int32_t* ldst; uint8_t* lop; int64_t* lts; int32_t* lpos;
  __device__ __forceinline__ void operator()(int64_t i, int64_t off, int64_t v) const {
    if (!v) return;
    lsrc[off] = g2l[src[i]];
    ldst[off] = g2l[f.dst[i]];
    lop[off] = op[i];
    lts[off] = ts[i];
    lpos[off] = static_cast<int32_t>(i);
  }
};

// ------------------------------------------------------------------ row exchange
// per-peer row counts of a list of owned local ids (each row goes to every rank in peers[v])
__global__ void k_count_peers(rtec_shard_t sh, const int32_t* __restrict__ list, const int64_t* n_list,
                              int64_t max_list, int64_t* peer_count) {
  RTEC_PDL_ENTRY();
  const int64_t n = n_list ? *n_list : max_list;
  for (int64_t i0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~int64_t(31); i0 < n;
       i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + lane_id();
    const uint32_t pm = i < n ? sh.peers[list ? list[i] : i] : 0u;
    for (int q = 0; q < sh.world; ++q) {
      const unsigned c = __popc(__ballot_sync(0xffffffffu, (pm >> q) & 1u));
      if (lane_id() == 0 && c) atomicAdd(reinterpret_cast<unsigned long long*>(peer_count + q), 1ull * c);
    }
  }
}

struct PackSrc {
  const float* m[kShardMaxMats];
  int32_t d[kShardMaxMats];
  int32_t k;
  int32_t width;
  int64_t off[kShardMaxWorld + 1];
};

__device__ __forceinline__ void pack_one(const rtec_shard_t& sh, const PackSrc& ps, int32_t v, int q,
                                         int64_t* cursor, int32_t* out_ids, int32_t* out_deg, float* out_rows) {
  int64_t slot = 0;
  if (lane_id() == 0) slot = ps.off[q] + atomicAdd(reinterpret_cast<unsigned long long*>(cursor + q), 1ull);
  slot = __shfl_sync(0xffffffffu, slot, 0);
  if (lane_id() == 0) {
    out_ids[slot] = sh.l2g[v];
    if (out_deg) out_deg[slot] = sh.gout[v];
  }
  float* o = out_rows + slot * ps.width;
  int c0 = 0;
  for (int j = 0; j < ps.k; ++j) {
    const float* r = ps.m[j] + static_cast<int64_t>(v) * ps.d[j];
    const int d = ps.d[j];
    if ((d & 3) == 0 && (c0 & 3) == 0 && (ps.width & 3) == 0) {
      for (int c = lane_id(); c < d / 4; c += 32)
        reinterpret_cast<float4*>(o + c0)[c] = __ldg(reinterpret_cast<const float4*>(r) + c);
    } else {
      for (int c = lane_id(); c < d; c += 32) o[c0 + c] = __ldg(r + c);
    }
    c0 += d;
  }
}

// list mode: (v, q) for every owned v of the list and every q in peers[v];
// pair mode: the explicit (send_u[k], send_q[k]) pairs of an admission
__global__ void __launch_bounds__(kSBlk) k_pack(rtec_shard_t sh, PackSrc ps, const int32_t* __restrict__ list,
                                                const int64_t* n_list, int64_t max_list,
                                                const int32_t* __restrict__ pair_u, const int32_t* __restrict__ pair_q,
                                                int64_t n_pairs, int64_t* cursor, int32_t* out_ids, int32_t* out_deg,
                                                float* out_rows) {
  RTEC_PDL_ENTRY();
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  if (pair_u) {
    for (int64_t k = warp; k < n_pairs; k += nw) pack_one(sh, ps, pair_u[k], pair_q[k], cursor, out_ids, out_deg, out_rows);
    return;
  }
  const int64_t n = n_list ? *n_list : max_list;
  for (int64_t i = warp; i < n; i += nw) {
    const int32_t v = list ? list[i] : static_cast<int32_t>(i);
    uint32_t pm = sh.peers[v];
    while (pm) {
      const int q = __ffs(pm) - 1;
      pm &= pm - 1;
      pack_one(sh, ps, v, q, cursor, out_ids, out_deg, out_rows);
    }
  }
}

// rows of received (global id, [rows...]) into the ghost rows of every matrix (+ degrees)
__global__ void __launch_bounds__(kSBlk) k_unpack_rows(rtec_shard_t sh, PackSrc ps, const int32_t* __restrict__ ids,
                                                       const int32_t* __restrict__ degs,
                                                       const float* __restrict__ rows, int64_t k, int32_t* out_local) {
  RTEC_PDL_ENTRY();
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < k; i += nw) {
    const int32_t lu = sh.g2l[ids[i]];
    if (lu < 0) continue;  // not local (cannot happen for a coherent peers[] / g2l pair)
    if (lane_id() == 0) {
      if (degs) sh.gout[lu] = sh.gout_prev[lu] = degs[i];
      if (out_local) out_local[i] = lu;
    }
    const float* src = rows + i * ps.width;
    int c0 = 0;
    for (int j = 0; j < ps.k; ++j) {
      float* o = const_cast<float*>(ps.m[j]) + static_cast<int64_t>(lu) * ps.d[j];
      for (int c = lane_id(); c < ps.d[j]; c += 32) o[c] = __ldg(src + c0 + c);
      c0 += ps.d[j];
    }
  }
}

// V_chg(l) of the shard, assembled over one or more exchange rounds: the received ghost
// rows of a round take positions pos_base + [0, k), the owned changed rows (own_list, last
// round) the positions after them.  Per received row either
//   glog mode:  glog[pos] = the overwritten pre-batch ghost row (the next layer retracts with it)
//   delta mode: delta[u] = c_new h_new - c_old h_old, c from the global out-degrees (GCN
//               1/sqrt(deg + off), else 1; 0 without out-edges) -- the next layer's source delta,
//               as the update epilogue writes it for owned rows (no DeltaLog at all)
struct ChgOut {
  float* glog;
  float* delta;
  int32_t coeff_gcn;
  float deg_off;
};

__device__ __forceinline__ float shard_coeff(const ChgOut& o, int32_t deg) {
  return deg > 0 ? (o.coeff_gcn ? 1.0f / sqrtf(static_cast<float>(deg) + o.deg_off) : 1.f) : 0.f;
}

template <bool V4>
__global__ void __launch_bounds__(kSBlk) k_unpack_changed(rtec_shard_t sh, int32_t d, const int32_t* __restrict__ ids,
                                                          const float* __restrict__ rows, int64_t k, int64_t pos_base,
                                                          float* H, const int32_t* __restrict__ own_list,
                                                          const int64_t* n_own, const float* __restrict__ own_log,
                                                          const int32_t* __restrict__ own_slot, ChgOut o,
                                                          uint32_t* bm_chg, int32_t* chg_slot, int32_t* chg_list,
                                                          int64_t* n_chg) {
  RTEC_PDL_ENTRY();
  const int64_t no = own_list ? *n_own : 0;
  const int64_t total = k + no;
  if (blockIdx.x == 0 && threadIdx.x == 0 && own_list) *n_chg = pos_base + total;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t p = warp; p < total; p += nw) {
    const bool recv = p < k;
    const int32_t u = recv ? sh.g2l[ids[p]] : own_list[p - k];
    if (u < 0) continue;
    const int64_t pos = pos_base + p;
    if (lane_id() == 0) {
      atomicOr(bm_chg + (u >> 5), 1u << (u & 31));
      chg_slot[u] = static_cast<int32_t>(pos);
      chg_list[pos] = u;
    }
    float* hrow = H + static_cast<int64_t>(u) * d;
    if (recv) {
      const float* nrow = rows + p * d;
      if (o.delta) {
        const float cn = shard_coeff(o, sh.gout[u]), co = shard_coeff(o, sh.gout_prev[u]);
        float* drow = o.delta + static_cast<int64_t>(u) * d;
        for (int c = lane_id(); c < d; c += 32) {
          const float nv = __ldg(nrow + c), ov = hrow[c];
          drow[c] = cn * nv - co * ov;
          hrow[c] = nv;
        }
      } else if (V4) {
        float* lrow = o.glog + pos * d;
        for (int c = lane_id(); c < d / 4; c += 32) {
          reinterpret_cast<float4*>(lrow)[c] = reinterpret_cast<const float4*>(hrow)[c];
          reinterpret_cast<float4*>(hrow)[c] = __ldg(reinterpret_cast<const float4*>(nrow) + c);
        }
      } else {
        float* lrow = o.glog + pos * d;
        for (int c = lane_id(); c < d; c += 32) {
          lrow[c] = hrow[c];
          hrow[c] = __ldg(nrow + c);
        }
      }
    } else if (!o.delta) {  // owned: the local DeltaLog row (delta mode: the epilogue wrote δ)
      float* lrow = o.glog + pos * d;
      const float* orow = own_log + static_cast<int64_t>(own_slot[u]) * d;
      if (V4) {
        for (int c = lane_id(); c < d / 4; c += 32)
          reinterpret_cast<float4*>(lrow)[c] = __ldg(reinterpret_cast<const float4*>(orow) + c);
      } else {
        for (int c = lane_id(); c < d; c += 32) lrow[c] = __ldg(orow + c);
      }
    }
  }
}

// ------------------------------------------------------------------ global degrees
__global__ void k_gdeg(rtec_shard_t sh, const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                       const uint8_t* __restrict__ op, const uint8_t* __restrict__ gst, int64_t B,
                       uint32_t* bm_touch) {
  RTEC_PDL_ENTRY();
  for (int64_t i0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~int64_t(31); i0 < B;
       i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + lane_id();
    const bool act = i < B && gst[i];
    int32_t s = 0, d = 0;
    if (act) {
      s = src[i];
      d = dst[i];
      const int32_t ls = sh.g2l[s];
      if (ls >= 0) atomicAdd(sh.gout + ls, op[i] == RTEC_OP_INSERT ? 1 : -1);  // graph.py:220-224
    }
    // owned endpoints (local id v / P) of applied updates: DegreeDelta candidates
    const bool os = act && owner_of(s, sh.world) == sh.rank;
    const bool od = act && owner_of(d, sh.world) == sh.rank;
    bm_set_warp(bm_touch, os ? s / sh.world : 0, os);
    bm_set_warp(bm_touch, od ? d / sh.world : 0, od);
  }
}

__global__ void k_gdeg_dg(rtec_shard_t sh, const int32_t* __restrict__ src, const uint8_t* __restrict__ gst, int64_t B,
                          uint32_t* dg_bm) {
  RTEC_PDL_ENTRY();
  for (int64_t i0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~int64_t(31); i0 < B;
       i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + lane_id();
    int32_t ls = -1;
    if (i < B && gst[i]) ls = sh.g2l[src[i]];
    const bool ch = ls >= 0 && sh.gout[ls] != sh.gout_prev[ls];
    bm_set_warp(dg_bm, ch ? ls : 0, ch);
  }
}

// owned touched vertices whose (in, out) degree changed -> DegreeDelta rows, ascending
// (owned local i <-> global rank + P i is monotone)
struct OwnedChanged {
  const uint32_t* touch;
  rtec_shard_t sh;
  const int32_t* in_deg; const int32_t* in_prev;
  __device__ __forceinline__ uint32_t changed(int64_t w) const {
    uint32_t t = touch[w], c = 0;
    while (t) {
      const int b = __ffs(t) - 1;
      t &= t - 1;
      const int64_t v = w * 32 + b;
      if (sh.gout[v] != sh.gout_prev[v] || in_deg[v] != in_prev[v]) c |= 1u << b;
    }
    return c;
  }
  __device__ __forceinline__ int64_t operator()(int64_t w) const { return __popc(changed(w)); }
};
struct OwnedDeltaRows {
  OwnedChanged f;
  int32_t* dv; int32_t* doi; int32_t* dni; int32_t* doo; int32_t* dno;
  __device__ __forceinline__ void operator()(int64_t w, int64_t off, int64_t) const {
    uint32_t c = f.changed(w);
    while (c) {
      const int b = __ffs(c) - 1;
      c &= c - 1;
      const int32_t v = static_cast<int32_t>(w * 32 + b);
      dv[off] = f.sh.rank + f.sh.world * v;
      doi[off] = f.in_prev[v];
      dni[off] = f.in_deg[v];
      doo[off] = f.sh.gout_prev[v];
      dno[off] = f.sh.gout[v];
      ++off;
    }
  }
};

__global__ void k_gdeg_commit(rtec_shard_t sh, const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                              const uint8_t* __restrict__ gst, int64_t B, uint32_t* dg_bm, uint32_t* bm_touch) {
  RTEC_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < B; i += (int64_t)gridDim.x * blockDim.x) {
    if (!gst[i]) continue;
    const int32_t s = src[i], d = dst[i];
    const int32_t ls = sh.g2l[s];
    if (ls >= 0) {
      sh.gout_prev[ls] = sh.gout[ls];
      dg_bm[ls >> 5] = 0;  // every set bit of the word is an applied update's source
    }
    if (owner_of(s, sh.world) == sh.rank) bm_touch[(s / sh.world) >> 5] = 0;
    if (owner_of(d, sh.world) == sh.rank) bm_touch[(d / sh.world) >> 5] = 0;
  }
}

static int shard_ok(const rtec_shard_t* sh) {
  if (!sh || sh->world < 1 || sh->world > kShardMaxWorld || sh->rank < 0 || sh->rank >= sh->world) {
    set_error("shard descriptor: world %d / rank %d out of range", sh ? sh->world : -1, sh ? sh->rank : -1);
    return RTEC_CONFIG_ERROR;
  }
  return RTEC_OK;
}

static int pack_src(PackSrc& ps, int32_t nmat, const float* const* mats, const int32_t* dims, int32_t world,
                    const int64_t* peer_off) {
  if (nmat < 1 || nmat > kShardMaxMats) {
    set_error("shard exchange: %d matrices (1..%d)", nmat, kShardMaxMats);
    return RTEC_CONFIG_ERROR;
  }
  ps = PackSrc{};
  ps.k = nmat;
  ps.width = 0;
  for (int j = 0; j < nmat; ++j) {
    ps.m[j] = mats[j];
    ps.d[j] = dims[j];
    ps.width += dims[j];
  }
  for (int q = 0; peer_off && q <= world; ++q) ps.off[q] = peer_off[q];
  return RTEC_OK;
}

}  // namespace rtec

using namespace rtec;

extern "C" {

int rtec_batch_validate(const int32_t* src, const int32_t* dst, int64_t B, int64_t n, uint64_t* err, void* ws,
                        size_t ws_bytes, rtec_stream_t stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  RTEC_CUDA(cudaMemsetAsync(err, 0xff, sizeof(uint64_t), s));
  if (B <= 0) return RTEC_OK;
  RTEC_PROF("batch_validate", s);
  Ws w(ws, ws_bytes);
  uint64_t* keys = w.alloc<uint64_t>(B);
  uint32_t* vals = w.alloc<uint32_t>(B);
  uint64_t* sk = w.alloc<uint64_t>(B);
  uint32_t* sv = w.alloc<uint32_t>(B);
  RTEC_WS_CHECK(w);
  const int grid = grid_for(B, kSBlk);
  launch(k_val_keys, grid, kSBlk, 0, s, src, dst, B, n, keys, vals, err);
  RTEC_TRY(sort_pairs(keys, vals, sk, sv, Count{nullptr, B}, B, bits_for(static_cast<uint64_t>(n) * n), w, s));
  launch(k_val_dups, grid, kSBlk, 0, s, sk, sv, B, n, err);
  RTEC_LAUNCH_CHECK("batch_validate");
  return RTEC_OK;
}

int rtec_shard_admit(const rtec_shard_t* sh, const int32_t* src, const int32_t* dst, const uint8_t* op, int64_t B,
                     uint64_t* err, uint32_t* bm_adm, int32_t* adm_list, int64_t* n_adm, int32_t* send_u,
                     int32_t* send_q, int64_t* n_send, int64_t* peer_count, void* ws, size_t ws_bytes,
                     rtec_stream_t stream) {
  RTEC_TRY(shard_ok(sh));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  RTEC_CUDA(cudaMemsetAsync(n_adm, 0, sizeof(int64_t), s));
  RTEC_CUDA(cudaMemsetAsync(n_send, 0, sizeof(int64_t), s));
  RTEC_CUDA(cudaMemsetAsync(peer_count, 0, sizeof(int64_t) * sh->world, s));
  if (B <= 0) return RTEC_OK;
  RTEC_PROF("shard_admit", s);
  launch(k_admit, grid_for(B, kSBlk), kSBlk, 0, s, *sh, src, dst, op, B, err, bm_adm, send_u, send_q, n_send, peer_count);
  RTEC_LAUNCH_CHECK("k_admit");
  Ws w(ws, ws_bytes);
  const int64_t words = (sh->n + 31) / 32;
  RTEC_TRY(exclusive_scan(AdmWord{bm_adm}, Count{nullptr, words}, words, AdmAssign{bm_adm, *sh, adm_list, err},
                          n_adm, w, s));
  launch(k_admit_commit, 1, 1, 0, s, sh->n_loc, n_adm, sh->cap);
  RTEC_LAUNCH_CHECK("k_admit_commit");
  return RTEC_OK;
}

int rtec_shard_localize(const rtec_shard_t* sh, const int32_t* src, const int32_t* dst, const uint8_t* op,
                        const int64_t* ts, int64_t B, const uint64_t* err, int32_t* lsrc, int32_t* ldst, uint8_t* lop,
                        int64_t* lts, int32_t* lpos, int64_t* n_local, void* ws, size_t ws_bytes,
                        rtec_stream_t stream) {
  RTEC_TRY(shard_ok(sh));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  RTEC_CUDA(cudaMemsetAsync(n_local, 0, sizeof(int64_t), s));
  if (B <= 0) return RTEC_OK;
  RTEC_PROF("shard_localize", s);
  Ws w(ws, ws_bytes);
  OwnedDst f{dst, sh->rank, sh->world, err};
  return exclusive_scan(f, Count{nullptr, B}, B, Localize{f, src, op, ts, sh->g2l, lsrc, ldst, lop, lts, lpos},
                        n_local, w, s);
}

int rtec_shard_count_peers(const rtec_shard_t* sh, const int32_t* list, const int64_t* n_list, int64_t max_list,
                           int64_t* peer_count, rtec_stream_t stream) {
  RTEC_TRY(shard_ok(sh));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  RTEC_CUDA(cudaMemsetAsync(peer_count, 0, sizeof(int64_t) * sh->world, s));
  if (max_list <= 0) return RTEC_OK;
  launch(k_count_peers, grid_for(max_list, kSBlk, kSMs * 8), kSBlk, 0, s, *sh, list, n_list, max_list, peer_count);
  RTEC_LAUNCH_CHECK("k_count_peers");
  return RTEC_OK;
}

int rtec_shard_pack(const rtec_shard_t* sh, int32_t nmat, const float* const* mats, const int32_t* dims,
                    const int64_t* peer_off, const int32_t* list, const int64_t* n_list, int64_t max_list,
                    const int32_t* pair_u, const int32_t* pair_q, int64_t n_pairs, int64_t* cursor, int32_t* out_ids,
                    int32_t* out_deg, float* out_rows, rtec_stream_t stream) {
  RTEC_TRY(shard_ok(sh));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  PackSrc ps;
  RTEC_TRY(pack_src(ps, nmat, mats, dims, sh->world, peer_off));
  RTEC_CUDA(cudaMemsetAsync(cursor, 0, sizeof(int64_t) * sh->world, s));
  const int64_t work = pair_u ? n_pairs : max_list;
  if (work <= 0) return RTEC_OK;
  RTEC_PROF("shard_pack", s);
  launch(k_pack, grid_for(work * 32, kSBlk, kSMs * 8), kSBlk, 0, s, *sh, ps, list, n_list, max_list, pair_u, pair_q,
                                                                 n_pairs, cursor, out_ids, out_deg, out_rows);
  RTEC_LAUNCH_CHECK("k_pack");
  return RTEC_OK;
}

int rtec_shard_unpack_rows(const rtec_shard_t* sh, int32_t nmat, float* const* mats, const int32_t* dims,
                           const int32_t* ids, const int32_t* degs, const float* rows, int64_t k, int32_t* out_local,
                           rtec_stream_t stream) {
  RTEC_TRY(shard_ok(sh));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  PackSrc ps;
  RTEC_TRY(pack_src(ps, nmat, const_cast<const float* const*>(mats), dims, sh->world, nullptr));
  if (k <= 0) return RTEC_OK;
  RTEC_PROF("shard_unpack", s);
  launch(k_unpack_rows, grid_for(k * 32, kSBlk, kSMs * 8), kSBlk, 0, s, *sh, ps, ids, degs, rows, k, out_local);
  RTEC_LAUNCH_CHECK("k_unpack_rows");
  return RTEC_OK;
}

int rtec_shard_unpack_changed(const rtec_shard_t* sh, int32_t d, const int32_t* ids, const float* rows, int64_t k,
                              int64_t pos_base, int32_t clear, float* H, const int32_t* own_list, const int64_t* n_own,
                              int64_t max_own, const float* own_log, const int32_t* own_slot, float* glog,
                              float* delta, int32_t coeff_gcn, float deg_off, uint32_t* bm_chg, int32_t* chg_slot,
                              int32_t* chg_list, int64_t* n_chg, rtec_stream_t stream) {
  RTEC_TRY(shard_ok(sh));
  if (!glog == !delta) {
    set_error("shard_unpack_changed: exactly one of glog / delta");
    return RTEC_CONFIG_ERROR;
  }
  if (own_list && glog && (!own_log || !own_slot)) {
    set_error("shard_unpack_changed: glog mode needs the owned DeltaLog rows");
    return RTEC_CONFIG_ERROR;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  RTEC_PROF("shard_unpack", s);
  if (clear) RTEC_CUDA(cudaMemsetAsync(bm_chg, 0, sizeof(uint32_t) * ((sh->cap + 31) / 32), s));
  const int64_t work = k + (own_list ? max_own : 0);
  if (work <= 0 && !own_list) return RTEC_OK;
  const int grid = grid_for((work > 0 ? work : 1) * 32, kSBlk, kSMs * 8);
  const ChgOut o{glog, delta, coeff_gcn, deg_off};
  if (d % 4 == 0)
    launch(k_unpack_changed<true>, grid, kSBlk, 0, s, *sh, d, ids, rows, k, pos_base, H, own_list, n_own, own_log, own_slot,
                                                  o, bm_chg, chg_slot, chg_list, n_chg);
  else
    launch(k_unpack_changed<false>, grid, kSBlk, 0, s, *sh, d, ids, rows, k, pos_base, H, own_list, n_own, own_log,
                                                   own_slot, o, bm_chg, chg_slot, chg_list, n_chg);
  RTEC_LAUNCH_CHECK("k_unpack_changed");
  return RTEC_OK;
}

int rtec_shard_degrees(const rtec_shard_t* sh, const int32_t* src, const int32_t* dst, const uint8_t* op,
                       const uint8_t* gstatus, int64_t B, const int32_t* in_deg, const int32_t* in_deg_prev,
                       uint32_t* bm_touch, uint32_t* dg_bm, int32_t* d_vertex, int32_t* d_old_in, int32_t* d_new_in,
                       int32_t* d_old_out, int32_t* d_new_out, int64_t* n_delta, void* ws, size_t ws_bytes,
                       rtec_stream_t stream) {
  RTEC_TRY(shard_ok(sh));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  RTEC_PROF("shard_degrees", s);
  if (B > 0) {
    launch(k_gdeg, grid_for(B, kSBlk), kSBlk, 0, s, *sh, src, dst, op, gstatus, B, bm_touch);
    launch(k_gdeg_dg, grid_for(B, kSBlk), kSBlk, 0, s, *sh, src, gstatus, B, dg_bm);
    RTEC_LAUNCH_CHECK("k_gdeg");
  }
  Ws w(ws, ws_bytes);
  const int64_t words = (sh->n_own + 31) / 32;
  OwnedChanged oc{bm_touch, *sh, in_deg, in_deg_prev};
  return exclusive_scan(oc, Count{nullptr, words}, words,
                        OwnedDeltaRows{oc, d_vertex, d_old_in, d_new_in, d_old_out, d_new_out}, n_delta, w, s);
}

int rtec_shard_commit(const rtec_shard_t* sh, const int32_t* src, const int32_t* dst, const uint8_t* gstatus,
                      int64_t B, uint32_t* dg_bm, uint32_t* bm_touch, rtec_stream_t stream) {
  RTEC_TRY(shard_ok(sh));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (B > 0) launch(k_gdeg_commit, grid_for(B, kSBlk), kSBlk, 0, s, *sh, src, dst, gstatus, B, dg_bm, bm_touch);
  RTEC_LAUNCH_CHECK("k_gdeg_commit");
  return RTEC_OK;
}

}  // extern "C"
